#!/bin/bash
# cfg3 GEMM phase study: per-phase stamps and timing with phases disabled
cd /root/repo
for F in s8 fp4; do
  echo "== stamps $F"; FMT=$F timeout 120 python tools/gemm_stamps.py 2>&1 | tail -9
done
for BK in TC_I8 TC_F4; do
  for D in 0 1 2 3 4 8 12 15; do
    echo -n "$BK dbg=$D: "; BACKEND=$BK TK_GEMM_DBG=$D timeout 120 python tools/prof_fc.py 2>&1 | grep gemm
  done
done
