#!/bin/bash
cd /root/repo
for D in 0 64; do
echo "== fp4 BN=64 S=1 dbg $D"; DBG=$D FMT=fp4 TK_GEMM_BN=64 TK_GEMM_SPLIT=1 timeout 120 python tools/gemm_stamps.py 2>&1 | tail -10
echo "== s8 BN=256 S=4 dbg $D"; DBG=$D FMT=s8 timeout 120 python tools/gemm_stamps.py 2>&1 | tail -10
done
