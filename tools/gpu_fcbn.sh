#!/bin/bash
cd /root/repo
for BK in TC_I8 TC_F4; do
  for BN in 64 128 256; do
    for S in 1 2 4; do
      echo -n "$BK BN=$BN S=$S: "; BACKEND=$BK TK_GEMM_BN=$BN TK_GEMM_SPLIT=$S timeout 120 python tools/prof_fc.py 2>&1 | grep -E "gemm|Error|mismatch" | tr '\n' ' '; echo
    done
  done
done
