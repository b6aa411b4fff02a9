#!/bin/bash
# FP4 GEMM bring-up: parity tests, then s8 vs fp4 cfg3 timing per split
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_linalg.py -x -q 2>&1 | tail -15
for BK in TC_I8 TC_F4; do
  BACKEND=$BK timeout 120 python tools/prof_fc.py 2>&1 | tail -2
  for S in 1 2 4 8; do BACKEND=$BK TK_GEMM_SPLIT=$S timeout 120 python tools/prof_fc.py 2>&1 | tail -1; done
done
for BN in 64 128; do BACKEND=TC_F4 TK_GEMM_BN=$BN timeout 120 python tools/prof_fc.py 2>&1 | tail -1; done
