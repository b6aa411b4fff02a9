#!/bin/bash
cd /root/repo
TK_GEMM_MC=4 timeout 900 python -m pytest tests/test_gpu_linalg.py -x -q 2>&1 | tail -3
TK_GEMM_MC=2 timeout 900 python -m pytest tests/test_gpu_linalg.py -x -q -k "level_operand or fc_" 2>&1 | tail -3
for BK in TC_F4 TC_I8; do
  for cfg in "64 1 1" "64 1 2" "64 1 4" "128 1 1" "128 1 2" "128 1 4"; do set -- $cfg
    echo -n "$BK BN=$1 S=$2 MC=$3: "; TK_GEMM_MC=$3 BACKEND=$BK TK_GEMM_BN=$1 TK_GEMM_SPLIT=$2 timeout 120 python tools/prof_fc.py 2>&1 | grep -E "gemm|Error|mismatch" | tr '\n' ' '; echo
  done
done
for MC in 1 2 4; do echo "== fp4 BN=64 S=1 MC=$MC"; TK_GEMM_MC=$MC FMT=fp4 TK_GEMM_BN=64 TK_GEMM_SPLIT=1 timeout 120 python tools/gemm_stamps.py 2>&1 | tail -7; done
