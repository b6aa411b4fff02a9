#!/bin/bash
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_linalg.py -x -q 2>&1 | tail -3
for cfg in "64 1" "128 2" "256 4"; do set -- $cfg
for FU in "" 1; do
echo "== fp4 BN=$1 S=$2 fused=$FU"; FUSED=$FU GRAPHS=1 FMT=fp4 TK_GEMM_BN=$1 TK_GEMM_SPLIT=$2 timeout 120 python tools/gemm_stamps.py 2>&1 | grep -E "graph of 20|launch 4|reduction|mma_issued|slices_out|cluster_bar|end "; done; done
