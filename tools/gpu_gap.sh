#!/bin/bash
cd /root/repo
for cfg in "128 2" "256 4"; do set -- $cfg
echo "== fp4 BN=$1 S=$2"; FMT=fp4 TK_GEMM_BN=$1 TK_GEMM_SPLIT=$2 timeout 120 python tools/gemm_stamps.py 2>&1 | grep -E "reduction|cluster_bar"; done
