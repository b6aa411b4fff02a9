#!/bin/bash
cd /root/repo
BACKEND=TC_F4 TK_GEMM_BN=128 TK_GEMM_SPLIT=2 timeout 120 python tools/prof_fc.py || exit 1
BACKEND=TC_F4 TK_GEMM_BN=128 TK_GEMM_SPLIT=2 timeout 600 ncu --section WarpStateStats --section SourceCounters --warp-sampling-interval 0 --import-source on --clock-control none -k regex:k_gemm_tc -s 3 -c 1 -o gpurun_out/gemm_f4_128_2 python tools/prof_fc.py > gpurun_out/ncu_gemm.log 2>&1
tail -3 gpurun_out/ncu_gemm.log
