#!/bin/bash
cd /root/repo
for V in kd2 kd4 kd2b; do
  echo "== $V"
  TK_LIB_PATH=tools/lib_ab_$V.so BACKEND=TC_F4 timeout 120 python tools/prof_fc.py 2>&1 | grep -E "gemm|mismatch|Error"
  TK_LIB_PATH=tools/lib_ab_$V.so timeout 300 python tools/fc_cold_sweep.py 2>&1 | grep "cold"
done
TK_LIB_PATH=tools/lib_ab_kd2.so timeout 600 python -m pytest tests/test_gpu_linalg.py -x -q 2>&1 | tail -1
