#!/bin/bash
cd /root/repo
timeout 300 python -m pytest tests/test_gpu_net.py -x -q > gpurun_out/pt.txt 2>&1; tail -1 gpurun_out/pt.txt
for A in 0 1 0 1; do
  echo -n "skip_tma=$A: "
  TK_CONV_SKIP_TMA=$A MODES=0 REPS=5 timeout 300 python tools/conv_probe.py 2>&1 | tail -21 | awk '$1==1||$1==3||$1==6||$1==8||$1==11||$1==13||$1==16||$1==18{printf "%s ", $3} /sum/{print "sum", $2}'
done
