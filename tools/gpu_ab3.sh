#!/bin/bash
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_net.py -x -q 2>&1 | tail -1
for V in pre new2 pre new2; do
  echo "== $V"
  TK_LIB_PATH=tools/lib_ab_$V.so MODES=0 REPS=5 timeout 600 python tools/conv_probe.py 2>&1 | tail -21 | awk '$1==1||$1==3||$1==4||$1==6||$1==8||$1==11||$1==13||$1==16||/sum/' | tr '\n' ' '; echo
done
for V in pre new2; do
  TK_LIB_PATH=tools/lib_ab_$V.so timeout 900 python bench.py --workload resnet50 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$V r50', d['value'], d['ms_per_step'])"
done
