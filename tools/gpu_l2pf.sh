#!/bin/bash
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_net.py -x -q 2>&1 | tail -1
MODES=2048,0,2048,0 REPS=5 timeout 900 python tools/conv_probe.py 2>&1 | tail -21
for D in 2048 0; do TK_CONV_DBG=$D timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dbg $D r18', d['value'], d['ms_per_step'])"; done
