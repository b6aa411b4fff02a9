#!/bin/bash
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_net.py -x -q 2>&1 | tail -1
MODES=0 REPS=7 timeout 600 python tools/conv_probe.py 2>&1 | tail -21
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('r18', d['value'], d['ms_per_step'], d['e2e']['value'])"
timeout 900 python bench.py --workload resnet50 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('r50', d['value'], d['ms_per_step'], d['e2e']['value'])"
