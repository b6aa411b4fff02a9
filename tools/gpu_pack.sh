#!/bin/bash
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_net.py -x -q 2>&1 | tail -1
for O in 1 "" 1 ""; do
  if [ -n "$O" ]; then export TK_PACK_INPUT_OLD=1; else unset TK_PACK_INPUT_OLD; fi
  echo -n "old=$O: "; timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('r18', d['value'], d['ms_per_step'])"
done
