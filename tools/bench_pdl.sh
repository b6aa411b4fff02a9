#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
python -m pytest tests/test_gpu_net.py -q -x 2>&1 | tail -1
for v in pdl nopdl pdl; do
  if [ $v = pdl ]; then export TK_PDL=1; else unset TK_PDL; fi
  python bench.py --workload ${W:-resnet18} --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/b_$v.json
  python - $v <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/b_{sys.argv[1]}.json").read())
print(sys.argv[1], d["value"], d["ms_per_step"], d["roofline"]["frac"])
PY
done
