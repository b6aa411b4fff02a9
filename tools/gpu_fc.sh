#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_codec.py -x -q 2>&1 | tail -3
timeout 300 python bench.py --workload fc --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_fc.json 2> gpurun_out/bench_fc.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_fc.json').read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"], "roofline", d["roofline"]["achieved"], d["roofline"]["frac"], d["roofline"]["avg_launch_ms"])
PY
for S in 1 2 4 8; do TK_GEMM_SPLIT=$S timeout 120 python tools/prof_fc.py 2>&1 | tail -1; done
