#!/bin/bash
cd /root/repo
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 300 python bench.py --workload fc --steps 20 --warmup 5 > gpurun_out/bench_fc.json 2> gpurun_out/bench_fc.err; echo "fc rc=$?"
timeout 300 python bench.py --workload conv --steps 20 --warmup 5 > gpurun_out/bench_conv.json 2> gpurun_out/bench_conv.err; echo "conv rc=$?"
python - <<'PY'
import json
for w in ("fc", "conv"):
    d = json.loads(open(f"gpurun_out/bench_{w}.json").read().strip().splitlines()[-1])
    print(w, "value", d["value"], d["unit"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], "roof", d["roofline"]["achieved"], d["roofline"]["frac"], d["roofline"]["avg_launch_ms"], d["config"].get("backend"), d["config"].get("step_ms_by_backend"))
PY
