#!/bin/bash
cd /root/repo
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
mkdir -p gpurun_out/prof
for w in resnet18 resnet50 fc dot conv; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/prof/bench_$w.json 2> gpurun_out/prof/bench_$w.err; echo "$w rc=$?"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>/dev/null | tail -1 > gpurun_out/prof/bench_reference_resnet18.json; echo "ref rc=$?"
head -c 600 gpurun_out/prof/bench_reference_resnet18.json
