#!/bin/bash
# quick iteration: build, net parity tests, per-conv probe
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_net.py -x -q 2>&1 | tail -3
for hs in ${HS_LIST:-8}; do
  echo "== HS cap $hs"; TK_CONV_HS=$hs DEPTH=${DEPTH:-18} B=${B:-256} MODES=${MODES:-0,4} timeout 300 python tools/conv_probe.py 2>&1 | tail -${TAILN:-22}
done
