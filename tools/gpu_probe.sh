#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_microbench tools/tc_microbench.cu && timeout 120 tools/tc_microbench > gpurun_out/tc_micro.txt 2>&1
DEPTH=18 B=256 timeout 300 python tools/conv_probe.py > gpurun_out/probe18.txt 2>&1
python tools/prof_net.py > gpurun_out/profnet18.txt 2>&1
DEPTH=50 B=256 MODES=0,1,4,5 timeout 300 python tools/conv_probe.py > gpurun_out/probe50.txt 2>&1
cat gpurun_out/tc_micro.txt gpurun_out/probe18.txt gpurun_out/profnet18.txt gpurun_out/probe50.txt
