#!/bin/bash
# Round profiling (run under gpurun from the repo root): bench lines for every
# workload and the reference arm, the ncu launch list of the default bench
# command, DRAM traffic per launch of each workload's dominant kernel, and one
# full-set capture of the top ResNet-18 conv.  Outputs: gpurun_out/prof/
set -x
mkdir -p gpurun_out/prof
for w in resnet18 resnet50 fc dot conv; do
  timeout -s KILL 900 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/prof/bench_$w.json 2> gpurun_out/prof/bench_$w.err
  timeout -s KILL 900 python bench.py --workload $w --impl reference --steps 5 --warmup 3 > gpurun_out/prof/ref_$w.json 2> gpurun_out/prof/ref_$w.err
done
# launch list of the default bench command (kernel durations, serialised: compare shares)
timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/prof/plain.log 2>&1 &&
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/prof/launches_resnet18.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
  > /dev/null 2>&1
# DRAM traffic of the dominant kernels (cold caches as ncu replays them)
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout -s KILL 300 python tools/prof_net.py > /dev/null 2>&1 &&
timeout -s KILL 900 ncu --metrics $M --clock-control none --csv -k regex:k_conv_tc -c 19 \
  --log-file gpurun_out/prof/traffic_resnet18.csv python tools/prof_net.py > /dev/null 2>&1
DEPTH=50 B=128 timeout -s KILL 300 python tools/prof_net.py > /dev/null 2>&1 &&
DEPTH=50 B=128 timeout -s KILL 900 ncu --metrics $M --clock-control none --csv -k regex:k_conv_tc -c 52 \
  --log-file gpurun_out/prof/traffic_resnet50.csv python tools/prof_net.py > /dev/null 2>&1
BACKEND=TC_F4 timeout -s KILL 300 python tools/prof_fc.py > /dev/null 2>&1 &&
BACKEND=TC_F4 timeout -s KILL 600 ncu --metrics $M --clock-control none --csv -k regex:k_gemm_tc -c 1 \
  --log-file gpurun_out/prof/traffic_fc.csv python tools/prof_fc.py > /dev/null 2>&1
timeout -s KILL 600 ncu --metrics $M --clock-control none --csv -k regex:k_dot -c 1 \
  --log-file gpurun_out/prof/traffic_dot.csv python bench.py --workload dot --steps 3 --warmup 3 \
  --no-cpu-baseline > /dev/null 2>&1
# one full-set capture of the top ResNet-18 conv (stage-1 block-0 conv2: f32 skip x + f32 out)
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_conv_tc -s 1 -c 1 \
  -o gpurun_out/prof/full_r18_conv1 python tools/prof_net.py > gpurun_out/prof/full.log 2>&1
# and of the cfg3 FC GEMM (FP4 pipe, bench tile choice)
BACKEND=TC_F4 timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:k_gemm_tc -s 2 -c 1 \
  -o gpurun_out/prof/full_fc_gemm python tools/prof_fc.py > gpurun_out/prof/full_fc.log 2>&1
# and of the split-TF32 stem conv (256 images)
timeout -s KILL 300 python tools/prof_stem.py > /dev/null 2>&1 &&
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:k_stem_tc -s 3 -c 1 \
  -o gpurun_out/prof/full_stem python tools/prof_stem.py > gpurun_out/prof/full_stem.log 2>&1
ls -la gpurun_out/prof
