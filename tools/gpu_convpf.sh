#!/bin/bash
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_net.py -x -q 2>&1 | tail -1
MODES=0 REPS=9 timeout 600 python tools/conv_probe.py 2>&1 | tail -21
