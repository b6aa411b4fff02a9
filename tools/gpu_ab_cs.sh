#!/bin/bash
cd /root/repo
for V in base cs base cs; do
  echo -n "== $V: "
  TK_LIB_PATH=tools/lib_ab_$V.so MODES=0 REPS=5 timeout 600 python tools/conv_probe.py 2>&1 | tail -21 | awk '$1==1||$1==3||$1==6||$1==8||$1==11||$1==13||$1==16||$1==18||/sum/' | awk '{printf "%s ", $NF} END {print ""}'
done
