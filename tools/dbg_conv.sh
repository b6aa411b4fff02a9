# per-conv device times of the ResNet-18 body under TK_CONV_DBG variants
for d in 0 1 2 4 7; do
  TK_CONV_DBG=$d ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dbg_$d.csv -s 23 -c 21 python tools/prof_net.py > /dev/null 2>&1
  echo "== dbg=$d"; python tools/launches.py gpurun_out/dbg_$d.csv | head -8
done
