for d in 7 15 9 8; do
  TK_CONV_DBG=$d ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dbg_$d.csv -s 23 -c 12 python tools/prof_net.py > /dev/null 2>&1
  echo "== dbg=$d"; python tools/launches.py gpurun_out/dbg_$d.csv 2>/dev/null | head -10
done
