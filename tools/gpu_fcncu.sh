#!/bin/bash
cd /root/repo
run() {  # label, env...
  local label=$1; shift
  env "$@" timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,smsp__cycles_active.avg --clock-control none -k regex:k_gemm_tc -c 12 --csv python tools/prof_fc.py > gpurun_out/ncu_$label.csv 2>/dev/null
  python - "$label" <<'PY'
import csv, sys, io
label = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/ncu_{label}.csv")) if len(r) > 10]
hdr = rows[0]; i_name = hdr.index("Metric Name"); i_val = hdr.index("Metric Value")
vals = {}
for r in rows[1:]:
    vals.setdefault(r[i_name], []).append(float(r[i_val].replace(",", "")))
print(label, {k: round(sum(v[3:]) / len(v[3:]), 1) for k, v in vals.items()})
PY
}
run i8_256_4 BACKEND=TC_I8
run i8_256_4_dbg15 BACKEND=TC_I8 TK_GEMM_DBG=15
run f4_64_1 BACKEND=TC_F4 TK_GEMM_BN=64 TK_GEMM_SPLIT=1
run f4_64_1_dbg15 BACKEND=TC_F4 TK_GEMM_BN=64 TK_GEMM_SPLIT=1 TK_GEMM_DBG=15
run f4_128_2 BACKEND=TC_F4 TK_GEMM_BN=128 TK_GEMM_SPLIT=2
