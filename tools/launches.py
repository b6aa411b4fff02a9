"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
i_name, i_val = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot = 0.0
for r in rows[1:]:
    v = float(r[i_val].replace(",", "")) / 1000
    tot += v
    print(f"{v:9.1f} us  {r[i_name].replace('(anonymous namespace)::', '')[:60]}")
print(f"total {tot:.1f} us over {len(rows) - 1} launches")
