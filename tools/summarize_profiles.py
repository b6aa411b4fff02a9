"""Turn the raw outputs of tools/profile_round.sh (gpurun_out/prof/) into the
tracked summaries under profiles/:

* bench_r02_<workload>.json      -- the bench line of each workload
* ncu_launches_r02_resnet18.{csv,txt} -- launch list of the default bench command
* traffic_r02.json               -- DRAM bytes per launch of each dominant kernel
* ncu_full_r02_<name>.txt        -- key metrics of each `ncu --set full` capture

Run here (ncu -i reads the .ncu-rep files without a GPU)."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RAW = os.path.join(ROOT, "gpurun_out", "prof")
OUT = os.path.join(ROOT, "profiles")
TRAFFIC_SRC = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (tools/profile_round.sh), "
               "cold caches")


def ncu_rows(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    if not rows:
        return []
    hdr = rows[0]
    return [dict(zip(hdr, r)) for r in rows[1:]]


def per_launch(path):
    """{launch id: {"kernel": name, metric: value}} from an ncu --metrics csv."""
    out = {}
    for r in ncu_rows(path):
        d = out.setdefault(r["ID"], {"kernel": r["Kernel Name"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return [out[k] for k in sorted(out, key=int)]


def bench_lines():
    for w in ("resnet18", "resnet50", "fc", "dot", "conv"):
        p = os.path.join(RAW, f"bench_{w}.json")
        if not os.path.exists(p):
            continue
        lines = [ln for ln in open(p).read().splitlines() if ln.startswith("{")]
        if lines:
            with open(os.path.join(OUT, f"bench_r02_{w}.json"), "w") as f:
                f.write(lines[-1] + "\n")
        p = os.path.join(RAW, f"ref_{w}.json")
        lines = [ln for ln in open(p).read().splitlines() if ln.startswith("{")] if os.path.exists(p) else []
        if lines:
            with open(os.path.join(OUT, f"bench_r02_reference_{w}.json"), "w") as f:
                f.write(lines[-1] + "\n")
            print("bench", w, json.loads(lines[-1])["value"])


def launches():
    p = os.path.join(RAW, "launches_resnet18.csv")
    if not os.path.exists(p):
        return
    ls = per_launch(p)
    with open(os.path.join(OUT, "ncu_launches_r02_resnet18.csv"), "w") as f:
        f.write(open(p).read())
    with open(os.path.join(OUT, "ncu_launches_r02_resnet18.txt"), "w") as f:
        f.write("ncu --metrics gpu__time_duration.sum --clock-control none: python bench.py --steps 3 --warmup 3\n")
        f.write("(serialised, cold-cache per-launch times; shares, not absolutes, compare with the bench)\n\n")
        tot = {}
        for d in ls:
            us = d.get("gpu__time_duration.sum", 0.0) / 1e3
            name = d["kernel"]
            short = name.split("(")[0]
            tot[short] = tot.get(short, 0.0) + us
            f.write(f"{us:9.1f} us  {name[:90]}\n")
        f.write("\nper kernel (sum over the run):\n")
        grand = sum(tot.values())
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            f.write(f"{v:10.1f} us  {100 * v / grand:5.1f}%  {k}\n")
    print("launch list:", len(ls), "launches")


def traffic():
    path = os.path.join(OUT, "traffic_r02.json")
    old = {}
    specs = {"resnet18": 256, "resnet50": 128, "fc": None, "dot": None}
    for w, batch in specs.items():
        p = os.path.join(RAW, f"traffic_{w}.csv")
        if not os.path.exists(p):
            continue
        ls = per_launch(p)
        if not ls:
            continue
        b = [d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in ls]
        ms = [d.get("gpu__time_duration.sum", 0) / 1e6 for d in ls]
        old[w] = {"bytes_per_launch": sum(b) / len(b), "launches": len(ls),
                  "kernel": ls[0]["kernel"].split("(")[0], "ncu_ms_per_launch": sum(ms) / len(ms),
                  "per_launch_bytes": b if len(b) > 1 else None, "source": TRAFFIC_SRC, "batch": batch}
        print("traffic", w, f"{sum(b) / len(b) / 1e6:.1f} MB/launch over {len(ls)} launches")
    with open(path, "w") as f:
        json.dump(old, f, indent=1)


KEYS = ("Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L2 Cache Throughput",
        "L1/TEX Cache Throughput", "Issue Slots Busy", "Executed Ipc Active", "Registers Per Thread",
        "Achieved Occupancy", "Dynamic Shared Memory Per Block", "L2 Hit Rate", "Mem Busy", "Max Bandwidth",
        "DRAM Frequency", "SM Frequency", "Grid Size", "Block Size", "Cluster Size")


def full(name, rep, note):
    p = os.path.join(RAW, rep)
    if not os.path.exists(p):
        return
    txt = subprocess.run(["ncu", "-i", p, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    if not rows:
        return
    hdr = rows[0]
    ik, isec, iname, iunit, ival = (hdr.index(h) for h in ("Kernel Name", "Section Name", "Metric Name",
                                                             "Metric Unit", "Metric Value"))
    raw = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,"
                          "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,"
                          "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active,"
                          "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,"
                          "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"],
                         capture_output=True, text=True).stdout
    with open(os.path.join(OUT, f"ncu_full_r02_{name}.txt"), "w") as f:
        f.write(note + "\n\n")
        f.write(f"kernel: {rows[1][ik]}\n")
        seen = set()
        for r in rows[1:]:
            if len(r) <= ival or r[iname] not in KEYS or (r[isec], r[iname]) in seen:
                continue
            seen.add((r[isec], r[iname]))
            f.write(f"{r[isec][:28]:28s} {r[iname]:34s} {r[ival]:>14s} {r[iunit]}\n")
        rr = list(csv.reader(raw.splitlines()))
        if len(rr) >= 3:
            f.write("\nraw:\n")
            for h, u, v in zip(rr[0], rr[1], rr[2]):
                if "__" in h:
                    f.write(f"  {h:70s} {v:>16s} {u}\n")
    print("full capture summarised:", name)


def main():
    if not os.path.isdir(RAW):
        sys.exit(f"no {RAW}")
    bench_lines()
    launches()
    traffic()
    full("r18_conv1", "full_r18_conv1.ncu-rep",
         "ncu --set full --clock-control none -k regex:k_conv_tc -s 1 -c 1 python tools/prof_net.py\n"
         "(ResNet-18 b256, second conv launch = stage-1 block-0 conv2: 3x3 64->64, f32 skip add (x, NCHW), f32 (channel-blocked) + s8 out)")
    full("fc_gemm", "full_fc_gemm.ncu-rep",
         "BACKEND=TC_F4 ncu --set full --clock-control none -k regex:k_gemm_tc -s 2 -c 1 python tools/prof_fc.py\n"
         "(cfg3 FC 4096x4096 b256, FP4 pipe, int32 out, tile chosen by the launcher; ncu flushes caches)")
    full("stem", "full_stem.ncu-rep",
         "ncu --set full --clock-control none -k regex:k_stem_tc -s 3 -c 1 python tools/prof_stem.py\n"
         "(ResNet stem 7x7/2 3->64, 256 x 224x224 images, split-TF32 tcgen05 kind::tf32: 84 MMAs 128x64x8 "
         "per 128-position tile; the kernel is bound by the MMAs' shared-memory operand reads)")


if __name__ == "__main__":
    main()
