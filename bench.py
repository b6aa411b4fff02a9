#!/usr/bin/env python
"""Benchmark of the FATNN ternary hot path on B200 (contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload resnet18|resnet50|fc|conv|dot]

Metric (BASELINE.json): "ternary GEMM Tops/s & ResNet-18 img/s vs roofline at
1/2/4/8 B200".  The default workload is ResNet-18 ternary inference at batch
256 per GPU (cfg4; images sharded over GPUs with no collective -> weak
scaling); `--workload fc` measures the cfg3 4096x4096 FC GEMM in Tops/s.

* value   -- units/s with inputs resident in HBM (device CUDA-event time per
             step, L2 flushed between steps, max over ranks).
* e2e     -- the same metric through the public API with host buffers: pinned
             H2D of the step's input and D2H of its result inside the timed
             region.
* roofline-- the dominant kernel's algorithmic work per launch / its average
             launch time (CUDA events on its stream), against the measured
             peak of its pipe (profiles/peaks_r01.json).
* cpu_baseline -- the reference's own CPU implementation (oracle/_ref, the
             unmodified headers) on this host, on a bounded sample.
`--impl reference` times that same reference CPU implementation on all host
threads for the same workload and prints the line with "impl": "reference".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ternary GEMM Tops/s & ResNet-18 img/s vs roofline at 1/2/4/8 B200"
PEAKS_FILE = os.path.join(ROOT, "profiles", "peaks_r01.json")


# ---------------------------------------------------------------------------
# helpers

def load_peaks() -> dict:
    p = {"hbm_gbs": 6549.4, "bf16_tflops": 1637.5, "source": "fallback"}
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        with open(mp) as f:
            p.update(json.load(f))
        p["source"] = "MEASURED_PEAKS.json"
    if os.path.exists(PEAKS_FILE):
        with open(PEAKS_FILE) as f:
            p.update({k: v for k, v in json.load(f).items() if k.endswith(("_tops", "_gbs"))})
    # int8 tensor pipe: measured cuBLASLt int8 GEMM (torch._int_mm) if recorded,
    # else 2x the measured bf16 dense figure (same pipe, twice the rate)
    p.setdefault("i8_tc_tops", 2 * p["bf16_tflops"])
    # LOP3+POPC pipe: 16 POPC/clk/SM measured (tools/pipe_bench.cu), 32 ops/POPC
    p.setdefault("popc_tops", 148 * 16 * 32 * p.get("sm_max_mhz", 1965.0) * 1e6 / 1e12)
    return p


class ClockSampler:
    """nvidia-smi sampling during the timed region (clocks + throttle reasons)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self) -> dict:
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 3 + i and r[3 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def dist_setup(n_gpus: int):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class L2Flush:
    """Writes a buffer larger than the 126 MB L2 between timed steps."""

    def __init__(self):
        import torch
        self.buf = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device="cuda")

    def __call__(self):
        self.buf.fill_(1.0)


# ---------------------------------------------------------------------------
# workloads (ours)

class FcWorkload:
    """cfg3: ternary FC 4096x4096, batch 256: quantize+pack -> GEMM -> folded BN."""

    name = "fc"

    def __init__(self, batch=256, cin=4096, cout=4096, seed=0):
        import numpy as np
        import torch
        from paper_2008_05101_b200 import ternkit as tk
        self.tk = tk
        rng = np.random.default_rng(seed)
        self.B, self.C, self.N = batch, cin, cout
        self.wq = rng.integers(-1, 2, (cout, cin)).astype(np.int8)
        gain = (rng.uniform(0.5, 1.5, cout) / 64).astype(np.float32)
        bias = rng.standard_normal(cout).astype(np.float32)
        self.layer = tk.make_packed_conv_layer(self.wq, tk.ConvGeometry(cin, cout, 1, 1, 1, 0),
                                               tk.QuantThresholds(), tk.QuantThresholds(0.5, 0.9), True,
                                               tk.ChannelAffine(gain, bias))
        self.x_host = np.abs(rng.standard_normal((batch, cin))).astype(np.float32)
        self.x = torch.from_numpy(self.x_host).cuda()
        self.x_pin = torch.from_numpy(self.x_host).pin_memory()
        self.y_pin = torch.empty((batch, cout), dtype=torch.float32).pin_memory()
        self.x_dev2 = torch.empty_like(self.x)
        self.units_per_step = 2.0 * batch * cin * cout / 1e12  # Tera-ops
        self.unit = "Tops/s"
        self.launches_per_step = 2
        self.config = {"workload": "cfg3 ternary FC 4096x4096 batch 256 (quantize+pack -> GEMM -> folded BN)",
                       "batch": batch, "in": cin, "out": cout, "backend": "auto",
                       "l2": "flushed between steps (256 MB write)"}

    def step(self):
        return self.tk.fully_connected_ternary(self.x, self.B, self.layer, check_errors=False)

    def step_e2e(self):
        self.x_dev2.copy_(self.x_pin, non_blocking=True)
        y = self.tk.fully_connected_ternary(self.x_dev2, self.B, self.layer, check_errors=False)
        self.y_pin.copy_(y, non_blocking=True)
        return y

    def e2e_bytes(self):
        return self.x_host.nbytes, self.B * self.N * 4

    def dominant(self):
        """(description, algorithmic work per launch, unit, bound, launcher)."""
        tk = self.tk
        layer = self.layer
        be = layer.backend_for(self.B)
        rows = tk.quantize_and_pack_rows(self.x, tk.QuantThresholds(0.5, 0.9), tk.QuantMode.kActivationNonneg)
        buf = tk.Im2colBuffer(rows, rows.shape[1], self.B, self.C, True, self.B, 1, 1)
        flops = 2.0 * self.B * self.C * self.N
        return (f"ternary GEMM ({be.name})", flops / 1e12, "TFLOP/s", "tensor" if be == tk.Backend.TC_I8 else "int",
                lambda: tk.packed_gemm(buf, layer), be)

    def verify(self):
        import numpy as np
        from oracle.oracle import Oracle
        O = Oracle()
        y = self.step().cpu().numpy()
        xs = np.ascontiguousarray(self.x_host[:4])
        st, ref = O.conv2d_ternary(xs, 4, self.C, 1, 1, self.wq, self.N, 1, 1, 0, (0.5, 0.9), True,
                                   self.layer.fused.gain, self.layer.fused.bias, 1.0)
        return st == 0 and np.array_equal(y[:4].view(np.int32), ref.reshape(4, self.N).view(np.int32))

    def cpu_baseline(self, threads: int) -> dict:
        """The reference (oracle/_ref) on a bounded sample: im2col_quantize_pack +
        packed_gemm with the reference's worker threads."""
        import ctypes as C
        import numpy as np
        from oracle.oracle import Reference, ptr, _f32p, _i8p
        R = Reference()
        rows = 64
        xs = np.ascontiguousarray(self.x_host[:rows])
        sec = C.c_double()
        st = R.lib.ref_time_fc_gemm(ptr(xs, _f32p), rows, self.C, ptr(self.wq, _i8p), self.N, 0.5, 0.9,
                                    threads, 1, C.byref(sec), None)
        assert st == 0
        t = sec.value
        return {"value": 2.0 * rows * self.C * self.N / t / 1e12, "unit": self.unit, "cores": threads,
                "kind": "reference", "sample": f"{rows} of {self.B} rows, 1 call (rows are independent)",
                "seconds": t}


def build_workload(name: str):
    if name == "fc":
        return FcWorkload()
    if name in ("resnet18", "resnet50"):
        from paper_2008_05101_b200.resnet import ResNetWorkload
        return ResNetWorkload(name)
    raise SystemExit(f"unknown workload {name}")


def time_dominant(w, iters: int = 20) -> tuple[float, str, float, str, str]:
    import torch
    desc, work, unit, bound, fn, be = w.dominant()
    for _ in range(3):
        fn()
    flush = L2Flush()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot = 0.0
    for _ in range(iters):
        flush()
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / iters, desc, work, unit, bound


def run_ours(args) -> None:
    import torch
    rank, world, local = dist_setup(args.gpus)
    w = build_workload(args.workload)
    assert w.verify(), "parity check failed before timing"
    flush = L2Flush()
    stream = torch.cuda.current_stream()
    # ---- device-resident timing ----
    for _ in range(args.warmup):
        w.step()
    torch.cuda.synchronize()
    barrier(world)
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier(world)
        for i in range(args.steps):
            flush()
            e0[i].record(stream)
            w.step()
            e1[i].record(stream)
        torch.cuda.synchronize()
    barrier(world)
    ms = sum(a.elapsed_time(b) for a, b in zip(e0, e1)) / args.steps
    ms = max_over_ranks(ms, world)
    value = w.units_per_step * world / (ms / 1e3)
    # ---- end to end through the public API with host buffers ----
    for _ in range(max(1, args.warmup)):
        w.step_e2e()
    torch.cuda.synchronize()
    barrier(world)
    ee0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ee1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for i in range(args.steps):
        flush()
        ee0[i].record(stream)
        w.step_e2e()
        ee1[i].record(stream)
    torch.cuda.synchronize()
    ems = max_over_ranks(sum(a.elapsed_time(b) for a, b in zip(ee0, ee1)) / args.steps, world)
    e2e_value = w.units_per_step * world / (ems / 1e3)
    # ---- roofline of the dominant kernel ----
    dms, desc, work, unit, bound = time_dominant(w)
    peaks = load_peaks()
    if bound == "tensor":
        peak, psrc = peaks["i8_tc_tops"], "measured int8 tensor GEMM (profiles/peaks_r01.json)"
    elif bound == "int":
        peak, psrc = peaks["popc_tops"], "measured POPC pipe x 32 ops (tools/pipe_bench.cu)"
    else:
        peak, psrc = peaks["hbm_gbs"], "MEASURED_PEAKS.json hbm_gbs"
    achieved = work / (dms / 1e3)
    roof = {"kernel": desc, "bound": "tensor" if bound == "tensor" else ("int" if bound == "int" else "hbm"),
            "achieved": round(achieved, 3), "peak": round(peak, 2), "unit": unit,
            "frac": round(achieved / peak, 4), "traffic": getattr(w, "traffic", None),
            "peak_source": psrc, "avg_launch_ms": round(dms, 5)}
    line = {"metric": METRIC, "value": round(value, 3), "unit": w.unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int8/2-bit ternary",
            "data": "synthetic (numpy seeded inputs, random ternary weights)", "config": w.config,
            "e2e": {"value": round(e2e_value, 3), "unit": w.unit, "ms_per_step": round(ems, 5),
                    "h2d_bytes_per_step": w.e2e_bytes()[0], "d2h_bytes_per_step": w.e2e_bytes()[1]},
            "gpu_launches": w.launches_per_step * args.steps, "roofline": roof,
            "clocks": clk.summary()}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = w.cpu_baseline(os.cpu_count() or 1)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.oracle import reference_lib_path
    if reference_lib_path() is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built for this host"}))
        return
    threads = os.cpu_count() or 1
    if args.workload == "fc":
        import numpy as np
        rng = np.random.default_rng(0)
        w = FcWorkload.__new__(FcWorkload)
        w.B, w.C, w.N = 256, 4096, 4096
        w.wq = rng.integers(-1, 2, (w.N, w.C)).astype(np.int8)
        rng.uniform(0.5, 1.5, w.N); rng.standard_normal(w.N)
        w.x_host = np.abs(rng.standard_normal((w.B, w.C))).astype(np.float32)
        w.unit = "Tops/s"
        w.config = {"workload": "cfg3 ternary FC 4096x4096 batch 256", "batch": 256, "in": 4096, "out": 4096}
        vals = []
        for i in range(args.warmup + args.steps):
            cb = w.cpu_baseline(threads)
            if i >= args.warmup:
                vals.append(cb["value"])
        v = statistics.mean(vals)
        cb["value"] = v
        line = {"metric": METRIC, "impl": "reference", "value": round(v, 5), "unit": w.unit, "n_gpus": 0,
                "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "config": w.config,
                "cpu_baseline": cb, "e2e": {"value": round(v, 5), "unit": w.unit, "h2d_bytes_per_step": 0,
                                            "d2h_bytes_per_step": 0}}
    else:
        from paper_2008_05101_b200.resnet import reference_cpu_run
        line = reference_cpu_run(args, METRIC, threads)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=os.environ.get("TK_BENCH_WORKLOAD", "resnet18"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
