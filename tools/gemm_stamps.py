"""Phase timeline of the tensor-core GEMM (cfg3 shape) from in-kernel
globaltimer stamps (env TK_GEMM_DBG |= 16)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _profile  # noqa: E402,F401  (the -DTK_PROFILE build: experiment knobs)
os.environ["TK_GEMM_DBG"] = str(16 | int(os.environ.get("DBG", "0")))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2008_05101_b200 import _lib, ternkit as tk  # noqa: E402


def main():
    B, N = int(os.environ.get("B", 256)), int(os.environ.get("N", 4096))
    rng = np.random.default_rng(0)
    wq = rng.integers(-1, 2, (N, N)).astype(np.int8)
    layer = tk.make_packed_conv_layer(wq, tk.ConvGeometry(N, N, 1, 1, 1, 0), tk.QuantThresholds(),
                                      tk.QuantThresholds(0.5, 0.9), True)
    x = torch.from_numpy(np.abs(rng.standard_normal((B, N))).astype(np.float32)).cuda()
    fmt = os.environ.get("FMT", "s8")
    a8 = tk.quantize_levels(x, tk.QuantThresholds(0.5, 0.9), tk.QuantMode.kActivationNonneg,
                            tk.layer_k_pad(layer, fmt), fmt)
    fused = bool(os.environ.get("FUSED"))  # f32 folded-BN rows instead of int32
    out = torch.empty((B, N), dtype=torch.float32 if fused else torch.int32, device="cuda")
    flush = torch.empty(256 * 2**20 // 4, device="cuda")
    for _ in range(3):
        tk.gemm_levels(a8, layer, fused=fused, out=out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()  # back-to-back launches without host gaps
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(5):
                if os.environ.get("FLUSH"):
                    flush.fill_(1.0)
                tk.gemm_levels(a8, layer, fused=fused, out=out)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"graph of 5 launches: {e0.elapsed_time(e1) * 1e3 / 5:.2f} us per launch")
    if os.environ.get("GRAPHS"):
        for n in (1, 5, 20, 50):
            g2 = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                with torch.cuda.graph(g2, stream=s):
                    for _ in range(n):
                        tk.gemm_levels(a8, layer, fused=fused, out=out)
            torch.cuda.synchronize()
            g2.replay()
            torch.cuda.synchronize()
            e0.record()
            for _ in range(5):
                g2.replay()
            e1.record()
            torch.cuda.synchronize()
            print(f"  graph of {n}: {e0.elapsed_time(e1) * 1e3 / 5 / n:.2f} us per launch")
    st = np.zeros(512 * 28, np.uint64)
    assert _lib.lib().tk_debug_gemm_stamps(st.ctypes.data) == 0
    gts = st[512 * 8:512 * 12].reshape(2, 512, 2).astype(np.int64)
    n = int((gts[0, :, 0] > 0).sum())
    a, b = gts[0, :n], gts[1, :n]  # the graph's last two launches, in start order
    if a[:, 0].min() > b[:, 0].min():
        a, b = b, a
    print(f"launch 4 span {a[:, 1].max() - a[:, 0].min()} ns; gap to launch 5 first start "
          f"{b[:, 0].min() - a[:, 1].max()} ns; launch 5 span {b[:, 1].max() - b[:, 0].min()} ns, "
          f"starts over {b[:, 0].max() - b[:, 0].min()} ns; launch-to-launch {b[:, 0].min() - a[:, 0].min()} ns")
    s2 = st[512 * 12:].reshape(512, 16).astype(np.int64)
    s = st[:512 * 8].reshape(512, 8).astype(np.int64)
    if s2[:, 12].any():
        k = s2[:, 12] > 0
        rel = s2[k] - s[k, 5:6]
        med = lambda i: int(np.median(rel[:, i])) if (s2[k, i] > 0).all() else None  # noqa: E731
        print("reduction after the cluster barrier: loop start", med(0), "iterations", [med(i) for i in range(1, 9)],
              "loop done", med(12), "sync", med(13), "stores issued", med(14), "stores read", med(15))
    s = s[s[:, 0] > 0]
    names = ["start", "setup", "staged_smem", "mma_issued", "slices_out", "cluster_bar", "reduced", "end"]
    print(f"{len(s)} CTAs; SM clock cycles after each CTA's own start (1965 cycles = 1 us)")
    for i, n in enumerate(names):
        v = s[:, i] - s[:, 0]
        v = v[s[:, i] > 0]
        if len(v):
            print(f"{n:16s} min {v.min():8d}  med {int(np.median(v)):8d}  max {v.max():8d}")


if __name__ == "__main__":
    main()
