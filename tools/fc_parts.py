"""cfg3 FC step parts (L2 flushed before each replay): quantize alone, GEMM
alone, both (the bench step), each as a one-launch CUDA graph."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    w = bench.FcWorkload()
    flush = bench.L2Flush()
    tk = w.tk
    q = lambda: tk.quantize_levels(w.x, tk.QuantThresholds(0.5, 0.9), tk.QuantMode.kActivationNonneg,  # noqa
                                   tk.layer_k_pad(w.layer, w.fmt), w.fmt)
    g = lambda: tk.gemm_levels(w.a8, w.layer, fused=True, out=w.y)  # noqa
    empty = torch.empty(1, device="cuda")
    for name, fn in (("empty graph", lambda: empty.add_(0)), ("quantize", q), ("gemm", g), ("step", w.step)):
        ms = bench._time_graph(bench.graph_of(fn), flush, n=30)
        ms_warm = bench._time_graph(bench.graph_of(fn), lambda: None, n=30)
        print(f"{name:12s} cold {ms * 1e3:7.2f} us   warm {ms_warm * 1e3:7.2f} us")


if __name__ == "__main__":
    main()
