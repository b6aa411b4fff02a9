"""Profiling driver for the cfg3 FC GEMM (run plain first, then under ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2008_05101_b200 import ternkit as tk  # noqa: E402


def main():
    B = int(os.environ.get("B", 256))
    C = N = int(os.environ.get("N", 4096))
    rng = np.random.default_rng(0)
    wq = rng.integers(-1, 2, (N, C)).astype(np.int8)
    layer = tk.make_packed_conv_layer(wq, tk.ConvGeometry(C, N, 1, 1, 1, 0), tk.QuantThresholds(),
                                      tk.QuantThresholds(0.5, 0.9), True)
    backend = os.environ.get("BACKEND", "TC_I8")
    layer.set_backend(tk.Backend[backend])
    fmt = "fp4" if backend == "TC_F4" else "s8"
    x = torch.from_numpy(np.abs(rng.standard_normal((B, C))).astype(np.float32)).cuda()
    a8 = tk.quantize_levels(x, tk.QuantThresholds(0.5, 0.9), tk.QuantMode.kActivationNonneg,
                            tk.layer_k_pad(layer, fmt), fmt)
    out = torch.empty((B, N), dtype=torch.int32, device="cuda")
    for _ in range(3):
        tk.gemm_levels(a8, layer, out=out)
    torch.cuda.synchronize()
    # timing with graph replay (no host gaps)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(10):
                tk.gemm_levels(a8, layer, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{fmt} gemm {B}x{N}x{C}: {ms * 1e3:.2f} us/launch (L2-warm, back-to-back) = "
          f"{2 * B * N * C / ms / 1e9:.1f} TOPS")
    lv = tk.unpack(tk.PackedTernaryVector(tk.quantize_and_pack_rows(x[:2], tk.QuantThresholds(0.5, 0.9),
                   tk.QuantMode.kActivationNonneg).view(-1), 2 * C)).cpu().numpy().reshape(2, C) + 1
    want = lv.astype(np.int64) @ wq.T.astype(np.int64)
    assert np.array_equal(out[:2].cpu().numpy(), want), "mismatch"
    print("ok")


if __name__ == "__main__":
    main()
