"""Phase timeline of the tensor-core GEMM (cfg3 shape) from in-kernel
globaltimer stamps (env TK_GEMM_DBG |= 16)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
    a8 = tk.quantize_levels(x, tk.QuantThresholds(0.5, 0.9), tk.QuantMode.kActivationNonneg, tk.layer_k_pad(layer))
    out = torch.empty((B, N), dtype=torch.int32, device="cuda")
    flush = torch.empty(256 * 2**20 // 4, device="cuda")
    for _ in range(5):
        if os.environ.get("FLUSH"):
            flush.fill_(1.0)
        tk.gemm_levels(a8, layer, out=out)
    torch.cuda.synchronize()
    st = np.zeros(512 * 8, np.uint64)
    assert _lib.lib().tk_debug_gemm_stamps(st.ctypes.data) == 0
    s = st.reshape(512, 8).astype(np.int64)
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
