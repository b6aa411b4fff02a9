"""cfg3 GEMM tile / split-K A/B of k_gemm_tc_i8 on s8 and fp4 level operands
(profiling build: TK_GEMM_BN / TK_GEMM_SPLIT force the tile width and the
cluster K split); warm = 20 back-to-back launches in one graph, cold = 256 MB
L2 flush before each single launch (event resolution on the B200 boxes is
2.048 us, so single-launch numbers are quantized; the warm ones are not)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _profile  # noqa: E402,F401

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2008_05101_b200 import ternkit as tk  # noqa: E402


def main():
    B = int(os.environ.get("B", 256))
    C = N = int(os.environ.get("N", 4096))
    rng = np.random.default_rng(0)
    wq = rng.integers(-1, 2, (N, C)).astype(np.int8)
    layer = tk.make_packed_conv_layer(wq, tk.ConvGeometry(C, N, 1, 1, 1, 0), tk.QuantThresholds(),
                                      tk.QuantThresholds(0.5, 0.9), True,
                                      tk.ChannelAffine(np.ones(N, np.float32), np.zeros(N, np.float32)))
    x = torch.from_numpy(np.abs(rng.standard_normal((B, C))).astype(np.float32)).cuda()
    flush = torch.empty(256 * 2**20 // 4, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ref = None
    for fmt in ("fp4", "s8"):
        a = tk.quantize_levels(x, tk.QuantThresholds(0.5, 0.9), tk.QuantMode.kActivationNonneg,
                               tk.layer_k_pad(layer, fmt), fmt)
        out = torch.empty((B, N), dtype=torch.float32, device="cuda")
        configs = [("auto", {})]
        for mc in (2, 4, 8):
            configs.append((f"A multicast x{mc}", {"TK_GEMM_MC": str(mc)}))
        for bn, sp in [tuple(map(int, c.split("x"))) for c in os.environ.get("FC_TILES", "").split(",") if c]:
            configs.append((f"BN{bn} S{sp}", {"TK_GEMM_BN": str(bn), "TK_GEMM_SPLIT": str(sp)}))
        for kern, env in configs:
            for k in ("TK_GEMM_BN", "TK_GEMM_SPLIT", "TK_GEMM_MC"):
                os.environ.pop(k, None)
            os.environ.update(env)
            for _ in range(3):
                tk.gemm_levels(a, layer, fused=True, out=out)
            torch.cuda.synchronize()
            if ref is None:
                ref = out.clone()
            assert torch.equal(out, ref), (fmt, kern)
            s = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    for _ in range(20):
                        tk.gemm_levels(a, layer, fused=True, out=out)
            torch.cuda.synchronize()
            e0.record(); g.replay(); e1.record(); e1.synchronize()
            warm = e0.elapsed_time(e1) / 20 * 1e3
            cold = []
            for _ in range(20):
                flush.fill_(1.0)
                e0.record()
                tk.gemm_levels(a, layer, fused=True, out=out)
                e1.record()
                e1.synchronize()
                cold.append(e0.elapsed_time(e1) * 1e3)
            print(f"{fmt} {kern:20s} warm {warm:7.2f} us  cold {np.median(cold):7.2f} us "
                  f"({2 * B * N * C / np.median(cold) / 1e6:.0f} TOPS cold)")


if __name__ == "__main__":
    main()
