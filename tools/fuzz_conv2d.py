"""Parity fuzz: random conv2d_ternary problems (channels 64/128/256, 1x1 and
3x3, stride 1/2, ragged planes, batch 1-4, random thresholds / BN / out_scale)
on every backend (AUTO, TC_CONV, TC_I8, TC_F4, POPC) vs the C oracle,
bit-exact f32.  Test infrastructure only (runs the oracle as the checker)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Oracle  # noqa: E402
from paper_2008_05101_b200 import ternkit as tk  # noqa: E402


def main():
    o = Oracle()
    bad = 0
    for seed in range(2000, 2040):
        rng = np.random.default_rng(seed)
        c = int(rng.choice([64, 128, 256]))
        oc = int(rng.choice([64, 128, 256]))
        k = int(rng.choice([1, 3]))
        s = int(rng.choice([1, 2]))
        h = int(rng.integers(8, 30)) & ~(s - 1)
        w = int(rng.integers(8, 30)) & ~(s - 1)
        n = int(rng.integers(1, 5))
        ta = tuple(sorted(rng.uniform(0.3, 1.2, 2)))
        wq = rng.integers(-1, 2, (oc, c * k * k)).astype(np.int8)
        gain = (rng.uniform(-1.5, 1.5, oc) / 16).astype(np.float32)
        bias = rng.standard_normal(oc).astype(np.float32)
        scale = float(rng.choice([1.0, 0.37]))
        x = np.abs(rng.standard_normal(n * c * h * w)).astype(np.float32)
        st, want = o.conv2d_ternary(x, n, c, h, w, wq, oc, k, s, k // 2, ta, True, gain, bias, scale)
        assert st == 0
        for be in ("AUTO", "TC_CONV", "TC_I8", "TC_F4", "POPC"):
            layer = tk.make_packed_conv_layer(wq, tk.ConvGeometry(c, oc, k, k, s, k // 2), tk.QuantThresholds(1.0, 1.0),
                                              tk.QuantThresholds(*ta), True, tk.ChannelAffine(gain, bias), scale)
            layer.set_backend(tk.Backend[be])
            y = tk.conv2d_ternary(x, tk.TensorShape(n, c, h, w), layer).data.cpu().numpy()
            m = np.count_nonzero(y.view(np.int32) != want.view(np.int32))
            if m:
                bad += 1
                print("seed", seed, be, (c, oc, k, s, h, w, n), "mismatches", m)
    print("fuzz done, bad =", bad)


if __name__ == "__main__":
    main()
