"""Stem conv A/B: the split-TF32 tensor-core kernel (default) vs the fp32 SIMT
kernel (TK_STEM_SIMT=1, profiling build): max error against an fp64 conv
relative to sum |x||w| per output, and device time per call (K calls between
one event pair) at 32 and 256 images."""
import os

import _profile  # noqa: F401  (profiling build: the TK_STEM_SIMT knob)
import torch

from paper_2008_05101_b200 import _lib as T
from paper_2008_05101_b200 import ternkit as tk


def run(x, w, y):
    T.check(T.lib().tk_stem_conv7x7s2(tk.context(), x.data_ptr(), x.shape[0], x.shape[2], x.shape[3], w.data_ptr(),
                                      y.data_ptr(), tk._stream()), "stem")


def main():
    g = torch.Generator(device="cuda").manual_seed(0)
    w = torch.randn(64, 3, 7, 7, device="cuda", generator=g) / (3 * 49) ** 0.5
    for mode in ("tc", "simt"):
        os.environ["TK_STEM_SIMT"] = "1" if mode == "simt" else "0"
        x = torch.rand(4, 3, 224, 224, device="cuda", generator=g) * 2 - 0.5
        y = torch.empty(4, 64, 112, 112, device="cuda")
        run(x, w, y)
        ref = torch.nn.functional.conv2d(x.double(), w.double(), stride=2, padding=3)
        scale = torch.nn.functional.conv2d(x.double().abs(), w.double().abs(), stride=2, padding=3)
        err = ((y.double() - ref).abs() / scale).max().item()
        for n in (32, 256):
            xs = torch.rand(n, 3, 224, 224, device="cuda", generator=g)
            ys = torch.empty(n, 64, 112, 112, device="cuda")
            for _ in range(3):
                run(xs, w, ys)
            torch.cuda.synchronize()
            k = 20
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(k):
                run(xs, w, ys)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / k * 1e3
            print(f"stem {mode:4s} n={n:3d}: {us:8.1f} us ({us / n:5.2f} us/img)  max rel err {err:.2e}")


if __name__ == "__main__":
    main()
