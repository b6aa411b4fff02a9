"""Time the two stem kernels separately (batch 256): tk_stem_conv7x7s2 and
tk_affine_relu_maxpool."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2008_05101_b200 import _lib as T, ternkit as tk  # noqa: E402
from paper_2008_05101_b200.resnet import TernaryResNet  # noqa: E402


def t(fn, n=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / n


B = int(os.environ.get("B", 256))
net = TernaryResNet(18, B, 0)
img = torch.rand(B, 3, 224, 224, device="cuda")
y = torch.empty((B, 64, 112, 112), device="cuda")
out = torch.empty((B, 64, 56, 56), device="cuda")
conv = lambda: T.lib().tk_stem_conv7x7s2(tk.context(), img.data_ptr(), B, 224, 224, net.stem_w.data_ptr(),  # noqa
                                         y.data_ptr(), tk._stream())
pool = lambda: T.lib().tk_affine_relu_maxpool(tk.context(), y.data_ptr(), B, 64, 112, 112,  # noqa
                                              net.stem_gain.data_ptr(), net.stem_bias.data_ptr(), out.data_ptr(),
                                              tk._stream())
print(f"stem conv {t(conv):.3f} ms   affine+relu+maxpool {t(pool):.3f} ms   whole stem {t(lambda: net.stem(img)):.3f} ms")
