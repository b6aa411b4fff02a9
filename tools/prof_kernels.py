"""Profiling driver for the integer-pipe and packing kernels (run plain first,
then under ncu): the LOP3+POPC GEMM on the cfg3 FC and cfg2 conv shapes,
quantize+pack on the cfg1 rows, conv2d_ternary's input packing (cfg2) and
the ResNet body's input packing (cfg4 b256), each after an L2 flush."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2008_05101_b200 import ternkit as tk  # noqa: E402
from paper_2008_05101_b200.resnet import TernaryBody, resnet_spec  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    flush = torch.empty(256 * 2**20 // 4, device="cuda")
    QT, QM = tk.QuantThresholds, tk.QuantMode
    # cfg3 FC on the POPC pipe
    wq = rng.integers(-1, 2, (4096, 4096)).astype(np.int8)
    fc = tk.make_packed_conv_layer(wq, tk.ConvGeometry(4096, 4096, 1, 1, 1, 0), QT(), QT(0.5, 0.9), True)
    fc.set_backend(tk.Backend.POPC)
    x = torch.from_numpy(np.abs(rng.standard_normal((256, 4096))).astype(np.float32)).cuda()
    # cfg2 conv on the POPC pipe and on the fused path (k_pack_input)
    wc = rng.integers(-1, 2, (64, 576)).astype(np.int8)
    cv = tk.make_packed_conv_layer(wc, tk.ConvGeometry(64, 64, 3, 3, 1, 1), QT(1, 1), QT(0.5, 0.5), True)
    xc = torch.from_numpy(np.abs(rng.standard_normal(64 * 56 * 56)).astype(np.float32)).cuda()
    shape = tk.TensorShape(1, 64, 56, 56)
    # cfg1 rows: quantize + pack of 65536 x 4096 floats
    x1 = torch.randn((65536, 4096), device="cuda").abs_()
    # cfg4 body input packing
    body = TernaryBody(resnet_spec(18, 0), 256, 64, 56, 56)
    xb = torch.relu(torch.randn(256, 64, 56, 56, device="cuda"))
    for _ in range(2):
        for f in (lambda: tk.fully_connected_ternary(x, 256, fc, check_errors=False),
                  lambda: (cv.set_backend(tk.Backend.POPC), tk.conv2d_ternary(xc, shape, cv, check_errors=False)),
                  lambda: (cv.set_backend(tk.Backend.AUTO), tk.conv2d_ternary(xc, shape, cv, check_errors=False)),
                  lambda: tk.quantize_and_pack_rows(x1, QT(0.5, 0.9), QM.kActivationNonneg),
                  lambda: body.forward(xb, check_errors=False)):
            flush.fill_(1.0)
            f()
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
