"""Profiling driver: the ResNet body forward a few times (plain or under ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2008_05101_b200.resnet import TernaryBody, resnet_spec, body_macs  # noqa: E402


def main():
    depth = int(os.environ.get("DEPTH", 18))
    batch = int(os.environ.get("B", 256))
    iters = int(os.environ.get("ITERS", 3))
    blocks = resnet_spec(depth, 0)
    body = TernaryBody(blocks, batch, 64, 56, 56)
    x = torch.relu(torch.randn(batch, 64, 56, 56, device="cuda"))
    pooled = torch.empty(batch, body.out_shape[0], device="cuda")
    for _ in range(2):
        body.forward(x, pooled=pooled, check_errors=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        body.forward(x, pooled=pooled, check_errors=False)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / iters
    print(f"resnet{depth} b{batch}: {ms:.3f} ms/step, {batch / ms * 1e3:.0f} img/s, "
          f"{2 * body_macs(blocks) * batch / ms / 1e9:.1f} TOPS")


if __name__ == "__main__":
    main()
