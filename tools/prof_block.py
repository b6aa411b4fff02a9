"""One residual block (stage-1 shape of ResNet-18 by default) forward a few
times: the target of single-kernel ncu captures of k_conv_tc."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2008_05101_b200.resnet import TernaryBody, _conv  # noqa: E402


def main():
    c = int(os.environ.get("C", 64))
    hw = int(os.environ.get("HW", 56))
    batch = int(os.environ.get("B", 256))
    rng = np.random.default_rng(0)
    blocks = [dict(convs=[_conv(rng, c, c, 3, 1, (0.5, 0.9)), _conv(rng, c, c, 3, 1, (0.45, 0.85), False)])]
    body = TernaryBody(blocks, batch, c, hw, hw)
    x = torch.relu(torch.randn(batch, c, hw, hw, device="cuda"))
    for _ in range(int(os.environ.get("ITERS", 3))):
        body.forward(x, check_errors=False)
    torch.cuda.synchronize()
    ms, macs = body.conv_times(x, reps=3)
    print("conv ms:", [round(float(m), 4) for m in ms])


if __name__ == "__main__":
    main()
