"""Per-conv device time of a ResNet body under the TK_CONV_DBG knobs
(1 no MMA, 2 no halo TMA, 4 no epilogue math/stores): attributes each conv's
time to its pipeline roles.  Usage: DEPTH=18 B=256 python tools/conv_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _profile  # noqa: E402,F401  (the -DTK_PROFILE build: experiment knobs)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2008_05101_b200.resnet import TernaryBody, resnet_spec  # noqa: E402


def main():
    depth = int(os.environ.get("DEPTH", 18))
    batch = int(os.environ.get("B", 256))
    modes = [int(m) for m in os.environ.get("MODES", "0,1,2,4,5,6,7").split(",")]
    blocks = resnet_spec(depth, 0)
    x = torch.relu(torch.randn(batch, 64, 56, 56, device="cuda"))
    flush = torch.empty(256 * 2**20 // 4, device="cuda")
    rows = {}
    macs = None
    for m in modes:
        os.environ["TK_CONV_DBG"] = str(m)
        body = TernaryBody(blocks, batch, 64, 56, 56)
        runs = []
        for _ in range(int(os.environ.get("REPS", 15))):
            ms, macs = body.conv_times(x, flush=lambda: flush.fill_(1.0), reps=1)
            runs.append(ms)
        rows[m] = np.median(np.stack(runs), axis=0)  # per conv, robust to outliers
        del body
    os.environ.pop("TK_CONV_DBG", None)
    print("conv  gmac   " + "  ".join(f"dbg{m:<3d}" for m in modes))
    for i in range(len(macs)):
        print(f"{i:4d} {macs[i] / 1e9:6.2f}  " + "  ".join(f"{rows[m][i] * 1e3:6.1f}" for m in modes))
    print("sum         " + "  ".join(f"{rows[m].sum() * 1e3:6.1f}" for m in modes), "(us)")


if __name__ == "__main__":
    main()
