"""Per-conv device times of a ResNet body under experiment knobs (profiling
build): LAYER_AB="NAME=VAL,..;NAME=VAL" runs one body per ';'-separated
setting and prints the per-conv ms side by side.  DEPTH / B select the body."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _profile  # noqa: E402,F401

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2008_05101_b200.resnet import TernaryBody, resnet_spec  # noqa: E402


def main():
    depth = int(os.environ.get("DEPTH", 50))
    batch = int(os.environ.get("B", 256))
    settings = [s for s in os.environ.get("LAYER_AB", "").split(";")]
    blocks = resnet_spec(depth, 0)
    x = torch.relu(torch.randn(batch, 64, 56, 56, device="cuda"))
    flush = torch.empty(256 * 2**20 // 4, device="cuda")
    cols, names = [], []
    for st in settings:
        env = dict(kv.split("=") for kv in st.split(",") if kv)
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        body = TernaryBody(blocks, batch, 64, 56, 56)
        for _ in range(3):  # first launches load the kernels (lazy module loading)
            body.forward(x, check_errors=False)
        torch.cuda.synchronize()
        ms, _ = body.conv_times(x, flush=lambda: flush.fill_(1.0), reps=5)
        cols.append(ms)
        names.append(st or "default")
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        del body
        torch.cuda.synchronize()
    print("conv  " + "  ".join(f"{n:>18s}" for n in names))
    for i in range(len(cols[0])):
        print(f"{i:4d}  " + "  ".join(f"{c[i] * 1e3:18.1f}" for c in cols))
    print("sum   " + "  ".join(f"{c.sum() * 1e3:18.1f}" for c in cols))


if __name__ == "__main__":
    main()
