"""Ternary body device time vs batch size (the e2e pipeline runs the body on
32-128-image groups), with and without programmatic dependent launch between
the convs (TK_PDL, profiling build); K forwards between one event pair."""
import os

import _profile  # noqa: F401  (profiling build: the TK_PDL knob)
import torch

from paper_2008_05101_b200.resnet import TernaryBody, resnet_spec


def main():
    depth = int(os.environ.get("DEPTH", 18))
    blocks = resnet_spec(depth, 0)
    for b in [int(v) for v in os.environ.get("BATCHES", "32,64,128,256").split(",")]:
        body = TernaryBody(blocks, b, 64, 56, 56)
        x = torch.rand(b, 64, 56, 56, device="cuda")
        pooled = torch.empty((b, body.out_shape[0]), device="cuda")
        row = []
        for pdl in ("0", "1"):
            os.environ["TK_PDL"] = pdl
            for _ in range(3):
                body.forward(x, pooled=pooled, check_errors=False)
            torch.cuda.synchronize()
            k = 20
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(k):
                body.forward(x, pooled=pooled, check_errors=False)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / k
            row.append(f"pdl={pdl} {ms * 1e3:7.1f} us ({ms * 1e3 / b:5.2f} us/img)")
        print(f"b={b:4d}  " + "   ".join(row))
        del body
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
