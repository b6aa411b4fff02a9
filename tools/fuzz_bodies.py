"""Parity fuzz: 60 random residual bodies (tests/test_gpu_net.py::_random_body,
seeds 1000-1059) through the fused kernels vs the C oracle, bit-exact f32.
Test infrastructure only (runs the oracle as the checker)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from tests.test_gpu_net import _random_body
from oracle.oracle import Oracle
from paper_2008_05101_b200.resnet import TernaryBody
o = Oracle()
bad = 0
for seed in range(1000, 1060):
    blocks, (n, c, h, w), x = _random_body(seed)
    body = TernaryBody(blocks, n, c, h, w)
    pooled, out = body.forward(torch.from_numpy(x.reshape(n, c, h, w)).cuda(), want_out=True)
    st, want = o.net_body(blocks, x, n, c, h, w)
    mism = np.count_nonzero(out.cpu().numpy().view(np.int32) != want.view(np.int32))
    if mism or not body.fused:
        bad += 1
        print("seed", seed, "fused", body.fused, "mismatches", mism)
    del body
print("fuzz done, bad =", bad)
