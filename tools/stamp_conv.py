"""Per-CTA phase timestamps of one fused conv (TK_CONV_DBG=16|x)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _profile  # noqa: E402,F401  (the -DTK_PROFILE build: experiment knobs)
os.environ["TK_CONV_DBG"] = str(16 | int(os.environ.get("DBG", "0")))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2008_05101_b200 import _lib  # noqa: E402
from paper_2008_05101_b200.resnet import TernaryBody, _conv  # noqa: E402


def main():
    c = int(os.environ.get("C", 64))
    hw = int(os.environ.get("HW", 56))
    batch = int(os.environ.get("B", 256))
    rng = np.random.default_rng(0)
    if os.environ.get("INNER"):  # trace the inner (integer-threshold epilogue) conv of a 2-conv block
        os.environ["TK_CONV_DBG_ONLY"] = "0"
        blocks = [dict(convs=[_conv(rng, c, c, 3, 1, (0.5, 0.9)), _conv(rng, c, c, 3, 1, (0.45, 0.85), False)])]
    else:
        blocks = [dict(convs=[_conv(rng, c, c, 3, 1, (0.5, 0.9), False)])]
    body = TernaryBody(blocks, batch, c, hw, hw)
    x = torch.relu(torch.randn(batch, c, hw, hw, device="cuda"))
    for _ in range(3):
        body.forward(x, check_errors=False)
    torch.cuda.synchronize()
    st = np.zeros(148 * 8 + 8 * 32, np.uint64)
    L = _lib.lib()
    L.tk_debug_conv_stamps.argtypes = [C.c_void_p]
    assert L.tk_debug_conv_stamps(st.ctypes.data) == 0
    tr = st[148 * 8:].reshape(8, 32).astype(np.int64)
    s = st[:148 * 8].reshape(148, 8).astype(np.int64)
    base = tr[tr > 0].min()
    cols = [(6, "mma_top"), (1, "after_aempty"), (7, "after_fence"), (2, "after_hfull"), (4, "after_taps"),
            (5, "after_commits"), (0, "producer"), (3, "epi_afull")]
    print("CTA0 trace, SM clocks: " + " ".join(f"{n:>12s}" for _, n in cols))
    for i in range(int(os.environ.get('ROWS', 10))):
        print(f"{i:2d} " + " ".join(f"{tr[r, i] - base:12d}" if tr[r, i] else f"{'-':>12s}" for r, _ in cols))
    t0 = s[:, 0].min()
    rel = (s[:, :6] - t0) / 1000.0
    names = ["start", "mma_setup", "w_res_ready", "mma_done", "epi_done", "end"]
    for i, n in enumerate(names):
        print(f"{n:12s} min {rel[:, i].min():8.2f} us  med {np.median(rel[:, i]):8.2f}  max {rel[:, i].max():8.2f}")


if __name__ == "__main__":
    main()
