"""cfg3 GEMM alone, L2 flushed before each launch (as the bench roofline),
stream launch, for several tile / split choices (TK_GEMM_BN / TK_GEMM_SPLIT)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _profile  # noqa: E402,F401  (the -DTK_PROFILE build: experiment knobs)
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    w = bench.FcWorkload()
    flush = bench.L2Flush()
    gemm = lambda: w.tk.gemm_levels(w.a8, w.layer, fused=True, out=w.y)  # noqa: E731
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for cfg in ("auto", "64,1", "128,1", "128,2", "256,2", "256,4", "128,4"):
        if cfg == "auto":
            os.environ.pop("TK_GEMM_BN", None)
            os.environ.pop("TK_GEMM_SPLIT", None)
        else:
            bn, sp = cfg.split(",")
            os.environ["TK_GEMM_BN"], os.environ["TK_GEMM_SPLIT"] = bn, sp
        for warm in (False, True):
            tot, n = 0.0, 20
            gemm()
            for _ in range(n):
                if not warm:
                    flush()
                e0.record()
                gemm()
                e1.record()
                e1.synchronize()
                tot += e0.elapsed_time(e1)
            print(f"{cfg:6s} {'warm' if warm else 'cold'} {tot / n * 1e3:7.2f} us")


if __name__ == "__main__":
    main()
