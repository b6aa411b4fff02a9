"""ResNet e2e schedule A/B: PipelinedResNet (host images -> slices on a copy
stream -> stem per slice -> ternary body per group of slices -> head) for
several (chunks, groups) settings; K steps between one event pair, as bench.py."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("PROFILE"):  # the -DTK_PROFILE build (experiment knobs such as TK_PDL)
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import _profile  # noqa: E402,F401
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2008_05101_b200.resnet import PipelinedResNet, TernaryResNet  # noqa: E402


def main():
    depth = int(os.environ.get("DEPTH", 18))
    batch = int(os.environ.get("B", 256))
    net = TernaryResNet(depth, batch, 0)
    imgs = torch.rand(batch, 3, 224, 224, generator=torch.Generator().manual_seed(1)).pin_memory()
    out_host = torch.empty((batch, 1000)).pin_memory()
    settings = [(8, [3, 5]), (8, [4, 4]), (8, [2, 2, 2, 2]), (8, [1] * 8), (8, [2, 2, 2, 1, 1]), (8, [4, 2, 1, 1]),
                (8, [3, 3, 2]), (16, [4, 4, 4, 4]), (16, [2] * 8), (16, [4, 4, 4, 2, 2]), (16, [1] * 16),
                (4, [1] * 4)]
    if os.environ.get("SETTINGS"):  # e.g. "8:3,5;16:4,4,4,4" or with uneven slices "32,32,48,16:1,1,2"
        settings = []
        for item in os.environ["SETTINGS"].split(";"):
            c, gs = item.split(":")
            settings.append(([int(v) for v in c.split(",")] if "," in c else int(c), [int(g) for g in gs.split(",")]))
    for chunks, groups in settings:
        if isinstance(chunks, list):
            pipe = PipelinedResNet(net, batch, len(chunks), groups, slices=chunks)
        else:
            pipe = PipelinedResNet(net, batch, chunks, groups)

        def step():
            y = pipe.forward(imgs)
            out_host.copy_(y, non_blocking=True)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        ms, _, _ = bench.flushed_loop_ms(lambda: [step() for _ in range(10)], lambda: None)
        print(f"chunks {str(chunks):>12s} groups {str(groups):14s} {ms / 10:.3f} ms/step  {batch / (ms / 10) * 1e3:,.0f} img/s")
        del pipe
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
