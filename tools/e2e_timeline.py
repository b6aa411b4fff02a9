"""Event timeline of one pipelined ResNet e2e step (copy stream vs compute
stream), relative to the step start (ms)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import ResNetWorkload  # noqa: E402
from paper_2008_05101_b200.resnet import PipelinedResNet  # noqa: E402


def main():
    w = ResNetWorkload(os.environ.get("W", "resnet18"))
    if os.environ.get("PIPE_GROUPS"):  # e.g. PIPE_GROUPS=5,3 (bash reserves GROUPS) (CHUNKS default 8)
        sl = [int(c) for c in os.environ["SLICES"].split(",")] if os.environ.get("SLICES") else None
        w.pipe = PipelinedResNet(w.net, w.B, int(os.environ.get("CHUNKS", 8)),
                                 [int(g) for g in os.environ["PIPE_GROUPS"].split(",")], slices=sl)
    pipe = w.pipe
    for _ in range(3):
        w.step_e2e()
    torch.cuda.synchronize()
    cs = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    t0 = ev()
    t0.record(cs)
    marks = []
    pipe.copy_stream.wait_stream(cs)
    with torch.cuda.stream(pipe.copy_stream):
        for i in range(pipe.chunks):
            pipe.copy_stream.wait_event(pipe.ev_consumed[i])
            pipe.img[i].copy_(w.images_host[pipe.off[i]:pipe.off[i + 1]], non_blocking=True)
            pipe.ev_copied[i].record(pipe.copy_stream)
            e = ev()
            e.record(pipe.copy_stream)
            marks.append((f"h2d {i} done", e))
    i = 0
    for gi, g in enumerate(pipe.groups):
        g0 = pipe.off[i]
        for _ in range(g):
            cs.wait_event(pipe.ev_copied[i])
            pipe.net.stem(pipe.img[i], out=pipe.xg[gi][pipe.off[i] - g0:pipe.off[i + 1] - g0])
            pipe.ev_consumed[i].record(cs)
            e = ev()
            e.record(cs)
            marks.append((f"stem {i} done", e))
            i += 1
        n = pipe.gsize[gi]
        pipe.bodies[n].forward(pipe.xg[gi], pooled=pipe.pooled[g0:g0 + n], check_errors=False)
        e = ev()
        e.record(cs)
        marks.append((f"body group {gi} ({g} slices, {n} images) done", e))
    pipe.net.head(pipe.pooled, out=pipe.logits)
    e = ev()
    e.record(cs)
    marks.append(("head done", e))
    torch.cuda.synchronize()
    for name, e in sorted(marks, key=lambda m: t0.elapsed_time(m[1])):
        print(f"{t0.elapsed_time(e):7.3f} ms  {name}")


if __name__ == "__main__":
    main()
