"""Time the parts of the ResNet e2e step (H2D, stem, body, head, D2H)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import ResNetWorkload  # noqa: E402


def t(fn, n=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / n


w = ResNetWorkload(os.environ.get("W", "resnet18"))
net = w.net
buf = torch.empty_like(w.images_dev)
print("h2d   ms", t(lambda: buf.copy_(w.images_host, non_blocking=True)))
print("stem  ms", t(lambda: net.stem(w.images_dev)))
print("body  ms", t(lambda: net.body.forward(w.x, pooled=w.pooled, check_errors=False)))
print("head  ms", t(lambda: torch.addmm(net.head_b, w.pooled, net.head_w.t())))
print("e2e   ms", t(w.step_e2e))
pipe = w.pipe
cb = pipe.slices[0]
img = torch.empty((cb, 3, 224, 224), device="cuda")
print(f"chunk of {cb}: h2d ms", t(lambda: img.copy_(w.images_host[:cb], non_blocking=True)),
      "stem+body ms", t(lambda: pipe.bodies[min(pipe.bodies)].forward(net.stem(img), pooled=pipe.pooled[:cb], check_errors=False)))
