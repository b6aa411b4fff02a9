"""Stem variants (fp32, no TF32): time per batch of 256 images."""
import torch
import torch.nn.functional as F

torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False
B = 256
x = torch.rand(B, 3, 224, 224, device="cuda")
w = torch.randn(64, 3, 7, 7, device="cuda") / 12
g = torch.rand(64, device="cuda") + 0.5
b = torch.randn(64, device="cuda") * 0.1


def t(fn, n=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / n


def base():
    y = F.conv2d(x, w, stride=2, padding=3)
    y = torch.relu(y * g.view(1, -1, 1, 1) + b.view(1, -1, 1, 1))
    return F.max_pool2d(y, 3, 2, 1)


print("baseline NCHW          ", t(base))
torch.backends.cudnn.benchmark = True
print("cudnn.benchmark NCHW   ", t(base))
xc = x.contiguous(memory_format=torch.channels_last)
wc = (w * g.view(-1, 1, 1, 1)).contiguous(memory_format=torch.channels_last)


def cl():
    y = F.conv2d(xc, wc, b, stride=2, padding=3)
    y = torch.relu_(y)
    return F.max_pool2d(y, 3, 2, 1)


print("channels_last folded   ", t(cl))
print("conv only NHWC         ", t(lambda: F.conv2d(xc, wc, b, stride=2, padding=3)))
print("conv only NCHW         ", t(lambda: F.conv2d(x, w, stride=2, padding=3)))
