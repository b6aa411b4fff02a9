import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2008_05101_b200 import _lib as T, ternkit as tk
x = torch.rand(256, 3, 224, 224, device="cuda")
w = torch.randn(64, 3, 7, 7, device="cuda")
y = torch.empty(256, 64, 112, 112, device="cuda")
def f():
    T.check(T.lib().tk_stem_conv7x7s2(tk.context(), x.data_ptr(), 256, 224, 224, w.data_ptr(), y.data_ptr(), tk._stream()), "s")
f(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): f()
e1.record(); e1.synchronize()
print("stem conv ms", e0.elapsed_time(e1) / 5)
