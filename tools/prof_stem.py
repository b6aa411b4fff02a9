"""Driver for an ncu capture of the stem conv (product library): ResNet stem
7x7/2 3->64 on 256 synthetic 224x224 images, 4 launches (capture -s 3 -c 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2008_05101_b200 import _lib as T  # noqa: E402
from paper_2008_05101_b200 import ternkit as tk  # noqa: E402


def main():
    n = int(os.environ.get("B", 256))
    g = torch.Generator(device="cuda").manual_seed(0)
    w = torch.randn(64, 3, 7, 7, device="cuda", generator=g) / (3 * 49) ** 0.5
    x = torch.rand(n, 3, 224, 224, device="cuda", generator=g)
    y = torch.empty(n, 64, 112, 112, device="cuda")
    for _ in range(4):
        T.check(T.lib().tk_stem_conv7x7s2(tk.context(), x.data_ptr(), n, 224, 224, w.data_ptr(), y.data_ptr(),
                                          tk._stream()), "stem")
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
