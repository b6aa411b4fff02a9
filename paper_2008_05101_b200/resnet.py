"""ResNet-18/50-shaped ternary networks on the fused B200 pipeline.

The reference has no ResNet definition; these networks apply
its network composition pattern -- packed_forward, R:tinynet.hpp:713-735 --
to conv layers: every quantized layer is conv2d_ternary (R:linalg.hpp:301-328)
with its folded BN, inner convs are followed by ReLU, and each block ends with
z = max(conv(h) + shortcut, 0).  As in the paper's protocol
the first (7x7 stem) and last (FC head) layers stay in float.

    TernaryBody      -- the ternary hot path (tk_net_* C-ABI, CUDA)
    TernaryResNet    -- float stem (split-TF32 tensor cores) + TernaryBody + float head
    resnet_spec()    -- synthetic random-weight ResNet-18 / ResNet-50 bodies
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _lib as T
from ._lib import check
from . import ternkit as tk


# ---------------------------------------------------------------------------
# synthetic specs

def _conv(rng, in_c, out_c, k, stride, ta, relu_follows=True):
    K = in_c * k * k
    # folded BN: gain normalises the ternary accumulator to ~unit variance
    # (E[a^2] ~ 1.8 for levels of half-normal inputs, E[w^2] = 2/3) so every
    # quantization level keeps occurring layer after layer.
    gain = (rng.uniform(0.8, 1.2, out_c) / math.sqrt(K * 1.2)).astype(np.float32)
    bias = (rng.standard_normal(out_c) * 0.25 - (0.0 if relu_follows else 0.3)).astype(np.float32)
    return dict(in_c=in_c, out_c=out_c, k=k, stride=stride, pad=k // 2,
                weights=rng.integers(-1, 2, (out_c, K)).astype(np.int8),
                ta=ta, tw=(1.0, 1.0), gain=gain, bias=bias, out_scale=1.0)


def resnet_spec(depth: int = 18, seed: int = 0, width: int = 64, variant: str = "v1.5"):
    """Body blocks (after the stem, input width x 56 x 56) of a ResNet-depth."""
    rng = np.random.default_rng(seed)
    blocks = []
    c = width
    ta = lambda: (float(np.float32(rng.uniform(0.4, 0.6))), float(np.float32(rng.uniform(0.8, 1.0))))  # noqa: E731
    if depth == 18:
        for stage, (w, n) in enumerate([(64, 2), (128, 2), (256, 2), (512, 2)]):
            for i in range(n):
                s = 2 if (stage > 0 and i == 0) else 1
                t1 = ta()
                blk = dict(convs=[_conv(rng, c, w, 3, s, t1), _conv(rng, w, w, 3, 1, ta(), False)])
                if s != 1 or c != w:
                    blk["down"] = _conv(rng, c, w, 1, s, t1, False)
                blocks.append(blk)
                c = w
    elif depth == 50:
        # v1.5 bottleneck (the stride sits on the 3x3 conv): 3.969 GMAC/img,
        # the count SURVEY.md §8(d) uses for cfg5; variant="v1" puts it on the
        # first 1x1 (3.738 GMAC/img)
        for stage, (w, n) in enumerate([(64, 3), (128, 4), (256, 6), (512, 3)]):
            for i in range(n):
                s = 2 if (stage > 0 and i == 0) else 1
                s1, s3 = (s, 1) if variant == "v1" else (1, s)
                t1 = ta()
                blk = dict(convs=[_conv(rng, c, w, 1, s1, t1), _conv(rng, w, w, 3, s3, ta()),
                                  _conv(rng, w, 4 * w, 1, 1, ta(), False)])
                if s != 1 or c != 4 * w:
                    blk["down"] = _conv(rng, c, 4 * w, 1, s, t1, False)
                blocks.append(blk)
                c = 4 * w
    else:
        raise ValueError("depth must be 18 or 50")
    return blocks


def body_macs(blocks, h=56, w=56) -> int:
    """Ternary multiply-accumulates per image of a body spec."""
    macs = 0
    for blk in blocks:
        hh, ww = h, w
        for cv in blk["convs"]:
            hh = (hh + 2 * cv["pad"] - cv["k"]) // cv["stride"] + 1
            ww = (ww + 2 * cv["pad"] - cv["k"]) // cv["stride"] + 1
            macs += hh * ww * cv["out_c"] * cv["in_c"] * cv["k"] ** 2
        if blk.get("down") is not None:
            d = blk["down"]
            macs += hh * ww * d["out_c"] * d["in_c"]
        h, w = hh, ww
    return macs


def body_bytes(blocks, batch: int, in_c: int = 64, h: int = 56, w: int = 56) -> int:
    """Algorithmic HBM bytes of one fused body forward (the roofline's HBM
    view): every conv reads its s8 level input once (1 B / element) and its
    weights once; inner convs write the next conv's levels (1 B); a block's
    last conv reads the skip (f32 identity, 4 B; s16 downsample
    accumulators, 2 B) and writes the f32 block output (4 B) plus the next
    block's levels (1 B, none after the last block); a downsample conv writes
    its s16 accumulators (2 B).  Halo re-reads, padding rows and duplicate
    quantizer outputs are not counted."""
    total = 0
    c, hh, ww = in_c, h, w
    for bi, blk in enumerate(blocks):
        last_blk = bi == len(blocks) - 1
        h_in, w_in, c_in = hh, ww, c
        for ci, cv in enumerate(blk["convs"]):
            ho = (hh + 2 * cv["pad"] - cv["k"]) // cv["stride"] + 1
            wo = (ww + 2 * cv["pad"] - cv["k"]) // cv["stride"] + 1
            total += batch * cv["in_c"] * hh * ww + cv["out_c"] * cv["in_c"] * cv["k"] ** 2
            out = batch * cv["out_c"] * ho * wo
            if ci < len(blk["convs"]) - 1:
                total += out
            else:
                total += out * (2 if blk.get("down") is not None else 4)  # skip read
                total += out * 4 + (0 if last_blk else out)
            hh, ww, c = ho, wo, cv["out_c"]
        if blk.get("down") is not None:
            d = blk["down"]
            total += batch * d["in_c"] * h_in * w_in + d["out_c"] * d["in_c"] + batch * d["out_c"] * hh * ww * 2
    return total


# ---------------------------------------------------------------------------
# the ternary body on the GPU

def _desc(cv, keep) -> T.ConvDesc:
    w = np.ascontiguousarray(cv["weights"], dtype=np.int8)
    g = np.ascontiguousarray(cv["gain"], dtype=np.float32)
    b = np.ascontiguousarray(cv["bias"], dtype=np.float32)
    keep += [w, g, b]
    tw = cv.get("tw", (1.0, 1.0))
    return T.ConvDesc(cv["in_c"], cv["out_c"], cv["k"], cv["stride"], cv["pad"],
                      w.ctypes.data_as(C.POINTER(C.c_int8)), tw[0], tw[1], cv["ta"][0], cv["ta"][1],
                      g.ctypes.data_as(C.POINTER(C.c_float)), b.ctypes.data_as(C.POINTER(C.c_float)),
                      cv.get("out_scale", 1.0))


class TernaryBody:
    """Residual ternary conv body (tk_net).  forward(x) takes the body input
    [batch][C][H][W] f32 on the device; returns pooled [batch][C'] and, if
    asked, the full [batch][C'][H'][W'] output."""

    def __init__(self, blocks, batch: int, in_c: int, in_h: int, in_w: int,
                 mode: int = T.TK_NET_AUTO):
        self.blocks = blocks
        self.batch, self.in_c, self.in_h, self.in_w = batch, in_c, in_h, in_w
        keep: list = []
        arr = (T.BlockDesc * len(blocks))()
        for i, blk in enumerate(blocks):
            arr[i].n_convs = len(blk["convs"])
            for j, cv in enumerate(blk["convs"]):
                arr[i].conv[j] = _desc(cv, keep)
            if blk.get("down") is not None:
                arr[i].has_down = 1
                arr[i].down = _desc(blk["down"], keep)
        h = C.c_void_p()
        check(T.lib().tk_net_create(tk.context(), C.cast(arr, C.c_void_p), len(blocks), batch, in_c,
                                    in_h, in_w, mode, C.byref(h)), "tk_net_create")
        self._h = h.value
        oc, oh, ow = C.c_int(), C.c_int(), C.c_int()
        check(T.lib().tk_net_out_shape(self._h, C.byref(oc), C.byref(oh), C.byref(ow)), "out_shape")
        self.out_shape = (oc.value, oh.value, ow.value)
        self.fused = bool(T.lib().tk_net_is_fused(self._h))

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                T.lib().tk_net_destroy(self._h)
            except Exception:
                pass
            self._h = None

    def conv_times(self, x: torch.Tensor, flush=None, reps: int = 5):
        """Per-conv device times (ms, averaged over reps forwards, L2 flushed
        before each by `flush`) and MACs per conv for the whole batch."""
        n = T.lib().tk_net_num_convs(self._h)
        check(T.lib().tk_net_set_timing(self._h, 1), "set_timing")
        ms = np.zeros(n, np.float32)
        acc = np.zeros(n, np.float64)
        macs = np.zeros(n, np.float64)
        for _ in range(reps):
            if flush:
                flush()
            self.forward(x, check_errors=False)
            check(T.lib().tk_net_conv_times(self._h, ms.ctypes.data, macs.ctypes.data), "conv_times")
            acc += ms
        check(T.lib().tk_net_set_timing(self._h, 0), "set_timing")
        return acc / reps, macs

    def launches(self, with_out=False, with_pooled=True) -> int:
        return T.lib().tk_net_launches(self._h, int(with_out), int(with_pooled))

    def forward(self, x: torch.Tensor, want_out: bool = False, pooled: torch.Tensor | None = None,
                out: torch.Tensor | None = None, check_errors: bool = True):
        assert x.is_cuda and x.dtype == torch.float32 and x.is_contiguous()
        assert x.numel() == self.batch * self.in_c * self.in_h * self.in_w
        c, h, w = self.out_shape
        if pooled is None:
            pooled = torch.empty((self.batch, c), dtype=torch.float32, device="cuda")
        if want_out and out is None:
            out = torch.empty((self.batch, c, h, w), dtype=torch.float32, device="cuda")
        check(T.lib().tk_net_forward(tk.context(), self._h, x.data_ptr(),
                                     out.data_ptr() if want_out else None, pooled.data_ptr(),
                                     tk._stream()), "tk_net_forward")
        if check_errors:
            tk.sync("tk_net_forward")
        return (pooled, out) if want_out else pooled


class TernaryResNet:
    """Float stem + ternary body + float head, images [batch][3][224][224]."""

    def __init__(self, depth: int = 18, batch: int = 256, seed: int = 0, classes: int = 1000):
        g = torch.Generator().manual_seed(seed)
        self.batch = batch
        self.stem_w = (torch.randn(64, 3, 7, 7, generator=g) / math.sqrt(3 * 49)).cuda()
        self.stem_gain = (torch.rand(64, generator=g) * 0.5 + 0.75).cuda()
        self.stem_bias = (torch.randn(64, generator=g) * 0.1).cuda()
        self.blocks = resnet_spec(depth, seed)
        self.body = TernaryBody(self.blocks, batch, 64, 56, 56)
        c = self.body.out_shape[0]
        self.head_w = (torch.randn(classes, c, generator=g) / math.sqrt(c)).cuda()
        self.head_b = torch.zeros(classes).cuda()

    def stem(self, images: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """fp32-class 7x7/2 conv (tk_stem_conv7x7s2: split-TF32 tcgen05,
        x_hi w_hi + x_hi w_lo + x_lo w_hi, error <= 4e-6 x sum |x||w|), then one
        fused pass of folded BN (fmaf), ReLU and 3x3/2 max-pool
        (tk_affine_relu_maxpool)."""
        images = images.contiguous()
        n = images.shape[0]
        y = torch.empty((n, 64, 112, 112), dtype=torch.float32, device="cuda")
        check(T.lib().tk_stem_conv7x7s2(tk.context(), images.data_ptr(), n, images.shape[2], images.shape[3],
                                        self.stem_w.data_ptr(), y.data_ptr(), tk._stream()),
              "tk_stem_conv7x7s2")
        n, c, h, w = y.shape
        if out is None:
            out = torch.empty((n, c, (h + 1) // 2, (w + 1) // 2), dtype=torch.float32, device="cuda")
        check(T.lib().tk_affine_relu_maxpool(tk.context(), y.data_ptr(), n, c, h, w, self.stem_gain.data_ptr(),
                                             self.stem_bias.data_ptr(), out.data_ptr(), tk._stream()),
              "tk_affine_relu_maxpool")
        return out

    def head(self, pooled: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """fp32 dense head (tk_dense_f32: four K-quarter FMA chains per logit, summed in order)."""
        pooled = pooled.contiguous()
        if out is None:
            out = torch.empty((pooled.shape[0], self.head_w.shape[0]), dtype=torch.float32, device="cuda")
        check(T.lib().tk_dense_f32(tk.context(), pooled.data_ptr(), self.head_w.data_ptr(), self.head_b.data_ptr(),
                                   pooled.shape[0], pooled.shape[1], self.head_w.shape[0], out.data_ptr(),
                                   tk._stream()), "tk_dense_f32")
        return out

    def forward(self, images: torch.Tensor, check_errors: bool = False) -> torch.Tensor:
        x = self.stem(images)
        pooled = self.body.forward(x, check_errors=check_errors)
        return self.head(pooled)


class PipelinedResNet:
    """End-to-end inference from host images.  The batch is uploaded in
    slices on a copy stream (`chunks` equal slices, or the image counts in
    `slices`); each slice's stem runs (compute stream) as soon as it has
    landed, and the ternary body runs on groups of consecutive slices
    (`groups`: slices per body launch sequence, default one group per slice)
    once their stems are done -- so the body of an early group overlaps the
    upload of later slices, and only the last group's stem + body follow the
    final copy.  Shares the stem/head parameters and block spec of `net`."""

    def __init__(self, net: TernaryResNet, batch: int, chunks: int = 4, groups: list[int] | None = None,
                 slices: list[int] | None = None):
        if slices is None:
            assert batch % chunks == 0
            slices = [batch // chunks] * chunks
        slices = list(slices)
        assert sum(slices) == batch and all(c > 0 for c in slices)
        chunks = len(slices)
        groups = list(groups) if groups else [1] * chunks
        assert sum(groups) == chunks and all(g > 0 for g in groups)
        self.net, self.batch, self.chunks, self.groups, self.slices = net, batch, chunks, groups, slices
        self.off = [sum(slices[:i]) for i in range(chunks + 1)]  # image offset of slice i
        first = [sum(groups[:gi]) for gi in range(len(groups))]   # first slice of group gi
        self.gsize = [self.off[f + g] - self.off[f] for f, g in zip(first, groups)]  # images per group
        self.bodies = {n: TernaryBody(net.blocks, n, 64, 56, 56) for n in sorted(set(self.gsize))}
        self.body = self.bodies[max(self.gsize)]
        self.copy_stream = torch.cuda.Stream()
        self.img = [torch.empty((c, 3, 224, 224), device="cuda") for c in slices]
        # stem outputs of a group, contiguous so the group's body reads one tensor
        self.xg = [torch.empty((n, 64, 56, 56), device="cuda") for n in self.gsize]
        self.ev_copied = [torch.cuda.Event() for _ in range(chunks)]
        self.ev_consumed = [torch.cuda.Event() for _ in range(chunks)]
        self.pooled = torch.empty((batch, self.body.out_shape[0]), device="cuda")
        self.logits = torch.empty((batch, net.head_w.shape[0]), device="cuda")
        self._first = True

    def forward(self, images_host: torch.Tensor) -> torch.Tensor:
        cs = torch.cuda.current_stream()
        # Slice i's upload waits only for the previous call's stem of slice i
        # (ev_consumed), not for the previous call's bodies: back-to-back calls
        # overlap the next batch's upload with this batch's last body and head
        # (the copy engine would otherwise idle through them).  The first call
        # orders its uploads after the caller's earlier work on this stream.
        if self._first:
            self.copy_stream.wait_stream(cs)
        with torch.cuda.stream(self.copy_stream):
            for i in range(self.chunks):
                if not self._first:  # the previous step's stem has read this buffer
                    self.copy_stream.wait_event(self.ev_consumed[i])
                self.img[i].copy_(images_host[self.off[i]:self.off[i + 1]], non_blocking=True)
                self.ev_copied[i].record(self.copy_stream)
        i = 0
        for gi, g in enumerate(self.groups):
            g0 = self.off[i]
            for _ in range(g):
                cs.wait_event(self.ev_copied[i])
                self.net.stem(self.img[i], out=self.xg[gi][self.off[i] - g0:self.off[i + 1] - g0])
                self.ev_consumed[i].record(cs)
                i += 1
            n = self.gsize[gi]
            self.bodies[n].forward(self.xg[gi], pooled=self.pooled[g0:g0 + n], check_errors=False)
        self._first = False
        return self.net.head(self.pooled, out=self.logits)
