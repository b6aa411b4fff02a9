"""GPU parity of network-level inference: the fused tensor-core conv pipeline
and the generic layer-by-layer path vs the C oracle's restatement of the
reference composition (which tests/test_oracle_golden.py pins to the compiled
reference).  Body outputs are compared bit-exactly as f32 -- the integer
accumulators, folded-BN FMA, skip add, ReLU and every intermediate
quantization must all agree for that to hold."""
import numpy as np
import pytest
import torch

from tests.netspec import conv_spec, tiny_body

pytestmark = pytest.mark.gpu


def _run(blocks, x, n, c, h, w, mode=0):
    from paper_2008_05101_b200.resnet import TernaryBody
    body = TernaryBody(blocks, n, c, h, w, mode=mode)
    pooled, out = body.forward(torch.from_numpy(x.reshape(n, c, h, w)).cuda(), want_out=True)
    return body, pooled.cpu().numpy(), out.cpu().numpy()


def _check(oracle, blocks, x, n, c, h, w, expect_fused):
    body, pooled, out = _run(blocks, x, n, c, h, w)
    assert body.fused == expect_fused
    st, want = oracle.net_body(blocks, x, n, c, h, w)
    assert st == 0
    assert out.shape == want.shape
    mism = np.count_nonzero(out.view(np.int32) != want.view(np.int32))
    assert mism == 0, f"{mism} of {out.size} body outputs differ"
    np.testing.assert_allclose(pooled, want.reshape(n, want.shape[1], -1).mean(-1), rtol=1e-5, atol=1e-5)
    assert (want > 0).mean() > 0.1
    return body, out


def test_generic_path_tiny_body(oracle):
    blocks, (n, c, h, w), x = tiny_body(seed=3)
    _check(oracle, blocks, x, n, c, h, w, expect_fused=False)


def fused_small(seed=0, n=3, h=16, w=16):
    rng = np.random.default_rng(seed)
    blocks = [
        dict(convs=[conv_spec(rng, 64, 64, 3, 1, 1), conv_spec(rng, 64, 64, 3, 1, 1, (0.45, 0.8))]),
        dict(convs=[conv_spec(rng, 64, 128, 3, 2, 1), conv_spec(rng, 128, 128, 3, 1, 1)],
             down=conv_spec(rng, 64, 128, 1, 2, 0)),
        dict(convs=[conv_spec(rng, 128, 64, 1, 1, 0), conv_spec(rng, 64, 64, 3, 1, 1, (0.4, 0.7)),
                    conv_spec(rng, 64, 128, 1, 1, 0)]),
        dict(convs=[conv_spec(rng, 128, 128, 1, 2, 0), conv_spec(rng, 128, 128, 3, 1, 1),
                    conv_spec(rng, 128, 256, 1, 1, 0)],
             down=conv_spec(rng, 128, 256, 1, 2, 0, (0.6, 1.0))),
        dict(convs=[conv_spec(rng, 256, 512, 3, 1, 1), conv_spec(rng, 512, 256, 3, 1, 1)]),
    ]
    x = np.abs(rng.standard_normal(n * 64 * h * w)).astype(np.float32)
    return blocks, (n, 64, h, w), x


def test_fused_path_small_body(oracle):
    """Basic, strided-with-downsample and bottleneck blocks (incl. a stride-2
    1x1, a 512-channel conv split over two N tiles and a downsample whose
    quantizer differs from its sibling conv's) through the fused kernels."""
    blocks, (n, c, h, w), x = fused_small()
    _check(oracle, blocks, x, n, c, h, w, expect_fused=True)


def _edge_conv(rng, in_c, out_c, k, pad, near, neg_gain):
    """A conv whose accumulators reach their extremes (weights all +1 or all
    -1 per row, a few zeros, on level-2 inputs: +-2 nnz at interior positions,
    kmax = 2 in_c k^2) and whose folded BN puts both quantizer thresholds
    within a few counts of them (alpha2 - alpha1 = 0.4 = 3 counts)."""
    K = in_c * k * k
    sign = rng.choice([1, -1], size=out_c, p=[0.75, 0.25]).astype(np.int8)
    w = np.repeat(sign[:, None], K, axis=1)
    w[:, ::97] = 0
    peak = 2 * np.count_nonzero(w, axis=1).astype(np.float64)  # |acc| at interior positions
    g = np.full(out_c, 0.4 / 3, np.float64)
    if neg_gain:
        g[::5] *= -1
    ta = (0.5, 0.9)
    j = np.arange(out_c)
    acc_t = np.where(sign > 0, peak - near - j % 7, -peak + j % 5)  # alpha1 crossing
    b = ta[0] - g * (acc_t + 0.5)
    return dict(in_c=in_c, out_c=out_c, k=k, stride=1, pad=pad, weights=w, ta=ta, tw=(1.0, 1.0),
                gain=g.astype(np.float32), bias=b.astype(np.float32), out_scale=1.0)


@pytest.mark.parametrize("neg_gain", [False, True])
def test_fused_extreme_accumulators(oracle, neg_gain):
    """Inner-conv integer thresholds at the accumulator extremes: 512-channel
    1x1 and 3x3 convs (kmax 1024 / 9216) on level-2 inputs with weights mostly
    +1 or -1, thresholds within a few counts of +-kmax -- the s16x2 DPX form
    (all gains positive) and the general signed form (some negative)."""
    rng = np.random.default_rng(11 + neg_gain)
    c, n, h, w = 512, 2, 6, 6
    blocks = [dict(convs=[_edge_conv(rng, c, c, 1, 0, 2, neg_gain), _edge_conv(rng, c, c, 3, 1, 2, neg_gain),
                          conv_spec(rng, c, c, 1, 1, 0)])]
    x = (2.0 + rng.random(n * c * h * w)).astype(np.float32)  # every level 2
    body, out = _check(oracle, blocks, x, n, c, h, w, expect_fused=True)


def _random_body(seed):
    """A random residual body the fused path accepts: basic or bottleneck
    blocks, 64/128/256/512 channels, stride-1/2 transitions with downsample,
    per-conv quantizer thresholds and BN drawn at random."""
    rng = np.random.default_rng(seed)
    c, h = 64, int(rng.choice([16, 24, 32]))
    blocks = []
    for _ in range(int(rng.integers(3, 6))):
        out = (2 * c if rng.random() < 0.6 else c) if c < 512 else c
        stride = 2 if out != c and h % 2 == 0 and h >= 8 else 1
        if stride == 1 and out != c:
            out = c
        ta = lambda: tuple(sorted(rng.uniform(0.3, 1.1, 2)))  # noqa: E731
        if rng.random() < 0.5:  # basic block
            convs = [conv_spec(rng, c, out, 3, stride, 1, ta()), conv_spec(rng, out, out, 3, 1, 1, ta())]
        else:  # bottleneck
            mid = max(64, out // 4) if out >= 256 else 64
            convs = [conv_spec(rng, c, mid, 1, 1, 0, ta()), conv_spec(rng, mid, mid, 3, stride, 1, ta()),
                     conv_spec(rng, mid, out, 1, 1, 0, ta())]
        blk = dict(convs=convs)
        if stride != 1 or out != c:
            blk["down"] = conv_spec(rng, c, out, 1, stride, 0, ta())
        blocks.append(blk)
        c, h = out, h // stride
    n = int(rng.integers(1, 4))
    h0 = h * 2 ** sum(1 for b in blocks if b.get("down") is not None and b["down"]["stride"] == 2)
    x = np.abs(rng.standard_normal(n * 64 * h0 * h0)).astype(np.float32)
    return blocks, (n, 64, h0, h0), x


@pytest.mark.parametrize("seed", [101, 202, 303, 404])
def test_fused_random_bodies(oracle, seed):
    """Random block structures through the fused kernels (every tiling rule:
    MT, column split, integer / DPX thresholds, resident vs streamed weights)
    bit-exact against the oracle."""
    blocks, (n, c, h, w), x = _random_body(seed)
    _check(oracle, blocks, x, n, c, h, w, expect_fused=True)


def test_fused_equals_generic(oracle):
    from paper_2008_05101_b200 import _lib as T
    blocks, (n, c, h, w), x = fused_small(seed=5, n=2, h=12, w=20)
    _, _, fused = _run(blocks, x, n, c, h, w, mode=T.TK_NET_AUTO)
    _, _, generic = _run(blocks, x, n, c, h, w, mode=T.TK_NET_GENERIC)
    assert np.array_equal(fused.view(np.int32), generic.view(np.int32))


def test_resnet18_body_subsample(oracle):
    """cfg4 network at full resolution (56x56 body input, 8 blocks), 2 images."""
    from paper_2008_05101_b200.resnet import resnet_spec
    blocks = resnet_spec(18, seed=0)
    rng = np.random.default_rng(1)
    x = np.maximum(rng.standard_normal(2 * 64 * 56 * 56), 0).astype(np.float32)
    _check(oracle, blocks, x, 2, 64, 56, 56, expect_fused=True)


def test_resnet50_body_subsample(oracle):
    """cfg5 network (16 bottleneck blocks), 1 image."""
    from paper_2008_05101_b200.resnet import resnet_spec
    blocks = resnet_spec(50, seed=0)
    rng = np.random.default_rng(2)
    x = np.maximum(rng.standard_normal(64 * 56 * 56), 0).astype(np.float32)
    _check(oracle, blocks, x, 1, 64, 56, 56, expect_fused=True)


def _full_batch_samples(oracle, depth, batch, images, seed):
    """The body exactly as the bench times it (one TernaryBody over the whole
    batch: persistent tile loop, late work items, the last partial M tile and
    the pad ring), sampled at the first, a middle and the last image."""
    from paper_2008_05101_b200.resnet import TernaryBody, resnet_spec
    blocks = resnet_spec(depth, seed=0)
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn((batch, 64, 56, 56), generator=g, device="cuda").relu_()
    body = TernaryBody(blocks, batch, 64, 56, 56)
    assert body.fused
    _, out = body.forward(x, want_out=True)
    got = out[images].cpu().numpy()
    del out
    xs = x[images].cpu().numpy()
    st, want = oracle.net_body(blocks, xs, len(images), 64, 56, 56)
    assert st == 0
    mism = np.count_nonzero(got.view(np.int32) != want.view(np.int32))
    assert mism == 0, f"{mism} of {got.size} body outputs differ"


def test_resnet18_full_batch_samples(oracle):
    """cfg4 at its timed batch (256): images 0, 127, 255 vs the oracle."""
    _full_batch_samples(oracle, 18, 256, [0, 127, 255], seed=11)


def test_resnet50_full_batch_samples(oracle):
    """cfg5 at its timed batch (1024 on one GPU): images 0, 511, 1023 vs the oracle."""
    _full_batch_samples(oracle, 50, 1024, [0, 511, 1023], seed=12)


def test_batch_independence_large_batch():
    """Images are independent: image i of a batch-64 run equals a batch-1 run."""
    from paper_2008_05101_b200.resnet import resnet_spec
    blocks = resnet_spec(18, seed=4)
    rng = np.random.default_rng(3)
    x = np.maximum(rng.standard_normal(64 * 64 * 56 * 56), 0).astype(np.float32)
    _, _, big = _run(blocks, x, 64, 64, 56, 56)
    for i in (0, 37, 63):
        _, _, one = _run(blocks, x.reshape(64, -1)[i].copy(), 1, 64, 56, 56)
        assert np.array_equal(big[i].view(np.int32), one[0].view(np.int32))


def test_net_errors(tk):
    from paper_2008_05101_b200.resnet import TernaryBody
    blocks, (n, c, h, w), x = fused_small(n=1)
    body = TernaryBody(blocks, n, c, h, w)
    xb = torch.from_numpy(x.reshape(n, c, h, w).copy()).cuda()
    xb[0, 5, 3, 3] = -1.0  # negative activation: R:quantizer.hpp:53-55
    with pytest.raises(tk.InvalidArgument):
        body.forward(xb)
    bad = [dict(convs=[conv_spec(np.random.default_rng(0), 64, 64, 3, 1, 1),
                       conv_spec(np.random.default_rng(0), 64, 32, 3, 1, 1)])]  # identity shape mismatch
    with pytest.raises(tk.InvalidArgument):
        TernaryBody(bad, 1, 64, 8, 8)


def test_pipelined_e2e_matches_serial_chunks(tk):
    """PipelinedResNet (chunked H2D overlapping compute) == the same chunks run
    serially through stem -> body -> head; stem pooling == torch reference."""
    from paper_2008_05101_b200.resnet import PipelinedResNet, TernaryBody, TernaryResNet
    net = TernaryResNet(18, 16, seed=3)
    pipe = PipelinedResNet(net, 16, chunks=4)
    g = torch.Generator().manual_seed(5)
    imgs = torch.rand(16, 3, 224, 224, generator=g).pin_memory()
    got = pipe.forward(imgs).clone()
    body4 = TernaryBody(net.blocks, 4, 64, 56, 56)
    pooled = torch.cat([body4.forward(net.stem(imgs[4 * i:4 * i + 4].cuda())) for i in range(4)])
    torch.cuda.synchronize()
    assert torch.equal(pipe.pooled, pooled)  # stem + ternary body, chunk by chunk: bit-exact
    assert torch.equal(got, net.head(pooled))  # (one head GEMM over the whole batch, as the pipeline does)
    # body launched on groups of 2 + 1 + 1 uploaded slices: the same bits
    pipe_g = PipelinedResNet(net, 16, chunks=4, groups=[2, 1, 1])
    got_g = pipe_g.forward(imgs).clone()
    torch.cuda.synchronize()
    assert torch.equal(pipe_g.pooled, pooled) and torch.equal(got_g, got)
    # back-to-back calls without a host sync (the next upload overlaps this
    # call's last body and head): each call's logits are its own
    imgs2 = torch.rand(16, 3, 224, 224, generator=g).pin_memory()
    want2 = pipe.forward(imgs2).clone()
    torch.cuda.synchronize()
    outs = []
    for im in (imgs, imgs2, imgs, imgs2):
        outs.append(pipe.forward(im).clone())
    torch.cuda.synchronize()
    assert all(torch.equal(o, w) for o, w in zip(outs, (got, want2, got, want2)))
    # uneven slices (4 + 8 + 4 images), bodies on 12 + 4 images: the same bits
    pipe_u = PipelinedResNet(net, 16, groups=[2, 1], slices=[4, 8, 4])
    got_u = pipe_u.forward(imgs).clone()
    torch.cuda.synchronize()
    assert torch.equal(pipe_u.pooled, pooled) and torch.equal(got_u, got)
    # stem (split-TF32 conv, fused affine + ReLU + max-pool) vs fp64: within
    # the conv's stated bound (4e-6 x sum |x||w|, here <= ~8) x max |gain|
    x = imgs[:2].cuda().double()
    y = torch.nn.functional.conv2d(x, net.stem_w.double(), stride=2, padding=3)
    ref = torch.nn.functional.max_pool2d(torch.relu(torch.addcmul(net.stem_bias.double().view(1, -1, 1, 1), y,
                                                                  net.stem_gain.double().view(1, -1, 1, 1))), 3, 2, 1)
    scale = torch.nn.functional.conv2d(x.abs(), net.stem_w.double().abs(), stride=2, padding=3).max().item()
    err = (net.stem(imgs[:2].cuda()).double() - ref).abs().max().item()
    assert err <= 4e-6 * scale * net.stem_gain.abs().max().item() + 1e-6, err


def test_stem_conv_matches_fp32_reference(tk):
    """tk_stem_conv7x7s2 (split-TF32: x_hi w_hi + x_hi w_lo + x_lo w_hi, f32
    accumulation) vs an fp64 conv: error <= 4e-6 x sum |x||w| per output (fp32
    class; measured 1.4e-6), on positive and mixed-sign inputs and odd sizes."""
    from paper_2008_05101_b200.resnet import TernaryResNet
    from paper_2008_05101_b200 import _lib as T
    net = TernaryResNet(18, 2, seed=1)
    g = torch.Generator(device="cuda").manual_seed(2)
    for (n, h, w, lo) in ((3, 224, 224, 0.0), (2, 224, 224, -1.0), (2, 37, 51, -1.0), (1, 9, 240, 0.0)):
        x = torch.rand(n, 3, h, w, device="cuda", generator=g) * (1 - lo) + lo
        ho, wo = (h - 1) // 2 + 1, (w - 1) // 2 + 1
        y = torch.full((n, 64, ho, wo), float("nan"), device="cuda")
        T.check(T.lib().tk_stem_conv7x7s2(tk.context(), x.data_ptr(), n, h, w, net.stem_w.data_ptr(),
                                          y.data_ptr(), tk._stream()), "stem")
        ref = torch.nn.functional.conv2d(x.double(), net.stem_w.double(), stride=2, padding=3)
        scale = torch.nn.functional.conv2d(x.double().abs(), net.stem_w.double().abs(), stride=2, padding=3)
        assert ((y.double() - ref).abs() <= 4e-6 * scale + 1e-30).all(), (n, h, w)
    # wider than one band of the kernel: refused, not silently wrong; n = 0 is a no-op
    x = torch.rand(1, 3, 8, 256, device="cuda")
    y = torch.empty(1, 64, 4, 128, device="cuda")
    assert T.lib().tk_stem_conv7x7s2(tk.context(), x.data_ptr(), 1, 8, 256, net.stem_w.data_ptr(), y.data_ptr(),
                                     tk._stream()) == T.TK_ERR_UNSUPPORTED
    assert T.lib().tk_stem_conv7x7s2(tk.context(), x.data_ptr(), 0, 8, 240, net.stem_w.data_ptr(), y.data_ptr(),
                                     tk._stream()) == T.TK_OK


def test_dense_head_matches_fp64(tk):
    """tk_dense_f32 (the ResNet head, one fp32 FMA chain per logit) vs an fp64
    matmul, ragged tiles included."""
    from paper_2008_05101_b200 import _lib as T
    for (b, k, o) in ((256, 512, 1000), (5, 2048, 70), (64, 17, 64)):
        x = torch.randn(b, k, device="cuda")
        w = torch.randn(o, k, device="cuda") / k ** 0.5
        bias = torch.randn(o, device="cuda")
        y = torch.empty(b, o, device="cuda")
        T.check(T.lib().tk_dense_f32(tk.context(), x.data_ptr(), w.data_ptr(), bias.data_ptr(), b, k, o,
                                     y.data_ptr(), tk._stream()), "dense")
        ref = x.double() @ w.double().t() + bias.double()
        scale = x.double().abs() @ w.double().abs().t() + bias.double().abs()
        assert ((y.double() - ref).abs() / scale).max().item() < k * 1.2e-7
