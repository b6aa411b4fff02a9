"""FATN packed models: the reference's file format and its
packed_forward on the GPU.  Fixtures tests/golden/pf_{cal,nocal}.fatn were
written by the reference's own serializer (oracle/make_golden.py), and the
reference's load_model + packed_forward produced golden["pf_logits*"]."""
import os
import struct

import numpy as np
import pytest

from paper_2008_05101_b200.model import ParseError, decode_words, parse_model, serialize_model

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def fixture(tag):
    with open(os.path.join(GOLD, f"pf_{tag}.fatn"), "rb") as f:
        return f.read()


@pytest.mark.parametrize("tag", ["cal", "nocal"])
def test_parse_and_byte_identical_round_trip(golden, tag):
    data = fixture(tag)
    m = parse_model(data)
    batch, in_dim, hidden, ncls, nb = map(int, golden["pf_dims"])
    assert (m.in_dim, m.hidden, m.n_classes, len(m.blocks)) == (in_dim, hidden, ncls, nb)
    assert np.array_equal(m.stem_w, golden["pf_stem_w"]) and np.array_equal(m.head_w, golden["pf_head_w"])
    for i, b in enumerate(m.blocks):
        assert np.array_equal(decode_words(b.words, b.patch_len), golden[f"pf_b{i}_w"])
        assert np.array_equal(b.weight_sums, golden[f"pf_b{i}_w"].astype(np.int32).sum(axis=1))
        assert (b.cal_gain is not None) == (tag == "cal") and b.nonneg
    assert serialize_model(m) == data  # R:docs/format.md: save/load/save is byte-identical


def test_decode_words_matches_oracle(oracle):
    rng = np.random.default_rng(3)
    v = rng.integers(-1, 2, 77).astype(np.int8)
    st, w = oracle.pack(v)
    assert np.array_equal(decode_words(w, 77), v)
    # the non-canonical zero code 0b10 decodes to 0 (R:codec.hpp:38-40)
    assert decode_words(np.array([0b10], np.uint64), 1)[0] == 0


def test_parse_errors_mirror_the_reference():
    good = fixture("cal")
    cases = {
        "bad model magic": b"FATX" + good[4:],
        "unsupported model version": good[:4] + struct.pack("<I", 2) + good[8:],
        "model needs stem and head": good[:8] + struct.pack("<I", 1) + good[12:],
        "trailing bytes": good + b"\0",
        "unexpected end of file": good[:-3],
    }
    for msg, data in cases.items():
        with pytest.raises(ParseError, match=msg):
            parse_model(data)
    # first block record starts after the stem record; corrupt its packed byte count
    m = parse_model(good)
    stem_len = 2 + 24 + 4 * (m.in_dim * m.hidden + m.hidden)
    b0 = m.blocks[0]
    off = 12 + stem_len + 2 + 24 + 20 + 8 * b0.out_c + 8 * b0.in_c + 4 * b0.out_c
    bad = good[:off] + struct.pack("<Q", b0.words.size * 8 + 8) + good[off + 8:]
    with pytest.raises(ParseError, match="byte count mismatch"):
        parse_model(bad)
    bad_tag = good[:12] + b"\x07" + good[13:]
    with pytest.raises(ParseError, match="unknown layer tag"):
        parse_model(bad_tag)


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["cal", "nocal"])
def test_packed_forward_gpu_matches_reference(tk, golden, tag):
    from paper_2008_05101_b200.model import PackedModel, argmax_rows, packed_forward
    m = PackedModel(parse_model(fixture(tag)))
    batch = int(golden["pf_dims"][0])
    logits = packed_forward(m, golden["pf_x"], batch).cpu().numpy()
    want = golden["pf_logits" if tag == "cal" else "pf_logits_nocal"]
    assert np.array_equal(logits.view(np.int32), want.view(np.int32))
    assert np.array_equal(argmax_rows(logits), want.argmax(axis=1))


@pytest.mark.gpu
def test_packed_forward_rejects_block_width_mismatch(tk, golden):
    """A block whose width differs from `hidden` is an InvalidArgument (the
    reference's FC size check, R:linalg.hpp:332-343), never an out-of-bounds
    residual add."""
    import dataclasses
    from paper_2008_05101_b200.model import PackedModel, packed_forward
    spec = parse_model(fixture("nocal"))
    b0 = spec.blocks[0]
    out_c = b0.out_c - 1
    wpr = b0.words.shape[1]
    narrow = dataclasses.replace(b0, out_c=out_c, words=b0.words[:out_c].copy(), weight_sums=b0.weight_sums[:out_c],
                                 gain=b0.gain[:out_c], bias=b0.bias[:out_c])
    assert narrow.words.shape == (out_c, wpr)
    m = PackedModel(dataclasses.replace(spec, blocks=[narrow] + spec.blocks[1:]))
    batch = int(golden["pf_dims"][0])
    with pytest.raises(tk.InvalidArgument):
        packed_forward(m, golden["pf_x"], batch)
