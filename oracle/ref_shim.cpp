// ref_shim.cpp -- extern "C" bindings over the UNMODIFIED reference headers.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file
// against /root/reference/proj/include (read in place, never copied) with the
// reference's own default flags (-std=gnu++20 -O3 -march=..., R:CMakeLists.txt
// :3-20) into oracle/_ref/libternkit_ref_<isa>.so.  The tests use it to pin
// the C restatement (oracle/ternkit_oracle.c) and to make tests/golden/; the
// bench's `--impl reference` arm times it as the reference CPU implementation.
// Nothing on the product path links it.
//
// Every entry converts reference exceptions (std::invalid_argument) into the
// status codes of include/ternkit_b200.h.

#include <chrono>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "ternkit/bench.hpp"
#include "ternkit/bitkernels.hpp"
#include "ternkit/codec.hpp"
#include "ternkit/linalg.hpp"
#include "ternkit/model_io.hpp"
#include "ternkit/quantizer.hpp"
#include "ternkit/tinynet.hpp"

#include "netdesc.h"

using namespace ternkit;

namespace {

constexpr int kOk = 0, kInvalid = 1, kNonfinite = 4, kNegative = 5;

template <class F>
int guard(F&& f) {
  try {
    f();
    return kOk;
  } catch (const std::invalid_argument& e) {
    const std::string m = e.what();
    if (m.find("not finite") != std::string::npos) return kNonfinite;
    if (m.find("p >= 0") != std::string::npos) return kNegative;
    return kInvalid;
  } catch (...) {
    return 99;
  }
}

QuantMode qmode(int mode) {
  return mode == 0 ? QuantMode::kWeight : QuantMode::kActivationNonneg;
}

PackedConvLayer build_layer(const nd_conv& c) {
  ConvGeometry g{c.in_c, c.out_c, c.k, c.k, c.stride, c.pad};
  ChannelAffine aff;
  if (c.gain) {
    aff.gain.assign(c.gain, c.gain + c.out_c);
    aff.bias.assign(c.bias, c.bias + c.out_c);
  }
  std::span<const std::int8_t> w(c.weights,
                                 static_cast<std::size_t>(c.out_c) * g.patch_len());
  return make_packed_conv_layer(w, g, {c.tw1, c.tw2}, {c.ta1, c.ta2}, true,
                                std::move(aff), c.out_scale);
}

struct RefBlock {
  std::vector<PackedConvLayer> convs;
  bool has_down = false;
  PackedConvLayer down;
};

struct RefNet {
  std::vector<RefBlock> blocks;
};

// One image (or one batch) through the body with the reference's own calls.
std::vector<float> run_body(const RefNet& net, std::vector<float> x,
                            TensorShape shape, TensorShape* out_shape) {
  for (const RefBlock& b : net.blocks) {
    std::vector<float> h = x;
    TensorShape hs = shape;
    ConvResult z;
    for (std::size_t i = 0; i < b.convs.size(); ++i) {
      z = conv2d_ternary(h, hs, b.convs[i]);
      if (i + 1 < b.convs.size()) {
        for (auto& v : z.data) v = std::max(v, 0.0f);
        h = std::move(z.data);
        hs = z.shape;
      }
    }
    std::vector<float> sc;
    if (b.has_down) {
      sc = conv2d_ternary(x, shape, b.down).data;
    } else {
      sc = std::move(x);
    }
    if (sc.size() != z.data.size()) throw std::invalid_argument("shortcut shape");
    for (std::size_t i = 0; i < sc.size(); ++i) {
      z.data[i] = std::max(z.data[i] + sc[i], 0.0f);  // R:tinynet.hpp:727
    }
    x = std::move(z.data);
    shape = z.shape;
  }
  if (out_shape) *out_shape = shape;
  return x;
}

}  // namespace

extern "C" {

int ref_quantize_weight_value(float p, float a1, float a2, int* level) {
  return guard([&] { *level = quantize_weight_value(p, {a1, a2}); });
}

int ref_quantize_activation_value(float p, float a1, float a2, int* level) {
  return guard([&] { *level = quantize_activation_value(p, {a1, a2}); });
}

int ref_pack(const std::int8_t* v, std::size_t n, std::uint64_t* words) {
  return guard([&] {
    PackedTernaryVector p = pack(std::span<const std::int8_t>(v, n));
    std::memcpy(words, p.words.data(), p.words.size() * 8);
  });
}

int ref_quantize_and_pack(const float* x, std::size_t n, float a1, float a2,
                          int mode, std::uint64_t* words) {
  return guard([&] {
    PackedTernaryVector p =
        quantize_and_pack(std::span<const float>(x, n), {a1, a2}, qmode(mode));
    std::memcpy(words, p.words.data(), p.words.size() * 8);
  });
}

std::uint64_t ref_ternary_multiply_word(std::uint64_t x, std::uint64_t y) {
  return ternary_multiply_word(x, y);
}

// out[p] = ternary_dot(x_p, y_p), or ternary_dot_nonneg when wsum != NULL
int ref_ternary_dot_batched(const std::uint64_t* x, const std::uint64_t* y,
                            std::size_t lanes, std::size_t pairs,
                            const std::int64_t* wsum, std::int64_t* out) {
  return guard([&] {
    const std::size_t nw = words_for_lanes(lanes);
    PackedTernaryVector a, b;
    a.logical_len = b.logical_len = lanes;
    a.nonneg_offset = wsum != nullptr;
    for (std::size_t p = 0; p < pairs; ++p) {
      a.words.assign(x + p * nw, x + (p + 1) * nw);
      b.words.assign(y + p * nw, y + (p + 1) * nw);
      out[p] = wsum ? ternary_dot_nonneg(a, b, wsum[p]) : ternary_dot(a, b);
    }
  });
}

int ref_im2col_quantize_pack(const float* x, int n, int c, int h, int w, int kh,
                             int kw, int stride, int pad, float a1, float a2,
                             int mode, std::uint64_t* rows) {
  return guard([&] {
    const TensorShape s{n, c, h, w};
    const ConvGeometry g{c, 1, kh, kw, stride, pad};
    Im2colBuffer buf = im2col_quantize_pack(std::span<const float>(x, s.count()),
                                            s, {a1, a2}, g, qmode(mode));
    std::memcpy(rows, buf.words.data(), buf.words.size() * 8);
  });
}

// packed_gemm on rows produced by im2col_quantize_pack of the given input.
int ref_conv_gemm(const float* x, int n, int c, int h, int w, const std::int8_t* wq,
                  int out_c, int k, int stride, int pad, float ta1, float ta2,
                  int nonneg, int mask_mode, int workers, std::int32_t* out) {
  return guard([&] {
    const TensorShape s{n, c, h, w};
    const ConvGeometry g{c, out_c, k, k, stride, pad};
    PackedConvLayer layer = make_packed_conv_layer(
        std::span<const std::int8_t>(wq, static_cast<std::size_t>(out_c) * g.patch_len()),
        g, {1, 1}, {ta1, ta2}, nonneg != 0);
    if (mask_mode) layer.precompute_masks();
    Im2colBuffer buf = im2col_quantize_pack(
        std::span<const float>(x, s.count()), s, {ta1, ta2}, g,
        nonneg ? QuantMode::kActivationNonneg : QuantMode::kWeight);
    std::vector<std::int32_t> r = packed_gemm(
        buf, layer, mask_mode ? MaskMode::kPrecomputed : MaskMode::kOnTheFly, workers);
    std::memcpy(out, r.data(), r.size() * 4);
  });
}

int ref_conv2d_ternary(const float* x, int n, int c, int h, int w,
                       const nd_conv* conv, int nonneg, int workers, float* out) {
  return guard([&] {
    nd_conv cc = *conv;
    const ConvGeometry g{cc.in_c, cc.out_c, cc.k, cc.k, cc.stride, cc.pad};
    ChannelAffine aff;
    if (cc.gain) {
      aff.gain.assign(cc.gain, cc.gain + cc.out_c);
      aff.bias.assign(cc.bias, cc.bias + cc.out_c);
    }
    PackedConvLayer layer = make_packed_conv_layer(
        std::span<const std::int8_t>(cc.weights,
                                     static_cast<std::size_t>(cc.out_c) * g.patch_len()),
        g, {cc.tw1, cc.tw2}, {cc.ta1, cc.ta2}, nonneg != 0, std::move(aff),
        cc.out_scale);
    const TensorShape s{n, c, h, w};
    ConvResult r = conv2d_ternary(std::span<const float>(x, s.count()), s, layer,
                                  MaskMode::kOnTheFly, workers);
    std::memcpy(out, r.data.data(), r.data.size() * 4);
  });
}

int ref_fully_connected_ternary(const float* x, int batch, const nd_conv* conv,
                                int nonneg, float* out) {
  return guard([&] {
    nd_conv cc = *conv;
    const ConvGeometry g{cc.in_c, cc.out_c, cc.k, cc.k, cc.stride, cc.pad};
    ChannelAffine aff;
    if (cc.gain) {
      aff.gain.assign(cc.gain, cc.gain + cc.out_c);
      aff.bias.assign(cc.bias, cc.bias + cc.out_c);
    }
    PackedConvLayer layer = make_packed_conv_layer(
        std::span<const std::int8_t>(cc.weights,
                                     static_cast<std::size_t>(cc.out_c) * g.patch_len()),
        g, {cc.tw1, cc.tw2}, {cc.ta1, cc.ta2}, nonneg != 0, std::move(aff),
        cc.out_scale);
    std::vector<float> r = fully_connected_ternary(
        std::span<const float>(x, static_cast<std::size_t>(batch) * cc.in_c), batch,
        layer);
    std::memcpy(out, r.data(), r.size() * 4);
  });
}

int ref_fuse_bn(const float* mean, const float* var, const float* gamma,
                const float* beta, float eps, int c, float* gain, float* bias) {
  return guard([&] {
    ChannelAffine a = fuse_bn(std::span<const float>(mean, c),
                              std::span<const float>(var, c),
                              std::span<const float>(gamma, c),
                              std::span<const float>(beta, c), eps);
    std::memcpy(gain, a.gain.data(), c * 4);
    std::memcpy(bias, a.bias.data(), c * 4);
  });
}

// packed_forward (R:tinynet.hpp:713-735) over a PackedModel assembled from
// raw arrays: float stem, `n_blocks` hidden x hidden ternary FC blocks with
// optional calibration affine, float head.
int ref_packed_forward(const float* x, int batch, int in_dim, int hidden,
                       int n_classes, const float* stem_w, const float* stem_b,
                       int n_blocks, const nd_conv* blocks, const float* cal_gain,
                       const float* cal_bias, const float* head_w,
                       const float* head_b, float* logits) {
  return guard([&] {
    PackedModel m;
    m.in_dim = in_dim;
    m.hidden = hidden;
    m.n_classes = n_classes;
    m.stem_w.assign(stem_w, stem_w + static_cast<std::size_t>(hidden) * in_dim);
    m.stem_b.assign(stem_b, stem_b + hidden);
    m.head_w.assign(head_w, head_w + static_cast<std::size_t>(n_classes) * hidden);
    m.head_b.assign(head_b, head_b + n_classes);
    for (int i = 0; i < n_blocks; ++i) {
      PackedBlock pb;
      pb.layer = build_layer(blocks[i]);
      if (cal_gain) {
        pb.has_calibration = true;
        pb.cal_gain.assign(cal_gain + static_cast<std::size_t>(i) * hidden,
                           cal_gain + static_cast<std::size_t>(i + 1) * hidden);
        pb.cal_bias.assign(cal_bias + static_cast<std::size_t>(i) * hidden,
                           cal_bias + static_cast<std::size_t>(i + 1) * hidden);
      }
      m.blocks.push_back(std::move(pb));
    }
    std::vector<float> r = packed_forward(
        m, std::span<const float>(x, static_cast<std::size_t>(batch) * in_dim), batch);
    std::memcpy(logits, r.data(), r.size() * 4);
  });
}

// The same model written as a FATN file by the reference's own serializer
// (R:model_io.hpp:151-207), for the loader fixtures of tests/golden.
int ref_save_packed_model(const char* path, int in_dim, int hidden, int n_classes, const float* stem_w,
                          const float* stem_b, int n_blocks, const nd_conv* blocks, const float* cal_gain,
                          const float* cal_bias, const float* head_w, const float* head_b) {
  return guard([&] {
    PackedModel m;
    m.in_dim = in_dim;
    m.hidden = hidden;
    m.n_classes = n_classes;
    m.stem_w.assign(stem_w, stem_w + static_cast<std::size_t>(hidden) * in_dim);
    m.stem_b.assign(stem_b, stem_b + hidden);
    m.head_w.assign(head_w, head_w + static_cast<std::size_t>(n_classes) * hidden);
    m.head_b.assign(head_b, head_b + n_classes);
    for (int i = 0; i < n_blocks; ++i) {
      PackedBlock pb;
      pb.layer = build_layer(blocks[i]);
      if (cal_gain) {
        pb.has_calibration = true;
        pb.cal_gain.assign(cal_gain + static_cast<std::size_t>(i) * hidden,
                           cal_gain + static_cast<std::size_t>(i + 1) * hidden);
        pb.cal_bias.assign(cal_bias + static_cast<std::size_t>(i) * hidden,
                           cal_bias + static_cast<std::size_t>(i + 1) * hidden);
      }
      m.blocks.push_back(std::move(pb));
    }
    save_model(m, path);
  });
}

// load_model + packed_forward with the reference's own code (R:model_io.hpp:
// 209-301, R:tinynet.hpp:713-735)
int ref_load_and_forward(const char* path, const float* x, int batch, float* logits, int* n_classes) {
  return guard([&] {
    PackedModel m = load_model(path);
    std::vector<float> r = packed_forward(m, std::span<const float>(x, static_cast<std::size_t>(batch) * m.in_dim),
                                          batch);
    std::memcpy(logits, r.data(), r.size() * 4);
    *n_classes = m.n_classes;
  });
}

// ---- paper baselines (R:bitkernels.hpp:99-224) ----
int ref_pack_binary(const std::int8_t* v, std::size_t n, std::uint64_t* words) {
  return guard([&] {
    PackedBinaryVector p = pack_binary(std::span<const std::int8_t>(v, n));
    std::memcpy(words, p.words.data(), p.words.size() * 8);
  });
}

int ref_binary_dot(const std::uint64_t* x, const std::uint64_t* y, std::size_t words, std::size_t logical_len,
                   std::int64_t* out) {
  return guard([&] {
    PackedBinaryVector a, b;
    a.words.assign(x, x + words);
    b.words.assign(y, y + words);
    a.logical_len = b.logical_len = logical_len;
    *out = binary_dot(a, b);
  });
}

int ref_multibit_dot(const std::uint64_t* x, int m, const std::uint64_t* y, int k, const double* sx,
                     const double* sy, std::size_t words, std::size_t logical_len, double* out) {
  return guard([&] {
    MultiBitVector a, b;
    for (int i = 0; i < m; ++i) {
      PackedBinaryVector p;
      p.words.assign(x + i * words, x + (i + 1) * words);
      p.logical_len = logical_len;
      a.planes.push_back(std::move(p));
      a.scales.push_back(sx[i]);
    }
    for (int i = 0; i < k; ++i) {
      PackedBinaryVector p;
      p.words.assign(y + i * words, y + (i + 1) * words);
      p.logical_len = logical_len;
      b.planes.push_back(std::move(p));
      b.scales.push_back(sy[i]);
    }
    *out = multibit_dot(a, b);
  });
}

// ---- network body (ResNet-shaped residual blocks) ----

void* ref_net_create(const nd_block* blocks, int n_blocks) {
  RefNet* net = new RefNet;
  try {
    for (int i = 0; i < n_blocks; ++i) {
      RefBlock rb;
      for (int j = 0; j < blocks[i].n_convs; ++j)
        rb.convs.push_back(build_layer(blocks[i].conv[j]));
      rb.has_down = blocks[i].has_down != 0;
      if (rb.has_down) rb.down = build_layer(blocks[i].down);
      net->blocks.push_back(std::move(rb));
    }
  } catch (...) {
    delete net;
    return nullptr;
  }
  return net;
}

void ref_net_destroy(void* h) { delete static_cast<RefNet*>(h); }

// Runs `n` images through the body, images sharded over `threads` host
// threads (images are independent, R:tests/test_linalg.cpp:289-304); every
// image goes through the reference's conv2d_ternary with workers = 1.
// Returns the wall time of the run in *seconds (timing harness only).
int ref_net_run(void* h, const float* x, int n, int c, int hh, int ww,
                int threads, float* out, double* seconds) {
  const RefNet& net = *static_cast<RefNet*>(h);
  const std::size_t in_img = static_cast<std::size_t>(c) * hh * ww;
  // probe output geometry on image 0 lazily inside workers
  std::vector<int> status(threads > 0 ? threads : 1, kOk);
  std::size_t out_img = 0;
  {
    // output size per image from the block list (cheap geometry walk)
    int ch = c, H = hh, W = ww;
    for (const RefBlock& b : net.blocks) {
      for (const auto& l : b.convs) {
        H = l.geom.out_h(H);
        W = l.geom.out_w(W);
        ch = l.geom.out_c;
      }
    }
    out_img = static_cast<std::size_t>(ch) * H * W;
  }
  const int nt = threads > 0 ? threads : 1;
  auto t0 = std::chrono::steady_clock::now();
  auto work = [&](int t) {
    status[t] = guard([&] {
      for (int i = t; i < n; i += nt) {
        std::vector<float> xi(x + i * in_img, x + (i + 1) * in_img);
        std::vector<float> y = run_body(net, std::move(xi), {1, c, hh, ww}, nullptr);
        if (out) std::memcpy(out + i * out_img, y.data(), out_img * 4);
      }
    });
  };
  if (nt == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
  }
  if (seconds)
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  for (int s : status)
    if (s != kOk) return s;
  return kOk;
}

// Times packed_gemm on a fixed im2col buffer (the FC GEMM of cfg3) using the
// reference's own worker threads.  Returns seconds per call over `iters`.
int ref_time_fc_gemm(const float* x, int batch, int in_c, const std::int8_t* wq,
                     int out_c, float ta1, float ta2, int workers, int iters,
                     double* seconds_per_call, std::int32_t* out) {
  return guard([&] {
    const TensorShape s{batch, in_c, 1, 1};
    const ConvGeometry g{in_c, out_c, 1, 1, 1, 0};
    PackedConvLayer layer = make_packed_conv_layer(
        std::span<const std::int8_t>(wq, static_cast<std::size_t>(out_c) * in_c), g,
        {1, 1}, {ta1, ta2}, true);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::int32_t> r;
    for (int i = 0; i < iters; ++i) {
      Im2colBuffer buf = im2col_quantize_pack(std::span<const float>(x, s.count()), s,
                                              {ta1, ta2}, g,
                                              QuantMode::kActivationNonneg);
      r = packed_gemm(buf, layer, MaskMode::kOnTheFly, workers);
    }
    *seconds_per_call =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() /
        iters;
    if (out) std::memcpy(out, r.data(), r.size() * 4);
  });
}

// cfg1 timing: `pairs` ternary_dot_nonneg calls (R:bitkernels.hpp:151-159) on
// vectors packed once up front, pairs sharded over `threads` host threads
// (the reference's dot is single-threaded; pairs are independent).
int ref_time_dot(const std::uint64_t* x, const std::uint64_t* y, std::size_t lanes,
                 std::size_t pairs, const std::int64_t* wsum, int threads,
                 double* seconds, std::int64_t* out) {
  return guard([&] {
    const std::size_t nw = words_for_lanes(lanes);
    std::vector<PackedTernaryVector> xs(pairs), ys(pairs);
    for (std::size_t p = 0; p < pairs; ++p) {
      xs[p].words.assign(x + p * nw, x + (p + 1) * nw);
      ys[p].words.assign(y + p * nw, y + (p + 1) * nw);
      xs[p].logical_len = ys[p].logical_len = lanes;
      xs[p].nonneg_offset = true;
    }
    std::vector<std::int64_t> r(pairs);
    const int nt = threads > 0 ? threads : 1;
    auto t0 = std::chrono::steady_clock::now();
    auto work = [&](int t) {  // contiguous ranges: no false sharing on r[]
      const std::size_t lo = pairs * t / nt, hi = pairs * (t + 1) / nt;
      for (std::size_t p = lo; p < hi; ++p) r[p] = ternary_dot_nonneg(xs[p], ys[p], wsum[p]);
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (out) std::memcpy(out, r.data(), pairs * 8);
  });
}

// cfg2 timing: conv2d_ternary (R:linalg.hpp:301-328) with the reference's own
// worker threads on a layer built once; seconds per call over `iters`.
int ref_time_conv(const float* x, int n, int c, int h, int w, const nd_conv* conv,
                  int workers, int iters, double* seconds_per_call, float* out) {
  return guard([&] {
    PackedConvLayer layer = build_layer(*conv);
    const TensorShape s{n, c, h, w};
    ConvResult r;
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < iters; ++i)
      r = conv2d_ternary(std::span<const float>(x, s.count()), s, layer, MaskMode::kOnTheFly,
                         workers);
    *seconds_per_call =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / iters;
    if (out) std::memcpy(out, r.data.data(), r.data.size() * 4);
  });
}

// ---- A10: the reference's own layer build (R:linalg.hpp:118-144) ----
// Packed weight rows ([out_c][words] u64, byte for byte) and weight sums.
int ref_make_packed_conv_layer(const std::int8_t* wq, int in_c, int out_c, int kh, int kw,
                               std::uint64_t* words, std::int32_t* wsums) {
  return guard([&] {
    const ConvGeometry g{in_c, out_c, kh, kw, 1, 0};
    PackedConvLayer layer = make_packed_conv_layer(
        std::span<const std::int8_t>(wq, static_cast<std::size_t>(out_c) * g.patch_len()), g,
        {1, 1}, {1, 1}, true);
    const std::size_t nw = words_for_lanes(g.patch_len());
    for (int o = 0; o < out_c; ++o) {
      std::memcpy(words + o * nw, layer.weights[o].words.data(), nw * 8);
      wsums[o] = layer.weight_sums[o];
    }
  });
}

// ---- CPU-baseline protocol: the reference's own time_runs (R:bench.hpp:64-99:
// `warmup` discarded runs, each measured run looped to >= min_run_s, mean /
// stddev / median over `repeats`, stable = stddev <= 15% of the mean) ----
struct ref_run_stats {
  double mean_us, stddev_us, median_us;
  int stable, repeats, warmup;
  double min_run_s;
};

static void fill_stats(const RunStats& r, int repeats, int warmup, double min_run_s,
                       ref_run_stats* st) {
  st->mean_us = r.mean_us;
  st->stddev_us = r.stddev_us;
  st->median_us = r.median_us;
  st->stable = r.stable ? 1 : 0;
  st->repeats = repeats;
  st->warmup = warmup;
  st->min_run_s = min_run_s;
}

// one call = the ResNet body on n images over `threads` host threads (ref_net_run)
int ref_time_runs_net(void* h, const float* x, int n, int c, int hh, int ww, int threads,
                      int repeats, int warmup, double min_run_s, ref_run_stats* st) {
  int status = kOk;
  RunStats r = time_runs([&] {
    int s = ref_net_run(h, x, n, c, hh, ww, threads, nullptr, nullptr);
    if (s != kOk) status = s;
  }, repeats, warmup, min_run_s);
  fill_stats(r, repeats, warmup, min_run_s, st);
  return status;
}

// one call = im2col_quantize_pack + packed_gemm(workers) of the FC (cfg3)
int ref_time_runs_fc(const float* x, int batch, int in_c, const std::int8_t* wq, int out_c,
                     float ta1, float ta2, int workers, int repeats, int warmup,
                     double min_run_s, ref_run_stats* st) {
  return guard([&] {
    const TensorShape s{batch, in_c, 1, 1};
    const ConvGeometry g{in_c, out_c, 1, 1, 1, 0};
    PackedConvLayer layer = make_packed_conv_layer(
        std::span<const std::int8_t>(wq, static_cast<std::size_t>(out_c) * in_c), g,
        {1, 1}, {ta1, ta2}, true);
    RunStats r = time_runs([&] {
      Im2colBuffer buf = im2col_quantize_pack(std::span<const float>(x, s.count()), s,
                                              {ta1, ta2}, g, QuantMode::kActivationNonneg);
      std::vector<std::int32_t> o = packed_gemm(buf, layer, MaskMode::kOnTheFly, workers);
    }, repeats, warmup, min_run_s);
    fill_stats(r, repeats, warmup, min_run_s, st);
  });
}

// one call = conv2d_ternary(workers) on the whole input (cfg2)
int ref_time_runs_conv(const float* x, int n, int c, int h, int w, const nd_conv* conv,
                       int workers, int repeats, int warmup, double min_run_s,
                       ref_run_stats* st) {
  return guard([&] {
    PackedConvLayer layer = build_layer(*conv);
    const TensorShape s{n, c, h, w};
    RunStats r = time_runs([&] {
      ConvResult o = conv2d_ternary(std::span<const float>(x, s.count()), s, layer,
                                    MaskMode::kOnTheFly, workers);
    }, repeats, warmup, min_run_s);
    fill_stats(r, repeats, warmup, min_run_s, st);
  });
}

// one call = `pairs` ternary_dot_nonneg over `threads` host threads (cfg1),
// vectors packed once outside the timed calls
int ref_time_runs_dot(const std::uint64_t* x, const std::uint64_t* y, std::size_t lanes,
                      std::size_t pairs, const std::int64_t* wsum, int threads, int repeats,
                      int warmup, double min_run_s, ref_run_stats* st) {
  return guard([&] {
    const std::size_t nw = words_for_lanes(lanes);
    std::vector<PackedTernaryVector> xs(pairs), ys(pairs);
    for (std::size_t p = 0; p < pairs; ++p) {
      xs[p].words.assign(x + p * nw, x + (p + 1) * nw);
      ys[p].words.assign(y + p * nw, y + (p + 1) * nw);
      xs[p].logical_len = ys[p].logical_len = lanes;
      xs[p].nonneg_offset = true;
    }
    std::vector<std::int64_t> r(pairs);
    const int nt = threads > 0 ? threads : 1;
    auto work = [&](int t) {
      const std::size_t lo = pairs * t / nt, hi = pairs * (t + 1) / nt;
      for (std::size_t p = lo; p < hi; ++p) r[p] = ternary_dot_nonneg(xs[p], ys[p], wsum[p]);
    };
    RunStats rs = time_runs([&] {
      std::vector<std::thread> pool;
      for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
      work(0);
      for (auto& th : pool) th.join();
    }, repeats, warmup, min_run_s);
    fill_stats(rs, repeats, warmup, min_run_s, st);
  });
}

}  // extern "C"
