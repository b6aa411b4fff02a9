// ternkit_b200/ternkit.hpp -- drop-in C++ front end of the B200 library.
//
// Mirrors the reference's header-only API (namespace ternkit, same type and
// function names, same argument meaning, value semantics and
// std::invalid_argument errors; R: = /root/reference/proj/include/ternkit/)
// on top of the C-ABI in include/ternkit_b200.h.  A reference user switches
// by replacing `#include "ternkit/linalg.hpp"` (etc.) with this header and
// linking libternkit_b200.so + cudart:
//
//     g++ -std=c++20 -I include app.cpp -L paper_2008_05101_b200 -lternkit_b200 -lcudart
//
// Every compute entry point runs on the GPU (device 0 by default, the CUDA
// default stream) and synchronises before returning, so errors surface as in
// the reference.  `workers` arguments are accepted and ignored: the CUDA grid
// replaces the CPU row partition (R:linalg.hpp:278-291).  PackedConvLayer
// additionally owns the device copy of its weights (uploaded once).
#pragma once

#include <cuda_runtime.h>

#include <bit>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../ternkit_b200.h"

namespace ternkit {

inline constexpr int kLanesPerWord = 32;                     // R:codec.hpp:32
inline constexpr std::uint64_t kAuxi = 0x5555555555555555ull;  // R:codec.hpp:35

namespace b200 {

inline void check(int st, const char* where) {
  if (st == TK_OK) return;
  if (st == TK_ERR_CUDA) throw std::runtime_error(std::string(where) + ": CUDA error");
  throw std::invalid_argument(std::string(where) + ": " + tk_status_string(st));
}

// process-wide context on the current device
inline tk_context* ctx() {
  static std::unique_ptr<tk_context, int (*)(tk_context*)> c = [] {
    int dev = 0;
    cudaGetDevice(&dev);
    tk_context* p = nullptr;
    check(tk_context_create(dev, &p), "tk_context_create");
    return std::unique_ptr<tk_context, int (*)(tk_context*)>(p, tk_context_destroy);
  }();
  return c.get();
}

inline void sync(const char* where) { check(tk_context_sync(ctx(), nullptr), where); }

template <class T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(std::size_t n) {
    if (n && cudaMalloc(&p, n * sizeof(T)) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
  }
  DevBuf(const T* host, std::size_t n) : DevBuf(n) {
    if (n) cudaMemcpy(p, host, n * sizeof(T), cudaMemcpyHostToDevice);
  }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  std::vector<T> host(std::size_t n) const {
    std::vector<T> v(n);
    if (n) cudaMemcpy(v.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost);
    return v;
  }
};

}  // namespace b200

// ---- codec (R:codec.hpp) ---------------------------------------------------

inline int decode_lane(unsigned code) noexcept { return std::popcount(code & 3u) - 1; }

inline unsigned encode_lane(int value) {
  switch (value) {
    case -1: return 0b00u;
    case 0: return 0b01u;
    case 1: return 0b11u;
    default:
      throw std::invalid_argument("ternary value out of range {-1,0,1}: " + std::to_string(value));
  }
}

struct QuantThresholds {
  float alpha1 = 1.0f;
  float alpha2 = 1.0f;
  void validate() const {
    if (!(alpha1 > 0.0f) || !(alpha2 > 0.0f))
      throw std::invalid_argument("quantizer step sizes must be positive");
  }
};

struct PackedTernaryVector {
  std::vector<std::uint64_t> words;
  std::size_t logical_len = 0;
  bool nonneg_offset = false;
  std::size_t lane_capacity() const noexcept { return words.size() * kLanesPerWord; }
};

inline std::size_t words_for_lanes(std::size_t n) noexcept { return (n + kLanesPerWord - 1) / kLanesPerWord; }

inline PackedTernaryVector pack(std::span<const std::int8_t> values) {
  PackedTernaryVector out;
  out.logical_len = values.size();
  const std::size_t nw = words_for_lanes(values.size());
  b200::DevBuf<std::int8_t> v(values.data(), values.size());
  b200::DevBuf<std::uint64_t> w(nw);
  b200::check(tk_pack(b200::ctx(), v.p, values.size(), w.p, nullptr), "pack");
  b200::sync("pack");
  out.words = w.host(nw);
  return out;
}
inline PackedTernaryVector pack(const std::vector<std::int8_t>& v) {
  return pack(std::span<const std::int8_t>(v));
}

inline std::vector<std::int8_t> unpack(const PackedTernaryVector& v) {
  b200::DevBuf<std::uint64_t> w(v.words.data(), v.words.size());
  b200::DevBuf<std::int8_t> o(v.logical_len);
  b200::check(tk_unpack(b200::ctx(), w.p, v.logical_len, o.p, nullptr), "unpack");
  b200::sync("unpack");
  return o.host(v.logical_len);
}

// ---- quantizer (R:quantizer.hpp) ---------------------------------------------

enum class QuantMode { kWeight, kActivationNonneg };

inline int tk_mode(QuantMode m) { return m == QuantMode::kWeight ? TK_MODE_WEIGHT : TK_MODE_ACTIVATION_NONNEG; }

inline PackedTernaryVector quantize_and_pack(std::span<const float> x, const QuantThresholds& t, QuantMode mode) {
  t.validate();
  PackedTernaryVector out;
  out.logical_len = x.size();
  out.nonneg_offset = mode == QuantMode::kActivationNonneg;
  const std::size_t nw = words_for_lanes(x.size());
  b200::DevBuf<float> xd(x.data(), x.size());
  b200::DevBuf<std::uint64_t> w(nw);
  b200::check(tk_quantize_pack(b200::ctx(), xd.p, 1, x.size(), t.alpha1, t.alpha2, tk_mode(mode), w.p, nullptr),
              "quantize_and_pack");
  b200::sync("quantize_and_pack");
  out.words = w.host(nw);
  return out;
}

inline std::vector<std::int8_t> quantize_weight(std::span<const float> p, const QuantThresholds& t) {
  return unpack(quantize_and_pack(p, t, QuantMode::kWeight));
}

inline std::vector<std::int8_t> quantize_activation_nonneg(std::span<const float> p, const QuantThresholds& t) {
  std::vector<std::int8_t> q = unpack(quantize_and_pack(p, t, QuantMode::kActivationNonneg));
  for (auto& v : q) v = static_cast<std::int8_t>(v + 1);
  return q;
}

inline int quantize_weight_value(float p, const QuantThresholds& t) {
  return quantize_weight(std::span<const float>(&p, 1), t)[0];
}

inline int quantize_activation_value(float p, const QuantThresholds& t) {
  return quantize_activation_nonneg(std::span<const float>(&p, 1), t)[0];
}

// ---- bit kernels (R:bitkernels.hpp) -------------------------------------------

inline std::uint64_t ternary_zero_seed(std::uint64_t yw) noexcept { return (yw ^ (yw >> 1)) & kAuxi; }

inline std::uint64_t ternary_multiply_word(std::uint64_t xw, std::uint64_t yw) noexcept {
  const std::uint64_t d = ternary_zero_seed(yw);
  return (~(xw ^ yw) | d) & ~(d << 1);
}

// R:bitkernels.hpp:66-72: the zero seed supplied by the caller
inline std::uint64_t ternary_multiply_word_premask(std::uint64_t xw, std::uint64_t yw, std::uint64_t d) noexcept {
  return (~(xw ^ yw) | d) & ~(d << 1);
}

namespace detail {

// R:bitkernels.hpp:76-85 (the reference's raw-pointer entry), on the GPU:
// host words in, sum popcount(TM) - 32 * words out.  Like the reference it
// does not throw; a CUDA failure terminates (there is no CPU fallback).
inline std::int64_t ternary_dot_words(const std::uint64_t* x, const std::uint64_t* y, std::size_t words) noexcept {
  b200::DevBuf<std::uint64_t> xd(x, words), yd(y, words);
  b200::DevBuf<std::int64_t> o(1);
  b200::check(tk_ternary_dot_batched(b200::ctx(), xd.p, yd.p, words, 1, nullptr, o.p, nullptr), "ternary_dot_words");
  b200::sync("ternary_dot_words");
  return o.host(1)[0];
}

// R:bitkernels.hpp:87-97: the same with the zero seeds supplied (used as given)
inline std::int64_t ternary_dot_words_premask(const std::uint64_t* x, const std::uint64_t* y,
                                              const std::uint64_t* seed, std::size_t words) noexcept {
  b200::DevBuf<std::uint64_t> xd(x, words), yd(y, words), sd(seed, words);
  b200::DevBuf<std::int64_t> o(1);
  b200::check(tk_ternary_dot_premask_batched(b200::ctx(), xd.p, yd.p, sd.p, words, 1, nullptr, o.p, nullptr),
              "ternary_dot_words_premask");
  b200::sync("ternary_dot_words_premask");
  return o.host(1)[0];
}

}  // namespace detail

inline std::int64_t ternary_dot(const PackedTernaryVector& x, const PackedTernaryVector& y) {
  if (x.logical_len != y.logical_len) throw std::invalid_argument("ternary_dot: length mismatch");
  const std::size_t nw = x.words.size();
  b200::DevBuf<std::uint64_t> xd(x.words.data(), nw), yd(y.words.data(), nw);
  b200::DevBuf<std::int64_t> o(1);
  b200::check(tk_ternary_dot_batched(b200::ctx(), xd.p, yd.p, nw, 1, nullptr, o.p, nullptr), "ternary_dot");
  b200::sync("ternary_dot");
  return o.host(1)[0];
}

inline std::vector<std::uint64_t> make_zero_seeds(const PackedTernaryVector& y) {
  std::vector<std::uint64_t> s(y.words.size());
  for (std::size_t i = 0; i < s.size(); ++i) s[i] = ternary_zero_seed(y.words[i]);
  return s;
}

inline std::int64_t ternary_dot_premask(const PackedTernaryVector& x, const PackedTernaryVector& y,
                                        std::span<const std::uint64_t> seeds) {
  if (x.logical_len != y.logical_len) throw std::invalid_argument("ternary_dot_premask: length mismatch");
  if (seeds.size() != y.words.size()) throw std::invalid_argument("ternary_dot_premask: seed buffer mismatch");
  const std::size_t nw = x.words.size();
  b200::DevBuf<std::uint64_t> xd(x.words.data(), nw), yd(y.words.data(), nw), sd(seeds.data(), nw);
  b200::DevBuf<std::int64_t> o(1);
  b200::check(tk_ternary_dot_premask_batched(b200::ctx(), xd.p, yd.p, sd.p, nw, 1, nullptr, o.p, nullptr),
              "ternary_dot_premask");
  b200::sync("ternary_dot_premask");
  return o.host(1)[0];
}

inline std::int64_t ternary_dot_nonneg(const PackedTernaryVector& a, const PackedTernaryVector& w,
                                       std::int64_t w_sum) {
  if (!a.nonneg_offset)
    throw std::invalid_argument("ternary_dot_nonneg: activation vector lacks the nonneg offset flag");
  return ternary_dot(a, w) + w_sum;
}

// ---- linalg (R:linalg.hpp) ---------------------------------------------------

struct TensorShape {
  int n = 0, c = 0, h = 0, w = 0;
  std::size_t count() const noexcept { return static_cast<std::size_t>(n) * c * h * w; }
};

struct ConvGeometry {
  int in_c = 0, out_c = 0;
  int kh = 3, kw = 3;
  int stride = 1, pad = 1;
  int patch_len() const noexcept { return in_c * kh * kw; }
  void validate(const TensorShape& x) const {
    if (in_c <= 0 || out_c <= 0 || kh <= 0 || kw <= 0 || stride <= 0 || pad < 0)
      throw std::invalid_argument("conv geometry: nonpositive dimension");
    if (x.c != in_c) throw std::invalid_argument("conv geometry: channel count mismatch");
    if (x.h + 2 * pad < kh || x.w + 2 * pad < kw)
      throw std::invalid_argument("conv geometry: kernel exceeds padded input");
  }
  int out_h(int h) const noexcept { return (h + 2 * pad - kh) / stride + 1; }
  int out_w(int w) const noexcept { return (w + 2 * pad - kw) / stride + 1; }
};

struct ChannelAffine {
  std::vector<float> gain;
  std::vector<float> bias;
  static ChannelAffine identity(int channels) {
    return {std::vector<float>(channels, 1.0f), std::vector<float>(channels, 0.0f)};
  }
};

inline ChannelAffine fuse_bn(std::span<const float> mean, std::span<const float> var, std::span<const float> gamma,
                             std::span<const float> beta, float eps) {
  const std::size_t c = mean.size();
  if (var.size() != c || gamma.size() != c || beta.size() != c)
    throw std::invalid_argument("fuse_bn: per-channel stat size mismatch");
  ChannelAffine out;
  out.gain.resize(c);
  out.bias.resize(c);
  b200::check(tk_fuse_bn(mean.data(), var.data(), gamma.data(), beta.data(), eps, static_cast<int>(c),
                         out.gain.data(), out.bias.data()),
              "fuse_bn");
  return out;
}

struct PackedConvLayer {
  ConvGeometry geom;
  std::vector<PackedTernaryVector> weights;
  std::vector<std::int32_t> weight_sums;
  std::vector<std::vector<std::uint64_t>> weight_mask_seeds;
  QuantThresholds thr_w, thr_a;
  float out_scale = 1.0f;
  ChannelAffine fused;
  bool activation_nonneg = true;
  std::shared_ptr<tk_layer> device;  // uploaded packed rows, masks, s8 operand, affine

  bool masks_ready() const noexcept { return weight_mask_seeds.size() == weights.size(); }
  void precompute_masks() {
    weight_mask_seeds.clear();
    for (const auto& w : weights) weight_mask_seeds.push_back(make_zero_seeds(w));
    if (device) b200::check(tk_layer_precompute_masks(device.get()), "precompute_masks");
  }
};

inline PackedConvLayer make_packed_conv_layer(std::span<const std::int8_t> ternary_weights, const ConvGeometry& geom,
                                              QuantThresholds thr_w, QuantThresholds thr_a, bool activation_nonneg,
                                              ChannelAffine fused = {}, float out_scale = 1.0f) {
  const std::size_t k = static_cast<std::size_t>(geom.patch_len());
  if (ternary_weights.size() != k * geom.out_c)
    throw std::invalid_argument("make_packed_conv_layer: weight size mismatch");
  PackedConvLayer layer;
  layer.geom = geom;
  layer.thr_w = thr_w;
  layer.thr_a = thr_a;
  layer.out_scale = out_scale;
  layer.activation_nonneg = activation_nonneg;
  layer.fused = fused.gain.empty() ? ChannelAffine::identity(geom.out_c) : std::move(fused);
  tk_layer* h = nullptr;
  b200::check(tk_layer_create(b200::ctx(), ternary_weights.data(), geom.in_c, geom.out_c, geom.kh, geom.kw,
                              geom.stride, geom.pad, thr_w.alpha1, thr_w.alpha2, thr_a.alpha1, thr_a.alpha2,
                              activation_nonneg ? 1 : 0, layer.fused.gain.data(), layer.fused.bias.data(),
                              out_scale, &h),
              "make_packed_conv_layer");
  layer.device = std::shared_ptr<tk_layer>(h, [](tk_layer* p) { tk_layer_destroy(p); });
  const std::size_t wpr = words_for_lanes(k);
  std::vector<std::uint64_t> words(wpr * geom.out_c);
  layer.weight_sums.resize(geom.out_c);
  b200::check(tk_layer_words_host(h, words.data(), layer.weight_sums.data()), "layer words");
  for (int o = 0; o < geom.out_c; ++o) {
    PackedTernaryVector v;
    v.logical_len = k;
    v.words.assign(words.begin() + o * wpr, words.begin() + (o + 1) * wpr);
    layer.weights.push_back(std::move(v));
  }
  return layer;
}

inline PackedConvLayer make_packed_conv_layer_from_float(std::span<const float> weights, const ConvGeometry& geom,
                                                         QuantThresholds thr_w, QuantThresholds thr_a,
                                                         bool activation_nonneg, ChannelAffine fused = {},
                                                         float out_scale = 1.0f) {
  std::vector<std::int8_t> q = quantize_weight(weights, thr_w);
  return make_packed_conv_layer(q, geom, thr_w, thr_a, activation_nonneg, std::move(fused), out_scale);
}

struct Im2colBuffer {
  std::vector<std::uint64_t> words;
  std::size_t words_per_row = 0;
  std::size_t row_count = 0;
  std::size_t row_len = 0;
  bool nonneg_offset = false;
  int batch = 0, out_h = 0, out_w = 0;
  std::span<const std::uint64_t> row(std::size_t r) const { return {words.data() + r * words_per_row, words_per_row}; }
};

inline Im2colBuffer im2col_quantize_pack(std::span<const float> x, const TensorShape& shape, const QuantThresholds& t,
                                         const ConvGeometry& geom, QuantMode mode) {
  geom.validate(shape);
  t.validate();
  if (x.size() != shape.count()) throw std::invalid_argument("im2col: input size does not match shape");
  Im2colBuffer buf;
  buf.batch = shape.n;
  buf.out_h = geom.out_h(shape.h);
  buf.out_w = geom.out_w(shape.w);
  buf.row_len = static_cast<std::size_t>(geom.patch_len());
  buf.words_per_row = words_for_lanes(buf.row_len);
  buf.row_count = static_cast<std::size_t>(shape.n) * buf.out_h * buf.out_w;
  buf.nonneg_offset = mode == QuantMode::kActivationNonneg;
  b200::DevBuf<float> xd(x.data(), x.size());
  b200::DevBuf<std::uint64_t> rows(buf.row_count * buf.words_per_row);
  b200::check(tk_im2col_quantize_pack(b200::ctx(), xd.p, shape.n, shape.c, shape.h, shape.w, geom.kh, geom.kw,
                                      geom.stride, geom.pad, t.alpha1, t.alpha2, tk_mode(mode), rows.p, nullptr),
              "im2col_quantize_pack");
  b200::sync("im2col_quantize_pack");
  buf.words = rows.host(buf.row_count * buf.words_per_row);
  return buf;
}

enum class MaskMode { kOnTheFly, kPrecomputed };

inline std::vector<std::int32_t> packed_gemm(const Im2colBuffer& a, const PackedConvLayer& layer,
                                             MaskMode mask_mode = MaskMode::kOnTheFly, int /*workers*/ = 1) {
  if (static_cast<int>(layer.weights.size()) != layer.geom.out_c)
    throw std::invalid_argument("packed_gemm: layer weight rows != out_c");
  if (mask_mode == MaskMode::kPrecomputed && !layer.masks_ready())
    throw std::invalid_argument("packed_gemm: masks not precomputed");
  b200::DevBuf<std::uint64_t> rows(a.words.data(), a.words.size());
  b200::DevBuf<std::int32_t> out(a.row_count * layer.geom.out_c);
  b200::check(tk_packed_gemm(b200::ctx(), layer.device.get(), rows.p, a.row_count, a.row_len, a.nonneg_offset ? 1 : 0,
                             mask_mode == MaskMode::kPrecomputed ? TK_MASK_PRECOMPUTED : TK_MASK_ON_THE_FLY, out.p,
                             nullptr),
              "packed_gemm");
  b200::sync("packed_gemm");
  return out.host(a.row_count * layer.geom.out_c);
}

struct ConvResult {
  std::vector<float> data;
  TensorShape shape;
};

inline ConvResult conv2d_ternary(std::span<const float> x, const TensorShape& shape, const PackedConvLayer& layer,
                                 MaskMode mask_mode = MaskMode::kOnTheFly, int /*workers*/ = 1) {
  layer.geom.validate(shape);
  if (x.size() != shape.count()) throw std::invalid_argument("im2col: input size does not match shape");
  if (mask_mode == MaskMode::kPrecomputed && !layer.masks_ready())
    throw std::invalid_argument("packed_gemm: masks not precomputed");
  ConvResult r;
  r.shape = {shape.n, layer.geom.out_c, layer.geom.out_h(shape.h), layer.geom.out_w(shape.w)};
  b200::DevBuf<float> xd(x.data(), x.size());
  b200::DevBuf<float> out(r.shape.count());
  b200::check(tk_conv2d_ternary(b200::ctx(), layer.device.get(), xd.p, shape.n, shape.h, shape.w,
                                mask_mode == MaskMode::kPrecomputed ? TK_MASK_PRECOMPUTED : TK_MASK_ON_THE_FLY, out.p,
                                nullptr),
              "conv2d_ternary");
  b200::sync("conv2d_ternary");
  r.data = out.host(r.shape.count());
  return r;
}

inline std::vector<float> fully_connected_ternary(std::span<const float> x, int batch, const PackedConvLayer& layer,
                                                  MaskMode mask_mode = MaskMode::kOnTheFly) {
  if (layer.geom.kh != 1 || layer.geom.kw != 1 || layer.geom.pad != 0)
    throw std::invalid_argument("fully_connected_ternary: expects 1x1 geometry");
  const TensorShape shape{batch, layer.geom.in_c, 1, 1};
  return conv2d_ternary(x, shape, layer, mask_mode).data;
}

}  // namespace ternkit
