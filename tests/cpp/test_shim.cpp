// test_shim.cpp -- the reference's own hot-path unit tests, re-expressed
// against the drop-in C++ header include/ternkit_b200/ternkit.hpp (so every
// call runs on the B200 kernels).  Cases follow R:tests/test_codec.cpp,
// test_bitkernels.cpp, test_quantizer.cpp and test_linalg.cpp (cited per
// case).  A tiny CHECK harness replaces Catch2 (absent in this image).
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "ternkit_b200/ternkit.hpp"

using namespace ternkit;

static int g_checks = 0, g_fail = 0;
#define CHECK(c)                                                      \
  do {                                                                \
    ++g_checks;                                                       \
    if (!(c)) {                                                       \
      ++g_fail;                                                       \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);        \
    }                                                                 \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                      \
  do {                                                                \
    ++g_checks;                                                       \
    bool thrown_ = false;                                             \
    try {                                                             \
      (void)(expr);                                                   \
    } catch (const T&) {                                              \
      thrown_ = true;                                                 \
    }                                                                 \
    if (!thrown_) {                                                   \
      ++g_fail;                                                       \
      std::printf("FAIL %s:%d: no throw: %s\n", __FILE__, __LINE__, #expr); \
    }                                                                 \
  } while (0)

static std::vector<float> random_floats(std::size_t n, unsigned seed, bool nonneg = false) {
  std::mt19937 rng(seed);
  std::normal_distribution<float> d(0.0f, 1.0f);
  std::vector<float> v(n);
  for (auto& e : v) e = nonneg ? std::abs(d(rng)) : d(rng);
  return v;
}
static std::vector<std::int8_t> random_ternary(std::size_t n, unsigned seed) {
  std::mt19937 rng(seed);
  std::uniform_int_distribution<int> t(-1, 1);
  std::vector<std::int8_t> v(n);
  for (auto& e : v) e = static_cast<std::int8_t>(t(rng));
  return v;
}

static void codec() {
  // R:tests/test_codec.cpp:31-37
  PackedTernaryVector p = pack(std::vector<std::int8_t>{-1, 0, 0, 1});
  CHECK(p.words.size() == 1 && (p.words[0] & 0xFF) == 0b11010100u && p.logical_len == 4);
  // :46-51 padding lanes hold the canonical zero code
  p = pack(std::vector<std::int8_t>{1});
  CHECK((p.words[0] >> 2) == (kAuxi >> 2) && p.lane_capacity() == 32);
  // :53-55
  CHECK_THROWS_AS(pack(std::vector<std::int8_t>{0, 3}), std::invalid_argument);
  // :71-80 round trip incl. length 37
  std::mt19937 rng(3);
  std::uniform_int_distribution<int> val(-1, 1);
  for (int it = 0; it < 200; ++it) {
    const std::size_t n = it == 0 ? 37 : static_cast<std::size_t>(it % 130);
    std::vector<std::int8_t> v(n);
    for (auto& e : v) e = static_cast<std::int8_t>(val(rng));
    CHECK(unpack(pack(v)) == v);
  }
  // :102-106, :108-112
  const std::vector<float> x{0.6f, -0.7f, 0.1f};
  CHECK((unpack(quantize_and_pack(x, {1.0f, 1.0f}, QuantMode::kWeight)) == std::vector<std::int8_t>{1, -1, 0}));
  PackedTernaryVector z = quantize_and_pack(std::vector<float>(64, 0.0f), {0.7f, 1.3f}, QuantMode::kWeight);
  for (auto w : z.words) CHECK(w == kAuxi);
  // :114-118
  const std::vector<float> bad{0.1f, std::nanf("")};
  CHECK_THROWS_AS(quantize_and_pack(bad, {1.0f, 1.0f}, QuantMode::kWeight), std::invalid_argument);
}

static void quantizer() {
  // R:tests/test_quantizer.cpp:9-34
  const QuantThresholds t{1.0f, 1.0f};
  CHECK(quantize_weight_value(0.6f, t) == 1);
  CHECK(quantize_weight_value(-0.3f, t) == 0);
  CHECK(quantize_weight_value(-0.7f, t) == -1);
  CHECK(quantize_weight_value(0.5f, t) == 0);   // bankers tie
  CHECK(quantize_weight_value(-0.5f, t) == 0);
  const QuantThresholds a{0.5f, 1.0f};
  CHECK(quantize_activation_value(0.4f, a) == 1);
  CHECK(quantize_activation_value(1.6f, a) == 2);
  CHECK(quantize_activation_value(0.1f, a) == 0);
  CHECK_THROWS_AS(quantize_activation_value(-0.1f, {1.0f, 1.0f}), std::invalid_argument);
  CHECK_THROWS_AS(quantize_weight(std::vector<float>{0.1f}, {0.0f, 1.0f}), std::invalid_argument);
}

static void bitkernels() {
  // R:tests/test_bitkernels.cpp:23-35 truth table
  for (unsigned xc = 0; xc < 4; ++xc)
    for (unsigned yc = 0; yc < 4; ++yc) {
      const std::uint64_t tm = ternary_multiply_word((kAuxi & ~3ull) | xc, (kAuxi & ~3ull) | yc);
      const unsigned zc = static_cast<unsigned>(tm & 3);
      CHECK(decode_lane(zc) == decode_lane(xc) * decode_lane(yc));
    }
  // :77-80
  CHECK(ternary_dot(pack(std::vector<std::int8_t>{1, 0, -1, 1}), pack(std::vector<std::int8_t>{-1, 0, 1, 1})) == -1);
  // :87-97 fuzz vs naive
  std::mt19937 rng(7);
  std::uniform_int_distribution<int> v(-1, 1), len(1, 700);
  for (int it = 0; it < 60; ++it) {
    const int n = len(rng);
    std::vector<std::int8_t> x(n), y(n);
    std::int64_t want = 0;
    for (int i = 0; i < n; ++i) {
      x[i] = static_cast<std::int8_t>(v(rng));
      y[i] = static_cast<std::int8_t>(v(rng));
      want += x[i] * y[i];
    }
    CHECK(ternary_dot(pack(x), pack(y)) == want);
  }
  // :112-119 mismatches rejected
  PackedTernaryVector a = pack(std::vector<std::int8_t>{1, 0}), b = pack(std::vector<std::int8_t>{1, 0, -1});
  CHECK_THROWS_AS(ternary_dot(a, b), std::invalid_argument);
  CHECK_THROWS_AS(ternary_dot_premask(a, a, std::vector<std::uint64_t>{}), std::invalid_argument);
  CHECK_THROWS_AS(ternary_dot_nonneg(a, a, 0), std::invalid_argument);
  // :121-135 nonneg hand example
  std::vector<std::int8_t> st{1, -1, 0};  // a = {2, 0, 1} stored as a - 1
  PackedTernaryVector ap = pack(st);
  ap.nonneg_offset = true;
  CHECK(ternary_dot_nonneg(ap, pack(std::vector<std::int8_t>{1, -1, 1}), 1) == 3);
  // R:bitkernels.hpp:66-97: the raw-pointer detail:: entries and the premask
  // forms; with make_zero_seeds they equal ternary_dot, and supplied seeds are
  // used as given (here: all-zero seeds = every lane treated as nonzero)
  {
    const std::vector<std::int8_t> xs = random_ternary(1000, 21), ys = random_ternary(1000, 22);
    const PackedTernaryVector xp = pack(xs), yp = pack(ys);
    const std::vector<std::uint64_t> seeds = make_zero_seeds(yp);
    const std::int64_t want = ternary_dot(xp, yp);
    CHECK(detail::ternary_dot_words(xp.words.data(), yp.words.data(), xp.words.size()) == want);
    CHECK(detail::ternary_dot_words_premask(xp.words.data(), yp.words.data(), seeds.data(), xp.words.size()) == want);
    CHECK(ternary_dot_premask(xp, yp, seeds) == want);
    const std::vector<std::uint64_t> zero(seeds.size(), 0);
    std::int64_t host = 0;
    for (std::size_t i = 0; i < xp.words.size(); ++i)
      host += __builtin_popcountll(ternary_multiply_word_premask(xp.words[i], yp.words[i], 0));
    host -= static_cast<std::int64_t>(xp.words.size()) * kLanesPerWord;
    CHECK(ternary_dot_premask(xp, yp, zero) == host);
    CHECK(detail::ternary_dot_words_premask(xp.words.data(), yp.words.data(), zero.data(), xp.words.size()) == host);
    for (std::size_t i = 0; i < xp.words.size(); ++i)
      CHECK(ternary_multiply_word_premask(xp.words[i], yp.words[i], seeds[i]) ==
            ternary_multiply_word(xp.words[i], yp.words[i]));
  }
}

static void linalg() {
  // R:tests/test_linalg.cpp:65-70 fuse_bn identity
  std::vector<float> m{0, 0}, var{1, 1}, g{1, 1}, be{0, 0};
  ChannelAffine aff = fuse_bn(m, var, g, be, 0.0f);
  CHECK(aff.gain[0] == 1.0f && aff.bias[1] == 0.0f);
  CHECK_THROWS_AS(fuse_bn(std::vector<float>{0}, std::vector<float>{0}, std::vector<float>{0},
                          std::vector<float>{0}, 0.0f),
                  std::invalid_argument);
  // :113-128 3x3 pad-1 corners
  Im2colBuffer buf = im2col_quantize_pack(std::vector<float>(9, 1.0f), {1, 1, 3, 3}, {1, 1}, {1, 1, 3, 3, 1, 1},
                                          QuantMode::kWeight);
  PackedTernaryVector row;
  row.words.assign(buf.row(0).begin(), buf.row(0).end());
  row.logical_len = buf.row_len;
  int zeros = 0, ones = 0;
  for (auto e : unpack(row)) (e == 0 ? zeros : ones)++;
  CHECK(zeros == 5 && ones == 4);
  // :165-175 validation
  CHECK_THROWS_AS(im2col_quantize_pack(random_floats(32, 34), {1, 2, 4, 4}, {1, 1}, {3, 1, 3, 3, 1, 1},
                                       QuantMode::kWeight),
                  std::invalid_argument);
  // :192-213 packed gemm == naive integer matmul
  {
    const int rows = 8, inner = 16, ocs = 4;
    auto wq = random_ternary(static_cast<std::size_t>(ocs) * inner, 36);
    const ConvGeometry gm{inner, ocs, 1, 1, 1, 0};
    PackedConvLayer layer = make_packed_conv_layer(wq, gm, {1, 1}, {0.5f, 0.5f}, true);
    auto x = random_floats(static_cast<std::size_t>(rows) * inner, 37, true);
    Im2colBuffer b2 = im2col_quantize_pack(x, {rows, inner, 1, 1}, layer.thr_a, gm, QuantMode::kActivationNonneg);
    auto out = packed_gemm(b2, layer);
    for (int r = 0; r < rows; ++r)
      for (int o = 0; o < ocs; ++o) {
        std::int64_t want = 0;
        for (int j = 0; j < inner; ++j)
          want += quantize_activation_value(x[r * inner + j], layer.thr_a) * wq[o * inner + j];
        CHECK(out[r * ocs + o] == want);
      }
    // :215-231 mask modes agree
    CHECK_THROWS_AS(packed_gemm(b2, layer, MaskMode::kPrecomputed), std::invalid_argument);
    layer.precompute_masks();
    CHECK(packed_gemm(b2, layer, MaskMode::kPrecomputed) == out);
    CHECK(packed_gemm(b2, layer, MaskMode::kOnTheFly, 3) == out);
  }
  // :289-304 batch independence (exact)
  {
    const ConvGeometry gm{3, 5, 3, 3, 1, 1};
    auto wq = random_ternary(static_cast<std::size_t>(gm.out_c) * gm.patch_len(), 45);
    PackedConvLayer layer = make_packed_conv_layer(wq, gm, {1, 1}, {0.5f, 0.5f}, true);
    auto xa = random_floats(108, 46, true), xb = random_floats(108, 47, true);
    std::vector<float> both(xa);
    both.insert(both.end(), xb.begin(), xb.end());
    ConvResult ra = conv2d_ternary(xa, {1, 3, 6, 6}, layer), rb = conv2d_ternary(xb, {1, 3, 6, 6}, layer);
    ConvResult rc = conv2d_ternary(both, {2, 3, 6, 6}, layer);
    std::vector<float> want(ra.data);
    want.insert(want.end(), rb.data.begin(), rb.data.end());
    CHECK(rc.data == want);
  }
  // :342-380 FC == naive, geometry check, zero input -> bias
  {
    const int in = 20, out = 6, batch = 3;
    auto wq = random_ternary(static_cast<std::size_t>(out) * in, 52);
    PackedConvLayer layer = make_packed_conv_layer(wq, {in, out, 1, 1, 1, 0}, {1, 1}, {0.5f, 0.5f}, true);
    auto x = random_floats(static_cast<std::size_t>(batch) * in, 53, true);
    auto y = fully_connected_ternary(x, batch, layer);
    for (int b = 0; b < batch; ++b)
      for (int o = 0; o < out; ++o) {
        std::int64_t want = 0;
        for (int j = 0; j < in; ++j) want += quantize_activation_value(x[b * in + j], layer.thr_a) * wq[o * in + j];
        CHECK(y[b * out + o] == static_cast<float>(want));
      }
    auto wq3 = random_ternary(static_cast<std::size_t>(out) * in * 9, 54);
    PackedConvLayer bad = make_packed_conv_layer(wq3, {in, out, 3, 3, 1, 1}, {1, 1}, {0.5f, 0.5f}, true);
    CHECK_THROWS_AS(fully_connected_ternary(x, batch, bad), std::invalid_argument);
    ChannelAffine a2{{1.0f, 2.0f, 3.0f}, {0.5f, -0.5f, 4.0f}};
    PackedConvLayer l3 = make_packed_conv_layer(random_ternary(24, 55), {8, 3, 1, 1, 1, 0}, {1, 1}, {0.5f, 0.5f},
                                                true, a2);
    auto yz = fully_connected_ternary(std::vector<float>(8, 0.0f), 1, l3);
    CHECK(yz[0] == 0.5f && yz[1] == -0.5f && yz[2] == 4.0f);
  }
  // :382-387
  CHECK_THROWS_AS(make_packed_conv_layer(std::vector<std::int8_t>(7, 0), {4, 2, 1, 1, 1, 0}, {1, 1}, {1, 1}, true),
                  std::invalid_argument);
}

int main() {
  codec();
  quantizer();
  bitkernels();
  linalg();
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
