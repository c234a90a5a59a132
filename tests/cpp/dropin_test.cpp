// Drop-in check: reference-style unit checks written against the quake::
// API of include/quake_b200/quake.hpp (the reference's kernels.hpp/nonlin.hpp
// signatures), linked against libquake_b200.so. Mirrors known answers from
// the reference's tests/test_kernels.cpp:63-131 and tests/test_nonlin.cpp:
// 42-62, 123-138, 218-229 (paths relative to /root/reference/proj/).
// Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <limits>
#include <random>
#include <stdexcept>
#include <vector>

#include "quake_b200/quake.hpp"

static int failures = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);    \
      ++failures;                                                  \
    }                                                              \
  } while (0)

template <typename Fn>
static bool throws_invalid(Fn&& fn) {
  try {
    fn();
  } catch (const std::invalid_argument&) {
    return true;
  }
  return false;
}

int main() {
  using quake::KernelChoice;
  using quake::QuadCoeffs;
  const float inf = std::numeric_limits<float>::infinity();

  // test_kernels.cpp:63-73
  const quake::AffineCoeffs b2 = quake::base2_coeffs(false);
  const quake::ClampRange r = quake::clamp_for(b2);
  CHECK(quake::quake(0.5f, b2, r) == 1.5f);
  CHECK(quake::quake(3.0f, b2, r) == 8.0f);
  // :75-81
  CHECK(quake::quake2(0.5f, b2, QuadCoeffs::continuity(), r) == (1.5f * 1.5f + 2.0f) / 3.0f);
  // :83-92 exact at 2^k (buffer form, one GPU call per kernel)
  std::vector<float> ks;
  for (int k = -100; k <= 100; ++k) ks.push_back(static_cast<float>(k));
  const quake::NumericBuffer y1 = quake::quake_buffer(ks, b2, r);
  const quake::NumericBuffer y2 = quake::quake2_buffer(ks, b2, QuadCoeffs::continuity(), r);
  for (std::size_t i = 0; i < ks.size(); ++i) {
    CHECK(y1[i] == std::ldexp(1.0f, static_cast<int>(ks[i])));
    CHECK(y2[i] == std::ldexp(1.0f, static_cast<int>(ks[i])));
  }
  // :123-131 saturation
  const quake::AffineCoeffs ne = quake::natural_exp_coeffs(true);
  const quake::ClampRange rn = quake::clamp_for(ne);
  const std::vector<float> sat{rn.lo - 50.0f, rn.hi + 50.0f, -inf, inf, std::nanf(""), rn.lo, rn.hi};
  const quake::NumericBuffer s = quake::quake_buffer(sat, ne, rn);
  CHECK(s[0] == s[5] && s[2] == s[5]);
  CHECK(s[1] == s[6] && s[3] == s[6] && s[4] == s[6]);
  // test_nonlin.cpp:42-62 constant rows
  for (const KernelChoice k : {KernelChoice::Exact, KernelChoice::Quake, KernelChoice::Quake2}) {
    const std::vector<float> v(4096, 5.25f);
    const quake::NumericBuffer out = quake::softmax_row(v, quake::SoftmaxParams{}, k);
    for (const float y : out) CHECK(y == out[0]);
  }
  // :123-138 input rejection, out untouched
  std::vector<float> out4(4, 7.0f);
  CHECK(throws_invalid([] {
    quake::softmax_row(std::vector<float>{}, quake::SoftmaxParams{}, KernelChoice::Exact);
  }));
  CHECK(throws_invalid([&] {
    quake::softmax_rows(std::vector<float>{1.0f, 2.0f, std::nanf(""), 3.0f}, 2,
                        quake::SoftmaxParams{}, KernelChoice::Quake2, out4);
  }));
  for (const float v : out4) CHECK(v == 7.0f);
  CHECK(throws_invalid([] { quake::coeffs_for(0.0f, 1.0f); }));
  // :218-229 buffer == scalar (logistic), GPU scalar form vs GPU buffer form
  std::mt19937 rng(59);
  std::uniform_real_distribution<float> dist(-30.0f, 30.0f);
  std::vector<float> xs(2000), lo(2000);
  for (auto& x : xs) x = dist(rng);
  for (const KernelChoice k : {KernelChoice::Quake, KernelChoice::Quake2}) {
    quake::logistic_buffer(xs, lo, k);
    for (std::size_t i = 0; i < xs.size(); i += 97) CHECK(lo[i] == quake::logistic(xs[i], k));
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAIL" : "PASS", failures);
  return failures;
}
