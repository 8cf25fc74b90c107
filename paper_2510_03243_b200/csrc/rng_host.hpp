// Host restatements shared by the product's host code (csrc/host.cpp: the
// build_pairs stream) and the synthetic-workload tool (tools/workload):
// the reference's Rng (rng.hpp:22-75) and its integer formatting.
#pragma once

#include <cmath>
#include <cstdint>
#include <random>
#include <string>
#include <utility>
#include <vector>

namespace pars_b200 {

// The reference's Rng (rng.hpp:22-75): mt19937_64 + hand-coded samplers.
class Rng {
 public:
  explicit Rng(uint64_t seed) : eng_(seed) {}
  uint64_t u64() { return eng_(); }
  double uniform01() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t n) {
    return static_cast<uint64_t>((static_cast<unsigned __int128>(eng_()) * n) >> 64);
  }
  double exponential(double rate) { return -std::log1p(-uniform01()) / rate; }
  double normal() {
    if (have_spare_) {
      have_spare_ = false;
      return spare_;
    }
    constexpr double kTwoPi = 6.283185307179586476925286766559;
    double u1 = 1.0 - uniform01();
    double u2 = uniform01();
    double r = std::sqrt(-2.0 * std::log(u1));
    double a = kTwoPi * u2;
    spare_ = r * std::sin(a);
    have_spare_ = true;
    return r * std::cos(a);
  }
  template <class T>
  void shuffle(std::vector<T>& v) {
    for (size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[below(i)]);
  }

 private:
  std::mt19937_64 eng_;
  double spare_ = 0.0;
  bool have_spare_ = false;
};

inline void append_u64(std::string& s, uint64_t v) {
  char buf[24];
  int n = 0;
  do {
    buf[n++] = (char)('0' + v % 10);
    v /= 10;
  } while (v);
  while (n) s.push_back(buf[--n]);
}
inline void append_i64(std::string& s, int64_t v) {
  if (v < 0) {
    s.push_back('-');
    append_u64(s, (uint64_t)(-(v + 1)) + 1);
  } else {
    append_u64(s, (uint64_t)v);
  }
}

}  // namespace pars_b200
