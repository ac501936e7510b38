// rmpc_oracle_rng.hpp — TEST INFRASTRUCTURE ONLY.
#pragma once

#include <cstdint>

namespace oracle {

// xoshiro256++ with splitmix64 seeding, restated from rng.hpp:15-75 (stream constructor
// Rng(seed, stream)).
struct Rng {
  uint64_t s[4];
  static uint64_t splitmix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  Rng(uint64_t seed, uint64_t stream) {
    uint64_t x = seed ^ splitmix(stream + 0x9e3779b97f4a7c15ULL);
    for (auto& w : s) {
      x += 0x9e3779b97f4a7c15ULL;
      w = splitmix(x);
    }
  }
  uint64_t next() {
    const uint64_t r = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }  // rng.hpp:41
  int uniform_int(int n) { return static_cast<int>(next() % static_cast<uint64_t>(n)); }  // rng.hpp:43
};


}  // namespace oracle
