// Counter-based R-MAT edge stream shared by the host (datagen.cpp) and device
// (datagen_dev.cu) generators so both produce identical relations.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define FJGEN_HD __host__ __device__ __forceinline__
#else
#define FJGEN_HD inline
#endif

namespace fjgen {

FJGEN_HD uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
// value i of stream (seed, stream)
FJGEN_HD uint64_t rng(uint64_t seed, uint64_t stream, uint64_t i) {
  return splitmix64(splitmix64(seed * 0x100000001b3ULL + stream) ^ (i * 0xd1b54a32d192ed03ULL));
}
FJGEN_HD double u01(uint64_t x) { return (double)(x >> 11) * (1.0 / 9007199254740992.0); }

// R-MAT edge i: `scale` quadrant draws with probabilities (a, b, c, 1-a-b-c);
// returns (src << 32) | dst.
FJGEN_HD uint64_t rmat_edge(uint64_t seed, uint64_t i, int scale, double a, double b, double c) {
  uint64_t s = 0, d = 0;
  for (int l = 0; l < scale; ++l) {
    const double r = u01(rng(seed, 1000 + l, i));
    uint64_t sb = 0, db = 0;
    if (r < a) {
    } else if (r < a + b) {
      db = 1;
    } else if (r < a + b + c) {
      sb = 1;
    } else {
      sb = db = 1;
    }
    s = (s << 1) | sb;
    d = (d << 1) | db;
  }
  return (s << 32) | d;
}

}  // namespace fjgen
