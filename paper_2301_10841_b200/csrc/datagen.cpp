// Seeded synthetic inputs for the BASELINE.json configs (libfjgen.so).
//
// The paper measured on JOB/LSQB, which are absent here;
// BASELINE.json's five configs stand in for them with seeded synthetic data
// (SURVEY.md §8(d)). Every generator is a pure function of (parameters, seed)
// built on a counter-based RNG, so the oracle and the device read identical
// bytes on any machine. "M" = 2^20 rows (SURVEY.md §8 config shorthand).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "rmat.hpp"

namespace {

using fjgen::rmat_edge;
using fjgen::rng;
using fjgen::splitmix64;
using fjgen::u01;

template <class F>
void parallel_for(uint64_t n, F&& f) {
  unsigned T = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (n < 65536) T = 1;
  std::vector<std::thread> th;
  for (unsigned t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      const uint64_t lo = n * t / T, hi = n * (t + 1) / T;
      for (uint64_t i = lo; i < hi; ++i) f(i);
    });
  for (auto& x : th) x.join();
}

std::string g_err;

}  // namespace

extern "C" {

const char* fjgen_last_error(void) { return g_err.c_str(); }

// Uniform int32 column values in [0, domain): column `col` of a table, seed s.
void fjgen_uniform(uint64_t seed, uint32_t col, uint64_t n, uint64_t domain, int32_t* out) {
  parallel_for(n, [&](uint64_t i) { out[i] = (int32_t)(rng(seed, col, i) % domain); });
}

// Zipf(s) over [0, k): P(v) ∝ 1/(v+1)^s, by inverse CDF.
int fjgen_zipf(uint64_t seed, uint32_t stream, uint64_t n, uint64_t k, double s, int32_t* out) {
  try {
    std::vector<double> cdf(k);
    double acc = 0;
    for (uint64_t v = 0; v < k; ++v) {
      acc += 1.0 / std::pow((double)(v + 1), s);
      cdf[v] = acc;
    }
    for (auto& x : cdf) x /= acc;
    cdf[k - 1] = 1.0;
    parallel_for(n, [&](uint64_t i) {
      const double r = u01(rng(seed, stream, i));
      out[i] = (int32_t)(std::upper_bound(cdf.begin(), cdf.end(), r) - cdf.begin());
      if (out[i] >= (int32_t)k) out[i] = (int32_t)(k - 1);
    });
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

// R-MAT graph with exactly m distinct directed edges, no self-loops: the
// first m distinct non-loop edges of the seeded candidate stream, in stream
// order (so rows are in random order, not sorted).
int fjgen_rmat(uint64_t seed, int scale, uint64_t m, double a, double b, double c, int32_t* src, int32_t* dst) {
  try {
    if (scale < 1 || scale > 31) throw std::runtime_error("scale must be 1..31");
    uint64_t K = m + m / 4 + 1024;
    while (true) {
      std::vector<uint64_t> cand(K);
      parallel_for(K, [&](uint64_t i) { cand[i] = rmat_edge(seed, i, scale, a, b, c); });
      // (key, index) pairs; keep the first occurrence of each non-loop key
      std::vector<std::pair<uint64_t, uint64_t>> kv(K);
      parallel_for(K, [&](uint64_t i) { kv[i] = {cand[i], i}; });
      std::sort(kv.begin(), kv.end());
      std::vector<uint64_t> first;
      first.reserve(m + 16);
      for (uint64_t i = 0; i < K; ++i) {
        if (i && kv[i].first == kv[i - 1].first) continue;
        if ((kv[i].first >> 32) == (kv[i].first & 0xffffffffULL)) continue;
        first.push_back(kv[i].second);
      }
      if (first.size() >= m) {
        std::sort(first.begin(), first.end());
        for (uint64_t i = 0; i < m; ++i) {
          const uint64_t e = cand[first[i]];
          src[i] = (int32_t)(e >> 32);
          dst[i] = (int32_t)(e & 0xffffffffULL);
        }
        return 0;
      }
      K = K + K / 2;
    }
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory in fjgen_rmat";
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

// Orient an edge list for clique counting: symmetrise, dedup, drop loops,
// orient every undirected edge from lower to higher (degree, id) rank, output
// in a seeded pseudo-random order. Returns the number of oriented edges
// written to (osrc, odst) (capacity n).
int64_t fjgen_orient(uint64_t seed, const int32_t* src, const int32_t* dst, uint64_t n, int32_t* osrc,
                     int32_t* odst) {
  try {
    std::vector<uint64_t> und;
    und.reserve(n);
    for (uint64_t i = 0; i < n; ++i) {
      uint32_t u = (uint32_t)src[i], v = (uint32_t)dst[i];
      if (u == v) continue;
      if (u > v) std::swap(u, v);
      und.push_back(((uint64_t)u << 32) | v);
    }
    std::sort(und.begin(), und.end());
    und.erase(std::unique(und.begin(), und.end()), und.end());
    uint32_t maxv = 0;
    for (uint64_t e : und) maxv = std::max<uint32_t>(maxv, (uint32_t)(e & 0xffffffffULL));
    std::vector<uint32_t> deg((uint64_t)maxv + 1, 0);
    for (uint64_t e : und) {
      ++deg[e >> 32];
      ++deg[e & 0xffffffffULL];
    }
    std::vector<std::pair<uint64_t, uint64_t>> out;  // (shuffle key, oriented edge)
    out.reserve(und.size());
    for (uint64_t e : und) {
      uint32_t u = (uint32_t)(e >> 32), v = (uint32_t)(e & 0xffffffffULL);
      const bool u_first = deg[u] < deg[v] || (deg[u] == deg[v] && u < v);
      if (!u_first) std::swap(u, v);
      const uint64_t oe = ((uint64_t)u << 32) | v;
      out.push_back({splitmix64(oe ^ splitmix64(seed)), oe});
    }
    std::sort(out.begin(), out.end());
    for (uint64_t i = 0; i < out.size(); ++i) {
      osrc[i] = (int32_t)(out[i].second >> 32);
      odst[i] = (int32_t)(out[i].second & 0xffffffffULL);
    }
    return (int64_t)out.size();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"
