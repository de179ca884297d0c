// ORACLE GENERATORS — TEST / BASELINE INFRASTRUCTURE ONLY. A second, independent
// implementation of the seeded synthetic inputs of the BASELINE.json configs
// (the product's libfjgen.so, paper_2301_10841_b200/csrc/datagen.cpp, defines
// them), so that the reference arm of bench.py and the oracle-side tests can
// produce the inputs without loading any product library. Same definitions,
// different code: parallel generation and a parallel hash-bucketed dedup instead
// of one global sort. tests/test_oracle_workloads.py checks both produce identical
// bytes.
//
// Definitions (seeded, counter-based, "M" = 2^20):
//   rng(seed, stream, i) = splitmix64(splitmix64(seed*0x100000001b3 + stream) ^ i*0xd1b54a32d192ed03)
//   uniform:  value i of column c = rng(seed, c, i) mod domain
//   zipf(s):  P(v) ∝ (v+1)^-s over [0,k), inverse CDF of u01(rng(seed, stream, i))
//   rmat:     candidate edge i draws `scale` quadrants, level l from
//             u01(rng(seed, 1000+l, i)); the relation is the first m distinct
//             non-loop candidates in stream order, from K = m + m/4 + 1024
//             candidates (K grows by K/2 until m are found)
//   orient:   symmetrise, dedup, drop loops, orient (deg, id) ascending, order
//             rows by splitmix64(edge ^ splitmix64(seed)), ties by edge
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace {

inline uint64_t sm64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
inline uint64_t draw(uint64_t seed, uint64_t stream, uint64_t i) {
  return sm64(sm64(seed * 0x100000001b3ULL + stream) ^ (i * 0xd1b54a32d192ed03ULL));
}
inline double unit(uint64_t x) { return static_cast<double>(x >> 11) * (1.0 / 9007199254740992.0); }

int threads() {
  const unsigned h = std::thread::hardware_concurrency();
  return static_cast<int>(std::max(1u, std::min(64u, h)));
}

// f(lo, hi) over [0, n) in T contiguous slices
template <class F>
void par(uint64_t n, F&& f) {
  const int T = n < 65536 ? 1 : threads();
  std::vector<std::thread> ts;
  for (int t = 0; t < T; ++t) ts.emplace_back([&, t] { f(n * t / T, n * (t + 1) / T); });
  for (auto& x : ts) x.join();
}

uint64_t rmat_candidate(uint64_t seed, uint64_t i, int scale, double a, double b, double c) {
  uint64_t s = 0, d = 0;
  for (int l = 0; l < scale; ++l) {
    const double r = unit(draw(seed, 1000 + l, i));
    const uint64_t sb = r >= a + b ? 1 : 0;                       // quadrants c, d
    const uint64_t db = (r >= a && r < a + b) || r >= a + b + c;  // quadrants b, d
    s = (s << 1) | sb;
    d = (d << 1) | db;
  }
  return (s << 32) | d;
}

}  // namespace

extern "C" {

void og_uniform(uint64_t seed, uint32_t col, uint64_t n, uint64_t domain, int32_t* out) {
  par(n, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) out[i] = static_cast<int32_t>(draw(seed, col, i) % domain);
  });
}

int og_zipf(uint64_t seed, uint32_t stream, uint64_t n, uint64_t k, double s, int32_t* out) {
  if (k == 0) return 1;
  std::vector<double> cdf(k);
  double acc = 0;
  for (uint64_t v = 0; v < k; ++v) {
    acc += 1.0 / std::pow(static_cast<double>(v + 1), s);
    cdf[v] = acc;
  }
  for (auto& x : cdf) x /= acc;
  cdf[k - 1] = 1.0;
  par(n, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) {
      const double r = unit(draw(seed, stream, i));
      const uint64_t v = static_cast<uint64_t>(std::upper_bound(cdf.begin(), cdf.end(), r) - cdf.begin());
      out[i] = static_cast<int32_t>(std::min(v, k - 1));
    }
  });
  return 0;
}

// Exactly m distinct non-loop directed edges: the first m such candidates in
// stream order. Dedup: candidates are bucketed by a hash of the key (a
// counting-sort pass), each bucket sorted by (key, index) in parallel, and the
// first occurrence of every non-loop key flagged; the flagged indices in
// increasing order are the stream-order firsts.
int og_rmat(uint64_t seed, int scale, uint64_t m, double a, double b, double c, int32_t* src, int32_t* dst) {
  if (scale < 1 || scale > 31) return 1;
  uint64_t K = m + m / 4 + 1024;
  for (;;) {
    std::vector<uint64_t> cand(K);
    par(K, [&](uint64_t lo, uint64_t hi) {
      for (uint64_t i = lo; i < hi; ++i) cand[i] = rmat_candidate(seed, i, scale, a, b, c);
    });
    const int bits = 12;  // buckets by a hash of the key: equal keys share a bucket, sizes stay even
    auto bucket = [&](uint64_t key) { return static_cast<uint32_t>(sm64(key) >> (64 - bits)); };
    const uint32_t NB = 1u << bits;
    const int T = K < 65536 ? 1 : threads();
    std::vector<std::vector<uint64_t>> hist(T, std::vector<uint64_t>(NB + 1, 0));
    std::vector<std::thread> ts;
    for (int t = 0; t < T; ++t)
      ts.emplace_back([&, t] {
        for (uint64_t i = K * t / T; i < K * (t + 1) / T; ++i) ++hist[t][bucket(cand[i])];
      });
    for (auto& x : ts) x.join();
    ts.clear();
    std::vector<uint64_t> bstart(NB + 1, 0);
    std::vector<std::vector<uint64_t>> pos(T, std::vector<uint64_t>(NB));
    uint64_t run = 0;
    for (uint32_t bk = 0; bk < NB; ++bk) {
      bstart[bk] = run;
      for (int t = 0; t < T; ++t) {
        pos[t][bk] = run;
        run += hist[t][bk];
      }
    }
    bstart[NB] = run;
    std::vector<uint32_t> idx(K);  // candidate indices, bucketed (stable within a thread slice)
    for (int t = 0; t < T; ++t)
      ts.emplace_back([&, t] {
        for (uint64_t i = K * t / T; i < K * (t + 1) / T; ++i) idx[pos[t][bucket(cand[i])]++] = static_cast<uint32_t>(i);
      });
    for (auto& x : ts) x.join();
    ts.clear();
    std::vector<uint8_t> keep(K, 0);
    std::atomic<uint32_t> next{0};
    for (int t = 0; t < T; ++t)
      ts.emplace_back([&] {
        for (;;) {
          const uint32_t bk = next.fetch_add(1);
          if (bk >= NB) break;
          uint32_t* lo = idx.data() + bstart[bk];
          uint32_t* hi = idx.data() + bstart[bk + 1];
          std::sort(lo, hi, [&](uint32_t x, uint32_t y) { return cand[x] != cand[y] ? cand[x] < cand[y] : x < y; });
          for (uint32_t* p = lo; p < hi; ++p) {
            const uint64_t key = cand[*p];
            if (p > lo && cand[p[-1]] == key) continue;
            if ((key >> 32) == (key & 0xffffffffULL)) continue;
            keep[*p] = 1;
          }
        }
      });
    for (auto& x : ts) x.join();
    uint64_t w = 0;
    for (uint64_t i = 0; i < K && w < m; ++i)
      if (keep[i]) {
        src[w] = static_cast<int32_t>(cand[i] >> 32);
        dst[w] = static_cast<int32_t>(cand[i] & 0xffffffffULL);
        ++w;
      }
    if (w == m) return 0;
    K = K + K / 2;
  }
}

// Returns the number of oriented edges written (capacity n).
int64_t og_orient(uint64_t seed, const int32_t* src, const int32_t* dst, uint64_t n, int32_t* osrc,
                  int32_t* odst) {
  std::vector<uint64_t> und;
  und.reserve(n);
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t u = static_cast<uint32_t>(src[i]), v = static_cast<uint32_t>(dst[i]);
    if (u != v) und.push_back(u < v ? (static_cast<uint64_t>(u) << 32) | v : (static_cast<uint64_t>(v) << 32) | u);
  }
  std::sort(und.begin(), und.end());
  und.erase(std::unique(und.begin(), und.end()), und.end());
  uint64_t nv = 0;
  for (const uint64_t e : und) nv = std::max<uint64_t>(nv, (e & 0xffffffffULL) + 1);
  std::vector<uint32_t> deg(nv, 0);
  for (const uint64_t e : und) {
    ++deg[e >> 32];
    ++deg[e & 0xffffffffULL];
  }
  const uint64_t salt = sm64(seed);
  std::vector<std::pair<uint64_t, uint64_t>> rows(und.size());
  for (size_t i = 0; i < und.size(); ++i) {
    uint32_t u = static_cast<uint32_t>(und[i] >> 32), v = static_cast<uint32_t>(und[i] & 0xffffffffULL);
    if (deg[v] < deg[u] || (deg[v] == deg[u] && v < u)) std::swap(u, v);
    const uint64_t oe = (static_cast<uint64_t>(u) << 32) | v;
    rows[i] = {sm64(oe ^ salt), oe};
  }
  std::sort(rows.begin(), rows.end());
  for (size_t i = 0; i < rows.size(); ++i) {
    osrc[i] = static_cast<int32_t>(rows[i].second >> 32);
    odst[i] = static_cast<int32_t>(rows[i].second & 0xffffffffULL);
  }
  return static_cast<int64_t>(rows.size());
}

}  // extern "C"
