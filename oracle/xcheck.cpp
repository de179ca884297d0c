// XCHECK — TEST INFRASTRUCTURE ONLY. Independent graph-pattern counters used to
// cross-check the Free Join oracle (oracle/fj_oracle.cpp) and the device path on
// the graph configs ("oracle equivalence").
//
// Nothing here follows the Free Join / COLT algorithm: the counters work on a
// plain CSR adjacency (sorted out-neighbour lists) with a per-thread bitmap, the
// textbook way to list triangles and cliques. They share only the output
// definition with the oracle:
//   count    = number of output tuples (edges are distinct, so every output
//              tuple has multiplicity 1);
//   checksum = sum over outputs of fmix64(TupleHash(t)) mod 2^64, t in the
//              query's head-variable order (value.hpp:61-67 TupleHash; the
//              checksum convention of SURVEY.md §8(c), fj_oracle.cpp:41-53).
//
// xc_triangles: Q(a,b,c) :- E(a,b),E(b,c),E(a,c) over directed edges (C2, C5).
// xc_clique4:   Q(a,b,c,d) :- Eab,Eac,Ebc,Ead,Ebd,Ecd over one oriented edge
//               set (C4): a->b, a->c, b->c, a->d, b->d, c->d.
// xc_path_walks: number of 5-edge walks (1^T A^5 1) mod 2^64 and mod two primes
//               (C5 5-path, count only).
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

inline uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}
inline uint64_t th_step(uint64_t h, int64_t v) { return (h ^ static_cast<uint64_t>(v)) * 0x100000001b3ULL; }
constexpr uint64_t kSeed = 0x811c9dc5ULL;

struct Csr {
  uint32_t nv = 0;
  std::vector<uint64_t> off;   // nv + 1
  std::vector<int32_t> adj;    // sorted per vertex
};

// Counting-sort CSR over out-neighbours; lists sorted ascending.
Csr build_csr(const int32_t* src, const int32_t* dst, uint64_t m, int nthreads) {
  Csr g;
  int32_t mx = -1;
  for (uint64_t i = 0; i < m; ++i) mx = std::max(mx, std::max(src[i], dst[i]));
  g.nv = static_cast<uint32_t>(mx + 1);
  g.off.assign(static_cast<uint64_t>(g.nv) + 1, 0);
  for (uint64_t i = 0; i < m; ++i) ++g.off[static_cast<uint32_t>(src[i]) + 1];
  for (uint32_t v = 0; v < g.nv; ++v) g.off[v + 1] += g.off[v];
  g.adj.resize(m);
  std::vector<uint64_t> cur(g.off.begin(), g.off.end() - 1);
  for (uint64_t i = 0; i < m; ++i) g.adj[cur[static_cast<uint32_t>(src[i])]++] = dst[i];
  std::atomic<uint32_t> next{0};
  std::vector<std::thread> ts;
  for (int t = 0; t < nthreads; ++t)
    ts.emplace_back([&] {
      for (;;) {
        const uint32_t v0 = next.fetch_add(4096);
        if (v0 >= g.nv) break;
        const uint32_t v1 = std::min<uint32_t>(g.nv, v0 + 4096);
        for (uint32_t v = v0; v < v1; ++v) std::sort(g.adj.begin() + g.off[v], g.adj.begin() + g.off[v + 1]);
      }
    });
  for (auto& t : ts) t.join();
  return g;
}

struct Acc {
  unsigned __int128 count = 0;
  uint64_t checksum = 0;
};

// Vertices handed out in chunks from an atomic counter, heaviest (by out-degree)
// first so that the hubs do not end up on one thread at the end.
template <class F>
Acc run_vertices(const Csr& g, int nthreads, F&& per_vertex) {
  std::vector<uint32_t> order(g.nv);
  for (uint32_t v = 0; v < g.nv; ++v) order[v] = v;
  std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) {
    return (g.off[x + 1] - g.off[x]) > (g.off[y + 1] - g.off[y]);
  });
  std::atomic<uint64_t> next{0};
  std::vector<Acc> acc(nthreads);
  std::vector<std::thread> ts;
  for (int t = 0; t < nthreads; ++t)
    ts.emplace_back([&, t] {
      std::vector<uint64_t> bits((static_cast<uint64_t>(g.nv) + 63) / 64, 0);
      Acc a;
      for (;;) {
        const uint64_t i0 = next.fetch_add(64);
        if (i0 >= g.nv) break;
        const uint64_t i1 = std::min<uint64_t>(g.nv, i0 + 64);
        for (uint64_t i = i0; i < i1; ++i) per_vertex(order[i], bits, a);
      }
      acc[t] = a;
    });
  for (auto& t : ts) t.join();
  Acc r;
  for (auto& a : acc) {
    r.count += a.count;
    r.checksum += a.checksum;
  }
  return r;
}

inline void set_bits(std::vector<uint64_t>& b, const int32_t* p, uint64_t n, bool on) {
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t c = static_cast<uint32_t>(p[i]);
    if (on)
      b[c >> 6] |= 1ULL << (c & 63);
    else
      b[c >> 6] &= ~(1ULL << (c & 63));
  }
}
inline bool test_bit(const std::vector<uint64_t>& b, int32_t c) {
  return (b[static_cast<uint32_t>(c) >> 6] >> (static_cast<uint32_t>(c) & 63)) & 1;
}

}  // namespace

extern "C" {

// count returned as two 64-bit limbs. nparts > 1: only outputs whose first
// variable a has partition_of(a, nparts) == part (fmix64(a ^ 0x5bd1e995) mod
// nparts, the multi-GPU partition function, fj_oracle.cpp:55-57).
int xc_triangles(const int32_t* src, const int32_t* dst, uint64_t m, int nthreads, uint32_t nparts,
                 uint32_t part, uint64_t* count_lo, uint64_t* count_hi, uint64_t* checksum) {
  if (nthreads < 1) nthreads = 1;
  const Csr g = build_csr(src, dst, m, nthreads);
  const Acc r = run_vertices(g, nthreads, [&](uint32_t a, std::vector<uint64_t>& bits, Acc& acc) {
    if (nparts > 1 && fmix64(static_cast<uint64_t>(static_cast<int64_t>(a)) ^ 0x5bd1e995ULL) % nparts != part)
      return;
    const int32_t* na = g.adj.data() + g.off[a];
    const uint64_t da = g.off[a + 1] - g.off[a];
    if (da == 0) return;
    set_bits(bits, na, da, true);  // out(a)
    const uint64_t ha = th_step(kSeed, a);
    for (uint64_t i = 0; i < da; ++i) {
      const int32_t b = na[i];
      const int32_t* nb = g.adj.data() + g.off[b];
      const uint64_t db = g.off[b + 1] - g.off[b];
      const uint64_t hab = th_step(ha, b);
      if (db <= da) {  // c in out(b), test c in out(a)
        for (uint64_t j = 0; j < db; ++j)
          if (test_bit(bits, nb[j])) {
            ++acc.count;
            acc.checksum += fmix64(th_step(hab, nb[j]));
          }
      } else {  // c in out(a), test c in out(b) by binary search
        for (uint64_t j = 0; j < da; ++j)
          if (std::binary_search(nb, nb + db, na[j])) {
            ++acc.count;
            acc.checksum += fmix64(th_step(hab, na[j]));
          }
      }
    }
    set_bits(bits, na, da, false);
  });
  *count_lo = static_cast<uint64_t>(r.count);
  *count_hi = static_cast<uint64_t>(r.count >> 64);
  *checksum = r.checksum;
  return 0;
}

int xc_clique4(const int32_t* src, const int32_t* dst, uint64_t m, int nthreads, uint64_t* count_lo,
               uint64_t* count_hi, uint64_t* checksum) {
  if (nthreads < 1) nthreads = 1;
  const Csr g = build_csr(src, dst, m, nthreads);
  const Acc r = run_vertices(g, nthreads, [&](uint32_t a, std::vector<uint64_t>& bits, Acc& acc) {
    const int32_t* na = g.adj.data() + g.off[a];
    const uint64_t da = g.off[a + 1] - g.off[a];
    if (da < 3) return;
    set_bits(bits, na, da, true);
    const uint64_t ha = th_step(kSeed, a);
    std::vector<int32_t> ab, abc;
    for (uint64_t i = 0; i < da; ++i) {
      const int32_t b = na[i];
      ab.clear();
      for (uint64_t j = g.off[b]; j < g.off[b + 1]; ++j)
        if (test_bit(bits, g.adj[j])) ab.push_back(g.adj[j]);  // c in out(a) & out(b), sorted
      if (ab.size() < 2) continue;
      const uint64_t hab = th_step(ha, b);
      for (const int32_t c : ab) {
        const int32_t* nc = g.adj.data() + g.off[c];
        const uint64_t dc = g.off[c + 1] - g.off[c];
        abc.clear();
        std::set_intersection(ab.begin(), ab.end(), nc, nc + dc, std::back_inserter(abc));
        const uint64_t habc = th_step(hab, c);
        for (const int32_t d : abc) {
          ++acc.count;
          acc.checksum += fmix64(th_step(habc, d));
        }
      }
    }
    set_bits(bits, na, da, false);
  });
  *count_lo = static_cast<uint64_t>(r.count);
  *count_hi = static_cast<uint64_t>(r.count >> 64);
  *checksum = r.checksum;
  return 0;
}

// Walks with `len` edges: x_0 = 1, x_{k+1}[u] = sum_{u->v} x_k[v]; result sum x_len.
// Exact modulo 2^64 and modulo each of `nmods` primes (out[0] = mod 2^64, out[1+i]).
int xc_walks(const int32_t* src, const int32_t* dst, uint64_t m, int len, const uint64_t* mods, int nmods,
             int nthreads, uint64_t* out) {
  if (nthreads < 1) nthreads = 1;
  const Csr g = build_csr(src, dst, m, nthreads);
  for (int k = -1; k < nmods; ++k) {
    const uint64_t p = k < 0 ? 0 : mods[k];
    std::vector<uint64_t> x(g.nv, 1), y(g.nv);
    for (int step = 0; step < len; ++step) {
      std::atomic<uint32_t> next{0};
      std::vector<std::thread> ts;
      for (int t = 0; t < nthreads; ++t)
        ts.emplace_back([&] {
          for (;;) {
            const uint32_t v0 = next.fetch_add(8192);
            if (v0 >= g.nv) break;
            const uint32_t v1 = std::min<uint32_t>(g.nv, v0 + 8192);
            for (uint32_t u = v0; u < v1; ++u) {
              unsigned __int128 s = 0;
              for (uint64_t j = g.off[u]; j < g.off[u + 1]; ++j) s += x[g.adj[j]];
              y[u] = p ? static_cast<uint64_t>(s % p) : static_cast<uint64_t>(s);
            }
          }
        });
      for (auto& t : ts) t.join();
      x.swap(y);
    }
    unsigned __int128 s = 0;
    for (uint32_t u = 0; u < g.nv; ++u) s += x[u];
    out[k + 1] = p ? static_cast<uint64_t>(s % p) : static_cast<uint64_t>(s);
  }
  return 0;
}

}  // extern "C"
