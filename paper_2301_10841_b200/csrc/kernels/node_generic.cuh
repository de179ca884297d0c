// node_generic: generic node kernel k_expand (Fig 13) and its per-candidate state
// Included by engine.cu (one translation unit: the kernels share templates and helpers).
#pragma once

// ============================================================================
// k_expand: iterate cover, probe, compact / aggregate  (Fig 13)
// ============================================================================
enum ExpandMode { EXPAND_WRITE = 0, EXPAND_COUNT = 1, EXPAND_ENUM = 2, EXPAND_MEMO = 3 };

__device__ __forceinline__ uint64_t upper_bound_u64(const uint64_t* __restrict__ a, uint64_t lo, uint64_t hi,
                                                    uint64_t x) {
  // first index in [lo, hi] with a[idx] > x (a[hi] > x guaranteed)
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) > x)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

// Load-balanced search, pass 1: bounds[t] = entry owning candidate c0 + t*TILE
// (bounds[ntiles] = F-1). Each k_expand tile then searches only
// [bounds[t], bounds[t+1]] instead of the whole scan.
constexpr int TILE = 256;
#ifndef FJG_LAST_CHUNK_LOG
#define FJG_LAST_CHUNK_LOG 31  // with ticketed chunks one launch is best (C2 last node 3.20 ms at 2^27, 3.03 at 2^31)
#endif
static_assert(FJG_LAST_CHUNK_LOG >= 12 && FJG_LAST_CHUNK_LOG <= 31,
              "k_chunk_marks uses 32-bit candidate offsets within a launch: FJG_LAST_CHUNK_LOG must be <= 31");
constexpr uint64_t kLastChunk = 1ull << FJG_LAST_CHUNK_LOG;  // last-node candidates per launch
__global__ void k_tile_bounds(const uint64_t* __restrict__ scan, uint64_t F, uint64_t c0, uint64_t c1,
                              uint64_t* __restrict__ bounds) {
  const uint64_t ntiles = (c1 - c0 + TILE - 1) / TILE;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t <= ntiles;
       t += (uint64_t)gridDim.x * blockDim.x)
    bounds[t] = (t == ntiles) ? F - 1 : upper_bound_u64(scan, 0, F - 1, c0 + t * TILE);
}

// Owner of every CHUNK-candidate chunk of [c0, c1) (the binding containing the
// chunk's first candidate), pass 1: each binding marks the first chunk start
// inside its candidate range (owner[] zeroed first); an inclusive max-scan
// then fills the rest (owners grow with the chunk index). owner[nchunks] =
// owner of c1 - 1. A thread's run then searches only [owner[t], owner[t+1]],
// which is usually a single binding.
__global__ void k_chunk_marks(const uint64_t* __restrict__ scan, uint64_t F, uint64_t c0, uint64_t c1, uint32_t chunk,
                              uint32_t* __restrict__ owner) {
  // chunk is a power of two and c1 - c0 <= kLastChunk (2^31): 32-bit shifts, no 64-bit division
  const uint32_t sh = __ffs(chunk) - 1;
  const uint32_t nch = (uint32_t)(c1 - c0 + chunk - 1) >> sh;
  // only the bindings whose candidates overlap [c0, c1): a contiguous range of
  // the frontier (a launch that starts at 0 / ends at the total skips the search;
  // the zero-candidate bindings it then visits fall through lo >= hi)
  const uint64_t elo = c0 == 0 ? 0 : upper_bound_u64(scan, 0, F - 1, c0);
  const uint64_t ehi = c1 >= __ldg(scan + F - 1) ? F - 1 : upper_bound_u64(scan, 0, F - 1, c1 - 1);
  for (uint64_t e = elo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e <= ehi;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t prev = e ? __ldg(scan + e - 1) : 0ull, se = __ldg(scan + e);
    const uint64_t lo = max(prev, c0), hi = min(se, c1);
    if (lo >= hi) continue;
    const uint32_t c = ((uint32_t)(lo - c0) + chunk - 1) >> sh;
    if (((uint64_t)c << sh) + c0 < hi) owner[c] = (uint32_t)e;
    if (hi == c1) owner[nch] = (uint32_t)e;
  }
}

// Register-resident helpers: W bounds the variables / atoms of the query at
// compile time so every per-candidate array stays in registers.
// (arithmetic blends: a plain `if (u == v) a[u] = x` is pattern-matched back
// into an indexed local-memory store)
template <int W>
__device__ __forceinline__ int32_t sel(const int32_t (&a)[W], int v) {
  int32_t x = 0;
#pragma unroll
  for (int u = 0; u < W; ++u) x |= a[u] & -(int32_t)(u == v);
  return x;
}

template <int W>
__device__ __forceinline__ void put(int32_t (&a)[W], int v, int32_t x) {
#pragma unroll
  for (int u = 0; u < W; ++u) {
    const int32_t m = -(int32_t)(u == v);
    a[u] = (x & m) | (a[u] & ~m);
  }
}

template <int W>
__device__ __forceinline__ void put2(uint32_t (&a)[W], uint32_t (&b)[W], int v, uint32_t x, uint32_t y) {
#pragma unroll
  for (int u = 0; u < W; ++u) {
    const uint32_t m = 0u - (uint32_t)(u == v);
    a[u] = (x & m) | (a[u] & ~m);
    b[u] = (y & m) | (b[u] & ~m);
  }
}

template <int W>
__device__ __forceinline__ uint32_t selu_(const uint32_t (&a)[W], int v) {
  uint32_t x = 0;
#pragma unroll
  for (int u = 0; u < W; ++u) x |= a[u] & (0u - (uint32_t)(u == v));
  return x;
}

// Per-candidate binding state. Narrow queries (W = 4) keep it in registers
// with arithmetic-blend selects; wider ones (W >= 8, where a blend costs W
// instructions per access) keep it in shared memory, variable-major so the
// lanes of a warp hit distinct banks.
template <int W>
struct RegState {
  int32_t val[W];
  uint32_t cp[W], cl[W];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int u = 0; u < W; ++u) val[u] = cp[u] = cl[u] = 0;
  }
  __device__ __forceinline__ int32_t get(int v) const { return sel(val, v); }
  __device__ __forceinline__ void set(int v, int32_t x) { put(val, v, x); }
  __device__ __forceinline__ int32_t at(int u) const { return val[u]; }
  __device__ __forceinline__ void seta(int u, int32_t x) { val[u] = x; }
  __device__ __forceinline__ void setc(int a, uint32_t p, uint32_t l) { put2(cp, cl, a, p, l); }
  __device__ __forceinline__ void setca(int a, uint32_t p, uint32_t l) {
    cp[a] = p;
    cl[a] = l;
  }
  __device__ __forceinline__ uint32_t cpa(int a) const { return cp[a]; }
  __device__ __forceinline__ uint32_t cla(int a) const { return cl[a]; }
  __device__ __forceinline__ uint32_t cpd(int a) const { return selu_(cp, a); }
};

template <int W>
struct SmemState {
  int32_t* val;
  uint32_t *cp, *cl;
  __device__ __forceinline__ SmemState(int32_t* sv, uint32_t* sp, uint32_t* sl)
      : val(sv + threadIdx.x), cp(sp + threadIdx.x), cl(sl + threadIdx.x) {}
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int u = 0; u < W; ++u) val[u * TILE] = cp[u * TILE] = cl[u * TILE] = 0;
  }
  __device__ __forceinline__ int32_t get(int v) const { return val[v * TILE]; }
  __device__ __forceinline__ void set(int v, int32_t x) { val[v * TILE] = x; }
  __device__ __forceinline__ int32_t at(int u) const { return val[u * TILE]; }
  __device__ __forceinline__ void seta(int u, int32_t x) { val[u * TILE] = x; }
  __device__ __forceinline__ void setc(int a, uint32_t p, uint32_t l) {
    cp[a * TILE] = p;
    cl[a * TILE] = l;
  }
  __device__ __forceinline__ void setca(int a, uint32_t p, uint32_t l) { setc(a, p, l); }
  __device__ __forceinline__ uint32_t cpa(int a) const { return cp[a * TILE]; }
  __device__ __forceinline__ uint32_t cla(int a) const { return cl[a * TILE]; }
  __device__ __forceinline__ uint32_t cpd(int a) const { return cp[a * TILE]; }
};

template <class St, int W>
__device__ __forceinline__ St make_state(uint32_t* smem) {
  if constexpr (W >= 8) {
    return St(reinterpret_cast<int32_t*>(smem), smem + W * TILE, smem + 2 * W * TILE);
  } else {
    return St();
  }
}

// One candidate: iterate the chosen cover at position j of entry e, then probe
// every other subatom of the node in order. Returns false if the candidate dies.
template <int MODE, int W, class St>
__device__ __forceinline__ bool run_candidate(const KNode& N, uint64_t e, uint64_t j, St& st, uint64_t& mult,
                                              uint64_t& probes, uint64_t& misses, uint64_t& body) {
#pragma unroll
  for (int v = 0; v < W; ++v)
    if ((N.in_vars >> v) & 1u) st.seta(v, __ldg(N.in_var[v] + e));
  if (MODE == EXPAND_WRITE) {
#pragma unroll
    for (int a = 0; a < W; ++a)
      if ((N.in_atoms >> a) & 1u) st.setca(a, __ldg(N.in_p[a] + e), __ldg(N.in_len[a] + e));
  }
  if (N.in_mult) mult = __ldg(N.in_mult + e);
  // ---- iterate the chosen cover (Fig 12 iter) ----
  const int ci = N.chosen[e];
  const KSub& S = N.sub[ci];
  uint32_t p, len;
  subtrie_of(S, e, p, len);
  if (p == kSingleton) {
    st.setc(S.atom, kSingleton, 1u);
  } else {
    const uint32_t pos = p + (uint32_t)j;
    if (!S.stream) {
      // forced map: distinct keys are the child starts
      const uint32_t c = __ldg(S.cnt + pos);
      if (c == 0) return false;
      st.setc(S.atom, pos, c);
    } else {
      st.setc(S.atom, kSingleton, 1u);  // suffix: stream values at the offsets
    }
#pragma unroll
    for (int t = 0; t < MAXK; ++t)
      if (t < S.nv) {
        const int32_t x = __ldg(S.src[t] + pos);
        const int v = S.var[t];
        if ((S.bound_mask >> t) & 1) {
          if (st.get(v) != x) return false;  // cover re-binds a bound variable
        } else {
          st.set(v, x);
        }
      }
  }
  ++body;  // the node body runs for this cover tuple (ExecStats.node_body_entries)
  // ---- probe every other subatom in node order (Fig 13 inner loop) ----
  for (int s = 0; s < N.nsub; ++s) {
    if (s == ci) continue;
    const KSub& P = N.sub[s];
    uint32_t pp, pl;
    subtrie_of(P, e, pp, pl);
    uint32_t q = kSingleton, ql = 1;
    if (pp != kSingleton) {
      int32_t key[MAXK];
#pragma unroll
      for (int t = 0; t < MAXK; ++t) key[t] = t < P.nv ? st.get(P.var[t]) : 0;
      ++probes;
      if (!colt_get(P, pp, pl, key, q, ql)) {
        ++misses;
        return false;
      }
    }
    if (P.last)
      mult *= ql;  // residual leaf vector: its offsets are the multiplicity
    else
      st.setc(P.atom, q, ql);
  }
  return true;
}

#ifndef FJG_EXPAND_MINBLOCKS
#define FJG_EXPAND_MINBLOCKS 1
#endif
template <int MODE, int W>
__global__ void __launch_bounds__(TILE, FJG_EXPAND_MINBLOCKS) k_expand(const __grid_constant__ KNode N, uint64_t c0,
                                                                       uint64_t c1, uint64_t F,
                                                                       const uint64_t* __restrict__ bounds,
                                                                       int min_var, int32_t* __restrict__ out_tuples,
                                                                       uint64_t out_cap, DevCounters* ctr) {
  __shared__ uint32_t s_warp[TILE / 32];
  __shared__ uint32_t s_base;
  extern __shared__ uint32_t s_state[];  // W >= 8: 3 * W * TILE words
  uint64_t acc_lo = 0, acc_hi = 0, acc_sum = 0, probes = 0, misses = 0, body = 0;
  long long acc_min = LLONG_MAX;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t* __restrict__ scan = N.scan;
  using St = typename std::conditional<(W >= 8), SmemState<W>, RegState<W>>::type;

  for (uint64_t base = c0 + (uint64_t)blockIdx.x * TILE; base < c1; base += (uint64_t)gridDim.x * TILE) {
    const uint64_t t = (base - c0) / TILE;
    const uint64_t lo = __ldg(bounds + t), hi = __ldg(bounds + t + 1);
    const uint64_t i = base + threadIdx.x;
    bool alive = i < c1;
    St st = make_state<St, W>(s_state);
    st.init();
    uint64_t mult = 1;
    if (alive) {
      const uint64_t e = upper_bound_u64(scan, lo, hi, i);
      const uint64_t j = i - (e ? __ldg(scan + e - 1) : 0ull);
      alive = run_candidate<MODE, W>(N, e, j, st, mult, probes, misses, body);
    }
    if (MODE == EXPAND_WRITE) {
      const unsigned bal = __ballot_sync(0xffffffffu, alive);
      if (lane == 0) s_warp[warp] = __popc(bal);
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t tot = 0;
        for (int w = 0; w < TILE / 32; ++w) {
          const uint32_t c = s_warp[w];
          s_warp[w] = tot;
          tot += c;
        }
        s_base = tot ? atomicAdd(&ctr->survivors, tot) : 0u;
      }
      __syncthreads();
      if (alive) {
        const uint32_t o = s_base + s_warp[warp] + __popc(bal & ((1u << lane) - 1));
#pragma unroll
        for (int v = 0; v < W; ++v)
          if ((N.out_vars >> v) & 1u) N.out_var[v][o] = st.at(v);
#pragma unroll
        for (int a = 0; a < W; ++a)
          if ((N.out_atoms >> a) & 1u) {
            N.out_p[a][o] = st.cpa(a);
            N.out_len[a][o] = st.cla(a);
          }
        if (N.out_mult) N.out_mult[o] = mult;
      }
      __syncthreads();
    } else if (alive) {
      if (MODE == EXPAND_COUNT || MODE == EXPAND_ENUM) {  // enumerating folds the count / checksum too
        uint64_t h = fj::kTupleHashSeed;
#pragma unroll
        for (int v = 0; v < W; ++v)
          if (v < N.nhead) h = fj::tuple_hash_step(h, (int64_t)st.at(v));
        acc_sum += mult * fj::checksum_word(h);
        acc_lo += mult;
        if (acc_lo < mult) ++acc_hi;
        if (min_var >= 0) acc_min = min(acc_min, (long long)st.get(min_var));
      } else if (MODE == EXPAND_MEMO) {
        // memoised chain suffix: this binding contributes mult * count(child of the carrier)
        const uint64_t g = __ldg(N.memo_gid + st.cpd(N.memo_atom)) - 1u;
        const unsigned __int128 mv =
            ((unsigned __int128)N.memo[2ull * g + 1] << 64) | (unsigned __int128)N.memo[2ull * g];
        const unsigned __int128 c = mv * mult + (((unsigned __int128)acc_hi << 64) | acc_lo);
        acc_lo = (uint64_t)c;
        acc_hi = (uint64_t)(c >> 64);
      }
      if (MODE == EXPAND_ENUM) {
        const unsigned long long o = atomicAdd((unsigned long long*)&ctr->out_rows, (unsigned long long)mult);
        for (uint64_t r = 0; r < mult && o + r < out_cap; ++r)
#pragma unroll
          for (int v = 0; v < W; ++v)
            if (v < N.nhead) out_tuples[(o + r) * N.nhead + v] = st.at(v);
      }
    }
  }
  // ---- flush per-thread accumulators: one atomic per warp ----
  probes = warp_sum(probes);
  misses = warp_sum(misses);
  body = warp_sum(body);
  if (lane == 0) {
    if (probes) {
      atomicAdd((unsigned long long*)&ctr->probes, (unsigned long long)probes);
      atomicAdd((unsigned long long*)&ctr->node_probes[N.k], (unsigned long long)probes);
    }
    if (misses) atomicAdd((unsigned long long*)&ctr->misses, (unsigned long long)misses);
    if (body) atomicAdd((unsigned long long*)&ctr->body[N.k], (unsigned long long)body);
  }
  if (MODE == EXPAND_COUNT || MODE == EXPAND_MEMO || MODE == EXPAND_ENUM) {
    // 128-bit count: carry out of the low word
    uint64_t lo = acc_lo, hi = acc_hi;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t l2 = __shfl_xor_sync(0xffffffffu, lo, o);
      const uint64_t h2 = __shfl_xor_sync(0xffffffffu, hi, o);
      const uint64_t s = lo + l2;
      hi += h2 + (s < lo ? 1 : 0);
      lo = s;
    }
    acc_sum = warp_sum(acc_sum);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc_min = min(acc_min, __shfl_xor_sync(0xffffffffu, acc_min, o));
    if (lane == 0) {
      if (lo) {
        const unsigned long long old = atomicAdd((unsigned long long*)&ctr->count_lo, (unsigned long long)lo);
        if (old + lo < old) ++hi;
      }
      if (hi) atomicAdd((unsigned long long*)&ctr->count_hi, (unsigned long long)hi);
      if (acc_sum) atomicAdd((unsigned long long*)&ctr->checksum, (unsigned long long)acc_sum);
      if (acc_min != LLONG_MAX) atomicMin(&ctr->minv, acc_min);
    }
  }
}

