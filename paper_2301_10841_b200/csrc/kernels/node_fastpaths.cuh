// node_fastpaths: shape-specialised node kernels: GJ last / frontier nodes, stream-cover pipeline
// Included by engine.cu (one translation unit: the kernels share templates and helpers).
#pragma once

// Fast path for the Generic-Join-shaped aggregating last node: every subatom
// is a cover over the same single new variable x. Per candidate: binding
// lookup, one coalesced cover read, NS-1 bucket probes, fold into count /
// checksum -- no generic state machinery. Used when x is not the last head
// variable (the hash then needs x in the middle of the tuple); the common
// case (triangle C2/C5, 4-clique C4) runs k_last_gj_bf below.
template <int NS, int W>
__global__ void __launch_bounds__(TILE) k_last_gj(const __grid_constant__ KNode N, uint64_t c0, uint64_t c1,
                                                  uint64_t F, const uint64_t* __restrict__ bounds, int xvar,
                                                  int min_var, DevCounters* ctr) {
  uint64_t acc_lo = 0, acc_hi = 0, acc_sum = 0, probes = 0, misses = 0, body = 0;
  long long acc_min = LLONG_MAX;
  const int lane = threadIdx.x & 31;
  const uint64_t* __restrict__ scan = N.scan;
  for (uint64_t base = c0 + (uint64_t)blockIdx.x * TILE; base < c1; base += (uint64_t)gridDim.x * TILE) {
    const uint64_t t = (base - c0) / TILE;
    const uint64_t lo = __ldg(bounds + t), hi = __ldg(bounds + t + 1);
    const uint64_t i = base + threadIdx.x;
    // binding of candidate i (search within the tile's bounds)
    const uint64_t e = i < c1 ? upper_bound_u64(scan, lo, hi, i) : lo;
    const uint64_t j = i - (e ? __ldg(scan + e - 1) : 0ull);
    if (i >= c1) continue;
    const int ci = N.chosen[e];
    uint32_t sp[NS], sl[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const KSub& P = N.sub[s];
      if (P.in_p) {
        sp[s] = __ldg(P.in_p + e);
        sl[s] = __ldg(P.in_len + e);
      } else {
        sp[s] = 0;
        sl[s] = *P.rregion;  // root: its probe region
      }
    }
    uint64_t mult = N.in_mult ? __ldg(N.in_mult + e) : 1ull;
    int32_t hv[W];  // bound head variables, prefetched off the critical path
#pragma unroll
    for (int v = 0; v < W; ++v) hv[v] = (v < N.nhead && v != xvar) ? __ldg(N.in_var[v] + e) : 0;
    uint32_t cpos = 0;
    const int32_t* csrc = nullptr;
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if (s == ci) {
        cpos = sp[s] + (uint32_t)j;
        csrc = N.sub[s].src[0];
      }
    const int32_t x = __ldg(csrc + cpos);
    ++body;
    bool alive = true;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      if (s == ci || !alive) continue;
      const KSub& P = N.sub[s];
      ++probes;
      const uint32_t kw = (uint32_t)x;
      uint64_t b = region_bucket(sp[s], sl[s], kw);
      const uint64_t blo = region_lo(sp[s]), bhi = region_hi(sp[s], sl[s]);
      const uint4* __restrict__ tb = reinterpret_cast<const uint4*>(P.table);
      uint32_t q = kEmpty;
      while (true) {
        const uint4 h0 = __ldg(tb + 2 * b);
        if (h0.y == kEmpty) break;
        if (h0.x == kw) { q = h0.y; break; }
        if (h0.w == kEmpty) break;
        if (h0.z == kw) { q = h0.w; break; }
        const uint4 h1 = __ldg(tb + 2 * b + 1);
        if (h1.y == kEmpty) break;
        if (h1.x == kw) { q = h1.y; break; }
        if (h1.w == kEmpty) break;
        if (h1.z == kw) { q = h1.w; break; }
        if (++b == bhi) b = blo;
      }
      if (q == kEmpty) {
        ++misses;
        alive = false;
      } else if (P.last) {
        mult *= __ldg(P.cnt + q);
      }
    }
    if (!alive) continue;
    uint64_t h = fj::kTupleHashSeed;
#pragma unroll
    for (int v = 0; v < W; ++v)
      if (v < N.nhead) {
        const int32_t val = (v == xvar) ? x : hv[v];
        h = fj::tuple_hash_step(h, (int64_t)val);
        if (v == min_var) acc_min = min(acc_min, (long long)val);
      }
    acc_sum += mult * fj::checksum_word(h);
    acc_lo += mult;
    if (acc_lo < mult) ++acc_hi;
  }
  probes = warp_sum(probes);
  misses = warp_sum(misses);
  body = warp_sum(body);
  uint64_t lo2 = acc_lo, hi2 = acc_hi;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t l2 = __shfl_xor_sync(0xffffffffu, lo2, o);
    const uint64_t h2 = __shfl_xor_sync(0xffffffffu, hi2, o);
    const uint64_t sm = lo2 + l2;
    hi2 += h2 + (sm < lo2 ? 1 : 0);
    lo2 = sm;
  }
  acc_sum = warp_sum(acc_sum);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc_min = min(acc_min, __shfl_xor_sync(0xffffffffu, acc_min, o));
  if (lane == 0) {
    if (probes) {
      atomicAdd((unsigned long long*)&ctr->probes, (unsigned long long)probes);
      atomicAdd((unsigned long long*)&ctr->node_probes[N.k], (unsigned long long)probes);
    }
    if (misses) atomicAdd((unsigned long long*)&ctr->misses, (unsigned long long)misses);
    if (body) atomicAdd((unsigned long long*)&ctr->body[N.k], (unsigned long long)body);
    if (lo2) {
      const unsigned long long old = atomicAdd((unsigned long long*)&ctr->count_lo, (unsigned long long)lo2);
      if (old + lo2 < old) ++hi2;
    }
    if (hi2) atomicAdd((unsigned long long*)&ctr->count_hi, (unsigned long long)hi2);
    if (acc_sum) atomicAdd((unsigned long long*)&ctr->checksum, (unsigned long long)acc_sum);
    if (acc_min != LLONG_MAX) atomicMin(&ctr->minv, acc_min);
  }
}

#ifndef FJG_GJ_BF_MINB
#define FJG_GJ_BF_MINB 4
#endif
#ifndef FJG_STREAM_MINB
#define FJG_STREAM_MINB 4
#endif
#ifndef FJG_STREAM_R
#define FJG_STREAM_R 2
#endif
#ifndef FJG_GJ_TICKET
#define FJG_GJ_TICKET 16  // C2 last node 3.46 -> 3.20 ms, C5 1873 -> 1587 ms (vs static striding)
#endif
#ifndef FJG_GJ_BF_MINB3
#define FJG_GJ_BF_MINB3 4  // 4 resident blocks (64 registers): C4 last node 107.7 -> 98.4 ms
#endif
// One 32-byte bucket (4 slots) in a single 256-bit load (LDG.E.ENL2.256).
struct Bucket8 {
  uint32_t k0, q0, k1, q1, k2, q2, k3, q3;
};
__device__ __forceinline__ Bucket8 ld_bucket(const Slot* table, uint64_t b) {
  Bucket8 r;
  asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.k0), "=r"(r.q0), "=r"(r.k1), "=r"(r.q1), "=r"(r.k2), "=r"(r.q2), "=r"(r.k3), "=r"(r.q3)
               : "l"(table + 4 * b));
  return r;
}
// Branch-free match over a bucket: slots fill in order, so a priority select
// finds the key; `more` = all four slots taken and none matched (the probe
// continues in the next bucket of the region).
__device__ __forceinline__ uint32_t bucket_match(const Bucket8& a, uint32_t kw, bool& more) {
  uint32_t q = (a.q3 != kEmpty && a.k3 == kw) ? a.q3 : kEmpty;
  q = (a.q2 != kEmpty && a.k2 == kw) ? a.q2 : q;
  q = (a.q1 != kEmpty && a.k1 == kw) ? a.q1 : q;
  q = (a.q0 != kEmpty && a.k0 == kw) ? a.q0 : q;
  more = a.q3 != kEmpty && q == kEmpty;
  return q;
}

// Per-warp queue of surviving candidates (binding, cover value, probe
// results): the checksum / multiplicity fold runs on full batches of 32 with
// every lane busy instead of on the ~7% of lanes that hit (C2).
#ifndef FJG_GJ_QC
#define FJG_GJ_QC 128  // survivor ring slots per warp (power of two, > 32 * FJG_GJ_R + 31)
#endif
template <int NS>
struct HitQueue {  // per-warp ring buffers
  static constexpr int NW = TILE / 32, QC = FJG_GJ_QC;
  int32_t x[NW][QC];
  uint32_t e[NW][QC];
  uint32_t q[NS - 1][NW][QC];
  uint8_t c[NW][QC];
  uint32_t tail[NW];
};

// GJ-shaped last node when x is the last head variable (tuple hash =
// step(prefix(binding), x)): each thread owns a run of R consecutive
// candidates (its binding found inside the warp's 64-candidate chunk owner
// range, split at binding boundaries); binding state is loaded once per run,
// cover reads are coalesced, and the R probes are issued back to back. The
// probed subatoms are selected by index (s = j + (j >= chosen)) so one code
// path serves every cover choice; each probe is one 256-bit bucket load and a
// priority select; survivors are folded from a per-warp queue (leaf
// multiplicities, head-prefix hash, checksum, MIN) with every lane busy.
template <int NS, int R, int W>
__global__ void __launch_bounds__(TILE, NS == 2 ? FJG_GJ_BF_MINB : FJG_GJ_BF_MINB3) k_last_gj_bf(const __grid_constant__ KNode N, uint64_t c0,
                                                                     uint64_t c1, uint64_t F,
                                                                     const uint32_t* __restrict__ owner,
                                                                     const uint32_t* __restrict__ perm,
                                                                     int min_var, DevCounters* ctr) {
  // a warp leaves at most 31 unfolded survivors plus 32 per candidate of a run
  static_assert(R >= 1 && (R & (R - 1)) == 0, "k_last_gj_bf: R must be a power of two (chunk_owners)");
  static_assert(32 * R + 31 < HitQueue<NS>::QC, "k_last_gj_bf: survivor ring too small for R");
  __shared__ HitQueue<NS> Q;
  uint64_t acc_lo = 0, acc_hi = 0, acc_sum = 0, probes = 0, misses = 0, body = 0;
  long long acc_min = LLONG_MAX;
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const uint64_t* __restrict__ scan = N.scan;
  const int nhead = N.nhead;
  uint32_t head = 0;  // warp-uniform ring head
  if (lane == 0) Q.tail[wi] = 0;
  __syncwarp();

  auto fold = [&](uint32_t h0, uint32_t n) {  // lanes < n fold ring entries h0 + lane
    if ((uint32_t)lane < n) {
      const uint32_t slot = (h0 + lane) & (HitQueue<NS>::QC - 1);
      const int32_t x = Q.x[wi][slot];
      const uint32_t e = Q.e[wi][slot];
      const int ci = Q.c[wi][slot];
      uint64_t mu = N.in_mult ? __ldg(N.in_mult + e) : 1ull;
#pragma unroll
      for (int j = 0; j < NS - 1; ++j) {
        const uint32_t* cnt = j >= ci ? N.sub[j + 1].cnt : N.sub[j].cnt;
        const bool plast = j >= ci ? N.sub[j + 1].last : N.sub[j].last;
        const uint32_t* ldup = j >= ci ? N.sub[j + 1].ldup : N.sub[j].ldup;
        if (plast && *ldup) mu *= __ldg(cnt + Q.q[j][wi][slot]);  // leaf multiplicity (1 on unit levels)
      }
      uint64_t pre = fj::kTupleHashSeed;
      long long bmin = LLONG_MAX;
#pragma unroll
      for (int v = 0; v < W; ++v)
        if (v < nhead - 1) {
          const int32_t hvv = __ldg(N.in_var[v] + e);
          pre = fj::tuple_hash_step(pre, (int64_t)hvv);
          if (v == min_var) bmin = hvv;
        }
      const uint64_t h = fj::tuple_hash_step(pre, (int64_t)x);
      acc_sum += mu * fj::checksum_word(h);
      acc_lo += mu;
      if (acc_lo < mu) ++acc_hi;
      if (min_var >= 0) acc_min = min(acc_min, min_var == nhead - 1 ? (long long)x : bmin);
    }
  };

  // warps walk the launch's 32*R-candidate chunks: statically strided, or
  // (FJG_GJ_TICKET) by tickets of FJG_GJ_TICKET chunks from a device counter,
  // which keeps every warp near the same front of the candidate range
  const uint64_t nchunks = (c1 - c0 + 32 * R - 1) / (32 * R);
#if FJG_GJ_TICKET
  uint64_t tk = 0, tk_end = 0;
  auto next_chunk = [&]() -> uint64_t {
    if (tk == tk_end) {
      unsigned long long t0 = 0;
      if (lane == 0) t0 = atomicAdd(&ctr->ticket, (unsigned long long)FJG_GJ_TICKET);
      tk = __shfl_sync(0xffffffffu, t0, 0);
      tk_end = tk + FJG_GJ_TICKET;
    }
    return tk++;
  };
  for (uint64_t ch = next_chunk(); ch < nchunks; ch = next_chunk()) {
#else
  for (uint64_t ch = (uint64_t)blockIdx.x * (TILE / 32) + wi; ch < nchunks; ch += (uint64_t)gridDim.x * (TILE / 32)) {
#endif
    uint64_t i = c0 + ch * (32 * R) + (uint64_t)lane * R;
    const uint64_t iend = min(i + R, c1);
    if (i < iend) {
      const uint64_t t = ch;  // this warp's chunk
      uint64_t e = upper_bound_u64(scan, __ldg(owner + t), __ldg(owner + t + 1), i);
      while (i < iend) {
        const uint64_t se = __ldg(scan + e);
        const uint64_t prev = e ? __ldg(scan + e - 1) : 0ull;
        const uint64_t bend = min(iend, se);
        // bindings may be visited in probe-region order: scan is then over the
        // permuted sequence and perm maps a position to the binding
        const uint32_t eb = perm ? __ldg(perm + e) : (uint32_t)e;
        const int ci = N.chosen[eb];
        uint32_t sp[NS], sl[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          const KSub& P = N.sub[s];
          if (P.in_p) {
            sp[s] = __ldg(P.in_p + eb);
            sl[s] = __ldg(P.in_len + eb);
          } else {
            sp[s] = 0;
            sl[s] = *P.rregion;  // root: its probe region
          }
        }
        uint32_t cbase = sp[0];
        const int32_t* csrc = N.sub[0].src[0];
#pragma unroll
        for (int s = 1; s < NS; ++s)
          if (s == ci) {
            cbase = sp[s];
            csrc = N.sub[s].src[0];
          }
        cbase += (uint32_t)(i - prev);
        int32_t x[R];
        bool live[R];
        uint32_t qv[R][NS - 1];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          live[r] = i + r < bend;
          x[r] = live[r] ? __ldg(csrc + cbase + r) : 0;
          body += live[r] ? 1 : 0;
        }
#pragma unroll
        for (int j = 0; j < NS - 1; ++j) {
          // probed subatom s = j + (j >= ci), selected without branching
          const Slot* tb = j >= ci ? N.sub[j + 1].table : N.sub[j].table;
          const uint32_t p = j >= ci ? sp[j + 1] : sp[j];
          const uint32_t len = j >= ci ? sl[j + 1] : sl[j];
          Bucket8 h[R];
          uint64_t b0[R];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            b0[r] = region_bucket(p, len, (uint32_t)x[r]);
            if (live[r]) h[r] = ld_bucket(tb, b0[r]);
          }
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (!live[r]) continue;
            ++probes;
            const uint32_t kw = (uint32_t)x[r];
            bool more;
            uint32_t q = bucket_match(h[r], kw, more);
            if (more) {
              uint64_t b = b0[r];
              const uint64_t blo = region_lo(p), bhi = region_hi(p, len);
              do {
                if (++b == bhi) b = blo;
                q = bucket_match(ld_bucket(tb, b), kw, more);
              } while (more);
            }
            if (q == kEmpty) {
              ++misses;
              live[r] = false;
            }
            qv[r][j] = q;
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (!live[r]) continue;
          const uint32_t slot = atomicAdd(&Q.tail[wi], 1u) & (HitQueue<NS>::QC - 1);
          Q.x[wi][slot] = x[r];
          Q.e[wi][slot] = eb;
          Q.c[wi][slot] = (uint8_t)ci;
#pragma unroll
          for (int j = 0; j < NS - 1; ++j) Q.q[j][wi][slot] = qv[r][j];
        }
        i = bend;
        ++e;
      }
    }
    // warp-convergent: fold full batches of 32 (at most 32*R + 31 < QC pending)
    __syncwarp();
    const uint32_t tail = *(volatile uint32_t*)&Q.tail[wi];
    while (tail - head >= 32) {
      fold(head, 32);
      head += 32;
    }
    __syncwarp();
  }
  __syncwarp();
  fold(head, *(volatile uint32_t*)&Q.tail[wi] - head);
  probes = warp_sum(probes);
  misses = warp_sum(misses);
  body = warp_sum(body);
  uint64_t lo2 = acc_lo, hi2 = acc_hi;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t l2 = __shfl_xor_sync(0xffffffffu, lo2, o);
    const uint64_t h2 = __shfl_xor_sync(0xffffffffu, hi2, o);
    const uint64_t sm = lo2 + l2;
    hi2 += h2 + (sm < lo2 ? 1 : 0);
    lo2 = sm;
  }
  acc_sum = warp_sum(acc_sum);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc_min = min(acc_min, __shfl_xor_sync(0xffffffffu, acc_min, o));
  if (lane == 0) {
    if (probes) {
      atomicAdd((unsigned long long*)&ctr->probes, (unsigned long long)probes);
      atomicAdd((unsigned long long*)&ctr->node_probes[N.k], (unsigned long long)probes);
    }
    if (misses) atomicAdd((unsigned long long*)&ctr->misses, (unsigned long long)misses);
    if (body) atomicAdd((unsigned long long*)&ctr->body[N.k], (unsigned long long)body);
    if (lo2) {
      const unsigned long long old = atomicAdd((unsigned long long*)&ctr->count_lo, (unsigned long long)lo2);
      if (old + lo2 < old) ++hi2;
    }
    if (hi2) atomicAdd((unsigned long long*)&ctr->count_hi, (unsigned long long)hi2);
    if (acc_sum) atomicAdd((unsigned long long*)&ctr->checksum, (unsigned long long)acc_sum);
    if (acc_min != LLONG_MAX) atomicMin(&ctr->minv, acc_min);
  }
}

// Sort key of every binding entering a GJ last node: the start of the subtrie
// region its (first) probed subatom will be probed in. Visiting bindings in
// this order makes consecutive bindings probe the same region, so a region is
// read from HBM about once per batch instead of once per probing binding.
template <int NS>
__global__ void k_probe_keys(const __grid_constant__ KNode N, uint64_t F, uint32_t* __restrict__ keys,
                             uint32_t* __restrict__ vals) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < F; e += (uint64_t)gridDim.x * blockDim.x) {
    const int ci = N.chosen[e];
    const int s = ci == 0 ? 1 : 0;
    const KSub& P = N.sub[s];
    keys[e] = P.in_p ? __ldg(P.in_p + e) : 0u;
    vals[e] = (uint32_t)e;
  }
}

__global__ void k_gather_m(const uint64_t* __restrict__ m, const uint32_t* __restrict__ perm, uint64_t F,
                           uint64_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < F; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = __ldg(m + __ldg(perm + i));
}

#ifndef FJG_GJW_RR
#define FJG_GJW_RR 4  // 64-candidate double steps per warp chunk (chunk = 64 * RR candidates)
#endif
#ifndef FJG_GJW_RR_UNSORTED
#define FJG_GJW_RR_UNSORTED 1  // double steps per chunk when the bindings are not ordered by probe region (C2)
#endif
#ifndef FJG_GJW_MINB3
#define FJG_GJW_MINB3 5
#endif
#ifndef FJG_GJ_TICKET3
#define FJG_GJ_TICKET3 FJG_GJ_TICKET
#endif
#ifndef FJG_GJW_RR3
#define FJG_GJW_RR3 1  // three-subatom nodes (C4): one double step per chunk (last node 71.6 -> 70.2 ms; 2: 70.9, 4: 71.6, 8: 74.5)
#endif
#ifndef FJG_GJW_MINB
#define FJG_GJW_MINB 5  // 48 registers: C5 last node 1017 -> 973 ms vs 6 blocks (40 registers + spills)
#endif
#ifndef FJG_GJW
#define FJG_GJW 1  // k_last_gj_warp instead of k_last_gj_bf for the GJ last node
#endif

// Binding state of a GJ last node (one frontier entry), loaded once per
// binding by the whole warp (uniform addresses, broadcast loads).
template <int NS>
struct GjBind {
  // candidate range [prev, end) of the binding, relative to the launch's c0 in
  // 32 bits (a launch spans <= 2^31 candidates): end clamped to the launch end,
  // prev wraps below 0 for a binding that began in an earlier launch (cover
  // offsets i - prev are computed mod 2^32 and stay exact)
  uint32_t prev, end;
  uint32_t eb;          // binding index (after the probe-region permutation)
  int ci;               // chosen cover
  uint32_t cb;          // cover subtrie start
  uint32_t p[NS - 1], len[NS - 1];  // probed subtrie regions, probe order
};

template <int NS>
__device__ __forceinline__ void gj_load_bind(const KNode& N, const uint64_t* __restrict__ scan,
                                             const uint32_t* __restrict__ perm, uint32_t e, uint64_t c0,
                                             uint32_t lmax, GjBind<NS>& B) {
  const uint64_t end = __ldg(scan + e);
  B.end = (uint32_t)min(end - c0, (uint64_t)lmax);
  B.prev = (uint32_t)((e ? __ldg(scan + e - 1) : 0ull) - c0);
  B.eb = perm ? __ldg(perm + e) : (uint32_t)e;
  B.ci = N.chosen[B.eb];
  uint32_t sp[NS], sl[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const KSub& P = N.sub[s];
    if (P.in_p) {
      sp[s] = __ldg(P.in_p + B.eb);
      sl[s] = __ldg(P.in_len + B.eb);
    } else {
      sp[s] = 0;
      sl[s] = *P.rregion;
    }
  }
  B.cb = sp[0];
#pragma unroll
  for (int s = 1; s < NS; ++s)
    if (s == B.ci) B.cb = sp[s];
  FJG_ASSERT(end >= c0 && B.ci >= 0 && B.ci < NS);
#pragma unroll
  for (int s = 0; s < NS; ++s)
    FJG_ASSERT(sp[s] == kSingleton || (uint64_t)sp[s] + sl[s] <= (uint64_t)N.sub[s].root_n + (N.sub[s].in_p ? 0 : 1));
#pragma unroll
  for (int j = 0; j < NS - 1; ++j) {
    B.p[j] = j >= B.ci ? sp[j + 1] : sp[j];
    B.len[j] = j >= B.ci ? sl[j + 1] : sl[j];
  }
}

// Three-subatom GJ nodes: candidates alive after the first probe wait in a
// per-warp ring and the second probe runs on full batches of 32 (C4: 27% of
// the candidates survive the first probe, so probing the second subatom in
// place ran every step at a quarter of its lanes).
template <int NS>
struct GjStage1 {
  static constexpr int NW = TILE / 32, QC = NS == 3 ? FJG_GJ_QC : 1;
  int32_t x[NW][QC];
  uint32_t e[NW][QC], q0[NW][QC], p1[NW][QC], len1[NW][QC];
  uint8_t c[NW][QC];
};

// GJ-shaped last node, warp-uniform bindings: a warp walks chunks of 64 * RR
// consecutive candidates (tickets from a device counter, as k_last_gj_bf) in
// double steps of 64 (lane l takes candidates base + l and base + 32 + l, so
// cover reads are two coalesced loads and two 256-bit bucket loads are in
// flight per lane). A double step inside one binding -- the common case, a
// binding has 300 candidates on C5 -- uses the warp's binding state held in
// registers and costs no per-lane bookkeeping; a step crossing binding ends
// walks each lane to its own binding. Survivors are folded from the per-warp
// ring exactly as in k_last_gj_bf.
template <int NS, int W, int RR, bool ENUMR = false>
__global__ void __launch_bounds__(TILE, NS == 3 ? FJG_GJW_MINB3 : FJG_GJW_MINB) k_last_gj_warp(const __grid_constant__ KNode N, uint64_t c0,
                                                                    uint64_t c1, uint64_t F,
                                                                    const uint32_t* __restrict__ owner,
                                                                    const uint32_t* __restrict__ perm, int min_var,
                                                                    DevCounters* ctr, int32_t* __restrict__ out_tuples = nullptr,
                                                                    uint64_t out_cap = 0) {
  static_assert(64 + 63 < HitQueue<NS>::QC, "k_last_gj_warp: survivor ring too small");
  __shared__ HitQueue<NS> Q;
  __shared__ GjStage1<NS> S1;
  uint32_t h1 = 0, t1 = 0;  // stage-1 ring cursors (NS == 3), warp-uniform
  uint64_t acc_lo = 0, acc_hi = 0, acc_sum = 0, probes = 0, misses = 0, body = 0;
  long long acc_min = LLONG_MAX;
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const uint64_t* __restrict__ scan = N.scan;
  const int nhead = N.nhead;
  // ring cursors, warp-uniform registers: entries [head, tail) are pending
  uint32_t head = 0, tail = 0;
  const unsigned lt_mask = (1u << lane) - 1u;
  // warp-aggregated enqueue (every lane calls it): one ballot, no atomics
  auto enqueue = [&](bool hit, int32_t x, uint32_t eb, int ci, const uint32_t (&qv)[NS - 1]) {
    const unsigned hm = __ballot_sync(0xffffffffu, hit);
    if (hit) {
      const uint32_t slot = (tail + __popc(hm & lt_mask)) & (HitQueue<NS>::QC - 1);
      Q.x[wi][slot] = x;
      Q.e[wi][slot] = eb;
      Q.c[wi][slot] = (uint8_t)ci;
#pragma unroll
      for (int j = 0; j < NS - 1; ++j) Q.q[j][wi][slot] = qv[j];
    }
    tail += __popc(hm);
  };

  auto fold = [&](uint32_t h0, uint32_t n) {
    int32_t row[W];  // enumerate mode: the output tuple (bound head variables, then x)
    uint64_t rmu = 0;
    if ((uint32_t)lane < n) {
      const uint32_t slot = (h0 + lane) & (HitQueue<NS>::QC - 1);
      const int32_t x = Q.x[wi][slot];
      const uint32_t e = Q.e[wi][slot];
      const int ci = Q.c[wi][slot];
      uint64_t mu = N.in_mult ? __ldg(N.in_mult + e) : 1ull;
#pragma unroll
      for (int j = 0; j < NS - 1; ++j) {
        const uint32_t* cnt = j >= ci ? N.sub[j + 1].cnt : N.sub[j].cnt;
        const bool plast = j >= ci ? N.sub[j + 1].last : N.sub[j].last;
        const uint32_t* ldup = j >= ci ? N.sub[j + 1].ldup : N.sub[j].ldup;
        if (plast && *ldup) mu *= __ldg(cnt + Q.q[j][wi][slot]);
      }
      uint64_t pre = fj::kTupleHashSeed;
      long long bmin = LLONG_MAX;
#pragma unroll
      for (int v = 0; v < W; ++v)
        if (v < nhead - 1) {
          const int32_t hvv = __ldg(N.in_var[v] + e);
          pre = fj::tuple_hash_step(pre, (int64_t)hvv);
          if (v == min_var) bmin = hvv;
          if (ENUMR) row[v] = hvv;
        }
      const uint64_t h = fj::tuple_hash_step(pre, (int64_t)x);
      acc_sum += mu * fj::checksum_word(h);
      acc_lo += mu;
      if (acc_lo < mu) ++acc_hi;
      if (min_var >= 0) acc_min = min(acc_min, min_var == nhead - 1 ? (long long)x : bmin);
      if (ENUMR) {
#pragma unroll
        for (int v = 0; v < W; ++v)
          if (v == nhead - 1) row[v] = x;
        rmu = mu;
      }
    }
    if (ENUMR) {  // the batch's rows: one global atomic per warp, lane offsets by scan
      uint64_t off = rmu;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint64_t o = __shfl_up_sync(0xffffffffu, off, d);
        if (lane >= d) off += o;
      }
      const uint64_t total = __shfl_sync(0xffffffffu, off, 31);
      unsigned long long base = 0;
      if (lane == 0 && total) base = atomicAdd((unsigned long long*)&ctr->out_rows, (unsigned long long)total);
      base = __shfl_sync(0xffffffffu, base, 0) + off - rmu;
      for (uint64_t r = 0; r < rmu && base + r < out_cap; ++r)
#pragma unroll
        for (int v = 0; v < W; ++v)
          if (v < nhead) out_tuples[(base + r) * nhead + v] = row[v];
    }
  };
  // probe candidate x of a binding in its probed regions; survivors enqueue
  // second probe of 32 (or the last n) stage-1 entries, one per lane
  auto stage2 = [&](uint32_t n) {
    if (NS != 3) return;
    const bool live = (uint32_t)lane < n;
    const uint32_t slot = (h1 + lane) & (GjStage1<NS>::QC - 1);
    int32_t x = 0;
    uint32_t eb = 0, q0 = 0, q1 = kEmpty;
    int ci = 0;
    if (live) {
      x = S1.x[wi][slot];
      eb = S1.e[wi][slot];
      q0 = S1.q0[wi][slot];
      ci = S1.c[wi][slot];
      const uint32_t p1 = S1.p1[wi][slot], len1 = S1.len1[wi][slot];
      const Slot* tb = 1 >= ci ? N.sub[NS - 1].table : N.sub[1].table;
      ++probes;
      const uint32_t kw = (uint32_t)x;
      uint64_t b = region_bucket(p1, len1, kw);
      bool more;
      q1 = bucket_match(ld_bucket(tb, b), kw, more);
      while (more) {
        if (++b == region_hi(p1, len1)) b = region_lo(p1);
        q1 = bucket_match(ld_bucket(tb, b), kw, more);
      }
      if (q1 == kEmpty) ++misses;
    }
    h1 += n;
    uint32_t qv[NS - 1];
    qv[0] = q0;
    if (NS == 3) qv[NS - 2] = q1;
    enqueue(live && q1 != kEmpty, x, eb, ci, qv);
  };
  auto probe_one = [&](bool live, int32_t x, const GjBind<NS>& B) {
    if (NS == 3) {  // first probe here, survivors queue for stage2
      uint32_t q = kEmpty;
      if (live) {
        const Slot* tb = 0 >= B.ci ? N.sub[1].table : N.sub[0].table;
        ++probes;
        const uint32_t kw = (uint32_t)x;
        uint64_t b = region_bucket(B.p[0], B.len[0], kw);
        bool more;
        q = bucket_match(ld_bucket(tb, b), kw, more);
        while (more) {
          if (++b == region_hi(B.p[0], B.len[0])) b = region_lo(B.p[0]);
          q = bucket_match(ld_bucket(tb, b), kw, more);
        }
        if (q == kEmpty) ++misses;
      }
      const bool hit = live && q != kEmpty;
      const unsigned hm = __ballot_sync(0xffffffffu, hit);
      if (hit) {
        const uint32_t slot = (t1 + __popc(hm & lt_mask)) & (GjStage1<NS>::QC - 1);
        S1.x[wi][slot] = x;
        S1.e[wi][slot] = B.eb;
        S1.q0[wi][slot] = q;
        S1.c[wi][slot] = (uint8_t)B.ci;
        S1.p1[wi][slot] = B.p[NS - 2];
        S1.len1[wi][slot] = B.len[NS - 2];
      }
      t1 += __popc(hm);
      return;
    }
    uint32_t qv[NS - 1];
#pragma unroll
    for (int j = 0; j < NS - 1; ++j) {
      qv[j] = kEmpty;
      if (!live) continue;
      const Slot* tb = j >= B.ci ? N.sub[j + 1].table : N.sub[j].table;
      ++probes;
      const uint32_t kw = (uint32_t)x;
      uint64_t b = region_bucket(B.p[j], B.len[j], kw);
      bool more;
      uint32_t q = bucket_match(ld_bucket(tb, b), kw, more);
      while (more) {
        if (++b == region_hi(B.p[j], B.len[j])) b = region_lo(B.p[j]);
        q = bucket_match(ld_bucket(tb, b), kw, more);
      }
      if (q == kEmpty) {
        ++misses;
        live = false;
      }
      qv[j] = q;
    }
    enqueue(live, x, B.eb, B.ci, qv);
  };

  constexpr uint32_t CH = 64 * RR;
  const uint32_t lmax = (uint32_t)(c1 - c0);  // candidates of this launch (<= 2^31)
  const uint32_t nchunks = (lmax + CH - 1) / CH;
  uint64_t tk = 0, tk_end = 0;
  auto next_chunk = [&]() -> uint64_t {
    if (tk == tk_end) {
      unsigned long long t0 = 0;
      if (lane == 0) t0 = atomicAdd(&ctr->ticket, (unsigned long long)(NS == 3 ? FJG_GJ_TICKET3 : FJG_GJ_TICKET));
      tk = __shfl_sync(0xffffffffu, t0, 0);
      tk_end = tk + (NS == 3 ? FJG_GJ_TICKET3 : FJG_GJ_TICKET);
    }
    return tk++;
  };
  for (uint64_t ch = next_chunk(); ch < nchunks; ch = next_chunk()) {
    // candidate positions below are local to the launch: c0 + local
    const uint32_t s0 = (uint32_t)ch * CH, s1 = min(s0 + CH, lmax);
    uint32_t e = __ldg(owner + ch);
    GjBind<NS> B;
    gj_load_bind<NS>(N, scan, perm, e, c0, lmax, B);
#pragma unroll 1
    for (int rr = 0; rr < RR; ++rr) {
      const uint32_t base = s0 + 64u * rr;
      if (base >= s1) break;
      while (B.end <= base) gj_load_bind<NS>(N, scan, perm, ++e, c0, lmax, B);  // warp-uniform
      if (base + 64 <= min(B.end, s1)) {
        const int32_t* __restrict__ cs = (B.ci == 0 ? N.sub[0].src[0] : (B.ci == 1 ? N.sub[1].src[0]
                                                                                   : N.sub[NS - 1].src[0])) +
                                         B.cb + (base - B.prev);
        const int32_t xa = __ldg(cs + lane), xb = __ldg(cs + 32 + lane);
        body += 2;
        if (NS == 2) {  // both buckets in flight before either is matched
          const Slot* tb = B.ci == 0 ? N.sub[1].table : N.sub[0].table;
          uint64_t ba = region_bucket(B.p[0], B.len[0], (uint32_t)xa);
          uint64_t bb = region_bucket(B.p[0], B.len[0], (uint32_t)xb);
          const Bucket8 ha = ld_bucket(tb, ba), hb = ld_bucket(tb, bb);
          probes += 2;
          bool ma, mb;
          uint32_t qa = bucket_match(ha, (uint32_t)xa, ma), qb = bucket_match(hb, (uint32_t)xb, mb);
          const uint64_t bhi = region_hi(B.p[0], B.len[0]);
          while (ma) {
            if (++ba == bhi) ba = region_lo(B.p[0]);
            qa = bucket_match(ld_bucket(tb, ba), (uint32_t)xa, ma);
          }
          while (mb) {
            if (++bb == bhi) bb = region_lo(B.p[0]);
            qb = bucket_match(ld_bucket(tb, bb), (uint32_t)xb, mb);
          }
          misses += (qa == kEmpty) + (qb == kEmpty);
          const uint32_t qva[NS - 1] = {qa}, qvb[NS - 1] = {qb};
          enqueue(qa != kEmpty, xa, B.eb, B.ci, qva);
          enqueue(qb != kEmpty, xb, B.eb, B.ci, qvb);
        } else {
          probe_one(true, xa, B);
          probe_one(true, xb, B);
        }
      } else {
        // the double step crosses binding ends (or the chunk end). Lane j holds
        // the end of binding e + j; when the window's bindings are among those
        // 32 and none is empty, each lane finds its two candidates' bindings by
        // popcounts over the window's end positions and fetches their state
        // with shuffles from the lane that loaded it.
        const unsigned FULL = 0xffffffffu;
        const uint64_t wend = c0 + min(base + 64, s1);  // absolute, as scan
        const uint32_t ej = e + lane;
        const uint64_t endj = ej < F ? __ldg(scan + ej) : ~0ull;
        const uint64_t rel = endj - (c0 + base);  // >= 1: binding e ends after base
        const bool inwin = endj < wend;
        const unsigned lo_bits = __reduce_or_sync(FULL, inwin && rel < 32 ? 1u << rel : 0u);
        const unsigned hi_bits = __reduce_or_sync(FULL, inwin && rel >= 32 ? 1u << (rel - 32) : 0u);
        const int nin = __popc(__ballot_sync(FULL, inwin));
        const bool fits = __shfl_sync(FULL, endj, 31) >= wend && __popc(lo_bits) + __popc(hi_bits) == nin;
        if (fits) {
          // lanes 0..nin load the state of bindings e..e+nin
          GjBind<NS> S = B;
          if (lane > 0 && lane <= nin) gj_load_bind<NS>(N, scan, perm, ej, c0, lmax, S);
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const uint32_t pos = 32 * t + lane;  // candidate base + pos
            const uint32_t i = base + pos;
            const bool live = i < s1;
            const unsigned below = pos >= 31 ? 0xffffffffu : ((2u << pos) - 1u);
            const int seg = t == 0 ? __popc(lo_bits & below)
                                   : __popc(lo_bits) + __popc(hi_bits & (lane >= 31 ? 0xffffffffu : ((2u << lane) - 1u)));
            GjBind<NS> L;
            L.prev = __shfl_sync(FULL, S.prev, seg);
            L.eb = __shfl_sync(FULL, S.eb, seg);
            L.ci = __shfl_sync(FULL, S.ci, seg);
            L.cb = __shfl_sync(FULL, S.cb, seg);
#pragma unroll
            for (int j = 0; j < NS - 1; ++j) {
              L.p[j] = __shfl_sync(FULL, S.p[j], seg);
              L.len[j] = __shfl_sync(FULL, S.len[j], seg);
            }
            const int32_t* cs =
                L.ci == 0 ? N.sub[0].src[0] : (L.ci == 1 ? N.sub[1].src[0] : N.sub[NS - 1].src[0]);
            const int32_t x = live ? __ldg(cs + L.cb + (i - L.prev)) : 0;
            body += live ? 1 : 0;
            probe_one(live, x, L);
          }
        } else {
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const uint32_t i = base + 32 * t + lane;
            const bool live = i < s1;
            GjBind<NS> L = B;
            if (live && i >= L.end) {
              uint32_t el = e + 1;
              while (__ldg(scan + el) <= c0 + i) ++el;
              gj_load_bind<NS>(N, scan, perm, el, c0, lmax, L);
            }
            const int32_t* cs =
                L.ci == 0 ? N.sub[0].src[0] : (L.ci == 1 ? N.sub[1].src[0] : N.sub[NS - 1].src[0]);
            const int32_t x = live ? __ldg(cs + L.cb + (i - L.prev)) : 0;
            body += live ? 1 : 0;
            probe_one(live, x, L);
          }
        }
      }
      if (NS == 3) {  // second probes on full batches (at most 64 + 31 stage-1 entries pending)
        while (t1 - h1 >= 32) {
          __syncwarp();  // the stage-1 entries other lanes wrote
          stage2(32);
          if (tail - head >= 32) {
            __syncwarp();
            do {
              fold(head, 32);
              head += 32;
            } while (tail - head >= 32);
          }
        }
        __syncwarp();
      }
      // warp-convergent: fold full batches of 32 (at most 64 + 31 pending)
      if (tail - head >= 32) {
        __syncwarp();  // the ring entries other lanes wrote
        do {
          fold(head, 32);
          head += 32;
        } while (tail - head >= 32);
        __syncwarp();
      }
    }
  }
  __syncwarp();
  if (NS == 3) {
    while (t1 != h1) {
      stage2(min(32u, t1 - h1));
      __syncwarp();
      if (tail - head >= 32) {
        fold(head, 32);
        head += 32;
        __syncwarp();
      }
    }
  }
  fold(head, tail - head);
  probes = warp_sum(probes);
  misses = warp_sum(misses);
  body = warp_sum(body);
  uint64_t lo2 = acc_lo, hi2 = acc_hi;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t l2 = __shfl_xor_sync(0xffffffffu, lo2, o);
    const uint64_t h2 = __shfl_xor_sync(0xffffffffu, hi2, o);
    const uint64_t sm = lo2 + l2;
    hi2 += h2 + (sm < lo2 ? 1 : 0);
    lo2 = sm;
  }
  acc_sum = warp_sum(acc_sum);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc_min = min(acc_min, __shfl_xor_sync(0xffffffffu, acc_min, o));
  if (lane == 0) {
    if (probes) {
      atomicAdd((unsigned long long*)&ctr->probes, (unsigned long long)probes);
      atomicAdd((unsigned long long*)&ctr->node_probes[N.k], (unsigned long long)probes);
    }
    if (misses) atomicAdd((unsigned long long*)&ctr->misses, (unsigned long long)misses);
    if (body) atomicAdd((unsigned long long*)&ctr->body[N.k], (unsigned long long)body);
    if (lo2) {
      const unsigned long long old = atomicAdd((unsigned long long*)&ctr->count_lo, (unsigned long long)lo2);
      if (old + lo2 < old) ++hi2;
    }
    if (hi2) atomicAdd((unsigned long long*)&ctr->count_hi, (unsigned long long)hi2);
    if (acc_sum) atomicAdd((unsigned long long*)&ctr->checksum, (unsigned long long)acc_sum);
    if (acc_min != LLONG_MAX) atomicMin(&ctr->minv, acc_min);
  }
}

#ifndef FJG_GJ_R
#define FJG_GJ_R 2
#endif
#ifndef FJG_GJ_WRITE
#define FJG_GJ_WRITE 1
#endif
#ifndef FJG_STREAM_WRITE
#define FJG_STREAM_WRITE 1
#endif

// GJ-shaped frontier-writing node: every subatom is a one-variable cover of the
// new variable x; atoms whose subatom is not their last continue with the
// child of their cover (keys mode) or probe (q, cnt[q]). Each thread takes
// RW candidates per tile (rounds of 32-candidate warp chunks), and the
// survivors of all rounds are block-compacted at once (one barrier pair and
// one global atomic per RW*TILE candidates).
#ifndef FJG_WRITE_RW
#define FJG_WRITE_RW 4
#endif
#ifndef FJG_WRITE_TICKET
#define FJG_WRITE_TICKET 1  // C4 frontier node -2 ms
#endif
template <int NS, bool ONE>
__device__ __forceinline__ bool gj_write_cand(const KNode& N, uint64_t c0, uint64_t i,
                                              const uint32_t* __restrict__ owner, uint32_t& e_out, int32_t& x,
                                              uint64_t& mult, uint32_t (&chp)[NS], uint32_t (&chl)[NS],
                                              uint32_t& probes, uint32_t& misses, uint32_t& body) {
  const uint64_t* __restrict__ scan = N.scan;
  uint64_t e = 0, j = i;  // ONE: a single binding (node 0), candidate = offset
  if (!ONE) {
    const uint64_t t = (i - c0) / 32;  // this warp's 32-candidate chunk
    e = upper_bound_u64(scan, __ldg(owner + t), __ldg(owner + t + 1), i);
    j = i - (e ? __ldg(scan + e - 1) : 0ull);
  }
  e_out = (uint32_t)e;
  if (ONE) {  // keys iteration over a forced map: most offsets are not child starts
    const int ci = N.chosen[0];
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if (s == ci && !N.sub[s].stream && __ldg(N.sub[s].cnt + (N.sub[s].in_p ? __ldg(N.sub[s].in_p) : 0u) + (uint32_t)j) == 0)
        return false;
  }
  const int ci = N.chosen[e];
  uint32_t sp[NS], sl[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const KSub& P = N.sub[s];
    if (P.in_p) {
      sp[s] = __ldg(P.in_p + e);
      sl[s] = __ldg(P.in_len + e);
    } else {
      sp[s] = 0;
      sl[s] = *P.rregion;  // root: its probe region
    }
  }
  mult = N.in_mult ? __ldg(N.in_mult + e) : 1ull;
  bool alive = true;
#pragma unroll
  for (int s = 0; s < NS; ++s)
    if (s == ci) {
      const KSub& S = N.sub[s];
      const uint32_t pos = sp[s] + (uint32_t)j;
      if (!S.stream) {  // forced map: distinct keys are the child starts
        const uint32_t c = __ldg(S.cnt + pos);
        if (c == 0) alive = false;
        chp[s] = pos;
        chl[s] = c;
      } else {
        chp[s] = kSingleton;
        chl[s] = 1;
      }
      x = alive ? __ldg(S.src[0] + pos) : 0;
    }
  if (!alive) return false;
  ++body;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    if (s == ci) continue;
    const KSub& P = N.sub[s];
    ++probes;
    const uint32_t kw = (uint32_t)x;
    uint64_t b = region_bucket(sp[s], sl[s], kw);
    const uint64_t blo = region_lo(sp[s]), bhi = region_hi(sp[s], sl[s]);
    bool more;
    uint32_t q = bucket_match(ld_bucket(P.table, b), kw, more);
    while (more) {
      if (++b == bhi) b = blo;
      q = bucket_match(ld_bucket(P.table, b), kw, more);
    }
    if (q == kEmpty) {
      ++misses;
      return false;
    }
    const uint32_t ql = __ldg(P.cnt + q);
    if (P.last)
      mult *= ql;
    else {
      chp[s] = q;
      chl[s] = ql;
    }
  }
  return true;
}

template <int NS, int W, bool ONE>
__device__ __forceinline__ void write_gj_body(const KNode& N, uint64_t c0, uint64_t c1,
                                              const uint32_t* __restrict__ owner, int xvar, DevCounters* ctr);

template <int NS, int W>
__global__ void __launch_bounds__(TILE) k_write_gj(const __grid_constant__ KNode N, uint64_t c0, uint64_t c1,
                                                   uint64_t F, const uint32_t* __restrict__ owner, int xvar,
                                                   DevCounters* ctr) {
  if (F == 1)
    write_gj_body<NS, W, true>(N, c0, c1, owner, xvar, ctr);
  else
    write_gj_body<NS, W, false>(N, c0, c1, owner, xvar, ctr);
}

template <int NS, int W, bool ONE>
__device__ __forceinline__ void write_gj_body(const KNode& N, uint64_t c0, uint64_t c1,
                                              const uint32_t* __restrict__ owner, int xvar, DevCounters* ctr) {
  constexpr int RW = FJG_WRITE_RW;
  __shared__ uint32_t s_warp[TILE / 32];
  __shared__ uint32_t s_base;
  uint32_t probes = 0, misses = 0, body = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
#if FJG_WRITE_TICKET
  // blocks take their next tile from a device counter (one front, see k_last_gj_bf)
  __shared__ uint64_t s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(&ctr->ticket, 1ull);
  __syncthreads();
  for (uint64_t base = c0 + s_tile * TILE * RW; base < c1;) {
#else
  for (uint64_t base = c0 + (uint64_t)blockIdx.x * TILE * RW; base < c1; base += (uint64_t)gridDim.x * TILE * RW) {
#endif
    bool alive[RW];
    uint32_t e[RW];
    int32_t x[RW];
    uint64_t mult[RW];
    uint32_t chp[RW][NS], chl[RW][NS];
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      // round r: warp w takes the 32-candidate chunk base + (r * TILE/32 + w) * 32
      const uint64_t i = base + (uint64_t)r * TILE + threadIdx.x;
#pragma unroll
      for (int s = 0; s < NS; ++s) chp[r][s] = chl[r][s] = 0;
      e[r] = 0;
      x[r] = 0;
      mult[r] = 1;
      alive[r] = i < c1 && gj_write_cand<NS, ONE>(N, c0, i, owner, e[r], x[r], mult[r], chp[r], chl[r], probes, misses,
                                             body);
    }
    unsigned bal[RW];
    uint32_t wtot = 0;
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      bal[r] = __ballot_sync(0xffffffffu, alive[r]);
      wtot += __popc(bal[r]);
    }
    if (lane == 0) s_warp[warp] = wtot;
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
    uint32_t o = s_base + s_warp[warp];
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      if (alive[r]) {
        const uint32_t at = o + __popc(bal[r] & lt_mask);
#pragma unroll
        for (int v = 0; v < W; ++v)
          if ((N.out_vars >> v) & 1u) N.out_var[v][at] = (v == xvar) ? x[r] : __ldg(N.in_var[v] + e[r]);
#pragma unroll
        for (int a = 0; a < W; ++a)
          if ((N.out_atoms >> a) & 1u) {
            uint32_t pa = 0, la = 0;
            bool here = false;
#pragma unroll
            for (int s = 0; s < NS; ++s)
              if (N.sub[s].atom == a) {
                pa = chp[r][s];
                la = chl[r][s];
                here = true;
              }
            if (!here) {
              pa = __ldg(N.in_p[a] + e[r]);
              la = __ldg(N.in_len[a] + e[r]);
            }
            N.out_p[a][at] = pa;
            N.out_len[a][at] = la;
          }
        if (N.out_mult) N.out_mult[at] = mult[r];
      }
      o += __popc(bal[r]);
    }
#if FJG_WRITE_TICKET
    if (threadIdx.x == 0) s_tile = atomicAdd(&ctr->ticket, 1ull);
    __syncthreads();
    base = c0 + s_tile * TILE * RW;
#else
    __syncthreads();
#endif
  }
  const uint64_t tp = warp_sum((uint64_t)probes), tm = warp_sum((uint64_t)misses), tb = warp_sum((uint64_t)body);
  if (lane == 0) {
    if (tp) {
      atomicAdd((unsigned long long*)&ctr->probes, (unsigned long long)tp);
      atomicAdd((unsigned long long*)&ctr->node_probes[N.k], (unsigned long long)tp);
    }
    if (tm) atomicAdd((unsigned long long*)&ctr->misses, (unsigned long long)tm);
    if (tb) atomicAdd((unsigned long long*)&ctr->body[N.k], (unsigned long long)tb);
  }
}

// Binary-join-pipeline node (frontier-writing): one cover iterated in stream
// mode, every other subatom a single-variable probe keyed on a variable the
// cover binds (C1 chain, C3 star node 0). Cover columns are loaded lazily, in
// probe order, so a candidate that dies at its first probe reads one column.
template <int W>
__global__ void __launch_bounds__(TILE) k_write_stream(const __grid_constant__ KNode N, uint64_t c0, uint64_t c1,
                                                       uint64_t F, const uint64_t* __restrict__ bounds,
                                                       DevCounters* ctr) {
  __shared__ uint32_t s_warp[TILE / 32];
  __shared__ uint32_t s_base;
  uint64_t probes = 0, misses = 0, body = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t* __restrict__ scan = N.scan;
  const int ci = N.cov[0];
  const KSub& S = N.sub[ci];
  for (uint64_t base = c0 + (uint64_t)blockIdx.x * TILE; base < c1; base += (uint64_t)gridDim.x * TILE) {
    const uint64_t t = (base - c0) / TILE;
    const uint64_t lo = __ldg(bounds + t), hi = __ldg(bounds + t + 1);
    const uint64_t i = base + threadIdx.x;
    bool alive = i < c1;
    uint64_t e = 0, mult = 1;
    uint32_t pos = 0;
    int32_t xv[MAXK];
    uint32_t have = 0;  // bit t: cover column t loaded
    uint32_t chp[MAXS], chl[MAXS];
#pragma unroll
    for (int k = 0; k < MAXK; ++k) xv[k] = 0;
#pragma unroll
    for (int s = 0; s < MAXS; ++s) chp[s] = chl[s] = 0;
    if (alive) {
      e = upper_bound_u64(scan, lo, hi, i);
      const uint64_t j = i - (e ? __ldg(scan + e - 1) : 0ull);
      uint32_t p;
      if (S.in_p) {
        p = __ldg(S.in_p + e);
      } else {
        p = 0;
      }
      pos = p + (uint32_t)j;
      if (N.in_mult) mult = __ldg(N.in_mult + e);
      ++body;
#pragma unroll
      for (int s = 0; s < MAXS; ++s) {
        if (s >= N.nsub || s == ci || !alive) continue;
        const KSub& P = N.sub[s];
        // key: the cover column bound to P's variable (loaded on first use)
        int tk = 0;
#pragma unroll
        for (int k = 0; k < MAXK; ++k)
          if (k < S.nv && S.var[k] == P.var[0]) tk = k;
        int32_t key = 0;
#pragma unroll
        for (int k = 0; k < MAXK; ++k)
          if (k == tk) {
            if (!((have >> k) & 1u)) {
              xv[k] = __ldg(S.src[k] + pos);
              have |= 1u << k;
            }
            key = xv[k];
          }
        uint32_t pp, pl;
        if (P.in_p) {
          pp = __ldg(P.in_p + e);
          pl = __ldg(P.in_len + e);
        } else {
          pp = 0;
          pl = *P.rregion;  // root: its probe region
        }
        ++probes;
        const uint32_t kw = (uint32_t)key;
        uint64_t b = region_bucket(pp, pl, kw);
        const uint64_t blo = region_lo(pp), bhi = region_hi(pp, pl);
        const uint4* __restrict__ tb = reinterpret_cast<const uint4*>(P.table);
        uint32_t q = kEmpty;
        while (true) {
          const uint4 h0 = __ldg(tb + 2 * b);
          if (h0.y == kEmpty) break;
          if (h0.x == kw) { q = h0.y; break; }
          if (h0.w == kEmpty) break;
          if (h0.z == kw) { q = h0.w; break; }
          const uint4 h1 = __ldg(tb + 2 * b + 1);
          if (h1.y == kEmpty) break;
          if (h1.x == kw) { q = h1.y; break; }
          if (h1.w == kEmpty) break;
          if (h1.z == kw) { q = h1.w; break; }
          if (++b == bhi) b = blo;
        }
        if (q == kEmpty) {
          ++misses;
          alive = false;
        } else {
          const uint32_t ql = __ldg(P.cnt + q);
          if (P.last)
            mult *= ql;
          else {
            chp[s] = q;
            chl[s] = ql;
          }
        }
      }
    }
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
        if ((N.out_vars >> v) & 1u) {
          int32_t val = 0;
          bool cov = false;
#pragma unroll
          for (int k = 0; k < MAXK; ++k)
            if (k < S.nv && S.var[k] == v) {
              val = ((have >> k) & 1u) ? xv[k] : __ldg(S.src[k] + pos);
              cov = true;
            }
          N.out_var[v][o] = cov ? val : __ldg(N.in_var[v] + e);
        }
#pragma unroll
      for (int a = 0; a < W; ++a)
        if ((N.out_atoms >> a) & 1u) {
          uint32_t pa = 0, la = 0;
          bool here = false;
#pragma unroll
          for (int s = 0; s < MAXS; ++s)
            if (s < N.nsub && N.sub[s].atom == a) {
              pa = s == ci ? kSingleton : chp[s];
              la = s == ci ? 1u : chl[s];
              here = true;
            }
          if (!here) {
            pa = __ldg(N.in_p[a] + e);
            la = __ldg(N.in_len[a] + e);
          }
          N.out_p[a][o] = pa;
          N.out_len[a][o] = la;
        }
      if (N.out_mult) N.out_mult[o] = mult;
    }
    __syncthreads();
  }
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
}

// Single-binding stream node (F == 1: node 0 of a plan whose first node
// iterates a base table, C1 chain / C3 star): no binding search at all, the
// candidate index is the row. Each warp owns 32*R consecutive rows, lane l the
// rows base + r*32 + l (every column load is coalesced); the probes are issued
// subatom by subatom with the R bucket loads of a lane back to back, and a
// warp stops as soon as none of its rows is alive (most star rows die at the
// first dimension). The probe key columns are resolved on the host (SProbe),
// child lengths are read only for survivors, and survivors take one
// warp-aggregated atomic -- no block barriers.
struct SProbe {
  int np;          // probed subatoms
  int8_t s[4];     // subatom index of probe j (node order)
  int8_t kc[4];    // cover column (index into the cover's src[]) holding probe j's key
};

// probe one key in a subtrie region: 256-bit bucket loads until a match or a free slot
__device__ __forceinline__ uint32_t probe_region_one(const Slot* table, uint32_t p, uint32_t len, uint32_t kw) {
  uint64_t b = (uint32_t)region_bucket(p, len, kw);
  bool more;
  uint32_t q = bucket_match(ld_bucket(table, b), kw, more);
  while (more) {
    if (++b == region_hi(p, len)) b = region_lo(p);
    q = bucket_match(ld_bucket(table, b), kw, more);
  }
  return q;
}

#ifndef FJG_STREAM_BULK
#define FJG_STREAM_BULK 0  // 1: k_stream_one stages its key column with cp.async.bulk + mbarrier (measured 5% slower on C3 node 0 than the per-lane 4-byte cp.async: one mbarrier wait per 64-key chunk; profiles/README.md)
#endif
constexpr int kStreamStages = 4;  // bulk-copy pipeline depth per warp
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
// global -> shared bulk copy (TMA engine, SASS UBLKCP): 16-byte aligned, size a multiple of 16
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int NP, int R>
struct StreamOneQC {
  static constexpr int QC = R <= 7 ? 256 : 512;  // per-warp ring capacity per stage (>= 32*R + 31)
};

// Write one surviving row (lanes with live set) to the next frontier. qlast is
// the last probe's result; earlier probes are repeated (survivors only).
template <int NP, int W>
__device__ __forceinline__ void stream_one_write(const KNode& N, const SProbe& SP, const KSub& S, bool live,
                                                 uint32_t row, uint32_t qlast, uint32_t pos0, uint64_t mult0,
                                                 const uint32_t (&pp)[NP], const uint32_t (&pl)[NP],
                                                 DevCounters* ctr, int lane) {
  const unsigned bal = __ballot_sync(0xffffffffu, live);
  if (!bal) return;
  uint32_t o = 0;
  if (lane == 0) o = atomicAdd(&ctr->survivors, (uint32_t)__popc(bal));
  o = __shfl_sync(0xffffffffu, o, 0);
  if (!live) return;
  const uint32_t at = o + __popc(bal & ((1u << lane) - 1u));
  const uint32_t pos = pos0 + row;
  uint64_t mult = mult0;
  uint32_t chp[NP], chl[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const KSub& P = N.sub[SP.s[j]];
    const uint32_t q =
        j == NP - 1 ? qlast
                    : probe_region_one(P.table, pp[j], pl[j], (uint32_t)__ldg(S.src[SP.kc[j]] + pos));
    const uint32_t ql = __ldg(P.cnt + q);
    chp[j] = P.last ? 0u : q;
    chl[j] = P.last ? 0u : ql;
    if (P.last) mult *= ql;
  }
#pragma unroll
  for (int v = 0; v < W; ++v)
    if ((N.out_vars >> v) & 1u) {
      int32_t val = 0;
      bool cov = false;
#pragma unroll
      for (int k = 0; k < MAXK; ++k)
        if (k < S.nv && S.var[k] == v) {
          val = __ldg(S.src[k] + pos);
          cov = true;
        }
      N.out_var[v][at] = cov ? val : __ldg(N.in_var[v]);
    }
#pragma unroll
  for (int a = 0; a < W; ++a)
    if ((N.out_atoms >> a) & 1u) {
      uint32_t pa = 0, la = 0;
      bool here = false;
      if (S.atom == a) {
        pa = kSingleton;
        la = 1u;
        here = true;
      }
#pragma unroll
      for (int j = 0; j < NP; ++j)
        if (N.sub[SP.s[j]].atom == a) {
          pa = chp[j];
          la = chl[j];
          here = true;
        }
      if (!here) {
        pa = __ldg(N.in_p[a]);
        la = __ldg(N.in_len[a]);
      }
      N.out_p[a][at] = pa;
      N.out_len[a][at] = la;
    }
  if (N.out_mult) N.out_mult[at] = mult;
}

template <int NP, int R, int W>
__global__ void __launch_bounds__(TILE, FJG_STREAM_MINB) k_stream_one(const __grid_constant__ KNode N, const SProbe SP, uint64_t c0,
                                                        uint64_t c1, DevCounters* ctr) {
  constexpr int QC = StreamOneQC<NP, R>::QC;
  constexpr int NQ = NP > 1 ? NP - 1 : 1;
  __shared__ uint32_t Q[NQ][TILE / 32][QC];  // stage j+1 input: rows alive after probe j
  uint32_t probes = 0, misses = 0, body = 0;
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int ci = N.cov[0];
  const KSub& S = N.sub[ci];
  const uint32_t pos0 = S.in_p ? __ldg(S.in_p) : 0u;
  const uint64_t mult0 = N.in_mult ? __ldg(N.in_mult) : 1ull;
  uint32_t pp[NP], pl[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const KSub& P = N.sub[SP.s[j]];
    if (P.in_p) {
      pp[j] = __ldg(P.in_p);
      pl[j] = __ldg(P.in_len);
    } else {
      pp[j] = 0;
      pl[j] = *P.rregion;
    }
  }
  uint32_t qhead[NQ], qtail[NQ];  // warp-uniform ring cursors
#pragma unroll
  for (int j = 0; j < NQ; ++j) qhead[j] = qtail[j] = 0;

  // push rows alive after probe j into stage j+1's queue, or write them (last probe)
  auto advance = [&](int j, bool live, uint32_t row, uint32_t q) {
    if (j == NP - 1) {
      stream_one_write<NP, W>(N, SP, S, live, row, q, pos0, mult0, pp, pl, ctr, lane);
    } else {
      const unsigned bal = __ballot_sync(0xffffffffu, live);
#pragma unroll
      for (int t = 0; t < NQ; ++t)
        if (t == j) {
          if (live) Q[t][wi][(qtail[t] + __popc(bal & lt_mask)) & (QC - 1)] = row;
          qtail[t] += __popc(bal);
        }
    }
  };
  // stage j >= 1: n (<= 32) queued rows, one per lane
  auto stage = [&](int j, uint32_t n) {
    bool live = (uint32_t)lane < n;
    uint32_t row = 0;
#pragma unroll
    for (int t = 0; t < NQ; ++t)
      if (t == j - 1) {
        if (live) row = Q[t][wi][(qhead[t] + lane) & (QC - 1)];
        qhead[t] += n;
      }
    __syncwarp();
    uint32_t q = kEmpty;
#pragma unroll
    for (int t = 1; t < NP; ++t)
      if (t == j && live) {
        const KSub& P = N.sub[SP.s[t]];
        ++probes;
        q = probe_region_one(P.table, pp[t], pl[t], (uint32_t)__ldg(S.src[SP.kc[t]] + pos0 + row));
        if (q == kEmpty) {
          ++misses;
          live = false;
        }
      }
#pragma unroll
    for (int t = 1; t < NP; ++t)
      if (t == j) advance(t, live, row, q);
  };

  // F == 1: candidates are positions of one subtrie (< 2^31), 32-bit indices
  const uint32_t gstep = gridDim.x * (TILE / 32) * 32u * R;
  const uint32_t e1 = (uint32_t)c1;
  const int32_t* __restrict__ kcol0 = S.src[SP.kc[0]] + pos0;
  const KSub& P0 = N.sub[SP.s[0]];
  uint32_t base = (uint32_t)c0 + (blockIdx.x * (TILE / 32) + wi) * 32u * R;
#if FJG_STREAM_BULK
  // software pipeline: the first-probe keys of the warp's next chunks stream
  // into shared memory as bulk copies (cp.async.bulk, one 128*R-byte copy per
  // chunk issued by lane 0, completion on a per-warp mbarrier per stage;
  // kStreamStages - 1 chunks in flight) while this chunk probes. A chunk that
  // is ragged (the column's end) or not 16-byte aligned is loaded by its lanes.
  __shared__ __align__(16) uint32_t KB[kStreamStages][TILE / 32][32 * R];
  __shared__ uint64_t MB[kStreamStages][TILE / 32];
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStreamStages; ++s) mbar_init(&MB[s][wi], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncwarp();
  const bool bulk_ok = ((reinterpret_cast<uintptr_t>(kcol0) & 15u) == 0) && ((base & 3u) == 0);
  auto prefetch = [&](uint32_t b, int stg) {
    if (b >= e1) return;
    if (bulk_ok && e1 - b >= 32u * R) {
      if (lane == 0) {
        mbar_expect_tx(&MB[stg][wi], 32u * R * 4u);
        bulk_g2s(&KB[stg][wi][0], kcol0 + b, 32u * R * 4u, &MB[stg][wi]);
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t i = b + r * 32 + lane;
        KB[stg][wi][r * 32 + lane] = i < e1 ? (uint32_t)__ldg(kcol0 + i) : 0u;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&MB[stg][wi]);
    }
  };
#pragma unroll
  for (int s = 0; s < kStreamStages - 1; ++s) prefetch(base + s * gstep, s);
  for (uint32_t it = 0; base < e1; base += gstep, ++it) {
    const int buf = it % kStreamStages;
    __syncwarp();  // every lane has read the stage refilled below (one iteration ago)
    prefetch(base + (kStreamStages - 1) * gstep, (it + kStreamStages - 1) % kStreamStages);
    mbar_wait(&MB[buf][wi], (it / kStreamStages) & 1u);
#else
  // software pipeline: the next chunk's first-probe keys stream into shared
  // memory (cp.async, double buffer) while this chunk probes; each lane copies
  // and reads only its own slots, so no warp barrier is needed.
  __shared__ uint32_t KB[2][TILE / 32][32 * R];
  auto prefetch = [&](uint32_t b, int buf) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t i = b + r * 32 + lane;
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&KB[buf][wi][r * 32 + lane]);
      const int32_t* src = kcol0 + (i < e1 ? i : 0u);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(i < e1 ? 4 : 0));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  prefetch(base, 0);
  int buf = 0;
  for (; base < e1; base += gstep, buf ^= 1) {
    prefetch(base + gstep, buf ^ 1);
    asm volatile("cp.async.wait_group 1;\n" ::);
#endif
    uint32_t kw[R], b0[R];
    bool live[R];
    Bucket8 h[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      live[r] = base + r * 32 + lane < e1;
      body += live[r] ? 1u : 0u;
      kw[r] = KB[buf][wi][r * 32 + lane];
      b0[r] = (uint32_t)region_bucket(pp[0], pl[0], kw[r]);
      if (live[r]) h[r] = ld_bucket(P0.table, b0[r]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      uint32_t q = kEmpty;
      if (live[r]) {
        ++probes;
        bool more;
        q = bucket_match(h[r], kw[r], more);
        if (more) {
          uint64_t b = b0[r];
          do {
            if (++b == region_hi(pp[0], pl[0])) b = region_lo(pp[0]);
            q = bucket_match(ld_bucket(P0.table, b), kw[r], more);
          } while (more);
        }
        if (q == kEmpty) {
          ++misses;
          live[r] = false;
        }
      }
      advance(0, live[r], base + r * 32 + lane, q);
    }
    // later stages on full batches of 32 queued rows
#pragma unroll
    for (int j = 1; j < NP; ++j)
      while (qtail[j - 1] - qhead[j - 1] >= 32) stage(j, 32);
  }
#if !FJG_STREAM_BULK
  asm volatile("cp.async.wait_group 0;\n" ::);
#endif
  // drain the partial batches, stage by stage
#pragma unroll
  for (int j = 1; j < NP; ++j)
    while (qtail[j - 1] != qhead[j - 1]) stage(j, min(32u, qtail[j - 1] - qhead[j - 1]));
  const uint64_t tprobes = warp_sum((uint64_t)probes), tmisses = warp_sum((uint64_t)misses),
                 tbody = warp_sum((uint64_t)body);
  if (lane == 0) {
    if (tprobes) {
      atomicAdd((unsigned long long*)&ctr->probes, (unsigned long long)tprobes);
      atomicAdd((unsigned long long*)&ctr->node_probes[N.k], (unsigned long long)tprobes);
    }
    if (tmisses) atomicAdd((unsigned long long*)&ctr->misses, (unsigned long long)tmisses);
    if (tbody) atomicAdd((unsigned long long*)&ctr->body[N.k], (unsigned long long)tbody);
  }
}

// Fused Cartesian tail (TailPlan): thread per binding of node k's frontier;
// a binding whose product exceeds 8 tuples is expanded by its whole warp
// (lanes stride the product). Each output tuple = the binding's values plus one
// row of every tail subtrie (mixed-radix index, last tail node fastest); counts,
// checksum and MIN fold as in the last node, or tuples are written (ENUM).
template <int MODE, int W, int NT>
__device__ __forceinline__ void tail_expand(const KNode& N, const TailPlan& T, uint64_t e, uint64_t start,
                                            uint32_t step, bool own, int min_var, int32_t* __restrict__ out_tuples,
                                            uint64_t out_cap, DevCounters* ctr, uint64_t& acc_lo, uint64_t& acc_hi,
                                            uint64_t& acc_sum, long long& acc_min, uint64_t (&inputs)[NT],
                                            uint64_t (&body)[NT], unsigned long long obase_in = 0) {
  int32_t val[W];
#pragma unroll
  for (int v = 0; v < W; ++v) val[v] = ((N.in_vars >> v) & 1u) ? __ldg(N.in_var[v] + e) : 0;
  const uint64_t mult = N.in_mult ? __ldg(N.in_mult + e) : 1ull;
  uint32_t tp[NT], tl[NT];
  uint64_t prod = 1;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    if (j >= T.ntail) continue;
    if (T.open[j]) {
      tp[j] = __ldg(T.in_p[j] + e);
      tl[j] = __ldg(T.in_len[j] + e);
    } else {
      tp[j] = 0;
      tl[j] = T.sub[j].root_n;
    }
    const uint32_t c = tp[j] == kSingleton ? 1u : tl[j];
    if (own) inputs[j] += prod;
    prod *= c;
    if (own) body[j] += prod;
  }
  const bool narrow = prod <= 0xFFFFFFFFull;
  // enumerate: the binding's prod * mult rows are reserved with one atomic (by
  // the thread that owns it, or lane 0 for a warp-expanded binding)
  unsigned long long obase = 0;
  if (MODE == EXPAND_ENUM) {
    if (own) {  // reserved by k_tail for its warp (a big binding's own call writes no rows)
      obase = obase_in;
    } else {
      if (start == 0 && prod) obase = atomicAdd((unsigned long long*)&ctr->out_rows, (unsigned long long)(prod * mult));
      obase = __shfl_sync(0xffffffffu, obase, 0);
    }
  }
  for (uint64_t idx = start; idx < prod; idx += step) {
    uint64_t rest = idx;
#pragma unroll
    for (int j = NT - 1; j >= 0; --j) {
      if (j >= T.ntail) continue;
      const uint32_t c = tp[j] == kSingleton ? 1u : tl[j];
      uint32_t off;
      if (j == 0) {  // outermost: the remaining index is the offset
        off = (uint32_t)rest;
      } else if (narrow) {
        off = (uint32_t)rest % c;
        rest = (uint32_t)rest / c;
      } else {
        off = (uint32_t)(rest % c);
        rest /= c;
      }
      if (tp[j] == kSingleton) continue;
      const KSub& S = T.sub[j];
#pragma unroll
      for (int t = 0; t < MAXK; ++t)
        if (t < S.nv) put(val, S.var[t], __ldg(S.src[t] + tp[j] + off));
    }
    {  // count / checksum / MIN (also when enumerating: one pass yields both)
      uint64_t h = fj::kTupleHashSeed;
#pragma unroll
      for (int v = 0; v < W; ++v)
        if (v < N.nhead) h = fj::tuple_hash_step(h, (int64_t)val[v]);
      acc_sum += mult * fj::checksum_word(h);
      acc_lo += mult;
      if (acc_lo < mult) ++acc_hi;
      if (min_var >= 0) acc_min = min(acc_min, (long long)sel(val, min_var));
    }
    if (MODE == EXPAND_ENUM) {
      const unsigned long long o = obase + idx * mult;
      for (uint64_t r = 0; r < mult && o + r < out_cap; ++r)
#pragma unroll
        for (int v = 0; v < W; ++v)
          if (v < N.nhead) out_tuples[(o + r) * N.nhead + v] = val[v];
    }
  }
}

// dF (optional): the frontier size on the device (the previous node's
// survivor count, no host round trip); node k's inputs are then counted here.
template <int MODE, int W, int NT>
__global__ void __launch_bounds__(TILE) k_tail(const __grid_constant__ KNode N, const __grid_constant__ TailPlan T,
                                               uint64_t F, const uint32_t* __restrict__ dF, int min_var,
                                               int32_t* __restrict__ out_tuples, uint64_t out_cap,
                                               DevCounters* ctr) {
  if (dF) {
    F = *dF;
    if (blockIdx.x == 0 && threadIdx.x == 0 && F)
      atomicAdd((unsigned long long*)&ctr->tail_inputs[T.node[0]], (unsigned long long)F);
  }
  uint64_t acc_lo = 0, acc_hi = 0, acc_sum = 0;
  long long acc_min = LLONG_MAX;
  uint64_t inputs[NT], body[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) inputs[j] = body[j] = 0;
  const int lane = threadIdx.x & 31;
  for (uint64_t b = (uint64_t)blockIdx.x * TILE; b < F; b += (uint64_t)gridDim.x * TILE) {
    const uint64_t e = b + threadIdx.x;
    bool big = false;
    unsigned long long own_rows = 0;
    if (e < F) {
      uint64_t prod = 1;
#pragma unroll
      for (int j = 0; j < NT; ++j)
        if (j < T.ntail) {
          const uint32_t p = T.open[j] ? __ldg(T.in_p[j] + e) : 0u;
          const uint32_t l = T.open[j] ? __ldg(T.in_len[j] + e) : T.sub[j].root_n;
          prod *= p == kSingleton ? 1u : l;
        }
      big = prod > 8;
      own_rows = big ? 0ull : prod * (N.in_mult ? __ldg(N.in_mult + e) : 1ull);
    }
    unsigned long long obase = 0;
    if (MODE == EXPAND_ENUM) {  // the warp's own rows: one atomic, lane offsets by scan
      unsigned long long off = own_rows;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long o = __shfl_up_sync(0xffffffffu, off, d);
        if (lane >= d) off += o;
      }
      const unsigned long long total = __shfl_sync(0xffffffffu, off, 31);
      unsigned long long base = 0;
      if (lane == 0 && total) base = atomicAdd((unsigned long long*)&ctr->out_rows, total);
      obase = __shfl_sync(0xffffffffu, base, 0) + off - own_rows;
    }
    if (e < F)  // small products: this thread alone (and it counts the binding's inputs/body)
      tail_expand<MODE, W, NT>(N, T, e, big ? ~0ull : 0ull, 1u, true, min_var, out_tuples, out_cap, ctr, acc_lo,
                           acc_hi, acc_sum, acc_min, inputs, body, obase);
    unsigned bm = __ballot_sync(0xffffffffu, big);
    uint64_t none[NT], nb[NT];
    while (bm) {  // big products: the whole warp strides them
      const int src = __ffs(bm) - 1;
      bm &= bm - 1;
      const uint64_t eb = __shfl_sync(0xffffffffu, e, src);
      tail_expand<MODE, W, NT>(N, T, eb, lane, 32u, false, min_var, out_tuples, out_cap, ctr, acc_lo, acc_hi, acc_sum,
                           acc_min, none, nb);
    }
  }
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
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    inputs[j] = warp_sum(inputs[j]);
    body[j] = warp_sum(body[j]);
  }
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < NT; ++j)
      if (j < T.ntail) {
        // node k's inputs are counted on the host (run_node)
        if (j > 0 && inputs[j]) atomicAdd((unsigned long long*)&ctr->tail_inputs[T.node[j]], (unsigned long long)inputs[j]);
        if (body[j]) atomicAdd((unsigned long long*)&ctr->body[T.node[j]], (unsigned long long)body[j]);
      }
    if (MODE == EXPAND_COUNT || MODE == EXPAND_ENUM) {
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

// The stream fast path: a single cover in stream mode whose subtrie is never a
// singleton, all its variables fresh; every other subatom probes one variable
// the cover binds.
static bool stream_write_ok(const DevNode& N, const KNode& G) {
  if (N.ncov != 1 || N.nsub < 2) return false;
  const DevSub& C = N.sub[N.cov[0]];
  if (!C.stream || C.bound_mask || C.nv < 1) return false;
  if (G.sub[N.cov[0]].in_p == nullptr && C.depth != 0) return false;
  for (int s = 0; s < N.nsub; ++s) {
    if (s == N.cov[0]) continue;
    const DevSub& P = N.sub[s];
    if (P.nv != 1) return false;
    bool found = false;
    for (int t = 0; t < C.nv; ++t)
      if (C.var[t] == P.var[0]) found = true;
    if (!found) return false;
  }
  return true;
}

// A frontier-writing node is GJ-shaped when every subatom is a one-variable
// cover of the same fresh variable (levels of depth >= 0, no bound check).
static int gj_write_var(const DevNode& N, int width) {
  if (N.nsub < 2 || N.nsub > 3 || N.ncov != N.nsub || width > 8) return -1;
  int x = -1;
  for (int s = 0; s < N.nsub; ++s) {
    const DevSub& D = N.sub[s];
    if (D.nv != 1 || D.bound_mask) return -1;
    if (x >= 0 && D.var[0] != x) return -1;
    x = D.var[0];
  }
  return x;
}

// The GJ fast path applies when every subatom of the node is a one-variable
// cover of the same new, unbound variable, and no subtrie can be a streamed
// singleton (all subatoms keys-or-stream levels of depth >= 0 with nv == 1).
static int gj_last_var(const KNode& G, const DevNode& N) {
  if (N.nsub < 2 || N.nsub > 3 || N.ncov != N.nsub || N.nhead > 8) return -1;
  int x = -1;
  for (int s = 0; s < N.nsub; ++s) {
    const DevSub& D = N.sub[s];
    if (D.nv != 1 || D.bound_mask || !D.stream) return -1;
    if (x >= 0 && D.var[0] != x) return -1;
    x = D.var[0];
  }
  // every earlier subatom of these atoms bound variables (no singleton residuals)
  for (int s = 0; s < N.nsub; ++s)
    if (G.sub[s].in_p == nullptr && N.sub[s].depth != 0) return -1;
  return x;
}

