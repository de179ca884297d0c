// select: k_select: dynamic cover, candidate counts, force claims
// Included by engine.cu (one translation unit: the kernels share templates and helpers).
#pragma once

// ============================================================================
// k_select: cover choice, candidate counts, force claims
// ============================================================================
__device__ __forceinline__ void claim_subtrie(const DevTrie* tries, DevCounters* ctr, const KSub& S, uint32_t p,
                                              uint32_t len, bool need) {
  // Warp-level dedup of identical subtries (bindings of one parent are
  // adjacent in the frontier), a CAS on the state word, then one list append
  // per warp (the list counter is a single hot address).
  const unsigned act = __activemask();
  const unsigned want = __ballot_sync(act, need);
  if (!want) return;
  const int lane = threadIdx.x & 31;
  bool lead = false;
  if (need) {
    const unsigned grp = __match_any_sync(want, p);
    lead = lane == __ffs(grp) - 1;
  }
  if (S.depth == 0) {
    if (lead) ctr->root_need[S.trie] = 1;
    return;
  }
  const DevLevel& L = tries[S.trie].lev[S.depth];
  bool won = false;
  if (lead && atomicCAS(&L.sn[p].state, 0u, 1u) == 0u) {
    won = true;
    L.cursor[p] = 0;
    L.sn[p].nkeys = 0;
  }
  const unsigned wm = __ballot_sync(act, won);
  if (!wm) return;
  const int first = __ffs(wm) - 1;
  uint32_t base = 0;
  // the claimed offsets, so the force sizes its owner map by them, not by the level
  const uint32_t tot = __reduce_add_sync(act, won ? len : 0u);
  if (lane == first) {
    base = atomicAdd(&ctr->list_count[S.trie * MAXL + S.depth], (uint32_t)__popc(wm));
    atomicAdd(&ctr->list_total[S.trie * MAXL + S.depth], tot);
  }
  base = __shfl_sync(act, base, first);
  if (won) {
    const uint32_t idx = base + __popc(wm & ((1u << lane) - 1u));
    L.list_p[idx] = p;
    L.list_len[idx] = len;
  }
}

__global__ void k_select(const __grid_constant__ KNode N, const DevTrie* __restrict__ tries, uint64_t F,
                         int dynamic, DevCounters* ctr) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t start = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t iters = (F + stride - 1) / stride;
  for (uint64_t it = 0; it < iters; ++it) {
    const uint64_t e = start + it * stride;
    const bool ok = e < F;
    int best = N.cov[0];
    uint32_t bp = 0, bl = 0;
    if (ok) {
      subtrie_of(N.sub[best], e, bp, bl);
      if (dynamic && N.ncov > 1) {
        uint64_t best_est = estimate(N.sub[best], bp, bl);
        for (int ci = 1; ci < N.ncov; ++ci) {
          const int s = N.cov[ci];
          uint32_t p, l;
          subtrie_of(N.sub[s], e, p, l);
          const uint64_t est = estimate(N.sub[s], p, l);
          if (est < best_est) {  // ties keep the lowest position
            best_est = est;
            best = s;
            bp = p;
            bl = l;
          }
        }
      }
      N.chosen[e] = (uint8_t)best;
      N.m[e] = (bp == kSingleton) ? 1ull : (uint64_t)bl;
    }
    // claims: the keys-iterated cover and every probed subatom must be forced
    for (int s = 0; s < N.nsub; ++s) {
      const KSub& S = N.sub[s];
      uint32_t p = 0, l = 0;
      bool need = false;
      if (ok) {
        subtrie_of(S, e, p, l);
        need = (p != kSingleton) && (s != best || !S.stream);
        if (need) need = *((volatile const uint32_t*)&S.sn[S.depth == 0 ? 0u : p].state) == 0u;
      }
      claim_subtrie(tries, ctr, S, p, l, need);
    }
  }
}


#ifndef FJG_SELECT_ILP
#define FJG_SELECT_ILP 1  // bindings per thread and trip (2 measured equal on C5: the kernel is bound by random DRAM sectors, not by latency)
#endif
// k_select for nodes of at most NS subatoms: each subatom's subtrie and state
// word are read once per binding and reused by the cover choice and the claims
// (the generic kernel re-reads them for the claims).
template <int NS>
__global__ void k_select_ns(const __grid_constant__ KNode N, const DevTrie* __restrict__ tries, uint64_t F,
                            int dynamic, DevCounters* ctr) {
  // U bindings per thread and trip: their subtrie ranges, then their {state,
  // key count} records are loaded back to back, the claims run after
  constexpr int U = FJG_SELECT_ILP;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t start = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t iters = (F + U * stride - 1) / (U * stride);
  for (uint64_t it = 0; it < iters; ++it) {
    uint64_t e[U];
    bool ok[U];
    uint32_t p[U][NS], l[U][NS], st[U][NS], nk[U][NS];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      e[u] = start + (it * U + u) * stride;
      ok[u] = e[u] < F;
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        p[u][s] = l[u][s] = nk[u][s] = 0;
        st[u][s] = 1;
        if (ok[u] && s < N.nsub) subtrie_of(N.sub[s], e[u], p[u][s], l[u][s]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int s = 0; s < NS; ++s)
        if (ok[u] && s < N.nsub && p[u][s] != kSingleton) {
          const KSub& S = N.sub[s];
          const uint2 sn = ld_substate(S.sn + (S.depth == 0 ? 0u : p[u][s]));  // state + key count: one load
          st[u][s] = sn.x;
          nk[u][s] = sn.y;
        }
    const bool est_all = dynamic && N.ncov > 1;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int best = N.cov[0];
      if (ok[u]) {
        auto est = [&](int s) -> uint64_t {
          uint64_t v = 0;
#pragma unroll
          for (int t = 0; t < NS; ++t)
            if (t == s) v = p[u][t] == kSingleton ? 1ull : (st[u][t] == 2u ? (uint64_t)nk[u][t] : l[u][t]);
          return v;
        };
        if (est_all) {
          uint64_t best_est = est(best);
          for (int ci = 1; ci < N.ncov; ++ci) {
            const int s = N.cov[ci];
            const uint64_t v = est(s);
            if (v < best_est) {  // ties keep the lowest position
              best_est = v;
              best = s;
            }
          }
        }
        uint32_t bp = 0, bl = 0;
#pragma unroll
        for (int t = 0; t < NS; ++t)
          if (t == best) {
            bp = p[u][t];
            bl = l[u][t];
          }
        N.chosen[e[u]] = (uint8_t)best;
        N.m[e[u]] = (bp == kSingleton) ? 1ull : (uint64_t)bl;
      }
      // claims: the keys-iterated cover and every probed subatom must be forced
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        if (s >= N.nsub) break;
        const KSub& S = N.sub[s];
        const bool need = ok[u] && p[u][s] != kSingleton && (s != best || !S.stream) && st[u][s] == 0u;
        claim_subtrie(tries, ctr, S, p[u][s], l[u][s], need);
      }
    }
  }
}

// Inclusive scan of a small frontier's candidate counts in one block (F <=
// kSmallScan), total written to DevCounters::total_m: one launch instead of
// the look-back scan's tile machinery.
constexpr uint64_t kSmallScan = 1024ull * 32;
__global__ void __launch_bounds__(1024) k_scan_small(const uint64_t* __restrict__ m, uint64_t* __restrict__ scan,
                                                     uint32_t F, DevCounters* ctr) {
  __shared__ uint64_t tmp[32];
  const uint32_t per = (F + 1023) / 1024;
  const uint32_t b = threadIdx.x * per, e = min(F, b + per);
  uint64_t local = 0;
  for (uint32_t i = b; i < e; ++i) local += m[i];
  uint64_t excl, total;
  excl = prims::block_excl_scan<1024>(local, total, tmp, prims::OpSum(), (uint64_t)0);
  for (uint32_t i = b; i < e; ++i) {
    excl += m[i];
    scan[i] = excl;
  }
  if (threadIdx.x == 0) ctr->total_m = total;
}
