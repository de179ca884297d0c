// force: batched lazy COLT forcing (Fig 12 force)
// Included by engine.cu (one translation unit: the kernels share templates and helpers).
#pragma once

// ============================================================================
// force: clear -> insert -> assign -> scatter -> finalize  (Fig 12 `force`)
//
// Optimistic members (FJG_FORCE_OPT; the claimed subtries of a level >= 1 with
// one-column keys, while no force of that level has met a repeated key): the
// insert assumes every key of a subtrie is distinct -- the winner's CAS writes
// the final slot {key, child start = its own position} and the same thread
// writes the unit child count and the clustered values, so clear + insert is
// the whole force (no scratch arrays, no second pass over the rows; a level of
// deduplicated graph edges always ends here). A repeated key flags the member,
// and the redo launches (clear, insert with phase 1; they exit at once
// otherwise) run the general counting protocol over the same subtries.
// ============================================================================
#ifndef FJG_FORCE_OPT
#define FJG_FORCE_OPT 1
#endif
#ifndef FJG_CLEAR_STREAM
#define FJG_CLEAR_STREAM 1
#endif
// Position iteration over the union of claimed ranges. single: one subtrie
// (p0, len0) given by value (the root BaseScan).
struct ForceRange {
  const uint32_t* list_p;
  const uint32_t* list_len;
  const uint32_t* list_scan;   // inclusive
  const uint32_t* list_count;  // device count
  const uint32_t* owner;       // list entry of every forced offset index (max-scan of start markers)
  uint32_t p0, len0;
  int single;
  int trie, lev;      // the (trie, level) this member forces
  uint32_t slot_off;  // its offset into the tmp_slot / tmp_rank scratch
};

// Forces launched together (blockIdx.y = member): every root a node claims in
// one set of launches; a level >= 1 force is a batch of one.
struct ForceBatch {
  int n;
  ForceRange R[MAXT];
};

__device__ __forceinline__ uint32_t force_total(const ForceRange& R) {
  if (R.single) return R.len0;
  const uint32_t c = *R.list_count;
  return c ? R.list_scan[c - 1] : 0u;
}

__device__ __forceinline__ void force_locate(const ForceRange& R, uint32_t i, uint32_t& p, uint32_t& len,
                                             uint32_t& pos) {
  if (R.single) {
    p = R.p0;
    len = R.len0;
    pos = R.p0 + i;
    return;
  }
  const uint32_t lo = __ldg(R.owner + i);
  const uint32_t before = lo ? R.list_scan[lo - 1] : 0u;
  p = R.list_p[lo];
  len = R.list_len[lo];
  pos = p + (i - before);
}

// owner map, pass 1: mark the first offset index of every listed subtrie
__global__ void k_force_marks(const uint32_t* __restrict__ list_scan, const uint32_t* __restrict__ list_count,
                              uint32_t* __restrict__ marks) {
  const uint32_t c = *list_count;
  for (uint32_t li = blockIdx.x * blockDim.x + threadIdx.x; li < c; li += gridDim.x * blockDim.x)
    marks[li ? list_scan[li - 1] : 0u] = li;
}

// clear the slot regions (one 4-slot bucket per position) and child counts of
// the claimed subtries
__global__ void k_force_clear(const DevTrie* __restrict__ tries, const __grid_constant__ ForceBatch B,
                              DevCounters* ctr, int phase, int opt_ok) {
  const int y = blockIdx.y;
  const ForceRange& R = B.R[y];
  const int lev = R.lev;
  const DevLevel& L = tries[R.trie].lev[lev];
  // phase 1 (redo): only a member whose optimistic insert met a repeated key
  if (phase == 1 && !(ctr->fopt[y] && ctr->fdup[y])) return;
  const uint32_t total = force_total(R);
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // this member's counters (read by the later kernels only)
    ctr->fnew[y] = 0;
    if (phase == 0) {
      ctr->fdup[y] = 0;
      int ncl = 0;  // clustered columns of this level (the optimistic insert copies at most two)
      for (int c = 0; c < tries[R.trie].ncols; ++c) ncl += L.cval[c] ? 1 : 0;
      ctr->fopt[y] = (opt_ok && !R.single && ncl <= 2 && !ctr->level_dup[R.trie * MAXL + lev]) ? 1u : 0u;
    }
    if (R.single) {
      L.cursor[lev == 0 ? 0 : R.p0] = 0;
      L.sn[lev == 0 ? 0 : R.p0].nkeys = 0;
    }
  }
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    uint32_t p, len, pos;
    force_locate(R, i, p, len, pos);
    uint4* t = reinterpret_cast<uint4*>(L.table) + 2ull * FJG_RS * pos;  // this position's buckets
#if FJG_CLEAR_STREAM
    // streaming (evict-first) stores: the cleared lines must not stay resident in
    // L2, where they crowd out the lines the insert's CAS traffic reuses
#pragma unroll
    for (int u = 0; u < 2 * FJG_RS; ++u) __stcs(t + u, make_uint4(kEmpty, kEmpty, kEmpty, kEmpty));
    __stcs(L.cnt + pos, 0u);
#else
#pragma unroll
    for (int u = 0; u < 2 * FJG_RS; ++u) t[u] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    L.cnt[pos] = 0;
#endif
    if (phase == 1 && pos == p) {  // the optimistic insert set them to the unit grouping
      L.cursor[p] = 0;
      L.sn[p].nkeys = 0;
    }
    if (L.srep)
#pragma unroll
      for (int u = 0; u < FJG_RS; ++u) reinterpret_cast<uint4*>(L.srep)[(uint64_t)FJG_RS * pos + u] = make_uint4(0u, 0u, 0u, 0u);
  }
}

// Insert every offset of the claimed subtries: claim a slot for its key (CAS
// on the 8-byte slot), then count it (the pending slot's q word is the group
// counter; the returned value is the offset's rank inside its child group).
#ifndef FJG_FORCE_MINB
#define FJG_FORCE_MINB 4
#endif
#ifndef FJG_FORCE_SYNC_ALL
#define FJG_FORCE_SYNC_ALL 0  // 1: roots reconverge every trip too
#endif
// OPTK: the kernel of a batch that may hold optimistic members (level >= 1,
// one-column keys); roots and multi-column keys run the plain instantiation
// (48 registers, 5 blocks per SM, no per-trip reconvergence: on a root's wide
// region the lanes that run ahead hide latency, C1 chain 0.47 vs 0.50 ms).
template <bool MULTI, bool OPTK>
__global__ void __launch_bounds__(256, OPTK ? FJG_FORCE_MINB : 5) k_force_insert(const DevTrie* __restrict__ tries, const __grid_constant__ ForceBatch B,
                               uint32_t* __restrict__ tmp_slot, uint32_t* __restrict__ tmp_rank,
                               DevCounters* ctr, int phase) {
  const int y = blockIdx.y;
  const ForceRange& R = B.R[y];
  const int trie = R.trie, lev = R.lev;
  const bool fopt = OPTK && !MULTI && ctr->fopt[y] != 0;
  if (phase == 1 && !(fopt && ctr->fdup[y])) return;
  const bool opt = fopt && phase == 0;  // optimistic: slots receive their final value
  tmp_slot += R.slot_off;
  tmp_rank += R.slot_off;
  const DevTrie& T = tries[trie];
  const DevLevel& L = T.lev[lev];
  const uint32_t total = force_total(R);
  const int nk = L.nk;
  const int32_t* src[MAXK];
#pragma unroll
  for (int t = 0; t < MAXK; ++t) src[t] = t < nk ? level_src(T, lev, L.keycol[t]) : nullptr;
  bool sawdup = false;  // a repeated key: flagged once per block at the end (one hot address)
  uint32_t wins = 0;     // slots this thread claimed (new keys), summed once per block at the end
  // block-uniform trip count (the end-of-kernel block reduction needs every thread)
  // optimistic members copy their (at most two: k_force_clear checks) clustered
  // columns in place; the pointers are loaded once
  const int32_t *osrc0 = nullptr, *osrc1 = nullptr;
  int32_t *odst0 = nullptr, *odst1 = nullptr;
  if (opt)
    for (int c = 0; c < T.ncols; ++c)
      if (L.cval[c]) {
        if (!odst0) {
          osrc0 = level_src(T, lev, c);
          odst0 = L.cval[c];
        } else {
          osrc1 = level_src(T, lev, c);
          odst1 = L.cval[c];
        }
      }
  for (uint32_t b0 = blockIdx.x * blockDim.x; b0 < total; b0 += gridDim.x * blockDim.x) {
    const uint32_t i = b0 + threadIdx.x;
    const bool live = i < total;
    bool won = false;
    uint64_t h = 0;
    uint32_t p = 0, len = 0, pos = 0;
    if (live) {
      force_locate(R, i, p, len, pos);
      int32_t vals[MAXK];
#pragma unroll
      for (int t = 0; t < MAXK; ++t) vals[t] = t < nk ? src[t][pos] : 0;
      const uint32_t kw = key_word_r(nk, vals);
      // the winner's CAS already counts it (rank 0); repeated keys add to the count
      // (optimistic: the final slot, child start = this position)
      const unsigned long long mine = ((unsigned long long)(opt ? pos : (kPendBit | 1u)) << 32) | kw;
      const uint64_t lo = 4ull * region_lo(p), hi = 4ull * region_hi(p, len);
      h = 4ull * region_bucket(p, len, kw);
      FJG_ASSERT(lo <= h && h < hi && pos >= p && pos < (uint64_t)p + len);
      bool first = R.single;  // roots: wide regions, the home slot is usually free
      while (true) {
        unsigned long long* addr = reinterpret_cast<unsigned long long*>(L.table + h);
        // a root's home slot is tried with a CAS straight away (a cleared slot
        // is all ones, so a free home slot costs one atomic and no load); other
        // slots -- and every slot of a small subtrie region, where the keys
        // crowd a few buckets -- are read first
        unsigned long long cur = first ? kEmpty64 : *((volatile unsigned long long*)addr);
        first = false;
        if (cur == kEmpty64) {
          const unsigned long long old = atomicCAS(addr, kEmpty64, mine);
          if (old == kEmpty64) {
            won = true;
            if (MULTI) {
              *((volatile uint32_t*)(L.srep + h)) = pos + 1;
              __threadfence();
            }
            break;
          }
          cur = old;
        }
        if ((uint32_t)cur == kw) {
          if (!MULTI) {
            sawdup = true;
            break;
          }
          uint32_t r;
          while ((r = *((volatile uint32_t*)(L.srep + h))) == 0u) {
          }
          bool eq = true;
#pragma unroll
          for (int t = 0; t < MAXK; ++t)
            if (t < nk && src[t][r - 1] != vals[t]) eq = false;
          if (eq) {
            sawdup = true;
            break;
          }
        }
        if (++h == hi) h = lo;
      }
    }
    // Reconverge the warp (every lane reaches this: the trip count is block
    // uniform). Lanes leave the probe loop at different times; left alone, the
    // early ones run ahead into the stores and the next trip, the warp splits
    // into fragments of ~13 lanes and every coalesced load and store of a trip
    // is issued once per fragment (ncu source view: 2x the instructions, L2
    // sectors and DRAM bytes of the converged kernel).
    if (OPTK || FJG_FORCE_SYNC_ALL) __syncwarp();
    if (live) {
      if (opt) {
        // unit child group of this row (force_unique_body's work, same thread)
        L.cnt[pos] = 1;
        if (pos == p) {
          L.sn[p].nkeys = len;
          L.cursor[p] = len;
        }
        if (odst0) odst0[pos] = osrc0[pos];
        if (odst1) odst1[pos] = osrc1[pos];
      } else {
        const uint32_t rank = won ? 0u : (atomicAdd(&L.table[h].q, 1u) & ~kPendBit);
        tmp_slot[pos] = (uint32_t)h;
        tmp_rank[pos] = rank;
      }
    }
    wins += won ? 1u : 0u;
    if (OPTK || FJG_FORCE_SYNC_ALL) __syncwarp();
  }
  // new keys and the repeated-key flag: one atomic per block (k_force_assign
  // finds the new slots as the rank-0 offsets, so no slot list is appended)
  __shared__ uint32_t rtmp[8];
  const uint32_t bw = prims::block_sum<256>(wins, rtmp);
  if (threadIdx.x == 0 && bw) atomicAdd(&ctr->fnew[y], bw);
  if (__syncthreads_or(sawdup) && threadIdx.x == 0) {
    ctr->fdup[y] = 1u;
    ctr->level_dup[trie * MAXL + lev] = 1u;
  }
}

// Child-range allocation: q = p + (running sum of child sizes of p).
template <bool SINGLE>
__global__ void k_force_assign(const DevTrie* __restrict__ tries, const __grid_constant__ ForceBatch B,
                               const uint32_t* __restrict__ tmp_slot, const uint32_t* __restrict__ tmp_rank,
                               DevCounters* ctr) {
  const int y = blockIdx.y;
  const ForceRange& R = B.R[y];
  if (!ctr->fdup[y]) return;  // the all-distinct case is k_force_scatter's identity grouping
  const uint32_t p0 = R.p0;
  tmp_slot += R.slot_off;
  tmp_rank += R.slot_off;
  const DevLevel& L = tries[R.trie].lev[R.lev];
  const uint32_t total = force_total(R);
  __shared__ uint32_t tmp[8];
  __shared__ uint32_t s_base;
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t iters = (total + stride - 1) / stride;
  for (uint32_t it = 0; it < iters; ++it) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x + it * stride;
    // the new slots are the rank-0 offsets (the winner of each key's CAS)
    bool ok = false;
    uint32_t h = 0, c = 0, p = 0;
    if (i < total) {
      uint32_t len, pos;
      force_locate(R, i, p, len, pos);
      if (tmp_rank[pos] == 0) {
        ok = true;
        h = tmp_slot[pos];
        c = L.table[h].q & ~kPendBit;
      }
    }
    uint32_t q = 0;
    if (SINGLE) {
      uint32_t excl, blk_total;
      excl = prims::block_excl_scan<256>(c, blk_total, tmp, prims::OpSum(), 0u);
      const uint32_t nb = __syncthreads_count(ok);
      if (threadIdx.x == 0 && nb) {
        s_base = p0 + atomicAdd(&L.cursor[p0], blk_total);
        atomicAdd(&L.sn[p0].nkeys, nb);
      }
      __syncthreads();
      q = s_base + excl;
      __syncthreads();
    } else if (ok) {
      const unsigned act = __activemask();
      const unsigned grp = __match_any_sync(act, p);
      const int lane = threadIdx.x & 31;
      const int leader = __ffs(grp) - 1;
      uint32_t pre = 0, tot = 0;
      unsigned m = grp;
      while (m) {
        const int l = __ffs(m) - 1;
        m &= m - 1;
        const uint32_t cl = __shfl_sync(grp, c, l);
        if (l < lane) pre += cl;
        tot += cl;
      }
      uint32_t base = 0;
      if (lane == leader) {
        base = atomicAdd(&L.cursor[p], tot);
        atomicAdd(&L.sn[p].nkeys, (uint32_t)__popc(grp));
      }
      base = __shfl_sync(grp, base, leader);
      q = p + base + pre;
    }
    if (ok) {
      L.table[h].q = q;
      L.cnt[q] = c;
    }
  }
}

__device__ void force_unique_body(const DevTrie* __restrict__ tries, int trie, int lev, const ForceRange& R,
                                  const uint32_t* __restrict__ tmp_slot);

// Scatter the clustered columns to their child ranges (repeated keys met), or
// the identity grouping (k_force_unique's body) when every key was distinct.
// Also finalizes the member (its subtries' state = forced, keys counted):
// only later kernels read those, and they are stream-ordered after this one.
__global__ void k_force_scatter(const DevTrie* __restrict__ tries, const __grid_constant__ ForceBatch B,
                                const uint32_t* __restrict__ tmp_slot, const uint32_t* __restrict__ tmp_rank,
                                DevCounters* ctr) {
  const int y = blockIdx.y;
  const ForceRange& R = B.R[y];
  const int trie = R.trie, lev = R.lev;
  tmp_slot += R.slot_off;
  tmp_rank += R.slot_off;
  {
    const DevLevel& L = tries[trie].lev[lev];
    if (blockIdx.x == 0 && threadIdx.x == 0)  // members of a batch finalize concurrently
      atomicAdd((unsigned long long*)&ctr->keys_inserted, (unsigned long long)ctr->fnew[y]);
    if (R.single) {
      if (blockIdx.x == 0 && threadIdx.x == 0) L.sn[lev == 0 ? 0 : R.p0].state = 2u;
    } else {
      const uint32_t c = *R.list_count;
      for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < c; i += gridDim.x * blockDim.x)
        L.sn[R.list_p[i]].state = 2u;
    }
  }
  if (!ctr->fdup[y]) {
    if (!ctr->fopt[y]) force_unique_body(tries, trie, lev, R, tmp_slot);  // (an optimistic insert did it)
    return;
  }
  const DevTrie& T = tries[trie];
  const DevLevel& L = T.lev[lev];
  const uint32_t total = force_total(R);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    uint32_t p, len, pos;
    force_locate(R, i, p, len, pos);
    const uint32_t h = tmp_slot[pos];
    const uint32_t dst = L.table[h].q + tmp_rank[pos];
    for (int c = 0; c < T.ncols; ++c) {
      int32_t* out = L.cval[c];
      if (out) out[dst] = level_src(T, lev, c)[pos];
    }
  }
}

// All keys distinct (no repeated key met by k_force_insert): every row is its
// own child group, so the grouping is the identity -- child start = the row's
// position, count 1, clustered columns copied in place. Replaces assign +
// scatter (a graph level of deduplicated edges always takes this path).
__device__ void force_unique_body(const DevTrie* __restrict__ tries, int trie, int lev, const ForceRange& R,
                                  const uint32_t* __restrict__ tmp_slot) {
  const DevTrie& T = tries[trie];
  const DevLevel& L = T.lev[lev];
  const uint32_t total = force_total(R);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    uint32_t p, len, pos;
    force_locate(R, i, p, len, pos);
    L.table[tmp_slot[pos]].q = pos;
    L.cnt[pos] = 1;
    if (pos == p) {
      L.sn[lev == 0 ? 0 : p].nkeys = len;
      L.cursor[lev == 0 ? 0 : p] = len;
    }
    for (int c = 0; c < T.ncols; ++c) {
      int32_t* out = L.cval[c];
      if (out) out[pos] = level_src(T, lev, c)[pos];
    }
  }
}



// ---------------------------------------------------------------------------
// Sort-based force of a root (the single subtrie [0, n) of level 0) with a
// key of arity <= 1: radix-sort (key, row), mark group starts, insert one slot
// per distinct key (no contention), gather the clustered columns. Produces the
// same structure as the atomic path without per-row atomics on hot keys.
// pay: the sort payload is this column's values (two-column relations: the
// sort then lays out both clustered columns, no gather), else the row ids
__global__ void k_root_keys(const DevTrie* __restrict__ tries, int trie, uint32_t n, uint32_t* __restrict__ keys,
                            uint32_t* __restrict__ rows, int pay) {
  const DevTrie& T = tries[trie];
  const DevLevel& L = T.lev[0];
  const int32_t* kc = L.nk ? T.base[L.keycol[0]] : nullptr;
  const int32_t* pc = pay >= 0 ? T.base[pay] : nullptr;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    keys[i] = kc ? (uint32_t)kc[i] : 0u;
    rows[i] = pc ? (uint32_t)pc[i] : i;
  }
}

__global__ void k_root_starts(const uint32_t* __restrict__ skeys, uint32_t n, uint8_t* __restrict__ flags) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    flags[i] = (i == 0 || skeys[i] != skeys[i - 1]) ? 1 : 0;
}

// clear the sorted root's G-bucket slot region and all n child counts
__global__ void k_root_clear(const DevTrie* __restrict__ tries, int trie, uint32_t n,
                             const uint32_t* __restrict__ ngroups, DevCounters* ctr) {
  const DevLevel& L = tries[trie].lev[0];
  const uint32_t G = max(*ngroups, 1u);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    L.cnt[i] = 0;
    if (i < G) {
      uint4* t = reinterpret_cast<uint4*>(L.table) + 2ull * FJG_RS * i;
#pragma unroll
      for (int u = 0; u < 2 * FJG_RS; ++u) t[u] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr->root_region[trie] = G;
}

// one thread per distinct key: its group is [starts[g], starts[g+1])
__global__ void k_root_insert(const DevTrie* __restrict__ tries, int trie, uint32_t n, const uint32_t* __restrict__ skeys,
                              const uint32_t* __restrict__ starts, const uint32_t* __restrict__ ngroups,
                              DevCounters* ctr) {
  const DevLevel& L = tries[trie].lev[0];
  const uint32_t G = *ngroups;
  bool sawdup = false;
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < G; g += gridDim.x * blockDim.x) {
    const uint32_t q = starts[g];
    const uint32_t c = (g + 1 < G ? starts[g + 1] : n) - q;
    const uint32_t kw = skeys[q];
    const uint32_t RG = max(G, 1u);  // region: one bucket per distinct key
    const uint64_t lo = 0, hi = 4ull * region_hi(0u, RG);
    uint64_t h = 4ull * region_bucket(0u, RG, kw);
    const unsigned long long mine = ((unsigned long long)q << 32) | kw;
    while (true) {
      unsigned long long* addr = reinterpret_cast<unsigned long long*>(L.table + h);
      if (atomicCAS(addr, kEmpty64, mine) == kEmpty64) break;
      if (++h == hi) h = lo;
    }
    L.cnt[q] = c;
    sawdup |= c > 1;
  }
  if (__any_sync(0xffffffffu, sawdup) && (threadIdx.x & 31) == 0) ctr->level_dup[trie * MAXL] = 1u;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    L.sn[0].nkeys = G;
    L.sn[0].state = 2u;
    ctr->newslots = G;
    atomicAdd((unsigned long long*)&ctr->keys_inserted, (unsigned long long)G);
  }
}

__global__ void k_root_gather(const DevTrie* __restrict__ tries, int trie, uint32_t n,
                              const uint32_t* __restrict__ srows) {
  const DevTrie& T = tries[trie];
  const DevLevel& L = T.lev[0];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t r = srows[i];
    for (int c = 0; c < T.ncols; ++c)
      if (L.cval[c]) L.cval[c][i] = T.base[c][r];
  }
}

// Eager (SIMPLE backend) level list: every key of a fully forced level l-1
// names a child subtrie (start q, length cnt[q]) to force at level l.
// (Same bookkeeping as a claim in k_select: the child's cursor / key count restart.)
__global__ void k_eager_list(const Slot* __restrict__ table, uint64_t nslots, const uint32_t* __restrict__ cnt,
                             DevLevel child, uint32_t* __restrict__ list_count,
                             const uint32_t* __restrict__ root_region) {
  uint32_t* __restrict__ list_p = child.list_p;
  uint32_t* __restrict__ list_len = child.list_len;
  if (root_region) nslots = 4ull * FJG_RS * *root_region;  // a root's live slots
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nslots; s += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t q = table[s].q;
    if (q == kEmpty) continue;
    child.cursor[q] = 0;
    child.sn[q].nkeys = 0;
    const uint32_t i = atomicAdd(list_count, 1u);
    list_p[i] = q;
    list_len[i] = cnt[q];
  }
}
