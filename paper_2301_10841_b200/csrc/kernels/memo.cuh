// memo: memoised chain count (count_factorized extension)
// Included by engine.cu (one translation unit: the kernels share templates and helpers).
#pragma once

__device__ __forceinline__ void atomic_add_u128(unsigned long long* m, unsigned __int128 v) {
  const unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
  const unsigned long long old = atomicAdd(m, lo);
  const unsigned long long carry = (old + lo < old) ? 1ull : 0ull;
  if (hi + carry) atomicAdd(m + 1, hi + carry);
}

// group index of every level-0 position, step 1: 1 at group starts (the
// inclusive sum then numbers groups 1..G)
__global__ void k_start_flags(const uint32_t* __restrict__ cnt, uint64_t n, uint32_t* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = cnt[i] ? 1u : 0u;
}

// every memo array over one trie's groups: 0, or the group size for a pass
// without fresh atoms (every row counts 1); plus the dense key -> group map
__global__ void k_memo_init(const __grid_constant__ MemoInit I) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < I.n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = __ldg(I.cnt + i);
    if (!c) continue;
    const uint64_t g = __ldg(I.gid + i) - 1u;
#pragma unroll
    for (int k = 0; k < kMemoInitMax; ++k)
      if (k < I.nout) {
        I.out[k][2 * g] = I.group_size[k] ? (unsigned long long)c : 0ull;
        I.out[k][2 * g + 1] = 0ull;
      }
    if (I.dense) {
      const uint32_t key = (uint32_t)__ldg(I.key + i);
      if (key < I.dense_n) I.dense[key] = (uint32_t)g;
    }
  }
}

// per row: probe the fresh atoms' roots once; child gid of the continuing one,
// product of the leaf lengths of the others
__global__ void __launch_bounds__(256) k_memo_resolve(const __grid_constant__ MemoPass M) {
  for (uint64_t pos = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < M.n;
       pos += (uint64_t)gridDim.x * blockDim.x) {
    int32_t t[MAXK];
#pragma unroll
    for (int k = 0; k < MAXK; ++k) t[k] = k < M.cnv ? __ldg(M.cvals[k] + pos) : 0;
    if (M.direct) {  // single continuing fresh atom over a dense sorted root: one read
      const uint32_t key = (uint32_t)t[M.cpos[0][0]];
      M.child[pos] = key < M.direct_n ? __ldg(M.direct + key) : kMemoMiss;
      continue;
    }
    uint32_t child = kMemoMiss;
    uint64_t coef = 1;
    for (int x = 0; x < M.nfresh; ++x) {
      const KSub& X = M.fresh[x];
      int32_t key[MAXK];
#pragma unroll
      for (int k = 0; k < MAXK; ++k) {
        int32_t v = 0;
#pragma unroll
        for (int u = 0; u < MAXK; ++u) v |= t[u] & -(int32_t)(u == M.cpos[x][k]);
        key[k] = k < X.nv ? v : 0;
      }
      uint32_t q, ql;
      const bool hit = x == M.cont_x ? colt_get<false>(X, 0u, X.root_n, key, q, ql)
                                     : colt_get<true>(X, 0u, X.root_n, key, q, ql);
      if (!hit) {
        coef = 0;
        child = kMemoMiss;
        break;
      }
      if (x == M.cont_x)
        child = __ldg(M.gid_next + q) - 1u;
      else
        coef *= ql;
    }
    if (M.cont_x >= 0) M.child[pos] = coef ? child : kMemoMiss;
    if (M.has_coef) M.coef[pos] = coef;
  }
}

// u128 helpers for the warp-segmented sums below
__device__ __forceinline__ void add128(unsigned long long& lo, unsigned long long& hi, unsigned long long blo,
                                       unsigned long long bhi) {
  const unsigned long long s = lo + blo;
  hi += bhi + (s < lo ? 1ull : 0ull);
  lo = s;
}

// one pass: memo_out[group(pos)] += coef(pos) * memo_next[child(pos)]. The rows
// of a group are contiguous: a warp forms segmented sums over its 32 rows
// (head flags by ballot, 5 shuffle steps) and the last lane of each segment
// adds it to the group with one u128 atomic.
__global__ void __launch_bounds__(256) k_memo_gather(const __grid_constant__ MemoPass M) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t iters = (M.n + stride - 1) / stride;
  for (uint64_t it = 0; it < iters; ++it) {
    const uint64_t pos = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x + it * stride;
    const bool ok = pos < M.n;
    uint32_t g = 0xffffffffu;
    unsigned long long lo = 0, hi = 0;
    if (ok) {
      g = __ldg(M.gid + pos) - 1u;
      const uint64_t coef = M.has_coef ? __ldg(M.coef + pos) : 1ull;
      if (M.cont_x >= 0) {
        const uint32_t c = __ldg(M.child + pos);
        if (c != kMemoMiss && coef) {
          const ulonglong2 mv = __ldg(reinterpret_cast<const ulonglong2*>(M.memo_next) + c);
          const unsigned __int128 f = (((unsigned __int128)mv.y << 64) | (unsigned __int128)mv.x) * coef;
          lo = (unsigned long long)f;
          hi = (unsigned long long)(f >> 64);
        }
      } else {
        lo = coef;
      }
    }
    const uint32_t gprev = __shfl_up_sync(FULL, g, 1);
    const unsigned heads = __ballot_sync(FULL, lane == 0 || g != gprev);
    const int seg = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));  // first lane of this lane's segment
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long ol = __shfl_up_sync(FULL, lo, d), oh = __shfl_up_sync(FULL, hi, d);
      if (lane - d >= seg) add128(lo, hi, ol, oh);
    }
    const uint32_t gnext = __shfl_down_sync(FULL, g, 1);
    const bool tail = lane == 31 || gnext != g;
    if (ok && tail && (lo | hi)) atomic_add_u128(M.memo_out + 2ull * g, ((unsigned __int128)hi << 64) | lo);
  }
}

// Top of the chain when node 0 streams the rows of the pass-0 carrier's
// relation and probes the root pass 0 resolved against (C5 5-path: E1 over E,
// probing the shared E root): its count is sum over those rows of
// memo_0[child(row)], read from pass 0's resolved children.
__global__ void __launch_bounds__(256) k_memo_total(const uint32_t* __restrict__ child, uint64_t n,
                                                    const unsigned long long* __restrict__ memo, int node,
                                                    DevCounters* ctr) {
  unsigned long long lo = 0, hi = 0;
  uint64_t rows = 0, misses = 0;
  for (uint64_t pos = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < n;
       pos += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = __ldg(child + pos);
    ++rows;
    if (c == kMemoMiss) {
      ++misses;
      continue;
    }
    const ulonglong2 mv = __ldg(reinterpret_cast<const ulonglong2*>(memo) + c);
    add128(lo, hi, mv.x, mv.y);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long ol = __shfl_xor_sync(0xffffffffu, lo, o), oh = __shfl_xor_sync(0xffffffffu, hi, o);
    add128(lo, hi, ol, oh);
  }
  rows = warp_sum(rows);
  misses = warp_sum(misses);
  if ((threadIdx.x & 31) == 0) {
    if (lo | hi) {
      const unsigned long long old = atomicAdd((unsigned long long*)&ctr->count_lo, lo);
      if (old + lo < old) ++hi;
      if (hi) atomicAdd((unsigned long long*)&ctr->count_hi, hi);
    }
    if (rows) {  // node 0's ExecStats: every row iterated and probed once
      atomicAdd((unsigned long long*)&ctr->body[node], (unsigned long long)rows);
      atomicAdd((unsigned long long*)&ctr->node_probes[node], (unsigned long long)rows);
      atomicAdd((unsigned long long*)&ctr->probes, (unsigned long long)rows);
    }
    if (misses) atomicAdd((unsigned long long*)&ctr->misses, (unsigned long long)misses);
  }
}


