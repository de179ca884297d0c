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

// memo_out[g] = 0, or the group size when the pass has no fresh atom (every
// row of the group contributes 1)
__global__ void k_memo_init(const __grid_constant__ MemoPass M) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M.n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = __ldg(M.cnt + i);
    if (!c) continue;
    const uint64_t g = __ldg(M.gid + i) - 1u;
    M.memo_out[2 * g] = M.nfresh == 0 ? (unsigned long long)c : 0ull;
    M.memo_out[2 * g + 1] = 0ull;
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
      if (!colt_get(X, 0u, X.root_n, key, q, ql)) {
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

// one pass: memo_out[group(pos)] += coef(pos) * memo_next[child(pos)]; the
// rows of a group are contiguous, so lanes of one group add inside the warp
__global__ void __launch_bounds__(256) k_memo_gather(const __grid_constant__ MemoPass M) {
  const unsigned FULL = 0xffffffffu;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t iters = (M.n + stride - 1) / stride;
  for (uint64_t it = 0; it < iters; ++it) {
    const uint64_t pos = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x + it * stride;
    const bool ok = pos < M.n;
    uint32_t g = 0;
    unsigned __int128 f = 0;
    if (ok) {
      g = __ldg(M.gid + pos) - 1u;
      const uint64_t coef = M.has_coef ? __ldg(M.coef + pos) : 1ull;
      if (M.cont_x >= 0) {
        const uint32_t c = __ldg(M.child + pos);
        if (c != kMemoMiss && coef) {
          const ulonglong2 mv = __ldg(reinterpret_cast<const ulonglong2*>(M.memo_next) + c);
          f = (((unsigned __int128)mv.y << 64) | (unsigned __int128)mv.x) * coef;
        }
      } else {
        f = coef;
      }
    }
    const unsigned act = __ballot_sync(FULL, ok && f != 0);
    if (ok && f != 0) {
      const unsigned grp = __match_any_sync(act, g);
      const int lane = threadIdx.x & 31;
      const int leader = __ffs(grp) - 1;
      unsigned long long lo = (unsigned long long)f, hi = (unsigned long long)(f >> 64);
      unsigned long long slo = 0, shi = 0;
      unsigned m = grp;
      while (m) {
        const int l = __ffs(m) - 1;
        m &= m - 1;
        const unsigned long long a = __shfl_sync(grp, lo, l), b = __shfl_sync(grp, hi, l);
        const unsigned long long s2 = slo + a;
        shi += b + (s2 < slo ? 1ull : 0ull);
        slo = s2;
      }
      if (lane == leader) atomic_add_u128(M.memo_out + 2ull * g, ((unsigned __int128)shi << 64) | slo);
    }
  }
}

struct MaxOp {
  __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};

