// memo: memoised chain count (count_factorized extension)
// Included by engine.cu (one translation unit: the kernels share templates and helpers).
#pragma once

__device__ __forceinline__ void atomic_add_u128(unsigned long long* m, unsigned __int128 v) {
  const unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
  const unsigned long long old = atomicAdd(m, lo);
  const unsigned long long carry = (old + lo < old) ? 1ull : 0ull;
  if (hi + carry) atomicAdd(m + 1, hi + carry);
}

__global__ void __launch_bounds__(256) k_memo_pass(const __grid_constant__ MemoPass M) {
  const unsigned FULL = 0xffffffffu;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t iters = (M.n + stride - 1) / stride;
  for (uint64_t it = 0; it < iters; ++it) {
    const uint64_t pos = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x + it * stride;
    const bool ok = pos < M.n;
    uint32_t g = 0;
    unsigned __int128 f = 0;
    if (ok) {
      g = M.owner[pos];
      int32_t t[MAXK];
#pragma unroll
      for (int k = 0; k < MAXK; ++k) t[k] = k < M.cnv ? __ldg(M.cvals[k] + pos) : 0;
      f = 1;
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
          f = 0;
          break;
        }
        if (M.cont[x])
          f *= ((unsigned __int128)M.memo_next[2ull * q + 1] << 64) | (unsigned __int128)M.memo_next[2ull * q];
        else
          f *= ql;
      }
    }
    // positions of one group are contiguous: aggregate per group inside the warp
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
__global__ void k_group_starts(const uint32_t* cnt, uint64_t n, uint32_t* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = cnt[i] ? (uint32_t)i : 0u;
}

