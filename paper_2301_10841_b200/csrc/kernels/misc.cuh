// misc: tuple hash, filter, partition kernels
// Included by engine.cu (one translation unit: the kernels share templates and helpers).
#pragma once

// ============================================================================
// misc kernels
// ============================================================================
__global__ void k_tuple_hash(const int64_t* vals, int arity, uint64_t n, uint64_t* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t h = fj::kTupleHashSeed;
    for (int t = 0; t < arity; ++t) h = fj::tuple_hash_step(h, vals[i * arity + t]);
    out[i] = h;
  }
}

__device__ __forceinline__ bool cmp_eval(int cmp, int64_t a, int64_t b) {
  switch (cmp) {
    case FJG_CMP_EQ: return a == b;
    case FJG_CMP_NE: return a != b;
    case FJG_CMP_LT: return a < b;
    case FJG_CMP_LE: return a <= b;
    case FJG_CMP_GT: return a > b;
    default: return a >= b;
  }
}

struct DevPreds {
  int n;
  fjg_predicate p[8];
  const int32_t* cols[MAXC];
};

__global__ void k_filter_flags(DevPreds P, uint64_t n, uint32_t* flags) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    bool ok = true;
    for (int k = 0; k < P.n; ++k) {
      const int64_t a = P.cols[P.p[k].column][i];
      const int64_t b = P.p[k].is_column ? (int64_t)P.cols[P.p[k].rhs_column][i] : P.p[k].constant;
      ok = ok && cmp_eval(P.p[k].cmp, a, b);
    }
    flags[i] = ok ? 1u : 0u;
  }
}

__global__ void k_compact_col(const int32_t* in, const uint32_t* flags, const uint32_t* excl, uint64_t n, int32_t* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    if (flags[i]) out[excl[i]] = in[i];
}

// int64 column ingestion (fj::Value is int64, value.hpp:31): narrows a staged
// chunk of int64 values to the engine's int32 column, four values per thread
// (two 128-bit loads, one 128-bit store). A value outside int32 records the
// lowest offending row in *bad_row (UINT64_MAX = none); its slot is left 0.
__global__ void k_narrow_i64(const long long* __restrict__ in, uint64_t n, uint64_t row0, int32_t* __restrict__ out,
                             unsigned long long* bad_row) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t nq = n >> 2;
  unsigned long long bad = ~0ull;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += stride) {
    const longlong2 a = __ldg(reinterpret_cast<const longlong2*>(in) + 2 * q);
    const longlong2 b = __ldg(reinterpret_cast<const longlong2*>(in) + 2 * q + 1);
    const long long v[4] = {a.x, a.y, b.x, b.y};
    int4 o;
    int32_t* op = &o.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool fits = v[j] == (long long)(int32_t)v[j];
      op[j] = fits ? (int32_t)v[j] : 0;
      if (!fits) bad = min(bad, (unsigned long long)(row0 + 4 * q + j));
    }
    reinterpret_cast<int4*>(out)[q] = o;
  }
  for (uint64_t i = (nq << 2) + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const long long v = in[i];
    const bool fits = v == (long long)(int32_t)v;
    out[i] = fits ? (int32_t)v : 0;
    if (!fits) bad = min(bad, (unsigned long long)(row0 + i));
  }
  if (bad != ~0ull) atomicMin(bad_row, bad);
}

// Stable hash partition (multi-GPU sharding on the first plan variable):
// counting sort by destination. Block b owns rows [b*kPartChunk, ...); hist is
// destination-major (d * nblocks + b) so its exclusive scan gives every
// (destination, block) its output base.
constexpr uint32_t kPartChunk = 2048;  // 8 rounds of 256 rows: more resident blocks hide the per-round latency
constexpr int PART_WARPS = 8;

struct DevPartCols {
  int ncols;
  const int32_t* in[MAXC];
  int32_t* out[MAXC];
};

__global__ void k_part_count(const int32_t* __restrict__ key, uint64_t n, int nparts, uint32_t nblocks,
                             uint32_t* __restrict__ hist) {
  extern __shared__ uint32_t s_cnt[];
  for (int d = threadIdx.x; d < nparts; d += blockDim.x) s_cnt[d] = 0;
  __syncthreads();
  const uint64_t lo = (uint64_t)blockIdx.x * kPartChunk, hi = min(n, lo + kPartChunk);
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x)
    atomicAdd(&s_cnt[fj::partition_of(key[i], (uint32_t)nparts)], 1u);
  __syncthreads();
  for (int d = threadIdx.x; d < nparts; d += blockDim.x) hist[(uint64_t)d * nblocks + blockIdx.x] = s_cnt[d];
}

__global__ void k_part_scatter(DevPartCols pc, int col, uint64_t n, int nparts, uint32_t nblocks,
                               const uint32_t* __restrict__ offs) {
  extern __shared__ uint32_t s_mem[];
  uint32_t* s_run = s_mem;               // [nparts] rows already placed per destination
  uint32_t* s_wc = s_mem + nparts;       // [PART_WARPS][nparts] per-warp counts of this round
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < nparts; d += blockDim.x) s_run[d] = 0;
  const uint64_t lo = (uint64_t)blockIdx.x * kPartChunk, hi = min(n, lo + kPartChunk);
  for (uint64_t r0 = lo; r0 < hi; r0 += blockDim.x) {
    for (int t = threadIdx.x; t < PART_WARPS * nparts; t += blockDim.x) s_wc[t] = 0;
    __syncthreads();
    const uint64_t i = r0 + threadIdx.x;
    const bool ok = i < hi;
    const uint32_t d = ok ? fj::partition_of(pc.in[col][i], (uint32_t)nparts) : 0u;
    const unsigned act = __ballot_sync(0xffffffffu, ok);
    unsigned grp = 0;
    if (ok) {
      grp = __match_any_sync(act, d);
      if (lane == __ffs(grp) - 1) s_wc[warp * nparts + d] = __popc(grp);
    }
    __syncthreads();
    if (ok) {
      uint32_t before = s_run[d];
      for (int w = 0; w < warp; ++w) before += s_wc[w * nparts + d];
      const uint64_t o = (uint64_t)offs[(uint64_t)d * nblocks + blockIdx.x] + before +
                         __popc(grp & ((1u << lane) - 1));
      for (int c = 0; c < pc.ncols; ++c) pc.out[c][o] = pc.in[c][i];
    }
    __syncthreads();
    for (int dd = threadIdx.x; dd < nparts; dd += blockDim.x) {
      uint32_t add = 0;
      for (int w = 0; w < PART_WARPS; ++w) add += s_wc[w * nparts + dd];
      s_run[dd] += add;
    }
    __syncthreads();
  }
}

// tot[d] = base of destination d (tot[nparts] = n)
__global__ void k_part_totals(const uint32_t* __restrict__ offs, int nparts, uint32_t nblocks, uint32_t* tot) {
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d <= nparts; d += gridDim.x * blockDim.x)
    tot[d] = offs[(uint64_t)d * nblocks];
}


// row-major tuples (enumerate output) -> columnar relation
__global__ void k_transpose_rows(const int32_t* __restrict__ rows, uint64_t n, DevPartCols pc) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    for (int c = 0; c < pc.ncols; ++c) pc.out[c][i] = rows[i * pc.ncols + c];
}
