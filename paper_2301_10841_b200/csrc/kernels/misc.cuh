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

__global__ void k_partition_flags(const int32_t* col, uint64_t n, int nparts, int part, uint32_t* flags) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    flags[i] = fj::partition_of(col[i], (uint32_t)nparts) == (uint32_t)part ? 1u : 0u;
}

