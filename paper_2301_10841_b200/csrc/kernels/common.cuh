// common: device helpers: hashing, COLT get, estimated_key_count
// Included by engine.cu (one translation unit: the kernels share templates and helpers).
#pragma once

// ============================================================================
// device helpers
// ============================================================================
__device__ __forceinline__ const int32_t* level_src(const DevTrie& T, int depth, int col) {
  return depth == 0 ? T.base[col] : T.lev[depth - 1].cval[col];
}

template <int N>
__device__ __forceinline__ uint32_t key_word_r(int nk, const int32_t (&vals)[N]) {
  if (nk == 0) return 0u;
  if (nk == 1) return static_cast<uint32_t>(vals[0]);
  uint64_t h = fj::kTupleHashSeed;
#pragma unroll
  for (int t = 0; t < N; ++t)
    if (t < nk) h = fj::tuple_hash_step(h, vals[t]);
  return static_cast<uint32_t>(fj::fmix64(h));
}

// first bucket (4 slots) of key word kw inside the region of subtrie (p, len)
__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  h ^= h >> 16;
  return h;
}
// Subtrie regions: the subtrie at positions [p, p+len) owns buckets
// [FJG_RS*p, FJG_RS*(p+len)) of its level's table (4 slots = 32 B each), so
// regions of different subtries never overlap. FJG_RS = 2 halves the load
// (0.125 per slot): a missed probe then rarely finds its home bucket full.
#ifndef FJG_RS
#define FJG_RS 1
#endif
// FJG_CHECK=1 (scripts/build_variant.py ... -DFJG_CHECK=1): device-side
// invariant checks at the probe, force and output sites; a violation traps
// (the launch fails with an illegal-instruction error naming the kernel).
// compute-sanitizer is not available on this pool (profiles/r02_checked_build.md).
#ifndef FJG_CHECK
#define FJG_CHECK 0
#endif
#if FJG_CHECK
#define FJG_ASSERT(c)                                                                 \
  do {                                                                                \
    if (!(c)) {                                                                       \
      printf("FJG_CHECK failed: %s (%s:%d) block %d thread %d\n", #c, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                      \
      __trap();                                                                       \
    }                                                                                 \
  } while (0)
#else
#define FJG_ASSERT(c) ((void)0)
#endif
__device__ __forceinline__ uint64_t region_lo(uint32_t p) { return (uint64_t)p * FJG_RS; }
__device__ __forceinline__ uint64_t region_hi(uint32_t p, uint32_t len) { return ((uint64_t)p + len) * FJG_RS; }
#ifndef FJG_HASH_MUL
#define FJG_HASH_MUL 1  // multiplicative (Fibonacci) bucket hash (C5 last node 924 -> 907 ms, C4 82 -> 77 ms); 0: fmix32
#endif
__device__ __forceinline__ uint64_t region_bucket(uint32_t p, uint32_t len, uint32_t kw) {
#if FJG_HASH_MUL
  const uint32_t h = kw * 0x9e3779b1u;  // the high bits pick the bucket (mul.hi with len)
#else
  const uint32_t h = fmix32(kw ^ 0x9e3779b9u);
#endif
  return region_lo(p) + (((uint64_t)h * ((uint64_t)len * FJG_RS)) >> 32);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Probe region (buckets) of a subtrie: its length, except for a root, whose
// region is set by its force (rows, or distinct keys when force-sorted).
__device__ __forceinline__ uint32_t probe_region(const KSub& S, uint32_t len) {
  return S.in_p ? len : *S.rregion;
}

// COLT get (Fig 12 `get` = force, then lookup): the subtrie was forced by an
// earlier kernel of this node, so this is a pure lookup in its slot region:
// read a bucket (one sector, as two 16-byte halves), stop at a match or at the
// first free slot.
template <bool WANT_LEN = true>
__device__ __forceinline__ bool colt_get(const KSub& P, uint32_t p, uint32_t len, const int32_t (&key)[MAXK],
                                         uint32_t& q, uint32_t& ql) {
  const int nk = P.nv;
  const uint32_t kw = key_word_r(nk, key);
  len = probe_region(P, len);
  FJG_ASSERT(len > 0 && (uint64_t)p + len <= (P.in_p ? (uint64_t)P.root_n : (uint64_t)P.root_n + 1));
  uint64_t b = region_bucket(p, len, kw);
  const uint64_t blo = region_lo(p), bhi = region_hi(p, len);
  const uint4* __restrict__ tb = reinterpret_cast<const uint4*>(P.table);
  while (true) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const uint4 s = __ldg(tb + 2 * b + half);
      // slot (s.x, s.y) then (s.z, s.w)
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        const uint32_t sk = w ? s.z : s.x, sq = w ? s.w : s.y;
        if (sq == kEmpty) return false;
        if (sk == kw) {
          bool eq = true;
          if (nk >= 2) {
#pragma unroll
            for (int t = 0; t < MAXK; ++t)
              if (t < nk && __ldg(P.kcmp[t] + sq) != key[t]) eq = false;
          }
          if (eq) {
            q = sq;
            ql = WANT_LEN ? __ldg(P.cnt + sq) : 0u;  // the child length costs a random read
            return true;
          }
        }
      }
    }
    if (++b == bhi) b = blo;
  }
}

__device__ __forceinline__ void subtrie_of(const KSub& S, uint64_t e, uint32_t& p, uint32_t& len) {
  if (S.in_p) {
    p = __ldg(S.in_p + e);
    len = __ldg(S.in_len + e);
  } else {
    p = 0;
    len = S.root_n;
  }
}

// {state, key count} of a subtrie in one 8-byte load (not cached in L1: claims
// and forces of earlier kernels of this stream must be seen)
__device__ __forceinline__ uint2 ld_substate(const SubState* p) {
  uint2 v;
  asm volatile("ld.volatile.global.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}

// estimated_key_count: forced map -> #keys, vector -> its
// length, BaseScan -> cardinality. Never forces.
__device__ __forceinline__ uint64_t estimate(const KSub& S, uint32_t p, uint32_t len) {
  if (p == kSingleton) return 1;
  const uint32_t id = S.depth == 0 ? 0u : p;
  const uint2 sn = ld_substate(S.sn + id);  // state and key count: one 8-byte load
  if (sn.x == 2u) return sn.y;
  return len;
}

