// prims: the device-wide primitives of the build and frontier path, hand-written
// for sm_100a (no library kernels on the hot path):
//   * single-pass prefix scans (sum / max, inclusive / exclusive) and flagged
//     selection, each tile finding its prefix by decoupled look-back over its
//     predecessors' published aggregates (one read and one write per element);
//   * a stable LSD radix sort of (u32 key, u32 value) pairs: one histogram
//     kernel for every pass, then per pass one kernel that ranks a tile of 8192
//     keys in shared memory (warp match_any multi-split), finds each digit's
//     global offset by decoupled look-back and writes the tile digit-sorted
//     from shared memory (coalesced runs) -- one read and one write of the pairs
//     per pass, 9-bit digits (27-bit vertex keys sort in 3 passes);
//   * a max reduction (the key bits a sorted root sorts on).
// Tiles are numbered by a ticket counter (never reset: the host keeps the
// running base), so a tile's predecessors are always resident or done; look-back
// words carry a 30-bit epoch so no per-call reset is needed.
// Included by engine.cu (one translation unit).
#pragma once

namespace prims {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned lane_lt_mask() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

struct OpSum {
  template <class T>
  __device__ __forceinline__ T operator()(T a, T b) const { return a + b; }
};
struct OpMax {
  template <class T>
  __device__ __forceinline__ T operator()(T a, T b) const { return a > b ? a : b; }
};

template <class T, class Op>
__device__ __forceinline__ T warp_incl_scan(T v, Op op) {
  const unsigned lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T u = __shfl_up_sync(kFull, v, o);
    if (lane >= (unsigned)o) v = op(u, v);
  }
  return v;
}

template <class T, class Op>
__device__ __forceinline__ T warp_reduce(T v, Op op) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// Exclusive block scan (identity `id`); `total` = the block's reduction.
// `sm` holds NT/32 values; the call ends with a barrier so `sm` is reusable.
template <int NT, class T, class Op>
__device__ __forceinline__ T block_excl_scan(T v, T& total, T* sm, Op op, T id) {
  constexpr int NW = NT / 32;
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T inc = warp_incl_scan(v, op);
  if (lane == 31) sm[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < (unsigned)NW ? sm[lane] : id;
    w = warp_incl_scan(w, op);
    if (lane < (unsigned)NW) sm[lane] = w;
  }
  __syncthreads();
  T ex = __shfl_up_sync(kFull, inc, 1);
  if (lane == 0) ex = id;
  const T r = warp ? op(sm[warp - 1], ex) : ex;
  total = sm[NW - 1];
  __syncthreads();
  return r;
}

template <int NT, class T>
__device__ __forceinline__ T block_sum(T v, T* sm) {
  T total;
  block_excl_scan<NT>(v, total, sm, OpSum(), T(0));
  return total;
}

// ---------------------------------------------------------------------------
// decoupled look-back (scans): one 16-byte descriptor per tile. Each 64-bit
// half carries the tag (epoch << 2 | status: 1 = the tile's aggregate, 2 = its
// inclusive prefix) in its high word and one 32-bit half of the value in its
// low word, so a descriptor is published with one 128-bit store and read with
// one 128-bit load -- no fence, no dependent second load. A reader accepts a
// descriptor only when both halves carry the same tag of this epoch (a half is
// written once per status, so equal tags mean both halves belong to one write).
// ---------------------------------------------------------------------------
struct __align__(16) LBTile {
  unsigned long long a, b;
};

__device__ __forceinline__ void lb_publish(LBTile* t, bool inclusive, unsigned long long v, uint32_t epoch) {
  const unsigned long long tag = (unsigned long long)((epoch << 2) | (inclusive ? 2u : 1u)) << 32;
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};\n" ::"l"(t), "l"(tag | (v & 0xffffffffull)),
               "l"(tag | (v >> 32))
               : "memory");
}

// Warp 0 of tile `tile` (> 0): the exclusive prefix over tiles [0, tile).
template <class T, class Op>
__device__ T lb_lookback(LBTile* st, uint64_t tile, uint32_t epoch, Op op, T id) {
  const unsigned lane = threadIdx.x & 31;
  T prefix = id;
  int64_t t = (int64_t)tile - 1;
  while (true) {
    const int64_t tt = t - (int64_t)lane;
    unsigned status = 2;
    T v = id;
    if (tt >= 0) {
      unsigned long long a, b;
      do {
        asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(a), "=l"(b) : "l"(st + tt) : "memory");
      } while ((uint32_t)(a >> 34) != epoch || (a >> 32) != (b >> 32));
      status = (unsigned)(a >> 32) & 3u;
      v = (T)((a & 0xffffffffull) | (b << 32));
    }
    const unsigned pm = __ballot_sync(kFull, status == 2u);
    // lanes up to (and including) the nearest inclusive prefix contribute
    const int first = pm ? __ffs(pm) - 1 : 31;
    if ((int)lane > first) v = id;
    prefix = op(prefix, warp_reduce(v, op));  // (a tile's window runs back in tile order: op is commutative here)
    if (pm) break;
    t -= 32;
  }
  return prefix;
}

// Single-pass scan: out[i] = op(in[0..i]) (EXCL: op(in[0..i-1]), identity first).
// In may alias out. `total` (optional) receives the reduction of all n.
#ifndef FJG_SCAN_ITEMS
#define FJG_SCAN_ITEMS 8
#endif
constexpr int kScanThreads = 256, kScanItems = FJG_SCAN_ITEMS, kScanTile = kScanThreads * kScanItems;
template <class In, class T, class Op, bool EXCL>
__global__ void __launch_bounds__(kScanThreads) k_scan_lb(const In* in, T* out, uint64_t n, LBTile* st,
                                                          unsigned long long* ticket, uint64_t tbase,
                                                          uint32_t epoch, T* total) {
  __shared__ T s_v[kScanTile];
  __shared__ T s_red[kScanThreads / 32];
  __shared__ uint64_t s_tile;
  __shared__ T s_prefix;
  Op op;
  const T id = T(0);
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1ull) - tbase;
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t base = tile * kScanTile;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t idx = base + i * kScanThreads + threadIdx.x;
    s_v[i * kScanThreads + threadIdx.x] = idx < n ? (T)in[idx] : id;
  }
  __syncthreads();
  T v[kScanItems];
  T acc = id;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = s_v[threadIdx.x * kScanItems + i];
    acc = op(acc, v[i]);
  }
  T tot;
  const T ex = block_excl_scan<kScanThreads>(acc, tot, s_red, op, id);
  if (threadIdx.x < 32) {
    T prefix = id;
    if (tile == 0) {
      if (threadIdx.x == 0) lb_publish(st, true, (unsigned long long)tot, epoch);
    } else {
      if (threadIdx.x == 0) lb_publish(st + tile, false, (unsigned long long)tot, epoch);
      prefix = lb_lookback<T>(st, tile, epoch, op, id);
      if (threadIdx.x == 0) lb_publish(st + tile, true, (unsigned long long)op(prefix, tot), epoch);
    }
    if (threadIdx.x == 0) s_prefix = prefix;
  }
  __syncthreads();
  T r = op(s_prefix, ex);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const T before = r;
    r = op(r, v[i]);
    s_v[threadIdx.x * kScanItems + i] = EXCL ? before : r;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t idx = base + i * kScanThreads + threadIdx.x;
    if (idx < n) out[idx] = s_v[i * kScanThreads + threadIdx.x];
  }
  if (total && threadIdx.x == 0 && base + kScanTile >= n) *total = op(s_prefix, tot);
}

// Flagged selection of indices: out[j] = the j-th i (in order) with flags[i] != 0;
// *count = the number selected. 16 flags per thread, one 16-byte load.
constexpr int kSelItems = 16, kSelTile = kScanThreads * kSelItems;
__global__ void __launch_bounds__(kScanThreads) k_select_flagged(const uint8_t* __restrict__ flags,
                                                                 uint32_t* __restrict__ out, uint64_t n,
                                                                 LBTile* st, unsigned long long* ticket,
                                                                 uint64_t tbase, uint32_t epoch, uint32_t* count) {
  __shared__ uint32_t s_red[kScanThreads / 32];
  __shared__ uint64_t s_tile;
  __shared__ uint32_t s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1ull) - tbase;
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t b = tile * kSelTile + (uint64_t)threadIdx.x * kSelItems;
  uint8_t f[kSelItems];
  if (b + kSelItems <= n) {
    const uint4 w = *reinterpret_cast<const uint4*>(flags + b);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int i = 0; i < kSelItems; ++i) f[i] = (uint8_t)(ws[i >> 2] >> (8 * (i & 3)));
  } else {
#pragma unroll
    for (int i = 0; i < kSelItems; ++i) f[i] = (b + i < n) ? flags[b + i] : 0;
  }
  uint32_t c = 0;
#pragma unroll
  for (int i = 0; i < kSelItems; ++i) c += f[i] ? 1u : 0u;
  uint32_t tot;
  const uint32_t ex = block_excl_scan<kScanThreads>(c, tot, s_red, OpSum(), 0u);
  if (threadIdx.x < 32) {
    uint32_t prefix = 0;
    if (tile == 0) {
      if (threadIdx.x == 0) lb_publish(st, true, tot, epoch);
    } else {
      if (threadIdx.x == 0) lb_publish(st + tile, false, tot, epoch);
      prefix = lb_lookback<uint32_t>(st, tile, epoch, OpSum(), 0u);
      if (threadIdx.x == 0) lb_publish(st + tile, true, prefix + tot, epoch);
    }
    if (threadIdx.x == 0) s_prefix = prefix;
  }
  __syncthreads();
  uint32_t pos = s_prefix + ex;
#pragma unroll
  for (int i = 0; i < kSelItems; ++i)
    if (f[i]) out[pos++] = (uint32_t)(b + i);
  if (threadIdx.x == 0 && tile * kSelTile + kSelTile >= n) *count = s_prefix + tot;
}

// max over n u32 values into *out (which the caller zeroed)
__global__ void k_reduce_max_u32(const uint32_t* __restrict__ in, uint64_t n, uint32_t* out) {
  __shared__ uint32_t s_red[8];
  uint32_t m = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    m = max(m, in[i]);
  uint32_t tot;
  block_excl_scan<256>(m, tot, s_red, OpMax(), 0u);
  if (threadIdx.x == 0 && tot) atomicMax(out, tot);
}

// ---------------------------------------------------------------------------
// radix sort of (u32 key, u32 value) pairs
// ---------------------------------------------------------------------------
#ifndef FJG_RADIX_ITEMS
#define FJG_RADIX_ITEMS 16
#endif
#ifndef FJG_RADIX_MINB
#define FJG_RADIX_MINB 2
#endif
constexpr int kRadixThreads = 512, kRadixItems = FJG_RADIX_ITEMS, kRadixTile = kRadixThreads * kRadixItems;
constexpr int kRadixBins = 512, kRadixMaxPasses = 4, kRadixWarps = kRadixThreads / 32;
constexpr size_t kRadixSmem = (size_t)kRadixTile * 8 + (size_t)kRadixWarps * kRadixBins * 2 + kRadixBins * 8 + 64;

// histograms of every pass's digit in one read of the keys (hist zeroed by the
// caller); pass p sorts bits [lo + p*dbits, min(lo + (p+1)*dbits, hi))
__device__ __forceinline__ uint32_t radix_digit(uint32_t k, int shift, int bits) {
  return (k >> shift) & ((1u << bits) - 1u);
}
__global__ void __launch_bounds__(256) k_radix_hist(const uint32_t* __restrict__ keys, uint64_t n, int lo,
                                                    int dbits, int npass, int hi, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[kRadixMaxPasses * kRadixBins];
  for (int i = threadIdx.x; i < npass * kRadixBins; i += blockDim.x) h[i] = 0;
  __syncthreads();
  int sh[kRadixMaxPasses], nb[kRadixMaxPasses];
#pragma unroll
  for (int p = 0; p < kRadixMaxPasses; ++p) {
    sh[p] = lo + p * dbits;
    nb[p] = p < npass ? min(dbits, hi - sh[p]) : 0;
  }
  const uint64_t n4 = n / 4;
  const uint4* k4 = reinterpret_cast<const uint4*>(keys);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 w = k4[i];
    const uint32_t ks[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int p = 0; p < kRadixMaxPasses; ++p)
        if (p < npass) atomicAdd(&h[p * kRadixBins + radix_digit(ks[j], sh[p], nb[p])], 1u);
  }
  for (uint64_t i = n4 * 4 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
#pragma unroll
    for (int p = 0; p < kRadixMaxPasses; ++p)
      if (p < npass) atomicAdd(&h[p * kRadixBins + radix_digit(keys[i], sh[p], nb[p])], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < npass * kRadixBins; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// One pass: digit = (key >> shift) & (2^dbits - 1), dbits <= 9; stable.
// Look-back word per (tile, digit): epoch << 34 | flag << 32 | count.
__global__ void __launch_bounds__(kRadixThreads, FJG_RADIX_MINB) k_radix_pass(const uint32_t* __restrict__ kin,
                                                                 const uint32_t* __restrict__ vin,
                                                                 uint32_t* __restrict__ kout,
                                                                 uint32_t* __restrict__ vout, uint64_t n, int shift,
                                                                 int dbits, const uint32_t* __restrict__ hist,
                                                                 unsigned long long* st, unsigned long long* ticket,
                                                                 uint64_t tbase, uint32_t epoch) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* sk = reinterpret_cast<uint32_t*>(smem);
  uint32_t* sv = sk + kRadixTile;
  uint16_t* wc = reinterpret_cast<uint16_t*>(sv + kRadixTile);  // [warp][digit]
  uint32_t* lstart = reinterpret_cast<uint32_t*>(wc + kRadixWarps * kRadixBins);
  uint32_t* gbase = lstart + kRadixBins;
  uint32_t* s_red = gbase + kRadixBins;  // 16 words
  __shared__ uint64_t s_tile;
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
  if (tid == 0) s_tile = atomicAdd(ticket, 1ull) - tbase;
  for (int i = lane; i < kRadixBins; i += 32) wc[warp * kRadixBins + i] = 0;
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t base = tile * kRadixTile;
  const uint32_t mask = (1u << dbits) - 1u;
  // warp-striped: warp w holds items base + w*512 + i*32 + lane (input order = (w, i, lane))
  uint32_t k[kRadixItems], v[kRadixItems];
  uint16_t rk[kRadixItems];
  const uint64_t wb = base + (uint64_t)warp * (32 * kRadixItems) + lane;
#pragma unroll
  for (int i = 0; i < kRadixItems; ++i) {
    const uint64_t idx = wb + i * 32;
    k[i] = idx < n ? kin[idx] : 0u;
    v[i] = idx < n ? vin[idx] : 0u;
  }
  uint16_t* mine = wc + warp * kRadixBins;
  const unsigned lt = lane_lt_mask();
#pragma unroll
  for (int i = 0; i < kRadixItems; ++i) {
    const bool valid = wb + i * 32 < n;
    const uint32_t d = valid ? ((k[i] >> shift) & mask) : 0xffffu;
    const unsigned peers = __match_any_sync(kFull, d);
    const uint32_t before = valid ? mine[d] : 0u;
    __syncwarp();
    if (valid && lane == (unsigned)(__ffs(peers) - 1)) mine[d] = (uint16_t)(before + __popc(peers));
    __syncwarp();
    rk[i] = (uint16_t)(before + __popc(peers & lt));
  }
  __syncthreads();
  // per digit (thread = digit): warp offsets, tile count, tile-local start
  const uint32_t d = tid;
  uint32_t run = 0;
#pragma unroll
  for (int w = 0; w < kRadixWarps; ++w) {
    const uint32_t c = wc[w * kRadixBins + d];
    wc[w * kRadixBins + d] = (uint16_t)run;
    run += c;
  }
  uint32_t tt;
  const uint32_t ls = block_excl_scan<kRadixThreads>(run, tt, s_red, OpSum(), 0u);
  lstart[d] = ls;
  // global start of digit d in this pass (exclusive over the pass histogram)
  const uint32_t gd = block_excl_scan<kRadixThreads>(hist[d], tt, s_red, OpSum(), 0u);
  // decoupled look-back for digit d
  uint32_t prefix = 0;
  unsigned long long* my = st + tile * kRadixBins + d;
  const unsigned long long ep = (unsigned long long)epoch << 34;
  if (tile == 0) {
    *reinterpret_cast<volatile unsigned long long*>(my) = ep | (2ull << 32) | run;
  } else {
    *reinterpret_cast<volatile unsigned long long*>(my) = ep | (1ull << 32) | run;
    int64_t t = (int64_t)tile - 1;
    while (true) {
      volatile unsigned long long* w = reinterpret_cast<volatile unsigned long long*>(st + (uint64_t)t * kRadixBins + d);
      unsigned long long s;
      do {
        s = *w;
      } while ((s >> 34) != (unsigned long long)epoch);
      prefix += (uint32_t)s;
      if (((s >> 32) & 3ull) == 2ull) break;
      --t;
    }
    *reinterpret_cast<volatile unsigned long long*>(my) = ep | (2ull << 32) | (uint32_t)(prefix + run);
  }
  gbase[d] = gd + prefix - ls;
  __syncthreads();
  // digit-sorted tile in shared memory
#pragma unroll
  for (int i = 0; i < kRadixItems; ++i) {
    if (wb + i * 32 < n) {
      const uint32_t dd = (k[i] >> shift) & mask;
      const uint32_t pos = lstart[dd] + wc[warp * kRadixBins + dd] + rk[i];
      sk[pos] = k[i];
      sv[pos] = v[i];
    }
  }
  __syncthreads();
  const uint32_t tn = n - base < (uint64_t)kRadixTile ? (uint32_t)(n - base) : (uint32_t)kRadixTile;
  for (uint32_t j = tid; j < tn; j += kRadixThreads) {
    const uint32_t kk = sk[j];
    const uint32_t o = gbase[(kk >> shift) & mask] + j;
    kout[o] = kk;
    vout[o] = sv[j];
  }
}

}  // namespace prims
