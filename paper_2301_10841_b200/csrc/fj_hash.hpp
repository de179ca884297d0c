// Hash functions shared by host and device code.
//
// tuple_hash() restates the reference's TupleHash (proj/include/fj/value.hpp:61-67)
// for integer tuples: h = 0x811c9dc5; h = (h ^ v.hash()) * 0x100000001b3 per
// value, where Value::hash() of an Int (value.hpp:49-53) is the libstdc++
// std::hash<int64_t> (identity) xor'ed with index 0 * 0x9e3779b97f4a7c15 = 0.
// Pinned by tests/golden/tuplehash_kats.json, generated from the reference
// header itself (oracle/_ref).
//
// The output checksum (BASELINE.json north_star: "sum of a 64-bit hash of each
// output tuple") is  sum over outputs of  mult * fmix64(tuple_hash(t))  mod 2^64
// with t in head-variable order; fmix64 is the MurmurHash3
// 64-bit finaliser (the plain FNV fold has weak low bits).
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define FJ_HD __host__ __device__ __forceinline__
#else
#define FJ_HD inline
#endif

namespace fj {

constexpr uint64_t kTupleHashSeed = 0x811c9dc5ULL;
constexpr uint64_t kTupleHashMul = 0x100000001b3ULL;

FJ_HD uint64_t tuple_hash_step(uint64_t h, int64_t v) {
  return (h ^ static_cast<uint64_t>(v)) * kTupleHashMul;
}

FJ_HD uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}

FJ_HD uint64_t checksum_word(uint64_t tuple_h) { return fmix64(tuple_h); }

// Index hash for the device COLT tables: (parent subtrie id, 32-bit key word).
FJ_HD uint64_t slot_hash(uint32_t parent, uint32_t key) {
  return fmix64((static_cast<uint64_t>(parent) << 32) | key);
}

// Hash-partition function for multi-GPU sharding on the first plan variable.
FJ_HD uint32_t partition_of(int32_t v, uint32_t nparts) {
  const uint64_t h = fmix64(static_cast<uint64_t>(static_cast<int64_t>(v)) ^ 0x5bd1e995ULL);
  // power-of-two rank counts (1/2/4/8 GPUs): a mask, the same value as h % nparts
  // without the 64-bit division subroutine on the device
  if ((nparts & (nparts - 1)) == 0) return static_cast<uint32_t>(h & (nparts - 1));
  return static_cast<uint32_t>(h % nparts);
}

}  // namespace fj
