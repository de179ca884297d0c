// Device R-MAT generator (bench input for the 2^27-vertex scale config): the
// same counter-based edge stream and selection rule as fjgen_rmat (first m
// distinct non-loop edges in stream order), so the output is bit-identical to
// the host generator; a CUB radix sort replaces the host sort.
#include <cuda_runtime.h>

#include <cstdint>
#include <cub/cub.cuh>
#include <string>

#include "rmat.hpp"

namespace {
std::string g_dev_err;

__global__ void k_cand(uint64_t seed, int scale, double a, double b, double c, uint64_t K, uint64_t* keys,
                       uint32_t* idx) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < K; i += (uint64_t)gridDim.x * blockDim.x) {
    keys[i] = fjgen::rmat_edge(seed, i, scale, a, b, c);
    idx[i] = (uint32_t)i;
  }
}

__global__ void k_first(const uint64_t* keys, uint64_t K, uint8_t* flags) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < K; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    const bool loop = (k >> 32) == (k & 0xffffffffULL);
    flags[i] = (!loop && (i == 0 || keys[i - 1] != k)) ? 1 : 0;
  }
}

__global__ void k_gather(uint64_t seed, int scale, double a, double b, double c, const uint32_t* sel, uint64_t m,
                         int32_t* src, int32_t* dst) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t e = fjgen::rmat_edge(seed, sel[i], scale, a, b, c);
    src[i] = (int32_t)(e >> 32);
    dst[i] = (int32_t)(e & 0xffffffffULL);
  }
}

struct Bufs {
  void* p[8] = {};
  ~Bufs() {
    for (void* x : p)
      if (x) cudaFree(x);
  }
};

#define DCK(x)                                   \
  do {                                           \
    cudaError_t _e = (x);                        \
    if (_e != cudaSuccess) {                     \
      g_dev_err = std::string(#x) + ": " + cudaGetErrorString(_e); \
      return 4;                                  \
    }                                            \
  } while (0)
}  // namespace

extern "C" {

const char* fjgen_device_last_error(void) { return g_dev_err.c_str(); }

// Writes m edges into device buffers dev_src / dev_dst on `device`.
int fjgen_rmat_device(int device, uint64_t seed, int scale, uint64_t m, double a, double b, double c,
                      int32_t* dev_src, int32_t* dev_dst) {
  DCK(cudaSetDevice(device));
  if (scale < 1 || scale > 31) {
    g_dev_err = "scale must be 1..31";
    return 3;
  }
  uint64_t K = m + m / 4 + 1024;
  while (true) {
    if (K >= (1ull << 32)) {
      g_dev_err = "candidate stream too long";
      return 4;
    }
    Bufs B;
    uint64_t *keys, *keys2;
    uint32_t *idx, *idx2, *sel;
    uint8_t* flags;
    int* nsel;
    DCK(cudaMalloc(&B.p[0], K * 8));
    DCK(cudaMalloc(&B.p[1], K * 8));
    DCK(cudaMalloc(&B.p[2], K * 4));
    DCK(cudaMalloc(&B.p[3], K * 4));
    DCK(cudaMalloc(&B.p[4], K));
    DCK(cudaMalloc(&B.p[5], K * 4));
    DCK(cudaMalloc(&B.p[6], 8));
    keys = (uint64_t*)B.p[0];
    keys2 = (uint64_t*)B.p[1];
    idx = (uint32_t*)B.p[2];
    idx2 = (uint32_t*)B.p[3];
    flags = (uint8_t*)B.p[4];
    sel = (uint32_t*)B.p[5];
    nsel = (int*)B.p[6];
    const int n = (int)K;
    k_cand<<<148 * 16, 256>>>(seed, scale, a, b, c, K, keys, idx);
    DCK(cudaGetLastError());
    size_t tb = 0, tb2 = 0, tb3 = 0;
    DCK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, idx, idx2, n));
    DCK(cub::DeviceSelect::Flagged(nullptr, tb2, idx2, flags, sel, nsel, n));
    DCK(cub::DeviceRadixSort::SortKeys(nullptr, tb3, sel, idx, n));
    size_t tmp_bytes = std::max(tb, std::max(tb2, tb3));
    DCK(cudaMalloc(&B.p[7], tmp_bytes));
    size_t t = tmp_bytes;
    // stable sort by edge key: within a key, stream order (first occurrence first)
    DCK(cub::DeviceRadixSort::SortPairs(B.p[7], t, keys, keys2, idx, idx2, n));
    k_first<<<148 * 16, 256>>>(keys2, K, flags);
    DCK(cudaGetLastError());
    t = tmp_bytes;
    DCK(cub::DeviceSelect::Flagged(B.p[7], t, idx2, flags, sel, nsel, n));
    int U = 0;
    DCK(cudaMemcpy(&U, nsel, sizeof(int), cudaMemcpyDeviceToHost));
    if ((uint64_t)U >= m) {
      t = tmp_bytes;
      DCK(cub::DeviceRadixSort::SortKeys(B.p[7], t, sel, idx, U));  // stream order
      k_gather<<<148 * 16, 256>>>(seed, scale, a, b, c, idx, m, dev_src, dev_dst);
      DCK(cudaGetLastError());
      DCK(cudaDeviceSynchronize());
      return 0;
    }
    K = K + K / 2;
  }
}

}  // extern "C"
