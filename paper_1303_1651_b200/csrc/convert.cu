// Storage-order conversion on the GPU: CSR of M -> CSR of M^T, which is the
// CSC of M (formats.py:302-329 csr_to_csc; a CSC passed as the CSR view of its
// transpose gives formats.py:332-357 csc_to_csr). The reference's conversion
// is a stable counting scatter over the entries in major order, so within
// each output slice the minor indices ascend; here the same order comes from a
// stable radix sort of (column key, entry index) pairs (CUB, CUDA toolkit
// headers) followed by a gather. Not on the north-star path: it serves
// multiply_mixed's single conversion (kernels.py:417-438).
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include "convert.cuh"
#include "device.cuh"

namespace spmmm {
namespace {

__global__ void k_tr_init(DevCsr in, uint64_t base, uint64_t n, uint32_t* __restrict__ keys,
                          uint32_t* __restrict__ perm, unsigned long long* __restrict__ err) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t c = ld_idx(in.ci + base + i);
    if (c >= in.cols) atomicOr(err, 1ull);
    keys[i] = uint32_t(c);
    perm[i] = uint32_t(i);
  }
}

__global__ void k_tr_rows(DevCsr in, uint64_t base, uint64_t n,
                          unsigned long long* __restrict__ err) {
  for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < in.rows;
       r += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t lo = ld_idx(in.rp + r), hi = ld_idx(in.rp + r + 1);
    if (hi < lo || lo < base || hi > base + n) atomicOr(err, 2ull);
  }
}

// entry i (relative to base) -> its row: the last r with rp[r] - base <= i
__device__ __forceinline__ uint64_t row_of(const uint64_t* rp, uint64_t rows, uint64_t base,
                                           uint64_t i) {
  uint64_t lo = 0, hi = rows;  // answer in [0, rows)
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) >> 1;
    if (ld_idx(rp + mid) - base <= i) lo = mid;
    else hi = mid;
  }
  return lo;
}

__global__ void k_tr_gather(DevCsr in, uint64_t base, uint64_t n, const uint32_t* __restrict__ perm,
                            uint64_t* __restrict__ out_ci, double* __restrict__ out_v) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t e = perm[i];
    out_ci[i] = row_of(in.rp, in.rows, base, e);
    out_v[i] = ld_val(in.v + base + e);
  }
}

// out_rp[c] = first sorted position with key >= c
__global__ void k_tr_ptr(const uint32_t* __restrict__ keys, uint64_t n, uint64_t cols,
                         uint64_t* __restrict__ out_rp) {
  for (uint64_t c = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; c <= cols;
       c += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (uint64_t(keys[mid]) < c) lo = mid + 1;
      else hi = mid;
    }
    out_rp[c] = lo;
  }
}

int bits_for(uint64_t x) {
  int b = 1;
  while (b < 32 && (uint64_t(1) << b) < x) ++b;
  return b;
}

}  // namespace

size_t transpose_scratch_bytes(uint64_t n, uint64_t cols) {
  size_t cub_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, static_cast<const uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr),
                                  static_cast<const uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr), int64_t(n), 0,
                                  bits_for(cols + 1));
  return 4 * size_t(n) * sizeof(uint32_t) + cub_bytes + 256;
}

cudaError_t transpose_csr(const DevCsr& in, uint64_t base, uint64_t n, uint64_t* out_rp,
                          uint64_t* out_ci, double* out_v, void* scratch, size_t scratch_bytes,
                          unsigned long long* err, int sms, cudaStream_t s) {
  uint32_t* keys = static_cast<uint32_t*>(scratch);
  uint32_t* keys2 = keys + n;
  uint32_t* perm = keys2 + n;
  uint32_t* perm2 = perm + n;
  void* temp = perm2 + n;
  size_t temp_bytes = scratch_bytes - 4 * size_t(n) * sizeof(uint32_t);
  const unsigned grid = unsigned(sms) * 8;
  if (in.rows) k_tr_rows<<<grid, 256, 0, s>>>(in, base, n, err);
  if (n) {
    k_tr_init<<<grid, 256, 0, s>>>(in, base, n, keys, perm, err);
    cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys, keys2, perm, perm2,
                                                    int64_t(n), 0, bits_for(in.cols + 1), s);
    if (e != cudaSuccess) return e;
    k_tr_gather<<<grid, 256, 0, s>>>(in, base, n, perm2, out_ci, out_v);
  }
  k_tr_ptr<<<grid, 256, 0, s>>>(keys2, n, in.cols, out_rp);
  return cudaGetLastError();
}

}  // namespace spmmm
