// Storage-order conversion (transpose of the index structure), convert.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "device.cuh"

namespace spmmm {

// Scratch for n entries and `cols` columns of the input (keys, permutation,
// CUB temporary storage).
size_t transpose_scratch_bytes(uint64_t n, uint64_t cols);

// CSR `in` (entries [base, base + n) of its arrays) -> CSR of in^T:
// out_rp[cols + 1], out_ci[n] (input row indices), out_v[n]; within each
// output row the entries keep the input's row order. *err |= 1 for a column
// index >= in.cols, |= 2 for a malformed row pointer.
cudaError_t transpose_csr(const DevCsr& in, uint64_t base, uint64_t n, uint64_t* out_rp,
                          uint64_t* out_ci, double* out_v, void* scratch, size_t scratch_bytes,
                          unsigned long long* err, int sms, cudaStream_t s);

}  // namespace spmmm
