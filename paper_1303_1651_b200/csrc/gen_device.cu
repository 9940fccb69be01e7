// Device-side operand generators for the stencil configs (C1, the C2 sweep,
// C4): every row is independent and its first entry has a closed form, so
// each thread writes its rows straight into HBM — no host generation and no
// upload. Bit-identical to the host generators (genmat.cpp; gen_fd restates
// sparsemm/genmat.py:79-103). The random families (C3's gen_random_k,
// genmat.py:106-130, and C5's Zipf rows) stay on the host: each matrix is ONE
// splitmix64 stream whose draws shift with every rejected duplicate column,
// so row r's first draw depends on every row before it.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/spmmm_gen.h"

namespace {

// 5-point Laplacian, row i = x + g*y: entries (y>0: i-g) (x>0: i-1) i
// (x<g-1: i+1) (y<g-1: i+g), -1 off the diagonal, 4 on it. Entries before
// row i: 5i minus the rows (before i) on each of the four borders.
__global__ void k_gen_fd(uint64_t g, uint64_t* __restrict__ rp, uint64_t* __restrict__ ci,
                         double* __restrict__ v) {
  const uint64_t n = g * g;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i <= n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t x0 = (i + g - 1) / g;                 // rows with x == 0
    const uint64_t x1 = i / g;                           // rows with x == g-1
    const uint64_t y0 = i < g ? i : g;                   // rows with y == 0
    const uint64_t y1 = i > (g - 1) * g ? i - (g - 1) * g : 0;  // rows with y == g-1
    uint64_t pos = g == 1 ? i : 5 * i - x0 - x1 - y0 - y1;
    rp[i] = pos;
    if (i == n) break;
    const uint64_t x = i % g, y = i / g;
    if (y > 0) { ci[pos] = i - g; v[pos++] = -1.0; }
    if (x > 0) { ci[pos] = i - 1; v[pos++] = -1.0; }
    ci[pos] = i; v[pos++] = 4.0;
    if (x + 1 < g) { ci[pos] = i + 1; v[pos++] = -1.0; }
    if (y + 1 < g) { ci[pos] = i + g; v[pos++] = -1.0; }
  }
}

// 27-point stencil, row i = x + g*y + g^2*z, neighbours in (dz, dy, dx)
// lexicographic order (ascending columns), 26 on the diagonal, -1 elsewhere.
// Per axis a coordinate t has c(t) in-range offsets (2 at a face, 3 inside)
// and S(t) = sum of c over the coordinates before t = 3t - 1 (t >= 1); with
// T = 3g - 2 per axis, the entries before row i are
// S(z) T^2 + c(z) (S(y) T + c(y) S(x)).
__device__ __forceinline__ uint64_t axis_c(uint64_t t, uint64_t g) {
  return (t > 0) + 1 + (t + 1 < g);
}
__device__ __forceinline__ uint64_t axis_s(uint64_t t) { return t ? 3 * t - 1 : 0; }

__global__ void k_gen_fd3(uint64_t g, uint64_t* __restrict__ rp, uint64_t* __restrict__ ci,
                          double* __restrict__ v) {
  const uint64_t g2 = g * g, n = g2 * g, T = 3 * g - 2;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i <= n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    if (i == n) {
      rp[n] = T * T * T;
      break;
    }
    const uint64_t x = i % g, y = (i / g) % g, z = i / g2;
    uint64_t pos = axis_s(z) * T * T + axis_c(z, g) * (axis_s(y) * T + axis_c(y, g) * axis_s(x));
    if (g == 1) pos = 0;
    rp[i] = pos;
    for (int dz = -1; dz <= 1; ++dz) {
      if ((dz < 0 && z == 0) || (dz > 0 && z + 1 >= g)) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        if ((dy < 0 && y == 0) || (dy > 0 && y + 1 >= g)) continue;
        for (int dx = -1; dx <= 1; ++dx) {
          if ((dx < 0 && x == 0) || (dx > 0 && x + 1 >= g)) continue;
          const uint64_t j = uint64_t(int64_t(i) + dx + int64_t(g) * dy + int64_t(g2) * dz);
          ci[pos] = j;
          v[pos++] = j == i ? 26.0 : -1.0;
        }
      }
    }
  }
}

int launch(void (*k)(uint64_t, uint64_t*, uint64_t*, double*), uint64_t g, uint64_t rows,
           uint64_t* rp, uint64_t* ci, double* v, void* stream) {
  if (g < 1 || !rp || !ci || !v) return 2;
  const uint64_t blocks = (rows + 1 + 255) / 256;
  k<<<unsigned(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0,
      static_cast<cudaStream_t>(stream)>>>(g, rp, ci, v);
  if (cudaGetLastError() != cudaSuccess) return 3;
  return cudaStreamSynchronize(static_cast<cudaStream_t>(stream)) == cudaSuccess ? 0 : 3;
}

}  // namespace

extern "C" {

int spmmm_gen_fd_device(uint64_t grid, uint64_t* row_ptr, uint64_t* col_idx, double* values,
                        void* stream) {
  return launch(k_gen_fd, grid, grid * grid, row_ptr, col_idx, values, stream);
}

int spmmm_gen_fd3_device(uint64_t grid, uint64_t* row_ptr, uint64_t* col_idx, double* values,
                         void* stream) {
  return launch(k_gen_fd3, grid, grid * grid * grid, row_ptr, col_idx, values, stream);
}

}  // extern "C"
