// Kernels of the multi-GPU row-block product.
//
// Product-balanced partition: rows of C are independent (kernels.py:323-329),
// so GPU g of G takes rows [lower_bound(P, g·T/G), lower_bound(P, (g+1)·T/G))
// of A, where P is the exclusive prefix of per-row product counts (the count
// pass, `prod`) and T = Σ prod. Every GPU holds all of A and B after the
// operand all-gather and runs the same integer arithmetic, so every rank
// derives the same bounds without a collective. Same targets and lower_bound
// as distributed.partition_rows (host numpy), which the tests compare against.
#pragma once

#include <cstdint>

namespace spmmm {

constexpr int kPartChunkRows = 4096;   // rows per chunk of the two-level scan (minimum)
constexpr int kPartMaxChunks = 4096;   // chunk sums one block scans in shared memory
constexpr int kPartMaxParts = 64;

// chunk sums of prod: one block per chunk of `L` rows
__global__ void k_part_chunk_sums(const uint32_t* __restrict__ prod, uint64_t rows, uint32_t L,
                                  unsigned long long* __restrict__ sums) {
  const uint64_t r0 = uint64_t(blockIdx.x) * L;
  const uint64_t r1 = r0 + L < rows ? r0 + L : rows;
  unsigned long long s = 0;
  for (uint64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) s += prod[r];
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
  __shared__ unsigned long long ws[32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += ws[w];
    sums[blockIdx.x] = t;
  }
}

// One block of 1024 threads: inclusive scan of the chunk sums, then one warp
// per target g·T/parts (g = 1 .. parts-1) finds its chunk by binary search and
// the row inside it by a warp scan. out[0..parts] = bounds, out[parts+1] = T.
// `out` is mapped host memory (the caller's pinned words).
__global__ void k_partition(const uint32_t* __restrict__ prod, uint64_t rows, uint32_t L,
                            const unsigned long long* __restrict__ sums, uint32_t nchunks,
                            int parts, unsigned long long* __restrict__ out) {
  __shared__ unsigned long long incl[kPartMaxChunks];
  __shared__ unsigned long long wtot[32];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  // each thread scans 4 consecutive chunk sums, then a block scan of the totals
  constexpr uint32_t kPer = kPartMaxChunks / 1024;
  unsigned long long v[kPer], run = 0;
#pragma unroll
  for (uint32_t u = 0; u < kPer; ++u) {
    const uint32_t i = tid * kPer + u;
    run += i < nchunks ? sums[i] : 0ull;
    v[u] = run;
  }
  unsigned long long x = run;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, d);
    if (int(lane) >= d) x += y;
  }
  if (lane == 31) wtot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = wtot[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, w, d);
      if (int(lane) >= d) w += y;
    }
    wtot[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  const unsigned long long base = (x - run) + (warp ? wtot[warp - 1] : 0ull);
#pragma unroll
  for (uint32_t u = 0; u < kPer; ++u) incl[tid * kPer + u] = base + v[u];
  __syncthreads();
  const unsigned long long total = nchunks ? incl[nchunks - 1] : 0ull;
  for (int g = int(warp) + 1; g < parts; g += int(blockDim.x >> 5)) {
    const unsigned long long t =
        (unsigned long long)((unsigned __int128)total * (unsigned)g / (unsigned)parts);
    uint64_t bound = 0;
    if (t > 0) {
      // first chunk whose inclusive prefix reaches t (exists: t <= total)
      uint32_t lo = 0, hi = nchunks - 1;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (incl[mid] >= t) hi = mid; else lo = mid + 1;
      }
      unsigned long long acc = lo ? incl[lo - 1] : 0ull;  // < t
      const uint64_t r0 = uint64_t(lo) * L;
      const uint64_t r1 = r0 + L < rows ? r0 + L : rows;
      bound = r1;
      for (uint64_t r = r0; r < r1; r += 32) {
        const uint64_t rr = r + lane;
        unsigned long long s = rr < r1 ? prod[rr] : 0u;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const unsigned long long y = __shfl_up_sync(0xffffffffu, s, d);
          if (int(lane) >= d) s += y;
        }
        // prefix after rows r..rr inclusive: the bound is rr + 1 for the first lane reaching t
        const unsigned hit = __ballot_sync(0xffffffffu, rr < r1 && acc + s >= t);
        if (hit) {
          bound = r + uint64_t(__ffs(hit) - 1) + 1;
          break;
        }
        acc += __shfl_sync(0xffffffffu, s, 31);
      }
    }
    if (lane == 0) reinterpret_cast<volatile unsigned long long*>(out)[g] = bound;
  }
  if (tid == 0) {
    volatile unsigned long long* o = out;
    o[0] = 0;
    o[parts] = rows;
    o[parts + 1] = total;
  }
}

// row pointers of a downloaded block, shifted by the nnz of the blocks before it
__global__ void k_copy_offset(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst,
                              uint64_t n, uint64_t off) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    dst[i] = src[i] + off;
}

}  // namespace spmmm
