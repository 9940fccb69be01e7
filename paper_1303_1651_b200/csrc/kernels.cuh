// sm_100a kernels of the spMMM pipeline (see DESIGN.md §3 for the dataflow).
// k_count / k_collect / k_long are in aux_kernels.cuh:
//   k_count    per-row product counts (estimate_nnz / count_mults per row),
//              their total and maximum, structural validation of A and B.
//   k_collect  lists the rows too long for the fused kernel (only when any).
//   k_long     block-per-row product of those rows into a staging buffer.
//   k_fused    one persistent pass over all rows: computes each row (short
//              rows in registers, medium rows in a shared-memory table),
//              obtains the row's output offset by a decoupled look-back scan
//              over tiles, and writes C.row_ptr / C.col_idx / C.values once.
#pragma once

#include "device.cuh"

namespace spmmm {

// ---------------------------------------------------------------------------
// K4: the fused, persistent, single-pass kernel. Must be launched
// cooperatively (all blocks co-resident): tile t is processed by block
// t mod gridDim.x and waits only on tiles < t (look-back), so the smallest
// unfinished tile can always progress.
struct FusedParams {
  DevCsr A, B;
  const uint32_t* prod;
  const uint32_t* lmap;
  const uint64_t* l_off;
  const uint32_t* l_nnz;
  const uint64_t* l_ci;
  const double* l_v;
  uint64_t* c_rp;
  uint64_t* c_ci;
  double* c_v;
  uint64_t* status;
  uint64_t ntiles;
  uint32_t epoch;
  uint32_t medium_limit;
  uint32_t* st_min;
  uint32_t* st_max;
  uint32_t* st_touch;
};

// WARPS warps per block; each warp owns R consecutive rows of a tile
// (R > 1 only without a table). T = shared-memory table slots per warp (0 =
// short rows only). WIDE = 64-bit sort keys (columns too large to pack).
template <int WARPS, int R, int T, bool WIDE, bool STATS>
__global__ void __launch_bounds__(WARPS * 32) k_fused(const FusedParams p) {
  static_assert(WARPS * R <= 32, "tile rows must fit one warp scan");
  static_assert(T == 0 || R == 1, "medium rows keep their table until written");
  constexpr int kRows = WARPS * R;
  constexpr int EMAX = T > 0 ? T / 32 : 1;
  constexpr int LOGT = T > 0 ? __builtin_ctz(T) : 5;
  using K = typename std::conditional<WIDE, unsigned long long, uint32_t>::type;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t s_nnz[kRows];
  __shared__ uint64_t s_base[kRows];

  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  uint32_t* keys = nullptr;
  double* vals = nullptr;
  if constexpr (T > 0) {
    vals = reinterpret_cast<double*>(smem_raw) + size_t(warp) * T;
    keys = reinterpret_cast<uint32_t*>(smem_raw + size_t(WARPS) * T * sizeof(double)) +
           size_t(warp) * T;
    for (uint32_t s = lane; s < uint32_t(T); s += 32) keys[s] = kEmptyKey;
    __syncwarp();
  }

  for (uint64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
    const uint64_t r0 = tile * kRows + uint64_t(warp) * R;
    ShortOut so[R];
    int cls[R];
    uint32_t nnz[R];
    K mk[EMAX];
    int mE = 1;
    uint64_t lidx = 0;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const uint64_t r = r0 + i;
      cls[i] = kRowZero;
      nnz[i] = 0;
      if (r < p.A.rows) {
        const uint64_t lo = ld_idx(p.A.rp + r), hi = ld_idx(p.A.rp + r + 1);
        const uint32_t pr = p.prod[r];
        cls[i] = classify(pr, hi - lo, p.medium_limit);
        uint32_t smin = kEmptyKey, smax = 0, stouch = 0;
        if (cls[i] == kRowShort) {
          nnz[i] = short_row<WIDE, STATS>(p.A, p.B, lo, uint32_t(hi - lo), so[i], smin, smax,
                                          stouch);
        } else if (cls[i] == kRowMedium) {
          if constexpr (T > 0) {
            uint32_t touches = 0;
            medium_accumulate<T, STATS>(p.A, p.B, lo, hi, keys, vals, touches);
            __syncwarp();
            const uint32_t cnt = medium_compact<T, STATS>(keys, vals, smin, smax);
            nnz[i] = cnt;
            int E = 1;
            while (uint32_t(E) * 32u < cnt) E <<= 1;
            mE = E;
#pragma unroll
            for (int e = 0; e < EMAX; ++e) {
              const uint32_t idx = uint32_t(e) * 32u + lane;
              mk[e] = (e < E && idx < cnt) ? ((K(keys[idx]) << LOGT) | K(idx)) : ~K(0);
            }
            bitonic_sort_dyn(mk, E);
            if (STATS) {
#pragma unroll
              for (int d = 16; d > 0; d >>= 1) touches += __shfl_xor_sync(kFull, touches, d);
              stouch = touches;
            }
          }
        } else if (cls[i] == kRowLong) {
          lidx = p.lmap[r];
          nnz[i] = p.l_nnz[lidx];
        }
        if (STATS && lane == 0 && cls[i] != kRowLong) {
          p.st_min[r] = smin;
          p.st_max[r] = smax;
          p.st_touch[r] = stouch;
        }
      }
      if (lane == 0) s_nnz[warp * R + i] = nnz[i];
    }
    __syncthreads();
    if (warp == 0) {
      const uint64_t v = lane < uint32_t(kRows) ? uint64_t(s_nnz[lane]) : 0ull;
      const uint64_t incl = warp_incl_scan64(v);
      const uint64_t agg = __shfl_sync(kFull, incl, 31);
      const uint64_t excl = lookback(p.status, tile, agg, p.epoch);
      if (lane < uint32_t(kRows)) s_base[lane] = excl + incl - v;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const uint64_t r = r0 + i;
      if (r >= p.A.rows) break;
      const uint64_t base = s_base[warp * R + i];
      if (lane == 0) p.c_rp[r + 1] = base + nnz[i];
      if (cls[i] == kRowShort) {
        if (so[i].keep) {
          p.c_ci[base + so[i].rank] = so[i].col;
          p.c_v[base + so[i].rank] = so[i].val;
        }
      } else if (cls[i] == kRowMedium) {
        if constexpr (T > 0) {
#pragma unroll
          for (int e = 0; e < EMAX; ++e) {
            const uint32_t idx = uint32_t(e) * 32u + lane;
            if (e < mE && idx < nnz[i]) {
              const K key = mk[e];
              p.c_ci[base + idx] = uint64_t(key >> LOGT);
              p.c_v[base + idx] = vals[uint32_t(key) & uint32_t(T - 1)];
            }
          }
          __syncwarp();
          for (uint32_t s = lane; s < uint32_t(T); s += 32) keys[s] = kEmptyKey;
          __syncwarp();
        }
      } else if (cls[i] == kRowLong) {
        const uint64_t off = p.l_off[lidx];
        for (uint32_t t = lane; t < nnz[i]; t += 32) {
          p.c_ci[base + t] = p.l_ci[off + t];
          p.c_v[base + t] = p.l_v[off + t];
        }
      }
    }
  }
}

}  // namespace spmmm
