// Device-side building blocks for the sm_100a spMMM pipeline: warp scans, the
// register bitonic sort and the decoupled look-back. The per-row paths are in
// rows.cuh, the kernels in kernels.cuh / aux_kernels.cuh.
//
// Numerics: every product is fl(a*b) via __dmul_rn and every accumulation
// step fl(acc + p) via __dadd_rn, so nvcc cannot contract them into DFMA.
// Together with the per-column left fold in ascending A-entry order this
// reproduces the reference's arithmetic exactly (kernels.py:167-174).
#pragma once

#include <cstdint>
#include <type_traits>

#include <cuda_runtime.h>

namespace spmmm {

constexpr uint32_t kFull = 0xffffffffu;
constexpr uint32_t kEmptyKey = 0xffffffffu;

// Row classes (decided from the per-row product count of the count pass).
enum RowClass : int {
  kRowZero = 0,   // no products: empty C row
  kRowShort = 1,  // <= 32 products and <= 32 A entries: one product per lane
  kRowMedium = 2, // <= medium limit products: warp + shared-memory hash table
  kRowLong = 3    // anything longer: block-per-row kernel, staged in a buffer
};

struct DevCsr {
  const uint64_t* __restrict__ rp;  // rows+1 (rp[0] may be nonzero for row blocks)
  const uint64_t* __restrict__ ci;  // nnz
  const double* __restrict__ v;     // nnz
  uint64_t rows, cols, nnz;
};

__device__ __forceinline__ int classify(uint32_t prod, uint64_t na, uint32_t medium_limit) {
  if (prod == 0) return kRowZero;
  if (prod <= 32 && na <= 32) return kRowShort;
  if (prod <= medium_limit) return kRowMedium;
  return kRowLong;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---- operand loads (read-only for the whole kernel: non-coherent path) ----
__device__ __forceinline__ uint64_t ld_idx(const uint64_t* p) {
  return __ldg(reinterpret_cast<const unsigned long long*>(p));
}
__device__ __forceinline__ double ld_val(const double* p) { return __ldg(p); }

// ---- relaxed gpu-scope accesses for the look-back status words ----
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---- warp collectives ----
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, x, d);
    if (lane >= uint32_t(d)) x += t;
  }
  return x;
}

__device__ __forceinline__ uint64_t warp_incl_scan64(uint64_t x) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t t = __shfl_up_sync(kFull, x, d);
    if (lane >= uint32_t(d)) x += t;
  }
  return x;
}

__device__ __forceinline__ uint64_t warp_sum64(uint64_t x) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(kFull, x, d);
  return x;
}

template <typename K>
__device__ __forceinline__ K shfl_xor_key(K k, int m) {
  return __shfl_xor_sync(kFull, k, m);
}

// Bitonic sort of E*32 keys held E per lane (element index e*32 + lane),
// ascending. Distances >= 32 are in-register exchanges, shorter ones are
// lane shuffles. N >= E is the register array capacity.
template <int E, int N, typename K>
__device__ __forceinline__ void bitonic_sort(K (&key)[N]) {
  static_assert(E <= N, "sort width exceeds register capacity");
  const uint32_t lane = lane_id();
  constexpr int n = E * 32;
#pragma unroll
  for (int k = 2; k <= n; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int je = j >> 5;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if ((e & je) == 0) {
            const int e2 = e | je;
            const bool up = ((e << 5) & k) == 0;
            const K a = key[e], b = key[e2];
            const K lo = a < b ? a : b;
            const K hi = a < b ? b : a;
            key[e] = up ? lo : hi;
            key[e2] = up ? hi : lo;
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const K p = shfl_xor_key(key[e], j);
          const uint32_t i = uint32_t(e) * 32u + lane;
          const bool up = (i & uint32_t(k)) == 0;
          const bool lower = (lane & uint32_t(j)) == 0;
          const K mn = key[e] < p ? key[e] : p;
          const K mx = key[e] < p ? p : key[e];
          key[e] = (lower == up) ? mn : mx;
        }
      }
    }
  }
}

// R independent one-key-per-lane bitonic sorts (32 keys each), interleaved so
// the shuffle chains of different rows overlap.
template <int R, typename K>
__device__ __forceinline__ void bitonic32_multi(K (&key)[R]) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const bool up = (lane & uint32_t(k)) == 0;
      const bool lower = (lane & uint32_t(j)) == 0;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const K p = shfl_xor_key(key[i], j);
        const K mn = key[i] < p ? key[i] : p;
        const K mx = key[i] < p ? p : key[i];
        key[i] = (lower == up) ? mn : mx;
      }
    }
  }
}

// Runtime-width dispatch of the bitonic sort (E a power of two <= N).
template <int N, typename K>
__device__ __forceinline__ void bitonic_sort_dyn(K (&key)[N], int E) {
  if (E <= 1) { bitonic_sort<1>(key); return; }
  if constexpr (N >= 2) { if (E == 2) { bitonic_sort<2>(key); return; } }
  if constexpr (N >= 4) { if (E == 4) { bitonic_sort<4>(key); return; } }
  if constexpr (N >= 8) { if (E == 8) { bitonic_sort<8>(key); return; } }
  if constexpr (N >= 16) { if (E == 16) { bitonic_sort<16>(key); return; } }
  if constexpr (N >= 32) { if (E == 32) { bitonic_sort<32>(key); return; } }
}

// ---------------------------------------------------------------------------
// Two-level decoupled look-back (single-pass exclusive scan of tile nnz).
//
// Status word: [63:62] flag (0 invalid, 1 aggregate, 2 inclusive prefix),
// [61:46] epoch (per call, so the arrays never need clearing), [45:0] value.
// Level 1: one word per tile. Level 2: one word per group of 32 tiles,
// holding the group's aggregate or its inclusive prefix. With thousands of
// warp tiles in flight a flat look-back would walk a whole wave of tiles;
// with groups it reads at most its own group's tiles plus a few group words.
// A walker that meets a group word nobody has written yet builds it from
// the group's 32 tile words (benign race: every writer stores a correct value).
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagPrefix = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 46) - 1;
constexpr int kGroupShift = 5;

__device__ __forceinline__ uint32_t status_flag(uint64_t w, uint32_t epoch) {
  return ((w >> 46) & 0xffffu) == (epoch & 0xffffu) ? uint32_t(w >> 62) : 0u;
}

__device__ __forceinline__ uint64_t status_word(uint64_t flag, uint32_t epoch, uint64_t v) {
  return flag | (uint64_t(epoch & 0xffffu) << 46) | v;
}

// The 32 tile words of group g -> the group's word (its inclusive prefix if
// some tile already has one, else its aggregate). Warp-collective; every
// tile word must be published.
__device__ __forceinline__ uint64_t group_word(const uint64_t* tstat, uint64_t g, uint32_t epoch) {
  const uint32_t lane = lane_id();
  const uint64_t tw = ld_relaxed(&tstat[(g << kGroupShift) + lane]);
  const uint32_t tpm = __ballot_sync(kFull, status_flag(tw, epoch) == 2);
  const uint32_t first = tpm ? 31u - __clz(tpm) : 0u;
  const uint64_t v = warp_sum64(lane >= first ? (tw & kValMask) : 0ull);
  return status_word(tpm ? kFlagPrefix : kFlagAgg, epoch, v);
}

// Publish a tile's aggregate (tile 0 publishes its prefix). The last tile of
// a group to publish (per-group counter) also publishes the group's word, so
// walkers never have to assemble it. Warp-collective.
__device__ __forceinline__ void publish_aggregate(uint64_t* tstat, uint64_t* gstat,
                                                  uint32_t* gcount, uint64_t tile, uint64_t agg,
                                                  uint64_t ntiles, uint32_t epoch) {
  const uint32_t lane = lane_id();
  const uint64_t g = tile >> kGroupShift;
  const bool full_group = ((g + 1) << kGroupShift) <= ntiles;
  uint32_t old = 0;
  if (lane == 0) {
    st_relaxed(&tstat[tile], status_word(tile == 0 ? kFlagPrefix : kFlagAgg, epoch, agg));
    if (full_group) {
      // acq_rel: our word is released before it is counted, and the 31 words
      // counted before us are visible if we are the last
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                   : "=r"(old) : "l"(gcount + g) : "memory");
    }
  }
  old = __shfl_sync(kFull, old, 0);
  if (full_group && old == 31) {
    const uint64_t gw = group_word(tstat, g, epoch);
    if (lane == 0) st_relaxed(&gstat[g], gw);
  }
}

// Warp-collective. The tile's aggregate must already be published. Returns
// its exclusive prefix and publishes the inclusive one (and the group's, for
// the last tile of a group).
__device__ __forceinline__ uint64_t lookback(uint64_t* tstat, uint64_t* gstat, uint64_t tile,
                                             uint64_t agg, uint32_t epoch) {
  const uint32_t lane = lane_id();
  const uint64_t g = tile >> kGroupShift;
  const uint32_t q = uint32_t(tile & 31u);
  uint64_t excl = 0;
  bool done = tile == 0;
  // ---- level 1: earlier tiles of the same group ----
  if (!done && q > 0) {
    const bool in = lane < q;
    int spins = 0;
    while (true) {
      uint64_t w = 0;
      uint32_t flag = 0;
      if (in) {
        w = ld_relaxed(&tstat[(g << kGroupShift) + lane]);
        flag = status_flag(w, epoch);
      }
      const uint32_t pm = __ballot_sync(kFull, in && flag == 2);
      const uint32_t first = pm ? 31u - __clz(pm) : 0u;  // nearest prefix
      const uint32_t need = ((1u << q) - 1u) & ~((1u << first) - 1u);
      if (__ballot_sync(kFull, in && flag == 0) & need) {
        __nanosleep(32u << (spins < 5 ? spins++ : 5));
        continue;
      }
      excl = warp_sum64((in && lane >= first) ? (w & kValMask) : 0ull);
      done = pm != 0;
      break;
    }
  }
  // ---- level 2: earlier groups ----
  if (!done && g > 0) {
    int64_t gb = int64_t(g) - 1;
    int spins = 0;
    while (true) {
      const int64_t gi = gb - int64_t(lane);
      uint64_t w = 0;
      uint32_t flag = 2;  // before group 0: an implicit prefix of 0
      if (gi >= 0) {
        w = ld_relaxed(&gstat[gi]);
        flag = status_flag(w, epoch);
      }
      const uint32_t pm = __ballot_sync(kFull, flag == 2);
      const uint32_t lim = pm ? uint32_t(__ffs(pm) - 1) : 31u;
      const uint32_t window = lim == 31 ? kFull : ((2u << lim) - 1u);
      if (__ballot_sync(kFull, flag == 0) & window) {
        __nanosleep(32u << (spins < 5 ? spins++ : 5));
        continue;
      }
      excl += warp_sum64((lane <= lim && gi >= 0) ? (w & kValMask) : 0ull);
      if (pm) break;
      gb -= 32;
    }
  }
  if (lane == 0) {
    if (tile != 0) st_relaxed(&tstat[tile], status_word(kFlagPrefix, epoch, excl + agg));
    if (q == 31) st_relaxed(&gstat[g], status_word(kFlagPrefix, epoch, excl + agg));
  }
  return excl;
}

}  // namespace spmmm
