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
  uint64_t pol;  // L2 cache policy for this operand's loads (0 = default)
};

// L2 eviction policies (createpolicy): B is re-read across rows and should
// stay in L2; A (when it is not also B) and C stream through once.
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

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
__device__ __forceinline__ uint64_t ld_idx(const uint64_t* p, uint64_t pol) {
  uint64_t v;
  asm("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_val(const double* p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t ld_u32(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}

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

// compare-exchange half: keep the smaller or the larger key (VIMNMX + predicate)
__device__ __forceinline__ uint32_t keep_minmax(uint32_t a, uint32_t b, bool take_min) {
  return take_min ? umin(a, b) : umax(a, b);
}
__device__ __forceinline__ unsigned long long keep_minmax(unsigned long long a,
                                                          unsigned long long b, bool take_min) {
  return take_min ? ullmin(a, b) : ullmax(a, b);
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
            key[e] = keep_minmax(a, b, up);
            key[e2] = keep_minmax(a, b, !up);
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const K p = shfl_xor_key(key[e], j);
          const uint32_t i = uint32_t(e) * 32u + lane;
          const bool up = (i & uint32_t(k)) == 0;
          const bool lower = (lane & uint32_t(j)) == 0;
          key[e] = keep_minmax(key[e], p, lower == up);
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
      for (int i = 0; i < R; ++i) key[i] = keep_minmax(key[i], shfl_xor_key(key[i], j), lower == up);
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
// Hierarchical decoupled look-back (single-pass exclusive scan of tile nnz).
//
// Status word: [63:62] flag (0 invalid, 1 aggregate, 2 inclusive prefix),
// [61:46] epoch (per call, so the arrays never need clearing), [45:0] value.
// Level 0 has one word per tile, level l one word per 32^l tiles (the item's
// aggregate, or its inclusive prefix). Thousands of tiles are in flight, so
// the nearest published prefix is usually a whole "wave" of tiles back; with
// three levels a look-back reads at most one chunk of 32 siblings per level.
// An item word is written by the last of its 32 children to publish (per-item
// acq_rel counter) and upgraded to a prefix by the last tile it covers.
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagPrefix = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 46) - 1;
constexpr int kLevels = 3;

struct LookbackState {
  uint64_t* stat[kLevels];   // status words per level
  unsigned long long* count[kLevels];  // [1..] per item: children << 46 | their sum (zeroed per call)
  uint64_t n[kLevels];       // items per level
  uint32_t epoch;
  unsigned long long* fault;  // watchdog report (ctrl word), 0 = none
};

// Watchdog: a wait that outlives ~2^20 back-off rounds (about a second) is a
// bug, not a slow predecessor. Record where it happened and stop waiting so
// the host reports an error instead of hanging the process.
constexpr int kSpinLimit = 1 << 20;
__device__ __forceinline__ bool watchdog(const LookbackState& lb, int spins, uint32_t site,
                                         uint64_t tile) {
  if (spins < kSpinLimit) return false;
  if (lane_id() == 0)
    atomicCAS(lb.fault, 0ull, (1ull << 63) | (uint64_t(site) << 48) | (tile & ((1ull << 48) - 1)));
  return true;
}

__device__ __forceinline__ uint32_t status_flag(uint64_t w, uint32_t epoch) {
  return ((w >> 46) & 0xffffu) == (epoch & 0xffffu) ? uint32_t(w >> 62) : 0u;
}

__device__ __forceinline__ uint64_t status_word(uint64_t flag, uint32_t epoch, uint64_t v) {
  return flag | (uint64_t(epoch & 0xffffu) << 46) | v;
}

__device__ __forceinline__ void backoff(int& spins) {
  __nanosleep(spins < 5 ? (32u << spins) : 1024u);
  ++spins;
}

// Publishing a tile: store its word, then add (1 << 46 | aggregate) to the
// enclosing level-1 item's counter. The counter carries the data itself, so
// the child whose add completes the item (count reaches 32) gets the item's
// sum from the atomic's return value and publishes the item word — no fences,
// no re-reading of the children. Higher levels cascade the same way.
constexpr unsigned long long kCountOne = 1ull << 46;

__device__ __forceinline__ void publish_aggregate(const LookbackState& lb, uint64_t tile,
                                                  uint64_t agg) {
  if (lane_id() != 0) return;
  st_relaxed(&lb.stat[0][tile], status_word(tile == 0 ? kFlagPrefix : kFlagAgg, lb.epoch, agg));
  uint64_t sum = agg;
#pragma unroll
  for (int l = 1; l < kLevels; ++l) {
    const uint64_t item = tile >> (5 * l);
    if (((item + 1) << (5 * l)) > lb.n[0]) return;  // incomplete item: never looked up
    const unsigned long long old = atomicAdd(lb.count[l] + item, kCountOne | sum);
    if ((old >> 46) != 31) return;
    sum += old & kValMask;  // the whole item
    st_relaxed(&lb.stat[l][item], status_word(kFlagAgg, lb.epoch, sum));
  }
}

// Warp-collective. The tile's aggregate must be published. Returns the
// exclusive prefix; publishes the inclusive prefix of the tile and of every
// item the tile closes.
__device__ __forceinline__ uint64_t lookback(const LookbackState& lb, uint64_t tile,
                                             uint64_t agg) {
  const uint32_t lane = lane_id();
  const uint32_t epoch = lb.epoch;
  uint64_t excl = 0;
  bool done = tile == 0;
#pragma unroll
  for (int l = 0; l < kLevels && !done; ++l) {
    const uint64_t idx = tile >> (5 * l);
    const uint64_t* st = lb.stat[l];
    if (l < kLevels - 1) {
      // earlier siblings inside the enclosing level-(l+1) item
      const uint32_t q = uint32_t(idx & 31u);
      if (q == 0) continue;
      const uint64_t base = idx - q;
      const bool in = lane < q;
      int spins = 0;
      while (true) {
        uint64_t w = 0;
        uint32_t f = 0;
        if (in) {
          w = ld_relaxed(&st[base + lane]);
          f = status_flag(w, epoch);
        }
        const uint32_t pm = __ballot_sync(kFull, in && f == 2);
        const uint32_t first = pm ? 31u - __clz(pm) : 0u;  // nearest prefix
        const uint32_t need = ((1u << q) - 1u) & ~((1u << first) - 1u);
        if ((__ballot_sync(kFull, in && f == 0) & need) && !watchdog(lb, spins, 2 + l, tile)) {
          backoff(spins);
          continue;
        }
        excl += warp_sum64((in && lane >= first) ? (w & kValMask) : 0ull);
        done = pm != 0;
        break;
      }
    } else {
      // top level: walk back until a prefix (or the start)
      int64_t gb = int64_t(idx) - 1;
      int spins = 0;
      while (gb >= 0) {
        const int64_t gi = gb - int64_t(lane);
        uint64_t w = 0;
        uint32_t f = 2;  // before item 0: an implicit prefix of 0
        if (gi >= 0) {
          w = ld_relaxed(&st[gi]);
          f = status_flag(w, epoch);
        }
        const uint32_t pm = __ballot_sync(kFull, f == 2);
        const uint32_t lim = pm ? uint32_t(__ffs(pm) - 1) : 31u;
        const uint32_t window = lim == 31 ? kFull : ((2u << lim) - 1u);
        if ((__ballot_sync(kFull, f == 0) & window) && !watchdog(lb, spins, 8, tile)) {
          backoff(spins);
          continue;
        }
        excl += warp_sum64((lane <= lim && gi >= 0) ? (w & kValMask) : 0ull);
        if (pm) break;
        gb -= 32;
      }
      done = true;
    }
  }
  if (lane == 0) {
    const uint64_t incl = excl + agg;
    if (tile != 0) st_relaxed(&lb.stat[0][tile], status_word(kFlagPrefix, epoch, incl));
#pragma unroll
    for (int l = 1; l < kLevels; ++l) {
      const uint64_t span = 1ull << (5 * l);
      if (((tile + 1) & (span - 1)) == 0)
        st_relaxed(&lb.stat[l][tile >> (5 * l)], status_word(kFlagPrefix, epoch, incl));
    }
  }
  return excl;
}

}  // namespace spmmm
