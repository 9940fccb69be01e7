// Device-side building blocks for the sm_100a spMMM pipeline: warp scans, the
// register bitonic sort, the decoupled look-back, and the per-row
// accumulation paths (short / medium). Kernels live in kernels.cuh.
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
        constexpr int dummy = 0;
        (void)dummy;
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
// Decoupled look-back over tiles (single pass exclusive scan of tile nnz).
// Status word: [63:62] flag (0 invalid, 1 aggregate, 2 inclusive prefix),
// [61:46] epoch (per call, so the array never needs clearing), [45:0] value.
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagPrefix = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 46) - 1;

// Warp-collective (call with all 32 lanes). Publishes `agg` for `tile` and
// returns the exclusive prefix of all earlier tiles.
__device__ __forceinline__ uint64_t lookback(uint64_t* status, uint64_t tile, uint64_t agg,
                                             uint32_t epoch) {
  const uint32_t lane = lane_id();
  const uint64_t ep = uint64_t(epoch & 0xffffu) << 46;
  if (tile == 0) {
    if (lane == 0) st_relaxed(&status[0], kFlagPrefix | ep | agg);
    return 0;
  }
  if (lane == 0) st_relaxed(&status[tile], kFlagAgg | ep | agg);
  uint64_t excl = 0;
  int64_t base = int64_t(tile) - 1;
  while (true) {
    const int64_t idx = base - int64_t(lane);
    uint64_t w = 0;
    uint32_t flag = 2;  // before tile 0: an implicit prefix of 0
    uint32_t pmask, lim, inval;
    int spins = 0;
    while (true) {
      if (idx >= 0) {
        w = ld_relaxed(&status[idx]);
        flag = ((w >> 46) & 0xffffu) == (epoch & 0xffffu) ? uint32_t(w >> 62) : 0u;
      }
      pmask = __ballot_sync(kFull, flag == 2);
      lim = pmask ? uint32_t(__ffs(pmask) - 1) : 31u;
      const uint32_t window = lim == 31 ? kFull : ((2u << lim) - 1u);
      inval = __ballot_sync(kFull, flag == 0) & window;
      if (!inval) break;
      if (++spins > 4) __nanosleep(64);
    }
    const uint64_t val = (lane <= lim && idx >= 0) ? (w & kValMask) : 0ull;
    excl += warp_sum64(val);
    if (pmask) break;
    base -= 32;
  }
  if (lane == 0) st_relaxed(&status[tile], kFlagPrefix | ep | (excl + agg));
  return excl;
}

// ---------------------------------------------------------------------------
// Short rows: <= 32 products, <= 32 A entries. One product per lane,
// expand -> bitonic sort by (column, product index) -> segmented left fold.
//
// Product q of the row is entry j of B row k where k runs over the A entries
// in ascending column order; lane order therefore is the reference's k order
// (kernels.py:167-171), and sorting by (col, lane) keeps each column's
// products in that order for the fold.
struct ShortOut {
  uint32_t col;
  uint32_t rank;
  double val;
  bool keep;
};

template <bool WIDE, bool STATS>
__device__ __forceinline__ uint32_t short_row(const DevCsr& A, const DevCsr& B, uint64_t lo,
                                              uint32_t na, ShortOut& out, uint32_t& smin,
                                              uint32_t& smax, uint32_t& stouch) {
  using K = typename std::conditional<WIDE, unsigned long long, uint32_t>::type;
  const uint32_t lane = lane_id();
  uint32_t len = 0;
  uint64_t bs = 0;
  double av = 0.0;
  if (lane < na) {
    const uint64_t k = ld_idx(A.ci + lo + lane);
    av = ld_val(A.v + lo + lane);
    bs = ld_idx(B.rp + k);
    len = uint32_t(ld_idx(B.rp + k + 1) - bs);
  }
  const uint32_t incl = warp_incl_scan(len);
  const uint32_t excl = incl - len;
  const uint32_t tot = __shfl_sync(kFull, incl, 31);
  // entry owning product `lane`: largest i with excl_i <= lane
  int i = 0;
#pragma unroll
  for (int st = 16; st > 0; st >>= 1) {
    const uint32_t ex = __shfl_sync(kFull, excl, i + st);
    if (ex <= lane) i += st;
  }
  const uint64_t bsrc = __shfl_sync(kFull, bs, i);
  const double a = __shfl_sync(kFull, av, i);
  const uint32_t j = lane - __shfl_sync(kFull, excl, i);
  const bool valid = lane < tot;
  uint32_t col = 0;
  double p = 0.0;
  if (valid) {
    col = uint32_t(ld_idx(B.ci + bsrc + j));
    p = __dmul_rn(a, ld_val(B.v + bsrc + j));
  }
  K key[1];
  key[0] = valid ? ((K(col) << 5) | K(lane)) : ~K(0);
  bitonic_sort<1>(key);
  col = uint32_t(key[0] >> 5);
  const uint32_t src = uint32_t(key[0]) & 31u;
  const double v = __shfl_sync(kFull, p, src);
  const uint32_t prev = __shfl_up_sync(kFull, col, 1);
  const bool head = valid && (lane == 0 || prev != col);
  double acc = v;
  uint32_t touches = 1;
  for (int d = 1; d < 32; ++d) {
    const uint32_t c = __shfl_down_sync(kFull, col, d);
    const double t = __shfl_down_sync(kFull, v, d);
    const bool cond = head && (lane + uint32_t(d) < tot) && c == col;
    if (!__any_sync(kFull, cond)) break;
    if (cond) {
      if (STATS && acc == 0.0) ++touches;  // re-touch after a transient zero
      acc = __dadd_rn(acc, t);
    }
  }
  const bool keep = head && (acc != 0.0);  // kernels.py:296 drops exact zeros
  const uint32_t km = __ballot_sync(kFull, keep);
  out.col = col;
  out.val = acc;
  out.keep = keep;
  out.rank = __popc(km & lanemask_lt());
  if (STATS) {
    smin = __shfl_sync(kFull, col, 0);
    smax = __shfl_sync(kFull, col, (tot - 1) & 31u);
    uint32_t t = head ? touches : 0u;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) t += __shfl_xor_sync(kFull, t, d);
    stouch = t;
  }
  return __popc(km);
}

// ---------------------------------------------------------------------------
// Medium rows: warp + open-addressing table of T slots in shared memory.
// Products are streamed in chunks of up to 32 in (k, j) order. A chunk is cut
// at B-row boundaries whenever possible, so most chunks hold one B row whose
// columns are distinct: all lanes update the table in one step. Chunks that
// span several B rows are applied in rounds where each column's products go
// in ascending product order (rank among equal columns via match_any), which
// keeps every table entry a left fold in reference order.

template <int T>
__device__ __forceinline__ uint32_t table_hash(uint32_t col) {
  constexpr int kLog = __builtin_ctz(T);
  return (col * 0x9E3779B1u) >> (32 - kLog);
}

template <int T, bool STATS>
__device__ __forceinline__ void table_apply(uint32_t* keys, double* vals, uint32_t col,
                                            double p, uint32_t& touches) {
  volatile uint32_t* vk = keys;
  uint32_t h = table_hash<T>(col);
  bool fresh = false;
  while (true) {
    const uint32_t k = vk[h];
    if (k == col) break;
    if (k == kEmptyKey) {
      const uint32_t old = atomicCAS(keys + h, kEmptyKey, col);
      if (old == kEmptyKey) { fresh = true; break; }
      if (old == col) break;
    }
    h = (h + 1) & (T - 1);
  }
  volatile double* vv = vals;
  const double cur = fresh ? 0.0 : vv[h];  // fresh slot == dense[x] == 0.0
  if (STATS && cur == 0.0) ++touches;
  vv[h] = __dadd_rn(cur, p);
}

template <int T, bool STATS>
__device__ __forceinline__ void medium_accumulate(const DevCsr& A, const DevCsr& B, uint64_t lo,
                                                  uint64_t hi, uint32_t* keys, double* vals,
                                                  uint32_t& touches) {
  const uint32_t lane = lane_id();
  for (uint64_t abase = lo; abase < hi; abase += 32) {
    const uint64_t e = abase + lane;
    uint32_t len = 0;
    uint64_t bs = 0;
    double av = 0.0;
    if (e < hi) {
      const uint64_t k = ld_idx(A.ci + e);
      av = ld_val(A.v + e);
      bs = ld_idx(B.rp + k);
      len = uint32_t(ld_idx(B.rp + k + 1) - bs);
    }
    const uint32_t incl = warp_incl_scan(len);
    const uint32_t excl = incl - len;
    const uint32_t gtot = __shfl_sync(kFull, incl, 31);
    uint32_t cs = 0;
    while (cs < gtot) {
      const uint32_t lim = cs + 32;
      const uint32_t bm = __ballot_sync(kFull, incl > cs && incl <= lim);
      const uint32_t ce =
          bm ? __shfl_sync(kFull, incl, 31 - __clz(bm)) : (lim < gtot ? lim : gtot);
      const uint32_t q = cs + lane;
      const bool act = q < ce;
      int i = 0;
#pragma unroll
      for (int st = 16; st > 0; st >>= 1) {
        const uint32_t ex = __shfl_sync(kFull, excl, i + st);
        if (ex <= q) i += st;
      }
      const uint64_t bsrc = __shfl_sync(kFull, bs, i);
      const double a = __shfl_sync(kFull, av, i);
      const uint32_t j = q - __shfl_sync(kFull, excl, i);
      uint32_t col = kEmptyKey;
      double p = 0.0;
      if (act) {
        col = uint32_t(ld_idx(B.ci + bsrc + j));
        p = __dmul_rn(a, ld_val(B.v + bsrc + j));
      }
      const int i_first = __shfl_sync(kFull, i, 0);
      const int i_last = __shfl_sync(kFull, i, (ce - cs - 1) & 31u);
      if (i_first == i_last) {
        if (act) table_apply<T, STATS>(keys, vals, col, p, touches);
        __syncwarp();
      } else {
        const uint32_t am = __ballot_sync(kFull, act);
        const uint32_t peers = __match_any_sync(kFull, col) & am;
        const uint32_t rank = __popc(peers & lanemask_lt());
        const uint32_t rounds = __reduce_max_sync(kFull, act ? rank : 0u) + 1u;
        for (uint32_t rr = 0; rr < rounds; ++rr) {
          if (act && rank == rr) table_apply<T, STATS>(keys, vals, col, p, touches);
          __syncwarp();
        }
      }
      cs = ce;
    }
  }
}

// After accumulation: compact the occupied nonzero slots to the front of the
// table (in place) and return their count. STATS: min/max over every occupied
// slot, zero-valued ones included (they were touched: kernels.py:175-178).
template <int T, bool STATS>
__device__ __forceinline__ uint32_t medium_compact(uint32_t* keys, double* vals, uint32_t& smin,
                                                   uint32_t& smax) {
  const uint32_t lane = lane_id();
  uint32_t cnt = 0;
  uint32_t mn = kEmptyKey, mx = 0;
#pragma unroll 4
  for (uint32_t s0 = 0; s0 < uint32_t(T); s0 += 32) {
    const uint32_t s = s0 + lane;
    const uint32_t k = keys[s];
    const double v = vals[s];
    const bool occ = k != kEmptyKey;
    const bool keep = occ && (v != 0.0);
    if (STATS && occ) {
      mn = k < mn ? k : mn;
      mx = k > mx ? k : mx;
    }
    const uint32_t m = __ballot_sync(kFull, keep);
    __syncwarp();
    if (keep) {
      const uint32_t pos = cnt + __popc(m & lanemask_lt());
      keys[pos] = k;
      vals[pos] = v;
    }
    cnt += __popc(m);
    __syncwarp();
  }
  if (STATS) {
    smin = __reduce_min_sync(kFull, mn);
    smax = __reduce_max_sync(kFull, mx);
  }
  return cnt;
}

}  // namespace spmmm
