// Split-mode rows by expand–sort–compress (ESC), for skewed inputs (C5).
//
// In split mode the non-short rows are computed before k_fused and staged
// (see run_long in spmmm.cu). When a row's products hit mostly distinct
// columns — C5's rows are random, nnz(C) ≈ products — a hash table is pure
// overhead: every product is inserted once and the table must still be sorted
// afterwards. ESC instead
//   expand:   writes every product of the row to shared memory in product
//             order q (q runs through (k, j) in A-entry order, i.e. the
//             reference's k order, kernels.py:163-180): value p_q = fl(a·b)
//             indexed by q, key (column, q);
//   sort:     sorts the keys by (column, q) — equal columns stay in q order;
//   compress: folds each run of equal columns left to right from 0.0 with
//             separately rounded adds (the reference's dense[x] += p) and
//             keeps a run iff its sum != 0.0 (kernels.py:296-298).
// So C[r, x] is bit-identical to the reference, like every other path.
//
//   k_esc_warp:  rows of <= kEscWarpLimit products, one warp per row, keys
//                sorted in registers (bitonic network per width).
//   k_esc_plan:  rows past kEscBlockCap products: cut into column-range parts
//                whose products are staged in q order.
//   k_esc_block: work items of <= kEscBlockCap products (the rows between,
//                whole, and the parts), one block each: one counting pass
//                partitions the keys into column-range buckets of 24-48 keys
//                (so a bucket is a small independent sort), one warp sorts
//                and folds each bucket in registers.
// Keys are 32-bit: (column << 9 | q) in the warp kernel (columns < 2^23,
// checked on the host), (column offset in bucket << qbits | q) in the block
// kernel.
#pragma once

#include "aux_kernels.cuh"
#include "kernels.cuh"

namespace spmmm {

constexpr int kEscWarps = 8;
constexpr int kEscQBits = 9;
constexpr uint32_t kEscWarpLimit = 1u << kEscQBits;  // products per warp row
constexpr int kEscColBits = 32 - kEscQBits;           // columns < 2^23

constexpr int kEscThreads = 512;
#ifndef SPMMM_BUCKET_AVG
#define SPMMM_BUCKET_AVG 48
#endif
constexpr uint32_t kEscBucketAvg = SPMMM_BUCKET_AVG;  // target keys per bucket (measured: 24 and 64 slower)
constexpr uint32_t kEscMaxBuckets = 1024;
// rows of (kEscWarpLimit, kEscBlockCap] products; two blocks per SM. In-bucket
// keys: qb = log2(cap) = 12 bits of q, so a bucket spans <= 2^20 columns
// (nb >= 32 buckets over < 2^23 columns: <= 2^18).
constexpr uint32_t kEscBlockCap = kHugeMin;

__host__ __device__ constexpr size_t esc_warp_smem_bytes() {
  return size_t(kEscWarps) * kEscWarpLimit * (sizeof(uint32_t) + sizeof(double));
}

// ---- register bitonic sort of a run of keys in shared memory -----------------
// E*32 keys, E per lane (element e*32 + lane). E = 1, 2: the fully unrolled
// network (device.cuh); larger E: the stage loops run at run time and only
// the per-element work is unrolled (small code — the sizes vary per row).
template <int JE, int E>
__device__ __forceinline__ void bitonic_reg_exchange(uint32_t (&key)[E], uint32_t k) {
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if ((e & JE) == 0) {
      const int e2 = e | JE;
      const bool up = ((uint32_t(e) << 5) & k) == 0;
      const uint32_t a = key[e], b = key[e2];
      key[e] = keep_minmax(a, b, up);
      key[e2] = keep_minmax(a, b, !up);
    }
  }
}

template <int E>
__device__ __forceinline__ void bitonic_loop(uint32_t (&key)[E]) {
  const uint32_t lane = lane_id();
#pragma unroll 1
  for (uint32_t k = 2; k <= uint32_t(E) * 32u; k <<= 1) {
#pragma unroll 1
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const uint32_t je = j >> 5;
        if constexpr (E > 1) { if (je == 1) bitonic_reg_exchange<1>(key, k); }
        if constexpr (E > 2) { if (je == 2) bitonic_reg_exchange<2>(key, k); }
        if constexpr (E > 4) { if (je == 4) bitonic_reg_exchange<4>(key, k); }
        if constexpr (E > 8) { if (je == 8) bitonic_reg_exchange<8>(key, k); }
      } else {
        const bool lower = (lane & j) == 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint32_t p = __shfl_xor_sync(kFull, key[e], j);
          const bool up = (((uint32_t(e) << 5) | lane) & k) == 0;
          key[e] = keep_minmax(key[e], p, lower == up);
        }
      }
    }
  }
}

template <int E>
__device__ __forceinline__ void sort_run_fixed(uint32_t* kb, uint32_t n) {
  const uint32_t lane = lane_id();
  uint32_t key[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t idx = uint32_t(e) * 32u + lane;
    key[e] = idx < n ? kb[idx] : kEmptyKey;
  }
  if constexpr (E <= 2) bitonic_sort<E>(key);
  else bitonic_loop<E>(key);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t idx = uint32_t(e) * 32u + lane;
    if (idx < n) kb[idx] = key[e];
  }
}

__device__ void warp_sort_smem(uint32_t* k, uint32_t n);

// Sort kb[0..n) ascending in place (warp-collective, n warp-uniform).
__device__ __forceinline__ void sort_run(uint32_t* kb, uint32_t n) {
  if (n <= 32) sort_run_fixed<1>(kb, n);
  else if (n <= 64) sort_run_fixed<2>(kb, n);
  else if (n <= 128) sort_run_fixed<4>(kb, n);
  else if (n <= 256) sort_run_fixed<8>(kb, n);
  else if (n <= 512) sort_run_fixed<16>(kb, n);
  else warp_sort_smem(kb, n);
  __syncwarp();
}

// In-place ascending sort of n keys in shared memory by one warp, for any n
// (buckets that outgrow the register sort: clustered columns). Bitonic with
// the "flip" first step, so every comparator is ascending and the virtual
// +inf padding past n never moves — pairs reaching past n are skipped.
__device__ __noinline__ void warp_sort_smem(uint32_t* k, uint32_t n) {
  const uint32_t lane = lane_id();
  uint32_t np = 1;
  while (np < n) np <<= 1;
  for (uint32_t m = 2; m <= np; m <<= 1) {
    // flip: i pairs with i ^ (m - 1) inside each block of m
    for (uint32_t t = lane; t < np / 2; t += 32) {
      const uint32_t i = (t / (m / 2)) * m + (t % (m / 2));
      const uint32_t pj = i ^ (m - 1);
      if (pj < n) {
        const uint32_t a = k[i], b = k[pj];
        if (a > b) { k[i] = b; k[pj] = a; }
      }
    }
    __syncwarp();
    for (uint32_t j = m / 4; j > 0; j >>= 1) {
      for (uint32_t t = lane; t < np / 2; t += 32) {
        const uint32_t i = 2 * t - (t & (j - 1));
        if (i + j < n) {
          const uint32_t a = k[i], b = k[i + j];
          if (a > b) { k[i] = b; k[i + j] = a; }
        }
      }
      __syncwarp();
    }
  }
}

// ---- the fold over a sorted run of keys --------------------------------------
// keys[0..n) sorted by (column part << qb | q); vals indexed by q. For
// element i of this lane: head = first of its column run; acc = left fold of
// the run from 0.0 in q order. Returns the head flag.
template <bool STATS>
__device__ __forceinline__ bool fold_at(const uint32_t* keys, const double* vals, uint32_t n,
                                        uint32_t i, uint32_t qb, double& acc,
                                        uint32_t& touches) {
  const uint32_t qmask = (1u << qb) - 1u;
  const uint32_t key = keys[i];
  const uint32_t col = key >> qb;
  const bool head = i == 0 || (keys[i - 1] >> qb) != col;
  acc = 0.0;
  if (head) {
    acc = __dadd_rn(0.0, vals[key & qmask]);  // dense[x] == 0.0: a touch
    if (STATS) ++touches;
    for (uint32_t j = i + 1; j < n; ++j) {
      const uint32_t kj = keys[j];
      if ((kj >> qb) != col) break;
      if (STATS && acc == 0.0) ++touches;  // re-touch after an exact zero
      acc = __dadd_rn(acc, vals[kj & qmask]);
    }
  }
  return head;
}

// ---- k_esc_warp ----------------------------------------------------------------
template <bool STATS>
__global__ void __launch_bounds__(kEscWarps * 32, 4) k_esc_warp(const RowsParams p_in) {
  extern __shared__ __align__(16) unsigned char esc_sm[];
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  double* sval = reinterpret_cast<double*>(esc_sm) + warp * kEscWarpLimit;
  uint32_t* skey =
      reinterpret_cast<uint32_t*>(esc_sm + kEscWarps * kEscWarpLimit * sizeof(double)) +
      warp * kEscWarpLimit;
  RowsParams p = p_in;
  p.B.pol = policy_evict_last();
  p.A.pol = policy_evict_first();
  const uint64_t n_sub = *p.n_sub;  // this kernel's own sub-list: no rows to skip
  // rows are taken kEscWarpTake at a time (they are small: one atomic per
  // row was 16% of the kernel's stall samples); lane j keeps row j's index
  constexpr uint32_t kEscWarpTake = 4;
  // the batch: rows taken, next one; lane j holds row j's list index, row,
  // products and entry range (the chain sub -> list -> prod / row_ptr once
  // per batch, not per row)
  uint32_t nb = 0, pos = 0, my_li = 0, my_r = 0, my_P = 0;
  uint64_t my_lo = 0, my_hi = 0;
#pragma unroll 1
  while (true) {
    if (pos == nb) {
      unsigned long long t = 0;
      if (lane == 0) t = atomicAdd(p.ticket, (unsigned long long)kEscWarpTake);
      const uint64_t t0 = __shfl_sync(kFull, t, 0);
      if (t0 >= n_sub) break;
      nb = uint32_t(n_sub - t0 < kEscWarpTake ? n_sub - t0 : kEscWarpTake);
      pos = 0;
      if (lane < nb) {
        my_li = p.sub[t0 + lane];
        my_r = p.list[my_li];
        my_P = p.prod[my_r];
        my_lo = ld_idx(p.A.rp + my_r);
        my_hi = ld_idx(p.A.rp + my_r + 1);
      }
    }
    const uint64_t li = __shfl_sync(kFull, my_li, pos);
    const uint32_t r = __shfl_sync(kFull, my_r, pos);
    const uint32_t P = __shfl_sync(kFull, my_P, pos);
    const uint64_t lo = __shfl_sync(kFull, my_lo, pos), hi = __shfl_sync(kFull, my_hi, pos);
    ++pos;
    // ---- expand: product q -> skey[q] = col << 9 | q, sval[q] = a * b ----
    uint32_t base = 0;
#pragma unroll 1
    for (uint64_t ab = lo; ab < hi; ab += 32) {
      const uint32_t na = uint32_t(hi - ab < 32 ? hi - ab : 32);
      uint64_t bs = 0;
      uint32_t len = 0;
      double av = 0.0;
      if (lane < na) {
        const uint64_t k = ld_idx(p.A.ci + ab + lane, p.A.pol);
        av = ld_val(p.A.v + ab + lane, p.A.pol);
        bs = ld_idx(p.B.rp + k, p.B.pol);
        len = uint32_t(ld_idx(p.B.rp + k + 1, p.B.pol) - bs);
      }
      const uint32_t incl = warp_incl_scan(len);
      const uint32_t excl = incl - len;
      const uint32_t tot = __shfl_sync(kFull, incl, 31);  // lanes past na: len 0
      // four chunks of 32 products per round: their loads are in flight together
#pragma unroll 1
      for (uint32_t c = 0; c < tot; c += 128) {
        uint32_t col[4];
        double bv[4], a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t q = c + 32u * u + lane;
          int i = 0;  // owner: the largest entry with excl <= q
#pragma unroll
          for (int st = 16; st > 0; st >>= 1) {
            const uint32_t ex = __shfl_sync(kFull, excl, i + st);
            if (ex <= q) i += st;
          }
          const uint64_t src = __shfl_sync(kFull, bs, i) + (q - __shfl_sync(kFull, excl, i));
          a[u] = __shfl_sync(kFull, av, i);
          col[u] = 0;
          bv[u] = 0.0;
          if (q < tot) {
            col[u] = uint32_t(ld_idx(p.B.ci + src, p.B.pol));
            bv[u] = ld_val(p.B.v + src, p.B.pol);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t q = c + 32u * u + lane;
          if (q < tot) {
            skey[base + q] = (col[u] << kEscQBits) | (base + q);
            sval[base + q] = __dmul_rn(a[u], bv[u]);
          }
        }
      }
      base += tot;
    }
    __syncwarp();
    // ---- sort (column, q) ----
    sort_run(skey, P);
    // ---- compress: fold runs, drop exact zeros, write out in column order ----
    unsigned long long off = 0;
    if (lane == 0) off = atomicAdd(p.cursor, (unsigned long long)P);  // upper bound
    off = __shfl_sync(kFull, off, 0);
    uint32_t cnt = 0, touches = 0;
#pragma unroll 1
    for (uint32_t i0 = 0; i0 < P; i0 += 32) {
      const uint32_t i = i0 + lane;
      double acc = 0.0;
      bool keep = false;
      if (i < P) keep = fold_at<STATS>(skey, sval, P, i, kEscQBits, acc, touches) && acc != 0.0;
      const uint32_t m = __ballot_sync(kFull, keep);
      if (keep) {
        const uint64_t pos = off + cnt + __popc(m & lanemask_lt());
        __stcs(p.l_ci + pos, skey[i] >> kEscQBits);
        __stcs(p.l_v + pos, acc);
      }
      cnt += __popc(m);
    }
    if (STATS) {
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) touches += __shfl_xor_sync(kFull, touches, d);
    }
    if (lane == 0) {
      p.l_off[li] = off;
      p.l_nnz[li] = cnt;
      if (STATS) {
        p.st_min[r] = skey[0] >> kEscQBits;
        p.st_max[r] = skey[P - 1] >> kEscQBits;
        p.st_touch[r] = touches;
      }
    }
    __syncwarp();
  }
}


// ---- k_esc_dom -------------------------------------------------------------------
// Rows dominated by one long B row (aux_kernels.cuh dom_eligible): the
// dominant entry's L products — a·(B row), columns ascending and distinct, the
// storage contract of formats.py:40-46 — are streamed, 32 per step, straight
// from B to the staged result, and merged on the way with the row's other
// <= kDomRCap products, which are expanded and sorted as in k_esc_warp (key
// col << kDomQBits | qR, qR their product order). A column of the others is folded
// left to right in product order from 0.0; where the dominant row has the
// same column its product joins the fold at its place in the order: after the
// products of earlier A entries (qR < n_before), before the later ones. So
// C[r, x] keeps the reference's k order (kernels.py:163-180), exact zeros are
// dropped (kernels.py:296-298), and a step's outputs are placed by counting:
// a dominant column after the kept columns before it, a merged column after
// the kept dominant columns below it. A B row whose columns do not ascend is
// reported (kCfUnsorted) and the product redone without this kernel.
constexpr int kDomWarps = 8;
#ifndef SPMMM_DOM_BLOCKS
#define SPMMM_DOM_BLOCKS 4
#endif
constexpr int kDomBlocks = SPMMM_DOM_BLOCKS;  // resident blocks per SM
// (2, 3, 4, 6 measured the same on C5 once the long rows start first)
#ifndef SPMMM_DOM_AHEAD
#define SPMMM_DOM_AHEAD 2
#endif
constexpr int kDomAhead = SPMMM_DOM_AHEAD;  // steps of the dominant run in flight
constexpr int kDomQBits = kDomRCap <= 256 ? 8 : 9;
static_assert(kDomRCap <= 512 && kDomQBits <= kEscQBits, "the others: one warp sort, ESC-mode column bits");
static_assert((1u << kDomQBits) >= kDomRCap, "qR bits");

__host__ __device__ constexpr size_t esc_dom_smem_bytes() {
  return size_t(kDomWarps) * kDomRCap * (sizeof(uint32_t) + sizeof(double));
}

template <bool STATS>
__global__ void __launch_bounds__(kDomWarps * 32, kDomBlocks) k_esc_dom(const LongParams p_in) {
  extern __shared__ __align__(16) unsigned char esc_sm[];
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  double* sval = reinterpret_cast<double*>(esc_sm) + warp * kDomRCap;
  uint32_t* skey =
      reinterpret_cast<uint32_t*>(esc_sm + kDomWarps * kDomRCap * sizeof(double)) + warp * kDomRCap;
  LongParams p = p_in;
  p.B.pol = policy_evict_last();
  p.A.pol = policy_evict_first();
  const uint32_t n_rows = uint32_t(*(volatile const unsigned long long*)p.n_sub);
  const uint32_t n_first = p.first ? uint32_t(*(volatile const unsigned long long*)p.n_first) : 0u;
  constexpr uint32_t qmask = (1u << kDomQBits) - 1u;
#pragma unroll 1
  while (true) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(p.ticket, 1ull);
    const uint32_t tr = uint32_t(__shfl_sync(kFull, t, 0));
    // the longer rows first (a 4096-entry dominant run is 128 dependent
    // steps: started last it would be the kernel's tail), then the others
    if (tr >= n_first + n_rows) break;
    const uint32_t li = tr < n_first ? p.first[tr] : p.sub[tr - n_first];
    const uint32_t r = p.list[li];
    const uint32_t P = p.prod[r];
    if (tr >= n_first && P > p.first_min) continue;  // taken above
    const uint64_t lo = ld_idx(p.A.rp + r), hi = ld_idx(p.A.rp + r + 1);
    const uint64_t ed = lo + p.dom[r];  // the dominant entry
    const uint64_t kd = ld_idx(p.A.ci + ed, p.A.pol);
    const double ad = ld_val(p.A.v + ed, p.A.pol);
    const uint64_t bsd = ld_idx(p.B.rp + kd, p.B.pol);
    const uint32_t L = uint32_t(ld_idx(p.B.rp + kd + 1, p.B.pol) - bsd);
    const uint32_t nR = P - L;
    // ---- expand the other entries: skey[qR] = col << kDomQBits | qR, sval[qR] = a * b ----
    uint32_t base = 0, n_before = 0;
#pragma unroll 1
    for (uint64_t ab = lo; ab < hi && nR; ab += 32) {
      const uint32_t na = uint32_t(hi - ab < 32 ? hi - ab : 32);
      uint64_t bs = 0;
      uint32_t len = 0;
      double av = 0.0;
      if (lane < na && ab + lane != ed) {
        const uint64_t k = ld_idx(p.A.ci + ab + lane, p.A.pol);
        av = ld_val(p.A.v + ab + lane, p.A.pol);
        bs = ld_idx(p.B.rp + k, p.B.pol);
        len = uint32_t(ld_idx(p.B.rp + k + 1, p.B.pol) - bs);
      }
      n_before += __reduce_add_sync(kFull, ab + lane < ed ? len : 0u);
      const uint32_t incl = warp_incl_scan(len);
      const uint32_t excl = incl - len;
      const uint32_t tot = __shfl_sync(kFull, incl, 31);
#pragma unroll 1
      for (uint32_t c = 0; c < tot; c += 64) {
        uint32_t col[2];
        double bv[2], a[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t q = c + 32u * u + lane;
          int i = 0;  // owner: the largest entry with excl <= q
#pragma unroll
          for (int st = 16; st > 0; st >>= 1) {
            const uint32_t ex = __shfl_sync(kFull, excl, i + st);
            if (ex <= q) i += st;
          }
          const uint64_t src = __shfl_sync(kFull, bs, i) + (q - __shfl_sync(kFull, excl, i));
          a[u] = __shfl_sync(kFull, av, i);
          col[u] = 0;
          bv[u] = 0.0;
          if (q < tot) {
            col[u] = uint32_t(ld_idx(p.B.ci + src, p.B.pol));
            bv[u] = ld_val(p.B.v + src, p.B.pol);
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t q = c + 32u * u + lane;
          if (q < tot) {
            skey[base + q] = (col[u] << kDomQBits) | (base + q);
            sval[base + q] = __dmul_rn(a[u], bv[u]);
          }
        }
      }
      base += tot;
    }
    __syncwarp();
    if (nR > 1) sort_run(skey, nR);
    unsigned long long off = 0;
    if (lane == 0) off = atomicAdd(p.ctrl + kCtrlStageCursor, (unsigned long long)P);  // upper bound
    off = __shfl_sync(kFull, off, 0);
    // ---- stream the dominant run, merging the others in ----
    uint32_t out = 0, rpos = 0, touches = 0, prev_last = 0;
    bool unsorted = false;
    // kDomAhead steps' loads in flight beside the one being merged
    uint32_t ncol[kDomAhead];
    double nval[kDomAhead];
#pragma unroll
    for (int a = 0; a < kDomAhead; ++a) {
      ncol[a] = 0;
      nval[a] = 0.0;
      if (32u * a + lane < L) {
        ncol[a] = uint32_t(ld_idx(p.B.ci + bsd + 32u * a + lane, p.B.pol));
        nval[a] = ld_val(p.B.v + bsd + 32u * a + lane, p.B.pol);
      }
    }
#pragma unroll 1
    for (uint32_t j0 = 0; j0 < L; j0 += 32) {
      const bool valid = j0 + lane < L;
      const uint32_t cd = valid ? ncol[0] : kEmptyKey;
      const double pd = __dmul_rn(ad, nval[0]);
#pragma unroll
      for (int a = 0; a + 1 < kDomAhead; ++a) {
        ncol[a] = ncol[a + 1];
        nval[a] = nval[a + 1];
      }
      if (j0 + 32u * kDomAhead + lane < L) {
        ncol[kDomAhead - 1] = uint32_t(ld_idx(p.B.ci + bsd + j0 + 32u * kDomAhead + lane, p.B.pol));
        nval[kDomAhead - 1] = ld_val(p.B.v + bsd + j0 + 32u * kDomAhead + lane, p.B.pol);
      }
      uint32_t prevc = __shfl_up_sync(kFull, cd, 1);
      if (lane == 0) prevc = prev_last;
      unsorted |= valid && (j0 + lane) > 0 && cd <= prevc;
      prev_last = __shfl_sync(kFull, cd, 31);
      const bool last = j0 + 32 >= L;
      const uint32_t limit = last ? kEmptyKey : prev_last;  // the others up to this column
      const double accd = __dadd_rn(0.0, pd);
      uint32_t km = __ballot_sync(kFull, valid && accd != 0.0);  // dominant-only columns kept
      uint32_t rbefore = 0, rk = 0, absorbed = 0;
      // the others up to `limit`, 32 per round, one per lane in sorted order
#pragma unroll 1
      while (rpos < nR) {
        const uint32_t x = rpos + lane;
        const uint32_t kx = x < nR ? skey[x] : kEmptyKey;
        const uint32_t cx = kx >> kDomQBits;
        const bool in = x < nR && cx <= limit;
        const uint32_t inm = __ballot_sync(kFull, in);  // (a prefix of the lanes)
        if (!inm) break;
        const bool head = in && (x == 0 || (skey[x - 1] >> kDomQBits) != cx);
        // jd: the step's dominant columns below cx (they ascend; lanes past L hold ~0)
        uint32_t jd = 0;
#pragma unroll
        for (int st = 16; st > 0; st >>= 1) {
          const uint32_t c = __shfl_sync(kFull, cd, jd + st - 1);
          if (c < cx) jd += st;
        }
        const uint32_t cj = __shfl_sync(kFull, cd, jd);
        const double pm = __shfl_sync(kFull, pd, jd);
        if (jd == 31 && cj < cx) jd = 32;
        const bool match = head && jd < 32 && cj == cx;
        double acc = 0.0;
        if (head) {
          bool pend = match;
          uint32_t t2 = x;
          do {
            const uint32_t kt = skey[t2];
            if ((kt >> kDomQBits) != cx) break;
            const uint32_t q = kt & qmask;
            if (pend && q >= n_before) {
              if (STATS && acc == 0.0) ++touches;
              acc = __dadd_rn(acc, pm);
              pend = false;
            }
            if (STATS && acc == 0.0) ++touches;
            acc = __dadd_rn(acc, sval[q]);
            ++t2;
          } while (t2 < nR);
          if (pend) {
            if (STATS && acc == 0.0) ++touches;
            acc = __dadd_rn(acc, pm);
          }
        }
        const uint32_t ab = __reduce_or_sync(kFull, match ? (1u << jd) : 0u);
        km &= ~ab;  // those columns are the merged ones' now
        absorbed |= ab;
        const bool keepx = head && acc != 0.0;
        const uint32_t kmx = __ballot_sync(kFull, keepx);
        if (keepx) {  // after the kept dominant-only columns below it and the kept merged before it
          const uint32_t dbelow = jd >= 32 ? km : (km & ((1u << jd) - 1u));
          const uint64_t pos = off + out + __popc(dbelow) + rk + __popc(kmx & lanemask_lt());
          __stcs(p.l_ci + pos, cx);
          __stcs(p.l_v + pos, acc);
        }
        // a dominant-only column: the kept merged columns below it (this round's:
        // the others' columns ascend over the lanes)
        {
          const uint32_t ce = in ? cx : kEmptyKey;
          uint32_t ix = 0;
#pragma unroll
          for (int st = 16; st > 0; st >>= 1) {
            const uint32_t c = __shfl_sync(kFull, ce, ix + st - 1);
            if (c < cd) ix += st;
          }
          const uint32_t c31 = __shfl_sync(kFull, ce, 31);
          if (ix == 31 && c31 < cd) ix = 32;
          rbefore += __popc(ix >= 32 ? kmx : (kmx & ((1u << ix) - 1u)));
        }
        rk += __popc(kmx);
        const uint32_t cnt = __popc(inm);
        rpos += cnt;
        if (cnt < 32) break;
      }
      if ((km >> lane) & 1u) {
        const uint64_t pos = off + out + __popc(km & lanemask_lt()) + rbefore;
        __stcs(p.l_ci + pos, cd);
        __stcs(p.l_v + pos, accd);
      }
      if (STATS && valid && !((absorbed >> lane) & 1u)) ++touches;
      out += __popc(km) + rk;
    }
    if (__ballot_sync(kFull, unsorted) && lane == 0)
      atomicOr(p.ctrl + kCtrlCfFlags, (unsigned long long)kCfUnsorted);
    if (STATS) touches = __reduce_add_sync(kFull, touches);
    if (lane == 0) {
      p.l_off[li] = off;
      p.l_nnz[li] = out;
      if (STATS) {
        // (touches: summed over the lanes below)
        const uint32_t c0 = uint32_t(ld_idx(p.B.ci + bsd, p.B.pol));
        const uint32_t c1 = uint32_t(ld_idx(p.B.ci + bsd + L - 1, p.B.pol));
        const uint32_t r0 = nR ? skey[0] >> kDomQBits : c0;
        const uint32_t r1 = nR ? skey[nR - 1] >> kDomQBits : c1;
        p.st_min[r] = c0 < r0 ? c0 : r0;
        p.st_max[r] = c1 > r1 ? c1 : r1;
        p.st_touch[r] = touches;
      }
    }
    __syncwarp();
  }
}

// ---- k_esc_plan ------------------------------------------------------------------
// Huge rows (> kHugeMin products): one block per row cuts the row's column
// range [cmin, cmax] into nparts equal ranges (~kPartTarget products each)
// and stages every product, in q order, into its part's scratch region. Each
// part is then an independent k_esc_block work item of <= kEscBlockCap
// products; a column lives in exactly one part, so its fold order is
// untouched. The row's A entries are cut into one contiguous segment per
// warp (segments are contiguous in q); pass 1 counts each warp's products per
// part, a scan over warps gives every (warp, part) its first slot, pass 2
// stages the products (chunks of 32 in q order, ranks in lane order: a
// stable scatter). A row whose busiest part outgrows its region (columns far
// from uniform over the range), or that finds the scratch full, goes to
// k_long instead.
// x / w for x, w < 2^24 (exact in fp32): a float estimate, corrected by one
// step either way (the estimate is off by at most one). ~6 instructions
// against ~25 for an integer division.
__device__ __forceinline__ uint32_t div_small(uint32_t x, uint32_t w, float inv_w) {
  uint32_t q = __float2uint_rz(float(x) * inv_w);
  if (q * w > x) --q;
  else if ((q + 1) * w <= x) ++q;
  return q;
}

#ifndef SPMMM_PART_TARGET
#define SPMMM_PART_TARGET 4096
#endif
constexpr uint32_t kPartTarget = SPMMM_PART_TARGET;  // products per part (1536-3584 measured slower; 4096: -0.6% on C5)
constexpr uint32_t kMaxParts = 64;
constexpr uint32_t kGiantRow = 16384;  // planned first
constexpr int kPlanThreads = 512;

// One warp's segment [e0, e1) of A entries: count (SCATTER = false) or stage
// (SCATTER = true) its products per part. cnt: this warp's per-part counters
// (pass 1) or next free slot (pass 2).
template <bool SCATTER>
__device__ __forceinline__ void plan_segment(const LongParams& pp, uint64_t es, uint64_t ehi,
                                             uint32_t gq, uint32_t qs, uint32_t qe, uint32_t cmn,
                                             uint32_t width, uint32_t region, uint64_t sbase,
                                             uint32_t* cnt) {
  const uint32_t lane = lane_id();
  const float inv_w = 1.0f / float(width);
  // entries from es (whose first product is row product gq) until product qe.
  // Two-deep software pipeline over the chunks of 32 entries: while chunk i's
  // products are loaded and placed, chunk i+1's B.row_ptr pairs and chunk
  // i+2's A entries are in flight (the walk is a chain of dependent loads:
  // A.col_idx -> B.row_ptr -> B.col_idx; unpipelined it is four round trips
  // per ~170 products)
  constexpr uint64_t kNone = ~0ull;
  auto load_a = [&](uint64_t ab, uint64_t& k, double& av) {
    k = kNone;
    av = 0.0;
    if (ab < ehi && ab + lane < ehi) {
      k = ld_idx(pp.A.ci + ab + lane, pp.A.pol);
      if (SCATTER) av = ld_val(pp.A.v + ab + lane, pp.A.pol);
    }
  };
  auto load_b = [&](uint64_t k, uint64_t& bs, uint32_t& len) {
    bs = 0;
    len = 0;
    if (k != kNone) {
      bs = ld_idx(pp.B.rp + k, pp.B.pol);
      len = uint32_t(ld_idx(pp.B.rp + k + 1, pp.B.pol) - bs);
    }
  };
  uint64_t k1, k2, bs_n;
  uint32_t len_n;
  double av_n, av2;
  load_a(es, k1, av_n);          // chunk 0's entries
  load_b(k1, bs_n, len_n);       // chunk 0's B rows
  load_a(es + 32, k2, av2);      // chunk 1's entries
#pragma unroll 1
  for (uint64_t ab = es; ab < ehi && gq < qe; ab += 32) {
    const uint64_t bs = bs_n;
    const uint32_t len = len_n;
    const double av = av_n;
    av_n = av2;
    load_b(k2, bs_n, len_n);          // chunk i+1's B rows
    load_a(ab + 64, k2, av2);         // chunk i+2's entries
    const uint32_t incl = warp_incl_scan(len);
    const uint32_t excl = incl - len;
    const uint32_t tot = __shfl_sync(kFull, incl, 31);
    // this segment's products of the group: local q in [qlo, qhi)
    const uint32_t qlo = qs > gq ? qs - gq : 0u;
    const uint32_t qhi = qe - gq < tot ? qe - gq : tot;
    gq += tot;
#pragma unroll 1
    for (uint32_t c = qlo; c < qhi; c += 128) {
      uint32_t col[4];
      double bv[4], a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t q = c + 32u * u + lane;
        int i = 0;
#pragma unroll
        for (int st = 16; st > 0; st >>= 1) {
          const uint32_t ex = __shfl_sync(kFull, excl, i + st);
          if (ex <= q) i += st;
        }
        const uint64_t src = __shfl_sync(kFull, bs, i) + (q - __shfl_sync(kFull, excl, i));
        a[u] = SCATTER ? __shfl_sync(kFull, av, i) : 0.0;
        col[u] = 0;
        bv[u] = 0.0;
        if (q < qhi) {
          col[u] = uint32_t(ld_idx(pp.B.ci + src, pp.B.pol));
          if (SCATTER) bv[u] = ld_val(pp.B.v + src, pp.B.pol);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t q = c + 32u * u + lane;
        const bool act = q < qhi;
        const uint32_t part = act ? div_small(col[u] - cmn, width, inv_w) : kEmptyKey;
        const uint32_t peers = __match_any_sync(kFull, part);
        const uint32_t leader = __ffs(peers) - 1;
        uint32_t old = 0;
        if (act && lane == leader) {
          old = cnt[part];
          cnt[part] = old + __popc(peers);
        }
        if (SCATTER) {
          const uint32_t pos = __shfl_sync(kFull, old, leader) + __popc(peers & lanemask_lt());
          if (act) {
            const uint64_t slot = sbase + uint64_t(part) * region + pos;
            __stcg(pp.scr_col + slot, col[u]);
            __stcg(pp.scr_val + slot, __dmul_rn(a[u], bv[u]));
          }
        }
        __syncwarp();
      }
    }
  }
}

template <bool STATS>
__global__ void __launch_bounds__(kPlanThreads, 2) k_esc_plan(LongParams p) {
  constexpr int NW = kPlanThreads / 32;
  __shared__ uint32_t s_cnt[NW][kMaxParts];
  __shared__ uint32_t s_h, s_min, s_max, s_over;
  __shared__ unsigned long long s_sbase;
  __shared__ uint64_t s_seg_e[NW];
  __shared__ uint32_t s_seg_q[NW];
  __shared__ uint32_t s_scan[NW + 1];
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = lane_id();
  LongParams pp = p;
  pp.B.pol = policy_evict_last();
  pp.A.pol = policy_evict_first();
  const uint32_t n_huge = uint32_t(p.ctrl[kCtrlHugeRows]);
#pragma unroll 1
  while (true) {
    if (tid == 0) {
      s_h = uint32_t(atomicAdd(p.ctrl + kCtrlPlanTicket, 1ull));
      s_min = kEmptyKey;
      s_max = 0;
      s_over = 0;
    }
    __syncthreads();
    // two sweeps over the list: rows past kGiantRow products first, so the
    // longest rows do not start last and set the kernel's tail
    const uint32_t t = s_h;
    if (t >= 2 * n_huge) break;
    const uint32_t h = t < n_huge ? t : t - n_huge;
    const uint32_t li = p.huge[h];
    const uint32_t r = p.list[li];
    const uint32_t P = p.prod[r];
    if ((t < n_huge) != (P > kGiantRow)) {
      __syncthreads();  // everyone has read s_h before the loop head rewrites it
      continue;
    }
    const uint64_t lo = ld_idx(pp.A.rp + r), hi = ld_idx(pp.A.rp + r + 1);
    // column range of the row (first and last column of every B row), and
    // where each warp's equal share of the row's products starts: the entry
    // holding product qs_w = w*P/NW and that entry's first product
    uint32_t cmn = kEmptyKey, cmx = 0, run = 0;
#pragma unroll 1
    for (uint64_t e0 = lo; e0 < hi; e0 += kPlanThreads) {
      const uint64_t e = e0 + tid;
      uint64_t bs = 0, be = 0;
      if (e < hi) {
        const uint64_t k = ld_idx(pp.A.ci + e, pp.A.pol);
        bs = ld_idx(pp.B.rp + k, pp.B.pol);
        be = ld_idx(pp.B.rp + k + 1, pp.B.pol);
      }
      if (be > bs) {
        const uint32_t c0 = uint32_t(ld_idx(pp.B.ci + bs, pp.B.pol));
        const uint32_t c1 = uint32_t(ld_idx(pp.B.ci + be - 1, pp.B.pol));
        cmn = c0 < cmn ? c0 : cmn;
        cmx = c1 > cmx ? c1 : cmx;
      }
      const uint32_t len = uint32_t(be - bs);
      uint32_t total;
      const uint32_t ex = run + block_excl_scan<kPlanThreads>(len, s_scan, total);
      if (len) {
#pragma unroll 1
        for (int w = 0; w < NW; ++w) {
          const uint32_t qs = uint32_t(uint64_t(w) * P / NW);
          if (ex <= qs && qs < ex + len) {
            s_seg_e[w] = e;
            s_seg_q[w] = ex;
          }
        }
      }
      run += total;
    }
    cmn = __reduce_min_sync(kFull, cmn);
    cmx = __reduce_max_sync(kFull, cmx);
    if (lane == 0) {
      atomicMin(&s_min, cmn);
      atomicMax(&s_max, cmx);
    }
    for (uint32_t j = lane; j < kMaxParts; j += 32) s_cnt[warp][j] = 0;
    __syncthreads();
    cmn = s_min;
    cmx = s_max;
    uint32_t nparts = (P + kPartTarget - 1) / kPartTarget;
    nparts = nparts < kMaxParts ? nparts : kMaxParts;
    const uint32_t width = (cmx - cmn) / nparts + 1;
    // region per part: 5/4 of the mean part plus slack, at most a block's cap
    uint32_t region = P / nparts + P / nparts / 4 + 64;
    region = region < kEscBlockCap ? region : kEscBlockCap;
    // this warp's segment of A entries
    // this warp's products [qs, qe) of the row, starting in entry es
    const uint32_t qs = uint32_t(uint64_t(warp) * P / NW);
    const uint32_t qe = uint32_t(uint64_t(warp + 1) * P / NW);
    const uint64_t es = s_seg_e[warp];
    const uint32_t gq = s_seg_q[warp];
    plan_segment<false>(pp, es, hi, gq, qs, qe, cmn, width, region, 0, s_cnt[warp]);
    __syncthreads();
    // per part: exclusive scan over warps -> each warp's first slot
    if (tid < nparts) {
      uint32_t run = 0;
      for (int w = 0; w < NW; ++w) {
        const uint32_t c = s_cnt[w][tid];
        s_cnt[w][tid] = run;
        run += c;
      }
      if (run > region) atomicOr(&s_over, 1u);
    }
    __syncthreads();
    if (tid == 0) {
      uint64_t sb = 0;
      if (!s_over) {
        sb = atomicAdd(p.ctrl + kCtrlScrCursor, (unsigned long long)nparts * region);
        if (sb + uint64_t(nparts) * region > p.scr_cap) s_over = 1;
      }
      s_sbase = sb;
      if (s_over) {
        p.ovf[atomicAdd(p.ctrl + kCtrlOvfRows, 1ull)] = li;
        p.row_np[h] = 0;
      }
    }
    __syncthreads();
    const bool over = s_over != 0;
    __syncthreads();  // everyone has read s_over before the loop head resets it
    if (over) continue;
    const uint64_t sbase = s_sbase;
    plan_segment<true>(pp, es, hi, gq, qs, qe, cmn, width, region, sbase, s_cnt[warp]);
    __syncthreads();
    // after pass 2 the last warp's cursors are the part totals
    if (warp == 0) {
      uint32_t nz = 0;
      for (uint32_t j0 = 0; j0 < nparts; j0 += 32) {
        const uint32_t j = j0 + lane;
        nz += __popc(__ballot_sync(kFull, j < nparts && s_cnt[NW - 1][j] > 0));
      }
      unsigned long long pbase = 0;
      if (lane == 0) pbase = atomicAdd(p.ctrl + kCtrlParts, (unsigned long long)nz);
      pbase = __shfl_sync(kFull, pbase, 0);
      uint32_t rank = 0;
      for (uint32_t j0 = 0; j0 < nparts; j0 += 32) {
        const uint32_t j = j0 + lane;
        const uint32_t tot = j < nparts ? s_cnt[NW - 1][j] : 0u;
        const uint32_t m = __ballot_sync(kFull, tot > 0);
        if (tot > 0) {
          PartDesc d;
          d.li = li;
          d.cnt = tot;
          d.off = sbase + uint64_t(j) * region;
          p.parts[pbase + rank + __popc(m & lanemask_lt())] = d;
        }
        rank += __popc(m);
      }
      if (lane == 0) {
        p.row_pbase[h] = uint32_t(pbase);
        p.row_np[h] = nz;
        p.l_nnz[li] = 0;
        if (STATS) {
          p.st_min[r] = cmn;
          p.st_max[r] = cmx;
          p.st_touch[r] = 0;
        }
      }
    }
    __syncthreads();
  }
}

// ---- k_esc_block ---------------------------------------------------------------

__host__ __device__ constexpr size_t esc_block_smem_bytes(uint32_t cap) {
  return size_t(cap) * (sizeof(double) + 2 * sizeof(uint32_t)) +
         size_t(kEscMaxBuckets) * 3 * sizeof(uint32_t);
}

// Rows of (kEscWarpLimit, cap] products (LongParams.sub), one block per row.
template <bool STATS>
__global__ void __launch_bounds__(kEscThreads, 2) k_esc_block(LongParams p, uint32_t cap) {
  constexpr int NT = kEscThreads;
  extern __shared__ __align__(16) unsigned char esc_sm[];
  double* sval = reinterpret_cast<double*>(esc_sm);               // [cap] by q
  uint32_t* scol = reinterpret_cast<uint32_t*>(sval + cap);       // [cap] column by q
  uint32_t* bkey = scol + cap;                                    // [cap] bucketed keys
  uint32_t* hist = bkey + cap;                                    // [kEscMaxBuckets]
  uint32_t* start = hist + kEscMaxBuckets;                        // bucket starts
  uint32_t* kept = start + kEscMaxBuckets;                        // kept per bucket, then out offsets
  __shared__ uint32_t s_excl[NT + 1];
  __shared__ uint64_t s_bs[NT];
  __shared__ double s_av[NT];
  __shared__ uint32_t s_scan[NT / 32 + 1];
  __shared__ uint32_t s_min, s_max, s_touch, s_bt;
  __shared__ unsigned long long s_off;
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  uint32_t qb = 1;
  while ((1u << qb) < cap) ++qb;
  LongParams pp = p;
  pp.B.pol = policy_evict_last();
  pp.A.pol = policy_evict_first();
  const uint32_t n_sub = uint32_t(*(volatile const unsigned long long*)p.n_sub);
  const uint32_t n_parts =
      p.parts ? uint32_t(*(volatile const unsigned long long*)(p.ctrl + kCtrlParts)) : 0u;
  // A work item's descriptor — ticket -> sub-list / part -> list -> products and
  // entry range, a chain of four dependent loads — is fetched by thread 0 one
  // item ahead, while the block sorts the current item's buckets (the items
  // are independent; at the top of an item the chain was ~2.5 us with all 16
  // warps waiting on it, ~50 times per block).
  struct ItemDesc {
    uint32_t t_row, li, r, P;
    unsigned long long scr, lo, hi;
  };
  __shared__ ItemDesc s_next;
  auto fetch_item = [&]() {  // thread 0
    ItemDesc d;
    d.t_row = uint32_t(atomicAdd(p.ticket, 1ull));
    d.li = d.r = d.P = 0;
    d.scr = d.lo = d.hi = 0;
    if (d.t_row < n_sub + n_parts) {
      if (d.t_row >= n_sub) {
        const PartDesc pd = p.parts[d.t_row - n_sub];
        d.li = pd.li;
        d.P = pd.cnt;
        d.scr = pd.off;
        d.r = p.list[d.li];
      } else {
        d.li = p.sub[d.t_row];
        d.r = p.list[d.li];
        d.P = p.prod[d.r];
        d.lo = ld_idx(pp.A.rp + d.r);
        d.hi = ld_idx(pp.A.rp + d.r + 1);
      }
    }
    s_next = d;
  };
  if (tid == 0) fetch_item();
#pragma unroll 1
  while (true) {
    if (tid == 0) {
      s_min = kEmptyKey;
      s_max = 0;
      s_touch = 0;
    }
    __syncthreads();
    const ItemDesc cur = s_next;
    const uint32_t t_row = cur.t_row;
    if (t_row >= n_sub + n_parts) break;
    // work item: a whole mid row, or one column-range part of a huge row
    const bool is_part = t_row >= n_sub;
    const uint32_t li = cur.li, P = cur.P, r = cur.r;
    const uint64_t scr = cur.scr, lo = cur.lo, hi = cur.hi;
    uint32_t base = 0, cmn = kEmptyKey, cmx = 0;
    // part: its products are staged in q order by k_esc_plan
    for (uint32_t i = tid; is_part && i < P; i += NT) {
      const uint32_t c = __ldcs(p.scr_col + scr + i);
      scol[i] = c;
      sval[i] = __ldcs(p.scr_val + scr + i);
      cmn = c < cmn ? c : cmn;
      cmx = c > cmx ? c : cmx;
    }
    // ---- expand (whole rows) ----
#pragma unroll 1
    for (uint64_t ab = lo; ab < hi; ab += NT) {
      const uint64_t e = ab + tid;
      uint32_t len = 0;
      uint64_t bs = 0;
      double av = 0.0;
      if (e < hi) {
        const uint64_t k = ld_idx(pp.A.ci + e, pp.A.pol);
        av = ld_val(pp.A.v + e, pp.A.pol);
        bs = ld_idx(pp.B.rp + k, pp.B.pol);
        len = uint32_t(ld_idx(pp.B.rp + k + 1, pp.B.pol) - bs);
      }
      uint32_t total;
      const uint32_t ex = block_excl_scan<NT>(len, s_scan, total);
      s_excl[tid] = ex;
      s_bs[tid] = bs;
      s_av[tid] = av;
      if (tid == 0) s_excl[NT] = total;
      __syncthreads();
#pragma unroll 1
      for (uint32_t c = 0; c < total; c += 4 * NT) {
        uint32_t col[4];
        double bv[4], a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t q = c + uint32_t(u) * NT + tid;
          col[u] = 0;
          bv[u] = 0.0;
          a[u] = 0.0;
          if (q < total) {
            int i = 0;
#pragma unroll
            for (int st = NT / 2; st > 0; st >>= 1)
              if (s_excl[i + st] <= q) i += st;
            const uint64_t src = s_bs[i] + (q - s_excl[i]);
            a[u] = s_av[i];
            col[u] = uint32_t(ld_idx(pp.B.ci + src, pp.B.pol));
            bv[u] = ld_val(pp.B.v + src, pp.B.pol);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t q = c + uint32_t(u) * NT + tid;
          if (q < total) {
            scol[base + q] = col[u];
            sval[base + q] = __dmul_rn(a[u], bv[u]);
            cmn = col[u] < cmn ? col[u] : cmn;
            cmx = col[u] > cmx ? col[u] : cmx;
          }
        }
      }
      base += total;
      __syncthreads();  // s_excl / s_bs / s_av reused by the next A chunk
    }
    cmn = __reduce_min_sync(kFull, cmn);
    cmx = __reduce_max_sync(kFull, cmx);
    if (lane == 0) {
      atomicMin(&s_min, cmn);
      atomicMax(&s_max, cmx);
    }
    // buckets: nb (power of two) column ranges of 2^sh columns from cmin,
    // ~kEscBucketAvg keys each; in-bucket key = offset << qb | q
    // nb: the smallest power of two >= max(2, P / kEscBucketAvg), at most kEscMaxBuckets
    const uint32_t want = (P + kEscBucketAvg - 1) / kEscBucketAvg;
    uint32_t nb = want <= 2 ? 2u : 1u << (32 - __clz(want - 1));
    nb = nb < kEscMaxBuckets ? nb : kEscMaxBuckets;
    for (uint32_t b = tid; b < nb; b += NT) hist[b] = 0;
    if (tid == 0) s_bt = NT / 32;  // buckets below were taken statically
    __syncthreads();
    const uint32_t cmin = s_min, range = s_max - cmin;
    // the smallest sh with (range >> sh) < nb: bits(range) - log2(nb), if positive
    const int shs = (32 - __clz(range)) - (31 - __clz(nb));
    const uint32_t sh = shs > 0 ? uint32_t(shs) : 0u;
    // ---- partition: histogram, bucket starts, scatter ----
    for (uint32_t q = tid; q < P; q += NT) atomicAdd(hist + ((scol[q] - cmin) >> sh), 1u);
    __syncthreads();
    {
      const uint32_t h0 = 2 * tid < nb ? hist[2 * tid] : 0u;
      const uint32_t h1 = 2 * tid + 1 < nb ? hist[2 * tid + 1] : 0u;
      uint32_t tot;
      const uint32_t ex = block_excl_scan<NT>(h0 + h1, s_scan, tot);
      if (2 * tid < nb) {
        start[2 * tid] = ex;
        kept[2 * tid] = ex;  // scatter cursors for now
      }
      if (2 * tid + 1 < nb) {
        start[2 * tid + 1] = ex + h0;
        kept[2 * tid + 1] = ex + h0;
      }
    }
    __syncthreads();
    const uint32_t omask = (1u << sh) - 1u;
    for (uint32_t q = tid; q < P; q += NT) {
      const uint32_t rel = scol[q] - cmin;
      const uint32_t pos = atomicAdd(kept + (rel >> sh), 1u);
      bkey[pos] = ((rel & omask) << qb) | q;
    }
    __syncthreads();
    // ---- per bucket (one warp): sort, fold; heads' sums go to sval[q] ----
    // (every thread has read s_next; thread 0 fetches the next item's now)
    if (tid == 0) fetch_item();
    uint32_t touches = 0;
#pragma unroll 1
    // buckets taken dynamically (sort costs vary with the bucket size)
    for (uint32_t b = warp;;) {
      if (b >= nb) break;
      const uint32_t sz = hist[b];
      uint32_t* kb = bkey + start[b];
      if (sz > 1) sort_run(kb, sz);
      uint32_t cnt = 0;
      for (uint32_t i0 = 0; i0 < sz; i0 += 32) {
        const uint32_t i = i0 + lane;
        double acc = 0.0;
        bool head = false;
        if (i < sz) {
          head = fold_at<STATS>(kb, sval, sz, i, qb, acc, touches);
          if (head) sval[kb[i] & ((1u << qb) - 1u)] = acc;  // only this head reads it again
        }
        cnt += __popc(__ballot_sync(kFull, head && acc != 0.0));
      }
      if (lane == 0) kept[b] = cnt;
      uint32_t nb2 = 0;
      if (lane == 0) nb2 = atomicAdd(&s_bt, 1u);
      b = __shfl_sync(kFull, nb2, 0);
    }
    __syncthreads();
    // ---- output offsets per bucket, then the row ----
    uint32_t n_out;
    {
      const uint32_t k0 = 2 * tid < nb ? kept[2 * tid] : 0u;
      const uint32_t k1 = 2 * tid + 1 < nb ? kept[2 * tid + 1] : 0u;
      const uint32_t ex = block_excl_scan<NT>(k0 + k1, s_scan, n_out);
      if (STATS) {
        uint32_t t = touches;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) t += __shfl_xor_sync(kFull, t, d);
        if (lane == 0 && t) atomicAdd(&s_touch, t);
      }
      if (2 * tid < nb) kept[2 * tid] = ex;
      if (2 * tid + 1 < nb) kept[2 * tid + 1] = ex + k0;
    }
    if (tid == 0) {
      s_off = n_out ? atomicAdd(p.ctrl + kCtrlStageCursor, (unsigned long long)n_out) : 0ull;
      if (is_part) {
        p.part_off[t_row - n_sub] = s_off;
        p.part_nnz[t_row - n_sub] = n_out;
        atomicAdd(p.l_nnz + li, n_out);  // the row's total (zeroed by k_esc_plan)
      } else {
        p.l_off[li] = s_off;
        p.l_nnz[li] = n_out;
      }
    }
    __syncthreads();
    const uint64_t off = s_off;
#pragma unroll 1
    for (uint32_t b = warp; b < nb; b += NT / 32) {
      const uint32_t sz = hist[b];
      const uint32_t* kb = bkey + start[b];
      const uint32_t blo = cmin + (b << sh);
      uint32_t o = kept[b];
      for (uint32_t i0 = 0; i0 < sz; i0 += 32) {
        const uint32_t i = i0 + lane;
        bool keep = false;
        uint32_t key = 0;
        double v = 0.0;
        if (i < sz) {
          key = kb[i];
          const bool head = i == 0 || (kb[i - 1] >> qb) != (key >> qb);
          v = sval[key & ((1u << qb) - 1u)];
          keep = head && v != 0.0;
        }
        const uint32_t m = __ballot_sync(kFull, keep);
        if (keep) {
          const uint64_t pos = off + o + __popc(m & lanemask_lt());
          __stcs(p.l_ci + pos, blo + (key >> qb));
          __stcs(p.l_v + pos, v);
        }
        o += __popc(m);
      }
    }
    if (STATS && tid == 0) {
      if (is_part) {  // range set by k_esc_plan
        atomicAdd(p.st_touch + r, s_touch);
      } else {
        p.st_min[r] = cmin;
        p.st_max[r] = s_max;
        p.st_touch[r] = s_touch;
      }
    }
    __syncthreads();
  }
}

}  // namespace spmmm
