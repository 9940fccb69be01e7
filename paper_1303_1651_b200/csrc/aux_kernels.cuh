// Count, long-row-listing and long-row kernels (used only by spmmm.cu).
#pragma once

#include <cooperative_groups.h>

#include "device.cuh"
#include "rows.cuh"

namespace spmmm {

// ctrl words (device, zeroed before every multiply)
constexpr int kCtrlCfWords = 32;
enum Ctrl : int {
  kCtrlTotal = 0,     // Σ products (estimate_nnz)
  kCtrlMaxProd = 1,   // max products of one row
  kCtrlNeedTable = 2, // some row needs the medium/long machinery
  kCtrlError = 3,     // bit flags: 1 A.row_ptr, 2 A.col_idx range, 4 B.row_ptr, 8 row too long
  kCtrlLongRows = 4,  // number of rows listed by k_collect
  kCtrlStageCursor = 5,
  kCtrlTicket = 6,    // k_fused's dynamic tile counter
  kCtrlFault = 7,     // k_fused watchdog report
  kCtrlNonShort = 8,  // rows that are not short (> 32 products or > 32 A entries)
  kCtrlLongTicket = 9,  // k_long's dynamic row counter
  kCtrlRowsTicket = 10, // k_rows's dynamic row counter
  kCtrlLongSmemTicket = 11, // k_long_smem's dynamic row counter
  kCtrlMidRows = 12,    // sub-list: rows for k_long_smem (one block per row)
  kCtrlHugeRows = 13,   // sub-list: rows for the cluster variant (8 blocks per row)
  kCtrlOvfRows = 14,    // sub-list: rows the cluster variant handed to k_long
  kCtrlHugeTicket = 15, // cluster variant's dynamic row counter; ESC mode: k_esc_dom's
  kCtrlCopyTickets = 16, // k_copy_long: block rows
  kCtrlDomBigRows = 17, // sub-list: k_esc_dom's rows past the block-copy limit
  kCtrlBMaxLen = 18,    // longest B row referenced by A (entries)
  kCtrlKMinInv = 19,    // ~(smallest column of A), 0 if A has no entries
  kCtrlKMax1 = 20,      // largest column of A + 1, 0 if none
  kCtrlNnz = 21,        // nnz(C), written by k_fused's last tile
  kCtrlHugeProducts = 22, // Σ products of rows past kHugeMin (k_esc_plan scratch size)
  kCtrlParts = 23,      // column-range parts written by k_esc_plan
  kCtrlPlanTicket = 24, // k_esc_plan's dynamic row counter
  kCtrlScrCursor = 25,  // k_esc_plan's scratch allocator (slots)
  kCtrlCfFlags = 26,    // count-free path: kCf* bits, then [27] longest A row, [28] longest B row
  kCtrlDone = 29,       // count-free path: k_fused warps finished (the last one reports)
  kCtrlCfEll = 30,      // count-free path: B's referenced rows were packed into ELL records
  kCtrlDomRows = 31,    // sub-list: rows dominated by one long B row (k_esc_dom)
  // (words past 31 belong to the counted path only: the count-free path's
  // last warp reports and clears words 0..31, kCtrlCfWords)
  kCtrlWarpRows = 32,   // sub-list: rows for k_esc_warp (one warp per row)
  kCtrlCountTicket = 33, // k_count's dynamic row-chunk counter
  kCtrlWords = 40
};

// rows past this many products are split into column-range parts in ESC mode
// (esc.cuh); k_count sums their products for the host
#ifndef SPMMM_HUGE_MIN
#define SPMMM_HUGE_MIN 5120
#endif
constexpr uint32_t kHugeMin = SPMMM_HUGE_MIN;

// Rows with a dominant B row (skewed inputs: an A row that hits a long B
// row — 40% of C5's products sit in such rows): the longest B row of the row
// has L >= kDomMinRun entries and at most kDomRCap of the row's P products
// come from the other entries (one warp sorts those). Such a row is the
// dominant run — already sorted, distinct columns — merged with the sorted
// others (esc.cuh k_esc_dom) instead of P keys sorted from scratch. k_count
// records the dominant entry (its offset in the A row; the first of the
// longest).
// (measured on C5, final kernels: others <= 512 / run >= 64 / any share of the
// row, the rule below, 2.82 ms; run >= 32: 2.84, >= 96: 2.84, >= 128: 2.86;
// others <= 384: 2.88; others <= 256 and at least half of the row — the rule
// before k_esc_dom took its long rows first and k_esc_block fetched its items
// ahead: 2.90. -DSPMMM_DOM_HALF asks for half of the row again.)
#ifndef SPMMM_DOM_RCAP
#define SPMMM_DOM_RCAP 512
#endif
#ifndef SPMMM_DOM_MINRUN
#define SPMMM_DOM_MINRUN 64
#endif
constexpr uint32_t kDomRCap = SPMMM_DOM_RCAP;
constexpr uint32_t kDomMinRun = SPMMM_DOM_MINRUN;
constexpr uint32_t kNoDom = 0xffffffffu;
__host__ __device__ inline bool dom_eligible(uint64_t P, uint64_t L) {
#ifdef SPMMM_DOM_HALF
  if (2 * L < P) return false;
#endif
  return L >= kDomMinRun && P - L <= kDomRCap;
}

// Split-mode row lists, built by k_count itself on the assumption that the
// product will run in split mode with the ESC kernels (the host knows only
// after reading k_count's totals; when it decides otherwise it resets the
// counters and k_collect lists the rows by that mode's limits). Saves the
// k_collect pass on skewed inputs (C5: 0.08 ms).
struct RowLists {
  uint32_t* list;       // every non-short row (null: k_count builds no lists)
  uint32_t* lmap;       // row -> its index in list
  uint32_t* mid_list;   // rows past mid_min products (one block each)
  uint32_t* huge_list;  // rows past huge_min products (column-range parts)
  uint32_t* dom_list;   // dominated rows (k_esc_dom), whatever their size
  uint32_t* dom_big;    // ... those past mid_min (block copy)
  uint32_t* warp_list;  // the other rows up to mid_min products (one warp each)
  uint32_t mid_min, huge_min;
};

// Append this warp's long rows (lane: row r, pr products, dominant entry dv)
// to the lists; every lane of the warp calls it.
__device__ __forceinline__ void list_rows(const RowLists& L, unsigned long long* ctrl, bool is_long,
                                          uint64_t r, uint32_t pr, uint32_t dv) {
  const uint32_t m = __ballot_sync(kFull, is_long);
  if (!m) return;
  const bool is_dom = is_long && dv != 0xffffffffu;
  const bool is_warp = is_long && !is_dom && pr <= L.mid_min;
  const uint32_t md = __ballot_sync(kFull, is_dom);
  const uint32_t mw = __ballot_sync(kFull, is_warp);
  uint32_t base = 0, dbase = 0, wbase = 0;
  if (lane_id() == 0) {
    base = uint32_t(atomicAdd(ctrl + kCtrlLongRows, (unsigned long long)__popc(m)));
    if (md) dbase = uint32_t(atomicAdd(ctrl + kCtrlDomRows, (unsigned long long)__popc(md)));
    if (mw) wbase = uint32_t(atomicAdd(ctrl + kCtrlWarpRows, (unsigned long long)__popc(mw)));
  }
  base = __shfl_sync(kFull, base, 0);
  dbase = __shfl_sync(kFull, dbase, 0);
  wbase = __shfl_sync(kFull, wbase, 0);
  if (is_long) {
    const uint32_t idx = base + __popc(m & lanemask_lt());
    L.list[idx] = uint32_t(r);
    L.lmap[r] = idx;
    // rows per computing kernel (the others are few: plain atomics)
    if (is_dom) {
      L.dom_list[dbase + __popc(md & lanemask_lt())] = idx;
      if (pr > L.mid_min) L.dom_big[atomicAdd(ctrl + kCtrlDomBigRows, 1ull)] = idx;
    } else if (pr > L.huge_min) {
      L.huge_list[atomicAdd(ctrl + kCtrlHugeRows, 1ull)] = idx;
    } else if (pr > L.mid_min) {
      L.mid_list[atomicAdd(ctrl + kCtrlMidRows, 1ull)] = idx;
    } else {
      L.warp_list[wbase + __popc(mw & lanemask_lt())] = idx;
    }
  }
}

// (64 registers, 4 blocks per SM: with the per-row dominant-entry tracking the
// kernel took 90 and ran 2; C5 0.30 -> 0.22 ms, C4 0.13 -> 0.10)
#ifndef SPMMM_COUNT_BLOCKS
#define SPMMM_COUNT_BLOCKS 4
#endif
__global__ void __launch_bounds__(256, SPMMM_COUNT_BLOCKS) k_count(DevCsr A, DevCsr B, uint32_t* __restrict__ prod,
                                               unsigned long long* __restrict__ ctrl,
                                               unsigned long long* __restrict__ zero,
                                               uint64_t nzero, uint4* __restrict__ ell_self,
                                               uint4* __restrict__ ell_all,
                                               uint32_t* __restrict__ dom, const RowLists lists) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nzero;
       i += uint64_t(gridDim.x) * blockDim.x)
    zero[i] = 0;
  const uint32_t lane = lane_id();
  uint64_t tot = 0, mx = 0, nonshort = 0, bmax = 0, kmin = ~0ull, kmax1 = 0, huge = 0;
  uint32_t need = 0, err = 0;
  constexpr uint64_t kSerial = 32;  // rows up to this many entries: one thread
  // chunks of 32 rows, taken dynamically: with a static assignment the warps
  // that met the long rows of a skewed input were the kernel's tail (23% of
  // the stall samples sat at the block's final barrier on C5)
  while (true) {
    unsigned long long chunk = 0;
    if (lane == 0) chunk = atomicAdd(ctrl + kCtrlCountTicket, 1ull);
    const uint64_t base = __shfl_sync(kFull, chunk, 0) * 32;
    if (base >= A.rows) break;
    const uint64_t r = base + lane;
    uint64_t lo = 0, hi = 0;
    if (r < A.rows) {
      lo = ld_idx(A.rp + r);
      hi = ld_idx(A.rp + r + 1);
      if (hi < lo || hi > A.nnz) {
        err |= 1u;
        hi = lo;
      }
    }
    uint64_t p = 0;
    uint64_t rl = 0;   // the row's longest B row and the (first) entry holding it
    uint32_t re = 0;
    // rows past kSerial entries: the whole warp, one row at a time. When only
    // a few rows of the warp pass 8 entries (skewed inputs), those go to the
    // warp too, so 31 short rows do not wait on one lane's 30-entry loop.
    const uint32_t few = __popc(__ballot_sync(kFull, hi - lo > 8));
    const bool serial = hi - lo <= (few <= 4 ? 8 : kSerial);
    if (serial) {
      // four entries per round: their two dependent load levels overlap
      for (uint64_t e0 = lo; e0 < hi; e0 += 4) {
        uint64_t k[4], b0[4], b1[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) k[u] = e0 + u < hi ? ld_idx(A.ci + e0 + u) : ~0ull;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          b0[u] = b1[u] = 0;
          if (k[u] != ~0ull && k[u] < B.rows) {
            b0[u] = ld_idx(B.rp + k[u]);
            b1[u] = ld_idx(B.rp + k[u] + 1);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (k[u] == ~0ull) continue;
          if (k[u] >= B.rows) { err |= 2u; continue; }
          if (b1[u] < b0[u] || b1[u] > B.nnz) { err |= 4u; continue; }
          const uint64_t l = b1[u] - b0[u];
          p += l;
          if (l > rl) {
            rl = l;
            re = uint32_t(e0 + u - lo);
          }
          bmax = l > bmax ? l : bmax;
          kmin = k[u] < kmin ? k[u] : kmin;
          kmax1 = k[u] + 1 > kmax1 ? k[u] + 1 : kmax1;
        }
      }
    }
    // long A rows: the whole warp, one row at a time
    uint32_t big = __ballot_sync(kFull, !serial);
    while (big) {
      const uint32_t src = __ffs(big) - 1;
      big &= big - 1;
      const uint64_t blo = __shfl_sync(kFull, lo, src), bhi = __shfl_sync(kFull, hi, src);
      uint64_t s = 0, sl = 0;
      uint32_t se = 0;
      // four entries per lane per round: a 4096-entry row is 32 rounds of two
      // dependent loads, not 128 (such rows set the kernel's tail)
      for (uint64_t e0 = blo + lane; e0 < bhi; e0 += 128) {
        uint64_t k[4], b0[4], b1[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint64_t e = e0 + 32u * u;
          k[u] = e < bhi ? ld_idx(A.ci + e) : ~0ull;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          b0[u] = b1[u] = 0;
          if (k[u] != ~0ull && k[u] < B.rows) {
            b0[u] = ld_idx(B.rp + k[u]);
            b1[u] = ld_idx(B.rp + k[u] + 1);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (k[u] == ~0ull) continue;
          if (k[u] >= B.rows) { err |= 2u; continue; }
          if (b1[u] < b0[u] || b1[u] > B.nnz) { err |= 4u; continue; }
          const uint64_t l = b1[u] - b0[u];
          s += l;
          if (l > sl) {  // (a lane's entries ascend: its first longest)
            sl = l;
            se = uint32_t(e0 + 32u * u - blo);
          }
          bmax = l > bmax ? l : bmax;
          kmin = k[u] < kmin ? k[u] : kmin;
          kmax1 = k[u] + 1 > kmax1 ? k[u] + 1 : kmax1;
        }
      }
      s = warp_sum64(s);
      // longest, then lowest entry
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        const uint64_t ol = __shfl_xor_sync(kFull, sl, d);
        const uint32_t oe = __shfl_xor_sync(kFull, se, d);
        if (ol > sl || (ol == sl && oe < se)) {
          sl = ol;
          se = oe;
        }
      }
      if (lane == src) {
        p = s;
        rl = sl;
        re = se;
      }
    }
    // C = A·A: row r of A is row r of B — its ELL record is written here, from
    // entries this lane has just read, instead of by a k_pack_ell pass
    if (ell_self && r < A.rows && hi - lo <= uint64_t(kEllSlots)) pack_ell_record(A, r, lo, hi, ell_self);
    uint32_t dv = kNoDom;
    if (r < A.rows) {
      if (p > 0x7fffffffull) err |= 8u;
      prod[r] = uint32_t(p > 0x7fffffffull ? 0x7fffffffull : p);
      if (p <= 0x7fffffffull && dom_eligible(p, rl)) dv = re;
      if (dom) dom[r] = dv;
      tot += p;
      huge += p > kHugeMin ? p : 0;
      mx = p > mx ? p : mx;
      if (p > 32 || (p > 0 && hi - lo > 32)) {
        need = 1;
        ++nonshort;
      }
    }
    if (lists.list)
      list_rows(lists, ctrl, r < A.rows && (p > 32 || (p > 0 && hi - lo > 32)), r,
                uint32_t(p > 0x7fffffffull ? 0x7fffffffull : p), dv);
  }
  // speculative ELL copy of every B row (A != B, B rows of ~kEllSlots
  // entries): the bandwidth-bound copy interleaves with the latency-bound
  // count instead of following it; used only if k_count's results call for ELL
  if (ell_all) {
    for (uint64_t rb = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; rb < B.rows;
         rb += uint64_t(gridDim.x) * blockDim.x) {
      uint64_t bh = ld_idx(B.rp + rb + 1);
      bh = bh < B.nnz ? bh : B.nnz;
      uint64_t bl = ld_idx(B.rp + rb);
      bl = bl < bh ? bl : bh;
      pack_ell_record(B, rb, bl, bh, ell_all);
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const uint64_t ob = __shfl_xor_sync(kFull, bmax, d);
    bmax = ob > bmax ? ob : bmax;
    const uint64_t ok0 = __shfl_xor_sync(kFull, kmin, d);
    kmin = ok0 < kmin ? ok0 : kmin;
    const uint64_t ok1 = __shfl_xor_sync(kFull, kmax1, d);
    kmax1 = ok1 > kmax1 ? ok1 : kmax1;
    tot += __shfl_xor_sync(kFull, tot, d);
    huge += __shfl_xor_sync(kFull, huge, d);
    nonshort += __shfl_xor_sync(kFull, nonshort, d);
    const uint64_t o = __shfl_xor_sync(kFull, mx, d);
    mx = o > mx ? o : mx;
    need |= __shfl_xor_sync(kFull, need, d);
    err |= __shfl_xor_sync(kFull, err, d);
  }
  // block-level combine, then one set of atomics per block (same-address
  // atomics from every warp serialise in L2)
  __shared__ unsigned long long s_red[9][8];
  const uint32_t warp = threadIdx.x >> 5;
  if (lane == 0) {
    s_red[0][warp] = tot;
    s_red[1][warp] = nonshort;
    s_red[2][warp] = mx;
    s_red[3][warp] = bmax;
    s_red[4][warp] = ~kmin;
    s_red[5][warp] = kmax1;
    s_red[6][warp] = need;
    s_red[7][warp] = err;
    s_red[8][warp] = huge;
  }
  __syncthreads();
  if (threadIdx.x < 9) {
    const uint32_t f = threadIdx.x;
    unsigned long long x = 0;
    for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
      const unsigned long long y = s_red[f][w];
      x = (f < 2 || f == 8) ? x + y : (f < 6 ? (y > x ? y : x) : (x | y));
    }
    if (x) {
      switch (f) {
        case 0: atomicAdd(ctrl + kCtrlTotal, x); break;
        case 1: atomicAdd(ctrl + kCtrlNonShort, x); break;
        case 2: atomicMax(ctrl + kCtrlMaxProd, x); break;
        case 3: atomicMax(ctrl + kCtrlBMaxLen, x); break;
        case 4: atomicMax(ctrl + kCtrlKMinInv, x); break;
        case 5: atomicMax(ctrl + kCtrlKMax1, x); break;
        case 6: atomicOr(ctrl + kCtrlNeedTable, 1ull); break;
        case 8: atomicAdd(ctrl + kCtrlHugeProducts, x); break;
        default: atomicOr(ctrl + kCtrlError, x); break;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// ELL copy of B (rows <= kEllSlots entries): one 64-byte record per row, written
// with four 16-byte stores (consecutive threads, consecutive records).
// Whether the short variant reads B through ELL records, from k_count's
// results — evaluated identically by k_pack_ell (device) and the host.
__host__ __device__ inline bool ell_wanted(const unsigned long long* w, uint64_t rows) {
  const uint64_t total = w[kCtrlTotal], bmax = w[kCtrlBMaxLen];
  const uint64_t k0 = ~w[kCtrlKMinInv], k1 = w[kCtrlKMax1];
  const bool need = w[kCtrlNeedTable] != 0;
  const bool split = need && w[kCtrlNonShort] * 4 <= rows;
  if (need && !split) return false;  // medium variant
  if (bmax > uint64_t(kEllSlots) || k1 <= k0) return false;
  // worth it when the referenced B rows (>= total / longest) are not much
  // fewer than the rows the copy spans
  return 10 * (total / (bmax ? bmax : 1)) >= 7 * (k1 - k0);
}

// ---------------------------------------------------------------------------
// The count-free path. When every row of C is short by construction — A
// rows of <= kEllEntries entries and B rows of <= kEllSlots (the ELL flavour:
// B read through its ELL records), or A rows of na entries and B rows of nb
// with na <= 32 and na·nb <= 32 (the CSR flavour, e.g. a row block of A
// against a whole B) — the fused kernel needs neither the per-row product
// counts nor the host decisions k_count feeds. This pass only measures the
// longest A and B rows, checks both row_ptr arrays, packs B's ELL records
// (ELL flavour) and zeroes the look-back counters; k_fused follows it on the
// stream with no host round trip, checks the verdict itself (cf_applies) and
// returns at once when it does not apply. The host then runs the counted
// path, which also yields the reference's exact error for bad input.
// (CfFlags and cf_applies: rows.cuh, beside the ELL layout)

// The count-free path's first pass as a kernel (small products run the same
// pass, prep_pass in rows.cuh, inside k_fused: the PREP instantiations; this
// kernel keeps its own copy of the body — routed through the shared device
// function it compiled 17% slower on C2, 0.118 -> 0.138 ms, measured).
// MODE 0, C = A·A (A square, its rows are B's rows): one pass over the rows
// measures both and checks A's columns while packing them as B's records.
// MODE 1, A spans most of B: A's rows and columns, then every B row (checked,
// measured, packed). MODE 2, A a row block of a larger matrix: A only — its
// rows, its columns against B.rows and their range [kmin, kmax] — and
// k_prep_b takes the B rows in that range.
template <int MODE>
__global__ void __launch_bounds__(256) k_prep(DevCsr A, DevCsr B,
                                              unsigned long long* __restrict__ ctrl,
                                              unsigned long long* __restrict__ zero,
                                              uint64_t nzero, uint4* __restrict__ ell) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const uint64_t t0 = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (uint64_t i = t0; i < nzero; i += stride) zero[i] = 0;
  unsigned f = 0;
  unsigned long long ma = 0, mb = 0, kmin = ~0ull, kmax1 = 0;
  if (MODE != 0) {
    for (uint64_t r = t0; r < A.rows; r += stride) {
      const uint64_t lo = ld_idx(A.rp + r), hi = ld_idx(A.rp + r + 1);
      if (hi < lo || hi > A.nnz) f |= kCfBadA;
      else ma = hi - lo > ma ? hi - lo : ma;
    }
    // every column of A's rows must name a row of B (k_fused trusts them);
    // coalesced over the entries of the rows' span
    uint64_t e0 = ld_idx(A.rp), e1 = ld_idx(A.rp + A.rows);
    e1 = e1 < A.nnz ? e1 : A.nnz;
    for (uint64_t e = e0 + t0; e < e1; e += stride) {
      const uint64_t k = ld_idx(A.ci + e);
      if (k >= B.rows) f |= kCfBadCol;
      if (MODE == 2) {
        kmin = k < kmin ? k : kmin;
        kmax1 = k + 1 > kmax1 ? k + 1 : kmax1;
      }
    }
  }
  if (MODE != 2) {
    for (uint64_t r = t0; r < B.rows; r += stride) {
      const uint64_t lo = ld_idx(B.rp + r), hi = ld_idx(B.rp + r + 1);
      if (hi < lo || hi > B.nnz) {
        f |= MODE == 0 ? (kCfBadB | kCfBadA) : kCfBadB;
        continue;
      }
      mb = hi - lo > mb ? hi - lo : mb;
      if (MODE == 0)
        for (uint64_t e = lo; e < hi; ++e)
          if (ld_idx(B.ci + e) >= B.rows) f |= kCfBadCol;  // (L1 hits: the record's loads)
      if (ell) pack_ell_record(B, r, lo, hi, ell);  // (longer rows: truncated, never read)
    }
    if (MODE == 0) ma = mb;
  }
  f = __reduce_or_sync(kFull, f);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const unsigned long long oa = __shfl_xor_sync(kFull, ma, d), ob = __shfl_xor_sync(kFull, mb, d);
    ma = oa > ma ? oa : ma;
    mb = ob > mb ? ob : mb;
    if (MODE == 2) {
      const unsigned long long o0 = __shfl_xor_sync(kFull, kmin, d);
      const unsigned long long o1 = __shfl_xor_sync(kFull, kmax1, d);
      kmin = o0 < kmin ? o0 : kmin;
      kmax1 = o1 > kmax1 ? o1 : kmax1;
    }
  }
  if (lane_id() == 0) {
    if (f) atomicOr(ctrl + kCtrlCfFlags, (unsigned long long)f);
    if (ma) atomicMax(ctrl + kCtrlCfFlags + 1, ma);
    if (mb) atomicMax(ctrl + kCtrlCfFlags + 2, mb);
    if (MODE == 2 && kmax1) {
      atomicMax(ctrl + kCtrlKMinInv, ~kmin);
      atomicMax(ctrl + kCtrlKMax1, kmax1);
    }
    if (MODE != 2 && ell && blockIdx.x == 0 && threadIdx.x == 0) ctrl[kCtrlCfEll] = 1;
  }
}

// The B rows A references, [kmin, kmax] from k_prep: checked, measured and
// (when A references most of them: at least 7/10 of the range, by A's entry
// count) packed into ELL records — the counted path's rule (ell_wanted).
// Rows outside the range are never read, like k_count leaves them unchecked.
__global__ void __launch_bounds__(256, 8) k_prep_b(DevCsr A, DevCsr B,
                                                unsigned long long* __restrict__ ctrl,
                                                uint4* __restrict__ ell) {
  const uint64_t k0 = ~ctrl[kCtrlKMinInv], k1 = ctrl[kCtrlKMax1];
  if (k1 <= k0) return;  // A has no entries
  uint64_t e0 = ld_idx(A.rp), e1 = ld_idx(A.rp + A.rows);
  e1 = e1 < A.nnz ? e1 : A.nnz;
  const bool pack = ell != nullptr && e1 > e0 && 10 * (e1 - e0) >= 7 * (k1 - k0);
  if (pack && blockIdx.x == 0 && threadIdx.x == 0) ctrl[kCtrlCfEll] = 1;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  unsigned f = 0;
  unsigned long long mb = 0;
  for (uint64_t r = k0 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < k1; r += stride) {
    const uint64_t lo = ld_idx(B.rp + r), hi = ld_idx(B.rp + r + 1);
    if (hi < lo || hi > B.nnz) {
      f |= kCfBadB;
      continue;
    }
    mb = hi - lo > mb ? hi - lo : mb;
    if (pack) pack_ell_record(B, r, lo, hi, ell);
  }
  f = __reduce_or_sync(kFull, f);
  mb = __reduce_max_sync(kFull, uint32_t(mb > 0xffffffffull ? 0xffffffffull : mb));
  if (lane_id() == 0) {
    if (f) atomicOr(ctrl + kCtrlCfFlags, (unsigned long long)f);
    if (mb) atomicMax(ctrl + kCtrlCfFlags + 2, mb);
  }
}

// Only the rows A references ([kmin, kmax], from k_count) are packed; rows in
// between that are longer than a record are truncated and never read. Runs
// right behind k_count, while the host reads k_count's results back.
__global__ void __launch_bounds__(256) k_pack_ell(DevCsr B, uint64_t a_rows,
                                                  const unsigned long long* __restrict__ ctrl,
                                                  uint4* __restrict__ ell) {
  if (!ell_wanted(ctrl, a_rows)) return;
  const uint64_t r0 = ~ctrl[kCtrlKMinInv], r1 = ctrl[kCtrlKMax1];
  for (uint64_t r = r0 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < r1;
       r += uint64_t(gridDim.x) * blockDim.x) {
    // unreferenced rows are not validated by k_count: clamp to the arrays
    uint64_t hi = ld_idx(B.rp + r + 1);
    hi = hi < B.nnz ? hi : B.nnz;
    uint64_t lo = ld_idx(B.rp + r);
    lo = lo < hi ? lo : hi;
    pack_ell_record(B, r, lo, hi, ell);
  }
}

// ---------------------------------------------------------------------------
// K2: list the long rows (warp-aggregated append; order is irrelevant).
__global__ void __launch_bounds__(256) k_collect(DevCsr A, const uint32_t* __restrict__ prod,
                                                 uint32_t medium_limit,
                                                 unsigned long long* __restrict__ ctrl,
                                                 const uint32_t* __restrict__ dom,
                                                 const RowLists lists) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const uint64_t start = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  // warp-uniform trip count so the ballots are full-warp
  const uint64_t span = (A.rows + stride - 1) / stride;
  for (uint64_t it = 0; it < span; ++it) {
    const uint64_t r = start + it * stride;
    bool is_long = false;
    uint32_t pr = 0;
    if (r < A.rows) {
      const uint64_t na = ld_idx(A.rp + r + 1) - ld_idx(A.rp + r);
      pr = prod[r];
      is_long = classify(pr, na, medium_limit) == kRowLong;
    }
    list_rows(lists, ctrl, is_long, r, pr, (is_long && dom) ? dom[r] : kNoDom);
  }
}

// ---------------------------------------------------------------------------
// K3: long rows, one 512-thread block per row, workspace in global memory
// (hash table + column bitmap per resident block, restored after each row).
//
// Order: products are enumerated in chunks of 512 in (k, j) order. Within a
// chunk, products hitting the same column are applied in rounds: each round
// every pending product bids its global product index with atomicMin on its
// slot's owner word; the lowest index wins and adds, so each column sees its
// products in ascending order — the reference's left fold (kernels.py:167-174).
// Output order: the bitmap over [min col, max col] is scanned in order, so the
// row comes out sorted without a comparison sort (the paper's BruteForce-bool
// lookup idea, kernels.py:106-113 / 216-227, on the GPU).
constexpr int kLongThreads = 512;

struct PartDesc {  // one column range of a huge row, products staged in q order
  uint32_t li;     // list index of the row
  uint32_t cnt;    // products in the range
  uint64_t off;    // first scratch slot
};

struct LongParams {
  DevCsr A, B;
  const uint32_t* prod;
  const uint32_t* list;
  unsigned long long* ctrl;
  uint64_t* l_off;
  uint32_t* l_nnz;
  uint32_t* l_ci;  // staged columns (u32: columns < 2^32; widened by k_copy_long)
  double* l_v;
  uint32_t* ws_keys;   // [grid][slots]
  double* ws_vals;     // [grid][slots]
  uint32_t* ws_owner;  // [grid][slots]
  uint32_t* ws_bits;   // [grid][words + swords]: column bitmap, then its summary
                       // (bit w of the summary: bitmap word w is nonzero)
  uint64_t ws_slots;   // power of two >= 2 * max products of a long row
  uint64_t ws_words;   // ceil(cols / 32)
  uint64_t ws_swords;  // ceil(ws_words / 32)
  const uint32_t* sub;                // this kernel's rows, as indices into list
  const unsigned long long* n_sub;    // their count
  unsigned long long* ticket;         // dynamic row counter
  uint32_t* ovf;                      // cluster variant: rows handed on to k_long
  const uint32_t* dom;                // k_esc_dom: the dominant entry of each of its rows
  const uint32_t* first;              // k_esc_dom: its rows past first_min products (taken first)
  const unsigned long long* n_first;
  uint32_t first_min;
  // ESC mode (esc.cuh): column-range parts of the huge rows
  struct PartDesc* parts;             // [max parts]
  uint64_t* part_off;                 // staging offset per part
  uint32_t* part_nnz;                 // entries per part
  uint32_t* row_pbase;                // per huge-list position: first part
  uint32_t* row_np;                   // per huge-list position: parts (0: whole row staged)
  const uint32_t* huge;               // huge sub-list
  uint32_t* scr_col;                  // part scratch: columns
  double* scr_val;                    // part scratch: products
  uint64_t scr_cap;                   // scratch slots
  uint64_t max_parts;
  uint32_t* st_min;
  uint32_t* st_max;
  uint32_t* st_touch;
};

// full-avalanche 32-bit mixer (the table is masked to its low bits)
__device__ __forceinline__ uint32_t long_hash(uint32_t x, uint32_t mask) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x & mask;
}

__device__ __forceinline__ uint32_t long_probe(const uint32_t* keys, uint32_t col, uint32_t mask) {
  uint32_t h = long_hash(col, mask);
  while (__ldcg(keys + h) != col) h = (h + 1) & mask;
  return h;
}

template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* scratch, uint32_t& total) {
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t incl = warp_incl_scan(x);
  if (lane == 31) scratch[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = lane < uint32_t(NT / 32) ? scratch[lane] : 0u;
    const uint32_t wi = warp_incl_scan(w);
    if (lane < uint32_t(NT / 32)) scratch[lane] = wi - w;
    if (lane == 31) scratch[NT / 32] = wi;
  }
  __syncthreads();
  const uint32_t res = scratch[warp] + incl - x;
  total = scratch[NT / 32];
  __syncthreads();
  return res;
}

template <bool STATS>
__global__ void __launch_bounds__(kLongThreads) k_long(LongParams p) {
  constexpr int NT = kLongThreads;
  constexpr int kDupSlots = 4 * NT;  // per-chunk duplicate detector
  __shared__ uint32_t s_excl[NT + 1];
  __shared__ uint64_t s_bs[NT];
  __shared__ double s_av[NT];
  __shared__ uint32_t s_scan[NT / 32 + 1];
  __shared__ uint32_t s_dup[kDupSlots];
  __shared__ uint32_t s_min, s_max, s_touch, s_zero;
  __shared__ unsigned long long s_off;

  const uint32_t tid = threadIdx.x;
  uint32_t* keys = p.ws_keys + uint64_t(blockIdx.x) * p.ws_slots;
  double* vals = p.ws_vals + uint64_t(blockIdx.x) * p.ws_slots;
  uint32_t* owner = p.ws_owner + uint64_t(blockIdx.x) * p.ws_slots;
  uint32_t* bits = p.ws_bits + uint64_t(blockIdx.x) * (p.ws_words + p.ws_swords);
  uint32_t* sum = bits + p.ws_words;
  const uint32_t n_sub = uint32_t(*(volatile const unsigned long long*)p.n_sub);
  for (uint32_t s = tid; s < uint32_t(kDupSlots); s += NT) s_dup[s] = kEmptyKey;

  // rows are taken dynamically: their costs are heavy-tailed
  __shared__ uint32_t s_li;
  while (true) {
    if (tid == 0) s_li = uint32_t(atomicAdd(p.ticket, 1ull));
    __syncthreads();
    const uint32_t t = s_li;
    __syncthreads();
    if (t >= n_sub) break;
    const uint32_t li = p.sub[t];
    const uint32_t r = p.list[li];
    const uint32_t prod = p.prod[r];
    const uint64_t lo = ld_idx(p.A.rp + r), hi = ld_idx(p.A.rp + r + 1);
    uint32_t tsize = 64;
    while (uint64_t(tsize) < 2ull * prod && uint64_t(tsize) < p.ws_slots) tsize <<= 1;
    const uint32_t mask = tsize - 1;
    if (tid == 0) { s_min = kEmptyKey; s_max = 0; s_touch = 0; s_zero = 0; }
    __syncthreads();
    uint32_t touches = 0;
    uint32_t seq_base = 0;
    for (uint64_t abase = lo; abase < hi; abase += NT) {
      const uint64_t e = abase + tid;
      uint32_t len = 0;
      uint64_t bs = 0;
      double av = 0.0;
      if (e < hi) {
        const uint64_t k = ld_idx(p.A.ci + e);
        av = ld_val(p.A.v + e);
        bs = ld_idx(p.B.rp + k);
        len = uint32_t(ld_idx(p.B.rp + k + 1) - bs);
      }
      uint32_t total;
      const uint32_t ex = block_excl_scan<NT>(len, s_scan, total);
      s_excl[tid] = ex;
      s_bs[tid] = bs;
      s_av[tid] = av;
      if (tid == 0) s_excl[NT] = total;
      __syncthreads();
      for (uint32_t cb = 0; cb < total; cb += NT) {
        const uint32_t q = cb + tid;
        const bool act = q < total;
        uint32_t col = 0, slot = 0, dslot = kEmptyKey;
        double pv = 0.0;
        bool dup = false;
        if (act) {
          // largest i with s_excl[i] <= q
          int i = 0;
#pragma unroll
          for (int st = NT / 2; st > 0; st >>= 1)
            if (s_excl[i + st] <= q) i += st;
          const uint64_t src = s_bs[i] + (q - s_excl[i]);
          col = uint32_t(ld_idx(p.B.ci + src));
          pv = __dmul_rn(s_av[i], ld_val(p.B.v + src));
          uint32_t h = long_hash(col, mask);
          while (true) {
            const uint32_t k = __ldcg(keys + h);
            if (k == col) break;
            if (k == kEmptyKey) {
              const uint32_t old = atomicCAS(keys + h, kEmptyKey, col);
              if (old == kEmptyKey) {
                if (!(atomicOr(bits + (col >> 5), 1u << (col & 31))))
                  atomicOr(sum + (col >> 10), 1u << ((col >> 5) & 31));  // word became nonzero
                atomicMin(&s_min, col);
                atomicMax(&s_max, col);
                break;
              }
              if (old == col) break;
            }
            h = (h + 1) & mask;
          }
          slot = h;
          // does another product of this chunk hit the same column?
          uint32_t d = long_hash(col, kDupSlots - 1);
          while (true) {
            const uint32_t old = atomicCAS(s_dup + d, kEmptyKey, col);
            if (old == kEmptyKey) { dslot = d; break; }  // ours to reset
            if (old == col) { dup = true; break; }
            d = (d + 1) & (kDupSlots - 1);
          }
        }
        if (!__syncthreads_or(dup)) {
          // all columns of the chunk distinct: every product adds directly
          if (act) {
            const double cur = __ldcg(vals + slot);
            if (STATS && cur == 0.0) ++touches;
            __stcg(vals + slot, __dadd_rn(cur, pv));
          }
        } else {
          // equal columns: rounds, lowest product index first (left fold order)
          const uint32_t seq = seq_base + q;
          bool pending = act;
          while (__syncthreads_or(pending)) {
            if (pending) atomicMin(owner + slot, seq);
            __syncthreads();
            if (pending && atomicAdd(owner + slot, 0u) == seq) {
              const double cur = __ldcg(vals + slot);
              if (STATS && cur == 0.0) ++touches;
              __stcg(vals + slot, __dadd_rn(cur, pv));
              atomicExch(owner + slot, kEmptyKey);
              pending = false;
            }
            __syncthreads();
          }
        }
        // reset the duplicate detector for the next chunk (inserters only)
        if (dslot != kEmptyKey) s_dup[dslot] = kEmptyKey;
        __syncthreads();
      }
      seq_base += total;
      __syncthreads();
    }
    // ---- ordered extraction: summary words -> nonzero bitmap words -> bits ----
    const uint32_t cmin = s_min, cmax = s_max;
    uint32_t s_begin = 0, s_end = 0, mine = 0;
    if (cmin <= cmax) {
      const uint32_t s0 = cmin >> 10, s1 = cmax >> 10;
      const uint32_t per = (s1 - s0 + 1 + NT - 1) / NT;
      s_begin = s0 + tid * per;
      s_end = s_begin + per;
      if (s_begin > s1 + 1) s_begin = s1 + 1;
      if (s_end > s1 + 1) s_end = s1 + 1;
      for (uint32_t sw = s_begin; sw < s_end; ++sw) {
        uint32_t sb = __ldcg(sum + sw);
        while (sb) {
          const uint32_t j = __ffs(sb) - 1;
          sb &= sb - 1;
          mine += __popc(__ldcg(bits + ((sw << 5) | j)));
        }
      }
    }
    uint32_t n_out;
    const uint32_t my_base = block_excl_scan<NT>(mine, s_scan, n_out);
    if (tid == 0) s_off = atomicAdd(p.ctrl + kCtrlStageCursor, (unsigned long long)n_out);
    __syncthreads();
    const uint64_t off = s_off;
    uint64_t pos = off + my_base;
    bool zero = false;
    for (uint32_t sw = s_begin; sw < s_end; ++sw) {
      uint32_t sb = __ldcg(sum + sw);
      while (sb) {
        const uint32_t j = __ffs(sb) - 1;
        sb &= sb - 1;
        const uint32_t w = (sw << 5) | j;
        uint32_t b = __ldcg(bits + w);
        __stcg(bits + w, 0u);  // restore as we go (the bits are in registers)
        while (b) {
          const uint32_t bit = __ffs(b) - 1;
          b &= b - 1;
          const uint32_t col = (w << 5) | bit;
          const double v = __ldcg(vals + long_probe(keys, col, mask));
          zero |= v == 0.0;
          p.l_ci[pos] = uint32_t(col);
          p.l_v[pos] = v;
          ++pos;
        }
      }
      __stcg(sum + sw, 0u);
    }
    if (STATS) {
      uint32_t t = touches;
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) t += __shfl_xor_sync(kFull, t, d);
      if (lane_id() == 0 && t) atomicAdd(&s_touch, t);
    }
    uint32_t nz_total = n_out;
    if (__syncthreads_or(zero)) {
      // exact cancellations (kernels.py:296-298 drops them): compact in place
      uint32_t out = 0;
      for (uint32_t c0 = 0; c0 < n_out; c0 += NT) {
        const uint32_t i = c0 + tid;
        uint32_t ci = 0;
        double v = 0.0;
        bool keep = false;
        if (i < n_out) {
          ci = p.l_ci[off + i];
          v = p.l_v[off + i];
          keep = v != 0.0;
        }
        uint32_t kept;
        const uint32_t ex = block_excl_scan<NT>(keep ? 1u : 0u, s_scan, kept);
        if (keep) {
          p.l_ci[off + out + ex] = ci;
          p.l_v[off + out + ex] = v;
        }
        out += kept;
        __syncthreads();
      }
      nz_total = out;
    }
    // restore the workspace for the next row
    for (uint32_t s = tid; s < tsize; s += NT) {
      __stcg(keys + s, kEmptyKey);
      __stcg(vals + s, 0.0);
    }
    if (tid == 0) {
      p.l_off[li] = off;
      p.l_nnz[li] = nz_total;
      if (STATS) {
        p.st_min[r] = cmin;
        p.st_max[r] = cmax;
        p.st_touch[r] = s_touch;
      }
    }
    __syncthreads();
  }
}


// Long rows: staged by k_long, placed at their final offsets after k_fused.
struct CopyParams {
  const uint32_t* list;      // pre-computed rows (k_collect)
  const uint32_t* prod;
  const uint32_t* big;       // mid then huge sub-lists (rows = A.rows apart)
  const uint32_t* dom_big;   // k_esc_dom's rows past long_min (null: none)
  const unsigned long long* ctrl;
  unsigned long long* tickets;  // [0] big rows, [1] other rows
  const uint64_t* l_off;
  const uint32_t* l_nnz;
  const uint32_t* l_ci;
  const double* l_v;
  const uint64_t* c_rp;
  uint64_t* c_ci;
  double* c_v;
  uint64_t rows;
  uint32_t long_min;         // rows past it are in the sub-lists
  const uint32_t* row_np;    // ESC mode: parts per huge row (else null)
  const uint32_t* row_pbase;
  const uint64_t* part_off;
  const uint32_t* part_nnz;
  uint64_t c_cap;                  // entries reserved for C: nothing is copied past it
  unsigned long long* overflow;    // ctrl word: kCfOverflow when a run would pass it
};

// Copy the staged rows into their slots of C (after k_fused wrote row_ptr).
// Rows of the sub-lists (long: up to tens of thousands of entries) are copied
// by whole blocks first; the remaining listed rows (<= long_min products) by
// one warp each. Both take rows dynamically.
// One staged run to its slot of C: U loads in flight per thread (a plain
// load -> store loop is one memory round trip per step).
#ifndef SPMMM_COPY_U
#define SPMMM_COPY_U 4
#endif
template <int U>
__device__ __forceinline__ void copy_run(unsigned long long* __restrict__ dci,
                                         double* __restrict__ dv,
                                         const uint32_t* __restrict__ sci,
                                         const double* __restrict__ sv, uint32_t n,
                                         uint32_t t0, uint32_t step) {
  // U loads in flight per thread whatever n is (most staged rows are a few
  // dozen entries: a loop that needs U * step of them to unroll never does)
  for (uint32_t i = t0; i < n; i += U * step) {
    unsigned long long c[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = i + u * step;
      c[u] = 0;
      v[u] = 0.0;
      if (j < n) {
        c[u] = (unsigned long long)__ldcs(sci + j);
        v[u] = __ldcs(sv + j);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = i + u * step;
      if (j < n) {
        __stcs(dci + j, c[u]);
        __stcs(dv + j, v[u]);
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_copy_long(CopyParams p) {
  __shared__ uint32_t s_t;
  unsigned long long* cci = reinterpret_cast<unsigned long long*>(p.c_ci);
  const uint32_t n_mid = uint32_t(p.ctrl[kCtrlMidRows]);
  const uint32_t n_big = n_mid + uint32_t(p.ctrl[kCtrlHugeRows]);
  const uint32_t n_dom = p.dom_big ? uint32_t(p.ctrl[kCtrlDomBigRows]) : 0u;
  while (true) {
    if (threadIdx.x == 0) s_t = uint32_t(atomicAdd(p.tickets, 1ull));
    __syncthreads();
    const uint32_t t = s_t;
    __syncthreads();
    if (t >= n_big + n_dom) break;
    if (t >= n_big) {  // dominated rows past long_min (the shorter ones: warps, below)
      const uint32_t dl = p.dom_big[t - n_big];
      const uint32_t dr = p.list[dl];
      const uint64_t ddst = p.c_rp[dr];
      const uint32_t dcnt = p.l_nnz[dl];
      if (ddst + dcnt > p.c_cap) {
        if (threadIdx.x == 0) atomicOr(p.overflow, (unsigned long long)kCfOverflow);
        continue;
      }
      const uint64_t dsrc = p.l_off[dl];
      copy_run<SPMMM_COPY_U>(cci + ddst, p.c_v + ddst, p.l_ci + dsrc, p.l_v + dsrc, dcnt, threadIdx.x,
                  blockDim.x);
      continue;
    }
    const uint32_t li = t < n_mid ? p.big[t] : p.big[p.rows + (t - n_mid)];
    const uint64_t dst = p.c_rp[p.list[li]];
    const uint32_t np = (t >= n_mid && p.row_np) ? p.row_np[t - n_mid] : 0u;
    if (np) {  // ESC parts of a huge row, in column order
      const uint32_t pb = p.row_pbase[t - n_mid];
      uint64_t d = dst;
      for (uint32_t j = 0; j < np; ++j) {
        const uint64_t so = p.part_off[pb + j];
        const uint32_t pc = p.part_nnz[pb + j];
        if (d + pc > p.c_cap) {
          if (threadIdx.x == 0) atomicOr(p.overflow, (unsigned long long)kCfOverflow);
          break;
        }
        copy_run<SPMMM_COPY_U>(cci + d, p.c_v + d, p.l_ci + so, p.l_v + so, pc, threadIdx.x, blockDim.x);
        d += pc;
      }
      continue;
    }
    const uint64_t src = p.l_off[li];
    const uint32_t cnt = p.l_nnz[li];
    if (dst + cnt > p.c_cap) {
      if (threadIdx.x == 0) atomicOr(p.overflow, (unsigned long long)kCfOverflow);
      continue;
    }
    copy_run<SPMMM_COPY_U>(cci + dst, p.c_v + dst, p.l_ci + src, p.l_v + src, cnt, threadIdx.x, blockDim.x);
  }
  // the other listed rows (<= long_min products): one warp each, static
  // assignment (their costs are alike; no ticket traffic)
  const uint32_t lane = lane_id();
  const uint32_t n = uint32_t(p.ctrl[kCtrlLongRows]);
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t li = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); li < n; li += nwarps) {
    const uint32_t r = p.list[li];
    if (p.prod[r] > p.long_min) continue;  // copied above
    const uint64_t dst = p.c_rp[r];
    const uint64_t src = p.l_off[li];
    const uint32_t cnt = p.l_nnz[li];
    if (dst + cnt > p.c_cap) {
      if (lane == 0) atomicOr(p.overflow, (unsigned long long)kCfOverflow);
      continue;
    }
    copy_run<SPMMM_COPY_U>(cci + dst, p.c_v + dst, p.l_ci + src, p.l_v + src, cnt, lane, 32);
  }
}

// ---------------------------------------------------------------------------
// K3b: long rows that fit shared memory (<= kLongSmemProducts products):
// one 512-thread block per row, everything on chip.
//  * accumulate: open-addressing table of up to kLongSmemSlots slots in shared
//    memory (sized per row for <= 3/4 load); products in chunks of 512 in
//    (k, j) order; equal columns inside a chunk are applied in rounds, lowest
//    product index first, arbitrated by a small shared table (column, min
//    index) — the reference's left fold per column (kernels.py:167-174);
//  * extract: the row's table region is bitonic-sorted in shared memory by
//    column (empty and exactly-zero slots sort last and are dropped,
//    kernels.py:296-298), then written out coalesced.
constexpr uint32_t kLongSmemSlots = 16384;
constexpr uint32_t kLongSmemProducts = kLongSmemSlots * 3 / 4;
constexpr int kLongDupSlots = 2048;

__host__ __device__ constexpr size_t long_smem_bytes() {
  return size_t(kLongSmemSlots) * (sizeof(uint32_t) + sizeof(double)) +
         size_t(kLongDupSlots) * 2 * sizeof(uint32_t);
}

// lower_bound of x in the sorted column run B.ci[lo, hi)
__device__ __forceinline__ uint64_t col_lower_bound(const uint64_t* ci, uint64_t lo, uint64_t hi,
                                                    uint64_t x) {
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (ld_idx(ci + mid) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// PARTS == 1: one block per row of (min, kLongSmemProducts] products.
// PARTS > 1: a thread-block cluster of PARTS blocks per longer row. Block i
// owns the i-th of PARTS equal column ranges of the row: it walks the whole
// A row but only the slice of each B row inside its range (binary search),
// so every column still folds in k order on one block. Counts, offsets and
// row stats are exchanged through distributed shared memory; the parts are
// staged back to back in column order. A part whose distinct columns outgrow
// the table hands the whole row to k_long (global tables).
template <bool STATS, int PARTS>
__global__ void __launch_bounds__(kLongThreads, 1) k_long_smem(LongParams p) {
  namespace cg = cooperative_groups;
  constexpr int NT = kLongThreads;
  constexpr uint32_t kCap = kLongSmemSlots * 7 / 8;  // PARTS > 1: inserts before hand-off
  extern __shared__ __align__(16) unsigned char sm[];
  double* vals = reinterpret_cast<double*>(sm);
  uint32_t* keys = reinterpret_cast<uint32_t*>(sm + kLongSmemSlots * sizeof(double));
  uint32_t* dkey = keys + kLongSmemSlots;
  uint32_t* dmin = dkey + kLongDupSlots;
  __shared__ uint32_t s_excl[NT + 1];
  __shared__ uint64_t s_bs[NT];
  __shared__ double s_av[NT];
  __shared__ uint32_t s_scan[NT / 32 + 1];
  __shared__ uint32_t s_li, s_tk, s_min, s_max, s_touch, s_kmin, s_kmax, s_cmin, s_cmax;
  __shared__ uint32_t s_x[2];  // PARTS > 1: this part's nnz, overflow flag
  __shared__ uint32_t s_ins;
  __shared__ unsigned long long s_off;
  const uint32_t tid = threadIdx.x;
  uint32_t rank = 0;
  if constexpr (PARTS > 1) rank = cg::this_cluster().block_rank();
  for (uint32_t s = tid; s < kLongSmemSlots; s += NT) keys[s] = kEmptyKey;
  for (uint32_t s = tid; s < uint32_t(kLongDupSlots); s += NT) {
    dkey[s] = kEmptyKey;
    dmin[s] = kEmptyKey;
  }
  if (tid == 0) {
    s_kmin = kEmptyKey;
    s_kmax = 0;
    s_cmin = kEmptyKey;
    s_cmax = 0;
  }
  const uint32_t n_sub = uint32_t(*(volatile const unsigned long long*)p.n_sub);
  while (true) {
    if constexpr (PARTS == 1) {
      if (tid == 0) s_li = uint32_t(atomicAdd(p.ticket, 1ull));
      __syncthreads();
    } else {
      if (rank == 0 && tid == 0) s_tk = uint32_t(atomicAdd(p.ticket, 1ull));
      cg::this_cluster().sync();
      if (tid == 0) s_li = *cg::this_cluster().map_shared_rank(&s_tk, 0);
      __syncthreads();
    }
    const uint32_t t_row = s_li;
    if (t_row >= n_sub) break;
    const uint32_t li = p.sub[t_row];
    const uint32_t r = p.list[li];
    const uint32_t prod = p.prod[r];
    uint32_t tsize = kLongSmemSlots;
    if constexpr (PARTS == 1) {
      tsize = 64;
      while (tsize * 3 < prod * 4) tsize <<= 1;  // load <= 3/4
    }
    const uint32_t mask = tsize - 1;
    const uint64_t lo = ld_idx(p.A.rp + r), hi = ld_idx(p.A.rp + r + 1);
    // PARTS > 1: this block's column range [clo, chi)
    uint64_t clo = 0, chi = ~0ull;
    if constexpr (PARTS > 1) {
      uint32_t cmn = kEmptyKey, cmx = 0;
      // four entries per thread per round: the three dependent loads of each
      // entry overlap across the four
      for (uint64_t e0 = lo + tid; e0 < hi; e0 += 4 * NT) {
        uint64_t k[4], bs[4], be[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint64_t e = e0 + uint64_t(u) * NT;
          k[u] = e < hi ? ld_idx(p.A.ci + e) : ~0ull;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          bs[u] = be[u] = 0;
          if (k[u] != ~0ull) {
            bs[u] = ld_idx(p.B.rp + k[u]);
            be[u] = ld_idx(p.B.rp + k[u] + 1);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (be[u] > bs[u]) {
            const uint32_t c0 = uint32_t(ld_idx(p.B.ci + bs[u]));
            const uint32_t c1 = uint32_t(ld_idx(p.B.ci + be[u] - 1));
            cmn = c0 < cmn ? c0 : cmn;
            cmx = c1 > cmx ? c1 : cmx;
          }
        }
      }
      cmn = __reduce_min_sync(kFull, cmn);
      cmx = __reduce_max_sync(kFull, cmx);
      if (lane_id() == 0) {
        atomicMin(&s_cmin, cmn);
        atomicMax(&s_cmax, cmx);
      }
      __syncthreads();
      const uint64_t w = uint64_t(s_cmax - s_cmin) / PARTS + 1;
      clo = s_cmin + rank * w;
      chi = clo + w;
    }
    if (tid == 0) { s_min = kEmptyKey; s_max = 0; s_touch = 0; s_ins = 0; }
    uint32_t touches = 0, seq_base = 0;
    bool over = false;
    __syncthreads();
    for (uint64_t abase = lo; abase < hi && !over; abase += NT) {
      const uint64_t e = abase + tid;
      uint32_t len = 0;
      uint64_t bs = 0;
      double av = 0.0;
      if (e < hi) {
        const uint64_t k = ld_idx(p.A.ci + e);
        av = ld_val(p.A.v + e);
        bs = ld_idx(p.B.rp + k);
        uint64_t be = ld_idx(p.B.rp + k + 1);
        if constexpr (PARTS > 1) {
          if (be - bs <= 8) {  // short B row: one round of loads, then count
            uint32_t c[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
              c[u] = bs + u < be ? uint32_t(ld_idx(p.B.ci + bs + u)) : kEmptyKey;
            uint32_t nlo = 0, nhi = 0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              nlo += (bs + u < be && c[u] < clo) ? 1u : 0u;
              nhi += (bs + u < be && c[u] < chi) ? 1u : 0u;
            }
            be = bs + nhi;
            bs = bs + nlo;
          } else {
            bs = col_lower_bound(p.B.ci, bs, be, clo);
            be = col_lower_bound(p.B.ci, bs, be, chi);
          }
        }
        len = uint32_t(be - bs);
      }
      uint32_t total;
      const uint32_t ex = block_excl_scan<NT>(len, s_scan, total);
      s_excl[tid] = ex;
      s_bs[tid] = bs;
      s_av[tid] = av;
      if (tid == 0) s_excl[NT] = total;
      __syncthreads();
      for (uint32_t cb = 0; cb < total; cb += NT) {
        if constexpr (PARTS > 1) {
          // room for a whole chunk of new columns, or hand the row on
          if (s_ins + NT > kCap) {
            over = true;
            break;
          }
        }
        const uint32_t q = cb + tid;
        const bool act = q < total;
        uint32_t col = 0, slot = 0, d = 0;
        double pv = 0.0;
        bool fresh = false, dup = false, dins = false;
        if (act) {
          int i = 0;
#pragma unroll
          for (int st = NT / 2; st > 0; st >>= 1)
            if (s_excl[i + st] <= q) i += st;
          const uint64_t src = s_bs[i] + (q - s_excl[i]);
          col = uint32_t(ld_idx(p.B.ci + src));
          pv = __dmul_rn(s_av[i], ld_val(p.B.v + src));
          uint32_t h = long_hash(col, mask);
          while (true) {
            const uint32_t k = keys[h];
            if (k == col) break;
            if (k == kEmptyKey) {
              const uint32_t old = atomicCAS(keys + h, kEmptyKey, col);
              if (old == kEmptyKey) { fresh = true; break; }
              if (old == col) break;
            }
            h = (h + 1) & mask;
          }
          slot = h;
          d = long_hash(col, kLongDupSlots - 1);
          while (true) {
            const uint32_t old = atomicCAS(dkey + d, kEmptyKey, col);
            if (old == kEmptyKey) { dins = true; break; }
            if (old == col) { dup = true; break; }
            d = (d + 1) & (kLongDupSlots - 1);
          }
          if (fresh) vals[slot] = 0.0;  // new column: dense[x] == 0.0
        }
        if constexpr (PARTS > 1) {
          if (fresh) atomicAdd(&s_ins, 1u);  // read after the next barrier
        }
        if (!__syncthreads_or(dup)) {
          if (act) {
            const double cur = vals[slot];
            if (STATS && cur == 0.0) ++touches;
            vals[slot] = __dadd_rn(cur, pv);
          }
        } else {
          const uint32_t seq = seq_base + q;
          bool pending = act;
          while (__syncthreads_or(pending)) {
            if (pending) atomicMin(dmin + d, seq);
            __syncthreads();
            if (pending && dmin[d] == seq) {
              const double cur = vals[slot];
              if (STATS && cur == 0.0) ++touches;
              vals[slot] = __dadd_rn(cur, pv);
              dmin[d] = kEmptyKey;
              pending = false;
            }
            __syncthreads();
          }
        }
        if (dins) dkey[d] = kEmptyKey;
        __syncthreads();
      }
      seq_base += total;
      __syncthreads();
    }
    // ---- extract in column order ----
    // P0: drop exact zeros (kernels.py:296-298); count and range of the rest
    uint32_t mn = kEmptyKey, mx = 0, keep_cnt = 0, kmn = kEmptyKey, kmx = 0;
    for (uint32_t s = tid; s < tsize; s += NT) {
      const uint32_t k = keys[s];
      if (k != kEmptyKey) {
        if (STATS) {
          mn = k < mn ? k : mn;
          mx = k > mx ? k : mx;
        }
        if (vals[s] != 0.0 && !over) {
          ++keep_cnt;
          kmn = k < kmn ? k : kmn;
          kmx = k > kmx ? k : kmx;
        } else {
          keys[s] = kEmptyKey;
        }
      }
    }
    kmn = __reduce_min_sync(kFull, kmn);
    kmx = __reduce_max_sync(kFull, kmx);
    if (lane_id() == 0 && kmn != kEmptyKey) {
      atomicMin(&s_kmin, kmn);
      atomicMax(&s_kmax, kmx);
    }
    if (STATS) {
      uint32_t t = touches;
#pragma unroll
      for (int dd = 16; dd > 0; dd >>= 1) t += __shfl_xor_sync(kFull, t, dd);
      mn = __reduce_min_sync(kFull, mn);
      mx = __reduce_max_sync(kFull, mx);
      if (lane_id() == 0) {
        if (t) atomicAdd(&s_touch, t);
        atomicMin(&s_min, mn);
        atomicMax(&s_max, mx);
      }
    }
    uint32_t n_out;
    block_excl_scan<NT>(keep_cnt, s_scan, n_out);  // (its barriers order the atomics)
    bool handed_on = false;
    if constexpr (PARTS == 1) {
      if (tid == 0) {
        s_off = n_out ? atomicAdd(p.ctrl + kCtrlStageCursor, (unsigned long long)n_out) : 0ull;
        p.l_off[li] = s_off;
        p.l_nnz[li] = n_out;
        if (STATS) {
          p.st_min[r] = s_min;
          p.st_max[r] = s_max;
          p.st_touch[r] = s_touch;
        }
      }
      __syncthreads();
    } else {
      cg::cluster_group cluster = cg::this_cluster();
      if (tid == 0) {  // (`over` is block-uniform)
        s_x[0] = n_out;
        s_x[1] = over ? 1u : 0u;
      }
      cluster.sync();  // (A) parts' counts, flags and stats are final
      uint32_t prefix = 0, total = 0, any_over = 0;
#pragma unroll
      for (int j = 0; j < PARTS; ++j) {
        const uint32_t* x = cluster.map_shared_rank(s_x, j);
        const uint32_t nj = x[0];
        any_over |= x[1];
        prefix += uint32_t(j) < rank ? nj : 0u;
        total += nj;
      }
      if (rank == 0 && tid == 0) {
        if (any_over) {
          p.ovf[atomicAdd(p.ctrl + kCtrlOvfRows, 1ull)] = li;
        } else {
          s_off = total ? atomicAdd(p.ctrl + kCtrlStageCursor, (unsigned long long)total) : 0ull;
          p.l_off[li] = s_off;
          p.l_nnz[li] = total;
          if (STATS) {
            uint32_t a0 = kEmptyKey, a1 = 0, a2 = 0;
            for (int j = 0; j < PARTS; ++j) {
              const uint32_t mj = *cluster.map_shared_rank(&s_min, j);
              const uint32_t xj = *cluster.map_shared_rank(&s_max, j);
              a0 = mj < a0 ? mj : a0;
              a1 = xj > a1 ? xj : a1;
              a2 += *cluster.map_shared_rank(&s_touch, j);
            }
            p.st_min[r] = a0;
            p.st_max[r] = a1;
            p.st_touch[r] = a2;
          }
        }
      }
      cluster.sync();  // (B) the row's staging offset is known
      if (any_over) {
        handed_on = true;
        for (uint32_t s = tid; s < tsize; s += NT) keys[s] = kEmptyKey;
      } else if (tid == 0) {
        s_off = *cluster.map_shared_rank(&s_off, 0) + prefix;
      }
      __syncthreads();
    }
    // P1: bucket histogram. Buckets are column ranges (monotone), about 16
    // columns each, so every bucket is a small independent sort.
    const uint32_t kmin = s_kmin, range = s_kmax - kmin;
    uint32_t nb = 2;
    while (nb * 16 < n_out && nb < uint32_t(kLongDupSlots) / 2) nb <<= 1;
    while ((range >> 26) >= nb) nb <<= 1;  // bucket width <= 2^26: 32-bit sort keys
    uint32_t sh = 0;
    while ((range >> sh) >= nb) ++sh;
    uint32_t* hist = dkey;  // the duplicate table is idle now
    uint32_t* cursor = dmin;
    if (n_out && !handed_on) {
      const uint64_t off = s_off;
      for (uint32_t b = tid; b < nb; b += NT) hist[b] = 0;
      __syncthreads();
      for (uint32_t s = tid; s < tsize; s += NT) {
        const uint32_t k = keys[s];
        if (k != kEmptyKey) atomicAdd(hist + ((k - kmin) >> sh), 1u);
      }
      __syncthreads();
      // exclusive bucket offsets (two buckets per thread; nb <= 2 * NT)
      const uint32_t h0 = 2 * tid < nb ? hist[2 * tid] : 0u;
      const uint32_t h1 = 2 * tid + 1 < nb ? hist[2 * tid + 1] : 0u;
      uint32_t tot;
      const uint32_t ex = block_excl_scan<NT>(h0 + h1, s_scan, tot);
      if (2 * tid < nb) {
        cursor[2 * tid] = ex;
        cursor[2 * tid + 1] = ex + h0;
      }
      __syncthreads();
      // P2: scatter into the staged row by bucket; clears the table
      for (uint32_t s = tid; s < tsize; s += NT) {
        const uint32_t k = keys[s];
        if (k != kEmptyKey) {
          const uint32_t pos = atomicAdd(cursor + ((k - kmin) >> sh), 1u);
          __stcg(p.l_ci + off + pos, uint32_t(k));
          __stcg(p.l_v + off + pos, vals[s]);
          keys[s] = kEmptyKey;
        }
      }
      __syncthreads();
      // P3: one warp per bucket of <= 64: register bitonic sort in place
      const uint32_t lane = lane_id(), warp = tid >> 5;
      bool big = false;
      for (uint32_t b = warp; b < nb; b += NT / 32) {
        const uint32_t sz = hist[b];
        if (sz == 0) continue;
        if (sz > 64) {
          big = true;
          continue;
        }
        const uint64_t base = off + cursor[b] - sz;
        const uint32_t blo = kmin + (b << sh);  // bucket's first column
        uint32_t key[2];
        double v[2];
#pragma unroll
        for (int e2 = 0; e2 < 2; ++e2) {
          const uint32_t idx = uint32_t(e2) * 32u + lane;
          key[e2] = ~0u;
          v[e2] = 0.0;
          if (idx < sz) {
            key[e2] = ((__ldcg(p.l_ci + base + idx) - blo) << 6) | idx;
            v[e2] = __ldcg(p.l_v + base + idx);
          }
        }
        if (sz <= 32) bitonic_sort<1>(key);  // the common size (about 16 per bucket)
        else bitonic_sort<2>(key);
#pragma unroll
        for (int e2 = 0; e2 < 2; ++e2) {
          const uint32_t idx = uint32_t(e2) * 32u + lane;
          const uint32_t pos = key[e2] & 63u;
          const double t0 = __shfl_sync(kFull, v[0], pos & 31u);
          const double t1 = __shfl_sync(kFull, v[1], pos & 31u);
          if (idx < sz) {
            __stcg(p.l_ci + base + idx, uint32_t(blo + (key[e2] >> 6)));
            __stcg(p.l_v + base + idx, (pos >> 5) ? t1 : t0);
          }
        }
      }
      // P4 (clustered columns only): buckets past 64, sorted by the whole
      // block in the idle table
      if (__syncthreads_or(big)) {
        for (uint32_t b = 0; b < nb; ++b) {
          const uint32_t sz = hist[b];
          if (sz <= 64) continue;
          const uint64_t base = off + cursor[b] - sz;
          uint32_t np = 1;
          while (np < sz) np <<= 1;
          for (uint32_t t = tid; t < np; t += NT) {
            keys[t] = t < sz ? __ldcg(p.l_ci + base + t) : kEmptyKey;
            if (t < sz) vals[t] = __ldcg(p.l_v + base + t);
          }
          __syncthreads();
          for (uint32_t k2 = 2; k2 <= np; k2 <<= 1) {
            for (uint32_t j = k2 >> 1; j > 0; j >>= 1) {
              for (uint32_t t = tid; t < (np >> 1); t += NT) {
                const uint32_t i = 2 * t - (t & (j - 1));
                const uint32_t ka = keys[i], kb = keys[i + j];
                if ((ka > kb) == ((i & k2) == 0)) {
                  keys[i] = kb;
                  keys[i + j] = ka;
                  const double tv = vals[i];
                  vals[i] = vals[i + j];
                  vals[i + j] = tv;
                }
              }
              __syncthreads();
            }
          }
          for (uint32_t t = tid; t < sz; t += NT) {
            __stcg(p.l_ci + base + t, keys[t]);
            __stcg(p.l_v + base + t, vals[t]);
          }
          __syncthreads();
          for (uint32_t t = tid; t < np; t += NT) keys[t] = kEmptyKey;
          __syncthreads();
        }
      }
      __syncthreads();
      for (uint32_t b = tid; b < nb; b += NT) {
        hist[b] = kEmptyKey;
        cursor[b] = kEmptyKey;
      }
    }
    __syncthreads();
    if (tid == 0) {
      s_kmin = kEmptyKey;
      s_kmax = 0;
      s_cmin = kEmptyKey;
      s_cmax = 0;
    }
    __syncthreads();
  }
  if constexpr (PARTS > 1) cg::this_cluster().sync();  // no block leaves while read remotely
}

}  // namespace spmmm
