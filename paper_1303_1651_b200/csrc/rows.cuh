// Per-row accumulation paths of the fused kernel.
//
// Order contract (the reason parity is bit-exact, kernels.py:163-180): for an
// output column x the value is the left fold, from 0.0, of fl(a_rk * b_kx)
// over the A-row entries k in ascending column order, each step one
// separately rounded fp64 add. Product q of a row is entry j of B row k, with
// q running through (k, j) in A-entry order — that is, q order *is* the
// reference's k order, and every path below applies a column's products in
// ascending q.
#pragma once

#include "device.cuh"

namespace spmmm {

// ---------------------------------------------------------------------------
// Short rows (<= 32 products, <= 32 A entries): one product per lane,
// expand -> bitonic sort by (column, q) -> segmented left fold. R rows of a
// warp tile go through every phase together, so their four dependent load
// levels (A.row_ptr, A entries, B.row_ptr, B entries) overlap.
struct ShortOut {
  uint32_t col;
  uint32_t rank;
  double val;
  bool keep;
};

// ELL copy of B for matrices whose rows have <= kEllSlots entries: one 64-byte
// record per B row, u32 col[6] (unused slots 0xffffffff) then f64 val[5].
// A tile row with <= kEllEntries A entries then maps product (entry e, slot j)
// to lane 5e + j — lane order is still the reference's (k, j) order — and
// needs no B.row_ptr loads, no scan and no search: one 64-byte block per
// referenced B row.
constexpr int kEllSlots = 5;
constexpr int kEllWords = 16;   // 64 B per record
constexpr int kEllValOff = 6;   // values start after 6 column words (byte 24)
constexpr uint32_t kEllEntries = 32 / kEllSlots;  // 6

// One ELL record: u32 col[6] (unused 0xffffffff) then f64 val[5] — B row r's
// entries [lo, hi) (at most kEllSlots are stored).
__device__ __forceinline__ void pack_ell_record(const DevCsr& B, uint64_t r, uint64_t lo,
                                                uint64_t hi, uint4* __restrict__ ell) {
  uint32_t c[kEllSlots + 1];
  double v[kEllSlots];
#pragma unroll
  for (int j = 0; j < kEllSlots; ++j) {
    const bool in = lo + j < hi;
    c[j] = in ? uint32_t(ld_idx(B.ci + lo + j)) : kEmptyKey;
    v[j] = in ? ld_val(B.v + lo + j) : 0.0;
  }
  c[kEllSlots] = kEmptyKey;
  auto lo32 = [](double x) { return uint32_t(__double_as_longlong(x)); };
  auto hi32 = [](double x) { return uint32_t(uint64_t(__double_as_longlong(x)) >> 32); };
  uint4* rec = ell + r * 4;
  rec[0] = make_uint4(c[0], c[1], c[2], c[3]);
  rec[1] = make_uint4(c[4], c[5], lo32(v[0]), hi32(v[0]));
  rec[2] = make_uint4(lo32(v[1]), hi32(v[1]), lo32(v[2]), hi32(v[2]));
  rec[3] = make_uint4(lo32(v[3]), hi32(v[3]), lo32(v[4]), hi32(v[4]));
}

// The count-free path's verdict (k_prep in aux_kernels.cuh measures the rows).
enum CfFlags : unsigned {
  kCfBadA = 1,      // A.row_ptr decreasing or past nnz
  kCfBadB = 2,      // B.row_ptr decreasing or past nnz
  kCfBadCol = 4,    // an A column >= B.rows
  kCfOverflow = 32,  // C outgrew its reservation (found by k_fused; nothing past it written)
  kCfUnsorted = 64   // k_esc_dom met a B row whose columns do not ascend (redone without it)
};

// ctrl + kCtrlCfFlags: [flags, longest A row, longest B row]. Every row of C
// then has <= max_a * max_b <= 32 products: the short path takes them all.
__host__ __device__ inline bool cf_applies(unsigned long long flags, unsigned long long max_a,
                                           unsigned long long max_b) {
  if (flags & (kCfBadA | kCfBadB | kCfBadCol)) return false;
  return max_a <= 32 && max_a * max_b <= 32;
}
// ... and B is read through its ELL records (when k_prep packed them)
__host__ __device__ inline bool cf_ell(unsigned long long max_a, unsigned long long max_b) {
  return max_a <= uint64_t(kEllEntries) && max_b <= uint64_t(kEllSlots);
}

// The count-free path's first pass. MODE 0, C = A·A (A square, its rows are
// B's rows): one pass over the rows measures both and checks A's columns
// while packing them as B's records. MODE 1, A spans most of B: A's rows and
// columns, then every B row (checked, measured, packed). MODE 2, A a row
// block of a larger matrix: A only — its rows, its columns against B.rows and
// their range [kmin, kmax] — and k_prep_b takes the B rows in that range.
// Runs as k_prep (aux_kernels.cuh) or as the prologue of k_fused (small
// products). Also zeroes the look-back counters.
struct CfWords {
  unsigned long long* flags;     // [0] kCf* bits, [1] longest A row, [2] longest B row
  unsigned long long* kmin_inv;  // ~(smallest column of A) (MODE 2)
  unsigned long long* kmax1;     // largest column of A + 1 (MODE 2)
  unsigned long long* ell;       // B's ELL records were packed
};

template <int MODE>
__device__ __forceinline__ void prep_pass(const DevCsr& A, const DevCsr& B, const CfWords& w,
                                          unsigned long long* __restrict__ zero, uint64_t nzero,
                                          uint4* __restrict__ ell, uint64_t t0, uint64_t stride) {
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
    if (f) atomicOr(w.flags, (unsigned long long)f);
    if (ma) atomicMax(w.flags + 1, ma);
    if (mb) atomicMax(w.flags + 2, mb);
    if (MODE == 2 && kmax1) {
      atomicMax(w.kmin_inv, ~kmin);
      atomicMax(w.kmax1, kmax1);
    }
    if (MODE != 2 && ell && t0 == 0) *w.ell = 1;
  }
}



template <int R, bool WIDE, bool STATS, bool ELLOK, bool CF = false>
__device__ __forceinline__ void short_rows(const DevCsr& A, const DevCsr& B,
                                           const uint32_t* __restrict__ ell,
                                           const uint64_t (&lo)[R], const uint32_t (&na)[R],
                                           const bool (&on)[R], ShortOut (&out)[R],
                                           uint32_t (&nnz)[R], uint32_t (&smin)[R],
                                           uint32_t (&smax)[R], uint32_t (&stouch)[R],
                                           uint32_t (&prods)[R], const void* pf = nullptr,
                                           bool self = false, uint64_t row0 = 0) {
  using K = typename std::conditional<WIDE, unsigned long long, uint32_t>::type;
  // narrow variant: every index and offset fits 32 bits (checked on the host)
  using Off = typename std::conditional<WIDE, uint64_t, uint32_t>::type;
  const uint32_t lane = lane_id();
  K key[R];
  double p[R];
  uint32_t tot[R];
  bool fast = false;
  if constexpr (ELLOK) {
    fast = ell != nullptr;
    if (!self) {
#pragma unroll
      for (int i = 0; i < R; ++i) fast &= !on[i] || na[i] <= kEllEntries;
    }
  }
  if (fast) {
    const uint32_t e = lane / kEllSlots, j = lane - e * kEllSlots;
    uint32_t col[R];
    double bv[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      col[i] = kEmptyKey;
      p[i] = 0.0;
      bv[i] = 0.0;
      if (self) {
        // C = A·A, row for row: row r's A entries are its own record — no
        // A.row_ptr / A.col_idx / A.values loads, one dependent level less
        if (on[i] && e < uint32_t(kEllSlots)) {
          const uint32_t* mine = ell + (row0 + uint64_t(i)) * kEllWords;
          const uint32_t k = ld_u32(mine + e, B.pol);
          p[i] = ld_val(reinterpret_cast<const double*>(mine + kEllValOff) + e, B.pol);
          if (k != kEmptyKey) {
            const uint32_t* rec = ell + uint64_t(k) * kEllWords;
            col[i] = ld_u32(rec + j, B.pol);
            bv[i] = ld_val(reinterpret_cast<const double*>(rec + kEllValOff) + j, B.pol);
          }
        }
      } else if (on[i] && e < na[i]) {
        const uint64_t k = ld_idx(A.ci + lo[i] + e, A.pol);
        p[i] = ld_val(A.v + lo[i] + e, A.pol);
        // (count-free path: k_prep has checked every A column against B.rows)
        const uint32_t* rec = ell + k * kEllWords;
        col[i] = ld_u32(rec + j, B.pol);
        bv[i] = ld_val(reinterpret_cast<const double*>(rec + kEllValOff) + j, B.pol);
      }
    }
    // the next group's records into L2 while this group waits on its own
    if (pf) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(pf));
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const bool valid = col[i] != kEmptyKey;
      p[i] = valid ? __dmul_rn(p[i], bv[i]) : 0.0;
      tot[i] = __popc(__ballot_sync(kFull, valid));
      key[i] = valid ? ((K(col[i]) << 5) | K(lane)) : ~K(0);
    }
  } else {
    Off kk[R];
    double av[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      kk[i] = 0;
      av[i] = 0.0;
      if (on[i] && lane < na[i]) {
        kk[i] = Off(ld_idx(A.ci + lo[i] + lane, A.pol));
        av[i] = ld_val(A.v + lo[i] + lane, A.pol);
      }
    }
    Off bs[R];
    uint32_t len[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      bs[i] = 0;
      len[i] = 0;
      if (on[i] && lane < na[i]) {
        const uint64_t b0 = ld_idx(B.rp + kk[i], B.pol);
        bs[i] = Off(b0);
        len[i] = uint32_t(ld_idx(B.rp + kk[i] + 1, B.pol) - b0);
      }
    }
    // widest A row of the tile bounds the scan and search depth (warp-uniform)
    uint32_t na_max = 1;
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (on[i] && na[i] > na_max) na_max = na[i];
    uint32_t incl[R];
#pragma unroll
    for (int i = 0; i < R; ++i) incl[i] = len[i];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      if (uint32_t(d) >= na_max) break;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const uint32_t t = __shfl_up_sync(kFull, incl[i], d);
        if (lane >= uint32_t(d)) incl[i] += t;
      }
    }
    uint32_t excl[R];
    int src[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      excl[i] = incl[i] - len[i];
      tot[i] = __shfl_sync(kFull, incl[i], (na[i] - 1) & 31u);
      if (lane >= na[i]) excl[i] = tot[i];  // beyond the row: never owns a product
      src[i] = 0;
    }
    // entry owning product q = lane: the largest i with excl_i <= lane
#pragma unroll
    for (int st = 16; st > 0; st >>= 1) {
      if (uint32_t(st) >= na_max) continue;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const uint32_t ex = __shfl_sync(kFull, excl[i], src[i] + st);
        if (ex <= lane) src[i] += st;
      }
    }
    uint32_t col[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const Off bsrc = __shfl_sync(kFull, bs[i], src[i]) + (lane - __shfl_sync(kFull, excl[i], src[i]));
      const double a = __shfl_sync(kFull, av[i], src[i]);
      col[i] = 0;
      p[i] = a;
      if (lane < tot[i]) {
        col[i] = uint32_t(ld_idx(B.ci + bsrc, B.pol));
        p[i] = ld_val(B.v + bsrc, B.pol);  // multiplied below, after the loads are in flight
      }
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const bool valid = lane < tot[i];
      const double a = __shfl_sync(kFull, av[i], src[i]);
      p[i] = valid ? __dmul_rn(a, p[i]) : 0.0;
      key[i] = valid ? ((K(col[i]) << 5) | K(lane)) : ~K(0);
    }
  }  // generic path
  bitonic32_multi<R>(key);
  uint32_t col[R];
  double v[R], acc[R];
  bool head[R];
  uint32_t seg[R], touches[R];
  uint32_t max_seg = 0;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    col[i] = uint32_t(key[i] >> 5);
    v[i] = __shfl_sync(kFull, p[i], uint32_t(key[i]) & 31u);
    const uint32_t prev = __shfl_up_sync(kFull, col[i], 1);
    head[i] = lane < tot[i] && (lane == 0 || prev != col[i]);
    // segment = this head's run of equal columns: up to the next head (or tot)
    const uint32_t hm = __ballot_sync(kFull, head[i]);
    const uint32_t above = hm & ~((2u << lane) - 1u);
    const uint32_t nxt = above ? uint32_t(__ffs(above) - 1) : tot[i];
    seg[i] = head[i] ? nxt - lane : 0u;
    max_seg = seg[i] > max_seg ? seg[i] : max_seg;
    acc[i] = v[i];
    touches[i] = 1;
  }
  max_seg = __reduce_max_sync(kFull, max_seg);
  // left fold of each segment in lane (= reference k) order
  for (uint32_t d = 1; d < max_seg; ++d) {
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const double t = __shfl_down_sync(kFull, v[i], d);
      if (d < seg[i]) {
        if (STATS && acc[i] == 0.0) ++touches[i];  // re-touch after a transient zero
        acc[i] = __dadd_rn(acc[i], t);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const bool keep = head[i] && (acc[i] != 0.0);  // kernels.py:296 drops exact zeros
    const uint32_t km = __ballot_sync(kFull, keep);
    out[i].col = col[i];
    out[i].val = acc[i];
    out[i].keep = keep;
    out[i].rank = __popc(km & lanemask_lt());
    nnz[i] = __popc(km);
    if (CF) prods[i] = tot[i];
    if (STATS && on[i]) {
      smin[i] = __shfl_sync(kFull, col[i], 0);
      smax[i] = __shfl_sync(kFull, col[i], (tot[i] - 1) & 31u);
      uint32_t t = head[i] ? touches[i] : 0u;
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) t += __shfl_xor_sync(kFull, t, d);
      stouch[i] = t;
    }
  }
}

// ---------------------------------------------------------------------------
// Several short rows in one pass (skewed inputs: most rows of C5 have a
// handful of products, so a pass per row leaves the warp nearly empty). The
// NR rows' A entries share the lanes (entry lane l belongs to the row whose
// entry range holds l), their products share the lanes in row order, and the
// sort key carries the row slot above the column: one expand -> sort -> fold
// pass yields the rows' results back to back, in row order, each row's
// columns folded in the reference's k order exactly as short_rows does.
// Needs sum(na) <= 32 and sum(products) <= 32 over the rows that are on, and
// columns < 2^kPackColBits in the narrow variant (the caller checks).
constexpr int kPackSlotBits = 2;  // NR <= 4 rows per pass
constexpr int kPackColBits = 32 - 5 - kPackSlotBits;

template <int NR, int G, bool WIDE>
__device__ __forceinline__ void packed_rows(const DevCsr& A, const DevCsr& B,
                                            const uint64_t (&lo)[G][NR],
                                            const uint32_t (&na)[G][NR], const bool (&on)[G][NR],
                                            ShortOut (&out)[G], uint32_t (&nnz)[G][NR]) {
  static_assert(NR <= (1 << kPackSlotBits), "row slots per packed pass");
  using K = typename std::conditional<WIDE, unsigned long long, uint32_t>::type;
  using Off = typename std::conditional<WIDE, uint64_t, uint32_t>::type;
  constexpr int kSlotShift = int(sizeof(K)) * 8 - kPackSlotBits;
  const uint32_t lane = lane_id();
  // G independent passes in lockstep (their dependent loads overlap).
  // entry lane -> (row slot, entry of that row)
  uint32_t slot[G], e[G];
  uint64_t rlo[G];
  bool ent[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    uint32_t eb = 0;
    slot[g] = 0;
    e[g] = 0;
    rlo[g] = 0;
    ent[g] = false;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const uint32_t n = on[g][i] ? na[g][i] : 0u;
      if (lane >= eb && lane < eb + n) {
        slot[g] = uint32_t(i);
        e[g] = lane - eb;
        rlo[g] = lo[g][i];
        ent[g] = true;
      }
      eb += n;
    }
  }
  Off kk[G], bs[G];
  double av[G];
  uint32_t len[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    kk[g] = 0;
    av[g] = 0.0;
    if (ent[g]) {
      kk[g] = Off(ld_idx(A.ci + rlo[g] + e[g], A.pol));
      av[g] = ld_val(A.v + rlo[g] + e[g], A.pol);
    }
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
    bs[g] = 0;
    len[g] = 0;
    if (ent[g]) {
      const uint64_t b0 = ld_idx(B.rp + kk[g], B.pol);
      bs[g] = Off(b0);
      len[g] = uint32_t(ld_idx(B.rp + kk[g] + 1, B.pol) - b0);
    }
  }
  // products of a pass's rows, in (row, k, j) order, one per lane
  uint32_t incl[G];
#pragma unroll
  for (int g = 0; g < G; ++g) incl[g] = len[g];
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t t = __shfl_up_sync(kFull, incl[g], d);
      if (lane >= uint32_t(d)) incl[g] += t;
    }
  }
  uint32_t excl[G], tot[G];
  int src[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    excl[g] = incl[g] - len[g];  // lanes past the entries: == tot, never an owner
    tot[g] = __shfl_sync(kFull, incl[g], 31);
    src[g] = 0;
  }
#pragma unroll
  for (int st = 16; st > 0; st >>= 1) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t ex = __shfl_sync(kFull, excl[g], src[g] + st);
      if (ex <= lane) src[g] += st;
    }
  }
  uint32_t col[G];
  double p[G];
  K key[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const Off bsrc = __shfl_sync(kFull, bs[g], src[g]) + (lane - __shfl_sync(kFull, excl[g], src[g]));
    col[g] = 0;
    p[g] = 0.0;
    if (lane < tot[g]) {
      col[g] = uint32_t(ld_idx(B.ci + bsrc, B.pol));
      p[g] = ld_val(B.v + bsrc, B.pol);  // multiplied below, after the loads are in flight
    }
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const double a = __shfl_sync(kFull, av[g], src[g]);
    const uint32_t pslot = __shfl_sync(kFull, slot[g], src[g]);
    const bool valid = lane < tot[g];
    p[g] = valid ? __dmul_rn(a, p[g]) : 0.0;
    key[g] = valid ? ((K(pslot) << kSlotShift) | (K(col[g]) << 5) | K(lane)) : ~K(0);
  }
  bitonic32_multi<G>(key);
  // sorted by (row slot, column, q): valid keys fill lanes [0, tot)
  K ck[G];
  double v[G], acc[G];
  bool head[G];
  uint32_t seg[G];
  uint32_t max_seg = 0;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    ck[g] = key[g] >> 5;  // slot and column
    v[g] = __shfl_sync(kFull, p[g], uint32_t(key[g]) & 31u);
    const K prev = __shfl_up_sync(kFull, ck[g], 1);
    head[g] = lane < tot[g] && (lane == 0 || prev != ck[g]);
    const uint32_t hm = __ballot_sync(kFull, head[g]);
    const uint32_t above = hm & ~((2u << lane) - 1u);
    const uint32_t nxt = above ? uint32_t(__ffs(above) - 1) : tot[g];
    seg[g] = head[g] ? nxt - lane : 0u;
    max_seg = seg[g] > max_seg ? seg[g] : max_seg;
    acc[g] = v[g];
  }
  max_seg = __reduce_max_sync(kFull, max_seg);
  for (uint32_t d = 1; d < max_seg; ++d) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const double t = __shfl_down_sync(kFull, v[g], d);
      if (d < seg[g]) acc[g] = __dadd_rn(acc[g], t);
    }
  }
  constexpr K kColMask = WIDE ? K(0xffffffffu) : K((1u << kPackColBits) - 1u);
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const bool keep = head[g] && (acc[g] != 0.0);  // kernels.py:296 drops exact zeros
    const uint32_t km = __ballot_sync(kFull, keep);
    out[g].col = uint32_t(ck[g] & kColMask);
    out[g].val = acc[g];
    out[g].keep = keep;
    out[g].rank = __popc(km & lanemask_lt());
    const uint32_t sid = uint32_t(key[g] >> kSlotShift);
#pragma unroll
    for (int i = 0; i < NR; ++i)
      nnz[g][i] = __popc(km & __ballot_sync(kFull, lane < tot[g] && sid == uint32_t(i)));
  }
}

// One packed pass over up to 8 rows of a warp tile (the split-mode
// instantiation, kernels.cuh SPLIT): lane i < 8 holds row i of the tile — its
// first A entry, its entry and product counts — and `on` says whether the row
// belongs to this pass (the caller cuts the tile's short rows into passes of
// <= 32 entries and <= 32 products). Same scheme as packed_rows with the row
// data taken from the lanes: entry and product offsets by a scan over the 8
// lanes, an entry lane finds its row by a shuffle search. Returns the number
// of entries kept; `my_nnz` is set in the lanes of the pass's rows.
constexpr int kTileSlotBits = 3;
constexpr int kTileColBits = 32 - 5 - kTileSlotBits;

template <bool WIDE>
__device__ __forceinline__ uint32_t packed_tile_pass(const DevCsr& A, const DevCsr& B, uint64_t my_lo,
                                                     uint32_t my_na, uint32_t my_prod, bool on,
                                                     ShortOut& out, uint32_t& my_nnz) {
  using K = typename std::conditional<WIDE, unsigned long long, uint32_t>::type;
  using Off = typename std::conditional<WIDE, uint64_t, uint32_t>::type;
  constexpr int kSlotShift = int(sizeof(K)) * 8 - kTileSlotBits;
  const uint32_t lane = lane_id();
  const uint32_t n_eff = on ? my_na : 0u, p_eff = on ? my_prod : 0u;
  const uint32_t w = p_eff | (n_eff << 16);
  uint32_t x = w;  // inclusive scan over lanes 0..7 (the other lanes hold 0)
#pragma unroll
  for (int d = 1; d < 8; d <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, x, d);
    if (lane >= uint32_t(d)) x += t;
  }
  const uint32_t eoff = (x - w) >> 16, poff = (x - w) & 0xffffu;
  // entry lane -> row slot: the last slot whose entries start at or before it
  int slot = 0;
#pragma unroll
  for (int st = 4; st > 0; st >>= 1) {
    const uint32_t eo = __shfl_sync(kFull, eoff, slot + st);
    if (eo <= lane) slot += st;
  }
  const uint32_t e = lane - __shfl_sync(kFull, eoff, slot);
  const bool ent = e < __shfl_sync(kFull, n_eff, slot);
  const uint64_t rlo = __shfl_sync(kFull, my_lo, slot);
  Off kk = 0, bs = 0;
  double av = 0.0;
  uint32_t len = 0;
  if (ent) {
    kk = Off(ld_idx(A.ci + rlo + e, A.pol));
    av = ld_val(A.v + rlo + e, A.pol);
  }
  if (ent) {
    const uint64_t b0 = ld_idx(B.rp + kk, B.pol);
    bs = Off(b0);
    len = uint32_t(ld_idx(B.rp + kk + 1, B.pol) - b0);
  }
  const uint32_t incl = warp_incl_scan(len);
  const uint32_t excl = incl - len;  // lanes past the entries: == tot, never an owner
  const uint32_t tot = __shfl_sync(kFull, incl, 31);
  int src = 0;
#pragma unroll
  for (int st = 16; st > 0; st >>= 1) {
    const uint32_t ex = __shfl_sync(kFull, excl, src + st);
    if (ex <= lane) src += st;
  }
  const Off bsrc = __shfl_sync(kFull, bs, src) + (lane - __shfl_sync(kFull, excl, src));
  const double a = __shfl_sync(kFull, av, src);
  const uint32_t pslot = __shfl_sync(kFull, uint32_t(slot), src);
  const bool valid = lane < tot;
  uint32_t col = 0;
  double pv = 0.0;
  if (valid) {
    col = uint32_t(ld_idx(B.ci + bsrc, B.pol));
    pv = ld_val(B.v + bsrc, B.pol);
  }
  pv = valid ? __dmul_rn(a, pv) : 0.0;
  K key[1];
  key[0] = valid ? ((K(pslot) << kSlotShift) | (K(col) << 5) | K(lane)) : ~K(0);
  bitonic32_multi<1>(key);
  const K ck = key[0] >> 5;  // slot and column
  const double v = __shfl_sync(kFull, pv, uint32_t(key[0]) & 31u);
  const K prev = __shfl_up_sync(kFull, ck, 1);
  const bool head = valid && (lane == 0 || prev != ck);
  const uint32_t hm = __ballot_sync(kFull, head);
  const uint32_t above = hm & ~((2u << lane) - 1u);
  const uint32_t nxt = above ? uint32_t(__ffs(above) - 1) : tot;
  const uint32_t seg = head ? nxt - lane : 0u;
  const uint32_t max_seg = __reduce_max_sync(kFull, seg);
  double acc = v;
  for (uint32_t d = 1; d < max_seg; ++d) {
    const double t = __shfl_down_sync(kFull, v, d);
    if (d < seg) acc = __dadd_rn(acc, t);
  }
  const bool keep = head && (acc != 0.0);  // kernels.py:296 drops exact zeros
  const uint32_t km = __ballot_sync(kFull, keep);
  constexpr K kColMask = WIDE ? K(0xffffffffu) : K((1u << kTileColBits) - 1u);
  out.col = uint32_t(ck & kColMask);
  out.val = acc;
  out.keep = keep;
  out.rank = __popc(km & lanemask_lt());
  // a row's products fill lanes [poff, poff + products) of the sorted order
  if (on) {
    const uint32_t m = (p_eff >= 32u ? kFull : ((1u << p_eff) - 1u)) << poff;
    my_nnz = __popc(km & m);
  }
  return __popc(km);
}

// ---------------------------------------------------------------------------
// Medium rows: a warp and an open-addressing table (column -> running sum).
// The table lives in shared memory (kSmemSlots per warp); a row whose distinct
// columns pass 3/4 of that restarts on the warp's slice of a global table
// (kGlobalSlots, sized for the medium product limit), so correctness never
// depends on guessing the row's output size.

constexpr int kSmemSlots = 256;
constexpr int kGlobalSlots = 2048;
constexpr int kPosBits = 11;  // log2(kGlobalSlots): packed sort key = col << 11 | position
constexpr uint32_t kMediumLimit = 1024;  // products; longer rows go to k_long

template <int T, bool GLOBAL>
struct Table {
  uint32_t* keys;
  double* vals;
  static constexpr int kSlots = T;
  __device__ __forceinline__ uint32_t ldk(uint32_t h) const {
    if constexpr (GLOBAL) return __ldcg(keys + h);
    else return static_cast<volatile uint32_t*>(keys)[h];
  }
  __device__ __forceinline__ double ldv(uint32_t h) const {
    if constexpr (GLOBAL) return __ldcg(vals + h);
    else return static_cast<volatile double*>(vals)[h];
  }
  __device__ __forceinline__ void stv(uint32_t h, double v) const {
    if constexpr (GLOBAL) __stcg(vals + h, v);
    else static_cast<volatile double*>(vals)[h] = v;
  }
  __device__ __forceinline__ void stk(uint32_t h, uint32_t k) const {
    if constexpr (GLOBAL) __stcg(keys + h, k);
    else static_cast<volatile uint32_t*>(keys)[h] = k;
  }
  __device__ __forceinline__ static uint32_t hash(uint32_t col) {
    constexpr int kLog = __builtin_ctz(T);
    return (col * 0x9E3779B1u) >> (32 - kLog);
  }
  // dense[col] += p with the reference's touch accounting; returns true if
  // the column was new. Columns applied in one call are distinct across lanes.
  template <bool STATS>
  __device__ __forceinline__ bool apply(uint32_t col, double p, uint32_t& touches) const {
    uint32_t h = hash(col);
    bool fresh = false;
    while (true) {
      const uint32_t k = ldk(h);
      if (k == col) break;
      if (k == kEmptyKey) {
        const uint32_t old = atomicCAS(keys + h, kEmptyKey, col);
        if (old == kEmptyKey) { fresh = true; break; }
        if (old == col) break;
      }
      h = (h + 1) & (T - 1);
    }
    const double cur = fresh ? 0.0 : ldv(h);  // fresh slot == dense[x] == 0.0
    if (STATS && cur == 0.0) ++touches;
    stv(h, __dadd_rn(cur, p));
    return fresh;
  }
  __device__ __forceinline__ void clear() const {
    const uint32_t lane = lane_id();
    for (uint32_t s = lane; s < uint32_t(T); s += 32) stk(s, kEmptyKey);
    __syncwarp();
  }
  // Copy the occupied nonzero keys to out[0..cnt) (table left intact);
  // STATS: min/max over every occupied slot.
  template <bool STATS>
  __device__ __forceinline__ uint32_t gather_keys(uint32_t* out, uint32_t& smin,
                                                  uint32_t& smax) const {
    const uint32_t lane = lane_id();
    uint32_t cnt = 0, mn = kEmptyKey, mx = 0;
    for (uint32_t s0 = 0; s0 < uint32_t(T); s0 += 32) {
      const uint32_t k = ldk(s0 + lane);
      const bool occ = k != kEmptyKey;
      const bool keep = occ && (ldv(s0 + lane) != 0.0);
      if (STATS && occ) {
        mn = k < mn ? k : mn;
        mx = k > mx ? k : mx;
      }
      const uint32_t m = __ballot_sync(kFull, keep);
      if (keep) __stcg(out + cnt + __popc(m & lanemask_lt()), k);
      cnt += __popc(m);
    }
    if (STATS) {
      smin = __reduce_min_sync(kFull, mn);
      smax = __reduce_max_sync(kFull, mx);
    }
    __syncwarp();
    return cnt;
  }
  // value of a key known to be present
  __device__ __forceinline__ double lookup(uint32_t col) const {
    uint32_t h = hash(col);
    while (ldk(h) != col) h = (h + 1) & (T - 1);
    return ldv(h);
  }
  // Compact the occupied nonzero slots to the front (in place); returns the
  // count. STATS: min/max over every occupied slot, zero-valued ones included.
  template <bool STATS>
  __device__ __forceinline__ uint32_t compact(uint32_t& smin, uint32_t& smax) const {
    const uint32_t lane = lane_id();
    uint32_t cnt = 0, mn = kEmptyKey, mx = 0;
    for (uint32_t s0 = 0; s0 < uint32_t(T); s0 += 32) {
      const uint32_t s = s0 + lane;
      const uint32_t k = ldk(s);
      const double v = ldv(s);
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
        stk(pos, k);
        stv(pos, v);
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
};

// Overflowed rows (more distinct columns than the shared table holds):
// sort up to kMediumLimit column keys staged in global memory, in registers
// (32 per lane), out of line so the main kernel keeps its small footprint.
static __device__ __noinline__ void sort_keys_global(uint32_t* keys, uint32_t n) {
  const uint32_t lane = lane_id();
  constexpr int N = kMediumLimit / 32;
  uint32_t k[N];
  int E = 1;
  while (uint32_t(E) * 32u < n) E <<= 1;
#pragma unroll
  for (int e = 0; e < N; ++e) {
    const uint32_t idx = uint32_t(e) * 32u + lane;
    k[e] = (e < E && idx < n) ? __ldcg(keys + idx) : kEmptyKey;
  }
  bitonic_sort_dyn(k, E);
#pragma unroll
  for (int e = 0; e < N; ++e) {
    const uint32_t idx = uint32_t(e) * 32u + lane;
    if (e < E && idx < n) __stcg(keys + idx, k[e]);
  }
  __syncwarp();
}

// One chunk of up to 32 consecutive products of a group of <= 32 A entries.
// The walk keeps a cursor (entry i, offset within its B row). A chunk is
//  * single: up to 32 products of one B row (distinct columns) — the common
//    case for long B rows; no search, every lane takes product `off + lane`;
//  * packed: whole consecutive short B rows up to 32 products, located per
//    lane by a binary search over the entries' exclusive offsets.
// The B loads are issued when the chunk is made and consumed when applied.
struct Chunk {
  uint32_t n;       // products in the chunk (0: walk finished)
  bool single;      // all products from one B row: columns distinct
  uint64_t col;
  double bv;
  double a;
  uint32_t i_next;  // cursor after this chunk
  uint32_t off_next;
};

struct Group {  // one group of <= 32 A entries, one entry per lane
  uint32_t len, incl, excl, nent;
  uint64_t bs;
  double av;
};

__device__ __forceinline__ Chunk make_chunk(const DevCsr& B, const Group& g, uint32_t i,
                                            uint32_t off) {
  Chunk c;
  c.n = 0;
  c.single = true;
  c.col = kEmptyKey;
  c.bv = 0.0;
  c.a = 0.0;
  const uint32_t lane = lane_id();
  // skip exhausted / empty entries (warp-uniform)
  uint32_t li = i < g.nent ? __shfl_sync(kFull, g.len, i & 31u) : 0u;
  while (i < g.nent && off >= li) {
    ++i;
    off = 0;
    li = i < g.nent ? __shfl_sync(kFull, g.len, i & 31u) : 0u;
  }
  if (i >= g.nent) {
    c.i_next = i;
    c.off_next = 0;
    return c;
  }
  const uint32_t rem = li - off;
  const uint32_t nxt = i + 1 < g.nent ? __shfl_sync(kFull, g.len, (i + 1) & 31u) : 64u;
  if (rem >= 32 || rem + nxt > 32) {
    // single B row
    c.n = rem < 32 ? rem : 32;
    const uint64_t bsrc = __shfl_sync(kFull, g.bs, i & 31u) + off;
    c.a = __shfl_sync(kFull, g.av, i & 31u);
    if (lane < c.n) {
      c.col = ld_idx(B.ci + bsrc + lane, B.pol);
      c.bv = ld_val(B.v + bsrc + lane, B.pol);
    }
    off += c.n;
    if (off >= li) {
      ++i;
      off = 0;
    }
    c.i_next = i;
    c.off_next = off;
    return c;
  }
  // packed: from (i, off) through the last entry that still fits in 32
  c.single = false;
  const uint32_t cs = __shfl_sync(kFull, g.excl, i & 31u) + off;
  const uint32_t lim = cs + 32;
  const uint32_t bm = __ballot_sync(kFull, lane < g.nent && g.incl > cs && g.incl <= lim);
  const uint32_t last = 31 - __clz(bm);  // bm != 0: entry i itself ends within lim
  const uint32_t ce = __shfl_sync(kFull, g.incl, last);
  c.n = ce - cs;
  const uint32_t q = cs + lane;
  int e = int(i);
#pragma unroll
  for (int st = 16; st > 0; st >>= 1) {
    const uint32_t ex = __shfl_sync(kFull, g.excl, (e + st) & 31);
    if (e + st <= int(last) && ex <= q) e += st;
  }
  const uint64_t bsrc = __shfl_sync(kFull, g.bs, e);
  c.a = __shfl_sync(kFull, g.av, e);
  const uint32_t j = q - __shfl_sync(kFull, g.excl, e);
  if (lane < c.n) {
    c.col = ld_idx(B.ci + bsrc + j, B.pol);
    c.bv = ld_val(B.v + bsrc + j, B.pol);
  }
  c.i_next = last + 1;
  c.off_next = 0;
  return c;
}

// Apply one chunk; returns the number of new columns it inserted.
template <class Tab, bool STATS>
__device__ __forceinline__ uint32_t apply_chunk(const Tab& tab, const Chunk& c,
                                                uint32_t& touches) {
  const uint32_t lane = lane_id();
  const bool act = lane < c.n;
  const uint32_t col = uint32_t(c.col);
  const double p = __dmul_rn(c.a, c.bv);
  bool fresh = false;
  if (c.single) {
    if (act) fresh = tab.template apply<STATS>(col, p, touches);
    __syncwarp();
  } else {
    // equal columns from different B rows: apply in rounds, lowest product first
    const uint32_t am = __ballot_sync(kFull, act);
    const uint32_t peers = __match_any_sync(kFull, act ? col : kEmptyKey) & am;
    const uint32_t rank = __popc(peers & lanemask_lt());
    const uint32_t rounds = __reduce_max_sync(kFull, act ? rank : 0u) + 1u;
    for (uint32_t rr = 0; rr < rounds; ++rr) {
      if (act && rank == rr) fresh |= tab.template apply<STATS>(col, p, touches);
      __syncwarp();
    }
  }
  return __popc(__ballot_sync(kFull, fresh));
}

// One whole B row (<= 32 entries) as a chunk: entry i of the group, one
// product per lane (distinct columns). The fast path of medium_accumulate for
// groups whose B rows all fit a warp and are long enough that packing several
// into one chunk would not pay (C4: 27-entry rows) — no cursor bookkeeping.
__device__ __forceinline__ Chunk entry_chunk(const DevCsr& B, const Group& g, uint32_t i) {
  Chunk c;
  c.n = 0;
  c.single = true;
  c.col = kEmptyKey;
  c.bv = 0.0;
  c.a = 0.0;
  c.i_next = i + 1;
  c.off_next = 0;
  if (i < g.nent) {  // warp-uniform
    const uint32_t lane = lane_id();
    c.n = __shfl_sync(kFull, g.len, i & 31u);
    const uint64_t bs = __shfl_sync(kFull, g.bs, i & 31u);
    c.a = __shfl_sync(kFull, g.av, i & 31u);
    if (lane < c.n) {
      c.col = ld_idx(B.ci + bs + lane, B.pol);
      c.bv = ld_val(B.v + bs + lane, B.pol);
    }
  }
  return c;
}

// Accumulate the whole row into `tab`. Returns false (and leaves the table
// dirty) if the row's distinct columns exceed `limit`.
template <class Tab, bool STATS>
__device__ __forceinline__ bool medium_accumulate(const DevCsr& A, const DevCsr& B, uint64_t lo,
                                                  uint64_t hi, const Tab& tab, uint32_t limit,
                                                  uint32_t& touches) {
  const uint32_t lane = lane_id();
  uint32_t inserted = 0;
  for (uint64_t abase = lo; abase < hi; abase += 32) {
    Group g;
    g.nent = uint32_t(hi - abase < 32 ? hi - abase : 32);
    const uint64_t e = abase + lane;
    g.len = 0;
    g.bs = 0;
    g.av = 0.0;
    if (lane < g.nent) {
      const uint64_t k = ld_idx(A.ci + e, A.pol);
      g.av = ld_val(A.v + e, A.pol);
      g.bs = ld_idx(B.rp + k, B.pol);
      g.len = uint32_t(ld_idx(B.rp + k + 1, B.pol) - g.bs);
    }
    g.incl = warp_incl_scan(g.len);
    g.excl = g.incl - g.len;
    const uint32_t lmax = __reduce_max_sync(kFull, g.len);
    if (lmax <= 32 && __shfl_sync(kFull, g.incl, 31) >= 16u * g.nent) {
      // every B row is one chunk, three in flight, applied in entry order
      Chunk e0 = entry_chunk(B, g, 0), e1 = entry_chunk(B, g, 1), e2 = entry_chunk(B, g, 2);
#pragma unroll 1
      for (uint32_t i = 0; i < g.nent; i += 3) {
        inserted += apply_chunk<Tab, STATS>(tab, e0, touches);
        if (inserted > limit) return false;
        e0 = entry_chunk(B, g, i + 3);
        if (i + 1 >= g.nent) break;
        inserted += apply_chunk<Tab, STATS>(tab, e1, touches);
        if (inserted > limit) return false;
        e1 = entry_chunk(B, g, i + 4);
        if (i + 2 >= g.nent) break;
        inserted += apply_chunk<Tab, STATS>(tab, e2, touches);
        if (inserted > limit) return false;
        e2 = entry_chunk(B, g, i + 5);
      }
      continue;
    }
    // three chunks in flight
    Chunk c0 = make_chunk(B, g, 0, 0);
    Chunk c1 = make_chunk(B, g, c0.i_next, c0.off_next);
    Chunk c2 = make_chunk(B, g, c1.i_next, c1.off_next);
    while (c0.n) {
      inserted += apply_chunk<Tab, STATS>(tab, c0, touches);
      if (inserted > limit) return false;
      c0 = make_chunk(B, g, c2.i_next, c2.off_next);
      if (!c1.n) break;
      inserted += apply_chunk<Tab, STATS>(tab, c1, touches);
      if (inserted > limit) return false;
      c1 = make_chunk(B, g, c0.i_next, c0.off_next);
      if (!c2.n) break;
      inserted += apply_chunk<Tab, STATS>(tab, c2, touches);
      if (inserted > limit) return false;
      c2 = make_chunk(B, g, c1.i_next, c1.off_next);
    }
  }
  return true;
}

}  // namespace spmmm
