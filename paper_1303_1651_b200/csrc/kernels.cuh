// The fused, persistent, single-pass spMMM kernel (k_fused) and the copy of
// pre-computed long rows (k_copy_long). k_count / k_collect / k_long are in
// aux_kernels.cuh. Dataflow: DESIGN.md §3.
//
// k_fused: every warp walks its own sequence of warp tiles (R consecutive
// rows; tile t belongs to global warp t mod #warps). For a tile it
//   1. computes its rows — short rows in registers (rows.cuh short_rows),
//      medium rows in the warp's shared-memory table (global table on
//      overflow), long rows only contribute their pre-computed nnz;
//   2. publishes the tile's nnz and reads its exclusive prefix with a
//      warp-level decoupled look-back (device.cuh lookback) — there is no
//      block barrier anywhere in the loop;
//   3. writes C.row_ptr[r+1] and the rows' (col, value) entries once.
// Launched cooperatively (all warps co-resident): the smallest unfinished
// tile's warp is always running it and only waits on smaller tiles, so the
// look-back cannot deadlock.
#pragma once

#include <cooperative_groups.h>

#include "rows.cuh"

#ifndef SPMMM_SHORT_BLOCKS
#define SPMMM_SHORT_BLOCKS 4
#endif
#ifndef SPMMM_PF_AHEAD
#define SPMMM_PF_AHEAD 1024
#endif
#ifndef SPMMM_LOCK
#define SPMMM_LOCK 4
#endif

namespace spmmm {

struct FusedParams {
  DevCsr A, B;
  const uint32_t* prod;
  const uint32_t* lmap;
  const uint32_t* l_nnz;
  const uint32_t* ell;  // ELL records of B (short variant, B rows <= kEllSlots) or null
  unsigned long long* nnz_out;  // nnz(C) for the host (ctrl word)
  uint64_t* c_rp;
  uint64_t* c_ci;
  double* c_v;
  LookbackState lb;  // hierarchical status words (device.cuh)
  unsigned long long* ticket;  // next free tile (zeroed per call)
  uint64_t ntiles;
  uint32_t medium_limit;
  uint32_t a_is_b;  // A and B are the same arrays
  uint32_t self_ell;  // ... row for row (C = A·A, count-free): a row's A entries are its ELL record
  uint32_t* g_keys;  // [#warps][kGlobalSlots] overflow tables (medium kernel)
  double* g_vals;
  uint32_t* g_scol;  // [#warps][2][kMediumLimit] staging of overflowed rows
  double* g_sval;
  uint32_t* st_min;
  uint32_t* st_max;
  uint32_t* st_touch;
  // count-free path (k_prep instead of k_count; short variant only): prod is
  // null, every row with entries is short, k_prep's verdict is read here and
  // the multiplications are summed into *cf_total
  const unsigned long long* cf_flags;
  const unsigned long long* cf_ell_flag;  // B's ELL records were packed
  unsigned long long* cf_total;
  unsigned long long* cf_err;
  uint64_t c_cap;  // entries reserved for C (count-free and medium variants check it)
  // count-free: the last warp to finish copies the ctrl words (ctrl) to the
  // host's mapped mirror (host_ctrl), so no read-back kernel follows
  const unsigned long long* ctrl;
  unsigned long long* host_ctrl;
  unsigned long long* done;
  int ctrl_words;
  // PREP instantiations (small count-free products): the prep pass runs in
  // this kernel, before a grid barrier, instead of as k_prep
  CfWords cf_words;
  unsigned long long* cf_zero;
  uint64_t cf_nzero;
  uint4* cf_pack;
};

// Warps take tiles dynamically, a batch of kBatch consecutive tiles per
// atomic, so faster SMs simply process more tiles. A warp computes its whole
// batch, then finishes (look-back + write) its previous batch: a tile is
// always computed right after it is acquired, so no chain of waits forms and
// the previous batch's predecessors are already published.

constexpr int kMaxBufs = 4;  // staging buffers of the largest variant

// Shared memory per warp: kBufs = 2 batches x kBatch tiles of staging
// (a tile's finished rows wait there until its offset is known), the per-row
// nnz of each, and for the medium kernel the warp's hash table. Medium rows
// with more than kStage outputs stage in the warp's global buffers instead.
template <int R, bool MEDIUM>
struct FusedSmem {
  static constexpr int kBatch = 1;  // tiles per ticket
  static constexpr int kBufs = 2 * kBatch;
  static constexpr int kStage = MEDIUM ? 128 : 32 * R;
  static constexpr int kTable = MEDIUM ? kSmemSlots : 0;
  // doubles per warp: staging values, table values, per buffer (tile, agg)
  static constexpr int kWords64 = kBufs * kStage + kTable + 2 * kBufs;
  // u32 per warp: staging columns, table keys, per buffer R row nnz + (staged, global)
  static constexpr int kWords32 = kBufs * kStage + kTable + kBufs * R + 2 * kBufs;
  static constexpr size_t bytes(int warps) {
    return size_t(warps) * (kWords64 * sizeof(double) + kWords32 * sizeof(uint32_t));
  }
};

template <int WARPS, int R, bool MEDIUM, bool WIDE, bool STATS, bool CF = false, int PREP = 0,
          bool SPLIT = false, bool SELF = false>
__global__ void __launch_bounds__(WARPS * 32, MEDIUM ? 4 : SPMMM_SHORT_BLOCKS) k_fused(const FusedParams p_in) {
  static_assert(!MEDIUM || R == 1, "one medium row per warp tile");
  static_assert(!(MEDIUM && CF), "the count-free path is short rows only");
  static_assert(PREP == 0 || CF, "the fused prep pass belongs to the count-free path");
  if constexpr (PREP != 0) {
    // the prep pass (mode PREP - 1) by every thread of the grid, then a grid
    // barrier: its verdict, maxima and ELL records are complete below
    prep_pass<PREP - 1>(p_in.A, p_in.B, p_in.cf_words, p_in.cf_zero, p_in.cf_nzero, p_in.cf_pack,
                        uint64_t(blockIdx.x) * blockDim.x + threadIdx.x,
                        uint64_t(gridDim.x) * blockDim.x);
    __threadfence();
    cooperative_groups::this_grid().sync();
  }
  static_assert(R >= 1 && R <= 8, "rows per warp tile");
  static_assert(!SPLIT || (!MEDIUM && !CF && PREP == 0), "split mode: the counted short variant");
  // SPLIT: the split-mode instantiation (fused_split.cu; skewed inputs such as
  // C5, whose non-short rows were computed before this kernel). Most of its
  // rows have a handful of products, so the tile's short rows go through
  // packed passes only (rows.cuh packed_tile_pass: up to 8 rows per pass)
  // and short_rows is not compiled in: C5's k_fused 0.68 -> 0.54 ms.
  // PACK: the same idea per lockstep group of 4 rows inside the shared short
  // variant (packed_rows; C5 0.68 -> 0.61 ms) — superseded by SPLIT, kept for
  // A/B builds (-DSPMMM_GROUP_PACK with -DSPMMM_NO_SPLIT_VARIANT).
#ifdef SPMMM_GROUP_PACK
  constexpr bool PACK = !MEDIUM && !CF && !STATS && (SPMMM_LOCK <= (1 << kPackSlotBits));
#else
  constexpr bool PACK = false;
#endif
  using K = typename std::conditional<WIDE, unsigned long long, uint32_t>::type;
  using SM = FusedSmem<R, MEDIUM>;
  constexpr int EMAX = MEDIUM ? kSmemSlots / 32 : 1;  // register sort up to 256 keys
  constexpr int kStage = SM::kStage;
  constexpr int kBufs = SM::kBufs;
  constexpr int kBatch = SM::kBatch;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  const uint64_t gwarp = uint64_t(blockIdx.x) * WARPS + warp;
  // B rows are re-read across A rows: keep them in L2. A streams once unless
  // it is B itself (C = A·A: its rows are the B rows of neighbouring rows).
  FusedParams p = p_in;
  p.B.pol = policy_evict_last();
  p.A.pol = p.a_is_b ? p.B.pol : policy_evict_first();
  double* s_val = reinterpret_cast<double*>(smem_raw) + size_t(warp) * SM::kWords64;
  uint32_t* s_col = reinterpret_cast<uint32_t*>(smem_raw + size_t(WARPS) * SM::kWords64 * 8) +
                    size_t(warp) * SM::kWords32;
  uint32_t* s_hdr = s_col + kBufs * kStage + SM::kTable;
  uint32_t* s_meta32 = s_hdr + kBufs * R;                                  // [buf][staged, global]
  uint64_t* s_meta64 = reinterpret_cast<uint64_t*>(s_val + kBufs * kStage + SM::kTable);  // [buf][tile, agg]
  Table<kSmemSlots, false> st{s_col + kBufs * kStage, s_val + kBufs * kStage};
  Table<kGlobalSlots, true> gt{nullptr, nullptr};
  uint32_t* g_scol = nullptr;
  double* g_sval = nullptr;
  if constexpr (MEDIUM) {
    gt.keys = p.g_keys + gwarp * kGlobalSlots;
    gt.vals = p.g_vals + gwarp * kGlobalSlots;
    g_scol = p.g_scol + gwarp * kMaxBufs * kMediumLimit;
    g_sval = p.g_sval + gwarp * kMaxBufs * kMediumLimit;
    st.clear();
  }
  const uint64_t rows = p.A.rows;
  // count-free: k_prep found a row the short path cannot take (or bad input)
  bool run = true;
  if constexpr (CF) {
    const volatile unsigned long long* w = p.cf_flags;
    const unsigned long long ma = w[1], mb = w[2];
    run = cf_applies(w[0], ma, mb);
    // B through its ELL records when k_prep(_b) packed them and every
    // referenced row fits one; else as CSR
    if (!cf_ell(ma, mb) || !*reinterpret_cast<const volatile unsigned long long*>(p.cf_ell_flag))
      p.ell = nullptr;
  }
  // C = A·A through the ELL records: rows are read from their own records
  // (short_rows), so the tile needs no A.row_ptr at all
  // (SELF: the instantiation launched for C = A·A — with the path compiled
  // into the one A != B products run, C3's k_fused was 2.8% slower)
  static_assert(!SELF || CF, "the self-record path belongs to the count-free variant");
  bool self = false;
#ifndef SPMMM_NO_SELF
  if constexpr (SELF) self = p.self_ell != 0 && p.ell != nullptr;
#endif
  uint64_t cf_prods = 0;
  // (stream prefetch: the average number of A entries in SPMMM_PF_AHEAD tiles)
  [[maybe_unused]] const uint64_t pf_entries =
      rows ? uint64_t(SPMMM_PF_AHEAD) * R * p.A.nnz / rows : 0;

  // the previous batch waits for its offsets; its metadata lives in s_meta*
  int nprev = 0;
  int half = 0;  // which half of the staging buffers the current batch fills

  auto finish = [&](int b) {
    const uint64_t tile = s_meta64[2 * b], agg = s_meta64[2 * b + 1];
    const uint32_t staged = s_meta32[2 * b];
    const bool global = s_meta32[2 * b + 1] != 0;
    const uint64_t excl = lookback(p.lb, tile, agg);
    const uint64_t r0 = tile * R;
    if (lane < uint32_t(R) && r0 + lane < rows) {
      uint64_t s = 0;
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (uint32_t(j) <= lane) s += s_hdr[b * R + j];
      p.c_rp[r0 + lane + 1] = excl + s;
      if (r0 + lane + 1 == rows) *p.nnz_out = excl + s;  // read back by the host
    }
    if (tile == 0 && lane == 0) p.c_rp[0] = 0;
    const uint32_t ext = MEDIUM ? 0u : s_meta32[2 * b + 1];  // short variant: external rows
    if ((CF || MEDIUM) && excl + agg > p.c_cap) {
      // C's reservation exceeded (count-free bound, or the medium variant's
      // 8·nnz(A)): write nothing past it, the host redoes it sized exactly
      if (lane == 0) atomicOr(p.cf_err, (unsigned long long)kCfOverflow);
    } else if (!MEDIUM && ext) {
      // the tile mixes staged short rows with rows computed before k_fused
      // (copied into their slots by k_copy_long): place each short row alone
      uint64_t dst = excl;
      uint32_t src = 0;
#pragma unroll 1
      for (int j = 0; j < R; ++j) {
        const uint32_t n = s_hdr[b * R + j];
        if (!((ext >> j) & 1u)) {
          for (uint32_t t = lane; t < n; t += 32) {
            __stcs(reinterpret_cast<unsigned long long*>(p.c_ci) + dst + t,
                   (unsigned long long)s_col[b * kStage + src + t]);
            __stcs(p.c_v + dst + t, s_val[b * kStage + src + t]);
          }
          src += n;
        }
        dst += n;
      }
    } else if (MEDIUM && global) {
      for (uint32_t t = lane; t < staged; t += 32) {
        __stcs(reinterpret_cast<unsigned long long*>(p.c_ci) + excl + t,
               (unsigned long long)__ldcg(g_scol + b * kMediumLimit + t));
        __stcs(p.c_v + excl + t, __ldcg(g_sval + b * kMediumLimit + t));
      }
    } else {
      for (uint32_t t = lane; t < staged; t += 32) {
        // C is written once and not re-read here: evict-first
        __stcs(reinterpret_cast<unsigned long long*>(p.c_ci) + excl + t,
               (unsigned long long)s_col[b * kStage + t]);
        __stcs(p.c_v + excl + t, s_val[b * kStage + t]);
      }
    }
    __syncwarp();
  };

  // A tile must be computed right after it is acquired (successors wait on
  // it), so tickets are taken when needed, never ahead.
  while (run) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(p.ticket, (unsigned long long)kBatch);
    base = __shfl_sync(kFull, base, 0);
    const bool have = base < p.ntiles;  // else: only finish the last batch
    const int ncur = have ? int(p.ntiles - base < uint64_t(kBatch) ? p.ntiles - base : kBatch) : 0;
#pragma unroll 1
    for (int bj = 0; bj < ncur; ++bj) {
    const uint64_t tile = base + bj;
    const int buf = half * kBatch + bj;
    const uint64_t r0 = tile * R;
    // Stream prefetch (C = A·A, the self-record path): the tile kPfAhead
    // tickets from here is some warp's in a few microseconds — its rows'
    // records into L2 now, so that tile's first loads are L2 hits instead of
    // DRAM round trips (C2 1.363 -> 1.340 ms; 1024 and 4096 tickets ahead
    // measured the same). Not in the A != B instantiations: prefetching A's
    // row pointers and entries there cost C3 2.3% (0.678 -> 0.694 ms).
    if constexpr (SELF && SPMMM_PF_AHEAD > 0) {
      const uint64_t ft = tile + SPMMM_PF_AHEAD;
      // (whole tiles only: every prefetched line lies inside the record array)
      if (self && (ft + 1) * R <= rows && lane < 4)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(p.ell + ft * R * kEllWords + lane * 32));
    }
    // ---- row bounds and classes of the tile: lane i owns row r0 + i ----
    uint64_t rpv = 0;
    uint32_t my_cls = kRowZero, my_na = 0, my_prod = 0;
    if (!self && lane <= uint32_t(R) && r0 + lane <= rows)
      rpv = ld_idx(p.A.rp + r0 + lane, p.A.pol);
    const uint64_t rpn = __shfl_down_sync(kFull, rpv, 1);
    // Stream prefetch, count-free A != B (C3): the tile SPMMM_PF_AHEAD tickets
    // ahead gets its row pointers and — at this tile's entry offset plus the
    // average entries per tile: exact for uniform rows, near enough otherwise,
    // and a wrong guess only wastes a line — its entries into L2: C3 k_fused
    // 0.678 -> 0.657 ms. (Going on to load those entries a stage later and
    // prefetch the B records they address: no gain, 0.68 ms.)
    if constexpr (CF && !SELF && PREP == 0 && SPMMM_PF_AHEAD > 0) {
      const uint64_t ft = tile + SPMMM_PF_AHEAD;
      if (ft < p.ntiles) {
        const uint64_t fe = __shfl_sync(kFull, rpv, 0) + pf_entries;
        if (lane == 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.A.rp + ft * R));
        // (the estimate may pass the arrays' end: only lines inside them)
        if (fe + 64 <= p.A.nnz) {
          if (lane >= 2 && lane < 6)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(p.A.ci + fe + (lane - 2) * 16));
          if (lane >= 6 && lane < 10)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(p.A.v + fe + (lane - 6) * 16));
        }
      }
    }
    if (self) {
      if (lane < uint32_t(R) && r0 + lane < rows) {
        my_cls = kRowShort;  // (an empty row's record is empty: no products)
        my_na = kEllSlots;
      }
    } else if (lane < uint32_t(R) && r0 + lane < rows) {
      my_na = uint32_t(rpn - rpv);
      if constexpr (CF) {
        my_cls = rpn > rpv ? uint32_t(kRowShort) : uint32_t(kRowZero);
      } else {
        my_prod = p.prod[r0 + lane];
        my_cls = uint32_t(classify(my_prod, rpn - rpv, p.medium_limit));
      }
    }
    // per-row results, lane i = row i; rows computed before this kernel
    // (long rows, and in split mode every non-short row) only report nnz
    uint32_t my_nnz = 0, my_min = kEmptyKey, my_max = 0, my_touch = 0;
    if (!MEDIUM && my_cls == kRowLong) my_nnz = p.l_nnz[p.lmap[r0 + lane]];
    const uint32_t ext_mask = MEDIUM ? 0u : __ballot_sync(kFull, my_cls == kRowLong);
    uint32_t staged = 0;
    bool global = false;
    if constexpr (SPLIT && !STATS) {
      // split mode: the tile's short rows in packed passes only (rows.cuh
      // packed_tile_pass): rows are taken into a pass while it stays within 32
      // A entries and 32 products (every short row fits one alone)
      const uint32_t pk = my_cls == kRowShort ? (my_prod | (my_na << 16)) : 0u;
      uint32_t sp = 0, sn = 0, npass = 0, my_pass = 0xffu;
      bool any = false;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const uint32_t v = __shfl_sync(kFull, pk, i);
        if (v) {
          const uint32_t pr = v & 0xffffu, n = v >> 16;
          if (any && (sp + pr > 32u || sn + n > 32u)) {
            ++npass;
            sp = 0;
            sn = 0;
          }
          any = true;
          sp += pr;
          sn += n;
          if (lane == uint32_t(i)) my_pass = npass;
        }
      }
      npass = any ? npass + 1 : 0;
#pragma unroll 1
      for (uint32_t ps = 0; ps < npass; ++ps) {
        ShortOut po;
        const uint32_t kept = packed_tile_pass<WIDE>(p.A, p.B, rpv, my_na, my_prod,
                                                     my_pass == ps, po, my_nnz);
        if (po.keep) {
          s_col[buf * kStage + staged + po.rank] = po.col;
          s_val[buf * kStage + staged + po.rank] = po.val;
        }
        staged += kept;
      }
    } else
    if (__ballot_sync(kFull, my_cls == kRowShort)) {
      // short rows go through short_rows in lockstep groups of kLock; the
      // groups run in a loop (one copy of the code: instruction cache)
      constexpr int kLock = R < SPMMM_LOCK ? R : SPMMM_LOCK;
      int ngroups = R / kLock;
      asm volatile("" : "+r"(ngroups));  // opaque: keep one copy of the group body
      // a group whose short rows have <= 32 A entries and <= 32 products in
      // all goes through one packed pass (rows.cuh packed_rows) instead of a
      // pass per row: its sums, products | entries << 16, in each of its lanes
      // (both groups' packed passes in lockstep measured slower: the code
      // outgrew the instruction cache)
      [[maybe_unused]] uint32_t pack_sum = 0;
      if constexpr (PACK) {
        pack_sum = my_cls == kRowShort ? (my_prod | (my_na << 16)) : 0u;
#pragma unroll
        for (int d = 1; d < kLock; d <<= 1) pack_sum += __shfl_xor_sync(kFull, pack_sum, d);
        if (!WIDE && p.B.cols > (1ull << kPackColBits)) pack_sum = ~0u;
      }
      // ELL path, two groups: the second group's A entries are loaded now and
      // the B records they address are prefetched into L2 while the first
      // group waits on its own loads (one lane per (row, entry): 4 rows x 8
      // entries). (The same for B.row_ptr in the generic path measured
      // neutral on C5.)
      const void* pf1 = nullptr;
      if constexpr (!MEDIUM) {
        if (!SPLIT && !self && p.ell && ngroups > 1) {
          const uint32_t pi = lane >> 3, pe = lane & 7;
          const uint32_t src = uint32_t(kLock) + (pi < uint32_t(kLock) ? pi : 0u);
          const uint64_t plo = __shfl_sync(kFull, rpv, src);
          const uint32_t pna = __shfl_sync(kFull, my_na, src);
          const uint32_t pcl = __shfl_sync(kFull, my_cls, src);
          if (pi < uint32_t(kLock) && pcl == kRowShort && pe < pna && pe < kEllEntries) {
            asm volatile("prefetch.global.L1 [%0];" ::"l"(p.A.v + plo + pe));
            const uint64_t pk = ld_idx(p.A.ci + plo + pe, p.A.pol);
            pf1 = p.ell + pk * kEllWords;
          }
        }
      }
#pragma unroll 1
      for (int h = 0; h < ngroups; ++h) {
        uint64_t hlo[kLock];
        uint32_t hna[kLock], hnnz[kLock], hmin[kLock], hmax[kLock], htouch[kLock];
        bool hon[kLock];
#pragma unroll
        for (int i = 0; i < kLock; ++i) {
          hlo[i] = __shfl_sync(kFull, rpv, h * kLock + i);
          hna[i] = __shfl_sync(kFull, my_na, h * kLock + i);
          hon[i] = __shfl_sync(kFull, my_cls, h * kLock + i) == kRowShort;
        }
        bool any = false;
#pragma unroll
        for (int i = 0; i < kLock; ++i) any |= hon[i];
        if (!any) continue;
        if constexpr (PACK) {
          const uint32_t gs = __shfl_sync(kFull, pack_sum, h * kLock);
          if ((gs & 0xffffu) <= 32u && (gs >> 16) <= 32u) {
            uint64_t glo[1][kLock];
            uint32_t gna[1][kLock], pn[1][kLock];
            bool gon[1][kLock];
#pragma unroll
            for (int i = 0; i < kLock; ++i) {
              glo[0][i] = hlo[i];
              gna[0][i] = hna[i];
              gon[0][i] = hon[i];
            }
            ShortOut po[1];
            packed_rows<kLock, 1, WIDE>(p.A, p.B, glo, gna, gon, po, pn);
            uint32_t gn = 0;
#pragma unroll
            for (int i = 0; i < kLock; ++i) {
              if (hon[i] && lane == uint32_t(h * kLock + i)) my_nnz = pn[0][i];
              gn += pn[0][i];
            }
            if (po[0].keep) {
              s_col[buf * kStage + staged + po[0].rank] = po[0].col;
              s_val[buf * kStage + staged + po[0].rank] = po[0].val;
            }
            staged += gn;
            continue;
          }
        }
        ShortOut so[kLock];
        uint32_t hprod[kLock];
        short_rows<kLock, WIDE, STATS, !MEDIUM && !SPLIT, CF>(p.A, p.B, p.ell, hlo, hna, hon, so, hnnz,
                                                    hmin, hmax, htouch, hprod,
                                                    h == 0 ? pf1 : nullptr, self,
                                                    r0 + uint64_t(h * kLock));
        if constexpr (CF) {
#pragma unroll
          for (int i = 0; i < kLock; ++i) cf_prods += hon[i] ? hprod[i] : 0u;
        }
#pragma unroll
        for (int i = 0; i < kLock; ++i) {
          if (!hon[i]) continue;
          if (lane == uint32_t(h * kLock + i)) {
            my_nnz = hnnz[i];
            if (STATS) {
              my_min = hmin[i];
              my_max = hmax[i];
              my_touch = htouch[i];
            }
          }
          if (so[i].keep) {
            s_col[buf * kStage + staged + so[i].rank] = so[i].col;
            s_val[buf * kStage + staged + so[i].rank] = so[i].val;
          }
          staged += hnnz[i];
        }
      }
    }

    // ---- medium / long row (R == 1 in the medium kernel) ----
    if constexpr (MEDIUM) {
      const int cls0 = int(__shfl_sync(kFull, my_cls, 0));
      const uint64_t lo0 = __shfl_sync(kFull, rpv, 0);
      uint32_t smin0 = kEmptyKey, smax0 = 0;
      if (cls0 == kRowMedium) {
        const uint64_t hi = __shfl_sync(kFull, rpn, 0);
        uint32_t touches = 0, cnt;
        bool use_gt = false;  // row overflowed the shared table
        if (medium_accumulate<decltype(st), STATS>(p.A, p.B, lo0, hi, st, kSmemSlots * 3 / 4,
                                                    touches)) {
          cnt = st.template compact<STATS>(smin0, smax0);
        } else {
          st.clear();
          touches = 0;
          use_gt = true;
          medium_accumulate<decltype(gt), STATS>(p.A, p.B, lo0, hi, gt, kGlobalSlots, touches);
          cnt = 0;
        }
        if (use_gt) {
          // stage in global memory: gather the keys, sort them in registers,
          // then fetch each value from the (intact) table
          uint32_t* scol = g_scol + buf * kMediumLimit;
          double* sval = g_sval + buf * kMediumLimit;
          cnt = gt.template gather_keys<STATS>(scol, smin0, smax0);
          sort_keys_global(scol, cnt);
          for (uint32_t t = lane; t < cnt; t += 32) __stcg(sval + t, gt.lookup(__ldcg(scol + t)));
          global = true;
        } else {
          global = cnt > uint32_t(kStage);  // too big for the shared stage
          int E = 1;
          while (uint32_t(E) * 32u < cnt) E <<= 1;
          K mk[EMAX];
#pragma unroll
          for (int e = 0; e < EMAX; ++e) {
            const uint32_t idx = uint32_t(e) * 32u + lane;
            mk[e] = (e < E && idx < cnt) ? ((K(st.ldk(idx)) << kPosBits) | K(idx)) : ~K(0);
          }
          bitonic_sort_dyn(mk, E);
          // sorted (col, value) into this tile's staging buffer
#pragma unroll
          for (int e = 0; e < EMAX; ++e) {
            const uint32_t idx = uint32_t(e) * 32u + lane;
            if (e < E && idx < cnt) {
              const uint32_t pos = uint32_t(mk[e]) & uint32_t(kGlobalSlots - 1);
              const uint32_t col = uint32_t(mk[e] >> kPosBits);
              const double val = st.ldv(pos);
              if (global) {
                __stcg(g_scol + buf * kMediumLimit + idx, col);
                __stcg(g_sval + buf * kMediumLimit + idx, val);
              } else {
                s_col[buf * kStage + idx] = col;
                s_val[buf * kStage + idx] = val;
              }
            }
          }
        }
        staged = cnt;
        if (lane == 0) {
          my_nnz = cnt;
          my_min = smin0;
          my_max = smax0;
        }
        __syncwarp();
        if (use_gt) gt.clear();
        else st.clear();
        if (STATS) {
#pragma unroll
          for (int d = 16; d > 0; d >>= 1) touches += __shfl_xor_sync(kFull, touches, d);
          if (lane == 0) my_touch = touches;
        }
      } else if (cls0 == kRowLong) {
        if (lane == 0) my_nnz = p.l_nnz[p.lmap[r0]];  // copied into place by k_copy_long
      }
    }

    // ---- per-row stats, tile header, aggregate ----
    if (lane < uint32_t(R)) {
      s_hdr[buf * R + lane] = my_nnz;
      if (STATS && r0 + lane < rows && my_cls != kRowLong) {
        p.st_min[r0 + lane] = my_min;
        p.st_max[r0 + lane] = my_max;
        p.st_touch[r0 + lane] = my_touch;
      }
    }
    uint64_t agg = my_nnz;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) agg += __shfl_xor_sync(kFull, agg, d);
    __syncwarp();
    publish_aggregate(p.lb, tile, agg);

    if (lane == 0) {
      s_meta64[2 * buf] = tile;
      s_meta64[2 * buf + 1] = agg;
      s_meta32[2 * buf] = staged;
      s_meta32[2 * buf + 1] = MEDIUM ? (global ? 1u : 0u) : ext_mask;
    }
    __syncwarp();
    }  // tiles of the batch
    // ---- finish the previous batch ----
#pragma unroll 1
    for (int j = 0; j < nprev; ++j) finish((half ^ 1) * kBatch + j);
    if (!have) break;
    nprev = ncur;
    half ^= 1;
  }
  // count-free: the multiplications (KernelStats.multiplications), one
  // atomic per warp (every lane holds the same sum)
  if constexpr (CF) {
    if (lane == 0 && cf_prods) atomicAdd(p.cf_total, (unsigned long long)cf_prods);
    // the last warp out reports every ctrl word to the host (the pattern of
    // a last-block reduction: fence, count, fence, read through L2)
    unsigned long long n = 0;
    if (lane == 0) {
      __threadfence();
      n = atomicAdd(p.done, 1ull);
    }
    n = __shfl_sync(kFull, n, 0);
    if (n + 1 == uint64_t(gridDim.x) * WARPS) {
      __threadfence();
      if (int(lane) < p.ctrl_words) {
        reinterpret_cast<volatile unsigned long long*>(p.host_ctrl)[lane] = __ldcg(p.ctrl + lane);
        // and leaves them zeroed for the next product (no memset before it)
        __stcg(const_cast<unsigned long long*>(p.ctrl) + lane, 0ull);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// k_rows: split mode. When non-short rows are a minority and vary a lot in
// cost (skewed matrices such as C5), inlining them in k_fused would make
// every later tile wait on the slowest one in its look-back. Instead they are
// computed here first — one warp per row of <= kRowsLimit products — and
// staged with their nnz; k_fused then treats them like long rows.
//
// Per warp: an open-addressing table of kRowsSlots slots in shared memory,
// used over a per-row power-of-two region sized for <= 3/4 load (so no
// overflow path exists). After the row: the region's nonzero (column, value)
// pairs are compacted to its front in place, bitonic-sorted there by column
// with a loop (small code: I-cache pressure was this kernel's bound), and
// written out coalesced.
struct RowsParams {
  DevCsr A, B;
  const uint32_t* prod;
  const uint32_t* dom;  // rows with a dominant entry are k_esc_dom's (null: none are)
  const uint32_t* sub;  // k_esc_warp: its rows, as indices into list
  const unsigned long long* n_sub;
  const uint32_t* list;
  const unsigned long long* n_list;
  unsigned long long* cursor;  // staging allocator
  unsigned long long* ticket;  // dynamic row counter
  uint64_t* l_off;
  uint32_t* l_nnz;
  uint32_t* l_ci;
  double* l_v;
  uint32_t* st_min;
  uint32_t* st_max;
  uint32_t* st_touch;
};

constexpr int kRowsWarps = 8;
constexpr uint32_t kRowsSlots = 1024;
constexpr uint32_t kRowsLimit = kRowsSlots * 3 / 4;  // products; longer rows: k_long_smem

__host__ __device__ constexpr size_t rows_smem_bytes() {
  return size_t(kRowsWarps) * kRowsSlots * (sizeof(double) + sizeof(uint32_t));
}

// Table over a runtime power-of-two region (mask), for medium_accumulate.
struct RegionTable {
  uint32_t* keys;
  double* vals;
  uint32_t mask;
  uint32_t shift;  // 32 - log2(region)
  template <bool STATS>
  __device__ __forceinline__ bool apply(uint32_t col, double p, uint32_t& touches) const {
    volatile uint32_t* vk = keys;
    volatile double* vv = vals;
    uint32_t h = (col * 0x9E3779B1u) >> shift;
    bool fresh = false;
    while (true) {
      const uint32_t k = vk[h];
      if (k == col) break;
      if (k == kEmptyKey) {
        const uint32_t old = atomicCAS(keys + h, kEmptyKey, col);
        if (old == kEmptyKey) { fresh = true; break; }
        if (old == col) break;
      }
      h = (h + 1) & mask;
    }
    const double cur = fresh ? 0.0 : vv[h];  // fresh slot == dense[x] == 0.0
    if (STATS && cur == 0.0) ++touches;
    vv[h] = __dadd_rn(cur, p);
    return fresh;
  }
};

template <bool STATS>
__global__ void __launch_bounds__(kRowsWarps * 32, 2) k_rows(const RowsParams p_in) {
  extern __shared__ __align__(16) unsigned char rows_sm[];
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  double* vals = reinterpret_cast<double*>(rows_sm) + warp * kRowsSlots;
  uint32_t* keys =
      reinterpret_cast<uint32_t*>(rows_sm + kRowsWarps * kRowsSlots * sizeof(double)) +
      warp * kRowsSlots;
  volatile uint32_t* vk = keys;
  volatile double* vv = vals;
  RowsParams p = p_in;
  p.B.pol = policy_evict_last();
  p.A.pol = policy_evict_first();
  for (uint32_t s = lane; s < kRowsSlots; s += 32) vk[s] = kEmptyKey;
  __syncwarp();
  const uint64_t n = *p.n_list;
#pragma unroll 1
  while (true) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(p.ticket, 1ull);
    const uint64_t li = __shfl_sync(kFull, t, 0);
    if (li >= n) break;
    const uint32_t r = p.list[li];
    const uint32_t prod = p.prod[r];
    if (prod > kRowsLimit) continue;  // k_long_smem / k_long
    uint32_t lg = 6;
    while ((1u << lg) * 3u < prod * 4u) ++lg;  // region: load <= 3/4
    const uint32_t region = 1u << lg;
    const RegionTable tab{keys, vals, region - 1, 32 - lg};
    const uint64_t lo = ld_idx(p.A.rp + r), hi = ld_idx(p.A.rp + r + 1);
    uint32_t touches = 0;
    medium_accumulate<RegionTable, STATS>(p.A, p.B, lo, hi, tab, region, touches);
    // compact nonzero pairs to the front, in place (each 32-slot window is
    // read completely before any lane writes; writes never pass the window)
    uint32_t cnt = 0, mn = kEmptyKey, mx = 0;
#pragma unroll 1
    for (uint32_t s0 = 0; s0 < region; s0 += 32) {
      const uint32_t s = s0 + lane;
      const uint32_t k = vk[s];
      const double v = vv[s];
      const bool occ = k != kEmptyKey;
      const bool keep = occ && (v != 0.0);  // kernels.py:296 drops exact zeros
      if (STATS && occ) {
        mn = k < mn ? k : mn;
        mx = k > mx ? k : mx;
      }
      const uint32_t m = __ballot_sync(kFull, keep);
      __syncwarp();
      vk[s] = kEmptyKey;
      __syncwarp();
      if (keep) {
        const uint32_t pos = cnt + __popc(m & lanemask_lt());
        vk[pos] = k;
        vv[pos] = v;
      }
      cnt += __popc(m);
    }
    __syncwarp();
    // bitonic sort of the first pow2 >= cnt pairs (the rest are empty keys)
    uint32_t np = 1;
    while (np < cnt) np <<= 1;
#pragma unroll 1
    for (uint32_t k2 = 2; k2 <= np; k2 <<= 1) {
#pragma unroll 1
      for (uint32_t j = k2 >> 1; j > 0; j >>= 1) {
        for (uint32_t t2 = lane; t2 < (np >> 1); t2 += 32) {
          const uint32_t i = 2 * t2 - (t2 & (j - 1));
          const uint32_t ka = vk[i], kb = vk[i + j];
          const bool up = (i & k2) == 0;
          if ((ka > kb) == up) {
            vk[i] = kb;
            vk[i + j] = ka;
            const double va = vv[i];
            vv[i] = vv[i + j];
            vv[i + j] = va;
          }
        }
        __syncwarp();
      }
    }
    unsigned long long off = 0;
    if (lane == 0) off = atomicAdd(p.cursor, (unsigned long long)cnt);
    off = __shfl_sync(kFull, off, 0);
    for (uint32_t t2 = lane; t2 < cnt; t2 += 32) {
      __stcs(p.l_ci + off + t2, vk[t2]);
      __stcs(p.l_v + off + t2, vv[t2]);
      vk[t2] = kEmptyKey;
    }
    __syncwarp();
    if (STATS) {
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) touches += __shfl_xor_sync(kFull, touches, d);
      mn = __reduce_min_sync(kFull, mn);
      mx = __reduce_max_sync(kFull, mx);
    }
    if (lane == 0) {
      p.l_off[li] = off;
      p.l_nnz[li] = cnt;
      if (STATS) {
        p.st_min[r] = mn;
        p.st_max[r] = mx;
        p.st_touch[r] = touches;
      }
    }
  }
}

}  // namespace spmmm
