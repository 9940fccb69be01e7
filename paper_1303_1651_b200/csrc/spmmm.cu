// Host side of libspmmm.so: contexts, device memory, the launch sequence of
// one C = A·B, and the C ABI declared in include/spmmm.h.
//
// One multiply (device-resident operands) is either
//   count-free (every row of C short by construction, aux_kernels.cuh k_prep):
//     k_prep -> k_fused (its last warp reports to the host) -> [sync]
//   or counted:
//     memset(ctrl) -> k_count -> [read-back, sync]         (size C, pick the kernel)
//     [k_collect -> ESC / long-row kernels]  only when some row is too long for k_fused
//     k_fused (cooperative, persistent) [-> k_copy_long] -> [read-back, sync]
// The reference does the same two steps host-side: estimate_nnz then one
// reservation (kernels.py:314, formats.py:199-205), then the row loop.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <atomic>
#include <functional>
#include <condition_variable>
#include <immintrin.h>
#include <mutex>
#include <thread>
#include <sched.h>
#include <unistd.h>
#include <string>
#include <vector>

#include "../../include/spmmm.h"
#include "aux_kernels.cuh"
#include "convert.cuh"
#include "dist_kernels.cuh"
#include "esc.cuh"
#include "fused_launch.cuh"

using namespace spmmm;

namespace {

// SPMMM_TRACE=1: host-side phase timestamps of spmmm_multiply on stderr
struct Trace {
  bool on;
  std::chrono::steady_clock::time_point t0;
  Trace() : on(std::getenv("SPMMM_TRACE") != nullptr), t0(std::chrono::steady_clock::now()) {}
  void mark(const char* what) const {
    if (!on) return;
    const double us =
        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "[spmmm] %10.1f us  %s\n", us, what);
  }
};

thread_local std::string g_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_error = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess) {                                                              \
      return fail(_e == cudaErrorMemoryAllocation ? SPMMM_ERR_OOM : SPMMM_ERR_CUDA,       \
                  "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__,        \
                  __LINE__);                                                              \
    }                                                                                     \
  } while (0)

// Grow-only device buffer allocated from the stream-ordered pool.
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
};

cudaError_t ensure(DevBuf& b, size_t bytes, cudaStream_t s, bool* grown = nullptr) {
  if (grown) *grown = false;
  if (bytes == 0) bytes = 16;
  if (b.cap >= bytes) return cudaSuccess;
  if (b.p) {
    cudaError_t e = cudaFreeAsync(b.p, s);
    if (e != cudaSuccess) return e;
    b.p = nullptr;
    b.cap = 0;
  }
  size_t want = std::max(bytes, size_t(256));
  cudaError_t e = cudaMallocAsync(&b.p, want, s);
  if (e != cudaSuccess) return e;
  b.cap = want;
  if (grown) *grown = true;
  return cudaSuccess;
}

void release(DevBuf& b, cudaStream_t s) {
  if (b.p) cudaFreeAsync(b.p, s);
  b.p = nullptr;
  b.cap = 0;
}

const char* const kKernelNames[] = {"k_count", "k_collect", "k_long", "k_fused", "k_copy_long",
                                    "k_rows", "k_long_smem", "k_long_cluster", "k_pack_ell",
                                    "k_esc_warp", "k_esc_block", "k_esc_plan", "k_prep",
                                    "k_esc_dom"};
constexpr int kNumKernels = 14;
#ifndef SPMMM_NO_SPLIT_VARIANT
constexpr bool kSplitVariant = true;  // split mode (no stats) runs fused_split.cu's instantiation
#else
constexpr bool kSplitVariant = false;
#endif
constexpr int kMaxPipeBlocks = 16;  // spmmm_multiply_host row blocks
constexpr uint64_t kNarrowMin = 1 << 20;  // results past this many products: u32 indices down

}  // namespace

namespace {
struct Stager;
}

struct spmmm_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int sms = 148;
  std::mutex mu;
  DevBuf ctrl, prod, lmap, list, status, l_off, l_nnz, ws, gtab;
  uint64_t gtab_warps = 0;
  DevBuf a_rp, a_ci, a_v, b_rp, b_ci, b_v;
  unsigned long long* h_ctrl = nullptr;  // pinned mirror of ctrl
  uint32_t epoch = 0;
  uint64_t status_cap_tiles = 0;
  uint64_t ws_slots = 0, ws_words = 0;
  int ws_grid = 0;
  DevBuf stage_ci, stage_v;  // staged pre-computed rows (run_long -> k_copy_long)
  bool long_smem_attr[2] = {false, false};  // k_long_smem opt-in smem set
  bool rows_attr[2] = {false, false};       // k_rows opt-in smem set
  bool esc_attr[2] = {false, false};        // k_esc_* opt-in smem set
  int long_clusters = 0;                     // resident kLongParts-block clusters
  DevBuf sub;                                // per-kernel row sub-lists
  DevBuf dom;                                // per row: its dominant entry (k_count -> k_esc_dom)
  bool no_dom = false;                       // the next counted product runs without k_esc_dom
  bool lists_from_count = false;             // k_count built the split-mode (ESC) row lists
  DevBuf ell;                                // ELL records of B (short rows)
  DevBuf tr_scratch;                         // storage-order conversion scratch
  DevBuf parts, part_off, part_nnz, row_parts, scr_col, scr_val;  // ESC parts of huge rows
  // spmmm_multiply_host: copy streams (uploads, downloads) and their events
  cudaStream_t s_up = nullptr, s_down = nullptr;
  cudaEvent_t pev[5 * kMaxPipeBlocks + 2] = {};
  DevBuf ci32, rp32;                   // narrowed column indices / row pointers of C blocks
  DevBuf d16, dbase;                   // u16 column deltas of C blocks and their chunk bases
  // split mode: k_esc_warp runs on its own stream beside k_esc_plan/k_esc_block
  cudaStream_t s_aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  DevBuf aux;                          // per-block max columns
  unsigned long long* h_aux = nullptr; // pinned mirror
  // multi-GPU: partition scratch (chunk sums), its pinned result words, and
  // the shifted row pointers of a download at an offset
  DevBuf part_sums, dl_rp;
  unsigned long long* h_part = nullptr;
  // operands the count-free path last declined (not retried for them)
  uint64_t cf_skip[5] = {0, 0, 0, 0, 0};
  // ctrl was zeroed behind the last count-free product (off the critical path)
  bool ctrl_clean = false;
  // the next counted product reserves C at the product count (an overflow redo)
  bool exact_reserve = false;
  // page-locked staging of pageable uploads (spmmm_multiply_host), lazily
  Stager* stager = nullptr;
  // freed product arrays kept for reuse: at most this many bytes
  size_t cache_limit = size_t(16) << 30;
  // freed product arrays, reused by later products (a fresh cudaMallocAsync
  // of hundreds of MB can cost tens of milliseconds of pool growth)
  std::vector<std::pair<void*, size_t>> cache;
  size_t cache_bytes = 0;
  cudaEvent_t ev[2 * kNumKernels] = {};
  cudaEvent_t ev_count = nullptr;  // k_count's results are on the host
  bool ev_used[kNumKernels] = {};
  double last_ms[kNumKernels] = {};
  int last_count = 0;
  int last_launches = 0;
};

struct spmmm_product {
  spmmm_context* ctx = nullptr;
  uint64_t rows = 0, cols = 0, nnz = 0, mults = 0;
  uint64_t* rp = nullptr;
  uint64_t* ci = nullptr;
  double* v = nullptr;
  uint32_t* st = nullptr;  // 3 * rows (min, max, touched) when row stats were requested
  size_t cap[4] = {0, 0, 0, 0};  // allocation sizes of rp, ci, v, st (context cache)
};

namespace {

// ---- product array cache ----------------------------------------------------


// Best fit among cached blocks of [bytes, 2*bytes + 1 MiB], else a new one.
cudaError_t cache_alloc(spmmm_context* c, size_t bytes, void** out, size_t* cap) {
  bytes = std::max(bytes, size_t(256));
  int best = -1;
  for (int i = 0; i < int(c->cache.size()); ++i) {
    const size_t s = c->cache[i].second;
    if (s >= bytes && s <= 2 * bytes + (size_t(1) << 20) &&
        (best < 0 || s < c->cache[best].second))
      best = i;
  }
  if (best >= 0) {
    *out = c->cache[best].first;
    *cap = c->cache[best].second;
    c->cache_bytes -= *cap;
    c->cache.erase(c->cache.begin() + best);
    return cudaSuccess;
  }
  *cap = bytes;
  return cudaMallocAsync(out, bytes, c->stream);
}

// Return a block (stream-ordered on the context stream, so a later product
// on the same stream may reuse it at once); the oldest blocks past the limit
// go back to the pool.
void cache_free(spmmm_context* c, void* ptr, size_t cap) {
  if (!ptr) return;
  c->cache.emplace_back(ptr, cap);
  c->cache_bytes += cap;
  while (c->cache_bytes > c->cache_limit && !c->cache.empty()) {
    cudaFreeAsync(c->cache.front().first, c->stream);
    c->cache_bytes -= c->cache.front().second;
    c->cache.erase(c->cache.begin());
  }
}

void product_release(spmmm_context* c, spmmm_product* p) {
  cache_free(c, p->rp, p->cap[0]);
  cache_free(c, p->ci, p->cap[1]);
  cache_free(c, p->v, p->cap[2]);
  cache_free(c, p->st, p->cap[3]);
  p->rp = nullptr;
  p->ci = nullptr;
  p->v = nullptr;
  p->st = nullptr;
}

// ---- operand views --------------------------------------------------------

int check_view(const spmmm_csr* m, const char* name) {
  if (!m) return fail(SPMMM_ERR_INVALID, "%s is NULL", name);
  if (!m->row_ptr) return fail(SPMMM_ERR_INVALID, "%s.row_ptr is NULL", name);
  if (m->nnz && (!m->col_idx || !m->values))
    return fail(SPMMM_ERR_INVALID, "%s has nnz=%llu but NULL arrays", name,
                (unsigned long long)m->nnz);
  if (m->memory != SPMMM_MEM_HOST && m->memory != SPMMM_MEM_DEVICE)
    return fail(SPMMM_ERR_INVALID, "%s.memory=%d is not host/device", name, m->memory);
  return SPMMM_OK;
}

int stage_h2d(spmmm_context* c, void* dst, const void* src, size_t bytes);

// Upload a host CSR view into context buffers; return a device view.
int upload(spmmm_context* c, const spmmm_csr* m, DevBuf& rp, DevBuf& ci, DevBuf& v, DevCsr* out) {
  const size_t rpb = (m->rows + 1) * sizeof(uint64_t);
  const size_t cib = m->nnz * sizeof(uint64_t), vb = m->nnz * sizeof(double);
  CUDA_TRY(ensure(rp, rpb, c->stream));
  CUDA_TRY(ensure(ci, cib, c->stream));
  CUDA_TRY(ensure(v, vb, c->stream));
  int rc = stage_h2d(c, rp.p, m->row_ptr, rpb);
  if (!rc && m->nnz) rc = stage_h2d(c, ci.p, m->col_idx, cib);
  if (!rc && m->nnz) rc = stage_h2d(c, v.p, m->values, vb);
  if (rc) return rc;
  out->rp = static_cast<const uint64_t*>(rp.p);
  out->ci = static_cast<const uint64_t*>(ci.p);
  out->v = static_cast<const double*>(v.p);
  out->rows = m->rows;
  out->cols = m->cols;
  out->nnz = m->nnz;
  return SPMMM_OK;
}

int resolve(spmmm_context* c, const spmmm_csr* a, const spmmm_csr* b, DevCsr* A, DevCsr* B) {
  if (a->memory == SPMMM_MEM_DEVICE) {
    *A = DevCsr{a->row_ptr, a->col_idx, a->values, a->rows, a->cols, a->nnz};
  } else {
    int rc = upload(c, a, c->a_rp, c->a_ci, c->a_v, A);
    if (rc) return rc;
  }
  if (b->memory == SPMMM_MEM_DEVICE) {
    *B = DevCsr{b->row_ptr, b->col_idx, b->values, b->rows, b->cols, b->nnz};
  } else if (a->memory == SPMMM_MEM_HOST && a->row_ptr == b->row_ptr &&
             a->col_idx == b->col_idx && a->values == b->values && a->rows == b->rows &&
             a->nnz == b->nnz) {
    *B = *A;  // C = A·A: one upload (C1, C2, C4 are squares of one matrix)
    B->cols = b->cols;
  } else {
    int rc = upload(c, b, c->b_rp, c->b_ci, c->b_v, B);
    if (rc) return rc;
  }
  return SPMMM_OK;
}

// ---- timing helpers ---------------------------------------------------------

struct Timer {
  spmmm_context* c;
  bool on;
  void begin(int k, cudaStream_t s = nullptr) {
    if (on) { cudaEventRecord(c->ev[2 * k], s ? s : c->stream); c->ev_used[k] = true; }
  }
  void end(int k, cudaStream_t s = nullptr) {
    if (on) cudaEventRecord(c->ev[2 * k + 1], s ? s : c->stream);
  }
};

// ---- small readbacks -----------------------------------------------------------
// Control words reach the host through a kernel storing into page-locked host
// memory (UVA-mapped), not cudaMemcpy: in the pipelined host path the copy
// engine is busy streaming C down, and a tiny memcpy would queue behind it.
__global__ void k_readback(const unsigned long long* __restrict__ src,
                           unsigned long long* __restrict__ host, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    volatile unsigned long long* h = host + i;
    *h = src[i];
  }
}

cudaError_t readback(const unsigned long long* dsrc, unsigned long long* hdst, int n,
                     cudaStream_t s) {
  k_readback<<<1, 64, 0, s>>>(dsrc, hdst, n);
  return cudaGetLastError();
}

// ---- the count pass ----------------------------------------------------------

// Look-back state of k_fused: the level-1.. counters first (zeroed by k_count
// for the largest layout a call can use: one row per tile), then the status
// words of every level.
uint64_t lb_counters_max(uint64_t rows) {
  uint64_t n = rows, total = 0;
  for (int l = 1; l < kLevels; ++l) {
    n = (n + 31) / 32;
    total += n;
  }
  return total;
}

// The row lists in the context's buffers (list, lmap; sub: mid, huge, overflow,
// dominated, dominated past the block-copy limit, warp rows — `rows` entries each).
RowLists row_lists(spmmm_context* c, uint64_t rows, uint32_t mid_min, uint32_t huge_min) {
  RowLists l{};
  l.list = static_cast<uint32_t*>(c->list.p);
  l.lmap = static_cast<uint32_t*>(c->lmap.p);
  l.mid_list = static_cast<uint32_t*>(c->sub.p);
  l.huge_list = l.mid_list + rows;
  l.dom_list = l.mid_list + 3 * rows;
  l.dom_big = l.mid_list + 4 * rows;
  l.warp_list = l.mid_list + 5 * rows;
  l.mid_min = mid_min;
  l.huge_min = huge_min;
  return l;
}

int run_count(spmmm_context* c, const DevCsr& A, const DevCsr& B, Timer& tm, bool pack = false) {
  CUDA_TRY(ensure(c->prod, std::max<uint64_t>(A.rows, 1) * sizeof(uint32_t), c->stream));
  CUDA_TRY(ensure(c->dom, std::max<uint64_t>(A.rows, 1) * sizeof(uint32_t), c->stream));
  // the product path: k_count also lists the non-short rows as split mode
  // with the ESC kernels wants them (RowLists, aux_kernels.cuh)
  RowLists lists{};
  c->lists_from_count = false;
  static const bool env_no_dom = std::getenv("SPMMM_NO_DOM") != nullptr;
  static const bool env_no_esc = std::getenv("SPMMM_NO_ESC") != nullptr;
  if (pack && A.rows && !env_no_dom && !env_no_esc && !c->no_dom &&
      B.cols <= (1ull << kEscColBits)) {
    CUDA_TRY(ensure(c->lmap, A.rows * sizeof(uint32_t), c->stream));
    CUDA_TRY(ensure(c->list, A.rows * sizeof(uint32_t), c->stream));
    CUDA_TRY(ensure(c->sub, 6 * A.rows * sizeof(uint32_t), c->stream));
    lists = row_lists(c, A.rows, kEscWarpLimit, kEscBlockCap);
    c->lists_from_count = true;
  }
  // status: counters + words for one row per tile (the medium layout, the largest)
  const uint64_t ncnt = pack ? lb_counters_max(A.rows) : 0;
  if (pack) {
    bool grown = false;
    uint64_t words = 0, n = A.rows;
    for (int l = 0; l < kLevels; ++l) {
      words += n;
      n = (n + 31) / 32;
    }
    CUDA_TRY(ensure(c->status, (words + ncnt) * sizeof(uint64_t), c->stream, &grown));
    if (grown || c->epoch >= 0xffffu) {
      CUDA_TRY(cudaMemsetAsync(c->status.p, 0, c->status.cap, c->stream));
      c->epoch = 0;
    }
  }
  if (pack) CUDA_TRY(ensure(c->ell, std::max<uint64_t>(B.rows, 1) * 64, c->stream));
  CUDA_TRY(cudaMemsetAsync(c->ctrl.p, 0, kCtrlWords * sizeof(unsigned long long), c->stream));
  c->ctrl_clean = false;
  // C = A·A with A's rows its own B rows: k_count writes the ELL copy itself
  const bool self_pack = pack && A.rows && A.rp == B.rp && A.ci == B.ci && A.v == B.v &&
                         A.rows == B.rows;
  // otherwise, B rows of about kEllSlots entries on average and A spanning
  // most of B: k_count also copies every B row (speculatively)
  static const bool no_spec = std::getenv("SPMMM_NO_SPEC_ELL") != nullptr;
  const bool spec_pack = pack && !self_pack && !no_spec && A.rows && B.rows &&
                         B.nnz <= uint64_t(kEllSlots) * B.rows + B.rows / 8 &&
                         2 * A.rows >= B.rows;
  if (A.rows) {
    const uint64_t blocks = std::min<uint64_t>((A.rows + 255) / 256, uint64_t(c->sms) * 8);
    tm.begin(0);
    k_count<<<unsigned(blocks), 256, 0, c->stream>>>(
        A, B, static_cast<uint32_t*>(c->prod.p), static_cast<unsigned long long*>(c->ctrl.p),
        static_cast<unsigned long long*>(c->status.p), ncnt,
        self_pack ? static_cast<uint4*>(c->ell.p) : nullptr,
        spec_pack ? static_cast<uint4*>(c->ell.p) : nullptr, static_cast<uint32_t*>(c->dom.p),
        lists);
    CUDA_TRY(cudaGetLastError());
    tm.end(0);
    ++c->last_launches;
  }
  ++c->last_launches;  // (k_readback)
  CUDA_TRY(readback(static_cast<const unsigned long long*>(c->ctrl.p), c->h_ctrl, kCtrlWords,
                    c->stream));
  CUDA_TRY(cudaEventRecord(c->ev_count, c->stream));
  if (pack && A.rows && !self_pack && !spec_pack) {
    // the ELL copy of B (if k_count's results call for it) overlaps the readback
    tm.begin(8);
    k_pack_ell<<<unsigned(c->sms) * 16, 256, 0, c->stream>>>(
        B, A.rows, static_cast<const unsigned long long*>(c->ctrl.p), static_cast<uint4*>(c->ell.p));
    CUDA_TRY(cudaGetLastError());
    tm.end(8);
    ++c->last_launches;
  }
  CUDA_TRY(cudaEventSynchronize(c->ev_count));
  const unsigned long long err = c->h_ctrl[kCtrlError];
  if (err & 1) return fail(SPMMM_ERR_INVALID, "malformed a.row_ptr (decreasing or past nnz)");
  if (err & 2) return fail(SPMMM_ERR_INVALID, "a.col_idx entry >= b.rows");
  if (err & 4) return fail(SPMMM_ERR_INVALID, "malformed b.row_ptr (decreasing or past nnz)");
  if (err & 8) return fail(SPMMM_ERR_UNSUPPORTED, "a row of C needs more than 2^31 products");
  return SPMMM_OK;
}

// ---- fused-kernel launch: instantiations live in fused_short.cu / fused_medium.cu ----

int fused_call(spmmm_context* c, bool medium, int op, const FusedParams& prm, bool wide,
               bool stats, unsigned grid, int* occ, bool count_free = false, int prep = 0,
               bool split = false) {
  FusedLaunchEnv env{c->device, c->sms, c->stream};
  cudaError_t e = count_free ? fused_cf(op, prm, env, wide, stats, grid, occ, prep, prm.self_ell != 0)
                  : medium   ? fused_medium(op, prm, env, wide, stats, grid, occ)
                  : split    ? fused_split(op, prm, env, wide, stats, grid, occ)
                             : fused_short(op, prm, env, wide, stats, grid, occ);
  if (e != cudaSuccess)
    return fail(e == cudaErrorMemoryAllocation ? SPMMM_ERR_OOM : SPMMM_ERR_CUDA,
                "k_fused<%s> %s: %s", medium ? "medium" : "short", op ? "launch" : "occupancy",
                cudaGetErrorString(e));
  return SPMMM_OK;
}

// ---- per-warp global overflow tables and sort/staging scratch ------------------

struct GtabView {
  uint32_t* keys;
  double* vals;
  uint32_t* scol;
  double* sval;
};

int ensure_gtab(spmmm_context* c, uint64_t warps, GtabView* v) {
  const size_t per_warp = kGlobalSlots * (sizeof(uint32_t) + sizeof(double)) +
                          kMaxBufs * kMediumLimit * (sizeof(uint32_t) + sizeof(double));
  bool grown = false;
  CUDA_TRY(ensure(c->gtab, warps * per_warp, c->stream, &grown));
  if (grown || c->gtab_warps < warps) {
    CUDA_TRY(cudaMemsetAsync(c->gtab.p, 0xff, c->gtab.cap, c->stream));  // keys empty
    c->gtab_warps = c->gtab.cap / per_warp;
  }
  char* g = static_cast<char*>(c->gtab.p);
  const uint64_t n = c->gtab_warps;
  v->vals = reinterpret_cast<double*>(g);
  v->sval = reinterpret_cast<double*>(g + n * kGlobalSlots * 8);
  v->keys = reinterpret_cast<uint32_t*>(g + n * (kGlobalSlots + kMaxBufs * kMediumLimit) * 8);
  v->scol = v->keys + n * kGlobalSlots;
  return SPMMM_OK;
}

// ---- the long-row path ------------------------------------------------------

#ifndef SPMMM_LONG_PARTS
#define SPMMM_LONG_PARTS 4
#endif
constexpr int kLongParts = SPMMM_LONG_PARTS;  // blocks per cluster for rows past kLongSmemProducts

// k_long_smem, one block per row or (cluster) kLongParts blocks per row
template <bool S>
int launch_long_smem(spmmm_context* c, const LongParams& lp, bool cluster) {
  const size_t smem = long_smem_bytes();
  auto* k1 = k_long_smem<S, 1>;
  auto* k8 = k_long_smem<S, kLongParts>;
  if (!c->long_smem_attr[S]) {  // once per context (device)
    CUDA_TRY(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    CUDA_TRY(cudaFuncSetAttribute(k8, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    c->long_smem_attr[S] = true;
  }
  if (!cluster) {
    k1<<<c->sms, kLongThreads, smem, c->stream>>>(lp);
    CUDA_TRY(cudaGetLastError());
    return SPMMM_OK;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kLongParts;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kLongThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (c->long_clusters <= 0) {
    cfg.gridDim = dim3(kLongParts * 64);
    int n = 0;
    CUDA_TRY(cudaOccupancyMaxActiveClusters(&n, k8, &cfg));
    if (n <= 0) return fail(SPMMM_ERR_UNSUPPORTED, "no %d-block cluster fits a GPC", kLongParts);
    c->long_clusters = n;
  }
  cfg.gridDim = dim3(unsigned(kLongParts * c->long_clusters));
  CUDA_TRY(cudaLaunchKernelEx(&cfg, k8, lp));
  return SPMMM_OK;
}

// Rows computed before k_fused: the long rows (> kMediumLimit products, k_long)
// and, in split mode, every other non-short row (k_rows). They are listed by
// k_collect (rows of class long for `list_limit`), staged with their nnz, and
// copied into place by k_copy_long after k_fused.
int run_long(spmmm_context* c, const DevCsr& A, const DevCsr& B, uint64_t max_prod,
             uint32_t list_limit, bool split, bool esc, uint64_t total, bool stats,
             spmmm_product* p,
             DevBuf& stage_ci, DevBuf& stage_v, Timer& tm) {
  const Trace tr;
  const uint64_t rows = A.rows;
  bool esc_forked = false;
  auto join_esc = [&]() -> int {
    if (esc_forked) {
      esc_forked = false;
      if (cudaStreamWaitEvent(c->stream, c->ev_join, 0) != cudaSuccess)
        return fail(SPMMM_ERR_CUDA, "joining the k_esc_warp stream failed");
    }
    return SPMMM_OK;
  };
  CUDA_TRY(ensure(c->lmap, rows * sizeof(uint32_t), c->stream));
  CUDA_TRY(ensure(c->list, rows * sizeof(uint32_t), c->stream));
  CUDA_TRY(ensure(c->l_off, rows * sizeof(uint64_t), c->stream));
  CUDA_TRY(ensure(c->l_nnz, rows * sizeof(uint32_t), c->stream));
  CUDA_TRY(ensure(c->sub, 6 * rows * sizeof(uint32_t), c->stream));
  uint32_t* mid_list = static_cast<uint32_t*>(c->sub.p);
  uint32_t* huge_list = mid_list + rows;
  uint32_t* ovf_list = mid_list + 2 * rows;
  uint32_t* dom_list = mid_list + 3 * rows;  // (+ 4 * rows: those past the block-copy limit)
  // ESC mode: rows dominated by one long B row go to k_esc_dom (SPMMM_NO_DOM=1,
  // or a B row found unsorted by it: all of them through the other kernels)
  static const bool env_no_dom = std::getenv("SPMMM_NO_DOM") != nullptr;
  const uint32_t* dom = (esc && !env_no_dom && !c->no_dom) ? static_cast<const uint32_t*>(c->dom.p)
                                                         : nullptr;
  // split mode: k_rows (k_esc_warp) takes rows up to kRowsLimit
  // (kEscWarpLimit); else k_fused up to kMediumLimit
  const uint32_t long_min = esc ? kEscWarpLimit : split ? kRowsLimit : kMediumLimit;
  // rows past huge_min: the cluster variant (and k_long for its overflow)
  const uint32_t huge_min = esc ? kEscBlockCap : kLongSmemProducts;
  tr.mark("  run_long: lists");
  CUDA_TRY(ensure(stage_ci, total * sizeof(uint32_t), c->stream));
  CUDA_TRY(ensure(stage_v, total * sizeof(double), c->stream));
  tr.mark("  run_long: buffers");
  const bool any_huge = max_prod > huge_min;  // some row needs the cluster / k_long
  // workspace: one table (>= 2x the distinct columns a row can have) and one
  // column bitmap per resident block
  uint64_t distinct = std::min<uint64_t>(max_prod, std::max<uint64_t>(B.cols, 1));
  uint64_t slots = 64;
  while (slots < 2 * distinct) slots <<= 1;
  uint64_t words = std::max<uint64_t>((B.cols + 31) / 32, 1);
  // grow-only: a bigger table or bitmap than this product needs works as well
  // (k_long restores both after every row), and the row blocks of one
  // pipelined product differ in their longest row
  const bool grow = any_huge && (!c->ws.p || slots > c->ws_slots || words > c->ws_words);
  slots = std::max<uint64_t>(slots, c->ws_slots);
  words = std::max<uint64_t>(words, c->ws_words);
  const uint64_t swords = (words + 31) / 32;
  const uint64_t per_block = slots * (4 + 8 + 4) + (words + swords) * 4;
  int grid = 2 * c->sms;
  const uint64_t budget = 8ull << 30;  // cap the workspace at 8 GiB
  while (grid > 1 && uint64_t(grid) * per_block > budget) grid /= 2;
  if (grow) {
    release(c->ws, c->stream);
    CUDA_TRY(ensure(c->ws, size_t(grid) * per_block, c->stream));
    char* base = static_cast<char*>(c->ws.p);
    const size_t n = size_t(grid) * slots;
    CUDA_TRY(cudaMemsetAsync(base, 0xff, n * 4, c->stream));                   // keys
    CUDA_TRY(cudaMemsetAsync(base + n * 4, 0, n * 8, c->stream));             // vals
    CUDA_TRY(cudaMemsetAsync(base + n * 12, 0xff, n * 4, c->stream));         // owner
    CUDA_TRY(cudaMemsetAsync(base + n * 16, 0, size_t(grid) * (words + swords) * 4,
                             c->stream));  // bitmaps + summaries
    c->ws_slots = slots;
    c->ws_words = words;
    c->ws_grid = grid;
  }
  tr.mark("  run_long: workspace");
  if (!(c->lists_from_count && esc && dom)) {
    // k_count's lists (if any) assumed split mode with every ESC kernel:
    // list the rows by this mode's limits instead
    unsigned long long* ctrl = static_cast<unsigned long long*>(c->ctrl.p);
    if (c->lists_from_count) {
      CUDA_TRY(cudaMemsetAsync(ctrl + kCtrlLongRows, 0, 8, c->stream));
      CUDA_TRY(cudaMemsetAsync(ctrl + kCtrlMidRows, 0, 16, c->stream));  // (and kCtrlHugeRows)
      CUDA_TRY(cudaMemsetAsync(ctrl + kCtrlDomBigRows, 0, 8, c->stream));
      CUDA_TRY(cudaMemsetAsync(ctrl + kCtrlDomRows, 0, 16, c->stream));  // (and kCtrlWarpRows)
    }
    const uint64_t blocks = std::min<uint64_t>((rows + 255) / 256, uint64_t(c->sms) * 8);
    tm.begin(1);
    k_collect<<<unsigned(blocks), 256, 0, c->stream>>>(
        A, static_cast<const uint32_t*>(c->prod.p), list_limit, ctrl, dom,
        row_lists(c, rows, long_min, huge_min));
    CUDA_TRY(cudaGetLastError());
    tm.end(1);
    ++c->last_launches;
  }
  if (split) {
    RowsParams rp;
    rp.A = A;
    rp.B = B;
    rp.prod = static_cast<const uint32_t*>(c->prod.p);
    rp.dom = dom;
    rp.sub = mid_list + 5 * rows;  // (RowLists.warp_list)
    rp.n_sub = static_cast<const unsigned long long*>(c->ctrl.p) + kCtrlWarpRows;
    rp.list = static_cast<const uint32_t*>(c->list.p);
    rp.n_list = static_cast<const unsigned long long*>(c->ctrl.p) + kCtrlLongRows;
    rp.cursor = static_cast<unsigned long long*>(c->ctrl.p) + kCtrlStageCursor;
    rp.ticket = static_cast<unsigned long long*>(c->ctrl.p) + kCtrlRowsTicket;
    rp.l_off = static_cast<uint64_t*>(c->l_off.p);
    rp.l_nnz = static_cast<uint32_t*>(c->l_nnz.p);
    rp.l_ci = static_cast<uint32_t*>(stage_ci.p);
    rp.l_v = static_cast<double*>(stage_v.p);
    rp.st_min = p->st;
    rp.st_max = p->st ? p->st + rows : nullptr;
    rp.st_touch = p->st ? p->st + 2 * rows : nullptr;
    if (esc) {
      const size_t smem = esc_warp_smem_bytes();
      if (!c->esc_attr[stats]) {  // once per context (device)
        auto set = [&](const void* f, size_t bytes) {
          return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
        };
        CUDA_TRY(set(reinterpret_cast<const void*>(stats ? k_esc_warp<true> : k_esc_warp<false>),
                     smem));
        CUDA_TRY(set(reinterpret_cast<const void*>(stats ? k_esc_block<true> : k_esc_block<false>),
                     esc_block_smem_bytes(kEscBlockCap)));
        c->esc_attr[stats] = true;
      }
      if (dom) {
        // the dominated rows first, with the whole GPU: a latency-bound stream of
        // B rows to the staged result (behind the other ESC kernels' resident
        // blocks it got one block per SM and took 1.3 ms instead of 0.3)
        LongParams dp{};
        dp.A = A;
        dp.B = B;
        dp.prod = rp.prod;
        dp.list = rp.list;
        dp.ctrl = static_cast<unsigned long long*>(c->ctrl.p);
        dp.l_off = rp.l_off;
        dp.l_nnz = rp.l_nnz;
        dp.l_ci = rp.l_ci;
        dp.l_v = rp.l_v;
        dp.sub = dom_list;
        dp.n_sub = dp.ctrl + kCtrlDomRows;
        dp.ticket = dp.ctrl + kCtrlHugeTicket;  // (the cluster variant's: unused in ESC mode)
        dp.dom = dom;
        dp.first = mid_list + 4 * rows;  // (RowLists.dom_big: the rows past the warp-row limit)
        dp.n_first = dp.ctrl + kCtrlDomBigRows;
        dp.first_min = long_min;
        dp.st_min = rp.st_min;
        dp.st_max = rp.st_max;
        dp.st_touch = rp.st_touch;
        tm.begin(13);
        if (stats) k_esc_dom<true><<<unsigned(c->sms) * kDomBlocks, kDomWarps * 32, esc_dom_smem_bytes(), c->stream>>>(dp);
        else k_esc_dom<false><<<unsigned(c->sms) * kDomBlocks, kDomWarps * 32, esc_dom_smem_bytes(), c->stream>>>(dp);
        CUDA_TRY(cudaGetLastError());
        tm.end(13);
        ++c->last_launches;
      }
      // the warp rows are independent of the block rows: their kernel runs on
      // a second stream, overlapping k_esc_plan / k_esc_block (all three are
      // latency bound); the context stream joins it before k_fused
      static const bool serial = std::getenv("SPMMM_SERIAL_ESC") != nullptr;
      cudaStream_t ws = c->stream;
      if (!serial) {
        if (!c->s_aux) {
          CUDA_TRY(cudaStreamCreateWithFlags(&c->s_aux, cudaStreamNonBlocking));
          CUDA_TRY(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
          CUDA_TRY(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
        }
        CUDA_TRY(cudaEventRecord(c->ev_fork, c->stream));
        CUDA_TRY(cudaStreamWaitEvent(c->s_aux, c->ev_fork, 0));
        ws = c->s_aux;
        esc_forked = true;
      }
      const unsigned grid_rows = unsigned(c->sms) * 4;  // (2 beside the block kernel measured slower)
      tm.begin(9, ws);
      if (stats) k_esc_warp<true><<<grid_rows, kEscWarps * 32, smem, ws>>>(rp);
      else k_esc_warp<false><<<grid_rows, kEscWarps * 32, smem, ws>>>(rp);
      CUDA_TRY(cudaGetLastError());
      tm.end(9, ws);
      ++c->last_launches;
      if (esc_forked) CUDA_TRY(cudaEventRecord(c->ev_join, c->s_aux));
      tr.mark("  run_long: k_esc_warp launched");
    } else {
    const size_t smem = rows_smem_bytes();
    if (!c->rows_attr[stats]) {  // once per context (device)
      if (stats)
        CUDA_TRY(cudaFuncSetAttribute(k_rows<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(smem)));
      else
        CUDA_TRY(cudaFuncSetAttribute(k_rows<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(smem)));
      c->rows_attr[stats] = true;
    }
    const unsigned grid_rows = unsigned(c->sms) * 2;
    tm.begin(5);
    if (stats) k_rows<true><<<grid_rows, kRowsWarps * 32, smem, c->stream>>>(rp);
    else k_rows<false><<<grid_rows, kRowsWarps * 32, smem, c->stream>>>(rp);
    CUDA_TRY(cudaGetLastError());
    tm.end(5);
    ++c->last_launches;
    tr.mark("  run_long: k_rows launched");
    }
  }
  if (max_prod <= long_min) return join_esc();
  LongParams lp;
  lp.A = A;
  lp.B = B;
  lp.prod = static_cast<const uint32_t*>(c->prod.p);
  lp.list = static_cast<const uint32_t*>(c->list.p);
  lp.ctrl = static_cast<unsigned long long*>(c->ctrl.p);
  lp.l_off = static_cast<uint64_t*>(c->l_off.p);
  lp.l_nnz = static_cast<uint32_t*>(c->l_nnz.p);
  lp.l_ci = static_cast<uint32_t*>(stage_ci.p);
  lp.l_v = static_cast<double*>(stage_v.p);
  char* base = static_cast<char*>(c->ws.p);
  const size_t n = size_t(c->ws_grid) * c->ws_slots;
  lp.ws_keys = reinterpret_cast<uint32_t*>(base);
  lp.ws_vals = reinterpret_cast<double*>(base + n * 4);
  lp.ws_owner = reinterpret_cast<uint32_t*>(base + n * 12);
  lp.ws_bits = reinterpret_cast<uint32_t*>(base + n * 16);
  lp.ws_slots = c->ws_slots;
  lp.ws_words = c->ws_words;
  lp.ws_swords = (c->ws_words + 31) / 32;
  lp.st_min = p->st;
  lp.st_max = p->st ? p->st + rows : nullptr;
  lp.st_touch = p->st ? p->st + 2 * rows : nullptr;
  unsigned long long* ctrl = static_cast<unsigned long long*>(c->ctrl.p);
  lp.ovf = ovf_list;
  lp.dom = nullptr;
  lp.parts = nullptr;
  lp.part_off = nullptr;
  lp.part_nnz = nullptr;
  lp.row_pbase = nullptr;
  lp.row_np = nullptr;
  lp.huge = huge_list;
  lp.scr_col = nullptr;
  lp.scr_val = nullptr;
  lp.scr_cap = 0;
  lp.max_parts = 0;
  if (esc && any_huge) {
    // parts: sum over huge rows of ceil(P / kPartTarget) <= 1.5 * huge / kPartTarget;
    // scratch slots <= 1.25 * huge + 64 per part (k_esc_plan's regions)
    const uint64_t huge = c->h_ctrl[kCtrlHugeProducts];
    const uint64_t max_parts = huge / (kPartTarget / 2) + 16;
    const uint64_t max_rows = huge / kHugeMin + 16;
    const uint64_t slots = huge + huge / 2 + 4096;
    CUDA_TRY(ensure(c->parts, max_parts * sizeof(PartDesc), c->stream));
    CUDA_TRY(ensure(c->part_off, max_parts * sizeof(uint64_t), c->stream));
    CUDA_TRY(ensure(c->part_nnz, max_parts * sizeof(uint32_t), c->stream));
    CUDA_TRY(ensure(c->row_parts, 2 * max_rows * sizeof(uint32_t), c->stream));
    CUDA_TRY(ensure(c->scr_col, slots * sizeof(uint32_t), c->stream));
    CUDA_TRY(ensure(c->scr_val, slots * sizeof(double), c->stream));
    lp.parts = static_cast<PartDesc*>(c->parts.p);
    lp.part_off = static_cast<uint64_t*>(c->part_off.p);
    lp.part_nnz = static_cast<uint32_t*>(c->part_nnz.p);
    lp.row_pbase = static_cast<uint32_t*>(c->row_parts.p);
    lp.row_np = lp.row_pbase + max_rows;
    lp.scr_col = static_cast<uint32_t*>(c->scr_col.p);
    lp.scr_val = static_cast<double*>(c->scr_val.p);
    lp.scr_cap = slots;
    lp.max_parts = max_parts;
  }
  // rows of (long_min, kLongSmemProducts] products: a block and on-chip tables
  lp.sub = mid_list;
  lp.n_sub = ctrl + kCtrlMidRows;
  lp.ticket = ctrl + kCtrlLongSmemTicket;
  int rc = SPMMM_OK;
  if (esc) {
    if (any_huge) {
      tm.begin(11);
      if (stats) k_esc_plan<true><<<c->sms * 2, kPlanThreads, 0, c->stream>>>(lp);
      else k_esc_plan<false><<<c->sms * 2, kPlanThreads, 0, c->stream>>>(lp);
      CUDA_TRY(cudaGetLastError());
      tm.end(11);
      ++c->last_launches;
    }
    const size_t smem = esc_block_smem_bytes(kEscBlockCap);
    tm.begin(10);
    if (stats) k_esc_block<true><<<c->sms * 2, kEscThreads, smem, c->stream>>>(lp, kEscBlockCap);
    else k_esc_block<false><<<c->sms * 2, kEscThreads, smem, c->stream>>>(lp, kEscBlockCap);
    CUDA_TRY(cudaGetLastError());
    tm.end(10);
  } else {
    tm.begin(6);
    rc = stats ? launch_long_smem<true>(c, lp, false) : launch_long_smem<false>(c, lp, false);
    if (rc) {
      join_esc();
      return rc;
    }
    tm.end(6);
  }
  ++c->last_launches;
  if (any_huge) {
    if (!esc) {
    // longer rows: a cluster of blocks per row, one column range each
    lp.sub = huge_list;
    lp.n_sub = ctrl + kCtrlHugeRows;
    lp.ticket = ctrl + kCtrlHugeTicket;
    tm.begin(7);
    rc = stats ? launch_long_smem<true>(c, lp, true) : launch_long_smem<false>(c, lp, true);
    if (rc) {
      join_esc();
      return rc;
    }
    tm.end(7);
    ++c->last_launches;
    }
    // rows whose column ranges outgrew the on-chip tables: global tables
    lp.sub = ovf_list;
    lp.n_sub = ctrl + kCtrlOvfRows;
    lp.ticket = ctrl + kCtrlLongTicket;
    tm.begin(2);
    if (stats) k_long<true><<<c->ws_grid, kLongThreads, 0, c->stream>>>(lp);
    else k_long<false><<<c->ws_grid, kLongThreads, 0, c->stream>>>(lp);
    CUDA_TRY(cudaGetLastError());
    tm.end(2);
    ++c->last_launches;
  }
  return join_esc();
}

// ---- the count-free path (k_prep -> k_fused, one host round trip) ----------
//
// aux_kernels.cuh (k_prep) and rows.cuh (cf_applies) say when it applies:
// every row of C is short by construction, so k_fused runs without k_count's
// per-row products and without the host reading k_count's results first. C
// is reserved at the bound that construction gives (30 or 32 entries per A
// row, 5 per A entry) instead of the exact product count. When the verdict
// is no (or the input is malformed) nothing was written and the counted path
// runs; those operands are then not tried again.

constexpr int kCfFallback = -1;
// count-free products up to this many rows (of A and B) run the prep pass
// inside k_fused (SPMMM_PREP_FUSED_ROWS overrides)
// (C1 40.5 -> 38.4 us; at 65K rows the separate, wider k_prep is faster)
constexpr uint64_t kPrepFusedRows = 1u << 14;
// internal multiply_impl flag: take the counted path (the pipelined host path's
// blocks: measured faster there)
constexpr uint32_t kFlagCounted = 1u << 30;

uint64_t lookback_words(uint64_t rows) {
  uint64_t words = 0, n = rows;
  for (int l = 0; l < kLevels; ++l) {
    words += n;
    n = (n + 31) / 32;
  }
  return words;
}

// Look-back status words + counters for `rows` one-row tiles (the largest
// layout); the counters are zeroed by k_count / k_prep.
cudaError_t ensure_lookback(spmmm_context* c, uint64_t rows) {
  bool grown = false;
  cudaError_t e = ensure(c->status, (lookback_words(rows) + lb_counters_max(rows)) * 8, c->stream,
                         &grown);
  if (e != cudaSuccess) return e;
  if (grown || c->epoch >= 0xffffu) {
    e = cudaMemsetAsync(c->status.p, 0, c->status.cap, c->stream);
    c->epoch = 0;
  }
  return e;
}

void fill_lookback(spmmm_context* c, uint64_t rows, uint64_t ntiles, FusedParams& fp) {
  uint64_t nl[kLevels];
  nl[0] = ntiles;
  for (int l = 1; l < kLevels; ++l) nl[l] = (nl[l - 1] + 31) / 32;
  c->epoch += 1;
  unsigned long long* cnt = static_cast<unsigned long long*>(c->status.p);
  uint64_t* w = reinterpret_cast<uint64_t*>(cnt + lb_counters_max(rows));
  fp.lb.count[0] = nullptr;
  for (int l = 0; l < kLevels; ++l) {
    fp.lb.stat[l] = w;
    fp.lb.n[l] = nl[l];
    w += nl[l];
    if (l > 0) {
      fp.lb.count[l] = cnt;
      cnt += nl[l];
    }
  }
  fp.lb.epoch = c->epoch;
  fp.lb.fault = static_cast<unsigned long long*>(c->ctrl.p) + kCtrlFault;
}

// Operands the path declined are not retried: keyed by where the caller's
// arrays are (host addresses for host operands — the upload buffers are
// reused by every call — device addresses otherwise) and the shapes.
void cf_key(const spmmm_csr* a, const spmmm_csr* b, uint64_t (&key)[5]) {
  key[0] = reinterpret_cast<uint64_t>(a->row_ptr);
  key[1] = reinterpret_cast<uint64_t>(a->col_idx);
  key[2] = reinterpret_cast<uint64_t>(b->row_ptr);
  key[3] = a->rows;
  key[4] = b->rows;
}

bool cf_candidate(spmmm_context* c, const DevCsr& A, const DevCsr& B, const uint64_t (&key)[5]) {
  static const bool off = std::getenv("SPMMM_NO_COUNT_FREE") != nullptr;
  if (off || A.rows == 0 || B.rows == 0) return false;
  if (B.nnz > 32 * B.rows + B.rows) return false;  // the longest B row is then > 32
  return std::memcmp(key, c->cf_skip, sizeof key) != 0;
}

int multiply_count_free(spmmm_context* c, const DevCsr& A, const DevCsr& B, bool stats, bool wide,
                        const uint64_t (&key)[5], Timer& tm, spmmm_product** out) {
  const uint64_t rows = A.rows;
  // B's rows may fit ELL records (on average they do); whether they all do,
  // and whether A references enough of them to pay for the packing, is
  // decided on the device (k_prep / k_prep_b)
  const bool same = A.rp == B.rp && A.ci == B.ci && A.rows == B.rows && A.nnz == B.nnz;
  const bool use_ell = B.nnz <= uint64_t(kEllSlots) * B.rows + B.rows / 8;
  CUDA_TRY(ensure_lookback(c, rows));
  if (use_ell) CUDA_TRY(ensure(c->ell, B.rows * 64, c->stream));
  if (!c->ctrl_clean)
    CUDA_TRY(cudaMemsetAsync(c->ctrl.p, 0, kCtrlWords * sizeof(unsigned long long), c->stream));
  c->ctrl_clean = false;
  auto* ctrl = static_cast<unsigned long long*>(c->ctrl.p);
  const uint64_t ncnt = lb_counters_max(rows);
  uint4* ell = use_ell ? static_cast<uint4*>(c->ell.p) : nullptr;
  // A spanning most of B: one pass packs all of B; a row block of A: its
  // column range first, then only the B rows in it (k_prep_b)
  const bool block = !same && 2 * rows < B.rows;
  const unsigned pgrid = unsigned(std::min<uint64_t>((std::max(rows, B.rows) + 255) / 256,
                                                     uint64_t(c->sms) * 8));
  unsigned long long* zero = static_cast<unsigned long long*>(c->status.p);
  // small products: the prep pass inside k_fused (one launch, a grid barrier)
  static const uint64_t prep_rows = std::getenv("SPMMM_PREP_FUSED_ROWS")
                                        ? std::strtoull(std::getenv("SPMMM_PREP_FUSED_ROWS"), nullptr, 10)
                                        : kPrepFusedRows;
  const int prep = (!block && std::max(rows, B.rows) <= prep_rows) ? (same ? 1 : 2) : 0;
  if (!prep) tm.begin(12);
  if (prep) {
    // (launched with k_fused below)
  } else if (same) {
    k_prep<0><<<pgrid, 256, 0, c->stream>>>(A, B, ctrl, zero, ncnt, ell);
  } else if (!block) {
    k_prep<1><<<pgrid, 256, 0, c->stream>>>(A, B, ctrl, zero, ncnt, ell);
  } else {
    k_prep<2><<<pgrid, 256, 0, c->stream>>>(A, B, ctrl, zero, ncnt, nullptr);
  }
  if (!prep) {
    CUDA_TRY(cudaGetLastError());
    ++c->last_launches;
  }
  if (block) {  // the B rows A references
    k_prep_b<<<pgrid, 256, 0, c->stream>>>(A, B, ctrl, ell);
    CUDA_TRY(cudaGetLastError());
    ++c->last_launches;
  }
  if (!prep) tm.end(12);

  auto* p = new (std::nothrow) spmmm_product;
  if (!p) return fail(SPMMM_ERR_OOM, "host allocation failed");
  p->ctx = c;
  p->rows = rows;
  p->cols = B.cols;
  auto cleanup = [&](int code) {
    product_release(c, p);
    delete p;
    return code;
  };
  // the reservation: <= 32 products per row; with B rows of <= 5 entries,
  // <= 5 per A entry. k_fused writes nothing past it (kCfOverflow: redone).
  const uint64_t cap = use_ell ? std::min<uint64_t>(uint64_t(kEllSlots) * A.nnz, 32 * rows)
                               : 32 * rows;
  cudaError_t e = cache_alloc(c, (rows + 1) * 8, reinterpret_cast<void**>(&p->rp), &p->cap[0]);
  if (e == cudaSuccess)
    e = cache_alloc(c, std::max<uint64_t>(cap, 1) * 8, reinterpret_cast<void**>(&p->ci), &p->cap[1]);
  if (e == cudaSuccess)
    e = cache_alloc(c, std::max<uint64_t>(cap, 1) * 8, reinterpret_cast<void**>(&p->v), &p->cap[2]);
  if (e == cudaSuccess && stats)
    e = cache_alloc(c, rows * 3 * sizeof(uint32_t), reinterpret_cast<void**>(&p->st), &p->cap[3]);
  if (e != cudaSuccess)
    return cleanup(fail(e == cudaErrorMemoryAllocation ? SPMMM_ERR_OOM : SPMMM_ERR_CUDA,
                        "allocating C (%llu entries): %s", (unsigned long long)cap,
                        cudaGetErrorString(e)));
  const uint64_t ntiles = (rows + kShortRowsPerTile - 1) / kShortRowsPerTile;
  FusedParams fp{};
  fill_lookback(c, rows, ntiles, fp);
  fp.ticket = ctrl + kCtrlTicket;
  fp.nnz_out = ctrl + kCtrlNnz;
  fp.A = A;
  fp.B = B;
  fp.prod = nullptr;
  fp.lmap = nullptr;
  fp.l_nnz = nullptr;
  fp.c_rp = p->rp;
  fp.c_ci = p->ci;
  fp.c_v = p->v;
  fp.ntiles = ntiles;
  fp.medium_limit = 0;
  fp.a_is_b = (A.ci == B.ci && A.v == B.v) ? 1u : 0u;
  fp.self_ell = (same && A.v == B.v && use_ell) ? 1u : 0u;
  fp.ell = reinterpret_cast<const uint32_t*>(ell);
  fp.st_min = p->st;
  fp.st_max = p->st ? p->st + rows : nullptr;
  fp.st_touch = p->st ? p->st + 2 * rows : nullptr;
  fp.cf_flags = ctrl + kCtrlCfFlags;
  fp.cf_ell_flag = ctrl + kCtrlCfEll;
  fp.cf_total = ctrl + kCtrlTotal;
  fp.cf_err = ctrl + kCtrlCfFlags;  // (kCfOverflow)
  fp.c_cap = cap;
  fp.ctrl = ctrl;
  fp.host_ctrl = c->h_ctrl;
  fp.done = ctrl + kCtrlDone;
  fp.ctrl_words = kCtrlCfWords;
  fp.cf_words = CfWords{ctrl + kCtrlCfFlags, ctrl + kCtrlKMinInv, ctrl + kCtrlKMax1, ctrl + kCtrlCfEll};
  fp.cf_zero = zero;
  fp.cf_nzero = ncnt;
  fp.cf_pack = ell;
  int occ = 0;
  int rc = fused_call(c, false, 0, fp, wide, stats, 0, &occ, true, prep);
  if (rc) return cleanup(rc);
  const unsigned grid = unsigned(std::min<uint64_t>((ntiles + kFusedWarps - 1) / kFusedWarps,
                                                    uint64_t(occ) * uint64_t(c->sms)));
  tm.begin(3);
  rc = fused_call(c, false, 1, fp, wide, stats, grid, nullptr, true, prep);
  if (rc) return cleanup(rc);
  tm.end(3);
  ++c->last_launches;
  // k_fused's last warp has copied every ctrl word (verdict, multiplications,
  // nnz, watchdog) to h_ctrl: the one host round trip
  e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cleanup(fail(SPMMM_ERR_CUDA, "multiply: %s", cudaGetErrorString(e)));
  // the last warp also zeroed ctrl for the next product (no memset before it)
  c->ctrl_clean = true;
  const unsigned long long* h = c->h_ctrl;
  if (!cf_applies(h[kCtrlCfFlags], h[kCtrlCfFlags + 1], h[kCtrlCfFlags + 2]) ||
      (h[kCtrlCfFlags] & kCfOverflow)) {
    std::memcpy(c->cf_skip, key, sizeof(c->cf_skip));
    cleanup(0);
    return kCfFallback;
  }
  if (h[kCtrlFault]) {
    const unsigned long long f = h[kCtrlFault];
    return cleanup(fail(SPMMM_ERR_CUDA, "k_fused look-back watchdog: site %llu tile %llu",
                        (f >> 48) & 0x7fff, f & ((1ull << 48) - 1)));
  }
  p->nnz = h[kCtrlNnz];
  p->mults = h[kCtrlTotal];
  *out = p;
  return SPMMM_OK;
}

int multiply_impl(spmmm_context* c, const spmmm_csr* a, const spmmm_csr* b, int strategy,
                  uint32_t flags, spmmm_product** out) {
  if (!out) return fail(SPMMM_ERR_INVALID, "out is NULL");
  *out = nullptr;
  if (strategy < SPMMM_STRATEGY_BFDOUBLE || strategy > SPMMM_STRATEGY_COMBINED)
    return fail(SPMMM_ERR_INVALID, "unknown strategy %d", strategy);
  int rc = check_view(a, "a");
  if (rc) return rc;
  rc = check_view(b, "b");
  if (rc) return rc;
  if (a->cols != b->rows)
    return fail(SPMMM_ERR_DIMENSION, "dimension mismatch: %llu (cols of a) != %llu (rows of b)",
                (unsigned long long)a->cols, (unsigned long long)b->rows);
  if (b->cols > 0xffffffffull)
    return fail(SPMMM_ERR_UNSUPPORTED, "b.cols=%llu exceeds the 32-bit column range",
                (unsigned long long)b->cols);
  if (a->rows >= 0xffffffffull)
    return fail(SPMMM_ERR_UNSUPPORTED, "a.rows=%llu exceeds the 32-bit row range",
                (unsigned long long)a->rows);
  const bool stats = flags & SPMMM_FLAG_ROW_STATS;
  Timer tm{c, bool(flags & SPMMM_FLAG_TIMING)};
  for (int k = 0; k < kNumKernels; ++k) c->ev_used[k] = false;
  c->last_count = 0;
  c->last_launches = 0;
  CUDA_TRY(cudaSetDevice(c->device));

  DevCsr A, B;
  rc = resolve(c, a, b, &A, &B);
  if (rc) return rc;
  const uint64_t rows = A.rows;

  const Trace tr;
  uint64_t key[5];
  cf_key(a, b, key);
  if (!(flags & kFlagCounted) && cf_candidate(c, A, B, key)) {
    const bool wide_s = B.cols > (1ull << 27) || B.nnz >= (1ull << 32) || A.nnz >= (1ull << 32) ||
                        B.rows >= (1ull << 32);
    rc = multiply_count_free(c, A, B, stats, wide_s, key, tm, out);
    if (rc != kCfFallback) {
      if (rc == SPMMM_OK && tm.on) {
        for (int k = 0; k < kNumKernels; ++k) {
          if (!c->ev_used[k]) continue;
          float ms = 0.f;
          cudaEventElapsedTime(&ms, c->ev[2 * k], c->ev[2 * k + 1]);
          c->last_ms[k] = ms;
        }
      }
      tr.mark("count-free product done");
      return rc;
    }
    // (k_prep's time and launches stay in the record: they were spent)
    tr.mark("count-free path declined: counted path");
  }
  rc = run_count(c, A, B, tm, true);
  if (rc) return rc;
  tr.mark("count done (host has totals)");
  const uint64_t total = c->h_ctrl[kCtrlTotal];
  const uint64_t max_prod = c->h_ctrl[kCtrlMaxProd];
  const bool need_table = c->h_ctrl[kCtrlNeedTable] != 0;

  // Medium kernel (per-warp tables) only when some row needs it; rows past
  // kMediumLimit products are computed by k_long before the fused pass.
  // Kernel shape. Without non-short rows: the short variant. When non-short
  // rows are a minority (skewed matrices) they vary a lot in cost, so they are
  // computed up front (split mode: k_rows / k_long) and the short variant
  // runs with them as pre-computed rows. Otherwise (most rows medium, e.g.
  // C4) medium rows are computed inline by the medium variant.
  const uint64_t nonshort = c->h_ctrl[kCtrlNonShort];
  const bool split = need_table && nonshort * 4 <= rows;
  // split-mode rows by expand-sort-compress (esc.cuh) when the 32-bit sort
  // keys can hold the columns; SPMMM_NO_ESC=1 keeps the hash-table kernels
  static const bool no_esc = std::getenv("SPMMM_NO_ESC") != nullptr;
  const bool esc = split && !no_esc && B.cols <= (1ull << kEscColBits);
  const bool medium = need_table && !split;
  const uint32_t medium_limit = medium ? kMediumLimit : 0u;
  const int pos_bits = medium ? kPosBits : 5;
  // narrow (32-bit keys and offsets) unless columns, entries or rows outgrow it
  const bool wide = B.cols > (1ull << (32 - pos_bits)) || B.nnz >= (1ull << 32) ||
                    A.nnz >= (1ull << 32) || B.rows >= (1ull << 32);
  const int rows_per_tile = medium ? 1 : kShortRowsPerTile;

  auto* p = new (std::nothrow) spmmm_product;
  if (!p) return fail(SPMMM_ERR_OOM, "host allocation failed");
  p->ctx = c;
  p->rows = rows;
  p->cols = B.cols;
  p->mults = total;
  auto cleanup = [&](int code) {
    product_release(c, p);
    delete p;
    return code;
  };
  // C storage: one reservation. The reference's own capacity rule is the
  // product count (CsrBuilder(..., estimate_nnz(a, b)), kernels.py:314); on
  // the device that is physical memory, not lazily touched pages
  // (formats.py:161-163), and for long medium rows it is far above nnz(C)
  // (C4: 705M products, 120.6M entries). The medium variant reserves
  // min(products, 8 nnz(A)) entries (SPMMM_C_RESERVE overrides 8); a product
  // that outgrows it writes nothing past it and is redone sized exactly.
  static const uint64_t reserve_factor = std::getenv("SPMMM_C_RESERVE")
                                             ? std::strtoull(std::getenv("SPMMM_C_RESERVE"), nullptr, 10)
                                             : 8;
  const uint64_t cap = (medium && !c->exact_reserve)
                           ? std::min<uint64_t>(total, std::max<uint64_t>(reserve_factor * A.nnz, 1u << 20))
                           : total;
  cudaError_t e = cache_alloc(c, (rows + 1) * 8, reinterpret_cast<void**>(&p->rp), &p->cap[0]);
  if (e == cudaSuccess)
    e = cache_alloc(c, std::max<uint64_t>(cap, 1) * 8, reinterpret_cast<void**>(&p->ci), &p->cap[1]);
  if (e == cudaSuccess)
    e = cache_alloc(c, std::max<uint64_t>(cap, 1) * 8, reinterpret_cast<void**>(&p->v), &p->cap[2]);
  if (e == cudaSuccess && stats)
    e = cache_alloc(c, std::max<uint64_t>(rows, 1) * 3 * sizeof(uint32_t),
                    reinterpret_cast<void**>(&p->st), &p->cap[3]);
  if (e != cudaSuccess)
    return cleanup(fail(e == cudaErrorMemoryAllocation ? SPMMM_ERR_OOM : SPMMM_ERR_CUDA,
                        "allocating C (%llu entries): %s", (unsigned long long)total,
                        cudaGetErrorString(e)));
  if (!rows) {  // otherwise k_fused's first tile writes row_ptr[0]
    e = cudaMemsetAsync(p->rp, 0, sizeof(uint64_t), c->stream);
    if (e != cudaSuccess) return cleanup(fail(SPMMM_ERR_CUDA, "%s", cudaGetErrorString(e)));
  }
  tr.mark("C allocated");

  // staging of pre-computed rows: context buffers, grown on demand and kept
  // (a per-call cudaMallocAsync of this size costs milliseconds of pool work)
  DevBuf& stage_ci = c->stage_ci;
  DevBuf& stage_v = c->stage_v;
  auto fail_staged = [&](int code) { return cleanup(code); };
  const bool has_long = split || (medium && max_prod > medium_limit);
  if (rows && has_long) {
    rc = run_long(c, A, B, max_prod, medium_limit, split, esc, total, stats, p, stage_ci,
                  stage_v, tm);
    if (rc) return fail_staged(rc);
    tr.mark("long rows launched");
  }

  if (rows) {
    const uint64_t ntiles = (rows + rows_per_tile - 1) / rows_per_tile;
    // look-back levels: words per level, then counters of levels 1..
    uint64_t nl[kLevels];
    nl[0] = ntiles;
    for (int l = 1; l < kLevels; ++l) nl[l] = (nl[l - 1] + 31) / 32;
    c->epoch += 1;
    FusedParams fp{};
    {
      // counters at the front (zeroed by k_count), then the status words
      unsigned long long* cnt = static_cast<unsigned long long*>(c->status.p);
      uint64_t* w = reinterpret_cast<uint64_t*>(cnt + lb_counters_max(rows));
      fp.lb.count[0] = nullptr;
      for (int l = 0; l < kLevels; ++l) {
        fp.lb.stat[l] = w;
        fp.lb.n[l] = nl[l];
        w += nl[l];
        if (l > 0) {
          fp.lb.count[l] = cnt;
          cnt += nl[l];
        }
      }
      fp.lb.epoch = c->epoch;
      fp.lb.fault = static_cast<unsigned long long*>(c->ctrl.p) + kCtrlFault;
    }
    fp.ticket = static_cast<unsigned long long*>(c->ctrl.p) + kCtrlTicket;
    fp.nnz_out = static_cast<unsigned long long*>(c->ctrl.p) + kCtrlNnz;
    fp.A = A;
    fp.B = B;
    fp.prod = static_cast<const uint32_t*>(c->prod.p);
    fp.lmap = static_cast<const uint32_t*>(c->lmap.p);
    fp.l_nnz = static_cast<const uint32_t*>(c->l_nnz.p);
    fp.c_rp = p->rp;
    fp.c_ci = p->ci;
    fp.c_v = p->v;
    fp.ntiles = ntiles;
    fp.medium_limit = medium_limit;
    fp.a_is_b = (A.ci == B.ci && A.v == B.v) ? 1u : 0u;
    fp.ell = nullptr;
    // short variant over a B whose rows all fit an ELL record: pack B once per
    // call (one 64-byte record per row; a referenced B row is then one block)
    if (ell_wanted(c->h_ctrl, rows)) fp.ell = static_cast<const uint32_t*>(c->ell.p);
    fp.g_keys = nullptr;
    fp.g_vals = nullptr;
    fp.g_scol = nullptr;
    fp.g_sval = nullptr;
    fp.st_min = p->st;
    fp.st_max = p->st ? p->st + rows : nullptr;
    fp.st_touch = p->st ? p->st + 2 * rows : nullptr;
    fp.cf_flags = nullptr;
    fp.cf_total = nullptr;
    fp.cf_err = static_cast<unsigned long long*>(c->ctrl.p) + kCtrlCfFlags;  // (kCfOverflow)
    fp.c_cap = cap;
    // split mode without stats: the packed-passes instantiation (its narrow
    // sort key holds row slot, column and lane: columns < 2^24)
    const bool split_variant = kSplitVariant && split && !stats &&
                               (wide || B.cols <= (1ull << kTileColBits));
    int occ = 0;
    rc = fused_call(c, medium, 0, fp, wide, stats, 0, &occ, false, 0, split_variant);
    if (rc) return fail_staged(rc);
    const unsigned grid = unsigned(std::min<uint64_t>(
        (ntiles + kFusedWarps - 1) / kFusedWarps, uint64_t(occ) * uint64_t(c->sms)));
    if (medium) {
      GtabView gv;
      rc = ensure_gtab(c, uint64_t(grid) * kFusedWarps, &gv);
      if (rc) return fail_staged(rc);
      fp.g_keys = gv.keys;
      fp.g_vals = gv.vals;
      fp.g_scol = gv.scol;
      fp.g_sval = gv.sval;
    }
    tm.begin(3);
    rc = fused_call(c, medium, 1, fp, wide, stats, grid, nullptr, false, 0, split_variant);
    if (rc) return fail_staged(rc);
    tm.end(3);
    ++c->last_launches;
    if (has_long) {
      tm.begin(4);
      CopyParams cp;
      cp.list = static_cast<const uint32_t*>(c->list.p);
      cp.prod = static_cast<const uint32_t*>(c->prod.p);
      cp.big = static_cast<const uint32_t*>(c->sub.p);
      static const bool env_no_dom = std::getenv("SPMMM_NO_DOM") != nullptr;
      cp.dom_big = (esc && !env_no_dom && !c->no_dom) ? cp.big + 4 * rows : nullptr;
      cp.ctrl = static_cast<const unsigned long long*>(c->ctrl.p);
      cp.tickets = static_cast<unsigned long long*>(c->ctrl.p) + kCtrlCopyTickets;
      cp.l_off = static_cast<const uint64_t*>(c->l_off.p);
      cp.l_nnz = static_cast<const uint32_t*>(c->l_nnz.p);
      cp.l_ci = static_cast<const uint32_t*>(stage_ci.p);
      cp.l_v = static_cast<const double*>(stage_v.p);
      cp.c_rp = p->rp;
      cp.c_ci = p->ci;
      cp.c_v = p->v;
      cp.rows = rows;
      cp.long_min = esc ? kEscWarpLimit : split ? kRowsLimit : kMediumLimit;
      const bool parts = esc && max_prod > kEscBlockCap;
      cp.row_pbase = parts ? static_cast<const uint32_t*>(c->row_parts.p) : nullptr;
      cp.row_np = parts ? cp.row_pbase + (c->h_ctrl[kCtrlHugeProducts] / kHugeMin + 16) : nullptr;
      cp.part_off = parts ? static_cast<const uint64_t*>(c->part_off.p) : nullptr;
      cp.part_nnz = parts ? static_cast<const uint32_t*>(c->part_nnz.p) : nullptr;
      cp.c_cap = cap;
      cp.overflow = static_cast<unsigned long long*>(c->ctrl.p) + kCtrlCfFlags;
      k_copy_long<<<c->sms * 8, 256, 0, c->stream>>>(cp);
      e = cudaGetLastError();
      if (e != cudaSuccess) return fail_staged(fail(SPMMM_ERR_CUDA, "k_copy_long: %s",
                                                    cudaGetErrorString(e)));
      tm.end(4);
      ++c->last_launches;
    }
  }
  tr.mark("fused + copy launched");
  // one read-back: the watchdog word through nnz(C) and the overflow word
  // (rows == 0: nnz is 0)
  static_assert(kCtrlNnz > kCtrlFault && kCtrlCfFlags > kCtrlNnz, "ctrl layout");
  if (!rows) {
    c->h_ctrl[kCtrlNnz] = 0;
    c->h_ctrl[kCtrlCfFlags] = 0;
  }
  ++c->last_launches;  // (k_readback)
  e = readback(static_cast<const unsigned long long*>(c->ctrl.p) + kCtrlFault, c->h_ctrl + kCtrlFault,
               rows ? kCtrlCfFlags - kCtrlFault + 1 : 1, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cleanup(fail(SPMMM_ERR_CUDA, "multiply: %s", cudaGetErrorString(e)));
  if (c->h_ctrl[kCtrlFault]) {
    const unsigned long long f = c->h_ctrl[kCtrlFault];
    return cleanup(fail(SPMMM_ERR_CUDA, "k_fused look-back watchdog: site %llu tile %llu",
                        (f >> 48) & 0x7fff, f & ((1ull << 48) - 1)));
  }
  if (c->h_ctrl[kCtrlCfFlags] & kCfUnsorted) {
    // a B row whose columns do not ascend (outside the storage contract, but
    // the other kernels sort whatever they are given): once more without
    // k_esc_dom, which merges its dominant B row as it is stored
    cleanup(0);
    tr.mark("unsorted B row met by k_esc_dom: redone without it");
    c->no_dom = true;
    rc = multiply_impl(c, a, b, strategy, flags, out);
    c->no_dom = false;
    return rc;
  }
  if (c->h_ctrl[kCtrlCfFlags] & kCfOverflow) {
    // C outgrew the reservation: once more, sized by the product count
    cleanup(0);
    tr.mark("C outgrew its reservation: redone sized exactly");
    c->exact_reserve = true;
    rc = multiply_impl(c, a, b, strategy, flags, out);
    c->exact_reserve = false;
    return rc;
  }
  p->nnz = c->h_ctrl[kCtrlNnz];
  tr.mark("done");
  if (tm.on) {
    for (int k = 0; k < kNumKernels; ++k) {
      if (!c->ev_used[k]) continue;
      float ms = 0.f;
      cudaEventElapsedTime(&ms, c->ev[2 * k], c->ev[2 * k + 1]);
      c->last_ms[k] = ms;
    }
  }
  *out = p;
  return SPMMM_OK;
}


// ---- block-pipelined product of host operands (spmmm_multiply_host) ---------
//
// PCIe, not the kernels, bounds a product whose operands and result live on
// the host (C2: 0.37 GB up, 0.91 GB down against ~1.4 ms of kernels). A goes
// up in G row blocks of about equal nnz — row pointers, columns, values —
// (for A != B all of B first: any A row may read any B row); there is no
// global count pass. Block j is computed as soon as every B row it reads is
// resident (for C = A·A a small kernel on the upload stream finds the
// block's largest column, which names the last row of B = A it reads), by
// the ordinary device product of a row block of A (rows are independent,
// kernels.py:323-329: its own count validates it and sizes its part of C),
// and its part of C streams down while the next block computes, so uploads,
// kernels and downloads overlap (PCIe is full duplex). Its row_ptr is
// shifted by the nnz before it on the device and it lands at its offset in
// one result, so the bytes are those of spmmm_multiply. Pageable operands go
// up through page-locked staging on an uploader thread (Stager).

constexpr int kPipeSplit = 64;

struct PipeBounds {
  uint64_t r[kMaxPipeBlocks + 1];
};

__global__ void k_block_maxcol(const uint64_t* __restrict__ rp, const uint64_t* __restrict__ ci,
                               const PipeBounds bounds, unsigned long long* __restrict__ out) {
  // kPipeSplit blocks per row block, each a slice of its entries
  const uint32_t j = blockIdx.x / kPipeSplit, part = blockIdx.x % kPipeSplit;
  const uint64_t e0 = rp[bounds.r[j]], e1 = rp[bounds.r[j + 1]];
  uint64_t m = 0;
  for (uint64_t e = e0 + uint64_t(part) * blockDim.x + threadIdx.x; e < e1;
       e += uint64_t(kPipeSplit) * blockDim.x)
    m = ci[e] > m ? ci[e] : m;
  m = __reduce_max_sync(0xffffffffu, uint32_t(m));  // columns < 2^32 (checked)
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out + j, (unsigned long long)m);
}

// C's column indices go down as u32 (columns < 2^32 are checked): half the
// PCIe bytes of col_idx; host threads widen them while the values follow.
__global__ void k_narrow(const uint64_t* __restrict__ src, uint32_t* __restrict__ dst,
                         uint64_t n) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    dst[i] = uint32_t(__ldcs(reinterpret_cast<const unsigned long long*>(src) + i));
}

// Stencil-like results: each 64-entry chunk of C's columns (chunks aligned
// to the global entry index) spans < 2^16 columns, so the columns go down as
// u16 deltas from a per-chunk base — half the bytes of u32. A block whose
// chunks do not all fit clears *ok (mapped host word) and goes down as u32.
// ci: the block's columns (global entries [off, off + n)); base: per chunk of
// the block, from chunk off >> 6.
__global__ void k_delta16(const uint64_t* __restrict__ ci, uint64_t off, uint64_t n,
                          uint32_t* __restrict__ base, uint16_t* __restrict__ delta,
                          unsigned int* __restrict__ ok) {
  const uint64_t c0 = off >> 6, c1 = (off + n + 63) >> 6;
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t nw = uint64_t(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t c = c0 + uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); c < c1;
       c += nw) {
    const uint64_t lo = c * 64 > off ? c * 64 : off, hi = (c + 1) * 64 < off + n ? (c + 1) * 64 : off + n;
    uint32_t v[2];
    uint32_t mn = 0xffffffffu, mx = 0;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint64_t e = lo + lane + 32u * u;
      v[u] = e < hi ? uint32_t(__ldcs(reinterpret_cast<const unsigned long long*>(ci) + (e - off)))
                    : 0u;
      if (e < hi) {
        mn = v[u] < mn ? v[u] : mn;
        mx = v[u] > mx ? v[u] : mx;
      }
    }
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (hi > lo && mx - mn >= 65536u && lane == 0) *reinterpret_cast<volatile unsigned int*>(ok) = 0;
    if (lane == 0) base[c - c0] = mn;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint64_t e = lo + lane + 32u * u;
      if (e < hi) delta[e] = uint16_t(v[u] - mn);
    }
  }
}

__global__ void k_zero_u64(uint64_t* p, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = 0;
}

__global__ void k_add_offset(uint64_t* __restrict__ rp, uint64_t n, uint64_t off) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    rp[i] += off;
}

int pipe_setup(spmmm_context* c) {
  if (c->s_up) return SPMMM_OK;
  CUDA_TRY(cudaStreamCreateWithFlags(&c->s_up, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&c->s_down, cudaStreamNonBlocking));
  for (cudaEvent_t& ev : c->pev) CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  // the widening workers sleep on these instead of spinning next to the
  // thread that issues the work
  for (int j = 0; j < kMaxPipeBlocks; ++j) {
    cudaEvent_t& ev = c->pev[2 + 3 * kMaxPipeBlocks + j];
    CUDA_TRY(cudaEventDestroy(ev));
    CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming | cudaEventBlockingSync));
  }
  CUDA_TRY(cudaMallocHost(&c->h_aux, 2 * kMaxPipeBlocks * sizeof(unsigned long long)));
  return SPMMM_OK;
}

// u32 -> u64 widening of downloaded column indices (host). AVX2 with
// streaming stores when the CPU has it: the result is written once and not
// read back soon, so skipping the read-for-ownership halves the memory
// traffic that competes with the DMA landing the next blocks.
__attribute__((target("avx2"))) void widen_avx2(const uint32_t* in, uint64_t* out, uint64_t n) {
  uint64_t i = 0;
  while (i < n && (reinterpret_cast<uintptr_t>(out + i) & 31)) {
    out[i] = in[i];
    ++i;
  }
  for (; i + 8 <= n; i += 8) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(in + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(in + i + 4));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(out + i), _mm256_cvtepu32_epi64(a));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(out + i + 4), _mm256_cvtepu32_epi64(b));
  }
  for (; i < n; ++i) out[i] = in[i];
  _mm_sfence();
}

// out[i] = base[(i >> 6) - cb] + delta[i] for global entries i in [i0, i1)
__attribute__((target("avx2"))) void widen16_avx2(const uint16_t* delta, const uint32_t* base,
                                                   uint64_t cb, uint64_t* out, uint64_t i0,
                                                   uint64_t i1) {
  uint64_t i = i0;
  for (; i < i1 && (i & 3); ++i) out[i] = uint64_t(base[(i >> 6) - cb]) + delta[i];
  for (; i + 4 <= i1; i += 4) {  // 4 entries never straddle a 64-entry chunk
    const __m256i b = _mm256_set1_epi64x(static_cast<long long>(base[(i >> 6) - cb]));
    const __m128i d = _mm_loadl_epi64(reinterpret_cast<const __m128i*>(delta + i));
    const __m256i w = _mm256_add_epi64(_mm256_cvtepu16_epi64(d), b);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(out + i), w);
  }
  for (; i < i1; ++i) out[i] = uint64_t(base[(i >> 6) - cb]) + delta[i];
  _mm_sfence();
}

void widen16(const uint16_t* delta, const uint32_t* base, uint64_t cb, uint64_t* out,
             uint64_t i0, uint64_t i1) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (avx2 && (reinterpret_cast<uintptr_t>(out) & 31) == 0) {
    widen16_avx2(delta, base, cb, out, i0, i1);
    return;
  }
  for (uint64_t i = i0; i < i1; ++i) out[i] = uint64_t(base[(i >> 6) - cb]) + delta[i];
}

void widen(const uint32_t* in, uint64_t* out, uint64_t n) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (avx2) {
    widen_avx2(in, out, n);
    return;
  }
  for (uint64_t i = 0; i < n; ++i) out[i] = in[i];
}

int host_alloc_internal(uint64_t bytes, void** ptr) { return spmmm_host_alloc(bytes, ptr); }
int host_free_internal(void* ptr) { return ptr ? spmmm_host_free(ptr) : SPMMM_OK; }

// ---- uploads from pageable host memory -------------------------------------
//
// cudaMemcpyAsync from pageable memory stages through the driver's own small
// buffers at the speed of one host thread, serialised with the caller. The
// reference's callers hand over ordinary numpy arrays (formats.py:35-58), so
// the pipelined path stages them itself: a few page-locked slots, each chunk
// copied into a slot by several host threads while the copy engine moves the
// previous slots to the device.
class CopyPool {
 public:
  explicit CopyPool(int n) {
    for (int i = 0; i < n; ++i) th_.emplace_back([this, i]() { loop(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_.store(true);
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return int(th_.size()); }
  // dst[0, n) = src[0, n), split over the pool's threads and the caller.
  // Workers spin briefly before sleeping: chunks follow each other within
  // microseconds and a condition-variable wake-up costs tens of them.
  void copy(void* dst, const void* src, size_t n) {
    dst_ = static_cast<char*>(dst);
    src_ = static_cast<const char*>(src);
    n_ = n;
    pending_.store(size(), std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> lk(mu_);
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    piece(size());
    while (pending_.load(std::memory_order_acquire) != 0) _mm_pause();
  }

 private:
  void piece(int i) {
    const size_t parts = size_t(size()) + 1;
    const size_t a = n_ * size_t(i) / parts, b = n_ * size_t(i + 1) / parts;
    if (b > a) std::memcpy(dst_ + a, src_ + a, b - a);
  }
  void loop(int i) {
    uint64_t seen = 0;
    while (true) {
      uint64_t g = gen_.load(std::memory_order_acquire);
      for (int spin = 0; g == seen && spin < 20000 && !stop_.load(); ++spin) {
        _mm_pause();
        g = gen_.load(std::memory_order_acquire);
      }
      if (g == seen) {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&]() { return stop_.load() || gen_.load() != seen; });
        g = gen_.load(std::memory_order_acquire);
      }
      if (stop_.load()) return;
      seen = g;
      piece(i);
      pending_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::atomic<bool> stop_{false};
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> pending_{0};
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t n_ = 0;
};

struct Stager {
  static constexpr int kSlots = 8;
  static constexpr size_t kSlotBytes = size_t(4) << 20;
  void* slot[kSlots] = {};
  cudaEvent_t done[kSlots] = {};
  int next = 0;
  CopyPool* pool = nullptr;
  ~Stager() {
    for (int k = 0; k < kSlots; ++k) {
      if (done[k]) cudaEventSynchronize(done[k]);
      if (slot[k]) spmmm_host_free(slot[k]);
      if (done[k]) cudaEventDestroy(done[k]);
    }
    delete pool;
  }
  cudaError_t init() {
    if (pool) return cudaSuccess;
    for (int k = 0; k < kSlots; ++k) {
      if (spmmm_host_alloc(kSlotBytes, &slot[k]) != SPMMM_OK) return cudaErrorMemoryAllocation;
      cudaError_t e = cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    cpu_set_t cs;
    const int ncpu = sched_getaffinity(0, sizeof(cs), &cs) == 0 ? CPU_COUNT(&cs) : 8;
    static const int env = std::getenv("SPMMM_STAGE_THREADS")
                               ? std::atoi(std::getenv("SPMMM_STAGE_THREADS")) : 0;
    // 6 on a 16-core host (C3 pageable e2e 21.7 / 19.7 / 19.9 ms with 4 / 6 / 8)
    pool = new CopyPool(std::max(0, (env > 0 ? env : std::max(1, std::min(ncpu * 3 / 8, 6))) - 1));
    return cudaSuccess;
  }
  // host (pageable) -> device on stream s, through the slots
  cudaError_t copy(void* dst, const void* src, size_t bytes, cudaStream_t s,
                   const std::atomic<bool>& abort) {
    for (size_t off = 0; off < bytes && !abort.load(std::memory_order_relaxed);
         off += kSlotBytes) {
      const size_t n = std::min(kSlotBytes, bytes - off);
      const int k = next++ % kSlots;
      cudaError_t e = cudaEventSynchronize(done[k]);  // the slot's last copy has left
      if (e != cudaSuccess) return e;
      pool->copy(slot[k], static_cast<const char*>(src) + off, n);
      e = cudaMemcpyAsync(static_cast<char*>(dst) + off, slot[k], n, cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) return e;
      e = cudaEventRecord(done[k], s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
};

bool host_pinned(const void* p) {
  if (!p) return true;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// One host->device copy on the context stream: pageable sources of 8 MiB and
// more go through the page-locked staging slots (several host threads), the
// rest straight to the copy engine.
int stage_h2d(spmmm_context* c, void* dst, const void* src, size_t bytes) {
  if (!bytes) return SPMMM_OK;
  static const bool no_stage = std::getenv("SPMMM_NO_STAGE") != nullptr;
  if (bytes >= (size_t(8) << 20) && !no_stage && !host_pinned(src)) {
    if (!c->stager) c->stager = new (std::nothrow) Stager;
    if (!c->stager) return fail(SPMMM_ERR_OOM, "host allocation failed");
    CUDA_TRY(c->stager->init());
    const std::atomic<bool> no_abort{false};
    CUDA_TRY(c->stager->copy(dst, src, bytes, c->stream, no_abort));
    return SPMMM_OK;
  }
  CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
  return SPMMM_OK;
}

int multiply_host_impl(spmmm_context* c, const spmmm_csr* a, const spmmm_csr* b, int strategy,
                       uint32_t flags, int blocks, spmmm_host_csr* out) {
  if (!out) return fail(SPMMM_ERR_INVALID, "out is NULL");
  if (strategy < SPMMM_STRATEGY_BFDOUBLE || strategy > SPMMM_STRATEGY_COMBINED)
    return fail(SPMMM_ERR_INVALID, "unknown strategy %d", strategy);
  int rc = check_view(a, "a");
  if (rc) return rc;
  rc = check_view(b, "b");
  if (rc) return rc;
  if (a->memory != SPMMM_MEM_HOST || b->memory != SPMMM_MEM_HOST)
    return fail(SPMMM_ERR_INVALID, "spmmm_multiply_host takes host operands");
  if (flags & SPMMM_FLAG_ROW_STATS)
    return fail(SPMMM_ERR_INVALID, "row stats need spmmm_multiply");
  if (a->cols != b->rows)
    return fail(SPMMM_ERR_DIMENSION, "dimension mismatch: %llu (cols of a) != %llu (rows of b)",
                (unsigned long long)a->cols, (unsigned long long)b->rows);
  if (b->cols > 0xffffffffull)
    return fail(SPMMM_ERR_UNSUPPORTED, "b.cols=%llu exceeds the 32-bit column range",
                (unsigned long long)b->cols);
  if (a->rows >= 0xffffffffull)
    return fail(SPMMM_ERR_UNSUPPORTED, "a.rows=%llu exceeds the 32-bit row range",
                (unsigned long long)a->rows);
  const uint64_t* arp = a->row_ptr;
  CUDA_TRY(cudaSetDevice(c->device));
  const Trace tr;
  rc = pipe_setup(c);
  if (rc) return rc;
  const bool same = a->row_ptr == b->row_ptr && a->col_idx == b->col_idx &&
                    a->values == b->values && a->rows == b->rows && a->nnz == b->nnz;
  const int G = std::max(1, std::min(blocks, kMaxPipeBlocks));
  cudaEvent_t* ev_struct = &c->pev[0];
  cudaEvent_t* ev_bv = &c->pev[1];
  cudaEvent_t* ev_av = &c->pev[2];
  cudaEvent_t* ev_comp = &c->pev[2 + kMaxPipeBlocks];
  cudaEvent_t* ev_down = &c->pev[2 + 2 * kMaxPipeBlocks];
  // device operands
  const size_t rpb = (a->rows + 1) * 8;
  CUDA_TRY(ensure(c->a_rp, rpb, c->stream));
  CUDA_TRY(ensure(c->a_ci, a->nnz * 8, c->stream));
  CUDA_TRY(ensure(c->a_v, a->nnz * 8, c->stream));
  if (!same) {
    CUDA_TRY(ensure(c->b_rp, (b->rows + 1) * 8, c->stream));
    CUDA_TRY(ensure(c->b_ci, b->nnz * 8, c->stream));
    CUDA_TRY(ensure(c->b_v, b->nnz * 8, c->stream));
  }
  CUDA_TRY(ensure(c->aux, (2 * kMaxPipeBlocks + 2) * 8, c->stream));
  // buffers (re)allocated on the context stream must exist before s_up uses them
  CUDA_TRY(cudaEventRecord(*ev_struct, c->stream));
  // SPMMM_TRACE: a GPU timeline of the call (upload, compute, download of
  // every block, relative to this point), printed at the end
  cudaEvent_t tl[1 + 3 * kMaxPipeBlocks] = {};
  if (tr.on) {
    for (cudaEvent_t& ev : tl) cudaEventCreate(&ev);
    cudaEventRecord(tl[0], c->stream);
  }
  CUDA_TRY(cudaStreamWaitEvent(c->s_up, *ev_struct, 0));
  uint64_t* d_arp = static_cast<uint64_t*>(c->a_rp.p);
  uint64_t* d_aci = static_cast<uint64_t*>(c->a_ci.p);
  double* d_av = static_cast<double*>(c->a_v.p);
  // row blocks of about equal nnz(A)
  uint64_t bound[kMaxPipeBlocks + 1];
  bound[0] = 0;
  for (int j = 1; j < G; ++j) {
    const uint64_t target = a->nnz * uint64_t(j) / uint64_t(G);
    bound[j] = uint64_t(std::lower_bound(arp, arp + a->rows + 1, target) - arp);
    bound[j] = std::max(bound[j], bound[j - 1]);
    bound[j] = std::min<uint64_t>(bound[j], a->rows);
  }
  bound[G] = a->rows;
  // the uploads below trust these entries (each block's k_count checks the rest)
  for (int j = 0; j < G && a->rows; ++j)
    if (arp[bound[j]] > arp[bound[j + 1]] || arp[bound[j + 1]] > a->nnz)
      return fail(SPMMM_ERR_INVALID, "malformed a.row_ptr (decreasing or past nnz)");
  // 1. uploads, in the order the blocks need them. A != B: all of B first
  // (any A row may read any B row). Then A block by block — row pointers,
  // columns, values — and for C = A·A each block's largest column as soon as
  // its columns are up: it names the last row of B = A that the block reads.
  // No global count pass: block 0 starts as soon as its inputs are resident
  // (each block's own count validates it and sizes its part of C).
  cudaEvent_t* ev_maxc = &c->pev[2 + 4 * kMaxPipeBlocks];
  uint64_t* d_aux = static_cast<uint64_t*>(c->aux.p);
  // Pageable operands (ordinary numpy arrays) go up through page-locked
  // staging on an uploader thread; the compute loop below waits for each
  // block's upload step to be issued (events must be recorded before a
  // stream can wait on them). Pinned operands are issued right here.
  const bool pageable = !host_pinned(a->row_ptr) || !host_pinned(a->col_idx) ||
                        !host_pinned(a->values) ||
                        (!same && (!host_pinned(b->row_ptr) || !host_pinned(b->col_idx) ||
                                   !host_pinned(b->values)));
  static const bool no_stage = std::getenv("SPMMM_NO_STAGE") != nullptr;
  const bool staged = pageable && !no_stage;
  if (staged) {
    if (!c->stager) c->stager = new (std::nothrow) Stager;
    if (!c->stager) return fail(SPMMM_ERR_OOM, "host allocation failed");
    CUDA_TRY(c->stager->init());
  }
  std::atomic<bool> up_abort{false};
  std::atomic<int> up_issued{0};  // upload steps issued: 1 (B) + one per A block
  std::atomic<int> up_error{0};
  std::string up_msg;
  std::mutex up_mu;
  std::condition_variable up_cv;
  auto h2d = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
    if (!bytes) return cudaSuccess;
    if (staged) return c->stager->copy(dst, src, bytes, c->s_up, up_abort);
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->s_up);
  };
  auto issue_uploads = [&]() -> int {
    cudaSetDevice(c->device);
    auto step_done = [&](int n) {
      {
        std::lock_guard<std::mutex> lk(up_mu);
        up_issued.store(n, std::memory_order_release);
      }
      up_cv.notify_all();
    };
    if (!same) {
      CUDA_TRY(h2d(c->b_rp.p, b->row_ptr, (b->rows + 1) * 8));
      CUDA_TRY(h2d(c->b_ci.p, b->col_idx, b->nnz * 8));
      CUDA_TRY(h2d(c->b_v.p, b->values, b->nnz * 8));
    }
    CUDA_TRY(cudaEventRecord(*ev_bv, c->s_up));
    step_done(1);
    for (int j = 0; j < G && !up_abort.load(); ++j) {
      const uint64_t r0 = bound[j], r1 = bound[j + 1];
      const uint64_t e0 = a->rows ? arp[r0] : 0, e1 = a->rows ? arp[r1] : 0;
      CUDA_TRY(h2d(d_arp + r0, arp + r0, (r1 - r0 + 1) * 8));
      if (e1 > e0) CUDA_TRY(h2d(d_aci + e0, a->col_idx + e0, (e1 - e0) * 8));
      if (same && r1 > r0) {
        PipeBounds pb;
        pb.r[0] = r0;
        pb.r[1] = r1;
        k_zero_u64<<<1, 32, 0, c->s_up>>>(d_aux + j, 1);
        k_block_maxcol<<<kPipeSplit, 256, 0, c->s_up>>>(
            d_arp, d_aci, pb, reinterpret_cast<unsigned long long*>(d_aux + j));
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(readback(reinterpret_cast<const unsigned long long*>(d_aux + j), c->h_aux + j, 1,
                          c->s_up));
        CUDA_TRY(cudaEventRecord(ev_maxc[j], c->s_up));
      }
      if (e1 > e0) CUDA_TRY(h2d(d_av + e0, a->values + e0, (e1 - e0) * 8));
      CUDA_TRY(cudaEventRecord(ev_av[j], c->s_up));
      if (tr.on) cudaEventRecord(tl[1 + j], c->s_up);
      step_done(j + 2);
    }
    return SPMMM_OK;
  };
  std::thread uploader;
  if (staged) {
    uploader = std::thread([&]() {
      const int rc_up = issue_uploads();
      if (rc_up) {
        std::lock_guard<std::mutex> lk(up_mu);
        up_msg = g_error;  // (thread-local: carried over to the caller's thread)
        up_error.store(rc_up);
      }
      {
        std::lock_guard<std::mutex> lk(up_mu);
        up_issued.store(G + 2, std::memory_order_release);  // nothing more will come
      }
      up_cv.notify_all();
    });
  } else {
    rc = issue_uploads();
    if (rc) {
      cudaStreamSynchronize(c->s_up);
      return rc;
    }
  }
  auto join_uploader = [&]() {
    if (uploader.joinable()) {
      up_abort.store(true);
      uploader.join();
    }
  };
  // until the uploader has issued step n (1: B, j + 2: A block j)
  auto wait_upload = [&](int n) -> int {
    if (!staged) return SPMMM_OK;
    std::unique_lock<std::mutex> lk(up_mu);
    up_cv.wait(lk, [&]() { return up_issued.load(std::memory_order_acquire) >= n; });
    if (up_error.load()) return fail(up_error.load(), "%s", up_msg.c_str());
    return SPMMM_OK;
  };
  DevCsr B{d_arp, d_aci, d_av, a->rows, a->cols, a->nnz};
  if (!same)
    B = DevCsr{static_cast<const uint64_t*>(c->b_rp.p), static_cast<const uint64_t*>(c->b_ci.p),
               static_cast<const double*>(c->b_v.p), b->rows, b->cols, b->nnz};
  B.cols = b->cols;
  auto drain = [&](int code) {
    join_uploader();
    cudaStreamSynchronize(c->s_up);
    cudaStreamSynchronize(c->s_down);
    cudaStreamSynchronize(c->stream);
    return code;
  };
  tr.mark(staged ? "pipe: staged uploads started" : "pipe: uploads issued");
  // 4. the result, in pinned host memory from the pool: 8 nnz(A) entries
  // (C2 2.6, C3 5, C4 4.6, C5 6 nnz(C) per A entry); should a block overflow
  // that, the product is redone in one shot (below).
  const char* cap_knob = std::getenv("SPMMM_PIPE_CAP");  // test knob, read per call
  const uint64_t cap_env = cap_knob ? std::strtoull(cap_knob, nullptr, 10) : 0;
  const uint64_t cap = cap_env ? cap_env : std::max<uint64_t>(8 * a->nnz, 1ull << 20);
  void *hrp = nullptr, *hci = nullptr, *hv = nullptr;
  rc = host_alloc_internal(rpb, &hrp);
  if (!rc) rc = host_alloc_internal(std::max<uint64_t>(cap, 1) * 8, &hci);
  if (!rc) rc = host_alloc_internal(std::max<uint64_t>(cap, 1) * 8, &hv);
  auto free_out = [&]() {
    host_free_internal(hrp);
    host_free_internal(hci);
    host_free_internal(hv);
    hrp = hci = hv = nullptr;
  };
  if (rc) {
    free_out();
    return drain(rc);
  }
  tr.mark("pipe: outputs allocated");
  uint64_t* out_rp = static_cast<uint64_t*>(hrp);
  uint64_t* out_ci = static_cast<uint64_t*>(hci);
  double* out_v = static_cast<double*>(hv);
  out_rp[0] = 0;
  // 5. blocks: compute when their inputs are resident, then stream down.
  // Column indices travel as u32 into a pinned staging area; worker threads
  // widen each block into the result as soon as its indices have landed.
  cudaEvent_t* ev_ci = &c->pev[2 + 3 * kMaxPipeBlocks];
  static const bool no_narrow = std::getenv("SPMMM_NO_NARROW") != nullptr;
  static const int widen_threads = std::getenv("SPMMM_WIDEN_THREADS")
                                       ? std::atoi(std::getenv("SPMMM_WIDEN_THREADS")) : 0;
  const bool narrow = cap >= kNarrowMin && cap < (1ull << 32) && !no_narrow;
  void* hci32 = nullptr;
  void* hrp32 = nullptr;
  void* hd16 = nullptr;
  void* hbase = nullptr;
  const uint64_t max_chunks = cap / 64 + 2 * uint64_t(G) + 16;
  if (narrow) {
    CUDA_TRY(ensure(c->ci32, cap * 4, c->stream));
    CUDA_TRY(ensure(c->rp32, (a->rows + 1) * 4, c->stream));
    CUDA_TRY(ensure(c->d16, cap * 2, c->stream));
    CUDA_TRY(ensure(c->dbase, max_chunks * 4, c->stream));
    rc = host_alloc_internal((a->rows + 1) * 4, &hrp32);
    if (!rc) rc = host_alloc_internal(cap * 2, &hd16);
    if (!rc) rc = host_alloc_internal(max_chunks * 4, &hbase);
    if (!rc) rc = host_alloc_internal(cap * 4, &hci32);
    if (rc) {
      free_out();
      return drain(rc);
    }
  }
  uint32_t* d_ci32 = static_cast<uint32_t*>(c->ci32.p);
  uint32_t* h_ci32 = static_cast<uint32_t*>(hci32);
  uint32_t* d_rp32 = static_cast<uint32_t*>(c->rp32.p);
  uint32_t* h_rp32 = static_cast<uint32_t*>(hrp32);
  uint16_t* d_d16 = static_cast<uint16_t*>(c->d16.p);
  uint16_t* h_d16 = static_cast<uint16_t*>(hd16);
  uint32_t* d_base = static_cast<uint32_t*>(c->dbase.p);
  uint32_t* h_base = static_cast<uint32_t*>(hbase);
  static const bool no_delta = std::getenv("SPMMM_NO_DELTA16") != nullptr;
  uint64_t blk_off[kMaxPipeBlocks] = {}, blk_n[kMaxPipeBlocks] = {};
  uint64_t blk_r0[kMaxPipeBlocks] = {}, blk_r1[kMaxPipeBlocks] = {};
  uint64_t blk_cb[kMaxPipeBlocks] = {};  // first chunk base of the block (u16 mode)
  bool blk_on[kMaxPipeBlocks] = {}, blk_16[kMaxPipeBlocks] = {};
  uint64_t cb_next = 0, d2h = 0;
  std::atomic<int> issued{0};
  std::mutex issue_mu;
  std::condition_variable issue_cv;
  auto publish = [&](int n) {
    {
      std::lock_guard<std::mutex> lk(issue_mu);
      issued.store(n, std::memory_order_release);
    }
    issue_cv.notify_all();
  };
  std::atomic<bool> abort_widen{false};
  std::vector<std::thread> workers;
  int nthreads = 1;
  if (narrow) {
    cpu_set_t cs;
    int ncpu = sched_getaffinity(0, sizeof(cs), &cs) == 0 ? CPU_COUNT(&cs) : 8;
    nthreads = widen_threads > 0 ? widen_threads : std::max(1, std::min(ncpu / 4, 4));
    for (int w = 0; w < nthreads; ++w) {
      workers.emplace_back([&, w]() {
        cudaSetDevice(c->device);
        for (int j = 0; j < G; ++j) {
          {
            std::unique_lock<std::mutex> lk(issue_mu);
            issue_cv.wait(lk, [&]() {
              return issued.load(std::memory_order_acquire) > j ||
                     abort_widen.load(std::memory_order_relaxed);
            });
          }
          if (abort_widen.load(std::memory_order_relaxed)) return;
          if (!blk_on[j]) continue;
          if (cudaEventSynchronize(ev_ci[j]) != cudaSuccess) return;
          const uint64_t n = blk_n[j];
          const uint64_t i0 = blk_off[j] + n * uint64_t(w) / uint64_t(nthreads);
          const uint64_t i1 = blk_off[j] + n * uint64_t(w + 1) / uint64_t(nthreads);
          if (blk_16[j])
            widen16(h_d16, h_base + blk_cb[j], blk_off[j] >> 6, out_ci, i0, i1);
          else
            widen(h_ci32 + i0, out_ci + i0, i1 - i0);
          const uint64_t nr = blk_r1[j] - blk_r0[j] + 1;  // row pointers r0..r1
          const uint64_t q0 = blk_r0[j] + nr * uint64_t(w) / uint64_t(nthreads);
          const uint64_t q1 = blk_r0[j] + nr * uint64_t(w + 1) / uint64_t(nthreads);
          widen(h_rp32 + q0, out_rp + q0, q1 - q0);
        }
      });
    }
  }
  auto stop_workers = [&]() {
    abort_widen.store(true);
    publish(G + 1);
    for (auto& t : workers) t.join();
    workers.clear();
    // the copy engines may still be writing into the staging blocks: drain
    // both copy streams before they go back to the pool (another thread may
    // be handed them by spmmm_host_alloc at once)
    cudaStreamSynchronize(c->s_down);
    cudaStreamSynchronize(c->s_up);
    if (hci32) host_free_internal(hci32);
    if (hrp32) host_free_internal(hrp32);
    if (hd16) host_free_internal(hd16);
    if (hbase) host_free_internal(hbase);
    hci32 = hrp32 = hd16 = hbase = nullptr;
  };
  spmmm_product* prods[kMaxPipeBlocks] = {};
  auto release_all = [&]() {
    for (int j = 0; j < G; ++j)
      if (prods[j]) {
        product_release(c, prods[j]);
        delete prods[j];
        prods[j] = nullptr;
      }
  };
  // every early return below (CUDA_TRY included) stops the workers, drains the
  // streams and returns the blocks and the result arrays
  struct Guard {
    std::function<void()> f;
    ~Guard() {
      if (f) f();
    }
  } guard{[&]() {
    stop_workers();
    drain(0);
    release_all();
    free_out();
  }};
  uint64_t off = 0, mults = 0;
  bool overflow = false;
  for (int j = 0; j < G; ++j) {
    const uint64_t r0 = bound[j], r1 = bound[j + 1];
    if (r1 == r0) continue;
    int u = j;  // the last A block this block needs resident
    rc = wait_upload(j + 2);
    if (rc) return rc;  // (the guard cleans up)
    if (same && a->rows) {
      CUDA_TRY(cudaEventSynchronize(ev_maxc[j]));
      const uint64_t row = c->h_aux[j];  // rows [0, row] of B = A (row_ptr to row + 1)
      const int uu = int(std::upper_bound(bound, bound + G + 1, row) - bound) - 1;
      u = std::min(std::max(uu, j), G - 1);
    }
    rc = wait_upload(u + 2);
    if (rc) return rc;
    CUDA_TRY(cudaStreamWaitEvent(c->stream, ev_av[u], 0));
    if (!same) CUDA_TRY(cudaStreamWaitEvent(c->stream, *ev_bv, 0));
    spmmm_csr va{r1 - r0, a->cols, a->nnz, d_arp + r0, d_aci, d_av, SPMMM_MEM_DEVICE, 0};
    spmmm_csr vb{B.rows, B.cols, B.nnz, B.rp, B.ci, B.v, SPMMM_MEM_DEVICE, 0};
    static const bool cf_blocks = std::getenv("SPMMM_PIPE_COUNT_FREE") != nullptr;
    rc = multiply_impl(c, &va, &vb, strategy,
                       (flags & SPMMM_FLAG_TIMING) | (cf_blocks ? 0u : kFlagCounted), &prods[j]);
    if (rc) return rc;  // (the guard cleans up)
    spmmm_product* p = prods[j];
    if (off + p->nnz > cap) {
      overflow = true;
      break;
    }
    if (off) {
      k_add_offset<<<std::max<unsigned>(1, unsigned(std::min<uint64_t>((r1 - r0 + 256) / 256, 1024))),
                     256, 0, c->stream>>>(p->rp, r1 - r0 + 1, off);
      CUDA_TRY(cudaGetLastError());
    }
    if (narrow) {
      // row pointers and columns go down as u32 (the reservation is < 2^32
      // entries), widened by the workers once ev_ci[j] has fired
      k_narrow<<<std::max(1u, std::min<unsigned>(unsigned((r1 - r0 + 256) / 256),
                                                  unsigned(c->sms) * 8)),
                 256, 0, c->stream>>>(p->rp, d_rp32 + r0, r1 - r0 + 1);
      CUDA_TRY(cudaGetLastError());
      const uint64_t nch = p->nnz ? ((off + p->nnz + 63) >> 6) - (off >> 6) : 0;
      bool use16 = false;
      if (p->nnz && !no_delta) {
        // u16 deltas if every 64-entry chunk spans < 2^16 columns (stencils)
        volatile unsigned long long* okw = c->h_aux + kMaxPipeBlocks + j;
        *okw = 1;
        k_delta16<<<std::max(1u, std::min<unsigned>(unsigned((nch + 7) / 8),
                                                     unsigned(c->sms) * 8)),
                    256, 0, c->stream>>>(p->ci, off, p->nnz, d_base + cb_next, d_d16,
                                         reinterpret_cast<unsigned int*>(
                                             const_cast<unsigned long long*>(okw)));
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        use16 = (*okw & 0xffffffffull) != 0;
      }
      if (p->nnz && !use16) {
        k_narrow<<<std::min<unsigned>(unsigned((p->nnz + 255) / 256), unsigned(c->sms) * 8), 256,
                   0, c->stream>>>(p->ci, d_ci32 + off, p->nnz);
        CUDA_TRY(cudaGetLastError());
      }
      CUDA_TRY(cudaEventRecord(ev_comp[j], c->stream));
      CUDA_TRY(cudaStreamWaitEvent(c->s_down, ev_comp[j], 0));
      CUDA_TRY(cudaMemcpyAsync(h_rp32 + r0, d_rp32 + r0, (r1 - r0 + 1) * 4,
                               cudaMemcpyDeviceToHost, c->s_down));
      d2h += (r1 - r0 + 1) * 4 + p->nnz * 8;
      if (use16) {
        CUDA_TRY(cudaMemcpyAsync(h_base + cb_next, d_base + cb_next, nch * 4,
                                 cudaMemcpyDeviceToHost, c->s_down));
        CUDA_TRY(cudaMemcpyAsync(h_d16 + off, d_d16 + off, p->nnz * 2, cudaMemcpyDeviceToHost,
                                 c->s_down));
        d2h += nch * 4 + p->nnz * 2;
      } else if (p->nnz) {
        CUDA_TRY(cudaMemcpyAsync(h_ci32 + off, d_ci32 + off, p->nnz * 4, cudaMemcpyDeviceToHost,
                                 c->s_down));
        d2h += p->nnz * 4;
      }
      blk_16[j] = use16;
      blk_cb[j] = cb_next;
      if (use16) cb_next += nch;
      CUDA_TRY(cudaEventRecord(ev_ci[j], c->s_down));
      if (p->nnz)
        CUDA_TRY(cudaMemcpyAsync(out_v + off, p->v, p->nnz * 8, cudaMemcpyDeviceToHost,
                                 c->s_down));
    } else {
      CUDA_TRY(cudaEventRecord(ev_comp[j], c->stream));
      CUDA_TRY(cudaStreamWaitEvent(c->s_down, ev_comp[j], 0));
      CUDA_TRY(cudaMemcpyAsync(out_rp + r0, p->rp, (r1 - r0 + 1) * 8, cudaMemcpyDeviceToHost,
                               c->s_down));
      if (p->nnz) {
        CUDA_TRY(cudaMemcpyAsync(out_ci + off, p->ci, p->nnz * 8, cudaMemcpyDeviceToHost,
                                 c->s_down));
        CUDA_TRY(cudaMemcpyAsync(out_v + off, p->v, p->nnz * 8, cudaMemcpyDeviceToHost,
                                 c->s_down));
      }
    }
    CUDA_TRY(cudaEventRecord(ev_down[j], c->s_down));  // (arrays live until the end)
    if (tr.on) {
      cudaEventRecord(tl[1 + kMaxPipeBlocks + j], c->stream);
      cudaEventRecord(tl[1 + 2 * kMaxPipeBlocks + j], c->s_down);
    }
    blk_off[j] = off;
    blk_n[j] = p->nnz;
    blk_r0[j] = r0;
    blk_r1[j] = r1;
    blk_on[j] = narrow;
    publish(j + 1);
    off += p->nnz;
    mults += p->mults;
    tr.mark("pipe: block computed, download issued");
  }
  if (overflow) {
    // the reservation was too small: one product over the resident operands
    // into exact-size arrays (the operands are all up once s_up drains)
    stop_workers();
    if (uploader.joinable()) uploader.join();  // every upload issued (no abort)
    if (up_error.load()) return fail(up_error.load(), "%s", up_msg.c_str());
    CUDA_TRY(cudaStreamSynchronize(c->s_down));
    CUDA_TRY(cudaStreamSynchronize(c->s_up));
    release_all();
    free_out();
    guard.f = nullptr;
    tr.mark("pipe: reservation overflowed, one-shot product");
    spmmm_csr va{a->rows, a->cols, a->nnz, d_arp, d_aci, d_av, SPMMM_MEM_DEVICE, 0};
    spmmm_csr vb{B.rows, B.cols, B.nnz, B.rp, B.ci, B.v, SPMMM_MEM_DEVICE, 0};
    spmmm_product* p = nullptr;
    rc = multiply_impl(c, &va, &vb, strategy, flags & SPMMM_FLAG_TIMING, &p);
    if (rc) return rc;
    rc = host_alloc_internal(rpb, &hrp);
    if (!rc) rc = host_alloc_internal(std::max<uint64_t>(p->nnz, 1) * 8, &hci);
    if (!rc) rc = host_alloc_internal(std::max<uint64_t>(p->nnz, 1) * 8, &hv);
    cudaError_t e = rc ? cudaSuccess : cudaMemcpyAsync(hrp, p->rp, rpb, cudaMemcpyDeviceToHost,
                                                       c->stream);
    if (!rc && e == cudaSuccess && p->nnz)
      e = cudaMemcpyAsync(hci, p->ci, p->nnz * 8, cudaMemcpyDeviceToHost, c->stream);
    if (!rc && e == cudaSuccess && p->nnz)
      e = cudaMemcpyAsync(hv, p->v, p->nnz * 8, cudaMemcpyDeviceToHost, c->stream);
    if (!rc && e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    const uint64_t nnz = p->nnz, m = p->mults;
    product_release(c, p);
    delete p;
    if (!rc && e != cudaSuccess) rc = fail(SPMMM_ERR_CUDA, "%s", cudaGetErrorString(e));
    if (rc) {
      free_out();
      return rc;
    }
    out->rows = a->rows;
    out->cols = b->cols;
    out->nnz = nnz;
    out->mults = m;
    out->row_ptr = static_cast<uint64_t*>(hrp);
    out->col_idx = static_cast<uint64_t*>(hci);
    out->values = static_cast<double*>(hv);
    out->h2d_bytes = rpb + a->nnz * 16 + (same ? 0 : (b->rows + 1) * 8 + b->nnz * 16);
    out->d2h_bytes = rpb + nnz * 16;
    return SPMMM_OK;
  }
  publish(G);  // (skipped empty blocks)
  if (tr.on) {
    cudaStreamSynchronize(c->s_down);
    tr.mark("pipe: downloads done (trace only: waits before joining)");
  }
  for (auto& t : workers) t.join();
  if (uploader.joinable()) uploader.join();  // (its last step was waited for above)
  tr.mark("pipe: widening done");
  workers.clear();
  if (hci32) host_free_internal(hci32);
  hci32 = nullptr;
  CUDA_TRY(cudaStreamSynchronize(c->s_down));
  CUDA_TRY(cudaStreamSynchronize(c->s_up));
  tr.mark("pipe: downloads done");
  if (tr.on) {
    cudaDeviceSynchronize();
    for (int j = 0; j < G; ++j) {
      float up = 0, comp = 0, down = 0;
      cudaEventElapsedTime(&up, tl[0], tl[1 + j]);
      cudaEventElapsedTime(&comp, tl[0], tl[1 + kMaxPipeBlocks + j]);
      cudaEventElapsedTime(&down, tl[0], tl[1 + 2 * kMaxPipeBlocks + j]);
      std::fprintf(stderr, "[spmmm] block %2d: uploaded %7.3f ms, computed %7.3f ms, downloaded %7.3f ms\n",
                   j, up, comp, down);
    }
    for (cudaEvent_t ev : tl) cudaEventDestroy(ev);
  }
  guard.f = nullptr;  // success: the result arrays are the caller's
  for (void* hp : {hrp32, hd16, hbase}) host_free_internal(hp);
  hrp32 = hd16 = hbase = nullptr;
  release_all();
  out->rows = a->rows;
  out->cols = b->cols;
  out->nnz = off;
  out->mults = mults;
  out->h2d_bytes = rpb + a->nnz * 16 + (same ? 0 : (b->rows + 1) * 8 + b->nnz * 16);
  out->d2h_bytes = narrow ? d2h : rpb + off * 16;
  out->row_ptr = out_rp;
  out->col_idx = out_ci;
  out->values = out_v;
  return SPMMM_OK;
}
}  // namespace

// =============================================================================
// C ABI
// =============================================================================
extern "C" {

int spmmm_abi_version(void) { return SPMMM_ABI_VERSION; }

const char* spmmm_last_error(void) { return g_error.c_str(); }

int spmmm_device_count(int* count) {
  if (!count) return fail(SPMMM_ERR_INVALID, "count is NULL");
  *count = 0;
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    return fail(SPMMM_ERR_CUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  }
  return SPMMM_OK;
}

int spmmm_context_create(int device, void* cuda_stream, spmmm_context** out) {
  if (!out) return fail(SPMMM_ERR_INVALID, "out is NULL");
  *out = nullptr;
  int n = 0;
  CUDA_TRY(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n)
    return fail(SPMMM_ERR_INVALID, "device %d out of range (%d devices)", device, n);
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    return fail(SPMMM_ERR_UNSUPPORTED, "device %d is sm_%d%d; libspmmm is built for sm_100a",
                device, prop.major, prop.minor);
  if (!prop.cooperativeLaunch)
    return fail(SPMMM_ERR_UNSUPPORTED, "device %d lacks cooperative launch", device);
  auto* c = new (std::nothrow) spmmm_context;
  if (!c) return fail(SPMMM_ERR_OOM, "host allocation failed");
  c->device = device;
  c->sms = prop.multiProcessorCount;
  // product cache: a quarter of the device's memory unless
  // SPMMM_DEVICE_CACHE_BYTES says otherwise
  const char* dcl = std::getenv("SPMMM_DEVICE_CACHE_BYTES");
  c->cache_limit = dcl ? size_t(std::strtoull(dcl, nullptr, 10)) : size_t(prop.totalGlobalMem / 4);
  // keep freed blocks in the pool: repeated products reuse their memory
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaError_t e = cudaSuccess;
  if (cuda_stream) {
    c->stream = static_cast<cudaStream_t>(cuda_stream);
  } else {
    e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    c->own_stream = true;
  }
  if (e == cudaSuccess) e = cudaMallocHost(&c->h_ctrl, kCtrlWords * sizeof(unsigned long long));
  for (int k = 0; k < 2 * kNumKernels && e == cudaSuccess; ++k) e = cudaEventCreate(&c->ev[k]);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_count, cudaEventDisableTiming);
  if (e == cudaSuccess) e = ensure(c->ctrl, kCtrlWords * sizeof(unsigned long long), c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    delete c;
    return fail(SPMMM_ERR_CUDA, "context_create: %s", cudaGetErrorString(e));
  }
  *out = c;
  return SPMMM_OK;
}

int spmmm_context_destroy(spmmm_context* c) {
  if (!c) return SPMMM_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (DevBuf* b : {&c->ctrl, &c->prod, &c->lmap, &c->list, &c->status, &c->l_off, &c->l_nnz,
                    &c->ws, &c->gtab, &c->sub, &c->dom, &c->ell, &c->tr_scratch, &c->stage_ci, &c->stage_v, &c->a_rp, &c->a_ci,
                    &c->a_v, &c->b_rp, &c->b_ci, &c->b_v, &c->parts, &c->part_off, &c->part_nnz,
                    &c->row_parts, &c->scr_col, &c->scr_val, &c->aux, &c->ci32, &c->rp32, &c->d16, &c->dbase,
                    &c->part_sums, &c->dl_rp})
    release(*b, c->stream);
  for (auto& cb : c->cache) cudaFreeAsync(cb.first, c->stream);
  c->cache.clear();
  cudaStreamSynchronize(c->stream);
  for (int k = 0; k < 2 * kNumKernels; ++k)
    if (c->ev[k]) cudaEventDestroy(c->ev[k]);
  if (c->ev_count) cudaEventDestroy(c->ev_count);
  for (cudaEvent_t ev : c->pev)
    if (ev) cudaEventDestroy(ev);
  if (c->s_up) cudaStreamDestroy(c->s_up);
  if (c->s_aux) cudaStreamDestroy(c->s_aux);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->s_down) cudaStreamDestroy(c->s_down);
  if (c->h_aux) cudaFreeHost(c->h_aux);
  if (c->h_part) cudaFreeHost(c->h_part);
  delete c->stager;
  if (c->h_ctrl) cudaFreeHost(c->h_ctrl);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
  return SPMMM_OK;
}

int spmmm_synchronize(spmmm_context* c) {
  if (!c) return fail(SPMMM_ERR_INVALID, "context is NULL");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return SPMMM_OK;
}

int spmmm_multiply(spmmm_context* c, const spmmm_csr* a, const spmmm_csr* b, int strategy,
                   uint32_t flags, spmmm_product** out) {
  if (!c) return fail(SPMMM_ERR_INVALID, "context is NULL");
  std::lock_guard<std::mutex> lock(c->mu);
  return multiply_impl(c, a, b, strategy, flags & (SPMMM_FLAG_ROW_STATS | SPMMM_FLAG_TIMING), out);
}

int spmmm_multiply_host(spmmm_context* c, const spmmm_csr* a, const spmmm_csr* b, int strategy,
                        uint32_t flags, int blocks, spmmm_host_csr* out) {
  if (!c) return fail(SPMMM_ERR_INVALID, "context is NULL");
  std::lock_guard<std::mutex> lock(c->mu);
  return multiply_host_impl(c, a, b, strategy, flags, blocks, out);
}

int spmmm_product_shape(const spmmm_product* p, uint64_t* rows, uint64_t* cols, uint64_t* nnz,
                        uint64_t* mults) {
  if (!p) return fail(SPMMM_ERR_INVALID, "product is NULL");
  if (rows) *rows = p->rows;
  if (cols) *cols = p->cols;
  if (nnz) *nnz = p->nnz;
  if (mults) *mults = p->mults;
  return SPMMM_OK;
}

int spmmm_row_classes(uint32_t out[5]) {
  if (!out) return fail(SPMMM_ERR_INVALID, "NULL argument");
  out[0] = kEscWarpLimit;
  out[1] = kHugeMin;
  out[2] = kDomRCap;
  out[3] = kDomMinRun;
#ifdef SPMMM_DOM_HALF
  out[4] = 1;
#else
  out[4] = 0;
#endif
  return SPMMM_OK;
}

int spmmm_product_reserved_bytes(const spmmm_product* p, uint64_t* bytes) {
  if (!p || !bytes) return fail(SPMMM_ERR_INVALID, "NULL argument");
  *bytes = p->cap[0] + p->cap[1] + p->cap[2] + p->cap[3];
  return SPMMM_OK;
}

int spmmm_product_device_arrays(const spmmm_product* p, const uint64_t** rp, const uint64_t** ci,
                                const double** v) {
  if (!p) return fail(SPMMM_ERR_INVALID, "product is NULL");
  if (rp) *rp = p->rp;
  if (ci) *ci = p->ci;
  if (v) *v = p->v;
  return SPMMM_OK;
}

int spmmm_product_download(spmmm_product* p, uint64_t* rp, uint64_t* ci, double* v) {
  if (!p) return fail(SPMMM_ERR_INVALID, "product is NULL");
  spmmm_context* c = p->ctx;
  std::lock_guard<std::mutex> lock(c->mu);
  CUDA_TRY(cudaSetDevice(c->device));
  if (rp) CUDA_TRY(cudaMemcpyAsync(rp, p->rp, (p->rows + 1) * 8, cudaMemcpyDeviceToHost, c->stream));
  if (p->nnz) {
    if (ci) CUDA_TRY(cudaMemcpyAsync(ci, p->ci, p->nnz * 8, cudaMemcpyDeviceToHost, c->stream));
    if (v) CUDA_TRY(cudaMemcpyAsync(v, p->v, p->nnz * 8, cudaMemcpyDeviceToHost, c->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return SPMMM_OK;
}

int spmmm_product_copy_device(spmmm_product* p, uint64_t* rp, uint64_t* ci, double* v) {
  if (!p) return fail(SPMMM_ERR_INVALID, "product is NULL");
  spmmm_context* c = p->ctx;
  std::lock_guard<std::mutex> lock(c->mu);
  CUDA_TRY(cudaSetDevice(c->device));
  if (rp) CUDA_TRY(cudaMemcpyAsync(rp, p->rp, (p->rows + 1) * 8, cudaMemcpyDeviceToDevice, c->stream));
  if (p->nnz) {
    if (ci) CUDA_TRY(cudaMemcpyAsync(ci, p->ci, p->nnz * 8, cudaMemcpyDeviceToDevice, c->stream));
    if (v) CUDA_TRY(cudaMemcpyAsync(v, p->v, p->nnz * 8, cudaMemcpyDeviceToDevice, c->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return SPMMM_OK;
}

int spmmm_product_row_stats(spmmm_product* p, uint64_t* mn, uint64_t* mx, uint64_t* touched) {
  if (!p) return fail(SPMMM_ERR_INVALID, "product is NULL");
  if (!p->st) return fail(SPMMM_ERR_INVALID, "product was computed without SPMMM_FLAG_ROW_STATS");
  spmmm_context* c = p->ctx;
  std::lock_guard<std::mutex> lock(c->mu);
  std::vector<uint32_t> h(size_t(p->rows) * 3);
  CUDA_TRY(cudaSetDevice(c->device));
  if (p->rows) {
    CUDA_TRY(cudaMemcpyAsync(h.data(), p->st, h.size() * 4, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  for (uint64_t r = 0; r < p->rows; ++r) {
    const uint32_t lo = h[r], hi = h[p->rows + r], t = h[2 * p->rows + r];
    const bool none = t == 0;
    if (mn) mn[r] = none ? ~0ull : lo;
    if (mx) mx[r] = none ? 0ull : hi;
    if (touched) touched[r] = t;
  }
  return SPMMM_OK;
}

int spmmm_product_destroy(spmmm_product* p) {
  if (!p) return SPMMM_OK;
  spmmm_context* c = p->ctx;
  std::lock_guard<std::mutex> lock(c->mu);
  cudaSetDevice(c->device);
  product_release(c, p);
  delete p;
  return SPMMM_OK;
}

int spmmm_estimate_nnz(spmmm_context* c, const spmmm_csr* a, const spmmm_csr* b, uint64_t* out) {
  if (!c || !out) return fail(SPMMM_ERR_INVALID, "NULL argument");
  std::lock_guard<std::mutex> lock(c->mu);
  int rc = check_view(a, "a");
  if (!rc) rc = check_view(b, "b");
  if (rc) return rc;
  if (a->cols != b->rows)
    return fail(SPMMM_ERR_DIMENSION, "dimension mismatch: %llu (cols of a) != %llu (rows of b)",
                (unsigned long long)a->cols, (unsigned long long)b->rows);
  CUDA_TRY(cudaSetDevice(c->device));
  DevCsr A, B;
  rc = resolve(c, a, b, &A, &B);
  if (rc) return rc;
  Timer tm{c, false};
  c->last_launches = 0;
  rc = run_count(c, A, B, tm);
  if (rc) return rc;
  *out = c->h_ctrl[kCtrlTotal];
  return SPMMM_OK;
}

int spmmm_transpose(spmmm_context* c, const spmmm_csr* m, spmmm_product** out) {
  if (!c || !out) return fail(SPMMM_ERR_INVALID, "NULL argument");
  *out = nullptr;
  std::lock_guard<std::mutex> lock(c->mu);
  int rc = check_view(m, "m");
  if (rc) return rc;
  if (m->rows >= 0xffffffffull || m->cols >= 0xffffffffull)
    return fail(SPMMM_ERR_UNSUPPORTED, "conversion needs rows and cols < 2^32 - 1");
  CUDA_TRY(cudaSetDevice(c->device));
  c->last_launches = 0;
  DevCsr M;
  uint64_t base = 0, end = 0;
  if (m->memory == SPMMM_MEM_DEVICE) {
    M = DevCsr{m->row_ptr, m->col_idx, m->values, m->rows, m->cols, m->nnz};
    CUDA_TRY(cudaMemcpyAsync(c->h_ctrl, m->row_ptr, sizeof(uint64_t), cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->h_ctrl + 1, m->row_ptr + m->rows, sizeof(uint64_t),
                             cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    base = c->h_ctrl[0];
    end = c->h_ctrl[1];
  } else {
    base = m->row_ptr[0];
    end = m->row_ptr[m->rows];
    if (base != 0) return fail(SPMMM_ERR_INVALID, "host row_ptr must start at 0");
    rc = upload(c, m, c->a_rp, c->a_ci, c->a_v, &M);
    if (rc) return rc;
  }
  if (end < base || end > m->nnz)
    return fail(SPMMM_ERR_INVALID, "malformed row_ptr (row_ptr[rows] < row_ptr[0] or past nnz)");
  const uint64_t n = end - base;
  if (n >= 0xffffffffull) return fail(SPMMM_ERR_UNSUPPORTED, "conversion needs nnz < 2^32 - 1");
  auto* p = new (std::nothrow) spmmm_product;
  if (!p) return fail(SPMMM_ERR_OOM, "host allocation failed");
  p->ctx = c;
  p->rows = m->cols;
  p->cols = m->rows;
  p->nnz = n;
  p->mults = 0;
  cudaError_t e = cache_alloc(c, (p->rows + 1) * 8, reinterpret_cast<void**>(&p->rp), &p->cap[0]);
  if (e == cudaSuccess)
    e = cache_alloc(c, std::max<uint64_t>(n, 1) * 8, reinterpret_cast<void**>(&p->ci), &p->cap[1]);
  if (e == cudaSuccess)
    e = cache_alloc(c, std::max<uint64_t>(n, 1) * 8, reinterpret_cast<void**>(&p->v), &p->cap[2]);
  const size_t sb = transpose_scratch_bytes(n, m->cols);
  if (e == cudaSuccess) e = ensure(c->tr_scratch, sb, c->stream);
  if (e == cudaSuccess)
    e = cudaMemsetAsync(c->ctrl.p, 0, kCtrlWords * sizeof(unsigned long long), c->stream);
  c->ctrl_clean = false;
  unsigned long long* err = static_cast<unsigned long long*>(c->ctrl.p) + kCtrlError;
  if (e == cudaSuccess)
    e = transpose_csr(M, base, n, p->rp, p->ci, p->v, c->tr_scratch.p, c->tr_scratch.cap, err,
                      c->sms, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(c->h_ctrl + kCtrlError, err, sizeof(uint64_t), cudaMemcpyDeviceToHost,
                        c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    product_release(c, p);
    delete p;
    return fail(e == cudaErrorMemoryAllocation ? SPMMM_ERR_OOM : SPMMM_ERR_CUDA, "transpose: %s",
                cudaGetErrorString(e));
  }
  const unsigned long long f = c->h_ctrl[kCtrlError];
  if (f) {
    product_release(c, p);
    delete p;
    return fail(SPMMM_ERR_INVALID, (f & 2) ? "malformed row_ptr" : "col_idx entry >= cols");
  }
  c->last_launches = 4;
  *out = p;
  return SPMMM_OK;
}

int spmmm_row_products_prefix(spmmm_context* c, const spmmm_csr* a, const spmmm_csr* b,
                              uint64_t* out) {
  if (!c || !out) return fail(SPMMM_ERR_INVALID, "NULL argument");
  std::lock_guard<std::mutex> lock(c->mu);
  int rc = check_view(a, "a");
  if (!rc) rc = check_view(b, "b");
  if (rc) return rc;
  if (a->cols != b->rows)
    return fail(SPMMM_ERR_DIMENSION, "dimension mismatch: %llu (cols of a) != %llu (rows of b)",
                (unsigned long long)a->cols, (unsigned long long)b->rows);
  CUDA_TRY(cudaSetDevice(c->device));
  DevCsr A, B;
  rc = resolve(c, a, b, &A, &B);
  if (rc) return rc;
  Timer tm{c, false};
  c->last_launches = 0;
  rc = run_count(c, A, B, tm);
  if (rc) return rc;
  std::vector<uint32_t> h(A.rows);
  if (A.rows) {
    CUDA_TRY(cudaMemcpyAsync(h.data(), c->prod.p, A.rows * 4, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  out[0] = 0;
  for (uint64_t r = 0; r < A.rows; ++r) out[r + 1] = out[r] + h[r];
  return SPMMM_OK;
}

int spmmm_partition_rows(spmmm_context* c, const spmmm_csr* a, const spmmm_csr* b, int parts,
                         uint64_t* bounds, uint64_t* total) {
  if (!c || !bounds) return fail(SPMMM_ERR_INVALID, "NULL argument");
  if (parts < 1 || parts > kPartMaxParts)
    return fail(SPMMM_ERR_INVALID, "parts=%d outside [1, %d]", parts, kPartMaxParts);
  std::lock_guard<std::mutex> lock(c->mu);
  int rc = check_view(a, "a");
  if (!rc) rc = check_view(b, "b");
  if (rc) return rc;
  if (a->cols != b->rows)
    return fail(SPMMM_ERR_DIMENSION, "dimension mismatch: %llu (cols of a) != %llu (rows of b)",
                (unsigned long long)a->cols, (unsigned long long)b->rows);
  if (a->rows >= 0xffffffffull)
    return fail(SPMMM_ERR_UNSUPPORTED, "a.rows=%llu exceeds the 32-bit row range",
                (unsigned long long)a->rows);
  CUDA_TRY(cudaSetDevice(c->device));
  DevCsr A, B;
  rc = resolve(c, a, b, &A, &B);
  if (rc) return rc;
  Timer tm{c, false};
  c->last_launches = 0;
  rc = run_count(c, A, B, tm);  // validates A and B, per-row products in c->prod
  if (rc) return rc;
  if (!c->h_part) CUDA_TRY(cudaMallocHost(&c->h_part, (kPartMaxParts + 2) * 8));
  const uint64_t rows = A.rows;
  if (rows == 0) {
    for (int g = 0; g <= parts; ++g) bounds[g] = 0;
    if (total) *total = 0;
    return SPMMM_OK;
  }
  uint64_t L = kPartChunkRows;
  while ((rows + L - 1) / L > uint64_t(kPartMaxChunks)) L *= 2;
  const uint32_t nchunks = uint32_t((rows + L - 1) / L);
  CUDA_TRY(ensure(c->part_sums, nchunks * 8, c->stream));
  auto* sums = static_cast<unsigned long long*>(c->part_sums.p);
  k_part_chunk_sums<<<nchunks, 256, 0, c->stream>>>(static_cast<const uint32_t*>(c->prod.p), rows,
                                                     uint32_t(L), sums);
  CUDA_TRY(cudaGetLastError());
  k_partition<<<1, 1024, 0, c->stream>>>(static_cast<const uint32_t*>(c->prod.p), rows,
                                         uint32_t(L), sums, nchunks, parts, c->h_part);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->last_launches += 2;
  uint64_t prev = 0;
  for (int g = 0; g <= parts; ++g) {
    uint64_t v = std::min<uint64_t>(c->h_part[g], rows);
    prev = std::max(prev, v);
    bounds[g] = prev;
  }
  bounds[0] = 0;
  bounds[parts] = rows;
  if (total) *total = c->h_part[parts + 1];
  return SPMMM_OK;
}

int spmmm_product_download_offset(spmmm_product* p, uint64_t offset, uint64_t* rp, uint64_t* ci,
                                  double* v) {
  if (!p) return fail(SPMMM_ERR_INVALID, "product is NULL");
  spmmm_context* c = p->ctx;
  std::lock_guard<std::mutex> lock(c->mu);
  CUDA_TRY(cudaSetDevice(c->device));
  if (rp) {
    const uint64_t n = p->rows + 1;
    const uint64_t* src = p->rp;
    if (offset) {
      CUDA_TRY(ensure(c->dl_rp, n * 8, c->stream));
      k_copy_offset<<<unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(c->sms) * 8)), 256, 0,
                      c->stream>>>(p->rp, static_cast<uint64_t*>(c->dl_rp.p), n, offset);
      CUDA_TRY(cudaGetLastError());
      src = static_cast<const uint64_t*>(c->dl_rp.p);
    }
    CUDA_TRY(cudaMemcpyAsync(rp, src, n * 8, cudaMemcpyDeviceToHost, c->stream));
  }
  if (p->nnz) {
    if (ci) CUDA_TRY(cudaMemcpyAsync(ci, p->ci, p->nnz * 8, cudaMemcpyDeviceToHost, c->stream));
    if (v) CUDA_TRY(cudaMemcpyAsync(v, p->v, p->nnz * 8, cudaMemcpyDeviceToHost, c->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return SPMMM_OK;
}

int spmmm_host_register(void* ptr, uint64_t bytes) {
  if (!ptr || !bytes) return fail(SPMMM_ERR_INVALID, "NULL or empty range");
  CUDA_TRY(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable));
  return SPMMM_OK;
}

int spmmm_host_unregister(void* ptr) {
  if (!ptr) return fail(SPMMM_ERR_INVALID, "ptr is NULL");
  CUDA_TRY(cudaHostUnregister(ptr));
  return SPMMM_OK;
}

int spmmm_last_timings(spmmm_context* c, const char** names, double* ms, int cap, int* count) {
  if (!c || !count) return fail(SPMMM_ERR_INVALID, "NULL argument");
  int n = 0;
  for (int k = 0; k < kNumKernels; ++k) {
    if (!c->ev_used[k]) continue;
    if (n < cap) {
      if (names) names[n] = kKernelNames[k];
      if (ms) ms[n] = c->last_ms[k];
    }
    ++n;
  }
  *count = n;
  return SPMMM_OK;
}

int spmmm_last_launch_count(spmmm_context* c, int* count) {
  if (!c || !count) return fail(SPMMM_ERR_INVALID, "NULL argument");
  *count = c->last_launches;
  return SPMMM_OK;
}

}  // extern "C"

// =============================================================================
// Pinned host pool (process-wide): size-bucketed free lists of cudaHostAlloc
// blocks. Pinning is expensive (page locking), so blocks are recycled.
// =============================================================================
namespace {

struct HostPool {
  std::mutex mu;
  std::multimap<uint64_t, void*> free_blocks;  // capacity -> block
  std::map<void*, uint64_t> live;              // block -> capacity
  uint64_t in_use = 0, cached = 0;
  // page-locked bytes kept for reuse: an eighth of the host's memory unless
  // SPMMM_HOST_CACHE_BYTES says otherwise
  uint64_t cache_limit = 0;
  HostPool() {
    const char* e = std::getenv("SPMMM_HOST_CACHE_BYTES");
    const long pages = sysconf(_SC_PHYS_PAGES), page = sysconf(_SC_PAGESIZE);
    cache_limit = e ? std::strtoull(e, nullptr, 10)
                    : (pages > 0 && page > 0 ? uint64_t(pages) * uint64_t(page) / 8 : 8ull << 30);
  }

  static uint64_t bucket(uint64_t bytes) {
    // round up to 1/8 steps of the next power of two to bound waste
    if (bytes <= 4096) return 4096;
    uint64_t p = 1;
    while (p < bytes) p <<= 1;
    const uint64_t step = p / 8;
    return (bytes + step - 1) / step * step;
  }
};

HostPool& host_pool() {
  static HostPool* pool = new HostPool;  // leaked on purpose: lives until exit
  return *pool;
}

}  // namespace

extern "C" {

int spmmm_host_alloc(uint64_t bytes, void** ptr) {
  if (!ptr) return fail(SPMMM_ERR_INVALID, "ptr is NULL");
  HostPool& hp = host_pool();
  const uint64_t cap = HostPool::bucket(bytes ? bytes : 1);
  {
    std::lock_guard<std::mutex> lock(hp.mu);
    auto it = hp.free_blocks.lower_bound(cap);
    if (it != hp.free_blocks.end() && it->first <= cap + cap / 4) {
      *ptr = it->second;
      hp.live[it->second] = it->first;
      hp.cached -= it->first;
      hp.in_use += it->first;
      hp.free_blocks.erase(it);
      return SPMMM_OK;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaHostAlloc(&p, cap, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    // release the cache and retry once
    std::lock_guard<std::mutex> lock(hp.mu);
    for (auto& kv : hp.free_blocks) cudaFreeHost(kv.second);
    hp.free_blocks.clear();
    hp.cached = 0;
    e = cudaHostAlloc(&p, cap, cudaHostAllocPortable);
    if (e != cudaSuccess)
      return fail(SPMMM_ERR_OOM, "cudaHostAlloc(%llu): %s", (unsigned long long)cap,
                  cudaGetErrorString(e));
  }
  std::lock_guard<std::mutex> lock(hp.mu);
  hp.live[p] = cap;
  hp.in_use += cap;
  *ptr = p;
  return SPMMM_OK;
}

int spmmm_host_free(void* ptr) {
  if (!ptr) return SPMMM_OK;
  HostPool& hp = host_pool();
  std::lock_guard<std::mutex> lock(hp.mu);
  auto it = hp.live.find(ptr);
  if (it == hp.live.end()) return fail(SPMMM_ERR_INVALID, "pointer not from spmmm_host_alloc");
  const uint64_t cap = it->second;
  hp.live.erase(it);
  hp.in_use -= cap;
  if (hp.cached + cap > hp.cache_limit) {
    cudaFreeHost(ptr);
  } else {
    hp.free_blocks.emplace(cap, ptr);
    hp.cached += cap;
  }
  return SPMMM_OK;
}

int spmmm_host_pool_bytes(uint64_t* in_use, uint64_t* cached) {
  HostPool& hp = host_pool();
  std::lock_guard<std::mutex> lock(hp.mu);
  if (in_use) *in_use = hp.in_use;
  if (cached) *cached = hp.cached;
  return SPMMM_OK;
}

}  // extern "C"
