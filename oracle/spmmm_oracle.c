/*
 * spmmm_oracle.c — CPU restatement of the reference spMMM hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the parity checker for the CUDA
 * library and the CPU baseline arm of bench.py. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it. The product path (paper_1303_1651_b200) never links or calls it.
 *
 * What it restates (reference = /root/reference/pkg/src/sparsemm):
 *   oracle_estimate_nnz       formats.py:276-289  (Σ over A nonzeros of rownnz_B)
 *   oracle_count_mults        perfmodel.py:63-76  (same number, per-entry loop)
 *   oracle_multiply_rowmajor  kernels.py:302-332 with the COMBINED strategy:
 *       RowAccumulator.__init__          kernels.py:75-83  (dense[cols]=0, touched=[], min=cols, max=0)
 *       accumulate, COMBINED branch      kernels.py:163-180
 *           if dense[x] == 0.0: touched.append(x)   (re-touch after a transient zero)
 *           dense[x] += av * bv                     (fp64 mul, then fp64 add; no FMA)
 *       store_row, COMBINED branch       kernels.py:255-266
 *           combined_select              kernels.py:186-191  (MinMax iff range < 2*len(touched))
 *           _store_range                 kernels.py:271-282
 *           _store_sorted                kernels.py:285-299  (sort, skip duplicates, drop == 0.0)
 *       CsrBuilder append/finalize       formats.py:165-187
 *   Row choices are reported per row exactly as KernelStats.row_choices records them
 *   (kernels.py:257-258): -1 = no record (row touched nothing), 0 = MinMax, 1 = Sort.
 *
 * The arithmetic must not be contracted into FMAs: the Makefile builds this file
 * with -ffp-contract=off, matching CPython's separately rounded float ops.
 *
 * oracle_multiply_rowmajor_mt runs the same serial algorithm on P row blocks in P
 * threads (rows of C are independent: kernels.py:323-329) and concatenates; its
 * output is byte-identical to the serial one. It is the multi-core CPU baseline.
 *
 * Pinned against the reference by tests/test_oracle.py (golden fixtures written by
 * tests/golden/make_golden.py, which imports the reference package itself).
 */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>

/* Large private buffers: 2 MiB aligned and hinted for transparent huge pages,
 * so first-touch page faults do not dominate the multi-threaded baseline. */
static void* big_alloc(size_t bytes) {
  const size_t align = (size_t)2 << 20;
  if (bytes < align) return malloc(bytes ? bytes : 1);
  void* p = NULL;
  bytes = (bytes + align - 1) / align * align;
  if (posix_memalign(&p, align, bytes)) return NULL;
  madvise(p, bytes, MADV_HUGEPAGE);
  return p;
}

#define ORACLE_OK 0
#define ORACLE_ERR_DIM 1
#define ORACLE_ERR_ARG 2
#define ORACLE_ERR_NOMEM 5
#define ORACLE_ERR_CAPACITY 7

typedef struct {
  uint64_t rows, cols;
  const uint64_t* rp;
  const uint64_t* ci;
  const double* v;
} ocsr;

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return (x > y) - (x < y);
}

static void sort_u64(uint64_t* a, uint64_t n) {
  if (n < 24) { /* insertion sort for the common short rows */
    for (uint64_t i = 1; i < n; ++i) {
      uint64_t x = a[i];
      uint64_t j = i;
      while (j > 0 && a[j - 1] > x) { a[j] = a[j - 1]; --j; }
      a[j] = x;
    }
    return;
  }
  qsort(a, (size_t)n, sizeof(uint64_t), cmp_u64);
}

/* formats.py:276-289 */
uint64_t oracle_estimate_nnz(uint64_t a_rows, const uint64_t* a_rp, const uint64_t* a_ci,
                             const uint64_t* b_rp) {
  uint64_t total = 0;
  for (uint64_t e = a_rp[0]; e < a_rp[a_rows]; ++e) {
    uint64_t k = a_ci[e];
    total += b_rp[k + 1] - b_rp[k];
  }
  return total;
}

/* perfmodel.py:63-76 walks A's stored entries; the sum is the same number. */
uint64_t oracle_count_mults(uint64_t a_rows, const uint64_t* a_rp, const uint64_t* a_ci,
                            const uint64_t* b_rp) {
  return oracle_estimate_nnz(a_rows, a_rp, a_ci, b_rp);
}

/* Per-row product counts (the quantity estimate_nnz sums), used by tests to
 * pin the GPU count pass row by row. */
void oracle_row_products(uint64_t a_rows, const uint64_t* a_rp, const uint64_t* a_ci,
                         const uint64_t* b_rp, uint64_t* out) {
  for (uint64_t r = 0; r < a_rows; ++r) {
    uint64_t p = 0;
    for (uint64_t e = a_rp[r]; e < a_rp[r + 1]; ++e) p += b_rp[a_ci[e] + 1] - b_rp[a_ci[e]];
    out[r] = p;
  }
}

/*
 * Serial COMBINED row-major product of rows [r0, r1) of A with B.
 * out_rp receives r1-r0+1 entries starting at 0. Entries go to out_ci/out_v
 * (capacity cap). choice (optional) receives one int8 per row.
 * Returns the number of entries written, or UINT64_MAX on capacity/alloc error.
 */
static uint64_t combined_rows(const ocsr* a, const ocsr* b, uint64_t r0, uint64_t r1,
                              uint64_t* out_rp, uint64_t* out_ci, double* out_v, uint64_t cap,
                              int8_t* choice) {
  const uint64_t length = b->cols;
  /* kernels.py:78; calloc keeps untouched columns as lazily zeroed pages */
  double* dense = (double*)calloc(length ? length : 1, sizeof(double));
  uint64_t tcap = 64, tlen = 0;
  uint64_t* touched = (uint64_t*)malloc(tcap * sizeof(uint64_t));
  if (!dense || !touched) { free(dense); free(touched); return UINT64_MAX; }
  uint64_t min_idx = length, max_idx = 0; /* kernels.py:82-83 */
  uint64_t cursor = 0;
  out_rp[0] = 0;
  for (uint64_t r = r0; r < r1; ++r) {
    const uint64_t lo = a->rp[r], hi = a->rp[r + 1];
    if (choice) choice[r - r0] = -1;
    if (lo != hi) { /* kernels.py:325-327 */
      /* accumulate, COMBINED branch: kernels.py:163-180 */
      for (uint64_t pos = lo; pos < hi; ++pos) {
        const double av = a->v[pos];
        const uint64_t k = a->ci[pos];
        for (uint64_t q = b->rp[k]; q < b->rp[k + 1]; ++q) {
          const uint64_t x = b->ci[q];
          if (dense[x] == 0.0) {
            if (tlen == tcap) {
              tcap *= 2;
              uint64_t* t2 = (uint64_t*)realloc(touched, tcap * sizeof(uint64_t));
              if (!t2) { free(dense); free(touched); return UINT64_MAX; }
              touched = t2;
            }
            touched[tlen++] = x;
          }
          const double prod = av * b->v[q];
          dense[x] = dense[x] + prod;
          if (x < min_idx) min_idx = x;
          if (x > max_idx) max_idx = x;
        }
      }
      /* store_row, COMBINED branch: kernels.py:255-266 */
      if (min_idx <= max_idx) {
        const int use_minmax = (max_idx - min_idx + 1) < 2 * tlen; /* combined_select */
        if (choice) choice[r - r0] = use_minmax ? 0 : 1;
        if (use_minmax) { /* _store_range: kernels.py:271-282 */
          for (uint64_t x = min_idx; x <= max_idx; ++x) {
            const double val = dense[x];
            if (val != 0.0) {
              if (cursor >= cap) { free(dense); free(touched); return UINT64_MAX; }
              out_ci[cursor] = x;
              out_v[cursor++] = val;
              dense[x] = 0.0;
            }
          }
        } else { /* _store_sorted: kernels.py:285-299 */
          sort_u64(touched, tlen);
          uint64_t prev = UINT64_MAX;
          for (uint64_t t = 0; t < tlen; ++t) {
            const uint64_t x = touched[t];
            if (x == prev) continue; /* re-touched after a transient exact zero */
            prev = x;
            const double val = dense[x];
            if (val != 0.0) {
              if (cursor >= cap) { free(dense); free(touched); return UINT64_MAX; }
              out_ci[cursor] = x;
              out_v[cursor++] = val;
              dense[x] = 0.0;
            }
          }
        }
        tlen = 0;
        min_idx = length;
        max_idx = 0;
      }
    }
    out_rp[r - r0 + 1] = cursor; /* builder.finalize(): formats.py:182-187 */
  }
  free(dense);
  free(touched);
  return cursor;
}

/*
 * C = A·B (kernels.py:302-332). out_rp has a_rows+1 entries; out_ci/out_v have
 * capacity `cap` (the reference reserves estimate_nnz entries). *nnz gets the
 * result size, *mults the multiplication count (KernelStats.multiplications).
 */
int oracle_multiply_rowmajor(uint64_t a_rows, uint64_t a_cols, const uint64_t* a_rp,
                             const uint64_t* a_ci, const double* a_v, uint64_t b_rows,
                             uint64_t b_cols, const uint64_t* b_rp, const uint64_t* b_ci,
                             const double* b_v, uint64_t* out_rp, uint64_t* out_ci,
                             double* out_v, uint64_t cap, int8_t* choice, uint64_t* nnz,
                             uint64_t* mults) {
  if (a_cols != b_rows) return ORACLE_ERR_DIM; /* kernels.py:312-313 */
  ocsr a = {a_rows, a_cols, a_rp, a_ci, a_v};
  ocsr b = {b_rows, b_cols, b_rp, b_ci, b_v};
  uint64_t n = combined_rows(&a, &b, 0, a_rows, out_rp, out_ci, out_v, cap, choice);
  if (n == UINT64_MAX) return ORACLE_ERR_CAPACITY;
  if (nnz) *nnz = n;
  if (mults) *mults = oracle_estimate_nnz(a_rows, a_rp, a_ci, b_rp);
  return ORACLE_OK;
}

/* ---- row-parallel variant (same bytes; the multi-core CPU baseline) ----
 * Three parallel phases: per-row product counts, the product of each of P
 * product-balanced row blocks into private buffers, then the concatenation
 * (each thread copies its own block). Rows are independent, so the output is
 * byte-identical to the serial product. */

typedef struct {
  const ocsr* a;
  const ocsr* b;
  uint64_t r0, r1, cap;
  uint64_t* prod; /* phase 0 output (rows) */
  uint64_t* rp;   /* phase 1: private row_ptr (r1-r0+1) */
  uint64_t* ci;
  double* v;
  uint64_t n;
  /* phase 2 */
  uint64_t base;
  uint64_t* out_rp;
  uint64_t* out_ci;
  double* out_v;
  int phase;
} ojob;

static void* run_job(void* p) {
  ojob* j = (ojob*)p;
  if (j->phase == 0) {
    for (uint64_t r = j->r0; r < j->r1; ++r) {
      uint64_t s = 0;
      for (uint64_t e = j->a->rp[r]; e < j->a->rp[r + 1]; ++e)
        s += j->b->rp[j->a->ci[e] + 1] - j->b->rp[j->a->ci[e]];
      j->prod[r] = s;
    }
  } else if (j->phase == 1) {
    j->n = combined_rows(j->a, j->b, j->r0, j->r1, j->rp, j->ci, j->v, j->cap, NULL);
  } else {
    for (uint64_t i = 0; i < j->r1 - j->r0; ++i) j->out_rp[j->r0 + i + 1] = j->base + j->rp[i + 1];
    memcpy(j->out_ci + j->base, j->ci, j->n * sizeof(uint64_t));
    memcpy(j->out_v + j->base, j->v, j->n * sizeof(double));
  }
  return NULL;
}

static void run_phase(ojob* jobs, pthread_t* th, int n, int phase) {
  for (int t = 0; t < n; ++t) {
    jobs[t].phase = phase;
    pthread_create(&th[t], NULL, run_job, &jobs[t]);
  }
  for (int t = 0; t < n; ++t) pthread_join(th[t], NULL);
}

int oracle_multiply_rowmajor_mt(int nthreads, uint64_t a_rows, uint64_t a_cols,
                                const uint64_t* a_rp, const uint64_t* a_ci, const double* a_v,
                                uint64_t b_rows, uint64_t b_cols, const uint64_t* b_rp,
                                const uint64_t* b_ci, const double* b_v, uint64_t* out_rp,
                                uint64_t* out_ci, double* out_v, uint64_t cap, uint64_t* nnz) {
  if (a_cols != b_rows) return ORACLE_ERR_DIM;
  if (nthreads < 1) nthreads = 1;
  if ((uint64_t)nthreads > a_rows) nthreads = a_rows ? (int)a_rows : 1;
  ocsr a = {a_rows, a_cols, a_rp, a_ci, a_v};
  ocsr b = {b_rows, b_cols, b_rp, b_ci, b_v};
  uint64_t* prod = (uint64_t*)malloc((a_rows + 1) * sizeof(uint64_t));
  ojob* jobs = (ojob*)calloc((size_t)nthreads, sizeof(ojob));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  if (!prod || !jobs || !th) { free(prod); free(jobs); free(th); return ORACLE_ERR_NOMEM; }
  /* phase 0: per-row product counts over equal row ranges */
  for (int t = 0; t < nthreads; ++t) {
    jobs[t].a = &a; jobs[t].b = &b; jobs[t].prod = prod;
    jobs[t].r0 = a_rows * (uint64_t)t / (uint64_t)nthreads;
    jobs[t].r1 = a_rows * (uint64_t)(t + 1) / (uint64_t)nthreads;
  }
  run_phase(jobs, th, nthreads, 0);
  uint64_t total = 0;
  for (uint64_t r = 0; r < a_rows; ++r) total += prod[r];
  /* product-balanced blocks */
  int rc = ORACLE_OK;
  uint64_t r = 0, acc = 0;
  for (int t = 0; t < nthreads; ++t) {
    const uint64_t target = (t + 1 == nthreads) ? total : total / nthreads * (t + 1);
    uint64_t r1 = r, blk = 0;
    while (r1 < a_rows && acc + prod[r1] <= target) { acc += prod[r1]; blk += prod[r1]; ++r1; }
    if (t + 1 == nthreads) while (r1 < a_rows) { blk += prod[r1]; ++r1; }
    jobs[t].r0 = r; jobs[t].r1 = r1; jobs[t].cap = blk;
    jobs[t].rp = (uint64_t*)malloc((r1 - r + 1) * sizeof(uint64_t));
    jobs[t].ci = (uint64_t*)big_alloc((blk ? blk : 1) * sizeof(uint64_t));
    jobs[t].v = (double*)big_alloc((blk ? blk : 1) * sizeof(double));
    if (!jobs[t].rp || !jobs[t].ci || !jobs[t].v) rc = ORACLE_ERR_NOMEM;
    r = r1;
  }
  if (rc == ORACLE_OK) {
    run_phase(jobs, th, nthreads, 1);
    uint64_t base = 0;
    out_rp[0] = 0;
    for (int t = 0; t < nthreads; ++t) {
      if (jobs[t].n == UINT64_MAX || base + jobs[t].n > cap) { rc = ORACLE_ERR_CAPACITY; break; }
      jobs[t].base = base;
      jobs[t].out_rp = out_rp; jobs[t].out_ci = out_ci; jobs[t].out_v = out_v;
      base += jobs[t].n;
    }
    if (rc == ORACLE_OK) {
      run_phase(jobs, th, nthreads, 2);
      if (nnz) *nnz = base;
    }
  }
  for (int t = 0; t < nthreads; ++t) { free(jobs[t].rp); free(jobs[t].ci); free(jobs[t].v); }
  free(prod); free(jobs); free(th);
  return rc;
}
