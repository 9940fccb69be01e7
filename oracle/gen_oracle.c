/*
 * gen_oracle.c — CPU restatement of the operand generators, for the CPU
 * reference arm of bench.py (`--impl reference`) and the tests.
 *
 * TEST INFRASTRUCTURE (like spmmm_oracle.c): the reference arm must not map
 * the product library, so it builds its operands here. Plain C, one thread.
 *
 *   splitmix64      sparsemm/genmat.py:28-39 (state += gamma, then the mix)
 *   next_unit       sparsemm/genmat.py:46-48 ((next >> 11) + 1) * 2^-53, in (0, 1]
 *   gen_fd          sparsemm/genmat.py:79-103 (5-point Laplacian, -1 / 4, sorted)
 *   gen_random_k    sparsemm/genmat.py:106-130 (one stream: column = next % n,
 *                   a value drawn only for an accepted (new) column; the row is
 *                   then sorted by column)
 *   gen_fd3         config C4: 27-point stencil, (dz, dy, dx)
 *                   lexicographic neighbours, 26 on the diagonal, -1 elsewhere
 *   gen_zipf        config C5: length = clipped Zipf(2) by
 *                   inverse CDF over the fp64 table sum_{j<=l} j^-2 / zeta(2),
 *                   u = (next >> 11) * 2^-53; distinct uniform columns by
 *                   rejection; values 2 u - 1 in [-1, 1)
 * The tests pin these against the reference's own fingerprints
 * (tests/golden/fingerprints.json) and against the product's generators.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static uint64_t sm_next(uint64_t* s) {
  *s += 0x9E3779B97F4A7C15ull;
  uint64_t z = *s;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int oracle_splitmix64(uint64_t seed, uint64_t n, uint64_t* out) {
  uint64_t s = seed;
  for (uint64_t i = 0; i < n; ++i) out[i] = sm_next(&s);
  return 0;
}

void oracle_gen_fd_size(uint64_t g, uint64_t* rows, uint64_t* nnz) {
  *rows = g * g;
  *nnz = 5 * g * g - 4 * g;
}

int oracle_gen_fd(uint64_t g, uint64_t* rp, uint64_t* ci, double* v) {
  const uint64_t n = g * g;
  uint64_t pos = 0;
  rp[0] = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t x = i % g, y = i / g;
    if (y > 0) { ci[pos] = i - g; v[pos++] = -1.0; }
    if (x > 0) { ci[pos] = i - 1; v[pos++] = -1.0; }
    ci[pos] = i; v[pos++] = 4.0;
    if (x + 1 < g) { ci[pos] = i + 1; v[pos++] = -1.0; }
    if (y + 1 < g) { ci[pos] = i + g; v[pos++] = -1.0; }
    rp[i + 1] = pos;
  }
  return 0;
}

void oracle_gen_fd3_size(uint64_t g, uint64_t* rows, uint64_t* nnz) {
  const uint64_t per_axis = 3 * g - 2;
  *rows = g * g * g;
  *nnz = per_axis * per_axis * per_axis;
}

int oracle_gen_fd3(uint64_t g, uint64_t* rp, uint64_t* ci, double* v) {
  const int64_t G = (int64_t)g, G2 = G * G, n = G2 * G;
  uint64_t pos = 0;
  rp[0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t x = i % G, y = (i / G) % G, z = i / G2;
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          if (z + dz < 0 || z + dz >= G || y + dy < 0 || y + dy >= G || x + dx < 0 ||
              x + dx >= G)
            continue;
          const int64_t j = i + dx + G * dy + G2 * dz;
          ci[pos] = (uint64_t)j;
          v[pos++] = j == i ? 26.0 : -1.0;
        }
    rp[i + 1] = pos;
  }
  return 0;
}

/* per-row set of drawn columns (open addressing) and the row's entries */
typedef struct {
  uint64_t* slot;
  uint64_t mask;
} colset;

static int set_reset(colset* s, uint64_t expected) {
  uint64_t cap = 16;
  while (cap < 2 * expected) cap <<= 1;
  if (cap - 1 != s->mask) {
    free(s->slot);
    s->slot = (uint64_t*)malloc(cap * sizeof(uint64_t));
    if (!s->slot) return -1;
    s->mask = cap - 1;
  }
  memset(s->slot, 0xff, (s->mask + 1) * sizeof(uint64_t));
  return 0;
}

static int set_insert(colset* s, uint64_t x) { /* 1 if new */
  uint64_t h = (x * 0x9E3779B97F4A7C15ull >> 20) & s->mask;
  for (;;) {
    if (s->slot[h] == ~0ull) { s->slot[h] = x; return 1; }
    if (s->slot[h] == x) return 0;
    h = (h + 1) & s->mask;
  }
}

typedef struct {
  uint64_t c;
  double v;
} entry;

static int by_col(const void* a, const void* b) {
  const uint64_t x = ((const entry*)a)->c, y = ((const entry*)b)->c;
  return x < y ? -1 : x > y;
}

int oracle_gen_random_k(uint64_t n, uint64_t k, uint64_t seed, uint64_t* rp, uint64_t* ci,
                        double* v) {
  if (k < 1 || k > n) return 2;
  uint64_t s = seed, pos = 0;
  colset set = {NULL, 0};
  entry* row = (entry*)malloc(k * sizeof(entry));
  if (!row) return 5;
  rp[0] = 0;
  for (uint64_t r = 0; r < n; ++r) {
    if (set_reset(&set, k)) { free(row); return 5; }
    uint64_t len = 0;
    while (len < k) {
      const uint64_t c = sm_next(&s) % n;
      if (!set_insert(&set, c)) continue; /* a repeat draws no value */
      row[len].c = c;
      row[len++].v = (double)((sm_next(&s) >> 11) + 1) * 0x1.0p-53;
    }
    qsort(row, k, sizeof(entry), by_col);
    for (uint64_t e = 0; e < k; ++e) { ci[pos] = row[e].c; v[pos++] = row[e].v; }
    rp[r + 1] = pos;
  }
  free(row);
  free(set.slot);
  return 0;
}

/* Two passes (nnz, then fill) over the same stream when rp is NULL. */
int oracle_gen_zipf(uint64_t n, uint64_t lmax, uint64_t seed, uint64_t* nnz_out, uint64_t* rp,
                    uint64_t* ci, double* v) {
  if (n < 1 || lmax < 1) return 2;
  const double zeta = M_PI * M_PI / 6.0;
  const uint64_t cap = lmax < n ? lmax : n, nt = lmax > 1 ? lmax - 1 : 0;
  double* cdf = (double*)malloc((nt ? nt : 1) * sizeof(double));
  entry* row = (entry*)malloc(cap * sizeof(entry));
  colset set = {NULL, 0};
  if (!cdf || !row) { free(cdf); free(row); return 5; }
  double partial = 0.0;
  for (uint64_t l = 1; l < lmax; ++l) {
    partial += 1.0 / pow((double)l, 2.0);
    cdf[l - 1] = partial / zeta;
  }
  uint64_t s = seed, pos = 0;
  if (rp) rp[0] = 0;
  for (uint64_t r = 0; r < n; ++r) {
    const double u = (double)(sm_next(&s) >> 11) * 0x1.0p-53;
    /* upper_bound: the number of table entries <= u */
    uint64_t lo = 0, hi = nt;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) / 2;
      if (cdf[mid] <= u) lo = mid + 1; else hi = mid;
    }
    uint64_t len = lo + 1;
    if (len > cap) len = cap;
    if (set_reset(&set, len)) { free(cdf); free(row); return 5; }
    uint64_t got = 0;
    while (got < len) {
      const uint64_t c = sm_next(&s) % n;
      if (!set_insert(&set, c)) continue;
      row[got].c = c;
      row[got++].v = 2.0 * ((double)(sm_next(&s) >> 11) * 0x1.0p-53) - 1.0;
    }
    if (rp) {
      qsort(row, len, sizeof(entry), by_col);
      for (uint64_t e = 0; e < len; ++e) { ci[pos] = row[e].c; v[pos++] = row[e].v; }
      rp[r + 1] = pos;
    } else {
      pos += len;
    }
  }
  *nnz_out = pos;
  free(cdf);
  free(row);
  free(set.slot);
  return 0;
}
