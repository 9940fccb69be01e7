// Seeded operand generators (host code, C ABI declared in include/spmmm_gen.h).
//
// Not on the spMMM hot path: these only build the synthetic operands for the
// BASELINE configs. The first three restate the reference package's
// generators bit for bit:
//   splitmix64   sparsemm/genmat.py:28-48
//   gen_fd       sparsemm/genmat.py:79-103
//   gen_random_k sparsemm/genmat.py:106-130  (one shared stream, a value is
//                drawn only for an accepted column, rows sorted by column)
// gen_fd3 (C4) and gen_zipf (C5) are new; their construction is the one laid
// out in SURVEY.md §8(d).
#include "../../include/spmmm_gen.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <utility>
#include <vector>

namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kMix1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kMix2 = 0x94D049BB133111EBull;

struct SplitMix64 {
  uint64_t state;
  explicit SplitMix64(uint64_t seed) : state(seed) {}
  uint64_t next() {
    state += kGamma;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * kMix1;
    z = (z ^ (z >> 27)) * kMix2;
    return z ^ (z >> 31);
  }
  // (0, 1]: top 53 bits plus one, times 2^-53 (genmat.py:46-48)
  double unit_open0() { return double((next() >> 11) + 1) * 0x1.0p-53; }
  // [0, 1): top 53 bits times 2^-53
  double unit_closed0() { return double(next() >> 11) * 0x1.0p-53; }
};

// Small open-addressing set of uint64 used for per-row rejection of repeats.
class RowSet {
 public:
  void reset(size_t expected) {
    size_t cap = 16;
    while (cap < expected * 2) cap <<= 1;
    if (slots_.size() != cap) slots_.assign(cap, kEmpty);
    else std::fill(slots_.begin(), slots_.end(), kEmpty);
    mask_ = cap - 1;
  }
  // true if inserted, false if already present
  bool insert(uint64_t x) {
    size_t h = size_t((x * 0x9E3779B97F4A7C15ull) >> 20) & mask_;
    while (true) {
      if (slots_[h] == kEmpty) { slots_[h] = x; return true; }
      if (slots_[h] == x) return false;
      h = (h + 1) & mask_;
    }
  }

 private:
  static constexpr uint64_t kEmpty = ~0ull;
  std::vector<uint64_t> slots_;
  size_t mask_ = 0;
};

}  // namespace

extern "C" {

int spmmm_splitmix64(uint64_t seed, uint64_t n, uint64_t* out) {
  if (!out && n) return 2;
  SplitMix64 rng(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = rng.next();
  return 0;
}

int spmmm_gen_fd_size(uint64_t grid, uint64_t* rows, uint64_t* nnz) {
  if (grid < 1 || !rows || !nnz) return 2;
  *rows = grid * grid;
  *nnz = 5 * grid * grid - 4 * grid;
  return 0;
}

int spmmm_gen_fd(uint64_t g, uint64_t* rp, uint64_t* ci, double* v) {
  if (g < 1 || !rp || !ci || !v) return 2;
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

int spmmm_gen_fd3_size(uint64_t g, uint64_t* rows, uint64_t* nnz) {
  if (g < 1 || !rows || !nnz) return 2;
  // per axis, the number of (coordinate, offset) pairs that stay inside: 3g - 2
  const uint64_t per_axis = 3 * g - 2;
  *rows = g * g * g;
  *nnz = per_axis * per_axis * per_axis;
  return 0;
}

int spmmm_gen_fd3(uint64_t g, uint64_t* rp, uint64_t* ci, double* v) {
  if (g < 1 || !rp || !ci || !v) return 2;
  const uint64_t n = g * g * g, g2 = g * g;
  uint64_t pos = 0;
  rp[0] = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const int64_t x = int64_t(i % g), y = int64_t((i / g) % g), z = int64_t(i / g2);
    // (dz, dy, dx) lexicographic with dz outermost gives ascending columns
    for (int dz = -1; dz <= 1; ++dz) {
      if (z + dz < 0 || z + dz >= int64_t(g)) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        if (y + dy < 0 || y + dy >= int64_t(g)) continue;
        for (int dx = -1; dx <= 1; ++dx) {
          if (x + dx < 0 || x + dx >= int64_t(g)) continue;
          const uint64_t j = uint64_t(int64_t(i) + dx + int64_t(g) * dy + int64_t(g2) * dz);
          ci[pos] = j;
          v[pos++] = (j == i) ? 26.0 : -1.0;
        }
      }
    }
    rp[i + 1] = pos;
  }
  return 0;
}

int spmmm_gen_random_k(uint64_t n, uint64_t k, uint64_t seed, uint64_t* rp, uint64_t* ci,
                       double* v) {
  if (k < 1 || k > n || !rp || !ci || !v) return 2;
  SplitMix64 rng(seed);
  RowSet seen;
  std::vector<std::pair<uint64_t, double>> row;
  row.reserve(k);
  uint64_t pos = 0;
  rp[0] = 0;
  for (uint64_t r = 0; r < n; ++r) {
    row.clear();
    seen.reset(k);
    while (row.size() < k) {
      const uint64_t c = rng.next() % n;
      if (!seen.insert(c)) continue;  // rejected repeats draw no value
      row.emplace_back(c, rng.unit_open0());
    }
    std::sort(row.begin(), row.end(),
              [](const auto& a, const auto& b) { return a.first < b.first; });
    for (const auto& e : row) { ci[pos] = e.first; v[pos++] = e.second; }
    rp[r + 1] = pos;
  }
  return 0;
}

int spmmm_gen_zipf(uint64_t n, double s, uint64_t lmax, uint64_t seed, uint64_t* nnz_out,
                   uint64_t* rp, uint64_t* ci, double* v) {
  if (n < 1 || lmax < 1 || !(s > 1.0) || !nnz_out) return 2;
  const bool fill = rp && ci && v;
  const uint64_t cap = std::min(lmax, n);
  // Inverse-CDF table for lengths 1..lmax-1, normalised by zeta(s); the
  // remaining mass (the clipped tail) maps to lmax.
  double zeta = 0.0;
  if (s == 2.0) {
    zeta = M_PI * M_PI / 6.0;
  } else {
    for (uint64_t j = 1; j < 10000000; ++j) zeta += std::pow(double(j), -s);
  }
  std::vector<double> cdf(lmax > 1 ? lmax - 1 : 0);
  double partial = 0.0;
  for (uint64_t l = 1; l < lmax; ++l) {
    partial += 1.0 / std::pow(double(l), s);
    cdf[l - 1] = partial / zeta;
  }
  SplitMix64 rng(seed);
  RowSet seen;
  std::vector<std::pair<uint64_t, double>> row;
  uint64_t pos = 0;
  if (fill) rp[0] = 0;
  for (uint64_t r = 0; r < n; ++r) {
    const double u = rng.unit_closed0();
    uint64_t len = uint64_t(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin()) + 1;
    if (len > cap) len = cap;
    row.clear();
    seen.reset(len);
    while (row.size() < len) {
      const uint64_t c = rng.next() % n;
      if (!seen.insert(c)) continue;
      row.emplace_back(c, 2.0 * rng.unit_closed0() - 1.0);
    }
    if (fill) {
      std::sort(row.begin(), row.end(),
                [](const auto& a, const auto& b) { return a.first < b.first; });
      for (const auto& e : row) { ci[pos] = e.first; v[pos++] = e.second; }
      rp[r + 1] = pos;
    } else {
      pos += len;
    }
  }
  *nnz_out = pos;
  return 0;
}

}  // extern "C"
