// Matrix Market coordinate I/O (ASCII, 1-based, "matrix coordinate real
// general"), native and multi-threaded: the reference's mtxio.py:1-72 with the
// same acceptance rules and error messages (entries in any order, comments
// and blank lines skipped, duplicates / out-of-range / wrong count rejected;
// the writer emits row-major order with %.17g values, which round-trips
// every double bit for bit — Python's '{:.17g}' and C's "%.17g" agree).
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/spmmm_mtx.h"

namespace {

thread_local std::string g_mtx_err;

int mtx_fail(int code, const std::string& msg) {
  g_mtx_err = msg;
  return code;
}

constexpr const char* kHeader = "%%MatrixMarket matrix coordinate real general";

unsigned n_threads() {
  unsigned t = std::thread::hardware_concurrency();
  return std::max(1u, std::min(t, 32u));
}

bool is_blank(const char* s, const char* e) {
  for (; s < e; ++s)
    if (!std::isspace(static_cast<unsigned char>(*s))) return false;
  return true;
}

std::string strip(const char* s, const char* e) {
  while (s < e && std::isspace(static_cast<unsigned char>(*s))) ++s;
  while (e > s && std::isspace(static_cast<unsigned char>(e[-1]))) --e;
  return std::string(s, e);
}

// Python repr of a plain ASCII string (the messages quote lines with !r)
std::string py_repr(const std::string& s) {
  const bool dq = s.find('\'') != std::string::npos && s.find('"') == std::string::npos;
  std::string out(1, dq ? '"' : '\'');
  for (char ch : s) {
    if (ch == '\\') out += "\\\\";
    else if (ch == '\t') out += "\\t";
    else if (!dq && ch == '\'') out += "\\'";
    else out += ch;
  }
  out += dq ? '"' : '\'';
  return out;
}

// whitespace-separated fields of [s, e)
void split_fields(const char* s, const char* e, std::vector<std::string>& out) {
  out.clear();
  while (s < e) {
    while (s < e && std::isspace(static_cast<unsigned char>(*s))) ++s;
    const char* t = s;
    while (t < e && !std::isspace(static_cast<unsigned char>(*t))) ++t;
    if (t > s) out.emplace_back(s, t);
    s = t;
  }
}

bool parse_int(const std::string& f, long long* v) {
  if (f.empty()) return false;
  errno = 0;
  char* end = nullptr;
  const long long x = std::strtoll(f.c_str(), &end, 10);
  if (errno || *end) return false;
  *v = x;
  return true;
}

bool parse_real(const std::string& f, double* v) {
  if (f.empty()) return false;
  // Python's float() takes no hexadecimal literals
  if (f.find('x') != std::string::npos || f.find('X') != std::string::npos) return false;
  char* end = nullptr;
  const double x = std::strtod(f.c_str(), &end);
  if (*end) return false;
  *v = x;
  return true;
}

struct Chunk {
  std::vector<uint32_t> r, c;
  std::vector<double> v;
  size_t err_pos = SIZE_MAX;  // byte offset of the first bad line in this chunk
  int err_code = 0;
  std::string err_msg;
};

struct Mtx {
  uint64_t rows = 0, cols = 0, nnz = 0;
  std::vector<uint64_t> rp, ci;
  std::vector<double> v;
};

}  // namespace

struct spmmm_mtx : Mtx {};

extern "C" {

const char* spmmm_mtx_last_error(void) { return g_mtx_err.c_str(); }

int spmmm_mtx_write(const char* path, const spmmm_csr* m) {
  if (!path || !m || !m->row_ptr) return mtx_fail(SPMMM_ERR_INVALID, "NULL argument");
  if (m->memory != SPMMM_MEM_HOST) return mtx_fail(SPMMM_ERR_INVALID, "host arrays required");
  const uint64_t rows = m->rows;
  const unsigned T = rows > 65536 ? n_threads() : 1;
  std::vector<std::string> parts(T);
  std::vector<std::thread> th;
  for (unsigned t = 0; t < T; ++t) {
    th.emplace_back([&, t] {
      const uint64_t r0 = rows * t / T, r1 = rows * (t + 1) / T;
      std::string& s = parts[t];
      s.reserve((m->row_ptr[r1] - m->row_ptr[r0]) * 40);
      char buf[96];
      for (uint64_t r = r0; r < r1; ++r)
        for (uint64_t p = m->row_ptr[r]; p < m->row_ptr[r + 1]; ++p) {
          const int n = std::snprintf(buf, sizeof buf, "%" PRIu64 " %" PRIu64 " %.17g\n", r + 1,
                                      m->col_idx[p] + 1, m->values[p]);
          s.append(buf, size_t(n));
        }
    });
  }
  for (auto& x : th) x.join();
  FILE* f = std::fopen(path, "wb");
  if (!f) return mtx_fail(SPMMM_ERR_INVALID, std::string("cannot open ") + path);
  const uint64_t nnz = m->row_ptr[rows] - m->row_ptr[0];
  std::fprintf(f, "%s\n%" PRIu64 " %" PRIu64 " %" PRIu64 "\n", kHeader, rows, m->cols, nnz);
  for (auto& s : parts) std::fwrite(s.data(), 1, s.size(), f);
  if (std::fclose(f) != 0) return mtx_fail(SPMMM_ERR_INVALID, std::string("write failed: ") + path);
  return SPMMM_OK;
}

int spmmm_mtx_read(const char* path, spmmm_mtx** out) {
  if (!path || !out) return mtx_fail(SPMMM_ERR_INVALID, "NULL argument");
  *out = nullptr;
  FILE* f = std::fopen(path, "rb");
  if (!f) return mtx_fail(SPMMM_ERR_INVALID, std::string("cannot open ") + path);
  std::string data;
  {
    std::fseek(f, 0, SEEK_END);
    const long sz = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    data.resize(sz > 0 ? size_t(sz) : 0);
    if (sz > 0 && std::fread(&data[0], 1, data.size(), f) != data.size()) {
      std::fclose(f);
      return mtx_fail(SPMMM_ERR_INVALID, std::string("read failed: ") + path);
    }
    std::fclose(f);
  }
  const char* s = data.data();
  const char* end = s + data.size();
  auto line_end = [&](const char* p) {
    const char* q = static_cast<const char*>(std::memchr(p, '\n', size_t(end - p)));
    return q ? q : end;
  };
  // header (mtxio.py:31-37)
  const char* le = line_end(s);
  std::string header(s, le);
  {
    std::string low = header;
    for (auto& ch : low) ch = char(std::tolower(static_cast<unsigned char>(ch)));
    std::vector<std::string> fl;
    split_fields(low.data(), low.data() + low.size(), fl);
    const std::vector<std::string> want = {"%%matrixmarket", "matrix", "coordinate", "real",
                                           "general"};
    if (fl != want)
      return mtx_fail(SPMMM_ERR_INVALID, "unsupported Matrix Market header: " +
                                             py_repr(strip(header.data(),
                                                           header.data() + header.size())));
  }
  const char* p = le < end ? le + 1 : end;
  // size line: the first line that is neither a comment nor blank (:38-42)
  while (true) {
    if (p >= end) return mtx_fail(SPMMM_ERR_INVALID, "missing size line");
    le = line_end(p);
    if (*p != '%' && !is_blank(p, le)) break;
    p = le < end ? le + 1 : end;
  }
  std::vector<std::string> fl;
  split_fields(p, le, fl);
  long long dims[3];
  if (fl.size() != 3 || !parse_int(fl[0], dims) || !parse_int(fl[1], dims + 1) ||
      !parse_int(fl[2], dims + 2))
    return mtx_fail(SPMMM_ERR_INVALID, "malformed size line: " + py_repr(strip(p, le)));
  if (dims[0] < 0 || dims[1] < 0 || dims[2] < 0 || dims[0] >= (1ll << 32) ||
      dims[1] >= (1ll << 32))
    return mtx_fail(SPMMM_ERR_UNSUPPORTED, "matrix dimensions outside the supported range");
  const uint64_t rows = uint64_t(dims[0]), cols = uint64_t(dims[1]), nnz = uint64_t(dims[2]);
  const char* body = le < end ? le + 1 : end;
  // entries: parsed in parallel chunks cut at line boundaries (:44-52)
  const size_t blen = size_t(end - body);
  const unsigned T = blen > (1u << 20) ? n_threads() : 1;
  std::vector<const char*> cut(T + 1);
  cut[0] = body;
  cut[T] = end;
  for (unsigned t = 1; t < T; ++t) {
    const char* q = body + blen * t / T;
    q = std::max(q, cut[t - 1]);
    const char* nl = static_cast<const char*>(std::memchr(q, '\n', size_t(end - q)));
    cut[t] = nl ? nl + 1 : end;
  }
  std::vector<Chunk> ch(T);
  std::vector<std::thread> th;
  for (unsigned t = 0; t < T; ++t) {
    th.emplace_back([&, t] {
      Chunk& c = ch[t];
      std::vector<std::string> f2;
      for (const char* q = cut[t]; q < cut[t + 1];) {
        const char* e = static_cast<const char*>(std::memchr(q, '\n', size_t(cut[t + 1] - q)));
        if (!e) e = cut[t + 1];
        const char* a = q;
        while (a < e && std::isspace(static_cast<unsigned char>(*a))) ++a;
        if (a < e && *a != '%') {
          split_fields(a, e, f2);
          long long r, cc;
          double v;
          if (f2.size() != 3 || !parse_int(f2[0], &r) || !parse_int(f2[1], &cc) ||
              !parse_real(f2[2], &v)) {
            c.err_pos = size_t(q - body);
            c.err_code = SPMMM_ERR_INVALID;
            c.err_msg = "malformed entry line: " + py_repr(strip(a, e));
            return;
          }
          if (!(r >= 1 && uint64_t(r - 1) < rows && cc >= 1 && uint64_t(cc - 1) < cols)) {
            c.err_pos = size_t(q - body);
            c.err_code = SPMMM_ERR_INVALID;
            c.err_msg = "entry (" + f2[0] + ", " + f2[1] + ") outside " + std::to_string(rows) +
                        " x " + std::to_string(cols);
            return;
          }
          c.r.push_back(uint32_t(r - 1));
          c.c.push_back(uint32_t(cc - 1));
          c.v.push_back(v);
        }
        q = e < cut[t + 1] ? e + 1 : e;
      }
    });
  }
  for (auto& x : th) x.join();
  for (auto& c : ch)  // the first bad line in file order
    if (c.err_code) return mtx_fail(c.err_code, c.err_msg);
  uint64_t got = 0;
  for (auto& c : ch) got += c.r.size();
  if (got != nnz)
    return mtx_fail(SPMMM_ERR_INVALID, "size line promises " + std::to_string(nnz) +
                                           " entries, file holds " + std::to_string(got));
  // row-major order (:53-67): counting sort by row, then columns within a row
  auto* m = new spmmm_mtx;
  m->rows = rows;
  m->cols = cols;
  m->nnz = nnz;
  m->rp.assign(rows + 1, 0);
  for (auto& c : ch)
    for (uint32_t r : c.r) ++m->rp[r + 1];
  for (uint64_t r = 0; r < rows; ++r) m->rp[r + 1] += m->rp[r];
  std::vector<uint64_t> next(m->rp.begin(), m->rp.end() - 1);
  std::vector<std::pair<uint32_t, double>> ent(nnz);
  for (auto& c : ch)
    for (size_t i = 0; i < c.r.size(); ++i) ent[next[c.r[i]]++] = {c.c[i], c.v[i]};
  m->ci.resize(nnz);
  m->v.resize(nnz);
  for (uint64_t r = 0; r < rows; ++r) {
    auto b = ent.begin() + int64_t(m->rp[r]), e = ent.begin() + int64_t(m->rp[r + 1]);
    std::stable_sort(b, e, [](const auto& x, const auto& y) { return x.first < y.first; });
    for (auto it = b; it != e; ++it) {
      if (it != b && it->first == (it - 1)->first) {
        const uint64_t col = it->first;
        delete m;
        return mtx_fail(SPMMM_ERR_INVALID, "duplicate entry at row " + std::to_string(r + 1) +
                                               ", column " + std::to_string(col + 1));
      }
      m->ci[size_t(it - ent.begin())] = it->first;
      m->v[size_t(it - ent.begin())] = it->second;
    }
  }
  *out = m;
  return SPMMM_OK;
}

int spmmm_mtx_shape(const spmmm_mtx* m, uint64_t* rows, uint64_t* cols, uint64_t* nnz) {
  if (!m) return mtx_fail(SPMMM_ERR_INVALID, "NULL argument");
  if (rows) *rows = m->rows;
  if (cols) *cols = m->cols;
  if (nnz) *nnz = m->nnz;
  return SPMMM_OK;
}

int spmmm_mtx_copy(const spmmm_mtx* m, uint64_t* row_ptr, uint64_t* col_idx, double* values) {
  if (!m) return mtx_fail(SPMMM_ERR_INVALID, "NULL argument");
  if (row_ptr) std::memcpy(row_ptr, m->rp.data(), m->rp.size() * sizeof(uint64_t));
  if (col_idx && m->nnz) std::memcpy(col_idx, m->ci.data(), m->nnz * sizeof(uint64_t));
  if (values && m->nnz) std::memcpy(values, m->v.data(), m->nnz * sizeof(double));
  return SPMMM_OK;
}

int spmmm_mtx_free(spmmm_mtx* m) {
  delete m;
  return SPMMM_OK;
}

}  // extern "C"
