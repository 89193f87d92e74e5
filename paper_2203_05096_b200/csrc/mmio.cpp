// Native, multi-threaded parser of the entry lines of a coordinate Matrix
// Market file -- the body loop of the reference's read_matrix_market
// (io.py:96-206) for large files.  Strict: any line outside the plain
// grammar (signed decimal indices, a strtod-parsable decimal value, the
// declared token count, indices in range, no skew-symmetric diagonal, the
// declared entry count) makes the call fail, and the Python loop re-reads
// the body to raise the reference's exact error with its line number.
// Accepted inputs therefore parse to exactly what the Python loop yields.

#include <omp.h>

#include <cerrno>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/csrk.h"

namespace csrk {
void set_error(const char *fmt, ...);  // abi.cu
}

namespace {

inline bool is_space(char c) {
  return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f';
}

// a data line: not blank, not a comment (after leading whitespace)
inline bool is_data(const char *a, const char *b) {
  while (a < b && is_space(*a)) ++a;
  return a < b && *a != '%';
}

inline bool parse_int(const char *a, const char *b, int64_t *out) {
  const char *p = a;
  if (p < b && (*p == '+' || *p == '-')) ++p;
  if (p == b) return false;
  for (const char *q = p; q < b; ++q)
    if (*q < '0' || *q > '9') return false;
  if (b - p > 18) return false;  // beyond int64 range checks: let Python decide
  char tmp[32];
  std::memcpy(tmp, a, b - a);
  tmp[b - a] = '\0';
  *out = std::strtoll(tmp, nullptr, 10);
  return true;
}

inline bool parse_real(const char *a, const char *b, double *out) {
  if (b - a > 64) return false;
  for (const char *q = a; q < b; ++q)  // decimal syntax only (no hex, no nan(...))
    if (*q == 'x' || *q == 'X' || *q == '(' || *q == '_' || *q == 'p' || *q == 'P')
      return false;
  char tmp[72];
  std::memcpy(tmp, a, b - a);
  tmp[b - a] = '\0';
  char *end = nullptr;
  errno = 0;
  *out = std::strtod(tmp, &end);
  return end == tmp + (b - a);
}

// parse one data line into (i, j, v); false on anything unusual
inline bool parse_line(const char *a, const char *b, int ntok, int64_t n_rows, int64_t n_cols,
                       bool skew, int64_t *i, int64_t *j, double *v) {
  const char *tok[4][2];
  int n = 0;
  const char *p = a;
  while (p < b) {
    while (p < b && is_space(*p)) ++p;
    if (p == b) break;
    const char *s = p;
    while (p < b && !is_space(*p)) ++p;
    if (n == 3) return false;
    tok[n][0] = s;
    tok[n][1] = p;
    ++n;
  }
  if (n != ntok) return false;
  if (!parse_int(tok[0][0], tok[0][1], i) || !parse_int(tok[1][0], tok[1][1], j)) return false;
  if (*i < 1 || *i > n_rows || *j < 1 || *j > n_cols) return false;
  if (skew && *i == *j) return false;
  *v = 1.0;
  if (ntok == 3 && !parse_real(tok[2][0], tok[2][1], v)) return false;
  return true;
}

}  // namespace

extern "C" int csrk_mm_parse(const char *buf, int64_t len, int64_t n_entries, int with_value,
                             int64_t n_rows, int64_t n_cols, int skew, int64_t *rows,
                             int64_t *cols, double *vals) {
  if (!buf || len < 0 || n_entries < 0 || (n_entries > 0 && (!rows || !cols || !vals))) {
    csrk::set_error("invalid argument to csrk_mm_parse");
    return CSRK_EINVAL;
  }
  const int threads = omp_get_max_threads();
  const int chunks = len < (1 << 20) ? 1 : threads * 4;
  // chunk bounds on line starts
  std::vector<int64_t> start(chunks + 1, len);
  start[0] = 0;
  for (int c = 1; c < chunks; ++c) {
    int64_t pos = len * c / chunks;
    if (pos < start[c - 1]) pos = start[c - 1];
    while (pos < len && pos > 0 && buf[pos - 1] != '\n') ++pos;
    start[c] = pos;
  }
  start[chunks] = len;
  // pass 1: data lines per chunk
  std::vector<int64_t> count(chunks + 1, 0);
#pragma omp parallel for schedule(dynamic, 1)
  for (int c = 0; c < chunks; ++c) {
    int64_t k = 0;
    const char *p = buf + start[c], *e = buf + start[c + 1];
    while (p < e) {
      const char *nl = static_cast<const char *>(std::memchr(p, '\n', e - p));
      const char *le = nl ? nl : e;
      k += is_data(p, le);
      p = nl ? nl + 1 : e;
    }
    count[c + 1] = k;
  }
  for (int c = 0; c < chunks; ++c) count[c + 1] += count[c];
  if (count[chunks] != n_entries) {
    csrk::set_error("entry count differs from the header");
    return CSRK_EINVAL;
  }
  // pass 2: parse into place
  int bad = 0;
  const int ntok = with_value ? 3 : 2;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
  for (int c = 0; c < chunks; ++c) {
    int64_t k = count[c];
    const char *p = buf + start[c], *e = buf + start[c + 1];
    while (p < e && !bad) {
      const char *nl = static_cast<const char *>(std::memchr(p, '\n', e - p));
      const char *le = nl ? nl : e;
      if (is_data(p, le)) {
        int64_t i = 0, j = 0;
        double v = 1.0;
        if (!parse_line(p, le, ntok, n_rows, n_cols, skew != 0, &i, &j, &v)) {
          bad = 1;
          break;
        }
        rows[k] = i - 1;
        cols[k] = j - 1;
        vals[k] = v;
        ++k;
      }
      p = nl ? nl + 1 : e;
    }
  }
  if (bad) {
    csrk::set_error("entry outside the plain grammar");
    return CSRK_EINVAL;
  }
  return CSRK_OK;
}
