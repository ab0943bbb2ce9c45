// Native edge-list and layout loaders ("fast
// edge-list and layout loaders"; the reference parses line by line in
// Python, graphio.py:46-117).
//
// Host code only.  The parsers accept the common, unambiguous subset of the
// reference's formats and report GLR_EFALLBACK for anything whose meaning
// depends on Python's rules (non-ASCII text, \r / \v / \f line breaks,
// underscores or other int()/float() spellings, inf/nan, over-long ids,
// malformed lines): the Python layer then runs its restatement of the
// reference parser, which produces the reference's exact result or error.
// Inside the subset the results are identical: integers are decimal digit
// strings, and reals go through strtod, which rounds correctly like
// Python's float().
#include <cerrno>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace glr {
namespace {

inline bool is_ws(char c) { return c == ' ' || c == '\t'; }

// the buffer is plain ASCII with '\n' line breaks only
bool plain_ascii(const char *b, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    const unsigned char c = (unsigned char)b[i];
    if (c >= 0x80 || c == '\r' || c == '\v' || c == '\f' || (c < 0x20 && c != '\n' && c != '\t') ||
        c == 0x1c || c == 0x1d || c == 0x1e)
      return false;
  }
  return true;
}

// [+]digits (<= 18 digits) -> value; false if anything else
bool parse_uint(const char *s, const char *e, int64_t *v) {
  if (s < e && *s == '+') ++s;
  if (s == e || e - s > 18) return false;
  int64_t x = 0;
  for (const char *p = s; p < e; ++p) {
    if (*p < '0' || *p > '9') return false;
    x = x * 10 + (*p - '0');
  }
  *v = x;
  return true;
}

// [+-]digits (<= 18 digits)
bool parse_int(const char *s, const char *e, int64_t *v) {
  bool neg = false;
  if (s < e && (*s == '-' || *s == '+')) {
    neg = *s == '-';
    ++s;
  }
  if (s < e && (*s == '+' || *s == '-')) return false;
  int64_t x;
  if (!parse_uint(s, e, &x)) return false;
  *v = neg ? -x : x;
  return true;
}

// [+-](digits[.digits*] | .digits)[(e|E)[+-]digits] -> strtod (correctly
// rounded, as Python's float()); rejects every other spelling
bool parse_real(const char *s, const char *e, double *v) {
  const char *p = s;
  if (p < e && (*p == '+' || *p == '-')) ++p;
  const char *d0 = p;
  while (p < e && *p >= '0' && *p <= '9') ++p;
  int digits = (int)(p - d0);
  if (p < e && *p == '.') {
    ++p;
    const char *f0 = p;
    while (p < e && *p >= '0' && *p <= '9') ++p;
    digits += (int)(p - f0);
  }
  if (digits == 0) return false;
  if (p < e && (*p == 'e' || *p == 'E')) {
    ++p;
    if (p < e && (*p == '+' || *p == '-')) ++p;
    const char *x0 = p;
    while (p < e && *p >= '0' && *p <= '9') ++p;
    if (p == x0) return false;
  }
  if (p != e || e - s > 400) return false;
  char tmp[416];
  memcpy(tmp, s, (size_t)(e - s));
  tmp[e - s] = '\0';
  errno = 0;
  char *end = nullptr;
  const double x = strtod(tmp, &end);
  if (end != tmp + (e - s)) return false;
  *v = x;  // overflow gives +-inf, which the caller treats like Python (non-finite)
  return true;
}

void trim(const char *&s, const char *&e) {
  while (s < e && is_ws(*s)) ++s;
  while (e > s && is_ws(e[-1])) --e;
}

}  // namespace
}  // namespace glr

extern "C" {

int glr_parse_edgelist(const char *buf, size_t len, int64_t *out, int64_t cap, int64_t *count) {
  using namespace glr;
  if ((buf == nullptr && len > 0) || count == nullptr || cap < 0) {
    set_error("glr_parse_edgelist: invalid arguments");
    return GLR_EARG;
  }
  if (!plain_ascii(buf, len)) {
    set_error("glr_parse_edgelist: text needs the Python parser");
    return GLR_EFALLBACK;
  }
  int64_t n = 0;
  const char *p = buf, *end = buf + len;
  while (p < end) {
    const char *nl = static_cast<const char *>(memchr(p, '\n', (size_t)(end - p)));
    const char *le = nl ? nl : end;
    const char *s = p, *e = le;
    p = nl ? nl + 1 : end;
    trim(s, e);
    if (s == e || *s == '#') continue;
    // exactly two whitespace-separated tokens
    const char *a0 = s, *a1 = s;
    while (a1 < e && !is_ws(*a1)) ++a1;
    const char *b0 = a1;
    while (b0 < e && is_ws(*b0)) ++b0;
    const char *b1 = b0;
    while (b1 < e && !is_ws(*b1)) ++b1;
    int64_t u, v;
    if (b0 == e || b1 != e || !parse_uint(a0, a1, &u) || !parse_uint(b0, b1, &v)) {
      set_error("glr_parse_edgelist: line needs the Python parser");
      return GLR_EFALLBACK;
    }
    if (out != nullptr && n < cap) {
      out[2 * n] = u;
      out[2 * n + 1] = v;
    }
    ++n;
  }
  *count = n;
  return GLR_OK;
}

int glr_parse_layout(const char *buf, size_t len, int64_t *ids, double *xy, int64_t cap,
                     int64_t *count) {
  using namespace glr;
  if ((buf == nullptr && len > 0) || count == nullptr || cap < 0) {
    set_error("glr_parse_layout: invalid arguments");
    return GLR_EARG;
  }
  if (!plain_ascii(buf, len)) {
    set_error("glr_parse_layout: text needs the Python parser");
    return GLR_EFALLBACK;
  }
  const char *p = buf, *end = buf + len;
  int64_t n = 0;
  bool header = true;
  while (p < end) {
    const char *nl = static_cast<const char *>(memchr(p, '\n', (size_t)(end - p)));
    const char *le = nl ? nl : end;
    const char *s = p, *e = le;
    p = nl ? nl + 1 : end;
    if (header) {  // exactly "id,x,y" up to spaces around the fields
      const char *f[4];
      int k = 0;
      f[0] = s;
      for (const char *q = s; q < e && k < 3; ++q)
        if (*q == ',') f[++k] = q + 1;
      const char *want[3] = {"id", "x", "y"};
      bool ok = k == 2;
      for (int i = 0; ok && i < 3; ++i) {
        const char *a = f[i];
        const char *b = i < 2 ? f[i + 1] - 1 : e;
        trim(a, b);
        ok = (size_t)(b - a) == strlen(want[i]) && memcmp(a, want[i], (size_t)(b - a)) == 0;
      }
      if (!ok) {
        set_error("glr_parse_layout: header needs the Python parser");
        return GLR_EFALLBACK;
      }
      header = false;
      continue;
    }
    const char *s2 = s, *e2 = e;
    trim(s2, e2);
    if (s2 == e2) continue;
    const char *c1 = static_cast<const char *>(memchr(s, ',', (size_t)(e - s)));
    const char *c2 = c1 ? static_cast<const char *>(memchr(c1 + 1, ',', (size_t)(e - c1 - 1)))
                        : nullptr;
    if (c1 == nullptr || c2 == nullptr || memchr(c2 + 1, ',', (size_t)(e - c2 - 1)) != nullptr) {
      set_error("glr_parse_layout: row needs the Python parser");
      return GLR_EFALLBACK;
    }
    const char *i0 = s, *i1 = c1, *x0 = c1 + 1, *x1 = c2, *y0 = c2 + 1, *y1 = e;
    trim(i0, i1);
    trim(x0, x1);
    trim(y0, y1);
    int64_t vid;
    double x, y;
    if (!parse_int(i0, i1, &vid) || !parse_real(x0, x1, &x) || !parse_real(y0, y1, &y) ||
        !std::isfinite(x) || !std::isfinite(y)) {
      set_error("glr_parse_layout: row needs the Python parser");
      return GLR_EFALLBACK;
    }
    if (ids != nullptr && n < cap) {
      ids[n] = vid;
      xy[2 * n] = x;
      xy[2 * n + 1] = y;
    }
    ++n;
  }
  if (header) {
    set_error("glr_parse_layout: empty file needs the Python parser");
    return GLR_EFALLBACK;
  }
  *count = n;
  return GLR_OK;
}

}  // extern "C"
