// Native edge-list and layout loaders ("fast
// edge-list and layout loaders"; the reference parses line by line in
// Python, graphio.py:46-117).
//
// Host code only, and the whole input grammar: the text is UTF-8, cut into
// lines at every boundary Python's str.splitlines() knows (\n, \r, \r\n,
// \v, \f, \x1c-\x1e, U+0085, U+2028, U+2029), trimmed and split at every
// code point str.isspace() accepts, and numbers follow int() / float() of a
// str: any Unicode decimal digit (Nd) counts as its ASCII digit, single
// underscores may sit between digits, int() refuses more than 4300 digits
// (sys.get_int_max_str_digits()), float() takes inf / infinity / nan in any
// case and rounds correctly (strtod).  Errors are reported as a kind, a line
// number and a byte span of the line (glr_parse_status); the Python layer
// formats the reference's message from them (graphio.py), so no text is
// ever re-parsed in Python.  Unicode tables: Python 3.12 / Unicode 15.0
// (tools/gen_unicode_tables.py).
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace glr {
namespace {

// code points with Unicode decimal value 0 (each starts a run 0..9)
const uint32_t kDigitZeros[] = {
    0x30,    0x660,   0x6f0,   0x7c0,   0x966,   0x9e6,   0xa66,   0xae6,   0xb66,   0xbe6,
    0xc66,   0xce6,   0xd66,   0xde6,   0xe50,   0xed0,   0xf20,   0x1040,  0x1090,  0x17e0,
    0x1810,  0x1946,  0x19d0,  0x1a80,  0x1a90,  0x1b50,  0x1bb0,  0x1c40,  0x1c50,  0xa620,
    0xa8d0,  0xa900,  0xa9d0,  0xa9f0,  0xaa50,  0xabf0,  0xff10,  0x104a0, 0x10d30, 0x11066,
    0x110f0, 0x11136, 0x111d0, 0x112f0, 0x11450, 0x114d0, 0x11650, 0x116c0, 0x11730, 0x118e0,
    0x11950, 0x11c50, 0x11d50, 0x11da0, 0x11f50, 0x16a60, 0x16ac0, 0x16b50, 0x1d7ce, 0x1d7d8,
    0x1d7e2, 0x1d7ec, 0x1d7f6, 0x1e140, 0x1e2f0, 0x1e4f0, 0x1e950, 0x1fbf0};

// decimal value of a code point, or -1
int digit_of(uint32_t c) {
  if (c < 0x80) return (c >= '0' && c <= '9') ? (int)(c - '0') : -1;
  const uint32_t *e = kDigitZeros + sizeof(kDigitZeros) / sizeof(kDigitZeros[0]);
  const uint32_t *z = std::upper_bound(kDigitZeros, e, c);
  if (z == kDigitZeros) return -1;
  const uint32_t d = c - z[-1];
  return d < 10 ? (int)d : -1;
}

// str.isspace()
bool is_space(uint32_t c) {
  if (c < 0x80) return c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f);
  return c == 0x85 || c == 0xa0 || c == 0x1680 || (c >= 0x2000 && c <= 0x200a) ||
         c == 0x2028 || c == 0x2029 || c == 0x202f || c == 0x205f || c == 0x3000;
}

// str.splitlines() boundaries (\r\n is handled by the line cutter)
bool is_break(uint32_t c) {
  return c == '\n' || c == '\r' || c == 0x0b || c == 0x0c || c == 0x1c || c == 0x1d ||
         c == 0x1e || c == 0x85 || c == 0x2028 || c == 0x2029;
}

// Strict UTF-8 as Python's decoder: no overlong forms, no surrogates, at
// most U+10FFFF, no truncated sequences.
bool utf8_valid(const unsigned char *b, size_t n) {
  size_t i = 0;
  while (i < n) {
    const unsigned c = b[i];
    if (c < 0x80) { ++i; continue; }
    int len;
    unsigned lo = 0x80, hi = 0xbf;
    if (c >= 0xc2 && c <= 0xdf) len = 2;
    else if (c == 0xe0) { len = 3; lo = 0xa0; }
    else if (c == 0xed) { len = 3; hi = 0x9f; }
    else if (c >= 0xe1 && c <= 0xef) len = 3;
    else if (c == 0xf0) { len = 4; lo = 0x90; }
    else if (c == 0xf4) { len = 4; hi = 0x8f; }
    else if (c >= 0xf1 && c <= 0xf3) len = 4;
    else return false;
    if (i + (size_t)len > n) return false;
    if (b[i + 1] < lo || b[i + 1] > hi) return false;
    for (int k = 2; k < len; ++k)
      if (b[i + k] < 0x80 || b[i + k] > 0xbf) return false;
    i += (size_t)len;
  }
  return true;
}

// code point at p (valid UTF-8), its byte length in *len
uint32_t cp_at(const unsigned char *p, int *len) {
  const unsigned c = p[0];
  if (c < 0x80) { *len = 1; return c; }
  if (c < 0xe0) { *len = 2; return ((c & 0x1fu) << 6) | (p[1] & 0x3fu); }
  if (c < 0xf0) {
    *len = 3;
    return ((c & 0x0fu) << 12) | ((p[1] & 0x3fu) << 6) | (p[2] & 0x3fu);
  }
  *len = 4;
  return ((c & 0x07u) << 18) | ((p[1] & 0x3fu) << 12) | ((p[2] & 0x3fu) << 6) | (p[3] & 0x3fu);
}

// code point ending at e (valid UTF-8, e > s), its byte length in *len
uint32_t cp_before(const unsigned char *s, const unsigned char *e, int *len) {
  const unsigned char *p = e - 1;
  while (p > s && (*p & 0xc0) == 0x80) --p;
  return cp_at(p, len);
}

struct Span {
  const unsigned char *s, *e;
  bool empty() const { return s == e; }
};

Span strip(Span t) {
  int l;
  while (t.s < t.e && is_space(cp_at(t.s, &l))) t.s += l;
  while (t.e > t.s && is_space(cp_before(t.s, t.e, &l))) t.e -= l;
  return t;
}

// Next line of str.splitlines() starting at *p; false when none is left.
bool next_line(const unsigned char **p, const unsigned char *end, Span *line) {
  if (*p >= end) return false;
  const unsigned char *q = *p;
  while (q < end) {
    int l;
    const uint32_t c = cp_at(q, &l);
    if (is_break(c)) {
      *line = {*p, q};
      q += l;
      if (c == '\r' && q < end && *q == '\n') ++q;
      *p = q;
      return true;
    }
    q += l;
  }
  *line = {*p, end};
  *p = end;
  return true;
}

// The number's characters with decimal digits mapped to ASCII ('?' for any
// other non-ASCII code point, which no grammar accepts), as int()/float()
// see them after _PyUnicode_TransformDecimalAndSpaceToASCII.
std::string to_ascii(Span t) {
  std::string a;
  a.reserve((size_t)(t.e - t.s));
  for (const unsigned char *p = t.s; p < t.e;) {
    int l;
    const uint32_t c = cp_at(p, &l);
    p += l;
    if (c < 0x80) {
      a.push_back((char)c);
    } else {
      const int d = digit_of(c);
      a.push_back(d >= 0 ? (char)('0' + d) : '?');
    }
  }
  return a;
}

// digits with single underscores strictly between digits, from a[i]; returns
// the end index (== i when there is no digit) or -1 on a misplaced '_'
long digit_run(const std::string &a, size_t i, std::string *out, size_t *ndig) {
  size_t j = i;
  while (j < a.size()) {
    const char c = a[j];
    if (c >= '0' && c <= '9') {
      out->push_back(c);
      ++*ndig;
      ++j;
    } else if (c == '_') {
      if (j == i || j + 1 >= a.size() || a[j + 1] < '0' || a[j + 1] > '9') return -1;
      ++j;
    } else {
      break;
    }
  }
  return (long)j;
}

enum IntStatus { kIntOk, kIntBig, kIntBad };

// int(str) of a token without surrounding whitespace; *v its value when it
// fits int64 (kIntBig: valid but outside int64)
IntStatus py_int(Span t, int64_t *v) {
  const std::string a = to_ascii(t);
  size_t i = 0;
  bool neg = false;
  if (i < a.size() && (a[i] == '+' || a[i] == '-')) neg = a[i++] == '-';
  std::string dig;
  size_t nd = 0;
  const long j = digit_run(a, i, &dig, &nd);
  if (j < 0 || (size_t)j == i || (size_t)j != a.size() || nd > 4300) return kIntBad;
  // magnitude with overflow detection (|INT64_MIN| = 2^63 fits as negative)
  unsigned long long m = 0;
  bool big = false;
  for (char c : dig) {
    const unsigned d = (unsigned)(c - '0');
    if (m > (~0ull - d) / 10ull) { big = true; break; }
    m = m * 10ull + d;
  }
  if (!big && (neg ? m > (1ull << 63) : m > (unsigned long long)INT64_MAX)) big = true;
  if (big) return kIntBig;
  *v = neg ? (int64_t)(0ull - m) : (int64_t)m;
  return kIntOk;
}

bool ieq(const std::string &a, size_t i, const char *w) {
  const size_t n = strlen(w);
  if (a.size() - i != n) return false;
  for (size_t k = 0; k < n; ++k)
    if ((char)tolower((unsigned char)a[i + k]) != w[k]) return false;
  return true;
}

// float(str) of a token without surrounding whitespace
bool py_float(Span t, double *v) {
  const std::string a = to_ascii(t);
  size_t i = 0;
  bool neg = false;
  if (i < a.size() && (a[i] == '+' || a[i] == '-')) neg = a[i++] == '-';
  if (ieq(a, i, "inf") || ieq(a, i, "infinity")) {
    *v = neg ? -HUGE_VAL : HUGE_VAL;
    return true;
  }
  if (ieq(a, i, "nan")) {
    *v = neg ? -NAN : NAN;
    return true;
  }
  std::string num(neg ? "-" : "");
  size_t nd = 0, nfrac = 0;
  long j = digit_run(a, i, &num, &nd);
  if (j < 0) return false;
  size_t p = (size_t)j;
  if (p < a.size() && a[p] == '.') {
    num.push_back('.');
    j = digit_run(a, p + 1, &num, &nfrac);
    if (j < 0) return false;
    p = (size_t)j;
  }
  if (nd + nfrac == 0) return false;
  if (p < a.size() && (a[p] == 'e' || a[p] == 'E')) {
    num.push_back('e');
    ++p;
    if (p < a.size() && (a[p] == '+' || a[p] == '-')) num.push_back(a[p++]);
    size_t ne = 0;
    j = digit_run(a, p, &num, &ne);
    if (j < 0 || ne == 0) return false;
    p = (size_t)j;
  }
  if (p != a.size()) return false;
  errno = 0;
  char *end = nullptr;
  *v = strtod(num.c_str(), &end);  // correctly rounded; overflow -> +-inf like float()
  return end == num.c_str() + num.size();
}

// Error record of the last parse on this thread (glr_parse_status).
struct ParseStatus {
  int64_t kind = 0, lineno = 0, a = 0, b = 0;
};
thread_local ParseStatus g_status;

int fail(int64_t kind, int64_t lineno, int64_t a, int64_t b) {
  g_status = {kind, lineno, a, b};
  set_error("glr_parse: error kind %lld at line %lld", (long long)kind, (long long)lineno);
  return GLR_EPARSE;
}

int64_t off(const unsigned char *base, const unsigned char *p) { return (int64_t)(p - base); }

}  // namespace
}  // namespace glr

extern "C" {

int glr_parse_status(int64_t *info) {
  if (info == nullptr) return GLR_EARG;
  info[0] = glr::g_status.kind;
  info[1] = glr::g_status.lineno;
  info[2] = glr::g_status.a;
  info[3] = glr::g_status.b;
  return GLR_OK;
}

int glr_parse_edgelist(const char *buf, size_t len, int64_t *out, int64_t cap, int64_t *count) {
  using namespace glr;
  if ((buf == nullptr && len > 0) || count == nullptr || cap < 0) {
    set_error("glr_parse_edgelist: invalid arguments");
    return GLR_EARG;
  }
  g_status = ParseStatus{};
  const unsigned char *b = reinterpret_cast<const unsigned char *>(buf), *end = b + len;
  if (!utf8_valid(b, len)) return fail(GLR_PARSE_UTF8, 0, 0, 0);
  int64_t n = 0, lineno = 0, big_line = 0;
  const unsigned char *p = b;
  Span line;
  while (next_line(&p, end, &line)) {
    ++lineno;
    const Span t = strip(line);
    if (t.empty() || *t.s == '#') continue;
    // whitespace-separated tokens (str.split()): exactly two
    Span tok[3];
    int nt = 0;
    for (const unsigned char *q = t.s; q < t.e && nt < 3;) {
      int l;
      while (q < t.e && is_space(cp_at(q, &l))) q += l;
      if (q >= t.e) break;
      const unsigned char *s0 = q;
      while (q < t.e && !is_space(cp_at(q, &l))) q += l;
      tok[nt++] = {s0, q};
    }
    if (nt != 2) return fail(GLR_PARSE_TOKENS, lineno, off(b, t.s), off(b, t.e));
    int64_t v[2];
    IntStatus st[2];
    for (int k = 0; k < 2; ++k) {
      st[k] = py_int(tok[k], &v[k]);
      if (st[k] == kIntBad) return fail(GLR_PARSE_NOT_INT, lineno, off(b, t.s), off(b, t.e));
    }
    for (int k = 0; k < 2; ++k) {
      const bool negative = st[k] == kIntBig ? *to_ascii(tok[k]).c_str() == '-' : v[k] < 0;
      if (negative) return fail(GLR_PARSE_NEGATIVE, lineno, 0, 0);
    }
    if (st[0] == kIntBig || st[1] == kIntBig) {
      // normalize_edges' int64 conversion fails only after the whole file
      if (big_line == 0) big_line = lineno;
    } else if (out != nullptr && n < cap) {
      out[2 * n] = v[0];
      out[2 * n + 1] = v[1];
    }
    ++n;
  }
  if (n == 0) return fail(GLR_PARSE_NO_EDGES, 0, 0, 0);
  if (big_line) return fail(GLR_PARSE_OVERFLOW, big_line, 0, 0);
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
  g_status = ParseStatus{};
  const unsigned char *b = reinterpret_cast<const unsigned char *>(buf), *end = b + len;
  if (!utf8_valid(b, len)) return fail(GLR_PARSE_UTF8, 0, 0, 0);
  const unsigned char *p = b;
  Span line;
  if (!next_line(&p, end, &line)) return fail(GLR_PARSE_EMPTY_LAYOUT, 0, 0, 0);
  {  // header: the comma-separated fields, stripped, are exactly id, x, y
    const char *want[3] = {"id", "x", "y"};
    int k = 0;
    bool ok = true;
    const unsigned char *f = line.s;
    for (const unsigned char *q = line.s;; ++q) {
      if (q == line.e || *q == ',') {
        const Span fs = strip({f, q});
        ok = ok && k < 3 && (size_t)(fs.e - fs.s) == strlen(want[k]) &&
             memcmp(fs.s, want[k], (size_t)(fs.e - fs.s)) == 0;
        ++k;
        f = q + 1;
        if (q == line.e) break;
      }
    }
    if (!ok || k != 3) return fail(GLR_PARSE_HEADER, 1, off(b, line.s), off(b, line.e));
  }
  // rows up to the first failing one; duplicates are resolved afterwards
  std::vector<int64_t> rid, rline;
  int64_t lineno = 1, err_kind = 0, err_line = 0, big_line = 0;
  Span err_span{b, b};
  while (next_line(&p, end, &line)) {
    ++lineno;
    if (strip(line).empty()) continue;
    Span part[3];
    int k = 0;
    const unsigned char *f = line.s;
    for (const unsigned char *q = line.s;; ++q) {
      if (q == line.e || *q == ',') {
        if (k < 3) part[k] = strip({f, q});
        ++k;
        f = q + 1;
        if (q == line.e) break;
      }
    }
    if (k != 3) {
      err_kind = GLR_PARSE_FIELDS;
      err_line = lineno;
      err_span = line;
      break;
    }
    int64_t vid = 0;
    double x, y;
    const IntStatus st = py_int(part[0], &vid);
    if (st == kIntBad || !py_float(part[1], &x) || !py_float(part[2], &y)) {
      err_kind = GLR_PARSE_MALFORMED;
      err_line = lineno;
      err_span = line;
      break;
    }
    if (!std::isfinite(x) || !std::isfinite(y)) {
      err_kind = GLR_PARSE_NONFINITE;
      err_line = lineno;
      break;
    }
    if (st == kIntBig) {  // a valid Python int that no int64 id array holds
      if (big_line == 0) big_line = lineno;
      continue;
    }
    const int64_t r = (int64_t)rid.size();
    if (ids != nullptr && r < cap) {
      ids[r] = vid;
      xy[2 * r] = x;
      xy[2 * r + 1] = y;
    }
    rid.push_back(vid);
    rline.push_back(lineno);
  }
  // the first repeated id in file order (it precedes any failing row)
  int64_t dup_line = 0, dup_id = 0;
  if (rid.size() > 1) {
    std::vector<int64_t> ord(rid.size());
    for (size_t i = 0; i < ord.size(); ++i) ord[i] = (int64_t)i;
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t c) { return rid[a] < rid[c]; });
    for (size_t i = 1; i < ord.size(); ++i)
      if (rid[ord[i]] == rid[ord[i - 1]] && (dup_line == 0 || rline[ord[i]] < dup_line)) {
        dup_line = rline[ord[i]];
        dup_id = rid[ord[i]];
      }
  }
  if (dup_line) return fail(GLR_PARSE_DUPLICATE, dup_line, dup_id, 0);
  if (err_kind) return fail(err_kind, err_line, off(b, err_span.s), off(b, err_span.e));
  if (rid.empty() && big_line == 0) return fail(GLR_PARSE_NO_ROWS, 0, 0, 0);
  if (big_line) return fail(GLR_PARSE_OVERFLOW, big_line, 0, 0);
  *count = (int64_t)rid.size();
  return GLR_OK;
}

}  // extern "C"
