// mm.cu -- Matrix Market ingest (io.hpp:38-123 parse_matrix_market) on the
// host, feeding the device CSR build (graph.cu graph_from_edges, the
// build_csr layout of graph.hpp:132-162).  Same acceptance rules, same error
// lines and messages as the reference:
//   header '%%MatrixMarket matrix coordinate <real|integer|pattern>
//   <general|symmetric>' (:56-71), comments and blank lines skipped, size
//   line (:73-86, square only), entries 1-based (:93-117; pattern -> weight
//   1.0, force_unit_weights, finite and non-negative weights, bounds,
//   symmetric mirroring of off-diagonal entries when expand_symmetric), the
//   declared entry count (:107-111, :118-121).
// Numbers are parsed with std::from_chars (the reference uses istream >>,
// which agrees on every well-formed decimal; both round-to-nearest).
#include <charconv>
#include <cmath>
#include <cstring>
#include <limits>
#include <type_traits>
#include <string>
#include <vector>

#include "impl.hpp"

namespace gfb {

struct EdgeList {
  uint64_t n = 0;
  std::vector<uint32_t> src, dst;
  std::vector<double> w;
};

thread_local uint64_t g_parse_line = 0;

[[noreturn]] static void parse_error(uint64_t line, const std::string& what) {
  g_parse_line = line;
  fail(GFB_EPARSE, "line " + std::to_string(line) + ": " + what);
}

namespace {

struct Cursor {
  const char* p;
  const char* end;
  uint64_t lineno = 0;
  const char* ls = nullptr;  // current line [ls, le)
  const char* le = nullptr;
  bool next_line() {
    if (p >= end) return false;
    ls = p;
    const void* nl = std::memchr(p, '\n', (size_t)(end - p));
    le = nl ? static_cast<const char*>(nl) : end;
    p = nl ? le + 1 : end;
    ++lineno;
    return true;
  }
};

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// whitespace-separated tokens of [a, b), like istream >> std::string
struct Tokens {
  const char* a;
  const char* b;
  bool next(const char** ts, const char** te) {
    while (a < b && is_space(*a)) ++a;
    if (a >= b) return false;
    *ts = a;
    while (a < b && !is_space(*a)) ++a;
    *te = a;
    return true;
  }
  template <class T>
  bool num(T* out) {  // istream >> T: leading whitespace, then a number
    while (a < b && is_space(*a)) ++a;
    if (a >= b) return false;
    const char* s = a;
    if constexpr (std::is_floating_point_v<T>) {
      if (*s == '+') ++s;  // from_chars rejects a leading '+', istream accepts it
      // istream >> double takes decimal numbers only (no inf / nan / hex)
      const char* q = (s < b && *s == '-') ? s + 1 : s;
      if (q >= b || !((*q >= '0' && *q <= '9') || *q == '.')) return false;
      auto r = std::from_chars(s, b, *out);
      if (r.ec != std::errc()) return false;
      a = r.ptr;
      return true;
    } else {
      // istream >> integer: optional sign; an unsigned target takes '-' and
      // negates modulo 2^N (strtoull semantics, as libstdc++'s num_get)
      bool neg = false;
      if (*s == '+' || *s == '-') {
        neg = *s == '-';
        ++s;
      }
      if (s >= b || *s < '0' || *s > '9') return false;
      std::make_unsigned_t<T> u = 0;
      auto r = std::from_chars(s, b, u);
      if (r.ec != std::errc()) return false;
      if constexpr (std::is_signed_v<T>) {
        const auto lim = (std::make_unsigned_t<T>)std::numeric_limits<T>::max();
        if (u > lim + (neg ? 1u : 0u)) return false;  // out of range: failbit
        *out = neg ? (T)(0 - u) : (T)u;
      } else {
        *out = neg ? (T)(0 - u) : u;
      }
      a = r.ptr;
      return true;
    }
  }
};

}  // namespace

EdgeList* mm_parse(const char* text, size_t len, bool force_unit, bool expand_symmetric) {
  Cursor c{text, text + len};
  if (!c.next_line()) parse_error(1, "empty input");  // io.hpp:56
  std::string tok[5];
  {
    Tokens t{c.ls, c.le};
    for (auto& s : tok) {
      const char *a, *b;
      if (t.next(&a, &b)) s.assign(a, b);
    }
  }
  if (tok[0] != "%%MatrixMarket" || tok[1] != "matrix" || tok[2] != "coordinate")
    parse_error(c.lineno, "malformed header, expected '%%MatrixMarket matrix coordinate ...'");
  const bool pattern = tok[3] == "pattern";
  if (tok[3] != "real" && tok[3] != "integer" && !pattern)
    parse_error(c.lineno, "unsupported field type '" + tok[3] + "'");
  const bool symmetric = tok[4] == "symmetric";
  if (tok[4] != "general" && !symmetric)
    parse_error(c.lineno, "unsupported symmetry '" + tok[4] + "'");
  unsigned long long rows = 0, cols = 0, declared = 0;
  for (;;) {  // size line, after comments (io.hpp:73-82)
    if (!c.next_line()) parse_error(c.lineno + 1, "missing size line");
    if (c.ls == c.le || *c.ls == '%') continue;
    Tokens t{c.ls, c.le};
    if (!(t.num(&rows) && t.num(&cols) && t.num(&declared)))
      parse_error(c.lineno, "malformed size line");
    break;
  }
  if (rows != cols)
    parse_error(c.lineno, "rectangular matrix (" + std::to_string(rows) + "x" +
                              std::to_string(cols) + "), graphs must be square");
  if (rows >= (1ull << 32)) parse_error(c.lineno, "more than 2^32 - 1 vertices");
  auto el = std::make_unique<EdgeList>();
  el->n = rows;
  const size_t reserve = (size_t)std::min<unsigned long long>(declared, 1ull << 28);
  el->src.reserve(reserve);
  el->dst.reserve(reserve);
  el->w.reserve(reserve);
  unsigned long long found = 0;
  while (c.next_line()) {  // io.hpp:93-117
    if (c.ls == c.le || *c.ls == '%') continue;
    Tokens t{c.ls, c.le};
    long long i = 0, j = 0;
    double w = 1.0;
    if (!(t.num(&i) && t.num(&j))) parse_error(c.lineno, "malformed entry");
    if (!pattern && !t.num(&w)) parse_error(c.lineno, "entry missing value");
    if (i < 1 || (unsigned long long)i > rows || j < 1 || (unsigned long long)j > cols)
      parse_error(c.lineno, "index out of declared bounds");
    if (force_unit) w = 1.0;
    if (!std::isfinite(w)) parse_error(c.lineno, "non-finite weight");
    if (w < 0) parse_error(c.lineno, "negative weight");
    ++found;
    if (found > declared)
      parse_error(c.lineno, "entry count mismatch: header declares " + std::to_string(declared) +
                                " entries, found more");
    const uint32_t s = (uint32_t)(i - 1), d = (uint32_t)(j - 1);
    el->src.push_back(s);
    el->dst.push_back(d);
    el->w.push_back(w);
    if (symmetric && expand_symmetric && s != d) {
      el->src.push_back(d);
      el->dst.push_back(s);
      el->w.push_back(w);
    }
  }
  if (found != declared)
    parse_error(c.lineno, "entry count mismatch: header declares " + std::to_string(declared) +
                              " entries, found " + std::to_string(found));
  return el.release();
}

void edge_list_free(EdgeList* e) { delete e; }
void edge_list_info(const EdgeList* e, uint64_t* n, uint64_t* m) {
  if (n) *n = e->n;
  if (m) *m = e->src.size();
}
void edge_list_read(const EdgeList* e, uint32_t* src, uint32_t* dst, double* w) {
  const size_t m = e->src.size();
  if (src && m) std::memcpy(src, e->src.data(), m * 4);
  if (dst && m) std::memcpy(dst, e->dst.data(), m * 4);
  if (w && m) std::memcpy(w, e->w.data(), m * 8);
}
const uint32_t* edge_list_src(const EdgeList* e) { return e->src.data(); }
const uint32_t* edge_list_dst(const EdgeList* e) { return e->dst.data(); }
const double* edge_list_w(const EdgeList* e) { return e->w.data(); }
uint64_t parse_error_line() { return g_parse_line; }

}  // namespace gfb
