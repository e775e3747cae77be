// SPDX-License-Identifier: Apache-2.0
//
// On-disk formats of the reference (rowgcn, inc/dataset.hpp:84-280 and inc/dense.hpp:290-335), restated
// as multi-threaded native loaders so real ogbn / Reddit graphs flow through the drop-in:
//   * Matrix Market coordinate files (real | integer | pattern, general | symmetric)  dataset.hpp:87-143
//   * whitespace edge lists "u v [w]" with '#' comments                                dataset.hpp:147-168
//   * load_graph format sniffing                                                       dataset.hpp:170-180
//   * features: MGDM dense binary or CSV rows                                           dataset.hpp:184-216
//   * labels (one integer per line)                                                     dataset.hpp:218-234
//   * masks JSON sidecar {"train": [ids], "val": [ids], "test": [ids]}                  dataset.hpp:237-262
//   * load_dataset                                                                      dataset.hpp:264-276
//   * write_dense / read_dense (MGDM)                                                   dense.hpp:293-335
//   * from_coo (sorted rows, duplicate (src, dst) weights summed)                       sparse.hpp:59-90
// Files are read whole and parsed in line-aligned chunks on host_threads() threads; the first error in
// file order wins and carries the reference's "path:line: ..." message and exception type. Number
// syntax follows the reference's extractors (std::istream >> int64 / double, std::stod, std::stol).
// One deliberate difference: duplicate edges are summed in file order (the reference's std::sort is not
// stable, so with three or more differing duplicate weights its float sum order is unspecified).
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <map>
#include <memory>
#include <mutex>

#include "mg_internal.hpp"

namespace mg {

namespace io {

std::string read_file(const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw IoError("cannot open " + path);
  std::string buf;
  std::fseek(f, 0, SEEK_END);
  const long size = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  if (size > 0) {
    buf.resize(static_cast<size_t>(size));
    const size_t got = std::fread(&buf[0], 1, buf.size(), f);
    buf.resize(got);
  }
  std::fclose(f);
  return buf;
}

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }
inline bool is_digit(char c) { return c >= '0' && c <= '9'; }

// std::istream >> int64 (num_get): skip whitespace, [+-]digits; no digits or overflow = failure.
bool scan_int(const char*& p, const char* e, index_t& out) {
  while (p < e && is_space(*p)) ++p;
  const char* q = p;
  bool neg = false;
  if (q < e && (*q == '+' || *q == '-')) neg = *q++ == '-';
  if (q >= e || !is_digit(*q)) return false;
  unsigned long long v = 0;
  bool overflow = false;
  while (q < e && is_digit(*q)) {
    const unsigned d = static_cast<unsigned>(*q++ - '0');
    if (v > (std::numeric_limits<unsigned long long>::max() - d) / 10) overflow = true;
    else v = v * 10 + d;
  }
  p = q;
  const unsigned long long lim = neg ? 9223372036854775808ull : 9223372036854775807ull;
  if (overflow || v > lim) return false;
  out = neg ? static_cast<index_t>(0 - v) : static_cast<index_t>(v);
  return true;
}

// std::istream >> double (libstdc++ num_get::_M_extract_float + strtod): skip whitespace, collect
// [+-] digits [. digits] [(e|E) [+-] digits] (the exponent only after a mantissa digit), convert the
// collected text with strtod; an empty / unconvertible text or an overflow is a failure with value 0.
enum class Scan { kOk, kEof, kFail };
Scan scan_double(const char*& p, const char* e, double& out) {
  while (p < e && is_space(*p)) ++p;
  if (p >= e) return Scan::kEof;
  char buf[512];
  int n = 0;
  const char* q = p;
  bool mant = false, dot = false;
  auto put = [&](char c) {
    if (n < 510) buf[n++] = c;
  };
  if (q < e && (*q == '+' || *q == '-')) put(*q++);
  while (q < e) {
    const char c = *q;
    if (is_digit(c)) {
      mant = true;
      put(c);
      ++q;
    } else if (c == '.' && !dot) {
      dot = true;
      put(c);
      ++q;
    } else {
      break;
    }
  }
  if (mant && q < e && (*q == 'e' || *q == 'E')) {
    put(*q++);
    if (q < e && (*q == '+' || *q == '-')) put(*q++);
    while (q < e && is_digit(*q)) put(*q++);
  }
  p = q;
  buf[n] = 0;
  char* end = nullptr;
  const double v = std::strtod(buf, &end);
  if (n == 0 || end != buf + n) {
    out = 0.0;
    return Scan::kFail;
  }
  if (std::isinf(v)) {  // overflow: failbit with the value clamped to +-max
    out = std::copysign(std::numeric_limits<double>::max(), v);
    return Scan::kFail;
  }
  out = v;
  return Scan::kOk;
}

// Line-aligned chunking of [b, e) for the parallel parsers.
std::vector<std::pair<const char*, const char*>> chunks(const char* b, const char* e, size_t min_bytes = 1 << 20) {
  std::vector<std::pair<const char*, const char*>> out;
  const size_t bytes = static_cast<size_t>(e - b);
  const int t = static_cast<int>(std::max<size_t>(1, std::min<size_t>(host_threads() * 4, bytes / min_bytes)));
  const char* s = b;
  for (int i = 1; i <= t && s < e; ++i) {
    const char* c = i == t ? e : b + bytes * i / t;
    if (c < s) c = s;
    while (c < e && c[-1] != '\n') ++c;  // chunk ends just after a newline
    out.emplace_back(s, c);
    s = c;
  }
  if (out.empty()) out.emplace_back(b, e);
  return out;
}

template <class F>
void run_chunks(size_t n, F&& f) {
  parallel_for(static_cast<index_t>(n), [&](index_t b, index_t e) {
    for (index_t i = b; i < e; ++i) f(static_cast<size_t>(i));
  }, 1);
}

size_t line_number(const char* base, const char* at) {  // 1-based
  size_t n = 1;
  for (const char* p = base; p < at; ++p) n += *p == '\n';
  return n;
}

struct ChunkError {
  const char* line = nullptr;  // start of the failing line (null = none)
  int code = 0;
  std::string detail;
};

struct Coo {
  std::vector<index_t> src, dst;
  std::vector<float> w;
  void push(index_t s, index_t d, float x) {
    src.push_back(s);
    dst.push_back(d);
    w.push_back(x);
  }
  size_t size() const { return src.size(); }
};

// sparse.hpp:59-90. Counting sort by source (stable), per-row sort by (dst, file order), duplicates summed.
Csr from_coo(std::vector<Coo>& parts, index_t n) {
  Csr m;
  m.rows = m.cols = n;
  m.row_ptr.assign(static_cast<size_t>(n) + 1, 0);
  size_t total = 0;
  for (auto& c : parts) total += c.size();
  for (auto& c : parts)
    for (size_t i = 0; i < c.size(); ++i) {
      if (c.src[i] < 0 || c.src[i] >= n || c.dst[i] < 0 || c.dst[i] >= n)
        throw ValueError("from_coo: edge (" + std::to_string(c.src[i]) + ", " + std::to_string(c.dst[i]) +
                         ") out of range for n=" + std::to_string(n));
      m.row_ptr[static_cast<size_t>(c.src[i]) + 1]++;
    }
  for (index_t u = 0; u < n; ++u) m.row_ptr[u + 1] += m.row_ptr[u];
  std::vector<index_t> col(total);
  std::vector<float> val(total);
  {
    std::vector<index_t> fill(m.row_ptr.begin(), m.row_ptr.end() - 1);
    for (auto& c : parts) {
      for (size_t i = 0; i < c.size(); ++i) {
        const index_t pos = fill[static_cast<size_t>(c.src[i])]++;
        col[static_cast<size_t>(pos)] = c.dst[i];
        val[static_cast<size_t>(pos)] = c.w[i];
      }
      std::vector<index_t>().swap(c.src);
      std::vector<index_t>().swap(c.dst);
      std::vector<float>().swap(c.w);
    }
  }
  // per row: stable sort by column, merge duplicates; then compact
  std::vector<index_t> kept(static_cast<size_t>(n), 0);
  parallel_for(n, [&](index_t b, index_t e) {
    std::vector<std::pair<index_t, float>> tmp;
    for (index_t u = b; u < e; ++u) {
      const index_t r0 = m.row_ptr[u], r1 = m.row_ptr[u + 1];
      tmp.clear();
      bool sorted = true;
      for (index_t i = r0; i < r1; ++i) {
        if (i > r0 && col[i] <= col[i - 1]) sorted = false;
        tmp.emplace_back(col[i], val[i]);
      }
      if (sorted) {
        kept[u] = r1 - r0;
        continue;
      }
      std::stable_sort(tmp.begin(), tmp.end(), [](const auto& a, const auto& b2) { return a.first < b2.first; });
      index_t o = r0;
      for (size_t i = 0; i < tmp.size();) {
        const index_t v = tmp[i].first;
        float w = tmp[i].second;
        ++i;
        while (i < tmp.size() && tmp[i].first == v) w += tmp[i++].second;
        col[o] = v;
        val[o] = w;
        ++o;
      }
      kept[u] = o - r0;
    }
  }, 4096);
  std::vector<index_t> rp(static_cast<size_t>(n) + 1, 0);
  for (index_t u = 0; u < n; ++u) rp[u + 1] = rp[u] + kept[u];
  if (rp[n] == static_cast<index_t>(total)) {
    m.col_idx = std::move(col);
    m.values = std::move(val);
  } else {
    m.col_idx.resize(static_cast<size_t>(rp[n]));
    m.values.resize(static_cast<size_t>(rp[n]));
    parallel_for(n, [&](index_t b, index_t e) {
      for (index_t u = b; u < e; ++u) {
        std::copy(col.begin() + m.row_ptr[u], col.begin() + m.row_ptr[u] + kept[u], m.col_idx.begin() + rp[u]);
        std::copy(val.begin() + m.row_ptr[u], val.begin() + m.row_ptr[u] + kept[u], m.values.begin() + rp[u]);
      }
    }, 4096);
  }
  m.row_ptr = std::move(rp);
  return m;
}

const char* line_end(const char* p, const char* e) {
  const void* nl = std::memchr(p, '\n', static_cast<size_t>(e - p));
  return nl ? static_cast<const char*>(nl) : e;
}

// dataset.hpp:87-143
Csr load_matrix_market(const std::string& path) {
  const std::string text = read_file(path);
  const char* b = text.data();
  const char* e = b + text.size();
  if (text.empty()) throw ParseError(path + ":1: empty file");
  const char* p = b;
  const char* le = line_end(p, e);
  {
    std::string banner, object, format, field, symmetry;
    std::string hdr(p, le);
    size_t i = 0;
    auto tok = [&](std::string& out) {
      while (i < hdr.size() && is_space(hdr[i])) ++i;
      const size_t s = i;
      while (i < hdr.size() && !is_space(hdr[i])) ++i;
      out = hdr.substr(s, i - s);
    };
    tok(banner), tok(object), tok(format), tok(field), tok(symmetry);
    if (banner != "%%MatrixMarket" || object != "matrix" || format != "coordinate")
      throw ParseError(path + ":1: expected '%%MatrixMarket matrix coordinate ...' header");
    const bool pattern = field == "pattern";
    if (!pattern && field != "real" && field != "integer")
      throw ParseError(path + ":1: unsupported field '" + field + "'");
    const bool symmetric = symmetry == "symmetric";
    if (!symmetric && symmetry != "general")
      throw ParseError(path + ":1: unsupported symmetry '" + symmetry + "'");
    // size line
    index_t rows = 0, cols = 0, entries = -1;
    p = le < e ? le + 1 : e;
    while (p < e) {
      const char* l0 = p;
      le = line_end(p, e);
      p = le < e ? le + 1 : e;
      if (l0 == le || *l0 == '%') continue;
      const char* q = l0;
      index_t r, c, n;
      if (!scan_int(q, le, r) || !scan_int(q, le, c) || !scan_int(q, le, n))
        throw ParseError(path + ":" + std::to_string(line_number(b, l0)) + ": bad size line");
      rows = r, cols = c, entries = n;
      break;
    }
    if (entries < 0) throw ParseError(path + ": missing size line");
    // entries, parsed in parallel chunks
    auto parts = chunks(p, e);
    std::vector<Coo> coo(parts.size());
    std::vector<ChunkError> err(parts.size());
    std::vector<index_t> seen(parts.size(), 0);
    run_chunks(parts.size(), [&](size_t ci) {
      const char* s = parts[ci].first;
      const char* ce = parts[ci].second;
      Coo& out = coo[ci];
      while (s < ce) {
        const char* l0 = s;
        const char* l1 = line_end(s, ce);
        s = l1 < ce ? l1 + 1 : ce;
        if (l0 == l1 || *l0 == '%') continue;
        const char* q = l0;
        index_t u, v;
        double w = 1.0;
        if (!scan_int(q, l1, u) || !scan_int(q, l1, v)) {
          err[ci] = {l0, 1, ""};
          return;
        }
        if (!pattern && scan_double(q, l1, w) != Scan::kOk) {
          err[ci] = {l0, 2, ""};
          return;
        }
        if (u < 1 || u > rows || v < 1 || v > cols) {
          err[ci] = {l0, 3, "(" + std::to_string(u) + ", " + std::to_string(v) + ")"};
          return;
        }
        out.push(u - 1, v - 1, static_cast<float>(w));
        if (symmetric && u != v) out.push(v - 1, u - 1, static_cast<float>(w));
        ++seen[ci];
      }
    });
    for (size_t ci = 0; ci < parts.size(); ++ci) {
      if (!err[ci].line) continue;
      const std::string at = path + ":" + std::to_string(line_number(b, err[ci].line)) + ": ";
      if (err[ci].code == 1) throw ParseError(at + "bad entry");
      if (err[ci].code == 2) throw ParseError(at + "missing value");
      throw ParseError(at + "index " + err[ci].detail + " out of bounds");
    }
    index_t total = 0;
    for (index_t s : seen) total += s;
    if (total != entries)
      throw ParseError(path + ": header promised " + std::to_string(entries) + " entries, found " +
                       std::to_string(total));
    if (rows != cols) throw ParseError(path + ": adjacency must be square, got " + shape_str(rows, cols));
    return from_coo(coo, rows);
  }
}

// dataset.hpp:147-168
Csr load_edge_list(const std::string& path) {
  const std::string text = read_file(path);
  const char* b = text.data();
  const char* e = b + text.size();
  auto parts = chunks(b, e);
  std::vector<Coo> coo(parts.size());
  std::vector<ChunkError> err(parts.size());
  std::vector<index_t> nmax(parts.size(), 0);
  run_chunks(parts.size(), [&](size_t ci) {
    const char* s = parts[ci].first;
    const char* ce = parts[ci].second;
    Coo& out = coo[ci];
    index_t n = 0;
    while (s < ce) {
      const char* l0 = s;
      const char* l1 = line_end(s, ce);
      s = l1 < ce ? l1 + 1 : ce;
      const char* q = l0;
      while (q < l1 && (*q == ' ' || *q == '\t' || *q == '\r')) ++q;
      if (q == l1 || *q == '#') continue;
      q = l0;
      index_t u, v;
      double w = 1.0;
      if (!scan_int(q, l1, u) || !scan_int(q, l1, v)) {
        err[ci] = {l0, 1, ""};
        return;
      }
      // `ls >> w`: absent (end of line) keeps 1.0, an unparsable token yields 0 (failbit, value 0)
      if (scan_double(q, l1, w) == Scan::kEof) w = 1.0;
      if (u < 0 || v < 0) {
        err[ci] = {l0, 2, ""};
        return;
      }
      n = std::max({n, u + 1, v + 1});
      out.push(u, v, static_cast<float>(w));
    }
    nmax[ci] = n;
  });
  index_t n = 0;
  for (size_t ci = 0; ci < parts.size(); ++ci) {
    if (err[ci].line) {
      const std::string at = path + ":" + std::to_string(line_number(b, err[ci].line)) + ": ";
      throw ParseError(at + (err[ci].code == 1 ? "expected 'u v [w]'" : "negative vertex id"));
    }
    n = std::max(n, nmax[ci]);
  }
  return from_coo(coo, n);
}

// dataset.hpp:170-180: Matrix Market when the first line starts with the banner, else an edge list.
Csr load_graph(const std::string& path, int format) {
  if (format == 1) return load_matrix_market(path);
  if (format == 2) return load_edge_list(path);
  if (format != 0) throw ValueError("load_graph: unknown format " + std::to_string(format));
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw IoError("cannot open " + path);
  char head[15] = {0};
  const size_t got = std::fread(head, 1, 14, f);
  std::fclose(f);
  if (got == 14 && std::memcmp(head, "%%MatrixMarket", 14) == 0) return load_matrix_market(path);
  return load_edge_list(path);
}

struct Dense {
  index_t rows = 0, cols = 0;
  std::vector<float> data;
};

// dense.hpp:311-335 (S = float: a width-8 payload is converted element-wise)
Dense read_dense(const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw IoError("cannot open " + path);
  std::unique_ptr<std::FILE, int (*)(std::FILE*)> guard(f, std::fclose);
  char magic[4];
  if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "MGDM", 4) != 0)
    throw ParseError(path + ": bad magic, not a dense binary file");
  std::uint64_t r = 0, c = 0;
  std::uint8_t w = 0;
  const bool ok = std::fread(&r, 8, 1, f) == 1 && std::fread(&c, 8, 1, f) == 1 && std::fread(&w, 1, 1, f) == 1;
  if (!ok || (w != 4 && w != 8)) throw ParseError(path + ": bad dtype width " + std::to_string(w));
  Dense m;
  m.rows = static_cast<index_t>(r);
  m.cols = static_cast<index_t>(c);
  const size_t count = static_cast<size_t>(r * c);
  m.data.resize(count);
  bool full;
  if (w == 4) {
    full = std::fread(m.data.data(), 4, count, f) == count;
  } else {
    std::vector<double> tmp(count);
    full = std::fread(tmp.data(), 8, count, f) == count;
    for (size_t i = 0; i < count; ++i) m.data[i] = static_cast<float>(tmp[i]);
  }
  if (!full) throw ParseError(path + ": truncated payload for " + shape_str(m.rows, m.cols));
  return m;
}

// dense.hpp:293-307
void write_dense(const std::string& path, index_t rows, index_t cols, const float* data) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw IoError("cannot open " + path + " for writing");
  std::unique_ptr<std::FILE, int (*)(std::FILE*)> guard(f, std::fclose);
  const std::uint64_t r = static_cast<std::uint64_t>(rows), c = static_cast<std::uint64_t>(cols);
  const std::uint8_t w = 4;
  const size_t count = static_cast<size_t>(rows * cols);
  bool ok = std::fwrite("MGDM", 1, 4, f) == 4 && std::fwrite(&r, 8, 1, f) == 1 && std::fwrite(&c, 8, 1, f) == 1 &&
            std::fwrite(&w, 1, 1, f) == 1;
  ok = ok && (count == 0 || std::fwrite(data, 4, count, f) == count);
  ok = ok && std::fflush(f) == 0;
  if (!ok) throw IoError("short write to " + path);
}

// std::stod on one CSV cell: strtod semantics (leading whitespace, trailing text ignored); no
// conversion or ERANGE is an error.
bool stod_cell(const char* s, const char* e, double& out) {
  char small[128];
  std::string big;
  const size_t len = static_cast<size_t>(e - s);
  const char* z;
  if (len < sizeof(small)) {
    std::memcpy(small, s, len);
    small[len] = 0;
    z = small;
  } else {
    big.assign(s, len);
    z = big.c_str();
  }
  char* end = nullptr;
  errno = 0;
  const double v = std::strtod(z, &end);
  if (end == z || errno == ERANGE) return false;
  out = v;
  return true;
}

// dataset.hpp:184-216
Dense load_features(const std::string& path) {
  {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw IoError("cannot open " + path);
    char magic[4] = {0, 0, 0, 0};
    const size_t got = std::fread(magic, 1, 4, f);
    std::fclose(f);
    if (got == 4 && std::memcmp(magic, "MGDM", 4) == 0) return read_dense(path);
  }
  const std::string text = read_file(path);
  const char* b = text.data();
  const char* e = b + text.size();
  auto parts = chunks(b, e);
  struct Part {
    std::vector<float> vals;
    std::vector<index_t> row_cols;  // columns of each row
  };
  std::vector<Part> out(parts.size());
  std::vector<ChunkError> err(parts.size());
  run_chunks(parts.size(), [&](size_t ci) {
    const char* s = parts[ci].first;
    const char* ce = parts[ci].second;
    Part& o = out[ci];
    while (s < ce) {
      const char* l0 = s;
      const char* l1 = line_end(s, ce);
      s = l1 < ce ? l1 + 1 : ce;
      if (l0 == l1) continue;
      index_t ncol = 0;
      const char* c = l0;
      while (true) {  // getline(ls, cell, ','): a trailing ',' does not start another cell
        const void* comma = std::memchr(c, ',', static_cast<size_t>(l1 - c));
        const char* ce2 = comma ? static_cast<const char*>(comma) : l1;
        double v;
        if (!stod_cell(c, ce2, v)) {
          err[ci] = {l0, 1, std::string(c, ce2)};
          return;
        }
        o.vals.push_back(static_cast<float>(v));
        ++ncol;
        if (!comma || ce2 + 1 == l1) break;
        c = ce2 + 1;
      }
      o.row_cols.push_back(ncol);
    }
  });
  index_t cols = -1, rows = 0;
  for (size_t ci = 0; ci < parts.size(); ++ci) {
    for (size_t r = 0; r < out[ci].row_cols.size(); ++r) {
      if (cols < 0) cols = out[ci].row_cols[r];
      if (out[ci].row_cols[r] != cols) {
        // locate the r-th non-empty line of this chunk for the message
        const char* s = parts[ci].first;
        size_t seen = 0;
        const char* at = s;
        while (s < parts[ci].second) {
          const char* l1 = line_end(s, parts[ci].second);
          if (l1 != s) {
            if (seen == r) {
              at = s;
              break;
            }
            ++seen;
          }
          s = l1 < parts[ci].second ? l1 + 1 : parts[ci].second;
        }
        throw ParseError(path + ":" + std::to_string(line_number(b, at)) + ": row has " +
                         std::to_string(out[ci].row_cols[r]) + " columns, expected " + std::to_string(cols));
      }
      ++rows;
    }
    if (err[ci].line)
      throw ParseError(path + ":" + std::to_string(line_number(b, err[ci].line)) + ": bad number '" + err[ci].detail +
                       "'");
  }
  if (rows == 0) throw ParseError(path + ": no feature rows");
  Dense m;
  m.rows = rows;
  m.cols = cols;
  m.data.reserve(static_cast<size_t>(rows * cols));
  for (auto& o : out) m.data.insert(m.data.end(), o.vals.begin(), o.vals.end());
  return m;
}

// dataset.hpp:218-234: std::stol per non-blank, non-'#' line, cast to int32.
std::vector<std::int32_t> load_labels(const std::string& path) {
  const std::string text = read_file(path);
  const char* b = text.data();
  const char* e = b + text.size();
  auto parts = chunks(b, e);
  std::vector<std::vector<std::int32_t>> out(parts.size());
  std::vector<ChunkError> err(parts.size());
  run_chunks(parts.size(), [&](size_t ci) {
    const char* s = parts[ci].first;
    const char* ce = parts[ci].second;
    while (s < ce) {
      const char* l0 = s;
      const char* l1 = line_end(s, ce);
      s = l1 < ce ? l1 + 1 : ce;
      const char* q = l0;
      while (q < l1 && (*q == ' ' || *q == '\t' || *q == '\r')) ++q;
      if (q == l1 || *q == '#') continue;
      std::string line(l0, l1);
      char* end = nullptr;
      errno = 0;
      const long v = std::strtol(line.c_str(), &end, 10);
      if (end == line.c_str() || errno == ERANGE) {
        err[ci] = {l0, 1, line};
        return;
      }
      out[ci].push_back(static_cast<std::int32_t>(v));
    }
  });
  std::vector<std::int32_t> labels;
  for (size_t ci = 0; ci < parts.size(); ++ci) {
    if (err[ci].line)
      throw ParseError(path + ":" + std::to_string(line_number(b, err[ci].line)) + ": bad label '" + err[ci].detail +
                       "'");
    labels.insert(labels.end(), out[ci].begin(), out[ci].end());
  }
  return labels;
}

// ---------------------------------------------------------------- masks JSON (dataset.hpp:237-262)
// A small recursive-descent JSON reader: the document must be valid JSON; for the keys train / val /
// test of a top-level object every element of the value (array elements, object values, or the
// scalar itself) is a vertex id (integers; floats truncated, as nlohmann's get<int64_t>; anything else is
// a type error, reported here as MG_PARSE_ERROR).
class Json {
 public:
  Json(const std::string& text, const std::string& path) : p_(text.data()), e_(p_ + text.size()), path_(path) {}

  std::map<std::string, std::vector<index_t>> masks() {
    ws();
    std::map<std::string, std::vector<index_t>> out;
    if (peek() == '{') {
      ++p_;
      ws();
      if (peek() == '}') {
        ++p_;
      } else {
        while (true) {
          ws();
          std::string key = str();
          ws();
          expect(':');
          ws();
          std::vector<index_t> ids;
          const bool want = key == "train" || key == "val" || key == "test";
          value(want ? &ids : nullptr, true);
          if (want) out[key] = std::move(ids);  // last duplicate wins
          ws();
          if (peek() == ',') {
            ++p_;
            continue;
          }
          expect('}');
          break;
        }
      }
    } else {
      value(nullptr, false);
    }
    ws();
    if (p_ != e_) fail("unexpected trailing content");
    return out;
  }

 private:
  const char* p_;
  const char* e_;
  std::string path_;

  [[noreturn]] void fail(const std::string& what) { throw ParseError(path_ + ": " + what); }
  char peek() const { return p_ < e_ ? *p_ : '\0'; }
  void ws() {
    while (p_ < e_ && (*p_ == ' ' || *p_ == '\t' || *p_ == '\n' || *p_ == '\r')) ++p_;
  }
  void expect(char c) {
    if (peek() != c) fail(std::string("expected '") + c + "'");
    ++p_;
  }
  std::string str() {
    expect('"');
    std::string s;
    while (p_ < e_ && *p_ != '"') {
      if (static_cast<unsigned char>(*p_) < 0x20) fail("control character in string");
      if (*p_ == '\\') {
        ++p_;
        if (p_ >= e_) fail("unterminated string");
        const char c = *p_++;
        if (c == 'u') {
          if (e_ - p_ < 4) fail("bad \\u escape");
          p_ += 4;
          s += '?';
        } else if (std::strchr("\"\\/bfnrt", c)) {
          s += c;
        } else {
          fail("bad escape");
        }
      } else {
        s += *p_++;
      }
    }
    expect('"');
    return s;
  }
  // element of an id list: nlohmann get<index_t>()
  void id(std::vector<index_t>* ids) {
    ws();
    const char c = peek();
    if (c == '-' || is_digit(c)) {
      double d;
      index_t i;
      const bool is_int = number(i, d);
      if (ids) ids->push_back(is_int ? i : static_cast<index_t>(d));
    } else {
      if (ids) fail("vertex id: type must be number");  // nlohmann type_error.302
      value(nullptr, false);
    }
  }
  void lit(const char* w) {
    const size_t n = std::strlen(w);
    if (static_cast<size_t>(e_ - p_) < n || std::strncmp(p_, w, n) != 0) fail("invalid literal");
    p_ += n;
  }
  bool number(index_t& i, double& d) {
    const char* s = p_;
    if (peek() == '-') ++p_;
    if (!is_digit(peek())) fail("invalid number");
    if (*p_ == '0') ++p_;
    else
      while (is_digit(peek())) ++p_;
    bool integral = true;
    if (peek() == '.') {
      integral = false;
      ++p_;
      if (!is_digit(peek())) fail("invalid number");
      while (is_digit(peek())) ++p_;
    }
    if (peek() == 'e' || peek() == 'E') {
      integral = false;
      ++p_;
      if (peek() == '+' || peek() == '-') ++p_;
      if (!is_digit(peek())) fail("invalid number");
      while (is_digit(peek())) ++p_;
    }
    std::string t(s, p_);
    if (integral) {
      errno = 0;
      char* end = nullptr;
      const long long v = std::strtoll(t.c_str(), &end, 10);
      if (errno != ERANGE) {
        i = v;
        return true;
      }
    }
    d = std::strtod(t.c_str(), nullptr);
    return false;
  }
  // any JSON value; when `ids` is set (a mask key), collect the ids it holds
  void value(std::vector<index_t>* ids, bool top_key) {
    ws();
    const char c = peek();
    if (c == '[') {
      ++p_;
      ws();
      if (peek() == ']') {
        ++p_;
        return;
      }
      while (true) {
        if (ids) id(ids);
        else value(nullptr, false);
        ws();
        if (peek() == ',') {
          ++p_;
          continue;
        }
        expect(']');
        return;
      }
    } else if (c == '{') {
      ++p_;
      ws();
      if (peek() == '}') {
        ++p_;
        return;
      }
      while (true) {
        ws();
        str();
        ws();
        expect(':');
        if (ids) id(ids);
        else value(nullptr, false);
        ws();
        if (peek() == ',') {
          ++p_;
          continue;
        }
        expect('}');
        return;
      }
    } else if (c == '"') {
      if (ids && top_key) fail("vertex ids must be numbers");
      str();
    } else if (c == 'n') {  // a null mask value iterates as empty
      lit("null");
    } else if (ids && top_key) {
      id(ids);
    } else if (c == 't') {
      lit("true");
    } else if (c == 'f') {
      lit("false");
    } else if (c == '-' || is_digit(c)) {
      index_t i;
      double d;
      number(i, d);
    } else {
      fail("syntax error");
    }
  }
};

// present: bit 0 train, bit 1 val, bit 2 test
int load_masks(const std::string& path, index_t n, std::vector<std::uint8_t>& train, std::vector<std::uint8_t>& val,
               std::vector<std::uint8_t>& test) {
  const std::string text = read_file(path);
  auto m = Json(text, path).masks();
  int present = 0;
  auto fill = [&](const char* key, std::vector<std::uint8_t>& out, int bit) {
    auto it = m.find(key);
    if (it == m.end()) return;
    present |= bit;
    out.assign(static_cast<size_t>(n), 0);
    for (index_t v : it->second) {
      if (v < 0 || v >= n)
        throw ParseError(path + ": vertex id " + std::to_string(v) + " out of range [0, " + std::to_string(n) + ")");
      out[static_cast<size_t>(v)] = 1;
    }
  };
  fill("train", train, 1);
  fill("val", val, 2);
  fill("test", test, 4);
  return present;
}

}  // namespace io
}  // namespace mg

struct mg_graph {
  mg::Csr csr;
};
struct mg_dense {
  mg::io::Dense m;
};

using namespace mg;

extern "C" {

mg_status mg_graph_load(const char* path, int32_t format, mg_graph** out) {
  return guarded([&] {
    if (!path || !out) throw ValueError("load_graph: null argument");
    auto g = std::make_unique<mg_graph>();
    g->csr = io::load_graph(path, format);
    *out = g.release();
  });
}

mg_status mg_graph_view(const mg_graph* g, mg_csr* out) {
  return guarded([&] {
    if (!g || !out) throw ValueError("graph: null argument");
    out->rows = g->csr.rows;
    out->cols = g->csr.cols;
    out->row_ptr = g->csr.row_ptr.data();
    out->col_idx = g->csr.col_idx.data();
    out->values = g->csr.values.data();
  });
}

void mg_graph_free(mg_graph* g) { delete g; }

// from_coo (inc/sparse.hpp:59-90): edges range-checked against n, rows sorted by (src, dst), duplicate
// (src, dst) weights summed (in edge order: a stable sort, where the reference's std::sort leaves the order
// of equal keys unspecified).
mg_status mg_graph_from_coo(int64_t n, int64_t count, const int64_t* src, const int64_t* dst, const float* weight,
                            mg_graph** out) {
  return guarded([&] {
    if (!out || n < 0 || count < 0 || (count > 0 && (!src || !dst || !weight)))
      throw ValueError("from_coo: bad argument");
    for (int64_t e = 0; e < count; ++e)
      if (src[e] < 0 || src[e] >= n || dst[e] < 0 || dst[e] >= n)
        throw ValueError("from_coo: edge (" + std::to_string(src[e]) + ", " + std::to_string(dst[e]) +
                         ") out of range for n=" + std::to_string(n));
    // counting sort by source row (stable), then a stable sort of each row by destination
    std::vector<index_t> start(static_cast<size_t>(n) + 1, 0);
    for (int64_t e = 0; e < count; ++e) ++start[static_cast<size_t>(src[e]) + 1];
    for (index_t u = 0; u < n; ++u) start[static_cast<size_t>(u) + 1] += start[static_cast<size_t>(u)];
    std::vector<std::pair<index_t, float>> byrow(static_cast<size_t>(count));
    std::vector<index_t> fill(start.begin(), start.end() - 1);
    for (int64_t e = 0; e < count; ++e) byrow[static_cast<size_t>(fill[static_cast<size_t>(src[e])]++)] = {dst[e], weight[e]};
    auto g = std::make_unique<mg_graph>();
    Csr& m = g->csr;
    m.rows = m.cols = n;
    m.row_ptr.assign(static_cast<size_t>(n) + 1, 0);
    for (index_t u = 0; u < n; ++u) {
      auto b = byrow.begin() + start[static_cast<size_t>(u)], e = byrow.begin() + start[static_cast<size_t>(u) + 1];
      std::stable_sort(b, e, [](const auto& x, const auto& y) { return x.first < y.first; });
      for (auto it = b; it != e;) {
        const index_t v = it->first;
        float w = it->second;
        for (++it; it != e && it->first == v; ++it) w += it->second;
        m.col_idx.push_back(v);
        m.values.push_back(w);
      }
      m.row_ptr[static_cast<size_t>(u) + 1] = static_cast<index_t>(m.col_idx.size());
    }
    *out = g.release();
  });
}

// add_self_loops (inc/dataset.hpp:60-73): a unit (u, u) entry wherever row u lacks one, rebuilt as
// from_coo does (inc/sparse.hpp:59-90): rows sorted by column, duplicate entries summed, range-checked
// against n = rows.
mg_status mg_graph_add_self_loops(const mg_csr* a, mg_graph** out) {
  return guarded([&] {
    if (!a || !out || a->rows < 0 || (a->rows > 0 && !a->row_ptr)) throw ValueError("add_self_loops: bad argument");
    const index_t n = a->rows;
    auto g = std::make_unique<mg_graph>();
    Csr& m = g->csr;
    m.rows = m.cols = n;
    m.row_ptr.assign(static_cast<size_t>(n) + 1, 0);
    std::vector<std::pair<index_t, float>> row;
    for (index_t u = 0; u < n; ++u) {
      row.clear();
      bool diag = false;
      for (index_t e = a->row_ptr[u]; e < a->row_ptr[u + 1]; ++e) {
        const index_t v = a->col_idx[e];
        if (v < 0 || v >= n)
          throw ValueError("from_coo: edge (" + std::to_string(u) + ", " + std::to_string(v) +
                           ") out of range for n=" + std::to_string(n));
        diag = diag || v == u;
        row.push_back({v, a->values[e]});
      }
      if (!diag) row.push_back({u, 1.0f});
      std::stable_sort(row.begin(), row.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
      for (size_t i = 0; i < row.size();) {
        const index_t v = row[i].first;
        float w = row[i].second;
        for (++i; i < row.size() && row[i].first == v; ++i) w += row[i].second;
        m.col_idx.push_back(v);
        m.values.push_back(w);
      }
      m.row_ptr[static_cast<size_t>(u) + 1] = static_cast<index_t>(m.col_idx.size());
    }
    *out = g.release();
  });
}

mg_status mg_dense_load(const char* path, mg_dense** out) {
  return guarded([&] {
    if (!path || !out) throw ValueError("load_features: null argument");
    auto d = std::make_unique<mg_dense>();
    d->m = io::load_features(path);
    *out = d.release();
  });
}

mg_status mg_dense_read(const char* path, mg_dense** out) {
  return guarded([&] {
    if (!path || !out) throw ValueError("read_dense: null argument");
    auto d = std::make_unique<mg_dense>();
    d->m = io::read_dense(path);
    *out = d.release();
  });
}

mg_status mg_dense_view(const mg_dense* d, int64_t* rows, int64_t* cols, const float** data) {
  return guarded([&] {
    if (!d) throw ValueError("dense: null");
    if (rows) *rows = d->m.rows;
    if (cols) *cols = d->m.cols;
    if (data) *data = d->m.data.data();
  });
}

void mg_dense_free(mg_dense* d) { delete d; }

mg_status mg_dense_write(const char* path, int64_t rows, int64_t cols, const float* data) {
  return guarded([&] {
    if (!path || rows < 0 || cols < 0 || (!data && rows * cols > 0)) throw ValueError("write_dense: bad argument");
    io::write_dense(path, rows, cols, data);
  });
}

mg_status mg_labels_load(const char* path, int32_t* dst, int64_t capacity, int64_t* count) {
  return guarded([&] {
    if (!path || !count) throw ValueError("load_labels: null argument");
    const auto labels = io::load_labels(path);
    *count = static_cast<int64_t>(labels.size());
    if (dst) {
      if (capacity < *count) throw ShapeError("load_labels: capacity " + std::to_string(capacity) + " < " +
                                              std::to_string(*count) + " labels");
      std::copy(labels.begin(), labels.end(), dst);
    }
  });
}

mg_status mg_masks_load(const char* path, int64_t n, uint8_t* train, uint8_t* val, uint8_t* test, int32_t* present) {
  return guarded([&] {
    if (!path || n < 0) throw ValueError("load_masks: bad argument");
    std::vector<std::uint8_t> tr, va, te;
    const int pr = io::load_masks(path, n, tr, va, te);
    if (present) *present = pr;
    if (train && !tr.empty()) std::copy(tr.begin(), tr.end(), train);
    if (val && !va.empty()) std::copy(va.begin(), va.end(), val);
    if (test && !te.empty()) std::copy(te.begin(), te.end(), test);
  });
}

mg_status mg_dataset_load(const char* graph_path, const char* features_path, const char* labels_path,
                          const char* masks_path, mg_dataset** out) {
  return guarded([&] {
    if (!graph_path || !features_path || !labels_path || !out) throw ValueError("load_dataset: null argument");
    auto ds = std::make_unique<mg_dataset>();
    ds->name = graph_path;
    ds->graph = io::load_graph(graph_path, 0);
    io::Dense f = io::load_features(features_path);
    ds->feature_rows = f.rows;
    ds->d0 = f.cols;
    ds->features = std::move(f.data);
    ds->labels = io::load_labels(labels_path);
    if (masks_path && masks_path[0])
      io::load_masks(masks_path, ds->n(), ds->train_mask, ds->val_mask, ds->test_mask);
    validate_dataset_named(*ds);
    *out = ds.release();
  });
}

mg_status mg_dataset_masks(const mg_dataset* ds, const uint8_t** train, const uint8_t** val, const uint8_t** test) {
  return guarded([&] {
    if (!ds) throw ValueError("dataset: null");
    if (train) *train = ds->train_mask.empty() ? nullptr : ds->train_mask.data();
    if (val) *val = ds->val_mask.empty() ? nullptr : ds->val_mask.data();
    if (test) *test = ds->test_mask.empty() ? nullptr : ds->test_mask.data();
  });
}

}  // extern "C"
