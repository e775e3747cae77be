// SPDX-License-Identifier: Apache-2.0
//
// The JSON documents the reference's API emits, produced natively so the drop-in needs no JSON library:
//   * config_to_json (inc/driver.hpp:59-71) — the checkpoint sidecar <path>.json (driver.hpp:272-273)
//   * BreakdownReport::to_json / text_table (inc/breakdown.hpp:27-58)
// The reference serialises with nlohmann::json::dump(indent); this writer reproduces that text byte for
// byte for these documents: object keys in sorted order, `indent` spaces per level ("key": value, one
// member per line) or the compact form for indent < 0, integers as integers, and doubles as the shortest
// round-trip digits laid out like nlohmann's format_buffer (fixed notation for decimal exponents in
// (-4, 15], otherwise d.ddde±XX with at least two exponent digits, a ".0" on integral values).
// Also the checkpoint files themselves (MGDM blocks, driver.hpp:255-299) and add_self_loops
// (inc/dataset.hpp:60-73).
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <system_error>
#include <vector>

#include "mg_internal.hpp"

namespace mg {
namespace {

// ---------------------------------------------------------------- a minimal JSON value + nlohmann-style dump
struct JVal {
  enum Kind { Int, Uint, Num, Bool, Arr, Obj } kind = Int;
  long long i = 0;
  unsigned long long u = 0;
  double d = 0;
  bool b = false;
  std::vector<JVal> arr;
  std::map<std::string, JVal> obj;  // std::map: keys come out sorted, like nlohmann::json's object_t
  static JVal integer(long long v) { JVal j; j.kind = Int; j.i = v; return j; }
  static JVal uinteger(unsigned long long v) { JVal j; j.kind = Uint; j.u = v; return j; }
  static JVal number(double v) { JVal j; j.kind = Num; j.d = v; return j; }
  static JVal boolean(bool v) { JVal j; j.kind = Bool; j.b = v; return j; }
};

// Shortest round-trip decimal digits of v and the layout of nlohmann's dtoa_impl::format_buffer.
std::string format_double(double v) {
  if (!std::isfinite(v)) return "null";
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char sci[64];
  const auto r = std::to_chars(sci, sci + sizeof(sci), v, std::chars_format::scientific);
  const std::string s(sci, r.ptr);  // [-]d[.ddd]e±XX, shortest digits
  std::string out;
  size_t p = 0;
  if (s[0] == '-') {
    out += '-';
    p = 1;
  }
  const size_t epos = s.find('e');
  std::string digits;
  for (size_t q = p; q < epos; ++q)
    if (s[q] != '.') digits += s[q];
  const int e10 = std::atoi(s.c_str() + epos + 1);  // value = d.ddd * 10^e10
  const int k = static_cast<int>(digits.size());
  const int n = e10 + 1;  // decimal point position: value = 0.d1..dk * 10^n
  constexpr int kMinExp = -4, kMaxExp = 15;
  if (k <= n && n <= kMaxExp) {
    out += digits + std::string(static_cast<size_t>(n - k), '0') + ".0";
  } else if (0 < n && n <= kMaxExp) {
    out += digits.substr(0, static_cast<size_t>(n)) + "." + digits.substr(static_cast<size_t>(n));
  } else if (kMinExp < n && n <= 0) {
    out += "0." + std::string(static_cast<size_t>(-n), '0') + digits;
  } else {
    out += digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    const int e = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof(eb), "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
    out += eb;
  }
  return out;
}

void dump(const JVal& v, int indent, int level, std::string& out) {
  const bool pretty = indent >= 0;
  const std::string pad_in = pretty ? std::string(static_cast<size_t>(indent * (level + 1)), ' ') : "";
  const std::string pad = pretty ? std::string(static_cast<size_t>(indent * level), ' ') : "";
  switch (v.kind) {
    case JVal::Int: out += std::to_string(v.i); return;
    case JVal::Uint: out += std::to_string(v.u); return;
    case JVal::Num: out += format_double(v.d); return;
    case JVal::Bool: out += v.b ? "true" : "false"; return;
    case JVal::Arr: {
      if (v.arr.empty()) {
        out += "[]";
        return;
      }
      out += pretty ? "[\n" : "[";
      for (size_t i = 0; i < v.arr.size(); ++i) {
        if (i) out += pretty ? ",\n" : ",";
        out += pad_in;
        dump(v.arr[i], indent, level + 1, out);
      }
      out += pretty ? "\n" + pad + "]" : "]";
      return;
    }
    case JVal::Obj: {
      if (v.obj.empty()) {
        out += "{}";
        return;
      }
      out += pretty ? "{\n" : "{";
      bool first = true;
      for (const auto& kv : v.obj) {
        if (!first) out += pretty ? ",\n" : ",";
        first = false;
        out += pad_in + "\"" + kv.first + (pretty ? "\": " : "\":");
        dump(kv.second, indent, level + 1, out);
      }
      out += pretty ? "\n" + pad + "}" : "}";
      return;
    }
  }
}

std::string dump(const JVal& v, int indent) {
  std::string s;
  dump(v, indent, 0, s);
  return s;
}

// config_to_json (driver.hpp:59-71): the GcnConfig keys only (no device modes).
JVal config_json(const mg_config* c) {
  JVal j;
  j.kind = JVal::Obj;
  JVal dims;
  dims.kind = JVal::Arr;
  for (int32_t i = 0; i < c->n_dims; ++i) dims.arr.push_back(JVal::integer(c->layer_dims[i]));
  j.obj["layer_dims"] = dims;
  j.obj["lr"] = JVal::number(c->lr);
  j.obj["beta1"] = JVal::number(c->beta1);
  j.obj["beta2"] = JVal::number(c->beta2);
  j.obj["epsilon"] = JVal::number(c->epsilon);
  j.obj["epochs"] = JVal::integer(c->epochs);
  j.obj["seed"] = JVal::uinteger(c->seed);
  j.obj["permute"] = JVal::boolean(c->permute != 0);
  j.obj["overlap"] = JVal::boolean(c->overlap != 0);
  j.obj["skip_first_backward_spmm"] = JVal::boolean(c->skip_first_backward_spmm != 0);
  j.obj["order_swap"] = JVal::boolean(c->order_swap != 0);
  return j;
}

// BreakdownReport (breakdown.hpp:17-61) over totals {spmm, gemm, activation, loss, adam, comm}.
constexpr const char* kBuckets[6] = {"spmm", "gemm", "activation", "loss", "adam", "comm"};
double bucket_total(const double* t) { return t[0] + t[1] + t[2] + t[3] + t[4] + t[5]; }
double bucket_frac(const double* t, double v) {
  const double tot = bucket_total(t);
  return tot > 0 ? v / tot : 0.0;
}
JVal breakdown_json(const double* t) {
  JVal tot, fr, j;
  tot.kind = fr.kind = j.kind = JVal::Obj;
  for (int b = 0; b < 6; ++b) {
    tot.obj[kBuckets[b]] = JVal::number(t[b]);
    fr.obj[kBuckets[b]] = JVal::number(bucket_frac(t, t[b]));
  }
  j.obj["totals_us"] = tot;
  j.obj["fractions"] = fr;
  return j;
}

void copy_out(const std::string& s, char* buf, int64_t capacity, int64_t* length) {
  if (length) *length = static_cast<int64_t>(s.size());
  if (buf && capacity > 0) {
    const size_t n = std::min<size_t>(s.size(), static_cast<size_t>(capacity - 1));
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
}

}  // namespace
}  // namespace mg

struct mg_checkpoint {
  std::vector<mg::index_t> rows, cols;
  std::vector<std::vector<float>> data;
};

using namespace mg;

extern "C" {

mg_status mg_config_to_json(const mg_config* cfg, int32_t indent, char* buf, int64_t capacity, int64_t* length) {
  return guarded([&] {
    if (!cfg || (cfg->n_dims > 0 && !cfg->layer_dims)) throw ValueError("config_to_json: null config");
    copy_out(dump(config_json(cfg), indent), buf, capacity, length);
  });
}

mg_status mg_breakdown_to_json(const double totals_us[6], int32_t indent, char* buf, int64_t capacity,
                               int64_t* length) {
  return guarded([&] {
    if (!totals_us) throw ValueError("breakdown: null totals");
    copy_out(dump(breakdown_json(totals_us), indent), buf, capacity, length);
  });
}

mg_status mg_breakdown_text(const double totals_us[6], char* buf, int64_t capacity, int64_t* length) {
  return guarded([&] {
    if (!totals_us) throw ValueError("breakdown: null totals");
    std::string s = "kernel               time_us fraction\n";
    char line[96];
    for (int b = 0; b < 7; ++b) {
      const double v = b < 6 ? totals_us[b] : bucket_total(totals_us);
      std::snprintf(line, sizeof(line), "%-12s %14.1f %8.3f\n", b < 6 ? kBuckets[b] : "total", v,
                    bucket_frac(totals_us, v));
      s += line;
    }
    copy_out(s, buf, capacity, length);
  });
}

// write_checkpoint (driver.hpp:255-274): each W as an MGDM block back to back, then <path>.json.
mg_status mg_checkpoint_write(const char* path, int32_t count, const int64_t* rows, const int64_t* cols,
                              const float* const* data, const mg_config* cfg) {
  return guarded([&] {
    if (!path || count < 0 || (count > 0 && (!rows || !cols || !data)) || !cfg)
      throw ValueError("write_checkpoint: bad argument");
    const std::string p = path;
    {
      std::FILE* f = std::fopen(path, "wb");
      if (!f) throw IoError("cannot open " + p + " for writing");
      std::unique_ptr<std::FILE, int (*)(std::FILE*)> guard(f, std::fclose);
      bool ok = true;
      for (int32_t i = 0; i < count && ok; ++i) {
        const std::uint64_t r = static_cast<std::uint64_t>(rows[i]), c = static_cast<std::uint64_t>(cols[i]);
        const std::uint8_t width = 4;
        const size_t n = static_cast<size_t>(r * c);
        ok = std::fwrite("MGDM", 1, 4, f) == 4 && std::fwrite(&r, 8, 1, f) == 1 && std::fwrite(&c, 8, 1, f) == 1 &&
             std::fwrite(&width, 1, 1, f) == 1 && (n == 0 || std::fwrite(data[i], 4, n, f) == n);
      }
      if (!ok || std::fflush(f) != 0) throw IoError("short write to " + p);
    }
    const std::string side = dump(config_json(cfg), 1) + "\n";
    if (std::FILE* s = std::fopen((p + ".json").c_str(), "wb")) {  // unchecked, like the reference's ofstream
      std::fwrite(side.data(), 1, side.size(), s);
      std::fclose(s);
    }
  });
}

// read_checkpoint<float> (driver.hpp:276-299): the blocks back, dtype width checked.
mg_status mg_checkpoint_read(const char* path, mg_checkpoint** out) {
  return guarded([&] {
    if (!path || !out) throw ValueError("read_checkpoint: null argument");
    const std::string p = path;
    std::FILE* f = std::fopen(path, "rb");
    if (!f) throw IoError("cannot open " + p);
    std::unique_ptr<std::FILE, int (*)(std::FILE*)> guard(f, std::fclose);
    auto ck = std::make_unique<mg_checkpoint>();
    while (true) {
      char magic[4];
      if (std::fread(magic, 1, 4, f) != 4) break;
      if (std::memcmp(magic, "MGDM", 4) != 0) throw ParseError(p + ": bad checkpoint block magic");
      std::uint64_t r = 0, c = 0;
      std::uint8_t width = 0;
      const bool hdr = std::fread(&r, 8, 1, f) == 1 && std::fread(&c, 8, 1, f) == 1 && std::fread(&width, 1, 1, f) == 1;
      if (!hdr || width != 4)
        throw ParseError(p + ": checkpoint dtype width " + std::to_string(hdr ? width : 0) +
                         " does not match run dtype 4");
      std::vector<float> w(static_cast<size_t>(r * c));
      if (!w.empty() && std::fread(w.data(), 4, w.size(), f) != w.size())
        throw ParseError(p + ": truncated checkpoint block");
      ck->rows.push_back(static_cast<index_t>(r));
      ck->cols.push_back(static_cast<index_t>(c));
      ck->data.push_back(std::move(w));
    }
    *out = ck.release();
  });
}

int32_t mg_checkpoint_count(const mg_checkpoint* ck) { return ck ? static_cast<int32_t>(ck->data.size()) : 0; }

mg_status mg_checkpoint_view(const mg_checkpoint* ck, int32_t i, int64_t* rows, int64_t* cols, const float** data) {
  return guarded([&] {
    if (!ck || i < 0 || i >= static_cast<int32_t>(ck->data.size())) throw ValueError("checkpoint: bad block index");
    if (rows) *rows = ck->rows[static_cast<size_t>(i)];
    if (cols) *cols = ck->cols[static_cast<size_t>(i)];
    if (data) *data = ck->data[static_cast<size_t>(i)].data();
  });
}

void mg_checkpoint_free(mg_checkpoint* ck) { delete ck; }

}  // extern "C"
