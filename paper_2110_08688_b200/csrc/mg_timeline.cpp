// SPDX-License-Identifier: Apache-2.0
//
// Host half of the timeline: export in the reference schema, the reference's two
// audits and the runtime breakdown, over mg_timeline_event arrays recorded from CUDA events
// (mg_group_timeline) or built by the caller.
//   export_timeline   inc/timeline.hpp:31-36     audit_timeline     inc/timeline.hpp:64-94
//   audit_staged_run  inc/timeline.hpp:96-126    runtime_breakdown  inc/breakdown.hpp:63-82
#include <cstdio>
#include <map>
#include <memory>
#include <string>

#include "mg_internal.hpp"

using namespace mg;

namespace {

struct IoErr : Error { explicit IoErr(const std::string& m) : Error(MG_IO_ERROR, m) {} };

std::string json_str(const char* s) {
  std::string o = "\"";
  for (const char* p = s; *p; ++p) {
    const unsigned char c = static_cast<unsigned char>(*p);
    if (c == '"' || c == '\\') {
      o += '\\';
      o += static_cast<char>(c);
    } else if (c < 0x20) {
      char b[8];
      std::snprintf(b, sizeof(b), "\\u%04x", c);
      o += b;
    } else {
      o += static_cast<char>(c);
    }
  }
  return o + "\"";
}

std::string num(double v) {
  char b[40];
  std::snprintf(b, sizeof(b), "%.17g", v);
  return b;
}

void check_args(const mg_timeline_event* ev, int64_t count) {
  if (count < 0 || (count > 0 && !ev)) throw ValueError("timeline: bad event array");
}

}  // namespace

extern "C" {

mg_status mg_timeline_export(const char* path, const mg_timeline_event* ev, int64_t count) {
  return guarded([&] {
    check_args(ev, count);
    if (!path) throw ValueError("timeline: null path");
    std::FILE* f = std::fopen(path, "w");
    if (!f) throw IoErr(std::string("cannot open ") + path + " for writing");
    std::unique_ptr<std::FILE, int (*)(std::FILE*)> guard(f, std::fclose);
    std::string out = "[";
    for (int64_t i = 0; i < count; ++i) {
      const auto& e = ev[i];
      out += i ? ",\n {" : "\n {";
      out += "\n  \"worker\": " + std::to_string(e.worker) + ",\n  \"lane\": " + std::to_string(e.lane) +
             ",\n  \"stage\": " + std::to_string(e.stage) + ",\n  \"kind\": " + json_str(e.kind) +
             ",\n  \"op\": " + json_str(e.op) + ",\n  \"t_start_us\": " + num(e.t_start_us) +
             ",\n  \"t_end_us\": " + num(e.t_end_us) + ",\n  \"task\": " + std::to_string(e.task) + ",\n  \"deps\": [";
      for (int32_t d = 0; d < e.n_deps; ++d) out += (d ? ", " : "") + std::to_string(e.deps[d]);
      out += "]\n }";
    }
    out += count ? "\n]\n" : "]\n";
    if (std::fwrite(out.data(), 1, out.size(), f) != out.size() || std::fflush(f) != 0)
      throw IoErr(std::string("short write to ") + path);
  });
}

mg_status mg_timeline_audit(const mg_timeline_event* ev, int64_t count) {
  return guarded([&] {
    check_args(ev, count);
    std::map<std::pair<int, int>, std::vector<const mg_timeline_event*>> lanes;
    std::map<uint64_t, const mg_timeline_event*> by_task;
    for (int64_t i = 0; i < count; ++i) {
      const auto& e = ev[i];
      if (e.t_start_us > e.t_end_us)
        throw ValueError("timeline: event on worker " + std::to_string(e.worker) + " has t_start > t_end");
      lanes[{e.worker, e.lane}].push_back(&e);
      if (e.task) by_task[e.task] = &e;
    }
    for (auto& [key, vec] : lanes) {
      std::stable_sort(vec.begin(), vec.end(), [](const mg_timeline_event* a, const mg_timeline_event* b) {
        return a->t_start_us < b->t_start_us;
      });
      for (size_t i = 1; i < vec.size(); ++i)
        if (vec[i]->t_start_us < vec[i - 1]->t_end_us)
          throw ValueError("timeline: overlapping events on worker " + std::to_string(key.first) + " lane " +
                           std::to_string(key.second));
    }
    for (int64_t i = 0; i < count; ++i) {
      const auto& e = ev[i];
      for (int32_t k = 0; k < e.n_deps; ++k) {
        const uint64_t d = e.deps[k];
        auto it = by_task.find(d);
        if (it == by_task.end())
          throw ValueError("timeline: task " + std::to_string(e.task) + " depends on missing task " +
                           std::to_string(d));
        if (it->second->t_end_us > e.t_start_us)
          throw ValueError("timeline: dependency " + std::to_string(d) + " of task " + std::to_string(e.task) +
                           " finished after the dependent started");
      }
    }
  });
}

mg_status mg_timeline_audit_staged(const mg_timeline_event* ev, int64_t count, int32_t world, int32_t overlapped) {
  return guarded([&] {
    check_args(ev, count);
    for (int w = 0; w < world; ++w) {
      std::map<int, const mg_timeline_event*> bcast, mult;
      for (int64_t i = 0; i < count; ++i) {
        const auto& e = ev[i];
        if (e.worker != w || e.stage < 0) continue;
        if (std::string(e.kind) == "broadcast") bcast[e.stage] = &e;
        if (std::string(e.kind) == "spmm") mult[e.stage] = &e;
      }
      if (bcast.size() != mult.size())
        throw ValueError("staged audit: worker " + std::to_string(w) + " has " + std::to_string(bcast.size()) +
                         " broadcasts but " + std::to_string(mult.size()) + " multiplies");
      const int stages = static_cast<int>(bcast.size());
      for (int j = 0; j < stages; ++j) {
        if (!bcast.count(j) || !mult.count(j))
          throw ValueError("staged audit: worker " + std::to_string(w) + " missing stage " + std::to_string(j));
        if (mult[j]->t_start_us < bcast[j]->t_end_us)
          throw ValueError("staged audit: spmm(" + std::to_string(j) + ") started before broadcast(" +
                           std::to_string(j) + ") finished on worker " + std::to_string(w));
        const int guard = overlapped ? j - 2 : j - 1;
        if (guard >= 0 && bcast[j]->t_start_us < mult[guard]->t_end_us)
          throw ValueError("staged audit: broadcast(" + std::to_string(j) + ") started before spmm(" +
                           std::to_string(guard) + ") finished on worker " + std::to_string(w));
      }
    }
  });
}

mg_status mg_timeline_breakdown(const mg_timeline_event* ev, int64_t count, double totals_us[6]) {
  return guarded([&] {
    check_args(ev, count);
    if (!totals_us) throw ValueError("breakdown: null output");
    if (count == 0) throw ValueError("runtime_breakdown: no events recorded");
    double t[6] = {0, 0, 0, 0, 0, 0};  // spmm, gemm, activation, loss, adam, comm
    for (int64_t i = 0; i < count; ++i) {
      const auto& e = ev[i];
      const std::string kind = e.kind, op = e.op;
      const double d = e.t_end_us - e.t_start_us;
      if (kind == "broadcast" || kind == "reduce") t[5] += d;
      else if (kind == "spmm") t[0] += d;
      else if (kind == "gemm") t[1] += d;
      else if (op == "relu" || op == "relu_bwd") t[2] += d;
      else if (op == "loss") t[3] += d;
      else if (op == "adam" || op == "wgrad_final") t[4] += d;
    }
    std::copy(t, t + 6, totals_us);
  });
}

}  // extern "C"
