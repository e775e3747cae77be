// TEST INFRASTRUCTURE ONLY. Compiles the reference's own callers of its training API — run_train
// (proj/tools/main.cpp:56-101) and the train_run / grad_run test cases of proj/tests/test_gcn.cpp:213-348 —
// UNCHANGED against the drop-in header include/mggcn/rowgcn.hpp (only S = double -> float), then runs
// them on the GPU. The reference text is extracted at build time by tests/dropin/extract.py into
// tests/dropin/_build/*.inc (git-ignored; never committed). A doctest stand-in provides TEST_CASE / CHECK /
// REQUIRE (doctest itself is not vendored in the reference tree).
//
//   dropin_main cases                                  run the extracted test cases
//   dropin_main train GRAPH FEATS LABELS CONFIG CKPT [WORKERS]   run_train<float> as the CLI calls it
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include <json.hpp>

#include "mggcn/rowgcn.hpp"

namespace rowgcn = mggcn::rowgcn;
using namespace rowgcn;

namespace shim {
struct Abort {};
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
inline int& failures() {
  static int f = 0;
  return f;
}
inline bool add(const char* name, void (*fn)()) {
  cases().push_back({name, fn});
  return true;
}
inline bool check(bool ok, const char* expr, const char* file, int line) {
  if (!ok) {
    ++failures();
    std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", file, line, expr);
  }
  return ok;
}
}  // namespace shim

#define DT_CAT2(a, b) a##b
#define DT_CAT(a, b) DT_CAT2(a, b)
#define TEST_CASE(name)                                                                   \
  void DT_CAT(dt_case_, __LINE__)();                                                      \
  const bool DT_CAT(dt_reg_, __LINE__) = shim::add(name, DT_CAT(dt_case_, __LINE__));     \
  void DT_CAT(dt_case_, __LINE__)()
#define CHECK(...) shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                      \
  do {                                                                                    \
    if (!shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__))   \
      throw shim::Abort();                                                                \
  } while (0)

namespace {
#include "_build/run_train.inc"
#include "_build/test_gcn_cases.inc"
}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cases";
  try {
    if (mode == "cases") {
      for (const auto& c : shim::cases()) {
        const int before = shim::failures();
        try {
          c.fn();
        } catch (const shim::Abort&) {
        }
        std::printf("%s: %s\n", shim::failures() == before ? "ok" : "FAILED", c.name);
      }
      std::printf("%zu cases, %d failed checks\n", shim::cases().size(), shim::failures());
      return shim::failures() == 0 ? 0 : 1;
    }
    if (mode == "train" && argc >= 7) {
      CommonFlags flags;
      flags.workers = argc > 7 ? std::atoi(argv[7]) : 1;
      flags.permute = true;
      return run_train<float>(flags, argv[2], argv[3], argv[4], "", argv[5], argv[6]);
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
  std::fprintf(stderr, "usage: dropin_main cases | train GRAPH FEATS LABELS CONFIG CKPT [WORKERS]\n");
  return 2;
}
