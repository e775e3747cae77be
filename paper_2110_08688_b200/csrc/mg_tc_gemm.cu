// SPDX-License-Identifier: Apache-2.0
#include <string>

#include "mg_internal.hpp"
#include "mg_tc_gemm.cuh"

namespace mg {
namespace tc {
bool available() { return false; }
int gemm(int mode, bool, bool, int64_t, int64_t, int64_t, const float*, int64_t, const float*, int64_t, float*,
         int64_t, int, cudaStream_t) {
  throw ValueError("gemm_mode " + std::to_string(mode) + ": tcgen05 path not built");
}
}  // namespace tc
}  // namespace mg
