// SPDX-License-Identifier: Apache-2.0
// tcgen05 (5th-gen tensor core) GeMMs for the TF32X3 / TF32 modes — see mg_tc_gemm.cu.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace mg {
namespace tc {
bool available();
// C = op(A) op(B) (+ epilogue), row-major with leading dimensions; returns kernels launched.
int gemm(int mode, bool ta, bool tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B,
         int64_t ldb, float* C, int64_t ldc, int epi, cudaStream_t s);
}  // namespace tc
}  // namespace mg
