// SPDX-License-Identifier: Apache-2.0
// tcgen05 (5th-gen tensor core) GeMMs for the TF32X3 / TF32 modes — see mg_tc_gemm.cu.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

#include "mg_epi.cuh"

namespace mg {
namespace tc {
bool available();
// C = op(A) op(B) (+ epilogue), row-major with leading dimensions; returns kernels launched.
// TN (ta) needs a split-K workspace of tn_workspace_bytes(M, N, K) (one per concurrent stream).
int gemm(int mode, bool ta, bool tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B,
         int64_t ldb, float* C, int64_t ldc, int epi, float* ws, size_t ws_bytes, cudaStream_t s,
         const k::Epi& ep = k::Epi{}, const float* rmax_in = nullptr);
// rmax_in: per-row max |A| pairs (k::Epi::rmax of A's producer); with it, TF32X3 NN / NT run the scaled fp16
// two-term split (v3, "gemm_f16"), without it the 3xTF32 split. ep.rmax: write this GeMM's own row maxima.
size_t tn_workspace_bytes(int64_t M, int64_t N, int64_t K);
// W-grad over up to 8 canonical row blocks in one launch: stage + g*block_stride (M x N, ld ldc) =
// H[begin_g : begin_g + len_g]^T G[same rows]; empty blocks are written as zeros. Deterministic and
// independent of how the rows are distributed over workers (chunks are relative to each block start).
int gemm_tn_blocks(int mode, int nblocks, const int64_t* begin, const int64_t* len, int64_t M, int64_t N,
                   const float* H, int64_t ldh, const float* G, int64_t ldg, float* stage, int64_t ldc,
                   int64_t block_stride, float* ws, size_t ws_bytes, cudaStream_t s);
// NN / NT (v2 kernel) pre-split W into K-major hi/lo planes: nn_workspace_bytes(N, K).
size_t nn_workspace_bytes(int64_t N, int64_t K);
void set_tn_chunk(int rows);
void set_gemm_version(int v);
void set_w3_bytes(int bytes);
void set_epi_chunks3(int c);  // v3 epilogue 32x32 buffers per warp (1 or 2) without the relu_backward mask  // v3 W ring budget
void set_gemm3_cluster(int c);
void set_gemm_f16(int on);
void set_gemm_f16_min_k(int k);
bool f16_enabled();  // gemm_f16 on and the v3 kernels selected (groups then keep row maxima)  // the fp16 split only for K above this (default 128)  // v3 NN / NT: scaled fp16 two-term split (1, default) or 3xTF32 (0)
  // v3 W multicast cluster (1 or 2)  // 1 = both operands in smem (SS), 2 = A split into TMEM (TS, default)  // TN split-K chunk length (rows, multiple of 32); set before creating groups
}  // namespace tc
}  // namespace mg
