// SPDX-License-Identifier: Apache-2.0
//
// Fused output epilogue shared by the SpMM kernels (mg_kernels.cuh) and the GeMMs (mg_tc_gemm.cu).
#pragma once

#include <cuda_runtime.h>

namespace mg {
namespace k {

__device__ __forceinline__ float relu0(float x) { return x > 0.0f ? x : 0.0f; }  // dense.hpp:214

// ---------------------------------------------------------------- fused output epilogue (bias, dropout)
// The optional bias + dropout of a layer's output, applied where the output is produced (the last stage
// of the staged SpMM, or the NN GeMM when layer 0 aggregates first / under order_swap): y = x + b, then
// relu (hidden layers), then dropout y = keep ? y / (1 - p) : 0. The keep mask is a counter-based hash of
// (seed, step, layer) and the element's GLOBAL (row, column): deterministic, P-invariant, and never
// stored — the backward pass recovers it from the output itself (y > 0 <=> kept and active), so the
// relu_backward epilogue only multiplies by 1 / (1 - p). Off (bias == nullptr, thr == 0) the epilogue
// is the identity and every exact-mode result stays bitwise. No reference analogue: the reference has no
// bias or dropout, so these are default-off extensions without a parity claim.
struct Epi {
  const float* bias = nullptr;  // ld-padded (padding entries 0); nullptr = no bias
  unsigned long long key = 0;   // dropout stream of this (seed, step, layer)
  unsigned thr = 0;             // drop when hash < thr (p * 2^32); 0 = no dropout
  float scale = 1.0f;           // 1 / (1 - p)
  long long row0 = 0;           // global row of local row 0
  // Row magnitudes for the next GeMM's scaled fp16 split (mg_tc_gemm.cu F16): when set, the producer writes
  // rmax[2 * row + slot] = max |y| over the values it stored in that row (local row index). A SpMM writes
  // slot 0 and zeroes slot 1; an NN GeMM tile writes slot = its 128-column tile (at most two tiles).
  float* rmax = nullptr;
  int rmax_acc = 0;  // 1: a later column slab of the same rows — fold the stored max in instead of overwriting
};
__device__ __forceinline__ float absmax4(float m, float4 v) {
  return fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
}
// max over the G lanes of a row group; lane 0 of the group writes {max, 0} for local row `row`
__device__ __forceinline__ void rmax_group_store(float m, unsigned gmask, int lane, int G, const Epi& e, long long row) {
  for (int o = G / 2; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(gmask, m, o, G));
  if (lane == 0) {
    float* r = e.rmax + 2 * row;
    *reinterpret_cast<float2*>(r) = make_float2(e.rmax_acc ? fmaxf(m, r[0]) : m, 0.0f);
  }
}
__host__ __device__ __forceinline__ unsigned long long mix64(unsigned long long z) {  // splitmix64 finaliser
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ unsigned dropout_hash(unsigned long long key, long long row, int col) {
  return static_cast<unsigned>(mix64(key + static_cast<unsigned long long>(row * 65536ll + col) * 0x9E3779B97F4A7C15ull) >> 32);
}
__device__ __forceinline__ float epi1(float x, int relu, const Epi& e, long long row, int col) {
  if (e.bias) x = __fadd_rn(x, __ldg(e.bias + col));
  if (relu) x = relu0(x);
  if (e.thr) x = dropout_hash(e.key, e.row0 + row, col) >= e.thr ? __fmul_rn(x, e.scale) : 0.0f;
  return x;
}
__device__ __forceinline__ float4 epi4(float4 a, int relu, const Epi& e, long long row, int col) {
  if (!e.bias && !e.thr) return relu ? make_float4(relu0(a.x), relu0(a.y), relu0(a.z), relu0(a.w)) : a;
  return make_float4(epi1(a.x, relu, e, row, col), epi1(a.y, relu, e, row, col + 1), epi1(a.z, relu, e, row, col + 2),
                     epi1(a.w, relu, e, row, col + 3));
}

}  // namespace k
}  // namespace mg
