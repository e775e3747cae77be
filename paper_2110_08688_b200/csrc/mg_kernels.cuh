// SPDX-License-Identifier: Apache-2.0
//
// sm_100a kernels of the training step (CUDA C++, no libraries):
//   * SpMM over one CSR tile (rowgcn::spmm, inc/sparse.hpp:140-188)  — the hot path
//   * exact SIMT GeMMs (rowgcn::gemm, inc/dense.hpp:140-204) with the fused ReLU epilogues
//   * fused masked softmax cross-entropy + gradient + argmax (inc/dense.hpp:241-277, gcn.hpp:271-290)
//   * fused canonical W-grad block sum + Adam (inc/gcn.hpp:365-377, :61-85)
//   * rank-order reduction for the in-process transport (inc/collectives.hpp:76-94)
// Device layout: every dense activation is row-major with a leading dimension padded to a multiple of
// 4 floats (16-byte rows for float4 traffic); padding columns are kept at +0.0 by every producer.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "mg_epi.cuh"

namespace mg {
namespace k {

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ float fma_free(float acc, float a, float b) {  // acc + a*b, two roundings
  return __fadd_rn(acc, __fmul_rn(a, b));
}
__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void axpy4(float4& acc, float v, const float4& x) {
  acc.x = fma_free(acc.x, v, x.x);
  acc.y = fma_free(acc.y, v, x.y);
  acc.z = fma_free(acc.z, v, x.z);
  acc.w = fma_free(acc.w, v, x.w);
}
__device__ __forceinline__ float relu1(float x) { return x > 0.0f ? x : 0.0f; }  // dense.hpp:214


// FAST-mode edge records carry a hub class in the top 4 bits of the column (mg_device.cu upload_tile):
// class k in 1..7 = the column is among the 10000 * 2^(k-1) most gathered of its tile, 0 = no class.
constexpr int kColMask = 0x0FFFFFFF;

// Edge records are streamed once per (column-slab) pass: mark them evict-first in L2 so they do not
// displace the h rows being gathered (which are what L2 reuse is for).
__device__ __forceinline__ int2 ld_edge(const int2* p) {
  int2 v;
  asm volatile(
      "{\n"
      ".reg .b64 pol;\n"
      "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
      "ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0, %1}, [%2], pol;\n"
      "}\n"
      : "=r"(v.x), "=r"(v.y)
      : "l"(p));
  return v;
}

// ============================================================================ SpMM (exact)
// One row per group of G lanes (G | 32); lane l of the group owns the float4 column chunks
// c = l + k*G (k < CPL). Every output element is a left fold over the row's nonzeros in column
// order with a separate multiply and add — exactly rowgcn::detail::spmm_rows (sparse.hpp:144-153) —
// so the result is bitwise equal to the reference and independent of the launch geometry.
// Rows are visited in `order` (sorted by decreasing length on the host) so the long rows start first.
// Edge records {col, val} are loaded cooperatively (one per lane) and broadcast with shuffles; the
// h-row gathers of U consecutive nonzeros are issued before any of them is consumed (memory-level
// parallelism without changing the accumulation order).
template <int G, int CPL>
__global__ void __launch_bounds__(256) spmm_exact_rows(const int* __restrict__ row_ptr, const int2* __restrict__ edges,
                                                       const int* __restrict__ order, int n_order,
                                                       const float* __restrict__ h, float* __restrict__ out, int ld,
                                                       int nchunk, int accumulate, int relu, Epi ep) {
  constexpr int U = (CPL <= 2) ? 4 : 2;
  const int lane = threadIdx.x & (G - 1);
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
  const int groups = gridDim.x * (blockDim.x / G);
  for (int idx = blockIdx.x * (blockDim.x / G) + threadIdx.x / G; idx < n_order; idx += groups) {
    const int r = order ? __ldg(order + idx) : idx;
    const int e0 = __ldg(row_ptr + r), e1 = __ldg(row_ptr + r + 1);
    float* orow = out + (size_t)r * ld;
    float4 acc[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      const int c = lane + k * G;
      acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (accumulate && c < nchunk) acc[k] = *reinterpret_cast<const float4*>(orow + 4 * c);
    }
    for (int base = e0; base < e1; base += G) {
      const int cnt = min(G, e1 - base);
      const int2 my = lane < cnt ? ld_edge(edges + base + lane) : make_int2(0, 0);
      int j = 0;
      for (; j + U <= cnt; j += U) {
        float4 x[U][CPL];
        float v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int col = __shfl_sync(gmask, my.x, j + u, G);
          v[u] = __int_as_float(__shfl_sync(gmask, my.y, j + u, G));
          const float* hr = h + (size_t)col * ld;
#pragma unroll
          for (int k = 0; k < CPL; ++k) {
            const int c = lane + k * G;
            x[u][k] = c < nchunk ? ldg4(hr + 4 * c) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int k = 0; k < CPL; ++k) axpy4(acc[k], v[u], x[u][k]);
      }
      for (; j < cnt; ++j) {
        const int col = __shfl_sync(gmask, my.x, j, G);
        const float v = __int_as_float(__shfl_sync(gmask, my.y, j, G));
        const float* hr = h + (size_t)col * ld;
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          const int c = lane + k * G;
          if (c < nchunk) axpy4(acc[k], v, ldg4(hr + 4 * c));
        }
      }
    }
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      const int c = lane + k * G;
      if (c < nchunk) *reinterpret_cast<float4*>(orow + 4 * c) = epi4(acc[k], relu, ep, r, 4 * c);
    }
  }
}

// ============================================================================ SpMM (fast)
// MG_SPMM_FAST: the same lane-group gather, with two differences that trade bitwise parity with the
// reference for speed (the result stays deterministic and within fp32 rounding of it):
//   * fused multiply-add per nonzero;
//   * rows with >= heavy_row nonzeros are cut into fixed segments of `seg` nonzeros that are gathered
//     in parallel like ordinary rows into a scratch buffer, then summed in segment order by
//     spmm_fast_hubs — the hub rows no longer serialise on one CTA.
// Work items are int4 {e_begin, e_end, dst, 0}: dst >= 0 is an output row (accumulate / relu apply),
// dst < 0 is scratch segment -dst-1 (plain store).
__device__ __forceinline__ void fma4(float4& acc, float v, const float4& x) {
  acc.x = fmaf(v, x.x, acc.x);
  acc.y = fmaf(v, x.y, acc.y);
  acc.z = fmaf(v, x.z, acc.z);
  acc.w = fmaf(v, x.w, acc.w);
}

template <int G, int CPL>
__global__ void __launch_bounds__(256) spmm_fast_items(const int4* __restrict__ items, int n_items,
                                                       const int2* __restrict__ edges, const float* __restrict__ h,
                                                       float* __restrict__ out, float* __restrict__ scratch, int ld,
                                                       int nchunk, int accumulate, int relu, Epi ep) {
  constexpr int U = (CPL <= 2) ? 4 : 2;
  const int lane = threadIdx.x & (G - 1);
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
  const int groups = gridDim.x * (blockDim.x / G);
  for (int idx = blockIdx.x * (blockDim.x / G) + threadIdx.x / G; idx < n_items; idx += groups) {
    const int4 it = __ldg(items + idx);
    const int e0 = it.x, e1 = it.y;
    const bool seg = it.z < 0;
    float* orow = seg ? scratch + (size_t)(-it.z - 1) * ld : out + (size_t)it.z * ld;
    float4 acc[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      const int c = lane + k * G;
      acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (!seg && accumulate && c < nchunk) acc[k] = *reinterpret_cast<const float4*>(orow + 4 * c);
    }
    for (int base = e0; base < e1; base += G) {
      const int cnt = min(G, e1 - base);
      const int2 my = lane < cnt ? ld_edge(edges + base + lane) : make_int2(0, 0);
      int j = 0;
      for (; j + U <= cnt; j += U) {
        float4 x[U][CPL];
        float v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int col = __shfl_sync(gmask, my.x, j + u, G) & kColMask;
          v[u] = __int_as_float(__shfl_sync(gmask, my.y, j + u, G));
          const float* hr = h + (size_t)col * ld;
#pragma unroll
          for (int k = 0; k < CPL; ++k) {
            const int c = lane + k * G;
            x[u][k] = c < nchunk ? ldg4(hr + 4 * c) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int k = 0; k < CPL; ++k) fma4(acc[k], v[u], x[u][k]);
      }
      for (; j < cnt; ++j) {
        const int col = __shfl_sync(gmask, my.x, j, G) & kColMask;
        const float v = __int_as_float(__shfl_sync(gmask, my.y, j, G));
        const float* hr = h + (size_t)col * ld;
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          const int c = lane + k * G;
          if (c < nchunk) fma4(acc[k], v, ldg4(hr + 4 * c));
        }
      }
    }
    float m = 0.0f;
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      const int c = lane + k * G;
      if (c < nchunk) {
        const float4 y = seg ? acc[k] : epi4(acc[k], relu, ep, it.z, 4 * c);
        *reinterpret_cast<float4*>(orow + 4 * c) = y;
        m = absmax4(m, y);
      }
    }
    if (!seg && ep.rmax) rmax_group_store(m, gmask, lane, G, ep, it.z);
  }
}

// MG_SPMM_FAST, cp.async-pipelined: the same per-lane FMA chain as spmm_fast_items (bitwise identical
// results), but the h-row gathers land in a per-group shared-memory ring (LDGSTS, no registers held while
// in flight), so D-1 stages of E nonzeros stay in flight per group instead of U. The gather addresses come
// from edge records held in three rotating G-record register windows (current, next, prefetched), so no
// gather waits on its own edge-record load. Requires E | G and (D - 1) * E <= G.
__device__ __forceinline__ void cp_async16_cg(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ void cp_async16_hint(void* smem, const void* gmem, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem), "l"(pol)
               : "memory");
}

// hub_max >= 0: gathers of columns of class 1..hub_max are marked L2 evict_last (they stay resident:
// the hub rows of the power-law graph are re-gathered by many rows), every other gather evict_first.
template <int G, int CPL, int E, int D, bool HINT>
__global__ void __launch_bounds__(128) spmm_fast_async(const int4* __restrict__ items, int n_items,
                                                       const int2* __restrict__ edges, const float* __restrict__ h,
                                                       float* __restrict__ out, float* __restrict__ scratch, int ld,
                                                       int nchunk, int accumulate, int relu, int hub_max, Epi ep) {
  static_assert(G % E == 0 && (D - 1) * E <= G, "pipeline depth must stay within one record window");
  uint64_t pol_last = 0, pol_first = 0;
  if (HINT) {
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol_last));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol_first));
  }
  extern __shared__ float4 ring_all[];
  const int lane = threadIdx.x & (G - 1);
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
  float4* ring = ring_all + (size_t)(threadIdx.x / G) * (D * E * CPL * G);  // [D][E][CPL][G]
  const int groups = gridDim.x * (blockDim.x / G);
  for (int idx = blockIdx.x * (blockDim.x / G) + threadIdx.x / G; idx < n_items; idx += groups) {
    const int4 it = __ldg(items + idx);
    const int e0 = it.x, n = it.y - it.x;
    const bool seg = it.z < 0;
    float* orow = seg ? scratch + (size_t)(-it.z - 1) * ld : out + (size_t)it.z * ld;
    float4 acc[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      const int c = lane + k * G;
      acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (!seg && accumulate && c < nchunk) acc[k] = *reinterpret_cast<const float4*>(orow + 4 * c);
    }
    auto win = [&](int w) {
      const int i = w * G + lane;
      return i < n ? ld_edge(edges + e0 + i) : make_int2(0, 0);
    };
    int2 wa = win(0), wb = win(1), wc = win(2);  // records of windows wi, wi + 1, wi + 2
    int wi = 0;
    const int nst = (n + E - 1) / E;
    auto issue = [&](int t) {  // gathers of stage t (edges t*E .. t*E+E-1) into slot t % D
      float4* slot = ring + (t % D) * (E * CPL * G);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = t * E + e;
        const int src = (i / G == wi) ? wa.x : wb.x;
        const int rec = __shfl_sync(gmask, src, i & (G - 1), G);
        if (i < n) {
          const float* hr = h + (size_t)(rec & kColMask) * ld;
          if (HINT) {
            const int cls = static_cast<int>(static_cast<unsigned>(rec) >> 28);
            const uint64_t pol = (cls != 0 && cls <= hub_max) ? pol_last : pol_first;
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              const int c = lane + k * G;
              if (c < nchunk) cp_async16_hint(slot + (e * CPL + k) * G + lane, hr + 4 * c, pol);
            }
          } else {
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              const int c = lane + k * G;
              if (c < nchunk) cp_async16_cg(slot + (e * CPL + k) * G + lane, hr + 4 * c);
            }
          }
        }
      }
    };
#pragma unroll
    for (int t = 0; t < D - 1; ++t) {
      if (t < nst) issue(t);
      cp_async_commit();
    }
    for (int t = 0; t < nst; ++t) {
      if (t > 0 && (t * E) % G == 0) {  // consumption enters window wi + 1
        wa = wb;
        wb = wc;
        ++wi;
        wc = win(wi + 2);
      }
      if (t + D - 1 < nst) issue(t + D - 1);
      cp_async_commit();
      cp_async_wait<D - 1>();
      const float4* slot = ring + (t % D) * (E * CPL * G);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = t * E + e;
        const float v = __int_as_float(__shfl_sync(gmask, wa.y, i & (G - 1), G));
        if (i < n) {
#pragma unroll
          for (int k = 0; k < CPL; ++k)
            if (lane + k * G < nchunk) fma4(acc[k], v, slot[(e * CPL + k) * G + lane]);
        }
      }
    }
    cp_async_wait<0>();
    float m = 0.0f;
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      const int c = lane + k * G;
      if (c < nchunk) {
        const float4 y = seg ? acc[k] : epi4(acc[k], relu, ep, it.z, 4 * c);
        *reinterpret_cast<float4*>(orow + 4 * c) = y;
        m = absmax4(m, y);
      }
    }
    if (!seg && ep.rmax) rmax_group_store(m, gmask, lane, G, ep, it.z);
  }
}

// MG_SPMM_FAST, row-streaming: the cp.async ring of spmm_fast_async kept full ACROSS rows. A work item is
// a piece {r0, r1, e0, e1} of consecutive light rows (their edges contiguous, e0 = rp[r0], e1 = rp[r1])
// or a hub-row segment {-(seg+1), 0, e0, e1}; the group streams the piece's nonzeros through the ring in
// stages of E and closes a row (epilogue store, accumulator reset) when the consumption cursor crosses
// the row's end, read from register windows of G row ends (lane l holds the end of row rb + l). Short rows no longer pay one DRAM latency each (spmm_fast_async drains its ring at every
// row end): the pipeline drains once per piece. Per output element the FMA chain is the same as
// spmm_fast_async's (acc = accumulate ? old : 0, then one fmaf per nonzero in column order), so results
// are bitwise identical. With accumulate the next row's old output is prefetched into registers when a
// row starts. Requires E | G and (D - 1) * E <= G.
template <int G, int CPL, int E, int D, bool HINT>
__global__ void __launch_bounds__(128) spmm_fast_stream(const int4* __restrict__ pieces, int n_pieces,
                                                        const int* __restrict__ row_ptr, const int2* __restrict__ edges,
                                                        const float* __restrict__ h, float* __restrict__ out,
                                                        float* __restrict__ scratch, int ld, int nchunk, int accumulate,
                                                        int relu, int hub_max, Epi ep) {
  static_assert(G % E == 0 && (D - 1) * E <= G, "pipeline depth must stay within one record window");
  uint64_t pol_last = 0, pol_first = 0;
  if (HINT) {
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol_last));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol_first));
  }
  extern __shared__ float4 ring_all[];
  const int lane = threadIdx.x & (G - 1);
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
  float4* ring = ring_all + (size_t)(threadIdx.x / G) * (D * E * CPL * G);  // [D][E][CPL][G]
  const int groups = gridDim.x * (blockDim.x / G);
  for (int idx = blockIdx.x * (blockDim.x / G) + threadIdx.x / G; idx < n_pieces; idx += groups) {
    const int4 pc = __ldg(pieces + idx);
    const bool seg = pc.x < 0;
    const int e0 = pc.z, n = pc.w - pc.z;
    const int nrows = seg ? 1 : pc.y - pc.x;
    const bool acc_in = accumulate && !seg;
    // row ends relative to e0 in two register windows of G rows (rows rb + lane, rb + G + lane; n past the
    // piece); the window after next is loaded when consumption enters the second one
    auto rwin = [&](int base) {
      const int r = base + lane;
      return (!seg && r < nrows) ? __ldg(row_ptr + pc.x + r + 1) - e0 : n;
    };
    int rb = 0, rend = rwin(0), rend2 = rwin(G);
    auto orow = [&](int r) -> float* {
      return seg ? scratch + (size_t)(-pc.x - 1) * ld : out + (size_t)(pc.x + r) * ld;
    };
    float4 acc[CPL], nxt[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      const int c = lane + k * G;
      acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      nxt[k] = acc[k];
      if (acc_in && c < nchunk) {
        acc[k] = *reinterpret_cast<const float4*>(orow(0) + 4 * c);
        if (nrows > 1) nxt[k] = *reinterpret_cast<const float4*>(orow(1) + 4 * c);
      }
    }
    int cur = 0;
    int cur_end = __shfl_sync(gmask, rend, 0, G);
    // closes row `cur` and opens the next one (accumulator from the prefetched old output)
    auto close_row = [&]() {
      float* o = orow(cur);
      float m = 0.0f;
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        const int c = lane + k * G;
        if (c < nchunk) {
          const float4 y = seg ? acc[k] : epi4(acc[k], relu, ep, pc.x + cur, 4 * c);
          *reinterpret_cast<float4*>(o + 4 * c) = y;
          m = absmax4(m, y);
        }
      }
      if (!seg && ep.rmax) rmax_group_store(m, gmask, lane, G, ep, pc.x + cur);
      ++cur;
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        const int c = lane + k * G;
        acc[k] = acc_in ? nxt[k] : make_float4(0.f, 0.f, 0.f, 0.f);
        if (acc_in && cur + 1 < nrows && c < nchunk) nxt[k] = *reinterpret_cast<const float4*>(orow(cur + 1) + 4 * c);
      }
      if (cur - rb == G) {
        rb += G;
        rend = rend2;
        rend2 = rwin(rb + G);
      }
      cur_end = __shfl_sync(gmask, rend, cur - rb, G);
    };
    auto win = [&](int w) {
      const int i = w * G + lane;
      return i < n ? ld_edge(edges + e0 + i) : make_int2(0, 0);
    };
    int2 wa = win(0), wb = win(1), wc = win(2);  // records of windows wi, wi + 1, wi + 2
    int wi = 0;
    const int nst = (n + E - 1) / E;
    auto issue = [&](int t) {  // gathers of stage t (edges t*E .. t*E+E-1) into slot t % D
      float4* slot = ring + (t % D) * (E * CPL * G);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = t * E + e;
        const int src = (i / G == wi) ? wa.x : wb.x;
        const int rec = __shfl_sync(gmask, src, i & (G - 1), G);
        if (i < n) {
          const float* hr = h + (size_t)(rec & kColMask) * ld;
          if (HINT) {
            const int cls = static_cast<int>(static_cast<unsigned>(rec) >> 28);
            const uint64_t pol = (cls != 0 && cls <= hub_max) ? pol_last : pol_first;
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              const int c = lane + k * G;
              if (c < nchunk) cp_async16_hint(slot + (e * CPL + k) * G + lane, hr + 4 * c, pol);
            }
          } else {
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              const int c = lane + k * G;
              if (c < nchunk) cp_async16_cg(slot + (e * CPL + k) * G + lane, hr + 4 * c);
            }
          }
        }
      }
    };
#pragma unroll
    for (int t = 0; t < D - 1; ++t) {
      if (t < nst) issue(t);
      cp_async_commit();
    }
    for (int t = 0; t < nst; ++t) {
      if (t > 0 && (t * E) % G == 0) {  // consumption enters window wi + 1
        wa = wb;
        wb = wc;
        ++wi;
        wc = win(wi + 2);
      }
      if (t + D - 1 < nst) issue(t + D - 1);
      cp_async_commit();
      cp_async_wait<D - 1>();
      const float4* slot = ring + (t % D) * (E * CPL * G);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = t * E + e;
        const float v = __int_as_float(__shfl_sync(gmask, wa.y, i & (G - 1), G));
        if (i < n) {
          while (i >= cur_end) close_row();  // uniform across the group
#pragma unroll
          for (int k = 0; k < CPL; ++k)
            if (lane + k * G < nchunk) fma4(acc[k], v, slot[(e * CPL + k) * G + lane]);
        }
      }
    }
    cp_async_wait<0>();
    while (cur < nrows) close_row();  // the last row and trailing empty rows
  }
}

// Upload time, FAST work lists: sort keys for the light rows (ht - length; hub rows 2 ht) and the items.
__global__ void light_keys(const int* __restrict__ rp, int rows, int ht, int* __restrict__ keys, int* __restrict__ ids) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    const int len = rp[r + 1] - rp[r];
    keys[r] = len < ht ? ht - len : 2 * ht;
    ids[r] = r;
  }
}
__global__ void light_fill(const int* __restrict__ rp, const int* __restrict__ ids, int n_light, int4* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_light; i += gridDim.x * blockDim.x) {
    const int r = ids[i];
    out[i] = make_int4(rp[r], rp[r + 1], r, 0);
  }
}

// Upload time: interleave the tile's column and value arrays into {col, value bits} records.
__global__ void pack_edges(const int* __restrict__ col, const float* __restrict__ val, long nnz,
                           int2* __restrict__ edges) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < nnz; i += (long)gridDim.x * blockDim.x)
    edges[i] = make_int2(col[i], __float_as_int(val[i]));
}

// Hub classes of a FAST tile (upload time): gather counts per column, a histogram of the counts (capped),
// and the tag pass: class k in 1..7 when count >= thr[k-1] (thr non-increasing), else 0.
constexpr int kHubCountCap = 1 << 16;
struct HubTiers {
  int thr[7];
};
__global__ void hub_count(const int2* __restrict__ edges, long nnz, int* __restrict__ cnt) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < nnz; i += (long)gridDim.x * blockDim.x)
    atomicAdd(cnt + (edges[i].x & kColMask), 1);
}
__global__ void hub_count_hist(const int* __restrict__ cnt, long cols, int* __restrict__ hist) {
  for (long c = blockIdx.x * (long)blockDim.x + threadIdx.x; c < cols; c += (long)gridDim.x * blockDim.x)
    atomicAdd(hist + min(cnt[c], kHubCountCap), 1);
}
__global__ void hub_tag(int2* __restrict__ edges, long nnz, const int* __restrict__ cnt, HubTiers t) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < nnz; i += (long)gridDim.x * blockDim.x) {
    const int col = edges[i].x & kColMask;
    const int c = cnt[col];
    int k = 0;
#pragma unroll
    for (int q = 6; q >= 0; --q)
      if (c >= t.thr[q]) k = q + 1;
    edges[i].x = col | (k << 28);
  }
}

// hubs[i] = {row, first segment, segment count}: out[row] = (acc ? out[row] : 0) + sum of its segments in
// order, then relu. One CTA per hub row, threads over float4 chunks.
__global__ void __launch_bounds__(256) spmm_fast_hubs(const int4* __restrict__ hubs, const float* __restrict__ scratch,
                                                      float* __restrict__ out, int ld, int accumulate, int relu, Epi ep) {
  const int4 hb = hubs[blockIdx.x];
  float* orow = out + (size_t)hb.x * ld;
  float m = 0.0f;
  for (int c = threadIdx.x; c < ld / 4; c += blockDim.x) {
    float4 s = accumulate ? *reinterpret_cast<const float4*>(orow + 4 * c) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
    for (int q = 0; q < hb.z; ++q) {  // unrolled: the segment loads go out together, the sum stays in order
      const float4 p = *reinterpret_cast<const float4*>(scratch + (size_t)(hb.y + q) * ld + 4 * c);
      s.x += p.x;
      s.y += p.y;
      s.z += p.z;
      s.w += p.w;
    }
    const float4 y = epi4(s, relu, ep, hb.x, 4 * c);
    *reinterpret_cast<float4*>(orow + 4 * c) = y;
    m = absmax4(m, y);
  }
  if (ep.rmax) {  // block max of the hub row
    __shared__ float red[8];
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) m = fmaxf(m, red[w]);
      *reinterpret_cast<float2*>(ep.rmax + 2 * hb.x) = make_float2(m, 0.0f);
    }
  }
}

// Long rows (hubs of the power-law graph): one CTA per (row, 64-column slab), warp-specialised.
// Warps 2-3 (producers) stream the row's h-slabs into an NST-deep ring of 32-nonzero stages with
// 16-byte cp.async (completion tracked per stage by cp.async.mbarrier.arrive); the stage's edge
// records arrive ahead of time in a second ring by one TMA bulk copy per stage (per-nonzero bulk copies
// were measured to be issue-bound on the TMA unit). Warps 0-1 (consumers, one output column per
// thread) fold each stage in column order with a separate multiply and add — the same left fold as
// above, so still bitwise exact — and release the stage through a second mbarrier.
constexpr int kHeavySlab = 64;
constexpr int kHeavyB = 32;
constexpr int kHeavyNst = 8;
constexpr int kHeavyThreads = 128;  // warps 0-1 consume (one column each), warps 2-3 produce
constexpr int kHeavyEslots = 16;  // edge-record ring (2 x the stage ring: reuse needs consumption)
constexpr size_t kHeavySmem = sizeof(float) * kHeavyNst * kHeavyB * kHeavySlab + 8 * kHeavyEslots * (kHeavyB + 2) +
                              8 * (2 * kHeavyNst + kHeavyEslots) + 128;
constexpr int kEdgePad = 2;  // edge arrays carry 2 spare records so the aligned bulk copies stay in bounds

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

__global__ void __launch_bounds__(kHeavyThreads) spmm_exact_heavy(const int* __restrict__ row_ptr,
                                                                  const int2* __restrict__ edges,
                                                                  const int* __restrict__ heavy, int nslab,
                                                                  const float* __restrict__ h, float* __restrict__ out,
                                                                  int ld, int accumulate, int relu, Epi ep) {
  extern __shared__ __align__(128) float smem[];
  float* buf = smem;                                                            // [NST][B][SLAB] h slabs
  int2* ering = reinterpret_cast<int2*>(smem + kHeavyNst * kHeavyB * kHeavySlab);  // [ESLOTS][B + 2] edge records
  uint64_t* full = reinterpret_cast<uint64_t*>(ering + kHeavyEslots * (kHeavyB + 2));
  uint64_t* empty = full + kHeavyNst;
  uint64_t* efull = empty + kHeavyNst;
  const int r = heavy[blockIdx.x / nslab];
  const int col0 = (blockIdx.x % nslab) * kHeavySlab;
  const int e0 = row_ptr[r], e1 = row_ptr[r + 1];
  const int nst_total = (e1 - e0 + kHeavyB - 1) / kHeavyB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t slab_bytes = static_cast<uint32_t>(min(kHeavySlab, ld - col0)) * 4u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kHeavyNst; ++s) {
      mbar_init(&full[s], 64);  // one cp.async.mbarrier.arrive.noinc per producer thread
      mbar_init(&empty[s], 64);
    }
    for (int s = 0; s < kHeavyEslots; ++s) mbar_init(&efull[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // Edge records of stage q arrive by one bulk copy (16-byte aligned start, so the copy may begin one
  // record early and end one late: the edge array is padded) into slot q % ESLOTS, kHeavyNst stages
  // ahead of use; the slot's previous occupant (stage q - ESLOTS) is long consumed by then.
  auto issue_edges = [&](int q) {
    const int base = e0 + q * kHeavyB;
    const int al = base & ~1;
    const int n = (min(kHeavyB, e1 - base) + (base - al) + 1) & ~1;
    const int slot = q % kHeavyEslots;
    mbar_arrive_tx(&efull[slot], static_cast<uint32_t>(n) * 8u);
    bulk_g2s(ering + slot * (kHeavyB + 2), edges + al, static_cast<uint32_t>(n) * 8u, &efull[slot]);
  };
  if (warp >= 2) {  // producers (warps 2-3): 16-byte cp.async per thread, completion tracked per stage
    const int pt = threadIdx.x - 64;  // 0..63
    const int nchunk = static_cast<int>(slab_bytes / 16);
    if (pt == 0)
      for (int q = 0; q < min(kHeavyNst, nst_total); ++q) issue_edges(q);
    for (int st = 0; st < nst_total; ++st) {
      const int s = st % kHeavyNst;
      if (st >= kHeavyNst) mbar_wait(&empty[s], ((st / kHeavyNst) - 1) & 1);  // consumer is done with st - NST
      if (pt == 0 && st + kHeavyNst < nst_total) issue_edges(st + kHeavyNst);
      const int slot = st % kHeavyEslots;
      mbar_wait(&efull[slot], (st / kHeavyEslots) & 1);
      const int base = e0 + st * kHeavyB;
      const int cnt = min(kHeavyB, e1 - base);
      const int2* er = ering + slot * (kHeavyB + 2) + (base & 1);
      float* dst = buf + (size_t)s * kHeavyB * kHeavySlab;
      for (int q = pt; q < cnt * (kHeavySlab / 4); q += 64) {
        const int b = q / (kHeavySlab / 4), c = q % (kHeavySlab / 4);
#ifdef MG_RACECHECK_PLAIN_COPIES
        // racecheck build only (build.py --racecheck): the same ring protocol with plain loads / stores and a
        // per-thread arrival, a form compute-sanitizer racecheck models (it does not model cp.async
        // completion through mbarriers)
        if (c < nchunk)
          *reinterpret_cast<float4*>(dst + b * kHeavySlab + 4 * c) =
              *reinterpret_cast<const float4*>(h + (size_t)er[b].x * ld + col0 + 4 * c);
      }
      mbar_arrive(&full[s]);
#else
        if (c < nchunk) cp_async16(dst + b * kHeavySlab + 4 * c, h + (size_t)er[b].x * ld + col0 + 4 * c);
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_addr(&full[s])) : "memory");
#endif
    }
  } else {  // consumers: one column each
    const int t = threadIdx.x;
    const int my_col = col0 + t;
    const bool active = my_col < ld;
    float acc = 0.0f;
    if (active && accumulate) acc = out[(size_t)r * ld + my_col];
    for (int st = 0; st < nst_total; ++st) {
      const int s = st % kHeavyNst;
      mbar_wait(&full[s], (st / kHeavyNst) & 1);
      const int base = e0 + st * kHeavyB;
      const int cnt = min(kHeavyB, e1 - base);
      const float* bs = buf + (size_t)s * kHeavyB * kHeavySlab + t;
      const int2* er = ering + (st % kHeavyEslots) * (kHeavyB + 2) + (base & 1);
      if (active) {
        if (cnt == kHeavyB) {  // full stage: all 64 smem loads in flight, then the 32-long add chain
          float x[kHeavyB], v[kHeavyB];
#pragma unroll
          for (int b = 0; b < kHeavyB; ++b) {
            v[b] = __int_as_float(er[b].y);
            x[b] = bs[b * kHeavySlab];
          }
#pragma unroll
          for (int b = 0; b < kHeavyB; ++b) acc = fma_free(acc, v[b], x[b]);
        } else {
          for (int b = 0; b < cnt; ++b) acc = fma_free(acc, __int_as_float(er[b].y), bs[b * kHeavySlab]);
        }
      }
      mbar_arrive(&empty[s]);  // per consumer thread (an elected arrival after __syncwarp is not modelled by racecheck)
    }
    if (active) out[(size_t)r * ld + my_col] = (ep.bias || ep.thr) ? epi1(acc, relu, ep, r, my_col) : (relu ? relu1(acc) : acc);
  }
}

// ============================================================================ GeMM (exact SIMT)
// C[M,N] = op(A) op(B) with the reference's per-element order: k ascending, separate multiply and
// add; NN/TN skip zero A entries (dense.hpp:165, :177); NT forms the dot product then adds it to a
// zeroed output (dense.hpp:189-191, i.e. 0 + acc). 64x64 tiles, 256 threads, 4x4 outputs each.
// EPI 0: store; 1: relu_backward in place, C = C_old > 0 ? r : 0 (dense.hpp:221-231); 2: relu. EPI 0 / 2
// add the optional bias and apply the optional dropout (Epi); EPI 1 scales the kept entries by 1 / (1 - p).
constexpr int kGBM = 64, kGBN = 64, kGBK = 16;

template <bool TA, bool TB, int EPI>
__global__ void __launch_bounds__(256) gemm_exact(int M, int N, int K, const float* __restrict__ A, long lda,
                                                  const float* __restrict__ B, long ldb, float* __restrict__ C,
                                                  long ldc, Epi ep) {
  __shared__ float As[kGBK][kGBM + 4];
  __shared__ float Bs[kGBK][kGBN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const long m0 = (long)blockIdx.x * kGBM;  // M (rows of the activations) on x: no 65535 limit
  const int n0 = blockIdx.y * kGBN;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
  for (int k0 = 0; k0 < K; k0 += kGBK) {
    // A tile -> As[kk][i]
    for (int q = tid; q < kGBK * kGBM; q += 256) {
      int kk, i;
      if (TA) { kk = q / kGBM; i = q % kGBM; } else { i = q / kGBK; kk = q % kGBK; }
      const long m = m0 + i;
      const int kx = k0 + kk;
      float v = 0.0f;
      if (m < M && kx < K) v = TA ? A[(long)kx * lda + m] : A[m * lda + kx];
      As[kk][i] = v;
    }
    for (int q = tid; q < kGBK * kGBN; q += 256) {
      int kk, j;
      if (TB) { j = q / kGBK; kk = q % kGBK; } else { kk = q / kGBN; j = q % kGBN; }
      const int n = n0 + j;
      const int kx = k0 + kk;
      float v = 0.0f;
      if (n < N && kx < K) v = TB ? B[(long)n * ldb + kx] : B[(long)kx * ldb + n];
      Bs[kk][j] = v;
    }
    __syncthreads();
    const int kmax = min(kGBK, K - k0);
    for (int kk = 0; kk < kmax; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (!TB && a[i] == 0.0f) continue;  // NN/TN zero skip
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma_free(acc[i][j], a[i], b[j]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const long m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float r = acc[i][j];
      if (TB) r = __fadd_rn(0.0f, r);  // out(i,j) += acc on a zeroed out
      float* cp = C + m * ldc + n;
      if (EPI == 1) r = (*cp > 0.0f) ? (ep.thr ? __fmul_rn(r, ep.scale) : r) : 0.0f;  // dropout-kept: x 1/(1-p)
      else r = epi1(r, EPI == 2, ep, m, n);
      *cp = r;
    }
  }
}

// ============================================================================ loss
// Masked softmax cross-entropy over the logits rows, gradient written in place (softmax - onehot) /
// denom (dense.hpp:241-277), argmax with first-max-wins ties (gcn.hpp:279-282). One warp per row,
// C <= 32*kLossCpl. Per-block partial sums (fp64) land in `partials`; finalize_stats sums them in a
// fixed order so the reported loss is run-to-run deterministic.
constexpr int kLossCpl = 8;

template <int CPL, int LPR = 32>  // LPR lanes per row (32 or 16: two rows per warp), C <= LPR * CPL
__global__ void __launch_bounds__(256) softmax_xent(float* __restrict__ logits, int ld, int rows, int C,
                                                    const int* __restrict__ labels, const uint8_t* __restrict__ mask,
                                                    float inv_denom, double* __restrict__ partials) {
  static_assert(LPR == 32 || LPR == 16 || LPR == 8, "a row spans a warp, a half or a quarter warp");
  constexpr int RPW = 32 / LPR;  // rows per warp
  __shared__ double s_loss[8], s_corr[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lr = lane & (LPR - 1), slot = lane / LPR;
  double my_loss = 0.0, my_corr = 0.0;
  const int stride = gridDim.x * 8 * RPW;
  // the next row's logits, label and mask are loaded while the current row is reduced (one row per warp
  // in flight was latency-bound); rows past the end read as masked
  auto load = [&](int r, float* z, int& label, int& m) {
    m = 0;
    label = 0;
#pragma unroll
    for (int q = 0; q < CPL; ++q) z[q] = -INFINITY;
    if (r >= rows) return;
    m = mask[r];
    label = labels[r];
    const float* row = logits + (size_t)r * ld;
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int j = lr + LPR * q;
      if (j < C) z[q] = row[j];
    }
  };
  float zn[CPL];
  int label_n = 0, m_n = 0;
  load((blockIdx.x * 8 + warp) * RPW + slot, zn, label_n, m_n);
  // warp-uniform loop over groups of RPW rows: every lane takes part in every shuffle
  for (int base = (blockIdx.x * 8 + warp) * RPW; base < rows; base += stride) {
    const int r = base + slot;
    float z[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) z[q] = zn[q];
    const int label = label_n, m = m_n;
    load(r + stride, zn, label_n, m_n);
    float mx = -INFINITY;
    int arg = 0x7fffffff;
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int j = lr + LPR * q;
      if (j < C && (arg == 0x7fffffff || z[q] > mx)) {
        mx = z[q];
        arg = j;
      }
    }
    // (max, first index) reduction over the row's lanes: strictly greater wins, ties keep the smaller index
#pragma unroll
    for (int off = LPR / 2; off; off >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, mx, off);
      const int oa = __shfl_xor_sync(0xffffffffu, arg, off);
      if (oa != 0x7fffffff && (arg == 0x7fffffff || om > mx || (om == mx && oa < arg))) {
        mx = om;
        arg = oa;
      }
    }
    float se = 0.0f, ex[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int j = lr + LPR * q;
      ex[q] = j < C ? expf(z[q] - mx) : 0.0f;
      if (j < C) se += ex[q];
    }
#pragma unroll
    for (int off = LPR / 2; off; off >>= 1) se += __shfl_xor_sync(0xffffffffu, se, off);
    float zlab = 0.0f;
#pragma unroll
    for (int q = 0; q < CPL; ++q)
      if (label == lr + LPR * q) zlab = z[q];
    zlab = __shfl_sync(0xffffffffu, zlab, label & (LPR - 1), LPR);
    if (r < rows) {
      float* row = logits + (size_t)r * ld;
      if (!m) {
        for (int j = lr; j < ld; j += LPR) row[j] = 0.0f;
      } else {
        if (lr == 0) {
          my_loss += (double)(logf(se) - (zlab - mx));
          my_corr += (arg == label) ? 1.0 : 0.0;
        }
        const float scale = __fdiv_rn(inv_denom, se);  // one division per row: g = e^(z - max) * (1/denom) / sum
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
          const int j = lr + LPR * q;
          if (j < C) {
            float g = __fmul_rn(ex[q], scale);
            if (j == label) g = __fsub_rn(g, inv_denom);
            row[j] = g;
          }
        }
        for (int j = C + lr; j < ld; j += LPR) row[j] = 0.0f;
      }
    }
  }
  // the other row slots' leaders (lanes LPR, 2 LPR, ...) hand their sums to lane 0
#pragma unroll
  for (int off = LPR; off < 32; off <<= 1) {
    my_loss += __shfl_down_sync(0xffffffffu, my_loss, off);
    my_corr += __shfl_down_sync(0xffffffffu, my_corr, off);
  }
  if (lane == 0) {
    s_loss[warp] = my_loss;
    s_corr[warp] = my_corr;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < 8; ++w) {
      a += s_loss[w];
      b += s_corr[w];
    }
    partials[2 * blockIdx.x] = a;
    partials[2 * blockIdx.x + 1] = b;
  }
}

__global__ void finalize_stats(const double* __restrict__ partials, int nblocks, double* __restrict__ stats) {
  // one warp: lane l sums blocks l, l + 32, ... in order, then a fixed xor tree — the same order every
  // run (a serial sum over ~1200 partial pairs took ~80 us)
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nblocks; i += 32) {
    a += partials[2 * i];
    b += partials[2 * i + 1];
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, off);
    b += __shfl_xor_sync(0xffffffffu, b, off);
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    stats[0] = a;
    stats[1] = b;
  }
}

// ============================================================================ W-grad finalize + Adam
// w_grad = 0 + stage[0] + ... + stage[7] in block order (gcn.hpp:365-377), then Adam with the
// reference's float constants and operation order (gcn.hpp:61-85), grads zeroed afterwards.
// Works on the padded d_l x ld_{l+1} arrays; padding stays exactly 0.
struct AdamConsts {
  float b1, one_m_b1, b2, one_m_b2, lr, eps, corr1, corr2;
};

__global__ void finalize_adam(int size, int blocks, const float* __restrict__ stage, float* __restrict__ w,
                              float* __restrict__ g, float* __restrict__ m, float* __restrict__ v, int run_adam,
                              AdamConsts c) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < size; i += gridDim.x * blockDim.x) {
    float s = 0.0f;
    for (int b = 0; b < blocks; ++b) s = __fadd_rn(s, stage[(size_t)b * size + i]);
    if (!run_adam) {
      g[i] = s;
      continue;
    }
    const float mi = __fadd_rn(__fmul_rn(c.b1, m[i]), __fmul_rn(c.one_m_b1, s));
    const float vi = __fadd_rn(__fmul_rn(c.b2, v[i]), __fmul_rn(__fmul_rn(c.one_m_b2, s), s));
    const float mhat = __fdiv_rn(mi, c.corr1);
    const float vhat = __fdiv_rn(vi, c.corr2);
    m[i] = mi;
    v[i] = vi;
    w[i] = __fsub_rn(w[i], __fdiv_rn(__fmul_rn(c.lr, mhat), __fadd_rn(__fsqrt_rn(vhat), c.eps)));
    g[i] = 0.0f;
  }
}

// ============================================================================ bias gradient (extension)
// dL/db_l = column sums of dL/dz_l over the rows of each canonical W-grad block (gcn.hpp:309-331 applied to
// a bias row), deterministic: fixed 1024-row chunks from the block's first local row, each folded
// sequentially per column, then the chunk partials summed in chunk order. For P | 8 no block spans two
// workers (uniform_partition bounds coincide), so the result is bitwise P-invariant like W_G.
constexpr int kBiasChunk = 1024;
struct BlockRanges {
  long long begin[8], len[8];
};
__global__ void bias_partials(const float* __restrict__ G, int ld, BlockRanges br, int max_chunks,
                              float* __restrict__ partial) {
  const int b = blockIdx.y, c = blockIdx.x;
  const long long r0 = br.begin[b] + static_cast<long long>(c) * kBiasChunk;
  const long long r1 = min(r0 + kBiasChunk, br.begin[b] + br.len[b]);
  for (int col = threadIdx.x; col < ld; col += blockDim.x) {
    float acc = 0.0f;
    for (long long r = r0; r < r1; ++r) acc = __fadd_rn(acc, G[r * ld + col]);
    partial[(static_cast<long long>(b) * max_chunks + c) * ld + col] = acc;
  }
}
__global__ void bias_reduce(const float* __restrict__ partial, BlockRanges br, int max_chunks, int ld,
                            float* __restrict__ out, long long block_stride) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 8 * ld; i += gridDim.x * blockDim.x) {
    const int b = i / ld, col = i % ld;
    const int nch = static_cast<int>((br.len[b] + kBiasChunk - 1) / kBiasChunk);
    float s = 0.0f;
    for (int c = 0; c < nch; ++c) s = __fadd_rn(s, partial[(static_cast<long long>(b) * max_chunks + c) * ld + col]);
    out[b * block_stride + col] = s;
  }
}

// ============================================================================ in-process reduction
// DeviceGroup::all_reduce_sum (inc/collectives.hpp:76-94): acc = 0 + b_0 + b_1 + ... in rank order,
// written back to every participant. Used by the LOCAL transport (several workers per device).
constexpr int kMaxLocal = 16;
template <class T>
struct PtrList {
  T* p[kMaxLocal];
};

template <class T>
__global__ void rank_order_allreduce(PtrList<T> bufs, int nranks, long count) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (long)gridDim.x * blockDim.x) {
    T acc = T(0);
    for (int r = 0; r < nranks; ++r) acc = acc + bufs.p[r][i];
    for (int r = 0; r < nranks; ++r) bufs.p[r][i] = acc;
  }
}

// zero fill (float4 granularity when aligned)
__global__ void fill_zero(float* __restrict__ p, long n) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) p[i] = 0.0f;
}

}  // namespace k
}  // namespace mg
