// SPDX-License-Identifier: Apache-2.0
//
// tcgen05 GeMMs of the training step (TF32X3 and TF32 modes): TMA-fed, warp-specialised, persistent.
//
//   NN  C[M,N] = A[M,K] W[K,N]       forward HW = H W             (rowgcn gemm NN, dense.hpp:158-169)
//   NT  C[M,N] = A[M,K] W[N,K]^T     H-grad with relu_backward fused (dense.hpp:182-193, :221-231)
//   TN  stage[g] = H[rows_g]^T G[rows_g] for the 8 canonical row blocks g (W-grad, gcn.hpp:316-331)
//
// Per 16-deep K block, warp 0 (one lane) issues TMA tensor loads of the raw fp32 tiles straight into
// the UMMA canonical smem layouts: K-major operands (A of NN/NT, B of NT) as SWIZZLE_64B boxes
// {16 k, rows}; MN-major operands (B = W of NN, both operands of TN, which are K x M row-major in HBM)
// as SWIZZLE_128B boxes {32 mn, 16 k} — no transposition anywhere. Warps 2-5 split each element
// in place, x = hi + lo with hi exact in TF32 (split_hi / split_lo below, MG_TC_SPLIT_RN), and
// mask TN rows past the chunk end. Warp 1 (one lane) issues tcgen05.mma.kind::tf32 (M = 128,
// N <= 256, K = 8) into one of two TMEM accumulators:
//   TF32X3: D += A_lo B_hi + A_hi B_lo + A_hi B_hi      TF32: D += A_hi B_hi
// Warps 6-9 drain TMEM with tcgen05.ld (warp w owns lanes 32*(w%4)) and apply the fused epilogue on
// the way to HBM. The tensor core accumulates with truncation, so the long-K TN GeMM is "promoted":
// every 256 rows the TMEM partial is drained and added in fp32 round-to-nearest into the work item's
// partial tile (L2 resident); partials of fixed 4096-row chunks (relative to the block start) are then
// summed in chunk order — deterministic and independent of the number of workers P.
// mbarriers: full[s] (TMA bytes) -> conv[s] (split done) -> empty[s] (tcgen05.commit) for the smem
// ring; tfull[b] (tcgen05.commit) / tempty[b] (epilogue) for the two TMEM accumulators.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "mg_internal.hpp"
#include "mg_tc_gemm.cuh"

namespace mg {
namespace tc {

#define TC_CUDA(x)                                                                                     \
  do {                                                                                                 \
    cudaError_t _e = (x);                                                                              \
    if (_e != cudaSuccess) {                                                                           \
      (void)cudaGetLastError();                                                                        \
      throw CudaError(std::string(#x) + ": " + cudaGetErrorString(_e));                                \
    }                                                                                                  \
  } while (0)

constexpr int BM = 128;            // tile rows = TMEM lanes
constexpr int BK = 16;             // K per pipeline stage
constexpr int kMaxStages = 8;
constexpr int kTraceStages = 256, kTraceItems = 16;  // MGGCN_TC_TRACE clock trace sizes
constexpr int kThreads = 320;      // 10 warps: 0 TMA, 1 MMA, 2-5 split, 6-9 epilogue
constexpr int kPromoteKb = 16;     // TN: drain TMEM every 16 K blocks (256 rows)
constexpr int kSmemBudget = 200 * 1024;  // smem stage ring
constexpr int kEpiSmem = 4 * 32 * 33 * 4;  // epilogue transpose, one 32 x 33 tile per epilogue warp
static int g_split_rows = 4096;    // TN chunk (rows), fixed relative to the block start ("tn_chunk")

enum { NN = 0, NT = 1, TN = 2 };

// TF32X3 split rounding: 0 = truncated, hi = x & 0xFFFFE000 and lo = x - hi (default); 1 = hi and lo rounded
// to nearest TF32. Measured on C4 (scripts/gemm_bias_probe.py, A/B on one box): round-to-nearest lowers the
// normwise GeMM error 1.3-2x (1.0e-6 vs 1.4e-6 at K = 100, 4e-6 vs 5.5e-6 for non-negative operands at
// K = 306K) but costs 1.6 ms of GeMM per epoch (11.4 vs 9.8 ms: the split warps are on the critical path).
// Both are far inside the 1e-4 tolerance; the step-level deviations from the reference are ReLU-mask flips
// at pre-activations within rounding of 0, which no split removes (tests/test_gpu_scale.py).
#ifndef MG_TC_SPLIT_RN
#define MG_TC_SPLIT_RN 0
#endif

struct Params {
  long M, N, K;          // NN/NT: C is M x N, reduction K. TN: M, N = output dims; rows given per block
  int np;                // N padded to 16 (MMA N)
  int npb;               // B rows held in smem per stage (np for K-major B, np rounded to 32 for MN-major)
  int tstride;           // TMEM columns per accumulator (npb rounded to 32)
  int nst;               // smem stages
  int m_tiles;
  int n_items;           // work items
  int terms;             // 3 = TF32X3, 1 = TF32
  float* C;
  long ldc;
  int epi;               // 0 store, 1 relu_backward mask in place, 2 relu
  // TN
  int chunk_rows;
  int nblocks;
  long blk_begin[8], blk_len[8];
  int blk_first[9];      // first work item of each block (prefix over blocks)
  float* partial;        // [n_items][BM][npb]
  float* dbg;            // debugging aid (MGGCN_TC_DEBUG): first stage tiles + first TMEM rows, else null
  long long* trace;      // MGGCN_TC_TRACE: CTA 0 clock64 per stage [kTraceStages][4] + per item [..][2]
  // v2
  int n_tiles;           // output column tiles of <= 128
  int bnr;               // B rows (tile columns) loaded per stage: min(np, 128) (TN: rounded to 32)
  int nwst;              // v3: W ring stages (nst = A ring stages)
  int epi_chunks;        // v3: 32 x 32 epilogue buffers per epilogue warp (2, or 4 with the relu_backward mask)
  k::Epi ep;             // fused bias / dropout (EPI 0, 2) and the dropout scale of the relu_backward mask (EPI 1)
  // v3 F16 (scaled two-term fp16 split on kind::f16): per-row max |A| pairs from A's producer (Epi::rmax)
  // and the per-column inverse scales of the pre-split W
  const float* rmax_in;
  const float* tinv;
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {  // non-blocking phase check
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// K-major SWIZZLE_64B: 8-row x 64-byte atoms, SBO = 512 B between 8-row groups, LBO unused (16 B).
__device__ __forceinline__ uint64_t desc_k64(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(512 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(4) << 61);
}
// MN-major 32-bit operands use the SWIZZLE_128B_BASE32B layout (UMMA layout type 1; TMA
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B): 4 k-rows x 128-byte (32 fp32 along M/N) atoms, 32-byte chunks
// XOR-swizzled by the row. LBO = 2048 B between atoms along M/N (one {32, 16} TMA box each),
// SBO = 512 B between consecutive 4-row atoms along K; one K = 8 MMA spans two of them.
__device__ __forceinline__ uint64_t desc_mn128(uint32_t saddr, uint32_t lbo = 2048) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>(lbo >> 4) << 16) |
         (static_cast<uint64_t>(512 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(1) << 61);
}
// kind::tf32 instruction descriptor: D f32 (bit 4), A/B tf32 (2 at bits 7, 10), majors (bits 15, 16),
// N >> 3 at bit 17, M >> 4 at bit 24.
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(a_mn) << 15) | (static_cast<uint32_t>(b_mn) << 16) |
         (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
// Warp-wide issue: every lane of the MMA warp executes these with warp-uniform operands and elect.sync
// picks the issuing lane inside the asm. Issuing from a lane-0 branch instead makes ptxas wrap every
// tcgen05.mma in an ELECT / R2UR.BROADCAST loop over the active lanes, which measured ~56 cycles per MMA
// (scripts/mma_probe.cu) against the 24 (N = 48) / 64 (N = 128) cycles the tensor core needs.
__device__ __forceinline__ void mma_tf32_e(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit_e(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// 3xTF32 splits (MG_TC_SPLIT_RN above): x = hi + lo, hi exact in TF32; the tensor core reads lo's top 19
// bits and the omitted lo*lo product is below 2^-22 |x|.
__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ float tf32_tr(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
__device__ __forceinline__ float split_hi(float x) { return MG_TC_SPLIT_RN ? tf32_rn(x) : tf32_tr(x); }
__device__ __forceinline__ float split_lo(float x, float hi) {
  return MG_TC_SPLIT_RN ? tf32_rn(__fsub_rn(x, hi)) : __fsub_rn(x, hi);
}
// lo part for an operand whose hi part is the raw fp32 tile (kind::tf32 truncates it: hi = x & 0xFFFFE000)
__device__ __forceinline__ float split_lo_trunc(float x) {
  const float d = __fsub_rn(x, tf32_tr(x));
  return MG_TC_SPLIT_RN ? tf32_rn(d) : d;
}
__device__ __forceinline__ float4 split4(float4 x, float4& lo) {
  float4 h;
  h.x = split_hi(x.x);
  h.y = split_hi(x.y);
  h.z = split_hi(x.z);
  h.w = split_hi(x.w);
  lo = make_float4(split_lo(x.x, h.x), split_lo(x.y, h.y), split_lo(x.z, h.z), split_lo(x.w, h.w));
  return h;
}

// The NN / NT epilogue on 4 consecutive outputs of row `row`, columns col..col+3: 1 = relu_backward mask
// (kept entries x 1/(1-p) under dropout), 2 = relu, 0 = store; bias / dropout per mg_epi.cuh only in the
// EXT instantiations (the default kernels carry no bias / dropout code: warp-specialised kernels are
// sensitive to code size, measured 2.5x slower GeMMs with the extension inlined into every kernel).
template <bool EXT>
__device__ __forceinline__ float4 gemm_epi(float4 o, float4 old, const Params& p, long row, int col) {
  if (!EXT) {
    if (p.epi == 1)
      return make_float4(old.x > 0.0f ? o.x : 0.0f, old.y > 0.0f ? o.y : 0.0f, old.z > 0.0f ? o.z : 0.0f,
                         old.w > 0.0f ? o.w : 0.0f);
    if (p.epi == 2) return make_float4(fmaxf(o.x, 0.0f), fmaxf(o.y, 0.0f), fmaxf(o.z, 0.0f), fmaxf(o.w, 0.0f));
    return o;
  }
  if (p.epi == 1) {
    if (p.ep.thr) o = make_float4(__fmul_rn(o.x, p.ep.scale), __fmul_rn(o.y, p.ep.scale), __fmul_rn(o.z, p.ep.scale),
                                  __fmul_rn(o.w, p.ep.scale));
    return make_float4(old.x > 0.0f ? o.x : 0.0f, old.y > 0.0f ? o.y : 0.0f, old.z > 0.0f ? o.z : 0.0f,
                       old.w > 0.0f ? o.w : 0.0f);
  }
  return k::epi4(o, p.epi == 2, p.ep, row, col);
}

// Ring cursor (slot, phase parity, wrapped) for rings whose depth is a runtime value: replaces sc % n and
// sc / n (an integer division per stage in every role's loop).
struct RingPos {
  int n, idx = 0;
  uint32_t phase = 0;
  bool wrapped = false;
  __device__ explicit RingPos(int n_) : n(n_) {}
  __device__ void next() {
    if (++idx == n) {
      idx = 0;
      phase ^= 1u;
      wrapped = true;
    }
  }
};
// ---------------------------------------------------------------- work decomposition
struct Item {
  long row0;    // NN/NT: first output row. TN: first K row (local)
  long k_end;   // TN: one past the last K row of this item
  int mt;       // TN: m tile
  int nkb;      // K blocks of the item
};

__device__ __forceinline__ Item item_of(const Params& p, int MODE_, int it, int bk = BK) {
  Item r{};
  if (MODE_ != TN) {
    r.row0 = static_cast<long>(it) * BM;
    r.nkb = static_cast<int>((p.K + bk - 1) / bk);
    return r;
  }
  int g = 0;
  while (g + 1 < p.nblocks && it >= p.blk_first[g + 1]) ++g;
  const int local = it - p.blk_first[g];
  const int c = local / p.m_tiles;
  r.mt = local % p.m_tiles;
  r.row0 = p.blk_begin[g] + static_cast<long>(c) * p.chunk_rows;
  const long end = p.blk_begin[g] + p.blk_len[g];
  r.k_end = (r.row0 + p.chunk_rows < end) ? r.row0 + p.chunk_rows : end;
  r.nkb = static_cast<int>((r.k_end - r.row0 + bk - 1) / bk);
  return r;
}

// ---------------------------------------------------------------- the kernel
template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) gemm_tc(const __grid_constant__ CUtensorMap map_a,
                                                       const __grid_constant__ CUtensorMap map_b, Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kMaxStages], conv[kMaxStages], empty[kMaxStages], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr bool A_MN = MODE == TN;
  constexpr bool B_MN = MODE != NT;
  const int a_bytes = BM * BK * 4;          // 8 KB
  const int b_bytes = p.npb * BK * 4;
  const int half = a_bytes + b_bytes;       // hi (TMA target) part of a stage; lo part follows
  const int stage = p.terms == 3 ? 2 * half : half;
  const uint32_t tx_bytes = static_cast<uint32_t>(half);
  const uint32_t tmem_cols = 2 * p.tstride <= 32 ? 32 : 2 * p.tstride <= 64 ? 64 : 2 * p.tstride <= 128 ? 128
                             : 2 * p.tstride <= 256 ? 256 : 512;

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_s)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t sc = 0;
      for (int it = blockIdx.x; it < p.n_items; it += gridDim.x) {
        const Item I = item_of(p, MODE, it);
        for (int kb = 0; kb < I.nkb; ++kb, ++sc) {
          const int s = sc % p.nst;
          if (sc >= static_cast<uint32_t>(p.nst)) mbar_wait(&empty[s], ((sc / p.nst) - 1) & 1);
          uint8_t* a = smem + s * stage;
          uint8_t* b = a + a_bytes;
          mbar_arrive_tx(&full[s], tx_bytes);
          if (MODE == TN) {
            const int k0 = static_cast<int>(I.row0) + kb * BK;
            for (int j = 0; j < BM / 32; ++j) tma_load_2d(a + j * 2048, &map_a, I.mt * BM + j * 32, k0, &full[s]);
            for (int j = 0; j < p.npb / 32; ++j) tma_load_2d(b + j * 2048, &map_b, j * 32, k0, &full[s]);
          } else {
            const int k0 = kb * BK;
            tma_load_2d(a, &map_a, k0, static_cast<int>(I.row0), &full[s]);
            if (B_MN) {
              for (int j = 0; j < p.npb / 32; ++j) tma_load_2d(b + j * 2048, &map_b, j * 32, k0, &full[s]);
            } else {
              tma_load_2d(b, &map_b, k0, 0, &full[s]);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = idesc_tf32(BM, p.np, A_MN ? 1 : 0, B_MN ? 1 : 0);
    uint32_t sc = 0, ac = 0;
    for (int it = blockIdx.x; it < p.n_items; it += gridDim.x) {
      const Item I = item_of(p, MODE, it);
      const int groups = MODE == TN ? (I.nkb + kPromoteKb - 1) / kPromoteKb : 1;
      for (int gi = 0; gi < groups; ++gi, ++ac) {
        const int kb0 = MODE == TN ? gi * kPromoteKb : 0;
        const int kb1 = MODE == TN ? min(I.nkb, kb0 + kPromoteKb) : I.nkb;
        const int buf = ac & 1;
        if (ac >= 2) mbar_wait(&tempty[buf], ((ac >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + static_cast<uint32_t>(buf * p.tstride);
        for (int kb = kb0; kb < kb1; ++kb, ++sc) {
          const int s = sc % p.nst;
          mbar_wait(&conv[s], (sc / p.nst) & 1);
          tc_fence_after();
          {  // whole warp, elected issue (see mma_tf32_e)
            const uint32_t ah = smem_u32(smem + s * stage), bh = ah + a_bytes;
            const uint32_t al = ah + half, bl = bh + half;
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const uint32_t ao = A_MN ? kk * 1024 : kk * 32, bo = B_MN ? kk * 1024 : kk * 32;
              const uint64_t dah = A_MN ? desc_mn128(ah + ao) : desc_k64(ah + ao);
              const uint64_t dbh = B_MN ? desc_mn128(bh + bo) : desc_k64(bh + bo);
              const uint32_t first = (kb == kb0 && kk == 0) ? 0u : 1u;
              if (p.terms == 3) {
                const uint64_t dal = A_MN ? desc_mn128(al + ao) : desc_k64(al + ao);
                const uint64_t dbl = B_MN ? desc_mn128(bl + bo) : desc_k64(bl + bo);
                mma_tf32_e(d, dal, dbh, idesc, first);
                mma_tf32_e(d, dah, dbl, idesc, 1u);
                mma_tf32_e(d, dah, dbh, idesc, 1u);
              } else {
                mma_tf32_e(d, dah, dbh, idesc, first);
              }
            }
            mma_commit_e(&empty[s]);
          }
          __syncwarp();
        }
        mma_commit_e(&tfull[buf]);
        __syncwarp();
      }
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------ split (+ TN chunk-end mask)
    const int t = threadIdx.x - 64;  // 0..127
    uint32_t sc = 0;
    for (int it = blockIdx.x; it < p.n_items; it += gridDim.x) {
      const Item I = item_of(p, MODE, it);
      for (int kb = 0; kb < I.nkb; ++kb, ++sc) {
        const int s = sc % p.nst;
        mbar_wait(&full[s], (sc / p.nst) & 1);
        uint8_t* hi = smem + s * stage;
        uint8_t* lo = hi + half;
        if (p.dbg && sc == 0 && blockIdx.x == 0)
          for (int q = t; q < half / 4; q += 128) p.dbg[q] = reinterpret_cast<float*>(hi)[q];
        const int valid_rows = MODE == TN ? static_cast<int>(min(static_cast<long>(BK), I.k_end - (I.row0 + kb * BK))) : BK;
        if (p.terms == 3 || valid_rows < BK) {
          for (int q = t; q < half / 16; q += 128) {
            float4 x = reinterpret_cast<float4*>(hi)[q];
            if (MODE == TN && valid_rows < BK && q < a_bytes / 16) {
              const int krow = ((q * 16) % 2048) >> 7;  // row of the MN-major box
              if (krow >= valid_rows) x = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            if (p.terms == 3) {
              float4 l;
              const float4 h = split4(x, l);
              reinterpret_cast<float4*>(hi)[q] = h;
              reinterpret_cast<float4*>(lo)[q] = l;
            } else {
              reinterpret_cast<float4*>(hi)[q] = x;
            }
          }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[s]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;
    const int row = q * 32 + lane;
    uint32_t ac = 0;
    for (int it = blockIdx.x; it < p.n_items; it += gridDim.x) {
      const Item I = item_of(p, MODE, it);
      const int groups = MODE == TN ? (I.nkb + kPromoteKb - 1) / kPromoteKb : 1;
      for (int gi = 0; gi < groups; ++gi, ++ac) {
        const int buf = ac & 1;
        mbar_wait(&tfull[buf], (ac >> 1) & 1);
        tc_fence_after();
        const uint32_t tbase = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(buf * p.tstride);
        // TMEM gives each lane one row; a 32 x 33 smem transpose per warp turns that into 128-byte
        // row segments so every global load/store of the epilogue is fully coalesced.
        float* stg = reinterpret_cast<float*>(smem + p.nst * stage) + q * (32 * 33);
        for (int c0 = 0; c0 < p.np; c0 += 32) {
          float v[32];
          tmem_ld32(tbase + c0, v);
          if (p.dbg && ac == 0 && blockIdx.x == 0 && c0 == 0)
            for (int i = 0; i < 32; ++i) p.dbg[16384 + row * 32 + i] = v[i];
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 32; ++i) stg[lane * 33 + i] = v[i];
          __syncwarp();
          const int c = c0 + lane;
          if (MODE == TN) {
            if (c < p.npb) {
              float* dst = p.partial + (static_cast<long>(it) * BM + q * 32) * p.npb + c;
              float prev[32];
              if (gi > 0) {  // all 32 row loads in flight before the first add
#pragma unroll
                for (int r = 0; r < 32; ++r) prev[r] = dst[static_cast<long>(r) * p.npb];
              }
#pragma unroll
              for (int r = 0; r < 32; ++r) {
                float x = stg[r * 33 + lane];
                if (gi > 0) x = __fadd_rn(prev[r], x);
                dst[static_cast<long>(r) * p.npb] = x;
              }
            }
          } else if (c < p.N) {
            const long g0 = I.row0 + q * 32;
            const int nrows = static_cast<int>(min(32L, p.M - g0));
            float* dst = p.C + g0 * p.ldc + c;
            float old[32];
            if (p.epi == 1) {  // relu_backward mask: issue every row load before the first store
#pragma unroll
              for (int r = 0; r < 32; ++r) old[r] = r < nrows ? dst[static_cast<long>(r) * p.ldc] : 0.0f;
            }
#pragma unroll
            for (int r = 0; r < 32; ++r) {
              if (r < nrows) {
                float x = stg[r * 33 + lane];
                if (p.epi == 1) x = old[r] > 0.0f ? (p.ep.thr ? __fmul_rn(x, p.ep.scale) : x) : 0.0f;
                else x = k::epi1(x, p.epi == 2, p.ep, g0 + r, static_cast<int>(c));
                dst[static_cast<long>(r) * p.ldc] = x;
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        if (p.trace && blockIdx.x == 0 && q == 0 && lane == 0 && ac < kTraceItems)
          p.trace[kTraceStages * 4 + ac * 2 + 1] = clock64();
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(tmem_cols));
}

// ================================================================ v2: A operand in TMEM ("TS" MMAs)
// Same pipeline, but the split A operand never goes back to shared memory: the four split warps own
// the 128 TMEM lanes (= tile rows) and write A_hi / A_lo of each 16-deep K block straight into a TMEM
// stage with tcgen05.st; the MMA reads A from TMEM and only B from smem. For NN / NT the B operand (W)
// is split and laid out K-major once per call (split_b), so its hi / lo tiles arrive by TMA ready to use.
// Output tiles are 128 x (<= 128) columns, so the two TMEM accumulators always double-buffer (wider N
// runs as adjacent column tiles of the same row tile, issued back to back so A comes from L2 the
// second time). TMEM: accumulators in columns [0, 256), A stages in [256, 256 + 32 * nst).
// Epilogue: each epilogue warp owns 32 rows and up to four 32 x 32 fp32 smem buffers (SWIZZLE_128B,
// the TMA layout). NN / NT: the relu_backward mask source (epi 1) is TMA-prefetched into the buffers
// before the accumulator is ready, results are written back in place and leave with TMA bulk stores.
// TN: the buffers hold the running fp32 sum of the promoted partials of the work item (no global
// read-modify-write), stored once per item.
constexpr int kAcol = 256;
constexpr int kTileN = 128;
constexpr int kEpiBuf = 4 * 4 * 4096;  // 4 warps x 4 chunks x (32 x 32 fp32)

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}
// One 16-K stage of 3xTF32 (2 K steps x 3 terms) behind one elect; BOFF = the descriptor increment of one
// K step (+1024 B = 64 for the MN-major SWIZZLE_128B_BASE32B B tiles, +32 B = 2 for K-major SWIZZLE_64B).
template <int BOFF>
__device__ __forceinline__ void mma6_tf32_ts_e(uint32_t d, uint32_t ah, uint32_t al, uint64_t bh, uint64_t bl,
                                               uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      ".reg .b32 ah1, al1;\n"
      ".reg .b64 bh1, bl1;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %6, 0;\n"
      "add.u32 ah1, %1, 8;\nadd.u32 al1, %2, 8;\n"
      "add.u64 bh1, %3, %7;\nadd.u64 bl1, %4, %7;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %5, p;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al1], bh1, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah1], bl1, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah1], bh1, %5, 1;\n"
      "}\n" ::"r"(d),
      "r"(ah), "r"(al), "l"(bh), "l"(bl), "r"(idesc), "r"(acc), "n"(BOFF));
}
// One 32-K stage of 3xTF32 (4 K steps x 3 terms) behind one elect, the K-step operand offsets computed
// inside the asm (+8 TMEM columns, +32 bytes = +2 in a K-major SWIZZLE_128B descriptor's address field).
template <int BOFF = 2>
__device__ __forceinline__ void mma12_tf32_ts_e(uint32_t d, uint32_t ah, uint32_t al, uint64_t bh, uint64_t bl,
                                                uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      ".reg .b32 ah1, ah2, ah3, al1, al2, al3;\n"
      ".reg .b64 bh1, bh2, bh3, bl1, bl2, bl3;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %6, 0;\n"
      "add.u32 ah1, %1, 8;\nadd.u32 ah2, %1, 16;\nadd.u32 ah3, %1, 24;\n"
      "add.u32 al1, %2, 8;\nadd.u32 al2, %2, 16;\nadd.u32 al3, %2, 24;\n"
      "add.u64 bh1, %3, %7;\nadd.u64 bh2, %3, %8;\nadd.u64 bh3, %3, %9;\n"
      "add.u64 bl1, %4, %7;\nadd.u64 bl2, %4, %8;\nadd.u64 bl3, %4, %9;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %5, p;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al1], bh1, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah1], bl1, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah1], bh1, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al2], bh2, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah2], bl2, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah2], bh2, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al3], bh3, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah3], bl3, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah3], bh3, %5, 1;\n"
      "}\n" ::"r"(d),
      "r"(ah), "r"(al), "l"(bh), "l"(bl), "r"(idesc), "r"(acc), "n"(BOFF), "n"(2 * BOFF), "n"(3 * BOFF));
}
// The three 3xTF32 terms of one K = 8 step, lo*hi + hi*lo + hi*hi, behind one elect (the operand
// conversions to uniform registers are shared by the three instructions).
__device__ __forceinline__ void mma3_tf32_ts_e(uint32_t tmem_d, uint32_t a_hi, uint32_t a_lo, uint64_t b_hi,
                                               uint64_t b_lo, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %6, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %5, p;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %5, 1;\n"
      "}\n" ::"r"(tmem_d),
      "r"(a_hi), "r"(a_lo), "l"(b_hi), "l"(b_lo), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_tf32_ts_e(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                              uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}
// One 32-K stage of the scaled fp16 split (2 K = 16 steps x 3 terms, kind::f16) behind one elect: A hi / lo
// from TMEM (16 fp16 pairs = 8 columns per K step), B hi / lo K-major SWIZZLE_64B (+32 B = +2 per K step).
__device__ __forceinline__ void mma6_f16_ts_e(uint32_t d, uint32_t ah, uint32_t al, uint64_t bh, uint64_t bl,
                                              uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      ".reg .b32 ah1, al1;\n"
      ".reg .b64 bh1, bl1;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %6, 0;\n"
      "add.u32 ah1, %1, 8;\nadd.u32 al1, %2, 8;\n"
      "add.u64 bh1, %3, 2;\nadd.u64 bl1, %4, 2;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %3, %5, p;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %4, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %3, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [al1], bh1, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ah1], bl1, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ah1], bh1, %5, 1;\n"
      "}\n" ::"r"(d),
      "r"(ah), "r"(al), "l"(bh), "l"(bl), "r"(idesc), "r"(acc));
}
// kind::f16 instruction descriptor: D f32 (bit 4), A / B f16 (0 at bits 7, 10), both K-major, N >> 3, M >> 4.
__host__ __device__ constexpr uint32_t idesc_f16(int m, int n) {
  return (1u << 4) | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}
// Power-of-two scale exponent for a block of values with max |x| = m: m * 2^e in [2^14, 2^15), so the fp16
// hi part keeps 11 significant bits of every element within 2^13 of the max and the lo part (2^-11 of hi)
// stays a normal fp16; clamped so the scale and its inverse are normal fp32 numbers.
__device__ __forceinline__ int f16_scale_exp(float m) {
  if (!(m > 0.0f)) return 0;
  int e;
  (void)frexpf(m, &e);  // m = f * 2^e, f in [0.5, 1): m in [2^(e-1), 2^e)
  // +-60: the epilogue multiplies by the product of a row's and a column's inverse scales, which then stays
  // a normal fp32 power of two (exact)
  return max(-60, min(60, 15 - e));
}
__device__ __forceinline__ uint32_t h2_bits(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
// x (already scaled) -> fp16 hi / lo pair for two consecutive K elements (a = even k in the low half)
__device__ __forceinline__ void split_f16x2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(a, b);
  const float2 hf = __half22float2(h);
  hi = h2_bits(h);
  lo = h2_bits(__floats2half2_rn(__fsub_rn(a, hf.x), __fsub_rn(b, hf.y)));
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int x, int y, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
// Row r's 16-byte chunk j of a 32 x 32 fp32 SWIZZLE_128B box.
__device__ __forceinline__ float4* sw128(float* buf, int r, int j) {
  return reinterpret_cast<float4*>(buf + r * 32 + ((j ^ (r & 7)) << 2));
}

// W (padded ld) -> B_hi / B_lo, K-major (np x kp): NN reads W as K x N (transpose), NT as N x K.
__global__ void split_b(const float* __restrict__ W, long ldw, int trans, int np, int kp, long nvalid, long kvalid,
                        int terms, float* __restrict__ hi, float* __restrict__ lo) {
  const long total = static_cast<long>(np) * kp;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const long n = i / kp, k = i % kp;
    float x = 0.0f;
    if (n < nvalid && k < kvalid) x = trans ? W[k * ldw + n] : W[n * ldw + k];
    const float h = terms == 3 ? split_hi(x) : x;
    hi[i] = h;
    lo[i] = terms == 3 ? split_lo(x, h) : 0.0f;
  }
}

// W -> per-column scaled fp16 hi / lo planes, K-major (np x kp, kp a multiple of 8) for the v3 F16 kernels:
// column n (an output column) is scaled by 2^e_n from its max |W[., n]| (f16_scale_exp); tinv[n] = 2^-e_n
// is applied by the epilogue. One block per column.
__global__ void split_b16(const float* __restrict__ W, long ldw, int trans, int np, int kp, long nvalid, long kvalid,
                          __half* __restrict__ hi, __half* __restrict__ lo, float* __restrict__ tinv) {
  __shared__ float red[32];
  const int n = blockIdx.x;
  float m = 0.0f;
  if (n < nvalid)
    for (long k = threadIdx.x; k < kvalid; k += blockDim.x) m = fmaxf(m, fabsf(trans ? W[k * ldw + n] : W[n * ldw + k]));
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) red[0] = m;
  }
  __syncthreads();
  const int e = f16_scale_exp(red[0]);
  const float sc = ldexpf(1.0f, e);
  if (threadIdx.x == 0) tinv[n] = ldexpf(1.0f, -e);
  for (long k = threadIdx.x; k < kp; k += blockDim.x) {
    const float x = (n < nvalid && k < kvalid) ? __fmul_rn(trans ? W[k * ldw + n] : W[n * ldw + k], sc) : 0.0f;
    const __half h = __float2half_rn(x);
    hi[static_cast<long>(n) * kp + k] = h;
    lo[static_cast<long>(n) * kp + k] = __float2half_rn(__fsub_rn(x, __half2float(h)));
  }
}

struct Item2 {
  Item k;   // rows / K range (TN: of the m-item)
  int mi;   // TN: m-item (index into the partial tiles); NN/NT: row tile
  int n0;   // first output column of the tile
  int nw;   // tile columns (multiple of 16, <= 128)
};
__device__ __forceinline__ Item2 item2_of(const Params& p, int MODE_, int it, int bk = BK) {
  Item2 r;
  r.mi = it / p.n_tiles;
  const int nt = it - r.mi * p.n_tiles;
  r.n0 = nt * kTileN;
  r.nw = min(kTileN, p.np - r.n0);
  r.k = item_of(p, MODE_, r.mi, bk);
  return r;
}

// TN: 4 extra warps (10-13) split the B tile in smem while warps 2-5 split A into TMEM.
constexpr int kThreadsTN = 448;
template <int MODE>
constexpr int threads2() { return MODE == TN ? kThreadsTN : kThreads; }
// v2 K rows per stage: TN streams 32 (one 12-MMA issue block per stage, half the per-stage barrier and
// commit overhead of 16), NN / NT keep 16 (their K-major SWIZZLE_64B B tiles).
template <int MODE>
__host__ __device__ constexpr int bk2() { return MODE == TN ? 32 : BK; }
constexpr int kPromoteRows = 256;  // TN: drain TMEM every 256 K rows

template <int MODE, bool EXT>
__global__ void __launch_bounds__(threads2<MODE>(), 1) gemm_tc2(const __grid_constant__ CUtensorMap map_a,
                                                        const __grid_constant__ CUtensorMap map_bh,
                                                        const __grid_constant__ CUtensorMap map_bl,
                                                        const __grid_constant__ CUtensorMap map_c, Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kMaxStages], conv[kMaxStages], empty[kMaxStages], tfull[2], tempty[2], oldbar[4];
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr bool B_MN = MODE == TN;  // NN/NT read the pre-split K-major B
  constexpr int BKV = bk2<MODE>();
  constexpr int kPromote = kPromoteRows / BKV;  // TN: K blocks per TMEM drain
  constexpr uint32_t kBox = 32 * BKV * 4;      // TN: bytes of one {32 n, BKV k} B box (LBO along N)
  const int a_bytes = BM * BKV * 4;    // raw A tile (no swizzle): NN/NT [128 rows][16 k], TN [32 k][128 m]
  const int b_bytes = p.bnr * BKV * 4;  // one B tile (bnr = tile columns held per stage)
  const int stage = a_bytes + 2 * b_bytes;  // A raw | B hi | B lo

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], MODE == TN && p.terms == 3 ? 8 : 4);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    for (int q = 0; q < 4; ++q) mbar_init(&oldbar[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_bh)) : "memory");
    if (MODE != TN) asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_bl)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tmem_base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t sc = 0;
      RingPos rp(p.nst);
      // single-term TF32 never reads B lo: do not load it
      const uint32_t tx = static_cast<uint32_t>(MODE == TN || p.terms != 3 ? a_bytes + b_bytes : stage);
      for (int it = blockIdx.x; it < p.n_items; it += gridDim.x) {
        const Item2 I = item2_of(p, MODE, it, BKV);
        for (int kb = 0; kb < I.k.nkb; ++kb, ++sc, rp.next()) {
          const int s = rp.idx;
          if (rp.wrapped) mbar_wait(&empty[s], rp.phase ^ 1u);
          if (p.trace && blockIdx.x == 0 && sc < kTraceStages) p.trace[sc * 4 + 0] = clock64();
          uint8_t* a = smem + s * stage;
          uint8_t* b = a + a_bytes;
          mbar_arrive_tx(&full[s], tx);
          if (MODE == TN) {
            const int k0 = static_cast<int>(I.k.row0) + kb * BKV;
            tma_load_2d(a, &map_a, I.k.mt * BM, k0, &full[s]);
            for (int j = 0; j < p.bnr / 32; ++j) tma_load_2d(b + j * kBox, &map_bh, I.n0 + j * 32, k0, &full[s]);
          } else {
            const int k0 = kb * BKV;
            tma_load_2d(a, &map_a, k0, static_cast<int>(I.k.row0), &full[s]);
            tma_load_2d(b, &map_bh, k0, I.n0, &full[s]);
            if (p.terms == 3) tma_load_2d(b + b_bytes, &map_bl, k0, I.n0, &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (A from TMEM)
    uint32_t sc = 0, ac = 0;
    RingPos rp(p.nst);
    for (int it = blockIdx.x; it < p.n_items; it += gridDim.x) {
      const Item2 I = item2_of(p, MODE, it, BKV);
      const uint32_t idesc = idesc_tf32(BM, I.nw, 0, B_MN ? 1 : 0);
      const int groups = MODE == TN ? (I.k.nkb + kPromote - 1) / kPromote : 1;
      for (int gi = 0; gi < groups; ++gi, ++ac) {
        const int kb0 = MODE == TN ? gi * kPromote : 0;
        const int kb1 = MODE == TN ? min(I.k.nkb, kb0 + kPromote) : I.k.nkb;
        const int buf = static_cast<int>(ac & 1);
        if (ac >= 2u) mbar_wait(&tempty[buf], ((ac >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + static_cast<uint32_t>(buf * kTileN);
        for (int kb = kb0; kb < kb1; ++kb, ++sc, rp.next()) {
          const int s = rp.idx;
          mbar_wait(&conv[s], rp.phase);
          tc_fence_after();
          if (p.trace && blockIdx.x == 0 && lane == 0 && sc < kTraceStages) p.trace[sc * 4 + 3] = clock64();
          {  // whole warp, elected issue (see mma_tf32_e)
            const uint32_t bh = smem_u32(smem + s * stage + a_bytes), bl = bh + b_bytes;
            const uint32_t ah = tmem + static_cast<uint32_t>(kAcol + s * 2 * BKV), al = ah + BKV;
            if (p.terms == 3) {
              const uint64_t dbh = B_MN ? desc_mn128(bh, kBox) : desc_k64(bh);
              const uint64_t dbl = B_MN ? desc_mn128(bl, kBox) : desc_k64(bl);
              if (BKV == 32) mma12_tf32_ts_e<B_MN ? 64 : 2>(d, ah, al, dbh, dbl, idesc, kb == kb0 ? 0u : 1u);
              else mma6_tf32_ts_e<B_MN ? 64 : 2>(d, ah, al, dbh, dbl, idesc, kb == kb0 ? 0u : 1u);
            } else {
#pragma unroll
              for (int kk = 0; kk < BKV / 8; ++kk) {
                const uint32_t bo = B_MN ? kk * 1024 : kk * 32;
                mma_tf32_ts_e(d, ah + kk * 8, B_MN ? desc_mn128(bh + bo, kBox) : desc_k64(bh + bo), idesc,
                              (kb == kb0 && kk == 0) ? 0u : 1u);
              }
            }
            mma_commit_e(&empty[s]);
          }
          __syncwarp();
        }
        mma_commit_e(&tfull[buf]);
        __syncwarp();
      }
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------ split A into TMEM (+ split B for TN)
    // Explicit shared-space loads of the raw tile (the aligned dynamic-smem pointer is generic to the compiler).
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int t = threadIdx.x - 64;
    uint32_t sc = 0;
    RingPos rp(p.nst);
    for (int it = blockIdx.x; it < p.n_items; it += gridDim.x) {
      const Item2 I = item2_of(p, MODE, it, BKV);
      for (int kb = 0; kb < I.k.nkb; ++kb, ++sc, rp.next()) {
        const int s = rp.idx;
        mbar_wait(&full[s], rp.phase);  // also implies the MMAs of this stage's last use are done
        if (p.trace && blockIdx.x == 0 && q == 0 && lane == 0 && sc < kTraceStages) p.trace[sc * 4 + 1] = clock64();
        const uint32_t araw = smem_u32(smem + s * stage);
        float x[BKV];
        if (MODE == TN) {
          const int valid = static_cast<int>(min(static_cast<long>(BKV), I.k.k_end - (I.k.row0 + kb * BKV)));
#pragma unroll
          for (int k = 0; k < BKV; ++k) {
            float v;
            asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(v) : "r"(araw + 4u * (k * BM + row)));
            x[k] = k < valid ? v : 0.0f;
          }
        } else {
#pragma unroll
          for (int k4 = 0; k4 < BKV / 4; ++k4)
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                         : "=f"(x[4 * k4]), "=f"(x[4 * k4 + 1]), "=f"(x[4 * k4 + 2]), "=f"(x[4 * k4 + 3])
                         : "r"(araw + 4u * (row * BKV + 4 * k4)));
        }
        uint32_t hi[BKV], lo[BKV];
#pragma unroll
        for (int k = 0; k < BKV; ++k) {
          const float h = p.terms == 3 ? split_hi(x[k]) : x[k];
          hi[k] = __float_as_uint(h);
          lo[k] = __float_as_uint(p.terms == 3 ? split_lo(x[k], h) : 0.0f);
        }
        const uint32_t ta = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(kAcol + s * 2 * BKV);
#pragma unroll
        for (int c = 0; c < BKV / 16; ++c) {
          tmem_st16(ta + 16 * c, hi + 16 * c);
          if (p.terms == 3) tmem_st16(ta + BKV + 16 * c, lo + 16 * c);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[s]);
        if (p.trace && blockIdx.x == 0 && q == 0 && lane == 0 && sc < kTraceStages) p.trace[sc * 4 + 2] = clock64();
      }
    }
  } else if (warp >= 10) {
    // ------------------------------------------------------------ TN: B (G rows) lo copy
    // kind::tf32 reads the raw fp32 tile as its hi part: the tensor core drops the low 13 mantissa bits
    // (hi = x & 0xFFFFE000), so only lo = x - hi is written (half the shared-memory stores of rewriting hi
    // in place; the kernel is shared-memory-bandwidth bound at this stage).
    if (MODE == TN && p.terms == 3) {
      const int t = threadIdx.x - 320;
      RingPos rp(p.nst);
      for (int it = blockIdx.x; it < p.n_items; it += gridDim.x) {
        const Item2 I = item2_of(p, MODE, it, BKV);
        for (int kb = 0; kb < I.k.nkb; ++kb, rp.next()) {
          const int s = rp.idx;
          mbar_wait(&full[s], rp.phase);
          const uint32_t bh = smem_u32(smem + s * stage + a_bytes);
          const uint32_t bl = bh + static_cast<uint32_t>(b_bytes);
          for (int q4 = t; q4 < b_bytes / 16; q4 += 128) {
            float4 v, l;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                         : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "r"(bh + 16u * q4));
            l = make_float4(split_lo_trunc(v.x), split_lo_trunc(v.y), split_lo_trunc(v.z), split_lo_trunc(v.w));
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(bl + 16u * q4), "f"(l.x), "f"(l.y),
                         "f"(l.z), "f"(l.w)
                         : "memory");
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&conv[s]);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;
    uint32_t ac = 0, tiles = 0;
    float* bufs = reinterpret_cast<float*>(smem + p.nst * stage) + q * (4 * 1024);  // 4 chunks of 32 x 32
    for (int it = blockIdx.x; it < p.n_items; it += gridDim.x, ++tiles) {
      const Item2 I = item2_of(p, MODE, it, BKV);
      const int nch = (I.nw + 31) / 32;
      // buffers are free once the previous tile's bulk stores have read them
      if (lane == 0) bulk_wait_read0();
      __syncwarp();
      const long grow0 = (MODE == TN ? static_cast<long>(I.mi) * BM : I.k.row0) + q * 32;
      if (MODE != TN && p.epi == 1 && lane == 0) {  // prefetch the relu_backward mask source
        mbar_arrive_tx(&oldbar[q], static_cast<uint32_t>(nch * 4096));
        for (int c = 0; c < nch; ++c)
          tma_load_2d(bufs + c * 1024, &map_c, I.n0 + c * 32, static_cast<int>(grow0), &oldbar[q]);
      }
      const int groups = MODE == TN ? (I.k.nkb + kPromote - 1) / kPromote : 1;
      for (int gi = 0; gi < groups; ++gi, ++ac) {
        const int buf = static_cast<int>(ac & 1);
        mbar_wait(&tfull[buf], (ac >> 1) & 1);
        tc_fence_after();
        if (p.trace && blockIdx.x == 0 && q == 0 && lane == 0 && ac < kTraceItems)
          p.trace[kTraceStages * 4 + ac * 2 + 0] = clock64();
        if (MODE != TN && p.epi == 1) mbar_wait(&oldbar[q], tiles & 1);
        const uint32_t tbase = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(buf * kTileN);
        for (int c = 0; c < nch; ++c) {
          float v[32];
          tmem_ld32(tbase + c * 32, v);
          float* b = bufs + c * 1024;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4 o = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            float4* dst = sw128(b, lane, j);
            if (MODE == TN) {
              if (gi > 0) {
                const float4 pv = *dst;
                o = make_float4(__fadd_rn(pv.x, o.x), __fadd_rn(pv.y, o.y), __fadd_rn(pv.z, o.z), __fadd_rn(pv.w, o.w));
              }
            } else {
              o = gemm_epi<EXT>(o, p.epi == 1 ? *dst : o, p, grow0 + lane, I.n0 + c * 32 + 4 * j);
            }
            *dst = o;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        if (p.trace && blockIdx.x == 0 && q == 0 && lane == 0 && ac < kTraceItems)
          p.trace[kTraceStages * 4 + ac * 2 + 1] = clock64();
      }
      // the finished 32-row slab leaves with bulk tensor stores (rows / columns past the end are clipped)
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        for (int c = 0; c < nch; ++c) tma_store_2d(&map_c, I.n0 + c * 32, static_cast<int>(grow0), bufs + c * 1024);
        bulk_commit();
      }
    }
    if (lane == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// ================================================================ v3 (NN / NT): wide stages, decoupled rings
// The MGGCN_TC_TRACE clock trace of v2 showed the K-block pipeline stepping at ~900 cycles against 384
// MMA cycles: the TMA engine was bounded by the number of 64-byte row segments per stage (A, W hi and W lo
// boxes of 16 fp32 per row), not by bytes. v3 moves 32 K per stage with 128-byte rows (SWIZZLE_128B boxes,
// half the segments per byte), and decouples the rings: the streamed operand A (HBM) has its own ring of
// raw 16 KB tiles, released as soon as the split warps hold them in registers; W hi / lo (L2-resident)
// have a shallow ring with their own producer warp; the 4 TMEM A slots (64 columns: hi | lo of 32 K) are
// released by the MMA's own commit. Warps: 0 A producer, 1 MMA, 2-5 split, 6-9 epilogue, 10 W producer.
constexpr int kThreads3 = 352;
constexpr int BK3 = 32;
constexpr int kMaxA3 = 12, kMaxW3 = 4, kTSlots3 = 4;

// K-major SWIZZLE_128B: 8-row x 128-byte atoms, SBO = 1024 B between 8-row groups, LBO unused (16 B).
__device__ __forceinline__ uint64_t desc_k128(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(2) << 61);
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar,
                                               uint32_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, "
      "%3}], [%4], %5;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "h"(static_cast<uint16_t>(mask))
      : "memory");
}
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint32_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(mask))
      : "memory");
}
__device__ __forceinline__ void mma_commit_mc_e(uint64_t* bar, uint32_t mask) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "h"(static_cast<uint16_t>(mask))
      : "memory");
}

constexpr int kRS3 = 4;  // F16: per-row scale buffers (split warps -> epilogue), one per item in flight

// F16 = scaled two-term fp16 split on kind::f16 (K = 16 per MMA: half the MMAs of 3xTF32): the split warps
// scale every A row by a power of two from its max |x| over the whole K range (read from global memory,
// the next item's row during the current item's stages), W columns are pre-scaled by split_b16, and the
// epilogue multiplies each output by both inverse scales (exact).
// arrive on the mbarrier at the same shared-memory offset in CTA `peer` of the cluster (release, cluster scope)
__device__ __forceinline__ void mbar_arrive_peer(uint64_t* bar, uint32_t peer) {
  asm volatile(
      "{\n"
      ".reg .b32 ra;\n"
      "mapa.shared::cluster.u32 ra, %0, %1;\n"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(peer)
      : "memory");
}

template <int MODE, int CL, bool EXT, bool F16>
__global__ void __launch_bounds__(kThreads3, 1) gemm_tc3(const __grid_constant__ CUtensorMap map_a,
                                                         const __grid_constant__ CUtensorMap map_bh,
                                                         const __grid_constant__ CUtensorMap map_bl,
                                                         const __grid_constant__ CUtensorMap map_c, Params p) {
  static_assert(MODE != TN, "v3 covers NN / NT");
  static_assert(CL == 1 || CL == 2, "cluster of 1 or 2");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t fullA[kMaxA3], emptyA[kMaxA3], fullW[kMaxW3], emptyW[kMaxW3], conv[kTSlots3], tslot[kTSlots3];
  __shared__ uint64_t tfull[2], tempty[2], oldbar[4];
  __shared__ uint64_t rsready[F16 ? kRS3 : 1], rsfree[F16 ? kRS3 : 1];
  __shared__ float rsinv[F16 ? kRS3 : 1][F16 ? BM : 1];
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nA = p.nst, nW = p.nwst;
  constexpr int a_bytes = BM * BK3 * 4;  // raw A tile [128 rows][32 k], SWIZZLE_128B
  // one W tile (hi or lo), K-major [bnr][32 k]: fp32 SWIZZLE_128B, or fp16 SWIZZLE_64B under F16
  const int b_bytes = p.bnr * BK3 * (F16 ? 2 : 4);
  uint8_t* aring = smem;                 // nA x a_bytes
  uint8_t* wring = smem + nA * a_bytes;  // nW x (hi | lo)
  float* epib = reinterpret_cast<float*>(wring + nW * 2 * b_bytes);

  if (threadIdx.x == 0) {
    for (int s = 0; s < nA; ++s) {
      mbar_init(&fullA[s], 1);
      mbar_init(&emptyA[s], 4 * CL);  // CL = 2: both CTAs' split warps (A is multicast into both)
    }
    for (int s = 0; s < nW; ++s) {
      mbar_init(&fullW[s], 1);
      mbar_init(&emptyW[s], 1);
    }
    for (int s = 0; s < kTSlots3; ++s) {
      mbar_init(&conv[s], 4);
      mbar_init(&tslot[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    for (int q = 0; q < 4; ++q) mbar_init(&oldbar[q], 1);
    if (F16)
      for (int b = 0; b < kRS3; ++b) {
        mbar_init(&rsready[b], 128);  // every split thread releases its own row's scale
        mbar_init(&rsfree[b], 128);   // every epilogue thread has read its row's scale
      }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_bh)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_bl)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tmem_base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync();  // peers' barriers are initialised before any multicast reaches them
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  const int nkb = static_cast<int>((p.K + BK3 - 1) / BK3);
  // CL = 2 (N > 128): the two CTAs of a cluster take the two 128-column tiles of the same row tile, so they
  // stream the same A tiles in the same order: each loads half of every A stage and multicasts it to both
  const int rank = static_cast<int>(blockIdx.x % CL), pair0 = static_cast<int>(blockIdx.x / CL);
  const int npairs = static_cast<int>(gridDim.x / CL);
  const int npi = CL == 1 ? p.m_tiles * p.n_tiles : p.m_tiles;
  auto item_of3 = [&](int pi) {
    Item2 r;
    const int nt = CL == 1 ? pi % p.n_tiles : rank;
    r.mi = CL == 1 ? pi / p.n_tiles : pi;
    r.n0 = nt * kTileN;
    r.nw = min(kTileN, p.np - r.n0);
    r.k.row0 = static_cast<long>(r.mi) * BM;
    r.k.nkb = nkb;
    return r;
  };

  if (warp == 0) {
    // ------------------------------------------------------------ A producer (HBM stream, deep ring)
    if (lane == 0) {
      uint32_t sc = 0;
      RingPos r(nA);
      for (int pi = pair0; pi < npi; pi += npairs) {
        const Item2 I = item_of3(pi);
        for (int kb = 0; kb < nkb; ++kb, ++sc, r.next()) {
          const int s = r.idx;
          if (r.wrapped) mbar_wait(&emptyA[s], r.phase ^ 1u);
          if (p.trace && blockIdx.x == 0 && sc < kTraceStages) p.trace[sc * 4 + 0] = clock64();
          mbar_arrive_tx(&fullA[s], static_cast<uint32_t>(a_bytes));
          if (CL == 1)
            tma_load_2d(aring + s * a_bytes, &map_a, kb * BK3, static_cast<int>(I.k.row0), &fullA[s]);
          else  // this CTA's half of the rows, into both CTAs' slot s
            tma_load_2d_mc(aring + s * a_bytes + rank * (a_bytes / 2), &map_a, kb * BK3,
                           static_cast<int>(I.k.row0) + rank * (BM / 2), &fullA[s], 3u);
        }
      }
    }
  } else if (warp == 10) {
    // ------------------------------------------------------------ W producer (L2-resident, shallow ring)
    if (lane == 0) {
      RingPos r(nW);
      const uint32_t tx = static_cast<uint32_t>(p.terms == 3 ? 2 * b_bytes : b_bytes);
      for (int pi = pair0; pi < npi; pi += npairs) {
        const Item2 I = item_of3(pi);
        for (int kb = 0; kb < nkb; ++kb, r.next()) {
          const int s = r.idx;
          if (r.wrapped) mbar_wait(&emptyW[s], r.phase ^ 1u);
          uint8_t* b = wring + s * 2 * b_bytes;
          mbar_arrive_tx(&fullW[s], tx);
          tma_load_2d(b, &map_bh, kb * BK3, I.n0, &fullW[s]);  // this CTA's own column tile
          if (p.terms == 3) tma_load_2d(b + b_bytes, &map_bl, kb * BK3, I.n0, &fullW[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (A from TMEM slots)
    uint32_t sc = 0, ac = 0;
    RingPos rw(nW);
    for (int pi = pair0; pi < npi; pi += npairs, ++ac) {
      const Item2 I = item_of3(pi);
      const uint32_t idesc = F16 ? idesc_f16(BM, I.nw) : idesc_tf32(BM, I.nw, 0, 0);
      const int buf = static_cast<int>(ac & 1);
      if (ac >= 2u) mbar_wait(&tempty[buf], ((ac >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t d = tmem + static_cast<uint32_t>(buf * kTileN);
      for (int kb = 0; kb < nkb; ++kb, ++sc, rw.next()) {
        const int j = sc % kTSlots3, w = rw.idx;
        mbar_wait(&conv[j], (sc / kTSlots3) & 1);
        mbar_wait(&fullW[w], rw.phase);
        tc_fence_after();
        if (p.trace && blockIdx.x == 0 && lane == 0 && sc < kTraceStages) p.trace[sc * 4 + 3] = clock64();
        {  // whole warp, elected issue (see mma_tf32_e)
          const uint32_t bh = smem_u32(wring + w * 2 * b_bytes), bl = bh + b_bytes;
          const uint32_t ah = tmem + static_cast<uint32_t>(kAcol + j * 64), al = ah + 32;
          static_assert(BK3 == 32, "mma12_tf32_ts_e issues one 32-K stage");
          if (F16) {
            mma6_f16_ts_e(d, ah, ah + 16, desc_k64(bh), desc_k64(bl), idesc, kb == 0 ? 0u : 1u);
          } else if (p.terms == 3) {
            mma12_tf32_ts_e(d, ah, al, desc_k128(bh), desc_k128(bl), idesc, kb == 0 ? 0u : 1u);
          } else {
#pragma unroll
            for (int kk = 0; kk < BK3 / 8; ++kk)
              mma_tf32_ts_e(d, ah + kk * 8, desc_k128(bh + kk * 32), idesc, (kb == 0 && kk == 0) ? 0u : 1u);
          }
          mma_commit_e(&tslot[j]);  // TMEM A slot j reusable
          mma_commit_e(&emptyW[w]);  // W slot w reusable
        }
        __syncwarp();
      }
      mma_commit_e(&tfull[buf]);
      __syncwarp();
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------ split: raw A (smem) -> hi / lo (TMEM slot)
    const int q = warp & 3;
    const int row = q * 32 + lane;
    uint32_t sc = 0, ic = 0;
    RingPos ra(nA);
    // F16: max |A| of this thread's row, written by A's producer (SpMM / GeMM epilogue, Epi::rmax: two
    // slots per row); the next item's pair is loaded one item ahead
    auto row_max = [&](int pi) -> float2 {
      const long grow = item_of3(pi).k.row0 + row;
      return grow < p.M ? __ldg(reinterpret_cast<const float2*>(p.rmax_in) + grow) : make_float2(0.0f, 0.0f);
    };
    float2 rm_next = make_float2(0.0f, 0.0f);
    if (F16 && pair0 < npi) rm_next = row_max(pair0);
    for (int pi = pair0; pi < npi; pi += npairs, ++ic) {
      float rscale = 1.0f;
      if (F16) {
        const int e = f16_scale_exp(fmaxf(rm_next.x, rm_next.y));
        if (pi + npairs < npi) rm_next = row_max(pi + npairs);
        rscale = ldexpf(1.0f, e);
        const int b = static_cast<int>(ic % kRS3);
        if (ic >= static_cast<uint32_t>(kRS3)) mbar_wait(&rsfree[b], ((ic / kRS3) - 1) & 1);
        rsinv[b][row] = ldexpf(1.0f, -e);
        mbar_arrive(&rsready[b]);  // per thread: each arrival releases exactly the write it orders
      }
      for (int kb = 0; kb < nkb; ++kb, ++sc, ra.next()) {
        const int s = ra.idx, j = sc % kTSlots3;
        mbar_wait(&fullA[s], ra.phase);
        if (p.trace && blockIdx.x == 0 && q == 0 && lane == 0 && sc < kTraceStages) p.trace[sc * 4 + 1] = clock64();
        // row r's 16-byte chunk c sits at r * 128 + ((c ^ (r & 7)) * 16) (SWIZZLE_128B)
        const uint32_t rbase = smem_u32(aring + s * a_bytes) + static_cast<uint32_t>(row * 128);
        float x[BK3];
#pragma unroll
        for (int c = 0; c < BK3 / 4; ++c)
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                       : "=f"(x[4 * c]), "=f"(x[4 * c + 1]), "=f"(x[4 * c + 2]), "=f"(x[4 * c + 3])
                       : "r"(rbase + static_cast<uint32_t>(((c ^ (row & 7)) << 4))));
        __syncwarp();
        if (lane == 0) {  // the raw tile is in registers: the producer(s) may refill (CL = 2: both write it)
          mbar_arrive(&emptyA[s]);
          if (CL == 2) mbar_arrive_peer(&emptyA[s], static_cast<uint32_t>(rank ^ 1));
        }
        uint32_t hi[BK3], lo[BK3];
        if (F16) {  // 16 fp16 pairs of hi, then 16 of lo: TMEM columns [0, 16) and [16, 32) of the slot
#pragma unroll
          for (int k = 0; k < BK3 / 2; ++k)
            split_f16x2(__fmul_rn(x[2 * k], rscale), __fmul_rn(x[2 * k + 1], rscale), hi[k], lo[k]);
        } else {
#pragma unroll
          for (int k = 0; k < BK3; ++k) {
            const float h = p.terms == 3 ? split_hi(x[k]) : x[k];
            hi[k] = __float_as_uint(h);
            lo[k] = __float_as_uint(p.terms == 3 ? split_lo(x[k], h) : 0.0f);
          }
        }
        if (sc >= static_cast<uint32_t>(kTSlots3)) mbar_wait(&tslot[j], ((sc / kTSlots3) - 1) & 1);
        tc_fence_after();
        const uint32_t ta = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(kAcol + j * 64);
        if (F16) {
          tmem_st16(ta, hi);
          tmem_st16(ta + 16, lo);
        } else {
          tmem_st16(ta, hi);
          tmem_st16(ta + 16, hi + 16);
          if (p.terms == 3) {
            tmem_st16(ta + 32, lo);
            tmem_st16(ta + 48, lo + 16);
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[j]);
        if (p.trace && blockIdx.x == 0 && q == 0 && lane == 0 && sc < kTraceStages) p.trace[sc * 4 + 2] = clock64();
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (NN / NT)
    // p.epi_chunks 32 x 32 buffers per warp. NN: 2, a 128-column tile leaves in two halves, each with its
    // own bulk stores, and the shared memory saved goes to a deeper W ring. NT with the relu_backward mask:
    // 4, the whole tile's mask prefetched at once (a second HBM round trip per tile measured slower).
    const int q = warp & 3;
    const int ech = p.epi_chunks;
    uint32_t ac = 0, mph = 0;
    float rinv = 1.0f, omax = 0.0f;
    float* bufs = epib + q * (ech * 1024);
    for (int pi = pair0; pi < npi; pi += npairs, ++ac) {
      const Item2 I = item_of3(pi);
      const int nch = (I.nw + 31) / 32;
      const long grow0 = I.k.row0 + q * 32;
      const int buf = static_cast<int>(ac & 1);
      const uint32_t tbase = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(buf * kTileN);
      for (int c0 = 0; c0 < nch; c0 += ech) {
        const int cn = min(ech, nch - c0);
        if (lane == 0) bulk_wait_read0();  // the buffers' previous bulk stores have read them
        __syncwarp();
        if (p.epi == 1 && lane == 0) {  // prefetch the relu_backward mask source
          mbar_arrive_tx(&oldbar[q], static_cast<uint32_t>(cn * 4096));
          for (int c = 0; c < cn; ++c)
            tma_load_2d(bufs + c * 1024, &map_c, I.n0 + (c0 + c) * 32, static_cast<int>(grow0), &oldbar[q]);
        }
        if (c0 == 0) {
          mbar_wait(&tfull[buf], (ac >> 1) & 1);
          tc_fence_after();
          if (p.trace && blockIdx.x == 0 && q == 0 && lane == 0 && ac < kTraceItems)
            p.trace[kTraceStages * 4 + ac * 2 + 0] = clock64();
          if (F16) {
            const int rb = static_cast<int>(ac % kRS3);
            mbar_wait(&rsready[rb], (ac / kRS3) & 1);
            rinv = rsinv[rb][q * 32 + lane];
            mbar_arrive(&rsfree[rb]);
          }
        }
        if (p.epi == 1) mbar_wait(&oldbar[q], (mph++) & 1);
        for (int c = 0; c < cn; ++c) {
          float v[32];
          tmem_ld32(tbase + (c0 + c) * 32, v);
          float* b = bufs + c * 1024;
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            float4 o = make_float4(v[4 * jj], v[4 * jj + 1], v[4 * jj + 2], v[4 * jj + 3]);
            const int col = I.n0 + (c0 + c) * 32 + 4 * jj;  // columns >= nw are stale TMEM: never stored
            if (F16) {  // row x column inverse scale: a power of two within 2^+-120, so one exact multiply
              const float4 t = col < p.np ? __ldg(reinterpret_cast<const float4*>(p.tinv + col))
                                          : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
              o = make_float4(__fmul_rn(o.x, __fmul_rn(rinv, t.x)), __fmul_rn(o.y, __fmul_rn(rinv, t.y)),
                              __fmul_rn(o.z, __fmul_rn(rinv, t.z)), __fmul_rn(o.w, __fmul_rn(rinv, t.w)));
            }
            float4* dst = sw128(b, lane, jj);
            o = gemm_epi<EXT>(o, p.epi == 1 ? *dst : o, p, grow0 + lane, col);
            *dst = o;
            if (p.ep.rmax) {
              if (col + 3 < p.N) omax = k::absmax4(omax, o);
              else if (col < p.N)
                omax = k::absmax4(omax, make_float4(o.x, col + 1 < p.N ? o.y : 0.0f, col + 2 < p.N ? o.z : 0.0f, 0.0f));
            }
          }
        }
        if (c0 + ech >= nch) {  // the whole accumulator has been read: the MMA may reuse it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[buf]);
          if (p.ep.rmax && grow0 + lane < p.M) {  // this tile's row max for the next GeMM's F16 split
            float* r = p.ep.rmax + 2 * (grow0 + lane);
            if (p.n_tiles == 1) *reinterpret_cast<float2*>(r) = make_float2(omax, 0.0f);
            else r[I.n0 / kTileN] = omax;
          }
          omax = 0.0f;
          if (p.trace && blockIdx.x == 0 && q == 0 && lane == 0 && ac < kTraceItems)
            p.trace[kTraceStages * 4 + ac * 2 + 1] = clock64();
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          for (int c = 0; c < cn; ++c)
            tma_store_2d(&map_c, I.n0 + (c0 + c) * 32, static_cast<int>(grow0), bufs + c * 1024);
          bulk_commit();
        }
      }
    }
    if (lane == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync();  // no CTA leaves while a peer may still multicast into it or arrive on it
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// Fixed-order sum of the TN partials of every block: stage[g][m][n] = 0 + p_0 + p_1 + ... (chunk order).
__global__ void reduce_partials(Params p, float* __restrict__ stage, long block_stride) {
  const long per = p.M * p.N;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < per * p.nblocks;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i / per);
    const long e = i % per;
    const long m = e / p.N, n = e % p.N;
    const long t = m / BM, r = m % BM;
    float s = 0.0f;
    for (int it = p.blk_first[g] + static_cast<int>(t); it < p.blk_first[g + 1]; it += p.m_tiles)
      s = __fadd_rn(s, p.partial[(static_cast<long>(it) * BM + r) * p.npb + n]);
    stage[g * block_stride + m * p.ldc + n] = s;
  }
}

// ---------------------------------------------------------------- host side
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    TC_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !f) throw CudaError("cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// 2-D fp32 map over a row-major matrix [outer][inner] with row pitch ld floats.
CUtensorMap make_map(const void* base, long inner, long outer, long ld, int box_inner, int box_outer,
                     CUtensorMapSwizzle sw, bool f16 = false) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(std::max<long>(inner, 1)),
                              static_cast<cuuint64_t>(std::max<long>(outer, 1))};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * (f16 ? 2 : 4)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_outer)};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = encode_fn()(&m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                                 const_cast<void*>(base), dims, strides, box,
                                 es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
  return m;
}

int cur_dev() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

int num_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

void finish_params(Params& p, long N, bool b_mn, int terms) {
  p.np = static_cast<int>((N + 15) / 16 * 16);
  p.npb = b_mn ? (p.np + 31) / 32 * 32 : p.np;
  p.tstride = (p.npb + 31) / 32 * 32;
  p.terms = terms;
  const int half = BM * BK * 4 + p.npb * BK * 4;
  const int stage = terms == 3 ? 2 * half : half;
  p.nst = std::max(2, std::min(kMaxStages, kSmemBudget / stage));
}

inline int smem_bytes(const Params& p) {
  const int half = BM * BK * 4 + p.npb * BK * 4;
  return p.nst * (p.terms == 3 ? 2 * half : half) + kEpiSmem + 1024;
}

template <int MODE>
void launch(const CUtensorMap& a, const CUtensorMap& b, const Params& p, cudaStream_t s) {
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr, cur_dev()))
    TC_CUDA(cudaFuncSetAttribute(gemm_tc<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSmemBudget + kEpiSmem + 1024));
  const int grid = std::max(1, std::min(p.n_items, num_sms()));
  gemm_tc<MODE><<<grid, kThreads, smem_bytes(p), s>>>(a, b, p);
  TC_CUDA(cudaGetLastError());
}

void check_ptr(const void* p, long ld, const char* what) {
  if ((reinterpret_cast<uintptr_t>(p) & 15) || ld % 4)
    throw ValueError(std::string("tc gemm: ") + what + " must be 16-byte aligned with ld % 4 == 0");
}

// ---- v2 (A in TMEM) host side
int g_gemm_version = 3;

constexpr int kSmemBudget2 = 160 * 1024;  // v2 stage ring (+ kEpiBuf epilogue buffers)

void finish_params2(Params& p, long N, bool tn, int terms) {
  p.np = static_cast<int>((N + 15) / 16 * 16);
  p.npb = tn ? (p.np + 31) / 32 * 32 : p.np;  // TN partial row stride
  p.tstride = 0;
  p.terms = terms;
  p.n_tiles = (p.np + kTileN - 1) / kTileN;
  p.bnr = std::min(p.np, kTileN);
  if (tn) p.bnr = (p.bnr + 31) / 32 * 32;
  const int bk = tn ? bk2<TN>() : bk2<NN>();
  const int stage = BM * bk * 4 + 2 * p.bnr * bk * 4;
  // TMEM: the A slots (2 * bk columns each, hi | lo) live above the two 128-column accumulators
  const int tmem_slots = (512 - kAcol) / (2 * bk);
  p.nst = std::max(2, std::min({kMaxStages, tmem_slots, kSmemBudget2 / stage}));
}

inline int smem_bytes2(const Params& p, int bk) { return p.nst * (BM * bk * 4 + 2 * p.bnr * bk * 4) + kEpiBuf + 1024; }

// v3 (NN / NT): A ring as deep as the shared memory left after the W ring and the epilogue buffers.
constexpr int kSmemMax3 = 232448 - 2048;  // sm_100 per-block maximum, minus static barriers and alignment
int g_epi_chunks3 = 2;  // v3 NN / NT epilogue buffers per warp without the relu_backward mask ("gemm3_epi", 1 or 2)
int g_w3_bytes = 96 * 1024;  // v3 W ring budget ("gemm3_wring", bytes): 3 stages of a 128-column tile
void finish_params3(Params& p, bool f16) {
  const int wst = 2 * p.bnr * BK3 * (f16 ? 2 : 4), ast = BM * BK3 * 4;
  p.epi_chunks = p.epi == 1 ? 4 : g_epi_chunks3;
  const int wbytes = p.epi == 1 ? std::min(g_w3_bytes, 64 * 1024) : g_w3_bytes;
  p.nwst = std::max(2, std::min(kMaxW3, wbytes / wst));
  const int avail = kSmemMax3 - (f16 ? 4096 : 0);  // F16: the per-row scale buffers are static shared memory
  p.nst = std::max(2, std::min(kMaxA3, (avail - 1024 - 4 * p.epi_chunks * 4096 - p.nwst * wst) / ast));
}
inline int smem_bytes3(const Params& p, bool f16) {
  return p.nst * BM * BK3 * 4 + p.nwst * 2 * p.bnr * BK3 * (f16 ? 2 : 4) + 4 * p.epi_chunks * 4096 + 1024;
}
int g_gemm3_cluster = 1;  // v3 NN / NT: 2 = 2-CTA clusters multicasting A to both column tiles ("gemm3_cluster")
// v3 NN / NT in TF32X3 mode: scaled fp16 two-term split on kind::f16 ("gemm_f16"). Off by default: in the
// step it measured neutral to +0.1 ms per C4 epoch against 3xTF32 on three boxes (the A stream, not the
// MMA issue, paces these kernels)
int g_gemm_f16 = 0;
// ... only above this K ("gemm_f16_min_k"): with <= 4 32-K stages per 128-row tile the per-tile epilogue,
// not the MMA issue, paces the kernel and the split's extra epilogue work made it slower (ncu, C4:
// NN K = 100 1.09 -> 1.21 ms, NT K = 47 1.09 -> 1.19 ms; K = 256: 1.52 -> 1.40 and 1.71 -> 1.46 ms)
int g_f16_min_k = 128;
template <int MODE, int CL, bool EXT, bool F16 = false>
void launch3x(const CUtensorMap& a, const CUtensorMap& bh, const CUtensorMap& bl, const CUtensorMap& c, const Params& p,
              cudaStream_t s) {
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr, cur_dev()))
    TC_CUDA(cudaFuncSetAttribute(gemm_tc3<MODE, CL, EXT, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSmemMax3 - (F16 ? 4096 : 0)));
  const int npi = CL == 1 ? p.m_tiles * p.n_tiles : p.m_tiles;  // CL = 2: one row tile per cluster item
  const int grid = CL * std::max(1, std::min(npi, num_sms() / CL));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads3);
  cfg.dynamicSmemBytes = static_cast<size_t>(smem_bytes3(p, F16));
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  TC_CUDA(cudaLaunchKernelEx(&cfg, gemm_tc3<MODE, CL, EXT, F16>, a, bh, bl, c, p));
}
// bias / dropout epilogue (Params::ep) only in the EXT instantiation
inline bool epi_ext(const Params& p) { return p.ep.bias != nullptr || p.ep.thr != 0; }
template <int MODE, int CL>
void launch3(const CUtensorMap& a, const CUtensorMap& bh, const CUtensorMap& bl, const CUtensorMap& c, const Params& p,
             cudaStream_t s) {
  if (epi_ext(p)) launch3x<MODE, CL, true>(a, bh, bl, c, p, s);
  else launch3x<MODE, CL, false>(a, bh, bl, c, p, s);
}
template <int MODE>
void launch3f16(const CUtensorMap& a, const CUtensorMap& bh, const CUtensorMap& bl, const CUtensorMap& c,
                const Params& p, cudaStream_t s) {
  if (epi_ext(p)) launch3x<MODE, 1, true, true>(a, bh, bl, c, p, s);
  else launch3x<MODE, 1, false, true>(a, bh, bl, c, p, s);
}

template <int MODE, bool EXT>
void launch2x(const CUtensorMap& a, const CUtensorMap& bh, const CUtensorMap& bl, const CUtensorMap& c, const Params& p,
              cudaStream_t s) {
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr, cur_dev()))
    TC_CUDA(cudaFuncSetAttribute(gemm_tc2<MODE, EXT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSmemBudget2 + kEpiBuf + 1024));
  const int grid = std::max(1, std::min(p.n_items, num_sms()));
  gemm_tc2<MODE, EXT><<<grid, threads2<MODE>(), smem_bytes2(p, bk2<MODE>()), s>>>(a, bh, bl, c, p);
  TC_CUDA(cudaGetLastError());
}
template <int MODE>
void launch2(const CUtensorMap& a, const CUtensorMap& bh, const CUtensorMap& bl, const CUtensorMap& c, const Params& p,
             cudaStream_t s) {
  if (MODE != TN && epi_ext(p)) launch2x<MODE, true>(a, bh, bl, c, p, s);
  else launch2x<MODE, false>(a, bh, bl, c, p, s);
}

}  // namespace

size_t nn_workspace_bytes(int64_t N, int64_t K) {
  const size_t np = static_cast<size_t>((N + 15) / 16 * 16);
  const size_t f32 = 2 * sizeof(float) * np * static_cast<size_t>((K + 3) / 4 * 4);
  const size_t f16 = 2 * sizeof(__half) * np * static_cast<size_t>((K + 7) / 8 * 8) + sizeof(float) * np + 256;
  return std::max(f32, f16);
}

void set_gemm_f16(int on) { g_gemm_f16 = on != 0 ? 1 : 0; }
bool f16_enabled() { return g_gemm_f16 != 0 && g_gemm_version == 3; }
void set_gemm_f16_min_k(int k) {
  if (k < 0) throw ValueError("tuning: gemm_f16_min_k must be >= 0");
  g_f16_min_k = k;
}

void set_gemm3_cluster(int c) {
  if (c != 1 && c != 2) throw ValueError("tuning: gemm3_cluster must be 1 or 2");
  g_gemm3_cluster = c;
}

void set_epi_chunks3(int c) {
  if (c != 1 && c != 2) throw ValueError("tuning: gemm3_epi must be 1 or 2");
  g_epi_chunks3 = c;
}

void set_w3_bytes(int bytes) {
  if (bytes < 16 * 1024 || bytes > 160 * 1024) throw ValueError("tuning: gemm3_wring must be 16..160 KiB");
  g_w3_bytes = bytes;
}

void set_gemm_version(int v) {
  if (v < 1 || v > 3) throw ValueError("tuning: gemm_kernel must be 1 (SS), 2 (A in TMEM) or 3 (v2 + decoupled rings)");
  g_gemm_version = v;
}

bool available() { return true; }

void set_tn_chunk(int rows) {
  if (rows < BK * kPromoteKb || rows % (BK * kPromoteKb))
    throw ValueError("tuning: tn_chunk must be a positive multiple of 256");
  g_split_rows = rows;
}

size_t tn_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  const long npb = ((N + 15) / 16 * 16 + 31) / 32 * 32;
  const long m_tiles = (M + BM - 1) / BM;
  const long chunks = (K + g_split_rows - 1) / g_split_rows + 8;  // + one partial chunk per block boundary
  return sizeof(float) * static_cast<size_t>(chunks * m_tiles * BM * npb);
}

// MGGCN_TC_TRACE: CTA 0's clock64 per pipeline stage (issue, data in smem, A in TMEM, MMA issue) and per
// accumulator (ready, drained), printed after the launch. Debug aid; it synchronises the device.
long long* trace_buffer() {
  static long long* t = [] {
    long long* d = nullptr;
    if (std::getenv("MGGCN_TC_TRACE"))
      TC_CUDA(cudaMallocManaged(&d, sizeof(long long) * (kTraceStages * 4 + kTraceItems * 2)));
    return d;
  }();
  if (t) std::fill(t, t + kTraceStages * 4 + kTraceItems * 2, 0LL);
  return t;
}
void print_trace(const Params& p, const char* what) {
  if (!p.trace) return;
  TC_CUDA(cudaDeviceSynchronize());
  const long long* t = p.trace;
  const long long t0 = t[0];
  std::fprintf(stderr, "[tc trace] %s M=%ld N=%ld K=%ld nst=%d items=%d (per stage: issue, full, conv, mma)\n", what,
               p.M, p.N, p.K, p.nst, p.n_items);
  for (int i = 0; i < 48; ++i)
    std::fprintf(stderr, "  s%-3d %8lld %8lld %8lld %8lld\n", i, t[i * 4] - t0, t[i * 4 + 1] - t0, t[i * 4 + 2] - t0,
                 t[i * 4 + 3] - t0);
  for (int i = 0; i < kTraceItems; ++i)
    std::fprintf(stderr, "  acc%-2d ready %8lld drained %8lld\n", i, t[kTraceStages * 4 + 2 * i] - t0,
                 t[kTraceStages * 4 + 2 * i + 1] - t0);
}

int gemm(int mode, bool ta, bool tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B,
         int64_t ldb, float* C, int64_t ldc, int epi, float* ws, size_t ws_bytes, cudaStream_t s, const k::Epi& ep,
         const float* rmax_in) {
  if (ta) {
    const int64_t begin[1] = {0}, len[1] = {K};
    return gemm_tn_blocks(mode, 1, begin, len, M, N, A, lda, B, ldb, C, ldc, 0, ws, ws_bytes, s);
  }
  if (mode != MG_GEMM_TF32X3 && mode != MG_GEMM_TF32) throw ValueError("tc gemm: bad mode");
  if (N > 256) throw ValueError("tc gemm: N > 256 not supported (" + std::to_string(N) + ")");
  if (M <= 0 || N <= 0) return 0;
  if (K <= 0) throw ValueError("tc gemm: K must be >= 1");
  check_ptr(A, lda, "A");
  check_ptr(B, ldb, "B");
  Params p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.C = C;
  p.ldc = ldc;
  p.epi = epi;
  p.ep = ep;
  if (g_gemm_version >= 2) {
    finish_params2(p, N, false, mode == MG_GEMM_TF32X3 ? 3 : 1);
    check_ptr(C, ldc, "C");
    p.m_tiles = static_cast<int>((M + BM - 1) / BM);
    p.n_items = p.m_tiles * p.n_tiles;
    const int kp = static_cast<int>((K + 3) / 4 * 4);
    if (!ws || ws_bytes < nn_workspace_bytes(N, K)) throw ValueError("tc gemm: B split workspace too small");
    if (g_gemm_version == 3 && g_gemm_f16 && p.terms == 3 && g_gemm3_cluster == 1 && rmax_in && K > g_f16_min_k) {
      // scaled fp16 two-term split (kind::f16): W -> per-column scaled fp16 hi / lo planes + inverse scales
      const int kp16 = static_cast<int>((K + 7) / 8 * 8);
      __half* h16 = reinterpret_cast<__half*>(ws);
      __half* l16 = h16 + static_cast<size_t>(p.np) * kp16;
      float* tinv = reinterpret_cast<float*>(
          (reinterpret_cast<uintptr_t>(l16 + static_cast<size_t>(p.np) * kp16) + 255) & ~uintptr_t(255));
      split_b16<<<p.np, 128, 0, s>>>(B, ldb, tb ? 0 : 1, p.np, kp16, N, K, h16, l16, tinv);
      TC_CUDA(cudaGetLastError());
      p.rmax_in = rmax_in;
      p.tinv = tinv;
      p.trace = trace_buffer();
      finish_params3(p, true);
      const CUtensorMap mc = make_map(C, N, M, ldc, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B);
      const CUtensorMap ma3 = make_map(A, K, M, lda, BK3, BM, CU_TENSOR_MAP_SWIZZLE_128B);
      const CUtensorMap mbh = make_map(h16, kp16, p.np, kp16, BK3, p.bnr, CU_TENSOR_MAP_SWIZZLE_64B, true);
      const CUtensorMap mbl = make_map(l16, kp16, p.np, kp16, BK3, p.bnr, CU_TENSOR_MAP_SWIZZLE_64B, true);
      if (!tb) launch3f16<NN>(ma3, mbh, mbl, mc, p, s);
      else launch3f16<NT>(ma3, mbh, mbl, mc, p, s);
      print_trace(p, tb ? "NT f16" : "NN f16");
      return 2;
    }
    float* bh = ws;
    float* bl = ws + static_cast<size_t>(p.np) * kp;
    const long tot = static_cast<long>(p.np) * kp;
    split_b<<<static_cast<int>(std::min<long>(1024, (tot + 255) / 256)), 256, 0, s>>>(B, ldb, tb ? 0 : 1, p.np, kp, N, K,
                                                                                       p.terms, bh, bl);
    TC_CUDA(cudaGetLastError());
    const CUtensorMap ma = make_map(A, K, M, lda, BK, BM, CU_TENSOR_MAP_SWIZZLE_NONE);
    const CUtensorMap mbh = make_map(bh, kp, p.np, kp, BK, p.bnr, CU_TENSOR_MAP_SWIZZLE_64B);
    const CUtensorMap mbl = make_map(bl, kp, p.np, kp, BK, p.bnr, CU_TENSOR_MAP_SWIZZLE_64B);
    const CUtensorMap mc = make_map(C, N, M, ldc, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B);
    p.trace = trace_buffer();
    if (g_gemm_version == 3) {  // 32-K stages, SWIZZLE_128B boxes
      finish_params3(p, false);
      const CUtensorMap ma3 = make_map(A, K, M, lda, BK3, BM, CU_TENSOR_MAP_SWIZZLE_128B);
      const int CL = (g_gemm3_cluster == 2 && p.n_tiles == 2) ? 2 : 1;  // A multicast needs two column tiles
      const CUtensorMap mbh3 = make_map(bh, kp, p.np, kp, BK3, p.bnr, CU_TENSOR_MAP_SWIZZLE_128B);
      const CUtensorMap mbl3 = make_map(bl, kp, p.np, kp, BK3, p.bnr, CU_TENSOR_MAP_SWIZZLE_128B);
      const CUtensorMap ma3h = make_map(A, K, M, lda, BK3, BM / 2, CU_TENSOR_MAP_SWIZZLE_128B);  // CL = 2 halves
      if (CL == 2) {
        if (!tb) launch3<NN, 2>(ma3h, mbh3, mbl3, mc, p, s);
        else launch3<NT, 2>(ma3h, mbh3, mbl3, mc, p, s);
      } else {
        if (!tb) launch3<NN, 1>(ma3, mbh3, mbl3, mc, p, s);
        else launch3<NT, 1>(ma3, mbh3, mbl3, mc, p, s);
      }
    } else if (!tb) {
      launch2<NN>(ma, mbh, mbl, mc, p, s);
    } else {
      launch2<NT>(ma, mbh, mbl, mc, p, s);
    }
    print_trace(p, tb ? "NT" : "NN");
    return 2;
  }
  finish_params(p, N, !tb, mode == MG_GEMM_TF32X3 ? 3 : 1);
  p.m_tiles = static_cast<int>((M + BM - 1) / BM);
  p.n_items = p.m_tiles;
  static float* dbg = [] {
    float* d = nullptr;
    if (std::getenv("MGGCN_TC_DEBUG")) TC_CUDA(cudaMallocManaged(&d, sizeof(float) * 65536));
    return d;
  }();
  p.dbg = dbg;
  if (dbg) std::fill(dbg, dbg + 65536, -7.0f);
  const CUtensorMap ma = make_map(A, K, M, lda, BK, BM, CU_TENSOR_MAP_SWIZZLE_64B);
  if (!tb) {  // NN: W is K x N row-major -> MN-major boxes {32 n, 16 k}
    const CUtensorMap mb = make_map(B, N, K, ldb, 32, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    launch<NN>(ma, mb, p, s);
  } else {    // NT: W is N x K row-major -> K-major box {16 k, np rows}
    const CUtensorMap mb = make_map(B, K, N, ldb, BK, p.np, CU_TENSOR_MAP_SWIZZLE_64B);
    launch<NT>(ma, mb, p, s);
  }
  if (dbg) {
    TC_CUDA(cudaDeviceSynchronize());
    std::fprintf(stderr, "[tc dbg] M=%ld N=%ld K=%ld np=%d npb=%d nst=%d terms=%d\n  A tile:", static_cast<long>(M),
                 static_cast<long>(N), static_cast<long>(K), p.np, p.npb, p.nst, p.terms);
    for (int i = 0; i < 24; ++i) std::fprintf(stderr, " %.4g", dbg[i]);
    std::fprintf(stderr, "\n  B tile:");
    for (int i = 0; i < 24; ++i) std::fprintf(stderr, " %.4g", dbg[2048 + i]);
    std::fprintf(stderr, "\n  TMEM row0:");
    for (int i = 0; i < 8; ++i) std::fprintf(stderr, " %.4g", dbg[16384 + i]);
    std::fprintf(stderr, "\n  TMEM row1:");
    for (int i = 0; i < 8; ++i) std::fprintf(stderr, " %.4g", dbg[16384 + 32 + i]);
    std::fprintf(stderr, "\n");
  }
  return 1;
}

int gemm_tn_blocks(int mode, int nblocks, const int64_t* begin, const int64_t* len, int64_t M, int64_t N,
                   const float* H, int64_t ldh, const float* G, int64_t ldg, float* stage, int64_t ldc,
                   int64_t block_stride, float* ws, size_t ws_bytes, cudaStream_t s) {
  if (mode != MG_GEMM_TF32X3 && mode != MG_GEMM_TF32) throw ValueError("tc gemm: bad mode");
  if (N > 256) throw ValueError("tc gemm: N > 256 not supported (" + std::to_string(N) + ")");
  if (nblocks < 1 || nblocks > 8) throw ValueError("tc gemm: 1..8 blocks");
  if (M <= 0 || N <= 0) return 0;
  check_ptr(H, ldh, "H");
  check_ptr(G, ldg, "G");
  Params p{};
  p.M = M;
  p.N = N;
  p.C = stage;
  p.ldc = ldc;
  if (g_gemm_version >= 2)
    finish_params2(p, N, true, mode == MG_GEMM_TF32X3 ? 3 : 1);
  else
    finish_params(p, N, true, mode == MG_GEMM_TF32X3 ? 3 : 1);
  p.m_tiles = static_cast<int>((M + BM - 1) / BM);
  p.chunk_rows = g_split_rows;
  p.nblocks = nblocks;
  int64_t rows_hi = 0;
  p.blk_first[0] = 0;
  for (int g = 0; g < nblocks; ++g) {
    p.blk_begin[g] = begin[g];
    p.blk_len[g] = std::max<int64_t>(0, len[g]);
    const long chunks = (p.blk_len[g] + p.chunk_rows - 1) / p.chunk_rows;
    p.blk_first[g + 1] = p.blk_first[g] + static_cast<int>(chunks) * p.m_tiles;
    // the operand maps end at the last row a block actually covers: a 32-row box past it is zero-filled by
    // TMA instead of reading past the end of H / G (an empty block's begin can lie anywhere)
    if (p.blk_len[g] > 0) rows_hi = std::max<int64_t>(rows_hi, begin[g] + len[g]);
  }
  p.n_items = p.blk_first[nblocks] * (g_gemm_version >= 2 ? p.n_tiles : 1);
  const size_t need = sizeof(float) * static_cast<size_t>(p.blk_first[nblocks]) * BM * p.npb;
  if (p.n_items > 0 && (!ws || ws_bytes < need)) throw ValueError("tc gemm: TN split-K workspace too small");
  p.partial = ws;
  int kernels = 0;
  if (p.n_items > 0) {
    const int bk = g_gemm_version >= 2 ? bk2<TN>() : BK;  // K rows per stage of the kernel that runs
    const CUtensorMap mb = make_map(G, N, rows_hi, ldg, 32, bk, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    if (g_gemm_version >= 2) {  // A = H rows land raw ([16 k][128 m]) and go to TMEM transposed per lane
      const CUtensorMap ma = make_map(H, M, rows_hi, ldh, BM, bk, CU_TENSOR_MAP_SWIZZLE_NONE);
      const CUtensorMap mc = make_map(ws, p.npb, static_cast<long>(p.blk_first[nblocks]) * BM, p.npb, 32, 32,
                                      CU_TENSOR_MAP_SWIZZLE_128B);
      p.trace = trace_buffer();
      launch2<TN>(ma, mb, mb, mc, p, s);
      print_trace(p, "TN");
    } else {
      const CUtensorMap ma = make_map(H, M, rows_hi, ldh, 32, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
      launch<TN>(ma, mb, p, s);
    }
    ++kernels;
  }
  const long total = M * N * nblocks;
  reduce_partials<<<static_cast<int>(std::min<long>(4096, (total + 255) / 256)), 256, 0, s>>>(p, stage, block_stride);
  TC_CUDA(cudaGetLastError());
  return kernels + 1;
}

}  // namespace tc
}  // namespace mg
