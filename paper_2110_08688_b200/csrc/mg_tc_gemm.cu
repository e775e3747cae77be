// SPDX-License-Identifier: Apache-2.0
//
// tcgen05 GeMMs of the training step (TF32X3 and TF32 modes), hand-written PTX for sm_100a.
//
//   NN  C[M,N] = A[M,K] W[K,N]       forward HW = H W            (rowgcn gemm NN, dense.hpp:158-169)
//   NT  C[M,N] = A[M,K] W[N,K]^T     H-grad, relu_backward fused (dense.hpp:182-193, :221-231)
//   TN  C[M,N] = A[K,M]^T B[K,N]     W-grad per canonical block  (dense.hpp:170-181), deterministic split-K
//
// Operands are staged by SIMT producer threads: float4 global loads, split x = hi + lo with
// hi = x & 0xffffe000 (exactly representable in TF32, so the tensor core reads it unchanged) and
// lo = x - hi (exact in fp32), written into the canonical UMMA K-major SWIZZLE_128B layout (8-row x
// 128-byte atoms, 16-byte chunk c of row r stored at chunk c ^ (r & 7)). One elected thread issues
// tcgen05.mma.kind::tf32 (M = 128, N <= 256, K = 8 per instruction) accumulating
//   D += A_hi B_hi + A_hi B_lo + A_lo B_hi        (TF32X3: fp32-level accuracy, ~2^-21 relative)
//   D += A_hi B_hi                                (TF32:   the 1-term mode, reported separately)
// into TMEM; tcgen05.commit arrives on an mbarrier per smem stage (double buffered, the next K block is
// staged while the tensor core consumes the current one). The epilogue reads TMEM with tcgen05.ld
// (warp w owns TMEM lanes 32*(w%4)..+31 = tile rows) and applies the fused epilogue on the way to HBM.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "mg_internal.hpp"
#include "mg_tc_gemm.cuh"

namespace mg {
namespace tc {

#define TC_CUDA(x)                                                                                     \
  do {                                                                                                 \
    cudaError_t _e = (x);                                                                              \
    if (_e != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(_e));           \
  } while (0)

constexpr int BM = 128;       // tile rows (TMEM lanes)
constexpr int BK = 32;        // fp32 per 128-byte swizzle row
constexpr int kThreads = 256;
static int g_split_rows = 4096;  // TN split-K chunk (rows), fixed relative to the block start (tuning "tn_chunk")

__host__ __device__ constexpr int a_bytes() { return BM * BK * 4; }           // 16 KB
__host__ __device__ constexpr int b_bytes(int np) { return np * BK * 4; }     // <= 32 KB
__host__ __device__ constexpr int stage_bytes(int np, int terms) {
  return terms == 1 ? a_bytes() + b_bytes(np) : 2 * (a_bytes() + b_bytes(np));
}
inline int smem_bytes(int np, int terms) { return 2 * stage_bytes(np, terms) + 1024 + 64; }

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity));
}

// SWIZZLE_128B K-major matrix descriptor (sm_100 "version 1"): start >> 4, LBO = 16 B (unused for
// swizzled K-major), SBO = 1024 B between 8-row groups, layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major, N >> 3 at bit 17, M >> 4 at bit 24.
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
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

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

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

// byte offset of (row, 16-byte chunk) inside a K-major SW128 tile of 128-byte rows
__device__ __forceinline__ uint32_t sw128_off(int row, int chunk) {
  return static_cast<uint32_t>((row >> 3) * 1024 + (row & 7) * 128 + ((chunk ^ (row & 7)) << 4));
}

__device__ __forceinline__ void split(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  lo = __fsub_rn(x, hi);
}

// ---------------------------------------------------------------- operand staging
// "direct": source row-major with K contiguous (rows = tile rows). Each 16-byte chunk is one float4.
template <bool SPLIT>
__device__ __forceinline__ void stage_direct(uint8_t* hi, uint8_t* lo, const float* __restrict__ src, long ld,
                                             long row0, long rows_valid, int rows_tile, int k0, int kpad) {
  const int nchunks = rows_tile * (BK / 4);
  for (int q = threadIdx.x; q < nchunks; q += kThreads) {
    const int r = q >> 3, c = q & 7;
    const long gr = row0 + r;
    const int k = k0 + 4 * c;
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (gr < rows_valid && k < kpad) x = __ldg(reinterpret_cast<const float4*>(src + gr * ld + k));
    const uint32_t off = sw128_off(r, c);
    if (SPLIT) {
      float4 h, l;
      split(x.x, h.x, l.x);
      split(x.y, h.y, l.y);
      split(x.z, h.z, l.z);
      split(x.w, h.w, l.w);
      *reinterpret_cast<float4*>(hi + off) = h;
      *reinterpret_cast<float4*>(lo + off) = l;
    } else {
      *reinterpret_cast<float4*>(hi + off) = x;
    }
  }
}

// "transposed": source row-major K x R (K = rows of the source, R contiguous). Lanes cover 8 k x 4
// float4 groups so the global reads are full 32-byte sectors and the scattered 4-byte smem writes
// hit at most 2 ways of every bank.
template <bool SPLIT>
__device__ __forceinline__ void stage_trans(uint8_t* hi, uint8_t* lo, const float* __restrict__ src, long ld,
                                            long k_row0, long k_rows_valid, int r0, int r_valid, int rows_tile) {
  const int groups = rows_tile / 4;  // float4 groups along R
  const int total = BK * groups;
  for (int q = threadIdx.x; q < total; q += kThreads) {
    const int lane = q & 31, wq = q >> 5;
    const int kk = (lane & 7) + 8 * (wq % (BK / 8));
    const int g4 = (lane >> 3) + 4 * (wq / (BK / 8));
    if (g4 >= groups) continue;
    const long gk = k_row0 + kk;
    const int rr = 4 * g4;
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (gk < k_rows_valid && r0 + rr < r_valid) x = __ldg(reinterpret_cast<const float4*>(src + gk * ld + r0 + rr));
    const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t off = sw128_off(rr + i, kk >> 2) + ((kk & 3) << 2);
      if (SPLIT) {
        float h, l;
        split(xs[i], h, l);
        *reinterpret_cast<float*>(hi + off) = h;
        *reinterpret_cast<float*>(lo + off) = l;
      } else {
        *reinterpret_cast<float*>(hi + off) = xs[i];
      }
    }
  }
}

struct Params {
  long M, N, K;          // logical sizes (K: reduction length; for TN the rows of A/B)
  const float* A;
  long lda;
  const float* B;
  long ldb;
  float* C;
  long ldc;
  int np;                // padded N (multiple of 16, <= 256)
  int kpad;              // K padded to the source's 4-float granularity (direct operands)
  int epi;               // 0 store, 1 relu_backward mask in place, 2 relu
  float* partial;        // TN: [n_chunks][m_tiles][BM][np]
  int n_chunks, m_tiles, k_chunk;
};

// MODE 0: NN (A direct, B transposed: W is K x N); 1: NT (A direct, B direct: W is N x K);
// 2: TN (A transposed: H is K x M, B transposed: G is K x N), split-K partials.
template <int MODE, int TERMS>
__global__ void __launch_bounds__(kThreads, 1) gemm_tc(Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t mbar[2];
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x >> 5;
  constexpr bool SPLIT = TERMS == 3;
  const int np = p.np;
  const int sb = stage_bytes(np, TERMS);

  // work item
  long m0, k_begin, k_end;
  int chunk = 0, mtile = 0;
  if (MODE == 2) {
    mtile = blockIdx.x % p.m_tiles;
    chunk = blockIdx.x / p.m_tiles;
    m0 = static_cast<long>(mtile) * BM;
    k_begin = static_cast<long>(chunk) * p.k_chunk;
    k_end = (p.K < k_begin + p.k_chunk) ? p.K : k_begin + p.k_chunk;
  } else {
    m0 = static_cast<long>(blockIdx.x) * BM;
    k_begin = 0;
    k_end = p.K;
  }

  if (threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    const uint32_t cols = np <= 32 ? 32 : np <= 64 ? 64 : np <= 128 ? 128 : 256;
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_s)),
                 "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  const uint32_t idesc = idesc_tf32(BM, np);

  const int nk = static_cast<int>((k_end - k_begin + BK - 1) / BK);
  uint32_t phase[2] = {0, 0};
  for (int it = 0; it < nk; ++it) {
    const int s = it & 1;
    if (it >= 2) {
      mbar_wait(&mbar[s], phase[s]);
      phase[s] ^= 1;
    }
    uint8_t* a_hi = smem + s * sb;
    uint8_t* a_lo = a_hi + a_bytes();
    uint8_t* b_hi = SPLIT ? a_lo + a_bytes() : a_hi + a_bytes();
    uint8_t* b_lo = b_hi + b_bytes(np);
    const long k0 = k_begin + static_cast<long>(it) * BK;
    if (MODE == 2) {
      stage_trans<SPLIT>(a_hi, a_lo, p.A, p.lda, k0, k_end, static_cast<int>(m0), static_cast<int>(p.M), BM);
      stage_trans<SPLIT>(b_hi, b_lo, p.B, p.ldb, k0, k_end, 0, static_cast<int>(p.N), np);
    } else {
      stage_direct<SPLIT>(a_hi, a_lo, p.A, p.lda, m0, p.M, BM, static_cast<int>(k0), p.kpad);
      if (MODE == 0)
        stage_trans<SPLIT>(b_hi, b_lo, p.B, p.ldb, k0, p.K, 0, static_cast<int>(p.N), np);
      else
        stage_direct<SPLIT>(b_hi, b_lo, p.B, p.ldb, 0, p.N, np, static_cast<int>(k0), p.kpad);
    }
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_fence_after();
      const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), bh = smem_u32(b_hi), bl = smem_u32(b_lo);
#pragma unroll
      for (int kk = 0; kk < BK / 8; ++kk) {
        const uint32_t off = kk * 32;  // 8 tf32 = 32 bytes along the swizzled row
        const uint32_t acc0 = (it > 0 || kk > 0) ? 1u : 0u;
        if (SPLIT) {
          mma_tf32(tmem, sw128_desc(al + off), sw128_desc(bh + off), idesc, acc0);
          mma_tf32(tmem, sw128_desc(ah + off), sw128_desc(bl + off), idesc, 1u);
          mma_tf32(tmem, sw128_desc(ah + off), sw128_desc(bh + off), idesc, 1u);
        } else {
          mma_tf32(tmem, sw128_desc(ah + off), sw128_desc(bh + off), idesc, acc0);
        }
      }
      mma_commit(&mbar[s]);
    }
  }
  // the last commit tracks every MMA issued before it
  if (nk > 0) {
    const int s = (nk - 1) & 1;
    mbar_wait(&mbar[s], phase[s]);
  }
  tc_fence_after();

  // epilogue: warps w and w+4 share TMEM lanes 32*(w%4) (tile rows), splitting the columns
  const int q = warp & 3;
  const int half = warp >> 2;
  const int row = q * 32 + (threadIdx.x & 31);
  const long grow = m0 + row;
  const int cols_half = (((np + 31) / 32) + 1) / 2 * 32;
  const int c_begin = half * cols_half, c_end = min(np, c_begin + cols_half);
  for (int c0 = c_begin; c0 < c_end; c0 += 32) {
    float v[32];
    if (nk > 0) {
      tmem_ld32(tmem + (static_cast<uint32_t>(q * 32) << 16) + c0, v);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = 0.f;
    }
    if (MODE == 2) {
      float* dst = p.partial + ((static_cast<long>(chunk) * p.m_tiles + mtile) * BM + row) * np + c0;
#pragma unroll
      for (int i = 0; i < 32; i += 4)  // np % 16 == 0: a float4 is wholly inside or outside the row
        if (c0 + i < np) *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    } else if (grow < p.M) {
      float* dst = p.C + grow * p.ldc;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const long c = c0 + i;
        if (c < p.N) {
          float r = v[i];
          if (p.epi == 1) r = dst[c] > 0.0f ? r : 0.0f;
          if (p.epi == 2) r = r > 0.0f ? r : 0.0f;
          dst[c] = r;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    const uint32_t cols = np <= 32 ? 32 : np <= 64 ? 64 : np <= 128 ? 128 : 256;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(cols));
  }
}

// Fixed-order sum of the split-K partials: C[m][n] = 0 + p_0 + p_1 + ... (chunk order).
__global__ void reduce_partials(const float* __restrict__ partial, int n_chunks, int m_tiles, int np, long M, long N,
                                float* __restrict__ C, long ldc) {
  const long total = M * N;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const long m = i / N, n = i % N;
    const long t = m / BM, r = m % BM;
    float s = 0.0f;
    for (int c = 0; c < n_chunks; ++c) s = __fadd_rn(s, partial[((static_cast<long>(c) * m_tiles + t) * BM + r) * np + n]);
    C[m * ldc + n] = s;
  }
}

bool available() { return true; }

void set_tn_chunk(int rows) {
  if (rows < BK || rows % BK) throw ValueError("tuning: tn_chunk must be a positive multiple of 32");
  g_split_rows = rows;
}

namespace {
template <int MODE, int TERMS>
void launch(const Params& p, int grid, cudaStream_t s) {
  const int sm = smem_bytes(p.np, TERMS);
  static bool attr = false;
  if (!attr) {
    TC_CUDA(cudaFuncSetAttribute(gemm_tc<MODE, TERMS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem_bytes(256, TERMS)));
    attr = true;
  }
  gemm_tc<MODE, TERMS><<<grid, kThreads, sm, s>>>(p);
  TC_CUDA(cudaGetLastError());
}
}  // namespace

size_t tn_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  const int np = static_cast<int>((N + 15) / 16 * 16);
  const long m_tiles = (M + BM - 1) / BM;
  const long chunks = (K + g_split_rows - 1) / g_split_rows;
  return sizeof(float) * static_cast<size_t>(chunks * m_tiles * BM * np);
}

int gemm(int mode, bool ta, bool tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B,
         int64_t ldb, float* C, int64_t ldc, int epi, float* ws, size_t ws_bytes, cudaStream_t s) {
  if (mode != MG_GEMM_TF32X3 && mode != MG_GEMM_TF32) throw ValueError("tc gemm: bad mode");
  if (N > 256) throw ValueError("tc gemm: N > 256 not supported (" + std::to_string(N) + ")");
  if (ta && tb) throw ValueError("gemm: transposed A and B together is not on the training path");
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15 || lda % 4 || ldb % 4)
    throw ValueError("tc gemm: operands must be 16-byte aligned with ld % 4 == 0");
  Params p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.A = A;
  p.lda = lda;
  p.B = B;
  p.ldb = ldb;
  p.C = C;
  p.ldc = ldc;
  p.np = static_cast<int>((N + 15) / 16 * 16);
  p.kpad = static_cast<int>((K + 3) / 4 * 4);
  p.epi = epi;
  const bool x3 = mode == MG_GEMM_TF32X3;
  if (!ta) {
    const int grid = static_cast<int>((M + BM - 1) / BM);
    if (!tb) {
      x3 ? launch<0, 3>(p, grid, s) : launch<0, 1>(p, grid, s);
    } else {
      x3 ? launch<1, 3>(p, grid, s) : launch<1, 1>(p, grid, s);
    }
    return 1;
  }
  // TN: split-K over fixed 4096-row chunks, then the fixed-order reduction (epilogue must be 0)
  if (epi != 0) throw ValueError("tc gemm: TN has no fused epilogue");
  p.m_tiles = static_cast<int>((M + BM - 1) / BM);
  p.k_chunk = g_split_rows;
  p.n_chunks = static_cast<int>(std::max<int64_t>(1, (K + p.k_chunk - 1) / p.k_chunk));
  if (!ws || ws_bytes < tn_workspace_bytes(M, N, std::max<int64_t>(K, 1)))
    throw ValueError("tc gemm: TN split-K workspace too small");
  p.partial = ws;
  const int grid = p.m_tiles * p.n_chunks;
  x3 ? launch<2, 3>(p, grid, s) : launch<2, 1>(p, grid, s);
  const long total = M * N;
  const int rb = static_cast<int>(std::min<long>(4096, (total + 255) / 256));
  reduce_partials<<<rb, 256, 0, s>>>(p.partial, p.n_chunks, p.m_tiles, p.np, M, N, C, ldc);
  TC_CUDA(cudaGetLastError());
  return 2;
}

}  // namespace tc
}  // namespace mg
