// Probe: issue cost of tcgen05.mma kind::tf32 (M = 128, K = 8) against N, A source (TMEM "ts" / SMEM "ss")
// and accumulator reuse. One CTA per SM, one thread issues back-to-back MMAs in groups of 12 (one
// 32-K stage of the 3xTF32 GeMM), committing each group to an mbarrier nobody waits on until the end.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_probe scripts/mma_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc_k128(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(2) << 61);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

template <bool TS>
__device__ __forceinline__ void mma(uint32_t d, uint32_t a_tmem, uint64_t a_desc, uint64_t b, uint32_t idesc) {
  if (TS)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                 ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc));
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(a_desc), "l"(b), "r"(idesc));
}

__device__ volatile int g_stop;

// contention modes: bit 0 = 4 warps tcgen05.st 64 TMEM columns in a loop, bit 1 = 4 warps ld.shared.v4 in a
// loop (each over its own 16 KB), bit 2 = 4 warps tcgen05.ld 32 columns in a loop
__device__ __forceinline__ void mma_ts_elect(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
               "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
               ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

// the GeMM's issue loop: descriptors from a rotating W slot, lane 0 only (WARP = 0) or warp-wide with
// elect.sync inside the asm (WARP = 1)
template <int N, int WARP, int FENCE = 0>
__global__ void __launch_bounds__(128, 1) probe_loop(long long* out, int groups) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar2, done_bar;
  __shared__ uint32_t tbase;
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&done_bar)));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&done_bar)) : "memory");
  }
  for (int i = threadIdx.x; i < (4 * 2 * N * 128) / 16; i += blockDim.x) reinterpret_cast<int4*>(s)[i] = make_int4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tbase;
  const int b_bytes = N * 128;
  if (threadIdx.x < 32) {
    const uint32_t idesc = idesc_tf32(128, N);
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      const int w = g % 4, j = g % 4;
      const uint32_t d = tmem + static_cast<uint32_t>((g / 8) & 1) * 128u;
      const uint32_t bh = smem_u32(s + w * 2 * b_bytes), bl = bh + b_bytes;
      const uint32_t ah = tmem + 256u + static_cast<uint32_t>(j * 64), al = ah + 32;
      if (FENCE >= 2)
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n"
                     ::"r"(smem_u32(&done_bar)) : "memory");
      if (FENCE >= 1) asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      if (FENCE >= 3) {
        if ((threadIdx.x & 31) == 0)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar2))
                       : "memory");
        __syncwarp();
      }
      if (WARP == 0) {
        if ((threadIdx.x & 31) == 0) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t dbh = desc_k128(bh + kk * 32), dbl = desc_k128(bl + kk * 32);
            const uint32_t first = (g % 8 == 0 && kk == 0) ? 0u : 1u;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                         ::"r"(d), "r"(al + kk * 8), "l"(dbh), "r"(idesc), "r"(first));
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                         ::"r"(d), "r"(ah + kk * 8), "l"(dbl), "r"(idesc), "r"(1u));
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                         ::"r"(d), "r"(ah + kk * 8), "l"(dbh), "r"(idesc), "r"(1u));
          }
        }
        __syncwarp();
      } else {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t dbh = desc_k128(bh + kk * 32), dbl = desc_k128(bl + kk * 32);
          const uint32_t first = (g % 8 == 0 && kk == 0) ? 0u : 1u;
          mma_ts_elect(d, al + kk * 8, dbh, idesc, first);
          mma_ts_elect(d, ah + kk * 8, dbl, idesc, 1u);
          mma_ts_elect(d, ah + kk * 8, dbh, idesc, 1u);
        }
        __syncwarp();
      }
    }
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar2))
                   : "memory");
      asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n"
                   ::"r"(smem_u32(&bar2)) : "memory");
    }
    __syncwarp();
    long long t2 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

template <int N, int WARP, int FENCE = 0>
void run_loop(const char* name, long long* d_out, int nsm) {
  const int groups = 2000;
  const size_t smem = 4 * 2 * N * 128 + 1024;
  cudaFuncSetAttribute(probe_loop<N, WARP, FENCE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe_loop<N, WARP, FENCE><<<nsm, 128, smem>>>(d_out, 10);
  cudaDeviceSynchronize();
  probe_loop<N, WARP, FENCE><<<nsm, 128, smem>>>(d_out, groups);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  long long h[2];
  cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-26s issue %6.1f cyc/mma  complete %6.1f cyc/mma\n", name, h[0] / (groups * 12.0), h[1] / (groups * 12.0));
}

// kind::f16 (fp16 inputs, fp32 accumulate): D f32 (bit 4), A/B f16 (format 0 at bits 7, 10), K = 16.
__host__ __device__ constexpr uint32_t idesc_f16(int m, int n) {
  return (1u << 4) | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}
template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) probe_f16(long long* out, int groups) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar2;
  __shared__ uint32_t tbase;
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < (2 * 256 * 128 + 128 * 128) / 16; i += blockDim.x) reinterpret_cast<int4*>(s)[i] = make_int4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tbase;
  if (threadIdx.x < 32) {
    const uint32_t idesc = idesc_f16(128, N);
    const uint32_t bs = smem_u32(s), as = bs + 2 * 256 * 128;
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {  // 4 K steps of 16 = one 64-K stage
        const uint64_t b = desc_k128(bs + kk * 32), a = desc_k128(as + kk * 32);
        const uint32_t at = tmem + 256 + kk * 8;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          if (TS)
            asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, 1, 0;\n"
                         "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                         ::"r"(tmem), "r"(at), "l"(b), "r"(idesc));
          else
            asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, 1, 0;\n"
                         "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                         ::"r"(tmem), "l"(a), "l"(b), "r"(idesc));
        }
      }
      __syncwarp();
    }
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar2)) : "memory");
      asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n"
                   ::"r"(smem_u32(&bar2)) : "memory");
    }
    __syncwarp();
    long long t2 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}
template <int N, bool TS>
void run_f16(const char* name, long long* d_out, int nsm) {
  const int groups = 2000;
  const size_t smem = 2 * 256 * 128 + 128 * 128 + 1024;
  cudaFuncSetAttribute(probe_f16<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe_f16<N, TS><<<nsm, 128, smem>>>(d_out, 10);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe_f16<N, TS><<<nsm, 128, smem>>>(d_out, groups);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long h[2];
  cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  const double mmas = groups * 12.0;
  printf("%-26s issue %6.1f cyc/mma  complete %6.1f cyc/mma  %.0f f16 TFLOP/s (K = 16 per MMA)\n", name, h[0] / mmas,
         h[1] / mmas, 2.0 * 128 * N * 16 * mmas * nsm / (ms * 1e-3) / 1e12);
}

template <int N, bool TS, int NACC, int CONT, int ORD>
__global__ void __launch_bounds__(384, 1) probe(long long* out, int groups, const float* gsrc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2, tbar[2];
  __shared__ uint32_t tbase;
  __shared__ volatile int done;
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < (2 * 256 * 128 + 128 * 128) / 16; i += blockDim.x)
    reinterpret_cast<int4*>(s)[i] = make_int4(0x3f800000, 0, 0x3f000000, 0);
  if (threadIdx.x == 0) {
    done = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar2)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&tbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&tbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_tf32(128, N);
    const uint32_t bs = smem_u32(s), as = bs + 2 * 256 * 128;
    const uint32_t a_t = tmem + 256 + (NACC == 2 && N > 128 ? 0 : 0);
    long long t0 = clock64();
    uint32_t phase = 0;
    for (int g = 0; g < groups; ++g) {
      const uint32_t d = tmem + (NACC == 2 ? static_cast<uint32_t>((g & 1) * (N <= 128 ? 128 : 0)) : 0u);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t b = desc_k128(bs + kk * 32);
        const uint64_t a = desc_k128(as + kk * 32);
        // ORD 0: same A / B; 1: A alternates hi, lo; 2: B alternates hi, lo; 3: the GeMM's (lo,hi) (hi,lo) (hi,hi);
        // 4: (hi,hi) (lo,hi) (hi,lo)
        const uint32_t ah = a_t + kk * 8, al = ah + 32;
        const uint64_t bh = b, bl = desc_k128(bs + N * 128 + kk * 32);
        const uint64_t adh = a, adl = desc_k128(as + 64 * 128 + kk * 32);
        if (ORD == 0) { mma<TS>(d, ah, adh, bh, idesc); mma<TS>(d, ah, adh, bh, idesc); mma<TS>(d, ah, adh, bh, idesc); }
        if (ORD == 1) { mma<TS>(d, al, adl, bh, idesc); mma<TS>(d, ah, adh, bh, idesc); mma<TS>(d, al, adl, bh, idesc); }
        if (ORD == 2) { mma<TS>(d, ah, adh, bl, idesc); mma<TS>(d, ah, adh, bh, idesc); mma<TS>(d, ah, adh, bl, idesc); }
        if (ORD == 3) { mma<TS>(d, al, adl, bh, idesc); mma<TS>(d, ah, adh, bl, idesc); mma<TS>(d, ah, adh, bh, idesc); }
        if (ORD == 4) { mma<TS>(d, ah, adh, bh, idesc); mma<TS>(d, al, adl, bh, idesc); mma<TS>(d, ah, adh, bl, idesc); }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar))
                   : "memory");
      (void)phase;
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar2))
                 : "memory");
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n"
                 ::"r"(smem_u32(&bar2)) : "memory");
    long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
    done = 1;
  } else if (threadIdx.x >= 128 && threadIdx.x < 256 && (CONT & 1)) {
    const int q = (threadIdx.x >> 5) & 3;
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = threadIdx.x + i;
    while (!done) {
      const uint32_t ta = tmem + (static_cast<uint32_t>(q * 32) << 16) + 448u;
      for (int c = 0; c < 4; ++c)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
                     ::"r"(ta + c * 16), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
                     "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
                     "r"(v[15]) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }
  } else if (threadIdx.x >= 128 && threadIdx.x < 256 && (CONT & 4)) {
    const int q = (threadIdx.x >> 5) & 3;
    uint32_t acc = 0;
    while (!done) {
      uint32_t r[16];
      const uint32_t ta = tmem + (static_cast<uint32_t>(q * 32) << 16) + 448u;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                   : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      for (int i = 0; i < 16; ++i) acc += r[i];
    }
    if (acc == 12345) out[2] = acc;
  } else if (threadIdx.x == 256 && (CONT & 8)) {
    // bulk global -> shared copies of 16 KB into a 2-slot ring after the operands (the GeMM's A stream)
    const uint32_t ring = smem_u32(s) + 2 * 256 * 128 + 128 * 128;
    uint32_t n = 0;
    while (!done) {
      const int slot = n & 1;
      if (n >= 2) {
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                     ::"r"(smem_u32(&tbar[slot])), "r"(((n >> 1) - 1) & 1) : "memory");
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&tbar[slot])), "r"(16384) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                   ::"r"(ring + slot * 16384), "l"(gsrc + (size_t)((blockIdx.x * 64 + (n & 63)) % 4096) * 4096), "r"(16384),
                     "r"(smem_u32(&tbar[slot])) : "memory");
      ++n;
    }
    for (int k = 0; k < 2 && n >= 1; ++k) {
      const uint32_t m = n - 1 - k;
      asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                   ::"r"(smem_u32(&tbar[m & 1])), "r"((m >> 1) & 1) : "memory");
      if (m == 0) break;
    }
  } else if (threadIdx.x >= 256 && (CONT & 2)) {
    const uint32_t base = smem_u32(s) + static_cast<uint32_t>(((threadIdx.x - 256) & 127) * 128);
    float a = 0.f;
    while (!done) {
      for (int c = 0; c < 8; ++c) {
        float x0, x1, x2, x3;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(x0), "=f"(x1), "=f"(x2), "=f"(x3)
                     : "r"(base + static_cast<uint32_t>(((c ^ (threadIdx.x & 7)) << 4))));
        a += x0 + x1 + x2 + x3;
      }
    }
    if (a == 1.2345f) out[2] = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

static const float* g_src;
template <int N, bool TS, int NACC, int CONT = 0, int ORD = 0>
void run(const char* name, long long* d_out, int nsm) {
  const int groups = 2000;
  const size_t smem = 2 * 256 * 128 + 128 * 128 + 2 * 16384 + 1024;
  cudaFuncSetAttribute(probe<N, TS, NACC, CONT, ORD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe<N, TS, NACC, CONT, ORD><<<nsm, 384, smem>>>(d_out, 10, g_src);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<N, TS, NACC, CONT, ORD><<<nsm, 384, smem>>>(d_out, groups, g_src);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long h[2];
  cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  const double mmas = groups * 12.0;
  const double tf = 2.0 * 128 * N * 8 * mmas * nsm / (ms * 1e-3) / 1e12;
  printf("%-22s issue %6.1f cyc/mma  complete %6.1f cyc/mma  %.3f ms  %.0f TF32 TFLOP/s\n", name, h[0] / mmas,
         h[1] / mmas, ms, tf);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  cudaMalloc(&d, 32);
  float* src;
  cudaMalloc(&src, 4096ull * 4096 * 4);  // 64 MB: an L2-sized stream
  cudaMemset(src, 0, 4096ull * 4096 * 4);
  g_src = src;
  run_loop<128, 1, 0>("tf32 loop N=128 elect", d, nsm);
  run_f16<128, false>("f16 ss N=128", d, nsm);
  run_f16<128, true>("f16 ts N=128", d, nsm);
  run_f16<256, true>("f16 ts N=256", d, nsm);
  run_f16<48, true>("f16 ts N=48", d, nsm);
  return 0;
}
