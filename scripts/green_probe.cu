// Probe: SM partitioning with green contexts on B200.
//  1. runtime-allocated memory + runtime <<<>>> launches into green-context streams (does it work,
//     are the SM sets disjoint?);
//  2. bandwidth of a 1 KB-row random gather (the SpMM access pattern) against the SM count;
//  3. a gather on one partition concurrently with an FMA loop on the other.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/green_probe scripts/green_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)
#define CD(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s:%d %s\n", __FILE__, __LINE__, s); exit(1); } } while (0)

__global__ void smid_kernel(int* out) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
}

// each warp gathers `per_warp` random rows of 256 floats (1 KB) and sums them into out
__global__ void gather_kernel(const float4* __restrict__ h, const int* __restrict__ idx, long n_idx, float4* out) {
  const int lane = threadIdx.x & 31;
  const long warps = (long)gridDim.x * (blockDim.x / 32);
  float4 acc[2] = {make_float4(0, 0, 0, 0), make_float4(0, 0, 0, 0)};
  for (long w = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; w * 8 < n_idx; w += warps) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const long r = __ldg(idx + w * 8 + e);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        float4 v = __ldg(h + r * 64 + lane + 32 * k);
        acc[k].x += v.x; acc[k].y += v.y; acc[k].z += v.z; acc[k].w += v.w;
      }
    }
  }
  out[(blockIdx.x * blockDim.x + threadIdx.x) % 4096] = make_float4(acc[0].x + acc[1].x, acc[0].y, acc[0].z, acc[0].w);
}

__global__ void fma_kernel(float* out, int iters) {
  float a = threadIdx.x * 1e-3f, b = 1.0001f, c = 0.5f, d = 0.25f;
  for (int i = 0; i < iters; ++i) {
    a = fmaf(a, b, c); c = fmaf(c, b, d); d = fmaf(d, b, a);
  }
  if (a + c + d == 12345.f) out[0] = a;
}

struct Part { CUgreenCtx g; CUstream s; int sms; };

static std::vector<Part> split(CUdevice dev, int first_sms) {
  CUdevResource all, res[2], rem;
  CD(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  unsigned n = 1;
  CD(cuDevSmResourceSplitByCount(res, &n, &all, &rem, 0, first_sms));
  std::vector<Part> out;
  CUdevResource* rs[2] = {&res[0], &rem};
  for (int i = 0; i < 2; ++i) {
    CUdevResourceDesc d;
    CD(cuDevResourceGenerateDesc(&d, rs[i], 1));
    Part p;
    CD(cuGreenCtxCreate(&p.g, d, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CD(cuGreenCtxStreamCreate(&p.s, p.g, CU_STREAM_NON_BLOCKING, 0));
    p.sms = rs[i]->sm.smCount;
    out.push_back(p);
  }
  return out;
}

int main() {
  CK(cudaSetDevice(0));
  CK(cudaFree(0));
  CUdevice dev;
  CD(cuDeviceGet(&dev, 0));
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const long rows = 2449029, n_idx = 124L << 20;
  float4* h;
  int* idx;
  float4* out;
  float* fout;
  CK(cudaMalloc(&h, rows * 1024));
  CK(cudaMalloc(&idx, n_idx * 4));
  CK(cudaMalloc(&out, 4096 * 16));
  CK(cudaMalloc(&fout, 16));
  CK(cudaMemset(h, 0, rows * 1024));
  {
    std::vector<int> hi(n_idx);
    unsigned long long x = 88172645463325252ull;
    for (long i = 0; i < n_idx; ++i) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      hi[i] = (int)(x % rows);
    }
    CK(cudaMemcpy(idx, hi.data(), n_idx * 4, cudaMemcpyHostToDevice));
  }
  int* smids;
  CK(cudaMalloc(&smids, 4096 * 4));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto time_gather = [&](cudaStream_t s, int sms) {
    const int grid = sms * 8;
    gather_kernel<<<grid, 256, 0, s>>>(h, idx, n_idx, out);
    CK(cudaEventRecord(a, s));
    for (int r = 0; r < 3; ++r) gather_kernel<<<grid, 256, 0, s>>>(h, idx, n_idx, out);
    CK(cudaEventRecord(b, s));
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms / 3;
  };
  const double gbytes = n_idx * 1024.0 / 1e9;
  float base = time_gather(0, nsm);
  printf("full device (%d SMs): gather %.2f ms, %.0f GB/s\n", nsm, base, gbytes / base * 1e3);
  for (int g : {16, 24, 32, 40, 48}) {
    std::vector<Part> p = split(dev, g);
    // disjointness
    std::vector<int> ids0(p[0].sms * 4), ids1(p[1].sms * 4);
    smid_kernel<<<p[0].sms * 4, 32, 0, (cudaStream_t)p[0].s>>>(smids);
    smid_kernel<<<p[1].sms * 4, 32, 0, (cudaStream_t)p[1].s>>>(smids + 2048);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(ids0.data(), smids, ids0.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ids1.data(), smids + 2048, ids1.size() * 4, cudaMemcpyDeviceToHost));
    unsigned long long m0[3] = {0, 0, 0}, m1[3] = {0, 0, 0};
    for (int v : ids0) m0[v / 64] |= 1ull << (v % 64);
    for (int v : ids1) m1[v / 64] |= 1ull << (v % 64);
    int c0 = 0, c1 = 0, ov = 0;
    for (int i = 0; i < 3; ++i) {
      c0 += __builtin_popcountll(m0[i]);
      c1 += __builtin_popcountll(m1[i]);
      ov += __builtin_popcountll(m0[i] & m1[i]);
    }
    float tg = time_gather((cudaStream_t)p[1].s, p[1].sms);
    // FMA alone on part 0, then both concurrently
    const int iters = 1 << 20;
    CK(cudaEventRecord(a, (cudaStream_t)p[0].s));
    fma_kernel<<<p[0].sms * 4, 256, 0, (cudaStream_t)p[0].s>>>(fout, iters);
    CK(cudaEventRecord(b, (cudaStream_t)p[0].s));
    CK(cudaEventSynchronize(b));
    float tf;
    CK(cudaEventElapsedTime(&tf, a, b));
    cudaEvent_t c, d;
    CK(cudaEventCreate(&c));
    CK(cudaEventCreate(&d));
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a, (cudaStream_t)p[1].s));
    for (int r = 0; r < 3; ++r) gather_kernel<<<p[1].sms * 8, 256, 0, (cudaStream_t)p[1].s>>>(h, idx, n_idx, out);
    CK(cudaEventRecord(b, (cudaStream_t)p[1].s));
    CK(cudaEventRecord(c, (cudaStream_t)p[0].s));
    fma_kernel<<<p[0].sms * 4, 256, 0, (cudaStream_t)p[0].s>>>(fout, iters);
    CK(cudaEventRecord(d, (cudaStream_t)p[0].s));
    CK(cudaDeviceSynchronize());
    float tg2, tf2;
    CK(cudaEventElapsedTime(&tg2, a, b));
    CK(cudaEventElapsedTime(&tf2, c, d));
    printf("split %3d/%3d SMs (seen %d/%d, overlap %d): gather on %d SMs %.2f ms (%.0f GB/s); fma alone %.2f ms; "
           "together gather %.2f ms (%.0f GB/s), fma %.2f ms\n",
           p[0].sms, p[1].sms, c0, c1, ov, p[1].sms, tg, gbytes / tg * 1e3, tf, tg2 / 3, gbytes / (tg2 / 3) * 1e3, tf2);
    for (auto& q : p) {
      CD(cuStreamDestroy(q.s));
      CD(cuGreenCtxDestroy(q.g));
    }
  }
  printf("ok\n");
  return 0;
}
