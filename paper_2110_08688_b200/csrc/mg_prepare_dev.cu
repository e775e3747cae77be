// SPDX-License-Identifier: Apache-2.0
//
// Device partitioner: rowgcn::prepare_data (inc/driver.hpp:87-117) with the graph
// work on the GPU, bit-identical to the host partitioner in mg_host.cpp (and so to the reference):
//   * random_permutation (partition.hpp:69-79) and permute_rows / permute_values stay on the host
//     (one sequential mt19937_64 pass; O(n d0) copies);
//   * permute_graph (partition.hpp:101-116): every entry (u, v) -> key (pi(u) << 32 | pi(v)), one radix
//     sort of (key, value) pairs = rows in order, columns sorted — no COO on the host;
//   * transpose (sparse.hpp:110-129): keys swapped to (col << 32 | row) and sorted again; entries are
//     unique, so the order equals the reference's stable counting sort;
//   * normalize_in_degree (sparse.hpp:94-107): column sums accumulated left to right over the transposed
//     rows (the reference's order: increasing source row), then one IEEE division per entry;
//   * tile_rows (partition.hpp:173-225): per-row split points by binary search, per-tile scans, local
//     columns. Tiles come back to the host partition (mg_partition), so every consumer is unchanged.
// Device memory: ~ 28 bytes per nonzero at the peak (keys and values double-buffered by the sort).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <numeric>

#include "mg_internal.hpp"

namespace mg {

void random_permutation(index_t n, std::uint64_t seed, std::vector<index_t>& forward);  // mg_host.cpp

namespace {

#define PD_CUDA(x)                                                                                      \
  do {                                                                                                  \
    cudaError_t _e = (x);                                                                               \
    if (_e != cudaSuccess) {                                                                            \
      (void)cudaGetLastError();                                                                         \
      throw CudaError(std::string("prepare_device: ") + #x + ": " + cudaGetErrorString(_e));            \
    }                                                                                                   \
  } while (0)

template <class T>
struct DBuf {  // owning device buffer
  T* p = nullptr;
  size_t n = 0;
  explicit DBuf(size_t count = 0) { alloc(count); }
  void alloc(size_t count) {
    free();
    n = count;
    if (count) PD_CUDA(cudaMalloc(&p, sizeof(T) * count));
  }
  void free() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { free(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
};

inline int grid_for(size_t n) { return static_cast<int>(std::min<size_t>((n + 255) / 256, 148 * 16)); }

// key = (pi(u) << 32) | pi(v) for every entry of the input CSR (warp per row keeps hub rows balanced)
__global__ void build_keys(const index_t* __restrict__ rp, const index_t* __restrict__ ci,
                           const index_t* __restrict__ fwd, index_t n, unsigned long long* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  for (index_t u = (blockIdx.x * (index_t)blockDim.x + threadIdx.x) >> 5; u < n;
       u += (gridDim.x * (index_t)blockDim.x) >> 5) {
    const unsigned long long r = static_cast<unsigned long long>(fwd ? fwd[u] : u) << 32;
    for (index_t k = rp[u] + lane; k < rp[u + 1]; k += 32) {
      const index_t v = ci[k];
      keys[k] = r | static_cast<unsigned long long>(fwd ? fwd[v] : v);
    }
  }
}

__global__ void swap_keys(const unsigned long long* __restrict__ in, unsigned long long* __restrict__ out, size_t m) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x) {
    const unsigned long long k = in[i];
    out[i] = (k << 32) | (k >> 32);
  }
}

// row counts from sorted keys: cnt[row]++ (row = key >> 32)
__global__ void row_counts(const unsigned long long* __restrict__ keys, size_t m, index_t* __restrict__ cnt) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(cnt + (keys[i] >> 32)), 1ull);
}

// normalize_in_degree: col_sum[v] = sum over row v of A^T, left to right (the reference's order)
__global__ void col_sums(const index_t* __restrict__ trp, const float* __restrict__ tv, index_t n,
                         float* __restrict__ cs) {
  for (index_t v = blockIdx.x * (index_t)blockDim.x + threadIdx.x; v < n; v += gridDim.x * (index_t)blockDim.x) {
    float s = 0.0f;
    for (index_t k = trp[v]; k < trp[v + 1]; ++k) s += tv[k];
    cs[v] = s;
  }
}

// a.v[k] /= col_sum[col(k)]  (A),  at.v[k] /= col_sum[row(k)]  (A^T): the low / high key half
__global__ void normalize(const unsigned long long* __restrict__ keys, float* __restrict__ v, size_t m,
                          const float* __restrict__ cs, int by_high) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    const float s = cs[by_high ? (k >> 32) : (k & 0xffffffffull)];
    v[i] = s != 0.0f ? __fdiv_rn(v[i], s) : 0.0f;
  }
}

// split[r * (P + 1) + j] = first entry of row (r0 + r) with column >= bounds[j]
__global__ void row_splits(const index_t* __restrict__ rp, const unsigned long long* __restrict__ keys, index_t r0,
                           index_t rows, const index_t* __restrict__ bounds, int P, index_t* __restrict__ split) {
  for (index_t r = blockIdx.x * (index_t)blockDim.x + threadIdx.x; r < rows; r += gridDim.x * (index_t)blockDim.x) {
    const index_t b = rp[r0 + r], e = rp[r0 + r + 1];
    for (int j = 0; j < P; ++j) {
      index_t lo = b, hi = e;  // lower_bound on the column (low key half)
      const unsigned long long target = static_cast<unsigned long long>(bounds[j]);
      while (lo < hi) {
        const index_t mid = (lo + hi) >> 1;
        if ((keys[mid] & 0xffffffffull) < target) lo = mid + 1;
        else hi = mid;
      }
      split[r * (P + 1) + j] = lo;
    }
    split[r * (P + 1) + P] = e;
  }
}

__global__ void tile_counts(const index_t* __restrict__ split, index_t rows, int P, int j, index_t* __restrict__ cnt) {
  for (index_t r = blockIdx.x * (index_t)blockDim.x + threadIdx.x; r < rows; r += gridDim.x * (index_t)blockDim.x)
    cnt[r] = split[r * (P + 1) + j + 1] - split[r * (P + 1) + j];
}

__global__ void tile_fill(const index_t* __restrict__ split, const index_t* __restrict__ trp,
                          const unsigned long long* __restrict__ keys, const float* __restrict__ vals, index_t rows,
                          int P, int j, std::int32_t base, std::int32_t* __restrict__ col, float* __restrict__ val) {
  const int lane = threadIdx.x & 31;
  for (index_t r = (blockIdx.x * (index_t)blockDim.x + threadIdx.x) >> 5; r < rows;
       r += (gridDim.x * (index_t)blockDim.x) >> 5) {
    const index_t s0 = split[r * (P + 1) + j], s1 = split[r * (P + 1) + j + 1], o = trp[r];
    for (index_t k = s0 + lane; k < s1; k += 32) {
      col[o + (k - s0)] = static_cast<std::int32_t>(keys[k] & 0xffffffffull) - base;
      val[o + (k - s0)] = vals[k];
    }
  }
}

template <class T>
void up(T* d, const T* h, size_t n) {
  if (n) PD_CUDA(cudaMemcpy(d, h, sizeof(T) * n, cudaMemcpyHostToDevice));
}
template <class T>
void down(T* h, const T* d, size_t n) {
  if (n) PD_CUDA(cudaMemcpy(h, d, sizeof(T) * n, cudaMemcpyDeviceToHost));
}

// Sorts (keys, vals) in place (through the alternate buffers); bits = significant key bits.
void sort_pairs(DBuf<unsigned long long>& k, DBuf<unsigned long long>& k2, DBuf<float>& v, DBuf<float>& v2, size_t m,
                int bits) {
  if (m == 0) return;
  cub::DoubleBuffer<unsigned long long> kb(k.p, k2.p);
  cub::DoubleBuffer<float> vb(v.p, v2.p);
  size_t tmp = 0;
  PD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, static_cast<int64_t>(m), 0, bits));
  DBuf<unsigned char> t(tmp);
  PD_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, kb, vb, static_cast<int64_t>(m), 0, bits));
  if (kb.Current() != k.p) std::swap(k.p, k2.p);
  if (vb.Current() != v.p) std::swap(v.p, v2.p);
}

// Row pointers (n + 1, exclusive scan of per-row counts) of a key-sorted entry list.
void row_pointers(const DBuf<unsigned long long>& k, size_t m, index_t n, DBuf<index_t>& rp) {
  DBuf<index_t> cnt(static_cast<size_t>(n) + 1);
  PD_CUDA(cudaMemset(cnt.p, 0, sizeof(index_t) * (n + 1)));
  if (m) row_counts<<<grid_for(m), 256>>>(k.p, m, cnt.p);
  PD_CUDA(cudaGetLastError());
  rp.alloc(static_cast<size_t>(n) + 1);
  size_t tmp = 0;
  PD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.p, rp.p, static_cast<int64_t>(n + 1)));
  DBuf<unsigned char> t(tmp);
  PD_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, cnt.p, rp.p, static_cast<int64_t>(n + 1)));
}

// tile_rows for row block i of a key-sorted matrix (row pointers rp) into host tiles.
std::vector<Tile> tiles_of(const DBuf<index_t>& rp, const DBuf<unsigned long long>& k, const DBuf<float>& v,
                           const std::vector<index_t>& bounds, const DBuf<index_t>& dbounds, int i) {
  const int P = static_cast<int>(bounds.size()) - 1;
  const index_t r0 = bounds[i], rows = bounds[i + 1] - r0;
  std::vector<Tile> tiles(P);
  DBuf<index_t> split(static_cast<size_t>(std::max<index_t>(rows, 1)) * (P + 1));
  if (rows) row_splits<<<grid_for(rows), 256>>>(rp.p, k.p, r0, rows, dbounds.p, P, split.p);
  PD_CUDA(cudaGetLastError());
  DBuf<index_t> cnt(static_cast<size_t>(rows) + 1), trp(static_cast<size_t>(rows) + 1);
  for (int j = 0; j < P; ++j) {
    Tile& t = tiles[j];
    t.rows = rows;
    t.cols = bounds[j + 1] - bounds[j];
    PD_CUDA(cudaMemset(cnt.p, 0, sizeof(index_t) * (rows + 1)));
    if (rows) tile_counts<<<grid_for(rows), 256>>>(split.p, rows, P, j, cnt.p);
    PD_CUDA(cudaGetLastError());
    size_t tmp = 0;
    PD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.p, trp.p, static_cast<int64_t>(rows + 1)));
    DBuf<unsigned char> tb(tmp);
    PD_CUDA(cub::DeviceScan::ExclusiveSum(tb.p, tmp, cnt.p, trp.p, static_cast<int64_t>(rows + 1)));
    t.row_ptr.resize(static_cast<size_t>(rows) + 1);
    down(t.row_ptr.data(), trp.p, static_cast<size_t>(rows) + 1);
    const index_t nnz = t.row_ptr[rows];
    DBuf<std::int32_t> col(static_cast<size_t>(nnz));
    DBuf<float> val(static_cast<size_t>(nnz));
    if (nnz)
      tile_fill<<<grid_for(static_cast<size_t>(rows) * 32), 256>>>(split.p, trp.p, k.p, v.p, rows, P, j,
                                                                   static_cast<std::int32_t>(bounds[j]), col.p, val.p);
    PD_CUDA(cudaGetLastError());
    t.col.resize(static_cast<size_t>(nnz));
    t.val.resize(static_cast<size_t>(nnz));
    down(t.col.data(), col.p, static_cast<size_t>(nnz));
    down(t.val.data(), val.p, static_cast<size_t>(nnz));
  }
  return tiles;
}

int key_bits(index_t n) {
  int b = 1;
  while ((index_t(1) << b) < n) ++b;
  return b;
}

}  // namespace
}  // namespace mg

using namespace mg;

extern "C" mg_status mg_prepare_device(const mg_dataset* ds, const mg_config* cfgp, int32_t workers, int32_t only_rank,
                                       int32_t device, mg_partition** out) {
  return guarded([&] {
    if (!ds || !out) throw ValueError("prepare: null argument");
    const Config cfg = to_config(cfgp);
    if (cfg.dims.front() != ds->d0)
      throw ConfigError("config: layer_dims[0]=" + std::to_string(cfg.dims.front()) +
                        " but dataset features have width " + std::to_string(ds->d0));
    if (workers <= 0) throw ValueError("uniform_partition: P must be >= 1, got " + std::to_string(workers));
    if (only_rank >= workers) throw ValueError("prepare: only_rank " + std::to_string(only_rank) + " >= P");
    validate_dataset_named(*ds);
    const index_t n = ds->n(), d0 = ds->d0, m = ds->graph.nnz();
    if (n >= (index_t(1) << 31)) throw ValueError("prepare: n >= 2^31 not supported");
    PD_CUDA(cudaSetDevice(device));
    auto p = std::make_unique<mg_partition>();
    p->n = n;
    p->d0 = d0;
    p->parts = workers;
    p->only_rank = only_rank;
    if (cfg.permute) {
      random_permutation(n, cfg.seed, p->perm_forward);
    } else {
      p->perm_forward.resize(n);
      std::iota(p->perm_forward.begin(), p->perm_forward.end(), index_t(0));
    }
    const auto& fwd = p->perm_forward;
    p->features.resize(static_cast<size_t>(n * d0));
    p->labels.resize(n);
    p->mask.resize(n);
    parallel_for(n, [&](index_t b, index_t e) {  // permute_rows / permute_values (partition.hpp:118-140)
      for (index_t u = b; u < e; ++u) {
        const index_t v = fwd[u];
        std::memcpy(&p->features[v * d0], &ds->features[u * d0], sizeof(float) * d0);
        p->labels[v] = ds->labels[u];
        p->mask[v] = ds->train_mask.empty() ? 1 : ds->train_mask[u];
      }
    });
    for (auto mk : p->mask) p->mask_count += mk ? 1 : 0;
    if (p->mask_count == 0) throw ValueError("training mask is empty");
    p->bounds.resize(workers + 1);
    for (int i = 0; i <= workers; ++i) p->bounds[i] = static_cast<index_t>(i) * n / workers;

    // ---- graph on the device
    const int bits = 32 + key_bits(n);  // row in the high word, column in the low word
    DBuf<unsigned long long> k(static_cast<size_t>(m)), k2(static_cast<size_t>(m));
    DBuf<float> v(static_cast<size_t>(m)), v2(static_cast<size_t>(m));
    {
      DBuf<index_t> rp(static_cast<size_t>(n) + 1), ci(static_cast<size_t>(m)), dfwd(cfg.permute ? n : 0);
      up(rp.p, ds->graph.row_ptr.data(), static_cast<size_t>(n) + 1);
      up(ci.p, ds->graph.col_idx.data(), static_cast<size_t>(m));
      up(v.p, ds->graph.values.data(), static_cast<size_t>(m));
      if (cfg.permute) up(dfwd.p, fwd.data(), static_cast<size_t>(n));
      if (n) build_keys<<<grid_for(static_cast<size_t>(n) * 32), 256>>>(rp.p, ci.p, cfg.permute ? dfwd.p : nullptr, n,
                                                                         k.p);
      PD_CUDA(cudaGetLastError());
    }
    sort_pairs(k, k2, v, v2, static_cast<size_t>(m), bits);  // A' (permute_graph): rows, sorted columns
    DBuf<unsigned long long> tk(static_cast<size_t>(m)), tk2(static_cast<size_t>(m));
    DBuf<float> tv(static_cast<size_t>(m)), tv2(static_cast<size_t>(m));
    if (m) {
      swap_keys<<<grid_for(static_cast<size_t>(m)), 256>>>(k.p, tk.p, static_cast<size_t>(m));
      PD_CUDA(cudaGetLastError());
      PD_CUDA(cudaMemcpy(tv.p, v.p, sizeof(float) * m, cudaMemcpyDeviceToDevice));
    }
    sort_pairs(tk, tk2, tv, tv2, static_cast<size_t>(m), bits);  // A'^T (transpose)
    k2.free();
    v2.free();
    tk2.free();
    tv2.free();
    DBuf<index_t> arp, trp;
    row_pointers(k, static_cast<size_t>(m), n, arp);
    row_pointers(tk, static_cast<size_t>(m), n, trp);
    {  // normalize_in_degree on both
      DBuf<float> cs(static_cast<size_t>(std::max<index_t>(n, 1)));
      if (n) col_sums<<<grid_for(static_cast<size_t>(n)), 256>>>(trp.p, tv.p, n, cs.p);
      PD_CUDA(cudaGetLastError());
      if (m) {
        normalize<<<grid_for(static_cast<size_t>(m)), 256>>>(k.p, v.p, static_cast<size_t>(m), cs.p, 0);
        normalize<<<grid_for(static_cast<size_t>(m)), 256>>>(tk.p, tv.p, static_cast<size_t>(m), cs.p, 1);
        PD_CUDA(cudaGetLastError());
      }
    }
    DBuf<index_t> dbounds(static_cast<size_t>(workers) + 1);
    up(dbounds.p, p->bounds.data(), static_cast<size_t>(workers) + 1);
    for (int d = 0; d < 2; ++d) p->tiles[d].resize(workers);
    for (int i = 0; i < workers; ++i) {
      if (!p->has_row(i)) continue;
      p->tiles[0][i] = tiles_of(trp, tk, tv, p->bounds, dbounds, i);  // forward tiles of A_hat^T
      p->tiles[1][i] = tiles_of(arp, k, v, p->bounds, dbounds, i);    // backward tiles of A_hat
    }
    PD_CUDA(cudaDeviceSynchronize());
    *out = p.release();
  });
}
