// SPDX-License-Identifier: Apache-2.0
//
// Device half of libmggcn.so: the per-GPU GcnWorker state (L+3 buffer plan in HBM), the
// communicator (NCCL, or the in-process rank-order transport when several workers share a device),
// the staged 1D row-broadcast SpMM schedule on two streams with CUDA events, and the training step.
// Reference: rowgcn inc/gcn.hpp (GcnWorker), inc/dist_spmm.hpp (staged SpMM), inc/collectives.hpp.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <future>
#include <memory>
#include <map>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "mg_internal.hpp"
#include "mg_kernels.cuh"
#include "mg_tc_gemm.cuh"

namespace mg {

#define MG_CUDA(x)                                                                                     \
  do {                                                                                                 \
    cudaError_t _e = (x);                                                                              \
    if (_e != cudaSuccess) {                                                                           \
      (void)cudaGetLastError(); /* non-sticky errors must not leak into the next launch check */       \
      throw CudaError(std::string(#x) + ": " + cudaGetErrorString(_e) + " (" + __FILE__ + ":" +        \
                      std::to_string(__LINE__) + ")");                                                 \
    }                                                                                                  \
  } while (0)
// Communicators are non-blocking (ncclCommInitRankConfig, blocking = 0) so a lost peer can be detected and
// the communicator aborted: calls may return ncclInProgress, and nccl_settle() completes them.
#define MG_NCCL(x)                                                                                     \
  do {                                                                                                 \
    ncclResult_t _r = (x);                                                                             \
    if (_r != ncclSuccess && _r != ncclInProgress)                                                     \
      throw NcclError(std::string(#x) + ": " + ncclGetErrorString(_r));                                \
  } while (0)
#define MG_LAUNCHED() MG_CUDA(cudaGetLastError())

namespace {

inline index_t pad4(index_t d) { return (d + 3) / 4 * 4; }
inline int ceil_div(index_t a, index_t b) { return static_cast<int>((a + b - 1) / b); }

std::atomic<int> g_heavy_row{4096};
std::atomic<long long> g_watchdog_ms{0};  // host-wait timeout before the group is aborted (0 = none)
std::atomic<long long> g_debug_stall_us{0};  // test hook: a spin kernel of this length at every step start
std::atomic<int> g_nccl_single{0};  // test hook: one-rank groups also get an NCCL communicator (exercised path)
std::atomic<int> g_profile{0};
std::atomic<int> g_step_graph{1};  // one-worker training steps replayed from a captured CUDA graph
// Opt-in ("ax_cache", default off; the bench headline never uses it): under aggregate_first, layer 0's SpMM
// Â·X depends on the inputs only, so a one-process group computes it once and keeps it until the features
// are written (mg_group_write) or the tuning changes. Results are bitwise those of the uncached step (the
// same kernel wrote the same buffer); the reference recomputes it every epoch (its order_swap path).
std::atomic<int> g_ax_cache{0};
std::atomic<uint64_t> g_tuning_epoch{1};  // bumped by every mg_set_tuning: a captured step graph is stale
std::atomic<int> g_spmm_slab{0};  // floats per column-slab pass of the SpMM (0 = the whole width, <= 1024)
std::atomic<int> g_narrow_group{0};  // lanes per row for widths of 33..64 floats (0 = 16, or 4 / 8)
int narrow_group() { return g_narrow_group.load(); }
int heavy_threshold() { return g_heavy_row.load(); }
// float4 chunks per SpMM launch: each launch walks every row's nonzeros for one column slab, so a slab of
// the gathered matrix (rows x slab x 4 B) can stay L2-resident while the edge stream passes through.
int slab_chunks() {
  const int s = g_spmm_slab.load();
  return s > 0 ? std::max(1, std::min(256, s / 4)) : 256;
}

int num_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

// ---------------------------------------------------------------- device CSR tile
struct DevTile {
  index_t rows = 0, cols = 0, nnz = 0;
  int* row_ptr = nullptr;   // rows + 1 (int32)
  int2* edges = nullptr;    // {col, float bits}
  int* light = nullptr;     // rows with nnz < heavy threshold, by decreasing length
  int n_light = 0;
  int* heavy = nullptr;     // rows with nnz >= heavy threshold
  int n_heavy = 0;
  // MG_SPMM_FAST work lists: items {e0, e1, dst, 0} (dst < 0: scratch segment), hubs {row, seg0, nseg, 0}
  int4* items = nullptr;
  int n_items = 0;
  int4* hubs = nullptr;
  int n_hubs = 0;
  int n_segments = 0;
  // MG_SPMM_FAST row-streaming pieces {r0, r1, e0, e1} (<= kPieceRows consecutive light rows) and hub-row
  // segments {-(seg+1), 0, e0, e1}, by decreasing nonzeros (spmm_fast_stream)
  int4* pieces = nullptr;
  int n_pieces = 0;
  bool hubs_classed = false;  // FAST: column hub classes in the top 4 bits of each edge record
};

std::atomic<int> g_fast_segment{2048};
// "stage_fold" = k (MG_SPMM_FAST, P > 2; 0 / 1 = off): up to k consecutive received stages are folded into
// one SpMM launch over a merged tile (the stages' tiles side by side, each block's columns shifted by the
// sizes of the blocks before it) reading the blocks from one k-block receive buffer: the output is
// read-modified-written once per group instead of once per stage. A group never contains the rank's own
// block (that stage reads its h in place). Off by default (the reference's stage-by-stage schedule and
// timeline); read at group creation.
std::atomic<int> g_stage_fold{0};
std::atomic<int> g_adaptive_cuts{1};  // "adaptive_cuts": FAST hub threshold / segment scaled to the tile

// MG_SPMM_FAST cut points of one tile: rows with >= ht nonzeros are hub rows cut into segments of seg
// nonzeros. One work item's gathers are serial in one lane group (~12 nonzeros per memory latency), so an
// item much longer than the launch's average share is the launch's tail: ncu of the C2 (arxiv-shaped)
// SpMM showed every SM idle after ~30% of the launch while one group folded a ~4000-nonzero row. The
// segment is therefore scaled to the tile: nnz / (SMs x 64) rounded down to a power of two, clamped to
// [64, fast_segment], and rows from 2 segments up are hubs (never above heavy_row).
struct FastCuts {
  int ht, seg;
};
int num_sms();
FastCuts fast_cuts(index_t nnz) {
  FastCuts c{g_heavy_row.load(), g_fast_segment.load()};
  if (!g_adaptive_cuts.load()) return c;
  const index_t share = nnz / (static_cast<index_t>(num_sms()) * 64);
  int seg = 64;
  while (seg * 2 <= share && seg * 2 <= c.seg) seg *= 2;
  c.seg = std::min(seg, c.seg);
  c.ht = std::max(1, std::min(c.ht, 2 * c.seg));
  return c;
}

// MGGCN_TIMING=1: host-side phase timings of group creation on stderr.
struct Stopwatch {
  bool on = std::getenv("MGGCN_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void lap(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[mggcn] %-12s %9.1f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// Fast-mode work lists: every hub row (>= heavy threshold) is cut into fixed segments of g_fast_segment
// nonzeros (gathered in parallel, summed in order afterwards); segments first, then the ordinary rows
// by decreasing length.
void build_fast_items(const std::vector<index_t>& rp, std::vector<int4>& items, std::vector<int4>& hubs, int& nseg) {
  const index_t rows = static_cast<index_t>(rp.size()) - 1;
  const FastCuts cuts = fast_cuts(rp.back());
  const int ht = cuts.ht, seg = cuts.seg;
  std::vector<int> light;
  items.clear();
  hubs.clear();
  nseg = 0;
  for (index_t r = 0; r < rows; ++r) {
    const index_t len = rp[r + 1] - rp[r];
    if (len < ht) {
      light.push_back(static_cast<int>(r));
      continue;
    }
    const int first = nseg;
    for (index_t e = rp[r]; e < rp[r + 1]; e += seg, ++nseg)
      items.push_back(make_int4(static_cast<int>(e), static_cast<int>(std::min<index_t>(e + seg, rp[r + 1])),
                                -(nseg + 1), 0));
    hubs.push_back(make_int4(static_cast<int>(r), first, nseg - first, 0));
  }
  // light rows by decreasing length, ties in row order: a counting sort (stable), O(rows + max length)
  index_t maxlen = 0;
  for (int r : light) maxlen = std::max(maxlen, rp[r + 1] - rp[r]);
  std::vector<index_t> cnt(static_cast<size_t>(maxlen) + 2, 0);
  for (int r : light) cnt[maxlen - (rp[r + 1] - rp[r]) + 1]++;
  for (size_t i = 1; i < cnt.size(); ++i) cnt[i] += cnt[i - 1];
  const size_t base = items.size();
  items.resize(base + light.size());
  for (int r : light)
    items[base + static_cast<size_t>(cnt[maxlen - (rp[r + 1] - rp[r])]++)] =
        make_int4(static_cast<int>(rp[r]), static_cast<int>(rp[r + 1]), r, 0);
}

// Row-streaming work list (spmm_fast_stream): maximal runs of consecutive light rows cut into pieces of at
// most kPieceRows rows and about piece_nnz nonzeros (a row is never split), plus one piece per hub-row
// segment; ordered by decreasing nonzeros (stable), so the grid's first wave takes the longest pieces.
constexpr int kPieceRows = 32;
std::atomic<int> g_piece_nnz{1024};
void build_stream_pieces(const std::vector<index_t>& rp, const std::vector<int4>& seg_items, std::vector<int4>& pieces) {
  const index_t rows = static_cast<index_t>(rp.size()) - 1;
  const FastCuts cuts = fast_cuts(rp.back());
  const int ht = cuts.ht;
  const index_t cap = std::min<index_t>(g_piece_nnz.load(), cuts.seg);
  pieces.clear();
  for (const int4& it : seg_items) pieces.push_back(make_int4(it.z, 0, it.x, it.y));
  index_t r = 0;
  while (r < rows) {
    if (rp[r + 1] - rp[r] >= ht) {
      ++r;
      continue;
    }
    const index_t r0 = r;
    while (r < rows && r - r0 < kPieceRows && rp[r + 1] - rp[r] < ht && (r == r0 || rp[r + 1] - rp[r0] <= cap)) ++r;
    pieces.push_back(make_int4(static_cast<int>(r0), static_cast<int>(r), static_cast<int>(rp[r0]),
                               static_cast<int>(rp[r])));
  }
  std::stable_sort(pieces.begin(), pieces.end(), [](const int4& a, const int4& b) { return a.w - a.z > b.w - b.z; });
}

// Hub-row half of build_fast_items: segment items + hub descriptors; *n_light = rows below the threshold.
void build_hub_segments(const std::vector<index_t>& rp, std::vector<int4>& items, std::vector<int4>& hubs, int& nseg,
                        index_t& n_light) {
  const index_t rows = static_cast<index_t>(rp.size()) - 1;
  const FastCuts cuts = fast_cuts(rp.back());
  const int ht = cuts.ht, seg = cuts.seg;
  items.clear();
  hubs.clear();
  nseg = 0;
  n_light = 0;
  for (index_t r = 0; r < rows; ++r) {
    const index_t len = rp[r + 1] - rp[r];
    if (len < ht) {
      ++n_light;
      continue;
    }
    const int first = nseg;
    for (index_t e = rp[r]; e < rp[r + 1]; e += seg, ++nseg)
      items.push_back(make_int4(static_cast<int>(e), static_cast<int>(std::min<index_t>(e + seg, rp[r + 1])),
                                -(nseg + 1), 0));
    hubs.push_back(make_int4(static_cast<int>(r), first, nseg - first, 0));
  }
}

// Device blocks released by destroyed groups and by group-creation temporaries stay cached for later
// allocations of the same (rounded) size on the same device: cudaMalloc / cudaFree of GB-sized blocks
// (page mapping; cudaFree synchronises the device) made group creation take 5-70 ms or 0.1-0.7 s from
// run to run. A failed cudaMalloc releases the device's cached blocks and retries.
class BlockCache {
 public:
  static constexpr size_t kCap = size_t(32) << 30;  // cached bytes per device
  static size_t round(size_t bytes) {
    const size_t q = bytes >= (size_t(1) << 20) ? (size_t(1) << 20) : 4096;
    return (std::max<size_t>(bytes, 16) + q - 1) / q * q;
  }
  void* get(int dev, size_t bytes) {  // bytes already rounded; the caller has set the device
    {
      std::lock_guard<std::mutex> lk(mu_);
      auto it = free_.find({dev, bytes});
      if (it != free_.end()) {
        void* p = it->second;
        free_.erase(it);
        cached_[dev] -= bytes;
        return p;
      }
    }
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      (void)cudaGetLastError();
      release(dev);
      MG_CUDA(cudaMalloc(&p, bytes));
    }
    return p;
  }
  std::atomic<bool> enabled{true};  // "block_cache" 0: every block goes back to the driver (cold-start runs)
  void put(int dev, void* p, size_t bytes) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(mu_);
    if (!enabled.load() || cached_[dev] + bytes > kCap) {  // bounded: torch / NCCL need memory too
      cudaFree(p);
      return;
    }
    free_.insert({{dev, bytes}, p});
    cached_[dev] += bytes;
  }
  void release(int dev) {
    std::lock_guard<std::mutex> lk(mu_);
    for (auto it = free_.begin(); it != free_.end();) {
      if (it->first.first == dev) {
        cudaFree(it->second);
        it = free_.erase(it);
      } else {
        ++it;
      }
    }
    cached_[dev] = 0;
  }

 private:
  std::mutex mu_;
  std::multimap<std::pair<int, size_t>, void*> free_;
  std::map<int, size_t> cached_;
};
BlockCache& block_cache() {
  static BlockCache* c = new BlockCache();  // process lifetime
  return *c;
}
int cur_device() {
  int d = 0;
  MG_CUDA(cudaGetDevice(&d));
  return d;
}
// A create-time temporary from the cache (released with tmp_free once its users have completed).
template <class T>
T* tmp_alloc(size_t count, size_t& bytes) {
  bytes = BlockCache::round(sizeof(T) * count);
  return static_cast<T*>(block_cache().get(cur_device(), bytes));
}
inline void tmp_free(void* p, size_t bytes) { block_cache().put(cur_device(), p, bytes); }

// Light-row half on the device: key = ht - length for rows below the threshold (2 ht for the others, which
// sort last), a stable radix sort of (key, row), then {e0, e1, row, 0} items for the first n_light rows.
void light_items_device(const int* rp, index_t rows, int ht, index_t n_light, int4* out) {
  size_t bk = 0, bt = 0;
  int* keys = tmp_alloc<int>(rows, bk);
  int* keys2 = tmp_alloc<int>(rows, bk);
  int* ids = tmp_alloc<int>(rows, bk);
  int* ids2 = tmp_alloc<int>(rows, bk);
  const int blocks = static_cast<int>(std::min<index_t>((rows + 255) / 256, 148 * 16));
  k::light_keys<<<blocks, 256, 0, cudaStreamLegacy>>>(rp, static_cast<int>(rows), ht, keys, ids);
  MG_LAUNCHED();
  cub::DoubleBuffer<int> kb(keys, keys2), vb(ids, ids2);
  int bits = 1;
  while ((1 << bits) <= 2 * ht) ++bits;
  size_t tmp = 0;
  MG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, static_cast<int>(rows), 0, bits, cudaStreamLegacy));
  void* t = tmp_alloc<char>(tmp, bt);
  MG_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, kb, vb, static_cast<int>(rows), 0, bits, cudaStreamLegacy));
  k::light_fill<<<blocks, 256, 0, cudaStreamLegacy>>>(rp, vb.Current(), static_cast<int>(n_light), out);
  MG_LAUNCHED();
  MG_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
  for (void* q : {static_cast<void*>(keys), static_cast<void*>(keys2), static_cast<void*>(ids),
                  static_cast<void*>(ids2)})
    tmp_free(q, bk);
  tmp_free(t, bt);
}

// Host-side construction of the launch lists for a tile (row order by decreasing length).
void build_orders(const std::vector<index_t>& rp, std::vector<int>& light, std::vector<int>& heavy) {
  const index_t rows = static_cast<index_t>(rp.size()) - 1;
  const int ht = heavy_threshold();
  light.clear();
  heavy.clear();
  for (index_t r = 0; r < rows; ++r) ((rp[r + 1] - rp[r]) >= ht ? heavy : light).push_back(static_cast<int>(r));
  auto longer = [&](int a, int b) { return (rp[a + 1] - rp[a]) > (rp[b + 1] - rp[b]); };
  std::stable_sort(light.begin(), light.end(), longer);
  std::stable_sort(heavy.begin(), heavy.end(), longer);
}

}  // namespace

// ---------------------------------------------------------------- kernel launchers (shared with C ABI)
struct SpmmLaunch {
  const int* row_ptr;
  const int2* edges;
  const int* light;
  int n_light;
  const int* heavy;
  int n_heavy;
};

template <int G, int CPL>
static void launch_rows(const SpmmLaunch& t, const float* h, float* out, int ld, int nchunk, int acc, int relu,
                        const k::Epi& ep, cudaStream_t s) {
  if (t.n_light <= 0) return;
  const int gpb = 256 / G;
  const int blocks = std::min(ceil_div(t.n_light, gpb), num_sms() * 16);
  k::spmm_exact_rows<G, CPL><<<blocks, 256, 0, s>>>(t.row_ptr, t.edges, t.light, t.n_light, h, out, ld, nchunk, acc,
                                                    relu, ep);
  MG_LAUNCHED();
}

// Light rows: pick the lane-group size G and chunks-per-lane CPL from the float4 width; widths above
// 1024 floats are processed in column slabs (each slab re-walks the row's nonzeros).
static int spmm_light(const SpmmLaunch& t, const float* h, float* out, index_t ld, int acc, int relu, const k::Epi& ep0,
                      cudaStream_t s) {
  const int nchunk_all = static_cast<int>(ld / 4);
  int launches = 0;
  const int step = slab_chunks();
  for (int c0 = 0; c0 < nchunk_all; c0 += step) {
    const int nchunk = std::min(step, nchunk_all - c0);
    const float* hs = h + 4 * c0;
    float* os = out + 4 * c0;
    const int L = static_cast<int>(ld);
    k::Epi ep = ep0;
    if (ep.bias) ep.bias += 4 * c0;
    ep.key += static_cast<unsigned long long>(4 * c0) * 0x9E3779B97F4A7C15ull;  // column offset of the slab
    if (nchunk <= 1) launch_rows<1, 1>(t, hs, os, L, nchunk, acc, relu, ep, s);
    else if (nchunk <= 2) launch_rows<2, 1>(t, hs, os, L, nchunk, acc, relu, ep, s);
    else if (nchunk <= 4) launch_rows<4, 1>(t, hs, os, L, nchunk, acc, relu, ep, s);
    else if (nchunk <= 8) launch_rows<8, 1>(t, hs, os, L, nchunk, acc, relu, ep, s);
    else if (nchunk <= 16 && narrow_group() == 4 && nchunk <= 12) launch_rows<4, 3>(t, hs, os, L, nchunk, acc, relu, ep, s);
    else if (nchunk <= 16 && narrow_group() == 8) launch_rows<8, 2>(t, hs, os, L, nchunk, acc, relu, ep, s);
    else if (nchunk <= 16) launch_rows<16, 1>(t, hs, os, L, nchunk, acc, relu, ep, s);
    else if (nchunk <= 32) launch_rows<32, 1>(t, hs, os, L, nchunk, acc, relu, ep, s);
    else if (nchunk <= 64) launch_rows<32, 2>(t, hs, os, L, nchunk, acc, relu, ep, s);
    else if (nchunk <= 96) launch_rows<32, 3>(t, hs, os, L, nchunk, acc, relu, ep, s);
    else if (nchunk <= 128) launch_rows<32, 4>(t, hs, os, L, nchunk, acc, relu, ep, s);
    else if (nchunk <= 192) launch_rows<32, 6>(t, hs, os, L, nchunk, acc, relu, ep, s);
    else launch_rows<32, 8>(t, hs, os, L, nchunk, acc, relu, ep, s);
    ++launches;
  }
  return launches;
}

struct FastLaunch {
  const int4* items;
  int n_items;
  const int4* hubs;
  int n_hubs;
  const int2* edges;
  float* scratch;  // n_segments x ld
  bool hubs_classed = false;  // edge records carry hub classes (upload_tile, FAST mode)
  index_t src_rows = 0;       // rows of the gathered block (the tile's columns)
  const int4* pieces = nullptr;  // row-streaming work list (spmm_fast_stream)
  int n_pieces = 0;
  const int* row_ptr = nullptr;
  double nnz_per_row = 0.0;
};

template <int G, int CPL>
static void launch_fast(const FastLaunch& t, const float* h, float* out, float* scratch, int ld, int nchunk, int acc,
                        int relu, const k::Epi& ep, cudaStream_t s) {
  const int gpb = 256 / G;
  const int blocks = std::min(ceil_div(t.n_items, gpb), num_sms() * 16);
  k::spmm_fast_items<G, CPL><<<blocks, 256, 0, s>>>(t.items, t.n_items, t.edges, h, out, scratch, ld, nchunk, acc,
                                                    relu, ep);
  MG_LAUNCHED();
}

std::atomic<int> g_spmm_async{1};  // MG_SPMM_FAST gathers through the cp.async ring (spmm_fast_async)
constexpr double kL2Bytes = 126.0 * (1 << 20);
std::atomic<long long> g_hub_bytes{96ll << 20};  // L2 footprint of evict_last hub rows per gather (0 = no hints)

// Largest hub class whose rows (10000 * 2^(k-1) of them, ld floats each) fit the hub footprint; -1 = no hints.
int hub_class_max(int ld) {
  const long long budget = g_hub_bytes.load();
  if (budget <= 0) return -1;
  int k = 0;
  while (k < 7 && 10000ll * (1ll << k) * ld * 4 <= budget) ++k;
  return k;
}

// Masked softmax-CE over `rows` logits rows of C classes: up to 48 classes a row takes a quarter warp (four
// rows per warp, 3 shuffle rounds per reduction), up to 176 (papers: 172) half a warp, wider rows a warp.
static void launch_softmax_xent(int C, int blocks, cudaStream_t s, float* logits, int ld, int rows, const int* labels,
                                const uint8_t* mask, float inv_denom, double* partials) {
  if (C <= 16) k::softmax_xent<2, 8><<<blocks, 256, 0, s>>>(logits, ld, rows, C, labels, mask, inv_denom, partials);
  else if (C <= 32) k::softmax_xent<4, 8><<<blocks, 256, 0, s>>>(logits, ld, rows, C, labels, mask, inv_denom, partials);
  else if (C <= 48) k::softmax_xent<6, 8><<<blocks, 256, 0, s>>>(logits, ld, rows, C, labels, mask, inv_denom, partials);
  else if (C <= 96) k::softmax_xent<6, 16><<<blocks, 256, 0, s>>>(logits, ld, rows, C, labels, mask, inv_denom, partials);
  else if (C <= 176) k::softmax_xent<11, 16><<<blocks, 256, 0, s>>>(logits, ld, rows, C, labels, mask, inv_denom, partials);
  else if (C <= 192) k::softmax_xent<6><<<blocks, 256, 0, s>>>(logits, ld, rows, C, labels, mask, inv_denom, partials);
  else k::softmax_xent<k::kLossCpl><<<blocks, 256, 0, s>>>(logits, ld, rows, C, labels, mask, inv_denom, partials);
  MG_LAUNCHED();
}

// adam_step's constants (gcn.hpp:61-70): cast to float, bias corrections via std::pow in double.
static k::AdamConsts adam_consts(double lr, double beta1, double beta2, double eps, int t) {
  if (t < 1) throw ValueError("adam_step: step index must be >= 1, got " + std::to_string(t));
  k::AdamConsts c{};
  c.b1 = static_cast<float>(beta1);
  c.b2 = static_cast<float>(beta2);
  c.one_m_b1 = 1.0f - c.b1;
  c.one_m_b2 = 1.0f - c.b2;
  c.lr = static_cast<float>(lr);
  c.eps = static_cast<float>(eps);
  c.corr1 = 1.0f - static_cast<float>(std::pow(beta1, t));
  c.corr2 = 1.0f - static_cast<float>(std::pow(beta2, t));
  return c;
}

template <int G, int CPL, int E, int D, bool HINT>
static void launch_fast_async_v(const FastLaunch& t, const float* h, float* out, float* scratch, int ld, int nchunk,
                                int acc, int relu, int hub_max, const k::Epi& ep, cudaStream_t s) {
  constexpr int kThreads = 128;
  constexpr size_t smem = sizeof(float4) * kThreads * D * E * CPL;
  static std::atomic<unsigned long long> attr{0};
  static std::atomic<int> blocks_per_sm{1};
  if (first_on_device(attr, cur_device())) {
    MG_CUDA(cudaFuncSetAttribute(k::spmm_fast_async<G, CPL, E, D, HINT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    int b = 0;
    MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k::spmm_fast_async<G, CPL, E, D, HINT>, kThreads, smem));
    blocks_per_sm = std::max(1, b);
  }
  const int gpb = kThreads / G;
  const int blocks = std::min(ceil_div(t.n_items, gpb), num_sms() * blocks_per_sm);
  k::spmm_fast_async<G, CPL, E, D, HINT><<<blocks, kThreads, smem, s>>>(t.items, t.n_items, t.edges, h, out, scratch,
                                                                        ld, nchunk, acc, relu, hub_max, ep);
  MG_LAUNCHED();
}

// MG_SPMM_FAST row-streaming kernel (spmm_fast_stream): 0 off, 1 on, 2 auto = tiles averaging fewer than
// kStreamRowNnz nonzeros per row (measured: C4 P = 8 stage tiles, 6.3 per row, 12.8 -> 11.7 ms per rank;
// slower on C2 / C3 / C4 at P = 1, 13.6-490 per row)
std::atomic<int> g_spmm_stream{2};
constexpr double kStreamRowNnz = 10.0;

template <int G, int CPL, int E, int D, bool HINT>
static void launch_fast_stream_v(const FastLaunch& t, const float* h, float* out, float* scratch, int ld, int nchunk,
                                 int acc, int relu, int hub_max, const k::Epi& ep, cudaStream_t s) {
  constexpr int kThreads = 128;
  constexpr size_t smem = sizeof(float4) * kThreads * D * E * CPL;
  static std::atomic<unsigned long long> attr{0};
  static std::atomic<int> blocks_per_sm{1};
  if (first_on_device(attr, cur_device())) {
    MG_CUDA(cudaFuncSetAttribute(k::spmm_fast_stream<G, CPL, E, D, HINT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    int b = 0;
    MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k::spmm_fast_stream<G, CPL, E, D, HINT>, kThreads, smem));
    blocks_per_sm = std::max(1, b);
  }
  const int gpb = kThreads / G;
  const int blocks = std::min(ceil_div(t.n_pieces, gpb), num_sms() * blocks_per_sm);
  k::spmm_fast_stream<G, CPL, E, D, HINT><<<blocks, kThreads, smem, s>>>(t.pieces, t.n_pieces, t.row_ptr, t.edges, h, out,
                                                                         scratch, ld, nchunk, acc, relu, hub_max, ep);
  MG_LAUNCHED();
}

template <int G, int CPL, int E, int D>
static void launch_fast_async(const FastLaunch& t, const float* h, float* out, float* scratch, int ld, int nchunk,
                              int acc, int relu, const k::Epi& ep, cudaStream_t s) {
  // hub hints only when the gathered block is well beyond the L2 (a block of a few L2 sizes is better
  // served by plain LRU, which then keeps a large share of every row resident)
  const bool big = static_cast<double>(t.src_rows) * ld * 4 > 4.0 * kL2Bytes;
  const int hub_max = t.hubs_classed && big ? hub_class_max(ld) : -1;
  const int sm = g_spmm_stream.load();
  if ((sm == 1 || (sm == 2 && t.nnz_per_row < kStreamRowNnz)) && t.pieces && t.n_pieces > 0) {
    if (hub_max >= 0) launch_fast_stream_v<G, CPL, E, D, true>(t, h, out, scratch, ld, nchunk, acc, relu, hub_max, ep, s);
    else launch_fast_stream_v<G, CPL, E, D, false>(t, h, out, scratch, ld, nchunk, acc, relu, -1, ep, s);
    return;
  }
  if (hub_max >= 0) launch_fast_async_v<G, CPL, E, D, true>(t, h, out, scratch, ld, nchunk, acc, relu, hub_max, ep, s);
  else launch_fast_async_v<G, CPL, E, D, false>(t, h, out, scratch, ld, nchunk, acc, relu, -1, ep, s);
}

// cp.async-pipelined variants for rows of >= 32 floats; false = use the register-gather kernel.
static bool launch_fast_pipelined(const FastLaunch& t, const float* hs, float* os, float* ss, int L, int nchunk,
                                  int acc, int relu, const k::Epi& ep, cudaStream_t s) {
  if (!g_spmm_async.load() || nchunk < 8) return false;
  if (nchunk <= 16) launch_fast_async<16, 1, 4, 4>(t, hs, os, ss, L, nchunk, acc, relu, ep, s);
  else if (nchunk <= 32) launch_fast_async<32, 1, 4, 4>(t, hs, os, ss, L, nchunk, acc, relu, ep, s);
  else if (nchunk <= 64) launch_fast_async<32, 2, 4, 4>(t, hs, os, ss, L, nchunk, acc, relu, ep, s);
  else if (nchunk <= 128) launch_fast_async<32, 4, 2, 4>(t, hs, os, ss, L, nchunk, acc, relu, ep, s);
  else return false;
  return true;
}

// MG_SPMM_FAST: one gather pass over rows + hub segments, then the ordered hub-segment sum.
static int spmm_fast(const FastLaunch& t, const float* h, float* out, index_t ld, int acc, int relu, const k::Epi& ep0,
                     cudaStream_t s) {
  int launches = 0;
  const int nchunk_all = static_cast<int>(ld / 4);
  if (t.n_items > 0) {
    const int step = slab_chunks();
    for (int c0 = 0; c0 < nchunk_all; c0 += step) {
      const int nchunk = std::min(step, nchunk_all - c0);
      const float* hs = h + 4 * c0;
      float* os = out + 4 * c0;
      float* ss = t.scratch ? t.scratch + 4 * c0 : nullptr;
      const int L = static_cast<int>(ld);
      k::Epi ep = ep0;
      if (ep.bias) ep.bias += 4 * c0;
      ep.rmax_acc = c0 > 0;  // column slabs: each pass folds its columns into the row maxima
      ep.key += static_cast<unsigned long long>(4 * c0) * 0x9E3779B97F4A7C15ull;  // column offset of the slab
      if (launch_fast_pipelined(t, hs, os, ss, L, nchunk, acc, relu, ep, s)) {
      } else if (nchunk <= 1) launch_fast<1, 1>(t, hs, os, ss, L, nchunk, acc, relu, ep, s);
      else if (nchunk <= 2) launch_fast<2, 1>(t, hs, os, ss, L, nchunk, acc, relu, ep, s);
      else if (nchunk <= 4) launch_fast<4, 1>(t, hs, os, ss, L, nchunk, acc, relu, ep, s);
      else if (nchunk <= 8) launch_fast<8, 1>(t, hs, os, ss, L, nchunk, acc, relu, ep, s);
      else if (nchunk <= 12 && narrow_group() == 4) launch_fast<4, 3>(t, hs, os, ss, L, nchunk, acc, relu, ep, s);
      else if (nchunk <= 16 && narrow_group() == 8) launch_fast<8, 2>(t, hs, os, ss, L, nchunk, acc, relu, ep, s);
      else if (nchunk <= 16) launch_fast<16, 1>(t, hs, os, ss, L, nchunk, acc, relu, ep, s);
      else if (nchunk <= 32) launch_fast<32, 1>(t, hs, os, ss, L, nchunk, acc, relu, ep, s);
      else if (nchunk <= 64) launch_fast<32, 2>(t, hs, os, ss, L, nchunk, acc, relu, ep, s);
      else if (nchunk <= 96) launch_fast<32, 3>(t, hs, os, ss, L, nchunk, acc, relu, ep, s);
      else if (nchunk <= 128) launch_fast<32, 4>(t, hs, os, ss, L, nchunk, acc, relu, ep, s);
      else if (nchunk <= 192) launch_fast<32, 6>(t, hs, os, ss, L, nchunk, acc, relu, ep, s);
      else launch_fast<32, 8>(t, hs, os, ss, L, nchunk, acc, relu, ep, s);
      ++launches;
    }
  }
  if (t.n_hubs > 0) {
    const int th = static_cast<int>(std::max<index_t>(32, std::min<index_t>(256, (ld / 4 + 31) / 32 * 32)));
    k::spmm_fast_hubs<<<t.n_hubs, th, 0, s>>>(t.hubs, t.scratch, out, static_cast<int>(ld), acc, relu, ep0);
    MG_LAUNCHED();
    ++launches;
  }
  return launches;
}

static int spmm_heavy(const SpmmLaunch& t, const float* h, float* out, index_t ld, int acc, int relu, const k::Epi& ep,
                      cudaStream_t s) {
  if (t.n_heavy <= 0) return 0;
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr, cur_device()))
    MG_CUDA(cudaFuncSetAttribute(k::spmm_exact_heavy, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(k::kHeavySmem)));
  const int nslab = ceil_div(ld, k::kHeavySlab);
  k::spmm_exact_heavy<<<t.n_heavy * nslab, k::kHeavyThreads, k::kHeavySmem, s>>>(t.row_ptr, t.edges, t.heavy, nslab, h, out,
                                                                   static_cast<int>(ld), acc, relu, ep);
  MG_LAUNCHED();
  return 1;
}

// GeMM dispatch: exact SIMT or tcgen05 (mg_tc_gemm.cuh).
// mg_dev_gemm only: per-row max |A| pairs {max, 0} (in the training step the producers of A write them)
__global__ void row_absmax_pairs(const float* __restrict__ A, long lda, long M, long K, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (long r = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; r < M;
       r += static_cast<long>(gridDim.x) * blockDim.x / 32) {
    float m = 0.0f;
    for (long k = lane; k < K; k += 32) m = fmaxf(m, fabsf(A[r * lda + k]));
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) *reinterpret_cast<float2*>(out + 2 * r) = make_float2(m, 0.0f);
  }
}

static int gemm_launch(int mode, bool ta, bool tb, index_t M, index_t N, index_t K, const float* A, index_t lda,
                       const float* B, index_t ldb, float* Cm, index_t ldc, int epi, cudaStream_t s,
                       float* ws = nullptr, size_t ws_bytes = 0, const k::Epi& ep = k::Epi{},
                       const float* rmax_in = nullptr) {
  if (M <= 0 || N <= 0) return 0;
  if (mode != MG_GEMM_EXACT)
    return tc::gemm(mode, ta, tb, M, N, K, A, lda, B, ldb, Cm, ldc, epi, ws, ws_bytes, s, ep, rmax_in);
  dim3 grid(ceil_div(M, k::kGBM), ceil_div(N, k::kGBN));
#define MG_G(TA, TB, E) k::gemm_exact<TA, TB, E><<<grid, 256, 0, s>>>((int)M, (int)N, (int)K, A, lda, B, ldb, Cm, ldc, ep)
  if (!ta && !tb) {
    if (epi == 0) MG_G(false, false, 0); else if (epi == 1) MG_G(false, false, 1); else MG_G(false, false, 2);
  } else if (ta && !tb) {
    if (epi == 0) MG_G(true, false, 0); else if (epi == 1) MG_G(true, false, 1); else MG_G(true, false, 2);
  } else if (!ta && tb) {
    if (epi == 0) MG_G(false, true, 0); else if (epi == 1) MG_G(false, true, 1); else MG_G(false, true, 2);
  } else {
    throw ValueError("gemm: transposed A and B together is not on the training path");
  }
#undef MG_G
  MG_LAUNCHED();
  return 1;
}

// ======================================================================== worker
struct Worker {
  int rank = 0, device = 0;
  index_t r0 = 0, rows = 0;
  cudaStream_t s0 = nullptr, s1 = nullptr, s2 = nullptr;  // compute (lane 0), comm (lane 1), heavy-row side
  std::vector<DevTile> tiles[2];
  // stage folding: SpMM steps as [first, last] stage pairs (last == first: one stage), the step of every
  // stage, and the merged tiles of the folded pairs (ftiles[dir][first])
  std::vector<int> step_first, step_last, step_of;
  std::vector<DevTile> ftiles[2];
  float* x = nullptr;
  int* labels = nullptr;
  uint8_t* mask = nullptr;
  std::vector<float*> ahw;
  float *hw = nullptr, *bc1 = nullptr, *bc2 = nullptr;
  float* ax = nullptr;  // Â·X (rows x ld0) when Config::aggregate_first()
  // TF32X3 + FAST: per-row max |y| pairs (k::Epi::rmax) of the GeMM A operands, written by their producers
  // for the scaled fp16 split: slot l < L for ahw[l], L for hw, L + 1 for ax; rows x 2 floats each
  float* rm = nullptr;
  float* rm_slot(int s) const { return rm ? rm + static_cast<size_t>(s) * 2 * std::max<index_t>(rows, 1) : nullptr; }
  std::vector<float*> W, WG, M, V, stage;
  double* partials = nullptr;
  float* seg_scratch = nullptr;  // MG_SPMM_FAST hub-row segment partials (max segments x ld_max)
  float* ws = nullptr;  // tcgen05 TN split-K partials (W-grad), private to this worker's stream
  size_t ws_bytes = 0;
  float* bias_part = nullptr;  // cfg.bias: per-chunk column sums of the bias gradient
  int bias_chunks = 0;
  double* stats = nullptr;
  double* h_stats = nullptr;  // pinned
  int loss_blocks = 0;
  ncclComm_t comm = nullptr;
  // events (reused every step)
  cudaEvent_t prior, heavy_fork, heavy_join, loss_done, stats_done, src_ready, copy_done, ar_ready, ar_done;
  cudaEvent_t join1 = nullptr, join2 = nullptr;  // step graph: s1 / s2 work enqueued before a graph launch
  std::vector<cudaEvent_t> bc_done, mult, wg_done, red_done;
  cudaEvent_t t_start, t_end;
  // timeline recorder (mg_group_set_timeline): timing events on the task's lane stream, base on s0
  std::vector<cudaEvent_t> tl_pool;
  size_t tl_used = 0;
  cudaEvent_t tl_base = nullptr;
  uint64_t last_task[2] = {0, 0};  // last recorded task per lane (WorkerCtx::last, collectives.hpp)
  std::vector<std::pair<void*, size_t>> allocs;  // block cache entries (pointer, rounded bytes)
  index_t bytes = 0;
};

}  // namespace mg

struct mg_group {
  mg::Config cfg;
  int world = 1;
  int transport = MG_TRANSPORT_NCCL;
  mg::index_t n = 0, mask_count = 0;
  std::vector<mg::index_t> bounds;
  mg::index_t wblocks[9] = {};  // canonical W-grad blocks uniform_partition(n, 8), driver.hpp:156
  std::vector<mg::index_t> ld;  // padded widths per dim
  mg::index_t ld_max = 4, max_part = 0;
  int fold = 0;  // stage folding group size (g_stage_fold >= 2, FAST mode, P > 2), 0 = off
  // floats per layer parameter array: W (ld_l x ld_{l+1}) plus, with cfg.bias, the bias row after it; the
  // same layout for W_G, Adam m / v and each canonical staging block, so the W-grad all-reduce, the block
  // sum and Adam cover the bias with no extra launches
  mg::index_t pstride(int l) const { return (ld[l] + (cfg.bias ? 1 : 0)) * ld[l + 1]; }
  std::vector<std::unique_ptr<mg::Worker>> workers;
  bool sealed = false;  // set after construction: allocations afterwards count as step allocations
  mg::index_t step_allocs = 0;
  bool labels_ok = true;
  std::string label_error;
  int kernels_last = 0;
  int64_t kernels_total = 0;  // since the last mg_group_last_profile
  std::vector<cudaEvent_t> prof_pool;
  size_t prof_used = 0;
  std::vector<std::pair<int, int>> prof_pending;  // (kind, index of the start event)
  double last_loss = 0, last_acc = 0;
  bool stats_pending = false;
  // DeviceGroup::abort (collectives.cpp:42-52): a request from any thread, served by the next host wait
  std::atomic<bool> abort_requested{false};
  bool aborted = false;
  std::string abort_reason;
  // timeline (rowgcn::TimelineEvent, collectives.hpp:24-34): one record per task, times resolved on drain
  struct TlRec {
    int worker_k, lane, stage;
    const char* kind;
    const char* op;
    uint64_t task;
    std::vector<uint64_t> deps;
    size_t ev;  // start event index in the worker's pool (end = ev + 1)
  };
  bool tl_on = false;
  uint64_t tl_next = 1;
  std::vector<TlRec> tl;
  std::vector<mg_timeline_event> tl_out;  // last drained events (deps point into tl)
  // The training step captured once as a CUDA graph (one-worker groups, `step_graph` tuning): replayed
  // with cudaGraphLaunch, the Adam launches' step-dependent constants patched per step.
  struct StepGraph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    struct AdamNode {
      cudaGraphNode_t node;
      cudaKernelNodeParams p;
      int size, blocks, run;
      const float* stage;
      float *w, *g, *m, *v;
      mg::k::AdamConsts c;
      void* args[9];
    };
    std::vector<AdamNode> adam;
    int kernels = 0;
    uint64_t epoch = 0;
    bool ax_cached = false;  // captured without layer 0's Â·X SpMM
  } sg;
  int64_t graph_replays = 0, graph_captures = 0;
  uint64_t ax_epoch = 0;  // g_tuning_epoch when Â·X was last computed under "ax_cache" (0: not cached)
};

namespace mg {
namespace {

void* dalloc(mg_group& g, Worker& w, size_t bytes) {
  if (g.sealed) g.step_allocs++;
  MG_CUDA(cudaSetDevice(w.device));
  const size_t rb = BlockCache::round(bytes);
  void* p = block_cache().get(w.device, rb);
  MG_CUDA(cudaMemset(p, 0, std::max<size_t>(bytes, 16)));
  w.allocs.push_back({p, rb});
  w.bytes += static_cast<index_t>(bytes);
  return p;
}

template <class T>
T* dalloc_t(mg_group& g, Worker& w, size_t count) {
  return static_cast<T*>(dalloc(g, w, sizeof(T) * count));
}

// Host -> device uploads go through a process-wide pair of pinned staging buffers: each chunk is produced
// straight into pinned memory by the host threads (packing / narrowing / copying) while the previous
// chunk's DMA is in flight, so no pageable copy and no full-size host temporary is needed. The copies
// run on the legacy default stream, after dalloc's zero-fill (cudaMemset, also the legacy stream), and
// upload() returns only when they are complete.
class Stager {
 public:
  static constexpr size_t kChunk = size_t(128) << 20;
  // fill(dst, first_byte, bytes) writes bytes [first_byte, first_byte + bytes) of the payload into dst
  void upload(void* dev, size_t bytes, const std::function<void(char*, size_t, size_t)>& fill) {
    std::lock_guard<std::mutex> lk(mu_);
    const cudaStream_t s = cudaStreamLegacy;
    init();
    using clk = std::chrono::steady_clock;
    double t_wait = 0, t_fill = 0;
    const auto t0 = clk::now();
    for (size_t off = 0, b = 0; off < bytes; off += kChunk, b ^= 1) {
      const size_t len = std::min(kChunk, bytes - off);
      auto a = clk::now();
      MG_CUDA(cudaEventSynchronize(done_[b]));  // the previous DMA out of this buffer has finished
      auto c = clk::now();
      fill(buf_[b], off, len);
      t_wait += std::chrono::duration<double, std::milli>(c - a).count();
      t_fill += std::chrono::duration<double, std::milli>(clk::now() - c).count();
      MG_CUDA(cudaMemcpyAsync(static_cast<char*>(dev) + off, buf_[b], len, cudaMemcpyHostToDevice, s));
      MG_CUDA(cudaEventRecord(done_[b], s));
    }
    MG_CUDA(cudaStreamSynchronize(s));
    if (std::getenv("MGGCN_TIMING") && bytes > (size_t(16) << 20))
      std::fprintf(stderr, "[mggcn] stage %7.1f MB: total %6.1f ms, fill %6.1f ms, wait %6.1f ms\n", bytes / 1e6,
                   std::chrono::duration<double, std::milli>(clk::now() - t0).count(), t_fill, t_wait);
  }
  template <class T>
  void upload_array(T* dev, const T* src, size_t count) {
    upload(dev, count * sizeof(T), [&](char* dst, size_t off, size_t len) {
      parallel_for(static_cast<index_t>(len), [&](index_t b, index_t e) {
        std::memcpy(dst + b, reinterpret_cast<const char*>(src) + off + b, static_cast<size_t>(e - b));
      }, index_t(1) << 20);
    });
  }

 private:
  void init() {
    if (buf_[0]) return;
    for (int i = 0; i < 2; ++i) {
      MG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&buf_[i]), kChunk));
      MG_CUDA(cudaEventCreateWithFlags(&done_[i], cudaEventDisableTiming));
      MG_CUDA(cudaEventRecord(done_[i], cudaStreamLegacy));
    }
  }
  std::mutex mu_;
  char* buf_[2] = {nullptr, nullptr};
  cudaEvent_t done_[2] = {nullptr, nullptr};
};
Stager& stager() {
  static Stager* s = new Stager();  // process lifetime (pinned memory is released at exit)
  return *s;
}

std::atomic<int> g_bwd_transpose{1};  // P = 1: the backward tile is built on the device ("bwd_transpose")

// A warp per row (hub rows hold up to ~1e5 nonzeros; the lanes stride through the row, coalesced).
// key = column << row_bits | row.
__global__ void transpose_keys(const int* __restrict__ rp, const int2* __restrict__ edges, int rows, long nnz,
                               int row_bits, unsigned long long* __restrict__ keys, unsigned int* __restrict__ vals) {
  (void)nnz;
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    const int e1 = rp[r + 1];
    for (int e = rp[r] + lane; e < e1; e += 32) {
      const int2 rec = edges[e];
      keys[e] = (static_cast<unsigned long long>(rec.x & k::kColMask) << row_bits) | static_cast<unsigned>(r);
      vals[e] = static_cast<unsigned>(rec.y);
    }
  }
}
__global__ void transpose_fill(const unsigned long long* __restrict__ keys, const unsigned int* __restrict__ vals,
                               long nnz, int row_bits, int2* __restrict__ edges, int* __restrict__ cnt) {
  const unsigned long long row_mask = (1ull << row_bits) - 1ull;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < nnz; i += (long)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    edges[i] = make_int2(static_cast<int>(k & row_mask), static_cast<int>(vals[i]));
    atomicAdd(cnt + (k >> row_bits), 1);
  }
}

// P = 1: the backward tile (Â, bwd) is the transpose of the forward tile (Âᵀ) — the same values with
// (row, column) swapped, columns ascending within a row as tile_rows leaves them — so it is built on the
// device from the uploaded forward tile (a radix sort of (column, row) keys, then a count + scan for the
// row pointers) instead of a second 8-bytes-per-nonzero upload. The host tile only provides the shapes.
void transpose_tile_device(const DevTile& f, DevTile& d) {
  const size_t nnz = static_cast<size_t>(d.nnz);
  size_t bk = 0, bv = 0, bc = 0, bt = 0;
  auto* k1 = tmp_alloc<unsigned long long>(nnz, bk);
  auto* k2 = tmp_alloc<unsigned long long>(nnz, bk);
  auto* v1 = tmp_alloc<unsigned int>(nnz, bv);
  auto* v2 = tmp_alloc<unsigned int>(nnz, bv);
  int* cnt = tmp_alloc<int>(static_cast<size_t>(d.rows) + 1, bc);
  const cudaStream_t s = cudaStreamLegacy;
  const int gb = num_sms() * 8;
  int row_bits = 1, col_bits = 1;
  while ((index_t(1) << row_bits) < std::max<index_t>(f.rows, 2)) ++row_bits;
  while ((index_t(1) << col_bits) < std::max<index_t>(f.cols, 2)) ++col_bits;
  transpose_keys<<<gb, 256, 0, s>>>(f.row_ptr, f.edges, static_cast<int>(f.rows), static_cast<long>(nnz), row_bits,
                                    k1, v1);
  MG_LAUNCHED();
  cub::DoubleBuffer<unsigned long long> kb(k1, k2);
  cub::DoubleBuffer<unsigned int> vb(v1, v2);
  size_t tmp = 0;
  MG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kb, vb, nnz, 0, row_bits + col_bits, s));
  void* t = tmp_alloc<char>(tmp, bt);
  MG_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, kb, vb, nnz, 0, row_bits + col_bits, s));
  MG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int) * (d.rows + 1), s));
  transpose_fill<<<gb, 256, 0, s>>>(kb.Current(), vb.Current(), static_cast<long>(nnz), row_bits, d.edges, cnt);
  MG_LAUNCHED();
  size_t stmp = 0;
  MG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, stmp, cnt, d.row_ptr, static_cast<int>(d.rows + 1), s));
  size_t bs = 0;
  void* st = tmp_alloc<char>(stmp, bs);
  MG_CUDA(cub::DeviceScan::ExclusiveSum(st, stmp, cnt, d.row_ptr, static_cast<int>(d.rows + 1), s));
  MG_CUDA(cudaStreamSynchronize(s));
  tmp_free(k1, bk);
  tmp_free(k2, bk);
  tmp_free(v1, bv);
  tmp_free(v2, bv);
  tmp_free(cnt, bc);
  tmp_free(t, bt);
  tmp_free(st, bs);
}

void upload_tile(mg_group& g, Worker& w, const Tile& t, DevTile& d, const DevTile* transpose_of = nullptr) {
  d.rows = t.rows;
  d.cols = t.cols;
  d.nnz = t.nnz();
  if (d.nnz >= (index_t(1) << 31)) throw ValueError("tile has >= 2^31 nonzeros; split the graph over more workers");
  d.row_ptr = dalloc_t<int>(g, w, t.rows + 1);
  d.edges = dalloc_t<int2>(g, w, d.nnz + k::kEdgePad);
  Stager& st = stager();
  if (transpose_of) {
    if (transpose_of->rows != t.cols || transpose_of->cols != t.rows || transpose_of->nnz != d.nnz)
      throw ValueError("upload: the backward tile is not the forward tile's transpose");
    Stopwatch sw0;
    if (d.nnz) transpose_tile_device(*transpose_of, d);
    else MG_CUDA(cudaMemset(d.row_ptr, 0, sizeof(int) * (t.rows + 1)));
    sw0.lap("  transpose");
  } else {
  st.upload(d.row_ptr, sizeof(int) * (t.rows + 1), [&](char* dst, size_t off, size_t len) {
    int* o = reinterpret_cast<int*>(dst);
    const index_t r0 = static_cast<index_t>(off / sizeof(int));
    parallel_for(static_cast<index_t>(len / sizeof(int)), [&](index_t b, index_t e) {
      for (index_t i = b; i < e; ++i) o[i] = static_cast<int>(t.row_ptr[r0 + i]);
    }, index_t(1) << 18);
  });
  }
  Stopwatch sw;
  if (d.nnz && !transpose_of) {  // {col, value bits} records: both arrays go up as they are, the device interleaves them
    size_t bc = 0, bv = 0;
    int* tcol = tmp_alloc<int>(static_cast<size_t>(d.nnz), bc);
    float* tval = tmp_alloc<float>(static_cast<size_t>(d.nnz), bv);
    if (is_pinned_host(t.col.data()) && is_pinned_host(t.val.data())) {  // one DMA each, no staging copy
      MG_CUDA(cudaMemcpyAsync(tcol, t.col.data(), sizeof(int) * d.nnz, cudaMemcpyHostToDevice, cudaStreamLegacy));
      MG_CUDA(cudaMemcpyAsync(tval, t.val.data(), sizeof(float) * d.nnz, cudaMemcpyHostToDevice, cudaStreamLegacy));
    } else {
      st.upload_array(tcol, t.col.data(), static_cast<size_t>(d.nnz));
      st.upload_array(tval, t.val.data(), static_cast<size_t>(d.nnz));
    }
    k::pack_edges<<<num_sms() * 8, 256, 0, cudaStreamLegacy>>>(tcol, tval, d.nnz, d.edges);
    MG_LAUNCHED();
    MG_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
    tmp_free(tcol, bc);
    tmp_free(tval, bv);
  }
  sw.lap("  arrays");
  // FAST mode: tag each record with its column's hub class (top 4 bits), computed on the device from the
  // uploaded records: per-column gather counts, a histogram of the counts, and per-tier count thresholds
  // (class k = gathered at least as often as the 10000 * 2^(k-1)-th most gathered column).
  if (g.cfg.spmm_mode == MG_SPMM_FAST && g_hub_bytes.load() > 0 && d.nnz && t.cols < (index_t(1) << 28)) {
    size_t bc = 0, bh = 0;
    int* cnt = tmp_alloc<int>(static_cast<size_t>(t.cols), bc);
    int* chist = tmp_alloc<int>(static_cast<size_t>(k::kHubCountCap + 1), bh);
    MG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int) * t.cols, cudaStreamLegacy));
    MG_CUDA(cudaMemsetAsync(chist, 0, sizeof(int) * (k::kHubCountCap + 1), cudaStreamLegacy));
    const int gb = num_sms() * 8;
    k::hub_count<<<gb, 256, 0, cudaStreamLegacy>>>(d.edges, d.nnz, cnt);
    k::hub_count_hist<<<gb, 256, 0, cudaStreamLegacy>>>(cnt, t.cols, chist);
    std::vector<int> h(k::kHubCountCap + 1);
    MG_CUDA(cudaMemcpy(h.data(), chist, sizeof(int) * h.size(), cudaMemcpyDeviceToHost));
    k::HubTiers tiers{};
    index_t seen = 0;
    int tier = 0;
    for (int c = k::kHubCountCap; c >= 1 && tier < 7; --c) {  // most gathered first
      seen += h[c];
      while (tier < 7 && seen >= 10000 * (index_t(1) << tier)) tiers.thr[tier++] = c;
    }
    for (; tier < 7; ++tier) tiers.thr[tier] = 1;  // fewer columns than the tier: everything gathered is in
    k::hub_tag<<<gb, 256, 0, cudaStreamLegacy>>>(d.edges, d.nnz, cnt, tiers);
    MG_LAUNCHED();
    MG_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
    tmp_free(cnt, bc);
    tmp_free(chist, bh);
    d.hubs_classed = true;
  }
  sw.lap("  hub class");
  if (g.cfg.spmm_mode == MG_SPMM_FAST) {
    // FAST work lists: hub-row segments on the host (few rows), then the light rows by decreasing length
    // (ties in row order) as a stable device radix sort of (ht - length, row) — the same list
    // build_fast_items makes on the host.
    std::vector<int4> seg_items, hubs;
    index_t n_light = 0;
    build_hub_segments(t.row_ptr, seg_items, hubs, d.n_segments, n_light);
    const size_t n_items = seg_items.size() + static_cast<size_t>(n_light);
    d.items = dalloc_t<int4>(g, w, std::max<size_t>(1, n_items));
    d.hubs = dalloc_t<int4>(g, w, std::max<size_t>(1, hubs.size()));
    d.n_items = static_cast<int>(n_items);
    d.n_hubs = static_cast<int>(hubs.size());
    if (!seg_items.empty())
      MG_CUDA(cudaMemcpy(d.items, seg_items.data(), sizeof(int4) * seg_items.size(), cudaMemcpyHostToDevice));
    if (!hubs.empty()) MG_CUDA(cudaMemcpy(d.hubs, hubs.data(), sizeof(int4) * hubs.size(), cudaMemcpyHostToDevice));
    if (n_light > 0) light_items_device(d.row_ptr, t.rows, fast_cuts(d.nnz).ht, n_light, d.items + seg_items.size());
    // row-streaming pieces only where the stream kernel will run ("spmm_stream", read here at creation)
    std::vector<int4> pieces;
    const int smode = g_spmm_stream.load();
    const double avg_nnz = t.rows ? static_cast<double>(d.nnz) / static_cast<double>(t.rows) : 0.0;
    if (smode == 1 || (smode == 2 && avg_nnz < kStreamRowNnz)) build_stream_pieces(t.row_ptr, seg_items, pieces);
    d.pieces = dalloc_t<int4>(g, w, std::max<size_t>(1, pieces.size()));
    d.n_pieces = static_cast<int>(pieces.size());
    if (!pieces.empty())
      MG_CUDA(cudaMemcpy(d.pieces, pieces.data(), sizeof(int4) * pieces.size(), cudaMemcpyHostToDevice));
    sw.lap("  lists");
    return;
  }
  std::vector<int> light, heavy;
  build_orders(t.row_ptr, light, heavy);
  d.light = dalloc_t<int>(g, w, std::max<size_t>(1, light.size()));
  d.heavy = dalloc_t<int>(g, w, std::max<size_t>(1, heavy.size()));
  d.n_light = static_cast<int>(light.size());
  d.n_heavy = static_cast<int>(heavy.size());
  if (!light.empty()) MG_CUDA(cudaMemcpy(d.light, light.data(), sizeof(int) * light.size(), cudaMemcpyHostToDevice));
  if (!heavy.empty()) MG_CUDA(cudaMemcpy(d.heavy, heavy.data(), sizeof(int) * heavy.size(), cudaMemcpyHostToDevice));
}

// Stage folding: tiles j0..j1 of one row block side by side (row r = tile j0's row r, then tile j0 + 1's with
// its columns shifted by block j0's size, ...): a CSR over the blocks stacked in one receive buffer.
Tile merge_tiles(const std::vector<const Tile*>& t) {
  Tile m;
  const index_t rows = t[0]->rows;
  m.rows = rows;
  std::vector<std::int32_t> shift(t.size(), 0);
  for (size_t q = 0; q < t.size(); ++q) {
    if (q) shift[q] = shift[q - 1] + static_cast<std::int32_t>(t[q - 1]->cols);
    m.cols += t[q]->cols;
  }
  m.row_ptr.assign(rows + 1, 0);
  for (index_t r = 0; r < rows; ++r) {
    index_t len = 0;
    for (const Tile* x : t) len += x->row_ptr[r + 1] - x->row_ptr[r];
    m.row_ptr[r + 1] = m.row_ptr[r] + len;
  }
  m.col.resize(m.row_ptr[rows]);
  m.val.resize(m.row_ptr[rows]);
  parallel_for(rows, [&](index_t s0, index_t e0) {
    for (index_t r = s0; r < e0; ++r) {
      index_t o = m.row_ptr[r];
      for (size_t q = 0; q < t.size(); ++q)
        for (index_t k = t[q]->row_ptr[r]; k < t[q]->row_ptr[r + 1]; ++k, ++o) {
          m.col[o] = t[q]->col[k] + shift[q];
          m.val[o] = t[q]->val[k];
        }
    }
  }, 4096);
  return m;
}

// Copies rows x cols (host, dense) into a device buffer with leading dimension ld (padding = 0).
void upload_padded(float* dst, const float* src, index_t rows, index_t cols, index_t ld) {
  if (cols == ld && rows * cols > 0 && is_pinned_host(src)) {
    MG_CUDA(cudaMemcpyAsync(dst, src, sizeof(float) * rows * cols, cudaMemcpyHostToDevice, cudaStreamLegacy));
    MG_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
    return;
  }
  if (cols == ld && rows * cols > 0) {
    stager().upload_array(dst, src, static_cast<size_t>(rows * cols));
    return;
  }
  if (cols == ld) {
    MG_CUDA(cudaMemcpy(dst, src, sizeof(float) * rows * cols, cudaMemcpyHostToDevice));
    return;
  }
  MG_CUDA(cudaMemcpy2D(dst, sizeof(float) * ld, src, sizeof(float) * cols, sizeof(float) * cols, rows,
                       cudaMemcpyHostToDevice));
}

void download_padded(float* dst, const float* src, index_t rows, index_t cols, index_t ld) {
  if (cols == ld) {
    MG_CUDA(cudaMemcpy(dst, src, sizeof(float) * rows * cols, cudaMemcpyDeviceToHost));
    return;
  }
  MG_CUDA(cudaMemcpy2D(dst, sizeof(float) * cols, src, sizeof(float) * ld, sizeof(float) * cols, rows,
                       cudaMemcpyDeviceToHost));
}

// The bias rows of the 8 canonical staging blocks (stride block_stride from `out`) from the local rows of G.
int bias_grad_blocks(Worker& w, const float* G, index_t ld, const int64_t* begin, const int64_t* len, float* out,
                     index_t block_stride, cudaStream_t s) {
  k::BlockRanges br{};
  for (int b = 0; b < 8; ++b) {
    br.begin[b] = begin[b];
    br.len[b] = len[b];
  }
  if (w.bias_chunks > 0) {
    k::bias_partials<<<dim3(w.bias_chunks, 8), 256, 0, s>>>(G, static_cast<int>(ld), br, w.bias_chunks, w.bias_part);
    MG_LAUNCHED();
  }
  k::bias_reduce<<<std::max(1, static_cast<int>((8 * ld + 255) / 256)), 256, 0, s>>>(
      w.bias_part, br, w.bias_chunks, static_cast<int>(ld), out, block_stride);
  MG_LAUNCHED();
  return w.bias_chunks > 0 ? 2 : 1;
}

cudaEvent_t mk_event(bool timing = false) {
  cudaEvent_t e;
  MG_CUDA(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
  return e;
}

void nccl_settle(mg_group& g);
void check_alive(mg_group& g);

// Test hook ("debug_stall_us"): a kernel that spins for `us` microseconds (a stand-in for a peer that never
// arrives, so the watchdog / abort path can be exercised on one device).
__global__ void stall_kernel(long long ns) {
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 >= ns) break;
    __nanosleep(1000);
  }
}

// "ax_cache": groups whose ranks all live in this process only (a write to one rank's features must not
// let the ranks of a multi-process job disagree on whether the layer-0 broadcasts run)
bool ax_cache_applies(const mg_group& g) {
  return g_ax_cache.load() && g.cfg.aggregate_first() && static_cast<int>(g.workers.size()) == g.world;
}
bool ax_cached(const mg_group& g) { return ax_cache_applies(g) && g.ax_epoch == g_tuning_epoch.load(); }

// ---------------------------------------------------------------- the step (one process, all local workers)
class Step {
 public:
  explicit Step(mg_group& g) : g_(g), cfg_(g.cfg), L_(g.cfg.layers()), P_(g.world) {}
  // training pass (dropout active) of step t, vs an evaluation forward (mg_group_forward / loss_only)
  void set_training(int t) {
    train_ = true;
    t_ = t;
  }

  // The fused output epilogue of layer l on worker w (mg_epi.cuh): its bias row and, for a hidden layer in
  // a training pass, the dropout stream of (seed, step, layer).
  k::Epi out_epi(const Worker& w, int l, bool hidden) const {
    k::Epi e;
    if (cfg_.bias) e.bias = w.W[l] + g_.ld[l] * g_.ld[l + 1];
    if (hidden && train_ && cfg_.dropout > 0.0) {
      e.thr = static_cast<unsigned>(std::min(4294967295.0, std::floor(cfg_.dropout * 4294967296.0)));
      e.scale = static_cast<float>(1.0 / (1.0 - cfg_.dropout));
      e.key = k::mix64(cfg_.seed ^ k::mix64(static_cast<unsigned long long>(t_) * 1024ull + static_cast<unsigned>(l) + 1ull));
    }
    e.row0 = w.r0;
    return e;
  }

  Worker& W(size_t k) { return *g_.workers[k]; }
  size_t nloc() const { return g_.workers.size(); }
  void dev(Worker& w) { MG_CUDA(cudaSetDevice(w.device)); }

  // -------------------------------------------------------------- collectives
  // DeviceGroup::broadcast_bytes (collectives.cpp:110-125) on the comm streams.
  void bcast(int root, size_t count, const std::vector<float*>& bufs) {
    if ((P_ == 1 && !W(0).comm) || g_.transport == MG_TRANSPORT_SOLO) return;
    if (g_.transport == MG_TRANSPORT_NCCL) {
      MG_NCCL(ncclGroupStart());
      for (size_t k = 0; k < nloc(); ++k) {
        Worker& w = W(k);
        dev(w);
        MG_NCCL(ncclBroadcast(bufs[k], bufs[k], count, ncclFloat, root, w.comm, w.s1));
      }
      MG_NCCL(ncclGroupEnd());
      nccl_settle(g_);
      return;
    }
    // in-process: receivers copy from the root's buffer once it is ready; the root's comm stream then
    // waits for every copy so nothing downstream of the broadcast can overwrite the source early.
    size_t rk = 0;
    for (size_t k = 0; k < nloc(); ++k)
      if (W(k).rank == root) rk = k;
    Worker& R = W(rk);
    dev(R);
    MG_CUDA(cudaEventRecord(R.src_ready, R.s1));
    for (size_t k = 0; k < nloc(); ++k) {
      if (k == rk) continue;
      Worker& w = W(k);
      dev(w);
      MG_CUDA(cudaStreamWaitEvent(w.s1, R.src_ready, 0));
      MG_CUDA(cudaMemcpyAsync(bufs[k], bufs[rk], sizeof(float) * count, cudaMemcpyDeviceToDevice, w.s1));
      MG_CUDA(cudaEventRecord(w.copy_done, w.s1));
      dev(R);
      MG_CUDA(cudaStreamWaitEvent(R.s1, w.copy_done, 0));
    }
  }

  // DeviceGroup::all_reduce_sum (collectives.hpp:76-94), no-op at P == 1.
  template <class T>
  void allreduce(size_t count, const std::vector<T*>& bufs) {
    if ((P_ == 1 && !W(0).comm) || count == 0 || g_.transport == MG_TRANSPORT_SOLO) return;
    if (g_.transport == MG_TRANSPORT_NCCL) {
      MG_NCCL(ncclGroupStart());
      for (size_t k = 0; k < nloc(); ++k) {
        Worker& w = W(k);
        dev(w);
        MG_NCCL(ncclAllReduce(bufs[k], bufs[k], count, sizeof(T) == 8 ? ncclDouble : ncclFloat, ncclSum, w.comm, w.s1));
      }
      MG_NCCL(ncclGroupEnd());
      nccl_settle(g_);
      return;
    }
    Worker& R = W(0);
    for (size_t k = 1; k < nloc(); ++k) {
      Worker& w = W(k);
      dev(w);
      MG_CUDA(cudaEventRecord(w.ar_ready, w.s1));
      dev(R);
      MG_CUDA(cudaStreamWaitEvent(R.s1, w.ar_ready, 0));
    }
    dev(R);
    k::PtrList<T> pl{};
    for (size_t k = 0; k < nloc(); ++k) pl.p[W(k).rank] = bufs[k];
    const int blocks = std::min<long>(1024, (static_cast<long>(count) + 255) / 256);
    k::rank_order_allreduce<T><<<blocks, 256, 0, R.s1>>>(pl, P_, static_cast<long>(count));
    MG_LAUNCHED();
    ++g_.kernels_last;
    MG_CUDA(cudaEventRecord(R.ar_done, R.s1));
    for (size_t k = 1; k < nloc(); ++k) {
      Worker& w = W(k);
      dev(w);
      MG_CUDA(cudaStreamWaitEvent(w.s1, R.ar_done, 0));
    }
  }

  // -------------------------------------------------------------- staged SpMM
  // staged_spmm_submit (inc/dist_spmm.hpp:57-103): stage j broadcasts worker j's rows of `src` into
  // bc[j % 2] (or bc1 without overlap) on the comm stream, then every worker multiplies its (me, j)
  // tile on the compute stream, accumulating for j > 0. Event edges:
  //   spmm(j) <- broadcast(j);   broadcast(j) <- spmm(j-2) overlapped / spmm(j-1) otherwise / prior.
  // relu_last fuses the forward ReLU into the final stage's epilogue.
  // rm_slot >= 0: the last stage also writes the output's per-row max pairs into Worker::rm_slot(rm_slot)
  void staged_spmm(int dir, index_t width, const std::vector<float*>& src, const std::vector<float*>& out,
                   bool relu_last, int epi_layer = -1, int rm_slot = -1) {
    const index_t ld = pad4(width);
    const bool ov = cfg_.overlap;
    std::vector<uint64_t> prior_task(nloc());
    std::vector<std::vector<uint64_t>> mult_task(nloc(), std::vector<uint64_t>(P_, 0));
    for (size_t k = 0; k < nloc(); ++k) {
      dev(W(k));
      MG_CUDA(cudaEventRecord(W(k).prior, W(k).s0));
      prior_task[k] = W(k).last_task[0];
    }
    for (int j = 0; j < P_; ++j) {
      std::vector<float*> recv(nloc());
      std::vector<int> tb(nloc(), -1);
      for (size_t k = 0; k < nloc(); ++k) {
        Worker& w = W(k);
        dev(w);
        // the step that consumes stage j and the buffer it reads (steps alternate BC1 / BC2 under overlap);
        // without folding a step is a stage (inc/dist_spmm.hpp:75-88)
        const int sj = w.step_of.empty() ? j : w.step_of[j];
        const int first = w.step_of.empty() ? j : w.step_first[sj];
        cudaEvent_t dep = ov ? (sj >= 2 ? w.mult[sj - 2] : w.prior) : (sj >= 1 ? w.mult[sj - 1] : w.prior);
        MG_CUDA(cudaStreamWaitEvent(w.s1, dep, 0));
        const uint64_t dep_task = ov ? (sj >= 2 ? mult_task[k][sj - 2] : prior_task[k])
                                     : (sj >= 1 ? mult_task[k][sj - 1] : prior_task[k]);
        tb[k] = tl_begin(k, 1, "broadcast", "h_stage", j, {dep_task});
        float* buf = (!ov || sj % 2 == 0) ? w.bc1 : w.bc2;
        buf += (g_.bounds[j] - g_.bounds[first]) * ld;  // block j's place in a folded group (0 if unfolded)
        recv[k] = (w.rank == j) ? src[k] : buf;
      }
      const size_t count = static_cast<size_t>((g_.bounds[j + 1] - g_.bounds[j]) * ld);
      bcast(j, count, recv);
      for (size_t k = 0; k < nloc(); ++k) {
        Worker& w = W(k);
        dev(w);
        const uint64_t bc_task = tl_end(k, tb[k]);
        MG_CUDA(cudaEventRecord(w.bc_done[j], w.s1));
        MG_CUDA(cudaStreamWaitEvent(w.s0, w.bc_done[j], 0));
        const int sj = w.step_of.empty() ? j : w.step_of[j];
        if (!w.step_of.empty() && w.step_last[sj] != j) continue;  // a group's SpMM waits for its last block
        const bool folded = !w.step_of.empty() && w.step_first[sj] != j;
        const int first = folded ? w.step_first[sj] : j;
        const float* hsrc = folded ? ((!ov || sj % 2 == 0) ? w.bc1 : w.bc2) : recv[k];
        const int ts = tl_begin(k, 0, "spmm", "stage", first, {bc_task});
        const DevTile& t = folded ? w.ftiles[dir][first] : w.tiles[dir][j];
        SpmmLaunch sl{t.row_ptr, t.edges, t.light, t.n_light, t.heavy, t.n_heavy};
        const int acc = sj > 0, relu = relu_last && j == P_ - 1;
        // the layer's bias / dropout ride on the final stage's output write
        k::Epi ep = (epi_layer >= 0 && j == P_ - 1) ? out_epi(w, epi_layer, relu_last) : k::Epi{};
        if (j == P_ - 1 && rm_slot >= 0 && cfg_.spmm_mode == MG_SPMM_FAST) ep.rmax = w.rm_slot(rm_slot);
        const int pi = prof_begin(w);
        if (cfg_.spmm_mode == MG_SPMM_FAST) {
          FastLaunch fl{t.items, t.n_items, t.hubs, t.n_hubs, t.edges, w.seg_scratch, t.hubs_classed, t.cols,
                        t.pieces, t.n_pieces, t.row_ptr, t.rows ? static_cast<double>(t.nnz) / t.rows : 0.0};
          g_.kernels_last += spmm_fast(fl, hsrc, out[k], ld, acc, relu, ep, w.s0);
          prof_end(w, pi, 0);
          mult_task[k][sj] = tl_end(k, ts);
          MG_CUDA(cudaEventRecord(w.mult[sj], w.s0));
          continue;
        }
        if (t.n_heavy > 0) {  // hub rows run beside the light rows on the side stream
          MG_CUDA(cudaEventRecord(w.heavy_fork, w.s0));
          MG_CUDA(cudaStreamWaitEvent(w.s2, w.heavy_fork, 0));
          g_.kernels_last += spmm_heavy(sl, hsrc, out[k], ld, acc, relu, ep, w.s2);
          MG_CUDA(cudaEventRecord(w.heavy_join, w.s2));
        }
        g_.kernels_last += spmm_light(sl, hsrc, out[k], ld, acc, relu, ep, w.s0);
        if (t.n_heavy > 0) MG_CUDA(cudaStreamWaitEvent(w.s0, w.heavy_join, 0));
        prof_end(w, pi, 0);
        mult_task[k][sj] = tl_end(k, ts);
        MG_CUDA(cudaEventRecord(w.mult[sj], w.s0));
      }
    }
  }

  // one GeMM task ("gemm", op, layer) on the compute lane, depending on the lane's previous task
  void gemm(size_t k, const char* op, int layer, bool ta, bool tb, index_t M, index_t N, index_t K, const float* A,
            index_t lda, const float* B, index_t ldb, float* Cm, index_t ldc, int epi, const k::Epi& ep = k::Epi{},
            const float* rmax_in = nullptr) {
    Worker& w = W(k);
    const int th = tl_begin(k, 0, "gemm", op, layer, {w.last_task[0]});
    const int pi = prof_begin(w);
    g_.kernels_last += gemm_launch(cfg_.gemm_mode, ta, tb, M, N, K, A, lda, B, ldb, Cm, ldc, epi, w.s0, w.ws, w.ws_bytes,
                                   ep, rmax_in);
    prof_end(w, pi, 1);
    tl_end(k, th);
  }

  // -------------------------------------------------------------- timeline (collectives.hpp:119-140)
  // Every task the reference submits to a lane (WorkerCtx::submit) is bracketed by a timing-event pair
  // on the matching stream: lane 0 = compute stream, lane 1 = comm stream. Returns a handle for tl_end.
  int tl_begin(size_t k, int lane, const char* kind, const char* op, int stage, std::vector<uint64_t> deps) {
    if (!g_.tl_on) return -1;
    Worker& w = W(k);
    if (w.tl_used + 2 > w.tl_pool.size())
      for (int i = 0; i < 256; ++i) w.tl_pool.push_back(mk_event(true));
    const size_t ev = w.tl_used;
    w.tl_used += 2;
    MG_CUDA(cudaEventRecord(w.tl_pool[ev], lane == 0 ? w.s0 : w.s1));
    deps.erase(std::remove(deps.begin(), deps.end(), uint64_t{0}), deps.end());
    g_.tl.push_back({static_cast<int>(k), lane, stage, kind, op, g_.tl_next++, std::move(deps), ev});
    return static_cast<int>(g_.tl.size() - 1);
  }
  uint64_t tl_end(size_t k, int h) {
    if (h < 0) return 0;
    Worker& w = W(k);
    auto& r = g_.tl[static_cast<size_t>(h)];
    MG_CUDA(cudaEventRecord(w.tl_pool[r.ev + 1], r.lane == 0 ? w.s0 : w.s1));
    w.last_task[r.lane] = r.task;
    return r.task;
  }
  uint64_t tl_task(int h) const { return h < 0 ? 0 : g_.tl[static_cast<size_t>(h)].task; }

  // -------------------------------------------------------------- optional per-kernel timing
  // Event pairs on the launching (compute) stream of the first local worker; enabled with
  // mg_set_tuning("profile", 1), summed by mg_group_last_profile. kind 0 = SpMM stage, 1 = GeMM, 2 = other.
  int prof_begin(Worker& w) {
    if (!g_profile.load() || &w != g_.workers[0].get()) return -1;
    if (g_.prof_used + 2 > g_.prof_pool.size()) {
      for (int i = 0; i < 512; ++i) g_.prof_pool.push_back(mk_event(true));
    }
    const int idx = static_cast<int>(g_.prof_used);
    g_.prof_used += 2;
    MG_CUDA(cudaEventRecord(g_.prof_pool[idx], w.s0));
    return idx;
  }
  void prof_end(Worker& w, int idx, int kind) {
    if (idx < 0) return;
    MG_CUDA(cudaEventRecord(g_.prof_pool[idx + 1], w.s0));
    g_.prof_pending.emplace_back(kind, idx);
  }

  // -------------------------------------------------------------- forward (gcn.hpp:238-267)
  void forward() {
    for (int l = 0; l < L_; ++l) {
      const index_t dl = cfg_.dims[l], dl1 = cfg_.dims[l + 1];
      const index_t ldl = g_.ld[l], ldl1 = g_.ld[l + 1];
      const bool swap = cfg_.order_swap && dl < dl1;  // gcn.hpp:145-148
      std::vector<float*> src(nloc()), out(nloc());
      if (l == 0 && cfg_.aggregate_first()) {  // ax = Â·X (d0 wide), ahw[0] = ax·W0 (+ReLU)
        if (!ax_cached(g_)) {
          for (size_t k = 0; k < nloc(); ++k) {
            src[k] = W(k).x;
            out[k] = W(k).ax;
          }
          staged_spmm(0, dl, src, out, false, -1, L_ + 1);
          if (ax_cache_applies(g_)) g_.ax_epoch = g_tuning_epoch.load();
        }
        for (size_t k = 0; k < nloc(); ++k) {
          Worker& w = W(k);
          dev(w);
          k::Epi ep = out_epi(w, 0, L_ > 1);
          if (L_ > 1) ep.rmax = w.rm_slot(0);  // ahw[0] is the next NN's A
          gemm(k, "hw", 0, false, false, w.rows, ldl1, dl, w.ax, ldl, w.W[0], ldl1, w.ahw[0], ldl1, L_ > 1 ? 2 : 0,
               ep, w.rm_slot(L_ + 1));
        }
        continue;
      }
      // ahw[l-1]'s row maxima exist when its producer wrote them: a FAST SpMM (l - 1 > 0 or no aggregation)
      // or the aggregated layer 0's NN GeMM
      const bool rm_in = l > 0 && !(cfg_.order_swap && cfg_.dims[l - 1] < cfg_.dims[l]);
      for (size_t k = 0; k < nloc(); ++k) {
        Worker& w = W(k);
        dev(w);
        const float* h_in = l == 0 ? w.x : w.ahw[l - 1];
        if (!swap) {
          gemm(k, "hw", l, false, false, w.rows, ldl1, dl, h_in, ldl, w.W[l], ldl1, w.hw, ldl1, 0, k::Epi{},
               rm_in ? w.rm_slot(l - 1) : nullptr);
          src[k] = w.hw;
        } else {
          src[k] = const_cast<float*>(h_in);
        }
        out[k] = swap ? w.hw : w.ahw[l];
      }
      staged_spmm(0, swap ? dl : dl1, src, out, !swap && l < L_ - 1, swap ? -1 : l, (!swap && l < L_ - 1) ? l : -1);
      if (swap) {
        for (size_t k = 0; k < nloc(); ++k) {
          Worker& w = W(k);
          dev(w);
          gemm(k, "hw", l, false, false, w.rows, ldl1, dl, w.hw, ldl, w.W[l], ldl1, w.ahw[l], ldl1, l < L_ - 1 ? 2 : 0,
               out_epi(w, l, l < L_ - 1));
        }
      }
    }
  }

  // -------------------------------------------------------------- loss (gcn.hpp:271-290)
  void loss_grad() {
    const index_t C = cfg_.dims[L_];
    const float inv_denom = 1.0f / static_cast<float>(g_.mask_count);
    std::vector<double*> st(nloc());
    std::vector<int> tr(nloc(), -1);
    for (size_t k = 0; k < nloc(); ++k) {
      Worker& w = W(k);
      dev(w);
      const int th = tl_begin(k, 0, "other", "loss", -1, {w.last_task[0]});
      const int pi = prof_begin(w);
      if (w.rows > 0) {
        launch_softmax_xent(static_cast<int>(C), w.loss_blocks, w.s0, w.ahw[L_ - 1], static_cast<int>(g_.ld[L_]),
                            static_cast<int>(w.rows), w.labels, w.mask, inv_denom, w.partials);
        ++g_.kernels_last;
      }
      k::finalize_stats<<<1, 32, 0, w.s0>>>(w.partials, w.rows > 0 ? w.loss_blocks : 0, w.stats);
      MG_LAUNCHED();
      ++g_.kernels_last;
      prof_end(w, pi, 2);
      const uint64_t loss_task = tl_end(k, th);
      MG_CUDA(cudaEventRecord(w.loss_done, w.s0));
      MG_CUDA(cudaStreamWaitEvent(w.s1, w.loss_done, 0));
      tr[k] = tl_begin(k, 1, "reduce", "loss", -1, {loss_task});
      st[k] = w.stats;
    }
    allreduce<double>(2, st);
    for (size_t k = 0; k < nloc(); ++k) {
      Worker& w = W(k);
      dev(w);
      MG_CUDA(cudaMemcpyAsync(w.h_stats, w.stats, 2 * sizeof(double), cudaMemcpyDeviceToHost, w.s1));
      tl_end(k, tr[k]);
      MG_CUDA(cudaEventRecord(w.stats_done, w.s1));
    }
  }

  // -------------------------------------------------------------- backward (gcn.hpp:292-350)
  void backward() {
    for (int l = L_ - 1; l >= 0; --l) {
      const index_t dl = cfg_.dims[l], dl1 = cfg_.dims[l + 1];
      const index_t ldl = g_.ld[l], ldl1 = g_.ld[l + 1];
      const bool agg = l == 0 && cfg_.aggregate_first();  // W0 grad = (Â·X)^T G0, no backward SpMM
      const bool skip = l == 0 && (cfg_.skip_first_backward_spmm || agg);
      std::vector<float*> grad_rows(nloc());
      if (!skip) {
        std::vector<float*> src(nloc()), out(nloc());
        for (size_t k = 0; k < nloc(); ++k) {
          src[k] = W(k).ahw[l];
          out[k] = W(k).hw;
        }
        staged_spmm(1, dl1, src, out, false, -1, L_);  // hw's row maxima: the H-grad NT's A
        grad_rows = out;
      } else {
        for (size_t k = 0; k < nloc(); ++k) grad_rows[k] = W(k).ahw[l];
      }
      // W_G staging over the 8 canonical row blocks (gcn.hpp:309-331), then one all-reduce.
      std::vector<float*> stg(nloc());
      std::vector<int> trd(nloc(), -1);
      const index_t bs = g_.pstride(l);
      for (size_t k = 0; k < nloc(); ++k) {
        Worker& w = W(k);
        dev(w);
        const float* h_in = l == 0 ? (agg ? w.ax : w.x) : w.ahw[l - 1];
        const int tw = tl_begin(k, 0, "gemm", "wgrad", l, {w.last_task[0]});
        if (cfg_.gemm_mode != MG_GEMM_EXACT) {  // one tcgen05 launch for all 8 blocks (+ ordered reduction)
          int64_t begin[8], len[8];
          for (int b = 0; b < 8; ++b) {
            const index_t a = std::max(g_.wblocks[b], w.r0), e = std::min(g_.wblocks[b + 1], w.r0 + w.rows);
            begin[b] = std::max<index_t>(0, a - w.r0);
            len[b] = std::max<index_t>(0, e - a);
          }
          const int pi = prof_begin(w);
          g_.kernels_last += tc::gemm_tn_blocks(cfg_.gemm_mode, 8, begin, len, ldl, ldl1, h_in, ldl, grad_rows[k], ldl1,
                                                w.stage[l], ldl1, bs, w.ws, w.ws_bytes, w.s0);
          prof_end(w, pi, 1);
        } else {
          for (int b = 0; b < 8; ++b) {
            const index_t a = std::max(g_.wblocks[b], w.r0), e = std::min(g_.wblocks[b + 1], w.r0 + w.rows);
            float* dst = w.stage[l] + b * bs;
            if (a >= e) {
              MG_CUDA(cudaMemsetAsync(dst, 0, sizeof(float) * bs, w.s0));
              continue;
            }
            const int pi = prof_begin(w);
            g_.kernels_last += gemm_launch(cfg_.gemm_mode, true, false, ldl, ldl1, e - a, h_in + (a - w.r0) * ldl, ldl,
                                           grad_rows[k] + (a - w.r0) * ldl1, ldl1, dst, ldl1, 0, w.s0, w.ws, w.ws_bytes);
            prof_end(w, pi, 1);
          }
        }
        if (cfg_.bias) {  // the bias row of every canonical block: column sums of dL/dz_l = ahw[l]
          int64_t begin[8], len[8];
          for (int b = 0; b < 8; ++b) {
            const index_t a = std::max(g_.wblocks[b], w.r0), e = std::min(g_.wblocks[b + 1], w.r0 + w.rows);
            begin[b] = std::max<index_t>(0, a - w.r0);
            len[b] = std::max<index_t>(0, e - a);
          }
          g_.kernels_last += bias_grad_blocks(w, w.ahw[l], ldl1, begin, len, w.stage[l] + ldl * ldl1, bs, w.s0);
        }
        const uint64_t wg_task = tl_end(k, tw);
        MG_CUDA(cudaEventRecord(w.wg_done[l], w.s0));
        MG_CUDA(cudaStreamWaitEvent(w.s1, w.wg_done[l], 0));
        trd[k] = tl_begin(k, 1, "reduce", "wgrad", l, {wg_task});
        stg[k] = w.stage[l];
      }
      allreduce<float>(static_cast<size_t>(8 * bs), stg);
      for (size_t k = 0; k < nloc(); ++k) {
        Worker& w = W(k);
        dev(w);
        red_task_[k].push_back(tl_end(k, trd[k]));
        MG_CUDA(cudaEventRecord(w.red_done[l], w.s1));
      }
      if (l > 0) {  // H_G = HW_G W^T fused with relu_backward into ahw[l-1] (gcn.hpp:337-348)
        for (size_t k = 0; k < nloc(); ++k) {
          Worker& w = W(k);
          dev(w);
          gemm(k, "hgrad", l, false, true, w.rows, ldl, dl1, grad_rows[k], ldl1, w.W[l], ldl1, w.ahw[l - 1], ldl, 1,
               out_epi(w, l - 1, true), skip ? nullptr : w.rm_slot(L_));
        }
      }
      (void)dl;
    }
  }

  // -------------------------------------------------------------- finalize (gcn.hpp:354-377 + adam :61-85)
  void finalize(bool adam, int t) {
    const k::AdamConsts c = adam ? adam_consts(cfg_.lr, cfg_.beta1, cfg_.beta2, cfg_.epsilon, t) : k::AdamConsts{};
    for (size_t k = 0; k < nloc(); ++k) {
      Worker& w = W(k);
      dev(w);
      for (int l = 0; l < L_; ++l) MG_CUDA(cudaStreamWaitEvent(w.s0, w.red_done[l], 0));
      std::vector<uint64_t> deps = red_task_[k];
      deps.push_back(w.last_task[0]);
      const int th = tl_begin(k, 0, "other", adam ? "adam" : "wgrad_final", -1, std::move(deps));
      const int pi = prof_begin(w);
      for (int l = 0; l < L_; ++l) {
        const int size = static_cast<int>(g_.pstride(l));
        k::finalize_adam<<<std::min(1024, (size + 255) / 256), 256, 0, w.s0>>>(size, 8, w.stage[l], w.W[l], w.WG[l],
                                                                              w.M[l], w.V[l], adam ? 1 : 0, c);
        MG_LAUNCHED();
        ++g_.kernels_last;
      }
      prof_end(w, pi, 2);
      tl_end(k, th);
    }
  }

  void begin() {
    g_.kernels_last = 0;
    check_alive(g_);
    if (!g_.labels_ok) throw ValueError(g_.label_error);
    if (const long long us = g_debug_stall_us.load()) {
      dev(W(0));
      stall_kernel<<<1, 1, 0, W(0).s0>>>(us * 1000);
      MG_LAUNCHED();
    }
    for (size_t k = 0; k < nloc(); ++k) {
      Worker& w = W(k);
      dev(w);
      // the previous step's stats read-back (comm stream) must finish before the stats are rewritten
      MG_CUDA(cudaStreamWaitEvent(w.s0, w.stats_done, 0));
      MG_CUDA(cudaEventRecord(w.t_start, w.s0));
    }
  }

  void end() {
    for (size_t k = 0; k < nloc(); ++k) {
      Worker& w = W(k);
      dev(w);
      MG_CUDA(cudaEventRecord(w.t_end, w.s0));
    }
    g_.kernels_total += g_.kernels_last;
  }

 private:
  mg_group& g_;
  const Config& cfg_;
  int L_, P_;
  std::vector<std::vector<uint64_t>> red_task_ = std::vector<std::vector<uint64_t>>(g_.workers.size());
  bool train_ = false;
  int t_ = 1;
};

// ---------------------------------------------------------------- failure handling
// Every host wait polls instead of blocking: it serves mg_group_abort requests, surfaces asynchronous NCCL
// errors (a peer that died or never arrived) and enforces the "watchdog_ms" timeout. Any of them aborts
// the group — ncclCommAbort on its communicators, which releases the device from a collective waiting
// for a lost peer — and raises ShutdownError, like DeviceGroup::abort (collectives.cpp:33-52) wakes every
// waiter with ShutdownError. An aborted group refuses further work.
[[noreturn]] void abort_group(mg_group& g, const std::string& why) {
  if (!g.aborted) {
    g.aborted = true;
    g.abort_reason = why;
    for (auto& wp : g.workers)
      if (wp->comm) {
        cudaSetDevice(wp->device);
        ncclCommAbort(wp->comm);
        wp->comm = nullptr;
      }
  }
  throw ShutdownError("device group aborted: " + g.abort_reason);
}

void check_alive(mg_group& g) {
  if (g.aborted) throw ShutdownError("device group aborted: " + g.abort_reason);
  if (g.abort_requested.load()) abort_group(g, "abort requested");
}

// Polls done() until it returns cudaSuccess; cudaErrorNotReady keeps waiting, anything else throws.
template <class Query>
void wait_for(mg_group& g, Query done, const char* what) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  const long long limit = g_watchdog_ms.load();
  for (int spin = 0;; ++spin) {
    const cudaError_t e = done();
    if (e == cudaSuccess) return;
    if (e != cudaErrorNotReady) {
      (void)cudaGetLastError();
      throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
    }
    check_alive(g);
    for (auto& wp : g.workers)
      if (wp->comm) {
        ncclResult_t st = ncclSuccess;
        ncclCommGetAsyncError(wp->comm, &st);
        if (st != ncclSuccess && st != ncclInProgress)
          abort_group(g, std::string("NCCL error on rank ") + std::to_string(wp->rank) + ": " + ncclGetErrorString(st));
      }
    if (limit > 0 && std::chrono::duration<double, std::milli>(clk::now() - t0).count() > static_cast<double>(limit))
      abort_group(g, std::string(what) + " did not complete within watchdog_ms=" + std::to_string(limit));
    if (spin < 256) std::this_thread::yield();
    else std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

// Completes non-blocking NCCL calls (init, grouped collectives) on every local communicator.
void nccl_settle(mg_group& g) {
  for (auto& wp : g.workers) {
    if (!wp->comm) continue;
    ncclComm_t c = wp->comm;
    wait_for(g, [c] {
      ncclResult_t st = ncclSuccess;
      ncclCommGetAsyncError(c, &st);
      if (st == ncclInProgress) return cudaErrorNotReady;
      if (st != ncclSuccess) throw NcclError(std::string("NCCL: ") + ncclGetErrorString(st));
      return cudaSuccess;
    }, "NCCL call");
  }
}

void sync_all(mg_group& g) {
  check_alive(g);
  for (auto& wp : g.workers) {
    MG_CUDA(cudaSetDevice(wp->device));
    for (cudaStream_t s : {wp->s0, wp->s1, wp->s2}) wait_for(g, [s] { return cudaStreamQuery(s); }, "stream");
  }
}

void read_stats(mg_group& g) {
  Worker& w = *g.workers[0];
  MG_CUDA(cudaSetDevice(w.device));
  cudaEvent_t e = w.stats_done;
  wait_for(g, [e] { return cudaEventQuery(e); }, "step statistics");
  g.last_loss = w.h_stats[0] / static_cast<double>(g.mask_count);
  g.last_acc = w.h_stats[1] / static_cast<double>(g.mask_count);
}

// ---------------------------------------------------------------- the step as a CUDA graph
// One-worker groups (no collectives) replay a captured graph of the whole step: at small sizes (C1, C2) the
// step is ~30 launches of a few microseconds each, and the graph removes the per-launch host cost and
// the inter-kernel launch gaps. The step's schedule depends only on the group and the tuning (captured
// again after any mg_set_tuning); what changes from step to step — Adam's bias corrections — is
// patched into the captured finalize_adam nodes. Not used with the timeline, the profiler (their events
// are per step), dropout (its key depends on t), the stall hook or the GeMM debug environment.
bool step_graph_ok(const mg_group& g) {
  static const bool debug_env = std::getenv("MGGCN_TC_TRACE") || std::getenv("MGGCN_TC_DEBUG");
  return g_step_graph.load() && !debug_env && g.workers.size() == 1 && g.world == 1 && !g.workers[0]->comm &&
         !g.tl_on && !g_profile.load() && !g_debug_stall_us.load() && !(g.cfg.dropout > 0.0);
}

void set_adam_nodes(mg_group& g, int t) {
  const Config& c = g.cfg;
  const k::AdamConsts ac = adam_consts(c.lr, c.beta1, c.beta2, c.epsilon, t);
  for (auto& a : g.sg.adam) {
    a.c = ac;
    MG_CUDA(cudaGraphExecKernelNodeSetParams(g.sg.exec, a.node, &a.p));
  }
}

// Events recorded inside a stream capture can only be waited on inside it: record each once outside, so
// the stream path (and the host waits) can use them again.
void release_captured_events(Worker& w) {
  for (cudaEvent_t e : {w.prior, w.heavy_fork, w.heavy_join, w.loss_done, w.stats_done, w.src_ready, w.copy_done,
                        w.ar_ready, w.ar_done, w.join1, w.join2})
    cudaEventRecord(e, w.s0);
  for (auto* vec : {&w.bc_done, &w.mult, &w.wg_done, &w.red_done})
    for (cudaEvent_t e : *vec) cudaEventRecord(e, w.s0);
  MG_LAUNCHED();
}

void capture_step(mg_group& g, Step& st) {
  Worker& w = *g.workers[0];
  if (g.sg.exec) MG_CUDA(cudaGraphExecDestroy(g.sg.exec));
  if (g.sg.graph) MG_CUDA(cudaGraphDestroy(g.sg.graph));
  g.sg = mg_group::StepGraph{};
  g.kernels_last = 0;
  MG_CUDA(cudaStreamBeginCapture(w.s0, cudaStreamCaptureModeRelaxed));
  cudaGraph_t graph = nullptr;
  try {
    st.forward();
    st.loss_grad();
    st.backward();
    st.finalize(true, 1);
    // every forked stream joins s0 before the capture ends
    cudaStreamCaptureStatus cs;
    for (auto [s, e] : {std::pair{w.s1, w.join1}, std::pair{w.s2, w.join2}}) {
      MG_CUDA(cudaStreamIsCapturing(s, &cs));
      if (cs != cudaStreamCaptureStatusActive) continue;
      MG_CUDA(cudaEventRecord(e, s));
      MG_CUDA(cudaStreamWaitEvent(w.s0, e, 0));
    }
  } catch (...) {
    cudaStreamEndCapture(w.s0, &graph);
    if (graph) cudaGraphDestroy(graph);
    (void)cudaGetLastError();
    release_captured_events(w);
    throw;
  }
  MG_CUDA(cudaStreamEndCapture(w.s0, &graph));
  g.sg.graph = graph;
  release_captured_events(w);
  MG_CUDA(cudaGraphInstantiate(&g.sg.exec, graph, 0));
  g.sg.kernels = g.kernels_last;
  g.sg.epoch = g_tuning_epoch.load();
  g.sg.ax_cached = ax_cached(g);
  g.graph_captures++;
  size_t n = 0;
  MG_CUDA(cudaGraphGetNodes(graph, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  MG_CUDA(cudaGraphGetNodes(graph, nodes.data(), &n));
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType ty;
    MG_CUDA(cudaGraphNodeGetType(nd, &ty));
    if (ty != cudaGraphNodeTypeKernel) continue;
    cudaKernelNodeParams kp{};
    MG_CUDA(cudaGraphKernelNodeGetParams(nd, &kp));
    if (kp.func != reinterpret_cast<void*>(k::finalize_adam)) continue;
    g.sg.adam.emplace_back();
    auto& a = g.sg.adam.back();
    a.node = nd;
    a.p = kp;
    void** v = kp.kernelParams;
    a.size = *static_cast<int*>(v[0]);
    a.blocks = *static_cast<int*>(v[1]);
    a.stage = *static_cast<const float**>(v[2]);
    a.w = *static_cast<float**>(v[3]);
    a.g = *static_cast<float**>(v[4]);
    a.m = *static_cast<float**>(v[5]);
    a.v = *static_cast<float**>(v[6]);
    a.run = *static_cast<int*>(v[7]);
    a.c = *static_cast<k::AdamConsts*>(v[8]);
  }
  // argument storage lives in the vector's final elements
  for (auto& a : g.sg.adam) {
    void* args[9] = {&a.size, &a.blocks, &a.stage, &a.w, &a.g, &a.m, &a.v, &a.run, &a.c};
    std::copy(args, args + 9, a.args);
    a.p.kernelParams = a.args;
    a.p.extra = nullptr;
  }
  if (static_cast<int>(g.sg.adam.size()) != g.cfg.layers())
    throw CudaError("step graph: expected one Adam launch per layer, captured " + std::to_string(g.sg.adam.size()));
}

void enqueue_train_graph(mg_group& g, int t) {
  Worker& w = *g.workers[0];
  MG_CUDA(cudaSetDevice(w.device));
  check_alive(g);
  if (!g.labels_ok) throw ValueError(g.label_error);
  if (!g.sg.exec || g.sg.epoch != g_tuning_epoch.load() || g.sg.ax_cached != ax_cached(g)) {
    Step st(g);
    st.set_training(t);
    capture_step(g, st);
  }
  set_adam_nodes(g, t);
  // the graph runs on s0 after everything enqueued before on s0 / s1 / s2 (the previous step's stats
  // read-back included), and later s1 / s2 work runs after it
  MG_CUDA(cudaEventRecord(w.join1, w.s1));
  MG_CUDA(cudaEventRecord(w.join2, w.s2));
  MG_CUDA(cudaStreamWaitEvent(w.s0, w.join1, 0));
  MG_CUDA(cudaStreamWaitEvent(w.s0, w.join2, 0));
  MG_CUDA(cudaStreamWaitEvent(w.s0, w.stats_done, 0));
  MG_CUDA(cudaEventRecord(w.t_start, w.s0));
  MG_CUDA(cudaGraphLaunch(g.sg.exec, w.s0));
  MG_CUDA(cudaEventRecord(w.stats_done, w.s0));
  MG_CUDA(cudaEventRecord(w.t_end, w.s0));
  MG_CUDA(cudaStreamWaitEvent(w.s1, w.t_end, 0));
  MG_CUDA(cudaStreamWaitEvent(w.s2, w.t_end, 0));
  g.kernels_last = g.sg.kernels;
  g.kernels_total += g.sg.kernels;
  g.graph_replays++;
  g.stats_pending = true;
}

}  // namespace
}  // namespace mg

using namespace mg;

// ======================================================================== C ABI (device half)
extern "C" {

mg_status mg_set_tuning(const char* key, int64_t value) {
  return guarded([&] {
    const std::string k = key ? key : "";
    g_tuning_epoch.fetch_add(1);
    if (k == "heavy_row") {
      if (value < 1) throw ValueError("tuning: heavy_row must be >= 1");
      g_heavy_row = static_cast<int>(std::min<int64_t>(value, 1 << 30));
    } else if (k == "watchdog_ms") {
      if (value < 0) throw ValueError("tuning: watchdog_ms must be >= 0 (0 = no timeout)");
      g_watchdog_ms = value;
    } else if (k == "debug_stall_us") {
      if (value < 0) throw ValueError("tuning: debug_stall_us must be >= 0");
      g_debug_stall_us = value;
    } else if (k == "nccl_single") {
      g_nccl_single = value != 0 ? 1 : 0;
    } else if (k == "profile") {
      g_profile = value != 0 ? 1 : 0;
    } else if (k == "step_graph") {
      g_step_graph = value != 0 ? 1 : 0;
    } else if (k == "ax_cache") {
      g_ax_cache = value != 0 ? 1 : 0;
    } else if (k == "spmm_narrow_group") {
      if (value != 0 && value != 4 && value != 8) throw ValueError("tuning: spmm_narrow_group must be 0, 4 or 8");
      g_narrow_group = static_cast<int>(value);
    } else if (k == "spmm_slab") {
      if (value < 0 || value % 4) throw ValueError("tuning: spmm_slab must be 0 or a multiple of 4 floats");
      g_spmm_slab = static_cast<int>(std::min<int64_t>(value, 1024));
    } else if (k == "spmm_hub_bytes") {
      if (value < 0) throw ValueError("tuning: spmm_hub_bytes must be >= 0");
      g_hub_bytes = value;
    } else if (k == "block_cache") {
      block_cache().enabled = value != 0;
      if (!value)
        for (int d = 0; d < 64 && d < mg_device_count(); ++d) block_cache().release(d);
    } else if (k == "bwd_transpose") {
      g_bwd_transpose = value != 0 ? 1 : 0;
    } else if (k == "adaptive_cuts") {
      g_adaptive_cuts = value != 0 ? 1 : 0;
    } else if (k == "spmm_stream") {
      if (value < 0 || value > 2) throw ValueError("tuning: spmm_stream must be 0 (off), 1 (on) or 2 (auto)");
      g_spmm_stream = static_cast<int>(value);
    } else if (k == "piece_nnz") {
      if (value < 1) throw ValueError("tuning: piece_nnz must be >= 1");
      g_piece_nnz = static_cast<int>(std::min<int64_t>(value, 1 << 30));
    } else if (k == "spmm_async") {
      g_spmm_async = value != 0 ? 1 : 0;
    } else if (k == "fast_segment") {
      if (value < 32) throw ValueError("tuning: fast_segment must be >= 32");
      g_fast_segment = static_cast<int>(std::min<int64_t>(value, 1 << 24));
    } else if (k == "tn_chunk") {
      tc::set_tn_chunk(static_cast<int>(value));
    } else if (k == "gemm3_cluster") {
      tc::set_gemm3_cluster(static_cast<int>(value));
    } else if (k == "gemm3_epi") {
      tc::set_epi_chunks3(static_cast<int>(value));
    } else if (k == "gemm3_wring") {
      tc::set_w3_bytes(static_cast<int>(value));
    } else if (k == "l2_persist_mb") {  // L2 set-aside for persisting (evict_last) lines on the current device
      if (value < 0) throw ValueError("tuning: l2_persist_mb must be >= 0");
      int dev = 0, maxp = 0;
      MG_CUDA(cudaGetDevice(&dev));
      MG_CUDA(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev));
      MG_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize,
                                 std::min<size_t>(static_cast<size_t>(value) << 20, static_cast<size_t>(maxp))));
    } else if (k == "stage_fold") {
      if (value < 0 || value > 64) throw ValueError("tuning: stage_fold must be 0 (off) or a group size 2..64");
      g_stage_fold = static_cast<int>(value);
    } else if (k == "gemm_f16_min_k") {
      tc::set_gemm_f16_min_k(static_cast<int>(value));
    } else if (k == "gemm_f16") {
      tc::set_gemm_f16(static_cast<int>(value));
    } else if (k == "gemm_kernel") {
      tc::set_gemm_version(static_cast<int>(value));
    } else {
      throw ValueError("tuning: unknown key '" + k + "'");
    }
  });
}

int32_t mg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();  // clear the sticky "no device" status
    return 0;
  }
  return n;
}

mg_status mg_nccl_unique_id(uint8_t id[128]) {
  return guarded([&] {
    ncclUniqueId u;
    MG_NCCL(ncclGetUniqueId(&u));
    static_assert(sizeof(u) == 128, "ncclUniqueId size");
    std::memcpy(id, &u, 128);
  });
}

mg_status mg_group_create(const mg_config* cfgp, const mg_partition* p, int32_t world, int32_t n_local,
                          const int32_t* local_ranks, const int32_t* devices, const uint8_t* nccl_id,
                          int32_t transport, mg_group** out) {
  return guarded([&] {
    if (!p || !out || n_local < 1 || !local_ranks || !devices) throw ValueError("group: bad arguments");
    // a failure part-way releases what was built (streams, events, device blocks, communicators)
    std::unique_ptr<mg_group, void (*)(mg_group*)> g(new mg_group(), mg_group_destroy);
    g->cfg = to_config(cfgp);
    const Config& cfg = g->cfg;
    if (cfg.dims.front() != p->d0)
      throw ConfigError("config: layer_dims[0]=" + std::to_string(cfg.dims.front()) +
                        " but dataset features have width " + std::to_string(p->d0));
    if (world != p->parts)
      throw ValueError("group: world " + std::to_string(world) + " but the partition has P=" +
                       std::to_string(p->parts));
    if (cfg.dims.back() > 32 * k::kLossCpl)
      throw ValueError("loss: more than " + std::to_string(32 * k::kLossCpl) + " classes is not supported");
    if (cfg.gemm_mode != MG_GEMM_EXACT && !tc::available())
      throw ValueError("gemm_mode " + std::to_string(cfg.gemm_mode) + " needs the tcgen05 kernels (sm_100a)");
    g->world = world;
    g->fold = (g_stage_fold.load() >= 2 && cfg.spmm_mode == MG_SPMM_FAST && world > 2) ? g_stage_fold.load() : 0;
    g->n = p->n;
    g->mask_count = p->mask_count;
    g->bounds = p->bounds;
    for (index_t d : cfg.dims) g->ld.push_back(pad4(d));
    for (size_t i = 1; i < g->ld.size(); ++i) g->ld_max = std::max(g->ld_max, g->ld[i]);
    if (cfg.order_swap || cfg.aggregate_first()) g->ld_max = std::max(g->ld_max, g->ld[0]);
    for (int i = 0; i < world; ++i) g->max_part = std::max(g->max_part, p->bounds[i + 1] - p->bounds[i]);
    for (int b = 0; b <= 8; ++b) g->wblocks[b] = static_cast<index_t>(b) * p->n / 8;  // driver.hpp:156
    // transport
    std::vector<int> devs(devices, devices + n_local);
    std::vector<int> sorted = devs;
    std::sort(sorted.begin(), sorted.end());
    const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    const bool one_device = sorted.front() == sorted.back();
    if (transport == MG_TRANSPORT_AUTO) transport = (distinct || n_local < world) ? MG_TRANSPORT_NCCL : MG_TRANSPORT_LOCAL;
    if (transport == MG_TRANSPORT_SOLO && n_local != 1)
      throw ValueError("group: the solo transport (measurement only) drives exactly one rank");
    if (transport < MG_TRANSPORT_NCCL || transport > MG_TRANSPORT_SOLO) throw ValueError("group: unknown transport");
    if (transport == MG_TRANSPORT_LOCAL && n_local != world)
      throw ValueError("group: the in-process transport needs every rank local");
    // LOCAL's peer copies and rank-order reduction dereference every worker's buffers from worker 0's device:
    // no peer access is set up, so it is only legal when every worker shares one device.
    if (transport == MG_TRANSPORT_LOCAL && !one_device)
      throw ValueError("group: the in-process transport needs every worker on one device (got a mix of devices; "
                       "use one device per worker for NCCL)");
    if (transport == MG_TRANSPORT_LOCAL && world > k::kMaxLocal)
      throw ValueError("group: the in-process transport supports at most " + std::to_string(k::kMaxLocal) + " workers");
    if (transport == MG_TRANSPORT_NCCL && !distinct)
      throw ValueError("group: NCCL needs one device per local worker");
    if (transport == MG_TRANSPORT_NCCL && n_local < world && !nccl_id)
      throw ValueError("group: ranks in other processes need the shared nccl_id");
    g->transport = transport;
    // labels in range for masked rows (checked where the reference checks, at the loss: dense.hpp:263)
    const index_t C = cfg.dims.back();
    for (index_t i = 0; i < p->rows_stored() && g->labels_ok; ++i)
      if (p->mask[i] && (p->labels[i] < 0 || p->labels[i] >= C)) {
        g->labels_ok = false;
        g->label_error = "softmax_xent: label " + std::to_string(p->labels[i]) + " out of range [0, " +
                         std::to_string(C) + ") at row " + std::to_string(p->row0 + i);
      }
    const int L = cfg.layers();
    Stopwatch sw;
    for (int k = 0; k < n_local; ++k) {
      auto wp = std::make_unique<Worker>();
      Worker& w = *wp;
      w.rank = local_ranks[k];
      w.device = devices[k];
      if (w.rank < 0 || w.rank >= world) throw ValueError("group: rank out of range");
      if (!p->has_row(w.rank)) throw ValueError("group: partition lacks row block " + std::to_string(w.rank));
      w.r0 = p->bounds[w.rank];
      w.rows = p->bounds[w.rank + 1] - w.r0;
      if (w.r0 < p->row0 || w.r0 + w.rows > p->row0 + p->rows_stored())
        throw ValueError("group: partition lacks the rows of block " + std::to_string(w.rank));
      const index_t lr0 = w.r0 - p->row0;  // first row of this block in the partition's row storage
      MG_CUDA(cudaSetDevice(w.device));
      MG_CUDA(cudaStreamCreateWithFlags(&w.s0, cudaStreamNonBlocking));
      MG_CUDA(cudaStreamCreateWithFlags(&w.s1, cudaStreamNonBlocking));
      MG_CUDA(cudaStreamCreateWithFlags(&w.s2, cudaStreamNonBlocking));
      for (auto* e : {&w.prior, &w.heavy_fork, &w.heavy_join, &w.loss_done, &w.stats_done, &w.src_ready, &w.copy_done,
                      &w.ar_ready, &w.ar_done, &w.join1, &w.join2})
        *e = mk_event();
      for (int j = 0; j < world; ++j) {
        w.bc_done.push_back(mk_event());
        w.mult.push_back(mk_event());
      }
      for (int l = 0; l < L; ++l) {
        w.wg_done.push_back(mk_event());
        w.red_done.push_back(mk_event());
      }
      w.t_start = mk_event(true);
      w.t_end = mk_event(true);
      if (g->fold) {  // SpMM steps: groups of <= fold consecutive received stages, the own stage alone
        w.step_of.assign(world, 0);
        for (int j = 0; j < world;) {
          int e = j + 1;
          if (j != w.rank)
            while (e < world && e - j < g->fold && e != w.rank) ++e;
          w.step_first.push_back(j);
          w.step_last.push_back(e - 1);
          for (int q = j; q < e; ++q) w.step_of[q] = static_cast<int>(w.step_first.size()) - 1;
          j = e;
        }
      }
      // rows: x_local (gcn.hpp:127-132). Page-locked features of the padded width go up on a copy stream
      // while the backward tiles are processed (after the forward tiles' DMAs, so the two do not share
      // the link); otherwise synchronously after the tiles.
      w.x = dalloc_t<float>(*g, w, std::max<index_t>(1, w.rows * g->ld[0]));
      const float* xsrc = p->features.data() + lr0 * p->d0;
      const bool x_async = p->d0 == g->ld[0] && w.rows > 0 && is_pinned_host(xsrc);
      cudaStream_t xs = nullptr;
      // tiles
      int max_segments = 0;
      for (int d = 0; d < 2; ++d) {
        w.tiles[d].resize(world);
        if (d == 1 && x_async) {
          MG_CUDA(cudaStreamCreateWithFlags(&xs, cudaStreamNonBlocking));
          MG_CUDA(cudaStreamSynchronize(cudaStreamLegacy));  // w.x's zero-fill precedes the copy stream's DMA
          MG_CUDA(cudaMemcpyAsync(w.x, xsrc, sizeof(float) * w.rows * p->d0, cudaMemcpyHostToDevice, xs));
        }
        for (int j = 0; j < world; ++j) {
          // a stage folded into a group is only ever read through the group's merged tile (below)
          if (g->fold && w.step_first[w.step_of[j]] != w.step_last[w.step_of[j]]) continue;
          const bool tr = d == 1 && world == 1 && g_bwd_transpose.load();
          upload_tile(*g, w, p->tiles[d][w.rank][j], w.tiles[d][j], tr ? &w.tiles[0][0] : nullptr);
          max_segments = std::max(max_segments, w.tiles[d][j].n_segments);
        }
        if (g->fold) {  // merged tiles of the folded stage pairs
          w.ftiles[d].resize(world);
          for (size_t st = 0; st < w.step_first.size(); ++st) {
            const int j0 = w.step_first[st], j1 = w.step_last[st];
            if (j1 == j0) continue;
            std::vector<const Tile*> parts;
            for (int q = j0; q <= j1; ++q) parts.push_back(&p->tiles[d][w.rank][q]);
            upload_tile(*g, w, merge_tiles(parts), w.ftiles[d][j0]);
            max_segments = std::max(max_segments, w.ftiles[d][j0].n_segments);
          }
        }
      }
      if (max_segments > 0) w.seg_scratch = dalloc_t<float>(*g, w, static_cast<size_t>(max_segments) * g->ld_max);
      sw.lap("tiles");
      if (xs) {
        MG_CUDA(cudaStreamSynchronize(xs));
        MG_CUDA(cudaStreamDestroy(xs));
      } else {
        upload_padded(w.x, xsrc, w.rows, p->d0, g->ld[0]);
      }
      w.labels = dalloc_t<int>(*g, w, std::max<index_t>(1, w.rows));
      w.mask = dalloc_t<uint8_t>(*g, w, std::max<index_t>(1, w.rows));
      if (w.rows) {
        MG_CUDA(cudaMemcpy(w.labels, p->labels.data() + lr0, sizeof(int) * w.rows, cudaMemcpyHostToDevice));
        MG_CUDA(cudaMemcpy(w.mask, p->mask.data() + lr0, w.rows, cudaMemcpyHostToDevice));
      }
      sw.lap("rows");
      // the L + 3 buffer plan (gcn.hpp:134-140)
      for (int l = 0; l < L; ++l) w.ahw.push_back(dalloc_t<float>(*g, w, std::max<index_t>(1, w.rows * g->ld[l + 1])));
      w.hw = dalloc_t<float>(*g, w, std::max<index_t>(1, w.rows * g->ld_max));
      const index_t bc_rows = std::max(1, g->fold) * g->max_part;  // a folded group's blocks stacked
      w.bc1 = dalloc_t<float>(*g, w, std::max<index_t>(1, bc_rows * g->ld_max));
      w.bc2 = dalloc_t<float>(*g, w, std::max<index_t>(1, bc_rows * g->ld_max));
      if (cfg.aggregate_first()) w.ax = dalloc_t<float>(*g, w, std::max<index_t>(1, w.rows * g->ld[0]));
      if (cfg.gemm_mode == MG_GEMM_TF32X3 && cfg.spmm_mode == MG_SPMM_FAST && tc::f16_enabled()) {
        const size_t n_rm = static_cast<size_t>(L + 2) * 2 * std::max<index_t>(1, w.rows);
        w.rm = dalloc_t<float>(*g, w, n_rm);
        // test hook: row maxima start as 8e37, so a row read before its producer wrote it breaks training
        if (std::getenv("MGGCN_POISON_RM")) MG_CUDA(cudaMemset(w.rm, 0x7E, sizeof(float) * n_rm));
      }
      // parameters, Adam state, W-grad staging (gcn.hpp:150-158), padded ld_l x ld_{l+1}
      for (int l = 0; l < L; ++l) {
        const index_t sz = g->pstride(l);
        w.W.push_back(dalloc_t<float>(*g, w, sz));
        w.WG.push_back(dalloc_t<float>(*g, w, sz));
        w.M.push_back(dalloc_t<float>(*g, w, sz));
        w.V.push_back(dalloc_t<float>(*g, w, sz));
        w.stage.push_back(dalloc_t<float>(*g, w, 8 * sz));
      }
      if (cfg.gemm_mode != MG_GEMM_EXACT) {  // largest W-grad block this worker can own
        index_t kmax = 1;
        for (int b = 0; b < 8; ++b) {
          const index_t a = std::max(g->wblocks[b], w.r0), e = std::min(g->wblocks[b + 1], w.r0 + w.rows);
          kmax = std::max(kmax, e - a);
        }
        for (int l = 0; l < L; ++l)
          w.ws_bytes = std::max({w.ws_bytes, tc::tn_workspace_bytes(g->ld[l], g->ld[l + 1], std::max<index_t>(1, w.rows)),
                                 tc::nn_workspace_bytes(g->ld[l + 1], g->ld[l]),
                                 tc::nn_workspace_bytes(g->ld[l], g->ld[l + 1])});
        w.ws = static_cast<float*>(dalloc(*g, w, w.ws_bytes));
      }
      if (cfg.bias) {
        index_t kmax = 0;
        for (int b = 0; b < 8; ++b) {
          const index_t a = std::max(g->wblocks[b], w.r0), e = std::min(g->wblocks[b + 1], w.r0 + w.rows);
          kmax = std::max(kmax, e - a);
        }
        w.bias_chunks = static_cast<int>((kmax + k::kBiasChunk - 1) / k::kBiasChunk);
        w.bias_part = dalloc_t<float>(*g, w, std::max<size_t>(1, static_cast<size_t>(8) * w.bias_chunks * g->ld_max));
      }
      w.loss_blocks = std::max(1, std::min(ceil_div(w.rows, 8), num_sms() * 8));
      w.partials = dalloc_t<double>(*g, w, 2 * w.loss_blocks);
      w.stats = dalloc_t<double>(*g, w, 2);
      MG_CUDA(cudaMallocHost(&w.h_stats, 2 * sizeof(double)));
      g->workers.push_back(std::move(wp));
      sw.lap("buffers");
    }
    if (transport == MG_TRANSPORT_NCCL && (world > 1 || g_nccl_single.load())) {
      // non-blocking communicators (see MG_NCCL): a peer that never arrives surfaces as a watchdog abort
      // instead of a hang inside ncclCommInitRank
      ncclUniqueId u;
      if (nccl_id) std::memcpy(&u, nccl_id, 128);
      else MG_NCCL(ncclGetUniqueId(&u));  // every rank is in this process
      ncclConfig_t nc = NCCL_CONFIG_INITIALIZER;
      nc.blocking = 0;
      MG_NCCL(ncclGroupStart());
      for (int k = 0; k < n_local; ++k) {
        MG_CUDA(cudaSetDevice(g->workers[k]->device));
        MG_NCCL(ncclCommInitRankConfig(&g->workers[k]->comm, world, u, g->workers[k]->rank, &nc));
      }
      MG_NCCL(ncclGroupEnd());
      nccl_settle(*g);
    }
    sw.lap("nccl");
    for (auto& wp : g->workers) {
      MG_CUDA(cudaSetDevice(wp->device));
      MG_CUDA(cudaDeviceSynchronize());
    }
    sw.lap("sync");
    g->sealed = true;
    *out = g.release();
  });
}

// GcnWorker::init_params (gcn.hpp:163-173): one Rng(seed) across layers, Glorot-uniform in double,
// cast to float; identical on every worker (the reference broadcasts rank 0's draw).
// DeviceGroup::abort (collectives.cpp:42-52): callable from any thread; the next (or current) host wait on
// the group aborts its communicators and raises ShutdownError, and the group refuses further work.
mg_status mg_group_abort(mg_group* g) {
  return guarded([&] {
    if (!g) throw ValueError("group: null");
    g->abort_requested = true;
  });
}

mg_status mg_group_init_params(mg_group* g) {
  return guarded([&] {
    Rng rng(g->cfg.seed);
    const int L = g->cfg.layers();
    for (int l = 0; l < L; ++l) {
      const index_t dl = g->cfg.dims[l], dl1 = g->cfg.dims[l + 1];
      const double limit = std::sqrt(6.0 / static_cast<double>(dl + dl1));
      std::vector<float> w(dl * dl1);
      for (auto& x : w) x = static_cast<float>(rng.uniform(-limit, limit));
      for (auto& wp : g->workers) {
        MG_CUDA(cudaSetDevice(wp->device));
        upload_padded(wp->W[l], w.data(), dl, dl1, g->ld[l + 1]);
        const size_t sz = sizeof(float) * g->pstride(l);
        if (g->cfg.bias) MG_CUDA(cudaMemset(wp->W[l] + g->ld[l] * g->ld[l + 1], 0, sizeof(float) * g->ld[l + 1]));
        MG_CUDA(cudaMemset(wp->M[l], 0, sz));
        MG_CUDA(cudaMemset(wp->V[l], 0, sz));
        MG_CUDA(cudaMemset(wp->WG[l], 0, sz));
      }
    }
  });
}

static void enqueue_train(mg_group* g, int t, bool adam) {
  // a step that has to (re)compute the cached Â·X runs on the stream path; the graph is captured without it
  if (adam && mg::step_graph_ok(*g) && (!mg::ax_cache_applies(*g) || mg::ax_cached(*g))) {
    mg::enqueue_train_graph(*g, t);
    return;
  }
  Step st(*g);
  st.set_training(t);
  st.begin();
  st.forward();
  st.loss_grad();
  st.backward();
  st.finalize(adam, t);
  st.end();
  g->stats_pending = true;
}

mg_status mg_group_train_step_async(mg_group* g, int32_t t) {
  return guarded([&] { enqueue_train(g, t, true); });
}

mg_status mg_group_sync(mg_group* g) {
  return guarded([&] {
    sync_all(*g);
    if (g->stats_pending) {
      read_stats(*g);
      g->stats_pending = false;
    }
  });
}

mg_status mg_group_last_stats(mg_group* g, double* loss, double* acc) {
  return guarded([&] {
    if (g->stats_pending) {
      read_stats(*g);
      g->stats_pending = false;
    }
    if (loss) *loss = g->last_loss;
    if (acc) *acc = g->last_acc;
  });
}

mg_status mg_group_train_step(mg_group* g, int32_t t, double* loss, double* acc, double* wall_us) {
  return guarded([&] {
    enqueue_train(g, t, true);
    sync_all(*g);
    read_stats(*g);
    g->stats_pending = false;
    if (loss) *loss = g->last_loss;
    if (acc) *acc = g->last_acc;
    if (wall_us) {
      Worker& w = *g->workers[0];
      float ms = 0.f;
      MG_CUDA(cudaEventElapsedTime(&ms, w.t_start, w.t_end));
      *wall_us = 1000.0 * ms;
    }
  });
}

mg_status mg_group_compute_gradients(mg_group* g, double* loss, double* acc) {
  return guarded([&] {
    enqueue_train(g, 1, false);
    sync_all(*g);
    read_stats(*g);
    g->stats_pending = false;
    if (loss) *loss = g->last_loss;
    if (acc) *acc = g->last_acc;
  });
}

mg_status mg_group_forward(mg_group* g) {
  return guarded([&] {
    Step st(*g);
    st.begin();
    st.forward();
    st.end();
    sync_all(*g);
  });
}

// GcnWorker::submit_backward + submit_finalize(false) (gcn.hpp:292-377): backward from whatever gradient
// the logits buffer ahw[L-1] holds (e.g. written with mg_group_write), W_G finalized, no Adam.
mg_status mg_group_backward(mg_group* g) {
  return guarded([&] {
    Step st(*g);
    st.begin();
    st.backward();
    st.finalize(false, 0);
    st.end();
    sync_all(*g);
  });
}

// GcnWorker::loss_only (gcn.hpp:189-205): forward, then the masked loss without touching the logits.
// The loss kernel writes gradients in place, so the logits are preserved through hw (never larger).
mg_status mg_group_loss_only(mg_group* g, double* loss) {
  return guarded([&] {
    Step st(*g);
    st.begin();
    st.forward();
    const int L = g->cfg.layers();
    const index_t ldc = g->ld[L];
    for (auto& wp : g->workers) {  // keep a copy of the logits in hw (n x ld_L <= n x ld_max)
      MG_CUDA(cudaSetDevice(wp->device));
      MG_CUDA(cudaMemcpyAsync(wp->hw, wp->ahw[L - 1], sizeof(float) * wp->rows * ldc, cudaMemcpyDeviceToDevice, wp->s0));
    }
    st.loss_grad();
    for (auto& wp : g->workers) {
      MG_CUDA(cudaSetDevice(wp->device));
      MG_CUDA(cudaMemcpyAsync(wp->ahw[L - 1], wp->hw, sizeof(float) * wp->rows * ldc, cudaMemcpyDeviceToDevice, wp->s0));
    }
    st.end();
    sync_all(*g);
    read_stats(*g);
    g->stats_pending = false;
    if (loss) *loss = g->last_loss;
  });
}

static Worker& find_worker(mg_group* g, int32_t rank) {
  for (auto& wp : g->workers)
    if (wp->rank == rank) return *wp;
  throw ValueError("group: rank " + std::to_string(rank) + " is not local to this process");
}

struct TensorView {
  float* p;
  index_t rows, cols, ld;
};

static TensorView tensor_view(mg_group* g, Worker& w, int which, int layer) {
  const int L = g->cfg.layers();
  auto need_layer = [&] {
    if (layer < 0 || layer >= L) throw ValueError("tensor: layer " + std::to_string(layer) + " out of range");
  };
  switch (which) {
    case MG_T_W: need_layer(); return {w.W[layer], g->cfg.dims[layer], g->cfg.dims[layer + 1], g->ld[layer + 1]};
    case MG_T_WGRAD: need_layer(); return {w.WG[layer], g->cfg.dims[layer], g->cfg.dims[layer + 1], g->ld[layer + 1]};
    case MG_T_ADAM_M: need_layer(); return {w.M[layer], g->cfg.dims[layer], g->cfg.dims[layer + 1], g->ld[layer + 1]};
    case MG_T_ADAM_V: need_layer(); return {w.V[layer], g->cfg.dims[layer], g->cfg.dims[layer + 1], g->ld[layer + 1]};
    case MG_T_AHW: need_layer(); return {w.ahw[layer], w.rows, g->cfg.dims[layer + 1], g->ld[layer + 1]};
    case MG_T_HW: need_layer(); return {w.hw, w.rows, g->cfg.dims[layer + 1], g->ld[layer + 1]};
    case MG_T_X: return {w.x, w.rows, g->cfg.dims[0], g->ld[0]};
    case MG_T_WSTAGE: {
      need_layer();
      // 8 blocks of (ld_l x ld_{l+1}); exposed as 8 d_l x d_{l+1} blocks stacked
      return {w.stage[layer], 8 * g->cfg.dims[layer], g->cfg.dims[layer + 1], g->ld[layer + 1]};
    }
    case MG_T_BIAS:
    case MG_T_BIAS_GRAD: {
      need_layer();
      if (!g->cfg.bias) throw ValueError("tensor: the group has no bias (config bias = 0)");
      float* base = which == MG_T_BIAS ? w.W[layer] : w.WG[layer];
      return {base + g->ld[layer] * g->ld[layer + 1], 1, g->cfg.dims[layer + 1], g->ld[layer + 1]};
    }
    case MG_T_ROWMAX: {  // the f16 split's per-row max pairs of slot `layer` (rows x 2; diagnostics)
      if (!w.rm) throw ValueError("tensor: the group keeps no row maxima (TF32X3 + FAST only)");
      if (layer < 0 || layer > g->cfg.layers() + 1) throw ValueError("tensor: row-max slot out of range");
      return {w.rm_slot(layer), w.rows, 2, 2};
    }
    default: throw ValueError("tensor: unknown id " + std::to_string(which));
  }
}

mg_status mg_group_read(mg_group* g, int32_t rank, int32_t which, int32_t layer, float* dst, int64_t count) {
  return guarded([&] {
    Worker& w = find_worker(g, rank);
    MG_CUDA(cudaSetDevice(w.device));
    sync_all(*g);
    TensorView v = tensor_view(g, w, which, layer);
    if (count != v.rows * v.cols)
      throw ShapeError("tensor: count " + std::to_string(count) + " != " + shape_str(v.rows, v.cols));
    if (which == MG_T_WSTAGE) {
      const index_t dl = g->cfg.dims[layer], bs = g->pstride(layer);
      for (int b = 0; b < 8; ++b) download_padded(dst + b * dl * v.cols, v.p + b * bs, dl, v.cols, v.ld);
      return;
    }
    download_padded(dst, v.p, v.rows, v.cols, v.ld);
  });
}

mg_status mg_group_write(mg_group* g, int32_t rank, int32_t which, int32_t layer, const float* src, int64_t count) {
  return guarded([&] {
    auto write_one = [&](Worker& w) {
      MG_CUDA(cudaSetDevice(w.device));
      TensorView v = tensor_view(g, w, which, layer);
      if (which == MG_T_WSTAGE) throw ValueError("tensor: the staging buffer is read-only");
      if (count != v.rows * v.cols)
        throw ShapeError("tensor: count " + std::to_string(count) + " != " + shape_str(v.rows, v.cols));
      upload_padded(v.p, src, v.rows, v.cols, v.ld);
    };
    sync_all(*g);
    if (which == MG_T_X) g->ax_epoch = 0;  // the cached Â·X is stale
    if (rank < 0) {  // replicated tensors: write every local worker
      for (auto& wp : g->workers) write_one(*wp);
    } else {
      write_one(find_worker(g, rank));
    }
  });
}

// FNV-1a over the unpadded W bytes of every layer (gcn.hpp:87-94, :221-226).
mg_status mg_group_w_hash(mg_group* g, int32_t rank, uint64_t* hash) {
  return guarded([&] {
    Worker& w = find_worker(g, rank);
    MG_CUDA(cudaSetDevice(w.device));
    sync_all(*g);
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (int l = 0; l < g->cfg.layers(); ++l) {
      const index_t dl = g->cfg.dims[l], dl1 = g->cfg.dims[l + 1];
      std::vector<float> buf(dl * dl1);
      download_padded(buf.data(), w.W[l], dl, dl1, g->ld[l + 1]);
      const auto* p = reinterpret_cast<const unsigned char*>(buf.data());
      for (size_t i = 0; i < buf.size() * 4; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
      }
    }
    *hash = h;
  });
}

mg_status mg_group_rows(mg_group* g, int32_t rank, int64_t* row_begin, int64_t* rows) {
  return guarded([&] {
    Worker& w = find_worker(g, rank);
    if (row_begin) *row_begin = w.r0;
    if (rows) *rows = w.rows;
  });
}

mg_status mg_group_buffer_audit(mg_group* g, int32_t* large_buffers, int64_t* step_allocations, int64_t* device_bytes) {
  return guarded([&] {
    // ahw[L] + hw + bc1 + bc2 (+ Â·X under aggregate_first)
    if (large_buffers) *large_buffers = g->cfg.layers() + 3 + (g->cfg.aggregate_first() ? 1 : 0);
    if (step_allocations) *step_allocations = g->step_allocs;
    if (device_bytes) *device_bytes = g->workers[0]->bytes;
  });
}

mg_status mg_group_last_profile(mg_group* g, double* spmm_us, double* gemm_us, double* other_us, int64_t* kernels) {
  return guarded([&] {
    sync_all(*g);
    double t[3] = {0, 0, 0};
    for (auto& [kind, idx] : g->prof_pending) {
      float ms = 0.f;
      MG_CUDA(cudaEventElapsedTime(&ms, g->prof_pool[idx], g->prof_pool[idx + 1]));
      t[kind] += 1000.0 * ms;
    }
    g->prof_pending.clear();
    g->prof_used = 0;
    if (spmm_us) *spmm_us = t[0];
    if (gemm_us) *gemm_us = t[1];
    if (other_us) *other_us = t[2];
    if (kernels) *kernels = g->kernels_total;
    g->kernels_total = 0;
  });
}

mg_status mg_group_graph_steps(mg_group* g, int64_t* replays, int64_t* captures) {
  return guarded([&] {
    if (!g) throw ValueError("group: null");
    if (replays) *replays = g->graph_replays;
    if (captures) *captures = g->graph_captures;
  });
}

void mg_group_destroy(mg_group* g) {
  if (!g) return;
  for (auto& wp : g->workers) {
    Worker& w = *wp;
    cudaSetDevice(w.device);
    cudaDeviceSynchronize();
    (void)cudaGetLastError();
    // an aborted communicator is gone already; a drained one has nothing in flight, so abort = release
    if (w.comm) ncclCommAbort(w.comm);
    for (auto& a : w.allocs) block_cache().put(w.device, a.first, a.second);
    if (w.h_stats) cudaFreeHost(w.h_stats);
    for (cudaEvent_t e : {w.prior, w.heavy_fork, w.heavy_join, w.loss_done, w.stats_done, w.src_ready, w.copy_done,
                          w.ar_ready, w.ar_done, w.join1, w.join2, w.t_start, w.t_end})
      if (e) cudaEventDestroy(e);
    for (auto* vec : {&w.bc_done, &w.mult, &w.wg_done, &w.red_done, &w.tl_pool})
      for (cudaEvent_t e : *vec) cudaEventDestroy(e);
    if (w.tl_base) cudaEventDestroy(w.tl_base);
    for (cudaStream_t st : {w.s0, w.s1, w.s2})
      if (st) cudaStreamDestroy(st);
  }
  if (!g->workers.empty()) cudaSetDevice(g->workers[0]->device);
  if (g->sg.exec) cudaGraphExecDestroy(g->sg.exec);
  if (g->sg.graph) cudaGraphDestroy(g->sg.graph);
  for (cudaEvent_t e : g->prof_pool) cudaEventDestroy(e);
  delete g;
}

// ---------------------------------------------------------------- timeline / bench-spmm
mg_status mg_group_set_timeline(mg_group* g, int32_t on) {
  return guarded([&] {
    if (!g) throw ValueError("group: null");
    sync_all(*g);
    if (on) {
      g->tl.clear();
      g->tl_out.clear();
      g->tl_next = 1;
      for (auto& wp : g->workers) {
        Worker& w = *wp;
        MG_CUDA(cudaSetDevice(w.device));
        if (!w.tl_base) w.tl_base = mk_event(true);
        MG_CUDA(cudaEventRecord(w.tl_base, w.s0));
        w.tl_used = 0;
        w.last_task[0] = w.last_task[1] = 0;
      }
    }
    g->tl_on = on != 0;
  });
}

mg_status mg_group_timeline(mg_group* g, mg_timeline_event* out, int64_t capacity, int64_t* count) {
  return guarded([&] {
    if (!g || !count) throw ValueError("timeline: null argument");
    sync_all(*g);
    g->tl_out.clear();
    for (const auto& r : g->tl) {
      Worker& w = *g->workers[static_cast<size_t>(r.worker_k)];
      MG_CUDA(cudaSetDevice(w.device));
      float a = 0.f, b = 0.f;
      MG_CUDA(cudaEventElapsedTime(&a, w.tl_base, w.tl_pool[r.ev]));
      MG_CUDA(cudaEventElapsedTime(&b, w.tl_base, w.tl_pool[r.ev + 1]));
      mg_timeline_event e{};
      e.worker = w.rank;
      e.lane = r.lane;
      e.stage = r.stage;
      e.n_deps = static_cast<int32_t>(r.deps.size());
      std::snprintf(e.kind, sizeof(e.kind), "%s", r.kind);
      std::snprintf(e.op, sizeof(e.op), "%s", r.op);
      e.t_start_us = 1000.0 * a;
      e.t_end_us = 1000.0 * b;
      e.task = r.task;
      e.deps = r.deps.empty() ? nullptr : r.deps.data();
      g->tl_out.push_back(e);
    }
    *count = static_cast<int64_t>(g->tl_out.size());
    if (out)
      std::copy(g->tl_out.begin(), g->tl_out.begin() + std::min<int64_t>(capacity, *count), out);
  });
}

mg_status mg_group_bench_spmm(mg_group* g, int32_t dir, double* wall_us) {
  return guarded([&] {
    if (!g) throw ValueError("group: null");
    if (dir != 0 && dir != 1) throw ValueError("bench_spmm: dir must be 0 (forward) or 1 (backward)");
    if (pad4(g->cfg.dims[0]) > g->ld_max)
      throw ValueError("bench_spmm: width " + std::to_string(g->cfg.dims[0]) +
                       " exceeds the group's buffer width " + std::to_string(g->ld_max) +
                       " (create the group with layer_dims[0] <= the widest hidden layer, or order_swap)");
    Step st(*g);
    std::vector<float*> src, out;
    for (auto& wp : g->workers) {
      src.push_back(wp->x);
      out.push_back(wp->hw);
    }
    Worker& w0 = *g->workers[0];
    MG_CUDA(cudaSetDevice(w0.device));
    MG_CUDA(cudaEventRecord(w0.t_start, w0.s0));
    st.staged_spmm(dir, g->cfg.dims[0], src, out, false);
    MG_CUDA(cudaSetDevice(w0.device));
    MG_CUDA(cudaEventRecord(w0.t_end, w0.s0));
    sync_all(*g);
    float ms = 0.f;
    MG_CUDA(cudaEventElapsedTime(&ms, w0.t_start, w0.t_end));
    if (wall_us) *wall_us = 1000.0 * ms;
  });
}

// ---------------------------------------------------------------- kernel-level entry points
mg_status mg_dev_spmm(int64_t rows, const int32_t* row_ptr, const void* edges, const float* h, float* out, int64_t w,
                      int64_t ld, int32_t accumulate, int32_t relu, int32_t mode, void* stream) {
  return guarded([&] {
    if (ld % 4 != 0 || ld < w) throw ValueError("spmm: ld must be a multiple of 4 and >= w");
    if (mode != MG_SPMM_EXACT && mode != MG_SPMM_FAST) throw ValueError("spmm: unknown mode");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::vector<int> rp32(rows + 1);
    MG_CUDA(cudaMemcpy(rp32.data(), row_ptr, sizeof(int) * (rows + 1), cudaMemcpyDeviceToHost));
    std::vector<index_t> rp(rp32.begin(), rp32.end());
    if (mode == MG_SPMM_FAST) {
      std::vector<int4> items, hubs;
      int nseg = 0;
      build_fast_items(rp, items, hubs, nseg);
      int4 *di = nullptr, *dh = nullptr;
      float* sc = nullptr;
      MG_CUDA(cudaMalloc(&di, sizeof(int4) * std::max<size_t>(1, items.size())));
      MG_CUDA(cudaMalloc(&dh, sizeof(int4) * std::max<size_t>(1, hubs.size())));
      MG_CUDA(cudaMalloc(&sc, sizeof(float) * std::max<size_t>(1, static_cast<size_t>(nseg) * ld)));
      if (!items.empty()) MG_CUDA(cudaMemcpy(di, items.data(), sizeof(int4) * items.size(), cudaMemcpyHostToDevice));
      if (!hubs.empty()) MG_CUDA(cudaMemcpy(dh, hubs.data(), sizeof(int4) * hubs.size(), cudaMemcpyHostToDevice));
      std::vector<int4> seg_items, pieces;
      for (const int4& it : items)
        if (it.z < 0) seg_items.push_back(it);
      build_stream_pieces(rp, seg_items, pieces);
      int4* dp = nullptr;
      MG_CUDA(cudaMalloc(&dp, sizeof(int4) * std::max<size_t>(1, pieces.size())));
      if (!pieces.empty()) MG_CUDA(cudaMemcpy(dp, pieces.data(), sizeof(int4) * pieces.size(), cudaMemcpyHostToDevice));
      FastLaunch fl{di, static_cast<int>(items.size()), dh, static_cast<int>(hubs.size()),
                    static_cast<const int2*>(edges), sc, false, 0, dp, static_cast<int>(pieces.size()), row_ptr,
                    rows ? static_cast<double>(rp.back()) / rows : 0.0};
      spmm_fast(fl, h, out, ld, accumulate, relu, k::Epi{}, s);
      MG_CUDA(cudaStreamSynchronize(s));
      cudaFree(di);
      cudaFree(dh);
      cudaFree(sc);
      cudaFree(dp);
      return;
    }
    std::vector<int> light, heavy;
    build_orders(rp, light, heavy);
    int *dl = nullptr, *dh = nullptr;
    MG_CUDA(cudaMalloc(&dl, sizeof(int) * std::max<size_t>(1, light.size())));
    MG_CUDA(cudaMalloc(&dh, sizeof(int) * std::max<size_t>(1, heavy.size())));
    if (!light.empty()) MG_CUDA(cudaMemcpy(dl, light.data(), sizeof(int) * light.size(), cudaMemcpyHostToDevice));
    if (!heavy.empty()) MG_CUDA(cudaMemcpy(dh, heavy.data(), sizeof(int) * heavy.size(), cudaMemcpyHostToDevice));
    // the hub-row kernel bulk-copies edge records from 16-byte aligned starts: give it a padded copy
    int2* ep = nullptr;
    if (!heavy.empty()) {
      const index_t nnz = rp.back();
      MG_CUDA(cudaMalloc(&ep, sizeof(int2) * (nnz + k::kEdgePad)));
      MG_CUDA(cudaMemsetAsync(ep, 0, sizeof(int2) * (nnz + k::kEdgePad), s));
      MG_CUDA(cudaMemcpyAsync(ep, edges, sizeof(int2) * nnz, cudaMemcpyDeviceToDevice, s));
    }
    SpmmLaunch sl{row_ptr, ep ? ep : static_cast<const int2*>(edges), dl, static_cast<int>(light.size()), dh,
                  static_cast<int>(heavy.size())};
    spmm_heavy(sl, h, out, ld, accumulate, relu, k::Epi{}, s);
    spmm_light(sl, h, out, ld, accumulate, relu, k::Epi{}, s);
    MG_CUDA(cudaStreamSynchronize(s));
    cudaFree(dl);
    cudaFree(dh);
    if (ep) cudaFree(ep);
  });
}

mg_status mg_dev_gemm(int32_t ta, int32_t tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                      const float* B, int64_t ldb, float* Cm, int64_t ldc, int32_t epilogue, int32_t mode,
                      void* stream) {
  return guarded([&] {
    if (epilogue < 0 || epilogue > 2) throw ValueError("gemm: unknown epilogue");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // workspaces come from the block cache (no cudaMalloc / cudaFree per call) and go back to it after a
    // stream synchronise
    const int dev = cur_device();
    float* ws = nullptr;
    size_t wsb = 0, wsr = 0, rmr = 0;
    float* rm = nullptr;  // NN / NT fp16 split: A's per-row max pairs, as the training step's producers write them
    if (mode != MG_GEMM_EXACT) {
      wsb = ta ? tc::tn_workspace_bytes(M, N, std::max<int64_t>(K, 1)) : tc::nn_workspace_bytes(N, K);
      wsr = BlockCache::round(wsb);
      ws = static_cast<float*>(block_cache().get(dev, wsr));
      if (!ta && mode == MG_GEMM_TF32X3 && M > 0 && tc::f16_enabled()) {
        rmr = BlockCache::round(sizeof(float) * 2 * M);
        rm = static_cast<float*>(block_cache().get(dev, rmr));
        row_absmax_pairs<<<static_cast<int>(std::min<int64_t>(4096, (M + 7) / 8)), 256, 0, st>>>(A, lda, M, K, rm);
        MG_LAUNCHED();
      }
    }
    try {
      gemm_launch(mode, ta != 0, tb != 0, M, N, K, A, lda, B, ldb, Cm, ldc, epilogue, st, ws, wsb, k::Epi{}, rm);
    } catch (...) {
      cudaStreamSynchronize(st);
      block_cache().put(dev, ws, wsr);
      block_cache().put(dev, rm, rmr);
      throw;
    }
    if (ws) {
      MG_CUDA(cudaStreamSynchronize(st));
      block_cache().put(dev, ws, wsr);
      block_cache().put(dev, rm, rmr);
    }
  });
}

mg_status mg_dev_softmax_xent(float* logits, int64_t rows, int64_t classes, int64_t ld, const int32_t* labels,
                              const uint8_t* mask, int64_t denom, double* stats, void* stream) {
  return guarded([&] {
    if (rows < 0 || classes < 1 || ld < classes) throw ShapeError("softmax_xent: bad shape");
    if (classes > 32 * k::kLossCpl)
      throw ValueError("softmax_xent: at most " + std::to_string(32 * k::kLossCpl) + " classes per row");
    if (denom <= 0) throw ValueError("softmax_xent: empty mask");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // the reference's label contract (dense.hpp:261-264), checked on the masked rows like the group's upload
    std::vector<int32_t> hl(rows);
    std::vector<uint8_t> hm(rows);
    if (rows > 0) {
      MG_CUDA(cudaMemcpyAsync(hl.data(), labels, sizeof(int32_t) * rows, cudaMemcpyDeviceToHost, s));
      MG_CUDA(cudaMemcpyAsync(hm.data(), mask, rows, cudaMemcpyDeviceToHost, s));
      MG_CUDA(cudaStreamSynchronize(s));
    }
    for (int64_t v = 0; v < rows; ++v)
      if (hm[v] && (hl[v] < 0 || hl[v] >= classes))
        throw ValueError("softmax_xent: label " + std::to_string(hl[v]) + " out of range [0, " +
                         std::to_string(classes) + ") at row " + std::to_string(v));
    const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, 8), num_sms() * 8)));
    double* part = nullptr;
    MG_CUDA(cudaMalloc(&part, sizeof(double) * (2 * blocks + 2)));
    const float inv = 1.0f / static_cast<float>(denom);
    const int R = static_cast<int>(rows), Cc = static_cast<int>(classes), L = static_cast<int>(ld);
    if (rows > 0) launch_softmax_xent(Cc, blocks, s, logits, L, R, labels, mask, inv, part);
    k::finalize_stats<<<1, 32, 0, s>>>(part, rows > 0 ? blocks : 0, part + 2 * blocks);
    MG_LAUNCHED();
    MG_CUDA(cudaMemcpyAsync(stats, part + 2 * blocks, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    MG_CUDA(cudaStreamSynchronize(s));
    cudaFree(part);
  });
}

mg_status mg_dev_adam(float* w, float* grad, float* m, float* v, int64_t size, double lr, double beta1, double beta2,
                      double epsilon, int32_t t, void* stream) {
  return guarded([&] {
    const k::AdamConsts c = adam_consts(lr, beta1, beta2, epsilon, t);
    if (size < 0 || size > INT32_MAX) throw ShapeError("adam_step: bad parameter count");
    if (size == 0) return;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    float* stage = nullptr;  // finalize_adam reads the gradient as a one-block stage and zeroes `grad`
    MG_CUDA(cudaMalloc(&stage, sizeof(float) * size));
    MG_CUDA(cudaMemcpyAsync(stage, grad, sizeof(float) * size, cudaMemcpyDeviceToDevice, s));
    const int n = static_cast<int>(size);
    k::finalize_adam<<<std::min(1024, (n + 255) / 256), 256, 0, s>>>(n, 1, stage, w, grad, m, v, 1, c);
    MG_LAUNCHED();
    MG_CUDA(cudaStreamSynchronize(s));
    cudaFree(stage);
  });
}

}  // extern "C"
