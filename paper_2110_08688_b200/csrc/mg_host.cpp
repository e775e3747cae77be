// SPDX-License-Identifier: Apache-2.0
//
// Host half of libmggcn.so: error plumbing, the platform-pinned RNG, the synthetic power-law
// generator and the partitioner (prepare_data). Everything here is bit-identical to the reference
// (rowgcn) by construction — the orders of every floating-point accumulation are the reference's —
// but restructured for a many-core host: counting sorts, per-row sorts and per-column sums run in
// parallel where the reference's result does not depend on the order of independent work.
#include <algorithm>
#include <limits>
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <numeric>

#include <cuda_runtime.h>

#include "mg_internal.hpp"

namespace mg {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

bool pinned_host_available() {
  static const bool ok = [] {
    int n = 0;
    if (std::getenv("MGGCN_NO_PINNED") || cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      return false;
    }
    return true;
  }();
  return ok;
}
void* pinned_host_alloc(size_t bytes, bool* pinned) {
  *pinned = false;
  void* p = nullptr;
  if (bytes >= (size_t(1) << 20) && pinned_host_available() &&
      cudaHostAlloc(&p, bytes, cudaHostAllocPortable) == cudaSuccess) {
    *pinned = true;
    return p;
  }
  cudaGetLastError();
  p = std::malloc(bytes ? bytes : 1);
  if (!p) throw std::bad_alloc();
  return p;
}
bool is_pinned_host(const void* p) {  // also true for interior pointers of a pinned block
  if (!p || !pinned_host_available()) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}
void pinned_host_free(void* p, bool pinned) {
  if (!p) return;
  if (pinned) cudaFreeHost(p);
  else std::free(p);
}

int host_threads() {
  static const int t = [] {
    const char* env = std::getenv("MGGCN_HOST_THREADS");
    int n = env ? std::atoi(env) : static_cast<int>(std::thread::hardware_concurrency());
    return std::max(1, std::min(n, 64));
  }();
  return t;
}

void parallel_for(index_t n, const std::function<void(index_t, index_t)>& f, index_t min_chunk) {
  if (n <= 0) return;
  const int t = static_cast<int>(std::min<index_t>(host_threads(), std::max<index_t>(1, n / min_chunk)));
  if (t <= 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> pool;
  std::exception_ptr err;
  std::mutex mu;
  const index_t chunk = (n + t - 1) / t;
  for (int i = 0; i < t; ++i) {
    const index_t b = std::min(n, i * chunk), e = std::min(n, (i + 1) * chunk);
    if (b >= e) break;
    pool.emplace_back([&, b, e] {
      try {
        f(b, e);
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        if (!err) err = std::current_exception();
      }
    });
  }
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

// ---------------------------------------------------------------- Rng: std::mt19937_64 (inc/rng.hpp)
Rng::Rng(std::uint64_t seed) {
  mt_[0] = seed;
  for (int i = 1; i < 312; ++i) mt_[i] = 6364136223846793005ULL * (mt_[i - 1] ^ (mt_[i - 1] >> 62)) + i;
  idx_ = 312;
}

void Rng::twist() {  // the mt19937_64 recurrence, split so no index needs a modulo
  constexpr std::uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
  int i = 0;
  for (; i < 156; ++i) {
    const std::uint64_t x = (mt_[i] & UM) | (mt_[i + 1] & LM);
    mt_[i] = mt_[i + 156] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
  }
  for (; i < 311; ++i) {
    const std::uint64_t x = (mt_[i] & UM) | (mt_[i + 1] & LM);
    mt_[i] = mt_[i - 156] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
  }
  const std::uint64_t x = (mt_[311] & UM) | (mt_[0] & LM);
  mt_[311] = mt_[155] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
  idx_ = 0;
}

std::uint64_t Rng::next() {
  if (idx_ >= 312) twist();
  std::uint64_t y = mt_[idx_++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

void Rng::discard(std::uint64_t k) {
  while (k) {
    if (idx_ >= 312) twist();
    const std::uint64_t a = std::min<std::uint64_t>(k, static_cast<std::uint64_t>(312 - idx_));
    idx_ += static_cast<int>(a);
    k -= a;
  }
}

// ---------------------------------------------------------------- config (inc/gcn.hpp:14-36)
Config to_config(const mg_config* c) {
  if (!c) throw ConfigError("config: null");
  Config cfg;
  if (c->n_dims > 0 && !c->layer_dims) throw ConfigError("config: layer_dims is null");
  cfg.dims.assign(c->layer_dims, c->layer_dims + std::max(0, c->n_dims));
  cfg.lr = c->lr;
  cfg.beta1 = c->beta1;
  cfg.beta2 = c->beta2;
  cfg.epsilon = c->epsilon;
  cfg.epochs = c->epochs;
  cfg.seed = c->seed;
  cfg.permute = c->permute != 0;
  cfg.overlap = c->overlap != 0;
  cfg.skip_first_backward_spmm = c->skip_first_backward_spmm != 0;
  cfg.order_swap = c->order_swap != 0;
  cfg.gemm_mode = c->gemm_mode;
  cfg.spmm_mode = c->spmm_mode;
  if (c->aggregate_input != 0 && c->aggregate_input != 1)
    throw ConfigError("config: aggregate_input must be 0 or 1, got " + std::to_string(c->aggregate_input));
  cfg.aggregate_input = c->aggregate_input != 0;
  if (c->bias != 0 && c->bias != 1) throw ConfigError("config: bias must be 0 or 1, got " + std::to_string(c->bias));
  cfg.bias = c->bias != 0;
  if (!(c->dropout >= 0.0 && c->dropout < 1.0))
    throw ConfigError("config: dropout must be in [0, 1), got " + std::to_string(c->dropout));
  cfg.dropout = c->dropout;
  if (cfg.layers() < 1)
    throw ConfigError("config: need at least one layer (layer_dims has " + std::to_string(cfg.dims.size()) +
                      " entries)");
  for (index_t d : cfg.dims)
    if (d < 1) throw ConfigError("config: layer dimension " + std::to_string(d) + " < 1");
  if (cfg.epochs < 0) throw ConfigError("config: negative epochs");
  if (cfg.gemm_mode < MG_GEMM_EXACT || cfg.gemm_mode > MG_GEMM_TF32)
    throw ConfigError("config: unknown gemm_mode " + std::to_string(cfg.gemm_mode));
  if (cfg.spmm_mode < MG_SPMM_EXACT || cfg.spmm_mode > MG_SPMM_FAST)
    throw ConfigError("config: unknown spmm_mode " + std::to_string(cfg.spmm_mode));
  return cfg;
}

// ---------------------------------------------------------------- CSR validation (inc/sparse.hpp:37-54)
void Csr::validate() const {
  if (static_cast<index_t>(row_ptr.size()) != rows + 1)
    throw ValueError("csr: row_ptr length " + std::to_string(row_ptr.size()) + " != rows+1");
  if (row_ptr[0] != 0) throw ValueError("csr: row_ptr[0] != 0");
  if (row_ptr[rows] != nnz()) throw ValueError("csr: row_ptr[rows] != nnz");
  if (values.size() != col_idx.size()) throw ValueError("csr: values/col_idx length mismatch");
  // Rows are checked in parallel chunks; each chunk keeps its first violation in (row, entry) order and the
  // lowest row wins, so the error is the one the reference's serial scan reports first, with its message.
  struct Bad {
    index_t row = -1, col = 0;
    int kind = 0;
  };
  std::mutex mu;
  Bad first;
  std::atomic<index_t> first_row{std::numeric_limits<index_t>::max()};
  parallel_for(rows, [&](index_t b, index_t e) {
    Bad mine;
    for (index_t u = b; u < e && mine.row < 0 && u < first_row.load(); ++u) {
      if (row_ptr[u] > row_ptr[u + 1]) {
        mine = {u, 0, 1};
        break;
      }
      for (index_t k = row_ptr[u]; k < row_ptr[u + 1]; ++k) {
        if (col_idx[k] < 0 || col_idx[k] >= cols) {
          mine = {u, col_idx[k], 2};
          break;
        }
        if (k > row_ptr[u] && col_idx[k] <= col_idx[k - 1]) {
          mine = {u, 0, 3};
          break;
        }
      }
    }
    if (mine.row < 0) return;
    std::lock_guard<std::mutex> lk(mu);
    if (first.row < 0 || mine.row < first.row) {
      first = mine;
      first_row = mine.row;
    }
  });
  if (first.row >= 0) {
    const std::string r = std::to_string(first.row);
    if (first.kind == 1) throw ValueError("csr: row_ptr not nondecreasing");
    if (first.kind == 2) throw ValueError("csr: col " + std::to_string(first.col) + " out of range in row " + r);
    throw ValueError("csr: columns not strictly increasing in row " + r);
  }
}

namespace {

// Internal compact graph: int64 row_ptr, int32 column, fp32 value (n < 2^31 at every config).
struct G32 {
  index_t n = 0;
  std::vector<index_t> rp;
  std::vector<std::int32_t> ci;
  std::vector<float> v;
  index_t nnz() const { return static_cast<index_t>(ci.size()); }
};

void exclusive_scan_inplace(std::vector<index_t>& a) {  // a[0..n] counts at [1..n] -> prefix
  for (size_t i = 1; i < a.size(); ++i) a[i] += a[i - 1];
}

// Sorts (col, val) pairs of one row by column. Columns are unique within a row.
void sort_row(std::int32_t* c, float* v, index_t len, std::vector<std::uint64_t>& scratch) {
  bool sorted = true;
  for (index_t i = 1; i < len && sorted; ++i) sorted = c[i - 1] < c[i];
  if (sorted) return;
  scratch.resize(static_cast<size_t>(len));
  for (index_t i = 0; i < len; ++i) {
    std::uint32_t bits;
    std::memcpy(&bits, &v[i], 4);
    scratch[i] = (static_cast<std::uint64_t>(static_cast<std::uint32_t>(c[i])) << 32) | bits;
  }
  std::sort(scratch.begin(), scratch.end());
  for (index_t i = 0; i < len; ++i) {
    c[i] = static_cast<std::int32_t>(scratch[i] >> 32);
    const std::uint32_t bits = static_cast<std::uint32_t>(scratch[i]);
    std::memcpy(&v[i], &bits, 4);
  }
}

// rowgcn::permute_graph (inc/partition.hpp:101-116): a'(pi(u), pi(v)) = a(u, v), rows sorted by column.
// from_coo's sort + merge reduces to a per-row sort because a valid CSR has no duplicate entries.
G32 permute_graph(const Csr& a, const std::vector<index_t>& fwd) {
  G32 out;
  out.n = a.rows;
  out.rp.assign(a.rows + 1, 0);
  for (index_t u = 0; u < a.rows; ++u) out.rp[fwd[u] + 1] = a.row_ptr[u + 1] - a.row_ptr[u];
  exclusive_scan_inplace(out.rp);
  out.ci.resize(a.nnz());
  out.v.resize(a.nnz());
  parallel_for(a.rows, [&](index_t b, index_t e) {
    std::vector<std::uint64_t> scratch;
    for (index_t u = b; u < e; ++u) {
      index_t pos = out.rp[fwd[u]];
      const index_t start = pos;
      for (index_t k = a.row_ptr[u]; k < a.row_ptr[u + 1]; ++k, ++pos) {
        out.ci[pos] = static_cast<std::int32_t>(fwd[a.col_idx[k]]);
        out.v[pos] = a.values[k];
      }
      sort_row(out.ci.data() + start, out.v.data() + start, pos - start, scratch);
    }
  }, 1024);
  return out;
}

G32 copy_graph(const Csr& a) {
  G32 out;
  out.n = a.rows;
  out.rp = a.row_ptr;
  out.ci.resize(a.nnz());
  out.v = a.values;
  parallel_for(a.nnz(), [&](index_t b, index_t e) {
    for (index_t k = b; k < e; ++k) out.ci[k] = static_cast<std::int32_t>(a.col_idx[k]);
  });
  return out;
}

// rowgcn::transpose (inc/sparse.hpp:110-129): stable counting sort; row v of the result lists its
// entries in increasing source row. Parallel version: per-chunk column histograms give every chunk
// its own write cursor per column, so the placement equals the sequential stable fill.
G32 transpose(const G32& a) {
  G32 t;
  t.n = a.n;
  t.rp.assign(a.n + 1, 0);
  t.ci.resize(a.nnz());
  t.v.resize(a.nnz());
  const int T = std::max(1, std::min<int>(host_threads(), static_cast<int>(a.n / 4096 + 1)));
  const index_t chunk = (a.n + T - 1) / T;
  std::vector<std::vector<std::int32_t>> cnt(T);
  {
    std::vector<std::thread> pool;
    for (int th = 0; th < T; ++th)
      pool.emplace_back([&, th] {
        cnt[th].assign(a.n, 0);
        const index_t b = std::min(a.n, th * chunk), e = std::min(a.n, (th + 1) * chunk);
        for (index_t k = a.rp[b]; k < a.rp[e]; ++k) cnt[th][a.ci[k]]++;
      });
    for (auto& p : pool) p.join();
  }
  for (index_t c = 0; c < a.n; ++c) {
    index_t s = 0;
    for (int th = 0; th < T; ++th) s += cnt[th][c];
    t.rp[c + 1] = s;
  }
  exclusive_scan_inplace(t.rp);
  // convert counts to per-chunk cursors: cursor[th][c] = rp[c] + sum_{th' < th} cnt[th'][c]
  std::vector<std::vector<index_t>> cur(T);
  parallel_for(T, [&](index_t b, index_t e) {
    for (index_t th = b; th < e; ++th) cur[th].assign(a.n, 0);
  }, 1);
  parallel_for(a.n, [&](index_t b, index_t e) {
    for (index_t c = b; c < e; ++c) {
      index_t s = t.rp[c];
      for (int th = 0; th < T; ++th) {
        cur[th][c] = s;
        s += cnt[th][c];
      }
    }
  });
  cnt.clear();
  {
    std::vector<std::thread> pool;
    for (int th = 0; th < T; ++th)
      pool.emplace_back([&, th] {
        const index_t b = std::min(a.n, th * chunk), e = std::min(a.n, (th + 1) * chunk);
        auto& cu = cur[th];
        for (index_t u = b; u < e; ++u)
          for (index_t k = a.rp[u]; k < a.rp[u + 1]; ++k) {
            const index_t pos = cu[a.ci[k]]++;
            t.ci[pos] = static_cast<std::int32_t>(u);
            t.v[pos] = a.v[k];
          }
      });
    for (auto& p : pool) p.join();
  }
  return t;
}

// rowgcn::tile_rows (inc/partition.hpp:173-225) for row block i of `a`: every row's sorted columns
// split at the part bounds; local column = v - begin(j).
std::vector<Tile> tile_row_block(const G32& a, const std::vector<index_t>& bounds, int i) {
  const int P = static_cast<int>(bounds.size()) - 1;
  const index_t r0 = bounds[i], r1 = bounds[i + 1], rows = r1 - r0;
  std::vector<Tile> tiles(P);
  // split[u][j] = first entry of row u with column >= bounds[j]; (rows) x (P + 1)
  std::vector<index_t> split(static_cast<size_t>(rows) * (P + 1));
  parallel_for(rows, [&](index_t b, index_t e) {
    for (index_t r = b; r < e; ++r) {
      const index_t u = r0 + r;
      const std::int32_t* beg = a.ci.data() + a.rp[u];
      const std::int32_t* end = a.ci.data() + a.rp[u + 1];
      index_t* s = &split[static_cast<size_t>(r) * (P + 1)];
      for (int j = 0; j < P; ++j)
        s[j] = a.rp[u] + (std::lower_bound(beg, end, static_cast<std::int32_t>(bounds[j])) - beg);
      s[P] = a.rp[u + 1];
    }
  });
  for (int j = 0; j < P; ++j) {
    Tile& t = tiles[j];
    t.rows = rows;
    t.cols = bounds[j + 1] - bounds[j];
    t.row_ptr.assign(rows + 1, 0);
    for (index_t r = 0; r < rows; ++r) {
      const index_t* s = &split[static_cast<size_t>(r) * (P + 1)];
      t.row_ptr[r + 1] = t.row_ptr[r] + (s[j + 1] - s[j]);
    }
    t.col.resize(t.row_ptr[rows]);
    t.val.resize(t.row_ptr[rows]);
    const std::int32_t base = static_cast<std::int32_t>(bounds[j]);
    parallel_for(rows, [&](index_t b, index_t e) {
      for (index_t r = b; r < e; ++r) {
        const index_t* s = &split[static_cast<size_t>(r) * (P + 1)];
        index_t pos = t.row_ptr[r];
        for (index_t k = s[j]; k < s[j + 1]; ++k, ++pos) {
          t.col[pos] = a.ci[k] - base;
          t.val[pos] = a.v[k];
        }
      }
    });
  }
  return tiles;
}

}  // namespace

// rowgcn::random_permutation (inc/partition.hpp:69-79)
void random_permutation(index_t n, std::uint64_t seed, std::vector<index_t>& forward) {
  std::vector<index_t> inverse(n);
  std::iota(inverse.begin(), inverse.end(), index_t(0));
  Rng rng(seed);
  for (index_t i = n - 1; i > 0; --i) {
    const index_t j = static_cast<index_t>(rng.below(static_cast<std::uint64_t>(i) + 1));
    std::swap(inverse[i], inverse[j]);
  }
  forward.assign(n, 0);
  for (index_t i = 0; i < n; ++i) forward[inverse[i]] = i;
}

}  // namespace mg

using namespace mg;

// ======================================================================== C ABI (host half)
// Dataset::validate (inc/dataset.hpp:30-44)
void mg::validate_dataset_named(const mg_dataset& ds) {
  ds.graph.validate();
  const std::string who = "dataset " + ds.name + ": ";
  if (ds.graph.rows != ds.graph.cols)
    throw ShapeError(who + "adjacency is " + shape_str(ds.graph.rows, ds.graph.cols) + ", expected square");
  if (ds.feature_rows != ds.graph.rows)
    throw ShapeError(who + "features have " + std::to_string(ds.feature_rows) + " rows but graph has " +
                     std::to_string(ds.graph.rows) + " vertices");
  if (static_cast<index_t>(ds.labels.size()) != ds.graph.rows)
    throw ShapeError(who + std::to_string(ds.labels.size()) + " labels but graph has " +
                     std::to_string(ds.graph.rows) + " vertices");
  if (!ds.train_mask.empty() && static_cast<index_t>(ds.train_mask.size()) != ds.graph.rows)
    throw ShapeError(who + "train mask length " + std::to_string(ds.train_mask.size()) + " != n " +
                     std::to_string(ds.graph.rows));
}
extern "C" {

const char* mg_last_error(void) { return g_last_error.c_str(); }
int32_t mg_abi_version(void) { return MG_ABI_VERSION; }

void mg_config_defaults(mg_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->lr = 0.01;
  c->beta1 = 0.9;
  c->beta2 = 0.999;
  c->epsilon = 1e-8;
  c->epochs = 100;
  c->seed = 1;
  c->gemm_mode = MG_GEMM_TF32X3;
  c->spmm_mode = MG_SPMM_FAST;
  c->aggregate_input = 1;
}

mg_status mg_config_validate(const mg_config* cfg) {
  return guarded([&] { (void)to_config(cfg); });
}

// rowgcn::synth_graph<float> (inc/dataset.hpp:287-334). The RNG stream is consumed in exactly the
// reference's order (stub draws row by row, then features, then labels); the sort + unique of the
// symmetric pair list is done per source row in parallel, which yields the same sorted set.
mg_status mg_dataset_synth(int64_t n, double avg_degree, double exponent, uint64_t seed, int64_t feature_dim,
                           int32_t classes, mg_dataset** out) {
  return guarded([&] {
    if (!out) throw ValueError("synth_graph: out is null");
    if (n < 2) throw ValueError("synth_graph: need n >= 2");
    if (avg_degree < 1.0) throw ValueError("synth_graph: need avg_degree >= 1");
    if (avg_degree >= static_cast<double>(n - 1))
      throw ValueError("synth_graph: avg_degree " + std::to_string(avg_degree) + " infeasible for n=" +
                       std::to_string(n));
    if (classes < 1) throw ValueError("synth_graph: classes must be >= 1");
    if (n >= (index_t(1) << 31)) throw ValueError("synth_graph: n >= 2^31 not supported by the host generator");
    Rng rng(seed);
    std::vector<double> weight(n);
    double wsum = 0;
    for (index_t u = 0; u < n; ++u) {
      weight[u] = std::pow(static_cast<double>(u + 1), -exponent);
      wsum += weight[u];
    }
    const double stubs_total = avg_degree * static_cast<double>(n) / 2.0;
    // stubs of row u are sv[so[u] .. so[u+1])
    std::vector<index_t> so(n + 1, 0);
    std::vector<std::int32_t> sv;
    sv.reserve(static_cast<size_t>(stubs_total * 1.05) + 16);
    for (index_t u = 0; u < n; ++u) {
      const double exact = stubs_total * weight[u] / wsum;
      index_t k = static_cast<index_t>(exact);
      if (rng.uniform() < exact - static_cast<double>(k)) ++k;
      k = std::min<index_t>(k, n - 1);
      for (index_t t = 0; t < k; ++t) {
        const index_t v = static_cast<index_t>(rng.below(static_cast<std::uint64_t>(n)));
        if (v == u) continue;
        sv.push_back(static_cast<std::int32_t>(v));
      }
      so[u + 1] = static_cast<index_t>(sv.size());
    }
    std::vector<double>().swap(weight);
    // symmetric bucket: row u holds its own stubs then the reverse of every stub targeting u
    std::vector<index_t> start(n + 1, 0);
    for (index_t u = 0; u < n; ++u) start[u + 1] += so[u + 1] - so[u];
    for (std::int32_t v : sv) start[v + 1]++;
    exclusive_scan_inplace(start);
    std::vector<std::int32_t> adj(start[n]);
    std::vector<index_t> fill(n);
    parallel_for(n, [&](index_t b, index_t e) {
      for (index_t u = b; u < e; ++u) {
        index_t p = start[u];
        for (index_t k = so[u]; k < so[u + 1]; ++k) adj[p++] = sv[k];
        fill[u] = p;
      }
    });
    for (index_t u = 0; u < n; ++u)
      for (index_t k = so[u]; k < so[u + 1]; ++k) adj[fill[sv[k]]++] = static_cast<std::int32_t>(u);
    std::vector<std::int32_t>().swap(sv);
    std::vector<index_t>().swap(so);
    std::vector<index_t> uniq(n + 1, 0);
    parallel_for(n, [&](index_t b, index_t e) {
      for (index_t u = b; u < e; ++u) {
        std::int32_t* row = adj.data() + start[u];
        const index_t len = start[u + 1] - start[u];
        std::sort(row, row + len);
        index_t w = 0;
        for (index_t i = 0; i < len; ++i)
          if (w == 0 || row[i] != row[w - 1]) row[w++] = row[i];
        uniq[u + 1] = w;
      }
    }, 256);
    exclusive_scan_inplace(uniq);
    auto ds = std::make_unique<mg_dataset>();
    ds->graph.rows = ds->graph.cols = n;
    ds->graph.row_ptr = uniq;
    ds->graph.col_idx.resize(uniq[n]);
    ds->graph.values.assign(uniq[n], 1.0f);
    parallel_for(n, [&](index_t b, index_t e) {
      for (index_t u = b; u < e; ++u)
        for (index_t i = 0; i < uniq[u + 1] - uniq[u]; ++i) ds->graph.col_idx[uniq[u] + i] = adj[start[u] + i];
    });
    ds->d0 = feature_dim;
    ds->feature_rows = n;
    ds->name = "synth-n" + std::to_string(n) + "-d" + std::to_string(avg_degree);  // dataset.hpp:326
    ds->features.resize(static_cast<size_t>(n * feature_dim));
    for (auto& x : ds->features) x = static_cast<float>(rng.uniform(-1.0, 1.0));
    ds->labels.resize(n);
    for (auto& l : ds->labels) l = static_cast<std::int32_t>(rng.below(static_cast<std::uint64_t>(classes)));
    *out = ds.release();
  });
}

mg_status mg_dataset_from_arrays(const mg_csr* graph, const float* features, int64_t d0, const int32_t* labels,
                                 const uint8_t* train_mask, mg_dataset** out) {
  return guarded([&] {
    if (!graph || !out || !graph->row_ptr) throw ValueError("dataset: null argument");
    auto ds = std::make_unique<mg_dataset>();
    const index_t n = graph->rows;
    if (n < 0 || d0 < 0) throw ValueError("dataset: negative dimension");
    ds->graph.rows = n;
    ds->graph.cols = graph->cols;
    ds->graph.row_ptr.assign(graph->row_ptr, graph->row_ptr + n + 1);
    const index_t nnz = ds->graph.row_ptr[n];
    if (nnz < 0) throw ValueError("csr: row_ptr[rows] < 0");
    ds->graph.col_idx.assign(graph->col_idx, graph->col_idx + nnz);
    ds->graph.values.assign(graph->values, graph->values + nnz);
    ds->d0 = d0;
    ds->feature_rows = n;
    ds->features.assign(features, features + n * d0);
    ds->labels.assign(labels, labels + n);
    if (train_mask) ds->train_mask.assign(train_mask, train_mask + n);
    *out = ds.release();
  });
}

mg_status mg_dataset_view(const mg_dataset* ds, mg_csr* graph, const float** features, int64_t* d0,
                          const int32_t** labels, const uint8_t** train_mask) {
  return guarded([&] {
    if (!ds) throw ValueError("dataset: null");
    if (graph) {
      graph->rows = ds->graph.rows;
      graph->cols = ds->graph.cols;
      graph->row_ptr = ds->graph.row_ptr.data();
      graph->col_idx = ds->graph.col_idx.data();
      graph->values = ds->graph.values.data();
    }
    if (features) *features = ds->features.data();
    if (d0) *d0 = ds->d0;
    if (labels) *labels = ds->labels.data();
    if (train_mask) *train_mask = ds->train_mask.empty() ? nullptr : ds->train_mask.data();
  });
}

int32_t mg_dataset_num_classes(const mg_dataset* ds) {
  std::int32_t c = 0;
  for (auto l : ds->labels) c = std::max(c, l);
  return c + 1;
}

static void validate_dataset(const mg_dataset& ds) { mg::validate_dataset_named(ds); }

mg_status mg_dataset_validate(const mg_dataset* ds) {
  return guarded([&] {
    if (!ds) throw ValueError("dataset: null");
    validate_dataset(*ds);
  });
}

void mg_dataset_free(mg_dataset* ds) { delete ds; }

// rowgcn::prepare_data (inc/driver.hpp:87-117)
mg_status mg_prepare(const mg_dataset* ds, const mg_config* cfgp, int32_t workers, int32_t only_rank,
                     mg_partition** out) {
  return guarded([&] {
    if (!ds || !out) throw ValueError("prepare: null argument");
    const Config cfg = to_config(cfgp);
    if (cfg.dims.front() != ds->d0)
      throw ConfigError("config: layer_dims[0]=" + std::to_string(cfg.dims.front()) +
                        " but dataset features have width " + std::to_string(ds->d0));
    if (workers <= 0) throw ValueError("uniform_partition: P must be >= 1, got " + std::to_string(workers));
    if (only_rank >= workers) throw ValueError("prepare: only_rank " + std::to_string(only_rank) + " >= P");
    validate_dataset(*ds);
    const index_t n = ds->n(), d0 = ds->d0;
    if (n >= (index_t(1) << 31)) throw ValueError("prepare: n >= 2^31 not supported");
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
        p->mask[v] = ds->train_mask.empty() ? 1 : ds->train_mask[u];  // effective_mask (dataset.hpp:46-49)
      }
    });
    for (auto m : p->mask) p->mask_count += m ? 1 : 0;
    if (p->mask_count == 0) throw ValueError("training mask is empty");
    p->bounds.resize(workers + 1);  // uniform_partition (partition.hpp:42-49)
    for (int i = 0; i <= workers; ++i) p->bounds[i] = static_cast<index_t>(i) * n / workers;

    G32 a = cfg.permute ? permute_graph(ds->graph, fwd) : copy_graph(ds->graph);
    G32 at = transpose(a);
    // normalize_in_degree (sparse.hpp:94-107): col_sum[v] accumulated over A's entries of column v in
    // increasing row order == row v of the stable transpose, summed left to right.
    std::vector<float> col_sum(n, 0.0f);
    parallel_for(n, [&](index_t b, index_t e) {
      for (index_t v = b; v < e; ++v) {
        float s = 0.0f;
        for (index_t k = at.rp[v]; k < at.rp[v + 1]; ++k) s += at.v[k];
        col_sum[v] = s;
      }
    });
    parallel_for(n, [&](index_t b, index_t e) {
      for (index_t u = b; u < e; ++u) {
        for (index_t k = a.rp[u]; k < a.rp[u + 1]; ++k) {
          const float s = col_sum[a.ci[k]];
          a.v[k] = s != 0.0f ? a.v[k] / s : 0.0f;
        }
        const float s = col_sum[u];  // row u of A^T holds column u of A
        for (index_t k = at.rp[u]; k < at.rp[u + 1]; ++k) at.v[k] = s != 0.0f ? at.v[k] / s : 0.0f;
      }
    });
    for (int d = 0; d < 2; ++d) p->tiles[d].resize(workers);
    for (int i = 0; i < workers; ++i) {
      if (!p->has_row(i)) continue;
      p->tiles[0][i] = tile_row_block(at, p->bounds, i);  // forward tiles of A_hat^T
      p->tiles[1][i] = tile_row_block(a, p->bounds, i);   // backward tiles of A_hat
    }
    *out = p.release();
  });
}

mg_status mg_partition_info(const mg_partition* p, int64_t* n, int64_t* mask_count, int64_t* bounds) {
  return guarded([&] {
    if (!p) throw ValueError("partition: null");
    if (n) *n = p->n;
    if (mask_count) *mask_count = p->mask_count;
    if (bounds) std::copy(p->bounds.begin(), p->bounds.end(), bounds);
  });
}

static const Tile& get_tile(const mg_partition* p, int32_t dir, int32_t i, int32_t j) {
  if (!p) throw ValueError("partition: null");
  if (dir < 0 || dir > 1) throw ValueError("partition: dir must be 0 or 1");
  if (i < 0 || i >= p->parts || j < 0 || j >= p->parts)
    throw ValueError("partition: tile (" + std::to_string(i) + ", " + std::to_string(j) + ") out of range");
  if (!p->has_row(i)) throw ValueError("partition: row block " + std::to_string(i) + " was not built");
  return p->tiles[dir][i][j];
}

mg_status mg_partition_tile_info(const mg_partition* p, int32_t dir, int32_t i, int32_t j, int64_t* rows,
                                 int64_t* cols, int64_t* nnz) {
  return guarded([&] {
    const Tile& t = get_tile(p, dir, i, j);
    if (rows) *rows = t.rows;
    if (cols) *cols = t.cols;
    if (nnz) *nnz = t.nnz();
  });
}

mg_status mg_partition_tile_export(const mg_partition* p, int32_t dir, int32_t i, int32_t j, int64_t* row_ptr,
                                   int64_t* col_idx, float* values) {
  return guarded([&] {
    const Tile& t = get_tile(p, dir, i, j);
    if (row_ptr) std::copy(t.row_ptr.begin(), t.row_ptr.end(), row_ptr);
    if (col_idx)
      for (index_t k = 0; k < t.nnz(); ++k) col_idx[k] = t.col[k];
    if (values) std::copy(t.val.begin(), t.val.end(), values);
  });
}

mg_status mg_partition_rows_export(const mg_partition* p, float* features, int32_t* labels, uint8_t* mask,
                                   int64_t* perm_forward) {
  return guarded([&] {
    if (!p) throw ValueError("partition: null");
    if (features) std::copy(p->features.begin(), p->features.end(), features);
    if (labels) std::copy(p->labels.begin(), p->labels.end(), labels);
    if (mask) std::copy(p->mask.begin(), p->mask.end(), mask);
    if (perm_forward) std::copy(p->perm_forward.begin(), p->perm_forward.end(), perm_forward);
  });
}

mg_status mg_partition_rows_info(const mg_partition* p, int64_t* row0, int64_t* rows) {
  return guarded([&] {
    if (!p) throw ValueError("partition: null");
    if (row0) *row0 = p->row0;
    if (rows) *rows = p->rows_stored();
  });
}

void mg_partition_free(mg_partition* p) { delete p; }

}  // extern "C"
