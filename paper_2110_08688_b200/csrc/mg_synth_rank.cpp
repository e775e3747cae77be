// SPDX-License-Identifier: Apache-2.0
// Per-rank synthetic input path for papers scale: rowgcn::synth_graph
// (inc/dataset.hpp:287-334) followed by rowgcn::prepare_data (inc/driver.hpp:87-117) for ONE row block of a
// P-way job, without the whole graph or all features in one process.
//
// What a rank needs from the reference's pipeline, and where it comes from here:
//   * the stub stream: every rank replays the generator's mt19937_64 stream (one uniform per vertex for
//     the stochastic rounding, then k uniform targets); the raw stubs (u -> v, v != u) are kept as one
//     int32 per stub (6.4 GB at 1.6 B stubs), grouped by u as they are drawn;
//   * its rows of P·A·P^T: the symmetrised pair list of the reference ((u, v) and (v, u) per stub, sorted,
//     unique, permuted) restricted to the rows the rank owns is, row by row, the sorted unique set of
//     fwd[v] over the stubs (u, v) and (v, u) with fwd[u] in the block — bucketed with atomic cursors,
//     then every row sorted and deduplicated (the order of the bucket fill does not matter);
//   * normalize_in_degree (inc/sparse.hpp:94-107): every value of A is 1, so column v's float sum is its
//     entry count = deg(v), the row length of v in the symmetric matrix. Forward tiles (A_hat^T) of row u
//     carry 1/deg(u), known locally; backward tiles (A_hat) carry 1/deg(v) for every column v, the one
//     thing a rank needs from the others (an all-gather of n int32, or P local block passes);
//   * features and labels: drawn after all stubs, n x d0 uniforms then n label draws; the rank keeps the
//     rows it owns and discards the rest of the stream (state twists only).
// Bit-identical to row block `rank` of the reference's prepare_data(synth_graph(...)) (tests/test_synth_rank.py
// against digests of the compiled reference, tests/golden/make_scale_golden.py c5s64).
#include <atomic>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>

#include "mg_internal.hpp"

using namespace mg;

struct mg_synth_rank {
  index_t n = 0, d0 = 0;
  int classes = 0, P = 1, rank = 0;
  bool graph_only = false, finished = false;
  std::vector<index_t> bounds;
  std::vector<index_t> fwd;       // permutation forward map (partition.hpp:69-79)
  std::vector<index_t> so;        // stubs of original vertex u: sv[so[u] .. so[u+1])
  std::vector<std::int32_t> sv;   // stub targets in draw order (v != u), relabelled to fwd[v] once drawn
  std::vector<index_t> rp;        // the rank's rows (permuted ids bounds[rank] ..): sorted unique columns
  std::vector<std::int32_t> ci;
  UploadVec<float> features;      // rows x d0
  std::vector<std::int32_t> labels;
  index_t row0() const { return bounds[rank]; }
  index_t rows() const { return bounds[rank + 1] - bounds[rank]; }
};

namespace {

// f(s, e) over [0, total) in chunks of `chunk`, claimed dynamically by host_threads() workers (the stub
// store is power-law skewed by vertex id: static splits over vertices leave one thread most of the work).
void dynamic_for(index_t total, index_t chunk, const std::function<void(index_t, index_t)>& f) {
  std::atomic<index_t> next{0};
  parallel_for(host_threads(), [&](index_t, index_t) {
    for (index_t s; (s = next.fetch_add(chunk)) < total;) f(s, std::min(total, s + chunk));
  }, 1);
}

// Every stub k in [s, e) with its drawing vertex u (so[u] <= k < so[u+1]): g(u, k_begin, k_end) per run.
template <class G>
void stub_runs(const mg_synth_rank& h, index_t s, index_t e, G&& g) {
  const index_t* so = h.so.data();
  index_t u = std::upper_bound(so, so + h.n + 1, s) - so - 1;
  for (index_t k = s; k < e; ++u) {
    const index_t ke = std::min(e, so[u + 1]);
    if (ke > k) g(u, k, ke);
    k = std::max(k, ke);
  }
}

// Rows bounds[b] .. bounds[b+1] of the permuted symmetric adjacency: sorted unique permuted columns.
void build_block(const mg_synth_rank& h, int b, std::vector<index_t>& rp, std::vector<std::int32_t>& ci) {
  const index_t b0 = h.bounds[b], b1 = h.bounds[b + 1], rows = b1 - b0;
  const index_t stubs = h.so[h.n];
  constexpr index_t kChunk = index_t(1) << 20;
  const index_t* fwd = h.fwd.data();
  const std::int32_t* sv = h.sv.data();
  std::unique_ptr<std::atomic<index_t>[]> cur(new std::atomic<index_t>[rows + 1]);
  parallel_for(rows + 1, [&](index_t s, index_t e) {
    for (index_t r = s; r < e; ++r) cur[r].store(0, std::memory_order_relaxed);
  });
  auto in_block = [b0, b1](index_t x) { return x >= b0 && x < b1; };
  // count: row fu gets fv for its own stubs, row fv gets fu for every stub (u, v)
  dynamic_for(stubs, kChunk, [&](index_t s, index_t e) {
    stub_runs(h, s, e, [&](index_t u, index_t k0, index_t k1) {
      const index_t fu = fwd[u];
      if (in_block(fu)) cur[fu - b0 + 1].fetch_add(k1 - k0, std::memory_order_relaxed);
      for (index_t k = k0; k < k1; ++k)
        if (in_block(sv[k])) cur[sv[k] - b0 + 1].fetch_add(1, std::memory_order_relaxed);
    });
  });
  std::vector<index_t> raw(rows + 1, 0);
  for (index_t r = 0; r < rows; ++r) raw[r + 1] = raw[r] + cur[r + 1].load(std::memory_order_relaxed);
  parallel_for(rows, [&](index_t s, index_t e) {
    for (index_t r = s; r < e; ++r) cur[r].store(raw[r], std::memory_order_relaxed);
  });
  std::vector<std::int32_t> buf(static_cast<size_t>(raw[rows]));
  dynamic_for(stubs, kChunk, [&](index_t s, index_t e) {
    stub_runs(h, s, e, [&](index_t u, index_t k0, index_t k1) {
      const index_t fu = fwd[u];
      const bool mine = in_block(fu);
      index_t pos = mine ? cur[fu - b0].fetch_add(k1 - k0, std::memory_order_relaxed) : 0;
      for (index_t k = k0; k < k1; ++k) {
        const index_t fv = sv[k];
        if (mine) buf[pos++] = static_cast<std::int32_t>(fv);
        if (in_block(fv)) buf[cur[fv - b0].fetch_add(1, std::memory_order_relaxed)] = static_cast<std::int32_t>(fu);
      }
    });
  });
  cur.reset();
  // per row: sort + unique (the reference's std::sort + std::unique over the pair list, restricted to a row)
  std::vector<index_t> len(rows + 1, 0);
  dynamic_for(rows, 4096, [&](index_t s, index_t e) {
    for (index_t r = s; r < e; ++r) {
      std::int32_t* row = buf.data() + raw[r];
      const index_t l = raw[r + 1] - raw[r];
      std::sort(row, row + l);
      index_t w = 0;
      for (index_t i = 0; i < l; ++i)
        if (w == 0 || row[i] != row[w - 1]) row[w++] = row[i];
      len[r + 1] = w;
    }
  });
  rp.assign(rows + 1, 0);
  for (index_t r = 0; r < rows; ++r) rp[r + 1] = rp[r] + len[r + 1];
  ci.resize(static_cast<size_t>(rp[rows]));
  parallel_for(rows, [&](index_t s, index_t e) {
    for (index_t r = s; r < e; ++r) std::memcpy(ci.data() + rp[r], buf.data() + raw[r], sizeof(std::int32_t) * (rp[r + 1] - rp[r]));
  }, 1024);
}

void row_lengths(const std::vector<index_t>& rp, std::int32_t* out) {
  for (size_t r = 0; r + 1 < rp.size(); ++r) out[r] = static_cast<std::int32_t>(rp[r + 1] - rp[r]);
}

}  // namespace

extern "C" {

mg_status mg_synth_rank_open(int64_t n, double avg_degree, double exponent, uint64_t seed, int64_t feature_dim,
                             int32_t classes, const mg_config* cfgp, int32_t workers, int32_t rank, int32_t flags,
                             mg_synth_rank** out) {
  return guarded([&] {
    if (!out) throw ValueError("synth_graph: out is null");
    // synth_graph's argument checks (dataset.hpp:290-295), then prepare_data's (driver.hpp:87-117)
    if (n < 2) throw ValueError("synth_graph: need n >= 2");
    if (avg_degree < 1.0) throw ValueError("synth_graph: need avg_degree >= 1");
    if (avg_degree >= static_cast<double>(n - 1))
      throw ValueError("synth_graph: avg_degree " + std::to_string(avg_degree) + " infeasible for n=" +
                       std::to_string(n));
    if (classes < 1) throw ValueError("synth_graph: classes must be >= 1");
    if (n >= (index_t(1) << 31)) throw ValueError("synth_graph: n >= 2^31 not supported by the host generator");
    const Config cfg = to_config(cfgp);
    if (cfg.dims.front() != feature_dim)
      throw ConfigError("config: layer_dims[0]=" + std::to_string(cfg.dims.front()) +
                        " but dataset features have width " + std::to_string(feature_dim));
    if (workers <= 0) throw ValueError("uniform_partition: P must be >= 1, got " + std::to_string(workers));
    if (rank < 0 || rank >= workers)
      throw ValueError("synth_rank: rank " + std::to_string(rank) + " out of range for P=" + std::to_string(workers));
    auto h = std::make_unique<mg_synth_rank>();
    h->n = n;
    h->d0 = feature_dim;
    h->classes = classes;
    h->P = workers;
    h->rank = rank;
    h->graph_only = (flags & MG_SYNTH_GRAPH_ONLY) != 0;
    h->bounds.resize(workers + 1);  // uniform_partition (partition.hpp:42-49)
    for (int i = 0; i <= workers; ++i) h->bounds[i] = static_cast<index_t>(i) * n / workers;
    if (cfg.permute) {
      random_permutation(n, cfg.seed, h->fwd);
    } else {
      h->fwd.resize(n);
      std::iota(h->fwd.begin(), h->fwd.end(), index_t(0));
    }
    // the stub stream (dataset.hpp:296-318), drawn exactly as the reference draws it
    Rng rng(seed);
    std::vector<double> weight(n);
    double wsum = 0;
    for (index_t u = 0; u < n; ++u) {
      weight[u] = std::pow(static_cast<double>(u + 1), -exponent);
      wsum += weight[u];
    }
    const double stubs_total = avg_degree * static_cast<double>(n) / 2.0;
    h->so.assign(n + 1, 0);
    h->sv.reserve(static_cast<size_t>(stubs_total * 1.02) + 16);
    for (index_t u = 0; u < n; ++u) {
      const double exact = stubs_total * weight[u] / wsum;
      index_t k = static_cast<index_t>(exact);
      if (rng.uniform() < exact - static_cast<double>(k)) ++k;
      k = std::min<index_t>(k, n - 1);
      for (index_t t = 0; t < k; ++t) {
        const index_t v = static_cast<index_t>(rng.below(static_cast<std::uint64_t>(n)));
        if (v == u) continue;
        h->sv.push_back(static_cast<std::int32_t>(v));
      }
      h->so[u + 1] = static_cast<index_t>(h->sv.size());
    }
    std::vector<double>().swap(weight);
    // every later pass reads stubs by their permuted ids only: relabel once (one parallel gather) so the
    // block passes stream the stub store instead of gathering fwd[] per stub
    {
      std::int32_t* sv = h->sv.data();
      const index_t* fwd = h->fwd.data();
      parallel_for(static_cast<index_t>(h->sv.size()), [&](index_t s, index_t e) {
        for (index_t k = s; k < e; ++k) sv[k] = static_cast<std::int32_t>(fwd[sv[k]]);
      }, 1 << 20);
    }
    build_block(*h, rank, h->rp, h->ci);
    if (!h->graph_only) {
      // features (n x d0 uniforms in [-1, 1)) then labels (n draws), dataset.hpp:327-331; permute_rows /
      // permute_values (partition.hpp:118-140) place original row u at fwd[u]
      const index_t b0 = h->row0(), b1 = b0 + h->rows(), d0 = feature_dim;
      h->features.resize(static_cast<size_t>(h->rows() * d0));
      for (index_t u = 0; u < n; ++u) {
        const index_t f = h->fwd[u];
        if (f >= b0 && f < b1) {
          float* x = h->features.data() + (f - b0) * d0;
          for (index_t c = 0; c < d0; ++c) x[c] = static_cast<float>(rng.uniform(-1.0, 1.0));
        } else {
          rng.discard(static_cast<std::uint64_t>(d0));
        }
      }
      h->labels.resize(h->rows());
      for (index_t u = 0; u < n; ++u) {
        const index_t f = h->fwd[u];
        if (f >= b0 && f < b1)
          h->labels[f - b0] = static_cast<std::int32_t>(rng.below(static_cast<std::uint64_t>(classes)));
        else
          rng.discard(1);
      }
    }
    *out = h.release();
  });
}

mg_status mg_synth_rank_info(const mg_synth_rank* h, int64_t* row0, int64_t* rows, int64_t* nnz, int64_t* stubs) {
  return guarded([&] {
    if (!h) throw ValueError("synth_rank: null handle");
    if (row0) *row0 = h->row0();
    if (rows) *rows = h->rows();
    if (nnz) *nnz = h->rp.empty() ? 0 : h->rp.back();
    if (stubs) *stubs = h->so.empty() ? 0 : h->so.back();
  });
}

mg_status mg_synth_rank_degrees(const mg_synth_rank* h, int32_t* degrees) {
  return guarded([&] {
    if (!h || !degrees) throw ValueError("synth_rank: null argument");
    if (h->finished) throw ValueError("synth_rank: already finished");
    row_lengths(h->rp, degrees);
  });
}

mg_status mg_synth_rank_block_degrees(mg_synth_rank* h, int32_t block, int32_t* degrees) {
  return guarded([&] {
    if (!h || !degrees) throw ValueError("synth_rank: null argument");
    if (h->finished) throw ValueError("synth_rank: already finished");
    if (block < 0 || block >= h->P) throw ValueError("synth_rank: block " + std::to_string(block) + " out of range");
    if (block == h->rank) return row_lengths(h->rp, degrees);
    std::vector<index_t> rp;
    std::vector<std::int32_t> ci;
    build_block(*h, block, rp, ci);
    row_lengths(rp, degrees);
  });
}

mg_status mg_synth_rank_finish(mg_synth_rank* h, const int32_t* degrees, mg_partition** out) {
  return guarded([&] {
    if (!h || !out) throw ValueError("synth_rank: null argument");
    if (h->finished) throw ValueError("synth_rank: already finished");
    if (h->graph_only) throw ValueError("synth_rank: opened with MG_SYNTH_GRAPH_ONLY (no features)");
    const index_t n = h->n, b0 = h->row0(), rows = h->rows();
    std::vector<std::int32_t> deg;
    if (!degrees) {
      deg.resize(n);
      for (int b = 0; b < h->P; ++b) {
        const mg_status st = mg_synth_rank_block_degrees(h, b, deg.data() + h->bounds[b]);
        if (st != MG_OK) throw Error(st, mg_last_error());
      }
      degrees = deg.data();
    }
    for (index_t r = 0; r < rows; ++r)
      if (degrees[b0 + r] != h->rp[r + 1] - h->rp[r])
        throw ValueError("synth_rank: degree of vertex " + std::to_string(b0 + r) + " is " +
                         std::to_string(degrees[b0 + r]) + " in the exchanged degrees but " +
                         std::to_string(h->rp[r + 1] - h->rp[r]) + " in this rank's rows");
    // the sv / so stub store is no longer needed: release it before the tiles are built
    std::vector<std::int32_t>().swap(h->sv);
    std::vector<index_t>().swap(h->so);
    auto p = std::make_unique<mg_partition>();
    p->n = n;
    p->d0 = h->d0;
    p->parts = h->P;
    p->only_rank = h->rank;
    p->bounds = h->bounds;
    p->row0 = b0;
    p->mask_count = n;  // synth_graph sets no train mask: effective_mask is all ones (dataset.hpp:46-49)
    const int P = h->P;
    for (int d = 0; d < 2; ++d) p->tiles[d].resize(P);
    // tile_rows (partition.hpp:173-225) of A_hat^T (forward, value 1/deg(row)) and A_hat (backward,
    // value 1/deg(column)) for row block `rank`: the two share the symmetric structure
    std::vector<index_t> split(static_cast<size_t>(rows) * (P + 1));
    parallel_for(rows, [&](index_t s, index_t e) {
      for (index_t r = s; r < e; ++r) {
        const std::int32_t* beg = h->ci.data() + h->rp[r];
        const std::int32_t* end = h->ci.data() + h->rp[r + 1];
        index_t* sp = &split[static_cast<size_t>(r) * (P + 1)];
        for (int j = 0; j < P; ++j)
          sp[j] = h->rp[r] + (std::lower_bound(beg, end, static_cast<std::int32_t>(h->bounds[j])) - beg);
        sp[P] = h->rp[r + 1];
      }
    });
    for (int d = 0; d < 2; ++d) {
      auto& row_tiles = p->tiles[d][h->rank];
      row_tiles.resize(P);
      for (int j = 0; j < P; ++j) {
        Tile& t = row_tiles[j];
        t.rows = rows;
        t.cols = h->bounds[j + 1] - h->bounds[j];
        t.row_ptr.assign(rows + 1, 0);
        for (index_t r = 0; r < rows; ++r) {
          const index_t* sp = &split[static_cast<size_t>(r) * (P + 1)];
          t.row_ptr[r + 1] = t.row_ptr[r] + (sp[j + 1] - sp[j]);
        }
        t.col.resize(t.row_ptr[rows]);
        t.val.resize(t.row_ptr[rows]);
        const std::int32_t base = static_cast<std::int32_t>(h->bounds[j]);
        parallel_for(rows, [&](index_t s, index_t e) {
          for (index_t r = s; r < e; ++r) {
            const index_t* sp = &split[static_cast<size_t>(r) * (P + 1)];
            const float row_inv = 1.0f / static_cast<float>(degrees[b0 + r]);
            index_t pos = t.row_ptr[r];
            for (index_t k = sp[j]; k < sp[j + 1]; ++k, ++pos) {
              const std::int32_t c = h->ci[k];
              t.col[pos] = c - base;
              t.val[pos] = d == 0 ? row_inv : 1.0f / static_cast<float>(degrees[c]);
            }
          }
        });
      }
    }
    p->features = std::move(h->features);
    p->labels = std::move(h->labels);
    p->mask.assign(rows, 1);
    p->perm_forward = std::move(h->fwd);
    std::vector<index_t>().swap(h->rp);
    std::vector<std::int32_t>().swap(h->ci);
    h->finished = true;
    *out = p.release();
  });
}

void mg_synth_rank_free(mg_synth_rank* h) { delete h; }

}  // extern "C"
