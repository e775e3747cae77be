// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE ONLY — the checker, never the product.
//
// extern "C" shim over the UNMODIFIED reference headers (rowgcn, /root/reference/proj/include),
// compiled in place by oracle/build_ref.sh into oracle/_ref/librowgcn_ref.so with the reference's own
// Release flags (-O3 -DNDEBUG, no -march, so GCC emits no FMA). No reference source is
// copied into this repository: this file only calls the reference API.
//
// Entry points mirror what the parity tests need:
//   * dataset construction (synth_graph dataset.hpp:287-334, or caller arrays),
//   * prepare_data (driver.hpp:87-117) with tile/perm export,
//   * kernels: spmm (sparse.hpp:161-188), gemm (dense.hpp:140-204), softmax_xent_sum
//     (dense.hpp:241-277), adam_step (gcn.hpp:61-85),
//   * model: train_run (driver.hpp:140-206), grad_run (driver.hpp:216-251) and a teacher-forced
//     single step dump built from GcnWorker's public step pieces (gcn.hpp:238-362).
// Only tests/, bench.py's cpu_baseline/reference arm and __graft_entry__.smoke() load this library.

#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "rowgcn/breakdown.hpp"
#include "rowgcn/driver.hpp"
#include "rowgcn/timeline.hpp"

using namespace rowgcn;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ShapeError& e) {
    g_err = e.what();
    return 1;
  } catch (const ValueError& e) {
    g_err = e.what();
    return 2;
  } catch (const ProtocolError& e) {
    g_err = e.what();
    return 3;
  } catch (const ShutdownError& e) {
    g_err = e.what();
    return 4;
  } catch (const ParseError& e) {
    g_err = e.what();
    return 5;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 6;
  } catch (const IoError& e) {
    g_err = e.what();
    return 7;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 99;
  }
}

struct RefCfg {
  const int64_t* dims;
  int32_t n_dims;
  double lr, beta1, beta2, epsilon;
  int32_t epochs;
  uint64_t seed;
  uint8_t permute, overlap, skip_first_backward_spmm, order_swap;
};

GcnConfig to_cfg(const RefCfg* c) {
  GcnConfig cfg;
  cfg.layer_dims.assign(c->dims, c->dims + c->n_dims);
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
  return cfg;
}

template <class S>
CsrMatrix<S> csr_from(int64_t rows, int64_t cols, const int64_t* rp, const int64_t* ci, const S* v) {
  CsrMatrix<S> m;
  m.rows = rows;
  m.cols = cols;
  m.row_ptr.assign(rp, rp + rows + 1);
  const int64_t nnz = rp[rows];
  m.col_idx.assign(ci, ci + nnz);
  m.values.assign(v, v + nnz);
  return m;
}

template <class S>
Dataset<S>* ds_from_arrays(int64_t n, const int64_t* rp, const int64_t* ci, const S* v, int64_t d0,
                           const S* feats, const int32_t* labels, const uint8_t* mask) {
  auto* ds = new Dataset<S>();
  ds->name = "arrays";
  ds->graph = csr_from<S>(n, n, rp, ci, v);
  ds->features = DenseMatrix<S>(n, d0);
  std::memcpy(ds->features.data(), feats, sizeof(S) * static_cast<size_t>(n * d0));
  ds->labels.assign(labels, labels + n);
  if (mask) ds->train_mask.assign(mask, mask + n);
  return ds;
}

template <class S>
struct Shared {
  PreparedData<S> prep;
  GcnConfig cfg;
  typename GcnWorker<S>::Shared sh;
  Shared(const Dataset<S>& ds, const GcnConfig& c, int workers) : prep(prepare_data(ds, c, workers)), cfg(c) {
    sh.cfg = &cfg;
    sh.fwd_tiles = &prep.fwd_tiles;
    sh.bwd_tiles = &prep.bwd_tiles;
    sh.features = &prep.features;
    sh.labels = &prep.labels;
    sh.mask = &prep.mask;
    sh.global_mask_count = prep.mask_count;
    sh.wgrad_blocks = uniform_partition(ds.n(), 8);
  }
};

// Teacher-forced single train step (== GcnWorker::train_step(1), gcn.hpp:175-184, split into its
// public pieces so the intermediate tensors can be captured). All row-indexed outputs are gathered
// into global (permuted) row order.
template <class S>
int step_dump(const Dataset<S>* ds, const RefCfg* c, int workers, const S* w_init, S* ahw_fwd,
              S* loss_grad, S* ahw_bwd, S* hw_last, S* wgrad, S* w_after, double* loss) {
  return guarded([&] {
    const GcnConfig cfg = to_cfg(c);
    Shared<S> shared(*ds, cfg, workers);
    const int L = cfg.layers();
    const index_t n = ds->n();
    std::vector<index_t> act_off(L + 1, 0);
    for (int l = 0; l < L; ++l) act_off[l + 1] = act_off[l] + n * cfg.layer_dims[l + 1];
    index_t w_total = 0;
    for (int l = 0; l < L; ++l) w_total += cfg.layer_dims[l] * cfg.layer_dims[l + 1];
    std::vector<double> loss_r(workers, 0.0);
    DeviceGroup group(workers);
    group.run([&](WorkerCtx& ctx) {
      GcnWorker<S> w(ctx, shared.sh);
      w.init_params();
      if (w_init) {
        index_t off = 0;
        for (auto& p : w.params()) {
          std::memcpy(p.w.data(), w_init + off, sizeof(S) * p.w.size());
          off += p.w.size();
        }
      }
      const index_t r0 = w.row_begin(), rows = w.local_rows();
      auto gather = [&](S* dst, int l, const S* src) {
        const index_t d = cfg.layer_dims[l + 1];
        if (dst)
          for (index_t i = 0; i < rows; ++i)
            std::memcpy(dst + act_off[l] + (r0 + i) * d, src + i * d, sizeof(S) * d);
      };
      const S lo = w.loss_only();  // forward + loss (same arithmetic as softmax_xent_sum)
      if (ctx.rank() == 0) *loss = static_cast<double>(lo);
      // loss_only leaves the forward activations in the L+3 pool; reuse them for the step.
      for (int l = 0; l < L; ++l) gather(ahw_fwd, l, w.pool().ahw[l].data());
      const TaskId stats = w.submit_loss_grad();
      ctx.wait(stats);
      if (loss_grad) {
        const index_t C = cfg.layer_dims[L];
        for (index_t i = 0; i < rows; ++i)
          std::memcpy(loss_grad + (r0 + i) * C, w.logits_view().data + i * C, sizeof(S) * C);
      }
      w.submit_backward();
      ctx.wait(w.submit_finalize(false, 1));
      for (int l = 0; l < L; ++l) gather(ahw_bwd, l, w.pool().ahw[l].data());
      if (hw_last) {
        const index_t d = cfg.layer_dims[1];  // layer-0 backward SpMM output (meaningless with skip)
        for (index_t i = 0; i < rows; ++i)
          std::memcpy(hw_last + (r0 + i) * d, w.pool().hw.data() + i * d, sizeof(S) * d);
      }
      if (ctx.rank() == 0) {
        index_t off = 0;
        for (auto& p : w.params()) {
          if (wgrad) std::memcpy(wgrad + off, p.w_grad.data(), sizeof(S) * p.w_grad.size());
          off += p.w_grad.size();
        }
      }
      adam_step(w.params(), 1, cfg);
      if (ctx.rank() == 0) {
        index_t off = 0;
        for (auto& p : w.params()) {
          if (w_after) std::memcpy(w_after + off, p.w.data(), sizeof(S) * p.w.size());
          off += p.w.size();
        }
      }
    });
    (void)w_total;
  });
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_spmm_threads(int t) { spmm_threads() = t; }

// ---------------------------------------------------------------- datasets
#define DS_FUNCS(S, SUF)                                                                                   \
  void* ref_ds_synth_##SUF(int64_t n, double deg, double expo, uint64_t seed, int64_t d0, int32_t classes) { \
    Dataset<S>* out = nullptr;                                                                             \
    if (guarded([&] { out = new Dataset<S>(synth_graph<S>(n, deg, expo, seed, d0, classes)); })) return nullptr; \
    return out;                                                                                            \
  }                                                                                                        \
  void* ref_ds_from_arrays_##SUF(int64_t n, const int64_t* rp, const int64_t* ci, const S* v, int64_t d0,   \
                                 const S* feats, const int32_t* labels, const uint8_t* mask) {             \
    Dataset<S>* out = nullptr;                                                                             \
    if (guarded([&] { out = ds_from_arrays<S>(n, rp, ci, v, d0, feats, labels, mask); })) return nullptr;  \
    return out;                                                                                            \
  }                                                                                                        \
  void ref_ds_info_##SUF(void* h, int64_t* n, int64_t* nnz, int64_t* d0) {                                 \
    auto* ds = static_cast<Dataset<S>*>(h);                                                                \
    *n = ds->n();                                                                                          \
    *nnz = ds->graph.nnz();                                                                                \
    *d0 = ds->features.cols();                                                                             \
  }                                                                                                        \
  void ref_ds_export_##SUF(void* h, int64_t* rp, int64_t* ci, S* v, S* feats, int32_t* labels) {           \
    auto* ds = static_cast<Dataset<S>*>(h);                                                                \
    if (rp) std::memcpy(rp, ds->graph.row_ptr.data(), 8 * ds->graph.row_ptr.size());                       \
    if (ci) std::memcpy(ci, ds->graph.col_idx.data(), 8 * ds->graph.col_idx.size());                       \
    if (v) std::memcpy(v, ds->graph.values.data(), sizeof(S) * ds->graph.values.size());                   \
    if (feats) std::memcpy(feats, ds->features.data(), sizeof(S) * ds->features.size());                   \
    if (labels) std::memcpy(labels, ds->labels.data(), 4 * ds->labels.size());                             \
  }                                                                                                        \
  void ref_ds_free_##SUF(void* h) { delete static_cast<Dataset<S>*>(h); }

DS_FUNCS(float, f32)
DS_FUNCS(double, f64)

// ---------------------------------------------------------------- partitioner
int ref_random_permutation(int64_t n, uint64_t seed, int64_t* forward, int64_t* inverse) {
  return guarded([&] {
    const Permutation p = random_permutation(n, seed);
    if (forward) std::memcpy(forward, p.forward.data(), 8 * n);
    if (inverse) std::memcpy(inverse, p.inverse.data(), 8 * n);
  });
}

int ref_uniform_partition(int64_t n, int32_t parts, int64_t* bounds) {
  return guarded([&] {
    const PartitionVector p = uniform_partition(n, parts);
    std::memcpy(bounds, p.bounds.data(), 8 * p.bounds.size());
  });
}

void* ref_prepare_f32(void* ds, const RefCfg* c, int32_t workers) {
  PreparedData<float>* out = nullptr;
  if (guarded([&] {
        out = new PreparedData<float>(prepare_data(*static_cast<Dataset<float>*>(ds), to_cfg(c), workers));
      }))
    return nullptr;
  return out;
}
void ref_prep_free_f32(void* h) { delete static_cast<PreparedData<float>*>(h); }

void ref_prep_info_f32(void* h, int64_t* mask_count, int64_t* bounds) {
  auto* p = static_cast<PreparedData<float>*>(h);
  *mask_count = p->mask_count;
  std::memcpy(bounds, p->partition.bounds.data(), 8 * p->partition.bounds.size());
}

void ref_prep_tile_info_f32(void* h, int32_t dir, int32_t i, int32_t j, int64_t* rows, int64_t* cols, int64_t* nnz) {
  auto* p = static_cast<PreparedData<float>*>(h);
  const auto& t = (dir == 0 ? p->fwd_tiles : p->bwd_tiles).tiles[i][j];
  *rows = t.rows;
  *cols = t.cols;
  *nnz = t.nnz();
}

void ref_prep_tile_export_f32(void* h, int32_t dir, int32_t i, int32_t j, int64_t* rp, int64_t* ci, float* v) {
  auto* p = static_cast<PreparedData<float>*>(h);
  const auto& t = (dir == 0 ? p->fwd_tiles : p->bwd_tiles).tiles[i][j];
  std::memcpy(rp, t.row_ptr.data(), 8 * t.row_ptr.size());
  std::memcpy(ci, t.col_idx.data(), 8 * t.col_idx.size());
  std::memcpy(v, t.values.data(), 4 * t.values.size());
}

void ref_prep_rows_export_f32(void* h, float* feats, int32_t* labels, uint8_t* mask, int64_t* perm_fwd) {
  auto* p = static_cast<PreparedData<float>*>(h);
  if (feats) std::memcpy(feats, p->features.data(), 4 * p->features.size());
  if (labels) std::memcpy(labels, p->labels.data(), 4 * p->labels.size());
  if (mask) std::memcpy(mask, p->mask.data(), p->mask.size());
  if (perm_fwd) std::memcpy(perm_fwd, p->perm.forward.data(), 8 * p->perm.forward.size());
}

// ---------------------------------------------------------------- kernels (f32 and f64)
#define KERNEL_FUNCS(S, SUF)                                                                                \
  int ref_spmm_##SUF(int64_t rows, int64_t cols, const int64_t* rp, const int64_t* ci, const S* v,           \
                     const S* h, int64_t w, int32_t accumulate, S* out) {                                   \
    return guarded([&] {                                                                                    \
      const CsrMatrix<S> a = csr_from<S>(rows, cols, rp, ci, v);                                            \
      spmm<S>(a, CMatView<S>(h, cols, w), accumulate != 0, MatView<S>{out, rows, w});                       \
    });                                                                                                     \
  }                                                                                                         \
  int ref_gemm_##SUF(const S* a, int64_t ar, int64_t ac, const S* b, int64_t br, int64_t bc, int32_t ta,    \
                     int32_t tb, int32_t acc, S* out, int64_t orows, int64_t ocols) {                       \
    return guarded([&] {                                                                                    \
      gemm<S>(CMatView<S>(a, ar, ac), CMatView<S>(b, br, bc), ta != 0, tb != 0, acc != 0,                   \
              MatView<S>{out, orows, ocols});                                                               \
    });                                                                                                     \
  }                                                                                                         \
  int ref_softmax_xent_sum_##SUF(const S* logits, int64_t rows, int64_t cols, const int32_t* labels,        \
                                 const uint8_t* mask, S* grad, int64_t denom, double* loss_sum) {           \
    return guarded([&] {                                                                                    \
      const S r = softmax_xent_sum<S>(CMatView<S>(logits, rows, cols),                                      \
                                      std::span<const int32_t>(labels, rows),                               \
                                      std::span<const uint8_t>(mask, rows), MatView<S>{grad, rows, cols},   \
                                      denom);                                                               \
      *loss_sum = static_cast<double>(r);                                                                   \
    });                                                                                                     \
  }                                                                                                         \
  int ref_adam_##SUF(S* w, S* g, S* m, S* v, int64_t size, int32_t t, double lr, double b1, double b2,      \
                     double eps) {                                                                          \
    return guarded([&] {                                                                                    \
      std::vector<LayerParams<S>> ps;                                                                       \
      ps.push_back({DenseMatrix<S>(1, size), DenseMatrix<S>(1, size), DenseMatrix<S>(1, size),              \
                    DenseMatrix<S>(1, size)});                                                              \
      std::memcpy(ps[0].w.data(), w, sizeof(S) * size);                                                     \
      std::memcpy(ps[0].w_grad.data(), g, sizeof(S) * size);                                                \
      std::memcpy(ps[0].adam_m.data(), m, sizeof(S) * size);                                                \
      std::memcpy(ps[0].adam_v.data(), v, sizeof(S) * size);                                                \
      GcnConfig cfg;                                                                                        \
      cfg.layer_dims = {1, 1};                                                                              \
      cfg.lr = lr;                                                                                          \
      cfg.beta1 = b1;                                                                                       \
      cfg.beta2 = b2;                                                                                       \
      cfg.epsilon = eps;                                                                                    \
      adam_step(ps, t, cfg);                                                                                \
      std::memcpy(w, ps[0].w.data(), sizeof(S) * size);                                                     \
      std::memcpy(g, ps[0].w_grad.data(), sizeof(S) * size);                                                \
      std::memcpy(m, ps[0].adam_m.data(), sizeof(S) * size);                                                \
      std::memcpy(v, ps[0].adam_v.data(), sizeof(S) * size);                                                \
    });                                                                                                     \
  }

KERNEL_FUNCS(float, f32)
KERNEL_FUNCS(double, f64)

// ---------------------------------------------------------------- model entry points
#define MODEL_FUNCS(S, SUF)                                                                                 \
  int ref_train_run_##SUF(void* dsh, const RefCfg* c, int32_t workers, double* loss, double* acc,           \
                          double* wall_us, uint64_t* hashes, S* final_w, S* logits) {                       \
    return guarded([&] {                                                                                    \
      const auto& ds = *static_cast<Dataset<S>*>(dsh);                                                      \
      const GcnConfig cfg = to_cfg(c);                                                                      \
      TrainOptions opts;                                                                                    \
      opts.workers = workers;                                                                               \
      opts.collect_logits = logits != nullptr;                                                              \
      const auto art = train_run(ds, cfg, opts);                                                            \
      for (int e = 0; e < cfg.epochs; ++e) {                                                                \
        if (loss) loss[e] = art.epoch_loss[e];                                                              \
        if (acc) acc[e] = art.epoch_acc[e];                                                                 \
        if (wall_us) wall_us[e] = art.epoch_wall_us[e];                                                     \
        if (hashes)                                                                                         \
          for (int r = 0; r < workers; ++r) hashes[e * workers + r] = art.w_hashes[e][r];                   \
      }                                                                                                     \
      if (final_w) {                                                                                        \
        index_t off = 0;                                                                                    \
        for (const auto& w : art.final_w) {                                                                 \
          std::memcpy(final_w + off, w.data(), sizeof(S) * w.size());                                       \
          off += w.size();                                                                                  \
        }                                                                                                   \
      }                                                                                                     \
      if (logits) std::memcpy(logits, art.logits.data(), sizeof(S) * art.logits.size());                    \
    });                                                                                                     \
  }                                                                                                         \
  int ref_grad_run_##SUF(void* dsh, const RefCfg* c, int32_t workers, double* loss, S* wgrad,               \
                         uint64_t* hashes) {                                                                \
    return guarded([&] {                                                                                    \
      const auto art = grad_run(*static_cast<Dataset<S>*>(dsh), to_cfg(c), workers);                        \
      *loss = art.loss;                                                                                     \
      index_t off = 0;                                                                                      \
      for (const auto& g : art.w_grad) {                                                                    \
        std::memcpy(wgrad + off, g.data(), sizeof(S) * g.size());                                           \
        off += g.size();                                                                                    \
      }                                                                                                     \
      if (hashes)                                                                                           \
        for (int r = 0; r < workers; ++r) hashes[r] = art.grad_hash_per_rank[r];                            \
    });                                                                                                     \
  }                                                                                                         \
  int ref_step_dump_##SUF(void* dsh, const RefCfg* c, int32_t workers, const S* w_init, S* ahw_fwd,         \
                          S* loss_grad, S* ahw_bwd, S* hw_last, S* wgrad, S* w_after, double* loss) {       \
    return step_dump<S>(static_cast<Dataset<S>*>(dsh), c, workers, w_init, ahw_fwd, loss_grad, ahw_bwd,     \
                        hw_last, wgrad, w_after, loss);                                                     \
  }

MODEL_FUNCS(float, f32)
MODEL_FUNCS(double, f64)

uint64_t ref_fnv1a(const void* data, uint64_t len, uint64_t h) { return fnv1a(data, len, h); }

// write_checkpoint<float> (driver.hpp:255-274) and config_to_json(cfg).dump(indent) (driver.hpp:59-71).
int ref_write_checkpoint_f32(const char* path, int32_t count, const int64_t* rows, const int64_t* cols,
                             const float* const* data, const RefCfg* c) {
  return guarded([&] {
    std::vector<DenseMatrix<float>> ws;
    for (int32_t i = 0; i < count; ++i) {
      DenseMatrix<float> w(rows[i], cols[i]);
      std::memcpy(w.data(), data[i], sizeof(float) * static_cast<size_t>(rows[i] * cols[i]));
      ws.push_back(std::move(w));
    }
    write_checkpoint(path, ws, to_cfg(c));
  });
}
int ref_config_json(const RefCfg* c, int32_t indent, char* buf, int64_t cap, int64_t* len) {
  return guarded([&] {
    const std::string s = config_to_json(to_cfg(c)).dump(indent);
    *len = static_cast<int64_t>(s.size());
    if (buf && cap > 0) {
      const size_t n = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
  });
}
int ref_breakdown_json(const double* t, int32_t indent, char* buf, int64_t cap, int64_t* len) {
  return guarded([&] {
    BreakdownReport r;
    r.spmm_us = t[0];
    r.gemm_us = t[1];
    r.activation_us = t[2];
    r.loss_us = t[3];
    r.adam_us = t[4];
    r.comm_us = t[5];
    const std::string s = r.to_json().dump(indent) + "\n" + r.text_table();
    *len = static_cast<int64_t>(s.size());
    if (buf && cap > 0) {
      const size_t n = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
  });
}

// ---------------------------------------------------------------- on-disk formats (dataset.hpp:84-280)
// Datasets returned here may be partial (graph only / features only); ref_ds_info / ref_ds_export and
// ref_ds_feat_shape read them.
int ref_load_graph_f32(const char* path, int32_t fmt, void** out) {
  return guarded([&] {
    auto ds = std::make_unique<Dataset<float>>();
    ds->graph = fmt == 1 ? load_matrix_market<float>(path) : fmt == 2 ? load_edge_list<float>(path)
                                                                       : load_graph<float>(path);
    *out = ds.release();
  });
}
int ref_load_features_f32(const char* path, void** out) {
  return guarded([&] {
    auto ds = std::make_unique<Dataset<float>>();
    ds->features = load_features<float>(path);
    *out = ds.release();
  });
}
int ref_read_dense_f32(const char* path, void** out) {
  return guarded([&] {
    auto ds = std::make_unique<Dataset<float>>();
    ds->features = read_dense<float>(path);
    *out = ds.release();
  });
}
void ref_ds_feat_shape_f32(void* h, int64_t* rows, int64_t* cols) {
  auto* ds = static_cast<Dataset<float>*>(h);
  *rows = ds->features.rows();
  *cols = ds->features.cols();
}
int ref_write_dense_f32(const char* path, int64_t rows, int64_t cols, const float* data) {
  return guarded([&] {
    DenseMatrix<float> m(rows, cols);
    if (rows * cols) std::memcpy(m.data(), data, sizeof(float) * static_cast<size_t>(rows * cols));
    write_dense<float>(path, m.view());
  });
}
int ref_load_labels(const char* path, int32_t* dst, int64_t cap, int64_t* count) {
  return guarded([&] {
    const auto l = load_labels(path);
    *count = static_cast<int64_t>(l.size());
    if (dst) std::memcpy(dst, l.data(), 4 * std::min<size_t>(l.size(), static_cast<size_t>(cap)));
  });
}
int ref_load_masks(const char* path, int64_t n, uint8_t* train, uint8_t* val, uint8_t* test, int32_t* present) {
  return guarded([&] {
    std::vector<uint8_t> tr, va, te;
    load_masks(path, n, tr, va, te);
    *present = (tr.empty() ? 0 : 1) | (va.empty() ? 0 : 2) | (te.empty() ? 0 : 4);
    if (!tr.empty()) std::memcpy(train, tr.data(), tr.size());
    if (!va.empty()) std::memcpy(val, va.data(), va.size());
    if (!te.empty()) std::memcpy(test, te.data(), te.size());
  });
}
int ref_load_dataset_f32(const char* g, const char* f, const char* l, const char* m, void** out) {
  return guarded([&] { *out = new Dataset<float>(load_dataset<float>(g, f, l, m ? m : "")); });
}
// ---------------------------------------------------------------- timeline (timeline.hpp, breakdown.hpp)
// Loads a timeline JSON with the reference's own load_timeline, runs audit_timeline, optionally
// audit_staged_run (world > 0), and returns runtime_breakdown totals {spmm, gemm, activation, loss, adam,
// comm} and the event count.
int ref_timeline_check(const char* path, int32_t world, int32_t overlapped, double* totals, int64_t* count) {
  return guarded([&] {
    const auto ev = load_timeline(path);
    *count = static_cast<int64_t>(ev.size());
    audit_timeline(ev);
    if (world > 0) audit_staged_run(ev, world, overlapped != 0);
    const auto rep = runtime_breakdown(ev);
    const double t[6] = {rep.spmm_us, rep.gemm_us, rep.activation_us, rep.loss_us, rep.adam_us, rep.comm_us};
    std::memcpy(totals, t, sizeof(t));
  });
}
// The reference's own training-run timeline (DeviceGroup, threads as GPUs) exported to path: the
// structural template the device timeline mirrors (kinds, ops, stages, lanes, dependency shape).
int ref_train_timeline_f32(void* dsh, const RefCfg* c, int32_t workers, const char* path) {
  return guarded([&] {
    TrainOptions opts;
    opts.workers = workers;
    const auto art = train_run<float>(*static_cast<Dataset<float>*>(dsh), to_cfg(c), opts);
    export_timeline(path, art.timeline);
  });
}

void ref_ds_masks_f32(void* h, uint8_t* train, uint8_t* val, uint8_t* test, int32_t* present) {
  auto* ds = static_cast<Dataset<float>*>(h);
  *present = (ds->train_mask.empty() ? 0 : 1) | (ds->val_mask.empty() ? 0 : 2) | (ds->test_mask.empty() ? 0 : 4);
  if (!ds->train_mask.empty()) std::memcpy(train, ds->train_mask.data(), ds->train_mask.size());
  if (!ds->val_mask.empty()) std::memcpy(val, ds->val_mask.data(), ds->val_mask.size());
  if (!ds->test_mask.empty()) std::memcpy(test, ds->test_mask.data(), ds->test_mask.size());
}

}  // extern "C"
