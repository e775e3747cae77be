// SPDX-License-Identifier: Apache-2.0
//
// mggcn/rowgcn.hpp — C++ drop-in for the reference's training API (rowgcn, proj/include/rowgcn/),
// header-only on top of the C ABI in mggcn.h (link with -lmggcn). Same names, argument meaning and
// exception types as the reference, so a caller of rowgcn switches by changing the include and the
// namespace:
//
//   rowgcn (reference)                                   mggcn::rowgcn (this header)
//   ShapeError/ValueError/... inc/errors.hpp:10-39        same names, same what() text
//   GcnConfig                 inc/gcn.hpp:14-36           + gemm_mode / spmm_mode
//   parse_config / materialize_config  driver.hpp:24-57   same (generic over the JSON type)
//   CsrMatrix / DenseMatrix / Dataset   sparse.hpp / dense.hpp / dataset.hpp
//   synth_graph<S>            inc/dataset.hpp:287-334     bit-identical output
//   add_self_loops<S>         inc/dataset.hpp:60-73
//   load_dataset<S> / load_graph<S> / load_features<S> / load_labels / load_masks / read_dense<S> /
//   write_dense<S>            inc/dataset.hpp:84-280, dense.hpp:290-335
//   prepare_data / PreparedData  driver.hpp:75-117        bit-identical tiles
//   GroupOptions / TrainOptions / TrainArtifacts / train_run<S>  driver.hpp:119-206, collectives.hpp:41-44
//   GradArtifacts / grad_run<S>  driver.hpp:209-251
//   config_to_json            driver.hpp:59-71            byte-identical dump()
//   write_checkpoint / read_checkpoint<S>  driver.hpp:255-299  (MGDM blocks + <path>.json sidecar)
//   runtime_breakdown / BreakdownReport / export_timeline / audits  breakdown.hpp, timeline.hpp
//
// The device work runs on the GPUs of this process (one GcnWorker per rank, two CUDA streams each,
// NCCL or the in-process transport between them). The templates are instantiable for S = float only:
// S = double is rejected at compile time (the B200 step trains in fp32; train_run<double> stays with the
// CPU reference), so a reference caller compiles unchanged for float.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "mggcn.h"

namespace mggcn {
namespace rowgcn {

using index_t = std::int64_t;

// ---------------------------------------------------------------- errors (inc/errors.hpp)
struct ShapeError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ValueError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ProtocolError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ShutdownError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ParseError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NcclError : std::runtime_error { using std::runtime_error::runtime_error; };

// The device path computes in fp32: every rowgcn template here is instantiable for S = float only.
template <class S>
constexpr void require_float() {
  static_assert(std::is_same<S, float>::value,
                "mggcn::rowgcn: the B200 training step runs in float (fp32 with 3xTF32 GeMMs); "
                "instantiate with S = float (rowgcn<double> stays with the CPU reference)");
}

inline void check(mg_status s) {
  if (s == MG_OK) return;
  const std::string m = mg_last_error();
  switch (s) {
    case MG_SHAPE_ERROR: throw ShapeError(m);
    case MG_VALUE_ERROR: throw ValueError(m);
    case MG_PROTOCOL_ERROR: throw ProtocolError(m);
    case MG_SHUTDOWN_ERROR: throw ShutdownError(m);
    case MG_PARSE_ERROR: throw ParseError(m);
    case MG_CONFIG_ERROR: throw ConfigError(m);
    case MG_IO_ERROR: throw IoError(m);
    case MG_CUDA_ERROR: throw CudaError(m);
    case MG_NCCL_ERROR: throw NcclError(m);
    default: throw std::runtime_error(m);
  }
}

// ---------------------------------------------------------------- Rng (inc/rng.hpp)
// std::mt19937_64 (standard-mandated stream) with modulo bounded draws and 53-bit uniforms: the same
// numbers as the reference's Rng and as the library's generator / Glorot init.
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : gen_(seed) {}
  std::uint64_t next() { return gen_(); }
  std::uint64_t below(std::uint64_t n) { return gen_() % n; }
  double uniform() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }

 private:
  std::mt19937_64 gen_;
};

// ---------------------------------------------------------------- containers
template <class S>
struct CooEdge {  // inc/sparse.hpp:16-21
  index_t src = 0;
  index_t dst = 0;
  S weight = S(1);
};

template <class S>
struct CsrMatrix {  // inc/sparse.hpp:25-55
  index_t rows = 0, cols = 0;
  std::vector<index_t> row_ptr, col_idx;
  std::vector<S> values;
  index_t nnz() const { return static_cast<index_t>(col_idx.size()); }
};

template <class S>
class DenseMatrix {  // inc/dense.hpp:73-118 (row-major, ld = cols)
 public:
  DenseMatrix() = default;
  DenseMatrix(index_t r, index_t c) : rows_(r), cols_(c), data_(static_cast<size_t>(r * c), S(0)) {
    if (r < 0 || c < 0) throw ValueError("DenseMatrix: negative dimension");
  }
  index_t rows() const { return rows_; }
  index_t cols() const { return cols_; }
  index_t size() const { return rows_ * cols_; }
  S* data() { return data_.data(); }
  const S* data() const { return data_.data(); }
  S& operator()(index_t i, index_t j) { return data_[static_cast<size_t>(i * cols_ + j)]; }
  S operator()(index_t i, index_t j) const { return data_[static_cast<size_t>(i * cols_ + j)]; }

 private:
  index_t rows_ = 0, cols_ = 0;
  std::vector<S> data_;
};

template <class S>
struct Dataset {  // inc/dataset.hpp:19-56
  CsrMatrix<S> graph;
  DenseMatrix<S> features;
  std::vector<std::int32_t> labels;
  std::vector<std::uint8_t> train_mask, val_mask, test_mask;
  std::string name;
  index_t n() const { return graph.rows; }
  void validate() const;  // Dataset::validate (inc/dataset.hpp:30-44), defined below
  std::vector<std::uint8_t> effective_mask() const {  // inc/dataset.hpp:46-49
    if (!train_mask.empty()) return train_mask;
    return std::vector<std::uint8_t>(static_cast<size_t>(n()), 1);
  }
  int num_classes() const {
    std::int32_t c = 0;
    for (auto l : labels) c = l > c ? l : c;
    return c + 1;
  }
};

// ---------------------------------------------------------------- config (inc/gcn.hpp:14-36)
struct GcnConfig {
  std::vector<index_t> layer_dims;
  double lr = 0.01, beta1 = 0.9, beta2 = 0.999, epsilon = 1e-8;
  int epochs = 100;
  std::uint64_t seed = 1;
  bool permute = false, overlap = false, skip_first_backward_spmm = false, order_swap = false;
  int gemm_mode = MG_GEMM_TF32X3;  // see DESIGN.md: EXACT is bitwise, TF32X3/FAST meet rel 1e-4
  int spmm_mode = MG_SPMM_FAST;
  bool aggregate_input = true;  // FAST only: layer 0 as (A X) W0 (mggcn.h)
  bool bias = false;            // default-off extensions, no reference analogue (mggcn.h)
  double dropout = 0.0;
  int layers() const { return static_cast<int>(layer_dims.size()) - 1; }
  mg_config c() const {
    mg_config m;
    mg_config_defaults(&m);
    m.layer_dims = layer_dims.data();
    m.n_dims = static_cast<std::int32_t>(layer_dims.size());
    m.lr = lr;
    m.beta1 = beta1;
    m.beta2 = beta2;
    m.epsilon = epsilon;
    m.epochs = epochs;
    m.seed = seed;
    m.permute = permute;
    m.overlap = overlap;
    m.skip_first_backward_spmm = skip_first_backward_spmm;
    m.order_swap = order_swap;
    m.gemm_mode = gemm_mode;
    m.spmm_mode = spmm_mode;
    m.aggregate_input = aggregate_input;
    m.bias = bias;
    m.dropout = dropout;
    return m;
  }
  void validate() const {
    const mg_config m = c();
    check(mg_config_validate(&m));
  }
};

struct ConfigFile {  // inc/driver.hpp:19-22
  std::vector<index_t> hidden_dims{16};
  GcnConfig cfg;
};

// inc/driver.hpp:24-47, generic over the JSON type (nlohmann::json in the reference's callers).
template <class Json>
ConfigFile parse_config(const Json& j) {
  static const char* known[] = {"hidden_dims", "lr", "beta1", "beta2", "epsilon", "epochs", "seed", "permute",
                                "overlap", "skip_first_backward_spmm", "order_swap"};
  for (auto it = j.begin(); it != j.end(); ++it) {
    bool ok = false;
    for (const char* k : known) ok = ok || it.key() == k;
    if (!ok) throw ConfigError("config: unknown key '" + it.key() + "'");
  }
  ConfigFile cf;
  if (j.contains("hidden_dims")) cf.hidden_dims = j.at("hidden_dims").template get<std::vector<index_t>>();
  auto& c = cf.cfg;
  c.lr = j.value("lr", c.lr);
  c.beta1 = j.value("beta1", c.beta1);
  c.beta2 = j.value("beta2", c.beta2);
  c.epsilon = j.value("epsilon", c.epsilon);
  c.epochs = j.value("epochs", c.epochs);
  c.seed = j.value("seed", c.seed);
  c.permute = j.value("permute", c.permute);
  c.overlap = j.value("overlap", c.overlap);
  c.skip_first_backward_spmm = j.value("skip_first_backward_spmm", c.skip_first_backward_spmm);
  c.order_swap = j.value("order_swap", c.order_swap);
  return cf;
}

inline GcnConfig materialize_config(const ConfigFile& cf, index_t d0, int classes) {  // driver.hpp:49-57
  GcnConfig cfg = cf.cfg;
  cfg.layer_dims.clear();
  cfg.layer_dims.push_back(d0);
  for (index_t h : cf.hidden_dims) cfg.layer_dims.push_back(h);
  cfg.layer_dims.push_back(classes);
  cfg.validate();
  return cfg;
}

// ---------------------------------------------------------------- RAII handles over the C ABI
namespace detail {
struct DatasetHandle {
  mg_dataset* p = nullptr;
  ~DatasetHandle() { mg_dataset_free(p); }
};
struct PartitionDel {
  void operator()(mg_partition* p) const { mg_partition_free(p); }
};
struct GroupDel {
  void operator()(mg_group* g) const { mg_group_destroy(g); }
};

inline DatasetHandle to_handle(const Dataset<float>& ds) {
  DatasetHandle h;
  const mg_csr g{ds.graph.rows, ds.graph.cols, ds.graph.row_ptr.data(), ds.graph.col_idx.data(),
                 ds.graph.values.data()};
  check(mg_dataset_from_arrays(&g, ds.features.data(), ds.features.cols(), ds.labels.data(),
                               ds.train_mask.empty() ? nullptr : ds.train_mask.data(), &h.p));
  return h;
}
}  // namespace detail

namespace detail {
inline Dataset<float> from_handle(mg_dataset* p, const std::string& name) {
  mg_csr g;
  const float* f = nullptr;
  const std::int32_t* lab = nullptr;
  const std::uint8_t* mask = nullptr;
  std::int64_t d0 = 0;
  check(mg_dataset_view(p, &g, &f, &d0, &lab, &mask));
  const std::uint8_t *tr = nullptr, *va = nullptr, *te = nullptr;
  check(mg_dataset_masks(p, &tr, &va, &te));
  const index_t n = g.rows;
  Dataset<float> ds;
  ds.name = name;
  ds.graph.rows = g.rows;
  ds.graph.cols = g.cols;
  ds.graph.row_ptr.assign(g.row_ptr, g.row_ptr + n + 1);
  ds.graph.col_idx.assign(g.col_idx, g.col_idx + g.row_ptr[n]);
  ds.graph.values.assign(g.values, g.values + g.row_ptr[n]);
  ds.features = DenseMatrix<float>(n, d0);
  if (n * d0 > 0) std::memcpy(ds.features.data(), f, sizeof(float) * static_cast<size_t>(n * d0));
  ds.labels.assign(lab, lab + n);
  if (tr) ds.train_mask.assign(tr, tr + n);
  if (va) ds.val_mask.assign(va, va + n);
  if (te) ds.test_mask.assign(te, te + n);
  return ds;
}
inline CsrMatrix<float> graph_view(const mg_graph* h) {
  mg_csr g;
  check(mg_graph_view(h, &g));
  CsrMatrix<float> m;
  m.rows = g.rows;
  m.cols = g.cols;
  m.row_ptr.assign(g.row_ptr, g.row_ptr + g.rows + 1);
  m.col_idx.assign(g.col_idx, g.col_idx + g.row_ptr[g.rows]);
  m.values.assign(g.values, g.values + g.row_ptr[g.rows]);
  return m;
}
inline CsrMatrix<float> graph_from(int32_t format, const std::string& path) {
  mg_graph* h = nullptr;
  check(mg_graph_load(path.c_str(), format, &h));
  std::unique_ptr<mg_graph, void (*)(mg_graph*)> guard(h, mg_graph_free);
  return graph_view(h);
}
inline DenseMatrix<float> dense_from(mg_status (*fn)(const char*, mg_dense**), const std::string& path) {
  mg_dense* h = nullptr;
  check(fn(path.c_str(), &h));
  std::unique_ptr<mg_dense, void (*)(mg_dense*)> guard(h, mg_dense_free);
  std::int64_t r = 0, c = 0;
  const float* d = nullptr;
  check(mg_dense_view(h, &r, &c, &d));
  DenseMatrix<float> m(r, c);
  if (r * c > 0) std::memcpy(m.data(), d, sizeof(float) * static_cast<size_t>(r * c));
  return m;
}
}  // namespace detail

// rowgcn::synth_graph<S> (inc/dataset.hpp:287-334), bit-identical.
template <class S>
Dataset<S> synth_graph(index_t n, double avg_degree, double exponent, std::uint64_t seed, index_t feature_dim = 16,
                       int classes = 4) {
  require_float<S>();
  detail::DatasetHandle h;
  check(mg_dataset_synth(n, avg_degree, exponent, seed, feature_dim, classes, &h.p));
  return detail::from_handle(h.p, "synth-n" + std::to_string(n) + "-d" + std::to_string(avg_degree));
}

template <class S>
inline void Dataset<S>::validate() const {
  require_float<S>();
  auto h = detail::to_handle(*this);
  check(mg_dataset_validate(h.p));
}

// from_coo (inc/sparse.hpp:59-90).
template <class S>
CsrMatrix<S> from_coo(std::vector<CooEdge<S>> edges, index_t n) {
  require_float<S>();
  std::vector<std::int64_t> src(edges.size()), dst(edges.size());
  std::vector<float> w(edges.size());
  for (size_t e = 0; e < edges.size(); ++e) {
    src[e] = edges[e].src;
    dst[e] = edges[e].dst;
    w[e] = edges[e].weight;
  }
  mg_graph* g = nullptr;
  check(mg_graph_from_coo(n, static_cast<std::int64_t>(edges.size()), src.data(), dst.data(), w.data(), &g));
  std::unique_ptr<mg_graph, void (*)(mg_graph*)> guard(g, mg_graph_free);
  return detail::graph_view(g);
}

// add_self_loops (inc/dataset.hpp:60-73).
template <class S>
CsrMatrix<S> add_self_loops(const CsrMatrix<S>& a) {
  require_float<S>();
  const mg_csr c{a.rows, a.cols, a.row_ptr.data(), a.col_idx.data(), a.values.data()};
  mg_graph* g = nullptr;
  check(mg_graph_add_self_loops(&c, &g));
  std::unique_ptr<mg_graph, void (*)(mg_graph*)> guard(g, mg_graph_free);
  return detail::graph_view(g);
}

// On-disk formats (inc/dataset.hpp:84-280, inc/dense.hpp:290-335): native multi-threaded loaders,
// same syntax, messages and exception types as the reference.
template <class S>
CsrMatrix<S> load_matrix_market(const std::string& path) {
  require_float<S>();
  return detail::graph_from(1, path);
}
template <class S>
CsrMatrix<S> load_edge_list(const std::string& path) {
  require_float<S>();
  return detail::graph_from(2, path);
}
template <class S>
CsrMatrix<S> load_graph(const std::string& path) {
  require_float<S>();
  return detail::graph_from(0, path);
}
template <class S>
DenseMatrix<S> load_features(const std::string& path) {
  require_float<S>();
  return detail::dense_from(mg_dense_load, path);
}
template <class S>
DenseMatrix<S> read_dense(const std::string& path) {
  require_float<S>();
  return detail::dense_from(mg_dense_read, path);
}
template <class S>
void write_dense(const std::string& path, const DenseMatrix<S>& m) {
  require_float<S>();
  check(mg_dense_write(path.c_str(), m.rows(), m.cols(), m.data()));
}
inline std::vector<std::int32_t> load_labels(const std::string& path) {
  std::int64_t n = 0;
  check(mg_labels_load(path.c_str(), nullptr, 0, &n));
  std::vector<std::int32_t> out(static_cast<size_t>(n));
  check(mg_labels_load(path.c_str(), out.data(), n, &n));
  return out;
}
inline void load_masks(const std::string& path, index_t n, std::vector<std::uint8_t>& train,
                       std::vector<std::uint8_t>& val, std::vector<std::uint8_t>& test) {
  std::vector<std::uint8_t> a(static_cast<size_t>(n)), b(static_cast<size_t>(n)), c(static_cast<size_t>(n));
  std::int32_t present = 0;
  check(mg_masks_load(path.c_str(), n, a.data(), b.data(), c.data(), &present));
  if (present & 1) train = std::move(a);
  if (present & 2) val = std::move(b);
  if (present & 4) test = std::move(c);
}
template <class S>
Dataset<S> load_dataset(const std::string& graph_path, const std::string& features_path,
                        const std::string& labels_path, const std::string& masks_path = "") {
  require_float<S>();
  detail::DatasetHandle h;
  check(mg_dataset_load(graph_path.c_str(), features_path.c_str(), labels_path.c_str(),
                        masks_path.empty() ? nullptr : masks_path.c_str(), &h.p));
  return detail::from_handle(h.p, graph_path);
}

// rowgcn::PreparedData (inc/driver.hpp:75-85): owns the bit-exact tiles of this process's ranks.
struct PreparedData {
  std::unique_ptr<mg_partition, detail::PartitionDel> p;
  int workers = 1;
  std::vector<index_t> bounds() const {
    std::vector<index_t> b(static_cast<size_t>(workers) + 1);
    check(mg_partition_info(p.get(), nullptr, nullptr, b.data()));
    return b;
  }
  CsrMatrix<float> tile(int dir, int i, int j) const {  // dir 0: A_hat^T (forward), 1: A_hat
    CsrMatrix<float> t;
    std::int64_t nnz = 0;
    check(mg_partition_tile_info(p.get(), dir, i, j, &t.rows, &t.cols, &nnz));
    t.row_ptr.resize(static_cast<size_t>(t.rows) + 1);
    t.col_idx.resize(static_cast<size_t>(nnz));
    t.values.resize(static_cast<size_t>(nnz));
    check(mg_partition_tile_export(p.get(), dir, i, j, t.row_ptr.data(), t.col_idx.data(), t.values.data()));
    return t;
  }
};

inline PreparedData prepare_data(const Dataset<float>& ds, const GcnConfig& cfg, int workers, int only_rank = -1) {
  auto h = detail::to_handle(ds);
  const mg_config c = cfg.c();
  mg_partition* p = nullptr;
  check(mg_prepare(h.p, &c, workers, only_rank, &p));
  PreparedData out;
  out.p.reset(p);
  out.workers = workers;
  return out;
}

// ---------------------------------------------------------------- driver (inc/driver.hpp:119-251)
// rowgcn::GroupOptions (inc/collectives.hpp:41-44). Accepted for source compatibility and ignored: the
// link delay is an injected cost of the reference's simulated links; here the links are NVLink / NCCL.
struct GroupOptions {
  double link_delay_ns_per_byte = 0.0;
};

struct TrainOptions {
  int workers = 1;
  GroupOptions group;  // ignored (see GroupOptions)
  bool collect_logits = false;
  std::function<void(int, double, double, double)> on_epoch;  // (epoch, loss, acc, wall_us) on rank 0
  std::vector<int> devices;  // CUDA device per rank; default rank % #devices
  int transport = MG_TRANSPORT_AUTO;
};

// rowgcn::TimelineEvent (inc/collectives.hpp:24-34), recorded from CUDA events (mggcn.h timeline).
struct TimelineEvent {
  int worker = 0, lane = 0, stage = -1;
  std::string kind, op;
  double t_start_us = 0, t_end_us = 0;
  std::uint64_t task = 0;
  std::vector<std::uint64_t> deps;
};

namespace detail {
inline std::vector<TimelineEvent> timeline(mg_group* g) {
  std::int64_t n = 0;
  check(mg_group_timeline(g, nullptr, 0, &n));
  std::vector<mg_timeline_event> raw(static_cast<size_t>(n));
  check(mg_group_timeline(g, raw.data(), n, &n));
  std::vector<TimelineEvent> out;
  out.reserve(raw.size());
  for (const auto& e : raw)
    out.push_back({e.worker, e.lane, e.stage, e.kind, e.op, e.t_start_us, e.t_end_us, e.task,
                   std::vector<std::uint64_t>(e.deps, e.deps + e.n_deps)});
  return out;
}
inline std::vector<mg_timeline_event> to_c(const std::vector<TimelineEvent>& ev) {
  std::vector<mg_timeline_event> out(ev.size());
  for (size_t i = 0; i < ev.size(); ++i) {
    auto& o = out[i];
    o.worker = ev[i].worker;
    o.lane = ev[i].lane;
    o.stage = ev[i].stage;
    o.n_deps = static_cast<std::int32_t>(ev[i].deps.size());
    std::snprintf(o.kind, sizeof(o.kind), "%s", ev[i].kind.c_str());
    std::snprintf(o.op, sizeof(o.op), "%s", ev[i].op.c_str());
    o.t_start_us = ev[i].t_start_us;
    o.t_end_us = ev[i].t_end_us;
    o.task = ev[i].task;
    o.deps = ev[i].deps.data();
  }
  return out;
}
}  // namespace detail

// export_timeline / audit_timeline / audit_staged_run (inc/timeline.hpp:31-126), native.
inline void export_timeline(const std::string& path, const std::vector<TimelineEvent>& ev) {
  const auto c = detail::to_c(ev);
  check(mg_timeline_export(path.c_str(), c.data(), static_cast<std::int64_t>(c.size())));
}
inline void audit_timeline(const std::vector<TimelineEvent>& ev) {
  const auto c = detail::to_c(ev);
  check(mg_timeline_audit(c.data(), static_cast<std::int64_t>(c.size())));
}
inline void audit_staged_run(const std::vector<TimelineEvent>& ev, int world, bool overlapped) {
  const auto c = detail::to_c(ev);
  check(mg_timeline_audit_staged(c.data(), static_cast<std::int64_t>(c.size()), world, overlapped ? 1 : 0));
}

// A JSON document the reference returns as nlohmann::json (config_to_json, BreakdownReport::to_json):
// dump(indent) gives the same text nlohmann::json::dump(indent) does (mggcn.h).
class JsonText {
 public:
  explicit JsonText(std::function<mg_status(int, char*, std::int64_t, std::int64_t*)> f) : f_(std::move(f)) {}
  std::string dump(int indent = -1) const {
    std::int64_t n = 0;
    check(f_(indent, nullptr, 0, &n));
    std::string s(static_cast<size_t>(n) + 1, '\0');
    check(f_(indent, &s[0], n + 1, &n));
    s.resize(static_cast<size_t>(n));
    return s;
  }

 private:
  std::function<mg_status(int, char*, std::int64_t, std::int64_t*)> f_;
};

// config_to_json (inc/driver.hpp:59-71).
inline JsonText config_to_json(const GcnConfig& cfg) {
  return JsonText([cfg](int indent, char* b, std::int64_t cap, std::int64_t* n) {
    const mg_config c = cfg.c();
    return mg_config_to_json(&c, indent, b, cap, n);
  });
}

// BreakdownReport / runtime_breakdown (inc/breakdown.hpp:17-82) over the CUDA-event timeline.
struct BreakdownReport {
  double spmm_us = 0, gemm_us = 0, activation_us = 0, loss_us = 0, adam_us = 0, comm_us = 0;
  double total_us() const { return spmm_us + gemm_us + activation_us + loss_us + adam_us + comm_us; }
  double frac(double v) const {
    const double t = total_us();
    return t > 0 ? v / t : 0.0;
  }
  JsonText to_json() const {
    const std::vector<double> t{spmm_us, gemm_us, activation_us, loss_us, adam_us, comm_us};
    return JsonText([t](int indent, char* b, std::int64_t cap, std::int64_t* n) {
      return mg_breakdown_to_json(t.data(), indent, b, cap, n);
    });
  }
  std::string text_table() const {
    const double t[6] = {spmm_us, gemm_us, activation_us, loss_us, adam_us, comm_us};
    std::int64_t n = 0;
    check(mg_breakdown_text(t, nullptr, 0, &n));
    std::string s(static_cast<size_t>(n) + 1, '\0');
    check(mg_breakdown_text(t, &s[0], n + 1, &n));
    s.resize(static_cast<size_t>(n));
    return s;
  }
};

inline BreakdownReport runtime_breakdown(const std::vector<TimelineEvent>& ev) {
  const auto c = detail::to_c(ev);
  double t[6] = {0, 0, 0, 0, 0, 0};
  check(mg_timeline_breakdown(c.data(), static_cast<std::int64_t>(c.size()), t));
  BreakdownReport r;
  r.spmm_us = t[0];
  r.gemm_us = t[1];
  r.activation_us = t[2];
  r.loss_us = t[3];
  r.adam_us = t[4];
  r.comm_us = t[5];
  return r;
}

template <class S>
struct TrainArtifacts {
  std::vector<double> epoch_loss, epoch_acc, epoch_wall_us;
  std::vector<TimelineEvent> timeline;  // every task of every epoch (CUDA events)
  std::vector<std::vector<std::uint64_t>> w_hashes;  // [epoch][rank]
  std::vector<DenseMatrix<S>> final_w;               // rank 0's replicas
  DenseMatrix<S> logits;                             // gathered post-training logits (permuted order)
  int workers = 1;
  double final_loss() const { return epoch_loss.empty() ? 0.0 : epoch_loss.back(); }
  double final_acc() const { return epoch_acc.empty() ? 0.0 : epoch_acc.back(); }
};

template <class S>
struct GradArtifacts {
  std::vector<DenseMatrix<S>> w_grad;
  std::vector<std::uint64_t> grad_hash_per_rank;
  double loss = 0.0;
};

namespace detail {
inline std::unique_ptr<mg_group, GroupDel> make_group(const GcnConfig& cfg, const PreparedData& prep, int workers,
                                                      std::vector<int> devices, int transport) {
  std::vector<std::int32_t> ranks(static_cast<size_t>(workers));
  if (devices.empty()) {
    int nd = mg_device_count();
    if (nd < 1) nd = 1;
    for (int r = 0; r < workers; ++r) devices.push_back(r % nd);
  }
  for (int r = 0; r < workers; ++r) ranks[static_cast<size_t>(r)] = r;
  const mg_config c = cfg.c();
  mg_group* g = nullptr;
  check(mg_group_create(&c, prep.p.get(), workers, workers, ranks.data(), devices.data(), nullptr, transport, &g));
  return std::unique_ptr<mg_group, GroupDel>(g);
}

inline DenseMatrix<float> read(mg_group* g, int rank, int which, int layer, index_t rows, index_t cols) {
  DenseMatrix<float> m(rows, cols);
  check(mg_group_read(g, rank, which, layer, m.data(), m.size()));
  return m;
}
}  // namespace detail

template <class S>
TrainArtifacts<S> train_run(const Dataset<S>& ds, const GcnConfig& cfg, const TrainOptions& opts) {
  require_float<S>();
  cfg.validate();
  if (cfg.layer_dims.front() != ds.features.cols())
    throw ConfigError("config: layer_dims[0]=" + std::to_string(cfg.layer_dims.front()) +
                      " but dataset features have width " + std::to_string(ds.features.cols()));
  const PreparedData prep = prepare_data(ds, cfg, opts.workers);
  auto g = detail::make_group(cfg, prep, opts.workers, opts.devices, opts.transport);
  check(mg_group_init_params(g.get()));
  TrainArtifacts<float> art;
  art.workers = opts.workers;
  check(mg_group_set_timeline(g.get(), 1));
  for (int e = 1; e <= cfg.epochs; ++e) {
    double loss = 0, acc = 0, wall = 0;
    check(mg_group_train_step(g.get(), e, &loss, &acc, &wall));
    art.epoch_loss.push_back(loss);
    art.epoch_acc.push_back(acc);
    art.epoch_wall_us.push_back(wall);
    std::vector<std::uint64_t> hs(static_cast<size_t>(opts.workers));
    for (int r = 0; r < opts.workers; ++r) check(mg_group_w_hash(g.get(), r, &hs[static_cast<size_t>(r)]));
    art.w_hashes.push_back(std::move(hs));
    if (opts.on_epoch) opts.on_epoch(e, loss, acc, wall);
  }
  art.timeline = detail::timeline(g.get());
  check(mg_group_set_timeline(g.get(), 0));
  const int L = cfg.layers();
  if (opts.collect_logits) {
    double l = 0;
    check(mg_group_loss_only(g.get(), &l));
    art.logits = DenseMatrix<float>(ds.n(), cfg.layer_dims.back());
    for (int r = 0; r < opts.workers; ++r) {
      std::int64_t b = 0, rows = 0;
      check(mg_group_rows(g.get(), r, &b, &rows));
      check(mg_group_read(g.get(), r, MG_T_AHW, L - 1, art.logits.data() + b * cfg.layer_dims.back(),
                          rows * cfg.layer_dims.back()));
    }
  }
  for (int l = 0; l < L; ++l)
    art.final_w.push_back(detail::read(g.get(), 0, MG_T_W, l, cfg.layer_dims[static_cast<size_t>(l)],
                                       cfg.layer_dims[static_cast<size_t>(l) + 1]));
  return art;
}

template <class S>
GradArtifacts<S> grad_run(const Dataset<S>& ds, const GcnConfig& cfg, int workers) {
  require_float<S>();
  cfg.validate();
  const PreparedData prep = prepare_data(ds, cfg, workers);
  auto g = detail::make_group(cfg, prep, workers, {}, MG_TRANSPORT_AUTO);
  check(mg_group_init_params(g.get()));
  GradArtifacts<float> art;
  double acc = 0;
  check(mg_group_compute_gradients(g.get(), &art.loss, &acc));
  const int L = cfg.layers();
  for (int r = 0; r < workers; ++r) {
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (int l = 0; l < L; ++l) {
      auto m = detail::read(g.get(), r, MG_T_WGRAD, l, cfg.layer_dims[static_cast<size_t>(l)],
                            cfg.layer_dims[static_cast<size_t>(l) + 1]);
      const auto* p = reinterpret_cast<const unsigned char*>(m.data());
      for (size_t i = 0; i < sizeof(float) * static_cast<size_t>(m.size()); ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
      }
      if (r == 0) art.w_grad.push_back(std::move(m));
    }
    art.grad_hash_per_rank.push_back(h);
  }
  return art;
}

// write_checkpoint (inc/driver.hpp:255-274): every W as an MGDM block back to back, plus <path>.json with
// config_to_json(cfg); byte-identical files (mggcn.h).
template <class S>
void write_checkpoint(const std::string& path, const std::vector<DenseMatrix<S>>& ws, const GcnConfig& cfg) {
  require_float<S>();
  std::vector<std::int64_t> rows, cols;
  std::vector<const float*> data;
  for (const auto& w : ws) {
    rows.push_back(w.rows());
    cols.push_back(w.cols());
    data.push_back(w.data());
  }
  const mg_config c = cfg.c();
  check(mg_checkpoint_write(path.c_str(), static_cast<std::int32_t>(ws.size()), rows.data(), cols.data(), data.data(),
                            &c));
}

// read_checkpoint<S> (inc/driver.hpp:276-299).
template <class S>
std::vector<DenseMatrix<S>> read_checkpoint(const std::string& path) {
  require_float<S>();
  mg_checkpoint* ck = nullptr;
  check(mg_checkpoint_read(path.c_str(), &ck));
  std::unique_ptr<mg_checkpoint, void (*)(mg_checkpoint*)> guard(ck, mg_checkpoint_free);
  std::vector<DenseMatrix<S>> ws;
  for (std::int32_t i = 0; i < mg_checkpoint_count(ck); ++i) {
    std::int64_t r = 0, c = 0;
    const float* d = nullptr;
    check(mg_checkpoint_view(ck, i, &r, &c, &d));
    DenseMatrix<S> w(r, c);
    if (r * c > 0) std::memcpy(w.data(), d, sizeof(float) * static_cast<size_t>(r * c));
    ws.push_back(std::move(w));
  }
  return ws;
}

}  // namespace rowgcn
}  // namespace mggcn
