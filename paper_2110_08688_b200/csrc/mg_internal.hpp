// SPDX-License-Identifier: Apache-2.0
// Internal host-side types shared by the host (mg_host.cpp) and device (mg_device.cu) halves of
// libmggcn.so. Nothing here is part of the ABI (include/mggcn.h is).
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "mggcn.h"

namespace mg {

using index_t = std::int64_t;

// Error taxonomy mirroring rowgcn (inc/errors.hpp:10-39); each maps to one mg_status.
struct Error : std::runtime_error {
  mg_status code;
  Error(mg_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
struct ShapeError : Error { explicit ShapeError(const std::string& m) : Error(MG_SHAPE_ERROR, m) {} };
struct ValueError : Error { explicit ValueError(const std::string& m) : Error(MG_VALUE_ERROR, m) {} };
struct ProtocolError : Error { explicit ProtocolError(const std::string& m) : Error(MG_PROTOCOL_ERROR, m) {} };
struct ShutdownError : Error { explicit ShutdownError(const std::string& m) : Error(MG_SHUTDOWN_ERROR, m) {} };
struct ConfigError : Error { explicit ConfigError(const std::string& m) : Error(MG_CONFIG_ERROR, m) {} };
struct CudaError : Error { explicit CudaError(const std::string& m) : Error(MG_CUDA_ERROR, m) {} };
struct NcclError : Error { explicit NcclError(const std::string& m) : Error(MG_NCCL_ERROR, m) {} };
struct ParseError : Error { explicit ParseError(const std::string& m) : Error(MG_PARSE_ERROR, m) {} };
struct IoError : Error { explicit IoError(const std::string& m) : Error(MG_IO_ERROR, m) {} };

void set_last_error(const std::string& msg);

template <class F>
mg_status guarded(F&& f) {
  try {
    f();
    return MG_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed (std::bad_alloc)");
    return MG_INTERNAL_ERROR;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return MG_INTERNAL_ERROR;
  }
}

inline std::string shape_str(index_t r, index_t c) { return std::to_string(r) + "x" + std::to_string(c); }

// Per-device one-time setup (kernel attributes such as the dynamic shared-memory limit live in each
// device's context): true the first time it is called with `dev` for this `seen` mask (devices < 64).
inline bool first_on_device(std::atomic<unsigned long long>& seen, int dev) {
  const unsigned long long bit = 1ull << (static_cast<unsigned>(dev) & 63u);
  return (seen.fetch_or(bit) & bit) == 0;
}

// ---------------------------------------------------------------- host parallel_for
int host_threads();
// Runs f(begin, end) over [0, n) split into contiguous chunks, one per thread.
void parallel_for(index_t n, const std::function<void(index_t, index_t)>& f, index_t min_chunk = 4096);

// ---------------------------------------------------------------- RNG (inc/rng.hpp:13-28)
// std::mt19937_64 restated so the host generator, permutation and Glorot init are platform-pinned.
class Rng {
 public:
  explicit Rng(std::uint64_t seed);
  std::uint64_t next();
  std::uint64_t below(std::uint64_t n) { return next() % n; }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  // std::mt19937_64::discard(k): advances the stream by k draws (state twists only, no tempering).
  void discard(std::uint64_t k);

 private:
  void twist();
  std::uint64_t mt_[312];
  int idx_;
};

// rowgcn::random_permutation (inc/partition.hpp:69-79): forward map old id -> new id.
void random_permutation(index_t n, std::uint64_t seed, std::vector<index_t>& forward);

// ---------------------------------------------------------------- config
struct Config {
  std::vector<index_t> dims;
  double lr = 0.01, beta1 = 0.9, beta2 = 0.999, epsilon = 1e-8;
  int epochs = 100;
  std::uint64_t seed = 1;
  bool permute = false, overlap = false, skip_first_backward_spmm = false, order_swap = false;
  int gemm_mode = MG_GEMM_TF32X3;
  int spmm_mode = MG_SPMM_EXACT;
  bool aggregate_input = false;
  bool bias = false;     // default-off extension: learned bias per layer (mggcn.h)
  double dropout = 0.0;  // default-off extension: dropout probability of hidden-layer outputs (mggcn.h)
  int layers() const { return static_cast<int>(dims.size()) - 1; }
  // Layer 0 as (Â·X)·W0 with Â·X kept for W0's gradient: one d0-wide SpMM replaces the d1-wide forward
  // and backward ones. Reassociation changes the float order, so only in MG_SPMM_FAST.
  bool aggregate_first() const {
    return aggregate_input && spmm_mode == MG_SPMM_FAST && !skip_first_backward_spmm && dims[0] < 2 * dims[1];
  }
};
Config to_config(const mg_config* c);  // validates (inc/gcn.hpp:29-35)

// ---------------------------------------------------------------- CSR / dataset
struct Csr {  // int64 row_ptr/col_idx like rowgcn::CsrMatrix (inc/sparse.hpp:25-55)
  index_t rows = 0, cols = 0;
  std::vector<index_t> row_ptr, col_idx;
  std::vector<float> values;
  index_t nnz() const { return static_cast<index_t>(col_idx.size()); }
  void validate() const;
};

}  // namespace mg

struct mg_dataset {
  mg::Csr graph;
  std::vector<float> features;  // feature_rows x d0 (feature_rows == n once validated)
  mg::index_t d0 = 0;
  mg::index_t feature_rows = 0;
  std::vector<std::int32_t> labels;
  std::vector<std::uint8_t> train_mask;  // empty = all
  std::vector<std::uint8_t> val_mask, test_mask;
  std::string name;
  mg::index_t n() const { return graph.rows; }
};

namespace mg {

void validate_dataset_named(const mg_dataset& ds);  // Dataset::validate (inc/dataset.hpp:30-44)

// Host storage for what group creation uploads (tile arrays, permuted features): page-locked when a CUDA
// device is present, so the upload is one DMA at full link speed with no staging copy (pinning happens at
// prepare time); plain heap memory otherwise (CPU-only hosts). Zero-initialised like std::vector.
bool pinned_host_available();
void* pinned_host_alloc(size_t bytes, bool* pinned);
void pinned_host_free(void* p, bool pinned);
bool is_pinned_host(const void* p);

template <class T>
struct UploadAlloc {
  using value_type = T;
  UploadAlloc() = default;
  template <class U>
  UploadAlloc(const UploadAlloc<U>&) {}
  T* allocate(size_t n) {
    bool pinned = false;
    return static_cast<T*>(pinned_host_alloc(n * sizeof(T), &pinned));
  }
  void deallocate(T* p, size_t) { pinned_host_free(p, is_pinned_host(p)); }
  template <class U>
  bool operator==(const UploadAlloc<U>&) const { return true; }
  template <class U>
  bool operator!=(const UploadAlloc<U>&) const { return false; }
};
template <class T>
using UploadVec = std::vector<T, UploadAlloc<T>>;

// One tile of the symmetric row tiling (rowgcn::TilePlan, inc/partition.hpp:158-171) in the device
// staging format: int64 row_ptr (host), int32 local column, fp32 value.
struct Tile {
  index_t rows = 0, cols = 0;
  std::vector<index_t> row_ptr;
  UploadVec<std::int32_t> col;
  UploadVec<float> val;
  index_t nnz() const { return static_cast<index_t>(col.size()); }
};

}  // namespace mg

struct mg_partition {
  mg::index_t n = 0, d0 = 0, mask_count = 0;
  int parts = 1;
  int only_rank = -1;
  std::vector<mg::index_t> bounds;
  std::vector<mg::index_t> perm_forward;
  // features / labels / mask hold permuted rows [row0, row0 + rows_stored()): every row for mg_prepare,
  // the rank's row block for the per-rank synthetic path (mg_synth_rank_finish)
  mg::index_t row0 = 0;
  mg::UploadVec<float> features;  // permuted, rows_stored() x d0
  std::vector<std::int32_t> labels;
  std::vector<std::uint8_t> mask;
  // tiles[dir][i][j]; rows i != only_rank are left empty when only_rank >= 0
  std::vector<std::vector<mg::Tile>> tiles[2];
  bool has_row(int i) const { return only_rank < 0 || only_rank == i; }
  mg::index_t rows_stored() const { return static_cast<mg::index_t>(labels.size()); }
};
