/* SPDX-License-Identifier: Apache-2.0
 *
 * mggcn.h — C ABI of the B200-native MG-GCN full-batch training step (libmggcn.so).
 *
 * This is the drop-in boundary for the reference's training API (rowgcn, proj/include/rowgcn/):
 * plain pointers and sizes, no C++ or torch types. Every entry point cites the reference interface it
 * replaces. C++ callers use include/mggcn/rowgcn.hpp (same names and exceptions as rowgcn); Python
 * callers use paper_2110_08688_b200 (ctypes). All calls return an mg_status; the message of the last
 * failure on the calling thread is mg_last_error(). Status codes map 1:1 onto the reference's
 * exception taxonomy (inc/errors.hpp:10-39) plus CUDA/NCCL failures.
 *
 * Ownership: objects returned through `**out` are owned by the caller and released with the matching
 * *_free / *_destroy. Input arrays are borrowed for the duration of the call (copied when kept).
 * Threading: calls on one object are not re-entrant (like train_run, inc/driver.hpp:140); distinct
 * objects may be used from distinct threads.
 */
#ifndef MGGCN_H_
#define MGGCN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MG_ABI_VERSION 3

typedef enum mg_status {
  MG_OK = 0,
  MG_SHAPE_ERROR = 1,    /* rowgcn::ShapeError    inc/errors.hpp:10 */
  MG_VALUE_ERROR = 2,    /* rowgcn::ValueError    inc/errors.hpp:15 */
  MG_PROTOCOL_ERROR = 3, /* rowgcn::ProtocolError inc/errors.hpp:20 */
  MG_SHUTDOWN_ERROR = 4, /* rowgcn::ShutdownError inc/errors.hpp:25 */
  MG_PARSE_ERROR = 5,    /* rowgcn::ParseError    inc/errors.hpp:30 */
  MG_CONFIG_ERROR = 6,   /* rowgcn::ConfigError   inc/errors.hpp:35 */
  MG_IO_ERROR = 7,       /* rowgcn::IoError       inc/errors.hpp:39 */
  MG_CUDA_ERROR = 8,     /* CUDA runtime / launch failure (no reference analogue) */
  MG_NCCL_ERROR = 9,     /* NCCL failure (the reference's collectives are in-process) */
  MG_INTERNAL_ERROR = 10
} mg_status;

/* Borrowed CSR view, entry (u, v) = edge u -> v in row u (rowgcn::CsrMatrix, inc/sparse.hpp:25-55). */
typedef struct mg_csr {
  int64_t rows, cols;
  const int64_t* row_ptr; /* rows + 1 */
  const int64_t* col_idx; /* nnz, strictly increasing per row */
  const float* values;    /* nnz */
} mg_csr;

/* Arithmetic modes of the device kernels (reported next to every number). */
typedef enum mg_gemm_mode {
  MG_GEMM_EXACT = 0,  /* SIMT, k-ascending separate mul/add: bitwise equal to rowgcn::gemm (f32) */
  MG_GEMM_TF32X3 = 1, /* tcgen05, 3-term split (hi*hi + hi*lo + lo*hi): fp32-level accuracy. kind::tf32 for the
                       * W-grad and (default) NN / NT; opt-in "gemm_f16": NN / NT fed by FAST SpMM on per-row /
                       * per-column scaled fp16 pairs, kind::f16 */
  MG_GEMM_TF32 = 2    /* tcgen05 kind::tf32, single term (reported separately, rel ~1e-3) */
} mg_gemm_mode;

typedef enum mg_spmm_mode {
  MG_SPMM_EXACT = 0, /* per-row column-order separate mul/add: bitwise equal to rowgcn::spmm (f32) */
  MG_SPMM_FAST = 1   /* long rows split across warps + fixed-order second pass (deterministic, tolerance) */
} mg_spmm_mode;

/* rowgcn::GcnConfig (inc/gcn.hpp:14-36) plus the device arithmetic modes. */
typedef struct mg_config {
  const int64_t* layer_dims; /* [d0, d1, ..., dL] */
  int32_t n_dims;
  double lr, beta1, beta2, epsilon;
  int32_t epochs;
  uint64_t seed;
  uint8_t permute, overlap, skip_first_backward_spmm, order_swap;
  int32_t gemm_mode; /* mg_gemm_mode */
  int32_t spmm_mode; /* mg_spmm_mode */
  /* 1: in MG_SPMM_FAST, layer 0 runs as (Â·X)·W0 and W0's gradient as (Â·X)^T·G0 (Â·X kept from the
   * forward) whenever d0 < 2·d1 and skip_first_backward_spmm is off: one d0-wide SpMM replaces the
   * forward and backward d1-wide ones (the association inc/gcn.hpp:254-260 uses under order_swap, carried
   * into the backward). Mathematically the same gradient; float order differs, so EXACT ignores it. */
  int32_t aggregate_input;
  /* Default-off extensions (no reference analogue: the reference has neither; no parity claim;
   * not part of the config JSON schema). bias = 1: every layer adds a learned bias row b_l (zero-initialised,
   * Adam-updated, its gradient reduced over the canonical W-grad blocks like W_G). dropout = p in [0, 1):
   * during train_step / compute_gradients each hidden layer's output (after bias + ReLU) is kept with
   * probability 1 - p and scaled by 1 / (1 - p); the mask is a counter hash of (seed, step, layer, global
   * row, column), fused into the producing kernel's epilogue and recovered by relu_backward from the
   * output itself. loss_only / forward (evaluation) apply no dropout. */
  int32_t bias;
  double dropout;
} mg_config;

/* Fills the reference defaults (inc/gcn.hpp:16-25): lr 0.01, betas 0.9/0.999, eps 1e-8, 100 epochs,
 * seed 1, flags off; gemm_mode TF32X3, spmm_mode FAST (both within rel 1e-4 of the reference; EXACT gives
 * bitwise parity). layer_dims left NULL. */
void mg_config_defaults(mg_config* cfg);
/* GcnConfig::validate (inc/gcn.hpp:29-35) -> MG_CONFIG_ERROR. */
mg_status mg_config_validate(const mg_config* cfg);

const char* mg_last_error(void);
int32_t mg_abi_version(void);
/* Process-wide tuning knobs (no reference analogue; defaults in DESIGN.md):
 *   "heavy_row"  nonzeros from which a tile row takes the cp.async hub-row SpMM path (default 4096)
 *   "profile"    1 = record per-kernel CUDA events during steps (mg_group_last_profile)
 *   "step_graph" 1 (default): training steps of one-worker groups (no collectives) are captured once as a
 *                CUDA graph and replayed (Adam's per-step constants patched into the graph); not used with
 *                the timeline, "profile", dropout or the stall hook; 0: every kernel launched per step
 *   "ax_cache"   1: under aggregate_input (MG_SPMM_FAST), a one-process group computes layer 0's Â·X once
 *                and reuses it until the features are written (mg_group_write MG_T_X) or the tuning changes
 *                (bitwise the same steps; one d0-wide SpMM fewer per step); 0 (default): every step, like
 *                the reference
 *   "tn_chunk"   W-grad split-K chunk in rows (multiple of 256, default 4096)
 *   "fast_segment"  hub-row segment length of MG_SPMM_FAST (default 2048)
 *   "spmm_slab" / "spmm_narrow_group"  SpMM launch-geometry experiments (default 0 = off)
 *   "spmm_async"   MG_SPMM_FAST gathers through the cp.async shared-memory ring (default 1)
 *   "spmm_hub_bytes"  L2 footprint of the rows given evict_last priority (default 96 MiB; 0 = no hints)
 *   "gemm_kernel"  tcgen05 GeMM variant: 1 = both split operands in smem, 2 = A split into TMEM,
 *                  3 = 2 with 32-K stages and decoupled A / W rings for NN / NT (default)
 *   "gemm3_wring"  v3 W-ring budget in bytes (default 96 KiB); "gemm3_cluster" 2: NN / NT with two 128-column
 *                  tiles run as 2-CTA clusters that multicast each A stage to both tiles (one A read from
 *                  HBM / L2 per row tile), 1: one CTA per tile
 *   "gemm_f16"     1: TF32X3 NN / NT whose A has producer-written row maxima (FAST SpMM; groups created
 *                  while it is on) run the scaled fp16 two-term split on kind::f16 when K > "gemm_f16_min_k"
 *                  (default 128); 0 (default): the 3xTF32 split everywhere
 *   "stage_fold"   k >= 2: MG_SPMM_FAST with P > 2 folds up to k consecutive received stages into one SpMM
 *                  launch over a merged tile (one output read-modify-write pass per group; receive buffers
 *                  k blocks deep); 0 (default) or 1: stage by stage
 *   "spmm_stream" 0 / 1 / 2 (auto, default): the row-streaming FAST SpMM for short-row tiles
 *   "adaptive_cuts" 1 (default): FAST hub-row cut points scaled to the tile; "piece_nnz" stream piece size
 *   "l2_persist_mb"  L2 set-aside for persisting (evict_last) lines on the current device (default 0;
 *                  measured: the SpMM gains < 1 ms, the GeMMs lose 3-5 ms per C4 epoch)
 *   "gemm_f16_min_k"  K above which the opt-in fp16 split runs (default 128)
 *   "bwd_transpose"  one worker: build the backward tile on the device from the forward one (default 1)
 *   "block_cache"  1 (default): device blocks of destroyed groups are kept for reuse; 0: released (cold runs)
 *   "watchdog_ms"  host-wait timeout after which a group is aborted with MG_SHUTDOWN_ERROR (default 0 = none)
 *   "debug_stall_us" / "nccl_single"  test hooks: a spin kernel at every step start; an NCCL communicator
 *                  (and NCCL collectives) for one-rank groups too */
mg_status mg_set_tuning(const char* key, int64_t value);

/* ---------------------------------------------------------------- host datasets
 * rowgcn::Dataset (inc/dataset.hpp:19-56). Held in host memory, float32. */
typedef struct mg_dataset mg_dataset;

/* rowgcn::synth_graph<float> (inc/dataset.hpp:287-334), bit-identical output. */
mg_status mg_dataset_synth(int64_t n, double avg_degree, double exponent, uint64_t seed, int64_t feature_dim,
                           int32_t classes, mg_dataset** out);
/* Copies caller arrays into a dataset (the Dataset struct fields). train_mask may be NULL (= all). */
mg_status mg_dataset_from_arrays(const mg_csr* graph, const float* features, int64_t d0, const int32_t* labels,
                                 const uint8_t* train_mask, mg_dataset** out);
/* Borrowed views into the dataset (valid until mg_dataset_free). *train_mask is NULL when absent. */
mg_status mg_dataset_view(const mg_dataset* ds, mg_csr* graph, const float** features, int64_t* d0,
                          const int32_t** labels, const uint8_t** train_mask);
/* Dataset::num_classes (inc/dataset.hpp:51-55). */
int32_t mg_dataset_num_classes(const mg_dataset* ds);
/* Dataset::validate (inc/dataset.hpp:30-44) + CsrMatrix::validate (inc/sparse.hpp:37-54). */
mg_status mg_dataset_validate(const mg_dataset* ds);
void mg_dataset_free(mg_dataset* ds);
/* Borrowed val / test / train masks (NULL when the dataset has none); Dataset::{train,val,test}_mask. */
mg_status mg_dataset_masks(const mg_dataset* ds, const uint8_t** train, const uint8_t** val, const uint8_t** test);

/* ---------------------------------------------------------------- on-disk formats
 * rowgcn loaders (inc/dataset.hpp:84-280, inc/dense.hpp:290-335), multi-threaded, same accepted syntax,
 * same exception types (MG_IO_ERROR: cannot open / short write; MG_PARSE_ERROR: "path:line: ..." for
 * malformed text) and messages. Graphs are built like from_coo (inc/sparse.hpp:59-90): rows sorted,
 * duplicate (u, v) weights summed (in file order). */
typedef struct mg_graph mg_graph;  /* owned CSR */
typedef struct mg_dense mg_dense;  /* owned row-major float matrix */

/* load_dataset<float>(graph, features, labels, masks) (dataset.hpp:264-276); masks_path NULL or "" = none.
 * The graph format is sniffed like load_graph; validates like Dataset::validate (name = graph_path). */
mg_status mg_dataset_load(const char* graph_path, const char* features_path, const char* labels_path,
                          const char* masks_path, mg_dataset** out);
/* format 0 = load_graph (sniff "%%MatrixMarket", dataset.hpp:170-180), 1 = load_matrix_market
 * (:87-143), 2 = load_edge_list (:147-168). */
mg_status mg_graph_load(const char* path, int32_t format, mg_graph** out);
mg_status mg_graph_view(const mg_graph* g, mg_csr* out); /* borrowed, valid until mg_graph_free */
void mg_graph_free(mg_graph* g);
/* load_features<float> (dataset.hpp:184-216): MGDM binary (by magic) or CSV rows. */
mg_status mg_dense_load(const char* path, mg_dense** out);
/* read_dense<float> (dense.hpp:311-335): MGDM only; f64 payloads are converted. */
mg_status mg_dense_read(const char* path, mg_dense** out);
mg_status mg_dense_view(const mg_dense* d, int64_t* rows, int64_t* cols, const float** data);
void mg_dense_free(mg_dense* d);
/* write_dense<float> (dense.hpp:293-307): "MGDM", u64 rows, u64 cols, u8 4, payload. */
mg_status mg_dense_write(const char* path, int64_t rows, int64_t cols, const float* data);
/* from_coo<float> (sparse.hpp:59-90): n x n CSR from `count` edges (src[e] -> dst[e], weight[e]); rows
 * sorted, duplicate (src, dst) weights summed (in edge order). ValueError on an out-of-range endpoint. */
mg_status mg_graph_from_coo(int64_t n, int64_t count, const int64_t* src, const int64_t* dst, const float* weight,
                            mg_graph** out);
/* add_self_loops<float> (dataset.hpp:60-73): a unit (u, u) entry in every row that lacks one, rebuilt like
 * from_coo (sparse.hpp:59-90). The result is an owned graph (mg_graph_view / mg_graph_free). */
mg_status mg_graph_add_self_loops(const mg_csr* a, mg_graph** out);
/* load_labels (dataset.hpp:218-234). *count = number of labels; dst (capacity entries) may be NULL to
 * query the count first. */
mg_status mg_labels_load(const char* path, int32_t* dst, int64_t capacity, int64_t* count);
/* load_masks (dataset.hpp:237-262) for n vertices; each non-NULL output gets n bytes when its key is
 * present. *present: bit 0 train, bit 1 val, bit 2 test. */
mg_status mg_masks_load(const char* path, int64_t n, uint8_t* train, uint8_t* val, uint8_t* test, int32_t* present);

/* ---------------------------------------------------------------- checkpoints and JSON documents
 * write_checkpoint / read_checkpoint<float> (inc/driver.hpp:255-299): every W as an MGDM block ("MGDM",
 * u64 rows, u64 cols, u8 width 4, payload) back to back, plus the sidecar <path>.json holding
 * config_to_json(cfg) (driver.hpp:59-71) as nlohmann::json::dump(1) writes it (byte-identical).
 * Errors: MG_IO_ERROR "cannot open <path> ..." / "short write to <path>"; MG_PARSE_ERROR on a bad magic,
 * a dtype width other than 4 or a truncated block. */
typedef struct mg_checkpoint mg_checkpoint;
mg_status mg_checkpoint_write(const char* path, int32_t count, const int64_t* rows, const int64_t* cols,
                              const float* const* data, const mg_config* cfg);
mg_status mg_checkpoint_read(const char* path, mg_checkpoint** out);
int32_t mg_checkpoint_count(const mg_checkpoint* ck);
mg_status mg_checkpoint_view(const mg_checkpoint* ck, int32_t i, int64_t* rows, int64_t* cols, const float** data);
void mg_checkpoint_free(mg_checkpoint* ck);
/* config_to_json(cfg).dump(indent) (driver.hpp:59-71; indent < 0 = compact) and BreakdownReport::to_json()
 * .dump(indent) / text_table() (inc/breakdown.hpp:27-58) over runtime_breakdown totals
 * {spmm, gemm, activation, loss, adam, comm}. *length = text length; buf (capacity bytes, may be NULL)
 * receives the NUL-terminated text, truncated to capacity - 1. */
mg_status mg_config_to_json(const mg_config* cfg, int32_t indent, char* buf, int64_t capacity, int64_t* length);
mg_status mg_breakdown_to_json(const double totals_us[6], int32_t indent, char* buf, int64_t capacity,
                               int64_t* length);
mg_status mg_breakdown_text(const double totals_us[6], char* buf, int64_t capacity, int64_t* length);

/* ---------------------------------------------------------------- partitioner
 * rowgcn::prepare_data (inc/driver.hpp:87-117): random_permutation (partition.hpp:69-79), permute
 * rows/graph (:101-140), uniform_partition (:42-49), normalize_in_degree (sparse.hpp:94-107),
 * transpose (:110-129), tile_rows (partition.hpp:173-225). Bit-identical to the reference.
 * only_rank = -1 builds every row block's tiles; r >= 0 builds only row block r (one process per GPU). */
typedef struct mg_partition mg_partition;

mg_status mg_prepare(const mg_dataset* ds, const mg_config* cfg, int32_t workers, int32_t only_rank,
                     mg_partition** out);
/* The same partition (bit-identical tiles), with permute_graph / transpose / normalize_in_degree /
 * tile_rows run on CUDA device `device` as radix sorts of (row, column) keys — the papers-scale path
 * (SURVEY §8f row 1): no host COO, ~28 bytes of device memory per nonzero at the peak. */
mg_status mg_prepare_device(const mg_dataset* ds, const mg_config* cfg, int32_t workers, int32_t only_rank,
                            int32_t device, mg_partition** out);
/* n, global mask count and the P+1 part bounds (PartitionVector::bounds). */
mg_status mg_partition_info(const mg_partition* p, int64_t* n, int64_t* mask_count, int64_t* bounds);
/* dir 0 = forward tiles of A_hat^T, dir 1 = backward tiles of A_hat (PreparedData::fwd/bwd_tiles). */
mg_status mg_partition_tile_info(const mg_partition* p, int32_t dir, int32_t i, int32_t j, int64_t* rows,
                                 int64_t* cols, int64_t* nnz);
mg_status mg_partition_tile_export(const mg_partition* p, int32_t dir, int32_t i, int32_t j, int64_t* row_ptr,
                                   int64_t* col_idx, float* values);
/* Permuted features, labels and mask of the stored rows (rows_info: [row0, row0 + rows); every row for
 * mg_prepare / mg_prepare_device, the rank's row block for mg_synth_rank_finish) and the permutation's
 * forward map over all n vertices (old id -> new id). */
mg_status mg_partition_rows_export(const mg_partition* p, float* features, int32_t* labels, uint8_t* mask,
                                   int64_t* perm_forward);
mg_status mg_partition_rows_info(const mg_partition* p, int64_t* row0, int64_t* rows);
void mg_partition_free(mg_partition* p);

/* ---------------------------------------------------------------- per-rank synthetic input (papers scale)
 * synth_graph (inc/dataset.hpp:287-334) + prepare_data (inc/driver.hpp:87-117) fused for ONE rank of a
 * P-way job, without materialising the whole graph or all features: the rank replays the generator's
 * mt19937_64 stream (stub draws, then the feature and label draws with the other ranks' rows skipped),
 * keeps the adjacency rows it owns after the permutation, and needs from the other ranks only the
 * deduplicated degree of every vertex (normalize_in_degree's column sums; a symmetric graph's column sum
 * is its row length). The partition it returns is bit-identical to row block `rank` of
 * prepare_data(synth_graph(...), cfg, P) (only_rank = rank).
 *   open    replays the stub stream, builds the rank's rows; flags MG_SYNTH_GRAPH_ONLY skips features
 *   degrees the rank's row lengths (degrees of vertices row0 .. row0 + rows - 1, permuted ids)
 *   block_degrees  the same for any row block b, computed from the kept stub stream (a lone process
 *           derives every degree this way: P passes of 1/P of the graph each, no collective)
 *   finish  takes every vertex's degree (n entries, permuted ids; NULL = compute via block_degrees) and
 *           emits the rank's forward and backward tiles, rows and labels; the handle's graph state is
 *           released. */
typedef struct mg_synth_rank mg_synth_rank;
#define MG_SYNTH_GRAPH_ONLY 1
mg_status mg_synth_rank_open(int64_t n, double avg_degree, double exponent, uint64_t seed, int64_t feature_dim,
                             int32_t classes, const mg_config* cfg, int32_t workers, int32_t rank, int32_t flags,
                             mg_synth_rank** out);
mg_status mg_synth_rank_info(const mg_synth_rank* h, int64_t* row0, int64_t* rows, int64_t* nnz,
                             int64_t* stubs);
mg_status mg_synth_rank_degrees(const mg_synth_rank* h, int32_t* degrees);
mg_status mg_synth_rank_block_degrees(mg_synth_rank* h, int32_t block, int32_t* degrees);
mg_status mg_synth_rank_finish(mg_synth_rank* h, const int32_t* degrees, mg_partition** out);
void mg_synth_rank_free(mg_synth_rank* h);

/* ---------------------------------------------------------------- device training group
 * The set of GcnWorkers (inc/gcn.hpp:101-398) living in this process, plus their communicator
 * (the reference's DeviceGroup, inc/collectives.hpp:58-203). One compute stream (lane 0) and one comm
 * stream (lane 1) per worker; the staged SpMM's dependency graph (inc/dist_spmm.hpp:57-103) is
 * reproduced with CUDA events.
 *   world      total number of workers P (all processes)
 *   n_local    workers driven by this process, with their ranks and CUDA devices
 *   nccl_id    128-byte ncclUniqueId shared by all processes (mg_nccl_unique_id on one process), or
 *              NULL when every rank is local.
 *   transport  MG_TRANSPORT_AUTO picks NCCL when each local worker owns a distinct device (or the group
 *              spans processes) and the in-process peer-copy transport otherwise (several workers per
 *              device — the reference's DeviceGroup semantics, used to test P > #GPUs). */
typedef struct mg_group mg_group;

/* MG_TRANSPORT_SOLO (measurement only): ONE rank of a P-way job alone in the process, its collectives
 * skipped (the receive buffers keep whatever they hold): times one rank's device work on its real
 * partition — e.g. rank 0 of the papers-shaped graph at P = 8 on one GPU — without the other ranks. The
 * numbers it computes are not a training result. */
typedef enum mg_transport {
  MG_TRANSPORT_AUTO = 0,
  MG_TRANSPORT_NCCL = 1,
  MG_TRANSPORT_LOCAL = 2,
  MG_TRANSPORT_SOLO = 3
} mg_transport;

/* Number of visible CUDA devices (0 without a driver/GPU: the host half of the library still works). */
int32_t mg_device_count(void);
mg_status mg_nccl_unique_id(uint8_t id[128]);
mg_status mg_group_create(const mg_config* cfg, const mg_partition* p, int32_t world, int32_t n_local,
                          const int32_t* local_ranks, const int32_t* devices, const uint8_t* nccl_id,
                          int32_t transport, mg_group** out);
/* DeviceGroup::abort (collectives.cpp:42-52), callable from any thread: the current or next host wait on the
 * group aborts its NCCL communicators (ncclCommAbort) and fails with MG_SHUTDOWN_ERROR "device group aborted:
 * ..."; every later call on the group fails the same way (mg_group_destroy still releases it). Host waits
 * also abort on an asynchronous NCCL error (a peer that died) and, with mg_set_tuning("watchdog_ms", T), when
 * a step, a collective or communicator creation has not completed within T ms (a peer that never arrived). */
mg_status mg_group_abort(mg_group* g);
/* GcnWorker::init_params (inc/gcn.hpp:163-173): Glorot from Rng(seed) on the host, replicated. */
mg_status mg_group_init_params(mg_group* g);
/* GcnWorker::train_step(t) (inc/gcn.hpp:175-184). Synchronous; loss = global masked mean, acc =
 * correct / mask count. wall_us (nullable) = device time from step start to optimizer completion on the
 * first local worker (the reference's epoch wall_us, inc/driver.hpp:170-173). */
mg_status mg_group_train_step(mg_group* g, int32_t t, double* loss, double* acc, double* wall_us);
/* GcnWorker::compute_gradients (inc/gcn.hpp:208-217): W_G materialised, no update. */
mg_status mg_group_compute_gradients(mg_group* g, double* loss, double* acc);
/* GcnWorker::loss_only (inc/gcn.hpp:189-205): forward + masked loss, logits left in place. */
mg_status mg_group_loss_only(mg_group* g, double* loss);
/* GcnWorker::submit_forward (inc/gcn.hpp:238-267), synchronous. */
mg_status mg_group_forward(mg_group* g);
/* GcnWorker::submit_backward + submit_finalize(false) (gcn.hpp:292-377): the backward pass from the
 * gradient currently in the logits buffer (MG_T_AHW of layer L-1), then W_G (MG_T_WGRAD) finalized without
 * Adam. H_G lands in MG_T_AHW of layer 0 (masked by relu_backward), as in the reference. */
mg_status mg_group_backward(mg_group* g);
/* Asynchronous train step: enqueue only (no host sync). Results via mg_group_sync + mg_group_last_stats. */
mg_status mg_group_train_step_async(mg_group* g, int32_t t);
mg_status mg_group_sync(mg_group* g);
mg_status mg_group_last_stats(mg_group* g, double* loss, double* acc);

typedef enum mg_tensor {
  MG_T_W = 0,      /* d_l x d_{l+1}      LayerParams::w      */
  MG_T_WGRAD = 1,  /* d_l x d_{l+1}      LayerParams::w_grad */
  MG_T_AHW = 2,    /* local_rows x d_{l+1}  BufferPool::ahw[l] */
  MG_T_HW = 3,     /* local_rows x width    BufferPool::hw (width = d_{layer+1}, caller's view) */
  MG_T_X = 4,      /* local_rows x d0     x_local */
  MG_T_ADAM_M = 5,
  MG_T_ADAM_V = 6,
  MG_T_WSTAGE = 7, /* 8 d_l x d_{l+1}   the canonical-block W-grad staging buffer */
  MG_T_BIAS = 8,   /* 1 x d_{l+1}        bias row of layer l (cfg.bias) */
  MG_T_BIAS_GRAD = 9, /* 1 x d_{l+1}      its gradient (like MG_T_WGRAD) */
  MG_T_ROWMAX = 10 /* local_rows x 2    row-max pairs of the f16 GeMM split, slot `layer` (l < L: ahw[l],
                    * L: hw, L + 1: Â·X); TF32X3 + FAST groups only (diagnostics, read-only use) */
} mg_tensor;

/* Copies a tensor of local worker `rank` to/from host memory in the reference's dense layout
 * (row-major, leading dimension = cols); count must equal the tensor's element count. */
mg_status mg_group_read(mg_group* g, int32_t rank, int32_t which, int32_t layer, float* dst, int64_t count);
mg_status mg_group_write(mg_group* g, int32_t rank, int32_t which, int32_t layer, const float* src, int64_t count);
/* GcnWorker::w_hash (inc/gcn.hpp:221-226): FNV-1a over the W bytes of local worker `rank`. */
mg_status mg_group_w_hash(mg_group* g, int32_t rank, uint64_t* hash);
/* Local rows of worker `rank`: [row_begin, row_begin + rows). */
mg_status mg_group_rows(mg_group* g, int32_t rank, int64_t* row_begin, int64_t* rows);
/* BufferPool::large_buffer_count (inc/gcn.hpp:57) and the device allocation counter used by the L+3
 * buffer audit (tests/test_gcn.cpp:350-368): allocations made inside steps must stay 0. */
mg_status mg_group_buffer_audit(mg_group* g, int32_t* large_buffers, int64_t* step_allocations,
                                int64_t* device_bytes);
/* Device time accumulated since the previous call (then reset), in microseconds, measured with CUDA
 * events on the launching stream of the first local worker when mg_set_tuning("profile", 1) is on:
 * SpMM stages (light + hub-row kernels), GeMMs, and other kernels (loss, finalize/Adam); plus the number
 * of kernels this library launched over the same steps (always counted). */
mg_status mg_group_last_profile(mg_group* g, double* spmm_us, double* gemm_us, double* other_us,
                                int64_t* kernels);
/* Training steps of this group replayed from its captured CUDA graph ("step_graph"), and captures made. */
mg_status mg_group_graph_steps(mg_group* g, int64_t* replays, int64_t* captures);
void mg_group_destroy(mg_group* g);

/* ---------------------------------------------------------------- timeline
 * rowgcn::TimelineEvent (inc/collectives.hpp:24-34): one record per task the reference submits to a
 * worker lane — lane 0 compute ("gemm" hw|wgrad|hgrad, "spmm" stage, "other" loss|adam|wgrad_final),
 * lane 1 comm ("broadcast" h_stage, "reduce" loss|wgrad) — timed by CUDA events on the lane's stream
 * (lane 0 = compute stream, lane 1 = comm stream), microseconds from the worker's base event. stage is
 * the staged-SpMM stage (or the layer for gemm / wgrad reduce, -1 otherwise), as in the reference.
 * The forward ReLU and relu_backward are fused into the SpMM / hgrad epilogues and have no own task. */
typedef struct mg_timeline_event {
  int32_t worker, lane, stage, n_deps;
  char kind[16];
  char op[16];
  double t_start_us, t_end_us;
  uint64_t task;         /* > 0, unique within the group */
  const uint64_t* deps;  /* n_deps task ids this task waited for */
} mg_timeline_event;

/* on != 0: clear and start recording every subsequent step (and mg_group_bench_spmm); 0: stop. */
mg_status mg_group_set_timeline(mg_group* g, int32_t on);
/* Synchronises and returns the recorded events (borrowed, valid until the next timeline call on g):
 * *count = number of events; the first min(count, capacity) are copied to out (out may be NULL). */
mg_status mg_group_timeline(mg_group* g, mg_timeline_event* out, int64_t capacity, int64_t* count);
/* export_timeline (inc/timeline.hpp:31-36): JSON array, one object per event, reference schema. */
mg_status mg_timeline_export(const char* path, const mg_timeline_event* ev, int64_t count);
/* audit_timeline (timeline.hpp:64-94): well formed, per-(worker, lane) non-overlapping, every dependency
 * finished before its dependent started. MG_VALUE_ERROR with the reference's message on violation. */
mg_status mg_timeline_audit(const mg_timeline_event* ev, int64_t count);
/* audit_staged_run (timeline.hpp:96-126) on the events of ONE staged SpMM. */
mg_status mg_timeline_audit_staged(const mg_timeline_event* ev, int64_t count, int32_t world, int32_t overlapped);
/* runtime_breakdown (inc/breakdown.hpp:63-82): totals_us = {spmm, gemm, activation, loss, adam, comm}. */
mg_status mg_timeline_breakdown(const mg_timeline_event* ev, int64_t count, double totals_us[6]);

/* bench-spmm (proj/tools/main.cpp:120-178): one staged SpMM of this group's local feature rows X
 * (width d0) over the dir tiles (0 forward Â^T, 1 backward Â) into the HW buffer (read with MG_T_HW),
 * synchronously. Recorded in the timeline when it is on. *wall_us = device time of the run on rank 0's
 * compute stream. */
mg_status mg_group_bench_spmm(mg_group* g, int32_t dir, double* wall_us);

/* ---------------------------------------------------------------- kernel-level entry points
 * Device pointers, caller's stream (cudaStream_t passed as void*, NULL = legacy default stream).
 * Used by the parity tests and the micro-benchmarks (the reference's bench-spmm, proj/tools/main.cpp:120-178). */

/* rowgcn::spmm (inc/sparse.hpp:161-188) on one tile: out[u, :w] = (accumulate ? out[u] : 0) +
 * sum_e val_e * h[col_e, :w] over row u in column order. h and out are row-major with leading dimension
 * ld (ld % 4 == 0, ld >= w, 16-byte aligned). edges = nnz {int32 col, float val} pairs. relu applies
 * max(0, x) to the final value (the fused relu_forward of the last forward stage, dense.hpp:208-215). */
mg_status mg_dev_spmm(int64_t rows, const int32_t* row_ptr, const void* edges, const float* h, float* out,
                      int64_t w, int64_t ld, int32_t accumulate, int32_t relu, int32_t mode, void* stream);
/* rowgcn::gemm (inc/dense.hpp:140-204) for the three step shapes, row-major with leading dims:
 *   NN: C[M,N] = A[M,K] B[K,N]     TN: C[M,N] = A[K,M]^T B[K,N]     NT: C[M,N] = A[M,K] B[N,K]^T
 * epilogue 0 = store, 1 = relu_backward mask: C = (C_old > 0 ? result : 0) (dense.hpp:221-231),
 * 2 = relu_forward on the result. mode = mg_gemm_mode. */
mg_status mg_dev_gemm(int32_t ta, int32_t tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                      const float* B, int64_t ldb, float* Cm, int64_t ldc, int32_t epilogue, int32_t mode,
                      void* stream);

/* rowgcn::softmax_xent_sum (inc/dense.hpp:241-277) plus the argmax correct count (inc/gcn.hpp:279-282) on
 * device rows: logits[rows, classes] with leading dimension ld is replaced by the gradient
 * (softmax - onehot) / denom on masked rows and 0 elsewhere (columns classes..ld zeroed). stats (HOST,
 * 2 doubles) = {loss sum over masked rows, correct count}. Errors as the reference: ValueError for
 * denom <= 0 ("empty mask") and for a masked label outside [0, classes); classes <= 256. Synchronous. */
mg_status mg_dev_softmax_xent(float* logits, int64_t rows, int64_t classes, int64_t ld, const int32_t* labels,
                              const uint8_t* mask, int64_t denom, double* stats, void* stream);
/* rowgcn::adam_step (inc/gcn.hpp:61-85) on one device parameter array of `size` floats: m, v, w updated
 * with the reference's float constants and operation order, grad zeroed. t >= 1 (ValueError otherwise).
 * Synchronous. */
mg_status mg_dev_adam(float* w, float* grad, float* m, float* v, int64_t size, double lr, double beta1, double beta2,
                      double epsilon, int32_t t, void* stream);

#ifdef __cplusplus
} /* extern "C" */
#endif
#endif /* MGGCN_H_ */
