"""Python mirror of the reference's training API (rowgcn, proj/include/rowgcn/) on top of libmggcn.so.

Same names, argument meaning and error behaviour as the C++ reference so parity tests read like the
reference's own tests:
  errors      inc/errors.hpp:10-39          ShapeError, ValueError, ... (+ CudaError, NcclError)
  GcnConfig   inc/gcn.hpp:14-36             + gemm_mode / spmm_mode (device arithmetic)
  parse_config / materialize_config / config_to_json   inc/driver.hpp:19-71
  write_checkpoint / read_checkpoint        inc/driver.hpp:255-299
  from_coo / add_self_loops                 inc/sparse.hpp:59-90, inc/dataset.hpp:60-73
  Dataset, synth_graph                      inc/dataset.hpp:19-56, :287-334
  load_dataset / load_graph / load_matrix_market / load_edge_list / load_features / load_labels /
  load_masks, read_dense / write_dense      inc/dataset.hpp:84-280, inc/dense.hpp:290-335
  prepare_data / PreparedData               inc/driver.hpp:75-117
  Group (the GcnWorkers of this process)    inc/gcn.hpp:101-398
  TrainOptions / TrainArtifacts / train_run inc/driver.hpp:119-206
  GradArtifacts / grad_run                  inc/driver.hpp:209-251
  fnv1a                                     inc/gcn.hpp:87-94
Every call goes through the C ABI (include/mggcn.h); nothing here computes on the CPU.
"""
from __future__ import annotations

import builtins
import ctypes as C
import json
import sys
from dataclasses import dataclass, field, fields
from typing import Callable, Optional

import numpy as np

from ._lib import lib, mg_config, mg_csr, mg_timeline_event


def _finalizing() -> bool:
    """True during interpreter shutdown, when module globals (lib, ctypes) may already be torn down: the
    process exit releases the native objects then."""
    return sys is None or sys.is_finalizing() or lib is None or C is None

# ----------------------------------------------------------------------------- errors (inc/errors.hpp)


class RowgcnError(RuntimeError):
    pass


class ShapeError(RowgcnError):
    pass


class ValueError(RowgcnError, builtins.ValueError):  # noqa: A001 - mirrors rowgcn::ValueError
    pass


class ProtocolError(RowgcnError):
    pass


class ShutdownError(RowgcnError):
    pass


class ParseError(RowgcnError):
    pass


class ConfigError(RowgcnError):
    pass


class IoError(RowgcnError):
    pass


class CudaError(RowgcnError):
    pass


class NcclError(RowgcnError):
    pass


_STATUS = {1: ShapeError, 2: ValueError, 3: ProtocolError, 4: ShutdownError, 5: ParseError, 6: ConfigError,
           7: IoError, 8: CudaError, 9: NcclError, 10: RowgcnError}

GEMM_EXACT, GEMM_TF32X3, GEMM_TF32 = 0, 1, 2
SPMM_EXACT, SPMM_FAST = 0, 1
TRANSPORT_AUTO, TRANSPORT_NCCL, TRANSPORT_LOCAL, TRANSPORT_SOLO = 0, 1, 2, 3
T_W, T_WGRAD, T_AHW, T_HW, T_X, T_ADAM_M, T_ADAM_V, T_WSTAGE, T_BIAS, T_BIAS_GRAD, T_ROWMAX = range(11)


def _check(rc: int):
    if rc != 0:
        msg = lib().mg_last_error().decode(errors="replace")
        raise _STATUS.get(rc, RowgcnError)(msg)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ----------------------------------------------------------------------------- config (inc/gcn.hpp:14-36)


@dataclass
class GcnConfig:
    layer_dims: list = field(default_factory=list)
    lr: float = 0.01
    beta1: float = 0.9
    beta2: float = 0.999
    epsilon: float = 1e-8
    epochs: int = 100
    seed: int = 1
    permute: bool = False
    overlap: bool = False
    skip_first_backward_spmm: bool = False
    order_swap: bool = False
    gemm_mode: int = GEMM_TF32X3  # production default; GEMM_EXACT/SPMM_EXACT give bitwise parity
    spmm_mode: int = SPMM_FAST
    aggregate_input: bool = True  # FAST only: layer 0 as (A X) W0, A X reused for W0's gradient (mggcn.h)
    bias: bool = False     # default-off extension (no reference analogue): learned bias per layer
    dropout: float = 0.0   # default-off extension: dropout probability of hidden-layer outputs (training)

    def layers(self) -> int:
        return len(self.layer_dims) - 1

    def _c(self):
        dims = np.ascontiguousarray(np.asarray(self.layer_dims, dtype=np.int64))
        c = mg_config(dims.ctypes.data_as(C.c_void_p), len(dims), self.lr, self.beta1, self.beta2, self.epsilon,
                      self.epochs, self.seed, int(self.permute), int(self.overlap),
                      int(self.skip_first_backward_spmm), int(self.order_swap), self.gemm_mode, self.spmm_mode,
                      int(self.aggregate_input), int(self.bias), float(self.dropout))
        c._keep = dims
        return c

    def validate(self):
        _check(lib().mg_config_validate(C.byref(self._c())))


@dataclass
class ConfigFile:
    hidden_dims: list = field(default_factory=lambda: [16])
    cfg: GcnConfig = field(default_factory=GcnConfig)


_KNOWN_KEYS = ("hidden_dims", "lr", "beta1", "beta2", "epsilon", "epochs", "seed", "permute", "overlap",
               "skip_first_backward_spmm", "order_swap")


def parse_config(j) -> ConfigFile:
    """inc/driver.hpp:24-47: one JSON document, unknown keys rejected with ConfigError."""
    if isinstance(j, (str, bytes)):
        try:
            j = json.loads(j)
        except json.JSONDecodeError as e:
            raise ParseError(f"config: {e}") from None
    for k in j:
        if k not in _KNOWN_KEYS:
            raise ConfigError(f"config: unknown key '{k}'")
    cf = ConfigFile()
    if "hidden_dims" in j:
        cf.hidden_dims = [int(x) for x in j["hidden_dims"]]
    for k in _KNOWN_KEYS[1:]:
        if k in j:
            setattr(cf.cfg, k, type(getattr(cf.cfg, k))(j[k]))
    return cf


def materialize_config(cf: ConfigFile, d0: int, classes: int) -> GcnConfig:
    """inc/driver.hpp:49-57: layer_dims = [d0, hidden..., classes], validated."""
    kw = {f.name: getattr(cf.cfg, f.name) for f in fields(GcnConfig)}
    kw["layer_dims"] = [int(d0)] + list(cf.hidden_dims) + [int(classes)]
    cfg = GcnConfig(**kw)
    cfg.validate()
    return cfg


def config_to_json(cfg: GcnConfig) -> dict:
    """inc/driver.hpp:59-71"""
    return {"layer_dims": list(cfg.layer_dims), "lr": cfg.lr, "beta1": cfg.beta1, "beta2": cfg.beta2,
            "epsilon": cfg.epsilon, "epochs": cfg.epochs, "seed": cfg.seed, "permute": cfg.permute,
            "overlap": cfg.overlap, "skip_first_backward_spmm": cfg.skip_first_backward_spmm,
            "order_swap": cfg.order_swap}


def _text(fn, *args) -> str:
    n = C.c_int64()
    _check(fn(*args, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(fn(*args, buf, n.value + 1, C.byref(n)))
    return buf.raw[:n.value].decode()


def config_to_json_text(cfg: GcnConfig, indent: int = -1) -> str:
    """config_to_json(cfg).dump(indent) as the reference's nlohmann::json writes it (byte-identical)."""
    return _text(lib().mg_config_to_json, C.byref(cfg._c()), int(indent))


def write_checkpoint(path, ws, cfg: GcnConfig):
    """write_checkpoint<float> (driver.hpp:255-274): MGDM blocks back to back + <path>.json sidecar."""
    arrs = [np.ascontiguousarray(w, np.float32) for w in ws]
    for a in arrs:
        if a.ndim != 2:
            raise ShapeError(f"write_checkpoint: expected matrices, got shape {a.shape}")
    rows = np.array([a.shape[0] for a in arrs], np.int64)
    cols = np.array([a.shape[1] for a in arrs], np.int64)
    ptrs = (C.c_void_p * max(1, len(arrs)))(*[a.ctypes.data for a in arrs])
    _check(lib().mg_checkpoint_write(_enc(path), len(arrs), _p(rows), _p(cols), ptrs, C.byref(cfg._c())))


def read_checkpoint(path) -> list:
    """read_checkpoint<float> (driver.hpp:276-299)."""
    h = C.c_void_p()
    _check(lib().mg_checkpoint_read(_enc(path), C.byref(h)))
    try:
        out = []
        for i in range(lib().mg_checkpoint_count(h)):
            r, c, d = C.c_int64(), C.c_int64(), C.c_void_p()
            _check(lib().mg_checkpoint_view(h, i, C.byref(r), C.byref(c), C.byref(d)))
            n = r.value * c.value
            out.append(np.zeros((r.value, c.value), np.float32) if n == 0 else
                       np.ctypeslib.as_array(C.cast(d, C.POINTER(C.c_float)), (n,)).reshape(r.value, c.value).copy())
        return out
    finally:
        lib().mg_checkpoint_free(h)


# ----------------------------------------------------------------------------- dataset (inc/dataset.hpp)


class Dataset:
    """rowgcn::Dataset in host memory (owned by libmggcn)."""

    def __init__(self, handle, name: str = ""):
        self._h = C.c_void_p(handle)
        self.name = name

    @classmethod
    def from_arrays(cls, row_ptr, col_idx, values, features, labels, train_mask=None, name="arrays"):
        rp = np.ascontiguousarray(row_ptr, np.int64)
        ci = np.ascontiguousarray(col_idx, np.int64)
        v = np.ascontiguousarray(values, np.float32)
        x = np.ascontiguousarray(features, np.float32)
        lab = np.ascontiguousarray(labels, np.int32)
        m = None if train_mask is None else np.ascontiguousarray(train_mask, np.uint8)
        n = len(rp) - 1
        g = mg_csr(n, n, _p(rp), _p(ci), _p(v))
        out = C.c_void_p()
        _check(lib().mg_dataset_from_arrays(C.byref(g), _p(x), x.shape[1] if x.ndim == 2 else 0, _p(lab), _p(m),
                                            C.byref(out)))
        return cls(out.value, name)

    def __del__(self, _fin=_finalizing):  # bound at definition: module globals may be gone at exit
        h = getattr(self, "_h", None)
        if h and h.value and not _fin():
            try:
                lib().mg_dataset_free(h)
            except Exception:  # interpreter teardown: the process exit releases the native object
                return
            self._h = C.c_void_p()

    def _view(self):
        g = mg_csr()
        f = C.c_void_p()
        d0 = C.c_int64()
        lab = C.c_void_p()
        m = C.c_void_p()
        _check(lib().mg_dataset_view(self._h, C.byref(g), C.byref(f), C.byref(d0), C.byref(lab), C.byref(m)))
        return g, f, d0.value, lab, m

    def n(self) -> int:
        return int(self._view()[0].rows)

    @property
    def graph(self):
        """(row_ptr, col_idx, values) as numpy copies."""
        g = self._view()[0]
        n = g.rows
        rp = np.ctypeslib.as_array(C.cast(g.row_ptr, C.POINTER(C.c_int64)), (n + 1,)).copy()
        nnz = int(rp[-1])
        ci = np.ctypeslib.as_array(C.cast(g.col_idx, C.POINTER(C.c_int64)), (max(nnz, 1),))[:nnz].copy()
        v = np.ctypeslib.as_array(C.cast(g.values, C.POINTER(C.c_float)), (max(nnz, 1),))[:nnz].copy()
        return rp, ci, v

    @property
    def features(self):
        g, f, d0, _, _ = self._view()
        return np.ctypeslib.as_array(C.cast(f, C.POINTER(C.c_float)), (g.rows * d0,)).reshape(g.rows, d0).copy()

    @property
    def labels(self):
        g, _, _, lab, _ = self._view()
        return np.ctypeslib.as_array(C.cast(lab, C.POINTER(C.c_int32)), (g.rows,)).copy()

    @property
    def nnz(self) -> int:
        return int(self.graph[0][-1])

    @property
    def d0(self) -> int:
        return self._view()[2]

    def num_classes(self) -> int:
        return int(lib().mg_dataset_num_classes(self._h))

    def validate(self):
        _check(lib().mg_dataset_validate(self._h))


def _masks(ds_handle):
    tr, va, te = C.c_void_p(), C.c_void_p(), C.c_void_p()
    _check(lib().mg_dataset_masks(ds_handle, C.byref(tr), C.byref(va), C.byref(te)))
    return tr.value, va.value, te.value


def _mask_array(ptr, n):
    if not ptr:
        return np.zeros(0, np.uint8)
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), (n,)).copy()


Dataset.train_mask = property(lambda self: _mask_array(_masks(self._h)[0], self.n()),
                              doc="Dataset::train_mask (empty = all vertices)")
Dataset.val_mask = property(lambda self: _mask_array(_masks(self._h)[1], self.n()), doc="Dataset::val_mask")
Dataset.test_mask = property(lambda self: _mask_array(_masks(self._h)[2], self.n()), doc="Dataset::test_mask")


# ----------------------------------------------------------------------------- on-disk formats
# (inc/dataset.hpp:84-280, inc/dense.hpp:290-335) — native multi-threaded loaders in libmggcn.


def _enc(path) -> bytes:
    return str(path).encode()


def _graph(fmt: int, path) -> tuple:
    h = C.c_void_p()
    _check(lib().mg_graph_load(_enc(path), fmt, C.byref(h)))
    try:
        g = mg_csr()
        _check(lib().mg_graph_view(h, C.byref(g)))
        n = g.rows
        rp = np.ctypeslib.as_array(C.cast(g.row_ptr, C.POINTER(C.c_int64)), (n + 1,)).copy()
        nnz = int(rp[-1])
        if nnz == 0:
            return rp, np.zeros(0, np.int64), np.zeros(0, np.float32)
        ci = np.ctypeslib.as_array(C.cast(g.col_idx, C.POINTER(C.c_int64)), (nnz,)).copy()
        v = np.ctypeslib.as_array(C.cast(g.values, C.POINTER(C.c_float)), (nnz,)).copy()
        return rp, ci, v
    finally:
        lib().mg_graph_free(h)


def _graph_out(h) -> tuple:
    try:
        g = mg_csr()
        _check(lib().mg_graph_view(h, C.byref(g)))
        n = g.rows
        rp = np.ctypeslib.as_array(C.cast(g.row_ptr, C.POINTER(C.c_int64)), (n + 1,)).copy()
        nnz = int(rp[-1])
        if nnz == 0:
            return rp, np.zeros(0, np.int64), np.zeros(0, np.float32)
        ci = np.ctypeslib.as_array(C.cast(g.col_idx, C.POINTER(C.c_int64)), (nnz,)).copy()
        v = np.ctypeslib.as_array(C.cast(g.values, C.POINTER(C.c_float)), (nnz,)).copy()
        return rp, ci, v
    finally:
        lib().mg_graph_free(h)


def from_coo(src, dst, weight, n: int) -> tuple:
    """from_coo<float> (sparse.hpp:59-90): (row_ptr, col_idx, values), rows sorted, duplicates summed."""
    s = np.ascontiguousarray(src, np.int64)
    d = np.ascontiguousarray(dst, np.int64)
    w = np.ascontiguousarray(weight, np.float32)
    if not (len(s) == len(d) == len(w)):
        raise ShapeError("from_coo: src / dst / weight lengths differ")
    h = C.c_void_p()
    _check(lib().mg_graph_from_coo(int(n), len(s), _p(s), _p(d), _p(w), C.byref(h)))
    return _graph_out(h)


def add_self_loops(row_ptr, col_idx, values, cols=None) -> tuple:
    """add_self_loops<float> (dataset.hpp:60-73)."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    ci = np.ascontiguousarray(col_idx, np.int64)
    v = np.ascontiguousarray(values, np.float32)
    n = len(rp) - 1
    g = mg_csr(n, n if cols is None else int(cols), rp.ctypes.data, ci.ctypes.data, v.ctypes.data)
    h = C.c_void_p()
    _check(lib().mg_graph_add_self_loops(C.byref(g), C.byref(h)))
    return _graph_out(h)


def load_graph(path):
    """load_graph<float> (dataset.hpp:170-180): (row_ptr, col_idx, values) of the sorted, deduplicated CSR."""
    return _graph(0, path)


def load_matrix_market(path):
    """load_matrix_market<float> (dataset.hpp:87-143)."""
    return _graph(1, path)


def load_edge_list(path):
    """load_edge_list<float> (dataset.hpp:147-168)."""
    return _graph(2, path)


def _dense(fn, path) -> np.ndarray:
    h = C.c_void_p()
    _check(fn(_enc(path), C.byref(h)))
    try:
        r, c, d = C.c_int64(), C.c_int64(), C.c_void_p()
        _check(lib().mg_dense_view(h, C.byref(r), C.byref(c), C.byref(d)))
        n = r.value * c.value
        if n == 0:
            return np.zeros((r.value, c.value), np.float32)
        return np.ctypeslib.as_array(C.cast(d, C.POINTER(C.c_float)), (n,)).reshape(r.value, c.value).copy()
    finally:
        lib().mg_dense_free(h)


def load_features(path) -> np.ndarray:
    """load_features<float> (dataset.hpp:184-216): MGDM binary or CSV."""
    return _dense(lib().mg_dense_load, path)


def read_dense(path) -> np.ndarray:
    """read_dense<float> (dense.hpp:311-335)."""
    return _dense(lib().mg_dense_read, path)


def write_dense(path, m):
    """write_dense<float> (dense.hpp:293-307)."""
    a = np.ascontiguousarray(m, np.float32)
    if a.ndim != 2:
        raise ShapeError(f"write_dense: expected a matrix, got shape {a.shape}")
    _check(lib().mg_dense_write(_enc(path), a.shape[0], a.shape[1], _p(a)))


def load_labels(path) -> np.ndarray:
    """load_labels (dataset.hpp:218-234)."""
    cnt = C.c_int64()
    _check(lib().mg_labels_load(_enc(path), None, 0, C.byref(cnt)))
    out = np.zeros(cnt.value, np.int32)
    _check(lib().mg_labels_load(_enc(path), _p(out), cnt.value, C.byref(cnt)))
    return out[: cnt.value]


def load_masks(path, n: int):
    """load_masks (dataset.hpp:237-262) -> (train, val, test); an absent key gives an empty array."""
    arrs = [np.zeros(n, np.uint8) for _ in range(3)]
    present = C.c_int32()
    _check(lib().mg_masks_load(_enc(path), int(n), *[_p(a) for a in arrs], C.byref(present)))
    return tuple(a if present.value & (1 << i) else np.zeros(0, np.uint8) for i, a in enumerate(arrs))


def load_dataset(graph_path, features_path, labels_path, masks_path="") -> Dataset:
    """load_dataset<float> (dataset.hpp:264-276); validates like Dataset::validate."""
    out = C.c_void_p()
    _check(lib().mg_dataset_load(_enc(graph_path), _enc(features_path), _enc(labels_path),
                                 _enc(masks_path) if masks_path else None, C.byref(out)))
    return Dataset(out.value, str(graph_path))


def synth_graph(n, avg_degree, exponent, seed, feature_dim=16, classes=4) -> Dataset:
    """rowgcn::synth_graph<float> (inc/dataset.hpp:287-334), bit-identical output."""
    out = C.c_void_p()
    _check(lib().mg_dataset_synth(int(n), float(avg_degree), float(exponent), int(seed), int(feature_dim),
                                  int(classes), C.byref(out)))
    return Dataset(out.value, f"synth-n{n}-d{avg_degree}")


# ----------------------------------------------------------------------------- partitioner (driver.hpp:75-117)


class PreparedData:
    def __init__(self, handle, workers: int):
        self._h = C.c_void_p(handle)
        self.workers = workers
        n = C.c_int64()
        mc = C.c_int64()
        b = np.zeros(workers + 1, np.int64)
        _check(lib().mg_partition_info(self._h, C.byref(n), C.byref(mc), _p(b)))
        self.n = n.value
        self.mask_count = mc.value
        self.bounds = b

    def __del__(self, _fin=_finalizing):  # bound at definition: module globals may be gone at exit
        h = getattr(self, "_h", None)
        if h and h.value and not _fin():
            try:
                lib().mg_partition_free(h)
            except Exception:  # interpreter teardown: the process exit releases the native object
                return
            self._h = C.c_void_p()

    def tile(self, direction: int, i: int, j: int):
        """(row_ptr, col_idx, values) of tile (i, j); direction 0 = A_hat^T (forward), 1 = A_hat."""
        r, c, z = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib().mg_partition_tile_info(self._h, direction, i, j, C.byref(r), C.byref(c), C.byref(z)))
        rp = np.zeros(r.value + 1, np.int64)
        ci = np.zeros(max(z.value, 1), np.int64)
        v = np.zeros(max(z.value, 1), np.float32)
        _check(lib().mg_partition_tile_export(self._h, direction, i, j, _p(rp), _p(ci), _p(v)))
        return rp, ci[:z.value], v[:z.value]

    def rows_info(self):
        """(row0, rows): the permuted rows whose features / labels / mask this partition holds."""
        r0, r = C.c_int64(), C.c_int64()
        _check(lib().mg_partition_rows_info(self._h, C.byref(r0), C.byref(r)))
        return r0.value, r.value

    def rows_export(self, d0: int):
        """Permuted features, labels and mask of the stored rows (rows_info), and the forward permutation."""
        rows = self.rows_info()[1]
        x = np.zeros((rows, d0), np.float32)
        lab = np.zeros(rows, np.int32)
        m = np.zeros(rows, np.uint8)
        pf = np.zeros(self.n, np.int64)
        _check(lib().mg_partition_rows_export(self._h, _p(x), _p(lab), _p(m), _p(pf)))
        return x, lab, m, pf


def prepare_data(ds: Dataset, cfg: GcnConfig, workers: int, only_rank: int = -1,
                 device: Optional[int] = None) -> PreparedData:
    """inc/driver.hpp:87-117. device=None: host partitioner; device=k: the graph work on CUDA device k
    (mg_prepare_device: radix sorts of (row, column) keys), bit-identical tiles."""
    out = C.c_void_p()
    if device is None:
        _check(lib().mg_prepare(ds._h, C.byref(cfg._c()), int(workers), int(only_rank), C.byref(out)))
    else:
        _check(lib().mg_prepare_device(ds._h, C.byref(cfg._c()), int(workers), int(only_rank), int(device),
                                       C.byref(out)))
    return PreparedData(out.value, workers)


class SynthRank:
    """One rank's share of synth_graph + prepare_data without the whole graph (mg_synth_rank_*, mggcn.h):
    open replays the generator's stream and keeps the rank's rows; degrees() are the rank's row lengths,
    block_degrees(b) any block's (from the kept stub stream); finish(all_degrees) emits the partition."""

    def __init__(self, n, avg_degree, exponent, seed, feature_dim, classes, cfg: GcnConfig, workers: int,
                 rank: int, graph_only: bool = False):
        out = C.c_void_p()
        self._h = C.c_void_p()
        _check(lib().mg_synth_rank_open(int(n), float(avg_degree), float(exponent), int(seed), int(feature_dim),
                                        int(classes), C.byref(cfg._c()), int(workers), int(rank),
                                        1 if graph_only else 0, C.byref(out)))
        self._h = C.c_void_p(out.value)
        self.n, self.workers, self.rank = int(n), int(workers), int(rank)
        r0, r, z, st = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib().mg_synth_rank_info(self._h, C.byref(r0), C.byref(r), C.byref(z), C.byref(st)))
        self.row0, self.rows, self.nnz, self.stubs = r0.value, r.value, z.value, st.value

    def __del__(self, _fin=_finalizing):  # bound at definition: module globals may be gone at exit
        h = getattr(self, "_h", None)
        if h and h.value and not _fin():
            try:
                lib().mg_synth_rank_free(h)
            except Exception:  # interpreter teardown: the process exit releases the native object
                return
            self._h = C.c_void_p()

    def degrees(self) -> np.ndarray:
        d = np.zeros(max(self.rows, 1), np.int32)
        _check(lib().mg_synth_rank_degrees(self._h, _p(d)))
        return d[:self.rows]

    def block_degrees(self, block: int) -> np.ndarray:
        b0, b1 = int(block) * self.n // self.workers, (int(block) + 1) * self.n // self.workers
        d = np.zeros(max(b1 - b0, 1), np.int32)
        _check(lib().mg_synth_rank_block_degrees(self._h, int(block), _p(d)))
        return d[:b1 - b0]

    def finish(self, all_degrees: Optional[np.ndarray] = None) -> PreparedData:
        out = C.c_void_p()
        if all_degrees is not None:
            all_degrees = np.ascontiguousarray(all_degrees, np.int32)
            if all_degrees.shape != (self.n,):
                raise ValueError(f"synth_rank: need {self.n} degrees, got {all_degrees.shape}")
        _check(lib().mg_synth_rank_finish(self._h, _p(all_degrees) if all_degrees is not None else None,
                                          C.byref(out)))
        return PreparedData(out.value, self.workers)


def synth_prepare_rank(n, avg_degree, exponent, seed, feature_dim, classes, cfg: GcnConfig, workers: int,
                       rank: int, exchange=None) -> PreparedData:
    """Row block `rank` of prepare_data(synth_graph(n, avg_degree, exponent, seed, feature_dim, classes), cfg,
    workers) (inc/dataset.hpp:287-334, inc/driver.hpp:87-117), bit-identical, built from the generator's
    stream without the rest of the graph. exchange(local_degrees) -> all n degrees (e.g. an all-gather
    over the job's process group); None: this process derives every block's degrees itself."""
    h = SynthRank(n, avg_degree, exponent, seed, feature_dim, classes, cfg, workers, rank)
    degs = None if exchange is None else exchange(h.degrees())
    return h.finish(degs)


# ----------------------------------------------------------------------------- device group (gcn.hpp)


def set_tuning(key: str, value: int):
    _check(lib().mg_set_tuning(key.encode(), int(value)))


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().mg_nccl_unique_id(buf))
    return bytes(buf)


def device_count() -> int:
    return int(lib().mg_device_count())


class Group:
    """The GcnWorkers of this process (one per local rank), their streams and communicator."""

    def __init__(self, cfg: GcnConfig, prep: PreparedData, world: int, local_ranks=None, devices=None,
                 nccl_id: Optional[bytes] = None, transport: int = TRANSPORT_AUTO):
        self.cfg = cfg
        self.world = world
        local_ranks = list(range(world)) if local_ranks is None else list(local_ranks)
        if devices is None:
            nd = max(1, device_count())
            devices = [r % nd for r in local_ranks]
        self.local_ranks = local_ranks
        r = np.asarray(local_ranks, np.int32)
        d = np.asarray(devices, np.int32)
        idb = None if nccl_id is None else (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        out = C.c_void_p()
        self._prep = prep  # keep alive until the upload finished
        _check(lib().mg_group_create(C.byref(cfg._c()), prep._h, world, len(local_ranks), _p(r), _p(d), idb,
                                     transport, C.byref(out)))
        self._h = C.c_void_p(out.value)
        self.dims = list(cfg.layer_dims)

    def close(self):
        h = getattr(self, "_h", None)
        if h and h.value:
            lib().mg_group_destroy(h)
            self._h = C.c_void_p()

    def __del__(self, _fin=_finalizing):  # bound at definition: module globals may be gone at exit
        if not _fin():
            try:
                self.close()
            except Exception:  # interpreter teardown
                pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def abort(self):
        """DeviceGroup::abort (collectives.cpp:42-52): thread-safe; waits in progress and every later call on
        the group raise ShutdownError."""
        _check(lib().mg_group_abort(self._h))

    def init_params(self):
        _check(lib().mg_group_init_params(self._h))

    def train_step(self, t: int):
        loss, acc, wall = C.c_double(), C.c_double(), C.c_double()
        _check(lib().mg_group_train_step(self._h, int(t), C.byref(loss), C.byref(acc), C.byref(wall)))
        self.last_accuracy = acc.value
        self.last_wall_us = wall.value
        return loss.value

    def train_step_async(self, t: int):
        _check(lib().mg_group_train_step_async(self._h, int(t)))

    def sync(self):
        _check(lib().mg_group_sync(self._h))

    def last_stats(self):
        loss, acc = C.c_double(), C.c_double()
        _check(lib().mg_group_last_stats(self._h, C.byref(loss), C.byref(acc)))
        return loss.value, acc.value

    def compute_gradients(self):
        loss, acc = C.c_double(), C.c_double()
        _check(lib().mg_group_compute_gradients(self._h, C.byref(loss), C.byref(acc)))
        self.last_accuracy = acc.value
        return loss.value

    def loss_only(self):
        loss = C.c_double()
        _check(lib().mg_group_loss_only(self._h, C.byref(loss)))
        return loss.value

    def forward(self):
        _check(lib().mg_group_forward(self._h))

    def backward(self):
        """submit_backward + submit_finalize(false): backward from the gradient in the logits buffer."""
        _check(lib().mg_group_backward(self._h))

    def set_timeline(self, on: bool):
        """Start (clearing) / stop recording TimelineEvents from CUDA events (mg_group_set_timeline)."""
        _check(lib().mg_group_set_timeline(self._h, int(bool(on))))

    def timeline(self) -> list:
        """The recorded events (rowgcn::DeviceGroup::timeline)."""
        cnt = C.c_int64()
        _check(lib().mg_group_timeline(self._h, None, 0, C.byref(cnt)))
        buf = (mg_timeline_event * max(1, cnt.value))()
        _check(lib().mg_group_timeline(self._h, buf, cnt.value, C.byref(cnt)))
        return [_from_c_event(buf[i]) for i in range(cnt.value)]

    def bench_spmm(self, direction: int = 0) -> float:
        """One staged SpMM of the local X rows (mg_group_bench_spmm); returns its device time in us."""
        us = C.c_double()
        _check(lib().mg_group_bench_spmm(self._h, direction, C.byref(us)))
        return us.value

    def rows(self, rank: int):
        b, n = C.c_int64(), C.c_int64()
        _check(lib().mg_group_rows(self._h, rank, C.byref(b), C.byref(n)))
        return b.value, n.value

    def _shape(self, rank, which, layer):
        d = self.dims
        if which in (T_W, T_WGRAD, T_ADAM_M, T_ADAM_V):
            return (d[layer], d[layer + 1])
        if which in (T_BIAS, T_BIAS_GRAD):
            return (1, d[layer + 1])
        if which == T_WSTAGE:
            return (8 * d[layer], d[layer + 1])
        rows = self.rows(rank)[1]
        if which in (T_AHW, T_HW):
            return (rows, d[layer + 1])
        if which == T_X:
            return (rows, d[0])
        if which == T_ROWMAX:
            return (rows, 2)
        raise ValueError(f"tensor: unknown id {which}")

    def read(self, which: int, layer: int = 0, rank: Optional[int] = None) -> np.ndarray:
        rank = self.local_ranks[0] if rank is None else rank
        shape = self._shape(rank, which, layer)
        out = np.zeros(shape, np.float32)
        _check(lib().mg_group_read(self._h, rank, which, layer, _p(out), out.size))
        return out

    def write(self, which: int, layer: int, data, rank: int = -1):
        a = np.ascontiguousarray(data, np.float32)
        _check(lib().mg_group_write(self._h, rank, which, layer, _p(a), a.size))

    def params(self, rank: Optional[int] = None):
        return [self.read(T_W, l, rank) for l in range(len(self.dims) - 1)]

    def set_params(self, ws):
        for l, w in enumerate(ws):
            self.write(T_W, l, w)

    def w_grads(self, rank: Optional[int] = None):
        return [self.read(T_WGRAD, l, rank) for l in range(len(self.dims) - 1)]

    def w_hash(self, rank: Optional[int] = None) -> int:
        h = C.c_uint64()
        _check(lib().mg_group_w_hash(self._h, self.local_ranks[0] if rank is None else rank, C.byref(h)))
        return h.value

    def buffer_audit(self):
        lb, sa, by = C.c_int32(), C.c_int64(), C.c_int64()
        _check(lib().mg_group_buffer_audit(self._h, C.byref(lb), C.byref(sa), C.byref(by)))
        return lb.value, sa.value, by.value

    def kernels_last_step(self) -> int:
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        kk = C.c_int64()
        _check(lib().mg_group_last_profile(self._h, C.byref(a), C.byref(b), C.byref(c), C.byref(kk)))
        return kk.value

    def graph_steps(self):
        """(steps replayed from the captured CUDA graph, captures made) — see the "step_graph" tuning."""
        r, c = C.c_int64(), C.c_int64()
        _check(lib().mg_group_graph_steps(self._h, C.byref(r), C.byref(c)))
        return r.value, c.value

    def logits(self, rank: Optional[int] = None):
        return self.read(T_AHW, len(self.dims) - 2, rank)


# ----------------------------------------------------------------------------- driver (driver.hpp:119-251)


@dataclass
class TrainOptions:
    workers: int = 1
    collect_logits: bool = False
    on_epoch: Optional[Callable[[int, float, float, float], None]] = None
    devices: Optional[list] = None
    transport: int = TRANSPORT_AUTO


@dataclass
class TrainArtifacts:
    epoch_loss: list = field(default_factory=list)
    epoch_acc: list = field(default_factory=list)
    epoch_wall_us: list = field(default_factory=list)
    w_hashes: list = field(default_factory=list)  # [epoch][rank]
    final_w: list = field(default_factory=list)   # rank 0's replicas
    logits: Optional[np.ndarray] = None           # gathered post-training logits (permuted order)
    workers: int = 1
    timeline: list = field(default_factory=list)  # TimelineEvent per task, every epoch (CUDA events)

    def final_loss(self):
        return self.epoch_loss[-1] if self.epoch_loss else 0.0

    def final_acc(self):
        return self.epoch_acc[-1] if self.epoch_acc else 0.0


def train_run(ds: Dataset, cfg: GcnConfig, opts: TrainOptions = TrainOptions()) -> TrainArtifacts:
    """inc/driver.hpp:140-206: prepare_data, init_params, `epochs` train steps, artifacts."""
    cfg.validate()
    if cfg.layer_dims[0] != ds.d0:
        raise ConfigError(f"config: layer_dims[0]={cfg.layer_dims[0]} but dataset features have width {ds.d0}")
    prep = prepare_data(ds, cfg, opts.workers)
    art = TrainArtifacts(workers=opts.workers)
    with Group(cfg, prep, opts.workers, devices=opts.devices, transport=opts.transport) as g:
        g.init_params()
        g.set_timeline(True)
        for e in range(1, cfg.epochs + 1):
            loss = g.train_step(e)
            art.epoch_loss.append(loss)
            art.epoch_acc.append(g.last_accuracy)
            art.epoch_wall_us.append(g.last_wall_us)
            art.w_hashes.append([g.w_hash(r) for r in range(opts.workers)])
            if opts.on_epoch:
                opts.on_epoch(e, loss, g.last_accuracy, g.last_wall_us)
        art.timeline = g.timeline()
        g.set_timeline(False)
        if opts.collect_logits:
            g.loss_only()
            art.logits = np.concatenate([g.logits(r) for r in range(opts.workers)], axis=0)
        art.final_w = g.params(0)
    return art


@dataclass
class GradArtifacts:
    w_grad: list = field(default_factory=list)
    grad_hash_per_rank: list = field(default_factory=list)
    loss: float = 0.0


def grad_run(ds: Dataset, cfg: GcnConfig, workers: int, devices=None, transport=TRANSPORT_AUTO) -> GradArtifacts:
    """inc/driver.hpp:216-251: one forward/backward, W_G materialised, no update."""
    cfg.validate()
    prep = prepare_data(ds, cfg, workers)
    art = GradArtifacts()
    with Group(cfg, prep, workers, devices=devices, transport=transport) as g:
        g.init_params()
        art.loss = g.compute_gradients()
        for r in range(workers):
            art.grad_hash_per_rank.append(fnv1a(g.w_grads(r)))
        art.w_grad = g.w_grads(0)
    return art


def fnv1a(arrays, h: int = 0xcbf29ce484222325) -> int:
    """inc/gcn.hpp:87-94 over the raw bytes of each array in turn."""
    for a in arrays:
        b = np.frombuffer(np.ascontiguousarray(a).tobytes(), np.uint8)
        for byte in b:
            h ^= int(byte)
            h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


# ----------------------------------------------------------------------------- timeline (inc/timeline.hpp)


@dataclass
class TimelineEvent:
    """rowgcn::TimelineEvent (inc/collectives.hpp:24-34)."""
    worker: int = 0
    lane: int = 0
    stage: int = -1
    kind: str = ""
    op: str = ""
    t_start_us: float = 0.0
    t_end_us: float = 0.0
    task: int = 0
    deps: list = field(default_factory=list)


def _from_c_event(e) -> TimelineEvent:
    return TimelineEvent(e.worker, e.lane, e.stage, e.kind.decode(), e.op.decode(), e.t_start_us, e.t_end_us,
                         int(e.task), [int(e.deps[i]) for i in range(e.n_deps)])


def _to_c_events(events):
    arr = (mg_timeline_event * max(1, len(events)))()
    keep = []
    for i, e in enumerate(events):
        d = (C.c_uint64 * max(1, len(e.deps)))(*e.deps)
        keep.append(d)
        arr[i] = mg_timeline_event(e.worker, e.lane, e.stage, len(e.deps), e.kind.encode()[:15], e.op.encode()[:15],
                                   e.t_start_us, e.t_end_us, e.task, C.cast(d, C.POINTER(C.c_uint64)))
    return arr, keep


def timeline_to_json(events) -> list:
    """inc/timeline.hpp:15-28."""
    return [{"worker": e.worker, "lane": e.lane, "stage": e.stage, "kind": e.kind, "op": e.op,
             "t_start_us": e.t_start_us, "t_end_us": e.t_end_us, "task": e.task, "deps": list(e.deps)}
            for e in events]


def export_timeline(path, events):
    """inc/timeline.hpp:31-36 (native writer, mg_timeline_export)."""
    arr, _keep = _to_c_events(events)
    _check(lib().mg_timeline_export(_enc(path), arr, len(events)))


def parse_timeline(arr) -> list:
    """inc/timeline.hpp:38-55."""
    out = []
    for j in arr:
        out.append(TimelineEvent(int(j["worker"]), int(j["lane"]), int(j["stage"]), str(j["kind"]),
                                 str(j.get("op", "")), float(j["t_start_us"]), float(j["t_end_us"]),
                                 int(j.get("task", 0)), [int(d) for d in j.get("deps", [])]))
    return out


def load_timeline(path) -> list:
    """inc/timeline.hpp:57-63."""
    try:
        with open(path) as f:
            return parse_timeline(json.load(f))
    except OSError as ex:
        raise IoError(f"cannot open {path}") from ex


def audit_timeline(events):
    """inc/timeline.hpp:64-94 (native, mg_timeline_audit): raises ValueError on violation."""
    arr, _keep = _to_c_events(events)
    _check(lib().mg_timeline_audit(arr, len(events)))


def audit_staged_run(events, world: int, overlapped: bool):
    """inc/timeline.hpp:96-126 (native, mg_timeline_audit_staged) on one staged SpMM's events."""
    arr, _keep = _to_c_events(events)
    _check(lib().mg_timeline_audit_staged(arr, len(events), int(world), int(bool(overlapped))))


def timeline_span_us(events) -> float:
    """inc/timeline.hpp:128-137."""
    if not events:
        return 0.0
    return max(e.t_end_us for e in events) - min(e.t_start_us for e in events)


@dataclass
class BreakdownReport:
    """rowgcn::BreakdownReport (inc/breakdown.hpp:14-61)."""
    spmm_us: float = 0.0
    gemm_us: float = 0.0
    activation_us: float = 0.0
    loss_us: float = 0.0
    adam_us: float = 0.0
    comm_us: float = 0.0
    _KEYS = ("spmm", "gemm", "activation", "loss", "adam", "comm")

    def total_us(self) -> float:
        return self.spmm_us + self.gemm_us + self.activation_us + self.loss_us + self.adam_us + self.comm_us

    def frac(self, v: float) -> float:
        t = self.total_us()
        return v / t if t > 0 else 0.0

    def to_json(self) -> dict:
        vals = [getattr(self, k + "_us") for k in self._KEYS]
        return {"totals_us": dict(zip(self._KEYS, vals)), "fractions": {k: self.frac(v) for k, v in zip(self._KEYS, vals)}}

    def text_table(self) -> str:
        s = "kernel               time_us fraction\n"
        for k in self._KEYS:
            v = getattr(self, k + "_us")
            s += f"{k:<12} {v:14.1f} {self.frac(v):8.3f}\n"
        return s + f"{'total':<12} {self.total_us():14.1f} {self.frac(self.total_us()):8.3f}\n"


def runtime_breakdown(events) -> BreakdownReport:
    """inc/breakdown.hpp:63-82 (native, mg_timeline_breakdown)."""
    arr, _keep = _to_c_events(events)
    t = (C.c_double * 6)()
    _check(lib().mg_timeline_breakdown(arr, len(events), t))
    return BreakdownReport(*list(t))


def bench_spmm(ds: Dataset, workers: int = 1, permute: bool = True, overlap: bool = True, seed: int = 1,
               timeline_path: str = "", stage_csv: str = "", devices=None, transport=TRANSPORT_AUTO,
               spmm_mode: int = SPMM_FAST) -> dict:
    """`bench-spmm` (proj/tools/main.cpp:120-178): one staged SpMM of the dataset's features (width = d0)
    over the forward tiles on `workers` GPUs; audits the staged-run rules, optionally exports the timeline
    and the per-stage CSV (stage, worker, comm_us, comp_us); returns the summary (plus the output rows)."""
    width = ds.d0
    cfg = GcnConfig([width, width], epochs=1, seed=seed, permute=permute, overlap=overlap and workers > 1,
                    spmm_mode=spmm_mode)
    prep = prepare_data(ds, cfg, workers)
    with Group(cfg, prep, workers, devices=devices, transport=transport) as g:
        g.set_timeline(True)
        device_us = g.bench_spmm(0)
        events = g.timeline()
        g.set_timeline(False)
        out = np.concatenate([g.read(T_HW, 0, r) for r in range(workers)], axis=0)
    audit_staged_run(events, workers, cfg.overlap)
    if timeline_path:
        export_timeline(timeline_path, events)
    if stage_csv:
        with open(stage_csv, "w") as f:
            f.write("stage,worker,comm_us,comp_us\n")
            for stage in range(workers):
                for w in range(workers):
                    comm = sum(e.t_end_us - e.t_start_us for e in events
                               if e.worker == w and e.stage == stage and e.kind == "broadcast")
                    comp = sum(e.t_end_us - e.t_start_us for e in events
                               if e.worker == w and e.stage == stage and e.kind == "spmm")
                    f.write(f"{stage},{w},{comm:g},{comp:g}\n")
    nnz = sum(int(prep.tile(0, i, j)[0][-1]) for i in range(workers) for j in range(workers))
    # DeviceGroup::total_bytes_sent (collectives.hpp:127): each root counts its stage message once
    bytes_bc = sum((prep.bounds[j + 1] - prep.bounds[j]) * width * 4 for j in range(workers)) if workers > 1 else 0
    return {"n": ds.n(), "nnz": nnz, "width": width, "workers": workers, "overlap": cfg.overlap, "permute": permute,
            "wall_us": timeline_span_us(events), "device_us": device_us, "bytes_broadcast": int(bytes_bc),
            "out": out, "events": events}


# ----------------------------------------------------------------------------- kernel-level entry points


def dev_spmm(rows, row_ptr_ptr, edges_ptr, h_ptr, out_ptr, w, ld, accumulate=False, relu=False, mode=SPMM_EXACT,
             stream=0):
    """rowgcn::spmm on device pointers (see include/mggcn.h mg_dev_spmm)."""
    _check(lib().mg_dev_spmm(rows, C.c_void_p(row_ptr_ptr), C.c_void_p(edges_ptr), C.c_void_p(h_ptr),
                             C.c_void_p(out_ptr), w, ld, int(accumulate), int(relu), mode, C.c_void_p(stream)))


def dev_gemm(ta, tb, M, N, K, a_ptr, lda, b_ptr, ldb, c_ptr, ldc, epilogue=0, mode=GEMM_EXACT, stream=0):
    _check(lib().mg_dev_gemm(int(ta), int(tb), M, N, K, C.c_void_p(a_ptr), lda, C.c_void_p(b_ptr), ldb,
                             C.c_void_p(c_ptr), ldc, epilogue, mode, C.c_void_p(stream)))


def dev_softmax_xent(logits_ptr, rows, classes, ld, labels_ptr, mask_ptr, denom, stream=0):
    """rowgcn::softmax_xent_sum on device rows, gradient in place; returns (loss_sum, correct)."""
    st = (C.c_double * 2)()
    _check(lib().mg_dev_softmax_xent(C.c_void_p(logits_ptr), rows, classes, ld, C.c_void_p(labels_ptr),
                                     C.c_void_p(mask_ptr), denom, st, C.c_void_p(stream)))
    return st[0], st[1]


def dev_adam(w_ptr, grad_ptr, m_ptr, v_ptr, size, t, lr=0.01, beta1=0.9, beta2=0.999, epsilon=1e-8, stream=0):
    """rowgcn::adam_step on one device parameter array (grad zeroed)."""
    _check(lib().mg_dev_adam(C.c_void_p(w_ptr), C.c_void_p(grad_ptr), C.c_void_p(m_ptr), C.c_void_p(v_ptr), size,
                             lr, beta1, beta2, epsilon, t, C.c_void_p(stream)))
