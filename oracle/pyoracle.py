"""TEST INFRASTRUCTURE ONLY — numpy/ctypes front end to the two CPU oracles.

* ``Ref``  — the UNMODIFIED reference (rowgcn headers) compiled by ``oracle/build_ref.sh`` into
  ``oracle/_ref/librowgcn_ref.so`` (kind "reference").
* ``Port`` — the plain-C restatement ``oracle/oracle.c`` built by ``oracle/build_oracle.sh`` into
  ``oracle/_build/liboracle_{f32,f64}.so`` (kind "port").

Only ``tests/``, ``bench.py``'s cpu_baseline / reference arm and ``__graft_entry__.smoke()`` import this
module; the product (``paper_2110_08688_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "librowgcn_ref.so")
PORT_LIBS = {np.float32: os.path.join(HERE, "_build", "liboracle_f32.so"),
             np.float64: os.path.join(HERE, "_build", "liboracle_f64.so")}

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class Dataset:
    """Mirror of rowgcn::Dataset (inc/dataset.hpp:19-56) as numpy arrays (CSR int64)."""
    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    features: np.ndarray
    labels: np.ndarray
    train_mask: np.ndarray | None = None

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def d0(self) -> int:
        return int(self.features.shape[1])

    def astype(self, dtype):
        return Dataset(self.n, self.row_ptr, self.col_idx, self.values.astype(dtype),
                       self.features.astype(dtype), self.labels, self.train_mask)


@dataclass
class Prepared:
    """Mirror of rowgcn::PreparedData (inc/driver.hpp:75-85); tiles[dir][i][j] = (row_ptr, col_idx, values),
    dir 0 = forward tiles of A_hat^T, dir 1 = backward tiles of A_hat."""
    bounds: np.ndarray
    mask_count: int
    features: np.ndarray
    labels: np.ndarray
    mask: np.ndarray
    perm_forward: np.ndarray
    tiles: list = field(default_factory=list)


class _RefCfg(C.Structure):
    _fields_ = [("dims", C.c_void_p), ("n_dims", C.c_int32), ("lr", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("epsilon", C.c_double), ("epochs", C.c_int32), ("seed", C.c_uint64),
                ("permute", C.c_uint8), ("overlap", C.c_uint8), ("skip_first_backward_spmm", C.c_uint8),
                ("order_swap", C.c_uint8)]


def make_cfg(dims, epochs=1, seed=1, lr=0.01, beta1=0.9, beta2=0.999, epsilon=1e-8, permute=False,
             overlap=False, skip_first_backward_spmm=False, order_swap=False):
    d = np.ascontiguousarray(np.asarray(dims, dtype=np.int64))
    c = _RefCfg(d.ctypes.data_as(C.c_void_p), len(d), lr, beta1, beta2, epsilon, epochs, seed,
                int(permute), int(overlap), int(skip_first_backward_spmm), int(order_swap))
    c._keep = d  # keep dims alive
    return c


def _suffix(dtype):
    return "f32" if np.dtype(dtype) == np.float32 else "f64"


class OracleError(RuntimeError):
    pass


class Ref:
    """The compiled reference (kind "reference")."""

    def __init__(self, path: str = REF_LIB):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run oracle/build_ref.sh (needs /root/reference)")
        self.lib = C.CDLL(path)
        self.lib.ref_last_error.restype = C.c_char_p
        for s in ("f32", "f64"):
            getattr(self.lib, f"ref_ds_synth_{s}").restype = C.c_void_p
            getattr(self.lib, f"ref_ds_from_arrays_{s}").restype = C.c_void_p
        self.lib.ref_prepare_f32.restype = C.c_void_p
        self.lib.ref_fnv1a.restype = C.c_uint64
        self.lib.ref_fnv1a.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]

    def _check(self, rc):
        if rc != 0:
            e = OracleError(f"reference error {rc}: {self.lib.ref_last_error().decode()}")
            e.code = rc  # 1 ShapeError, 2 ValueError, ..., 5 ParseError, 7 IoError (ref_shim.cpp guarded)
            e.message = self.lib.ref_last_error().decode()
            raise e

    # ------------------------------------------------------------ on-disk formats (dataset.hpp:84-280)
    def _partial_graph(self, h):
        try:
            nn, nnz, d0 = C.c_int64(), C.c_int64(), C.c_int64()
            self.lib.ref_ds_info_f32(C.c_void_p(h), C.byref(nn), C.byref(nnz), C.byref(d0))
            rp = np.zeros(nn.value + 1, np.int64)
            ci = np.empty(nnz.value, np.int64)
            v = np.empty(nnz.value, np.float32)
            if nn.value or nnz.value:
                self.lib.ref_ds_export_f32(C.c_void_p(h), _ptr(rp), _ptr(ci), _ptr(v), None, None)
            return rp, ci, v
        finally:
            self.lib.ref_ds_free_f32(C.c_void_p(h))

    def load_graph(self, path, fmt=0):
        """load_graph / load_matrix_market (fmt 1) / load_edge_list (fmt 2) -> (row_ptr, col_idx, values)."""
        h = C.c_void_p()
        self._check(self.lib.ref_load_graph_f32(str(path).encode(), C.c_int32(fmt), C.byref(h)))
        return self._partial_graph(h.value)

    def _partial_features(self, h):
        try:
            r, c = C.c_int64(), C.c_int64()
            self.lib.ref_ds_feat_shape_f32(C.c_void_p(h), C.byref(r), C.byref(c))
            x = np.zeros((r.value, c.value), np.float32)
            if x.size:
                self.lib.ref_ds_export_f32(C.c_void_p(h), None, None, None, _ptr(x), None)
            return x
        finally:
            self.lib.ref_ds_free_f32(C.c_void_p(h))

    def load_features(self, path):
        h = C.c_void_p()
        self._check(self.lib.ref_load_features_f32(str(path).encode(), C.byref(h)))
        return self._partial_features(h.value)

    def read_dense(self, path):
        h = C.c_void_p()
        self._check(self.lib.ref_read_dense_f32(str(path).encode(), C.byref(h)))
        return self._partial_features(h.value)

    def write_dense(self, path, m):
        a = np.ascontiguousarray(m, np.float32)
        self._check(self.lib.ref_write_dense_f32(str(path).encode(), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]),
                                                 _ptr(a)))

    def load_labels(self, path):
        cnt = C.c_int64()
        self._check(self.lib.ref_load_labels(str(path).encode(), None, C.c_int64(0), C.byref(cnt)))
        out = np.zeros(cnt.value, np.int32)
        self._check(self.lib.ref_load_labels(str(path).encode(), _ptr(out), C.c_int64(cnt.value), C.byref(cnt)))
        return out

    def load_masks(self, path, n):
        arrs = [np.zeros(n, np.uint8) for _ in range(3)]
        pr = C.c_int32()
        self._check(self.lib.ref_load_masks(str(path).encode(), C.c_int64(n), *[_ptr(a) for a in arrs], C.byref(pr)))
        return tuple(a if pr.value & (1 << i) else np.zeros(0, np.uint8) for i, a in enumerate(arrs))

    def timeline_check(self, path, world=0, overlapped=False):
        """The reference's load_timeline + audit_timeline (+ audit_staged_run when world > 0) on a JSON
        file; returns (event count, runtime_breakdown totals dict). Raises OracleError on violation."""
        t = np.zeros(6, np.float64)
        cnt = C.c_int64()
        self._check(self.lib.ref_timeline_check(str(path).encode(), C.c_int32(world), C.c_int32(int(overlapped)),
                                                _ptr(t), C.byref(cnt)))
        return cnt.value, dict(zip(("spmm", "gemm", "activation", "loss", "adam", "comm"), t.tolist()))

    def train_timeline(self, ds: Dataset, cfg, workers: int, path):
        """Exports the reference trainer's own timeline (train_run<float>) to path."""
        h = self._ds_handle(ds, np.float32)
        try:
            self._check(self.lib.ref_train_timeline_f32(C.c_void_p(h), C.byref(cfg), C.c_int32(workers),
                                                        str(path).encode()))
        finally:
            self._ds_free(h, np.float32)

    def load_dataset(self, g, f, l, m=""):
        """load_dataset<float> -> (Dataset, (train, val, test))."""
        h = C.c_void_p()
        self._check(self.lib.ref_load_dataset_f32(str(g).encode(), str(f).encode(), str(l).encode(),
                                                  str(m).encode() if m else None, C.byref(h)))
        try:
            nn, nnz, d0 = C.c_int64(), C.c_int64(), C.c_int64()
            self.lib.ref_ds_info_f32(h, C.byref(nn), C.byref(nnz), C.byref(d0))
            rp = np.empty(nn.value + 1, np.int64)
            ci = np.empty(nnz.value, np.int64)
            v = np.empty(nnz.value, np.float32)
            x = np.empty((nn.value, d0.value), np.float32)
            lab = np.empty(nn.value, np.int32)
            self.lib.ref_ds_export_f32(h, _ptr(rp), _ptr(ci), _ptr(v), _ptr(x), _ptr(lab))
            arrs = [np.zeros(nn.value, np.uint8) for _ in range(3)]
            pr = C.c_int32()
            self.lib.ref_ds_masks_f32(h, *[_ptr(a) for a in arrs], C.byref(pr))
            masks = tuple(a if pr.value & (1 << i) else np.zeros(0, np.uint8) for i, a in enumerate(arrs))
        finally:
            self.lib.ref_ds_free_f32(h)
        return Dataset(nn.value, rp, ci, v, x, lab), masks

    def set_spmm_threads(self, t: int):
        self.lib.ref_set_spmm_threads(C.c_int(t))

    # ------------------------------------------------------------ datasets
    def _ds_handle(self, ds: Dataset, dtype):
        s = _suffix(dtype)
        vals = np.ascontiguousarray(ds.values, dtype=dtype)
        feats = np.ascontiguousarray(ds.features, dtype=dtype)
        h = getattr(self.lib, f"ref_ds_from_arrays_{s}")(
            C.c_int64(ds.n), _ptr(np.ascontiguousarray(ds.row_ptr, np.int64)),
            _ptr(np.ascontiguousarray(ds.col_idx, np.int64)), _ptr(vals), C.c_int64(ds.d0), _ptr(feats),
            _ptr(np.ascontiguousarray(ds.labels, np.int32)),
            _ptr(None if ds.train_mask is None else np.ascontiguousarray(ds.train_mask, np.uint8)))
        if not h:
            self._check(99)
        return h

    def _ds_free(self, h, dtype):
        getattr(self.lib, f"ref_ds_free_{_suffix(dtype)}")(C.c_void_p(h))

    def synth(self, n, avg_degree, exponent, seed, feature_dim=16, classes=4, dtype=np.float32) -> Dataset:
        s = _suffix(dtype)
        h = getattr(self.lib, f"ref_ds_synth_{s}")(C.c_int64(n), C.c_double(avg_degree), C.c_double(exponent),
                                                  C.c_uint64(seed), C.c_int64(feature_dim), C.c_int32(classes))
        if not h:
            self._check(2)
        try:
            nn, nnz, d0 = C.c_int64(), C.c_int64(), C.c_int64()
            getattr(self.lib, f"ref_ds_info_{s}")(C.c_void_p(h), C.byref(nn), C.byref(nnz), C.byref(d0))
            rp = np.empty(nn.value + 1, np.int64)
            ci = np.empty(nnz.value, np.int64)
            v = np.empty(nnz.value, dtype)
            x = np.empty((nn.value, d0.value), dtype)
            lab = np.empty(nn.value, np.int32)
            getattr(self.lib, f"ref_ds_export_{s}")(C.c_void_p(h), _ptr(rp), _ptr(ci), _ptr(v), _ptr(x), _ptr(lab))
        finally:
            self._ds_free(h, dtype)
        return Dataset(nn.value, rp, ci, v, x, lab)

    # ------------------------------------------------------------ partitioner
    def random_permutation(self, n, seed):
        f = np.empty(n, np.int64)
        inv = np.empty(n, np.int64)
        self._check(self.lib.ref_random_permutation(C.c_int64(n), C.c_uint64(seed), _ptr(f), _ptr(inv)))
        return f, inv

    def uniform_partition(self, n, parts):
        b = np.empty(parts + 1, np.int64)
        self._check(self.lib.ref_uniform_partition(C.c_int64(n), C.c_int32(parts), _ptr(b)))
        return b

    def prepare(self, ds: Dataset, cfg, workers: int) -> Prepared:
        h = self._ds_handle(ds, np.float32)
        try:
            p = self.lib.ref_prepare_f32(C.c_void_p(h), C.byref(cfg), C.c_int32(workers))
            if not p:
                self._check(99)
        finally:
            self._ds_free(h, np.float32)
        try:
            mc = C.c_int64()
            b = np.empty(workers + 1, np.int64)
            self.lib.ref_prep_info_f32(C.c_void_p(p), C.byref(mc), _ptr(b))
            x = np.empty((ds.n, ds.d0), np.float32)
            lab = np.empty(ds.n, np.int32)
            m = np.empty(ds.n, np.uint8)
            pf = np.empty(ds.n, np.int64)
            self.lib.ref_prep_rows_export_f32(C.c_void_p(p), _ptr(x), _ptr(lab), _ptr(m), _ptr(pf))
            tiles = []
            for d in (0, 1):
                grid = []
                for i in range(workers):
                    row = []
                    for j in range(workers):
                        r, c_, z = C.c_int64(), C.c_int64(), C.c_int64()
                        self.lib.ref_prep_tile_info_f32(C.c_void_p(p), d, i, j, C.byref(r), C.byref(c_), C.byref(z))
                        rp = np.empty(r.value + 1, np.int64)
                        ci = np.empty(z.value, np.int64)
                        v = np.empty(z.value, np.float32)
                        self.lib.ref_prep_tile_export_f32(C.c_void_p(p), d, i, j, _ptr(rp), _ptr(ci), _ptr(v))
                        row.append((rp, ci, v))
                    grid.append(row)
                tiles.append(grid)
        finally:
            self.lib.ref_prep_free_f32(C.c_void_p(p))
        return Prepared(b, mc.value, x, lab, m, pf, tiles)

    # ------------------------------------------------------------ kernels
    def spmm(self, rows, cols, rp, ci, v, h, accumulate=False, out=None):
        dtype = h.dtype
        w = h.shape[1]
        out = np.zeros((rows, w), dtype) if out is None else np.ascontiguousarray(out, dtype).copy()
        self._check(getattr(self.lib, f"ref_spmm_{_suffix(dtype)}")(
            C.c_int64(rows), C.c_int64(cols), _ptr(np.ascontiguousarray(rp, np.int64)),
            _ptr(np.ascontiguousarray(ci, np.int64)), _ptr(np.ascontiguousarray(v, dtype)),
            _ptr(np.ascontiguousarray(h)), C.c_int64(w), C.c_int32(int(accumulate)), _ptr(out)))
        return out

    def gemm(self, a, b, ta=False, tb=False, accumulate=False, out=None):
        dtype = a.dtype
        m = a.shape[1] if ta else a.shape[0]
        n = b.shape[0] if tb else b.shape[1]
        out = np.zeros((m, n), dtype) if out is None else np.ascontiguousarray(out, dtype).copy()
        self._check(getattr(self.lib, f"ref_gemm_{_suffix(dtype)}")(
            _ptr(np.ascontiguousarray(a)), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]),
            _ptr(np.ascontiguousarray(b)), C.c_int64(b.shape[0]), C.c_int64(b.shape[1]), C.c_int32(int(ta)),
            C.c_int32(int(tb)), C.c_int32(int(accumulate)), _ptr(out), C.c_int64(m), C.c_int64(n)))
        return out

    def softmax_xent_sum(self, logits, labels, mask, denom):
        dtype = logits.dtype
        grad = np.empty_like(logits)
        ls = C.c_double()
        self._check(getattr(self.lib, f"ref_softmax_xent_sum_{_suffix(dtype)}")(
            _ptr(np.ascontiguousarray(logits)), C.c_int64(logits.shape[0]), C.c_int64(logits.shape[1]),
            _ptr(np.ascontiguousarray(labels, np.int32)), _ptr(np.ascontiguousarray(mask, np.uint8)), _ptr(grad),
            C.c_int64(denom), C.byref(ls)))
        return ls.value, grad

    def adam(self, w, g, m, v, t, lr=0.01, b1=0.9, b2=0.999, eps=1e-8):
        arrs = [np.ascontiguousarray(x).copy() for x in (w, g, m, v)]
        self._check(getattr(self.lib, f"ref_adam_{_suffix(w.dtype)}")(
            *[_ptr(x) for x in arrs], C.c_int64(w.size), C.c_int32(t), C.c_double(lr), C.c_double(b1),
            C.c_double(b2), C.c_double(eps)))
        return arrs

    # ------------------------------------------------------------ model
    def train_run(self, ds: Dataset, cfg, workers: int, dtype=np.float32, collect_logits=False):
        s = _suffix(dtype)
        E = cfg.epochs
        dims = list(cfg._keep)
        loss = np.zeros(E)
        acc = np.zeros(E)
        wall = np.zeros(E)
        hashes = np.zeros(E * workers, np.uint64)
        wsz = sum(dims[i] * dims[i + 1] for i in range(len(dims) - 1))
        fw = np.zeros(wsz, dtype)
        logits = np.zeros((ds.n, dims[-1]), dtype) if collect_logits else None
        h = self._ds_handle(ds, dtype)
        try:
            self._check(getattr(self.lib, f"ref_train_run_{s}")(
                C.c_void_p(h), C.byref(cfg), C.c_int32(workers), _ptr(loss), _ptr(acc), _ptr(wall), _ptr(hashes),
                _ptr(fw), _ptr(logits)))
        finally:
            self._ds_free(h, dtype)
        return dict(loss=loss, acc=acc, wall_us=wall, w_hashes=hashes.reshape(E, workers),
                    final_w=split_w(fw, dims), logits=logits)

    def grad_run(self, ds: Dataset, cfg, workers: int, dtype=np.float32):
        s = _suffix(dtype)
        dims = list(cfg._keep)
        wsz = sum(dims[i] * dims[i + 1] for i in range(len(dims) - 1))
        g = np.zeros(wsz, dtype)
        hashes = np.zeros(workers, np.uint64)
        loss = C.c_double()
        h = self._ds_handle(ds, dtype)
        try:
            self._check(getattr(self.lib, f"ref_grad_run_{s}")(C.c_void_p(h), C.byref(cfg), C.c_int32(workers),
                                                                C.byref(loss), _ptr(g), _ptr(hashes)))
        finally:
            self._ds_free(h, dtype)
        return dict(loss=loss.value, w_grad=split_w(g, dims), hashes=hashes)

    def step_dump(self, ds: Dataset, cfg, workers: int, dtype=np.float32, w_init=None):
        """Teacher-forced train_step(1) with captured tensors (global permuted rows)."""
        s = _suffix(dtype)
        dims = list(cfg._keep)
        n = ds.n
        L = len(dims) - 1
        act = sum(n * d for d in dims[1:])
        wsz = sum(dims[i] * dims[i + 1] for i in range(L))
        ahw_fwd = np.zeros(act, dtype)
        lg = np.zeros((n, dims[-1]), dtype)
        ahw_bwd = np.zeros(act, dtype)
        hw_last = np.zeros((n, dims[1]), dtype)
        wg = np.zeros(wsz, dtype)
        wa = np.zeros(wsz, dtype)
        loss = C.c_double()
        wi = None if w_init is None else np.ascontiguousarray(np.concatenate([np.ravel(x) for x in w_init]), dtype)
        h = self._ds_handle(ds, dtype)
        try:
            self._check(getattr(self.lib, f"ref_step_dump_{s}")(
                C.c_void_p(h), C.byref(cfg), C.c_int32(workers), _ptr(wi), _ptr(ahw_fwd), _ptr(lg), _ptr(ahw_bwd),
                _ptr(hw_last), _ptr(wg), _ptr(wa), C.byref(loss)))
        finally:
            self._ds_free(h, dtype)
        return dict(loss=loss.value, ahw_fwd=split_act(ahw_fwd, n, dims), loss_grad=lg,
                    ahw_bwd=split_act(ahw_bwd, n, dims), hw_last=hw_last, w_grad=split_w(wg, dims),
                    w_after=split_w(wa, dims))

    def fnv1a(self, arrays) -> int:
        h = 0xcbf29ce484222325
        for a in arrays:
            a = np.ascontiguousarray(a)
            h = self.lib.ref_fnv1a(a.ctypes.data_as(C.c_void_p), C.c_uint64(a.nbytes), C.c_uint64(h))
        return h


def fnv1a(arrays) -> int:
    """FNV-1a 64 over the raw bytes of each array in turn (inc/gcn.hpp:87-94, w_hash :221-226)."""
    h = 0xcbf29ce484222325
    for a in arrays:
        for byte in np.ascontiguousarray(a).view(np.uint8).tobytes():
            h ^= byte
            h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def split_w(flat, dims):
    out, off = [], 0
    for i in range(len(dims) - 1):
        sz = dims[i] * dims[i + 1]
        out.append(flat[off:off + sz].reshape(dims[i], dims[i + 1]))
        off += sz
    return out


def split_act(flat, n, dims):
    out, off = [], 0
    for d in dims[1:]:
        out.append(flat[off:off + n * d].reshape(n, d))
        off += n * d
    return out


class Port:
    """The plain-C restatement (kind "port")."""

    def __init__(self, dtype=np.float32):
        self.dtype = np.dtype(dtype).type
        path = PORT_LIBS[self.dtype]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run oracle/build_oracle.sh")
        self.lib = C.CDLL(path)
        self.s = _suffix(dtype)
        for name in ("or_synth_graph", "or_ds_from_arrays", "or_prepare", "or_model_create"):
            getattr(self.lib, f"{name}_{self.s}").restype = C.c_void_p

    def f(self, name):
        return getattr(self.lib, f"{name}_{self.s}")

    def rng_first(self, seed, count):
        out = np.empty(count, np.uint64)
        self.f("or_rng_first")(C.c_uint64(seed), C.c_int32(count), _ptr(out))
        return out

    def random_permutation(self, n, seed):
        f = np.empty(n, np.int64)
        inv = np.empty(n, np.int64)
        self.f("or_random_permutation")(C.c_int64(n), C.c_uint64(seed), _ptr(f), _ptr(inv))
        return f, inv

    def uniform_partition(self, n, parts):
        b = np.empty(parts + 1, np.int64)
        self.f("or_uniform_partition")(C.c_int64(n), C.c_int32(parts), _ptr(b))
        return b

    def _export_ds(self, h) -> Dataset:
        nn, nnz, d0 = C.c_int64(), C.c_int64(), C.c_int64()
        self.f("or_ds_info")(C.c_void_p(h), C.byref(nn), C.byref(nnz), C.byref(d0))
        rp = np.empty(nn.value + 1, np.int64)
        ci = np.empty(nnz.value, np.int64)
        v = np.empty(nnz.value, self.dtype)
        x = np.empty((nn.value, d0.value), self.dtype)
        lab = np.empty(nn.value, np.int32)
        self.f("or_ds_export")(C.c_void_p(h), _ptr(rp), _ptr(ci), _ptr(v), _ptr(x), _ptr(lab))
        return Dataset(nn.value, rp, ci, v, x, lab)

    def synth(self, n, avg_degree, exponent, seed, feature_dim=16, classes=4) -> Dataset:
        h = self.f("or_synth_graph")(C.c_int64(n), C.c_double(avg_degree), C.c_double(exponent), C.c_uint64(seed),
                                     C.c_int64(feature_dim), C.c_int32(classes))
        if not h:
            raise OracleError("synth_graph: invalid arguments")
        try:
            return self._export_ds(h)
        finally:
            self.f("or_ds_free")(C.c_void_p(h))

    def _ds_handle(self, ds: Dataset):
        return self.f("or_ds_from_arrays")(
            C.c_int64(ds.n), _ptr(np.ascontiguousarray(ds.row_ptr, np.int64)),
            _ptr(np.ascontiguousarray(ds.col_idx, np.int64)), _ptr(np.ascontiguousarray(ds.values, self.dtype)),
            C.c_int64(ds.d0), _ptr(np.ascontiguousarray(ds.features, self.dtype)),
            _ptr(np.ascontiguousarray(ds.labels, np.int32)))

    def prepare_handle(self, ds: Dataset, permute: bool, seed: int, workers: int):
        h = self._ds_handle(ds)
        try:
            mask = None if ds.train_mask is None else np.ascontiguousarray(ds.train_mask, np.uint8)
            return self.f("or_prepare")(C.c_void_p(h), _ptr(mask), C.c_int32(int(permute)), C.c_uint64(seed),
                                        C.c_int32(workers))
        finally:
            self.f("or_ds_free")(C.c_void_p(h))

    def prepare(self, ds: Dataset, permute: bool, seed: int, workers: int) -> Prepared:
        p = self.prepare_handle(ds, permute, seed, workers)
        try:
            mc = C.c_int64()
            b = np.empty(workers + 1, np.int64)
            self.f("or_prep_info")(C.c_void_p(p), C.byref(mc), _ptr(b))
            x = np.empty((ds.n, ds.d0), self.dtype)
            lab = np.empty(ds.n, np.int32)
            m = np.empty(ds.n, np.uint8)
            pf = np.empty(ds.n, np.int64)
            self.f("or_prep_rows_export")(C.c_void_p(p), _ptr(x), _ptr(lab), _ptr(m), _ptr(pf))
            tiles = []
            for d in (0, 1):
                grid = []
                for i in range(workers):
                    row = []
                    for j in range(workers):
                        r, c_, z = C.c_int64(), C.c_int64(), C.c_int64()
                        self.f("or_prep_tile_info")(C.c_void_p(p), d, i, j, C.byref(r), C.byref(c_), C.byref(z))
                        rp = np.empty(r.value + 1, np.int64)
                        ci = np.empty(z.value, np.int64)
                        v = np.empty(z.value, self.dtype)
                        self.f("or_prep_tile_export")(C.c_void_p(p), d, i, j, _ptr(rp), _ptr(ci), _ptr(v))
                        row.append((rp, ci, v))
                    grid.append(row)
                tiles.append(grid)
            return Prepared(b, mc.value, x, lab, m, pf, tiles)
        finally:
            self.f("or_prep_free")(C.c_void_p(p))

    def spmm(self, rows, cols, rp, ci, v, h, accumulate=False, out=None):
        w = h.shape[1]
        out = np.zeros((rows, w), self.dtype) if out is None else np.ascontiguousarray(out, self.dtype).copy()
        self.f("or_spmm")(C.c_int64(rows), C.c_int64(cols), _ptr(np.ascontiguousarray(rp, np.int64)),
                          _ptr(np.ascontiguousarray(ci, np.int64)), _ptr(np.ascontiguousarray(v, self.dtype)),
                          _ptr(np.ascontiguousarray(h, self.dtype)), C.c_int64(w), C.c_int32(int(accumulate)),
                          _ptr(out))
        return out

    def gemm(self, a, b, ta=False, tb=False, accumulate=False, out=None):
        m = a.shape[1] if ta else a.shape[0]
        n = b.shape[0] if tb else b.shape[1]
        out = np.zeros((m, n), self.dtype) if out is None else np.ascontiguousarray(out, self.dtype).copy()
        self.f("or_gemm")(_ptr(np.ascontiguousarray(a, self.dtype)), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]),
                          _ptr(np.ascontiguousarray(b, self.dtype)), C.c_int64(b.shape[0]), C.c_int64(b.shape[1]),
                          C.c_int32(int(ta)), C.c_int32(int(tb)), C.c_int32(int(accumulate)), _ptr(out))
        return out

    def softmax_xent_sum(self, logits, labels, mask, denom):
        grad = np.empty_like(np.ascontiguousarray(logits, self.dtype))
        ls = C.c_double()
        rc = self.f("or_softmax_xent_sum")(_ptr(np.ascontiguousarray(logits, self.dtype)), C.c_int64(logits.shape[0]),
                                           C.c_int64(logits.shape[1]), _ptr(np.ascontiguousarray(labels, np.int32)),
                                           _ptr(np.ascontiguousarray(mask, np.uint8)), _ptr(grad), C.c_int64(denom),
                                           C.byref(ls))
        if rc:
            raise OracleError("softmax_xent: ValueError")
        return ls.value, grad

    def adam(self, w, g, m, v, t, lr=0.01, b1=0.9, b2=0.999, eps=1e-8):
        arrs = [np.ascontiguousarray(x, self.dtype).copy() for x in (w, g, m, v)]
        rc = self.f("or_adam")(*[_ptr(x) for x in arrs], C.c_int64(w.size), C.c_int32(t), C.c_double(lr),
                               C.c_double(b1), C.c_double(b2), C.c_double(eps))
        if rc:
            raise OracleError("adam_step: ValueError")
        return arrs

    def model(self, ds: Dataset, dims, workers=1, seed=1, permute=False, lr=0.01, beta1=0.9, beta2=0.999,
              epsilon=1e-8, skip_first_backward_spmm=False, order_swap=False):
        return PortModel(self, ds, dims, workers, seed, permute, lr, beta1, beta2, epsilon,
                         skip_first_backward_spmm, order_swap)


class PortModel:
    """Restated GcnWorker group (inc/gcn.hpp) over a prepared dataset."""

    def __init__(self, port: Port, ds, dims, workers, seed, permute, lr, b1, b2, eps, skip, swap):
        self.port = port
        self.dims = [int(d) for d in dims]
        self.n = ds.n
        self.prep = port.prepare_handle(ds, permute, seed, workers)
        d = np.ascontiguousarray(np.asarray(self.dims, np.int64))
        self.h = port.f("or_model_create")(C.c_void_p(self.prep), _ptr(d), C.c_int32(len(d)), C.c_double(lr),
                                           C.c_double(b1), C.c_double(b2), C.c_double(eps), C.c_uint64(seed),
                                           C.c_int32(int(skip)), C.c_int32(int(swap)))

    def __del__(self):
        try:
            self.port.f("or_model_free")(C.c_void_p(self.h))
            self.port.f("or_prep_free")(C.c_void_p(self.prep))
        except Exception:
            pass

    def get_w(self):
        flat = np.empty(sum(self.dims[i] * self.dims[i + 1] for i in range(len(self.dims) - 1)), self.port.dtype)
        self.port.f("or_model_get_w")(C.c_void_p(self.h), _ptr(flat))
        return split_w(flat, self.dims)

    def set_w(self, ws):
        flat = np.ascontiguousarray(np.concatenate([np.ravel(w) for w in ws]), self.port.dtype)
        self.port.f("or_model_set_w")(C.c_void_p(self.h), _ptr(flat))

    def step(self, t=1, mode=0, dumps=False):
        n, dims = self.n, self.dims
        act = sum(n * d for d in dims[1:])
        wsz = sum(dims[i] * dims[i + 1] for i in range(len(dims) - 1))
        dt = self.port.dtype
        af = np.zeros(act, dt) if dumps else None
        lg = np.zeros((n, dims[-1]), dt) if dumps else None
        ab = np.zeros(act, dt) if dumps else None
        wg = np.zeros(wsz, dt) if dumps else None
        loss, acc = C.c_double(), C.c_double()
        rc = self.port.f("or_model_step")(C.c_void_p(self.h), C.c_int32(t), C.c_int32(mode), C.byref(loss),
                                          C.byref(acc), _ptr(af), _ptr(lg), _ptr(ab), _ptr(wg))
        if rc:
            raise OracleError("model step: ValueError")
        out = dict(loss=loss.value, acc=acc.value)
        if dumps:
            out.update(ahw_fwd=split_act(af, n, dims), loss_grad=lg, ahw_bwd=split_act(ab, n, dims),
                       w_grad=split_w(wg, dims))
        return out
