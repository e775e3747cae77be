"""The C++ / Python drop-in against the reference's own API surface (CPU only, no device work):

* checkpoint files and their <path>.json sidecar are byte-identical to the compiled reference's
  write_checkpoint (inc/driver.hpp:255-274), and config_to_json / BreakdownReport dumps are
  byte-identical to nlohmann::json::dump (driver.hpp:59-71, breakdown.hpp:27-58);
* read_checkpoint errors and round trip (driver.hpp:276-299, tests/test_dataset.cpp:211-236);
* from_coo / add_self_loops semantics (sparse.hpp:59-90, dataset.hpp:60-73);
* the reference's own callers — run_train (tools/main.cpp:56-101) and the train_run / grad_run cases of
  tests/test_gcn.cpp:213-348 — compile UNCHANGED against include/mggcn/rowgcn.hpp (extracted at build time
  by tests/dropin/extract.py), and S = double is rejected at compile time with a message.
"""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from oracle.pyoracle import make_cfg
from paper_2110_08688_b200 import rowgcn as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REFERENCE = "/root/reference/proj/include/rowgcn"
JSON_DIR = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"

CONFIGS = [
    dict(dims=[3, 4, 2], epochs=100),
    dict(dims=[100, 256, 256, 47], lr=0.05, epochs=3, seed=12345678901234, permute=True, overlap=True),
    dict(dims=[7, 1], epochs=7, lr=1e-5, beta1=0.5, beta2=0.25, epsilon=1e-12, skip_first_backward_spmm=True,
         order_swap=True),
    dict(dims=[2, 3], lr=123.0, beta1=0.0001, beta2=1e20, epsilon=2.5e-7, epochs=0),
    dict(dims=[5, 5], epochs=1, lr=0.1 + 0.2, beta1=1 / 3, beta2=1e15, epsilon=1e16, seed=2 ** 64 - 1),
]


def ours_cfg(c):
    kw = {k: v for k, v in c.items() if k != "dims"}
    return R.GcnConfig(list(c["dims"]), **kw)


def upstream_arrays(text, indent):
    """The oracle build's json.hpp is cudnn_frontend's bundled nlohmann 3.11.3, which carries one local edit
    ("Custom from FE": integer arrays stay on one line under pretty printing). The reference vendors upstream
    3.11.3, whose dump(indent) puts every array element on its own line; map the edit back.
    Only top-level members hold arrays in these documents (layer_dims), so the nesting level is 1."""
    import re
    if indent < 0:
        return text
    inner, outer = " " * (2 * indent), " " * indent
    return re.sub(r"\[(-?\d+(?:,-?\d+)*)\]",
                  lambda m: "[\n" + ",\n".join(inner + x for x in m.group(1).split(",")) + "\n" + outer + "]", text)


def ref_text(ref, fn, *args):
    n = C.c_int64()
    buf = C.create_string_buffer(1 << 16)
    assert getattr(ref.lib, fn)(*args, buf, 1 << 16, C.byref(n)) == 0
    return buf.raw[:n.value].decode()


@pytest.mark.parametrize("i", range(len(CONFIGS)))
@pytest.mark.parametrize("indent", [-1, 0, 1, 2, 4])
def test_config_to_json_bytes(ref, i, indent):
    c = CONFIGS[i]
    rc = make_cfg(**c)
    theirs = upstream_arrays(ref_text(ref, "ref_config_json", C.byref(rc), indent), indent)
    assert R.config_to_json_text(ours_cfg(c), indent) == theirs


@pytest.mark.parametrize("totals", [[0] * 6, [1.5, 2.25, 0, 1e-3, 7, 123456.789], [3e7, 1, 2, 3, 4, 5]])
@pytest.mark.parametrize("indent", [-1, 1, 2])
def test_breakdown_json_and_table_bytes(ref, totals, indent):
    t = (C.c_double * 6)(*totals)
    ours = R._text(R.lib().mg_breakdown_to_json, t, indent) + "\n" + R._text(R.lib().mg_breakdown_text, t)
    assert ours == ref_text(ref, "ref_breakdown_json", t, indent)


@pytest.mark.parametrize("i", range(len(CONFIGS)))
def test_checkpoint_bytes_equal_reference(ref, tmp_path, i):
    c = CONFIGS[i]
    rng = np.random.default_rng(i)
    dims = c["dims"]
    ws = [rng.standard_normal((dims[l], dims[l + 1])).astype(np.float32) for l in range(len(dims) - 1)]
    ours, theirs = tmp_path / "ours.ckpt", tmp_path / "ref.ckpt"
    R.write_checkpoint(ours, ws, ours_cfg(c))
    rows = np.array([w.shape[0] for w in ws], np.int64)
    cols = np.array([w.shape[1] for w in ws], np.int64)
    ptrs = (C.c_void_p * len(ws))(*[w.ctypes.data for w in ws])
    rc = make_cfg(**c)
    assert ref.lib.ref_write_checkpoint_f32(str(theirs).encode(), len(ws), rows.ctypes.data_as(C.c_void_p),
                                            cols.ctypes.data_as(C.c_void_p), ptrs, C.byref(rc)) == 0
    assert ours.read_bytes() == theirs.read_bytes()
    side = upstream_arrays((tmp_path / "ref.ckpt.json").read_text(), 1)
    assert (tmp_path / "ours.ckpt.json").read_text() == side
    back = R.read_checkpoint(theirs)  # and we read the reference's file back bit for bit
    assert len(back) == len(ws) and all(np.array_equal(a.view(np.uint32), b.view(np.uint32)) for a, b in zip(back, ws))


def test_checkpoint_errors(tmp_path):
    # tests/test_dataset.cpp:211-236 round trip + the read_checkpoint failure modes (driver.hpp:276-299)
    p = tmp_path / "ck.bin"
    ws = [np.arange(12, dtype=np.float32).reshape(3, 4), np.ones((4, 2), np.float32)]
    R.write_checkpoint(p, ws, R.GcnConfig([3, 4, 2]))
    import json
    assert json.loads((tmp_path / "ck.bin.json").read_text())["layer_dims"] == [3, 4, 2]
    raw = p.read_bytes()
    (tmp_path / "magic.bin").write_bytes(b"XGDM" + raw[4:])
    with pytest.raises(R.ParseError, match="bad checkpoint block magic"):
        R.read_checkpoint(tmp_path / "magic.bin")
    (tmp_path / "trunc.bin").write_bytes(raw[:-3])
    with pytest.raises(R.ParseError, match="truncated checkpoint block"):
        R.read_checkpoint(tmp_path / "trunc.bin")
    (tmp_path / "f64.bin").write_bytes(raw[:20] + bytes([8]) + raw[21:])
    with pytest.raises(R.ParseError, match="dtype width 8 does not match run dtype 4"):
        R.read_checkpoint(tmp_path / "f64.bin")
    with pytest.raises(R.IoError, match="cannot open"):
        R.read_checkpoint(tmp_path / "missing.bin")
    with pytest.raises(R.IoError, match="for writing"):
        R.write_checkpoint(tmp_path / "no" / "dir.bin", ws, R.GcnConfig([3, 4, 2]))


def test_from_coo_and_self_loops():
    rng = np.random.default_rng(3)
    n, m = 50, 400
    s, d = rng.integers(0, n, m), rng.integers(0, n, m)
    w = rng.integers(1, 4, m).astype(np.float32)  # small integers: sums are exact in any order
    rp, ci, v = R.from_coo(s, d, w, n)
    dense = np.zeros((n, n), np.float64)
    np.add.at(dense, (s, d), w)
    nz = np.nonzero(dense)
    assert np.array_equal(rp, np.concatenate([[0], np.cumsum(np.bincount(nz[0], minlength=n))]))
    assert np.array_equal(ci, nz[1]) and np.array_equal(v, dense[nz].astype(np.float32))
    with pytest.raises(R.ValueError, match=r"from_coo: edge \(3, 50\) out of range for n=50"):
        R.from_coo([3], [50], [1.0], n)
    rp2, ci2, v2 = R.add_self_loops(rp, ci, v)
    dense2 = dense.copy()
    for u in range(n):
        if dense2[u, u] == 0:
            dense2[u, u] = 1.0
    nz2 = np.nonzero(dense2)
    assert np.array_equal(ci2, nz2[1]) and np.array_equal(v2, dense2[nz2].astype(np.float32))
    assert np.array_equal(rp2[1:] - rp2[:-1], np.bincount(nz2[0], minlength=n))


def _compile(src, out, extra=()):
    return subprocess.run(["g++", "-std=gnu++20", "-O0", "-fsyntax-only" if out is None else "-O1",
                           "-I", os.path.join(ROOT, "include"), "-I", JSON_DIR, *extra, str(src),
                           *([] if out is None else ["-L", os.path.join(ROOT, "paper_2110_08688_b200"), "-lmggcn",
                                                     "-o", str(out)])],
                          capture_output=True, text=True)


@pytest.mark.skipif(not os.path.isdir(REFERENCE), reason="reference callers are extracted in the build container")
def test_reference_callers_compile_unchanged():
    r = subprocess.run(["bash", os.path.join(ROOT, "tests", "dropin", "build_dropin.sh")], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert os.access(os.path.join(ROOT, "tests", "dropin", "_build", "dropin_main"), os.X_OK)


def test_double_is_rejected_at_compile_time(tmp_path):
    src = tmp_path / "dbl.cpp"
    src.write_text('#include "mggcn/rowgcn.hpp"\nnamespace R = mggcn::rowgcn;\n'
                   "int main() { auto ds = R::synth_graph<double>(10, 2.0, 0.7, 1); (void)ds; }\n")
    r = _compile(src, None)
    assert r.returncode != 0 and "runs in float" in r.stderr
    src.write_text('#include "mggcn/rowgcn.hpp"\nnamespace R = mggcn::rowgcn;\n'
                   "int main() { auto ds = R::synth_graph<float>(10, 2.0, 0.7, 1); (void)ds; }\n")
    assert _compile(src, None).returncode == 0
