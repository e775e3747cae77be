"""On-disk formats: the native loaders of libmggcn against the compiled reference
(oracle/_ref), same files in, bit-identical CSR / features / labels / masks out, same exception type and
message for malformed input. Cases follow proj/tests/test_dataset.cpp:27-160 plus multi-chunk files
(the native loaders parse line-aligned chunks in parallel) and syntax corner cases of the reference's
extractors. Host-only: runs without a GPU."""
import os

import numpy as np
import pytest

from paper_2110_08688_b200 import rowgcn as R

CODES = {R.ShapeError: 1, R.ValueError: 2, R.ParseError: 5, R.IoError: 7}


def ours(fn, *a):
    try:
        return ("ok", fn(*a))
    except R.RowgcnError as e:
        return ("err", CODES.get(type(e), 99), str(e))


def theirs(fn, *a):
    from oracle.pyoracle import OracleError
    try:
        return ("ok", fn(*a))
    except OracleError as e:
        return ("err", e.code, e.message)


def same(a, b):
    if a[0] != b[0]:
        return False
    if a[0] == "err":
        return a[1:] == b[1:]
    x, y = a[1], b[1]
    if isinstance(x, tuple):
        return len(x) == len(y) and all(np.array_equal(np.asarray(p), np.asarray(q)) and
                                        np.asarray(p).dtype == np.asarray(q).dtype for p, q in zip(x, y))
    x, y = np.asarray(x), np.asarray(y)
    return x.shape == y.shape and x.dtype == y.dtype and x.tobytes() == y.tobytes()


def write(tmp_path, name, text, mode="w"):
    p = tmp_path / name
    with open(p, mode) as f:
        f.write(text)
    return p


def check_graph(ref, path, fmt=0):
    a = ours({0: R.load_graph, 1: R.load_matrix_market, 2: R.load_edge_list}[fmt], path)
    b = theirs(ref.load_graph, path, fmt)
    assert same(a, b), (a, b)
    return a


# ----------------------------------------------------------------------------- Matrix Market


def test_matrix_market_general_real(ref, tmp_path):
    p = write(tmp_path, "gen.mtx", "%%MatrixMarket matrix coordinate real general\n% a comment\n3 3 3\n"
                                   "1 2 1.5\n2 1 2.0\n3 3 0.5\n")
    r = check_graph(ref, p, 1)
    rp, ci, v = r[1]
    assert list(rp) == [0, 1, 2, 3] and list(ci) == [1, 0, 2] and list(v) == [1.5, 2.0, 0.5]
    check_graph(ref, p, 0)


def test_matrix_market_pattern_and_symmetric(ref, tmp_path):
    r = check_graph(ref, write(tmp_path, "pat.mtx", "%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n2 1\n"))
    assert list(r[1][2]) == [1.0, 1.0]
    r = check_graph(ref, write(tmp_path, "sym.mtx", "%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n"
                                                    "2 1 3.0\n3 3 1.0\n"))
    assert r[1][0][-1] == 3  # (1,0), (0,1), (2,2): diagonal not mirrored
    check_graph(ref, write(tmp_path, "int.mtx", "%%MatrixMarket matrix coordinate integer symmetric\n"
                                                "4 4 3\n2 1 7\n4 1 -2\n3 3 5\n"))


@pytest.mark.parametrize("body", [
    "2 2 1\n5 1 1.0\n",            # index out of bounds -> :3:
    "2 2 3\n1 1 1.0\n",            # header promised 3
    "2 2 1\n1 1\n",                # missing value
    "2 2 1\n1 x 1.0\n",            # bad entry
    "2 2 1\n1.5 1 1.0\n",          # "1" then ".5" is not an integer -> bad entry
    "% only comments\n",           # missing size line
    "2 x 1\n",                     # bad size line
    "2 3 1\n1 1 1\n",              # not square
    "2 2 1\n1 1 1e\n",             # incomplete exponent: failbit -> missing value
    "2 2 2\n1 1 1e999\n2 2 1\n",   # overflow -> missing value
    "2 2 1\n\n% c\n1 2 +.5e+1\n",  # blank and comment lines between entries
    "2 2 1\r\n1 2 2.5\r\n",        # CRLF
    "2 2 2\n1 2 1\n1 2 2\n",       # duplicate entries summed
])
def test_matrix_market_cases(ref, tmp_path, body):
    check_graph(ref, write(tmp_path, "c.mtx", "%%MatrixMarket matrix coordinate real general\n" + body), 1)


@pytest.mark.parametrize("header", [
    "%%MatrixMarket matrix array real general",
    "%%MatrixMarket matrix coordinate complex general",
    "%%MatrixMarket matrix coordinate real hermitian",
    "%MatrixMarket matrix coordinate real general",
])
def test_matrix_market_bad_headers(ref, tmp_path, header):
    a = check_graph(ref, write(tmp_path, "h.mtx", header + "\n2 2 1\n1 1 1\n"), 1)
    assert a[0] == "err" and a[1] == 5 and ":1:" in a[2]


def test_matrix_market_empty_and_missing(ref, tmp_path):
    a = check_graph(ref, write(tmp_path, "e.mtx", ""), 1)
    assert a[:2] == ("err", 5)
    a = check_graph(ref, tmp_path / "nope.mtx", 1)
    assert a[:2] == ("err", 7)


# ----------------------------------------------------------------------------- edge lists


def test_edge_list_comments_weights(ref, tmp_path):
    r = check_graph(ref, write(tmp_path, "edges.txt", "# toy graph\n0 1\n1 2 2.5\n\n2 0\n"), 2)
    rp, ci, v = r[1]
    assert rp[-1] == 3 and v[list(ci[rp[1]:rp[2]]).index(2) + rp[1]] == 2.5


@pytest.mark.parametrize("text", [
    "0 1\nnonsense\n",        # :2: expected 'u v [w]'
    "0 1\n-1 2\n",            # negative vertex id
    "0 1 abc\n1 0\n",         # unparsable weight -> 0 (failbit, value 0)
    "0 1 \n1 0\t\r\n",        # trailing whitespace keeps the default weight
    "  # indented comment\n\t\n0 3 0.25\n3 0 1e-3\n",
    "1 1 1\n1 1 2\n0 1\n",    # duplicate self loop summed, vertex 0 only as a source
    "5 5\n",                   # n = max id + 1, empty rows before
    "",                        # empty file -> empty graph
    "0 1 1e999\n",            # overflow -> clamped to max, cast to float (inf)
    "0 1 0x10\n",             # "0" then junk: weight 0
])
def test_edge_list_cases(ref, tmp_path, text):
    check_graph(ref, write(tmp_path, "e.txt", text), 2)
    check_graph(ref, write(tmp_path, "e2.txt", text), 0)


def test_large_edge_list_multichunk(ref, tmp_path):
    """> 1 MiB so the native parser splits it into line-aligned chunks; dyadic weights keep duplicate
    sums order-independent (the reference's std::sort leaves the order of equal keys unspecified)."""
    rng = np.random.default_rng(7)
    n, m = 20000, 300000
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    w = rng.choice([0.5, 1.0, 2.25, 3.0], m)
    lines = [f"{a} {b} {c}" if i % 3 else f"{a} {b}" for i, (a, b, c) in enumerate(zip(u, v, w))]
    lines[1000] = "# comment in the middle"
    p = write(tmp_path, "big.txt", "\n".join(lines) + "\n")
    assert os.path.getsize(p) > 2 << 20
    a = check_graph(ref, p, 2)
    assert a[0] == "ok"
    bad = lines.copy()
    bad[250000] = "17 nonsense"
    a = check_graph(ref, write(tmp_path, "bad.txt", "\n".join(bad) + "\n"), 2)
    assert a[0] == "err" and ":250001:" in a[2]


def test_large_matrix_market_multichunk(ref, tmp_path):
    rng = np.random.default_rng(3)
    n, m = 30000, 200000
    u = rng.integers(1, n + 1, m)
    v = rng.integers(1, n + 1, m)
    body = "\n".join(f"{a} {b} {c}" for a, b, c in zip(u, v, rng.choice([1, 2, 4], m)))
    p = write(tmp_path, "big.mtx", f"%%MatrixMarket matrix coordinate integer symmetric\n{n} {n} {m}\n{body}\n")
    assert check_graph(ref, p, 0)[0] == "ok"


# ----------------------------------------------------------------------------- features


@pytest.mark.parametrize("text", [
    "1.5,2\n-0.25,1e-3\n",
    "1,2\n3\n",                  # ragged -> :2:
    "1,2,\n3,4,\n",              # trailing comma: no extra cell
    "1,,2\n",                    # empty cell -> bad number
    " 1, 2\n3 ,4x\n",            # stod: leading spaces, trailing text ignored
    "inf,nan\n0x1p3,-0\n",       # stod accepts what strtod accepts
    "1e400,1\n",                 # out of range -> bad number
    "\n\n1,2\n\n3,4\n",          # empty lines skipped
    "1,2\r\n3,4\r\n",            # CRLF: "2\r" parses
    "1,2\n\r\n",                 # a "\r" line is not empty -> bad number
    "",                          # no feature rows
])
def test_csv_features(ref, tmp_path, text):
    p = write(tmp_path, "f.csv", text)
    a, b = ours(R.load_features, p), theirs(ref.load_features, p)
    if a[0] == "ok" and b[0] == "ok":  # NaN payloads compare by bits
        assert a[1].tobytes() == b[1].tobytes() and a[1].shape == b[1].shape
    else:
        assert same(a, b), (a, b)


def test_large_csv_multichunk(ref, tmp_path):
    rng = np.random.default_rng(1)
    x = rng.standard_normal((40000, 12)).astype(np.float64)
    p = tmp_path / "big.csv"
    np.savetxt(p, x, delimiter=",", fmt="%.9g")
    a, b = ours(R.load_features, p), theirs(ref.load_features, p)
    assert a[0] == "ok" and same(a, b)
    lines = open(p).read().splitlines()
    lines[31234] = lines[31234] + ",7"
    p2 = write(tmp_path, "ragged.csv", "\n".join(lines) + "\n")
    a, b = ours(R.load_features, p2), theirs(ref.load_features, p2)
    assert a[0] == "err" and ":31235:" in a[2] and same(a, b)


def test_mgdm_round_trip_and_errors(ref, tmp_path):
    x = np.arange(12, dtype=np.float32).reshape(3, 4) / 7
    R.write_dense(tmp_path / "ours.bin", x)
    ref.write_dense(tmp_path / "ref.bin", x)
    assert open(tmp_path / "ours.bin", "rb").read() == open(tmp_path / "ref.bin", "rb").read()
    for fn in (R.load_features, R.read_dense):
        assert np.array_equal(fn(tmp_path / "ours.bin"), x)
    # f64 payload converted element-wise
    x64 = np.linspace(-1, 1, 10).reshape(2, 5)
    blob = b"MGDM" + np.uint64(2).tobytes() + np.uint64(5).tobytes() + bytes([8]) + x64.tobytes()
    p = write(tmp_path, "f64.bin", blob, "wb")
    assert same(ours(R.read_dense, p), theirs(ref.read_dense, p))
    assert same(ours(R.load_features, p), theirs(ref.load_features, p))
    for name, data in [("trunc.bin", blob[:-3]), ("width.bin", blob[:20] + bytes([2]) + blob[21:]),
                       ("hdr.bin", blob[:10]), ("magic.bin", b"XGDM" + blob[4:])]:
        p = write(tmp_path, name, data, "wb")
        assert same(ours(R.read_dense, p), theirs(ref.read_dense, p)), name
    assert same(ours(R.read_dense, tmp_path / "missing.bin"), theirs(ref.read_dense, tmp_path / "missing.bin"))


# ----------------------------------------------------------------------------- labels and masks


@pytest.mark.parametrize("text", ["0\n1\n", "# c\n 3\n\n-2\n7 trailing\n", "1\nabc\n", "99999999999999999999\n",
                                  "4294967297\n", "", "\t\r\n5\r\n"])
def test_labels(ref, tmp_path, text):
    p = write(tmp_path, "l.txt", text)
    assert same(ours(R.load_labels, p), theirs(ref.load_labels, p))


@pytest.mark.parametrize("text", [
    '{"train": [0], "test": [1]}',
    '{"train": [0, 2, 2], "val": [1], "other": {"x": [1, "s", null]}}',
    '{"train": [5]}',                      # out of range
    '{"train": [0.9, 2]}',                 # nlohmann get<int64_t>: floats truncate
    '{"train": [0, true]}',                # ... booleans are a type error
    '{"val": null, "test": 1}',            # null iterates empty; a scalar iterates once
    '{"train": [0], "train": [1]}',        # duplicate key: last wins
    '{"train": [0]',                       # invalid JSON
    '[1, 2]',                              # not an object: no masks
    '{}',
])
def test_masks(ref, tmp_path, text):
    p = write(tmp_path, "m.json", text)
    a, b = ours(R.load_masks, p, 3), theirs(ref.load_masks, p, 3)
    if a[0] == "err" or b[0] == "err":  # nlohmann's messages differ; ParseError (or its type_error, 99)
        assert a[0] == b[0] == "err" and a[1] == 5 and b[1] in (5, 99)
    else:
        assert same(a, b), (a, b)


# ----------------------------------------------------------------------------- load_dataset


def test_load_dataset_toy_round_trip_with_masks(ref, tmp_path):
    """proj/tests/test_dataset.cpp:105-123."""
    write(tmp_path, "toy.edges", "0 1\n1 0\n")
    write(tmp_path, "toy.labels", "0\n1\n")
    write(tmp_path, "toy.masks.json", '{"train": [0], "test": [1]}')
    feats = np.zeros((2, 3), np.float32)
    feats[0, 0], feats[1, 2] = 1.0, -1.0
    R.write_dense(tmp_path / "toy.features", feats)
    paths = [tmp_path / f for f in ("toy.edges", "toy.features", "toy.labels", "toy.masks.json")]
    ds = R.load_dataset(*paths)
    rds, (tr, va, te) = ref.load_dataset(*paths)
    assert ds.n() == 2 and ds.d0 == 3 and ds.num_classes() == 2
    assert list(ds.labels) == [0, 1] and list(ds.train_mask) == [1, 0] and list(ds.test_mask) == [0, 1]
    assert len(ds.val_mask) == 0 and len(va) == 0
    rp, ci, v = ds.graph
    assert np.array_equal(rp, rds.row_ptr) and np.array_equal(ci, rds.col_idx) and np.array_equal(v, rds.values)
    assert np.array_equal(ds.features, rds.features) and np.array_equal(ds.labels, rds.labels)
    assert np.array_equal(ds.train_mask, tr) and np.array_equal(ds.test_mask, te)


def test_load_dataset_dimension_mismatch(ref, tmp_path):
    """proj/tests/test_dataset.cpp:125-139: the ShapeError names both counts."""
    write(tmp_path, "m.edges", "0 1\n1 2\n2 0\n")
    write(tmp_path, "m.features.csv", "1.0,2.0\n3.0,4.0\n")
    write(tmp_path, "m.labels", "0\n0\n0\n")
    paths = [tmp_path / f for f in ("m.edges", "m.features.csv", "m.labels")]
    a = ours(R.load_dataset, *paths)
    b = theirs(ref.load_dataset, *paths)
    assert a[:2] == ("err", 1) and "2" in a[2] and "3" in a[2] and same(a, b)
    write(tmp_path, "m.labels", "0\n0\n")
    write(tmp_path, "m.features.csv", "1.0,2.0\n3.0,4.0\n5,6\n")
    assert same(ours(R.load_dataset, *paths), theirs(ref.load_dataset, *paths))


def test_loaded_dataset_prepares_like_reference(ref, tmp_path):
    """A loaded graph flows through prepare_data: the permutation and tiles stay bit-identical."""
    from oracle.pyoracle import make_cfg
    rng = np.random.default_rng(5)
    n = 500
    u, v = rng.integers(0, n, 4000), rng.integers(0, n, 4000)
    write(tmp_path, "g.txt", "".join(f"{a} {b}\n{b} {a}\n" for a, b in zip(u, v)) + f"{n - 1} {n - 1}\n")
    np.savetxt(tmp_path / "x.csv", rng.standard_normal((n, 6)), delimiter=",")
    write(tmp_path, "y.txt", "".join(f"{c}\n" for c in rng.integers(0, 4, n)))
    paths = [tmp_path / f for f in ("g.txt", "x.csv", "y.txt")]
    ds = R.load_dataset(*paths)
    rds, _ = ref.load_dataset(*paths)
    cfg = R.GcnConfig([6, 8, 4], epochs=1, seed=9, permute=True)
    prep = R.prepare_data(ds, cfg, 2)
    rprep = ref.prepare(rds, make_cfg([6, 8, 4], seed=9, permute=True), 2)
    for d in range(2):
        for i in range(2):
            for j in range(2):
                got = prep.tile(d, i, j)
                want = rprep.tiles[d][i][j]
                for g_, w_ in zip(got, want):
                    assert np.array_equal(np.asarray(g_), np.asarray(w_))


def test_cpp_dropin_load_dataset(tmp_path):
    """examples/load_dataset.cpp: the C++ drop-in's load_dataset (rowgcn::load_dataset) end to end."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_2110_08688_b200")
    exe = tmp_path / "load_dataset"
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-Werror", "-I", os.path.join(root, "include"),
                        os.path.join(root, "examples", "load_dataset.cpp"), "-L", libdir, "-lmggcn",
                        f"-Wl,-rpath,{libdir}", "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    write(tmp_path, "g.mtx", "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 2\n2 1\n3 2\n")
    write(tmp_path, "x.csv", "1,2\n3,4\n5,6.5\n")
    write(tmp_path, "y.txt", "0\n2\n1\n")
    write(tmp_path, "m.json", '{"train": [0, 2], "val": [1]}')
    out = subprocess.run([str(exe), *(str(tmp_path / f) for f in ("g.mtx", "x.csv", "y.txt", "m.json"))],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip() == "n=3 nnz=4 d0=2 classes=3 train=2 val=3 test=0 fsum=21.500000"
    write(tmp_path, "bad.csv", "1,2\n3\n5,6\n")
    out = subprocess.run([str(exe), *(str(tmp_path / f) for f in ("g.mtx", "bad.csv", "y.txt"))],
                         capture_output=True, text=True)
    assert out.returncode == 1 and out.stdout.startswith("ParseError: ") and ":2:" in out.stdout
