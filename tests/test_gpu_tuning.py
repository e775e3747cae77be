"""Launch-geometry knobs must not change results: the column-slab SpMM keeps every output element's
fold order, so exact mode stays bitwise and fast mode stays identical to its unslabbed self."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from test_gpu_kernels import random_tile, run_spmm  # noqa: E402
from gpu_util import bits_equal  # noqa: E402

from paper_2110_08688_b200 import rowgcn as R  # noqa: E402


@pytest.mark.parametrize("slab", [4, 8, 16, 64])
@pytest.mark.parametrize("w", [8, 47, 256])
def test_spmm_slab_exact_bitwise(port32, slab, w):
    rng = np.random.default_rng(slab * 7 + w)
    rows, cols = 200, 400
    rp, ci, v = random_tile(rng, rows, cols, 0.03)
    h = rng.uniform(-1, 1, (cols, w)).astype(np.float32)
    o0 = rng.uniform(-1, 1, (rows, w)).astype(np.float32)
    ref = port32.spmm(rows, cols, rp, ci, v, h, True, o0)
    R.set_tuning("spmm_slab", slab)
    try:
        exact = run_spmm(rp, ci, v, h, True, o0)
        fast = run_spmm(rp, ci, v, h, True, o0, mode=R.SPMM_FAST)
    finally:
        R.set_tuning("spmm_slab", 0)
    assert bits_equal(exact, ref)
    assert bits_equal(fast, run_spmm(rp, ci, v, h, True, o0, mode=R.SPMM_FAST))


@pytest.mark.parametrize("group", [4, 8])
@pytest.mark.parametrize("w", [36, 47, 48, 64])
def test_spmm_narrow_group_variants(port32, group, w):
    rng = np.random.default_rng(group + w)
    rows, cols = 300, 500
    rp, ci, v = random_tile(rng, rows, cols, 0.02)
    h = rng.uniform(-1, 1, (cols, w)).astype(np.float32)
    o0 = rng.uniform(-1, 1, (rows, w)).astype(np.float32)
    ref = port32.spmm(rows, cols, rp, ci, v, h, True, o0)
    base_fast = run_spmm(rp, ci, v, h, True, o0, mode=R.SPMM_FAST)
    R.set_tuning("spmm_narrow_group", group)
    try:
        exact = run_spmm(rp, ci, v, h, True, o0)
        fast = run_spmm(rp, ci, v, h, True, o0, mode=R.SPMM_FAST)
    finally:
        R.set_tuning("spmm_narrow_group", 0)
    assert bits_equal(exact, ref)
    assert bits_equal(fast, base_fast)


def test_slab_training_equals_default():
    ds = R.synth_graph(3000, 10.0, 0.7, 2, 12, 5)
    cfg = R.GcnConfig([12, 40, 5], epochs=3, seed=2, permute=True)
    a = R.train_run(ds, cfg, R.TrainOptions(devices=[0]))
    R.set_tuning("spmm_slab", 8)
    try:
        b = R.train_run(ds, cfg, R.TrainOptions(devices=[0]))
    finally:
        R.set_tuning("spmm_slab", 0)
    assert a.epoch_loss == b.epoch_loss and a.w_hashes == b.w_hashes


@pytest.mark.parametrize("w", [32, 40, 47, 64, 100, 128, 256, 300, 512])
def test_spmm_async_pipeline_bitwise(w):
    """The cp.async-pipelined FAST gather keeps each lane's FMA chain: bitwise equal to the register
    gather, with hub segments, accumulate and relu, rows shorter and longer than the record windows."""
    rng = np.random.default_rng(w + 11)
    rows, cols = 400, 700
    rp, ci, v = random_tile(rng, rows, cols, 0.05, hub_rows=(3, 17, 200), hub_len=650)
    h = rng.uniform(-1, 1, (cols, w)).astype(np.float32)
    o0 = rng.uniform(-1, 1, (rows, w)).astype(np.float32)
    R.set_tuning("heavy_row", 128)
    try:
        outs = {}
        # register gather; cp.async ring per row (spmm_fast_async); row-streaming pieces (spmm_fast_stream)
        for key, (on, stream) in {"reg": (0, 0), "async": (1, 0), "stream": (1, 1)}.items():  # 2 = auto
            R.set_tuning("spmm_async", on)
            R.set_tuning("spmm_stream", stream)
            outs[key] = (run_spmm(rp, ci, v, h, mode=R.SPMM_FAST),
                         run_spmm(rp, ci, v, h, True, o0, relu=True, mode=R.SPMM_FAST))
    finally:
        R.set_tuning("spmm_async", 1)
        R.set_tuning("spmm_stream", 2)
        R.set_tuning("heavy_row", 4096)
    for key in ("async", "stream"):
        for a, b in zip(outs["reg"], outs[key]):
            assert bits_equal(a, b), key
    outs[1] = outs["stream"]
    ref = (rp, ci, v)
    dense = np.zeros((rows, cols), np.float64)
    for r in range(rows):
        dense[r, ci[rp[r]:rp[r + 1]]] = v[rp[r]:rp[r + 1]]
    assert np.max(np.abs(outs[1][0] - dense @ h.astype(np.float64))) <= 1e-4 * max(1.0, np.max(np.abs(dense @ h)))
    del ref


@pytest.mark.parametrize("hub_bytes", [0, 1 << 20, 96 << 20])
def test_hub_l2_hints_do_not_change_results(hub_bytes):
    """FAST edge records carry a hub class in the column's top bits; the L2 evict_last / evict_first hints
    they select change caching only: training is bitwise identical with and without them."""
    ds = R.synth_graph(30000, 20.0, 0.7, 8, 24, 5)
    cfg = R.GcnConfig([24, 64, 5], epochs=2, seed=1, permute=True, spmm_mode=R.SPMM_FAST)
    a = R.train_run(ds, cfg, R.TrainOptions(devices=[0]))
    R.set_tuning("spmm_hub_bytes", hub_bytes)
    try:
        b = R.train_run(ds, cfg, R.TrainOptions(devices=[0]))
    finally:
        R.set_tuning("spmm_hub_bytes", 96 << 20)
    assert a.epoch_loss == b.epoch_loss and a.w_hashes == b.w_hashes


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_backward_tile_transposed_on_device(mode):
    """P = 1 builds the backward tile (Â) on the device as the transpose of the uploaded forward tile (Âᵀ):
    training is bitwise the same as with the uploaded backward tile (weighted graph: the values matter)."""
    kw = dict(gemm_mode=R.GEMM_EXACT, spmm_mode=R.SPMM_EXACT) if mode == "exact" else {}
    rng = np.random.default_rng(4)
    n, m = 3000, 40000
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    keys = np.unique(u * n + v)
    rows, cols = keys // n, keys % n
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    rp = np.cumsum(rp)
    vals = rng.uniform(0.1, 2.0, len(keys)).astype(np.float32)
    x = rng.uniform(-1, 1, (n, 12)).astype(np.float32)
    lab = rng.integers(0, 5, n).astype(np.int32)
    ds = R.Dataset.from_arrays(rp, cols.astype(np.int64), vals, x, lab)
    cfg = R.GcnConfig([12, 32, 5], epochs=3, seed=7, permute=True, **kw)
    runs = []
    for flag in (0, 1):
        R.set_tuning("bwd_transpose", flag)
        try:
            runs.append(R.train_run(ds, cfg, R.TrainOptions(devices=[0])))
        finally:
            R.set_tuning("bwd_transpose", 1)
    assert runs[0].epoch_loss == runs[1].epoch_loss
    for a, b in zip(runs[0].final_w, runs[1].final_w):
        assert a.tobytes() == b.tobytes()


def test_block_cache_reuses_memory_across_groups():
    """Destroyed groups' device blocks are cached and reused: creating and destroying groups of the same
    shape repeatedly does not grow the device's used memory, and results do not change."""
    ds = R.synth_graph(20000, 10.0, 0.7, 5, 32, 6)
    cfg = R.GcnConfig([32, 64, 6], epochs=2, seed=3, permute=True)
    first = R.train_run(ds, cfg, R.TrainOptions(devices=[0]))
    torch.cuda.synchronize()
    free0, total = torch.cuda.mem_get_info()
    for _ in range(4):
        again = R.train_run(ds, cfg, R.TrainOptions(devices=[0]))
        assert again.epoch_loss == first.epoch_loss
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < 64 << 20  # the repeats ran out of the cache


@pytest.mark.parametrize("w", [32, 40, 128, 256, 512])
@pytest.mark.parametrize("density,piece_nnz", [(0.002, 1024), (0.002, 1), (0.02, 7), (0.02, 100000)])
def test_spmm_stream_pieces_bitwise(w, density, piece_nnz):
    """Row-streaming pieces (spmm_fast_stream): many empty and 1-2 nonzero rows, pieces of one row
    (piece_nnz 1) up to 32 rows, hub segments in the same work list, accumulate (prefetched old rows) and
    relu: bitwise equal to the per-row cp.async kernel."""
    rng = np.random.default_rng(int(w / density) + piece_nnz)
    rows, cols = 1000, 900
    rp, ci, v = random_tile(rng, rows, cols, density, hub_rows=(0, 31, 32, 500, 999), hub_len=700)
    h = rng.uniform(-1, 1, (cols, w)).astype(np.float32)
    o0 = rng.uniform(-1, 1, (rows, w)).astype(np.float32)
    R.set_tuning("heavy_row", 256)
    R.set_tuning("fast_segment", 64)
    R.set_tuning("piece_nnz", piece_nnz)
    try:
        outs = {}
        for stream in (0, 1):
            R.set_tuning("spmm_stream", stream)
            outs[stream] = (run_spmm(rp, ci, v, h, mode=R.SPMM_FAST),
                            run_spmm(rp, ci, v, h, True, o0, mode=R.SPMM_FAST),
                            run_spmm(rp, ci, v, h, True, o0, relu=True, mode=R.SPMM_FAST))
    finally:
        R.set_tuning("spmm_stream", 2)
        R.set_tuning("piece_nnz", 1024)
        R.set_tuning("heavy_row", 4096)
        R.set_tuning("fast_segment", 2048)
    for a, b in zip(outs[0], outs[1]):
        assert bits_equal(a, b)


def test_spmm_stream_training_bitwise():
    """Whole training steps (P = 1 and the staged P = 3 with accumulating stages) are bitwise identical with
    the row-streaming kernel on and off."""
    ds = R.synth_graph(20000, 9.0, 0.7, 4, 40, 6)
    for P in (1, 3):
        cfg = R.GcnConfig([40, 64, 64, 6], epochs=2, seed=2, permute=True, overlap=P > 1, gemm_mode=R.GEMM_TF32X3,
                          spmm_mode=R.SPMM_FAST, aggregate_input=True)
        opts = R.TrainOptions(workers=P, devices=[0] * P, transport=R.TRANSPORT_NCCL if P == 1 else R.TRANSPORT_LOCAL)
        try:
            R.set_tuning("spmm_stream", 0)
            a = R.train_run(ds, cfg, opts)
            R.set_tuning("spmm_stream", 1)
            b = R.train_run(ds, cfg, opts)
        finally:
            R.set_tuning("spmm_stream", 2)
        assert a.epoch_loss == b.epoch_loss and a.w_hashes == b.w_hashes, P


@pytest.mark.parametrize("P,overlap,k", [(3, True, 2), (4, False, 2), (8, True, 2), (8, True, 4), (8, False, 7)])
def test_stage_fold(ref, P, overlap, k):
    """stage_fold = k (FAST, P > 2): up to k received stages in one SpMM over a merged tile — the same sums in
    another association. Teacher-forced step 1: W_G and the H-grads within 1e-5 (normwise) of the
    stage-by-stage schedule; 3 epochs: losses of both schedules within 1e-4 of the f64 reference (the
    product contract; W after Adam amplifies the reassociation of tiny gradients, so the two trajectories are
    compared through the reference, not to each other). In-process transport."""
    from gpu_util import normwise
    from oracle.pyoracle import make_cfg
    dims = [24, 64, 32, 6]
    ds = R.synth_graph(6000, 20.0, 0.9, 3, dims[0], dims[-1])
    cfg = R.GcnConfig(dims, epochs=3, seed=5, permute=True, overlap=overlap,
                      gemm_mode=R.GEMM_TF32X3, spmm_mode=R.SPMM_FAST, aggregate_input=True)
    opts = dict(workers=P, devices=[0] * P, transport=R.TRANSPORT_LOCAL)
    prep = R.prepare_data(ds, cfg, P)

    def step1():
        with R.Group(cfg, prep, P, devices=[0] * P, transport=R.TRANSPORT_LOCAL) as g:
            g.init_params()
            loss = g.compute_gradients()
            return loss, [g.read(R.T_WGRAD, l) for l in range(3)], [g.read(R.T_AHW, l, r) for l in range(2) for r in range(P)]

    base1, base = step1(), R.train_run(ds, cfg, R.TrainOptions(**opts))
    R.set_tuning("stage_fold", k)
    try:
        fold1, fold = step1(), R.train_run(ds, cfg, R.TrainOptions(**opts))
    finally:
        R.set_tuning("stage_fold", 0)
    assert abs(fold1[0] - base1[0]) <= 1e-6 * abs(base1[0])
    for a, b in zip(fold1[1] + fold1[2], base1[1] + base1[2]):
        assert normwise(a, b) <= 1e-5
    assert fold1[1][0].tobytes() != base1[1][0].tobytes()  # the folded schedule ran (another association)
    r64 = ref.train_run(ref.synth(6000, 20.0, 0.9, 3, dims[0], dims[-1], dtype=np.float64),
                        make_cfg(dims, epochs=3, seed=5, permute=True, overlap=overlap), P, np.float64)
    for e in range(3):
        assert abs(base.epoch_loss[e] - r64["loss"][e]) <= 1e-4 * abs(r64["loss"][e])
        assert abs(fold.epoch_loss[e] - r64["loss"][e]) <= 1e-4 * abs(r64["loss"][e])


def test_solo_transport_steps():
    """MG_TRANSPORT_SOLO (measurement only): one rank of a P-way job alone, collectives skipped — it creates,
    steps and reports; more than one local rank is refused."""
    ds = R.synth_graph(4000, 10.0, 0.7, 2, 16, 4)
    cfg = R.GcnConfig([16, 32, 4], epochs=2, seed=2, permute=True, overlap=True, gemm_mode=R.GEMM_TF32X3,
                      spmm_mode=R.SPMM_FAST, aggregate_input=True)
    prep = R.synth_prepare_rank(4000, 10.0, 0.7, 2, 16, 4, cfg, 4, 1)
    with R.Group(cfg, prep, 4, local_ranks=[1], devices=[0], transport=R.TRANSPORT_SOLO) as g:
        g.init_params()
        for t in (1, 2):
            g.train_step(t)
    full = R.prepare_data(ds, cfg, 4)
    with pytest.raises(R.ValueError, match="solo"):
        R.Group(cfg, full, 4, local_ranks=[0, 1], devices=[0, 0], transport=R.TRANSPORT_SOLO)


@pytest.mark.parametrize("P", [1, 3])
def test_f16_split_training(ref, P):
    """gemm_f16 (opt-in): NN / NT on the scaled fp16 split with producer-written row maxima, in the training
    step — losses within 1e-4 of the f64 reference over 4 epochs (the product contract), at P = 1 and on the
    in-process transport, including a layer whose N is not a multiple of 32 (stale TMEM columns past N)."""
    from oracle.pyoracle import make_cfg
    dims = [20, 48, 24, 5]
    ds = R.synth_graph(3000, 8.0, 0.7, 11, dims[0], dims[-1])
    cfg = R.GcnConfig(dims, epochs=4, seed=2, permute=True, overlap=P > 1, gemm_mode=R.GEMM_TF32X3,
                      spmm_mode=R.SPMM_FAST, aggregate_input=True)
    import os
    R.set_tuning("gemm_f16", 1)
    R.set_tuning("gemm_f16_min_k", 0)
    os.environ["MGGCN_POISON_RM"] = "1"  # row maxima start as 8e37: any row read before its producer wrote it
    try:                                  # would scale its A row to zero and break the trajectory
        got = R.train_run(ds, cfg, R.TrainOptions(workers=P, devices=[0] * P,
                                                 transport=R.TRANSPORT_NCCL if P == 1 else R.TRANSPORT_LOCAL))
        with R.Group(cfg, R.prepare_data(ds, cfg, P), P, devices=[0] * P,
                     transport=R.TRANSPORT_NCCL if P == 1 else R.TRANSPORT_LOCAL) as g:
            g.init_params()
            g.forward()
            a0 = g.read(R.T_AHW, 0)
            rm = g.read(R.T_ROWMAX, 0)
            assert np.array_equal(np.maximum(rm[:, 0], rm[:, 1]), np.abs(a0).max(1))  # producer-written maxima
    finally:
        os.environ.pop("MGGCN_POISON_RM", None)
        R.set_tuning("gemm_f16", 0)
        R.set_tuning("gemm_f16_min_k", 128)
    r64 = ref.train_run(ref.synth(3000, 8.0, 0.7, 11, dims[0], dims[-1], dtype=np.float64),
                        make_cfg(dims, epochs=4, seed=2, permute=True, overlap=P > 1), P, np.float64)
    for e in range(4):
        assert abs(got.epoch_loss[e] - r64["loss"][e]) <= 1e-4 * abs(r64["loss"][e])
