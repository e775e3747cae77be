"""World-size-2 tests of the multi-rank host logic on CPU (gloo), the way bench.py drives the device
path under torchrun: per-rank prepare_data(only_rank), the shared NCCL id exchange, and the staged
1D row-broadcast protocol (inc/dist_spmm.hpp:57-103) plus the canonical-block W-grad all-reduce
(inc/gcn.hpp:316-335) replayed with torch.distributed collectives over the rank's own tiles. The
arithmetic is the C oracle's (test infrastructure), so the checks are bitwise."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    from oracle.pyoracle import Port
    from paper_2110_08688_b200 import rowgcn as R
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        port32 = Port(np.float32)
        # 1. the shared NCCL unique id (bench.py: rank 0 creates it, torch.distributed broadcasts it)
        obj = [R.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
        ids = [None] * world
        dist.all_gather_object(ids, nid)
        assert all(i == ids[0] for i in ids) and len(nid) == 128
        # 2. per-rank partition == the corresponding row block of the full partition
        n, w = 900, 12
        ds = R.synth_graph(n, 9.0, 0.7, 3, 5, 3)
        cfg = R.GcnConfig([5, w, 3], seed=4, permute=True)
        mine = R.prepare_data(ds, cfg, world, only_rank=rank)
        full = R.prepare_data(ds, cfg, world)
        for d in (0, 1):
            for j in range(world):
                for a, b in zip(mine.tile(d, rank, j), full.tile(d, rank, j)):
                    assert np.array_equal(a, b)
        # 2b. the per-rank synthetic input path with the degree all-gather bench.py uses under torchrun
        #     (mg_synth_rank_*): identical to the same row block of the whole-graph partition
        from paper_2110_08688_b200.torchdist import degree_exchange
        sr = R.synth_prepare_rank(n, 9.0, 0.7, 3, 5, 3, cfg, world, rank, exchange=degree_exchange(dist, n, world))
        for d in (0, 1):
            for j in range(world):
                for a, b_ in zip(sr.tile(d, rank, j), full.tile(d, rank, j)):
                    assert np.array_equal(a, b_)
        xs, ls, _, _ = sr.rows_export(5)
        xf, lf, _, _ = full.rows_export(5)
        q0, q1 = int(full.bounds[rank]), int(full.bounds[rank + 1])
        assert sr.rows_info() == (q0, q1 - q0)
        assert np.array_equal(xs, xf[q0:q1]) and np.array_equal(ls, lf[q0:q1])
        b = mine.bounds
        r0, r1 = int(b[rank]), int(b[rank + 1])
        # 3. staged SpMM over torch.distributed broadcasts: out_i = sum_j tile(i, j) H^j, stages in order
        rng = np.random.default_rng(7)
        H = rng.uniform(-1, 1, (n, w)).astype(np.float32)  # same on every rank; each owns rows [r0, r1)
        h_local = H[r0:r1].copy()
        out = np.zeros((r1 - r0, w), np.float32)
        for j in range(world):
            rows_j = int(b[j + 1] - b[j])
            buf = torch.from_numpy(h_local.copy()) if j == rank else torch.zeros(rows_j, w)
            dist.broadcast(buf, src=j)
            rp, ci, v = mine.tile(0, rank, j)
            out = port32.spmm(r1 - r0, rows_j, rp, ci, v, buf.numpy(), accumulate=j > 0, out=out)
        gathered = [torch.zeros(int(b[i + 1] - b[i]), w) for i in range(world)]
        dist.all_gather(gathered, torch.from_numpy(out))
        staged = torch.cat(gathered).numpy()
        # monolithic reference: the P=1 partition's single tile
        mono_prep = R.prepare_data(ds, cfg, 1)
        rp, ci, v = mono_prep.tile(0, 0, 0)
        mono = port32.spmm(n, n, rp, ci, v, H)
        assert np.array_equal(staged.view(np.uint32), mono.view(np.uint32))
        # 4. canonical 8-block W-grad staging + rank-order all-reduce == single worker, bitwise
        X = rng.uniform(-1, 1, (n, 5)).astype(np.float32)
        G = rng.uniform(-1, 1, (n, w)).astype(np.float32)
        wb = [i * n // 8 for i in range(9)]
        stage = np.zeros((8, 5, w), np.float32)
        for g in range(8):
            a, e = max(wb[g], r0), min(wb[g + 1], r1)
            if a < e:
                stage[g] = port32.gemm(X[a:e], G[a:e], ta=True)
        t = torch.from_numpy(stage)
        dist.all_reduce(t)  # one nonzero contributor per block: x + 0 is exact in any order
        wg = np.zeros((5, w), np.float32)
        for g in range(8):
            wg = (wg + t.numpy()[g]).astype(np.float32)
        ref_stage = [port32.gemm(X[wb[g]:wb[g + 1]], G[wb[g]:wb[g + 1]], ta=True) for g in range(8)]
        ref = np.zeros((5, w), np.float32)
        for g in range(8):
            ref = (ref + ref_stage[g]).astype(np.float32)
        assert np.array_equal(wg.view(np.uint32), ref.view(np.uint32))
        q.put((rank, "ok"))
    except Exception as ex:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_world_size_2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(60)
    assert results == {0: "ok", 1: "ok"}, results


def test_cpp_dropin_header_compiles(tmp_path):
    """The C++ drop-in (include/mggcn/rowgcn.hpp) compiles and links against libmggcn.so."""
    import subprocess
    exe = tmp_path / "train_products"
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "examples", "train_products.cpp"), "-L",
                        os.path.join(ROOT, "paper_2110_08688_b200"), "-lmggcn", "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
