"""The per-rank synthetic input path (mg_synth_rank_*, mggcn.h): one rank of a P-way
job builds its row block of prepare_data(synth_graph(...)) (inc/dataset.hpp:287-334, inc/driver.hpp:87-117)
from the generator's stream, without the whole graph or all features.

* against the compiled reference (tests/golden/scale_ranks.json, tests/golden/make_scale_golden.py ranks):
  the papers-shaped graph at 1/64 scale (1.74 M vertices, 50 M directed edges, [128,128,128,172]) at
  P = 8, every rank: its features / labels / mask rows and its forward and backward tiles are
  bit-identical (sha256) to the reference's whole-graph partition cut at that rank; both degree sources
  (exchanged, and derived locally by block passes) are exercised;
* against the host partitioner (itself pinned to the reference) on small graphs, permute on/off, P up to
  8 and P > n, plus the error paths.
"""
import json
import os

import numpy as np
import pytest

from scale_common import RANK_CASES, SCALE, sha, tile_digest

from paper_2110_08688_b200 import rowgcn as R

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "scale_ranks.json")


@pytest.mark.parametrize("name,P", RANK_CASES)
def test_ranks_bit_identical_to_reference(name, P):
    gold = json.load(open(GOLD))[f"{name}:{P}"]
    c = SCALE[name]
    dims, n = c["dims"], c["n"]
    cfg = R.GcnConfig(dims, seed=1, permute=True, overlap=True)
    handles = [R.SynthRank(n, c["deg"], 0.7, 1, dims[0], dims[-1], cfg, P, r) for r in range(P)]
    all_deg = np.concatenate([h.degrees() for h in handles])  # what the all-gather of a P-process job delivers
    assert sum(h.nnz for h in handles) == gold["nnz"]
    for r, h in enumerate(handles):
        g = gold["ranks"][str(r)]
        # rank 0 derives the degrees itself (P block passes), the others take the exchanged ones
        prep = h.finish(None if r == 0 else all_deg)
        assert [int(b) for b in prep.bounds] == gold["bounds"] and prep.mask_count == gold["mask_count"]
        x, lab, m, pf = prep.rows_export(dims[0])
        assert prep.rows_info() == (gold["bounds"][r], gold["bounds"][r + 1] - gold["bounds"][r])
        assert sha(pf) == gold["perm_forward"]
        assert sha(x) == g["features"] and sha(lab) == g["labels"] and sha(m) == g["mask"], r
        for d in (0, 1):
            for j in range(P):
                assert tile_digest(*prep.tile(d, r, j)) == g["tiles"][f"{d},{j}"], (r, d, j)
        handles[r] = None


def _same_block(prep, full, r, d0):
    for d in (0, 1):
        for j in range(full.workers):
            for a, b in zip(prep.tile(d, r, j), full.tile(d, r, j)):
                assert a.dtype == b.dtype and np.array_equal(a, b), (d, r, j)
    x, lab, m, pf = prep.rows_export(d0)
    xf, lf, mf, pff = full.rows_export(d0)
    r0, r1 = int(full.bounds[r]), int(full.bounds[r + 1])
    assert np.array_equal(pf, pff)
    assert np.array_equal(x.view(np.uint32), xf[r0:r1].view(np.uint32))
    assert np.array_equal(lab, lf[r0:r1]) and np.array_equal(m, mf[r0:r1])
    assert prep.mask_count == full.mask_count


@pytest.mark.parametrize("n,deg,d0,C,P,permute", [(300, 8.0, 7, 3, 1, True), (300, 8.0, 7, 3, 3, True),
                                                  (1000, 20.0, 5, 4, 4, False), (4000, 12.0, 9, 5, 8, True),
                                                  (7, 2.0, 3, 2, 8, True)])
def test_ranks_match_host_partitioner(n, deg, d0, C, P, permute):
    cfg = R.GcnConfig([d0, 16, C], seed=3, permute=permute)
    full = R.prepare_data(R.synth_graph(n, deg, 0.7, 5, d0, C), cfg, P)
    hs = [R.SynthRank(n, deg, 0.7, 5, d0, C, cfg, P, r) for r in range(P)]
    all_deg = np.concatenate([h.degrees() for h in hs])
    for r in range(P):
        assert np.array_equal(hs[r].block_degrees((r + 1) % P), all_deg[full.bounds[(r + 1) % P]:full.bounds[(r + 1) % P + 1]])
        _same_block(hs[r].finish(all_deg if r % 2 else None), full, r, d0)


def test_errors():
    cfg = R.GcnConfig([4, 8, 3], seed=1, permute=True)
    with pytest.raises(R.ValueError, match="need n >= 2"):
        R.SynthRank(1, 1.0, 0.7, 1, 4, 3, cfg, 2, 0)
    with pytest.raises(R.ValueError, match="out of range"):
        R.SynthRank(100, 4.0, 0.7, 1, 4, 3, cfg, 2, 2)
    with pytest.raises(R.ConfigError, match="layer_dims"):
        R.SynthRank(100, 4.0, 0.7, 1, 5, 3, cfg, 2, 0)
    h = R.SynthRank(100, 4.0, 0.7, 1, 4, 3, cfg, 2, 0)
    bad = np.zeros(100, np.int32)
    with pytest.raises(R.ValueError, match="exchanged degrees"):
        h.finish(bad)
    h.finish(None)
    with pytest.raises(R.ValueError, match="already finished"):
        h.finish(None)
    g = R.SynthRank(100, 4.0, 0.7, 1, 4, 3, cfg, 2, 1, graph_only=True)
    assert g.degrees().shape == (50,)
    with pytest.raises(R.ValueError, match="GRAPH_ONLY"):
        g.finish(None)
