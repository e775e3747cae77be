"""CPU half of the full-size parity pins (tests/test_gpu_scale.py has the rest): the host generator and
host partitioner of libmggcn at the full C2 arxiv shape (169,343 vertices, 2.3 M edges) are bit-identical to
the compiled reference's synth_graph + prepare_data at P = 1 and P = 2 (tests/golden/scale_partition.json)."""
import json
import os

import pytest

from scale_common import SCALE, dataset_digest
from test_gpu_scale import check_partition

from paper_2110_08688_b200 import rowgcn as R

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "scale_partition.json")


@pytest.mark.parametrize("P", [1, 2])
def test_c2_partition_bit_identical(P):
    gold = json.load(open(GOLD))["c2"]
    c = SCALE["c2"]
    ds = R.synth_graph(c["n"], c["deg"], 0.7, 1, c["dims"][0], c["dims"][-1])
    rp, ci, v = ds.graph
    assert dataset_digest(rp, ci, v, ds.features, ds.labels) == gold["dataset"]
    check_partition(R.prepare_data(ds, R.GcnConfig(c["dims"], seed=1, permute=True, overlap=P > 1), P), ds, gold, P)
