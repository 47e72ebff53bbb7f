"""Parity at BASELINE.json's full sizes, in the configuration bench.py times
(same generators, same library defaults), bit-exact against the oracle for every
strategy: config 2 (TM-1, 1M subscribers, bulk 1M), config 3 (TPC-B, 1,000
branches, bulk 4M, uniform and hot-branch), config 4 (TPC-C NO+Payment, 64
warehouses, bulk 1M)."""
import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import compare, gpu_db

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CASES = {
    "tm1_nurand": (W.TM1, W.Tm1Dims(1_000_000), 1_000_000, dict(dist="nurand")),
    "tpcb_uniform": (W.TPCB, W.TpcbDims(1000, 10, 100_000), 4_000_000, dict(remote_pct=15.0)),
    "tpcb_hot": (W.TPCB, W.TpcbDims(1000, 10, 100_000), 1_000_000, dict(remote_pct=15.0, alpha=0.1)),
    "tpcc": (W.TPCC, W.TpccDims(64, 10, 3000, 100_000), 1_000_000, {}),
    # NEXT-1 (ADD conflict rule): the bench's *_add workloads
    "tpcb_hot_add": (W.TPCB, W.TpcbDims(1000, 10, 100_000), 4_000_000, dict(remote_pct=15.0, alpha=0.1)),
    "tpcc_add": (W.TPCC, W.TpccDims(64, 10, 3000, 100_000), 1_000_000, {}),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_full_size_all_strategies(case):
    schema, dims, n, kw = CASES[case]
    add_rule = case.endswith("_add")
    image = W.make_db(schema, dims, seed=1)
    bulk = W.make_bulk(schema, dims, n, seed=2, **kw)
    ref = oracle.run(schema, dims.dims, image, bulk)
    depth = None
    for strategy in ("kset", "part", "tpl"):
        db = gpu_db(schema, dims, image, n, insert_capacity=2, add_rule=add_rule)
        db.submit(bulk)
        st = db.execute(strategy)
        compare(schema, ref, db, image, label=f"{case} {strategy}")
        if strategy == "kset":
            depth = db.depths()
            assert st["depth"] == int(depth.max())
        db.close()
    # rank fixpoint = T-dependency-graph depth of every transaction
    assert np.array_equal(depth, oracle.depths(schema, dims.dims, image, bulk, add_rule=add_rule))
