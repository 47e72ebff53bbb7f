"""Spine-streaming rank: the depth of every transaction -- its k-set, the
longest path to it in the T-dependency graph -- must equal the oracle's
on bulks built to stress the chain walk: tiny dimensions (nearly every transaction has
cross-chain predecessors, read runs on customers before a Payment's write), hot branches
(one long chain), micro skew (one tuple's chain holds a tenth of the bulk), and the
iterative rank it replaced must give the same depths."""
import os

import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import compare, gpu_db

pytestmark = pytest.mark.gpu

CASES = {
    "tpcc_tiny": (W.TPCC, W.TpccDims(3, 2, 30, 40), 6000,
                  dict(remote_line_pct=30.0, remote_pay_pct=40.0, rbk_pct=10.0)),
    "tpcc_std": (W.TPCC, W.TpccDims(4, 10, 3000, 5000), 20_000, {}),
    "tpcb_remote": (W.TPCB, W.TpcbDims(8, 10, 50), 20_000, dict(remote_pct=60.0)),
    "tpcb_hot": (W.TPCB, W.TpcbDims(16, 10, 2000), 20_000, dict(remote_pct=15.0, alpha=0.5)),
    "tpcb_withdraw": (W.TPCB, W.TpcbDims(8, 10, 100), 20_000, dict(withdraw_pct=30.0)),
    "micro_skew": (W.MICRO, W.MicroDims(5000, 8, 0), 30_000, dict(alpha=0.1)),
}


def _db(schema, dims, image, n, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return gpu_db(schema, dims, image, n)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("case", list(CASES))
def test_spine_depths_and_results(case):
    schema, dims, n, kw = CASES[case]
    image = W.make_db(schema, dims, seed=1)
    bulk = W.make_bulk(schema, dims, n, seed=3, **kw)
    ref_d = oracle.depths(schema, dims.dims, image, bulk)
    ref = oracle.run(schema, dims.dims, image, bulk)
    for env in ({}, {"GPUTX_RANK_SPINE": "0"}):
        db = _db(schema, dims, image, n, env)
        try:
            db.submit(bulk)
            st = db.execute("kset")
            d = db.depths()
            assert np.array_equal(d, ref_d), f"{case} {env}: depths differ at {np.nonzero(d != ref_d)[0][:10]}"
            assert st["depth"] == ref_d.max() and st["zero_set"] == int((ref_d == 0).sum())
            compare(schema, ref, db, image, label=f"{case} {env}")
        finally:
            db.close()
