"""GPU parity for the micro benchmark (§6.1): bit-exact float results of the
T-branch procedure under every strategy, with and without type grouping,
with lock skew alpha (deep T-dependency graphs)."""
import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import compare, gpu_db, run_both

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("strategy", ["kset", "part", "tpl"])
@pytest.mark.parametrize("T,x,alpha", [(8, 1, 0.0), (32, 2, 0.05), (1, 0, 0.5), (16, 1, 0.0)])
def test_micro_parity(strategy, T, x, alpha):
    d = W.MicroDims(20_000, T, x)
    image = W.micro_db(d, seed=1)
    bulks = [W.micro_bulk(d, 9000, seed=s, alpha=alpha) for s in (2, 3)]
    run_both(W.MICRO, d, image, bulks, strategy)


@pytest.mark.parametrize("p", [1, 2, 4, 16])
def test_micro_grouping_keeps_results(p):
    """Type grouping changes the execution order inside a k-set only."""
    d = W.MicroDims(5000, 16, 1)
    image = W.micro_db(d, seed=1)
    bulk = W.micro_bulk(d, 8000, seed=4, alpha=0.01)
    ref = oracle.run(W.MICRO, d.dims, image, bulk)
    db = gpu_db(W.MICRO, d, image, bulk.n)
    db.set_grouping(p)
    db.submit(bulk)
    db.execute("kset")
    compare(W.MICRO, ref, db, image, label=f"p={p}")
    # within each k-set the order is by (type group), stable by ts
    dep = db.depths()
    perm = db.perm()
    key = dep[perm].astype(np.int64) * 16 + (bulk.type[perm].astype(np.int64) * p) // 16
    assert (np.diff(key) >= 0).all()
    db.close()


def test_micro_rejects_bad_params():
    from paper_1103_3105_b200.gputx import GputxError
    d = W.MicroDims(100, 4, 1)
    db = gpu_db(W.MICRO, d, W.micro_db(d), 10)
    bad = W.micro_bulk(d, 10, seed=1)
    bad.param_words[3] = 100                      # tuple out of range
    with pytest.raises(GputxError):
        db.submit(bad)
    bad2 = W.micro_bulk(d, 10, seed=1)
    bad2.type[2] = 4                              # type >= T
    with pytest.raises(GputxError):
        db.submit(bad2)
    with pytest.raises(GputxError):
        db.set_grouping(5)
    db.close()
