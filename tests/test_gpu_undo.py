"""Undo-log recovery for a non-two-phase type:
TPC-B WITHDRAW debits account, teller and branch and aborts AFTERWARDS if the account went
negative, rolling its updates back from its undo log.  Every strategy must still give the
serial result (ts order; the relaxed ones: their witnessed order), including under the
ADD rule where the teller/branch rollback is a compensating increment."""
import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import gpu_db, run_both

pytestmark = pytest.mark.gpu

DIMS = W.TpcbDims(8, 10, 200)


@pytest.mark.parametrize("add_rule", [False, True])
@pytest.mark.parametrize("strategy", ["kset", "part", "tpl", "auto"])
def test_withdraw_rollback_parity(strategy, add_rule):
    image = W.tpcb_db(DIMS)
    bulks = [W.tpcb_bulk(DIMS, 9000, seed=s, remote_pct=15.0, withdraw_pct=40.0) for s in (1, 2)]
    db = gpu_db(W.TPCB, DIMS, image, 9000, add_rule=add_rule)
    stats = run_both(W.TPCB, DIMS, image, bulks, strategy, db=db)
    assert all(s["aborted"] > 500 for s in stats)            # rollbacks really happened
    db.close()


@pytest.mark.parametrize("strategy", ["tpl_relaxed", "part_relaxed"])
def test_withdraw_relaxed_witness(strategy):
    image = W.tpcb_db(DIMS)
    bulk = W.tpcb_bulk(DIMS, 9000, seed=3, remote_pct=15.0, withdraw_pct=40.0)
    db = gpu_db(W.TPCB, DIMS, image, bulk.n)
    db.submit(bulk)
    db.execute(strategy)
    ref = oracle.run(W.TPCB, DIMS.dims, image, bulk, order=db.serial_order())
    st, out = db.read_results()
    assert np.array_equal(st, ref.status) and np.array_equal(out, ref.out)
    got = db.read_image(image)
    for k in image:
        assert np.array_equal(got[k], ref.db[k]), k
    db.close()


def test_withdraw_in_the_pool():
    image = W.tpcb_db(DIMS)
    bulk = W.tpcb_bulk(DIMS, 6000, seed=4, remote_pct=15.0, withdraw_pct=40.0)
    ref = oracle.run(W.TPCB, DIMS.dims, image, bulk)
    db = gpu_db(W.TPCB, DIMS, image, bulk.n)
    st = np.full(bulk.n, 255, np.uint8)
    for a in range(0, bulk.n, 1500):
        db.pool_submit(bulk.slice(a, a + 1500))
        db.pool_step()
        ts, s, _ = db.pool_read()
        st[ts] = s
    while db.pool_pending():
        db.pool_step()
        ts, s, _ = db.pool_read()
        st[ts] = s
    assert np.array_equal(st, ref.status)
    got = db.read_image(image)
    for k in image:
        assert np.array_equal(got[k], ref.db[k]), k
    db.close()


def test_withdraw_must_be_local():
    from paper_1103_3105_b200.gputx import GputxError
    image = W.tpcb_db(DIMS)
    bulk = W.tpcb_bulk(DIMS, 50, seed=5, withdraw_pct=100.0)
    bulk.param_words[0] = (bulk.param_words[2] + 1) % DIMS.branches * DIMS.accounts_per_branch   # remote account
    db = gpu_db(W.TPCB, DIMS, image, 50)
    with pytest.raises(GputxError):
        db.submit(bulk)
    db.close()
