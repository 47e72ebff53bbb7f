"""Streaming K-SET over a live pool:
arrivals submitted in chunks, one 0-set executed per step, the rest kept with their
original timestamps.  After the pool drains, the database, every transaction's (status,
output) and the insert tables (as row sets) equal the oracle's serial run of all
arrivals in ts order (Definition 1)."""
import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import gpu_db

pytestmark = pytest.mark.gpu

CASES = {
    "tm1": (W.TM1, W.Tm1Dims(2000), dict(dist="nurand")),
    "tpcb": (W.TPCB, W.TpcbDims(8, 10, 1000), dict(remote_pct=15.0)),
    "tpcb_hot": (W.TPCB, W.TpcbDims(8, 10, 1000), dict(remote_pct=15.0, alpha=0.3)),
    "tpcc": (W.TPCC, W.TpccDims(2, 10, 300, 2000), {}),
    "micro": (W.MICRO, W.MicroDims(3000, 8, 1), dict(alpha=0.05)),
}


def _rows(tab):
    cols = sorted(tab)
    return sorted(zip(*[np.asarray(tab[c]).tolist() for c in cols])) if cols else []


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("steps_per_chunk", [1, 3])
def test_pool_streaming_equals_serial(case, steps_per_chunk):
    schema, dims, kw = CASES[case]
    image = W.make_db(schema, dims, seed=1)
    bulk = W.make_bulk(schema, dims, 6000, seed=2, **kw)
    ref = oracle.run(schema, dims.dims, image, bulk)
    add_rule = False
    db = gpu_db(schema, dims, image, bulk.n, insert_capacity=2)
    n = bulk.n
    st = np.full(n, 255, np.uint8)
    out = np.zeros((n, ref.out.shape[1]), np.uint8)
    done = np.zeros(n, np.int64)
    chunks = np.linspace(0, n, 9).astype(int)
    steps = 0
    for a, b in zip(chunks[:-1], chunks[1:]):
        first = db.pool_submit(bulk.slice(int(a), int(b)))
        assert first == a
        for _ in range(steps_per_chunk):
            s = db.pool_step()
            steps += 1
            ts, s_st, s_out = db.pool_read()
            assert len(ts) == s["executed"] == s["n"]
            assert np.all(np.diff(ts.astype(np.int64)) > 0)           # ts order within a step
            st[ts] = s_st
            out[ts] = s_out
            done[ts] += 1
    while db.pool_pending():
        s = db.pool_step()
        steps += 1
        assert s["executed"] > 0                                       # progress every step
        ts, s_st, s_out = db.pool_read()
        st[ts] = s_st
        out[ts] = s_out
        done[ts] += 1
    assert (done == 1).all()
    assert np.array_equal(st, ref.status)
    assert np.array_equal(out, ref.out)
    got = db.read_image(image)
    for k in image:
        assert np.array_equal(got[k], ref.db[k]), k
    ins = db.inserts()
    for tab, cols in ref.inserts.items():
        assert _rows(ins[tab]) == _rows(cols), tab
    if case in ("tpcb_hot", "micro"):
        assert steps > 10                       # deep chains stay in the pool across steps
    db.close()


def test_pool_zero_set_is_the_depth_zero_set():
    """The first step executes exactly the transactions of depth 0."""
    schema, dims, kw = CASES["tpcb_hot"]
    image = W.make_db(schema, dims, seed=1)
    bulk = W.make_bulk(schema, dims, 4000, seed=3, **kw)
    dep = oracle.depths(schema, dims.dims, image, bulk)
    db = gpu_db(schema, dims, image, bulk.n)
    db.pool_submit(bulk)
    db.pool_step()
    ts, _, _ = db.pool_read()
    assert np.array_equal(np.sort(ts), np.flatnonzero(dep == 0))
    assert db.pool_pending() == bulk.n - int((dep == 0).sum())
    db.close()


def test_pool_rejects_and_blocks_bulk_api():
    from paper_1103_3105_b200.gputx import GputxError
    schema, dims, kw = CASES["tpcb"]
    image = W.make_db(schema, dims, seed=1)
    bulk = W.make_bulk(schema, dims, 100, seed=3, **kw)
    db = gpu_db(schema, dims, image, 150)
    db.pool_submit(bulk)
    with pytest.raises(GputxError):
        db.submit(bulk)                                # pool not empty
    with pytest.raises(GputxError):
        db.pool_submit(bulk)                           # 200 > max_bulk 150
    bad = W.make_bulk(schema, dims, 10, seed=4, **kw)
    bad.param_words[0] = 10 ** 9
    with pytest.raises(GputxError):
        db.pool_submit(bad)
    assert db.pool_pending() == 100
    db.reset()
    assert db.pool_pending() == 0
    db.submit(bulk)
    db.execute("kset")
    db.close()
