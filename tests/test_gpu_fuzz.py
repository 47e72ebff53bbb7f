"""Randomised small bulks through every strategy (including the relaxed ones, the pool and
run_bulks), each compared with the oracle element by element: ragged sizes (0, 1, odd,
a few tiles), extreme skew, tiny databases where nearly every pair of transactions
conflicts, both conflict rules.  Seeds are fixed: a failure is reproducible."""
import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import compare, gpu_db

pytestmark = pytest.mark.gpu

STRATS = ["kset", "part", "tpl", "auto"]


def _cases():
    rng = np.random.default_rng(2024)
    for k in range(24):
        schema = [W.TPCB, W.TM1, W.TPCC, W.MICRO][k % 4]
        n = int(rng.choice([0, 1, 2, 7, 33, 257, 1025, 5000]))
        seed = int(rng.integers(1, 1 << 30))
        add = bool(k % 3 == 0) and schema in (W.TPCB, W.TPCC)
        yield pytest.param(schema, n, seed, add, id=f"s{schema}-n{n}-seed{seed % 1000}-add{int(add)}")


def _make(schema, n, seed):
    rng = np.random.default_rng(seed)
    if schema == W.TPCB:
        dims = W.TpcbDims(int(rng.integers(1, 6)), int(rng.integers(1, 4)), int(rng.integers(2, 50)))
        kw = dict(remote_pct=float(rng.choice([0.0, 30.0])), alpha=float(rng.choice([0.0, 0.5])),
                  withdraw_pct=float(rng.choice([0.0, 40.0])))
    elif schema == W.TM1:
        dims = W.Tm1Dims(int(rng.integers(1, 40)))
        kw = dict(dist=str(rng.choice(["uniform", "nurand"])))
    elif schema == W.TPCC:
        dims = W.TpccDims(int(rng.integers(1, 4)), int(rng.integers(1, 4)), int(rng.integers(3, 20)),
                          int(rng.integers(5, 60)))
        kw = dict(remote_line_pct=float(rng.choice([0.0, 20.0])), remote_pay_pct=float(rng.choice([0.0, 40.0])),
                  rbk_pct=float(rng.choice([0.0, 10.0])))
    else:
        dims = W.MicroDims(int(rng.integers(1, 100)), int(rng.integers(1, 33)), int(rng.integers(0, 3)))
        kw = dict(alpha=float(rng.choice([0.0, 0.3])))
    image = W.make_db(schema, dims, seed=seed % 97)
    bulk = W.make_bulk(schema, dims, n, seed, **kw)
    return dims, image, bulk


@pytest.mark.parametrize("schema,n,seed,add", list(_cases()))
def test_fuzz_all_strategies(schema, n, seed, add):
    dims, image, bulk = _make(schema, n, seed)
    ref = oracle.run(schema, dims.dims, image, bulk)
    db = gpu_db(schema, dims, image, max(1, n), add_rule=add, insert_capacity=16)
    try:
        for s in STRATS:
            db.reset()
            db.submit(bulk)
            db.execute(s)
            compare(schema, ref, db, image, label=f"{s}")
        for s in ("tpl_relaxed", "part_relaxed"):
            db.reset()
            db.submit(bulk)
            db.execute(s)
            rr = oracle.run(schema, dims.dims, image, bulk, order=db.serial_order())
            st, out = db.read_results()
            assert np.array_equal(st, rr.status) and np.array_equal(out, rr.out), s
            got = db.read_image(image)
            for c in image:
                assert np.array_equal(got[c], rr.db[c]), (s, c)
        # the pool, in two chunks, drained
        db.reset()
        half = n // 2
        st = np.full(n, 255, np.uint8)
        for a, b in ((0, half), (half, n)):
            db.pool_submit(bulk.slice(a, b))
            db.pool_step()
            ts, s_, _ = db.pool_read()
            st[ts] = s_
        while db.pool_pending():
            db.pool_step()
            ts, s_, _ = db.pool_read()
            st[ts] = s_
        assert np.array_equal(st, ref.status)
        got = db.read_image(image)
        for c in image:
            assert np.array_equal(got[c], ref.db[c]), ("pool", c)
    finally:
        db.close()
