"""GPU parity: the CUDA path through the C ABI vs the oracle (Definition 1,
PAPER.md:73), bit-exact on final database, statuses, outputs and inserted rows,
for TPL / PART / K-SET on TPC-B, TM-1 and TPC-C."""
import os

import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import compare, gpu_db, run_both

pytestmark = pytest.mark.gpu

STRATS = ["kset", "part", "tpl"]


@pytest.mark.parametrize("strategy", STRATS)
def test_tpcb_tiny_config1(strategy):
    """BASELINE config 1: 1 branch, 10 tellers, 100k accounts, 4,096 deposits."""
    dims = W.TpcbDims(1, 10, 100_000)
    image = W.tpcb_db(dims)
    bulk = W.tpcb_bulk(dims, 4096, seed=1)
    db = gpu_db(W.TPCB, dims, image, 4096)
    st = run_both(W.TPCB, dims, image, [bulk], strategy, db=db)[0]
    if strategy == "kset":
        assert np.array_equal(db.depths(), np.arange(4096))       # one path: depth(t) = t
        assert st["depth"] == 4095 and st["zero_set"] == 1
    db.close()


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("n", [1, 37, 9000])
def test_tpcb_multibranch(strategy, n):
    dims = W.TpcbDims(16, 10, 2000)
    image = W.tpcb_db(dims)
    run_both(W.TPCB, dims, image, [W.tpcb_bulk(dims, n, seed=n, remote_pct=15.0)], strategy)


@pytest.mark.parametrize("add_rule", [False, True])
@pytest.mark.parametrize("strategy", STRATS)
def test_tpcb_hot_branch(strategy, add_rule):
    """Hot-branch skew: branch 0 holds half the bulk, far more records
    than one warp's share, so the root-local rank falls back to the grid-wide scan
    (kernels.cuh RR_SPLIT); depths and state must still equal the oracle's."""
    dims = W.TpcbDims(16, 10, 2000)
    image = W.tpcb_db(dims)
    bulk = W.tpcb_bulk(dims, 9000, seed=4, remote_pct=15.0, alpha=0.5)
    db = gpu_db(W.TPCB, dims, image, bulk.n, add_rule=add_rule)
    run_both(W.TPCB, dims, image, [bulk], strategy, db=db)
    if strategy == "kset":
        assert np.array_equal(db.depths(), oracle.depths(W.TPCB, dims.dims, image, bulk, add_rule=add_rule))
    db.close()


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("dist", ["nurand", "uniform"])
def test_tm1(strategy, dist):
    dims = W.Tm1Dims(20_000)
    image = W.tm1_db(dims, seed=3)
    bulks = [W.tm1_bulk(dims, 30_011, seed=5, dist=dist), W.tm1_bulk(dims, 7_000, seed=6, dist=dist)]
    run_both(W.TM1, dims, image, bulks, strategy, max_bulk=40_000)


@pytest.mark.parametrize("strategy", STRATS)
def test_tpcc(strategy):
    dims = W.TpccDims(4, 10, 3000, 100_000)
    image = W.tpcc_db(dims, seed=2)
    bulks = [W.tpcc_bulk(dims, 12_345, seed=7), W.tpcc_bulk(dims, 3_000, seed=8)]
    run_both(W.TPCC, dims, image, bulks, strategy, max_bulk=20_000)


@pytest.mark.parametrize("strategy", STRATS)
def test_tpcc_tiny_contention(strategy):
    """Tiny dimensions: many remote lines/customers, duplicate items, by-name, aborts."""
    dims = W.TpccDims(3, 2, 30, 40)
    image = W.tpcc_db(dims, seed=4)
    bulk = W.tpcc_bulk(dims, 5000, seed=9, remote_line_pct=30.0, remote_pay_pct=40.0, rbk_pct=10.0)
    run_both(W.TPCC, dims, image, [bulk], strategy)


@pytest.mark.parametrize("schema,dims,kw", [
    (W.TPCB, W.TpcbDims(8, 10, 1000), dict(remote_pct=15.0)),
    (W.TM1, W.Tm1Dims(5000), dict(dist="nurand")),
    (W.TPCC, W.TpccDims(2, 10, 3000, 1000), {}),
])
def test_kset_depths_match_oracle(schema, dims, kw):
    """A5: the rank fixpoint equals the T-dependency-graph depth."""
    image = W.make_db(schema, dims, seed=3)
    bulk = W.make_bulk(schema, dims, 20_000, 11, **kw)
    db = gpu_db(schema, dims, image, bulk.n)
    db.submit(bulk)
    st = db.execute("kset")
    d = db.depths()
    ref = oracle.depths(schema, dims.dims, image, bulk)
    assert np.array_equal(d, ref)
    assert st["depth"] == ref.max() and st["zero_set"] == int((ref == 0).sum())
    # A6: perm is a permutation ordered by (depth, type)
    perm = db.perm()
    assert np.array_equal(np.sort(perm), np.arange(bulk.n))
    key = ref[perm].astype(np.int64) * 8 + bulk.type[perm]
    assert (np.diff(key) >= 0).all()
    db.close()


@pytest.mark.parametrize("strategy", STRATS)
def test_grid_shape_independence(strategy):
    dims = W.Tm1Dims(3000)
    image = W.tm1_db(dims, seed=1)
    bulk = W.tm1_bulk(dims, 20_000, seed=2)
    ref = oracle.run(W.TM1, dims.dims, image, bulk)
    for grid, cluster in [(1, "0"), (7, "0"), (8, "8"), (16, "8"), (0, "8"), (0, "16")]:
        os.environ["GPUTX_KSET_CLUSTER"] = cluster
        try:
            db = gpu_db(W.TM1, dims, image, bulk.n)
        finally:
            os.environ.pop("GPUTX_KSET_CLUSTER", None)
        db.set_launch(exec_grid=grid)
        db.submit(bulk)
        db.execute(strategy)
        compare(W.TM1, ref, db, image, label=f"grid {grid} cluster {cluster}")
        db.close()


def test_empty_bulk():
    dims = W.TpcbDims(2, 10, 100)
    image = W.tpcb_db(dims)
    db = gpu_db(W.TPCB, dims, image, 16)
    empty = W.tpcb_bulk(dims, 0, seed=1)
    for s in STRATS:
        db.submit(empty)
        st = db.execute(s)
        assert st["n"] == 0
    db.close()


def test_errors():
    from paper_1103_3105_b200 import GputxError
    dims = W.Tm1Dims(100)
    image = W.tm1_db(dims, seed=1)
    db = gpu_db(W.TM1, dims, image, 64)
    with pytest.raises(GputxError) as e:
        db.register_types([0, 1, 1])
    assert e.value.name == "EDUP_TYPE"
    with pytest.raises(GputxError) as e:
        db.register_types([9])
    assert e.value.name == "EUNKNOWN_TYPE"
    db.register_types([0, 4])                        # GSD and UL only
    b = W.tm1_bulk(dims, 20, seed=1)                 # contains other types
    with pytest.raises(GputxError) as e:
        db.submit(b)
    assert e.value.name == "EUNKNOWN_TYPE"
    db.register_types(list(range(7)))
    with pytest.raises(GputxError) as e:
        db.submit(W.tm1_bulk(dims, 65, seed=1))
    assert e.value.name == "ECAPACITY"
    bad = W.tm1_bulk(dims, 10, seed=1)
    bad.param_words = bad.param_words.copy()
    i = int(np.nonzero(bad.type == W.TM1_GSD)[0][0])
    bad.param_words[bad.param_off[i]] = 10_000        # s_id out of range
    with pytest.raises(GputxError) as e:
        db.submit(bad)
    assert e.value.name == "EINVAL"
    with pytest.raises(GputxError) as e:
        db.execute("kset")
    assert e.value.name == "ESTATE"
    db.submit(W.tm1_bulk(dims, 10, seed=2))
    with pytest.raises(GputxError) as e:
        db.submit(W.tm1_bulk(dims, 10, seed=3))
    assert e.value.name == "ESTATE"
    db.execute("tpl")
    db.close()


def test_reset_restores_pristine():
    dims = W.TpcbDims(4, 10, 1000)
    image = W.tpcb_db(dims)
    db = gpu_db(W.TPCB, dims, image, 5000)
    db.submit(W.tpcb_bulk(dims, 5000, seed=1))
    db.execute("kset")
    db.reset()
    got = db.read_image(image)
    for k in image:
        assert np.array_equal(got[k], image[k])
    assert db.inserts()["history"]["h_ts"].size == 0
    run_both(W.TPCB, dims, image, [W.tpcb_bulk(dims, 5000, seed=1)], "part", db=db)
    db.close()


TS_COLUMNS = {"h_ts", "o_entry_d", "h_date"}     # insert columns that hold the transaction's ts


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("schema", [W.TPCB, W.TPCC])
def test_explicit_timestamps(strategy, schema):
    """gputx_bulk.ts (caller-given global timestamps): same execution order as
    position order, and the ts-valued insert columns carry the given timestamps."""
    if schema == W.TPCB:
        dims = W.TpcbDims(8, 10, 500)
        bulk = W.tpcb_bulk(dims, 5000, seed=21, remote_pct=20.0)
    else:
        dims = W.TpccDims(4, 10, 300, 2000)
        bulk = W.tpcc_bulk(dims, 4000, seed=22, remote_line_pct=5.0)
    image = W.make_db(schema, dims, seed=5)
    ts = (np.arange(bulk.n, dtype=np.int64) * 7 + 1000).astype(np.uint32)
    ref = oracle.run(schema, dims.dims, image, bulk)
    for tab, cols in ref.inserts.items():
        for c in cols:
            if c in TS_COLUMNS:
                cols[c] = ts[cols[c].astype(np.int64)].astype(cols[c].dtype)
    db = gpu_db(schema, dims, image, bulk.n)
    try:
        db.submit(bulk, ts=ts)
        db.execute(strategy)
        compare(schema, ref, db, image, label=f"{strategy} explicit ts")
    finally:
        db.close()


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("schema", [W.TPCB, W.TPCC])
def test_add_rule_parity_and_depths(strategy, schema):
    """GPUTX_FLAG_ADD_RULE (PAPER.md:475(c)): increments of teller /
    branch balances and W_YTD / D_YTD do not conflict with each other.  The final state,
    outputs and inserts still equal serial execution; K-SET depths equal the oracle's
    ADD-rule recurrence and are much shallower than under the R/W rule."""
    if schema == W.TPCB:
        dims = W.TpcbDims(4, 10, 300)
        bulk = W.tpcb_bulk(dims, 20_000, seed=31, remote_pct=20.0)
    else:
        dims = W.TpccDims(4, 10, 300, 2000)
        bulk = W.tpcc_bulk(dims, 8000, seed=32, remote_line_pct=5.0)
    image = W.make_db(schema, dims, seed=6)
    ref = oracle.run(schema, dims.dims, image, bulk)
    db = gpu_db(schema, dims, image, bulk.n, add_rule=True)
    try:
        db.submit(bulk)
        st = db.execute(strategy)
        compare(schema, ref, db, image, label=f"{strategy} add rule")
        if strategy == "kset":
            want = oracle.depths(schema, dims.dims, image, bulk, add_rule=True)
            assert np.array_equal(db.depths(), want)
            assert st["depth"] < oracle.depths(schema, dims.dims, image, bulk).max()
    finally:
        db.close()


BIG = 1 << 62


@pytest.mark.parametrize("schema,dims,n,kw", [
    (W.TPCB, W.TpcbDims(16, 10, 2000), 9000, dict(remote_pct=15.0)),
    (W.TM1, W.Tm1Dims(20_000), 30_000, dict(dist="nurand")),
    (W.TPCC, W.TpccDims(4, 10, 3000, 100_000), 12_000, {}),
])
@pytest.mark.parametrize("want", ["kset", "part", "tpl"])
def test_auto_strategy_algorithm1(schema, dims, n, kw, want):
    """NEXT-3: GPUTX_AUTO computes w0, d, c equal to the oracle's and
    runs the strategy Algorithm 1 picks; thresholds are set so that
    each branch is taken, and the result is bit-exact against serial execution."""
    image = W.make_db(schema, dims, seed=3)
    bulk = W.make_bulk(schema, dims, n, 12, **kw)
    ref = oracle.structure(schema, dims.dims, image, bulk)
    if want == "kset":
        bars = (ref["w0"], BIG, 0)                 # w0 >= w0_bar
    elif want == "part":
        bars = (ref["w0"] + 1, BIG, ref["c"])      # c <= c_bar
    else:
        if ref["c"] == 0:
            pytest.skip("no cross-partition transaction (TM-1): Algorithm 1 never returns TPL")
        bars = (ref["w0"] + 1, ref["d"] + 1, ref["c"] - 1)
    assert oracle.choose_strategy(ref["w0"], ref["d"], ref["c"], *bars) == want
    db = gpu_db(schema, dims, image, n)
    db.set_chooser(*bars)
    st = run_both(schema, dims, image, [bulk], "auto", db=db)[0]
    assert st["strategy"] == want
    assert (st["zero_set"], st["depth"], st["cross"]) == (ref["w0"], ref["d"], ref["c"])
    db.close()


@pytest.mark.parametrize("add_rule", [False, True])
@pytest.mark.parametrize("wbits,n", [(8, 5_000), (10, 3 * 1024 + 1), (12, 4096), (13, 100)])
def test_tpcc_windowed_rank(monkeypatch, wbits, n, add_rule):
    """A5 windowed: windows of 2^wbits transactions,
    a ragged last window, a bulk that is exactly whole windows and one smaller than a
    window; depths equal the T-dependency-graph depths and the state
    equals serial execution, with and without the ADD rule."""
    monkeypatch.setenv("GPUTX_RANK_WINDOW", str(wbits))
    dims = W.TpccDims(3, 4, 300, 2_000)
    image = W.tpcc_db(dims, seed=5)
    bulk = W.tpcc_bulk(dims, n, seed=13, remote_line_pct=20.0, remote_pay_pct=30.0)
    db = gpu_db(W.TPCC, dims, image, n, add_rule=add_rule)
    run_both(W.TPCC, dims, image, [bulk], "kset", db=db)
    assert np.array_equal(db.depths(), oracle.depths(W.TPCC, dims.dims, image, bulk, add_rule=add_rule))
    db.close()


@pytest.mark.parametrize("runmax", [0, 1024])
def test_kset_round_runs(monkeypatch, runmax):
    """K-SET runs of one-CTA rounds (and, with GPUTX_KSET_RUNMAX, of narrow rounds up to
    1,024 transactions) inside CTA 0: deep TM-1 NURand tail and TPC-B with few branches."""
    monkeypatch.setenv("GPUTX_KSET_RUNMAX", str(runmax))
    for schema, dims, n, kw in [(W.TM1, W.Tm1Dims(3_000), 20_000, dict(dist="nurand")),
                                (W.TPCB, W.TpcbDims(3, 10, 1000), 6_000, dict(remote_pct=30.0))]:
        image = W.make_db(schema, dims, seed=2)
        bulk = W.make_bulk(schema, dims, n, 17, **kw)
        db = gpu_db(schema, dims, image, n)
        run_both(schema, dims, image, [bulk], "kset", db=db)
        assert np.array_equal(db.depths(), oracle.depths(schema, dims.dims, image, bulk))
        db.close()
