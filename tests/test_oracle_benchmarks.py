"""Pins for the serial executor (Definition 1) against closed forms,
consistency invariants and per-item projections of the benchmark definitions
(DESIGN.md §3), none of which re-run the oracle's own transaction loop."""
import numpy as np
import pytest

import oracle
import workloads as W


# ------------------------------------------------------------------------------ TPC-B
def _prefix_by_key(keys, vals):
    """Running sum of vals per key, in array order."""
    order = np.argsort(keys, kind="stable")
    k, v = keys[order], vals[order]
    cs = np.cumsum(v)
    start = np.r_[0, np.nonzero(k[1:] != k[:-1])[0] + 1]
    base = np.zeros_like(cs)
    seg = np.zeros(len(k), np.int64)
    seg[start] = 1
    seg = np.cumsum(seg) - 1
    base = (cs - v)[start][seg]
    out = np.empty_like(cs)
    out[order] = cs - base
    return out


@pytest.mark.parametrize("dims,remote", [(W.TpcbDims(1, 10, 100_000), 0.0),
                                          (W.TpcbDims(8, 10, 1000), 15.0),
                                          (W.TpcbDims(4, 3, 50), 40.0)])
def test_tpcb_closed_forms(dims, remote):
    n = 4096
    db = W.tpcb_db(dims)
    b = W.tpcb_bulk(dims, n, seed=3, remote_pct=remote)
    r = oracle.run(W.TPCB, dims.dims, db, b, first_ts=100)
    p = b.param_words.reshape(n, 4).astype(np.int64)
    aid, tid, bid = p[:, 0], p[:, 1], p[:, 2]
    delta = p[:, 3].astype(np.uint32).view(np.int32).astype(np.int64)
    assert (r.status == 0).all()                                  # TPC-B never aborts
    acc = np.zeros(dims.branches * dims.accounts_per_branch, np.int64)
    np.add.at(acc, aid, delta)
    assert np.array_equal(r.db["acc_bal"], acc)                    # A = sum of deltas
    tel = np.zeros(dims.branches * dims.tellers_per_branch, np.int64)
    np.add.at(tel, tid, delta)
    assert np.array_equal(r.db["tel_bal"], tel)
    br = np.zeros(dims.branches, np.int64)
    np.add.at(br, bid, delta)
    assert np.array_equal(r.db["br_bal"], br)
    # Sum A = Sum T = Sum B = Sum history.delta (Ext TPC-B consistency)
    s = r.db["acc_bal"].sum()
    assert s == r.db["tel_bal"].sum() == r.db["br_bal"].sum() == r.inserts["history"]["h_delta"].sum()
    # output = account balance after its own update = prefix sum per account
    out = r.out.view(np.int64).reshape(-1)
    assert np.array_equal(out, _prefix_by_key(aid, delta))
    h = r.inserts["history"]
    assert np.array_equal(h["h_ts"], 100 + np.arange(n))
    assert np.array_equal(h["h_aid"], aid) and np.array_equal(h["h_tid"], tid)
    # tellers belong to the branch, accounts to the branch unless remote
    assert np.array_equal(tid // dims.tellers_per_branch, bid)
    if remote == 0:
        assert np.array_equal(aid // dims.accounts_per_branch, bid)


def test_tpcb_tiny_depth_is_ts():
    """Config 1 (one branch): every pair conflicts on the branch, so the
    T-dependency graph is one path and depth(t) = t."""
    dims = W.TpcbDims(1, 10, 100_000)
    b = W.tpcb_bulk(dims, 4096, seed=1)
    d = oracle.depths(W.TPCB, dims.dims, W.tpcb_db(dims), b)
    assert np.array_equal(d, np.arange(4096))


def test_tpcb_paths_per_branch():
    """0% remote: the graph degrades to one path per branch, so
    depth(t) = #earlier transactions of the same branch."""
    dims = W.TpcbDims(16, 10, 1000)
    b = W.tpcb_bulk(dims, 5000, seed=2, remote_pct=0.0)
    bid = b.param_words.reshape(-1, 4)[:, 2].astype(np.int64)
    ones = np.ones_like(bid)
    expect = _prefix_by_key(bid, ones) - 1
    d = oracle.depths(W.TPCB, dims.dims, W.tpcb_db(dims), b)
    assert np.array_equal(d, expect)


# ------------------------------------------------------------------------------ TM-1
def test_tm1_projections():
    dims = W.Tm1Dims(2000)
    db = W.tm1_db(dims, seed=4)
    b = W.tm1_bulk(dims, 20000, seed=5, dist="nurand")
    r = oracle.run(W.TM1, dims.dims, db, b)
    t = b.type
    n = b.n
    P = dims.subscribers
    # static aborts: GAD fails iff the AI row is missing
    gad = np.nonzero(t == W.TM1_GAD)[0]
    for i in gad:
        s_id, ai = b.params(i)
        assert r.status[i] == (0 if db["ai_valid"][(s_id - 1) * 4 + ai - 1] else 1)
    # USD fails iff the SF row is missing
    for i in np.nonzero(t == W.TM1_USD)[0]:
        s_id, sf = b.params(i)[:2]
        assert r.status[i] == (0 if db["sf_valid"][(s_id - 1) * 4 + sf - 1] else 1)
    # vlr_location = the last UL value (UL never fails), else initial
    vlr = db["sub_vlr"].copy()
    nbr_to_s = {int(v): k for k, v in enumerate(db["sub_nbr"])}
    for i in np.nonzero(t == W.TM1_UL)[0]:
        lo, hi, v = b.params(i)
        vlr[nbr_to_s[int(lo) | (int(hi) << 32)]] = v
    assert np.array_equal(r.db["sub_vlr"], vlr)
    # bit_1 / data_a = last committed USD
    bits = db["sub_bits"].copy()
    da = db["sf_data_a"].copy()
    for i in np.nonzero((t == W.TM1_USD) & (r.status == 0))[0]:
        s_id, sf, b1, d_a = b.params(i)
        bits[s_id - 1] = (bits[s_id - 1] & 0xFFFE) | b1
        da[(s_id - 1) * 4 + sf - 1] = d_a
    assert np.array_equal(r.db["sub_bits"], bits)
    assert np.array_equal(r.db["sf_data_a"], da)
    # live CF rows = initial + committed ICF - committed DCF
    ok = r.status == 0
    assert int(r.db["cf_live"].sum()) == int(db["cf_live"].sum()) + int(((t == W.TM1_ICF) & ok).sum()) \
        - int(((t == W.TM1_DCF) & ok).sum())
    # read-only tables unchanged
    for k in ["sub_nbr", "sub_hex", "sub_msc", "ai_valid", "ai_data4", "sf_valid", "sf_active"]:
        assert np.array_equal(r.db[k], db[k])
    # GSD output: sub_nbr and hex are static
    gsd = np.nonzero(t == W.TM1_GSD)[0]
    o = r.out[gsd]
    s = b.param_words[b.param_off[gsd]].astype(np.int64) - 1
    assert np.array_equal(o[:, 0:8].copy().view(np.uint64).reshape(-1), db["sub_nbr"][s])
    assert (r.status[gsd] == 0).all()
    # abort rates near TATP's (statistical; parity-unpinned as a rate)
    gnd_fail = r.status[t == W.TM1_GND].mean()
    assert 0.6 < gnd_fail < 0.95
    assert 0.25 < r.status[t == W.TM1_GAD].mean() < 0.5


def test_tm1_gsd_sees_last_ul():
    """A read returns the last prior write (per-item projection on vlr_location)."""
    dims = W.Tm1Dims(50)
    db = W.tm1_db(dims, seed=1)
    b = W.tm1_bulk(dims, 3000, seed=2, dist="uniform", mix=(50, 0, 0, 0, 50, 0, 0))
    r = oracle.run(W.TM1, dims.dims, db, b)
    cur = db["sub_vlr"].copy()
    nbr_to_s = {int(v): k for k, v in enumerate(db["sub_nbr"])}
    for i in range(b.n):
        p = b.params(i)
        if b.type[i] == W.TM1_UL:
            cur[nbr_to_s[int(p[0]) | (int(p[1]) << 32)]] = p[2]
        else:
            assert r.out[i, 20:24].view(np.uint32)[0] == cur[p[0] - 1]


# ------------------------------------------------------------------------------ TPC-C
@pytest.mark.parametrize("dims", [W.TpccDims(4, 10, 3000, 100_000), W.TpccDims(3, 4, 60, 500)])
def test_tpcc_invariants(dims):
    n = 6000
    db = W.tpcc_db(dims, seed=2)
    b = W.tpcc_bulk(dims, n, seed=3)
    r = oracle.run(W.TPCC, dims.dims, db, b, first_ts=7)
    Wn, D, C, I = dims.dims
    f = r.db
    # W_YTD = sum of D_YTD (Ext TPC-C 3.3.2.1)
    assert np.array_equal(f["w_ytd"], f["d_ytd"].reshape(Wn, D).sum(axis=1))
    o, no, ol, h = (r.inserts[k] for k in ("order", "new_order", "order_line", "history"))
    wd_o = o["o_w"].astype(np.int64) * D + o["o_d"]
    # D_NEXT_O_ID - 1 = max(O_ID) per district; new ids contiguous from 3001 (3.3.2.2/3)
    for wd in range(Wn * D):
        ids = np.sort(o["o_id"][wd_o == wd])
        assert np.array_equal(ids, np.arange(3001, f["d_next_o_id"][wd]))
    assert np.array_equal(np.sort(no["no_o_id"]), np.sort(o["o_id"]))
    # sum O_OL_CNT = #ORDER_LINE (3.3.2.4)
    assert int(o["o_ol_cnt"].sum()) == len(ol["ol_o_id"])
    # NewOrder rolls back iff its last item is unused (2.4.2.3)
    is_no = b.type == W.TPCC_NEWORDER
    last_bad = np.array([b.params(i)[4 + 3 * (b.params(i)[3] - 1)] >= I if is_no[i] else False
                         for i in range(n)])
    assert np.array_equal(r.status.astype(bool), last_bad)
    assert len(o["o_id"]) == int((is_no & ~last_bad).sum())
    # delta W_YTD = sum of h_amount of home Payments
    hw = np.zeros(Wn, np.int64)
    np.add.at(hw, h["h_w"].astype(np.int64), h["h_amount"].astype(np.int64))
    assert np.array_equal(f["w_ytd"] - db["w_ytd"], hw)
    # C_BALANCE + C_YTD_PAYMENT constant; payment count = #payments
    assert np.array_equal(f["c_balance"] + f["c_ytd_payment"], db["c_balance"] + db["c_ytd_payment"])
    cidx = (h["h_cw"].astype(np.int64) * D + h["h_cd"]) * C + h["h_c"]
    cnt = np.zeros(Wn * D * C, np.int64)
    np.add.at(cnt, cidx, 1)
    assert np.array_equal(f["c_payment_cnt"].astype(np.int64) - db["c_payment_cnt"], cnt)
    # delta S_YTD = sum ol_quantity; S_ORDER_CNT = #lines; S_REMOTE_CNT = #remote lines
    sidx = ol["ol_supply_w"].astype(np.int64) * I + ol["ol_i_id"]
    ytd = np.zeros(Wn * I, np.int64)
    np.add.at(ytd, sidx, ol["ol_quantity"].astype(np.int64))
    assert np.array_equal(f["s_ytd"] - db["s_ytd"], ytd)
    oc = np.zeros(Wn * I, np.int64)
    np.add.at(oc, sidx, 1)
    assert np.array_equal(f["s_order_cnt"].astype(np.int64), oc)
    rc = np.zeros(Wn * I, np.int64)
    np.add.at(rc, sidx, (ol["ol_supply_w"] != ol["ol_w"]).astype(np.int64))
    assert np.array_equal(f["s_remote_cnt"].astype(np.int64), rc)
    # stock quantity: per-item projection, replaying each stock's lines in ts order
    q = db["s_quantity"].astype(np.int64).copy()
    for s, qty in zip(sidx, ol["ol_quantity"].astype(np.int64)):
        q[s] = q[s] - qty if q[s] >= qty + 10 else q[s] - qty + 91
    assert np.array_equal(f["s_quantity"].astype(np.int64), q)
    assert (f["s_quantity"] >= 1).all() and (f["s_quantity"] <= 100).all()
    # ORDER_LINE amount = qty * I_PRICE
    assert np.array_equal(ol["ol_amount"].astype(np.int64),
                          ol["ol_quantity"].astype(np.int64) * db["i_price"][ol["ol_i_id"]])
    # Payment output: c_balance after = initial - running sum of that customer's payments
    pay = np.nonzero(b.type == W.TPCC_PAYMENT)[0]
    out_c = r.out[pay, 0:4].copy().view(np.uint32).reshape(-1).astype(np.int64)
    out_bal = r.out[pay, 8:16].copy().view(np.int64).reshape(-1)
    cw = np.array([b.params(i)[2] for i in pay], np.int64)
    cd = np.array([b.params(i)[3] for i in pay], np.int64)
    amt = np.array([b.params(i)[6] for i in pay], np.int64)
    key = (cw * D + cd) * C + out_c
    assert np.array_equal(out_bal, db["c_balance"][key] - _prefix_by_key(key, amt))
    # by-name: the chosen customer has that C_LAST and is the ceil(n/2)-th by C_FIRST
    for j, i in enumerate(pay[:300]):
        p = b.params(i)
        if p[4]:
            base = (p[2] * D + p[3]) * C
            same = np.nonzero(db["c_last"][base:base + C] == p[5])[0]
            firsts = np.sort(db["c_first"][base + same])
            assert db["c_last"][base + out_c[j]] == p[5]
            assert firsts[(len(same) + 1) // 2 - 1] == db["c_first"][base + out_c[j]]
        else:
            assert out_c[j] == p[5]
    # NewOrder total from the order lines (Ext TPC-C 2.4.2.2, rates in 1e-4, half up)
    for i in np.nonzero(is_no & ~last_bad)[0][:300]:
        p = b.params(i)
        w, d, c, k = p[0], p[1], p[2], p[3]
        lines = p[4:4 + 3 * k].reshape(k, 3).astype(np.int64)
        s = int((lines[:, 2] * db["i_price"][lines[:, 0]]).sum())
        disc = int(db["c_discount"][(w * D + d) * C + c])
        tax = int(db["w_tax"][w]) + int(db["d_tax"][w * D + d])
        x = s * (10000 - disc) * (10000 + tax)
        assert r.out[i, 8:16].view(np.int64)[0] == (2 * x + 10 ** 8) // (2 * 10 ** 8)
        assert r.out[i, 4:8].view(np.uint32)[0] == k


# ------------------------------------------------------------------------------ brute force
def _rows(tab):
    cols = sorted(tab)
    return sorted(zip(*[tab[c].tolist() for c in cols])) if cols else []


def _same(schema, a, b):
    for k in a.db:
        if not np.array_equal(a.db[k], b.db[k]):
            return False
    if not (np.array_equal(a.status, b.status) and np.array_equal(a.out, b.out)):
        return False
    return all(_rows(a.inserts[t]) == _rows(b.inserts[t]) for t in a.inserts)


def _graph(schema, dims, db, bulk, drop=None):
    from oracle import depgraph as g
    off, items, modes = oracle.footprint(schema, dims.dims, db, bulk)
    pool = []
    for i in range(bulk.n):
        ops = [(int(items[j]), 'W' if modes[j] else 'R') for j in range(off[i], off[i + 1])]
        if drop is not None and drop(bulk.type[i]):
            ops = []
        pool.append(ops)
    return g.graph_by_definition(pool)


CASES = [
    (W.TPCB, W.TpcbDims(2, 2, 3), dict(remote_pct=30.0)),
    (W.TM1, W.Tm1Dims(3), dict(dist="uniform")),
    (W.TPCC, W.TpccDims(2, 2, 3, 4), dict(remote_line_pct=30.0, remote_pay_pct=30.0, rbk_pct=10.0)),
]


@pytest.mark.parametrize("schema,dims,kw", CASES)
def test_every_linear_extension_equals_serial(schema, dims, kw):
    """Any execution order that respects the T-dependency graph built from the
    declared footprints yields the serial result (shows the footprints are
    complete; Definition 1 + PAPER.md:111)."""
    from oracle import depgraph as g
    db = W.make_db(schema, dims, seed=3)
    total = 0
    for seed in range(12):
        bulk = W.make_bulk(schema, dims, 6, seed, **kw)
        ref = oracle.run(schema, dims.dims, db, bulk)
        edges = _graph(schema, dims, db, bulk)
        exts = g.linear_extensions(bulk.n, edges, limit=200)
        for order in exts:
            got = oracle.run_sequence(schema, dims.dims, db, bulk, order)
            assert _same(schema, ref, got), (seed, order)
        total += len(exts)
    assert total > 50


def test_dropped_footprint_is_detected():
    """Negative control: without GSD's read operations some extension differs."""
    from oracle import depgraph as g
    dims = W.Tm1Dims(2)
    db = W.tm1_db(dims, seed=3)
    bad = 0
    for seed in range(40):
        bulk = W.tm1_bulk(dims, 6, seed, dist="uniform", mix=(50, 0, 0, 0, 50, 0, 0))
        ref = oracle.run(W.TM1, dims.dims, db, bulk)
        edges = _graph(W.TM1, dims, db, bulk, drop=lambda t: t == W.TM1_GSD)
        for order in g.linear_extensions(bulk.n, edges, limit=50):
            if not _same(W.TM1, ref, oracle.run_sequence(W.TM1, dims.dims, db, bulk, order)):
                bad += 1
    assert bad > 0


@pytest.mark.parametrize("schema,dims,kw", CASES)
def test_kset_order_equals_serial(schema, dims, kw):
    """Executing k-set by k-set (any order inside a k-set) equals serial order
    (§5.3)."""
    rng = np.random.default_rng(0)
    db = W.make_db(schema, dims, seed=3)
    for seed in range(20):
        bulk = W.make_bulk(schema, dims, 40, seed, **kw)
        ref = oracle.run(schema, dims.dims, db, bulk)
        d = oracle.depths(schema, dims.dims, db, bulk)
        order = np.lexsort((rng.random(bulk.n), d))
        assert _same(schema, ref, oracle.run_sequence(schema, dims.dims, db, bulk, order))


def test_shard_split_covers_bulk_once():
    """Sharding helpers (workloads): every transaction has exactly one home shard, homes
    keep the bulk's order, and owned row ranges tile each table."""
    dims = W.TpccDims(6, 10, 30, 500)
    bulk = W.tpcc_bulk(dims, 2000, seed=4)
    for G in (1, 2, 4):
        parts = W.split_home(bulk, dims, G)
        ts = np.concatenate([p.ts for p in parts])
        assert np.array_equal(np.sort(ts), np.arange(bulk.n))
        for r, p in enumerate(parts):
            assert np.all(np.diff(p.ts.astype(np.int64)) > 0)
            assert np.all(W.shard_of(W.home_roots(p), G, 6) == r)
            for k in range(min(p.n, 20)):
                assert np.array_equal(p.params(k), bulk.params(int(p.ts[k])))
        rows = [W.shard_rows(W.TPCC, dims, G, r)["stock"] for r in range(G)]
        assert rows[0][0] == 0 and rows[-1][1] == 6 * 500
        assert all(rows[r][1] == rows[r + 1][0] for r in range(G - 1))


def test_tpcb_add_rule_depth_closed_form():
    """ADD rule: teller and branch balances are increments, so deposits conflict only
    on the account row: depth(t) = number of earlier deposits to the same account."""
    dims = W.TpcbDims(2, 10, 50)
    image = W.tpcb_db(dims)
    bulk = W.tpcb_bulk(dims, 3000, seed=8, remote_pct=30.0)
    d = oracle.depths(W.TPCB, dims.dims, image, bulk, add_rule=True)
    aid = bulk.param_words[0::4].astype(np.int64)
    seen = {}
    want = []
    for a in aid:
        want.append(seen.get(a, 0))
        seen[a] = seen.get(a, 0) + 1
    assert np.array_equal(d, np.array(want))
    # without the rule every deposit of a branch is one chain (depth >= branch position)
    d0 = oracle.depths(W.TPCB, dims.dims, image, bulk)
    assert d0.max() > 1000 and d.max() < 200


def test_tpcb_withdraw_non_two_phase_by_projection():
    """WITHDRAW (type 1, NEXT-4 / PAPER.md:441-443) debits first and aborts afterwards if
    the account went negative; its undo must leave no trace.  Per-account projection: a
    withdrawal commits iff the balance before it covers the amount; teller and branch
    balances are the sums of committed signed amounts; Sum A = Sum T = Sum B; only
    deposits add history rows."""
    dims = W.TpcbDims(4, 3, 40)
    db = W.tpcb_db(dims)
    b = W.tpcb_bulk(dims, 6000, seed=9, remote_pct=20.0, withdraw_pct=45.0)
    r = oracle.run(W.TPCB, dims.dims, db, b)
    p = b.param_words.reshape(-1, 4).astype(np.int64)
    amt = p[:, 3].astype(np.uint32).view(np.int32).astype(np.int64)
    acc = np.zeros(dims.branches * dims.accounts_per_branch, np.int64)
    tel = np.zeros(dims.branches * dims.tellers_per_branch, np.int64)
    br = np.zeros(dims.branches, np.int64)
    aborts = 0
    for i in range(b.n):
        a, t, bb = p[i, 0], p[i, 1], p[i, 2]
        if b.type[i] == W.TPCB_WITHDRAW:
            assert a // dims.accounts_per_branch == bb                 # always a local account
            if acc[a] >= amt[i]:
                acc[a] -= amt[i]; tel[t] -= amt[i]; br[bb] -= amt[i]
                assert r.status[i] == 0 and r.out[i].view(np.int64)[0] == acc[a]
            else:
                aborts += 1
                assert r.status[i] == 1 and not r.out[i].any()
        else:
            acc[a] += amt[i]; tel[t] += amt[i]; br[bb] += amt[i]
            assert r.status[i] == 0 and r.out[i].view(np.int64)[0] == acc[a]
    assert np.array_equal(r.db["acc_bal"], acc) and np.array_equal(r.db["tel_bal"], tel)
    assert np.array_equal(r.db["br_bal"], br)
    assert acc.sum() == tel.sum() == br.sum()
    assert len(r.inserts["history"]["h_ts"]) == int((b.type == 0).sum())
    assert 100 < aborts < int((b.type == 1).sum())
