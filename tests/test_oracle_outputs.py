"""Pins for every output field and abort predicate of the serial executor (Definition 1,
PAPER.md:73) that the closed-form / invariant pins of test_oracle_benchmarks.py leave
open.  Each pin is a per-item PROJECTION written from the public benchmark definitions
(Ext TATP, Ext TPC-C; SURVEY.md §8(c) "per-item projection cross-check"): the state of
one item (a CF slot, a stock row, a district counter, a subscriber's bit_1) is replayed
in ts order from the bulk's parameters alone, and the oracle's status and output record
must equal what that replay predicts.  None of these helpers calls the oracle's
transaction loop; a dropped term, a wrong comparison or a swapped field in oracle.c
fails one of them."""
import numpy as np
import pytest

import oracle
import workloads as W
from oracle import depgraph as g


def _u32(row, at):
    return int(row[at:at + 4].copy().view(np.uint32)[0])


def _i32(row, at):
    return int(row[at:at + 4].copy().view(np.int32)[0])


def _u64(row, at):
    return int(row[at:at + 8].copy().view(np.uint64)[0])


def _i64(row, at):
    return int(row[at:at + 8].copy().view(np.int64)[0])


def _nbr_map(db):
    return {int(v): k for k, v in enumerate(db["sub_nbr"])}


# ----------------------------------------------------------------------------- TM-1
# TATP (Ext), read as DESIGN.md R-S12:
#  GET_NEW_DESTINATION returns cf.numberx of the CF rows of (s, sf) with
#    sf.is_active = 1  AND  cf.start_time <= start  AND  end < cf.end_time,
#  in start_time order; no such row -> the transaction fails.
#  INSERT_CALL_FORWARDING fails on a missing SF row (foreign key) or an existing
#    (s, sf, start) row (primary key); DELETE_CALL_FORWARDING fails when no row goes.
@pytest.mark.parametrize("seed,P,n,dist", [(11, 40, 6000, "uniform"), (12, 3000, 30000, "nurand")])
def test_tm1_cf_projection_predicts_gnd_icf_dcf(seed, P, n, dist):
    dims = W.Tm1Dims(P)
    db = W.tm1_db(dims, seed=seed)
    # a mix heavy in the call-forwarding types so every slot sees several of them
    b = W.tm1_bulk(dims, n, seed=seed + 1, dist=dist, mix=(5, 30, 5, 5, 5, 25, 25))
    r = oracle.run(W.TM1, dims.dims, db, b)
    nbr = _nbr_map(db)
    live = {}          # (s, sf, start) -> (end, numberx) of the live row
    for k in range(4 * P):
        for j in range(3):
            if db["cf_live"][k * 3 + j]:
                live[(k // 4, k % 4 + 1, 8 * j)] = (int(db["cf_end"][k * 3 + j]), int(db["cf_numberx"][k * 3 + j]))
    seen = {1: 0, 5: 0, 6: 0}
    hits = 0
    for i in range(n):
        t = int(b.type[i])
        p = [int(x) for x in b.params(i)]
        row = r.out[i]
        if t == W.TM1_GND:
            s, sf, start, end = p[0] - 1, p[1], p[2], p[3]
            f = s * 4 + sf - 1
            rows = []
            if db["sf_valid"][f] and db["sf_active"][f]:
                for st in (0, 8, 16):
                    x = live.get((s, sf, st))
                    if x is not None and st <= start and end < x[0]:
                        rows.append(x[1])
            want_status = 0 if rows else 1
            assert r.status[i] == want_status, (i, "GND status")
            if rows:
                hits += 1
                assert _u32(row, 0) == len(rows)
                assert [_u64(row, 8 + 8 * k) for k in range(len(rows))] == rows
                assert not row[8 + 8 * len(rows):].any()
            else:
                assert not row.any()
        elif t in (W.TM1_ICF, W.TM1_DCF):
            s = nbr.get(p[0] | (p[1] << 32), -1)
            sf, st = p[2], p[3]
            key = (s, sf, st)
            if t == W.TM1_ICF:
                ok = s >= 0 and bool(db["sf_valid"][s * 4 + sf - 1]) and key not in live
                if ok:
                    live[key] = (p[4], p[5] | (p[6] << 32))
            else:
                ok = s >= 0 and key in live
                if ok:
                    del live[key]
            assert r.status[i] == (0 if ok else 1), (i, t)
            assert not row.any()                      # no output record
        if t in seen:
            seen[t] += int(r.status[i] == 0)
    # the replay's final CF image equals the oracle's, field by field for live rows
    got_live = {(k // 4, k % 4 + 1, 8 * j) for k in range(4 * P) for j in range(3) if r.db["cf_live"][k * 3 + j]}
    assert got_live == set(live)
    for (s, sf, st), (end, num) in live.items():
        c = (s * 4 + sf - 1) * 3 + st // 8
        assert int(r.db["cf_end"][c]) == end and int(r.db["cf_numberx"][c]) == num
    assert hits > 20 and all(v > 10 for v in seen.values()), (hits, seen)


def test_tm1_gsd_gad_usd_outputs_by_projection():
    """GSD returns the subscriber row with bit_1 / vlr_location as last written before
    it (USD / UL); GAD returns the AI row or fails when it is missing; USD fails on a
    missing SF row and then writes nothing."""
    P = 60
    dims = W.Tm1Dims(P)
    db = W.tm1_db(dims, seed=21)
    b = W.tm1_bulk(dims, 8000, seed=22, dist="uniform", mix=(35, 0, 25, 20, 20, 0, 0))
    r = oracle.run(W.TM1, dims.dims, db, b)
    nbr = _nbr_map(db)
    bits = db["sub_bits"].astype(np.int64).copy()
    vlr = db["sub_vlr"].astype(np.int64).copy()
    da = db["sf_data_a"].astype(np.int64).copy()
    counts = np.zeros(7, int)
    for i in range(b.n):
        t = int(b.type[i])
        p = [int(x) for x in b.params(i)]
        row = r.out[i]
        counts[t] += 1
        if t == W.TM1_GSD:
            s = p[0] - 1
            assert r.status[i] == 0
            assert _u64(row, 0) == int(db["sub_nbr"][s])
            assert _u64(row, 8) == int(db["sub_hex"][s])
            assert _u32(row, 16) == int(db["sub_msc"][s])
            assert _u32(row, 20) == vlr[s]
            assert int(row[24:26].copy().view(np.uint16)[0]) == bits[s]
            assert bytes(row[26:36]) == bytes(db["sub_byte2"][s])
            assert not row[36:].any()
        elif t == W.TM1_GAD:
            a = (p[0] - 1) * 4 + p[1] - 1
            if db["ai_valid"][a]:
                assert r.status[i] == 0
                assert row[0] == db["ai_data1"][a] and row[1] == db["ai_data2"][a]
                assert _u32(row, 4) == int(db["ai_data3"][a]) and _u64(row, 8) == int(db["ai_data4"][a])
            else:
                assert r.status[i] == 1 and not row.any()
        elif t == W.TM1_USD:
            s, f = p[0] - 1, (p[0] - 1) * 4 + p[1] - 1
            if db["sf_valid"][f]:
                assert r.status[i] == 0
                bits[s] = (bits[s] & ~1) | (p[2] & 1)
                da[f] = p[3]
            else:
                assert r.status[i] == 1
        elif t == W.TM1_UL:
            s = nbr[p[0] | (p[1] << 32)]
            assert r.status[i] == 0
            vlr[s] = p[2]
    assert np.array_equal(r.db["sub_bits"].astype(np.int64), bits)
    assert np.array_equal(r.db["sf_data_a"].astype(np.int64), da)
    assert np.array_equal(r.db["sub_vlr"].astype(np.int64), vlr)
    assert (counts[[0, 2, 3, 4]] > 500).all()


# ----------------------------------------------------------------------------- TPC-C
@pytest.mark.parametrize("dims", [W.TpccDims(2, 3, 40, 60), W.TpccDims(4, 10, 300, 2000)])
def test_tpcc_neworder_line_outputs_and_payment_credit(dims):
    """NewOrder (Ext TPC-C 2.4.2.2): o_id = D_NEXT_O_ID before the increment; per
    line, the S_QUANTITY read BEFORE its update (a stock row repeated inside one
    order sees the earlier line's update), ol_amount = qty * I_PRICE and brand =
    I_ORIGINAL and S_ORIGINAL.  Payment (2.5.2.2): output c_credit of the chosen
    customer and C_BALANCE after the payment."""
    n = 4000
    Wn, D, C, I = dims.dims
    db = W.tpcc_db(dims, seed=5)
    b = W.tpcc_bulk(dims, n, seed=6)
    r = oracle.run(W.TPCC, dims.dims, db, b)
    q = db["s_quantity"].astype(np.int64).copy()
    dnext = db["d_next_o_id"].astype(np.int64).copy()
    bal = db["c_balance"].astype(np.int64).copy()
    repeats = lines = credit_bc = 0
    for i in range(n):
        p = [int(x) for x in b.params(i)]
        row = r.out[i]
        if b.type[i] == W.TPCC_NEWORDER:
            w, d, k = p[0], p[1], p[3]
            L = [(p[4 + 3 * l], p[5 + 3 * l], p[6 + 3 * l]) for l in range(k)]
            if any(it >= I for it, _, _ in L):
                assert r.status[i] == 1 and not row.any()
                continue
            assert r.status[i] == 0
            assert _u32(row, 0) == dnext[w * D + d]
            dnext[w * D + d] += 1
            assert _u32(row, 4) == k
            seen = set()
            for l, (it, sw, qty) in enumerate(L):
                s = sw * I + it
                repeats += s in seen
                seen.add(s)
                before = q[s]
                q[s] = before - qty if before >= qty + 10 else before - qty + 91
                o = 16 + 12 * l
                assert _i32(row, o) == before, (i, l)
                assert _i32(row, o + 4) == qty * int(db["i_price"][it])
                assert row[o + 8] == (1 if db["i_original"][it] and db["s_original"][s] else 0)
                assert not row[o + 9:o + 12].any()
                lines += 1
            assert not row[16 + 12 * k:].any()
        else:
            assert r.status[i] == 0
            cw, cd, h = p[2], p[3], p[6]
            c = _u32(row, 0)
            key = (cw * D + cd) * C + c
            assert _u32(row, 4) == int(db["c_credit"][key])
            bal[key] -= h
            assert _i64(row, 8) == bal[key]
            credit_bc += int(db["c_credit"][key] != 0)
    assert np.array_equal(r.db["s_quantity"].astype(np.int64), q)
    assert np.array_equal(r.db["d_next_o_id"].astype(np.int64), dnext)
    assert lines > 1000 and credit_bc > 0
    if D * C < 200:
        assert repeats > 0           # the tiny case exercises a repeated stock row


def test_appendix_b_rejects_add_operations():
    """Appendix B is defined for reads and writes only."""
    with pytest.raises(ValueError):
        g.graph_appendix_b([[(0, 'A')], [(0, 'R')]])
