"""Pins of the strategy chooser's oracle: Algorithm 1
 on every branch and boundary, and the structural parameters
w0, d, c on hand-built bulks whose values are fixed by
construction, not by the oracle."""
import numpy as np
import pytest

import oracle
import workloads as W


@pytest.mark.parametrize("w0,d,c,want", [
    (100, 0, 0, "kset"),        # w0 >= w0_bar (line 2)
    (99, 5000, 9999, "part"),   # d >= d_bar (line 7)
    (99, 10, 3, "part"),        # c <= c_bar (line 7)
    (99, 10, 4, "tpl"),         # neither (line 10)
    (100, 10, 4, "kset"),       # the w0 test comes first and is ">="
    (99, 20, 4, "part"),        # ">=" on d
    (99, 19, 4, "tpl"),
])
def test_algorithm1_branches(w0, d, c, want):
    assert oracle.choose_strategy(w0, d, c, w0_bar=100, d_bar=20, c_bar=3) == want


def _bulk(schema, types, rows):
    return W._pack(schema, np.asarray(types, np.uint8), [np.asarray(r, np.uint32) for r in rows])


def test_cross_partition_tpcb_by_construction():
    # 3 branches x 2 tellers x 5 accounts; deposit [aid, tid, bid, delta]
    dims = W.TpcbDims(3, 2, 5)
    b = _bulk(W.TPCB, [0] * 4, [[0, 0, 0, 5], [7, 1, 0, 5], [14, 5, 2, 3], [4, 2, 1, 1]])
    got = oracle.cross_partition(W.TPCB, dims.dims, b, np.zeros(4, np.uint8))
    assert got.tolist() == [False, True, False, True]     # account 7 is branch 1's, 4 is branch 0's


def test_cross_partition_tpcc_by_construction():
    dims = W.TpccDims(3, 2, 30, 40)
    image = W.tpcc_db(dims, seed=1)
    rows = [
        [0, 0, 1, 5] + [1, 0, 1, 2, 0, 1, 3, 0, 1, 4, 0, 1, 5, 0, 1],     # NO, all lines local
        [1, 1, 2, 5] + [1, 1, 1, 2, 1, 1, 3, 2, 1, 4, 1, 1, 5, 1, 1],     # NO, line 3 from w 2
        [2, 0, 3, 5] + [1, 2, 1, 2, 0, 1, 3, 2, 1, 4, 2, 1, 40, 2, 1],    # NO, remote line, unused item 40 -> aborts
        [0, 1, 0, 1, 0, 7, 100],                                          # Payment, local customer
        [0, 1, 2, 0, 0, 7, 100],                                          # Payment, customer of w 2
    ]
    b = _bulk(W.TPCC, [0, 0, 0, 1, 1], rows)
    st = oracle.run(W.TPCC, dims.dims, image, b).status
    assert st.tolist() == [0, 0, 1, 0, 0]
    assert oracle.cross_partition(W.TPCC, dims.dims, b, st).tolist() == [False, True, False, False, True]


def test_structure_tpcb_one_branch_closed_form():
    """One branch: every deposit writes the branch balance, so the graph is one path
    (depth(t) = t): w0 = 1, d = n - 1, c = 0 (no other branch)."""
    dims = W.TpcbDims(1, 10, 1000)
    b = W.tpcb_bulk(dims, 300, seed=2)
    s = oracle.structure(W.TPCB, dims.dims, W.tpcb_db(dims), b)
    assert s == {"w0": 1, "d": 299, "c": 0}


def test_structure_tm1_single_partition():
    """TM-1 transactions touch one subscriber: c = 0 for any bulk."""
    dims = W.Tm1Dims(500)
    image = W.tm1_db(dims, seed=3)
    b = W.tm1_bulk(dims, 2000, seed=4)
    s = oracle.structure(W.TM1, dims.dims, image, b)
    assert s["c"] == 0 and s["w0"] >= 1 and s["d"] >= 1
