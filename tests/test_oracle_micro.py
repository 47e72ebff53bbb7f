"""Pins for the micro-benchmark procedure of the oracle (§6.1; DESIGN.md
R-M1): "each transaction reads a tuple, and performs computation, and then writes the
result back to the tuple; the amount of computation is simulated with calling the _sinf
function (100 * x) times".  Checked against the mathematics it approximates (math.sin in
float64), its special case x = 0 (identity), the T-dependency graph closed form of
single-tuple writes, and the every-linear-extension brute force."""
import math

import numpy as np
import pytest

import oracle
import workloads as W
from oracle import depgraph as g


def _f32(bits):
    return float(np.uint32(bits).view(np.float32))


def test_x0_is_identity():
    """x = 0: no computation; the transaction writes back what it read and returns it."""
    d = W.MicroDims(500, 8, 0)
    db = W.micro_db(d, seed=2)
    b = W.micro_bulk(d, 3000, seed=3)
    r = oracle.run(W.MICRO, d.dims, db, b)
    tup = b.param_words.astype(np.int64)
    assert np.array_equal(r.db["tuple"], db["tuple"])
    assert np.array_equal(r.out.view(np.uint32).reshape(-1), db["tuple"][tup])
    assert (r.status == 0).all()


@pytest.mark.parametrize("t", [0, 5, 17, 31])
def test_one_call_is_sin_of_affine_argument(t):
    """One call of type t maps v to ~sin(A_t v + B_t), A_t = 15/16 - t/128, B_t =
    (t - 15.5)/1024: the degree-5 Taylor polynomial on |u| <= 1 is within 1/5040 of sin,
    plus float rounding.  100 calls (x = 1) of a contraction stay within 2e-3 of the
    float64 iteration of math.sin."""
    A = 0.9375 - t / 128.0
    B = (t - 15.5) / 1024.0
    vals = np.linspace(-0.5, 0.5, 41, dtype=np.float32)
    d = W.MicroDims(len(vals), 32, 1)
    db = {"tuple": vals.view(np.uint32).copy()}
    from workloads import Bulk
    b = Bulk(W.MICRO, np.full(len(vals), t, np.uint8), np.arange(len(vals) + 1, dtype=np.uint32),
             np.arange(len(vals), dtype=np.uint32))
    r = oracle.run(W.MICRO, d.dims, db, b)
    got = r.out.view(np.float32).reshape(-1).astype(np.float64)
    for v0, y in zip(vals.astype(np.float64), got):
        v = v0
        for _ in range(100):
            v = math.sin(A * v + B)
        assert abs(y - v) < 2e-3, (t, v0, y, v)


def test_types_are_distinct_functions():
    """The T branches compute different functions (the switch cannot be collapsed)."""
    d = W.MicroDims(32, 32, 2)
    v0 = np.full(32, np.float32(0.25)).view(np.uint32)
    from workloads import Bulk
    b = Bulk(W.MICRO, np.arange(32, dtype=np.uint8), np.arange(33, dtype=np.uint32), np.arange(32, dtype=np.uint32))
    r = oracle.run(W.MICRO, d.dims, {"tuple": v0.copy()}, b)
    assert len(set(r.out.view(np.uint32).reshape(-1).tolist())) == 32


def test_depth_is_number_of_earlier_transactions_on_the_tuple():
    """Every micro transaction writes one tuple, so the T-dependency graph is one path per
    tuple: depth(t) = #earlier transactions on its tuple.  With
    skew alpha the deepest path is tuple 0's."""
    d = W.MicroDims(5000, 8, 1)
    b = W.micro_bulk(d, 20000, seed=4, alpha=0.2)
    dep = oracle.depths(W.MICRO, d.dims, W.micro_db(d), b)
    tup = b.param_words.astype(np.int64)
    seen = {}
    want = np.zeros(b.n, np.int64)
    for i, x in enumerate(tup):
        want[i] = seen.get(x, 0)
        seen[x] = want[i] + 1
    assert np.array_equal(dep, want)
    assert dep.max() == int((tup == 0).sum()) - 1 and dep.max() > 3000


def test_every_linear_extension_equals_serial():
    """Any order respecting the per-tuple chains gives the serial result, and an order
    that swaps two transactions of different types on one tuple does not."""
    d = W.MicroDims(3, 4, 1)
    db = W.micro_db(d, seed=5)
    swapped_differs = 0
    for seed in range(8):
        b = W.micro_bulk(d, 6, seed)
        ref = oracle.run(W.MICRO, d.dims, db, b)
        off, items, modes = oracle.footprint(W.MICRO, d.dims, db, b)
        pool = [[(int(items[j]), 'W')] for j in range(b.n)]
        for order in g.linear_extensions(b.n, g.graph_by_definition(pool), limit=100):
            got = oracle.run_sequence(W.MICRO, d.dims, db, b, order)
            assert np.array_equal(got.db["tuple"], ref.db["tuple"]) and np.array_equal(got.out, ref.out)
        tup = b.param_words
        for i in range(b.n):
            for j in range(i + 1, b.n):
                if tup[i] == tup[j] and b.type[i] != b.type[j]:
                    order = list(range(b.n))
                    order[i], order[j] = order[j], order[i]
                    got = oracle.run_sequence(W.MICRO, d.dims, db, b, order)
                    swapped_differs += not np.array_equal(got.db["tuple"], ref.db["tuple"])
    assert swapped_differs > 0
