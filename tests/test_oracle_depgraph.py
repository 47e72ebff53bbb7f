"""Pins for the depth / k-set oracle (§4): the Figure-1 worked values,
the definition's O(n^3) edge test, Appendix B, topological sort, O(n^2) brute
force and the streaming recurrence in oracle.c must all agree, and k-sets must
satisfy Properties 1 and 2."""
import itertools
import json
import os
import random

import numpy as np
import pytest

import oracle
from oracle import depgraph as g

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _streaming(pool):
    """oracle.c orc_depths on a pool of (item, mode) lists."""
    items, modes, off = [], [], [0]
    names = {}
    for txn in pool:
        m = {}
        for it, md in txn:
            old = m.get(it)
            m[it] = md if old in (None, md) else 'W'
        for it, md in m.items():
            items.append(names.setdefault(it, len(names)))
            modes.append({'R': 0, 'W': 1, 'A': 2}[md])
        off.append(len(items))
    return list(oracle.depths_from_ops(np.array(off, np.uint64), np.array(items, np.uint64),
                                       np.array(modes, np.uint8)))


def test_figure1_worked_example():
    fx = json.load(open(os.path.join(GOLD, "figure1.json")))
    pool = [[tuple(op) for op in t] for t in fx["pool"]]
    edges = g.graph_by_definition(pool)
    assert edges == {tuple(e) for e in fx["edges"]}
    for e in fx["absent_edges"]:
        assert tuple(e) not in edges
    assert g.graph_appendix_b(pool) == edges
    assert g.topo_depths(len(pool), edges) == fx["depths"]
    assert g.depths_bruteforce(pool) == fx["depths"]
    assert _streaming(pool) == fx["depths"]
    assert g.literal_rank_rule(pool) == fx["ranks_group_a"]   # single-item pool: rule is exact
    assert g.ksets(fx["depths"]) == fx["ksets"]


def test_literal_rank_rule_counterexample():
    fx = json.load(open(os.path.join(GOLD, "rank_rule_counterexample.json")))
    pool = [[tuple(op) for op in t] for t in fx["pool"]]
    assert g.literal_rank_rule(pool) == fx["literal_rule_depths"]
    assert g.topo_depths(3, g.graph_by_definition(pool)) == fx["true_depths"]
    assert _streaming(pool) == fx["true_depths"]
    ok, _ = g.check_properties(pool, fx["literal_rule_depths"])
    assert not ok                                       # literal k-sets violate Property 1


def _closure(n, edges):
    reach = [set() for _ in range(n)]
    for v in range(n - 1, -1, -1):
        for a, b in edges:
            if a == v:
                reach[v] |= {b} | reach[b]
    return reach


def _same_order(n, e_def, e_b):
    """Appendix B adds edges per item and does not test condition (c) across items,
    so it may add t1 -> t2 implied by a path through a third transaction
    (DESIGN.md R-S8): a superset with the same reachability (hence depths)."""
    return e_def <= e_b and _closure(n, e_def) == _closure(n, e_b)


def _footprints(items):
    fps = []
    for k in range(1, len(items) + 1):
        for sub in itertools.combinations(items, k):
            for modes in itertools.product("RW", repeat=k):
                fps.append(list(zip(sub, modes)))
    return fps


def test_exhaustive_small_pools():
    """Every pool of <= 3 transactions over 3 items (26 footprints each)."""
    fps = _footprints(["a", "b", "c"])
    assert len(fps) == 26
    count = 0
    for n in (1, 2, 3):
        for pool in itertools.product(fps, repeat=n):
            pool = list(pool)
            edges = g.graph_by_definition(pool)
            eb = g.graph_appendix_b(pool)
            assert _same_order(n, edges, eb)
            d = g.topo_depths(n, edges)
            assert g.topo_depths(n, eb) == d
            assert g.depths_bruteforce(pool) == d
            ok, msg = g.check_properties(pool, d)
            assert ok, msg
            count += 1
    assert count == 26 + 26 ** 2 + 26 ** 3


def test_streaming_matches_graph_random():
    rng = random.Random(5)
    for _ in range(400):
        n = rng.randint(1, 12)
        nitems = rng.randint(1, 5)
        pool = [[(rng.randrange(nitems), rng.choice("RW")) for _ in range(rng.randint(0, 3))]
                for _ in range(n)]
        edges = g.graph_by_definition(pool)
        d = g.topo_depths(n, edges)
        eb = g.graph_appendix_b(pool)
        assert _same_order(n, edges, eb)
        assert g.topo_depths(n, eb) == d
        assert g.depths_bruteforce(pool) == d
        assert _streaming(pool) == d
        ok, msg = g.check_properties(pool, d)
        assert ok, msg


def test_literal_rule_exact_for_single_op_transactions():
    rng = random.Random(9)
    for _ in range(300):
        n = rng.randint(1, 15)
        pool = [[(rng.randrange(3), rng.choice("RW"))] for _ in range(n)]
        assert g.literal_rank_rule(pool) == g.depths_bruteforce(pool)


def test_reads_only_single_kset():
    pool = [[("x", "R")] for _ in range(10)]
    assert _streaming(pool) == [0] * 10
    assert g.graph_by_definition(pool) == set()


def test_empty_pool():
    assert _streaming([]) == []
    assert g.depths_bruteforce([]) == []


def test_add_rule_exhaustive_small_pools():
    """ADD rule: modes R/W/A, two adds of one item do not conflict.
    Every pool of <= 3 transactions over 2 items: the streaming recurrence of
    oracle.c equals the longest path of the graph built from the definition, and
    equals the O(n^2) brute force; Properties 1-2 hold."""
    fps = []
    for k in (1, 2):
        for sub in itertools.combinations(["a", "b"], k):
            for modes in itertools.product("RWA", repeat=k):
                fps.append(list(zip(sub, modes)))
    assert len(fps) == 3 + 3 + 9
    count = 0
    for n in (1, 2, 3):
        for pool in itertools.product(fps, repeat=n):
            pool = list(pool)
            d = g.topo_depths(n, g.graph_by_definition(pool))
            assert g.depths_bruteforce(pool) == d
            assert _streaming(pool) == d, pool
            ok, msg = g.check_properties(pool, d)
            assert ok, msg
            count += 1
    assert count == 15 + 15 ** 2 + 15 ** 3


def test_add_rule_random_pools():
    rng = random.Random(11)
    for _ in range(400):
        n = rng.randint(1, 14)
        nitems = rng.randint(1, 4)
        pool = [[(rng.randrange(nitems), rng.choice("RWAA")) for _ in range(rng.randint(0, 3))]
                for _ in range(n)]
        d = g.depths_bruteforce(pool)
        assert g.topo_depths(n, g.graph_by_definition(pool)) == d
        assert _streaming(pool) == d


def test_add_rule_special_cases():
    """Closed forms: adds only -> one k-set; add/read alternation on one item -> a chain
    of runs; a write after adds waits for all of them."""
    assert _streaming([[("x", "A")]] * 6) == [0] * 6
    assert _streaming([[("x", "A")], [("x", "A")], [("x", "R")], [("x", "R")], [("x", "A")]]) == [0, 0, 1, 1, 2]
    assert _streaming([[("x", "A")], [("x", "A")], [("x", "W")], [("x", "A")]]) == [0, 0, 1, 2]


def test_run_order_matches_one_at_a_time_replay():
    """orc_run_order (the witness replay of the relaxed strategies) equals
    executing the transactions one at a time in that order (run_sequence), and with the
    identity order equals Definition 1."""
    import numpy as np
    import oracle
    import workloads as W
    for schema, dims, kw in [(W.TPCB, W.TpcbDims(2, 2, 5), dict(remote_pct=30.0)), (W.TM1, W.Tm1Dims(4), {}),
                             (W.TPCC, W.TpccDims(2, 2, 3, 4), dict(rbk_pct=10.0)), (W.MICRO, W.MicroDims(5, 4, 1), {})]:
        db = W.make_db(schema, dims, seed=2)
        bulk = W.make_bulk(schema, dims, 40, 3, **kw)
        order = np.random.default_rng(1).permutation(bulk.n)
        a = oracle.run(schema, dims.dims, db, bulk, order=order)
        b = oracle.run_sequence(schema, dims.dims, db, bulk, order)
        for k in a.db:
            assert np.array_equal(a.db[k], b.db[k]), (schema, k)
        assert np.array_equal(a.status, b.status) and np.array_equal(a.out, b.out)
        for t in a.inserts:
            for c in a.inserts[t]:
                assert np.array_equal(a.inserts[t][c], b.inserts[t][c]), (schema, t, c)
        ident = oracle.run(schema, dims.dims, db, bulk, order=np.arange(bulk.n))
        ref = oracle.run(schema, dims.dims, db, bulk)
        assert np.array_equal(ident.out, ref.out) and all(np.array_equal(ident.db[k], ref.db[k]) for k in ref.db)
