"""T-dependency graph on small pools — TEST INFRASTRUCTURE ONLY (pure Python).

A pool is a list of transactions in timestamp order; each transaction is a list
of basic operations (item, mode) with mode 'R' or 'W' (§4.1), or 'A'
(a commutative increment) under the ADD rule (PAPER.md:475(c):
two adds of an item do not conflict; an add conflicts with reads and writes).
These loops are for small pools (n <= a few hundred); full-size depths use
oracle.depths() (the streaming recurrence in oracle.c).
"""
from __future__ import annotations

import itertools
from collections import defaultdict


def _norm(txn):
    """Merge same-item operations of one transaction; W dominates, differing modes
    merge to W (DESIGN.md R-S3)."""
    m = {}
    for item, mode in txn:
        old = m.get(item)
        m[item] = mode if old in (None, mode) else 'W'
    return m


def _ops_conflict(x: str, y: str) -> bool:
    """Two operations on one item conflict unless both read or both add."""
    return not (x == y and x in ('R', 'A'))


def conflicting(t1, t2) -> bool:
    """two transactions conflict iff they have two operations on the
    same data item and at least one is a write (and, ADD rule, not both adds)."""
    a, b = _norm(t1), _norm(t2)
    return any(x in b and _ops_conflict(a[x], b[x]) for x in a)


def graph_by_definition(pool):
    """Edges t1 -> t2 iff (a) conflicting, (b) ts(t1) < ts(t2), (c) no t strictly
    between them conflicts with both.  O(n^3)."""
    n = len(pool)
    C = [[conflicting(pool[i], pool[j]) if i != j else False for j in range(n)] for i in range(n)]
    edges = set()
    for i in range(n):
        for j in range(i + 1, n):
            if C[i][j] and not any(C[i][k] and C[k][j] for k in range(i + 1, j)):
                edges.add((i, j))
    return edges


def graph_appendix_b(pool):
    """Appendix B: add transactions in ts order; per item keep the
    ascending list of transactions that accessed it.  A write scans back from the
    tail to the last writer t_w: edge t_w -> t if t_w is the tail, else edges from
    EVERY reader between the tail and t_w (reading R-S8).  A read adds t_w -> t.
    Appendix B knows reads and writes only: an 'A' operation raises ValueError."""
    lists = defaultdict(list)          # item -> [(txn, mode)]
    edges = set()
    for t, txn in enumerate(pool):
        for item, mode in _norm(txn).items():
            if mode not in ('R', 'W'):
                raise ValueError(f"graph_appendix_b: mode {mode!r} (Appendix B has R/W only)")
            L = lists[item]
            if L:
                if mode == 'W':
                    k = len(L) - 1
                    readers = []
                    while k >= 0 and L[k][1] != 'W':
                        readers.append(L[k][0])
                        k -= 1
                    if not readers:            # t_w is the tail
                        edges.add((L[-1][0], t))
                    else:
                        for r in readers:
                            edges.add((r, t))
                else:
                    k = len(L) - 1
                    while k >= 0 and L[k][1] != 'W':
                        k -= 1
                    if k >= 0:
                        edges.add((L[k][0], t))
            L.append((t, mode))
    return edges


def topo_depths(n, edges):
    """Topological sort; depth(v) = 1 + max depth of v's predecessors, sources 0
    (PAPER.md:135)."""
    preds = defaultdict(list)
    indeg = [0] * n
    succ = defaultdict(list)
    for a, b in edges:
        preds[b].append(a)
        succ[a].append(b)
        indeg[b] += 1
    depth = [0] * n
    ready = [v for v in range(n) if indeg[v] == 0]
    seen = 0
    while ready:
        v = ready.pop()
        seen += 1
        depth[v] = 1 + max((depth[u] for u in preds[v]), default=-1)
        for w in succ[v]:
            indeg[w] -= 1
            if indeg[w] == 0:
                ready.append(w)
    assert seen == n, "cycle"
    return depth


def depths_bruteforce(pool):
    """depth(j) = max over earlier conflicting i of depth(i) + 1 (0 if none)."""
    d = []
    for j in range(len(pool)):
        d.append(max((d[i] + 1 for i in range(j) if conflicting(pool[i], pool[j])), default=0))
    return d


def literal_rank_rule(pool):
    """The five-step rule of PAPER.md:137-149 read literally (per-group ranks only,
    then max per transaction).  Exact only when every txn has <= 1 operation
    (DESIGN.md R-S1); kept to document the correction."""
    groups = defaultdict(list)
    for t, txn in enumerate(pool):
        for item, mode in _norm(txn).items():
            groups[item].append((t, mode))
    rank = [0] * len(pool)
    for item, ops in groups.items():
        r = 0
        for k, (t, mode) in enumerate(ops):
            if k == 0:
                r = 0
            elif mode == 'W' or ops[k - 1][1] == 'W':
                r = r + 1
            rank[t] = max(rank[t], r)
    return rank


def ksets(depth):
    out = defaultdict(list)
    for t, d in enumerate(depth):
        out[d].append(t)
    return [out[k] for k in range(max(depth) + 1)] if depth else []


def check_properties(pool, depth):
    """Property 1 (k-sets conflict-free) and Property 2 (each member of the k-set,
    k >= 1, conflicts with some member of the (k-1)-set)."""
    ks = ksets(depth)
    for k, members in enumerate(ks):
        for a, b in itertools.combinations(members, 2):
            if conflicting(pool[a], pool[b]):
                return False, f"P1: {a},{b} in {k}-set conflict"
        if k >= 1:
            for t in members:
                if not any(conflicting(pool[t], pool[u]) for u in ks[k - 1]):
                    return False, f"P2: {t} in {k}-set has no conflict in {k-1}-set"
    return True, ""


def linear_extensions(n, edges, limit=None):
    """Every topological order of the DAG (for tiny n)."""
    preds = [set() for _ in range(n)]
    for a, b in edges:
        preds[b].add(a)
    out = []
    order = []
    placed = [False] * n

    def rec():
        if limit is not None and len(out) >= limit:
            return
        if len(order) == n:
            out.append(list(order))
            return
        for v in range(n):
            if not placed[v] and all(placed[u] for u in preds[v]):
                placed[v] = True
                order.append(v)
                rec()
                order.pop()
                placed[v] = False

    rec()
    return out
