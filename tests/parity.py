"""Helpers for GPU-vs-oracle parity tests (imported by tests only)."""
import numpy as np

import oracle
import workloads as W


def gpu_db(schema, dims, image, max_bulk, **kw):
    from paper_1103_3105_b200 import Database
    return Database(schema, dims.dims, max_bulk, image, **kw)


def compare(schema, ref, db, image, label=""):
    """Bit-exact comparison of final image, status, outputs and insert tables."""
    got = db.read_image(image)
    for k in image:
        a, b = ref.db[k], got[k]
        if not np.array_equal(a, b):
            bad = np.nonzero(a.reshape(-1) != b.reshape(-1))[0]
            raise AssertionError(f"{label}: column {k} differs at {bad[:10]} ({len(bad)} cells): "
                                 f"oracle {a.reshape(-1)[bad[:5]]} gpu {b.reshape(-1)[bad[:5]]}")
    st, out = db.read_results()
    if not np.array_equal(st, ref.status):
        bad = np.nonzero(st != ref.status)[0]
        raise AssertionError(f"{label}: status differs at {bad[:10]} ({len(bad)})")
    if not np.array_equal(out, ref.out):
        bad = np.nonzero((out != ref.out).any(axis=1))[0]
        raise AssertionError(f"{label}: output differs at txns {bad[:10]} ({len(bad)}): "
                             f"oracle {ref.out[bad[0]][:24]} gpu {out[bad[0]][:24]}")
    ins = db.inserts()
    for tab, cols in ref.inserts.items():
        for c, a in cols.items():
            b = ins[tab][c]
            if not np.array_equal(a, b):
                raise AssertionError(f"{label}: insert {tab}.{c} differs (oracle {len(a)} rows, gpu {len(b)})")


def run_both(schema, dims, image, bulks, strategy, db=None, max_bulk=None, **kw):
    """Execute `bulks` in sequence on the oracle and the GPU; compare after each
    (insert tables accumulate across bulks on both sides)."""
    own = db is None
    if own:
        db = gpu_db(schema, dims, image, max_bulk or max(1, max(b.n for b in bulks)), **kw)
    cur = image
    ts = 0
    stats = []
    acc = None
    try:
        for k, b in enumerate(bulks):
            ref = oracle.run(schema, dims.dims, cur, b, first_ts=ts)
            if acc is None:
                acc = ref.inserts
            else:
                acc = {t: {c: np.concatenate([acc[t][c], ref.inserts[t][c]]) for c in cols}
                       for t, cols in ref.inserts.items()}
            first = db.submit(b)
            assert first == ts
            stats.append(db.execute(strategy))
            compare(schema, oracle.Result(ref.db, ref.status, ref.out, acc), db, image,
                    label=f"{strategy} bulk {k}")
            cur = ref.db
            ts += b.n
    finally:
        if own:
            db.close()
    return stats


def compare_sharded(schema, dims, ref, dbs, homes, image, label=""):
    """Sharded run vs the oracle: every shard's owned rows, untouched foreign rows, home
    results in submission order, and the union of the insert tables (each shard's rows
    in ts order, the union compared as a multiset)."""
    G = len(dbs)
    R = W.n_roots(schema, dims)
    for r, db in enumerate(dbs):
        lo = (r * R + G - 1) // G
        hi = ((r + 1) * R + G - 1) // G
        got = db.read_image(image)
        for k in image:
            a, b, init = ref.db[k].reshape(-1), got[k].reshape(-1), np.asarray(image[k]).reshape(-1)
            if schema == W.TPCC and k.startswith("i_"):
                assert np.array_equal(a, b), f"{label}: replicated {k} changed on shard {r}"
                continue
            assert a.size % R == 0, k
            f = a.size // R
            own = slice(lo * f, hi * f)
            if not np.array_equal(a[own], b[own]):
                bad = np.nonzero(a[own] != b[own])[0] + lo * f
                raise AssertionError(f"{label}: shard {r} column {k} differs at {bad[:10]} ({len(bad)} cells): "
                                     f"oracle {a[bad[:5]]} gpu {b[bad[:5]]}")
            rest = np.ones(a.size, bool)
            rest[own] = False
            assert np.array_equal(b[rest], init[rest]), f"{label}: shard {r} wrote foreign rows of {k}"
        st, out = db.read_results()
        idx = homes[r].ts.astype(np.int64)
        if not np.array_equal(st, ref.status[idx]):
            bad = np.nonzero(st != ref.status[idx])[0]
            raise AssertionError(f"{label}: shard {r} status differs at {bad[:10]}")
        if not np.array_equal(out, ref.out[idx]):
            bad = np.nonzero((out != ref.out[idx]).any(axis=1))[0]
            raise AssertionError(f"{label}: shard {r} output differs at home txns {bad[:10]} ({len(bad)}): "
                                 f"oracle {ref.out[idx][bad[0]][:24]} gpu {out[bad[0]][:24]}")
    ins = [db.inserts() for db in dbs]
    for tab, cols in ref.inserts.items():
        names = list(cols)
        want = np.stack([cols[c].astype(np.int64) for c in names], axis=1)
        have = np.concatenate([np.stack([i[tab][c].astype(np.int64) for c in names], axis=1) for i in ins])
        assert want.shape == have.shape, f"{label}: insert {tab}: oracle {want.shape[0]} rows, gpu {have.shape[0]}"
        ow = np.lexsort(want.T[::-1])
        oh = np.lexsort(have.T[::-1])
        assert np.array_equal(want[ow], have[oh]), f"{label}: insert table {tab} differs"
