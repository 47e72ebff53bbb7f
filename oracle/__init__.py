"""GPUTx oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow, single-threaded CPU implementation of what the bulk-execution hot
path computes (Definition 1): see oracle.c for the serial executor,
the conflict footprint and the streaming depth recurrence, and depgraph.py for
the small-pool graph algorithms of §4 / Appendix B.

May be imported only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg.  The product package
(paper_1103_3105_b200) never imports it, and it never imports the product.

Parity pins: tests/test_oracle_*.py (no function here is "parity unpinned").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

TPCB, TM1, TPCC, MICRO = 1, 2, 3, 4

# column order of oracle.c per schema
COLS = {
    TPCB: ["br_bal", "tel_bal", "acc_bal"],
    TM1: ["sub_nbr", "sub_bits", "sub_hex", "sub_byte2", "sub_msc", "sub_vlr",
          "ai_valid", "ai_data1", "ai_data2", "ai_data3", "ai_data4",
          "sf_valid", "sf_active", "sf_error", "sf_data_a", "sf_data_b",
          "cf_live", "cf_end", "cf_numberx"],
    TPCC: ["w_ytd", "w_tax", "d_ytd", "d_tax", "d_next_o_id", "c_balance", "c_ytd_payment",
           "c_payment_cnt", "c_discount", "c_credit", "c_last", "c_first", "i_price",
           "i_original", "s_quantity", "s_ytd", "s_order_cnt", "s_remote_cnt", "s_original"],
    MICRO: ["tuple"],
}

# insert tables: (table, [(column, dtype)], rows-per-txn bound)
INSERTS = {
    TPCB: [("history", [("h_tid", np.uint32), ("h_bid", np.uint32), ("h_aid", np.uint32),
                        ("h_delta", np.int32), ("h_ts", np.uint32)], 1)],
    TM1: [],
    MICRO: [],
    TPCC: [("order", [("o_id", np.uint32), ("o_d", np.uint32), ("o_w", np.uint32), ("o_c", np.uint32),
                      ("o_entry_d", np.uint32), ("o_ol_cnt", np.uint32), ("o_all_local", np.uint32)], 1),
           ("new_order", [("no_o_id", np.uint32), ("no_d", np.uint32), ("no_w", np.uint32)], 1),
           ("order_line", [("ol_o_id", np.uint32), ("ol_d", np.uint32), ("ol_w", np.uint32),
                           ("ol_number", np.uint32), ("ol_i_id", np.uint32), ("ol_supply_w", np.uint32),
                           ("ol_quantity", np.uint32), ("ol_amount", np.int32)], 15),
           ("history", [("h_c", np.uint32), ("h_cd", np.uint32), ("h_cw", np.uint32), ("h_d", np.uint32),
                        ("h_w", np.uint32), ("h_date", np.uint32), ("h_amount", np.int32)], 1)],
}

OUT_STRIDE = {TPCB: 8, TM1: 40, TPCC: 200, MICRO: 4}


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain -O2, single-threaded)."""
    with _lock:
        if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            tmp = _LIB + f".tmp{os.getpid()}"
            # -ffp-contract=off: the micro benchmark's float procedure is evaluated exactly
            # as written (fmaf where the text says fma, separate rounding elsewhere)
            subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared", "-o", tmp, _SRC,
                                   "-lm"])
            os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        lib.orc_run.argtypes = [ctypes.c_int, P, P, ctypes.c_uint64, P, P, P, ctypes.c_uint64, P, P, P, P]
        lib.orc_run.restype = ctypes.c_int
        lib.orc_footprint.argtypes = [ctypes.c_int, P, P, ctypes.c_uint64, P, P, P, P, P, P, ctypes.c_uint64,
                                      ctypes.c_int]
        lib.orc_footprint.restype = ctypes.c_int64
        lib.orc_run_order.argtypes = [ctypes.c_int, P, P, ctypes.c_uint64, P, P, P, ctypes.c_uint64, P, P, P, P, P]
        lib.orc_run_order.restype = ctypes.c_int
        lib.orc_depths.argtypes = [ctypes.c_uint64, P, P, P, P]
        lib.orc_depths.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags.c_contiguous
    return a.ctypes.data


def _ptrs(arrs) -> ctypes.Array:
    return (ctypes.c_void_p * max(1, len(arrs)))(*[_ptr(a) for a in arrs])


def _dims(dims) -> np.ndarray:
    d = np.zeros(4, np.uint32)
    d[:len(dims)] = dims
    return d


class Result:
    """Outcome of serial execution: final db image, status u8[n], out u8[n, stride], inserts."""

    def __init__(self, db, status, out, inserts):
        self.db, self.status, self.out, self.inserts = db, status, out, inserts


def run(schema: int, dims, db: dict, bulk, first_ts: int = 0, order=None) -> Result:
    """Definition 1: execute `bulk` serially in ts order on a COPY of `db`.  With `order`
    (a permutation of range(n)): serially in that order, each transaction keeping its own
    ts (orc_run_order; the witness replay of the relaxed strategies)."""
    lib = _load()
    work = {k: np.ascontiguousarray(v).copy() for k, v in db.items()}
    cols = [work[k] for k in COLS[schema]]
    n = bulk.n
    stride = OUT_STRIDE[schema]
    status = np.zeros(n, np.uint8)
    out = np.zeros((n, stride), np.uint8)
    ins_cols, ins_tabs = [], []
    for tab, cl, per in INSERTS[schema]:
        arrs = [np.zeros(max(1, n * per), dt) for _, dt in cl]
        ins_cols += arrs
        ins_tabs.append((tab, cl, arrs))
    nrows = np.zeros(max(1, len(ins_tabs)), np.uint64)
    tp = np.ascontiguousarray(bulk.type, np.uint8)
    po = np.ascontiguousarray(bulk.param_off, np.uint32)
    pw = np.ascontiguousarray(bulk.param_words, np.uint32)
    if pw.size == 0:
        pw = np.zeros(1, np.uint32)
    dm = _dims(dims)
    t0 = time.perf_counter()
    if order is None:
        rc = lib.orc_run(schema, _ptr(dm), _ptrs(cols), n, _ptr(tp), _ptr(po), _ptr(pw), first_ts,
                         _ptr(status), _ptr(out), _ptrs(ins_cols), _ptr(nrows))
    else:
        od = np.ascontiguousarray(order, np.uint32)
        if od.shape != (n,) or not np.array_equal(np.sort(od), np.arange(n, dtype=np.uint32)):
            raise ValueError("order must be a permutation of range(n)")
        rc = lib.orc_run_order(schema, _ptr(dm), _ptrs(cols), n, _ptr(tp), _ptr(po), _ptr(pw), first_ts,
                               _ptr(od if n else np.zeros(1, np.uint32)), _ptr(status), _ptr(out),
                               _ptrs(ins_cols), _ptr(nrows))
    secs = time.perf_counter() - t0
    if rc != 0:
        raise RuntimeError(f"orc_run failed: {rc}")
    inserts = {}
    for k, (tab, cl, arrs) in enumerate(ins_tabs):
        m = int(nrows[k])
        inserts[tab] = {name: a[:m].copy() for (name, _), a in zip(cl, arrs)}
    r = Result(work, status, out, inserts)
    r.seconds = secs          # time of the serial loop alone (one host core)
    return r


def footprint(schema: int, dims, db: dict, bulk, add_rule: bool = False):
    """(ops_off u64[n+1], items u64[m], modes u8[m]) — basic operations per txn.
    modes: 0 read, 1 write, 2 add (only with add_rule: TPC-B teller/branch balances,
    TPC-C W_YTD/D_YTD, which are only incremented and never read by an output)."""
    lib = _load()
    cols = [np.ascontiguousarray(db[k]) for k in COLS[schema]]
    n = bulk.n
    cap = 16 * max(1, n)
    ops_off = np.zeros(n + 1, np.uint64)
    items = np.zeros(cap, np.uint64)
    modes = np.zeros(cap, np.uint8)
    tp = np.ascontiguousarray(bulk.type, np.uint8)
    po = np.ascontiguousarray(bulk.param_off, np.uint32)
    pw = np.ascontiguousarray(bulk.param_words, np.uint32)
    if pw.size == 0:
        pw = np.zeros(1, np.uint32)
    m = lib.orc_footprint(schema, _ptr(_dims(dims)), _ptrs(cols), n, _ptr(tp), _ptr(po), _ptr(pw),
                          _ptr(ops_off), _ptr(items), _ptr(modes), cap, int(add_rule))
    if m < 0:
        raise RuntimeError("footprint capacity")
    return ops_off, items[:m].copy(), modes[:m].copy()


def depths_from_ops(ops_off: np.ndarray, items: np.ndarray, modes: np.ndarray) -> np.ndarray:
    """Streaming depth recurrence (oracle.c orc_depths) on an explicit op list."""
    lib = _load()
    n = ops_off.shape[0] - 1
    ops_off = np.ascontiguousarray(ops_off, np.uint64)
    items = np.ascontiguousarray(items, np.uint64)
    modes = np.ascontiguousarray(modes, np.uint8)
    if items.size == 0:
        items = np.zeros(1, np.uint64)
        modes = np.zeros(1, np.uint8)
    out = np.zeros(max(1, n), np.uint32)
    if lib.orc_depths(n, _ptr(ops_off), _ptr(items), _ptr(modes), _ptr(out)) != 0:
        raise RuntimeError("orc_depths")
    return out[:n]


def depths(schema: int, dims, db: dict, bulk, add_rule: bool = False) -> np.ndarray:
    """T-dependency-graph depth of every transaction of `bulk` against `db`
    (add_rule: two increments of one item do not conflict)."""
    return depths_from_ops(*footprint(schema, dims, db, bulk, add_rule))


def run_sequence(schema: int, dims, db: dict, bulk, order, first_ts: int = 0) -> Result:
    """Execute the transactions of `bulk` one at a time in the given ORDER (a
    permutation of range(n)), each keeping its own timestamp first_ts + i.
    Used by the every-linear-extension brute force: status/out are indexed by
    the original transaction, insert rows appear in execution order."""
    work = {k: np.ascontiguousarray(v).copy() for k, v in db.items()}
    n = bulk.n
    stride = OUT_STRIDE[schema]
    status = np.zeros(n, np.uint8)
    out = np.zeros((n, stride), np.uint8)
    inserts = {tab: {c: [] for c, _ in cl} for tab, cl, _ in INSERTS[schema]}
    for i in order:
        one = bulk.slice(int(i), int(i) + 1)
        r = run(schema, dims, work, one, first_ts=first_ts + int(i))
        work = r.db
        status[i] = r.status[0]
        out[i] = r.out[0]
        for tab, cols in r.inserts.items():
            for c, a in cols.items():
                inserts[tab][c].append(a)
    ins = {}
    for tab, cl, _ in INSERTS[schema]:
        ins[tab] = {c: (np.concatenate(inserts[tab][c]) if inserts[tab][c] else np.zeros(0, dt))
                    for c, dt in cl}
    return Result(work, status, out, ins)


# ---------------------------------------------------------------------------------------
# Strategy chooser: Algorithm 1, PAPER.md:416-437 (Appendix D,
# "Choosing the suitable execution strategy"), on the structural parameters of the
# T-dependency graph listed at PAPER.md:408-413.
# ---------------------------------------------------------------------------------------
def cross_partition(schema: int, dims, bulk, status: np.ndarray) -> np.ndarray:
    """bool[n]: the transaction accesses more than one PART partition (PAPER.md:413, 430:
    "cross-partition transactions").  Partitions (DESIGN.md R-S10 / R-S20): TPC-B branch,
    TPC-C warehouse, TM-1 128 subscribers (a TM-1 transaction touches one subscriber).
    Accesses are those the procedure performs in the serial run: a transaction that
    aborts in its first phase (TPC-C NewOrder with an unused item, by-name Payment
    with no such customer) touches only its home partition."""
    n = bulk.n
    out = np.zeros(n, bool)
    po = bulk.param_off.astype(np.int64)
    pw = bulk.param_words
    for i in range(n):
        p = pw[po[i]:po[i + 1]]
        if schema == TPCB:
            # deposit [aid, tid, bid, delta]; accounts per branch = dims[2]
            out[i] = int(p[0]) // int(dims[2]) != int(p[2])
        elif schema == TPCC and status[i] == 0:
            w = int(p[0])
            if bulk.type[i] == 0:      # NewOrder [w, d, c, ol_cnt, (i, supply_w, qty) x ol_cnt]
                out[i] = any(int(p[5 + 3 * l]) != w for l in range(int(p[3])))
            else:                      # Payment [w, d, cw, cd, by_name, c_or_last, h_amount]
                out[i] = int(p[2]) != w
    return out


def choose_strategy(w0: int, d: int, c: int, w0_bar: int, d_bar: int, c_bar: int) -> str:
    """Algorithm 1, line by line."""
    if w0 >= w0_bar:                  # 2: if w0 >= w0_bar then
        return "kset"                 # 3:   return K-SET
    if c <= c_bar or d >= d_bar:      # 7: if c <= c_bar or d >= d_bar then
        return "part"                 # 8:   return PART
    return "tpl"                      # 10: return TPL


def structure(schema: int, dims, db: dict, bulk, add_rule: bool = False) -> dict:
    """w0 = |0-set|, d = depth of the T-dependency graph, c = cross-partition
    transactions of `bulk` against `db`."""
    dep = depths(schema, dims, db, bulk, add_rule)
    st = run(schema, dims, db, bulk).status
    return {"w0": int((dep == 0).sum()), "d": int(dep.max()) if bulk.n else 0,
            "c": int(cross_partition(schema, dims, bulk, st).sum())}
