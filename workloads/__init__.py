"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module is the ONLY code both sides use.  It holds no arithmetic of the
method (no procedure, no footprint, no depth/rank, no lock key, no partition
map): it draws initial database images and transaction bulks from seeded
numpy generators, with the shapes and distributions of the paper's
benchmarks (App. E) as read in DESIGN.md §"Input recipe".

Everything is 0-based: warehouse w in [0, W), district d in [0, D), customer
c in [0, C), item i in [0, I) (i == I is the TPC-C "unused item" that makes a
NewOrder roll back), TM-1 s_id in [1, P] (TATP's 1-based id, kept because
sub_nbr is its 15-digit decimal string).

A bulk is the transaction signature SoA of PAPER.md:95 (<id, type, params>,
id implicit = submission order):
    type        u8[n]
    param_off   u32[n+1]   params of txn i are param_words[param_off[i]:param_off[i+1]]
    param_words u32[...]
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# --------------------------------------------------------------------------------------
# schemas and type ids (interface constants, mirrored by include/gputx.h)
# --------------------------------------------------------------------------------------
TPCB, TM1, TPCC, MICRO = 1, 2, 3, 4

TPCB_DEPOSIT = 0
TM1_GSD, TM1_GND, TM1_GAD, TM1_USD, TM1_UL, TM1_ICF, TM1_DCF = range(7)
TPCC_NEWORDER, TPCC_PAYMENT = 0, 1

# TATP standard mix, percent (GSD 35, GND 10, GAD 35, USD 2, UL 14, ICF 2, DCF 2)
TM1_MIX = (35, 10, 35, 2, 14, 2, 2)
# TPC-C NewOrder : Payment = 45 : 43 (the two-type subset of the standard mix)
TPCC_MIX = (45, 43)

# output record stride (bytes) per schema; layouts documented in include/gputx.h
OUT_STRIDE = {TPCB: 8, TM1: 40, TPCC: 200, MICRO: 4}


@dataclass
class Bulk:
    schema: int
    type: np.ndarray
    param_off: np.ndarray
    param_words: np.ndarray
    meta: dict = field(default_factory=dict)
    ts: np.ndarray | None = None     # global timestamps (u32, increasing); None: position order

    @property
    def n(self) -> int:
        return int(self.type.shape[0])

    def params(self, i: int) -> np.ndarray:
        return self.param_words[self.param_off[i]:self.param_off[i + 1]]

    def take(self, idx: np.ndarray, ts: np.ndarray | None = None) -> "Bulk":
        """The transactions at positions idx (increasing), optionally with timestamps."""
        idx = np.asarray(idx, np.int64)
        lens = (self.param_off[idx + 1].astype(np.int64) - self.param_off[idx])
        off = np.zeros(idx.size + 1, np.int64)
        np.cumsum(lens, out=off[1:])
        src = np.repeat(self.param_off[idx].astype(np.int64) - off[:-1], lens) + np.arange(off[-1])
        return Bulk(self.schema, self.type[idx].copy(), off.astype(np.uint32), self.param_words[src].copy(),
                    dict(self.meta), None if ts is None else np.asarray(ts, np.uint32))

    def slice(self, lo: int, hi: int) -> "Bulk":
        off = self.param_off[lo:hi + 1]
        return Bulk(self.schema, self.type[lo:hi].copy(), (off - off[0]).astype(np.uint32),
                    self.param_words[off[0]:off[-1]].copy(), dict(self.meta))


def _pack(schema: int, types: np.ndarray, rows: list[np.ndarray] | None = None,
          fixed: np.ndarray | None = None) -> Bulk:
    """Pack per-transaction parameter lists into the SoA signature arrays."""
    n = types.shape[0]
    if fixed is not None:                      # every txn has fixed.shape[1] words
        k = fixed.shape[1]
        off = (np.arange(n + 1, dtype=np.uint64) * k).astype(np.uint32)
        return Bulk(schema, types.astype(np.uint8), off, fixed.astype(np.uint32).reshape(-1))
    lens = np.fromiter((r.shape[0] for r in rows), dtype=np.uint64, count=n)
    off = np.zeros(n + 1, dtype=np.uint64)
    np.cumsum(lens, out=off[1:])
    words = np.concatenate(rows).astype(np.uint32) if n else np.zeros(0, np.uint32)
    return Bulk(schema, types.astype(np.uint8), off.astype(np.uint32), words)


def _rng(seed: int, tag: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([int(seed) & 0xFFFFFFFF, tag]))


def nurand(rng: np.random.Generator, A: int, x: int, y: int, size, C: int = 0) -> np.ndarray:
    """TPC-C 2.1.6 NURand(A, x, y) = (((rand[0,A] | rand[x,y]) + C) % (y-x+1)) + x."""
    a = rng.integers(0, A + 1, size=size, dtype=np.int64)
    b = rng.integers(x, y + 1, size=size, dtype=np.int64)
    return (((a | b) + C) % (y - x + 1)) + x


def zipf_keys(rng: np.random.Generator, theta: float, nkeys: int, size) -> np.ndarray:
    """Zipf(theta) over keys [0, nkeys): P(k) ~ 1/(k+1)^theta (theta=0 -> uniform)."""
    if theta <= 0.0:
        return rng.integers(0, nkeys, size=size, dtype=np.int64)
    w = 1.0 / np.power(np.arange(1, nkeys + 1, dtype=np.float64), theta)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    u = rng.random(size=size)
    return np.minimum(np.searchsorted(cdf, u, side="right"), nkeys - 1).astype(np.int64)


def bcd15(v: np.ndarray) -> np.ndarray:
    """15-digit zero-padded decimal string packed one digit per nibble (most
    significant digit in the high nibble): TATP's sub_nbr / numberx strings
    as a u64 (reading R-S24)."""
    v = np.asarray(v, dtype=np.uint64).copy()
    out = np.zeros(v.shape, dtype=np.uint64)
    for k in range(15):
        out |= (v % np.uint64(10)) << np.uint64(4 * k)
        v //= np.uint64(10)
    return out


def _split64(x: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    x = np.asarray(x, dtype=np.uint64)
    return (x & np.uint64(0xFFFFFFFF)).astype(np.uint32), (x >> np.uint64(32)).astype(np.uint32)


# --------------------------------------------------------------------------------------
# TPC-B (Ext TPC-B)
# --------------------------------------------------------------------------------------
@dataclass(frozen=True)
class TpcbDims:
    branches: int = 1
    tellers_per_branch: int = 10
    accounts_per_branch: int = 100_000

    @property
    def dims(self):
        return (self.branches, self.tellers_per_branch, self.accounts_per_branch, 0)


def tpcb_db(dims: TpcbDims) -> dict[str, np.ndarray]:
    """Initial TPC-B image: all balances 0 (Ext TPC-B)."""
    B, T, A = dims.branches, dims.tellers_per_branch, dims.accounts_per_branch
    return {
        "br_bal": np.zeros(B, np.int64),
        "tel_bal": np.zeros(B * T, np.int64),
        "acc_bal": np.zeros(B * A, np.int64),
    }


TPCB_WITHDRAW = 1


def tpcb_bulk(dims: TpcbDims, n: int, seed: int, remote_pct: float = 15.0,
              alpha: float = 0.0, zipf_theta: float = 0.0, home_range: tuple | None = None,
              withdraw_pct: float = 0.0) -> Bulk:
    """n deposit transactions, params [aid, tid, bid, delta(i32 as u32)].

    withdraw_pct > 0: that share are WITHDRAW [aid, tid, bid, amount] (type 1, SURVEY.md
    NEXT-4 / PAPER.md:441-443: a NON-two-phase type -- it debits, then aborts if the account
    went negative; always a local account), amount uniform in [1, 999999] cents.

    Branch: hot-branch alpha model (branch 0 w.p. alpha, else uniform)
    or Zipf(theta) over branches; teller uniform within the branch; account in the
    branch, or w.p. remote_pct% uniform in another branch (Ext TPC-B);
    delta uniform in [-999999, 999999] cents.
    """
    rng = _rng(seed, 0xB)
    B, T, A = dims.branches, dims.tellers_per_branch, dims.accounts_per_branch
    lo, hi = home_range if home_range is not None else (0, B)   # home branches (sharded generation)
    if zipf_theta > 0:
        bid = lo + zipf_keys(rng, zipf_theta, hi - lo, n)
    else:
        bid = rng.integers(lo, hi, size=n, dtype=np.int64)
        if alpha > 0:
            hot = rng.random(n) < alpha
            bid = np.where(hot, lo, bid)
    tid = bid * T + rng.integers(0, T, size=n, dtype=np.int64)
    abr = bid.copy()
    if B > 1 and remote_pct > 0:
        remote = rng.random(n) < remote_pct / 100.0
        other = rng.integers(0, B - 1, size=n, dtype=np.int64)
        other = np.where(other >= bid, other + 1, other)
        abr = np.where(remote, other, bid)
    aid = abr * A + rng.integers(0, A, size=n, dtype=np.int64)
    delta = rng.integers(-999_999, 1_000_000, size=n, dtype=np.int64)
    types = np.zeros(n, np.uint8)
    if withdraw_pct > 0:
        rw = _rng(seed, 0xBD)
        wd = rw.random(n) < withdraw_pct / 100.0
        types[wd] = TPCB_WITHDRAW
        aid = np.where(wd, bid * A + rw.integers(0, A, size=n, dtype=np.int64), aid)
        delta = np.where(wd, rw.integers(1, 1_000_000, size=n, dtype=np.int64), delta)
    fixed = np.stack([aid, tid, bid, delta.astype(np.int32).view(np.uint32).astype(np.int64)], axis=1)
    b = _pack(TPCB, types, fixed=fixed.astype(np.uint32))
    b.meta = dict(dims=dims.dims, seed=seed, remote_pct=remote_pct, alpha=alpha, zipf=zipf_theta,
                  withdraw_pct=withdraw_pct)
    return b


# --------------------------------------------------------------------------------------
# TM-1 / TATP (Ext TATP)
# --------------------------------------------------------------------------------------
@dataclass(frozen=True)
class Tm1Dims:
    subscribers: int = 1_000_000

    @property
    def dims(self):
        return (self.subscribers, 0, 0, 0)


def _random_subset_mask(rng, rows: int, k: int) -> np.ndarray:
    """For each row pick a uniform count in [1, k] and a uniform subset of that size
    of k slots; returns bool[rows, k]."""
    cnt = rng.integers(1, k + 1, size=rows)
    keys = rng.random((rows, k))
    order = np.argsort(keys, axis=1)
    rank = np.empty_like(order)
    np.put_along_axis(rank, order, np.arange(k)[None, :].repeat(rows, 0), axis=1)
    return rank < cnt[:, None]


def _letters(rng, size, nchar: int) -> np.ndarray:
    """nchar random upper-case ASCII letters packed little-endian into a u64."""
    out = np.zeros(size, np.uint64)
    for k in range(nchar):
        out |= rng.integers(65, 91, size=size).astype(np.uint64) << np.uint64(8 * k)
    return out


def tm1_db(dims: Tm1Dims, seed: int = 7) -> dict[str, np.ndarray]:
    """TATP population.  Row index s = s_id - 1; AI/SF rows at [s*4 + type-1];
    CF rows at [(s*4 + sf_type-1)*3 + start_time/8] with a liveness flag."""
    rng = _rng(seed, 0x7A7)
    P = dims.subscribers
    s_id = np.arange(1, P + 1, dtype=np.uint64)
    db = {
        "sub_nbr": bcd15(s_id),
        "sub_bits": rng.integers(0, 1 << 10, size=P).astype(np.uint16),     # bit_1 = bit 0
        "sub_hex": rng.integers(0, 1 << 40, size=P, dtype=np.int64).astype(np.uint64),
        "sub_byte2": rng.integers(0, 256, size=(P, 10)).astype(np.uint8),
        "sub_msc": rng.integers(0, 1 << 32, size=P, dtype=np.int64).astype(np.uint32),
        "sub_vlr": rng.integers(0, 1 << 32, size=P, dtype=np.int64).astype(np.uint32),
    }
    ai = _random_subset_mask(rng, P, 4).reshape(-1)
    db["ai_valid"] = ai.astype(np.uint8)
    db["ai_data1"] = rng.integers(0, 256, size=4 * P).astype(np.uint8)
    db["ai_data2"] = rng.integers(0, 256, size=4 * P).astype(np.uint8)
    db["ai_data3"] = _letters(rng, 4 * P, 3).astype(np.uint32)
    db["ai_data4"] = _letters(rng, 4 * P, 5)
    sf = _random_subset_mask(rng, P, 4).reshape(-1)
    db["sf_valid"] = sf.astype(np.uint8)
    db["sf_active"] = (rng.random(4 * P) < 0.85).astype(np.uint8)
    db["sf_error"] = rng.integers(0, 256, size=4 * P).astype(np.uint8)
    db["sf_data_a"] = rng.integers(0, 256, size=4 * P).astype(np.uint8)
    db["sf_data_b"] = _letters(rng, 4 * P, 5)
    # call forwarding: 0..3 rows per existing SF row, start_time subset of {0, 8, 16}
    cnt = rng.integers(0, 4, size=4 * P)
    keys = rng.random((4 * P, 3))
    order = np.argsort(keys, axis=1)
    rank = np.empty_like(order)
    np.put_along_axis(rank, order, np.arange(3)[None, :].repeat(4 * P, 0), axis=1)
    live = (rank < cnt[:, None]) & sf[:, None]
    db["cf_live"] = live.reshape(-1).astype(np.uint8)
    start = np.array([0, 8, 16], np.int64)[None, :]
    db["cf_end"] = (start + rng.integers(1, 9, size=(4 * P, 3))).reshape(-1).astype(np.uint8)
    db["cf_numberx"] = bcd15(rng.integers(0, 10**15, size=12 * P, dtype=np.int64).astype(np.uint64))
    return db


def tm1_bulk(dims: Tm1Dims, n: int, seed: int, dist: str = "nurand", mix=TM1_MIX,
             home_range: tuple | None = None) -> Bulk:
    """n TATP transactions.  s_id = NURand(A, 1, P) ("nurand", TATP standard with
    A = 65535 / 1048575 / 2097151 by P) or uniform in [1, P].

    Param words per type:
      GSD [s_id]                       GND [s_id, sf, st, et]
      GAD [s_id, ai]                   USD [s_id, sf, bit1, data_a]
      UL  [nbr_lo, nbr_hi, vlr]        ICF [nbr_lo, nbr_hi, sf, st, et, numx_lo, numx_hi]
      DCF [nbr_lo, nbr_hi, sf, st]
    UL/ICF/DCF carry the subscriber's sub_nbr string.
    """
    rng = _rng(seed, 0x7A1)
    lo, hi = home_range if home_range is not None else (0, dims.subscribers)   # subscribers lo+1..hi
    P = hi - lo
    if dist == "nurand":
        A = 65535 if P <= 1_000_000 else (1048575 if P <= 10_000_000 else 2097151)
        s_id = lo + nurand(rng, A, 1, P, n)
    elif dist == "uniform":
        s_id = lo + rng.integers(1, P + 1, size=n, dtype=np.int64)
    else:
        raise ValueError(dist)
    p = np.asarray(mix, np.float64)
    types = rng.choice(7, size=n, p=p / p.sum()).astype(np.uint8)
    sf = rng.integers(1, 5, size=n, dtype=np.int64)
    ai = rng.integers(1, 5, size=n, dtype=np.int64)
    st = rng.integers(0, 3, size=n, dtype=np.int64) * 8
    et_gnd = rng.integers(1, 25, size=n, dtype=np.int64)
    et_icf = st + rng.integers(1, 9, size=n, dtype=np.int64)
    bit1 = rng.integers(0, 2, size=n, dtype=np.int64)
    data_a = rng.integers(0, 256, size=n, dtype=np.int64)
    vlr = rng.integers(0, 1 << 32, size=n, dtype=np.int64)
    nlo, nhi = _split64(bcd15(s_id.astype(np.uint64)))
    xlo, xhi = _split64(bcd15(rng.integers(0, 10**15, size=n, dtype=np.int64).astype(np.uint64)))
    W = np.zeros((n, 7), np.int64)
    L = np.zeros(n, np.int64)
    t = types
    def put(mask, cols):
        idx = np.nonzero(mask)[0]
        for k, c in enumerate(cols):
            W[idx, k] = c[idx]
        L[idx] = len(cols)
    put(t == TM1_GSD, [s_id])
    put(t == TM1_GND, [s_id, sf, st, et_gnd])
    put(t == TM1_GAD, [s_id, ai])
    put(t == TM1_USD, [s_id, sf, bit1, data_a])
    put(t == TM1_UL, [nlo.astype(np.int64), nhi.astype(np.int64), vlr])
    put(t == TM1_ICF, [nlo.astype(np.int64), nhi.astype(np.int64), sf, st, et_icf,
                       xlo.astype(np.int64), xhi.astype(np.int64)])
    put(t == TM1_DCF, [nlo.astype(np.int64), nhi.astype(np.int64), sf, st])
    off = np.zeros(n + 1, np.int64)
    np.cumsum(L, out=off[1:])
    mask = np.arange(7)[None, :] < L[:, None]
    words = W[mask].astype(np.uint32)
    b = Bulk(TM1, types, off.astype(np.uint32), words)
    b.meta = dict(dims=dims.dims, seed=seed, dist=dist, root=(s_id - 1).astype(np.int64))
    return b


# --------------------------------------------------------------------------------------
# TPC-C NewOrder + Payment (Ext TPC-C)
# --------------------------------------------------------------------------------------
@dataclass(frozen=True)
class TpccDims:
    warehouses: int = 64
    districts: int = 10
    customers: int = 3000        # per district
    items: int = 100_000

    @property
    def dims(self):
        return (self.warehouses, self.districts, self.customers, self.items)

    @property
    def names(self) -> int:      # distinct C_LAST codes
        return min(1000, self.customers)


def tpcc_db(dims: TpccDims, seed: int = 11) -> dict[str, np.ndarray]:
    """TPC-C initial image (Ext TPC-C 4.3.3.1, numeric columns only; DESIGN.md R-S24/S25).

    Row layouts: district [w*D + d], customer [(w*D + d)*C + c], stock [w*I + i].
    C_LAST is the 0..999 syllable code: c < 1000 -> c, else NURand(255, 0, 999)
    (clipped to the name range for tiny test dimensions).
    """
    rng = _rng(seed, 0xCC)
    W, D, C, I = dims.warehouses, dims.districts, dims.customers, dims.items
    NC = W * D * C
    nm = dims.names
    last = nurand(rng, 255, 0, 999, NC) % nm
    cidx = np.tile(np.arange(C), W * D)
    last = np.where(cidx < nm, cidx, last)
    return {
        "w_ytd": np.full(W, D * 3_000_000, np.int64),      # 30,000,000 at D = 10
        "w_tax": rng.integers(0, 2001, size=W).astype(np.int32),
        "d_ytd": np.full(W * D, 3_000_000, np.int64),
        "d_tax": rng.integers(0, 2001, size=W * D).astype(np.int32),
        "d_next_o_id": np.full(W * D, 3001, np.uint32),
        "c_balance": np.full(NC, -1000, np.int64),
        "c_ytd_payment": np.full(NC, 1000, np.int64),
        "c_payment_cnt": np.ones(NC, np.uint32),
        "c_discount": rng.integers(0, 5001, size=NC).astype(np.int32),
        "c_credit": (rng.random(NC) < 0.10).astype(np.uint8),      # 1 = "BC"
        "c_last": last.astype(np.uint16),
        "c_first": rng.integers(0, 1 << 62, size=NC, dtype=np.int64).astype(np.uint64),
        "i_price": rng.integers(100, 10001, size=I).astype(np.int32),
        "i_original": (rng.random(I) < 0.10).astype(np.uint8),
        "s_quantity": rng.integers(10, 101, size=W * I).astype(np.int32),
        "s_ytd": np.zeros(W * I, np.int64),
        "s_order_cnt": np.zeros(W * I, np.uint32),
        "s_remote_cnt": np.zeros(W * I, np.uint32),
        "s_original": (rng.random(W * I) < 0.10).astype(np.uint8),
    }


def tpcc_bulk(dims: TpccDims, n: int, seed: int, mix=TPCC_MIX, remote_line_pct: float = 1.0,
              remote_pay_pct: float = 15.0, byname_pct: float = 60.0, rbk_pct: float = 1.0,
              home_w: np.ndarray | None = None) -> Bulk:
    """NewOrder [w, d, c, ol_cnt, (i, supply_w, qty) x ol_cnt] and
    Payment [w, d, cw, cd, by_name, c_or_last, h_amount] (Ext TPC-C 2.4.1, 2.5.1).
    home_w optionally fixes each transaction's home warehouse (sharded generation)."""
    rng = _rng(seed, 0xC1)
    W, D, C, I = dims.warehouses, dims.districts, dims.customers, dims.items
    p = np.asarray(mix, np.float64)
    types = rng.choice(2, size=n, p=p / p.sum()).astype(np.uint8)
    w = rng.integers(0, W, size=n, dtype=np.int64) if home_w is None else np.asarray(home_w, np.int64)
    d = rng.integers(0, D, size=n, dtype=np.int64)
    # NewOrder fields
    c_no = nurand(rng, 1023, 0, C - 1, n) if C > 1 else np.zeros(n, np.int64)
    ol_cnt = rng.integers(5, 16, size=n, dtype=np.int64)
    rbk = rng.random(n) < rbk_pct / 100.0
    items = nurand(rng, 8191, 0, I - 1, (n, 15)) if I > 1 else np.zeros((n, 15), np.int64)
    last_pos = ol_cnt - 1
    items[np.arange(n), last_pos] = np.where(rbk, I, items[np.arange(n), last_pos])
    rl = (rng.random((n, 15)) < remote_line_pct / 100.0) & (W > 1)
    other = rng.integers(0, max(W - 1, 1), size=(n, 15), dtype=np.int64)
    other = np.where(other >= w[:, None], other + 1, other)
    supply = np.where(rl, other, w[:, None])
    qty = rng.integers(1, 11, size=(n, 15), dtype=np.int64)
    # Payment fields
    rp = (rng.random(n) < remote_pay_pct / 100.0) & (W > 1)
    ow = rng.integers(0, max(W - 1, 1), size=n, dtype=np.int64)
    ow = np.where(ow >= w, ow + 1, ow)
    cw = np.where(rp, ow, w)
    cd = np.where(rp, rng.integers(0, D, size=n, dtype=np.int64), d)
    byname = rng.random(n) < byname_pct / 100.0
    last = nurand(rng, 255, 0, 999, n) % dims.names
    c_pay = nurand(rng, 1023, 0, C - 1, n) if C > 1 else np.zeros(n, np.int64)
    c_or_last = np.where(byname, last, c_pay)
    h = rng.integers(100, 500_001, size=n, dtype=np.int64)

    is_no = types == TPCC_NEWORDER
    L = np.where(is_no, 4 + 3 * ol_cnt, 7)
    off = np.zeros(n + 1, np.int64)
    np.cumsum(L, out=off[1:])
    Wm = np.zeros((n, 49), np.int64)
    Wm[:, 0] = w
    Wm[:, 1] = d
    Wm[:, 2] = np.where(is_no, c_no, cw)
    Wm[:, 3] = np.where(is_no, ol_cnt, cd)
    lines = np.stack([items, supply, qty], axis=2).reshape(n, 45)
    pay = np.stack([byname.astype(np.int64), c_or_last, h], axis=1)
    Wm[:, 4:49] = np.where(is_no[:, None], lines, np.pad(pay, ((0, 0), (0, 42))))
    mask = np.arange(49)[None, :] < L[:, None]
    words = Wm[mask].astype(np.uint32)
    b = Bulk(TPCC, types, off.astype(np.uint32), words)
    b.meta = dict(dims=dims.dims, seed=seed)
    return b


# --------------------------------------------------------------------------------------
# Micro benchmark (§6.1): N tuples; a bulk of single-tuple transactions
# spread evenly over T types (the branches of the combined switch kernel); each reads
# its tuple, computes (x units of 100 sin evaluations, the procedure's cost) and writes
# the result back.  Skew: the first tuple with probability alpha, the others uniformly
# ("transactions acquire the first lock with a probability of alpha").
# --------------------------------------------------------------------------------------
@dataclass(frozen=True)
class MicroDims:
    tuples: int = 8_000_000       # PAPER.md:258 "the number of tuples is fixed to be eight millions"
    types: int = 8                # T (default 8)
    x: int = 16                   # computation units (default 16)

    @property
    def dims(self):
        return (self.tuples, self.types, self.x, 0)


def micro_db(dims: MicroDims, seed: int = 7) -> dict[str, np.ndarray]:
    """Tuple values: f32 uniform in [-0.5, 0.5), stored as their u32 bit patterns."""
    rng = _rng(seed, 0x3C0)
    v = (rng.random(dims.tuples, dtype=np.float32) - np.float32(0.5)).astype(np.float32)
    return {"tuple": v.view(np.uint32).copy()}


def micro_bulk(dims: MicroDims, n: int, seed: int, alpha: float = 0.0, theta: float = 0.0,
               types: int | None = None) -> Bulk:
    """n transactions [tuple id]; type uniform over the T types ("transactions are evenly
    assigned with a transaction type"); tuple 0 w.p. alpha, else uniform (or Zipf theta)."""
    rng = _rng(seed, 0x3C1)
    T = dims.types if types is None else types
    t = rng.integers(0, T, size=n).astype(np.uint8)
    if theta > 0.0:
        tup = zipf_keys(rng, theta, dims.tuples, n)
    else:
        tup = rng.integers(0, dims.tuples, size=n, dtype=np.int64)
    if alpha > 0.0:
        tup = np.where(rng.random(n) < alpha, 0, tup)
    b = _pack(MICRO, t, fixed=tup.reshape(n, 1))
    b.meta = dict(dims=dims.dims, seed=seed, alpha=alpha, root=tup.astype(np.int64))
    return b


def make_db(schema: int, dims, seed: int = 7) -> dict[str, np.ndarray]:
    if schema == TPCB:
        return tpcb_db(dims)
    if schema == TM1:
        return tm1_db(dims, seed)
    if schema == TPCC:
        return tpcc_db(dims, seed)
    if schema == MICRO:
        return micro_db(dims, seed)
    raise ValueError(schema)


def make_bulk(schema: int, dims, n: int, seed: int, **kw) -> Bulk:
    if schema == TPCB:
        return tpcb_bulk(dims, n, seed, **kw)
    if schema == TM1:
        return tm1_bulk(dims, n, seed, **kw)
    if schema == TPCC:
        return tpcc_bulk(dims, n, seed, **kw)
    if schema == MICRO:
        return micro_bulk(dims, n, seed, **kw)
    raise ValueError(schema)


# --------------------------------------------------------------------------------------
# Sharding by root key: TPC-B branch, TPC-C warehouse, TM-1 subscriber.
# Shard r of G owns roots x with x*G // R == r.  These only select which rank submits a
# transaction (its "home"); the engine splits cross-shard transactions itself.

def n_roots(schema: int, dims) -> int:
    return int(dims.dims[0])


def home_roots(bulk: Bulk) -> np.ndarray:
    """Home root key of every transaction (TPC-B teller's branch, TPC-C w, TM-1 s_id-1)."""
    first = bulk.param_off[:-1].astype(np.int64)
    if bulk.schema == TPCB:
        return bulk.param_words[first + 2].astype(np.int64)
    if bulk.schema == TPCC:
        return bulk.param_words[first].astype(np.int64)
    return np.asarray(bulk.meta["root"], np.int64)


def shard_of(root: np.ndarray, G: int, R: int) -> np.ndarray:
    return (np.asarray(root, np.int64) * G) // R


def split_home(bulk: Bulk, dims, G: int) -> list[Bulk]:
    """Per shard, its home transactions with their global timestamps (bulk positions)."""
    owner = shard_of(home_roots(bulk), G, n_roots(bulk.schema, dims))
    out = []
    for r in range(G):
        idx = np.nonzero(owner == r)[0]
        out.append(bulk.take(idx, ts=idx.astype(np.uint32)))
    return out


def shard_rows(schema: int, dims, G: int, r: int) -> dict:
    """Row ranges [lo, hi) of each root-partitioned column owned by shard r (columns
    not listed are read-only and replicated)."""
    R = n_roots(schema, dims)
    lo = (r * R + G - 1) // G
    hi = ((r + 1) * R + G - 1) // G
    d = dims.dims
    if schema == TPCB:
        return {"branch": (lo, hi), "teller": (lo * d[1], hi * d[1]), "account": (lo * d[2], hi * d[2])}
    if schema == TPCC:
        D, C, I = d[1], d[2], d[3]
        return {"warehouse": (lo, hi), "district": (lo * D, hi * D), "customer": (lo * D * C, hi * D * C),
                "stock": (lo * I, hi * I)}
    return {"subscriber": (lo, hi)}


def scaled_dims(schema: int, dims, G: int):
    """The global dimensions of a weak-scaled run: G times the root keys of `dims`."""
    if schema == TPCB:
        return TpcbDims(dims.branches * G, dims.tellers_per_branch, dims.accounts_per_branch)
    if schema == TM1:
        return Tm1Dims(dims.subscribers * G)
    return TpccDims(dims.warehouses * G, dims.districts, dims.customers, dims.items)


def shard_bulk(schema: int, gdims, n: int, seed: int, r: int, G: int, **kw) -> Bulk:
    """Shard r's n home transactions of a G-shard run over the global dims: home roots
    drawn in r's root range with the single-GPU distribution, remote accounts / supply
    warehouses / customers over all roots; global ts = i*G + r (interleaved, unique)."""
    R = n_roots(schema, gdims)
    lo, hi = (r * R + G - 1) // G, ((r + 1) * R + G - 1) // G
    s = seed * 1009 + r
    if schema == TPCB:
        b = tpcb_bulk(gdims, n, s, home_range=(lo, hi), **kw)
    elif schema == TM1:
        b = tm1_bulk(gdims, n, s, home_range=(lo, hi), **kw)
    else:
        w = np.random.default_rng(np.random.SeedSequence([s, 0x5EA])).integers(lo, hi, size=n, dtype=np.int64)
        b = tpcc_bulk(gdims, n, s, home_w=w, **kw)
    b.ts = (np.arange(n, dtype=np.int64) * G + r).astype(np.uint32)
    return b
