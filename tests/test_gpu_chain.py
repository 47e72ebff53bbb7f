"""K-SET chain executor (TPC-B; DESIGN.md §4 "Chain owners", "Deposit runs"): a warp per
branch chain executes the chain's members in k-set order; runs of deposits on distinct
accounts with no cross-chain waiter but the first execute lane-parallel.  Bulks built to
break the runs every way -- repeated accounts inside a chain (few accounts per branch),
cross-chain links (remote accounts), WITHDRAWs (non-two-phase, undo on abort), random
per-transaction delays -- must give the oracle's serial result (Definition 1)
element by element."""
import os

import pytest

import oracle
import workloads as W
from tests.parity import compare, gpu_db

pytestmark = pytest.mark.gpu

STAT_CHAIN = 16           # GPUTX_STAT_KSET_CHAIN
JITTER = 1024             # GPUTX_KSET_DIAG: random 0..2 us sleep before every transaction

CASES = {
    "dup_accounts": (W.TpcbDims(8, 10, 40), 20_000, dict(remote_pct=0.0)),
    "remote_heavy": (W.TpcbDims(16, 10, 200), 30_000, dict(remote_pct=60.0)),
    "withdraw_mix": (W.TpcbDims(8, 10, 100), 20_000, dict(withdraw_pct=30.0, remote_pct=15.0)),
    "hot": (W.TpcbDims(32, 10, 5000), 50_000, dict(remote_pct=15.0, alpha=0.5)),
    "wide": (W.TpcbDims(1000, 10, 1000), 100_000, dict(remote_pct=15.0)),
}


def _open(dims, image, n, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return gpu_db(W.TPCB, dims, image, n)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("jitter", [False, True])
@pytest.mark.parametrize("runs", [True, False])
def test_chain_executor_parity(case, jitter, runs):
    dims, n, kw = CASES[case]
    image = W.make_db(W.TPCB, dims, seed=1)
    bulk = W.make_bulk(W.TPCB, dims, n, seed=5, **kw)
    ref = oracle.run(W.TPCB, dims.dims, image, bulk)
    env = {"GPUTX_KSET_DIAG": str(JITTER)} if jitter else {}
    if not runs:
        env["GPUTX_CHAIN_RUNS"] = "0"
    db = _open(dims, image, n, env)
    try:
        for rep in range(2 if jitter else 3):
            db.reset()
            db.submit(bulk)
            st = db.execute("kset")
            assert st["flags"] & STAT_CHAIN, "the chain executor ran"
            compare(W.TPCB, ref, db, image, label=f"chain {case} jitter {jitter} rep {rep}")
    finally:
        db.close()
