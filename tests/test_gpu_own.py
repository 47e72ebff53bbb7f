"""K-SET with owner-local rounds (DESIGN.md §4 "Owner-local rounds"): every warp executes
the k-sets of its own transactions in increasing k (Property 1 inside a k-set, PAPER.md:
123-125; §5.3), waiting only for cross-warp predecessors.  The result must be the serial
one (Definition 1) whatever the owner map, the grid and the timing; every run
is compared with the oracle element by element."""
import os

import pytest

import oracle
import workloads as W
from tests.parity import compare, gpu_db

pytestmark = pytest.mark.gpu

STAT_OWNER = 4            # GPUTX_STAT_KSET_OWNER
JITTER = 1024             # GPUTX_KSET_DIAG: random 0..2 us sleep before every transaction
GLOBAL_WAITS = 8192       # every cross-owner wait becomes a wait for all warps
ANY_OWNER = 16384         # owner = hash(transaction index): cross-owner edges everywhere

CASES = {
    "tm1": (W.TM1, W.Tm1Dims(4096), 8192, {}),
    "tm1_big": (W.TM1, W.Tm1Dims(20_000), 60_000, {}),
    "tpcb": (W.TPCB, W.TpcbDims(4, 10, 1000), 4096, dict(remote_pct=15.0)),
    "tpcb_wide": (W.TPCB, W.TpcbDims(64, 10, 1000), 50_000, dict(remote_pct=15.0)),
    "tpcb_withdraw": (W.TPCB, W.TpcbDims(16, 10, 100), 20_000, dict(withdraw_pct=30.0)),
    "micro": (W.MICRO, W.MicroDims(3000, 8, 1), 20_000, dict(alpha=0.05)),
}


def _open(schema, dims, image, n, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return gpu_db(schema, dims, image, n)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _run(case, env, grid=0, reps=1):
    schema, dims, n, kw = CASES[case]
    image = W.make_db(schema, dims, seed=1)
    bulk = W.make_bulk(schema, dims, n, seed=2, **kw)
    ref = oracle.run(schema, dims.dims, image, bulk)
    db = _open(schema, dims, image, n, env)
    try:
        if grid:
            db.set_launch(exec_grid=grid)
        flags = []
        for rep in range(reps):
            db.reset()
            db.submit(bulk)
            st = db.execute("kset")
            flags.append(st["flags"])
            compare(schema, ref, db, image, label=f"{case} {env} grid {grid} rep {rep}")
        return flags
    finally:
        db.close()


@pytest.mark.parametrize("case", list(CASES))
def test_owner_rounds_default(case):
    flags = _run(case, {})
    assert all(f & STAT_OWNER for f in flags), "owner-local rounds are the K-SET default here"


@pytest.mark.parametrize("case", ["tm1", "tpcb", "micro"])
def test_global_rounds_still_available(case):
    flags = _run(case, {"GPUTX_KSET_OWN": "0"})
    assert not any(f & STAT_OWNER for f in flags)


@pytest.mark.parametrize("case", ["tm1", "tpcb", "tpcb_withdraw", "micro"])
@pytest.mark.parametrize("diag", [ANY_OWNER, ANY_OWNER | GLOBAL_WAITS])
def test_arbitrary_owners_with_jitter(case, diag):
    """Owners unrelated to the root keys: nearly every T-dependency edge crosses warps, so
    the dependency pass (foreign predecessors, read runs, global waits) carries the result."""
    _run(case, {"GPUTX_KSET_DIAG": str(diag | JITTER)}, reps=3)


@pytest.mark.parametrize("case", ["tm1", "tpcb"])
@pytest.mark.parametrize("grid", [1, 3, 37])
def test_owner_rounds_any_grid(case, grid):
    _run(case, {"GPUTX_KSET_DIAG": str(JITTER)}, grid=grid, reps=3)
