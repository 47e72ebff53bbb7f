"""K-SET hand-off stress (VERDICT r1 "correctness gate"): the round schedule must give the
serial result (Definition 1; Property 1) whatever the launch
shape and whatever order the CTAs happen to finish in.  Every run below is compared with
the oracle element by element (image, statuses, outputs, inserts)."""
import os

import pytest

import oracle
import workloads as W
from tests.parity import compare, gpu_db

pytestmark = pytest.mark.gpu

JITTER = 1024          # GPUTX_KSET_DIAG: random 0..2 us sleep before every transaction
NO_CLUSTER_LAUNCH = 512  # GPUTX_KSET_DIAG: launch without the cluster attribute


def _open(schema, dims, image, n, cluster=None, diag=0):
    env = {"GPUTX_KSET_DIAG": str(diag)}
    if cluster is not None:
        env["GPUTX_KSET_CLUSTER"] = str(cluster)
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


CASES = {
    "tm1": (W.TM1, W.Tm1Dims(4096), 8192, {}),                                   # smoke() config
    "tpcb": (W.TPCB, W.TpcbDims(4, 10, 1000), 4096, dict(remote_pct=15.0)),
    "tpcc": (W.TPCC, W.TpccDims(2, 10, 300, 2000), 2048, {}),
}


@pytest.mark.parametrize("case", ["tm1", "tpcb"])
@pytest.mark.parametrize("cluster", [0, 8])
@pytest.mark.parametrize("grid", [1, 7, 37, 0])
def test_kset_stress_grid_cluster_jitter(case, cluster, grid):
    schema, dims, n, kw = CASES[case]
    image = W.make_db(schema, dims, seed=1)
    bulk = W.make_bulk(schema, dims, n, seed=2, **kw)
    ref = oracle.run(schema, dims.dims, image, bulk)
    db = _open(schema, dims, image, n, cluster=cluster, diag=JITTER)
    try:
        if grid and cluster and grid % cluster:
            grid = max(cluster, grid // cluster * cluster)
        db.set_launch(exec_grid=grid)
        for rep in range(10):
            db.reset()
            db.submit(bulk)
            db.execute("kset")
            compare(schema, ref, db, image, label=f"{case} grid {grid} cluster {cluster} rep {rep}")
    finally:
        db.close()


@pytest.mark.parametrize("case", ["tm1", "tpcb", "tpcc"])
def test_kset_survives_launch_without_clusters(case):
    """GPUTEST_r01: under ncu the executor's cluster launch ran every CTA as a cluster of
    one, the cluster barriers synchronised nothing and TM-1 GSD read stale vlr values.
    The kernel now reads %cluster_nctarank and falls back to counter hand-offs; diag 512
    reproduces that launch without a profiler."""
    schema, dims, n, kw = CASES[case]
    image = W.make_db(schema, dims, seed=1)
    bulk = W.make_bulk(schema, dims, n, seed=2, **kw)
    ref = oracle.run(schema, dims.dims, image, bulk)
    import os as _os
    _os.environ["GPUTX_KSET_DF"] = "0"           # the round executor (TPC-C defaults to dataflow)
    try:
        db = _open(schema, dims, image, n, cluster=8, diag=NO_CLUSTER_LAUNCH | JITTER)
    finally:
        _os.environ.pop("GPUTX_KSET_DF", None)
    try:
        for rep in range(5):
            db.reset()
            db.submit(bulk)
            st = db.execute("kset")
            assert st["flags"] & 1, "the executor did not notice the missing clusters"
            compare(schema, ref, db, image, label=f"{case} no-cluster launch rep {rep}")
    finally:
        db.close()


def test_kset_watchdog_returns_edeadlock():
    """A K-SET round that waits for a signal that never comes (diag 2048) must not hang:
    the spin watchdog trips, the call returns EDEADLOCK, the handle is poisoned until
    gputx_reset (include/gputx.h)."""
    from paper_1103_3105_b200.gputx import GputxError
    schema, dims, n, kw = CASES["tm1"]
    image = W.make_db(schema, dims, seed=1)
    bulk = W.make_bulk(schema, dims, n, seed=2, **kw)
    os.environ["GPUTX_WATCHDOG_MS"] = "300"
    try:
        db = _open(schema, dims, image, n, cluster=0, diag=2048)
    finally:
        os.environ.pop("GPUTX_WATCHDOG_MS", None)
    try:
        db.submit(bulk)
        with pytest.raises(GputxError) as e:
            db.execute("kset")
        assert e.value.name == "EDEADLOCK"
        with pytest.raises(GputxError) as e2:
            db.submit(bulk)
        assert e2.value.name == "ESTATE"
        db.reset()
        db.submit(bulk)                         # usable again after reset
    finally:
        db.close()
        os.environ["GPUTX_WATCHDOG_MS"] = "10000"   # restore the process-wide default
        try:
            _open(schema, dims, image, n).close()
        finally:
            os.environ.pop("GPUTX_WATCHDOG_MS", None)
