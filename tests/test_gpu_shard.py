"""GPU parity of the sharded path (include/gputx.h "Sharding"): G shard
handles on one GPU, cross-shard transactions exchanged as packed records (device copies
stand in for the NCCL all-to-all), each shard executing its fragments in global ts order.
The union of the shards must equal serial execution of the whole bulk (Definition 1)."""
import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import compare_sharded

pytestmark = pytest.mark.gpu

STRATS = ["kset", "part", "tpl"]


def _run(schema, dims, image, bulk, G, strategy, p2p=False, **kw):
    from paper_1103_3105_b200 import Database
    from paper_1103_3105_b200.shard import LocalShards
    ref = oracle.run(schema, dims.dims, image, bulk)
    homes = W.split_home(bulk, dims, G)
    dbs = [Database(schema, dims.dims, bulk.n, image, shard=r, nshards=G, **kw) for r in range(G)]
    try:
        stats = LocalShards(dbs, p2p=p2p).step(homes, strategy)
        compare_sharded(schema, dims, ref, dbs, homes, image, label=f"{strategy} G={G}")
        return stats
    finally:
        for db in dbs:
            db.close()


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("G", [2, 3])
def test_tpcb_sharded(strategy, G):
    dims = W.TpcbDims(12, 10, 500)
    image = W.tpcb_db(dims)
    bulk = W.tpcb_bulk(dims, 6000, seed=3, remote_pct=40.0)
    stats = _run(W.TPCB, dims, image, bulk, G, strategy)
    assert sum(s["n"] for s in stats) > bulk.n          # remote accounts crossed shards


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("G", [2, 4])
def test_tpcc_sharded(strategy, G):
    dims = W.TpccDims(8, 10, 300, 2000)
    image = W.tpcc_db(dims, seed=2)
    bulk = W.tpcc_bulk(dims, 5000, seed=9, remote_line_pct=10.0, remote_pay_pct=30.0)
    stats = _run(W.TPCC, dims, image, bulk, G, strategy)
    assert sum(s["n"] for s in stats) > bulk.n


def test_tpcc_sharded_tiny_contention():
    """Few items and customers: duplicate lines, by-name misses, aborts, hot stock."""
    dims = W.TpccDims(3, 2, 30, 40)
    image = W.tpcc_db(dims, seed=4)
    bulk = W.tpcc_bulk(dims, 3000, seed=5, remote_line_pct=30.0, remote_pay_pct=40.0)
    for s in STRATS:
        _run(W.TPCC, dims, image, bulk, 3, s)


@pytest.mark.parametrize("strategy", STRATS)
def test_tm1_sharded(strategy):
    dims = W.Tm1Dims(5000)
    image = W.tm1_db(dims, seed=3)
    bulk = W.tm1_bulk(dims, 20_000, seed=4, dist="nurand")
    stats = _run(W.TM1, dims, image, bulk, 2, strategy)
    assert sum(s["n"] for s in stats) == bulk.n          # single-subscriber: nothing crosses


def test_sharded_errors():
    from paper_1103_3105_b200 import Database, GputxError
    dims = W.TpcbDims(4, 10, 100)
    image = W.tpcb_db(dims)
    bulk = W.tpcb_bulk(dims, 100, seed=1)
    db = Database(W.TPCB, dims.dims, 100, image, shard=0, nshards=2)
    try:
        with pytest.raises(GputxError) as e:
            db.submit(bulk)                                   # sharded handles use shard_pack/submit
        assert e.value.name == "ESTATE"
        home = bulk.take(np.arange(bulk.n), ts=np.arange(bulk.n, dtype=np.uint32))
        db.shard_pack(home)                                   # includes the other shard's txns
        with pytest.raises(GputxError) as e:
            db.shard_submit(None, 0)
        assert e.value.name == "ECROSS"
    finally:
        db.close()


@pytest.mark.parametrize("schema,dims,n,kw", [
    (W.TPCB, W.TpcbDims(12, 10, 500), 6000, dict(remote_pct=40.0)),
    (W.TPCC, W.TpccDims(8, 10, 300, 2000), 5000, dict(remote_line_pct=10.0, remote_pay_pct=30.0)),
])
def test_auto_sharded(schema, dims, n, kw):
    """GPUTX_AUTO on shards: each shard runs Algorithm 1 on its local graph (the choice
    may differ between shards; every strategy is shard-local) and the union still
    equals serial execution."""
    image = W.make_db(schema, dims, seed=2)
    bulk = W.make_bulk(schema, dims, n, 9, **kw)
    stats = _run(schema, dims, image, bulk, 2, "auto")
    assert all(s["strategy"] in ("kset", "part", "tpl") for s in stats)


@pytest.mark.parametrize("bad", ["nonmonotone", "toolong", "firstoff"])
def test_shard_pack_rejects_malformed_offsets(bad):
    """a malformed home bulk must be rejected (EINVAL) before any kernel reads
    or writes through its offsets -- no out-of-bounds merge of parameter words."""
    from paper_1103_3105_b200 import Database
    from paper_1103_3105_b200.gputx import GputxError
    dims = W.TpccDims(4, 10, 30, 500)
    image = W.tpcc_db(dims, seed=1)
    bulk = W.tpcc_bulk(dims, 400, seed=2)
    home = W.split_home(bulk, dims, 2)[0]
    off = home.param_off.astype(np.int64).copy()
    if bad == "nonmonotone":
        off[5] = off[7] + 3
    elif bad == "toolong":
        off[6] = off[5] + 50              # > 49 words (the TPC-C maximum) for transaction 5
    else:
        off[0] = 1                        # param_off[0] must be 0
    home.param_off = off.astype(np.uint32)
    db = Database(W.TPCC, dims.dims, bulk.n, image, shard=0, nshards=2)
    with pytest.raises(GputxError) as e:
        db.shard_pack(home)
    assert e.value.name in ("EINVAL", "ECAPACITY")
    db.close()


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("case", ["tpcb", "tpcc", "tm1"])
@pytest.mark.parametrize("G", [2, 4])
def test_fused_peer_exchange(case, G, strategy):
    """The library's fused exchange over peer memory (gputx_shard_dispatch / receive /
    return / collect): the dispatching kernel writes the records straight into the owner
    shard's arena; the union of the shards equals the serial run of the whole bulk."""
    if case == "tpcb":
        dims = W.TpcbDims(12, 10, 500)
        image, bulk = W.tpcb_db(dims), W.tpcb_bulk(dims, 6000, seed=3, remote_pct=40.0)
        schema = W.TPCB
    elif case == "tpcc":
        dims = W.TpccDims(8, 10, 30, 1000)
        image, bulk = W.tpcc_db(dims, seed=2), W.tpcc_bulk(dims, 5000, seed=4, remote_line_pct=10.0,
                                                           remote_pay_pct=30.0)
        schema = W.TPCC
    else:
        dims = W.Tm1Dims(4000)
        image, bulk = W.tm1_db(dims, seed=2), W.tm1_bulk(dims, 6000, seed=5)
        schema = W.TM1
    stats = _run(schema, dims, image, bulk, G, strategy, p2p=True)
    if case != "tm1":
        assert sum(s["n"] for s in stats) > bulk.n          # cross-shard records moved


def test_fused_peer_exchange_repeated_epochs():
    """Several bulks back to back through the same arenas (epochs, counter resets)."""
    from paper_1103_3105_b200 import Database
    from paper_1103_3105_b200.shard import LocalShards
    dims = W.TpccDims(6, 10, 30, 1000)
    image = W.tpcc_db(dims, seed=2)
    G = 3
    dbs = [Database(W.TPCC, dims.dims, 6000, image, shard=r, nshards=G, insert_capacity=6) for r in range(G)]
    ls = LocalShards(dbs, p2p=True)
    cur, ts0 = image, 0
    try:
        for k in range(4):
            bulk = W.tpcc_bulk(dims, 3000, seed=20 + k, remote_line_pct=10.0, remote_pay_pct=30.0)
            bulk.ts = (ts0 + np.arange(bulk.n)).astype(np.uint32)
            ref = oracle.run(W.TPCC, dims.dims, cur, bulk, first_ts=ts0)
            homes = W.split_home(bulk, dims, G)
            for h in homes:
                h.ts = (h.ts.astype(np.int64) + ts0).astype(np.uint32)
            ls.step(homes, "kset")
            for r, db in enumerate(dbs):
                st, out = db.read_results()
                idx = homes[r].ts.astype(np.int64) - ts0
                assert np.array_equal(st, ref.status[idx]) and np.array_equal(out, ref.out[idx]), (k, r)
            cur, ts0 = ref.db, ts0 + bulk.n
    finally:
        for db in dbs:
            db.close()


def test_bench_cli_two_ranks_strong_tpcc():
    """`GPUTX_DIST_BACKEND=gloo python bench.py --gpus 2 --workload tpcc
    --scaling strong` on one GPU spawns 2 ranks, runs the fused peer exchange between them
    (CUDA IPC on one device) and prints one line with n_gpus 2 (a functional check: two
    ranks sharing one GPU say nothing about scaling)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["GPUTX_DIST_BACKEND"] = "gloo"
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--workload", "tpcc", "--scaling", "strong",
                          "--steps", "2", "--warmup", "3", "--also", "none", "--others", "", "--no-cpu-baseline"],
                         cwd=root, capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert "fused" in d["config"]["exchange"]
