"""The N > 1 host path on CPU (gloo, world_size 2): per-rank shards, max-over-ranks
timing, and the reference arm under torchrun (rank 0 prints, others exit quietly)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import torch
    import bench
    import workloads as W
    from paper_1103_3105_b200.shard import all_to_all_records
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = bench.WORKLOADS["tpcc"]
    small = dict(wl, dims=W.TpccDims(4, 10, 30, 1000), n=500)
    dims, image, bulks = bench.make_inputs(small, rank, world, 1, seed=3)
    roots = W.home_roots(bulks[0])
    # exchange: rank r sends r+1 records to every peer (stride 3: [ts, src, dst])
    stride = 3
    counts = [(rank + 1) if q != rank else 0 for q in range(world)]
    recs = [[1000 * rank + j, rank, q] for q in range(world) for j in range(counts[q])]
    send = torch.tensor(recs, dtype=torch.int32).reshape(-1)
    recv, nrecv = all_to_all_records(send, counts, stride)
    got = recv[:nrecv * stride].reshape(-1, stride).tolist()
    x = bench.reduce_max(dist, float(rank + 1) * 1.5)
    q.put((rank, x, dims.dims, int(roots.min()), int(roots.max()), bulks[0].ts[:3].tolist(), got))
    dist.destroy_process_group()


def test_gloo_two_ranks_shards_exchange_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29000 + os.getpid() % 1000
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == res[1][1] == 3.0               # max over ranks
    assert res[0][2] == res[1][2] == (8, 10, 30, 1000)  # weak scaling: 2 x 4 warehouses, same image
    assert (res[0][3], res[0][4]) == (0, 3) and (res[1][3], res[1][4]) == (4, 7)   # home roots per shard
    assert res[0][5] == [0, 2, 4] and res[1][5] == [1, 3, 5]                       # interleaved global ts
    assert res[0][6] == [[1000, 1, 0], [1001, 1, 0]]   # rank 0 received rank 1's two records
    assert res[1][6] == [[0, 0, 1]]


def test_reference_arm_torchrun_two_ranks():
    port = 30000 + os.getpid() % 1000
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl", "reference",
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--workload", "tpcb_tiny"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"


def test_bench_self_spawns_ranks_for_gpus_n():
    """`bench.py --gpus 2` without a launcher re-runs itself under torch.distributed.run
    with two ranks (--gpus was parsed and ignored); rank 0 prints n_gpus 2."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    cmd = [sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "2", "--warmup", "1",
           "--workload", "tpcb_tiny", "--scaling", "strong"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"


def test_strong_scaling_inputs_partition_one_bulk():
    """--scaling strong (BASELINE config 4): the configuration's database and ONE bulk in
    total; every transaction is submitted by exactly one rank (its home warehouse's), with
    its global timestamp."""
    sys.path.insert(0, ROOT)
    import bench
    import workloads as W
    wl = dict(bench.WORKLOADS["tpcc"], dims=W.TpccDims(8, 10, 30, 1000), n=3000)
    parts = [bench.make_inputs_strong(wl, r, 4, 1, seed=5) for r in range(4)]
    assert all(p[0].dims == (8, 10, 30, 1000) for p in parts)
    ts = np.concatenate([p[2][0].ts for p in parts]).astype(np.int64)
    assert np.array_equal(np.sort(ts), np.arange(3000))
    for r, p in enumerate(parts):
        assert np.all(W.shard_of(W.home_roots(p[2][0]), 4, 8) == r)
