"""Boundary features of SURVEY.md §8(b): device memory through the caller's allocator
(cfg.alloc / cfg.free = PyTorch's caching allocator) and gputx_snapshot."""
import numpy as np
import pytest

import workloads as W
from tests.parity import gpu_db, run_both

pytestmark = pytest.mark.gpu


def test_torch_caching_allocator_hooks():
    import torch
    dims = W.TpccDims(2, 10, 300, 2000)
    image = W.tpcc_db(dims, seed=1)
    bulk = W.tpcc_bulk(dims, 3000, seed=2)
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated(0)
    db = gpu_db(W.TPCC, dims, image, bulk.n, torch_memory=True)
    held = torch.cuda.memory_allocated(0) - before
    assert held > 10 << 20                      # the engine's buffers live in torch's pool
    for s in ("kset", "tpl", "part"):
        db.reset()
        run_both(W.TPCC, dims, image, [bulk], s, db=db)
    db.close()
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated(0) - before < (1 << 20)   # all of it returned


def test_snapshot_matches_columns_and_inserts():
    dims = W.TpcbDims(4, 10, 1000)
    image = W.tpcb_db(dims)
    bulk = W.tpcb_bulk(dims, 5000, seed=3, withdraw_pct=20.0)
    db = gpu_db(W.TPCB, dims, image, bulk.n)
    db.submit(bulk)
    db.execute("kset")
    snap = db.snapshot()
    assert snap["schema"] == W.TPCB and snap["dims"] == list(dims.dims)
    got = db.read_image(image)
    for k in image:
        assert np.array_equal(snap["columns"][k].view(image[k].dtype), got[k].reshape(-1)), k
    ins = db.inserts()
    for c, a in ins["history"].items():
        assert np.array_equal(snap["tables"]["history"][c], a.view(np.uint32)), c
    db.close()


@pytest.mark.parametrize("schema", [W.TM1, W.TPCC, W.TPCB])
def test_run_bulks_overlapped_equals_serial(schema):
    """gputx_run_bulks (overlapped H2D / D2H, two copy streams) gives every bulk's results
    and the final state of the serial run of the bulks one after another."""
    import oracle
    import torch
    dims = {W.TM1: W.Tm1Dims(5000), W.TPCC: W.TpccDims(2, 10, 300, 2000), W.TPCB: W.TpcbDims(4, 10, 1000)}[schema]
    image = W.make_db(schema, dims, seed=1)
    bulks = [W.make_bulk(schema, dims, 3000 + 500 * k, seed=10 + k) for k in range(5)]
    db = gpu_db(schema, dims, image, 6000, insert_capacity=8)
    stride = db.stride
    st = [torch.empty(b.n, dtype=torch.uint8).pin_memory().numpy() for b in bulks]
    out = [torch.empty(b.n * stride, dtype=torch.uint8).pin_memory().numpy().reshape(b.n, stride) for b in bulks]
    stats = db.run_bulks(bulks, "kset", st, out, stats=True)
    cur, ts = image, 0
    for k, b in enumerate(bulks):
        ref = oracle.run(schema, dims.dims, cur, b, first_ts=ts)
        assert np.array_equal(st[k], ref.status), k
        assert np.array_equal(out[k], ref.out), k
        assert stats[k]["n"] == b.n
        cur, ts = ref.db, ts + b.n
    got = db.read_image(image)
    for c in image:
        assert np.array_equal(got[c], cur[c]), c
    db.close()


@pytest.mark.parametrize("strategy", ["kset", "part", "tpl", "auto"])
def test_execute_async_wait_equals_execute(strategy):
    """gputx_execute_async + gputx_wait give gputx_execute's results and stats; the
    handle refuses other calls (ESTATE) while the execute is pending."""
    import oracle
    from paper_1103_3105_b200.gputx import GputxError
    dims = W.Tm1Dims(5000)
    image = W.make_db(W.TM1, dims, seed=1)
    bulk = W.make_bulk(W.TM1, dims, 4000, seed=7)
    db = gpu_db(W.TM1, dims, image, bulk.n, insert_capacity=8)
    db.submit(bulk)
    db.execute_async(strategy)
    with pytest.raises(GputxError):
        db.read_results()
    with pytest.raises(GputxError):
        db.execute(strategy)
    st = db.wait()
    with pytest.raises(GputxError):
        db.wait()                                   # nothing pending any more
    assert st["n"] == bulk.n and st["committed"] + st["aborted"] == bulk.n
    ref = oracle.run(W.TM1, dims.dims, image, bulk)
    status, out = db.read_results()
    assert np.array_equal(status, ref.status) and np.array_equal(out, ref.out)
    got = db.read_image(image)
    for c in image:
        assert np.array_equal(got[c], ref.db[c]), c
    db.close()
