"""GPUTX_FLAG_PACKED_OUT (include/gputx.h): variable-size output records at submit-time
offsets, so the result transfer the paper counts in the bulk time
moves only what the procedures return.  Every record must be the first bytes of the
oracle's fixed-stride record, with the rest of that record zero; the offsets must follow
the documented size rule."""
import numpy as np
import pytest

import oracle
import workloads as W
from paper_1103_3105_b200.gputx import GputxError, unpack_outputs
from tests.parity import compare, gpu_db

pytestmark = pytest.mark.gpu

CASES = {
    "tm1": (W.TM1, W.Tm1Dims(4096), 8192, {}),
    "tpcb": (W.TPCB, W.TpcbDims(4, 10, 1000), 4096, dict(remote_pct=15.0)),
    "tpcc": (W.TPCC, W.TpccDims(2, 10, 300, 2000), 2048, {}),
    "micro": (W.MICRO, W.MicroDims(3000, 8, 1), 8192, dict(alpha=0.05)),
}


def documented_sizes(schema, bulk):
    """The record sizes of include/gputx.h GPUTX_FLAG_PACKED_OUT, from types and params."""
    t = bulk.type.astype(np.int64)
    if schema == W.TPCB:
        return np.full(bulk.n, 8, np.int64)
    if schema == W.MICRO:
        return np.full(bulk.n, 4, np.int64)
    if schema == W.TM1:
        return np.array([40, 32, 16, 0, 0, 0, 0], np.int64)[t]
    cnt = bulk.param_words[bulk.param_off[:-1].astype(np.int64) + 3].astype(np.int64)
    return np.where(t == 0, (16 + 12 * cnt + 7) // 8 * 8, 16)


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("strategy", ["kset", "part", "tpl"])
def test_packed_outputs_match_oracle(case, strategy):
    schema, dims, n, kw = CASES[case]
    image = W.make_db(schema, dims, seed=1)
    bulk = W.make_bulk(schema, dims, n, seed=2, **kw)
    ref = oracle.run(schema, dims.dims, image, bulk)
    db = gpu_db(schema, dims, image, n, packed_out=True)
    try:
        db.submit(bulk)
        off = db.read_out_offsets()
        sizes = documented_sizes(schema, bulk)
        assert off[0] == 0 and np.array_equal(np.diff(off.astype(np.int64)), sizes)
        db.execute(strategy)
        compare(schema, ref, db, image, label=f"packed {case} {strategy}")
        _, raw = db.read_results(raw=True)
        assert raw.size == int(sizes.sum()) <= n * db.stride
        # the bytes beyond a record's packed size are zero in the oracle's record
        for s in np.unique(sizes):
            rows = np.nonzero(sizes == s)[0]
            assert not ref.out[rows, s:].any()
    finally:
        db.close()


@pytest.mark.parametrize("case", ["tm1", "tpcc"])
def test_packed_run_bulks(case):
    """gputx_run_bulks moves out_off[n] bytes per bulk; unpacked they equal the oracle's
    outputs of the same bulks run in sequence."""
    schema, dims, n, kw = CASES[case]
    image = W.make_db(schema, dims, seed=1)
    bulks = [W.make_bulk(schema, dims, n, seed=10 + k, **kw) for k in range(3)]
    db = gpu_db(schema, dims, image, n, packed_out=True, insert_capacity=8)
    try:
        status = [np.zeros(b.n, np.uint8) for b in bulks]
        out = [np.zeros(b.n * db.stride, np.uint8) for b in bulks]
        db.run_bulks(bulks, "kset", status, out)
        cur, ts = image, 0
        for k, b in enumerate(bulks):
            ref = oracle.run(schema, dims.dims, cur, b, first_ts=ts)
            off = np.concatenate([[0], np.cumsum(documented_sizes(schema, b))]).astype(np.uint32)
            assert np.array_equal(status[k], ref.status), f"bulk {k} status"
            assert np.array_equal(unpack_outputs(out[k], off, db.stride), ref.out), f"bulk {k} outputs"
            cur, ts = ref.db, ts + b.n
    finally:
        db.close()


def test_packed_rejects_pool():
    schema, dims, n, kw = CASES["tpcb"]
    image = W.make_db(schema, dims, seed=1)
    bulk = W.make_bulk(schema, dims, 64, seed=2, **kw)
    db = gpu_db(schema, dims, image, n, packed_out=True)
    try:
        with pytest.raises(GputxError) as e:
            db.pool_submit(bulk)
        assert e.value.name == "EINVAL"
    finally:
        db.close()
