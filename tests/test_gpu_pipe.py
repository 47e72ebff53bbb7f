"""Pipelined gputx_run_bulks (TM-1 / micro K-SET): bulks are submitted and executed without
a host round trip between them, so validation errors surface after the run.  The results
must equal the oracle's serial execution of the bulks in sequence (Definition 1,
PAPER.md:73), and a bulk that fails validation must leave the database as the bulks
before it left it -- it and every later bulk of the run execute as empty."""
import numpy as np
import pytest

import oracle
import workloads as W
from paper_1103_3105_b200.gputx import GputxError, unpack_outputs
from tests.parity import gpu_db

pytestmark = pytest.mark.gpu

STAT_PIPELINED = 8
CASES = {
    "tm1": (W.TM1, W.Tm1Dims(4096), 8192, {}),
    "tm1_big": (W.TM1, W.Tm1Dims(50_000), 100_000, {}),
    "micro": (W.MICRO, W.MicroDims(3000, 8, 1), 8192, dict(alpha=0.05)),
}
SIZES = {W.TM1: np.array([40, 32, 16, 0, 0, 0, 0], np.int64), W.MICRO: None}


def offsets(schema, bulk, stride, packed):
    if not packed:
        return None
    sz = SIZES[schema][bulk.type.astype(np.int64)] if schema == W.TM1 else np.full(bulk.n, 4, np.int64)
    return np.concatenate([[0], np.cumsum(sz)]).astype(np.uint32)


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("packed", [False, True])
def test_pipelined_run_bulks_parity(case, packed):
    schema, dims, n, kw = CASES[case]
    image = W.make_db(schema, dims, seed=1)
    bulks = [W.make_bulk(schema, dims, n, seed=20 + k, **kw) for k in range(4)]
    db = gpu_db(schema, dims, image, n, packed_out=packed)
    try:
        status = [np.zeros(b.n, np.uint8) for b in bulks]
        out = [np.zeros(b.n * db.stride, np.uint8) for b in bulks]
        sts = db.run_bulks(bulks, "kset", status, out, stats=True)
        cur, ts = image, 0
        for k, b in enumerate(bulks):
            ref = oracle.run(schema, dims.dims, cur, b, first_ts=ts)
            assert sts[k]["flags"] & STAT_PIPELINED
            assert sts[k]["committed"] == int((ref.status == 0).sum())
            assert np.array_equal(status[k], ref.status), f"bulk {k} status"
            off = offsets(schema, b, db.stride, packed)
            got = unpack_outputs(out[k], off, db.stride) if packed else out[k].reshape(b.n, db.stride)
            assert np.array_equal(got, ref.out), f"bulk {k} outputs"
            cur, ts = ref.db, ts + b.n
        img = db.read_image(image)
        for c in image:
            assert np.array_equal(img[c], cur[c]), c
        st, o = db.read_results()                      # the last bulk's results stay readable
        assert np.array_equal(st, status[-1])
    finally:
        db.close()


@pytest.mark.parametrize("bad_at", [0, 1, 2])
def test_pipelined_error_stops_the_run(bad_at):
    schema, dims, n, kw = CASES["tm1"]
    image = W.make_db(schema, dims, seed=1)
    bulks = [W.make_bulk(schema, dims, n, seed=30 + k, **kw) for k in range(3)]
    bad = bulks[bad_at]
    bad.param_words = bad.param_words.copy()
    i = int(np.nonzero(bad.type == W.TM1_GSD)[0][5])
    bad.param_words[bad.param_off[i]] = 10 ** 7        # s_id out of range
    db = gpu_db(schema, dims, image, n)
    try:
        with pytest.raises(GputxError) as e:
            db.run_bulks(bulks, "kset", [np.zeros(b.n, np.uint8) for b in bulks], None)
        assert e.value.name == "EINVAL" and f"bulk {bad_at}" in str(e.value)
        cur, ts = image, 0
        for b in bulks[:bad_at]:
            cur = oracle.run(schema, dims.dims, cur, b, first_ts=ts).db
            ts += b.n
        img = db.read_image(image)
        for c in image:
            assert np.array_equal(img[c], cur[c]), f"{c}: a failed / later bulk changed the database"
        db.reset()                                     # usable again
        db.run_bulks([bulks[(bad_at + 1) % 3]], "kset", None, None)
    finally:
        db.close()
