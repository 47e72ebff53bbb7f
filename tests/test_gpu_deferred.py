"""GPUTX_FLAG_DEFERRED_CHECK (include/gputx.h): submit enqueues the validation without waiting
for its verdict; the verdict comes with execute.  Results must equal the oracle's serial
execution (Definition 1), and a bulk that fails validation must leave the
database unchanged whatever the strategy."""
import numpy as np
import pytest

import oracle
import workloads as W
from paper_1103_3105_b200.gputx import GputxError
from tests.parity import compare, gpu_db

pytestmark = pytest.mark.gpu

CASES = {
    "tm1": (W.TM1, W.Tm1Dims(4096), 8192, {}),
    "micro": (W.MICRO, W.MicroDims(3000, 8, 1), 8192, dict(alpha=0.05)),
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("strategy", ["kset", "part", "tpl"])
@pytest.mark.parametrize("packed", [False, True])
def test_deferred_parity(case, strategy, packed):
    schema, dims, n, kw = CASES[case]
    image = W.make_db(schema, dims, seed=1)
    bulk = W.make_bulk(schema, dims, n, seed=2, **kw)
    ref = oracle.run(schema, dims.dims, image, bulk)
    db = gpu_db(schema, dims, image, n, deferred_check=True, packed_out=packed)
    try:
        db.submit(bulk)
        db.execute(strategy)
        compare(schema, ref, db, image, label=f"deferred {case} {strategy}")
    finally:
        db.close()


@pytest.mark.parametrize("strategy", ["kset", "tpl"])
def test_deferred_error_leaves_db_unchanged(strategy):
    schema, dims, n, kw = CASES["tm1"]
    image = W.make_db(schema, dims, seed=1)
    bad = W.make_bulk(schema, dims, n, seed=2, **kw)
    bad.param_words = bad.param_words.copy()
    i = int(np.nonzero(bad.type == W.TM1_GSD)[0][7])
    bad.param_words[bad.param_off[i]] = 10 ** 7         # s_id out of range
    db = gpu_db(schema, dims, image, n, deferred_check=True, packed_out=True)
    try:
        db.submit(bad)                                  # no verdict yet
        with pytest.raises(GputxError) as e:
            db.execute(strategy)
        assert e.value.name == "EINVAL"
        img = db.read_image(image)
        for c in image:
            assert np.array_equal(img[c], image[c]), f"{c} changed by a failed bulk"
        good = W.make_bulk(schema, dims, n, seed=3, **kw)
        ref = oracle.run(schema, dims.dims, image, good)
        assert db.submit(good) == 0, "the failed bulk must not consume timestamps"
        db.execute(strategy)
        compare(schema, ref, db, image, label="after a failed deferred bulk")
    finally:
        db.close()
