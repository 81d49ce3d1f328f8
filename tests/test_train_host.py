"""CPU checks of the estimator-training boundary (no GPU): the host-side
init_estimator_params restatement against the reference, and the reference's
validation messages through the C ABI."""
import numpy as np
import pytest

from oracle.bindings import Ref
from paper_2603_19289_b200 import engine


@pytest.mark.parametrize("shape", [(64, 2, 4, 16, 4, 7), (96, 3, 2, 20, 5, 1), (2048, 2, 4, 128, 48, 1)])
def test_estimator_init_matches_reference(shape):
    d, m, n, E, L, seed = shape
    ref = Ref()
    want = ref.estimator_flat(ref.estimator_init(d, m, n, E, L, 1e-5, seed))
    got = engine.estimator_init(d, m, n, E, L, 1e-5, seed)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("kw,msg", [
    (dict(m=1), "estimator: m and n must be > 1"),
    (dict(d=63), "estimator: d must be divisible by m"),
    (dict(k=0), "train: invalid k"),
    (dict(k=17), "train: invalid k"),
    (dict(val_fraction=1.0), "train: no training tokens after split"),
])
def test_train_validation_messages(kw, msg):
    a = dict(d=64, m=2, n=4, E=16, L=4, k=2, val_fraction=0.1)
    a.update(kw)
    T = 10
    inp = np.zeros((T, a["L"] - 1, a["d"]), np.float32)
    tgt = np.zeros((T, a["L"] - 1, a["E"]), np.float32)
    with pytest.raises(ValueError, match=msg):
        engine.train_estimator(inp, tgt, a["d"], a["m"], a["n"], a["E"], a["L"], k=a["k"],
                               val_fraction=a["val_fraction"], max_steps=1)
