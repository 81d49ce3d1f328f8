"""Estimator distillation on the GPU against the reference's
own train_estimator (estimator.cpp:374-450, oracle/_ref): trained parameters
and the validation curve must be bit-identical."""
import numpy as np
import pytest

from oracle.bindings import Ref
from paper_2603_19289_b200 import engine

CASES = [
    # d, m, n, E, L, tokens, batch, steps, eval_every, k, val_fraction, early_stop
    (64, 2, 4, 16, 4, 40, 4, 10, 3, 2, 0.1, 0.0),
    (96, 3, 2, 20, 5, 23, 3, 7, 2, 3, 0.2, 0.0),     # ragged tiles (latent 32, mlp 64, E 20)
    (256, 2, 4, 64, 6, 64, 8, 5, 5, 4, 0.1, 0.0),    # multi-tile chains
    (64, 2, 4, 16, 4, 40, 4, 10, 3, 2, 0.1, 0.01),   # early stop at the first evaluation
    (64, 2, 4, 16, 4, 40, 4, 0, 3, 2, 0.1, 0.0),     # max_steps = 0: init params, one curve point
]


def _data(T, L, d, E, seed):
    rng = np.random.default_rng(seed)
    inp = rng.standard_normal((T, L - 1, d)).astype(np.float32)
    tgt = (2.0 * rng.standard_normal((T, L - 1, E))).astype(np.float32)
    return inp, tgt


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_train_estimator_matches_reference(case):
    d, m, n, E, L, T, B, steps, ev, k, vf, es = case
    inp, tgt = _data(T, L, d, E, d + T)
    ref = Ref()
    kw = dict(eps=1e-5, seed=11, lr=3e-3, batch=B, max_steps=steps, eval_every=ev, val_fraction=vf,
              hseed=5, k=k, early_stop=es)
    rp, rc = ref.train_estimator(inp, tgt, d, m, n, E, L, **kw)
    gp, gc, _ = engine.train_estimator(inp, tgt, d, m, n, E, L, **kw)
    assert gc.shape == rc.shape
    np.testing.assert_array_equal(gc, rc)
    bad = np.flatnonzero(gp.view(np.uint32) != rp.view(np.uint32))
    assert bad.size == 0, f"{bad.size} params differ, first at {bad[:5]}: {gp[bad[:5]]} vs {rp[bad[:5]]}"
    if steps and not es:
        assert not np.array_equal(gp, engine.estimator_init(d, m, n, E, L, 1e-5, 11))


@pytest.mark.gpu
def test_train_estimator_on_model_trace():
    """Distillation data from a real decode: quasi-hidden inputs are replaced by
    the traced post-attention state s_{l+1} (DistillInput::kSNext, speculation.cpp:463-467)
    and targets by the traced true router logits of layer l+1."""
    from paper_2603_19289_b200 import ModelConfig, Session
    cfg = dict(layers=8, experts=16, top_k=4, hidden=64, expert_hidden=128, vocab=256, head_dim=32, seed=3)
    s = Session(ModelConfig(**cfg), max_positions=128)
    s.init_weights_seeded()
    T = 48
    s.reset(T, True)
    s.prefill(list(range(1, T + 1)))
    st = s.trace("s", T).reshape(T, 8, 64)
    lg = s.trace("lg_true", T).reshape(T, 8, 16)
    inp = np.ascontiguousarray(st[:, 1:, :])
    tgt = np.ascontiguousarray(lg[:, 1:, :])
    ref = Ref()
    kw = dict(seed=2, lr=1e-2, batch=8, max_steps=12, eval_every=4, hseed=1, k=4)
    rp, rc = ref.train_estimator(inp, tgt, 64, 2, 4, 16, 8, **kw)
    gp, gc, _ = engine.train_estimator(inp, tgt, 64, 2, 4, 16, 8, **kw)
    np.testing.assert_array_equal(gc, rc)
    assert np.array_equal(gp.view(np.uint32), rp.view(np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["quasi", "s-next"])
def test_distill_dataset_and_training_match_reference(mode):
    """build_distill_dataset (speculation.cpp:476-484) on the GPU from a captured
    decode, against the reference's builder over the reference's own trace of
    the same model and prompt; then both train on it (bit-exact end to end)."""
    from paper_2603_19289_b200 import ModelConfig, Session
    from oracle.bindings import Config
    cfg = dict(layers=8, experts=16, top_k=4, hidden=64, expert_hidden=128, vocab=256, head_dim=32, seed=5)
    ref = Ref()
    rm = ref.build_model(Config(**cfg))
    prompt = [int(x) for x in np.random.default_rng(1).integers(0, 256, 40)]
    table = None
    s = Session(ModelConfig(**cfg), max_positions=128)
    s.init_weights_seeded()
    if mode == "quasi":
        table = rm.calibrate(64, 7, 32)
        d, _ = ref.table_get(table)
        s.load_default_vectors(d)
    T = len(prompt)
    s.reset(T, True)
    s.prefill(prompt)
    gi, gt = s.build_distill_dataset(0, T, mode)
    ri, rt = rm.distill_dataset(prompt, table, mode)
    assert np.array_equal(gt, rt)
    assert np.array_equal(gi.view(np.uint32), ri.view(np.uint32))
    kw = dict(seed=2, lr=1e-2, batch=8, max_steps=8, eval_every=4, hseed=1, k=4)
    rp, rc = ref.train_estimator(ri, rt, 64, 2, 4, 16, 8, **kw)
    gp, gc, _ = engine.train_estimator(gi, gt, 64, 2, 4, 16, 8, **kw)
    np.testing.assert_array_equal(gc, rc)
    assert np.array_equal(gp.view(np.uint32), rp.view(np.uint32))
