"""Batched decode (B independent sequences sharing weight streams and expert
loads; BASELINE configs 2-3 ask for batch 1-16).  Parity at batch B means B
independent streams (SURVEY "Batch"): every sequence's tokens and logits must
equal its own single-sequence run, which tests/test_gpu.py pins to the
reference."""
import numpy as np
import pytest

TOY = dict(layers=8, experts=16, top_k=4, hidden=64, expert_hidden=128, vocab=256, head_dim=32, seed=11)


def _single(s, prompt, n_new, mode):
    P = len(prompt)
    S = P + n_new - 1
    s.reset(S, True)
    s.prefill(prompt)
    if n_new > 1:
        s.decode(mode, n_new - 1)
    toks = s.tokens(S)[P - 1:]
    lg = s.trace("logits", S)[P - 1:]
    return toks, lg


def _session(cfg, frac):
    from paper_2603_19289_b200 import ModelConfig, Session
    s = Session(ModelConfig(**cfg), cache_fraction=frac, max_positions=128)
    s.init_weights_seeded()
    d, _ = s.calibrate(64, 2, 32)
    s.load_default_vectors(d)
    s.set_predictor("router-pf")
    return s


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["on_demand", "prefetch"])
@pytest.mark.parametrize("B,frac", [(1, 1.0), (5, 0.5), (16, 0.25)])
def test_batch_generate_equals_independent_sequences(mode, B, frac):
    s = _session(TOY, frac)
    P, n_new = 4, 9
    prompts = np.random.default_rng(B).integers(0, 256, (B, P)).astype(np.int32)
    toks, lg = s.batch_generate(prompts, n_new, mode, logits=True)
    for b in range(B):
        want_t, want_lg = _single(s, prompts[b], n_new, mode)
        assert np.array_equal(toks[b], want_t), (b, toks[b], want_t)
        assert np.array_equal(lg[b].view(np.uint32), want_lg.view(np.uint32)), b
    s.close()


@pytest.mark.gpu
def test_batch_generate_gptoss_shape_batch8():
    """GPT-OSS-20B layer shapes (H 2880, 32 experts top-4), depth-truncated, batch 8."""
    cfg = dict(layers=2, experts=32, top_k=4, hidden=2880, expert_hidden=2880, vocab=256, head_dim=64, seed=3,
               gating="topk-softmax")
    s = _session(cfg, 0.25)
    prompts = np.random.default_rng(8).integers(0, 256, (8, 3)).astype(np.int32)
    for mode in ("prefetch", "on_demand"):
        toks = s.batch_generate(prompts, 5, mode)
        for b in range(8):
            want_t, _ = _single(s, prompts[b], 5, mode)
            assert np.array_equal(toks[b], want_t), (mode, b)
    s.close()


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["baseline-s", "est-pf", "hybrid"])
def test_batch_generate_other_predictors(kind):
    """baseline-s, est-pf (the Mixtral config's lightweight estimator, run as chain
    GEMMs) and a hybrid per-layer map, batched, against single-sequence runs."""
    from paper_2603_19289_b200 import engine
    s = _session(TOY, 0.5)
    flat = engine.estimator_init(64, 4, 2, 16, 8, 1e-5, 9)
    s.load_estimator(64, 4, 2, 16, 8, 1e-5, flat)
    hybrid = ["est-pf", "router-pf", "baseline-s", "est-pf", "router-pf", "baseline-s", "est-pf"]
    s.set_predictor(kind, hybrid if kind == "hybrid" else None)
    prompts = np.random.default_rng(3).integers(0, 256, (6, 4)).astype(np.int32)
    toks, lg = s.batch_generate(prompts, 8, "prefetch", logits=True)
    for b in range(6):
        want_t, want_lg = _single(s, prompts[b], 8, "prefetch")
        assert np.array_equal(toks[b], want_t), (kind, b)
        assert np.array_equal(lg[b].view(np.uint32), want_lg.view(np.uint32)), (kind, b)
    s.close()


@pytest.mark.gpu
def test_batch_generate_rejects_oracle():
    s = _session(TOY, 1.0)
    s.set_predictor("oracle")
    with pytest.raises(ValueError, match="oracle"):
        s.batch_generate(np.zeros((2, 3), np.int32), 3, "prefetch")
    s.close()


@pytest.mark.gpu
def test_batch_generate_mixtral_shape_batch16_est_pf():
    """Mixtral-8x7B layer shapes (H 4096, Hm 14336, 8 experts top-2) with the
    lightweight estimator (est-pf), depth-truncated, batch 16, half the experts cached."""
    from paper_2603_19289_b200 import engine
    cfg = dict(layers=2, experts=8, top_k=2, hidden=4096, expert_hidden=14336, vocab=256, head_dim=128, seed=1,
               gating="topk-softmax")
    s = _session(cfg, 0.5)
    s.load_estimator(4096, 8, 4, 8, 2, 1e-5, engine.estimator_init(4096, 8, 4, 8, 2, 1e-5, 5))
    s.set_predictor("est-pf")
    prompts = np.random.default_rng(16).integers(0, 256, (16, 3)).astype(np.int32)
    toks = s.batch_generate(prompts, 4, "prefetch")
    for b in range(16):
        want_t, _ = _single(s, prompts[b], 4, "prefetch")
        assert np.array_equal(toks[b], want_t), b
    s.close()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["on_demand", "prefetch"])
@pytest.mark.parametrize("frac", [1.0, 0.5])
def test_batch_generate_expert_parallel_two_ranks(mode, frac):
    """Batched decode under expert parallelism (SURVEY §8e, B > 1): two ranks
    sharing this GPU, each computing only its experts' rows of the step's B·k
    entries and exchanging them through peer stores + one system-scope
    arrival per rank per layer (k_pf_ep_publish / k_pf_ep_wait).  Both ranks
    return the single-GPU batch's tokens and logits bit for bit — resident
    experts (device-built work lists, CUDA graph) and an offloaded cache
    (host-driven waves, Algorithm 1 copies of local experts only)."""
    import threading
    from paper_2603_19289_b200 import ModelConfig, Session
    ref = Session(ModelConfig(**TOY), cache_fraction=1.0, max_positions=128)
    ref.init_weights_seeded()
    d, _ = ref.calibrate(64, 2, 32)
    ref.load_default_vectors(d)
    ref.set_predictor("router-pf")
    B, P, n_new = 6, 4, 7
    prompts = np.random.default_rng(31).integers(0, 256, (B, P)).astype(np.int32)
    want_t, want_lg = ref.batch_generate(prompts, n_new, mode, logits=True)
    ref.close()
    ranks = [Session(ModelConfig(**TOY), cache_fraction=frac, max_positions=128, ep_rank=r, ep_world=2)
             for r in (0, 1)]
    for s in ranks:
        s.init_weights_seeded()
        s.load_default_vectors(d)
        s.set_predictor("router-pf")
        if frac == 1.0:
            s.preload_all()
    bufs = [s.ep_buffers() for s in ranks]
    for s in ranks:
        s.ep_connect([b[0] for b in bufs], [b[1] for b in bufs])
    out, errs = [None, None], []

    def run(i):
        try:
            out[i] = ranks[i].batch_generate(prompts, n_new, mode, logits=True)
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in (0, 1)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not errs, errs
    for toks, lg in out:
        assert np.array_equal(toks, want_t)
        assert np.array_equal(lg.view(np.uint32), want_lg.view(np.uint32))
    for s in ranks:
        s.close()
