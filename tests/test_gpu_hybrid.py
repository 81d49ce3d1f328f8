"""Hybrid-map selection end to end on the GPU: measure the
per-layer online hit rates of router-pf and est-pf on the same teacher-forced
stream, select the map, decode with it, and check the hybrid
decode against the oracle's hybrid predictor with the same map."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOY = dict(layers=8, experts=16, top_k=4, hidden=64, expert_hidden=128, vocab=256, head_dim=32,
           seed=4)


@pytest.fixture(scope="module")
def lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2603_19289_b200 import load_library
    return load_library()


def test_select_and_run_hybrid_map(lib):
    from oracle.bindings import Config, Oracle
    from paper_2603_19289_b200 import ModelConfig, Session, layer_hit_rates, select_hybrid_map
    orc = Oracle()
    om = orc.build_model(Config(**TOY), round_bf16=True)
    table = om.calibrate(128, 2, 32)
    est = orc.estimator(TOY["hidden"], 2, 4, TOY["experts"], TOY["layers"], seed=5)
    s = Session(ModelConfig(**TOY), cache_fraction=0.5, max_positions=256)
    s.init_weights_seeded()
    s.load_default_vectors(np.array(table.d))
    s.load_estimator(TOY["hidden"], 2, 4, TOY["experts"], TOY["layers"], 1e-5, np.array(est.flat))
    prompt = [5, 77, 200, 13, 9]
    forced = np.random.default_rng(2).integers(0, 256, 40).astype(np.int32)
    P, N = len(prompt), 40
    rates = {}
    for kind in ("router-pf", "est-pf", "baseline-s"):
        s.set_predictor(kind)
        s.reset(P + N, False)
        s.prefill(prompt)
        s.decode_stream("prefetch", forced)
        rates[kind] = layer_hit_rates(s.trace("id_exec", P + N)[P:], s.trace("id_true", P + N)[P:])
    hmap = select_hybrid_map(rates)
    assert len(hmap) == TOY["layers"] - 1
    for l, k in enumerate(hmap):  # the chosen predictor has the best rate at that layer
        assert rates[k][l] == max(r[l] for r in rates.values())
    s.set_predictor("hybrid", hmap)
    s.reset(P + N, False)
    s.prefill(prompt)
    s.decode_stream("prefetch", forced)
    got = s.trace("id_exec", P + N)
    want = om.generate_trace(prompt, N + 1, orc.make_predictor("hybrid", om, table, est, hmap), forced=forced)
    assert np.array_equal(got, want.ids)
    s.close()
