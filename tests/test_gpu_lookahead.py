"""Multi-layer-ahead prediction on the GPU: depth-1
predictions from captured traces reproduce the decode's own router-pf
predictions; deeper lookahead feeds the cache simulator."""
import numpy as np
import pytest

TOY = dict(layers=8, experts=16, top_k=4, hidden=64, expert_hidden=128, vocab=256, head_dim=32, seed=7)


@pytest.mark.gpu
def test_predict_ahead_depth1_equals_router_pf_and_feeds_simulator():
    from paper_2603_19289_b200 import ModelConfig, Session, engine
    s = Session(ModelConfig(**TOY), cache_fraction=0.5, max_positions=128)
    s.init_weights_seeded()
    d, _ = s.calibrate(64, 2, 32)
    s.load_default_vectors(d)
    s.set_predictor("router-pf")
    P, n = 4, 24
    S = P + n - 1
    s.reset(S, True)
    s.prefill([5, 6, 7, 8])
    s.decode("prefetch", n - 1)
    ids1 = s.predict_ahead(0, S, 1)
    pred = s.trace("id_pred", S).reshape(S, 8, 4)
    ex = s.trace("id_exec", S).reshape(S, 8, 4)
    steps = range(P, S)  # decode steps: the predictor ran on these
    for t in steps:
        for l in range(1, 8):
            assert sorted(ids1[t, l]) == sorted(pred[t, l]), (t, l)
    assert (ids1[:, 0] == -1).all()
    ids2 = s.predict_ahead(0, S, 2)
    assert (ids2[:, :2] == -1).all() and (ids2[:, 2:] >= 0).all()
    one = engine.simulate_cache(ex[P:], 0.014, 0.005, 0.021, 0.178, capacity=4, lookahead=1, pred_ids=ids1[P:])
    two = engine.simulate_cache(ex[P:], 0.014, 0.005, 0.021, 0.178, capacity=8, lookahead=2, pred_ids=ids1[P:],
                                pred2_ids=ids2[P:])
    assert one["tpot"] > 0 and two["tpot"] > 0
    s.close()
