"""Hybrid-map selection from per-layer hit rates
and per-layer online hit rates, host-only (no GPU)."""
import json

import numpy as np
import pytest

from paper_2603_19289_b200 import hybrid_map_json, layer_hit_rates, select_hybrid_map


def test_layer_hit_rates_are_recall_at_k_per_layer():
    rng = np.random.default_rng(0)
    steps, L, k = 7, 5, 3
    true = np.stack([[rng.permutation(10)[:k] for _ in range(L)] for _ in range(steps)]).astype(np.int32)
    exe = true.copy()
    exe[:, 2, 0] = 99          # one miss per step at layer 2
    exe[::2, 4, :] = 98        # all miss on even steps at layer 4
    r = layer_hit_rates(exe, true)
    assert r.shape == (L - 1,)
    want = [1.0, 2 / 3, 1.0, 1.0 - 4 / 7]
    assert np.allclose(r, want)


def test_select_best_per_layer_and_threshold_rule():
    rates = {"router-pf": [0.9, 0.4, 0.7, 0.95], "est-pf": [0.8, 0.6, 0.7, 0.99],
             "baseline-s": [0.5, 0.65, 0.2, 0.1]}
    # best per layer, ties to the earlier candidate
    assert select_hybrid_map(rates) == ["router-pf", "baseline-s", "router-pf", "est-pf"]
    # the paper's rule: router-pf unless its hit rate is low, then the best other
    assert select_hybrid_map(rates, threshold=0.75) == ["router-pf", "baseline-s", "est-pf", "router-pf"]
    m = json.loads(hybrid_map_json(["router-pf", "est-pf"]))
    assert m == {"0": "router-pf", "1": "est-pf"}  # load_hybrid_map's format


def test_select_rejects_non_concrete_kinds():
    with pytest.raises(ValueError, match="concrete"):
        select_hybrid_map({"router-pf": [0.5], "oracle": [0.9]})
