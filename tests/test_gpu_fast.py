"""Tolerance decode mode (smoe_set_decode_mode(1): packed-FFMA partial sums in
every decode GEMV, column-split GEMVs for qkv / routers / unembed) against the
CPU oracle, teacher-forced layer by layer (tests/parity_check.py with rtol):

* every hidden-state / logit vector within RTOL of the reference's value on
  the GPU's own inputs (norm-relative error, the largest per field reported);
* router, predictor and executed ids, and the greedy token, equal to the
  reference's unless the oracle's gap at the deciding boundary is below
  EPS_TIE (reported as a near-tie, never hidden);
* in both offload modes, at the toy shape, the Qwen3-30B-A3B layer shapes
  and the headline run itself (48 layers, 25 % cache, calibrated default
  vectors, 32-token prompt, teacher-forced stream).

The exact mode (default) stays bit-identical (tests/test_gpu*.py)."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RTOL = 2e-5     # ||gpu - ref|| / ||ref|| per vector
EPS_TIE = 1e-5  # boundary gap (probabilities / logits) below which a flipped id is a near-tie

TOY = dict(layers=8, experts=16, top_k=4, hidden=64, expert_hidden=128, vocab=256, head_dim=32, seed=4)
Q30 = dict(layers=48, experts=128, top_k=8, hidden=2048, expert_hidden=768, vocab=256,
           head_dim=128, seed=1)


@pytest.fixture(scope="module")
def lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2603_19289_b200 import load_library
    return load_library()


def _report(name, obj):
    print(f"\n[parity-fast] {name}: {json.dumps(obj, default=str)}")
    d = os.environ.get("PARITY_REPORT_DIR")
    if d:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, f"{name}.json"), "w") as f:
            json.dump(obj, f, indent=1, default=str)


def _run(cfg, P, N, frac, calib, label):
    from oracle.bindings import Config, Oracle
    from paper_2603_19289_b200 import ModelConfig, Session
    from parity_check import check_traces, gpu_trace
    orc = Oracle()
    prompt = orc.token_stream(P, cfg["vocab"], 3)
    forced = orc.token_stream(N, cfg["vocab"], 4)
    s = Session(ModelConfig(**cfg), cache_fraction=1.0, max_positions=max(P + N + 8, 300))
    s.init_weights_seeded()
    s.preload_all()
    dv, _ = s.calibrate(calib, 2, 256)  # exact mode (the reference's accumulator)
    s.set_cache_fraction(frac)
    s.set_predictor("router-pf")
    s.set_decode_mode("fast")
    runs = []
    for mode in ("on_demand", "prefetch"):
        s.reset(P + N, True)
        s.prefill(prompt)
        s.decode_stream(mode, forced)
        runs.append((mode, gpu_trace(s, P + N, P), mode))
    s.close()
    om = orc.build_model(Config(**cfg), round_bf16=True, lazy=True)
    reps = check_traces(orc, om, cfg, runs, table=dv, eps_tie=EPS_TIE, rtol=RTOL)
    for mode, rep in reps.items():
        summ = rep.summary()
        summ.update({"config": label, "mode": mode, "decode_mode": "fast", "eps_tie": EPS_TIE})
        _report(f"fast_{label}_{mode}", summ)
        assert rep.ok(), summ
        assert 0 < rep.max_rel_err.get("m", 0.0) <= RTOL  # really a different summation, within RTOL
    return reps


def test_fast_mode_toy_teacher_forced(lib):
    _run(TOY, 12, 16, 0.5, 64, "toy")


def test_fast_mode_q30_layers_teacher_forced(lib):
    _run(dict(Q30, layers=3), 16, 8, 0.25, 256, "q30_L3")


def test_fast_mode_long_context_toy(lib):
    """Flash-decoding attention over 700+ positions (several CTAs, ragged slices)."""
    _run(dict(TOY, layers=3), 700, 6, 0.5, 64, "toy_long")


def test_fast_mode_two_level_attention_merge_toy(lib):
    """2200+ positions: more than 32 attention CTAs, so the partials merge in
    two levels (groups of 32, then the group partials)."""
    _run(dict(TOY, layers=2), 2200, 4, 0.5, 64, "toy_2k_two_level")


def test_fast_mode_long_context_q30_layers(lib):
    """head_dim 128 (float4 lanes) over 1100+ positions."""
    _run(dict(Q30, layers=2), 1100, 4, 0.25, 256, "q30_L2_long")


def test_fast_mode_headline_q30_48_layers(lib):
    """The bench's headline workload in the tolerance mode."""
    reps = _run(Q30, 32, 12, 0.25, 2000, "q30_L48")
    assert reps["prefetch"].checked["lg_pred"] == 12 * 47


def test_fast_mode_switch_rebuilds_graphs(lib):
    """Exact -> fast -> exact on one session: the exact tokens come back bit for bit."""
    from paper_2603_19289_b200 import ModelConfig, Session
    cfg = dict(TOY, layers=4)
    s = Session(ModelConfig(**cfg), cache_fraction=0.5, max_positions=64)
    s.init_weights_seeded()
    s.load_default_vectors(np.zeros((4, 16, 64), np.float32))
    s.set_predictor("router-pf")
    out = []
    for mode in ("exact", "fast", "exact"):
        s.set_decode_mode(mode)
        got, _ = s.run_offloaded_decode([3, 1, 4, 1, 5], 8, "prefetch")
        out.append(np.asarray(got))
    s.close()
    assert np.array_equal(out[0], out[2])


def test_fast_mode_one_launch_ffn_toy(lib, monkeypatch):
    """The opt-in one-launch tolerance FFN (k_ffn_cs, SMOE_FFN_CS_FUSED=1):
    gate/up units then claimed down items in one grid, same tolerance."""
    monkeypatch.setenv("SMOE_FFN_CS_FUSED", "1")
    _run(TOY, 12, 16, 0.5, 64, "toy_ffn_cs")


def test_fast_mode_column_split_down_toy(lib, monkeypatch):
    """The opt-in gate/up + column-split down path (k_ffn_gud + k_down_reduce,
    SMOE_FFN_GUD=1): each gate/up CTA also computes the down partial over its
    16 columns of h; the partials are summed in slice order. Same tolerance."""
    monkeypatch.setenv("SMOE_FFN_GUD", "1")
    _run(TOY, 12, 16, 0.5, 64, "toy_ffn_gud")


def test_fast_mode_column_split_down_q30_layers(lib, monkeypatch):
    """The same at the Q30 layer shape (Hm 768: 48 column slices, the 64-wide
    in-flight batches of the reduction), two layers, offloaded prefetch."""
    monkeypatch.setenv("SMOE_FFN_GUD", "1")
    _run(dict(Q30, layers=2), 10, 8, 0.25, 64, "q30_L2_ffn_gud")


def test_fast_mode_per_expert_down_toy(lib, monkeypatch):
    """The previous down projection (k_ffn_down: one warp per (row block,
    expert), last-of-k CTA mixes; SMOE_DOWN_RB=0) next to the default
    row-block kernel (k_ffn_down_rb) the other tests run. Same tolerance."""
    monkeypatch.setenv("SMOE_DOWN_RB", "0")
    _run(TOY, 12, 16, 0.5, 64, "toy_down_per_expert")


def test_fast_mode_per_expert_down_q30_layers(lib, monkeypatch):
    """The same at the Q30 layer shape, two layers, offloaded prefetch."""
    monkeypatch.setenv("SMOE_DOWN_RB", "0")
    _run(dict(Q30, layers=2), 10, 8, 0.25, 64, "q30_L2_down_per_expert")
