"""The CPU oracle (oracle/specmoe_oracle.c) pinned against fixtures produced by
the reference library itself (tests/golden/make_golden.py), plus the SPEC
invariants the reference states but never tests."""
import os

import numpy as np
import pytest

from oracle.bindings import Config

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TINY = dict(layers=3, experts=6, top_k=2, hidden=16, expert_hidden=24, vocab=32, head_dim=8,
            seed=11)
BASE = dict(layers=4, experts=32, top_k=4, hidden=512, expert_hidden=1024, vocab=256,
            head_dim=64, seed=1)
KINDS = ("none", "baseline-s", "router-pf", "est-pf", "hybrid", "oracle")
HYBRID_TINY = ["router-pf", "est-pf"]


def gold(name):
    return np.load(os.path.join(G, name))


# ---------------------------------------------------------------- numerics --

def test_softmax_kats(orc):
    k = gold("kat.npz")
    for name, v in (("softmax_0000", [0, 0, 0, 0]), ("softmax_1000_0", [1000, 0]),
                    ("softmax_210", [2, 1, 0])):
        assert np.array_equal(orc.softmax(v), k[name])
    with pytest.raises(ValueError):
        orc.softmax([np.nan])


def test_softmax_sums_to_one(orc):  # test_numerics.cpp:32-45
    rng = np.random.default_rng(42)
    for _ in range(200):
        v = ((rng.random(int(rng.integers(1, 129))) * 2 - 1) * 1e4).astype(np.float32)
        p = orc.softmax(v)
        assert (p >= 0).all() and abs(p.astype(np.float64).sum() - 1.0) < 1e-5


def test_top_k_kats_and_ties(orc):
    k = gold("kat.npz")
    assert np.array_equal(orc.top_k([5, 1, 9], 1), k["topk_519_1"])
    assert np.array_equal(orc.top_k([3, 3, 3], 2), k["topk_333_2"])
    rng = np.random.default_rng(7)
    for _ in range(300):  # vs a stable full sort (test_numerics.cpp:72-90)
        n = int(rng.integers(1, 65))
        kk = int(rng.integers(1, n + 1))
        v = (rng.integers(0, 8, n)).astype(np.float32)
        want = np.argsort(-v, kind="stable")[:kk]
        assert np.array_equal(orc.top_k(v, kk), want)
    with pytest.raises(ValueError):
        orc.top_k([1, 2], 3)


def test_rms_norm_and_silu_kats(orc):
    k = gold("kat.npz")
    assert np.array_equal(orc.rms_norm([1, 1, 1, 1], [1, 1, 1, 1], 1e-12), k["rms_ones"])
    assert np.array_equal(orc.rms_norm([0, 0, 0], [2, 3, 4], 1e-5), k["rms_zero"])
    assert np.array_equal(orc.rms_norm([3, 4], [1, 1], 0.0), k["rms_34"])
    got = np.array([orc.silu(x) for x in (0.0, 30.0, 1.0, -3.5, 1e-3)], np.float32)
    assert np.array_equal(got, k["silu"])


def test_make_decision_vs_reference(orc):
    """router/make_decision cases incl. forced ties, both gating orders, bit-exact."""
    k = gold("kat.npz")
    for row, ids, gates in zip(k["dec_in"], k["dec_ids"], k["dec_gates"]):
        E, kk, gating = int(row[0]), int(row[1]), int(row[2])
        gi, gg = orc.make_decision(row[3:3 + E], kk, gating)
        assert np.array_equal(gi, ids[:kk])
        assert np.array_equal(gg, gates[:kk])


def test_linear_and_rng(orc):
    k = gold("kat.npz")
    assert np.array_equal(orc.linear(k["linear_w"], k["linear_x"]), k["linear_y"])
    seeds = [orc.derive_seed(s, l) for s, l in [(0, "embedding"), (11, "layer2.expert5.w_down"),
                                               (1, "token-stream"), (7, "estimator.a")]]
    assert np.array_equal(np.array(seeds, np.uint64), k["derive_seed"])
    g = orc.gaussian_stream(12345, np.float32(0.4) / np.sqrt(np.float32(16)), 257)
    assert np.array_equal(g, k["gauss"])


# ------------------------------------------------------------------- model --

def test_weights_match_reference_init(orc):
    c = gold("tiny_common.npz")
    m = orc.build_model(Config(**TINY), round_bf16=True)
    raw = orc.build_model(Config(**TINY), round_bf16=False)
    assert np.array_equal(m.tensor("layer1.expert5.w_down"), c["w_l1e5_down"])
    assert np.array_equal(raw.tensor("layer1.expert5.w_down"), c["w_l1e5_down_f32"])
    assert np.array_equal(raw.tensor("embedding"), c["w_emb_f32"])
    assert np.array_equal(m.tensor("layer2.gate"), c["w_l2_gate"])


@pytest.fixture(scope="module")
def tiny_setup(orc):
    c = gold("tiny_common.npz")
    m = orc.build_model(Config(**TINY), round_bf16=True)
    table = orc.table(c["dv"], c["dv_counts"])
    est = orc.estimator(TINY["hidden"], 2, 4, TINY["experts"], TINY["layers"], flat=c["est_flat"])
    return m, table, est, c


def test_default_vectors_match_reference(orc, tiny_setup):
    m, _, _, c = tiny_setup
    t = m.calibrate(200, 2, 16)
    assert np.array_equal(np.array(t.d), c["dv"])
    assert np.array_equal(np.array(t.counts), c["dv_counts"])


def test_estimator_init_matches_reference(orc, tiny_setup):
    _, _, _, c = tiny_setup
    est = orc.estimator(TINY["hidden"], 2, 4, TINY["experts"], TINY["layers"], seed=5)
    assert np.array_equal(np.array(est.flat), c["est_flat"])


@pytest.mark.parametrize("kind", KINDS)
def test_generation_traces_match_reference(orc, tiny_setup, kind):
    """speculative_forward / forward_decode per-(step, layer) records, bit-exact."""
    m, table, est, c = tiny_setup
    g = gold(f"tiny_{kind}.npz")
    pred = None if kind == "none" else orc.make_predictor(
        kind, m, table, est, HYBRID_TINY if kind == "hybrid" else None)
    t = m.generate_trace(c["prompt"], int(c["n_new"]), pred, outputs=True)
    for f in ("tokens", "s", "r", "m", "logits", "ids", "gates", "outputs", "final_logits"):
        assert np.array_equal(getattr(t, f), g[f]), f
    if pred is not None:
        for f in ("pred_logits", "pred_ids", "pred_gates"):
            assert np.array_equal(getattr(t, f), g[f]), f


def test_baseline_config_generation(orc):
    """BASELINE configs[0] (L4 H512 E32 k4): 64 tokens, true router and router-pf
    with the reference's 2000-token default vectors, ids bit-exact."""
    g = gold("baseline.npz")
    m = orc.build_model(Config(**BASE), round_bf16=True)
    table = orc.table(g["dv"], g["dv_counts"])
    for kind in ("none", "router-pf"):
        pred = None if kind == "none" else orc.make_predictor(kind, m, table)
        t = m.generate_trace(g["prompt"], 64, pred)
        assert np.array_equal(t.tokens, g[f"{kind}_tokens"])
        assert np.array_equal(t.ids, g[f"{kind}_ids"])
        assert np.array_equal(t.final_logits[-8:], g[f"{kind}_final_logits"])
        if pred is not None:
            assert np.array_equal(t.pred_ids, g[f"{kind}_pred_ids"])


# ----------------------------------------------------- SPEC invariants -------

def test_oracle_equivalence(orc, tiny_setup):
    """speculative decode with the Oracle predictor is bit-identical
    to the true path."""
    m, _, _, c = tiny_setup
    a = m.generate_trace(c["prompt"], 12)
    b = m.generate_trace(c["prompt"], 12, orc.make_predictor("oracle", m))
    for f in ("tokens", "s", "m", "ids", "gates", "final_logits"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


def test_zero_table_router_pf_is_router_on_normed_residual(orc, tiny_setup):
    """d = 0 collapses router-pf to the router over rms_norm(r_l)."""
    m, _, _, c = tiny_setup
    L, E, H = TINY["layers"], TINY["experts"], TINY["hidden"]
    zero = orc.table(np.zeros((L, E, H), np.float32))
    t = m.generate_trace(c["prompt"], 6, orc.make_predictor("router-pf", m, zero))
    P = len(c["prompt"])
    for s in range(P, t.r.shape[0]):
        for l in range(L - 1):
            q = orc.rms_norm(t.r[s, l], m.tensor(f"layer{l + 1}.moe_norm_gain"), 1e-5)
            lg = orc.linear(m.tensor(f"layer{l + 1}.gate").reshape(E, H), q)
            assert np.array_equal(lg, t.pred_logits[s, l])


def test_single_expert_model_identical_to_true_path(orc):
    """SPEC.md:251 example — E=1, k=1 with any predictor equals the true path."""
    cfg = Config(layers=3, experts=1, top_k=1, hidden=16, expert_hidden=8, vocab=32, head_dim=4,
                 seed=3)
    m = orc.build_model(cfg)
    table = m.calibrate(16, 2, 8)
    a = m.generate_trace([1, 2, 3], 6)
    b = m.generate_trace([1, 2, 3], 6, orc.make_predictor("router-pf", m, table))
    assert np.array_equal(a.tokens, b.tokens)
    assert np.array_equal(a.final_logits, b.final_logits)


def test_recall_at_k(orc):
    assert orc.recall_at_k([1, 2, 3, 4], [4, 3, 9, 8]) == 0.5
    assert orc.recall_at_k([1, 2], [1, 2]) == 1.0


# ------------------------------------------- oracle vs the reference itself --

@pytest.mark.parametrize("gating", ["softmax-topk-renorm", "topk-softmax"])
def test_oracle_vs_reference_library_live(orc, ref, gating):
    """Where the reference library is built (this container), run both on a fresh
    config with the topk-softmax gating order too."""
    cfg = Config(layers=4, experts=12, top_k=3, hidden=32, expert_hidden=40, vocab=64,
                 head_dim=8, seed=21, gating=gating)
    rm, om = ref.build_model(cfg), orc.build_model(cfg)
    rt = rm.calibrate(64, 2, 16)
    ot = om.calibrate(64, 2, 16)
    d, cnt = ref.table_get(rt)
    assert np.array_equal(d, np.array(ot.d))
    pr = ref.make_predictor("router-pf", cfg.layers, rt)
    po = orc.make_predictor("router-pf", om, ot)
    a = rm.generate_trace([5, 9, 2], 10, pr, outputs=True)
    b = om.generate_trace([5, 9, 2], 10, po, outputs=True)
    for f in ("tokens", "s", "m", "logits", "ids", "gates", "outputs", "final_logits",
              "pred_ids", "pred_gates", "pred_logits"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


def test_handle_views_keep_their_handle_alive():
    """`np.array(model.calibrate(...).d)` drops the table handle while its
    view is read: the view must keep the C table alive (the bench's
    reference arm crashed on exactly this expression)."""
    import gc
    from oracle.bindings import Config, Oracle
    cfg = Config(layers=2, experts=8, top_k=2, hidden=64, expert_hidden=96, vocab=64, head_dim=16, seed=3)
    om = Oracle().build_model(cfg, round_bf16=True)
    held = om.calibrate(16, 2, 16)
    want = np.array(held.d)
    v = om.calibrate(16, 2, 16).d  # the table handle is unreachable except through the view
    gc.collect()
    _ = [np.zeros(1 << 16) for _ in range(8)]  # churn the allocator
    assert np.array_equal(np.array(v), want)
    assert np.array_equal(np.array(om.calibrate(16, 2, 16).d), want)
