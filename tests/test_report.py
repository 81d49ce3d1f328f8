"""Reporting in the C ABI vs the reference library itself:
the two-lane schedule simulator, breakdown, Eq. 1, per-token breakdown of a
measured event log, recall@k / rank alignment.  Host-only: runs without a GPU."""
import ctypes as C

import numpy as np
import pytest

from paper_2603_19289_b200 import Event, breakdown, recall_at_k, simulate


@pytest.mark.parametrize("seed", range(6))
def test_simulator_matches_reference(ref, seed):
    rng = np.random.default_rng(seed)
    L = int(rng.integers(1, 50))
    a, g, e, c = (rng.random(L) * s for s in (3.0, 0.5, 2.0, 12.0))
    cold = -1.0 if seed % 2 else float(rng.random() * 20)
    for mode in ("on_demand", "prefetch"):
        tp, fr, an = simulate(a, g, e, c, mode, cold)
        rtp, rfr, ran = ref.simulate(a, g, e, c, mode == "prefetch", cold)
        assert tp == rtp and an == ran
        assert np.array_equal(fr, rfr)


def test_spec_examples():
    """SPEC.md examples: uniform 1/1/10/2 over 48 layers -> 672; copy = compute ->
    analytic speedup 2; t_copy = 0 -> both modes equal sum of compute."""
    L = 48
    tp, fr, _ = simulate([1] * L, [1] * L, [2] * L, [10] * L, "on_demand")
    assert tp == 672.0 and abs(fr[1] - 10 / 14) < 1e-12
    _, _, an = simulate([1] * L, [1] * L, [2] * L, [4] * L, "prefetch")
    assert an == 4 * L
    t0, _, _ = simulate([1] * L, [1] * L, [2] * L, [0] * L, "prefetch")
    t1, _, _ = simulate([1] * L, [1] * L, [2] * L, [0] * L, "on_demand")
    assert t0 == t1 == 4 * L
    with pytest.raises(ValueError, match="negative"):
        simulate([-1], [0], [0], [0], "on_demand")


def test_breakdown_of_event_log_matches_reference(ref):
    rng = np.random.default_rng(3)
    evs = []
    for tok in range(5):
        t = tok * 1000.0
        for l in range(6):
            for kind, d in ((0, rng.random() * 5), (1, rng.random()), (2, rng.random() * 3)):
                evs.append(Event(0, kind, l, tok, t, t + d))
                t += d
            s0 = t - rng.random() * 4
            evs.append(Event(1, 3, l, tok, s0, s0 + rng.random() * 10))
    fr, tp = breakdown(evs)
    n = len(evs)
    cols = [np.array([getattr(e, f) for e in evs], np.int32) for f in ("lane", "kind", "layer", "token")]
    st = np.array([e.start_ms for e in evs], np.float64)
    en = np.array([e.end_ms for e in evs], np.float64)
    rfr = np.zeros(3)
    rtp = C.c_double()
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    assert ref.lib.ref_breakdown_events(*[p(c) for c in cols], p(st), p(en), n, p(rfr),
                                        C.byref(rtp)) == 0
    assert np.allclose(fr, rfr, rtol=0, atol=1e-12) and abs(tp - rtp.value) < 1e-9
    assert abs(fr.sum() - 1.0) < 1e-9


def test_recall_and_rank_alignment(orc):
    r, m = recall_at_k([3, 1, 4, 9], [4, 3, 8, 9])
    assert r == orc.recall_at_k([3, 1, 4, 9], [4, 3, 8, 9]) == 0.75
    assert list(m) == [False, False, False, True]


def _disjoint_trace(T, L, K):
    """Every (token, layer) executes K experts never used before: every request misses."""
    ids = np.arange(T, dtype=np.int32)[:, None, None] * K + np.arange(K, dtype=np.int32)[None, None, :]
    return np.ascontiguousarray(np.broadcast_to(ids, (T, L, K)))


@pytest.mark.parametrize("seed", range(4))
def test_cache_simulator_reduces_to_reference_when_all_miss(ref, seed):
    """Cache model pinned to the reference's simulate_on_demand /
    simulate_prefetch (schedule.cpp:92-148): capacity k per layer, each token's
    experts new, predictions exact -> every layer copies k experts, prefetched one
    layer ahead; per-layer copy = k * t_copy_expert."""
    from paper_2603_19289_b200 import engine
    rng = np.random.default_rng(seed)
    T, L, K = 5, int(rng.integers(2, 20)), int(rng.integers(1, 9))
    a, g, e = (rng.integers(0, 16, L).astype(np.float64) * 0.25 for _ in range(3))
    tc = float(rng.integers(1, 12)) * 0.25
    ids = _disjoint_trace(T, L, K)
    for la, mode in ((0, False), (1, True)):
        got = engine.simulate_cache(ids, a, g, e, tc, capacity=K, lookahead=la, pred_ids=ids)
        rtp, _, _ = ref.simulate(a, g, e, np.full(L, K * tc), mode, -1.0)
        assert got["tpot"] == pytest.approx(rtp, rel=1e-12)
        assert got["stall_copies"] == (L * K if la == 0 else K)
        assert got["useful_prefetch"] == (0 if la == 0 else (L - 1) * K)


def test_cache_simulator_hits_and_lookahead():
    from paper_2603_19289_b200 import engine
    rng = np.random.default_rng(0)
    T, L, K, E = 64, 8, 4, 16
    ids = np.stack([np.stack([rng.choice(E, K, replace=False) for _ in range(L)]) for _ in range(T)]).astype(np.int32)
    base = dict(t_attn=1.0, t_gate=0.25, t_expert=2.0, t_copy_expert=1.5)
    # resident working set: no copies after warm-up, TPOT = sum of compute
    r = engine.simulate_cache(ids, **base, capacity=E, lookahead=0, warm_tokens=T // 2)
    assert r["stall_copies"] == 0 and r["tpot"] == pytest.approx(L * 3.25)
    # exact predictions: one-ahead hides copies, two-ahead hides at least as much
    lo = engine.simulate_cache(ids, **base, capacity=K, lookahead=0)
    one = engine.simulate_cache(ids, **base, capacity=2 * K, lookahead=1, pred_ids=ids)
    two = engine.simulate_cache(ids, **base, capacity=3 * K, lookahead=2, pred_ids=ids, pred2_ids=ids)
    assert one["tpot"] < lo["tpot"] and two["tpot"] <= one["tpot"]
    assert two["stall_copies"] <= one["stall_copies"] <= lo["stall_copies"]
    lfu = engine.simulate_cache(ids, **base, capacity=K + 2, policy="lfu", lookahead=1, pred_ids=ids)
    assert lfu["tpot"] > 0
    with pytest.raises(ValueError, match="lookahead 2"):
        engine.simulate_cache(ids, **base, capacity=K, lookahead=2, pred_ids=ids)
