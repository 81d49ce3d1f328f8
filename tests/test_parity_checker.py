"""CPU test of the teacher-forced layer-wise checker (tests/parity_check.py)
itself: an oracle-produced decode, laid out like a GPU trace, must check clean
in both offload modes, and a single flipped bit in any recorded field must be
caught at the right (position, layer)."""
import numpy as np
import pytest

from oracle.bindings import Config, Oracle
from parity_check import check_traces

CFG = dict(layers=4, experts=8, top_k=2, hidden=32, expert_hidden=48, vocab=64, head_dim=16, seed=9)


def as_gpu_trace(orc, want, cfg, prompt, forced, spec):
    """The oracle's Trace in the GPU trace layout (smoe_read_trace fields)."""
    L, K, E = cfg["layers"], cfg["top_k"], cfg["experts"]
    S = want.s.shape[0]
    P = len(prompt)
    tr = {"s": want.s, "r": want.r, "m": want.m, "lg_true": want.logits, "y": want.outputs,
          "logits": want.final_logits, "id_exec": want.ids, "g_exec": want.gates, "P": P}
    tr["id_true"] = np.zeros((S, L, K), np.int32)
    tr["g_true"] = np.zeros((S, L, K), np.float32)
    for t in range(S):
        for l in range(L):
            tr["id_true"][t, l], tr["g_true"][t, l] = orc.make_decision(want.logits[t, l], K, 0)
    tr["id_pred"] = np.full((S, L, K), -1, np.int32)
    tr["g_pred"] = np.zeros((S, L, K), np.float32)
    tr["lg_pred"] = np.zeros((S, L, E), np.float32)
    if spec:
        tr["id_pred"][:, 1:] = want.pred_ids
        tr["g_pred"][:, 1:] = want.pred_gates
        tr["lg_pred"][:, 1:] = want.pred_logits
    tr["tok_in"] = np.concatenate([prompt, forced[: S - P]]).astype(np.int32)
    tr["tokens"] = np.argmax(want.final_logits, axis=1).astype(np.int32)
    return tr


@pytest.fixture(scope="module")
def setup():
    orc = Oracle()
    om = orc.build_model(Config(**CFG), round_bf16=True)
    table = om.calibrate(48, 2, 16)
    lazy = orc.build_model(Config(**CFG), round_bf16=True, lazy=True)
    prompt = np.array([3, 14, 15, 9], np.int32)
    forced = np.array([(7 * i + 5) % CFG["vocab"] for i in range(12)], np.int32)
    runs = {}
    for mode in ("on_demand", "prefetch"):
        pred = orc.make_predictor("router-pf", om, table) if mode == "prefetch" else None
        want = om.generate_trace(prompt, 13, pred, outputs=True, forced=forced)
        runs[mode] = as_gpu_trace(orc, want, CFG, prompt, forced, mode == "prefetch")
    return orc, lazy, np.array(table.d), runs


def test_oracle_trace_checks_clean(setup):
    orc, lazy, table, runs = setup
    reps = check_traces(orc, lazy, CFG, [(m, runs[m], m) for m in runs], table=table, threads=4)
    for m, rep in reps.items():
        assert rep.ok(), (m, rep.summary())
        assert not rep.near_ties
        assert all(rep.exact[f] == rep.checked[f] for f in rep.checked)
        assert rep.checked["y"] == runs[m]["s"].shape[0] * CFG["layers"] * CFG["top_k"]
    assert reps["prefetch"].checked["lg_pred"] > 0


@pytest.mark.parametrize("field,where", [("r", (6, 2)), ("y", (9, 1)), ("lg_pred", (7, 3)),
                                         ("m", (5, 0)), ("logits", (8, None))])
def test_one_flipped_bit_is_caught(setup, field, where):
    orc, lazy, table, runs = setup
    tr = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in runs["prefetch"].items()}
    t, l = where
    a = tr[field]
    idx = (t,) if l is None else (t, l)
    flat = a[idx].reshape(-1).view(np.uint32)
    flat[0] ^= 1
    rep = check_traces(orc, lazy, CFG, [("p", tr, "prefetch")], table=table, threads=4)["p"]
    assert not rep.ok()
    hits = {(f, tt, ll) for f, tt, ll, _ in rep.mismatches}
    expect = {"r": "attn_r", "y": "y", "lg_pred": "lg_pred", "m": "m", "logits": "logits"}[field]
    assert any(f == expect and tt == t and (l is None or ll == l) for f, tt, ll in hits), rep.summary()
