"""Generates tests/golden/*.npz from the REFERENCE LIBRARY ITSELF
(oracle/_ref/libspecmoe_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile).  Run in the build container (where /root/reference exists):

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures pin the C restatement (oracle/specmoe_oracle.c) and, through
it, the GPU path.  Contents:
  kat.npz       known-answer tests of test_numerics.cpp / test_model.cpp
                (softmax, top_k, rms_norm, silu, make_decision, linear,
                derive_seed, gaussian stream) evaluated by the reference.
  tiny_*.npz    tests/test_util.hpp tiny_config (L3 E6 k2 H16 Hm24 V32 D8,
                seed 11), bf16-rounded weights: per-step traces of greedy
                generation with every predictor kind.
  baseline.npz  BASELINE.json configs[0] (L4 H512 E32 k4; Hm 1024, vocab 256,
                head_dim 64 stated), seed 1: default vectors from 2000
                calibration tokens (seed 2, seq_len 256), a 16-token prompt
                (seed 3) and 64 generated tokens with router-pf and with the
                true router; executed / predicted ids per step.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.bindings import Config, Ref  # noqa: E402

TINY = dict(layers=3, experts=6, top_k=2, hidden=16, expert_hidden=24, vocab=32, head_dim=8,
            seed=11)
BASE = dict(layers=4, experts=32, top_k=4, hidden=512, expert_hidden=1024, vocab=256,
            head_dim=64, seed=1)
HYBRID_TINY = ["router-pf", "est-pf"]


def kat(ref: Ref):
    out = {}
    out["softmax_0000"] = ref.softmax([0, 0, 0, 0])
    out["softmax_1000_0"] = ref.softmax([1000, 0])
    out["softmax_210"] = ref.softmax([2, 1, 0])
    out["topk_519_1"] = ref.top_k([5, 1, 9], 1)
    out["topk_333_2"] = ref.top_k([3, 3, 3], 2)
    out["rms_ones"] = ref.rms_norm([1, 1, 1, 1], [1, 1, 1, 1], 1e-12)
    out["rms_zero"] = ref.rms_norm([0, 0, 0], [2, 3, 4], 1e-5)
    out["rms_34"] = ref.rms_norm([3, 4], [1, 1], 0.0)
    out["silu"] = np.array([ref.silu(x) for x in (0.0, 30.0, 1.0, -3.5, 1e-3)], np.float32)
    rng = np.random.default_rng(31)
    cases_l, cases_ids, cases_g = [], [], []
    for it in range(200):  # router vs exhaustive oracle (test_model.cpp:105-129) style inputs
        E = int(2 + rng.integers(0, 12))
        k = int(1 + rng.integers(0, E))
        lg = np.zeros(16, np.float32)
        lg[:E] = (rng.random(E) * 6 - 3).astype(np.float32)
        if it % 5 == 0:
            lg[:E] = np.round(lg[:E])  # forced ties
        for gating in (0, 1):
            ids, g = ref.make_decision(lg[:E], k, gating)
            a = np.full(16, -1, np.int32)
            a[:k] = ids
            b = np.zeros(16, np.float32)
            b[:k] = g
            cases_l.append(np.concatenate([[E, k, gating], lg]).astype(np.float32))
            cases_ids.append(a)
            cases_g.append(b)
    out["dec_in"] = np.stack(cases_l)
    out["dec_ids"] = np.stack(cases_ids)
    out["dec_gates"] = np.stack(cases_g)
    w = (rng.random((8, 4)) - 0.5).astype(np.float32)
    x = (rng.random(4) - 0.5).astype(np.float32)
    out["linear_w"], out["linear_x"], out["linear_y"] = w, x, ref.linear(w, x)
    out["derive_seed"] = np.array([ref.derive_seed(s, l) for s, l in
                                   [(0, "embedding"), (11, "layer2.expert5.w_down"),
                                    (1, "token-stream"), (7, "estimator.a")]], np.uint64)
    out["gauss"] = ref.gaussian_stream(12345, np.float32(0.4) / np.sqrt(np.float32(16)), 257)
    np.savez_compressed(os.path.join(HERE, "kat.npz"), **out)


def tiny(ref: Ref):
    cfg = Config(**TINY)
    m = ref.build_model(cfg, True)
    raw = ref.build_model(cfg, False)
    table = m.calibrate(200, 2, 16)
    d, cnt = ref.table_get(table)
    est = ref.estimator_init(TINY["hidden"], 2, 4, TINY["experts"], TINY["layers"], seed=5)
    prompt = np.array([3, 1, 4, 1, 5], np.int32)
    n_new = 8
    common = dict(prompt=prompt, n_new=n_new, dv=d, dv_counts=cnt,
                  est_flat=ref.estimator_flat(est),
                  w_l1e5_down=m.tensor("layer1.expert5.w_down"),
                  w_l1e5_down_f32=raw.tensor("layer1.expert5.w_down"),
                  w_emb_f32=raw.tensor("embedding"), w_l2_gate=m.tensor("layer2.gate"))
    np.savez_compressed(os.path.join(HERE, "tiny_common.npz"), **common)
    for kind in ("none", "baseline-s", "router-pf", "est-pf", "hybrid", "oracle"):
        pred = None if kind == "none" else ref.make_predictor(
            kind, cfg.layers, table, est, HYBRID_TINY if kind == "hybrid" else None)
        t = m.generate_trace(prompt, n_new, pred, outputs=True)
        rec = dict(tokens=t.tokens, s=t.s, r=t.r, m=t.m, logits=t.logits, ids=t.ids,
                   gates=t.gates, outputs=t.outputs, final_logits=t.final_logits)
        if pred is not None:
            rec.update(pred_logits=t.pred_logits, pred_ids=t.pred_ids, pred_gates=t.pred_gates)
        np.savez_compressed(os.path.join(HERE, f"tiny_{kind}.npz"), **rec)


def baseline(ref: Ref):
    from oracle.bindings import Oracle
    cfg = Config(**BASE)
    m = ref.build_model(cfg, True)
    table = m.calibrate(2000, 2, 256)
    d, cnt = ref.table_get(table)
    prompt = Oracle().token_stream(16, BASE["vocab"], 3)
    out = dict(dv=d, dv_counts=cnt, prompt=prompt)
    for kind in ("none", "router-pf"):
        pred = None if kind == "none" else ref.make_predictor(kind, cfg.layers, table)
        t = m.generate_trace(prompt, 64, pred)
        out[f"{kind}_tokens"] = t.tokens
        out[f"{kind}_ids"] = t.ids
        out[f"{kind}_true_ids"] = t.ids if pred is None else None
        out[f"{kind}_final_logits"] = t.final_logits[-8:]
        if pred is not None:
            out[f"{kind}_pred_ids"] = t.pred_ids
            # online ids: the true router on the speculative stream (for hit rates)
            out[f"{kind}_true_logits_last"] = t.logits[-1]
            tid = np.zeros_like(t.ids)
            for s in range(t.logits.shape[0]):
                for l in range(cfg.layers):
                    tid[s, l] = ref.make_decision(t.logits[s, l], cfg.top_k, 0)[0]
            out[f"{kind}_true_ids"] = tid
    out = {k: v for k, v in out.items() if v is not None}
    np.savez_compressed(os.path.join(HERE, "baseline.npz"), **out)


if __name__ == "__main__":
    r = Ref()
    kat(r)
    tiny(r)
    if "--no-baseline" not in sys.argv:
        baseline(r)
    print("golden fixtures written to", HERE)
