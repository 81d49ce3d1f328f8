"""Exploratory GPU-vs-oracle comparison (prints a report; tests/ holds the asserts)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle.bindings import Config, Oracle  # noqa: E402
from paper_2603_19289_b200 import ModelConfig, Session  # noqa: E402


def cmp(name, a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        print(f"  {name}: SHAPE {a.shape} vs {b.shape}")
        return
    eq = np.mean(a == b) if a.size else 1.0
    md = float(np.max(np.abs(a.astype(np.float64) - b.astype(np.float64)))) if a.size else 0.0
    print(f"  {name}: exact {eq:.6f} maxdiff {md:.3e}")


def run(cfg, P=5, n_new=8, kinds=("none", "router-pf", "baseline-s", "oracle", "est-pf", "hybrid"),
        frac=0.5):
    orc = Oracle()
    om = orc.build_model(Config(**cfg), True)
    t0 = time.time()
    table = om.calibrate(128, 2, 32)
    print("oracle calibrate", time.time() - t0)
    E, L, H = cfg["experts"], cfg["layers"], cfg["hidden"]
    est = orc.estimator(H, 2, 4, E, L, seed=5)
    s = Session(ModelConfig(**cfg), cache_fraction=frac, max_positions=256)
    t0 = time.time()
    s.init_weights_seeded()
    print("gpu init", time.time() - t0)
    t0 = time.time()
    d, cnt = s.calibrate(128, 2, 32)
    print("gpu calibrate", time.time() - t0)
    cmp("dv", d, table.d)
    cmp("dv counts", cnt, table.counts)
    s.load_estimator(H, 2, 4, E, L, 1e-5, np.array(est.flat))
    rng = np.random.default_rng(0)
    prompt = rng.integers(0, cfg["vocab"], P).astype(np.int32)
    for kind in kinds:
        hyb = None
        if kind == "hybrid":
            hyb = [["router-pf", "est-pf", "baseline-s"][l % 3] for l in range(L - 1)]
        pred = None if kind == "none" else orc.make_predictor(kind, om, table, est, hyb)
        want = om.generate_trace(prompt, n_new, pred, outputs=True)
        if kind != "none":
            s.set_predictor(kind, hyb)
        modes = ["on_demand"] if kind == "none" else ["prefetch"]
        for mode in modes:
            S = P + n_new - 1
            s.reset(S, True)
            s.prefill(prompt)
            s.decode(mode, n_new - 1)
            toks = s.tokens(S)[P - 1:]
            print(f"[{kind}/{mode}] tokens gpu {list(toks)} oracle {list(want.tokens)}")
            cmp("s", s.trace("s", S), want.s)
            cmp("r", s.trace("r", S), want.r)
            cmp("m", s.trace("m", S), want.m)
            cmp("logits_true", s.trace("lg_true", S), want.logits)
            cmp("ids_exec", s.trace("id_exec", S), want.ids)
            cmp("gates_exec", s.trace("g_exec", S), want.gates)
            cmp("y", s.trace("y", S), want.outputs)
            cmp("final", s.trace("logits", S), want.final_logits)
            if kind != "none":
                gp = s.trace("id_pred", S)[:, 1:, :]
                cmp("pred_ids(decode)", gp[P:], want.pred_ids[P:])
                cmp("pred_logits(decode)", s.trace("lg_pred", S)[P:, 1:, :], want.pred_logits[P:])
            c = s.counters()
            print("  counters", c["hits"].sum(), c["misses"].sum(), c["h2d_bytes"], c["requests"],
                  "copy_ms", round(c["copy_ms"], 3))
    s.close()


if __name__ == "__main__":
    tiny = dict(layers=3, experts=6, top_k=2, hidden=16, expert_hidden=24, vocab=32, head_dim=8,
                seed=11)
    toy = dict(layers=8, experts=16, top_k=4, hidden=64, expert_hidden=128, vocab=256,
               head_dim=32, seed=4)
    run(tiny, kinds=("none", "router-pf"))
    run(toy)
    big = dict(layers=4, experts=32, top_k=4, hidden=512, expert_hidden=1024, vocab=256,
               head_dim=64, seed=1)
    run(big, P=8, n_new=16, kinds=("none", "router-pf"), frac=0.25)
