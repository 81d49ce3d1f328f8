"""Predictor choice for the headline workload (tools only; DESIGN.md §5 "Copy
overlap"): per-layer online hit rates of router-pf, baseline-s and est-pf on a
SELECTION stream (random_token_stream seed 5, never the bench's seed 4), the
hybrid map chosen from them (speculation.cpp:145-165 format, the paper's
best-per-layer rule), then the bench's stream workload (Q30, 25 % cache,
prompt seed 3, forced seed 4) decoded with each predictor in both offload
modes: TPOT, misses per token, recall.  Also saves the executed ids of each
predictor for tools/overlap_sim.py.

    python tools/hybrid_study.py [steps] [est_tokens]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    from paper_2603_19289_b200 import ModelConfig, Session, engine, layer_hit_rates, select_hybrid_map
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    est_tokens = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    dm = os.environ.get("SMOE_DECODE_MODE", "fast")
    c = dict(bench.CONFIGS["q30"])
    L, H, E, K = c["layers"], c["hidden"], c["experts"], c["top_k"]
    P, W, NS = 32, 4, 128
    cap = max(P + W + steps, P + NS, 256) + 16
    s = Session(ModelConfig(**c), cache_fraction=1.0, max_positions=cap)
    s.init_weights_seeded()
    s.preload_all()
    s.calibrate(2000, 2, 256)
    s.set_decode_mode(dm)
    out = {"decode_mode": dm}
    # est-pf: estimator distilled on the GPU from on-demand streams with
    # distinct prompts (seeds 100+i / 200+i; one stream overfits its context)
    t0 = time.time()
    m, n = 8, 4
    nst = max(1, est_tokens // 96)
    inps, tgts = [], []
    for i in range(nst):
        s.reset(32 + 96 + 8, True)
        s.prefill(list(bench.token_stream(32, c["vocab"], 100 + i)))
        s.decode_stream("on_demand", bench.token_stream(96, c["vocab"], 200 + i))
        a, b = s.build_distill_dataset(32, 96, "quasi")
        inps.append(a)
        tgts.append(b)
    inp, tgt = np.concatenate(inps), np.concatenate(tgts)
    steps_tr = int(os.environ.get("EST_STEPS", "1500"))
    flat, curve, ms = engine.train_estimator(inp, tgt, H, m, n, E, L, seed=1, lr=1e-3, batch=32,
                                             max_steps=steps_tr, eval_every=steps_tr // 5, val_fraction=0.1,
                                             hseed=1, k=K)
    s.load_estimator(H, m, n, E, L, 1e-5, flat)
    out["estimator"] = dict(train_tokens=int(inp.shape[0]), streams=nst, steps=steps_tr,
                            val_hit_rate=float(curve[-1][2]), train_ms=ms, wall_s=time.time() - t0)
    prompt = bench.token_stream(P, c["vocab"], 3)
    sel = bench.token_stream(NS, c["vocab"], 5)
    rates = {}
    for kind in ("router-pf", "baseline-s", "est-pf"):
        s.set_predictor(kind)
        s.reset(P + NS, False)
        s.prefill(prompt)
        s.decode_stream("prefetch", sel)
        rates[kind] = layer_hit_rates(s.trace("id_exec", P + NS)[P:], s.trace("id_true", P + NS)[P:])
    out["layer_hit_rates"] = {k: [round(float(x), 4) for x in v] for k, v in rates.items()}
    out["mean_hit_rate"] = {k: float(np.mean(v)) for k, v in rates.items()}
    hmap = select_hybrid_map(rates)
    out["hybrid_map"] = hmap
    out["hybrid_map_counts"] = {k: hmap.count(k) for k in set(hmap)}
    forced = bench.token_stream(W + steps, c["vocab"], 4)
    S = P + W + steps
    ids = {}
    res = {}
    for pred in ("router-pf", "hybrid"):
        if pred == "hybrid":
            s.set_predictor("hybrid", hmap)
        else:
            s.set_predictor(pred)
        # executed ids with experts resident (routing does not depend on the cache)
        s.set_cache_fraction(1.0)
        for mode in ("on_demand", "prefetch"):
            s.reset(S, False)
            s.prefill(prompt)
            s.decode_stream(mode, forced)
            ids[f"{pred}_{mode}"] = s.trace("id_exec", S)[P:]
            ids[f"{pred}_{mode}_true"] = s.trace("id_true", S)[P:]
        s.set_cache_fraction(0.25)
        r = {}
        for mode in ("on_demand", "prefetch"):
            tp, mi = [], []
            for run in range(3):
                s.reset(S, False)
                s.prefill(prompt)
                s.decode_stream(mode, forced[:W])
                s.clear_stats()
                s.decode_stream(mode, forced[W:])
                tp.append(float(np.mean(s.token_ms())))
                mi.append(int(s.counters()["misses"].sum()) / steps)
            r[mode] = dict(tpot_ms=tp, misses_per_token=mi)
        ex, tr = ids[f"{pred}_prefetch"], ids[f"{pred}_prefetch_true"]
        r["recall"] = float(np.mean([len(set(ex[t, l]) & set(tr[t, l])) / K
                                     for t in range(ex.shape[0]) for l in range(1, L)]))
        res[pred] = r
    out["stream"] = res
    s.close()
    path = os.path.join(ROOT, "gpurun_out", "hybrid_ids.npz")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    np.savez(path, **ids)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
