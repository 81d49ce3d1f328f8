"""Cache policy x prefetch lookahead on the Q30 stream workload.

    python tools/lookahead_study.py [steps] [calib_tokens]

Decodes the bench's headline workload (Q30 shape, 25 % cache, router-pf,
teacher-forced random_token_stream(4)) with full trace capture and measures
TPOT, then replays the captured executed ids through the cache simulator
(smoe_simulate_cache) with router-pf predictions 1 and 2 layers ahead computed
on the GPU from the same trace (smoe_predict_ahead).  The simulator's
per-layer compute times come from the resident decode TPOT split by the
device-side kernel timeline (profiles/r01_ktrace_q30_greedy.txt ratios), the
copy time from the measured link rate.  Tool only (prints a table).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2603_19289_b200 import ModelConfig, Session, engine  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    calib = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    c = dict(bench.CONFIGS["q30"])
    L, E, K = c["layers"], c["experts"], c["top_k"]
    P, W = 32, 8
    s = Session(ModelConfig(**c), cache_fraction=1.0, max_positions=max(P + W + steps + 16, 300))
    s.init_weights_seeded()
    s.preload_all()
    dv, _ = s.calibrate(calib, 2, 256)
    prompt = bench.token_stream(P, c["vocab"], 3)
    forced = bench.token_stream(W + steps, c["vocab"], 4)
    S = P + W + steps
    s.set_predictor("router-pf")

    def run(frac, mode):
        s.set_cache_fraction(frac)
        s.reset(S, True)
        s.prefill(prompt)
        s.decode_stream(mode, forced[:W])
        s.clear_stats()
        s.decode_stream(mode, forced[W:])
        return float(np.mean(s.token_ms()))

    resident = run(1.0, "prefetch")
    measured = {m: run(0.25, m) for m in ("on_demand", "prefetch")}
    # trace of the prefetch run (Algorithm 1): executed = predicted for l >= 1
    sl = slice(P + W, S)
    ex = s.trace("id_exec", S).reshape(S, L, K)[sl]
    true = s.trace("id_true", S).reshape(S, L, K)[sl]
    ids1 = s.predict_ahead(0, S, 1)[sl]
    ids2 = s.predict_ahead(0, S, 2)[sl]
    assert all(sorted(ids1[t, l]) == sorted(ex[t, l]) for t in range(len(ex)) for l in range(1, L))
    gbps = s.measure_link(32)
    expert_bytes = 3 * c["hidden"] * c["expert_hidden"] * 2
    t_copy = expert_bytes / (gbps * 1e6)  # ms per expert copy
    # per-layer compute split (device timeline, greedy resident: qkv+attn+wo 14.0,
    # router 5.0, gate/up+down 21.0 us of 40 us) scaled to the measured resident TPOT
    per_layer = resident / L
    ta, tg, te = per_layer * 14.0 / 40.0, per_layer * 5.0 / 40.0, per_layer * 21.0 / 40.0
    C = E // 4
    rows = []
    cases = [("on-demand (true ids)", 0, true, None, None),
             ("prefetch 1 ahead (Algorithm 1)", 1, ex, ids1, None),
             ("prefetch 1 ahead + warm 2 ahead", 2, ex, ids1, ids2)]
    for pol in ("lru", "lfu"):
        for name, la, exe, p1, p2 in cases:
            r = engine.simulate_cache(exe, ta, tg, te, t_copy, capacity=C, policy=pol, lookahead=la,
                                      pred_ids=p1, pred2_ids=p2, warm_tokens=4)
            rows.append(dict(case=name, policy=pol, **{k: round(v, 4) for k, v in r.items()}))
    # how much of the executed (1-ahead) set the 2-ahead prediction already names
    rec2 = np.mean([len(set(ids2[t, l]) & set(ex[t, l])) / K for t in range(len(ex)) for l in range(2, L)])
    rec1 = np.mean([len(set(ids1[t, l]) & set(true[t, l])) / K for t in range(len(ex)) for l in range(1, L)])
    out = dict(link_GBps=gbps, measured_tpot_ms=measured, resident_tpot_ms=resident, t_copy_expert_ms=t_copy,
               recall_1ahead_vs_true=rec1, overlap_2ahead_vs_executed=rec2, sim=rows)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
