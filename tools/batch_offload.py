"""Batched decode under offload, speculative prefetch vs on-demand (BASELINE
configs 2-3; VERDICT r01 "configs 2-3 under offload").

    python tools/batch_offload.py g20 [steps] [cache] [B ...]
    python tools/batch_offload.py mx  [steps] [cache] [B ...]

g20: GPT-OSS-20B shape (24 layers, 32 experts top-4, H = Hm = 2880, topk-softmax),
     router-pf predictor.
mx:  Mixtral-8x7B shape (32 layers, 8 experts top-2, H 4096, Hm 14336,
     topk-softmax) with the lightweight estimator (est-pf, d/m = 512 latent,
     n = 4): trained on the GPU by KL distillation (smoe_train_estimator) on a
     decode captured from the same model, as the paper prescribes.
Weights seeded bf16, default vectors from a 64-token GPU calibration, 8-token
random prompts; for each B: smoe_batch_generate in both modes with the HBM
expert cache capped at `cache` of the experts per layer; wall clock per batch
step (prompt excluded), tokens/s, expert bytes copied.  Prints one JSON line.
Tools only.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2603_19289_b200 import ModelConfig, Session, engine  # noqa: E402

CFG = {
    "g20": dict(layers=24, experts=32, top_k=4, hidden=2880, expert_hidden=2880, vocab=256, head_dim=64, seed=1,
                gating="topk-softmax"),
    "mx": dict(layers=32, experts=8, top_k=2, hidden=4096, expert_hidden=14336, vocab=256, head_dim=128, seed=1,
               gating="topk-softmax"),
}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "g20"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    frac = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
    batches = [int(x) for x in sys.argv[4:]] or ([1, 2, 4, 8] if name == "g20" else [1, 2, 4, 8, 16])
    c = dict(CFG[name])
    t0 = time.time()
    s = Session(ModelConfig(**c), cache_fraction=1.0, max_positions=300)
    s.init_weights_seeded()
    s.preload_all()
    d, _ = s.calibrate(64, 2, 256)
    pred = "router-pf"
    info = {"config": name, "cache_fraction": frac, "steps": steps, "prompt_len": 8}
    if name == "mx":  # est-pf with a GPU-distilled estimator
        L, H, E = c["layers"], c["hidden"], c["experts"]
        m, n = 8, 4
        rng = np.random.default_rng(1)
        T = 96
        s.reset(T + 8, True)
        s.prefill(list(rng.integers(0, 256, 8)))
        s.decode_stream("on_demand", rng.integers(0, 256, T).astype(np.int32))
        inp, tgt = s.build_distill_dataset(8, T, "quasi")
        flat, curve, ms = engine.train_estimator(inp, tgt, H, m, n, E, L, seed=1, lr=1e-3, batch=32,
                                                 max_steps=150, eval_every=50, val_fraction=0.1, hseed=1,
                                                 k=c["top_k"])
        s.load_estimator(H, m, n, E, L, 1e-5, flat)
        pred = "est-pf"
        info["estimator"] = {"latent": H // m, "mlp": H // m * n, "train_tokens": T, "steps": 150,
                             "val_hit_rate": float(curve[-1][2]), "train_ms": ms}
    s.set_predictor(pred)
    s.set_cache_fraction(frac)
    info["predictor"] = pred
    info["slots_per_layer"] = s.cache_slots()
    info["setup_s"] = time.time() - t0
    rng = np.random.default_rng(0)
    rows = []
    for B in batches:
        pr = rng.integers(0, 256, (B, 8)).astype(np.int32)
        row = {"B": B}
        for mode in ("on_demand", "prefetch"):
            s.batch_generate(pr, 2, mode)  # warm-up (batch buffers)
            s.clear_stats()
            _, ms = s.batch_generate(pr, steps + 1, mode, timing=True)
            cnt = s.counters()
            miss = int(cnt["misses"].sum())  # prompt steps included
            row[mode] = {"ms_per_step": ms, "tokens_per_s": B * 1e3 / ms, "expert_copies": miss,
                         "h2d_wire_bytes": int(cnt["h2d_bytes"])}  # packed store: ~0.75 of raw
        row["prefetch_gain_pct"] = 100.0 * (row["on_demand"]["ms_per_step"] - row["prefetch"]["ms_per_step"]) / \
            row["on_demand"]["ms_per_step"]
        rows.append(row)
        print(json.dumps(row), flush=True)
    info["rows"] = rows
    print(json.dumps(info))
    s.close()


if __name__ == "__main__":
    main()
