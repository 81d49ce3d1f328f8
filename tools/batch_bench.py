"""Batched decode throughput (BASELINE configs 2-3: batch 1-16) on one B200.

    python tools/batch_bench.py [config] [steps] [cache_fraction]

config: q30 | g20 (GPT-OSS-20B shape, 24 layers) | g20-8 (depth 8).  For B in
1, 2, 4, 8, 16: decode `steps` tokens per sequence through
smoe_batch_generate after an 8-token prompt and print tokens/s and ms per
batch step (the batch buffers allocated by a warm-up call; wall clock per decode step,
prompt excluded).  The single-sequence graph decode TPOT is printed for reference.
Tools only.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2603_19289_b200 import ModelConfig, Session  # noqa: E402

CFG = {
    "q30": dict(layers=48, experts=128, top_k=8, hidden=2048, expert_hidden=768, vocab=256, head_dim=128, seed=1),
    "g20": dict(layers=24, experts=32, top_k=4, hidden=2880, expert_hidden=2880, vocab=256, head_dim=64, seed=1,
                gating="topk-softmax"),
}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "g20"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    frac = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
    c = dict(CFG[name.split("-")[0]])
    if "-" in name:
        c["layers"] = int(name.split("-")[1])
    s = Session(ModelConfig(**c), cache_fraction=1.0, max_positions=300)
    s.init_weights_seeded()
    s.preload_all()
    d, _ = s.calibrate(64, 2, 256)
    s.load_default_vectors(d)
    s.set_predictor("router-pf")
    s.set_cache_fraction(frac)
    P = 8
    rng = np.random.default_rng(0)
    for mode in ("prefetch", "on_demand"):
        _, per = s.run_offloaded_decode(list(rng.integers(0, 256, P)), steps + 1, mode)
        print(f"{name} {mode}: single-sequence graph decode TPOT {np.mean(per):.3f} ms")
        for B in (1, 2, 4, 8, 16):
            pr = rng.integers(0, 256, (B, P)).astype(np.int32)
            s.batch_generate(pr, 3, mode)  # warm-up (allocates the batch buffers)
            _, ms = s.batch_generate(pr, steps + 1, mode, timing=True)
            print(f"  B={B:2d}: {ms:7.3f} ms per batch step, {B * 1e3 / ms:8.1f} tokens/s")

if __name__ == "__main__":
    main()
