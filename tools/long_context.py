"""Decode TPOT after a long prompt (tools only): Q30 shape, prompt through the
batched prefill, then teacher-forced decode steps; resident experts and the
25 % cache, both attention variants (SMOE_ATTN_SPLIT is read per process).

    python tools/long_context.py [prompt_len] [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2603_19289_b200 import ModelConfig, Session  # noqa: E402


def main():
    plen = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    c = dict(bench.CONFIGS["q30"])
    s = Session(ModelConfig(**c), cache_fraction=1.0, max_positions=plen + steps + 32)
    s.init_weights_seeded()
    s.preload_all()
    d, _ = s.calibrate(256, 2, min(256, plen + steps))
    s.load_default_vectors(d)
    s.set_predictor("router-pf")
    prompt = bench.token_stream(plen, c["vocab"], 5)
    forced = bench.token_stream(steps + 4, c["vocab"], 4)
    for frac in (1.0, 0.25):
        s.set_cache_fraction(frac)
        if frac == 1.0:
            s.preload_all()
        for mode in ("prefetch", "on_demand"):
            s.reset(plen + steps + 4, False)
            s.prefill_batched(prompt)
            s.decode_stream(mode, forced[:4])
            s.clear_stats()
            s.decode_stream(mode, forced[4:])
            cnt = s.counters()
            print(f"prompt {plen} cache {frac} {mode}: TPOT {np.mean(s.token_ms()):.3f} ms, "
                  f"H2D {cnt['h2d_bytes'] / steps / 1e6:.1f} MB/token")
    s.close()


if __name__ == "__main__":
    main()
