"""Decode TPOT after long prompts (tools only; bench.py reports the same
measurement as `long_context`): Q30 shape, 25 % cache, prompt through the
batched prefill, then teacher-forced decode steps in both offload modes and
both decode arithmetic modes.

    python tools/long_context.py [steps] [prompt_len ...]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2603_19289_b200 import ModelConfig, Session  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    plens = [int(x) for x in sys.argv[2:]] or [1024, 4096, 16384]
    c = dict(bench.CONFIGS["q30"])
    cap = max(plens) + steps + 32
    s = Session(ModelConfig(**c), cache_fraction=1.0, max_positions=cap)
    s.init_weights_seeded()
    s.preload_all()
    d, _ = s.calibrate(256, 2, 256)
    s.load_default_vectors(d)
    s.set_predictor("router-pf")
    s.set_cache_fraction(0.25)
    forced = bench.token_stream(steps + 4, c["vocab"], 4)
    out = []
    for plen in plens:
        prompt = bench.token_stream(plen, c["vocab"], 5)
        row = {"prompt_len": plen}
        for dm in ("fast", "exact"):
            s.set_decode_mode(dm)
            for mode in ("prefetch", "on_demand"):
                s.reset(plen + steps + 4, False)
                t0 = time.perf_counter()
                s.prefill_batched(prompt)
                row["prefill_ms"] = (time.perf_counter() - t0) * 1e3
                s.decode_stream(mode, forced[:4])
                s.clear_stats()
                s.decode_stream(mode, forced[4:])
                ms = s.token_ms()
                row[f"{dm}_{mode}_tpot_ms"] = float(np.mean(ms))
                row[f"{dm}_{mode}_tpot_sd"] = float(np.std(ms))
        print(json.dumps(row), flush=True)
        out.append(row)
    s.close()


if __name__ == "__main__":
    main()
