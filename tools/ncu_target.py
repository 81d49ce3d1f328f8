"""Short decode workload for ncu: Q30 layer shapes, depth-truncated (per-layer
kernels are identical to the full model's), cache 25%, router-pf."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2603_19289_b200 import ModelConfig, Session

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = ModelConfig(layers=L, experts=128, top_k=8, hidden=2048, expert_hidden=768, vocab=256,
                  head_dim=128, seed=1)
resident = "--resident" in sys.argv
s = Session(cfg, cache_fraction=1.0 if resident else 0.25, max_positions=512)
s.init_weights_seeded()
if resident:
    s.preload_all()  # no copy-lane waits: ncu serialises streams
s.calibrate(32, 2, 256)
s.set_predictor("router-pf")
import os
s.set_decode_mode(os.environ.get("SMOE_DECODE_MODE", "fast"))
prompt = (np.arange(8) * 37 % 256).astype(np.int32)
s.reset(64)
s.prefill(prompt)
ranged = "--profile-range" in sys.argv  # with `ncu --profile-from-start off`: decode only
if ranged:
    import torch
    torch.cuda.init()
    torch.cuda.profiler.start()
s.decode("prefetch", steps)
s.decode("on_demand", steps)
if ranged:
    torch.cuda.profiler.stop()
print("ok", s.token_ms())
