"""Per-kernel launch times (CUDA events, L back-to-back launches) on a
depth-truncated Q30-shaped model held resident in HBM.  Tools only."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_19289_b200 import ModelConfig, Session  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfg = ModelConfig(layers=L, experts=128, top_k=8, hidden=2048, expert_hidden=768, vocab=256,
                  head_dim=128, seed=1)
s = Session(cfg, cache_fraction=1.0, max_positions=256)
s.init_weights_seeded()
s.load_default_vectors(np.zeros((L, 128, 2048), np.float32))
s.set_predictor("router-pf")
s.preload_all()
s.reset(64, False)
s.prefill(list(range(32)))
for _ in range(2):
    p = s.profile_kernels(reps=5)
print({k: round(v, 2) for k, v in p.items()})
gu = 8 * 2 * 768 * 2048 * 2
print(f"ffn_gate_up {gu / p['ffn_gate_up'] / 1e3:.0f} GB/s; ffn_down {gu / 2 / p['ffn_down'] / 1e3:.0f} GB/s; ffn (as launched) {1.5 * gu / p['ffn'] / 1e3:.0f} GB/s; path {s.path_info()}")
s.close()
