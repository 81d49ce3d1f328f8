"""Per-kernel launch times (CUDA events, L back-to-back launches) on a
depth-truncated Q30-shaped model held resident in HBM.  Tools only."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_19289_b200.engine as E  # noqa: E402

if os.environ.get("SMOE_LIB"):  # a variant build (tools only)
    E.load_library(os.environ["SMOE_LIB"])
from paper_2603_19289_b200 import ModelConfig, Session  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfg = ModelConfig(layers=L, experts=128, top_k=8, hidden=2048, expert_hidden=768, vocab=256,
                  head_dim=128, seed=1)
s = Session(cfg, cache_fraction=1.0, max_positions=int(os.environ.get("KB_CAP", "256")))
s.init_weights_seeded()
s.load_default_vectors(np.zeros((L, 128, 2048), np.float32))
s.set_predictor("router-pf")
s.preload_all()
if os.environ.get("SMOE_DECODE_MODE"):
    s.set_decode_mode(os.environ["SMOE_DECODE_MODE"])
s.reset(max(64, int(os.environ.get("KB_PROMPT", "32")) + 16), False)
s.prefill([t % 256 for t in range(int(os.environ.get("KB_PROMPT", "32")))])
s.decode("prefetch", 2)  # predicted decisions of every layer in place (prefetch-form timing)
for _ in range(2):
    p = s.profile_kernels(reps=5)
s.reset(max(64, int(os.environ.get("KB_PROMPT", "32")) + 16), False)
s.prefill(list(range(32)))
s.decode("prefetch", 4)
s.decode("prefetch", 16)
tp = float(np.mean(s.token_ms()))
s.decode("on_demand", 4)
s.decode("on_demand", 16)
print(f"resident greedy TPOT ({L} layers): prefetch {tp:.3f} ms, on_demand {float(np.mean(s.token_ms())):.3f} ms")
print({k: round(v, 2) for k, v in p.items()})
gu = 8 * 2 * 768 * 2048 * 2
print(f"ffn_gate_up {gu / p['ffn_gate_up'] / 1e3:.0f} GB/s; ffn_down {gu / 2 / p['ffn_down'] / 1e3:.0f} GB/s; ffn (as launched) {1.5 * gu / p['ffn'] / 1e3:.0f} GB/s; ffn_gate_up prefetch form {gu / (p.get('ffn_gate_up_prefetch') or 1e9) / 1e3:.0f} GB/s; path {s.path_info()}")
s.close()
