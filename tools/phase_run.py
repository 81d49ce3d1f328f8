"""Per-phase cycle counts printed by the instrumented build (make -C
paper_2603_19289_b200/csrc phase): python tools/phase_run.py [on_demand|prefetch]."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_19289_b200.engine as E  # noqa: E402

E.load_library(os.path.join(os.path.dirname(os.path.abspath(__file__)), "phase", "libsmoe_b200.so"))
from paper_2603_19289_b200 import ModelConfig, Session  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "on_demand"
cfg = ModelConfig(layers=4, experts=128, top_k=8, hidden=2048, expert_hidden=768, vocab=256,
                  head_dim=128, seed=1)
s = Session(cfg, cache_fraction=1.0, max_positions=64)
s.init_weights_seeded()
s.preload_all()
s.load_default_vectors(np.zeros((4, 128, 2048), np.float32))
s.set_predictor("router-pf")
s.reset(16)
s.prefill([1, 2, 3])
s.decode(mode, 2, use_graph=True)
