import sys, numpy as np
sys.path.insert(0, ".")
import paper_2603_19289_b200.engine as E
E.load_library("tools/phase/libsmoe_b200.so")
from paper_2603_19289_b200 import ModelConfig, Session
cfg = ModelConfig(layers=2, experts=128, top_k=8, hidden=2048, expert_hidden=768, vocab=256, head_dim=128, seed=1)
s = Session(cfg, cache_fraction=1.0, max_positions=64)
s.init_weights_seeded(); s.preload_all()
s.reset(16); s.prefill([1, 2, 3]); s.decode("on_demand", 2, use_graph=False)
