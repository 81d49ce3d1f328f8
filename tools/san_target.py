"""Small workload for compute-sanitizer (tools only): the tolerance-mode decode
(column-split gate/up, flash-decoding attention, decision_fast) in both offload
modes with the packed store (k_xp_unpack on the copy lane), the tcgen05
prefill, and a batched decode under offload.

    compute-sanitizer --tool memcheck python tools/san_target.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_19289_b200 import ModelConfig, Session  # noqa: E402

cfg = ModelConfig(layers=3, experts=16, top_k=4, hidden=64, expert_hidden=128, vocab=256, head_dim=32, seed=4)
s = Session(cfg, cache_fraction=1.0, max_positions=400)
s.init_weights_seeded()
s.preload_all()
d, _ = s.calibrate(32, 2, 32)
s.load_default_vectors(d)
s.set_predictor("router-pf")
s.set_cache_fraction(0.5)
s.set_decode_mode("fast")
for mode in ("on_demand", "prefetch"):
    s.reset(64, True)
    s.prefill([5, 77, 200, 13])
    s.decode(mode, 6)
    print(mode, s.tokens(10)[3:].tolist(), flush=True)
s.set_prefill_mode("tensor")
prompt = np.random.default_rng(1).integers(0, 256, 300).astype(np.int32)
s.reset(320, False)
s.prefill_batched(prompt)
s.decode("on_demand", 2)
print("tensor prefill ok", flush=True)
toks = s.batch_generate(np.random.default_rng(2).integers(0, 256, (3, 4)).astype(np.int32), 4, "prefetch")
print("batch ok", toks.tolist(), flush=True)
s.close()
