"""Batched vs token-by-token prefill wall time (Q30 shape).  Tools only.
    python tools/prefill_bench.py [layers] [prompt_len] [cache_fraction] [batched,tensor,token]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_19289_b200 import ModelConfig, Session  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 48
P = int(sys.argv[2]) if len(sys.argv) > 2 else 512
frac = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
cfg = ModelConfig(layers=L, experts=128, top_k=8, hidden=2048, expert_hidden=768, vocab=256,
                  head_dim=128, seed=1)
s = Session(cfg, cache_fraction=1.0, max_positions=P + 64)
s.init_weights_seeded()
s.preload_all()
s.load_default_vectors(np.zeros((L, 128, 2048), np.float32))
s.set_cache_fraction(frac)
s.set_predictor("router-pf")
prompt = (np.arange(P) * 37 % 256).astype(np.int32)
res = {}
names = sys.argv[4].split(",") if len(sys.argv) > 4 else ["batched", "token"]
for name in names:  # batched (exact chains), tensor (tcgen05 expert GEMMs, tolerance), token
    s.set_prefill_mode("tensor" if name == "tensor" else "exact")
    for rep in range(2):
        s.reset(P + 4, False)
        t0 = time.perf_counter()
        (s.prefill if name == "token" else s.prefill_batched)(prompt)
        dt = time.perf_counter() - t0
    res[name] = dt
    tok = int(s.tokens(P)[P - 1])
    print(f"{name:8s} prefill of {P} tokens, {L} layers, cache {frac}: {dt * 1e3:9.1f} ms "
          f"({dt * 1e6 / P:8.1f} us/token), next token {tok}", flush=True)
for a in names[1:]:
    print(f"{a} / {names[0]}: {res[a] / res[names[0]]:.2f}x")
s.close()
