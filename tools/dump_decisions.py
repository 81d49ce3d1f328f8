"""Dump the executed expert decisions of the bench's stream workload (Q30,
router-pf, prefetch and on-demand) for offline cache-policy simulation
(tools/cache_sim.py).  Tools only."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_19289_b200 import ModelConfig, Session  # noqa: E402

L = 48
cfg = ModelConfig(layers=L, experts=128, top_k=8, hidden=2048, expert_hidden=768, vocab=256,
                  head_dim=128, seed=1)
s = Session(cfg, cache_fraction=1.0, max_positions=512)
s.init_weights_seeded()
s.preload_all()
s.calibrate(2000, 2, 256)
s.set_predictor("router-pf")


def token_stream(n, vocab, seed):
    # bench.py's random_token_stream equivalent is imported to stay identical
    import bench
    return bench.token_stream(n, vocab, seed)


P, N = 32, 128
prompt = token_stream(P, 256, 3)
forced = token_stream(N, 256, 4)
out = {}
for mode in ("prefetch", "on_demand"):
    S = P + N
    s.reset(S, True)
    s.prefill(prompt)
    s.decode_stream(mode, forced)
    out[mode + "_exec"] = s.trace("id_exec", S)[P:]
    out[mode + "_true"] = s.trace("id_true", S)[P:]
    out[mode + "_pred"] = s.trace("id_pred", S)[P:]
np.savez_compressed(os.path.join("gpurun_out", "decisions_q30.npz"), **out)
print({k: v.shape for k, v in out.items()})
s.close()
