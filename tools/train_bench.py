"""Estimator distillation throughput, GPU vs the reference's CPU train_estimator.

    python tools/train_bench.py [d m n E L tokens batch steps]

Defaults: the Qwen3-30B-A3B shape (d=2048, m=2, n=4 -> latent 1024, mlp 4096;
E=128, L=48), 512 synthetic tokens, batch 32, 20 steps.  Prints the GPU device
time per optimizer step (evaluation excluded) and the reference's CPU time per
step extrapolated from a bounded 1-token step (its cost is linear in tokens).
Tool only: the reference arm runs oracle/_ref.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2603_19289_b200 import engine  # noqa: E402


def main():
    a = [int(x) for x in sys.argv[1:]]
    d, m, n, E, L, T, B, steps = a + [2048, 2, 4, 128, 48, 512, 32, 20][len(a):]
    rng = np.random.default_rng(0)
    inp = rng.standard_normal((T, L - 1, d)).astype(np.float32)
    tgt = (2 * rng.standard_normal((T, L - 1, E))).astype(np.float32)
    kw = dict(seed=1, lr=1e-3, batch=B, eval_every=steps, val_fraction=0.02, hseed=1, k=8)
    engine.train_estimator(inp, tgt, d, m, n, E, L, max_steps=2, **kw)  # warm-up
    _, curve, ms = engine.train_estimator(inp, tgt, d, m, n, E, L, max_steps=steps, **kw)
    dm, mlp = d // m, d // m * n
    macs = (B * (L - 1)) * (2 * (dm * d + 2 * mlp * dm + E * dm) + 2 * mlp * dm + dm * d + E * dm)
    print(f"gpu: {ms / steps:.3f} ms/step ({B} tokens x {L - 1} layers), "
          f"{macs / (ms / steps * 1e-3) / 1e12:.2f} T chain-MAC/s, curve {curve[-1].tolist()}")
    try:
        from oracle.bindings import Ref
        ref = Ref()
    except Exception as e:  # noqa: BLE001
        print("reference unavailable:", e)
        return
    small = dict(kw, batch=1, val_fraction=0.0)
    Ts = 3
    t0 = time.perf_counter()
    ref.train_estimator(inp[:Ts], tgt[:Ts], d, m, n, E, L, max_steps=0, **small)
    t1 = time.perf_counter()
    ref.train_estimator(inp[:Ts], tgt[:Ts], d, m, n, E, L, max_steps=1, **small)
    t2 = time.perf_counter()
    per_tok = (t2 - t1) - (t1 - t0)
    print(f"reference cpu (1 thread): {per_tok * 1e3:.1f} ms per token-step -> "
          f"{per_tok * B * 1e3:.0f} ms/step at batch {B}; speed-up {per_tok * B * 1e3 / (ms / steps):.0f}x")


if __name__ == "__main__":
    main()
