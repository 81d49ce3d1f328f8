"""est-pf diagnostic (tools only): GPU-distilled estimator, its online logits
against a numpy restatement of estimator_forward (estimator.cpp:94-161) on the
same quasi-hidden inputs, and the recall of both against the true logits.

    python tools/est_check.py [layers] [tokens]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def np_forward(flat, q, l, d, m, n, E, L, eps=1e-5):
    dm, mlp = d // m, d // m * n
    o = 0
    A = flat[o:o + dm * d].reshape(dm, d); o += dm * d
    pos = flat[o:o + L * dm].reshape(L, dm); o += L * dm
    B = flat[o:o + mlp * dm].reshape(mlp, dm); o += mlp * dm
    Cm = flat[o:o + dm * mlp].reshape(dm, mlp); o += dm * mlp
    g = flat[o:o + dm]; o += dm
    b = flat[o:o + dm]; o += dm
    W = flat[o:o + E * dm].reshape(E, dm)
    z = A @ q + pos[l]
    u = B @ z
    act = u / (1 + np.exp(-u))
    h = z + Cm @ act
    xh = (h - h.mean()) / np.sqrt(h.var() + eps)
    return W @ (g * xh + b)


def recall(a, b, k):
    return len(set(np.argsort(-a)[:k]) & set(np.argsort(-b)[:k])) / k


def main():
    import bench
    from paper_2603_19289_b200 import ModelConfig, Session, engine
    Lr = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    c = dict(bench.CONFIGS["q30"], layers=Lr)
    L, H, E, K = c["layers"], c["hidden"], c["experts"], c["top_k"]
    s = Session(ModelConfig(**c), cache_fraction=1.0, max_positions=T + 64)
    s.init_weights_seeded()
    s.preload_all()
    s.calibrate(2000, 2, 256)
    s.set_decode_mode("fast")
    s.set_predictor("router-pf")
    s.reset(T + 8, True)
    s.prefill(list(bench.token_stream(8, c["vocab"], 7)))
    s.decode_stream("on_demand", bench.token_stream(T, c["vocab"], 6))
    inp, tgt = s.build_distill_dataset(8, T, "quasi")
    flat, curve, ms = engine.train_estimator(inp, tgt, H, 8, 4, E, L, seed=1, lr=1e-3, batch=32,
                                             max_steps=400, eval_every=100, val_fraction=0.1, hseed=1, k=K)
    print("curve", np.round(curve, 4).tolist())
    ntr = int(T * 0.9)
    for name, rng in (("train", range(0, 20)), ("val", range(ntr, ntr + 20))):
        r = np.mean([recall(np_forward(flat, inp[t, l], l, H, 8, 4, E, L), tgt[t, l], K)
                     for t in rng for l in range(L - 1)])
        print(f"numpy forward recall on {name} samples: {r:.3f}")
    s.load_estimator(H, 8, 4, E, L, 1e-5, flat)
    s.set_predictor("est-pf")
    P, N = 32, 24
    s.reset(P + N, True)
    s.prefill(list(bench.token_stream(P, c["vocab"], 3)))
    s.decode_stream("prefetch", bench.token_stream(N, c["vocab"], 5))
    i2, t2 = s.build_distill_dataset(P, N, "quasi")
    lgp = s.trace("lg_pred", P + N)[P:]
    lgt = s.trace("lg_true", P + N)[P:]
    errs, r_np, r_on = [], [], []
    for t in range(N):
        for l in range(L - 1):
            f = np_forward(flat, i2[t, l], l, H, 8, 4, E, L)
            errs.append(np.abs(f - lgp[t, l + 1]).max() / (np.abs(f).max() + 1e-30))
            r_np.append(recall(f, lgt[t, l + 1], K))
            r_on.append(recall(lgp[t, l + 1], lgt[t, l + 1], K))
    print(f"online vs numpy logits: max rel err {max(errs):.3e}; recall numpy {np.mean(r_np):.3f} online {np.mean(r_on):.3f}")
    print("dataset target == trace lg_true:", float(np.abs(t2[:, :, :] - lgt[:, 1:, :]).max()))
    s.close()


if __name__ == "__main__":
    main()
