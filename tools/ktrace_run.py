"""Device-side kernel timeline of one decode step (graph launch), from the
instrumented build (make -C paper_2603_19289_b200/csrc ktrace): per layer and
kernel the first CTA entry, first CTA past its PDL wait and last CTA exit,
in µs from the step start.  Tools only.

    python tools/ktrace_run.py [layers] [cache_fraction] [greedy|stream] [--prompt=N]
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_19289_b200.engine as E  # noqa: E402

LIB = os.path.join(ROOT, "tools", "ktrace", "libsmoe_b200.so")
E.load_library(LIB)
from paper_2603_19289_b200 import ModelConfig, Session  # noqa: E402

KINDS = {14: "l2_pf", 0: "embed", 1: "qkv", 2: "attn", 3: "wo", 4: "router", 5: "est0", 6: "est1", 7: "est2",
         8: "est3", 9: "ffn_gu", 10: "ffn_down", 11: "ep_mix", 12: "final", 13: "predictor",
         15: "ffn_fused", 16: "down_reduce"}
L = int(sys.argv[1]) if len(sys.argv) > 1 else 8
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
wl = sys.argv[3] if len(sys.argv) > 3 else "greedy"
use_graph = "--no-graph" not in sys.argv
plen = next((int(a.split("=")[1]) for a in sys.argv if a.startswith("--prompt=")), 32)
lib = C.CDLL(LIB)
lib.smoe_ktrace_read.argtypes = [C.c_void_p]
cfg = ModelConfig(layers=L, experts=128, top_k=8, hidden=2048, expert_hidden=768, vocab=256,
                  head_dim=128, seed=1)
s = Session(cfg, cache_fraction=frac, max_positions=max(512, plen + 96))
s.init_weights_seeded()
if frac == 1.0:
    s.preload_all()
s.calibrate(64, 2, 256)
s.set_predictor("router-pf")
s.set_decode_mode(os.environ.get("SMOE_DECODE_MODE", "exact"))
rng = np.random.default_rng(4)
forced = rng.integers(0, 256, 64).astype(np.int32)
for mode in ("prefetch", "on_demand"):
    s.reset(plen + 96)
    s.prefill_batched(list(rng.integers(0, 256, plen)) if plen > 32 else list(range(32)))
    if wl == "stream":
        s.decode_stream(mode, forced[:8])
    else:
        s.decode(mode, 8)
    lib.smoe_ktrace_reset()
    if wl == "stream":
        s.decode_stream(mode, forced[8:9])
    else:
        s.decode(mode, 1, use_graph=use_graph)
    buf = np.zeros((17 * 128, 4), np.uint64)
    lib.smoe_ktrace_read(buf.ctypes.data)
    t0 = min(int(r[0]) for r in buf if r[0] != np.uint64(~np.uint64(0)) and r[2] > 0)
    print(f"== {mode} ({wl}, cache {frac}, L={L}) step {float(s.token_ms()[-1]):.3f} ms ==")
    print(f"{'layer':>5} {'kernel':>9} {'entry':>8} {'waited':>8} {'exit':>8} {'run':>7} {'lastCTA':>8}")
    rows = []
    for kind, name in KINDS.items():
        for layer in range(L if kind not in (0, 12) else 1):
            r = buf[kind * 128 + layer]
            if r[2] == 0:
                continue
            e, w, x, lc = ((int(v) - t0) / 1e3 if int(v) != 2**64 - 1 else float("nan") for v in r)
            rows.append((x, layer, name, e, w, lc))
    for x, layer, name, e, w, lc in sorted(rows, key=lambda t: (t[3], t[0])):
        print(f"{layer:>5} {name:>9} {e:8.2f} {w:8.2f} {x:8.2f} {x - w:7.2f} {lc:8.2f}")
s.close()
