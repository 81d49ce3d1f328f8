"""Cache policy study (tools only): which slot-replacement policy minimises the
expert copies of the headline stream workload in each offload mode?

    python tools/cache_policy_study.py capture [steps]   # GPU: records id_true / id_exec
    python tools/cache_policy_study.py simulate          # CPU: replays them through policies

Capture: Q30 shape, resident experts (routing does not depend on the cache),
calibrated router-pf table, 32-token prompt, `steps` teacher-forced stream
tokens in prefetch mode; saves the true and executed ids of every decode row
to gpurun_out/policy_trace.npz.  Simulate: per layer a cache of C = 32 slots;
each decode token requests its executed set (misses = copies), with

  lru        recency of use (the engine's policy)
  lru+true   as lru, plus the true router's ids of the token touched after it
             (the logging router runs every layer anyway; speculation.cpp:370)
  lfu        uses while resident
"""
import os
import sys
from collections import OrderedDict

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "gpurun_out", "policy_trace.npz")


def capture(steps):
    import bench
    from paper_2603_19289_b200 import ModelConfig, Session
    c = dict(bench.CONFIGS["q30"])
    P = 32
    s = Session(ModelConfig(**c), cache_fraction=1.0, max_positions=P + steps + 16)
    s.init_weights_seeded()
    s.preload_all()
    s.calibrate(2000, 2, 256)
    s.set_predictor("router-pf")
    s.set_decode_mode("fast")
    prompt = bench.token_stream(P, c["vocab"], 3)
    forced = bench.token_stream(steps, c["vocab"], 4)
    out = {}
    for mode in ("prefetch", "on_demand"):
        s.reset(P + steps, False)
        s.prefill(prompt)
        s.decode_stream(mode, forced)
        out[f"{mode}_true"] = s.trace("id_true", P + steps)[P:]
        out[f"{mode}_exec"] = s.trace("id_exec", P + steps)[P:]
    s.close()
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    np.savez(OUT, **out)
    print("saved", OUT, {k: v.shape for k, v in out.items()})


def simulate(C=32, warm=5):
    d = np.load(OUT)
    for mode in ("prefetch", "on_demand"):
        ex, tr = d[f"{mode}_exec"], d[f"{mode}_true"]
        T, L, K = ex.shape
        for pol in ("lru", "lru+true", "lfu"):
            caches = [OrderedDict() for _ in range(L)]
            miss = 0
            for t in range(T):
                for l in range(L):
                    cache = caches[l]
                    req = [int(e) for e in ex[t, l]]
                    for e in req:
                        if e in cache:
                            if pol == "lfu":
                                cache[e] += 1
                            else:
                                cache.move_to_end(e)
                        else:
                            if t >= warm:
                                miss += 1
                            if len(cache) >= C:
                                if pol == "lfu":
                                    victim = min((k for k in cache if k not in req), key=lambda k: cache[k])
                                else:
                                    victim = next(k for k in cache if k not in req)
                                del cache[victim]
                            cache[e] = 1
                if pol == "lru+true":
                    for l in range(L):
                        for e in tr[t, l]:
                            if int(e) in caches[l]:
                                caches[l].move_to_end(int(e))
            print(f"{mode:9s} {pol:9s} misses/token {miss / (T - warm):6.2f}")


if __name__ == "__main__":
    if sys.argv[1] == "capture":
        capture(int(sys.argv[2]) if len(sys.argv) > 2 else 200)
    else:
        simulate()
