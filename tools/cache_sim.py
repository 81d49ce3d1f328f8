"""Offline cache-policy simulation on dumped decisions (tools only):
per layer C slots, each token-layer requests its k executed experts; a miss
copies one expert; eviction never removes an expert of the same request."""
import sys
from collections import OrderedDict, defaultdict

import numpy as np


def simulate(ids, C, policy, warm=8, count=32):
    T, L, K = ids.shape
    misses = 0
    for l in range(L):
        cache = OrderedDict()  # expert -> last use
        freq = defaultdict(float)
        for t in range(min(T, warm + count)):
            req = [int(e) for e in ids[t, l]]
            for e in req:
                freq[e] = freq[e] * 0.98 + 1.0 if policy == "lfu-decay" else freq[e] + 1
            for e in req:
                if e in cache:
                    cache.move_to_end(e)
                    continue
                if t >= warm:
                    misses += 1
                if len(cache) >= C:
                    cands = [x for x in cache if x not in req]
                    if policy == "lru":
                        victim = cands[0]
                    elif policy.startswith("lfu"):
                        victim = min(cands, key=lambda x: (freq[x], list(cache).index(x)))
                    elif policy == "belady":
                        def nxt(x):
                            for u in range(t + 1, T):
                                if x in ids[u, l]:
                                    return u
                            return 10**9
                        victim = max(cands, key=nxt)
                    del cache[victim]
                cache[e] = t
    return misses / count


d = np.load(sys.argv[1])
for mode in ("prefetch", "on_demand"):
    ids = d[mode + "_exec"]
    print(mode, {p: round(simulate(ids, 32, p), 2) for p in ("lru", "lfu", "lfu-decay", "belady")},
          "misses per token (C=32)")
