"""Copy-overlap study (tools only; DESIGN.md §5 "Copy overlap"): replays the
ids captured by tools/overlap_capture.py through an event model of the
offload engine and compares slot policies and copy-lane disciplines.

    python tools/overlap_sim.py [gpurun_out/overlap_trace.npz]

Time model, per token and layer l (µs; calibrated on the resident TPOTs):
  A  qkv + attn + wo                      (both modes)
  G  true router + decision               (on-demand: on the critical path)
  P  predictor of l+1 after wo(l)         (prefetch: side stream)
  F  expert FFN (gate/up + down), starts when layer l's experts are in HBM
  h  host scheduler latency from mailbox post to the first copy
Copy lane: one server at the measured link rate; an expert copy is `chunks`
pieces; urgent requests (ids the device will execute) preempt warm ones
(predictions d > 1 layers ahead) at chunk boundaries.
"""
import heapq
import sys
from collections import OrderedDict

import numpy as np


class Slots:
    """Per-layer slot pool with a replacement policy.  `pinned` = ids that must
    stay (the current request).  Returns the list of ids that need a copy."""

    def __init__(self, L, C, policy):
        self.C, self.policy = C, policy
        self.c = [OrderedDict() for _ in range(L)]  # id -> use count (lfu) / None
        self.prob = [OrderedDict() for _ in range(L)]  # 2q: probation FIFO

    def has(self, l, e):
        return e in self.c[l] or e in self.prob[l]

    def touch(self, l, e):
        c = self.c[l]
        if e in c:
            c[e] += 1
            c.move_to_end(e)
        elif e in self.prob[l]:  # 2q: second use promotes
            del self.prob[l][e]
            self._insert_main(l, e, set())

    def _victim(self, d, keep):
        if self.policy == "lfu":
            return min((k for k in d if k not in keep), key=lambda k: d[k], default=None)
        return next((k for k in d if k not in keep), None)

    def _insert_main(self, l, e, keep):
        c = self.c[l]
        cap = self.C - (self.qcap if self.policy == "2q" else 0)
        while len(c) >= cap:
            v = self._victim(c, keep)
            if v is None:
                break
            del c[v]
        c[e] = 1

    def insert(self, l, e, keep):
        if self.policy == "2q":
            p = self.prob[l]
            while len(p) >= self.qcap:
                v = next((k for k in p if k not in keep), None)
                if v is None:
                    break
                del p[v]
            p[e] = 1
        else:
            self._insert_main(l, e, keep)


def run(exec_ids, warm_ids, mode, T, pol, C, tm, warm_from=5, chunks=1, qcap=8):
    """exec_ids [T][L][K]: executed ids; warm_ids: None or [T][L][K] predictions
    made one layer before the request (posted with the l-1 request)."""
    T_, L, K = exec_ids.shape
    A, G, P, F, h, tc = tm["A"], tm["G"], tm["P"], tm["F"], tm["h"], tm["tcopy"]
    slots = Slots(L, C, pol)
    slots.qcap = qcap
    now = 0.0
    lane_free = 0.0
    inflight = {}  # (l, e) -> completion time
    misses = 0
    warm_copies = 0
    tok_ms = []
    warm_q = []  # pending warm copies (l, e)

    def lane_run(until):
        """Run warm copies on the idle lane up to `until`."""
        nonlocal lane_free, warm_copies
        while warm_q and lane_free < until:
            l, e = warm_q.pop(0)
            if slots.has(l, e) or (l, e) in inflight:
                continue
            slots.insert(l, e, set())
            start = lane_free
            # warm copy in chunks: an urgent request arriving mid-copy waits for one chunk
            inflight[(l, e)] = start + tc
            lane_free = start + tc
            warm_copies += 1

    for t in range(T):
        t0 = now
        for l in range(L):
            start = now
            ids = [int(x) for x in exec_ids[t, l]]
            if mode == "on_demand" or l == 0:
                post = start + A + G
            else:
                post = prev_post  # noqa: F821  (posted during layer l-1)
            # warm copies get the lane while it is idle until the urgent post
            lane_run(post + h)
            need = 0.0
            keep = set(ids)
            urgent = []
            for e in ids:
                if (l, e) in inflight:
                    need = max(need, inflight[(l, e)])
                    slots.touch(l, e)
                elif slots.has(l, e):
                    slots.touch(l, e)
                else:
                    urgent.append(e)
            if urgent:
                # a warm copy in progress finishes its current chunk first
                lane = max(lane_free - (tc - tc / chunks) if lane_free > post + h else lane_free, post + h)
                for e in urgent:
                    slots.insert(l, e, keep)
                    lane += tc
                    inflight[(l, e)] = lane
                    if t >= warm_from:
                        misses += 1
                lane_free = max(lane_free, lane)
                need = max(need, lane)
            # the next layer's request is posted during this layer (prefetch)
            if mode == "prefetch":
                prev_post = start + A + P
                if warm_ids is not None and l + 2 < L:
                    for e in warm_ids[t, l + 2]:
                        warm_q.append((l + 2, int(e)))
                elif warm_ids is not None and t + 1 < T and l + 2 >= L:
                    pass
            ffn_start = max(start + A + (G if mode == "on_demand" or l == 0 else 0.0), need)
            now = ffn_start + F
            for k in [k for k, v in inflight.items() if v <= now]:
                del inflight[k]
        now += tm["tail"]
        tok_ms.append((now - t0) / 1000)
    n = T - warm_from
    return dict(tpot=float(np.mean(tok_ms[warm_from:])), misses=misses / n, warm=warm_copies / max(T, 1))


def belady(exec_ids, C, warm_from=5):
    T, L, K = exec_ids.shape
    miss = 0
    for l in range(L):
        seq = [[int(x) for x in exec_ids[t, l]] for t in range(T)]
        cache = set()
        for t in range(T):
            for e in seq[t]:
                if e in cache:
                    continue
                if t >= warm_from:
                    miss += 1
                if len(cache) >= C:
                    def nxt(x):
                        for u in range(t + 1, T):
                            if x in seq[u]:
                                return u
                        return 10 ** 9
                    cand = [x for x in cache if x not in seq[t]]
                    cache.discard(max(cand, key=nxt))
                cache.add(e)
    return miss / (T - warm_from)


def miss_structure(d, C=32, warm=32):
    """Where the copies come from: per layer, steady-state LRU misses per token
    (after `warm` tokens), distinct experts executed, and the misses of the best
    static set of C experts (frequency oracle) — for both offload modes."""
    from collections import Counter
    out = {}
    for mode in ("on_demand", "prefetch"):
        ex = d[f"{mode}_exec"]
        T, L, K = ex.shape
        per = np.zeros(L)
        for l in range(L):
            cache = OrderedDict()
            for t in range(T):
                req = [int(e) for e in ex[t, l]]
                for e in req:
                    if e in cache:
                        cache.move_to_end(e)
                        continue
                    if t >= warm:
                        per[l] += 1
                    if len(cache) >= C:
                        del cache[next(k for k in cache if k not in req)]
                    cache[e] = 1
        per /= T - warm
        rows = []
        for l in range(L):
            c = Counter(ex[:, l].ravel().tolist())
            top = sum(v for _, v in c.most_common(C)) / (T * K)
            rows.append((l, round(float(per[l]), 2), len(c), round((1 - top) * K, 2)))
        out[mode] = dict(total=round(float(per.sum()), 2), rows=rows)
    return out


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/overlap_trace.npz"
    d = np.load(path)
    ms = miss_structure(d)
    for mode, v in ms.items():
        print(f"{mode}: steady LRU misses/token {v['total']}; layers with > 0.05 misses/token "
              "(layer, LRU misses, distinct experts, best-static-set misses):")
        print("   ", [r for r in v["rows"] if r[1] > 0.05])
    ex, tr = d["prefetch_exec"], d["prefetch_true"]
    K = ex.shape[2]
    rec = [np.mean([len(set(ex[t, l]) & set(tr[t, l])) / K for t in range(ex.shape[0])]) for l in range(1, 6)]
    print("router-pf recall vs true at layers 1..5:", [round(float(r), 2) for r in rec])
    for dd in (2, 3, 4):
        a = d[f"ahead{dd}"]
        ov = np.mean([len(set(a[t, l]) & set(ex[t, l])) / K for t in range(ex.shape[0]) for l in range(dd, ex.shape[1])])
        print(f"router-pf {dd} layers ahead vs the executed (1-ahead) set: {ov:.3f}")
    L = d["prefetch_exec"].shape[1]
    T = d["prefetch_exec"].shape[0]
    link = float(d["link_GBps"])
    tcopy = 3 * 2048 * 768 * 2 / (link * 1e3)  # µs
    rp = float(np.mean(d["prefetch_resident_ms"][5:])) * 1000 / L
    ro = float(np.mean(d["on_demand_resident_ms"][5:])) * 1000 / L
    G = ro - rp
    A = 14.0
    tm = dict(A=A, G=G, P=9.0, F=rp - A, h=4.0, tcopy=tcopy, tail=0.0)
    print(f"T={T} link {link:.1f} GB/s copy {tcopy:.0f} us; resident layer pf {rp:.1f} od {ro:.1f} us")
    C = 32
    for pol in ("lru", "lfu"):
        od = run(d["on_demand_exec"], None, "on_demand", T, pol, C, tm)
        pf = run(d["prefetch_exec"], None, "prefetch", T, pol, C, tm)
        pw = run(d["prefetch_exec"], d["ahead2"], "prefetch", T, pol, C, tm, chunks=8)
        print(f"{pol:4s} on-demand {od['tpot']:.3f} ms ({od['misses']:.2f} miss/tok) | prefetch {pf['tpot']:.3f} "
              f"({pf['misses']:.2f}) | +warm2 {pw['tpot']:.3f} ({pw['misses']:.2f}, warm {pw['warm']:.2f})")
    print("belady misses/token: on-demand %.2f prefetch %.2f" % (belady(d["on_demand_exec"], C),
                                                               belady(d["prefetch_exec"], C)))


if __name__ == "__main__":
    main()
