"""Teacher-forced, layer-by-layer parity checker.  TEST
INFRASTRUCTURE ONLY: used by the -m gpu tests to check a recorded GPU decode
against the CPU oracle (oracle/_ref/liboracle.so) one layer at a time.

For every recorded position t and layer l the checker takes the GPU's own
inputs to that layer and re-evaluates the reference's per-layer functions on
them (bf16-rounded weights, the values the GPU holds):

* attention (model.cpp:376-380): r_l from x_l = emb[token] (l = 0) or
  r_{l-1} + m_{l-1}, with the K/V history built from the recorded x_l of
  positions 0..t (``orc_attn_layer``);
* s_l = rms_norm(r_l, moe_gain_l) (numerics.cpp:72-84);
* the true router and make_decision (model.cpp:258-281);
* Algorithm 1's executed decision: the true one at layer 0, on demand and in
  the prompt; the one predicted at l-1 otherwise (speculation.cpp:366-371);
* the router-pf predictor for l+1: q_l = rms_norm(r_l + layer_default(exec_l),
  gain_{l+1}), gate_{l+1} . q_l, make_decision (speculation.cpp:104-121,
  206-228);
* every executed expert's raw output y_i = expert_ffn(W_e, s_l) and the
  mixture m_l = sum_i g_i y_i in decision order (model.cpp:283-304);
* the final logits (rms_norm + unembed) and the greedy argmax (model.cpp:384-396).

Only one layer's experts are generated at a time (lazy oracle model), so a
48-layer Q30 trace is checked within a few GB of host memory.  Every field is
compared for bit equality; a routing decision that differs is classified by the
oracle's logit gap at the deciding boundary (a near-tie when the gap is below
``eps``) and reported, never hidden.

With ``rtol > 0`` (the tolerance decode mode, smoe_set_decode_mode(1)) every
float vector is compared by its norm-relative error ||gpu - ref|| / ||ref||
against rtol instead (the largest error per field is reported), the ids and
the greedy token must still be equal unless the oracle's gap at the deciding
boundary is below ``eps`` (reported as a near-tie).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
from dataclasses import dataclass, field

import numpy as np

FIELDS = ("attn_r", "s", "lg_true", "id_true", "g_true", "exec", "lg_pred", "id_pred", "g_pred",
          "y", "m", "logits", "token")


@dataclass
class Report:
    checked: dict = field(default_factory=lambda: {f: 0 for f in FIELDS})
    exact: dict = field(default_factory=lambda: {f: 0 for f in FIELDS})
    near_ties: list = field(default_factory=list)   # (field, t, l, gap)
    mismatches: list = field(default_factory=list)  # (field, t, l, detail)
    min_boundary_gap: float = float("inf")
    max_rel_err: dict = field(default_factory=dict)  # tolerance mode: field -> largest error
    rtol: float = 0.0

    def add(self, f, ok):
        self.checked[f] += 1
        self.exact[f] += int(ok)

    def vec(self, f, want, got, t, l):
        """Bit equality, or (rtol > 0) norm-relative error within rtol."""
        want = np.asarray(want, np.float32)
        got = np.asarray(got, np.float32)
        if np.array_equal(want, got):
            self.add(f, True)
            return
        if self.rtol > 0:
            err = float(np.linalg.norm(got.astype(np.float64) - want) /
                        max(np.linalg.norm(want.astype(np.float64)), 1e-30))
            self.max_rel_err[f] = max(self.max_rel_err.get(f, 0.0), err)
            self.add(f, False)
            if err > self.rtol:
                self.mismatches.append((f, t, l, err))
            return
        self.add(f, False)
        self.mismatches.append((f, t, l, float(np.abs(want - got).max())))

    def ok(self) -> bool:
        return not self.mismatches

    def summary(self) -> dict:
        out = {"checked": self.checked, "exact": self.exact,
               "near_ties": len(self.near_ties), "near_tie_list": self.near_ties[:20],
               "mismatches": len(self.mismatches), "mismatch_list": self.mismatches[:20],
               "min_boundary_gap": self.min_boundary_gap}
        if self.rtol > 0:
            out.update({"rtol": self.rtol, "max_rel_err": self.max_rel_err})
        return out


def boundary_gap(orc, logits, k, gating):
    """Gap the decision hinges on: between the k-th and (k+1)-th largest value the
    top-k is taken over (probabilities for softmax-topk-renorm, logits for
    topk-softmax), and the smallest gap inside the top k (their order fixes the
    gates' rank order)."""
    v = orc.softmax(logits) if gating == 0 else np.asarray(logits, np.float32)
    srt = np.sort(v.astype(np.float64))[::-1]
    gaps = np.abs(np.diff(srt[: k + 1])) if len(srt) > k else np.abs(np.diff(srt[:k]))
    return float(gaps.min()) if gaps.size else float("inf")


def check_traces(orc, om, cfg: dict, runs, table=None, eps_tie: float = 1e-6,
                 threads: int | None = None, rtol: float = 0.0) -> dict:
    """runs: [(name, trace, mode)], each trace over S recorded positions (prompt
    rows first): tok_in [S], s/r/m [S][L][H], lg_true/lg_pred [S][L][E],
    id_*/g_* [S][L][K], y [S][L][K][H], logits [S][V], tokens [S] (argmax of
    each row), P = prompt length.  mode 'on_demand' or 'prefetch' (router-pf
    with `table`, [L][E][H]).  Layers are the outer loop, so one layer's experts
    (the union over every run) are generated once and released after it.
    Returns {name: Report}."""
    L, E, K, H = cfg["layers"], cfg["experts"], cfg["top_k"], cfg["hidden"]
    gating = {"softmax-topk-renorm": 0, "topk-softmax": 1}[cfg.get("gating", "softmax-topk-renorm")]
    eps = np.float32(cfg.get("eps", 1e-5))
    emb = om.tensor("embedding").reshape(cfg["vocab"], H)
    ones = np.ones(H, np.float32)
    pool = cf.ThreadPoolExecutor(max_workers=threads or os.cpu_count() or 1)
    tb = orc.table(np.asarray(table, np.float32)) if table is not None else None
    reps = {name: Report(rtol=rtol) for name, _, _ in runs}
    xs = {name: np.stack([emb[int(t)] for t in tr["tok_in"]]).astype(np.float32)
          for name, tr, _ in runs}  # x_0 of every row
    for l in range(L):
        ex = {}
        for name, tr, mode in runs:
            rep, spec, P = reps[name], mode == "prefetch", tr["P"]
            S = tr["s"].shape[0]
            r_gpu, s_gpu = tr["r"][:, l], tr["s"][:, l]
            R = om.attn_layer(l, xs[name])  # the K/V history needs every position
            for t in range(S):
                rep.vec("attn_r", R[t], r_gpu[t], t, l)
                s_ref = orc.rms_norm(r_gpu[t], ones, eps)
                rep.vec("s", s_ref, s_gpu[t], t, l)
                lg = om.linear(f"layer{l}.gate", E, s_gpu[t])
                rep.vec("lg_true", lg, tr["lg_true"][t, l], t, l)
                ids, gates = orc.make_decision(lg, K, gating)
                gap = boundary_gap(orc, lg, K, gating)
                rep.min_boundary_gap = min(rep.min_boundary_gap, gap)
                _decision(rep, ids, gates, tr["id_true"][t, l], tr["g_true"][t, l], "true", t, l, gap, eps_tie)
                decode_row = spec and t >= P and l >= 1
                want_exec = tr["id_pred"][t, l] if decode_row else tr["id_true"][t, l]
                ok = np.array_equal(tr["id_exec"][t, l], want_exec)
                rep.add("exec", ok)
                if not ok:
                    rep.mismatches.append(("exec", t, l, str(tr["id_exec"][t, l])))
                if spec and t >= P and l < L - 1:  # router-pf prediction for l + 1
                    e_ids = np.ascontiguousarray(tr["id_exec"][t, l], np.int32)
                    e_g = np.ascontiguousarray(tr["g_exec"][t, l], np.float32)
                    d = np.zeros(H, np.float32)
                    orc.lib.orc_layer_default(tb.h, e_ids.ctypes.data, e_g.ctypes.data, K, l,
                                              d.ctypes.data)
                    q = np.zeros(H, np.float32)
                    orc.lib.orc_quasi_hidden(np.ascontiguousarray(r_gpu[t]).ctypes.data, d.ctypes.data,
                                             ones.ctypes.data, H, eps, q.ctypes.data)
                    lgp = om.linear(f"layer{l + 1}.gate", E, q)
                    rep.vec("lg_pred", lgp, tr["lg_pred"][t, l + 1], t, l + 1)
                    pids, pg = orc.make_decision(lgp, K, gating)
                    gap = boundary_gap(orc, lgp, K, gating)
                    rep.min_boundary_gap = min(rep.min_boundary_gap, gap)
                    _decision(rep, pids, pg, tr["id_pred"][t, l + 1], tr["g_pred"][t, l + 1], "pred", t, l + 1,
                              gap, eps_tie)
            ex[name] = tr["id_exec"][:, l]
        # this layer's experts: the union over every run, generated once
        need = sorted({int(e) for name in ex for row in ex[name] for e in row})
        om.ensure_experts(l, need)
        for name, tr, mode in runs:
            rep = reps[name]
            S = tr["s"].shape[0]
            s_gpu, m_gpu = tr["s"][:, l], tr["m"][:, l]
            jobs = {(t, i): pool.submit(om.expert_ffn, l, int(ex[name][t][i]), s_gpu[t])
                    for t in range(S) for i in range(K)}
            for t in range(S):
                ys = []
                for i in range(K):
                    y = jobs[(t, i)].result()
                    ys.append(y)
                    rep.vec("y", y, tr["y"][t, l, i], t, l)
                mm = np.zeros(H, np.float32)
                g_ex = tr["g_exec"][t, l]
                for i in range(K):  # moe_block mixture, f32 in decision order
                    mm = mm + np.float32(g_ex[i]) * ys[i]
                rep.vec("m", mm, m_gpu[t], t, l)
            xs[name] = (tr["r"][:, l] + tr["m"][:, l]).astype(np.float32)  # next layer's input
        om.release_experts(l, need)
    for name, tr, mode in runs:  # final norm + unembed + greedy argmax
        rep = reps[name]
        for t in range(tr["s"].shape[0]):
            xn = orc.rms_norm(xs[name][t], ones, eps)
            lo = om.linear("unembed", cfg["vocab"], xn)
            rep.vec("logits", lo, tr["logits"][t], t, L)
            ok = int(np.argmax(lo)) == int(tr["tokens"][t])
            rep.add("token", ok)
            if not ok:
                top2 = np.sort(lo.astype(np.float64))[-2:]
                gap = float(top2[1] - top2[0])
                if rtol > 0 and gap < eps_tie:
                    rep.near_ties.append(("token", t, L, gap))
                else:
                    rep.mismatches.append(("token", t, L, int(np.argmax(lo))))
    pool.shutdown()
    return reps


def _decision(rep, ids, gates, got_ids, got_g, kind, t, l, gap, eps_tie):
    """Routing ids exact (a differing id at a boundary gap below eps_tie is a
    reported near-tie); gates exact, or within rtol in tolerance mode."""
    ok = np.array_equal(ids, got_ids)
    rep.add(f"id_{kind}", ok)
    if not ok:
        (rep.near_ties if gap < eps_tie else rep.mismatches).append((f"id_{kind}", t, l, gap))
        rep.add(f"g_{kind}", False)  # gates of another expert set: not comparable
        return
    rep.vec(f"g_{kind}", gates, got_g, t, l)


def gpu_trace(s, S: int, P: int) -> dict:
    """The recorded trace of a Session (smoe_reset(..., trace_full=1)) as numpy arrays."""
    tr = {f: s.trace(f, S) for f in ("s", "r", "m", "lg_true", "id_true", "g_true", "id_exec",
                                     "g_exec", "id_pred", "g_pred", "lg_pred", "y", "logits",
                                     "tok_in")}
    tr["tokens"] = s.tokens(S)
    tr["P"] = P
    return tr
