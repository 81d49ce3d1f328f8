"""ctypes binding of libsmoe_b200.so (include/smoe.h).

This is the Python face of the C ABI, used by tests/ and bench.py.  It mirrors
the reference's decode-path API (proj/include/specmoe): ``ModelConfig``,
``ExecutorOptions`` / ``OffloadMode``, ``make_predictor`` kinds and
``run_offloaded_decode``.  There is no CPU fallback: if the CUDA library is
missing or no GPU is present, constructing a ``Session`` raises.
"""
from __future__ import annotations

import atexit
import ctypes as C
import os
import weakref
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsmoe_b200.so")

PRED = {"none": -1, "baseline-s": 0, "router-pf": 1, "est-pf": 2, "hybrid": 3, "oracle": 4}
MODE = {"on_demand": 0, "prefetch": 1}
GATING = {"softmax-topk-renorm": 0, "topk-softmax": 1}

# Symbols declared by include/smoe.h (checked by tests/test_capi.py).
EXPORTS = [
    "smoe_last_error", "smoe_session_create", "smoe_session_destroy", "smoe_init_weights_seeded",
    "smoe_load_tensor", "smoe_load_default_vectors", "smoe_load_estimator", "smoe_set_predictor",
    "smoe_set_cache_fraction", "smoe_reset", "smoe_prefill", "smoe_decode",
    "smoe_run_offloaded_decode", "smoe_step", "smoe_calibrate", "smoe_steps_done",
    "smoe_read_tokens", "smoe_read_trace", "smoe_token_ms", "smoe_counters", "smoe_copy_events",
    "smoe_cache_slots", "smoe_debug_state", "smoe_clear_stats", "smoe_profile_kernels",
    "smoe_measure_link", "smoe_kernels_per_step", "smoe_preload_all", "smoe_decode_stream",
    "smoe_ep_buffers", "smoe_ep_ipc_handles", "smoe_ep_connect", "smoe_ep_connect_ipc",
    "smoe_timeline", "smoe_simulate", "smoe_breakdown", "smoe_recall_at_k",
    "smoe_write_trace_bundle", "smoe_prefill_batched", "smoe_estimator_param_count", "smoe_simulate_cache", "smoe_predict_ahead", "smoe_batch_generate", "smoe_exp", "smoe_build_distill_dataset",
    "smoe_estimator_init", "smoe_train_estimator", "smoe_run_offloaded_decode_ex", "smoe_path_info", "smoe_decide", "smoe_layer_hit_rates",
    "smoe_select_hybrid_map", "smoe_set_prefill_mode", "smoe_set_decode_mode", "smoe_xp_pack", "smoe_xp_unpack",
]


class _Config(C.Structure):
    _fields_ = [("layers", C.c_int32), ("experts", C.c_int32), ("top_k", C.c_int32),
                ("hidden", C.c_int32), ("expert_hidden", C.c_int32), ("vocab", C.c_int32),
                ("head_dim", C.c_int32), ("eps", C.c_float), ("seed", C.c_uint64),
                ("gating", C.c_int32)]


class _Options(C.Structure):
    _fields_ = [("device", C.c_int32), ("cache_fraction", C.c_float),
                ("max_positions", C.c_int32), ("copy_latency_us", C.c_int32),
                ("deadlock_s", C.c_double), ("ep_rank", C.c_int32), ("ep_world", C.c_int32)]


class _EstConfig(C.Structure):
    _fields_ = [("d", C.c_int32), ("m", C.c_int32), ("n", C.c_int32), ("experts", C.c_int32),
                ("layers", C.c_int32), ("eps", C.c_float)]


class _TrainHyper(C.Structure):
    _fields_ = [("lr", C.c_double), ("batch_tokens", C.c_int32), ("max_steps", C.c_int64),
                ("eval_every", C.c_int64), ("val_fraction", C.c_double), ("seed", C.c_uint64),
                ("k", C.c_int32), ("early_stop_hit_rate", C.c_double)]


class _CurvePoint(C.Structure):
    _fields_ = [("tokens_seen", C.c_int64), ("val_kl", C.c_double), ("val_hit_rate", C.c_double)]


class Event(C.Structure):
    """MeasuredEvent (executor.hpp:31-37): lane 0 compute / 1 copy; kind 0 attn /
    1 gate / 2 expert / 3 copy."""
    _fields_ = [("lane", C.c_int32), ("kind", C.c_int32), ("layer", C.c_int32),
                ("token", C.c_int32), ("start_ms", C.c_double), ("end_ms", C.c_double)]


class CopyEvent(C.Structure):
    _fields_ = [("seq", C.c_int32), ("layer", C.c_int32), ("step", C.c_int32),
                ("hits", C.c_int32), ("misses", C.c_int32), ("bytes", C.c_int64),
                ("start_ms", C.c_double), ("end_ms", C.c_double)]


@dataclass
class ModelConfig:
    """ModelConfig (model.hpp:28-47)."""
    layers: int
    experts: int
    top_k: int
    hidden: int
    expert_hidden: int
    vocab: int
    head_dim: int
    eps: float = 1e-5
    seed: int = 0
    gating: str = "softmax-topk-renorm"

    def _c(self):
        return _Config(self.layers, self.experts, self.top_k, self.hidden, self.expert_hidden,
                       self.vocab, self.head_dim, self.eps, self.seed, GATING[self.gating])

    def expert_bytes_bf16(self) -> int:
        return 3 * self.hidden * self.expert_hidden * 2


_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Loads the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build() first")
        lib = C.CDLL(path)
        lib.smoe_last_error.restype = C.c_char_p
        for name in EXPORTS:
            getattr(lib, name)  # raises AttributeError if not exported
        _lib = lib
    return _lib


class SmoeError(RuntimeError):
    pass


def simulate(t_attn, t_gate, t_expert, t_copy, mode: str, cold_start_copy: float = -1.0):
    """simulate_on_demand / simulate_prefetch + breakdown + analytic_improvement
    (schedule.cpp:92-217), host C++ — no GPU needed."""
    lib = load_library()
    arr = [np.ascontiguousarray(a, np.float64) for a in (t_attn, t_gate, t_expert, t_copy)]
    tpot = C.c_double()
    an = C.c_double()
    fr = np.zeros(3, np.float64)
    _check(lib.smoe_simulate(len(arr[0]), *[_p(a) for a in arr], C.c_double(cold_start_copy),
                             MODE[mode], C.byref(tpot), _p(fr), C.byref(an)))
    return tpot.value, fr, an.value


class _CacheSim(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("tokens", "layers", "k", "capacity", "policy", "lookahead",
                                         "warm_tokens")]


def simulate_cache(exec_ids, t_attn, t_gate, t_expert, t_copy_expert, capacity, policy="lru", lookahead=1,
                   pred_ids=None, pred2_ids=None, warm_tokens=0):
    """Trace-driven two-lane schedule with a per-layer slot cache.
    Returns {tpot, stall_copies, prefetch_copies, useful_prefetch} per measured token."""
    lib = load_library()
    ex = np.ascontiguousarray(exec_ids, np.int32)
    T, L, K = ex.shape
    pr = None if pred_ids is None else np.ascontiguousarray(pred_ids, np.int32)
    p2 = None if pred2_ids is None else np.ascontiguousarray(pred2_ids, np.int32)
    ts = [np.ascontiguousarray(np.broadcast_to(np.asarray(x, np.float64), (L,))) for x in (t_attn, t_gate, t_expert)]
    c = _CacheSim(T, L, K, capacity, {"lru": 0, "lfu": 1}[policy], lookahead, warm_tokens)
    out = np.zeros(4, np.float64)
    _check(lib.smoe_simulate_cache(C.byref(c), _p(ex), _p(pr), _p(p2), *[_p(x) for x in ts],
                                   C.c_double(t_copy_expert), _p(out)))
    return dict(zip(("tpot", "stall_copies", "prefetch_copies", "useful_prefetch"), out.tolist()))


def breakdown(events) -> tuple:
    """per_token_reports + breakdown (executor.cpp:361-382, schedule.cpp:205-217):
    mean {compute, copy, idle} fractions and mean TPOT over decode steps."""
    lib = load_library()
    n = len(events)
    arr = (Event * max(n, 1))(*events)
    fr = np.zeros(3, np.float64)
    tp = C.c_double()
    _check(lib.smoe_breakdown(arr, n, _p(fr), C.byref(tp)))
    return fr, tp.value


def layer_hit_rates(exec_ids, true_ids) -> np.ndarray:
    """Per-layer online hit rates [L-1] of a recorded decode (id_exec vs id_true,
    [steps][L][k]); entry l-1 belongs to the predictor dispatched at l-1."""
    lib = load_library()
    e = np.ascontiguousarray(exec_ids, np.int32)
    t = np.ascontiguousarray(true_ids, np.int32)
    steps, L, k = e.shape
    out = np.zeros(L - 1, np.float64)
    _check(lib.smoe_layer_hit_rates(_p(e), _p(t), steps, L, k, _p(out)))
    return out


def xp_pack(raw) -> bytes | None:
    """Exponent-packed (xp11) form of a bf16 block given as uint16 [n]; None when
    the block does not pack (the store then keeps it raw)."""
    lib = load_library()
    raw = np.ascontiguousarray(raw, np.uint16)
    out = np.zeros(raw.size * 2 + 64, np.uint8)
    nb = C.c_int64()
    _check(lib.smoe_xp_pack(_p(raw), C.c_int64(raw.size), _p(out), C.c_int64(out.size), C.byref(nb)))
    return out[: nb.value].tobytes() if nb.value else None


def xp_unpack(packed: bytes, n: int) -> np.ndarray:
    """Inverse of xp_pack -> uint16 [n]."""
    lib = load_library()
    buf = np.frombuffer(packed, np.uint8).copy()
    out = np.zeros(n, np.uint16)
    _check(lib.smoe_xp_unpack(_p(buf), _p(out), C.c_int64(n)))
    return out


def select_hybrid_map(rates: dict, threshold: float = 0.0) -> list:
    """Hybrid map (layers-1 predictor names) from per-layer hit rates {kind: [L-1]};
    the first kind is the default (threshold > 0: kept unless below it)."""
    lib = load_library()
    kinds = list(rates)
    r = np.ascontiguousarray(np.stack([np.asarray(rates[k], np.float64) for k in kinds]))
    codes = np.array([PRED[k] for k in kinds], np.int32)
    out = np.zeros(r.shape[1], np.int32)
    _check(lib.smoe_select_hybrid_map(_p(r), _p(codes), len(kinds), r.shape[1] + 1, C.c_double(threshold),
                                      _p(out)))
    inv = {v: k for k, v in PRED.items()}
    return [inv[int(c)] for c in out]


def hybrid_map_json(names) -> str:
    """The map in load_hybrid_map's format (speculation.cpp:145-165): {"layer": "kind"}."""
    import json
    return json.dumps({str(l): n for l, n in enumerate(names)})


def recall_at_k(pred, truth):
    """recall_at_k (metrics.cpp:9-20) and rank_alignment (metrics.cpp:22-28)."""
    lib = load_library()
    p = np.ascontiguousarray(pred, np.int32)
    t = np.ascontiguousarray(truth, np.int32)
    r = C.c_double()
    m = np.zeros(len(p), np.int32)
    _check(lib.smoe_recall_at_k(_p(p), _p(t), len(p), C.byref(r), _p(m)))
    return r.value, m.astype(bool)


def device_exp(x) -> np.ndarray:
    """exp on the GPU through the device restatement of glibc's exp(double)."""
    lib = load_library()
    x = np.ascontiguousarray(x, np.float64)
    y = np.zeros_like(x)
    _check(lib.smoe_exp(_p(x), _p(y), C.c_int64(x.size)))
    return y


def device_decide(logits, k: int, gating: str = "softmax-topk-renorm"):
    """make_decision of every row of `logits` [rows][E] on the GPU -> (ids, gates)."""
    lib = load_library()
    lg = np.ascontiguousarray(logits, np.float32)
    rows, E = lg.shape
    ids = np.zeros((rows, k), np.int32)
    gates = np.zeros((rows, k), np.float32)
    _check(lib.smoe_decide(_p(lg), rows, E, k, GATING[gating], _p(ids), _p(gates)))
    return ids, gates


def estimator_init(d, m, n, E, L, eps=1e-5, seed=0) -> np.ndarray:
    """init_estimator_params<float> (estimator.cpp:54-75): the flat parameter block."""
    lib = load_library()
    c = _EstConfig(d, m, n, E, L, eps)
    cnt = C.c_int64()
    _check(lib.smoe_estimator_param_count(C.byref(c), C.byref(cnt)))
    out = np.zeros(cnt.value, np.float32)
    _check(lib.smoe_estimator_init(C.byref(c), C.c_uint64(seed), _p(out), cnt))
    return out


def train_estimator(inputs, targets, d, m, n, E, L, eps=1e-5, seed=0, lr=1e-3, batch=32, max_steps=0,
                    eval_every=50, val_fraction=0.1, hseed=0, k=1, early_stop=0.0):
    """train_estimator (estimator.cpp:374-450) on the GPU.  inputs [tokens][L-1][d],
    targets [tokens][L-1][E].  Returns (flat params, curve [n][3] = tokens_seen, val_kl,
    val_hit_rate, device ms of the training steps)."""
    lib = load_library()
    inputs = np.ascontiguousarray(inputs, np.float32)
    targets = np.ascontiguousarray(targets, np.float32)
    tokens = inputs.size // ((L - 1) * d)
    c = _EstConfig(d, m, n, E, L, eps)
    cnt = C.c_int64()
    _check(lib.smoe_estimator_param_count(C.byref(c), C.byref(cnt)))
    params = np.zeros(cnt.value, np.float32)
    cap = int(max_steps // max(eval_every, 1)) + 3
    curve = (_CurvePoint * cap)()
    nc = C.c_int32()
    ms = C.c_double()
    h = _TrainHyper(lr, batch, max_steps, eval_every, val_fraction, hseed, k, early_stop)
    _check(lib.smoe_train_estimator(C.byref(c), C.c_uint64(seed), _p(inputs), _p(targets), C.c_int64(tokens),
                                    L - 1, C.byref(h), _p(params), cnt, curve, cap, C.byref(nc), C.byref(ms)))
    cv = np.array([(p.tokens_seen, p.val_kl, p.val_hit_rate) for p in curve[:nc.value]], np.float64)
    return params, cv.reshape(-1, 3), ms.value


def _check(rc):
    if rc != 0:
        msg = _lib.smoe_last_error().decode()
        raise (ValueError if rc == 1 else SmoeError)(msg)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


_LIVE: "weakref.WeakSet[Session]" = weakref.WeakSet()


@atexit.register
def _close_live_sessions():
    """Destroy sessions still open at interpreter exit while the CUDA runtime
    is alive (module teardown order would otherwise decide)."""
    for s in list(_LIVE):
        try:
            s.close()
        except Exception:
            pass


class Session:
    """One model on one GPU: pinned expert store + HBM slot cache + decode state."""

    def __init__(self, cfg: ModelConfig, device: int = 0, cache_fraction: float = 1.0,
                 max_positions: int = 4096, copy_latency_us: int = 0, deadlock_s: float = 10.0,
                 ep_rank: int = 0, ep_world: int = 1):
        lib = load_library()
        self.cfg = cfg
        self._h = C.c_void_p()
        opt = _Options(device, cache_fraction, max_positions, copy_latency_us, deadlock_s,
                       ep_rank, ep_world)
        c = cfg._c()
        _check(lib.smoe_session_create(C.byref(c), C.byref(opt), C.byref(self._h)))
        self.lib = lib
        _LIVE.add(self)

    def close(self):
        if self._h:
            _check(self.lib.smoe_session_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- weights / artifacts -------------------------------------------------
    def init_weights_seeded(self):
        _check(self.lib.smoe_init_weights_seeded(self._h))

    def load_tensor(self, name: str, data: np.ndarray):
        d = np.ascontiguousarray(data, np.float32).ravel()
        _check(self.lib.smoe_load_tensor(self._h, name.encode(), _p(d), C.c_int64(d.size)))

    def load_default_vectors(self, d: np.ndarray):
        d = np.ascontiguousarray(d, np.float32).ravel()
        _check(self.lib.smoe_load_default_vectors(self._h, _p(d), C.c_int64(d.size)))

    def load_estimator(self, d, m, n, E, L, eps, flat):
        f = np.ascontiguousarray(flat, np.float32).ravel()
        c = _EstConfig(d, m, n, E, L, eps)
        _check(self.lib.smoe_load_estimator(self._h, C.byref(c), _p(f), C.c_int64(f.size)))

    def set_predictor(self, kind: str, hybrid=None):
        hm = None
        if hybrid is not None:
            hm = np.ascontiguousarray([PRED[k] if isinstance(k, str) else k for k in hybrid],
                                      np.int32)
        _check(self.lib.smoe_set_predictor(self._h, PRED[kind], _p(hm)))

    def set_cache_fraction(self, f: float):
        _check(self.lib.smoe_set_cache_fraction(self._h, C.c_float(f)))

    def cache_slots(self) -> int:
        n = C.c_int32()
        _check(self.lib.smoe_cache_slots(self._h, C.byref(n)))
        return n.value

    # -- decode ----------------------------------------------------------------
    def reset(self, max_steps: int = 0, trace_full: bool = False):
        _check(self.lib.smoe_reset(self._h, max_steps, int(trace_full)))

    def prefill(self, tokens):
        t = np.ascontiguousarray(tokens, np.int32)
        _check(self.lib.smoe_prefill(self._h, _p(t), len(t)))

    def prefill_batched(self, tokens):
        """All prompt tokens per layer at once (same results as prefill)."""
        t = np.ascontiguousarray(tokens, np.int32)
        _check(self.lib.smoe_prefill_batched(self._h, _p(t), len(t)))

    def decode(self, mode: str, n_steps: int, use_graph: bool = True):
        _check(self.lib.smoe_decode(self._h, MODE[mode], n_steps, int(use_graph)))

    def decode_stream(self, mode: str, tokens):
        t = np.ascontiguousarray(tokens, np.int32)
        _check(self.lib.smoe_decode_stream(self._h, MODE[mode], _p(t), len(t)))

    def run_offloaded_decode_ex(self, prompt, n_new: int, mode: str, cap: int = 1 << 18):
        """run_offloaded_decode returning the whole ExecutorResult (executor.hpp:39-44):
        (tokens, events, per_token_ms, max_resident_layers), events from the same run."""
        p = np.ascontiguousarray(prompt, np.int32)
        toks = np.zeros(n_new, np.int32)
        per = np.zeros(max(n_new - 1, 1), np.float64)
        arr = (Event * cap)()
        n, mr = C.c_int32(), C.c_int32()
        _check(self.lib.smoe_run_offloaded_decode_ex(self._h, _p(p), len(p), n_new, MODE[mode],
                                                     _p(toks), _p(per), arr, cap, C.byref(n),
                                                     C.byref(mr)))
        return toks, [arr[i] for i in range(min(n.value, cap))], per[: n_new - 1], mr.value

    def run_offloaded_decode(self, prompt, n_new: int, mode: str):
        """run_offloaded_decode (executor.cpp:326-359): tokens + device-timed per-token ms."""
        p = np.ascontiguousarray(prompt, np.int32)
        toks = np.zeros(n_new, np.int32)
        per = np.zeros(max(n_new - 1, 1), np.float64)
        _check(self.lib.smoe_run_offloaded_decode(self._h, _p(p), len(p), n_new, MODE[mode],
                                                  _p(toks), _p(per)))
        return toks, per[: n_new - 1]

    def step(self, mode: str, token: int, logits: np.ndarray | None = None) -> int:
        nxt = C.c_int32()
        _check(self.lib.smoe_step(self._h, MODE[mode], token, _p(logits), C.byref(nxt)))
        return nxt.value

    def calibrate(self, ntok: int, seed: int, seq_len: int):
        c = self.cfg
        d = np.zeros((c.layers, c.experts, c.hidden), np.float32)
        cnt = np.zeros((c.layers, c.experts), np.int64)
        _check(self.lib.smoe_calibrate(self._h, C.c_int64(ntok), C.c_uint64(seed), seq_len,
                                       _p(d), _p(cnt)))
        return d, cnt

    # -- results ---------------------------------------------------------------
    def steps_done(self) -> int:
        n = C.c_int32()
        _check(self.lib.smoe_steps_done(self._h, C.byref(n)))
        return n.value

    def tokens(self, n: int) -> np.ndarray:
        out = np.zeros(n, np.int32)
        _check(self.lib.smoe_read_tokens(self._h, _p(out), n))
        return out

    def trace(self, field: str, steps: int) -> np.ndarray:
        c = self.cfg
        L, K, H, E, V = c.layers, c.top_k, c.hidden, c.experts, c.vocab
        shapes = {"id_true": (L, K), "id_exec": (L, K), "id_pred": (L, K), "g_true": (L, K),
                  "g_exec": (L, K), "g_pred": (L, K), "s": (L, H), "r": (L, H), "m": (L, H),
                  "lg_true": (L, E), "lg_pred": (L, E), "y": (L, K, H), "logits": (V,),
                  "tok_in": ()}
        dt = np.int32 if field.startswith("id_") or field == "tok_in" else np.float32
        out = np.zeros((steps,) + shapes[field], dt)
        _check(self.lib.smoe_read_trace(self._h, field.encode(), _p(out), C.c_int64(out.size)))
        return out

    def build_distill_dataset(self, first: int, n: int, mode: str = "quasi"):
        """build_distill_dataset (speculation.cpp:476-484) on captured steps -> (inputs, targets)."""
        L, H, E = self.cfg.layers, self.cfg.hidden, self.cfg.experts
        inp = np.zeros((n, L - 1, H), np.float32)
        tgt = np.zeros((n, L - 1, E), np.float32)
        _check(self.lib.smoe_build_distill_dataset(self._h, first, n, {"quasi": 0, "s-next": 1}[mode],
                                                   _p(inp), _p(tgt)))
        return inp, tgt

    def batch_generate(self, prompts, n_new: int, mode: str = "prefetch", logits: bool = False,
                       timing: bool = False):
        """B sequences decoded together; prompts [B][P] -> tokens [B][n_new] (and logits
        [B][n_new][V] with logits=True; mean ms per decode step with timing=True)."""
        pr = np.ascontiguousarray(prompts, np.int32)
        B, P = pr.shape
        out = np.zeros((B, n_new), np.int32)
        lg = np.zeros((B, n_new, self.cfg.vocab), np.float32) if logits else None
        ms = C.c_double()
        _check(self.lib.smoe_batch_generate(self._h, B, _p(pr), P, n_new, MODE[mode], _p(out), _p(lg),
                                            C.byref(ms)))
        res = (out,) + ((lg,) if logits else ()) + ((ms.value,) if timing else ())
        return res if len(res) > 1 else out

    def predict_ahead(self, first: int, n: int, depth: int) -> np.ndarray:
        """Router-pf ids `depth` layers ahead from captured steps -> [n][L][K] (-1 where l < depth)."""
        out = np.zeros((n, self.cfg.layers, self.cfg.top_k), np.int32)
        _check(self.lib.smoe_predict_ahead(self._h, first, n, depth, _p(out)))
        return out

    def write_trace_bundle(self, path: str, first: int, n: int, seq_len: int = 0,
                           source: str = "", seed: int = 0):
        """Trace bundle in the reference's format (TraceWriter, trace.cpp:60-122)."""
        _check(self.lib.smoe_write_trace_bundle(self._h, path.encode(), first, n, seq_len,
                                                source.encode(), C.c_uint64(seed)))

    def token_ms(self) -> np.ndarray:
        out = np.zeros(4096, np.float64)
        n = C.c_int32()
        _check(self.lib.smoe_token_ms(self._h, _p(out), len(out), C.byref(n)))
        return out[: min(n.value, len(out))].copy()

    def counters(self):
        L = self.cfg.layers
        hits = np.zeros(L, np.int64)
        misses = np.zeros(L, np.int64)
        b = C.c_int64()
        ms = C.c_double()
        req = C.c_int32()
        _check(self.lib.smoe_counters(self._h, _p(hits), _p(misses), C.byref(b), C.byref(ms),
                                      C.byref(req)))
        return {"hits": hits, "misses": misses, "h2d_bytes": b.value, "copy_ms": ms.value,
                "requests": req.value}

    # -- expert parallelism -----------------------------------------------------
    def ep_buffers(self):
        x = C.c_void_p()
        c = C.c_void_p()
        _check(self.lib.smoe_ep_buffers(self._h, C.byref(x), C.byref(c)))
        return x.value, c.value

    def ep_ipc_handles(self) -> bytes:
        buf = (C.c_ubyte * 128)()
        _check(self.lib.smoe_ep_ipc_handles(self._h, buf))
        return bytes(buf)

    def ep_connect(self, xbufs, cnts):
        W = len(xbufs)
        xa = (C.c_void_p * W)(*xbufs)
        ca = (C.c_void_p * W)(*cnts)
        _check(self.lib.smoe_ep_connect(self._h, xa, ca))

    def ep_connect_ipc(self, handles):
        blob = b"".join(handles)
        buf = (C.c_ubyte * len(blob)).from_buffer_copy(blob)
        _check(self.lib.smoe_ep_connect_ipc(self._h, buf))

    def preload_all(self):
        _check(self.lib.smoe_preload_all(self._h))

    def clear_stats(self):
        _check(self.lib.smoe_clear_stats(self._h))

    def profile_kernels(self, reps: int = 3) -> dict:
        out = np.zeros(9, np.float64)
        _check(self.lib.smoe_profile_kernels(self._h, reps, _p(out)))
        names = ["qkv", "attn", "wo", "router", "ffn_gate_up", "ffn_down", "final", "ffn",
                 "ffn_gate_up_prefetch"]
        return dict(zip(names, out.tolist()))

    def set_decode_mode(self, mode: str):
        """'exact' (sequential chains, bit parity) or 'fast' (packed FFMA partial sums, tolerance)."""
        _check(self.lib.smoe_set_decode_mode(self._h, {"exact": 0, "fast": 1}[mode]))

    def set_prefill_mode(self, mode: str):
        """'exact' (sequential chains, bit parity) or 'tensor' (tcgen05 expert GEMMs, tolerance)."""
        _check(self.lib.smoe_set_prefill_mode(self._h, {"exact": 0, "tensor": 1}[mode]))

    def path_info(self) -> dict:
        out = np.zeros(8, np.int32)
        _check(self.lib.smoe_path_info(self._h, _p(out), 8))
        return {"ffn_fused": bool(out[0]), "attn_ctas": int(out[1]), "host_ordered": bool(out[2]),
                "device_hit_path": bool(out[3]), "store_numa_node": int(out[4]),
                "store_packed_blocks": int(out[5]), "store_wire_per_raw": float(out[6]) / 1000.0,
                "copy_lane_kernels": int(out[7])}

    def measure_link(self, n_copies: int = 64) -> float:
        g = C.c_double()
        _check(self.lib.smoe_measure_link(self._h, n_copies, C.byref(g)))
        return g.value

    def kernels_per_step(self, mode: str) -> int:
        n = C.c_int32()
        _check(self.lib.smoe_kernels_per_step(self._h, MODE[mode], C.byref(n)))
        return n.value

    def timeline(self, mode: str, n_steps: int, tokens=None, cap: int = 1 << 20):
        """Decode n_steps with a measured lane timeline (list of Event)."""
        t = None if tokens is None else np.ascontiguousarray(tokens, np.int32)
        arr = (Event * cap)()
        n = C.c_int32()
        _check(self.lib.smoe_timeline(self._h, MODE[mode], _p(t), n_steps, arr, cap, C.byref(n)))
        return [arr[i] for i in range(min(n.value, cap))]

    def copy_events(self, cap: int = 65536):
        arr = (CopyEvent * cap)()
        n = C.c_int32()
        _check(self.lib.smoe_copy_events(self._h, arr, cap, C.byref(n)))
        return [arr[i] for i in range(min(n.value, cap))]
