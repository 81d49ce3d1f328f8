"""ctypes bindings for the CPU checkers.  TEST INFRASTRUCTURE ONLY.

* ``Ref``    -> oracle/_ref/libspecmoe_ref.so: the unmodified reference library
              (compiled from /root/reference/proj/src by oracle/Makefile) behind
              oracle/ref_driver.cpp.
* ``Oracle`` -> oracle/_ref/liboracle.so: our C restatement (specmoe_oracle.c).

Both expose the same Python surface so tests can run one against the other.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libspecmoe_ref.so")
ORC_SO = os.path.join(HERE, "_ref", "liboracle.so")

KINDS = {"baseline-s": 0, "router-pf": 1, "est-pf": 2, "hybrid": 3, "oracle": 4}
GATING = {"softmax-topk-renorm": 0, "topk-softmax": 1}

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")


@dataclass
class Config:
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

    def args(self):
        return (self.layers, self.experts, self.top_k, self.hidden, self.expert_hidden,
                self.vocab, self.head_dim, C.c_float(self.eps), C.c_uint64(self.seed),
                GATING[self.gating])


@dataclass
class Trace:
    """Per-(step, layer) records; layout of ref_driver.cpp:ref_generate_trace."""
    tokens: np.ndarray
    s: np.ndarray
    r: np.ndarray
    m: np.ndarray
    logits: np.ndarray
    ids: np.ndarray
    gates: np.ndarray
    outputs: np.ndarray | None
    final_logits: np.ndarray
    pred_logits: np.ndarray | None = None
    pred_ids: np.ndarray | None = None
    pred_gates: np.ndarray | None = None
    extra: dict = field(default_factory=dict)


def _alloc_trace(cfg: Config, P: int, n_new: int, outputs: bool, with_pred: bool):
    S = P + n_new - 1
    L, H, E, K, V = cfg.layers, cfg.hidden, cfg.experts, cfg.top_k, cfg.vocab
    t = Trace(
        tokens=np.zeros(n_new, np.int32),
        s=np.zeros((S, L, H), np.float32), r=np.zeros((S, L, H), np.float32),
        m=np.zeros((S, L, H), np.float32), logits=np.zeros((S, L, E), np.float32),
        ids=np.zeros((S, L, K), np.int32), gates=np.zeros((S, L, K), np.float32),
        outputs=np.zeros((S, L, K, H), np.float32) if outputs else None,
        final_logits=np.zeros((S, V), np.float32))
    if with_pred:
        t.pred_logits = np.zeros((S, max(L - 1, 1), E), np.float32)
        t.pred_ids = np.full((S, max(L - 1, 1), K), -1, np.int32)
        t.pred_gates = np.zeros((S, max(L - 1, 1), K), np.float32)
    return t


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class _Common:
    lib: C.CDLL

    def _check(self, rc):
        if rc != 0:
            msg = self.lib_err()
            raise (ValueError if rc == 1 else RuntimeError)(msg)


class Ref(_Common):
    """The reference library itself (oracle/_ref/libspecmoe_ref.so)."""

    def __init__(self, path: str = REF_SO):
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_model_tensor.restype = C.c_int64
        L.ref_model_set_tensor.restype = C.c_int64
        L.ref_model_set_tensor.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]
        L.ref_model_tensor.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]
        L.ref_derive_seed.restype = C.c_uint64
        L.ref_derive_seed.argtypes = [C.c_uint64, C.c_char_p]
        L.ref_silu.restype = C.c_float
        L.ref_silu.argtypes = [C.c_float]
        L.ref_gaussian_stream.argtypes = [C.c_uint64, C.c_float, C.c_int64, C.c_void_p]
        L.ref_offloaded_decode.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                           C.c_int, C.c_int64, C.c_double, C.c_void_p,
                                           C.c_void_p, C.c_void_p]
        L.ref_generate.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_calibrate_default_vectors.argtypes = [C.c_void_p, C.c_int64, C.c_uint64, C.c_int,
                                                    C.c_void_p]
        L.ref_estimator_init.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float,
                                         C.c_uint64, C.c_void_p, C.c_void_p]
        L.ref_rms_norm.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_float, C.c_void_p]
        L.ref_simulate.argtypes = [C.c_int] + [C.c_void_p] * 4 + [C.c_double, C.c_int] + [C.c_void_p] * 3
        for fn in ("ref_free_model", "ref_free_table", "ref_free_estimator", "ref_free_predictor"):
            getattr(L, fn).argtypes = [C.c_void_p]

    def lib_err(self):
        return self.lib.ref_last_error().decode()

    # -- model ---------------------------------------------------------------
    def build_model(self, cfg: Config, round_bf16: bool = True):
        h = C.c_void_p()
        self._check(self.lib.ref_build_model(*cfg.args(), int(round_bf16), C.byref(h)))
        return RefModel(self, h, cfg)

    def alloc_model(self, cfg: Config):
        """Model with the reference's shapes and zero weights (fill with set_tensor)."""
        h = C.c_void_p()
        self._check(self.lib.ref_alloc_model(*cfg.args(), C.byref(h)))
        return RefModel(self, h, cfg)

    def derive_seed(self, seed: int, label: str) -> int:
        return self.lib.ref_derive_seed(seed, label.encode())

    def gaussian_stream(self, seed: int, stddev: float, n: int) -> np.ndarray:
        out = np.zeros(n, np.float32)
        self.lib.ref_gaussian_stream(seed, stddev, n, _ptr(out))
        return out

    # -- leaf numerics -------------------------------------------------------
    def softmax(self, v):
        v = np.ascontiguousarray(v, np.float32)
        out = np.zeros_like(v)
        self._check(self.lib.ref_softmax(_ptr(v), len(v), _ptr(out)))
        return out

    def top_k(self, v, k):
        v = np.ascontiguousarray(v, np.float32)
        idx = np.zeros(k, np.int32)
        self._check(self.lib.ref_top_k(_ptr(v), len(v), k, _ptr(idx)))
        return idx

    def rms_norm(self, v, g, eps):
        v = np.ascontiguousarray(v, np.float32)
        g = np.ascontiguousarray(g, np.float32)
        out = np.zeros_like(v)
        self._check(self.lib.ref_rms_norm(_ptr(v), _ptr(g), len(v), eps, _ptr(out)))
        return out

    def silu(self, x):
        return self.lib.ref_silu(x)

    def make_decision(self, logits, k, gating=0):
        logits = np.ascontiguousarray(logits, np.float32)
        ids = np.zeros(k, np.int32)
        gates = np.zeros(k, np.float32)
        self._check(self.lib.ref_make_decision(_ptr(logits), len(logits), k, gating, _ptr(ids),
                                               _ptr(gates)))
        return ids, gates

    def linear(self, w, x):
        w = np.ascontiguousarray(w, np.float32)
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros(w.shape[0], np.float32)
        self._check(self.lib.ref_linear(_ptr(w), w.shape[0], w.shape[1], _ptr(x), _ptr(out)))
        return out

    # -- artifacts -----------------------------------------------------------
    def table_from(self, d: np.ndarray, counts: np.ndarray | None = None):
        L, E, H = d.shape
        d = np.ascontiguousarray(d, np.float32)
        cnt = None if counts is None else np.ascontiguousarray(counts, np.int64)
        h = C.c_void_p()
        self._check(self.lib.ref_table_from(L, E, H, _ptr(d), _ptr(cnt), C.byref(h)))
        return RefHandle(self, h, "ref_free_table", shape=(L, E, H))

    def table_get(self, t):
        L, E, H = t.shape
        d = np.zeros((L, E, H), np.float32)
        c = np.zeros((L, E), np.int64)
        self._check(self.lib.ref_table_get(t.h, _ptr(d), _ptr(c)))
        return d, c

    def estimator_init(self, d, m, n, E, L, eps=1e-5, seed=0):
        h = C.c_void_p()
        cnt = C.c_int64()
        self._check(self.lib.ref_estimator_init(d, m, n, E, L, eps, seed, C.byref(h), C.byref(cnt)))
        return RefHandle(self, h, "ref_free_estimator", count=cnt.value, E=E, d=d)

    def estimator_flat(self, est):
        out = np.zeros(est.count, np.float32)
        self._check(self.lib.ref_estimator_get(est.h, _ptr(out)))
        return out

    def estimator_set(self, est, flat):
        flat = np.ascontiguousarray(flat, np.float32)
        self._check(self.lib.ref_estimator_set(est.h, _ptr(flat)))

    def estimator_logits(self, est, q, layer):
        q = np.ascontiguousarray(q, np.float32)
        out = np.zeros(est.E, np.float32)
        self._check(self.lib.ref_estimator_logits(est.h, _ptr(q), layer, _ptr(out)))
        return out

    def train_estimator(self, inputs, targets, d, m, n, E, L, eps=1e-5, seed=0, lr=1e-3, batch=32,
                        max_steps=0, eval_every=50, val_fraction=0.1, hseed=0, k=1, early_stop=0.0):
        """train_estimator (estimator.cpp:374-450) -> (flat params, curve [n][3])."""
        inputs = np.ascontiguousarray(inputs, np.float32)
        targets = np.ascontiguousarray(targets, np.float32)
        tokens = inputs.size // ((L - 1) * d)
        est = self.estimator_init(d, m, n, E, L, eps, seed)
        params = np.zeros(est.count, np.float32)
        cap = int(max_steps // max(eval_every, 1)) + 3
        curve = np.zeros((cap, 3), np.float64)
        nc = C.c_int()
        L_ = self.lib
        L_.ref_train_estimator.argtypes = [C.c_int] * 5 + [C.c_float, C.c_uint64, C.c_void_p, C.c_void_p,
                                           C.c_int64, C.c_double, C.c_int, C.c_int64, C.c_int64,
                                           C.c_double, C.c_uint64, C.c_int, C.c_double, C.c_void_p,
                                           C.c_void_p, C.c_int, C.c_void_p]
        self._check(L_.ref_train_estimator(d, m, n, E, L, eps, seed, _ptr(inputs), _ptr(targets), tokens, lr,
                                           batch, max_steps, eval_every, val_fraction, hseed, k, early_stop,
                                           _ptr(params), _ptr(curve), cap, C.byref(nc)))
        return params, curve[:nc.value].copy()

    def make_predictor(self, kind: str, L: int, table=None, est=None, hybrid=None):
        h = C.c_void_p()
        hm = None if hybrid is None else np.ascontiguousarray(
            [KINDS[k] if isinstance(k, str) else k for k in hybrid], np.int32)
        self._check(self.lib.ref_make_predictor(KINDS[kind], table.h if table else None,
                                                est.h if est else None, _ptr(hm), L, C.byref(h)))
        return RefHandle(self, h, "ref_free_predictor", kind=kind)

    def simulate(self, attn, gate, expert, copy, prefetch, cold=-1.0):
        arrs = [np.ascontiguousarray(a, np.float64) for a in (attn, gate, expert, copy)]
        tpot = C.c_double()
        an = C.c_double()
        fr = np.zeros(3, np.float64)
        self._check(self.lib.ref_simulate(len(arrs[0]), *[_ptr(a) for a in arrs], cold,
                                          int(prefetch), C.byref(tpot), _ptr(fr), C.byref(an)))
        return tpot.value, fr, an.value


class RefHandle:
    def __init__(self, owner, h, free_fn, **kw):
        self.owner, self.h, self._free = owner, h, free_fn
        self.__dict__.update(kw)

    def __del__(self):
        try:
            getattr(self.owner.lib, self._free)(self.h)
        except Exception:
            pass


class RefModel:
    def __init__(self, ref: Ref, h, cfg: Config):
        self.ref, self.h, self.cfg = ref, h, cfg

    def __del__(self):
        try:
            self.ref.lib.ref_free_model(self.h)
        except Exception:
            pass

    def tensor(self, name: str) -> np.ndarray:
        n = self.ref.lib.ref_model_tensor(self.h, name.encode(), None)
        if n == 0:
            raise KeyError(name)
        out = np.zeros(n, np.float32)
        self.ref.lib.ref_model_tensor(self.h, name.encode(), _ptr(out))
        return out

    def set_tensor(self, name: str, v: np.ndarray):
        v = np.ascontiguousarray(v, np.float32).ravel()
        if self.ref.lib.ref_model_set_tensor(self.h, name.encode(), _ptr(v)) != v.size:
            raise KeyError(name)

    def calibrate(self, ntok: int, seed: int, seq_len: int):
        h = C.c_void_p()
        self.ref._check(self.ref.lib.ref_calibrate_default_vectors(self.h, ntok, seed, seq_len,
                                                                   C.byref(h)))
        c = self.cfg
        return RefHandle(self.ref, h, "ref_free_table", shape=(c.layers, c.experts, c.hidden))

    def distill_dataset(self, prompt, table=None, mode="quasi"):
        """DistillDatasetBuilder (speculation.cpp:437-471) over forward_decode(prompt)."""
        c = self.cfg
        t = np.ascontiguousarray(prompt, np.int32)
        inp = np.zeros((len(t), c.layers - 1, c.hidden), np.float32)
        tgt = np.zeros((len(t), c.layers - 1, c.experts), np.float32)
        self.ref._check(self.ref.lib.ref_distill_dataset(self.h, _ptr(t), len(t), table.h if table else None,
                                                         0 if mode == "quasi" else 1, _ptr(inp), _ptr(tgt)))
        return inp, tgt

    def write_trace(self, tokens, seq_len: int, path: str, source: str = "", seed: int = 0):
        """The reference's TraceWriter over stream_decode_trace (true path)."""
        t = np.ascontiguousarray(tokens, np.int32)
        self.ref._check(self.ref.lib.ref_write_trace(self.h, _ptr(t), C.c_int64(len(t)), seq_len,
                                                     path.encode(), source.encode(),
                                                     C.c_uint64(seed)))

    def generate_trace(self, prompt, n_new, pred=None, outputs=False) -> Trace:
        prompt = np.ascontiguousarray(prompt, np.int32)
        t = _alloc_trace(self.cfg, len(prompt), n_new, outputs, pred is not None)
        self.ref._check(self.ref.lib.ref_generate_trace(
            self.h, _ptr(prompt), len(prompt), n_new, pred.h if pred else None, _ptr(t.tokens),
            _ptr(t.s), _ptr(t.r), _ptr(t.m), _ptr(t.logits), _ptr(t.ids), _ptr(t.gates),
            _ptr(t.outputs), _ptr(t.final_logits), _ptr(t.pred_logits), _ptr(t.pred_ids),
            _ptr(t.pred_gates)))
        return t

    def generate(self, prompt, n_new, pred=None):
        prompt = np.ascontiguousarray(prompt, np.int32)
        toks = np.zeros(n_new, np.int32)
        pf = C.c_double()
        dc = C.c_double()
        self.ref._check(self.ref.lib.ref_generate(self.h, _ptr(prompt), len(prompt), n_new,
                                                  pred.h if pred else None, _ptr(toks),
                                                  C.byref(pf), C.byref(dc)))
        return toks, pf.value, dc.value

    def offloaded_decode(self, prompt, n_new, pred=None, mode="on_demand", latency_us=0,
                         deadlock_factor=100.0):
        prompt = np.ascontiguousarray(prompt, np.int32)
        toks = np.zeros(n_new, np.int32)
        per = np.zeros(max(n_new - 1, 1), np.float64)
        mr = C.c_int()
        self.ref._check(self.ref.lib.ref_offloaded_decode(
            self.h, _ptr(prompt), len(prompt), n_new, pred.h if pred else None,
            0 if mode == "on_demand" else 1, latency_us, deadlock_factor, _ptr(toks), _ptr(per),
            C.byref(mr)))
        return toks, per[: n_new - 1], mr.value


class Oracle(_Common):
    """Our C restatement (oracle/_ref/liboracle.so)."""

    def __init__(self, path: str = ORC_SO, threads: int | None = None):
        self.lib = C.CDLL(path)
        L = self.lib
        L.orc_last_error.restype = C.c_char_p
        L.orc_derive_seed.restype = C.c_uint64
        L.orc_derive_seed.argtypes = [C.c_uint64, C.c_char_p]
        L.orc_fill_gaussian.argtypes = [C.c_uint64, C.c_double, C.c_void_p, C.c_uint64]
        L.orc_model_build.restype = C.c_void_p
        L.orc_model_build.argtypes = [C.c_int] * 7 + [C.c_float, C.c_uint64, C.c_int, C.c_int]
        L.orc_model_build_lazy.restype = C.c_void_p
        L.orc_model_build_lazy.argtypes = [C.c_int] * 7 + [C.c_float, C.c_uint64, C.c_int, C.c_int]
        L.orc_model_ensure_experts.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int]
        L.orc_model_release_expert.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.orc_model_expert_ffn.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.orc_attn_layer.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p]
        L.orc_linear.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.orc_model_free.argtypes = [C.c_void_p]
        L.orc_model_tensor.restype = C.c_void_p
        L.orc_model_tensor.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]
        L.orc_table_new.restype = C.c_void_p
        L.orc_table_new.argtypes = [C.c_int, C.c_int, C.c_int]
        L.orc_table_free.argtypes = [C.c_void_p]
        L.orc_table_data.restype = C.c_void_p
        L.orc_table_data.argtypes = [C.c_void_p]
        L.orc_table_counts.restype = C.c_void_p
        L.orc_table_counts.argtypes = [C.c_void_p]
        L.orc_est_new.restype = C.c_void_p
        L.orc_est_new.argtypes = [C.c_int] * 5 + [C.c_float]
        L.orc_est_free.argtypes = [C.c_void_p]
        L.orc_est_flat.restype = C.c_void_p
        L.orc_est_flat.argtypes = [C.c_void_p, C.c_void_p]
        L.orc_est_init.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_est_logits.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
        L.orc_pred_new.restype = C.c_void_p
        L.orc_pred_new.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_pred_free.argtypes = [C.c_void_p]
        L.orc_generate_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int] + [C.c_void_p] * 13
        L.orc_generate_trace_forced.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                                 C.c_void_p, C.c_void_p] + [C.c_void_p] * 12
        L.orc_calibrate.argtypes = [C.c_void_p, C.c_int64, C.c_uint64, C.c_int, C.c_void_p]
        L.orc_silu.restype = C.c_float
        L.orc_silu.argtypes = [C.c_float]
        L.orc_rms_norm.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_float, C.c_void_p]
        L.orc_round_bf16.restype = C.c_float
        L.orc_round_bf16.argtypes = [C.c_float]
        L.orc_recall_at_k.restype = C.c_double
        L.orc_recall_at_k.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
        L.orc_token_stream.argtypes = [C.c_int64, C.c_int, C.c_uint64, C.c_void_p]
        L.orc_expert_ffn.argtypes = [C.c_void_p] * 3 + [C.c_int, C.c_int] + [C.c_void_p] * 3
        L.orc_layer_default.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                        C.c_void_p]
        L.orc_quasi_hidden.argtypes = [C.c_void_p] * 3 + [C.c_int, C.c_float, C.c_void_p]
        if threads:
            L.orc_set_threads(threads)
        else:  # ORC_THREADS overrides; at most 32 (fills and expert FFNs split into <= 64 jobs)
            L.orc_set_threads(int(os.environ.get("ORC_THREADS", min(os.cpu_count() or 1, 32))))

    def lib_err(self):
        return self.lib.orc_last_error().decode()

    def derive_seed(self, seed, label):
        return self.lib.orc_derive_seed(seed, label.encode())

    def gaussian_stream(self, seed, stddev, n):
        out = np.zeros(n, np.float32)
        self.lib.orc_fill_gaussian(seed, float(np.float32(stddev)), _ptr(out), n)
        return out

    def token_stream(self, n, vocab, seed):
        out = np.zeros(n, np.int32)
        self.lib.orc_token_stream(n, vocab, seed, _ptr(out))
        return out

    def build_model(self, cfg: Config, round_bf16: bool = True, lazy: bool = False):
        """lazy: dense weights only; experts generated on first use (ensure_experts,
        moe_block, tensor()) and releasable — the streaming per-layer checker."""
        fn = self.lib.orc_model_build_lazy if lazy else self.lib.orc_model_build
        h = fn(*cfg.args(), int(round_bf16))
        return OracleModel(self, h, cfg)

    def softmax(self, v):
        v = np.ascontiguousarray(v, np.float32)
        out = np.zeros_like(v)
        self._check(self.lib.orc_softmax(_ptr(v), len(v), _ptr(out)))
        return out

    def top_k(self, v, k):
        v = np.ascontiguousarray(v, np.float32)
        idx = np.zeros(k, np.int32)
        self._check(self.lib.orc_top_k(_ptr(v), len(v), k, _ptr(idx), None))
        return idx

    def rms_norm(self, v, g, eps):
        v = np.ascontiguousarray(v, np.float32)
        g = np.ascontiguousarray(g, np.float32)
        out = np.zeros_like(v)
        self.lib.orc_rms_norm(_ptr(v), _ptr(g), len(v), eps, _ptr(out))
        return out

    def silu(self, x):
        return self.lib.orc_silu(x)

    def make_decision(self, logits, k, gating=0):
        logits = np.ascontiguousarray(logits, np.float32)
        ids = np.zeros(k, np.int32)
        gates = np.zeros(k, np.float32)
        self._check(self.lib.orc_make_decision(_ptr(logits), len(logits), k, gating, _ptr(ids),
                                               _ptr(gates)))
        return ids, gates

    def linear(self, w, x):
        w = np.ascontiguousarray(w, np.float32)
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros(w.shape[0], np.float32)
        self.lib.orc_linear(_ptr(w), w.shape[0], w.shape[1], _ptr(x), _ptr(out))
        return out

    def expert_ffn(self, wg, wu, wd, x):
        H = x.shape[0]
        Hm = wg.shape[0]
        y = np.zeros(H, np.float32)
        scratch = np.zeros(2 * Hm, np.float32)
        self.lib.orc_expert_ffn(*[_ptr(np.ascontiguousarray(a, np.float32)) for a in (wg, wu, wd)],
                                H, Hm, _ptr(np.ascontiguousarray(x, np.float32)), _ptr(y),
                                _ptr(scratch))
        return y

    def recall_at_k(self, pred, truth):
        p = np.ascontiguousarray(pred, np.int32)
        t = np.ascontiguousarray(truth, np.int32)
        return self.lib.orc_recall_at_k(_ptr(p), _ptr(t), len(p))

    def table(self, d: np.ndarray, counts=None):
        L, E, H = d.shape
        h = self.lib.orc_table_new(L, E, H)
        tb = OracleHandle(self, h, "orc_table_free", shape=(L, E, H))
        tb.d[...] = d
        if counts is not None:
            tb.counts[...] = counts
        return tb

    def estimator(self, d, m, n, E, L, eps=1e-5, seed=None, flat=None):
        h = self.lib.orc_est_new(d, m, n, E, L, eps)
        est = OracleHandle(self, h, "orc_est_free", E=E, d=d)
        if seed is not None:
            self.lib.orc_est_init(h, seed)
        if flat is not None:
            est.flat[...] = flat
        return est

    def estimator_logits(self, est, q, layer):
        q = np.ascontiguousarray(q, np.float32)
        out = np.zeros(est.E, np.float32)
        self._check(self.lib.orc_est_logits(est.h, _ptr(q), layer, _ptr(out)))
        return out

    def make_predictor(self, kind, model, table=None, est=None, hybrid=None):
        hm = None if hybrid is None else np.ascontiguousarray(
            [KINDS[k] if isinstance(k, str) else k for k in hybrid], np.int32)
        h = self.lib.orc_pred_new(KINDS[kind], table.h if table else None,
                                  est.h if est else None, _ptr(hm), model.h)
        p = OracleHandle(self, h, "orc_pred_free", kind=kind)
        p._keep = (table, est, hm)
        return p


class _Owned(np.ndarray):
    """A view of C-owned memory that keeps its owning handle alive (so
    `np.array(handle_returning_call().d)` cannot read freed memory)."""


def _owned(arr: np.ndarray, owner) -> np.ndarray:
    v = arr.view(_Owned)
    v._owner = owner
    return v


class OracleHandle:
    def __init__(self, owner, h, free_fn, **kw):
        self.owner, self.h, self._free = owner, h, free_fn
        self.__dict__.update(kw)

    @property
    def d(self):
        L, E, H = self.shape
        p = self.owner.lib.orc_table_data(self.h)
        return _owned(np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_float)), (L, E, H)), self)

    @property
    def counts(self):
        L, E, H = self.shape
        p = self.owner.lib.orc_table_counts(self.h)
        return _owned(np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_int64)), (L, E)), self)

    @property
    def flat(self):
        n = C.c_int64()
        p = self.owner.lib.orc_est_flat(self.h, C.byref(n))
        return _owned(np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_float)), (n.value,)), self)

    def __del__(self):
        try:
            getattr(self.owner.lib, self._free)(C.c_void_p(self.h))
        except Exception:
            pass


class OracleModel:
    def __init__(self, orc: Oracle, h, cfg: Config):
        self.orc, self.h, self.cfg = orc, h, cfg

    def __del__(self):
        try:
            self.orc.lib.orc_model_free(C.c_void_p(self.h))
        except Exception:
            pass

    def tensor(self, name: str) -> np.ndarray:
        """Zero-copy view of a named tensor (mutable: writes change the model)."""
        n = C.c_int64()
        p = self.orc.lib.orc_model_tensor(self.h, name.encode(), C.byref(n))
        if not p:
            raise KeyError(name)
        return _owned(np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_float)), (n.value,)), self)

    def ensure_experts(self, layer: int, ids):
        ids = np.ascontiguousarray(ids, np.int32)
        self.orc.lib.orc_model_ensure_experts(self.h, layer, _ptr(ids), len(ids))

    def release_experts(self, layer: int, ids):
        for e in ids:
            self.orc.lib.orc_model_release_expert(self.h, layer, int(e))

    def expert_ffn(self, layer: int, e: int, x) -> np.ndarray:
        """expert_ffn (model.cpp:283-288) of a generated expert; releases the GIL,
        so a thread pool runs several at once."""
        x = np.ascontiguousarray(x, np.float32)
        y = np.zeros(self.cfg.hidden, np.float32)
        self.orc._check(self.orc.lib.orc_model_expert_ffn(self.h, layer, int(e), _ptr(x), _ptr(y)))
        return y

    def attn_layer(self, layer: int, X) -> np.ndarray:
        """Teacher-forced attention of one layer: R_j = x_j + attention_step over
        positions 0..n-1 with the K/V history built from the given inputs."""
        X = np.ascontiguousarray(X, np.float32)
        R = np.zeros_like(X)
        self.orc._check(self.orc.lib.orc_attn_layer(self.h, layer, _ptr(X), X.shape[0], _ptr(R)))
        return R

    def linear(self, name: str, rows: int, x) -> np.ndarray:
        """linear (numerics.cpp:136-147) with a named weight [rows][len(x)]."""
        x = np.ascontiguousarray(x, np.float32)
        w = self.tensor(name)
        out = np.zeros(rows, np.float32)
        self.orc.lib.orc_linear(w.ctypes.data, rows, len(x), _ptr(x), _ptr(out))
        return out

    def calibrate(self, ntok, seed, seq_len):
        c = self.cfg
        tb = self.orc.table(np.zeros((c.layers, c.experts, c.hidden), np.float32))
        self.orc._check(self.orc.lib.orc_calibrate(self.h, ntok, seed, seq_len, tb.h))
        return tb

    def generate_trace(self, prompt, n_new, pred=None, outputs=False, forced=None) -> Trace:
        """generate(); `forced` (n_new-1 tokens) teacher-forces the decode inputs."""
        prompt = np.ascontiguousarray(prompt, np.int32)
        t = _alloc_trace(self.cfg, len(prompt), n_new, outputs, pred is not None)
        fz = None if forced is None else np.ascontiguousarray(forced, np.int32)
        if fz is not None and len(fz) < n_new - 1:
            raise ValueError("forced stream shorter than n_new - 1")
        self.orc._check(self.orc.lib.orc_generate_trace_forced(
            self.h, _ptr(prompt), len(prompt), n_new, pred.h if pred else None, _ptr(fz),
            _ptr(t.tokens),
            _ptr(t.s), _ptr(t.r), _ptr(t.m), _ptr(t.logits), _ptr(t.ids), _ptr(t.gates),
            _ptr(t.outputs), _ptr(t.final_logits), _ptr(t.pred_logits), _ptr(t.pred_ids),
            _ptr(t.pred_gates)))
        return t
