"""GPU parity tests: the CUDA path (through the C ABI) against the reference's
golden fixtures and the CPU oracle.  Bit-exact for ids, gates, hidden states
and logits (the kernels keep the reference's operation
order); the only tolerance anywhere is the documented f64-reduction-order
caveat, which these tests have never needed.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TINY = dict(layers=3, experts=6, top_k=2, hidden=16, expert_hidden=24, vocab=32, head_dim=8,
            seed=11)
BASE = dict(layers=4, experts=32, top_k=4, hidden=512, expert_hidden=1024, vocab=256,
            head_dim=64, seed=1)
TOY = dict(layers=8, experts=16, top_k=4, hidden=64, expert_hidden=128, vocab=256, head_dim=32,
           seed=4)
HYBRID_TINY = ["router-pf", "est-pf"]


def gold(name):
    return np.load(os.path.join(G, name))


@pytest.fixture(scope="module")
def lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2603_19289_b200 import load_library
    return load_library()


def session(cfg, **kw):
    from paper_2603_19289_b200 import ModelConfig, Session
    kw.setdefault("max_positions", 512)
    s = Session(ModelConfig(**cfg), **kw)
    s.init_weights_seeded()
    return s


def run_trace(s, prompt, n_new, mode):
    P = len(prompt)
    S = P + n_new - 1
    s.reset(S, True)
    s.prefill(prompt)
    s.decode(mode, n_new - 1)
    out = {f: s.trace(f, S) for f in ("s", "r", "m", "lg_true", "id_exec", "g_exec", "y", "logits",
                                     "id_pred", "g_pred", "lg_pred", "id_true")}
    out["tokens"] = s.tokens(S)[P - 1:]
    return out


def assert_trace_equal(got, want, with_pred, P):
    assert np.array_equal(got["tokens"], want["tokens"])
    for g, w in (("s", "s"), ("r", "r"), ("m", "m"), ("lg_true", "logits"), ("id_exec", "ids"),
                 ("g_exec", "gates"), ("y", "outputs"), ("logits", "final_logits")):
        assert np.array_equal(got[g], want[w]), g
    if with_pred:  # predictions made during decode steps (prefill never predicts)
        assert np.array_equal(got["id_pred"][P:, 1:], want["pred_ids"][P:])
        assert np.array_equal(got["g_pred"][P:, 1:], want["pred_gates"][P:])


# ------------------------------------------------ reference golden fixtures --

@pytest.mark.parametrize("kind", ["none", "baseline-s", "router-pf", "est-pf", "hybrid", "oracle"])
def test_tiny_matches_reference_goldens(lib, kind):
    c = gold("tiny_common.npz")
    g = gold(f"tiny_{kind}.npz")
    s = session(TINY, cache_fraction=0.5)
    s.load_default_vectors(c["dv"])
    s.load_estimator(TINY["hidden"], 2, 4, TINY["experts"], TINY["layers"], 1e-5, c["est_flat"])
    mode = "on_demand"
    if kind != "none":
        s.set_predictor(kind, HYBRID_TINY if kind == "hybrid" else None)
        mode = "prefetch"
    got = run_trace(s, c["prompt"], int(c["n_new"]), mode)
    want = {k: g[k] for k in g.files}
    assert_trace_equal(got, want, kind != "none", len(c["prompt"]))
    s.close()


def test_default_vectors_bit_exact(lib):
    c = gold("tiny_common.npz")
    s = session(TINY)
    d, cnt = s.calibrate(200, 2, 16)
    assert np.array_equal(d, c["dv"]) and np.array_equal(cnt, c["dv_counts"])
    s.close()


def test_baseline_config_64_tokens(lib):
    """BASELINE configs[0] (L4 H512 E32 k4): default vectors from 2000 calibration
    tokens, then 64 generated tokens with the true router and with router-pf;
    tokens, executed ids and online hit rates identical to the reference."""
    g = gold("baseline.npz")
    s = session(BASE, cache_fraction=1.0, max_positions=512)
    s.preload_all()
    d, cnt = s.calibrate(2000, 2, 256)
    assert np.array_equal(d, g["dv"]) and np.array_equal(cnt, g["dv_counts"])
    s.set_cache_fraction(0.25)
    s.set_predictor("router-pf")
    P = len(g["prompt"])
    for kind, mode in (("none", "on_demand"), ("router-pf", "prefetch")):
        S = P + 63
        s.reset(S, False)
        s.prefill(g["prompt"])
        s.decode(mode, 63)
        assert np.array_equal(s.tokens(S)[P - 1:], g[f"{kind}_tokens"])
        assert np.array_equal(s.trace("id_exec", S), g[f"{kind}_ids"])
        assert np.array_equal(s.trace("id_true", S), g[f"{kind}_true_ids"])
        if kind == "router-pf":
            got_recall = np.mean([len(set(a) & set(b)) / 4 for a, b in
                                  zip(s.trace("id_exec", S)[P:, 1:].reshape(-1, 4),
                                      s.trace("id_true", S)[P:, 1:].reshape(-1, 4))])
            want_recall = np.mean([len(set(a) & set(b)) / 4 for a, b in
                                   zip(g["router-pf_ids"][P:, 1:].reshape(-1, 4),
                                       g["router-pf_true_ids"][P:, 1:].reshape(-1, 4))])
            assert got_recall == want_recall
    s.close()


# ------------------------------------------------------------ vs the oracle --

@pytest.fixture(scope="module")
def toy_oracle():
    from oracle.bindings import Config, Oracle
    orc = Oracle()
    om = orc.build_model(Config(**TOY), round_bf16=True)
    table = om.calibrate(128, 2, 32)
    est = orc.estimator(TOY["hidden"], 2, 4, TOY["experts"], TOY["layers"], seed=5)
    return orc, om, table, est


@pytest.mark.parametrize("kind", ["none", "baseline-s", "router-pf", "est-pf", "hybrid", "oracle"])
@pytest.mark.parametrize("frac", [0.25, 1.0])
def test_toy_all_predictors_vs_oracle(lib, toy_oracle, kind, frac):
    orc, om, table, est = toy_oracle
    L = TOY["layers"]
    hyb = [["router-pf", "est-pf", "baseline-s"][l % 3] for l in range(L - 1)]
    pred = None if kind == "none" else orc.make_predictor(kind, om, table, est,
                                                         hyb if kind == "hybrid" else None)
    prompt = np.array([5, 77, 200, 13, 9], np.int32)
    want = om.generate_trace(prompt, 10, pred, outputs=True)
    s = session(TOY, cache_fraction=frac)
    s.load_default_vectors(np.array(table.d))
    s.load_estimator(TOY["hidden"], 2, 4, TOY["experts"], L, 1e-5, np.array(est.flat))
    mode = "on_demand"
    if kind != "none":
        s.set_predictor(kind, hyb if kind == "hybrid" else None)
        mode = "prefetch"
    got = run_trace(s, prompt, 10, mode)
    w = dict(tokens=want.tokens, s=want.s, r=want.r, m=want.m, logits=want.logits, ids=want.ids,
             gates=want.gates, outputs=want.outputs, final_logits=want.final_logits,
             pred_ids=want.pred_ids, pred_gates=want.pred_gates)
    assert_trace_equal(got, w, kind != "none", len(prompt))
    s.close()


@pytest.mark.parametrize("plen", [130, 200])
def test_long_context_attention_chunks(lib, toy_oracle, plen):
    """Contexts past the two prefetched 64-position chunks: keys and values
    stream through the cp.async rings (k_attn), the current row arrives in a
    chunk loaded after the PDL wait, and ring slots are reused."""
    orc, om, table, est = toy_oracle
    rng = np.random.default_rng(plen)
    prompt = rng.integers(0, TOY["vocab"], plen).astype(np.int32)
    want = om.generate_trace(prompt, 6, orc.make_predictor("router-pf", om, table), outputs=True)
    s = session(TOY, cache_fraction=0.5)
    s.load_default_vectors(np.array(table.d))
    s.set_predictor("router-pf")
    got = run_trace(s, prompt, 6, "prefetch")
    w = dict(tokens=want.tokens, s=want.s, r=want.r, m=want.m, logits=want.logits, ids=want.ids,
             gates=want.gates, outputs=want.outputs, final_logits=want.final_logits,
             pred_ids=want.pred_ids, pred_gates=want.pred_gates)
    assert_trace_equal(got, w, True, len(prompt))
    s.close()


def test_topk_softmax_gating(lib):
    from oracle.bindings import Config, Oracle
    cfg = dict(TOY, gating="topk-softmax", seed=9)
    orc = Oracle()
    om = orc.build_model(Config(**cfg), round_bf16=True)
    table = om.calibrate(64, 2, 32)
    want = om.generate_trace([1, 2, 3], 8, orc.make_predictor("router-pf", om, table), outputs=True)
    s = session(cfg, cache_fraction=0.5)
    s.load_default_vectors(np.array(table.d))
    s.set_predictor("router-pf")
    got = run_trace(s, [1, 2, 3], 8, "prefetch")
    assert np.array_equal(got["tokens"], want.tokens)
    assert np.array_equal(got["g_exec"], want.gates)
    assert np.array_equal(got["logits"], want.final_logits)
    s.close()


def test_oracle_predictor_equals_true_path(lib):
    """SPEC.md:298 oracle equivalence on the GPU (prefetch with Oracle == on-demand)."""
    s = session(TOY, cache_fraction=0.25)
    s.set_predictor("oracle")
    a = run_trace(s, [7, 8, 9], 12, "on_demand")
    b = run_trace(s, [7, 8, 9], 12, "prefetch")
    for f in ("tokens", "s", "m", "id_exec", "g_exec", "logits"):
        assert np.array_equal(a[f], b[f]), f
    s.close()


def test_cache_fraction_never_changes_results(lib):
    """The slot cache changes which copies happen, never which experts run."""
    out = []
    for frac in (0.25, 0.5, 1.0):
        s = session(TOY, cache_fraction=frac)
        s.calibrate(64, 2, 32)
        s.set_predictor("router-pf")
        out.append(run_trace(s, [3, 1, 4, 1, 5], 10, "prefetch"))
        s.close()
    for o in out[1:]:
        for f in ("tokens", "m", "logits", "id_exec"):
            assert np.array_equal(o[f], out[0][f]), f


def test_load_tensor_from_f32_reference_model(lib):
    """smoe_load_tensor: a reference Model's f32 tensors, rounded to bf16 on the
    way in, reproduce the rounded oracle exactly."""
    from oracle.bindings import Config, Oracle
    orc = Oracle()
    cfg = dict(TINY, seed=23)
    raw = orc.build_model(Config(**cfg), round_bf16=False)
    rnd = orc.build_model(Config(**cfg), round_bf16=True)
    from paper_2603_19289_b200 import ModelConfig, Session
    s = Session(ModelConfig(**cfg), cache_fraction=0.5, max_positions=64)
    names = ["embedding", "unembed", "final_norm_gain"]
    for l in range(cfg["layers"]):
        names += [f"layer{l}.{t}" for t in ("attn_norm_gain", "moe_norm_gain", "wq", "wk", "wv",
                                             "wo", "gate")]
        names += [f"layer{l}.expert{e}.{t}" for e in range(cfg["experts"])
                  for t in ("w_gate", "w_up", "w_down")]
    for n in names:
        s.load_tensor(n, raw.tensor(n))
    want = rnd.generate_trace([4, 5, 6], 6, outputs=True)
    got = run_trace(s, [4, 5, 6], 6, "on_demand")
    assert np.array_equal(got["tokens"], want.tokens)
    assert np.array_equal(got["logits"], want.final_logits)
    s.close()


def test_single_expert_and_prompt_of_one(lib):
    from oracle.bindings import Config, Oracle
    cfg = dict(layers=2, experts=1, top_k=1, hidden=16, expert_hidden=8, vocab=32, head_dim=8,
               seed=3)
    orc = Oracle()
    om = orc.build_model(Config(**cfg), round_bf16=True)
    want = om.generate_trace([9], 5, outputs=True)
    s = session(cfg, cache_fraction=1.0)
    got = run_trace(s, [9], 5, "on_demand")
    assert np.array_equal(got["tokens"], want.tokens)
    assert np.array_equal(got["logits"], want.final_logits)
    s.close()


def test_step_api_end_to_end(lib, toy_oracle):
    """smoe_step: host token in, host logits out, equals the oracle's logits."""
    orc, om, table, est = toy_oracle
    want = om.generate_trace([11, 12], 4)
    s = session(TOY, cache_fraction=0.5)
    s.reset(16)
    s.prefill([11, 12])
    logits = np.zeros(TOY["vocab"], np.float32)
    tok = int(s.tokens(2)[1])
    for i in range(3):
        nxt = s.step("on_demand", tok, logits)
        assert np.array_equal(logits, want.final_logits[2 + i])
        assert nxt == want.tokens[i + 1]
        tok = nxt
    s.close()


# ------------------------------------------------- copy lane / cache logic --

def test_copy_lane_invariants(lib):
    """Copies are serialised on one FIFO lane (copy_lane_serialized,
    schedule.cpp:224-234), every request is accounted hit or miss, bytes match
    the misses, and every prefetch request precedes its layer's compute."""
    s = session(TOY, cache_fraction=0.25)
    s.calibrate(32, 2, 32)
    s.set_predictor("router-pf")
    s.reset(32)
    s.prefill([1, 2, 3])
    s.clear_stats()
    s.decode("prefetch", 6)
    ev = s.copy_events()
    c = s.counters()
    K = TOY["top_k"]
    assert c["requests"] == len(ev) == 6 * TOY["layers"]
    assert sum(e.hits + e.misses for e in ev) == len(ev) * K
    assert int(c["hits"].sum()) == sum(e.hits for e in ev)
    per = 3 * TOY["hidden"] * TOY["expert_hidden"] * 2  # toy dims need no tile padding
    # the link carries the store's wire format: raw bf16 or exponent-packed
    # (xp11, ~0.70 of raw; per-block size varies by a few escapes)
    ratio = s.path_info()["store_wire_per_raw"]
    assert all(abs(e.bytes - e.misses * per * ratio) <= e.misses * per * 0.003 for e in ev)
    spans = sorted((e.start_ms, e.end_ms) for e in ev if e.misses > 0)
    for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
        assert b0 >= a1 - 1e-3
    s.close()


def test_errors_are_loud(lib):
    s = session(TOY)
    with pytest.raises(ValueError, match="prefetch mode needs a predictor"):
        s.run_offloaded_decode([1, 2], 3, "prefetch")
    with pytest.raises(ValueError, match="default-vector table"):
        s.set_predictor("router-pf")
    with pytest.raises(ValueError, match="token out of vocab"):
        s.prefill([1, 999])
    with pytest.raises(ValueError, match="needs cache_fraction 1.0"):
        s2 = session(TOY, cache_fraction=0.5)
        s2.preload_all()
    s.close()


def test_q30_layer_shapes_vs_oracle(lib):
    """Qwen3-30B-A3B layer shapes (H2048 E128 k8 Hm768, head_dim 128),
    depth-truncated to 2 layers (per-layer weights depend only on (seed, label)),
    cache 25 %: prefetch decode bit-exact against the oracle."""
    from oracle.bindings import Config, Oracle
    cfg = dict(layers=2, experts=128, top_k=8, hidden=2048, expert_hidden=768, vocab=256,
               head_dim=128, seed=1)
    orc = Oracle()
    om = orc.build_model(Config(**cfg), round_bf16=True)
    table = om.calibrate(8, 2, 256)
    want = om.generate_trace([3, 30, 300 % 256], 4, orc.make_predictor("router-pf", om, table),
                             outputs=False)
    s = session(cfg, cache_fraction=0.25)
    s.load_default_vectors(np.array(table.d))
    s.set_predictor("router-pf")
    got = run_trace(s, [3, 30, 300 % 256], 4, "prefetch")
    assert np.array_equal(got["tokens"], want.tokens)
    assert np.array_equal(got["id_exec"], want.ids)
    assert np.array_equal(got["m"], want.m)
    assert np.array_equal(got["logits"], want.final_logits)
    s.close()


def test_stream_decode_vs_oracle_teacher_forced(lib, toy_oracle):
    """smoe_decode_stream (teacher-forced inputs, the bench's headline workload)
    equals the oracle's speculative_forward over the same token stream."""
    orc, om, table, est = toy_oracle
    forced = np.array([(37 * i + 11) % TOY["vocab"] for i in range(11)], np.int32)
    prompt = [5, 6, 7]
    want = om.generate_trace(prompt, 12, orc.make_predictor("router-pf", om, table),
                             outputs=True, forced=forced)
    s = session(TOY, cache_fraction=0.25)
    s.load_default_vectors(np.array(table.d))
    s.set_predictor("router-pf")
    for mode in ("prefetch", "on_demand"):
        S = 3 + 11
        s.reset(S, True)
        s.prefill(prompt)
        s.decode_stream(mode, forced)
        if mode == "prefetch":
            assert np.array_equal(s.tokens(S)[2:], want.tokens)
            assert np.array_equal(s.trace("m", S), want.m)
            assert np.array_equal(s.trace("id_exec", S), want.ids)
            assert np.array_equal(s.trace("logits", S), want.final_logits)
    s.close()


@pytest.mark.parametrize("shape", ["g20", "mx"])
def test_other_baseline_shapes_vs_oracle(lib, shape):
    """BASELINE configs[2] (GPT-OSS-20B shape, topk-softmax gating) and configs[3]
    (Mixtral-8x7B shape with the lightweight estimator, est-pf), depth-truncated
    to 2 layers: prefetch decode bit-exact against the oracle."""
    from oracle.bindings import Config, Oracle
    if shape == "g20":
        cfg = dict(layers=2, experts=32, top_k=4, hidden=2880, expert_hidden=2880, vocab=256,
                   head_dim=64, seed=1, gating="topk-softmax")
        kind = "router-pf"
    else:
        cfg = dict(layers=2, experts=8, top_k=2, hidden=4096, expert_hidden=14336, vocab=256,
                   head_dim=128, seed=1, gating="topk-softmax")
        kind = "est-pf"
    orc = Oracle()
    om = orc.build_model(Config(**cfg), round_bf16=True)
    table = om.calibrate(4, 2, 256)
    est = orc.estimator(cfg["hidden"], 8, 4, cfg["experts"], cfg["layers"], seed=5)
    prompt = [3, 30, 200]
    want = om.generate_trace(prompt, 4, orc.make_predictor(kind, om, table, est), outputs=False)
    s = session(cfg, cache_fraction=0.5)
    s.load_default_vectors(np.array(table.d))
    s.load_estimator(cfg["hidden"], 8, 4, cfg["experts"], cfg["layers"], 1e-5, np.array(est.flat))
    s.set_predictor(kind)
    got = run_trace(s, prompt, 4, "prefetch")
    assert np.array_equal(got["tokens"], want.tokens)
    assert np.array_equal(got["id_exec"], want.ids)
    assert np.array_equal(got["g_exec"], want.gates)
    assert np.array_equal(got["m"], want.m)
    assert np.array_equal(got["logits"], want.final_logits)
    s.close()


@pytest.mark.parametrize("mode", ["prefetch", "on_demand"])
def test_expert_parallel_two_ranks_bit_exact(lib, toy_oracle, mode):
    """EP with two ranks sharing this GPU: each rank stores, caches
    and copies only experts e % 2 == rank, the dense path is replicated, and
    the combine exchanges raw expert rows through peer stores + system-scope
    arrival counters.  Both ranks must equal the single-GPU / oracle result."""
    import threading
    orc, om, table, est = toy_oracle
    forced = np.array([(29 * i + 3) % TOY["vocab"] for i in range(9)], np.int32)
    prompt = [8, 9, 10, 11]
    pred = orc.make_predictor("router-pf", om, table) if mode == "prefetch" else None
    want = om.generate_trace(prompt, 10, pred, outputs=True, forced=forced)
    ranks = [session(TOY, cache_fraction=0.5, ep_rank=r, ep_world=2) for r in (0, 1)]
    for s in ranks:
        s.load_default_vectors(np.array(table.d))
        s.set_predictor("router-pf")
    bufs = [s.ep_buffers() for s in ranks]
    for s in ranks:
        s.ep_connect([b[0] for b in bufs], [b[1] for b in bufs])
    S = len(prompt) + 9
    out = [None, None]
    errs = []

    def run(i):
        try:
            s = ranks[i]
            s.reset(S, True)
            s.prefill(prompt)
            s.decode_stream(mode, forced)
            out[i] = dict(tokens=s.tokens(S)[len(prompt) - 1:], m=s.trace("m", S),
                          ids=s.trace("id_exec", S), logits=s.trace("logits", S),
                          y=s.trace("y", S), c=s.counters())
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in (0, 1)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not errs, errs
    for o in out:
        assert np.array_equal(o["tokens"], want.tokens)
        assert np.array_equal(o["ids"], want.ids)
        assert np.array_equal(o["m"], want.m)
        assert np.array_equal(o["y"], want.outputs)
        assert np.array_equal(o["logits"], want.final_logits)
    # each rank copied only its own shard
    for s in ranks:
        ev = s.copy_events()
        assert all(e.hits + e.misses <= TOY["top_k"] for e in ev)
    for s in ranks:
        s.close()


def test_timeline_event_log(lib, toy_oracle):
    """smoe_timeline: the measured lane log of run_offloaded_decode — 3 compute
    events per layer per step, copy events serialised, breakdown sums to 1, and
    the decode itself is unchanged (tokens equal the graph path's)."""
    from paper_2603_19289_b200 import breakdown
    orc, om, table, est = toy_oracle
    forced = np.array([(17 * i + 5) % TOY["vocab"] for i in range(6)], np.int32)
    s = session(TOY, cache_fraction=0.25)
    s.load_default_vectors(np.array(table.d))
    s.set_predictor("router-pf")
    for mode in ("on_demand", "prefetch"):
        S = 3 + 6
        s.reset(S, False)
        s.prefill([4, 5, 6])
        ev = s.timeline(mode, 6, forced)
        toks_tl = s.tokens(S)
        s.reset(S, False)
        s.prefill([4, 5, 6])
        s.decode_stream(mode, forced)
        assert np.array_equal(toks_tl, s.tokens(S))
        comp = [e for e in ev if e.lane == 0]
        per_step = TOY["layers"] * 3 + (1 if mode == "prefetch" else 0)  # + layer-0 predictor
        assert len(comp) == 6 * per_step
        assert all(e.end_ms >= e.start_ms for e in ev)
        cp = sorted((e.start_ms, e.end_ms) for e in ev if e.lane == 1)
        for (a0, a1), (b0, b1) in zip(cp, cp[1:]):
            assert b0 >= a1 - 1e-3
        fr, tp = breakdown(ev)
        assert abs(fr.sum() - 1.0) < 1e-9 and tp > 0
    s.close()


def test_trace_bundle_matches_reference_writer(lib, tmp_path):
    """§8f: the GPU's trace bundle (smoe_write_trace_bundle) equals, file for
    file and byte for byte, the bundle the reference writes itself
    (TraceWriter over stream_decode_trace, the `specmoe trace` workload) on the
    same bf16 model and token stream; manifests agree field by field."""
    import json

    from oracle.bindings import REF_SO, Config, Ref
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    cfg = dict(layers=3, experts=8, top_k=2, hidden=64, expert_hidden=96, vocab=64, head_dim=16,
               seed=21)
    N = 12
    toks = np.array([(7 * i + 3) % cfg["vocab"] for i in range(N)], np.int32)
    ref = Ref()
    rm = ref.build_model(Config(**cfg), round_bf16=True)
    rdir, gdir = str(tmp_path / "ref"), str(tmp_path / "gpu")
    rm.write_trace(toks, N, rdir, "parity", 5)
    s = session(cfg, cache_fraction=0.5)
    s.reset(N, True)
    s.prefill(toks)
    s.write_trace_bundle(gdir, 0, N, N, "parity", 5)
    s.close()
    for f in ("token_ids", "s", "r", "m", "router_logits", "expert_ids", "expert_gates",
              "expert_outputs"):
        a = open(os.path.join(rdir, f + ".moet"), "rb").read()
        b = open(os.path.join(gdir, f + ".moet"), "rb").read()
        assert a == b, f
    ja = json.load(open(os.path.join(rdir, "manifest.json")))
    jb = json.load(open(os.path.join(gdir, "manifest.json")))
    assert np.float32(ja["config"].pop("eps")) == np.float32(jb["config"].pop("eps"))
    assert ja == jb


def _decode_after(cfg, prompt, n_dec, batched, frac, pred="router-pf", table=None):
    from paper_2603_19289_b200 import ModelConfig, Session
    s = Session(ModelConfig(**cfg), cache_fraction=frac, max_positions=512)
    s.init_weights_seeded()
    if table is not None:
        s.load_default_vectors(table)
    if frac == 1.0:
        s.preload_all()
    s.set_predictor(pred)
    P = len(prompt)
    S = P + n_dec
    s.reset(S, True)
    (s.prefill_batched if batched else s.prefill)(prompt)
    s.decode("prefetch", n_dec)
    out = {f: s.trace(f, S)[P:] for f in ("s", "r", "m", "lg_true", "id_exec", "g_exec", "y",
                                         "logits", "id_pred")}
    out["tokens"] = s.tokens(S)[P - 1:]
    s.close()
    return out


@pytest.mark.parametrize("plen,frac", [(20, 0.25), (150, 1.0)])
def test_batched_prefill_matches_token_prefill(lib, toy_oracle, plen, frac):
    """§8f row 2: the batched prefill (all prompt tokens per layer, experts
    loaded in slot-pool waves) leaves exactly the state the token-by-token
    prefill leaves: the next token and every later decode step (tokens,
    hidden states, router logits, decisions, expert outputs, logits) are
    bit-identical; the token path itself is pinned to the reference."""
    orc, om, table, est = toy_oracle
    rng = np.random.default_rng(plen)
    prompt = rng.integers(0, TOY["vocab"], plen).astype(np.int32)
    a = _decode_after(TOY, prompt, 6, False, frac, table=np.array(table.d))
    b = _decode_after(TOY, prompt, 6, True, frac, table=np.array(table.d))
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_batched_prefill_q30_layer_shapes(lib):
    """Q30 layer shapes (H 2048, 128 experts top-8, Hm 768), 2 layers: batched
    and token-by-token prefill agree bit for bit on the following decode."""
    cfg = dict(layers=2, experts=128, top_k=8, hidden=2048, expert_hidden=768, vocab=256,
               head_dim=128, seed=1)
    prompt = (np.arange(24) * 37 % 256).astype(np.int32)
    dv = np.zeros((2, 128, 2048), np.float32)
    a = _decode_after(cfg, prompt, 3, False, 0.25, table=dv)
    b = _decode_after(cfg, prompt, 3, True, 0.25, table=dv)
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_batched_prefill_mixtral_layer_shapes(lib):
    """Mixtral layer shapes (H 4096, Hm 14336: the down kernel stages two
    tokens' h rows at a time), 2 layers, cache 0.5: batched and token-by-token
    prefill agree bit for bit on the following decode."""
    cfg = dict(layers=2, experts=8, top_k=2, hidden=4096, expert_hidden=14336, vocab=256,
               head_dim=128, seed=1, gating="topk-softmax")
    prompt = (np.arange(20) * 53 % 256).astype(np.int32)
    dv = np.zeros((2, 8, 4096), np.float32)
    a = _decode_after(cfg, prompt, 3, False, 0.5, table=dv)
    b = _decode_after(cfg, prompt, 3, True, 0.5, table=dv)
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_long_context_split_attention_vs_oracle(lib):
    """Contexts beyond 512 positions take the split attention (16 CTAs share the
    scores and the context outputs; the last one forms the softmax): decode after
    a 700-token prompt stays bit-identical to the oracle."""
    from oracle.bindings import Config, Oracle
    cfg = dict(TOY, seed=13)
    orc = Oracle()
    om = orc.build_model(Config(**cfg), round_bf16=True)
    table = om.calibrate(64, 2, 32)
    prompt = list(np.random.default_rng(7).integers(0, TOY["vocab"], 700))
    want = om.generate_trace(prompt, 4, orc.make_predictor("router-pf", om, table), outputs=True)
    s = session(cfg, cache_fraction=0.5, max_positions=800)
    s.load_default_vectors(np.array(table.d))
    s.set_predictor("router-pf")
    got = run_trace(s, prompt, 4, "prefetch")
    w = dict(tokens=want.tokens, s=want.s, r=want.r, m=want.m, logits=want.logits, ids=want.ids,
             gates=want.gates, outputs=want.outputs, final_logits=want.final_logits,
             pred_ids=want.pred_ids, pred_gates=want.pred_gates)
    assert_trace_equal(got, w, True, len(prompt))
    s.close()


@pytest.mark.parametrize("head_dim,plen", [(128, 701), (64, 555)])
def test_long_context_split_attention_wide_heads_vs_oracle(lib, head_dim, plen):
    """The split attention's cp.async staging branch (head_dim / 16 outputs per
    CTA, a multiple of 4: head_dim 64 and 128 as on the Q30 / Mixtral shapes)
    and its tail handling (prompt lengths that are not multiples of 4 or 32)
    against the oracle, bit for bit."""
    from oracle.bindings import Config, Oracle
    cfg = dict(TOY, head_dim=head_dim, seed=17)
    orc = Oracle()
    om = orc.build_model(Config(**cfg), round_bf16=True)
    table = om.calibrate(64, 2, 32)
    prompt = list(np.random.default_rng(head_dim).integers(0, TOY["vocab"], plen))
    want = om.generate_trace(prompt, 4, orc.make_predictor("router-pf", om, table), outputs=True)
    s = session(cfg, cache_fraction=0.5, max_positions=plen + 64)
    s.load_default_vectors(np.array(table.d))
    s.set_predictor("router-pf")
    got = run_trace(s, prompt, 4, "prefetch")
    w = dict(tokens=want.tokens, s=want.s, r=want.r, m=want.m, logits=want.logits, ids=want.ids,
             gates=want.gates, outputs=want.outputs, final_logits=want.final_logits,
             pred_ids=want.pred_ids, pred_gates=want.pred_gates)
    assert_trace_equal(got, w, True, len(prompt))
    s.close()


def test_config_beyond_kernel_limits_is_rejected(lib):
    """A config whose kernels cannot launch (here head_dim 256 with a 4096-position
    KV capacity: the attention CTA would need more shared memory than the SM
    has) fails at session creation with the kernel named, not at first decode."""
    from paper_2603_19289_b200 import ModelConfig, Session
    with pytest.raises(ValueError, match="k_attn needs"):
        Session(ModelConfig(**dict(TOY, head_dim=256)), max_positions=4096)


def test_device_exp_equals_host_libm(lib):
    """The f64 exp of every softmax / silu on the path (exp_glibc.cuh) equals
    the host libm's exp — the one the reference calls — bit for bit, where
    CUDA's own exp(double) differs in the last bit for ~6 % of arguments."""
    import math
    from paper_2603_19289_b200 import engine
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.uniform(-40, 0, 200000), rng.uniform(-1, 0, 100000),
                        rng.uniform(-745, 709, 100000), rng.uniform(-1e-3, 1e-3, 50000),
                        (rng.uniform(-20, 0, 50000).astype(np.float32)).astype(np.float64),
                        [0.0, -0.0, -1e-300, 709.7, -745.2, -np.inf, np.inf]])
    y = engine.device_exp(x)
    want = np.array([math.exp(v) if v < 709.8 else math.inf for v in x])
    bad = np.flatnonzero(y.view(np.uint64) != want.view(np.uint64))
    assert bad.size == 0, (x[bad[:5]], y[bad[:5]], want[bad[:5]])
