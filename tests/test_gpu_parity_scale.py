"""Parity at the benchmarked scale and on the paths that were only self-compared
(VERDICT r01 "Next round" item 1), against the CPU oracle:

* the headline run itself — Qwen3-30B-A3B shape, all 48 layers, HBM cache 25 %,
  default vectors from a 2000-token GPU calibration, 32-token prompt, 20
  teacher-forced stream steps, both offload modes — checked layer by layer,
  teacher-forced (tests/parity_check.py), with exact-match and near-tie counts;
* the GPU calibration at the Q30 shape (2-layer truncation, 2000 tokens)
  against the oracle's DefaultVectorAccumulator restatement;
* batched prefill and batched decode directly against oracle streams;
* the Qwen3-235B-A22B shape (2-layer truncation), single GPU and 2-rank EP.

Reports are printed and, when PARITY_REPORT_DIR is set, written there as JSON.
"""
import json
import os
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

Q30 = dict(layers=48, experts=128, top_k=8, hidden=2048, expert_hidden=768, vocab=256,
           head_dim=128, seed=1)
Q235 = dict(layers=2, experts=128, top_k=8, hidden=4096, expert_hidden=1536, vocab=256,
            head_dim=128, seed=1)
TOY = dict(layers=8, experts=16, top_k=4, hidden=64, expert_hidden=128, vocab=256, head_dim=32,
           seed=4)


@pytest.fixture(scope="module")
def lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2603_19289_b200 import load_library
    return load_library()


def _report(name, obj):
    print(f"\n[parity] {name}: {json.dumps(obj, default=str)}")
    d = os.environ.get("PARITY_REPORT_DIR")
    if d:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, f"{name}.json"), "w") as f:
            json.dump(obj, f, indent=1, default=str)


def _token_stream(n, vocab, seed):
    from oracle.bindings import Oracle
    return Oracle().token_stream(n, vocab, seed)


def test_headline_q30_48_layers_teacher_forced(lib):
    """The bench's headline workload, every layer of every recorded position."""
    from oracle.bindings import Config, Oracle
    from paper_2603_19289_b200 import ModelConfig, Session
    from parity_check import check_traces, gpu_trace
    P, N = 32, 20
    s = Session(ModelConfig(**Q30), cache_fraction=1.0, max_positions=300)
    s.init_weights_seeded()
    s.preload_all()
    dv, _ = s.calibrate(2000, 2, 256)
    s.set_cache_fraction(0.25)
    s.set_predictor("router-pf")
    prompt = _token_stream(P, Q30["vocab"], 3)
    forced = _token_stream(N, Q30["vocab"], 4)
    runs = []
    for mode in ("on_demand", "prefetch"):
        s.reset(P + N, True)
        s.prefill(prompt)
        s.clear_stats()
        s.decode_stream(mode, forced)
        c = s.counters()
        assert int(c["misses"].sum()) > 0  # the 25 % cache really copied
        runs.append((mode, gpu_trace(s, P + N, P), mode))
    s.close()
    orc = Oracle()
    om = orc.build_model(Config(**Q30), round_bf16=True, lazy=True)
    reps = check_traces(orc, om, Q30, runs, table=dv)
    for mode, rep in reps.items():
        summ = rep.summary()
        summ.update({"config": "q30 L48 cache 0.25, calib 2000, prompt 32, 20 stream steps",
                     "mode": mode})
        _report(f"headline_q30_{mode}", summ)
        assert rep.ok(), summ
        assert rep.checked["y"] == (P + N) * 48 * 8
    assert reps["prefetch"].checked["lg_pred"] == N * 47


def test_q30_calibration_vs_oracle_accumulator(lib):
    """smoe_calibrate at the Q30 layer shapes (2-layer truncation: per-layer
    weights depend only on (seed, label)), 2000 tokens, seq_len 256: default
    vectors and counts equal the oracle's accumulate_default_vectors."""
    from oracle.bindings import Config, Oracle
    from paper_2603_19289_b200 import ModelConfig, Session
    cfg = dict(Q30, layers=2)
    s = Session(ModelConfig(**cfg), cache_fraction=1.0, max_positions=300)
    s.init_weights_seeded()
    s.preload_all()
    d, cnt = s.calibrate(2000, 2, 256)
    s.close()
    om = Oracle().build_model(Config(**cfg), round_bf16=True)
    tb = om.calibrate(2000, 2, 256)
    exact = int(np.sum(d.view(np.uint32) == np.array(tb.d).view(np.uint32)))
    _report("q30_calibration", {"values": int(d.size), "exact": exact,
                                "counts_equal": bool(np.array_equal(cnt, np.array(tb.counts)))})
    assert np.array_equal(cnt, np.array(tb.counts))
    assert exact == d.size


def test_batched_prefill_vs_oracle(lib):
    """smoe_prefill_batched, then decode: every decode row equals the oracle's
    generate (not just the GPU's own token-by-token prefill)."""
    from oracle.bindings import Config, Oracle
    from paper_2603_19289_b200 import ModelConfig, Session
    orc = Oracle()
    om = orc.build_model(Config(**TOY), round_bf16=True)
    table = om.calibrate(64, 2, 32)
    prompt = np.random.default_rng(11).integers(0, TOY["vocab"], 77).astype(np.int32)
    want = om.generate_trace(prompt, 7, orc.make_predictor("router-pf", om, table), outputs=True)
    s = Session(ModelConfig(**TOY), cache_fraction=0.25, max_positions=256)
    s.init_weights_seeded()
    s.load_default_vectors(np.array(table.d))
    s.set_predictor("router-pf")
    P = len(prompt)
    S = P + 6
    s.reset(S, True)
    s.prefill_batched(prompt)
    s.decode("prefetch", 6)
    assert np.array_equal(s.tokens(S)[P - 1:], want.tokens)
    for f, w in (("m", want.m), ("s", want.s), ("id_exec", want.ids), ("y", want.outputs),
                 ("logits", want.final_logits)):
        assert np.array_equal(s.trace(f, S)[P:], w[P:]), f
    s.close()


@pytest.mark.parametrize("mode", ["on_demand", "prefetch"])
def test_batch_generate_vs_oracle_streams(lib, mode):
    """smoe_batch_generate: B = 5 sequences; each one's tokens and logits equal
    the oracle's own generate of that sequence."""
    from oracle.bindings import Config, Oracle
    from paper_2603_19289_b200 import ModelConfig, Session
    orc = Oracle()
    om = orc.build_model(Config(**TOY), round_bf16=True)
    table = om.calibrate(64, 2, 32)
    rng = np.random.default_rng(5)
    prompts = rng.integers(0, TOY["vocab"], (5, 9)).astype(np.int32)
    s = Session(ModelConfig(**TOY), cache_fraction=0.5, max_positions=128)
    s.init_weights_seeded()
    s.load_default_vectors(np.array(table.d))
    s.set_predictor("router-pf")
    toks, lg = s.batch_generate(prompts, 8, mode, logits=True)
    pred = orc.make_predictor("router-pf", om, table) if mode == "prefetch" else None
    for b in range(5):
        want = om.generate_trace(prompts[b], 8, pred)
        assert np.array_equal(toks[b], want.tokens), b
        assert np.array_equal(lg[b], want.final_logits[8:]), b
    s.close()


def _q235_oracle_trace(mode, prompt, forced, n_new):
    from oracle.bindings import Config, Oracle
    orc = Oracle()
    om = orc.build_model(Config(**Q235), round_bf16=True, lazy=True)
    table = om.calibrate(16, 2, 16)
    pred = orc.make_predictor("router-pf", om, table) if mode == "prefetch" else None
    return om.generate_trace(prompt, n_new, pred, outputs=True, forced=forced), np.array(table.d)


@pytest.mark.parametrize("mode", ["on_demand", "prefetch"])
def test_q235_shape_vs_oracle_single_and_two_rank_ep(lib, mode):
    """Qwen3-235B-A22B layer shapes (H 4096, 128 experts top-8, Hm 1536; 2-layer
    truncation): the single-GPU decode and the 2-rank expert-parallel decode
    (ranks sharing this GPU) both equal the oracle bit for bit."""
    from paper_2603_19289_b200 import ModelConfig, Session
    prompt = [17, 230, 5]
    forced = np.array([(41 * i + 7) % 256 for i in range(6)], np.int32)
    want, table = _q235_oracle_trace(mode, prompt, forced, 7)
    S = len(prompt) + 6

    def run(s):
        s.load_default_vectors(table)
        s.set_predictor("router-pf")
        s.reset(S, True)
        s.prefill(prompt)
        s.decode_stream(mode, forced)
        return dict(tokens=s.tokens(S)[len(prompt) - 1:], m=s.trace("m", S), ids=s.trace("id_exec", S),
                    logits=s.trace("logits", S))

    s = Session(ModelConfig(**Q235), cache_fraction=0.25, max_positions=64)
    s.init_weights_seeded()
    got = run(s)
    s.close()
    for k, w in (("tokens", want.tokens), ("m", want.m), ("ids", want.ids),
                 ("logits", want.final_logits)):
        assert np.array_equal(got[k], w), k
    ranks = [Session(ModelConfig(**Q235), cache_fraction=0.25, max_positions=64, ep_rank=r, ep_world=2)
             for r in (0, 1)]
    for r in ranks:
        r.init_weights_seeded()
    bufs = [r.ep_buffers() for r in ranks]
    for r in ranks:
        r.ep_connect([b[0] for b in bufs], [b[1] for b in bufs])
    out, errs = [None, None], []

    def worker(i):
        try:
            out[i] = run(ranks[i])
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=worker, args=(i,)) for i in (0, 1)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    for o in out:
        for k, w in (("tokens", want.tokens), ("m", want.m), ("ids", want.ids),
                     ("logits", want.final_logits)):
            assert np.array_equal(o[k], w), k
    for r in ranks:
        r.close()
