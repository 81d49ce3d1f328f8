"""GPU tests of the offload machinery's alternative orderings, against the oracle:

* the device-side hit path (a request whose experts are all resident releases
  its layer on the device, no host round trip) changes no result and no
  counter, only who writes the ready value;
* host-ordered mode (the compute stream waits for the copy stream on a CUDA
  event, no device spin; selected automatically under ncu / compute-sanitizer)
  gives the same results as the device-ordered decode;
* run_offloaded_decode_ex returns the whole ExecutorResult (executor.hpp:39-44)
  from one run.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOY = dict(layers=8, experts=16, top_k=4, hidden=64, expert_hidden=128, vocab=256, head_dim=32,
           seed=4)


@pytest.fixture(scope="module")
def lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2603_19289_b200 import load_library
    return load_library()


@pytest.fixture(scope="module")
def toy():
    from oracle.bindings import Config, Oracle
    orc = Oracle()
    om = orc.build_model(Config(**TOY), round_bf16=True)
    table = om.calibrate(128, 2, 32)
    return orc, om, table


def _session(env: dict, frac=0.25, **kw):
    from paper_2603_19289_b200 import ModelConfig, Session
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: v for k, v in env.items() if v is not None})
    for k, v in env.items():
        if v is None:
            os.environ.pop(k, None)
    try:
        s = Session(ModelConfig(**TOY), cache_fraction=frac, max_positions=256, **kw)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    s.init_weights_seeded()
    return s


def _decode(s, table, prompt, n, mode, stream=None):
    s.load_default_vectors(np.array(table.d))
    s.set_predictor("router-pf")
    P = len(prompt)
    S = P + n
    s.reset(S, True)
    s.prefill(prompt)
    s.clear_stats()
    if stream is None:
        s.decode(mode, n)
    else:
        s.decode_stream(mode, stream[:n])
    out = {f: s.trace(f, S) for f in ("id_exec", "id_true", "s", "m", "logits")}
    out["tokens"] = s.tokens(S)
    c = s.counters()
    out["hits"], out["misses"], out["bytes"] = c["hits"], c["misses"], c["h2d_bytes"]
    return out, s.copy_events()


@pytest.mark.parametrize("mode", ["on_demand", "prefetch"])
def test_device_hit_path_changes_nothing_but_the_round_trip(lib, toy, mode):
    orc, om, table = toy
    prompt = [5, 77, 200, 13, 9]
    stream = list(np.random.default_rng(3).integers(0, 256, 24))
    a = _session({"SMOE_NO_FAST_HIT": "1"})
    b = _session({"SMOE_NO_FAST_HIT": None})
    ra, eva = _decode(a, table, prompt, 24, mode, stream)
    rb, evb = _decode(b, table, prompt, 24, mode, stream)
    for k in ra:
        assert np.array_equal(ra[k], rb[k]), k
    # the oracle agrees (teacher-forced stream through the same predictor)
    pred = orc.make_predictor("router-pf", om, table) if mode == "prefetch" else None
    forced = np.array(stream[:24], np.int32)
    want = om.generate_trace(prompt, 25, pred, forced=forced)
    assert np.array_equal(rb["id_exec"], want.ids)
    # every request is accounted; all-hit requests moved no bytes
    assert len(eva) == len(evb)
    all_hit = [e for e in evb if e.misses == 0]
    assert len(all_hit) > 0 and all(e.bytes == 0 for e in all_hit)
    a.close()
    b.close()


@pytest.mark.parametrize("mode", ["on_demand", "prefetch"])
def test_host_ordered_mode_matches_oracle(lib, toy, mode):
    """SMOE_HOST_ORDERED=1 (what ncu / compute-sanitizer get automatically):
    no graphs, no device spin on the copy lane, same results."""
    orc, om, table = toy
    prompt = [5, 77, 200, 13, 9]
    s = _session({"SMOE_HOST_ORDERED": "1"})
    got, ev = _decode(s, table, prompt, 10, mode)
    pred = orc.make_predictor("router-pf", om, table) if mode == "prefetch" else None
    want = om.generate_trace(prompt, 11, pred, outputs=True)
    P = len(prompt)
    assert np.array_equal(got["tokens"][P - 1:], want.tokens)
    assert np.array_equal(got["id_exec"], want.ids)
    assert np.array_equal(got["m"], want.m)
    assert s.kernels_per_step(mode) == -1  # never captured
    assert any(e.misses > 0 for e in ev)   # the copy lane really ran
    s.close()


@pytest.mark.parametrize("mode", ["on_demand", "prefetch"])
def test_run_offloaded_decode_ex_executor_result(lib, toy, mode):
    orc, om, table = toy
    prompt = [5, 77, 200, 13, 9]
    s = _session({})
    s.load_default_vectors(np.array(table.d))
    s.set_predictor("router-pf")
    toks, _ = s.run_offloaded_decode(prompt, 8, mode)
    toks2, events, per, max_res = s.run_offloaded_decode_ex(prompt, 8, mode)
    assert np.array_equal(toks, toks2)
    assert len(per) == 7 and all(p > 0 for p in per)
    lanes = {(e.lane, e.kind) for e in events}
    assert {(0, 0), (0, 1), (0, 2)} <= lanes
    # at most two layers' experts requested and not yet consumed at once (the
    # reference's double-buffer bound, executor.cpp:159-162); on demand, one
    assert 1 <= max_res <= (2 if mode == "prefetch" else 1)
    s.close()


@pytest.mark.parametrize("mode", ["on_demand", "prefetch"])
def test_fused_expert_ffn_matches_oracle(lib, toy, mode):
    """The opt-in one-launch expert FFN (SMOE_FUSED_FFN=1: gate/up, then down
    row-block pairs claimed by the finished CTAs, two chains per lane) is
    bit-identical to the oracle."""
    orc, om, table = toy
    prompt = [5, 77, 200, 13, 9]
    stream = list(np.random.default_rng(8).integers(0, 256, 12))
    s = _session({"SMOE_FUSED_FFN": "1"})
    assert s.path_info()["ffn_fused"]
    got, _ = _decode(s, table, prompt, 12, mode, stream)
    pred = orc.make_predictor("router-pf", om, table) if mode == "prefetch" else None
    want = om.generate_trace(prompt, 13, pred, outputs=True, forced=np.array(stream, np.int32))
    assert np.array_equal(got["id_exec"], want.ids)
    assert np.array_equal(got["m"], want.m)
    assert np.array_equal(got["logits"], want.final_logits)
    s.close()


@pytest.mark.parametrize("E,K", [(8, 2), (32, 4), (128, 8), (256, 16), (300, 8)])
@pytest.mark.parametrize("gating", ["softmax-topk-renorm", "topk-softmax"])
def test_decision_routine_vs_oracle(lib, E, K, gating):
    """warp_decision (every router / predictor / estimator decision on the path)
    against the oracle's make_decision on random rows, rows with exact ties
    (duplicated logits, the lower index must win), near ties one ulp apart,
    and large / tiny magnitudes (probabilities that underflow f32)."""
    from oracle.bindings import Oracle
    from paper_2603_19289_b200.engine import device_decide
    orc = Oracle()
    rng = np.random.default_rng(E * 31 + K)
    rows = [rng.normal(0, 1, E), rng.normal(0, 30, E), rng.normal(0, 1e-3, E)]
    for _ in range(40):
        r = rng.normal(0, 2, E).astype(np.float32)
        dup = rng.integers(0, E, max(2, E // 4))
        r[dup] = r[dup[0]]                     # exact ties
        j = int(rng.integers(0, E - 1))
        r[j + 1] = np.nextafter(r[j], np.float32(np.inf))  # one-ulp neighbours
        rows.append(r)
    rows.append(np.zeros(E))                   # everything tied
    rows.append(np.concatenate([[200.0], np.full(E - 1, -200.0)]))  # probabilities underflow
    lg = np.stack(rows).astype(np.float32)
    gid = 0 if gating == "softmax-topk-renorm" else 1
    ids, gates = device_decide(lg, K, gating)
    for r in range(lg.shape[0]):
        wi, wg = orc.make_decision(lg[r], K, gid)
        assert np.array_equal(ids[r], wi), (r, ids[r], wi)
        assert np.array_equal(gates[r].view(np.uint32), wg.view(np.uint32)), (r, gates[r], wg)


@pytest.mark.parametrize("mode", ["on_demand", "prefetch"])
def test_packed_expert_store_is_lossless_on_the_copy_path(lib, toy, mode):
    """Experts travel exponent-packed (xp11) and k_xp_unpack restores them in
    the slot: same trace as the raw store, bit for bit, with ~3/4 of the link
    bytes; and both equal the oracle."""
    orc, om, table = toy
    prompt = [5, 77, 200, 13, 9]
    stream = list(np.random.default_rng(4).integers(0, 256, 24))
    raw = _session({"SMOE_STORE_PACK": "0"})
    pk = _session({"SMOE_STORE_PACK": None})
    assert raw.path_info()["store_packed_blocks"] == 0
    assert pk.path_info()["store_packed_blocks"] == TOY["layers"] * TOY["experts"]
    ra, eva = _decode(raw, table, prompt, 24, mode, stream)
    rb, evb = _decode(pk, table, prompt, 24, mode, stream)
    for k in ("id_exec", "id_true", "s", "m", "logits", "tokens", "hits", "misses"):
        assert np.array_equal(ra[k], rb[k]), k
    assert ra["bytes"] > 0 and 0.66 < rb["bytes"] / ra["bytes"] < 0.74
    pred = orc.make_predictor("router-pf", om, table) if mode == "prefetch" else None
    want = om.generate_trace(prompt, 25, pred, forced=np.array(stream[:24], np.int32))
    assert np.array_equal(rb["id_exec"], want.ids)
    raw.close()
    pk.close()
