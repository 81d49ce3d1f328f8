"""Regression: decode parity while another process keeps the GPU busy.

Contexts of different processes time-slice the GPU, which stretches the gap
between a host call returning and its device work landing.  A pageable
cudaMemcpy on the legacy stream is not ordered before kernels on the session's
non-blocking streams, so the first prefill once read stale prompt tokens under
this load (and the two-process EP test failed).  Every transfer outside the
decode graph is now ordered on the compute stream (engine.cpp h2d/d2h/dset)."""
import subprocess
import sys
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOY = dict(layers=4, experts=16, top_k=4, hidden=64, expert_hidden=128, vocab=256, head_dim=32,
           seed=4)
HOG = ("import torch, time\n"
       "a = torch.randn(4096, 4096, device='cuda')\n"
       "t0 = time.time()\n"
       "while time.time() - t0 < 30:\n"
       "    a = (a @ a).clamp_(-1, 1)\n"
       "    torch.cuda.synchronize()\n")


def test_decode_parity_while_gpu_time_sliced():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from oracle.bindings import Config, Oracle
    from paper_2603_19289_b200 import ModelConfig, Session
    orc = Oracle(threads=2)
    om = orc.build_model(Config(**TOY), round_bf16=True)
    table = om.calibrate(32, 2, 32)
    forced = np.array([(13 * i + 7) % TOY["vocab"] for i in range(6)], np.int32)
    want = om.generate_trace([1, 2, 3], 7, orc.make_predictor("router-pf", om, table), forced=forced)
    hog = subprocess.Popen([sys.executable, "-c", HOG])
    try:
        time.sleep(6)  # the hog's context is up and running kernels
        for frac in (0.5, 1.0):
            s = Session(ModelConfig(**TOY), cache_fraction=frac, max_positions=64)
            s.init_weights_seeded()
            s.load_default_vectors(np.array(table.d))
            s.set_predictor("router-pf")
            if frac == 1.0:
                s.preload_all()
            s.reset(9, True)
            s.prefill([1, 2, 3])
            s.decode_stream("prefetch", forced)
            assert np.array_equal(s.tokens(9)[2:], want.tokens)
            assert np.array_equal(s.trace("m", 9), want.m)
            assert np.array_equal(s.trace("logits", 9), want.final_logits)
            s.close()
    finally:
        hog.kill()
        hog.wait()
