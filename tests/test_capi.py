"""The C ABI library loads on a GPU-less host and exports every symbol
include/smoe.h declares; without a GPU it fails loudly (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "smoe.h")
LIB = os.path.join(ROOT, "paper_2603_19289_b200", "libsmoe_b200.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(smoe_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("smoe_session_create", "smoe_run_offloaded_decode", "smoe_set_predictor",
                 "smoe_load_default_vectors", "smoe_load_estimator", "smoe_counters",
                 "smoe_copy_events", "smoe_step", "smoe_calibrate"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.fail("libsmoe_b200.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_lists_every_symbol():
    from paper_2603_19289_b200.engine import EXPORTS
    assert sorted(EXPORTS) == declared_symbols()


def test_invalid_config_is_invalid_argument():
    from paper_2603_19289_b200 import ModelConfig, Session
    with pytest.raises(ValueError, match="k must satisfy"):
        Session(ModelConfig(layers=2, experts=4, top_k=5, hidden=8, expert_hidden=8, vocab=8,
                            head_dim=4))
    with pytest.raises(ValueError, match="head_dim must be even"):
        Session(ModelConfig(layers=2, experts=4, top_k=2, hidden=8, expert_hidden=8, vocab=8,
                            head_dim=3))


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_19289_b200 import ModelConfig, Session, SmoeError
    with pytest.raises(SmoeError):
        Session(ModelConfig(layers=2, experts=4, top_k=2, hidden=16, expert_hidden=8, vocab=8,
                            head_dim=8))
