"""The C++ drop-in (paper_2603_19289_b200/dropin/specmoe_b200.hpp) linked with
the UNMODIFIED reference objects (oracle/_ref/libdropin_check.so, built where
/root/reference exists): on the same reference Model (bf16-representable
weights), specmoe_b200::run_offloaded_decode / generate with predictors from
specmoe_b200::make_* return the reference's own tokens from
specmoe::run_offloaded_decode / generate (executor.hpp:51-52,
speculation.hpp:102-103); a CPU predictor from the reference's factories is
refused (no CPU fallback)."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SO = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                  "libdropin_check.so")


@pytest.fixture(scope="module")
def lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    if not os.path.exists(SO):
        pytest.skip("oracle/_ref/libdropin_check.so not built (needs the reference headers)")
    L = C.CDLL(SO)
    L.dropin_last_error.restype = C.c_char_p
    L.dropin_check.argtypes = [C.c_int] * 7 + [C.c_uint64, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int,
                                                C.c_float] + [C.c_void_p] * 5
    return L


@pytest.mark.parametrize("mode,kind,frac", [(0, -1, 0.25), (1, 1, 0.25), (1, 0, 0.5), (1, 1, 1.0)])
def test_dropin_matches_reference_tokens(lib, mode, kind, frac):
    cfg = (4, 16, 4, 64, 96, 256, 32)
    prompt = np.array([3, 1, 4, 1, 5, 9, 2, 6], np.int32)
    n = 10
    ref, got, gref, ggot = (np.zeros(n, np.int32) for _ in range(4))
    info = np.zeros(4, np.int32)
    rc = lib.dropin_check(*cfg, 7, mode, kind, prompt.ctypes.data, len(prompt), n, frac,
                          ref.ctypes.data, got.ctypes.data, gref.ctypes.data, ggot.ctypes.data,
                          info.ctypes.data)
    assert rc == 0, lib.dropin_last_error().decode()
    assert np.array_equal(ref, got), (ref, got)
    assert np.array_equal(gref, ggot), (gref, ggot)
    assert info[1] > 0 and 1 <= info[0] <= 2  # events filled, residency bound


def test_dropin_refuses_cpu_predictor(lib):
    rc = lib.dropin_reject_cpu_predictor()
    assert rc == 1
    assert "specmoe_b200::make_" in lib.dropin_last_error().decode()
