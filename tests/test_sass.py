"""Arithmetic-order guards on the compiled sm_100a code (CPU-only: cuobjdump).

The kernels reproduce the reference's separately rounded `acc += w * x`
(numerics.cpp:136-147).  Packed products (FMUL2) are used, but ptxas contracts
an FMUL2 feeding a packed add into FFMA2 even for the _rn intrinsics, which
would fuse the rounding; the library must therefore contain no FFMA2, and the
chain kernels must contain the FMUL2 / FADD pair the design relies on."""
import os
import shutil
import subprocess

import pytest

BUILD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                     "paper_2603_19289_b200", "csrc", "build")
OBJ = os.path.join(BUILD, "kernels.o")
# every object whose chains must keep the reference's separately rounded
# products and adds (decode, batched prefill / decode, estimator training).
# The decode library also holds the tolerance mode (smoe_set_decode_mode(1):
# packed FFMA partial sums by design), so the decode kernels are checked in
# the exact-only build of the same source (kernels_exact.o, -DSMOE_EXACT_ONLY).
CHAIN_OBJS = ("kernels_exact.o", "prefill.o", "train_dev.o")


def _sass(obj=OBJ):
    if not os.path.exists(obj) or not shutil.which("cuobjdump"):
        pytest.skip(f"{os.path.basename(obj)} or cuobjdump not available")
    return subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True,
                          check=True).stdout


def _functions(sass):
    out, cur = {}, None
    for line in sass.splitlines():
        if "Function :" in line:
            cur = line.split("Function :")[1].strip()
            out[cur] = []
        elif cur:
            out[cur].append(line)
    return out


@pytest.mark.parametrize("obj", CHAIN_OBJS)
def test_no_packed_fma_anywhere(obj):
    sass = _sass(os.path.join(BUILD, obj))
    assert "FFMA2" not in sass, obj


def test_chain_kernels_use_separate_products_and_adds():
    fns = _functions(_sass(os.path.join(BUILD, "kernels_exact.o")))
    for short in ("k_qkv", "k_ffn_gu", "k_ffn_down", "k_router", "k_final", "k_wo"):
        body = "\n".join(next(v for k, v in fns.items() if short in k))
        assert "FMUL2" in body, short
        assert "FADD" in body, short


def test_tolerance_mode_uses_packed_fma():
    """The shipped decode object does carry the tolerance mode's FFMA2 chains."""
    fns = _functions(_sass())
    for short in ("k_qkv", "k_ffn_gu", "k_ffn_down", "k_router", "k_final"):
        body = "\n".join(next(v for k, v in fns.items() if short in k))
        assert "FFMA2" in body, short
