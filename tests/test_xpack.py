"""Exponent-packed expert blocks (xp12, engine.h / xpack.cpp): the pinned
store's wire format must be lossless for every bf16 bit pattern, pack the
Gaussian-like expert weights to ~12 bits per weight, and refuse blocks that
would not shrink.  Host-only (no GPU): the device decoder k_xp_unpack is
covered by every bit-exact GPU test, which copies experts through it."""
import numpy as np
import pytest

from paper_2603_19289_b200 import xp_pack, xp_unpack


def _bf16(x):
    """Round-to-nearest-even f32 -> bf16 bit patterns."""
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def test_gaussian_block_packs_to_12_bits_losslessly():
    rng = np.random.default_rng(1)
    raw = _bf16(rng.normal(0.0, 0.4 / np.sqrt(2048), 3 * 2048 * 96))  # Q30 init scale
    packed = xp_pack(raw)
    assert packed is not None
    ratio = len(packed) / (raw.size * 2)
    assert 0.75 <= ratio < 0.76, ratio  # 12 bits per weight + header + a few escapes
    assert np.array_equal(xp_unpack(packed, raw.size), raw)


def test_every_bit_pattern_round_trips():
    """All 65536 bf16 patterns (zeros, subnormals, inf, NaN payloads) inside a
    Gaussian block: the out-of-window ones travel as escapes."""
    rng = np.random.default_rng(2)
    base = _bf16(rng.normal(0.0, 0.01, 1 << 22))
    raw = base.copy()
    idx = rng.choice(raw.size, 65536, replace=False)
    raw[np.sort(idx)] = np.arange(65536, dtype=np.uint16)
    packed = xp_pack(raw)
    assert packed is not None
    assert np.array_equal(xp_unpack(packed, raw.size), raw)


def test_window_edges_and_escape_order():
    # exponents exactly at base and base + 14 are codes; base - 1 and zero escape
    e_max = 127
    raw = np.full(4096, (e_max - 3) << 7, np.uint16)
    raw[5] = e_max << 7                # sets base = e_max - 14
    raw[6] = (e_max - 14) << 7 | 0x7f  # == base: a code
    raw[7] = (e_max - 15) << 7         # base - 1: escape
    raw[8] = 0x8000                    # -0: escape
    raw[4095] = 1                      # subnormal: escape
    packed = xp_pack(raw)
    assert packed is not None
    hdr = np.frombuffer(packed[:16], np.uint32)
    assert hdr[1] == e_max - 14
    n = raw.size
    esc = np.frombuffer(packed[16 + n // 2 + n:], np.uint32).reshape(-1, 2)
    assert np.all(np.diff(esc[:, 0].astype(np.int64)) > 0)  # ascending indices
    assert np.array_equal(xp_unpack(packed, n), raw)


def test_unpackable_blocks_are_refused():
    rng = np.random.default_rng(3)
    wide = rng.integers(0, 1 << 16, 4096, dtype=np.uint16)  # uniform bit patterns: ~90 % escapes
    assert xp_pack(wide) is None
    assert xp_pack(np.zeros(12, np.uint16)) is None  # n % 8 != 0


def test_unpack_rejects_foreign_bytes():
    with pytest.raises(ValueError):
        xp_unpack(bytes(64), 8)
