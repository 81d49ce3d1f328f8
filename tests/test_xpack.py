"""Exponent-packed expert blocks (xp11, engine.h / xpack.cpp): the pinned
store's wire format must be lossless for every bf16 bit pattern, pack the
Gaussian-like expert weights to ~11 bits per weight, and refuse blocks that
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
    assert 0.68 <= ratio < 0.71, ratio  # 2 + 8 bits, 4 more for the quarter outside the top-3 exponents
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


def test_primary_secondary_and_escapes():
    """Three most frequent exponents get 2-bit codes, the next binades 4-bit
    codes, and values outside the 15-binade secondary window escape (listed
    in ascending index order)."""
    rng = np.random.default_rng(5)
    n = 4096
    e = rng.choice([120, 121, 119], n, p=[0.5, 0.3, 0.2])     # primary exponents
    e[rng.choice(n, 300, replace=False)] = 117                 # secondary
    e[rng.choice(n, 40, replace=False)] = 90                   # far below the window: escapes
    raw = ((rng.integers(0, 2, n) << 15) | (e << 7) | rng.integers(0, 128, n)).astype(np.uint16)
    raw[17] = 0          # +0 (exponent 0)
    raw[4000] = 0x8001   # negative subnormal
    packed = xp_pack(raw)
    assert packed is not None
    hdr = np.frombuffer(packed[:32], np.uint32)
    assert sorted(hdr[4:7].tolist()) == [119, 120, 121]
    nesc = int(hdr[3])
    esc = np.frombuffer(packed[len(packed) - 8 * nesc:], np.uint32).reshape(-1, 2)
    assert nesc >= 40 and np.all(np.diff(esc[:, 0].astype(np.int64)) > 0)
    assert np.array_equal(xp_unpack(packed, n), raw)


def test_unpackable_blocks_are_refused():
    rng = np.random.default_rng(3)
    wide = rng.integers(0, 1 << 16, 4096, dtype=np.uint16)  # uniform bit patterns: ~90 % escapes
    assert xp_pack(wide) is None
    assert xp_pack(np.zeros(128, np.uint16)) is None  # n % 256 != 0


def test_unpack_rejects_foreign_bytes():
    with pytest.raises(ValueError):
        xp_unpack(bytes(64), 256)
