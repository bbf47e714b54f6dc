"""CPU: the arithmetic the byte-packed equality count relies on
(csrc/swar_eqcount.cu), checked exhaustively in numpy. The kernel itself is
covered on the GPU by tests/test_gpu_swar.py."""
from __future__ import annotations

import numpy as np


def differing_bytes(a4: np.ndarray, b4: np.ndarray) -> np.ndarray:
    """Count of differing byte lanes per word pair, as the kernel computes it:
    y = ((a ^ b) + 0x7F7F7F7F) & 0x80808080, count = bytes of y >> 7."""
    x = (a4 ^ b4).astype(np.uint64)
    y = (x + 0x7F7F7F7F) & 0x80808080
    y >>= 7
    return ((y & 0xFF) + ((y >> 8) & 0xFF) + ((y >> 16) & 0xFF) + (y >> 24)).astype(np.int64)


def test_byte_lane_zero_test_is_exact():
    """For every pair of 7-bit bytes, bit 7 of (a ^ b) + 0x7F is set exactly
    when a != b, and no carry leaves the byte (so lanes are independent)."""
    a, b = np.meshgrid(np.arange(128, dtype=np.uint64), np.arange(128, dtype=np.uint64))
    s = (a ^ b) + 0x7F
    assert (s < 0x100).all()  # no carry into the next lane
    assert np.array_equal((s & 0x80) != 0, a != b)


def test_packed_words_count_like_elementwise():
    """Random 4-lane words with adversarial lane mixes (equal, differing, the
    K padding pair 0 / 1): the packed count equals the elementwise count."""
    rng = np.random.default_rng(3)
    a = rng.integers(0, 128, (20000, 4)).astype(np.uint64)
    b = np.where(rng.random((20000, 4)) < 0.5, a, rng.integers(0, 128, (20000, 4))).astype(np.uint64)
    a[:100], b[:100] = 0, 1  # padding lanes always differ
    pack = lambda v: v[:, 0] | (v[:, 1] << 8) | (v[:, 2] << 16) | (v[:, 3] << 24)  # noqa: E731
    assert np.array_equal(differing_bytes(pack(a), pack(b)), (a != b).sum(axis=1))


def test_low_seven_bits_injective_on_any_128_window():
    """v -> v mod 128 (the packed byte) is injective on every window of 128
    consecutive int32 values, including windows crossing zero and the ends of
    the int32 range; a window of 129 values is not."""
    for lo in (-2**31, -200, -64, 0, 1000, 2**31 - 128):
        v = np.arange(lo, lo + 128, dtype=np.int64)
        assert len(np.unique(v.astype(np.int32).view(np.uint32) & 0x7F)) == 128
    v = np.arange(0, 129, dtype=np.int64)
    assert len(np.unique(v & 0x7F)) == 128


def test_byte_counters_fit_a_k_tile():
    """The per-tile partial holds 4 byte counters; each gains at most one per
    packed word, so a k tile of BK <= 255 words cannot overflow a lane."""
    bk = 32  # csrc/swar_eqcount.cu registers BK = 32
    assert bk <= 255
    per_lane = np.full(4, bk, dtype=np.uint64)
    word = per_lane[0] | (per_lane[1] << 8) | (per_lane[2] << 16) | (per_lane[3] << 24)
    assert ((word >> 8 * np.arange(4, dtype=np.uint64)) & 0xFF).sum() == 4 * bk
