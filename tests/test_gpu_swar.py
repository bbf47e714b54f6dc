"""GPU: the byte-packed equality-count variants (csrc/swar_eqcount.cu).

Four k of A and of B are packed as 7-bit bytes into one word and compared
four at a time, which is exact only when every value lies in one window of
128 consecutive integers (v mod 128 is then injective). These tests aim at
that condition and at the packing: windows away from zero and spanning
negative values, the window's edge (127 apart, then 128), the word padding of
K, sub-rectangles of a prior-valued R, and the guard that hands every other
input to the ordinary eqcount tile. Results are exact integers, compared
bit for bit with the oracle.
"""
from __future__ import annotations

import numpy as np
import pytest

from tests.helpers import oracle

pytestmark = pytest.mark.gpu


def swar_variants(plan):
    return [(vi, v.name) for vi, v in enumerate(plan.variants()) if "_swar_" in v.name]


def run(ctx, A, B, vi, R0=None, bounds=None):
    import torch

    import paper_2305_08872_b200 as P

    M, N = A.shape[0], B.shape[1]
    plan = ctx.plan("eqcount", "i32")
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    R = dev(np.zeros((M, N), np.int32) if R0 is None else R0.copy())
    b = P.Bounds(*bounds) if bounds else P.Bounds(0, M, 0, N, 0, A.shape[1])
    P.run_subtask(plan, P.Operands(dev(A), dev(B), R), P.TileParams(variant=vi), b)
    return R.cpu().numpy()


def want_of(A, B, R0=None, bounds=None):
    M, N = A.shape[0], B.shape[1]
    i0, i1, j0, j1, k0, k1 = bounds or (0, M, 0, N, 0, A.shape[1])
    R = np.zeros((M, N)) if R0 is None else R0.astype(np.float64)
    R[i0:i1, j0:j1] += oracle("eqcount", A[i0:i1, k0:k1].astype(np.float64),
                              B[k0:k1, j0:j1].astype(np.float64))
    return R


def test_swar_variants_registered(gpu_ctx):
    assert len(swar_variants(gpu_ctx.plan("eqcount", "i32"))) >= 2


@pytest.mark.parametrize("lo,hi", [(0, 16), (-8, 9), (1000, 1128), (-70, 58), (-2**31, -2**31 + 128),
                                   (2**31 - 128, 2**31 - 1)])
def test_window_exact(gpu_ctx, lo, hi):
    """Values inside one 128-wide window (the packed path), anywhere in the
    int32 range: exact. K = 20 (5 words, padded to 8) and K = 132."""
    rng = np.random.default_rng(abs(lo) % 1000 + 3)
    plan = gpu_ctx.plan("eqcount", "i32")
    for M, K, N in ((64, 20, 128), (97, 132, 36)):
        A = rng.integers(lo, hi, (M, K), dtype=np.int64).astype(np.int32)
        B = rng.integers(lo, hi, (K, N), dtype=np.int64).astype(np.int32)
        want = want_of(A, B)
        for vi, name in swar_variants(plan):
            got = run(gpu_ctx, A, B, vi)
            np.testing.assert_array_equal(got, want, err_msg=f"{name} [{lo}, {hi}) {M}x{K}x{N}")


@pytest.mark.parametrize("span", [127, 128, 1000, 2**32 - 1])
def test_window_edge_and_guard(gpu_ctx, span):
    """min and max exactly `span` apart: 127 stays on the packed path, wider
    spans go to the ordinary tile (values v and v + 128 would collide in 7
    bits, so the test puts such pairs in on purpose). Exact either way."""
    rng = np.random.default_rng(span % 997)
    M, K, N = 48, 64, 64
    base = -(2**31) if span == 2**32 - 1 else -40
    A = rng.integers(0, 8, (M, K)).astype(np.int64) + base
    B = rng.integers(0, 8, (K, N)).astype(np.int64) + base
    A[0, 0] = base + span
    if span >= 128:
        B[0, :] = base + 128 if span != 2**32 - 1 else base  # collides with base mod 128
        A[1, 0] = base + 128 if span != 2**32 - 1 else base + 2**32 - 1
    A, B = A.astype(np.int32), B.astype(np.int32)
    want = want_of(A, B)
    plan = gpu_ctx.plan("eqcount", "i32")
    for vi, name in swar_variants(plan):
        np.testing.assert_array_equal(run(gpu_ctx, A, B, vi), want, err_msg=f"{name} span {span}")


def test_sub_rectangle_prior_r(gpu_ctx):
    """A bounds sub-rectangle of an R holding prior values: only the rectangle
    changes, by exactly the counts over [k0, k1)."""
    rng = np.random.default_rng(5)
    M, K, N = 130, 200, 264
    A = rng.integers(0, 16, (M, K)).astype(np.int32)
    B = rng.integers(0, 16, (K, N)).astype(np.int32)
    R0 = rng.integers(-1000, 1000, (M, N)).astype(np.int32)
    bounds = (3, 121, 8, 200, 4, 180)
    want = want_of(A, B, R0, bounds)
    plan = gpu_ctx.plan("eqcount", "i32")
    for vi, name in swar_variants(plan):
        np.testing.assert_array_equal(run(gpu_ctx, A, B, vi, R0, bounds), want, err_msg=name)


def test_baseline_shape_sampled_rows(gpu_ctx):
    """Config 3b's shape and distribution (A, B uniform 0..15, M = 65536,
    N = 256, K = 1024) through each packed variant; sampled rows exact."""
    rng = np.random.default_rng(31)
    M, K, N = 65536, 1024, 256
    A = rng.integers(0, 16, (M, K)).astype(np.int32)
    B = rng.integers(0, 16, (K, N)).astype(np.int32)
    rows = np.unique(np.r_[0, M - 1, rng.integers(0, M, 10)])
    want = oracle("eqcount", A[rows].astype(np.float64), B.astype(np.float64))
    plan = gpu_ctx.plan("eqcount", "i32")
    for vi, name in swar_variants(plan):
        got = run(gpu_ctx, A, B, vi)
        np.testing.assert_array_equal(got[rows], want, err_msg=name)
