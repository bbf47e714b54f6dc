"""GPU: the per-element device executor (amlt_gpu_run_naive).

It evaluates the statement node by node in k order exactly like the
reference's run_naive (src/naive.cpp:65-117) and the C oracle restating it,
so on f64 it is bit-identical to the oracle even on real-valued data; f32 /
i32 see the same values rounded to the kernel dtype (int-valued: exact).
Also checks bounds, assignment statements, transposed / col-major operands
and the threshold classes, plus agreement with the tiled kernels.
"""
from __future__ import annotations

import numpy as np
import pytest

from tests.helpers import NP_DT, cast, check, make_inputs, oracle

pytestmark = pytest.mark.gpu

BODY_DTYPES = [("gemm", "f64"), ("gemm", "f32"), ("discount", "f64"), ("discount", "f32"),
               ("boost", "f64"), ("boost", "f32"), ("sqdiff", "f64"), ("sqdiff", "f32"),
               ("eqcount", "f64"), ("eqcount", "i32"), ("thrcount", "f64"), ("thrcount", "i32")]


def dev(x, dtype):
    import torch
    if x is None:
        return None
    return torch.from_numpy(np.ascontiguousarray(x.astype(NP_DT[dtype]))).cuda()


@pytest.mark.parametrize("body,dtype", BODY_DTYPES)
@pytest.mark.parametrize("dist", ["int", "baseline"])
def test_naive_matches_oracle(gpu_ctx, body, dtype, dist):
    import paper_2305_08872_b200 as P
    if dist == "baseline" and dtype == "i32" and body == "thrcount":
        pytest.skip("thrcount baseline data is real-valued")
    M, K, N = 67, 45, 131
    A, B, t, d = make_inputs(body, M, K, N, dist, seed=5)
    A, B, t, d = (cast(x, dtype) for x in (A, B, t, d))
    R0 = np.zeros((M, N))
    plan = gpu_ctx.plan(body, dtype)
    R = dev(R0, dtype)
    ops = P.Operands(dev(A, dtype), dev(B, dtype), R, dev(t, dtype), dev(d, dtype))
    el = P.run_naive(plan, ops, P.Bounds(0, M, 0, N, 0, K))
    assert el > 0
    want = oracle(body, A, B, t, d)
    got = R.cpu().numpy().astype(np.float64)
    if dtype == "f64" or dist == "int":
        check(body, dtype, got, want, exact=True, what="naive")
    else:
        check(body, dtype, got, want, A=A, B=B, what="naive f32")


def test_naive_bounds_accumulate_and_assign(gpu_ctx):
    import paper_2305_08872_b200 as P
    M, K, N = 40, 33, 50
    A, B, t, d = make_inputs("discount", M, K, N, "baseline", seed=3)
    R0 = np.arange(M * N, dtype=np.float64).reshape(M, N)
    b = (3, 31, 7, 45, 2, 29)
    for accumulate in (True, False):
        plan = gpu_ctx.plan("discount", "f64", accumulate=accumulate)
        R = dev(R0, "f64")
        ops = P.Operands(dev(A, "f64"), dev(B, "f64"), R, dev(t, "f64"), dev(d, "f64"))
        P.run_naive(plan, ops, P.Bounds(*b))
        want = oracle("discount", A, B, t, d, R0=R0, bounds=b, accumulate=accumulate)
        check("discount", "f64", R.cpu().numpy(), want, exact=True,
              what=f"naive bounds accumulate={accumulate}")


def test_naive_orientations_and_threshold_classes(gpu_ctx):
    import torch

    import paper_2305_08872_b200 as P
    M, K, N = 37, 29, 41
    rng = np.random.default_rng(11)
    A = rng.uniform(0, 10, (M, K))
    B = rng.uniform(1, 20, (K, N))
    tij = rng.uniform(20, 120, (M, N))
    want = np.zeros((M, N))
    for i in range(M):
        for j in range(N):
            acc = 0.0
            for k in range(K):
                p = A[i, k] * B[k, j]
                acc += p + (1.0 if p > tij[i, j] else 0.0) * (p - tij[i, j])
            want[i, j] = acc
    # A stored transposed (A[k][i]) and col-major B; thres[i][j] col-major
    At = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()           # K x M row-major
    Bc = torch.from_numpy(np.ascontiguousarray(B.T)).cuda().t()       # K x N col-major view
    Tc = torch.from_numpy(np.ascontiguousarray(tij.T)).cuda().t()     # M x N col-major view
    R = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    plan = gpu_ctx.plan("boost", "f64", layout_a=1, thres_class="ij")
    P.run_naive(plan, P.Operands(At, Bc, R, Tc, None), P.Bounds(0, M, 0, N, 0, K))
    got = R.cpu().numpy()
    assert np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300)) <= 1e-12
    # the tiled path on the same operands agrees with the naive one
    R2 = torch.zeros_like(R)
    P.run_subtask(plan, P.Operands(At, Bc, R2, Tc, None), P.TileParams(),
                  P.Bounds(0, M, 0, N, 0, K))
    assert np.max(np.abs(R2.cpu().numpy() - got) / np.maximum(np.abs(got), 1e-300)) <= 1e-12


def test_naive_constant_threshold_and_empty(gpu_ctx):
    import paper_2305_08872_b200 as P
    M, K, N = 16, 12, 24
    A, B, _, _ = make_inputs("thrcount", M, K, N, "baseline", seed=2)
    plan = gpu_ctx.plan("thrcount", "f64", thres_class="c", thres_value=100.0)
    R = dev(np.zeros((M, N)), "f64")
    ops = P.Operands(dev(A, "f64"), dev(B, "f64"), R)
    P.run_naive(plan, ops, P.Bounds(0, M, 0, N, 0, K))
    want = oracle("thrcount", A, B, np.full(N, 100.0))
    check("thrcount", "f64", R.cpu().numpy(), want, exact=True, what="q3 -tc")
    before = R.clone()
    P.run_naive(plan, ops, P.Bounds(0, 0, 0, N, 0, K))
    P.run_naive(plan, ops, P.Bounds(0, M, 0, N, 3, 3))
    assert bool((R == before).all())
