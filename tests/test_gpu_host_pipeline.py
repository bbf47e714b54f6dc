"""GPU parity of the host-buffer entry's copy / compute pipeline (row bands
of A / R, K panels of B), the tuned host entry (run_host_adaptive, the
reference's run_adaptive over host MatrixBuffers, src/engine.cpp:165-169),
and the row-band multi-GPU paths: the persistent single-process group
(amlt_sharded_*) and the one-process-per-GPU broadcast entry (torchrun).

The K panels split the reduction over k into consecutive launches that
accumulate into R, so integer-valued data (the reference's determinism
convention, acceptance.cpp:109-132) must stay bit-exact; the tests force
small panels with AMLT_HOST_PANEL_BYTES.
"""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

from tests.helpers import check, make_inputs, oracle

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture
def small_panels(monkeypatch):
    monkeypatch.setenv("AMLT_HOST_PANEL_BYTES", "65536")


@pytest.mark.parametrize("body", ["discount", "gemm", "boost", "eqcount", "sqdiff"])
@pytest.mark.parametrize("r_zero", [False, True])
def test_panels_and_bands_bit_exact(gpu_ctx, small_panels, body, r_zero):
    """1100 rows (several row bands) x K = 1000 (three K panels of B): the
    pipeline's result equals the oracle's bit for bit on int-valued data,
    R's prior values included."""
    import paper_2305_08872_b200 as P

    M, K, N = 1100, 1000, 300
    A, B, t, d = make_inputs(body, M, K, N, "int", seed=71)
    rng = np.random.default_rng(72)
    R0 = np.zeros((M, N)) if r_zero else rng.integers(-8, 9, (M, N)).astype(np.float64)
    want = oracle(body, A, B, t, d, R0=R0)
    R = R0.copy()
    plan = gpu_ctx.plan(body, "f64")
    el = P.run_host(plan, P.Operands(A, B, R, t, d), P.Bounds(0, M, 0, N, 0, K), r_zero=r_zero)
    assert el > 0
    check(body, "f64", R, want, exact=True, what=f"pipeline {body} r_zero={r_zero}")


def test_panels_sub_rectangle(gpu_ctx, small_panels):
    """Bounds with k0 > 0, j0 > 0 and a row sub-range: only R(bounds) moves."""
    import paper_2305_08872_b200 as P

    M, K, N = 1300, 1100, 260
    A, B, t, d = make_inputs("discount", M, K, N, "int", seed=73)
    R0 = np.random.default_rng(74).integers(-8, 9, (M, N)).astype(np.float64)
    b = (40, 1250, 6, 250, 64, 1090)
    want = oracle("discount", A, B, t, d, R0=R0, bounds=b)
    R = R0.copy()
    P.run_host(gpu_ctx.plan("discount", "f64"), P.Operands(A, B, R, t, d), P.Bounds(*b))
    check("discount", "f64", R, want, exact=True, what="pipeline sub-rectangle")


def test_panels_baseline_distribution(gpu_ctx, small_panels):
    """Config-0 distributions through the panelled pipeline: within 1e-12."""
    import paper_2305_08872_b200 as P

    M, K, N = 1024, 1024, 1024
    A, B, t, d = make_inputs("discount", M, K, N, "baseline", seed=75)
    want = oracle("discount", A, B, t, d)
    R = np.zeros((M, N))
    plan = gpu_ctx.plan("discount", "f64")
    names = [v.name for v in plan.variants()]
    theta = next(i for i, n in enumerate(names) if "_theta_" in n)
    for tile in (None, P.TileParams(variant=theta)):
        R[:] = 0
        P.run_host(plan, P.Operands(A, B, R, t, d), P.Bounds(0, M, 0, N, 0, K), params=tile, r_zero=True)
        check("discount", "f64", R, want, what=f"pipeline baseline tile={tile}")


def test_run_host_adaptive_tunes_then_reuses(gpu_ctx):
    """The first call of a shape tunes (row-band or scratch trials) and
    reports its trials; the second reuses the winner (from_cache) through the
    pipeline. Coverage: disjoint rectangles whose union is the bounds."""
    import paper_2305_08872_b200 as P

    M, K, N = 1536, 512, 640
    A, B, t, d = make_inputs("discount", M, K, N, "int", seed=76)
    want = oracle("discount", A, B, t, d)
    gpu_ctx.clear_tuning_cache()
    plan = gpu_ctx.plan("discount", "f64")
    reps = []
    for _ in range(2):
        R = np.zeros((M, N))
        reps.append(P.run_host_adaptive(plan, P.Operands(A, B, R, t, d), P.Bounds(0, M, 0, N, 0, K),
                                        r_zero=True))
        check("discount", "f64", R, want, exact=True, what="run_host_adaptive")
    first, second = reps
    assert first.trials and (first.tuned or first.scratch_tuned)
    assert not second.trials and second.from_cache and second.best_variant == first.best_variant
    for rep in reps:
        area = sum((c.i1 - c.i0) * (c.j1 - c.j0) * (c.k1 - c.k0) for c in rep.coverage)
        assert area == M * N * K
        cells = np.zeros((M, N), dtype=np.int32)
        for c in rep.coverage:
            if c.k0 == 0:
                cells[c.i0:c.i1, c.j0:c.j1] += 1
        assert (cells == 1).all()
        assert rep.total_seconds > 0


def test_bcast_flag_without_communicator(gpu_ctx, small_panels):
    """AMLT_HOST_BCAST_SHARED without a communicator: every operand comes
    from this rank's host memory."""
    import paper_2305_08872_b200 as P

    M, K, N = 300, 600, 200
    A, B, t, d = make_inputs("discount", M, K, N, "int", seed=77)
    want = oracle("discount", A, B, t, d)
    R = np.zeros((M, N))
    assert gpu_ctx.comm_size == 1
    P.run_host(gpu_ctx.plan("discount", "f64"), P.Operands(A, B, R, t, d), P.Bounds(0, M, 0, N, 0, K),
               bcast=True)
    check("discount", "f64", R, want, exact=True, what="bcast, no communicator")


@pytest.mark.parametrize("body", ["discount", "gemm"])
def test_broadcast_path_on_a_one_rank_communicator(small_panels, body):
    """The NCCL broadcast path of the host pipeline on one GPU: a real
    one-rank communicator (amlt_gpu_comm_unique_id / _attach), so every
    ncclBroadcast, group and stream / event hand-off of the multi-rank path
    runs (the broadcasts themselves are no-ops). B in several K panels; two
    calls (the first tunes); bit-exact."""
    import paper_2305_08872_b200 as P

    ctx = P.Context(0)
    try:
        ctx.attach_comm(0, 1)
        assert ctx.comm_size == 1
        M, K, N = 1100, 1000, 300
        A, B, t, d = make_inputs(body, M, K, N, "int", seed=80)
        want = oracle(body, A, B, t, d)
        plan = ctx.plan(body, "f64")
        for _ in range(2):
            R = np.zeros((M, N))
            P.run_host_adaptive(plan, P.Operands(A, B, R, t, d), P.Bounds(0, M, 0, N, 0, K), r_zero=True,
                                bcast=True)
            check(body, "f64", R, want, exact=True, what=f"one-rank broadcast path {body}")
        lay = ctx.last_host_layout()
        # every rank cuts B the same way: geometric panels from K and the panel count alone
        assert lay["bcast"] == 1 and lay["k_panels"] > 1 and lay["k_panel0"] < K // lay["k_panels"], lay
        ctx.detach_comm()
    finally:
        ctx.close()


def _pinned(x):
    """A page-locked (cudaHostAlloc, device-mapped) copy of a numpy array."""
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).pin_memory()


@pytest.mark.parametrize("body", ["discount", "gemm", "boost", "eqcount", "sqdiff"])
@pytest.mark.parametrize("r_zero", [False, True])
def test_zero_copy_result_bit_exact(gpu_ctx, small_panels, body, r_zero):
    """R in pinned host memory: the rows after band 0 run as one launch whose
    epilogue stores R straight into host memory (and reads R's prior values
    from there without R_ZERO); band 0 goes through the staged panels.
    Bit-exact against the oracle, and the trace shows the zero-copy layout."""
    import paper_2305_08872_b200 as P
    from tests.helpers import NP_DT

    dtype = {"eqcount": "i32", "sqdiff": "f32"}.get(body, "f64")
    npd = NP_DT[dtype]
    M, K, N = 1300, 1000, 300
    A, B, t, d = make_inputs(body, M, K, N, "int", seed=91)
    rng = np.random.default_rng(92)
    R0 = np.zeros((M, N)) if r_zero else rng.integers(-8, 9, (M, N)).astype(np.float64)
    want = oracle(body, A, B, t, d, R0=R0)
    R = _pinned(R0.astype(npd))
    ops = P.Operands(_pinned(A.astype(npd)), _pinned(B.astype(npd)), R,
                     None if t is None else t.astype(npd), None if d is None else d.astype(npd))
    plan = gpu_ctx.plan(body, dtype)
    P.run_host(plan, ops, P.Bounds(0, M, 0, N, 0, K), r_zero=r_zero)
    lay = gpu_ctx.last_host_layout()
    assert lay["zero_copy_r"] == 1 and lay["bands"] == 2 and lay["k_panels"] > 1, lay
    check(body, dtype, R.numpy().astype(np.float64), want, exact=True, what=f"zero-copy {body} r_zero={r_zero}")


def test_zero_copy_sub_rectangle_and_tuned_theta(gpu_ctx, small_panels):
    """Zero-copy R with a bounds sub-rectangle (k0, j0 > 0, a row range): R
    outside the bounds, in host memory, is never touched. Then the tuned
    path: run_host_adaptive tunes (staged, whole task), the second call runs
    the cached winner (theta form forced through TileParams too) with B
    prepared panel by panel into one whole-K preparation."""
    import paper_2305_08872_b200 as P

    M, K, N = 1400, 1100, 260
    A, B, t, d = make_inputs("discount", M, K, N, "int", seed=93)
    R0 = np.random.default_rng(94).integers(-8, 9, (M, N)).astype(np.float64)
    b = (40, 1350, 6, 250, 64, 1090)
    want = oracle("discount", A, B, t, d, R0=R0, bounds=b)
    plan = gpu_ctx.plan("discount", "f64")
    R = _pinned(R0)
    P.run_host(plan, P.Operands(A, B, R, t, d), P.Bounds(*b))
    assert gpu_ctx.last_host_layout()["zero_copy_r"] == 1
    check("discount", "f64", R.numpy(), want, exact=True, what="zero-copy sub-rectangle")

    theta = next(i for i, v in enumerate(plan.variants()) if "_theta_" in v.name)
    want0 = oracle("discount", A, B, t, d)
    R = _pinned(np.zeros((M, N)))
    P.run_host(plan, P.Operands(A, B, R, t, d), P.Bounds(0, M, 0, N, 0, K), params=P.TileParams(variant=theta),
               r_zero=True)
    assert gpu_ctx.last_host_layout()["zero_copy_r"] == 1
    check("discount", "f64", R.numpy(), want0, exact=True, what="zero-copy theta")
    gpu_ctx.clear_tuning_cache()
    for it in range(2):
        R = _pinned(np.zeros((M, N)))
        rep = P.run_host_adaptive(plan, P.Operands(A, B, R, t, d), P.Bounds(0, M, 0, N, 0, K), r_zero=True)
        check("discount", "f64", R.numpy(), want0, exact=True, what=f"run_host_adaptive zero-copy call {it}")
        assert rep.from_cache == (it == 1)
        lay = gpu_ctx.last_host_layout()
        # (the tuning call runs whole, staged; the cached winner, split-K or not, zero-copy)
        assert (lay["tuned"], lay["zero_copy_r"]) == ((1, 0) if it == 0 else (0, 1)), (lay, rep.best_kc)


def test_pageable_or_disabled_zero_copy_stays_staged(gpu_ctx, small_panels, monkeypatch):
    """Pageable R (numpy) and AMLT_HOST_NO_ZEROCOPY=1 keep the staged
    pipeline (R bands copied out); same results."""
    import paper_2305_08872_b200 as P

    M, K, N = 1300, 700, 200
    A, B, t, d = make_inputs("discount", M, K, N, "int", seed=95)
    want = oracle("discount", A, B, t, d)
    plan = gpu_ctx.plan("discount", "f64")
    R = np.zeros((M, N))
    P.run_host(plan, P.Operands(A, B, R, t, d), P.Bounds(0, M, 0, N, 0, K), r_zero=True)
    lay = gpu_ctx.last_host_layout()
    assert lay["zero_copy_r"] == 0 and lay["k_panels"] > 1, lay
    check("discount", "f64", R, want, exact=True, what="pageable R")
    monkeypatch.setenv("AMLT_HOST_NO_ZEROCOPY", "1")
    Rp = _pinned(np.zeros((M, N)))
    P.run_host(plan, P.Operands(A, B, Rp, t, d), P.Bounds(0, M, 0, N, 0, K), r_zero=True)
    assert gpu_ctx.last_host_layout()["zero_copy_r"] == 0
    check("discount", "f64", Rp.numpy(), want, exact=True, what="zero-copy disabled")


def _shard_rows(M, n):
    """First and last row of every device's band (64-row edges, as the group cuts)."""
    edges = [min(M, (M * d // n + 32) // 64 * 64) for d in range(n)] + [M]
    rows = set()
    for r0, r1 in zip(edges[:-1], edges[1:]):
        if r1 > r0:
            rows.update((r0, r1 - 1))
    return sorted(rows)


def test_sharded_group_all_devices(gpu_ctx, small_panels):
    """The persistent group over every visible device (one on a 1-GPU box):
    run twice (the second run reuses the tuned winners); the first and last
    row of every device's band match the oracle bit for bit."""
    import torch

    import paper_2305_08872_b200 as P

    n = torch.cuda.device_count()
    M, K, N = 256 * n + 70, 700, 300
    A, B, t, d = make_inputs("discount", M, K, N, "int", seed=78)
    rows = _shard_rows(M, n)
    want = oracle("discount", A[rows], B, t, d)
    g = P.ShardedGroup(list(range(n)))
    try:
        for it in range(2):
            R = np.zeros((M, N))
            el, reps = g.run(P.Operands(A, B, R, t, d), P.Bounds(0, M, 0, N, 0, K), body="discount",
                             r_zero=True)
            assert el > 0 and len(reps) == n
            check("discount", "f64", R[rows], want, exact=True, what=f"group run {it}")
            if it == 1:
                assert all(r.from_cache or not r.trials for r in reps)
        # R pinned: every device's band writes its rows straight into it (zero-copy)
        R = _pinned(np.zeros((M, N)))
        el, reps = g.run(P.Operands(A, B, R, t, d), P.Bounds(0, M, 0, N, 0, K), body="discount", r_zero=True)
        check("discount", "f64", R.numpy()[rows], want, exact=True, what="group run, pinned R")
        # a task text (generated body) through the same group
        src = ("where(i in [0..M] and j in [0..N] and k in [0..K]) {\n"
               "  R[i][j] += A[i][k]*B[k][j] + (A[i][k] > thres[j]);\n}\n")
        R = np.zeros((M, N))
        g.run(P.Operands(A, B, R, None, None, (t,)), P.Bounds(0, M, 0, N, 0, K), source=src)
        want2 = (A[rows] @ B) + (A[rows][:, :, None] > t[None, None, :]).sum(axis=1)
        check("discount", "f64", R[rows], want2, exact=True, what="group, generated body")
    finally:
        g.close()


@pytest.mark.skipif("not __import__('torch').cuda.is_available() or "
                    "__import__('torch').cuda.device_count() < 2", reason="needs >= 2 GPUs")
def test_torchrun_broadcast_entry(tmp_path):
    """One process per GPU (torchrun, NCCL): each rank attaches the
    communicator, rank 0 alone holds B / thres / dis in host memory, every
    rank its own A / R rows; the first and last row of every band match the
    oracle (tests/mp_bcast_worker.py)."""
    import torch

    n = torch.cuda.device_count()
    out = tmp_path / "rows.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29531",
           os.path.join(ROOT, "tests", "mp_bcast_worker.py"), str(out)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    z = np.load(out)
    assert z["bad"] == 0, f"{int(z['bad'])} mismatching rows"


@pytest.mark.parametrize("case", range(24))
def test_random_pipeline_cases_bit_exact(gpu_ctx, small_panels, case):
    """Randomised sweep of the host pipeline: shapes large enough for several
    row bands, B cut into K panels (small panels forced), a bounds
    sub-rectangle of a prior-valued (or zero, with AMLT_HOST_R_ZERO) R, every
    fixed body / dtype, transposed or col-major operands (which fall back to
    one band / one panel), run_host or run_host_adaptive; int-valued data, so
    bit-exact against the oracle, R outside the bounds untouched."""
    import paper_2305_08872_b200 as P
    from tests.helpers import NP_DT

    bodies = [("gemm", "f64"), ("gemm", "f32"), ("discount", "f64"), ("boost", "f64"), ("boost", "f32"),
              ("sqdiff", "f32"), ("eqcount", "i32"), ("thrcount", "f64")]
    rng = np.random.default_rng(7000 + case)
    body, dtype = bodies[case % len(bodies)]
    M, K, N = int(rng.integers(1024, 2600)), int(rng.integers(300, 1300)), int(rng.integers(64, 420))
    i0, j0, k0 = int(rng.integers(0, 200)), int(rng.integers(0, 40)), int(rng.integers(0, 100))
    i1, j1, k1 = int(rng.integers(M - 200, M + 1)), int(rng.integers(N - 30, N + 1)), int(rng.integers(K - 80, K + 1))
    at = bool(rng.random() < 0.2)
    bcm = bool(rng.random() < 0.2)
    r_zero = bool(rng.random() < 0.4)
    A, B, t, d = make_inputs(body, M, K, N, "int", seed=7100 + case)
    R0 = np.zeros((M, N)) if r_zero else rng.integers(-50, 50, (M, N)).astype(np.float64)
    b = (i0, i1, j0, j1, k0, k1)
    if r_zero:  # R starts at zero: only the bounds rows are zero-filled, so the bounds cover whole rows
        b = (i0, i1, 0, N, k0, k1)
    want = oracle(body, A, B, t, d, R0=R0, bounds=b)
    npd = NP_DT[dtype]
    Ab = np.ascontiguousarray(A.T if at else A).astype(npd)
    Bb = (np.asfortranarray(B) if bcm else np.ascontiguousarray(B)).astype(npd)
    R = R0.astype(npd).copy()
    if case % 2 == 1:  # pinned R: the zero-copy result path where it applies
        R = _pinned(R)
    plan = gpu_ctx.plan(body, dtype, layout_a=int(at))
    ops = P.Operands(Ab, Bb, R, None if t is None else t.astype(npd), None if d is None else d.astype(npd))
    if case % 3 == 0:
        gpu_ctx.clear_tuning_cache()
        P.run_host_adaptive(plan, ops, P.Bounds(*b), r_zero=r_zero)
    else:
        P.run_host(plan, ops, P.Bounds(*b), r_zero=r_zero)
    got = (R if isinstance(R, np.ndarray) else R.numpy()).astype(np.float64)
    bad = np.argwhere(got != want)
    assert bad.size == 0, (f"case {case}: {body}/{dtype} {M}x{K}x{N} bounds {b} at={at} bcm={bcm} "
                           f"r_zero={r_zero}: {len(bad)} mismatches, first {tuple(bad[0])} got "
                           f"{got[tuple(bad[0])]} want {want[tuple(bad[0])]}")
