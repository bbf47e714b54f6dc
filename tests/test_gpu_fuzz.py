"""GPU: randomized parity sweep over the fixed bodies.

Each case draws a body, dtype, shape (tiny and ragged included), a bounds
sub-rectangle of a larger R holding prior values, operand orientations and
storage orders, the threshold form, '=' or '+=', and how the task runs
(tuned, a named tile variant, a forced split-K depth, the host-buffer
entry, AMULET's tuner contract, or the per-element executor), on the reference's IntValued data so that every case must be
bit-exact against the C oracle (and R outside the bounds untouched).
"""
from __future__ import annotations

import numpy as np
import pytest

from tests.helpers import NP_DT, oracle

pytestmark = pytest.mark.gpu

BODIES = [("gemm", "f64"), ("gemm", "f32"), ("discount", "f64"), ("discount", "f32"),
          ("boost", "f64"), ("boost", "f32"), ("sqdiff", "f64"), ("sqdiff", "f32"),
          ("eqcount", "f64"), ("eqcount", "i32"), ("thrcount", "f64"), ("thrcount", "i32")]


def stored(x, transposed, col_major):
    """The buffer holding the statement operand x (logical rows x cols)."""
    buf = x.T if transposed else x
    return np.asfortranarray(buf) if col_major else np.ascontiguousarray(buf)


@pytest.mark.parametrize("case", range(192))
def test_random_cases_bit_exact(gpu_ctx, case):
    import torch

    import paper_2305_08872_b200 as P

    rng = np.random.default_rng(1000 + case)
    body, dtype = BODIES[case % len(BODIES)]
    M, K, N = (int(rng.integers(1, 200)), int(rng.integers(1, 160)), int(rng.integers(1, 220)))
    if case % 5 == 0:
        M, K, N = int(rng.integers(200, 700)), int(rng.integers(100, 600)), int(rng.integers(200, 700))
    i0, j0, k0 = (int(rng.integers(0, max(1, M // 3))), int(rng.integers(0, max(1, N // 3))),
                  int(rng.integers(0, max(1, K // 3))))
    i1, j1, k1 = (int(rng.integers(i0 + 1, M + 1)), int(rng.integers(j0 + 1, N + 1)),
                  int(rng.integers(k0 + 1, K + 1)))
    at, bt = bool(rng.integers(0, 2)), bool(rng.integers(0, 2))
    acm, bcm = bool(rng.integers(0, 2)), bool(rng.integers(0, 2))
    accumulate = rng.random() < 0.8
    tcls = "j"
    if body in ("discount", "boost", "thrcount"):
        tcls = str(rng.choice(["c", "i", "j", "ij"]))
    A = rng.integers(-8, 9, (M, K)).astype(np.float64)
    B = rng.integers(-8, 9, (K, N)).astype(np.float64)
    if body == "eqcount":
        A, B = np.abs(A) % 5, np.abs(B) % 5  # collisions likely
    R0 = rng.integers(-50, 50, (M, N)).astype(np.float64)
    tval = float(rng.integers(-8, 9))
    thres = {"c": None, "i": rng.integers(-8, 9, M).astype(np.float64),
             "j": rng.integers(-8, 9, N).astype(np.float64),
             "ij": rng.integers(-8, 9, (M, N)).astype(np.float64)}[tcls] \
        if body in ("discount", "boost", "thrcount") else None
    dis = rng.integers(-8, 9, N).astype(np.float64) if body == "discount" else None

    # oracle: thresholds as an (i, j) grid, one row at a time (its threshold
    # vector runs over j)
    b = (i0, i1, j0, j1, k0, k1)
    if body in ("discount", "boost", "thrcount"):
        T = {"c": np.full((M, N), tval), "i": None, "j": None, "ij": thres}[tcls]
        if tcls == "i":
            T = np.repeat(thres[:, None], N, 1)
        elif tcls == "j":
            T = np.repeat(thres[None, :], M, 0)
        want = R0.copy()
        for i in range(i0, i1):
            want[i] = oracle(body, A[i:i + 1], B, T[i], dis, R0=R0[i:i + 1],
                             bounds=(0, 1, j0, j1, k0, k1), accumulate=accumulate)[0]
    else:
        want = oracle(body, A, B, None, None, R0=R0, bounds=b, accumulate=accumulate)

    td = {"f64": torch.float64, "f32": torch.float32, "i32": torch.int32}[dtype]
    npd = NP_DT[dtype]
    dev = lambda x: None if x is None else torch.from_numpy(  # noqa: E731
        np.asarray(x.astype(npd), order="K")).to("cuda")
    Ab = stored(A, at, acm).astype(npd, order="K")
    Bb = stored(B, bt, bcm).astype(npd, order="K")
    plan = gpu_ctx.plan(body, dtype, accumulate=accumulate, layout_a=int(at), layout_b=int(bt),
                        thres_class=tcls, thres_value=tval)
    mode = case % 6
    if mode == 3:  # host-buffer entry
        R = R0.astype(npd).copy()
        ops = P.Operands(Ab, Bb, R, None if thres is None else thres.astype(npd),
                         None if dis is None else dis.astype(npd))
        P.run_host(plan, ops, P.Bounds(*b))
        got = R.astype(np.float64)
    else:
        R = dev(R0)
        At = torch.from_numpy(Ab).to("cuda") if Ab.flags.c_contiguous else \
            torch.from_numpy(np.ascontiguousarray(Ab.T)).to("cuda").t()
        Bt = torch.from_numpy(Bb).to("cuda") if Bb.flags.c_contiguous else \
            torch.from_numpy(np.ascontiguousarray(Bb.T)).to("cuda").t()
        ops = P.Operands(At, Bt, R, dev(thres), dev(dis))
        if mode == 0:
            P.adaptive_execute(plan, ops, P.Bounds(*b))
        elif mode == 4:  # AMULET's own tuner contract over the GPU executor
            P.engine.adaptive_execute_amulet(plan, ops, P.Bounds(*b))
        elif mode == 5:  # the per-element executor
            P.run_naive(plan, ops, P.Bounds(*b))
        elif mode == 1:
            vs = plan.variants()
            vi = int(rng.integers(0, len(vs)))
            try:
                P.run_subtask(plan, ops, P.TileParams(variant=vi), P.Bounds(*b))
            except P.EngineError:  # an aligned variant on unaligned operands: the planner's pick
                P.run_subtask(plan, ops, P.TileParams(), P.Bounds(*b))
        else:
            P.run_subtask(plan, ops, P.TileParams(kc=int(rng.integers(1, max(2, k1 - k0 + 1)))),
                          P.Bounds(*b))
        got = R.cpu().numpy().astype(np.float64)
    bad = np.argwhere(got != want)
    assert bad.size == 0, (f"case {case}: {body}/{dtype} {M}x{K}x{N} bounds {b} at={at} bt={bt} "
                           f"acm={acm} bcm={bcm} acc={accumulate} thres={tcls} mode={mode}: "
                           f"{len(bad)} mismatches, first {tuple(bad[0])} got "
                           f"{got[tuple(bad[0])]} want {want[tuple(bad[0])]}")


@pytest.mark.parametrize("case", range(40))
def test_random_generated_statements_on_subrectangles(gpu_ctx, case):
    """Generated bodies on a bounds sub-rectangle of an R holding prior
    values, with row/col-major storage, against the UNMODIFIED reference's
    execute_scalar_region on the same region (int data: bit-exact)."""
    import random

    import torch

    import paper_2305_08872_b200 as P
    from oracle import pyoracle as po
    from tests.test_gpu_generic import random_statement

    if not po.ref_available():
        pytest.skip("reference engine not built")
    rng = random.Random(5000 + case)
    src = random_statement(rng)
    M, K, N = 3 + rng.randrange(90), 1 + rng.randrange(80), 3 + rng.randrange(110)
    ref = po.RefTask.create(src, M, K, N, seed=case + 3, int_valued=True,
                            order_a=rng.randrange(2), order_b=rng.randrange(2))
    t = P.compile_task(src)
    R0 = np.array([[rng.randrange(-40, 40) for _ in range(N)] for _ in range(M)], dtype=np.float64)
    ref.set(t.result_name, R0)
    i0, j0, k0 = rng.randrange(M // 2 + 1), rng.randrange(N // 2 + 1), rng.randrange(K)
    i1, j1, k1 = rng.randrange(i0 + 1, M + 1), rng.randrange(j0 + 1, N + 1), rng.randrange(k0 + 1, K + 1)
    data = {}
    for name in ref.names():
        x = ref.get(name)  # logical view over the reference's storage order
        data[name] = torch.from_numpy(np.ascontiguousarray(x)).cuda() if x.flags.c_contiguous or \
            x.ndim == 1 else torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()
    data[t.result_name] = torch.from_numpy(R0.copy()).cuda()
    plan = gpu_ctx.plan_for(t, "f64")
    how = case % 3
    bnd = P.Bounds(i0, i1, j0, j1, k0, k1)
    ops = P.operands_of(t, data)
    if how == 0:
        P.adaptive_execute(plan, ops, bnd)
    elif how == 1:
        P.run_subtask(plan, ops, P.TileParams(kc=max(1, (k1 - k0) // 2)), bnd)
    else:
        P.run_naive(plan, ops, bnd)
    ref.run_scalar_region(i0, i1, j0, j1, k0, k1)
    want = ref.get(t.result_name)
    got = data[t.result_name].cpu().numpy()
    bad = np.argwhere(got != want)
    assert bad.size == 0, (f"{src} {M}x{K}x{N} bounds {(i0, i1, j0, j1, k0, k1)} how={how}: "
                           f"{len(bad)} mismatches, first {tuple(bad[0])}: {got[tuple(bad[0])]} "
                           f"vs {want[tuple(bad[0])]}")


@pytest.mark.parametrize("case", range(48))
def test_random_real_data_within_tolerance(gpu_ctx, case):
    """BASELINE distributions (helpers.make_inputs 'baseline') on random shapes
    with K up to 4096 and random entries: fp64 <= 1e-12, fp32 <= 1e-5
    (normwise for GEMM) against the fp64 oracle, int32 exact."""
    import torch

    import paper_2305_08872_b200 as P
    from tests.helpers import cast, check, make_inputs

    rng = np.random.default_rng(7000 + case)
    body, dtype = BODIES[case % len(BODIES)]
    M, N = int(rng.integers(1, 400)), int(rng.integers(1, 400))
    K = int(rng.choice([int(rng.integers(1, 300)), int(rng.integers(300, 4097))]))
    A, B, t, d = make_inputs(body, M, K, N, "baseline", seed=case)
    A, B, t, d = (cast(x, dtype) for x in (A, B, t, d))
    want = oracle(body, A, B, t, d)
    td = {"f64": torch.float64, "f32": torch.float32, "i32": torch.int32}[dtype]
    dev = lambda x: None if x is None else torch.from_numpy(x).to(td).cuda()  # noqa: E731
    R = torch.zeros((M, N), dtype=td, device="cuda")
    plan = gpu_ctx.plan(body, dtype)
    ops = P.Operands(dev(A), dev(B), R, dev(t), dev(d))
    mode = case % 3
    if mode == 0:
        P.adaptive_execute(plan, ops, P.Bounds(0, M, 0, N, 0, K))
    elif mode == 1:
        vs = plan.variants()
        vi = int(rng.integers(0, len(vs)))
        try:
            P.run_subtask(plan, ops, P.TileParams(variant=vi), P.Bounds(0, M, 0, N, 0, K))
        except P.EngineError:
            P.run_subtask(plan, ops, P.TileParams(), P.Bounds(0, M, 0, N, 0, K))
    else:
        P.run_subtask(plan, ops, P.TileParams(kc=int(rng.integers(32, max(33, K)))),
                      P.Bounds(0, M, 0, N, 0, K))
    check(body, dtype, R.cpu().numpy(), want, A=A, B=B,
          what=f"case {case} {body}/{dtype} {M}x{K}x{N} mode {mode}")


@pytest.mark.parametrize("case", range(36))
def test_random_degenerate_and_banded(gpu_ctx, case):
    """Bounds that may be empty in any dimension or a single row / column /
    k, and tall tasks (M >= 1024) that take the host pipeline's row bands
    (pinned R: zero-copy; pageable R: staged), through every entry; bit-exact
    on IntValued data, R outside the bounds untouched."""
    import torch

    import paper_2305_08872_b200 as P

    rng = np.random.default_rng(7000 + case)
    body, dtype = [("discount", "f64"), ("gemm", "f64"), ("eqcount", "i32"), ("boost", "f32"),
                   ("sqdiff", "f32"), ("gemm", "f32")][case % 6]
    tall = case % 3 == 0
    M = int(rng.integers(1024, 1600)) if tall else int(rng.integers(1, 120))
    K, N = int(rng.integers(1, 300)), int(rng.integers(1, 200))

    def extent(n):
        a = int(rng.integers(0, n + 1))
        kind = rng.integers(0, 4)
        b = a if kind == 0 else min(n, a + 1) if kind == 1 else int(rng.integers(a, n + 1))
        return a, b

    (i0, i1), (j0, j1), (k0, k1) = extent(M), extent(N), extent(K)
    if tall:
        i0, i1 = 0, M  # the whole tall band (the banded pipeline needs M >= 1024 rows)
    A = rng.integers(-8, 9, (M, K)).astype(np.float64)
    B = rng.integers(-8, 9, (K, N)).astype(np.float64)
    if body == "eqcount":
        A, B = np.abs(A) % 5, np.abs(B) % 5
    thres = rng.integers(-8, 9, N).astype(np.float64) if body in ("discount", "boost") else None
    dis = rng.integers(-8, 9, N).astype(np.float64) if body == "discount" else None
    R0 = rng.integers(-50, 50, (M, N)).astype(np.float64)
    b = (i0, i1, j0, j1, k0, k1)
    want = oracle(body, A, B, thres, dis, R0=R0, bounds=b)
    npd = NP_DT[dtype]
    plan = gpu_ctx.plan(body, dtype)
    mode = int(rng.integers(0, 6))
    host = mode >= 4 or tall and mode >= 2
    if host:
        pinned = mode != 5
        cv = (lambda x: None if x is None else torch.from_numpy(x.astype(npd)).pin_memory()) if pinned else \
            (lambda x: None if x is None else torch.from_numpy(x.astype(npd)))
        R = cv(R0)
        ops = P.Operands(cv(A), cv(B), R, cv(thres), cv(dis))
        if mode % 2:
            P.run_host_adaptive(plan, ops, P.Bounds(*b))
        else:
            P.run_host(plan, ops, P.Bounds(*b))
        got = R.numpy().astype(np.float64)
    else:
        dv = lambda x: None if x is None else torch.from_numpy(x.astype(npd)).cuda()  # noqa: E731
        R = dv(R0)
        ops = P.Operands(dv(A), dv(B), R, dv(thres), dv(dis))
        if mode == 0:
            P.adaptive_execute(plan, ops, P.Bounds(*b))
        elif mode == 1:
            P.run_naive(plan, ops, P.Bounds(*b))
        elif mode == 2:
            P.run_subtask(plan, ops, P.TileParams(kc=int(rng.integers(1, 200))), P.Bounds(*b))
        else:
            P.run_subtask(plan, ops, P.TileParams(), P.Bounds(*b))
        got = R.cpu().numpy().astype(np.float64)
    bad = np.argwhere(got != want)
    assert bad.size == 0, (f"case {case}: {body}/{dtype} {M}x{K}x{N} bounds {b} mode={mode}: "
                           f"{len(bad)} mismatches, first {tuple(bad[0])} got {got[tuple(bad[0])]} "
                           f"want {want[tuple(bad[0])]}")
