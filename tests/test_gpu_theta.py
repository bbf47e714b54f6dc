"""GPU: the theta-form discount variants (csrc/theta_discount.cu).

The mask p > t is evaluated as a > theta(k, j) with theta prepared on the B
side, so these tests aim at exactly the places that form can go wrong:
thresholds sitting on products (ties) and one ulp either side of them,
negative and zero b, c1 = 0 / negative, K tails and sub-rectangles, and the
guard that hands non-finite or out-of-range operands to the ordinary discount
kernel (whose result must then be bit-identical to that kernel's).
"""
from __future__ import annotations

import numpy as np
import pytest

from tests.helpers import check, int_valued, oracle

pytestmark = pytest.mark.gpu


def theta_variants(plan):
    return [(vi, v.name) for vi, v in enumerate(plan.variants()) if "_theta_" in v.name]


def ordinary(plan):
    """The shipped ordinary discount tile (32 x 128, 4 x 4 per thread)."""
    return [v.name for v in plan.variants()].index("discount_f64_32x128_t4x4_w8x1")


def run(ctx, A, B, t, d, vi, R0=None, bounds=None, tcls="j", tval=0.0):
    import torch

    import paper_2305_08872_b200 as P

    M, N = A.shape[0], B.shape[1]
    plan = ctx.plan("discount", "f64", thres_class=tcls, thres_value=tval)
    dev = lambda x: None if x is None else torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    R = dev(np.zeros((M, N)) if R0 is None else R0.copy())
    ops = P.Operands(dev(A), dev(B), R, dev(t), dev(d))
    b = P.Bounds(*bounds) if bounds else P.Bounds(0, M, 0, N, 0, A.shape[1])
    P.run_subtask(plan, ops, P.TileParams(variant=vi), b)
    return R.cpu().numpy()


# (the theta variants stage A by TMA: K and N even, as for every TMA variant)


def test_theta_variants_registered(gpu_ctx):
    plan = gpu_ctx.plan("discount", "f64")
    assert len(theta_variants(plan)) >= 2
    # per-output thresholds (T indexed by i or (i, j)) never get the theta form
    for cls in ("i", "ij"):
        assert not theta_variants(gpu_ctx.plan("discount", "f64", thres_class=cls))


@pytest.mark.parametrize("seed", range(6))
def test_int_valued_bit_exact_with_ties(gpu_ctx, seed):
    """IntValued data: products land exactly on thresholds often; every term
    and sum is exact, so the theta form must match the oracle bit for bit."""
    rng = np.random.default_rng(seed)
    M, K, N = [(64, 64, 64), (96, 130, 160), (257, 130, 66), (13, 18, 6), (200, 334, 258), (33, 8, 130)][seed]
    A, B = int_valued(rng, (M, K)), int_valued(rng, (K, N))
    t = int_valued(rng, N)
    d = rng.integers(-3, 4, N).astype(np.float64)  # c1 = 1 - d: 0, negative and > 1 included
    R0 = rng.integers(-50, 50, (M, N)).astype(np.float64)
    plan = gpu_ctx.plan("discount", "f64")
    for vi, name in theta_variants(plan):
        want = oracle("discount", A, B, t, d, R0=R0)
        got = run(gpu_ctx, A, B, t, d, vi, R0=R0)
        check("discount", "f64", got, want, exact=True, what=f"{name} {M}x{K}x{N}")


def test_constant_threshold_and_subrectangle(gpu_ctx):
    import paper_2305_08872_b200 as P  # noqa: F401

    rng = np.random.default_rng(11)
    M, K, N = 150, 170, 190
    A, B = int_valued(rng, (M, K)), int_valued(rng, (K, N))
    d = int_valued(rng, N)
    R0 = rng.integers(-50, 50, (M, N)).astype(np.float64)
    bounds = (5, 140, 8, 180, 2, 161)
    plan = gpu_ctx.plan("discount", "f64", thres_class="c", thres_value=3.0)
    for vi, name in theta_variants(plan):
        want = oracle("discount", A, B, np.full(N, 3.0), d, R0=R0, bounds=bounds)
        got = run(gpu_ctx, A, B, None, d, vi, R0=R0, bounds=bounds, tcls="c", tval=3.0)
        check("discount", "f64", got, want, exact=True, what=f"{name} const-t bounds {bounds}")


@pytest.mark.parametrize("seed", range(4))
def test_real_thresholds_on_products(gpu_ctx, seed):
    """Real data with every threshold equal to an actual product rn(a b) or
    one ulp either side of it: a mask error costs (1 - c1) p, far above the
    1e-12 tolerance, so theta must be exact at the boundary."""
    rng = np.random.default_rng(100 + seed)
    M, K, N = 96, 200, 130
    A = rng.uniform(-3, 3, (M, K))
    B = rng.uniform(-3, 3, (K, N))
    B[rng.random((K, N)) < 0.05] = 0.0
    ii, kk = rng.integers(0, M, N), rng.integers(0, K, N)
    t = A[ii, kk] * B[kk, np.arange(N)]
    shift = rng.integers(-1, 2, N)
    t = np.where(shift < 0, np.nextafter(t, -np.inf), np.where(shift > 0, np.nextafter(t, np.inf), t))
    d = rng.uniform(0, 0.5, N)
    plan = gpu_ctx.plan("discount", "f64")
    want = oracle("discount", A, B, t, d)
    base = run(gpu_ctx, A, B, t, d, ordinary(plan))
    # mixed signs cancel, so the bound is normwise:
    # |err| <= 1e-12 * sum_k |term_k|
    scale = np.abs(A) @ np.abs(B) * np.maximum(1.0, np.abs(1.0 - d))[None, :]
    for vi, name in theta_variants(plan):
        got = run(gpu_ctx, A, B, t, d, vi)
        for ref, what in ((want, "oracle"), (base, "ordinary kernel")):
            worst = float((np.abs(got - ref) / scale).max())
            assert worst <= 1e-12, f"{name} seed {seed} vs {what}: normwise {worst:.3e}"


def test_baseline_distribution_within_tolerance(gpu_ctx):
    from tests.helpers import make_inputs

    A, B, t, d = make_inputs("discount", 300, 1000, 260, "baseline", seed=5)
    want = oracle("discount", A, B, t, d)
    plan = gpu_ctx.plan("discount", "f64")
    for vi, name in theta_variants(plan):
        check("discount", "f64", run(gpu_ctx, A, B, t, d, vi), want, what=name)


@pytest.mark.parametrize("case", ["inf_b", "nan_t", "huge", "tiny", "inf_dis"])
def test_guard_hands_over_to_ordinary_kernel(gpu_ctx, case):
    """Operands the theta form cannot reproduce: the guard must route the whole
    launch to the ordinary discount kernel, bit-identical to it."""
    rng = np.random.default_rng(7)
    M, K, N = 70, 90, 66
    A, B = int_valued(rng, (M, K)), int_valued(rng, (K, N))
    t, d = int_valued(rng, N), rng.uniform(0, 0.5, N)
    if case == "inf_b":
        B[3, 5] = np.inf
    elif case == "nan_t":
        t[4] = np.nan
    elif case == "huge":
        A[2, 2], B[2, 7] = 1e200, 1e150
    elif case == "tiny":
        A[1, 1], B[1, 3] = 1e-200, 1e-150
    else:
        d[0] = -np.inf
    plan = gpu_ctx.plan("discount", "f64")
    base = run(gpu_ctx, A, B, t, d, ordinary(plan))
    for vi, name in theta_variants(plan):
        got = run(gpu_ctx, A, B, t, d, vi)
        np.testing.assert_array_equal(got, base, err_msg=f"{name} {case}")


def test_nonfinite_a_in_theta_form(gpu_ctx):
    """inf / NaN in A stay on the theta path; on IntValued data the result must
    equal the ordinary kernel's exactly, inf signs and NaN positions included
    (both evaluate p * (p > t ? c1 : 1); the finite entries also equal the
    oracle).

    Stated divergence: for a term whose product is infinite the
    fused kernels accumulate the IEEE value p * c (+-inf, or NaN for 0 * inf),
    while the reference's mask arithmetic ((m*A)*B)*dis multiplies 0 or 1 by
    inf and yields NaN. Every such output is non-finite on both sides, at the
    same positions; the values (+-inf vs NaN) may differ."""
    rng = np.random.default_rng(9)
    M, K, N = 40, 64, 34
    A, B = int_valued(rng, (M, K)), int_valued(rng, (K, N))
    t, d = int_valued(rng, N), rng.integers(-2, 3, N).astype(np.float64)
    A[3, 10], A[7, 20], A[11, 30] = np.inf, -np.inf, np.nan
    want = oracle("discount", A, B, t, d)
    plan = gpu_ctx.plan("discount", "f64")
    base = run(gpu_ctx, A, B, t, d, ordinary(plan))
    fin = np.isfinite(base)
    np.testing.assert_array_equal(fin, np.isfinite(want))  # non-finite at the same positions
    assert (~fin).any()
    np.testing.assert_array_equal(base[fin], want[fin])
    for vi, name in theta_variants(plan):
        got = run(gpu_ctx, A, B, t, d, vi)
        np.testing.assert_array_equal(got, base, err_msg=name)


def test_theta_skipped_when_planes_do_not_fit():
    """The tuner leaves out variants whose prepared operands would not fit in
    free HBM (here 1.6 GB of theta planes with ~1.5 GB free) instead of
    failing the call on cudaMalloc."""
    import torch

    import paper_2305_08872_b200 as P

    M, K, N = 2048, 4096, 16384
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randint(0, 10, (M, K), device="cuda", generator=g).double()
    B = torch.rand((K, N), device="cuda", dtype=torch.float64, generator=g) * 99 + 1
    t = torch.rand(N, device="cuda", dtype=torch.float64, generator=g) * 400 + 50
    d = torch.rand(N, device="cuda", dtype=torch.float64, generator=g) * 0.3
    R = torch.zeros((M, N), device="cuda", dtype=torch.float64)
    ctx = P.Context(0)
    plan = ctx.plan("discount", "f64")
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    hog = torch.empty(max(0, free - (1536 << 20)), dtype=torch.uint8, device="cuda")
    try:
        rep = P.adaptive_execute(plan, P.Operands(A, B, R, t, d), P.Bounds(0, M, 0, N, 0, K))
    finally:
        del hog
        torch.cuda.empty_cache()
    names = [plan.variants()[tr.value].name for tr in rep.trials]
    assert names and not any("_theta_" in n for n in names), names
    rows = [0, 777, M - 1]
    want = oracle("discount", A[rows].cpu().numpy(), B.cpu().numpy(), t.cpu().numpy(), d.cpu().numpy())
    check("discount", "f64", R[rows].cpu().numpy(), want, what="fallback tiles under memory pressure")


@pytest.mark.parametrize("kc", [128, 320, 512])
def test_theta_split_k_bit_exact(gpu_ctx, kc):
    """K segments for the theta tiles: partials per segment,
    reduced in segment order; exact on data whose products and sums are
    exact (A integers 0..9, integer B and thresholds, dis a multiple of 1/4),
    including a K tail, a prior-valued R and a sub-rectangle."""
    import torch

    import paper_2305_08872_b200 as P

    rng = np.random.default_rng(kc)
    M, K, N = 300, 1000, 260
    A = rng.integers(0, 10, (M, K)).astype(np.float64)
    B = rng.integers(1, 100, (K, N)).astype(np.float64)
    t = rng.integers(50, 450, N).astype(np.float64)
    d = rng.integers(0, 2, N) * 0.25
    R0 = rng.integers(-8, 9, (M, N)).astype(np.float64)
    plan = gpu_ctx.plan("discount", "f64")
    b = (5, 290, 2, 258, 64, 1000)
    want = oracle("discount", A, B, t, d, R0=R0, bounds=b)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    for vi, name in theta_variants(plan):
        R = dev(R0)
        log = P.ExecLog(capacity=8)
        P.run_subtask(plan, P.Operands(dev(A), dev(B), R, dev(t), dev(d)), P.TileParams(kc=kc, variant=vi),
                      P.Bounds(*b), log=log)
        assert log.records[0].splits == (936 + (kc + 15) // 16 * 16 - 1) // ((kc + 15) // 16 * 16)
        check("discount", "f64", R.cpu().numpy(), want, exact=True, what=f"{name} kc={kc}")


def test_config0_tunes_theta_with_k_segments(gpu_ctx):
    """Config 0 (1024^3): the tuner's candidates include the theta tiles with
    K segments, and whatever wins is within 1e-12 of the oracle."""
    import torch

    import paper_2305_08872_b200 as P
    from tests.helpers import make_inputs

    M = K = N = 1024
    A, B, t, d = make_inputs("discount", M, K, N, "baseline", seed=81)
    want = oracle("discount", A, B, t, d)
    plan = gpu_ctx.plan("discount", "f64")
    gpu_ctx.clear_tuning_cache()
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    R = dev(np.zeros((M, N)))
    rep = P.adaptive_execute(plan, P.Operands(dev(A), dev(B), R, dev(t), dev(d)), P.Bounds(0, M, 0, N, 0, K))
    names = [v.name for v in plan.variants()]
    tried = {(names[tr.value], tr.rows) for tr in rep.trials}
    assert any("_theta_" in n for n, _ in tried)
    assert rep.scratch_tuned and len(rep.trials) > len({n for n, _ in tried})  # split-K forms tried too
    check("discount", "f64", R.cpu().numpy(), want, what="config 0 tuned")


def test_scratch_trials_are_charged(gpu_ctx):
    """Whole-task trials on the scratch R are work the real task repeats: the
    report charges them (tuning_seconds, inside total_seconds) and counts no
    output rows for them (tuning_fraction 0)."""
    import torch

    import paper_2305_08872_b200 as P
    from tests.helpers import make_inputs

    M = K = N = 512
    A, B, t, d = make_inputs("discount", M, K, N, "baseline", seed=82)
    plan = gpu_ctx.plan("discount", "f64")
    gpu_ctx.clear_tuning_cache()
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    R = dev(np.zeros((M, N)))
    rep = P.adaptive_execute(plan, P.Operands(dev(A), dev(B), R, dev(t), dev(d)), P.Bounds(0, M, 0, N, 0, K))
    assert rep.scratch_tuned and rep.tuning_fraction == 0.0
    trials = sum(tr.elapsed for tr in rep.trials)
    # each candidate runs twice (five times for sub-millisecond tasks, as
    # here), the fastest scored; every run is charged
    assert trials <= rep.tuning_seconds <= 6.0 * trials
    assert rep.total_seconds > rep.tuning_seconds
