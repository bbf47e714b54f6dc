"""GPU parity: the sm_100a kernels through the C-ABI vs the CPU oracle.

Integer-valued data (the reference's own determinism convention,
test_support / acceptance.cpp:109-132): bit-exact for every body, dtype and
tile variant, on the acceptance dims including ragged ones. BASELINE
distributions: within BASELINE's tolerances (fp64 1e-12, fp32 1e-5 relative
vs the fp64 oracle; normwise for GEMM), int32 bit-exact.
"""
from __future__ import annotations

import numpy as np
import pytest

from tests.helpers import ACCEPT_DIMS, NP_DT, cast, check, make_inputs, oracle

pytestmark = pytest.mark.gpu

BODY_DTYPES = [("gemm", "f64"), ("gemm", "f32"), ("discount", "f64"), ("discount", "f32"),
               ("boost", "f64"), ("boost", "f32"), ("sqdiff", "f64"), ("sqdiff", "f32"),
               ("eqcount", "f64"), ("eqcount", "f32"), ("eqcount", "i32"),
               ("thrcount", "f64"), ("thrcount", "f32"), ("thrcount", "i32")]


def dev(x, dtype):
    import torch

    if x is None:
        return None
    return torch.from_numpy(np.ascontiguousarray(x.astype(NP_DT[dtype]))).cuda()


def run_gpu(ctx, body, dtype, A, B, thres=None, dis=None, R0=None, bounds=None, tile=None,
            adaptive=False, thres_class="j", thres_value=0.0):
    import paper_2305_08872_b200 as P

    M, N, K = A.shape[0], B.shape[1], A.shape[1]
    plan = ctx.plan(body, dtype, thres_class=thres_class, thres_value=thres_value)
    R = dev(np.zeros((M, N)) if R0 is None else R0, dtype)
    ops = P.Operands(dev(A, dtype), dev(B, dtype), R, dev(thres, dtype), dev(dis, dtype))
    b = P.Bounds(*bounds) if bounds else P.Bounds(0, M, 0, N, 0, K)
    if adaptive:
        rep = P.adaptive_execute(plan, ops, b)
        return R.cpu().numpy(), rep
    P.run_subtask(plan, ops, tile or P.TileParams(), b)
    return R.cpu().numpy(), None


@pytest.mark.parametrize("body,dtype", BODY_DTYPES)
def test_int_valued_all_variants_bit_exact(gpu_ctx, body, dtype):
    import paper_2305_08872_b200 as P

    plan = gpu_ctx.plan(body, dtype)
    for vi, v in enumerate(plan.variants()):
        for (M, K, N) in ACCEPT_DIMS:
            vn = 2 if dtype == "f64" else 4
            if not v.name.endswith("_u") and (K % vn or N % vn):
                continue  # 16-byte staging needs vector-multiple strides
            A, B, t, d = make_inputs(body, M, K, N, "int", seed=M * 7 + K)
            want = oracle(body, A, B, t, d)
            tile = P.TileParams(variant=vi)  # the unaligned variant runs on aligned data too
            got, _ = run_gpu(gpu_ctx, body, dtype, A, B, t, d, tile=tile)
            check(body, dtype, got, want, exact=True, what=f"{v.name} {M}x{K}x{N}")


@pytest.mark.parametrize("body,dtype", BODY_DTYPES)
def test_reference_goldens(gpu_ctx, body, dtype):
    """Against outputs of the UNMODIFIED reference (run_naive on its own
    seeded IntValued data), committed under tests/golden/."""
    from tests.golden.load import load_golden

    for case in load_golden(body):
        A, B, t, d, want = case["A"], case["B"], case.get("thres"), case.get("dis"), case["R"]
        tcls, tval = ("c", case["thres_const"]) if "thres_const" in case else ("j", 0.0)
        got, _ = run_gpu(gpu_ctx, body, dtype, A, B, t, d, adaptive=True, thres_class=tcls,
                         thres_value=tval)
        check(body, dtype, got, want, exact=True, what=f"golden {case['name']}")


@pytest.mark.parametrize("body,dtype", [("discount", "f64"), ("boost", "f64"), ("boost", "f32"),
                                        ("gemm", "f64"), ("gemm", "f32"), ("sqdiff", "f32"),
                                        ("eqcount", "i32"), ("discount", "f32"),
                                        ("thrcount", "f64")])
def test_baseline_distributions_tolerance(gpu_ctx, body, dtype):
    M, K, N = 384, 1000, 320
    A, B, t, d = make_inputs(body, M, K, N, "baseline", seed=11)
    A, B, t, d = (cast(x, dtype) for x in (A, B, t, d))
    want = oracle(body, A, B, t, d)
    got, _ = run_gpu(gpu_ctx, body, dtype, A, B, t, d, adaptive=True)
    check(body, dtype, got, want, A=A, B=B, what=f"{body}/{dtype} baseline dist")


def test_config0_discount_full(gpu_ctx):
    """Config 0 in full: discount fp64 1024^3, BASELINE distributions."""
    A, B, t, d = make_inputs("discount", 1024, 1024, 1024, "baseline", seed=1)
    want = oracle("discount", A, B, t, d)
    got, rep = run_gpu(gpu_ctx, "discount", "f64", A, B, t, d, adaptive=True)
    check("discount", "f64", got, want, what="config 0")


@pytest.mark.parametrize("body,dtype,M,K,N", [
    ("boost", "f32", 4096, 4096, 4096), ("boost", "f64", 4096, 4096, 4096),
    ("gemm", "f64", 2048, 8192, 2048), ("gemm", "f32", 2048, 8192, 2048),
    ("sqdiff", "f32", 65536, 1024, 256), ("eqcount", "i32", 65536, 1024, 256)])
def test_large_configs_sampled_rows(gpu_ctx, body, dtype, M, K, N):
    """BASELINE-size shapes; the oracle checks sampled rows (rows of R are
    independent, so the oracle on those rows of A is exact for them)."""
    A, B, t, d = make_inputs(body, M, K, N, "baseline", seed=5)
    A, B, t, d = (cast(x, dtype) for x in (A, B, t, d))
    got, rep = run_gpu(gpu_ctx, body, dtype, A, B, t, d, adaptive=True)
    rows = np.unique(np.r_[0, M - 1, np.random.default_rng(2).integers(0, M, 14)])
    want = oracle(body, A[rows], B, t, d)
    check(body, dtype, got[rows], want, A=A[rows], B=B, what=f"{body}/{dtype} {M}x{K}x{N}")


@pytest.mark.parametrize("body,dtype", [("discount", "f64"), ("boost", "f32"), ("eqcount", "i32"),
                                        ("gemm", "f64")])
def test_split_k_and_nc(gpu_ctx, body, dtype):
    import paper_2305_08872_b200 as P

    M, K, N = 300, 777, 200
    A, B, t, d = make_inputs(body, M, K, N, "int", seed=3)
    want = oracle(body, A, B, t, d)
    for kc in (64, 100, 256, 777, 5000):
        for nc in (0, 64, 128, 1000):
            got, _ = run_gpu(gpu_ctx, body, dtype, A, B, t, d, tile=P.TileParams(kc=kc, nc=nc))
            check(body, dtype, got, want, exact=True, what=f"kc={kc} nc={nc}")


@pytest.mark.parametrize("body,dtype", [("discount", "f64"), ("sqdiff", "f32"), ("eqcount", "i32")])
def test_subrectangle_isolation(gpu_ctx, body, dtype):
    """Only R inside the bounds changes (test_tiled.cpp:172-188); the rest of
    R keeps its prior values; k outside [k0,k1) never contributes."""
    M, K, N = 90, 70, 110
    A, B, t, d = make_inputs(body, M, K, N, "int", seed=9)
    R0 = np.random.default_rng(4).integers(-50, 50, (M, N)).astype(np.float64)
    for bounds in [(3, 77, 5, 101, 2, 61), (0, 1, 0, 1, 0, 1), (10, 10, 0, N, 0, K),
                   (0, M, 0, N, 30, 30), (5, 9, 7, 8, 0, K)]:
        want = oracle(body, A, B, t, d, R0=R0, bounds=bounds)
        got, _ = run_gpu(gpu_ctx, body, dtype, A, B, t, d, R0=R0, bounds=bounds)
        check(body, dtype, got, want, exact=True, what=f"bounds {bounds}")


@pytest.mark.parametrize("body,dtype", [("discount", "f64"), ("boost", "f32"), ("eqcount", "i32")])
def test_unaligned_operands(gpu_ctx, body, dtype):
    """Odd leading dimensions and odd offsets force the element-wise staging
    variant; results unchanged."""
    import torch

    import paper_2305_08872_b200 as P

    M, K, N = 77, 51, 93
    A, B, t, d = make_inputs(body, M, K, N, "int", seed=21)
    want = oracle(body, A, B, t, d)
    dt = NP_DT[dtype]
    Ab = dev(np.zeros((M, K + 3)), dtype)
    Ab[:, 1:K + 1] = dev(A, dtype)
    Bb = dev(np.zeros((K, N + 1)), dtype)
    Bb[:, :N] = dev(B, dtype)
    R = torch.zeros((M, N), dtype=Ab.dtype, device="cuda")
    plan = gpu_ctx.plan(body, dtype)
    ops = P.Operands(Ab[:, 1:K + 1], Bb[:, :N], R, dev(t, dtype), dev(d, dtype))
    P.run_subtask(plan, ops, P.TileParams(), P.Bounds(0, M, 0, N, 0, K))
    check(body, dtype, R.cpu().numpy(), want, exact=True, what="unaligned")
    del dt


@pytest.mark.parametrize("body,dtype", [("discount", "f64"), ("gemm", "f32"), ("eqcount", "i32")])
def test_assignment_last_k_wins(gpu_ctx, body, dtype):
    """`R[i][j] = ...` keeps only the k = k1-1 term (test_exec.cpp:159-171)."""
    import torch

    import paper_2305_08872_b200 as P

    M, K, N = 40, 6, 33
    A, B, t, d = make_inputs(body, M, K, N, "int", seed=13)
    want = oracle(body, A, B, t, d, accumulate=False)
    plan = gpu_ctx.plan(body, dtype, accumulate=False)
    R = torch.zeros((M, N), dtype=dev(A, dtype).dtype, device="cuda")
    P.run_subtask(plan, P.Operands(dev(A, dtype), dev(B, dtype), R, dev(t, dtype), dev(d, dtype)),
                  P.TileParams(), P.Bounds(0, M, 0, N, 0, K))
    check(body, dtype, R.cpu().numpy(), want, exact=True, what="assign")


def test_adaptive_coverage_exactly_once(gpu_ctx):
    import paper_2305_08872_b200 as P

    # thin 1-wave bands: every candidate fits in M / 4; M*N*K above the size
    # that is tuned whole on a scratch R instead
    M, K, N = 32768, 1280, 4096
    A, B, t, d = make_inputs("discount", M, K, N, "int", seed=17)
    want = oracle("discount", A[:64], B, t, d)
    log = P.ExecLog()
    plan = gpu_ctx.plan("discount", "f64")
    R = dev(np.zeros((M, N)), "f64")
    rep = P.adaptive_execute(plan, P.Operands(dev(A, "f64"), dev(B, "f64"), R, dev(t, "f64"),
                                              dev(d, "f64")), P.Bounds(0, M, 0, N, 0, K), log=log)
    assert rep.tuned and len(rep.trials) >= 2
    covered = np.zeros(M, dtype=np.int32)
    for c in rep.coverage:
        assert (c.j0, c.j1, c.k0, c.k1) == (0, N, 0, K)
        covered[c.i0:c.i1] += 1
    assert (covered == 1).all()
    assert len(log.records) == len(rep.coverage)
    # the winner: the best trial, or, when the short first-pass bands were
    # refined with 8-wave bands, the best of those last `refined` trials
    pool = rep.trials[-rep.refined:] if rep.refined else rep.trials
    best = min(pool, key=lambda tr: tr.score)
    assert rep.best_variant == best.value
    got = R.cpu().numpy()
    check("discount", "f64", got[:64], want, exact=True, what="adaptive rows")
    full = oracle("discount", A[-64:], B, t, d)
    check("discount", "f64", got[-64:], full, exact=True, what="adaptive tail rows")


def test_run_host_e2e(gpu_ctx):
    import paper_2305_08872_b200 as P

    M, K, N = 513, 300, 257
    A, B, t, d = make_inputs("discount", M, K, N, "baseline", seed=23)
    want = oracle("discount", A, B, t, d)
    R = np.zeros((M, N))
    plan = gpu_ctx.plan("discount", "f64")
    el = P.run_host(plan, P.Operands(A, B, R, t, d), P.Bounds(0, M, 0, N, 0, K))
    assert el > 0
    check("discount", "f64", R, want, what="run_host")


def test_edge_empty_and_tiny(gpu_ctx):
    for (M, K, N) in [(1, 1, 1), (1, 1000, 1), (2, 3, 1), (1, 2, 300)]:
        for body, dtype in [("discount", "f64"), ("eqcount", "i32"), ("boost", "f32")]:
            A, B, t, d = make_inputs(body, M, K, N, "int", seed=M + N + K)
            want = oracle(body, A, B, t, d)
            got, _ = run_gpu(gpu_ctx, body, dtype, A, B, t, d, adaptive=True)
            check(body, dtype, got, want, exact=True, what=f"tiny {M}x{K}x{N}")


def test_missing_binding_raises(gpu_ctx):
    import paper_2305_08872_b200 as P

    A, B, t, d = make_inputs("discount", 8, 8, 8, "int")
    plan = gpu_ctx.plan("discount", "f64")
    with pytest.raises(P.MissingBinding):
        P.run_subtask(plan, P.Operands(dev(A, "f64"), dev(B, "f64"), dev(np.zeros((8, 8)), "f64"),
                                       dev(t, "f64"), None), P.TileParams(), P.Bounds(0, 8, 0, 8, 0, 8))


@pytest.mark.parametrize("body,dtype", [("discount", "f64"), ("discount", "f32"), ("boost", "f64"),
                                        ("boost", "f32"), ("thrcount", "f64"),
                                        ("thrcount", "i32")])
@pytest.mark.parametrize("form", ["i", "ij", "c"])
def test_threshold_forms_all_variants(gpu_ctx, body, dtype, form):
    """Presets -ti / -tij / -tc (presets.cpp:52-61): thresholds indexed [i],
    [i][j] or a constant, every variant of the plan, ragged dims, bit-exact on
    int-valued data; the constant also as a named 1 x 1 scalar buffer."""
    import paper_2305_08872_b200 as P

    rng = np.random.default_rng(31)
    for (M, K, N) in [(96, 128, 160), (257, 129, 65), (13, 17, 5)]:
        A, B = (rng.integers(-8, 9, s).astype(np.float64) for s in ((M, K), (K, N)))
        dis = rng.integers(-8, 9, N).astype(np.float64) if body == "discount" else None
        if form == "i":
            thres = rng.integers(-8, 9, M).astype(np.float64)
        elif form == "ij":
            thres = rng.integers(-8, 9, (M, N)).astype(np.float64)
        else:
            thres = 3.0
        want = np.zeros((M, N))
        from oracle import pyoracle as po
        po.oracle_run({"discount": po.DISCOUNT, "boost": po.BOOST, "thrcount": po.THRCOUNT}[body],
                      A, B, want, thres=thres, dis=dis, thres_form=form)
        if form == "c":
            for named in (False, True):
                plan = gpu_ctx.plan(body, dtype, thres_class="c", thres_value=0.0 if named else 3.0)
                R = dev(np.zeros((M, N)), dtype)
                tb = dev(np.array([[3.0]]), dtype) if named else None
                P.adaptive_execute(plan, P.Operands(dev(A, dtype), dev(B, dtype), R, tb,
                                                    dev(dis, dtype)), P.Bounds(0, M, 0, N, 0, K))
                check(body, dtype, R.cpu().numpy(), want, exact=True, what=f"tc named={named}")
            continue
        plan = gpu_ctx.plan(body, dtype, thres_class=form)
        vn = 2 if dtype == "f64" else 4
        for vi, v in enumerate(plan.variants()):
            if not v.name.endswith("_u") and (K % vn or N % vn):
                continue
            R = dev(np.zeros((M, N)), dtype)
            P.run_subtask(plan, P.Operands(dev(A, dtype), dev(B, dtype), R, dev(thres, dtype),
                                           dev(dis, dtype)), P.TileParams(variant=vi),
                          P.Bounds(0, M, 0, N, 0, K))
            check(body, dtype, R.cpu().numpy(), want, exact=True, what=f"t{form} {v.name} {M}x{K}x{N}")
        # sub-rectangle: the threshold offsets follow the bounds
        R0 = rng.integers(-5, 5, (M, N)).astype(np.float64)
        bnd = (2, M - 1, 1, N, 3, K)
        want2 = R0.copy()
        po.oracle_run({"discount": po.DISCOUNT, "boost": po.BOOST, "thrcount": po.THRCOUNT}[body],
                      A, B, want2, thres=thres, dis=dis, thres_form=form, bounds=bnd)
        R = dev(R0, dtype)
        P.run_subtask(plan, P.Operands(dev(A, dtype), dev(B, dtype), R, dev(thres, dtype),
                                       dev(dis, dtype)), P.TileParams(), P.Bounds(*bnd))
        check(body, dtype, R.cpu().numpy(), want2, exact=True, what=f"t{form} bounds")


@pytest.mark.parametrize("body,dtype", [("discount", "f64"), ("boost", "f32"), ("gemm", "f64"),
                                        ("eqcount", "i32"), ("sqdiff", "f32")])
def test_orientations_and_storage_orders(gpu_ctx, body, dtype):
    """All four statement orientations (presets -ab/-atb/-abt/-atbt) over
    row- and col-major buffers (test_exec.cpp:109-130), and col-major R: the
    layouts the kernels do not stage directly are packed first, like the
    reference's packing (packing.hpp:11-18)."""
    import torch

    import paper_2305_08872_b200 as P
    from oracle import pyoracle as po

    M, K, N = 97, 61, 83
    A, B, t, d = make_inputs(body, M, K, N, "int", seed=41)
    R0 = np.random.default_rng(8).integers(-9, 9, (M, N)).astype(np.float64)
    bounds = (3, M - 2, 1, N, 2, K - 1)
    want = oracle(body, A, B, t, d, R0=R0, bounds=bounds)

    def buf(x, transposed, colmajor):
        """Buffer whose statement view is x: (x.T if transposed) stored row/col-major."""
        y = x.T if transposed else x
        tt = dev(np.ascontiguousarray(y), dtype)
        if colmajor:
            tt = tt.t().contiguous().t()  # same logical matrix, col-major strides
        return tt

    for at in (0, 1):
        for bt in (0, 1):
            plan = gpu_ctx.plan(body, dtype, layout_a=at, layout_b=bt)
            for acm in (False, True):
                for bcm in (False, True):
                    for rcm in (False, True):
                        Rb = dev(R0, dtype)
                        if rcm:
                            Rb = Rb.t().contiguous().t()
                        ops = P.Operands(buf(A, at, acm), buf(B, bt, bcm), Rb, dev(t, dtype),
                                         dev(d, dtype))
                        P.run_subtask(plan, ops, P.TileParams(), P.Bounds(*bounds))
                        check(body, dtype, Rb.cpu().numpy(), want, exact=True,
                              what=f"at={at} bt={bt} acm={acm} bcm={bcm} rcm={rcm}")
            # adaptive path too (one layout combination per orientation)
            Rb = dev(R0, dtype)
            ops = P.Operands(buf(A, at, True), buf(B, bt, False), Rb, dev(t, dtype), dev(d, dtype))
            P.adaptive_execute(plan, ops, P.Bounds(*bounds))
            check(body, dtype, Rb.cpu().numpy(), want, exact=True, what=f"adaptive at={at} bt={bt}")


@pytest.mark.parametrize("body,dtype", [("discount", "f64"), ("gemm", "f32"), ("eqcount", "i32")])
def test_amulet_tuner_contract_on_gpu(gpu_ctx, body, dtype):
    """AMULET's own tuner (find_kc / find_nc / remainder, autotuner.cpp)
    driving the GPU executor with real timing: the result is exact."""
    import paper_2305_08872_b200 as P

    M, K, N = 150, 700, 900
    A, B, t, d = make_inputs(body, M, K, N, "int", seed=51)
    want = oracle(body, A, B, t, d)
    plan = gpu_ctx.plan(body, dtype)
    R = dev(np.zeros((M, N)), dtype)
    log = P.ExecLog()
    rep = P.engine.adaptive_execute_amulet(
        plan, P.Operands(dev(A, dtype), dev(B, dtype), R, dev(t, dtype), dev(d, dtype)),
        P.Bounds(0, M, 0, N, 0, K), i_h=12, i_w=16, log=log)
    assert rep.tuned and rep.kc_trials and rep.nc_trials
    check(body, dtype, R.cpu().numpy(), want, exact=True, what="amulet tuner")


def test_run_sharded_single_process(gpu_ctx):
    """amlt_gpu_run_sharded: single-process row-band execution from host
    buffers (one band per device; here the box's one device), for A[i][k]
    row-major and A[k][i] col-major; other A layouts are refused."""
    import torch

    import paper_2305_08872_b200 as P

    ndev = torch.cuda.device_count()
    M, K, N = 700, 300, 260
    A, B, t, d = make_inputs("discount", M, K, N, "baseline", seed=61)
    want = oracle("discount", A, B, t, d)
    for at, Abuf in ((0, np.ascontiguousarray(A)), (1, np.asfortranarray(A.T))):
        plan = gpu_ctx.plan("discount", "f64", layout_a=at)
        R = np.zeros((M, N))
        el = P.engine.run_sharded_host(plan, P.Operands(Abuf, B, R, t, d),
                                       P.Bounds(0, M, 0, N, 0, K), list(range(ndev)), r_zero=True)
        assert el > 0
        check("discount", "f64", R, want, what=f"sharded layout_a={at}")
    plan = gpu_ctx.plan("discount", "f64", layout_a=1)
    with pytest.raises(P.UnsupportedExpression):
        P.engine.run_sharded_host(plan, P.Operands(np.ascontiguousarray(A.T), B, np.zeros((M, N)),
                                                   t, d), P.Bounds(0, M, 0, N, 0, K), [0])


@pytest.mark.parametrize("form", ["i", "ij"])
def test_run_sharded_row_indexed_thresholds(gpu_ctx, form):
    """Thresholds indexed by i follow the row split: on a sub-range of rows
    [i0, i1) the device sees thres from row i0 (a row-major [i][j] threshold
    is copied band by band like R)."""
    import paper_2305_08872_b200 as P

    M, K, N = 90, 70, 130
    A, B, _, d = make_inputs("discount", M, K, N, "int", seed=62)
    rng = np.random.default_rng(63)
    t = rng.integers(-8, 9, M if form == "i" else (M, N)).astype(np.float64)
    R0 = rng.integers(-8, 9, (M, N)).astype(np.float64)
    i0, i1 = 13, 77
    tv = np.broadcast_to(t[:, None], (M, N)) if form == "i" else t
    want = R0.copy()
    for i in range(i0, i1):
        p = A[i][:, None] * B  # K x N
        want[i] += (p - (p > tv[i]) * p * d).sum(axis=0)
    plan = gpu_ctx.plan("discount", "f64", thres_class=form)
    R = R0.copy()
    P.engine.run_sharded_host(plan, P.Operands(A, B, R, t, d), P.Bounds(i0, i1, 0, N, 0, K), [0])
    check("discount", "f64", R, want, exact=True, what=f"sharded thres[{form}]")


def test_config4_full_size_sampled_rows(gpu_ctx):
    """BASELINE config 4 at full size (32768 x 32768 x 8192 discount f64, the
    bench workload): inputs generated on the device with its distributions,
    the tuned run over the whole task, then the oracle on sampled rows
    (including the first and last row of every 8-way shard band) x sampled
    columns (including the first and last)."""
    import torch

    import paper_2305_08872_b200 as P

    M, K, N = 32768, 8192, 32768
    g = torch.Generator(device="cuda").manual_seed(11)
    A = torch.randint(0, 10, (M, K), device="cuda", generator=g).double()
    B = torch.rand((K, N), device="cuda", dtype=torch.float64, generator=g) * 99 + 1
    t = torch.rand(N, device="cuda", dtype=torch.float64, generator=g) * 400 + 50
    d = torch.rand(N, device="cuda", dtype=torch.float64, generator=g) * 0.3
    R = torch.zeros((M, N), device="cuda", dtype=torch.float64)
    plan = gpu_ctx.plan("discount", "f64")
    rep = P.adaptive_execute(plan, P.Operands(A, B, R, t, d), P.Bounds(0, M, 0, N, 0, K))
    assert sum((c.i1 - c.i0) for c in rep.coverage) == M
    bands = [M * r // 8 for r in range(9)]
    rows = sorted(set([b for b in bands[:-1]] + [b - 1 for b in bands[1:]]
                      + list(np.random.default_rng(4).integers(0, M, 8))))
    cols = sorted(set([0, N - 1] + list(np.random.default_rng(5).integers(0, N, 510))))
    idx = torch.tensor(rows, device="cuda")
    cdx = torch.tensor(cols, device="cuda")
    Ah = A[idx].cpu().numpy()
    got = R[idx][:, cdx].cpu().numpy()
    Bh, th, dh = B[:, cdx].cpu().numpy(), t[cdx].cpu().numpy(), d[cdx].cpu().numpy()
    want = oracle("discount", Ah, Bh, th, dh)  # rows x sampled columns: exact oracle entries
    check("discount", "f64", got, want, what="config 4 sampled rows x columns")


@pytest.mark.parametrize("dtype,order", [("f64", 0), ("f32", 1), ("i32", 0)])
def test_device_matrix_alloc_upload_download(gpu_ctx, dtype, order):
    """amlt_gpu_matrix_*: the library's own device matrices (f64 host values
    in, the plan's dtype on the device, f64 out), padded to 16 bytes, usable
    as operands."""
    import ctypes as C

    import paper_2305_08872_b200 as P
    from paper_2305_08872_b200 import _native as N

    L = N.lib()
    dt = {"f64": N.F64, "f32": N.F32, "i32": N.I32}[dtype]
    body = "eqcount" if dtype == "i32" else "gemm"
    M, K, N_ = 37, 29, 45
    A, B, _, _ = make_inputs(body, M, K, N_, "int", seed=71)

    def dev(x, order):
        m = N.Matrix()
        r, c = x.shape
        assert L.amlt_gpu_matrix_alloc(gpu_ctx.handle, r, c, order, dt, C.byref(m)) == N.OK
        assert m.ld * (8 if dt == N.F64 else 4) % 16 == 0
        host = np.ascontiguousarray(x if order == 0 else x.T)
        assert L.amlt_gpu_matrix_upload(gpu_ctx.handle, C.byref(m), host.ctypes.data,
                                        host.shape[1]) == N.OK
        return m, host

    ma, _ = dev(A, order)
    mb, _ = dev(B, 0)
    mr, _ = dev(np.zeros((M, N_)), 0)
    plan = gpu_ctx.plan(body, dtype)
    ops = N.OperandsC(ma, mb, mr, N.Matrix(), N.Matrix(), 0)
    b = N.BoundsC(0, M, 0, N_, 0, K)
    tp = N.TileParamsC(0, 0, 0, -1)
    el = C.c_double()
    assert L.amlt_gpu_run_subtask(gpu_ctx.handle, plan.handle, C.byref(ops), C.byref(tp),
                                  C.byref(b), N.CLOCK_FN(), None, None, C.byref(el)) == N.OK
    out = np.empty((M, N_))
    assert L.amlt_gpu_matrix_download(gpu_ctx.handle, C.byref(mr), out.ctypes.data, N_) == N.OK
    want = oracle(body, A, B)
    check(body, dtype, out, want, exact=True, what="device matrices")
    back = np.empty((A if order == 0 else A.T).shape)  # C-ordered storage rows
    L.amlt_gpu_matrix_download(gpu_ctx.handle, C.byref(ma), back.ctypes.data, back.shape[1])
    assert np.array_equal(back, A if order == 0 else A.T)
    for m in (ma, mb, mr):
        assert L.amlt_gpu_matrix_free(gpu_ctx.handle, C.byref(m)) == N.OK and not m.data


@pytest.mark.parametrize("name", ["gemm_f32_128x256_tcgen05_3xtf32",
                                  "gemm_f32_128x128_tcgen05_3xtf32_acc4"])
def test_tcgen05_gemm_edges(gpu_ctx, name):
    """The tensor-core f32 GEMM forced through: ragged M/N tiles, a
    sub-rectangle of a larger R (everything outside untouched, R0 accumulated),
    transposed / col-major operands (packed first), and BASELINE data within
    1e-5 normwise."""
    import torch

    import paper_2305_08872_b200 as P

    rng = np.random.default_rng(81)
    # ragged tiles, accumulate onto R0, sub-rectangle
    M, K, N = 300, 136, 520
    A = rng.integers(-8, 9, (M, K)).astype(np.float32)
    B = rng.integers(-8, 9, (K, N)).astype(np.float32)
    R0 = rng.integers(-100, 100, (M, N)).astype(np.float32)
    b = (17, 290, 12, 500, 8, 128)  # i0, i1, j0, j1, k0, k1 (k0, j0 keep 16-byte alignment)
    want = R0.astype(np.float64).copy()
    want[b[0]:b[1], b[2]:b[3]] += A[b[0]:b[1], b[4]:b[5]].astype(np.float64) @ \
        B[b[4]:b[5], b[2]:b[3]].astype(np.float64)
    for layout_a, layout_b in ((0, 0), (1, 0), (0, 1), (1, 1)):
        plan = gpu_ctx.plan("gemm", "f32", layout_a=layout_a, layout_b=layout_b)
        vi = [v.name for v in plan.variants()].index(name)
        Ab = torch.from_numpy(np.ascontiguousarray(A.T if layout_a else A)).cuda()
        Bb = torch.from_numpy(np.ascontiguousarray(B.T if layout_b else B)).cuda()
        R = torch.from_numpy(R0.copy()).cuda()
        P.run_subtask(plan, P.Operands(Ab, Bb, R), P.TileParams(variant=vi), P.Bounds(*b))
        assert np.array_equal(R.cpu().numpy().astype(np.float64), want), (name, layout_a, layout_b)
    # BASELINE distribution (N(0,1)), normwise against the fp64 oracle
    M, K, N = 512, 2048, 768
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    plan = gpu_ctx.plan("gemm", "f32")
    vi = [v.name for v in plan.variants()].index(name)
    R = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    P.run_subtask(plan, P.Operands(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), R),
                  P.TileParams(variant=vi), P.Bounds(0, M, 0, N, 0, K))
    want = A.astype(np.float64) @ B.astype(np.float64)
    check("gemm", "f32", R.cpu().numpy(), want, A=A.astype(np.float64), B=B.astype(np.float64),
          what=name)


def test_ozaki_f64_gemm_on_int8_tensor_cores():
    """The f64 GEMM on the int8 tensor cores (Ozaki slicing): exact on integer
    data (ragged tiles, sub-rectangles, every orientation), <= 1e-12 normwise
    on N(0,1) data at BASELINE's K, NaN for rows/columns holding inf/nan, and
    opt-in for the tuner (AMLT_CTX_F64_EMULATION)."""
    import torch

    import paper_2305_08872_b200 as P

    ctx = P.Context(0)
    rng = np.random.default_rng(91)
    name = "gemm_f64_128x64_tcgen05_ozaki_i8"
    M, K, N = 300, 136, 264
    A = rng.integers(-8, 9, (M, K)).astype(np.float64)
    B = rng.integers(-8, 9, (K, N)).astype(np.float64)
    R0 = rng.integers(-100, 100, (M, N)).astype(np.float64)
    b = (17, 290, 8, 250, 8, 128)
    want = R0.copy()
    want[b[0]:b[1], b[2]:b[3]] += A[b[0]:b[1], b[4]:b[5]] @ B[b[4]:b[5], b[2]:b[3]]
    for layout_a, layout_b in ((0, 0), (1, 0), (0, 1), (1, 1)):
        plan = ctx.plan("gemm", "f64", layout_a=layout_a, layout_b=layout_b)
        vi = [v.name for v in plan.variants()].index(name)
        R = torch.from_numpy(R0.copy()).cuda()
        P.run_subtask(plan, P.Operands(torch.from_numpy(np.ascontiguousarray(A.T if layout_a else A)).cuda(),
                                       torch.from_numpy(np.ascontiguousarray(B.T if layout_b else B)).cuda(), R),
                      P.TileParams(variant=vi), P.Bounds(*b))
        assert np.array_equal(R.cpu().numpy(), want), (layout_a, layout_b)
    # N(0,1) at K = 8192 (BASELINE config 2's depth), normwise vs the fp64 oracle
    plan = ctx.plan("gemm", "f64")
    vi = [v.name for v in plan.variants()].index(name)
    M, K, N = 256, 8192, 384
    A = rng.standard_normal((M, K))
    B = rng.standard_normal((K, N))
    R = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    P.run_subtask(plan, P.Operands(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), R),
                  P.TileParams(variant=vi), P.Bounds(0, M, 0, N, 0, K))
    check("gemm", "f64", R.cpu().numpy(), oracle("gemm", A, B), A=A, B=B, what="ozaki N(0,1)")
    # non-finite inputs: the affected row / column becomes NaN, the rest is exact
    A = rng.integers(-8, 9, (128, 64)).astype(np.float64)
    B = rng.integers(-8, 9, (64, 128)).astype(np.float64)
    A[5, 3] = np.inf
    B[7, 9] = np.nan
    R = torch.zeros((128, 128), dtype=torch.float64, device="cuda")
    P.run_subtask(plan, P.Operands(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), R),
                  P.TileParams(variant=vi), P.Bounds(0, 128, 0, 128, 0, 64))
    got = R.cpu().numpy()
    assert np.isnan(got[5]).all() and np.isnan(got[:, 9]).all()
    mask = np.ones_like(got, dtype=bool)
    mask[5] = False
    mask[:, 9] = False
    ref = np.nan_to_num(A, posinf=0.0) @ np.nan_to_num(B, nan=0.0)
    assert np.array_equal(got[mask], ref[mask])
    # opt-in: the default tuner never picks it; with the flag it is a candidate
    M = K = N = 1024
    A = torch.randn((M, K), device="cuda", dtype=torch.float64)
    B = torch.randn((K, N), device="cuda", dtype=torch.float64)
    R = torch.zeros((M, N), device="cuda", dtype=torch.float64)
    rep = P.adaptive_execute(plan, P.Operands(A, B, R), P.Bounds(0, M, 0, N, 0, K))
    assert all(plan.variants()[t.value].name != name for t in rep.trials)
    ectx = P.Context(0, f64_emulation=True)
    eplan = ectx.plan("gemm", "f64")
    R.zero_()
    rep = P.adaptive_execute(eplan, P.Operands(A, B, R), P.Bounds(0, M, 0, N, 0, K))
    assert any(eplan.variants()[t.value].name == name for t in rep.trials)


def test_tuning_cache_across_layouts_alignment_and_threshold_forms(gpu_ctx):
    """The per-shape tuning cache must not carry a winner into a call it cannot
    serve: same (M, N, K) with aligned then unaligned operands, and with a plan
    whose variants differ (thresholds indexed by i)."""
    import torch

    import paper_2305_08872_b200 as P

    M, K, N = 1500, 600, 700  # tunable size: the first call caches a winner
    A, B, t, d = make_inputs("discount", M, K, N, "int", seed=71)
    want = oracle("discount", A, B, t, d)
    ctx = P.Context(0)
    plan = ctx.plan("discount", "f64")
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    for rep in range(2):  # second run hits the cache
        R = torch.zeros((M, N), dtype=torch.float64, device="cuda")
        P.adaptive_execute(plan, P.Operands(dev(A), dev(B), R, dev(t), dev(d)), P.Bounds(0, M, 0, N, 0, K))
        check("discount", "f64", R.cpu().numpy(), want, exact=True, what=f"aligned run {rep}")
    # unaligned: A and B as views with an odd leading dimension
    Ab = torch.zeros((M, K + 1), dtype=torch.float64, device="cuda")
    Ab[:, :K] = dev(A)
    Bb = torch.zeros((K, N + 1), dtype=torch.float64, device="cuda")
    Bb[:, :N] = dev(B)
    R = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    P.adaptive_execute(plan, P.Operands(Ab[:, :K], Bb[:, :N], R, dev(t), dev(d)), P.Bounds(0, M, 0, N, 0, K))
    check("discount", "f64", R.cpu().numpy(), want, exact=True, what="unaligned after cached aligned")
    # same shape, thresholds indexed by i: a different variant family
    ti = np.random.default_rng(72).integers(-8, 9, M).astype(np.float64)
    iplan = ctx.plan("discount", "f64", thres_class="i")
    R = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    rep = P.adaptive_execute(iplan, P.Operands(dev(A), dev(B), R, dev(ti), dev(d)), P.Bounds(0, M, 0, N, 0, K))
    wi = np.zeros((M, N))
    for i in range(M):
        wi[i] = oracle("discount", A[i:i + 1], B, np.full(N, ti[i]), d)[0]
    check("discount", "f64", R.cpu().numpy(), wi, exact=True, what="thres[i] after cached thres[j]")
    assert rep.best_variant >= 0


@pytest.mark.parametrize("dtype,variant", [("f64", None), ("f32", None), ("f32", "cuda_core")])
def test_config2_full_size_sampled_rows(gpu_ctx, dtype, variant):
    """BASELINE config 2 at its full 8192^3 shape (plain GEMM, A and B
    N(0,1)): the tuned winner (DMMA for f64, the tcgen05 3xTF32 GEMM for
    f32) and, for f32, the fastest CUDA-core FFMA tile as the config is
    written; the oracle on the first / last rows plus random rows x sampled
    columns, normwise (|d| <= tol * sum_k |a b|)."""
    import torch

    import paper_2305_08872_b200 as P

    M = K = N = 8192
    td = {"f64": torch.float64, "f32": torch.float32}[dtype]
    g = torch.Generator(device="cuda").manual_seed(21)
    A = torch.randn((M, K), device="cuda", dtype=td, generator=g)
    B = torch.randn((K, N), device="cuda", dtype=td, generator=g)
    R = torch.zeros((M, N), device="cuda", dtype=td)
    plan = gpu_ctx.plan("gemm", dtype)
    ops = P.Operands(A, B, R, None, None)
    bounds = P.Bounds(0, M, 0, N, 0, K)
    names = [v.name for v in plan.variants()]
    if variant == "cuda_core":
        vi = names.index("gemm_f32_64x128_t8x4_w8x1")  # the cuda_core leg of bench.py
        P.run_subtask(plan, ops, P.TileParams(variant=vi), bounds)
        used = names[vi]
    else:
        rep = P.adaptive_execute(plan, ops, bounds)
        used = names[rep.best_variant]
        assert ("dmma" in used) if dtype == "f64" else ("tcgen05" in used)
    rows = sorted({0, M - 1, M // 2} | set(int(x) for x in np.random.default_rng(6).integers(0, M, 9)))
    cols = sorted({0, N - 1} | set(int(x) for x in np.random.default_rng(7).integers(0, N, 300)))
    idx = torch.tensor(rows, device="cuda")
    cdx = torch.tensor(cols, device="cuda")
    got = R[idx][:, cdx].double().cpu().numpy()
    Ah = A[idx].double().cpu().numpy()
    Bh = B[:, cdx].double().cpu().numpy()
    want = oracle("gemm", Ah, Bh)
    check("gemm", dtype, got, want, A=Ah, B=Bh, what=f"config 2 {dtype} {used}")


def test_context_stream_is_ordered_after_the_default_stream(gpu_ctx):
    """Operands made by PyTorch on its default stream (here a 1 GiB zero-fill
    of R queued right before the call) must be complete when the context's
    own stream runs the kernel: the own stream is a blocking stream. With a
    non-blocking one the zero-fill could land after the kernel (R all zero)."""
    import torch

    import paper_2305_08872_b200 as P

    M, K, N = 8192, 16, 16384
    A = torch.ones((M, K), device="cuda", dtype=torch.float64)
    B = torch.ones((K, N), device="cuda", dtype=torch.float64)
    plan = gpu_ctx.plan("gemm", "f64")
    for _ in range(3):
        R = torch.zeros((M, N), device="cuda", dtype=torch.float64)  # 1 GiB fill on the default stream
        P.run_subtask(plan, P.Operands(A, B, R, None, None), P.TileParams(), P.Bounds(0, M, 0, N, 0, K))
        assert bool((R == K).all())


@pytest.mark.parametrize("body,dtype", [("discount", "f64"), ("gemm", "f64"), ("eqcount", "i32"),
                                        ("boost", "f32"), ("gemm", "f32")])
def test_empty_bounds_leave_r_untouched(gpu_ctx, body, dtype):
    """Empty rectangles (no rows, no columns, or an empty k range) through
    every entry and every tile variant: R keeps its prior value exactly
    (tiled_executor.cpp:9-77 does nothing for an empty range), nothing is
    launched with a zero grid."""
    import torch

    import paper_2305_08872_b200 as P

    M, K, N = 70, 96, 128  # aligned: every variant (TMA ones included) runs the non-empty cases
    A, B, t, d = make_inputs(body, M, K, N, "int", seed=4)
    R0 = np.random.default_rng(4).integers(-8, 9, (M, N)).astype(np.float64)
    plan = gpu_ctx.plan(body, dtype)
    ops = lambda R: P.Operands(dev(A, dtype), dev(B, dtype), R, dev(t, dtype), dev(d, dtype))  # noqa: E731
    # (j0 = 7 / k0 = 31 offsets leave the operand views unaligned: an empty
    # rectangle must not care)
    empties = [P.Bounds(5, 5, 0, N, 0, K), P.Bounds(0, M, 7, 7, 0, K), P.Bounds(0, M, 0, N, 31, 31),
               P.Bounds(0, 0, 0, 0, 0, 0)]
    for b in empties:
        for vi, v in enumerate(plan.variants()):
            R = dev(R0, dtype)
            P.run_subtask(plan, ops(R), P.TileParams(variant=vi), b)
            assert np.array_equal(R.cpu().numpy().astype(np.float64), R0), (v.name, b)
        R = dev(R0, dtype)
        P.adaptive_execute(plan, ops(R), b)
        assert np.array_equal(R.cpu().numpy().astype(np.float64), R0), ("adaptive", b)
        hR = torch.from_numpy(R0.astype(NP_DT[dtype])).pin_memory()
        hops = P.Operands(*(torch.from_numpy(np.ascontiguousarray(x).astype(NP_DT[dtype])).pin_memory()
                            if x is not None else None for x in (A, B)), hR,
                          *(torch.from_numpy(x.astype(NP_DT[dtype])).pin_memory() if x is not None else None
                            for x in (t, d)))
        P.run_host(plan, hops, b)
        assert np.array_equal(hR.numpy().astype(np.float64), R0), ("run_host", b)


@pytest.mark.parametrize("stmt", ["+= A[i][k]*B[k][j] + u[i]*v[j] - (A[i][k] > s)*W[i][j]/4",
                                  "= A[i][k]*B[k][j] - (A[i][k]*B[k][j] > thres[j])*A[i][k]*B[k][j]*dis[j]",
                                  "+= A[i][k]*B[k][j]"])
def test_empty_bounds_generated_assign_naive_host(gpu_ctx, stmt):
    """Empty rectangles through a generated (NVRTC) body, an "=" statement
    (last k wins), the per-element executor and the tuned host entry: R
    keeps its prior value (R[j][j]-style views with unaligned offsets
    included)."""
    import torch

    import paper_2305_08872_b200 as P

    head = "where(i in [0..M] and j in [0..N] and k in [0..K]) {\n  R[i][j] "
    plan = gpu_ctx.plan_source(head + stmt + ";\n}\n", "f64")
    M, K, N = 40, 48, 64
    rng = np.random.default_rng(9)
    R0 = rng.integers(-8, 9, (M, N)).astype(np.float64)
    names = plan.aux_names
    aux_shape = {"u": (M,), "v": (N,), "s": (1, 1), "W": (M, N)}
    named = {"thres": rng.integers(-8, 9, N).astype(np.float64), "dis": rng.integers(-8, 9, N).astype(np.float64)}
    A = rng.integers(-8, 9, (M, K)).astype(np.float64)
    B = rng.integers(-8, 9, (K, N)).astype(np.float64)

    def operands(R, place):
        aux = tuple(place(rng.integers(-8, 9, aux_shape[n]).astype(np.float64)) for n in names)
        thres = place(named["thres"]) if "thres" in stmt else None
        dis = place(named["dis"]) if "dis" in stmt else None
        return P.Operands(place(A), place(B), R, thres, dis, aux=aux)

    to_dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    to_host = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory()  # noqa: E731
    for b in (P.Bounds(3, 3, 0, N, 0, K), P.Bounds(0, M, 5, 5, 0, K), P.Bounds(0, M, 0, N, 7, 7)):
        R = to_dev(R0)
        P.adaptive_execute(plan, operands(R, to_dev), b)
        P.run_naive(plan, operands(R, to_dev), b)
        for vi in range(len(plan.variants())):
            P.run_subtask(plan, operands(R, to_dev), P.TileParams(variant=vi), b)
        assert np.array_equal(R.cpu().numpy(), R0), (stmt, b)
        hR = to_host(R0)
        P.run_host_adaptive(plan, operands(hR, to_host), b)
        assert np.array_equal(hR.numpy(), R0), ("host", stmt, b)


@pytest.mark.parametrize("body,dtype,variant,kc", [
    ("discount", "f64", "discount_f64_48x128_theta_t6x4_w8x1", 208),  # B preparation + split-K reduce
    ("discount", "f64", "discount_f64_32x128_t4x4_w8x1", 0),
    ("gemm", "f32", "gemm_f32_128x256_tcgen05_3xtf32", 0),  # operand split pre-pass
    ("eqcount", "i32", "eqcount_i32_32x128_swar_t4x4_w8x1", 0),  # packing pre-pass + guarded pair
    ("gemm", "f64", "gemm_f64_64x128_dmma_w32x32_c2x4", 256)])
def test_graph_replay_matches_enqueue(gpu_ctx, body, dtype, variant, kc):
    """amlt_gpu_graph_capture: a captured step replayed N times gives what N
    plain enqueues give (bit-exact on IntValued data), and a launch after the
    context's workspaces were reallocated is refused, not run on freed
    memory."""
    import paper_2305_08872_b200 as P

    M, K, N = 300, 1024, 520
    A, B, t, d = make_inputs(body, M, K, N, "int", seed=12)
    if body == "eqcount":
        A, B = np.abs(A), np.abs(B)
    plan = gpu_ctx.plan(body, dtype)
    vi = [v.name for v in plan.variants()].index(variant)
    tp = P.TileParams(kc=kc, variant=vi)
    bnd = P.Bounds(0, M, 0, N, 0, K)
    R1, R2 = dev(np.zeros((M, N)), dtype), dev(np.zeros((M, N)), dtype)
    ops1 = P.Operands(dev(A, dtype), dev(B, dtype), R1, dev(t, dtype), dev(d, dtype))
    ops2 = P.Operands(ops1.a, ops1.b, R2, ops1.thres, ops1.dis)
    g = P.capture_graph(plan, ops2, tp, bnd)  # runs one plain step on R2 first
    for _ in range(3):
        P.enqueue(plan, ops1, tp, bnd)
        g.launch()
    P.enqueue(plan, ops1, tp, bnd)  # R1: 4 steps, R2: 1 (capture) + 3 replays
    got1, got2 = R1.cpu().numpy(), R2.cpu().numpy()
    assert np.array_equal(got1, got2), variant
    want = oracle(body, A, B, t, d)
    check(body, dtype, got2 / 4, want, exact=True, what=f"graph {variant}")
    # workspaces reallocated (a bigger split-K / preparation need): refused
    big = 4 * M
    Ab = np.tile(A, (4, 1))
    Rb = dev(np.zeros((big, N)), dtype)
    P.run_subtask(plan, P.Operands(dev(Ab, dtype), ops1.b, Rb, ops1.thres, ops1.dis),
                  P.TileParams(kc=64, variant=vi), P.Bounds(0, big, 0, N, 0, K))
    gpu_ctx_ws_grew = True
    try:
        g.launch()
        gpu_ctx_ws_grew = False  # nothing was reallocated: the replay is still valid
    except P.EngineError as e:
        assert "reallocated" in str(e)
    if not gpu_ctx_ws_grew:
        assert np.array_equal(R2.cpu().numpy(), got2 + got2 / 4)
    g.close()
