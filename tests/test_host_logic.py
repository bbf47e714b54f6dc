"""CPU: the C-ABI library and the host-side logic, without a GPU.

* the shared library loads and exports every symbol include/amlt_gpu.h
  declares (no compute calls);
* the executor / tuner run in DRY-RUN contexts (AMLT_CTX_DRY_RUN: dispatches
  are planned, logged and clocked through the Clock seam, no device touched),
  so the tuner's decisions are checked deterministically with scripted
  FakeClock intervals — the reference's own strategy for its tuner
  (tests/test_autotuner.cpp:60-171, acceptance c4/c5);
* error mapping onto the EngineError hierarchy (errors.hpp:10-60).
"""
from __future__ import annotations

import os
import re

import numpy as np
import pytest

import paper_2305_08872_b200 as P
from paper_2305_08872_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "amlt_gpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(amlt_\w+)\s*\(", text)) - {"amlt_clock_fn"})


def test_library_exports_every_header_symbol():
    import ctypes

    lib = ctypes.CDLL(N.LIB_PATH)
    names = header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), f"libamlt_gpu.so does not export {n}"
    assert set(N.EXPORTS) == set(names)
    assert N.lib().amlt_gpu_abi_version() == N.ABI_VERSION


def test_library_is_sm100a_only():
    """The fatbin carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_spr_and_nonpositive_time():
    # reference tests/test_engine.cpp:367-374 restated
    assert P.spr(1000, 1000, 1000, 1.0) == pytest.approx(1.0)
    assert P.spr(1024, 1024, 1024, 0.5) == pytest.approx(1024 ** 3 / 0.5e9)
    with pytest.raises(P.NonPositiveTime):
        P.spr(1, 1, 1, 0.0)
    with pytest.raises(P.NonPositiveTime):
        P.spr(1, 1, 1, -1.0)


def big_ops(M, K, N, body="discount", dtype=np.float64):
    """Untouched (virtual) buffers: dry-run contexts never read them."""
    A = np.empty((M, K), dtype)
    B = np.empty((K, N), dtype)
    R = np.empty((M, N), dtype)
    t = np.empty(N, dtype) if body in ("discount", "boost", "thrcount") else None
    d = np.empty(N, dtype) if body == "discount" else None
    return P.Operands(A, B, R, t, d)


def test_run_subtask_reads_clock_exactly_twice(dry_ctx):
    plan = dry_ctx.plan("discount", "f64")
    clk = P.FakeClock([0.25])
    el = P.run_subtask(plan, big_ops(64, 32, 64), P.TileParams(), P.Bounds(0, 64, 0, 64, 0, 32),
                       clock=clk)
    assert el == 0.25 and clk.consumed() == 1 and not clk.open
    with pytest.raises(IndexError):  # script exhausted -> loud failure, as FakeClock does
        P.run_subtask(plan, big_ops(64, 32, 64), P.TileParams(), P.Bounds(0, 64, 0, 64, 0, 32),
                      clock=clk)


def tuned_call(ctx, deltas, M=131072, K=64, N=1024):
    plan = ctx.plan("discount", "f64")
    ctx.clear_tuning_cache()
    clk = P.FakeClock(deltas)
    log = P.ExecLog()
    rep = P.adaptive_execute(plan, big_ops(M, K, N), P.Bounds(0, M, 0, N, 0, K), clock=clk,
                             log=log)
    return plan, rep, clk, log


def test_tuner_picks_argmin_score_and_covers_once(dry_ctx):
    rng = np.random.default_rng(97)
    for trial in range(40):
        deltas = list(rng.uniform(1e-4, 1.0, 16))
        plan, rep, clk, log = tuned_call(dry_ctx, deltas)
        assert rep.tuned
        n = len(rep.trials)
        assert n >= 2
        # every trial consumed one scripted interval, the remainder one more
        assert clk.consumed() == n + 1
        for i, t in enumerate(rep.trials):
            assert t.elapsed == pytest.approx(deltas[i])
            # elapsed / rows, scaled by c / ceil(c) for c CTAs per SM in the band
            assert deltas[i] / t.rows * 0.5 < t.score <= deltas[i] / t.rows * (1 + 1e-12)
        scores = [t.score for t in rep.trials]
        want = rep.trials[int(np.argmin(scores))].value  # ties keep the earlier
        assert rep.best_variant == want
        # exactly-once coverage of the rows, full N and K each
        cover = np.zeros(131072, dtype=np.int32)
        for c in rep.coverage:
            assert (c.j0, c.j1, c.k0, c.k1) == (0, 1024, 0, 64)
            cover[c.i0:c.i1] += 1
        assert (cover == 1).all()
        assert rep.total_seconds == pytest.approx(sum(deltas[:n + 1]))
        assert 0 < rep.tuning_fraction <= 0.25
        # the remainder ran with the winner
        assert log.records[-1].variant == rep.best_variant
        assert [r.variant for r in log.records[:n]] == [t.value for t in rep.trials]


def test_tuner_ties_keep_earlier_candidate(dry_ctx):
    plan, rep, clk, log = tuned_call(dry_ctx, [1.0] * 16)
    scores = [t.score for t in rep.trials]
    best = min(scores)
    assert rep.best_variant == rep.trials[scores.index(best)].value


def test_tuner_cache_reused_on_second_call(dry_ctx):
    plan, rep, clk, log = tuned_call(dry_ctx, [0.5, 0.1] + [0.9] * 14)
    clk2 = P.FakeClock([0.3])
    log2 = P.ExecLog()
    rep2 = P.adaptive_execute(plan, big_ops(131072, 64, 1024), P.Bounds(0, 131072, 0, 1024, 0, 64),
                              clock=clk2, log=log2)
    assert rep2.from_cache and not rep2.tuned
    assert rep2.best_variant == rep.best_variant
    assert len(log2.records) == 1 and clk2.consumed() == 1
    assert log2.records[0].variant == rep.best_variant


def test_small_task_runs_untuned_whole(dry_ctx):
    plan = dry_ctx.plan("discount", "f64")
    dry_ctx.clear_tuning_cache()
    clk = P.FakeClock([0.01])
    log = P.ExecLog()
    rep = P.adaptive_execute(plan, big_ops(300, 200, 100), P.Bounds(0, 300, 0, 100, 0, 200),
                             clock=clk, log=log)
    assert not rep.tuned and rep.trials == []
    assert len(rep.coverage) == 1 and len(log.records) == 1
    c = rep.coverage[0]
    assert (c.i0, c.i1, c.j0, c.j1, c.k0, c.k1) == (0, 300, 0, 100, 0, 200)


def test_small_output_large_k_splits_k(dry_ctx):
    """An output that cannot fill 148 SMs gets split-K (deterministic
    ordered reduction); config 0 (1024^3) is such a case."""
    plan = dry_ctx.plan("discount", "f64")
    dry_ctx.clear_tuning_cache()
    log = P.ExecLog()
    rep = P.adaptive_execute(plan, big_ops(256, 4096, 256), P.Bounds(0, 256, 0, 256, 0, 4096),
                             clock=P.FakeClock([0.01]), log=log)
    assert log.records[0].splits > 1
    assert rep.best_kc < 4096 and rep.best_kc % 16 == 0


@pytest.mark.parametrize("kc,want_splits", [(0, 1), (5000, 1), (1000, 1), (256, 4), (100, 9),
                                            (64, 16)])
def test_tile_kc_is_split_k(dry_ctx, kc, want_splits):
    plan = dry_ctx.plan("gemm", "f64")
    log = P.ExecLog()
    P.run_subtask(plan, big_ops(128, 1000, 128, "gemm"), P.TileParams(kc=kc),
                  P.Bounds(0, 128, 0, 128, 0, 1000), clock=P.FakeClock([1.0]), log=log)
    assert log.records[0].splits == want_splits


def test_nc_selects_tile_width(dry_ctx):
    plan = dry_ctx.plan("discount", "f64")
    vs = plan.variants()
    for nc in (64, 128, 1000):
        log = P.ExecLog()
        P.run_subtask(plan, big_ops(256, 64, 256), P.TileParams(nc=nc),
                      P.Bounds(0, 256, 0, 256, 0, 64), clock=P.FakeClock([1.0]), log=log)
        assert vs[log.records[0].variant].block_n <= nc


def test_unaligned_operands_pick_element_variant(dry_ctx):
    plan = dry_ctx.plan("discount", "f64")
    vs = plan.variants()
    A = np.empty((64, 33))  # odd leading dimension
    ops = P.Operands(A, np.empty((33, 64)), np.empty((64, 64)), np.empty(64), np.empty(64))
    log = P.ExecLog()
    P.run_subtask(plan, ops, P.TileParams(), P.Bounds(0, 64, 0, 64, 0, 33),
                  clock=P.FakeClock([1.0]), log=log)
    assert vs[log.records[0].variant].name.endswith("_u")
    with pytest.raises(P.EngineError):  # explicit TMA variant on unaligned operands
        P.run_subtask(plan, ops, P.TileParams(variant=0), P.Bounds(0, 64, 0, 64, 0, 33),
                      clock=P.FakeClock([1.0]))


def test_errors_map_to_reference_hierarchy(dry_ctx):
    plan = dry_ctx.plan("discount", "f64")
    ops = big_ops(16, 16, 16)
    ops.dis = None
    with pytest.raises(P.MissingBinding):
        P.run_subtask(plan, ops, P.TileParams(), P.Bounds(0, 16, 0, 16, 0, 16))
    with pytest.raises(P.EngineError):
        P.run_subtask(plan, big_ops(16, 16, 16), P.TileParams(), P.Bounds(0, 17, 0, 16, 0, 16))
    # A[k][i] / B[j][k] over row-major buffers are packed (packing.hpp:11-18)
    for lay in ({"layout_a": N.LAYOUT_TRANSPOSED}, {"layout_b": N.LAYOUT_TRANSPOSED}):
        tplan = dry_ctx.plan("gemm", "f64", **lay)
        assert P.run_subtask(tplan, big_ops(16, 16, 16, "gemm"), P.TileParams(),
                             P.Bounds(0, 16, 0, 16, 0, 16), clock=P.FakeClock([0.5])) == 0.5
    with pytest.raises(P.UnsupportedExpression):  # u[k] is not an MMLT leaf
        P.compile_task("where(i in [0..M] and j in [0..N] and k in [0..K]) {\n"
                       "  R[i][j] += A[i][k]*B[k][j]*u[k];\n}\n")
    # a recognised statement outside the fixed bodies: a generated body
    assert P.compile_task("where(i in [0..M] and j in [0..N] and k in [0..K]) {\n"
                          "  R[i][j] += A[i][k]*B[k][j] + u[i]*v[j];\n}\n").body == N.BODY_GENERIC
    # thresholds indexed [i]: accepted, and the vector must cover i1
    iplan = dry_ctx.plan("discount", "f64", thres_class="i")
    assert all(v.name.endswith(("_ti", "_ti_u")) for v in iplan.variants())
    ops_i = big_ops(16, 16, 16)
    P.run_subtask(iplan, ops_i, P.TileParams(), P.Bounds(0, 16, 0, 16, 0, 16),
                  clock=P.FakeClock([1.0]))
    ops_i.thres = np.empty(8)
    with pytest.raises(P.EngineError):
        P.run_subtask(iplan, ops_i, P.TileParams(), P.Bounds(0, 16, 0, 16, 0, 16))
    with pytest.raises(P.UnsupportedExpression):
        dry_ctx.plan("gemm", "i32")  # no int32 GEMM kernel
    with pytest.raises(P.EngineError):  # dtype mismatch
        P.run_subtask(plan, big_ops(16, 16, 16, dtype=np.float32), P.TileParams(),
                      P.Bounds(0, 16, 0, 16, 0, 16))


def test_transposed_statement_over_col_major_buffer_is_supported(dry_ctx):
    """A[k][i] stored col-major has i-rows contiguous along k: same layout the
    kernels stage, so it is accepted (layouts are resolved per element)."""
    plan = dry_ctx.plan("gemm", "f64", layout_a=N.LAYOUT_TRANSPOSED)
    At = np.empty((64, 32), order="F")  # buffer rows = k (64), cols = i (32)
    ops = P.Operands(At, np.empty((64, 48)), np.empty((32, 48)))
    el = P.run_subtask(plan, ops, P.TileParams(), P.Bounds(0, 32, 0, 48, 0, 64),
                       clock=P.FakeClock([0.5]))
    assert el == 0.5


def test_plan_variants_describe_tiles(dry_ctx):
    for body, dt in [("discount", "f64"), ("boost", "f32"), ("eqcount", "i32"), ("gemm", "f64")]:
        vs = dry_ctx.plan(body, dt).variants()
        assert vs
        for v in vs:
            assert v.block_m % v.thread_m == 0 or v.tensor_core
            assert v.smem_bytes <= 227 * 1024
            assert v.threads % 32 == 0
    assert any(v.tensor_core for v in dry_ctx.plan("gemm", "f64").variants())


def test_dry_run_refuses_host_entry(dry_ctx):
    plan = dry_ctx.plan("gemm", "f64")
    with pytest.raises(P.NoDevice):
        P.run_host(plan, big_ops(8, 8, 8, "gemm"), P.Bounds(0, 8, 0, 8, 0, 8))


def test_no_device_context_fails_loudly():
    """Without a GPU, a real (non-dry) context must fail, not fall back."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(P.NoDevice):
        P.Context(0)


def test_run_naive_validates_like_run_subtask(dry_ctx):
    """amlt_gpu_run_naive shares the operand rules (missing aux, bounds
    beyond an operand) and never reads the clock in a dry-run context."""
    plan = dry_ctx.plan("discount", "f64")
    ops = big_ops(16, 16, 16)
    assert P.run_naive(plan, ops, P.Bounds(0, 16, 0, 16, 0, 16)) == 0.0
    ops.dis = None
    with pytest.raises(P.MissingBinding):
        P.run_naive(plan, ops, P.Bounds(0, 16, 0, 16, 0, 16))
    with pytest.raises(P.EngineError):
        P.run_naive(plan, big_ops(16, 16, 16), P.Bounds(0, 16, 0, 17, 0, 16))


def test_sharded_group_dry_run_bands_and_plans():
    """The persistent row-band group (amlt_sharded_*) on CPU: dry-run
    contexts plan and validate each device's band; bands are 64-row aligned
    and tile [i0, i1) exactly once (the same cut as bench.py's row_band);
    a second run of the group reuses its plans; bad operands fail loudly."""
    from paper_2305_08872_b200.sharded import row_band

    g = P.ShardedGroup([0, 1, 2, 3, 4, 5, 6, 7], dry_run=True)
    try:
        for M in (32768, 1000, 70):
            ops = big_ops(M, 64, 256)
            for _ in range(2):
                _, reps = g.run(ops, P.Bounds(0, M, 0, 256, 0, 64), body="discount")
                edges = [(r.coverage[0].i0, r.coverage[0].i1) for r in reps]
                assert edges == [row_band(M, 8, d, align=64) for d in range(8)]
                assert edges[0][0] == 0 and edges[-1][1] == M
                assert all(a1 == b0 for (_, a1), (b0, _) in zip(edges, edges[1:]))
        # a generated body through the same group
        src = ("where(i in [0..M] and j in [0..N] and k in [0..K]) {\n"
               "  R[i][j] += A[i][k]*B[k][j] + u[i]*v[j];\n}\n")
        M = 512
        ops = P.Operands(np.empty((M, 64)), np.empty((64, 256)), np.empty((M, 256)), None, None,
                         (np.empty(M), np.empty(256)))
        g.run(ops, P.Bounds(0, M, 0, 256, 0, 64), source=src)
        with pytest.raises(P.MissingBinding):  # dis missing
            g.run(P.Operands(np.empty((M, 64)), np.empty((64, 256)), np.empty((M, 256)), np.empty(256)),
                  P.Bounds(0, M, 0, 256, 0, 64), body="discount")
    finally:
        g.close()


@pytest.mark.parametrize("bounds", [(0, 70, 7, 7, 0, 96), (5, 5, 0, 128, 0, 96), (0, 70, 0, 128, 31, 31),
                                    (0, 0, 0, 0, 0, 0)])
def test_adaptive_on_an_empty_rectangle(dry_ctx, bounds):
    """An empty rectangle takes the untuned path (autotuner.cpp:112-122):
    no trials, tuned = false, its one coverage rectangle; the band sizing
    must not divide by its zero column-tile count (it did: SIGFPE)."""
    plan = dry_ctx.plan("discount", "f64")
    M, K, N = 70, 96, 128
    ops = P.Operands(np.zeros((M, K)), np.zeros((K, N)), np.zeros((M, N)), np.zeros(N), np.zeros(N))
    rep = P.adaptive_execute(plan, ops, P.Bounds(*bounds))
    i0, i1, j0, j1, k0, k1 = bounds
    assert not rep.tuned and not rep.trials
    assert [(c.i0, c.i1, c.j0, c.j1, c.k0, c.k1) for c in rep.coverage] == [bounds]
