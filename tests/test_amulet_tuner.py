"""CPU: AMULET's own tuner contract on the GPU executor, decision for decision
against the UNMODIFIED reference tuner.

acceptance.cpp c5 (1000 scripted-clock tuner checks) and test_autotuner.cpp
drive the reference's run_adaptive with a FakeClock script and check the kc /
nc winners. Here the same scripts drive both the reference (oracle/_ref) and
amlt_gpu_adaptive_execute_amulet (dry-run context, same kernel shape i_h x
i_w): winners, tuned flag, number of clock intervals consumed and the (k, j)
coverage ledger must all be identical. acceptance c4 (exactly-once (i,j,k)
execution) is checked from the GPU executor's dispatch log.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2305_08872_b200 as P
from oracle import pyoracle as po

needs_ref = pytest.mark.skipif(not po.ref_available(), reason="reference engine not built")


def gpu_ops(M, K, N, dtype=np.float64):
    return P.Operands(np.empty((M, K), dtype), np.empty((K, N), dtype), np.empty((M, N), dtype))


@needs_ref
def test_tuner_decisions_match_reference_under_scripted_clocks(dry_ctx):
    rng = np.random.default_rng(97)
    src = po.preset_source("matmul")
    plan = dry_ctx.plan("gemm", "f64")
    for sample in range(300):
        K = 1 + int(rng.integers(0, 260))
        N = 64 + int(rng.integers(0, 237))
        M = 13
        deltas = list(rng.uniform(1e-4, 1.0, 64))
        ref = po.RefTask.create(src, M, K, N, seed=7)
        ih, iw = ref.shape()
        kc, nc, tuned, used, rects = ref.run_adaptive_scripted(deltas)
        clk = P.FakeClock(deltas)
        rep = P.engine.adaptive_execute_amulet(plan, gpu_ops(M, K, N), P.Bounds(0, M, 0, N, 0, K),
                                               i_h=ih, i_w=iw, clock=clk)
        what = f"sample {sample} K={K} N={N}"
        assert (rep.best_kc, rep.best_nc, rep.tuned) == (kc, nc, tuned), what
        assert clk.consumed() == used, what
        assert [(c.k0, c.k1, c.j0, c.j1) for c in rep.coverage] == rects, what


@needs_ref
def test_untuned_small_tasks_match_reference(dry_ctx):
    src = po.preset_source("q1")
    plan = dry_ctx.plan("discount", "f64")
    for (M, K, N) in [(13, 17, 5), (5, 300, 400), (64, 64, 40)]:
        ref = po.RefTask.create(src, M, K, N, seed=1)
        ih, iw = ref.shape()
        kc, nc, tuned, used, rects = ref.run_adaptive_scripted([0.5] * 8)
        ops = P.Operands(np.empty((M, K)), np.empty((K, N)), np.empty((M, N)), np.empty(N),
                         np.empty(N))
        rep = P.engine.adaptive_execute_amulet(plan, ops, P.Bounds(0, M, 0, N, 0, K), i_h=ih,
                                               i_w=iw, clock=P.FakeClock([0.5] * 8))
        assert (rep.best_kc, rep.best_nc, rep.tuned) == (kc, nc, tuned)
        assert [(c.k0, c.k1, c.j0, c.j1) for c in rep.coverage] == rects


def test_exactly_once_execution(dry_ctx):
    """acceptance c4: every (i, j, k) cell is executed exactly once, and the
    coverage rectangles tile K x N exactly once."""
    rng = np.random.default_rng(41)
    plan = dry_ctx.plan("gemm", "f64")
    for t in range(50):
        M = 1 + int(rng.integers(0, 64))
        K = 1 + int(rng.integers(0, 280))
        N = 1 + int(rng.integers(0, 300))
        log = P.ExecLog()
        rep = P.engine.adaptive_execute_amulet(plan, gpu_ops(M, K, N), P.Bounds(0, M, 0, N, 0, K),
                                               i_h=12, i_w=16, clock=P.FakeClock([0.1] * 200),
                                               log=log)
        cells = np.zeros((M, N, K), dtype=np.int8)
        for r in log.records:
            cells[r.i0:r.i1, r.j0:r.j1, r.k0:r.k1] += 1
        assert (cells == 1).all(), f"{M}x{K}x{N}"
        kj = np.zeros((K, N), dtype=np.int8)
        for c in rep.coverage:
            kj[c.k0:c.k1, c.j0:c.j1] += 1
        assert (kj == 1).all()


def test_kc_candidates_and_tuning_fraction(dry_ctx):
    """kc candidates K, ceil-halvings >= 16 (autotuner.cpp:8-16); the
    tuning fraction is (4 i_w + sum of tested nc) / N (autotuner.cpp:128-131)."""
    plan = dry_ctx.plan("gemm", "f64")
    M, K, N = 64, 1000, 1000
    rep = P.engine.adaptive_execute_amulet(plan, gpu_ops(M, K, N), P.Bounds(0, M, 0, N, 0, K),
                                           clock=P.FakeClock([1.0] * 64))
    assert [t.value for t in rep.kc_trials] == [1000, 500, 250, 125, 63, 32, 16]
    assert rep.tuning_fraction == pytest.approx(
        (4 * 16 + sum(t.value for t in rep.nc_trials)) / N)
    # equal scripted intervals: elapsed/kc is smallest for the largest kc
    assert rep.best_kc == 1000
