"""GPU counterparts of the reference's performance acceptance criteria for
this path (tests/acceptance.cpp:190-280), on the task the
reference uses for them: matmul at 1024^3, integer-valued data. The discount
body (config 0's shape) is checked the same way.

  c6  the tuned choice within 1.20x of the best fixed grid point. The
      reference's grid is (kc, nc) in {16..1024}^2 for one interpreted kernel;
      the GPU's is every tile variant the tuner may pick x K segments {K, K/2,
      K/4}. Samples interleave round-robin over 3 rounds, minimum per cell
      (acceptance.cpp:212-247). The adaptive side is the steady state: the
      GPU tuner caches its winner per shape (the reference re-tunes each call).
  c7  adaptive at least 2x faster than the naive executor
      (acceptance.cpp:250-258): amlt_gpu_run_naive, one IEEE operation per
      syntax-tree node, k ascending.
  c8  packing neutral (acceptance.cpp:261-282): transposed operands (presets
      -atbt, packed by the executor before the tile kernel) give the bit-same
      result as the normal layout on integer data, and their elapsed time is
      within [0.5, 1.5]x of it with the same tile.
"""
from __future__ import annotations

import numpy as np
import pytest

from tests.helpers import int_valued

pytestmark = pytest.mark.gpu

N3 = 1024


def _setup(ctx, body, layout_a=0, layout_b=0):
    import torch

    import paper_2305_08872_b200 as P

    rng = np.random.default_rng(5)
    A, B = int_valued(rng, (N3, N3)), int_valued(rng, (N3, N3))
    th = dis = None
    if body == "discount":
        th, dis = int_valued(rng, N3), int_valued(rng, N3)
    t = lambda x: None if x is None else torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    R = torch.zeros((N3, N3), dtype=torch.float64, device="cuda")
    plan = ctx.plan(body, "f64", layout_a=layout_a, layout_b=layout_b)
    ops = P.Operands(t(A.T if layout_a else A), t(B.T if layout_b else B), R, t(th), t(dis))
    return P, plan, ops, R, P.Bounds(0, N3, 0, N3, 0, N3)


def _grid(P, plan):
    """(name, TileParams) cells the tuner can choose from (the opt-in int8
    f64 GEMM and unaligned-operand variants excluded)."""
    cells = []
    for vi, v in enumerate(plan.variants()):
        if "ozaki" in v.name or v.name.endswith("_u"):
            continue
        for kc in (0, N3 // 2, N3 // 4):
            cells.append((f"{v.name} kc={kc or N3}", P.TileParams(kc=kc, variant=vi)))
    return cells


@pytest.mark.parametrize("body", ["gemm", "discount"])
def test_c6_adaptive_within_1_20_of_best_grid_point(gpu_ctx, body):
    P, plan, ops, R, bnd = _setup(gpu_ctx, body)
    gpu_ctx.clear_tuning_cache()
    P.adaptive_execute(plan, ops, bnd)  # tunes once and caches the winner
    cells = []
    for name, tp in _grid(P, plan):
        try:
            P.run_subtask(plan, ops, tp, bnd)  # warm-up; drops cells that do not run
            cells.append((name, tp))
        except P.EngineError:
            pass
    assert cells
    best = {name: float("inf") for name, _ in cells}
    adaptive = float("inf")
    for _ in range(3):
        adaptive = min(adaptive, P.adaptive_execute(plan, ops, bnd).total_seconds)
        for name, tp in cells:
            best[name] = min(best[name], P.run_subtask(plan, ops, tp, bnd))
    adaptive = min(adaptive, P.adaptive_execute(plan, ops, bnd).total_seconds)
    name, grid = min(best.items(), key=lambda x: x[1])
    print(f"c6 {body}: adaptive {adaptive * 1e6:.1f} us, best grid {grid * 1e6:.1f} us ({name}), "
          f"ratio {adaptive / grid:.3f}")
    assert adaptive <= 1.20 * grid, f"{body}: adaptive {adaptive * 1e6:.1f} us vs best grid {grid * 1e6:.1f} us ({name})"


@pytest.mark.parametrize("body", ["gemm", "discount"])
def test_c7_adaptive_at_least_2x_faster_than_naive(gpu_ctx, body):
    P, plan, ops, R, bnd = _setup(gpu_ctx, body)
    P.adaptive_execute(plan, ops, bnd)
    adaptive = min(P.adaptive_execute(plan, ops, bnd).total_seconds for _ in range(3))
    R.zero_()
    naive = P.run_naive(plan, ops, bnd)
    print(f"c7 {body}: naive {naive * 1e3:.2f} ms, adaptive {adaptive * 1e3:.3f} ms, {naive / adaptive:.1f}x")
    assert naive >= 2.0 * adaptive, f"{body}: naive {naive * 1e3:.2f} ms vs adaptive {adaptive * 1e3:.3f} ms"


@pytest.mark.parametrize("body", ["gemm", "discount"])
def test_c8_packing_neutral(gpu_ctx, body):
    P, plan, ops, R, bnd = _setup(gpu_ctx, body)
    Pt, plan_t, ops_t, R_t, _ = _setup(gpu_ctx, body, layout_a=1, layout_b=1)
    # the same tile on both layouts: the normal layout's tuned winner
    gpu_ctx.clear_tuning_cache()
    rep = P.adaptive_execute(plan, ops, bnd)
    names = [v.name for v in plan.variants()]
    win = names[rep.best_variant]
    tp = P.TileParams(kc=rep.best_kc if rep.best_kc < N3 else 0, variant=rep.best_variant)
    tp_t = P.TileParams(kc=tp.kc, variant=[v.name for v in plan_t.variants()].index(win))
    R.zero_()
    P.run_subtask(plan, ops, tp, bnd)
    R_t.zero_()
    P.run_subtask(plan_t, ops_t, tp_t, bnd)
    assert np.array_equal(R.cpu().numpy(), R_t.cpu().numpy()), f"{body}: packed result differs ({win})"
    plain = min(P.run_subtask(plan, ops, tp, bnd) for _ in range(3))
    packed = min(P.run_subtask(plan_t, ops_t, tp_t, bnd) for _ in range(3))
    ratio = packed / plain
    print(f"c8 {body}: packed {packed * 1e6:.1f} us, unpacked {plain * 1e6:.1f} us, ratio {ratio:.2f} ({win})")
    assert 0.5 <= ratio <= 1.5, f"{body}: packed/unpacked elapsed ratio {ratio:.2f} ({win})"
