"""CPU: pin the oracle (our C restatement of run_naive) against the reference.

* known answers from the reference's own spec and tests;
* bit-exact agreement with the UNMODIFIED reference engine (oracle/_ref) on
  every body, int-valued and real data, all orientations it can express;
* the committed golden fixtures (tests/golden/, generated from the reference).
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import pyoracle as po
from tests.golden.load import load_golden
from tests.helpers import BODY_KIND, oracle

needs_ref = pytest.mark.skipif(not po.ref_available(), reason="reference engine not built")


def test_known_answers_spec():
    # Query 1 DAG with A*B=10, thres=5, dis=0.5 -> 5.0; thres=20 -> 10.0
    assert po.oracle_eval(po.DISCOUNT, 10.0, 1.0, 5.0, 0.5) == 5.0
    assert po.oracle_eval(po.DISCOUNT, 10.0, 1.0, 20.0, 0.5) == 10.0
    assert po.oracle_eval(po.DISCOUNT, 2.0, 5.0, 5.0, 0.5) == 5.0


def test_known_answers_expr_dag():
    # tests/test_expr_dag.cpp:130-150 with A=3, B=-2, thres=5 (the cases that
    # are one of the GPU bodies)
    assert po.oracle_eval(po.GEMM, 3, -2) == -6
    # A*B - (A*B > thres)*A*B  (discount with dis = 1)
    assert po.oracle_eval(po.DISCOUNT, 3, -2, 5, 1.0) == -6
    # A*B > 100 -> 0
    assert po.oracle_eval(po.THRCOUNT, 3, -2, 100) == 0
    assert po.oracle_eval(po.EQCOUNT, 3, 3) == 1 and po.oracle_eval(po.EQCOUNT, 3, -2) == 0
    assert po.oracle_eval(po.SQDIFF, 3, -2) == 25
    assert po.oracle_eval(po.BOOST, 3, 4, 5) == 12 + 7


@needs_ref
@pytest.mark.parametrize("body", sorted(BODY_KIND))
@pytest.mark.parametrize("int_valued", [True, False])
def test_oracle_matches_reference_naive(body, int_valued):
    text = {"gemm": po.preset_source("matmul"), "discount": po.preset_source("q1"),
            "boost": po.preset_source("q2"), "thrcount": po.preset_source("q3"),
            "sqdiff": po.SQDIFF_TEXT, "eqcount": po.EQCOUNT_TEXT}[body]
    for (M, K, N) in [(13, 17, 21), (32, 24, 40), (5, 1, 7)]:
        t = po.RefTask.create(text, M, K, N, seed=7, int_valued=int_valued)
        A, B = t.get("A"), t.get("B")
        th = t.get("thres")[:, 0] if "thres" in t.names() else None
        ds = t.get("dis")[:, 0] if "dis" in t.names() else None
        R = np.zeros((M, N))
        if body == "thrcount":
            po.oracle_run(po.THRCOUNT, A, B, R, thres=100.0, thres_form="c")
        else:
            po.oracle_run(BODY_KIND[body], A, B, R, thres=th, dis=ds)
        t.run_naive()
        assert np.array_equal(R, t.get("R")), f"{body} {M}x{K}x{N}"


@needs_ref
@pytest.mark.parametrize("preset", ["q1-tj-atb", "q1-tj-abt", "q2-tj-atbt", "matmul-atb",
                                    "q1-tc", "q2-ti", "q1-tij"])
def test_oracle_orientations_and_threshold_forms(preset):
    """Transposed operands and -tc/-ti/-tij thresholds through strides."""
    src = po.preset_source(preset)
    M, K, N = 11, 9, 13
    t = po.RefTask.create(src, M, K, N, seed=3, int_valued=True)
    at, bt = "-atb" in preset or "-atbt" in preset, "-abt" in preset or "-atbt" in preset
    A = t.get("A").T if at else t.get("A")
    B = t.get("B").T if bt else t.get("B")
    form = "tc" if "-tc" in preset else "ti" if "-ti" in preset and "-tij" not in preset else \
        "tij" if "-tij" in preset else "tj"
    kind = po.DISCOUNT if preset.startswith("q1") else po.BOOST if preset.startswith("q2") else po.GEMM
    thres = None
    tf = "j"
    if kind != po.GEMM:
        if form == "tc":
            thres, tf = 100.0, "c"
        elif form == "ti":
            thres, tf = t.get("thres")[:, 0], "i"
        elif form == "tij":
            thres, tf = t.get("thres"), "ij"
        else:
            thres = t.get("thres")[:, 0]
    dis = t.get("dis")[:, 0] if "dis" in t.names() else None
    R = np.zeros((M, N))
    po.oracle_run(kind, A, B, R, thres=thres, dis=dis, thres_form=tf)
    t.run_naive()
    assert np.array_equal(R, t.get("R"))


@needs_ref
def test_reference_adaptive_equals_naive_int():
    """The reference's own tiled executor == its naive oracle on int data
    (acceptance c3), which is what makes int-valued parity bit-exact."""
    t = po.RefTask.create(po.preset_source("q1"), 64, 64, 64, seed=1, int_valued=True)
    t2 = po.RefTask.create(po.preset_source("q1"), 64, 64, 64, seed=1, int_valued=True)
    t.run_naive()
    t2.run_adaptive()
    assert np.array_equal(t.get("R"), t2.get("R"))


@pytest.mark.parametrize("body", sorted(BODY_KIND))
def test_oracle_matches_goldens(body):
    for case in load_golden(body):
        if "thres_const" in case:
            R = np.zeros_like(case["R"])
            po.oracle_run(BODY_KIND[body], case["A"], case["B"], R, thres=case["thres_const"],
                          thres_form="c")
        else:
            R = oracle(body, case["A"], case["B"], case.get("thres"), case.get("dis"))
        assert np.array_equal(R, case["R"]), case["name"]


def test_oracle_bounds_and_assignment():
    rng = np.random.default_rng(0)
    A = rng.integers(-8, 9, (9, 7)).astype(float)
    B = rng.integers(-8, 9, (7, 6)).astype(float)
    R0 = rng.integers(-5, 5, (9, 6)).astype(float)
    R = R0.copy()
    po.oracle_run(po.GEMM, A, B, R, bounds=(2, 5, 1, 4, 3, 6))
    want = R0.copy()
    want[2:5, 1:4] += A[2:5, 3:6] @ B[3:6, 1:4]
    assert np.array_equal(R, want)
    R = R0.copy()
    po.oracle_run(po.GEMM, A, B, R, accumulate=False)
    assert np.array_equal(R, np.outer(A[:, -1], B[-1, :]))
