"""Shared test helpers: seeded inputs (reference int-valued convention and the
BASELINE.json distributions), oracle evaluation, tolerance checks."""
from __future__ import annotations

import numpy as np

from oracle import pyoracle as po

BODY_KIND = {"gemm": po.GEMM, "discount": po.DISCOUNT, "boost": po.BOOST, "sqdiff": po.SQDIFF,
             "eqcount": po.EQCOUNT, "thrcount": po.THRCOUNT}
NP_DT = {"f64": np.float64, "f32": np.float32, "i32": np.int32}
# rel tolerances stated by BASELINE.json north_star (vs an fp64 oracle)
TOL = {"f64": 1e-12, "f32": 1e-5, "i32": 0.0}
# acceptance-suite dims (M, K, N), reference tests/acceptance.cpp:109-110
ACCEPT_DIMS = [(64, 64, 64), (96, 128, 160), (257, 129, 65), (13, 17, 5)]


def int_valued(rng, shape):
    """The reference's IntValued convention: integers in [-8, 8]
    (matrix.hpp:63-66). Every product/partial sum is then exact."""
    return rng.integers(-8, 9, shape).astype(np.float64)


def make_inputs(body, M, K, N, dist="int", seed=1):
    """float64 inputs for one body. dist: 'int' (reference convention) or
    'baseline' (BASELINE.json configs)."""
    rng = np.random.default_rng(seed)
    thres = dis = None
    if dist == "int":
        A, B = int_valued(rng, (M, K)), int_valued(rng, (K, N))
        if body in ("discount", "boost", "thrcount"):
            thres = int_valued(rng, N)
        if body == "discount":
            dis = int_valued(rng, N)
        return A, B, thres, dis
    if body == "discount":  # config 0 / 4
        A = rng.integers(0, 10, (M, K)).astype(np.float64)
        B = rng.uniform(1, 100, (K, N))
        thres = rng.uniform(50, 450, N)
        dis = rng.uniform(0, 0.3, N)
    elif body == "boost":  # config 1
        A, B = rng.uniform(0, 1, (M, K)), rng.uniform(0, 1, (K, N))
        thres = rng.uniform(0.25, 0.75, N)
    elif body == "gemm":  # config 2
        A, B = rng.standard_normal((M, K)), rng.standard_normal((K, N))
    elif body == "sqdiff":  # config 3a
        A, B = rng.uniform(-1, 1, (M, K)), rng.uniform(-1, 1, (K, N))
    elif body == "eqcount":  # config 3b
        A = rng.integers(0, 16, (M, K)).astype(np.float64)
        B = rng.integers(0, 16, (K, N)).astype(np.float64)
    elif body == "thrcount":
        A, B = rng.uniform(0, 20, (M, K)), rng.uniform(0, 20, (K, N))
        thres = rng.uniform(50, 150, N)
    return A, B, thres, dis


def cast(x, dtype):
    """Rounds inputs to the kernel dtype; the oracle then sees the same values
    upcast exactly to double (BASELINE: fp32/int32 parity vs the fp64 oracle)."""
    if x is None:
        return None
    return x.astype(NP_DT[dtype]).astype(np.float64)


def oracle(body, A, B, thres=None, dis=None, R0=None, bounds=None, accumulate=True):
    M, N = A.shape[0], B.shape[1]
    R = np.zeros((M, N)) if R0 is None else R0.astype(np.float64).copy()
    po.oracle_run(BODY_KIND[body], A, B, R, thres=thres, dis=dis, bounds=bounds,
                  accumulate=accumulate)
    return R


def normwise_bound(body, A, B, thres=None):
    """sum_k |term_k| per output: the scale for normwise fp tolerance (needed
    for GEMM on N(0,1) data)."""
    if body == "gemm":
        return np.abs(A) @ np.abs(B)
    if body == "sqdiff":
        return (A * A) @ np.ones_like(B) + np.ones_like(A) @ (B * B) + 2 * np.abs(A) @ np.abs(B)
    return None


def check(body, dtype, got, want, A=None, B=None, exact=False, what=""):
    got = np.asarray(got, dtype=np.float64)
    if exact or dtype == "i32" or body in ("eqcount", "thrcount"):
        bad = np.argwhere(got != want)
        assert bad.size == 0, (f"{what}: {len(bad)} mismatches, first at {tuple(bad[0])}: "
                               f"got {got[tuple(bad[0])]!r} want {want[tuple(bad[0])]!r}")
        return 0.0
    tol = TOL[dtype]
    err = np.abs(got - want)
    scale = np.abs(want)
    if body == "gemm":
        scale = normwise_bound(body, A, B)
    rel = err / np.maximum(scale, np.finfo(np.float64).tiny)
    worst = float(rel.max()) if rel.size else 0.0
    assert worst <= tol, f"{what}: max rel err {worst:.3e} > {tol:.0e}"
    return worst
