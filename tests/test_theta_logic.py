"""CPU: the claim behind the theta-form discount (csrc/theta_discount.cu),
restated in numpy and checked on adversarial samples.

For b > 0, rn(x * b) is nondecreasing in x, so the mask rn(a b) > t holds
exactly for a > theta with theta = max{x : rn(x b) <= t}; for b < 0 it is
nonincreasing and the mask is !(a > theta) with theta = max{x : rn(x b) > t}.
theta is found by a short nextafter walk from t / b and, failing that, a
bisection over the order-preserving int64 keys of the doubles — the same
search the prep kernel runs. The kernel itself is covered on the GPU by
tests/test_gpu_theta.py."""
from __future__ import annotations

import numpy as np

INF = np.inf


def okey(x: float) -> int:
    b = int(np.array(x, dtype=np.float64).view(np.int64))
    return b ^ ((b >> 63) & 0x7FFFFFFFFFFFFFFF)


def odec(k: int) -> float:
    b = k ^ ((k >> 63) & 0x7FFFFFFFFFFFFFFF)
    return float(np.array(b, dtype=np.int64).view(np.float64))


def pred(x: float, b: float, t: float) -> bool:
    y = float(np.float64(x) * np.float64(b))
    return y <= t if b > 0 else y > t


def theta_of(b: float, t: float) -> float:
    """max{x : pred(x)} for finite t and finite nonzero b (pred(-inf) holds)."""
    with np.errstate(all="ignore"):  # nextafter past DBL_MAX is inf: intended
        return _theta_of(b, t)


def _theta_of(b: float, t: float) -> float:
    with np.errstate(all="ignore"):
        x = float(np.float64(t) / np.float64(b))
    if x != x:
        x = 0.0
    for _ in range(8):
        if not pred(x, b, t):
            x = float(np.nextafter(x, -INF))
            continue
        up = float(np.nextafter(x, INF))
        if not pred(up, b, t):
            return x
        x = up
    lo, hi = okey(-INF), okey(INF)
    while hi - lo > 1:
        mid = lo + (hi - lo) // 2
        if pred(odec(mid), b, t):
            lo = mid
        else:
            hi = mid
    return odec(lo)


def mask_theta(a: float, b: float, theta: float) -> bool:
    return (a > theta) if b > 0 else not (a > theta)


def mask_ref(a: float, b: float, t: float) -> bool:
    return float(np.float64(a) * np.float64(b)) > t


def test_mask_exact_on_ties_and_neighbours():
    """a, b, t chosen so that a * b lands on t, and a one ulp either side."""
    rng = np.random.default_rng(11)
    for _ in range(400):
        b = float(rng.uniform(1, 100)) * (1 if rng.random() < 0.7 else -1)
        a0 = float(rng.integers(0, 10))
        t = float(np.float64(a0) * np.float64(b))  # a product exactly on the threshold
        th = theta_of(b, t)
        for a in (a0, float(np.nextafter(a0, INF)), float(np.nextafter(a0, -INF)), a0 + 1, a0 - 1):
            assert mask_theta(a, b, th) == mask_ref(a, b, t), (a, b, t, th)


def test_mask_exact_on_random_reals():
    rng = np.random.default_rng(12)
    for _ in range(300):
        b = float(rng.standard_normal() * 10 ** rng.uniform(-3, 3))
        t = float(rng.standard_normal() * 10 ** rng.uniform(-3, 3))
        if b == 0:
            continue
        th = theta_of(b, t)
        for a in rng.standard_normal(20) * 10 ** rng.uniform(-3, 3):
            a = float(a)
            assert mask_theta(a, b, th) == mask_ref(a, b, t), (a, b, t, th)
        # and right at theta and its neighbours
        for a in (th, float(np.nextafter(th, INF)), float(np.nextafter(th, -INF))):
            assert mask_theta(a, b, th) == mask_ref(a, b, t), (a, b, t, th)


def test_far_start_falls_back_to_bisection():
    """t / b far from theta (huge ratios): the walk gives up after 8 steps and
    the bisection still lands on the exact boundary."""
    for b, t in ((1e-300, 1e300), (3.0, 1e308), (-7.5, -1e-310), (1e300, 1e-300)):
        th = theta_of(b, t)
        with np.errstate(all="ignore"):
            assert pred(th, b, t) and not pred(float(np.nextafter(th, INF)), b, t)
