"""Generated bodies (AMLT_BODY_GENERIC): recognised statements outside the
six fixed bodies, compiled at plan time by NVRTC into the tile kernels.

Parity follows the reference's own strategy for arbitrary statements
(tests/test_engine.cpp:377-398 "adaptive and naive agree across random
statements and layouts"; tests/test_exec.cpp:269-285): random statements
over A, B, u[i], v[j], W[i][j], a scalar s and small constants with + - *
/2^n and comparisons, on the reference's IntValued data, must match the
UNMODIFIED reference's run_naive bit for bit (oracle/_ref, driven through
oracle/ref_shim.cpp). CPU cases check recognition, the generated source and
that NVRTC compiles it for sm_100a (no device needed).
"""
from __future__ import annotations

import random

import numpy as np
import pytest

import paper_2305_08872_b200 as P
from paper_2305_08872_b200 import _native as N
from oracle import pyoracle as po

HEAD = "where(i in [0..M] and j in [0..N] and k in [0..K]) {\n  R[i][j] "


def random_statement(rng: random.Random):
    """A random recognised statement (own generator; the shape of the
    reference's TaskGen: a product core plus a random subtree)."""
    at, bt = rng.random() < 0.3, rng.random() < 0.3
    A = "A[k][i]" if at else "A[i][k]"
    B = "B[j][k]" if bt else "B[k][j]"

    def leaf():
        return rng.choice([A, B, "u[i]", "v[j]", "W[i][j]", "s", str(rng.randrange(7))])

    def sub(d):
        if d >= 3 or rng.random() < 0.35:
            return leaf()
        lhs = sub(d + 1)
        if rng.random() < 0.1:
            return f"({lhs})/{2 << rng.randrange(3)}"
        ops = [" + ", " - ", "*", " > ", " >= ", " < ", " <= ", " == "]
        op = ops[rng.randrange(8 if rng.random() < 0.25 else 3)]
        return f"({lhs}){op}({sub(d + 1)})"

    core = f"{A}*{B}"
    rhs = core if rng.random() < 0.2 else core + rng.choice([" + ", " - "]) + "(" + sub(0) + ")"
    op = "+=" if rng.random() < 0.9 else "="
    return HEAD + f"{op} {rhs};\n}}\n"


def test_generated_bodies_compile_for_sm100a_without_a_device(dry_ctx):
    """NVRTC runs on the host: plan creation in a dry-run context compiles the
    generated kernels (tile variants, '=' kernel, per-element kernel)."""
    src = HEAD + "+= A[i][k]*B[k][j] + u[i]*v[j] - (A[i][k] > s)*W[i][j]/4;\n}\n"
    plan = dry_ctx.plan_source(src, "f64")
    assert plan.body == N.BODY_GENERIC
    assert plan.aux_names == ("u", "v", "s", "W")
    assert plan.aux_classes == (N.LEAF_VEC_I, N.LEAF_VEC_J, N.LEAF_CONSTANT, N.LEAF_MAT_IJ)
    vs = plan.variants()
    assert len(vs) == 4 and all(v.name.startswith("generic_f64_") for v in vs)
    assert all(v.name.endswith(("_ti", "_u_ti")) for v in vs)  # per-output aux state
    # operand rules: every aux leaf must be bound, by position
    M, K, N_ = 16, 8, 24
    ops = P.Operands(np.zeros((M, K)), np.zeros((K, N_)), np.zeros((M, N_)),
                     aux=(np.zeros(M), np.zeros(N_), np.zeros((1, 1)), np.zeros((M, N_))))
    assert P.run_subtask(plan, ops, P.TileParams(), P.Bounds(0, M, 0, N_, 0, K),
                         clock=P.FakeClock([0.25])) == 0.25
    ops.aux = ops.aux[:3]
    with pytest.raises(P.MissingBinding):
        P.run_subtask(plan, ops, P.TileParams(), P.Bounds(0, M, 0, N_, 0, K))
    ops.aux = (np.zeros(M - 1), np.zeros(N_), np.zeros((1, 1)), np.zeros((M, N_)))
    with pytest.raises(P.EngineError):
        P.run_subtask(plan, ops, P.TileParams(), P.Bounds(0, M, 0, N_, 0, K))
    f32 = dry_ctx.plan_source(src, "f32")
    assert all(v.name.startswith("generic_f32_") for v in f32.variants())
    with pytest.raises(P.UnsupportedExpression):
        dry_ctx.plan_source(src, "i32")


def test_generated_source_is_the_statement_node_by_node():
    import ctypes as C
    src = HEAD + "+= (A[i][k] - 1)*B[k][j]/8 + (v[j] >= A[i][k]);\n}\n"
    n = N.lib().amlt_gpu_generated_source(src.encode(), N.F64, None, 0)
    assert n > 0
    buf = C.create_string_buffer(int(n) + 1)
    N.lib().amlt_gpu_generated_source(src.encode(), N.F64, buf, n + 1)
    text = buf.value.decode()
    assert "struct BodyGen" in text and "HAS_AT = false" in text
    # /8 becomes an exact multiply by 2^-3; the comparison yields 1 / 0
    assert ("add_rn(mul_rn(mul_rn(sub_rn(a, T(0x1p+0)), b), T(0x1p-3)), "
            "((c.v[0]) >= (a) ? T(1) : T(0)))") in text
    fixed = HEAD + "+= A[i][k]*B[k][j];\n}\n"
    assert N.lib().amlt_gpu_generated_source(fixed.encode(), N.F64, None, 0) == -1


@pytest.mark.parametrize("seed", range(6))
def test_random_statements_recognised_and_compiled(dry_ctx, seed):
    rng = random.Random(1000 + seed)
    src = random_statement(rng)
    t = P.compile_task(src)
    plan = dry_ctx.plan_for(t, "f64")
    if t.body == N.BODY_GENERIC:  # (a bare A*B core is the fixed GEMM body)
        assert len(plan.variants()) == 4


# ---------------------------------------------------------------- GPU cases

def _gpu_run(gpu_ctx, src, ref, adaptive=True, dtype="f64", tile=None):
    import torch
    t = P.compile_task(src)
    plan = gpu_ctx.plan_for(t, dtype)
    td = {"f64": torch.float64, "f32": torch.float32}[dtype]
    data = {}
    for name in ref.names():
        x = ref.get(name) if name != t.result_name else np.zeros_like(ref.get(name))
        data[name] = torch.from_numpy(np.ascontiguousarray(x)).to(td).cuda()
    ops = P.operands_of(t, data)
    b = P.Bounds(0, ref.M, 0, ref.N, 0, ref.K)
    if adaptive:
        P.adaptive_execute(plan, ops, b)
    else:
        P.run_subtask(plan, ops, tile or P.TileParams(), b)
    return data[t.result_name].double().cpu().numpy()


@pytest.mark.gpu
@pytest.mark.skipif(not po.ref_available(), reason="reference engine not built")
@pytest.mark.parametrize("seed", range(30))
def test_random_statements_match_reference_naive_bit_for_bit(gpu_ctx, seed):
    rng = random.Random(seed)
    src = random_statement(rng)
    M, K, N_ = 5 + rng.randrange(60), 1 + rng.randrange(70), 5 + rng.randrange(90)
    ref = po.RefTask.create(src, M, K, N_, seed=seed + 1, int_valued=True,
                            order_a=seed % 2, order_b=int(seed % 3 == 0))
    assert ref.is_mmlt()
    got = _gpu_run(gpu_ctx, src, ref, adaptive=seed % 2 == 0,
                   tile=P.TileParams(kc=32) if seed % 4 == 1 else None)
    ref.run_naive()
    want = ref.get(ref.result_name())
    bad = np.argwhere(got != want)
    assert bad.size == 0, f"{src}: {len(bad)} mismatches, first {tuple(bad[0])}: " \
                          f"{got[tuple(bad[0])]} vs {want[tuple(bad[0])]}"


@pytest.mark.gpu
@pytest.mark.skipif(not po.ref_available(), reason="reference engine not built")
def test_generated_body_real_data_and_f32(gpu_ctx):
    src = HEAD + "+= A[i][k]*B[k][j]*s + u[i] - (A[i][k] > v[j])*W[i][j]/2;\n}\n"
    M, K, N_ = 300, 257, 190
    ref = po.RefTask.create(src, M, K, N_, seed=3, int_valued=False)
    ref.run_naive()
    want = ref.get(ref.result_name())
    got = _gpu_run(gpu_ctx, src, ref)
    assert np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300)) <= 1e-12
    # f32 on int-valued data: every term and partial sum stays below 2^24,
    # so the f32 kernels are exact too
    iref = po.RefTask.create(src, M, K, N_, seed=4, int_valued=True)
    iref.run_naive()
    got32 = _gpu_run(gpu_ctx, src, iref, dtype="f32")
    assert np.array_equal(got32, iref.get(iref.result_name()))


@pytest.mark.gpu
@pytest.mark.skipif(not po.ref_available(), reason="reference engine not built")
def test_generated_body_naive_and_host_paths(gpu_ctx):
    """The per-element executor and the host-buffer entry run generated
    bodies too (aux leaves staged with the other operands)."""
    import torch
    src = HEAD + "= A[k][i]*B[k][j] - (u[i] < B[k][j])*3;\n}\n"
    M, K, N_ = 70, 33, 90
    ref = po.RefTask.create(src, M, K, N_, seed=5, int_valued=True)
    ref.run_naive()
    want = ref.get(ref.result_name())
    t = P.compile_task(src)
    plan = gpu_ctx.plan_for(t, "f64")
    host = {n: np.ascontiguousarray(ref.get(n)) for n in ref.names()}
    host[t.result_name] = np.zeros((M, N_))
    dev = {n: torch.from_numpy(x).cuda() for n, x in host.items()}
    P.run_naive(plan, P.operands_of(t, dev), P.Bounds(0, M, 0, N_, 0, K))
    assert np.array_equal(dev[t.result_name].cpu().numpy(), want)
    P.run_host(plan, P.operands_of(t, host), P.Bounds(0, M, 0, N_, 0, K))
    assert np.array_equal(host[t.result_name], want)


def test_generated_kernels_are_cached_on_disk(tmp_path):
    """A generated body compiles once per machine: the cubin lands in
    $AMLT_GPU_JIT_CACHE and later processes load it; a damaged entry is
    ignored (recompiled), and "0" disables the cache."""
    import os
    import subprocess
    import sys

    code = ("import paper_2305_08872_b200 as P\n"
            "ctx = P.Context(0, dry_run=True)\n"
            "p = ctx.plan_source('" + HEAD.replace("\n", "\\n") +
            "+= A[i][k]*B[k][j] - v[j]*(B[k][j] > 2);\\n}\\n')\n"
            "print(len(p.variants()))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

    def run(cache):
        env = dict(os.environ, AMLT_GPU_JIT_CACHE=str(cache))
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        return r.stdout.strip()

    d = tmp_path / "jit"
    assert run(d) == "4"
    files = list(d.glob("jit-*.bin"))
    assert len(files) == 1 and files[0].stat().st_size > 10000
    assert run(d) == "4"  # served from the cache
    files[0].write_bytes(files[0].read_bytes()[:100])  # damaged entry: recompiled
    assert run(d) == "4"
    assert files[0].stat().st_size > 10000
    off = tmp_path / "off"
    env_dir = off / "x"
    assert run("0") == "4" and not env_dir.exists()


@pytest.mark.gpu
@pytest.mark.skipif(not po.ref_available(), reason="reference engine not built")
@pytest.mark.parametrize("w_order", ["C", "F"])
def test_sharded_source_with_row_indexed_leaves(gpu_ctx, w_order):
    """amlt_gpu_run_sharded_source on a sub-range of rows: [i] and [i][j]
    leaves are viewed / copied from the band's first row (row-major W is
    banded like R, col-major W replicated and offset)."""
    src = HEAD + "+= A[i][k]*B[k][j] + u[i]*v[j] - (A[i][k] > s)*W[i][j]/4;\n}\n"
    M, K, N_ = 64, 40, 72
    ref = po.RefTask.create(src, M, K, N_, seed=9, int_valued=True)
    t = P.compile_task(src)
    host = {n: np.ascontiguousarray(ref.get(n)) for n in ref.names()}
    host["W"] = np.asarray(host["W"], order=w_order)
    R0 = np.arange(M * N_, dtype=np.float64).reshape(M, N_)
    host[t.result_name] = R0.copy()
    ref.set(t.result_name, R0)
    i0, i1 = 7, 50
    el = P.engine.run_sharded_source(src, P.operands_of(t, host), P.Bounds(i0, i1, 0, N_, 0, K), [0])
    assert el > 0
    ref.run_naive()
    want = ref.get(ref.result_name())
    got = host[t.result_name]
    assert np.array_equal(got[i0:i1], want[i0:i1])
    assert np.array_equal(got[:i0], R0[:i0]) and np.array_equal(got[i1:], R0[i1:])
