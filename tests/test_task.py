"""CPU: the task front-end recognises exactly the GPU bodies.

Restates the reference's recognition conditions (recognize.cpp:84-166) and
checks the body match against the reference's own preset texts
(presets.cpp:52-94) and recognition verdicts (oracle/_ref).
"""
from __future__ import annotations

import pytest

import paper_2305_08872_b200 as P
from paper_2305_08872_b200 import _native as N
from paper_2305_08872_b200.task import TaskError, compile_task
from oracle import pyoracle as po

WRAP = "where(i in [0..M] and j in [0..N] and k in [0..K]) {{\n  R[i][j] {op} {rhs};\n}}\n"


def wrap(rhs, op="+="):
    return WRAP.format(op=op, rhs=rhs)


@pytest.mark.parametrize("rhs,body", [
    ("A[i][k]*B[k][j]", "gemm"),
    ("B[k][j]*A[i][k]", "gemm"),
    ("A[i][k]*B[k][j] - (A[i][k]*B[k][j] > thres[j])*A[i][k]*B[k][j]*dis[j]", "discount"),
    ("A[i][k]*B[k][j] + (A[i][k]*B[k][j] > thres[j])*(A[i][k]*B[k][j] - thres[j])", "boost"),
    ("(A[i][k] - B[k][j])*(A[i][k] - B[k][j])", "sqdiff"),
    ("A[i][k] == B[k][j]", "eqcount"),
    ("B[k][j] == A[i][k]", "eqcount"),
    ("(A[i][k]*B[k][j] > 100)", "thrcount"),
])
def test_bodies_recognised(rhs, body):
    t = compile_task(wrap(rhs))
    assert t.body_name == body
    assert t.a_name == "A" and t.b_name == "B" and t.result_name == "R"
    assert t.accumulate


def test_roles_and_forms():
    t = compile_task(wrap("A[i][k]*B[k][j] - (A[i][k]*B[k][j] > thres[j])*A[i][k]*B[k][j]*dis[j]"))
    assert (t.thres_name, t.dis_name, t.thres_class) == ("thres", "dis", N.LEAF_VEC_J)
    t = compile_task(wrap("(A[i][k]*B[k][j] > 100)"))
    assert t.thres_class == N.LEAF_CONSTANT and t.thres_value == 100.0
    t = compile_task(wrap("A[k][i]*B[j][k]"))
    assert (t.layout_a, t.layout_b) == (N.LAYOUT_TRANSPOSED, N.LAYOUT_TRANSPOSED)
    t = compile_task(wrap("A[i][k]*B[k][j]", "="))
    assert not t.accumulate
    # roles follow the target's subscripts, not loop declaration order
    t = compile_task("where(k in [0..K] and j in [0..N] and i in [0..M]) {\n"
                     "  R[i][j] += X[i][k]*Y[k][j];\n}\n")
    assert (t.a_name, t.b_name, t.var_k) == ("X", "Y", "k")
    # comments
    t = compile_task("// a comment\n" + wrap("A[i][k]*B[k][j]"))
    assert t.body_name == "gemm"


@pytest.mark.parametrize("rhs,aux", [
    ("A[i][k]*B[k][j] + u[i]*v[j]", (("u", N.LEAF_VEC_I), ("v", N.LEAF_VEC_J))),
    ("A[i][k]*B[k][j]*s + u[i] - v[j]*W[i][j]",
     (("s", N.LEAF_CONSTANT), ("u", N.LEAF_VEC_I), ("v", N.LEAF_VEC_J), ("W", N.LEAF_MAT_IJ))),
    ("(A[i][k] + 1)*(B[k][j] - 1)/2 + W[i][j]", (("W", N.LEAF_MAT_IJ),)),
    ("A[i][k]*B[k][j] - (A[i][k]*B[k][j] < thres[j])*A[i][k]*B[k][j]",
     (("thres", N.LEAF_VEC_J),)),
])
def test_other_mmlt_statements_get_generated_bodies(rhs, aux):
    """Recognised MMLT statements outside the six bodies (recognize.cpp:
    84-166) plan a generated body; aux leaves in first-use order."""
    t = compile_task(wrap(rhs))
    assert t.body == N.BODY_GENERIC and t.body_name == "generic"
    assert tuple(zip(t.aux_names, t.aux_classes)) == aux
    assert (t.a_name, t.b_name) == ("A", "B")


@pytest.mark.parametrize("rhs", [
    "A[i][k]*C[k][j]*B[k][j]",               # two k-indexed B-role arrays
    "A[i][k]*u[k]",                          # u[k] does not fit the pattern
    "A[i][k]*B[k][j]*W[j][i]",               # W[j][i] does not fit the pattern
])
def test_non_mmlt_statements_are_unsupported(rhs):
    with pytest.raises(P.UnsupportedExpression):
        compile_task(wrap(rhs))


def test_not_mmlt():
    with pytest.raises(P.UnsupportedExpression):
        compile_task("where(i in [0..M] and j in [0..N]) {\n  R[i][j] += A[i][j];\n}\n")
    with pytest.raises(P.UnsupportedExpression):
        compile_task(wrap("R[i][j]*A[i][k]*B[k][j]"))
    with pytest.raises(TaskError):
        compile_task("where(i in [0..M] {")


@pytest.mark.skipif(not po.ref_available(), reason="reference engine not built")
def test_reference_presets():
    """Every reference preset the reference recognises as an MMLT: q1/q2
    (any threshold form, any orientation), matmul and q3 map to their body;
    the reference and we agree on the operand roles."""
    names = (["matmul-" + o for o in ("ab", "atb", "abt", "atbt")]
             + [f"{q}-{f}-{o}" for q in ("q1", "q2", "q3") for f in ("tc", "ti", "tj", "tij")
                for o in ("ab", "atb", "abt", "atbt")])
    assert len(names) == 52
    want_body = {"matmul": "gemm", "q1": "discount", "q2": "boost", "q3": "thrcount"}
    for name in names:
        src = po.preset_source(name)
        t = compile_task(src)
        assert t.body_name == want_body[name.split("-")[0]], name
        ref = po.RefTask.create(src, 4, 4, 4)
        assert ref.is_mmlt()
        a, b, aux = ref.roles()
        assert (t.a_name, t.b_name) == (a, b)
        form = name.split("-")[1] if not name.startswith("matmul") else None
        if form:
            want_cls = {"tc": N.LEAF_CONSTANT, "ti": N.LEAF_VEC_I, "tj": N.LEAF_VEC_J,
                        "tij": N.LEAF_MAT_IJ}[form]
            assert t.thres_class == want_cls, name
        assert t.layout_a == (N.LAYOUT_TRANSPOSED if "-at" in name else N.LAYOUT_NORMAL)
        assert t.layout_b == (N.LAYOUT_TRANSPOSED if name.endswith("bt") else N.LAYOUT_NORMAL)


def native_recognize(src):
    import ctypes as C

    info = N.TaskInfoC()
    st = N.lib().amlt_gpu_recognize(src.encode(), C.byref(info))
    return st, info


CASES = [
    "A[i][k]*B[k][j]", "B[k][j]*A[i][k]", "A[k][i]*B[j][k]",
    "A[i][k]*B[k][j] - (A[i][k]*B[k][j] > thres[j])*A[i][k]*B[k][j]*dis[j]",
    "A[i][k]*B[k][j] + (A[i][k]*B[k][j] > thres[j])*(A[i][k]*B[k][j] - thres[j])",
    "A[i][k]*B[k][j] + (A[i][k]*B[k][j] > s)*(A[i][k]*B[k][j] - s)",
    "(A[i][k] - B[k][j])*(A[i][k] - B[k][j])", "A[i][k] == B[k][j]", "(A[i][k]*B[k][j] > 100)",
    "A[i][k]*B[k][j] + u[i]*v[j]", "A[i][k]*u[k]", "A[i][k]*C[k][j]*B[k][j]",
    "A[i][k]*B[k][j] - (A[i][k]*B[k][j] < thres[j])*A[i][k]*B[k][j]",
]


@pytest.mark.parametrize("rhs", CASES)
@pytest.mark.parametrize("op", ["+=", "="])
def test_native_recognizer_agrees_with_python(rhs, op):
    src = wrap(rhs, op)
    st, info = native_recognize(src)
    try:
        t = compile_task(src)
    except P.UnsupportedExpression:
        assert st == N.ERR_UNSUPPORTED
        return
    assert st == N.OK, N.lib().amlt_gpu_last_error(None)
    d = info.desc
    assert (d.body, d.accumulate, d.layout_a, d.layout_b, d.thres_class) == \
        (t.body, int(t.accumulate), t.layout_a, t.layout_b, t.thres_class)
    assert d.thres_value == t.thres_value
    assert (info.a.decode(), info.b.decode(), info.r.decode()) == (t.a_name, t.b_name, t.result_name)
    assert info.thres.decode() == (t.thres_name or "") and info.dis.decode() == (t.dis_name or "")


def test_native_recognizer_parse_error():
    st, _ = native_recognize("where(i in [0..M] {")
    assert st == N.ERR_ENGINE
    assert b"parse error" in N.lib().amlt_gpu_last_error(None)


# ---------------------------------------------------------------------------
# canonical matching: a fixed body written differently still
# runs its fused kernel; the reference DAG normalises the same way
# (expr_dag.cpp:182-245)

@pytest.mark.parametrize("rhs,body", [
    # q1 with the comparison reversed, the mask factor moved, re-associated
    ("A[i][k]*B[k][j] - (thres[j] < A[i][k]*B[k][j])*A[i][k]*B[k][j]*dis[j]", "discount"),
    ("A[i][k]*B[k][j] - A[i][k]*B[k][j]*dis[j]*(A[i][k]*B[k][j] > thres[j])", "discount"),
    ("B[k][j]*A[i][k] - dis[j]*(B[k][j]*A[i][k] > thres[j])*(A[i][k]*B[k][j])", "discount"),
    # q2 with the terms swapped and the comparison reversed
    ("(thres[j] < A[i][k]*B[k][j])*(A[i][k]*B[k][j] - thres[j]) + A[i][k]*B[k][j]", "boost"),
    ("100 < A[i][k]*B[k][j]", "thrcount"),
])
def test_canonical_forms_hit_fixed_bodies(rhs, body):
    assert compile_task(wrap(rhs)).body_name == body


@pytest.mark.parametrize("rhs", [
    "A[i][k]*B[k][j] - (A[i][k]*B[k][j] >= thres[j])*A[i][k]*B[k][j]*dis[j]",  # >= is not >
    "A[i][k]*B[k][j] + (A[i][k]*B[k][j] > thres[j])*A[i][k]*B[k][j]*dis[j]",  # + is not -
    "A[i][k]*B[k][j] - (A[i][k] > thres[j])*A[i][k]*B[k][j]*dis[j]",          # mask of A alone
    "(B[k][j] - A[i][k])*(A[i][k] - B[k][j])",
])
def test_near_misses_stay_generic(rhs):
    assert compile_task(wrap(rhs)).body == N.BODY_GENERIC


# ---------------------------------------------------------------------------
# the reference program's op counts (SURVEY §8(d) measure (B)), pinned
# against the unmodified reference's schedule_labelfs output

def _ref_program_counts(src):
    t = po.RefTask.create(src, 4, 4, 4)
    counts = {}
    for ln in t.program():
        op = ln.split()[0]
        counts[op] = counts.get(op, 0) + 1
    return counts


def _program_sources():
    srcs = [P.task.preset_source(n) for n in P.task.preset_names()]
    srcs += [wrap("(A[i][k] - B[k][j])*(A[i][k] - B[k][j])"), wrap("A[i][k] == B[k][j]"),
             wrap("A[i][k]*B[k][j] - (thres[j] < A[i][k]*B[k][j])*A[i][k]*B[k][j]*dis[j]"),
             wrap("A[i][k]*B[k][j] + u[i]*v[j]"), wrap("(A[i][k] + 1)*(B[k][j] - 1)/2 + W[i][j]"),
             wrap("A[i][k]*B[k][j]*s + u[i] - v[j]*W[i][j]"),
             wrap("(A[i][k] > v[j])*(B[k][j] + 2) - (A[i][k] < 1)*u[i] + 3"),
             wrap("A[i][k]*B[k][j]", "=")]
    return srcs


@pytest.mark.skipif(not po.ref_available(), reason="reference engine not built")
@pytest.mark.parametrize("src", _program_sources())
def test_program_op_counts_match_the_reference(src):
    t = compile_task(src)
    assert t.program == _ref_program_counts(src)


def test_body_op_flops_of_the_five_bodies():
    """(B) per SURVEY §8(d): discount / boost 6, gemm 2, sqdiff 3, eqcount 4."""
    flops = {"q1": 6, "q2": 6, "matmul": 2}
    for name, want in flops.items():
        assert compile_task(P.task.preset_source(name)).program_flops == want
    assert compile_task(wrap("(A[i][k] - B[k][j])*(A[i][k] - B[k][j])")).program_flops == 3
    assert compile_task(wrap("A[i][k] == B[k][j]")).program_flops == 4
