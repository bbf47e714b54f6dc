"""The task-level API (taskdata.py): bind_dims / make_task_data with the
reference's names, checked against the unmodified reference engine's own
make_task_data buffers (CPU), and verify_against_naive on the GPU."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2305_08872_b200 as P
from paper_2305_08872_b200 import matrix_io as io
from oracle import pyoracle as po

HEAD = "where(i in [0..M] and j in [0..N] and k in [0..K]) {\n  R[i][j] += "


@pytest.mark.skipif(not po.ref_available(), reason="reference engine not built")
@pytest.mark.parametrize("src,oa,ob,mode", [
    (P.task.preset_source("q1"), 0, 0, io.INT_VALUED),
    (P.task.preset_source("q2-tij-atb"), 1, 0, io.REAL),
    (P.task.preset_source("q3-ti-abt"), 0, 1, io.INT_VALUED),
    (HEAD + "A[i][k]*B[k][j] + u[i]*v[j] - (A[i][k] > s)*W[i][j];\n}\n", 1, 1, io.REAL),
])
def test_make_task_data_matches_reference(src, oa, ob, mode):
    t = P.compile_task(src)
    data = P.make_task_data(t, 13, 7, 17, seed=3, order_a=oa, order_b=ob, mode=mode)
    ref = po.RefTask.create(src, 13, 7, 17, seed=3, int_valued=mode == io.INT_VALUED,
                            order_a=oa, order_b=ob)
    for name in ref.names():
        want = ref.get(name)
        got = np.asarray(data.arrays[name], dtype=np.float64).reshape(want.shape)
        if name == t.result_name:
            assert not got.any()
            continue
        assert np.array_equal(got, want), name
    b, dims = P.bind_dims(t, 13, 7, 17)
    assert dims == (13, 7, 17) and (b.i1, b.j1, b.k1) == (13, 17, 7)


def test_bind_dims_numeric_and_conflicting_ends():
    t = P.compile_task("where(i in [0..64] and j in [0..N] and k in [0..N]) {\n"
                       "  R[i][j] += A[i][k]*B[k][j];\n}\n")
    b, dims = P.bind_dims(t, 5, 9, 9)
    assert dims == (64, 9, 9)
    with pytest.raises(P.EngineError, match="conflicting"):
        P.bind_dims(t, 5, 8, 9)


@pytest.mark.gpu
@pytest.mark.parametrize("preset,mode,dtype", [("q1", io.INT_VALUED, "f64"), ("q2", io.REAL, "f64"),
                                               ("matmul", io.REAL, "f32")])
def test_reference_sequence_on_the_gpu(gpu_ctx, preset, mode, dtype):
    """compile_task -> bind_dims -> make_task_data -> run_adaptive ->
    verify_against_naive, the reference engine's sequence, on the device."""
    t = P.compile_task(P.task.preset_source(preset))
    data = P.make_task_data(t, 300, 200, 260, seed=1, mode=mode, dtype=dtype, device="cuda:0")
    b, _ = P.bind_dims(t, 300, 200, 260)
    plan = gpu_ctx.plan_for(t, dtype)
    P.run_adaptive(plan, data.operands(), b)
    v = P.verify_against_naive(plan, data, b, mode)
    assert v.passed, v
    if mode == io.INT_VALUED:
        assert v.exact
