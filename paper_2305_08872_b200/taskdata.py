"""Task-level API over the GPU engine, with the reference engine's names
(src/engine.cpp:104-216, include/amlt/engine.hpp):

* ``bind_dims(task, M, K, N)``      loop extents -> (Bounds, (M, K, N))
* ``make_task_data(task, ...)``     every array the task names, generated with
                                    the reference's seeded generator straight
                                    into the kernel dtype (host or device)
* ``load_operand_file(data, ...)``  an AMLT matrix file in place of A or B
* ``verify_against_naive(...)``     the result against the per-element device
                                    executor: exact / max abs / max rel / pass
                                    (pass = exact on IntValued data, rel <= the
                                    dtype's bound on Real data; engine.cpp:186-210)

so a caller of the reference's ``compile_task -> bind_dims -> make_task_data ->
run_adaptive -> verify_against_naive`` sequence finds the same steps here.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, Optional, Tuple

from . import _native as N
from . import engine as E
from . import matrix_io as io
from .task import TaskPlan

TOLERANCE = {"f64": 1e-12, "f32": 1e-5, "i32": 0.0}


def bind_dims(task: TaskPlan, M: int, K: int, N_: int) -> Tuple[E.Bounds, Tuple[int, int, int]]:
    """bind_dims (src/engine.cpp:104-126): numeric range ends are fixed, named
    ends bind to M (the i loop), K (k) and N (j); one name bound to two values
    is an error."""
    bound: Dict[str, int] = {}
    out = []
    for end, value in zip(task.dims, (M, K, N_)):
        try:
            out.append(int(float(end)))
            continue
        except ValueError:
            pass
        if end in bound and bound[end] != value:
            raise E.EngineError(f"conflicting values for dimension '{end}': {bound[end]} vs {value}")
        bound[end] = value
        out.append(value)
    m, k, n = out
    return E.Bounds(0, m, 0, n, 0, k), (m, k, n)


@dataclass
class TaskData:
    """TaskData (engine.hpp:50-57): the task's arrays by name, R among them."""
    task: TaskPlan
    arrays: Dict[str, object] = field(default_factory=dict)
    dtype: str = "f64"

    @property
    def result_name(self) -> str:
        return self.task.result_name

    def result(self):
        return self.arrays[self.task.result_name]

    def operands(self, R=None) -> E.Operands:
        """make_operands (engine.cpp:153-163), optionally with another R."""
        arrays = dict(self.arrays)
        if R is not None:
            arrays[self.task.result_name] = R
        return E.operands_of(self.task, arrays)


def _shape_of(task: TaskPlan, name: str, M: int, K: int, N_: int, cls: Optional[int] = None):
    if name == task.a_name:
        return (K, M) if task.layout_a == N.LAYOUT_TRANSPOSED else (M, K)
    if name == task.b_name:
        return (N_, K) if task.layout_b == N.LAYOUT_TRANSPOSED else (K, N_)
    return {N.LEAF_CONSTANT: (1, 1), N.LEAF_VEC_I: (M, 1), N.LEAF_VEC_J: (N_, 1),
            N.LEAF_MAT_IJ: (M, N_)}[cls]


def make_task_data(task: TaskPlan, M: int, K: int, N_: int, seed: int = 1,
                   order_a: int = io.ROW_MAJOR, order_b: int = io.ROW_MAJOR,
                   mode: int = io.INT_VALUED, dtype: str = "f64", device=None) -> TaskData:
    """make_task_data (src/engine.cpp:128-151): each array from gen_matrix
    with the per-name seed seed ^ fnv1a(name) (bit-identical to the
    reference's buffers), A and B in the requested storage orders, R zero.
    device None gives host numpy arrays, else CUDA tensors."""
    if dtype == "i32" and mode == io.REAL:
        raise E.EngineError("i32 data needs the IntValued mode")
    _, (M, K, N_) = bind_dims(task, M, K, N_)
    data = TaskData(task, {}, dtype)

    def gen(name, shape, order):
        return io.gen_operand(seed, name, shape[0], shape[1], order, mode, dtype, device)

    data.arrays[task.a_name] = gen(task.a_name, _shape_of(task, task.a_name, M, K, N_), order_a)
    data.arrays[task.b_name] = gen(task.b_name, _shape_of(task, task.b_name, M, K, N_), order_b)
    if task.thres_name:
        data.arrays[task.thres_name] = gen(task.thres_name, _shape_of(task, task.thres_name, M, K, N_,
                                                                      task.thres_class), io.ROW_MAJOR)
    if task.dis_name:
        data.arrays[task.dis_name] = gen(task.dis_name, (N_, 1), io.ROW_MAJOR)
    for name, cls in zip(task.aux_names, task.aux_classes):
        data.arrays[name] = gen(name, _shape_of(task, name, M, K, N_, cls), io.ROW_MAJOR)
    if device is None:
        import numpy as np
        R = np.zeros((M, N_), dtype={"f64": np.float64, "f32": np.float32, "i32": np.int32}[dtype])
    else:
        import torch
        R = torch.zeros((M, N_), dtype={"f64": torch.float64, "f32": torch.float32,
                                        "i32": torch.int32}[dtype], device=device)
    data.arrays[task.result_name] = R
    return data


def load_operand_file(data: TaskData, name: str, path: str, device=None) -> None:
    """load_operand_file (amlt_main.cpp:117-128): an AMLT matrix file replaces
    the named array; its shape must match."""
    if name not in data.arrays:
        raise E.EngineError(f"task has no operand named {name}")
    cur = data.arrays[name]
    rows, cols = (int(v) for v in cur.shape)
    info = io.matrix_file_info(path)
    if (info.rows, info.cols) != (rows, cols):
        raise E.EngineError(f"operand file {path} is {info.rows}x{info.cols}, task needs {rows}x{cols}")
    data.arrays[name] = io.read_matrix_file(path, data.dtype, device)


@dataclass
class VerifyResult:
    """VerifyResult (engine.hpp): exact, max abs / rel error, pass."""
    exact: bool
    max_abs_err: float
    max_rel_err: float
    passed: bool


def verify_against_naive(plan: E.GpuPlan, data: TaskData, bounds: E.Bounds,
                         mode: int = io.INT_VALUED) -> VerifyResult:
    """verify_against_naive (src/engine.cpp:186-210) with the per-element
    device executor (amlt_gpu_run_naive) as the naive side: pass = exact on
    IntValued data, max rel <= TOLERANCE[dtype] on Real data."""
    import torch
    got = data.result()
    scratch = torch.zeros_like(got)
    E.run_naive(plan, data.operands(scratch), bounds)
    g, w = got.double(), scratch.double()
    err = (g - w).abs()
    mag = torch.maximum(g.abs(), w.abs())
    rel = torch.where(mag > 0, err / torch.where(mag > 0, mag, torch.ones_like(mag)),
                      torch.zeros_like(mag))
    exact = bool(torch.equal(g, w))
    max_abs = float(err.max()) if err.numel() else 0.0
    max_rel = float(rel.max()) if rel.numel() else 0.0
    ok = exact if mode == io.INT_VALUED else (exact or max_rel <= TOLERANCE[data.dtype])
    return VerifyResult(exact, max_abs, max_rel, ok)
