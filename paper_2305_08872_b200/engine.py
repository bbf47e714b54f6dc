"""Host-side mirror of the reference engine's executor/tuner interface.

Same names, argument meaning and error behaviour as the reference
(/root/reference/proj), over the B200 C-ABI (include/amlt_gpu.h):

====================================  =========================================
here                                  reference
====================================  =========================================
``compile_task(source, dtype)``       ``compile_task`` src/engine.cpp:86-102
``Bounds``, ``TileParams``            tiled_executor.hpp:11-21
``ExecRecord``, ``ExecLog``           tiled_executor.hpp:25-34
``run_subtask``                       tiled_executor.hpp:42-44
``Trial``, ``CoverRect``,             autotuner.hpp:11-34
``TuneReport``
``adaptive_execute``                  autotuner.hpp:68-70
``run_fixed``, ``run_adaptive``       engine.hpp:65-69
``spr``                               engine.hpp:83-85
``Clock``, ``SteadyClock``,           clock.hpp:12-55
``FakeClock``
``EngineError`` and subclasses        errors.hpp:10-60
====================================  =========================================

Operand buffers are torch tensors on the context's CUDA device (run_subtask,
adaptive_execute) or host numpy arrays / CPU tensors (run_host). The kernels
compute in the plan's dtype (f64, f32 or i32).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional

from . import _native as N
from .task import TaskPlan, compile_task  # noqa: F401  (re-exported)

# ---------------------------------------------------------------------------
# errors (errors.hpp:10-60)


class EngineError(RuntimeError):
    pass


class UnsupportedExpression(EngineError):
    pass


class MissingBinding(EngineError):
    pass


class NoFeasibleKernel(EngineError):
    pass


class NonPositiveTime(EngineError):
    pass


class CudaError(EngineError):
    pass


class NoDevice(EngineError):
    pass


_ERRS = {
    N.ERR_ENGINE: EngineError, N.ERR_UNSUPPORTED: UnsupportedExpression,
    N.ERR_MISSING_BINDING: MissingBinding, N.ERR_NO_FEASIBLE_KERNEL: NoFeasibleKernel,
    N.ERR_NON_POSITIVE_TIME: NonPositiveTime, N.ERR_INVALID_ARGUMENT: EngineError,
    N.ERR_CUDA: CudaError, N.ERR_NO_DEVICE: NoDevice,
}


def _raise(status: int, ctx_handle) -> None:
    if status == N.OK:
        return
    msg = N.lib().amlt_gpu_last_error(ctx_handle)
    msg = msg.decode() if msg else f"status {status}"
    raise _ERRS.get(status, EngineError)(msg)


# ---------------------------------------------------------------------------
# clock seam (clock.hpp:12-55)


class Clock:
    def now(self) -> float:  # seconds, monotonic
        raise NotImplementedError


class SteadyClock(Clock):
    def now(self) -> float:
        return time.perf_counter()


class FakeClock(Clock):
    """Scripted clock: now() alternates interval start / end; each completed
    interval advances time by the next scripted delta; raises when the script
    is exhausted (clock.hpp:29-55)."""

    def __init__(self, deltas=()):
        self.deltas = list(deltas)
        self.next = 0
        self.t = 0.0
        self.open = False

    def push(self, d: float) -> None:
        self.deltas.append(d)

    def now(self) -> float:
        if not self.open:
            self.open = True
            return self.t
        self.open = False
        if self.next >= len(self.deltas):
            raise IndexError("FakeClock: delta script exhausted")
        self.t += self.deltas[self.next]
        self.next += 1
        return self.t

    def consumed(self) -> int:
        return self.next


class _ClockBridge:
    """Wraps a Python Clock as an amlt_clock_fn; remembers a raised error."""

    def __init__(self, clock: Optional[Clock]):
        self.clock = clock
        self.error: Optional[BaseException] = None

        def cb(_user):
            try:
                return float(self.clock.now())
            except BaseException as e:  # noqa: BLE001 — re-raised after the call
                self.error = e
                return 0.0

        self.fn = N.CLOCK_FN(cb) if clock is not None else N.CLOCK_FN()

    def check(self):
        if self.error is not None:
            e, self.error = self.error, None
            raise e


# ---------------------------------------------------------------------------
# plain records (tiled_executor.hpp, autotuner.hpp)


@dataclass
class Bounds:
    i0: int = 0
    i1: int = 0
    j0: int = 0
    j1: int = 0
    k0: int = 0
    k1: int = 0

    def _c(self):
        return N.BoundsC(self.i0, self.i1, self.j0, self.j1, self.k0, self.k1)


@dataclass
class TileParams:
    """kc: K-segment depth (split-K when < K); nc: column-tile width selecting
    a variant; pack: accepted, no effect; variant: explicit index or -1."""
    kc: int = 0
    nc: int = 0
    pack: bool = False
    variant: int = -1

    def _c(self):
        return N.TileParamsC(self.kc, self.nc, int(self.pack), self.variant)


@dataclass
class ExecRecord:
    variant: int
    splits: int
    i0: int
    i1: int
    j0: int
    j1: int
    k0: int
    k1: int


@dataclass
class ExecLog:
    records: List[ExecRecord] = field(default_factory=list)
    capacity: int = 4096


@dataclass
class Trial:
    value: int
    rows: int
    elapsed: float
    score: float


@dataclass
class CoverRect:
    i0: int
    i1: int
    k0: int
    k1: int
    j0: int
    j1: int


@dataclass
class TuneReport:
    trials: List[Trial] = field(default_factory=list)
    best_variant: int = -1
    best_kc: int = 0
    tuned: bool = False
    from_cache: bool = False
    scratch_tuned: bool = False
    coverage: List[CoverRect] = field(default_factory=list)
    tuning_fraction: float = 0.0
    total_seconds: float = 0.0
    tuning_seconds: float = 0.0  # whole-task trials on the scratch R (included in total_seconds)
    refined: int = 0  # > 0: the winner is the best of the last `refined` (8-wave) trials


@dataclass
class VariantInfo:
    index: int
    name: str
    block_m: int
    block_n: int
    block_k: int
    thread_m: int
    thread_n: int
    threads: int
    stages: int
    smem_bytes: int
    tensor_core: bool


# ---------------------------------------------------------------------------
# operands


_TORCH_DT = None


def _dtype_code_of(x) -> int:
    import numpy as np
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return {torch.float64: N.F64, torch.float32: N.F32, torch.int32: N.I32}[x.dtype]
    except ImportError:
        pass
    return {np.dtype(np.float64): N.F64, np.dtype(np.float32): N.F32,
            np.dtype(np.int32): N.I32}[np.asarray(x).dtype]


@dataclass(frozen=True)
class Shape:
    """The shape of an operand another rank holds: with
    AMLT_HOST_BCAST_SHARED, ranks other than 0 describe B and the shared
    vectors by shape only (row-major, dense) and receive them by broadcast."""
    rows: int
    cols: int = 1
    dtype: str = "f64"


def matrix_of(x, expect_device: Optional[bool] = None) -> N.Matrix:
    """Describes a 1-D/2-D torch tensor or numpy array as an amlt_matrix
    (MatrixBuffer-like: rows, cols, leading stride, storage order)."""
    if x is None:
        return N.Matrix()
    if isinstance(x, Shape):
        return N.Matrix(None, x.rows, x.cols, max(x.cols, 1), N.ROW_MAJOR, DTYPES[x.dtype])
    try:
        import torch
        is_t = isinstance(x, torch.Tensor)
    except ImportError:
        is_t = False
    if is_t:
        if expect_device is True and not x.is_cuda:
            raise EngineError("operand must be a CUDA tensor for the device entry points")
        if expect_device is False and x.is_cuda:
            raise EngineError("operand must be a host tensor for run_host")
        shape, strides, ptr = tuple(x.shape), tuple(x.stride()), x.data_ptr()
    else:
        import numpy as np
        a = np.asarray(x)
        shape = a.shape
        strides = tuple(s // a.itemsize for s in a.strides)
        ptr = a.ctypes.data
    dt = _dtype_code_of(x)
    if len(shape) == 1:
        return N.Matrix(ptr, shape[0], 1, max(strides[0], 1), N.ROW_MAJOR, dt)
    if len(shape) != 2:
        raise EngineError("operands must be 1-D or 2-D")
    r, c = shape
    s0, s1 = strides
    if s1 == 1 or c == 1 or r == 0 or c == 0:
        return N.Matrix(ptr, r, c, max(s0, c, 1), N.ROW_MAJOR, dt)
    if s0 == 1 or r == 1:
        return N.Matrix(ptr, r, c, max(s1, r, 1), N.COL_MAJOR, dt)
    raise UnsupportedExpression("operand buffers need unit stride along one axis")


@dataclass
class Operands:
    """Operands (kernel_exec.hpp:17-24): A, B, R and the aux leaves the body
    names. Buffers follow MatrixBuffer conventions: A is M x K (or K x M for
    a transposed statement), B is K x N (or N x K), R is M x N, vectors are
    1-D or len x 1."""
    a: object
    b: object
    r: object
    thres: object = None
    dis: object = None
    aux: tuple = ()  # generated bodies: aux leaves by position (TaskPlan.aux_names)

    def _c(self, device: Optional[bool]):
        if len(self.aux) > N.MAX_AUX:
            raise UnsupportedExpression(f"at most {N.MAX_AUX} aux operands")
        aux = (N.Matrix * N.MAX_AUX)(*[matrix_of(x, device) for x in self.aux])
        return N.OperandsC(matrix_of(self.a, device), matrix_of(self.b, device),
                           matrix_of(self.r, device), matrix_of(self.thres, device),
                           matrix_of(self.dis, device), len(self.aux), aux)


# ---------------------------------------------------------------------------
# context + plan


class Context:
    """One B200 device context (amlt_gpu_ctx_create). dry_run=True plans,
    logs and clocks dispatches without touching a device (host-logic tests);
    f64_emulation=True lets the tuner pick the int8-tensor-core f64 GEMM
    (AMLT_CTX_F64_EMULATION)."""

    def __init__(self, device: int = 0, dry_run: bool = False, f64_emulation: bool = False):
        self._lib = N.lib()
        h = C.c_void_p()
        flags = (N.CTX_DRY_RUN if dry_run else 0) | (N.CTX_F64_EMULATION if f64_emulation else 0)
        st = self._lib.amlt_gpu_ctx_create(device, flags, C.byref(h))
        _raise(st, None)
        self.handle = h
        self.device = device
        self.dry_run = dry_run

    def close(self):
        if getattr(self, "handle", None):
            self._lib.amlt_gpu_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def attach_comm(self, rank: int, world_size: int, unique_id: Optional[bytes] = None,
                    exchange=None) -> None:
        """Attaches an NCCL communicator for the multi-process host entry
        (amlt_gpu_comm_attach): rank 0 makes the id; `exchange(id_or_None)`
        must return rank 0's id on every rank (e.g. a torch.distributed
        object broadcast). Collective: every rank must call it. A one-rank
        communicator is valid (its broadcasts are no-ops)."""
        if world_size <= 1 and unique_id is None and exchange is None:
            exchange = lambda uid: uid  # noqa: E731  (rank 0 is the only rank)
        if unique_id is None:
            if rank == 0:
                buf = C.create_string_buffer(N.NCCL_ID_BYTES)
                _raise(self._lib.amlt_gpu_comm_unique_id(buf), None)
                unique_id = buf.raw
            if exchange is None:
                raise EngineError("attach_comm needs the id or an exchange function")
            unique_id = exchange(unique_id)
        buf = C.create_string_buffer(bytes(unique_id), N.NCCL_ID_BYTES)
        _raise(self._lib.amlt_gpu_comm_attach(self.handle, buf, int(rank), int(world_size)), self.handle)

    def detach_comm(self) -> None:
        _raise(self._lib.amlt_gpu_comm_detach(self.handle), self.handle)

    @property
    def comm_size(self) -> int:
        return int(self._lib.amlt_gpu_comm_size(self.handle))

    def last_host_layout(self) -> dict:
        """How the last run_host / run_host_adaptive call on this context ran
        (amlt_gpu_last_host_layout)."""
        out = (C.c_int64 * N.HOST_LAYOUT_FIELDS)()
        _raise(self._lib.amlt_gpu_last_host_layout(self.handle, out), self.handle)
        keys = ("bands", "k_panels", "zero_copy_r", "band0_rows", "k_panel0", "bcast", "tuned")
        return {k: int(v) for k, v in zip(keys, out)}

    def set_stream(self, stream) -> None:
        """Launch on a torch.cuda.Stream (or raw cudaStream_t int); None
        restores the context's own stream."""
        if stream is None:
            ptr = None
        elif isinstance(stream, int):
            ptr = stream
        else:
            ptr = stream.cuda_stream
        _raise(self._lib.amlt_gpu_set_stream(self.handle, C.c_void_p(ptr)), self.handle)

    def clear_tuning_cache(self) -> None:
        self._lib.amlt_gpu_clear_tuning_cache(self.handle)

    def plan(self, body, dtype="f64", accumulate=True, layout_a=0, layout_b=0,
             thres_class="j", thres_value=0.0) -> "GpuPlan":
        return GpuPlan(self, body, dtype, accumulate, layout_a, layout_b, thres_class,
                       thres_value)

    def plan_for(self, task: TaskPlan, dtype="f64") -> "GpuPlan":
        if task.body == N.BODY_GENERIC:
            return GpuPlan.from_source(self, task.source, dtype)
        return GpuPlan(self, task.body, dtype, task.accumulate, task.layout_a, task.layout_b,
                       task.thres_class, task.thres_value)

    def plan_source(self, source: str, dtype="f64") -> "GpuPlan":
        """amlt_gpu_plan_from_source: recognise + plan a task text; statements
        that are not one of the fixed bodies get a generated body (compiled at
        plan time, cached per statement)."""
        return GpuPlan.from_source(self, source, dtype)


BODIES = {"gemm": N.BODY_GEMM, "matmul": N.BODY_GEMM, "discount": N.BODY_DISCOUNT,
          "q1": N.BODY_DISCOUNT, "boost": N.BODY_BOOST, "q2": N.BODY_BOOST,
          "sqdiff": N.BODY_SQDIFF, "eqcount": N.BODY_EQCOUNT, "thrcount": N.BODY_THRCOUNT,
          "q3": N.BODY_THRCOUNT}
DTYPES = {"f64": N.F64, "f32": N.F32, "i32": N.I32}
THRES_CLASSES = {"c": N.LEAF_CONSTANT, "i": N.LEAF_VEC_I, "j": N.LEAF_VEC_J,
                 "ij": N.LEAF_MAT_IJ}


class GpuPlan:
    """An immutable, shareable plan for one body/dtype (amlt_gpu_plan_create)."""

    def __init__(self, ctx: Context, body, dtype, accumulate, layout_a, layout_b, thres_class,
                 thres_value):
        self.ctx = ctx
        self.body = BODIES[body] if isinstance(body, str) else int(body)
        self.dtype = DTYPES[dtype] if isinstance(dtype, str) else int(dtype)
        tc = THRES_CLASSES[thres_class] if isinstance(thres_class, str) else int(thres_class)
        self.desc = N.BodyDesc(self.body, self.dtype, int(bool(accumulate)), int(layout_a),
                               int(layout_b), tc, float(thres_value))
        h = C.c_void_p()
        _raise(ctx._lib.amlt_gpu_plan_create(ctx.handle, C.byref(self.desc), C.byref(h)),
               ctx.handle)
        self.handle = h

    @classmethod
    def from_source(cls, ctx: Context, source: str, dtype="f64") -> "GpuPlan":
        self = cls.__new__(cls)
        self.ctx = ctx
        self.dtype = DTYPES[dtype] if isinstance(dtype, str) else int(dtype)
        info = N.TaskInfoC()
        h = C.c_void_p()
        self.handle = None
        _raise(ctx._lib.amlt_gpu_plan_from_source(ctx.handle, source.encode(), self.dtype,
                                                  C.byref(h), C.byref(info)), ctx.handle)
        self.handle = h
        self.desc = info.desc
        self.body = info.desc.body
        self.aux_names = tuple(info.aux_names[q].value.decode() for q in range(info.n_aux))
        self.aux_classes = tuple(int(info.aux_class[q]) for q in range(info.n_aux))
        return self

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.ctx._lib.amlt_gpu_plan_destroy(self.handle)
                self.handle = None
        except Exception:  # noqa: BLE001
            pass

    def variants(self) -> List[VariantInfo]:
        L = self.ctx._lib
        out = []
        for i in range(L.amlt_gpu_plan_num_variants(self.handle)):
            v = N.VariantInfoC()
            _raise(L.amlt_gpu_plan_variant(self.handle, i, C.byref(v)), self.ctx.handle)
            out.append(VariantInfo(v.index, v.name.decode(), v.block_m, v.block_n, v.block_k,
                                   v.thread_m, v.thread_n, v.threads, v.stages, v.smem_bytes,
                                   bool(v.tensor_core)))
        return out

    def default_variant(self, M, N_, K) -> int:
        return self.ctx._lib.amlt_gpu_plan_default_variant(self.handle, M, N_, K)


# ---------------------------------------------------------------------------
# executors


def _log_c(log: Optional[ExecLog]):
    if log is None:
        return None, None
    recs = (N.ExecRecordC * log.capacity)()
    lc = N.ExecLogC(C.cast(recs, C.POINTER(N.ExecRecordC)), log.capacity, 0, 0)
    return lc, recs


def _log_back(log: Optional[ExecLog], lc, recs) -> None:
    if log is None:
        return
    for i in range(lc.count):
        r = recs[i]
        log.records.append(ExecRecord(r.variant, r.splits, r.i0, r.i1, r.j0, r.j1, r.k0, r.k1))


def run_subtask(plan: GpuPlan, ops: Operands, params: TileParams, bounds: Bounds,
                clock: Optional[Clock] = None, log: Optional[ExecLog] = None) -> float:
    """R(bounds) (+)= body over bounds on the GPU, synchronously; returns the
    elapsed seconds between the clock's two reads (CUDA events if no clock).
    Mirrors run_subtask (tiled_executor.hpp:36-44)."""
    ctx = plan.ctx
    bridge = _ClockBridge(clock)
    oc = ops._c(None if ctx.dry_run else True)
    tp = params._c() if params is not None else TileParams()._c()
    bc = bounds._c()
    lc, recs = _log_c(log)
    el = C.c_double()
    st = ctx._lib.amlt_gpu_run_subtask(ctx.handle, plan.handle, C.byref(oc), C.byref(tp),
                                       C.byref(bc), bridge.fn, None,
                                       C.byref(lc) if lc is not None else None, C.byref(el))
    bridge.check()
    _raise(st, ctx.handle)
    _log_back(log, lc, recs)
    return el.value


def run_naive(plan: GpuPlan, ops: Operands, bounds: Bounds,
              clock: Optional[Clock] = None) -> float:
    """The per-element device executor (amlt_gpu_run_naive): the GPU
    counterpart of run_naive / execute_scalar_region (src/naive.cpp:157-166,
    src/kernel_exec.cpp:408-457) — untiled, k ascending, one IEEE operation
    per syntax-tree node. Synchronous; returns elapsed seconds."""
    ctx = plan.ctx
    bridge = _ClockBridge(clock)
    oc = ops._c(None if ctx.dry_run else True)
    bc = bounds._c()
    el = C.c_double()
    st = ctx._lib.amlt_gpu_run_naive(ctx.handle, plan.handle, C.byref(oc), C.byref(bc), bridge.fn,
                                     None, C.byref(el))
    bridge.check()
    _raise(st, ctx.handle)
    return el.value


def enqueue(plan: GpuPlan, ops: Operands, params: TileParams, bounds: Bounds) -> None:
    """Asynchronous run_subtask on the context stream (no clock, no sync)."""
    ctx = plan.ctx
    oc = ops._c(True)
    tp = params._c() if params is not None else TileParams()._c()
    bc = bounds._c()
    _raise(ctx._lib.amlt_gpu_enqueue(ctx.handle, plan.handle, C.byref(oc), C.byref(tp),
                                     C.byref(bc)), ctx.handle)


class Graph:
    """One enqueue of (plan, ops, params, bounds) captured into a CUDA graph
    (amlt_gpu_graph_capture): launch() replays every kernel of the step on
    the context's current stream with no per-launch host work. The operands
    (pointers and shapes) and the variant are fixed at capture."""

    def __init__(self, plan: GpuPlan, ops: Operands, params: TileParams, bounds: Bounds):
        self.plan = plan
        self._ops = ops  # keeps the operand tensors alive while the graph exists
        ctx = plan.ctx
        oc = ops._c(True)
        tp = params._c() if params is not None else TileParams()._c()
        bc = bounds._c()
        h = C.c_void_p()
        _raise(ctx._lib.amlt_gpu_graph_capture(ctx.handle, plan.handle, C.byref(oc), C.byref(tp),
                                               C.byref(bc), C.byref(h)), ctx.handle)
        self.handle = h

    def launch(self) -> None:
        _raise(self.plan.ctx._lib.amlt_gpu_graph_launch(self.handle), self.plan.ctx.handle)

    def close(self) -> None:
        if self.handle:
            self.plan.ctx._lib.amlt_gpu_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 (interpreter shutdown)
            pass


def capture_graph(plan: GpuPlan, ops: Operands, params: TileParams, bounds: Bounds) -> Graph:
    """amlt_gpu_graph_capture: the step enqueue() would run, as a CUDA graph."""
    return Graph(plan, ops, params, bounds)


def _report(rc: N.TuneReportC) -> TuneReport:
    rep = TuneReport()
    rep.trials = [Trial(rc.trials[i].value, rc.trials[i].rows, rc.trials[i].elapsed,
                        rc.trials[i].score) for i in range(rc.n_trials)]
    rep.best_variant = rc.best_variant
    rep.best_kc = rc.best_kc
    rep.tuned = bool(rc.tuned)
    rep.from_cache = bool(rc.from_cache)
    rep.scratch_tuned = bool(rc.scratch_tuned)
    rep.coverage = [CoverRect(c.i0, c.i1, c.k0, c.k1, c.j0, c.j1)
                    for c in rc.coverage[:rc.n_cover]]
    rep.tuning_fraction = rc.tuning_fraction
    rep.total_seconds = rc.total_seconds
    rep.tuning_seconds = rc.tuning_seconds
    rep.refined = rc.refined
    return rep


def adaptive_execute(plan: GpuPlan, ops: Operands, bounds: Bounds, pack: bool = False,
                     clock: Optional[Clock] = None, log: Optional[ExecLog] = None) -> TuneReport:
    """Measured tile choice on row bands of the real task, then the remainder
    with the winner; every output produced exactly once
    (adaptive_execute, autotuner.hpp:62-70)."""
    ctx = plan.ctx
    bridge = _ClockBridge(clock)
    oc = ops._c(None if ctx.dry_run else True)
    bc = bounds._c()
    lc, recs = _log_c(log)
    rc = N.TuneReportC()
    st = ctx._lib.amlt_gpu_adaptive_execute(ctx.handle, plan.handle, C.byref(oc), C.byref(bc),
                                            int(pack), bridge.fn, None,
                                            C.byref(lc) if lc is not None else None,
                                            C.byref(rc))
    bridge.check()
    _raise(st, ctx.handle)
    _log_back(log, lc, recs)
    return _report(rc)


@dataclass
class RefTrial:
    value: int
    elapsed: float
    score: float


@dataclass
class RefCoverRect:
    k0: int
    k1: int
    j0: int
    j1: int


@dataclass
class AmuletTuneReport:
    """The reference's TuneReport (autotuner.hpp:26-34)."""
    kc_trials: List[RefTrial] = field(default_factory=list)
    nc_trials: List[RefTrial] = field(default_factory=list)
    best_kc: int = 0
    best_nc: int = 0
    tuned: bool = False
    coverage: List[RefCoverRect] = field(default_factory=list)
    tuning_fraction: float = 0.0
    total_seconds: float = 0.0


def adaptive_execute_amulet(plan: GpuPlan, ops: Operands, bounds: Bounds, i_h: int = 12,
                            i_w: int = 16, clock: Optional[Clock] = None,
                            log: Optional[ExecLog] = None) -> AmuletTuneReport:
    """AMULET's own tuner contract over the GPU executor (find_kc / find_nc /
    remainder rectangles, autotuner.cpp:8-151). With the reference plan's
    (i_h, i_w) and the same clock script it makes the reference's choices."""
    ctx = plan.ctx
    bridge = _ClockBridge(clock)
    oc = ops._c(None if ctx.dry_run else True)
    bc = bounds._c()
    lc, recs = _log_c(log)
    rc = N.AmuletReportC()
    st = ctx._lib.amlt_gpu_adaptive_execute_amulet(ctx.handle, plan.handle, C.byref(oc),
                                                   C.byref(bc), i_h, i_w, bridge.fn, None,
                                                   C.byref(lc) if lc is not None else None,
                                                   C.byref(rc))
    bridge.check()
    _raise(st, ctx.handle)
    _log_back(log, lc, recs)
    rep = AmuletTuneReport()
    rep.kc_trials = [RefTrial(t.value, t.elapsed, t.score) for t in rc.kc_trials[:rc.n_kc_trials]]
    rep.nc_trials = [RefTrial(t.value, t.elapsed, t.score) for t in rc.nc_trials[:rc.n_nc_trials]]
    rep.best_kc, rep.best_nc, rep.tuned = rc.best_kc, rc.best_nc, bool(rc.tuned)
    rep.coverage = [RefCoverRect(c.k0, c.k1, c.j0, c.j1) for c in rc.coverage[:rc.n_cover]]
    rep.tuning_fraction, rep.total_seconds = rc.tuning_fraction, rc.total_seconds
    return rep


def _host_flags(r_zero: bool, bcast: bool) -> int:
    return (N.HOST_R_ZERO if r_zero else 0) | (N.HOST_BCAST_SHARED if bcast else 0)


def run_host(plan: GpuPlan, ops: Operands, bounds: Bounds, params: Optional[TileParams] = None,
             clock: Optional[Clock] = None, r_zero: bool = False, bcast: bool = False) -> float:
    """Host-buffer entry: operands in host memory (pinned for full speed).
    A / R row bands and B K-panels are pipelined against compute; R comes
    back into ops.r; returns elapsed seconds for all of it. r_zero=True
    states R starts at zero (zero-filled on the device, not copied in).
    bcast=True (a communicator attached): B and the shared vectors come
    from rank 0's host memory by NCCL broadcast (other ranks pass Shape)."""
    ctx = plan.ctx
    bridge = _ClockBridge(clock)
    oc = ops._c(False)
    bc = bounds._c()
    tp = params._c() if params is not None else None
    el = C.c_double()
    st = ctx._lib.amlt_gpu_run_host(ctx.handle, plan.handle, C.byref(oc),
                                    C.byref(tp) if tp is not None else None, C.byref(bc),
                                    _host_flags(r_zero, bcast), bridge.fn, None, C.byref(el))
    bridge.check()
    _raise(st, ctx.handle)
    return el.value


def run_host_adaptive(plan: GpuPlan, ops: Operands, bounds: Bounds, clock: Optional[Clock] = None,
                      r_zero: bool = False, bcast: bool = False) -> TuneReport:
    """run_adaptive over host buffers (amlt_gpu_run_host_adaptive): the
    tuner picks the tile on the first call of a shape (the task then runs
    whole through adaptive_execute), later calls reuse the winner through
    the copy / compute pipeline. The report's total_seconds covers the
    copies too."""
    ctx = plan.ctx
    bridge = _ClockBridge(clock)
    oc = ops._c(False)
    bc = bounds._c()
    rc = N.TuneReportC()
    el = C.c_double()
    st = ctx._lib.amlt_gpu_run_host_adaptive(ctx.handle, plan.handle, C.byref(oc), C.byref(bc),
                                             _host_flags(r_zero, bcast), bridge.fn, None,
                                             C.byref(rc), C.byref(el))
    bridge.check()
    _raise(st, ctx.handle)
    return _report(rc)


class ShardedGroup:
    """A persistent row-band group over several devices of this process
    (amlt_sharded_create): contexts, the NCCL communicator, plans and tuning
    winners are made once and reused by every run."""

    def __init__(self, devices, dry_run: bool = False):
        self._lib = N.lib()
        self.devices = list(devices)
        self.dry_run = dry_run
        devs = (C.c_int * len(self.devices))(*self.devices)
        h = C.c_void_p()
        st = self._lib.amlt_sharded_create(len(self.devices), devs, N.CTX_DRY_RUN if dry_run else 0,
                                           C.byref(h))
        if st != N.OK:
            raise _ERRS.get(st, EngineError)(self._lib.amlt_sharded_last_error(None).decode())
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            self._lib.amlt_sharded_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def run(self, ops: Operands, bounds: Bounds, body=None, source: Optional[str] = None,
            dtype="f64", r_zero: bool = False, **desc):
        """Runs the task on every device's row band; returns (elapsed seconds,
        one TuneReport per device). The plan: `source` (a task text), else
        `body` with the GpuPlan descriptor fields in **desc."""
        dt = DTYPES[dtype] if isinstance(dtype, str) else int(dtype)
        d = None
        if source is None:
            b = BODIES[body] if isinstance(body, str) else int(body)
            tc = desc.get("thres_class", "j")
            tc = THRES_CLASSES[tc] if isinstance(tc, str) else int(tc)
            d = N.BodyDesc(b, dt, int(bool(desc.get("accumulate", True))), int(desc.get("layout_a", 0)),
                           int(desc.get("layout_b", 0)), tc, float(desc.get("thres_value", 0.0)))
        oc = ops._c(False)
        bc = bounds._c()
        reps = (N.TuneReportC * len(self.devices))()
        el = C.c_double()
        st = self._lib.amlt_sharded_run(self.handle, C.byref(d) if d is not None else None,
                                        source.encode() if source is not None else None, dt,
                                        C.byref(oc), C.byref(bc), N.HOST_R_ZERO if r_zero else 0,
                                        reps, C.byref(el))
        if st != N.OK:
            raise _ERRS.get(st, EngineError)(self._lib.amlt_sharded_last_error(self.handle).decode())
        return el.value, [_report(r) for r in reps]


def run_sharded_host(desc_plan: GpuPlan, ops: Operands, bounds: Bounds, devices,
                     r_zero: bool = False) -> float:
    """Single-process row-band multi-GPU run (amlt_gpu_run_sharded): host
    operands, B and vectors NCCL-broadcast from devices[0], one band per
    device, R rows copied back. Returns elapsed seconds."""
    devs = (C.c_int * len(devices))(*devices)
    oc = ops._c(False)
    bc = bounds._c()
    el = C.c_double()
    st = N.lib().amlt_gpu_run_sharded(C.byref(desc_plan.desc), C.byref(oc), C.byref(bc),
                                      len(devices), devs, N.HOST_R_ZERO if r_zero else 0,
                                      C.byref(el))
    if st != N.OK:
        raise _ERRS.get(st, EngineError)(N.lib().amlt_gpu_sharded_last_error().decode())
    return el.value


def run_sharded_source(source: str, ops: Operands, bounds: Bounds, devices, dtype="f64",
                       r_zero: bool = False) -> float:
    """amlt_gpu_run_sharded_source: the single-process multi-GPU run for any
    recognised task text (generated bodies included; aux leaves in
    ops.aux by position). Returns elapsed seconds."""
    devs = (C.c_int * len(devices))(*devices)
    oc = ops._c(False)
    bc = bounds._c()
    el = C.c_double()
    dt = DTYPES[dtype] if isinstance(dtype, str) else int(dtype)
    st = N.lib().amlt_gpu_run_sharded_source(source.encode(), dt, C.byref(oc), C.byref(bc),
                                             len(devices), devs, N.HOST_R_ZERO if r_zero else 0,
                                             C.byref(el))
    if st != N.OK:
        raise _ERRS.get(st, EngineError)(N.lib().amlt_gpu_sharded_last_error().decode())
    return el.value


def run_fixed(plan: GpuPlan, ops: Operands, bounds: Bounds, kc: int, nc: int, pack=False,
              clock: Optional[Clock] = None, log: Optional[ExecLog] = None) -> float:
    """run_fixed (engine.hpp:67-68): one subtask over the whole bounds."""
    return run_subtask(plan, ops, TileParams(kc, nc, pack), bounds, clock, log)


def run_adaptive(plan: GpuPlan, ops: Operands, bounds: Bounds, pack=False,
                 clock: Optional[Clock] = None, log: Optional[ExecLog] = None) -> TuneReport:
    """run_adaptive (engine.hpp:65-66)."""
    return adaptive_execute(plan, ops, bounds, pack, clock, log)


def measure_peak(pipe: str) -> tuple:
    """(lane ops/s, SM GHz) of one pipe on the current device: 'dfma',
    'ffma', 'alu', 'dsetp', 'dmma' (roofline denominators)."""
    code = {"dfma": 0, "ffma": 1, "alu": 2, "dsetp": 3, "dmma": 4, "discount_f64": 5,
            "boost_f64": 6, "boost_f32": 7, "sqdiff_f32": 8, "eqcount_i32": 9, "gemm_f32": 10,
            "gemm_f64": 11, "ffma2": 12}[pipe]
    ops, ghz = C.c_double(), C.c_double()
    st = N.lib().amlt_gpu_measure_peak(code, C.byref(ops), C.byref(ghz))
    if st != N.OK:
        raise CudaError(f"measure_peak({pipe}) failed: status {st}")
    return ops.value, ghz.value


def spr(M: int, K: int, N_: int, seconds: float) -> float:
    """Scaled processing rate M*K*N / (1e9*T); NonPositiveTime for T <= 0
    (engine.cpp:212-216)."""
    out = C.c_double()
    st = N.lib().amlt_spr(M, K, N_, float(seconds), C.byref(out))
    if st == N.ERR_NON_POSITIVE_TIME:
        raise NonPositiveTime(f"elapsed time must be positive, got {seconds:f}")
    if st != N.OK:
        raise EngineError(f"spr: status {st}")
    return out.value


def bounds_of(task: TaskPlan, M: int, K: int, N_: int) -> Bounds:
    """bind_dims (engine.cpp:104-126) for a recognised task with [0..X]
    ranges: the (i, j, k) half-open rectangle."""
    return Bounds(0, M, 0, N_, 0, K)


def operands_of(task: TaskPlan, data: Dict[str, object]) -> Operands:
    """make_operands (engine.cpp:153-163): binds buffers by the task's role
    names; an aux leaf the body needs but `data` lacks -> MissingBinding."""
    def need(name):
        if name not in data:
            raise MissingBinding(f"missing binding for '{name}'")
        return data[name]
    thres = need(task.thres_name) if task.thres_name else None
    dis = need(task.dis_name) if task.dis_name else None
    aux = tuple(need(n) for n in task.aux_names)
    return Operands(need(task.a_name), need(task.b_name), need(task.result_name), thres, dis, aux)
