"""Input-side data formats of the hot path: AMLT matrix files and the
reference's seeded operand generator, landing directly in the kernel dtype.

* AMLT binary matrix file (reference README.md:146-157,
  src/matrix.cpp:64-114): 24-byte header — "AMLT", u32 rows, u32 cols (LE),
  u8 storage order (0 row-major, 1 col-major), 11 zero bytes — then
  rows*cols little-endian f64 values in storage order.
* gen_matrix (src/matrix.cpp:20-37) and the per-array seed of
  make_task_data (src/engine.cpp:17-24,147): mt19937_64 over
  seed_seq{seed ^ fnv1a(name), rows, cols, order, mode}.

Both are implemented natively in lib/libamlt_gpu.so (csrc/matrix_file.cpp);
this module only allocates the destination (numpy on the host or a torch
tensor on a CUDA device) and returns it shaped rows x cols with the file's
storage order expressed as strides, which is what ``engine.matrix_of``
reads back into an ``amlt_matrix``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

from . import _native as N
from .engine import EngineError, _ERRS

ROW_MAJOR, COL_MAJOR = N.ROW_MAJOR, N.COL_MAJOR
INT_VALUED, REAL = 0, 1
_DT = {"f64": N.F64, "f32": N.F32, "i32": N.I32}
_NP = {N.F64: "float64", N.F32: "float32", N.I32: "int32"}


def _check(status: int) -> None:
    if status == N.OK:
        return
    msg = N.lib().amlt_matrix_file_last_error()
    msg = msg.decode() if msg else f"status {status}"
    raise _ERRS.get(status, EngineError)(msg)


@dataclass(frozen=True)
class MatrixFileInfo:
    rows: int
    cols: int
    order: int  # ROW_MAJOR / COL_MAJOR


def _dt(dtype) -> int:
    if isinstance(dtype, str):
        if dtype not in _DT:
            raise EngineError(f"unknown dtype '{dtype}' (f64 | f32 | i32)")
        return _DT[dtype]
    return int(dtype)


def _alloc(rows: int, cols: int, order: int, dt: int, device):
    """Storage-order buffer of rows*cols values, returned as a rows x cols
    view (col-major = transposed view of a cols x rows array)."""
    sr, sc = (rows, cols) if order == ROW_MAJOR else (cols, rows)
    if device is None:
        import numpy as np
        buf = np.empty((sr, sc), dtype=_NP[dt])
        view = buf if order == ROW_MAJOR else buf.T
        return buf, view, buf.ctypes.data, 0
    import torch
    tdt = {N.F64: torch.float64, N.F32: torch.float32, N.I32: torch.int32}[dt]
    dev = torch.device(device)
    if dev.type != "cuda":
        raise EngineError("device must be a CUDA device (or None for host numpy)")
    buf = torch.empty((sr, sc), dtype=tdt, device=dev)
    view = buf if order == ROW_MAJOR else buf.t()
    return buf, view, buf.data_ptr(), 1


def matrix_file_info(path: str) -> MatrixFileInfo:
    r, c, o = C.c_int64(), C.c_int64(), C.c_int()
    _check(N.lib().amlt_matrix_file_info(str(path).encode(), C.byref(r), C.byref(c), C.byref(o)))
    return MatrixFileInfo(r.value, c.value, o.value)


def read_matrix_file(path: str, dtype="f64", device=None):
    """read_matrix_file (src/matrix.cpp:90-114). Returns a rows x cols numpy
    array (device None) or CUDA tensor in ``dtype``, storage order preserved
    through strides. Raises EngineError on a bad magic, unknown order,
    truncated payload or unopenable path."""
    info = matrix_file_info(path)
    dt = _dt(dtype)
    if device is not None:
        import torch
        torch.cuda.set_device(torch.device(device))
    buf, view, ptr, on_dev = _alloc(info.rows, info.cols, info.order, dt, device)
    if info.rows * info.cols:
        _check(N.lib().amlt_matrix_file_read(str(path).encode(), C.c_void_p(ptr), dt, on_dev))
    return view


def storage_order_of(x) -> int:
    """ROW_MAJOR / COL_MAJOR of a 2-D array or tensor the way the engine
    describes it (engine.matrix_of)."""
    from .engine import matrix_of
    return matrix_of(x).order


def write_matrix_file(path: str, x, order: Optional[int] = None) -> None:
    """write_matrix_file (src/matrix.cpp:64-88) of a 2-D f64/f32/i32 numpy
    array or tensor (host or CUDA). The storage order is the buffer's own
    (row- or col-major contiguous) unless ``order`` forces a copy."""
    from .engine import _dtype_code_of
    try:
        dt = _dtype_code_of(x)
    except KeyError:
        raise EngineError("matrix files are written from f64, f32 or i32 buffers") from None
    try:
        import torch
        is_t = isinstance(x, torch.Tensor)
    except ImportError:
        is_t = False
    if len(tuple(x.shape)) != 2:
        raise EngineError("matrix files hold 2-D matrices")
    rows, cols = (int(v) for v in x.shape)
    if order is None:
        try:
            order = storage_order_of(x) if rows and cols else ROW_MAJOR
        except EngineError:
            order = ROW_MAJOR
    # The storage-order buffer to stream: contiguous rows (row-major) or
    # contiguous columns (col-major).
    if is_t:
        s = x.contiguous() if order == ROW_MAJOR else x.t().contiguous()
        ptr, on_dev = s.data_ptr(), int(s.is_cuda)
    else:
        import numpy as np
        s = np.ascontiguousarray(x) if order == ROW_MAJOR else np.ascontiguousarray(np.asarray(x).T)
        ptr, on_dev = s.ctypes.data, 0
    _check(N.lib().amlt_matrix_file_write(str(path).encode(), C.c_void_p(ptr), rows, cols, order,
                                          dt, on_dev))


def operand_seed(seed: int, name: str) -> int:
    """seed ^ fnv1a(name) (src/engine.cpp:17-24,147)."""
    return int(N.lib().amlt_operand_seed(C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), name.encode()))


def gen_matrix(seed: int, rows: int, cols: int, order: int = ROW_MAJOR, mode: int = INT_VALUED,
               dtype="f64", device=None):
    """gen_matrix (src/matrix.cpp:20-37): deterministic rows x cols values,
    IntValued in [-8, 8] (mode 0) or Real in [0, 1) (mode 1), generated in
    storage order so the buffer is identical to the reference's."""
    dt = _dt(dtype)
    if device is not None:
        import torch
        torch.cuda.set_device(torch.device(device))
    buf, view, ptr, on_dev = _alloc(rows, cols, order, dt, device)
    _check(N.lib().amlt_gen_matrix(C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), rows, cols, order, mode,
                                   C.c_void_p(ptr), dt, on_dev))
    return view


def gen_operand(seed: int, name: str, rows: int, cols: int, order: int = ROW_MAJOR,
                mode: int = INT_VALUED, dtype="f64", device=None):
    """The array make_task_data binds to ``name`` (src/engine.cpp:128-151)."""
    return gen_matrix(operand_seed(seed, name), rows, cols, order, mode, dtype, device)
