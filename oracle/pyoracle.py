"""TEST INFRASTRUCTURE — NOT PRODUCT CODE.

ctypes front-ends for the two CPU checkers built by ``oracle/Makefile``:

* ``liboracle.so`` — our C restatement of the reference's naive oracle
  (``oracle/oracle.c``; reference ``src/naive.cpp:18-166``).
* ``_ref/libamlt_ref_v{3,4}.so`` — the unmodified reference engine plus
  ``ref_shim.cpp``: ``compile_task``/``make_task_data``/``run_naive``/
  ``run_adaptive``/``run_fixed`` exactly as the reference ships them.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

# Body ids shared with oracle.c (and, by value, with include/amlt_gpu.h).
GEMM, DISCOUNT, BOOST, SQDIFF, EQCOUNT, THRCOUNT = range(6)

_oracle = None
_ref = None


def _cpu_has_v4() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            flags = set()
            for line in f:
                if line.startswith("flags"):
                    flags = set(line.split(":", 1)[1].split())
                    break
    except OSError:
        return False
    return {"avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl"} <= flags


def build_if_needed() -> None:
    """Builds the checkers (``make -C oracle``) if the .so files are missing."""
    need = not os.path.exists(os.path.join(HERE, "liboracle.so"))
    need |= not os.path.exists(os.path.join(HERE, "_ref", "libamlt_ref_v3.so")) and os.path.isdir(
        "/root/reference/proj/src")
    if need:
        import subprocess

        subprocess.run(["make", "-C", HERE, "-j8"], check=True, stdout=subprocess.DEVNULL)


def oracle_lib():
    global _oracle
    if _oracle is None:
        build_if_needed()
        lib = C.CDLL(os.path.join(HERE, "liboracle.so"))
        lib.oracle_run.restype = C.c_int
        lib.oracle_eval.restype = C.c_double
        lib.oracle_eval.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_double]
        _oracle = lib
    return _oracle


class _View(C.Structure):
    _fields_ = [("p", C.POINTER(C.c_double)), ("s0", C.c_int64), ("s1", C.c_int64)]


def _view(arr, s0=None, s1=None):
    """(row, col) element strides of a float64 array view, or explicit ones."""
    if arr is None:
        return None
    a = np.asarray(arr)
    assert a.dtype == np.float64
    if s0 is None:
        if a.ndim == 2:
            s0, s1 = a.strides[0] // 8, a.strides[1] // 8
        else:
            s0, s1 = a.strides[0] // 8, 0
    v = _View(a.ctypes.data_as(C.POINTER(C.c_double)), s0, s1)
    v._keep = a
    return v


def oracle_eval(kind, a, b, t=0.0, dis=0.0) -> float:
    return oracle_lib().oracle_eval(kind, a, b, t, dis)


def oracle_run(kind, A, B, R, thres=None, dis=None, bounds=None, accumulate=True,
               thres_form="j"):
    """R[i0:i1, j0:j1] (+)= sum_k body(...) in place; every array float64.

    ``A`` is indexed (i, k) and ``B`` (k, j) — pass ``X.T`` views for the
    transposed orientations. ``thres`` is a scalar (form "c"), an M-vector
    ("i"), an N-vector ("j") or an M x N matrix ("ij"); ``dis`` an N-vector.
    """
    A = np.asarray(A)
    B = np.asarray(B)
    M, K = A.shape
    N = B.shape[1]
    if bounds is None:
        bounds = (0, M, 0, N, 0, K)
    i0, i1, j0, j1, k0, k1 = bounds
    assert R.dtype == np.float64
    tv = None
    keep = []
    if thres is not None:
        if thres_form == "c":
            tarr = np.array([float(thres)])
            keep.append(tarr)
            tv = _view(tarr, 0, 0)
        elif thres_form == "i":
            tv = _view(np.asarray(thres), np.asarray(thres).strides[0] // 8, 0)
        elif thres_form == "j":
            tv = _view(np.asarray(thres), 0, np.asarray(thres).strides[0] // 8)
        else:
            tv = _view(np.asarray(thres))
    dv = None
    if dis is not None:
        dv = _view(np.asarray(dis), 0, np.asarray(dis).strides[0] // 8)
    rc = oracle_lib().oracle_run(
        C.c_int(kind), C.c_int(1 if accumulate else 0), C.byref(_view(A)), C.byref(_view(B)),
        C.byref(tv) if tv is not None else None, C.byref(dv) if dv is not None else None,
        R.ctypes.data_as(C.POINTER(C.c_double)), C.c_int64(R.strides[0] // 8),
        C.c_int64(R.strides[1] // 8), C.c_int64(i0), C.c_int64(i1), C.c_int64(j0), C.c_int64(j1),
        C.c_int64(k0), C.c_int64(k1))
    if rc != 0:
        raise ValueError(f"oracle_run: unknown body {kind}")
    return R


# --------------------------------------------------------------------------
# The unmodified reference engine


def ref_lib():
    global _ref
    if _ref is None:
        build_if_needed()
        name = "libamlt_ref_v4.so" if _cpu_has_v4() else "libamlt_ref_v3.so"
        path = os.path.join(HERE, "_ref", name)
        if not os.path.exists(path):
            raise FileNotFoundError(f"reference engine not built: {path}")
        lib = C.CDLL(path)
        lib.ref_task_new.restype = C.c_void_p
        lib.ref_task_new.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_int64, C.c_uint64,
                                     C.c_int, C.c_int, C.c_int]
        for fn in ("ref_task_free", "ref_task_is_mmlt", "ref_task_num_arrays", "ref_task_shape",
                   "ref_task_array_name", "ref_task_result_name", "ref_task_array_shape",
                   "ref_task_array_get", "ref_task_array_set", "ref_task_bounds",
                   "ref_task_run_naive", "ref_task_run_adaptive", "ref_task_run_fixed",
                   "ref_task_run_scalar_region", "ref_task_run_adaptive_bands", "ref_task_roles",
                   "ref_task_program"):
            getattr(lib, fn).argtypes = None
        lib.ref_task_array_name.restype = C.c_char_p
        lib.ref_task_result_name.restype = C.c_char_p
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_gen_matrix.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int, C.c_int,
                                       C.c_void_p]
        lib.ref_write_matrix_file.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_int,
                                              C.c_void_p]
        lib.ref_read_matrix_file.argtypes = [C.c_char_p, C.POINTER(C.c_int64),
                                             C.POINTER(C.c_int64), C.POINTER(C.c_int),
                                             C.c_void_p, C.c_int64]
        _ref = lib
    return _ref


def ref_gen_matrix(seed: int, rows: int, cols: int, order: int, mode: int):
    """The reference's gen_matrix (src/matrix.cpp:20-37): the storage-order
    buffer as a flat float64 array."""
    import numpy as np
    out = np.empty(rows * cols, dtype=np.float64)
    if ref_lib().ref_gen_matrix(seed & 0xFFFFFFFFFFFFFFFF, rows, cols, order, mode,
                                out.ctypes.data) != 0:
        raise RuntimeError(ref_lib().ref_last_error().decode())
    return out


def ref_write_matrix_file(path: str, rows: int, cols: int, order: int, storage) -> None:
    """The reference's write_matrix_file (src/matrix.cpp:64-88)."""
    import numpy as np
    s = np.ascontiguousarray(storage, dtype=np.float64).ravel()
    if ref_lib().ref_write_matrix_file(str(path).encode(), rows, cols, order, s.ctypes.data) != 0:
        raise RuntimeError(ref_lib().ref_last_error().decode())


def ref_read_matrix_file(path: str):
    """The reference's read_matrix_file (src/matrix.cpp:90-114) ->
    (rows, cols, order, flat storage-order float64 array); raises
    RuntimeError carrying the reference's EngineError message."""
    import numpy as np
    r, c, o = C.c_int64(), C.c_int64(), C.c_int()
    lib = ref_lib()
    if lib.ref_read_matrix_file(str(path).encode(), C.byref(r), C.byref(c), C.byref(o), None, 0):
        raise RuntimeError(lib.ref_last_error().decode())
    out = np.empty(r.value * c.value, dtype=np.float64)
    if lib.ref_read_matrix_file(str(path).encode(), C.byref(r), C.byref(c), C.byref(o),
                                out.ctypes.data, out.size):
        raise RuntimeError(lib.ref_last_error().decode())
    return r.value, c.value, o.value, out


def ref_available() -> bool:
    try:
        ref_lib()
        return True
    except (FileNotFoundError, OSError):
        return False


def preset_source(name: str) -> str:
    lib = ref_lib()
    buf = C.create_string_buffer(4096)
    n = lib.ref_preset_source(name.encode(), buf, 4096)
    if n < 0:
        raise KeyError(name)
    return buf.value.decode()


def task_text(rhs: str, op: str = "+=") -> str:
    return ("where(i in [0..M] and j in [0..N] and k in [0..K]) {\n  R[i][j] " + op + " " + rhs
            + ";\n}\n")


SQDIFF_TEXT = task_text("(A[i][k] - B[k][j])*(A[i][k] - B[k][j])")
EQCOUNT_TEXT = task_text("A[i][k] == B[k][j]")


@dataclass
class RefTask:
    """One reference task: compile_task + bind_dims + make_task_data."""

    handle: int
    M: int
    K: int
    N: int

    @classmethod
    def create(cls, source: str, M: int, K: int, N: int, seed: int = 1, int_valued=True,
               order_a=0, order_b=0) -> "RefTask":
        lib = ref_lib()
        h = lib.ref_task_new(source.encode(), M, K, N, C.c_uint64(seed), order_a, order_b,
                             1 if int_valued else 0)
        if not h:
            raise RuntimeError("reference compile failed: " + lib.ref_last_error().decode())
        return cls(h, M, K, N)

    def __del__(self):
        if getattr(self, "handle", None):
            ref_lib().ref_task_free(C.c_void_p(self.handle))
            self.handle = None

    @property
    def _h(self):
        return C.c_void_p(self.handle)

    def is_mmlt(self) -> bool:
        return bool(ref_lib().ref_task_is_mmlt(self._h))

    def shape(self):
        ih, iw = C.c_int(), C.c_int()
        ref_lib().ref_task_shape(self._h, C.byref(ih), C.byref(iw))
        return ih.value, iw.value

    def names(self):
        lib = ref_lib()
        return [lib.ref_task_array_name(self._h, i).decode()
                for i in range(lib.ref_task_num_arrays(self._h))]

    def result_name(self) -> str:
        return ref_lib().ref_task_result_name(self._h).decode()

    def program(self) -> list:
        """The reference's compiled pseudo-program (schedule_labelfs +
        print_program): one "opcode dst src..." string per instruction."""
        buf = C.create_string_buffer(1 << 14)
        n = ref_lib().ref_task_program(self._h, buf, C.c_int(len(buf)))
        if n < 0:
            raise RuntimeError("not an MMLT task")
        return [ln for ln in buf.value.decode().splitlines() if ln.strip()]

    def roles(self):
        a, b, aux = (C.create_string_buffer(256) for _ in range(3))
        if ref_lib().ref_task_roles(self._h, a, b, aux, 256) != 0:
            return None
        return a.value.decode(), b.value.decode(), [x for x in aux.value.decode().split(",") if x]

    def get(self, name: str) -> np.ndarray:
        """The array in logical (rows, cols) orientation (a view over storage)."""
        lib = ref_lib()
        r, c, o = C.c_int64(), C.c_int64(), C.c_int()
        if lib.ref_task_array_shape(self._h, name.encode(), C.byref(r), C.byref(c), C.byref(o)):
            raise KeyError(name)
        buf = np.empty(r.value * c.value, dtype=np.float64)
        lib.ref_task_array_get(self._h, name.encode(), buf.ctypes.data_as(C.c_void_p))
        if o.value == 0:
            return buf.reshape(r.value, c.value)
        return buf.reshape(c.value, r.value).T

    def set(self, name: str, values: np.ndarray) -> None:
        lib = ref_lib()
        r, c, o = C.c_int64(), C.c_int64(), C.c_int()
        if lib.ref_task_array_shape(self._h, name.encode(), C.byref(r), C.byref(c), C.byref(o)):
            raise KeyError(name)
        v = np.asarray(values, dtype=np.float64).reshape(r.value, c.value)
        store = np.ascontiguousarray(v if o.value == 0 else v.T)
        lib.ref_task_array_set(self._h, name.encode(), store.ctypes.data_as(C.c_void_p))

    def bounds(self):
        out = (C.c_int64 * 6)()
        ref_lib().ref_task_bounds(self._h, out)
        return tuple(out)

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError("reference error: " + ref_lib().ref_last_error().decode())

    def run_naive(self) -> float:
        s = C.c_double()
        self._check(ref_lib().ref_task_run_naive(self._h, C.byref(s)))
        return s.value

    def run_adaptive(self, pack=False):
        s, kc, nc = C.c_double(), C.c_int64(), C.c_int64()
        self._check(ref_lib().ref_task_run_adaptive(self._h, int(pack), C.byref(s), C.byref(kc),
                                                    C.byref(nc)))
        return s.value, kc.value, nc.value

    def run_adaptive_scripted(self, deltas):
        """run_adaptive under the reference's FakeClock with `deltas`:
        (best_kc, best_nc, tuned, intervals consumed, [(k0, k1, j0, j1)])."""
        arr = (C.c_double * len(deltas))(*deltas)
        kc, nc, tuned, used, ncov = C.c_int64(), C.c_int64(), C.c_int(), C.c_int(), C.c_int(256)
        cov = (C.c_int64 * (4 * 256))()
        self._check(ref_lib().ref_task_run_adaptive_scripted(
            self._h, arr, C.c_int(len(deltas)), C.byref(kc), C.byref(nc), C.byref(tuned),
            C.byref(used), C.byref(ncov), cov))
        rects = [tuple(cov[4 * i:4 * i + 4]) for i in range(ncov.value)]
        return kc.value, nc.value, bool(tuned.value), used.value, rects

    def run_fixed(self, kc, nc, pack=False) -> float:
        s = C.c_double()
        self._check(ref_lib().ref_task_run_fixed(self._h, C.c_int64(kc), C.c_int64(nc), int(pack),
                                                 C.byref(s)))
        return s.value

    def run_scalar_region(self, i0, i1, j0, j1, k0, k1) -> None:
        self._check(ref_lib().ref_task_run_scalar_region(self._h, *(C.c_int64(x) for x in
                                                                    (i0, i1, j0, j1, k0, k1))))

    def run_adaptive_bands(self, nthreads, i0=None, i1=None, j0=None, j1=None) -> float:
        b = self.bounds()
        i0 = b[0] if i0 is None else i0
        i1 = b[1] if i1 is None else i1
        j0 = b[2] if j0 is None else j0
        j1 = b[3] if j1 is None else j1
        s = C.c_double()
        self._check(ref_lib().ref_task_run_adaptive_bands(
            self._h, C.c_int(nthreads), C.c_int64(i0), C.c_int64(i1), C.c_int64(j0),
            C.c_int64(j1), C.byref(s)))
        return s.value
