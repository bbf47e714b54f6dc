"""ctypes binding of the C-ABI in ``include/amlt_gpu.h`` (lib/libamlt_gpu.so).

This is the Python side of the drop-in boundary: every structure below is a
field-for-field mirror of the header. The library is required — there is no
CPU fallback; importing a missing or stale library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "lib", "libamlt_gpu.so")

ABI_VERSION = 4
MAX_AUX = 8

# amlt_status
OK, ERR_ENGINE, ERR_UNSUPPORTED, ERR_MISSING_BINDING, ERR_NO_FEASIBLE_KERNEL, \
    ERR_NON_POSITIVE_TIME, ERR_INVALID_ARGUMENT, ERR_CUDA, ERR_NO_DEVICE = range(9)

# amlt_body
BODY_GEMM, BODY_DISCOUNT, BODY_BOOST, BODY_SQDIFF, BODY_EQCOUNT, BODY_THRCOUNT, \
    BODY_GENERIC = range(7)
# amlt_dtype
F64, F32, I32 = range(3)
ROW_MAJOR, COL_MAJOR = 0, 1
LAYOUT_NORMAL, LAYOUT_TRANSPOSED = 0, 1
LEAF_CONSTANT, LEAF_VEC_I, LEAF_VEC_J, LEAF_MAT_IJ = range(4)
CTX_DRY_RUN = 1
CTX_F64_EMULATION = 2
MAX_TRIALS = 128
MAX_COVER = 64


class BodyDesc(C.Structure):
    _fields_ = [("body", C.c_int32), ("dtype", C.c_int32), ("accumulate", C.c_int32),
                ("layout_a", C.c_int32), ("layout_b", C.c_int32), ("thres_class", C.c_int32),
                ("thres_value", C.c_double)]


class Matrix(C.Structure):
    _fields_ = [("data", C.c_void_p), ("rows", C.c_int64), ("cols", C.c_int64),
                ("ld", C.c_int64), ("order", C.c_int32), ("dtype", C.c_int32)]


class OperandsC(C.Structure):
    _fields_ = [("a", Matrix), ("b", Matrix), ("r", Matrix), ("thres", Matrix), ("dis", Matrix),
                ("n_aux", C.c_int32), ("aux", Matrix * MAX_AUX)]


class BoundsC(C.Structure):
    _fields_ = [("i0", C.c_int64), ("i1", C.c_int64), ("j0", C.c_int64), ("j1", C.c_int64),
                ("k0", C.c_int64), ("k1", C.c_int64)]


class TileParamsC(C.Structure):
    _fields_ = [("kc", C.c_int64), ("nc", C.c_int64), ("pack", C.c_int32), ("variant", C.c_int32)]


class ExecRecordC(C.Structure):
    _fields_ = [("variant", C.c_int32), ("splits", C.c_int32), ("i0", C.c_int64),
                ("i1", C.c_int64), ("j0", C.c_int64), ("j1", C.c_int64), ("k0", C.c_int64),
                ("k1", C.c_int64)]


class ExecLogC(C.Structure):
    _fields_ = [("records", C.POINTER(ExecRecordC)), ("capacity", C.c_int32),
                ("count", C.c_int32), ("total", C.c_int32)]


class VariantInfoC(C.Structure):
    _fields_ = [("index", C.c_int32), ("body", C.c_int32), ("dtype", C.c_int32),
                ("block_m", C.c_int32), ("block_n", C.c_int32), ("block_k", C.c_int32),
                ("thread_m", C.c_int32), ("thread_n", C.c_int32), ("threads", C.c_int32),
                ("stages", C.c_int32), ("smem_bytes", C.c_int32), ("tensor_core", C.c_int32),
                ("name", C.c_char * 48)]


class TrialC(C.Structure):
    _fields_ = [("value", C.c_int64), ("rows", C.c_int64), ("elapsed", C.c_double),
                ("score", C.c_double)]


class CoverRectC(C.Structure):
    _fields_ = [("i0", C.c_int64), ("i1", C.c_int64), ("k0", C.c_int64), ("k1", C.c_int64),
                ("j0", C.c_int64), ("j1", C.c_int64)]


class TuneReportC(C.Structure):
    _fields_ = [("n_trials", C.c_int32), ("trials", TrialC * MAX_TRIALS),
                ("best_variant", C.c_int32), ("best_kc", C.c_int64), ("tuned", C.c_int32),
                ("from_cache", C.c_int32), ("scratch_tuned", C.c_int32), ("n_cover", C.c_int32),
                ("coverage", CoverRectC * MAX_COVER), ("tuning_fraction", C.c_double),
                ("total_seconds", C.c_double), ("tuning_seconds", C.c_double), ("refined", C.c_int32)]


MAX_REF_TRIALS = 64
MAX_REF_COVER = 128


class RefTrialC(C.Structure):
    _fields_ = [("value", C.c_int64), ("elapsed", C.c_double), ("score", C.c_double)]


class RefCoverC(C.Structure):
    _fields_ = [("k0", C.c_int64), ("k1", C.c_int64), ("j0", C.c_int64), ("j1", C.c_int64)]


class AmuletReportC(C.Structure):
    _fields_ = [("n_kc_trials", C.c_int32), ("kc_trials", RefTrialC * MAX_REF_TRIALS),
                ("n_nc_trials", C.c_int32), ("nc_trials", RefTrialC * MAX_REF_TRIALS),
                ("best_kc", C.c_int64), ("best_nc", C.c_int64), ("tuned", C.c_int32),
                ("n_cover", C.c_int32), ("coverage", RefCoverC * MAX_REF_COVER),
                ("tuning_fraction", C.c_double), ("total_seconds", C.c_double)]


PROG_OPCODES = ("mov", "add", "sub", "mul", "div", "gtcmp", "gecmp", "ltcmp", "lecmp", "eqcmp",
                "masksub", "maskadd")
PROG_NOPS = len(PROG_OPCODES)


class TaskInfoC(C.Structure):
    _fields_ = [("desc", BodyDesc), ("a", C.c_char * 64), ("b", C.c_char * 64),
                ("r", C.c_char * 64), ("thres", C.c_char * 64), ("dis", C.c_char * 64),
                ("n_aux", C.c_int32), ("aux_names", (C.c_char * 64) * MAX_AUX),
                ("aux_class", C.c_int32 * MAX_AUX), ("prog_counts", C.c_int32 * PROG_NOPS),
                ("prog_instrs", C.c_int32), ("prog_flops", C.c_int32)]


CLOCK_FN = C.CFUNCTYPE(C.c_double, C.c_void_p)

EXPORTS = [
    "amlt_gpu_abi_version", "amlt_gpu_ctx_create", "amlt_gpu_ctx_destroy", "amlt_gpu_last_error",
    "amlt_gpu_set_stream", "amlt_gpu_clear_tuning_cache", "amlt_gpu_plan_create",
    "amlt_gpu_plan_destroy", "amlt_gpu_plan_num_variants", "amlt_gpu_plan_variant",
    "amlt_gpu_plan_default_variant", "amlt_gpu_run_subtask", "amlt_gpu_enqueue",
    "amlt_gpu_adaptive_execute", "amlt_gpu_run_host", "amlt_spr", "amlt_gpu_measure_peak",
    "amlt_gpu_recognize", "amlt_gpu_plan_from_source", "amlt_gpu_adaptive_execute_amulet",
    "amlt_gpu_run_sharded", "amlt_gpu_sharded_last_error", "amlt_matrix_file_info",
    "amlt_matrix_file_read", "amlt_matrix_file_write", "amlt_matrix_file_last_error",
    "amlt_operand_seed", "amlt_gen_matrix", "amlt_gpu_run_naive", "amlt_gpu_generated_source",
    "amlt_gpu_run_sharded_source", "amlt_gpu_matrix_alloc", "amlt_gpu_matrix_free",
    "amlt_gpu_matrix_upload", "amlt_gpu_matrix_download", "amlt_gpu_run_host_adaptive",
    "amlt_gpu_comm_unique_id", "amlt_gpu_comm_attach", "amlt_gpu_comm_detach", "amlt_gpu_comm_size",
    "amlt_gpu_last_host_layout",
    "amlt_sharded_create", "amlt_sharded_destroy", "amlt_sharded_run", "amlt_sharded_size",
    "amlt_sharded_last_error", "amlt_gpu_graph_capture", "amlt_gpu_graph_launch", "amlt_gpu_graph_destroy",
]
HOST_LAYOUT_FIELDS = 7
HOST_R_ZERO = 1
HOST_BCAST_SHARED = 2
NCCL_ID_BYTES = 128

_lib = None


def lib():
    """Loads lib/libamlt_gpu.so once. Raises if it is missing (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2305_08872_b200.build` "
            "(there is no CPU fallback for the MMLT kernels)")
    L = C.CDLL(LIB_PATH)
    P = C.c_void_p
    L.amlt_gpu_abi_version.restype = C.c_int
    L.amlt_gpu_ctx_create.argtypes = [C.c_int, C.c_int, C.POINTER(P)]
    L.amlt_gpu_ctx_destroy.argtypes = [P]
    L.amlt_gpu_ctx_destroy.restype = None
    L.amlt_gpu_last_error.argtypes = [P]
    L.amlt_gpu_last_error.restype = C.c_char_p
    L.amlt_gpu_set_stream.argtypes = [P, P]
    L.amlt_gpu_clear_tuning_cache.argtypes = [P]
    L.amlt_gpu_clear_tuning_cache.restype = None
    L.amlt_gpu_plan_create.argtypes = [P, C.POINTER(BodyDesc), C.POINTER(P)]
    L.amlt_gpu_plan_destroy.argtypes = [P]
    L.amlt_gpu_plan_destroy.restype = None
    L.amlt_gpu_plan_num_variants.argtypes = [P]
    L.amlt_gpu_plan_variant.argtypes = [P, C.c_int, C.POINTER(VariantInfoC)]
    L.amlt_gpu_plan_default_variant.argtypes = [P, C.c_int64, C.c_int64, C.c_int64]
    L.amlt_gpu_run_subtask.argtypes = [P, P, C.POINTER(OperandsC), C.POINTER(TileParamsC),
                                       C.POINTER(BoundsC), CLOCK_FN, P, C.POINTER(ExecLogC),
                                       C.POINTER(C.c_double)]
    L.amlt_gpu_run_naive.argtypes = [P, P, C.POINTER(OperandsC), C.POINTER(BoundsC), CLOCK_FN, P,
                                      C.POINTER(C.c_double)]
    L.amlt_gpu_enqueue.argtypes = [P, P, C.POINTER(OperandsC), C.POINTER(TileParamsC),
                                   C.POINTER(BoundsC)]
    L.amlt_gpu_graph_capture.argtypes = [P, P, C.POINTER(OperandsC), C.POINTER(TileParamsC),
                                         C.POINTER(BoundsC), C.POINTER(P)]
    L.amlt_gpu_graph_launch.argtypes = [P]
    L.amlt_gpu_graph_destroy.argtypes = [P]
    L.amlt_gpu_graph_destroy.restype = None
    L.amlt_gpu_adaptive_execute.argtypes = [P, P, C.POINTER(OperandsC), C.POINTER(BoundsC),
                                            C.c_int, CLOCK_FN, P, C.POINTER(ExecLogC),
                                            C.POINTER(TuneReportC)]
    L.amlt_gpu_run_host.argtypes = [P, P, C.POINTER(OperandsC), C.POINTER(TileParamsC),
                                    C.POINTER(BoundsC), C.c_int, CLOCK_FN, P,
                                    C.POINTER(C.c_double)]
    L.amlt_gpu_run_host_adaptive.argtypes = [P, P, C.POINTER(OperandsC), C.POINTER(BoundsC), C.c_int,
                                             CLOCK_FN, P, C.POINTER(TuneReportC), C.POINTER(C.c_double)]
    L.amlt_gpu_comm_unique_id.argtypes = [C.c_void_p]
    L.amlt_gpu_comm_attach.argtypes = [P, C.c_void_p, C.c_int, C.c_int]
    L.amlt_gpu_comm_detach.argtypes = [P]
    L.amlt_gpu_comm_size.argtypes = [P]
    L.amlt_gpu_last_host_layout.argtypes = [P, C.POINTER(C.c_int64)]
    L.amlt_sharded_create.argtypes = [C.c_int, C.POINTER(C.c_int), C.c_int, C.POINTER(P)]
    L.amlt_sharded_destroy.argtypes = [P]
    L.amlt_sharded_destroy.restype = None
    L.amlt_sharded_run.argtypes = [P, C.POINTER(BodyDesc), C.c_char_p, C.c_int, C.POINTER(OperandsC),
                                   C.POINTER(BoundsC), C.c_int, C.POINTER(TuneReportC),
                                   C.POINTER(C.c_double)]
    L.amlt_sharded_size.argtypes = [P]
    L.amlt_sharded_last_error.argtypes = [P]
    L.amlt_sharded_last_error.restype = C.c_char_p
    L.amlt_gpu_measure_peak.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.amlt_gpu_adaptive_execute_amulet.argtypes = [P, P, C.POINTER(OperandsC), C.POINTER(BoundsC),
                                                   C.c_int, C.c_int, CLOCK_FN, P,
                                                   C.POINTER(ExecLogC), C.POINTER(AmuletReportC)]
    L.amlt_gpu_run_sharded.argtypes = [C.POINTER(BodyDesc), C.POINTER(OperandsC),
                                       C.POINTER(BoundsC), C.c_int, C.POINTER(C.c_int), C.c_int,
                                       C.POINTER(C.c_double)]
    L.amlt_gpu_sharded_last_error.restype = C.c_char_p
    L.amlt_gpu_run_sharded_source.argtypes = [C.c_char_p, C.c_int, C.POINTER(OperandsC),
                                              C.POINTER(BoundsC), C.c_int, C.POINTER(C.c_int),
                                              C.c_int, C.POINTER(C.c_double)]
    L.amlt_matrix_file_info.argtypes = [C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int)]
    L.amlt_matrix_file_read.argtypes = [C.c_char_p, C.c_void_p, C.c_int, C.c_int]
    L.amlt_matrix_file_write.argtypes = [C.c_char_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                                         C.c_int, C.c_int]
    L.amlt_matrix_file_last_error.restype = C.c_char_p
    L.amlt_operand_seed.argtypes = [C.c_uint64, C.c_char_p]
    L.amlt_operand_seed.restype = C.c_uint64
    L.amlt_gen_matrix.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_void_p,
                                  C.c_int, C.c_int]
    L.amlt_gpu_generated_source.argtypes = [C.c_char_p, C.c_int, C.c_char_p, C.c_int64]
    L.amlt_gpu_generated_source.restype = C.c_int64
    L.amlt_gpu_matrix_alloc.argtypes = [P, C.c_int64, C.c_int64, C.c_int, C.c_int, C.POINTER(Matrix)]
    L.amlt_gpu_matrix_free.argtypes = [P, C.POINTER(Matrix)]
    L.amlt_gpu_matrix_upload.argtypes = [P, C.POINTER(Matrix), C.c_void_p, C.c_int64]
    L.amlt_gpu_matrix_download.argtypes = [P, C.POINTER(Matrix), C.c_void_p, C.c_int64]
    L.amlt_gpu_recognize.argtypes = [C.c_char_p, C.POINTER(TaskInfoC)]
    L.amlt_gpu_plan_from_source.argtypes = [P, C.c_char_p, C.c_int, C.POINTER(P),
                                            C.POINTER(TaskInfoC)]
    L.amlt_spr.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_double, C.POINTER(C.c_double)]
    v = L.amlt_gpu_abi_version()
    if v != ABI_VERSION:
        raise ImportError(f"libamlt_gpu ABI {v} != expected {ABI_VERSION}; rebuild")
    _lib = L
    return L
