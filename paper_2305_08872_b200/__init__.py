"""B200-native (sm_100a) backend for AMULET's matrix-multiplication-like task.

    R[i][j] (+)= sum_k body(A[i][k], B[k][j], per-column vectors[j])

for the discount, threshold-boost, squared-difference, equality-count and
plain multiply-add bodies, behind the reference engine's executor / tuner
interface (see include/amlt_gpu.h and engine.py).
"""
from . import _native  # noqa: F401
from .engine import (Bounds, Clock, Context, CoverRect, EngineError, ExecLog, ExecRecord,  # noqa: F401
                     FakeClock, GpuPlan, MissingBinding, NoDevice, NoFeasibleKernel,
                     NonPositiveTime, Operands, SteadyClock, TileParams, Trial, TuneReport,
                     UnsupportedExpression, adaptive_execute, bounds_of, enqueue, operands_of,
                     run_adaptive, run_fixed, run_host, run_host_adaptive, run_naive, run_subtask,
                     Shape, ShardedGroup, spr, Graph, capture_graph)
from .task import TaskPlan, compile_task  # noqa: F401
from .taskdata import (TaskData, VerifyResult, bind_dims, load_operand_file,  # noqa: F401
                       make_task_data, verify_against_naive)

__all__ = [n for n in dir() if not n.startswith("_")]
