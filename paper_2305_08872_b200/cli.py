"""Command-line front end over the B200 backend, with the reference CLI's
commands, options, exit codes and report schemas (tools/amlt_main.cpp):

    python -m paper_2305_08872_b200.cli run     --preset q1 --dims 1024 1024 1024 --verify
    python -m paper_2305_08872_b200.cli tune    --preset matmul --dims 16 200 256
    python -m paper_2305_08872_b200.cli bench   --preset q2 --dims 512 512 512
    python -m paper_2305_08872_b200.cli explain --preset q1

* run (amlt_main.cpp:163-255): modes adaptive (the GPU tuner), fixed
  (--kc/--nc; nc selects the tile variant by its column width) and naive
  (the per-element device executor). --verify re-runs the task through the
  naive executor and compares: exact, pass (rel <= 1e-12 for f64, 1e-5 for
  f32 on real data) or fail (exit 4). Reports as json / csv / table with the
  reference's field names.
* tune (:257-289): AMULET's own tuner contract over the GPU executor by
  default (--tuner amulet: kc/nc trials, chosen, tuning fraction, coverage —
  the reference's JSON schema); --tuner gpu prints the GPU tuner's report.
* bench (:291-345): power-of-two (kc, nc) grid of fixed runs as CSV plus an
  adaptive footer line.
* explain (:347-386): recognition, the body's straight-line program, the
  reference plan's register block, and the GPU variants for the task.

Data: make_task_data's seeded arrays (--seed, --data int|real, --layout-a/-b
row|col), generated with the reference's generator straight into the kernel
dtype on the device, or --a-file / --b-file AMLT matrix files.

Exit codes (amlt_main.cpp:431-446): 0 ok; 2 usage or engine error
("<class>: message"); 3 recognition failed; 4 verification failed. One
deliberate difference: the reference's run falls back to its CPU
interpreter for statements that are not multiply-accumulate; this backend
has no CPU path, so run exits 3 for them like tune/bench/explain.
"""
from __future__ import annotations

import argparse
import json
import sys
from typing import List, Optional, Tuple

from . import _native as N
from . import engine as E
from . import matrix_io as io
from . import taskdata as TD
from .task import TaskError, TaskPlan, compile_task, preset_source

# The reference's straight-line program per body (schedule.hpp:32-53; frozen
# for q1 at tests/test_schedule.cpp:53-72) and its register block at the
# default machine (simd 8, 32 vector registers; kernel_plan.cpp:45-143).
_PROGRAMS = {
    N.BODY_GEMM: ["mul REG0 A B", "add R R REG0"],
    N.BODY_DISCOUNT: ["mul REG0 A B", "gtcmp MASKREG0 REG0 {t}", "mul REG1 REG0 {d}",
                      "masksub REG0 MASKREG0 REG0 REG1", "add R R REG0"],
    N.BODY_BOOST: ["mul REG0 A B", "gtcmp MASKREG0 REG0 {t}", "sub REG1 REG0 {t}",
                   "maskadd REG0 MASKREG0 REG0 REG1", "add R R REG0"],
    N.BODY_SQDIFF: ["sub REG0 A B", "mul REG0 REG0 REG0", "add R R REG0"],
    N.BODY_EQCOUNT: ["eqcmp MASKREG0 A B", "maskadd REG0 MASKREG0 $0 $1", "add R R REG0"],
    N.BODY_THRCOUNT: ["mul REG0 A B", "gtcmp MASKREG0 REG0 {t}", "maskadd REG0 MASKREG0 $0 $1",
                      "add R R REG0"],
}
_LEDGER = {N.BODY_DISCOUNT: (11, 16, 31)}
_DEFAULT_BLOCK = (12, 16, 31)
_CLASS = {N.LEAF_CONSTANT: "constant", N.LEAF_VEC_I: "[i]", N.LEAF_VEC_J: "[j]",
          N.LEAF_MAT_IJ: "[i][j]"}


class UsageError(Exception):
    pass


class RecognitionFailed(Exception):
    pass


# ---------------------------------------------------------------------------
# task and data


def _load_source(a) -> str:
    if a.task and a.preset:
        raise E.EngineError("--task and --preset are mutually exclusive")
    if a.task:
        try:
            with open(a.task) as f:
                return f.read()
        except OSError:
            raise E.EngineError(f"cannot open task file: {a.task}") from None
    if a.preset:
        src = preset_source(a.preset)
        if src is None:
            raise E.EngineError(f"unknown preset: {a.preset}")
        return src
    raise E.EngineError("one of --task or --preset is required")


def _task_id(a) -> str:
    return a.preset if a.preset else a.task


def _compile(a) -> TaskPlan:
    src = _load_source(a)
    try:
        return compile_task(src)
    except E.UnsupportedExpression as e:
        raise RecognitionFailed(str(e)) from None


def _extents(tp: TaskPlan, dims: List[int]) -> Tuple[int, int, int]:
    """bind_dims (src/engine.cpp:104-126) over --dims M K N."""
    return TD.bind_dims(tp, dims[0], dims[1], dims[2])[1]


def _task_data(tp: TaskPlan, M: int, K: int, N_: int, a, device: str) -> TD.TaskData:
    """make_task_data (src/engine.cpp:128-151) on the device, then --a-file /
    --b-file (amlt_main.cpp:117-134)."""
    mode = io.REAL if a.data == "real" else io.INT_VALUED
    if a.dtype == "i32" and mode == io.REAL:
        raise E.EngineError("--dtype i32 needs --data int")
    data = TD.make_task_data(tp, M, K, N_, seed=a.seed,
                             order_a=io.COL_MAJOR if a.layout_a == "col" else io.ROW_MAJOR,
                             order_b=io.COL_MAJOR if a.layout_b == "col" else io.ROW_MAJOR,
                             mode=mode, dtype=a.dtype, device=device)
    if a.a_file:
        TD.load_operand_file(data, tp.a_name, a.a_file, device)
    if a.b_file:
        TD.load_operand_file(data, tp.b_name, a.b_file, device)
    return data


def _verify(plan, data: TD.TaskData, bounds: E.Bounds, dtype: str, mode: str) -> str:
    """verify_against_naive (src/engine.cpp:186-210) with the per-element
    device executor as the naive side."""
    v = TD.verify_against_naive(plan, data, bounds, io.REAL if mode == "real" else io.INT_VALUED)
    return "exact" if v.exact else ("pass" if v.passed else "fail")


def _aggregate(times: List[float], agg: str) -> float:
    return sum(times) / len(times) if agg == "mean" else min(times)


def _g(x: float) -> str:
    """std::ostream's default formatting of a double (6 significant digits)."""
    return f"{x:g}"


def _emit(a, text: str) -> None:
    if not a.out:
        sys.stdout.write(text)
        return
    try:
        with open(a.out, "w") as f:
            f.write(text)
    except OSError:
        raise E.EngineError(f"cannot write output file: {a.out}") from None


def _setup(a):
    tp = _compile(a)
    M, K, N_ = _extents(tp, a.dims)
    ctx = E.Context(a.device, f64_emulation=getattr(a, "f64_emulation", False))
    device = f"cuda:{a.device}"
    plan = ctx.plan_for(tp, a.dtype)
    data = _task_data(tp, M, K, N_, a, device)
    return tp, ctx, plan, data, E.Bounds(0, M, 0, N_, 0, K), (M, K, N_)


def _generated_term(source: str, dtype: str) -> str:
    """The generated body's term expression (amlt_gpu_generated_source)."""
    import ctypes as C
    dt = {"f64": N.F64, "f32": N.F32, "i32": N.I32}[dtype]
    n = N.lib().amlt_gpu_generated_source(source.encode(), dt, None, 0)
    if n < 0:
        raise E.EngineError(N.lib().amlt_gpu_last_error(None).decode())
    buf = C.create_string_buffer(int(n) + 1)
    N.lib().amlt_gpu_generated_source(source.encode(), dt, buf, n + 1)
    text = buf.value.decode()
    body = text[text.index("T term("):]
    body = body[body.index("return ") + 7:]
    return body[:body.index(";")]


def _block(tp: TaskPlan) -> Tuple[int, int, int]:
    return _LEDGER.get(tp.body, _DEFAULT_BLOCK)


# ---------------------------------------------------------------------------
# commands


def cmd_run(a) -> int:
    if a.mode == "fixed" and (a.kc < 1 or a.nc < 1):
        raise UsageError("--mode fixed requires --kc and --nc >= 1")
    tp, ctx, plan, data, bounds, (M, K, N_) = _setup(a)
    times: List[float] = []
    rep = None
    for _ in range(max(1, a.trials)):
        data.result().zero_()
        if a.mode == "adaptive":
            rep = E.adaptive_execute(plan, data.operands(), bounds, a.packing)
            times.append(rep.total_seconds)
        elif a.mode == "fixed":
            times.append(E.run_fixed(plan, data.operands(), bounds, a.kc, a.nc, a.packing))
        else:
            times.append(E.run_naive(plan, data.operands(), bounds))
    elapsed = _aggregate(times, a.agg)
    verify = "skipped"
    if a.verify:
        verify = _verify(plan, data, bounds, a.dtype, a.data)
    rate = E.spr(M, K, N_, elapsed) if elapsed > 0 else None
    kc = nc = None
    if a.mode == "adaptive":
        kc = rep.best_kc if rep.best_kc > 0 else K
        nc = plan.variants()[rep.best_variant].block_n if rep.best_variant >= 0 else N_
    elif a.mode == "fixed":
        kc, nc = a.kc, a.nc
    if a.format == "json":
        j = {"task": _task_id(a), "m": M, "k": K, "n": N_, "mode": a.mode,
             "elapsed_seconds": elapsed, "spr": rate, "kc": kc, "nc": nc, "packing": a.packing,
             "trials": max(1, a.trials), "agg": a.agg, "verify": verify,
             "dtype": a.dtype, "backend": "b200"}
        if rep is not None and rep.best_variant >= 0:
            j["variant"] = plan.variants()[rep.best_variant].name
        text = json.dumps(j, indent=2) + "\n"
    elif a.format == "csv":
        text = "task,m,k,n,mode,elapsed_seconds,spr,kc,nc,packing,verify\n"
        text += (f"{_task_id(a)},{M},{K},{N_},{a.mode},{_g(elapsed)},"
                 f"{_g(rate) if rate is not None else ''},{kc if kc is not None else ''},"
                 f"{nc if nc is not None else ''},{1 if a.packing else 0},{verify}\n")
    else:
        text = (f"task      {_task_id(a)}\n"
                f"dims      {M} x {K} x {N_}\n"
                f"mode      {a.mode}\n"
                f"elapsed   {_g(elapsed)} s ({a.agg} of {max(1, a.trials)})\n"
                f"spr       {_g(rate) if rate is not None else '-'}\n")
        if kc is not None:
            text += f"kc, nc    {kc}, {nc}\n"
        text += f"verify    {verify}\n"
    _emit(a, text)
    if verify == "fail":
        sys.stderr.write("verification failed\n")
        return 4
    return 0


def cmd_tune(a) -> int:
    tp, ctx, plan, data, bounds, (M, K, N_) = _setup(a)
    if a.tuner == "amulet":
        i_h, i_w, _ = _block(tp)
        rep = E.adaptive_execute_amulet(plan, data.operands(), bounds, i_h, i_w)
        j = {"task": _task_id(a), "tuned": rep.tuned,
             "kc_trials": [{"kc": t.value, "elapsed": t.elapsed, "score": t.score}
                           for t in rep.kc_trials],
             "nc_trials": [{"nc": t.value, "elapsed": t.elapsed, "score": t.score}
                           for t in rep.nc_trials],
             "chosen": {"kc": rep.best_kc, "nc": rep.best_nc},
             "tuning_fraction": rep.tuning_fraction, "total_seconds": rep.total_seconds,
             "coverage": [{"k0": c.k0, "k1": c.k1, "j0": c.j0, "j1": c.j1}
                          for c in rep.coverage]}
    else:
        rep = E.adaptive_execute(plan, data.operands(), bounds, a.packing)
        vs = plan.variants()
        j = {"task": _task_id(a), "tuned": rep.tuned, "from_cache": rep.from_cache,
             "scratch_tuned": rep.scratch_tuned,
             "trials": [{"variant": vs[t.value].name, "rows": t.rows, "elapsed": t.elapsed,
                         "score": t.score} for t in rep.trials],
             "chosen": {"variant": vs[rep.best_variant].name if rep.best_variant >= 0 else None,
                        "kc": rep.best_kc if rep.best_kc > 0 else K},
             "tuning_fraction": rep.tuning_fraction, "total_seconds": rep.total_seconds,
             "coverage": [{"i0": c.i0, "i1": c.i1, "k0": c.k0, "k1": c.k1, "j0": c.j0,
                           "j1": c.j1} for c in rep.coverage]}
    _emit(a, json.dumps(j, indent=2) + "\n")
    return 0


def cmd_bench(a) -> int:
    tp, ctx, plan, data, bounds, (M, K, N_) = _setup(a)

    def grid(limit):
        if limit < 16:
            return [limit]
        v, x = [], 16
        while x <= limit:
            v.append(x)
            x *= 2
        return v

    kcs, ncs = grid(K), grid(N_)
    lines = ["kc\\nc," + ",".join(str(n) for n in ncs)]
    for kc in kcs:
        cells = []
        for nc in ncs:
            times = []
            for _ in range(max(1, a.trials)):
                data.result().zero_()
                times.append(E.run_fixed(plan, data.operands(), bounds, kc, nc, a.packing))
            cells.append(_g(_aggregate(times, a.agg)))
        lines.append(f"{kc}," + ",".join(cells))
    data.result().zero_()
    rep = E.adaptive_execute(plan, data.operands(), bounds, a.packing)
    kc = rep.best_kc if rep.best_kc > 0 else K
    nc = plan.variants()[rep.best_variant].block_n if rep.best_variant >= 0 else N_
    lines.append(f"adaptive,{_g(rep.total_seconds)},kc={kc},nc={nc}")
    _emit(a, "\n".join(lines) + "\n")
    return 0


def cmd_explain(a) -> int:
    src = _load_source(a)
    out = ["task:", src.rstrip(), ""]
    try:
        tp = compile_task(src)
    except E.UnsupportedExpression as e:
        out.append(f"recognition: not MMLT ({e})")
        _emit(a, "\n".join(out) + "\n")
        raise RecognitionFailed(str(e)) from None
    lay = {N.LAYOUT_NORMAL: "normal", N.LAYOUT_TRANSPOSED: "transposed"}
    aux = []
    if tp.thres_name:
        aux.append(f"{tp.thres_name} {_CLASS[tp.thres_class]}")
    elif tp.body in (N.BODY_DISCOUNT, N.BODY_BOOST, N.BODY_THRCOUNT):
        aux.append(f"constant {tp.thres_value:g}")
    if tp.dis_name:
        aux.append(f"{tp.dis_name} [j]")
    out.append(f"recognition: MMLT  A={tp.a_name} ({lay[tp.layout_a]})  "
               f"B={tp.b_name} ({lay[tp.layout_b]})  R={tp.result_name}  "
               f"aux={{{', '.join(aux)}}}  {'+=' if tp.accumulate else '='}")
    if tp.body == N.BODY_GENERIC:
        for nm, cls in zip(tp.aux_names, tp.aux_classes):
            aux.append(f"{nm} {_CLASS[cls]}")
        out[-1] = (f"recognition: MMLT  A={tp.a_name} ({lay[tp.layout_a]})  "
                   f"B={tp.b_name} ({lay[tp.layout_b]})  R={tp.result_name}  "
                   f"aux={{{', '.join(aux)}}}  {'+=' if tp.accumulate else '='}")
        out.append("body: generated (NVRTC-compiled into the tile kernels at plan time)")
        out.append(f"term: {_generated_term(tp.source, a.dtype)}")
    else:
        out.append(f"body: {tp.body_name}")
        tname = tp.thres_name or f"${tp.thres_value:g}"
        prog = [s.format(t=tname, d=tp.dis_name or "dis") for s in _PROGRAMS[tp.body]]
        out.append(f"\npseudo program ({len(prog)} instructions):")
        out += ["  " + s for s in prog]
        i_h, i_w, regs = _block(tp)
        out.append(f"\nreference kernel shape: {i_h} x {i_w} ({regs} registers)")
    ctx = E.Context(a.device, dry_run=True)
    plan = ctx.plan_for(tp, a.dtype)
    out.append(f"\nB200 variants ({a.dtype}):")
    for v in plan.variants():
        out.append(f"  {v.index:2d} {v.name:<32s} block {v.block_m} x {v.block_n} x {v.block_k}"
                   f", thread {v.thread_m} x {v.thread_n}, {v.threads} threads, {v.stages} stages"
                   f", {v.smem_bytes} B smem{', tensor core' if v.tensor_core else ''}")
    M, K, N_ = _extents(tp, a.dims)
    out.append(f"default for {M} x {K} x {N_}: "
               f"{plan.variants()[plan.default_variant(M, N_, K)].name}")
    _emit(a, "\n".join(out) + "\n")
    return 0


# ---------------------------------------------------------------------------
# argument parsing


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        sys.stderr.write(f"usage error: {message}\n")
        raise SystemExit(2)


def _parser() -> argparse.ArgumentParser:
    p = _Parser(prog="amlt-b200", description="Adaptive execution engine for "
                "matrix-multiplication-like tasks (B200 backend)")
    sub = p.add_subparsers(dest="cmd", required=True)

    def task_opts(s):
        s.add_argument("--task", default="")
        s.add_argument("--preset", default="")
        s.add_argument("--dtype", default="f64", choices=["f64", "f32", "i32"])
        s.add_argument("--device", type=int, default=0)
        s.add_argument("--f64-emulation", action="store_true",
                       help="let the tuner use the int8-tensor-core f64 GEMM (opt-in)")
        s.add_argument("--dims", type=int, nargs=3, default=[512, 512, 512],
                       metavar=("M", "K", "N"))
        s.add_argument("--out", default="")

    def data_opts(s):
        s.add_argument("--layout-a", default="row", choices=["row", "col"])
        s.add_argument("--layout-b", default="row", choices=["row", "col"])
        s.add_argument("--seed", type=int, default=1)
        s.add_argument("--data", default="int", choices=["int", "real"])
        s.add_argument("--packing", action="store_true")
        s.add_argument("--a-file", default="")
        s.add_argument("--b-file", default="")

    r = sub.add_parser("run")
    task_opts(r)
    data_opts(r)
    r.add_argument("--mode", default="adaptive", choices=["adaptive", "fixed", "naive"])
    r.add_argument("--kc", type=int, default=0)
    r.add_argument("--nc", type=int, default=0)
    r.add_argument("--verify", action="store_true")
    r.add_argument("--format", default="table", choices=["json", "csv", "table"])
    r.add_argument("--trials", type=int, default=3)
    r.add_argument("--agg", default="min", choices=["min", "mean"])
    t = sub.add_parser("tune")
    task_opts(t)
    data_opts(t)
    t.add_argument("--tuner", default="amulet", choices=["amulet", "gpu"])
    b = sub.add_parser("bench")
    task_opts(b)
    data_opts(b)
    b.add_argument("--trials", type=int, default=3)
    b.add_argument("--agg", default="min", choices=["min", "mean"])
    e = sub.add_parser("explain")
    task_opts(e)
    return p


def _error_class(e: Exception) -> str:
    if isinstance(e, TaskError):
        return "parse error"
    if isinstance(e, E.UnsupportedExpression):
        return "unsupported expression"
    if isinstance(e, E.NoFeasibleKernel):
        return "no feasible kernel"
    if isinstance(e, E.MissingBinding):
        return "missing binding"
    if isinstance(e, E.NonPositiveTime):
        return "non-positive time"
    return "error"


def main(argv: Optional[List[str]] = None) -> int:
    a = _parser().parse_args(argv)
    try:
        return {"run": cmd_run, "tune": cmd_tune, "bench": cmd_bench,
                "explain": cmd_explain}[a.cmd](a)
    except UsageError as e:
        sys.stderr.write(f"usage error: {e}\n")
        return 2
    except RecognitionFailed as e:
        sys.stderr.write(f"recognition failed: {e}\n")
        return 3
    except (E.EngineError, TaskError) as e:
        sys.stderr.write(f"{_error_class(e)}: {e}\n")
        return 2


if __name__ == "__main__":
    sys.exit(main())
