#!/usr/bin/env python
"""Benchmark of the MMLT hot path on B200 — one JSON line on rank 0.

Default workload = BASELINE config 4, the one quoted at 1/2/4/8 GPUs:
discount body, fp64, M = N = 32768, K = 8192, inputs drawn from config 0's
distributions (A integers 0..9, B U[1,100), thres U[50,450), dis U[0,0.3)),
R zero-initialised. A "step" is one pass of the hot path over that whole
problem: R += sum_k body(A, B, thres, dis).

Multi-GPU: `bench.py --gpus N` with WORLD_SIZE unset re-launches itself
under torch.distributed.run (one process per GPU, NCCL); under torchrun
WORLD_SIZE must equal --gpus. Rank r owns R / A rows [r*M/n, (r+1)*M/n)
(64-row edges); B and the per-column vectors come from rank 0 (NCCL
broadcast over NVLink), no reduction: rows of R are independent. The total
problem is fixed as n grows (strong scaling).

Legs:
  value     device-resident inputs; K timed steps of the tuned winner through
            the public API (one enqueue per step), CUDA events on the launch
            stream, max over ranks.
  verified  after the timed region: the same winner once more on a zeroed R,
            then the CPU oracle (oracle/, the checker only) on the first and
            last row of every rank's band plus random rows x sampled columns.
  e2e       the same metric through the host-buffer C-ABI entry
            (amlt_gpu_run_host) from pinned host memory: every step copies
            A (each rank its rows) and B / thres / dis (rank 0 only; NCCL
            broadcast to the other ranks inside the call, panel by panel) H2D
            and R D2H, all inside the timed region.
  roofline  (A) matmul-like flops (2 per inner iteration) against the pipe
            peak measured in this run; (B) the reference program's body-op
            flops (the statement's compiled pseudo-program, counted by the
            native recogniser); (C) pipe-busy % and DRAM bytes of the reported
            tile from its committed ncu capture (profiles/r*/ncu_keyed.json).
  cpu_baseline  the UNMODIFIED reference engine (oracle/_ref) on the box's
            host cores, rank 0 at N=1 only, on a bounded sample of the same
            workload, extrapolated by rate (reference arm: --impl reference).
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import socket
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("matmul-like GFLOP/s (inner iters/s) & fraction of FMA/tensor peak, "
          "1/2/4/8 B200")

WORKLOADS = {
    # name: (body, dtype, M, K, N)
    "cfg4_discount_f64": ("discount", "f64", 32768, 8192, 32768),
    "cfg0_discount_f64": ("discount", "f64", 1024, 1024, 1024),
    "cfg1_boost_f32": ("boost", "f32", 4096, 4096, 4096),
    "cfg1_boost_f64": ("boost", "f64", 4096, 4096, 4096),
    "cfg2_gemm_f64": ("gemm", "f64", 8192, 8192, 8192),
    "cfg2_gemm_f32": ("gemm", "f32", 8192, 8192, 8192),
    "cfg3_sqdiff_f32": ("sqdiff", "f32", 65536, 1024, 256),
    "cfg3_eqcount_i32": ("eqcount", "i32", 65536, 1024, 256),
}
TEXT = {"discount": "A[i][k]*B[k][j] - (A[i][k]*B[k][j] > thres[j])*A[i][k]*B[k][j]*dis[j]",
        "boost": "A[i][k]*B[k][j] + (A[i][k]*B[k][j] > thres[j])*(A[i][k]*B[k][j] - thres[j])",
        "gemm": "A[i][k]*B[k][j]", "sqdiff": "(A[i][k] - B[k][j])*(A[i][k] - B[k][j])",
        "eqcount": "A[i][k] == B[k][j]"}
PIPE = {"f64": "dfma", "f32": "ffma", "i32": "alu"}
TOL = {"f64": 1e-12, "f32": 1e-5, "i32": 0.0}  # BASELINE north_star tolerances vs the fp64 oracle


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    lrank = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, lrank


def task_source(body):
    return ("where(i in [0..M] and j in [0..N] and k in [0..K]) {\n  R[i][j] += "
            + TEXT[body] + ";\n}\n")


# ---------------------------------------------------------------------------
# rank launch


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: re-run this command as N ranks
    (torch.distributed.run, one process per GPU); rank 0's JSON line passes
    through on stdout."""
    import torch

    have = torch.cuda.device_count()
    if have < n and "--dry-run" not in sys.argv:
        log(f"bench.py: --gpus {n} but only {have} CUDA device(s) are visible")
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.abspath(__file__), *sys.argv[1:]]
    log("bench.py: launching", " ".join(cmd))
    return subprocess.call(cmd)


class NcclLog:
    """NCCL_DEBUG=INFO for the communicator lines (nranks, rank, NVLS /
    transport choices), written to a per-rank file and echoed to stderr at
    the end so stdout keeps exactly one JSON line."""

    def __init__(self, rank: int):
        self.path = None
        if "NCCL_DEBUG_FILE" not in os.environ:
            self.path = os.path.join(tempfile.gettempdir(), f"amlt_bench_nccl.{os.getpid()}.r{rank}.log")
            os.environ["NCCL_DEBUG_FILE"] = self.path
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,ENV")
        self.rank = rank

    def echo(self):
        if not self.path or not os.path.exists(self.path):
            return
        with open(self.path, errors="replace") as f:
            for line in f:
                if any(s in line for s in ("nranks", "Init COMPLETE", "NVLS", "comm ", "NCCL version")):
                    log(f"[nccl rank {self.rank}] {line.rstrip()}")
        os.unlink(self.path)


# ---------------------------------------------------------------------------
# clocks sampled during the timed region


class ClockSampler:
    def __init__(self, gpu_index: int):
        self.path = tempfile.mktemp(prefix="clocks_", suffix=".csv")
        self.proc = None
        self.gpu = gpu_index

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.f.close()
        sm, mx, pw, reasons = [], None, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx = float(parts[2])
                    pw.append(float(parts[3]))
                except ValueError:
                    continue
                for n, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        os.unlink(self.path)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(pw) if pw else None}


# ---------------------------------------------------------------------------
# data


def gen_shared(body, dtype, K, N, device):
    """B and the per-column vectors with BASELINE's distributions (seeded)."""
    import torch

    tdt = {"f64": torch.float64, "f32": torch.float32, "i32": torch.int32}[dtype]
    g = torch.Generator(device=device)
    g.manual_seed(1)
    th = ds = None
    if body == "discount":
        Bv = torch.empty((K, N), dtype=tdt, device=device).uniform_(1, 100, generator=g)
        th = torch.empty(N, dtype=tdt, device=device).uniform_(50, 450, generator=g)
        ds = torch.empty(N, dtype=tdt, device=device).uniform_(0, 0.3, generator=g)
    elif body == "boost":
        Bv = torch.rand((K, N), dtype=tdt, device=device, generator=g)
        th = torch.empty(N, dtype=tdt, device=device).uniform_(0.25, 0.75, generator=g)
    elif body == "gemm":
        Bv = torch.randn((K, N), dtype=tdt, device=device, generator=g)
    elif body == "sqdiff":
        Bv = torch.empty((K, N), dtype=tdt, device=device).uniform_(-1, 1, generator=g)
    else:  # eqcount
        Bv = torch.randint(0, 16, (K, N), dtype=tdt, device=device, generator=g)
    return Bv, th, ds


def gen_rows(body, dtype, rows, K, row0, device):
    """This rank's rows of A (seeded by the first row, so any split gives the
    same A for the same rows only per split; the oracle check uses the rows
    each rank actually holds)."""
    import torch

    tdt = {"f64": torch.float64, "f32": torch.float32, "i32": torch.int32}[dtype]
    ga = torch.Generator(device=device)
    ga.manual_seed(1000 + row0)
    if body == "discount":
        return torch.randint(0, 10, (rows, K), device=device, generator=ga).to(tdt)
    if body == "boost":
        return torch.rand((rows, K), dtype=tdt, device=device, generator=ga)
    if body == "gemm":
        return torch.randn((rows, K), dtype=tdt, device=device, generator=ga)
    if body == "sqdiff":
        return torch.empty((rows, K), dtype=tdt, device=device).uniform_(-1, 1, generator=ga)
    return torch.randint(0, 16, (rows, K), dtype=tdt, device=device, generator=ga)


# ---------------------------------------------------------------------------
# reference CPU arm


def reference_sample(body, M, K, N, threads):
    """A bounded sample of the workload for the reference engine: 12 rows per
    thread (>= the reference's i_h, so every band is tuned as in a full run)
    x min(N, 4096) columns x full K — about 10 s of CPU work at the
    reference's ~0.1 G iterations/s per thread on the interpreted bodies.
    Rows are independent, so the sample's rate is the workload's rate."""
    rows = min(M, 12 * threads)
    cols = min(N, 8192 if body == "gemm" else 4096)
    return rows, K, cols


def run_reference(body, M, K, N, steps, warmup, threads):
    import numpy as np

    from oracle import pyoracle as po

    text = {"discount": po.preset_source("q1"), "boost": po.preset_source("q2"),
            "gemm": po.preset_source("matmul"), "sqdiff": po.SQDIFF_TEXT,
            "eqcount": po.EQCOUNT_TEXT}[body]
    rows, K_, cols = reference_sample(body, M, K, N, threads)
    t = po.RefTask.create(text, rows, K_, cols, seed=1, int_valued=False)
    rng = np.random.default_rng(1)
    if body == "discount":
        t.set("A", rng.integers(0, 10, (rows, K_)).astype(np.float64))
        t.set("B", rng.uniform(1, 100, (K_, cols)))
        t.set("thres", rng.uniform(50, 450, cols))
        t.set("dis", rng.uniform(0, 0.3, cols))
    elif body == "boost":
        t.set("A", rng.uniform(0, 1, (rows, K_)))
        t.set("B", rng.uniform(0, 1, (K_, cols)))
        t.set("thres", rng.uniform(0.25, 0.75, cols))
    elif body == "gemm":
        t.set("A", rng.standard_normal((rows, K_)))
        t.set("B", rng.standard_normal((K_, cols)))
    elif body == "sqdiff":
        t.set("A", rng.uniform(-1, 1, (rows, K_)))
        t.set("B", rng.uniform(-1, 1, (K_, cols)))
    else:
        t.set("A", rng.integers(0, 16, (rows, K_)).astype(np.float64))
        t.set("B", rng.integers(0, 16, (K_, cols)).astype(np.float64))
    times = []
    for s in range(warmup + steps):
        el = t.run_adaptive_bands(threads)
        if s >= warmup:
            times.append(el)
    iters = rows * K_ * cols
    sec = sum(times) / len(times)
    return {"iters_per_s": iters / sec, "seconds_per_sample": sec,
            "sample_fraction": (rows * cols) / (M * N),
            "sample": f"{rows} rows x {cols} cols x K={K_} of the workload "
                      f"({iters / 1e9:.2f} G inner iterations), reference adaptive_execute "
                      f"on {threads} row bands (one std::thread each), seed-1 BASELINE "
                      f"distributions; the workload's rate is extrapolated from the sample's "
                      f"(rows of R are independent)"}


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# roofline helpers


def ncu_capture_for(workload, tile):
    """Pipe-busy % and DRAM bytes per launch of `tile` on `workload` from the
    newest committed keyed ncu capture (profiles/r*/ncu_keyed.json), or None."""
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_keyed.json")), reverse=True):
        try:
            d = json.load(open(path)).get(workload, {})
        except (OSError, ValueError):
            continue
        if tile in d:
            e = dict(d[tile])
            e["file"] = os.path.relpath(path, ROOT)
            return e
    return None


def algorithmic_bytes(body, dtype, M, K, N):
    """Compulsory HBM bytes per launch: A, B, R read + R write, vectors."""
    es = 8 if dtype == "f64" else 4
    vec = {"discount": 2, "boost": 1}.get(body, 0) * N
    return es * (M * K + K * N + 2 * M * N + vec)


def hbm_peak_gbs():
    """MEASURED_PEAKS.json's copy bandwidth (driver-written), or None."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return None


def cap_rows(cap, workload):
    """Rows of R the keyed capture's launch covered: the whole workload at
    N=1 (tools/capture_keyed.sh); a rank's band scales the traffic by its
    share of the rows."""
    return cap.get("rows") or WORKLOADS[workload][2]


def tensor_tf32_peak() -> float:
    """Dense TF32 tensor-core TFLOP/s: the driver-measured dense bf16 figure
    (MEASURED_PEAKS.json, burst) halved (TF32 runs at half the bf16 rate on
    B200); the B200_PROFILING.md fallback (2250 bf16) when absent."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"]) / 2.0
    except Exception:  # noqa: BLE001
        return 2250.0 / 2.0


def launches_of(name: str, split: bool) -> int:
    """Kernel launches one enqueue of the winner makes."""
    if "tcgen05_3xtf32" in name:
        return 3  # operand split of A, of B, the tensor-core GEMM
    if "ozaki" in name:
        return 5  # row / column exponents, A / B slicing, the int8 GEMM
    if "_theta_" in name:
        # B preparation and A scan in one launch, the tile, the guard-exited
        # fallback (+ the ordered split-K reduce)
        return 3 + (1 if split else 0)
    if "_swar_" in name:
        return 4  # B packing, A packing, the tile, the guard-exited fallback
    return 2 if split else 1


# ---------------------------------------------------------------------------
# legs


def verify_rows(P, plan, win, A, B, th, ds, R, body, dtype, rows, rank, row0, stream):
    """The timed winner once more on a zeroed R, then the oracle on this
    rank's first and last row plus random rows x sampled columns."""
    import numpy as np
    import torch

    from oracle import pyoracle as po

    M, K, N = rows, A.shape[1], B.shape[1]
    R.zero_()
    P.enqueue(plan, P.Operands(A, B, R, th, ds), win, P.Bounds(0, M, 0, N, 0, K))
    torch.cuda.synchronize()
    rng = np.random.default_rng(17 + rank)
    ri = sorted({0, M - 1} | set(int(x) for x in rng.integers(0, M, 4))) if M > 0 else []
    ci = sorted({0, N - 1} | set(int(x) for x in rng.integers(0, N, 510)))
    if not ri:
        return 0, len(ci), 0.0, 0
    idx = torch.tensor(ri, device=A.device)
    cdx = torch.tensor(ci, device=A.device)
    got = R[idx][:, cdx].double().cpu().numpy()
    Ah = A[idx].double().cpu().numpy()
    Bh = B[:, cdx].double().cpu().numpy()
    th_h = th[cdx].double().cpu().numpy() if th is not None else None
    ds_h = ds[cdx].double().cpu().numpy() if ds is not None else None
    return (len(ri), len(ci)) + check_rows(got, Ah, Bh, th_h, ds_h, body, dtype)


def check_rows(got, Ah, Bh, th_h, ds_h, body, dtype):
    """(max relative error, mismatches) of sampled R rows x columns against
    the C oracle on the same rows of A and columns of B / thres / dis."""
    import numpy as np

    from oracle import pyoracle as po

    kind = {"gemm": po.GEMM, "discount": po.DISCOUNT, "boost": po.BOOST, "sqdiff": po.SQDIFF,
            "eqcount": po.EQCOUNT}[body]
    ri = range(got.shape[0])
    ci = range(got.shape[1])
    want = np.zeros((len(ri), len(ci)))
    po.oracle_run(kind, Ah, Bh, want, thres=th_h, dis=ds_h)
    if dtype == "i32" or body == "eqcount":
        return 0.0, int((got != want).sum())
    err = np.abs(got - want)
    if body in ("gemm", "sqdiff"):  # normwise: |d| <= tol * sum_k |term_k|
        if body == "gemm":
            scale = np.abs(Ah) @ np.abs(Bh)
        else:
            scale = (Ah * Ah) @ np.ones_like(Bh) + np.ones_like(Ah) @ (Bh * Bh) + 2 * np.abs(Ah) @ np.abs(Bh)
    else:
        scale = np.abs(want)
    rel = err / np.maximum(scale, np.finfo(np.float64).tiny)
    return float(rel.max()), int((rel > TOL[dtype]).sum())


def cuda_core_leg(P, plan, ops, bounds, stream, steps, M, K, N, peak_ffma_tflops):
    """Config 2 fp32 as BASELINE writes it (the CUDA-core path): the fastest
    SIMT FFMA tile, timed like the value leg (the tuner picks the tcgen05
    3xTF32 GEMM for the headline)."""
    import torch

    best = None
    for vi, v in enumerate(plan.variants()):
        if v.tensor_core or "tcgen05" in v.name or v.name.endswith("_u"):
            continue
        tp = P.TileParams(variant=vi)
        try:
            P.enqueue(plan, ops, tp, bounds)
        except P.EngineError:
            continue
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(max(steps, 2)):
            P.enqueue(plan, ops, tp, bounds)
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / max(steps, 2)
        if best is None or t < best[1]:
            best = (v.name, t)
    if best is None:
        return None
    tf = 2 * M * K * N / best[1] / 1e12
    return {"value": tf * 1e3, "unit": "GFLOP/s", "tile": best[0], "ms_per_step": best[1] * 1e3,
            "frac_of_ffma_peak": tf / peak_ffma_tflops,
            "note": "BASELINE config 2 fp32 on the CUDA-core FFMA path, best SIMT tile; the headline "
                    "value is the tcgen05 3xTF32 tensor-core GEMM the tuner picks"}


# ---------------------------------------------------------------------------
# CPU dry run of the multi-rank plumbing


def dry_run(args, body, dtype, M, K, N, ws, rank):
    """The harness's multi-rank logic on CPU (gloo): each rank's row band,
    B and the vectors made on rank 0 and broadcast, a checksum of them
    gathered from every rank, the max-over-ranks reduction; rank 0 prints one
    JSON line with "dry_run": true and no measured value."""
    import torch

    from paper_2305_08872_b200.sharded import row_band

    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")
    row0, row1 = row_band(M, ws, rank, align=64)
    kk, nn = min(K, 64), min(N, 64)  # a corner of B stands in for the whole
    g = torch.Generator().manual_seed(1 + rank)  # ranks differ until the broadcast
    Bv = torch.rand((kk, nn), dtype=torch.float64, generator=g)
    vec = torch.rand(nn, dtype=torch.float64, generator=g)
    if dist is not None:
        dist.broadcast(Bv, src=0)
        dist.broadcast(vec, src=0)
    local = torch.tensor([float(row0), float(row1), float(Bv.sum() + vec.sum()), float(rank + 1)],
                         dtype=torch.float64)
    parts = [torch.zeros_like(local) for _ in range(ws)]
    if dist is not None:
        dist.all_gather(parts, local)
        el = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
    else:
        parts = [local]
        el = torch.tensor([1.0])
    if rank == 0:
        print(json.dumps({"dry_run": True, "value": None, "metric": METRIC, "n_gpus": ws,
                          "config": {"workload": args.workload, "body": body, "dtype": dtype,
                                     "M": M, "K": K, "N": N, "parallelism": f"rowshard{ws}"},
                          "bands": [[int(p[0].item()), int(p[1].item())] for p in parts],
                          "shared_checksums": [float(p[2].item()) for p in parts],
                          "max_over_ranks": float(el.item())}), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# main


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4_discount_f64", choices=sorted(WORKLOADS))
    ap.add_argument("--tile", default=None,
                    help="skip the tuner and run this tile variant (name from plan.variants()); "
                         "used to pin the tuned winner under ncu, whose serialised launches "
                         "change the trial timings")
    ap.add_argument("--kc", type=int, default=0, help="with --tile: the K-segment depth (split-K)")
    ap.add_argument("--no-graph", action="store_true",
                    help="value leg: plain enqueue per step instead of replaying the step from a "
                         "CUDA graph (amlt_gpu_graph_capture)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU only (gloo): rank launch, row bands, the broadcast of B / vectors and "
                         "the max-over-ranks reduction, with no kernel and no timing claim "
                         "(tests/test_bench_harness.py)")
    ap.add_argument("--proxy-band", type=int, default=0, metavar="N",
                    help="one GPU: time only rank 0's row band of an N-way split (what each rank "
                         "of an N-GPU run computes), B / vectors copied by this rank; the line is "
                         "labelled 'proxy' and is not a multi-GPU measurement")
    ap.add_argument("--f64-emulation", action="store_true",
                    help="let the tuner use the int8-tensor-core f64 GEMM (AMLT_CTX_F64_EMULATION)")
    args = ap.parse_args()
    body, dtype, M, K, N = WORKLOADS[args.workload]
    steps, warmup = args.steps, max(args.warmup, 0)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        return spawn_ranks(args.gpus)
    ws, rank, lrank = dist_env()
    if "WORLD_SIZE" in os.environ and ws != args.gpus:
        log(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; launch one rank per GPU")
        return 2

    proxy = args.proxy_band if args.proxy_band > 1 else 0
    if proxy and (ws > 1 or args.gpus > 1):
        log("bench.py: --proxy-band is a one-GPU measurement; run it with --gpus 1 outside torchrun")
        return 2

    if args.dry_run:
        return dry_run(args, body, dtype, M, K, N, ws, rank)

    if args.impl == "reference":
        if rank != 0:
            return 0
        threads = cpu_threads()
        r = run_reference(body, M, K, N, steps, warmup, threads)
        gf = 2 * r["iters_per_s"] / 1e9
        line = {"impl": "reference", "metric": METRIC, "value": gf, "unit": "GFLOP/s",
                "inner_iters_per_s": r["iters_per_s"], "n_gpus": args.gpus, "steps": steps,
                "warmup": warmup, "ms_per_step": r["seconds_per_sample"] * 1e3,
                "ms_per_step_note": "seconds of one bounded sample (see cpu_baseline.sample); the "
                                    "workload's rate is extrapolated from it",
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": {"workload": args.workload, "body": body, "M": M, "K": K, "N": N,
                           "parallelism": f"cpu_threads{threads}"},
                "cpu_baseline": {"value": gf, "unit": "GFLOP/s", "cores": threads,
                                 "kind": "reference", "sample": r["sample"],
                                 "extrapolated_from_sample": True,
                                 "sample_fraction": r["sample_fraction"], "cpu_model": cpu_model()},
                "e2e": {"value": gf, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    # the GPU arm always warms up at least 3 steps (the first one tunes)
    warmup = max(warmup, 3)
    nccl_log = NcclLog(rank) if ws > 1 else None
    import numpy as np
    import torch

    import paper_2305_08872_b200 as P
    from paper_2305_08872_b200.sharded import row_band
    from paper_2305_08872_b200.task import compile_task

    assert torch.cuda.is_available(), "bench.py needs a CUDA device"
    torch.cuda.set_device(lrank)
    device = torch.device("cuda", lrank)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=device)
    row0, row1 = row_band(M, proxy or ws, rank, align=64)
    rows = row1 - row0
    if proxy:
        M = rows  # the work of this step: rank 0's band

    ctx = P.Context(lrank, f64_emulation=args.f64_emulation)
    # one explicit (non-default) stream for torch and the kernels alike, so the
    # CUDA events below bracket exactly the launches
    stream = torch.cuda.Stream(device)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream)
    task = compile_task(task_source(body))
    plan = ctx.plan_for(task, dtype)

    # roofline denominator, measured on this GPU now
    pipe = PIPE[dtype] if not (body == "gemm" and dtype == "f64") else "dmma"
    peak_ops, peak_ghz = P.engine.measure_peak(pipe)
    if pipe == "alu":
        # integer bodies are issue-bound: the ceiling is the SM's issue rate,
        # 4 schedulers x 32 lanes per clock
        props = torch.cuda.get_device_properties(device)
        peak_tflops = 128 * props.multi_processor_count * peak_ghz * 1e9 / 1e12
    else:
        peak_tflops = 2 * peak_ops / 1e12

    B, th, ds = gen_shared(body, dtype, K, N, device)
    if dist is not None:  # input placement before timing: B and the vectors from rank 0
        for t in (B, th, ds):
            if t is not None:
                dist.broadcast(t, src=0)
    A = gen_rows(body, dtype, rows, K, row0, device)
    R = torch.zeros((rows, N), dtype=A.dtype, device=device)
    ops = P.Operands(A, B, R, th, ds)
    bounds = P.Bounds(0, rows, 0, N, 0, K)
    torch.cuda.synchronize()

    # warm-up: the first call tunes on row bands (AMULET-style), later calls
    # reuse the cached winner
    reports = []
    if args.tile:
        from types import SimpleNamespace

        vi = [v.name for v in plan.variants()].index(args.tile)
        for _ in range(warmup):
            P.run_subtask(plan, ops, P.TileParams(kc=args.kc, variant=vi), bounds)
        reports.append(SimpleNamespace(best_variant=vi, best_kc=args.kc if 0 < args.kc < K else K, tuned=False,
                                       scratch_tuned=False, trials=[]))
    else:
        for _ in range(warmup):
            reports.append(P.adaptive_execute(plan, ops, bounds))
    torch.cuda.synchronize()
    tuned = reports[0] if reports else None

    def barrier():
        if dist is not None:
            dist.barrier()

    # ---- value leg
    # Inputs that fit the 126 MB L2 (with margin) get an L2 flush between
    # timed steps; larger ones stream from HBM anyway.
    in_bytes = sum(x.numel() * x.element_size() for x in (A, B, R) if x is not None)
    flush = in_bytes < (256 << 20)
    flush_buf = torch.empty(512 << 20, dtype=torch.uint8, device=device) if flush else None
    sampler = ClockSampler(lrank)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    last = reports[-1] if reports else None
    win = P.TileParams(kc=last.best_kc if last and last.best_kc < K else 0,
                       variant=last.best_variant if last else -1)
    variants = plan.variants()
    win_name = variants[win.variant].name if win.variant is not None and win.variant >= 0 else ""
    split = bool(last and last.best_kc < K)
    # the step as a CUDA graph: every kernel of it, replayed with no
    # per-launch host work (the capture runs one plain step first)
    graph = None
    if not args.no_graph:
        try:
            graph = P.capture_graph(plan, ops, win, bounds)
        except P.EngineError as e:
            log(f"bench.py: graph capture failed ({e}); timing plain enqueues")
    step_launch = "cuda-graph replay" if graph is not None else "enqueue"
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.3)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    launches = 0
    for s in range(steps):
        if flush:
            flush_buf.zero_()  # evict L2 (outside the step's events)
        ev[s][0].record(stream)
        if graph is not None:
            graph.launch()
        else:
            P.enqueue(plan, ops, win, bounds)
        ev[s][1].record(stream)
        launches += launches_of(win_name, split)
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    el = t0.elapsed_time(t1) / 1e3
    per_launch = [a.elapsed_time(b) / 1e3 for a, b in ev]
    if flush:
        el = sum(per_launch)  # the flushes are not part of the work
    if dist is not None:
        tt = torch.tensor([el], dtype=torch.float64, device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        el = float(tt.item())
    iters_total = M * K * N * steps
    value = 2 * iters_total / el / 1e9
    kernel_s = sum(per_launch) / len(per_launch)
    achieved_tflops = 2 * rows * K * N / kernel_s / 1e12
    tensor_tf32 = "tcgen05_3xtf32" in win_name
    ozaki = "ozaki" in win_name
    if ozaki:
        # int8 tensor cores, 28 slice GEMMs per f64 GEMM (7 slices, diagonals
        # 2..8); int8 dense = 2 x bf16 dense on B200
        peak_tflops, pipe = tensor_tf32_peak() * 4.0 / 28.0, "tcgen05.kind::i8 (Ozaki, 28 slice GEMMs)"
        tensor_tf32 = True
    elif tensor_tf32:
        # 3 TF32 MMAs per product (3xTF32); TF32 dense is half the bf16 rate
        peak_tflops, pipe = tensor_tf32_peak() / 3.0, "tcgen05.kind::tf32 (3xTF32)"

    # ---- config 2 fp32 on the CUDA-core path, beside the tensor-core headline
    cuda_core = None
    if args.workload == "cfg2_gemm_f32" and rank == 0 and ws == 1:
        ffma_ops, _ = P.engine.measure_peak("ffma")
        cuda_core = cuda_core_leg(P, plan, ops, bounds, stream, steps, rows, K, N, 2 * ffma_ops / 1e12)

    # ---- verified: the timed winner, re-run once on a zeroed R, vs the oracle
    verified = None
    if not args.no_verify:
        nr, nc, worst, bad = verify_rows(P, plan, win, A, B, th, ds, R, body, dtype, rows, rank, row0,
                                         stream)
        if dist is not None:
            tt = torch.tensor([nr, worst, bad], dtype=torch.float64, device=device)
            parts = [torch.zeros_like(tt) for _ in range(ws)]
            dist.all_gather(parts, tt)
            nr = int(sum(p[0].item() for p in parts))
            worst = max(p[1].item() for p in parts)
            bad = int(sum(p[2].item() for p in parts))
        verified = {"rows": nr, "cols": nc, "max_rel": worst, "tol": TOL[dtype], "mismatches": bad,
                    "ok": bad == 0,
                    "how": "the timed winner re-run once on a zeroed R after the timed region; the "
                           "C oracle (oracle/liboracle.so, pinned to the reference's run_naive) on the "
                           "first and last row of every rank's band plus random rows x sampled columns"
                           + ("; normwise for gemm/sqdiff" if body in ("gemm", "sqdiff") else "")}

    # ---- e2e leg: host buffers through the C-ABI host entry
    e2e = None
    if not args.no_e2e:
        hA = A.cpu().pin_memory()
        hB = B.cpu().pin_memory() if rank == 0 else P.Shape(K, N, dtype)
        hth = (th.cpu().pin_memory() if rank == 0 else P.Shape(N, 1, dtype)) if th is not None else None
        hds = (ds.cpu().pin_memory() if rank == 0 else P.Shape(N, 1, dtype)) if ds is not None else None
        hR = torch.empty((rows, N), dtype=A.dtype).pin_memory()
        hops = P.Operands(hA, hB, hR, hth, hds)
        # columns kept for checking the e2e result afterwards (every rank)
        rng = np.random.default_rng(29 + rank)
        e_ci = sorted({0, N - 1} | set(int(x) for x in rng.integers(0, N, 254)))
        e_ri = sorted({0, rows - 1} | set(int(x) for x in rng.integers(0, rows, 6))) if rows > 0 else []
        cdx = torch.tensor(e_ci, device=B.device)
        e_B = B[:, cdx].double().cpu().numpy()
        e_th = th[cdx].double().cpu().numpy() if th is not None else None
        e_ds = ds[cdx].double().cpu().numpy() if ds is not None else None
        if graph is not None:
            graph.close()  # (it holds the value leg's operands)
            graph = None
        del A, B, R, ops
        torch.cuda.empty_cache()
        bcast = ws > 1
        e2e_error = None
        if bcast:
            def exchange(uid):
                box = [uid]
                dist.broadcast_object_list(box, src=0)
                return box[0]

            ctx.attach_comm(rank, ws, exchange=exchange)
        tms = []
        # --tile pins the e2e leg's tile too (else: the winner the value leg's
        # warm-up tuned and cached for this shape)
        e2e_tp = win if args.tile else None
        try:
            P.run_host(plan, hops, bounds, params=e2e_tp, r_zero=True, bcast=bcast)  # warm-up (staging alloc)
            barrier()
            for _ in range(steps):
                tms.append(P.run_host(plan, hops, bounds, params=e2e_tp, r_zero=True, bcast=bcast))
        except P.EngineError as e:  # reported in the line, not fatal to the value leg
            e2e_error = f"rank {rank}: {e}"
            log("bench.py: e2e leg failed:", e2e_error)
            tms = [float("inf")]
        e_el = sum(tms)
        layout = ctx.last_host_layout() if not e2e_error else {}
        if dist is not None:
            tt = torch.tensor([e_el], dtype=torch.float64, device=device)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_el = float(tt.item())
        es = hA.element_size()
        # bytes this rank copies per step: its A rows (+ B and the vectors on
        # rank 0, the only rank that reads them from host memory), its R rows
        shared = sum(x.numel() for x in (hB, hth, hds) if isinstance(x, torch.Tensor)) * es
        h2d_total, d2h_total = float(hA.numel() * es + shared), float(hR.numel() * es)
        if dist is not None:
            tt = torch.tensor([h2d_total, d2h_total], dtype=torch.float64, device=device)
            dist.all_reduce(tt)
            h2d_total, d2h_total = float(tt[0].item()), float(tt[1].item())
        e2e = {"value": 2 * iters_total / e_el / 1e9 if e_el != float("inf") else None, "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(h2d_total),
               "d2h_bytes_per_step": int(d2h_total),
               "ms_per_step": e_el / steps * 1e3,
               "path": ("amlt_gpu_run_host (C-ABI) from pinned host buffers: B in K panels and A in row "
                        "bands H2D (each rank its own A rows), pipelined against compute; band 0 computed "
                        "panel by panel as B lands "
                        "(its R zero-filled on the device, D2H afterwards); "
                        + ("the other rows in one launch whose epilogue writes R straight into the pinned "
                           "host buffer (zero-copy)" if layout.get("zero_copy_r") else
                           "the other row bands whole-K, each R band D2H as soon as it is done")
                        + ("; B / thres / dis read on rank 0 only and NCCL-broadcast panel by panel "
                           "inside the call" if bcast else "")),
               "layout": layout}
        if e2e_error:
            e2e["error"] = e2e_error
        if not args.no_verify:
            # the last timed step's R, as it landed in host memory (every rank
            # joins the gather below, a failed one with no rows checked)
            if e2e_error or not e_ri:
                worst, bad, nr = 0.0, 0, 0
            else:
                worst, bad = check_rows(hR[e_ri][:, e_ci].double().numpy(), hA[e_ri].double().numpy(), e_B,
                                        e_th, e_ds, body, dtype)
                nr = len(e_ri)
            if dist is not None:
                tt = torch.tensor([nr, worst, bad], dtype=torch.float64, device=device)
                parts = [torch.zeros_like(tt) for _ in range(ws)]
                dist.all_gather(parts, tt)
                nr = int(sum(p[0].item() for p in parts))
                worst = max(p[1].item() for p in parts)
                bad = int(sum(p[2].item() for p in parts))
            e2e["verified"] = {"rows": nr, "cols": len(e_ci), "max_rel": worst, "mismatches": bad, "ok": bad == 0,
                               "how": "the last timed step's R in host memory, sampled rows x columns, "
                                      "against the C oracle"}

    # ---- CPU baseline (rank 0, N = 1)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        try:
            threads = cpu_threads()
            r = run_reference(body, M, K, N, 1, 0, threads)
            # the reference's own single-threaded mode (run_adaptive) beside it
            r1 = run_reference(body, M, K, N, 1, 0, 1) if threads > 1 else r
            cpu = {"value": 2 * r["iters_per_s"] / 1e9, "unit": "GFLOP/s", "cores": threads,
                   "kind": "reference", "sample": r["sample"], "extrapolated_from_sample": True,
                   "sample_fraction": r["sample_fraction"], "cpu_model": cpu_model(),
                   "value_1thread": 2 * r1["iters_per_s"] / 1e9,
                   "sample_1thread": r1["sample"]}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "GFLOP/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        best = last.best_variant if last else -1
        tile = variants[best].name if best >= 0 else None
        cap = ncu_capture_for(args.workload, tile) if tile else None
        if cap is None:
            log(f"bench.py: no committed ncu capture of tile {tile} for {args.workload} "
                "(profiles/r*/ncu_keyed.json): roofline.pipe_busy and traffic are null")
        iters_per_s_kernel = rows * K * N / kernel_s
        body_flops = task.program_flops
        # (B): the reference program's body-op flops per second against the
        # same pipe peak in flops (2 per FMA lane op)
        frac_b = iters_per_s_kernel * body_flops / (peak_tflops * 1e12) if not tensor_tf32 else None
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s",
            "inner_iters_per_s": iters_total / el,
            "n_gpus": ws, "steps": steps, "warmup": warmup, "ms_per_step": el / steps * 1e3,
            "step_ms_rank0": {"best": min(per_launch) * 1e3, "median": sorted(per_launch)[len(per_launch) // 2] * 1e3,
                              "worst": max(per_launch) * 1e3, "n": len(per_launch)},
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": dtype, "data": "synthetic",
            "config": {"workload": args.workload, "body": body, "M": M, "K": K, "N": N,
                       "parallelism": f"rowshard{ws}",
                       "l2": ("flushed between timed steps (512 MiB memset outside the step "
                              "events; value from the sum of per-step kernel times)"
                              if flush else "inputs larger than L2 (no flush)"),
                       "tile": tile,
                       "split_k_kc": win.kc or None,
                       "step_launch": step_launch,
                       "tuning": ("pinned by --tile" if args.tile else
                                  "row-band trials" if tuned and tuned.tuned else
                                  "whole-task trials on scratch R" if tuned and tuned.scratch_tuned
                                  else "planner default"),
                       "tuning_trials": [(variants[t.value].name, round(t.score * 1e6, 4))
                                         for t in tuned.trials] if tuned else []},
            "roofline": {"bound": "tensor" if tensor_tf32 else
                         ("fp64" if dtype == "f64" else ("fp32" if dtype == "f32" else "int32")),
                         "pipe": pipe, "achieved": achieved_tflops, "peak": peak_tflops,
                         "unit": "TFLOP/s", "frac": achieved_tflops / peak_tflops,
                         "peak_source": ("measured in this run by amlt_gpu_measure_peak "
                                         f"({pipe} probe at {peak_ghz:.3f} GHz)" if not tensor_tf32 else
                                         "MEASURED_PEAKS.json dense bf16 (burst), scaled as the "
                                         "accounting states"),
                         "accounting": (
                             "(A) 2 flops per inner iteration (matmul-like); 28 int8 tensor-core "
                             "slice products per iteration (Ozaki, 7 slices), peak = measured dense "
                             "bf16 x 2 (int8 rate) / 28" if ozaki else
                             "(A) 2 flops per inner iteration (matmul-like); 3 TF32 tensor-core "
                             "products per iteration (3xTF32), peak = measured dense bf16 / 2 / 3"
                             if tensor_tf32 else
                             "(A) 2 ops per inner iteration (matmul-like); peak = the SM issue rate "
                             "(128 lane-instructions/clk/SM) at the probe's clock"
                             if pipe == "alu" else
                             "(A) 2 flops per inner iteration (matmul-like); peak = 2 x the measured "
                             f"{pipe} lane-op rate on this GPU"),
                         "body_program": task.program,
                         "body_flops_per_iter": body_flops,
                         "frac_body_flops": frac_b,
                         "frac_body_flops_note": "(B): the reference's compiled program for the "
                                                 "statement (csrc/task.cpp, pinned to schedule_labelfs "
                                                 "in tests/test_task.py), add/sub/mul/div/cmp 1, "
                                                 "masksub/maskadd 2, final add 1, x iterations/s, "
                                                 "over the same peak; above 1 when the kernel needs "
                                                 "fewer pipe ops than the program states",
                         "pipe_busy": cap.get("pipe_pct") if cap else None,
                         "issue_active_pct": cap.get("issue_active_pct") if cap else None,
                         "traffic": cap.get("dram_bytes") if cap else None,
                         "traffic_unit": "bytes per launch of the tile (ncu dram read+write)",
                         # achieved HBM rate: the capture's DRAM bytes over this run's kernel time,
                         # against MEASURED_PEAKS.json's copy bandwidth (north_star's HBM GB/s)
                         "hbm_gbps": (cap["dram_bytes"] * (rows / cap_rows(cap, args.workload)) / kernel_s / 1e9
                                      if cap and cap.get("dram_bytes") else None),
                         "hbm_frac": (cap["dram_bytes"] * (rows / cap_rows(cap, args.workload)) / kernel_s / 1e9
                                      / hbm_peak_gbs() if cap and cap.get("dram_bytes") and hbm_peak_gbs()
                                      else None),
                         "capture": (f"{cap['file']}: {cap.get('capture', '')}" if cap else
                                     f"none committed for tile {tile}"),
                         "algorithmic_bytes": algorithmic_bytes(body, dtype, M, K, N),
                         "kernel_ms": kernel_s * 1e3},
            "verified": verified,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if cuda_core is not None:
            line["cuda_core"] = cuda_core
        if proxy:
            line["proxy"] = {"of_gpus": proxy, "band_rows": rows, "full_M": WORKLOADS[args.workload][2],
                             "note": "rank 0's row band of an N-way split timed alone on one GPU: every "
                                     "value here is that band's rate (M in config = the band's rows); "
                                     "the e2e leg copies B / vectors H2D itself (rank 0's share of an "
                                     "N-GPU run, without its NCCL broadcast); not a multi-GPU "
                                     "measurement"}
            line["config"]["parallelism"] = f"proxy_band_of_{proxy}"
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    if nccl_log is not None:
        nccl_log.echo()
    return 0


if __name__ == "__main__":
    sys.exit(main())
