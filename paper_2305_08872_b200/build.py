"""Builds the sm_100a shared library ``lib/libamlt_gpu.so`` in-tree.

One nvcc job per (body, dtype) instantiation unit plus the host/ABI units,
run in parallel, then one link. Incremental: an object is rebuilt when its
source or any header under csrc/ or include/ is newer.

    python -m paper_2305_08872_b200.build [--force] [-j N]

AMLT_PTXAS_<UNIT>=<flag> (e.g. AMLT_PTXAS_THETA_DISCOUNT=-O1) passes one
extra ptxas flag to one unit (scheduling experiments; touch the source so it
is rebuilt).
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build", "obj")
LIB = os.path.join(PKG, "lib", "libamlt_gpu.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
GEN = os.path.join(PKG, "build", "gen")
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
              "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include"), "-I" + GEN]

# (body template name, amlt_body id, C type, amlt_dtype id)
PAIRS = [
    ("Gemm", 0, "double", 0), ("Discount", 1, "double", 0), ("Boost", 2, "double", 0),
    ("Sqdiff", 3, "double", 0), ("Eqcount", 4, "double", 0), ("Thrcount", 5, "double", 0),
    ("Gemm", 0, "float", 1), ("Discount", 1, "float", 1), ("Boost", 2, "float", 1),
    ("Sqdiff", 3, "float", 1), ("Eqcount", 4, "float", 1), ("Thrcount", 5, "float", 1),
    ("Eqcount", 4, "int", 2), ("Thrcount", 5, "int", 2),
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _headers():
    hs = []
    for d in (CSRC, os.path.join(ROOT, "include")):
        for f in os.listdir(d):
            if f.endswith((".h", ".cuh", ".hpp")):
                hs.append(os.path.join(d, f))
    return hs


def _jobs():
    jobs = []
    inst = os.path.join(CSRC, "kernels_inst.cu")
    for body, bid, ctype, dt in PAIRS:
        out = os.path.join(OBJ, f"k_{body}_{dt}.o")
        defs = [f"-DAMLT_BODY={body}", f"-DAMLT_BODY_ID={bid}", f"-DAMLT_T={ctype}", f"-DAMLT_DT={dt}"]
        jobs.append((inst, out, defs))
    for src in ("dmma_gemm.cu", "tcgen05_gemm.cu", "ozaki_gemm.cu", "theta_discount.cu", "swar_eqcount.cu", "register_all.cu", "amlt_gpu.cu", "peak.cu", "task.cpp",
                "sharded.cu", "matrix_file.cpp", "naive.cu", "jit.cu"):
        obj = os.path.splitext(src)[0] + ".o"
        jobs.append((os.path.join(CSRC, src), os.path.join(OBJ, obj), []))
    return jobs


def _embed_kernel_header() -> None:
    """build/gen/mmlt_kernel_src.inc: the tile-kernel header as a C++ raw
    string, compiled again at run time (NVRTC) around generated bodies."""
    os.makedirs(GEN, exist_ok=True)
    src = os.path.join(CSRC, "mmlt_kernel.cuh")
    out = os.path.join(GEN, "mmlt_kernel_src.inc")
    text = open(src).read()
    assert ")AMLT_SRC" not in text
    body = 'R"AMLT_SRC(' + text + ')AMLT_SRC"\n'
    if not os.path.exists(out) or open(out).read() != body:
        with open(out, "w") as f:
            f.write(body)


def build(force: bool = False, jobs: int | None = None, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    _embed_kernel_header()
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    hdr_mtime = max(os.path.getmtime(h) for h in _headers())
    todo = []
    for src, out, defs in _jobs():
        if force or not os.path.exists(out) or os.path.getmtime(out) < max(os.path.getmtime(src), hdr_mtime):
            todo.append((src, out, defs))
    exe = nvcc()
    logs = {}

    def run(job):
        src, out, defs = job
        extra = os.environ.get("AMLT_PTXAS_" + os.path.splitext(os.path.basename(src))[0].upper(), "")
        cmd = [exe, *ARCH, *NVCC_FLAGS, *defs, *(["-Xptxas", extra] if extra else []), "-c", src, "-o", out]
        r = subprocess.run(cmd, capture_output=True, text=True)
        logs[out] = r.stdout + r.stderr
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {os.path.basename(out)}:\n{r.stderr[-4000:]}")
        return out

    if todo:
        n = jobs or min(len(todo), os.cpu_count() or 4)
        with ThreadPoolExecutor(max_workers=n) as ex:
            list(ex.map(run, todo))
        with open(os.path.join(PKG, "build", "ptxas.log"), "a") as f:
            for k, v in logs.items():
                f.write(f"==== {os.path.basename(k)}\n{v}\n")
    objs = [out for _, out, _ in _jobs()]
    if todo or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [exe, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stderr[-4000:])
    if verbose:
        print(f"built {LIB} ({len(todo)} objects recompiled)")
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    a = ap.parse_args(argv)
    build(force=a.force, jobs=a.j, verbose=True)


if __name__ == "__main__":
    sys.exit(main())
