"""The C++ host side: the header-only layer over the C-ABI, and the reference
engine driving the backend through integration/amlt_ref_gpu_backend.hpp.

CPU (here): compile + run tests/cpp/test_shim.cpp (dry-run), and the adapter
demo in --dry-run mode (plumbing only).
GPU: the adapter demo for real — the reference's compile_task /
make_task_data produce the task and data, the B200 backend computes, and the
reference's own verify_against_naive checks the result (exact on int data,
rel <= 1e-12 on real data).
"""
from __future__ import annotations

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2305_08872_b200", "lib")
DEMO = os.path.join(ROOT, "oracle", "_ref", "adapter_demo")


def test_cpp_shim_dry_run(tmp_path):
    cxx = shutil.which("g++")
    if not cxx:
        pytest.skip("no g++")
    exe = str(tmp_path / "test_shim")
    subprocess.run([cxx, "-std=c++17", "-O1", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_shim.cpp"), "-L" + LIBDIR,
                    "-lamlt_gpu", "-Wl,-rpath," + LIBDIR, "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "PASS" in r.stdout, r.stdout + r.stderr


@pytest.mark.skipif(not os.path.exists(DEMO), reason="adapter demo not built (needs the reference)")
def test_reference_adapter_dry_run():
    r = subprocess.run([DEMO, "--dry-run"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "PASS" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_reference_adapter_on_gpu():
    assert os.path.exists(DEMO), "oracle/_ref/adapter_demo must be prebuilt and shipped"
    r = subprocess.run([DEMO], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("failures") and "PASS" in r.stdout, \
        r.stdout[-3000:] + r.stderr[-2000:]
