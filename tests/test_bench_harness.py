"""CPU (gloo) tests of bench.py's multi-rank harness: `--gpus N` outside
torchrun launches N ranks itself, a --gpus / WORLD_SIZE mismatch is an
error, every rank gets its 64-row band (the same cut as the native group,
csrc/sharded.cu), B and the vectors reach every rank from rank 0, the
reduction is the max over ranks, and stdout carries exactly one JSON line.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=e,
                          capture_output=True, text=True, timeout=300)


@pytest.mark.parametrize("n,workload", [(2, "cfg4_discount_f64"), (3, "cfg0_discount_f64")])
def test_gpus_n_spawns_n_ranks(n, workload):
    r = run_bench("--gpus", str(n), "--dry-run", "--workload", workload)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    out = json.loads(lines[0])
    assert out["dry_run"] and out["value"] is None and out["n_gpus"] == n
    M = out["config"]["M"]
    bands = out["bands"]
    assert bands[0][0] == 0 and bands[-1][1] == M
    for (a0, a1), (b0, b1) in zip(bands, bands[1:]):
        assert a1 == b0 and a1 % 64 == 0
    # the native group's cut (csrc/sharded.cu: (M d / n + 32) / 64 * 64)
    assert [b[0] for b in bands] == [min(M, (M * d // n + 32) // 64 * 64) for d in range(n)]
    assert len(set(out["shared_checksums"])) == 1  # every rank holds rank 0's B / vectors
    assert out["max_over_ranks"] == n


def test_gpus_world_size_mismatch_is_an_error():
    r = run_bench("--gpus", "4", "--dry-run", env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE" in r.stderr


def test_single_rank_dry_run():
    r = run_bench("--dry-run")
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip())
    assert out["n_gpus"] == 1 and out["bands"] == [[0, out["config"]["M"]]]


def test_proxy_band_refuses_multi_rank():
    """--proxy-band times one rank's band on ONE GPU; under torchrun or with
    --gpus > 1 it is refused before any work (bench.py)."""
    r = run_bench("--gpus", "2", "--proxy-band", "8", "--dry-run",
                  env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2 and "proxy-band" in r.stderr
