"""The command-line front end (paper_2305_08872_b200/cli.py), mirroring the
reference's tests/test_cli.cpp case by case: report schemas, exit codes,
operand files, --out. CPU cases need no device (explain plans in a dry-run
context; usage / recognition errors fail before any device work); the rest
run on the GPU.
"""
from __future__ import annotations

import json

import numpy as np
import pytest

from paper_2305_08872_b200 import cli
from paper_2305_08872_b200 import matrix_io as io

NOT_MMLT = ("where(i in [0..M] and j in [0..N] and k in [0..K]) {\n"
            "  R[i][j] += A[i][k]*B[k][j]*u[k];\n}\n")  # a k-indexed aux: not an MMLT


def run_cli(capsys, line: str):
    try:
        code = cli.main(line.split())
    except SystemExit as e:
        code = e.code
    out, err = capsys.readouterr()
    return code, out, err


# ---------------------------------------------------------------- CPU cases

def test_explain_prints_the_pipeline_for_a_recognized_task(capsys):
    code, out, _ = run_cli(capsys, "explain --preset q1")
    assert code == 0
    for s in ("MMLT", "mul REG0 A B", "masksub", "11 x 16", "31", "thres", "B200 variants"):
        assert s in out, s


def test_unknown_presets_and_missing_tasks_exit_2(capsys, tmp_path):
    code, _, err = run_cli(capsys, "run --preset nosuch --dims 8 8 8")
    assert code == 2 and "unknown preset" in err
    assert run_cli(capsys, "run --dims 8 8 8")[0] == 2
    assert run_cli(capsys, f"run --task {tmp_path}/no_such_file.task --dims 8 8 8")[0] == 2
    code, _, err = run_cli(capsys, "run --task x.task --preset matmul --dims 8 8 8")
    assert code == 2 and "mutually exclusive" in err


def test_parse_errors_exit_2(capsys, tmp_path):
    p = tmp_path / "bad.task"
    p.write_text("where(i in [0..M] and j in [0..N]) { R[i][j] += ; }\n")
    code, _, err = run_cli(capsys, f"run --task {p} --dims 8 8 8")
    assert code == 2 and "parse error" in err


def test_unrecognized_tasks_exit_3(capsys, tmp_path):
    p = tmp_path / "nm.task"
    p.write_text(NOT_MMLT)
    for cmd in ("run", "tune", "bench", "explain"):
        code, _, err = run_cli(capsys, f"{cmd} --task {p} --dims 12 10 14")
        assert code == 3 and "recognition failed" in err, cmd


def test_fixed_mode_needs_explicit_tile_sizes(capsys):
    code, _, err = run_cli(capsys, "run --preset matmul --dims 32 32 32 --mode fixed")
    assert code == 2 and "usage error" in err


def test_bad_flags_and_missing_subcommands_fail(capsys):
    assert run_cli(capsys, "run --preset matmul --no-such-flag")[0] != 0
    assert run_cli(capsys, "")[0] != 0
    assert run_cli(capsys, "run --preset matmul --dims 8 8")[0] != 0
    assert run_cli(capsys, "run --preset matmul --format yaml")[0] != 0


def test_explain_covers_every_preset(capsys):
    from paper_2305_08872_b200.task import preset_names
    for name in preset_names():
        code, out, _ = run_cli(capsys, f"explain --preset {name} --dims 24 16 24")
        assert code == 0 and "default for 24 x 16 x 24" in out, name


# ---------------------------------------------------------------- GPU cases

@pytest.mark.gpu
def test_run_reports_a_verified_adaptive_execution_as_json(capsys):
    code, out, _ = run_cli(capsys, "run --preset q1 --dims 48 32 40 --verify --format json")
    assert code == 0
    j = json.loads(out)
    assert (j["task"], j["m"], j["k"], j["n"], j["mode"]) == ("q1", 48, 32, 40, "adaptive")
    assert j["verify"] == "exact" and j["elapsed_seconds"] > 0
    assert j["kc"] >= 1 and j["nc"] >= 1 and j["packing"] is False and j["trials"] == 3


@pytest.mark.gpu
def test_run_emits_the_documented_csv_header(capsys):
    code, out, _ = run_cli(capsys, "run --preset matmul --dims 32 32 32 --format csv")
    assert code == 0
    header, row = out.splitlines()[:2]
    assert header == "task,m,k,n,mode,elapsed_seconds,spr,kc,nc,packing,verify"
    assert row.startswith("matmul,32,32,32,ad") and "skipped" in row


@pytest.mark.gpu
def test_run_table_format_names_the_fields(capsys):
    code, out, _ = run_cli(capsys, "run --preset q3-tij-atbt --dims 24 16 24 --verify")
    assert code == 0
    assert "task      q3-tij-atbt" in out and "dims      24 x 16 x 24" in out
    assert "verify    exact" in out


@pytest.mark.gpu
def test_fixed_and_naive_modes(capsys):
    code, out, _ = run_cli(capsys, "run --preset matmul --dims 32 32 32 --mode fixed --kc 16 "
                                   "--nc 16 --verify --trials 1")
    assert code == 0 and "exact" in out
    code, out, _ = run_cli(capsys, "run --preset q2 --dims 20 12 28 --mode naive --verify "
                                   "--format json")
    j = json.loads(out)
    assert code == 0 and j["mode"] == "naive" and j["verify"] == "exact"
    assert j["kc"] is None and j["nc"] is None


@pytest.mark.gpu
@pytest.mark.parametrize("extra", ["--data real", "--data real --dtype f32",
                                   "--dtype i32 --layout-a col", "--layout-b col --dtype f32"])
def test_run_verifies_across_dtypes_and_layouts(capsys, extra):
    preset = "q3-tj" if "i32" in extra else "q2-atb"
    code, out, _ = run_cli(capsys, f"run --preset {preset} --dims 70 33 90 --verify --format json "
                                   f"--trials 1 {extra}")
    j = json.loads(out)
    assert code == 0 and j["verify"] in ("exact", "pass"), out


@pytest.mark.gpu
def test_tune_prints_trials_winners_coverage_and_the_tuning_fraction(capsys):
    code, out, _ = run_cli(capsys, "tune --preset matmul --dims 16 200 256 --seed 5")
    assert code == 0
    j = json.loads(out)
    assert j["task"] == "matmul" and j["tuned"] is True
    assert [t["kc"] for t in j["kc_trials"]] == [200, 100, 50, 25]
    assert all(t["elapsed"] > 0 and t["score"] > 0 for t in j["kc_trials"])
    assert all(t["nc"] % 16 == 0 for t in j["nc_trials"])
    assert j["chosen"]["kc"] in [t["kc"] for t in j["kc_trials"]]
    assert 0.0 < j["tuning_fraction"] <= 1.0 and j["total_seconds"] > 0
    area = sum((c["k1"] - c["k0"]) * (c["j1"] - c["j0"]) for c in j["coverage"])
    assert area == 200 * 256


@pytest.mark.gpu
def test_tune_on_a_small_problem_reports_the_untuned_defaults(capsys):
    code, out, _ = run_cli(capsys, "tune --preset matmul --dims 16 100 32")
    j = json.loads(out)
    assert code == 0 and j["tuned"] is False
    assert j["chosen"] == {"kc": 100, "nc": 32}
    assert j["tuning_fraction"] == 0.0 and j["kc_trials"] == []


@pytest.mark.gpu
def test_tune_with_the_gpu_tuner(capsys):
    code, out, _ = run_cli(capsys, "tune --preset q1 --dims 2048 256 1024 --tuner gpu")
    j = json.loads(out)
    assert code == 0 and j["chosen"]["variant"].startswith("discount_f64")
    area = sum((c["i1"] - c["i0"]) * (c["j1"] - c["j0"]) for c in j["coverage"])
    assert area == 2048 * 1024


@pytest.mark.gpu
def test_bench_emits_the_grid_as_csv_with_an_adaptive_footer(capsys):
    code, out, _ = run_cli(capsys, "bench --preset matmul --dims 24 48 64 --trials 1")
    assert code == 0
    lines = out.splitlines()
    assert lines[0] == "kc\\nc,16,32,64"
    rows = [ln for ln in lines[1:] if not ln.startswith("adaptive,")]
    assert len(rows) == 2 and all(r.count(",") == 3 for r in rows)
    footer = lines[-1]
    assert footer.startswith("adaptive,") and "kc=" in footer and "nc=" in footer


@pytest.mark.gpu
def test_operand_files_override_generated_data(capsys, tmp_path):
    a = np.empty((12, 10), order="F")
    b = np.empty((10, 14))
    for i in range(12):
        for k in range(10):
            a[i, k] = (i * k) % 5 - 2
    for k in range(10):
        for j in range(14):
            b[k, j] = (k + j) % 7 - 3
    pa, pb = str(tmp_path / "a.amlt"), str(tmp_path / "b.amlt")
    io.write_matrix_file(pa, a)
    io.write_matrix_file(pb, b)
    out_path = str(tmp_path / "r.json")
    code, out, _ = run_cli(capsys, f"run --preset matmul --dims 12 10 14 --a-file {pa} "
                                   f"--b-file {pb} --verify --format json --trials 1 "
                                   f"--out {out_path}")
    assert code == 0 and out == ""
    j = json.load(open(out_path))
    assert j["task"] == "matmul" and j["verify"] == "exact"
    code, _, err = run_cli(capsys, f"run --preset matmul --dims 9 9 9 --a-file {pa}")
    assert code == 2 and "9x9" in err


GENERIC = ("where(i in [0..M] and j in [0..N] and k in [0..K]) {\n"
           "  R[i][j] += A[k][i]*B[k][j] + u[i]*v[j] - (A[k][i] > s)*W[i][j]/4;\n}\n")


def test_explain_a_generated_body(capsys, tmp_path):
    p = tmp_path / "g.task"
    p.write_text(GENERIC)
    code, out, _ = run_cli(capsys, f"explain --task {p} --dims 64 32 48")
    assert code == 0
    assert "body: generated" in out and "aux={u [i], v [j], s constant, W [i][j]}" in out
    assert "term: sub_rn(add_rn(mul_rn(a, b), mul_rn(c.v[0], c.v[1]))" in out


@pytest.mark.gpu
@pytest.mark.parametrize("extra", ["", "--mode naive", "--layout-a col --data real",
                                   "--dtype f32"])
def test_run_a_generated_body_verified(capsys, tmp_path, extra):
    p = tmp_path / "g.task"
    p.write_text(GENERIC)
    code, out, err = run_cli(capsys, f"run --task {p} --dims 70 33 90 --verify --format json "
                                     f"--trials 1 {extra}")
    j = json.loads(out)
    assert code == 0, err
    assert j["verify"] in (("exact", "pass") if "real" in extra else ("exact",)), out


@pytest.mark.gpu
@pytest.mark.parametrize("extra", ["--dtype f32", "--f64-emulation"])
def test_run_gemm_on_tensor_cores_verified(capsys, extra):
    """matmul through the CLI where the tuner may choose a tensor-core GEMM
    (tcgen05 3xTF32 for f32; the opt-in int8 Ozaki f64): integer data, exact."""
    code, out, err = run_cli(capsys, f"run --preset matmul --dims 1024 512 768 --verify "
                                     f"--format json --trials 1 {extra}")
    j = json.loads(out)
    assert code == 0, err
    assert j["verify"] == "exact", out
