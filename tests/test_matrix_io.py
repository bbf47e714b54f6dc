"""Input-side data formats: AMLT matrix files and the seeded generator.

Mirrors the reference's tests/test_engine.cpp:285-365 ("gen_matrix is
order-sensitive but value-deterministic", "matrix files round-trip bit
exactly", "the matrix file header is laid out exactly", "malformed matrix
files are rejected") against the native implementation in libamlt_gpu.so,
and pins it byte for byte against the unmodified reference (oracle/_ref,
driven through oracle/ref_shim.cpp) where that library is present.
"""
from __future__ import annotations

import os
import struct
import sys

import numpy as np
import pytest

from paper_2305_08872_b200 import EngineError
from paper_2305_08872_b200 import matrix_io as io

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle  # noqa: E402

needs_ref = pytest.mark.skipif(not pyoracle.ref_available(), reason="oracle/_ref not built")


def storage(x):
    """Flat storage-order values of a rows x cols view."""
    o = io.storage_order_of(x)
    return np.ascontiguousarray(x if o == io.ROW_MAJOR else np.asarray(x).T).ravel()


def test_gen_matrix_is_order_sensitive_but_value_deterministic():
    rm = io.gen_matrix(7, 9, 11, io.ROW_MAJOR, io.INT_VALUED)
    rm2 = io.gen_matrix(7, 9, 11, io.ROW_MAJOR, io.INT_VALUED)
    assert np.array_equal(rm, rm2)
    assert rm.min() >= -8 and rm.max() <= 8 and np.all(rm == np.round(rm))
    cm = io.gen_matrix(7, 9, 11, io.COL_MAJOR, io.INT_VALUED)
    assert cm.shape == (9, 11) and io.storage_order_of(cm) == io.COL_MAJOR
    assert not np.array_equal(rm, cm)  # order is part of the seed sequence
    real = io.gen_matrix(7, 9, 11, io.ROW_MAJOR, io.REAL)
    assert real.min() >= 0.0 and real.max() < 1.0
    assert np.any(real != np.floor(real))


@needs_ref
@pytest.mark.parametrize("seed,rows,cols,order,mode", [
    (7, 9, 11, 0, 0), (7, 9, 11, 1, 0), (123, 5, 7, 0, 1), (123, 5, 7, 1, 1),
    (1 ^ 0x5A5A, 64, 33, 0, 0), (0xFFFFFFFFFFFFFFFF, 3, 1, 1, 1), (5, 0, 4, 0, 0)])
def test_gen_matrix_matches_reference_bit_for_bit(seed, rows, cols, order, mode):
    mine = storage(io.gen_matrix(seed, rows, cols, order, mode))
    ref = pyoracle.ref_gen_matrix(seed, rows, cols, order, mode)
    assert mine.view(np.uint64).tolist() == ref.view(np.uint64).tolist()


def test_operand_seed_is_seed_xor_fnv1a():
    def fnv1a(s):
        h = 1469598103934665603
        for ch in s.encode():
            h ^= ch
            h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
        return h
    for seed in (0, 1, 42, 2**63 + 5):
        for name in ("A", "B", "thres", "dis", ""):
            assert io.operand_seed(seed, name) == seed ^ fnv1a(name)


@needs_ref
@pytest.mark.parametrize("preset,int_valued,order_a,order_b", [
    ("q1", True, 0, 0), ("q2", False, 1, 0), ("matmul", True, 0, 1)])
def test_gen_operand_matches_reference_task_data(preset, int_valued, order_a, order_b):
    """make_task_data's arrays (src/engine.cpp:128-151) at seed 1, every
    non-result array, both storage orders."""
    t = pyoracle.RefTask.create(pyoracle.preset_source(preset), 13, 5, 17, seed=1,
                                int_valued=int_valued, order_a=order_a, order_b=order_b)
    a_name, b_name, _ = t.roles()
    for name in t.names():
        if name == t.result_name():
            continue
        want = t.get(name)
        order = order_a if name == a_name else order_b if name == b_name else 0
        got = io.gen_operand(1, name, want.shape[0], want.shape[1], order,
                             io.INT_VALUED if int_valued else io.REAL)
        assert np.array_equal(got, want), name
        assert storage(got).view(np.uint64).tolist() == storage(want).view(np.uint64).tolist()


@pytest.mark.parametrize("order", [io.ROW_MAJOR, io.COL_MAJOR])
def test_matrix_files_round_trip_bit_exactly(tmp_path, order):
    path = str(tmp_path / "roundtrip.amlt")
    m = io.gen_matrix(123, 5, 7, order, io.REAL)
    io.write_matrix_file(path, m)
    info = io.matrix_file_info(path)
    assert (info.rows, info.cols, info.order) == (5, 7, order)
    back = io.read_matrix_file(path)
    assert back.shape == (5, 7) and io.storage_order_of(back) == order
    assert np.array_equal(back, m)
    assert storage(back).view(np.uint64).tolist() == storage(m).view(np.uint64).tolist()


def test_matrix_file_header_is_laid_out_exactly(tmp_path):
    path = str(tmp_path / "header.amlt")
    m = np.zeros((2, 3), dtype=np.float64, order="F")  # col-major
    m[0, 0] = 1.0
    m[1, 2] = -2.5
    io.write_matrix_file(path, m)
    b = open(path, "rb").read()
    assert len(b) == 24 + 6 * 8
    assert b[:4] == b"AMLT"
    assert struct.unpack("<II", b[4:12]) == (2, 3)
    assert b[12] == 1 and b[13:24] == bytes(11)
    vals = struct.unpack("<6d", b[24:])
    assert vals[0] == 1.0 and vals[5] == -2.5  # storage order: (0,0) first, (1,2) last


def test_malformed_matrix_files_are_rejected(tmp_path):
    path = str(tmp_path / "bad.amlt")
    open(path, "wb").write(b"NOPE")
    with pytest.raises(EngineError, match="bad magic"):
        io.read_matrix_file(path)
    io.write_matrix_file(path, np.zeros((4, 4)))
    b = open(path, "rb").read()
    open(path, "wb").write(b[:-8])
    with pytest.raises(EngineError, match="truncated"):
        io.read_matrix_file(path)
    bad_order = bytearray(b)
    bad_order[12] = 2
    open(path, "wb").write(bytes(bad_order))
    with pytest.raises(EngineError, match="storage order"):
        io.read_matrix_file(path)
    with pytest.raises(EngineError, match="cannot open"):
        io.read_matrix_file(str(tmp_path / "does_not_exist.amlt"))
    with pytest.raises(EngineError):
        io.read_matrix_file(path, dtype="f16")


@needs_ref
@pytest.mark.parametrize("order", [0, 1])
def test_matrix_files_interchange_with_reference(tmp_path, order):
    """Files written by either side read back identically on the other."""
    rows, cols = 11, 6
    ref_storage = pyoracle.ref_gen_matrix(99, rows, cols, order, 1)
    p_ref = str(tmp_path / "ref.amlt")
    pyoracle.ref_write_matrix_file(p_ref, rows, cols, order, ref_storage)
    mine = io.read_matrix_file(p_ref)
    assert io.storage_order_of(mine) == order
    assert storage(mine).view(np.uint64).tolist() == ref_storage.view(np.uint64).tolist()
    p_mine = str(tmp_path / "mine.amlt")
    io.write_matrix_file(p_mine, mine)
    assert open(p_mine, "rb").read() == open(p_ref, "rb").read()
    r, c, o, vals = pyoracle.ref_read_matrix_file(p_mine)
    assert (r, c, o) == (rows, cols, order)
    assert vals.view(np.uint64).tolist() == ref_storage.view(np.uint64).tolist()


@needs_ref
def test_reference_rejects_what_we_reject(tmp_path):
    path = str(tmp_path / "bad.amlt")
    open(path, "wb").write(b"AMLT" + bytes(20) + bytes(7))  # 0x0 header + junk is fine
    assert pyoracle.ref_read_matrix_file(path)[:3] == (0, 0, 0)
    assert io.read_matrix_file(path).shape == (0, 0)
    open(path, "wb").write(b"AMLT" + struct.pack("<II", 2, 2) + bytes(12) + bytes(24))
    with pytest.raises(RuntimeError, match="truncated"):
        pyoracle.ref_read_matrix_file(path)
    with pytest.raises(EngineError, match="truncated"):
        io.read_matrix_file(path)


@pytest.mark.parametrize("dtype,np_dt", [("f32", np.float32), ("i32", np.int32)])
def test_read_converts_to_kernel_dtype(tmp_path, dtype, np_dt):
    path = str(tmp_path / "m.amlt")
    m = io.gen_matrix(3, 17, 9, io.ROW_MAJOR, io.INT_VALUED)
    io.write_matrix_file(path, m)
    got = io.read_matrix_file(path, dtype=dtype)
    assert got.dtype == np_dt and np.array_equal(got, m.astype(np_dt))
    # and back: f32 / i32 buffers widen to exact f64 values on write
    p2 = str(tmp_path / "m2.amlt")
    io.write_matrix_file(p2, got)
    assert open(p2, "rb").read() == open(path, "rb").read()


def test_write_forced_order_and_strided_input(tmp_path):
    m = io.gen_matrix(4, 6, 5, io.ROW_MAJOR, io.REAL)
    p = str(tmp_path / "f.amlt")
    io.write_matrix_file(p, m, order=io.COL_MAJOR)
    back = io.read_matrix_file(p)
    assert io.storage_order_of(back) == io.COL_MAJOR and np.array_equal(back, m)
    big = io.gen_matrix(4, 12, 10, io.ROW_MAJOR, io.REAL)
    view = big[::2, ::2]  # no unit stride: written row-major
    io.write_matrix_file(p, view)
    back = io.read_matrix_file(p)
    assert io.storage_order_of(back) == io.ROW_MAJOR and np.array_equal(back, view)


@pytest.mark.gpu
@pytest.mark.parametrize("order", [io.ROW_MAJOR, io.COL_MAJOR])
@pytest.mark.parametrize("dtype", ["f64", "f32", "i32"])
def test_read_and_generate_straight_into_device_memory(tmp_path, order, dtype):
    import torch
    m = io.gen_matrix(11, 300, 129, order, io.INT_VALUED)
    p = str(tmp_path / "d.amlt")
    io.write_matrix_file(p, m)
    d = io.read_matrix_file(p, dtype=dtype, device="cuda:0")
    assert d.is_cuda and io.storage_order_of(d) == order
    want = torch.from_numpy(np.ascontiguousarray(m)).to(d.dtype)
    assert torch.equal(d.cpu(), want)
    g = io.gen_matrix(11, 300, 129, order, io.INT_VALUED, dtype=dtype, device="cuda:0")
    assert torch.equal(g.cpu(), want)
    p2 = str(tmp_path / "d2.amlt")
    io.write_matrix_file(p2, g)  # device source
    if dtype != "f64":
        io.write_matrix_file(p, torch.from_numpy(np.ascontiguousarray(m)).to(d.dtype),
                             order=order)
    assert open(p2, "rb").read() == open(p, "rb").read()
