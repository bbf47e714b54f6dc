"""CPU: the multi-GPU partitioner's host logic with world_size 2 over gloo.

Rank 0 holds A, B and the vectors; A rows are scattered, B and the per-column
vectors broadcast, each rank computes its band (the CPU oracle is injected as
the executor — no GPU here), R bands are gathered on rank 0 and must equal
the single-process oracle bit for bit (int-valued data)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from paper_2305_08872_b200.sharded import bands, row_band


def test_row_bands_partition_exactly():
    for M in (1, 7, 64, 1000, 32768):
        for n in (1, 2, 3, 4, 8):
            for align in (1, 16, 64):
                bs = bands(M, n, align)
                assert bs[0][0] == 0 and bs[-1][1] == M
                for (a0, a1), (b0, b1) in zip(bs, bs[1:]):
                    assert a1 == b0 and a0 <= a1
                if M >= 64 * n and align > 1:
                    assert all(b0 % align == 0 for b0, _ in bs)
    assert row_band(32768, 8, 3) == (12288, 16384)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, M, K, N, out_path):
    import torch
    import torch.distributed as dist

    from oracle import pyoracle as po
    from paper_2305_08872_b200.sharded import (broadcast_replicated, gather_rows, row_band,
                                               run_sharded, scatter_rows)

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    rng = np.random.default_rng(5)
    A_full = torch.from_numpy(rng.integers(-8, 9, (M, K)).astype(np.float64))
    if rank == 0:
        B = torch.from_numpy(rng.integers(-8, 9, (K, N)).astype(np.float64))
        thres = torch.from_numpy(rng.integers(-8, 9, N).astype(np.float64))
        dis = torch.from_numpy(rng.integers(-8, 9, N).astype(np.float64))
    else:
        B, thres, dis = torch.zeros((K, N), dtype=torch.float64), torch.zeros(N, dtype=torch.float64), \
            torch.zeros(N, dtype=torch.float64)
    broadcast_replicated([B, thres, dis], src=0)
    r0, r1 = row_band(M, ws, rank, align=16)
    a_band = torch.zeros((r1 - r0, K), dtype=torch.float64)
    scatter_rows(A_full if rank == 0 else None, a_band, M, src=0, align=16)
    r_band = torch.zeros((r1 - r0, N), dtype=torch.float64)

    def cpu_exec(a, b, r, t, d):
        rr = r.numpy()
        po.oracle_run(po.DISCOUNT, a.numpy(), b.numpy(), rr, thres=t.numpy(), dis=d.numpy())

    run_sharded(a_band, B, r_band, thres, dis, executor=cpu_exec)
    R = torch.zeros((M, N), dtype=torch.float64) if rank == 0 else None
    gather_rows(r_band, R, M, dst=0, align=16)
    if rank == 0:
        np.save(out_path, R.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("M", [100, 257])
def test_sharded_discount_gloo_ws2(tmp_path, M):
    import torch.multiprocessing as mp

    from oracle import pyoracle as po

    K, N = 37, 45
    out = str(tmp_path / "R.npy")
    mp.spawn(_worker, args=(2, _free_port(), M, K, N, out), nprocs=2, join=True)
    rng = np.random.default_rng(5)
    A = rng.integers(-8, 9, (M, K)).astype(np.float64)
    B = rng.integers(-8, 9, (K, N)).astype(np.float64)
    thres = rng.integers(-8, 9, N).astype(np.float64)
    dis = rng.integers(-8, 9, N).astype(np.float64)
    want = np.zeros((M, N))
    po.oracle_run(po.DISCOUNT, A, B, want, thres=thres, dis=dis)
    got = np.load(out)
    assert np.array_equal(got, want)
