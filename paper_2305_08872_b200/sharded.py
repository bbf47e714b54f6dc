"""Multi-GPU partitioner: R row bands across the ranks of one box.

Rows of R are independent: R[i, :] needs A[i, :], all of B and the
per-column vectors. So rank r of n owns rows [M*r/n, M*(r+1)/n) of A and R;
B and the per-j vectors are replicated with one NCCL broadcast each from the
rank that holds them (over NVLink 5 / NVSwitch on a B200 box); there is no
reduction on the data path. An optional gather returns R to one rank for
verification only. One process per GPU, torch.distributed for the plumbing
(backend "nccl" on the GPUs; "gloo" for the CPU tests of this logic).

There is no counterpart in the reference (single-threaded by design,
SPEC.md:8/267); the split is the same row-band split the reference's CPU
baseline uses for its all-cores measurement.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional, Sequence


def row_band(M: int, world_size: int, rank: int, align: int = 1):
    """Half-open row range of `rank`: balanced bands, interior boundaries on
    multiples of `align` (e.g. the CTA tile height) when M allows."""
    if world_size <= 0 or not (0 <= rank < world_size):
        raise ValueError("bad rank / world size")

    def edge(r):
        if r <= 0:
            return 0
        if r >= world_size:
            return M
        e = (M * r) // world_size
        if align > 1:
            e = min(M, (e + align // 2) // align * align)
        return e

    return edge(rank), edge(rank + 1)


def bands(M: int, world_size: int, align: int = 1):
    return [row_band(M, world_size, r, align) for r in range(world_size)]


def broadcast_replicated(tensors: Sequence, src: int = 0, group=None) -> None:
    """Replicates B and the per-column vectors from `src` to every rank, in
    place (one broadcast per tensor; None entries are skipped)."""
    import torch.distributed as dist

    for t in tensors:
        if t is not None:
            dist.broadcast(t, src=src, group=group)


def scatter_rows(full, band_out, M: int, src: int = 0, group=None, align: int = 1) -> None:
    """Sends each rank its A rows from `src` (point-to-point, batched)."""
    import torch.distributed as dist

    ws, rank = dist.get_world_size(group), dist.get_rank(group)
    if rank == src:
        ops = []
        for r, (r0, r1) in enumerate(bands(M, ws, align)):
            if r == src:
                band_out.copy_(full[r0:r1])
            elif r1 > r0:
                ops.append(dist.P2POp(dist.isend, full[r0:r1].contiguous(), r, group))
        for w in dist.batch_isend_irecv(ops) if ops else []:
            w.wait()
    elif band_out.shape[0] > 0:
        dist.recv(band_out, src=src, group=group)


def gather_rows(band, full_out, M: int, dst: int = 0, group=None, align: int = 1) -> None:
    """Collects every rank's R rows on `dst` (verification only)."""
    import torch.distributed as dist

    ws, rank = dist.get_world_size(group), dist.get_rank(group)
    if rank == dst:
        for r, (r0, r1) in enumerate(bands(M, ws, align)):
            if r == dst:
                full_out[r0:r1].copy_(band)
            elif r1 > r0:
                dist.recv(full_out[r0:r1], src=r, group=group)
    elif band.shape[0] > 0:
        dist.send(band.contiguous(), dst=dst, group=group)


@dataclass
class ShardedTask:
    """One rank's share of an MMLT task."""
    rank: int
    world_size: int
    row0: int
    row1: int
    K: int
    N: int


def run_sharded(a_band, b, r_band, thres=None, dis=None, *, plan=None,
                executor: Optional[Callable] = None, K: Optional[int] = None):
    """Runs this rank's band: R_band (+)= body(A_band, B, vectors). The
    default executor is the B200 adaptive executor (adaptive_execute on the
    rank's device); `executor(a, b, r, thres, dis)` may be injected (CPU
    tests). Returns the executor's result (a TuneReport on the GPU path)."""
    if executor is None:
        from . import engine as E

        if plan is None:
            raise ValueError("run_sharded needs a GpuPlan (or an executor)")
        rows, k = a_band.shape[0], (K if K is not None else a_band.shape[1])
        return E.adaptive_execute(plan, E.Operands(a_band, b, r_band, thres, dis),
                                  E.Bounds(0, rows, 0, b.shape[1], 0, k))
    return executor(a_band, b, r_band, thres, dis)
