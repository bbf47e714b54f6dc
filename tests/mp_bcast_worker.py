"""Worker of tests/test_gpu_host_pipeline.py::test_torchrun_broadcast_entry
(launched by torch.distributed.run, one process per GPU).

Each rank attaches an NCCL communicator to its context; rank 0 alone passes
B / thres / dis from host memory, the other ranks their shapes
(engine.Shape), and every rank its own A / R rows. run_host_adaptive then
broadcasts the shared operands panel by panel inside the pipeline. The first
and last row of every band are checked against the oracle; rank 0 writes
the mismatch count to argv[1].
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(out_path: str) -> int:
    import numpy as np
    import torch
    import torch.distributed as dist

    rank = int(os.environ["RANK"])
    ws = int(os.environ["WORLD_SIZE"])
    lrank = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(lrank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lrank))
    os.environ["AMLT_HOST_PANEL_BYTES"] = "65536"

    import paper_2305_08872_b200 as P
    from paper_2305_08872_b200.sharded import row_band
    from tests.helpers import make_inputs, oracle

    M, K, N = 256 * ws + 70, 700, 300
    A, B, t, d = make_inputs("discount", M, K, N, "int", seed=79)
    ctx = P.Context(lrank)

    def exchange(uid):
        box = [uid]
        dist.broadcast_object_list(box, src=0)
        return box[0]

    ctx.attach_comm(rank, ws, exchange=exchange)
    assert ctx.comm_size == ws
    r0, r1 = row_band(M, ws, rank, align=64)
    plan = ctx.plan("discount", "f64")
    Bh = B if rank == 0 else P.Shape(K, N)
    th = t if rank == 0 else P.Shape(N)
    dh = d if rank == 0 else P.Shape(N)
    Ab = np.ascontiguousarray(A[r0:r1])
    bad = 0
    for _ in range(2):  # the first run tunes, the second reuses the winner
        R = np.zeros((r1 - r0, N))
        P.run_host_adaptive(plan, P.Operands(Ab, Bh, R, th, dh), P.Bounds(0, r1 - r0, 0, N, 0, K),
                            r_zero=True, bcast=True)
        if r1 > r0:
            rows = sorted({0, r1 - r0 - 1})
            want = oracle("discount", Ab[rows], B, t, d)
            bad += int((R[rows] != want).any(axis=1).sum())
    tot = torch.tensor([bad], device="cuda")
    dist.all_reduce(tot)
    if rank == 0:
        np.savez(out_path, bad=int(tot.item()))
    dist.barrier()
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1]))
