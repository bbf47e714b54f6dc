import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2305_08872_b200 as P
from tests.helpers import oracle, check, make_inputs
ctx = P.Context(0)
plan = ctx.plan("gemm", "f32")
names = [v.name for v in plan.variants()]
vi = names.index("gemm_f32_128x256_tcgen05_3xtf32")
vj = names.index("gemm_f32_128x128_tcgen05_3xtf32_acc4")
print("variant", vi, flush=True)
import time
cases = [(128, 32, 256, "int"), (256, 96, 512, "int"), (300, 200, 260, "int"), (512, 1024, 768, "baseline"),
         (256, 4096, 512, "baseline"), (256, 8192, 512, "baseline"), (256, 16384, 512, "baseline")]
for (M, K, N, dist) in cases:
    A, B, _, _ = make_inputs("gemm", M, K, N, dist, seed=3)
    A32, B32 = A.astype(np.float32), B.astype(np.float32)
    R = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    ops = P.Operands(torch.from_numpy(A32).cuda(), torch.from_numpy(B32).cuda(), R)
    try:
        P.run_subtask(plan, ops, P.TileParams(variant=vi), P.Bounds(0, M, 0, N, 0, K))
        torch.cuda.synchronize()
        got = R.cpu().numpy().astype(np.float64)
        R3 = torch.zeros((M, N), dtype=torch.float32, device="cuda")
        P.run_subtask(plan, P.Operands(ops.a, ops.b, R3), P.TileParams(variant=vj), P.Bounds(0, M, 0, N, 0, K))
        got3 = R3.cpu().numpy().astype(np.float64)
        want = A32.astype(np.float64) @ B32.astype(np.float64)
        # FFMA kernel for comparison
        R2 = torch.zeros((M, N), dtype=torch.float32, device="cuda")
        P.run_subtask(plan, P.Operands(ops.a, ops.b, R2), P.TileParams(variant=1), P.Bounds(0, M, 0, N, 0, K))
        e2 = np.abs(R2.cpu().numpy().astype(np.float64) - want).max()
        err = np.abs(got - want).max()
        scale = (np.abs(A32.astype(np.float64)) @ np.abs(B32.astype(np.float64))).max()
        e3 = np.abs(got3 - want).max()
        print(M, K, N, dist, "wide", err / scale, "acc4", e3 / scale, "ffma", e2 / scale, flush=True)
    except Exception as e:
        print("ERR", M, K, N, e, flush=True)
        break

# speed at cfg2
M = K = N = 8192
A = torch.randn((M, K), device="cuda", dtype=torch.float32); B = torch.randn((K, N), device="cuda", dtype=torch.float32)
R = torch.zeros((M, N), device="cuda", dtype=torch.float32)
ops = P.Operands(A, B, R)
for v in (vi, vj, 1):
    P.run_subtask(plan, ops, P.TileParams(variant=v), P.Bounds(0, M, 0, N, 0, K))
    best = min(P.run_subtask(plan, ops, P.TileParams(variant=v), P.Bounds(0, M, 0, N, 0, K)) for _ in range(3))
    print(plan.variants()[v].name, "%.2f ms  %.1f TFLOP/s" % (best * 1e3, 2 * M * N * K / best / 1e12), flush=True)
