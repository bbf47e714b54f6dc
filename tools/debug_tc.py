import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2305_08872_b200 as P
from tests.helpers import make_inputs
ctx = P.Context(0)
plan = ctx.plan("gemm", "f32")
def peek(tag):
    import ctypes
    cudart = ctypes.CDLL("libcudart.so.12") if False else None
    e = torch.cuda.synchronize()
    print(tag, "ok", flush=True)
for vi, v in enumerate(plan.variants()):
    for (M, K, N) in [(64, 64, 64), (96, 128, 160)]:
        if v.name.endswith("_u") is False and (K % 4 or N % 4): continue
        A, B, _, _ = make_inputs("gemm", M, K, N, "int", seed=1)
        R = torch.zeros((M, N), dtype=torch.float32, device="cuda")
        ops = P.Operands(torch.from_numpy(A.astype(np.float32)).cuda(), torch.from_numpy(B.astype(np.float32)).cuda(), R)
        try:
            P.run_subtask(plan, ops, P.TileParams(variant=vi), P.Bounds(0, M, 0, N, 0, K))
            torch.cuda.synchronize()
            print(v.name, M, K, N, "ok", flush=True)
        except Exception as e:
            print(v.name, M, K, N, "ERR", e, flush=True)
plan64 = ctx.plan("gemm", "f64")
A, B, _, _ = make_inputs("gemm", 64, 64, 64, "int", seed=1)
R = torch.zeros((64, 64), dtype=torch.float64, device="cuda")
try:
    P.run_subtask(plan64, P.Operands(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), R), P.TileParams(variant=0), P.Bounds(0, 64, 0, 64, 0, 64))
    print("f64 after ok")
except Exception as e:
    print("f64 after ERR", e)
