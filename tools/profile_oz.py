import sys, torch
sys.path.insert(0, '.')
import paper_2305_08872_b200 as P
ctx = P.Context(0)
plan = ctx.plan("gemm", "f64")
vi = [v.name for v in plan.variants()].index("gemm_f64_128x64_tcgen05_ozaki_i8")
M = K = N = 8192
A = torch.randn((M, K), device="cuda", dtype=torch.float64); B = torch.randn((K, N), device="cuda", dtype=torch.float64)
R = torch.zeros((M, N), device="cuda", dtype=torch.float64)
el = P.run_subtask(plan, P.Operands(A, B, R), P.TileParams(variant=vi), P.Bounds(0, M, 0, N, 0, K))
print("%.2f ms" % (el * 1e3))
