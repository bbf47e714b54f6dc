"""Small-shape run of the tcgen05 GEMM variants and a generated body, for
compute-sanitizer (scratch tool)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2305_08872_b200 as P
ctx = P.Context(0)
plan = ctx.plan("gemm", "f32")
for vi, v in enumerate(plan.variants()):
    if "tcgen05" not in v.name: continue
    for (M, K, N) in [(64, 64, 64), (200, 96, 264), (129, 40, 300)]:
        A = torch.randint(-8, 9, (M, K), device="cuda").float(); B = torch.randint(-8, 9, (K, N), device="cuda").float()
        R = torch.zeros((M, N), device="cuda")
        P.run_subtask(plan, P.Operands(A, B, R), P.TileParams(variant=vi), P.Bounds(0, M, 0, N, 0, K))
        torch.cuda.synchronize()
        assert torch.equal(R.double(), A.double() @ B.double()), (v.name, M, K, N)
        print(v.name, M, K, N, "ok", flush=True)
