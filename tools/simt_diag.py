"""Diagnostic: f32 SIMT GEMM tiles at larger shapes vs an fp64 torch reference
(where wrong, how wrong, and is it repeatable)."""
import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2305_08872_b200 as P
ctx = P.Context(0)
plan = ctx.plan("gemm", "f32")
names = [v.name for v in plan.variants()]
M = K = N = 8192
g = torch.Generator(device="cuda").manual_seed(21)
A = torch.randn((M, K), device="cuda", dtype=torch.float32, generator=g)
B = torch.randn((K, N), device="cuda", dtype=torch.float32, generator=g)
ref = (A.double() @ B.double())
scale = (A.double().abs() @ B.double().abs())
for vn in ["gemm_f32_32x128_t4x4_w8x1", "gemm_f32_32x256_t8x8_w4x1", "gemm_f32_64x128_t8x4_w8x1"]:
    vi = names.index(vn)
    outs = []
    for rep in range(3):
        R = torch.zeros((M, N), device="cuda", dtype=torch.float32)
        P.run_subtask(plan, P.Operands(A, B, R, None, None), P.TileParams(variant=vi), P.Bounds(0, M, 0, N, 0, K))
        rel = (R.double() - ref).abs() / scale
        badm = rel > 1e-5
        nb = int(badm.sum().item())
        outs.append(R.clone())
        if nb:
            idx = badm.nonzero()
            rows = torch.unique(idx[:, 0]); cols = torch.unique(idx[:, 1])
            print(vn, rep, "bad", nb, "rows", rows[:8].tolist(), len(rows), "cols", cols[:8].tolist(), len(cols),
                  "R00", R[0, 0].item(), "ref00", ref[0, 0].item(), "ratio", (R[0,0].double()/ref[0,0]).item(), flush=True)
        else:
            print(vn, rep, "ok", flush=True)
    print(vn, "repeatable", all(torch.equal(outs[0], o) for o in outs[1:]), flush=True)
