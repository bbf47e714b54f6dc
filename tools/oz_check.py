import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2305_08872_b200 as P
ctx = P.Context(0)
plan = ctx.plan("gemm", "f64")
names = [v.name for v in plan.variants()]
vi = names.index("gemm_f64_128x64_tcgen05_ozaki_i8")
dm = names.index("gemm_f64_64x64_dmma_w32x32_c2x2")
print("variant", vi, flush=True)
rng = np.random.default_rng(5)
for (M, K, N, dist) in [(128, 128, 128, "int"), (300, 200, 264, "int"), (256, 1024, 512, "normal"), (200, 4096, 136, "normal"), (512, 8192, 512, "normal"), (128, 512, 128, "wide")]:
    if dist == "int":
        A = rng.integers(-8, 9, (M, K)).astype(np.float64); B = rng.integers(-8, 9, (K, N)).astype(np.float64)
    elif dist == "normal":
        A = rng.standard_normal((M, K)); B = rng.standard_normal((K, N))
    else:
        A = rng.standard_normal((M, K)) * np.exp(rng.uniform(-20, 20, (M, K))); B = rng.standard_normal((K, N))
    R = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    try:
        P.run_subtask(plan, P.Operands(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), R), P.TileParams(variant=vi), P.Bounds(0, M, 0, N, 0, K))
        torch.cuda.synchronize()
    except Exception as e:
        print("ERR", M, K, N, e, flush=True); break
    got = R.cpu().numpy()
    want = A @ B  # numpy f64 (blocked) — reference for the normwise check
    scale = np.abs(A) @ np.abs(B)
    err = (np.abs(got - want) / np.maximum(scale, 1e-300)).max()
    exact = np.array_equal(got, want) if dist == "int" else None
    print(M, K, N, dist, "normwise", err, "exact" if exact else "", flush=True)
M = K = N = 8192
A = torch.randn((M, K), device="cuda", dtype=torch.float64); B = torch.randn((K, N), device="cuda", dtype=torch.float64)
R = torch.zeros((M, N), device="cuda", dtype=torch.float64)
for v in (vi, dm):
    P.run_subtask(plan, P.Operands(A, B, R), P.TileParams(variant=v), P.Bounds(0, M, 0, N, 0, K))
    best = min(P.run_subtask(plan, P.Operands(A, B, R), P.TileParams(variant=v), P.Bounds(0, M, 0, N, 0, K)) for _ in range(3))
    print(plan.variants()[v].name, "%.2f ms  %.1f TFLOP/s" % (best * 1e3, 2 * M * N * K / best / 1e12), flush=True)
