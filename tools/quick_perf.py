"""Scratch timing of every tile variant on the BASELINE shapes (device-resident
inputs, CUDA events, best of a few reps). Not the bench contract — bench.py is."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_08872_b200 as P

CFGS = [("discount", "f64", 1024, 1024, 1024), ("boost", "f32", 4096, 4096, 4096),
        ("boost", "f64", 4096, 4096, 4096), ("gemm", "f64", 8192, 8192, 8192),
        ("gemm", "f32", 8192, 8192, 8192), ("sqdiff", "f32", 65536, 1024, 256),
        ("eqcount", "i32", 65536, 1024, 256), ("discount", "f64", 8192, 8192, 8192)]
if len(sys.argv) > 1:
    CFGS = [c for c in CFGS if c[0] + c[1] in sys.argv[1:] or c[0] in sys.argv[1:]]
ctx = P.Context(0)
TD = {"f64": torch.float64, "f32": torch.float32, "i32": torch.int32}
res = []
for body, dt, M, K, N in CFGS:
    g = torch.Generator(device="cuda").manual_seed(1)
    if dt == "i32":
        A = torch.randint(0, 16, (M, K), device="cuda", dtype=torch.int32, generator=g)
        B = torch.randint(0, 16, (K, N), device="cuda", dtype=torch.int32, generator=g)
    else:
        A = torch.rand((M, K), device="cuda", dtype=TD[dt], generator=g)
        B = torch.rand((K, N), device="cuda", dtype=TD[dt], generator=g)
    t = torch.rand(N, device="cuda", dtype=TD[dt], generator=g) * 0.5 + 0.25 if dt != "i32" else torch.randint(0, 16, (N,), device="cuda", dtype=torch.int32)
    d = torch.rand(N, device="cuda", dtype=TD[dt], generator=g) * 0.3 if dt != "i32" else None
    R = torch.zeros((M, N), device="cuda", dtype=TD[dt])
    plan = ctx.plan(body, dt)
    ops = P.Operands(A, B, R, t, d)
    bnd = P.Bounds(0, M, 0, N, 0, K)
    for vi, v in enumerate(plan.variants()):
        if v.name.endswith("_u"): continue
        tp = P.TileParams(variant=vi)
        P.run_subtask(plan, ops, tp, bnd)
        best = 1e9
        for _ in range(3):
            best = min(best, P.run_subtask(plan, ops, tp, bnd))
        it = M * N * K / best
        line = dict(body=body, dtype=dt, shape=[M, K, N], variant=v.name, ms=best * 1e3, giter_s=it / 1e9, gflops_mm=2 * it / 1e9)
        print(json.dumps(line), flush=True)
        res.append(line)
    del A, B, R
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/quick_perf.json", "w"), indent=1)
