"""Scratch check (not product code): repeat AMULET-style tuning of one BASELINE
config in one process and print each run's trial scores and winner, to see how
stable the row-band trials are."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_08872_b200 as P

body, dt, M, K, N = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
TD = {"f64": torch.float64, "f32": torch.float32, "i32": torch.int32}[dt]
ctx = P.Context(0)
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.rand((M, K), device="cuda", dtype=TD, generator=g)
B = torch.rand((K, N), device="cuda", dtype=TD, generator=g)
t = torch.rand(N, device="cuda", dtype=TD, generator=g) * 0.5 + 0.25
R = torch.zeros((M, N), device="cuda", dtype=TD)
plan = ctx.plan(body, dt)
names = [v.name for v in plan.variants()]
for rep in range(int(sys.argv[6]) if len(sys.argv) > 6 else 4):
    ctx.clear_tuning_cache()
    r = P.adaptive_execute(plan, P.Operands(A, B, R, t, None), P.Bounds(0, M, 0, N, 0, K))
    print(json.dumps({"rep": rep, "winner": names[r.best_variant], "total_ms": round(r.total_seconds * 1e3, 3),
                      "trials": [(names[x.value], round(x.score * 1e6, 4)) for x in r.trials]}), flush=True)
    for vi in sorted({x.value for x in r.trials}):
        R.zero_()
        best = min(P.run_subtask(plan, P.Operands(A, B, R, t, None), P.TileParams(variant=vi),
                                 P.Bounds(0, M, 0, N, 0, K)) for _ in range(3))
        print("   whole", names[vi], round(best * 1e3, 3), "ms")
