"""Whole-call times (B preparation included) of the tuner's pick against the
best ordinary and theta tiles, for tasks where the B preparation matters
(few rows, large K x N)."""
import sys, time, torch
sys.path.insert(0, '.')
import paper_2305_08872_b200 as P
from bench import gen_inputs
ctx = P.Context(0)
plan = ctx.plan("discount", "f64")
v = plan.variants()
for M, K, N in [(64, 8192, 32768), (256, 8192, 32768), (1024, 4096, 8192), (2048, 8192, 8192)]:
    A, B, th, ds = gen_inputs("discount", "f64", M, K, N, 0, 0, torch.device("cuda"), False)
    R = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    ops = P.Operands(A, B, R, th, ds)
    bnd = P.Bounds(0, M, 0, N, 0, K)
    ctx.clear_tuning_cache()
    rep = P.adaptive_execute(plan, ops, bnd)
    def call(tp=None):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        if tp is None: P.adaptive_execute(plan, ops, bnd)
        else: P.run_subtask(plan, ops, tp, bnd)
        torch.cuda.synchronize(); return (time.perf_counter() - t0) * 1e3
    pick = min(call() for _ in range(3))
    res = {}
    for vi, x in enumerate(v):
        if x.name.endswith("_u") or "_ti" in x.name: continue
        res[x.name] = min(call(P.TileParams(variant=vi)) for _ in range(2))
    best_o = min((t, n) for n, t in res.items() if "_theta_" not in n)
    best_t = min((t, n) for n, t in res.items() if "_theta_" in n)
    print(M, K, N, "pick", v[rep.best_variant].name, "kc", rep.best_kc, round(pick, 3), "ms | best ordinary",
          best_o[1], round(best_o[0], 3), "| best theta", best_t[1], round(best_t[0], 3), flush=True)
    del A, B, R, ops
    torch.cuda.empty_cache()
