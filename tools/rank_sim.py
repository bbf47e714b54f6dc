import sys, time, torch
sys.path.insert(0, '.')
import paper_2305_08872_b200 as P
from bench import gen_inputs
ctx = P.Context(0)
plan = ctx.plan("discount", "f64")
K, N = 8192, 32768
for ws in (2, 4, 8):
    rows = 32768 // ws
    A, B, th, ds = gen_inputs("discount", "f64", rows, K, N, 0, 0, torch.device("cuda"), False)
    R = torch.zeros((rows, N), dtype=torch.float64, device="cuda")
    ops = P.Operands(A, B, R, th, ds)
    bnd = P.Bounds(0, rows, 0, N, 0, K)
    ctx.clear_tuning_cache()
    rep = P.adaptive_execute(plan, ops, bnd)
    torch.cuda.synchronize()
    v = plan.variants()
    t0 = time.time(); rep2 = P.adaptive_execute(plan, ops, bnd); torch.cuda.synchronize(); el = time.time() - t0
    print(ws, rows, "tuned", rep.tuned, "scratch", rep.scratch_tuned, "frac", round(rep.tuning_fraction, 3),
          "winner", v[rep.best_variant].name, "second call", round(el * 1e3, 1), "ms",
          round(2 * rows * K * N / el / 1e12, 2), "TF", [(v[t.value].name[13:], t.rows, round(t.score * 1e6, 2)) for t in rep.trials])
    del A, B, R, ops
    torch.cuda.empty_cache()
