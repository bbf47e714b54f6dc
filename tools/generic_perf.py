"""Scratch timing of generated bodies vs the fixed bodies on one B200
(device-resident inputs, CUDA events, best of 3). Not the bench contract."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_08872_b200 as P

HEAD = "where(i in [0..M] and j in [0..N] and k in [0..K]) {\n  R[i][j] += "
STMTS = [
    ("q1 (fixed body)", "A[i][k]*B[k][j] - (A[i][k]*B[k][j] > thres[j])*A[i][k]*B[k][j]*dis[j]"),
    ("q1 with < (generated)", "A[i][k]*B[k][j] - (A[i][k]*B[k][j] < thres[j])*A[i][k]*B[k][j]*dis[j]"),
    ("A*B + u[i]*v[j]", "A[i][k]*B[k][j] + u[i]*v[j]"),
    ("A*B*s + u[i] - v[j]*W[i][j]", "A[i][k]*B[k][j]*s + u[i] - v[j]*W[i][j]"),
    ("(A+1)*(B-1)/2 + (A > v[j])", "(A[i][k] + 1)*(B[k][j] - 1)/2 + (A[i][k] > v[j])"),
]
M = K = N = int(os.environ.get("SIZE", "4096"))
ctx = P.Context(0)
g = torch.Generator(device="cuda").manual_seed(1)
for name, rhs in STMTS:
    src = HEAD + rhs + ";\n}\n"
    t = P.compile_task(src)
    t0 = time.time()
    plan = ctx.plan_for(t, "f64")
    plan_s = time.time() - t0
    shapes = {"A": (M, K), "B": (K, N), "R": (M, N), "thres": (N,), "dis": (N,), "u": (M,),
              "v": (N,), "s": (1, 1), "W": (M, N)}
    data = {n: torch.rand(shapes[n], device="cuda", dtype=torch.float64, generator=g)
            for n in [t.a_name, t.b_name, t.result_name] + list(t.aux_names)
            + [x for x in (t.thres_name, t.dis_name) if x]}
    ops = P.operands_of(t, data)
    b = P.Bounds(0, M, 0, N, 0, K)
    rep = P.adaptive_execute(plan, ops, b)
    best = 1e9
    for _ in range(3):
        best = min(best, P.run_subtask(plan, ops, P.TileParams(variant=rep.best_variant, kc=rep.best_kc), b))
    print(json.dumps({"stmt": name, "body": t.body_name, "plan_s": round(plan_s, 2),
                      "variant": plan.variants()[rep.best_variant].name, "ms": round(best * 1e3, 2),
                      "gflops_mm": round(2 * M * N * K / best / 1e9)}), flush=True)
