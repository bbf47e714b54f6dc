import sys, os, time, torch
sys.path.insert(0, "/root/repo")
import paper_2305_08872_b200 as P
from paper_2305_08872_b200.task import compile_task
import bench
M, K, N = 32768, 8192, 32768
ctx = P.Context(0)
plan = ctx.plan_for(compile_task(bench.task_source("discount")), "f64")
dev = torch.device("cuda", 0)
B, th, ds = bench.gen_shared("discount", "f64", K, N, dev)
A = bench.gen_rows("discount", "f64", M, K, 0, dev)
R = torch.zeros((M, N), dtype=torch.float64, device=dev)
rep = P.adaptive_execute(plan, P.Operands(A, B, R, th, ds), P.Bounds(0, M, 0, N, 0, K))
print("winner", plan.variants()[rep.best_variant].name, file=sys.stderr)
hops = P.Operands(A.cpu().pin_memory(), B.cpu().pin_memory(), torch.empty((M, N), dtype=torch.float64).pin_memory(), th.cpu().pin_memory(), ds.cpu().pin_memory())
del A, B, R; torch.cuda.empty_cache()
P.run_host(plan, hops, P.Bounds(0, M, 0, N, 0, K), r_zero=True)
os.environ["AMLT_HOST_TRACE"] = "1"
for _ in range(2):
    el = P.run_host(plan, hops, P.Bounds(0, M, 0, N, 0, K), r_zero=True)
    print("e2e", el, file=sys.stderr)
# copy bandwidths
h = torch.empty(1 << 30, dtype=torch.uint8).pin_memory(); d = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
for name, f in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    f(); torch.cuda.synchronize(); t = time.time(); [f() for _ in range(4)]; torch.cuda.synchronize()
    print(name, 4 / (time.time() - t), "GB/s", file=sys.stderr)
