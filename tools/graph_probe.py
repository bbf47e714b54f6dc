"""Scratch: one config-0 step (the tuned winner's launches) enqueued plainly
vs replayed from the library's CUDA graph of it (amlt_gpu_graph_capture). Device time per
step from CUDA events, best and median of 50."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2305_08872_b200 as P  # noqa: E402
from paper_2305_08872_b200.task import compile_task  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg0_discount_f64"
body, dtype, M, K, N = bench.WORKLOADS[wl]
ctx = P.Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream)
plan = ctx.plan_for(compile_task(bench.task_source(body)), dtype)
dev = torch.device("cuda", 0)
B, th, ds = bench.gen_shared(body, dtype, K, N, dev)
A = bench.gen_rows(body, dtype, M, K, 0, dev)
R = torch.zeros((M, N), dtype=A.dtype, device=dev)
ops = P.Operands(A, B, R, th, ds)
bnd = P.Bounds(0, M, 0, N, 0, K)
for _ in range(3):
    rep = P.adaptive_execute(plan, ops, bnd)
win = P.TileParams(variant=rep.best_variant, kc=rep.best_kc if rep.best_kc < K else 0)
print("winner", plan.variants()[rep.best_variant].name, "kc", rep.best_kc)


def timed(fn, n=50):
    ts = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[0], ts[len(ts) // 2]


for _ in range(5):
    P.enqueue(plan, ops, win, bnd)
torch.cuda.synchronize()
print("plain enqueue  best %.4f ms  median %.4f ms" % timed(lambda: P.enqueue(plan, ops, win, bnd)))
g = P.capture_graph(plan, ops, win, bnd)  # amlt_gpu_graph_capture
torch.cuda.synchronize()
print("graph replay   best %.4f ms  median %.4f ms" % timed(g.launch))
