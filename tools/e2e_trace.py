"""One BASELINE workload through the host entry with AMLT_HOST_TRACE=1: the
copy / compute pipeline's stage times (stderr), the layout it chose, and
pinned H2D / D2H bandwidth.  python tools/e2e_trace.py [workload]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2305_08872_b200 as P  # noqa: E402
from paper_2305_08872_b200.task import compile_task  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg4_discount_f64"
body, dtype, M, K, N = bench.WORKLOADS[wl]
ctx = P.Context(0)
plan = ctx.plan_for(compile_task(bench.task_source(body)), dtype)
dev = torch.device("cuda", 0)
B, th, ds = bench.gen_shared(body, dtype, K, N, dev)
A = bench.gen_rows(body, dtype, M, K, 0, dev)
R = torch.zeros((M, N), dtype=A.dtype, device=dev)
bounds = P.Bounds(0, M, 0, N, 0, K)
rep = P.adaptive_execute(plan, P.Operands(A, B, R, th, ds), bounds)
win = P.TileParams(variant=rep.best_variant, kc=rep.best_kc if rep.best_kc < K else 0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
stream = torch.cuda.current_stream()
ctx.set_stream(stream)
P.enqueue(plan, P.Operands(A, B, R, th, ds), win, bounds)
e0.record(stream)
for _ in range(3):
    P.enqueue(plan, P.Operands(A, B, R, th, ds), win, bounds)
e1.record(stream)
torch.cuda.synchronize()
ctx.set_stream(None)
print(wl, "winner", plan.variants()[rep.best_variant].name, "kc", rep.best_kc,
      f"device-resident step {e0.elapsed_time(e1) / 3:.3f} ms", file=sys.stderr)


def pin(x):
    return x.cpu().pin_memory() if x is not None else None


hops = P.Operands(pin(A), pin(B), torch.empty((M, N), dtype=A.dtype).pin_memory(), pin(th), pin(ds))
del A, B, R
torch.cuda.empty_cache()
P.run_host(plan, hops, bounds, r_zero=True)
for mode in ("zero-copy", "staged"):  # (pinned R: zero-copy unless AMLT_HOST_NO_ZEROCOPY)
    if mode == "staged":
        os.environ["AMLT_HOST_NO_ZEROCOPY"] = "1"
    os.environ["AMLT_HOST_TRACE"] = "1"
    P.run_host(plan, hops, bounds, r_zero=True)
    os.environ.pop("AMLT_HOST_TRACE")
    els = [P.run_host(plan, hops, bounds, r_zero=True) for _ in range(3)]
    print(f"e2e {mode}: best {min(els) * 1e3:.3f} ms of {[round(e * 1e3, 3) for e in els]}",
          ctx.last_host_layout(), file=sys.stderr)
os.environ.pop("AMLT_HOST_NO_ZEROCOPY")
# copy bandwidths
h = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
d = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
for name, f in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    f()
    torch.cuda.synchronize()
    t = time.time()
    for _ in range(4):
        f()
    torch.cuda.synchronize()
    print(name, 4 / (time.time() - t), "GB/s", file=sys.stderr)
