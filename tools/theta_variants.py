"""Scratch: every theta-discount variant at 8192^3 (device-resident, best of
3, uniform data as tools/quick_perf.py). Not the bench contract."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_08872_b200 as P  # noqa: E402

M = K = N = int(os.environ.get("SIZE", "8192"))
if os.environ.get("MKN"):  # e.g. MKN=8192,8192,32768
    M, K, N = (int(x) for x in os.environ["MKN"].split(","))
ctx = P.Context(0)
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.rand((M, K), device="cuda", dtype=torch.float64, generator=g)
B = torch.rand((K, N), device="cuda", dtype=torch.float64, generator=g)
t = torch.rand(N, device="cuda", dtype=torch.float64, generator=g) * 0.5 + 0.25
d = torch.rand(N, device="cuda", dtype=torch.float64, generator=g) * 0.3
R = torch.zeros((M, N), device="cuda", dtype=torch.float64)
plan = ctx.plan("discount", "f64")
ops = P.Operands(A, B, R, t, d)
bnd = P.Bounds(0, M, 0, N, 0, K)
ref = None
for vi, v in enumerate(plan.variants()):
    if "theta" not in v.name and v.name != "discount_f64_32x128_t4x4_w8x1":
        continue
    tp = P.TileParams(variant=vi)
    R.zero_()
    P.run_subtask(plan, ops, tp, bnd)
    out = R.clone()
    if ref is None:
        ref = out
    err = float(((out - ref).abs() / ref.abs().clamp_min(1e-300)).max())
    best = min(P.run_subtask(plan, ops, tp, bnd) for _ in range(3))
    print(f"{v.name:48s} {best * 1e3:8.2f} ms  {2 * M * N * K / best / 1e12:6.2f} TF  rel-vs-first {err:.1e}",
          flush=True)
