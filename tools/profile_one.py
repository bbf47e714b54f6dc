"""Runs one MMLT configuration a few times through the C-ABI (for ncu).

    python tools/profile_one.py <body> <dtype> M K N [variant] [reps]

Device-resident BASELINE-distribution inputs; prints per-launch ms.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2305_08872_b200 as P  # noqa: E402
from bench import gen_rows, gen_shared  # noqa: E402

body, dtype = sys.argv[1], sys.argv[2]
M, K, N = (int(x) for x in sys.argv[3:6])
variant = sys.argv[6] if len(sys.argv) > 6 else "-1"  # index or name
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 2
kc = int(sys.argv[8]) if len(sys.argv) > 8 else 0
dev = torch.device("cuda", 0)
ctx = P.Context(0)
plan = ctx.plan(body, dtype)
B, th, ds = gen_shared(body, dtype, K, N, dev)
A = gen_rows(body, dtype, M, K, 0, dev)
R = torch.zeros((M, N), dtype=A.dtype, device=dev)
ops = P.Operands(A, B, R, th, ds)
vs = plan.variants()
if not variant.lstrip("-").isdigit():
    variant = [v.name for v in vs].index(variant)
elif int(variant) < 0:
    variant = plan.default_variant(M, N, K)
variant = int(variant)
print("variant", vs[variant].name, flush=True)
for _ in range(reps):
    el = P.run_subtask(plan, ops, P.TileParams(kc=kc, variant=variant), P.Bounds(0, M, 0, N, 0, K))
    print(f"{el * 1e3:.3f} ms  {2 * M * N * K / el / 1e12:.3f} TFLOP/s", flush=True)
