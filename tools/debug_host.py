import faulthandler, sys, os
faulthandler.enable()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2305_08872_b200 as P
from tests.helpers import make_inputs, oracle
ctx = P.Context(0)
plan = ctx.plan("discount", "f64")
for (M, K, N) in [(513, 300, 257), (4096, 256, 512)]:
    A, B, t, d = make_inputs("discount", M, K, N, "baseline", seed=23)
    R = np.zeros((M, N))
    print("run_host", M, K, N, flush=True)
    try:
        el = P.run_host(plan, P.Operands(A, B, R, t, d), P.Bounds(0, M, 0, N, 0, K))
        want = oracle("discount", A, B, t, d)
        print(" ok", el, np.abs(R - want).max(), flush=True)
    except Exception as e:
        print(" ERR", e, flush=True)
        break
    hA = torch.from_numpy(A).pin_memory(); hB = torch.from_numpy(B).pin_memory()
    ht = torch.from_numpy(t).pin_memory(); hd = torch.from_numpy(d).pin_memory()
    hR = torch.zeros((M, N), dtype=torch.float64).pin_memory()
    el = P.run_host(plan, P.Operands(hA, hB, hR, ht, hd), P.Bounds(0, M, 0, N, 0, K), r_zero=True)
    print(" pinned ok", el, np.abs(hR.numpy() - want).max(), flush=True)
