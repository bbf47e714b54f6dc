"""Do the FP64 tensor path (DMMA) and the FP64 CUDA-core path (DFMA) share
hardware on B200? Time a DMMA GEMM and a DFMA-bound discount kernel alone and
on two concurrent streams (scratch experiment)."""
import sys, torch
sys.path.insert(0, '.')
import paper_2305_08872_b200 as P
ctx1, ctx2 = P.Context(0), P.Context(0)
M = K = N = 4096
A = torch.rand((M, K), device="cuda", dtype=torch.float64); B = torch.rand((K, N), device="cuda", dtype=torch.float64)
R1 = torch.zeros((M, N), device="cuda", dtype=torch.float64); R2 = torch.zeros_like(R1)
t = torch.rand(N, device="cuda", dtype=torch.float64); d = torch.rand(N, device="cuda", dtype=torch.float64) * 0.3
g = ctx1.plan("gemm", "f64"); q = ctx2.plan("discount", "f64")
gv = [v.name for v in g.variants()].index("gemm_f64_64x64_dmma_w32x32_c2x2")
qv = [v.name for v in q.variants()].index("discount_f64_32x128_t4x4_w8x1")
b = P.Bounds(0, M, 0, N, 0, K)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
ctx1.set_stream(s1); ctx2.set_stream(s2)
def run(which, reps=3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_event(e0); s2.wait_event(e0)
    for _ in range(reps):
        if "g" in which: P.enqueue(g, P.Operands(A, B, R1), P.TileParams(variant=gv), b)
        if "q" in which: P.enqueue(q, P.Operands(A, B, R2, t, d), P.TileParams(variant=qv), b)
    f1, f2 = torch.cuda.Event(), torch.cuda.Event(); f1.record(s1); f2.record(s2)
    torch.cuda.current_stream().wait_event(f1); torch.cuda.current_stream().wait_event(f2)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
run("gq")
tg, tq, tb = run("g"), run("q"), run("gq")
print(f"DMMA gemm alone {tg:.2f} ms, DFMA discount alone {tq:.2f} ms, both concurrently {tb:.2f} ms "
      f"(sum {tg + tq:.2f}, max {max(tg, tq):.2f})")
