import sys, time, numpy as np, torch
sys.path[:0] = ['.', 'tests']
import workloads, paper_2211_06320_b200 as fpe
cfg = 3
a = workloads.coefficients(cfg)
poly = fpe.precondition(a)
poly.set_profiling(True)
N = 1 << 26
pts = torch.from_numpy(workloads.points(cfg, N)).cuda()
for lg in (20, 21, 22, 23, 24, 25, 26):
    n = 1 << lg
    t = pts[:n]
    poly.evaluate(t); torch.cuda.synchronize()
    s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
    k = max(1, (1 << 26) // n)
    s0.record()
    for i in range(k):
        poly.evaluate(pts[(i * n) % N:(i * n) % N + n])
    s1.record(); torch.cuda.synchronize()
    ms = s0.elapsed_time(s1) / k
    print(f"n=2^{lg}: {ms:.3f} ms/batch, {ms * (1 << 26) / n:.2f} ms per 2^26 points", {a_: round(b_, 3) for a_, b_ in poly.last_stage_ms()})
