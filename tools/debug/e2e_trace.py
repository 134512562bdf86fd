import sys, time, numpy as np, torch
sys.path[:0] = ['.', 'tests']
import workloads, paper_2211_06320_b200 as fpe
a = workloads.coefficients(3)
poly = fpe.precondition(a)
n = 1 << 26
pts = workloads.points(3, n)
hp = torch.from_numpy(pts).pin_memory(); hv = torch.empty(n, dtype=torch.complex128).pin_memory(); he = torch.empty(n, dtype=torch.int64).pin_memory()
poly.evaluate_host_ptr(hp.data_ptr(), 1, n, hv.data_ptr(), he.data_ptr())
t0 = time.perf_counter(); poly.evaluate_host_ptr(hp.data_ptr(), 1, n, hv.data_ptr(), he.data_ptr()); print("wall %.2f ms" % ((time.perf_counter() - t0) * 1e3), file=sys.stderr)
