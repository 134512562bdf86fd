"""e2e (fpe_evaluate_host, pinned host buffers) time of cfg3 for several pipeline settings, each in its own
process (the library reads FPE_HOST_* once):  python tools/e2e_sweep.py 22:18:6 22:21:6:1 ...
(chunk log2 : first-chunk log2 : slots [: split D2H])"""
import os
import subprocess
import sys

CHILD = r'''
import sys, time, torch
sys.path[:0] = ['.']
import workloads, paper_2211_06320_b200 as fpe
poly = fpe.precondition(workloads.coefficients(3))
n = 1 << 26
pts = workloads.points(3, n)
hp = torch.from_numpy(pts).pin_memory(); hv = torch.empty(n, dtype=torch.complex128).pin_memory()
he = torch.empty(n, dtype=torch.int64).pin_memory()
poly.evaluate_host_ptr(hp.data_ptr(), 1, n, hv.data_ptr(), he.data_ptr())
ts = []
for _ in range(5):
    t0 = time.perf_counter(); poly.evaluate_host_ptr(hp.data_ptr(), 1, n, hv.data_ptr(), he.data_ptr())
    ts.append((time.perf_counter() - t0) * 1e3)
print(" ".join(f"{t:.2f}" for t in ts))
'''

for s in sys.argv[1:]:
    c, f, k, sp = (s.split(":") + ["0"])[:4]
    env = dict(os.environ, FPE_HOST_CHUNK_LOG2=c, FPE_HOST_FIRST_LOG2=f, FPE_HOST_SLOTS=k, FPE_HOST_SPLIT_D2H=sp)
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=600)
    print(s, r.stdout.strip() or r.stderr[-500:], flush=True)
