"""Max |P_gpu - P_ref| / S on long-window points (cfg3 polynomial, |z| within 2^-12 of 1) -- the points
whose pieces go to the tensor cores."""
import sys, numpy as np
sys.path[:0] = ['.', 'tests']
import oracle, workloads, paper_2211_06320_b200 as fpe
from parity import gpu_eval, abs_sum_log2, rel_err_vs
a = workloads.coefficients(3)
P = oracle.OraclePoly(a)
rng = np.random.default_rng(71)
n = 2048
pts = np.exp2(rng.uniform(-2.0 ** -12, 2.0 ** -12, n)) * np.exp(1j * rng.uniform(0, 2 * np.pi, n))
poly = fpe.precondition(a)
out = gpu_eval(poly, pts)
idx = np.arange(0, n, 4)
c = P.classify(pts[idx])
Q = P.fpe_eval(pts[idx], c)
err = rel_err_vs(Q, out["v"][idx], out["e"][idx], abs_sum_log2(a, pts[idx]))
print("K median", np.median(c["K"]), "max err/S = 2^%.2f" % np.log2(err.max()), "median 2^%.2f" % np.log2(np.median(err)))
