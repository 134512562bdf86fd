import sys, ctypes as C, numpy as np, torch
sys.path[:0] = ['.', 'tests']
import workloads, paper_2211_06320_b200 as fpe
from paper_2211_06320_b200 import _lib
L = _lib.lib()
f = L.fpe_debug_mma_stats
f.argtypes = [C.c_void_p, C.c_int]
for cfg, n in ((1, 1 << 16), (3, 1 << 24), (5, 1 << 24)):
    a = workloads.coefficients(cfg)
    poly = fpe.precondition(a)
    t = torch.from_numpy(workloads.points(cfg, n)).cuda()
    out = np.zeros(4, np.uint64)
    f(out.ctypes.data, 1)
    poly.evaluate(t); torch.cuda.synchronize()
    f(out.ctypes.data, 1)
    print(cfg, "pieces", out[0], "window coef", out[2], "mma coef", out[3], "frac", out[3] / max(out[2], 1))
