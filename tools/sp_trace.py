"""Chunk timeline of k_eval_sparse_coop (needs a build with FPE_EXTRA_FLAGS=-DFPE_ITEM_TRACE):
python tools/sp_trace.py [points]"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path[:0] = ['.']
import paper_2211_06320_b200 as fpe  # noqa: E402
import workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
L = fpe.lib()
L.fpe_debug_sp_trace.argtypes = [C.c_void_p, C.c_int, C.c_int]
L.fpe_debug_sp_trace.restype = C.c_int
poly = fpe.precondition(workloads.coefficients(4))
pts = torch.from_numpy(workloads.points(4, n)).cuda()
poly.evaluate(pts)
torch.cuda.synchronize()
L.fpe_debug_sp_trace(None, 0, 1)
poly.evaluate(pts)
torch.cuda.synchronize()
buf = np.zeros((1 << 20, 3), np.uint64)
m = L.fpe_debug_sp_trace(buf.ctypes.data, 1 << 20, 1)
b = buf[:m].astype(np.int64)
t0 = b[:, 0].min()
s, e = (b[:, 0] - t0) / 1e6, (b[:, 1] - t0) / 1e6
mk, sk = b[:, 2] >> 32, b[:, 2] & 0xffffffff
dur = e - s
print(f"{n} points: {m} chunks over {e.max():.3f} ms; chunk start max {s.max():.3f} ms")
for q in (0.5, 0.9, 0.99, 0.999):
    print(f"  chunk duration p{q*100:g}: {np.quantile(dur, q)*1e3:.1f} us")
for t in (1, 2, 4, 8, 16, 32, 64, 256, 1024):
    sel = mk >= t
    if sel.any():
        print(f"  max K >= {t}: {int(sel.sum())} chunks, mean dur {dur[sel].mean()*1e3:.1f} us")
for i in np.argsort(-dur)[:15]:
    print(f"  chunk start {s[i]:.3f} end {e[i]:.3f} dur {dur[i]*1e3:.1f} us maxK {mk[i]} sumK {sk[i]}")
ends = np.sort(e)
print("  fraction of chunks ended by t:", [(round(float(ends[int(f * (m - 1))]), 3), f) for f in (0.5, 0.9, 0.99, 0.999, 1.0)])
