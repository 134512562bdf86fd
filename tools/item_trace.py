"""Work-item timeline of k_eval_tiled (needs a build with FPE_EXTRA_FLAGS=-DFPE_ITEM_TRACE):
python tools/item_trace.py [points]"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path[:0] = ['.']
import paper_2211_06320_b200 as fpe  # noqa: E402
import workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 21
L = fpe.lib()
L.fpe_debug_item_trace.argtypes = [C.c_void_p, C.c_int, C.c_int]
L.fpe_debug_item_trace.restype = C.c_int
poly = fpe.precondition(workloads.coefficients(3))
pts = torch.from_numpy(workloads.points(3, n)).cuda()
poly.evaluate(pts)
torch.cuda.synchronize()
L.fpe_debug_item_trace(None, 0, 1)
poly.evaluate(pts)
torch.cuda.synchronize()
buf = np.zeros((1 << 20, 3), np.uint64)
m = L.fpe_debug_item_trace(buf.ctypes.data, 1 << 20, 1)
b = buf[:m].astype(np.int64)
t0 = b[:, 0].min()
s, e = (b[:, 0] - t0) / 1e6, (b[:, 1] - t0) / 1e6
kind = (b[:, 2] >> 60) & 3
folded = (b[:, 2] >> 59) & 1
info = b[:, 2] & ((1 << 20) - 1)
grp = (b[:, 2] >> 20) & ((1 << 39) - 1)
span = e.max()
print(f"{n} points: {m} items over {span:.3f} ms; multi pieces {int((kind == 1).sum())}, groups {int((kind == 2).sum())}")
dur = e - s
for q in (0.5, 0.9, 0.99):
    print(f"  item duration p{int(q*100)}: {np.quantile(dur, q):.4f} ms")
order = np.argsort(-dur)[:15]
for i in order:
    print(f"  kind {kind[i]} folded {folded[i]} group {grp[i]} info {info[i]} start {s[i]:.3f} end {e[i]:.3f} dur {dur[i]:.3f}")
m1 = kind == 1
print("multi pieces: median dur folded %.4f / not folded %.4f; max %.4f / %.4f" % (
    np.median(dur[m1 & (folded == 1)]), np.median(dur[m1 & (folded == 0)]), dur[m1 & (folded == 1)].max(), dur[m1 & (folded == 0)].max()))
# busy warps over time
for t in np.linspace(0, span, 21):
    print(f"  t={t:.3f} ms busy items {int(((s <= t) & (e > t)).sum())}")
# occupancy over time: items in flight (one per busy warp); the tail is the time after the first warp idles
ev = np.concatenate([np.stack([s, np.ones_like(s)], 1), np.stack([e, -np.ones_like(e)], 1)])
ev = ev[np.argsort(ev[:, 0], kind="stable")]
busy = np.cumsum(ev[:, 1])
peak = busy.max()
for frac in (0.99, 0.9, 0.5):
    t = ev[np.flatnonzero(busy >= frac * peak)[-1], 0]
    print(f"  last time >= {frac:.0%} of the {int(peak)} busy warps: {t:.3f} ms of {span:.3f} ({100 * (span - t) / span:.1f}% after)")
