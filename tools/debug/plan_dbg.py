import sys, numpy as np, torch
sys.path[:0] = ['.', 'tests']
import workloads, paper_2211_06320_b200 as fpe
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = 1 << 22
a = workloads.coefficients(cfg)
pts = workloads.points(cfg, n)
poly = fpe.precondition(a)
poly.set_profiling(True)
t = torch.from_numpy(pts).cuda()
for _ in range(2):
    v, e = poly.evaluate(t)
torch.cuda.synchronize()
print(poly.last_stage_ms())
ws = poly._ws.cpu().numpy()
al = lambda x: (x + 255) & ~255
o = al(n * 8) * 2
rec = ws[o:o + 32 * n].view(np.uint32).reshape(n, 8)
o += al(32 * n) + al(4 * n)
ppc = -(-(-(-n // 148)) // 1024) * 1024
nct = -(-n // ppc)
o += al(nct * 32768 * 4)
gcount = ws[o:o + 4 * 32769].view(np.uint32); o += al(32769 * 4)
bstart = ws[o:o + 4 * 32769].view(np.uint32)
print("n", n, "bstart[16384]", bstart[16384], "long points", gcount[16384:32768].sum(), "short", gcount[:16384].sum())
