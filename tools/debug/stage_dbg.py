import sys, numpy as np, torch
sys.path[:0] = ['.', 'tests']
import workloads, paper_2211_06320_b200 as fpe
a = workloads.coefficients(1)
pts = workloads.points(1)[:8]
poly = fpe.precondition(a)
t = torch.from_numpy(pts).cuda()
v, e = poly.evaluate(t)
torch.cuda.synchronize()
ws = poly._ws.cpu().numpy()
n = 8
al = lambda x: (x + 255) & ~255
o_rec = al(n * 8) * 2
rec = ws[o_rec:o_rec + 32 * n].view(np.float64).reshape(n, 4)
o_spos = o_rec + al(32 * n)
spos = ws[o_spos:o_spos + 4 * n].view(np.uint32)
print("spos", spos)
print("staged re,im", rec[:, :2])
print("staged E", rec[:, 2].view(np.int64))
print("vals", v.cpu().numpy(), e.cpu().numpy())
print("as ints", ws[o_rec:o_rec + 32 * n].view(np.int32).reshape(n, 8))
