import sys, numpy as np, torch
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import oracle, workloads, paper_2211_06320_b200 as fpe
from parity import gpu_eval, abs_sum_log2, rel_err_vs
a=workloads.coefficients(1); pts=workloads.points(1)
poly=fpe.precondition(a); P=oracle.OraclePoly(a)
out=gpu_eval(poly, pts)
c=P.classify(pts); Q=P.fpe_eval(pts,c); l2S=abs_sum_log2(a,pts)
err=rel_err_vs(Q,out['v'],out['e'],l2S)
bad=np.flatnonzero(~(err<=2**-45))
print("nbad",len(bad), "of", len(pts))
for i in bad[:12]:
    print(i, pts[i], abs(pts[i]), c['l'][i], c['r'][i], 'gpu', out['v'][i], out['e'][i], 'ref', Q.hi[i], Q.e[i], 'err', err[i])
# monomials
for n in [1,2,3,5,7,8,9,100,1001,1023]:
    m=np.zeros(n+1,complex); m[n]=1.0
    pm=fpe.precondition(m)
    z=np.array([8.021386289160132-0.06490685074726375j, 0.5+0.25j, 1.5j, -3.0+0j])
    o=gpu_eval(pm,z,diag=False)
    Pm=oracle.OraclePoly(m); Qm=Pm.fpe_eval(z)
    print(n, o['v'], o['e'], Qm.hi, Qm.e)
