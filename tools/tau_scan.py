import sys, numpy as np, time
sys.path.insert(0,'/root/repo')
from oracle import oracle as o
from paper_2104_03293_b200 import instances as inst, problems as pp
for n in [16, 20]:
    a, xs = inst.exact_cover(n, seed=0)
    h, J, C = pp.ising_from_exact_cover(a)
    r = pp.rescale_r(h, J)
    s, A, B = inst.dw_like_schedule()
    zs = int(sum(int(xs[i]) << i for i in range(n)))
    for p in [32, 64]:
        for tau in [0.02, 0.05, 0.1, 0.2, 0.4]:
            t0=time.time()
            psi = o.aqa_state(h, J, tau*p, p, s, 2*np.pi*A, 2*np.pi*B/r)
            print(n, p, tau, "P=%.3e" % o.success_prob(psi, [zs]), "unif=%.1e" % 2.0**-n, "E=%.3f" % (o.expect_hc(h,J,psi)+C), "%.1fs"%(time.time()-t0), flush=True)
