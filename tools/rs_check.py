import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
torch.cuda.set_device(0)
from paper_2104_03293_b200 import instances as inst, qsim as Q
n = 30
h, J = inst.random_ising(n, 1)
g = np.array([0.3, 0.5, 0.7]); b = np.array([-0.9, -0.6, -0.3])
with Q.QSim(n) as s:
    s.set_ising(h, J); s.init_plus(); s.apply_qaoa(g, b)
    a = s.amplitudes(0, 1 << 20); e = s.expect_hc()
np.save("/tmp/rs_%s.npy" % os.environ.get("QSIM_RUNSPLIT", "0"), a)
print("RUNSPLIT", os.environ.get("QSIM_RUNSPLIT"), "E", repr(e))
