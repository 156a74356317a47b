import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth
from paper_2006_16438_b200 import Cparls
T = synth.make("C1"); cfg = T.cfg
a = Cparls(T.dims, T.coords.cuda(), T.vals.cuda(), cfg.rank, tau=1e-6)
a.reset_stats()
ta = a.run(1, cfg.s, 9, iter0=0, fit_every=1)
st = a.stats()
print("trace", ta, "syncs", st["host_syncs"], "steps", st["mode_steps"], "fits", st["fits"])
print("fit after", a.fit())
b = Cparls(T.dims, T.coords.cuda(), T.vals.cuda(), cfg.rank, tau=1e-6)
for k in range(3):
    info = b.sample(k, cfg.s, 9, k); b.solve_mode(k)
print("b fit", b.fit())
for m in range(3):
    print(m, np.abs(a.get_factor(m)[0] - b.get_factor(m)[0]).max())
c = Cparls(T.dims, T.coords.cuda(), T.vals.cuda(), cfg.rank)
tc = c.run(2, cfg.s, 9, iter0=0, fit_every=1)
print("no-abort run trace", tc, c.stats()["host_syncs"])
