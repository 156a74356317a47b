import numpy as np, torch, synth
from paper_2006_16438_b200 import Cparls
T = synth.make("C2", device="cuda")
for p in (1, 3):
    g = Cparls(T.dims, T.coords, T.vals, 10, rhs_path=p, init_seed=5)
    A = [g.get_factor(m)[0] for m in range(4)]
    res = []
    for rep in range(3):
        for m in range(4): g.set_factor(m, A[m])
        g.sample(0, 1 << 16, 77, 0)
        s = g.get_sample()
        g.solve_mode(0)
        G, B = g.last_solve(0)
        res.append((s["w2"].copy(), G.copy(), B.copy(), g.get_factor(1)[0].copy(), g.get_ptilde(1).copy()))
    for i in range(5):
        print(p, i, [np.array_equal(res[0][i], res[j][i]) for j in (1, 2)], np.abs(res[0][i] - res[1][i]).max())
