"""Diagnostics (not product): shape of the sampled-fiber workload on a config.

For each mode step after a few warm iterations: s_bar, s_det, matched entries,
fiber-length quantiles, share of entries in long fibers, entries per touched
output row and the share held by the top rows.  Used to design the RHS kernel.
"""
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2006_16438_b200 import Cparls

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = synth.CONFIGS[cfgname]
dev = torch.device("cuda", 0)
T = synth.make(cfg, device=dev, index_dtype=torch.int32)
coords, vals = T.coords, T.vals
del T
torch.cuda.empty_cache()
g = Cparls(cfg.dims, coords, vals, cfg.rank, tau=-1.0, init_seed=cfg.init_seed)
del coords, vals
torch.cuda.empty_cache()
g.run(3, cfg.s, cfg.sample_seed, iter0=0, fit_every=0)
res = []
for k in range(len(cfg.dims)):
    info = g.sample(k, cfg.s, cfg.sample_seed, 3 * len(cfg.dims) + k)
    smp = g.get_sample()
    lens, out, val = g.get_fibers()
    mk = int(lens.sum())
    ls = np.sort(lens)[::-1]
    cs = np.cumsum(ls)
    d = {"mode": k, "n": int(cfg.dims[k]), "s_bar": int(len(lens)), "s_det": int(smp["is_det"].sum()),
         "mk": mk, "len_q": {q: int(np.quantile(lens, q)) for q in (0.5, 0.9, 0.99, 0.999, 1.0)},
         "nonempty": int((lens > 0).sum())}
    for L in (256, 1024, 4096, 16384, 65536):
        d[f"share_len_ge_{L}"] = float(lens[lens >= L].sum() / max(mk, 1))
        d[f"nfib_len_ge_{L}"] = int((lens >= L).sum())
    cnt = np.bincount(out, minlength=cfg.dims[k])
    tr = np.sort(cnt[cnt > 0])[::-1]
    d["touched_rows"] = int(len(tr))
    d["entries_per_row_q"] = {q: int(np.quantile(tr, q)) for q in (0.5, 0.9, 0.99, 1.0)}
    for top in (64, 1024, 16384, 131072):
        d[f"top{top}_rows_share"] = float(tr[:top].sum() / max(mk, 1))
    res.append(d)
    g.solve_mode(k)
    print(json.dumps(d), flush=True)
