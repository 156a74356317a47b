#!/usr/bin/env python
"""Measurement-only: exact-fit kernel time per streamed copy (cparls_opts.fit_mode)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2006_16438_b200 import Cparls  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1]]
T = synth.make(cfg, device="cuda", index_dtype=torch.int32)
torch.cuda.empty_cache()
for fm in [-1] + list(range(len(cfg.dims))):
    g = Cparls(cfg.dims, T.coords, T.vals, cfg.rank, tau=-1.0, init_seed=cfg.init_seed, fit_mode=fm)
    g.run(2, cfg.s, 3, iter0=0, fit_every=0)
    f0 = g.fit()
    g.reset_stats()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        f = g.fit()
    wall = (time.perf_counter() - t0) / 5
    st = g.stats()
    print(json.dumps({"config": cfg.name, "fit_mode": fm, "fit": f, "wall_ms": wall * 1e3,
                      "k_fit_ms": st["kernel_ms"]["fit"] / max(1, st["kernel_launches_by_id"]["fit"])}), flush=True)
    del g
    torch.cuda.empty_cache()
