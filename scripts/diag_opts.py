#!/usr/bin/env python
"""Measurement-only: per-iteration time and kernel times of one config under
several cparls_opts variants (argv: config, then JSON dicts of Cparls kwargs)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2006_16438_b200 import Cparls  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1]]
variants = [json.loads(a) for a in sys.argv[2:]] or [{}]
T = synth.make(cfg, device="cuda", index_dtype=torch.int32)
torch.cuda.empty_cache()
for kw in variants:
    g = Cparls(cfg.dims, T.coords, T.vals, cfg.rank, tau=-1.0, init_seed=cfg.init_seed, **kw)
    g.run(3, cfg.s, 3, iter0=0, fit_every=0)
    g.reset_stats()
    n = 20
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g.run(n, cfg.s, 3, iter0=3, fit_every=0)
    wall = time.perf_counter() - t0
    st = g.stats()
    print(json.dumps({"config": cfg.name, "opts": kw, "ms_per_iter_nofit": wall * 1000 / n,
                      "kernels": {k: st["kernel_ms"][k] / max(1, st["kernel_launches_by_id"][k])
                                  for k in st["kernel_ms"]},
                      "hot_rows": st["rhs_hot_rows"][:len(cfg.dims)],
                      "hot_share": st["rhs_hot_share"][:len(cfg.dims)]}), flush=True)
    del g
    torch.cuda.empty_cache()
