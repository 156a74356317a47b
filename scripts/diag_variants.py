#!/usr/bin/env python
"""Measurement-only: C4 kernel times for a library build (CPARLS_LIB) --
compile-time tuning variants (e.g. the RHS window size)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2006_16438_b200 import Cparls  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
T = synth.make(cfg, device="cuda", index_dtype=torch.int32)
torch.cuda.empty_cache()
g = Cparls(cfg.dims, T.coords, T.vals, cfg.rank, tau=-1.0, init_seed=cfg.init_seed)
del T
torch.cuda.empty_cache()
g.run(3, cfg.s, 3, iter0=0, fit_every=0)
g.reset_stats()
t0 = time.perf_counter()
g.run(5, cfg.s, 3, iter0=3, fit_every=5)
wall = time.perf_counter() - t0
st = g.stats()
out = {"lib": os.environ.get("CPARLS_LIB", "default"), "wall_ms_per_iter": wall * 200,
       "kernels": {k: st["kernel_ms"][k] / max(1, st["kernel_launches_by_id"][k]) for k in st["kernel_ms"]},
       "create_ms": st["create_ms"]}
print(json.dumps(out))
