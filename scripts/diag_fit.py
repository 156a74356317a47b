#!/usr/bin/env python
"""Measurement-only: exact-fit kernel time on C4 at different points of a run
(after create, after warm-up iterations, between timed iterations) and for
every choice of the streamed copy (opts.fit_mode)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2006_16438_b200 import Cparls  # noqa: E402


def fit_ms(g, reps=2):
    out = []
    for _ in range(reps):
        g.reset_stats()
        f = g.fit()
        st = g.stats()
        out.append(st["kernel_ms"]["fit"])
    return out, f


def main():
    cfg = synth.CONFIGS["C4"]
    dev = torch.device("cuda")
    T = synth.make(cfg, device=dev, index_dtype=torch.int32)
    torch.cuda.empty_cache()   # the generator's temporaries (torch's caching allocator)
    res = {}
    for fm in [int(x) for x in (sys.argv[1:] or ["-1"])]:
        g = Cparls(cfg.dims, T.coords, T.vals, cfg.rank, tau=-1.0, init_seed=cfg.init_seed, fit_mode=fm)
        r = {"lib": os.environ.get("CPARLS_LIB", "default")}
        r["after_create"] = fit_ms(g)
        g.run(3, cfg.s, 3, iter0=0, fit_every=0)
        r["after_3_iters"] = fit_ms(g)
        if os.environ.get("DIAG_FIT_LONG"):
            g.run(5, cfg.s, 3, iter0=3, fit_every=0)
            r["after_8_iters"] = fit_ms(g)
            g.reset_stats()
            g.run(5, cfg.s, 3, iter0=8, fit_every=1)
            torch.cuda.synchronize()
            st = g.stats()
            r["inside_run_fit_every_1"] = st["kernel_ms"]["fit"] / max(1, st["kernel_launches_by_id"]["fit"])
            r["rhs_avg"] = st["kernel_ms"]["rhs"] / max(1, st["kernel_launches_by_id"]["rhs"])
        res[fm] = r
        g.close()
        torch.cuda.empty_cache()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
