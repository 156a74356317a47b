#!/usr/bin/env python
"""Measurement-only: how the matched fiber entries of a C4 mode step spread
over output rows (decides whether aggregating the sampled RHS before its L2
reductions can pay).  For each mode k after W warm-up iterations:
  - m_k, distinct rows, entries per row (mean / max);
  - share of the entries landing in the top-K rows ranked by the step's own
    counts and by the row's nonzero degree (a static relabeling's view);
  - dedup factor of local aggregation: entries / distinct (group, row) pairs
    when groups are F consecutive fibers (device sample order is not exported;
    canonical order = key ascending), for F = 16 ... 4096.
Prints one JSON object."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2006_16438_b200 import Cparls  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
    warm = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    cfg = synth.CONFIGS[name]
    dev = torch.device("cuda")
    T = synth.make(cfg, device=dev, index_dtype=torch.int32)
    degs = []
    for m in range(len(cfg.dims)):
        d = torch.zeros(cfg.dims[m], dtype=torch.int64, device=dev)
        for lo in range(0, T.coords.shape[0], 1 << 27):
            d += torch.bincount(T.coords[lo:lo + (1 << 27), m].long(), minlength=cfg.dims[m])
        degs.append(d)
    torch.cuda.empty_cache()
    g = Cparls(cfg.dims, T.coords, T.vals, cfg.rank, tau=-1.0, init_seed=cfg.init_seed)
    del T
    torch.cuda.empty_cache()
    g.run(warm, cfg.s, cfg.sample_seed, iter0=0, fit_every=0)
    res = {"config": name, "warmup": warm, "modes": []}
    for k in range(len(cfg.dims)):
        info = g.sample(k, cfg.s, cfg.sample_seed, warm * len(cfg.dims) + k)
        lens, out, _ = g.get_fibers()
        out = torch.from_numpy(out).to(dev)
        lens_t = torch.from_numpy(lens).to(dev)
        n = cfg.dims[k]
        cnt = torch.bincount(out, minlength=n)
        mk = int(out.numel())
        srt = torch.sort(cnt, descending=True).values.double().cumsum(0)
        deg_rank = torch.argsort(degs[k], descending=True)
        by_deg = cnt[deg_rank].double().cumsum(0)
        tops = {}
        for K in (64, 256, 1024, 4096, 16384, 65536, 262144):
            if K <= n:
                tops[K] = {"by_count": float(srt[K - 1] / mk), "by_degree": float(by_deg[K - 1] / mk)}
        fid = torch.repeat_interleave(torch.arange(len(lens), device=dev), lens_t)
        dedup = {}
        for F in (16, 64, 256, 1024, 4096):
            key = (fid // F) * n + out
            u = torch.unique(key).numel()
            dedup[F] = mk / u
        # contiguous pieces of E entries in window-major order (RW-row windows,
        # fibers in canonical order or in a random order), the unit a CTA could
        # sort and aggregate in shared memory before its L2 reductions
        RW = (96 << 20) // 256
        win = out // RW
        pieces = {}
        for order in ("canonical", "random"):
            if order == "random":
                perm = torch.randperm(len(lens), device=dev, generator=torch.Generator(device=dev).manual_seed(0))
                fo = perm[fid]
            else:
                fo = fid
            # window-major, then fiber order, then row (fibers are row-sorted)
            okey = (win * len(lens) + fo) * n + out
            pos = torch.argsort(okey)
            o2 = out[pos]
            del okey, pos
            for E in (2048, 4096, 8192, 16384, 65536):
                ck = torch.arange(mk, device=dev) // E
                u = torch.unique(ck * n + o2).numel()
                pieces[f"{order}_E{E}"] = mk / u
                del ck
            del o2
        # fiber length distribution
        lq = torch.quantile(lens_t.double()[:min(len(lens), 1 << 24)], torch.tensor([0.5, 0.9, 0.99, 1.0], device=dev,
                                                                                    dtype=torch.float64))
        res["modes"].append({"k": k, "n_k": n, "s_bar": int(info.s_bar), "s_det": int(info.s_det), "m_k": mk,
                             "distinct_rows": int((cnt > 0).sum()), "max_per_row": int(cnt.max()),
                             "mean_per_touched_row": mk / max(1, int((cnt > 0).sum())),
                             "top_rows_share": tops, "dedup_groups_of_F_fibers": dedup, "dedup_pieces_window_major": pieces,
                             "fiber_len_q50_q90_q99_max": [float(x) for x in lq]})
        del out, cnt, fid
        torch.cuda.empty_cache()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
