"""N3: the paper's sec:exp-comb-repeat and sec:hybrid-rand studies,
re-run on the synthetic stand-ins with this library (not product code).

  python scripts/study_n3.py [--quick] [--out profiles/r01_n3_study.json]

1. Random vs hybrid: the Uber-shaped C2 tensor, rank 10, factors
   of modes 2-4 fixed to an exact CP-ALS solution (cparls_run_als from the seeded
   random init), the mode-1 least-squares problem.  For s = 2^7 ... 2^19 and
   tau = 1 (random) vs 1/s (hybrid), 10 seeds each: the relative residual
   difference |r(B~) - r(B*)| / max(1, r(B*)) with r(B) = ||Z B' - X'||_F^2
   evaluated without densification, r(B) = ||X||^2 - 2 <B, MTTKRP> + tr(B^T B V),
   B* the exact solution (host fp64 MTTKRP and V^+), B~ the sketched solve of
   the GPU; plus s_det, p_det and s_bar.
2. Combining repeated rows: the Amazon-shaped C4 tensor, rank 10,
   a CP-ALS solution (10 iterations of cparls_run_als), modes 1-3, s = 2^17,
   random and hybrid, 10 seeds: rows of the sketch and nonzeros of the sampled
   right-hand side with repeats combined (s_bar, m_k) and without (s, the sum of
   count x fiber length), and the GPU time of the sketched mode update.
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2006_16438_b200 import Cparls


def mttkrp_host(coords, vals, factors, k):
    """M = X_(k) (KRP of the other factors), fp64 on the host (C2 is small)."""
    D = coords.shape[1]
    z = np.ones((len(vals), factors[0].shape[1]))
    for m in range(D):
        if m != k:
            z *= factors[m][coords[:, m]]
    M = np.zeros((factors[k].shape[0], factors[k].shape[1]))
    np.add.at(M, coords[:, k], vals[:, None] * z)
    return M


def residual(B, Mk, V, normX2):
    return normX2 - 2.0 * float((B * Mk).sum()) + float(np.trace(B.T @ B @ V))


def random_vs_hybrid(quick):
    T = synth.make("C2", device="cuda")
    coords, vals = T.coords.cpu().numpy().astype(np.int64), T.vals.cpu().numpy().astype(np.float64)
    r, k = 10, 0
    g = Cparls(T.dims, T.coords, T.vals, r)
    g.run_als(30 if not quick else 5, fit_every=0)
    A = [g.get_factor(m)[0] for m in range(4)]
    lam = g.get_factor(0)[1]
    A[3] = A[3] * lam          # the model with unit lambda (the fixed factors of the LS problem)
    V = np.ones((r, r))
    for m in range(4):
        if m != k:
            V *= A[m].T @ A[m]
    Mk = mttkrp_host(coords, vals, A, k)
    w, Q = np.linalg.eigh(V)
    keep = w > r * np.finfo(float).eps * w.max()
    Bstar = Mk @ ((Q[:, keep] / w[keep]) @ Q[:, keep].T)
    normX2 = float((vals ** 2).sum())
    rstar = residual(Bstar, Mk, V, normX2)
    rows = []
    exps = range(7, 20) if not quick else (7, 12, 17)
    for e in exps:
        s = 1 << e
        for name, tau in (("random", 1.0), ("hybrid", -1.0)):
            g.set_tau(tau)
            diffs, sdet, pdet, sbar = [], [], [], []
            for seed in range(10 if not quick else 3):
                for m in range(4):
                    g.set_factor(m, A[m])
                info = g.sample(k, s, 1000 + seed, 0)
                g.solve_mode(k)
                _, Bt = g.last_solve(k)
                diffs.append(abs(residual(Bt, Mk, V, normX2) - rstar) / max(1.0, rstar))
                sdet.append(info.s_det); pdet.append(info.p_det); sbar.append(info.s_bar)
            rows.append({"s": s, "scheme": name, "rel_resid_diff_mean": float(np.mean(diffs)),
                         "rel_resid_diff_median": float(np.median(diffs)), "s_det": float(np.mean(sdet)),
                         "p_det": float(np.mean(pdet)), "s_bar": float(np.mean(sbar))})
            print(json.dumps(rows[-1]), flush=True)
    g.close()
    return {"tensor": "C2 (Uber-shaped 183 x 24 x 1140 x 1717, 3.3M nnz)", "rank": r, "mode": k,
            "residual_exact": rstar, "rows": rows}


def combine_repeats(quick):
    cfg = synth.CONFIGS["C4"]
    T = synth.make(cfg, device="cuda", index_dtype=torch.int32)
    coords, vals = T.coords, T.vals
    del T
    torch.cuda.empty_cache()
    r, s = 10, 1 << 17
    g = Cparls(cfg.dims, coords, vals, r)
    del coords, vals
    torch.cuda.empty_cache()
    g.run_als(10 if not quick else 2, fit_every=0)
    A = [g.get_factor(m)[0] for m in range(3)]
    lam = g.get_factor(0)[1]
    A[2] = A[2] * lam
    rows = []
    for k in range(3):
        for name, tau in (("random", 1.0), ("hybrid", -1.0)):
            g.set_tau(tau)
            acc = {"s_bar": [], "mk_combined": [], "mk_uncombined": [], "ms": [], "s_det": [], "p_det": []}
            for seed in range(10 if not quick else 2):
                for m in range(3):
                    g.set_factor(m, A[m])
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                info = g.sample(k, s, 2000 + seed, 0)
                sm = g.get_sample()
                lens = g.get_fiber_lengths()
                si = g.solve_mode(k)
                torch.cuda.synchronize()
                acc["ms"].append((time.perf_counter() - t0) * 1e3)
                acc["s_bar"].append(info.s_bar)
                acc["s_det"].append(info.s_det)
                acc["p_det"].append(info.p_det)
                acc["mk_combined"].append(si.matched_nnz)
                acc["mk_uncombined"].append(int((sm["counts"].astype(np.int64) * lens).sum()))
            row = {"mode": k, "scheme": name, "s": s, **{kk: float(np.mean(v)) for kk, v in acc.items()}}
            rows.append(row)
            print(json.dumps(row), flush=True)
    g.close()
    return {"tensor": "C4 (Amazon-shaped 4.8M x 1.8M x 1.8M, 1.74B nnz)", "rank": r, "rows": rows,
            "note": "uncombined rows = s; uncombined RHS nonzeros = sum over samples of count x fiber length; "
                    "ms = sample + export + solve through the ABI (includes host copies of the sample)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--out", default="profiles/r01_n3_study.json")
    a = ap.parse_args()
    res = {"random_vs_hybrid": random_vs_hybrid(a.quick), "combine_repeats": combine_repeats(a.quick)}
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
