#!/usr/bin/env python
"""CP-ARLS-LEV outer iterations/s on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

A "step" is one CP-ARLS-LEV outer iteration (all D mode updates: sample ->
KrpSamp/Gram -> fiber lookup -> RHS -> solve/normalize/leverage, Alg. 3
P:917-928) with the exact fit amortized once per epoch of eta = 5 iterations
(P:930): the timed K iterations include a fit after every 5th global
iteration.  Inputs are synthetic Zipf tensors shaped like the paper's
workloads (synth/).  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ETA = 5                       # epoch length
FIT_SAMPLES = 1 << 27         # s_fit of the paper's estimated fit on Amazon
FIT_SEED = 17
METRIC = "CP-ARLS-LEV ALS iterations/sec (r=25, s=2^17) and % of HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--tau", type=float, default=-1.0, help="-1 = 1/s (hybrid, P:999); 1 = random")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-phases", action="store_true", help="per-phase breakdown (stderr)")
    ap.add_argument("--sample-frac", type=float, default=0.001,
                    help="oracle sample: this fraction of the config's nonzeros (a prefix)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rk = int(os.environ.get("RANK", "0"))
    lrk = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rk, lrk


# ---------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1])); mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no nvidia-smi sample"], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "window": "warm-up + timed region"}


KERNEL_NAMES = {"rhs": "k_rhs", "fit": "k_fit_sub", "solve_rows": "k_solve_dmma", "lev_rows": "k_lev_rows_w"}


def kernel_names(r):
    """Timer labels (cparls_stats.kernel_ms ids) -> kernel names; the solve
    runs on FP64 tensor cores (k_solve_dmma) for r in 5..32."""
    names = dict(KERNEL_NAMES)
    if not (4 < r <= 32):
        names["solve_rows"] = "k_solve_rows_t"
    return names


def row_ld(r):
    """Row stride libcparls uses for r columns (cparls_create: r rounded up to 8, r <= 4: 4)."""
    return (r + 3) // 4 * 4 if r <= 4 else (r + 7) // 8 * 8


def rhs_row_stream(g, cfg, seed, window_rows, per_mode=1 << 25):
    """The output rows k_rhs reduces into, taken from the library itself: for
    every mode k a fresh sample (same s and tau as the run), its matched
    fiber entries in the sample's canonical order (cparls_get_fibers), those
    in the first output-row window, first `per_mode` of them."""
    import numpy as np
    import torch
    parts = []
    for k in range(len(cfg.dims)):
        g.sample(k, cfg.s, seed, 1_000_000 + k)
        _, out, _ = g.get_fibers()
        out = out[out < min(window_rows, cfg.dims[k])][:per_mode]
        parts.append(torch.from_numpy(out.astype(np.int32)))
        del out
    return torch.cat(parts).contiguous()


def measure_peaks(cfg, dev, window_rows, fit_rows, row_stream=None):
    """Ceilings of the hot kernels' own access patterns on this GPU, measured
    here (libcparls_peaks.so, not part of the method): r-lane reductions (fp64,
    and int64 for the fixed-point RHS) into random rows of an L2-sized window
    and into the tensor's own row stream (k_rhs), and r-wide fp64 row gathers
    from random rows of a factor-sized matrix (k_fit_sub)."""
    import ctypes as C
    import torch
    lib = C.CDLL(os.path.join(ROOT, "paper_2006_16438_b200", "libcparls_peaks.so"))
    lib.cparls_peak_red_f64.restype = C.c_double
    lib.cparls_peak_red_f64.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int]
    lib.cparls_peak_gather.restype = C.c_double
    lib.cparls_peak_gather.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int64, C.c_int, C.c_int, C.c_void_p]
    r = cfg.rank
    ld = row_ld(r)
    torch.cuda.synchronize()
    M = torch.zeros(window_rows * ld, dtype=torch.float64, device=dev)
    red = lib.cparls_peak_red_f64(M.data_ptr(), window_rows, r, ld, 8192, 148 * 8, 5)
    lib.cparls_peak_red_kind.restype = C.c_double
    lib.cparls_peak_red_kind.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int,
                                         C.c_int]
    red_u64 = lib.cparls_peak_red_kind(M.data_ptr(), window_rows, r, ld, 8192, 148 * 8, 5, 0)
    red_idx = {}
    if row_stream is not None and row_stream.numel() > 0:
        lib.cparls_peak_red_idx.restype = C.c_double
        lib.cparls_peak_red_idx.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                                            C.c_int]
        for name, kind in (("u64", 0), ("f64", 2)):
            red_idx[name] = lib.cparls_peak_red_idx(M.data_ptr(), row_stream.data_ptr(), row_stream.numel(), r, ld,
                                                    148 * 8, 5, kind)
    del M
    A = torch.rand(fit_rows * ld, dtype=torch.float64, device=dev)
    scr = torch.zeros(1, dtype=torch.float64, device=dev)
    gat = lib.cparls_peak_gather(A.data_ptr(), fit_rows, ld, 32768, 148 * 8, 5, scr.data_ptr())
    del A, scr
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return {"red_f64_lane_ops_per_s": red, "red_u64_lane_ops_per_s": red_u64,
            "red_stream_u64_lane_ops_per_s": red_idx.get("u64"), "red_stream_f64_lane_ops_per_s": red_idx.get("f64"),
            "red_stream_len": int(row_stream.numel()) if row_stream is not None else 0,
            "red_window_rows": window_rows,
            "gather_bytes_per_s": gat, "gather_rows": fit_rows, "rank": r, "ld": ld}


def traffic_for(kernel, config):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed ncu --set full capture (profiles/traffic.json), else None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        e = d[config][kernel]
        return float(e["dram_bytes_per_launch"])
    except Exception:
        return None


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------- oracle leg
def oracle_sample(cfg_name, frac, steps, tau):
    """Time the plain-C oracle (as it stands) for `steps` outer iterations on
    the first frac*nnz nonzeros of the config (a prefix of the same seeded
    draw sequence), same dims / r / s / tau.  Single-threaded."""
    import dataclasses
    import numpy as np
    import torch
    import oracle
    import synth
    cfg = synth.CONFIGS[cfg_name]
    nnz = max(1000, int(cfg.nnz * frac))
    sub = dataclasses.replace(cfg, nnz=nnz)
    T = synth.make(sub, device="cpu", index_dtype=torch.int64)
    o = oracle.Oracle(cfg.dims, T.coords.numpy(), T.vals.to(torch.float64).numpy(), cfg.rank)
    init = synth.uniform_init(cfg.dims, cfg.rank, cfg.init_seed)
    for k in range(len(cfg.dims)):
        o.set_factor(k, init[k].numpy())
    times = []
    D = len(cfg.dims)
    for t in range(steps):
        t0 = time.perf_counter()
        for k in range(D):
            o.sample(k, cfg.s, tau, cfg.sample_seed, t * D + k)
            o.solve_mode(k)
        if (t + 1) % ETA == 0:
            o.fit()
        times.append(time.perf_counter() - t0)
    # amortize one fit per ETA iterations even if steps < ETA
    tf0 = time.perf_counter(); o.fit(); tfit = time.perf_counter() - tf0
    nfits = steps // ETA
    total = sum(times) + (steps / ETA - nfits) * tfit
    return {"value": steps / total, "unit": "iterations/s", "cores": 1, "kind": "oracle", "host": host_info(),
            "sample": f"{steps} outer iteration(s) of the plain-C oracle (1 thread) on the first {nnz} "
                      f"nonzeros ({frac:.4%}) of {cfg_name}'s seeded draw sequence, full dims "
                      f"{cfg.dims}, r={cfg.rank}, s={cfg.s}, tau={'1/s' if tau < 0 else tau}, "
                      f"exact fit amortized 1/{ETA}"}


def host_info():
    """nproc, CPU model and host RAM (SURVEY 8(d) oracle timing)."""
    info = {"nproc": os.cpu_count()}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                info["ram_gb"] = round(int(line.split()[1]) / 2 ** 20, 1)
                break
    except OSError:
        pass
    return info


def run_reference(args):
    ws, rk, _ = dist_env()
    if rk != 0:
        return
    import synth
    cfg = synth.CONFIGS[args.config]
    steps = max(1, args.steps)
    # warmup iterations of a CPU program are not needed for timing; keep the
    # run bounded: W is honored only up to 1
    if args.warmup > 0:
        oracle_sample(args.config, args.sample_frac, 1, args.tau)
    cb = oracle_sample(args.config, args.sample_frac, steps, args.tau)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "iterations/s",
            "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 / cb["value"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "dims": list(cfg.dims), "rank": cfg.rank, "s": cfg.s,
                       "tau": "1/s" if args.tau < 0 else args.tau, "oracle_sample": cb["sample"]},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "iterations/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch
    import synth
    from paper_2006_16438_b200 import Cparls

    ws, rk, lrk = dist_env()
    torch.cuda.set_device(lrk)
    dev = torch.device("cuda", lrk)
    comm = None
    if ws > 1:
        # one process per GPU (torchrun); torch.distributed only carries the NCCL
        # id and the max-over-ranks timing, libcparls runs its own NCCL comm
        import torch.distributed as dist
        dist.init_process_group("gloo")
        from paper_2006_16438_b200 import Comm
        obj = [Comm.nccl_unique_id() if rk == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = Comm.nccl(ws, rk, obj[0])
    cfg = synth.CONFIGS[args.config]
    D = len(cfg.dims)
    t0 = time.perf_counter()
    # this rank's chunk of the COO only (cells rk, rk + ws, ... of the tensor);
    # cparls_create routes the nonzeros to the owners of their rows
    T = synth.make(cfg, device=dev, index_dtype=torch.int32, part=rk, parts=ws)
    coords, vals = T.coords, T.vals
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    nnz = cfg.nnz
    host = None
    if not args.no_e2e:
        host = (torch.empty(coords.shape, dtype=coords.dtype, pin_memory=True),
                torch.empty(vals.shape, dtype=vals.dtype, pin_memory=True))
        host[0].copy_(coords)
        host[1].copy_(vals)
        # the caller's pinned destination buffers for the factors read back
        host_out = [(torch.empty((cfg.dims[m], cfg.rank), dtype=torch.float64, pin_memory=True),
                     torch.empty(cfg.rank, dtype=torch.float64, pin_memory=True)) for m in range(D)]
    torch.cuda.empty_cache()
    stream = torch.cuda.current_stream(dev)
    t0 = time.perf_counter()
    # the paper's estimated-fit sample for its Amazon runs: s_fit = 2^27,
    # drawn once at create (single GPU; the exact fit is the headline)
    fit_samples = FIT_SAMPLES if ws == 1 else 0
    g = Cparls(cfg.dims, coords, vals, cfg.rank, tau=args.tau, init_seed=cfg.init_seed,
               stream=stream.cuda_stream, comm=comm, world_size=ws, world_rank=rk,
               fit_samples=fit_samples, fit_seed=FIT_SEED)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    create_phases = dict(zip(["setup_and_input_ms", "sorted_copies_ms", "dups_fibers_fit_sample_ms",
                              "factors_leverage_ms"], g.stats()["create_ms"]))
    create_phases["sorted_copies_split_ms"] = dict(zip(["cudaMalloc_free", "radix_sorts", "key_kernels_directory",
                                                        "hot_rows"], g.stats()["build_ms"]))
    del coords, vals, T
    torch.cuda.empty_cache()

    seed = cfg.sample_seed
    # clocks are sampled (200 ms nvidia-smi interval) from the first warm-up
    # iteration through the end of the timed region: the same workload, and a
    # short timed region (small configs) still gets samples
    clk = Clocks(lrk).__enter__()
    # warmup
    for t in range(args.warmup):
        g.run(1, cfg.s, seed, iter0=t, fit_every=0)
    if args.profile_phases:
        g.set_profiling(True)
    K = args.steps
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    g.reset_stats()
    if ws > 1:
        dist.barrier()
    try:
        ev0.record(stream)
        # K iterations with the exact fit at every epoch end (eta = 5, Alg. 3)
        trace = g.run(K, cfg.s, seed, iter0=args.warmup, fit_every=ETA)
        ev1.record(stream)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
    finally:
        clk.__exit__()
    ms = ev0.elapsed_time(ev1)
    if ws > 1:   # the job's time is the slowest rank's
        tt = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt[0])
    st = g.stats()          # resolves the per-kernel event timers of the timed region
    # k_rhs's own row stream at the state the timed run left (for its ceiling)
    row_stream = None
    if ws == 1:
        ld_ = row_ld(cfg.rank)
        row_stream = rhs_row_stream(g, cfg, seed, min(max(cfg.dims), (96 << 20) // (ld_ * 8)))
    # SURVEY 8(d) byte model of the timed region (cparls_stats counters: what
    # the method must touch, not the traffic) per iteration, against HBM
    model_bytes = sum(st[k] for k in st if k.startswith("bytes_")) / K
    iter_roofline = {"bytes_per_iteration": model_bytes, "achieved_GBps": model_bytes / (ms / K / 1e3) / 1e9,
                     "what": "SURVEY 8(d) algorithmic bytes per outer iteration (sample, Gram, lookup, RHS, "
                             "solve, leverage, exact fit / eta) over the measured ms per iteration"}
    # per-iteration CUDA-event times (no fit), mean and median over iterations 2..K
    per_it = []
    if ws == 1:
        for t in range(K):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.run(1, cfg.s, seed, iter0=args.warmup + t, fit_every=0)
            b.record(stream)
            b.synchronize()
            per_it.append(a.elapsed_time(b))
    tail = sorted(per_it[1:]) if len(per_it) > 1 else per_it
    per_iteration = {"mean_ms": sum(tail) / len(tail), "median_ms": tail[len(tail) // 2],
                     "what": "one outer iteration without the fit, iterations 2..K"} if tail else None
    # iterations/s with the exact fit every iteration (fit_every = 1)
    fe1 = None
    if ws == 1:
        K1 = min(K, 5)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        g.run(K1, cfg.s, seed, iter0=args.warmup, fit_every=1)
        b.record(stream)
        torch.cuda.synchronize()
        fe1 = {"value": K1 / (a.elapsed_time(b) / 1e3), "unit": "iterations/s", "iterations": K1}
    # secondary: the same K iterations with the paper's estimated fit
    # per epoch instead of the exact one (Alg. 3 as run on Amazon, s_fit = 2^27)
    est = None
    if fit_samples:
        g.reset_stats()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for t in range(K):
            g.run(1, cfg.s, seed, iter0=args.warmup + K + t, fit_every=0)
            if (t + 1) % ETA == 0:
                g.fit_estimate()
        e1.record(stream)
        torch.cuda.synchronize()
        st_est = g.stats()
        nf = st_est["kernel_launches_by_id"]["fit"]
        est = {"value": K / (e0.elapsed_time(e1) / 1000.0), "unit": "iterations/s", "s_fit": FIT_SAMPLES,
               "fit_alpha": 0.5, "fit_est_kernel_avg_ms": (st_est["kernel_ms"]["fit"] / nf) if nf else None,
               "fit_estimate": g.fit_estimate()[0],
               "what": "same K iterations, estimated fit (stratified sample, frozen at create) per epoch"}
    if st["fits"] == 0:     # K < ETA: time one fit so the fit kernel is still reported
        g.fit()
        st_fit = g.stats()
        st["kernel_ms"]["fit"] = st_fit["kernel_ms"]["fit"]
        st["kernel_launches_by_id"]["fit"] = st_fit["kernel_launches_by_id"]["fit"]
    value = K / (ms / 1000.0)
    vbytes = 4 if cfg.value_dtype == "f32" else 8
    # RRF initialization timed once, the paper's s_init = 1e5
    # (P:1691); it replaces the factors, so it runs after the timed regions
    rrf_ms = None
    if ws == 1:
        torch.cuda.synchronize()
        r0 = time.perf_counter()
        g.init_rrf(100000, 7)
        torch.cuda.synchronize()
        rrf_ms = (time.perf_counter() - r0) * 1e3
    # secondary: the exact CP-ALS baseline on the same
    # copies, with the exact fit every iteration (its stopping test)
    als = None
    if ws == 1:
        KA = 3
        g.reset_stats()
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True); a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        g.run_als(KA, fit_every=1)
        a1.record(stream)
        torch.cuda.synchronize()
        st_als = g.stats()
        va = KA / (a0.elapsed_time(a1) / 1000.0)
        als = {"value": va, "unit": "iterations/s", "iterations": KA, "fit_every": 1,
               "mttkrp_avg_ms": st_als["kernel_ms"]["rhs"] / max(1, st_als["kernel_launches_by_id"]["rhs"]),
               "cparls_iteration_speedup": value / va,
               "what": "exact CP-ALS (full sparse MTTKRP per mode + V^+ solve + exact fit) on the same GPU"}
    final_fit = g.fit()
    if args.profile_phases:
        sys.stderr.write(json.dumps({k: v for k, v in st.items()}, indent=1) + "\n")
    g.close()
    del g
    torch.cuda.empty_cache()
    kms, kn = st["kernel_ms"], st["kernel_launches_by_id"]
    # share of the timed region; a fit timed outside it (K < eta) is amortized 1/eta per step
    share = {k: kms[k] / ms for k in kms}
    if st["fits"] == 0 and kn["fit"]:
        share["fit"] = kms["fit"] / kn["fit"] / ETA / (ms / K)
    KN = kernel_names(cfg.rank)
    kernels = {KN[k]: {"launches": int(kn[k]), "avg_ms": (kms[k] / kn[k]) if kn[k] else None,
                                 "share_of_step": share[k]} for k in kms}
    dominant = max(share, key=lambda k: share[k])
    ld = row_ld(cfg.rank)
    window_rows = min(max(cfg.dims), (96 << 20) // (ld * 8))
    hbm_peak, peak_src = measured_peaks()
    # measured ceilings of the hot kernels' access patterns (same GPU, same run)
    row_stream = row_stream.to(dev) if row_stream is not None else None
    peaks = measure_peaks(cfg, dev, window_rows, int(sorted(cfg.dims)[len(cfg.dims) // 2]), row_stream)
    del row_stream
    iter_roofline.update({"peak_GBps": hbm_peak, "frac": iter_roofline["achieved_GBps"] / hbm_peak,
                          "frac_nominal_8TBps": iter_roofline["achieved_GBps"] / 8000.0})
    # k_rhs: algorithmic work = m_k * r fp64 reductions per launch (SURVEY 8(d):
    # every matched nonzero adds w^2 x z_j to its output row); bytes = matched
    # entries (out + value) + touched output rows read and written once
    n_rhs = max(1, kn["rhs"])
    rhs_red = st["sum_matched_nnz"] * cfg.rank / n_rhs
    rhs_bytes = st["sum_matched_nnz"] * (4 + vbytes) / n_rhs + sum(cfg.dims) / D * cfg.rank * 8 * 2
    rhs_avg_s = (kms["rhs"] / n_rhs) / 1000.0 if kn["rhs"] else None
    # exact fit: algorithmic bytes: every nonzero of the fit
    # mode's copy (key u64 + out i32 + value) plus every factor row once
    fit_alg_bytes = nnz * (8 + 4 + vbytes) + sum(cfg.dims) * cfg.rank * 8
    fit_avg_s = (kms["fit"] / max(1, kn["fit"])) / 1000.0 if kn["fit"] else None
    rl = {}
    if rhs_avg_s:
        pk = peaks["red_stream_u64_lane_ops_per_s"] or peaks["red_u64_lane_ops_per_s"]
        rl["rhs"] = {"bound": "hbm", "kernel": "k_rhs (sampled RHS, P:949-958)",
                     "achieved": rhs_bytes / rhs_avg_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
                     "frac": rhs_bytes / rhs_avg_s / 1e9 / hbm_peak,
                     "traffic": traffic_for("k_rhs", args.config), "alg_bytes_per_launch": rhs_bytes,
                     "avg_launch_ms": rhs_avg_s * 1e3, "peak_source": peak_src,
                     "alg_bytes_what": "SURVEY 8(d): matched entries m_k*(4+v) + the output rows of M read and "
                                       "written once (n_k*r*16), per launch",
                     "l2_reduction_view": {
                         "achieved": rhs_red / rhs_avg_s / 1e9, "peak": pk / 1e9,
                         "unit": "G int64 fixed-point reductions/s", "frac": (rhs_red / rhs_avg_s) / pk,
                         "peak_source": f"measured here: cparls_peak_red_idx, r-lane u64 red (nothing else) "
                                        f"into the rows of {peaks['red_stream_len']} matched fiber entries of "
                                        f"fresh samples in the first {window_rows}-row output window",
                         "what": "the kernel's binding ceiling: r-lane L2 reductions issued vs the rate the "
                                 "SM->L2 write path retires them (DESIGN.md section 8)"}}
    if fit_avg_s:
        gather_bytes = nnz * ld * 8.0     # one A_{k*} row per nonzero (the per-entry gather)
        rl["fit"] = {"bound": "hbm", "kernel": "k_fit_sub (exact fit, P:867-875)",
                     "achieved": fit_alg_bytes / fit_avg_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
                     "frac": fit_alg_bytes / fit_avg_s / 1e9 / hbm_peak,
                     "traffic": traffic_for("k_fit_sub", args.config), "alg_bytes_per_launch": fit_alg_bytes,
                     "avg_launch_ms": fit_avg_s * 1e3, "peak_source": peak_src,
                     "gather_view": {"achieved": gather_bytes / fit_avg_s / 1e9,
                                     "peak": peaks["gather_bytes_per_s"] / 1e9, "unit": "GB/s",
                                     "frac": gather_bytes / fit_avg_s / peaks["gather_bytes_per_s"],
                                     "what": "per-nonzero A_k* row gathers vs measured random-row gather rate"}}
    roofline = dict(rl.get(dominant, rl.get("rhs") or rl.get("fit") or {}))
    roofline["dominant"] = KN[dominant]
    roofline["others"] = {KN[k]: v for k, v in rl.items() if k != dominant}

    # e2e: public API from pinned host buffers (create + K iterations + fits + factors back)
    e2e = None
    if host is not None:
        torch.cuda.synchronize()
        # the driver reclaims the memory of the context closed above in the
        # background; cudaMalloc right after such a free waits for it (~0.4-1 s
        # on C4, profiles/r02_create_after_free_C4.json) -- a cost of this
        # benchmark's earlier context, not of the user's call, so let it settle
        time.sleep(5.0)
        hc, hv = host
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        w0 = time.perf_counter()
        g2 = Cparls(cfg.dims, hc.numpy(), hv.numpy(), cfg.rank, tau=args.tau, init_seed=cfg.init_seed,
                    stream=stream.cuda_stream, comm=comm, world_size=ws, world_rank=rk)
        w1 = time.perf_counter()
        d2h = 0
        g2.run(K, cfg.s, seed, iter0=0, fit_every=ETA)
        d2h += 8 * (K // ETA)
        w2 = time.perf_counter()
        for m in range(D):
            A, lam = g2.get_factor(m, out=host_out[m][0].numpy(), lam_out=host_out[m][1].numpy())
            d2h += A.nbytes + lam.nbytes
        e1.record(stream)
        torch.cuda.synchronize()
        w3 = time.perf_counter()
        ems = e0.elapsed_time(e1)
        if ws > 1:
            tt = torch.tensor([ems], dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt[0])
        create2 = dict(zip(["setup_and_input_ms", "sorted_copies_ms", "dups_fibers_fit_sample_ms",
                            "factors_leverage_ms"], g2.stats()["create_ms"]))
        create2["sorted_copies_split_ms"] = dict(zip(["cudaMalloc_free", "radix_sorts", "key_kernels_directory",
                                                      "hot_rows"], g2.stats()["build_ms"]))
        g2.close()
        h2d = hc.numel() * hc.element_size() + hv.numel() * hv.element_size()
        e2e = {"value": K / (ems / 1000.0), "unit": "iterations/s", "h2d_bytes_per_step": h2d // K,
               "d2h_bytes_per_step": d2h // K,
               "wall_s": {"create_from_host": w1 - w0, "run": w2 - w1, "factors_to_host": w3 - w2},
               "create_phases": create2,
               "includes": "cparls_create from pinned host COO (H2D + per-mode index build) + K iterations + "
                           "fits every 5 + factors back into pinned host buffers"}

    cpu = None
    if not args.no_cpu_baseline and rk == 0 and ws == 1:
        cpu = oracle_sample(args.config, args.sample_frac, 1, args.tau)

    line = {
        "metric": METRIC, "value": value, "unit": "iterations/s", "n_gpus": ws, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms / K, "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "dims": list(cfg.dims), "nnz": int(nnz), "rank": cfg.rank,
                   "s": cfg.s, "tau": "1/s" if args.tau < 0 else args.tau, "fit_every": ETA,
                   "values": cfg.value_dtype, "l2": "inputs larger than L2 (per-mode sorted copies "
                   f"{nnz * (16 if cfg.value_dtype == 'f32' else 20) * D / 1e9:.1f} GB >> 126 MB)",
                   "parallelism": f"row-sharded x{ws} (per mode step: sampled rows from their owners, p~ allgather, "
                                  f"r x r Gram allreduce; dense factors once per fit)" if ws > 1 else "single GPU"},
        "roofline": roofline,
        "kernels": kernels,
        "peaks_measured": peaks,
        "clocks": clk.summary(),
        "gpu_launches": int(st["kernel_launches"]),
        "host_syncs_in_timed_region": int(st["host_syncs"]),
        "e2e": e2e,
        "cpu_baseline": cpu,
        "fit": final_fit,
        "estimated_fit_variant": est,
        "cp_als_baseline": als,
        "setup": {"generate_s": t_gen, "create_s": t_build, "create_phases": create_phases, "rrf_init_ms": rrf_ms},
        "iteration_roofline": iter_roofline,
        "per_iteration": per_iteration,
        "fit_every_1": fe1,
        "phases_ms": {k[3:]: st[k] for k in st if k.startswith("ms_")} if args.profile_phases else None,
        "counters": {"last_matched_nnz": st["last_matched_nnz"], "last_s_bar": st["last_s_bar"],
                     "last_attempts": st["last_attempts"], "touched_rows": st["touched_rows"][:D]},
    }
    if rk == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
