# round-2 experiment (gpu call 40): the fit_overlap_sms option it sweeps was measured slower on C4 and removed
"""cparls_run (K iterations, exact fit every 5) on C4 for several
fit_overlap_sms settings (0 = inline fit): CUDA-event time per iteration and
the fit trace (identical up to the double-double rounding)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2006_16438_b200 import Cparls
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
settings = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,74,37,111").split(",")]
K = int(sys.argv[3]) if len(sys.argv) > 3 else 20
T = synth.make(cfg, device="cuda", index_dtype=torch.int32)
torch.cuda.synchronize(); torch.cuda.empty_cache()
st = torch.cuda.current_stream()
out = {}
ref = None
for sms in settings:
    g = Cparls(cfg.dims, T.coords, T.vals, cfg.rank, fit_overlap_sms=sms, stream=st.cuda_stream)
    g.run(5, cfg.s, cfg.sample_seed, iter0=0, fit_every=5)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    tr = g.run(K, cfg.s, cfg.sample_seed, iter0=5, fit_every=5)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    tr = [float(x) for x in tr if not np.isnan(x)]
    if ref is None:
        ref = tr
    out[sms] = {"ms_per_iter": ms, "it_per_s": 1000 / ms, "trace": tr,
                "max_trace_diff": max(abs(a - b) for a, b in zip(tr, ref))}
    print(sms, out[sms], flush=True)
    g.close(); del g
    torch.cuda.empty_cache()
print(json.dumps(out))
