"""A/B of a library build (CPARLS_LIB) on a config: ms per iteration of
cparls_run (K iterations, exact fit every 5) and the hot kernels' CUDA-event
times (cparls_stats.kernel_ms), after W warm-up iterations."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2006_16438_b200 import Cparls
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
T = synth.make(cfg, device="cuda", index_dtype=torch.int32)
torch.cuda.synchronize(); torch.cuda.empty_cache()
st = torch.cuda.current_stream()
g = Cparls(cfg.dims, T.coords, T.vals, cfg.rank, stream=st.cuda_stream)
del T
torch.cuda.empty_cache()
g.run(3, cfg.s, cfg.sample_seed, iter0=0, fit_every=0)
g.reset_stats()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(st)
tr = g.run(K, cfg.s, cfg.sample_seed, iter0=3, fit_every=5)
e1.record(st)
torch.cuda.synchronize()
s = g.stats()
out = {"lib": os.environ.get("CPARLS_LIB", "default"), "config": cfg.name, "ms_per_iter": e0.elapsed_time(e1) / K,
       "kernel_avg_ms": {k: s["kernel_ms"][k] / max(1, s["kernel_launches_by_id"][k]) for k in s["kernel_ms"]},
       "trace": [float(x) for x in tr]}
print(json.dumps(out))
