"""cparls_run (K iterations, exact fit every 5) with opts.fit_overlap 0 and 1:
CUDA-event ms per iteration and the fit traces."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2006_16438_b200 import Cparls
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
T = synth.make(cfg, device="cuda", index_dtype=torch.int32)
torch.cuda.synchronize(); torch.cuda.empty_cache()
st = torch.cuda.current_stream()
out = {"config": cfg.name, "K": K}
for rep in range(2):
    for fo in (0, 1):
        g = Cparls(cfg.dims, T.coords, T.vals, cfg.rank, fit_overlap=fo, stream=st.cuda_stream)
        g.run(5, cfg.s, cfg.sample_seed, iter0=0, fit_every=5)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        tr = g.run(K, cfg.s, cfg.sample_seed, iter0=5, fit_every=5)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        out[f"overlap{fo}_rep{rep}"] = {"ms_per_iter": ms, "it_per_s": 1000 / ms,
                                        "trace": [float(x) for x in tr if not np.isnan(x)]}
        g.close(); del g
        torch.cuda.empty_cache()
print(json.dumps(out))
