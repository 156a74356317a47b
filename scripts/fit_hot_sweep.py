# round-2 experiment (gpu call 38): the fit_hot_rows option it sweeps was measured slower and removed
"""Exact-fit kernel time on C4 for several fit_hot_rows settings (0 = off)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2006_16438_b200 import Cparls
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
T = synth.make(cfg, device="cuda", index_dtype=torch.int32)
torch.cuda.synchronize()
torch.cuda.empty_cache()
out = {"lib": os.environ.get("CPARLS_LIB", "default")}
for hot in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,128,256,448,1024").split(",")]:
    g = Cparls(cfg.dims, T.coords, T.vals, cfg.rank, fit_hot_rows=hot)
    g.run(1, cfg.s, cfg.sample_seed, iter0=0, fit_every=0)
    f0 = g.fit()
    g.reset_stats()
    for _ in range(3):
        f = g.fit()
    st = g.stats()
    out[hot] = {"fit_ms": st["kernel_ms"]["fit"] / 3, "fit": f, "rows": st["fit_hot_rows"], "share": st["fit_hot_share"]}
    print(hot, out[hot], flush=True)
    g.close(); del g
    torch.cuda.empty_cache()
print(json.dumps(out))
