"""cparls_create timing on C4: from device COO and from pinned host COO (with the
first context closed), with the library's create_ms / build_ms split."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2006_16438_b200 import Cparls
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
T = synth.make(cfg, device="cuda", index_dtype=torch.int32)
hc = torch.empty(T.coords.shape, dtype=T.coords.dtype, pin_memory=True); hc.copy_(T.coords)
hv = torch.empty(T.vals.shape, dtype=T.vals.dtype, pin_memory=True); hv.copy_(T.vals)
torch.cuda.synchronize()
t0 = time.perf_counter(); d = hc.cuda(); e = hv.cuda(); torch.cuda.synchronize(); t_h2d = time.perf_counter() - t0
del d, e
torch.cuda.empty_cache()
out = {"h2d_torch_s": t_h2d, "h2d_GBps": (hc.numel() * 4 + hv.numel() * 4) / t_h2d / 1e9}
for rep in range(3):
    if rep == 2:
        time.sleep(5.0)   # let the driver finish with the memory freed by the previous context
    t0 = time.perf_counter(); g = Cparls(cfg.dims, T.coords, T.vals, cfg.rank); torch.cuda.synchronize()
    st = g.stats()
    out[f"dev{rep}"] = {"s": time.perf_counter() - t0, "create_ms": st["create_ms"], "build_ms": st["build_ms"],
                        "after_sleep": rep == 2}
    g.close(); del g
del T
torch.cuda.empty_cache()
for rep in range(2):
    if rep == 1:
        g.close(); del g
        torch.cuda.empty_cache()
        time.sleep(5.0)
    t0 = time.perf_counter(); g = Cparls(cfg.dims, hc.numpy(), hv.numpy(), cfg.rank); torch.cuda.synchronize()
    st = g.stats()
    out[f"host{rep}"] = {"s": time.perf_counter() - t0, "create_ms": st["create_ms"], "build_ms": st["build_ms"],
                         "after_sleep": rep == 1}
print(json.dumps(out), flush=True)
