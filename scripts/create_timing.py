import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2006_16438_b200 import Cparls
cfg = synth.CONFIGS["C4"]
T = synth.make(cfg, device="cuda", index_dtype=torch.int32)
hc = torch.empty(T.coords.shape, dtype=T.coords.dtype, pin_memory=True); hc.copy_(T.coords)
hv = torch.empty(T.vals.shape, dtype=T.vals.dtype, pin_memory=True); hv.copy_(T.vals)
torch.cuda.synchronize()
t0 = time.perf_counter(); d = hc.cuda(); e = hv.cuda(); torch.cuda.synchronize(); t_h2d = time.perf_counter() - t0
del d, e
torch.cuda.empty_cache()
t0 = time.perf_counter(); g = Cparls(cfg.dims, T.coords, T.vals, cfg.rank); torch.cuda.synchronize(); t_dev = time.perf_counter() - t0
g.close(); del g
del T
torch.cuda.empty_cache()
t0 = time.perf_counter(); g = Cparls(cfg.dims, hc.numpy(), hv.numpy(), cfg.rank); torch.cuda.synchronize(); t_host = time.perf_counter() - t0
print(json.dumps({"h2d_torch_s": t_h2d, "h2d_GBps": (hc.numel() * 4 + hv.numel() * 4) / t_h2d / 1e9, "create_from_device_s": t_dev, "create_from_host_s": t_host}), flush=True)
