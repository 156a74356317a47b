"""Fraction of C4's nonzeros whose mode-k row is among the top-K rows by degree
(how much of the per-nonzero factor-row gather an L2-resident hot set could serve)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
cfg = synth.CONFIGS["C4"]
T = synth.make(cfg, device="cuda", index_dtype=torch.int32)
out = {}
for k in range(3):
    deg = torch.bincount(T.coords[:, k].long(), minlength=cfg.dims[k]).double()
    d, _ = torch.sort(deg, descending=True)
    cs = torch.cumsum(d, 0) / d.sum()
    out[k] = {K: float(cs[min(K, len(cs)) - 1]) for K in (256, 512, 1024, 2048, 4096, 10_000, 50_000, 100_000, 400_000)}
    out[k]["n"] = cfg.dims[k]
print(json.dumps(out))
