"""Feasibility timing (not product): device radix sort of RHS-sized pair arrays."""
import torch, time
n = 160_000_000
g = torch.Generator(device="cuda"); g.manual_seed(0)
keys = torch.randint(0, 4_800_000, (n,), device="cuda", dtype=torch.int32, generator=g)
vals = torch.randint(0, 2**62, (n,), device="cuda", dtype=torch.int64, generator=g)
for name, fn in [("sort_i32_stable", lambda: torch.sort(keys, stable=True)),
                 ("sort_i64_keys", lambda: torch.sort(keys.to(torch.int64) << 32 | (vals & 0xffffffff), stable=False))]:
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): fn()
    e1.record(); torch.cuda.synchronize()
    print(name, e0.elapsed_time(e1) / 5, "ms", flush=True)
