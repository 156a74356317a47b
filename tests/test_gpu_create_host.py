"""cparls_create from host COO: the chunked host->device copy (above 2^27
nonzeros: 4 chunks of 40/30/20/10% on a copy stream; every mode's composite keys of a chunk made and sorted
while later chunks are in flight, the sorted runs merged at the end) must give
the same context as a create from device memory (one full stable sort per
mode) -- identical sorted copies, hence identical samples, factors and fits,
bit for bit.  A C4-shaped tensor of 150M nonzeros plus 1M duplicated
coordinates (copies of chunk-0 nonzeros with other values, placed in the last
chunk: the merge must keep input order among equal keys) spans four chunks.  Also: factors read back into pinned and pageable host
buffers agree exactly."""
import dataclasses

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

NNZ = 150_000_123          # > 2^27: four chunks
NDUP = 1_000_000


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def test_create_from_host_chunks_equals_device():
    need_gpu()
    from paper_2006_16438_b200 import Cparls
    cfg = dataclasses.replace(synth.CONFIGS["C4"], nnz=NNZ)
    dev = torch.device("cuda", 0)
    T = synth.make(cfg, device=dev, index_dtype=torch.int32)
    dc = torch.cat([T.coords, T.coords[:NDUP]])
    dv = torch.cat([T.vals, T.vals[:NDUP] * 2 + 1])
    del T
    hc = torch.empty(dc.shape, dtype=dc.dtype, pin_memory=True)
    hv = torch.empty(dv.shape, dtype=dv.dtype, pin_memory=True)
    hc.copy_(dc)
    hv.copy_(dv)
    torch.cuda.synchronize()
    traces, facs = [], []
    for src in ("device", "pinned", "pageable"):
        if src == "device":
            c, v = dc, dv
        elif src == "pinned":
            c, v = hc.numpy(), hv.numpy()
        else:
            c, v = hc.numpy().copy(), hv.numpy().copy()
        g = Cparls(cfg.dims, c, v, cfg.rank, tau=-1.0, init_seed=cfg.init_seed)
        traces.append(g.run(3, cfg.s, cfg.sample_seed, iter0=0, fit_every=1))
        facs.append([g.get_factor(m) for m in range(len(cfg.dims))])
        if src == "pinned":
            # the same factors into pinned host and device destinations
            for m in range(len(cfg.dims)):
                po = torch.empty((cfg.dims[m], cfg.rank), dtype=torch.float64, pin_memory=True)
                pl = torch.empty(cfg.rank, dtype=torch.float64, pin_memory=True)
                A, lam = g.get_factor(m, out=po.numpy(), lam_out=pl.numpy())
                assert A.ctypes.data == po.data_ptr()
                assert np.array_equal(A, facs[-1][m][0]) and np.array_equal(lam, facs[-1][m][1])
        g.close()
    for t in traces[1:]:
        assert np.array_equal(t, traces[0]), (t, traces[0])
    for f in facs[1:]:
        for (A, lam), (A0, lam0) in zip(f, facs[0]):
            assert np.array_equal(A, A0) and np.array_equal(lam, lam0)
    assert np.all(np.isfinite(traces[0])) and traces[0][-1] > 0


def test_create_from_host_rejects_bad_coordinate_in_last_chunk():
    need_gpu()
    from paper_2006_16438_b200 import Cparls
    dims = (1000, 900, 800)
    n = (1 << 27) + 5
    rng = np.random.default_rng(0)
    coords = np.stack([rng.integers(0, d, n, dtype=np.int32) for d in dims], axis=1)
    vals = rng.random(n, dtype=np.float32)
    coords[-1, 2] = dims[2]          # out of range, in the last chunk
    with pytest.raises(Exception):
        Cparls(dims, coords, vals, 5, tau=-1.0, init_seed=1)
