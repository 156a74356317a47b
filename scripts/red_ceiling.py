"""fp64 r-lane reduction ceiling vs the size of the row window (diagnostics)."""
import ctypes as C, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
lib = C.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2006_16438_b200", "libcparls_peaks.so"))
lib.cparls_peak_red_f64.restype = C.c_double
lib.cparls_peak_red_f64.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int]
ld, r = 28, 25
for mb in (4, 16, 32, 64, 96, 128, 256, 1024):
    rows = (mb << 20) // (ld * 8)
    M = torch.zeros(rows * ld, dtype=torch.float64, device="cuda")
    for blocks in (148 * 8, 148 * 16):
        v = lib.cparls_peak_red_f64(M.data_ptr(), rows, r, ld, 4096, blocks, 5)
        print(json.dumps({"window_MB": mb, "blocks": blocks, "G_lane_ops_s": v / 1e9}), flush=True)
    del M

lib.cparls_peak_red_kind.restype = C.c_double
lib.cparls_peak_red_kind.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int]
for mb in (32, 96):
    rows = (mb << 20) // (ld * 8)
    M = torch.zeros(rows * ld, dtype=torch.float64, device="cuda")
    for kind, name in ((0, "u64"), (1, "f32")):
        v = lib.cparls_peak_red_kind(M.data_ptr(), rows, r, ld, 4096, 148 * 8, 5, kind)
        print(json.dumps({"window_MB": mb, "type": name, "G_lane_ops_s": v / 1e9}), flush=True)
    del M
