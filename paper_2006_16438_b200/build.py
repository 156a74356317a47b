"""Build libcparls.so (sm_100a) in-tree with nvcc."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "cparls.cu")
LIB = os.path.join(HERE, "libcparls.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
def _nccl_dir():
    """NCCL shipped with torch (the library torch.distributed loads)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    return None


NCCL = _nccl_dir()
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-O2", "-shared", "--expt-relaxed-constexpr", "-Xptxas", "-v"]
if NCCL:
    FLAGS += ["-I" + os.path.join(NCCL, "include"), "-L" + os.path.join(NCCL, "lib"),
              "-Xlinker", "-rpath," + os.path.join(NCCL, "lib")]


def sources():
    d = os.path.join(HERE, "csrc")
    return [os.path.join(d, f) for f in os.listdir(d) if f.endswith((".cu", ".cuh"))] + [
        os.path.join(HERE, "..", "include", "cparls.h")]


PEAKS_SRC = os.path.join(HERE, "csrc", "peaks.cu")
PEAKS_LIB = os.path.join(HERE, "libcparls_peaks.so")


def _nvcc(out, src, libs, verbose):
    cmd = [NVCC] + FLAGS + ["-o", out + ".tmp", src] + libs
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed: " + src)
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(out + ".tmp", out)


def build(force=False, verbose=False, lib=None, extra=()):
    """libcparls.so (the product) and libcparls_peaks.so (bench-only microbenchmarks).
    lib/extra: build a variant library (e.g. -D flags) at another path (experiments)."""
    if lib is not None:
        _nvcc(lib, SRC, ["-lcudart", "-l:libnccl.so.2"] + list(extra), verbose)
        return lib
    if force or not os.path.exists(PEAKS_LIB) or os.path.getmtime(PEAKS_LIB) < os.path.getmtime(PEAKS_SRC):
        _nvcc(PEAKS_LIB, PEAKS_SRC, ["-lcudart"], verbose)
    srcs = [s for s in sources() if s != PEAKS_SRC]
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(s) for s in srcs):
        return LIB
    _nvcc(LIB, SRC, ["-lcudart", "-l:libnccl.so.2"], verbose)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
