"""CPU-side checks of the boundary: libcparls.so builds for sm_100a, loads, and
exports every symbol include/cparls.h declares; the binding refuses to run
without a GPU (no CPU fallback).  No compute calls here."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cparls.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cparls_[a-z_]+)\s*\(", src)))


def test_library_builds_and_exports_all_declared_symbols():
    from paper_2006_16438_b200 import build
    lib_path = build.build()
    L = ctypes.CDLL(lib_path)
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), f"{s} declared in cparls.h but not exported"
    from paper_2006_16438_b200 import cparls
    assert set(syms) == set(cparls.EXPORTED)


def test_library_is_sm100a_code():
    from paper_2006_16438_b200 import build
    lib_path = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_string():
    from paper_2006_16438_b200 import build, cparls
    build.build()
    assert "sm_100a" in cparls.version()


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    from paper_2006_16438_b200 import Cparls
    with pytest.raises(RuntimeError):
        Cparls((2, 2, 2), np.zeros((1, 3), dtype=np.int32), np.ones(1), 1)


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2006_16438_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "cparls_oracle" not in txt and "or_create" not in txt, f


def _c_layout(struct, fields):
    """sizeof and offsetof(field) of a cparls.h struct, from gcc on the header."""
    import tempfile
    body = "\n".join(f'printf("%zu\\n", offsetof({struct}, {f}));' for f in fields)
    src = ("#include <stdio.h>\n#include <stddef.h>\n#include \"cparls.h\"\n"
           f"int main(void) {{ printf(\"%zu\\n\", sizeof({struct})); {body} return 0; }}\n")
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "l.c")
        exe = os.path.join(d, "l")
        open(c, "w").write(src)
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", exe, c], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    return [int(x) for x in out]


@pytest.mark.parametrize("name", ["Opts", "Stats", "SampleInfo", "SolveInfo"])
def test_binding_struct_layouts_match_header(name):
    """The ctypes mirrors of cparls_opts / cparls_stats / the info structs have
    the header's size and field offsets (struct_size versioning relies on it)."""
    from paper_2006_16438_b200 import cparls
    cls = getattr(cparls, name)
    cname = {"Opts": "cparls_opts", "Stats": "cparls_stats", "SampleInfo": "cparls_sample_info",
             "SolveInfo": "cparls_solve_info"}[name]
    fields = [f for f, _ in cls._fields_]
    got = _c_layout(cname, fields)
    assert got[0] == ctypes.sizeof(cls), (name, got[0], ctypes.sizeof(cls))
    for f, off in zip(fields, got[1:]):
        assert getattr(cls, f).offset == off, (name, f)


def test_no_environment_knobs_in_the_library():
    """Numerics and code paths are chosen through cparls_opts only (no getenv)."""
    csrc = os.path.join(ROOT, "paper_2006_16438_b200", "csrc")
    for f in os.listdir(csrc):
        txt = open(os.path.join(csrc, f)).read()
        assert "getenv" not in txt, f
