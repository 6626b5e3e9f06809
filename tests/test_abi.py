"""CPU: the C-ABI library builds for sm_100a, loads, and exports exactly the
entry points include/hapt_b200.h declares; the product path refuses to run
without a GPU (no CPU fallback)."""

import os
import re
import subprocess

import pytest
import torch

from conftest import REPO

HEADER = os.path.join(REPO, "include", "hapt_b200.h")


def declared() -> set:
    text = open(HEADER).read()
    return set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(hapt_[a-z0-9_]+)\(", text, re.M))


def test_library_builds_and_exports_header_symbols():
    from paper_2509_24859_b200 import _lib, build

    path = build.build()
    assert os.path.exists(path)
    names = declared()
    assert {"hapt_dp_sweep_batch", "hapt_tables_build", "hapt_sim_1f1b"} <= names
    h = _lib.load(path)
    for n in names:
        assert hasattr(h, n), n
    assert set(_lib.EXPORTED) == names
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (hapt_[a-z0-9_]+)", out))
    assert names <= exported


def test_sass_targets_sm100a():
    from paper_2509_24859_b200 import build

    path = build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    from paper_2509_24859_b200 import _lib
    from paper_2509_24859_b200.cluster import ClusterSpec, DeviceMesh
    from paper_2509_24859_b200.model_graph import uniform_layers
    from paper_2509_24859_b200.profiling import build_store

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.lib()
    with pytest.raises(RuntimeError):
        build_store(uniform_layers(2, 1e12, 1e9, 1e6),
                    ClusterSpec([DeviceMesh("m", 1, 1, 1e12, 1e12, 1e9, 1e9)], cross_bw=1e9))


def test_product_does_not_import_oracle():
    pkg = os.path.join(REPO, "paper_2509_24859_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                text = open(os.path.join(root, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "import meshpipe" not in text and "from meshpipe" not in text, f


def test_trace_entry_points_validate_arguments():
    """The trace-layout K3 entry points reject a missing or misaligned trace
    (argument checks run before any CUDA call, so this runs on CPU)."""
    import ctypes

    from paper_2509_24859_b200 import _lib, build

    h = _lib.load(build.build())
    h.hapt_last_error.restype = ctypes.c_char_p
    one = (ctypes.c_int32 * 4)(0, 1, 1, 1)
    dbl = (ctypes.c_double * 8)()
    off = (ctypes.c_int64 * 2)()
    odd = ctypes.addressof(dbl) + 8  # 8-byte aligned, not 16
    einval = 1
    rc = h.hapt_sim_1f1b_trace(1, one, dbl, dbl, dbl, one, one, dbl, None, off, 4, one, dbl,
                               ctypes.c_size_t(64), None)
    assert rc == einval and b"hapt_sim_1f1b_trace" in h.hapt_last_error()
    rc = h.hapt_sim_1f1b_trace(1, one, dbl, dbl, dbl, one, one, dbl, ctypes.c_void_p(odd), off,
                               4, one, dbl, ctypes.c_size_t(64), None)
    assert rc == einval and b"16-byte" in h.hapt_last_error()
    rc = h.hapt_analyze_1f1b_trace(1, 1, one, dbl, dbl, dbl, one, one, None,
                                   ctypes.c_void_p(odd), off, None, dbl, one, dbl, dbl, None)
    assert rc == einval and b"hapt_analyze_1f1b_trace" in h.hapt_last_error()
