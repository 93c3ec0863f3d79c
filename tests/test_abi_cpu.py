"""The C-ABI library loads and exports every entry point declared in include/pdilqr.h; host-side
validation works without a GPU (no compute calls here)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "pdilqr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pdilqr_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def P():
    import paper_2506_07823_b200 as P
    P.lib()
    return P


def test_header_declares_the_boundary():
    names = declared_functions()
    for f in ("pdilqr_create", "pdilqr_destroy", "pdilqr_workspace_bytes", "pdilqr_solve_lq",
              "pdilqr_linearize", "pdilqr_step"):
        assert f in names


def test_library_exports_every_declared_symbol(P):
    L = C.CDLL(P.LIB_PATH)
    for f in declared_functions():
        assert hasattr(L, f), f
    assert L.pdilqr_abi_version() == P.pdilqr.ABI_VERSION == 2


def test_library_is_sm100a(P):
    """The fatbin carries sm_100a SASS (checked with cuobjdump when available)."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def cfg(P, **kw):
    c = P.pdilqr.Config(N=50, n=12, m=12, batch=4096, dtype=0, model=1, n_alpha=10, armijo_c1=1e-4,
                        theta_max=0.0, leaf_chunk=0, export_policy=0)
    c.srbd.mass = 15.0; c.srbd.dt = 0.02; c.srbd.barrier_mu = 0.1; c.srbd.barrier_delta = 1.0
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def test_workspace_bytes_and_validation(P):
    L = P.lib()
    nb = C.c_size_t()
    assert L.pdilqr_workspace_bytes(C.byref(cfg(P)), C.byref(nb)) == 0
    assert nb.value > 100 * 2 ** 20          # B=4096, N=50 SRBD: > 100 MB of scan workspace
    nb2 = C.c_size_t()
    assert L.pdilqr_workspace_bytes(C.byref(cfg(P, leaf_chunk=1)), C.byref(nb2)) == 0
    assert nb2.value > nb.value               # the tree needs slot storage
    assert L.pdilqr_workspace_bytes(C.byref(cfg(P, n=13)), C.byref(nb)) == 2       # SRBD needs n = m = 12
    assert b"SRBD" in L.pdilqr_last_error()
    assert L.pdilqr_workspace_bytes(C.byref(cfg(P, model=0, n=300, m=4)), C.byref(nb)) == 5   # n > 256
    assert L.pdilqr_workspace_bytes(C.byref(cfg(P, model=0, n=74, m=32, batch=8, N=100)), C.byref(nb)) == 0
    assert L.pdilqr_workspace_bytes(C.byref(cfg(P, n_alpha=40)), C.byref(nb)) == 1
    assert L.pdilqr_workspace_bytes(C.byref(cfg(P, batch=0)), C.byref(nb)) == 2
    assert L.pdilqr_workspace_bytes(None, C.byref(nb)) == 1


def test_no_cpu_fallback_without_gpu(P):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    L = P.lib()
    h = C.c_void_p()
    buf = (C.c_ubyte * 1024)()
    st = L.pdilqr_create(C.byref(cfg(P, batch=1, N=2)), 0, C.cast(buf, C.c_void_p), 1024, C.byref(h))
    assert st in (3, 4)                       # workspace / CUDA error: the library never computes on the host
    with pytest.raises(Exception):
        P.PdIlqr(N=2, n=4, m=2, batch=1)
