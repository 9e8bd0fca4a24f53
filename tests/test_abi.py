"""CPU checks of the C-ABI library: it builds, loads without a GPU, exports every
symbol include/fdirw.h declares, and validates arguments before touching CUDA."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def fd():
    import __graft_entry__

    __graft_entry__.build()
    import paper_2408_11376_b200 as fd

    return fd


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "fdirw.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fdirw_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(fd):
    syms = declared_symbols()
    assert len(syms) >= 11
    out = subprocess.check_output(["nm", "-D", "--defined-only", fd._LIB_PATH]).decode()
    exported = set(re.findall(r" T (fdirw_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert set(fd.EXPORTS) == set(syms)


def test_no_oracle_in_product():
    """The product path never imports, links or calls the oracle."""
    pkg = os.path.join(ROOT, "paper_2408_11376_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "liboracle" not in txt, f
    out = subprocess.check_output(["ldd", os.path.join(pkg, "libfdirw.so")]).decode()
    assert "oracle" not in out


def _params(fd, **kw):
    d = dict(nx=8, ny=8, nz=8, dh=1.0, D_fast=1.0, D_slow=1e-3, dt=0.5, radius=2, n_fd=0, weights="bf16")
    d.update(kw)
    return fd.Params(**d)


@pytest.mark.parametrize("kw,status", [
    (dict(nx=0), 1), (dict(radius=0), 1), (dict(radius=9), 1), (dict(D_fast=0.0), 1),
    (dict(D_slow=-1.0), 1), (dict(dt=0.0), 1), (dict(dh=-1.0), 1), (dict(n_fd=-1), 1),
    (dict(n_fd=1, dt=1.0), 2),  # λ = 1 > 1/6
])
def test_validation_without_gpu(fd, kw, status):
    raw = _params(fd, **kw).c()
    m = np.ones(512, np.uint8)
    h = ctypes.c_void_p()
    rc = fd._lib.fdirw_build_kernels(ctypes.byref(raw), m.ctypes.data_as(ctypes.c_void_p), None, None,
                                     ctypes.byref(h))
    assert rc == status
    assert fd.last_error()
    assert not h.value


def test_bad_slab_and_format(fd):
    p = _params(fd)
    raw = p.c()
    raw.weights = 7
    h = ctypes.c_void_p()
    m = np.ones((8, 8, 8), np.uint8)
    rc = fd._lib.fdirw_build_kernels(ctypes.byref(raw), m.ctypes.data_as(ctypes.c_void_p), None, None,
                                     ctypes.byref(h))
    assert rc == fd.E_INVALID
    with pytest.raises(fd.FdirwError) as e:  # slab thinner than R
        fd.build_kernels(p, m, rank=0, world=4, z_begin=0, z_end=1, device=0, stream=0)
    assert e.value.status == fd.E_INVALID
    with pytest.raises(fd.FdirwError):  # rank 0 must start at z = 0
        fd.build_kernels(p, m, rank=0, world=2, z_begin=2, z_end=5, device=0, stream=0)
    assert fd._lib.fdirw_step(None, None, None, None) == fd.E_INVALID
    fd._lib.fdirw_destroy(None)  # no-op


def test_slabs_tile(fd):
    for nz in (12, 37, 192, 384):
        for w in (1, 2, 3, 8):
            sl = fd.slabs(nz, w)
            assert sl[0][0] == 0 and sl[-1][1] == nz
            assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))


def test_loaded_library_matches_sources(fd):
    """The loaded libfdirw.so was compiled from exactly the sources in the tree (content hash of
    sources, headers, flags and nvcc version, compiled in as fdirw_build_id)."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("fdirw_build", os.path.join(ROOT, "paper_2408_11376_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    assert fd.build_id() == b.source_sha()


def test_null_arguments_rejected_without_gpu(fd):
    """Every entry point added in round 2 validates its arguments before touching CUDA."""
    L = fd._lib
    d = ctypes.c_double()
    u, v = ctypes.c_uint64(), ctypes.c_uint64()
    ms = (ctypes.c_double * 5)()
    assert L.fdirw_step_host(None, None, None, None) == fd.E_INVALID
    assert L.fdirw_comm_init(None, None) == fd.E_INVALID
    assert L.fdirw_mass_local(None, None, ctypes.byref(d), None) == fd.E_INVALID
    assert L.fdirw_profile_phases(None, None, 4, None, ms) == fd.E_INVALID
    assert L.fdirw_debug_stage_canary(None, 1, ctypes.byref(u), ctypes.byref(v)) == fd.E_INVALID
    assert fd.last_error()


def test_slab_index_range_checked(fd):
    """slabs whose mask planes exceed 2^31 voxels are rejected (the window dedup and
    the N3 loop index a slab's voxels with 32-bit ints)."""
    p = _params(fd, nx=2048, ny=2048, nz=600, radius=1)
    plan = fd.fdirw_plan()
    rc = fd._lib.fdirw_make_plan(ctypes.byref(p.c()), None, ctypes.byref(plan))
    assert rc == fd.E_INVALID and "2^31" in fd.last_error()
    ok = _params(fd, nx=2048, ny=2048, nz=400, radius=1)
    assert fd._lib.fdirw_make_plan(ctypes.byref(ok.c()), None, ctypes.byref(plan)) == fd.FDIRW_OK
