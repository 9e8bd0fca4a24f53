"""CPU fp64 ORACLE for the FDiRW hot path (arXiv 2408.11376) — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2408_11376_b200``) never imports it and shares no code with it.

This module is argument marshalling (ctypes + numpy) around ``fdirw_oracle.c``;
every piece of the method's arithmetic lives in that C file, each function
citing the PAPER.md passage it follows.  See DESIGN.md §4 for the pins.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fdirw_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

FMT = {"fp32": 0, "fp16": 1, "bf16": 2}


def build(force: bool = False) -> str:
    """Compile fdirw_oracle.c with gcc (-O2, strict IEEE: no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(
            ["gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
             "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Params(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("dh", ctypes.c_double), ("D_fast", ctypes.c_double), ("D_slow", ctypes.c_double),
                ("dt", ctypes.c_double), ("R", ctypes.c_int32), ("n_fd", ctypes.c_int32)]


class _Derived(ctypes.Structure):
    _fields_ = [("n_fd", ctypes.c_int32), ("dt_fd", ctypes.c_double), ("lam_ff", ctypes.c_double),
                ("lam_fs", ctypes.c_double), ("lam_ss", ctypes.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P, D = ctypes.POINTER(_Params), ctypes.POINTER(_Derived)
        vp = ctypes.c_void_p
        L.oracle_derive.argtypes = [P, D]
        L.oracle_derive.restype = ctypes.c_int
        L.oracle_kernel.argtypes = [P, D, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp]
        L.oracle_build_kernels.argtypes = [P, D, vp, vp, vp]
        L.oracle_step_scatter.argtypes = [P, vp, vp, vp, vp, vp]
        L.oracle_step_scatter_omp.argtypes = [P, vp, vp, vp, vp, vp]
        L.oracle_quantize.argtypes = [P, vp, ctypes.c_long, ctypes.c_int, ctypes.c_int, vp, vp]
        L.oracle_fd_whole_grid.argtypes = [P, D, vp, vp, ctypes.c_int, ctypes.c_double, vp]
        L.oracle_f32_to_f16.argtypes = [ctypes.c_float]
        L.oracle_f32_to_f16.restype = ctypes.c_uint16
        L.oracle_f32_to_bf16.argtypes = [ctypes.c_float]
        L.oracle_f32_to_bf16.restype = ctypes.c_uint16
        L.oracle_f16_to_f64.argtypes = [ctypes.c_uint16]
        L.oracle_f16_to_f64.restype = ctypes.c_double
        L.oracle_bf16_to_f64.argtypes = [ctypes.c_uint16]
        L.oracle_bf16_to_f64.restype = ctypes.c_double
        L.oracle_round_fmt.argtypes = [ctypes.c_double, ctypes.c_int]
        L.oracle_round_fmt.restype = ctypes.c_double
        L.oracle_rel_l2.argtypes = [vp, vp, ctypes.c_long]
        L.oracle_rel_l2.restype = ctypes.c_double
        _lib = L
    return _lib


@dataclass
class Problem:
    """The paper's problem statement (Table 1) plus north_star's window radius."""
    mask: np.ndarray          # uint8 [nz][ny][nx], 1 = fast (liquid)
    dh: float
    D_fast: float             # effective diffusivity D·A/RT (A6)
    D_slow: float
    dt: float
    R: int
    n_fd: int = 0             # 0 = derive (a1)

    def __post_init__(self):
        self.mask = np.ascontiguousarray(self.mask, dtype=np.uint8)
        if self.mask.ndim != 3:
            raise ValueError("mask must be [nz][ny][nx]")

    @property
    def shape(self):
        return self.mask.shape

    @property
    def K(self):
        return (2 * self.R + 1) ** 3

    def _params(self) -> _Params:
        nz, ny, nx = self.mask.shape
        return _Params(nx, ny, nz, self.dh, self.D_fast, self.D_slow, self.dt, self.R, self.n_fd)


@dataclass
class Derived:
    n_fd: int
    dt_fd: float
    lam_ff: float
    lam_fs: float
    lam_ss: float


def derive(pb: Problem) -> Derived:
    p, d = pb._params(), _Derived()
    rc = lib().oracle_derive(ctypes.byref(p), ctypes.byref(d))
    if rc == 1:
        raise ValueError("invalid parameters")
    if rc == 2:
        raise ValueError("unstable: lambda_max > 1/6")
    return Derived(d.n_fd, d.dt_fd, d.lam_ff, d.lam_fs, d.lam_ss)


def _pd(pb: Problem):
    p, d = pb._params(), _Derived()
    rc = lib().oracle_derive(ctypes.byref(p), ctypes.byref(d))
    if rc != 0:
        raise ValueError("oracle_derive failed (%d)" % rc)
    return p, d


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def kernel(pb: Problem, s) -> np.ndarray:
    """W_s as an fp64 array [2R+1][2R+1][2R+1] indexed [oz+R][oy+R][ox+R]; s = (x, y, z)."""
    p, d = _pd(pb)
    L = 2 * pb.R + 1
    W = np.zeros(L ** 3, np.float64)
    lib().oracle_kernel(ctypes.byref(p), ctypes.byref(d), _ptr(pb.mask), int(s[0]), int(s[1]), int(s[2]), _ptr(W))
    return W.reshape(L, L, L)


def clip_box(pb: Problem, box):
    nz, ny, nx = pb.shape
    x0, x1, y0, y1, z0, z1 = box
    return (max(0, x0), min(nx, x1), max(0, y0), min(ny, y1), max(0, z0), min(nz, z1))


def build_kernels(pb: Problem, box=None) -> np.ndarray:
    """Kernels of all sources in box=(x0,x1,y0,y1,z0,z1) → fp64 [bz][by][bx][K]."""
    nz, ny, nx = pb.shape
    box = clip_box(pb, box or (0, nx, 0, ny, 0, nz))
    p, d = _pd(pb)
    bx, by, bz = box[1] - box[0], box[3] - box[2], box[5] - box[4]
    W = np.zeros((bz, by, bx, pb.K), np.float64)
    b = np.array(box, np.int32)
    lib().oracle_build_kernels(ctypes.byref(p), ctypes.byref(d), _ptr(pb.mask), _ptr(b), _ptr(W))
    return W


def quantize(pb: Problem, W: np.ndarray, fmt: str, mass_fix: bool = True, box=None) -> np.ndarray:
    """O5: the stored operator (decoded to fp64), diagonal in the centre slot.  With a far
    field (mask 2, N2) the kernels of windows that touch it keep their own mass M = ΣW;
    `box` = the source box of W (default: whole grid) locates those windows."""
    W = np.ascontiguousarray(W, np.float64)
    Wq = np.empty_like(W)
    ow = None
    if (pb.mask == 2).any():
        ow = np.ascontiguousarray(open_windows(pb, box).ravel().astype(np.uint8))
    lib().oracle_quantize(ctypes.byref(pb._params()), _ptr(W), W.size // pb.K, FMT[fmt], int(mass_fix), _ptr(Wq),
                          _ptr(ow) if ow is not None else None)
    return Wq


def open_windows(pb: Problem, box=None) -> np.ndarray:
    """bool [bz][by][bx]: does the source's window contain a far-field cell (mask 2)?"""
    nz, ny, nx = pb.shape
    box = clip_box(pb, box or (0, nx, 0, ny, 0, nz))
    R = pb.R
    far = np.pad(pb.mask == 2, R)
    out = np.zeros((box[5] - box[4], box[3] - box[2], box[1] - box[0]), bool)
    for oz in range(2 * R + 1):
        for oy in range(2 * R + 1):
            for ox in range(2 * R + 1):
                out |= far[box[4] + oz:box[5] + oz, box[2] + oy:box[3] + oy, box[0] + ox:box[1] + ox]
    return out


def step_scatter(pb: Problem, W: np.ndarray, sbox, C_old: np.ndarray, tbox, threads: bool = False) -> np.ndarray:
    """O4: targets in tbox from the sources in sbox (W from build_kernels(sbox)).  threads=True:
    the OpenMP form (target planes split between threads, same per-target order, same bits)."""
    C_old = np.ascontiguousarray(C_old, np.float64)
    assert C_old.shape == pb.shape
    sbox = clip_box(pb, sbox)
    tbox = clip_box(pb, tbox)
    W = np.ascontiguousarray(W, np.float64)
    assert W.shape[:3] == (sbox[5] - sbox[4], sbox[3] - sbox[2], sbox[1] - sbox[0])
    out = np.zeros((tbox[5] - tbox[4], tbox[3] - tbox[2], tbox[1] - tbox[0]), np.float64)
    sb, tb = np.array(sbox, np.int32), np.array(tbox, np.int32)
    fn = lib().oracle_step_scatter_omp if threads else lib().oracle_step_scatter
    fn(ctypes.byref(pb._params()), _ptr(W), _ptr(sb), _ptr(C_old), _ptr(tb), _ptr(out))
    return out


def step_box(pb: Problem, C_old: np.ndarray, tbox, fmt: str | None = None, mass_fix: bool = True,
             W: np.ndarray | None = None):
    """One FDiRW step for targets in tbox: build the kernels of every source that
    reaches tbox (tbox expanded by R), optionally quantise (O5), scatter (O4)."""
    R = pb.R
    sbox = clip_box(pb, (tbox[0] - R, tbox[1] + R, tbox[2] - R, tbox[3] + R, tbox[4] - R, tbox[5] + R))
    if W is None:
        W = build_kernels(pb, sbox)
    if fmt is not None:
        W = quantize(pb, W, fmt, mass_fix, box=sbox)
    return step_scatter(pb, W, sbox, C_old, tbox)


def step_full(pb: Problem, C_old: np.ndarray, steps: int = 1, fmt: str | None = None, mass_fix: bool = True,
              threads: bool = False, W: np.ndarray | None = None, checkpoints=()):
    """`steps` FDiRW steps on the whole grid (small grids only: N·K fp64 kernels).  threads:
    the OpenMP scatter (same bits); W: the kernels, if already built (fmt / mass_fix are then
    ignored); checkpoints: step counts at which to also return the field → (C, {k: C_k})."""
    nz, ny, nx = pb.shape
    box = (0, nx, 0, ny, 0, nz)
    if W is None:
        W = build_kernels(pb, box)
        if fmt is not None:
            W = quantize(pb, W, fmt, mass_fix)
    C = np.asarray(C_old, np.float64)
    snap = {}
    for k in range(1, steps + 1):
        C = step_scatter(pb, W, box, C, box, threads=threads)
        if k in checkpoints:
            snap[k] = C.copy()
    return (C, snap) if checkpoints else C


def fd_whole_grid(pb: Problem, C0: np.ndarray, nsub: int, c_far: float = 0.0) -> np.ndarray:
    """O6: nsub whole-grid explicit FD substeps (closed domain; far-field cells, mask 2,
    held at c_far)."""
    p, d = _pd(pb)
    C0 = np.ascontiguousarray(C0, np.float64)
    out = np.empty_like(C0)
    lib().oracle_fd_whole_grid(ctypes.byref(p), ctypes.byref(d), _ptr(pb.mask), _ptr(C0), int(nsub), float(c_far),
                               _ptr(out))
    return out


def f32_to_f16_bits(x: float) -> int:
    return int(lib().oracle_f32_to_f16(float(np.float32(x))))


def f32_to_bf16_bits(x: float) -> int:
    return int(lib().oracle_f32_to_bf16(float(np.float32(x))))


def round_fmt(x: float, fmt: str) -> float:
    return float(lib().oracle_round_fmt(float(x), FMT[fmt]))


def rel_l2(g: np.ndarray, o: np.ndarray) -> float:
    g = np.ascontiguousarray(g, np.float64).ravel()
    o = np.ascontiguousarray(o, np.float64).ravel()
    return float(lib().oracle_rel_l2(_ptr(g), _ptr(o), g.size))
