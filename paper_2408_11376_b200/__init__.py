"""paper_2408_11376_b200 — B200-native FDiRW hot path (arXiv 2408.11376).

Thin ctypes binding of ``include/fdirw.h`` (libfdirw.so, built in-tree for
sm_100a).  Argument marshalling only: every step of the method runs in the
library's CUDA kernels.  torch supplies device memory (tensors), streams and
the torch.distributed bootstrap of the NCCL id; nothing else.

There is no CPU fallback: importing this package raises if libfdirw.so is
missing, and every call raises ``FdirwError`` on a non-OK status.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libfdirw.so")

if not os.path.exists(_LIB_PATH):
    raise ImportError(
        "libfdirw.so not found at %s — build it with `python paper_2408_11376_b200/build.py` "
        "(or __graft_entry__.build()); there is no fallback path" % _LIB_PATH)

_lib = ctypes.CDLL(_LIB_PATH)

FDIRW_OK, E_INVALID, E_UNSTABLE, E_OOM, E_CUDA, E_NCCL, E_ALIAS, E_STATE = range(8)
STATUS_NAMES = ["OK", "E_INVALID", "E_UNSTABLE", "E_OOM", "E_CUDA", "E_NCCL", "E_ALIAS", "E_STATE"]
WEIGHTS = {"fp32": 0, "fp16": 1, "bf16": 2, "mx8": 3}
F_NO_MASS_FIX = 1
F_NO_DEDUP = 2
F_DEDUP_STORAGE = 4  # NEXT row N4: uniform chunks read shared class kernels (fewer HBM bytes)
F_KGEN_FP64 = 8  # kgen in fp64, the oracle's operation order (reading A22, debugging)
F_SYMMETRIC_RULE = 16  # exact regime only: gather weights = own kernel reflected (reading A24)
F_KGEN_DIRECT = 32  # kgen runs the n_fd substeps literally instead of the Chebyshev recurrence (reading A30)
F_NO_BULK_STREAM = 64  # superposition: per-thread weight loads instead of TMA-staged rows (same bits)
F_KGEN_COLUMNS = 128  # R = 5 kgen: one window column per thread (round-1 kernel) instead of pairs (A/B)
F_PBC_RESERVOIR = 256  # N2: p_BC by the reservoir's held-Dirichlet FD instead of 1 − row sum (A26 alternative)

EXPORTS = ["fdirw_make_plan", "fdirw_nccl_unique_id", "fdirw_build_kernels", "fdirw_step", "fdirw_run", "fdirw_mass",
           "fdirw_query", "fdirw_destroy", "fdirw_last_error", "fdirw_debug_upload_weights",
           "fdirw_export_kernels", "fdirw_step_virtual", "fdirw_coarse_build", "fdirw_coarse_step",
           "fdirw_coarse_run", "fdirw_coarse_query", "fdirw_coarse_export", "fdirw_coarse_destroy",
           "fdirw_far_init", "fdirw_far_init_virtual", "fdirw_far_get", "fdirw_absorb_run",
           "fdirw_set_precision_mode", "fdirw_coarse_far_init", "fdirw_coarse_far_get",
           "fdirw_coarse_export_pbc", "fdirw_p2p_export", "fdirw_p2p_attach", "fdirw_p2p_attach_local",
           "fdirw_p2p_check", "fdirw_read_ceiling", "fdirw_mass_local", "fdirw_profile_phases",
           "fdirw_comm_init", "fdirw_step_host", "fdirw_debug_stage_canary",
           "fdirw_build_id"]
TRANSPORTS = {"nccl": 0, "p2p": 1}
P2P_BLOB_BYTES = 256


class fdirw_params(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("dh", ctypes.c_double), ("D_fast", ctypes.c_double), ("D_slow", ctypes.c_double),
                ("dt", ctypes.c_double), ("radius", ctypes.c_int32), ("n_fd", ctypes.c_int32),
                ("weights", ctypes.c_int32), ("flags", ctypes.c_uint32), ("v_far", ctypes.c_double)]


class fdirw_dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("z_begin", ctypes.c_int32),
                ("z_end", ctypes.c_int32), ("device", ctypes.c_int32), ("nccl_id", ctypes.c_void_p),
                ("transport", ctypes.c_int32)]


class fdirw_info(ctypes.Structure):
    _fields_ = [("n_fd", ctypes.c_int32), ("K", ctypes.c_int32), ("z_begin", ctypes.c_int32),
                ("z_end", ctypes.c_int32), ("dt_fd", ctypes.c_double), ("lambda_fast", ctypes.c_double),
                ("lambda_fs", ctypes.c_double), ("lambda_slow", ctypes.c_double),
                ("weight_bytes", ctypes.c_uint64), ("state_bytes", ctypes.c_uint64),
                ("bytes_per_voxel_update", ctypes.c_uint64), ("voxels", ctypes.c_uint64),
                ("tile_chunks", ctypes.c_int32), ("n_tiles", ctypes.c_int32),
                ("kgen_sources", ctypes.c_uint64), ("kgen_windows", ctypes.c_uint64),
                ("chunks", ctypes.c_uint64), ("uniform_chunks", ctypes.c_uint64), ("uniform_classes", ctypes.c_int32),
                ("kgen_steps", ctypes.c_int32), ("kgen_kernel_ms", ctypes.c_double)]


class fdirw_plan(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "z_begin", "z_end", "src_z_begin", "src_z_end", "mask_z_begin", "mask_z_end", "tile_chunks",
        "tiles_per_plane", "n_tiles", "interior_tile_begin", "interior_tile_end", "peer_lo", "peer_hi", "n_fd")] + \
        [(n, ctypes.c_int64) for n in ("padded_x", "padded_y", "padded_z", "pad_x0", "halo_elems", "send_lo",
                                       "recv_lo", "send_hi", "recv_hi")] + \
        [("weight_bytes", ctypes.c_uint64), ("state_bytes", ctypes.c_uint64), ("kgen_steps", ctypes.c_int32)]


class fdirw_coarse_info(ctypes.Structure):
    _fields_ = [("n_fd", ctypes.c_int32), ("block", ctypes.c_int32), ("n_groups", ctypes.c_int64),
                ("n_region", ctypes.c_int64), ("p_bytes", ctypes.c_uint64), ("flops_per_step", ctypes.c_uint64),
                ("fd_passes", ctypes.c_int32)]


_vp = ctypes.c_void_p
_st = ctypes.c_int
_lib.fdirw_make_plan.argtypes = [ctypes.POINTER(fdirw_params), ctypes.POINTER(fdirw_dist), ctypes.POINTER(fdirw_plan)]
_lib.fdirw_make_plan.restype = _st
_lib.fdirw_nccl_unique_id.argtypes = [_vp]
_lib.fdirw_nccl_unique_id.restype = _st
_lib.fdirw_build_kernels.argtypes = [ctypes.POINTER(fdirw_params), _vp, ctypes.POINTER(fdirw_dist), _vp,
                                     ctypes.POINTER(_vp)]
_lib.fdirw_build_kernels.restype = _st
_lib.fdirw_step.argtypes = [_vp, _vp, _vp, _vp]
_lib.fdirw_step.restype = _st
_lib.fdirw_run.argtypes = [_vp, _vp, ctypes.c_int32, _vp]
_lib.fdirw_run.restype = _st
_lib.fdirw_mass.argtypes = [_vp, _vp, ctypes.POINTER(ctypes.c_double), _vp]
_lib.fdirw_mass.restype = _st
_lib.fdirw_build_id.argtypes = []
_lib.fdirw_build_id.restype = ctypes.c_char_p
_lib.fdirw_debug_stage_canary.argtypes = [_vp, ctypes.c_int32, ctypes.POINTER(ctypes.c_uint64),
                                          ctypes.POINTER(ctypes.c_uint64)]
_lib.fdirw_debug_stage_canary.restype = _st
_lib.fdirw_step_host.argtypes = [_vp, _vp, _vp, _vp]
_lib.fdirw_step_host.restype = _st
_lib.fdirw_comm_init.argtypes = [_vp, _vp]
_lib.fdirw_comm_init.restype = _st
_lib.fdirw_mass_local.argtypes = [_vp, _vp, ctypes.POINTER(ctypes.c_double), _vp]
_lib.fdirw_mass_local.restype = _st
_lib.fdirw_profile_phases.argtypes = [_vp, _vp, ctypes.c_int32, _vp, ctypes.POINTER(ctypes.c_double)]
_lib.fdirw_profile_phases.restype = _st
_lib.fdirw_read_ceiling.argtypes = [_vp, ctypes.c_int32, _vp, ctypes.POINTER(ctypes.c_double)]
_lib.fdirw_read_ceiling.restype = _st
_lib.fdirw_query.argtypes = [_vp, ctypes.POINTER(fdirw_info)]
_lib.fdirw_query.restype = _st
_lib.fdirw_destroy.argtypes = [_vp]
_lib.fdirw_destroy.restype = None
_lib.fdirw_last_error.argtypes = []
_lib.fdirw_last_error.restype = ctypes.c_char_p
_lib.fdirw_debug_upload_weights.argtypes = [_vp, _vp]
_lib.fdirw_debug_upload_weights.restype = _st
_lib.fdirw_export_kernels.argtypes = [_vp, _vp, _vp]
_lib.fdirw_export_kernels.restype = _st
_lib.fdirw_step_virtual.argtypes = [ctypes.POINTER(_vp), ctypes.c_int32, ctypes.POINTER(_vp),
                                    ctypes.POINTER(_vp), _vp]
_lib.fdirw_step_virtual.restype = _st
_lib.fdirw_coarse_build.argtypes = [ctypes.POINTER(fdirw_params), _vp, ctypes.c_int32, _vp, ctypes.POINTER(_vp)]
_lib.fdirw_coarse_build.restype = _st
_lib.fdirw_coarse_step.argtypes = [_vp, _vp, _vp, _vp]
_lib.fdirw_coarse_step.restype = _st
_lib.fdirw_coarse_run.argtypes = [_vp, _vp, ctypes.c_int32, _vp]
_lib.fdirw_coarse_run.restype = _st
_lib.fdirw_coarse_query.argtypes = [_vp, ctypes.POINTER(fdirw_coarse_info)]
_lib.fdirw_coarse_query.restype = _st
_lib.fdirw_coarse_export.argtypes = [_vp, _vp, _vp]
_lib.fdirw_coarse_export.restype = _st
_lib.fdirw_coarse_far_init.argtypes = [_vp, _vp, ctypes.c_double, ctypes.POINTER(ctypes.c_double), _vp]
_lib.fdirw_coarse_far_init.restype = _st
_lib.fdirw_coarse_far_get.argtypes = [_vp, ctypes.POINTER(ctypes.c_double), _vp]
_lib.fdirw_coarse_far_get.restype = _st
_lib.fdirw_coarse_export_pbc.argtypes = [_vp, _vp]
_lib.fdirw_coarse_export_pbc.restype = _st
_lib.fdirw_coarse_destroy.argtypes = [_vp]
_lib.fdirw_coarse_destroy.restype = None
_lib.fdirw_far_init.argtypes = [_vp, _vp, ctypes.c_double, ctypes.POINTER(ctypes.c_double), _vp]
_lib.fdirw_far_init.restype = _st
_lib.fdirw_far_init_virtual.argtypes = [ctypes.POINTER(_vp), ctypes.c_int32, ctypes.POINTER(_vp), ctypes.c_double,
                                        ctypes.POINTER(ctypes.c_double), _vp]
_lib.fdirw_far_init_virtual.restype = _st
_lib.fdirw_far_get.argtypes = [_vp, ctypes.POINTER(ctypes.c_double), _vp]
_lib.fdirw_far_get.restype = _st
_lib.fdirw_p2p_export.argtypes = [_vp, _vp]
_lib.fdirw_p2p_export.restype = _st
_lib.fdirw_p2p_attach.argtypes = [_vp, _vp, _vp]
_lib.fdirw_p2p_attach.restype = _st
_lib.fdirw_p2p_attach_local.argtypes = [ctypes.POINTER(_vp), ctypes.c_int32]
_lib.fdirw_p2p_attach_local.restype = _st
_lib.fdirw_p2p_check.argtypes = [_vp, ctypes.POINTER(ctypes.c_int32), _vp]
_lib.fdirw_p2p_check.restype = _st


class fdirw_absorb_params(ctypes.Structure):
    _fields_ = [("D_S", ctypes.c_double), ("k", ctypes.c_double), ("c_S_eq", ctypes.c_double),
                ("c_L_eq", ctypes.c_double)]


_lib.fdirw_absorb_run.argtypes = [_vp, ctypes.POINTER(fdirw_absorb_params), _vp, ctypes.c_int32, _vp, _vp]
_lib.fdirw_absorb_run.restype = _st
_lib.fdirw_set_precision_mode.argtypes = [_vp, ctypes.c_int32]
_lib.fdirw_set_precision_mode.restype = _st
PRECISION_MODES = {"default": 0, "fp32": 1, "mixed": 2, "fp16": 3}


class FdirwError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        super().__init__("%s: %s" % (STATUS_NAMES[status] if 0 <= status < 8 else status, msg))


def build_id() -> str:
    """sha256 of the sources the loaded library was compiled from (fdirw_build_id)."""
    return _lib.fdirw_build_id().decode()


def last_error() -> str:
    return _lib.fdirw_last_error().decode()


def _check(rc: int):
    if rc != FDIRW_OK:
        raise FdirwError(rc, last_error())


def _stream(stream):
    if stream is None:
        import torch

        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _dptr(t):
    """Device pointer of a contiguous fp32 CUDA tensor."""
    if not (t.is_cuda and t.is_contiguous() and str(t.dtype) == "torch.float32"):
        raise ValueError("expected a contiguous float32 CUDA tensor")
    return ctypes.c_void_p(t.data_ptr())


def _hptr(t):
    """Host pointer of a contiguous fp32 CPU tensor (pinned for asynchronous copies) or ndarray."""
    if isinstance(t, np.ndarray):
        if not (t.flags["C_CONTIGUOUS"] and t.dtype == np.float32):
            raise ValueError("expected a contiguous float32 array")
        return ctypes.c_void_p(t.ctypes.data)
    if t.is_cuda or not t.is_contiguous() or str(t.dtype) != "torch.float32":
        raise ValueError("expected a contiguous float32 CPU tensor")
    return ctypes.c_void_p(t.data_ptr())


@dataclass
class Params:
    nx: int
    ny: int
    nz: int
    dh: float
    D_fast: float
    D_slow: float
    dt: float
    radius: int
    n_fd: int = 0
    weights: str = "bf16"
    flags: int = 0
    v_far: float = 0.0  # N2: far-field reservoir volume (voxels); 0 = closed domain

    def c(self) -> fdirw_params:
        return fdirw_params(self.nx, self.ny, self.nz, self.dh, self.D_fast, self.D_slow, self.dt, self.radius,
                            self.n_fd, WEIGHTS[self.weights], self.flags, self.v_far)


class Context:
    """Owns an fdirw_ctx*; call destroy() (or use as a context manager)."""

    def __init__(self, handle: int, params: Params):
        self.handle = ctypes.c_void_p(handle)
        self.params = params

    def __enter__(self):
        return self

    def __exit__(self, *a):
        destroy(self)

    @property
    def info(self):
        return query(self)


def make_plan(params: Params, rank: int = 0, world: int = 1, z_begin: int | None = None,
              z_end: int | None = None) -> dict:
    """fdirw_make_plan: the host-side slab / halo / tile plan of one rank (no GPU needed)."""
    p = params.c()
    d = fdirw_dist(rank, world, 0 if z_begin is None else z_begin, params.nz if z_end is None else z_end, 0, None)
    pl = fdirw_plan()
    _check(_lib.fdirw_make_plan(ctypes.byref(p), ctypes.byref(d), ctypes.byref(pl)))
    return {f: getattr(pl, f) for f, _ in fdirw_plan._fields_}


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.fdirw_nccl_unique_id(buf))
    return buf.raw


def build_kernels(params: Params, phase: np.ndarray, rank: int = 0, world: int = 1, z_begin: int | None = None,
                  z_end: int | None = None, device: int | None = None, nccl_id: bytes | None = None,
                  stream=None, transport: str = "nccl") -> Context:
    """fdirw_build_kernels: phase = WHOLE-grid uint8 mask [nz][ny][nx] (host), 1 = fast.
    transport: "nccl" (halo via NCCL send/recv; nccl_id None + world > 1 = virtual ranks) or
    "p2p" (halo planes stored into the neighbours' memory by the superposition; attach with
    p2p_attach / p2p_attach_local before stepping)."""
    phase = np.ascontiguousarray(phase, dtype=np.uint8)
    if phase.shape != (params.nz, params.ny, params.nx):
        raise ValueError("phase shape %s != (nz, ny, nx)" % (phase.shape,))
    p = params.c()
    dist = None
    idbuf = None
    if world > 1 or z_begin is not None or device is not None:
        if device is None:
            import torch

            device = torch.cuda.current_device()
        if nccl_id is not None:
            idbuf = ctypes.create_string_buffer(nccl_id, 128)
        dist = fdirw_dist(rank, world, 0 if z_begin is None else z_begin, params.nz if z_end is None else z_end,
                          device, ctypes.cast(idbuf, ctypes.c_void_p) if idbuf is not None else None,
                          TRANSPORTS[transport])
    h = ctypes.c_void_p()
    _check(_lib.fdirw_build_kernels(ctypes.byref(p), phase.ctypes.data_as(ctypes.c_void_p),
                                    ctypes.byref(dist) if dist is not None else None, _stream(stream),
                                    ctypes.byref(h)))
    return Context(h.value, params)


def p2p_export(ctx: Context) -> bytes:
    """fdirw_p2p_export → the 256-byte blob (geometry + CUDA IPC handles) to all-gather."""
    buf = ctypes.create_string_buffer(P2P_BLOB_BYTES)
    _check(_lib.fdirw_p2p_export(ctx.handle, buf))
    return buf.raw


def p2p_attach(ctx: Context, lo_blob: bytes | None, hi_blob: bytes | None):
    lo = ctypes.create_string_buffer(lo_blob, P2P_BLOB_BYTES) if lo_blob is not None else None
    hi = ctypes.create_string_buffer(hi_blob, P2P_BLOB_BYTES) if hi_blob is not None else None
    _check(_lib.fdirw_p2p_attach(ctx.handle, lo, hi))


def p2p_attach_local(ctxs):
    H = (_vp * len(ctxs))(*[c.handle.value for c in ctxs])
    _check(_lib.fdirw_p2p_attach_local(H, len(ctxs)))


def p2p_check(ctx: Context, stream=None) -> bool:
    """True if a neighbour wait timed out (results invalid)."""
    t = ctypes.c_int32(0)
    _check(_lib.fdirw_p2p_check(ctx.handle, ctypes.byref(t), _stream(stream)))
    return bool(t.value)


def step(ctx: Context, c_in, c_out, stream=None):
    _check(_lib.fdirw_step(ctx.handle, _dptr(c_in), _dptr(c_out), _stream(stream)))


def step_host(ctx: Context, c_in_host, c_out_host, stream=None):
    """fdirw_step_host: host (pinned CPU tensor) slab in → step on the device → host slab out;
    asynchronous on the stream."""
    _check(_lib.fdirw_step_host(ctx.handle, _hptr(c_in_host), _hptr(c_out_host), _stream(stream)))


def run(ctx: Context, c, n_steps: int, stream=None):
    _check(_lib.fdirw_run(ctx.handle, _dptr(c), int(n_steps), _stream(stream)))


def mass(ctx: Context, c, stream=None) -> float:
    out = ctypes.c_double()
    _check(_lib.fdirw_mass(ctx.handle, _dptr(c), ctypes.byref(out), _stream(stream)))
    return out.value


def comm_init(ctx: Context, nccl_id: bytes):
    """fdirw_comm_init: the NCCL communicator of a P2P context (collective; for fdirw_mass)."""
    idbuf = ctypes.create_string_buffer(nccl_id, 128)
    _check(_lib.fdirw_comm_init(ctx.handle, idbuf))


def mass_local(ctx: Context, c, stream=None) -> float:
    """Σ c over this rank's slab (fdirw_mass_local)."""
    out = ctypes.c_double()
    _check(_lib.fdirw_mass_local(ctx.handle, _dptr(c), ctypes.byref(out), _stream(stream)))
    return out.value


PHASES = ("halo", "interior", "boundary", "tail", "step")


def profile_phases(ctx: Context, c, n_steps: int, stream=None) -> dict:
    """fdirw_profile_phases: mean device ms per step of each phase (halo, interior, boundary,
    tail, whole step), n_steps eager steps on c in place."""
    out = (ctypes.c_double * 5)()
    _check(_lib.fdirw_profile_phases(ctx.handle, _dptr(c), int(n_steps), _stream(stream), out))
    return dict(zip(PHASES, list(out)))


def read_ceiling(ctx: Context, reps: int = 5, stream=None) -> float:
    """fdirw_read_ceiling: GB/s of a pure read stream over the context's weights (best of reps)."""
    out = ctypes.c_double()
    _check(_lib.fdirw_read_ceiling(ctx.handle, int(reps), _stream(stream), ctypes.byref(out)))
    return out.value


def query(ctx: Context) -> dict:
    info = fdirw_info()
    _check(_lib.fdirw_query(ctx.handle, ctypes.byref(info)))
    return {f: getattr(info, f) for f, _ in fdirw_info._fields_}


def destroy(ctx: Context):
    if ctx.handle and ctx.handle.value:
        _lib.fdirw_destroy(ctx.handle)
        ctx.handle = ctypes.c_void_p()


def debug_upload_weights(ctx: Context, kernels: np.ndarray):
    k = np.ascontiguousarray(kernels, dtype=np.float64)
    _check(_lib.fdirw_debug_upload_weights(ctx.handle, k.ctypes.data_as(ctypes.c_void_p)))


def debug_stage_canary(ctx: Context, enable: bool = True):
    """fdirw_debug_stage_canary → (16-byte words checked, mismatches)."""
    a, b = ctypes.c_uint64(), ctypes.c_uint64()
    _check(_lib.fdirw_debug_stage_canary(ctx.handle, int(enable), ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def export_kernels(ctx: Context, box) -> np.ndarray:
    """Stored kernels of the sources in box = (x0,x1,y0,y1,z0,z1) → fp64 [bz][by][bx][K]."""
    b = np.array(box, np.int32)
    K = (2 * ctx.params.radius + 1) ** 3
    out = np.zeros((b[5] - b[4], b[3] - b[2], b[1] - b[0], K), np.float64)
    _check(_lib.fdirw_export_kernels(ctx.handle, b.ctypes.data_as(ctypes.c_void_p),
                                     out.ctypes.data_as(ctypes.c_void_p)))
    return out


def step_virtual(ctxs, c_in, c_out, stream=None):
    n = len(ctxs)
    H = (_vp * n)(*[c.handle.value for c in ctxs])
    I = (_vp * n)(*[_dptr(t).value for t in c_in])
    O = (_vp * n)(*[_dptr(t).value for t in c_out])
    _check(_lib.fdirw_step_virtual(H, n, I, O, _stream(stream)))


def slabs(nz: int, world: int):
    """Equal z-slabs [r·nz/P, (r+1)·nz/P)."""
    return [(r * nz // world, (r + 1) * nz // world) for r in range(world)]


# ---- NEXT row N1: coarse-mesh FDiRW (Eqs.10-15) ------------------------------
class Coarse:
    """Owns an fdirw_coarse*."""

    def __init__(self, handle: int, params: Params, shape):
        self.handle = ctypes.c_void_p(handle)
        self.params = params
        self.shape = shape

    def __enter__(self):
        return self

    def __exit__(self, *a):
        coarse_destroy(self)

    @property
    def info(self):
        return coarse_query(self)


def coarse_build(params: Params, region: np.ndarray, block: int = 5, stream=None) -> Coarse:
    """fdirw_coarse_build: region = uint8 [nz][ny][nx] (host), 1 = Ω_L, 2 = far field (v_far > 0)."""
    region = np.ascontiguousarray(region, dtype=np.uint8)
    if region.shape != (params.nz, params.ny, params.nx):
        raise ValueError("region shape %s != (nz, ny, nx)" % (region.shape,))
    p = params.c()
    h = ctypes.c_void_p()
    _check(_lib.fdirw_coarse_build(ctypes.byref(p), region.ctypes.data_as(ctypes.c_void_p), int(block),
                                   _stream(stream), ctypes.byref(h)))
    return Coarse(h.value, params, region.shape)


def coarse_step(ctx: Coarse, c_in, c_out, stream=None):
    _check(_lib.fdirw_coarse_step(ctx.handle, _dptr(c_in), _dptr(c_out), _stream(stream)))


def coarse_run(ctx: Coarse, c, n_steps: int, stream=None):
    _check(_lib.fdirw_coarse_run(ctx.handle, _dptr(c), int(n_steps), _stream(stream)))


def coarse_query(ctx: Coarse) -> dict:
    info = fdirw_coarse_info()
    _check(_lib.fdirw_coarse_query(ctx.handle, ctypes.byref(info)))
    return {f: getattr(info, f) for f, _ in fdirw_coarse_info._fields_}


def coarse_export(ctx: Coarse):
    """(P decoded fp64 [N][N] with the fp32 diagonal, group_of int32 [nz][ny][nx])."""
    N = coarse_query(ctx)["n_groups"]
    P = np.zeros((N, N), np.float64)
    g = np.zeros(ctx.shape, np.int32)
    _check(_lib.fdirw_coarse_export(ctx.handle, P.ctypes.data_as(ctypes.c_void_p), g.ctypes.data_as(ctypes.c_void_p)))
    return P, g


def coarse_export_pbc(ctx: Coarse):
    """P_BC as stored (fp32 → fp64) [N] (N2 far-field contexts only)."""
    pbc = np.zeros(coarse_query(ctx)["n_groups"], np.float64)
    _check(_lib.fdirw_coarse_export_pbc(ctx.handle, pbc.ctypes.data_as(ctypes.c_void_p)))
    return pbc


def coarse_far_init(ctx: Coarse, c, c_far0: float, stream=None) -> float:
    """fdirw_coarse_far_init → K0 = Σ_{Ω_L} c + c_far0·v_far (Eq.7 invariant)."""
    m = ctypes.c_double(0.0)
    _check(_lib.fdirw_coarse_far_init(ctx.handle, _dptr(c), float(c_far0), ctypes.byref(m), _stream(stream)))
    return m.value


def coarse_far_get(ctx: Coarse, stream=None) -> float:
    v = ctypes.c_double(0.0)
    _check(_lib.fdirw_coarse_far_get(ctx.handle, ctypes.byref(v), _stream(stream)))
    return v.value


def coarse_destroy(ctx: Coarse):
    if ctx.handle and ctx.handle.value:
        _lib.fdirw_coarse_destroy(ctx.handle)
        ctx.handle = ctypes.c_void_p()


# ---- NEXT row N2: far-field reservoir (Eq.7) ---------------------------------------
def far_init(ctx: Context, c, c_far0: float, stream=None) -> float:
    """fdirw_far_init: sets c_far(t0) and returns M0 = Σ c + c_far0·v_far (Eq.7's Σc_{S+L}(t0))."""
    m0 = ctypes.c_double()
    _check(_lib.fdirw_far_init(ctx.handle, _dptr(c), float(c_far0), ctypes.byref(m0), _stream(stream)))
    return m0.value


def far_init_virtual(ctxs, cs, c_far0: float, stream=None) -> float:
    n = len(ctxs)
    H = (_vp * n)(*[c.handle.value for c in ctxs])
    C = (_vp * n)(*[_dptr(t).value for t in cs])
    m0 = ctypes.c_double()
    _check(_lib.fdirw_far_init_virtual(H, n, C, float(c_far0), ctypes.byref(m0), _stream(stream)))
    return m0.value


def far_get(ctx: Context, stream=None) -> float:
    v = ctypes.c_double()
    _check(_lib.fdirw_far_get(ctx.handle, ctypes.byref(v), _stream(stream)))
    return v.value


# ---- NEXT row N3: integrated absorption loop + §3.3 precision modes ------------------------
def absorb_run(ctx: Context, c, n_steps: int, D_S: float, k: float, c_S_eq: float, c_L_eq: float,
               stream=None) -> np.ndarray:
    """fdirw_absorb_run → kinetics [n_steps][4] = (Q_S, Q_L, c_far, c̄_S)."""
    ap = fdirw_absorb_params(D_S, k, c_S_eq, c_L_eq)
    kin = np.zeros((max(int(n_steps), 1), 4), np.float64)
    _check(_lib.fdirw_absorb_run(ctx.handle, ctypes.byref(ap), _dptr(c), int(n_steps),
                                 kin.ctypes.data_as(ctypes.c_void_p), _stream(stream)))
    return kin[:n_steps]


def set_precision_mode(ctx: Context, mode):
    """'default' | 'fp32' | 'mixed' | 'fp16' (or 0..3), see include/fdirw.h."""
    _check(_lib.fdirw_set_precision_mode(ctx.handle, PRECISION_MODES.get(mode, mode)))
