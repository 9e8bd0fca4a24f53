"""ORACLE for NEXT row N2 — open domain with a far-field reservoir (Eq.7,
P:99-107 Eqs.8-9, Eq.14).  TEST INFRASTRUCTURE ONLY (same rules as oracle/__init__.py).

Phase codes of the mask: 0 slow (solid), 1 fast (near-field liquid), 2 far-field liquid.
The far field is a uniform reservoir c_far of volume V_far (voxel units).

  kernels      W_s from the window FD with far-field cells held at 0 (oracle_kernel):
               the response to c(t0) alone (Eq.8 first term); Σ_o W_s(o) < 1 when the
               window touches the far field — the rest flows into the reservoir;
  p_BC         Eq.8's boundary column, read as  p_BC(x) = 1 − Σ_s W_s(x − s)  (reading
               A26): the response to c_far = 1 held with c(t0) = 0 — for the whole-grid
               FD this IS 1 − row sum (linearity + a uniform field being stationary),
               pinned below against the held-Dirichlet FD where the windows are exact;
  step         c(t+Δt) = p c(t) + p_BC c_far(t)                                  (Eq.8)
  far update   c_far(t+Δt) = (Σc_{S+L}(t0) − Σ c_near(t+Δt) − Σ c_S(t+Δt)) / V_far  (Eq.7)
"""
from __future__ import annotations

import numpy as np

from . import Problem, build_kernels, clip_box, quantize, step_box, step_scatter


def nonfar(pb: Problem) -> np.ndarray:
    return (pb.mask != 2).astype(np.float64)


def p_bc_full(pb: Problem, W: np.ndarray) -> np.ndarray:
    """p_BC on the whole grid from whole-grid kernels W (fp64 or the O5-decoded ones)."""
    nz, ny, nx = pb.shape
    box = (0, nx, 0, ny, 0, nz)
    return (1.0 - step_scatter(pb, W, box, nonfar(pb), box)) * nonfar(pb)


def p_bc_reservoir(pb: Problem) -> np.ndarray:
    """p_BC by the reservoir's own held-Dirichlet FD (the alternative reading of A26):
    the response, after n_fd whole-grid substeps from a zero field, to the far field held at 1 —
    the fine-grid analogue of the paper's P_BC column (Eq.10 with the boundary source).
    Equal to p_bc_full where the windows are exact; ≥ 0 and 0 beyond the reservoir's reach
    everywhere."""
    from . import derive, fd_whole_grid

    zero = np.zeros(pb.shape, np.float64)
    return fd_whole_grid(pb, zero, derive(pb).n_fd, c_far=1.0) * nonfar(pb)


def step_full(pb: Problem, W: np.ndarray, C: np.ndarray, c_far: float, pbc: np.ndarray) -> np.ndarray:
    """Eq.8 on the whole grid (far-field voxels carry 0: their value is the scalar c_far)."""
    nz, ny, nx = pb.shape
    box = (0, nx, 0, ny, 0, nz)
    Cn = np.asarray(C, np.float64) * nonfar(pb)
    return (step_scatter(pb, W, box, Cn, box) + pbc * c_far) * nonfar(pb)


def far_update(M0: float, C_new: np.ndarray, V_far: float) -> float:
    """Eq.7: the reservoir takes whatever mass the near field + solid do not hold."""
    return (M0 - float(np.sum(C_new, dtype=np.float64))) / V_far


def run_full(pb: Problem, C0: np.ndarray, c_far0: float, V_far: float, steps: int, fmt: str | None = None):
    """`steps` FDiRW steps with the reservoir; returns (C, c_far, M0)."""
    W = build_kernels(pb)
    if fmt is not None:
        W = quantize(pb, W, fmt)
    pbc = p_bc_full(pb, W)
    C = np.asarray(C0, np.float64) * nonfar(pb)
    M0 = float(C.sum()) + c_far0 * V_far
    c_far = c_far0
    for _ in range(steps):
        C = step_full(pb, W, C, c_far, pbc)
        c_far = far_update(M0, C, V_far)
    return C, c_far, M0


def step_box_far(pb: Problem, C: np.ndarray, c_far: float, tbox, fmt: str | None = None) -> np.ndarray:
    """Eq.8 for the targets of tbox only (sampled parity at full size)."""
    tbox = clip_box(pb, tbox)
    sl = (slice(tbox[4], tbox[5]), slice(tbox[2], tbox[3]), slice(tbox[0], tbox[1]))
    nf = nonfar(pb)
    part = step_box(pb, np.asarray(C, np.float64) * nf, tbox, fmt=fmt)
    ones = step_box(pb, nf, tbox, fmt=fmt)
    return (part + (1.0 - ones) * c_far) * nf[sl]
