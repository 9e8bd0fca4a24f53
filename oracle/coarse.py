"""ORACLE for NEXT row N1 — coarse-mesh FDiRW (§3.1, Eqs.10-15).
TEST INFRASTRUCTURE ONLY (same rules as oracle/__init__.py).

The paper's own step, written out in its order and notation on the fine grid
of `Problem` (closed domain, reading A3; the far-field term P_BC·c_far is NEXT
row N2):

  region Ω_L   the fast-phase voxels the FDiRW handles (near-field liquid);
  groups I     Ω_L ∩ axis-aligned b×b×b blocks anchored at the origin, empty
               blocks dropped, numbered in block order (z, y, x) — P:113 "N = N_L/125",
               i.e. b = 5 (the paper's coarsening algorithm, ref 12, is unavailable;
               block groups follow SPEC S:259);
  P[:, J]      explicit FD over Ω_L (faces leaving Ω_L carry no flux) from the
               group-uniform source c⁰ = 1 on group J,
               n_fd substeps, then mapped (Eq.11/13)  — computed with
               oracle.fd_whole_grid on the mask Ω_L with D_slow = 0;
  step         'Mapping' C_I = Σ_{i∈I} c_i / N_I         (Eq.13)
               C'_I = Σ_J P_IJ C_J                       (Eq.14, closed domain)
               'Re-mapping' c'_i = C'_I for i ∈ I       (Eq.15); voxels ∉ Ω_L unchanged.

Reduced-precision storage of P ("P is stored in FP16"): off-diagonal
P̃_IJ = RNE_fmt(RNE_fp32(P_IJ)); diagonal fixed in fp32 so every column keeps the
mass it moves: Σ_I N_I P̃_IJ = N_J (the coarse analogue of reading A10).
"""
from __future__ import annotations

import numpy as np

from . import Problem, fd_whole_grid, round_fmt


def groups(region: np.ndarray, b: int = 5):
    """group_of[z, y, x] ∈ {−1, 0..N−1} and N_I (group sizes)."""
    region = np.asarray(region) == 1  # 2 = far-field reservoir (N2), not grouped
    nz, ny, nx = region.shape
    bz, by, bx = -(-nz // b), -(-ny // b), -(-nx // b)
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    block = ((z // b) * by + (y // b)) * bx + (x // b)
    used = np.zeros(bz * by * bx, bool)
    used[block[region]] = True
    ids = np.cumsum(used) - 1
    g = np.where(region, ids[block], -1).astype(np.int32)
    n = int(used.sum())
    sizes = np.bincount(g[region], minlength=n).astype(np.int64)
    return g, sizes


def map_fine_to_coarse(c: np.ndarray, g: np.ndarray, sizes: np.ndarray) -> np.ndarray:
    """Eq.13: C_I = Σ_{i∈I} c_i / N_I (fp64)."""
    m = g >= 0
    return np.bincount(g[m], weights=np.asarray(c, np.float64)[m], minlength=len(sizes)) / sizes


def remap_coarse_to_fine(C: np.ndarray, g: np.ndarray, c: np.ndarray) -> np.ndarray:
    """Eq.15: c_i = C_I for every grouped voxel; other voxels keep their value."""
    out = np.array(c, np.float64, copy=True)
    m = g >= 0
    out[m] = np.asarray(C, np.float64)[g[m]]
    return out


def region_problem(pb: Problem, region: np.ndarray) -> Problem:
    """FD over Ω_L only: Ω_L voxels are the fast phase, everything else impermeable
    (D_slow = 0 ⇒ harmonic-mean faces into it vanish, reading A23); region value 2 marks the
    far-field reservoir, held at c_far by oracle.fd_whole_grid (N2)."""
    return Problem(mask=np.asarray(region, np.uint8), dh=pb.dh, D_fast=pb.D_fast, D_slow=0.0, dt=pb.dt, R=1,
                   n_fd=pb.n_fd if pb.n_fd else 0)


def build_P(pb: Problem, region: np.ndarray, b: int = 5, n_fd: int | None = None):
    """Dense P (N×N, fp64), column J = map(FD^{n_fd}(1_J)) (Eq.10)."""
    import oracle

    g, sizes = groups(region, b)
    rp = region_problem(pb, region)
    n = oracle.derive(pb).n_fd if n_fd is None else n_fd
    N = len(sizes)
    P = np.zeros((N, N))
    for J in range(N):
        c0 = (g == J).astype(np.float64)
        P[:, J] = map_fine_to_coarse(fd_whole_grid(rp, c0, n), g, sizes)
    return P, g, sizes


def build_PBC(pb: Problem, region: np.ndarray, b: int = 5, n_fd: int | None = None) -> np.ndarray:
    """N2 on the coarse mesh: P_BC (Eq.10) = map of the FD over Ω_L from c = 0 with the far
    field held at 1."""
    import oracle

    g, sizes = groups(region, b)
    n = oracle.derive(pb).n_fd if n_fd is None else n_fd
    return map_fine_to_coarse(fd_whole_grid(region_problem(pb, region), np.zeros(region.shape), n, c_far=1.0),
                              g, sizes)


def quantize_P(P: np.ndarray, sizes: np.ndarray, fmt: str) -> np.ndarray:
    """Off-diagonal RNE_fmt(RNE_fp32(P_IJ)); fp32 diagonal keeping each column's mass
    M_J = Σ_I N_I P_IJ (= N_J in a closed domain; less with a far field, N2)."""
    N = P.shape[0]
    Q = np.empty_like(P)
    for I in range(N):
        for J in range(N):
            Q[I, J] = round_fmt(P[I, J], fmt) if I != J else 0.0
    s = sizes.astype(np.float64)
    for J in range(N):
        M = float(np.dot(s, P[:, J]))
        off = float(np.dot(s, Q[:, J]))  # Σ_{I≠J} N_I P̃_IJ (diagonal entry is 0 here)
        Q[J, J] = float(np.float32((M - off) / s[J]))
    return Q


def step(P: np.ndarray, g: np.ndarray, sizes: np.ndarray, c: np.ndarray) -> np.ndarray:
    """One coarse FDiRW step, Eqs.13-15."""
    C = map_fine_to_coarse(c, g, sizes)
    return remap_coarse_to_fine(P @ C, g, c)


def step_far(P: np.ndarray, PBC: np.ndarray, g: np.ndarray, sizes: np.ndarray, c: np.ndarray, c_far: float):
    """Eq.14 with the boundary term: C' = P·C + P_BC·c_far, then Eq.15."""
    C = map_fine_to_coarse(c, g, sizes)
    return remap_coarse_to_fine(P @ C + PBC * c_far, g, c)


def flop_count(N: int, N_L: int) -> int:
    """§4.3: N(N+1) + 2·N_L multiplications per step."""
    return N * (N + 1) + 2 * N_L
