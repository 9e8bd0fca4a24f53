"""ORACLE for NEXT row N3 — the integrated absorption loop (P:42 components 1-4, P:50-78
Eqs.1-7, Fig.4) and the precision modes of §3.3 (Figs.8-10).
TEST INFRASTRUCTURE ONLY (same rules as oracle/__init__.py).

Per macro step Δt (operator split; SPEC S:225, S:464 — the paper's flowchart, Fig.4, is not
reproduced in the text):
  (1) fast diffusion in the near-field liquid: FDiRW, Eq.8, with the far-field reservoir
      (N2) and the solid impermeable (D_slow = 0 in the liquid FD: all
      solid–liquid exchange happens in (3));
  (2) slow diffusion in the solid: explicit FD, D_S·A_S/RT, solid–solid faces only,
      n_s substeps with λ_S ≤ 0.1 (Table 1: exactly one substep);
  (3) interface absorption, pseudo-second order (Eqs.4-6): for every solid voxel s and
      every near-field liquid face neighbour l (pre-step values, Jacobi):
          q_sl = k · f_L(c_l) · f_S(c_s) · Δt,
          f_L = 0 if c_l ≤ c_L^eq else (c_l − c_L^eq)/c_L^eq,   f_S = max((c_S^eq − c_s)/c_S^eq, 0)
      mass moves from l to s; a liquid voxel never gives more than c_l − c_L^eq (the
      transfers it feeds are scaled down together; "transfer clamped to available
      mass"; reading A29);
  (4) far field, Eq.7: c_far = (Σc_{S+L}(t0) − Σc_near − Σc_S)/V_far;
  (5) kinetics: Q_S = Σ_solid c, Q_L = Σ_near-liquid c, c̄_S = Q_S/(N_S·c_S^eq) (Fig.6, Fig.10).

FDiRW precision modes (§3.3; Figs.8-10):
  "fp64"    weights, products and sums in fp64
  "fp32"    weights, concentrations, products and the running sum in fp32
  "mixed"   the paper's: P stored in fp16, C converted to fp16, each product rounded to
            fp16, accumulated in fp32
  "fp16"    as "mixed" with the running sum in fp16 too
Products are summed over sources in ascending order.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import Problem, build_kernels, derive, fd_whole_grid, quantize
from . import farfield


@dataclass
class Absorb:
    """Table 1 in effective form."""
    D_L: float        # D_L·A_L/RT
    D_S: float        # D_S·A_S/RT
    dh: float
    dt: float
    k: float          # PSO rate constant [1/s]
    c_S_eq: float
    c_L_eq: float
    V_far: float      # far-field volume in voxels
    R: int


def f_L(c, c_eq):
    """Eq.5."""
    return np.where(c <= c_eq, 0.0, (c - c_eq) / c_eq)


def f_S(c, c_eq):
    """Eq.6, clamped at 0 (no desorption)."""
    return np.maximum((c_eq - c) / c_eq, 0.0)


def rate(c_L, c_S, ab: Absorb):
    """Eq.4: (Ṙ_S, Ṙ_L)."""
    r = ab.k * f_L(c_L, ab.c_L_eq) * f_S(c_S, ab.c_S_eq)
    return r, -r


_DIRS = [(0, 0, -1), (0, 0, 1), (0, -1, 0), (0, 1, 0), (-1, 0, 0), (1, 0, 0)]  # (dz,dy,dx): −x,+x,−y,+y,−z,+z


def _shift(a, d, fill):
    """out[i] = a[i + d] (fill outside the grid)."""
    out = np.full_like(a, fill)
    src = [slice(None)] * 3
    dst = [slice(None)] * 3
    for ax, s in enumerate(d):
        n = a.shape[ax]
        if s > 0:
            src[ax], dst[ax] = slice(s, n), slice(0, n - s)
        elif s < 0:
            src[ax], dst[ax] = slice(0, n + s), slice(-s, n)
    out[tuple(dst)] = a[tuple(src)]
    return out


def react(c: np.ndarray, mask: np.ndarray, ab: Absorb) -> np.ndarray:
    """Component (2) of P:42, Eqs.4-6, one explicit step of length Δt with the clamp (A29)."""
    c = np.asarray(c, np.float64)
    solid, liq = mask == 0, mask == 1
    fS = f_S(c, ab.c_S_eq) * solid
    fL = f_L(c, ab.c_L_eq) * liq
    q = []  # q[f][s]: transfer into solid voxel s from its neighbour in direction f
    for d in _DIRS:
        q.append(ab.k * fS * _shift(fL, d, 0.0) * ab.dt)
    # total requested from each liquid voxel l: Σ over the solid neighbours s of l
    Q = np.zeros_like(c)
    for d, qf in zip(_DIRS, q):
        Q += _shift(qf, tuple(-x for x in d), 0.0)   # q of the solid at l − d, which points at l
    avail = np.maximum(c - ab.c_L_eq, 0.0) * liq
    alpha = np.where(Q > avail, np.divide(avail, Q, out=np.zeros_like(Q), where=Q > 0), 1.0)
    out = c.copy()
    for d, qf in zip(_DIRS, q):
        out += qf * _shift(alpha, d, 0.0)              # solid s gains α_l q_sl
    out -= alpha * Q                                    # liquid l loses α_l Q_l
    return out


def solid_fd(c: np.ndarray, mask: np.ndarray, ab: Absorb) -> np.ndarray:
    """Component (3): explicit FD over the solid only (solid–solid faces)."""
    pb = Problem(mask=(mask == 0).astype(np.uint8), dh=ab.dh, D_fast=ab.D_S, D_slow=0.0, dt=ab.dt, R=1)
    n_s = derive(pb).n_fd
    return fd_whole_grid(pb, c, n_s)


def liquid_problem(mask: np.ndarray, ab: Absorb) -> Problem:
    """FDiRW problem of component (1): fast = near-field liquid, solid impermeable, far = 2."""
    return Problem(mask=mask, dh=ab.dh, D_fast=ab.D_L, D_slow=0.0, dt=ab.dt, R=ab.R)


def _round(x, mode):
    if mode == "fp32":
        return x.astype(np.float32)
    if mode in ("mixed", "fp16"):
        return x.astype(np.float32).astype(np.float16)
    return x


def fdirw_step_mode(pb: Problem, W: np.ndarray, c: np.ndarray, c_far: float, pbc: np.ndarray, mode: str):
    """Eq.8 under one precision mode, gather over sources in ascending order (box = grid)."""
    if mode == "fp64":
        return farfield.step_full(pb, W, c, c_far, pbc)
    nz, ny, nx = pb.shape
    L, R = 2 * pb.R + 1, pb.R
    nf = (pb.mask != 2)
    cs = np.where(nf, np.asarray(c, np.float64), 0.0)
    Wm = _round(W, mode)                             # [z][y][x][K] per-source kernels
    cm = _round(cs, mode)
    acc_t = np.float16 if mode == "fp16" else np.float32
    acc = np.zeros((nz, ny, nx), acc_t)
    pad = ((R, R), (R, R), (R, R))
    Wp = np.pad(Wm, pad + ((0, 0),))
    cp = np.pad(cm, pad)
    # target x receives W_s(x−s) c_s for s = x − o; ascending source order = descending o
    for o in range(L ** 3 - 1, -1, -1):
        oz, oy, ox = o // (L * L) - R, (o // L) % L - R, o % L - R
        sl = (slice(R - oz, R - oz + nz), slice(R - oy, R - oy + ny), slice(R - ox, R - ox + nx))
        w = Wp[sl + (o,)]
        cc = cp[sl]
        if mode == "fp32":
            prod = (w * cc).astype(np.float32)
        else:
            prod = (w * cc).astype(np.float16)         # product rounded to fp16
        acc = (acc + prod.astype(acc_t)).astype(acc_t)
    bc = (_round(pbc, mode).astype(np.float64) * c_far)
    out = acc.astype(np.float64) + bc
    return out * nf


def run(mask: np.ndarray, c0: np.ndarray, c_far0: float, ab: Absorb, steps: int, mode: str = "fp64"):
    """The integrated loop; returns (c, c_far, kinetics list of (Q_S, Q_L, c_far, c̄_S))."""
    pb = liquid_problem(mask, ab)
    W = build_kernels(pb)
    # the paper stores P plainly in the mode's format: no diagonal fix-up here
    Wq = (quantize(pb, W, "fp16", mass_fix=False) if mode in ("mixed", "fp16")
          else (quantize(pb, W, "fp32", mass_fix=False) if mode == "fp32" else W))
    pbc = farfield.p_bc_full(pb, Wq)
    c = np.asarray(c0, np.float64) * (mask != 2)
    M0 = float(c.sum()) + c_far0 * ab.V_far
    c_far = c_far0
    n_s = int((mask == 0).sum())
    kin = []
    for _ in range(steps):
        c = fdirw_step_mode(pb, Wq, c, c_far, pbc, mode)       # (1)
        c = solid_fd(c, mask, ab)                               # (3) slow solid diffusion
        c = react(c, mask, ab)                                  # (2) interface absorption
        c_far = (M0 - float(c.sum())) / ab.V_far                # (4) Eq.7
        QS, QL = float(c[mask == 0].sum()), float(c[mask == 1].sum())
        kin.append((QS, QL, c_far, QS / (n_s * ab.c_S_eq)))
    return c, c_far, kin
