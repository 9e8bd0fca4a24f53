"""Seeded synthetic inputs for the FDiRW hot path — shared by the oracle tests,
the CUDA-path tests and bench.py.  Holds NONE of the method's arithmetic
(no stencil, no kernels, no superposition): only geometry masks, initial
concentration fields and the parameter presets of BASELINE.json's configs.

Geometry recipe (the paper's particles come from phase-field
modelling, Fig.1 caption / ref 20, which we cannot reproduce):
  * porous particle: a solid ball of radius r_p at the grid centre minus a
    union of pore spheres (centres uniform in the ball, radii uniform in a
    range) until the target porosity 1 − N_solid/N_ball is reached (P:241-249
    Fig.13: R25/R50/R75 particles; SPEC S:50-58 pore model);
  * porous waste-form block: the whole grid solid minus pores until the liquid
    fraction reaches the target (BASELINE configs[1]);
  * liquid not face-connected to the grid boundary is relabelled solid
    (SPEC S:53, S:77 trapped-cavity policy);
  * mask uint8 [nz][ny][nx], x fastest, 1 = fast phase (liquid), 0 = slow (solid).
Initial concentration "paper": c_L⁰ = 2.12e-3 in liquid, c_S⁰ = 1e-6 in solid
(Table 1); "random": U[0,1) from seed+100.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# Table 1: Δh = 10e-9 m, Δt = 500 µs, Δt_fd = 0.5 µs, D_S = 1e-17, D_L = 1e-14 m²/s,
# A_S/RT = A_L/RT = 2e3.  Effective diffusivities D·A/RT (reading A6).
TABLE1 = dict(dh=10e-9, dt=500e-6, dt_fd=0.5e-6, D_S=1.0e-17, D_L=1.0e-14, A_S_RT=2e3, A_L_RT=2e3,
              c_S0=1.0e-6, c_L0=2.12e-3)
D_FAST_SI = TABLE1["D_L"] * TABLE1["A_L_RT"]  # 2e-11 m²/s
D_SLOW_SI = TABLE1["D_S"] * TABLE1["A_S_RT"]  # 2e-14 m²/s


def _carve_sphere(solid: np.ndarray, c, r: float) -> int:
    """Set voxels whose centre lies within distance r of c to liquid; return #solid voxels removed."""
    nz, ny, nx = solid.shape
    lo = [max(0, int(np.floor(c[i] - r))) for i in range(3)]
    hi = [min(s, int(np.ceil(c[i] + r)) + 1) for i, s in enumerate((nx, ny, nz))]
    if hi[0] <= lo[0] or hi[1] <= lo[1] or hi[2] <= lo[2]:
        return 0
    z, y, x = np.ogrid[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
    inside = (x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2 <= r * r
    sub = solid[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
    removed = int(np.count_nonzero(sub & inside))
    sub[inside] = False
    return removed


def _relabel_trapped(liquid: np.ndarray) -> np.ndarray:
    """Liquid components (6-connectivity) that do not touch the grid boundary become solid."""
    from scipy import ndimage

    lab, n = ndimage.label(liquid)
    if n == 0:
        return liquid
    b = np.zeros(n + 1, bool)
    for sl in (lab[0], lab[-1], lab[:, 0], lab[:, -1], lab[:, :, 0], lab[:, :, -1]):
        b[np.unique(sl)] = True
    b[0] = False
    return b[lab]


def porous_particle(shape, r_p: float, pore_r=(2.0, 4.0), porosity: float = 0.3, seed: int = 0,
                    n_pores: int | None = None, center=None) -> np.ndarray:
    """Ball of radius r_p (solid) minus pores; returns uint8 mask, 1 = liquid."""
    if np.isscalar(shape):
        shape = (int(shape),) * 3
    nz, ny, nx = shape
    rng = np.random.Generator(np.random.PCG64(seed))
    c0 = center if center is not None else ((nx - 1) / 2.0, (ny - 1) / 2.0, (nz - 1) / 2.0)
    z, y, x = np.ogrid[0:nz, 0:ny, 0:nx]
    solid = (x - c0[0]) ** 2 + (y - c0[1]) ** 2 + (z - c0[2]) ** 2 <= r_p * r_p
    n_ball = int(np.count_nonzero(solid))
    n_solid = n_ball
    k = 0
    while True:
        if n_pores is not None:
            if k >= n_pores:
                break
        elif n_ball == 0 or 1.0 - n_solid / n_ball >= porosity:
            break
        # centre uniform in the ball (rejection from the cube), radius uniform in range
        while True:
            u = rng.uniform(-1.0, 1.0, 3)
            if u @ u <= 1.0:
                break
        r = rng.uniform(pore_r[0], pore_r[1])
        n_solid -= _carve_sphere(solid, (c0[0] + r_p * u[0], c0[1] + r_p * u[1], c0[2] + r_p * u[2]), r)
        k += 1
    liquid = _relabel_trapped(~solid)
    return liquid.astype(np.uint8)


def porous_block(shape, pore_r=(2.0, 4.0), porosity: float = 0.45, seed: int = 0) -> np.ndarray:
    """Whole-grid solid block minus overlapping pores until liquid fraction ≥ porosity."""
    if np.isscalar(shape):
        shape = (int(shape),) * 3
    nz, ny, nx = shape
    rng = np.random.Generator(np.random.PCG64(seed))
    solid = np.ones(shape, bool)
    n = solid.size
    n_solid = n
    while 1.0 - n_solid / n < porosity:
        c = (rng.uniform(0, nx), rng.uniform(0, ny), rng.uniform(0, nz))
        r = rng.uniform(pore_r[0], pore_r[1])
        n_solid -= _carve_sphere(solid, c, r)
    liquid = _relabel_trapped(~solid)
    return liquid.astype(np.uint8)


def tiled_particles(n_tile: int = 192, tiles=(2, 2, 2), r_p: float = 50, porosity: float = 0.3,
                    seeds=range(3, 11)) -> np.ndarray:
    """Multiple-particle system: tiles of independent porous particles."""
    tz, ty, tx = tiles
    out = np.empty((tz * n_tile, ty * n_tile, tx * n_tile), np.uint8)
    seeds = list(seeds)
    i = 0
    for a in range(tz):
        for b in range(ty):
            for c in range(tx):
                out[a * n_tile:(a + 1) * n_tile, b * n_tile:(b + 1) * n_tile, c * n_tile:(c + 1) * n_tile] = \
                    porous_particle(n_tile, r_p, porosity=porosity, seed=seeds[i % len(seeds)])
                i += 1
    return out


def near_field(mask: np.ndarray, r_p: float, margin: float = 5.0, center=None) -> np.ndarray:
    """Near-field liquid: liquid voxels whose centre lies within r_p + margin·Δh of
    the particle centre (Euclidean, boundary inclusive).  uint8 region."""
    nz, ny, nx = mask.shape
    c0 = center if center is not None else ((nx - 1) / 2.0, (ny - 1) / 2.0, (nz - 1) / 2.0)
    z, y, x = np.ogrid[0:nz, 0:ny, 0:nx]
    r = r_p + margin
    inside = (x - c0[0]) ** 2 + (y - c0[1]) ** 2 + (z - c0[2]) ** 2 <= r * r
    return ((mask == 1) & inside).astype(np.uint8)


def with_far_field(mask: np.ndarray, r_p: float, margin: float = 5.0, center=None) -> np.ndarray:
    """NEXT row N2 layout: liquid beyond r_p + margin·Δh of the particle centre becomes
    the far-field reservoir (label 2); the near field (solid + liquid within) keeps 0/1."""
    nf = near_field(mask, r_p, margin, center)
    out = mask.copy()
    out[(mask == 1) & (nf == 0)] = 2
    return out


def random_two_phase(shape, p_fast: float = 0.6, seed: int = 0) -> np.ndarray:
    """i.i.d. Bernoulli phases — a stress input for small parity cases (not a paper shape)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return (rng.random(shape) < p_fast).astype(np.uint8)


def initial_c(mask: np.ndarray, kind: str = "random", seed: int = 0) -> np.ndarray:
    """fp32 initial concentration [nz][ny][nx]."""
    if kind == "paper":
        return np.where(mask == 1, np.float32(TABLE1["c_L0"]), np.float32(TABLE1["c_S0"])).astype(np.float32)
    if kind == "random":
        rng = np.random.Generator(np.random.PCG64(seed + 100))
        return rng.random(mask.shape, dtype=np.float32)
    raise ValueError(kind)


@dataclass
class Config:
    """One BASELINE.json config: geometry recipe + the paper's problem parameters."""
    name: str
    shape: tuple
    R: int
    dh: float
    D_fast: float
    D_slow: float
    dt: float
    weights: str
    n_fd: int = 0
    geometry: dict = field(default_factory=dict)
    v_far: float = 0.0    # N2: far-field reservoir volume in voxels (0 = closed domain)
    c_far0: float = 0.0   # N2: initial far-field concentration

    @property
    def K(self) -> int:
        return (2 * self.R + 1) ** 3

    def mask(self) -> np.ndarray:
        g = dict(self.geometry)
        kind = g.pop("kind")
        far_margin = g.pop("far_margin", None)
        if kind == "particle":
            m = porous_particle(self.shape, **g)
            return with_far_field(m, g["r_p"], far_margin) if far_margin is not None else m
        if kind == "block":
            return porous_block(self.shape, **g)
        if kind == "tiled":
            return tiled_particles(**g)
        if kind == "random":
            return random_two_phase(self.shape, **g)
        raise ValueError(kind)


def lattice(n_fd: int):
    """Lattice units (dh = 1, D_fast = 1): Δt = λ*·n_fd with λ* = 0.1 → derived n_fd = n_fd."""
    return dict(dh=1.0, D_fast=1.0, dt=0.1 * n_fd)


def config(name: str, n_fd: int | None = None, weights: str | None = None) -> Config:
    """BASELINE.json configs[0..4] (cfg1..cfg5)."""
    if name == "cfg1":   # 16³ two-phase porous grid, D ratio 1e3, R2, fp32, 10 steps
        n = 1000 if n_fd is None else n_fd
        c = Config("cfg1", (16, 16, 16), 2, D_slow=1e-3, weights="fp32",
                   geometry=dict(kind="particle", r_p=5, pore_r=(1.0, 2.0), n_pores=4, seed=1), **lattice(n))
    elif name == "cfg2":  # 64³ random porous waste-form block, D ratio 1e5, R4, fp32 vs bf16
        n = 1000 if n_fd is None else n_fd
        c = Config("cfg2", (64, 64, 64), 4, D_slow=1e-5, weights="bf16",
                   geometry=dict(kind="block", pore_r=(2.0, 4.0), porosity=0.45, seed=2), **lattice(n))
    elif name == "cfg3":  # 192³ paper medium model (R50 particle), Table 1 SI parameters, R5, bf16
        c = Config("cfg3", (192, 192, 192), 5, dh=TABLE1["dh"], D_fast=D_FAST_SI, D_slow=D_SLOW_SI,
                   dt=TABLE1["dt"], weights="bf16",
                   geometry=dict(kind="particle", r_p=50, pore_r=(2.0, 4.0), porosity=0.3, seed=3))
    elif name == "cfg4":  # 384³ = 2×2×2 R50 particles, D ratio 1e3, R5, bf16, z-slabs
        c = Config("cfg4", (384, 384, 384), 5, dh=TABLE1["dh"], D_fast=D_FAST_SI, D_slow=D_SLOW_SI,
                   dt=TABLE1["dt"], weights="bf16",
                   geometry=dict(kind="tiled", n_tile=192, tiles=(2, 2, 2), r_p=50, porosity=0.3,
                                 seeds=tuple(range(3, 11))))
    elif name == "cfg5":  # cfg3 geometry, D ratio 1e8, R8 — kernel-generation-dominated
        c = Config("cfg5", (192, 192, 192), 8, dh=TABLE1["dh"], D_fast=D_FAST_SI, D_slow=D_FAST_SI * 1e-8,
                   dt=TABLE1["dt"], weights="bf16",
                   geometry=dict(kind="particle", r_p=50, pore_r=(2.0, 4.0), porosity=0.3, seed=3))
    elif name == "cfg3o":  # NEXT row N2: the paper's open R50 model — near field r_p+5Δh inside a
        # grid that just encloses it, far-field reservoir V_L^far = 1.80e-10 mL (Table 1) = 1.8e8 Δh³
        c = Config("cfg3o", (120, 120, 120), 5, dh=TABLE1["dh"], D_fast=D_FAST_SI, D_slow=D_SLOW_SI,
                   dt=TABLE1["dt"], weights="bf16",
                   geometry=dict(kind="particle", r_p=50, pore_r=(2.0, 4.0), porosity=0.3, seed=3, far_margin=5.0),
                   v_far=1.80e-16 / TABLE1["dh"] ** 3, c_far0=TABLE1["c_L0"])
    else:
        raise ValueError(name)
    if n_fd is not None and name in ("cfg3", "cfg4", "cfg5", "cfg3o"):
        c.n_fd = n_fd
    if weights is not None:
        c.weights = weights
    return c
