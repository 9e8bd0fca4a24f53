"""Shared test helpers: build oracle problems and library params from one config."""
import numpy as np

import fdirw_inputs as fi


def oracle_problem(cfg: fi.Config, mask=None, n_fd=None):
    import oracle

    return oracle.Problem(mask=cfg.mask() if mask is None else mask, dh=cfg.dh, D_fast=cfg.D_fast,
                          D_slow=cfg.D_slow, dt=cfg.dt, R=cfg.R, n_fd=cfg.n_fd if n_fd is None else n_fd)


def lib_params(cfg: fi.Config, weights=None, flags=0, v_far=None):
    import paper_2408_11376_b200 as fd

    nz, ny, nx = cfg.shape
    return fd.Params(nx=nx, ny=ny, nz=nz, dh=cfg.dh, D_fast=cfg.D_fast, D_slow=cfg.D_slow, dt=cfg.dt,
                     radius=cfg.R, n_fd=cfg.n_fd, weights=weights or cfg.weights, flags=flags,
                     v_far=cfg.v_far if v_far is None else v_far)


def small_cfg(shape, R, n_fd, D_slow=1e-3, weights="fp32", mask=None, seed=0, kind="random"):
    """Lattice-unit config for ad-hoc parity cases."""
    c = fi.Config("adhoc", tuple(shape), R, weights=weights, D_slow=D_slow, **fi.lattice(n_fd),
                  geometry=dict(kind="random", p_fast=0.6, seed=seed))
    return c


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))
