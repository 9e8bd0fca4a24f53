"""Diagnostic: per-weight error of the stored fp32 kernels vs the oracle's fp64 kernels
(cfg1 at n_fd = 1000), for the Chebyshev default and the direct substeps."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import fdirw_inputs as fi  # noqa: E402
import oracle  # noqa: E402
import paper_2408_11376_b200 as fd  # noqa: E402
from _util import lib_params, oracle_problem  # noqa: E402

oracle.build()
for name, kw in (("cfg1", {}), ("cfg2s", None)):
    if kw is None:
        from _util import small_cfg
        cfg = small_cfg((14, 13, 15), 4, 1000, D_slow=1e-5, weights="fp32")
        mask = fi.random_two_phase((14, 13, 15), 0.6, seed=4)
    else:
        cfg = fi.config("cfg1", n_fd=1000, weights="fp32")
        mask = cfg.mask()
    pb = oracle_problem(cfg, mask)
    Wo = oracle.build_kernels(pb)
    off = np.ones(pb.K, bool)
    off[pb.K // 2] = False
    nz, ny, nx = cfg.shape
    for flags in (0, fd.F_KGEN_DIRECT):
        ctx = fd.build_kernels(lib_params(cfg, flags=flags), mask)
        W = fd.export_kernels(ctx, (0, nx, 0, ny, 0, nz))
        fd.destroy(ctx)
        e = np.abs(W[..., off] - Wo[..., off])
        r = e / np.maximum(Wo[..., off], 1e-30)
        big = Wo[..., off] > 1e-3 * Wo.max()
        print("%s flags=%d: max abs %.3e (max W %.3e)  max rel (W>1e-3 max) %.3e  p99.9 rel %.3e  relL2 %.3e" % (
            name, flags, e.max(), Wo[..., off].max(), r[big].max(), np.quantile(r[big], 0.999),
            np.linalg.norm(e) / np.linalg.norm(Wo[..., off])))

# open windows (N2 far field): kernels keep M_s < 1, the rest went to the reservoir
from _util import small_cfg  # noqa: E402

shape = (14, 13, 15)
m = fi.porous_particle(shape, min(shape) / 2 - 4, pore_r=(1.0, 2.0), porosity=0.3, seed=4)
mask = fi.with_far_field(m, min(shape) / 2 - 4, margin=2.0)
cfg = small_cfg(shape, 3, 1000, D_slow=1e-3, weights="fp32")
pb = oracle_problem(cfg, mask)
Wo = oracle.build_kernels(pb)
off = np.ones(pb.K, bool)
off[pb.K // 2] = False
nz, ny, nx = shape
openw = Wo.sum(-1) < 0.999
for flags in (0, fd.F_KGEN_DIRECT):
    ctx = fd.build_kernels(lib_params(cfg, flags=flags, v_far=1000.0), mask)
    W = fd.export_kernels(ctx, (0, nx, 0, ny, 0, nz))
    fd.destroy(ctx)
    e = np.abs(W[..., off] - Wo[..., off])
    rows = openw & (mask != 2)
    mo, mg = Wo[rows].sum(-1), W[rows].sum(-1)
    print("open flags=%d: windows %d, mass left min %.3e; max |dW| %.3e (max W %.3e); kernel-mass rel err max %.3e" % (
        flags, rows.sum(), mo.min(), e[rows].max(), Wo[rows][:, off].max(), (np.abs(mg - mo) / mo).max()))
