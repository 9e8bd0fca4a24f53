"""Diagnostic (GPU): per-decade relative error of the stored fp32 kernels against the oracle's
fp64 kernels, Chebyshev default (reading A30) vs the literal substeps, plus each kernel's error
normalised by its own largest off-centre weight.  Prints one JSON line per case; the numbers set
the bounds of tests/test_gpu_kgen_tails.py."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import fdirw_inputs as fi  # noqa: E402
import oracle  # noqa: E402
import paper_2408_11376_b200 as fd  # noqa: E402
from _util import lib_params, oracle_problem, small_cfg  # noqa: E402


def cases():
    cfg = fi.config("cfg1", n_fd=1000, weights="fp32")
    yield "cfg1", cfg, cfg.mask()
    yield "r4_ratio1e5", small_cfg((14, 13, 15), 4, 1000, D_slow=1e-5), fi.random_two_phase((14, 13, 15), 0.6, seed=4)
    yield "r5_particle", small_cfg((22, 23, 21), 5, 1000, D_slow=1e-3), fi.porous_particle(
        (22, 23, 21), 7, pore_r=(1.0, 2.0), porosity=0.3, seed=3)


def decade_stats(W, Wo, off):
    out = {}
    g, o = W[..., off].ravel(), Wo[..., off].ravel()
    rel = np.abs(g - o) / np.maximum(o, 1e-300)
    for d in range(0, 13):
        sel = (o < 10.0 ** -d) & (o >= 10.0 ** -(d + 1))
        if sel.any():
            out["1e-%d" % (d + 1)] = dict(n=int(sel.sum()), max=float(rel[sel].max()),
                                          p99=float(np.quantile(rel[sel], 0.99)), med=float(np.median(rel[sel])))
    return out


oracle.build()
for name, cfg, mask in cases():
    pb = oracle_problem(cfg, mask)
    Wo = oracle.build_kernels(pb)
    off = np.ones(pb.K, bool)
    off[pb.K // 2] = False
    nz, ny, nx = cfg.shape
    for flags, label in ((0, "chebyshev"), (fd.F_KGEN_DIRECT, "direct")):
        ctx = fd.build_kernels(lib_params(cfg, "fp32", flags=flags), mask)
        W = fd.export_kernels(ctx, (0, nx, 0, ny, 0, nz))
        fd.destroy(ctx)
        e = np.abs(W[..., off] - Wo[..., off])
        kmax = Wo[..., off].max(-1, keepdims=True)
        print(json.dumps(dict(case=name, path=label, max_abs=float(e.max()),
                              max_abs_over_kernel_offmax=float((e / kmax).max()),
                              p999_abs_over_kernel_offmax=float(np.quantile(e / kmax, 0.999)),
                              neg=int((W < 0).sum()), decades=decade_stats(W, Wo, off))))
