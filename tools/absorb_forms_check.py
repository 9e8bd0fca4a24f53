"""A/B of the N3 tail forms on cfg3o (GPU): the nf path (default), FDIRW_ABSORB_FULL=1 (solid pass
sweeps the grid), FDIRW_ABSORB_SCALAR=1 (per-voxel sweeps): after 1 / 2 / 10 macro steps, the
fields' differences (where, by phase) and c_far.  Usage: python tools/absorb_forms_check.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fdirw_inputs as fi  # noqa: E402
import paper_2408_11376_b200 as fd  # noqa: E402

cfg = fi.config("cfg3o")
mask = cfg.mask()
nz, ny, nx = cfg.shape
T = fi.TABLE1
params = fd.Params(nx=nx, ny=ny, nz=nz, dh=cfg.dh, D_fast=cfg.D_fast, D_slow=0.0, dt=cfg.dt, radius=cfg.R,
                   n_fd=cfg.n_fd, weights=cfg.weights, v_far=cfg.v_far)
kin_p = dict(D_S=fi.D_SLOW_SI, k=0.05, c_S_eq=1.0, c_L_eq=1e-5)
c0 = np.where(mask == 1, T["c_L0"], np.where(mask == 0, T["c_S0"], 0.0)).astype(np.float32)
res = {}
for form in ("nf", "full", "scalar"):
    for ev in ("FDIRW_ABSORB_FULL", "FDIRW_ABSORB_SCALAR"):
        os.environ.pop(ev, None)
    if form != "nf":
        os.environ["FDIRW_ABSORB_" + form.upper()] = "1"
    ctx = fd.build_kernels(params, mask)
    c = torch.from_numpy(c0).cuda()
    fd.far_init(ctx, c, cfg.c_far0)
    ks = []
    for n in (1, 1, 8):
        k = fd.absorb_run(ctx, c, n, **kin_p)
        ks.append((c.cpu().numpy().copy(), k[-1].copy()))
    res[form] = ks
    fd.destroy(ctx)
for i, n in enumerate((1, 2, 10)):
    a, b, s = res["nf"][i], res["full"][i], res["scalar"][i]
    d = a[0] != b[0]
    print("after %d steps: nf vs full differ at %d voxels (phases %s), max %.3e; full vs scalar max %.3e; "
          "c_far nf %.10e full %.10e" % (n, d.sum(), np.bincount(mask[d], minlength=3), np.abs(a[0] - b[0]).max(),
                                         np.abs(b[0] - s[0]).max(), a[1][2], b[1][2]))
