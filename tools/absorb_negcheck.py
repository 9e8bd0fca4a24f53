"""Diagnostic (GPU): the N3 loop on cfg3o for 1000 macro steps in several weight formats / tail
forms; reports the minimum liquid value, where, and when it first goes negative (reading A26's
p_BC = 1 - row sum is negative at pore targets of the truncated windows).
Usage: python tools/absorb_negcheck.py"""
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import fdirw_inputs as fi, paper_2408_11376_b200 as fd
cfg = fi.config("cfg3o"); mask = cfg.mask(); nz, ny, nx = cfg.shape; T = fi.TABLE1
c0 = np.where(mask == 1, T["c_L0"], np.where(mask == 0, T["c_S0"], 0.0)).astype(np.float32)
for form, w in (("default","bf16"), ("scalar","bf16"), ("default","fp32"), ("default", "fp16"), ("pbc_reservoir", "bf16")):
    for ev in ("FDIRW_ABSORB_SCALAR",): os.environ.pop(ev, None)
    if form == "scalar": os.environ["FDIRW_ABSORB_SCALAR"] = "1"
    p = fd.Params(nx=nx, ny=ny, nz=nz, dh=cfg.dh, D_fast=cfg.D_fast, D_slow=0.0, dt=cfg.dt, radius=cfg.R,
                  n_fd=cfg.n_fd, weights=w, v_far=cfg.v_far,
                  flags=fd.F_PBC_RESERVOIR if form == "pbc_reservoir" else 0)
    ctx = fd.build_kernels(p, mask)
    c = torch.from_numpy(c0).cuda(); fd.far_init(ctx, c, cfg.c_far0)
    first = None
    for k in range(20):
        fd.absorb_run(ctx, c, 50, fi.D_SLOW_SI, 0.05, 1.0, 1e-5)
        g = c.cpu().numpy()
        mn = g[mask == 1].min()
        if mn < 0 and first is None: first = (k + 1) * 50
    g = c.cpu().numpy()
    liq = np.where(mask == 1, g, np.inf)
    i = np.unravel_index(np.argmin(liq), g.shape)
    nb = mask[max(i[0]-1,0):i[0]+2, max(i[1]-1,0):i[1]+2, max(i[2]-1,0):i[2]+2]
    print(form, w, "liquid min %.3e at %s (first negative after %s steps); #neg %d; solid max %.3e; neighbourhood phases %s" % (
        g[i], i, first, int((g[mask == 1] < 0).sum()), g[mask == 0].max(), np.bincount(nb.ravel(), minlength=3)))
    fd.destroy(ctx)
