#!/usr/bin/env python
"""Small end-to-end exercise of every CUDA entry point, for compute-sanitizer
(memcheck / racecheck / initcheck):  compute-sanitizer --tool memcheck python tools/sanitize_small.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fdirw_inputs as fi  # noqa: E402
import paper_2408_11376_b200 as fd  # noqa: E402


# SANITIZE_NO_BULK=1: every context streams weights with per-thread loads (the racecheck
# control run: racecheck does not model cp.async.bulk's mbarrier completion)
EXTRA = fd.F_NO_BULK_STREAM if os.environ.get("SANITIZE_NO_BULK") == "1" else 0


def params(shape, R, n_fd, fmt="bf16", flags=0, v_far=0.0):
    flags |= EXTRA
    nz, ny, nx = shape
    return fd.Params(nx=nx, ny=ny, nz=nz, dh=1.0, D_fast=1.0, D_slow=1e-3, dt=0.1 * n_fd, radius=R, n_fd=0,
                     weights=fmt, flags=flags, v_far=v_far)


def main():
    shape = (12, 11, 21)
    mask = fi.porous_particle(shape, 4, pore_r=(1.0, 1.5), n_pores=3, seed=1)
    c0 = torch.from_numpy(fi.initial_c(mask, "random", seed=1)).cuda()
    for fmt, flags in (("bf16", 0), ("fp32", fd.F_NO_DEDUP), ("fp16", fd.F_DEDUP_STORAGE)):
        with fd.build_kernels(params(shape, 3, 30, fmt, flags), mask) as ctx:
            out = torch.empty_like(c0)
            fd.step(ctx, c0, out)
            c = c0.clone()
            fd.run(ctx, c, 3)
            fd.mass(ctx, c)
            if not flags & fd.F_DEDUP_STORAGE:  # export needs the dense layout
                fd.export_kernels(ctx, (0, 5, 0, 4, 0, 3))
    # the two-columns-per-thread kgen (kgen_bal.cu: R5 two z segments, R8 three), Chebyshev and
    # literal passes, closed and open windows, and the column kernel it replaces (A/B flag)
    kshape = (9, 10, 11)
    kmask = fi.porous_particle(kshape, 4, pore_r=(1.0, 1.5), n_pores=3, seed=4)
    fkmask = fi.with_far_field(kmask, 4, 0.5)
    for R, m, flags, vf in ((5, kmask, 0, 0.0), (5, fkmask, 0, 100.0), (5, kmask, fd.F_KGEN_COLUMNS, 0.0),
                            (8, kmask, 0, 0.0), (8, kmask, fd.F_KGEN_DIRECT, 0.0)):
        with fd.build_kernels(params(kshape, R, 30, "bf16", flags, v_far=vf), m) as ctx:
            fd.export_kernels(ctx, (0, 3, 0, 3, 0, 3))
    # round 2 entry points: host-buffer step (plain and plane-chunk pipelined), phase profile,
    # slab mass, the staged-stream canary
    hin = c0.cpu().pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    with fd.build_kernels(params(shape, 3, 30, "bf16"), mask) as ctx:
        fd.step_host(ctx, hin, hout)
        c = c0.clone()
        fd.profile_phases(ctx, c, 2)
        fd.mass_local(ctx, c)
    pshape = (48, 11, 21)  # 48 planes >= 4R: the pipelined form (chunks of 8 planes)
    pmask = fi.porous_particle(pshape, 4, pore_r=(1.0, 1.5), n_pores=3, seed=3)
    pin = torch.from_numpy(fi.initial_c(pmask, "random", seed=3)).pin_memory()
    pout = torch.empty_like(pin).pin_memory()
    with fd.build_kernels(params(pshape, 3, 30, "bf16"), pmask) as ctx:
        fd.step_host(ctx, pin, pout)
        fd.step_host(ctx, pout, pin)
    # TMA-staged weight stream (needs >= 2 CTAs/SM of tiles: 40 planes x 8 tiles), dense and N4 mixed
    big = (40, 64, 256)
    bmask = fi.porous_particle(big, 14, pore_r=(1.0, 2.0), porosity=0.3, seed=2)
    cb = torch.from_numpy(fi.initial_c(bmask, "random", seed=2)).cuda()
    for flags in (0, fd.F_DEDUP_STORAGE):
        with fd.build_kernels(params(big, 1, 4, "bf16", flags), bmask) as ctx:
            assert ctx.info["n_tiles"] >= 2 * 148
            c = cb.clone()
            fd.run(ctx, c, 2)
            if not flags:
                fd.debug_stage_canary(ctx, True)
                fd.run(ctx, c, 1)
                assert fd.debug_stage_canary(ctx, True)[1] == 0
    # MX8 weights: expand + diag build pass, staged MX8 stream (tile 256 and a
    # runtime tile width), export
    if not EXTRA:
        for shp, R in ((shape, 3), (big, 1)):
            mk = mask if shp == shape else bmask
            with fd.build_kernels(params(shp, R, 30, "mx8"), mk) as ctx:
                c = (c0 if shp == shape else cb).clone()
                fd.run(ctx, c, 2)
                fd.mass(ctx, c)
                fd.export_kernels(ctx, (0, 5, 0, 4, 0, 3))
    # far field (N2)
    fmask = fi.with_far_field(fi.porous_particle(shape, 4, pore_r=(1.0, 1.5), n_pores=3, seed=1), 4, 2.0)
    with fd.build_kernels(params(shape, 2, 20, v_far=100.0), fmask) as ctx:
        c = c0.clone()
        fd.far_init(ctx, c, 0.5)
        fd.run(ctx, c, 2)
        fd.far_get(ctx)
    # N3 absorption loop (impermeable solid context): interface-group list, grouped sweeps,
    # in-place scatter, the replayed two-step graph and an odd tail; without a solid pass too
    nz, ny, nx = shape
    ap = fd.Params(nx=nx, ny=ny, nz=nz, dh=1.0, D_fast=1.0, D_slow=0.0, dt=2.0, radius=2, n_fd=0, weights="bf16",
                   flags=EXTRA, v_far=100.0)
    with fd.build_kernels(ap, fmask) as ctx:
        c = c0.clone() * torch.from_numpy((fmask != 2).astype(np.float32)).cuda()
        fd.far_init(ctx, c, 0.5)
        fd.absorb_run(ctx, c, 3, 0.01, 0.05, 1.0, 1e-5)
        fd.absorb_run(ctx, c, 2, 0.0, 0.05, 1.0, 1e-5)
    # virtual ranks
    sl = fd.slabs(shape[0], 3)
    ctxs = [fd.build_kernels(params(shape, 3, 20, v_far=100.0), fmask, rank=r, world=3, z_begin=a, z_end=b, device=0)
            for r, (a, b) in enumerate(sl)]
    cin = [c0[a:b].contiguous() for a, b in sl]
    cout = [torch.empty_like(t) for t in cin]
    fd.far_init_virtual(ctxs, cin, 0.5)
    fd.step_virtual(ctxs, cin, cout)
    for x in ctxs:
        fd.destroy(x)
    # coarse mesh (N1)
    region = fi.near_field(mask, 4, margin=2)
    with fd.coarse_build(params(shape, 1, 30), region, block=3) as cc:
        out = torch.empty_like(c0)
        fd.coarse_step(cc, c0, out)
        fd.coarse_run(cc, out, 2)
        fd.coarse_export(cc)
    torch.cuda.synchronize()
    print("sanitize_small: ok")


if __name__ == "__main__":
    main()
