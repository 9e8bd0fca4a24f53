"""Minimal compute-sanitizer target for the two-columns kgen (kgen_bal.cu, R5 and R8 builds on a
small porous grid):

    FDIRW_KGEN_SYNCCHECK=1 compute-sanitizer --tool synccheck python tools/kgen_synccheck.py
    compute-sanitizer --tool racecheck python tools/kgen_synccheck.py

(FDIRW_KGEN_SYNCCHECK=1 selects the barrier form synccheck accepts, kgen_common.cuh.)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fdirw_inputs as fi  # noqa: E402
import paper_2408_11376_b200 as fd  # noqa: E402

shape = (9, 10, 11)
mask = fi.porous_particle(shape, 4, pore_r=(1.0, 1.5), n_pores=3, seed=4)
for R in (5, 8):
    p = fd.Params(nx=shape[2], ny=shape[1], nz=shape[0], dh=1.0, D_fast=1.0, D_slow=1e-3, dt=3.0, radius=R, n_fd=0,
                  weights="bf16", flags=0, v_far=0.0)
    with fd.build_kernels(p, mask):
        pass
print("ok")
