"""§4.2 / Fig.10 analogue at full size (GPU): the paper's FP32, mixed FP32/FP16 and FP16 modes of the
superposition (the study kernels of fdirw_set_precision_mode) in the integrated absorption
loop on cfg3o (the open R50 model, Table 1 kinetics) for 1000 macro steps (t = 0.5 s), against the
product path with fp32 weights (compensated fp32 accumulation, fp32-pair diagonal) as the
reference — the fp64 oracle does not run 1000 steps of a 120³ grid; the product path is within
~1e-7 of it on the desk model (tests/test_gpu_absorb.py).  Reports the relative error of c̄_S(t)
(Fig.10c) and of the final liquid field, per mode.  Usage:
  python tools/precision_study.py [steps] [reservoir] > profiles/<round>_precision_study_cfg3o[_pbc_reservoir].json"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fdirw_inputs as fi  # noqa: E402
import paper_2408_11376_b200 as fd  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
PBC = fd.F_PBC_RESERVOIR if (len(sys.argv) > 2 and sys.argv[2] == "reservoir") else 0  # p_BC reading (A26)
cfg = fi.config("cfg3o")
mask = cfg.mask()
nz, ny, nx = cfg.shape
T = fi.TABLE1
kin_p = dict(D_S=fi.D_SLOW_SI, k=0.05, c_S_eq=1.0, c_L_eq=1e-5)
c0 = np.where(mask == 1, T["c_L0"], np.where(mask == 0, T["c_S0"], 0.0)).astype(np.float32)


def run(weights, mode, flags):
    p = fd.Params(nx=nx, ny=ny, nz=nz, dh=cfg.dh, D_fast=cfg.D_fast, D_slow=0.0, dt=cfg.dt, radius=cfg.R,
                  n_fd=cfg.n_fd, weights=weights, v_far=cfg.v_far, flags=flags | PBC)
    ctx = fd.build_kernels(p, mask)
    try:
        c = torch.from_numpy(c0).cuda()
        fd.far_init(ctx, c, cfg.c_far0)
        fd.set_precision_mode(ctx, mode)
        kin = fd.absorb_run(ctx, c, steps, **kin_p)
        return kin, c.cpu().numpy().astype(np.float64)
    finally:
        fd.destroy(ctx)


ref_kin, ref_c = run("fp32", "default", 0)
liq = mask == 1
out = {"workload": "cfg3o open R50 model, integrated absorption loop, %d macro steps (t = %.3f s)" % (steps, steps * cfg.dt),
       "reference": "product path, fp32 weights (compensated fp32 accumulation)",
       "p_bc": "reservoir FD (FDIRW_F_PBC_RESERVOIR)" if PBC else "1 - row sum (A26)",
       "paper": "P:199-201: relative errors ~1e-6 (FP32), ~1e-5 (mixed FP32/FP16), ~1e-2 (FP16); errors do not grow",
       "c_bar_S_final_ref": float(ref_kin[-1, 3]), "modes": {}}
# the paper's three modes as it states them (P stored plainly in the mode's format: no diagonal
# fix-up), then the same modes with this repo's fp32-pair diagonal fix-up (A10), then the
# product path (A9: weights only reduced, fp32 products and accumulation) with fp16 / bf16 weights
cases = [("fp32", "fp32", "fp32", fd.F_NO_MASS_FIX), ("mixed", "mixed", "fp16", fd.F_NO_MASS_FIX),
         ("fp16", "fp16", "fp16", fd.F_NO_MASS_FIX), ("mixed+mass_fix", "mixed", "fp16", 0),
         ("fp16+mass_fix", "fp16", "fp16", 0), ("product_fp16_weights", "default", "fp16", 0),
         ("product_bf16_weights", "default", "bf16", 0)]
for name, mode, w, flags in cases:
    try:
        kin, c = run(w, mode, flags)
    except fd.FdirwError as e:
        out["modes"][name] = {"unavailable": str(e)}
        continue
    re = np.abs(kin[:, 3] - ref_kin[:, 3]) / ref_kin[:, 3]
    out["modes"][name] = {
        "mode": mode,
        "mass_fix": not (flags & fd.F_NO_MASS_FIX),
        "weights": w,
        "c_bar_S_rel_err_max": float(re.max()),
        "c_bar_S_rel_err_final": float(re[-1]),
        "c_bar_S_rel_err_every_100": [float(x) for x in re[99::100]],
        "liquid_field_relL2_final": float(np.linalg.norm(c[liq] - ref_c[liq]) / np.linalg.norm(ref_c[liq])),
    }
print(json.dumps(out, indent=1))
