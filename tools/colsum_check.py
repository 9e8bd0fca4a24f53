"""Where does the fp32 long-run mass drift come from?  Column sums of the exported stored operator
(fp64 sums) → the drift one step of exact arithmetic would cause, vs the GPU's measured per-step
drift."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import fdirw_inputs as fi  # noqa: E402
import paper_2408_11376_b200 as fd  # noqa: E402
from _util import lib_params, small_cfg  # noqa: E402

shape = (36, 36, 36)
cfg = small_cfg(shape, 4, 1000, D_slow=1e-5)
mask = fi.porous_block(shape, pore_r=(2.0, 3.0), porosity=0.45, seed=6)
out = {}
for fmt in ("fp32", "bf16"):
    ctx = fd.build_kernels(lib_params(cfg, fmt), mask)
    W = fd.export_kernels(ctx, (0, 36, 0, 36, 0, 36))
    c0 = fi.initial_c(mask, "random", seed=6).astype(np.float32)
    cs = W.sum(-1) - 1.0
    pred = float((cs * c0.astype(np.float64)).sum() / c0.astype(np.float64).sum())
    c = torch.from_numpy(c0).cuda()
    m0 = fd.mass(ctx, c)
    fd.run(ctx, c, 100)
    m1 = fd.mass(ctx, c)
    fd.destroy(ctx)
    out[fmt] = {"colsum_dev_mean": float(cs.mean()), "colsum_dev_absmax": float(np.abs(cs).max()),
                "predicted_drift_per_step": pred, "measured_drift_per_step": (m1 - m0) / m0 / 100,
                "colsum_dev_mean_liquid": float(cs[mask == 1].mean()), "colsum_dev_mean_solid": float(cs[mask == 0].mean())}
print(json.dumps(out, indent=1))
