"""Mass drift of long runs (north_star: total mass to 1e-6 relative): relative change of Σc after
n macro steps for each weight format, on cfg3 (192³) and a 36³ D-ratio-1e5 block.  One JSON line."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import fdirw_inputs as fi  # noqa: E402
import paper_2408_11376_b200 as fd  # noqa: E402
from _util import lib_params, small_cfg  # noqa: E402

out = {}
cases = [("block36", small_cfg((36, 36, 36), 4, 1000, D_slow=1e-5), fi.porous_block((36, 36, 36), pore_r=(2.0, 3.0),
                                                                                    porosity=0.45, seed=6), "random"),
         ("cfg3", fi.config("cfg3"), None, "paper")]
for name, cfg, mask, init in cases:
    mask = cfg.mask() if mask is None else mask
    for fmt in ("fp32", "fp16", "bf16", "mx8"):
        ctx = fd.build_kernels(lib_params(cfg, fmt), mask)
        c = torch.from_numpy(fi.initial_c(mask, init, seed=6)).cuda()
        m0 = fd.mass(ctx, c)
        rec = {}
        done = 0
        for n in (10, 100, 1000):
            fd.run(ctx, c, n - done)
            done = n
            rec[n] = (fd.mass(ctx, c) - m0) / m0
        fd.destroy(ctx)
        out["%s_%s" % (name, fmt)] = rec
print(json.dumps(out))
