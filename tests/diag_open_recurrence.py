"""Diagnostic (GPU + oracle): kept kernel mass M_s of windows touching the N2 reservoir, the
Chebyshev recurrence (reduced-precision storage default) vs the literal substeps
(FDIRW_KGEN_OPEN_LITERAL=1), both against the oracle's fp64 kernels.  Prints max / median of
|M − M_oracle| for open windows.  Usage: python tests/diag_open_recurrence.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import fdirw_inputs as fi  # noqa: E402
import oracle  # noqa: E402
import paper_2408_11376_b200 as fd  # noqa: E402
from _util import lib_params, oracle_problem, small_cfg  # noqa: E402

oracle.build()
for fmt, R, shape in (("bf16", 5, (14, 13, 15)), ("fp16", 3, (14, 13, 15)), ("bf16", 8, (19, 18, 20))):
    m = fi.porous_particle(shape, min(shape) / 2 - 4, pore_r=(1.0, 2.0), porosity=0.3, seed=4)
    mask = fi.with_far_field(m, min(shape) / 2 - 4, margin=2.0)
    cfg = small_cfg(shape, R, 1000, D_slow=1e-3, weights=fmt)
    pb = oracle_problem(cfg, mask)
    Wo = oracle.build_kernels(pb).reshape(-1, pb.K)
    ow = oracle.open_windows(pb).reshape(-1) & (mask.reshape(-1) <= 1)
    Mo = Wo.sum(1)
    box = (0, shape[2], 0, shape[1], 0, shape[0])
    for form in ("recurrence", "literal"):
        if form == "literal":
            os.environ["FDIRW_KGEN_OPEN_LITERAL"] = "1"
        else:
            os.environ.pop("FDIRW_KGEN_OPEN_LITERAL", None)
        ctx = fd.build_kernels(lib_params(cfg, v_far=2000.0), mask)
        try:
            W = fd.export_kernels(ctx, box).reshape(-1, pb.K).astype(np.float64)
        finally:
            fd.destroy(ctx)
        dM = np.abs(W.sum(1) - Mo)[ow]
        rel = dM / Mo[ow]
        print("%s R%d %-10s open windows %d: |dM| max %.2e median %.2e; rel max %.2e median %.2e (M min %.2e)"
              % (fmt, R, form, ow.sum(), dM.max(), np.median(dM), rel.max(), np.median(rel), Mo[ow].min()))
