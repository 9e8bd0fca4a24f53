"""Per-rank superposition time for the slab a rank owns under N-way z-slab strong scaling of
cfg3 (192³ R5 bf16): one GPU, a closed 192×192×(192/N) grid (same tile count per launch as
a rank), device-timed with CUDA events.  Compares with the 1-GPU step / N (wave-quantisation
check for the scaling run).  `python tools/slab_timing.py [bf16|mx8]`."""
import sys

import torch

sys.path.insert(0, ".")
import fdirw_inputs as fi  # noqa: E402
import paper_2408_11376_b200 as fd  # noqa: E402

WEIGHTS = sys.argv[1] if len(sys.argv) > 1 else "bf16"
cfg = fi.config("cfg3")
full = cfg.mask()
for n in (1, 2, 4, 8):
    nz = 192 // n
    z0 = 96 - nz // 2
    mask = full[z0:z0 + nz].copy()
    p = fd.Params(nx=192, ny=192, nz=nz, dh=cfg.dh, D_fast=cfg.D_fast, D_slow=cfg.D_slow, dt=cfg.dt,
                  radius=5, n_fd=0, weights=WEIGHTS)
    with fd.build_kernels(p, mask) as ctx:
        c = torch.from_numpy(fi.initial_c(mask, "paper")).cuda()
        fd.run(ctx, c, 10)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = 200
        torch.cuda.synchronize()
        e0.record()
        fd.run(ctx, c, steps)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        print("N=%d slab %d planes, %d tiles: %.4f ms/step (ideal from N=1: see first line / N)" %
              (n, nz, ctx.info["n_tiles"], ms))
