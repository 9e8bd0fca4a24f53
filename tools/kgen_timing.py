"""Times fdirw_build_kernels (a1-a4) for a config several times in one process:
the first build includes CUDA lazy module loading; later ones show the steady cost."""
import sys
import time

import torch

sys.path.insert(0, ".")
import fdirw_inputs as fi  # noqa: E402
import paper_2408_11376_b200 as fd  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
cfg = fi.config(name)
mask = cfg.mask()
nz, ny, nx = cfg.shape
p = fd.Params(nx=nx, ny=ny, nz=nz, dh=cfg.dh, D_fast=cfg.D_fast, D_slow=cfg.D_slow, dt=cfg.dt, radius=cfg.R,
              n_fd=cfg.n_fd, weights=cfg.weights, v_far=cfg.v_far, flags=flags)
for i in range(reps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    ctx = fd.build_kernels(p, mask)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    info = ctx.info
    print("%s build %d: %.3f s  kgen kernel %.1f ms (%d passes/window)  windows %d  sources %d"
          % (name, i, dt, info["kgen_kernel_ms"], info["kgen_steps"], info["kgen_windows"], info["kgen_sources"]))
    fd.destroy(ctx)
