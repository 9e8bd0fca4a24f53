import sys, time
sys.path.insert(0, ".")
import torch, fdirw_inputs as fi, paper_2408_11376_b200 as fd
cfg = fi.config("cfg3"); mask = cfg.mask(); nz, ny, nx = cfg.shape
p = fd.Params(nx=nx, ny=ny, nz=nz, dh=cfg.dh, D_fast=cfg.D_fast, D_slow=cfg.D_slow, dt=cfg.dt, radius=cfg.R, n_fd=0, weights="bf16")
s = torch.cuda.current_stream()
for i in range(4):
    torch.cuda.synchronize(); t = time.perf_counter()
    ctx = fd.build_kernels(p, mask, device=0, stream=s)
    t1 = time.perf_counter() - t
    t = time.perf_counter(); fd.destroy(ctx); t2 = time.perf_counter() - t
    print("build %.3f s  destroy %.3f s" % (t1, t2))
