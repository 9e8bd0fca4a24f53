# Emulation (oracle, fp64 host) of an MX-style weight format for NEXT row N4: u8 mantissas with one
# power-of-two scale per gather block (8 targets x 1 slot), fp32 diagonal fix-up; relL2 after 10
# steps vs the exact kernels, beside bf16.  Design study for DESIGN.md §14, not product.
import sys, numpy as np
import os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, 'tests'))
import fdirw_inputs as fi, oracle
from _util import oracle_problem, small_cfg
oracle.build()

def gather_blocks_quant(W, R, mode):
    # W: [nz][ny][nx][K] source-major fp64; returns quantized W' (same layout) by gather blocks of 8 targets
    nz, ny, nx, K = W.shape
    L = 2*R+1
    Wq = np.zeros_like(W)
    offs = [(o % L - R, (o // L) % L - R, o // (L*L) - R) for o in range(K)]
    for o, (ox, oy, oz) in enumerate(offs):
        if o == K//2: continue
        # gather weight for target x: G[z,y,x] = W[z-oz, y-oy, x-ox, o]
        G = np.zeros((nz, ny, nx))
        zs = slice(max(0, oz), min(nz, nz+oz)); ys = slice(max(0, oy), min(ny, ny+oy)); xs = slice(max(0, ox), min(nx, nx+ox))
        zs2 = slice(max(0, -oz), min(nz, nz-oz)); ys2 = slice(max(0, -oy), min(ny, ny-oy)); xs2 = slice(max(0, -ox), min(nx, nx-ox))
        G[zs, ys, xs] = W[zs2, ys2, xs2, o]
        nxq = (nx+7)//8
        Gp = np.zeros((nz, ny, nxq*8)); Gp[:, :, :nx] = G
        B = Gp.reshape(nz, ny, nxq, 8)
        if mode == 'bf16':
            import torch
            Q = torch.from_numpy(B.astype(np.float32)).to(torch.bfloat16).double().numpy()
        else:
            mx = B.max(-1, keepdims=True)
            e = np.ceil(np.log2(np.maximum(mx, 1e-300) / 255.0))
            sc = np.where(mx > 0, 2.0**e, 1.0)
            Q = np.round(B / sc) * sc
        Gq = Q.reshape(nz, ny, nxq*8)[:, :, :nx]
        Wq[zs2, ys2, xs2, o] = Gq[zs, ys, xs]
    # fix-up diag per source
    Wq[..., K//2] = 1.0 - (Wq.sum(-1) - Wq[..., K//2])
    return Wq

for name, shape, R, Ds in (("cfg1", None, 2, 1e-3), ("cfg2s", (24, 22, 26), 4, 1e-5), ("R5", (22, 24, 26), 5, 1e-3)):
    if shape is None:
        cfg = fi.config("cfg1", n_fd=1000, weights="fp32"); mask = cfg.mask()
    else:
        cfg = small_cfg(shape, R, 1000, D_slow=Ds, weights="fp32")
        mask = fi.porous_particle(shape, min(shape)//2 - 3, pore_r=(1.0, 2.0), porosity=0.3, seed=5)
    pb = oracle_problem(cfg, mask)
    W = oracle.build_kernels(pb)
    nz, ny, nx = mask.shape
    box = (0, nx, 0, ny, 0, nz)
    c0 = fi.initial_c(mask, "paper").astype(np.float64)
    res = {}
    for mode in ("exact", "bf16", "mx8"):
        Wm = W if mode == "exact" else gather_blocks_quant(W, cfg.R, mode)
        C = c0.copy()
        for _ in range(10): C = oracle.step_scatter(pb, Wm, box, C, box)
        res[mode] = C
    ref = res["exact"]
    for mode in ("bf16", "mx8"):
        print(name, mode, "relL2 %.2e" % (np.linalg.norm(res[mode]-ref)/np.linalg.norm(ref)), "mass %.1e" % abs(res[mode].sum()/ref.sum()-1))
