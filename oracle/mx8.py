"""CPU ORACLE for the MX8 weight format — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import this.
It shares no code with the CUDA path (``csrc/mx8.cuh``).

MX8 is this repo's storage format, not the paper's (the paper's formats are FP64/FP32/FP16,
P:155-157 §3.3).  What it must preserve is the paper's operator: C_new(x) = Σ_s W_s(x−s)·C_old(s)
(Eq.8 with the windowed kernels of reading A1) with every column summing to 1 (mass
conservation of the closed domain, reading A10).  The definition, written out plainly:

* gather block = for one window offset o and one target row (z, y): the 8 targets
  x0 … x0+7 with x0 = 8·⌊x/8⌋ (the superposition's 8-target thread chunk).  Its 8 weights are
  W_{t−o}(o) for the 8 targets t (0 where t − o is outside the grid or t ≥ nx);
* scale s = 2^e, e the smallest integer with max(block)·2^−e ≤ 255, e ≥ −126
  (s = 2^−126 for an all-zero block);
* mantissa m = RNE(max(w, 0)/s) ∈ [0, 255]; decoded weight m·s;
* the centre weight (diagonal) = 1 − Σ_{o≠0} decoded W_s(o) (reading A10's fix-up).

The decision (the code m) is taken on the weight rounded to fp32 — the precision the CUDA
path quantises in — so both sides decide in the same precision (the kernels themselves differ
by the kgen fp32 round-off, which tests bound separately).
"""
from __future__ import annotations

import numpy as np


def block_scale_exp(M: np.ndarray) -> np.ndarray:
    """e per block: smallest integer with M·2^−e ≤ 255 (M ≥ 0, fp32 values), clamped to ≥ −126."""
    M = np.asarray(M, np.float64)
    f, k = np.frexp(M)                 # M = f·2^k, f ∈ [0.5, 1)  →  M ∈ [2^(k−1), 2^k)
    e = k - 8                          # M·2^−e ∈ [128, 256)
    e = np.where(np.ldexp(M, -e) > 255.0, e + 1, e)
    e = np.where(M > 0, e, -126)
    return np.maximum(e, -126).astype(np.int64)


def quantize_block(v: np.ndarray):
    """One block (…, 8) of weights → (m (…, 8) int, e (…,)): the format's definition."""
    v = np.asarray(v, np.float32).astype(np.float64)  # the decision is taken on fp32 weights
    e = block_scale_exp(np.maximum(v, 0.0).max(-1))
    m = np.rint(np.ldexp(np.maximum(v, 0.0), -e[..., None]))  # numpy rint: round half to even
    return np.minimum(m, 255).astype(np.int64), e


def quantize_mx8(W: np.ndarray, R: int) -> np.ndarray:
    """Source-major kernels W [nz][ny][nx][K] of the WHOLE grid (oracle.build_kernels) → the
    MX8-stored operator decoded to fp64, same layout, diagonal = the mass fix-up."""
    nz, ny, nx, K = W.shape
    L = 2 * R + 1
    assert K == L ** 3
    kc = K // 2
    nxq = (nx + 7) // 8
    Wq = np.zeros_like(W)
    for o in range(K):
        if o == kc:
            continue
        ox, oy, oz = o % L - R, (o // L) % L - R, o // (L * L) - R
        if abs(ox) >= nx or abs(oy) >= ny or abs(oz) >= nz:
            continue  # the offset leaves the grid from every source: no (source, target) pair
        # gather view: G[z, y, x] = W_{(z,y,x) − o}(o) for targets x in the grid, else 0
        G = np.zeros((nz, ny, nxq * 8))
        tz = slice(max(0, oz), min(nz, nz + oz)); sz = slice(max(0, -oz), min(nz, nz - oz))
        ty = slice(max(0, oy), min(ny, ny + oy)); sy = slice(max(0, -oy), min(ny, ny - oy))
        tx = slice(max(0, ox), min(nx, nx + ox)); sx = slice(max(0, -ox), min(nx, nx - ox))
        G[tz, ty, tx] = W[sz, sy, sx, o]
        m, e = quantize_block(G.reshape(nz, ny, nxq, 8))
        D = np.ldexp(m.astype(np.float64), e[..., None]).reshape(nz, ny, nxq * 8)
        Wq[sz, sy, sx, o] = D[tz, ty, tx]
    Wq[..., kc] = 1.0 - (Wq.sum(-1) - Wq[..., kc])
    return Wq
