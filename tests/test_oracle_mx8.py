"""Pins for the MX8 oracle (oracle/mx8.py): closed-form scales and codes,
the quantisation error bound, a brute-force source-centric loop for the block gather (the
indexing a transposed or shifted block would break), and mass conservation of the fix-up."""
import math

import numpy as np
import pytest

import fdirw_inputs as fi
from _util import oracle_problem, small_cfg
from oracle import mx8


@pytest.mark.parametrize("M,e", [
    (1.0, -7),                      # 1·2^7 = 128 ≤ 255, 1·2^8 = 256 > 255
    (255 * 2.0 ** -9, -9),          # exactly 255 quanta
    (255.5 * 2.0 ** -9, -8),        # just over: next power of two
    (128 * 2.0 ** -20, -20),        # 128 quanta
    (0.0, -126),                    # all-zero block
    (2.0 ** -140, -126),            # below the clamp: m = 2^−14 → 0
])
def test_block_scale_closed_form(M, e):
    assert int(mx8.block_scale_exp(np.array(M))) == e


def test_block_codes_closed_form():
    v = np.array([1.0, 0.5, 0.25, 1 / 128, 1 / 256, 3 / 256, -1e-10, 0.0])
    m, e = mx8.quantize_block(v)
    assert int(e) == -7
    # 1/256 = 0.5 quantum → 0 (half to even), 3/256 = 1.5 quanta → 2, negatives clamp to 0
    assert m.tolist() == [128, 64, 32, 1, 0, 2, 0, 0]


def test_error_bound_random_blocks():
    rng = np.random.default_rng(3)
    v = rng.random((2000, 8)) ** 6 * 10.0 ** rng.uniform(-12, 0, (2000, 1))
    m, e = mx8.quantize_block(v)
    s = np.ldexp(1.0, e)
    v32 = v.astype(np.float32).astype(np.float64)
    assert np.all(np.abs(m * s[:, None] - v32) <= 0.5 * s[:, None] * (1 + 1e-12))
    M = v32.max(-1)
    assert np.all(M / s <= 255) and np.all(M / s > 127.5)
    assert m.max() <= 255 and m.min() >= 0


def _brute(W, R):
    """Source-centric scalar loops: for every (source, offset) find its target's block by hand."""
    nz, ny, nx, K = W.shape
    L = 2 * R + 1
    out = np.zeros_like(W)
    for sz in range(nz):
        for sy in range(ny):
            for sx in range(nx):
                off = 0.0
                for o in range(K):
                    if o == K // 2:
                        continue
                    ox, oy, oz = o % L - R, (o // L) % L - R, o // (L * L) - R
                    tz, ty, tx = sz + oz, sy + oy, sx + ox
                    if not (0 <= tz < nz and 0 <= ty < ny and 0 <= tx < nx):
                        continue
                    x0 = tx - tx % 8
                    blk = []
                    for j in range(8):
                        ux = x0 + j
                        qz, qy, qx = tz - oz, ty - oy, ux - ox
                        ok = ux < nx and 0 <= qz < nz and 0 <= qy < ny and 0 <= qx < nx
                        blk.append(float(np.float32(W[qz, qy, qx, o])) if ok else 0.0)
                    M = max(max(blk), 0.0)
                    if M > 0:
                        fr, k = math.frexp(M)
                        e = k - 8
                        if math.ldexp(M, -e) > 255:
                            e += 1
                        e = max(e, -126)
                    else:
                        e = -126
                    w = blk[tx - x0]
                    m = min(round(math.ldexp(max(w, 0.0), -e)), 255)  # Python round: half to even
                    out[sz, sy, sx, o] = math.ldexp(m, e)
                    off += out[sz, sy, sx, o]
                out[sz, sy, sx, K // 2] = 1.0 - off
    return out


@pytest.mark.parametrize("R,shape", [
    (1, (3, 4, 11)),   # nx = 11: a full chunk and a ragged one
    (3, (2, 3, 5)),    # window larger than the grid in every direction
    (2, (1, 1, 17)),   # 1-D
])
def test_gather_blocks_vs_brute_force(R, shape):
    rng = np.random.default_rng(7)
    W = rng.random(shape + ((2 * R + 1) ** 3,)) ** 4
    W[rng.random(W.shape) < 0.1] = 0.0
    got = mx8.quantize_mx8(W, R)
    ref = _brute(W, R)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-15)


def test_oracle_kernels_mass_and_bound():
    cfg = small_cfg((6, 7, 13), 2, 60, D_slow=1e-3)
    pb = oracle_problem(cfg, fi.random_two_phase(cfg.shape, 0.6, seed=2))
    import oracle

    W = oracle.build_kernels(pb)
    Wq = mx8.quantize_mx8(W, pb.R)
    np.testing.assert_allclose(Wq.sum(-1), 1.0, atol=1e-14)  # every column conserves mass
    off = np.ones(pb.K, bool)
    off[pb.K // 2] = False
    # |error| ≤ s/2 < M/255, M ≤ the largest weight of that offset within ±7 sources in x
    nz, ny, nx, K = W.shape
    Mx = np.zeros_like(W)
    for dx in range(-7, 8):
        sh = np.zeros_like(W)
        if dx >= 0:
            sh[:, :, :nx - dx] = W[:, :, dx:]
        else:
            sh[:, :, -dx:] = W[:, :, :nx + dx]
        Mx = np.maximum(Mx, sh)
    err = np.abs(Wq - W)[..., off]
    assert np.all(err <= Mx[..., off] / 255 + 1e-9 * W.max())
    assert np.abs(Wq - W)[..., off].max() > 0  # it does quantise
