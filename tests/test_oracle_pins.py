"""Pins of the CPU fp64 oracle against what the paper and the mathematics fix
(SURVEY §8c pins P1–P12).  No GPU, no product code."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import fdirw_inputs as fi

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def lat(mask, R, n_fd, D_slow=1e-3, D_fast=1.0):
    import oracle

    return oracle.Problem(mask=mask, dh=1.0, D_fast=D_fast, D_slow=D_slow, dt=0.1 * n_fd, R=R, n_fd=0)


# ---------------------------------------------------------------- a1 / Table 1
def test_table1_derivation(oracle_lib):
    """Table 1: Δt/Δt_fd = 1000 and λ = 0.1 from the printed SI values."""
    g = json.load(open(os.path.join(GOLD, "table1.json")))
    D_f = g["D_L_m2_s"] * g["A_L_over_RT"]
    D_s = g["D_S_m2_s"] * g["A_S_over_RT"]
    pb = oracle_lib.Problem(mask=np.ones((4, 4, 4), np.uint8), dh=g["dh_m"], D_fast=D_f, D_slow=D_s,
                            dt=g["dt_s"], R=1)
    d = oracle_lib.derive(pb)
    assert d.n_fd == g["derived"]["n_fd"]
    assert d.dt_fd == pytest.approx(g["dt_fd_s"], rel=1e-12)
    assert d.lam_ff == pytest.approx(g["derived"]["lambda_fast"], rel=1e-12)
    assert d.lam_ss == pytest.approx(g["derived"]["lambda_slow"], rel=1e-12)
    # harmonic mean across phases (A4): 2·a·b/(a+b)
    assert d.lam_fs == pytest.approx(2 * 0.1 * 1e-4 / (0.1 + 1e-4), rel=1e-12)
    assert D_f / D_s == pytest.approx(g["derived"]["D_ratio"])


def test_derivation_guards(oracle_lib):
    pb = lat(np.ones((2, 2, 2), np.uint8), 1, 7)
    assert oracle_lib.derive(pb).n_fd == 7  # lattice preset reproduces n_fd exactly
    bad = oracle_lib.Problem(mask=np.ones((2, 2, 2), np.uint8), dh=1.0, D_fast=1.0, D_slow=0.0, dt=1.0, R=1, n_fd=1)
    with pytest.raises(ValueError, match="unstable"):
        oracle_lib.derive(bad)  # λ = 1 > 1/6
    with pytest.raises(ValueError):
        oracle_lib.derive(oracle_lib.Problem(mask=np.ones((2, 2, 2), np.uint8), dh=1.0, D_fast=-1.0,
                                             D_slow=0.0, dt=1.0, R=1))


# ---------------------------------------------------------------- P7 stencil
def test_one_substep_stencil(oracle_lib):
    """P7: one substep from δ → centre 1−6λ, faces λ, all else 0."""
    g = json.load(open(os.path.join(GOLD, "stencil_one_step.json")))
    pb = lat(np.ones((7, 7, 7), np.uint8), 2, 1)
    W = oracle_lib.kernel(pb, (3, 3, 3))
    R = 2
    exp = np.zeros_like(W)
    exp[R, R, R] = g["centre"]
    for a, b, c in [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]:
        exp[R + a, R + b, R + c] = g["face"]
    np.testing.assert_allclose(W, exp, rtol=0, atol=1e-15)


def test_harmonic_two_cell(oracle_lib):
    """Reading A4 closed form: 2 voxels (fast|slow), one substep from the fast one:
    [1−λ_fs, λ_fs] with λ_fs = Δt_fd·2·D_f·D_s/(D_f+D_s)/Δh²."""
    mask = np.array([[[1, 0]]], np.uint8)
    Df, Ds, dt_fd, dh = 3.0, 0.5, 0.02, 0.7
    pb = oracle_lib.Problem(mask=mask, dh=dh, D_fast=Df, D_slow=Ds, dt=dt_fd, R=1, n_fd=1)
    lam = dt_fd * 2 * Df * Ds / (Df + Ds) / dh ** 2
    W = oracle_lib.kernel(pb, (0, 0, 0))  # window slot [oz+1][oy+1][ox+1]
    assert W[1, 1, 1] == pytest.approx(1 - lam, abs=1e-15)
    assert W[1, 1, 2] == pytest.approx(lam, abs=1e-15)
    assert np.count_nonzero(W) == 2  # out-of-domain slots are 0 (A21)
    W2 = oracle_lib.kernel(pb, (1, 0, 0))
    assert W2[1, 1, 1] == pytest.approx(1 - lam, abs=1e-15) and W2[1, 1, 0] == pytest.approx(lam, abs=1e-15)


# ---------------------------------------------------------------- P11 1-D trinomials
@pytest.mark.parametrize("n", [3, 7])
def test_1d_trinomial(oracle_lib, n):
    """P11: ny = nz = 1, untruncated (n ≤ R, far from the ends): the kernel is the
    coefficient list of (1−2λ + λ z + λ z⁻¹)^n (lazy random walk)."""
    lam, R, nx = 0.1, 8, 41
    pb = lat(np.ones((1, 1, nx), np.uint8), R, n)
    W = oracle_lib.kernel(pb, (20, 0, 0))
    poly = np.array([1.0])
    for _ in range(n):
        poly = np.convolve(poly, [lam, 1 - 2 * lam, lam])
    exp = np.zeros(2 * R + 1)
    exp[R - n:R + n + 1] = poly
    np.testing.assert_allclose(W[R, R, :], exp, rtol=0, atol=1e-15)
    assert np.count_nonzero(W) == np.count_nonzero(W[R, R, :])


# ---------------------------------------------------------------- P6 moments
def test_homogeneous_moments(oracle_lib):
    """P6: lazy 3-D random walk moments; centre value = multinomial sum."""
    n, lam, R = 5, 0.1, 5
    pb = lat(np.ones((15, 15, 15), np.uint8), R, n)
    W = oracle_lib.kernel(pb, (7, 7, 7))
    o = np.arange(-R, R + 1, dtype=np.float64)
    Z, Y, X = np.meshgrid(o, o, o, indexing="ij")
    assert W.sum() == pytest.approx(1.0, abs=1e-14)
    assert abs((W * X).sum()) < 1e-15 and abs((W * Y).sum()) < 1e-15 and abs((W * Z).sum()) < 1e-15
    for A in (X, Y, Z):
        assert (W * A ** 2).sum() == pytest.approx(2 * lam * n, rel=1e-13)
        assert (W * A ** 4).sum() == pytest.approx(2 * lam * n + 3 * n * (n - 1) * (2 * lam) ** 2, rel=1e-13)
    assert (W * X ** 2 * Y ** 2).sum() == pytest.approx(n * (n - 1) * (2 * lam) ** 2, rel=1e-13)
    # centre: Σ n!/((a!)²(b!)²(c!)²(n−2a−2b−2c)!) λ^{2(a+b+c)} (1−6λ)^{n−2(a+b+c)}, exact rationals
    L = Fraction(1, 10)
    centre = Fraction(0)
    for a in range(n // 2 + 1):
        for b in range(n // 2 + 1):
            for c in range(n // 2 + 1):
                m = 2 * (a + b + c)
                if m > n:
                    continue
                mult = math.factorial(n) // (math.factorial(a) ** 2 * math.factorial(b) ** 2 *
                                             math.factorial(c) ** 2 * math.factorial(n - m))
                centre += mult * L ** m * (1 - 6 * L) ** (n - m)
    assert W[R, R, R] == pytest.approx(float(centre), rel=1e-13)
    assert float(centre) == pytest.approx(0.06664, abs=5e-6)  # SURVEY P6 value


# ---------------------------------------------------------------- P3/P4 mass & positivity
@pytest.mark.parametrize("n_fd", [2, 40])
def test_kernel_mass_and_positivity(oracle_lib, n_fd):
    """P3: Σ_o W_s(o) = 1 for every source, both regimes (reflecting window, A2);
    P4: W ≥ 0 (maximum principle)."""
    mask = fi.random_two_phase((9, 8, 7), 0.6, seed=5)
    pb = lat(mask, 2, n_fd, D_slow=1e-3)
    W = oracle_lib.build_kernels(pb)
    np.testing.assert_allclose(W.sum(-1), 1.0, rtol=0, atol=1e-13)
    assert W.min() >= 0.0


# ---------------------------------------------------------------- P5 symmetry
def _dense_P(oracle_lib, pb):
    """Dense N×N p (Eq.9): p[i, j] = mass moving j → i."""
    nz, ny, nx = pb.shape
    W = oracle_lib.build_kernels(pb)
    R, L = pb.R, 2 * pb.R + 1
    N = nx * ny * nz
    P = np.zeros((N, N))
    for sz in range(nz):
        for sy in range(ny):
            for sx in range(nx):
                j = (sz * ny + sy) * nx + sx
                Ws = W[sz, sy, sx].reshape(L, L, L)
                for oz in range(-R, R + 1):
                    for oy in range(-R, R + 1):
                        for ox in range(-R, R + 1):
                            x, y, z = sx + ox, sy + oy, sz + oz
                            if 0 <= x < nx and 0 <= y < ny and 0 <= z < nz:
                                P[(z * ny + y) * nx + x, j] = Ws[oz + R, oy + R, ox + R]
    return P


def test_symmetry_regimes(oracle_lib):
    """P5: P = Pᵀ in the exact regime (n_fd ≤ R, self-adjoint FD operator with
    harmonic-mean faces); the reflecting window edges break it when n_fd > R."""
    mask = fi.random_two_phase((7, 6, 5), 0.6, seed=11)
    P = _dense_P(oracle_lib, lat(mask, 2, 2, D_slow=0.05))
    assert np.abs(P - P.T).max() < 1e-15
    np.testing.assert_allclose(P.sum(1), 1.0, atol=1e-14)  # P9: rows sum to 1 too
    Pt = _dense_P(oracle_lib, lat(mask, 2, 30, D_slow=0.05))
    assert np.abs(Pt - Pt.T).max() > 1e-3
    np.testing.assert_allclose(Pt.sum(0), 1.0, atol=1e-13)  # columns still conserve mass


def test_dense_matvec_equals_scatter(oracle_lib):
    """O4 scatter == dense p·c (numpy matmul), Eq.8 with the column convention P:109."""
    mask = fi.random_two_phase((6, 5, 7), 0.5, seed=3)
    pb = lat(mask, 2, 9, D_slow=0.02)
    P = _dense_P(oracle_lib, pb)
    C = fi.initial_c(mask, "random", seed=3).astype(np.float64)
    out = oracle_lib.step_full(pb, C, 1)
    np.testing.assert_allclose(out.ravel(), P @ C.ravel(), rtol=0, atol=1e-15)


# ---------------------------------------------------------------- P1/P2 brute force
def test_exact_regime_equals_whole_grid_fd(oracle_lib):
    """P1: n_fd ≤ R ⇒ one FDiRW step == n_fd whole-grid FD substeps (light cone),
    and s steps == s·n_fd substeps, for any two-phase geometry."""
    mask = fi.random_two_phase((10, 9, 8), 0.55, seed=2)
    for n_fd, R in [(2, 2), (3, 3), (1, 1)]:
        pb = lat(mask, R, n_fd, D_slow=0.01)
        C = fi.initial_c(mask, "random", seed=1).astype(np.float64)
        got = oracle_lib.step_full(pb, C, steps=3)
        ref = oracle_lib.fd_whole_grid(pb, C, 3 * n_fd)
        assert oracle_lib.rel_l2(got, ref) < 1e-14
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-14)  # not resting on rel_l2 alone


def test_window_covering_domain_equals_whole_grid_fd(oracle_lib):
    """P2: R ≥ max dim − 1 ⇒ the window is the whole domain: exact for any n_fd."""
    mask = fi.random_two_phase((4, 5, 3), 0.5, seed=8)
    pb = lat(mask, 4, 60, D_slow=0.03)
    C = fi.initial_c(mask, "random", seed=2).astype(np.float64)
    got = oracle_lib.step_full(pb, C, steps=2)
    ref = oracle_lib.fd_whole_grid(pb, C, 120)
    assert oracle_lib.rel_l2(got, ref) < 1e-13
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-13)


def test_fd_whole_grid_independent(oracle_lib):
    """O6 against an independent numpy formulation of the same closed-domain update
    (array slicing instead of per-cell loops)."""
    mask = fi.random_two_phase((6, 7, 8), 0.5, seed=4)
    pb = lat(mask, 1, 5, D_slow=0.02)
    d = oracle_lib.derive(pb)
    ph = mask.astype(bool)
    C = fi.initial_c(mask, "random", seed=4).astype(np.float64)
    lamtab = {(True, True): d.lam_ff, (False, False): d.lam_ss, (True, False): d.lam_fs, (False, True): d.lam_fs}
    c = C.copy()
    for _ in range(5):
        new = c.copy()
        for ax in range(3):
            a = [slice(None)] * 3
            b = [slice(None)] * 3
            a[ax] = slice(0, -1)
            b[ax] = slice(1, None)
            pa, pbm = ph[tuple(a)], ph[tuple(b)]
            lam = np.where(pa & pbm, d.lam_ff, np.where(~pa & ~pbm, d.lam_ss, d.lam_fs))
            flux = lam * (c[tuple(b)] - c[tuple(a)])
            new[tuple(a)] += flux
            new[tuple(b)] -= flux
        c = new
    ref = oracle_lib.fd_whole_grid(pb, C, 5)
    np.testing.assert_allclose(ref, c, rtol=0, atol=1e-14)
    assert lamtab[(True, False)] == d.lam_fs


def _numpy_closed_fd(ph, c, lam_ff, lam_fs, lam_ss, n):
    """Closed-box explicit FD, array-slicing form (independent of the oracle's C loops)."""
    for _ in range(n):
        new = c.copy()
        for ax in range(3):
            a = [slice(None)] * 3
            b = [slice(None)] * 3
            a[ax] = slice(0, -1)
            b[ax] = slice(1, None)
            pa, pbm = ph[tuple(a)], ph[tuple(b)]
            lam = np.where(pa & pbm, lam_ff, np.where(~pa & ~pbm, lam_ss, lam_fs))
            flux = lam * (c[tuple(b)] - c[tuple(a)])
            new[tuple(a)] += flux
            new[tuple(b)] -= flux
        c = new
    return c


@pytest.mark.parametrize("R,n_fd", [(2, 60), (3, 40)])
def test_truncated_window_equals_boxed_fd(oracle_lib, R, n_fd):
    """Truncated regime (n_fd > R) on a porous two-phase grid: a source's window Ω_s is the
    box [s−R, s+R]³ clipped to the domain, with no flux across its faces (readings A2, A21), so
    W_s must equal a closed-domain FD run from δ_s on that sub-box alone.  Reference: the
    array-slicing FD above on the cut-out mask, λ from Δt/n_fd and the harmonic mean computed
    here; sources at a corner, an edge, a face, the interior and a slow voxel."""
    shape = (12, 11, 13)
    mask = fi.random_two_phase(shape, 0.55, seed=R + 30)
    D_slow = 0.02
    pb = lat(mask, R, n_fd, D_slow=D_slow)
    dt_fd = 0.1 * n_fd / n_fd
    lam_ff, lam_ss = dt_fd * 1.0, dt_fd * D_slow
    lam_fs = dt_fd * 2 * 1.0 * D_slow / (1.0 + D_slow)
    nz, ny, nx = shape
    L = 2 * R + 1
    slow = np.argwhere(mask[R:-R, R:-R, R:-R] == 0)[0] + R
    for sz, sy, sx in [(0, 0, 0), (0, 5, 0), (6, 0, 7), (6, 5, 7), tuple(slow), (nz - 1, ny - 1, nx - 1)]:
        W = oracle_lib.build_kernels(pb, (sx, sx + 1, sy, sy + 1, sz, sz + 1))[0, 0, 0].reshape(L, L, L)
        z0, z1 = max(sz - R, 0), min(sz + R + 1, nz)
        y0, y1 = max(sy - R, 0), min(sy + R + 1, ny)
        x0, x1 = max(sx - R, 0), min(sx + R + 1, nx)
        sub = mask[z0:z1, y0:y1, x0:x1].astype(bool)
        c = np.zeros(sub.shape)
        c[sz - z0, sy - y0, sx - x0] = 1.0
        ref = _numpy_closed_fd(sub, c, lam_ff, lam_fs, lam_ss, n_fd)
        win = W[z0 - sz + R:z1 - sz + R, y0 - sy + R:y1 - sy + R, x0 - sx + R:x1 - sx + R]
        np.testing.assert_allclose(win, ref, rtol=0, atol=1e-14)
        outside = W.copy()
        outside[z0 - sz + R:z1 - sz + R, y0 - sy + R:y1 - sy + R, x0 - sx + R:x1 - sx + R] = 0.0
        assert not outside.any()  # nothing outside the domain
        assert n_fd > R and np.count_nonzero(win) == win.size  # truncated regime: every cell reached


# ---------------------------------------------------------------- P8 impermeable solid
def test_impermeable_slow_phase(oracle_lib):
    """P8 (reading A23): D_slow = 0 ⇒ slow sources keep all their mass (W = δ), and
    mass is conserved per connected fast component."""
    from scipy import ndimage

    mask = fi.random_two_phase((8, 8, 8), 0.5, seed=9)
    pb = lat(mask, 2, 7, D_slow=0.0)
    W = oracle_lib.build_kernels(pb)
    c = (2 * pb.R + 1) ** 3 // 2
    slow = mask == 0
    assert np.all(W[slow][:, c] == 1.0) and np.all(W[slow].sum(-1) == 1.0)
    C = fi.initial_c(mask, "random", seed=9).astype(np.float64)
    out = oracle_lib.step_full(pb, C, 1, )
    lab, n = ndimage.label(mask == 1)
    for k in range(1, n + 1):
        assert out[lab == k].sum() == pytest.approx(C[lab == k].sum(), rel=1e-13)
    np.testing.assert_array_equal(out[slow], C[slow])


# ---------------------------------------------------------------- P9/P10
def test_uniform_and_linearity(oracle_lib):
    """P9 uniform field stationary in the exact regime; P10 linearity."""
    mask = fi.random_two_phase((7, 7, 7), 0.6, seed=12)
    pb = lat(mask, 2, 2, D_slow=0.01)
    out = oracle_lib.step_full(pb, np.full(mask.shape, 0.37), 1)
    np.testing.assert_allclose(out, 0.37, rtol=1e-14)
    pbt = lat(mask, 2, 25, D_slow=0.01)
    W = oracle_lib.build_kernels(pbt)
    box = (0, 7, 0, 7, 0, 7)
    a = fi.initial_c(mask, "random", 1).astype(np.float64)
    b = fi.initial_c(mask, "random", 2).astype(np.float64)
    lhs = oracle_lib.step_scatter(pbt, W, box, 2.5 * a - 0.75 * b, box)
    rhs = 2.5 * oracle_lib.step_scatter(pbt, W, box, a, box) - 0.75 * oracle_lib.step_scatter(pbt, W, box, b, box)
    np.testing.assert_allclose(lhs, rhs, rtol=1e-12, atol=1e-14)
    assert lhs.sum() == pytest.approx((2.5 * a - 0.75 * b).sum(), rel=1e-12)  # mass, truncated regime


# ---------------------------------------------------------------- P12 reflecting window limit
def test_reflecting_window_uniform_limit(oracle_lib):
    """P12: homogeneous reflecting window (fully inside the domain), n_fd → ∞:
    W → 1/K (doubly stochastic symmetric window operator).  R=2, λ=0.1: the
    second eigenvalue is 1−0.2(1−cos(π/5)) ≈ 0.962, so 0.962^1500 ≈ 1e-25."""
    pb = lat(np.ones((9, 9, 9), np.uint8), 2, 1500)
    W = oracle_lib.kernel(pb, (4, 4, 4))
    np.testing.assert_allclose(W, 1.0 / 125, rtol=1e-12)


def test_box_step_equals_full_step(oracle_lib):
    """step_box (sources = target box expanded by R) reproduces the full-grid step
    on the target box, including boxes touching the domain boundary."""
    mask = fi.porous_particle((12, 11, 10), 3.5, pore_r=(1, 1.5), n_pores=3, seed=4)
    pb = lat(mask, 2, 30, D_slow=1e-3)
    C = fi.initial_c(mask, "random", seed=7).astype(np.float64)
    full = oracle_lib.step_full(pb, C, 1)
    for tb in [(0, 4, 0, 5, 0, 3), (3, 10, 2, 9, 4, 12), (6, 10, 8, 11, 9, 12)]:
        part = oracle_lib.step_box(pb, C, tb)
        np.testing.assert_allclose(part, full[tb[4]:tb[5], tb[2]:tb[3], tb[0]:tb[1]], rtol=0, atol=1e-15)


def test_scatter_openmp_bitwise(oracle_lib):
    """The OpenMP scatter (timing form) adds each target's terms in the sequential
    order: bitwise the sequential O4, on a box with clipped sources and on the full grid."""
    mask = fi.porous_particle((14, 12, 13), 4, pore_r=(1, 1.5), n_pores=3, seed=6)
    pb = lat(mask, 2, 40, D_slow=1e-3)
    C = fi.initial_c(mask, "random", seed=6).astype(np.float64)
    for tb in [(0, 13, 0, 12, 0, 14), (3, 11, 2, 6, 5, 9)]:
        sb = oracle_lib.clip_box(pb, (tb[0] - 2, tb[1] + 2, tb[2] - 2, tb[3] + 2, tb[4] - 2, tb[5] + 2))
        W = oracle_lib.build_kernels(pb, sb)
        a = oracle_lib.step_scatter(pb, W, sb, C, tb)
        b = oracle_lib.step_scatter(pb, W, sb, C, tb, threads=True)
        np.testing.assert_array_equal(a, b)
