"""Pins of the N2 far-field oracle (oracle/farfield.py; Eq.7, Eq.8)."""
import numpy as np
import pytest

import fdirw_inputs as fi


@pytest.fixture(scope="module")
def ff(oracle_lib):
    from oracle import farfield

    return farfield


def lat(mask, R, n_fd, D_slow=1e-2):
    import oracle

    return oracle.Problem(mask=mask, dh=1.0, D_fast=1.0, D_slow=D_slow, dt=0.1 * n_fd, R=R)


def _open_mask(shape, seed):
    """solid/liquid with a far-field region (code 2) outside a sphere — the paper's layout."""
    m = fi.random_two_phase(shape, 0.6, seed=seed)
    nz, ny, nx = shape
    z, y, x = np.ogrid[0:nz, 0:ny, 0:nx]
    r2 = (x - (nx - 1) / 2) ** 2 + (y - (ny - 1) / 2) ** 2 + (z - (nz - 1) / 2) ** 2
    m[(r2 > (min(shape) / 2 - 1) ** 2) & (m == 1)] = 2
    return m


@pytest.mark.parametrize("n_fd,R", [(2, 2), (3, 3)])
def test_exact_regime_equals_dirichlet_fd(ff, oracle_lib, n_fd, R):
    """n_fd ≤ R: Eq.8 with p_BC = 1 − row sum equals n_fd whole-grid FD substeps with the
    far field held at c_far (light cone) — pins the absorbing kernels, the p_BC reading
    and the step together."""
    m = _open_mask((10, 11, 9), 3)
    assert (m == 2).any()
    pb = lat(m, R, n_fd)
    C = fi.initial_c(m, "random", seed=2).astype(np.float64) * (m != 2)
    W = oracle_lib.build_kernels(pb)
    pbc = ff.p_bc_full(pb, W)
    got = ff.step_full(pb, W, C, 0.37, pbc)
    ref = oracle_lib.fd_whole_grid(pb, C, n_fd, c_far=0.37) * (m != 2)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-14)


@pytest.mark.parametrize("n_fd,R", [(2, 2), (3, 4)])
def test_p_bc_reservoir_equals_row_sum_reading_where_exact(ff, oracle_lib, n_fd, R):
    """The alternative p_BC reading (the reservoir's held-Dirichlet FD response) equals A26's
    1 − row sum where the windows are exact (n_fd ≤ R); it is in [0, 1] and 0 on voxels farther
    than n_fd faces from the reservoir."""
    m = _open_mask((10, 11, 9), 3)
    pb = lat(m, R, n_fd)
    W = oracle_lib.build_kernels(pb)
    a, b = ff.p_bc_reservoir(pb), ff.p_bc_full(pb, W)
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-14)
    assert a.min() >= 0.0 and a.max() <= 1.0
    far = np.argwhere(m == 2)
    for idx in np.argwhere((m != 2)):
        if np.abs(far - idx).sum(1).min() > n_fd:
            assert a[tuple(idx)] == 0.0


def test_p_bc_reservoir_nonnegative_truncated(ff, oracle_lib):
    """In the truncated regime the two readings part: A26's 1 − row sum goes negative at targets
    whose row sum exceeds 1, the reservoir reading stays in [0, 1]."""
    m = _open_mask((12, 13, 11), 5)
    pb = lat(m, 2, 40)
    W = oracle_lib.build_kernels(pb)
    a, b = ff.p_bc_reservoir(pb), ff.p_bc_full(pb, W)
    assert a.min() >= 0.0 and a.max() <= 1.0
    assert np.abs(a - b).max() > 1e-3


def test_window_covering_domain_equals_dirichlet_fd(ff, oracle_lib):
    m = _open_mask((5, 4, 6), 4)
    pb = lat(m, 5, 70)
    C = fi.initial_c(m, "random", seed=3).astype(np.float64) * (m != 2)
    W = oracle_lib.build_kernels(pb)
    got = ff.step_full(pb, W, C, 0.81, ff.p_bc_full(pb, W))
    ref = oracle_lib.fd_whole_grid(pb, C, 70, c_far=0.81) * (m != 2)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-13)


def test_uniform_stationary_and_eq7(ff, oracle_lib):
    """Truncated regime: c ≡ c_far ≡ κ is stationary (row-sum identity);
    Eq.7 closes the global balance exactly (SPEC S:134 arithmetic example)."""
    m = _open_mask((9, 10, 11), 5)
    pb = lat(m, 2, 40)
    W = oracle_lib.build_kernels(pb)
    pbc = ff.p_bc_full(pb, W)
    C = 0.7 * (m != 2).astype(np.float64)
    np.testing.assert_allclose(ff.step_full(pb, W, C, 0.7, pbc)[m != 2], 0.7, rtol=1e-13)
    assert ff.far_update(100.0, np.array([30.0, 20.0]), 25.0) == 2.0
    C0 = fi.initial_c(m, "random", seed=6)
    Cn, cf, M0 = ff.run_full(pb, C0, 0.25, 1e3, 4)
    assert Cn.sum() + cf * 1e3 == pytest.approx(M0, rel=1e-14)
    assert np.all(Cn[m == 2] == 0)


def test_absorbing_kernel_mass(oracle_lib):
    """Windows touching the reservoir lose mass to it; closed windows keep Σ W = 1; the
    quantised columns keep each kernel's own mass M (A10 generalised)."""
    m = _open_mask((9, 9, 9), 7)
    pb = lat(m, 2, 30)
    W = oracle_lib.build_kernels(pb)
    ow = oracle_lib.open_windows(pb)
    s = W.sum(-1)
    src = m != 2
    assert np.all(s[src & ~ow] == pytest.approx(1.0, abs=1e-13))
    assert np.all(s[src & ow] < 1.0 - 1e-6)
    assert np.all(W[m == 2] == 0)
    for fmt in ("fp32", "bf16", "fp16"):
        Wq = oracle_lib.quantize(pb, W, fmt)
        np.testing.assert_allclose(Wq.sum(-1)[src], s[src], atol=1e-14)
