"""Host logic of kgen's Chebyshev evaluation (reading A30), no GPU needed.

After 8 direct substeps the library picks the degree m of p_m(y) = Σ_{k≤m} c_k T_k(y) ≈ x^n, x = αy + β on the window
spectrum [1 − 12λ_max, 1] (α = 6λ_max, β = 1 − 6λ_max), as the smallest m whose tail
Σ_{k>m} c_k ≤ 1e-10; it computes the c_k by a discrete Chebyshev transform.  This test
derives the same c_k a different way — as a probability: x^n = E[T_{|S_J|}(y)] where
J ~ Binomial(n, α) and S_J is a ±1 random walk of J steps (y^j = 2^{-j} Σ_i C(j,i) T_{|j−2i|}),
so c_k = P(|S_J| = k) ≥ 0 and Σ c_k = 1 — and checks the library's m against it."""
import math

import numpy as np
import pytest

import fdirw_inputs as fi
from _util import lib_params


def _walk_coeffs(n, lam_max):
    """c_k = P(|S_J| = k), J ~ Bin(n, 6λ), S a simple ±1 walk (fp64, log-space binomials)."""
    al = 6.0 * lam_max
    j = np.arange(n + 1)
    lg = np.array([math.lgamma(n + 1) - math.lgamma(i + 1) - math.lgamma(n - i + 1) for i in j])
    with np.errstate(divide="ignore"):
        pj = np.exp(lg + j * math.log(al) + (n - j) * math.log1p(-al))
    c = np.zeros(n + 1)
    dist = np.zeros(2 * n + 1)  # position of the walk after j steps, offset n
    dist[n] = 1.0
    for jj in range(n + 1):
        if jj:
            dist = 0.5 * (np.roll(dist, 1) + np.roll(dist, -1))
        if pj[jj] < 1e-300:
            continue
        pos = np.abs(np.arange(2 * n + 1) - n)
        np.add.at(c, pos, pj[jj] * dist)
    return c


def test_walk_coeffs_reproduce_power():
    """The pin itself: Σ c_k T_k(y) == x^n on [a, 1] (n small enough to sum every term)."""
    n, lam = 40, 0.1
    c = _walk_coeffs(n, lam)
    assert np.all(c >= 0) and abs(c.sum() - 1.0) < 1e-12
    x = np.linspace(1 - 12 * lam, 1.0, 101)
    y = (x - (1 - 6 * lam)) / (6 * lam)
    p = np.polynomial.chebyshev.chebval(y, c)
    np.testing.assert_allclose(p, x ** n, rtol=1e-10, atol=1e-14)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg5"])
def test_library_degree_matches_random_walk_tail(fd_cpu, name):
    cfg = fi.config(name)
    pl = fd_cpu.make_plan(lib_params(cfg))
    n = pl["n_fd"]
    assert n == 1000
    # λ_max = D_max Δt_fd / Δh² (Table 1: 0.1 for every preset)
    lam = max(cfg.D_fast, cfg.D_slow) * cfg.dt / n / cfg.dh ** 2
    pre = 8  # direct substeps before the recurrence (fdirw_api.cu kCheb_pre)
    c = _walk_coeffs(n - pre, lam)
    tail = 1.0 - np.cumsum(c)
    m = pl["kgen_steps"] - pre
    assert 100 < m < 300, m
    assert tail[m] <= 1.2e-10 and tail[m - 1] > 0.8e-10, (m, tail[m - 1], tail[m])
    # the FDIRW_F_KGEN_DIRECT flag (and FP64) keep the n_fd literal substeps
    assert fd_cpu.make_plan(lib_params(cfg, flags=fd_cpu.F_KGEN_DIRECT))["kgen_steps"] == n
    assert fd_cpu.make_plan(lib_params(cfg, flags=fd_cpu.F_KGEN_FP64))["kgen_steps"] == n


@pytest.mark.parametrize("n_fd", [2, 5, 20, 40])
def test_small_n_stays_direct(fd_cpu, n_fd):  # (n_fd ≤ 16 is always direct)
    """Where the recurrence would not save ≥ 20 % of the lane-ops, kgen keeps the substeps
    (so the exact-regime pin P1, n_fd ≤ R, runs the literal FD)."""
    pl = fd_cpu.make_plan(lib_params(fi.config("cfg1", n_fd=n_fd)))
    assert pl["kgen_steps"] == n_fd
