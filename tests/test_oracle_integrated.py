"""Pins of the N3 oracle (oracle/integrated.py): Eqs.4-6 worked examples, the interface
exchange in closed form, conservation of the integrated loop (Eq.7), absorption kinetics
monotonicity and the precision-mode error ordering of §4.2 (Figs.8-10)."""
import numpy as np
import pytest

import fdirw_inputs as fi


@pytest.fixture(scope="module")
def ig(oracle_lib):
    from oracle import integrated

    return integrated


def _ab(ig, **kw):
    T = fi.TABLE1
    d = dict(D_L=fi.D_FAST_SI, D_S=fi.D_SLOW_SI, dh=T["dh"], dt=T["dt"], k=0.05, c_S_eq=1.0, c_L_eq=1e-5,
             V_far=2e4, R=3)
    d.update(kw)
    return ig.Absorb(**d)


def test_eq4_6_examples(ig):
    """SPEC S:124-126 hand evaluations of Eqs.4-6 (k = 0.05)."""
    ab = _ab(ig)
    r, rl = ig.rate(np.array([ab.c_L_eq]), np.array([0.0]), ab)
    assert r[0] == 0.0 and rl[0] == 0.0                                      # c_L = c_eq → 0
    r, rl = ig.rate(np.array([2 * ab.c_L_eq]), np.array([0.0]), ab)
    assert r[0] == pytest.approx(0.05) and rl[0] == pytest.approx(-0.05)     # f_L = f_S = 1
    r, _ = ig.rate(np.array([2 * ab.c_L_eq]), np.array([0.25]), ab)
    assert r[0] == pytest.approx(0.0375)
    r, _ = ig.rate(np.array([1.0]), np.array([1.5]), ab)
    assert r[0] == 0.0                                                       # no desorption (f_S clamp)


def test_react_two_voxels(ig):
    """One solid|liquid face: the solid gains exactly k·f_L·f_S·Δt, the liquid loses it;
    with a huge k the liquid stops exactly at c_L^eq (clamp, A29)."""
    mask = np.array([[[0, 1]]], np.uint8)
    ab = _ab(ig, dt=1e-4)  # q = 8e-6 < c_l − c_eq = 2e-5: no clamp
    c = np.array([[[0.2, 3e-5]]])
    out = ig.react(c, mask, ab)
    q = ab.k * ((3e-5 - 1e-5) / 1e-5) * ((1.0 - 0.2) / 1.0) * ab.dt
    assert out[0, 0, 0] == pytest.approx(0.2 + q, rel=1e-14)
    assert out[0, 0, 1] == pytest.approx(3e-5 - q, rel=1e-12)
    big = ig.react(c, mask, _ab(ig, k=1e6))
    assert big[0, 0, 1] == pytest.approx(1e-5, rel=1e-12)
    assert big.sum() == pytest.approx(c.sum(), rel=1e-15)
    # two solids sharing one liquid voxel: both transfers scaled by the same factor
    mask3 = np.array([[[0, 1, 0]]], np.uint8)
    c3 = np.array([[[0.0, 3e-5, 0.5]]])
    o3 = ig.react(c3, mask3, _ab(ig, k=1e6))
    assert o3[0, 0, 1] == pytest.approx(1e-5, rel=1e-12)
    assert (o3[0, 0, 0] - 0.0) / (o3[0, 0, 2] - 0.5) == pytest.approx(1.0 / 0.5, rel=1e-9)  # ∝ f_S


def test_solid_fd_only_moves_solid_mass(ig):
    mask = fi.random_two_phase((6, 7, 8), 0.5, seed=2)
    c = fi.initial_c(mask, "random", seed=2).astype(np.float64)
    ab = _ab(ig)
    out = ig.solid_fd(c, mask, ab)
    np.testing.assert_array_equal(out[mask == 1], c[mask == 1])
    assert out[mask == 0].sum() == pytest.approx(c[mask == 0].sum(), rel=1e-14)


@pytest.fixture(scope="module")
def desk(ig):
    """A small porous particle in its near field, Table 1 SI parameters (20³, r_p = 6, R = 3)."""
    shape = (20, 20, 20)
    m = fi.with_far_field(fi.porous_particle(shape, 6, pore_r=(1.0, 2.0), porosity=0.3, seed=3), 6, 3.0)
    T = fi.TABLE1
    c0 = np.where(m == 1, T["c_L0"], np.where(m == 0, T["c_S0"], 0.0))
    ab = _ab(ig)
    runs = {mode: ig.run(m, c0, T["c_L0"], ab, 30, mode) for mode in ("fp64", "fp32", "mixed", "fp16")}
    return m, c0, ab, runs


def test_loop_conservation_and_kinetics(ig, desk):
    """Eq.7: Σc + c_far·V_far = Σc_{S+L}(t0) after every step; Q_S non-decreasing under
    Table 1 parameters; c_far non-increasing."""
    m, c0, ab, runs = desk
    c, cf, kin = runs["fp64"]
    M0 = float(c0.sum()) + fi.TABLE1["c_L0"] * ab.V_far
    assert c.sum() + cf * ab.V_far == pytest.approx(M0, rel=1e-13)
    QS = np.array([k[0] for k in kin])
    far = np.array([k[2] for k in kin])
    assert np.all(np.diff(QS) >= 0) and QS[-1] > QS[0]
    assert np.all(np.diff(far) <= 1e-18)


def test_precision_error_ordering(desk):
    """§4.2 / Fig.10: RE of c̄_S vs FP64 orders FP32 < mixed FP32/FP16 < FP16;
    FP32 ≈ 1e-9-level here, mixed within 1e-3 (the paper: FP32 ~1e-6, mixed ~1e-5, FP16 ~1e-2
    at N = 2515; this desk model has K = 343 terms per sum)."""
    _, _, _, runs = desk
    ref = np.array([k[3] for k in runs["fp64"][2]])
    re = {mode: np.max(np.abs(np.array([k[3] for k in runs[mode][2]]) - ref) / ref)
          for mode in ("fp32", "mixed", "fp16")}
    assert re["fp32"] < re["mixed"] < re["fp16"]
    assert re["fp32"] < 1e-6 and re["mixed"] < 1e-3
