"""Pins of the N1 coarse-mesh oracle (oracle/coarse.py; Eqs.10-15)."""
import json
import os

import numpy as np
import pytest

import fdirw_inputs as fi

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def co(oracle_lib):
    from oracle import coarse

    return coarse


def lat(mask, n_fd, D_slow=1e-3):
    import oracle

    return oracle.Problem(mask=mask, dh=1.0, D_fast=1.0, D_slow=D_slow, dt=0.1 * n_fd, R=1)


def test_groups_blocks(co):
    g, s = co.groups(np.ones((10, 10, 10), np.uint8), 5)
    assert len(s) == 8 and np.all(s == 125)
    g, s = co.groups(np.ones((5, 5, 5), np.uint8), 5)
    assert len(s) == 1 and s[0] == 125
    reg = np.zeros((6, 7, 11), np.uint8)
    reg[0, 0, 0] = reg[5, 6, 10] = reg[2, 3, 4] = 1
    g, s = co.groups(reg, 5)
    assert len(s) == 2 and list(s) == [2, 1] and g[0, 0, 0] == g[2, 3, 4] == 0 and g[5, 6, 10] == 1
    assert np.all(g[reg == 0] == -1)


def test_map_remap(co):
    reg = np.zeros((1, 1, 4), np.uint8) + 1
    g, s = co.groups(reg, 5)
    C = co.map_fine_to_coarse(np.array([[[1.0, 2.0, 3.0, 4.0]]]), g, s)
    assert C[0] == 2.5
    rng = np.random.default_rng(0)
    reg = fi.random_two_phase((12, 11, 13), 0.7, seed=1)
    g, s = co.groups(reg, 5)
    c = rng.random(reg.shape)
    C = co.map_fine_to_coarse(c, g, s)
    pc = co.remap_coarse_to_fine(C, g, c)
    np.testing.assert_allclose(co.map_fine_to_coarse(pc, g, s), C, rtol=1e-14)       # map∘remap = id
    np.testing.assert_allclose(co.remap_coarse_to_fine(co.map_fine_to_coarse(pc, g, s), g, pc), pc, rtol=1e-14)
    assert pc[reg == 1].sum() == pytest.approx(c[reg == 1].sum(), rel=1e-13)     # "explicitly conserve"
    np.testing.assert_array_equal(pc[reg == 0], c[reg == 0])


def test_P_invariants(co):
    """Row sums 1 (uniform field stationary), column mass Σ_I N_I P_IJ = N_J (closed
    domain), P ≥ 0; a single sealed group gives P = [[1]]."""
    mask = fi.porous_particle((16, 15, 17), 4, pore_r=(1, 1.5), n_pores=3, seed=2)
    reg = fi.near_field(mask, 4, margin=3)
    pb = lat(mask, 60)
    P, g, s = co.build_P(pb, reg, b=3)
    assert P.shape[0] == len(s) > 10
    np.testing.assert_allclose(P.sum(1), 1.0, atol=1e-12)
    np.testing.assert_allclose(s @ P, s, rtol=1e-12)
    assert P.min() >= 0
    one = np.ones((4, 4, 4), np.uint8)
    P1, _, _ = co.build_P(lat(one, 30), one, b=5)
    np.testing.assert_allclose(P1, [[1.0]], atol=1e-14)


def test_P_b1_equals_fine_operator(co, oracle_lib):
    """b = 1: each group one voxel, so P is the fine FD operator over Ω_L — the same
    matrix the windowed-kernel path gives when the window covers the domain (P2
    regime): two independent oracle code paths (oracle_kernel vs oracle_fd_whole_grid)."""
    reg = fi.random_two_phase((4, 3, 5), 0.7, seed=3)
    pb = lat(np.ones_like(reg), 25)
    P, g, s = co.build_P(pb, reg, b=1)
    kp = oracle_lib.Problem(mask=reg, dh=1.0, D_fast=1.0, D_slow=0.0, dt=0.1 * 25, R=5)
    W = oracle_lib.build_kernels(kp)
    L, R = 11, 5
    idx = np.argwhere(reg == 1)  # group order == voxel order for b = 1
    for J, (sz, sy, sx) in enumerate(idx):
        Wk = W[sz, sy, sx].reshape(L, L, L)
        for I, (z, y, x) in enumerate(idx):
            assert P[I, J] == pytest.approx(Wk[z - sz + R, y - sy + R, x - sx + R], abs=1e-14)


def test_groupwise_constant_exact(co, oracle_lib):
    """for a group-wise constant field the coarse step equals the mapped
    fine FD evolution over Δt (linearity of the columns)."""
    mask = fi.porous_particle((14, 14, 14), 4, pore_r=(1, 1.5), n_pores=2, seed=5)
    reg = fi.near_field(mask, 4, margin=2)
    pb = lat(mask, 40)
    P, g, s = co.build_P(pb, reg, b=4)
    rng = np.random.default_rng(1)
    C = rng.random(len(s))
    c = co.remap_coarse_to_fine(C, g, np.zeros(mask.shape))
    fine = oracle_lib.fd_whole_grid(co.region_problem(pb, reg), c, 40)
    np.testing.assert_allclose(P @ C, co.map_fine_to_coarse(fine, g, s), rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(co.step(P, g, s, c)[reg == 1],
                               co.remap_coarse_to_fine(co.map_fine_to_coarse(fine, g, s), g, c)[reg == 1], rtol=1e-12)


@pytest.mark.parametrize("fmt", ["fp32", "fp16", "bf16"])
def test_quantize_P_mass(co, fmt):
    mask = fi.porous_particle((12, 12, 12), 3, pore_r=(1, 1.5), n_pores=2, seed=6)
    reg = fi.near_field(mask, 3, margin=2)
    P, g, s = co.build_P(lat(mask, 50), reg, b=3)
    Q = co.quantize_P(P, s, fmt)
    np.testing.assert_allclose(s @ Q, s, rtol=2e-7)
    off = ~np.eye(len(s), dtype=bool)
    assert np.abs(Q[off] - P[off]).max() <= {"fp32": 1e-7, "fp16": 1e-3, "bf16": 4e-3}[fmt]


def test_flop_model_table3(co):
    """§4.3 FLOP model N(N+1)+2N_L on Table 3's counts."""
    t3 = json.load(open(os.path.join(GOLD, "table3.json")))
    for k in ("R25", "R50"):
        assert co.flop_count(t3[k]["N"], t3[k]["N_L"]) == t3[k]["flops"]


def test_near_field_region():
    """P:40 near-field = liquid within r_p + 5Δh (inclusive); our R50
    particle reproduces Table 3's R50 counts within 5 % (statistical similarity)."""
    m = np.ones((1, 1, 40), np.uint8)
    nf = fi.near_field(m, 10.0, center=(0.0, 0.0, 0.0))
    assert nf[0, 0, 15] == 1 and nf[0, 0, 16] == 0          # distance exactly 15 is inside
    t3 = json.load(open(os.path.join(GOLD, "table3.json")))["R50"]
    mask = fi.config("cfg3").mask()
    n_l = int(fi.near_field(mask, 50).sum())
    n_s = int((mask == 0).sum())
    assert abs(n_l - t3["N_L"]) / t3["N_L"] < 0.05 and abs(n_s - t3["N_S"]) / t3["N_S"] < 0.05


def test_coarse_far_field(co, oracle_lib):
    """N1 + N2 (Eq.10 with P_BC): the row-sum identity Σ_J P_IJ + P_BC_I = 1 (SPEC S:318,
    S:330), a uniform field with c_far equal to it is stationary, and b = 1 reproduces the
    held-Dirichlet fine FD exactly (linearity in (c, c_far))."""
    mask = fi.porous_particle((14, 15, 13), 4, pore_r=(1, 1.5), n_pores=2, seed=3)
    region = fi.with_far_field(mask, 4, 2.0)            # 1 near liquid, 2 far, 0 solid
    region = np.where(region == 0, 0, region).astype(np.uint8)
    pb = lat(mask, 40)
    P, g, s = co.build_P(pb, region, b=3)
    PBC = co.build_PBC(pb, region, b=3)
    np.testing.assert_allclose(P.sum(1) + PBC, 1.0, atol=1e-12)
    assert PBC.max() > 1e-3 and PBC.min() >= 0
    c = np.where(region == 1, 0.6, 0.0)
    np.testing.assert_allclose(co.step_far(P, PBC, g, s, c, 0.6)[region == 1], 0.6, rtol=1e-12)
    Q = co.quantize_P(P, s, "bf16")
    np.testing.assert_allclose(s @ Q, s @ P, rtol=2e-7)   # column masses kept (A10 generalised)
    # b = 1: P·c + P_BC·c_far == fine FD with the far field held at c_far
    reg = np.zeros((5, 4, 6), np.uint8)
    reg[1:4, 1:3, 1:5] = 1
    reg[0] = 2
    P1, g1, s1 = co.build_P(lat(np.ones_like(reg), 25), reg, b=1)
    B1 = co.build_PBC(lat(np.ones_like(reg), 25), reg, b=1)
    c1 = np.where(reg == 1, np.random.default_rng(0).random(reg.shape), 0.0)
    got = co.step_far(P1, B1, g1, s1, c1, 0.3)
    ref = oracle_lib.fd_whole_grid(co.region_problem(lat(np.ones_like(reg), 25), reg), c1, 25, c_far=0.3)
    np.testing.assert_allclose(got[reg == 1], ref[reg == 1], rtol=1e-12)
