"""GPU parity of NEXT row N3 — the integrated absorption loop (Eqs.1-7) and the §3.3
precision modes (Figs.8-10) — against oracle/integrated.py, through the C-ABI."""
import numpy as np
import pytest

import fdirw_inputs as fi
from _util import rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fd():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import __graft_entry__

    __graft_entry__.build()
    import paper_2408_11376_b200 as fd

    return fd


@pytest.fixture(scope="module")
def desk(oracle_lib):
    """The oracle's desk model: 20³, r_p = 6 particle, near field r_p + 3, Table 1 SI values."""
    from oracle import integrated as ig

    shape = (20, 20, 20)
    m = fi.with_far_field(fi.porous_particle(shape, 6, pore_r=(1.0, 2.0), porosity=0.3, seed=3), 6, 3.0)
    T = fi.TABLE1
    c0 = np.where(m == 1, T["c_L0"], np.where(m == 0, T["c_S0"], 0.0))
    ab = ig.Absorb(D_L=fi.D_FAST_SI, D_S=fi.D_SLOW_SI, dh=T["dh"], dt=T["dt"], k=0.05, c_S_eq=1.0, c_L_eq=1e-5,
                   V_far=2e4, R=3)
    runs = {mode: ig.run(m, c0, T["c_L0"], ab, 20, mode) for mode in ("fp64", "fp32", "mixed", "fp16")}
    return m, c0, ab, runs


def _gpu(fd, m, c0, ab, weights, mode, steps=20):
    import torch

    nz, ny, nx = m.shape
    p = fd.Params(nx=nx, ny=ny, nz=nz, dh=ab.dh, D_fast=ab.D_L, D_slow=0.0, dt=ab.dt, radius=ab.R, weights=weights,
                  v_far=ab.V_far, flags=fd.F_NO_MASS_FIX if mode != "default" else 0)
    ctx = fd.build_kernels(p, m)
    try:
        c = torch.from_numpy(c0.astype(np.float32)).cuda()
        M0 = fd.far_init(ctx, c, fi.TABLE1["c_L0"])
        fd.set_precision_mode(ctx, mode)
        kin = fd.absorb_run(ctx, c, steps, ab.D_S, ab.k, ab.c_S_eq, ab.c_L_eq)
        return c.cpu().numpy().astype(np.float64), kin, M0
    finally:
        fd.destroy(ctx)


def test_absorb_loop_vs_oracle(fd, desk):
    """Default product path (fp32 weights): field, kinetics (Q_S, c̄_S, c_far) and the Eq.7
    balance vs the oracle's fp64 loop."""
    m, c0, ab, runs = desk
    got, kin, M0 = _gpu(fd, m, c0, ab, "fp32", "default")
    ref, refcf, refkin = runs["fp64"]
    nf = m != 2
    assert rel_l2(got[nf], ref[nf]) <= 1e-5
    rk = np.array(refkin)
    np.testing.assert_allclose(kin[:, 0], rk[:, 0], rtol=1e-5)           # Q_S(t)
    np.testing.assert_allclose(kin[:, 3], rk[:, 3], rtol=1e-5)           # c̄_S(t)
    np.testing.assert_allclose(kin[:, 2], rk[:, 2], rtol=1e-5)           # c_far(t)
    assert np.all(np.diff(kin[:, 0]) >= -1e-9 * kin[0, 0])               # absorption only
    tot = got[nf].sum() + kin[-1, 2] * ab.V_far
    assert abs(tot - M0) / M0 <= 1e-6


def test_precision_modes_vs_oracle(fd, desk):
    """The paper's FP32 / mixed FP32-FP16 / FP16 modes on the GPU track the oracle's
    emulation of the same modes, and keep the §4.2 ordering of the error in c̄_S vs FP64."""
    m, c0, ab, runs = desk
    ref = np.array([k[3] for k in runs["fp64"][2]])
    re = {}
    for mode, w in (("fp32", "fp32"), ("mixed", "fp16"), ("fp16", "fp16")):
        _, kin, _ = _gpu(fd, m, c0, ab, w, mode)
        emu = np.array([k[3] for k in runs[mode][2]])
        re[mode] = np.max(np.abs(kin[:, 3] - ref) / ref)
        tol = {"fp32": 1e-5, "mixed": 5e-4, "fp16": 5e-3}[mode]
        assert np.max(np.abs(kin[:, 3] - emu) / emu) <= tol, mode
    assert re["fp32"] < re["mixed"] < re["fp16"]


def test_absorb_run_replay_consistent(fd, desk):
    """fdirw_absorb_run replays a captured two-macro-step graph (round 2): 7 + 6 steps in two
    calls (an odd tail, the graph reused) give the field and kinetics of 13 steps in one call
    bit for bit; changing a loop parameter between calls recaptures (a fresh context agrees)."""
    import torch

    m, c0, ab, _ = desk
    nz, ny, nx = m.shape
    p = fd.Params(nx=nx, ny=ny, nz=nz, dh=ab.dh, D_fast=ab.D_L, D_slow=0.0, dt=ab.dt, radius=ab.R, weights="bf16",
                  v_far=ab.V_far)

    def run(chunks, ks):
        ctx = fd.build_kernels(p, m)
        try:
            c = torch.from_numpy(c0.astype(np.float32)).cuda()
            fd.far_init(ctx, c, fi.TABLE1["c_L0"])
            kins = [fd.absorb_run(ctx, c, n, ab.D_S, k, ab.c_S_eq, ab.c_L_eq) for n, k in zip(chunks, ks)]
            return c.cpu().numpy(), np.concatenate(kins)
        finally:
            fd.destroy(ctx)

    a_c, a_k = run([13], [ab.k])
    b_c, b_k = run([7, 6], [ab.k, ab.k])
    np.testing.assert_array_equal(a_c, b_c)
    np.testing.assert_array_equal(a_k, b_k)
    # a parameter change between calls (k) must not replay the old graph
    c1, k1 = run([4, 4], [ab.k, 2 * ab.k])
    ctx = fd.build_kernels(p, m)
    try:
        c = torch.from_numpy(c0.astype(np.float32)).cuda()
        fd.far_init(ctx, c, fi.TABLE1["c_L0"])
        fd.absorb_run(ctx, c, 4, ab.D_S, ab.k, ab.c_S_eq, ab.c_L_eq)
        ctx2 = fd.build_kernels(p, m)
        try:
            # the second half on a context that never saw the first k: same result
            fd.far_init(ctx2, c, float(fd.far_get(ctx)))
            kk = fd.absorb_run(ctx2, c, 4, ab.D_S, 2 * ab.k, ab.c_S_eq, ab.c_L_eq)
        finally:
            fd.destroy(ctx2)
    finally:
        fd.destroy(ctx)
    np.testing.assert_allclose(c1, c.cpu().numpy(), rtol=1e-6, atol=1e-12)
    np.testing.assert_allclose(k1[4:, :2], kk[:, :2], rtol=1e-6)


def test_absorb_loop_many_tail_blocks(fd, oracle_lib):
    """A grid whose tail sweeps launch more than 592 blocks (56³: 686): the kinetics partial sums
    (2 doubles per block, up to kAbsorbMaxBlocks blocks) must fit their buffer.  Round 2's first
    replay version sized it for 592 blocks, so at cfg3o (2,368 blocks) react_apply wrote past it
    into far_state and the bench line's c_far / mass balance were garbage.  Checked against the
    oracle's fp64 loop (3 steps), the record against the returned field, and Eq.7's balance."""
    import torch
    from oracle import integrated as ig

    shape = (56, 56, 56)
    m = fi.with_far_field(fi.porous_particle(shape, 18, pore_r=(1.0, 2.0), porosity=0.3, seed=5), 18, 3.0)
    T = fi.TABLE1
    c0 = np.where(m == 1, T["c_L0"], np.where(m == 0, T["c_S0"], 0.0))
    ab = ig.Absorb(D_L=fi.D_FAST_SI, D_S=fi.D_SLOW_SI, dh=T["dh"], dt=T["dt"], k=0.05, c_S_eq=1.0, c_L_eq=1e-5,
                   V_far=2e5, R=3)
    steps = 3
    ref, _, refkin = ig.run(m, c0, T["c_L0"], ab, steps, "fp64")
    got, kin, M0 = _gpu(fd, m, c0, ab, "fp32", "default", steps=steps)
    nf = m != 2
    assert rel_l2(got[nf], ref[nf]) <= 1e-5
    np.testing.assert_allclose(kin, np.array(refkin), rtol=1e-5)
    np.testing.assert_allclose(kin[-1, 0], got[m == 0].sum(), rtol=1e-9)   # Q_S of the returned field
    np.testing.assert_allclose(kin[-1, 1], got[m == 1].sum(), rtol=1e-9)   # Q_L
    tot = got[nf].sum() + kin[-1, 2] * ab.V_far
    assert abs(tot - M0) / M0 <= 1e-6


@pytest.mark.parametrize("D_S,weights", [(fi.D_SLOW_SI, "fp32"), (0.0, "fp32"), (fi.D_SLOW_SI, "bf16")])
def test_absorb_grouped_tail_bitwise(fd, monkeypatch, D_S, weights):
    """The tail over groups of 4 x-voxels — by default (one solid pass) the liquid step skips its
    identity-chunk copy and the solid pass visits only the non-far groups, reading the solid values
    from the step's input; α / the apply / its in-place scatter visit only the interface groups
    (FDIRW_ABSORB_FULL=1: the solid pass sweeps the grid instead; FDIRW_ABSORB_SWEEP=1 sweeps all
    three) — against the per-voxel sweeps (FDIRW_ABSORB_SCALAR=1): every voxel's
    value is the same expression in the same face order, so one macro step's field is bitwise
    equal; the kinetics partials are summed per thread-group (another fixed order), so Q_S, Q_L,
    c_far agree to rounding, and after that c_far feeds the next step's p_BC·c_far term.  nx = 37
    (a ragged last group), R = 2, and the loop without a solid pass (D_S = 0)."""
    import torch

    shape = (23, 29, 37)
    m = fi.with_far_field(fi.porous_particle(shape, 8, pore_r=(1.0, 2.0), porosity=0.3, seed=7), 8, 2.0)
    T = fi.TABLE1
    c0 = np.where(m == 1, T["c_L0"], np.where(m == 0, T["c_S0"], 0.0)).astype(np.float32)
    nz, ny, nx = shape
    p = fd.Params(nx=nx, ny=ny, nz=nz, dh=T["dh"], D_fast=fi.D_FAST_SI, D_slow=0.0, dt=T["dt"], radius=2,
                  weights=weights, v_far=2e4)
    out = {}
    for form in ("default", "full", "sweep", "scalar"):
        for ev in ("FDIRW_ABSORB_SCALAR", "FDIRW_ABSORB_SWEEP", "FDIRW_ABSORB_FULL"):
            monkeypatch.delenv(ev, raising=False)
        if form != "default":
            monkeypatch.setenv("FDIRW_ABSORB_" + form.upper(), "1")
        ctx = fd.build_kernels(p, m)
        try:
            c = torch.from_numpy(c0).cuda()
            fd.far_init(ctx, c, T["c_L0"])
            k1 = fd.absorb_run(ctx, c, 1, D_S, 0.05, 1.0, 1e-5)
            c1 = c.cpu().numpy()
            k5 = fd.absorb_run(ctx, c, 5, D_S, 0.05, 1.0, 1e-5)
            out[form] = (c1, k1, c.cpu().numpy(), k5)
        finally:
            fd.destroy(ctx)
    b = out["scalar"]
    for a in (out["default"], out["full"], out["sweep"]):
        assert np.count_nonzero(a[0] != c0) > 0  # the step moved the field
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_allclose(a[1], b[1], rtol=1e-12)
        np.testing.assert_allclose(a[2], b[2], rtol=1e-6, atol=1e-12)
        np.testing.assert_allclose(a[3], b[3], rtol=1e-9)


def test_isolated_sources_exact_delta(fd):
    """With D_slow = 0 a solid voxel's every face number is 0: its kernel is exactly δ (kgen runs no
    pass for it — the Chebyshev recurrence would give Σ fp32(c_k)·δ, and an open window, which is
    not renormalised, would keep that as its mass: the identity rows of the N3 loop's liquid step
    would leak).  bf16 storage (open windows by the recurrence), R = 5 and 8, with a reservoir."""
    for R, shape in ((5, (22, 21, 23)), (8, (24, 23, 25))):
        m = fi.with_far_field(fi.porous_particle(shape, 7, pore_r=(1.0, 2.0), porosity=0.3, seed=5), 7, 3.0)
        nz, ny, nx = shape
        T = fi.TABLE1
        p = fd.Params(nx=nx, ny=ny, nz=nz, dh=T["dh"], D_fast=fi.D_FAST_SI, D_slow=0.0, dt=T["dt"], radius=R,
                      weights="bf16", v_far=2e4)
        ctx = fd.build_kernels(p, m)
        try:
            W = fd.export_kernels(ctx, (0, nx, 0, ny, 0, nz)).reshape(-1, (2 * R + 1) ** 3)
        finally:
            fd.destroy(ctx)
        sol = W[m.reshape(-1) == 0]
        c = sol.shape[1] // 2
        assert len(sol) > 100
        np.testing.assert_array_equal(sol[:, c], 1.0)
        assert np.count_nonzero(np.delete(sol, c, axis=1)) == 0


def test_absorb_cfg3o_sampled_vs_oracle(fd, oracle_lib):
    """One macro step of the integrated loop at full size (cfg3o: the open R50 model, Table 1 SI
    values, bf16 weights, the default tail — interface lists, nf path), against the oracle's
    components in the paper's order on sampled boxes: the liquid FDiRW step with p_BC·c_far
    (oracle.farfield.step_box_far on the box grown by 3 voxels), then oracle.integrated.solid_fd
    and react on that grown box; compared on the box interior (3 voxels in, past the stencils'
    reach of the grown box's edge), within the reduced-precision bar.  Boxes at the particle
    surface (solid, near-field liquid) and inside the particle (solid and pores)."""
    import torch
    from oracle import farfield as ff
    from oracle import integrated as ig

    cfg = fi.config("cfg3o")
    mask = cfg.mask()
    nz, ny, nx = cfg.shape
    T = fi.TABLE1
    ab = ig.Absorb(D_L=fi.D_FAST_SI, D_S=fi.D_SLOW_SI, dh=T["dh"], dt=T["dt"], k=0.05, c_S_eq=1.0, c_L_eq=1e-5,
                   V_far=cfg.v_far, R=cfg.R)
    c0 = np.where(mask == 1, T["c_L0"], np.where(mask == 0, T["c_S0"], 0.0))
    p = fd.Params(nx=nx, ny=ny, nz=nz, dh=cfg.dh, D_fast=cfg.D_fast, D_slow=0.0, dt=cfg.dt, radius=cfg.R,
                  n_fd=cfg.n_fd, weights="bf16", v_far=cfg.v_far)
    ctx = fd.build_kernels(p, mask)
    try:
        c = torch.from_numpy(c0.astype(np.float32)).cuda()
        fd.far_init(ctx, c, cfg.c_far0)
        fd.absorb_run(ctx, c, 1, ab.D_S, ab.k, ab.c_S_eq, ab.c_L_eq)
        got = c.cpu().numpy().astype(np.float64)
    finally:
        fd.destroy(ctx)
    pb = ig.liquid_problem(mask, ab)
    g = 3
    for box in [(107, 111, 58, 62, 58, 62), (76, 80, 58, 62, 58, 62)]:  # particle surface; pores inside
        gb = (box[0] - g, box[1] + g, box[2] - g, box[3] + g, box[4] - g, box[5] + g)
        msub = mask[gb[4]:gb[5], gb[2]:gb[3], gb[0]:gb[1]]
        assert (msub == 1).any() and (msub == 0).any(), box
        liq = ff.step_box_far(pb, c0 * (mask != 2), cfg.c_far0, gb, fmt=None)
        ref = ig.react(ig.solid_fd(liq, msub, ab), msub, ab)
        ref = ref[g:-g, g:-g, g:-g]
        sub = got[box[4]:box[5], box[2]:box[3], box[0]:box[1]]
        assert rel_l2(sub, ref) <= 5e-3, (box, rel_l2(sub, ref))
        # and the absorption moved mass at the interface (the comparison is not the identity)
        moved = rel_l2(c0[box[4]:box[5], box[2]:box[3], box[0]:box[1]], ref)
        assert moved > 10 * rel_l2(sub, ref), (box, moved, rel_l2(sub, ref))


@pytest.mark.parametrize("weights", ["fp32", "bf16"])
def test_absorb_without_solid_is_the_liquid_step(fd, weights):
    """Degenerate loop: an open domain with no solid voxel.  The interface and non-far lists hold no
    solid work, the reaction has no face pair, Q_S = c̄_S = 0 — and one macro step's field is bit for
    bit the plain far-field FDiRW step (fdirw_run) of the same context (c_far enters only the next
    step); Eq.7's balance closes."""
    import torch

    shape = (21, 19, 23)
    m = fi.with_far_field(np.ones(shape, np.uint8), 7, 2.0)
    assert not (m == 0).any() and (m == 2).any()
    T = fi.TABLE1
    c0 = np.where(m == 1, T["c_L0"] * (1.0 + 0.3 * np.sin(np.arange(m.size).reshape(shape))), 0.0).astype(np.float32)
    nz, ny, nx = shape
    p = fd.Params(nx=nx, ny=ny, nz=nz, dh=T["dh"], D_fast=fi.D_FAST_SI, D_slow=0.0, dt=T["dt"], radius=3,
                  weights=weights, v_far=2e4)
    out = []
    for kind in ("absorb", "run"):
        ctx = fd.build_kernels(p, m)
        try:
            c = torch.from_numpy(c0).cuda()
            M0 = fd.far_init(ctx, c, 0.5 * T["c_L0"])
            if kind == "absorb":
                kin = fd.absorb_run(ctx, c, 1, fi.D_SLOW_SI, 0.05, 1.0, 1e-5)
                assert kin[0, 0] == 0.0 and kin[0, 3] == 0.0
                got = c.cpu().numpy().astype(np.float64)
                assert abs(got[m != 2].sum() + kin[0, 2] * 2e4 - M0) / M0 <= 1e-9
            else:
                fd.run(ctx, c, 1)
            out.append(c.cpu().numpy())
        finally:
            fd.destroy(ctx)
    np.testing.assert_array_equal(out[0], out[1])


@pytest.mark.parametrize("flags", [0, "pbc_reservoir"])
def test_absorb_cfg3o_long_run_invariants(fd, flags):
    """1000 macro steps (t = 0.5 s, Fig.6's horizon) of the default loop on cfg3o (bf16): no NaN;
    Q_S never decreases (absorption only) and c̄_S stays in [0, 1]; every solid voxel stays
    ≤ c_S^eq (f_S ≥ 0 clamps at saturation); and Eq.7's balance Σ c + c_far·V_far = M0 holds to
    1e-9 at the end.  NOT asserted: liquid ≥ 0.  Under reading A26 (p_BC = 1 − row sum) the
    truncated windows give pore targets row sums up to ~1.6 — the fp64 oracle's own p_BC is −0.6 at
    a pore voxel 20 voxels from the far field — so p_BC·c_far drives depleted pores negative
    (measured min −6.3e-3 after 1000 steps, the same with fp32 / fp16 / bf16 weights and every tail
    form: `tools/absorb_negcheck.py`, reading A26).  With FDIRW_F_PBC_RESERVOIR (p_BC by
    the reservoir's held-Dirichlet FD, ≥ 0) every concentration stays ≥ 0, and that is asserted."""
    import torch

    cfg = fi.config("cfg3o")
    mask = cfg.mask()
    nz, ny, nx = cfg.shape
    T = fi.TABLE1
    c0 = np.where(mask == 1, T["c_L0"], np.where(mask == 0, T["c_S0"], 0.0)).astype(np.float32)
    p = fd.Params(nx=nx, ny=ny, nz=nz, dh=cfg.dh, D_fast=cfg.D_fast, D_slow=0.0, dt=cfg.dt, radius=cfg.R,
                  n_fd=cfg.n_fd, weights="bf16", v_far=cfg.v_far,
                  flags=fd.F_PBC_RESERVOIR if flags == "pbc_reservoir" else 0)
    ctx = fd.build_kernels(p, mask)
    try:
        c = torch.from_numpy(c0).cuda()
        M0 = fd.far_init(ctx, c, cfg.c_far0)
        kin = fd.absorb_run(ctx, c, 1000, fi.D_SLOW_SI, 0.05, 1.0, 1e-5)
        got = c.cpu().numpy().astype(np.float64)
    finally:
        fd.destroy(ctx)
    assert np.isfinite(kin).all() and np.isfinite(got).all()
    assert np.all(np.diff(kin[:, 0]) >= -1e-12 * kin[-1, 0])
    assert np.all((kin[:, 3] >= 0) & (kin[:, 3] <= 1))
    assert got[mask == 0].max() <= 1.0 + 1e-6
    assert abs(got[mask != 2].sum() + kin[-1, 2] * cfg.v_far - M0) / M0 <= 1e-9
    assert kin[-1, 3] > kin[0, 3]  # it absorbed
    if flags == "pbc_reservoir":  # p_BC ≥ 0 everywhere: every concentration stays ≥ 0
        assert got[mask != 2].min() >= 0.0
