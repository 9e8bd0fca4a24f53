"""GPU parity of NEXT row N2 — open domain with a far-field reservoir (Eq.7,
P:101-107 Eq.8) — against oracle/farfield.py, through the C-ABI."""
import numpy as np
import pytest

import fdirw_inputs as fi
from _util import lib_params, oracle_problem, rel_l2, small_cfg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fd():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import __graft_entry__

    __graft_entry__.build()
    import paper_2408_11376_b200 as fd

    return fd


def _open_mask(shape, seed):
    m = fi.porous_particle(shape, min(shape) / 2 - 4, pore_r=(1.0, 2.0), porosity=0.3, seed=seed)
    return fi.with_far_field(m, min(shape) / 2 - 4, margin=2.0)


def _gpu_far(fd, cfg, mask, c0, c_far0, steps, v_far, flags=0):
    import torch

    ctx = fd.build_kernels(lib_params(cfg, flags=flags, v_far=v_far), mask)
    try:
        c = torch.from_numpy(c0.astype(np.float32)).cuda()
        M0 = fd.far_init(ctx, c, c_far0)
        fd.run(ctx, c, steps)
        cf = fd.far_get(ctx)
        return c.cpu().numpy().astype(np.float64), cf, M0, ctx.info
    finally:
        fd.destroy(ctx)


@pytest.mark.parametrize("n_fd,R", [(2, 2), (4, 4)])
def test_far_exact_regime_vs_dirichlet_fd(fd, oracle_lib, n_fd, R):
    """n_fd ≤ R: one GPU step == n_fd whole-grid FD substeps with the reservoir held at c_far
    (oracle O6), and c_far(t+Δt) == Eq.7 on the GPU's own field."""
    shape = (13, 14, 15)
    mask = _open_mask(shape, 2)
    assert (mask == 2).sum() > 100
    cfg = small_cfg(shape, R, n_fd, D_slow=1e-2, weights="fp32")
    pb = oracle_problem(cfg, mask)
    c0 = fi.initial_c(mask, "random", seed=2).astype(np.float64) * (mask != 2)
    got, cf, M0, _ = _gpu_far(fd, cfg, mask, c0, 0.3, 1, v_far=500.0)
    ref = oracle_lib.fd_whole_grid(pb, c0, n_fd, c_far=0.3) * (mask != 2)
    assert rel_l2(got, ref) <= 1e-5
    assert np.all(got[mask == 2] == 0)
    assert M0 == pytest.approx(c0.astype(np.float32).astype(np.float64).sum() + 0.3 * 500.0, rel=1e-12)
    assert cf == pytest.approx((M0 - got.sum()) / 500.0, rel=1e-9)


@pytest.mark.parametrize("fmt", ["fp32", "bf16"])
def test_far_truncated_vs_oracle(fd, oracle_lib, fmt):
    """Truncated regime (n_fd = 300 > R), 3 steps with the reservoir: field, c_far and the
    conserved total (Eq.7) vs oracle.farfield.run_full (quantised the same way)."""
    from oracle import farfield as ff

    shape = (14, 13, 15)
    mask = _open_mask(shape, 4)
    cfg = small_cfg(shape, 3, 300, D_slow=1e-3, weights=fmt)
    pb = oracle_problem(cfg, mask)
    c0 = fi.initial_c(mask, "random", seed=4).astype(np.float64)
    V = 2000.0
    refC, refcf, refM0 = ff.run_full(pb, c0, 0.5, V, 3)
    got, cf, M0, _ = _gpu_far(fd, cfg, mask, c0, 0.5, 3, v_far=V)
    tol = 1e-5 if fmt == "fp32" else 5e-3
    nf = mask != 2
    assert rel_l2(got[nf], refC[nf]) <= tol
    assert abs(cf - refcf) / refcf <= (1e-6 if fmt == "fp32" else 1e-4)
    assert (got.sum() + cf * V - M0) / M0 == pytest.approx(0.0, abs=1e-9)   # Eq.7 closes the balance


def test_far_uniform_stationary(fd):
    """c ≡ c_far ≡ κ stays κ (p_BC = 1 − row sum)."""
    import torch

    shape = (12, 12, 12)
    mask = _open_mask(shape, 6)
    cfg = small_cfg(shape, 2, 100, weights="bf16")
    c0 = np.where(mask != 2, 0.8, 0.0)
    got, cf, M0, _ = _gpu_far(fd, cfg, mask, c0, 0.8, 4, v_far=1e4)
    np.testing.assert_allclose(got[mask != 2], 0.8, rtol=2e-6)
    assert cf == pytest.approx(0.8, rel=1e-6)


@pytest.mark.parametrize("world", [2, 3])
def test_far_virtual_ranks_bitwise(fd, world):
    """Slabs + Eq.7 with tile sums gathered in global order: bitwise equal to world = 1."""
    import torch

    shape = (12, 11, 13)
    mask = _open_mask(shape, 8)
    cfg = small_cfg(shape, 3, 60, weights="bf16")
    c0 = fi.initial_c(mask, "random", seed=8)
    V = 777.0
    ctx = fd.build_kernels(lib_params(cfg, v_far=V), mask)
    try:
        cin = torch.from_numpy(c0).cuda()
        out = torch.empty_like(cin)
        fd.far_init(ctx, cin, 0.4)
        fd.step(ctx, cin, out)
        fd.step(ctx, out, cin)
        one, cf1 = cin.cpu().numpy(), fd.far_get(ctx)
    finally:
        fd.destroy(ctx)
    sl = fd.slabs(shape[0], world)
    ctxs = [fd.build_kernels(lib_params(cfg, v_far=V), mask, rank=r, world=world, z_begin=a, z_end=b, device=0)
            for r, (a, b) in enumerate(sl)]
    try:
        cin = [torch.from_numpy(c0[a:b].copy()).cuda() for a, b in sl]
        cout = [torch.empty_like(t) for t in cin]
        fd.far_init_virtual(ctxs, cin, 0.4)
        fd.step_virtual(ctxs, cin, cout)
        fd.step_virtual(ctxs, cout, cin)
        got = np.concatenate([t.cpu().numpy() for t in cin], axis=0)
        cfs = [fd.far_get(c) for c in ctxs]
    finally:
        for c in ctxs:
            fd.destroy(c)
    np.testing.assert_array_equal(got, one)
    assert all(x == cf1 for x in cfs)


def test_cfg3o_open_r50_sampled(fd, oracle_lib):
    """The paper's open R50 model (near field r_p + 5Δh in a 120³ grid, V_far from Table 1),
    Table 1 SI parameters, R5, bf16: sampled boxes (particle surface; near-field edge next to
    the reservoir) vs oracle.farfield.step_box_far; Eq.7 balance."""
    import torch
    from oracle import farfield as ff

    cfg = fi.config("cfg3o")
    mask = cfg.mask()
    assert set(np.unique(mask)) == {0, 1, 2}
    pb = oracle_problem(cfg, mask)
    c0 = fi.initial_c(mask, "paper") * (mask != 2)
    ctx = fd.build_kernels(lib_params(cfg), mask)
    try:
        c = torch.from_numpy(c0).cuda()
        M0 = fd.far_init(ctx, c, cfg.c_far0)
        fd.run(ctx, c, 1)
        cf = fd.far_get(ctx)
        got = c.cpu().numpy()
    finally:
        fd.destroy(ctx)
    assert (got.astype(np.float64).sum() + cf * cfg.v_far - M0) / M0 == pytest.approx(0.0, abs=1e-9)
    for tb in [(107, 112, 57, 62, 58, 62), (112, 117, 58, 63, 57, 61)]:
        ref = ff.step_box_far(pb, c0.astype(np.float64), cfg.c_far0, tb, fmt=None)
        assert rel_l2(got[tb[4]:tb[5], tb[2]:tb[3], tb[0]:tb[1]], ref) <= 5e-3, tb


def test_identity_rows_bitwise(fd):
    """Impermeable solid (D_slow = 0, the N3 loop's liquid step) in an open domain: chunks whose
    non-far targets are all solid are identity rows and carry no weights (C_new = C_old by a
    copy).  Field, c_far and exported kernels bitwise equal to the uncompacted path
    (FDIRW_F_NO_DEDUP builds every window and streams every chunk)."""
    import torch

    shape = (26, 24, 28)
    mask = _open_mask(shape, 11)
    cfg = small_cfg(shape, 3, 60, D_slow=0.0, weights="bf16")
    c0 = fi.initial_c(mask, "random", seed=11)
    outs = []
    for flags in (0, fd.F_NO_DEDUP):
        ctx = fd.build_kernels(lib_params(cfg, flags=flags, v_far=500.0), mask)
        try:
            c = torch.from_numpy(c0.astype(np.float32)).cuda()
            fd.far_init(ctx, c, 0.3)
            fd.run(ctx, c, 3)
            W = fd.export_kernels(ctx, (0, 28, 0, 24, 0, 26)) if flags == 0 else None
            outs.append((c.cpu().numpy(), fd.far_get(ctx), ctx.info["weight_bytes"], W))
        finally:
            fd.destroy(ctx)
    nf = mask != 2
    np.testing.assert_array_equal(outs[0][0][nf], outs[1][0][nf])
    assert outs[0][1] == outs[1][1]
    assert outs[0][2] < outs[1][2]  # identity and all-far chunks store nothing
    W = outs[0][3]
    solid = mask == 0
    c = W.shape[-1] // 2
    np.testing.assert_array_equal(W[solid][:, c], 1.0)  # slow sources: W_s = δ


@pytest.mark.parametrize("fmt,R", [("bf16", 5), ("fp16", 3), ("bf16", 8)])
def test_open_windows_recurrence_reduced_precision(fd, oracle_lib, monkeypatch, fmt, R):
    """With fp16 / bf16 storage, windows touching the reservoir take the Chebyshev recurrence too
    (reading A30; fp32 storage keeps the literal substeps).  Against the literal substeps
    (FDIRW_KGEN_OPEN_LITERAL=1) on the same geometry: every stored weight within one storage ulp
    of the literal one, or within 2e-7 absolute (the recurrence's rounding, on the source's
    scale) where the weight is tiny; the kept masses M_s vs the oracle's within 2e-4 relative;
    one step of the field vs the oracle within the reduced-precision bar."""
    import torch
    from oracle import farfield as ff

    shape = (14, 13, 15) if R < 8 else (19, 18, 20)
    mask = _open_mask(shape, 4)
    cfg = small_cfg(shape, R, 1000, D_slow=1e-3, weights=fmt)
    box = (0, shape[2], 0, shape[1], 0, shape[0])
    out = {}
    for form in ("recurrence", "literal"):
        if form == "literal":
            monkeypatch.setenv("FDIRW_KGEN_OPEN_LITERAL", "1")
        else:
            monkeypatch.delenv("FDIRW_KGEN_OPEN_LITERAL", raising=False)
        ctx = fd.build_kernels(lib_params(cfg, v_far=2000.0), mask)
        try:
            out[form] = fd.export_kernels(ctx, box)
        finally:
            fd.destroy(ctx)
    K = (2 * R + 1) ** 3
    A, B = out["recurrence"].reshape(-1, K), out["literal"].reshape(-1, K)
    src = (mask.reshape(-1) <= 1)
    A, B = A[src], B[src]
    c = K // 2
    off = np.ones(K, bool)
    off[c] = False
    ulp = {"bf16": 2.0 ** -7, "fp16": 2.0 ** -10}[fmt]  # one ulp relative, at worst
    d = np.abs(A[:, off] - B[:, off])
    excess = d - ulp * np.abs(B[:, off])
    assert np.all(excess <= 2e-7), (excess.max(), np.count_nonzero(excess > 2e-7), d.max())
    # the kernels' kept masses M_s (a column sums to M_s through the fp32-pair diagonal) against
    # the oracle's fp64 kernels: the recurrence's rounding is absolute on the source's scale
    # (measured, tests/diag_open_recurrence.py: relative ≤ 5.7e-5 vs the literal substeps' 4.6e-6
    # on these grids) — bounded here at 2e-4, ten times below bf16's half-ulp 2^-9 that every
    # stored weight carries; the diagonals differ from the literal path's by the off-centre
    # weights' storage rounding on top
    pbo = oracle_problem(cfg, mask)
    Mo = oracle_lib.build_kernels(pbo).reshape(-1, K)[src].sum(1)
    ow = oracle_lib.open_windows(pbo).reshape(-1)[src]
    for W in (A, B):
        rel = np.abs(W.astype(np.float64).sum(1) - Mo)[ow] / Mo[ow]
        assert rel.max() <= 2e-4, rel.max()
    assert np.max(np.abs(A[:, c] - B[:, c])) <= 1e-4, np.max(np.abs(A[:, c] - B[:, c]))
    # and the stepped field against the oracle (exact kernels), 1 step
    pb = oracle_problem(cfg, mask)
    c0 = fi.initial_c(mask, "random", seed=4).astype(np.float64) * (mask != 2)
    monkeypatch.delenv("FDIRW_KGEN_OPEN_LITERAL", raising=False)
    got, cf, M0, _ = _gpu_far(fd, cfg, mask, c0, 0.5, 1, v_far=2000.0)
    refC, refcf, _ = ff.run_full(pb, c0, 0.5, 2000.0, 1)
    nf = mask != 2
    assert rel_l2(got[nf], refC[nf]) <= 5e-3
    assert (got.sum() + cf * 2000.0 - M0) / M0 == pytest.approx(0.0, abs=1e-9)


def test_pbc_reservoir_vs_oracle(fd, oracle_lib):
    """FDIRW_F_PBC_RESERVOIR: p_BC by the reservoir's held-Dirichlet FD (A26's alternative,
    oracle.farfield.p_bc_reservoir), truncated regime (n_fd = 300 > R = 3), fp32: one step vs the
    oracle's Eq.8 with that p_BC, and Eq.7's balance."""
    import torch
    from oracle import farfield as ff

    shape = (14, 13, 15)
    mask = _open_mask(shape, 4)
    cfg = small_cfg(shape, 3, 300, D_slow=1e-3, weights="fp32")
    pb = oracle_problem(cfg, mask)
    c0 = fi.initial_c(mask, "random", seed=4).astype(np.float64) * (mask != 2)
    Wq = oracle_lib.quantize(pb, oracle_lib.build_kernels(pb), "fp32")
    pbc = ff.p_bc_reservoir(pb)
    assert pbc.min() >= 0.0
    ref = ff.step_full(pb, Wq, c0, 0.5, pbc)
    got, cf, M0, _ = _gpu_far(fd, cfg, mask, c0, 0.5, 1, v_far=2000.0, flags=fd.F_PBC_RESERVOIR)
    nf = mask != 2
    assert rel_l2(got[nf], ref[nf]) <= 1e-5
    assert (got.sum() + cf * 2000.0 - M0) / M0 == pytest.approx(0.0, abs=1e-9)
    # and it differs from the row-sum reading here (the truncated regime)
    ref26 = ff.step_full(pb, Wq, c0, 0.5, ff.p_bc_full(pb, Wq))
    assert rel_l2(ref[nf], ref26[nf]) > 1e-4
