"""GPU parity: the CUDA path (through the C-ABI) against the CPU fp64 oracle on the
same seeded inputs.  Tolerances from north_star: fp32 relL2 ≤ 1e-5,
fp16/bf16 relL2 ≤ 5e-3, total mass ≤ 1e-6 relative; the superposition alone on the
oracle's own quantised weights ≤ 1e-6 (only fp32 accumulation order differs)."""
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


def _gpu_steps(fd, cfg, mask, c0, steps, weights=None, flags=0, use_run=True):
    import torch

    ctx = fd.build_kernels(lib_params(cfg, weights, flags), mask)
    try:
        c = torch.from_numpy(c0.astype(np.float32)).cuda()
        m0 = fd.mass(ctx, c)
        if use_run:
            fd.run(ctx, c, steps)
        else:
            out = torch.empty_like(c)
            for _ in range(steps):
                fd.step(ctx, c, out)
                c, out = out, c
        m1 = fd.mass(ctx, c)
        torch.cuda.synchronize()
        return c.cpu().numpy().astype(np.float64), m0, m1, ctx.info
    finally:
        fd.destroy(ctx)


# ------------------------------------------------------------------ cfg1 (16³, R2)
@pytest.mark.parametrize("n_fd,direct", [(2, False), (1000, False), (1000, True)])
def test_cfg1_fp32_10_steps(fd, oracle_lib, n_fd, direct):
    """BASELINE configs[0]: 16³ two-phase porous grid, D ratio 1e3, R2, fp32, 10 steps,
    exact (n_fd = 2 ≤ R) and truncated (n_fd = 1000) regimes; kgen by the Chebyshev
    recurrence (default at n_fd = 1000, reading A30) and by the literal substeps."""
    cfg = fi.config("cfg1", n_fd=n_fd, weights="fp32")
    mask = cfg.mask()
    pb = oracle_problem(cfg, mask)
    c0 = fi.initial_c(mask, "random", seed=1)
    ref = oracle_lib.step_full(pb, c0.astype(np.float64), steps=10)
    got, m0, m1, info = _gpu_steps(fd, cfg, mask, c0, 10, flags=fd.F_KGEN_DIRECT if direct else 0)
    assert info["n_fd"] == n_fd
    plan = fd.make_plan(lib_params(cfg, flags=fd.F_KGEN_DIRECT if direct else 0))
    assert info["kgen_steps"] == plan["kgen_steps"] == (n_fd if (direct or n_fd < 8) else 8 + 157)
    assert rel_l2(got, ref) <= 1e-5
    assert abs(m1 - m0) / abs(m0) <= 1e-6
    assert abs(got.sum() - c0.astype(np.float64).sum()) / c0.sum() <= 1e-6
    if n_fd == 2:  # P1 on the GPU: == 20 whole-grid FD substeps
        fdref = oracle_lib.fd_whole_grid(pb, c0.astype(np.float64), 20)
        assert rel_l2(got, fdref) <= 1e-5


@pytest.mark.parametrize("direct", [True, False])
@pytest.mark.parametrize("fmt", ["fp32", "fp16", "bf16"])
def test_kgen_matches_oracle_kernels(fd, oracle_lib, fmt, direct):
    """a3/a4 in isolation: the stored kernels (export) vs the oracle's quantised kernels (O5),
    kgen by the literal substeps and by the Chebyshev recurrence (reading A30)."""
    cfg = fi.config("cfg1", n_fd=1000, weights=fmt)
    mask = cfg.mask()
    pb = oracle_problem(cfg, mask)
    Wo = oracle_lib.quantize(pb, oracle_lib.build_kernels(pb), fmt)
    ctx = fd.build_kernels(lib_params(cfg, flags=fd.F_KGEN_DIRECT if direct else 0), mask)
    try:
        Wg = fd.export_kernels(ctx, (0, 16, 0, 16, 0, 16))
    finally:
        fd.destroy(ctx)
    ulp = {"fp32": 2e-6, "fp16": 2.0 ** -10, "bf16": 2.0 ** -7}[fmt]
    c = pb.K // 2
    off = np.ones(pb.K, bool)
    off[c] = False
    # off-centre: equal up to one storage ulp (the GPU's fp32 FD may round differently).  The
    # recurrence's fp32 rounding is absolute on the scale of the window (its t_k are O(‖v‖), not
    # O(W), reading A30), so fp32 adds a term scaled by EACH kernel's own largest off-centre
    # weight (not the global max, which includes near-1 diagonals): measured 6.5e-6 of it here
    # (r02_kgen_decades.jsonl; direct 3.9e-6) → bound 2e-5, about 3x.
    kmax = Wo[..., off].max(-1, keepdims=True)
    absol = 1e-7 if (direct or fmt != "fp32") else 2e-5 * kmax
    err = np.abs(Wg[..., off] - Wo[..., off])
    assert np.all(err <= ulp * np.maximum(np.abs(Wo[..., off]), 1e-30) + absol)
    if fmt == "fp32":
        assert rel_l2(Wg[..., off], Wo[..., off]) <= 2e-6
    np.testing.assert_allclose(Wg.sum(-1), 1.0, atol=1e-12)  # mass fix-up (fp32-pair diagonal, A10): Σ = 1
    assert np.all(Wg >= 0)


@pytest.mark.parametrize("fmt", ["fp32", "fp16", "bf16"])
def test_superposition_on_oracle_weights(fd, oracle_lib, fmt):
    """a5 in isolation: upload the oracle's O5 weights, one GPU step vs the oracle's fp64 scatter."""
    import torch

    cfg = small_cfg((13, 17, 21), 3, 40, D_slow=1e-3, weights=fmt)  # ragged: nx % 8 != 0
    mask = fi.random_two_phase(cfg.shape, 0.6, seed=5)
    pb = oracle_problem(cfg, mask)
    Wq = oracle_lib.quantize(pb, oracle_lib.build_kernels(pb), fmt)
    c0 = fi.initial_c(mask, "random", seed=5)
    ref = oracle_lib.step_scatter(pb, Wq, (0, 21, 0, 17, 0, 13), c0.astype(np.float64), (0, 21, 0, 17, 0, 13))
    ctx = fd.build_kernels(lib_params(cfg, fmt), mask)
    try:
        fd.debug_upload_weights(ctx, Wq)
        cin = torch.from_numpy(c0).cuda()
        out = torch.empty_like(cin)
        fd.step(ctx, cin, out)
        got = out.cpu().numpy()
    finally:
        fd.destroy(ctx)
    assert rel_l2(got, ref) <= 1e-6


# ------------------------------------------------------------------ edge cases
@pytest.mark.parametrize("shape,R,n_fd,fmt", [
    ((7, 9, 13), 3, 50, "fp32"),      # ragged, several tiles per plane
    ((1, 1, 37), 4, 9, "fp32"),       # 1-D grid
    ((5, 3, 4), 1, 1, "fp32"),        # tiny, R = 1, one substep
    ((6, 5, 9), 2, 300, "bf16"),
    ((4, 12, 19), 5, 60, "fp16"),     # window larger than the domain in z
    ((3, 3, 3), 8, 30, "bf16"),       # R = 8 > every dimension (P2 regime)
    # the two-columns kgen (R5, R8) on degenerate grids: 1-D rows, 2-D sheets, a thin slab
    ((1, 1, 23), 5, 40, "fp32"),
    ((2, 19, 1), 8, 40, "fp32"),
    ((13, 2, 3), 5, 1000, "fp32"),
    ((5, 21, 22), 8, 1000, "bf16"),
])
def test_edge_shapes(fd, oracle_lib, shape, R, n_fd, fmt):
    cfg = small_cfg(shape, R, n_fd, D_slow=2e-3, weights=fmt)
    mask = fi.random_two_phase(shape, 0.55, seed=R + n_fd)
    pb = oracle_problem(cfg, mask)
    c0 = fi.initial_c(mask, "random", seed=3)
    ref = oracle_lib.step_full(pb, c0.astype(np.float64), steps=3)
    got, m0, m1, _ = _gpu_steps(fd, cfg, mask, c0, 3)
    tol = 1e-5 if fmt == "fp32" else 5e-3
    assert rel_l2(got, ref) <= tol
    assert abs(m1 - m0) / m0 <= 1e-6


def test_impermeable_and_no_mass_fix(fd, oracle_lib):
    """D_slow = 0 (reading A23) and FDIRW_F_NO_MASS_FIX reproduce the oracle's variants."""
    cfg = small_cfg((8, 8, 8), 2, 30, D_slow=0.0, weights="bf16")
    mask = fi.random_two_phase(cfg.shape, 0.5, seed=2)
    pb = oracle_problem(cfg, mask)
    c0 = fi.initial_c(mask, "random", seed=2)
    ref = oracle_lib.step_full(pb, c0.astype(np.float64), steps=2)
    got, m0, m1, _ = _gpu_steps(fd, cfg, mask, c0, 2)
    assert rel_l2(got, ref) <= 5e-3
    np.testing.assert_allclose(got[mask == 0], c0[mask == 0], rtol=1e-6)  # slow voxels keep their mass
    refq = oracle_lib.step_full(pb, c0.astype(np.float64), steps=1, fmt="bf16", mass_fix=False)
    got2, _, _, _ = _gpu_steps(fd, cfg, mask, c0, 1, flags=1)
    assert rel_l2(got2, refq) <= 1e-4


def test_step_equals_run(fd):
    """fdirw_run (CUDA graph, padded ping-pong) is bitwise fdirw_step repeated."""
    cfg = small_cfg((12, 10, 11), 2, 20, weights="bf16")
    mask = fi.random_two_phase(cfg.shape, 0.6, seed=1)
    c0 = fi.initial_c(mask, "random", seed=1)
    a, _, _, _ = _gpu_steps(fd, cfg, mask, c0, 5, use_run=True)
    b, _, _, _ = _gpu_steps(fd, cfg, mask, c0, 5, use_run=False)
    np.testing.assert_array_equal(a, b)


# ------------------------------------------------------------------ cfg2 (64³, R4), sampled boxes
@pytest.mark.parametrize("fmt", ["fp32", "bf16"])
def test_cfg2_boxes(fd, oracle_lib, fmt):
    """BASELINE configs[1]: 64³ porous waste-form block, D ratio 1e5, R4, n_fd = 1000;
    one full-grid GPU step compared on target boxes (corner, ragged interior, far corner)."""
    import torch

    cfg = fi.config("cfg2", weights=fmt)
    mask = cfg.mask()
    pb = oracle_problem(cfg, mask)
    c0 = fi.initial_c(mask, "paper")
    ctx = fd.build_kernels(lib_params(cfg), mask)
    try:
        c = torch.from_numpy(c0).cuda()
        m0 = fd.mass(ctx, c)
        fd.run(ctx, c, 1)
        m1 = fd.mass(ctx, c)
        got = c.cpu().numpy()
    finally:
        fd.destroy(ctx)
    assert abs(m1 - m0) / m0 <= 1e-6
    tol = 1e-5 if fmt == "fp32" else 5e-3
    for tb in [(0, 9, 0, 8, 0, 7), (27, 38, 30, 37, 20, 29), (57, 64, 58, 64, 60, 64)]:
        ref = oracle_lib.step_box(pb, c0.astype(np.float64), tb)
        assert rel_l2(got[tb[4]:tb[5], tb[2]:tb[3], tb[0]:tb[1]], ref) <= tol, tb


# ------------------------------------------------------------------ cfg3 (192³, R5) — bench launch config
@pytest.mark.parametrize("fmt", ["bf16", "fp16"])
def test_cfg3_bench_config_sampled(fd, oracle_lib, fmt):
    """BASELINE configs[2] at full size in bench.py's launch configuration (fdirw_run):
    192³ R50 particle, Table 1 SI parameters (n_fd = 1000), R5, bf16 weights (the headline)
    and fp16 (the paper's storage format).  Sampled target boxes vs the oracle; total
    mass over the whole grid."""
    import torch

    cfg = fi.config("cfg3", weights=fmt)
    mask = cfg.mask()
    pb = oracle_problem(cfg, mask)
    c0 = fi.initial_c(mask, "paper")
    ctx = fd.build_kernels(lib_params(cfg), mask)
    try:
        assert ctx.info["n_fd"] == 1000
        c = torch.from_numpy(c0).cuda()
        m0 = fd.mass(ctx, c)
        fd.run(ctx, c, 1)
        m1 = fd.mass(ctx, c)
        got = c.cpu().numpy()
        fd.run(ctx, c, 2)
        m3 = fd.mass(ctx, c)
        got3 = c.cpu().numpy()
    finally:
        fd.destroy(ctx)
    assert abs(m1 - m0) / m0 <= 1e-6 and abs(m3 - m0) / m0 <= 1e-6
    # a box on the particle surface (r ≈ 50 from the centre), a ragged one at a domain corner and
    # one deep inside the particle (solid with pores: the slow-phase kernels)
    for tb in [(140, 146, 92, 98, 92, 97), (0, 5, 185, 192, 0, 3), (93, 99, 94, 100, 95, 99)]:
        ref = oracle_lib.step_box(pb, c0.astype(np.float64), tb)
        assert rel_l2(got[tb[4]:tb[5], tb[2]:tb[3], tb[0]:tb[1]], ref) <= 5e-3, tb
    # three dependent steps on a surface box: the oracle steps the box grown by 2R, then R, then
    # the box itself (each step needs the previous one's values R voxels around it)
    tb = (142, 146, 94, 98, 93, 97)
    C = c0.astype(np.float64)
    for k in (2, 1, 0):
        bk = oracle_lib.clip_box(pb, (tb[0] - k * 5, tb[1] + k * 5, tb[2] - k * 5, tb[3] + k * 5, tb[4] - k * 5,
                                      tb[5] + k * 5))
        part = oracle_lib.step_box(pb, C, bk)
        C = C.copy()
        C[bk[4]:bk[5], bk[2]:bk[3], bk[0]:bk[1]] = part
    assert rel_l2(got3[tb[4]:tb[5], tb[2]:tb[3], tb[0]:tb[1]], C[tb[4]:tb[5], tb[2]:tb[3], tb[0]:tb[1]]) <= 5e-3


# ------------------------------------------------------------------ slabs (virtual ranks)
@pytest.mark.parametrize("world", [2, 3, 4])
def test_virtual_ranks_bitwise(fd, oracle_lib, world):
    """P13: the slab decomposition with R-plane halos reproduces the 1-GPU result bitwise
    (thin slabs: thickness ≥ R, interior/boundary split exercised)."""
    import torch

    cfg = small_cfg((4 * 3, 11, 13), 3, 25, weights="bf16")
    mask = fi.random_two_phase(cfg.shape, 0.6, seed=world)
    c0 = fi.initial_c(mask, "random", seed=world)
    one, _, _, _ = _gpu_steps(fd, cfg, mask, c0, 1, use_run=False)
    nz = cfg.shape[0]
    sl = fd.slabs(nz, world)
    ctxs = [fd.build_kernels(lib_params(cfg), mask, rank=r, world=world, z_begin=a, z_end=b, device=0)
            for r, (a, b) in enumerate(sl)]
    try:
        cin = [torch.from_numpy(c0[a:b].copy()).cuda() for a, b in sl]
        cout = [torch.empty_like(t) for t in cin]
        fd.step_virtual(ctxs, cin, cout)
        got = np.concatenate([t.cpu().numpy() for t in cout], axis=0)
    finally:
        for c in ctxs:
            fd.destroy(c)
    np.testing.assert_array_equal(got, one.astype(np.float32))
    # and the sharded field against the oracle directly (not only against one GPU)
    ref = oracle_lib.step_full(oracle_problem(cfg, mask), c0.astype(np.float64), steps=1)
    assert rel_l2(got, ref) <= 5e-3


@pytest.mark.parametrize("R,fmt,far,direct", [(5, "fp32", False, False), (5, "bf16", False, False),
                                              (5, "fp32", True, False), (5, "fp32", False, True),
                                              (8, "fp32", False, False), (8, "bf16", True, False)])
def test_kgen_bal_equal_columns(fd, oracle_lib, R, fmt, far, direct):
    """R = 5 and 8: the two-columns-per-thread kgen (kgen_bal.cu, the default) against the one-column
    kernel (FDIRW_F_KGEN_COLUMNS) and the oracle.  The substep / recurrence arithmetic is the same
    operation for operation, so the stored weights agree except where the fp64 epilogue sum
    (grouped per thread differently) moves a renormalised weight across a rounding boundary:
    at most one fp32 ulp, on a small fraction of the weights.  Closed and open (N2) windows,
    Chebyshev and literal substeps, dedup and direct kgen."""
    shape = (21, 23, 22) if R == 5 else (13, 14, 12)
    mask = fi.porous_particle(shape, 7 if R == 5 else 5, pore_r=(1.0, 2.0), porosity=0.3, seed=3)
    if far:
        mask = fi.with_far_field(mask, 8 if R == 5 else 5, 3.0 if R == 5 else 1.0)
    cfg = small_cfg(shape, R, 1000, D_slow=1e-3, weights=fmt)
    pb = oracle_problem(cfg, mask)
    Wo = oracle_lib.quantize(pb, oracle_lib.build_kernels(pb), fmt)
    box = (0, shape[2], 0, shape[1], 0, shape[0])
    out = {}
    for name, flags in (("pairs", 0), ("columns", fd.F_KGEN_COLUMNS), ("pairs_nodedup", fd.F_NO_DEDUP)):
        flags |= fd.F_KGEN_DIRECT if direct else 0
        ctx = fd.build_kernels(lib_params(cfg, fmt, flags, v_far=1e3 if far else 0.0), mask)
        try:
            out[name] = fd.export_kernels(ctx, box)
        finally:
            fd.destroy(ctx)
    src = (mask != 2).reshape(-1)
    c = pb.K // 2
    off = np.ones(pb.K, bool)
    off[c] = False
    P, C = out["pairs"].reshape(-1, pb.K)[src], out["columns"].reshape(-1, pb.K)[src]
    np.testing.assert_array_equal(out["pairs"], out["pairs_nodedup"])  # dedup is bit-exact
    d = np.abs(P[:, off] - C[:, off])
    ulp = {"fp32": 2.0 ** -23, "bf16": 2.0 ** -7}[fmt]
    assert np.all(d <= ulp * np.abs(C[:, off]) + 1e-30)
    assert np.count_nonzero(d) <= 1e-3 * d.size
    np.testing.assert_allclose(P[:, c], C[:, c], rtol=1e-6, atol=1e-13)
    if fmt == "fp32" and not far:  # and as close to the oracle as the column kernel
        Wo2 = Wo.reshape(-1, pb.K)[src]
        ep, ec = rel_l2(P[:, off], Wo2[:, off]), rel_l2(C[:, off], Wo2[:, off])
        assert ep <= 1e-5 and ep <= 1.01 * ec, (ep, ec)


@pytest.mark.parametrize("fmt,far", [("fp32", False), ("bf16", False), ("fp16", True)])
def test_kgen_fp64_flag_equals_oracle_bits(fd, oracle_lib, fmt, far):
    """FDIRW_F_KGEN_FP64 (reading A22): fp64 substeps in the oracle's operation order and no
    renormalisation ⇒ every stored off-centre weight equals the oracle's O5 weight bit for bit
    (closed and open windows); the diagonal differs only by fp64 summation order."""
    shape = (9, 10, 11)
    mask = fi.random_two_phase(shape, 0.6, seed=11)
    if far:
        mask[:, :, :2][mask[:, :, :2] == 1] = 2
    cfg = small_cfg(shape, 3, 60, D_slow=1e-2, weights=fmt)
    pb = oracle_problem(cfg, mask)
    Wo = oracle_lib.quantize(pb, oracle_lib.build_kernels(pb), fmt)  # open windows keep M = ΣW
    for flags in (fd.F_KGEN_FP64, fd.F_KGEN_FP64 | fd.F_NO_DEDUP):
        ctx = fd.build_kernels(lib_params(cfg, fmt, flags, v_far=1e3 if far else 0.0), mask)
        try:
            Wg = fd.export_kernels(ctx, (0, shape[2], 0, shape[1], 0, shape[0]))
        finally:
            fd.destroy(ctx)
        src = (mask != 2).reshape(-1)
        c = pb.K // 2
        off = np.ones(pb.K, bool)
        off[c] = False
        Wg2, Wo2 = Wg.reshape(-1, pb.K)[src], Wo.reshape(-1, pb.K)[src]
        np.testing.assert_array_equal(Wg2[:, off], Wo2[:, off])
        np.testing.assert_allclose(Wg2[:, c], Wo2[:, c], rtol=0, atol=1e-13)  # fp32 pair: fp64 sum order only


def test_symmetric_rule(fd, oracle_lib):
    """FDIRW_F_SYMMETRIC_RULE (reading A24): in the exact regime (n_fd ≤ R) target x's gather
    weights are its own kernel reflected.  Matches the oracle and the default build; the slab
    decomposition (no halo sources) stays bitwise equal to one GPU; rejected when n_fd > R."""
    import torch

    cfg = small_cfg((12, 11, 13), 3, 3, D_slow=1e-2, weights="fp32")
    mask = fi.random_two_phase(cfg.shape, 0.6, seed=8)
    pb = oracle_problem(cfg, mask)
    c0 = fi.initial_c(mask, "random", seed=8)
    ref = oracle_lib.step_full(pb, c0.astype(np.float64), steps=2)
    sym, m0, m1, info = _gpu_steps(fd, cfg, mask, c0, 2, flags=fd.F_SYMMETRIC_RULE)
    dflt, _, _, _ = _gpu_steps(fd, cfg, mask, c0, 2)
    assert rel_l2(sym, ref) <= 1e-5 and rel_l2(sym, dflt) <= 1e-6
    assert abs(m1 - m0) / m0 <= 1e-6
    one, _, _, _ = _gpu_steps(fd, cfg, mask, c0, 1, use_run=False, flags=fd.F_SYMMETRIC_RULE)
    sl = fd.slabs(cfg.shape[0], 3)
    ctxs = [fd.build_kernels(lib_params(cfg, flags=fd.F_SYMMETRIC_RULE), mask, rank=r, world=3, z_begin=a,
                             z_end=b, device=0) for r, (a, b) in enumerate(sl)]
    try:
        assert ctxs[1].info["kgen_sources"] == (sl[1][1] - sl[1][0]) * 11 * 13  # own slab only
        cin = [torch.from_numpy(c0[a:b].copy()).cuda() for a, b in sl]
        cout = [torch.empty_like(t) for t in cin]
        fd.step_virtual(ctxs, cin, cout)
        got = np.concatenate([t.cpu().numpy() for t in cout], axis=0)
    finally:
        for c in ctxs:
            fd.destroy(c)
    np.testing.assert_array_equal(got, one.astype(np.float32))
    with pytest.raises(fd.FdirwError) as e:
        fd.build_kernels(lib_params(small_cfg((6, 6, 6), 2, 3), flags=fd.F_SYMMETRIC_RULE), np.ones((6, 6, 6), np.uint8))
    assert e.value.status == fd.E_INVALID


def test_profile_phases_equals_run(fd):
    """fdirw_profile_phases (tracing: CUDA events between the phases of eager steps) computes the
    same bits as fdirw_run, and its phases account for the step."""
    import torch

    cfg = small_cfg((20, 18, 40), 3, 30, weights="bf16")
    mask = fi.random_two_phase(cfg.shape, 0.6, seed=6)
    c0 = fi.initial_c(mask, "random", seed=6)
    ctx = fd.build_kernels(lib_params(cfg), mask)
    try:
        a = torch.from_numpy(c0).cuda()
        b = a.clone()
        fd.run(ctx, a, 5)
        ph = fd.profile_phases(ctx, b, 5)
        np.testing.assert_array_equal(a.cpu().numpy(), b.cpu().numpy())
        assert fd.mass_local(ctx, a) == fd.mass(ctx, a)
    finally:
        fd.destroy(ctx)
    assert ph["interior"] > 0 and ph["halo"] >= 0 and ph["boundary"] >= 0
    assert ph["step"] >= ph["interior"] and ph["step"] <= 1.5 * (ph["interior"] + ph["tail"]) + 0.05


@pytest.mark.parametrize("shape,R", [((96, 128, 256), 2), ((9, 10, 11), 2)])
def test_step_host_equals_run(fd, shape, R):
    """fdirw_step_host (host buffers: copy-in, step, copy-out on the caller's stream; on slabs of
    ≥ 8 tiles per SM — the 96×128×256 grid has 1,536 — a plane-chunk pipeline with copies
    overlapping the chunks' superpositions) chained three times equals fdirw_run(3) bit for bit."""
    import torch

    cfg = small_cfg(shape, R, 30, weights="bf16")
    mask = fi.random_two_phase(cfg.shape, 0.6, seed=12)
    c0 = fi.initial_c(mask, "random", seed=12)
    ctx = fd.build_kernels(lib_params(cfg), mask)
    try:
        ref = torch.from_numpy(c0).cuda()
        fd.run(ctx, ref, 3)
        h = [torch.from_numpy(c0.copy()).pin_memory(), torch.empty(cfg.shape, dtype=torch.float32).pin_memory()]
        for k in range(3):
            fd.step_host(ctx, h[k % 2], h[(k + 1) % 2])
        torch.cuda.synchronize()
        np.testing.assert_array_equal(h[1].numpy(), ref.cpu().numpy())
        with pytest.raises(fd.FdirwError):
            fd.step_host(ctx, h[0], h[0])
    finally:
        fd.destroy(ctx)


def test_errors(fd):
    import torch

    cfg = small_cfg((4, 4, 4), 1, 2)
    mask = np.ones(cfg.shape, np.uint8)
    ctx = fd.build_kernels(lib_params(cfg), mask)
    try:
        c = torch.zeros(cfg.shape, device="cuda")
        with pytest.raises(fd.FdirwError) as e:
            fd.step(ctx, c, c)
        assert e.value.status == fd.E_ALIAS
    finally:
        fd.destroy(ctx)


# ------------------------------------------------------------------ kgen: Chebyshev vs substeps
@pytest.mark.parametrize("shape,R,D_slow,fmt", [
    ((16, 16, 16), 2, 1e-3, "fp32"),    # cfg1 geometry class, D ratio 1e3
    ((14, 13, 15), 4, 1e-5, "fp32"),    # cfg2's D ratio 1e5, R4
    ((11, 12, 10), 3, 0.0, "fp32"),     # impermeable slow phase (reading A23): isolated cells
    ((13, 12, 14), 5, 1e-3, "bf16"),    # cfg3's R5, bf16 storage
])
def test_kgen_chebyshev_vs_substeps_and_oracle(fd, oracle_lib, shape, R, D_slow, fmt):
    """Reading A30: the default kgen runs 8 substeps, then evaluates A^992 by a Chebyshev
    recurrence of degree m = 157 (λ = 0.1; truncation ≤ 1e-10); FDIRW_F_KGEN_DIRECT runs the 1000
    literal substeps.  Both stored kernels against the oracle's fp64 kernels (unquantised),
    and against each other."""
    cfg = small_cfg(shape, R, 1000, D_slow=D_slow, weights=fmt)
    mask = fi.random_two_phase(shape, 0.6, seed=R)
    pb = oracle_problem(cfg, mask)
    Wo = oracle_lib.build_kernels(pb)  # fp64, [nz][ny][nx][K]
    nz, ny, nx = shape
    Wg, infos = [], []
    for flags in (0, fd.F_KGEN_DIRECT):
        ctx = fd.build_kernels(lib_params(cfg, flags=flags), mask)
        try:
            infos.append(ctx.info)
            Wg.append(fd.export_kernels(ctx, (0, nx, 0, ny, 0, nz)))
        finally:
            fd.destroy(ctx)
    assert infos[0]["kgen_steps"] == 8 + 157 and infos[1]["kgen_steps"] == 1000
    assert infos[0]["kgen_kernel_ms"] > 0
    c = pb.K // 2
    off = np.ones(pb.K, bool)
    off[c] = False
    # storage rounding (fp32: the FD's own fp32 error) + what each evaluation adds
    q = {"fp32": 2e-5, "bf16": 2.0 ** -8}[fmt]
    for W in Wg:
        assert np.all(W >= 0)
        np.testing.assert_allclose(W.sum(-1), 1.0, atol=3e-7)
        err = np.abs(W[..., off] - Wo[..., off])
        assert err.max() <= q * Wo[..., off].max() + 1e-9, err.max() / Wo[..., off].max()
        assert rel_l2(W[..., off], Wo[..., off]) <= (5e-6 if fmt == "fp32" else 4e-3)
    d = np.abs(Wg[0] - Wg[1])[..., off]
    assert d.max() <= q * Wo[..., off].max() + 1e-9


# per-decade relative error of the stored fp32 kernels vs the oracle's fp64 kernels, for every
# weight >= 1e-12: the solid-side tails of two-phase kernels are checked, not only the bulk.
# Bounds = 3x the largest relative error measured per decade over the three cases below
# (profiles/r02_kgen_decades.jsonl).  The literal substeps' fp32 error is relative (≤ 9e-5 at
# D ratio 1e5, where 1000 substeps accumulate rounding); the Chebyshev recurrence's is absolute on
# the window's scale (reading A30), so its relative error grows in the far tail: 2e-5 down to
# 1e-8, 9e-5 / 2e-4 / 4.6e-4 / 6.6e-4 in the 1e-9 ... 1e-12 decades.
_DECADE_BOUND = {
    "chebyshev": {1: 1e-4, 2: 1e-4, 3: 1e-4, 4: 1e-4, 5: 1e-4, 6: 1e-4, 7: 1e-4, 8: 1e-4, 9: 3e-4, 10: 6e-4,
                  11: 1.5e-3, 12: 2e-3},
    "direct": {d: 3e-4 for d in range(1, 13)},
}


@pytest.mark.parametrize("path", ["chebyshev", "direct"])
@pytest.mark.parametrize("case", ["cfg1", "r4_ratio1e5", "r5_particle"])
def test_kgen_tail_decades(fd, oracle_lib, case, path):
    if case == "cfg1":
        cfg = fi.config("cfg1", n_fd=1000, weights="fp32")
        mask = cfg.mask()
    elif case == "r4_ratio1e5":
        cfg = small_cfg((14, 13, 15), 4, 1000, D_slow=1e-5)
        mask = fi.random_two_phase((14, 13, 15), 0.6, seed=4)
    else:
        cfg = small_cfg((22, 23, 21), 5, 1000, D_slow=1e-3)
        mask = fi.porous_particle((22, 23, 21), 7, pore_r=(1.0, 2.0), porosity=0.3, seed=3)
    pb = oracle_problem(cfg, mask)
    Wo = oracle_lib.build_kernels(pb)
    nz, ny, nx = cfg.shape
    ctx = fd.build_kernels(lib_params(cfg, "fp32", flags=0 if path == "chebyshev" else fd.F_KGEN_DIRECT), mask)
    try:
        Wg = fd.export_kernels(ctx, (0, nx, 0, ny, 0, nz))
    finally:
        fd.destroy(ctx)
    off = np.ones(pb.K, bool)
    off[pb.K // 2] = False
    g, o = Wg[..., off].ravel(), Wo[..., off].ravel()
    rel = np.abs(g - o) / np.maximum(o, 1e-300)
    seen = 0
    for d, bound in _DECADE_BOUND[path].items():
        sel = (o < 10.0 ** -(d - 1)) & (o >= 10.0 ** -d)
        if sel.any():
            seen += 1
            assert rel[sel].max() <= bound, (d, float(rel[sel].max()))
    assert seen >= 7  # the kernels span at least 7 decades above 1e-12
    assert np.all(g >= 0)


# ------------------------------------------------------------------ TMA-staged weight stream
@pytest.mark.parametrize("cfgname,fmt", [("96", "fp32"), ("96", "bf16"), ("96", "fp16"), ("cfg3o", "bf16")])
def test_bulk_stream_bitwise(fd, cfgname, fmt):
    """The default superposition for launches of ≥ 2 CTAs/SM streams each tile's weights into
    shared-memory stages with cp.async.bulk; FDIRW_F_NO_BULK_STREAM uses per-thread loads.  Same
    arithmetic in the same order: bitwise equal fields (closed 96³ — 480 tiles; fp32 rows of
    56 KB take the 1-CTA/SM 3-stage form, bf16/fp16 2 CTAs × 4 stages — and the open cfg3o
    with the N2 p_BC term and per-tile sums)."""
    import torch

    if cfgname == "96":
        shape = (96, 96, 96)
        cfg = small_cfg(shape, 3, 100, D_slow=1e-3, weights=fmt)
        mask = fi.porous_particle(shape, 30, pore_r=(1.0, 3.0), porosity=0.3, seed=7)
    else:
        cfg = fi.config(cfgname, weights=fmt)
        mask = cfg.mask()
    c0 = fi.initial_c(mask, "random", seed=5).astype(np.float32)
    outs = []
    for flags in (0, fd.F_NO_BULK_STREAM):
        ctx = fd.build_kernels(lib_params(cfg, flags=flags), mask)
        try:
            assert ctx.info["n_tiles"] >= 2 * 148
            c = torch.from_numpy(c0).cuda()
            if cfg.v_far:
                fd.far_init(ctx, c, cfg.c_far0)
            fd.run(ctx, c, 3)
            outs.append(c.cpu().numpy())
        finally:
            fd.destroy(ctx)
    np.testing.assert_array_equal(outs[0], outs[1])


@pytest.mark.parametrize("fmt", ["fp32", "bf16"])
def test_bulk_stream_stage_canary(fd, fmt):
    """The staged stream's mbarrier protocol in practice (compute-sanitizer racecheck does not
    model cp.async.bulk's complete_tx ordering): every weight a compute thread takes
    from a stage equals the global copy both right after the full barrier and just before the
    warp releases the stage — no late copy, no premature refill — over 4 steps of 2 CTAs/SM
    (bf16) and 1 CTA/SM (fp32) launches; the field is unchanged by the checks."""
    import torch

    shape = (96, 96, 96)
    cfg = small_cfg(shape, 3, 100, D_slow=1e-3, weights=fmt)
    mask = fi.porous_particle(shape, 30, pore_r=(1.0, 3.0), porosity=0.3, seed=7)
    c0 = fi.initial_c(mask, "random", seed=5).astype(np.float32)
    ctx = fd.build_kernels(lib_params(cfg), mask)
    try:
        info = ctx.info
        assert info["n_tiles"] >= 2 * 148
        ref = torch.from_numpy(c0).cuda()
        fd.run(ctx, ref, 4)
        assert fd.debug_stage_canary(ctx, True) == (0, 0)
        c = torch.from_numpy(c0).cuda()
        fd.run(ctx, c, 4)
        checks, bad = fd.debug_stage_canary(ctx, True)
        np.testing.assert_array_equal(c.cpu().numpy(), ref.cpu().numpy())
    finally:
        fd.destroy(ctx)
    L = 7
    assert checks == 4 * 2 * info["chunks"] * (L ** 3 - 1) * (2 if fmt == "fp32" else 1)
    assert bad == 0


# ------------------------------------------------------------------ window de-duplication
@pytest.mark.parametrize("fmt,R,n_fd", [("bf16", 3, 100), ("fp32", 2, 1000), ("fp16", 4, 40)])
def test_dedup_bitwise(fd, fmt, R, n_fd):
    """kgen once per distinct window (default) == kgen on every source (FDIRW_F_NO_DEDUP),
    bitwise: stored kernels and stepped fields; on a particle geometry with many duplicates."""
    import torch

    shape = (30, 28, 33)
    mask = fi.porous_particle(shape, 9, pore_r=(1.0, 2.0), porosity=0.3, seed=4)
    cfg = small_cfg(shape, R, n_fd, D_slow=1e-3, weights=fmt)
    c0 = fi.initial_c(mask, "random", seed=4)
    outs, infos, kerns = [], [], []
    for flags in (0, fd.F_NO_DEDUP):
        ctx = fd.build_kernels(lib_params(cfg, flags=flags), mask)
        try:
            infos.append(ctx.info)
            kerns.append(fd.export_kernels(ctx, (0, 33, 0, 28, 0, 30)))
            c = torch.from_numpy(c0).cuda()
            fd.run(ctx, c, 3)
            outs.append(c.cpu().numpy())
        finally:
            fd.destroy(ctx)
    assert infos[0]["kgen_windows"] < 0.6 * infos[0]["kgen_sources"]  # 6204 / 9181 / 13148 of 27720
    assert infos[1]["kgen_windows"] == infos[1]["kgen_sources"] == 30 * 28 * 33
    np.testing.assert_array_equal(kerns[0], kerns[1])
    np.testing.assert_array_equal(outs[0], outs[1])


def test_cfg5_r8_sampled(fd, oracle_lib):
    """BASELINE configs[4]: cfg3 geometry, D ratio 1e8, R8 (K = 4913), bf16; one step,
    a sampled box at the particle surface vs the oracle; whole-grid mass."""
    import torch

    cfg = fi.config("cfg5")
    mask = cfg.mask()
    pb = oracle_problem(cfg, mask)
    c0 = fi.initial_c(mask, "paper")
    ctx = fd.build_kernels(lib_params(cfg), mask)
    try:
        info = ctx.info
        assert info["K"] == 4913 and info["n_fd"] == 1000
        c = torch.from_numpy(c0).cuda()
        m0 = fd.mass(ctx, c)
        fd.run(ctx, c, 1)
        m1 = fd.mass(ctx, c)
        got = c.cpu().numpy()
    finally:
        fd.destroy(ctx)
    assert abs(m1 - m0) / m0 <= 1e-6
    tb = (143, 147, 93, 97, 94, 97)
    ref = oracle_lib.step_box(pb, c0.astype(np.float64), tb)
    assert rel_l2(got[tb[4]:tb[5], tb[2]:tb[3], tb[0]:tb[1]], ref) <= 5e-3


def test_cfg4_384_one_gpu_sampled(fd, oracle_lib):
    """BASELINE configs[3]'s workload on ONE GPU (150.8 GB of bf16 weights resident): 384³ =
    2×2×2 R50 particles, Table 1 SI parameters, R5.  One step through fdirw_run; sampled boxes
    vs the oracle — a particle surface in the far octant, the seam between octants, and a
    ragged domain corner; whole-grid mass."""
    import torch

    cfg = fi.config("cfg4")
    mask = cfg.mask()
    pb = oracle_problem(cfg, mask)
    c0 = fi.initial_c(mask, "paper")
    ctx = fd.build_kernels(lib_params(cfg), mask)
    try:
        assert ctx.info["n_fd"] == 1000 and ctx.info["weight_bytes"] > 150e9
        c = torch.from_numpy(c0).cuda()
        m0 = fd.mass(ctx, c)
        fd.run(ctx, c, 1)
        m1 = fd.mass(ctx, c)
        got = c.cpu().numpy()
        del c
    finally:
        fd.destroy(ctx)
    assert abs(m1 - m0) / m0 <= 1e-6
    for tb in [(332, 338, 285, 291, 286, 290), (189, 195, 94, 99, 94, 98), (379, 384, 0, 6, 381, 384)]:
        ref = oracle_lib.step_box(pb, c0.astype(np.float64), tb)
        assert rel_l2(got[tb[4]:tb[5], tb[2]:tb[3], tb[0]:tb[1]], ref) <= 5e-3, tb


# ------------------------------------------------------------------ NEXT row N1: coarse-mesh FDiRW
@pytest.mark.parametrize("fmt,b,direct", [("fp32", 3, False), ("fp32", 3, True), ("bf16", 4, False), ("fp16", 5, False)])
def test_coarse_mesh_vs_oracle(fd, oracle_lib, fmt, b, direct):
    """N1 (Eqs.10-15): GPU-built P vs the oracle's P (FD from group-uniform
    sources, group means), and coarse steps vs the oracle's map → P·C → remap.  P columns by
    the Chebyshev evaluation (default, reading A30) and by the literal substeps."""
    import torch
    from oracle import coarse as oc

    shape = (22, 21, 23)
    mask = fi.porous_particle(shape, 6, pore_r=(1.0, 2.0), porosity=0.3, seed=7)
    region = fi.near_field(mask, 6, margin=3)
    cfg = small_cfg(shape, 1, 200, weights=fmt)
    pb = oracle_problem(cfg, mask)
    P, g, sizes = oc.build_P(pb, region, b=b)
    c0 = fi.initial_c(mask, "random", seed=7).astype(np.float64)
    ref = c0
    for _ in range(3):
        ref = oc.step(P, g, sizes, ref)
    ctx = fd.coarse_build(lib_params(cfg, fmt, flags=fd.F_KGEN_DIRECT if direct else 0), region, block=b)
    try:
        info = ctx.info
        assert info["fd_passes"] == (200 if direct else fd.make_plan(lib_params(cfg))["kgen_steps"])
        assert info["n_groups"] == len(sizes) and info["n_region"] == int(region.sum())
        assert info["flops_per_step"] == oc.flop_count(len(sizes), int(region.sum()))
        Pg, gg = fd.coarse_export(ctx)
        c = torch.from_numpy(c0.astype(np.float32)).cuda()
        out = torch.empty_like(c)
        fd.coarse_step(ctx, c, out)
        fd.coarse_run(ctx, out, 2)
        got = out.cpu().numpy()
    finally:
        fd.coarse_destroy(ctx)
    np.testing.assert_array_equal(gg, g)
    tolP = {"fp32": 2e-6, "fp16": 2e-3, "bf16": 8e-3}[fmt]
    off = ~np.eye(len(sizes), dtype=bool)
    assert np.abs(Pg[off] - P[off]).max() <= tolP * max(P.max(), 1e-30)
    np.testing.assert_allclose(sizes @ Pg, sizes, rtol=3e-7)        # column mass fix-up
    tol = 1e-5 if fmt == "fp32" else 5e-3
    assert rel_l2(got[region == 1], ref[region == 1]) <= tol
    np.testing.assert_array_equal(got[region == 0], c0.astype(np.float32)[region == 0])
    m0 = c0.astype(np.float32)[region == 1].astype(np.float64).sum()
    assert abs(got[region == 1].astype(np.float64).sum() - m0) / m0 <= 1e-6


@pytest.mark.parametrize("far", [False, True])
def test_coarse_run_group_space(fd, monkeypatch, far):
    """fdirw_coarse_run maps once, steps the group values and remaps once: against n
    whole coarse steps (fdirw_coarse_step: map, GEMV, remap each time) it differs only by the
    re-averaging rounding of the skipped map/remap pairs — relL2 ≤ 1e-6 over Ω_L, mass and c_far
    alike — and with FDIRW_COARSE_PER_STEP_REMAP=1 (the per-step form) it is bitwise n steps."""
    import torch

    shape = (22, 21, 23)
    mask = fi.porous_particle(shape, 6, pore_r=(1.0, 2.0), porosity=0.3, seed=7)
    region = fi.with_far_field(mask, 6, 3.0) if far else fi.near_field(mask, 6, margin=3)
    cfg = small_cfg(shape, 1, 200, weights="fp32")
    v_far = 4.0e4 if far else 0.0
    c0 = torch.from_numpy(np.where(region == 1, fi.initial_c(mask, "random", seed=9), 0.0).astype(np.float32)).cuda()
    n = 5

    def run(form):
        monkeypatch.delenv("FDIRW_COARSE_PER_STEP_REMAP", raising=False)
        if form == "per_step_run":
            monkeypatch.setenv("FDIRW_COARSE_PER_STEP_REMAP", "1")
        ctx = fd.coarse_build(lib_params(cfg, "fp32", v_far=v_far), region, block=3)
        try:
            c = c0.clone()
            if far:
                fd.coarse_far_init(ctx, c, 0.7)
            if form == "steps":
                out = torch.empty_like(c)
                for _ in range(n):
                    fd.coarse_step(ctx, c, out)
                    c, out = out, c
            else:
                fd.coarse_run(ctx, c, n)
            cf = fd.coarse_far_get(ctx) if far else 0.0
            return c.cpu().numpy().astype(np.float64), cf
        finally:
            fd.coarse_destroy(ctx)

    a, cfa = run("group_space")
    b, cfb = run("steps")
    p, cfp = run("per_step_run")
    np.testing.assert_array_equal(p, b)
    assert cfp == cfb
    m = region == 1
    assert rel_l2(a[m], b[m]) <= 1e-6
    np.testing.assert_array_equal(a[~m], b[~m])
    assert abs(a[m].sum() - b[m].sum()) <= 1e-6 * b[m].sum()
    if far:
        assert abs(cfa - cfb) <= 1e-6 * cfb


@pytest.mark.parametrize("fmt", ["fp32", "bf16"])
def test_coarse_bulk_gemv_bitwise(fd, fmt, monkeypatch):
    """The bulk-copy (cp.async.bulk + mbarrier ring) GEMV and the register GEMV
    (FDIRW_COARSE_GEMV=0) give identical bits: same lane partition and FMA order per row."""
    import torch

    shape = (30, 29, 31)
    mask = fi.porous_particle(shape, 9, pore_r=(1.0, 2.0), porosity=0.3, seed=4)
    region = fi.near_field(mask, 9, margin=4)
    cfg = small_cfg(shape, 1, 50, weights=fmt)
    c0 = torch.from_numpy(fi.initial_c(mask, "random", seed=4)).cuda()
    outs = []
    for mode in ("0", "1"):
        monkeypatch.setenv("FDIRW_COARSE_GEMV", mode)
        ctx = fd.coarse_build(lib_params(cfg, fmt), region, block=3)
        try:
            assert ctx.info["n_groups"] > 148  # several rows per CTA
            c = c0.clone()
            fd.coarse_run(ctx, c, 4)
            outs.append(c.cpu().numpy())
        finally:
            fd.coarse_destroy(ctx)
    np.testing.assert_array_equal(outs[0], outs[1])


@pytest.mark.parametrize("fmt,b", [("fp32", 3), ("fp16", 5)])
def test_coarse_far_vs_oracle(fd, oracle_lib, fmt, b):
    """N1 + N2 (Eq.10 with P_BC, Eq.7): GPU P_BC vs the oracle's held-Dirichlet FD, coarse
    steps with the boundary term and the device-side c_far update vs the oracle, and the
    Eq.7 balance Σ_{Ω_L} c + c_far·V_far = K0."""
    import torch
    from oracle import coarse as oc

    shape = (22, 21, 23)
    mask = fi.porous_particle(shape, 6, pore_r=(1.0, 2.0), porosity=0.3, seed=7)
    region = fi.with_far_field(mask, 6, 3.0)          # 1 near liquid, 2 far reservoir, 0 solid
    cfg = small_cfg(shape, 1, 200, weights=fmt)
    pb = oracle_problem(cfg, mask)
    P, g, sizes = oc.build_P(pb, region, b=b)
    PBC = oc.build_PBC(pb, region, b=b)
    Q = oc.quantize_P(P, sizes, fmt)
    v_far, cf0 = 4.0e4, 0.7
    c0 = np.where(region == 1, fi.initial_c(mask, "random", seed=9), 0.0).astype(np.float32)
    ref, cf = c0.astype(np.float64), cf0
    K0 = ref[region == 1].sum() + cf0 * v_far
    hist = []
    for _ in range(4):
        ref = oc.step_far(Q, PBC.astype(np.float32).astype(np.float64), g, sizes, ref, cf)
        cf = (K0 - ref[region == 1].sum()) / v_far        # Eq.7
        hist.append(cf)
    ctx = fd.coarse_build(lib_params(cfg, fmt, v_far=v_far), region, block=b)
    try:
        Pg, gg = fd.coarse_export(ctx)
        Bg = fd.coarse_export_pbc(ctx)
        c = torch.from_numpy(c0).cuda()
        out = torch.empty_like(c)
        K0g = fd.coarse_far_init(ctx, c, cf0)
        fd.coarse_step(ctx, c, out)
        cf1 = fd.coarse_far_get(ctx)
        fd.coarse_run(ctx, out, 3)
        cf4 = fd.coarse_far_get(ctx)
        got = out.cpu().numpy()
    finally:
        fd.coarse_destroy(ctx)
    np.testing.assert_array_equal(gg, g)
    assert np.abs(Bg - PBC).max() <= 2e-6 * PBC.max()                 # fp32 FD, as P (tolP)
    assert PBC.max() > 1e-3
    # column masses (absorbing): the literal fp32 FD with fp32 storage; with fp16 / bf16 storage the
    # open region's columns take the Chebyshev recurrence (reading A30), whose rounding is absolute
    # on the source's scale — bounded at 5e-5 relative, ten times below fp16's half-ulp 2^-11
    np.testing.assert_allclose(sizes @ Pg, sizes @ P, rtol=2e-6 if fmt == "fp32" else 5e-5)
    assert abs(K0g - K0) <= 1e-6 * K0
    tol = 1e-5 if fmt == "fp32" else 5e-3
    assert rel_l2(got[region == 1], ref[region == 1]) <= tol
    ctol = 1e-6 if fmt == "fp32" else 1e-5
    assert abs(cf1 - hist[0]) <= ctol * cf0 and abs(cf4 - hist[3]) <= ctol * cf0, (cf1 - hist[0], cf4 - hist[3])
    np.testing.assert_array_equal(got[region != 1], c0[region != 1])
    bal = got[region == 1].astype(np.float64).sum() + cf4 * v_far
    assert abs(bal - K0g) <= 1e-9 * K0g


# ------------------------------------------------------------------ NEXT row N4: uniform-chunk dedup
@pytest.mark.parametrize("cfgname,steps", [("small", 3), ("cfg3", 2)])
def test_dedup_storage_bitwise(fd, cfgname, steps):
    """FDIRW_F_DEDUP_STORAGE (uniform chunks read their shared class kernel) gives bitwise the
    dense path's field, on a particle geometry and on the full cfg3 workload."""
    import torch

    if cfgname == "small":
        shape = (40, 37, 48)
        mask = fi.porous_particle(shape, 8, pore_r=(1.0, 2.0), porosity=0.3, seed=9)
        cfg = small_cfg(shape, 3, 200, weights="bf16")
    else:
        cfg = fi.config("cfg3")
        mask = cfg.mask()
    c0 = fi.initial_c(mask, "random", seed=9)
    outs, infos = [], []
    for flags in (0, fd.F_DEDUP_STORAGE):
        ctx = fd.build_kernels(lib_params(cfg, flags=flags), mask)
        try:
            infos.append(ctx.info)
            c = torch.from_numpy(c0).cuda()
            fd.run(ctx, c, steps)
            outs.append(c.cpu().numpy())
        finally:
            fd.destroy(ctx)
    assert infos[0]["uniform_chunks"] == 0
    assert infos[1]["uniform_chunks"] > (0.2 * infos[1]["chunks"] if cfgname == "cfg3" else 0)
    np.testing.assert_array_equal(outs[0], outs[1])


def test_build_deterministic(fd):
    """Two builds of the same problem give the same bits (kernels and stepped field): resume =
    rebuild + saved C continues a run exactly."""
    import torch

    shape = (48, 40, 44)
    mask = fi.porous_particle(shape, 14, pore_r=(1.0, 2.5), porosity=0.3, seed=21)
    cfg = small_cfg(shape, 4, 1000, D_slow=1e-4, weights="fp16")
    c0 = fi.initial_c(mask, "random", seed=21)
    outs = []
    for _ in range(2):
        ctx = fd.build_kernels(lib_params(cfg), mask)
        try:
            W = fd.export_kernels(ctx, (10, 30, 8, 28, 12, 20))
            c = torch.from_numpy(c0).cuda()
            fd.run(ctx, c, 3)
            outs.append((W, c.cpu().numpy()))
        finally:
            fd.destroy(ctx)
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])


# ------------------------------------------------------------------ long runs
@pytest.mark.parametrize("fmt,tol", [("fp32", 1e-5), ("bf16", 5e-3)])
def test_long_run_error_does_not_grow(fd, oracle_lib, fmt, tol):
    """1000 macro steps (t = 0.5 s at Table 1's Δt: the run length of Fig.7) on a 36³
    porous waste-form block, D ratio 1e5, R4, n_fd = 1000: the GPU field stays within the bar of
    the fp64 oracle at steps 10, 100 and 1000, and its error does not keep growing — the paper's
    observation for its precision modes ("errors ... do not continue to grow over
    iterations"); mass to 1e-6."""
    import torch

    shape = (36, 36, 36)
    mask = fi.porous_block(shape, pore_r=(2.0, 3.0), porosity=0.45, seed=6)
    cfg = small_cfg(shape, 4, 1000, D_slow=1e-5, weights=fmt)
    pb = oracle_problem(cfg, mask)
    c0 = fi.initial_c(mask, "random", seed=6)
    _, ref = oracle_lib.step_full(pb, c0.astype(np.float64), steps=1000, threads=True, checkpoints=(10, 100, 1000))
    ctx = fd.build_kernels(lib_params(cfg), mask)
    errs = {}
    try:
        c = torch.from_numpy(c0).cuda()
        m0 = fd.mass(ctx, c)
        done = 0
        for k in (10, 100, 1000):
            fd.run(ctx, c, k - done)
            done = k
            errs[k] = rel_l2(c.cpu().numpy(), ref[k])
        m1 = fd.mass(ctx, c)
    finally:
        fd.destroy(ctx)
    print("long run %s: relL2 vs oracle %s" % (fmt, errs))
    assert all(e <= tol for e in errs.values()), errs
    assert errs[1000] <= 10 * errs[100], errs   # no faster than linear in the steps
    assert abs(m1 - m0) / m0 <= 1e-6
