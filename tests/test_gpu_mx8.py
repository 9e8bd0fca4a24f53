"""GPU parity for the MX8 weight format (FDIRW_W_MX8) through the C-ABI:
stored kernels vs the MX8 oracle (oracle/mx8.py) block by block, fields vs the exact fp64
oracle at north_star's reduced-precision bar (relL2 ≤ 5e-3, mass ≤ 1e-6), the full-size cfg3
bench configuration sampled, and the unsupported combinations rejected."""
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


def _cases():
    return {
        "cfg1": (fi.config("cfg1", n_fd=1000, weights="fp32"), None),
        "ragged_r4_1e5": (small_cfg((13, 22, 21), 4, 1000, D_slow=1e-5), "porous"),
        "particle_r5": (small_cfg((22, 24, 26), 5, 1000, D_slow=1e-3), "particle"),
    }


def _mask(cfg, kind):
    if kind is None:
        return cfg.mask()
    if kind == "porous":
        return fi.random_two_phase(cfg.shape, 0.6, seed=11)
    return fi.porous_particle(cfg.shape, min(cfg.shape) // 2 - 3, pore_r=(1.0, 2.0), porosity=0.3, seed=5)


@pytest.mark.parametrize("name", ["cfg1", "ragged_r4_1e5", "particle_r5"])
def test_mx8_kernels_vs_oracle(fd, oracle_lib, name):
    """Decoded stored weights vs the MX8 oracle on the oracle's kernels: within one quantum of
    the block (the GPU's fp32 kernels may flip a rounding or a block scale) plus the kgen fp32
    error; every column sums to 1; no negative weight."""
    from oracle import mx8

    cfg, kind = _cases()[name]
    mask = _mask(cfg, kind)
    pb = oracle_problem(cfg, mask)
    W = oracle_lib.build_kernels(pb)
    Wo = mx8.quantize_mx8(W, pb.R)
    nz, ny, nx = cfg.shape
    ctx = fd.build_kernels(lib_params(cfg, "mx8"), mask)
    try:
        Wg = fd.export_kernels(ctx, (0, nx, 0, ny, 0, nz))
        info = ctx.info
    finally:
        fd.destroy(ctx)
    K = pb.K
    assert info["bytes_per_voxel_update"] == ((K - 1) * 9 + 4) // 8 + 16
    off = np.ones(K, bool)
    off[K // 2] = False
    # quantum bound from the oracle side: s ≤ 2·M/255 with M the block max (≤ neighbours ±7 in x)
    Mx = np.zeros_like(W)
    for dx in range(-7, 8):
        sh = np.zeros_like(W)
        if dx >= 0:
            sh[:, :, :nx - dx] = W[:, :, dx:]
        else:
            sh[:, :, -dx:] = W[:, :, :nx + dx]
        Mx = np.maximum(Mx, sh)
    err = np.abs(Wg - Wo)[..., off]
    assert np.all(err <= 2.0 * Mx[..., off] / 255 + 1e-5 * W.max()), err.max()
    # nearly every code agrees exactly (differences only at rounding / scale boundaries)
    assert np.mean(err > 1e-5 * W.max()) < 0.01
    np.testing.assert_allclose(Wg.sum(-1), 1.0, atol=3e-7)
    assert np.all(Wg[..., off] >= 0)


@pytest.mark.parametrize("name", ["cfg1", "ragged_r4_1e5", "particle_r5"])
def test_mx8_field_vs_oracle(fd, oracle_lib, name):
    """10 steps (the paper's initial field) vs the exact fp64 oracle: relL2 ≤ 5e-3 (north_star's
    reduced-precision bar), total mass ≤ 1e-6; and vs the oracle run on MX8-quantised oracle
    kernels much closer (the same format, different kgen rounding)."""
    import torch
    from oracle import mx8

    cfg, kind = _cases()[name]
    mask = _mask(cfg, kind)
    pb = oracle_problem(cfg, mask)
    nz, ny, nx = cfg.shape
    box = (0, nx, 0, ny, 0, nz)
    c0 = fi.initial_c(mask, "paper").astype(np.float64)
    W = oracle_lib.build_kernels(pb)
    Wq = mx8.quantize_mx8(W, pb.R)
    ref, refq = c0.copy(), c0.copy()
    for _ in range(10):
        ref = oracle_lib.step_scatter(pb, W, box, ref, box)
        refq = oracle_lib.step_scatter(pb, Wq, box, refq, box)
    ctx = fd.build_kernels(lib_params(cfg, "mx8"), mask)
    try:
        c = torch.from_numpy(c0.astype(np.float32)).cuda()
        m0 = fd.mass(ctx, c)
        fd.run(ctx, c, 10)
        m1 = fd.mass(ctx, c)
        got = c.cpu().numpy().astype(np.float64)
    finally:
        fd.destroy(ctx)
    assert rel_l2(got, ref) <= 5e-3
    assert rel_l2(got, refq) <= 0.25 * rel_l2(got, ref) + 1e-5
    assert abs(m1 - m0) / abs(m0) <= 1e-6


def test_mx8_step_equals_run(fd):
    """fdirw_step (single launches) and fdirw_run (graph ping-pong) give identical bits."""
    import torch

    cfg = small_cfg((9, 17, 30), 3, 200, D_slow=1e-3)
    mask = fi.random_two_phase(cfg.shape, 0.6, seed=4)
    c0 = torch.from_numpy(fi.initial_c(mask, "random", seed=4)).cuda()
    ctx = fd.build_kernels(lib_params(cfg, "mx8"), mask)
    try:
        a = c0.clone()
        fd.run(ctx, a, 4)
        b, out = c0.clone(), torch.empty_like(c0)
        for _ in range(4):
            fd.step(ctx, b, out)
            b, out = out, b
        torch.cuda.synchronize()
        assert torch.equal(a, b)
    finally:
        fd.destroy(ctx)


def test_mx8_cfg3_bench_config_sampled(fd, oracle_lib):
    """BASELINE configs[2] at full size with MX8 weights, bench.py's launch (fdirw_run): sampled
    target boxes vs the exact oracle, total mass over the grid, and the weight bytes 9/16 of bf16's."""
    import torch

    cfg = fi.config("cfg3")
    mask = cfg.mask()
    pb = oracle_problem(cfg, mask)
    c0 = fi.initial_c(mask, "paper")
    ctx = fd.build_kernels(lib_params(cfg, "mx8"), mask)
    try:
        info = ctx.info
        c = torch.from_numpy(c0).cuda()
        m0 = fd.mass(ctx, c)
        fd.run(ctx, c, 1)
        m1 = fd.mass(ctx, c)
        got = c.cpu().numpy()
    finally:
        fd.destroy(ctx)
    K = pb.K
    n_w = info["weight_bytes"] - info["n_tiles"] * info["tile_chunks"] * 8 * 8  # fp32-pair diagonal
    assert n_w == info["n_tiles"] * info["tile_chunks"] * 8 * (K - 1) * 9 // 8
    assert abs(m1 - m0) / m0 <= 1e-6
    for tb in [(140, 146, 92, 98, 92, 97), (0, 5, 185, 192, 0, 3)]:
        ref = oracle_lib.step_box(pb, c0.astype(np.float64), tb)
        assert rel_l2(got[tb[4]:tb[5], tb[2]:tb[3], tb[0]:tb[1]], ref) <= 5e-3, tb


def test_mx8_rejected_combinations(fd):
    cfg = small_cfg((8, 8, 8), 2, 50)
    mask = fi.random_two_phase(cfg.shape, 0.6, seed=1)
    for flags in (fd.F_NO_MASS_FIX, fd.F_NO_DEDUP):
        with pytest.raises(fd.FdirwError):
            fd.build_kernels(lib_params(cfg, "mx8", flags=flags), mask)


@pytest.mark.parametrize("shape,R,n_fd", [
    ((7, 9, 13), 3, 50),      # ragged, several tiles per plane
    ((1, 1, 37), 4, 9),       # 1-D grid
    ((5, 3, 4), 1, 1),        # tiny, R = 1, one substep (exact regime)
    ((6, 5, 9), 2, 300),
    ((4, 12, 19), 5, 60),     # window larger than the domain in z
    ((3, 3, 3), 8, 30),       # R = 8 > every dimension
    ((6, 7, 40), 7, 120),     # R = 7, runtime tile width
])
def test_mx8_edge_shapes(fd, oracle_lib, shape, R, n_fd):
    """Edge cases with MX8 weights: 3 steps vs the oracle on its own MX8-quantised kernels
    (tight: only kgen round-off differs) and vs the exact oracle (north_star's 5e-3), mass."""
    from oracle import mx8

    cfg = small_cfg(shape, R, n_fd, D_slow=2e-3)
    mask = fi.random_two_phase(shape, 0.55, seed=R + n_fd)
    pb = oracle_problem(cfg, mask)
    nz, ny, nx = shape
    box = (0, nx, 0, ny, 0, nz)
    c0 = fi.initial_c(mask, "random", seed=3)
    W = oracle_lib.build_kernels(pb)
    Wq = mx8.quantize_mx8(W, R)
    ref, refq = c0.astype(np.float64), c0.astype(np.float64)
    for _ in range(3):
        ref = oracle_lib.step_scatter(pb, W, box, ref, box)
        refq = oracle_lib.step_scatter(pb, Wq, box, refq, box)
    import torch

    ctx = fd.build_kernels(lib_params(cfg, "mx8"), mask)
    try:
        c = torch.from_numpy(c0.astype(np.float32)).cuda()
        m0 = fd.mass(ctx, c)
        fd.run(ctx, c, 3)
        m1 = fd.mass(ctx, c)
        got = c.cpu().numpy().astype(np.float64)
    finally:
        fd.destroy(ctx)
    assert rel_l2(got, refq) <= 1e-3
    assert rel_l2(got, ref) <= 5e-3
    assert abs(m1 - m0) / m0 <= 1e-6


def test_mx8_r8_mass_drift(fd):
    """The fp32 partials are bounded in slots (R8: 2 rows per TwoSum): 200 steps
    over a mostly homogeneous 64×64×96 R8 grid (identical kernels: systematic round-off) keep
    the total mass to 1e-7 (4 rows per partial measured 8e-7 at cfg5)."""
    import torch

    cfg = small_cfg((64, 64, 96), 8, 400, D_slow=1e-3)
    mask = fi.porous_particle(cfg.shape, 20, pore_r=(1.0, 2.0), porosity=0.3, seed=3)
    c0 = torch.from_numpy(fi.initial_c(mask, "paper")).cuda()
    ctx = fd.build_kernels(lib_params(cfg, "mx8"), mask)
    try:
        c = c0.clone()
        m0 = fd.mass(ctx, c)
        fd.run(ctx, c, 200)
        m1 = fd.mass(ctx, c)
    finally:
        fd.destroy(ctx)
    assert abs(m1 - m0) / m0 <= 1e-7


@pytest.mark.parametrize("cfgname", ["cfg3", "liquid_r2"])
def test_mx8_dedup_storage(fd, oracle_lib, cfgname):
    """MX8 with N4 storage (uniform chunks read their class kernel, quantised as blocks of 8
    equal weights, plus a per-target diagonal): the same decoded operator as dense MX8 and the
    same summation grouping, so the field is bitwise dense MX8's; vs the exact oracle within
    5e-3; mass."""
    import torch

    if cfgname == "cfg3":
        cfg, mask, steps = fi.config("cfg3"), None, 2
        mask = cfg.mask()
    else:  # mostly liquid around a small particle: homogeneous windows, so uniform chunks
        cfg = small_cfg((12, 32, 64), 2, 60, D_slow=1e-3)  # 256 chunks per plane: N4 needs tile 256
        mask, steps = fi.porous_particle(cfg.shape, 5, pore_r=(1.0, 1.5), porosity=0.3, seed=4), 10
    c0 = torch.from_numpy(fi.initial_c(mask, "paper")).cuda()
    out = {}
    for flags in (0, fd.F_DEDUP_STORAGE):
        ctx = fd.build_kernels(lib_params(cfg, "mx8", flags=flags), mask)
        try:
            if flags:
                assert ctx.info["uniform_chunks"] > 0
            c = c0.clone()
            m0 = fd.mass(ctx, c)
            fd.run(ctx, c, steps)
            m1 = fd.mass(ctx, c)
            out[flags] = c.cpu().numpy().astype(np.float64)
            assert abs(m1 - m0) / m0 <= 1e-6
        finally:
            fd.destroy(ctx)
    np.testing.assert_array_equal(out[fd.F_DEDUP_STORAGE], out[0])  # same weights, same summation order
    if cfgname != "cfg3":
        pb = oracle_problem(cfg, mask)
        nz, ny, nx = cfg.shape
        box = (0, nx, 0, ny, 0, nz)
        W = oracle_lib.build_kernels(pb)
        ref = fi.initial_c(mask, "paper").astype(np.float64)
        for _ in range(steps):
            ref = oracle_lib.step_scatter(pb, W, box, ref, box)
        assert rel_l2(out[fd.F_DEDUP_STORAGE], ref) <= 5e-3


@pytest.mark.parametrize("world", [2, 3, 4])
def test_mx8_virtual_ranks_bitwise(fd, world):
    """MX8 over z-slabs (virtual ranks, R-plane halos): every rank's diagonal needs the blocks
    its sources write into the neighbours' targets, which it re-quantises from its own class
    kernels; the result is the 1-GPU MX8 field bitwise (and the kernels too, via export)."""
    import torch

    cfg = small_cfg((4 * 3, 11, 13), 3, 25)
    mask = fi.random_two_phase(cfg.shape, 0.6, seed=world)
    c0 = fi.initial_c(mask, "random", seed=world)
    ctx1 = fd.build_kernels(lib_params(cfg, "mx8"), mask)
    try:
        a = torch.from_numpy(c0.copy()).cuda()
        one = torch.empty_like(a)
        fd.step(ctx1, a, one)
        one = one.cpu().numpy()
        W1 = fd.export_kernels(ctx1, (0, 13, 0, 11, 0, 12))
    finally:
        fd.destroy(ctx1)
    sl = fd.slabs(cfg.shape[0], world)
    ctxs = [fd.build_kernels(lib_params(cfg, "mx8"), mask, rank=r, world=world, z_begin=a, z_end=b, device=0)
            for r, (a, b) in enumerate(sl)]
    try:
        cin = [torch.from_numpy(c0[a:b].copy()).cuda() for a, b in sl]
        cout = [torch.empty_like(t) for t in cin]
        fd.step_virtual(ctxs, cin, cout)
        got = np.concatenate([t.cpu().numpy() for t in cout], axis=0)
        # each rank's stored kernels: its targets' blocks and its own sources' diagonals
        Wr = [fd.export_kernels(c, (0, 13, 0, 11, 0, 12)) for c in ctxs]
    finally:
        for c in ctxs:
            fd.destroy(c)
    np.testing.assert_array_equal(got, one)
    K = cfg.K
    for (a, b), W in zip(sl, Wr):
        np.testing.assert_array_equal(W[a:b, ..., K // 2], W1[a:b, ..., K // 2])  # diagonals


def _open_mask(shape, seed):
    m = fi.porous_particle(shape, min(shape) / 2 - 4, pore_r=(1.0, 2.0), porosity=0.3, seed=seed)
    return fi.with_far_field(m, min(shape) / 2 - 4, margin=2.0)


def test_mx8_far_vs_oracle(fd):
    """MX8 with the N2 far-field reservoir (open windows keep their own mass M, so the diagonal
    is M − Σ decoded off-centre weights; all-far chunks compacted away): 3 steps vs the exact
    oracle (oracle/farfield.py), c_far, and the Eq.7 balance."""
    import torch
    from oracle import farfield as ff

    shape = (14, 13, 15)
    mask = _open_mask(shape, 4)
    cfg = small_cfg(shape, 3, 300, D_slow=1e-3)
    pb = oracle_problem(cfg, mask)
    c0 = fi.initial_c(mask, "random", seed=4).astype(np.float64)
    V = 2000.0
    refC, refcf, _ = ff.run_full(pb, c0, 0.5, V, 3)
    ctx = fd.build_kernels(lib_params(cfg, "mx8", v_far=V), mask)
    try:
        c = torch.from_numpy(c0.astype(np.float32)).cuda()
        M0 = fd.far_init(ctx, c, 0.5)
        fd.run(ctx, c, 3)
        cf = fd.far_get(ctx)
        got = c.cpu().numpy().astype(np.float64)
    finally:
        fd.destroy(ctx)
    nf = mask != 2
    assert rel_l2(got[nf], refC[nf]) <= 5e-3
    assert abs(cf - refcf) / refcf <= 1e-3
    assert (got.sum() + cf * V - M0) / M0 == pytest.approx(0.0, abs=1e-9)


@pytest.mark.parametrize("world", [2, 3])
def test_mx8_far_virtual_ranks_bitwise(fd, world):
    """MX8 + far field over slabs (no compaction there; Eq.7 from gathered tile sums): bitwise
    the one-rank result (which compacts the all-far chunks)."""
    import torch

    shape = (12, 11, 13)
    mask = _open_mask(shape, 8)
    cfg = small_cfg(shape, 3, 60)
    c0 = fi.initial_c(mask, "random", seed=8)
    V = 777.0
    ctx = fd.build_kernels(lib_params(cfg, "mx8", v_far=V), mask)
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
    ctxs = [fd.build_kernels(lib_params(cfg, "mx8", v_far=V), mask, rank=r, world=world, z_begin=a, z_end=b,
                             device=0) for r, (a, b) in enumerate(sl)]
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


def test_mx8_tile_split_bitwise(fd, monkeypatch):
    """One-wave launches split each tile into parts (2 bulk copies per slot per part); every
    thread's arithmetic is unchanged, so any split gives the whole-tile bits."""
    import torch

    cfg = small_cfg((6, 32, 64), 3, 80, D_slow=1e-3)  # 256 chunks per plane: 6 tiles of 256
    mask = fi.random_two_phase(cfg.shape, 0.6, seed=9)
    c0 = torch.from_numpy(fi.initial_c(mask, "random", seed=9)).cuda()
    outs = {}
    for nsub in ("1", "2", "4", None):
        if nsub is None:
            monkeypatch.delenv("FDIRW_MX8_NSUB", raising=False)
        else:
            monkeypatch.setenv("FDIRW_MX8_NSUB", nsub)
        ctx = fd.build_kernels(lib_params(cfg, "mx8"), mask)
        try:
            c = c0.clone()
            fd.run(ctx, c, 3)
            outs[nsub] = c.cpu().numpy()
        finally:
            fd.destroy(ctx)
    for k in ("2", "4", None):
        np.testing.assert_array_equal(outs[k], outs["1"])
