"""a6 over peer memory (FDIRW_TRANSPORT_P2P, csrc/p2p.cu): the halo planes are stored into
the neighbours' state by the superposition itself, ordered by per-step epoch flags.

Both tests run on ONE GPU: (1) n contexts of one process, each stepping on its own stream
concurrently (fdirw_p2p_attach_local); (2) two processes exchanging CUDA IPC handles of
their buffers over gloo (fdirw_p2p_export / fdirw_p2p_attach) — the same code path as one
process per GPU over NVLink, minus the link.  Both must equal the one-context result bit
for bit (P13)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import fdirw_inputs as fi
from _util import lib_params, small_cfg

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def fd():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import __graft_entry__

    __graft_entry__.build()
    import paper_2408_11376_b200 as fd

    return fd


def _one_gpu(fd, cfg, mask, c0, steps):
    import torch

    ctx = fd.build_kernels(lib_params(cfg), mask)
    try:
        c = torch.from_numpy(c0).cuda()
        fd.run(ctx, c, steps)
        torch.cuda.synchronize()
        return c.cpu().numpy()
    finally:
        fd.destroy(ctx)


@pytest.mark.parametrize("world,steps,R,shape", [(2, 5, 3, None), (3, 4, 2, None), (4, 3, 3, None),
                                                  (2, 3, 2, (80, 64, 256))])
def test_p2p_local_ranks_bitwise(fd, world, steps, R, shape):
    """(80, 64, 256): each slab has 320 tiles, so the ranks run the TMA-staged superposition
    (with its fused halo pushes) instead of the small-grid register-prefetch body."""
    import torch

    cfg = small_cfg(shape or (4 * 3 + 1, 11, 13), R, 25, weights="bf16")
    mask = fi.random_two_phase(cfg.shape, 0.6, seed=world + 20)
    c0 = fi.initial_c(mask, "random", seed=world)
    ref = _one_gpu(fd, cfg, mask, c0, steps)
    sl = fd.slabs(cfg.shape[0], world)
    ctxs = [fd.build_kernels(lib_params(cfg), mask, rank=r, world=world, z_begin=a, z_end=b, device=0,
                             transport="p2p") for r, (a, b) in enumerate(sl)]
    try:
        fd.p2p_attach_local(ctxs)
        streams = [torch.cuda.Stream() for _ in ctxs]
        cs = [torch.from_numpy(c0[a:b].copy()).cuda() for a, b in sl]
        torch.cuda.synchronize()
        for ctx, c, st in zip(ctxs, cs, streams):  # enqueued back to back: the ranks run concurrently
            fd.run(ctx, c, steps, stream=st)
        torch.cuda.synchronize()
        assert not any(fd.p2p_check(ctx) for ctx in ctxs)
        got = np.concatenate([c.cpu().numpy() for c in cs], axis=0)
        # no communicator (built without nccl_id): the whole-grid Σ is refused, the slab Σ is not
        with pytest.raises(fd.FdirwError) as e:
            fd.mass(ctxs[0], cs[0])
        assert e.value.status == fd.E_STATE
        tot = sum(fd.mass_local(ctx, c) for ctx, c in zip(ctxs, cs))
        assert abs(tot - got.astype(np.float64).sum()) <= 1e-9 * abs(tot)
        # fdirw_step (user buffers) on the same contexts: one more step from the result
        outs = [torch.empty_like(c) for c in cs]
        for ctx, c, o, st in zip(ctxs, cs, outs, streams):
            fd.step(ctx, c, o, stream=st)
        torch.cuda.synchronize()
        got2 = np.concatenate([o.cpu().numpy() for o in outs], axis=0)
    finally:
        for ctx in ctxs:
            fd.destroy(ctx)
    np.testing.assert_array_equal(got, ref)
    np.testing.assert_array_equal(got2, _one_gpu(fd, cfg, mask, c0, steps + 1))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_p2p_two_processes_ipc(fd, tmp_path):
    """Two processes, CUDA IPC handles exchanged over gloo, P2P stores into the other
    process's buffers; the 2-rank result equals the 1-context result bit for bit."""
    cfg = small_cfg((14, 12, 17), 3, 25, weights="bf16")
    mask = fi.random_two_phase(cfg.shape, 0.6, seed=31)
    c0 = fi.initial_c(mask, "random", seed=31)
    steps = 5
    ref = _one_gpu(fd, cfg, mask, c0, steps)
    port = _free_port()
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE="2")
    procs = []
    for r in range(2):
        e = dict(env, RANK=str(r))
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "_p2p_worker.py"), str(tmp_path),
                                       str(steps)], env=e, cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
    outs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=240)
        except subprocess.TimeoutExpired:
            p.kill()
            o, _ = p.communicate()
        outs.append(o.decode(errors="replace"))
    assert all(p.returncode == 0 for p in procs), "\n".join(outs)
    got = np.concatenate([np.load(tmp_path / ("rank%d.npy" % r)) for r in range(2)], axis=0)
    np.testing.assert_array_equal(got, ref)
