"""a6 across physical GPUs: one process per device, both halo transports (NCCL send/recv and
P2P peer stores over NVLink).  Needs >= 2 CUDA devices and skips otherwise — the build's GPU
box has one, so these run only where the driver provides several.  Each run must
equal the one-GPU field bit for bit (P13) and the oracle within the bf16 bar, with the
whole-grid mass from fdirw_mass (an NCCL all-reduce on both transports) conserved."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import fdirw_inputs as fi
from _util import lib_params, oracle_problem, rel_l2, small_cfg

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ndev():
    import torch

    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_multi_gpu_bitwise_and_oracle(oracle_lib, tmp_path, transport, world):
    if _ndev() < world:
        pytest.skip("needs %d CUDA devices (have %d)" % (world, _ndev()))
    import torch

    import __graft_entry__

    __graft_entry__.build()
    import paper_2408_11376_b200 as fd

    shape, R, steps = (4 * world, 19, 37), 3, 4   # slabs of 4 planes ≥ R: thin, halo-dominated
    cfg = small_cfg(shape, R, 25, weights="bf16")
    mask = fi.random_two_phase(cfg.shape, 0.6, seed=41)
    c0 = fi.initial_c(mask, "random", seed=41)
    ctx = fd.build_kernels(lib_params(cfg), mask)
    try:
        c = torch.from_numpy(c0).cuda()
        fd.run(ctx, c, steps + 1)
        one = c.cpu().numpy()
    finally:
        fd.destroy(ctx)
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), WORLD_SIZE=str(world))
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "_multi_worker.py"), str(tmp_path),
                               str(steps), transport, ",".join(map(str, shape)), str(R)],
                              env=dict(env, RANK=str(r)), cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
             for r in range(world)]
    outs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=300)
        except subprocess.TimeoutExpired:
            p.kill()
            o, _ = p.communicate()
        outs.append(o.decode(errors="replace"))
    assert all(p.returncode == 0 for p in procs), "\n".join(outs)
    got = np.concatenate([np.load(tmp_path / ("rank%d.npy" % r)) for r in range(world)], axis=0)
    np.testing.assert_array_equal(got, one)
    ref = oracle_lib.step_full(oracle_problem(cfg, mask), c0.astype(np.float64), steps=steps + 1)
    assert rel_l2(got, ref) <= 5e-3
    meta = [json.load(open(tmp_path / ("rank%d.json" % r))) for r in range(world)]
    m0 = float(c0.astype(np.float32).astype(np.float64).sum())
    for m in meta:  # every rank sees the whole-grid Σ
        assert abs(m["m0"] - m0) <= 1e-9 * m0
        assert abs(m["m1"] - m["m0"]) <= 1e-6 * m["m0"]
        assert m["phases"]["step"] > 0
