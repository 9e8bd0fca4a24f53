"""Multi-process (gloo, CPU) tests of the N>1 host logic: the slab plan that
libfdirw.so computes (fdirw_make_plan) drives a real 2-/3-rank halo exchange of the
padded state, and the bootstrap broadcasts an NCCL-id-sized blob the way bench.py
does.  The GPU transport itself (NCCL / virtual ranks) is covered by -m gpu tests."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shape, R, q):
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import paper_2408_11376_b200 as fd

        dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank, world_size=world)
        nz, ny, nx = shape
        params = fd.Params(nx=nx, ny=ny, nz=nz, dh=1.0, D_fast=1.0, D_slow=1e-3, dt=0.1 * 30, radius=R,
                           weights="bf16")
        z0, z1 = fd.slabs(nz, world)[rank]
        pl = fd.make_plan(params, rank, world, z0, z1)
        assert (pl["z_begin"], pl["z_end"]) == (z0, z1)
        assert pl["src_z_begin"] == max(0, z0 - R) and pl["src_z_end"] == min(nz, z1 + R)
        assert pl["mask_z_begin"] == max(0, z0 - 2 * R) and pl["mask_z_end"] == min(nz, z1 + 2 * R)
        tpp = pl["tiles_per_plane"]
        assert pl["n_tiles"] == (z1 - z0) * tpp
        if z1 - z0 > 2 * R:
            assert pl["interior_tile_begin"] == R * tpp and pl["interior_tile_end"] == (z1 - z0 - R) * tpp
        else:
            assert pl["interior_tile_begin"] == pl["interior_tile_end"]

        # bootstrap: rank 0's 128-byte id reaches every rank unchanged (bench.py path)
        blob = [bytes(np.random.default_rng(7).integers(0, 256, 128, dtype=np.uint8)) if rank == 0 else None]
        dist.broadcast_object_list(blob, src=0)
        assert len(blob[0]) == 128

        # padded state of this rank, interior filled from the global field
        G = np.random.default_rng(11).random(shape, dtype=np.float32)
        px, py, pz, x0 = pl["padded_x"], pl["padded_y"], pl["padded_z"], pl["pad_x0"]
        P = np.zeros(pz * py * px, np.float32)
        V = P.reshape(pz, py, px)
        V[R:R + (z1 - z0), R:R + ny, x0:x0 + nx] = G[z0:z1]
        T = torch.from_numpy(P)
        n = pl["halo_elems"]
        reqs = []
        for peer, s_off, r_off in ((pl["peer_lo"], pl["send_lo"], pl["recv_lo"]),
                                   (pl["peer_hi"], pl["send_hi"], pl["recv_hi"])):
            if peer >= 0:
                reqs.append(dist.isend(T[s_off:s_off + n].clone(), peer))
                buf = torch.empty(n)
                reqs.append((dist.irecv(buf, peer), buf, r_off))
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
                T[r[2]:r[2] + n] = r[1]
            else:
                r.wait()
        V = T.numpy().reshape(pz, py, px)
        # halo planes now hold the neighbours' boundary planes; the padding stays 0
        lo = G[z0 - R:z0] if z0 > 0 else np.zeros((R, ny, nx), np.float32)
        hi = G[z1:z1 + R] if z1 < nz else np.zeros((R, ny, nx), np.float32)
        np.testing.assert_array_equal(V[:R, R:R + ny, x0:x0 + nx], lo)
        np.testing.assert_array_equal(V[R + (z1 - z0):, R:R + ny, x0:x0 + nx], hi)
        mask = np.ones_like(V, bool)
        mask[:, R:R + ny, x0:x0 + nx] = False
        assert not V[mask].any()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        import traceback

        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world,shape,R", [(2, (12, 9, 13), 3), (3, (15, 7, 20), 2), (2, (10, 5, 8), 5)])
def test_gloo_halo_exchange(world, shape, R):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, R, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert res[r] == "ok", res[r]
