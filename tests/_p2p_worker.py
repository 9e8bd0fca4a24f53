"""One rank of tests/test_gpu_p2p.py::test_p2p_two_processes_ipc (not a test module).

Builds an FDIRW_TRANSPORT_P2P context for its slab on cuda:0, all-gathers the P2P blobs
over gloo, attaches its neighbours (CUDA IPC), runs the steps and saves its slab."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch
    import torch.distributed as dist

    import fdirw_inputs as fi
    import paper_2408_11376_b200 as fd
    from _util import lib_params, small_cfg

    out_dir, steps = sys.argv[1], int(sys.argv[2])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    cfg = small_cfg((14, 12, 17), 3, 25, weights="bf16")
    mask = fi.random_two_phase(cfg.shape, 0.6, seed=31)
    c0 = fi.initial_c(mask, "random", seed=31)
    z0, z1 = fd.slabs(cfg.shape[0], world)[rank]
    ctx = fd.build_kernels(lib_params(cfg), mask, rank=rank, world=world, z_begin=z0, z_end=z1, device=0,
                           transport="p2p")
    blobs = [None] * world
    dist.all_gather_object(blobs, fd.p2p_export(ctx))
    fd.p2p_attach(ctx, blobs[rank - 1] if rank > 0 else None, blobs[rank + 1] if rank < world - 1 else None)
    dist.barrier()
    c = torch.from_numpy(c0[z0:z1].copy()).cuda()
    fd.run(ctx, c, steps)
    torch.cuda.synchronize()
    assert not fd.p2p_check(ctx), "P2P wait timed out"
    np.save(os.path.join(out_dir, "rank%d.npy" % rank), c.cpu().numpy())
    dist.barrier()  # the neighbour may still store into our buffers until it is done
    fd.destroy(ctx)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
