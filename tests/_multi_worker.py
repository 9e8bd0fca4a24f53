"""One rank of tests/test_gpu_multi.py (not a test module): one process per GPU.

Rank r builds its z-slab context on cuda:r with the requested transport (NCCL: grouped
send/recv on a comm stream; P2P: CUDA IPC peer stores fused into the superposition), runs the
steps through fdirw_run, then one more through fdirw_step, and saves its slab plus the
whole-grid mass (fdirw_mass: an NCCL all-reduce on both transports)."""
import json
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

    out_dir, steps, transport, shape, R = sys.argv[1], int(sys.argv[2]), sys.argv[3], \
        tuple(int(v) for v in sys.argv[4].split(",")), int(sys.argv[5])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    cfg = small_cfg(shape, R, 25, weights="bf16")
    mask = fi.random_two_phase(cfg.shape, 0.6, seed=41)
    c0 = fi.initial_c(mask, "random", seed=41)
    z0, z1 = fd.slabs(cfg.shape[0], world)[rank]
    obj = [fd.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = fd.build_kernels(lib_params(cfg), mask, rank=rank, world=world, z_begin=z0, z_end=z1, device=rank,
                           nccl_id=obj[0] if transport == "nccl" else None, transport=transport)
    if transport == "p2p":
        blobs = [None] * world
        dist.all_gather_object(blobs, fd.p2p_export(ctx))
        fd.p2p_attach(ctx, blobs[rank - 1] if rank > 0 else None, blobs[rank + 1] if rank < world - 1 else None)
        fd.comm_init(ctx, obj[0])  # the communicator fdirw_mass reduces over
    dist.barrier()
    c = torch.from_numpy(c0[z0:z1].copy()).cuda()
    m0 = fd.mass(ctx, c)
    fd.run(ctx, c, steps)
    out = torch.empty_like(c)
    fd.step(ctx, c, out)
    m1 = fd.mass(ctx, out)
    ph = fd.profile_phases(ctx, out.clone(), 4)
    torch.cuda.synchronize()
    if transport == "p2p":
        assert not fd.p2p_check(ctx), "P2P wait timed out"
    np.save(os.path.join(out_dir, "rank%d.npy" % rank), out.cpu().numpy())
    json.dump({"m0": m0, "m1": m1, "phases": ph}, open(os.path.join(out_dir, "rank%d.json" % rank), "w"))
    dist.barrier()  # a neighbour may still store into our buffers until it is done
    fd.destroy(ctx)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
