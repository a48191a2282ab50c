"""Rank process for test_multigpu.test_p2p_fused_gather_two_processes: two processes on the box's
one GPU play two ranks of bench.py's multi-GPU frame with the fused trace + peer-memory hit scatter
(shard.PeerFrame: rank 0's frame buffer exported over CUDA IPC and mapped by rank 1, both ranks'
trace kernels storing hits straight into it). Control plane: gloo. Rank 0 writes the frame."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import inputs  # noqa: E402
from paper_2410_14128_b200 import shard, vf  # noqa: E402


def main(cfg, out):
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    vol = bench.make_volume(bench.CONFIGS[cfg][0])
    keys, rgba = inputs.voxels_device(vol)
    h = vf.build((keys, rgba, inputs.dims_of(vol)), bench.CONFIGS[cfg][2])
    del keys, rgba
    rays, perm = bench.make_rays(cfg)
    width = bench.frame_width(cfg)
    own = shard.shard(perm, width, rank, world)
    rl = torch.from_numpy(np.ascontiguousarray(rays[own])).to(dev)
    pf = shard.PeerFrame(len(rays), perm[own], dev)
    assert (pf.ptr != 0) and (rank == 0) == (pf.frame is not None)
    for rep in range(2):  # the frame buffer is reused across frames
        if rank == 0:
            pf.frame.fill_(0x7F7F7F7F)
            torch.cuda.synchronize()
        dist.barrier()
        pf.run(lambda r, ptr, sl: h.trace_scatter(r, ptr, sl), rl)
        torch.cuda.synchronize()
        dist.barrier()
    if rank == 0:
        np.save(out, pf.frame.cpu().numpy())
    pf.close()
    dist.barrier()
    dist.destroy_process_group()
    print(f"RANK {rank} OK")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
