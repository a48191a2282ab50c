"""Subprocess for test_full_frame.test_cfg5_tile_sharded_frame_assembled: simulate N = 2, 4, 8
ranks of bench.py's frame on one GPU. For every simulated rank r, a one-rank NCCL group runs
bench.FrameStep (chunked trace of rank r's interleaved tiles + NCCL gather) and the gathered shard
is placed into the frame with shard.assemble; the assembled image must equal the oracle's."""
import os
import socket
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import bench  # noqa: E402
import inputs  # noqa: E402
from paper_2410_14128_b200 import shard, vf  # noqa: E402
from parity import assert_parity  # noqa: E402


def main(tmp):
    ref = {"xyz": np.load(os.path.join(tmp, "ref_xyz.npy")), "t": np.load(os.path.join(tmp, "ref_t.npy"))}
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]), RANK="0", WORLD_SIZE="1")
    s.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    vol = bench.make_volume("sparse")
    keys, rgba = inputs.voxels_device(vol)
    h = vf.build((keys, rgba, inputs.dims_of(vol)), bench.CONFIGS["cfg5"][2])
    del keys, rgba
    rays, perm = bench.make_rays("cfg5")
    width = bench.frame_width("cfg5")
    n = len(rays)
    for world in (2, 4, 8):
        counts = shard.shard_counts(perm, width, world)
        bufs = []
        for r in range(world):
            own = shard.shard(perm, width, r, world)
            rl = torch.from_numpy(np.ascontiguousarray(rays[own])).cuda()
            # the bench's per-rank step, in a one-rank group: trace chunks + NCCL gather to rank 0
            step = bench.FrameStep(lambda rv, hv: h.trace(rv, hv), rl, [counts[r]], 0, 1, True, torch.device("cuda", 0),
                                   chunks=3, timed=False)
            got = step()
            torch.cuda.synchronize()
            bufs.append(got[0].cpu().numpy())
        img = shard.assemble(bufs, perm, width, world)  # row-major pixels
        out = img[perm]  # back to ray order
        assert out.shape == (n, 4)
        assert_parity(out[:, :3], out[:, 3].view(np.float32), ref, f"cfg5 tile-sharded frame N={world}")
    dist.destroy_process_group()
    print("FRAME OK")


if __name__ == "__main__":
    main(sys.argv[1])
