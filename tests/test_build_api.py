"""vf_build boundary behaviour: the vf_allocator hook ("PyTorch only for device
memory") and VF_ERR_OVERFLOW (stored offsets < 2^32 words, PAPER.md:86 / reading A15)."""
from __future__ import annotations

import ctypes
import time

import numpy as np
import pytest

import inputs

pytestmark = pytest.mark.gpu


def _one_voxel_per_brick(R: int, brick: int):
    """keys (x | y<<21 | z<<42) of one voxel in every brick^3 brick of an R^3 volume."""
    import torch
    c = np.arange(R // brick, dtype=np.int64) * brick + (brick // 2)
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    keys = (x.ravel() | (y.ravel() << 21) | (z.ravel() << 42)).astype(np.int64)
    rgba = np.full(len(keys), 0x7F3F1F0F, dtype=np.int32)
    return torch.from_numpy(keys).cuda(), torch.from_numpy(rgba).cuda()


def test_overflow_fails_fast_before_allocating():
    """R(6^3) R(6^3) at 4096^3 with one voxel in each of the 2^18 bricks: the brick tier would need
    2^18 x 2^18 = 2^36 words, so its offsets cannot be stored -> VF_ERR_OVERFLOW, raised before the
    256 GiB tier is allocated (fast, device memory unchanged)."""
    import torch
    from paper_2410_14128_b200 import vf
    keys, rgba = _one_voxel_per_brick(4096, 64)
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    t0 = time.perf_counter()
    with pytest.raises(vf.VfError) as ei:
        vf.build((keys, rgba, (4096, 4096, 4096)), "R(6^3) R(6^3)")
    assert ei.value.status == vf.VF_ERR_OVERFLOW, str(ei.value)
    assert "2^32" in vf.last_error()
    assert time.perf_counter() - t0 < 30
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated() == before  # every build temporary went back to torch
    # the same volume fits as a hierarchy with small bricks: R(3^3) G(9) -> offsets far below 2^32
    h = vf.build((keys, rgba, (4096, 4096, 4096)), "R(3^3) G(9)")
    assert h.stats()["nonempty_voxels"] == 2 ** 18
    h.close()


def test_single_raw_level_is_exempt_from_the_offset_limit():
    """Reading A15: a single-level Raw grid stores no offsets. R(11^3) at 2048^3 = 2^33 words
    (32 GiB) builds and traces with 64-bit cell indexing (one voxel, hit by one +x ray)."""
    import torch
    from paper_2410_14128_b200 import vf
    keys = torch.tensor([2000 | (1500 << 21) | (7 << 42)], dtype=torch.int64, device="cuda")
    rgba = torch.tensor([0x11223344], dtype=torch.int32, device="cuda")
    h = vf.build((keys, rgba, (2048, 2048, 2048)), "R(11^3)")
    assert h.bytes_used >= 4 * 2 ** 33
    rays = torch.tensor([[0.5, 1500.5, 7.5, 0.0, 1.0, 0.0, 0.0, float("inf")]], dtype=torch.float32, device="cuda")
    out = h.trace(rays).cpu().numpy()
    assert out[0, :3].tolist() == [2000, 1500, 7] and out[0, 3].view(np.float32) == np.float32(1999.5)
    h.close()


def test_torch_allocator_owns_the_handle_memory():
    """With the default allocator the format buffer lives in torch's caching allocator: allocated
    bytes grow by >= bytes_used while the handle lives and return to the baseline after close;
    the buffer and the trace are identical to a build with the library's cudaMalloc."""
    import torch
    from paper_2410_14128_b200 import vf
    from inputs import rays as R
    d = inputs.menger(128, 4)
    keys, rgba = inputs.voxels_device(d)
    rays = torch.from_numpy(R.perspective(64, 64, 60.0, (-40.3, 60.7, -70.1), (40.5, 40.5, 40.5))[0]).cuda()
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    ht = vf.build((keys, rgba, (128,) * 3), "R(3^3) G(4)")
    torch.cuda.synchronize()
    held = torch.cuda.memory_allocated() - before
    assert held >= ht.bytes_used
    hc = vf.build((keys, rgba, (128,) * 3), "R(3^3) G(4)", allocator=None)
    assert torch.cuda.memory_allocated() - before == held  # cudaMalloc: invisible to torch
    assert ht.bytes_used == hc.bytes_used
    assert np.array_equal(ht.buffer_words(), hc.buffer_words())
    assert torch.equal(ht.trace(rays), hc.trace(rays))
    ht.close()
    hc.close()
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated() == before


def test_custom_allocator_balanced_and_failure_is_oom():
    """A caller-supplied vf_allocator sees every allocation: alloc/free calls balance after
    vf_destroy (no leak), requests arrive on the build stream, and an allocator that refuses
    returns VF_ERR_OOM from vf_build with nothing leaked."""
    import torch
    from paper_2410_14128_b200 import vf
    live, log, streams = {}, [], set()
    limit = [None]

    def a(nbytes, ctx, stream):
        if limit[0] is not None and nbytes > limit[0]:
            return None
        p = torch.cuda.caching_allocator_alloc(int(nbytes), torch.cuda.current_device(), stream or 0)
        live[p] = nbytes
        log.append(nbytes)
        streams.add(stream or 0)
        return p

    def f(ptr, nbytes, ctx, stream):
        assert live.pop(ptr) == nbytes
        torch.cuda.caching_allocator_delete(ptr)

    A = vf.Allocator(vf._ALLOC_FN(a), vf._FREE_FN(f), None)
    d = inputs.menger(128, 4)
    keys, rgba = inputs.voxels_device(d)
    s = torch.cuda.Stream()
    h = vf.build((keys, rgba, (128,) * 3), "S(3) G(4)", allocator=A, stream=s)
    assert len(log) > 10 and streams == {s.cuda_stream}
    assert len(live) == 2  # the format buffer and the work counters
    h.close()
    assert not live
    limit[0] = 1 << 16  # refuse the larger requests
    with pytest.raises(vf.VfError) as ei:
        vf.build((keys, rgba, (128,) * 3), "S(3) G(4)", allocator=A, stream=s)
    assert ei.value.status == vf.VF_ERR_OOM
    assert not live
