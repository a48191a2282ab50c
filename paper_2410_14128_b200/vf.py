"""Thin ctypes binding of libvf.so (include/vf.h). Argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C ABI; there is no Python or
CPU fallback: if libvf.so is missing this module raises at import time. PyTorch supplies
device memory and streams (tensors' data_ptr / torch.cuda.Stream.cuda_stream).
"""
from __future__ import annotations

import atexit
import ctypes
import os
import re
import weakref

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VF_LIB") or os.path.join(PKG, "libvf.so")  # VF_LIB: A/B builds (tools)

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (or python -m "
                      f"paper_2410_14128_b200._build); there is no CPU fallback")

_lib = ctypes.CDLL(LIB_PATH)

VF_OK, VF_ERR_INVALID_ARG, VF_ERR_PARSE, VF_ERR_FORMAT, VF_ERR_UNSUPPORTED, VF_ERR_OVERFLOW, VF_ERR_OOM, VF_ERR_CUDA = range(8)
STATUS_NAMES = {0: "VF_OK", 1: "VF_ERR_INVALID_ARG", 2: "VF_ERR_PARSE", 3: "VF_ERR_FORMAT", 4: "VF_ERR_UNSUPPORTED",
                5: "VF_ERR_OVERFLOW", 6: "VF_ERR_OOM", 7: "VF_ERR_CUDA"}
VF_RAW, VF_SVO, VF_SVDAG, VF_NTREE, VF_DF = range(5)
VF_VOL_DENSE_DEVICE, VF_VOL_SPARSE_DEVICE = 0, 1
VF_BUILD_WHOLE_LEVEL_DEDUP = 1
VF_BUILD_ALIGN_NODES = 2
VF_BUILD_DEFAULT = VF_BUILD_WHOLE_LEVEL_DEDUP
VF_TRACE_RESTART_SV = 1
VF_TRACE_INCOHERENT = 2
VF_TRACE_SCHEDULE = 4  # longest-first block order from the previous launch over the same ray array
VF_TRACE_REGROUP = 8   # with VF_TRACE_SCHEDULE: rays regrouped into warps by their last iteration counts
VF_TRACE_PERSISTENT_WARPS = 1 << 30  # internal ablation flag (include/vf.h: bit 30 reserved)
VF_MAX_LEVELS = 16
VF_MAX_TIERS = 16
COUNTER_NAMES = ("rays", "hits", "cell_tests", "steps", "descents", "pops", "redescents", "locates", "near_ties",
                 "raw_cells", "svo_nodes", "svdag_nodes", "svdag_ptrs", "ntree_nodes", "leaf_words", "format_bytes",
                 "exact_calls", "warp_max_tests", "df_skips", "sector_reads", "unique_words", "unique_sectors")
VF_NCOUNTERS = len(COUNTER_NAMES)


class VfError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Level(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_uint32), ("log2_extent", ctypes.c_uint8 * 3), ("depth", ctypes.c_uint8),
                ("log2_fanout", ctypes.c_uint8), ("df_max", ctypes.c_uint8), ("reserved", ctypes.c_uint8 * 2)]


class Volume(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_uint32), ("dims", ctypes.c_uint32 * 3), ("rgba", ctypes.c_void_p),
                ("n_voxels", ctypes.c_uint64), ("keys", ctypes.c_void_p), ("values", ctypes.c_void_p)]


class IpcHandle(ctypes.Structure):  # vf_ipc_handle
    _fields_ = [("handle", ctypes.c_uint8 * 64), ("offset", ctypes.c_uint64)]


def ipc_export(tensor) -> bytes:
    """vf_ipc_export of a CUDA tensor's data pointer (bytes, for any host-side transport)."""
    h = IpcHandle()
    _check(_lib.vf_ipc_export(ctypes.c_void_p(tensor.data_ptr()), ctypes.byref(h)))
    return bytes(ctypes.string_at(ctypes.addressof(h), ctypes.sizeof(h)))


def ipc_open(blob: bytes, device: int) -> int:
    """vf_ipc_open: map another process's export on `device`; returns the device pointer (int)."""
    h = IpcHandle.from_buffer_copy(blob)
    out = ctypes.c_void_p(0)
    _check(_lib.vf_ipc_open(ctypes.byref(h), device, ctypes.byref(out)))
    return out.value


def ipc_close(ptr: int) -> None:
    _check(_lib.vf_ipc_close(ctypes.c_void_p(ptr)))


class Stats(ctypes.Structure):
    _fields_ = [("bytes_used", ctypes.c_uint64), ("paper_layout_bytes", ctypes.c_uint64),
                ("nonempty_voxels", ctypes.c_uint64), ("dims", ctypes.c_uint32 * 3), ("n_levels", ctypes.c_uint32),
                ("n_tiers", ctypes.c_uint32), ("root", ctypes.c_uint32),
                ("nodes_per_tier", ctypes.c_uint64 * VF_MAX_TIERS), ("words_per_tier", ctypes.c_uint64 * VF_MAX_TIERS),
                ("dedup_leaf_nodes", ctypes.c_uint64), ("build_ms", ctypes.c_double), ("compiled_in", ctypes.c_uint32),
                ("reserved_", ctypes.c_uint32)]


_vp = ctypes.c_void_p
_u32, _u64 = ctypes.c_uint32, ctypes.c_uint64
_ALLOC_FN = ctypes.CFUNCTYPE(_vp, ctypes.c_size_t, _vp, _vp)
_FREE_FN = ctypes.CFUNCTYPE(None, _vp, ctypes.c_size_t, _vp, _vp)


class Allocator(ctypes.Structure):  # vf_allocator
    _fields_ = [("alloc", _ALLOC_FN), ("free", _FREE_FN), ("ctx", _vp)]


def _torch_alloc(nbytes, ctx, stream):
    """vf_allocator.alloc backed by torch's caching allocator (the device is the current one:
    the library sets the handle's device around every call)."""
    import torch
    try:
        return torch.cuda.caching_allocator_alloc(int(nbytes), torch.cuda.current_device(), stream or 0)
    except Exception:  # out of memory: the library reports VF_ERR_OOM
        return None


def _torch_free(ptr, nbytes, ctx, stream):
    import torch
    torch.cuda.caching_allocator_delete(ptr)


# kept alive for the life of the module (the library holds the function pointers until vf_destroy)
_TORCH_ALLOC_FN, _TORCH_FREE_FN = _ALLOC_FN(_torch_alloc), _FREE_FN(_torch_free)
TORCH_ALLOCATOR = Allocator(_TORCH_ALLOC_FN, _TORCH_FREE_FN, None)
_sig = {
    "vf_last_error": ([], ctypes.c_char_p),
    "vf_abi_version": ([], ctypes.c_int),
    "vf_parse_format": ([ctypes.c_char_p, ctypes.POINTER(Level), _u32, ctypes.POINTER(_u32)], ctypes.c_int),
    "vf_format_to_string": ([ctypes.POINTER(Level), _u32, ctypes.c_char_p, ctypes.c_size_t], ctypes.c_int),
    "vf_format_resolution": ([ctypes.POINTER(Level), _u32, ctypes.POINTER(_u32)], ctypes.c_int),
    "vf_build": ([ctypes.POINTER(Volume), ctypes.POINTER(Level), _u32, _u32, ctypes.POINTER(Allocator), ctypes.c_int,
                  _vp, ctypes.POINTER(_vp), ctypes.POINTER(_u64)], ctypes.c_int),
    "vf_trace": ([_vp, _vp, _u64, _vp, _u32, _vp], ctypes.c_int),
    "vf_trace_host": ([_vp, _vp, _u64, _vp, _u32, _vp], ctypes.c_int),
    "vf_trace_scatter": ([_vp, _vp, _u64, _vp, _vp, _u32, _vp], ctypes.c_int),
    "vf_ipc_export": ([_vp, _vp], ctypes.c_int),
    "vf_ipc_open": ([_vp, ctypes.c_int, ctypes.POINTER(_vp)], ctypes.c_int),
    "vf_ipc_close": ([_vp], ctypes.c_int),
    "vf_trace_ex": ([_vp, _vp, _u64, _vp, _vp, _u32, _vp], ctypes.c_int),
    "vf_trace_launch_count": ([_vp, _vp, _u64, _u32, ctypes.POINTER(_u32)], ctypes.c_int),
    "vf_trace_counters": ([_vp, _vp, _u64, _vp, _u32, _vp, ctypes.POINTER(_u64)], ctypes.c_int),
    "vf_query": ([_vp, _vp, _u64, _vp, _vp], ctypes.c_int),
    "vf_stats_get": ([_vp, ctypes.POINTER(Stats)], ctypes.c_int),
    "vf_buffer": ([_vp, ctypes.POINTER(_vp), ctypes.POINTER(_u64)], ctypes.c_int),
    "vf_buffer_read": ([_vp, _u64, _u64, _vp], ctypes.c_int),
    "vf_destroy": ([_vp], None),
}
for _name, (_args, _res) in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_sig)


def _check(st: int):
    if st != VF_OK:
        raise VfError(st, _lib.vf_last_error().decode(errors="replace"))


def last_error() -> str:
    return _lib.vf_last_error().decode(errors="replace")


# ---------------------------------------------------------------- formats
def parse_format(sig: str):
    arr = (Level * VF_MAX_LEVELS)()
    n = _u32(0)
    _check(_lib.vf_parse_format(sig.encode(), arr, VF_MAX_LEVELS, ctypes.byref(n)))
    out = (Level * n.value)()
    ctypes.memmove(out, arr, ctypes.sizeof(Level) * n.value)
    return out


def format_to_string(levels) -> str:
    buf = ctypes.create_string_buffer(512)
    _check(_lib.vf_format_to_string(levels, len(levels), buf, 512))
    return buf.value.decode()


def format_resolution(levels):
    d = (_u32 * 3)()
    _check(_lib.vf_format_resolution(levels, len(levels), d))
    return (d[0], d[1], d[2])


_BASE = {"SVO": "S", "SVDAG": "G"}


def signature_from_baseline(text: str, resolution: int) -> str:
    """BASELINE.json notation -> paper signature (SURVEY.md §8(c) reading A16).
    "SVDAG->Raw<8>" at 256 -> "G(5) R(3, 3, 3)"; "N^3-tree<4>" = T(2, d); an unsized SVO/SVDAG/
    N^3-tree level takes the depth that fills the remaining resolution (at most one per
    signature); "Raw<k>" = R(log2 k) per axis."""
    parts = [p.strip() for p in re.split(r"->|→", text) if p.strip()]
    lg_total = resolution.bit_length() - 1
    if 1 << lg_total != resolution:
        raise ValueError("resolution must be a power of two")
    fixed, free = 0, None
    levels = []
    for p in parts:
        m = re.fullmatch(r"Raw<(\d+)>", p)
        if m:
            k = int(m.group(1)).bit_length() - 1
            levels.append(("R", k))
            fixed += k
            continue
        m = re.fullmatch(r"N\^?3-tree<(\d+)>(?:\[(\d+)\])?", p)
        if m:
            n = int(m.group(1)).bit_length() - 1
            if m.group(2):
                levels.append(("T", n, int(m.group(2))))
                fixed += n * int(m.group(2))
            else:
                levels.append(("T", n, None))
            continue
        if p in _BASE:
            levels.append((_BASE[p], None))
            continue
        raise ValueError(f"unknown level {p!r}")
    free = [i for i, l in enumerate(levels) if l[-1] is None]
    if len(free) > 1:
        raise ValueError("more than one unsized level")
    rem = lg_total - fixed
    out = []
    for i, l in enumerate(levels):
        if l[0] == "R":
            out.append(f"R({l[1]}, {l[1]}, {l[1]})")
        elif l[0] == "T":
            d = l[2]
            if d is None:
                if rem % l[1]:
                    raise ValueError("N^3-tree depth does not divide the remaining resolution")
                d = rem // l[1]
            out.append(f"T({l[1]}, {d})")
        else:
            out.append(f"{l[0]}({rem})")
    return " ".join(out)


# ---------------------------------------------------------------- handle
def _stream_ptr(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


class Handle:
    """An immutable built format on one device (owns the device buffer)."""

    def __init__(self, ptr, signature: str, levels, bytes_used: int):
        self._p = ptr
        self.signature = signature
        self.levels = levels
        self.bytes_used = bytes_used

    # -- the hot path
    @staticmethod
    def _flags(restart, persistent=False, incoherent=False, schedule=False):
        """schedule: False, True (VF_TRACE_SCHEDULE) or "regroup" (+ VF_TRACE_REGROUP)."""
        return ((VF_TRACE_RESTART_SV if restart else 0) | (VF_TRACE_PERSISTENT_WARPS if persistent else 0)
                | (VF_TRACE_INCOHERENT if incoherent else 0) | (VF_TRACE_SCHEDULE if schedule else 0)
                | (VF_TRACE_REGROUP if schedule == "regroup" else 0))

    def trace(self, rays, hits=None, restart: bool = False, stream=None, persistent: bool = False,
              incoherent: bool = False, schedule: bool = False):
        """rays: (n, 8) float32 CUDA tensor (vf_ray); hits: (n, 4) int32 CUDA tensor (vf_hit, t as
        float bits). Asynchronous on `stream`. Returns hits."""
        import torch
        n = rays.shape[0]
        if hits is None:
            hits = torch.empty((n, 4), dtype=torch.int32, device=rays.device)
        assert rays.is_cuda and rays.dtype == torch.float32 and rays.is_contiguous() and rays.shape[1] == 8
        assert hits.is_cuda and hits.dtype == torch.int32 and hits.is_contiguous() and hits.shape[0] >= n
        _check(_lib.vf_trace(self._p, ctypes.c_void_p(rays.data_ptr()), n, ctypes.c_void_p(hits.data_ptr()),
                             self._flags(restart, persistent, incoherent, schedule), _stream_ptr(stream)))
        return hits

    def launch_count(self, rays, restart: bool = False, incoherent: bool = False, schedule: bool = False) -> int:
        """vf_trace_launch_count: kernels one trace call over `rays` launches now (3 if scheduled, 4
        with regrouping)."""
        c = _u32(0)
        _check(_lib.vf_trace_launch_count(self._p, ctypes.c_void_p(rays.data_ptr()), rays.shape[0],
                                          self._flags(restart, False, incoherent, schedule), ctypes.byref(c)))
        return int(c.value)

    def trace_scatter(self, rays, hits, slots, restart: bool = False, stream=None, incoherent: bool = False,
                      schedule: bool = False):
        """vf_trace_scatter: the hit of ray i goes to row slots[i] of `hits` — a CUDA tensor, or a raw
        device pointer (int) such as a peer process's frame buffer from ipc_open. slots: (n,) int32
        CUDA tensor on the handle's device. Asynchronous on `stream`."""
        import torch
        n = rays.shape[0]
        assert rays.is_cuda and rays.dtype == torch.float32 and rays.is_contiguous() and rays.shape[1] == 8
        assert slots.is_cuda and slots.dtype == torch.int32 and slots.is_contiguous() and slots.shape[0] >= n
        ptr = hits if isinstance(hits, int) else hits.data_ptr()
        _check(_lib.vf_trace_scatter(self._p, ctypes.c_void_p(rays.data_ptr()), n, ctypes.c_void_p(ptr),
                                     ctypes.c_void_p(slots.data_ptr()), self._flags(restart, False, incoherent, schedule),
                                     _stream_ptr(stream)))
        return hits

    def trace_payload(self, rays, hits=None, payload=None, restart: bool = False, stream=None,
                      schedule: bool = False):
        """vf_trace_ex: hits plus closest-hit payload (n, 2) int32 {rgba, packed int8 normal}."""
        import torch
        n = rays.shape[0]
        if hits is None:
            hits = torch.empty((n, 4), dtype=torch.int32, device=rays.device)
        if payload is None:
            payload = torch.empty((n, 2), dtype=torch.int32, device=rays.device)
        _check(_lib.vf_trace_ex(self._p, ctypes.c_void_p(rays.data_ptr()), n, ctypes.c_void_p(hits.data_ptr()),
                                ctypes.c_void_p(payload.data_ptr()), self._flags(restart, schedule=schedule),
                                _stream_ptr(stream)))
        return hits, payload

    def counters(self, rays, hits=None, restart: bool = False, stream=None, persistent: bool = False,
                 incoherent: bool = False) -> dict:
        """Run the counting variant of the trace kernel once; totals over all rays (synchronous)."""
        import torch
        n = rays.shape[0]
        if hits is None:
            hits = torch.empty((n, 4), dtype=torch.int32, device=rays.device)
        c = (_u64 * VF_NCOUNTERS)()
        _check(_lib.vf_trace_counters(self._p, ctypes.c_void_p(rays.data_ptr()), n, ctypes.c_void_p(hits.data_ptr()),
                                      self._flags(restart, persistent, incoherent), _stream_ptr(stream), c))
        return {k: int(c[i]) for i, k in enumerate(COUNTER_NAMES)}

    def trace_host(self, rays, hits, restart: bool = False, stream=None, incoherent: bool = False,
                   schedule: bool = False):
        """End to end: host (pinned) rays (n,8) float32 -> host hits (n,4) int32, copies inside."""
        n = rays.shape[0]
        _check(_lib.vf_trace_host(self._p, ctypes.c_void_p(rays.data_ptr()), n, ctypes.c_void_p(hits.data_ptr()),
                                  self._flags(restart, False, incoherent, schedule), _stream_ptr(stream)))
        return hits

    def query(self, xyz, stream=None):
        """xyz: (n,3) int32 CUDA tensor -> (n,) int32 rgba (0 = empty)."""
        import torch
        n = xyz.shape[0]
        out = torch.empty(n, dtype=torch.int32, device=xyz.device)
        _check(_lib.vf_query(self._p, ctypes.c_void_p(xyz.data_ptr()), n, ctypes.c_void_p(out.data_ptr()),
                             _stream_ptr(stream)))
        return out

    def stats(self) -> dict:
        s = Stats()
        _check(_lib.vf_stats_get(self._p, ctypes.byref(s)))
        nt = s.n_tiers
        return dict(bytes_used=s.bytes_used, paper_layout_bytes=s.paper_layout_bytes,
                    nonempty_voxels=s.nonempty_voxels, dims=tuple(s.dims), n_levels=s.n_levels, n_tiers=nt,
                    root=s.root, nodes_per_tier=list(s.nodes_per_tier[:nt]),
                    words_per_tier=list(s.words_per_tier[:nt]), dedup_leaf_nodes=s.dedup_leaf_nodes,
                    build_ms=s.build_ms, compiled_in=bool(s.compiled_in))

    def buffer(self):
        """(device pointer, n_words) of the format buffer."""
        p = ctypes.c_void_p(0)
        n = _u64(0)
        _check(_lib.vf_buffer(self._p, ctypes.byref(p), ctypes.byref(n)))
        return p.value, n.value

    def buffer_words(self, first: int = 0, count: int | None = None):
        """Copy of (part of) the format buffer as a numpy uint32 array (tests / tools)."""
        import numpy as np
        _, n = self.buffer()
        if count is None:
            count = n - first
        out = np.empty(count, dtype=np.uint32)
        _check(_lib.vf_buffer_read(self._p, first, count, out.ctypes.data))
        return out

    def close(self):
        if self._p:
            _lib.vf_destroy(self._p)
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_LIVE = weakref.WeakSet()  # handles closed at interpreter exit, while torch (their allocator) still works


@atexit.register
def _close_live_handles():
    for h in list(_LIVE):
        h.close()


def build(volume, signature, flags: int = VF_BUILD_DEFAULT, device: int | None = None, stream=None,
          allocator="torch") -> Handle:
    """Build a format.

    allocator: "torch" (default) routes every device allocation of the build and of the handle
            through torch's caching allocator (vf_allocator); None uses the library's cudaMalloc; an
            Allocator instance is passed through as is.

    volume: a dense CUDA tensor (Rz, Ry, Rx) int32/uint32 RGBA (0 = empty), or a tuple
            (keys int64 CUDA tensor x|y<<21|z<<42, rgba int32 CUDA tensor, dims (Rx,Ry,Rz)).
    signature: paper signature text (e.g. "R(4^3) G(7)") or a Level array.
    """
    import torch
    levels = parse_format(signature) if isinstance(signature, str) else signature
    sig = format_to_string(levels)
    v = Volume()
    if isinstance(volume, tuple):
        keys, vals, dims = volume
        v.kind = VF_VOL_SPARSE_DEVICE
        for a in range(3):
            v.dims[a] = dims[a]
        v.n_voxels = keys.shape[0]
        v.keys = keys.data_ptr() if keys.numel() else None
        v.values = vals.data_ptr() if vals.numel() else None
        dev = keys.device
    else:
        assert volume.is_cuda and volume.dim() == 3 and volume.is_contiguous()
        v.kind = VF_VOL_DENSE_DEVICE
        Rz, Ry, Rx = volume.shape
        v.dims[0], v.dims[1], v.dims[2] = Rx, Ry, Rz
        v.rgba = volume.data_ptr()
        dev = volume.device
    if device is None:
        device = dev.index if dev.index is not None else torch.cuda.current_device()
    out = ctypes.c_void_p(0)
    used = _u64(0)
    if isinstance(allocator, Allocator):  # a caller-supplied vf_allocator (kept alive by the caller)
        alloc = ctypes.byref(allocator)
    else:
        alloc = ctypes.byref(TORCH_ALLOCATOR) if allocator == "torch" else None
    _check(_lib.vf_build(ctypes.byref(v), levels, len(levels), flags, alloc, device, _stream_ptr(stream),
                         ctypes.byref(out), ctypes.byref(used)))
    h = Handle(out, sig, levels, used.value)
    _LIVE.add(h)
    return h
