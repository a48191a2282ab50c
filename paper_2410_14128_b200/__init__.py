"""paper_2410_14128_b200 — B200-native first-hit ray tracing through hybrid voxel formats
(arXiv 2410.14128, "Hybrid Voxel Formats for Efficient Ray Tracing").

The product is libvf.so (C ABI in include/vf.h, CUDA sources in csrc/); ``vf`` is its thin
ctypes binding. Importing this package fails loudly if libvf.so has not been built.
"""
from . import vf  # noqa: F401
from .vf import Handle, VfError, build, format_resolution, format_to_string, parse_format  # noqa: F401

__all__ = ["vf", "Handle", "VfError", "build", "parse_format", "format_to_string", "format_resolution"]
