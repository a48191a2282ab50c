"""paper_2410_14128_b200 — B200-native first-hit ray tracing through hybrid voxel formats
(arXiv 2410.14128, "Hybrid Voxel Formats for Efficient Ray Tracing").

The product is libvf.so (C ABI in include/vf.h, CUDA sources in csrc/); ``vf`` is its thin
ctypes binding. The binding is imported lazily so that ``_build`` can compile libvf.so on a fresh
checkout; touching any public name (or ``import paper_2410_14128_b200.vf``) fails loudly if
libvf.so has not been built — there is no CPU fallback.
"""
import importlib

__all__ = ["vf", "Handle", "VfError", "build", "parse_format", "format_to_string", "format_resolution"]


def __getattr__(name):
    if name in __all__:
        vf = importlib.import_module(".vf", __name__)
        return vf if name == "vf" else getattr(vf, name)
    raise AttributeError(name)
