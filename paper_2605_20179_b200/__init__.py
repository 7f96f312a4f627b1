"""B200-native TIDE MoE layer-step (arXiv 2605.20179).

The product is libtide.so (C ABI in include/tide.h, sm_100a CUDA kernels in
csrc/); ``tide`` is its thin ctypes binding.  See DESIGN.md.
"""
from . import tide  # noqa: F401
from .tide import Context, TideError, make_desc, pack_expert, pack_layer  # noqa: F401
