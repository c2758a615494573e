"""B200-native residual path integral renderer (arXiv 2406.16302): sm_100a CUDA kernels behind the C ABI
of include/rr.h, with a thin ctypes binding.  See DESIGN.md."""
from .renderer import Renderer, RRError  # noqa: F401
