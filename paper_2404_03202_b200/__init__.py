"""B200-native ERP Gaussian-splatting hot path (OmniGS, arXiv 2404.03202).

The product is ``libosplat_b200.so`` (C ABI in include/osplat.h, sm_100a kernels in csrc/);
``native`` is its ctypes mirror of the reference render / backward / adam_step interface.
Importing the package loads the library and fails loudly if it has not been built.
"""
from . import scenes  # noqa: F401
from .native import (Config, Context, Frame, HostCloud, OsplatError, launch_count,  # noqa: F401
                     osplat_render, version)

__all__ = ["Config", "Context", "Frame", "HostCloud", "OsplatError", "launch_count", "osplat_render",
           "version", "scenes"]
