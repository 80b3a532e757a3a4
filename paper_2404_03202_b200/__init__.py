"""B200-native ERP Gaussian-splatting hot path (OmniGS, arXiv 2404.03202).

The product is ``libosplat_b200.so`` (C ABI in include/osplat.h, sm_100a kernels in csrc/);
``native`` is its ctypes mirror of the reference render / backward / adam_step interface.

``scenes`` (numpy scene generators) imports without the library; the product names below load
``libosplat_b200.so`` on first access and fail loudly if it has not been built. (The reference
arm of bench.py imports ``scenes`` only, so that process never maps the product library.)
"""
from . import scenes  # noqa: F401

_NATIVE = ("Config", "Context", "Frame", "HostCloud", "OsplatError", "launch_count", "osplat_render", "version")

__all__ = list(_NATIVE) + ["scenes"]


def __getattr__(name):
    if name in _NATIVE:
        from . import native
        return getattr(native, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
