"""B200-native LithOS TPC scheduler: the reference's gpuos:: scheduling path
(TPC quotas with stealing and revocation, kernel atomization, right-sizing)
on a persistent sm_100a dispatcher. See DESIGN.md.

The native library is the product (lib/libgpuos_b200.so); `api` binds it.
"""
from . import api  # noqa: F401

__all__ = ["api"]
