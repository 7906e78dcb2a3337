"""B200-native (sm_100a) HALO quantized linear-layer training path.

Drop-in for the reference's HALO operator (HaloLinearLayerT, HaloScheme,
quantize/transform/qmatmul primitives and the HQ-FSDP protocol).  Compute
runs only in libhalo_b200.so (hand-written CUDA for sm_100a); importing
``paper_2501_02625_b200.halo`` fails loudly if the library is missing.
"""
from . import _lib  # noqa: F401

__all__ = ["halo", "fsdp"]
