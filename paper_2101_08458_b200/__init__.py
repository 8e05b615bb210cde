"""tzc-b200: B200-native (sm_100a) backend for the UNIT/tzc tensorized-instruction
compiler (arXiv 2101.08458).

The product is ``libtzc_b200.so`` (C++ tzc host library + tcgen05 CUDA kernels
behind the C ABI in ``include/tzc_b200.h``).  This package only loads it:

* :mod:`._capi`  — ctypes declarations of the C ABI
* :mod:`.device` — torch-tensor wrappers for the device-level entry points
* :mod:`.ops`    — the reference-facing op-level entry (op text + host buffers)
* :mod:`.workloads` — op-text generators (reference layouts + batched NHWC / ResNet-50 bank)
"""
from ._capi import TzcError, lib  # noqa: F401

__version__ = "0.1.0"
