"""B200-native (sm_100a) stereo hot path of Chang & Maruyama, arXiv 2212.00488.

The compute path lives in the C-ABI library ``libstereo_b200.so`` (CUDA kernels
for sm_100a, declared in ``include/stereo.h``).  ``paper_2212_00488_b200.abi``
is the thin ctypes binding; importing this package does not load the library,
so the synthetic generators (``synth``) stay importable on a CPU-only box.
"""
__all__ = ["abi", "synth"]
