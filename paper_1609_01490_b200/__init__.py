"""B200-native block-space triangular thread map lambda(omega) (arXiv:1609.01490).

The product is the C-ABI library ``libtri.so`` (include/tri.h) with hand-written
sm_100a kernels; ``paper_1609_01490_b200.tri`` is its thin ctypes binding.
Importing this package does not load the library (so the seeded input
generators work on a CPU-only box); the first call into ``tri`` does, and fails
loudly if it is missing.  There is no CPU fallback.
"""
__all__ = ["tri", "inputs", "dist"]
