"""B200-native randUTV (arXiv:2002.06960, Sec. 3.1) behind a C ABI.

The product is ``librandutv.so`` (CUDA kernels for sm_100a + host driver,
``csrc/``, interface ``include/randutv.h``); ``randutv.py`` is its ctypes
binding.  ``inputs.py`` builds the seeded synthetic matrices of BASELINE.json,
``flops.py`` the algorithmic flop model used for GFLOP/s.  Importing the
package does not load the library; calling a compute entry point does, and
fails loudly if it is missing (there is no CPU fallback).
"""
