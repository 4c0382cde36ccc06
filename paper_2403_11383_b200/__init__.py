"""B200-native (sm_100a) hot path of the SBS quadruped MPC iteration (arxiv 2403.11383).

The product is the C-ABI library ``libsbs.so`` built from ``csrc/`` (declared in
``include/sbs.h``).  ``binding.py`` is a thin ctypes binding with the same names;
it fails loudly when the library is missing -- there is no CPU fallback.
"""
