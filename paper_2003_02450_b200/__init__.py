"""qswg: B200-native Lindblad expmv for quantum stochastic walks.

The product is libqswg.so (C++ host + sm_100a kernels, C ABI in
include/qswg.h); `paper_2003_02450_b200.api` is its Python mirror of the
reference library surface (importing it loads libqswg.so and fails loudly if
it is missing).  `graphs` holds the seeded synthetic workloads.
"""
