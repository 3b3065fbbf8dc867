"""B200-native matrix-free PA Lagrange hot path (arXiv 2112.07075 / ale_minihydro drop-in).

Public modules mirror the reference package: `tensor_basis`, `fespace`,
`operators`, `hydro`, `kernel_exec`.  The compute runs in the in-tree
sm_100a library `libb200hydro.so` (C-ABI: include/b200hydro.h).
"""

__version__ = "0.1.0"
