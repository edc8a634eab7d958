"""B200-native matrix-free finite-element operator apply (arXiv 2509.10226 hot path).

Host-side setup mirrors the reference package ``tetmf`` (mesh, DoF map, basis
tables, geometry); the apply runs in hand-written sm_100a FP64 tensor-core
kernels in ``libtetmf_b200.so`` behind the C-ABI of ``include/tetmf_b200.h``.
"""

__version__ = "0.1.0"
