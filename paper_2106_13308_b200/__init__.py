"""B200-native VQMC Max-Cut training step (arXiv 2106.13308), drop-in for the reference's
C++ API (see include/vqmc_b200.h and DESIGN.md).  The compute path is libvqmc_b200.so
(hand-written sm_100a CUDA); this package is the Python mirror of the reference API."""
from . import _capi  # noqa: F401  (fails loudly when the CUDA library is missing)
