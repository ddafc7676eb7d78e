"""B200-native (sm_100a) Modalities data-parallel training step.

Host code in Python mirrors the reference's component interfaces; all compute
runs in hand-written CUDA kernels behind the C-ABI in include/b2s.h
(libb2s.so, loaded by ``_lib``). See DESIGN.md.
"""

__version__ = "0.1.0"
