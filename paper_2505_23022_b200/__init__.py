"""B200-native (sm_100a) implementation of Scorpio's per-iteration scheduling hot
path (arXiv 2505.23022), behind the reference ``slosim`` scheduler/predictor API.

The compute path is ``lib/libscorpio_b200.so`` (hand-written CUDA, C ABI in
``include/scorpio_b200.h``); Python marshals reference-shaped objects to SoA
device buffers and back.  There is no CPU fallback.
"""

__version__ = "0.1.0"
