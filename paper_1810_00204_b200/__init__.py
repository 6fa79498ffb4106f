"""B200-native QV-Tree Search hot path (arXiv 1810.00204): libqvts.so (sm_100a CUDA + C ABI,
include/qvts.h) and its thin ctypes binding.  See DESIGN.md."""
from .qvts import *  # noqa: F401,F403
from .qvts import Model, QvtsError, lib  # noqa: F401
