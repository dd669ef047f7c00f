"""B200-native all-fold cross-validation XᵀX/XᵀY (arXiv 2401.13185).

``cvgram`` mirrors the reference C++ API (/root/reference/proj/include/cvgram);
``plan`` exposes the device-resident staged engine used by the benchmark and
the multi-GPU driver.  The sm_100a library is loaded at import: there is no
CPU fallback.
"""
from . import _lib

_lib.lib()  # fail loudly here if the engine was not built

from . import cvgram  # noqa: E402
from .cvgram import *  # noqa: E402,F401,F403

__all__ = ["cvgram"]
