"""CPU oracle for the all-fold CV XᵀX/XᵀY path — TEST INFRASTRUCTURE ONLY.

Restates the reference (/root/reference/proj/include/cvgram/{fast,baseline,
partition,core,random}.hpp) in plain C (``cvgram_oracle.c``), loaded here via
ctypes.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline legs may import this package; the product package never does.
"""
from .pyoracle import *  # noqa: F401,F403
