"""B200-native RLHF PPO step engine (arXiv 2312.11819 / FlexRLHF placement strategies).

Host engine in C++ (csrc/host), sm_100a kernels (csrc/kernels), C-ABI in
include/rlhf_engine.h + include/rlhf_kernels.h.  Python here is bindings only.
"""
from .capi import LIB_PATH, lib  # noqa: F401
