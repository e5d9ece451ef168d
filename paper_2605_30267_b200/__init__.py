"""B200-native hot path of Acc-Sinkhorn (arXiv 2605.30267).

The product is libotg.so (C-ABI: include/otg.h; sm_100a kernels in csrc/).
``paper_2605_30267_b200.ot`` mirrors the reference's ``ot::`` solver API on
top of it; ``include/otg.hpp`` is the same mirror for C++ callers.
"""
from . import ot  # noqa: F401
from .ot import *  # noqa: F401,F403

__all__ = ["ot"]
