"""B200-native multiple-observer siting engine (arXiv 2006.16783).

VIX -> FINDMAX -> VIEWSHED -> SITE as hand-written sm_100a kernels behind the
C-ABI in include/txsite_b200.h.  ``Engine`` mirrors the reference stage API.
"""
from .api import (Engine, TxsError, STOP, device_ok, make_params, max_words, partition,
                  ray_template, selftest)

__all__ = ["Engine", "TxsError", "STOP", "device_ok", "make_params", "max_words", "partition",
           "ray_template", "selftest"]
