"""B200-native multiple-observer siting engine (arXiv 2006.16783).

VIX -> FINDMAX -> VIEWSHED -> SITE as hand-written sm_100a kernels behind the
C-ABI in include/txsite_b200.h.  ``Engine`` mirrors the reference stage API.

The engine names load lazily (PEP 562): importing a pure-Python submodule such
as ``paper_2006_16783_b200.configs`` does not map libtxsite_b200.so, so
bench.py's CPU reference arm runs without the engine library in the process.
Touching any engine name loads the library (and fails loudly without it).
"""
__all__ = ["Engine", "Group", "plan_bands", "TxsError", "STOP", "LOS_ARITH", "device_ok", "make_params", "max_words", "partition",
           "ray_template", "selftest"]


def __getattr__(name):
    if name in __all__:
        from . import api
        return getattr(api, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
