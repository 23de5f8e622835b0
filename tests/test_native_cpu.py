"""CPU-side checks of the native library: it loads, exports every symbol the
C-ABI header declares, its host-side helpers are exact, and it refuses to run
without an sm_100 device (no CPU fallback)."""
import os
import re

import numpy as np

import oracle_lib as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    import paper_2006_16783_b200._native as N
    hdr = open(os.path.join(ROOT, "include", "txsite_b200.h")).read()
    declared = set(re.findall(r"\b(txs_[a-z_]+)\(", hdr))   # (function-pointer fields are "type (*name)(")
    assert declared, "no declarations parsed"
    for name in sorted(declared):
        assert hasattr(N.lib, name), f"{name} declared in include/txsite_b200.h but not exported"
    assert declared == set(N.EXPORTS)
    assert N.lib.txs_abi_version() == 1


def test_selftest_exact_division():
    import paper_2006_16783_b200 as T
    assert T.selftest()


def test_ray_template_matches_oracle():
    import paper_2006_16783_b200 as T
    for R in (1, 2, 3, 5, 17, 30, 64, 100, 200, 250):
        a, b = T.ray_template(R), O.ray_template(R)
        for x, y in zip(a, b):
            assert np.array_equal(x, y), R


def test_partition_api():
    import paper_2006_16783_b200 as T
    assert T.partition(1000, 1000, 30) == (10, 100, 100)
    assert T.partition(32000, 32000, 1000) == (334, 96, 96)
    assert T.partition(46400, 46400, 2000) == (667, 70, 70)
    assert T.partition(46400, 46400, 100, 400) == (400, 116, 116)
    assert T.partition(4096, 4096, 200, 128) == (128, 32, 32)
    try:
        T.partition(100, 100, 2)
        raise AssertionError("roi < 3 must fail (SPEC.md:232)")
    except T.TxsError as e:
        assert e.status == "INVALID_ARGUMENT"


def test_no_cpu_fallback():
    import paper_2006_16783_b200 as T
    if T.device_ok():
        return   # on a B200 the context opens; covered by the gpu suite
    try:
        T.Engine(0)
        raise AssertionError("Engine must not open without an sm_100 device")
    except T.TxsError as e:
        assert e.status == "CUDA"
