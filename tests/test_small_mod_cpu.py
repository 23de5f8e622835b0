"""The 32-bit-fold remainder of the VIX receiver draws (vix.cu SmallMod /
small_mod: x % (2R+1) for 64-bit splitmix outputs, R <= 255) restated in
Python: the constants make_smallmod picks and the fold sequence give x % d for
every d the engine can use, on random and edge-case x."""
import random


def make_smallmod(d):
    k32, k20 = (1 << 32) % d, (1 << 20) % d
    nmax = ((((d << 32) >> 20) + 1) * (d - 1)) + (1 << 20)
    for sh in range(31, 0, -1):
        P = 1 << (32 + sh)
        m = -(-P // d)
        if m >= 1 << 32:
            continue
        e = m * d - P
        assert e * nmax < P
        return k32, k20, m, sh
    raise AssertionError(d)


def small_mod(d, c, x):
    k32, k20, m, sh = c
    t = (x >> 32) * k32 + (x & 0xffffffff)
    assert t < 1 << 41
    n = ((t >> 20) * k20 + (t & 0xfffff)) & 0xffffffff
    assert n < 1 << 31
    q = ((n * m) >> 32) >> sh
    return n - q * d


def test_small_mod_all_spans():
    rng = random.Random(7)
    edge = [0, 1, (1 << 64) - 1, (1 << 63), (1 << 32) - 1, 1 << 32, (1 << 41) - 1]
    for R in range(1, 256):
        d = 2 * R + 1
        c = make_smallmod(d)
        xs = edge + [rng.getrandbits(64) for _ in range(300)] + [d * rng.getrandbits(55) + rng.randrange(d) for _ in range(50)]
        for x in xs:
            assert small_mod(d, c, x) == x % d, (d, x)
