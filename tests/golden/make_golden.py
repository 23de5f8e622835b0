"""Regenerate tests/golden/kat.json from the REFERENCE's own code.

Run in the build container (where /root/reference exists and
oracle/_ref/libtxs_ref.so was compiled from the reference headers
proj/include/txsite/{grid_walk,rng,parallel}.hpp by oracle/Makefile):

    make -C oracle && python tests/golden/make_golden.py

Every vector below is produced by the reference's walk_crossings
(grid_walk.hpp:27-77), SplitMix64 / mix_seed (rng.hpp:9-36) and
parallel_for_chunks (parallel.hpp:20-42), plus the SPEC.md:147 fp64
formulation of estimate_vix built on that walk (oracle/ref_shim.cpp) — the
vectors pin the oracle's restatement, which the GPU is then checked against.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_lib as O  # noqa: E402


def main():
    R = O.ref()
    if R is None:
        raise SystemExit("oracle/_ref/libtxs_ref.so missing: build it where /root/reference exists")
    kat = {"source": "reference headers proj/include/txsite/*.hpp via oracle/ref_shim.cpp"}
    # rng.hpp
    seeds = [0, 1, 42, 1234567, 2**63 + 12345, 2**64 - 1]
    kat["splitmix_next"] = {str(s): [str(int(x)) for x in O.splitmix(s, 8, 0, 0, R)] for s in seeds}
    kat["splitmix_next_below"] = {f"{s}/{n}": [str(int(x)) for x in O.splitmix(s, 8, 1, n, R)]
                                  for s in seeds for n in (3, 201, 401, 501, 46400)}
    kat["splitmix_next_double_bits"] = {str(s): [str(int(x)) for x in O.splitmix(s, 4, 2, 0, R)] for s in seeds}
    trip = [(0, 0, 0), (42, 0, 0), (42, 1, 0), (42, 0, 1), (42, 500, 500), (7, 46399, 46399),
            (2**64 - 1, 123, 456), (99, 2**40, 3)]
    kat["mix_seed"] = [[str(a), str(b), str(c), str(int(R.ref_mix_seed(a, b, c)))] for a, b, c in trip]
    # grid_walk.hpp: full lists for short segments, hashes for many more
    rng = np.random.default_rng(20200630)
    short = [(0, 0, 3, 7, 0), (0, 0, 2, 4, 1), (5, 5, 5, 9, 0), (5, 5, 9, 5, 1), (3, 3, 0, 0, 0),
             (10, 10, 4, 13, 1), (0, 0, 6, 6, 0), (0, 0, 1, 0, 1), (0, 0, 0, 0, 1), (7, 2, 2, 9, 0)]
    for _ in range(20):
        r0, c0 = (int(x) for x in rng.integers(0, 50, 2))
        r1, c1 = (int(x) for x in rng.integers(0, 50, 2))
        short.append((r0, c0, r1, c1, int(rng.integers(0, 2))))
    lists = []
    for (r0, c0, r1, c1, e) in short:
        t, r, c, k = O.walk(r0, c0, r1, c1, e, R)
        lists.append({"seg": [r0, c0, r1, c1, e], "t": t.tolist(), "row": r.tolist(), "col": c.tolist(),
                      "kind": k.tolist()})
    kat["walk_lists"] = lists
    hashes = []
    for i in range(600):
        span = [60, 260, 600, 2000][i % 4]
        r0, c0 = (int(x) for x in rng.integers(0, 46400, 2))
        dr, dc = (int(x) for x in rng.integers(-span, span + 1, 2))
        if i % 7 == 0:
            dr = 0
        if i % 11 == 0:
            dc = dr
        e = i % 2
        h, n = O.walk_hash(r0, c0, r0 + dr, c0 + dc, e, R)
        hashes.append([r0, c0, r0 + dr, c0 + dc, e, str(h), n])
    h, n = O.walk_hash(46000, 46000, 45900, 46071, 0, R)
    hashes.append([46000, 46000, 45900, 46071, 0, str(h), n])
    kat["walk_hashes"] = hashes
    # parallel.hpp
    kat["chunks"] = [[n, t, O.chunks(n, t, R)] for n in (0, 1, 2, 10, 17, 1000, 4096) for t in (1, 2, 3, 8, 64)]
    # fp64 formulation of estimate_vix on the reference walk, for the
    # differing-bits count against the exact-arithmetic oracle (DESIGN.md §2 D2)
    z = O.generate_fractal(96, 96, 0.5, 7, 0, 4000)
    fp = np.zeros((96, 96), np.uint8)
    R.ref_estimate_vix_fp64(O._p(z), 96, 96, 20, 10, 10, 10, 99, 0, O._p(fp), 0, 96)
    kat["vix_fp64"] = {"terrain": "generate_fractal(96,96,0.5,7,0,4000)", "roi": 20, "ht": 10, "hr": 10,
                       "samples": 10, "seed": 99, "scores": fp.ravel().tolist()}
    # SPEC.md:147 fp64 LOS decisions of the reference walk on a tie-heavy terrain:
    # elevations quantized to multiples of 50 with a flat band, so the terrain
    # often touches the LOS exactly (grazing ties that fp64 rounding decides).
    zq = (O.generate_fractal(80, 80, 0.6, 31, 0, 600) // 50 * 50).astype(np.int16)
    zq[30:40, :] = 100
    rng = np.random.default_rng(1234)
    pairs = rng.integers(0, 80, size=(6000, 4)).astype(np.int64)
    vis = [int(R.ref_is_visible_fp64(O._p(zq), 80, 80, int(a), int(b), 0, int(c), int(d), 0))
           for a, b, c, d in pairs]
    kat["los_fp64_ties"] = {"terrain": "generate_fractal(80,80,0.6,31,0,600)//50*50, rows 30..39 = 100",
                            "ht": 0, "hr": 0, "pairs": pairs.ravel().tolist(), "visible": vis}
    fq = np.zeros((80, 80), np.uint8)
    R.ref_estimate_vix_fp64(O._p(zq), 80, 80, 15, 0, 0, 12, 4242, 0, O._p(fq), 0, 80)
    kat["vix_fp64_ties"] = {"roi": 15, "ht": 0, "hr": 0, "samples": 12, "seed": 4242, "scores": fq.ravel().tolist()}
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kat, f, separators=(",", ":"))
    print("wrote", os.path.join(HERE, "kat.json"))


if __name__ == "__main__":
    main()
