"""ctypes bindings to the CPU oracle (oracle/liboracle.so) and, where it was
built, the reference-header shim (oracle/_ref/libtxs_ref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs; never by the product.
"""
import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.environ.get("ORACLE_SO", os.path.join(ROOT, "oracle", "liboracle.so"))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libtxs_ref.so")

i64, u64, i32, dbl, vp = C.c_int64, C.c_uint64, C.c_int32, C.c_double, C.c_void_p


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"oracle not built: {ORACLE_SO} (run `make -C oracle`)")
        L = C.CDLL(ORACLE_SO)
        L.txo_mix_seed.restype = u64
        L.txo_mix_seed.argtypes = [u64, u64, u64]
        L.txo_splitmix.argtypes = [u64, i64, C.c_int, u64, vp]
        L.txo_walk.restype = i64
        L.txo_walk.argtypes = [i64, i64, i64, i64, C.c_int, vp, vp, vp, vp, i64]
        L.txo_walk_hash.restype = u64
        L.txo_walk_hash.argtypes = [i64, i64, i64, i64, C.c_int, vp]
        L.txo_chunks.restype = i64
        L.txo_chunks.argtypes = [i64, C.c_uint, vp]
        L.txo_generate_fractal.restype = C.c_int
        L.txo_generate_fractal.argtypes = [i64, i64, dbl, u64, i32, i32, vp, C.c_uint]
        L.txo_is_visible.restype = C.c_int
        L.txo_is_visible.argtypes = [vp, i64, i64, i64, i64, i64, i64, i64, i64, C.c_int]
        L.txo_is_visible_batch.argtypes = [vp, i64, i64, vp, i64, i64, i64, vp, C.c_uint, C.c_int]
        L.txo_estimate_vix.argtypes = [vp, i64, i64, i64, i64, i64, i64, u64, C.c_uint, vp, i64, i64, C.c_int]
        L.txo_find_candidates.restype = i64
        L.txo_find_candidates.argtypes = [vp, i64, i64, i64, i64, vp, vp, vp, i64]
        L.txo_midpoint_circle_count.restype = i64
        L.txo_midpoint_circle_count.argtypes = [i64]
        L.txo_template.restype = i64
        L.txo_template.argtypes = [i64, vp, vp, vp, vp, vp, i64, i64, vp]
        L.txo_viewsheds.argtypes = [vp, i64, i64, i64, i64, i64, i64, vp, vp, vp, vp, i64, C.c_uint, C.c_int]
        L.txo_marginal_gain.restype = i64
        L.txo_marginal_gain.argtypes = [vp, vp, vp, i64, i64, C.c_int]
        L.txo_site.restype = C.c_int
        L.txo_site.argtypes = [i64, vp, vp, vp, vp, i64, i64, i64, dbl, i64, C.c_int,
                               vp, vp, vp, vp, vp, i64, vp, vp]
        _lib = L
    return _lib


def ref():
    """The reference-header shim, or None where /root/reference was absent at build."""
    global _ref
    if _ref is None and os.path.exists(REF_SO):
        R = C.CDLL(REF_SO)
        R.ref_mix_seed.restype = u64
        R.ref_mix_seed.argtypes = [u64, u64, u64]
        R.ref_splitmix.argtypes = [u64, i64, C.c_int, u64, vp]
        R.ref_walk.restype = i64
        R.ref_walk.argtypes = [i64, i64, i64, i64, C.c_int, vp, vp, vp, vp, i64]
        R.ref_walk_hash.restype = u64
        R.ref_walk_hash.argtypes = [i64, i64, i64, i64, C.c_int, vp]
        R.ref_chunks.restype = i64
        R.ref_chunks.argtypes = [i64, C.c_uint, vp]
        R.ref_is_visible_fp64.restype = C.c_int
        R.ref_is_visible_fp64.argtypes = [vp, i64, i64, i64, i64, i64, i64, i64, i64]
        R.ref_estimate_vix_fp64.argtypes = [vp, i64, i64, i64, i64, i64, i64, u64, C.c_uint, vp, i64, i64]
        _ref = R
    return _ref


# ---- thin numpy wrappers ----------------------------------------------------

def splitmix(seed, n, mode=0, arg=0, L=None):
    out = np.zeros(n, np.uint64)
    (L or lib()).txo_splitmix(seed, n, mode, arg, _p(out)) if L is None else L.ref_splitmix(seed, n, mode, arg, _p(out))
    return out


def walk(r0, c0, r1, c1, include_end, L=None):
    f = (lib().txo_walk if L is None else L.ref_walk)
    n = f(r0, c0, r1, c1, int(include_end), None, None, None, None, 0)
    t, r, c = (np.zeros(n) for _ in range(3))
    k = np.zeros(n, np.int32)
    f(r0, c0, r1, c1, int(include_end), _p(t), _p(r), _p(c), _p(k), n)
    return t, r, c, k


def walk_hash(r0, c0, r1, c1, include_end, L=None):
    f = (lib().txo_walk_hash if L is None else L.ref_walk_hash)
    cnt = C.c_int64(0)
    h = f(r0, c0, r1, c1, int(include_end), C.byref(cnt))
    return int(h), int(cnt.value)


def chunks(n, threads, L=None):
    out = np.zeros(2 * max(threads, 1) + 2, np.int64)
    f = (lib().txo_chunks if L is None else L.ref_chunks)
    m = f(n, threads, _p(out))
    return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(m)]


def generate_fractal(nrows, ncols, roughness, seed, zmin, zmax, threads=0):
    z = np.zeros((nrows, ncols), np.int16)
    rc = lib().txo_generate_fractal(nrows, ncols, roughness, seed, zmin, zmax, _p(z), threads)
    if rc != 0:
        raise ValueError("generate_fractal: invalid arguments")
    return z


# LOS arithmetic (txs_params.los_arith): "fp64" = SPEC.md:147's formula, the
# reference's and the engine's default; "exact" = exact rationals (SPEC.md:120's
# real-number predicate; differs from fp64 only at exact grazing ties).
ARITH = {"fp64": 0, "exact": 1, "fp64-euclid": 2}   # fp64-euclid: viewsheds only (oracle.cpp)


def is_visible(z, tr, tc, ht, rr, rc, hr, arith="fp64"):
    z = np.ascontiguousarray(z, np.int16)
    return bool(lib().txo_is_visible(_p(z), z.shape[0], z.shape[1], tr, tc, ht, rr, rc, hr, ARITH[arith]))


def is_visible_batch(z, pairs, ht, hr, threads=0, arith="fp64"):
    z = np.ascontiguousarray(z, np.int16)
    pairs = np.ascontiguousarray(pairs, np.int32)
    out = np.zeros(len(pairs), np.uint8)
    lib().txo_is_visible_batch(_p(z), z.shape[0], z.shape[1], _p(pairs), len(pairs), ht, hr, _p(out), threads,
                               ARITH[arith])
    return out


def estimate_vix(z, roi, ht, hr, samples, seed, threads=0, rows=None, arith="fp64"):
    z = np.ascontiguousarray(z, np.int16)
    out = np.zeros(z.shape, np.uint8)
    rb, re = rows if rows is not None else (0, z.shape[0])
    lib().txo_estimate_vix(_p(z), z.shape[0], z.shape[1], roi, ht, hr, samples, seed, threads, _p(out), rb, re,
                           ARITH[arith])
    return out


def estimate_vix_rows(z, roi, ht, hr, samples, seed, rows, threads=0, arith="fp64"):
    """VixMap rows `rows` only (len(rows) x ncols), same values as estimate_vix."""
    L = lib()
    L.txo_estimate_vix_rows.argtypes = [vp, i64, i64, i64, i64, i64, i64, u64, C.c_uint, vp, i64, vp, C.c_int]
    z = np.ascontiguousarray(z, np.int16)
    rows = np.ascontiguousarray(rows, np.int64)
    out = np.zeros((len(rows), z.shape[1]), np.uint8)
    L.txo_estimate_vix_rows(_p(z), z.shape[0], z.shape[1], roi, ht, hr, samples, seed, threads, _p(rows), len(rows),
                            _p(out), ARITH[arith])
    return out


def popcounts(words):
    """Per-row popcount of a 2-D uint64 array."""
    return np.bitwise_count(np.ascontiguousarray(words, np.uint64)).sum(axis=-1, dtype=np.int64)


def find_candidates(scores, block_width, per_block):
    scores = np.ascontiguousarray(scores, np.uint8)
    nr, nc = scores.shape
    n = lib().txo_find_candidates(_p(scores), nr, nc, block_width, per_block, None, None, None, 0)
    rows, cols, sc = (np.zeros(n, np.int32) for _ in range(3))
    lib().txo_find_candidates(_p(scores), nr, nc, block_width, per_block, _p(rows), _p(cols), _p(sc), n)
    return rows, cols, sc


def ray_template(roi):
    nc = C.c_int64(0)
    nr = lib().txo_template(roi, None, None, None, None, None, 0, 0, C.byref(nc))
    p, q = np.zeros(nr, np.int32), np.zeros(nr, np.int32)
    cb = np.zeros(nr + 1, np.int64)
    ca, cc = np.zeros(nc.value, np.int32), np.zeros(nc.value, np.int32)
    lib().txo_template(roi, _p(p), _p(q), _p(cb), _p(ca), _p(cc), nr, nc.value, None)
    return p, q, cb, ca, cc


def max_words(roi):
    s = 2 * roi + 1
    return (s * s + 63) // 64


def viewsheds(z, roi, ht, hr, rows, cols, threads=0, arith="fp64"):
    z = np.ascontiguousarray(z, np.int16)
    rows = np.ascontiguousarray(rows, np.int32)
    cols = np.ascontiguousarray(cols, np.int32)
    n = len(rows)
    stride = max_words(roi)
    wins = np.zeros((n, 4), np.int32)
    words = np.zeros((n, stride), np.uint64)
    lib().txo_viewsheds(_p(z), z.shape[0], z.shape[1], roi, ht, hr, n, _p(rows), _p(cols),
                        _p(wins), _p(words), stride, threads, ARITH[arith])
    return wins, words


def marginal_gain(win, v, cum, nrows, ncols, bitloop=False):
    win = np.ascontiguousarray(win, np.int32)
    v = np.ascontiguousarray(v, np.uint64)
    cum = np.ascontiguousarray(cum, np.uint64)
    return int(lib().txo_marginal_gain(_p(win), _p(v), _p(cum), nrows, ncols, int(bitloop)))


STOP_NAMES = {0: "target-reached", 1: "zero-gain", 2: "exhausted", 3: "max-selected"}


def site(rows, cols, wins, words, nrows, ncols, target, max_selected=0, naive=False):
    rows = np.ascontiguousarray(rows, np.int32)
    cols = np.ascontiguousarray(cols, np.int32)
    wins = np.ascontiguousarray(wins, np.int32)
    words = np.ascontiguousarray(words, np.uint64)
    n = len(rows)
    cap = n + 1
    idx = np.zeros(cap, np.int64)
    sr, sc = np.zeros(cap, np.int32), np.zeros(cap, np.int32)
    gain, cov = np.zeros(cap, np.int64), np.zeros(cap)
    ns = C.c_int64(0)
    cum = np.zeros((nrows * ncols + 63) // 64, np.uint64)
    stride = words.shape[1] if words.ndim == 2 else 0
    stop = lib().txo_site(n, _p(rows), _p(cols), _p(wins), _p(words), stride, nrows, ncols,
                          target, max_selected, int(naive), _p(idx), _p(sr), _p(sc), _p(gain),
                          _p(cov), cap, C.byref(ns), _p(cum))
    k = ns.value
    return dict(index=idx[:k], row=sr[:k], col=sc[:k], gain=gain[:k], coverage=cov[:k],
                stop=STOP_NAMES[stop], cum=cum)


def elevation_between(z0, z1, m, n):
    L = lib()
    L.txo_elevation_between.restype = dbl
    L.txo_elevation_between.argtypes = [i64, i64, i64, i64]
    return L.txo_elevation_between(z0, z1, m, n)


def random_observers(nrows, ncols, n, seed):
    L = lib()
    L.txo_random_observers.argtypes = [i64, i64, i64, u64, vp, vp]
    rows, cols = np.zeros(n, np.int32), np.zeros(n, np.int32)
    L.txo_random_observers(nrows, ncols, n, seed, _p(rows), _p(cols))
    return rows, cols


def unpack_window(win, words):
    """Window bitmap as a (h, w) uint8 array (LSB-first row-major, D8)."""
    h, w = int(win[2]), int(win[3])
    bits = np.unpackbits(np.ascontiguousarray(words, np.uint64).view(np.uint8), bitorder="little")
    return bits[: h * w].reshape(h, w)


def dense_bits(cum, nrows, ncols):
    bits = np.unpackbits(np.ascontiguousarray(cum, np.uint64).view(np.uint8), bitorder="little")
    return bits[: nrows * ncols].reshape(nrows, ncols)


def pack_dense(bits2d):
    flat = np.ascontiguousarray(bits2d, np.uint8).ravel()
    pad = (-len(flat)) % 64
    flat = np.concatenate([flat, np.zeros(pad, np.uint8)])
    return np.packbits(flat, bitorder="little").view(np.uint64).copy()


def viewshed_ties(z, roi, ht, hr, r, c):
    """(exact words, tie-cell words) of one viewshed (window layout, D8)."""
    L = lib()
    L.txo_viewshed_ties.argtypes = [vp, i64, i64, i64, i64, i64, i64, i64, vp, vp]
    z = np.ascontiguousarray(z, np.int16)
    w, t = np.zeros(max_words(roi), np.uint64), np.zeros(max_words(roi), np.uint64)
    L.txo_viewshed_ties(_p(z), z.shape[0], z.shape[1], roi, ht, hr, r, c, _p(w), _p(t))
    return w, t


def los_class(z, tr, tc, ht, rr, rc, hr):
    """1 blocked, 0 grazing tie (visible, touching), -1 visible with clearance."""
    L = lib()
    L.txo_los_class.restype = C.c_int
    L.txo_los_class.argtypes = [vp, i64, i64, i64, i64, i64, i64, i64, i64]
    z = np.ascontiguousarray(z, np.int16)
    return L.txo_los_class(_p(z), z.shape[0], z.shape[1], tr, tc, ht, rr, rc, hr)
