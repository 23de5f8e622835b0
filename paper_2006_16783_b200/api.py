"""Python face of the engine, mirroring the reference's stage API
(SPEC.md: terrain :22-104, los :117, vix :176, candidates :228/:238,
viewshed :285/:305, siting :364/:374/:384, cli :433) over the C-ABI.

Stage outputs stay resident in HBM inside an Engine; the methods copy to numpy
only when asked (``copy=True``), like the ``*_out`` pointers of the C-ABI.
"""
import ctypes as C

import numpy as np

from . import _native as N

STOP = N.STOP


class TxsError(RuntimeError):
    def __init__(self, status, message):
        super().__init__(f"{N.STATUS.get(status, status)}: {message}")
        self.status = N.STATUS.get(status, status)


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


LOS_ARITH = {"fp64": 0, "exact": 1}


def make_params(roi, tx_height=10, rx_height=10, samples=10, per_block=20, block_width=0,
                target=0.95, max_selected=0, seed=0, site_mode=0, los_arith="fp64"):
    """SiteParams plus block_width / seed / max_selected / site_mode /
    los_arith ("fp64" = SPEC.md:147's formula, the default; "exact" = exact rationals)."""
    return N.Params(roi=roi, tx_height=tx_height, rx_height=rx_height, samples_per_point=samples,
                    per_block=per_block, block_width=block_width, site_mode=site_mode,
                    los_arith=LOS_ARITH[los_arith],
                    target_coverage=target, max_selected=max_selected, seed=seed)


def partition(nrows, ncols, roi, block_width=0):
    """partition -> (block_width, blocks_x, blocks_y)."""
    bw, bx, by = C.c_int64(), C.c_int64(), C.c_int64()
    st = N.lib.txs_partition(nrows, ncols, roi, block_width, C.byref(bw), C.byref(bx), C.byref(by))
    if st:
        raise TxsError(st, "[findmax] partition: roi < 3 with the default block width, or bad dims")
    return bw.value, bx.value, by.value


def ray_template(roi):
    """The frozen D5 ray template (host-side; no GPU needed)."""
    nc = C.c_int64()
    nr = N.lib.txs_ray_template(roi, None, None, None, None, None, 0, 0, C.byref(nc))
    if nr < 0:
        raise TxsError(1, "bad roi")
    p, q = np.zeros(nr, np.int32), np.zeros(nr, np.int32)
    cb = np.zeros(nr + 1, np.int64)
    ca, cc = np.zeros(nc.value, np.int32), np.zeros(nc.value, np.int32)
    N.lib.txs_ray_template(roi, _p(p), _p(q), _p(cb), _p(ca), _p(cc), nr, nc.value, None)
    return p, q, cb, ca, cc


def selftest():
    return N.lib.txs_selftest() == 0


def device_ok():
    return bool(N.lib.txs_device_ok())


def record_words(roi):
    """u64 words per gathered viewshed record (txs_viewshed_record_words)."""
    return int(N.lib.txs_viewshed_record_words(roi))


def max_words(roi):
    s = 2 * roi + 1
    return (s * s + 63) // 64


class Engine:
    """One device context (txs_ctx).  Not thread-safe (the
    orchestrator is single-threaded)."""

    def __init__(self, device=0):
        h = C.c_void_p()
        st = N.lib.txs_create(device, C.byref(h))
        if st:
            raise TxsError(st, f"txs_create(device={device}) failed: no usable sm_100 device")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib = getattr(N, "lib", None)   # None during interpreter teardown
            if lib is not None:
                lib.txs_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _chk(self, st):
        if st:
            raise TxsError(st, N.lib.txs_last_error(self._h).decode())

    # ---- terrain ------------------------------------------------------------
    def set_terrain(self, z):
        z = np.ascontiguousarray(z, np.int16)
        self._chk(N.lib.txs_set_terrain(self._h, _p(z), z.shape[0], z.shape[1]))

    def generate_fractal(self, nrows, ncols, roughness, seed, zmin, zmax):
        self._chk(N.lib.txs_generate_fractal(self._h, nrows, ncols, roughness, seed, zmin, zmax))

    def fill_rows(self, row_begin, row_end, value):
        self._chk(N.lib.txs_fill_rows(self._h, row_begin, row_end, value))

    @property
    def dims(self):
        r, c = C.c_int64(), C.c_int64()
        self._chk(N.lib.txs_terrain_dims(self._h, C.byref(r), C.byref(c)))
        return r.value, c.value

    def terrain(self):
        nr, nc = self.dims
        z = np.empty((nr, nc), np.int16)
        self._chk(N.lib.txs_get_terrain(self._h, _p(z)))
        return z

    # ---- los ------------------------------------------------------------------
    def is_visible_batch(self, pairs, tx_height, rx_height, los_arith="fp64"):
        pairs = np.ascontiguousarray(pairs, np.int32).reshape(-1, 4)
        out = np.zeros(len(pairs), np.uint8)
        self._chk(N.lib.txs_is_visible_batch(self._h, _p(pairs), len(pairs), tx_height, rx_height,
                                             LOS_ARITH[los_arith], _p(out)))
        return out

    # ---- vix ------------------------------------------------------------------
    def estimate_vix(self, params, copy=True):
        out = np.empty(self.dims, np.uint8) if copy else None
        self._chk(N.lib.txs_estimate_vix(self._h, C.byref(params), _p(out)))
        return out

    def vix(self, row_begin=None, row_end=None):
        """Rows [row_begin, row_end) of the resident VixMap (default: all)."""
        nr, nc = self.dims
        rb = 0 if row_begin is None else row_begin
        re = nr if row_end is None else row_end
        out = np.empty((re - rb, nc), np.uint8)
        self._chk(N.lib.txs_get_vix(self._h, rb, re, _p(out)))
        return out

    def set_vix(self, scores):
        scores = np.ascontiguousarray(scores, np.uint8)
        self._chk(N.lib.txs_set_vix(self._h, _p(scores)))

    # ---- candidates -----------------------------------------------------------
    def find_candidates(self, params, copy=True):
        n = C.c_int64()
        self._chk(N.lib.txs_find_candidates(self._h, C.byref(params), C.byref(n), None, 0))
        return self.candidates() if copy else n.value

    def num_candidates(self):
        n = C.c_int64()
        self._chk(N.lib.txs_get_candidates(self._h, None, 0, C.byref(n)))
        return n.value

    def candidates(self):
        n = C.c_int64()
        self._chk(N.lib.txs_get_candidates(self._h, None, 0, C.byref(n)))
        buf = np.zeros((n.value, 4), np.int32)
        self._chk(N.lib.txs_get_candidates(self._h, _p(buf), n.value, None))
        return buf[:, 0].copy(), buf[:, 1].copy(), buf[:, 2].copy()

    def set_candidates(self, rows, cols, scores=None):
        n = len(rows)
        buf = np.zeros((n, 4), np.int32)
        buf[:, 0], buf[:, 1] = rows, cols
        if scores is not None:
            buf[:, 2] = scores
        self._chk(N.lib.txs_set_candidates(self._h, _p(buf), n))

    def random_observers(self, n, seed):
        self._chk(N.lib.txs_random_observers(self._h, n, seed))

    # ---- viewsheds --------------------------------------------------------------
    def compute_all_viewsheds(self, params):
        self._chk(N.lib.txs_compute_viewsheds(self._h, C.byref(params)))

    def viewsheds(self, roi, first=0, count=None):
        if count is None:
            n = C.c_int64()
            self._chk(N.lib.txs_get_candidates(self._h, None, 0, C.byref(n)))
            count = n.value - first
        stride = max_words(roi)
        wins = np.zeros((count, 4), np.int32)
        words = np.zeros((count, stride), np.uint64)
        pops = np.zeros(count, np.int64)
        self._chk(N.lib.txs_get_viewsheds(self._h, first, count, _p(wins), _p(words), stride, _p(pops)))
        return wins, words, pops

    def set_viewsheds(self, roi, rows, cols, wins, words):
        rows = np.ascontiguousarray(rows, np.int32)
        cols = np.ascontiguousarray(cols, np.int32)
        wins = np.ascontiguousarray(wins, np.int32)
        words = np.ascontiguousarray(words, np.uint64)
        self._chk(N.lib.txs_set_viewsheds(self._h, roi, len(rows), _p(rows), _p(cols), _p(wins), _p(words),
                                          words.shape[1]))

    # ---- siting -----------------------------------------------------------------
    def site(self, params, cap=None):
        if cap is None:
            n = C.c_int64()
            self._chk(N.lib.txs_get_candidates(self._h, None, 0, C.byref(n)))
            cap = n.value + 1
        steps = (N.Step * max(cap, 1))()
        ns, stop = C.c_int64(), C.c_int32()
        self._chk(N.lib.txs_site(self._h, C.byref(params), steps, cap, C.byref(ns), C.byref(stop)))
        return _steps_dict(steps, min(ns.value, cap), stop.value)

    def cumulative(self):
        nr, nc = self.dims
        out = np.zeros((nr * nc + 63) // 64, np.uint64)
        self._chk(N.lib.txs_get_cumulative(self._h, _p(out)))
        return out

    def marginal_gains(self, cum_dense):
        cum = np.ascontiguousarray(cum_dense, np.uint64)
        n = C.c_int64()
        self._chk(N.lib.txs_get_candidates(self._h, None, 0, C.byref(n)))
        out = np.zeros(max(n.value, 1), np.int64)
        self._chk(N.lib.txs_marginal_gains(self._h, _p(cum), _p(out)))
        return out[:n.value]

    # ---- pipeline ---------------------------------------------------------------
    def run_pipeline(self, params, cap=1 << 20):
        steps = (N.Step * cap)()
        ns, stop = C.c_int64(), C.c_int32()
        ms = (C.c_double * 4)()
        self._chk(N.lib.txs_run_pipeline(self._h, C.byref(params), steps, cap, C.byref(ns), C.byref(stop), ms))
        d = _steps_dict(steps, min(ns.value, cap), stop.value)
        d["stage_ms"] = dict(vix=ms[0], findmax=ms[1], viewshed=ms[2], site=ms[3])
        return d

    def run_pipeline_host(self, z, params, cap=1 << 20):
        """run_pipeline from a host terrain (row-major int16, ideally pinned):
        the upload overlaps VIX (txs_run_pipeline_host)."""
        z = np.ascontiguousarray(z, np.int16)
        steps = (N.Step * cap)()
        ns, stop = C.c_int64(), C.c_int32()
        ms = (C.c_double * 4)()
        self._chk(N.lib.txs_run_pipeline_host(self._h, _p(z), z.shape[0], z.shape[1], C.byref(params), steps, cap,
                                              C.byref(ns), C.byref(stop), ms))
        d = _steps_dict(steps, min(ns.value, cap), stop.value)
        d["stage_ms"] = dict(vix=ms[0], findmax=ms[1], viewshed=ms[2], site=ms[3])
        return d

    # ---- row-band shards --------------------------------------------
    def set_shard(self, nrows, ncols, row_begin, row_end, halo):
        self._chk(N.lib.txs_set_shard(self._h, nrows, ncols, row_begin, row_end, halo))

    def shard_info(self):
        a, b, c, d = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        self._chk(N.lib.txs_shard_info(self._h, C.byref(a), C.byref(b), C.byref(c), C.byref(d)))
        return a.value, b.value, c.value, d.value

    def set_candidate_base(self, gid0):
        self._chk(N.lib.txs_set_candidate_base(self._h, gid0))

    def site_shard_begin(self, params):
        self._chk(N.lib.txs_site_shard_begin(self._h, C.byref(params)))

    def site_shard_best(self):
        k = C.c_uint64()
        self._chk(N.lib.txs_site_shard_best(self._h, C.byref(k)))
        return k.value

    def site_shard_export(self, gid, roi):
        owned, r, c = C.c_int32(), C.c_int32(), C.c_int32()
        win = np.zeros(4, np.int32)
        words = np.zeros(max_words(roi), np.uint64)
        self._chk(N.lib.txs_site_shard_export(self._h, gid, C.byref(owned), C.byref(r), C.byref(c), _p(win),
                                              _p(words), len(words)))
        if not owned.value:
            return None
        return r.value, c.value, win, words

    def site_shard_apply(self, row, col, win, words):
        win = np.ascontiguousarray(win, np.int32)
        words = np.ascontiguousarray(words, np.uint64)
        self._chk(N.lib.txs_site_shard_apply(self._h, row, col, _p(win), _p(words)))

    # ---- device-resident shard rounds (pointers are device addresses, e.g. torch tensors' data_ptr())
    def site_shard_best_dev(self, d_key):
        self._chk(N.lib.txs_site_shard_best_dev(self._h, C.c_void_p(d_key)))

    def site_shard_export_dev(self, d_key, d_payload):
        self._chk(N.lib.txs_site_shard_export_dev(self._h, C.c_void_p(d_key), C.c_void_p(d_payload)))

    def site_shard_apply_dev(self, d_key, d_payload, total_candidates):
        self._chk(N.lib.txs_site_shard_apply_dev(self._h, C.c_void_p(d_key), C.c_void_p(d_payload), total_candidates))

    def site_shard_export_keyed_dev(self, d_key, d_out):
        self._chk(N.lib.txs_site_shard_export_keyed_dev(self._h, C.c_void_p(d_key), C.c_void_p(d_out)))

    def site_shard_select_dev(self, d_gathered, nranks, d_key, d_payload):
        self._chk(N.lib.txs_site_shard_select_dev(self._h, C.c_void_p(d_gathered), nranks, C.c_void_p(d_key),
                                                  C.c_void_p(d_payload)))

    def site_shard_payload_words(self):
        return int(N.lib.txs_site_shard_payload_words(self._h))

    def site_shard_result(self, cap):
        steps = (N.Step * max(1, cap))()
        ns, stop = C.c_int64(), C.c_int32()
        self._chk(N.lib.txs_site_shard_result(self._h, steps, cap, C.byref(ns), C.byref(stop)))
        d = _steps_dict(steps, min(ns.value, cap), 0)
        d["stop"] = STOP[stop.value] if stop.value >= 0 else None
        return d

    # ---- replicated SITE over gathered viewsheds ---------------------
    def viewsheds_pack(self, slots, d_records):
        """Resident viewsheds as `slots` records (txs_viewshed_record_words u64
        each) into the device buffer at d_records (stream-ordered); returns the
        record count."""
        n = C.c_int64()
        self._chk(N.lib.txs_viewsheds_pack(self._h, slots, C.c_void_p(d_records), C.byref(n)))
        return n.value

    def site_gathered(self, params, nrec, n_total, d_records, cap=None):
        cap = n_total + 1 if cap is None else cap
        steps = (N.Step * max(cap, 1))()
        ns, stop = C.c_int64(), C.c_int32()
        self._chk(N.lib.txs_site_gathered(self._h, C.byref(params), nrec, n_total, C.c_void_p(d_records), steps, cap,
                                          C.byref(ns), C.byref(stop)))
        return _steps_dict(steps, min(ns.value, cap), stop.value)

    def stream(self):
        return N.lib.txs_stream(self._h)

    def time_gain_pass(self, reps=5):
        """(ms per full gain pass, packed bytes per pass) against the current cum (after site())."""
        ms, b = C.c_double(), C.c_int64()
        self._chk(N.lib.txs_time_gain_pass(self._h, reps, C.byref(ms), C.byref(b)))
        return ms.value, b.value

    def measure_l2(self, nbytes=64 << 20, reps=20):
        """L2-resident read bandwidth in GB/s (txs_measure_cache_read)."""
        g = C.c_double()
        self._chk(N.lib.txs_measure_cache_read(self._h, nbytes, reps, C.byref(g)))
        return g.value

    def stats(self):
        s = N.Stats()
        self._chk(N.lib.txs_get_stats(self._h, C.byref(s)))
        return {k: (list(getattr(s, k)) if isinstance(getattr(s, k), C.Array) else getattr(s, k))
                for k, _ in N.Stats._fields_}

    def reset_stats(self):
        self._chk(N.lib.txs_reset_stats(self._h))

    def synchronize(self):
        self._chk(N.lib.txs_synchronize(self._h))

    def event_record(self, slot):
        self._chk(N.lib.txs_event_record(self._h, slot))

    def event_elapsed(self, a, b):
        ms = C.c_double()
        self._chk(N.lib.txs_event_elapsed(self._h, a, b, C.byref(ms)))
        return ms.value

    @property
    def handle(self):
        return self._h


def plan_bands(nrows, block, world):
    """txs_plan_bands: [(row_begin, row_end)] per rank over whole FINDMAX block rows."""
    out = np.zeros(2 * world, np.int64)
    st = N.lib.txs_plan_bands(nrows, block, world, _p(out))
    if st:
        raise TxsError(st, f"plan_bands: {world} ranks > block rows of {nrows} / {block}")
    return [(int(out[2 * k]), int(out[2 * k + 1])) for k in range(world)]


class Group:
    """Native multi-GPU group (txs_group, csrc/group.cu): N contexts as row-band
    shards of one grid, driven from this one process; SITE rounds exchange the
    winner over peer memory ("p2p", default), NCCL ("nccl") or the host ("host").
    `devices` may repeat a device (virtual ranks, tests).  `ops` (an address of a
    txs_engine_ops table) substitutes the stage entry points (CPU stand-in tests;
    host exchange only)."""

    def __init__(self, devices=(0,), exchange=None, ops=None):
        devs = np.ascontiguousarray(devices, np.int32)
        h = C.c_void_p()
        if ops is None:
            st = N.lib.txs_group_create(len(devs), _p(devs), C.byref(h))
        else:
            st = N.lib.txs_group_create_with_ops(len(devs), _p(devs), C.c_void_p(ops), C.byref(h))
        if st:
            raise TxsError(st, f"txs_group_create(devices={list(devices)}) failed")
        self._h = h
        self.n = len(devs)
        if exchange is not None:
            self.set_exchange(exchange)

    def close(self):
        if getattr(self, "_h", None):
            lib = getattr(N, "lib", None)
            if lib is not None:
                lib.txs_group_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _chk(self, st):
        if st:
            raise TxsError(st, N.lib.txs_group_last_error(self._h).decode())

    def set_exchange(self, name):
        if name == "nccl":
            # the engine dlopens libnccl.so.2 on first NCCL use and reuses a copy
            # already in the process: load torch's (newer) one first where torch is
            # installed, so a later `import torch` does not meet an older NCCL
            try:
                import torch  # noqa: F401
            except ImportError:
                pass
        self._chk(N.lib.txs_group_set_exchange(self._h, N.EXCHANGE[name]))

    def set_grid(self, nrows, ncols, params):
        self.dims = (nrows, ncols)
        self._chk(N.lib.txs_group_set_grid(self._h, nrows, ncols, C.byref(params)))

    def band(self, rank):
        a, b = C.c_int64(), C.c_int64()
        self._chk(N.lib.txs_group_band(self._h, rank, C.byref(a), C.byref(b)))
        return a.value, b.value

    def set_terrain(self, z):
        z = np.ascontiguousarray(z, np.int16)
        assert z.shape == tuple(self.dims)
        self._chk(N.lib.txs_group_set_terrain(self._h, _p(z)))

    def generate_fractal(self, roughness, seed, zmin, zmax):
        self._chk(N.lib.txs_group_generate_fractal(self._h, roughness, seed, zmin, zmax))

    def fill_rows(self, row_begin, row_end, value):
        self._chk(N.lib.txs_group_fill_rows(self._h, row_begin, row_end, value))

    def random_observers(self, n, seed):
        self._chk(N.lib.txs_group_random_observers(self._h, n, seed))

    def run_pipeline(self, params, cap=1 << 20):
        steps = (N.Step * cap)()
        ns, stop = C.c_int64(), C.c_int32()
        ms = (C.c_double * 4)()
        self._chk(N.lib.txs_group_run_pipeline(self._h, C.byref(params), steps, cap, C.byref(ns), C.byref(stop), ms))
        d = _steps_dict(steps, min(ns.value, cap), stop.value)
        d["stage_ms"] = dict(vix=ms[0], findmax=ms[1], viewshed=ms[2], site=ms[3])
        return d

    def cumulative(self):
        nr, nc = self.dims
        out = np.zeros((nr * nc + 63) // 64, np.uint64)
        self._chk(N.lib.txs_group_get_cumulative(self._h, _p(out)))
        return out

    def context(self, rank):
        return N.lib.txs_group_context(self._h, rank)


_STEP_DT = np.dtype([("index", "<i8"), ("row", "<i4"), ("col", "<i4"), ("gain", "<i8"), ("coverage", "<f8")])


def _steps_dict(steps, n, stop):
    a = np.frombuffer(C.string_at(C.addressof(steps), n * C.sizeof(N.Step)), dtype=_STEP_DT)
    return dict(index=a["index"].copy(), row=a["row"].copy(), col=a["col"].copy(),
                gain=a["gain"].copy(), coverage=a["coverage"].copy(), stop=STOP[stop])
