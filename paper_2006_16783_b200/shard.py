"""Row-band multi-GPU orchestration of the siting pipeline.

Rank k owns a contiguous band of FINDMAX block rows and holds terrain for the
band +- (roi+1) rows.  VIX, FINDMAX and VIEWSHED run independently per rank
(no data-path collective).  Global candidate ids are the exclusive prefix of
the per-band counts plus the local index, which reproduces single-GPU block
order.  SITE is the one exchange: every round each rank
reports its best (gain << 32 | ~gid) key.  Host rounds reduce the keys
(allreduce MAX) and the owner of the winner contributes its window and packed
words to an allreduce SUM that every other rank feeds zeros into (a broadcast
whose root is data-dependent).  Device rounds use one collective instead: each
rank contributes {its best key, that candidate's window and words}, one
allgather delivers every rank's entry, and each rank selects the largest key
(TXS_SHARD_EXCHANGE=reduce keeps the two-allreduce form).  Every rank then ORs
the window into its held cumulative rows and updates its local gains.  Stop
rules (decision D9) are evaluated identically on every rank from that key.

The default with device rounds (TXS_SHARD_EXCHANGE=replicate) needs no
collective per round at all: one allgather of every band's packed viewsheds,
then every rank runs the single-GPU SITE loop (~6 us per round at roi 100,
against a collective's latency per round) on the gathered set.

`ranks` is the list of (engine, band index) pairs this process drives: one per
process with TorchComm over NCCL (one GPU each), or several on one device with
LocalComm (the single-GPU emulation the tests use).  An "engine" is anything
with the shard methods of paper_2006_16783_b200.Engine.
"""
import os

import numpy as np

STOP_TARGET, STOP_ZERO, STOP_EXHAUSTED, STOP_MAX = "target-reached", "zero-gain", "exhausted", "max-selected"


def plan_bands(nrows, block, world):
    """Split the ceil(nrows/block) FINDMAX block rows over `world` ranks as
    evenly as possible; returns [(row_begin, row_end)].  A world larger than
    the block rows is rejected: a rank without a band would leave its peers
    blocked in the per-round collectives (txs_plan_bands refuses it likewise)."""
    nb = -(-nrows // block)
    if world < 1 or world > nb:
        raise ValueError(f"{world} ranks > {nb} FINDMAX block rows ({nrows} rows / block {block})")
    base, extra = divmod(nb, world)
    out, b = [], 0
    for k in range(world):
        cnt = base + (1 if k < extra else 0)
        out.append((min(nrows, b * block), min(nrows, (b + cnt) * block)))
        b += cnt
    return out


class LocalComm:
    """Collectives over a single process (all ranks local)."""
    world = 1

    def max_i64(self, x):
        return int(x)

    def sum_i64(self, arr):
        return arr

    def allgather_i64(self, arr):
        return np.asarray(arr, np.int64)

    # device-round collectives over the local ranks' device buffers (tests:
    # every engine's stream is drained, the reduction runs on torch's stream)
    def max_dev(self, tensors, engines):
        return self._reduce_dev(tensors, engines, "max")

    def sum_dev(self, tensors, engines):
        return self._reduce_dev(tensors, engines, "sum")

    def allgather_dev(self, sends, recvs, engines):
        import torch
        for e in engines:
            e.synchronize()
        cat = torch.cat(sends)
        for r in recvs:
            r.copy_(cat)
        torch.cuda.synchronize()

    @staticmethod
    def _reduce_dev(tensors, engines, op):
        import torch
        for e in engines:
            e.synchronize()
        if len(tensors) > 1:
            st = torch.stack(tensors)
            red = st.max(0).values if op == "max" else st.sum(0)
            for t in tensors:
                t.copy_(red)
            torch.cuda.synchronize()


class TorchComm:
    """Collectives through torch.distributed (NCCL on GPUs, gloo on CPU).  Keys
    are < 2^63 (gain < 2^31), so signed int64 MAX is exact; the winner payload
    is reinterpreted as int64 for a SUM with zeros (bit-exact)."""

    def __init__(self, device="cpu", graphs=True):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.device = torch, dist, device
        self.world = dist.get_world_size()
        self.graphs = graphs and str(device).startswith("cuda")   # capture device rounds as CUDA graphs

    def max_i64(self, x):
        t = self.torch.tensor([int(x)], dtype=self.torch.int64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return int(t.item())

    def sum_i64(self, arr):
        t = self.torch.from_numpy(np.ascontiguousarray(arr).view(np.int64).copy()).to(self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return t.cpu().numpy().view(np.uint64)

    def allgather_i64(self, arr):
        a = np.ascontiguousarray(arr, np.int64)
        t = self.torch.from_numpy(a.copy()).to(self.device)
        outs = [self.torch.zeros_like(t) for _ in range(self.world)]
        self.dist.all_gather(outs, t)
        return np.concatenate([o.cpu().numpy() for o in outs])

    # device-round collectives: issued on the engine's stream, so they order
    # with its kernels without any host wait (one engine per process)
    def max_dev(self, tensors, engines):
        self._on_stream(tensors[0], engines[0], self.dist.ReduceOp.MAX)

    def sum_dev(self, tensors, engines):
        self._on_stream(tensors[0], engines[0], self.dist.ReduceOp.SUM)

    def allgather_dev(self, sends, recvs, engines):
        s = self.torch.cuda.ExternalStream(engines[0].stream(), device=sends[0].device)
        with self.torch.cuda.stream(s):
            self.dist.all_gather_into_tensor(recvs[0], sends[0])

    def _on_stream(self, t, eng, op):
        s = self.torch.cuda.ExternalStream(eng.stream(), device=t.device)
        with self.torch.cuda.stream(s):
            self.dist.all_reduce(t, op=op)


def _mw(roi):
    s = 2 * roi + 1
    return (s * s + 63) // 64


def setup_sharded(ranks, cfg, nbands, host_terrain=None):
    """Give every local rank its band + (roi+1)-row halo of the configuration's
    terrain: generated on the device (cropped), or copied from `host_terrain`
    (the full grid, e.g. pinned host memory).  Returns the active ranks."""
    nr, nc, roi = cfg.nrows, cfg.ncols, cfg.roi
    bands = plan_bands(nr, cfg.block if cfg.block else max(1, roi), nbands)
    halo = roi + 1
    active = []
    for eng, k in ranks:
        r0, r1 = bands[k]
        if r1 <= r0:
            continue
        eng.set_shard(nr, nc, r0, r1, halo)
        if host_terrain is None:
            eng.generate_fractal(nr, nc, cfg.roughness, cfg.terrain_seed, cfg.zmin, cfg.zmax)
            if cfg.water_rows:
                eng.fill_rows(0, cfg.water_rows, 0)
        else:
            h0, hr, _, _ = eng.shard_info()
            eng.set_terrain(host_terrain[h0:h0 + hr])
        active.append((eng, k))
    return active


def run_sharded(ranks, comm, cfg, params, nbands, setup=True, with_cum=True, device_rounds=False):
    """Run one configuration (paper_2006_16783_b200.configs.Config) over row
    bands.  Returns dict(index,row,col,gain,coverage,stop,cum) with the global
    dense cumulative bitmap.  With setup=False the ranks already
    hold their terrain (setup_sharded).  device_rounds=True runs the SITE
    rounds on the device (txs_site_shard_*_dev): keys and winner payloads stay
    in device buffers and the two collectives per round are stream-ordered,
    so the host only polls for the stop every few rounds."""
    nr, nc, roi = cfg.nrows, cfg.ncols, cfg.roi
    bands = plan_bands(nr, cfg.block if cfg.block else max(1, roi), nbands)
    if setup:
        active = setup_sharded(ranks, cfg, nbands)
    else:
        active = [(e, k) for e, k in ranks if bands[k][1] > bands[k][0]]
    # ---- VIX + FINDMAX per band, global ids by prefix over band order --------
    counts = np.zeros(nbands, np.int64)
    for eng, k in active:
        if cfg.random_observers:
            eng.random_observers(cfg.random_observers, cfg.observer_seed)   # ids = global draw index
            counts[k] = 0
        else:
            eng.estimate_vix(params, copy=False)
            counts[k] = eng.find_candidates(params, copy=False)
    counts = comm.allgather_i64(counts).reshape(-1, nbands).sum(0)
    if cfg.random_observers:
        total_cand = cfg.random_observers
    else:
        prefix = np.concatenate([[0], np.cumsum(counts)[:-1]])
        for eng, k in active:
            eng.set_candidate_base(int(prefix[k]))
        total_cand = int(counts.sum())
    # ---- VIEWSHED per band --------------------------------------------------------
    mode = os.environ.get("TXS_SHARD_EXCHANGE") or "replicate"
    replicate = device_rounds and mode == "replicate"
    for eng, _ in active:
        eng.compute_all_viewsheds(params)
        if not replicate:
            eng.site_shard_begin(params)
    # ---- SITE ---------------------------------------------------------------------------
    if replicate:
        out = _replicated_site(active, comm, params, total_cand)
        if with_cum:
            out["cum"] = active[0][0].cumulative()   # every rank holds the whole grid's cum
        return out
    if device_rounds:
        out = _device_rounds(active, comm, total_cand, mode)
        if not with_cum:
            return out
        return _with_cum(out, active, comm, bands, nr, nc)
    total = float(nr) * float(nc)
    mw = _mw(roi)
    idx, rows, cols, gains, covs = [], [], [], [], []
    covered, stop = 0, STOP_EXHAUSTED
    target, max_sel = params.target_coverage, params.max_selected
    while True:
        if len(idx) >= total_cand:
            stop = STOP_EXHAUSTED
            break
        key = max([eng.site_shard_best() for eng, _ in active] + [0])
        key = comm.max_i64(key)
        g = key >> 32
        if g <= 0:
            stop = STOP_ZERO
            break
        gid = 0xFFFFFFFF - (key & 0xFFFFFFFF)
        payload = np.zeros(6 + mw, np.uint64)
        for eng, _ in active:
            ex = eng.site_shard_export(gid, roi)
            if ex is not None:
                r, c, win, words = ex
                payload[0], payload[1] = r, c
                payload[2:6] = win.astype(np.uint64)
                payload[6:] = words
        payload = comm.sum_i64(payload)
        r, c = int(payload[0]), int(payload[1])
        win = payload[2:6].astype(np.int32)
        words = np.ascontiguousarray(payload[6:])
        for eng, _ in active:
            eng.site_shard_apply(r, c, win, words)
        covered += g
        cov = covered / total
        idx.append(gid); rows.append(r); cols.append(c); gains.append(g); covs.append(cov)
        if cov >= target:
            stop = STOP_TARGET
            break
        if max_sel > 0 and len(idx) >= max_sel:
            stop = STOP_MAX
            break
    out = dict(index=np.array(idx, np.int64), row=np.array(rows, np.int32), col=np.array(cols, np.int32),
               gain=np.array(gains, np.int64), coverage=np.array(covs), stop=stop)
    if not with_cum:
        return out
    return _with_cum(out, active, comm, bands, nr, nc)


def _with_cum(out, active, comm, bands, nr, nc):
    """Global cumulative bitmap: each band's rows, summed (disjoint bits)."""
    nw = (nr * nc + 63) // 64
    cum = np.zeros(nw, np.uint64)
    for eng, k in active:
        r0, r1 = bands[k]
        part = eng.cumulative()
        bits = np.unpackbits(part.view(np.uint8), bitorder="little")[: nr * nc]
        mask = np.zeros(nr * nc, np.uint8)
        mask[r0 * nc: r1 * nc] = 1
        packed = np.packbits(np.concatenate([bits & mask, np.zeros(nw * 64 - nr * nc, np.uint8)]),
                             bitorder="little").view(np.uint64)
        cum |= packed
    out["cum"] = comm.sum_i64(cum)
    return out


def _replicated_site(active, comm, params, total_cand):
    """SITE without a collective per round: one allgather of every band's
    candidates and packed viewsheds (records of txs_viewshed_record_words), then
    the single-GPU SITE loop on the gathered set on every rank -- the same picks
    bit for bit (the gathered set is the single-GPU candidate list, each entry
    at its global id).  site_ms = device time of the pack + allgather (the
    engine's own SITE stage timer covers the rest)."""
    import torch
    from .api import record_words
    engines = [e for e, _ in active]
    rw = record_words(params.roi)
    n_local = max(e.num_candidates() for e in engines)
    n_max = max(1, int(comm.allgather_i64(np.array([n_local], np.int64)).max()))
    nranks = getattr(comm, "world", 1) if len(engines) == 1 else len(engines)
    dev = torch.device("cuda", torch.cuda.current_device())
    torch.cuda.synchronize()
    engines[0].event_record(12)
    sends = [torch.empty(n_max * rw, dtype=torch.int64, device=dev) for _ in engines]
    for e, sd in zip(engines, sends):
        e.viewsheds_pack(n_max, sd.data_ptr())
    recvs = [torch.empty(nranks * n_max * rw, dtype=torch.int64, device=dev) for _ in engines]
    comm.allgather_dev(sends, recvs, engines)
    engines[0].event_record(13)
    gather_ms = engines[0].event_elapsed(12, 13)
    del sends
    res = None
    for e, rv in zip(engines, recvs):
        r = e.site_gathered(params, nranks * n_max, total_cand, rv.data_ptr())
        res = res or r
    del recvs
    res["site_ms"] = gather_ms
    res["rounds_mode"] = "replicated"
    res["exchange"] = "one allgather of every band's packed viewsheds, then the single-GPU SITE loop on every rank"
    return res


def _device_rounds(active, comm, total_cand, mode="gather", poll_every=16):
    """SITE rounds with the keys and payloads in device buffers (see run_sharded).
    With one engine per process (TorchComm) a block of `poll_every` rounds --
    engine kernels and NCCL collectives, all on the engine's stream -- is
    captured once as a CUDA graph and replayed until the device reports the stop."""
    import torch
    engines = [e for e, _ in active]
    pw = engines[0].site_shard_payload_words()
    dev = torch.device("cuda", torch.cuda.current_device())
    keys = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in engines]
    pays = [torch.zeros(pw, dtype=torch.int64, device=dev) for _ in engines]
    nranks = getattr(comm, "world", 1) if len(engines) == 1 else len(engines)
    sends = [torch.zeros(pw + 1, dtype=torch.int64, device=dev) for _ in engines]
    recvs = [torch.zeros(nranks * (pw + 1), dtype=torch.int64, device=dev) for _ in engines]
    torch.cuda.synchronize()

    def round_gather():
        # one collective: every rank contributes {its best key, that candidate's
        # payload}; the largest key among the gathered entries is the winner
        for e, k, sd in zip(engines, keys, sends):
            e.site_shard_best_dev(k.data_ptr())
            e.site_shard_export_keyed_dev(k.data_ptr(), sd.data_ptr())
        comm.allgather_dev(sends, recvs, engines)
        for e, k, p, rv in zip(engines, keys, pays, recvs):
            e.site_shard_select_dev(rv.data_ptr(), nranks, k.data_ptr(), p.data_ptr())
            e.site_shard_apply_dev(k.data_ptr(), p.data_ptr(), total_cand)

    def round_reduce():
        # two collectives: allreduce(MAX) of the keys, then the owner's payload
        # broadcast as an allreduce(SUM) with zeros
        for e, k in zip(engines, keys):
            e.site_shard_best_dev(k.data_ptr())
        comm.max_dev(keys, engines)
        for e, k, p in zip(engines, keys, pays):
            e.site_shard_export_dev(k.data_ptr(), p.data_ptr())
        comm.sum_dev(pays, engines)
        for e, k, p in zip(engines, keys, pays):
            e.site_shard_apply_dev(k.data_ptr(), p.data_ptr(), total_cand)

    # per-round exchange (TXS_SHARD_EXCHANGE=gather|reduce): one allgather of
    # {key, payload}, or two allreduces (MAX of keys, SUM broadcast of the payload)
    one_round = round_reduce if mode == "reduce" else round_gather

    engines[0].event_record(14)
    one_round()                                   # eager: sizes the device step log
    done = 1
    graph = None
    if len(engines) == 1 and getattr(comm, "graphs", False):
        try:
            s = torch.cuda.ExternalStream(engines[0].stream(), device=dev)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=s):
                for _ in range(poll_every):
                    one_round()
        except Exception as ex:                   # capture unsupported here: eager rounds
            import sys
            print(f"shard: CUDA-graph capture of the SITE rounds failed ({ex!r}); eager rounds", file=sys.stderr)
            graph = None
            torch.cuda.synchronize()
    res = engines[0].site_shard_result(max(1, total_cand))
    while res["stop"] is None and done <= total_cand + 1:
        if graph is not None:
            graph.replay()
            done += poll_every
        else:
            for _ in range(poll_every):
                one_round()
            done += poll_every
        res = engines[0].site_shard_result(max(1, total_cand))
    engines[0].event_record(15)
    res = engines[0].site_shard_result(max(1, total_cand))
    if res["stop"] is None:
        raise RuntimeError("sharded SITE did not stop")
    res["site_ms"] = engines[0].event_elapsed(14, 15)   # device time of the rounds (rank-local)
    res["rounds_mode"] = "graph" if graph is not None else "eager"
    res["exchange"] = ("one allgather of {key, payload} per round" if mode != "reduce"
                       else "two allreduces per round (MAX of keys, SUM broadcast of the payload)")
    return res
