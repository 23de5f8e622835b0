#!/usr/bin/env python
"""Benchmark: end-to-end multiple-observer siting (VIX -> FINDMAX -> VIEWSHED
-> SITE) on a BASELINE.json configuration, one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl b200|reference]

A "step" is one full siting run of the configuration on its synthetic seeded
terrain.  `value` = device seconds per step with the terrain resident in HBM
(CUDA events on the engine stream, L2 flushed between steps, max over ranks);
`e2e` = the same run through the public API from pinned host memory: terrain
H2D, the pipeline, the step list and the cumulative bitmap D2H inside the
timed region.  `--impl reference` times the CPU oracle port (oracle/) on this
host's cores on a bounded, extrapolated sample of the same workload.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "end-to-end siting sec; VIEWSHED LOS samples/s; SITE GB/s vs HBM roofline"
DTYPE = "int32 exact LOS walks + fp64 tie re-test (SPEC.md:147 decisions); int16 terrain; u64 bitmaps"
DATA = "synthetic (seeded diamond-square terrain, BASELINE shapes)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", help="BASELINE config c1..c5 (default c3: the largest "
                    "single-GPU full pipeline)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--site-mode", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--threads", type=int, default=0, help="CPU threads for the oracle legs (0 = all)")
    ap.add_argument("--sharded", action="store_true", help="row-band path even at N=1 (NCCL world of 1)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ---------------------------------------------------------------------------
# CPU oracle leg (cpu_baseline and --impl reference).  Nothing here loads the
# engine library: paper_2006_16783_b200.configs is pure Python (the package
# resolves its engine names lazily).
# ---------------------------------------------------------------------------
# Per-config sample plan: VIX on every `vix_stride`-th row (offset rotating per
# step), VIEWSHED on every `vs_stride`-th candidate (rotating), FINDMAX in full,
# SITE in full (lazy greedy over every candidate's viewshed) except at C5,
# where 1M R=250 viewsheds cannot be built on the host in minutes: there SITE
# runs on the candidates of the top-left 1/16 sub-square with 1/16 of the picks.
SAMPLE_PLAN = {"c1": (1, 1, True), "c2": (1, 1, True), "c3": (256, 64, True), "c4": (1024, 64, True),
               "c5": (0, 1024, False)}


def config_dict(cfg):
    """The workload description both arms print (identical dicts)."""
    return {"workload": cfg.name, "nrows": cfg.nrows, "ncols": cfg.ncols, "roi": cfg.roi, "height": cfg.height,
            "vix_samples": cfg.samples, "block": cfg.block, "per_block": cfg.per_block,
            "random_observers": cfg.random_observers, "max_selected": cfg.max_selected,
            "target_coverage": cfg.target, "los_arith": "fp64 (SPEC.md:147)",
            "l2": "flushed between steps (256 MB write outside the timed events)"}


class CpuReference:
    """The oracle port (oracle/, std::thread workers like parallel.hpp) timed on
    this host on a bounded sample of the configuration, extrapolated per stage:
    est = VIX_sample * nrows / rows_sampled + FINDMAX + VIEWSHED_sample * n /
    sampled + SITE (full).  `cand` / `views`: the GPU's candidate list and
    downloaded viewsheds (cpu_baseline leg: the host work is then checked
    against the GPU's); without them (reference arm) candidates come from a
    seeded synthetic VixMap and the host builds every viewshed once at setup."""

    def __init__(self, cfg, threads, cand=None, views=None):
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import numpy as np
        import oracle_lib as O
        self.O, self.np, self.cfg = O, np, cfg
        self.threads = threads or (os.cpu_count() or 1)
        c = cfg
        t0 = time.perf_counter()
        self.z = O.generate_fractal(c.nrows, c.ncols, c.roughness, c.terrain_seed, c.zmin, c.zmax, self.threads)
        if c.water_rows:
            self.z[:c.water_rows] = 0
        self.vix_stride, self.vs_stride, self.site_full = SAMPLE_PLAN.get(c.name[:2], (64, 64, True))
        rng = np.random.default_rng(c.terrain_seed)
        if c.samples:
            # FINDMAX input for timing: a seeded synthetic VixMap (score levels 0..S)
            self.scores = rng.integers(0, c.samples + 1, (c.nrows, c.ncols)).astype(np.uint8)
        if cand is not None:
            self.cr, self.cc = cand
        elif c.samples:
            self.cr, self.cc, _ = O.find_candidates(self.scores, c.block, c.per_block)
        else:
            self.cr, self.cc = O.random_observers(c.nrows, c.ncols, c.random_observers, c.observer_seed)
        self.ncand = len(self.cr)
        if self.site_full:
            self.site_idx = np.arange(self.ncand)
            self.site_sel = c.max_selected
        else:
            self.site_idx = np.nonzero((self.cr < c.nrows // 4) & (self.cc < c.ncols // 4))[0]
            self.site_sel = max(1, c.max_selected // 16)
        if views is not None and self.site_full:
            self.sw, self.sv = views
        else:
            self.sw, self.sv = O.viewsheds(self.z, c.roi, c.height, c.height, self.cr[self.site_idx],
                                           self.cc[self.site_idx], self.threads)
        self.setup_s = time.perf_counter() - t0
        self.full = self.vix_stride <= 1 and self.vs_stride == 1 and self.site_full
        self.k = 0
        self.last = {}

    def step(self):
        """One sampled step: (estimated full-configuration seconds, per-stage
        estimates, measured wall seconds of the step)."""
        O, np, c = self.O, self.np, self.cfg
        parts, out = {}, {}
        w0 = time.perf_counter()
        if c.samples:
            rows = np.arange((self.k * 7919) % self.vix_stride, c.nrows, self.vix_stride)
            t0 = time.perf_counter()
            out["vix_rows"], out["vix"] = rows, O.estimate_vix_rows(self.z, c.roi, c.height, c.height, c.samples,
                                                                     c.vix_seed, rows, self.threads)
            parts["vix"] = (time.perf_counter() - t0) * c.nrows / len(rows)
            t0 = time.perf_counter()
            O.find_candidates(self.scores, c.block, c.per_block)
            parts["findmax"] = time.perf_counter() - t0
        # runs of 64 consecutive candidates (block-order neighbours share terrain in the host caches, as in
        # the full run), every vs_stride-th run
        runs = np.arange((self.k * 104729) % self.vs_stride, -(-self.ncand // 64), self.vs_stride)
        idx = (runs[:, None] * 64 + np.arange(64)[None, :]).ravel()
        idx = idx[idx < self.ncand]
        t0 = time.perf_counter()
        out["vs_idx"] = idx
        out["vs_wins"], out["vs_words"] = O.viewsheds(self.z, c.roi, c.height, c.height, self.cr[idx], self.cc[idx],
                                                      self.threads)
        parts["viewshed"] = (time.perf_counter() - t0) * self.ncand / len(idx)
        t0 = time.perf_counter()
        out["site"] = O.site(self.cr[self.site_idx], self.cc[self.site_idx], self.sw, self.sv, c.nrows, c.ncols,
                             c.target, self.site_sel)
        parts["site"] = (time.perf_counter() - t0) * (1 if self.site_full else 16)
        self.k += 1
        self.last = out
        return sum(parts.values()), parts, time.perf_counter() - w0

    def sample_desc(self):
        c = self.cfg
        s = []
        if c.samples:
            s.append("VIX on every %d-th row (%d of %d rows, x%d)" % (self.vix_stride, -(-c.nrows // self.vix_stride),
                                                                      c.nrows, self.vix_stride)
                     if self.vix_stride > 1 else "VIX in full")
            s.append("FINDMAX in full (seeded synthetic VixMap)")
        s.append("VIEWSHED on every %d-th run of 64 consecutive of %d observers (x%d)" % (self.vs_stride, self.ncand,
                                                                                        self.vs_stride)
                 if self.vs_stride > 1 else f"VIEWSHED in full ({self.ncand} observers)")
        s.append(f"SITE lazy greedy in full ({self.ncand} candidates, {self.site_sel} picks max)" if self.site_full
                 else f"SITE lazy greedy on the {len(self.site_idx)} candidates of the top-left 1/16 sub-square, "
                      f"{self.site_sel} picks (x16)")
        return "; ".join(s) + "; per-stage linear extrapolation to the full configuration"


def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    ref = CpuReference(cfg, args.threads)
    for _ in range(args.warmup):
        ref.step()
    vals, walls, parts_all = [], [], []
    for _ in range(args.steps):
        v, parts, wall = ref.step()
        vals.append(v)
        walls.append(wall)
        parts_all.append(parts)
    value = statistics.mean(vals)
    stages = {k: round(statistics.mean(p[k] for p in parts_all), 4) for k in parts_all[0]}
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(statistics.mean(walls) * 1e3, 2), "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp64 (SPEC.md:147 LOS arithmetic, oracle port)", "data": DATA,
        "config": config_dict(cfg),
        "cpu_baseline": {"value": round(value, 4), "unit": "s", "cores": ref.threads, "kind": "port",
                         "sample": ref.sample_desc()},
        "estimated": {"what": ("value = the measured full-configuration step (every stage in full)" if ref.full else
                               "value = full-configuration seconds estimated from each step's sample "
                               "(per-stage linear extrapolation); ms_per_step = the measured wall time of a "
                               "sampled step"), "extrapolated": not ref.full, "steps_s": [round(v, 3) for v in vals],
                      "stdev_s": round(statistics.pstdev(vals), 3), "setup_s": round(ref.setup_s, 1)},
        "stages_s": stages,
        "e2e": {"value": round(value, 4), "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def _lines(self):
        try:
            with open(self.f.name) as fh:
                return sum(1 for _ in fh)
        except OSError:
            return 0

    def start(self):
        """Start sampling every 200 ms and return once the sampler is live (its
        first line written), so that even a short timed region is covered."""
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-i", str(self.idx), "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
            return
        t0 = time.time()
        while self._lines() == 0 and time.time() - t0 < 10 and self.p.poll() is None:
            time.sleep(0.02)
        self.n0 = self._lines()

    def stop(self):
        if self.p is None:
            return None
        # at least one sample taken at or after the end of the timed region
        t0 = time.time()
        while self._lines() <= getattr(self, "n0", 0) and time.time() - t0 < 2 and self.p.poll() is None:
            time.sleep(0.02)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if "Active" in r[5 + i] and "Not" not in r[5 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def _load_json(*path):
    try:
        with open(os.path.join(ROOT, *path)) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def load_peaks():
    """HBM copy peak (MEASURED_PEAKS.json, driver-written; else the profiling
    recipe's fallback), the L2-resident read peak (profiles/l2_peak.json, a
    committed measurement -- fixed, not re-measured per run) and the warp
    instruction issue peak: 148 SMs x 4 schedulers x 1 warp-instruction/clk at
    the max SM clock."""
    d = _load_json("MEASURED_PEAKS.json")
    hbm = (float(d["hbm_gbs"]), "measured") if "hbm_gbs" in d else (6650.0, "fallback (B200_PROFILING.md)")
    mhz = float(d.get("sm_max_mhz", 1965.0))
    l2 = _load_json("profiles", "l2_peak.json")
    return {"hbm": hbm, "l2": (float(l2["gbs"]), l2.get("source", "profiles/l2_peak.json")) if "gbs" in l2 else (None, None),
            "issue": (148 * 4 * mhz * 1e6 / 1e9, f"148 SMs x 4 SMSPs x 1 warp-inst/clk x {mhz:.0f} MHz")}


def kernel_counts(cfg, kernel):
    """Per-launch ncu counters of `kernel` at this config (profiles/kernel_counts.json,
    from profiles/scripts/kernel_counts.sh: same config, same seeds, so the same
    data-dependent work as the live run)."""
    return _load_json("profiles", "kernel_counts.json").get(cfg.name[:2], {}).get(kernel)


def los_roof(name, kernel, kernel_ms, units, cfg, peaks):
    """VIX / VIEWSHED: issue-bound LOS walks.  achieved = ncu warp
    instructions per launch / the live kernel time; l2 = L2 bytes the kernel
    actually read (ncu) / live time against the committed L2 read peak; los =
    SURVEY §8(d)'s algorithmic LOS samples (every crossing, no early exit)."""
    r = {"stage": name, "kernel": kernel, "kernel_ms": round(kernel_ms, 3), "bound": "issue",
         "unit": "Gwarp-inst/s", "peak": round(peaks["issue"][0], 1), "peak_kind": peaks["issue"][1],
         "los": {"samples_per_launch": int(units),
                 "samples_per_s": round(units / (kernel_ms / 1e3), 1) if kernel_ms else None,
                 "algorithmic_gbs": round(4 * units / (kernel_ms / 1e3) / 1e9, 1) if kernel_ms else None}}
    k = kernel_counts(cfg, kernel)
    if k and kernel_ms:
        r["achieved"] = round(k["inst"] / (kernel_ms / 1e3) / 1e9, 1)
        r["frac"] = round(r["achieved"] / r["peak"], 4)
        r["inst_per_launch"] = int(k["inst"])
        r["inst_per_los_sample"] = round(k["inst"] / units, 3) if units else None
        r["traffic"] = int(k["dram_bytes"])
        l2p = peaks["l2"][0]
        r["l2"] = {"read_bytes_per_launch": int(k["l2_read_bytes"]),
                   "achieved_gbs": round(k["l2_read_bytes"] / (kernel_ms / 1e3) / 1e9, 1),
                   "peak_gbs": l2p, "frac": round(k["l2_read_bytes"] / (kernel_ms / 1e3) / 1e9 / l2p, 4) if l2p else None}
        r["ncu_issue_active_pct"] = k.get("issue_active_pct")
    else:
        r["achieved"] = r["frac"] = r["traffic"] = None
    return r


def stage_figures(st, K, cfg, site_mode, site_stream=None):
    """Per-stage device times and work figures from the engine's stats over K
    steps, and the roofline of the dominant stage's kernel."""
    peaks = load_peaks()
    stages = {}
    if cfg.samples:
        kern = ("k_vix_lanes" if cfg.samples <= 32 else "k_vix_quads") if cfg.roi <= 255 else "k_vix"
        stages["vix"] = {"ms": round(st["ms_vix"] / K, 3),
                         **los_roof("vix", kern, st["ms_vix_kernel"] / K, st["vix_crossings_full"] / K, cfg, peaks)}
        stages["findmax"] = {"ms": round(st["ms_findmax"] / K, 3), "kernel": "k_findmax"}
    kern = "k_viewshed_evk" if cfg.roi <= 250 else "k_viewshed"
    stages["viewshed"] = {"ms": round(st["ms_viewshed"] / K, 3),
                          **los_roof("viewshed", kern, st["ms_viewshed_kernel"] / K, st["viewshed_crossings"] / K,
                                     cfg, peaks)}
    site_ms = st["ms_site"] / K
    stages["site"] = {"ms": round(site_ms, 3), "iterations": int(st["site_iterations"] // K),
                      "kernel": ("k_batch_bmax+decide+winners+delta+update (batched rounds; k_site_loop1 on small grids)"
                                 if site_mode == 0 else "k_gain_full"),
                      "launches": int(st["site_launches"] // K),
                      "mode": "exact incremental, every local maximum per round" if site_mode == 0 else "full-rescan"}
    if site_stream:
        hbm = peaks["hbm"][0]
        site_stream["frac_of_hbm"] = round(site_stream["gbs"] / hbm, 4) if site_stream.get("gbs") else None
        site_stream["kernel_frac_of_hbm"] = (round(site_stream["kernel_gbs"] / hbm, 4)
                                             if site_stream.get("kernel_gbs") else None)
        k = kernel_counts(cfg, site_stream["kernel"])
        site_stream["traffic"] = int(k["dram_bytes"]) if k else None
        stages["site_stream"] = site_stream
    dom = max(("vix", "viewshed", "site"), key=lambda x: stages.get(x, {}).get("ms", -1))
    if dom in ("vix", "viewshed"):
        roofline = {k: v for k, v in stages[dom].items() if k != "ms"}
    else:   # SITE: the streaming gain pass against HBM
        ss = stages.get("site_stream", {})
        roofline = {"stage": "site", "kernel": ss.get("kernel"), "bound": "hbm", "unit": "GB/s",
                    "achieved": ss.get("kernel_gbs"), "peak": peaks["hbm"][0], "peak_kind": peaks["hbm"][1],
                    "frac": ss.get("kernel_frac_of_hbm"), "traffic": ss.get("traffic")}
    roofline["note"] = ("VIX/VIEWSHED are issue-bound exact LOS walks (DESIGN.md §3, §5): the roof is warp-instruction "
                        "issue; l2 = bytes the kernel actually read against the committed L2 read peak; SITE's "
                        "streaming gain pass is the HBM-bound kernel (stages.site_stream)")
    return stages, roofline, peaks


def run_b200(args, cfg):
    import numpy as np
    import torch
    import paper_2006_16783_b200 as T
    from paper_2006_16783_b200.configs import params_for, run, run_from_host, setup_terrain

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    eng = T.Engine(local)
    params = params_for(cfg, args.site_mode)
    setup_terrain(eng, cfg)
    z_host = torch.empty((cfg.nrows, cfg.ncols), dtype=torch.int16, pin_memory=True).numpy()
    z_host[:] = eng.terrain()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        run(eng, cfg, params)
    eng.synchronize()

    phys = os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[local] if os.environ.get(
        "CUDA_VISIBLE_DEVICES") else str(local)
    clocks = Clocks(phys)
    eng.reset_stats()
    torch.cuda.synchronize()
    barrier()
    clocks.start()
    step_ms = []
    res = None
    for _ in range(args.steps):
        flush.zero_()                  # evict L2 (256 MB > 126 MB) outside the timed events
        torch.cuda.synchronize()
        eng.event_record(0)
        res = run(eng, cfg, params)
        eng.event_record(1)
        step_ms.append(eng.event_elapsed(0, 1))
    eng.synchronize()
    torch.cuda.synchronize()
    clk = clocks.stop()
    st = eng.stats()
    barrier()
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], device=f"cuda:{local}", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms = total_ms / args.steps

    # ---- SITE streaming figure: the same SITE on the resident viewsheds with
    # the full-rescan strategy (every round re-reads every packed viewshed) ---
    import ctypes
    from paper_2006_16783_b200 import _native as N
    p1 = params_for(cfg, 1)
    p1.max_selected = min(cfg.max_selected or 64, 64)   # bounded: 64 rounds re-reading every viewshed
    eng.reset_stats()
    r1 = eng.site(p1, cap=p1.max_selected + 1)
    st1 = eng.stats()
    assert np.array_equal(r1["index"], res["index"][:len(r1["index"])]), "full-rescan SITE diverged from incremental"
    # rounds-only device time (the gain pass + argmax + commit of each round;
    # bucket/gain initialisation excluded -- it is in stages.site's ms)
    # kernel-level: the gain pass alone (CUDA events around back-to-back passes
    # against the final cum), the SURVEY §8(d) SITE roofline figure
    gp_ms, gp_bytes = eng.time_gain_pass(8)
    rms = st1["ms_site_rounds"]
    site_stream = {"ms": round(rms, 3), "ms_with_setup": round(st1["ms_site"], 3),
                   "iterations": int(st1["site_iterations"]), "bytes": int(st1["site_bytes"]),
                   "gbs": round(st1["site_bytes"] / (rms / 1e3) / 1e9, 1) if rms else None,
                   "kernel": "k_gain_full",
                   "layout": os.environ.get("TXS_GAIN_PASS") or "t8 (8x8-tile shadow of the viewsheds and the cum, DESIGN.md §3)",
                   "mode": "full-rescan (same picks as incremental)",
                   "kernel_ms_per_pass": round(gp_ms, 4), "kernel_bytes_per_pass": int(gp_bytes),
                   "kernel_gbs": round(gp_bytes / (gp_ms / 1e3) / 1e9, 1) if gp_ms else None}

    # ---- e2e through the public API from pinned host memory ---------------
    nw = (cfg.posts + 63) // 64
    cum_host = torch.empty(nw * 8, dtype=torch.uint8, pin_memory=True).numpy().view(np.uint64)
    e2e_ms = []
    launches_e2e = 0
    for _ in range(max(1, args.e2e_steps)):
        flush.zero_()
        torch.cuda.synchronize()
        before = eng.stats()["kernel_launches"]
        eng.event_record(2)
        r2 = run_from_host(eng, cfg, params, z_host)   # upload overlapped with VIX (public API)
        eng._chk(N.lib.txs_get_cumulative(eng.handle, ctypes.c_void_p(cum_host.ctypes.data)))
        eng.event_record(3)
        e2e_ms.append(eng.event_elapsed(2, 3))
        launches_e2e = eng.stats()["kernel_launches"] - before
    # median over the e2e steps: a host-side stall (seen as an occasional
    # 200-400 ms gap between the step's device events) does not set the figure;
    # every step's time is reported beside it
    assert np.array_equal(r2["index"], res["index"]) and r2["stop"] == res["stop"], "e2e picks differ"
    e2e = statistics.median(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e], device=f"cuda:{local}", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e = float(t.item())
    d2h = nw * 8 + len(r2["index"]) * 32

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    # ---- per-stage figures and the roofline of the dominant kernel -------
    K = args.steps
    stages, roofline, peaks = stage_figures(st, K, cfg, args.site_mode, site_stream)
    line = {
        "metric": METRIC, "value": round(ms / 1e3, 5), "unit": "s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": DTYPE, "data": DATA, "config": config_dict(cfg),
        "result": {"candidates": st["candidates"], "sited": int(len(res["index"])), "stop": res["stop"],
                   "coverage": float(res["coverage"][-1]) if len(res["coverage"]) else 0.0,
                   "parallelism": f"replicas{world}" if world > 1 else "single-gpu"},
        "stages": stages,
        "roofline": roofline,
        "e2e": {"value": round(e2e / 1e3, 5), "unit": "s", "h2d_bytes_per_step": cfg.posts * 2,
                "d2h_bytes_per_step": d2h, "kernel_launches_per_step": launches_e2e,
                "steps_ms": [round(x, 3) for x in e2e_ms], "statistic": "median"},
        "gpu_launches": st["kernel_launches"],
        "fp64_ties": {"vix_segments_retested": st["vix_fp64_ties"] // K, "vix_decisions_changed": st["vix_fp64_flips"] // K,
                      "viewshed_rays_retested": st["vs_fp64_ties"] // K, "viewshed_bits_changed": st["vs_fp64_flips"] // K},
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"], line["differing_bits"] = cpu_baseline_leg(args, cfg, eng, res)
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def cpu_baseline_leg(args, cfg, eng, res):
    """The oracle on this host on the bounded sample (rank 0, N = 1), fed with
    the GPU's candidate list and viewsheds; its sample outputs double as a live
    parity check of the timed run: differing VixMap scores on the sampled rows,
    differing bits of the sampled viewsheds, and the oracle's SITE sequence /
    cumulative bitmap against the GPU's."""
    import numpy as np
    rows, cols, _ = eng.candidates()
    plan = SAMPLE_PLAN.get(cfg.name[:2], (64, 64, True))
    views = eng.viewsheds(cfg.roi)[:2] if plan[2] else None
    ref = CpuReference(cfg, args.threads, cand=(rows, cols), views=views)
    v, parts, wall = ref.step()
    out = ref.last
    diff = {}
    if cfg.samples:
        g = np.concatenate([eng.vix(int(r), int(r) + 1) for r in out["vix_rows"]])
        diff["vix"] = {"rows_compared": int(len(out["vix_rows"])), "posts_compared": int(g.size),
                       "scores_differing": int((g != out["vix"]).sum())}
    idx = out["vs_idx"]
    if views is not None:
        gw, gv = views[0][idx], views[1][idx]
    else:
        got = [eng.viewsheds(cfg.roi, first=int(i), count=1)[:2] for i in idx]
        gw, gv = np.concatenate([x[0] for x in got]), np.concatenate([x[1] for x in got])
    area = int((out["vs_wins"][:, 2].astype(np.int64) * out["vs_wins"][:, 3]).sum())
    diff["viewshed"] = {"viewsheds_compared": int(len(idx)), "bits_compared": area,
                        "windows_differing": int((gw != out["vs_wins"]).any(1).sum()),
                        "bits_differing": int(np.bitwise_count(gv ^ out["vs_words"]).sum())}
    o = out["site"]
    if plan[2]:
        same = (o["stop"] == res["stop"] and len(o["index"]) == len(res["index"])
                and bool(np.array_equal(o["index"], res["index"])) and bool(np.array_equal(o["gain"], res["gain"])))
        diff["site"] = {"picks_compared": int(len(res["index"])), "sequence_identical": same,
                        "cum_bits_differing": int(np.bitwise_count(eng.cumulative() ^ o["cum"]).sum())}
    diff["reference"] = ("the cpu_baseline sample's own oracle outputs (SPEC.md:147 fp64 formula, oracle pinned to the "
                         "reference walk_crossings) against this run's GPU results")
    cpu = {"value": round(v, 3), "unit": "s", "cores": ref.threads, "kind": "port", "sample": ref.sample_desc(),
           "measured_wall_s": round(wall, 3), "stages_s": {k: round(x, 3) for k, x in parts.items()}}
    return cpu, diff


def run_b200_sharded(args, cfg):
    """N > 1: one configuration split into row bands over the N GPUs (strong
    scaling), SITE exchanging (gain,id) keys and winner windows over NCCL."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2006_16783_b200 as T
    from paper_2006_16783_b200.configs import params_for
    from paper_2006_16783_b200.shard import TorchComm, run_sharded, setup_sharded

    rank, world, local = dist_env()
    if "MASTER_ADDR" not in os.environ:   # --sharded without torchrun: a world of one
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(sk.getsockname()[1]), RANK="0", WORLD_SIZE="1")
        sk.close()
    torch.cuda.set_device(local)
    # NCCL may print its version line on stdout at communicator init (depending
    # on NCCL_DEBUG): keep stdout for the one JSON line by pointing fd 1 at
    # stderr while the communicator comes up
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        dist.init_process_group("nccl", init_method="env://", device_id=torch.device(f"cuda:{local}"))
        dist.barrier()
        torch.cuda.synchronize()
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)
    dev = f"cuda:{local}"
    comm = TorchComm(dev)
    eng = T.Engine(local)
    params = params_for(cfg, args.site_mode)
    ranks = [(eng, rank)]
    setup_sharded(ranks, cfg, world)
    h0, hr, b0, b1 = eng.shard_info()
    z_host = torch.empty((hr, cfg.ncols), dtype=torch.int16, pin_memory=True).numpy()
    z_host[:] = eng.terrain()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        run_sharded(ranks, comm, cfg, params, world, setup=False, with_cum=False, device_rounds=True)
    eng.reset_stats()
    torch.cuda.synchronize()
    dist.barrier()
    phys = os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[local] if os.environ.get(
        "CUDA_VISIBLE_DEVICES") else str(local)
    clocks = Clocks(phys)
    clocks.start()
    step_ms, res, site_ms = [], None, 0.0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        dist.barrier()
        eng.event_record(0)
        res = run_sharded(ranks, comm, cfg, params, world, setup=False, with_cum=False, device_rounds=True)
        eng.event_record(1)
        step_ms.append(eng.event_elapsed(0, 1))
        site_ms += res.get("site_ms", 0.0)
    clk = clocks.stop()
    st = eng.stats()
    # stage times: max over ranks; work units: summed over the bands
    extra_iters = 0 if res.get("rounds_mode") == "replicated" else args.steps * len(res["index"])
    tm = torch.tensor([st["ms_vix"], st["ms_findmax"], st["ms_viewshed"], st["ms_site"] + site_ms,
                       st["site_iterations"] + extra_iters, st["ms_vix_kernel"],
                       st["ms_viewshed_kernel"]], device=dev, dtype=torch.float64)
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    tc = torch.tensor([st["vix_crossings_full"], st["viewshed_crossings"], st["site_bytes"]], device=dev,
                      dtype=torch.float64)
    dist.all_reduce(tc, op=dist.ReduceOp.SUM)
    agg = dict(st)
    agg.update(ms_vix=tm[0].item(), ms_findmax=tm[1].item(), ms_viewshed=tm[2].item(), ms_site=tm[3].item(),
               site_iterations=int(tm[4].item()), ms_vix_kernel=tm[5].item(), ms_viewshed_kernel=tm[6].item(),
               vix_crossings_full=tc[0].item(), viewshed_crossings=tc[1].item(),
               site_bytes=tc[2].item())
    t = torch.tensor([sum(step_ms) / args.steps], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    e2e_ms = []
    for _ in range(max(1, args.e2e_steps)):
        flush.zero_()
        torch.cuda.synchronize()
        dist.barrier()
        eng.event_record(2)
        eng.set_shard(cfg.nrows, cfg.ncols, b0, b1, cfg.roi + 1)
        eng.set_terrain(z_host)
        r2 = run_sharded(ranks, comm, cfg, params, world, setup=False, with_cum=True, device_rounds=True)
        eng.event_record(3)
        e2e_ms.append(eng.event_elapsed(2, 3))
    t = torch.tensor([statistics.median(e2e_ms)], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e = float(t.item())
    launches = torch.tensor([st["kernel_launches"]], device=dev, dtype=torch.int64)
    dist.all_reduce(launches, op=dist.ReduceOp.SUM)
    if rank == 0:
        stages, roofline, _ = stage_figures(agg, args.steps, cfg, args.site_mode)
        line = {
            "metric": METRIC, "value": round(ms / 1e3, 5), "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": DTYPE, "data": DATA, "config": config_dict(cfg),
            "result": {"sited": int(len(res["index"])), "stop": res["stop"],
                       "parallelism": f"rowband{world} (halo roi+1; SITE {res.get('rounds_mode')}: "
                                      f"{res.get('exchange')})"},
            "e2e": {"value": round(e2e / 1e3, 5), "unit": "s", "h2d_bytes_per_step": cfg.posts * 2,
                    "d2h_bytes_per_step": ((cfg.posts + 63) // 64) * 8 + len(r2["index"]) * 32},
            "gpu_launches": int(launches.item()),
            "stages": stages,
            "roofline": roofline,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    from paper_2006_16783_b200.configs import CONFIGS
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    elif dist_env()[1] > 1 or args.sharded:
        run_b200_sharded(args, cfg)
    else:
        run_b200(args, cfg)


if __name__ == "__main__":
    main()
