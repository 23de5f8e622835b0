"""The five BASELINE.json configurations as engine parameters.

Seeded synthetic terrains (decision D10 generator) stand in for the paper's
NASADEM tiles and DEM1000 (not in the container); shapes, elevation ranges,
roughness, ROI, heights, sampling, blocking and SITE caps are BASELINE's.
"""
from dataclasses import dataclass


@dataclass(frozen=True)
class Config:
    name: str
    nrows: int
    ncols: int
    roughness: float
    zmin: int
    zmax: int
    roi: int
    height: int
    samples: int        # VIX samples per post (0: no VIX stage)
    block: int          # FINDMAX block width (0: no FINDMAX stage)
    per_block: int
    target: float
    max_selected: int
    terrain_seed: int
    vix_seed: int
    water_rows: int = 0          # rows [0, water_rows) clamped to 0
    random_observers: int = 0    # config 5: observers instead of VIX+FINDMAX
    observer_seed: int = 0

    @property
    def posts(self):
        return self.nrows * self.ncols


CONFIGS = {
    "c1": Config("c1-1000sq-roi100", 1000, 1000, 0.5, 0, 4000, 100, 10, 10, 100, 10, 0.95, 200, 2006, 1),
    "c2": Config("c2-4096sq-roi200", 4096, 4096, 0.6, 0, 3000, 200, 20, 20, 128, 16, 1.0, 1024, 2007, 2),
    "c3": Config("c3-16384sq-roi100-water", 16384, 16384, 0.5, 0, 4000, 100, 10, 10, 256, 32, 1.0, 4096, 2008, 3,
                 water_rows=2048),
    "c4": Config("c4-46400sq-roi100", 46400, 46400, 0.5, 0, 4000, 100, 10, 10, 400, 16, 1.0, 4096, 2009, 4),
    "c5": Config("c5-16384sq-roi250-1M-observers", 16384, 16384, 0.5, 0, 4000, 250, 50, 0, 0, 0, 1.0, 8192, 2010, 5,
                 random_observers=1 << 20, observer_seed=16783),
}


def params_for(cfg, site_mode=0):
    from .api import make_params
    return make_params(cfg.roi, cfg.height, cfg.height, samples=max(cfg.samples, 1),
                       per_block=max(cfg.per_block, 1), block_width=cfg.block, target=cfg.target,
                       max_selected=cfg.max_selected, seed=cfg.vix_seed, site_mode=site_mode)


def setup_terrain(engine, cfg):
    """Generate the config's terrain in HBM (untimed input plumbing)."""
    engine.generate_fractal(cfg.nrows, cfg.ncols, cfg.roughness, cfg.terrain_seed, cfg.zmin, cfg.zmax)
    if cfg.water_rows:
        engine.fill_rows(0, cfg.water_rows, 0)


def run(engine, cfg, params):
    """One end-to-end siting on the resident terrain; returns the result dict."""
    cap = cfg.max_selected + 1 if cfg.max_selected > 0 else 1 << 20
    if cfg.random_observers:
        engine.random_observers(cfg.random_observers, cfg.observer_seed)
        engine.compute_all_viewsheds(params)
        return engine.site(params, cap=min(cap, cfg.random_observers + 1))
    return engine.run_pipeline(params, cap=cap)


def run_from_host(engine, cfg, params, z_host):
    """The same siting from a host terrain through the public API: the upload
    overlaps VIX (txs_run_pipeline_host); configuration 5 (no VIX) uploads, then
    runs."""
    cap = cfg.max_selected + 1 if cfg.max_selected > 0 else 1 << 20
    if cfg.random_observers:
        engine.set_terrain(z_host)
        return run(engine, cfg, params)
    return engine.run_pipeline_host(z_host, params, cap=cap)
