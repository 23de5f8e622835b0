"""Where the e2e step's time goes beyond the resident pipeline (txs_run_pipeline_host + txs_get_cumulative):
python profiles/scripts/e2e_probe2.py c3 [iters]"""
import sys, time, ctypes
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2006_16783_b200 as T
from paper_2006_16783_b200 import _native as N
from paper_2006_16783_b200.configs import CONFIGS, params_for, setup_terrain, run, run_from_host
cfg = CONFIGS[sys.argv[1]]
e = T.Engine(0)
setup_terrain(e, cfg)
p = params_for(cfg)
z_host = torch.empty((cfg.nrows, cfg.ncols), dtype=torch.int16, pin_memory=True).numpy()
z_host[:] = e.terrain()
nw = (cfg.nrows * cfg.ncols + 63) // 64
cum_host = torch.empty(nw * 8, dtype=torch.uint8, pin_memory=True).numpy().view(np.uint64)
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
    e.synchronize()
    t0 = time.perf_counter()
    e.event_record(2)
    r = run_from_host(e, cfg, p, z_host); e.event_record(4)
    t2 = time.perf_counter()
    e._chk(N.lib.txs_get_cumulative(e.handle, ctypes.c_void_p(cum_host.ctypes.data))); e.event_record(5)
    t3 = time.perf_counter()
    sm = {k: round(v, 2) for k, v in r.get("stage_ms", {}).items()}
    print(i, "host-run", round(e.event_elapsed(2, 4), 2), "cum", round(e.event_elapsed(4, 5), 2),
          "wall", round((t2 - t0) * 1e3, 2), round((t3 - t2) * 1e3, 2), "stages", sm, "sum", round(sum(sm.values()), 2), flush=True)
    e.reset_stats()
for i in range(3):
    e.synchronize(); t0 = time.perf_counter()
    e.event_record(3); r = run(e, cfg, p); e.event_record(4)
    t1 = time.perf_counter()
    sm = {k: round(v, 2) for k, v in r.get("stage_ms", {}).items()}
    print("resident run", round(e.event_elapsed(3, 4), 2), "wall", round((t1 - t0) * 1e3, 2), sm, "sum", round(sum(sm.values()), 2))
