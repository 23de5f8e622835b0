import sys, time, ctypes
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2006_16783_b200 as T
from paper_2006_16783_b200 import _native as N
from paper_2006_16783_b200.configs import CONFIGS, params_for, setup_terrain, run
cfg = CONFIGS[sys.argv[1]]
e = T.Engine(0)
setup_terrain(e, cfg)
p = params_for(cfg)
z_host = torch.empty((cfg.nrows, cfg.ncols), dtype=torch.int16, pin_memory=True).numpy()
z_host[:] = e.terrain()
nw = (cfg.nrows * cfg.ncols + 63) // 64
cum_host = torch.empty(nw * 8, dtype=torch.uint8, pin_memory=True).numpy().view(np.uint64)
for i in range(4):
    e.synchronize()
    e.event_record(2); e.set_terrain(z_host); e.event_record(3)
    r = run(e, cfg, p); e.event_record(4)
    e._chk(N.lib.txs_get_cumulative(e.handle, ctypes.c_void_p(cum_host.ctypes.data))); e.event_record(5)
    st = e.stats()
    print(i, "h2d", round(e.event_elapsed(2, 3), 2), "run", round(e.event_elapsed(3, 4), 2), "cum", round(e.event_elapsed(4, 5), 2), flush=True)
    e.reset_stats()
for i in range(2):
    e.event_record(3); r = run(e, cfg, p); e.event_record(4)
    print("resident run", round(e.event_elapsed(3, 4), 2))
