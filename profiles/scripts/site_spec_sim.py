"""How many greedy picks could one SITE round commit?  (design probe for
multi-pick rounds, run on the GPU box)

Claim: at a round start let t1 > t2 > ... be the candidates in key order
(gain << 32 | ~id).  Committing t1 lowers only the gains of candidates whose
windows overlap t1's.  If t2's window does not overlap t1's, t2's key is
unchanged and every other key is unchanged or lower, so t2 is the next greedy
pick; inductively the longest prefix t1..tm in which no window overlaps an
earlier one is the next m picks.  This script runs a configuration on the
engine, downloads the viewsheds, replays the greedy exactly (gains recomputed
for the overlapping candidates after each pick, picks checked against the
engine's), and at each round start measures m.
  python profiles/scripts/site_spec_sim.py c3 [T]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2006_16783_b200 as T  # noqa: E402
from paper_2006_16783_b200.configs import CONFIGS, params_for, run, setup_terrain  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
TOP = int(sys.argv[2]) if len(sys.argv) > 2 else 32
cfg = CONFIGS[name]
R = cfg.roi
with T.Engine(0) as e:
    setup_terrain(e, cfg)
    p = params_for(cfg)
    res = run(e, cfg, p)
    rows, cols, _ = e.candidates()
    wins, words, pops = e.viewsheds(R)
    nr, nc = e.dims
picks = res["index"].astype(np.int64)
n = len(rows)
print(f"{name}: {n} candidates, {len(picks)} picks", flush=True)
rows = rows.astype(np.int64)
cols = cols.astype(np.int64)
cum = np.zeros((nr, nc), bool)


def vbits(i):
    r0, c0, h, w = (int(x) for x in wins[i])
    nb = h * w
    b = np.unpackbits(words[i][: (nb + 63) // 64].view(np.uint8), bitorder="little")[:nb]
    return r0, c0, h, w, b.reshape(h, w).astype(bool)


ids = np.arange(n, dtype=np.int64)
keys = pops.astype(np.int64) * (1 << 32) + ((1 << 32) - 1 - ids)
taken = np.zeros(n, bool)


def neighbours(i):
    return np.nonzero((np.abs(rows - rows[i]) <= 2 * R) & (np.abs(cols - cols[i]) <= 2 * R) & ~taken)[0]


t0 = time.time()
k = 0
ms = []
while k < len(picks):
    part = np.argpartition(-keys, TOP)[:TOP] if n > TOP else np.arange(n)
    top = part[np.argsort(-keys[part], kind="stable")]
    acc = [int(top[0])]
    for t in top[1:]:
        t = int(t)
        if any(abs(rows[t] - rows[a]) <= 2 * R and abs(cols[t] - cols[a]) <= 2 * R for a in acc):
            break
        acc.append(t)
    for a in acc:
        w = int(np.argmax(keys))
        assert w == a, (k, w, a)
        assert w == picks[k], (k, w, int(picks[k]))
        r0, c0, h, ww, b = vbits(w)
        cum[r0:r0 + h, c0:c0 + ww] |= b
        taken[w] = True
        keys[w] = -1
        for j in neighbours(w):
            jr0, jc0, jh, jw, jb = vbits(int(j))
            g = int((jb & ~cum[jr0:jr0 + jh, jc0:jc0 + jw]).sum())
            keys[j] = g * (1 << 32) + ((1 << 32) - 1 - int(j))
        k += 1
        if k == len(picks):
            break
    ms.append(len(acc))
ms = np.array(ms)
print(f"{name}: {len(picks)} picks in {len(ms)} rounds (mean {len(picks) / len(ms):.2f} picks per round, "
      f"top {TOP}); rounds with m = 1: {(ms == 1).mean():.3f}, m >= 4: {(ms >= 4).mean():.3f}, "
      f"max {ms.max()}; sim {time.time() - t0:.0f} s", flush=True)
print("histogram m: " + " ".join(f"{v}:{c}" for v, c in zip(*np.unique(ms, return_counts=True))))
