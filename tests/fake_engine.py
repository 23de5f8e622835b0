"""CPU stand-in for paper_2006_16783_b200.Engine's shard interface, built on
the oracle (TEST INFRASTRUCTURE ONLY).  Lets the multi-rank orchestration in
paper_2006_16783_b200/shard.py run across real processes over gloo on a
machine without GPUs."""
import numpy as np

import oracle_lib as O


class FakeShardEngine:
    def set_shard(self, nrows, ncols, r0, r1, halo):
        self.nr, self.nc, self.r0, self.r1, self.halo = nrows, ncols, r0, r1, halo

    def shard_info(self):
        h0 = max(0, self.r0 - self.halo)
        return h0, min(self.nr, self.r1 + self.halo) - h0, self.r0, self.r1

    def generate_fractal(self, nrows, ncols, rough, seed, zmin, zmax):
        self.z = O.generate_fractal(nrows, ncols, rough, seed, zmin, zmax)

    def fill_rows(self, a, b, v):
        self.z[a:b] = v

    def estimate_vix(self, p, copy=False):
        self.scores = O.estimate_vix(self.z, p.roi, p.tx_height, p.rx_height, p.samples_per_point, p.seed,
                                     rows=(self.r0, self.r1))

    def find_candidates(self, p, copy=False):
        r, c, _ = O.find_candidates(self.scores[self.r0:self.r1], p.block_width, p.per_block)
        self.rows, self.cols = r + self.r0, c
        self.gids = np.arange(len(r), dtype=np.int64)
        return len(r)

    def random_observers(self, n, seed):
        r, c = O.random_observers(self.nr, self.nc, n, seed)
        keep = (r >= self.r0) & (r < self.r1)
        self.rows, self.cols, self.gids = r[keep], c[keep], np.nonzero(keep)[0].astype(np.int64)

    def set_candidate_base(self, gid0):
        self.gids = gid0 + np.arange(len(self.rows), dtype=np.int64)

    def compute_all_viewsheds(self, p):
        self.roi = p.roi
        self.wins, self.words = O.viewsheds(self.z, p.roi, p.tx_height, p.rx_height, self.rows, self.cols)

    def site_shard_begin(self, p):
        self.cum = np.zeros((self.nr * self.nc + 63) // 64, np.uint64)

    def site_shard_best(self):
        best = 0
        for i in range(len(self.rows)):
            g = O.marginal_gain(self.wins[i], self.words[i], self.cum, self.nr, self.nc)
            best = max(best, (g << 32) | (0xFFFFFFFF - int(self.gids[i])))
        return best

    def site_shard_export(self, gid, roi):
        hit = np.nonzero(self.gids == gid)[0]
        if len(hit) == 0:
            return None
        i = int(hit[0])
        return int(self.rows[i]), int(self.cols[i]), self.wins[i].copy(), self.words[i].copy()

    def site_shard_apply(self, r, c, win, words):
        bits = O.dense_bits(self.cum, self.nr, self.nc).copy()
        r0, c0, h, w = (int(x) for x in win)
        bits[r0:r0 + h, c0:c0 + w] |= O.unpack_window(win, words)
        self.cum = O.pack_dense(bits)

    def cumulative(self):
        return self.cum
