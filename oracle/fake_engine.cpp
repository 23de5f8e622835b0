// TEST INFRASTRUCTURE ONLY.  A CPU stand-in for the engine's stage entry
// points (txs_engine_ops, include/txsite_b200.h), built on the oracle, so the
// native group orchestration (txs_group_*, csrc/group.cu) -- band plan, global
// ids, host-staged SITE rounds, stop rules, cum assembly -- runs with 2+ ranks
// on a machine without GPUs (tests/test_group_cpu.py).  Mirrors
// tests/fake_engine.py, the stand-in of the Python orchestration.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../include/txsite_b200.h"
#include "oracle.hpp"

namespace {

struct Fake {
    std::string err;
    int64_t nr = 0, nc = 0, r0 = 0, r1 = 0, halo = 0;
    std::vector<int16_t> z;        // whole grid; rows outside band +- halo stay 0 (never read)
    std::vector<uint8_t> scores;   // whole grid indexing (txo::estimate_vix)
    std::vector<int32_t> rows, cols, score;
    std::vector<int64_t> gids;
    int32_t roi = 0;
    std::vector<txo::Window> wins;
    std::vector<uint64_t> words;   // stride txo window words of 2roi+1
    int64_t stride = 0;
    std::vector<uint64_t> cum;     // dense whole grid
    bool cum_valid = false;
};

Fake* F(txs_ctx* c) { return reinterpret_cast<Fake*>(c); }
const Fake* F(const txs_ctx* c) { return reinterpret_cast<const Fake*>(c); }
txs_status bad(Fake* f, const char* m) { f->err = m; return TXS_ERR_STATE; }
txo::Grid grid(const Fake* f) { return txo::Grid{f->nr, f->nc, f->z.data()}; }

txs_status f_create(int, txs_ctx** out) { *out = reinterpret_cast<txs_ctx*>(new Fake()); return TXS_OK; }
void f_destroy(txs_ctx* c) { delete F(c); }
const char* f_last_error(const txs_ctx* c) { return F(c)->err.c_str(); }

txs_status f_set_shard(txs_ctx* c, int64_t nr, int64_t nc, int64_t rb, int64_t re, int32_t halo) {
    Fake* f = F(c);
    f->nr = nr; f->nc = nc; f->r0 = rb; f->r1 = re; f->halo = halo;
    f->z.assign((size_t)(nr * nc), 0);
    f->gids.clear(); f->rows.clear(); f->cols.clear(); f->score.clear();
    f->cum_valid = false;
    return TXS_OK;
}
txs_status f_shard_info(const txs_ctx* c, int64_t* h0, int64_t* hr, int64_t* b0, int64_t* b1) {
    const Fake* f = F(c);
    *h0 = std::max<int64_t>(0, f->r0 - f->halo);
    *hr = std::min<int64_t>(f->nr, f->r1 + f->halo) - *h0;
    *b0 = f->r0; *b1 = f->r1;
    return TXS_OK;
}
txs_status f_set_terrain(txs_ctx* c, const int16_t* z, int64_t nrows, int64_t ncols) {
    Fake* f = F(c);
    int64_t h0, hr, b0, b1;
    f_shard_info(c, &h0, &hr, &b0, &b1);
    if (nrows != hr || ncols != f->nc) { f->err = "[read] sharded context: band + halo rows"; return TXS_ERR_SIZE_MISMATCH; }
    std::copy(z, z + nrows * ncols, f->z.begin() + h0 * f->nc);
    return TXS_OK;
}
txs_status f_generate(txs_ctx* c, int64_t nr, int64_t nc, double rough, uint64_t seed, int32_t zmin, int32_t zmax) {
    Fake* f = F(c);
    if (nr != f->nr || nc != f->nc) return bad(f, "[read] generate the global grid dimensions");
    txo::generate_fractal(nr, nc, rough, seed, zmin, zmax, f->z.data(), 0);
    return TXS_OK;
}
txs_status f_fill_rows(txs_ctx* c, int64_t rb, int64_t re, int16_t v) {
    Fake* f = F(c);
    std::fill(f->z.begin() + rb * f->nc, f->z.begin() + re * f->nc, v);
    return TXS_OK;
}
txs_status f_vix(txs_ctx* c, const txs_params* p, uint8_t*) {
    Fake* f = F(c);
    f->scores.assign((size_t)(f->nr * f->nc), 0);
    txo::estimate_vix(grid(f), p->roi, p->tx_height, p->rx_height, p->samples_per_point, p->seed, 0,
                      f->scores.data(), f->r0, f->r1, p->los_arith);
    return TXS_OK;
}
txs_status f_findmax(txs_ctx* c, const txs_params* p, int64_t* n, txs_candidate*, int64_t) {
    Fake* f = F(c);
    const int64_t bw = p->block_width > 0 ? p->block_width : (p->roi + 2) / 3;
    const auto v = txo::find_candidates(f->scores.data() + f->r0 * f->nc, f->r1 - f->r0, f->nc, bw, p->per_block);
    f->rows.clear(); f->cols.clear(); f->score.clear(); f->gids.clear();
    for (size_t i = 0; i < v.size(); ++i) {
        f->rows.push_back(v[i].row + (int32_t)f->r0); f->cols.push_back(v[i].col); f->score.push_back(v[i].score);
        f->gids.push_back((int64_t)i);
    }
    *n = (int64_t)v.size();
    return TXS_OK;
}
txs_status f_observers(txs_ctx* c, int64_t n, uint64_t seed) {   // decision D11, band's draws, id = draw index
    Fake* f = F(c);
    txo::SplitMix64 s(seed);
    f->rows.clear(); f->cols.clear(); f->score.clear(); f->gids.clear();
    for (int64_t i = 0; i < n; ++i) {
        const int32_t r = (int32_t)s.next_below((uint64_t)f->nr), cc = (int32_t)s.next_below((uint64_t)f->nc);
        if (r >= f->r0 && r < f->r1) { f->rows.push_back(r); f->cols.push_back(cc); f->score.push_back(0); f->gids.push_back(i); }
    }
    return TXS_OK;
}
txs_status f_get_cands(txs_ctx* c, txs_candidate* out, int64_t cap, int64_t* n) {
    Fake* f = F(c);
    if (n) *n = (int64_t)f->rows.size();
    for (int64_t i = 0; out && i < std::min<int64_t>(cap, (int64_t)f->rows.size()); ++i)
        out[i] = txs_candidate{f->rows[(size_t)i], f->cols[(size_t)i], f->score[(size_t)i], 0};
    return TXS_OK;
}
txs_status f_base(txs_ctx* c, int64_t gid0) {
    Fake* f = F(c);
    for (size_t i = 0; i < f->gids.size(); ++i) f->gids[i] = gid0 + (int64_t)i;
    return TXS_OK;
}
txs_status f_viewsheds(txs_ctx* c, const txs_params* p) {
    Fake* f = F(c);
    f->roi = p->roi;
    f->stride = ((2LL * p->roi + 1) * (2LL * p->roi + 1) + 63) / 64;
    const size_t n = f->rows.size();
    f->wins.assign(n, txo::Window{});
    f->words.assign(n * (size_t)f->stride, 0);
    const txo::Grid g = grid(f);
    for (size_t i = 0; i < n; ++i) {
        if (p->los_arith == TXS_LOS_EXACT)
            txo::compute_viewshed(g, f->rows[i], f->cols[i], p->roi, p->tx_height, p->rx_height, &f->wins[i],
                                  f->words.data() + i * (size_t)f->stride);
        else
            txo::compute_viewshed_fp64(g, f->rows[i], f->cols[i], p->roi, p->tx_height, p->rx_height, &f->wins[i],
                                       f->words.data() + i * (size_t)f->stride);
    }
    return TXS_OK;
}
txs_status f_begin(txs_ctx* c, const txs_params*) {
    Fake* f = F(c);
    f->cum.assign((size_t)((f->nr * f->nc + 63) / 64), 0);
    f->cum_valid = true;
    return TXS_OK;
}
txs_status f_best(txs_ctx* c, uint64_t* key) {
    Fake* f = F(c);
    uint64_t best = 0;
    for (size_t i = 0; i < f->rows.size(); ++i) {
        const int64_t g = txo::marginal_gain(f->wins[i], f->words.data() + i * (size_t)f->stride, f->cum.data(),
                                             (int64_t)f->cum.size(), f->nc);
        best = std::max<uint64_t>(best, ((uint64_t)g << 32) | (0xffffffffull - (uint64_t)f->gids[i]));
    }
    *key = best;
    return TXS_OK;
}
txs_status f_export(txs_ctx* c, int64_t gid, int32_t* owned, int32_t* row, int32_t* col, txs_window* win,
                    uint64_t* words, int64_t stride) {
    Fake* f = F(c);
    *owned = 0;
    for (size_t i = 0; i < f->gids.size(); ++i) {
        if (f->gids[i] != gid) continue;
        *owned = 1; *row = f->rows[i]; *col = f->cols[i];
        const txo::Window& w = f->wins[i];
        *win = txs_window{w.row0, w.col0, w.h, w.w};
        std::fill(words, words + stride, 0ull);
        std::copy(f->words.begin() + (int64_t)i * f->stride, f->words.begin() + (int64_t)i * f->stride + txo::window_words(w), words);
        return TXS_OK;
    }
    return TXS_OK;
}
txs_status f_apply(txs_ctx* c, int32_t, int32_t, const txs_window* win, const uint64_t* words) {
    Fake* f = F(c);
    txo::union_into(txo::Window{win->row0, win->col0, win->h, win->w}, words, f->cum.data(), f->nc);
    return TXS_OK;
}
txs_status f_cum_rows(txs_ctx* c, int64_t rb, int64_t re, uint64_t* out) {
    Fake* f = F(c);
    if (!f->cum_valid) return bad(f, "[site] no cumulative viewshed");
    for (int64_t b = rb * f->nc; b < re * f->nc; ++b)
        if ((f->cum[(size_t)(b >> 6)] >> (b & 63)) & 1) __atomic_fetch_or(&out[b >> 6], 1ull << (b & 63), __ATOMIC_RELAXED);
    return TXS_OK;
}
txs_status f_stats(txs_ctx*, txs_stats* out) { *out = txs_stats{}; return TXS_OK; }

const txs_engine_ops kFakeOps = {
    f_create, f_destroy, f_last_error, f_set_shard, f_shard_info, f_set_terrain, f_generate, f_fill_rows,
    f_vix, f_findmax, f_observers, f_get_cands, f_base, f_viewsheds, f_begin, f_best, f_export, f_apply,
    f_cum_rows, f_stats,
};

}  // namespace

extern "C" const txs_engine_ops* txo_fake_engine_ops(void) { return &kFakeOps; }
