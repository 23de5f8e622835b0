// ORACLE — TEST INFRASTRUCTURE ONLY.  extern "C" surface of the oracle for the
// Python test-suite (ctypes) and bench.py's cpu_baseline / --impl reference.
#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "oracle.hpp"

using namespace txo;

template <class Fn>
static void par(int64_t n, unsigned threads, Fn&& fn) {
    if (threads == 0) { threads = std::thread::hardware_concurrency(); if (!threads) threads = 1; }
    if (n <= 0) return;
    if (threads <= 1 || n == 1) { fn(int64_t{0}, n); return; }
    if ((int64_t)threads > n) threads = (unsigned)n;
    const int64_t base = n / threads, extra = n % threads;
    std::vector<std::thread> pool;
    int64_t b = 0;
    for (unsigned w = 0; w < threads; ++w) {
        int64_t e = b + base + ((int64_t)w < extra ? 1 : 0);
        pool.emplace_back([b, e, &fn] { fn(b, e); });
        b = e;
    }
    for (auto& t : pool) t.join();
}

extern "C" {

int txo_abi_version() { return 1; }

uint64_t txo_mix_seed(uint64_t a, uint64_t b, uint64_t c) { return mix_seed(a, b, c); }

// n draws of one stream; mode 0 next(), 1 next_below(arg), 2 next_double bits
void txo_splitmix(uint64_t seed, int64_t n, int mode, uint64_t arg, uint64_t* out) {
    SplitMix64 s(seed);
    for (int64_t i = 0; i < n; ++i) {
        if (mode == 0) out[i] = s.next();
        else if (mode == 1) out[i] = s.next_below(arg);
        else { double d = s.next_double(); std::memcpy(&out[i], &d, 8); }
    }
}

int64_t txo_walk(int64_t r0, int64_t c0, int64_t r1, int64_t c1, int include_end,
                 double* t, double* row, double* col, int32_t* kind, int64_t cap) {
    int64_t n = 0;
    walk(r0, c0, r1, c1, include_end != 0, [&](const Crossing& x) {
        if (n < cap) { t[n] = x.t; row[n] = x.row; col[n] = x.col; kind[n] = x.kind; }
        ++n;
        return true;
    });
    return n;
}

// FNV-1a over the crossing list's (t,row,col) bit patterns and kind bytes.
uint64_t txo_walk_hash(int64_t r0, int64_t c0, int64_t r1, int64_t c1, int include_end, int64_t* count) {
    uint64_t h = 1469598103934665603ull;
    int64_t n = 0;
    auto mix = [&](const void* p, size_t len) {
        const unsigned char* b = (const unsigned char*)p;
        for (size_t i = 0; i < len; ++i) { h ^= b[i]; h *= 1099511628211ull; }
    };
    walk(r0, c0, r1, c1, include_end != 0, [&](const Crossing& x) {
        mix(&x.t, 8); mix(&x.row, 8); mix(&x.col, 8);
        unsigned char k = (unsigned char)x.kind; mix(&k, 1);
        ++n;
        return true;
    });
    if (count) *count = n;
    return h;
}

// parallel.hpp:20-42 chunk boundaries (begin,end) pairs; returns chunk count.
int64_t txo_chunks(int64_t n, unsigned threads, int64_t* out) {
    if (threads == 0) threads = 1;
    if (n <= 0) return 0;
    if (threads <= 1 || n == 1) { out[0] = 0; out[1] = n; return 1; }
    if ((int64_t)threads > n) threads = (unsigned)n;
    const int64_t base = n / threads, extra = n % threads;
    int64_t b = 0;
    for (unsigned w = 0; w < threads; ++w) {
        int64_t e = b + base + ((int64_t)w < extra ? 1 : 0);
        out[2 * w] = b; out[2 * w + 1] = e;
        b = e;
    }
    return threads;
}

int txo_generate_fractal(int64_t nrows, int64_t ncols, double roughness, uint64_t seed,
                         int32_t zmin, int32_t zmax, int16_t* out, unsigned threads) {
    return generate_fractal(nrows, ncols, roughness, seed, zmin, zmax, out, threads);
}

int txo_is_visible(const int16_t* z, int64_t nrows, int64_t ncols, int64_t tr, int64_t tc,
                   int64_t ht, int64_t rr, int64_t rc, int64_t hr, int arith) {
    Grid g{nrows, ncols, z};
    return is_visible_arith(g, tr, tc, ht, rr, rc, hr, arith) ? 1 : 0;
}

void txo_is_visible_batch(const int16_t* z, int64_t nrows, int64_t ncols, const int32_t* pairs,
                          int64_t n, int64_t ht, int64_t hr, uint8_t* out, unsigned threads, int arith) {
    Grid g{nrows, ncols, z};
    par(n, threads, [&](int64_t b, int64_t e) {
        for (int64_t i = b; i < e; ++i) {
            const int32_t* p = pairs + 4 * i;
            out[i] = is_visible_arith(g, p[0], p[1], ht, p[2], p[3], hr, arith) ? 1 : 0;
        }
    });
}

void txo_estimate_vix(const int16_t* z, int64_t nrows, int64_t ncols, int64_t roi, int64_t ht,
                      int64_t hr, int64_t samples, uint64_t seed, unsigned threads,
                      uint8_t* scores, int64_t row_begin, int64_t row_end, int arith) {
    Grid g{nrows, ncols, z};
    estimate_vix(g, roi, ht, hr, samples, seed, threads, scores, row_begin, row_end, arith);
}

// estimate_vix on an arbitrary set of rows: out is len(rows) x ncols.  Work is
// split over posts (not rows) so a few expensive rows do not serialise.
void txo_estimate_vix_rows(const int16_t* z, int64_t nrows, int64_t ncols, int64_t roi, int64_t ht,
                           int64_t hr, int64_t samples, uint64_t seed, unsigned threads,
                           const int64_t* rows, int64_t nsel, uint8_t* out, int arith) {
    Grid g{nrows, ncols, z};
    const int64_t span = 1024;   // posts per work item
    const int64_t per_row = (ncols + span - 1) / span;
    par(nsel * per_row, threads, [&](int64_t b, int64_t e) {
        for (int64_t it = b; it < e; ++it) {
            // rows interleaved, so every worker's static chunk mixes all sampled rows
            const int64_t i = it % nsel, c0 = (it / nsel) * span, c1 = std::min(ncols, c0 + span);
            estimate_vix_cols(g, roi, ht, hr, samples, seed, rows[i], c0, c1, out + i * ncols, arith);
        }
    });
}

int64_t txo_find_candidates(const uint8_t* scores, int64_t nrows, int64_t ncols, int64_t bw,
                            int64_t per_block, int32_t* rows, int32_t* cols, int32_t* sc,
                            int64_t cap) {
    auto v = find_candidates(scores, nrows, ncols, bw, per_block);
    for (int64_t i = 0; i < (int64_t)v.size() && i < cap; ++i) {
        rows[i] = v[i].row; cols[i] = v[i].col; sc[i] = v[i].score;
    }
    return (int64_t)v.size();
}

int64_t txo_midpoint_circle_count(int64_t roi) { return (int64_t)midpoint_circle(roi).size(); }

// Ray template: returns ray count; fills arrays when caps suffice.
int64_t txo_template(int64_t roi, int32_t* p, int32_t* q, int64_t* cell_begin, int32_t* ca,
                     int32_t* cb, int64_t cap_rays, int64_t cap_cells, int64_t* ncells) {
    const RayTemplate& T = ray_template(roi);
    const int64_t nr = (int64_t)T.p.size(), nc = (int64_t)T.ca.size();
    if (ncells) *ncells = nc;
    if (cap_rays >= nr && cap_cells >= nc) {
        std::copy(T.p.begin(), T.p.end(), p);
        std::copy(T.q.begin(), T.q.end(), q);
        std::copy(T.cell_begin.begin(), T.cell_begin.end(), cell_begin);
        std::copy(T.ca.begin(), T.ca.end(), ca);
        std::copy(T.cb.begin(), T.cb.end(), cb);
    }
    return nr;
}

void txo_viewsheds(const int16_t* z, int64_t nrows, int64_t ncols, int64_t roi, int64_t ht,
                   int64_t hr, int64_t n, const int32_t* rows, const int32_t* cols,
                   int32_t* wins, uint64_t* words, int64_t stride, unsigned threads, int arith) {
    Grid g{nrows, ncols, z};
    ray_template(roi);  // build once before fanning out
    par(n, threads, [&](int64_t b, int64_t e) {
        for (int64_t i = b; i < e; ++i) {
            Window w;
            if (arith == ArithExact) compute_viewshed(g, rows[i], cols[i], roi, ht, hr, &w, words + i * stride);
            else compute_viewshed_fp64(g, rows[i], cols[i], roi, ht, hr, &w, words + i * stride, arith == ArithFp64Euclid);
            wins[4 * i] = w.row0; wins[4 * i + 1] = w.col0; wins[4 * i + 2] = w.h; wins[4 * i + 3] = w.w;
        }
    });
}

// cum: dense (nrows*ncols+63)/64 words
int64_t txo_marginal_gain(const int32_t* win, const uint64_t* v, const uint64_t* cum,
                          int64_t nrows, int64_t ncols, int bitloop) {
    Window w{win[0], win[1], win[2], win[3]};
    const int64_t cw = (nrows * ncols + 63) / 64;
    if (bitloop) return marginal_gain_bitloop(w, v, cum, ncols);
    std::vector<uint64_t> padded(cum, cum + cw);
    padded.push_back(0);
    return marginal_gain(w, v, padded.data(), cw + 1, ncols);
}

int txo_site(int64_t n, const int32_t* rows, const int32_t* cols, const int32_t* wins,
             const uint64_t* words, int64_t stride, int64_t nrows, int64_t ncols, double target,
             int64_t max_selected, int naive, int64_t* idx, int32_t* srow, int32_t* scol,
             int64_t* gain, double* cov, int64_t cap, int64_t* nsteps, uint64_t* cum_out) {
    std::vector<Window> W((size_t)n);
    for (int64_t i = 0; i < n; ++i) W[i] = {wins[4 * i], wins[4 * i + 1], wins[4 * i + 2], wins[4 * i + 3]};
    std::vector<Step> steps;
    int stop = site(n, rows, cols, W.data(), words, stride, nrows, ncols, target, max_selected,
                    naive != 0, steps, cum_out);
    *nsteps = (int64_t)steps.size();
    for (int64_t i = 0; i < (int64_t)steps.size() && i < cap; ++i) {
        idx[i] = steps[i].index; srow[i] = steps[i].row; scol[i] = steps[i].col;
        gain[i] = steps[i].gain; cov[i] = steps[i].coverage;
    }
    return stop;
}

}  // extern "C"

extern "C" {

// elevation_between at the rational fraction m/n: z0*(1-m/n) + z1*m/n
double txo_elevation_between(int64_t z0, int64_t z1, int64_t m, int64_t n) {
    return (double)(z0 * (n - m) + z1 * m) / (double)n;
}

// decision D11: observers (next_below(nrows), next_below(ncols)) from SplitMix64(seed)
void txo_random_observers(int64_t nrows, int64_t ncols, int64_t n, uint64_t seed, int32_t* rows, int32_t* cols) {
    SplitMix64 s(seed);
    for (int64_t i = 0; i < n; ++i) {
        rows[i] = (int32_t)s.next_below((uint64_t)nrows);
        cols[i] = (int32_t)s.next_below((uint64_t)ncols);
    }
}

}  // extern "C"

extern "C" {

// Exact viewsheds plus the mask of their grazing-tie cells (tangent == horizon).
void txo_viewshed_ties(const int16_t* z, int64_t nrows, int64_t ncols, int64_t roi, int64_t ht, int64_t hr,
                       int64_t r, int64_t c, uint64_t* words, uint64_t* ties) {
    Grid g{nrows, ncols, z};
    Window w;
    compute_viewshed(g, r, c, roi, ht, hr, &w, words, ties);
}

// LOS classification for tie accounting: 1 blocked, 0 visible with a crossing
// exactly ON the LOS (grazing tie), -1 visible with clearance.
int txo_los_class(const int16_t* z, int64_t nrows, int64_t ncols, int64_t tr, int64_t tc,
                  int64_t ht, int64_t rr, int64_t rc, int64_t hr) {
    Grid g{nrows, ncols, z};
    if (!is_visible(g, tr, tc, ht, rr, rc, hr)) return 1;
    const int64_t E = g.at(tr, tc) + ht, Zt = g.at(rr, rc) + hr, D = Zt - E;
    const int64_t dr = rr - tr, dc = rc - tc, nr = std::llabs(dr), nc = std::llabs(dc);
    const int64_t sr = dr >= 0 ? 1 : -1, sc = dc >= 0 ? 1 : -1;
    bool tie = false;
    walk(0, 0, dr, dc, false, [&](const Crossing& x) {
        int64_t n, k, zn;
        if (x.kind == RowLine) {
            n = nr; k = x.ir;
            const int64_t num = k * nc, q = num / nr, m = num % nr, r = tr + sr * k;
            zn = g.at(r, tc + sc * q) * (n - m) + g.at(r, tc + sc * (q + 1)) * m;
        } else if (x.kind == ColLine) {
            n = nc; k = x.ic;
            const int64_t num = k * nr, q = num / nc, m = num % nc, c = tc + sc * k;
            zn = g.at(tr + sr * q, c) * (n - m) + g.at(tr + sr * (q + 1), c) * m;
        } else if (nr > 0) {
            n = nr; k = x.ir;
            zn = g.at(tr + sr * k, tc + sc * (k * nc / nr)) * n;
        } else {
            n = nc; k = x.ic;
            zn = g.at(tr, tc + sc * k) * n;
        }
        if (zn == E * n + k * D) tie = true;
        return true;
    });
    return tie ? 0 : -1;
}

}  // extern "C"
