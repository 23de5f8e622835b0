// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header comment).
//
// Built with -O3 -ffp-contract=off (the restated walk's fp64
// t/row/col must not be FMA-contracted to match the reference header bit for
// bit).  All LOS predicates are evaluated in exact integer arithmetic: the
// real-number predicate of SPEC.md:120,144 ("interpolated terrain strictly
// above the LOS") with no rounding at all.  DESIGN.md §2 D2 explains why this
// replaces SPEC.md:147's fp64 and how the differing bits against the fp64
// formula are counted (oracle/ref_fp64.cpp).
#include "oracle.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <numeric>
#include <queue>
#include <thread>
#include <tuple>

namespace txo {

// parallel.hpp:9-42 restated: static contiguous chunks, disjoint writes.
template <class Fn>
static void parallel_chunks(int64_t n, unsigned threads, Fn&& fn) {
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

uint64_t mix_seed(uint64_t a, uint64_t b, uint64_t c) {   // rng.hpp:31-36
    SplitMix64 s(a);
    uint64_t h = s.next() ^ (b * 0xFF51AFD7ED558CCDull);
    SplitMix64 t(h);
    return t.next() ^ (c * 0xC4CEB9FE1A85EC53ull);
}

// ---------------------------------------------------------------------------
// generate_fractal — SPEC.md:61-69; decision D10.
// Integer diamond-square on a (2^k+1)^2 canvas, displacement of canvas point
// (y,x) at amplitude A is SplitMix64(mix_seed(seed,y,x)).next() % (2A+1) - A,
// amplitudes amp[i] = floor(A0 * r^(i+1)) (corners use amp[0], level L uses
// amp[L+1]), averages use floor division, the top-left nrows x ncols crop is
// mapped z = mid + floor(v*(zmax-zmin) / 2^21), clamped to [zmin,zmax].
// ---------------------------------------------------------------------------
static inline int64_t floordiv(int64_t a, int64_t b) {
    int64_t q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
    return q;
}
static inline int32_t disp(uint64_t seed, int64_t y, int64_t x, int64_t A) {
    if (A <= 0) return 0;
    SplitMix64 s(mix_seed(seed, (uint64_t)y, (uint64_t)x));
    return (int32_t)((int64_t)(s.next() % (uint64_t)(2 * A + 1)) - A);
}

int generate_fractal(int64_t nrows, int64_t ncols, double roughness, uint64_t seed,
                     int32_t zmin, int32_t zmax, int16_t* out, unsigned threads) {
    if (nrows < 2 || ncols < 2 || zmin > zmax || !(roughness > 0.0) || roughness > 1.0) return 1;
    int k = 1;
    while (((int64_t)1 << k) + 1 < std::max(nrows, ncols)) ++k;
    const int64_t N = ((int64_t)1 << k) + 1;
    const int64_t A0 = (int64_t)1 << 20;
    std::vector<int64_t> amp(k + 1);
    double a = (double)A0;
    for (int i = 0; i <= k; ++i) { a *= roughness; amp[i] = (int64_t)std::floor(a); }
    std::vector<int32_t> cv((size_t)(N * N));
    auto C = [&](int64_t y, int64_t x) -> int32_t& { return cv[(size_t)(y * N + x)]; };
    for (int64_t y : {(int64_t)0, N - 1})
        for (int64_t x : {(int64_t)0, N - 1}) C(y, x) = disp(seed, y, x, amp[0]);
    for (int L = 0; L < k; ++L) {
        const int64_t s = (int64_t)1 << (k - L), h = s / 2, A = amp[L + 1];
        const int64_t nc = (N - 1) / s;           // squares per side
        // diamond: centres (h + i*s, h + j*s)
        parallel_chunks(nc, threads, [&](int64_t b, int64_t e) {
            for (int64_t i = b; i < e; ++i)
                for (int64_t j = 0; j < nc; ++j) {
                    const int64_t y = h + i * s, x = h + j * s;
                    int64_t sum = (int64_t)C(y - h, x - h) + C(y - h, x + h) + C(y + h, x - h) + C(y + h, x + h);
                    C(y, x) = (int32_t)(floordiv(sum, 4) + disp(seed, y, x, A));
                }
        });
        // square: points with (y/h + x/h) odd
        const int64_t nrow = (N - 1) / h + 1;
        parallel_chunks(nrow, threads, [&](int64_t b, int64_t e) {
            for (int64_t iy = b; iy < e; ++iy) {
                const int64_t y = iy * h;
                for (int64_t x = ((iy & 1) ? 0 : h); x < N; x += s) {
                    int64_t sum = 0, cnt = 0;
                    if (y - h >= 0) { sum += C(y - h, x); ++cnt; }
                    if (y + h < N) { sum += C(y + h, x); ++cnt; }
                    if (x - h >= 0) { sum += C(y, x - h); ++cnt; }
                    if (x + h < N) { sum += C(y, x + h); ++cnt; }
                    C(y, x) = (int32_t)(floordiv(sum, cnt) + disp(seed, y, x, A));
                }
            }
        });
    }
    const int64_t range = (int64_t)zmax - zmin;
    const int64_t mid = (int64_t)zmin + range / 2;
    parallel_chunks(nrows, threads, [&](int64_t b, int64_t e) {
        for (int64_t y = b; y < e; ++y)
            for (int64_t x = 0; x < ncols; ++x) {
                int64_t v = mid + floordiv((int64_t)C(y, x) * range, (int64_t)1 << 21);
                v = std::min<int64_t>(std::max<int64_t>(v, zmin), zmax);
                out[y * ncols + x] = (int16_t)v;
            }
    });
    return 0;
}

// ---------------------------------------------------------------------------
// is_visible — SPEC.md:117-126; strict '>'; posts read directly
// (SPEC.md:146); crossings from walk() (grid_walk.hpp:27) on relative
// coordinates (D1).  Exact: with n = |dr| (row line i, t = i/n) the test
// z(t) > E + t(Zt-E) is  z0*(n-m) + z1*m  >  E*n + i*(Zt-E),  m = i*|dc| mod n.
// ---------------------------------------------------------------------------
bool is_visible(const Grid& g, int64_t tr, int64_t tc, int64_t ht,
                int64_t rr, int64_t rc, int64_t hr) {
    const int64_t E = g.at(tr, tc) + ht, Zt = g.at(rr, rc) + hr, D = Zt - E;
    const int64_t dr = rr - tr, dc = rc - tc;
    const int64_t nr = std::llabs(dr), nc = std::llabs(dc);
    const int64_t sr = dr >= 0 ? 1 : -1, sc = dc >= 0 ? 1 : -1;
    return walk(0, 0, dr, dc, false, [&](const Crossing& x) {
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
        return !(zn > E * n + k * D);
    });
}

// ---------------------------------------------------------------------------
// estimate_vix — SPEC.md:176-195, draw order D6: per post one stream
// SplitMix64(mix_seed(seed,row,col)); per sample draw dr then dc with
// next_below(2R+1)-R, reject outside the lattice disk or the grid; self allowed.
// ---------------------------------------------------------------------------
// The VixMap score of one post (D6 draw order).
static uint8_t vix_score(const Grid& g, int64_t roi, int64_t ht, int64_t hr, int64_t samples, uint64_t seed,
                         int64_t r, int64_t c, int arith) {
    const uint64_t span = (uint64_t)(2 * roi + 1);
    const int64_t R2 = roi * roi;
    SplitMix64 s(mix_seed(seed, (uint64_t)r, (uint64_t)c));
    int64_t vis = 0;
    for (int64_t k = 0; k < samples; ++k) {
        int64_t dr, dc;
        for (;;) {
            dr = (int64_t)s.next_below(span) - roi;
            dc = (int64_t)s.next_below(span) - roi;
            if (dr * dr + dc * dc <= R2 && g.in(r + dr, c + dc)) break;
        }
        vis += is_visible_arith(g, r, c, ht, r + dr, c + dc, hr, arith) ? 1 : 0;
    }
    return (uint8_t)vis;
}

void estimate_vix(const Grid& g, int64_t roi, int64_t ht, int64_t hr, int64_t samples,
                  uint64_t seed, unsigned threads, uint8_t* scores,
                  int64_t row_begin, int64_t row_end, int arith) {
    const int64_t rows = row_end - row_begin;
    parallel_chunks(rows * g.ncols, threads, [&](int64_t b, int64_t e) {
        for (int64_t idx = b; idx < e; ++idx) {
            const int64_t r = row_begin + idx / g.ncols, c = idx % g.ncols;
            scores[r * g.ncols + c] = vix_score(g, roi, ht, hr, samples, seed, r, c, arith);
        }
    });
}

void estimate_vix_cols(const Grid& g, int64_t roi, int64_t ht, int64_t hr, int64_t samples, uint64_t seed,
                       int64_t r, int64_t c0, int64_t c1, uint8_t* row_out, int arith) {
    for (int64_t c = c0; c < c1; ++c) row_out[c] = vix_score(g, roi, ht, hr, samples, seed, r, c, arith);
}

// ---------------------------------------------------------------------------
// find_candidates — SPEC.md:238-259, D7: blocks in block-row-major order;
// within a block score desc, then (row, col) asc; min(per_block, size) each.
// ---------------------------------------------------------------------------
std::vector<Cand> find_candidates(const uint8_t* scores, int64_t nrows, int64_t ncols,
                                  int64_t bw, int64_t per_block, unsigned threads) {
    const int64_t by = (nrows + bw - 1) / bw, bx = (ncols + bw - 1) / bw;
    std::vector<std::vector<Cand>> rows_out((size_t)by);   // per block row, in block order
    parallel_chunks(by, threads, [&](int64_t b, int64_t e) {
        std::vector<Cand> tmp;
        for (int64_t i = b; i < e; ++i)
            for (int64_t j = 0; j < bx; ++j) {
                tmp.clear();
                for (int64_t r = i * bw; r < std::min(nrows, (i + 1) * bw); ++r)
                    for (int64_t c = j * bw; c < std::min(ncols, (j + 1) * bw); ++c)
                        tmp.push_back({(int32_t)r, (int32_t)c, scores[r * ncols + c]});
                const int64_t k = std::min<int64_t>(per_block, (int64_t)tmp.size());
                std::partial_sort(tmp.begin(), tmp.begin() + k, tmp.end(), [](const Cand& x, const Cand& y) {
                    if (x.score != y.score) return x.score > y.score;
                    if (x.row != y.row) return x.row < y.row;
                    return x.col < y.col;
                });
                rows_out[(size_t)i].insert(rows_out[(size_t)i].end(), tmp.begin(), tmp.begin() + k);
            }
    });
    std::vector<Cand> out;
    for (auto& v : rows_out) out.insert(out.end(), v.begin(), v.end());
    return out;
}

// ---------------------------------------------------------------------------
// Viewshed ray template — decision D5.
// Rays are the primitive directions of the midpoint-circle perimeter cells of
// radius R plus the 8 principal directions, in angle order.
// Every lattice-disk cell (a,b) != 0 is owned by the forward ray of least
// perpendicular distance (exact: min cross^2/L^2), ties to the lowest index.
// ---------------------------------------------------------------------------
std::vector<std::pair<int32_t,int32_t>> midpoint_circle(int64_t R) {
    std::vector<std::pair<int32_t,int32_t>> pts;
    int64_t x = R, y = 0, d = 1 - R;
    while (x >= y) {
        const int64_t P[8][2] = {{x, y}, {y, x}, {-y, x}, {-x, y}, {-x, -y}, {-y, -x}, {y, -x}, {x, -y}};
        for (auto& p : P) pts.emplace_back((int32_t)p[0], (int32_t)p[1]);
        ++y;
        if (d < 0) d += 2 * y + 1;
        else { --x; d += 2 * (y - x) + 1; }
    }
    std::sort(pts.begin(), pts.end());
    pts.erase(std::unique(pts.begin(), pts.end()), pts.end());
    return pts;
}

static int half_of(int64_t p, int64_t q) { return (p > 0 || (p == 0 && q > 0)) ? 0 : 1; }

static RayTemplate build_template(int64_t R) {
    RayTemplate T;
    T.roi = R;
    std::vector<std::pair<int32_t,int32_t>> dirs;
    for (auto [a, b] : midpoint_circle(R)) {
        int64_t g = std::gcd(std::llabs(a), std::llabs(b));
        dirs.emplace_back((int32_t)(a / g), (int32_t)(b / g));
    }
    const int32_t pr[8][2] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}, {1, 1}, {1, -1}, {-1, 1}, {-1, -1}};
    for (auto& d : pr) dirs.emplace_back(d[0], d[1]);
    std::sort(dirs.begin(), dirs.end());
    dirs.erase(std::unique(dirs.begin(), dirs.end()), dirs.end());
    // angle order, x = col (q), y = row (p), starting at direction (0,+1)
    std::sort(dirs.begin(), dirs.end(), [](auto A, auto B) {
        int ha = half_of(A.first, A.second), hb = half_of(B.first, B.second);
        if (ha != hb) return ha < hb;
        return (int64_t)A.second * B.first - (int64_t)A.first * B.second > 0;
    });
    const int64_t nr = (int64_t)dirs.size();
    for (auto [p, q] : dirs) { T.p.push_back(p); T.q.push_back(q); }
    std::vector<std::vector<std::tuple<int64_t,int32_t,int32_t>>> own(nr);
    for (int64_t a = -R; a <= R; ++a)
        for (int64_t b = -R; b <= R; ++b) {
            if ((a == 0 && b == 0) || a * a + b * b > R * R) continue;
            int64_t best = -1, bc2 = 0, bl2 = 1;
            for (int64_t r = 0; r < nr; ++r) {
                const int64_t p = T.p[r], q = T.q[r];
                if (a * p + b * q <= 0) continue;
                const int64_t cr = a * q - b * p, c2 = cr * cr, l2 = p * p + q * q;
                if (best < 0 || c2 * bl2 < bc2 * l2) { best = r; bc2 = c2; bl2 = l2; }
            }
            own[best].emplace_back(a * T.p[best] + b * T.q[best], (int32_t)a, (int32_t)b);
        }
    T.cell_begin.push_back(0);
    for (int64_t r = 0; r < nr; ++r) {
        std::sort(own[r].begin(), own[r].end());
        for (auto& [d, a, b] : own[r]) { T.ca.push_back(a); T.cb.push_back(b); }
        T.cell_begin.push_back((int64_t)T.ca.size());
    }
    return T;
}

const RayTemplate& ray_template(int64_t roi) {
    static std::mutex mu;
    static std::map<int64_t, RayTemplate> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(roi);
    if (it == cache.end()) it = cache.emplace(roi, build_template(roi)).first;
    return it->second;
}

Window window_of(int64_t nrows, int64_t ncols, int64_t r, int64_t c, int64_t R) {
    Window w;
    w.row0 = (int32_t)std::max<int64_t>(0, r - R);
    w.col0 = (int32_t)std::max<int64_t>(0, c - R);
    w.h = (int32_t)(std::min<int64_t>(nrows - 1, r + R) - w.row0 + 1);
    w.w = (int32_t)(std::min<int64_t>(ncols - 1, c + R) - w.col0 + 1);
    return w;
}

// compute_viewshed — SPEC.md:285-293 with D5: along each ray a cell owned by it
// is visible iff its receiver tangent (z+h_r-E)/(u_c*L) is >= the running max
// of terrain tangents (z-E)/(u_k*L) over in-grid crossings with u_k < u_c,
// u_c = dot/L^2 its projection (exact cross-multiplied integers).
void compute_viewshed(const Grid& g, int64_t r, int64_t c, int64_t R, int64_t ht, int64_t hr,
                      Window* win_out, uint64_t* words, uint64_t* ties) {
    const RayTemplate& T = ray_template(R);
    const Window win = window_of(g.nrows, g.ncols, r, c, R);
    *win_out = win;
    std::fill(words, words + window_words(win), 0ull);
    if (ties) std::fill(ties, ties + window_words(win), 0ull);
    auto setbit = [&](int64_t rr, int64_t cc, uint64_t* w = nullptr) {
        const int64_t k = (rr - win.row0) * win.w + (cc - win.col0);
        (w ? w : words)[k >> 6] |= 1ull << (k & 63);
    };
    setbit(r, c);
    const int64_t E = g.at(r, c) + ht;
    const int64_t nrays = (int64_t)T.p.size();
    for (int64_t ri = 0; ri < nrays; ++ri) {
        const int64_t cb = T.cell_begin[ri], ce = T.cell_begin[ri + 1];
        if (cb == ce) continue;
        const int64_t p = T.p[ri], q = T.q[ri], L2 = p * p + q * q;
        int64_t K = 1;
        for (int64_t i = cb; i < ce; ++i) {
            const int64_t d = T.ca[i] * p + T.cb[i] * q;
            K = std::max(K, (d + L2 - 1) / L2);
        }
        bool has = false;
        int64_t NH = 0, MH = 1;
        int64_t ci = cb;
        auto test = [&](int64_t i) {
            const int64_t a = T.ca[i], b = T.cb[i], rr = r + a, cc = c + b;
            if (!g.in(rr, cc)) return;
            const int64_t P = g.at(rr, cc) + hr - E, dot = a * p + b * q;
            if (!has || P * L2 * MH >= NH * dot) setbit(rr, cc);
            if (ties && has && P * L2 * MH == NH * dot) setbit(rr, cc, ties);   // tangent == horizon
        };
        const int64_t dr = K * p, dc = K * q;
        const int64_t nr = std::llabs(dr), nc = std::llabs(dc);
        const int64_t sr = dr >= 0 ? 1 : -1, sc = dc >= 0 ? 1 : -1;
        walk(0, 0, dr, dc, false, [&](const Crossing& x) {
            int64_t n, idx, zn;
            bool ok;
            if (x.kind == RowLine) {
                n = nr; idx = x.ir;
                const int64_t num = idx * nc, qd = num / nr, m = num % nr;
                const int64_t rr = r + sr * idx, c0 = c + sc * qd, c1 = c + sc * (qd + 1);
                ok = g.in(rr, c0) && g.in(rr, c1);
                zn = ok ? g.at(rr, c0) * (n - m) + g.at(rr, c1) * m : 0;
            } else if (x.kind == ColLine) {
                n = nc; idx = x.ic;
                const int64_t num = idx * nr, qd = num / nc, m = num % nc;
                const int64_t cc = c + sc * idx, r0 = r + sr * qd, r1 = r + sr * (qd + 1);
                ok = g.in(r0, cc) && g.in(r1, cc);
                zn = ok ? g.at(r0, cc) * (n - m) + g.at(r1, cc) * m : 0;
            } else {
                int64_t rr, cc;
                if (nr > 0) { n = nr; idx = x.ir; rr = r + sr * idx; cc = c + sc * (idx * nc / nr); }
                else { n = nc; idx = x.ic; rr = r; cc = c + sc * idx; }
                ok = g.in(rr, cc);
                zn = ok ? g.at(rr, cc) * n : 0;
            }
            // cells with u_c <= u_k (dot/L2 <= K*idx/n) do not see this crossing
            while (ci < ce && (T.ca[ci] * p + T.cb[ci] * q) * n <= K * idx * L2) test(ci++);
            if (ci == ce || !ok) return false;   // done, or left the grid (prefix)
            const int64_t N = zn - E * n, M = K * idx;
            if (!has || N * MH > NH * M) { has = true; NH = N; MH = M; }
            return true;
        });
        while (ci < ce) test(ci++);
    }
}


// ---------------------------------------------------------------------------
// fp64 forms ("All LOS arithmetic in double-precision floating
// point"), the reference formula: the restated walk's doubles (bit-identical
// to grid_walk.hpp:27-77, pinned in tests/test_oracle_kat.py), interpolation
// z0*(1-f) + z1*f with f = frac(col), LOS height E + t*(Zt-E);
// built -ffp-contract=off, so every operation is one IEEE rounding.
// ---------------------------------------------------------------------------
static inline bool interp_fp64(const Grid& g, int64_t tr, int64_t tc, const Crossing& x, double* zt) {
    int64_t r0, c0, r1, c1;
    double f;
    if (x.kind == Post) {
        r0 = r1 = tr + std::llround(x.row); c0 = c1 = tc + std::llround(x.col); f = 0.0;
        if (!g.in(r0, c0)) return false;
        *zt = (double)g.at(r0, c0);
        return true;
    }
    if (x.kind == RowLine) {
        const double cf = std::floor(x.col);
        f = x.col - cf;
        r0 = r1 = tr + std::llround(x.row); c0 = tc + (int64_t)cf; c1 = c0 + 1;
    } else {
        const double rf = std::floor(x.row);
        f = x.row - rf;
        c0 = c1 = tc + std::llround(x.col); r0 = tr + (int64_t)rf; r1 = r0 + 1;
    }
    if (!g.in(r0, c0) || !g.in(r1, c1)) return false;
    *zt = (double)g.at(r0, c0) * (1.0 - f) + (double)g.at(r1, c1) * f;
    return true;
}

bool is_visible_fp64(const Grid& g, int64_t tr, int64_t tc, int64_t ht,
                     int64_t rr, int64_t rc, int64_t hr) {
    const double E = (double)g.at(tr, tc) + (double)ht, Zt = (double)g.at(rr, rc) + (double)hr;
    return walk(0, 0, rr - tr, rc - tc, false, [&](const Crossing& x) {
        double zt = 0.0;
        interp_fp64(g, tr, tc, x, &zt);
        return !(zt > E + x.t * (Zt - E));
    });
}

bool is_visible_arith(const Grid& g, int64_t tr, int64_t tc, int64_t ht,
                      int64_t rr, int64_t rc, int64_t hr, int arith) {
    return arith == ArithExact ? is_visible(g, tr, tc, ht, rr, rc, hr)
                               : is_visible_fp64(g, tr, tc, ht, rr, rc, hr);
}

// compute_viewshed in fp64 (SPEC.md:321 tangent = rise over 2D
// run).  A crossing's tangent is SURVEY Appendix A D4's key (z - eye) /
// sqrt(row^2 + col^2) on the walk's own doubles; a cell's run is its distance
// along its owner ray (D5), dot / sqrt(L2) -- so in real numbers this is exactly
// compute_viewshed's predicate, and the two differ only where a cell's tangent
// EQUALS the horizon (a grazing tie, decided by fp64 rounding).  euclid = true
// takes the cell's own distance sqrt(a^2 + b^2) instead (D4 verbatim; used only
// to count the bits that choice moves, tests/test_oracle_spec.py).  Horizon =
// max over the owner ray's in-grid crossings before the cell (the exact u order
// of compute_viewshed); cell visible iff its tangent >= the horizon.
void compute_viewshed_fp64(const Grid& g, int64_t r, int64_t c, int64_t R, int64_t ht, int64_t hr,
                           Window* win_out, uint64_t* words, bool euclid) {
    const RayTemplate& T = ray_template(R);
    const Window win = window_of(g.nrows, g.ncols, r, c, R);
    *win_out = win;
    std::fill(words, words + window_words(win), 0ull);
    auto setbit = [&](int64_t rr, int64_t cc) {
        const int64_t k = (rr - win.row0) * win.w + (cc - win.col0);
        words[k >> 6] |= 1ull << (k & 63);
    };
    setbit(r, c);
    const double E = (double)g.at(r, c) + (double)ht;
    const int64_t nrays = (int64_t)T.p.size();
    for (int64_t ri = 0; ri < nrays; ++ri) {
        const int64_t cb = T.cell_begin[ri], ce = T.cell_begin[ri + 1];
        if (cb == ce) continue;
        const int64_t p = T.p[ri], q = T.q[ri], L2 = p * p + q * q;
        int64_t K = 1;
        for (int64_t i = cb; i < ce; ++i) {
            const int64_t d = T.ca[i] * p + T.cb[i] * q;
            K = std::max(K, (d + L2 - 1) / L2);
        }
        bool has = false;
        double H = 0.0;
        int64_t ci = cb;
        auto test = [&](int64_t i) {
            const int64_t a = T.ca[i], b = T.cb[i], rr = r + a, cc = c + b;
            if (!g.in(rr, cc)) return;
            const double run = euclid ? std::sqrt((double)(a * a + b * b))
                                      : (double)(a * p + b * q) / std::sqrt((double)L2);
            const double s = ((double)g.at(rr, cc) + (double)hr - E) / run;
            if (!has || s >= H) setbit(rr, cc);
        };
        const int64_t dr = K * p, dc = K * q;
        const int64_t nr = std::llabs(dr), nc = std::llabs(dc);
        walk(0, 0, dr, dc, false, [&](const Crossing& x) {
            const bool byc = x.kind == ColLine || (x.kind == Post && nr == 0);
            const int64_t n = byc ? nc : nr, idx = byc ? x.ic : x.ir;
            while (ci < ce && (T.ca[ci] * p + T.cb[ci] * q) * n <= K * idx * L2) test(ci++);
            double zt = 0.0;
            if (ci == ce || !interp_fp64(g, r, c, x, &zt)) return false;
            const double s = (zt - E) / std::sqrt(x.row * x.row + x.col * x.col);
            if (!has || s > H) { has = true; H = s; }
            return true;
        });
        while (ci < ce) test(ci++);
    }
}

// ---------------------------------------------------------------------------
// siting — SPEC.md:364-392, D9.  Cum is dense row-major over the terrain
// (SPEC.md:351), viewsheds dense row-major over their window.
// ---------------------------------------------------------------------------
int64_t popcount_words(const uint64_t* w, int64_t n) {
    int64_t s = 0;
    for (int64_t i = 0; i < n; ++i) s += __builtin_popcountll(w[i]);
    return s;
}

static inline uint64_t bits_at(const uint64_t* w, int64_t nwords, int64_t off) {
    const int64_t i = off >> 6, sh = off & 63;
    uint64_t lo = w[i] >> sh;
    if (sh && i + 1 < nwords) lo |= w[i + 1] << (64 - sh);
    return lo;
}

// word-wise AND-NOT with per-row sub-word shifts.
int64_t marginal_gain(const Window& win, const uint64_t* v, const uint64_t* cum,
                      int64_t cum_words, int64_t ncols) {
    const int64_t nv = window_words(win);
    int64_t g = 0;
    for (int64_t y = 0; y < win.h; ++y) {
        const int64_t ov = y * win.w, oc = (int64_t)(win.row0 + y) * ncols + win.col0;
        for (int64_t x = 0; x < win.w; x += 64) {
            const int64_t len = std::min<int64_t>(64, win.w - x);
            const uint64_t mask = len == 64 ? ~0ull : ((1ull << len) - 1);
            g += __builtin_popcountll(bits_at(v, nv, ov + x) & ~bits_at(cum, cum_words, oc + x) & mask);
        }
    }
    return g;
}

int64_t marginal_gain_bitloop(const Window& win, const uint64_t* v, const uint64_t* cum, int64_t ncols) {
    int64_t g = 0;
    for (int64_t y = 0; y < win.h; ++y)
        for (int64_t x = 0; x < win.w; ++x) {
            const int64_t kv = y * win.w + x, kc = (int64_t)(win.row0 + y) * ncols + win.col0 + x;
            if (((v[kv >> 6] >> (kv & 63)) & 1) && !((cum[kc >> 6] >> (kc & 63)) & 1)) ++g;
        }
    return g;
}

void union_into(const Window& win, const uint64_t* v, uint64_t* cum, int64_t ncols) {
    const int64_t nv = window_words(win);
    for (int64_t y = 0; y < win.h; ++y) {
        const int64_t ov = y * win.w, oc = (int64_t)(win.row0 + y) * ncols + win.col0;
        for (int64_t x = 0; x < win.w; x += 64) {
            const int64_t len = std::min<int64_t>(64, win.w - x);
            const uint64_t bits = bits_at(v, nv, ov + x) & (len == 64 ? ~0ull : ((1ull << len) - 1));
            const int64_t o = oc + x, i = o >> 6, sh = o & 63;
            cum[i] |= bits << sh;
            if (sh && (bits >> (64 - sh))) cum[i + 1] |= bits >> (64 - sh);
        }
    }
}

// Lazy greedy (max-heap keyed by (stale gain, stamp)) or the
// naive greedy re-evaluating every candidate each round (the test
// oracle).  Ties: lowest candidate index.
int site(int64_t n, const int32_t* orow, const int32_t* ocol,
         const Window* wins, const uint64_t* words, int64_t stride,
         int64_t nrows, int64_t ncols, double target, int64_t max_selected,
         bool naive, std::vector<Step>& steps, uint64_t* cum_out) {
    const int64_t total = nrows * ncols;
    std::vector<uint64_t> cum((size_t)((total + 63) / 64 + 1), 0);
    auto V = [&](int64_t i) { return words + i * stride; };
    const int64_t cw = (int64_t)cum.size();
    auto gain = [&](int64_t i) { return marginal_gain(wins[i], V(i), cum.data(), cw, ncols); };
    int64_t covered = 0;
    steps.clear();
    int stop = Exhausted;
    std::vector<char> taken((size_t)n, 0);
    using Key = std::tuple<int64_t, int64_t, int64_t>;   // (gain, -index, stamp)
    std::priority_queue<Key> heap;
    if (!naive)
        for (int64_t i = 0; i < n; ++i) heap.emplace(popcount_words(V(i), window_words(wins[i])), -i, 0);
    int64_t round = 0;
    for (;;) {
        if ((int64_t)steps.size() == n) { stop = Exhausted; break; }
        int64_t best = -1, bg = -1;
        if (naive) {
            for (int64_t i = 0; i < n; ++i) {
                if (taken[i]) continue;
                const int64_t gi = gain(i);
                if (gi > bg) { bg = gi; best = i; }
            }
        } else {
            for (;;) {
                auto [g, ni, stamp] = heap.top();
                heap.pop();
                if (stamp == round) { best = -ni; bg = g; break; }
                heap.emplace(gain(-ni), ni, round);
            }
        }
        if (bg <= 0) { stop = ZeroGain; break; }
        union_into(wins[best], V(best), cum.data(), ncols);
        taken[best] = 1;
        covered += bg;
        ++round;
        const double cov = (double)covered / (double)total;
        steps.push_back({best, orow[best], ocol[best], bg, cov});
        if (cov >= target) { stop = TargetReached; break; }
        if (max_selected > 0 && (int64_t)steps.size() >= max_selected) { stop = MaxSelected; break; }
    }
    if (cum_out) std::copy(cum.begin(), cum.begin() + (total + 63) / 64, cum_out);
    return stop;
}

}  // namespace txo
