// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Compiled against the reference's own shipped headers, straight from
// /root/reference/proj/include/txsite/ (never copied into this repo), into
// oracle/_ref/libtxs_ref.so by oracle/Makefile.  It exposes:
//   * the reference walk_crossings (grid_walk.hpp:27-77), SplitMix64/mix_seed
//     (rng.hpp:9-36) and parallel_for_chunks (parallel.hpp:20-42) so the
//     oracle's restatement is pinned bit-for-bit against the real code, and
//     so tests/golden/make_golden.py can write the known-answer fixtures;
//   * the SPEC.md:147 fp64 formulation of is_visible / estimate_vix built on
//     the reference walk_crossings, used only to COUNT the bits where the
//     exact-arithmetic semantics (DESIGN.md §2 D2) differ from fp64 rounding.
// The reference's src/*.cpp are absent, so this is the whole
// of the reference that can be compiled.
#include <txsite/grid_walk.hpp>
#include <txsite/parallel.hpp>
#include <txsite/rng.hpp>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

using txsite::CrossKind;

extern "C" {

uint64_t ref_mix_seed(uint64_t a, uint64_t b, uint64_t c) { return txsite::mix_seed(a, b, c); }

void ref_splitmix(uint64_t seed, int64_t n, int mode, uint64_t arg, uint64_t* out) {
    txsite::SplitMix64 s(seed);
    for (int64_t i = 0; i < n; ++i) {
        if (mode == 0) out[i] = s.next();
        else if (mode == 1) out[i] = s.next_below(arg);
        else { double d = s.next_double(); std::memcpy(&out[i], &d, 8); }
    }
}

int64_t ref_walk(int64_t r0, int64_t c0, int64_t r1, int64_t c1, int include_end,
                 double* t, double* row, double* col, int32_t* kind, int64_t cap) {
    int64_t n = 0;
    txsite::walk_crossings(r0, c0, r1, c1, include_end != 0,
                           [&](double tt, double rr, double cc, CrossKind k) {
                               if (n < cap) { t[n] = tt; row[n] = rr; col[n] = cc; kind[n] = (int32_t)k; }
                               ++n;
                               return true;
                           });
    return n;
}

uint64_t ref_walk_hash(int64_t r0, int64_t c0, int64_t r1, int64_t c1, int include_end, int64_t* count) {
    uint64_t h = 1469598103934665603ull;
    int64_t n = 0;
    auto mix = [&](const void* p, size_t len) {
        const unsigned char* b = (const unsigned char*)p;
        for (size_t i = 0; i < len; ++i) { h ^= b[i]; h *= 1099511628211ull; }
    };
    txsite::walk_crossings(r0, c0, r1, c1, include_end != 0,
                           [&](double tt, double rr, double cc, CrossKind k) {
                               mix(&tt, 8); mix(&rr, 8); mix(&cc, 8);
                               unsigned char kb = (unsigned char)k; mix(&kb, 1);
                               ++n;
                               return true;
                           });
    if (count) *count = n;
    return h;
}

// Records the (begin,end) chunks the reference scheduler hands out, in order.
int64_t ref_chunks(int64_t n, unsigned threads, int64_t* out) {
    std::mutex mu;
    std::vector<std::pair<int64_t,int64_t>> seen;
    txsite::parallel_for_chunks(n, threads, [&](int64_t b, int64_t e) {
        std::lock_guard<std::mutex> lk(mu);
        seen.emplace_back(b, e);
    });
    std::sort(seen.begin(), seen.end());
    for (size_t i = 0; i < seen.size(); ++i) { out[2 * i] = seen[i].first; out[2 * i + 1] = seen[i].second; }
    return (int64_t)seen.size();
}

// SPEC.md:117-147 in fp64 on the reference walk (relative coordinates, D1).
static bool vis_fp64(const int16_t* z, int64_t ncols, int64_t tr, int64_t tc, int64_t ht,
                     int64_t rr, int64_t rc, int64_t hr) {
    auto Z = [&](int64_t r, int64_t c) { return (double)z[r * ncols + c]; };
    const double E = Z(tr, tc) + (double)ht, Zt = Z(rr, rc) + (double)hr;
    return txsite::walk_crossings(0, 0, rr - tr, rc - tc, false,
        [&](double t, double row, double col, CrossKind k) {
            double zt;
            if (k == CrossKind::Post) {
                zt = Z(tr + std::llround(row), tc + std::llround(col));
            } else if (k == CrossKind::RowLine) {
                const double cf = std::floor(col), f = col - cf;
                const int64_t r = tr + std::llround(row), c = tc + (int64_t)cf;
                zt = Z(r, c) * (1.0 - f) + Z(r, c + 1) * f;
            } else {
                const double rf = std::floor(row), f = row - rf;
                const int64_t r = tr + (int64_t)rf, c = tc + std::llround(col);
                zt = Z(r, c) * (1.0 - f) + Z(r + 1, c) * f;
            }
            return !(zt > E + t * (Zt - E));
        });
}

int ref_is_visible_fp64(const int16_t* z, int64_t nrows, int64_t ncols, int64_t tr, int64_t tc,
                        int64_t ht, int64_t rr, int64_t rc, int64_t hr) {
    (void)nrows;
    return vis_fp64(z, ncols, tr, tc, ht, rr, rc, hr) ? 1 : 0;
}

// estimate_vix with the D6 draw order on the reference rng, fp64 LOS.
void ref_estimate_vix_fp64(const int16_t* z, int64_t nrows, int64_t ncols, int64_t roi,
                           int64_t ht, int64_t hr, int64_t samples, uint64_t seed,
                           unsigned threads, uint8_t* scores, int64_t row_begin, int64_t row_end) {
    const uint64_t span = (uint64_t)(2 * roi + 1);
    txsite::parallel_for_chunks((row_end - row_begin) * ncols, threads, [&](int64_t b, int64_t e) {
        for (int64_t idx = b; idx < e; ++idx) {
            const int64_t r = row_begin + idx / ncols, c = idx % ncols;
            txsite::SplitMix64 s(txsite::mix_seed(seed, (uint64_t)r, (uint64_t)c));
            int vis = 0;
            for (int64_t k = 0; k < samples; ++k) {
                int64_t dr, dc;
                for (;;) {
                    dr = (int64_t)s.next_below(span) - roi;
                    dc = (int64_t)s.next_below(span) - roi;
                    const int64_t rr = r + dr, cc = c + dc;
                    if (dr * dr + dc * dc <= roi * roi && rr >= 0 && rr < nrows && cc >= 0 && cc < ncols) break;
                }
                vis += vis_fp64(z, ncols, r, c, ht, r + dr, c + dc, hr) ? 1 : 0;
            }
            scores[r * ncols + c] = (uint8_t)vis;
        }
    });
}

}  // extern "C"
