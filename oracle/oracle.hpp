// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference's multiple-observer siting pipeline
// (arXiv 2006.16783 as specified by /root/reference/SPEC.md, built on the three
// shipped headers proj/include/txsite/{grid_walk,rng,parallel}.hpp).
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs may load this library, and only as the checker or the timed
// CPU baseline.  The product (paper_2006_16783_b200/) never links or calls it.
//
// Parity pinning: the restated walk_crossings / SplitMix64 / mix_seed /
// parallel_for_chunks are checked bit-for-bit against known-answer vectors
// produced by compiling the reference headers themselves (oracle/ref_kat.cpp
// -> oracle/_ref/, fixtures in tests/golden/).  The stage semantics SPEC leaves
// open are frozen in DESIGN.md §2 (decision register) and restated here.
#pragma once
#include <cstdint>
#include <vector>

namespace txo {

// ---- rng.hpp:9-36 restated -------------------------------------------------
struct SplitMix64 {
    uint64_t state;
    explicit SplitMix64(uint64_t s) : state(s) {}
    uint64_t next() {                       // rng.hpp:13-18
        uint64_t z = (state += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    uint64_t next_below(uint64_t n) { return next() % n; }          // rng.hpp:21
    double next_double() { return (double)(next() >> 11) * 0x1.0p-53; }  // rng.hpp:24
};
uint64_t mix_seed(uint64_t a, uint64_t b, uint64_t c = 0);           // rng.hpp:31-36

// ---- grid_walk.hpp:9-13 ----------------------------------------------------
enum Kind : int { RowLine = 0, ColLine = 1, Post = 2 };

// One crossing of walk(): the reference's (t,row,col,kind) plus the exact
// integer line indices (ir for row lines, ic for column lines) the
// exact-arithmetic predicates need.
struct Crossing {
    double t, row, col;
    int kind;
    int64_t ir, ic;   // 1-based indices of the crossed row / column line
};

// grid_walk.hpp:27-77 restated with exact integer ordering (ir*nc vs ic*nr);
// equivalent to the reference's 1e-13 merge tolerance for |d| < 2^25
// (distinct parameters differ by >= 1/(nr*nc)).  f returns false to stop.
template <class F>
bool walk(int64_t r0, int64_t c0, int64_t r1, int64_t c1, bool include_end, F&& f) {
    const int64_t dr = r1 - r0, dc = c1 - c0;
    const int64_t nr = dr < 0 ? -dr : dr, nc = dc < 0 ? -dc : dc;
    const int64_t sr = dr >= 0 ? 1 : -1, sc = dc >= 0 ? 1 : -1;
    int64_t ir = 1, ic = 1;
    while (ir <= nr || ic <= nc) {
        // exact: tr < tc  <=>  ir*nc < ic*nr  (absent lines compare as t=2)
        int cmp;
        if (ir > nr) cmp = 1;
        else if (ic > nc) cmp = -1;
        else { __int128 a = (__int128)ir * nc, b = (__int128)ic * nr; cmp = a < b ? -1 : (a > b ? 1 : 0); }
        Crossing x;
        x.ir = ir; x.ic = ic;
        bool at_end;
        if (cmp < 0) {
            x.t = (double)ir / (double)nr;
            x.row = (double)(r0 + sr * ir);
            x.col = (double)c0 + (dc == 0 ? 0.0 : x.t * (double)dc);
            x.kind = dc == 0 ? Post : RowLine;
            at_end = ir == nr;   // t == 1 here only when nc == 0 (else merged)
            ++ir;
        } else if (cmp > 0) {
            x.t = (double)ic / (double)nc;
            x.row = (double)r0 + (dr == 0 ? 0.0 : x.t * (double)dr);
            x.col = (double)(c0 + sc * ic);
            x.kind = dr == 0 ? Post : ColLine;
            at_end = ic == nc;
            ++ic;
        } else {
            x.t = (double)ir / (double)nr;
            x.row = (double)(r0 + sr * ir);
            x.col = (double)(c0 + sc * ic);
            x.kind = Post;
            at_end = ir == nr;
            ++ir; ++ic;
        }
        if (at_end) {
            if (include_end) {
                Crossing e{1.0, (double)r1, (double)c1, Post, nr, nc};
                return f(e);
            }
            return true;
        }
        if (!f(x)) return false;
    }
    return true;
}

// ---- terrain ---------------------------------------------
struct Grid {
    int64_t nrows = 0, ncols = 0;
    const int16_t* z = nullptr;
    int64_t at(int64_t r, int64_t c) const { return z[r * ncols + c]; }
    bool in(int64_t r, int64_t c) const { return r >= 0 && r < nrows && c >= 0 && c < ncols; }
};

// generate_fractal, decision D10.
int generate_fractal(int64_t nrows, int64_t ncols, double roughness, uint64_t seed,
                     int32_t zmin, int32_t zmax, int16_t* out, unsigned threads);

// ---- los, exact rational evaluation of SPEC.md:120,144 ----
bool is_visible(const Grid& g, int64_t tr, int64_t tc, int64_t ht,
                int64_t rr, int64_t rc, int64_t hr);

// SPEC.md:147 fp64 form (the reference formula) and the selector; arith is
// ArithFp64 (0, the default everywhere) or ArithExact (1, exact rationals).
enum Arith : int { ArithFp64 = 0, ArithExact = 1, ArithFp64Euclid = 2 /* viewsheds only */ };
bool is_visible_fp64(const Grid& g, int64_t tr, int64_t tc, int64_t ht,
                     int64_t rr, int64_t rc, int64_t hr);
bool is_visible_arith(const Grid& g, int64_t tr, int64_t tc, int64_t ht,
                      int64_t rr, int64_t rc, int64_t hr, int arith);

// ---- vix, decision D6 ---------------------------------------
void estimate_vix(const Grid& g, int64_t roi, int64_t ht, int64_t hr, int64_t samples,
                  uint64_t seed, unsigned threads, uint8_t* scores,
                  int64_t row_begin, int64_t row_end, int arith = ArithFp64);
// columns [c0, c1) of row r, written to row_out[c] (single-threaded)
void estimate_vix_cols(const Grid& g, int64_t roi, int64_t ht, int64_t hr, int64_t samples, uint64_t seed,
                       int64_t r, int64_t c0, int64_t c1, uint8_t* row_out, int arith = ArithFp64);

// ---- candidates, decision D7 -----------------------------
struct Cand { int32_t row, col, score; };
std::vector<Cand> find_candidates(const uint8_t* scores, int64_t nrows, int64_t ncols,
                                  int64_t block_width, int64_t per_block, unsigned threads = 0);

// ---- viewshed, decision D5/D8 ----------------------------
struct RayTemplate {
    int64_t roi = 0;
    std::vector<int32_t> p, q;              // primitive directions (row, col), angle order
    std::vector<int64_t> cell_begin;        // per ray offset into cells (size rays+1)
    std::vector<int32_t> ca, cb;            // owned cells (row off, col off), sorted by projection
};
const RayTemplate& ray_template(int64_t roi);
std::vector<std::pair<int32_t,int32_t>> midpoint_circle(int64_t roi);

struct Window { int32_t row0, col0, h, w; };
inline int64_t window_words(const Window& w) { return ((int64_t)w.h * w.w + 63) / 64; }
Window window_of(int64_t nrows, int64_t ncols, int64_t r, int64_t c, int64_t roi);
// ties (optional, window words): the cells whose tangent EQUALS their horizon
void compute_viewshed(const Grid& g, int64_t r, int64_t c, int64_t roi, int64_t ht, int64_t hr,
                      Window* win, uint64_t* words, uint64_t* ties = nullptr);
void compute_viewshed_fp64(const Grid& g, int64_t r, int64_t c, int64_t roi, int64_t ht, int64_t hr,
                           Window* win, uint64_t* words, bool euclid = false);

// ---- siting, decision D9 ---------------------------------
enum Stop : int { TargetReached = 0, ZeroGain = 1, Exhausted = 2, MaxSelected = 3 };
struct Step { int64_t index; int32_t row, col; int64_t gain; double coverage; };

int64_t popcount_words(const uint64_t* w, int64_t n);
int64_t marginal_gain(const Window& win, const uint64_t* v, const uint64_t* cum,
                      int64_t cum_words, int64_t ncols);
int64_t marginal_gain_bitloop(const Window& win, const uint64_t* v, const uint64_t* cum,
                              int64_t ncols);
void union_into(const Window& win, const uint64_t* v, uint64_t* cum, int64_t ncols);

int site(int64_t n, const int32_t* orow, const int32_t* ocol,
         const Window* wins, const uint64_t* words, int64_t stride,
         int64_t nrows, int64_t ncols, double target, int64_t max_selected,
         bool naive, std::vector<Step>& steps, uint64_t* cum_out);

}  // namespace txo
