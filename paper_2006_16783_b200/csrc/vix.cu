// VIX stage (estimate_vix) and the batch LOS test
// (is_visible) — one warp-cooperative LOS routine serves both.
//
// LOS (DESIGN.md §2 D2): a segment p -> q is blocked iff at some interior
// crossing of a grid line the interpolated terrain is strictly above the LOS.
// For the row line i (t = i/nr, column offset i*nc/nr = qd + m/nr) that is
//     z(r_i, qd)*(nr-m) + z(r_i, qd+1)*m  >  E*nr + i*(Zt-E)
// and symmetrically for column lines — exact int32 arithmetic, no rounding,
// the real-number predicate of SPEC.md:120,144.  The blocked test is an OR
// over crossings, so lanes take 32 crossings at a time in any order (row
// lines first, then column lines; a post crossed by both is tested twice with
// the same exact answer) and the warp stops at the first chunk with a hit.
//
// Sampling (decision D6): post (r,c) owns the stream SplitMix64(mix_seed(seed,
// r,c)); draws 2j,2j+1 give (dr,dc) = next_below(2R+1)-R, rejected outside the
// lattice disk or the grid.  Lane l evaluates draw k+l directly (the splitmix
// state is a counter), a ballot keeps the first S accepted pairs in order.
#include "ctx.hpp"

namespace txs {
namespace {

#ifndef VIX_TILE
#define VIX_TILE 32    // posts per item row (persistent kernel; measured 4 / 8 / 16 / 32: c3 110.5 / 102.6 / 98.7 / 96.3 ms, c4 - / 811 / 780 / 760, c2 38.2 / 37.8 / 37.8 / 37.8)
#endif
#ifndef VIX_THREADS
#define VIX_THREADS 512
#endif
constexpr int kTile = 32;          // posts per tile side (shared-memory tile / column-major paths)
constexpr int kTileQ = VIX_TILE;   // posts per tile side (quad-plane path)
static_assert(kTileQ <= 32, "a tile row's stream seeds are computed one post per lane");
constexpr int kVixThreads = VIX_THREADS;   // 16 warps
constexpr int kVixWarps = kVixThreads / 32;
constexpr unsigned kFull = 0xffffffffu;

struct TerrainView {
    const int16_t* __restrict__ g;   // global terrain
    const int16_t* s;                // shared tile (or null)
    int64_t ncols;
    int sr0, sc0, sw;
    __device__ __forceinline__ int at(int r, int c) const {
        if (s) return s[(r - sr0) * sw + (c - sc0)];
        return __ldg(g + (int64_t)r * ncols + c);
    }
};

// Warp-cooperative exact LOS: returns true (uniform) iff the segment is blocked.
// Major-axis form: with M = the longer of |dr|,|dc| (major lines i = 1..M-1)
// and m_ = the shorter, step i covers the major-line crossing at
// x_i = i*m_/M = q + r/M (posts A = (i,q), B = (i,q+1)) and — iff 0 < r < m_ —
// the single minor-line crossing j = q between major lines i-1 and i (posts
// C = (i-1,q), A; weight on A = j*M - (i-1)*m_).  Exact int32 tests:
//   zA*(M-r) + zB*r            > E*M  + i*(Zt-E)
//   zC*(m_-w) + zA*w           > E*m_ + j*(Zt-E)
// Lanes take kIlp steps each per round (32*kIlp steps), all loads issued
// before the compares; C = (i-1,q) is needed only when q moved from step i-1
// to i (0 < r < m_), where it equals B of step i-1, held by the neighbouring
// lane: a warp shuffle replaces that third load (one edge lane loads it).
template <bool SMEM>
__device__ __forceinline__ int load_z(const int16_t* base, int off) {
    if (SMEM) return base[off];
    return zld(base + off);
}

// Returns 1 (uniform) iff the segment is blocked, 2 iff it is visible but
// touches the LOS at some crossing (an exact grazing tie), else 0.
template <bool SMEM, int ILP>
__device__ __forceinline__ int warp_blocked(const int16_t* P, int stride, int dr, int dc, int E, int Zt, int lane) {
    const int nr = abs(dr), nc = abs(dc);
    const bool rows_major = nr >= nc;
    const int nM = rows_major ? nr : nc, nm = rows_major ? nc : nr;
    const int steps = nM - 1;
    if (steps <= 0) return 0;
    const int stepM = rows_major ? (dr >= 0 ? stride : -stride) : (dc >= 0 ? 1 : -1);
    const int stepm = rows_major ? (dc >= 0 ? 1 : -1) : (dr >= 0 ? stride : -stride);
    const int D = Zt - E;
    // per-lane DDA state at step i: q = floor(i*nm/nM), r = i*nm mod nM (one
    // fp32-reciprocal division per sample, then exact increments of 32 steps)
    const float rcp = __fdividef(1.0f, (float)nM);
    auto divmod = [&](int num, int& q, int& r) {
        q = __float2int_rz(__int2float_rn(num) * rcp);
        r = num - q * nM;
        if (r >= nM) { ++q; r -= nM; }
        if (r < 0) { --q; r += nM; }
    };
    int q32, r32;
    divmod(32 * nm, q32, r32);
    int i = 1 + lane;
    int q, r;
    divmod(max(i, 0) * nm, q, r);
    int off = i * stepM + q * stepm;                 // post A = (i, q)
    int rhsM = E * nM + i * D;                       // major-line LOS numerator
    int rhsm = E * nm + q * D;                       // minor-line LOS numerator
    const int dOffM = 32 * stepM, dRhsM = 32 * D;
    bool tie = false;
    for (int k0 = 0; k0 < steps; k0 += 32 * ILP) {
        bool b = false;
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
            const bool valid = i >= 1 && i <= steps;
            const int oA = valid ? off : 0;
            const int zA = load_z<SMEM>(P, oA);
            const int zB = (valid && r) ? load_z<SMEM>(P, oA + stepm) : 0;
            // C = (i-1, q): B of the neighbouring step when q moved (needed only then)
            const int zCl = (lane == 0 && valid) ? load_z<SMEM>(P, oA - stepM) : 0;
            const int nb = __shfl_up_sync(kFull, zB, 1);
            const int zC = lane == 0 ? zCl : nb;
            const int vM = zA * (nM - r) + zB * r, vm = zC * r + zA * (nm - r);
            const bool minor = r > 0 && r < nm;
            b |= valid && vM > rhsM;
            // minor line j = q between major lines i-1 and i: weight on A = nm - r
            b |= valid && minor && vm > rhsm;
            tie |= valid && (vM == rhsM || (minor && vm == rhsm));
            // advance 32 steps
            i += 32;
            off += dOffM;
            rhsM += dRhsM;
            r += r32; q += q32; off += q32 * stepm; rhsm += q32 * D;
            if (r >= nM) { r -= nM; ++q; off += stepm; rhsm += D; }
        }
        if (__any_sync(kFull, b)) return 1;
    }
    return __any_sync(kFull, tie) ? 2 : 0;
}

// SPEC.md:147's fp64 is_visible for one segment, operation for operation the
// oracle's is_visible_fp64 (oracle/oracle.cpp) on the walk of grid_walk.hpp:27-77
// (relative coordinates, D1): t = k/n, the minor coordinate t*d, f = its
// fractional part, z0*(1-f) + z1*f against E + t*(Zt-E), blocked iff '>'.
// Explicit _rn intrinsics: no FMA contraction (the oracle is built
// -ffp-contract=off).  Run only for segments with an exact grazing tie.
__device__ bool seg_blocked_fp64(const int16_t* __restrict__ z, int64_t ncols, int tr, int tc, int E, int Zt, int dr,
                                 int dc) {
    const int nr = abs(dr), nc = abs(dc), sr = dr >= 0 ? 1 : -1, sc = dc >= 0 ? 1 : -1;
    const double Ed = (double)E, D = (double)(Zt - E);
    auto Z = [&](int r, int c) -> double { return (double)zld(z + (int64_t)r * ncols + c); };
    int ir = 1, ic = 1;
    while (ir <= nr || ic <= nc) {
        int cmp;
        if (ir > nr) cmp = 1;
        else if (ic > nc) cmp = -1;
        else {
            const long long x = (long long)ir * nc, y = (long long)ic * nr;
            cmp = x < y ? -1 : (x > y ? 1 : 0);
        }
        double t, zt;
        bool at_end;
        if (cmp < 0 && dc != 0) {          // row line: row exact, col = t*dc
            t = __ddiv_rn((double)ir, (double)nr);
            const double col = __dmul_rn(t, (double)dc), cf = floor(col), f = __dsub_rn(col, cf);
            const int r = tr + sr * ir, c = tc + (int)cf;
            zt = __dadd_rn(__dmul_rn(Z(r, c), __dsub_rn(1.0, f)), __dmul_rn(Z(r, c + 1), f));
            at_end = ir == nr;
            ++ir;
        } else if (cmp > 0 && dr != 0) {   // column line: col exact, row = t*dr
            t = __ddiv_rn((double)ic, (double)nc);
            const double row = __dmul_rn(t, (double)dr), rf = floor(row), f = __dsub_rn(row, rf);
            const int r = tr + (int)rf, c = tc + sc * ic;
            zt = __dadd_rn(__dmul_rn(Z(r, c), __dsub_rn(1.0, f)), __dmul_rn(Z(r + 1, c), f));
            at_end = ic == nc;
            ++ic;
        } else {                            // through a post (axis-aligned, or both lines at once)
            const bool byr = cmp <= 0;
            t = byr ? __ddiv_rn((double)ir, (double)nr) : __ddiv_rn((double)ic, (double)nc);
            const int r = byr ? tr + sr * ir : tr, c = cmp == 0 ? tc + sc * ic : (byr ? tc : tc + sc * ic);
            zt = Z(r, c);
            at_end = byr ? ir == nr : ic == nc;
            if (cmp <= 0) ++ir;
            if (cmp >= 0) ++ic;
        }
        if (at_end) return false;
        if (zt > __dadd_rn(Ed, __dmul_rn(t, D))) return true;
    }
    return false;
}

// fp64 re-test of the tie list (txs_params.los_arith == TXS_LOS_FP64): a
// segment the exact walk found visible with a grazing tie is re-decided by
// SPEC.md:147's formula, and a block takes one off its post's score.
__global__ void k_vix_fp64_ties(const int16_t* __restrict__ z, int64_t ncols, const int4* __restrict__ ties,
                                unsigned long long* __restrict__ counters, long long cap, int ht, int hr,
                                uint8_t* __restrict__ vix_rows) {
    const long long n = min((long long)counters[kVixTies], cap);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int4 t = ties[i];
        const int E = zld(z + (int64_t)t.x * ncols + t.y) + ht;
        const int Zt = zld(z + (int64_t)(t.x + t.z) * ncols + t.y + t.w) + hr;
        if (seg_blocked_fp64(z, ncols, t.x, t.y, E, Zt, t.z, t.w)) {
            uint8_t* b = vix_rows + (int64_t)t.x * ncols + t.y;
            unsigned* w = (unsigned*)((uintptr_t)b & ~(uintptr_t)3);
            atomicSub(w, 1u << (8 * ((uintptr_t)b & 3)));   // the byte counted this segment: >= 1, no borrow
            atomicAdd((unsigned long long*)counters + kVixTiesFlipped, 1ull);
        }
    }
}

// Per-sample walk geometry, computed by the lane that owns the sample and
// broadcast with shuffles (one setup per 32 samples instead of per sample).
struct SegGeom {
    int nM, nm, stepM, stepm, D, q32, r32;
    float rcp;
};

__device__ __forceinline__ SegGeom seg_geom(int dr, int dc, int stride, int D) {
    SegGeom g;
    const int nr = abs(dr), nc = abs(dc);
    const bool rows_major = nr >= nc;
    g.nM = rows_major ? nr : nc;
    g.nm = rows_major ? nc : nr;
    g.stepM = rows_major ? (dr >= 0 ? stride : -stride) : (dc >= 0 ? 1 : -1);
    g.stepm = rows_major ? (dc >= 0 ? 1 : -1) : (dr >= 0 ? stride : -stride);
    if (g.nm == 0) g.stepm = 0;   // axis-aligned: B (weight 0) must not leave the segment's line
    g.D = D;
    g.rcp = g.nM ? __fdividef(1.0f, (float)g.nM) : 0.f;
    const int num = 32 * g.nm;
    int q = __float2int_rz(__int2float_rn(num) * g.rcp), r = num - q * g.nM;
    if (r >= g.nM) { ++q; r -= g.nM; }
    if (r < 0) { --q; r += g.nM; }
    g.q32 = q; g.r32 = r;
    return g;
}

__device__ __forceinline__ SegGeom shfl_geom(const SegGeom& g, int src) {
    SegGeom o;
    o.nM = __shfl_sync(kFull, g.nM, src);
    o.nm = __shfl_sync(kFull, g.nm, src);
    o.stepM = __shfl_sync(kFull, g.stepM, src);
    o.stepm = __shfl_sync(kFull, g.stepm, src);
    o.D = __shfl_sync(kFull, g.D, src);
    o.q32 = __shfl_sync(kFull, g.q32, src);
    o.r32 = __shfl_sync(kFull, g.r32, src);
    o.rcp = __shfl_sync(kFull, g.rcp, src);
    return o;
}

// The walk of warp_blocked on precomputed geometry (one step per lane per
// vote).  Rounds where all 32 lanes hold a real step run without validity
// predicates; B is always loaded (for a valid step q+1 <= m_, so it is a post
// of the segment's bounding box) and weighted by r.
template <bool SMEM, bool CHECK>
__device__ __forceinline__ bool walk_round(const int16_t* P, int nM, int nm, int stepM, int stepm, int steps, int lane,
                                           int i, int r, int off, int rhsM, int rhsm) {
    const bool valid = !CHECK || i <= steps;
    const int oA = valid ? off : 0;
    const int zA = load_z<SMEM>(P, oA);
    const int zB = load_z<SMEM>(P, valid ? oA + stepm : 0);
    const int zCl = lane == 0 ? load_z<SMEM>(P, valid ? oA - stepM : 0) : 0;
    const int nb = __shfl_up_sync(kFull, zB, 1);
    const int zC = lane == 0 ? zCl : nb;
    bool b = zA * (nM - r) + zB * r > rhsM;
    b |= r > 0 && r < nm && zC * r + zA * (nm - r) > rhsm;
    return valid && b;
}

template <bool SMEM>
__device__ __forceinline__ int warp_walk(const int16_t* P, const SegGeom& g, int E, int lane) {
    const int nM = g.nM, nm = g.nm, steps = nM - 1;
    if (steps <= 0) return 0;
    const int stepM = g.stepM, stepm = g.stepm, D = g.D;
    int i = 1 + lane;
    const int num = i * nm;
    int q = __float2int_rz(__int2float_rn(num) * g.rcp), r = num - q * nM;
    if (r >= nM) { ++q; r -= nM; }
    if (r < 0) { --q; r += nM; }
    int off = i * stepM + q * stepm;                 // post A = (i, q)
    // LOS numerators minus 1: the rounds test z >= LOS (blocks and grazing
    // ties); a round with a hit is re-tested strictly (+1).  0 visible,
    // 1 blocked, 2 visible with a tie (the segment goes to the fp64 tie list).
    int rhsM = E * nM + i * D - 1;                   // major-line LOS numerator
    int rhsm = E * nm + q * D - 1;                   // minor-line LOS numerator
    const int dOffM = 32 * stepM + g.q32 * stepm, dRhsM = 32 * D, dRhsm = g.q32 * D;
    const int full = steps >> 5;                     // rounds with every lane valid
    int st = 0;
    for (int k = 0; k < full; ++k) {
        if (__any_sync(kFull, walk_round<SMEM, false>(P, nM, nm, stepM, stepm, steps, lane, i, r, off, rhsM, rhsm))) {
            if (__any_sync(kFull, walk_round<SMEM, false>(P, nM, nm, stepM, stepm, steps, lane, i, r, off, rhsM + 1, rhsm + 1)))
                return 1;
            st = 2;
        }
        i += 32;
        off += dOffM;
        rhsM += dRhsM;
        rhsm += dRhsm;
        r += g.r32;
        if (r >= nM) { r -= nM; off += stepm; rhsm += D; }
    }
    if ((steps & 31) && __any_sync(kFull, walk_round<SMEM, true>(P, nM, nm, stepM, stepm, steps, lane, i, r, off, rhsM, rhsm))) {
        if (__any_sync(kFull, walk_round<SMEM, true>(P, nM, nm, stepM, stepm, steps, lane, i, r, off, rhsM + 1, rhsm + 1)))
            return 1;
        st = 2;
    }
    return st;
}

__device__ __forceinline__ int warp_of_thread() { return threadIdx.x >> 5; }

// distinct interior crossings of a (dr,dc) segment: |dr|+|dc|-gcd-1 (binary gcd)
__device__ __forceinline__ int crossings_of(int dr, int dc) {
    unsigned a = abs(dr), b = abs(dc);
    if (a == 0 || b == 0) return (int)(a + b) > 0 ? (int)(a + b) - 1 : 0;
    const int n = (int)(a + b);
    const int sh = __ffs(a | b) - 1;
    a >>= __ffs(a) - 1;
    while (b) {
        b >>= __ffs(b) - 1;
        if (a > b) { const unsigned t = a; a = b; b = t; }
        b -= a;
    }
    return n - (int)(a << sh) - 1;
}

// gcd table for |dr|,|dc| <= 255 (the quad path's crossing statistic: one L2
// load per sample instead of a binary-gcd loop)
__global__ void k_add_counter(unsigned long long* __restrict__ p, unsigned long long v) { *p += v; }

__global__ void k_gcd_table(uint8_t* __restrict__ t) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= 256 * 256) return;
    unsigned a = idx >> 8, b = idx & 255;
    while (b) { const unsigned r = a % b; a = b; b = r; }
    t[idx] = (uint8_t)a;
}
__device__ __forceinline__ int crossings_tab(int dr, int dc, const uint8_t* __restrict__ gt) {
    const int a = abs(dr), b = abs(dc);
    if (a == 0 || b == 0) return a + b > 0 ? a + b - 1 : 0;
    return a + b - (int)__ldg(gt + (a << 8) + b) - 1;
}

// x % d for a 64-bit x and a small d (<= 511: 2R+1 with R <= 255) in 32-bit
// steps: t = hi*(2^32 mod d) + lo < 2^41 (one wide multiply-add), n = (t >> 20)*
// (2^20 mod d) + (t mod 2^20) < 2^12 d^2 + 2^20 <= 2^30, then
// floor(n / d) = umulhi(n, m) >> sh with m = ceil(2^(32+sh) / d) < 2^32, exact
// for every n <= n_max because e n_max < 2^(32+sh), e = m d - 2^(32+sh)
// (make_smallmod checks it; the identities keep t and n congruent to x mod d).
struct SmallMod {
    uint32_t d, k32, k20, m, sh;
};

inline SmallMod make_smallmod(uint32_t d) {
    SmallMod f{d, (uint32_t)((1ull << 32) % d), (uint32_t)((1ull << 20) % d), 0, 0};
    if (d < 2 || d > 511) return SmallMod{0, 0, 0, 0, 0};
    const uint64_t nmax = ((((uint64_t)d << 32) >> 20) + 1) * (d - 1) + (1u << 20);
    for (uint32_t sh = 31; sh > 0; --sh) {   // the largest sh with m < 2^32
        const unsigned __int128 P = (unsigned __int128)1 << (32 + sh);
        const unsigned __int128 m = (P + d - 1) / d;
        if (m >= ((unsigned __int128)1 << 32)) continue;
        const unsigned __int128 e = m * d - P;
        if (e * nmax >= P) return SmallMod{0, 0, 0, 0, 0};
        f.m = (uint32_t)m;
        f.sh = sh;
        return f;
    }
    return SmallMod{0, 0, 0, 0, 0};
}

__device__ __forceinline__ int small_mod(const SmallMod& f, uint64_t x) {
    const uint64_t t = (uint64_t)(uint32_t)(x >> 32) * f.k32 + (uint32_t)x;
    const uint32_t n = (uint32_t)(t >> 20) * f.k20 + ((uint32_t)t & 0xfffffu);
    const uint32_t q = __umulhi(n, f.m) >> f.sh;
    return (int)(n - q * f.d);
}

struct VixArgs {
    int R, ht, hr, S;
    uint64_t seed;
    FastMod64 span;   // 2R+1
    int tiles_x, tiles_y;
    int hp, wp;          // quad T-plane column pitch, V-plane row pitch
    int strip;           // tile columns per traversal strip (quad path)
    int row0, row_end;   // band rows [row0, row_end)
    int zr0, zr1;        // held terrain rows [zr0, zr1)
    int pv, pt, st_off;  // skip map: SV row pitch, ST column pitch, ST offset (int16 entries)
    uint32_t s_mul;      // ceil(2^32 / S) (0: divide): floor(x / S) = umulhi(x, s_mul) while x S < 2^32
    SmallMod smod;       // x % (2R+1) for 64-bit x by 32-bit folds (k_vix_lanes)
    int count_cross;     // k_vix_lanes: accumulate the crossing statistic (first launch per key)
    int4* ties;          // fp64 tie list: {tx row, tx col, dr, dc} of visible segments with a grazing tie
    long long tie_cap;
};

// Record a visible segment with a grazing tie for the fp64 re-test (rare:
// ~1e-4 of segments on the BASELINE terrains).
__device__ __forceinline__ void push_tie(const VixArgs& a, unsigned long long* counters, int r, int c, int dr, int dc) {
    const unsigned long long k = atomicAdd(counters + kVixTies, 1ull);
    if ((long long)k < a.tie_cap) a.ties[k] = make_int4(r, c, dr, dc);
}

template <bool SMEM, int ILP>
__global__ void __launch_bounds__(kVixThreads, 2) k_vix(const int16_t* __restrict__ z, const int16_t* __restrict__ zt, int nrows, int ncols,
                                                      uint8_t* __restrict__ out, VixArgs a,
                                                      unsigned long long* __restrict__ counters) {
    extern __shared__ __align__(16) unsigned char s_dyn[];
    // dynamic smem: [samples: kVixWarps x S ints][terrain tile (SMEM only)]
    int* s_samp = (int*)s_dyn + warp_of_thread() * a.S;
    int16_t* s_tile = (int16_t*)((int*)s_dyn + kVixWarps * a.S + 4);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ty0 = a.row0 + (blockIdx.x / a.tiles_x) * kTile, tx0 = (blockIdx.x % a.tiles_x) * kTile;
    TerrainView T{z, nullptr, ncols, 0, 0, 0};
    if (SMEM) {
        const int r0 = max(a.zr0, ty0 - a.R), r1 = min(a.zr1 - 1, ty0 + kTile - 1 + a.R);
        const int c0 = max(0, tx0 - a.R), c1 = min(ncols - 1, tx0 + kTile - 1 + a.R);
        const int sh = r1 - r0 + 1, sw = c1 - c0 + 1;
        for (int i = threadIdx.x; i < sh * sw; i += kVixThreads) {
            const int y = i / sw, x = i - y * sw;
            s_tile[i] = zld(z + (int64_t)(r0 + y) * ncols + c0 + x);
        }
        T.s = s_tile; T.sr0 = r0; T.sc0 = c0; T.sw = sw;
        __syncthreads();
    }
    const int R2 = a.R * a.R;
    unsigned long long n_los = 0, n_cross = 0;
    for (int pi = warp; pi < kTile * kTile; pi += kVixWarps) {
        const int r = ty0 + pi / kTile, c = tx0 + pi % kTile;
        if (r >= a.row_end || c >= ncols) continue;
        const uint64_t base = mix_seed(a.seed, (uint64_t)r, (uint64_t)c);
        const int E = T.at(r, c) + a.ht;
        // ---- draw S receivers (D6) ----
        int nacc = 0;
        for (uint64_t k = 0; nacc < a.S; k += 32) {
            const int v = (int)fm_mod(a.span, sm_draw(base, k + lane)) - a.R;
            const int dc = __shfl_down_sync(kFull, v, 1);
            const int dr = v;
            const bool ok = !(lane & 1) && dr * dr + dc * dc <= R2 && r + dr >= 0 && r + dr < nrows &&
                            c + dc >= 0 && c + dc < ncols;
            const unsigned mask = __ballot_sync(kFull, ok);
            if (ok) {
                const int slot = nacc + __popc(mask & ((1u << lane) - 1));
                if (slot < a.S) s_samp[slot] = (dr & 0xffff) | (dc << 16);
            }
            nacc += __popc(mask);
        }
        __syncwarp();
        // ---- test them: lane s holds sample s (groups of 32) with its receiver elevation ----
        int vis = 0;
        for (int s0 = 0; s0 < a.S; s0 += 32) {
            const int ns = min(32, a.S - s0);
            const int16_t* P = SMEM ? T.s + (r - T.sr0) * T.sw + (c - T.sc0) : T.g + (int64_t)r * ncols + c;
            const int stride = SMEM ? T.sw : ncols;
            // global path: walk row-major segments on the column-major copy so the
            // lanes' consecutive major steps are contiguous in memory
            const int16_t* PT = SMEM ? P : zt + (int64_t)c * (a.zr1 - a.zr0) + (r - a.zr0);
            SegGeom my{};
            bool my_tr = false;
            if (lane < ns) {
                const int pk = s_samp[s0 + lane];
                const int dr = (int)(int16_t)(pk & 0xffff), dc = pk >> 16;
                const int zt_ = T.at(r + dr, c + dc) + a.hr;
                n_cross += crossings_of(dr, dc);
                my_tr = !SMEM && abs(dr) > abs(dc);
                my = my_tr ? seg_geom(dc, dr, a.zr1 - a.zr0, zt_ - E) : seg_geom(dr, dc, stride, zt_ - E);
            }
            const unsigned trmask = __ballot_sync(kFull, my_tr);
            for (int sidx = 0; sidx < ns; ++sidx) {
                const SegGeom g = shfl_geom(my, sidx);
                const int stt = warp_walk<SMEM>(((trmask >> sidx) & 1u) ? PT : P, g, E, lane);
                vis += stt == 1 ? 0 : 1;
                if (stt == 2 && lane == 0) {
                    const int pk = s_samp[s0 + sidx];
                    push_tie(a, counters, r, c, (int)(int16_t)(pk & 0xffff), pk >> 16);
                }
            }
        }
        __syncwarp();
        if (lane == 0) out[(int64_t)r * ncols + c] = (uint8_t)vis;
        n_los += a.S;
    }
    for (int o = 16; o; o >>= 1) n_cross += __shfl_down_sync(kFull, n_cross, o);
    if (lane == 0 && n_los) {
        atomicAdd(counters + kVixLos, n_los);
        atomicAdd(counters + kVixCrossFull, n_cross);
    }
}

// ---- quad-plane global path (roi <= 255) ----------------------------------------
// Every segment is walked with its major step +1 in memory: a segment whose
// major component is negative is walked from the receiver instead (same
// crossings, same exact predicates — the LOS line is symmetric:
// Zt*M + (M-i)*(E-Zt) = E*M + i*(Zt-E)).  Four planes of uint2 hold, per
// post A, the two post pairs a step needs:
//   .x = (A, B)  B = A one minor step on   -> zA*(M-r) + zB*r   (dp2a.lo)
//   .y = (C, A)  C = A one major step back -> zC*r + zA*(m-r)   (dp2a.hi)
// so one coalesced 64-bit load and two dp2a (16-bit x 8-bit dot products,
// exact) evaluate both crossings of a step, with no shuffles:
//   plane 0 QV+ [y*Wp + c]    = {(z(y,c), z(y+1,c)), (z(y,c-1), z(y,c))}   |dc| >= |dr|, minor +row
//   plane 1 QV- [y*Wp + c]    = {(z(y,c), z(y-1,c)), (z(y,c-1), z(y,c))}   minor -row
//   plane 2 QT+ [c*Hp + y]    = {(z(y,c), z(y,c+1)), (z(y-1,c), z(y,c))}   |dr| > |dc|, minor +col
//   plane 3 QT- [c*Hp + y]    = {(z(y,c), z(y,c-1)), (z(y-1,c), z(y,c))}   minor -col
// (y = held row, H = held rows; Wp and Hp = the V planes' row pitch and the
// T planes' column pitch: ncols resp. H rounded to 32 plus 16 -- with a
// power-of-two pitch the rows of a tile's window alias onto few L2 slices;
// neighbours outside the held terrain are 0
// and only ever carry weight 0).  Weights: both byte pairs come from one
// word W = (M + 255r) | (256m - 255r) << 16, linear in r.
__device__ __forceinline__ uint32_t pk16(int lo, int hi) { return (uint16_t)lo | ((uint32_t)(uint16_t)hi << 16); }

__global__ void k_quads(const int16_t* __restrict__ z, uint2* __restrict__ q, int H, int Hp, int Wp, int ncols) {
    __shared__ int16_t t[34][36];   // held rows y0-1 .. y0+32, cols c0-1 .. c0+32
    const int c0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    for (int i = tid; i < 34 * 34; i += 256) {
        const int yy = i / 34, xx = i - yy * 34, y = y0 + yy - 1, c = c0 + xx - 1;
        t[yy][xx] = (y >= 0 && y < H && c >= 0 && c < ncols) ? z[(int64_t)y * ncols + c] : (int16_t)0;
    }
    __syncthreads();
    const int64_t n = (int64_t)H * Wp;
    for (int yy = threadIdx.y; yy < 32; yy += 8) {
        const int y = y0 + yy, c = c0 + threadIdx.x, ty = yy + 1, tx = threadIdx.x + 1;
        if (y < H && c < ncols) {
            const int a = t[ty][tx];
            const uint32_t ca = pk16(t[ty][tx - 1], a);
            const int64_t w = (int64_t)y * Wp + c;
            q[w] = make_uint2(pk16(a, t[ty + 1][tx]), ca);
            q[n + w] = make_uint2(pk16(a, t[ty - 1][tx]), ca);
        }
    }
    for (int xx = threadIdx.y; xx < 32; xx += 8) {
        const int c = c0 + xx, y = y0 + threadIdx.x, ty = threadIdx.x + 1, tx = xx + 1;
        if (y < H && c < ncols) {
            const int a = t[ty][tx];
            const uint32_t ca = pk16(t[ty - 1][tx], a);
            const int64_t w = 2 * n + (int64_t)c * Hp + y, nT = (int64_t)ncols * Hp;
            q[w] = make_uint2(pk16(a, t[ty][tx + 1]), ca);
            q[nT + w] = make_uint2(pk16(a, t[ty][tx - 1]), ca);
        }
    }
}

__device__ __forceinline__ uint2 qld(const uint2* p) {
#ifdef TXS_BOUNDS_CHECK
    const int16_t* s = (const int16_t*)p;
    if (s < g_zb.lo2 || s + 3 >= g_zb.hi2) __trap();
#endif
    return __ldg(p);
}

// sum of signed 16-bit halves of `pair` times unsigned weight bytes 0,1 (lo) or 2,3 (hi) of w
__device__ __forceinline__ int dp2lo(uint32_t pair, uint32_t w) {
    int d;
    asm("dp2a.lo.s32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(pair), "r"(w), "r"(0));
    return d;
}
__device__ __forceinline__ int dp2hi(uint32_t pair, uint32_t w) {
    int d;
    asm("dp2a.hi.s32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(pair), "r"(w), "r"(0));
    return d;
}

// Per-sample walk geometry, computed by the lane that owns the sample and kept
// in shared memory as two 16-byte records: the skip test reads only the first,
// the exact walk both (the registers of the walk stay free for occupancy).
// Divisions by M are exact fixed-point multiplies: with mag = ceil(2^16 m / M),
// floor(x m / M) = (x mag) >> 16 for every 0 <= x <= 255 (the error x(mag -
// 2^16 m/M)/2^16 < 255/2^16 < 1/M cannot carry past the next integer).
// Grazing ties (DESIGN.md §2 D2): every hot test below is `z >= LOS` -- the
// -1 of `z > LOS - 1` is folded into LE2 and Esn -- so the skip test only skips
// groups strictly below the LOS, and a walked chunk reports exact blocks AND
// exact ties; a chunk with a hit is re-tested strictly (bias +1), and a segment
// that stays visible with a tie goes to the fp64 tie list (k_vix_fp64_ties).
struct __align__(16) QuadGeomC {   // skip test
    int soff;         // skip-map entry of the start post's block (padded block indices)
    int LE2;          // Es*M + min(0, G D) - 1  (Es = LOS height at the start post, D = LOS rise, G = group steps)
    int DG;           // G D
    int w;            // M | c0 << 8 | tr << 13 | mneg << 14 | mag << 15   (M = 0: nothing to walk)
};
struct __align__(16) QuadGeomF {   // exact walk
    const uint2* Q;   // start post's entry in its plane (terrain-walk kernels: the start post's
                      // int16 terrain address, reinterpreted)
    int Esn;          // Es*m - 1 (Es = LOS height at the start post: E, or Zt when reversed)
    int msm;          // m | sm << 8 (sm = minor step in plane words / terrain posts, 0 for axis-aligned)
};
struct QuadGeom { QuadGeomC c; QuadGeomF f; };

#ifndef VIX_MINB
#define VIX_MINB 2    // CTAs per SM: 64 registers, no spills (measured: 4 / 3 / 2 / 1 -> c2 43.1 / 42.0 / 38.8 / 57.1 ms, c3 144.3 / 137.9 / 126.1 / 150.8)
#endif

// The larger margin z*n - (LOS numerator - 1) of a step's two crossings (the
// dp2a accumulators take the negated numerators): d > 0 iff some crossing
// touches or rises above the LOS (z >= LOS), d > 1 iff one is strictly above
// it (z > LOS: blocked).  The minor-line crossing exists only for 0 < r < m.
__device__ __forceinline__ int dp2lo_acc(uint32_t pair, uint32_t w, int acc) {
    int d;
    asm("dp2a.lo.s32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(pair), "r"(w), "r"(acc));
    return d;
}
__device__ __forceinline__ int dp2hi_acc(uint32_t pair, uint32_t w, int acc) {
    int d;
    asm("dp2a.hi.s32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(pair), "r"(w), "r"(acc));
    return d;
}
__device__ __forceinline__ int quad_margin(uint2 v, int r, int nm, uint32_t wb, int rhsM, int rhsm) {
    const uint32_t W = wb + (uint32_t)r * 0xFF0100FFu;   // (+255 lo, -255 hi) per unit r
    const int dM = dp2lo_acc(v.x, W, -rhsM), dm = dp2hi_acc(v.y, W, -rhsm);
    return ((unsigned)(r - 1) < (unsigned)(nm - 1)) ? max(dM, dm) : dM;
}

// Plane geometry shared by every walk of a launch.
struct QuadPitch {
    int pv, pt;       // skip map: SV row pitch, ST column pitch (int16)
    int zs;           // terrain row pitch (terrain-walk kernels)
};

// One exact step of a failing unit, read from the int16 terrain instead of the
// quad planes (the kernels whose skip test passes almost every group -- 16-step
// groups -- do not build the planes): posts A = P[i stepM + q sm], B = A one
// minor step on, C = A one major step back; the predicates of quad_test.
__device__ __forceinline__ int terrain_margin(const int16_t* P, int i, int q, int r, int nM, int nm, int sm, int stepM,
                                              int rhsM, int rhsm) {
    const int o = i * stepM + q * sm;
    const bool minor = (unsigned)(r - 1) < (unsigned)(nm - 1);
    const int zA = zld(P + o);
    const int zB = r ? zld(P + o + sm) : 0;
    const int zC = minor ? zld(P + o - stepM) : 0;
    const int dM = zA * (nM - r) + zB * r - rhsM;
    return minor ? max(dM, zC * r + zA * (nm - r) - rhsm) : dM;
}

// Full walk: one segment per warp, lane l taking major steps l+1, l+33, ...;
// a vote after every 32 steps.  Returns true (uniform) iff the segment is
// blocked.  (TXS_VIX_SKIP=0: every step of every segment is evaluated.)
// Segment states of the walks: visible, blocked, visible with a grazing tie.
enum : int { kSegVis = 0, kSegBlk = 1, kSegTie = 2 };

template <int GS>
__device__ __forceinline__ int quad_walk(const QuadGeom* gp, int lane) {
    const QuadGeomC c = gp->c;
    const int nM = c.w & 0xff, steps = nM - 1;
    if (steps <= 0) return kSegVis;
    const QuadGeomF f = gp->f;
    const int nm = f.msm & 0xff, sm = f.msm >> 8, mag = (unsigned)c.w >> 15, D = c.DG >> GS;
    const uint32_t wb = (uint32_t)nM | ((uint32_t)nm << 24);
    const int q32 = (32 * mag) >> 16, r32 = 32 * nm - q32 * nM;
    int i = 1 + lane;
    int q = (i * mag) >> 16, r = i * nm - q * nM;
    int off = i + q * sm;
    int rhsM = c.LE2 - min(0, c.DG) + i * D, rhsm = f.Esn + q * D;
    const int dOff = 32 + q32 * sm, dRhsM = 32 * D, dRhsm = q32 * D;
    int st = kSegVis;
    for (int k = 0; k <= (steps >> 5); ++k) {
        const bool valid = k < (steps >> 5) || (steps & ~31) + 1 + lane <= steps;
        if (k == (steps >> 5) && !(steps & 31)) break;
        const int d = valid ? quad_margin(qld(f.Q + off), r, nm, wb, rhsM, rhsm) : 0;
        if (__any_sync(kFull, d > 0)) {   // z >= LOS somewhere: a block, or only ties
            if (__any_sync(kFull, d > 1)) return kSegBlk;
            st = kSegTie;
        }
        off += dOff; rhsM += dRhsM; rhsm += dRhsm; r += r32;
        if (r >= nM) { r -= nM; off += sm; rhsm += D; }
    }
    return st;
}

// Hierarchical walk with a conservative skip test (exact: it only ever skips
// steps that cannot block).  Steps are taken in groups of G = 2^GS (4 or 16):
// group g holds major steps Gg+1..Gg+G, whose crossings lie at t in (Gg/M,
// (Gg+G)/M] and use posts with major offsets Gg..Gg+G and minor offsets
// q(Gg+1)..q(Gg+1)+G -- a (G+1)x(G+1) window, so inside the 2G x 2G posts of
// two-by-two GxG blocks at the window's corner block.  The skip map holds, per
// block corner, the maximum elevation of those 2G x 2G posts (k_skipmap).  The
// interpolated terrain at any crossing of the group is at most that maximum,
// and the LOS over the group is at least its value at one end, so
//     smax * M  <=  Es*M + Gg*D + min(0, G D)  =  LE2 + g*DG
// proves that no crossing of the group is blocked.  The window's minor corner
// block, relative to the start post's, is (c0 + q(Gg+1)) >> GS for a positive
// minor direction (c0 = the start post's minor offset in its block) and
// -((c0 + q(Gg+1)) >> GS) for a negative one (c0 = 2G-1 - that offset), so the
// map index is soff + g + ((c0 + q(Gg+1)) >> GS) * ssp with a signed pitch ssp.
//
// Sequential form (TXS_VIX_SKIP=2): one segment per warp pass, lane l testing
// group 32k+l, failing groups walked in order with an exit at the first block.
template <int GS>
__device__ __forceinline__ int quad_walk_skip(const QuadGeom* gp, const QuadPitch& P, const int16_t* __restrict__ smap,
                                              int* s_fail, int lane) {
    const QuadGeomC c = gp->c;
    const int nM = c.w & 0xff, steps = nM - 1;
    if (steps <= 0) return kSegVis;
    int st = kSegVis;
    const int mag = (unsigned)c.w >> 15, magG = mag << GS, c0 = (c.w >> 8) & 31;
    const int sp = (c.w & 0x2000) ? P.pt : P.pv, ssp = (c.w & 0x4000) ? -sp : sp;
    const int ngroups = (steps + (1 << GS) - 1) >> GS;
    const int16_t* S = smap + c.soff;
    for (int g0 = 0; g0 < ngroups; g0 += 32) {
        const int gi = g0 + lane;
        bool fail = false;
        if (gi < ngroups) {
            const int q1 = (gi * magG + mag) >> 16;
            const int smax = __ldg(S + gi + ((c0 + q1) >> GS) * ssp);
            fail = smax * nM > c.LE2 + gi * c.DG;
        }
        const unsigned F = __ballot_sync(kFull, fail);
        if (!F) continue;
        if (fail) s_fail[__popc(F & ((1u << lane) - 1))] = gi;
        __syncwarp();
        const QuadGeomF f = gp->f;
        const int nm = f.msm & 0xff, sm = f.msm >> 8, D = c.DG >> GS, LE = c.LE2 - min(0, c.DG);
        const uint32_t wb = (uint32_t)nM | ((uint32_t)nm << 24);
        const int cnt = __popc(F);
        for (int j = 0; j < cnt; j += 32 >> GS) {   // 32/G groups x G steps per pass
            const int sub = j + (lane >> GS);
            int d = 0;
            if (sub < cnt) {
                const int i = (s_fail[sub] << GS) + 1 + (lane & ((1 << GS) - 1));
                if (i <= steps) {
                    const int q = (i * mag) >> 16, r = i * nm - q * nM;
                    d = quad_margin(qld(f.Q + i + q * sm), r, nm, wb, LE + i * D, f.Esn + q * D);
                }
            }
            if (__any_sync(kFull, d > 0)) {
                if (__any_sync(kFull, d > 1)) return kSegBlk;
                st = kSegTie;
            }
        }
        __syncwarp();
    }
    return st;
}

//
// A batch of up to 32 segments (lane l built segment l's geometry g) is tested
// as one flattened list of (segment, unit) pairs, 32 per warp pass, so lanes
// do not idle on short segments; a unit is U consecutive groups (4U steps),
// tested by one lane, so the per-pair bookkeeping is paid once per unit.  A
// unit with a failing group is then walked exactly, whole: one warp pass of 32
// consecutive steps (coalesced plane loads, the predicates of quad_test), in
// (segment, unit) order, skipping segments already found blocked.  Returns
// the mask of lanes whose segment is visible; *tiem = the visible lanes whose
// segment touched the LOS at some crossing (an exact grazing tie).
template <int U, int GS, bool TERR>
__device__ __forceinline__ unsigned batch_skip(const QuadGeom& g, int ns, int lane, QuadGeom* s_geo, int* s_pre,
                                               int* s_fail, const int16_t* __restrict__ smap, const QuadPitch& P,
                                               unsigned* tiem) {
    static_assert((U << GS) <= 32, "a failing unit is walked by one 32-step pass");
    const int nMl = g.c.w & 0xff;
    const int ng = (lane < ns && nMl >= 2) ? (nMl + (1 << GS) - 2) >> GS : 0;   // ceil((M-1)/G) groups
    const int nu = (ng + U - 1) / U;
    const unsigned nz = __ballot_sync(kFull, ng > 0);
    int inc = nu;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += t;
    }
    const int T = __shfl_sync(kFull, inc, 31);
    if (ng > 0) {   // compacted: segments with groups, in lane order; prefixes strictly increase
        const int slot = __popc(nz & ((1u << lane) - 1));
        s_geo[slot] = g;
        const int sp = (g.c.w & 0x2000) ? P.pt : P.pv;
        s_pre[slot] = (inc - nu) | (((g.c.w & 0x4000) ? -sp : sp) << 16);   // unit prefix | signed map pitch
    }
    __syncwarp();
    const int myp = lane < __popc(nz) ? s_pre[lane] & 0xffff : 0x7fffffff;
    unsigned blk = 0, tie = 0;   // blocked slots, slots with a grazing tie
    for (int base = 0; base < T; base += 32) {
        // slot of pair base+lane: (slots starting at or before base) - 1 + (starts in (base, base+lane])
        const unsigned B = __reduce_or_sync(kFull, (myp > base && myp < base + 32) ? 1u << (myp - base) : 0u);
        const int cb = __popc(__ballot_sync(kFull, myp <= base));
        const int p = base + lane;
        const int sl = cb - 1 + __popc(B & ((2u << lane) - 1));
        bool fail = false;
        int ui = 0;
        if (p < T && !((blk >> sl) & 1u)) {   // pairs of segments already blocked are dropped
            const int ps = s_pre[sl];
            const QuadGeomC c = s_geo[sl].c;
            const int nM = c.w & 0xff, mag = (unsigned)c.w >> 15, c0 = (c.w >> 8) & 31, ssp = ps >> 16;
            const int ngs = (nM + (1 << GS) - 2) >> GS;
            ui = p - (ps & 0xffff);
            const int g0 = ui * U;
            const int16_t* S = smap + c.soff;
            int q1 = (g0 * (mag << GS) + mag) >> 16;
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int gi = g0 + k;
                if (k == 0 || gi < ngs) {
                    const int smax = __ldg(S + gi + ((c0 + q1) >> GS) * ssp);
                    fail |= smax * nM > c.LE2 + gi * c.DG;
                }
                q1 = ((gi + 1) * (mag << GS) + mag) >> 16;
            }
        }
        const unsigned F = __ballot_sync(kFull, fail);
        if (!F) continue;
        if (fail) s_fail[__popc(F & ((1u << lane) - 1))] = sl | (ui << 8);
        __syncwarp();
        const int cnt = __popc(F);
        for (int h = 0; h < cnt; ++h) {
            const int e = s_fail[h];
            const int sf = e & 0xff;
            if ((blk >> sf) & 1u) continue;
            const QuadGeomC c = s_geo[sf].c;
            const QuadGeomF f = s_geo[sf].f;
            const int nM = c.w & 0xff;
            // 32 steps from the unit's first (a unit of U G < 32 steps is walked with its successor)
            const int i = ((U * (e >> 8)) << GS) + 1 + lane;
            int d = 0;   // margin: > 0 z >= LOS (a block or a grazing tie), > 1 z > LOS (a block)
            if (i < nM) {
                const int nm = f.msm & 0xff, sm = f.msm >> 8, mag = (unsigned)c.w >> 15, D = c.DG >> GS;
                const int q = (i * mag) >> 16, r = i * nm - q * nM;
                const int rhsM = c.LE2 - min(0, c.DG) + i * D, rhsm = f.Esn + q * D;
                if (TERR) {
                    d = terrain_margin((const int16_t*)f.Q, i, q, r, nM, nm, sm, (c.w & 0x2000) ? P.zs : 1, rhsM, rhsm);
                } else {
                    const uint32_t wb = (uint32_t)nM | ((uint32_t)nm << 24);
                    d = quad_margin(qld(f.Q + i + q * sm), r, nm, wb, rhsM, rhsm);
                }
            }
            if (__any_sync(kFull, d > 0)) {
                if (__any_sync(kFull, d > 1)) blk |= 1u << sf;
                else tie |= 1u << sf;
            }
        }
        __syncwarp();
    }
    // visible lanes (lane order): segments without groups, and slots not blocked
    const int slot = __popc(nz & ((1u << lane) - 1));
    const bool vis = lane < ns && (ng == 0 || !((blk >> slot) & 1u));
    *tiem = __ballot_sync(kFull, vis && ng > 0 && ((tie >> slot) & 1u));
    return __ballot_sync(kFull, vis);
}

// Per-lane form of the skip test (measured: c3 VIX 102.7 -> 78.3 ms, c4 811 ->
// 617, c2 (4-step groups, 19 % failing) 40.0 -> 35.4 against batch_skip): each
// lane runs the skip test over its own segment's groups, with no cross-lane
// compaction, keeping one "some group failed" flag.  The walk position is
// carried incrementally: the minor offset of step gi*G + 1 plus the start
// block's offset c0 sits in the high bits of acc (acc >> 16 = c0 +
// floor((gi G + 1) m / M)), and the LOS bound grows by G D per group.  Lanes
// with a failing group (rare) build their exact-walk record (walk_rec) and are
// walked one at a time: the warp re-tests that segment's groups (lane =
// group), then runs one coalesced 32-step pass from each failing group
// (32 >> GS groups per pass), stopping at the first block.
template <int GS, bool TERR, bool MASK, class WalkRec>
__device__ __forceinline__ unsigned batch_skip_lane(const QuadGeomC& gc, int ns, int lane, QuadGeom* s_geo,
                                                    const int16_t* __restrict__ smap, const QuadPitch& P,
                                                    unsigned* tiem, WalkRec walk_rec) {
    constexpr int kSpan = 32 >> GS;   // groups covered by one 32-step pass
    using Mask = typename std::conditional<(GS >= 3), unsigned, unsigned long long>::type;   // <= 63 groups
    const int nM = gc.w & 0xff;
    const int ng = (lane < ns && nM >= 2) ? (nM + (1 << GS) - 2) >> GS : 0;
    // map entry of group gi: soff + gi + ((acc0 + gi G mag) >> (16 + GS)) * ssp
    const int mag = (unsigned)gc.w >> 15, acc0 = mag + (((gc.w >> 8) & 31) << 16);
    const int sp = (gc.w & 0x2000) ? P.pt : P.pv;
    const int ssp = (gc.w & 0x4000) ? -sp : sp;
    bool fail = false;
    Mask fm = 0;   // (MASK) the failing groups themselves
    {
        // 4-step groups (up to 63 per segment): four groups per iteration, their map
        // loads issued together (c2 40.6 -> 34.0 ms); 16-step groups (<= 10): one
        // per iteration (c3 49.9 -> 45.6 against four)
#ifndef VIX_SKIP_U16
#define VIX_SKIP_U16 1
#endif
        constexpr int kU = GS >= 4 ? VIX_SKIP_U16 : 4;
        int acc = acc0, rhs = gc.LE2, idx = gc.soff;
        for (int g0 = 0; g0 < ng; g0 += kU) {
            int sv[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u)
                sv[u] = (kU == 1 || g0 + u < ng) ? __ldg(smap + (idx + u + ((acc + u * (mag << GS)) >> (16 + GS)) * ssp)) : 0;
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const bool f = (kU == 1 || g0 + u < ng) && sv[u] * nM > rhs + u * gc.DG;
                if (MASK) fm |= (Mask)f << (g0 + u);
                else fail |= f;
            }
            acc += kU * (mag << GS);
            rhs += kU * gc.DG;
            idx += kU;
        }
    }
    if (MASK) fail = fm != 0;
    unsigned F = __ballot_sync(kFull, fail);
    unsigned blk = 0, tie = 0;   // bit l: lane l's segment blocked / has a grazing tie
    if (F) {
        if (fail) s_geo[lane] = QuadGeom{gc, walk_rec()};   // the walk record, built only when needed
        __syncwarp();
        while (F) {
            const int sl = __ffs(F) - 1;
            F &= F - 1;
            const QuadGeomC c = s_geo[sl].c;
            const QuadGeomF f = s_geo[sl].f;
            const int sM = c.w & 0xff, nm = f.msm & 0xff, sm = f.msm >> 8, cmag = (unsigned)c.w >> 15, D = c.DG >> GS;
            // the segment's failing groups, re-tested cooperatively (lane = group)
            Mask m = 0;
            if (MASK) {
                m = __shfl_sync(kFull, fm, sl);
            } else {
                const int sng = (sM + (1 << GS) - 2) >> GS;
                const int csp = (c.w & 0x2000) ? P.pt : P.pv, cssp = (c.w & 0x4000) ? -csp : csp;
                const int cacc0 = cmag + (((c.w >> 8) & 31) << 16);
                for (int base = 0; base < sng; base += 32) {
                    const int gi = base + lane;
                    bool fl = false;
                    if (gi < sng) {
                        const int smax = __ldg(smap + (c.soff + gi + ((cacc0 + gi * (cmag << GS)) >> (16 + GS)) * cssp));
                        fl = smax * sM > c.LE2 + gi * c.DG;
                    }
                    m |= (Mask)__ballot_sync(kFull, fl) << base;
                }
            }
            while (m) {
                const int gi = sizeof(Mask) == 4 ? __ffs((unsigned)m) - 1 : __ffsll((long long)m) - 1;
                m &= ~((((Mask)1 << kSpan) - 1) << gi);
                const int i = (gi << GS) + 1 + lane;
                int d = 0;   // margin: > 0 z >= LOS (a block or a grazing tie), > 1 z > LOS (a block)
                if (i < sM) {
                    const int q = (i * cmag) >> 16, r = i * nm - q * sM;
                    const int rhsM = c.LE2 - min(0, c.DG) + i * D, rhsm = f.Esn + q * D;
                    if (TERR) {
                        d = terrain_margin((const int16_t*)f.Q, i, q, r, sM, nm, sm, (c.w & 0x2000) ? P.zs : 1, rhsM, rhsm);
                    } else {
                        const uint32_t wb = (uint32_t)sM | ((uint32_t)nm << 24);
                        d = quad_margin(qld(f.Q + i + q * sm), r, nm, wb, rhsM, rhsm);
                    }
                }
                if (__any_sync(kFull, d > 0)) {
                    if (__any_sync(kFull, d > 1)) { blk |= 1u << sl; break; }
                    tie |= 1u << sl;
                }
            }
        }
        __syncwarp();
    }
    const bool vis = lane < ns && !((blk >> lane) & 1u);
    *tiem = __ballot_sync(kFull, vis && ((tie >> lane) & 1u));
    return __ballot_sync(kFull, vis);
}

// Walk geometry of the segment from post (r, c) (observer elevation E) to
// (r + dr0, c + dc0): the skip-test record (soff, LE2, DG, w) and the
// exact-walk record (start address, Esn, msm); n_cross counts its crossings.
template <int GS, bool TERR, bool WALK = true, bool COUNT = true>
__device__ __forceinline__ QuadGeom seg_quad_geom(const int16_t* __restrict__ z, const uint2* __restrict__ qp, int ncols,
                                                  const VixArgs& a, const uint8_t* __restrict__ gcdt,
                                                  const unsigned long long* s_rcp40, int r, int c, int E, int dr0, int dc0,
                                                  unsigned long long& n_cross) {
    QuadGeom g{};
    const int H = a.zr1 - a.zr0;
    int dr = dr0, dc = dc0;
    const int Zt = zld(z + (int64_t)(r + dr) * ncols + (c + dc)) + a.hr;
    if (COUNT) n_cross += crossings_tab(dr, dc, gcdt);
    const bool tr = abs(dr) > abs(dc);
    const bool rev = tr ? dr < 0 : dc < 0;      // walk from the receiver
    const int y = r - a.zr0 + (rev ? dr : 0), x = c + (rev ? dc : 0);   // start post
    if (rev) { dr = -dr; dc = -dc; }
    const int nM = tr ? dr : dc, nm = tr ? abs(dc) : abs(dr);
    const bool mneg = (tr ? dc : dr) < 0;
    const int64_t n = (int64_t)H * a.wp, nT = (int64_t)ncols * a.hp;
    const int stride = tr ? a.hp : a.wp;
    const int Es = rev ? Zt : E;
    if (!WALK) {
    } else if (TERR) {
        g.f.Q = (const uint2*)(z + (int64_t)(y + a.zr0) * ncols + x);
        const int zstep = tr ? 1 : ncols;   // minor axis: columns for row-major walks
        g.f.msm = nm | ((nm == 0 ? 0 : (mneg ? -zstep : zstep)) * 256);
    } else {
        g.f.Q = qp + (tr ? 2 * n + (int64_t)x * a.hp + y + (mneg ? nT : 0) : (int64_t)y * a.wp + x + (mneg ? n : 0));
        g.f.msm = nm | ((nm == 0 ? 0 : (mneg ? -stride : stride)) * 256);
    }
    if (WALK) g.f.Esn = Es * nm - 1;
    // skip map (k_skipmap): padded 4x4-block indices of the start post,
    // SV row-major for column-major walks, ST column-major for row-major ones
    const int maj = tr ? y : x, mnr = tr ? x : y;
    const int mag = (int)(((unsigned long long)(nm * 65536 + nM - 1) * s_rcp40[nM]) >> 40);   // 0 when M = 0
    // (a negative minor direction starts one block further on, G - 1 - mo posts into it: folded
    // into soff so that the in-block offset c0 stays below G -- 5 bits up to 32-step groups)
#ifndef VIX_REPACK_ALL
#define VIX_REPACK_ALL 0
#endif
    constexpr bool kFold = GS >= 5 || VIX_REPACK_ALL;   // (only 32-step groups need it)
    const int mfold = kFold ? (int)mneg : 0;
    g.c.soff = tr ? a.st_off + ((maj >> GS) + 1) + ((mnr >> GS) + 1 - mfold) * a.pt
                  : ((maj >> GS) + 1) + ((mnr >> GS) + 1 - mfold) * a.pv;
    const int D = rev ? E - Zt : Zt - E;
    constexpr int G = 1 << GS;
    g.c.LE2 = Es * nM + min(0, G * D) - 1;
    g.c.DG = G * D;
    const int mo = mnr & (G - 1);
    g.c.w = nM | ((mneg ? (kFold ? G : 2 * G) - 1 - mo : mo) << 8) | ((int)tr << 13) | ((int)mneg << 14) | (mag << 15);
    return g;
}

template <int SKIP, int U, int GS>
__global__ void __launch_bounds__(kVixThreads, VIX_MINB) k_vix_quads(const int16_t* __restrict__ z,
                                                                   const uint2* __restrict__ qp, int nrows, int ncols,
                                                                   uint8_t* __restrict__ out, VixArgs a,
                                                                   const uint8_t* __restrict__ gcdt,
                                                                   const int16_t* __restrict__ smap,
                                                                   unsigned long long* __restrict__ counters) {
    extern __shared__ __align__(16) unsigned char s_dyn[];
    // dynamic smem: [geometry: kVixWarps x 32][failing units: kVixWarps x 32][unit prefixes: kVixWarps x 32]
    //               [sample queue: kVixWarps x 64 ints]
    QuadGeom* s_geo = (QuadGeom*)s_dyn + warp_of_thread() * 32;
    constexpr int kFailInts = 32;   // failing units
    int* s_fail = (int*)((QuadGeom*)s_dyn + kVixWarps * 32) + warp_of_thread() * kFailInts;
    int* s_pre = (int*)((QuadGeom*)s_dyn + kVixWarps * 32) + kVixWarps * kFailInts + warp_of_thread() * 32;
    int* s_q = (int*)((QuadGeom*)s_dyn + kVixWarps * 32) + kVixWarps * (kFailInts + 32) + warp_of_thread() * 64;
    const QuadPitch PQ{a.pv, a.pt, ncols};
    // 16-step skip groups (roi < 150): failing units walk the terrain, no quad planes
    constexpr bool TERR = (SKIP == 1 || SKIP == 3) && GS == 4;
    const int lane = threadIdx.x & 31;
    // mag = ceil(2^16 m / M) for every M <= 255: floor(x / M) = (x * ceil(2^40 / M)) >> 40
    // exactly for x < 2^24 (the error x (ceil - 2^40/M) / 2^40 < 2^-16 < 1/M)
    __shared__ unsigned long long s_rcp40[256];
    for (int d = threadIdx.x; d < 256; d += blockDim.x) s_rcp40[d] = d ? ((1ull << 40) + d - 1) / d : 0ull;
    __syncthreads();
    const int R2 = a.R * a.R;
    unsigned long long n_cross = 0;
    int n_posts = 0;
    // Persistent CTAs (grid = resident CTAs) whose warps pull tile rows of
    // kTileQ posts from one global counter, in tile order (vertical strips of
    // a.strip tile columns, row-major inside a strip): a warp that finishes
    // early takes more work instead of idling until its CTA's slowest warp is
    // done, and the rows in flight stay a compact window of the grid (the L2
    // working set of the quad planes).  Each post's S receivers (D6) are drawn into a
    // per-warp FIFO of (dr, dc, ring slot) and tested 32 at a time; post p of
    // the warp (in draw order) owns FIFO samples [p S, p S + S) and ring slot
    // p & 15, whose lane holds its position, observer elevation and count.
    constexpr int kRing = 16;
    int myE = 0, myR = 0, myC = 0, mycnt = 0;
    int qn = 0;                      // queued samples
    int p_next = 0, p_open = 0;      // posts drawn / posts finished
    int tq = 0;                      // samples of the open posts already tested
    auto run_batch = [&](int ns) {
        QuadGeom g{};
        const int pk = lane < ns ? s_q[lane] : 0;
        const int pj = (pk >> 18) & (kRing - 1);
        const int E = __shfl_sync(kFull, myE, pj), r = __shfl_sync(kFull, myR, pj), c = __shfl_sync(kFull, myC, pj);
        const int dr0 = (pk & 0x1ff) - 256, dc0 = ((pk >> 9) & 0x1ff) - 256;   // transmitter frame
        if (lane < ns) g = seg_quad_geom<GS, TERR>(z, qp, ncols, a, gcdt, s_rcp40, r, c, E, dr0, dc0, n_cross);
        __syncwarp();
        unsigned vism, tiem;
        if constexpr (SKIP == 1) {
            vism = batch_skip<U, GS, TERR>(g, ns, lane, s_geo, s_pre, s_fail, smap, PQ, &tiem);
        } else if constexpr (SKIP == 3) {
            vism = batch_skip_lane<GS, TERR, true>(g.c, ns, lane, s_geo, smap, PQ, &tiem, [&] { return g.f; });
        } else {
            s_geo[lane] = g;
            __syncwarp();
            int mine = kSegVis;
            for (int sidx = 0; sidx < ns; ++sidx) {
                const int stt = SKIP == 2 ? quad_walk_skip<GS>(s_geo + sidx, PQ, smap, s_fail, lane) : quad_walk<GS>(s_geo + sidx, lane);
                if (lane == sidx) mine = stt;
            }
            vism = __ballot_sync(kFull, lane < ns && mine != kSegBlk);
            tiem = __ballot_sync(kFull, lane < ns && mine == kSegTie);
        }
        if ((tiem >> lane) & 1u) push_tie(a, counters, r, c, dr0, dc0);
        // visible counts of the ring slots in this batch (posts p0 .. p1)
        const int p0 = p_open + (a.s_mul ? (int)__umulhi((unsigned)tq, a.s_mul) : tq / a.S);
        const int p1 = p_open + (a.s_mul ? (int)__umulhi((unsigned)(tq + ns - 1), a.s_mul) : (tq + ns - 1) / a.S);
        for (int pp = p0; pp <= p1; ++pp) {
            const int cj = __popc(vism & __ballot_sync(kFull, lane < ns && pj == (pp & (kRing - 1))));
            if (lane == (pp & (kRing - 1))) mycnt += cj;
        }
        tq += ns;
        // posts whose S samples are all tested: write their score, free the slot
        for (; p_open < p_next && a.S <= tq; ++p_open, tq -= a.S) {
            if (lane == (p_open & (kRing - 1))) {
                out[(int64_t)myR * ncols + myC] = (uint8_t)mycnt;
                mycnt = 0;
            }
        }
        // drop the tested samples from the FIFO
        const int rest = qn - ns;
        const int t0 = lane < rest ? s_q[ns + lane] : 0, t1 = lane + 32 < rest ? s_q[ns + lane + 32] : 0;
        __syncwarp();
        if (lane < rest) s_q[lane] = t0;
        if (lane + 32 < rest) s_q[lane + 32] = t1;
        __syncwarp();
        qn = rest;
    };
    const int strip_tiles = a.strip * a.tiles_y;
    for (;;) {
        long long item = 0;
        if (lane == 0) item = (long long)atomicAdd(counters + kVixNext, 1ull);
        item = __shfl_sync(kFull, item, 0);
        const int64_t tile = item / kTileQ;
        if (tile >= (int64_t)a.tiles_x * a.tiles_y) break;
        int ty, tx;
        {
            const int sidx = (int)(tile / strip_tiles), rem = (int)(tile - (int64_t)sidx * strip_tiles);
            const int sw = min(a.strip, a.tiles_x - sidx * a.strip);
            ty = rem / sw;
            tx = sidx * a.strip + (rem - ty * sw);
        }
        const int r = a.row0 + ty * kTileQ + item % kTileQ;
        if (r >= a.row_end) continue;
        // the row's stream seeds (D6) and observer elevations, one post per lane
        // (measured: c3 126.1 -> 113.3 ms; a wash at 32 registers, profiles/README.md)
        uint64_t rseed = 0;
        int rE = 0;
        if (lane < kTileQ && tx * kTileQ + lane < ncols) {
            rseed = mix_seed(a.seed, (uint64_t)r, (uint64_t)(tx * kTileQ + lane));
            rE = zld(z + (int64_t)r * ncols + tx * kTileQ + lane) + a.ht;
        }
        for (int j = 0; j < kTileQ; ++j) {
            const int c = tx * kTileQ + j;
            if (c >= ncols) break;
            if (p_next - p_open == kRing) run_batch(qn);   // ring full (S < 3): drain
            ++n_posts;
            const uint64_t base = __shfl_sync(kFull, rseed, j);
            const int E = __shfl_sync(kFull, rE, j);
            const int slot = p_next & (kRing - 1);
            if (lane == slot) { myE = E; myR = r; myC = c; }
            ++p_next;
            // ---- draw S receivers (D6) into the FIFO ----
            int nacc = 0;
            for (uint32_t k = 0; nacc < a.S; k += 32) {   // draw k + lane of the post's stream
                const int v = (int)fm_mod(a.span, sm_finalize(base + (uint64_t)(k + lane + 1) * kGamma)) - a.R;
                const int dc = __shfl_down_sync(kFull, v, 1);
                const int dr = v;
                const bool ok = !(lane & 1) && dr * dr + dc * dc <= R2 && (unsigned)(r + dr) < (unsigned)nrows &&
                                (unsigned)(c + dc) < (unsigned)ncols;
                const unsigned mask = __ballot_sync(kFull, ok);
                const int take = min(__popc(mask), a.S - nacc);
                if (ok) {
                    const int rank = __popc(mask & ((1u << lane) - 1));
                    if (rank < take) s_q[qn + rank] = (dr + 256) | ((dc + 256) << 9) | (slot << 18);
                }
                nacc += take;
                qn += take;
                __syncwarp();
                if (qn >= 32) run_batch(32);
            }
        }
    }
    while (qn > 0) run_batch(min(qn, 32));
    for (int o = 16; o; o >>= 1) n_cross += __shfl_down_sync(kFull, n_cross, o);
    if (lane == 0 && n_posts) {
        atomicAdd(counters + kVixLos, (unsigned long long)n_posts * a.S);
        atomicAdd(counters + kVixCrossFull, n_cross);
    }
}

// One post per lane (S <= kLaneDrawMaxS, item rows of 32 posts): lane l draws
// its own post's S receivers (D6: pair i of the post's stream is draws 2i,
// 2i+1; rejected pairs are skipped) into column l of the warp's
// [sample][lane] table, then batch k tests sample k of every post -- the
// lanes of a batch are the row's 32 posts, so the observer, its elevation and
// its visible count stay in the lane's registers (no receiver FIFO, no ring of
// open posts, no shuffles per batch).
constexpr int kLaneDrawMaxS = 32;
// P posts per lane (P = 2: the warp takes two item rows; each lane draws its
// first post's S receivers, then its second's, in one loop, so the warp's draw
// iterations are the max over lanes of the two posts' pair counts together --
// less divergence than twice the max of one).
// CC: the crossing statistic compiled in (1), out (0: the cached launches -- the walk geometry is
// then inlined once, not in both forms), or chosen by a.count_cross (-1).
template <int GS, bool MASK, bool LAZY, int P, int CC = -1>
__global__ void __launch_bounds__(kVixThreads, VIX_MINB) k_vix_lanes(const int16_t* __restrict__ z,
                                                                   const uint2* __restrict__ qp, int nrows, int ncols,
                                                                   uint8_t* __restrict__ out, VixArgs a,
                                                                   const uint8_t* __restrict__ gcdt,
                                                                   const int16_t* __restrict__ smap,
                                                                   unsigned long long* __restrict__ counters) {
    static_assert(kTileQ == 32, "one post per lane");
    static_assert(P == 1 || P == 2, "one or two posts per lane");
    extern __shared__ __align__(16) unsigned char s_dyn[];
    // dynamic smem: [geometry: kVixWarps x 32][samples: kVixWarps x P S x 32 ints]
    QuadGeom* s_geo = (QuadGeom*)s_dyn + warp_of_thread() * 32;
    int* s_smp = (int*)((QuadGeom*)s_dyn + kVixWarps * 32) + warp_of_thread() * a.S * 32 * P;
    const uint32_t smp_lane = (uint32_t)__cvta_generic_to_shared(s_smp) + 4u * (threadIdx.x & 31);   // column of this lane
    const QuadPitch PQ{a.pv, a.pt, ncols};
    constexpr bool TERR = GS >= 4;
    const int lane = threadIdx.x & 31;
    __shared__ unsigned long long s_rcp40[256];
    for (int d = threadIdx.x; d < 256; d += blockDim.x) s_rcp40[d] = d ? ((1ull << 40) + d - 1) / d : 0ull;
    __syncthreads();
    const int R2 = a.R * a.R, S = a.S;
    unsigned long long n_cross = 0;
    int n_posts = 0;
    const int strip_tiles = a.strip * a.tiles_y;
    const int64_t ntiles = (int64_t)a.tiles_x * a.tiles_y;
    for (;;) {
        long long item0 = 0;
        if (lane == 0) item0 = (long long)atomicAdd(counters + kVixNext, (unsigned long long)P);
        item0 = __shfl_sync(kFull, item0, 0);
        if (item0 / kTileQ >= ntiles) break;
        int rq[P], cq[P], Eq[P], npq[P];
        bool hq[P];
        uint64_t xq[P];
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const long long item = item0 + q;
            const int64_t tile = item / kTileQ;
            rq[q] = 0; cq[q] = 0; Eq[q] = 0; npq[q] = 0; hq[q] = false; xq[q] = 0;
            if (tile >= ntiles) continue;
            const int sidx = (int)(tile / strip_tiles), rem = (int)(tile - (int64_t)sidx * strip_tiles);
            const int sw = min(a.strip, a.tiles_x - sidx * a.strip);
            const int ty = rem / sw;
            const int tx = sidx * a.strip + (rem - ty * sw);
            const int r = a.row0 + ty * kTileQ + (int)(item % kTileQ);
            if (r >= a.row_end) continue;
            rq[q] = r;
            cq[q] = tx * kTileQ + lane;
            npq[q] = min(32, ncols - tx * kTileQ);   // posts of this item row: lanes 0 .. np-1
            hq[q] = lane < npq[q];
            if (hq[q]) {
                xq[q] = mix_seed(a.seed, (uint64_t)r, (uint64_t)cq[q]);
                Eq[q] = zld(z + (int64_t)r * ncols + cq[q]) + a.ht;
            }
            n_posts += npq[q] * (lane == 0);
        }
        // ---- draw: the lane's posts' S receivers each (D6), rows q S .. q S + S - 1 ----
        {
            int row = hq[0] ? 0 : S;
            const int limit = (P == 2 && hq[P - 1]) ? P * S : (hq[0] ? S : 0);
            uint64_t x = hq[0] ? xq[0] : xq[P - 1];
            int rr = hq[0] ? rq[0] : rq[P - 1], cc = hq[0] ? cq[0] : cq[P - 1];
            while (row < limit) {
                x += kGamma;
                const int dr = small_mod(a.smod, sm_finalize(x)) - a.R;
                x += kGamma;
                const int dc = small_mod(a.smod, sm_finalize(x)) - a.R;
                if (dr * dr + dc * dc <= R2 && (unsigned)(rr + dr) < (unsigned)nrows && (unsigned)(cc + dc) < (unsigned)ncols) {
                    asm volatile("st.shared.u32 [%0], %1;" ::"r"(smp_lane + (uint32_t)row * 128u),
                                 "r"((dr + 256) | ((dc + 256) << 9)));
                    ++row;
                    if (P == 2 && row == S) { x = xq[P - 1]; rr = rq[P - 1]; cc = cq[P - 1]; }   // the second post
                }
            }
        }
        __syncwarp();
        // ---- batch k of post q: sample k of the q-th row's 32 posts ----
#pragma unroll
        for (int q = 0; q < P; ++q) {
            if (npq[q] == 0) continue;   // (warp-uniform)
            const int r = rq[q], c = cq[q], E = Eq[q], np = npq[q];
            const bool has = hq[q];
            int cnt = 0;
            for (int k = 0; k < S; ++k) {
                QuadGeom g{};
                int dr0 = 0, dc0 = 0;
                if (has) {
                    const int pk = s_smp[(q * S + k) * 32 + lane];
                    dr0 = (pk & 0x1ff) - 256;
                    dc0 = ((pk >> 9) & 0x1ff) - 256;
                    if (CC >= 0)
                        g = seg_quad_geom<GS, TERR, !LAZY, CC == 1>(z, qp, ncols, a, gcdt, s_rcp40, r, c, E, dr0, dc0, n_cross);
                    else
                    g = a.count_cross ? seg_quad_geom<GS, TERR, !LAZY, true>(z, qp, ncols, a, gcdt, s_rcp40, r, c, E, dr0, dc0, n_cross)
                                      : seg_quad_geom<GS, TERR, !LAZY, false>(z, qp, ncols, a, gcdt, s_rcp40, r, c, E, dr0, dc0, n_cross);
                }
                unsigned tiem;
                const unsigned vism = batch_skip_lane<GS, TERR, MASK>(g.c, np, lane, s_geo, smap, PQ, &tiem, [&] {
                    if (!LAZY) return g.f;
                    unsigned long long unused = 0;
                    return seg_quad_geom<GS, TERR, true>(z, qp, ncols, a, gcdt, s_rcp40, r, c, E, dr0, dc0, unused).f;
                });
                if ((tiem >> lane) & 1u) push_tie(a, counters, r, c, dr0, dc0);
                cnt += (vism >> lane) & 1u;
            }
            if (has) out[(int64_t)r * ncols + c] = (uint8_t)cnt;
        }
        __syncwarp();
    }
    for (int o = 16; o; o >>= 1) n_cross += __shfl_down_sync(kFull, n_cross, o);
    if (lane == 0 && n_posts) {
        atomicAdd(counters + kVixLos, (unsigned long long)n_posts * a.S);
        atomicAdd(counters + kVixCrossFull, n_cross);
    }
}

// Group-size choice for k_vix_lanes (16- or 32-step skip groups).  32-step groups halve the
// skip tests of a segment, but a failing group costs a serial exact walk, so they pay only
// where nearly every group passes (c4's 46400^2 terrain: VIX 311 -> 263 ms; c3's rougher
// 16384^2: 40 -> 70).  k_vix_sample runs the 32-step test on pseudo-random segments of the
// launch's rows; k_vix_select picks 5 (32 steps) when at most thr/1024 of them have a failing
// group, else 4.  Both kernels are then launched and the one not chosen finds its work counter
// exhausted (k_vix_arm).
__global__ void k_vix_sample(const int16_t* __restrict__ z, int ncols, VixArgs a, const int16_t* __restrict__ smap,
                             unsigned long long* __restrict__ counters, int nsamp) {
    __shared__ unsigned long long s_rcp40[256];
    for (int d = threadIdx.x; d < 256; d += blockDim.x) s_rcp40[d] = d ? ((1ull << 40) + d - 1) / d : 0ull;
    __syncthreads();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    bool counted = false, failed = false;
    if (t < nsamp && a.row_end > a.row0) {
        const uint64_t h = sm_finalize(a.seed ^ ((uint64_t)(t + 1) * kGamma)), h2 = sm_finalize(h + kGamma);
        const int r = a.row0 + (int)((uint32_t)h % (uint32_t)(a.row_end - a.row0)), c = (int)((uint32_t)(h >> 32) % (uint32_t)ncols);
        const int span = 2 * a.R + 1;
        const int dr = (int)((uint32_t)(h2 & 0xffffu) % (uint32_t)span) - a.R, dc = (int)((uint32_t)((h2 >> 16) & 0xffffu) % (uint32_t)span) - a.R;
        if (dr * dr + dc * dc <= a.R * a.R && (dr | dc) != 0 && r + dr >= a.zr0 && r + dr < a.zr1 && (unsigned)(c + dc) < (unsigned)ncols) {
            unsigned long long unused = 0;
            const int E = zld(z + (int64_t)r * ncols + c) + a.ht;
            const QuadGeomC gc = seg_quad_geom<5, true, false, false>(z, nullptr, ncols, a, nullptr, s_rcp40, r, c, E, dr, dc, unused).c;
            const int nM = gc.w & 0xff, ng = nM >= 2 ? (nM + 30) >> 5 : 0;
            const int mag = (unsigned)gc.w >> 15, sp = (gc.w & 0x2000) ? a.pt : a.pv, ssp = (gc.w & 0x4000) ? -sp : sp;
            int acc = mag + (((gc.w >> 8) & 31) << 16), rhs = gc.LE2;
            for (int gi = 0; gi < ng; ++gi) {
                failed |= (int)__ldg(smap + (gc.soff + gi + (acc >> 21) * ssp)) * nM > rhs;
                acc += mag << 5;
                rhs += gc.DG;
            }
            counted = true;
        }
    }
    const unsigned cm = __ballot_sync(0xffffffffu, counted), fm = __ballot_sync(0xffffffffu, failed);
    if ((threadIdx.x & 31) == 0 && cm) {
        atomicAdd(counters + kVixSelTotal, (unsigned long long)__popc(cm));
        if (fm) atomicAdd(counters + kVixSelFail, (unsigned long long)__popc(fm));
    }
}

// the work counter of the next k_vix_lanes launch: 0 when its group size is the chosen one, else past
// every tile, so that its warps leave at their first pull (an early return inside the kernel costs
// the sweep 3 % more instructions: c3 40.6 -> 41.8 ms)
__global__ void k_vix_arm(unsigned long long* __restrict__ counters, int want) {
    counters[kVixNext] = (int)counters[kVixSel] == want ? 0ull : 1ull << 62;
}

__global__ void k_vix_select(unsigned long long* __restrict__ counters, int thr) {
    const unsigned long long fail = counters[kVixSelFail], total = counters[kVixSelTotal];
    counters[kVixSel] = (total >= 1024 && fail * 1024ull <= total * (unsigned long long)thr) ? 5ull : 4ull;
}

// Skip map of the skip tests.  Pass 1: per GxG block the maximum elevation,
// stored with one block of padding on every side (padded index = block + 1;
// padding blocks hold no posts: -32768).  Pass 2: per padded block corner
// (pr, pc) the maximum of blocks pr..pr+1 x pc..pc+1 -- the 2G x 2G posts from
// post (G(pr-1), G(pc-1)) -- written row-major (SV) and column-major (ST) so
// that lanes stepping along a walk's major axis read consecutive entries.
// padded block rows [pr0, pr1) of the (Hb+2) x (Wb+2) block maxima
__global__ void k_blockmax(const int16_t* __restrict__ z, int H, int W, int16_t* __restrict__ bp, int Hb, int Wb, int G,
                           int pr0, int pr1) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + (int64_t)pr0 * (Wb + 2);
    if (idx >= (int64_t)pr1 * (Wb + 2)) return;
    const int pr = (int)(idx / (Wb + 2)), pc = (int)(idx - (int64_t)pr * (Wb + 2));
    const int br = pr - 1, bc = pc - 1;
    int m = -32768;
    if (br >= 0 && br < Hb && bc >= 0 && bc < Wb) {
        for (int y = G * br; y < min(G * br + G, H); ++y)
            for (int x = G * bc; x < min(G * bc + G, W); ++x) m = max(m, (int)z[(int64_t)y * W + x]);
    }
    bp[idx] = (int16_t)m;
}

// padded block rows [pr0, pr1) of the 2G-block maxima from the G-block maxima (2 x 2 blocks each)
__global__ void k_blockmax2(const int16_t* __restrict__ bp, int Hb, int Wb, int16_t* __restrict__ bp2, int Hb2, int Wb2,
                            int pr0, int pr1) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + (int64_t)pr0 * (Wb2 + 2);
    if (idx >= (int64_t)pr1 * (Wb2 + 2)) return;
    const int pr = (int)(idx / (Wb2 + 2)), pc = (int)(idx - (int64_t)pr * (Wb2 + 2));
    const int br2 = pr - 1, bc2 = pc - 1;
    int m = -32768;
    if (br2 >= 0 && br2 < Hb2 && bc2 >= 0 && bc2 < Wb2) {
        for (int br = 2 * br2; br < min(2 * br2 + 2, Hb); ++br)
            for (int bc = 2 * bc2; bc < min(2 * bc2 + 2, Wb); ++bc) m = max(m, (int)bp[(int64_t)(br + 1) * (Wb + 2) + bc + 1]);
    }
    bp2[idx] = (int16_t)m;
}

// block-corner rows [q0, q1) of the skip map (from padded block rows q0 .. q1)
__global__ void k_skipmap(const int16_t* __restrict__ bp, int Hb, int Wb, int16_t* __restrict__ sv, int pv,
                          int16_t* __restrict__ st, int pt, int q0, int q1) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + (int64_t)q0 * (Wb + 1);
    if (idx >= (int64_t)q1 * (Wb + 1)) return;
    const int pr = (int)(idx / (Wb + 1)), pc = (int)(idx - (int64_t)pr * (Wb + 1));
    const int16_t* b = bp + (int64_t)pr * (Wb + 2) + pc;
    const int16_t m = max(max(b[0], b[1]), max(b[Wb + 2], b[Wb + 3]));
    sv[(int64_t)pr * pv + pc] = m;
    st[(int64_t)pc * pt + pr] = m;
}

// column-major copy of the terrain: zt[c*nrows + r] = z[r*ncols + c]
__global__ void k_transpose(const int16_t* __restrict__ z, int16_t* __restrict__ zt, int nrows, int ncols) {
    __shared__ int16_t t[32][33];
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int y = threadIdx.y; y < 32; y += 8) {
        const int r = r0 + y, c = c0 + threadIdx.x;
        if (r < nrows && c < ncols) t[y][threadIdx.x] = z[(int64_t)r * ncols + c];
    }
    __syncthreads();
    for (int x = threadIdx.y; x < 32; x += 8) {
        const int c = c0 + x, r = r0 + threadIdx.x;
        if (r < nrows && c < ncols) zt[(int64_t)c * nrows + r] = t[threadIdx.x][x];
    }
}

// one warp per pair; exact walk, tied segments re-decided in fp64 (fp64 = 1)
__global__ void k_los_batch(const int16_t* __restrict__ z, int nrows, int ncols, const int4* __restrict__ pairs,
                            int64_t n, int ht, int hr, int fp64, uint8_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (w >= n) return;
    const int4 p = pairs[w];
    const int16_t* P = z + (int64_t)p.x * ncols + p.y;
    const int E = zld(P) + ht, Zt = zld(z + (int64_t)p.z * ncols + p.w) + hr;
    const int st = warp_blocked<false, 1>(P, ncols, p.z - p.x, p.w - p.y, E, Zt, lane);
    if (lane == 0) {
        bool blocked = st == 1;
        if (st == 2 && fp64) blocked = seg_blocked_fp64(z, ncols, p.x, p.y, E, Zt, p.z - p.x, p.w - p.y);
        out[w] = blocked ? 0 : 1;
    }
}

}  // namespace

txs_status launch_vix(txs_ctx* c, const txs_params& p) {
    VixArgs a;
    a.R = p.roi; a.ht = p.tx_height; a.hr = p.rx_height; a.S = p.samples_per_point;
    // exact while x S < 2^32 for the x < 16 S + 32 it is applied to; larger S divides
    a.s_mul = a.S > 0 && a.S < 4096 ? (uint32_t)(((1ull << 32) + (uint64_t)a.S - 1) / (uint64_t)a.S) : 0u;
    a.seed = p.seed;
    a.span = make_fastmod((uint64_t)(2 * p.roi + 1));
    a.smod = make_smallmod((uint32_t)(2 * p.roi + 1));
    a.count_cross = 1;   // (d = 0: not usable; k_vix_lanes needs roi <= 255)
    // fp64 tie list (grazing ties: ~1e-4 of segments on the BASELINE terrains);
    // txs_estimate_vix re-runs the stage with a larger list on overflow
    {
        const int64_t los = (c->band_r1 - c->band_r0) * c->ncols * (int64_t)p.samples_per_point;
        const int64_t want = std::max<int64_t>(c->vix_tie_min, std::min<int64_t>(1 << 26, std::max<int64_t>(1 << 20, los / 1024)));
        if (ensure(c, "vix", (void**)&c->d_ties, &c->ties_cap, sizeof(int4) * (size_t)want) != TXS_OK)
            return TXS_ERR_OUT_OF_MEMORY;
        a.ties = c->d_ties;
        a.tie_cap = (long long)(c->ties_cap / sizeof(int4));
        TXS_CUDA(c, "vix", cudaMemsetAsync(c->d_counters + kVixTies, 0, sizeof(unsigned long long), c->stream));
    }
    a.tiles_x = (int)((c->ncols + kTile - 1) / kTile);
    a.tiles_y = (int)((c->band_r1 - c->band_r0 + kTile - 1) / kTile);
    const int tq = kTileQ;   // the quad path's tiles (see path 1 below)
    a.hp = (int)(((c->z_rows + 31) & ~(int64_t)31) + 16);
    a.wp = (int)(((c->ncols + 31) & ~(int64_t)31) + 16);
    // traversal order (measured, profiles/README.md): strips of 16 tile columns
    // at roi 200 (C2 60.2 -> 57.6 ms); row-major at roi 100 (C3: strips raise
    // the L2 hit rate 81 -> 99 % yet run 457 -> 550 ms)
    a.strip = p.roi >= 150 ? 16 : a.tiles_x;
    if (const char* e = getenv("TXS_VIX_STRIP")) a.strip = std::max(1, std::min(a.tiles_x, atoi(e)));
    a.row0 = (int)c->band_r0; a.row_end = (int)c->band_r1;
    a.zr0 = (int)c->z_off; a.zr1 = (int)(c->z_off + c->z_rows);
    const int64_t tiles = a.tiles_x * ((c->band_r1 - c->band_r0 + kTile - 1) / kTile);
    if (tiles > 0x7fffffff) return fail(c, TXS_ERR_RANGE, "vix", "grid too large");
    const int64_t side = kTile + 2 * (int64_t)p.roi;
    const size_t samp = sizeof(int) * (kVixWarps * (size_t)a.S + 4);
    const size_t smem = samp + sizeof(int16_t) * side * side;
    auto go = [&](auto kern, size_t sm) -> txs_status {
        if (sm > 48 * 1024) TXS_CUDA(c, "vix", cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        kern<<<(unsigned)tiles, kVixThreads, sm, c->stream>>>(c->zv(), c->d_zt, (int)c->nrows, (int)c->ncols,
                                                              c->d_vix - c->band_r0 * c->ncols, a, c->d_counters);
        return TXS_OK;
    };
    txs_status st;
    // path (measured on B200, profiles/README.md): the quad planes whenever
    // roi <= 255 (dp2a weight bytes) and their 32 B/post fit in half the free
    // HBM -- they beat the shared-memory tile at roi 100 and the column-major
    // copy at roi 200; else the shared-memory tile when two CTAs fit; else the
    // column-major copy.  TXS_VIX_PATH=smem|pairs|zt overrides (measurement).
    const size_t qbytes = sizeof(uint2) * (size_t)(2 * c->z_rows * (int64_t)a.wp + 2 * c->ncols * (int64_t)a.hp);
    // the free-memory query only when the scratch must grow (it can stall the
    // host inside the timed stage)
    size_t freeb = 0, totalb = 0;
    // (the default roi < 150 kernel walks the terrain and needs only the skip map)
    const bool terr_default = p.roi < 150 && !getenv("TXS_VIX_GROUP") && !getenv("TXS_VIX_SKIP");
    const size_t qneed = terr_default ? 0 : qbytes;
    if (p.roi <= 255 && qneed > c->pairs_cap) cudaMemGetInfo(&freeb, &totalb);
    const bool quads_ok = p.roi <= 255 && (qneed <= c->pairs_cap || qneed <= freeb / 2);
    int path = quads_ok ? 1 : (smem <= 110 * 1024 ? 0 : 2);
    if (const char* e = getenv("TXS_VIX_PATH")) {
        if (!strcmp(e, "smem") && smem <= 200 * 1024) path = 0;
        if (!strcmp(e, "pairs") && p.roi <= 255) path = 1;
        if (!strcmp(e, "zt")) path = 2;
    }
    set_zbounds(c->d_z, c->d_z + c->z_rows * c->ncols, c->stream);
    // an overlapped upload (txs_run_pipeline_host) has a banded form only on the
    // 16-step terrain-walk path; every other path waits for the whole terrain
    if (c->up_pending && path != 1) {
        txs_status w = wait_terrain_rows(c, c->z_rows);
        if (w != TXS_OK) return w;
    }
    if (path == 0) {
        cudaEventRecord(c->ev_k0, c->stream);
        st = go(k_vix<true, 1>, smem);
        cudaEventRecord(c->ev_k1, c->stream);
    } else if (path == 1) {
        const int64_t n = c->z_rows * c->ncols;
        int64_t nq = 2 * c->z_rows * (int64_t)a.wp + 2 * c->ncols * (int64_t)a.hp;
        // skip-test group size G = 2^gs (measured, profiles/README.md): 16 at roi < 150,
        // where the smooth C3/C4 terrain passes 16-step tests 99.97 % of the time
        // (one map load per 16 steps), 4 at roi >= 150 (C2: 59 % of 16-step groups
        // fail, 19 % of 4-step ones); TXS_VIX_GROUP=4|16 overrides
        int gs = p.roi >= 150 ? 2 : 4;
        // k_vix_lanes also has 32-step groups: TXS_VIX_GROUP=32 forces them; by default both
        // the 16- and the 32-step maps are built and k_vix_sample picks per launch (`dual`)
        const bool lanes_ok = p.samples_per_point <= kLaneDrawMaxS && a.smod.d != 0 && !getenv("TXS_VIX_SKIP") &&
                              !getenv("TXS_VIX_LANESKIP") && !getenv("TXS_VIX_LANEDRAW");
        bool dual = gs == 4 && lanes_ok && !getenv("TXS_VIX_GROUP") && !getenv("TXS_VIX_LMODE");
        if (const char* e = getenv("TXS_VIX_DUAL")) dual = dual && atoi(e) != 0;
        if (const char* e = getenv("TXS_VIX_GROUP")) gs = atoi(e) >= 32 && lanes_ok ? 5 : atoi(e) >= 16 ? 4 : 2;
        const int G = 1 << gs;
        // skip map (k_skipmap) behind the quad planes: SV, ST, then the block maxima
        const int Hb = (int)((c->z_rows + G - 1) / G), Wb = (int)((c->ncols + G - 1) / G);
        a.pv = ((Wb + 1) + 7) & ~7;
        a.pt = ((Hb + 1) + 7) & ~7;
        const int64_t nsv = (int64_t)(Hb + 1) * a.pv, nst = (int64_t)(Wb + 1) * a.pt;
        const int64_t nbp = (int64_t)(Hb + 2) * (Wb + 2);
        if (nsv + nst > 0x7fffffff) return fail(c, TXS_ERR_RANGE, "vix", "grid too large");
        a.st_off = (int)nsv;
        // 1: flattened (segment, unit) skip test, 2: per-segment skip test, 0: full walk.
        // Measured (profiles/README.md), ms: C2 55.4 / 45.8 / 48.9, C3 429 / 212 / 313,
        // C4 4273 / 1688 / 2508 (full / flattened / per segment)
        int skip = 1;
        if (a.pv >= 32768 || a.pt >= 32768) skip = 0;   // signed 16-bit map pitches (batch_skip)
        if (const char* e = getenv("TXS_VIX_SKIP")) skip = std::max(0, std::min(2, atoi(e)));
        // the 32-step maps (dual) sit behind the 16-step ones
        constexpr int G2 = 32;
        const int Hb2 = (int)((c->z_rows + G2 - 1) / G2), Wb2 = (int)((c->ncols + G2 - 1) / G2);
        const int pv2 = ((Wb2 + 1) + 7) & ~7, pt2 = ((Hb2 + 1) + 7) & ~7;
        const int64_t nsv2 = (int64_t)(Hb2 + 1) * pv2, nst2 = (int64_t)(Wb2 + 1) * pt2, nbp2 = (int64_t)(Hb2 + 2) * (Wb2 + 2);
        const int64_t n_fine = nsv + nst + nbp;
        dual = dual && skip == 1;
        const size_t map_bytes = skip ? sizeof(int16_t) * (size_t)(n_fine + (dual ? nsv2 + nst2 + nbp2 : 0)) : 0;
        // with 16-step skip groups the flattened kernel walks failing units on the
        // terrain itself: no quad planes (69 GB at C4) and no plane build
        const bool terr = skip == 1 && gs >= 4;
        if (terr) nq = 0;
        // rebuilt on every call (part of the timed stage; ~1 HBM pass of 34 B/post)
        if (ensure(c, "vix", (void**)&c->d_pairs, &c->pairs_cap, sizeof(uint2) * nq + map_bytes) != TXS_OK)
            return TXS_ERR_OUT_OF_MEMORY;
        const bool banded = c->up_pending && terr && !c->sharded;
        if (c->up_pending && !banded) {
            txs_status w = wait_terrain_rows(c, c->z_rows);
            if (w != TXS_OK) return w;
        }
        if (!terr) {
            dim3 tb(32, 8), tg((unsigned)((c->ncols + 31) / 32), (unsigned)((c->z_rows + 31) / 32));
            k_quads<<<tg, tb, 0, c->stream>>>(c->d_z, (uint2*)c->d_pairs, (int)c->z_rows, a.hp, a.wp, (int)c->ncols);
            TXS_LAUNCHED(c, "vix");
        }
        int16_t* smap = skip ? (int16_t*)((uint2*)c->d_pairs + nq) : nullptr;
        // overlapped terrain upload (txs_run_pipeline_host): the map and the walk go
        // band by band behind the arriving rows (16-step terrain walks only)
        int16_t* bp = skip ? smap + nsv + nst : nullptr;
        if (skip && !banded) {
            k_blockmax<<<(unsigned)((nbp + 255) / 256), 256, 0, c->stream>>>(c->d_z, (int)c->z_rows, (int)c->ncols, bp, Hb, Wb, G,
                                                                           0, Hb + 2);
            TXS_LAUNCHED(c, "vix");
            const int64_t ns = (int64_t)(Hb + 1) * (Wb + 1);
            k_skipmap<<<(unsigned)((ns + 255) / 256), 256, 0, c->stream>>>(bp, Hb, Wb, smap, a.pv, smap + nsv, a.pt, 0, Hb + 1);
            TXS_LAUNCHED(c, "vix");
            if (dual) {
                int16_t* smap2 = smap + n_fine;
                int16_t* bp2 = smap2 + nsv2 + nst2;
                k_blockmax2<<<(unsigned)((nbp2 + 255) / 256), 256, 0, c->stream>>>(bp, Hb, Wb, bp2, Hb2, Wb2, 0, Hb2 + 2);
                TXS_LAUNCHED(c, "vix");
                const int64_t ns2 = (int64_t)(Hb2 + 1) * (Wb2 + 1);
                k_skipmap<<<(unsigned)((ns2 + 255) / 256), 256, 0, c->stream>>>(bp2, Hb2, Wb2, smap2, pv2, smap2 + nsv2, pt2, 0,
                                                                               Hb2 + 1);
                TXS_LAUNCHED(c, "vix");
            }
        }
        const uint2* qp = (const uint2*)c->d_pairs;
        set_zbounds(c->d_z, c->d_z + n, c->stream, (const int16_t*)qp, (const int16_t*)(qp + nq));
        size_t qsm = (sizeof(QuadGeom) * 32 + sizeof(int) * (32 + 32 + 64)) * kVixWarps;
        // groups per skip unit (measured, profiles/README.md): 8 at roi 200 (C2 46.6 -> 43.5 ms
        // vs 4), 4 at roi 100 (C3 190.6 -> 180.2 vs 8)
        // G = 16: units of 2 groups (32 steps, TXS_VIX_UNIT=1 for 16)
        int unit = gs >= 4 ? 2 : (p.roi >= 150 ? 8 : 4);
        if (const char* e = getenv("TXS_VIX_UNIT")) unit = atoi(e);
        decltype(&k_vix_quads<1, 8, 2>) kq, kq32 = nullptr;   // kq32: the 32-step kernel of a dual launch
        bool lanes_kernel = false;
        if (skip == 1) {
            // per-lane skip tests (batch_skip_lane); TXS_VIX_LANESKIP=0: flattened units (batch_skip)
            static const bool lane_skip = !getenv("TXS_VIX_LANESKIP") || atoi(getenv("TXS_VIX_LANESKIP")) != 0;
            if (gs >= 4) kq = lane_skip ? k_vix_quads<3, 2, 4> : (unit == 1 ? k_vix_quads<1, 1, 4> : k_vix_quads<1, 2, 4>);
            else kq = lane_skip ? k_vix_quads<3, 8, 2> : (unit == 8 ? k_vix_quads<1, 8, 2> : k_vix_quads<1, 4, 2>);
            // one post per lane (k_vix_lanes) for S <= 32; TXS_VIX_LANEDRAW=0: the per-warp receiver FIFO
            static const bool lane_draw = !getenv("TXS_VIX_LANEDRAW") || atoi(getenv("TXS_VIX_LANEDRAW")) != 0;
            if (lane_skip && lane_draw && p.samples_per_point <= kLaneDrawMaxS && a.smod.d != 0) {
                // failing-group mask vs one flag + cooperative re-test; walk record eager vs
                // built only for failing lanes (TXS_VIX_LMODE = mask | lazy << 1)
                int lm = gs >= 4 ? 3 : 1;   // measured: profiles/README.md (VIX one post per lane)
                if (const char* e = getenv("TXS_VIX_LMODE")) lm = atoi(e) & 3;
                // posts per lane (TXS_VIX_PPL=1|2; measured, profiles/README.md): two on large
                // grids with few samples (c3 41.8 -> 40.2 ms, c4 322 -> 309), one otherwise
                // (c2, S = 20: 32.5 vs 53.6; c1, 1000^2: 1.87 vs 2.03)
                int ppl = p.samples_per_point <= 12 && (double)c->nrows * (double)c->ncols >= (double)(1 << 24) ? 2 : 1;
                if (const char* e = getenv("TXS_VIX_PPL")) ppl = atoi(e) == 2 && p.samples_per_point <= 20 ? 2 : 1;
                if (gs == 5) {   // (failing-group mask + lazy walk record only)
                    kq = ppl == 2 ? k_vix_lanes<5, true, true, 2> : k_vix_lanes<5, true, true, 1>;
                } else if (ppl == 2) {
                    if (gs == 4) kq = lm == 0 ? k_vix_lanes<4, false, false, 2> : lm == 1 ? k_vix_lanes<4, true, false, 2>
                                    : lm == 2 ? k_vix_lanes<4, false, true, 2> : k_vix_lanes<4, true, true, 2>;
                    else kq = lm == 0 ? k_vix_lanes<2, false, false, 2> : lm == 1 ? k_vix_lanes<2, true, false, 2>
                            : lm == 2 ? k_vix_lanes<2, false, true, 2> : k_vix_lanes<2, true, true, 2>;
                } else {
                    if (gs == 4) kq = lm == 0 ? k_vix_lanes<4, false, false, 1> : lm == 1 ? k_vix_lanes<4, true, false, 1>
                                    : lm == 2 ? k_vix_lanes<4, false, true, 1> : k_vix_lanes<4, true, true, 1>;
                    else kq = lm == 0 ? k_vix_lanes<2, false, false, 1> : lm == 1 ? k_vix_lanes<2, true, false, 1>
                            : lm == 2 ? k_vix_lanes<2, false, true, 1> : k_vix_lanes<2, true, true, 1>;
                }
                qsm = (sizeof(QuadGeom) * 32 + sizeof(int) * 32 * (size_t)ppl * (size_t)std::max(1, p.samples_per_point)) *
                      kVixWarps;
                lanes_kernel = true;
                if (dual) kq32 = ppl == 2 ? k_vix_lanes<5, true, true, 2> : k_vix_lanes<5, true, true, 1>;
            }
        } else if (skip == 2) {
            kq = gs == 4 ? k_vix_quads<2, 8, 4> : k_vix_quads<2, 8, 2>;
        } else {
            kq = gs == 4 ? k_vix_quads<0, 8, 4> : k_vix_quads<0, 8, 2>;
        }
        dual = dual && kq32 != nullptr;
        if (qsm > 40 * 1024) {   // (the kernels' static shared memory counts against the default 48 KB)
            TXS_CUDA(c, "vix", cudaFuncSetAttribute(kq, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qsm));
            if (dual) TXS_CUDA(c, "vix", cudaFuncSetAttribute(kq32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qsm));
        }
        if (!c->d_gcd) {
            TXS_CUDA(c, "vix", cudaMalloc((void**)&c->d_gcd, 256 * 256));
            k_gcd_table<<<256, 256, 0, c->stream>>>(c->d_gcd);
            TXS_LAUNCHED(c, "vix");
        }
        VixArgs aq = a;   // the quad path's own (smaller) tiles
        aq.tiles_x = (int)((c->ncols + tq - 1) / tq);
        aq.tiles_y = (int)((c->band_r1 - c->band_r0 + tq - 1) / tq);
        aq.strip = p.roi >= 150 ? 16 : aq.tiles_x;
        if (const char* e = getenv("TXS_VIX_STRIP")) aq.strip = std::max(1, std::min(aq.tiles_x, atoi(e)));
        const int64_t tiles_q = (int64_t)aq.tiles_x * aq.tiles_y;
        if (tiles_q > 0x7fffffff) return fail(c, TXS_ERR_RANGE, "vix", "grid too large");
        // persistent: as many CTAs as are resident (tiles are pulled in a loop)
        int per_sm = 0;
        TXS_CUDA(c, "vix", cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kq, kVixThreads, qsm));
        int64_t grid_q = std::min<int64_t>(tiles_q, (int64_t)std::max(1, per_sm) * c->num_sms);
        if (const char* e = getenv("TXS_VIX_GRID")) grid_q = std::min<int64_t>(tiles_q, std::max(1, atoi(e)));
        // the crossing statistic depends only on this key: counted once (over one launch or
        // the upload bands' launches), then cached
        const uint64_t key = mix_seed(mix_seed(p.seed, (uint64_t)p.roi * 4099 + (uint64_t)p.samples_per_point,
                                               (uint64_t)c->nrows * 1000003 + (uint64_t)c->ncols),
                                      (uint64_t)c->band_r0 * 1000003 + (uint64_t)c->band_r1,
                                      (uint64_t)c->z_off * 1000003 + (uint64_t)c->z_rows);
        const bool lanes = lanes_kernel;
        const bool cached = lanes && c->vix_cross_valid && c->vix_cross_key == key;
        aq.count_cross = cached ? 0 : 1;
        if (lanes) {   // the default forms with the statistic compiled in or out
            auto cc_form = [&](decltype(kq) f) -> decltype(kq) {
                if (f == k_vix_lanes<4, true, true, 2>) return cached ? k_vix_lanes<4, true, true, 2, 0> : k_vix_lanes<4, true, true, 2, 1>;
                if (f == k_vix_lanes<4, true, true, 1>) return cached ? k_vix_lanes<4, true, true, 1, 0> : k_vix_lanes<4, true, true, 1, 1>;
                if (f == k_vix_lanes<5, true, true, 2>) return cached ? k_vix_lanes<5, true, true, 2, 0> : k_vix_lanes<5, true, true, 2, 1>;
                if (f == k_vix_lanes<5, true, true, 1>) return cached ? k_vix_lanes<5, true, true, 1, 0> : k_vix_lanes<5, true, true, 1, 1>;
                return f;
            };
            if (!getenv("TXS_VIX_CCFORM") || atoi(getenv("TXS_VIX_CCFORM")) != 0) {
                kq = cc_form(kq);
                if (kq32) kq32 = cc_form(kq32);
                if (qsm > 40 * 1024) {
                    TXS_CUDA(c, "vix", cudaFuncSetAttribute(kq, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qsm));
                    if (kq32) TXS_CUDA(c, "vix", cudaFuncSetAttribute(kq32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qsm));
                }
                TXS_CUDA(c, "vix", cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kq, kVixThreads, qsm));
                grid_q = std::min<int64_t>(tiles_q, (int64_t)std::max(1, per_sm) * c->num_sms);
                if (const char* e = getenv("TXS_VIX_GRID")) grid_q = std::min<int64_t>(tiles_q, std::max(1, atoi(e)));
            }
        }
        unsigned long long before = 0;
        if (lanes && !cached)
            TXS_CUDA(c, "vix", cudaMemcpyAsync(&before, c->d_counters + kVixCrossFull, sizeof(before),
                                               cudaMemcpyDeviceToHost, c->stream));
        auto finish_cross = [&]() -> txs_status {
            if (cached) {
                k_add_counter<<<1, 1, 0, c->stream>>>(c->d_counters + kVixCrossFull, c->vix_cross_count);
                TXS_LAUNCHED(c, "vix");
            } else if (lanes) {
                unsigned long long after = 0;
                TXS_CUDA(c, "vix", cudaMemcpyAsync(&after, c->d_counters + kVixCrossFull, sizeof(after),
                                                   cudaMemcpyDeviceToHost, c->stream));
                TXS_CUDA(c, "vix", cudaStreamSynchronize(c->stream));
                c->vix_cross_count = after - before;
                c->vix_cross_key = key;
                c->vix_cross_valid = true;
            }
            return TXS_OK;
        };
        // one launch over args' rows; dual: sample the 32-step test on those rows, then both
        // group sizes' kernels, of which the one not chosen returns at once
        int dual_thr = 8;   // of 1024 sampled segments with a failing 32-step group (TXS_VIX_DUAL_THR)
        if (const char* e = getenv("TXS_VIX_DUAL_THR")) dual_thr = std::max(0, atoi(e));
        auto launch_rows = [&](VixArgs args, int64_t grid, uint8_t* out) -> txs_status {
            if (dual) {
                VixArgs a32 = args;
                a32.pv = pv2; a32.pt = pt2; a32.st_off = (int)nsv2;
                const int16_t* smap2 = smap + n_fine;
                constexpr int kSamples = 1 << 16;
                TXS_CUDA(c, "vix", cudaMemsetAsync(c->d_counters + kVixSelFail, 0, 3 * sizeof(unsigned long long), c->stream));
                k_vix_sample<<<kSamples / 256, 256, 0, c->stream>>>(c->zv(), (int)c->ncols, a32, smap2, c->d_counters, kSamples);
                TXS_LAUNCHED(c, "vix");
                k_vix_select<<<1, 1, 0, c->stream>>>(c->d_counters, dual_thr);
                TXS_LAUNCHED(c, "vix");
                if (getenv("TXS_VIX_VERBOSE")) {
                    unsigned long long h[3] = {0, 0, 0};
                    TXS_CUDA(c, "vix", cudaMemcpyAsync(h, c->d_counters + kVixSelFail, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
                    TXS_CUDA(c, "vix", cudaStreamSynchronize(c->stream));
                    fprintf(stderr, "[txs] VIX rows [%d, %d): %llu of %llu sampled segments fail a 32-step group -> %llu-step groups\n",
                            args.row0, args.row_end, h[0], h[1], 1ull << h[2]);
                }
                k_vix_arm<<<1, 1, 0, c->stream>>>(c->d_counters, 4);
                kq<<<(unsigned)grid, kVixThreads, qsm, c->stream>>>(c->zv(), qp, (int)c->nrows, (int)c->ncols, out, args, c->d_gcd,
                                                                   smap, c->d_counters);
                TXS_LAUNCHED(c, "vix");
                k_vix_arm<<<1, 1, 0, c->stream>>>(c->d_counters, 5);
                kq32<<<(unsigned)grid, kVixThreads, qsm, c->stream>>>(c->zv(), qp, (int)c->nrows, (int)c->ncols, out, a32, c->d_gcd,
                                                                     smap2, c->d_counters);
                return TXS_OK;
            }
            TXS_CUDA(c, "vix", cudaMemsetAsync(c->d_counters + kVixNext, 0, sizeof(unsigned long long), c->stream));
            kq<<<(unsigned)grid, kVixThreads, qsm, c->stream>>>(c->zv(), qp, (int)c->nrows, (int)c->ncols, out, args, c->d_gcd, smap,
                                                               c->d_counters);
            return TXS_OK;
        };
        if (!banded) {
            cudaEventRecord(c->ev_k0, c->stream);
            if ((st = launch_rows(aq, grid_q, c->d_vix - c->band_r0 * c->ncols)) != TXS_OK) return st;
            cudaEventRecord(c->ev_k1, c->stream);
            if ((st = finish_cross()) != TXS_OK) return st;
        } else {
            // band b = upload chunk b's rows; it needs the rows up to r1 + R + 4G (its
            // walks, and the map corners of their groups), so it waits for the chunk
            // holding them; block-max rows and map corner rows are built once each, as
            // soon as their terrain rows are in
            const int64_t H = c->z_rows;
            int pr_done = 0, q_done = 0, pr2_done = 0, q2_done = 0;
            const int Gneed = dual ? G2 : G;
            cudaEventRecord(c->ev_k0, c->stream);
            for (size_t b = 0; b < c->up_end.size(); ++b) {
                const int64_t r0 = b ? c->up_end[b - 1] : 0, r1 = c->up_end[b];
                const int64_t need = std::min(H, r1 + p.roi + 4 * (int64_t)Gneed);
                int64_t loaded = H;
                for (size_t k = b; k < c->up_end.size(); ++k)
                    if (c->up_end[k] >= need) { loaded = c->up_end[k]; break; }
                if ((st = wait_terrain_rows(c, need)) != TXS_OK) return st;
                const int pr_new = loaded >= H ? Hb + 2 : (int)(loaded / G) + 1;
                if (pr_new > pr_done) {
                    const int64_t cnt = (int64_t)(pr_new - pr_done) * (Wb + 2);
                    k_blockmax<<<(unsigned)((cnt + 255) / 256), 256, 0, c->stream>>>(c->d_z, (int)H, (int)c->ncols, bp, Hb, Wb,
                                                                                   G, pr_done, pr_new);
                    TXS_LAUNCHED(c, "vix");
                    pr_done = pr_new;
                }
                const int q_new = std::min(Hb + 1, pr_done - 1);
                if (q_new > q_done) {
                    const int64_t cnt = (int64_t)(q_new - q_done) * (Wb + 1);
                    k_skipmap<<<(unsigned)((cnt + 255) / 256), 256, 0, c->stream>>>(bp, Hb, Wb, smap, a.pv, smap + nsv, a.pt,
                                                                                  q_done, q_new);
                    TXS_LAUNCHED(c, "vix");
                    q_done = q_new;
                }
                if (dual) {
                    int16_t* smap2 = smap + n_fine;
                    int16_t* bp2 = smap2 + nsv2 + nst2;
                    const int pr2_new = loaded >= H ? Hb2 + 2 : (int)(loaded / G2) + 1;
                    if (pr2_new > pr2_done) {
                        const int64_t cnt = (int64_t)(pr2_new - pr2_done) * (Wb2 + 2);
                        k_blockmax2<<<(unsigned)((cnt + 255) / 256), 256, 0, c->stream>>>(bp, Hb, Wb, bp2, Hb2, Wb2, pr2_done,
                                                                                        pr2_new);
                        TXS_LAUNCHED(c, "vix");
                        pr2_done = pr2_new;
                    }
                    const int q2_new = std::min(Hb2 + 1, pr2_done - 1);
                    if (q2_new > q2_done) {
                        const int64_t cnt = (int64_t)(q2_new - q2_done) * (Wb2 + 1);
                        k_skipmap<<<(unsigned)((cnt + 255) / 256), 256, 0, c->stream>>>(bp2, Hb2, Wb2, smap2, pv2, smap2 + nsv2, pt2,
                                                                                      q2_done, q2_new);
                        TXS_LAUNCHED(c, "vix");
                        q2_done = q2_new;
                    }
                }
                VixArgs ab = aq;
                ab.row0 = (int)r0; ab.row_end = (int)r1;
                ab.tiles_y = (int)((r1 - r0 + tq - 1) / tq);
                const int64_t tb = (int64_t)ab.tiles_x * ab.tiles_y;
                const int64_t gb = std::min<int64_t>(tb, (int64_t)std::max(1, per_sm) * c->num_sms);
                if ((st = launch_rows(ab, gb, c->d_vix)) != TXS_OK) return st;
                TXS_LAUNCHED(c, "vix");
            }
            cudaEventRecord(c->ev_k1, c->stream);
            if ((st = finish_cross()) != TXS_OK) return st;
        }
        st = TXS_OK;
    } else {
        if (ensure(c, "vix", (void**)&c->d_zt, &c->zt_cap, sizeof(int16_t) * c->z_rows * c->ncols) != TXS_OK)
            return TXS_ERR_OUT_OF_MEMORY;
        {
            dim3 tb(32, 8), tg((unsigned)((c->ncols + 31) / 32), (unsigned)((c->z_rows + 31) / 32));
            k_transpose<<<tg, tb, 0, c->stream>>>(c->d_z, c->d_zt, (int)c->z_rows, (int)c->ncols);
            TXS_LAUNCHED(c, "vix");
        }
        set_zbounds(c->d_z, c->d_z + c->z_rows * c->ncols, c->stream, c->d_zt, c->d_zt + c->z_rows * c->ncols);
        cudaEventRecord(c->ev_k0, c->stream);
        st = go(k_vix<false, 1>, samp);
        cudaEventRecord(c->ev_k1, c->stream);
    }
    if (st != TXS_OK) return st;
    TXS_LAUNCHED(c, "vix");
    if (p.los_arith == TXS_LOS_FP64) {   // re-decide the tied segments in fp64
        k_vix_fp64_ties<<<(unsigned)(c->num_sms * 4), 256, 0, c->stream>>>(c->zv(), c->ncols, c->d_ties, c->d_counters,
                                                                          a.tie_cap, p.tx_height, p.rx_height,
                                                                          c->d_vix - c->band_r0 * c->ncols);
        TXS_LAUNCHED(c, "vix");
    }
    return TXS_OK;
}

txs_status launch_los_batch(txs_ctx* c, const int32_t* d_pairs, int64_t n, int32_t ht, int32_t hr, int32_t arith,
                            uint8_t* d_out) {
    const int64_t threads = n * 32;
    const unsigned blocks = (unsigned)((threads + 255) / 256);
    set_zbounds(c->d_z, c->d_z + c->z_rows * c->ncols, c->stream);
    k_los_batch<<<blocks, 256, 0, c->stream>>>(c->zv(), (int)c->nrows, (int)c->ncols, (const int4*)d_pairs, n, ht, hr,
                                                 arith == TXS_LOS_FP64 ? 1 : 0, d_out);
    TXS_LAUNCHED(c, "los");
    return TXS_OK;
}

}  // namespace txs
