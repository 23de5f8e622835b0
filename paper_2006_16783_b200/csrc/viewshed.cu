// VIEWSHED stage (compute_viewshed / compute_all_viewsheds)
// — R2 radial sweep, decision D5.
//
// One CTA per observer; thread t walks rays t, t+T, ... of the frozen ray
// template (raytemplate.cpp), so the 32 lanes of a warp walk 32 neighbouring
// rays and their terrain reads land in the same few L1 lines.  Along a ray
// (primitive direction (p,q), u = parameter, crossing row line i at u = i/|p|)
// each terrain crossing contributes the tangent N/M = (z - E)/u as an exact
// rational (N = z*|p| - E*|p| with z*|p| the integer interpolation, M = i);
// the horizon is their running max (compared by cross-multiplication in
// int64), and an owned cell (a,b) with projection u_c = dot/L2 is visible iff
//     P * L2 * M_h  >=  N_h * dot        (P = z_cell + h_r - E)
// i.e. its receiver tangent is >= the horizon of the crossings with u < u_c
// (">= the running horizon angle", SPEC.md:321 tangent, SPEC.md:324
// horizon from bare terrain).  Crossings needing an off-grid post end the ray
// (the in-grid crossings of a ray are a prefix).  Bits: window row-major,
// LSB-first in u64 words (decision D8), accumulated in shared memory.
#include <cub/cub.cuh>

#include <cstdlib>

#include "ctx.hpp"

namespace txs {
namespace {

struct VsArgs {
    int nrows, ncols, R, ht, hr, nrays;
    int64_t stride;       // u64 words per viewshed slot
    const int32_t* perm;  // processing order (spatially sorted), or null
    int64_t n;            // observers
    int sbits;            // smem bitmap u32 words per observer: (2R+1) rows x (2*Wmax+1) (odd pitch)
    long long tmpl_cross, tmpl_cells;   // template crossings / cells (interior observers)
    const uint32_t* pairs;  // pair planes of the held rows (interior K-observer path), or null
    int p2, pw;             // pair-plane row pitch (words, 2*pw) and posts per plane row
    int zoff;               // first held terrain row
    int2* ties;             // fp64 tie list: {candidate, ray} with a cell whose tangent equals the horizon
    long long tie_cap;
};

// A cell's receiver tangent EQUALS its horizon (an exact grazing tie, which
// fp64 rounding decides either way): the observer's ray goes to the fp64 tie
// list (k_vs_fp64_ties).  The sweeps flag candidates by the low 32 bits of the
// two cross products -- a superset of the exact ties (the re-test recomputes
// the whole ray, so a false positive costs time, not bits).
__device__ __forceinline__ void push_vs_tie(const VsArgs& a, unsigned long long* counters, int64_t cand, int ray) {
    const unsigned long long k = atomicAdd(counters + kVsTies, 1ull);
    if ((long long)k < a.tie_cap) a.ties[k] = make_int2((int)cand, ray);
}

// Pair planes for the interior K-observer sweep: held row y occupies p2 = 2*pw
// words, (H, V) interleaved per post (word 2x + 1 for a column crossing, so an
// event's pair offset is dr*p2 + 2*dc + col), H[x] = z(y,x) | z(y,x+1) << 16 and
// V[x] = z(y,x) | z(y+1,x) << 16 (0 past the last column / held row).  A grid
// crossing interpolates between exactly such a pair, so one 32-bit load and one
// dp2a (signed 16-bit halves x unsigned weight bytes, exact) replace two
// 16-bit loads and two multiplies; for a ray stepping to -col (-row) the pair
// one post back is read and the weight bytes are swapped.
__global__ void k_vs_pairs(const int16_t* __restrict__ z, uint32_t* __restrict__ out, int H, int ncols, int pw) {
    const int64_t total = (int64_t)H * pw;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int y = (int)(t / pw), x = (int)(t - (int64_t)y * pw);
        uint32_t hv = 0, vv = 0;
        if (x < ncols) {
            const int16_t* zr = z + (int64_t)y * ncols;
            const uint32_t a = (uint16_t)zr[x];
            hv = a | ((x + 1 < ncols ? (uint32_t)(uint16_t)zr[x + 1] : 0u) << 16);
            vv = a | ((y + 1 < H ? (uint32_t)(uint16_t)zr[x + ncols] : 0u) << 16);
        }
        uint32_t* row = out + (int64_t)y * 2 * pw;
        reinterpret_cast<uint2*>(row)[x] = make_uint2(hv, vv);   // interleaved: (H, V) per post
    }
}

// the same planes, four posts per thread (ncols % 4 == 0: 8-byte terrain loads, two 16-byte stores)
__global__ void k_vs_pairs4(const int16_t* __restrict__ z, uint32_t* __restrict__ out, int H, int ncols, int pw) {
    const int q = pw >> 2;   // groups of four posts per plane row (pw is a multiple of 16)
    const int64_t total = (int64_t)H * q;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int y = (int)(t / q), x = (int)(t - (int64_t)y * q) << 2;
        uint4 lo = make_uint4(0u, 0u, 0u, 0u), hi = lo;
        if (x < ncols) {
            const int16_t* zr = z + (int64_t)y * ncols + x;
            const uint2 a = __ldg(reinterpret_cast<const uint2*>(zr));   // posts x .. x+3 as 16-bit halves
            const uint2 b = y + 1 < H ? __ldg(reinterpret_cast<const uint2*>(zr + ncols)) : make_uint2(0u, 0u);
            const uint32_t nx = x + 4 < ncols ? (uint32_t)(uint16_t)__ldg(zr + 4) : 0u;
            const uint32_t z0 = a.x & 0xffffu, z1 = a.x >> 16, z2 = a.y & 0xffffu, z3 = a.y >> 16;
            lo = make_uint4(a.x, z0 | (b.x << 16), z1 | (z2 << 16), z1 | (b.x & 0xffff0000u));
            hi = make_uint4(a.y, z2 | (b.y << 16), z3 | (nx << 16), z3 | (b.y & 0xffff0000u));
        }
        uint4* row = reinterpret_cast<uint4*>(out + (int64_t)y * 2 * pw + 2 * x);
        row[0] = lo;
        row[1] = hi;
    }
}

__device__ __forceinline__ uint32_t vs_pld(const uint32_t* p) {
#ifdef TXS_BOUNDS_CHECK
    const int16_t* q = (const int16_t*)p;
    if (q < g_zb.lo2 || q + 1 >= g_zb.hi2) __trap();
#endif
    return __ldg(p);
}

// s_bits[word] |= bit when pred (predicated, no branch; 32-bit shared address)
__device__ __forceinline__ void red_or_shared(uint32_t saddr, uint32_t bit, bool pred) {
    asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p red.shared.or.b32 [%0], %1;\n}\n" ::"r"(saddr), "r"(bit),
                 "r"((uint32_t)pred)
                 : "memory");
}

// signed 32x32 -> 64-bit product in one IMAD.WIDE
__device__ __forceinline__ long long mulw(int a, int b) {
    long long d;
    asm("mul.wide.s32 %0, %1, %2;" : "=l"(d) : "r"(a), "r"(b));
    return d;
}

__device__ __forceinline__ int vs_dp2(uint32_t pair, uint32_t w) {
    int d;
    asm("dp2a.lo.s32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(pair), "r"(w), "r"(0));
    return d;
}

// Aligned output word b of window row y, gathered from the window-dense smem
// bitmap (row-major h x w bits): the smem copy stays compact (3 CTAs/SM at
// R=250) and the cum-aligned layout is produced on the way out.
__device__ __forceinline__ uint64_t aligned_word_from_dense(const uint32_t* sb, int y, int b, int col0, int w) {
    const int base = col0 & ~63;
    const int cl = max(col0, base + 64 * b), ch = min(col0 + w - 1, base + 64 * b + 63);
    if (cl > ch) return 0ull;
    const int off = y * w + (cl - col0), len = ch - cl + 1;
    const int w0 = off >> 5, sh = off & 31;
    const uint64_t lo = (uint64_t)sb[w0] | ((uint64_t)sb[w0 + 1] << 32);
    uint64_t seg = lo >> sh;
    if (sh) seg |= (uint64_t)sb[w0 + 2] << (64 - sh);
    if (len < 64) seg &= (1ull << len) - 1;
    return seg << (cl - base - 64 * b);
}

template <bool SMEM_BITS>
__global__ void k_viewshed(const int16_t* __restrict__ z, const int32_t* __restrict__ crow,
                           const int32_t* __restrict__ ccol, const int4* __restrict__ rays,
                           const uint32_t* __restrict__ cells, VsArgs a, uint64_t* __restrict__ words,
                           int4* __restrict__ wins, int32_t* __restrict__ pops,
                           unsigned long long* __restrict__ counters) {
    extern __shared__ __align__(16) uint32_t s_bits[];
    __shared__ int s_red[32];
    const int64_t cand = a.perm ? a.perm[blockIdx.x] : blockIdx.x;
    const int r = crow[cand], c = ccol[cand];
    const int row0 = max(0, r - a.R), col0 = max(0, c - a.R);
    const int h = min(a.nrows - 1, r + a.R) - row0 + 1, w = min(a.ncols - 1, c + a.R) - col0 + 1;
    // smem: window-dense bits (RS = w); global: cum-aligned rows (RS = nwr*64)
    const int nwr = win_nwr(col0, w);
    const int abase = SMEM_BITS ? col0 : (col0 & ~63);
    const int RS = SMEM_BITS ? w : nwr << 6;
    const int nw64 = h * nwr;
    uint64_t* out = words + cand * a.stride;
    if (SMEM_BITS) {
        for (int i = threadIdx.x; i < (h * w + 31) / 32 + 3; i += blockDim.x) s_bits[i] = 0u;
        __syncthreads();
    }
    auto set_bit = [&](int k) {
        if (SMEM_BITS) atomicOr(&s_bits[k >> 5], 1u << (k & 31));
        else atomicOr((unsigned long long*)&out[k >> 6], 1ull << (k & 63));
    };
    auto Z = [&](int rr, int cc) -> int { return zld(z + (int64_t)rr * a.ncols + cc); };
    const int E = Z(r, c) + a.ht;
    unsigned long long n_cross = 0, n_cells = 0;

    for (int ray = threadIdx.x; ray < a.nrays; ray += blockDim.x) {
        const int4 rd = __ldg(rays + ray);
        const int p = rd.x, q = rd.y, cb = rd.z, cnt = rd.w;
        const int ap = abs(p), aq = abs(q), sp = p >= 0 ? 1 : -1, sq = q >= 0 ? 1 : -1;
        const int L2 = p * p + q * q;
        // row crossing i: column offset i*aq/ap = qr + mr/ap ; column crossing j: row offset qc + mc/aq
        const int dqr = ap ? aq / ap : 0, dmr = ap ? aq % ap : 0;
        const int dqc = aq ? ap / aq : 0, dmc = aq ? ap % aq : 0;
        int i = 1, j = 1, qr = dqr, mr = dmr, qc = dqc, mc = dmc;
        bool has = false, alive = true, tied = false;
        int NH = 0, MH = 1;
        for (int k = 0; k < cnt; ++k) {
            const uint32_t cell = __ldg(cells + cb + k);
            const int ca = (int)(int16_t)(cell & 0xffffu), cbb = (int)(int16_t)(cell >> 16);
            const int dot = ca * p + cbb * q;
            while (alive) {
                bool isrow, iscol;
                if (ap == 0) { isrow = false; iscol = true; }
                else if (aq == 0) { isrow = true; iscol = false; }
                else {
                    const int cmp = i * aq - j * ap;
                    isrow = cmp <= 0; iscol = cmp >= 0;
                }
                const int idx = isrow ? i : j, n = isrow ? ap : aq;
                if ((long long)idx * L2 >= (long long)dot * n) break;   // u_k >= u_c
                int zn;
                if (isrow && iscol) {   // through a post
                    const int rr = r + sp * i, cc = c + sq * j;
                    if (rr < 0 || rr >= a.nrows || cc < 0 || cc >= a.ncols) { alive = false; break; }
                    zn = Z(rr, cc) * n;
                } else if (isrow) {
                    const int rr = r + sp * i, c0 = c + sq * qr;
                    if (rr < 0 || rr >= a.nrows || c0 < 0 || c0 >= a.ncols) { alive = false; break; }
                    zn = Z(rr, c0) * (n - mr);
                    if (mr) {
                        const int c1 = c0 + sq;
                        if (c1 < 0 || c1 >= a.ncols) { alive = false; break; }
                        zn += Z(rr, c1) * mr;
                    }
                } else {
                    const int cc = c + sq * j, r0 = r + sp * qc;
                    if (cc < 0 || cc >= a.ncols || r0 < 0 || r0 >= a.nrows) { alive = false; break; }
                    zn = Z(r0, cc) * (n - mc);
                    if (mc) {
                        const int r1 = r0 + sp;
                        if (r1 < 0 || r1 >= a.nrows) { alive = false; break; }
                        zn += Z(r1, cc) * mc;
                    }
                }
                const int N = zn - E * n;
                if (!has || (long long)N * MH > (long long)NH * idx) { has = true; NH = N; MH = idx; }
                ++n_cross;
                if (isrow) { ++i; qr += dqr; mr += dmr; if (mr >= ap) { mr -= ap; ++qr; } }
                if (iscol) { ++j; qc += dqc; mc += dmc; if (mc >= aq) { mc -= aq; ++qc; } }
            }
            const int rr = r + ca, cc = c + cbb;
            if (rr < 0 || rr >= a.nrows || cc < 0 || cc >= a.ncols) continue;
            ++n_cells;
            const int P = Z(rr, cc) + a.hr - E;
            const long long lhs = (long long)P * L2 * MH, rhs = (long long)NH * dot;
            if (!has || lhs >= rhs)
                set_bit((rr - row0) * RS + (cc - abase));
            tied |= has && lhs == rhs;
        }
        if (tied) push_vs_tie(a, counters, cand, ray);
    }
    if (threadIdx.x == 0) set_bit((r - row0) * RS + (c - abase));
    __syncthreads();
    int pc = 0;
    for (int i = threadIdx.x; i < nw64; i += blockDim.x) {
        uint64_t v;
        if (SMEM_BITS) {
            const int y = i / nwr;
            v = aligned_word_from_dense(s_bits, y, i - y * nwr, col0, w);
            out[i] = v;
        } else {
            v = out[i];
        }
        pc += __popcll(v);
    }
    // block reductions: popcount and counters
    for (int o = 16; o; o >>= 1) {
        pc += __shfl_down_sync(0xffffffffu, pc, o);
        n_cross += __shfl_down_sync(0xffffffffu, n_cross, o);
        n_cells += __shfl_down_sync(0xffffffffu, n_cells, o);
    }
    if ((threadIdx.x & 31) == 0) {
        s_red[threadIdx.x >> 5] = pc;
        atomicAdd(counters + kVsCross, n_cross);
        atomicAdd(counters + kVsCells, n_cells);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int k = 0; k < (int)((blockDim.x + 31) >> 5); ++k) t += s_red[k];
        pops[cand] = t;
        wins[cand] = make_int4(row0, col0, h, w);
    }
}

// Event-stream variant (roi <= kEvMaxRoi): the merged per-ray events of the
// template are read [step][lane] (one coalesced 8-byte-per-lane load per warp
// step) and every event — row/column/post crossing or owned cell — goes
// through the same branch-free arithmetic with one value v = z0*(n-m) + z1*m:
//   crossing:  X = v - E*n,        M = y (line index)     horizon candidate X/M
//   cell:      X = z + h_r - E,    M = L2*MH, y = dot      receiver tangent test
// and one pair of 32x32->64-bit products X*M vs NH*y against the horizon
// NH/MH (cells: P*L2*MH >= NH*dot, crossings: N*MH > NH*M).  Lanes of a warp
// are 32 neighbouring rays; the CTA's warps stride over the ray groups.
constexpr int kVsUnroll = 4;

template <bool INTERIOR>
__device__ __forceinline__ void vs_events(const int16_t* __restrict__ z, int r, int c, int E, int row0, int abase, int RS,
                                          const VsArgs& a, const int4* __restrict__ rays,
                                          const int2* __restrict__ groups, const uint2* __restrict__ events,
                                          int ngroups, uint32_t* s_bits, uint64_t* gout, bool smem_bits,
                                          unsigned long long& n_cross, unsigned long long& n_cells, int64_t cand,
                                          unsigned long long* counters) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int16_t* __restrict__ P = z + (int64_t)r * a.ncols + c;
    const int Ehr = E - a.hr;
    // cell (r+dr, c+dc) -> aligned bit (r+dr-row0)*RS + (c+dc-abase) = dr*RS + dc + K0
    const int K0 = (r - row0) * RS + (c - abase);
    for (int g = warp; g < ngroups; g += nwarps) {
        const int2 grp = __ldg(groups + g);
        const int ray = g * 32 + lane;
        int p = 0, q = 0;
        if (ray < a.nrays) { const int4 rd = __ldg(rays + ray); p = rd.x; q = rd.y; }
        const int L2 = p * p + q * q;
        bool has = false, alive = true, tied = false;
        int NH = 0, MH = 1, L2MH = L2;
        const uint2* ev = events + (int64_t)grp.x * 32 + lane;
        for (int st0 = 0; st0 < grp.y; st0 += kVsUnroll) {
            uint2 ee[kVsUnroll];
            int z0[kVsUnroll], z1[kVsUnroll], kb[kVsUnroll];
            bool ok[kVsUnroll];
#pragma unroll
            for (int u = 0; u < kVsUnroll; ++u)
                ee[u] = st0 + u < grp.y ? __ldg(ev + (int64_t)(st0 + u) * 32) : make_uint2((uint32_t)kEvNop, 0u);
#pragma unroll
            for (int u = 0; u < kVsUnroll; ++u) {
                const uint32_t e = ee[u].x, type = e & 7u;
                const int dr = ((int)(e << 20)) >> 23, F = ((int)(e << 10)) >> 22, dc = F >> 1;
                const bool isrow = type == kEvRow, iscol = type == kEvCol;
                bool inb = type != kEvNop;
                if (!INTERIOR) {   // both interpolation posts in the grid
                    const int rr = r + dr, cc = c + dc;
                    const int r1 = rr + (iscol ? 1 : 0), c1 = cc + (isrow ? 1 : 0);
                    inb = inb && rr >= 0 && rr < a.nrows && cc >= 0 && cc < a.ncols && r1 >= 0 && r1 < a.nrows &&
                          c1 >= 0 && c1 < a.ncols;
                }
                kb[u] = dr * RS + dc + K0;
                const int off0 = inb ? dr * a.ncols + dc : 0;
                const int off1 = inb ? off0 + (iscol ? a.ncols : (isrow ? 1 : 0)) : 0;
                z0[u] = zld(P + off0);
                z1[u] = zld(P + off1);
                ok[u] = inb;
            }
#pragma unroll
            for (int u = 0; u < kVsUnroll; ++u) {
                const uint32_t e = ee[u].x, type = e & 7u;
                const int y = (int)(ee[u].y & 0xffffffu);
                const int w0 = (int)(e >> 24), w1 = (int)(ee[u].y >> 24);
                const bool iscell = type == kEvCell, iscross = type <= kEvPost;
                const int v = z0[u] * w0 + z1[u] * w1;
                const int X = v - (iscell ? Ehr : (w0 + w1) * E);
                const long long lhs = (long long)X * (iscell ? L2MH : MH);
                const long long rhs = (long long)NH * y;
                if (iscross) {
                    if (!ok[u]) alive = false;
                    else if (alive) {
                        ++n_cross;
                        if (!has || lhs > rhs) { has = true; NH = X; MH = y; L2MH = L2 * y; }
                    }
                } else if (iscell && ok[u]) {
                    ++n_cells;
                    if (!has || lhs >= rhs) {
                        const int k = kb[u];
                        if (smem_bits) atomicOr(&s_bits[k >> 5], 1u << (k & 31));
                        else atomicOr((unsigned long long*)&gout[k >> 6], 1ull << (k & 63));
                    }
                    tied |= has && lhs == rhs;
                }
            }
        }
        if (tied) push_vs_tie(a, counters, cand, ray);
    }
}


// Interior fast path for K observers per CTA: each warp walks its ray group
// once, the event load/decode/offsets are shared and every observer keeps its
// own horizon (NH, MH) and bitmap — K independent dependency chains per lane.
// Interior observers have every post in the grid and an unclipped window, so
// no bounds tests and no counting (the template's totals are added instead).
//
// EDGE: the same sweep for CTAs holding observers near the grid edge (clipped
// windows): per observer, an event counts only if its posts are in the grid
// (a crossing that needs an off-grid post ends that observer's ray, cells
// outside the grid are skipped -- the rules of vs_events<false>), the cell bit
// uses the observer's own window pitch and origin, and the crossings / cells
// actually evaluated are counted.
//
// STEP: events per sweep iteration (event groups are padded to a multiple of 4
// steps, raytemplate.cpp) -- 4 at roi >= 225 (C5 1151 -> 1099 ms), 2 elsewhere
// (C3 20.9 vs 23.5 ms at 4; profiles/README.md)
template <int K, bool PAIRS, bool EDGE, int STEP>
__device__ __forceinline__ void vs_events_k(const int16_t* __restrict__ z, const int* rk, const int* ck, const int* Ek,
                                            const int* RSk, const int* K0k,
                                            const VsArgs& a, const int4* __restrict__ rays,
                                            const int2* __restrict__ groups, const uint2* __restrict__ events,
                                            int ngroups, uint32_t* s_bits, int bits_stride,
                                            unsigned long long& n_cross, unsigned long long& n_cells,
                                            unsigned long long* counters) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const uint32_t* __restrict__ B[K];   // PAIRS: the observer's word in the pair planes
    const int16_t* __restrict__ P[K];    // else: the observer's post
    int Ehr[K];
    uint32_t sb[K];                      // shared byte address of bitmap k
    const int RS0 = RSk[0], K00 = K0k[0];   // identical for every interior observer
    const int p2 = a.p2;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        if (PAIRS) {
            // (threadIdx.x >> 10) == 0 but not provably so: B lives in per-thread
            // registers, and B + off becomes one IMAD.WIDE instead of a 64-bit add chain
            B[k] = a.pairs + (int64_t)(rk[k] - a.zoff) * a.p2 + 2 * ck[k] + (threadIdx.x >> 10);
            asm("mov.b64 %0, %0;" : "+l"(B[k]));
        } else {
            P[k] = z + (int64_t)rk[k] * a.ncols + ck[k];
        }
        Ehr[k] = Ek[k] - a.hr;
        sb[k] = (uint32_t)__cvta_generic_to_shared(s_bits + k * bits_stride);
    }
    for (int g = warp; g < ngroups; g += nwarps) {
        const int2 grp = __ldg(groups + g);
        const int ray = g * 32 + lane;
        int p = 0, q = 0;
        if (ray < a.nrays) { const int4 rd = __ldg(rays + ray); p = rd.x; q = rd.y; }
        const int L2 = p * p + q * q;
        // horizon NH/MH, starting at a sentinel below every real tangent: any
        // crossing replaces it and every cell before the first crossing is
        // visible.  Exact for int16 terrain, heights <= 32767 (txs_params
        // check) and roi <= 250: a crossing's |X| <= 98302*255 < 2^30 <= 2^30*M,
        // a cell's |X|*L2 <= 98302*L2 < 2^30*dot (an owned cell lies ahead of
        // its ray: dot >= 0.7*|(p,q)|, and |(p,q)| <= 354)
        int NH[K], MH[K], L2MH[K];
        bool alive[K];
        uint32_t tied = 0;   // bit k: observer k met a cell whose tangent may equal its horizon
#pragma unroll
        for (int k = 0; k < K; ++k) { NH[k] = -(1 << 30); MH[k] = 1; L2MH[k] = L2; alive[k] = true; }
        const uint2* ev = events + (int64_t)grp.x * 32 + lane;
        for (int st0 = 0; st0 < grp.y; st0 += STEP, ev += 32 * STEP) {
            uint2 ee[STEP];
            uint32_t pr[STEP][K];
            int z0[STEP][K], z1[STEP][K];
            int dru[STEP], dcu[STEP];
            bool ok[STEP][K];
#pragma unroll
            for (int u = 0; u < STEP; ++u) {
                ee[u] = __ldg(ev + u * 32);   // groups hold an even number of steps
                const uint32_t e = ee[u].x, type = e & 7u;
                const int dr = ((int)(e << 20)) >> 23, F = ((int)(e << 10)) >> 22, dc = F >> 1;
                const bool isrow = type == kEvRow, iscol = type == kEvCol;
                dru[u] = dr; dcu[u] = F;   // dc = F >> 1
#pragma unroll
                for (int k = 0; k < K; ++k) {   // both interpolation posts (or the cell) in the grid
                    ok[u][k] = !EDGE || (type != kEvNop && (unsigned)(rk[k] + dr) < (unsigned)(a.nrows - (iscol ? 1 : 0)) &&
                                         (unsigned)(ck[k] + dc) < (unsigned)(a.ncols - (isrow ? 1 : 0)));
                }
                if (PAIRS) {   // the first post's H pair (its right neighbour) or, column crossing, V pair
                    const int off = dr * p2 + F;   // F = 2*dc + iscol; Nop events carry dr = F = 0
#pragma unroll
                    for (int k = 0; k < K; ++k) pr[u][k] = (!EDGE || ok[u][k]) ? vs_pld(B[k] + off) : 0u;
                } else {
                    const int off0 = type != kEvNop ? dr * a.ncols + dc : 0;
                    const int off1 = off0 + (iscol ? a.ncols : (isrow ? 1 : 0));
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        z0[u][k] = (!EDGE || ok[u][k]) ? zld(P[k] + off0) : 0;
                        z1[u][k] = (!EDGE || ok[u][k]) ? zld(P[k] + off1) : 0;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < STEP; ++u) {
                const uint32_t e = ee[u].x, type = e & 7u;
                const int y = (int)(ee[u].y & 0xffffffu);
                const uint32_t W = __byte_perm(e, ee[u].y, 0x73u);   // w0 | w1 << 8
                const int w0 = (int)(W & 0xffu), w1 = (int)((W >> 8) & 0xffu), n = w0 + w1;
                const bool iscell = type == kEvCell, iscross = type <= kEvPost;
                // interior observers share the window geometry (pitch 2R+1, origin
                // bit R*(2R+1)+R): the cell's word and bit are observer-independent
                const int kk = dru[u] * RS0 + (dcu[u] >> 1) + K00;
                const uint32_t cw4 = (uint32_t)(kk >> 5) << 2, cbit = 1u << (kk & 31);
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int v = PAIRS ? vs_dp2(pr[u][k], W) : z0[u][k] * w0 + z1[u][k] * w1;
                    const int X = v - (iscell ? Ehr[k] : n * Ek[k]);
                    const long long lhs = mulw(X, iscell ? L2MH[k] : MH[k]);
                    const long long rhs = mulw(NH[k], y);
                    bool upc = iscross, setc = iscell;
                    if (EDGE) {
                        if (iscross && !ok[u][k]) alive[k] = false;   // the ray needs an off-grid post: it ends
                        upc = iscross && alive[k];
                        setc = iscell && ok[u][k];
                        n_cross += upc;
                        n_cells += setc;
                    }
                    const bool up = upc & (lhs > rhs);
                    NH[k] = up ? X : NH[k];
                    MH[k] = up ? y : MH[k];
                    L2MH[k] = up ? L2 * y : L2MH[k];
                    if (EDGE) {
                        const int kb = dru[u] * RSk[k] + (dcu[u] >> 1) + K0k[k];
                        red_or_shared(sb[k] + ((uint32_t)(kb >> 5) << 2), 1u << (kb & 31), setc & (lhs >= rhs));
                    } else {
                        red_or_shared(sb[k] + cw4, cbit, setc & (lhs >= rhs));
                    }
                    tied |= (uint32_t)(setc & ((uint32_t)lhs == (uint32_t)rhs)) << k;
                }
            }
        }
        if (tied) {
#pragma unroll
            for (int k = 0; k < K; ++k)
                if ((tied >> k) & 1u) {   // observer k of this CTA (k_viewshed_evk's slot order)
                    const int64_t slot = (int64_t)blockIdx.x * K + k;
                    push_vs_tie(a, counters, a.perm ? a.perm[slot] : slot, g * 32 + lane);
                }
        }
    }
}

// Interior K-observer sweep on the interior event encoding (events3,
// raytemplate.cpp pack_ev3): per event one shared decode -- pair offset
// dr*p2 + F, weight word W, denominator n = w0 + w1 (a dp2a of W with
// (1, 1)), the receiver-height term, the cell's bitmap word and bit straight
// from the event -- then per observer
//     X   = dp2a(pair, W, hrc) - n*E          (crossing: z*n - E*n; cell: z + h_r - E)
//     lhs = X * M',  rhs = N * yv              (M' = L2*M: one product for both kinds)
//     crossing: horizon <- (X, yv) iff lhs > rhs;  cell: visible iff lhs >= rhs
// and a flag when the two products' low words agree (a superset of the exact
// ties, re-decided in fp64 by k_vs_fp64_ties).
template <int K, int STEP>
__device__ __forceinline__ void vs_events_k3(const int* rk, const int* ck, const int* Ek, const VsArgs& a,
                                             const int4* __restrict__ rays, const int2* __restrict__ groups,
                                             const uint2* __restrict__ events, int ngroups, uint32_t* s_bits,
                                             int bits_stride, unsigned long long* counters) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const uint32_t* __restrict__ B[K];
    int nE[K];
    uint32_t sb[K];
    const int p2 = a.p2, hr = a.hr;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        B[k] = a.pairs + (int64_t)(rk[k] - a.zoff) * a.p2 + 2 * ck[k] + (threadIdx.x >> 10);
        asm("mov.b64 %0, %0;" : "+l"(B[k]));
        nE[k] = -Ek[k];
        sb[k] = (uint32_t)__cvta_generic_to_shared(s_bits + k * bits_stride);
    }
    for (int g = warp; g < ngroups; g += nwarps) {
        const int2 grp = __ldg(groups + g);
        const int ray = g * 32 + lane;
        int p = 0, q = 0;
        if (ray < a.nrays) { const int4 rd = __ldg(rays + ray); p = rd.x; q = rd.y; }
        const int L2 = p * p + q * q;
        // horizon N/M' (M' = L2*M) from a sentinel below every real tangent (see vs_events_k)
        int NH[K], MH[K];
        bool tied[K];
#pragma unroll
        for (int k = 0; k < K; ++k) { NH[k] = -(1 << 30); MH[k] = L2; tied[k] = false; }
        const uint2* ev = events + (int64_t)grp.x * 32 + lane;
        // software pipeline: the next iteration's events are loaded while this
        // one computes (the stream is padded by STEP rows of Nops at its end)
        // (two-event iterations only: at STEP 4 the extra registers cost more, c5 1027 -> 1055 ms)
#ifndef VS_PRE4
#define VS_PRE4 0
#endif
        constexpr bool kPre = STEP == 2 || VS_PRE4;
        uint2 en[STEP];
#pragma unroll
        for (int u = 0; u < STEP; ++u) en[u] = kPre ? __ldg(ev + u * 32) : make_uint2(0u, 0u);
        for (int st0 = 0; st0 < grp.y; st0 += STEP, ev += 32 * STEP) {
            uint2 ee[STEP];
            uint32_t pr[STEP][K];
#pragma unroll
            for (int u = 0; u < STEP; ++u) {
                ee[u] = kPre ? en[u] : __ldg(ev + u * 32);
                const int dr = ((int)(ee[u].x << 21)) >> 23, F = ((int)(ee[u].x << 11)) >> 22;
                const int off = dr * p2 + F;   // Nop events carry dr = F = 0
#pragma unroll
                for (int k = 0; k < K; ++k) pr[u][k] = vs_pld(B[k] + off);
            }
            if (kPre) {
#pragma unroll
                for (int u = 0; u < STEP; ++u) en[u] = __ldg(ev + 32 * STEP + u * 32);
            }
#pragma unroll
            for (int u = 0; u < STEP; ++u) {
                const uint32_t x = ee[u].x, type = x & 3u;
                const bool iscell = type == kEv3Cell, iscross = type == kEv3Cross;
                const uint32_t aux = (x >> 21) | ((ee[u].y >> 25) << 11);
                const int yv = (int)(ee[u].y & 0x1ffffffu);
                const uint32_t W = iscell ? 1u : aux;
                const int n = vs_dp2(0x00010001u, W);   // w0 + w1 (1 for a cell)
                const int hrc = iscell ? hr : 0;
                const uint32_t cw4 = (aux >> 5) << 2, cbit = 1u << (aux & 31u);
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    int v;
                    asm("dp2a.lo.s32.u32 %0, %1, %2, %3;" : "=r"(v) : "r"(pr[u][k]), "r"(W), "r"(hrc));
                    const int X = v + n * nE[k];
                    const long long lhs = mulw(X, MH[k]);
                    const long long rhs = mulw(NH[k], yv);
                    const bool up = iscross & (lhs > rhs);
                    NH[k] = up ? X : NH[k];
                    MH[k] = up ? yv : MH[k];
                    red_or_shared(sb[k] + cw4, cbit, iscell & (lhs >= rhs));
                    tied[k] |= iscell & ((uint32_t)lhs == (uint32_t)rhs);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < K; ++k)
            if (tied[k]) {   // observer k of this CTA (k_viewshed_evk's slot order)
                const int64_t slot = (int64_t)blockIdx.x * K + k;
                push_vs_tie(a, counters, a.perm ? a.perm[slot] : slot, ray);
            }
    }
}

template <bool SMEM_BITS>
__global__ void k_viewshed_ev(const int16_t* __restrict__ z, const int32_t* __restrict__ crow,
                              const int32_t* __restrict__ ccol, const int4* __restrict__ rays,
                              const int2* __restrict__ groups, const uint2* __restrict__ events, int ngroups,
                              VsArgs a, uint64_t* __restrict__ words, int4* __restrict__ wins,
                              int32_t* __restrict__ pops, unsigned long long* __restrict__ counters) {
    extern __shared__ __align__(16) uint32_t s_bits[];
    __shared__ int s_red[32];
    const int64_t cand = a.perm ? a.perm[blockIdx.x] : blockIdx.x;
    const int r = crow[cand], c = ccol[cand];
    const int row0 = max(0, r - a.R), col0 = max(0, c - a.R);
    const int h = min(a.nrows - 1, r + a.R) - row0 + 1, w = min(a.ncols - 1, c + a.R) - col0 + 1;
    // smem: window-dense bits (RS = w); global: cum-aligned rows (RS = nwr*64)
    const int nwr = win_nwr(col0, w);
    const int abase = SMEM_BITS ? col0 : (col0 & ~63);
    const int RS = SMEM_BITS ? w : nwr << 6;
    const int nw64 = h * nwr;
    uint64_t* out = words + cand * a.stride;
    if (SMEM_BITS) {
        for (int i = threadIdx.x; i < (h * w + 31) / 32 + 3; i += blockDim.x) s_bits[i] = 0u;
        __syncthreads();
    }
    const int E = zld(z + (int64_t)r * a.ncols + c) + a.ht;
    unsigned long long n_cross = 0, n_cells = 0;
    // every crossing/cell post lies within roi+1 of the observer
    const bool interior = r - a.R - 1 >= 0 && r + a.R + 1 < a.nrows && c - a.R - 1 >= 0 && c + a.R + 1 < a.ncols;
    if (interior)
        vs_events<true>(z, r, c, E, row0, abase, RS, a, rays, groups, events, ngroups, s_bits, out, SMEM_BITS, n_cross, n_cells,
                        cand, counters);
    else
        vs_events<false>(z, r, c, E, row0, abase, RS, a, rays, groups, events, ngroups, s_bits, out, SMEM_BITS, n_cross, n_cells,
                         cand, counters);
    if (threadIdx.x == 0) {
        const int k = (r - row0) * RS + (c - abase);
        if (SMEM_BITS) atomicOr(&s_bits[k >> 5], 1u << (k & 31));
        else atomicOr((unsigned long long*)&out[k >> 6], 1ull << (k & 63));
    }
    __syncthreads();
    int pc = 0;
    for (int i = threadIdx.x; i < nw64; i += blockDim.x) {
        uint64_t v;
        if (SMEM_BITS) {
            const int y = i / nwr;
            v = aligned_word_from_dense(s_bits, y, i - y * nwr, col0, w);
            out[i] = v;
        }
        else v = out[i];
        pc += __popcll(v);
    }
    for (int o = 16; o; o >>= 1) {
        pc += __shfl_down_sync(0xffffffffu, pc, o);
        n_cross += __shfl_down_sync(0xffffffffu, n_cross, o);
        n_cells += __shfl_down_sync(0xffffffffu, n_cells, o);
    }
    if ((threadIdx.x & 31) == 0) {
        s_red[threadIdx.x >> 5] = pc;
        atomicAdd(counters + kVsCross, n_cross);
        atomicAdd(counters + kVsCells, n_cells);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += s_red[k];
        pops[cand] = t;
        wins[cand] = make_int4(row0, col0, h, w);
    }
}

// K observers per CTA (shared event stream, smem bitmaps); CTAs where some
// observer is not interior fall back to one observer at a time.
template <int K, int MAXREG, int STEP>
__global__ void __maxnreg__(MAXREG) k_viewshed_evk(const int16_t* __restrict__ z, const int32_t* __restrict__ crow,
                               const int32_t* __restrict__ ccol, const int4* __restrict__ rays,
                               const int2* __restrict__ groups, const uint2* __restrict__ events, int ngroups,
                               VsArgs a, uint64_t* __restrict__ words, int4* __restrict__ wins,
                               int32_t* __restrict__ pops, unsigned long long* __restrict__ counters,
                               const uint2* __restrict__ events3) {
    extern __shared__ __align__(16) uint32_t s_bits[];
    __shared__ int s_red[32];
    const int bits_stride = a.sbits;
    int64_t cand[K];
    int rk[K], ck[K], Ek[K], row0[K], col0[K], hh[K], ww[K], RSk[K], K0k[K], abk[K];
    bool all_int = true;
    int nk = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int64_t slot = (int64_t)blockIdx.x * K + k;
        cand[k] = slot < a.n ? (a.perm ? a.perm[slot] : slot) : -1;
        if (cand[k] < 0) {
            all_int = false;
            rk[k] = ck[k] = Ek[k] = row0[k] = col0[k] = hh[k] = ww[k] = RSk[k] = K0k[k] = abk[k] = 0;
            continue;
        }
        ++nk;
        const int r = crow[cand[k]], c = ccol[cand[k]];
        rk[k] = r; ck[k] = c;
        row0[k] = max(0, r - a.R); col0[k] = max(0, c - a.R);
        hh[k] = min(a.nrows - 1, r + a.R) - row0[k] + 1;
        ww[k] = min(a.ncols - 1, c + a.R) - col0[k] + 1;
        RSk[k] = ww[k];          // smem bitmap: window-dense rows
        abk[k] = col0[k];
        K0k[k] = (r - row0[k]) * RSk[k] + (c - abk[k]);
        Ek[k] = zld(z + (int64_t)r * a.ncols + c) + a.ht;
        all_int = all_int && r - a.R - 1 >= 0 && r + a.R + 1 < a.nrows && c - a.R - 1 >= 0 && c + a.R + 1 < a.ncols;
    }
    for (int i = threadIdx.x; i < K * bits_stride; i += blockDim.x) s_bits[i] = 0u;
    __syncthreads();
    unsigned long long n_cross = 0, n_cells = 0;
    if (all_int) {
        unsigned long long d0 = 0, d1 = 0;
        if (a.pairs && events3) vs_events_k3<K, STEP>(rk, ck, Ek, a, rays, groups, events3, ngroups, s_bits, bits_stride, counters);
        else if (a.pairs) vs_events_k<K, true, false, STEP>(z, rk, ck, Ek, RSk, K0k, a, rays, groups, events, ngroups, s_bits, bits_stride, d0, d1,
                                                       counters);
        else vs_events_k<K, false, false, STEP>(z, rk, ck, Ek, RSk, K0k, a, rays, groups, events, ngroups, s_bits, bits_stride, d0, d1,
                                                counters);
        if (threadIdx.x == 0) { n_cross = (unsigned long long)(K * a.tmpl_cross); n_cells = (unsigned long long)(K * a.tmpl_cells); }
    } else if (a.pairs && nk == K) {   // edge observers: the same shared sweep with per-observer grid bounds
        vs_events_k<K, true, true, STEP>(z, rk, ck, Ek, RSk, K0k, a, rays, groups, events, ngroups, s_bits, bits_stride,
                                   n_cross, n_cells, counters);
    } else {
        for (int k = 0; k < K; ++k) {
            if (cand[k] < 0) continue;
            const bool in = rk[k] - a.R - 1 >= 0 && rk[k] + a.R + 1 < a.nrows && ck[k] - a.R - 1 >= 0 &&
                            ck[k] + a.R + 1 < a.ncols;
            if (in)
                vs_events<true>(z, rk[k], ck[k], Ek[k], row0[k], abk[k], RSk[k], a, rays, groups, events, ngroups,
                                s_bits + k * bits_stride, nullptr, true, n_cross, n_cells, cand[k], counters);
            else
                vs_events<false>(z, rk[k], ck[k], Ek[k], row0[k], abk[k], RSk[k], a, rays, groups, events, ngroups,
                                 s_bits + k * bits_stride, nullptr, true, n_cross, n_cells, cand[k], counters);
        }
    }
#pragma unroll
    for (int k = 0; k < K; ++k)
        if (threadIdx.x == k && cand[k] >= 0) {
            const int b = K0k[k];   // the observer's own cell
            atomicOr(&s_bits[k * bits_stride + (b >> 5)], 1u << (b & 31));
        }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        if (cand[k] < 0) continue;
        const int nwr = win_nwr(col0[k], ww[k]);
        const int nw64 = hh[k] * nwr;
        uint64_t* out = words + cand[k] * a.stride;
        int pc = 0;
        for (int i = threadIdx.x; i < nw64; i += blockDim.x) {
            const int y = i / nwr;
            const uint64_t v = aligned_word_from_dense(s_bits + k * bits_stride, y, i - y * nwr, col0[k], ww[k]);
            out[i] = v;
            pc += __popcll(v);
        }
        for (int o = 16; o; o >>= 1) pc += __shfl_down_sync(0xffffffffu, pc, o);
        if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = pc;
        __syncthreads();
        if (threadIdx.x == 0) {
            int t = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_red[w];
            pops[cand[k]] = t;
            wins[cand[k]] = make_int4(row0[k], col0[k], hh[k], ww[k]);
        }
        __syncthreads();
    }
    for (int o = 16; o; o >>= 1) {
        n_cross += __shfl_down_sync(0xffffffffu, n_cross, o);
        n_cells += __shfl_down_sync(0xffffffffu, n_cells, o);
    }
    if ((threadIdx.x & 31) == 0 && (n_cross || n_cells)) {
        atomicAdd(counters + kVsCross, n_cross);
        atomicAdd(counters + kVsCells, n_cells);
    }
}

// fp64 re-decision of the tie list (txs_params.los_arith == TXS_LOS_FP64): the
// whole ray of each listed (observer, ray) is recomputed with SPEC.md:147's
// arithmetic, operation for operation the oracle's compute_viewshed_fp64
// (oracle/oracle.cpp): crossings of the walk (0,0) -> (Kp, Kq) in exact order
// with the walk's doubles t, row, col (grid_walk.hpp:27-77), interpolation
// z0*(1-f) + z1*f, crossing tangent (z - E) / sqrt(row^2 + col^2), cell tangent
// (z + h_r - E) / (dot / sqrt(L2)), visible iff >= the running max; the ray
// ends at the first crossing with an off-grid post.  Explicit _rn intrinsics
// (no FMA contraction).  Changed bits are flipped in the resident cum-aligned
// words and the popcount adjusted.
__global__ void k_vs_fp64_ties(const int16_t* __restrict__ z, const int32_t* __restrict__ crow,
                               const int32_t* __restrict__ ccol, const int4* __restrict__ rays,
                               const uint32_t* __restrict__ cells, VsArgs a, unsigned long long* __restrict__ counters,
                               uint64_t* __restrict__ words, int32_t* __restrict__ pops) {
    const long long nt = min((long long)counters[kVsTies], a.tie_cap);
    auto Z = [&](int rr, int cc) -> double { return (double)zld(z + (int64_t)rr * a.ncols + cc); };
    auto in = [&](int rr, int cc) { return rr >= 0 && rr < a.nrows && cc >= 0 && cc < a.ncols; };
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nt; t += (long long)gridDim.x * blockDim.x) {
        const int2 e = a.ties[t];
        const int64_t cand = e.x;
        const int r = crow[cand], c = ccol[cand];
        const int row0 = max(0, r - a.R), col0 = max(0, c - a.R), w = min(a.ncols - 1, c + a.R) - col0 + 1;
        const int RS = win_nwr(col0, w) << 6, abase = col0 & ~63;
        uint64_t* out = words + cand * a.stride;
        const int4 rd = __ldg(rays + e.y);
        const int p = rd.x, q = rd.y, cb = rd.z, cnt = rd.w, L2 = p * p + q * q;
        auto cell = [&](int i, int& ca, int& cbb) {
            const uint32_t v = __ldg(cells + cb + i);
            ca = (int)(int16_t)(v & 0xffffu); cbb = (int)(int16_t)(v >> 16);
        };
        int K = 1;
        for (int i = 0; i < cnt; ++i) {
            int ca, cbb;
            cell(i, ca, cbb);
            K = max(K, (ca * p + cbb * q + L2 - 1) / L2);
        }
        const int Ei = zld(z + (int64_t)r * a.ncols + c) + a.ht;
        const double E = (double)Ei, rootL = __dsqrt_rn((double)L2);
        bool has = false;
        double H = 0.0;
        int ci = 0;
        auto test = [&](int i) {
            int ca, cbb;
            cell(i, ca, cbb);
            const int rr = r + ca, cc = c + cbb;
            if (!in(rr, cc)) return;
            const double run = __ddiv_rn((double)(ca * p + cbb * q), rootL);
            const double s = __ddiv_rn((double)(zld(z + (int64_t)rr * a.ncols + cc) + a.hr - Ei), run);
            const bool vis = !has || s >= H;
            const int64_t k = (int64_t)(rr - row0) * RS + (cc - abase);
            const unsigned long long m = 1ull << (k & 63);
            unsigned long long* wp = (unsigned long long*)out + (k >> 6);
            const bool cur = (*(volatile unsigned long long*)wp & m) != 0ull;
            if (vis != cur) {
                if (vis) atomicOr(wp, m); else atomicAnd(wp, ~m);
                atomicAdd(pops + cand, vis ? 1 : -1);
                atomicAdd(counters + kVsTiesFlipped, 1ull);
            }
        };
        const int dr = K * p, dc = K * q, nr = abs(dr), nc = abs(dc), sr = dr >= 0 ? 1 : -1, sc = dc >= 0 ? 1 : -1;
        int ir = 1, ic = 1;
        while (ci < cnt && (ir <= nr || ic <= nc)) {
            int cmp;
            if (ir > nr) cmp = 1;
            else if (ic > nc) cmp = -1;
            else {
                const long long x = (long long)ir * nc, y = (long long)ic * nr;
                cmp = x < y ? -1 : (x > y ? 1 : 0);
            }
            double t, row, col;
            int n, idx, kind;   // kind: 0 row line, 1 column line, 2 post
            bool at_end;
            if (cmp < 0) {
                t = __ddiv_rn((double)ir, (double)nr); row = (double)(sr * ir); col = dc == 0 ? 0.0 : __dmul_rn(t, (double)dc);
                kind = dc == 0 ? 2 : 0; n = nr; idx = ir; at_end = ir == nr; ++ir;
            } else if (cmp > 0) {
                t = __ddiv_rn((double)ic, (double)nc); row = dr == 0 ? 0.0 : __dmul_rn(t, (double)dr); col = (double)(sc * ic);
                kind = dr == 0 ? 2 : 1; n = nc; idx = ic; at_end = ic == nc; ++ic;
            } else {
                t = __ddiv_rn((double)ir, (double)nr); row = (double)(sr * ir); col = (double)(sc * ic);
                kind = 2; n = nr; idx = ir; at_end = ir == nr; ++ir; ++ic;
            }
            (void)t;
            if (at_end) break;
            // cells with u_c <= u_k (dot / L2 <= K idx / n) do not see this crossing
            for (;;) {
                if (ci >= cnt) break;
                int ca, cbb;
                cell(ci, ca, cbb);
                if ((long long)(ca * p + cbb * q) * n > (long long)K * idx * L2) break;
                test(ci++);
            }
            if (ci >= cnt) break;
            double zt;
            if (kind == 2) {
                const int rr = r + (int)row, cc = c + (int)col;
                if (!in(rr, cc)) break;
                zt = Z(rr, cc);
            } else if (kind == 0) {
                const double cf = floor(col), f = __dsub_rn(col, cf);
                const int rr = r + (int)row, c0 = c + (int)cf;
                if (!in(rr, c0) || !in(rr, c0 + 1)) break;
                zt = __dadd_rn(__dmul_rn(Z(rr, c0), __dsub_rn(1.0, f)), __dmul_rn(Z(rr, c0 + 1), f));
            } else {
                const double rf = floor(row), f = __dsub_rn(row, rf);
                const int r0 = r + (int)rf, cc = c + (int)col;
                if (!in(r0, cc) || !in(r0 + 1, cc)) break;
                zt = __dadd_rn(__dmul_rn(Z(r0, cc), __dsub_rn(1.0, f)), __dmul_rn(Z(r0 + 1, cc), f));
            }
            const double s = __ddiv_rn(__dsub_rn(zt, E), __dsqrt_rn(__dadd_rn(__dmul_rn(row, row), __dmul_rn(col, col))));
            if (!has || s > H) { has = true; H = s; }
        }
        while (ci < cnt) test(ci++);
    }
}

__global__ void k_tile_keys(const int32_t* __restrict__ crow, const int32_t* __restrict__ ccol, int64_t n, int tiles_x,
                            int tshift, uint32_t* __restrict__ keys, int32_t* __restrict__ idx) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    keys[i] = (uint32_t)((crow[i] >> tshift) * tiles_x + (ccol[i] >> tshift));
    idx[i] = (int32_t)i;
}

}  // namespace

txs_status launch_viewsheds(txs_ctx* c, const txs_params& p) {
    RayTemplateDev* T = nullptr;
    txs_status st = get_template(c, p.roi, &T);
    if (st != TXS_OK) return st;
    const int64_t n = c->ncand, mw = aligned_stride(p.roi);   // engine-internal cum-aligned layout
    set_zbounds(c->d_z, c->d_z + c->z_rows * c->ncols, c->stream);
    TXS_CUDA(c, "viewshed", cudaStreamSynchronize(c->stream));
    if (ensure(c, "viewshed", (void**)&c->d_words, &c->words_cap, sizeof(uint64_t) * (n * mw + 8)) != TXS_OK ||
        ensure(c, "viewshed", (void**)&c->d_win, &c->win_cap, sizeof(int4) * std::max<int64_t>(1, n)) != TXS_OK ||
        ensure(c, "viewshed", (void**)&c->d_pop, &c->pop_cap, sizeof(int32_t) * std::max<int64_t>(1, n)) != TXS_OK)
        return fail(c, TXS_ERR_OUT_OF_MEMORY, "viewshed", "cannot hold the packed viewsheds");
    c->vs_roi = p.roi;
    c->vs_n = n;
    c->vs_stride = mw;
    if (n == 0) return TXS_OK;
    VsArgs a{(int)c->nrows, (int)c->ncols, p.roi, p.tx_height, p.rx_height, T->nrays, mw, nullptr, n, 0, 0, 0,
             nullptr, 0, 0, 0, nullptr, 0};
    // fp64 tie list (rays with a cell exactly at its horizon: ~2e-5 of cells at
    // roi 100, fewer at larger roi); txs_compute_viewsheds re-runs on overflow
    {
        const int64_t want = std::max<int64_t>(c->vs_tie_min,
                                               std::min<int64_t>(1 << 26, std::max<int64_t>(1 << 20, n * T->nrays / 256)));
        if (ensure(c, "viewshed", (void**)&c->d_ties, &c->ties_cap, sizeof(int2) * (size_t)want) != TXS_OK)
            return TXS_ERR_OUT_OF_MEMORY;
        a.ties = (int2*)c->d_ties;
        a.tie_cap = (long long)(c->ties_cap / sizeof(int2));
        TXS_CUDA(c, "viewshed", cudaMemsetAsync(c->d_counters + kVsTies, 0, sizeof(unsigned long long), c->stream));
    }
    // Process observers in 16x16-tile order so the CTAs resident at any moment
    // read overlapping terrain windows (L2 reuse; config 5's observers are
    // random over a 537 MB terrain).  Output slots keep candidate order.
    if (n >= 4096) {
        int tshift = 4;   // 16x16-post observer tiles (measured 4 / 5 / 6: c5 1262 / 1264 / 1276 ms, c2 / c3 flat)
        if (const char* e = getenv("TXS_VS_TILE_SHIFT")) tshift = std::max(0, std::min(12, atoi(e)));
        const int tiles_x = (int)((c->ncols + (1 << tshift) - 1) >> tshift);
        size_t tmp_bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (uint32_t*)nullptr, (uint32_t*)nullptr, (int32_t*)nullptr,
                                        (int32_t*)nullptr, (int)n);
        const size_t need = 16 * (size_t)n + tmp_bytes + 256;
        if (ensure(c, "viewshed", &c->d_scratch, &c->scratch_cap, need) != TXS_OK) return TXS_ERR_OUT_OF_MEMORY;
        uint32_t* keys = (uint32_t*)c->d_scratch;
        uint32_t* keys2 = keys + n;
        int32_t* idx = (int32_t*)(keys2 + n);
        int32_t* perm = idx + n;
        void* tmp = perm + n;
        k_tile_keys<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(c->d_crow, c->d_ccol, n, tiles_x, tshift, keys, idx);
        TXS_LAUNCHED(c, "viewshed");
        TXS_CUDA(c, "viewshed", cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, idx, perm, (int)n, 0, 32,
                                                                c->stream));
        a.perm = perm;
    }
    a.sbits = (int)(((2 * p.roi + 1) * (2 * p.roi + 1) + 31) / 32 + 4);   // window-dense smem bitmap (+pad)
    const size_t smem = sizeof(uint32_t) * (size_t)a.sbits;
    if (n > 0x7fffffff) return fail(c, TXS_ERR_RANGE, "viewshed", "too many candidates");
    const bool smem_bits = smem <= 160 * 1024;
    if (!smem_bits) TXS_CUDA(c, "viewshed", cudaMemsetAsync(c->d_words, 0, sizeof(uint64_t) * n * mw, c->stream));
    a.n = n;
    {
        const EventTemplate& Et = event_template(p.roi <= kEvMaxRoi ? p.roi : 1);
        long long cr = 0, ce = 0;
        for (const uint2& e : Et.events) { const uint32_t t = e.x & 7u; cr += t <= kEvPost; ce += t == kEvCell; }
        a.tmpl_cross = cr; a.tmpl_cells = ce;
    }
    // observers per CTA (measured on B200, profiles/README.md): 3 below roi 225
    // (C2 16.2 -> 15.3 ms, C3 27.0 -> 23.5, C4 50.4 -> 44.5 against K = 2), 2 at
    // roi >= 225 (C5 1324 ms vs 1519+ for K = 3), fewer when the grid would not
    // fill the SMs (C1's 1000 observers: K = 2)
    int kobs = 1;
    if (2 * smem <= 100 * 1024 && n >= (int64_t)2 * c->num_sms * 4) kobs = 2;
    if (p.roi < 225 && 3 * smem <= 100 * 1024 && n >= (int64_t)3 * c->num_sms * 8) kobs = 3;
    if (const char* kenv = getenv("TXS_VS_K")) kobs = atoi(kenv);
    if (T->events && smem_bits && (kobs == 2 || kobs == 3 || kobs == 4) && (size_t)kobs * smem <= 200 * 1024) {
        // warps per CTA (measured, profiles/README.md; resident warps vs ray-group
        // balance): 15 at roi >= 225 (C5 1496 -> 1325 ms), 8 at roi >= 150 (C2
        // 16.5 -> 15.9), else 6 (C3 34.3 -> 27.0); TXS_VS_WARPS overrides
        int best = p.roi >= 225 ? 15 : (p.roi >= 150 ? (kobs == 3 ? 12 : 8) : 6);   // K=3, roi 200: 12 (C2 15.3 vs 16.5 at 9)
        best = std::min(best, T->ngroups);
        if (const char* e = getenv("TXS_VS_WARPS")) best = std::max(1, std::min(32, atoi(e)));
        const int threads = 32 * best;
        const size_t sm = (size_t)kobs * smem;
        // registers (resident CTAs per SM at the chosen warps): 72 at roi 150..224
        // (C2 13.5 ms vs 14.0 at 64), 64 elsewhere (C3 23.2 vs 24.3 at 68, C4 44.3 vs
        // 46.6, C5 1276 vs 1717 at 72: 15-warp CTAs drop to one per SM)
        const bool cap64 = p.roi < 150 || p.roi >= 225;
        // 4 events per sweep iteration at roi >= 225 (K=2 only), TXS_VS_STEP=2/4 overrides
        bool step4 = p.roi >= 225;
        if (const char* e = getenv("TXS_VS_STEP")) step4 = atoi(e) == 4;
        const unsigned grid = (unsigned)((n + kobs - 1) / kobs);
        // pair planes of the held rows (rebuilt per call, part of the timed stage;
        // shares the VIX quad-plane scratch buffer) -- measured (profiles/README.md):
        // C2 19.3 -> 18.0 ms, C3 34.9 -> 32.3, C5 1816 -> 1590; TXS_VS_PAIRS=0/1 overrides
        bool use_pairs = true;
        if (const char* e = getenv("TXS_VS_PAIRS")) use_pairs = atoi(e) != 0;
        if (use_pairs) {
        a.pw = (int)(((c->ncols + 31) & ~(int64_t)31) + 16);
        a.p2 = 2 * a.pw;
        a.zoff = (int)c->z_off;
        const int64_t pwords = c->z_rows * (int64_t)a.p2;
        if (ensure(c, "viewshed", (void**)&c->d_pairs, &c->pairs_cap, sizeof(uint32_t) * pwords) != TXS_OK)
            return TXS_ERR_OUT_OF_MEMORY;
        if (c->ncols % 4 == 0 && !getenv("TXS_VS_PAIRS1"))   // (four posts per thread: c3 VIEWSHED 20.55 -> 20.13 ms; TXS_VS_PAIRS1=1: one post per thread)
            k_vs_pairs4<<<(unsigned)std::min<int64_t>((c->z_rows * (a.pw / 4) + 255) / 256, (int64_t)c->num_sms * 32), 256, 0,
                          c->stream>>>(c->d_z, (uint32_t*)c->d_pairs, (int)c->z_rows, (int)c->ncols, a.pw);
        else
            k_vs_pairs<<<(unsigned)std::min<int64_t>((c->z_rows * a.pw + 255) / 256, (int64_t)c->num_sms * 32), 256, 0,
                         c->stream>>>(c->d_z, (uint32_t*)c->d_pairs, (int)c->z_rows, (int)c->ncols, a.pw);
        TXS_LAUNCHED(c, "viewshed");
        a.pairs = (const uint32_t*)c->d_pairs;
        set_zbounds(c->d_z, c->d_z + c->z_rows * c->ncols, c->stream, (const int16_t*)a.pairs,
                    (const int16_t*)(a.pairs + pwords));
        }
        // interior observers sweep the interior event encoding (TXS_VS_EV3=0: the generic one)
        const uint2* ev3 = T->events3;
        if (const char* e = getenv("TXS_VS_EV3")) ev3 = atoi(e) ? T->events3 : nullptr;
        if (kobs == 3) {
            auto kern = cap64 ? k_viewshed_evk<3, 64, 2> : k_viewshed_evk<3, 72, 2>;
            if (sm > 48 * 1024)
                TXS_CUDA(c, "viewshed", cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            cudaEventRecord(c->ev_k0, c->stream);
            kern<<<grid, threads, sm, c->stream>>>(c->zv(), c->d_crow, c->d_ccol, T->rays, T->groups, T->events,
                                                                 T->ngroups, a, c->d_words, c->d_win, c->d_pop, c->d_counters,
                                                                 ev3);
        } else if (kobs == 2) {
            auto kern = cap64 ? (step4 ? k_viewshed_evk<2, 64, 4> : k_viewshed_evk<2, 64, 2>) : k_viewshed_evk<2, 72, 2>;
            if (const char* e = getenv("TXS_VS_REGS")) {   // A/B: register cap x events per iteration
                const int rg = atoi(e);
                if (rg == 80) kern = step4 ? k_viewshed_evk<2, 80, 4> : k_viewshed_evk<2, 80, 2>;
                else if (rg == 96) kern = step4 ? k_viewshed_evk<2, 96, 4> : k_viewshed_evk<2, 96, 2>;
            }
            if (sm > 48 * 1024)
                TXS_CUDA(c, "viewshed", cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            cudaEventRecord(c->ev_k0, c->stream);
            kern<<<grid, threads, sm, c->stream>>>(c->zv(), c->d_crow, c->d_ccol, T->rays, T->groups, T->events,
                                                                 T->ngroups, a, c->d_words, c->d_win, c->d_pop, c->d_counters,
                                                                 ev3);
        } else {
            auto kern = cap64 ? k_viewshed_evk<4, 64, 2> : k_viewshed_evk<4, 72, 2>;
            if (sm > 48 * 1024)
                TXS_CUDA(c, "viewshed", cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            cudaEventRecord(c->ev_k0, c->stream);
            kern<<<grid, threads, sm, c->stream>>>(c->zv(), c->d_crow, c->d_ccol, T->rays, T->groups, T->events,
                                                                 T->ngroups, a, c->d_words, c->d_win, c->d_pop, c->d_counters,
                                                                 ev3);
        }
    } else if (T->events) {
        // warps per CTA: the divisor of the group count closest to 12 (balanced strides)
        int best = 1;
        for (int wv = 1; wv <= 32; ++wv)
            if (T->ngroups % wv == 0 && std::abs(wv - 12) < std::abs(best - 12)) best = wv;
        if (best < 4) best = std::min(T->ngroups, 8);
        const int threads = 32 * best;
        if (smem_bits) {
            if (smem > 48 * 1024)
                TXS_CUDA(c, "viewshed", cudaFuncSetAttribute(k_viewshed_ev<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            cudaEventRecord(c->ev_k0, c->stream);
            k_viewshed_ev<true><<<(unsigned)n, threads, smem, c->stream>>>(c->zv(), c->d_crow, c->d_ccol, T->rays, T->groups,
                                                                          T->events, T->ngroups, a, c->d_words, c->d_win,
                                                                          c->d_pop, c->d_counters);
        } else {
            cudaEventRecord(c->ev_k0, c->stream);
            k_viewshed_ev<false><<<(unsigned)n, threads, 0, c->stream>>>(c->zv(), c->d_crow, c->d_ccol, T->rays, T->groups,
                                                                        T->events, T->ngroups, a, c->d_words, c->d_win,
                                                                        c->d_pop, c->d_counters);
        }
    } else {
        const int per = (T->nrays + 255) / 256;
        const int threads = ((T->nrays + per - 1) / per + 31) / 32 * 32;
        if (smem_bits) {
            if (smem > 48 * 1024)
                TXS_CUDA(c, "viewshed", cudaFuncSetAttribute(k_viewshed<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            cudaEventRecord(c->ev_k0, c->stream);
            k_viewshed<true><<<(unsigned)n, threads, smem, c->stream>>>(c->zv(), c->d_crow, c->d_ccol, T->rays, T->cells, a,
                                                                        c->d_words, c->d_win, c->d_pop, c->d_counters);
        } else {
            cudaEventRecord(c->ev_k0, c->stream);
            k_viewshed<false><<<(unsigned)n, threads, 0, c->stream>>>(c->zv(), c->d_crow, c->d_ccol, T->rays, T->cells, a,
                                                                     c->d_words, c->d_win, c->d_pop, c->d_counters);
        }
    }
    cudaEventRecord(c->ev_k1, c->stream);
    TXS_LAUNCHED(c, "viewshed");
    if (p.los_arith == TXS_LOS_FP64) {   // re-decide the tied rays in fp64
        k_vs_fp64_ties<<<(unsigned)(c->num_sms * 4), 128, 0, c->stream>>>(c->zv(), c->d_crow, c->d_ccol, T->rays, T->cells, a,
                                                                         c->d_counters, c->d_words, c->d_pop);
        TXS_LAUNCHED(c, "viewshed");
    }
    return TXS_OK;
}

}  // namespace txs
