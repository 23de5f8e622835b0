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

constexpr int kTile = 32;          // posts per tile side
constexpr int kVixThreads = 512;   // 16 warps
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

// exact floor(num / n) and remainder for 0 <= num < 2^24, n >= 1, via fp32 reciprocal + one fix-up
__device__ __forceinline__ void divmod_small(int num, int n, float rinv, int& q, int& m) {
    q = __float2int_rz(__int2float_rn(num) * rinv);
    m = num - q * n;
    if (m >= n) { ++q; m -= n; }
    if (m < 0) { --q; m += n; }
}

// Warp-cooperative exact LOS: returns true (uniform) iff the segment is blocked.
__device__ __forceinline__ bool warp_blocked(const TerrainView& T, int r, int c, int dr, int dc, int E, int Zt, int lane) {
    const int nr = abs(dr), nc = abs(dc);
    const int sr = dr >= 0 ? 1 : -1, sc = dc >= 0 ? 1 : -1;
    const int nrow = nr > 1 ? nr - 1 : 0, ncol = nc > 1 ? nc - 1 : 0, total = nrow + ncol;
    const int D = Zt - E;
    const float rr_inv = nr ? __frcp_rn((float)nr) : 0.f, rc_inv = nc ? __frcp_rn((float)nc) : 0.f;
    for (int g0 = 0; g0 < total; g0 += 32) {
        const int g = g0 + lane;
        bool b = false;
        if (g < nrow) {
            const int i = g + 1;
            int q, m;
            divmod_small(i * nc, nr, rr_inv, q, m);
            const int rr = r + sr * i, c0 = c + sc * q;
            int zn = T.at(rr, c0) * (nr - m);
            if (m) zn += T.at(rr, c0 + sc) * m;
            b = zn > E * nr + i * D;
        } else if (g < total) {
            const int j = g - nrow + 1;
            int q, m;
            divmod_small(j * nr, nc, rc_inv, q, m);
            const int cc = c + sc * j, r0 = r + sr * q;
            int zn = T.at(r0, cc) * (nc - m);
            if (m) zn += T.at(r0 + sr, cc) * m;
            b = zn > E * nc + j * D;
        }
        if (__any_sync(kFull, b)) return true;
    }
    return false;
}

__device__ __forceinline__ int warp_of_thread() { return threadIdx.x >> 5; }

__device__ __forceinline__ int gcd_i(int a, int b) {
    while (b) { const int t = a % b; a = b; b = t; }
    return a;
}

struct VixArgs {
    int R, ht, hr, S;
    uint64_t seed;
    FastMod64 span;   // 2R+1
    int tiles_x;
};

template <bool SMEM>
__global__ void __launch_bounds__(kVixThreads) k_vix(const int16_t* __restrict__ z, int nrows, int ncols,
                                                      uint8_t* __restrict__ out, VixArgs a,
                                                      unsigned long long* __restrict__ counters) {
    extern __shared__ __align__(16) unsigned char s_dyn[];
    // dynamic smem: [samples: kVixWarps x S ints][terrain tile (SMEM only)]
    int* s_samp = (int*)s_dyn + warp_of_thread() * a.S;
    int16_t* s_tile = (int16_t*)((int*)s_dyn + kVixWarps * a.S + 4);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ty0 = (blockIdx.x / a.tiles_x) * kTile, tx0 = (blockIdx.x % a.tiles_x) * kTile;
    TerrainView T{z, nullptr, ncols, 0, 0, 0};
    if (SMEM) {
        const int r0 = max(0, ty0 - a.R), r1 = min(nrows - 1, ty0 + kTile - 1 + a.R);
        const int c0 = max(0, tx0 - a.R), c1 = min(ncols - 1, tx0 + kTile - 1 + a.R);
        const int sh = r1 - r0 + 1, sw = c1 - c0 + 1;
        for (int i = threadIdx.x; i < sh * sw; i += kVixThreads) {
            const int y = i / sw, x = i - y * sw;
            s_tile[i] = __ldg(z + (int64_t)(r0 + y) * ncols + c0 + x);
        }
        T.s = s_tile; T.sr0 = r0; T.sc0 = c0; T.sw = sw;
        __syncthreads();
    }
    const int R2 = a.R * a.R;
    unsigned long long n_los = 0, n_cross = 0;
    for (int pi = warp; pi < kTile * kTile; pi += kVixWarps) {
        const int r = ty0 + pi / kTile, c = tx0 + pi % kTile;
        if (r >= nrows || c >= ncols) continue;
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
        // ---- test them ----
        int vis = 0;
        for (int sidx = 0; sidx < a.S; ++sidx) {
            const int pk = s_samp[sidx];
            const int dr = (int)(int16_t)(pk & 0xffff), dc = pk >> 16;
            const int Zt = T.at(r + dr, c + dc) + a.hr;
            vis += warp_blocked(T, r, c, dr, dc, E, Zt, lane) ? 0 : 1;
            if (lane == 0) {
                const int nr = abs(dr), nc = abs(dc);
                n_cross += (nr && nc) ? (nr + nc - gcd_i(nr, nc) - 1) : (nr + nc > 0 ? nr + nc - 1 : 0);
            }
        }
        __syncwarp();
        if (lane == 0) {
            out[(int64_t)r * ncols + c] = (uint8_t)vis;
            n_los += a.S;
        }
    }
    if (lane == 0 && n_los) {
        atomicAdd(counters + kVixLos, n_los);
        atomicAdd(counters + kVixCrossFull, n_cross);
    }
}

// one warp per pair
__global__ void k_los_batch(const int16_t* __restrict__ z, int nrows, int ncols, const int4* __restrict__ pairs,
                            int64_t n, int ht, int hr, uint8_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (w >= n) return;
    const int4 p = pairs[w];
    TerrainView T{z, nullptr, ncols, 0, 0, 0};
    const int E = T.at(p.x, p.y) + ht, Zt = T.at(p.z, p.w) + hr;
    const bool blocked = warp_blocked(T, p.x, p.y, p.z - p.x, p.w - p.y, E, Zt, lane);
    if (lane == 0) out[w] = blocked ? 0 : 1;
}

}  // namespace

txs_status launch_vix(txs_ctx* c, const txs_params& p) {
    VixArgs a;
    a.R = p.roi; a.ht = p.tx_height; a.hr = p.rx_height; a.S = p.samples_per_point;
    a.seed = p.seed;
    a.span = make_fastmod((uint64_t)(2 * p.roi + 1));
    a.tiles_x = (int)((c->ncols + kTile - 1) / kTile);
    const int64_t tiles = a.tiles_x * ((c->nrows + kTile - 1) / kTile);
    if (tiles > 0x7fffffff) return fail(c, TXS_ERR_RANGE, "vix", "grid too large");
    const int64_t side = kTile + 2 * (int64_t)p.roi;
    const size_t samp = sizeof(int) * (kVixWarps * (size_t)a.S + 4);
    const size_t smem = samp + sizeof(int16_t) * side * side;
    if (smem <= 110 * 1024) {   // two CTAs per SM
        TXS_CUDA(c, "vix", cudaFuncSetAttribute(k_vix<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_vix<true><<<(unsigned)tiles, kVixThreads, smem, c->stream>>>(c->d_z, (int)c->nrows, (int)c->ncols, c->d_vix, a, c->d_counters);
    } else {
        k_vix<false><<<(unsigned)tiles, kVixThreads, samp, c->stream>>>(c->d_z, (int)c->nrows, (int)c->ncols, c->d_vix, a, c->d_counters);
    }
    TXS_LAUNCHED(c, "vix");
    return TXS_OK;
}

txs_status launch_los_batch(txs_ctx* c, const int32_t* d_pairs, int64_t n, int32_t ht, int32_t hr, uint8_t* d_out) {
    const int64_t threads = n * 32;
    const unsigned blocks = (unsigned)((threads + 255) / 256);
    k_los_batch<<<blocks, 256, 0, c->stream>>>(c->d_z, (int)c->nrows, (int)c->ncols, (const int4*)d_pairs, n, ht, hr, d_out);
    TXS_LAUNCHED(c, "los");
    return TXS_OK;
}

}  // namespace txs
