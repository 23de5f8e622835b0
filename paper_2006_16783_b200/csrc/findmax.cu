// FINDMAX stage (SPEC.md:228 partition, :238 find_candidates) — decision D7:
// blocks in block-row-major order; inside a block the top-k posts by score
// desc, then (row, col) asc.  One CTA per block: a 256-bin score histogram
// picks the threshold score theta, one ordered pass compacts the posts above
// theta (sorted afterwards by rank counting, fewer than k of them) and the
// first k-#above posts equal to theta in row-major order (block scans built
// from warp ballots).  Candidate index = output position.
#include <vector>

#include "ctx.hpp"

namespace txs {
namespace {

constexpr int kFmThreads = 256;
constexpr int kFmWarps = kFmThreads / 32;
constexpr int kMaxPerBlock = 8192;

struct FmArgs {
    int nrows, ncols, bw, bx_count, k, by0;   // by0: first block row of the band
    int64_t row_total_full;   // candidates of one full-height block row
};

__global__ void __launch_bounds__(kFmThreads) k_findmax(const uint8_t* __restrict__ vix, FmArgs a,
                                                         int32_t* __restrict__ crow, int32_t* __restrict__ ccol,
                                                         int32_t* __restrict__ cscore) {
    __shared__ int hist[256];
    __shared__ int s_theta, s_gt, s_need;
    __shared__ int s_wgt[kFmWarps], s_weq[kFmWarps];
    __shared__ int s_run_gt, s_run_eq;
    extern __shared__ int2 s_list[];   // (score, linear index) of posts above theta
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int by = blockIdx.x / a.bx_count, bxi = blockIdx.x % a.bx_count;
    const int r0 = (a.by0 + by) * a.bw, c0 = bxi * a.bw;
    const int h = min(a.bw, a.nrows - r0), w = min(a.bw, a.ncols - c0), n = h * w;
    const int kk = min(a.k, n);
    const int64_t out0 = (int64_t)by * a.row_total_full + (int64_t)bxi * min(a.k, h * a.bw);

    for (int i = tid; i < 256; i += kFmThreads) hist[i] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += kFmThreads) {
        const int y = i / w, x = i - y * w;
        atomicAdd(&hist[vix[(int64_t)(r0 + y) * a.ncols + c0 + x]], 1);
    }
    __syncthreads();
    if (tid == 0) {
        int cum = 0, v = 255;
        for (; v > 0; --v) {
            if (cum + hist[v] >= kk) break;
            cum += hist[v];
        }
        s_theta = v; s_gt = cum; s_need = kk - cum;
        s_run_gt = 0; s_run_eq = 0;
    }
    __syncthreads();
    const int theta = s_theta, cnt_gt = s_gt, need = s_need;
    for (int base = 0; base < n; base += kFmThreads) {
        const int i = base + tid;
        int s = -1;
        if (i < n) {
            const int y = i / w, x = i - y * w;
            s = vix[(int64_t)(r0 + y) * a.ncols + c0 + x];
        }
        const bool fgt = s > theta, feq = s == theta;
        const unsigned bg = __ballot_sync(0xffffffffu, fgt), be = __ballot_sync(0xffffffffu, feq);
        if (lane == 0) { s_wgt[warp] = __popc(bg); s_weq[warp] = __popc(be); }
        __syncthreads();
        int pg = s_run_gt, pe = s_run_eq, tg = 0, te = 0;
        for (int q = 0; q < kFmWarps; ++q) {
            if (q < warp) { pg += s_wgt[q]; pe += s_weq[q]; }
            tg += s_wgt[q]; te += s_weq[q];
        }
        const unsigned lt = (1u << lane) - 1;
        pg += __popc(bg & lt);
        pe += __popc(be & lt);
        if (fgt) s_list[pg] = make_int2(s, i);
        if (feq && pe < need) {
            const int y = i / w, x = i - y * w;
            const int64_t o = out0 + cnt_gt + pe;
            crow[o] = r0 + y; ccol[o] = c0 + x; cscore[o] = s;
        }
        __syncthreads();
        if (tid == 0) { s_run_gt += tg; s_run_eq += te; }
        __syncthreads();
        if (s_run_gt >= cnt_gt && s_run_eq >= need) break;
    }
    // rank the (few) posts above theta: score desc, then row-major index asc
    for (int e = tid; e < cnt_gt; e += kFmThreads) {
        const int2 me = s_list[e];
        int rank = 0;
        for (int f = 0; f < cnt_gt; ++f) {
            const int2 o = s_list[f];
            rank += (o.x > me.x) || (o.x == me.x && o.y < me.y);
        }
        const int y = me.y / w, x = me.y - y * w;
        crow[out0 + rank] = r0 + y; ccol[out0 + rank] = c0 + x; cscore[out0 + rank] = me.x;
    }
}

__global__ void k_random_observers(int64_t n, uint64_t seed, FastMod64 mr, FastMod64 mc,
                                   int32_t* __restrict__ crow, int32_t* __restrict__ ccol, int32_t* __restrict__ cs) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        crow[i] = (int32_t)fm_mod(mr, sm_draw(seed, 2 * (uint64_t)i));
        ccol[i] = (int32_t)fm_mod(mc, sm_draw(seed, 2 * (uint64_t)i + 1));
        cs[i] = 0;
    }
}

}  // namespace

txs_status launch_findmax(txs_ctx* c, const txs_params& p, int64_t bw) {
    if (p.per_block > kMaxPerBlock) return fail(c, TXS_ERR_RANGE, "findmax", "per_block > 8192");
    FmArgs a;
    a.nrows = (int)c->nrows; a.ncols = (int)c->ncols; a.bw = (int)bw; a.k = p.per_block;
    a.bx_count = (int)((c->ncols + bw - 1) / bw);
    a.by0 = (int)(c->band_r0 / bw);
    const int64_t by_count = (c->band_r1 - c->band_r0 + bw - 1) / bw;
    const int64_t wlast = c->ncols - (int64_t)(a.bx_count - 1) * bw;
    auto row_total = [&](int64_t h) {
        return (int64_t)(a.bx_count - 1) * std::min<int64_t>(a.k, h * bw) + std::min<int64_t>(a.k, h * wlast);
    };
    a.row_total_full = row_total(bw);
    const int64_t hlast = std::min<int64_t>(bw, c->nrows - (a.by0 + by_count - 1) * bw);
    const int64_t n = (by_count - 1) * a.row_total_full + row_total(hlast);
    const int64_t nblocks = by_count * a.bx_count;
    if (nblocks > 0x7fffffff || n >= 0x7fffffff) return fail(c, TXS_ERR_RANGE, "findmax", "too many blocks");
    TXS_CUDA(c, "findmax", cudaStreamSynchronize(c->stream));
    const size_t need = sizeof(int32_t) * (size_t)std::max<int64_t>(n, 1);
    if (need > c->cand_cap || !c->d_crow) {
        for (int32_t** q : {&c->d_crow, &c->d_ccol, &c->d_cscore}) { if (*q) cudaFree(*q); *q = nullptr; }
        c->cand_cap = 0;
        for (int32_t** q : {&c->d_crow, &c->d_ccol, &c->d_cscore}) TXS_CUDA(c, "findmax", cudaMalloc(q, need));
        c->cand_cap = need;
    }
    const size_t smem = sizeof(int2) * (size_t)std::max(1, std::min<int>(a.k, a.bw * a.bw));
    if (smem > 48 * 1024)
        TXS_CUDA(c, "findmax", cudaFuncSetAttribute(k_findmax, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_findmax<<<(unsigned)nblocks, kFmThreads, smem, c->stream>>>(c->d_vix - c->band_r0 * c->ncols, a, c->d_crow,
                                                                  c->d_ccol, c->d_cscore);
    TXS_LAUNCHED(c, "findmax");
    c->ncand = n;
    return TXS_OK;
}

txs_status launch_random_observers(txs_ctx* c, int64_t n, uint64_t seed) {
    if (n == 0) return TXS_OK;
    const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)c->num_sms * 16);
    k_random_observers<<<blocks, 256, 0, c->stream>>>(n, seed, make_fastmod((uint64_t)c->nrows),
                                                      make_fastmod((uint64_t)c->ncols), c->d_crow, c->d_ccol, c->d_cscore);
    TXS_LAUNCHED(c, "findmax");
    return TXS_OK;
}

}  // namespace txs
