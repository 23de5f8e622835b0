// SITE stage (site, marginal_gain, coverage) — decision D9.
//
// Greedy max-coverage whose output equals naive greedy:
// each round the candidate with the largest marginal gain popc(v & ~cum) wins,
// ties to the lowest candidate index, then its window is ORed
// into the cumulative bitmap.  Two exact device strategies (txs_params.site_mode):
//   0  incremental: gains are kept exact; after committing winner w with newly
//      covered bits D = v_w & ~cum, only candidates whose window overlaps w's
//      change, by popc(v_i & D) (SPEC.md:404's lazy rule made exact instead of
//      lazy: gain_i(t+1) = gain_i(t) - popc(v_i & D)).  Neighbours come from a
//      CSR bucket grid of side roi over candidate positions.
//   1  full rescan: every round recomputes popc(v_i & ~cum) for all i — the
//      HBM-streaming pass (the SITE GB/s roofline figure).
// Per round: k_argmax (grid reduction of (gain<<32 | ~idx)), k_commit (one
// CTA: stop rules, delta/cum update, step record, neighbour ranges) and
// k_update / k_gain_full, captured as a CUDA graph of kRoundsPerGraph rounds;
// kernels become no-ops once the device flag `done` is set.
//
// Bitmaps inside the engine are row-padded (wpr = ceil(ncols/64) words per
// terrain row) so a window row maps to whole words; the dense row-major
// CumulativeShed of SPEC.md:351 is produced on download.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <cstdlib>
#include <cstring>
#include <vector>

#include "ctx.hpp"

namespace txs {
namespace {

namespace cg = cooperative_groups;

#ifndef SITE_ROUNDS_PER_GRAPH
#define SITE_ROUNDS_PER_GRAPH 64   // measured 16 / 64: c5 80.8 / 77.5 ms (fewer host polls)
#endif
constexpr int kRoundsPerGraph = SITE_ROUNDS_PER_GRAPH;
constexpr unsigned kFull = 0xffffffffu;

struct SiteArgs {
    int nrows, ncols, R, bsize, nbx, nby;
    int cr0, cr1;                     // cum region rows held [cr0, cr1)
    int dpitch;                       // delta window row pitch (words)
    int64_t wpr, n, stride, max_sel;
    double target, total;
    int prof;                         // k_site_loop1: accumulate per-phase device time (TXS_SITE_PROFILE=1)
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__global__ void k_init_gains(const int32_t* __restrict__ pop, int32_t* __restrict__ gain, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        gain[i] = pop[i];
}

__global__ void k_bucket_count(const int32_t* __restrict__ crow, const int32_t* __restrict__ ccol, int64_t n,
                               int bsize, int nbx, int32_t* __restrict__ counts) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&counts[(crow[i] / bsize) * nbx + ccol[i] / bsize], 1);
}

__global__ void k_bucket_fill(const int32_t* __restrict__ crow, const int32_t* __restrict__ ccol, int64_t n,
                              int bsize, int nbx, int32_t* __restrict__ cursor, int32_t* __restrict__ items) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        items[atomicAdd(&cursor[(crow[i] / bsize) * nbx + ccol[i] / bsize], 1)] = (int32_t)i;
}

__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) { return a > b ? a : b; }

struct LoopPtrs {
    const int32_t* crow;
    const int32_t* ccol;
    const int4* wins;
    const int32_t* bstart;
    txs_step* steps;
};

// Grid argmax of (gain << 32 | ~idx); the last CTA to finish takes the
// round's decision (SPEC.md:367 stop rules in decision-D9 order), records the
// step and the winner window, and computes the neighbour bucket ranges.
__global__ void k_argmax(const int32_t* __restrict__ gain, SiteArgs a, SiteState* st, LoopPtrs lp,
                         int2* __restrict__ dspan) {
    if (st->done) return;
    if (st->finish) {   // previous round committed the final pick
        if (blockIdx.x == 0 && threadIdx.x == 0) st->done = 1;
        return;
    }
    __shared__ unsigned long long s_red[32];
    __shared__ bool s_last;
    unsigned long long best = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = ((unsigned long long)(uint32_t)gain[i] << 32) | (0xffffffffull - (uint64_t)i);
        best = umax64(best, key);
    }
    for (int o = 16; o; o >>= 1) best = umax64(best, __shfl_xor_sync(kFull, best, o));
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        best = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) best = umax64(best, s_red[k]);
        if (best) atomicMax(&st->best_key, best);
        __threadfence();
        s_last = atomicAdd(&st->blocks_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    for (int y = threadIdx.x; y < 2 * a.R + 1; y += blockDim.x) dspan[y] = make_int2(0x7fffffff, -1);
    if (threadIdx.x != 0) return;
    __threadfence();
    const unsigned long long key = atomicAdd(&st->best_key, 0ull);
    st->best_key = 0ull;
    st->blocks_done = 0u;
    const int g = (int)(key >> 32);
    const int64_t idx = (int64_t)(0xffffffffull - (key & 0xffffffffull));
    if (st->nsel >= a.n) { st->done = 1; st->stop = TXS_STOP_EXHAUSTED; return; }
    if (g <= 0) { st->done = 1; st->stop = TXS_STOP_ZERO_GAIN; return; }
    const int4 win = lp.wins[idx];
    const int r = lp.crow[idx], c = lp.ccol[idx];
    const long long k = st->nsel;
    st->covered += g;
    const double cov = (double)st->covered / a.total;
    lp.steps[k] = txs_step{idx, r, c, (int64_t)g, cov};
    st->nsel = k + 1;
    st->w_idx = (int)idx; st->w_gain = g;
    st->w_row0 = win.x; st->w_col0 = win.y; st->w_h = win.z; st->w_w = win.w;
    if (cov >= a.target) { st->finish = 1; st->stop = TXS_STOP_TARGET_REACHED; }
    else if (a.max_sel > 0 && k + 1 >= a.max_sel) { st->finish = 1; st->stop = TXS_STOP_MAX_SELECTED; }
    // neighbours: candidates within 2R rows/cols of the winner (window overlap);
    // consecutive buckets of one bucket row are one CSR range
    const int by0 = max(0, (r - 2 * a.R) / a.bsize), by1 = min(a.nby - 1, (r + 2 * a.R) / a.bsize);
    const int bx0 = max(0, (c - 2 * a.R) / a.bsize), bx1 = min(a.nbx - 1, (c + 2 * a.R) / a.bsize);
    int nb = 0, pref = 0;
    for (int by = by0; by <= by1 && nb < kMaxNb; ++by) {
        const int s0 = lp.bstart[by * a.nbx + bx0], e0 = lp.bstart[by * a.nbx + bx1 + 1];
        st->nb_start[nb] = s0;
        st->nb_pref[nb] = pref;
        pref += e0 - s0;
        ++nb;
    }
    st->nb_pref[nb] = pref;
    st->nb_count = nb;
}

// Newly covered bits of the winner: d = v_w & ~cum per cum word of its window
// (the viewshed rows are cum-aligned, so word b of window row y IS cum word
// (row0+y, (col0>>6)+b)); cum |= d; d is stored in the window-shaped delta
// buffer and every row keeps the span [lo, hi] of its non-zero words.
// (sharded: the window comes from `xfer` and only the held cum rows are touched)
__device__ __forceinline__ void commit_body(const SiteArgs& a, int r0, int c0, int h, int w, const uint64_t* __restrict__ v,
                                            uint64_t* __restrict__ cum, uint64_t* __restrict__ dwin,
                                            int2* __restrict__ dspan, int tid, int nthreads) {
    const int wlo = c0 >> 6, nwr = win_nwr(c0, w);
    const int ya = max(r0, a.cr0), yb = min(r0 + h, a.cr1);   // held rows of the window
    for (int t = tid; t < (yb - ya) * nwr; t += nthreads) {
        const int y = ya + t / nwr, b = t % nwr;
        const int64_t o = (int64_t)y * a.wpr + wlo + b;
        const uint64_t cw = cum[o];
        const uint64_t d = v[(y - r0) * nwr + b] & ~cw;
        dwin[(int64_t)(y - r0) * a.dpitch + b] = d;
        if (d) {
            cum[o] = cw | d;
            atomicMin(&dspan[y - r0].x, b);
            atomicMax(&dspan[y - r0].y, b);
        }
    }
}

__global__ void k_commit(SiteArgs a, SiteState* st, const uint64_t* __restrict__ words, uint64_t* __restrict__ cum,
                         uint64_t* __restrict__ dwin, int2* __restrict__ dspan, const uint64_t* __restrict__ xfer) {
    if (st->done) return;
    const uint64_t* v = xfer ? xfer : words + (int64_t)st->w_idx * a.stride;
    commit_body(a, st->w_row0, st->w_col0, st->w_h, st->w_w, v, cum, dwin, dspan, blockIdx.x * blockDim.x + threadIdx.x,
                gridDim.x * blockDim.x);
}

// incremental: gain_i -= popc(v_i & delta) for the neighbours i whose window
// overlaps the winner's; one CTA per neighbour, its threads over the overlap
// rows, each row visiting only the delta span of non-zero words.
#ifndef SITE_UPD_THREADS
#define SITE_UPD_THREADS 128
#endif
constexpr int kUpdThreads = SITE_UPD_THREADS;
constexpr int kUpdPerSm = 32;   // k_update CTAs per SM
#ifndef SITE_UPD_U
#define SITE_UPD_U 4
#endif
constexpr int kUpdU = SITE_UPD_U;   // delta words in flight per row in the neighbour updates

// One CTA per neighbour f in [first, total) step `stride`: the CTA's threads
// take the overlap rows (short per-thread dependency chains — this loop is
// latency-bound), each row visiting only the delta span of non-zero words.
// nb_* describe the neighbour list (CSR bucket ranges).  Returns the SITE
// bytes touched (counted by thread 0).
template <bool kAtomic = false>
__device__ __forceinline__ unsigned long long update_body(const SiteArgs& a, int wr0, int wc0, int wh, int ww, int nb,
                                                          const int* nb_start, const int* nb_pref,
                                                          const int4* __restrict__ wins, const uint64_t* __restrict__ words,
                                                          const uint64_t* __restrict__ dwin, const int2* __restrict__ dspan,
                                                          const int32_t* __restrict__ items, int32_t* __restrict__ gain,
                                                          int first, int stride, int* s_red, int* s_cnt) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int total = nb_pref[nb];
    const int wr1 = wr0 + wh - 1, wc1 = wc0 + ww - 1, wlo_w = wc0 >> 6;
    unsigned long long bytes_all = 0;
    for (int f = first; f < total; f += stride) {
        int k = 0;
        while (k + 1 < nb && nb_pref[k + 1] <= f) ++k;
        const int i = items[nb_start[k] + (f - nb_pref[k])];
        const int4 win = wins[i];
        const int ra = max(win.x, wr0), rb = min(win.x + win.z - 1, wr1);
        const int cl = max(win.y, wc0), ch = min(win.y + win.w - 1, wc1);
        if (ra > rb || cl > ch) continue;   // uniform across the CTA
        const uint64_t* v = words + (int64_t)i * a.stride;
        const int blo = (cl >> 6) - wlo_w, bhi = (ch >> 6) - wlo_w;   // overlap words, winner-relative
        const int nwr_i = win_nwr(win.y, win.w), shift_i = wlo_w - (win.y >> 6);   // winner word b = i word b+shift
        int acc = 0, touched = 0;
        for (int y = ra + threadIdx.x; y <= rb; y += blockDim.x) {
            const int2 sp = dspan[y - wr0];
            const int lo = max(sp.x, blo), hi = min(sp.y, bhi);
            const uint64_t* vr = v + (int64_t)(y - win.x) * nwr_i + shift_i;
            const uint64_t* dr = dwin + (int64_t)(y - wr0) * a.dpitch;
            // kUpdU delta words in flight, then the viewshed words under the non-zero
            // ones (two dependent latencies per kUpdU words instead of per word)
            for (int b0 = lo; b0 <= hi; b0 += kUpdU) {
                uint64_t d[kUpdU];
#pragma unroll
                for (int u = 0; u < kUpdU; ++u) d[u] = b0 + u <= hi ? dr[b0 + u] : 0ull;
#pragma unroll
                for (int u = 0; u < kUpdU; ++u)
                    if (d[u]) {
                        acc += __popcll(vr[b0 + u] & d[u]);   // both zero outside their windows: the AND is the overlap
                        ++touched;
                    }
            }
        }
        for (int o = 16; o; o >>= 1) {
            acc += __shfl_down_sync(kFull, acc, o);
            touched += __shfl_down_sync(kFull, touched, o);
        }
        if (lane == 0) { s_red[warp] = acc; s_cnt[warp] = touched; }
        __syncthreads();
        if (threadIdx.x == 0) {
            int t = 0, tb = 0;
            for (int q = 0; q < nw; ++q) { t += s_red[q]; tb += s_cnt[q]; }
            if (t) {
                if (kAtomic) atomicSub(&gain[i], t);
                else gain[i] -= t;
            }
            bytes_all += 16ull * (unsigned long long)tb;
        }
        __syncthreads();
    }
    return bytes_all;
}

__global__ void __launch_bounds__(kUpdThreads) k_update(SiteArgs a, const SiteState* __restrict__ st,
                                                         const int4* __restrict__ wins,
                                                         const uint64_t* __restrict__ words,
                                                         const uint64_t* __restrict__ dwin,
                                                         const int2* __restrict__ dspan,
                                                         const int32_t* __restrict__ items,
                                                         int32_t* __restrict__ gain,
                                                         unsigned long long* __restrict__ counters) {
    if (st->done || st->finish) return;
    __shared__ int s_red[32], s_cnt[32];
    const unsigned long long bytes = update_body(a, st->w_row0, st->w_col0, st->w_h, st->w_w, st->nb_count, st->nb_start,
                                                 st->nb_pref, wins, words, dwin, dspan, items, gain, blockIdx.x,
                                                 gridDim.x, s_red, s_cnt);
    if (threadIdx.x == 0 && bytes) atomicAdd(counters + kSiteBytes, bytes);
}

// ---- persistent SITE loop (one cooperative launch for the whole greedy) ----------
// Phase A: per-CTA partial argmax of (gain << 32 | ~idx)            -> grid sync
// Phase B: every CTA reduces the partials (identical winner and stop
//          decisions everywhere); CTA 0 records the step; all CTAs commit
//          the winner window into cum and the delta                 -> grid sync
// Phase C: neighbour gains -= popc(v_i & delta)                      -> grid sync
// Delta spans are double-buffered so the next round's buffer is reset during
// the current commit.
#ifndef SITE_LOOP_THREADS
#define SITE_LOOP_THREADS 256
#endif
constexpr int kLoopThreads = SITE_LOOP_THREADS;

#ifdef SITE_LOOP_MAXREG
#define TXS_LOOP_REGS __maxnreg__(SITE_LOOP_MAXREG)
#else
#define TXS_LOOP_REGS __launch_bounds__(kLoopThreads)
#endif
__global__ void TXS_LOOP_REGS k_site_loop(SiteArgs a, SiteState* st, LoopPtrs lp,
                                                             int32_t* __restrict__ gain, const int32_t* __restrict__ items,
                                                             const uint64_t* __restrict__ words, uint64_t* __restrict__ cum,
                                                             uint64_t* __restrict__ dwin, int2* __restrict__ dspan0,
                                                             int2* __restrict__ dspan1,
                                                             unsigned long long* __restrict__ partials,
                                                             unsigned long long* __restrict__ counters) {
    cg::grid_group grid = cg::this_grid();
    __shared__ unsigned long long s_key[kLoopThreads / 32];
    __shared__ int s_red[32], s_cnt[32];
    __shared__ int s_nb, s_nbstart[kMaxNb], s_nbpref[kMaxNb + 1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gtid = blockIdx.x * blockDim.x + tid, gthreads = gridDim.x * blockDim.x;
    const int side = 2 * a.R + 1;
    if (blockIdx.x == 0)
        for (int y = tid; y < side; y += blockDim.x) dspan0[y] = make_int2(0x7fffffff, -1);
    grid.sync();
    long long nsel = 0, covered = 0;
    int stop = TXS_STOP_EXHAUSTED;
    unsigned long long bytes_all = 0;
    for (int it = 0;; ++it) {
        int2* sp = (it & 1) ? dspan1 : dspan0;
        int2* spn = (it & 1) ? dspan0 : dspan1;
        // ---- A: partial argmax
        unsigned long long best = 0;
        for (int64_t i = gtid; i < a.n; i += gthreads)
            best = umax64(best, ((unsigned long long)(uint32_t)gain[i] << 32) | (0xffffffffull - (uint64_t)i));
        for (int o = 16; o; o >>= 1) best = umax64(best, __shfl_xor_sync(kFull, best, o));
        if (lane == 0) s_key[warp] = best;
        __syncthreads();
        if (tid == 0) {
            unsigned long long b = 0;
            for (int k = 0; k < kLoopThreads / 32; ++k) b = umax64(b, s_key[k]);
            partials[blockIdx.x] = b;
        }
        grid.sync();
        // ---- B: global winner (redundantly in every CTA), step record, commit
        best = 0;
        for (int k = tid; k < (int)gridDim.x; k += blockDim.x) best = umax64(best, partials[k]);
        for (int o = 16; o; o >>= 1) best = umax64(best, __shfl_xor_sync(kFull, best, o));
        __syncthreads();   // s_key reuse
        if (lane == 0) s_key[warp] = best;
        __syncthreads();
        unsigned long long key = 0;
        for (int k = 0; k < kLoopThreads / 32; ++k) key = umax64(key, s_key[k]);
        const int g = (int)(key >> 32);
        const int64_t idx = (int64_t)(0xffffffffull - (key & 0xffffffffull));
        if (nsel >= a.n) { stop = TXS_STOP_EXHAUSTED; break; }
        if (g <= 0) { stop = TXS_STOP_ZERO_GAIN; break; }
        const int4 win = lp.wins[idx];
        const int r = lp.crow[idx], c = lp.ccol[idx];
        covered += g;
        const double cov = (double)covered / a.total;
        if (gtid == 0) lp.steps[nsel] = txs_step{idx, r, c, (int64_t)g, cov};
        ++nsel;
        commit_body(a, win.x, win.y, win.z, win.w, words + idx * a.stride, cum, dwin, sp, gtid, gthreads);
        if (blockIdx.x == 0)
            for (int y = tid; y < side; y += blockDim.x) spn[y] = make_int2(0x7fffffff, -1);
        if (cov >= a.target) { stop = TXS_STOP_TARGET_REACHED; break; }
        if (a.max_sel > 0 && nsel >= a.max_sel) { stop = TXS_STOP_MAX_SELECTED; break; }
        if (tid == 0) {
            const int by0 = max(0, (r - 2 * a.R) / a.bsize), by1 = min(a.nby - 1, (r + 2 * a.R) / a.bsize);
            const int bx0 = max(0, (c - 2 * a.R) / a.bsize), bx1 = min(a.nbx - 1, (c + 2 * a.R) / a.bsize);
            int nb = 0, pref = 0;
            for (int by = by0; by <= by1 && nb < kMaxNb; ++by) {
                const int s0 = lp.bstart[by * a.nbx + bx0], e0 = lp.bstart[by * a.nbx + bx1 + 1];
                s_nbstart[nb] = s0;
                s_nbpref[nb] = pref;
                pref += e0 - s0;
                ++nb;
            }
            s_nbpref[nb] = pref;
            s_nb = nb;
        }
        grid.sync();
        // ---- C: neighbour updates
        bytes_all += update_body(a, win.x, win.y, win.z, win.w, s_nb, s_nbstart, s_nbpref, lp.wins, words, dwin, sp,
                                 items, gain, blockIdx.x, gridDim.x, s_red, s_cnt);
        grid.sync();
    }
    if (tid == 0 && bytes_all) atomicAdd(counters + kSiteBytes, bytes_all);
    if (gtid == 0) {
        st->nsel = nsel;
        st->covered = covered;
        st->stop = stop;
        st->done = 1;
    }
}

// ---- persistent SITE loop with ONE grid barrier per round (site_mode 0) ---------
// Candidate i is owned by CTA i mod G, which keeps its gain and window in
// shared memory, so a gain is only ever updated by its owner and the per-CTA
// partial argmax needs no barrier after the updates.  Per round r (after the
// barrier):
//   1. every CTA reduces the G partials {key = gain << 32 | ~idx, position,
//      window} of round r-1 (double-buffered by parity): identical winner w_r
//      and stop decisions (decision D9) everywhere;
//   2. the previous winner's bits are ORed into cum, rows spread over the CTAs
//      (the commit of w_{r-1} happens one round late);
//   3. every CTA updates its owned candidates whose window overlaps w_r's:
//      gain_i -= popc(v_i & v_w & ~cum & ~v_{w_{r-1}}).  The reads of cum race
//      with step 2's writes, and either value of a word gives the same result:
//      cum through w_{r-2} | v_{w_{r-1}} is exactly cum through w_{r-1};
//   4. it writes its new partial -> barrier.
// The winner overlaps itself, so its gain drops to 0 (taken).  Exact: the same
// picks, gains and cum as the three-barrier loop and naive greedy.
struct __align__(16) SitePart {
    unsigned long long key;
    int r, c, row0, col0, h, w;
};

__device__ __forceinline__ void part_max(SitePart& a, const SitePart& b) {
    if (b.key > a.key) a = b;
}

__device__ __forceinline__ SitePart shfl_part(const SitePart& p, int o) {
    SitePart q;
    q.key = __shfl_xor_sync(kFull, p.key, o);
    q.r = __shfl_xor_sync(kFull, p.r, o); q.c = __shfl_xor_sync(kFull, p.c, o);
    q.row0 = __shfl_xor_sync(kFull, p.row0, o); q.col0 = __shfl_xor_sync(kFull, p.col0, o);
    q.h = __shfl_xor_sync(kFull, p.h, o); q.w = __shfl_xor_sync(kFull, p.w, o);
    return q;
}

#ifndef SITE_L1_THREADS
#define SITE_L1_THREADS 256
#endif
constexpr int kL1Threads = SITE_L1_THREADS;

// cum |= v over the window rows slot, slot + nslots, ... (the commit of one winner)
__device__ __forceinline__ void flush_rows(const SiteArgs& a, const SitePart& w, const uint64_t* __restrict__ v,
                                           uint64_t* __restrict__ cum, int slot, int nslots) {
    const int nwr = win_nwr(w.col0, w.w), wlo = w.col0 >> 6;
    const int nrow = (w.h + nslots - 1 - slot) / nslots;   // rows of this slot
    for (int t = threadIdx.x; t < nrow * nwr; t += blockDim.x) {
        const int y = slot + (t / nwr) * nslots, b = t % nwr;
        const uint64_t x = v[y * nwr + b];
        if (x)   // a reduction, not load-or-store: no round trip before the barrier
            atomicOr((unsigned long long*)(cum + (int64_t)(w.row0 + y) * a.wpr + wlo + b), (unsigned long long)x);
    }
}

__global__ void __launch_bounds__(kL1Threads, 2) k_site_loop1(SiteArgs a, SiteState* st, LoopPtrs lp,
                                                         const int32_t* __restrict__ pop, int32_t* __restrict__ gain,
                                                         const uint64_t* __restrict__ words, uint64_t* __restrict__ cum,
                                                         SitePart* __restrict__ parts,
                                                         unsigned long long* __restrict__ counters) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char s_dyn[];
    const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int m = (int)((a.n - cta + G - 1) / G);   // owned: i = cta + G j, j < m
    int4* s_win = (int4*)s_dyn;
    int2* s_rc = (int2*)(s_win + m);
    int* s_gain = (int*)(s_rc + m);
    int* s_nb = s_gain + m;                          // owned candidates overlapping the winner
    __shared__ SitePart s_part[kL1Threads / 32];
    __shared__ int s_nnb, s_nrows[kL1Threads];
    for (int j = tid; j < m; j += blockDim.x) {
        const int64_t i = cta + (int64_t)G * j;
        s_win[j] = lp.wins[i];
        s_rc[j] = make_int2(lp.crow[i], lp.ccol[i]);
        s_gain[j] = pop[i];
    }
    __syncthreads();
    // partial argmax of the owned gains -> parts[buf][cta]
    // (keys alone travel through the shuffles; the owner of the best key then
    // writes the payload from shared memory)
    __shared__ unsigned long long s_key[kL1Threads / 32];
    __shared__ int s_kj[kL1Threads / 32];
    auto write_partial = [&](SitePart* buf) {
        unsigned long long bk = 0ull;
        int bj = -1;
        for (int j = tid; j < m; j += blockDim.x) {
            const int64_t i = cta + (int64_t)G * j;
            const unsigned long long key = ((unsigned long long)(uint32_t)s_gain[j] << 32) | (0xffffffffull - (uint64_t)i);
            if (key > bk) { bk = key; bj = j; }
        }
        for (int o = 16; o; o >>= 1) {
            const unsigned long long k2 = __shfl_xor_sync(kFull, bk, o);
            const int j2 = __shfl_xor_sync(kFull, bj, o);
            if (k2 > bk) { bk = k2; bj = j2; }
        }
        if (lane == 0) { s_key[warp] = bk; s_kj[warp] = bj; }
        __syncthreads();
        if (tid == 0) {
            unsigned long long x = s_key[0];
            int xj = s_kj[0];
            for (int k = 1; k < kL1Threads / 32; ++k)
                if (s_key[k] > x) { x = s_key[k]; xj = s_kj[k]; }
            SitePart out{0ull, 0, 0, 0, 0, 0, 0};
            if (xj >= 0) {
                const int4 wv = s_win[xj];
                out = SitePart{x, s_rc[xj].x, s_rc[xj].y, wv.x, wv.y, wv.z, wv.w};
            }
            buf[cta] = out;
        }
    };
    write_partial(parts);
    grid.sync();
    long long nsel = 0, covered = 0;
    int stop = TXS_STOP_EXHAUSTED;
    bool have_prev = false;
    SitePart prev{};
    int64_t prev_idx = 0;
    unsigned long long bytes_all = 0;
    const bool prof = a.prof && cta == 0 && tid == 0;
    unsigned long long ph[5] = {0, 0, 0, 0, 0}, tp = prof ? gtimer() : 0;
    auto mark = [&](int k) {
        if (prof) { const unsigned long long t = gtimer(); ph[k] += t - tp; tp = t; }
    };
    for (int it = 0;; ++it) {
        const SitePart* pb = parts + (size_t)(it & 1) * G;
        SitePart* pn = parts + (size_t)((it + 1) & 1) * G;
        // ---- 1. global winner (redundantly in every CTA)
        SitePart best{0ull, 0, 0, 0, 0, 0, 0};
        {
            unsigned long long bk = 0ull;
            int bk_k = -1;
            for (int k = tid; k < G; k += blockDim.x) {
                const unsigned long long key = pb[k].key;
                if (key > bk) { bk = key; bk_k = k; }
            }
            for (int o = 16; o; o >>= 1) {
                const unsigned long long k2 = __shfl_xor_sync(kFull, bk, o);
                const int i2 = __shfl_xor_sync(kFull, bk_k, o);
                if (k2 > bk) { bk = k2; bk_k = i2; }
            }
            __syncthreads();   // s_key / s_part reuse
            if (lane == 0) { s_key[warp] = bk; s_kj[warp] = bk_k; }
            __syncthreads();
            unsigned long long x = s_key[0];
            int xk = s_kj[0];
            for (int k = 1; k < kL1Threads / 32; ++k)
                if (s_key[k] > x) { x = s_key[k]; xk = s_kj[k]; }
            // one 32-byte read of the winning partial (measured: cheaper than every
            // thread loading whole partials and handing the winner over in smem)
            if (xk >= 0) best = pb[xk];
        }
        mark(0);
        mark(1);
        const int g = (int)(best.key >> 32);
        const int64_t idx = (int64_t)(0xffffffffull - (best.key & 0xffffffffull));
        // a stop ends the loop before this round's end-of-round commit of w_{r-1}: do it here
        const bool stop_now = nsel >= a.n || g <= 0;
        if (stop_now && have_prev) flush_rows(a, prev, words + prev_idx * a.stride, cum, cta, G);
        if (nsel >= a.n) { stop = TXS_STOP_EXHAUSTED; break; }
        if (g <= 0) { stop = TXS_STOP_ZERO_GAIN; break; }
        covered += g;
        const double cov = (double)covered / a.total;
        if (cta == 0 && tid == 0) lp.steps[nsel] = txs_step{idx, best.r, best.c, (int64_t)g, cov};
        ++nsel;
        const uint64_t* vw = words + idx * a.stride;
        if (cov >= a.target || (a.max_sel > 0 && nsel >= a.max_sel)) {
            stop = cov >= a.target ? TXS_STOP_TARGET_REACHED : TXS_STOP_MAX_SELECTED;
            if (have_prev) flush_rows(a, prev, words + prev_idx * a.stride, cum, cta, G);
            flush_rows(a, best, vw, cum, cta, G);   // the final commit
            break;
        }
        // ---- 3. owned neighbours: gain -= popc(v_i & v_w & ~cum & ~v_prev)
        if (tid == 0) s_nnb = 0;
        __syncthreads();
        const int wr1 = best.row0 + best.h - 1, wc1 = best.col0 + best.w - 1;
        for (int j = tid; j < m; j += blockDim.x) {
            const int4 wv = s_win[j];
            if (wv.x <= wr1 && wv.x + wv.z - 1 >= best.row0 && wv.y <= wc1 && wv.y + wv.w - 1 >= best.col0)
                s_nb[atomicAdd(&s_nnb, 1)] = j;
        }
        __syncthreads();
        const int nnb = s_nnb;
        if (nnb > 0) {
            // (neighbour, overlap row) pairs flattened over the CTA
            const int nwr_w = win_nwr(best.col0, best.w), wlo_w = best.col0 >> 6;
            const int nwr_p = have_prev ? win_nwr(prev.col0, prev.w) : 0, wlo_p = prev.col0 >> 6;
            const uint64_t* vp = have_prev ? words + prev_idx * a.stride : nullptr;
            int total = 0;   // pairs (the overlap row counts of the neighbours, prefix in s_nrows)
            for (int k0 = 0; k0 < nnb; k0 += blockDim.x) {
                // rows per neighbour of this chunk, then a CTA prefix scan (chunk <= blockDim.x neighbours)
                int rows = 0;
                if (k0 + tid < nnb) {
                    const int4 wv = s_win[s_nb[k0 + tid]];
                    rows = min(wv.x + wv.z - 1, wr1) - max(wv.x, best.row0) + 1;
                }
                int incl = rows;
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o) incl += t;
                }
                __syncthreads();
                if (lane == 31) s_part[warp].r = incl;   // warp totals (s_part is free here)
                __syncthreads();
                int woff = 0;
                for (int q = 0; q < warp; ++q) woff += s_part[q].r;
                int ctot = 0;
                for (int q = 0; q < kL1Threads / 32; ++q) ctot += s_part[q].r;
                s_nrows[tid] = woff + incl;   // inclusive prefix of the chunk's neighbours
                __syncthreads();
                const int cn = min((int)blockDim.x, nnb - k0);
                for (int t = tid; t < ctot; t += blockDim.x) {
                    int lo = 0, hi = cn - 1;     // the neighbour holding pair t
                    while (lo < hi) { const int mid = (lo + hi) >> 1; if (s_nrows[mid] > t) hi = mid; else lo = mid + 1; }
                    const int j = s_nb[k0 + lo];
                    const int4 wv = s_win[j];
                    const int y = max(wv.x, best.row0) + t - (lo ? s_nrows[lo - 1] : 0);
                    const int cl = max(wv.y, best.col0), ch = min(wv.y + wv.w - 1, wc1);
                    const int64_t i = cta + (int64_t)G * j;
                    const uint64_t* vi = words + i * a.stride + (int64_t)(y - wv.x) * win_nwr(wv.y, wv.w) - (wv.y >> 6);
                    const uint64_t* vwr = vw + (int64_t)(y - best.row0) * nwr_w - wlo_w;
                    const bool prow = have_prev && y >= prev.row0 && y < prev.row0 + prev.h;
                    const uint64_t* vpr = prow ? vp + (int64_t)(y - prev.row0) * nwr_p - wlo_p : nullptr;
                    const uint64_t* cr = cum + (int64_t)y * a.wpr;
                    int acc = 0;
                    for (int B = cl >> 6; B <= (ch >> 6); ++B) {
                        const uint64_t x = __ldg(vi + B) & __ldg(vwr + B) & ~__ldcg(cr + B);
                        const uint64_t pv = (prow && B >= wlo_p && B < wlo_p + nwr_p) ? __ldg(vpr + B) : 0ull;
                        acc += __popcll(x & ~pv);
                    }
                    if (acc) atomicSub(&s_gain[j], acc);
                }
                total += ctot;
                __syncthreads();
            }
            bytes_all += 16ull * (unsigned long long)total;
        }
        __syncthreads();
        mark(2);
        // ---- 4. new partial, then the commit of the previous winner (its rows
        // spread over the CTAs; it overlaps the wait for the slowest CTA, and
        // every commit of w_{r-1} lands before barrier r, ahead of round r+1's
        // updates, which compensate only for w_r) -> barrier
        write_partial(pn);
        if (have_prev) flush_rows(a, prev, words + prev_idx * a.stride, cum, cta, G);
        mark(3);
        prev = best;
        prev_idx = idx;
        have_prev = true;
        grid.sync();
        mark(4);
    }
    if (prof)
        for (int k = 0; k < 5; ++k) st->phase_ns[k] = ph[k];
    for (int j = tid; j < m; j += blockDim.x) gain[cta + (int64_t)G * j] = s_gain[j];
    if (tid == 0 && bytes_all) atomicAdd(counters + kSiteBytes, bytes_all);
    if (cta == 0 && tid == 0) {
        st->nsel = nsel;
        st->covered = covered;
        st->stop = stop;
        st->done = 1;
    }
}

// ---- the same loop inside ONE thread-block cluster (site_mode 0, few neighbours per round) --
// When a round updates only tens of neighbours (roi 100: c3, c4) the round is
// the latency of its barrier and of its scans: a grid barrier costs ~1.2 us
// before any waiting (profiles/scripts/gridsync_bench.cu) and the 148-CTA loop
// spent 2.7 of its 5.3 us per round there.  A cluster of CS CTAs (16,
// non-portable size) runs the identical round structure with a hardware
// cluster barrier, and the per-CTA partial winners travel through distributed
// shared memory: CTA k stores its {key, position, window} into slot k of every
// peer's s_parts[parity], so the winner reduction reads local shared memory.
// Ownership follows the neighbour-bucket order (d_bucket_items, buckets of
// side R sorted row-major): the candidate at sorted position s belongs to CTA
// s mod CS, local slot s / CS, so the winner's neighbours are <= 5 contiguous
// local ranges (one per bucket row) instead of a scan of every owned
// candidate, and the per-CTA argmax keeps a maximum per chunk of 32 slots,
// recomputed only for the chunks those ranges touch (gains only change
// there).  Per candidate in shared memory: position (2 x u16), index, gain, a
// u16 neighbour-list slot.  Same picks, gains and cum as k_site_loop1 (commit
// of w_{r-1} one round late, racing cum reads compensated by ~v_prev).
#ifndef SITE_LC_THREADS
#define SITE_LC_THREADS 512
#endif
constexpr int kLcThreads = SITE_LC_THREADS;
constexpr int kLcMaxCluster = 16;
constexpr int kLcMaxRanges = 8;   // bucket rows within 2R of a winner: <= 5 at bucket side R

__device__ __forceinline__ int4 roi_box(const SiteArgs& a, int r, int c) {
    const int row0 = max(0, r - a.R), col0 = max(0, c - a.R);
    return make_int4(row0, col0, min(a.nrows - 1, r + a.R) - row0 + 1, min(a.ncols - 1, c + a.R) - col0 + 1);
}

__global__ void __launch_bounds__(kLcThreads, 1) k_site_loopc(SiteArgs a, SiteState* st, LoopPtrs lp,
                                                              const int32_t* __restrict__ pop, int32_t* __restrict__ gain,
                                                              const int32_t* __restrict__ items,
                                                              const uint64_t* __restrict__ words, uint64_t* __restrict__ cum,
                                                              unsigned long long* __restrict__ counters) {
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char s_dyn[];
    const int G = (int)cluster.num_blocks(), cta = (int)cluster.block_rank(), tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int kWarps = kLcThreads / 32;
    const int m = (int)((a.n - cta + G - 1) / G);   // owned: sorted positions s = cta + G j, j < m
    const int mmax = (int)((a.n + G - 1) / G);      // the same carve-up in every CTA
    const int nchunk = (mmax + 31) >> 5;
    uint32_t* s_pos = (uint32_t*)s_dyn;             // row << 16 | col
    int* s_idx = (int*)(s_pos + mmax);              // candidate index
    int* s_gain = s_idx + mmax;
    unsigned long long* s_ckey = (unsigned long long*)(s_gain + mmax + (mmax & 1));   // per chunk of 32 slots: best key
    int* s_cj = (int*)(s_ckey + nchunk);                                               // ... and its slot
    uint16_t* s_nb = (uint16_t*)(s_cj + nchunk);    // owned candidates overlapping the winner (mmax <= 65535)
    __shared__ SitePart s_parts[2][kLcMaxCluster];  // [parity][writer rank], written by the peers
    __shared__ unsigned long long s_key[kWarps];
    __shared__ int s_kj[kWarps], s_wsum[kWarps];
    __shared__ int s_nnb, s_nrows[kLcThreads];
    __shared__ int s_rng[2 * kLcMaxRanges];         // local slot ranges [lo, hi) of the winner's bucket rows
    for (int j = tid; j < m; j += blockDim.x) {
        const int i = items[cta + (int64_t)G * j];
        s_pos[j] = ((uint32_t)lp.crow[i] << 16) | (uint32_t)lp.ccol[i];
        s_idx[j] = i;
        s_gain[j] = pop[i];
    }
    __syncthreads();
    // best key of chunk ch (slots 32 ch .. 32 ch + 31), by one warp
    auto chunk_max = [&](int ch) {
        const int j = ch * 32 + lane;
        unsigned long long bk = 0ull;
        int bj = -1;
        if (j < m) { bk = ((unsigned long long)(uint32_t)s_gain[j] << 32) | (0xffffffffull - (uint64_t)(uint32_t)s_idx[j]); bj = j; }
        for (int o = 16; o; o >>= 1) {
            const unsigned long long k2 = __shfl_xor_sync(kFull, bk, o);
            const int j2 = __shfl_xor_sync(kFull, bj, o);
            if (k2 > bk) { bk = k2; bj = j2; }
        }
        if (lane == 0) { s_ckey[ch] = bk; s_cj[ch] = bj; }
    };
    // the CTA's best over its chunk maxima -> slot `cta` of every peer's s_parts[buf]
    auto write_partial = [&](int buf) {
        unsigned long long bk = 0ull;
        int bj = -1;
        for (int ch = tid; ch < nchunk; ch += blockDim.x) {
            const unsigned long long key = s_ckey[ch];
            if (key > bk) { bk = key; bj = s_cj[ch]; }
        }
        for (int o = 16; o; o >>= 1) {
            const unsigned long long k2 = __shfl_xor_sync(kFull, bk, o);
            const int j2 = __shfl_xor_sync(kFull, bj, o);
            if (k2 > bk) { bk = k2; bj = j2; }
        }
        if (lane == 0) { s_key[warp] = bk; s_kj[warp] = bj; }
        __syncthreads();
        if (tid < G) {   // thread k delivers this CTA's partial to peer k
            unsigned long long x = s_key[0];
            int xj = s_kj[0];
            for (int k = 1; k < kWarps; ++k)
                if (s_key[k] > x) { x = s_key[k]; xj = s_kj[k]; }
            SitePart out{0ull, 0, 0, 0, 0, 0, 0};
            if (xj >= 0) {
                const uint32_t rc = s_pos[xj];
                const int4 wv = roi_box(a, (int)(rc >> 16), (int)(rc & 0xffffu));
                out = SitePart{x, (int)(rc >> 16), (int)(rc & 0xffffu), wv.x, wv.y, wv.z, wv.w};
            }
            SitePart* peer = cluster.map_shared_rank(&s_parts[buf][cta], tid);
            *peer = out;
        }
    };
    for (int ch = warp; ch < nchunk; ch += kWarps) chunk_max(ch);
    __syncthreads();
    write_partial(0);
    cluster.sync();
    long long nsel = 0, covered = 0;
    int stop = TXS_STOP_EXHAUSTED;
    bool have_prev = false;
    SitePart prev{};
    int64_t prev_idx = 0;
    unsigned long long bytes_all = 0;
    const bool prof = a.prof && cta == 0 && tid == 0;
    unsigned long long ph[5] = {0, 0, 0, 0, 0}, tp = prof ? gtimer() : 0;
    auto mark = [&](int k) {
        if (prof) { const unsigned long long t = gtimer(); ph[k] += t - tp; tp = t; }
    };
    for (int it = 0;; ++it) {
        // ---- 1. global winner from the local copies of the G partials (every warp, by shuffles)
        SitePart best;
        {
            unsigned long long bk = lane < G ? s_parts[it & 1][lane].key : 0ull;
            int bw = lane < G ? lane : 0;
            for (int o = 16; o; o >>= 1) {
                const unsigned long long k2 = __shfl_xor_sync(kFull, bk, o);
                const int w2 = __shfl_xor_sync(kFull, bw, o);
                if (k2 > bk) { bk = k2; bw = w2; }
            }
            best = s_parts[it & 1][bw];
        }
        const int g = (int)(best.key >> 32);
        const int64_t idx = (int64_t)(0xffffffffull - (best.key & 0xffffffffull));
        // the winner's neighbour buckets: rows by0..by1, columns bx0..bx1 -> one sorted range per
        // bucket row -> local slots [ceil((s0 - cta) / G), ceil((s1 - cta) / G))
        const int by0 = max(0, (best.r - 2 * a.R) / a.bsize), by1 = min(a.nby - 1, (best.r + 2 * a.R) / a.bsize);
        const int bx0 = max(0, (best.c - 2 * a.R) / a.bsize), bx1 = min(a.nbx - 1, (best.c + 2 * a.R) / a.bsize);
        const int nrng = min(kLcMaxRanges, by1 - by0 + 1);
        if (g > 0 && tid < 2 * nrng) {
            const int by = by0 + (tid >> 1);
            const int sp = __ldg(lp.bstart + by * a.nbx + ((tid & 1) ? bx1 + 1 : bx0));
            s_rng[tid] = max(0, (sp - cta + G - 1) / G);
        }
        mark(0);
        mark(1);
        // a stop ends the loop before this round's end-of-round commit of w_{r-1}: do it here
        const bool stop_now = nsel >= a.n || g <= 0;
        if (stop_now && have_prev) flush_rows(a, prev, words + prev_idx * a.stride, cum, cta, G);
        if (nsel >= a.n) { stop = TXS_STOP_EXHAUSTED; break; }
        if (g <= 0) { stop = TXS_STOP_ZERO_GAIN; break; }
        covered += g;
        const double cov = (double)covered / a.total;
        if (cta == 0 && tid == 0) lp.steps[nsel] = txs_step{idx, best.r, best.c, (int64_t)g, cov};
        ++nsel;
        const uint64_t* vw = words + idx * a.stride;
        if (cov >= a.target || (a.max_sel > 0 && nsel >= a.max_sel)) {
            stop = cov >= a.target ? TXS_STOP_TARGET_REACHED : TXS_STOP_MAX_SELECTED;
            if (have_prev) flush_rows(a, prev, words + prev_idx * a.stride, cum, cta, G);
            flush_rows(a, best, vw, cum, cta, G);   // the final commit
            break;
        }
        // ---- 3. owned neighbours: gain -= popc(v_i & v_w & ~cum & ~v_prev)
        if (tid == 0) s_nnb = 0;
        __syncthreads();
        const int wr1 = best.row0 + best.h - 1, wc1 = best.col0 + best.w - 1;
        // windows overlap iff the origins are within 2R of each other in both axes
        // (clipping at the grid edge shortens both boxes on the same side)
        for (int q = 0; q < nrng; ++q) {
            const int lo = s_rng[2 * q], hi = min(m, s_rng[2 * q + 1]);
            for (int j = lo + tid; j < hi; j += blockDim.x) {
                const uint32_t rc = s_pos[j];
                if (abs((int)(rc >> 16) - best.r) <= 2 * a.R && abs((int)(rc & 0xffffu) - best.c) <= 2 * a.R)
                    s_nb[atomicAdd(&s_nnb, 1)] = (uint16_t)j;
            }
        }
        __syncthreads();
        const int nnb = s_nnb;
        if (nnb > 0) {
            const int nwr_w = win_nwr(best.col0, best.w), wlo_w = best.col0 >> 6;
            const int nwr_p = have_prev ? win_nwr(prev.col0, prev.w) : 0, wlo_p = prev.col0 >> 6;
            const uint64_t* vp = have_prev ? words + prev_idx * a.stride : nullptr;
            int total = 0;
            for (int k0 = 0; k0 < nnb; k0 += blockDim.x) {
                int rows = 0;
                if (k0 + tid < nnb) {
                    const uint32_t rc = s_pos[s_nb[k0 + tid]];
                    const int4 wv = roi_box(a, (int)(rc >> 16), (int)(rc & 0xffffu));
                    rows = max(0, min(wv.x + wv.z - 1, wr1) - max(wv.x, best.row0) + 1);
                }
                int incl = rows;
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o) incl += t;
                }
                __syncthreads();
                if (lane == 31) s_wsum[warp] = incl;
                __syncthreads();
                int woff = 0, ctot = 0;
                for (int q = 0; q < kWarps; ++q) {
                    const int v = s_wsum[q];
                    if (q < warp) woff += v;
                    ctot += v;
                }
                s_nrows[tid] = woff + incl;   // inclusive prefix of the chunk's neighbours
                __syncthreads();
                const int cn = min((int)blockDim.x, nnb - k0);
                for (int t = tid; t < ctot; t += blockDim.x) {
                    int lo = 0, hi = cn - 1;     // the neighbour holding pair t
                    while (lo < hi) { const int mid = (lo + hi) >> 1; if (s_nrows[mid] > t) hi = mid; else lo = mid + 1; }
                    const int j = s_nb[k0 + lo];
                    const uint32_t rc = s_pos[j];
                    const int4 wv = roi_box(a, (int)(rc >> 16), (int)(rc & 0xffffu));
                    const int y = max(wv.x, best.row0) + t - (lo ? s_nrows[lo - 1] : 0);
                    const int cl = max(wv.y, best.col0), ch = min(wv.y + wv.w - 1, wc1);
                    const int64_t i = s_idx[j];
                    const uint64_t* vi = words + i * a.stride + (int64_t)(y - wv.x) * win_nwr(wv.y, wv.w) - (wv.y >> 6);
                    const uint64_t* vwr = vw + (int64_t)(y - best.row0) * nwr_w - wlo_w;
                    const bool prow = have_prev && y >= prev.row0 && y < prev.row0 + prev.h;
                    const uint64_t* vpr = prow ? vp + (int64_t)(y - prev.row0) * nwr_p - wlo_p : nullptr;
                    const uint64_t* cr = cum + (int64_t)y * a.wpr;
                    int acc = 0;
                    for (int B = cl >> 6; B <= (ch >> 6); ++B) {
                        const uint64_t x = __ldg(vi + B) & __ldg(vwr + B) & ~__ldcg(cr + B);
                        const uint64_t pv = (prow && B >= wlo_p && B < wlo_p + nwr_p) ? __ldg(vpr + B) : 0ull;
                        acc += __popcll(x & ~pv);
                    }
                    if (acc) atomicSub(&s_gain[j], acc);
                }
                total += ctot;
                __syncthreads();
            }
            bytes_all += 16ull * (unsigned long long)total;
        }
        __syncthreads();
        mark(2);
        // ---- 4. chunk maxima of the touched ranges, the new partial to every peer, the commit
        // of the previous winner -> cluster barrier
        {
            int base = 0;   // (range, chunk) pairs flattened over the warps
            for (int q = 0; q < nrng; ++q) {
                const int lo = s_rng[2 * q], hi = min(m, s_rng[2 * q + 1]);
                if (hi <= lo) continue;
                const int c0 = lo >> 5, c1 = (hi - 1) >> 5;
                for (int ch = c0 + ((warp - base) % kWarps + kWarps) % kWarps; ch <= c1; ch += kWarps) chunk_max(ch);
                base += c1 - c0 + 1;
            }
        }
        __syncthreads();
        write_partial((it + 1) & 1);
        if (have_prev) flush_rows(a, prev, words + prev_idx * a.stride, cum, cta, G);
        mark(3);
        prev = best;
        prev_idx = idx;
        have_prev = true;
        cluster.sync();
        mark(4);
    }
    if (prof)
        for (int k = 0; k < 5; ++k) st->phase_ns[k] = ph[k];
    for (int j = tid; j < m; j += blockDim.x) gain[s_idx[j]] = s_gain[j];
    if (tid == 0 && bytes_all) atomicAdd(counters + kSiteBytes, bytes_all);
    if (cta == 0 && tid == 0) {
        st->nsel = nsel;
        st->covered = covered;
        st->stop = stop;
        st->done = 1;
    }
    cluster.sync();   // no CTA exits while a peer may still address its shared memory
}

// Streaming form over the cum-aligned layout: lane t of the candidate's warp
// reads word t (one coalesced, L1-bypassing load; the viewshed words are the
// only HBM stream) = word b of window row y, whose cum counterpart is the
// L2-resident cum word (row0+y, (col0>>6)+b): gain = sum popc(v & ~cum).
// (measured: 4 loads in flight per lane at 46 registers beat 8 or 16 in flight
// and tighter register bounds, profiles/README.md)
// T8: the same pass over the 8x8-tile shadow layout (below): `wins` holds the
// window in tile units (ty0, tx0, nty, ntx), word t is tile (t / ntx, t % ntx)
// and its cum counterpart is word (ty0 + t / ntx, tx0 + t % ntx) of the tile
// cum (pitch a.wpr tiles); `wins_alg` (the windows in posts) only feeds the
// algorithmic byte count.
#ifndef GAIN_T8_U
#define GAIN_T8_U 5   // (stream, cum) load pairs in flight per lane of the t8 pass; measured 4 / 5 / 6 / 8: c3 4.34 / 4.39 / 3.65 / 3.91 TB/s, c4 3.94 / 4.18 / 3.54 / 3.81
#endif
template <typename G, bool T8>
__global__ void k_gain_full(SiteArgs a, const SiteState* st, const int4* __restrict__ wins,
                            const uint64_t* __restrict__ words, const uint64_t* __restrict__ cum,
                            G* __restrict__ gain, unsigned long long* __restrict__ counters,
                            const int4* __restrict__ wins_alg, int64_t pf_ahead) {
    if (st && (st->done || st->finish)) return;
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long bytes = 0;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < a.n; i += warps) {
        const int4 win = wins[i];
        const int nwr = T8 ? win.w : win_nwr(win.y, win.w), total = win.z * nwr;
        const uint64_t* v = words + i * a.stride;
        const uint64_t* crow = cum + (int64_t)win.x * a.wpr + (T8 ? win.y : (win.y >> 6));
        if (T8 && pf_ahead >= 0 && i + pf_ahead < a.n) {
            // a tile cum larger than L2 (c4: 269 MB) misses on every pass, and a warp
            // stalled on scattered cum sectors holds back its stream loads: the
            // candidate's tile rows (lane = tile row, <= 3 lines each) go to L2 first
            // (measured at c4, look-ahead 0 / 8 / 148 / 1184 candidates: 3.94 / 3.84 /
            // 3.89 / 3.84 TB/s against 3.54 without; with the cum resident in L2 the
            // prefetches only cost issue slots, c3 4.34 -> 4.11)
            const int4 wf = pf_ahead ? wins[i + pf_ahead] : win;
            if (lane < wf.z) {
                const uint64_t* q = cum + (int64_t)(wf.x + lane) * a.wpr + wf.y;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(q + 16));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(q + wf.w - 1));
            }
        }
        // word t -> (y, b): y = t / nwr via incremental steps of 32 words
        int y = lane / nwr, b = lane - y * nwr;
        const int dy = 32 / nwr, db = 32 - dy * nwr;
        int acc = 0;
        constexpr int U = T8 ? GAIN_T8_U : 4;
#ifdef GAIN_PROBE_FOLD
        const int ymask = (a.prof & 2) ? 1 : -1;   // timing probe: cum reads folded onto two rows (wrong gains)
#else
        constexpr int ymask = -1;
#endif
        for (int t0 = lane; t0 < total; t0 += 32 * U) {
            uint64_t vw[U], cw[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool ok = t0 + 32 * u < total;
                vw[u] = ok ? __ldcs(v + t0 + 32 * u) : 0ull;
                cw[u] = ok ? __ldg(crow + (int64_t)(y & ymask) * a.wpr + b) : 0ull;
                y += dy; b += db;
                if (b >= nwr) { b -= nwr; ++y; }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) acc += __popcll(vw[u] & ~cw[u]);
        }
        for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(kFull, acc, o);
        if (lane == 0) {
            gain[i] = (G)acc;
            if (counters) {   // SPEC-layout (algorithmic) bytes
                const int4 wa = T8 ? wins_alg[i] : win;
                bytes += 8ull * (((unsigned long long)wa.z * wa.w + 63) >> 6);
            }
        }
    }
    if (counters && lane == 0 && bytes) atomicAdd(counters + kSiteBytes, bytes);
}

// ---- 8x8-tile ("t8") shadow layout of the streaming gain pass ---------------
// Word (TY, TX) of a tile bitmap holds terrain rows 8TY..8TY+7 x columns
// 8TX..8TX+7, bit (r & 7) * 8 + (c & 7).  A (2R+1)^2 window touches at most
// ((2R+7)/8 + 1)^2 tiles: 1.07x its packed size at roi 100 (1.04x at 200),
// where the cum-aligned rows -- padded to 64-bit terrain words in ONE
// dimension -- take 1.32x (1.16x).  The streaming pass reads exactly these
// words, so the padding is HBM traffic; the tile words keep the property the
// pass needs: word t of a candidate has ONE cum counterpart (no shifts).
// Tile columns are bytes of the cum-aligned words (8 | 64), so the conversion
// gathers one byte from each of 8 rows.
__host__ __device__ inline int t8_span(int lo, int len) { return ((lo + len - 1) >> 3) - (lo >> 3) + 1; }
inline int64_t t8_stride(int64_t roi) { const int64_t m = ((2 * roi + 7) >> 3) + 1; return m * m; }

__global__ void k_words_to_t8(int64_t n, const int4* __restrict__ wins, const uint64_t* __restrict__ words,
                              int64_t stride, uint64_t* __restrict__ t8, int64_t t8stride, int4* __restrict__ t8win) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
        const int4 win = wins[i];   // row0, col0, h, w
        const int nwr = win_nwr(win.y, win.w), wlo = win.y >> 6;
        const int ty0 = win.x >> 3, tx0 = win.y >> 3;
        const int nty = t8_span(win.x, win.z), ntx = t8_span(win.y, win.w);
        if (lane == 0) t8win[i] = make_int4(ty0, tx0, nty, ntx);
        const uint64_t* v = words + i * stride;
        uint64_t* o = t8 + i * t8stride;
        for (int t = lane; t < nty * ntx; t += 32) {
            const int ty = t / ntx, TX = tx0 + (t - ty * ntx);
            const int b = (TX >> 3) - wlo, sh = (TX & 7) * 8;
            uint64_t out = 0;
#pragma unroll
            for (int rr = 0; rr < 8; ++rr) {
                const int y = (ty0 + ty) * 8 + rr - win.x;
                if (y >= 0 && y < win.z) out |= ((v[y * nwr + b] >> sh) & 0xffull) << (rr * 8);
            }
            o[t] = out;
        }
    }
}

// row-padded cum (rows [cr0, cr1) held) -> tile cum of the whole grid
__global__ void k_cum_to_t8(const uint64_t* __restrict__ cum, int64_t wpr, int cr0, int cr1, int th, int tw,
                            uint64_t* __restrict__ t8cum) {
    const int64_t total = (int64_t)th * tw;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int TY = (int)(t / tw), TX = (int)(t - (int64_t)TY * tw);
        const int sh = (TX & 7) * 8;
        uint64_t out = 0;
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
            const int r = TY * 8 + rr;
            if (r >= cr0 && r < cr1) out |= ((cum[(int64_t)r * wpr + (TX >> 3)] >> sh) & 0xffull) << (rr * 8);
        }
        t8cum[t] = out;
    }
}

// the round's winner into the tile cum (beside k_commit's row-padded cum)
__global__ void k_commit_t8(const SiteState* st, const int4* __restrict__ t8win, const uint64_t* __restrict__ t8,
                            int64_t t8stride, uint64_t* __restrict__ t8cum, int tw) {
    if (st->done) return;
    const int4 win = t8win[st->w_idx];
    const uint64_t* v = t8 + (int64_t)st->w_idx * t8stride;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < win.z * win.w; t += gridDim.x * blockDim.x) {
        const int ty = t / win.w, tx = t - ty * win.w;
        const uint64_t x = v[t];
        if (x) t8cum[(int64_t)(win.x + ty) * tw + win.y + tx] |= x;
    }
}

// Bucket-tiled form of k_gain_full (mode-1 rounds): one CTA per candidate
// bucket (side bsize = roi, the CSR grid of mode 0) first copies the cum
// region every window of the bucket lies in -- rows [by*bs - R, (by+1)*bs + R),
// words [(bx*bs - R) >> 6, ((bx+1)*bs - 1 + R) >> 6] -- into shared memory,
// then its warps stream the bucket's candidates' packed words from HBM (8
// coalesced 256-byte loads in flight per warp) against that copy.  The cum is
// read from L2 once per bucket instead of once per candidate, so the L2 carries
// little more than the HBM stream itself.
constexpr int kTiledThreads = 512;

struct TileBox {
    int ry0, ry1, wx0, wx1;
};
__device__ __forceinline__ TileBox tile_box(const SiteArgs& a, int bkt) {
    const int by = bkt / a.nbx, bx = bkt - by * a.nbx;
    TileBox t;
    t.ry0 = max(max(0, a.cr0), by * a.bsize - a.R);
    t.ry1 = min(min(a.nrows, a.cr1), (by + 1) * a.bsize + a.R);
    t.wx0 = max(0, bx * a.bsize - a.R) >> 6;
    t.wx1 = (min(a.ncols - 1, (bx + 1) * a.bsize - 1 + a.R) >> 6) + 1;
    return t;
}

template <typename G>
__global__ void __launch_bounds__(kTiledThreads, 2) k_gain_tiled(SiteArgs a, const SiteState* st,
                                                               const int4* __restrict__ wins,
                                                               const uint64_t* __restrict__ words,
                                                               const uint64_t* __restrict__ cum,
                                                               const int32_t* __restrict__ bstart,
                                                               const int32_t* __restrict__ items,
                                                               G* __restrict__ gain,
                                                               unsigned long long* __restrict__ counters) {
    if (st && (st->done || st->finish)) return;
    extern __shared__ __align__(16) uint64_t s_cum[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int W = kTiledThreads / 32;
    const int nbk = a.nbx * a.nby;
    unsigned long long bytes = 0;
    for (int bkt = blockIdx.x; bkt < nbk; bkt += gridDim.x) {
        const int k0 = bstart[bkt], k1 = bstart[bkt + 1];
        if (k0 == k1) continue;
        const TileBox tb = tile_box(a, bkt);
        const int pw = tb.wx1 - tb.wx0;
        for (int t = tid; t < (tb.ry1 - tb.ry0) * pw; t += kTiledThreads) {
            const int y = t / pw, x = t - y * pw;
            s_cum[t] = cum[(int64_t)(tb.ry0 + y) * a.wpr + tb.wx0 + x];
        }
        __syncthreads();
        for (int k = k0 + warp; k < k1; k += W) {
            const int64_t i = items[k];
            const int4 win = wins[i];
            const int nwr = win_nwr(win.y, win.w), total = win.z * nwr;
            const uint64_t* v = words + i * a.stride;
            const uint64_t* crow = s_cum + (win.x - tb.ry0) * pw + ((win.y >> 6) - tb.wx0);
            int y = lane / nwr, b = lane - y * nwr;
            const int dy = 32 / nwr, db = 32 - dy * nwr;
            int acc = 0;
            constexpr int U = 8;
            for (int t0 = lane; t0 < total; t0 += 32 * U) {
                uint64_t vw[U];
                int co[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    vw[u] = t0 + 32 * u < total ? __ldcs(v + t0 + 32 * u) : 0ull;
                    co[u] = y * pw + b;
                    y += dy; b += db;
                    if (b >= nwr) { b -= nwr; ++y; }
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (t0 + 32 * u < total) acc += __popcll(vw[u] & ~crow[co[u]]);
            }
            for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(kFull, acc, o);
            if (lane == 0) {
                gain[i] = (G)acc;
                bytes += 8ull * (((unsigned long long)win.z * win.w + 63) >> 6);   // SPEC-layout (algorithmic) bytes
            }
        }
        __syncthreads();
    }
    if (counters && lane == 0 && bytes) atomicAdd(counters + kSiteBytes, bytes);
}

// Strip-tile form of the full gain pass: a tile is SH terrain rows x TX
// candidate buckets (side roi).  A task is one candidate's window rows inside
// one strip -- contiguous words of its cum-aligned viewshed; the task list,
// grouped by tile, is built once per candidate set (k_strip_count /
// k_strip_fill: the windows do not change between rounds).  Per tile a CTA
// stages the cum words its tasks can reach (the tile's rows, its bucket
// columns +- roi) in shared memory once, then its warps stream the tasks:
// each viewshed word is read from HBM once per pass and each cum word from L2
// a few times per pass (the per-candidate form reads a window of cum per
// candidate: at roi 100 as many L2 bytes as HBM bytes).  A task's words arrive
// by one bulk copy (cp.async.bulk, completion on an mbarrier) into one of
// kStripSlots slots of the warp's staging ring, so every warp keeps
// kStripSlots tasks in flight whatever their length; partial popcounts go to
// the gains by atomics (zeroed first by k_zero_gains).  Warp w takes the
// tile's tasks w, w + W, w + 2W, ... (even shares).
constexpr int kStripThreads = 256;
constexpr int kStripSlots = 4;

struct StripGeo {
    int SH, TX, ntx, nstrips, r_lo, r_hi;
};
__device__ __forceinline__ void strip_tile_box(const SiteArgs& a, const StripGeo& g, int tile, int* s0, int* s1,
                                               int* wx0, int* pw) {
    const int s = tile / g.ntx, tx = tile - s * g.ntx;
    *s0 = g.r_lo + s * g.SH;
    *s1 = min(g.r_hi, *s0 + g.SH);
    const int bx0 = tx * g.TX, bx1 = min(a.nbx, bx0 + g.TX);
    *wx0 = max(0, bx0 * a.bsize - a.R) >> 6;
    *pw = ((min(a.ncols - 1, bx1 * a.bsize - 1 + a.R) >> 6) + 1) - *wx0;
}

// tasks of candidate i: one per strip its window rows (held rows) meet
template <bool FILL>
__global__ void k_strip_tasks(SiteArgs a, StripGeo g, const int4* __restrict__ wins, const int32_t* __restrict__ ccol,
                              int32_t* __restrict__ cursor, int4* __restrict__ tasks, unsigned long long* alg) {
    unsigned long long bytes = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
        const int4 win = wins[i];
        if (!FILL) bytes += 8ull * (((unsigned long long)win.z * win.w + 63) >> 6);   // SPEC-layout (algorithmic) bytes
        const int ya0 = max(win.x, g.r_lo), yb0 = min(win.x + win.z, g.r_hi);
        if (ya0 >= yb0) continue;
        const int tx = (ccol[i] / a.bsize) / g.TX;
        const int nwr = win_nwr(win.y, win.w);
        for (int s = (ya0 - g.r_lo) / g.SH; s <= (yb0 - 1 - g.r_lo) / g.SH; ++s) {
            const int tile = s * g.ntx + tx;
            if (!FILL) { atomicAdd(cursor + tile, 1); continue; }
            int s0, s1, wx0, pw;
            strip_tile_box(a, g, tile, &s0, &s1, &wx0, &pw);
            const int ya = max(ya0, s0), yb = min(yb0, s1);
            const int k = atomicAdd(cursor + tile, 1);
            tasks[k] = make_int4((int)i, (ya - win.x) * nwr, (ya - s0) * pw + (win.y >> 6) - wx0,
                                 ((yb - ya) * nwr) | (nwr << 20));
        }
    }
    if (!FILL) {
        for (int o = 16; o; o >>= 1) bytes += __shfl_down_sync(kFull, bytes, o);
        if ((threadIdx.x & 31) == 0 && bytes) atomicAdd(alg, bytes);
    }
}

template <typename G>
__global__ void k_zero_gains(const SiteState* st, G* __restrict__ gain, int64_t n) {
    if (st && (st->done || st->finish)) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        gain[i] = 0;
}

__device__ __forceinline__ void gain_add(int32_t* g, int v) { atomicAdd(g, v); }
__device__ __forceinline__ void gain_add(int64_t* g, int v) {
    atomicAdd((unsigned long long*)g, (unsigned long long)(long long)v);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
// arm the barrier with the copy's byte count and start the copy (one lane)
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n @!p bra W;\n}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

template <typename G>
__global__ void __launch_bounds__(kStripThreads) k_gain_strips(SiteArgs a, StripGeo geo, const SiteState* st,
                                                              const uint64_t* __restrict__ words,
                                                              const uint64_t* __restrict__ cum,
                                                              const int32_t* __restrict__ tstart,
                                                              const int4* __restrict__ tasks,
                                                              G* __restrict__ gain,
                                                              unsigned long long* __restrict__ counters,
                                                              unsigned long long alg_bytes, int tile_words, int SW) {
    if (st && (st->done || st->finish)) return;
    extern __shared__ __align__(16) uint64_t s_cum[];   // cum tile (tile_words, even), then the staging rings
    __shared__ __align__(8) uint64_t s_bar[kStripThreads / 32][kStripSlots];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int W = kStripThreads / 32, S = kStripSlots;
    uint64_t* ring = s_cum + tile_words + (int64_t)warp * S * SW;
    const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
    const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(&s_bar[warp][0]);
    if (lane == 0)
        for (int k = 0; k < S; ++k) mbar_init(bar_s + 8 * k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    if (counters && blockIdx.x == 0 && tid == 0) atomicAdd(counters + kSiteBytes, alg_bytes);
    uint32_t phase = 0;   // bit k: parity of slot k's next completion
    int head = 0;         // oldest slot in flight
    const int wpr = (int)a.wpr;
    for (int tile = blockIdx.x; tile < geo.nstrips * geo.ntx; tile += gridDim.x) {
        const int t0 = tstart[tile], t1 = tstart[tile + 1];
        if (t0 == t1) continue;
        int s0, s1, wx0, pw;
        strip_tile_box(a, geo, tile, &s0, &s1, &wx0, &pw);
        for (int t = tid; t < (s1 - s0) * pw; t += kStripThreads) {
            const int y = t / pw, x = t - y * pw;
            s_cum[t] = __ldg(cum + (int64_t)(s0 + y) * wpr + wx0 + x);
        }
        __syncthreads();
        int4 fd = make_int4(0, 0, 0, 0);   // this lane's fetched task
        int fbase = t0 + warp, fcur = 32, fn = 0;   // lane l of a fetch: task fbase + W*l
        int si = 0, scb = 0, snwr = 1, soff = 0, snw = 0;   // slot info held by lane k
        int inflight = 0;
        for (;;) {
            while (inflight < S) {   // producer: keep S copies in flight
                if (fcur >= fn) {
                    if (fbase >= t1) break;
                    fn = min(32, (t1 - fbase + W - 1) / W);
                    if (lane < fn) fd = __ldg(tasks + fbase + W * lane);
                    fbase += W * 32;
                    fcur = 0;
                }
                const int j = fcur++;
                const int ij = __shfl_sync(kFull, fd.x, j), fwj = __shfl_sync(kFull, fd.y, j);
                const int cbj = __shfl_sync(kFull, fd.z, j), pk = __shfl_sync(kFull, fd.w, j);
                const int nwj = pk & 0xfffff;
                const int64_t src = (int64_t)ij * a.stride + fwj;
                const int64_t a0 = src & ~(int64_t)1;
                const int off = (int)(src - a0), span = (off + nwj + 1) & ~1;
                const int slot = (head + inflight) & (S - 1);
                if (lane == 0) bulk_load(ring_s + 8u * slot * SW, words + a0, 8u * span, bar_s + 8 * slot);
                if (lane == slot) { si = ij; scb = cbj; snwr = pk >> 20; soff = off; snw = nwj; }
                ++inflight;
            }
            if (inflight == 0) break;
            const int slot = head;   // consumer: the oldest slot
            const int ij = __shfl_sync(kFull, si, slot), cbj = __shfl_sync(kFull, scb, slot);
            const int nwrj = __shfl_sync(kFull, snwr, slot), offj = __shfl_sync(kFull, soff, slot);
            const int nwj = __shfl_sync(kFull, snw, slot);
            mbar_wait(bar_s + 8 * slot, (phase >> slot) & 1u);
            phase ^= 1u << slot;
            const uint64_t* v = ring + slot * SW + offj;
            const uint64_t* cr = s_cum + cbj;
            int y = lane / nwrj, b = lane - y * nwrj;
            const int dy = 32 / nwrj, db = 32 - dy * nwrj;
            int acc = 0;
            for (int t = lane; t < nwj; t += 32) {
                acc += __popcll(v[t] & ~cr[y * pw + b]);
                y += dy; b += db;
                if (b >= nwrj) { b -= nwrj; ++y; }
            }
            acc = __reduce_add_sync(kFull, acc);
            if (lane == 0 && acc) gain_add(gain + ij, acc);
            __syncwarp();
            head = (head + 1) & (S - 1);
            --inflight;
        }
        __syncthreads();
    }
}

// ---- layout conversion: SPEC dense rows <-> cum-aligned rows ------------------------
__global__ void k_aligned_to_dense(const uint64_t* __restrict__ al, int64_t astride, const int4* __restrict__ wins,
                                   int64_t count, uint64_t* __restrict__ dense, int64_t dstride) {
    const int64_t total = count * dstride;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / dstride;
        const int j = (int)(t - i * dstride);
        const int4 win = wins[i];
        const int w = win.w, nbits = win.z * w, nwr = win_nwr(win.y, w);
        uint64_t out = 0;
        if (64 * j < nbits) {
            const uint64_t* v = al + i * astride;
            int bit0 = 64 * j, rem = min(64, nbits - bit0), pos = 0;
            int y = bit0 / w, x = bit0 - y * w;
            while (rem > 0) {
                const int len = min(rem, w - x);
                const int col = (win.y & 63) + x;            // bit position inside the aligned row
                const int wo = col >> 6, sh = col & 63;
                const uint64_t* row = v + (int64_t)y * nwr;
                uint64_t seg = row[wo] >> sh;
                if (sh && wo + 1 < nwr) seg |= row[wo + 1] << (64 - sh);
                if (len < 64) seg &= (1ull << len) - 1;
                out |= seg << pos;
                pos += len; rem -= len; ++y; x = 0;
            }
        }
        dense[i * dstride + j] = out;
    }
}

__global__ void k_dense_to_aligned(const uint64_t* __restrict__ dense, int64_t dstride, const int4* __restrict__ wins,
                                   int64_t count, uint64_t* __restrict__ al, int64_t astride) {
    const int64_t total = count * astride;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / astride;
        const int k = (int)(t - i * astride);
        const int4 win = wins[i];
        const int w = win.w, nwr = win_nwr(win.y, w);
        uint64_t out = 0;
        if (k < win.z * nwr) {
            const int y = k / nwr, b = k - y * nwr;
            const int base = win.y & ~63;                  // column of bit 0 of word 0
            const int cl = max(win.y, base + 64 * b), ch = min(win.y + w - 1, base + 64 * b + 63);
            if (cl <= ch) {
                const uint64_t* dv = dense + i * dstride;
                const int len = ch - cl + 1;
                const long long off = (long long)y * w + (cl - win.y);
                const int64_t wd = off >> 6;
                const int sh = (int)(off & 63);
                uint64_t seg = dv[wd] >> sh;
                if (sh && 64 - sh < len) seg |= dv[wd + 1] << (64 - sh);
                if (len < 64) seg &= (1ull << len) - 1;
                out = seg << (cl - base - 64 * b);
            }
        }
        al[i * astride + k] = out;
    }
}

__global__ void k_dense_to_padded(const uint64_t* __restrict__ dense, uint64_t* __restrict__ pad, int64_t nrows,
                                  int64_t ncols, int64_t wpr) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nrows * wpr; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t y = t / wpr, wi = t - y * wpr;
        const int64_t off = y * ncols + wi * 64;
        const int64_t w = off >> 6;
        const int s = (int)(off & 63);
        uint64_t v = dense[w] >> s;
        if (s) v |= dense[w + 1] << (64 - s);
        const int64_t valid = min((int64_t)64, ncols - wi * 64);
        if (valid < 64) v &= (1ull << valid) - 1;
        pad[t] = v;
    }
}

// pad is indexed by global row; rows outside [cr0, cr1) read as zero
// dense words [t0, t1) of the whole grid are written to dense[0 .. t1-t0)
__global__ void k_padded_to_dense(const uint64_t* __restrict__ pad, uint64_t* __restrict__ dense, int64_t nrows,
                                  int64_t ncols, int64_t wpr, int64_t cr0, int64_t cr1, int64_t t0, int64_t t1) {
    const int64_t total = nrows * ncols;
    for (int64_t t = t0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < t1; t += (int64_t)gridDim.x * blockDim.x) {
        uint64_t v = 0;
        const int64_t b0 = t * 64, b1 = min(b0 + 64, total);
        int64_t b = b0;
        while (b < b1) {   // walk the (at most a few) row segments covered by this dense word
            const int64_t y = b / ncols, x = b - y * ncols;
            const int64_t len = min(b1 - b, ncols - x);
            const int64_t pw = x >> 6;
            const int s = (int)(x & 63);
            uint64_t seg = 0;
            if (y >= cr0 && y < cr1) {
                seg = pad[y * wpr + pw] >> s;
                if (s && pw + 1 < wpr) seg |= pad[y * wpr + pw + 1] << (64 - s);
            }
            if (len < 64) seg &= (1ull << len) - 1;
            v |= seg << (b - b0);
            b += len;
        }
        dense[t - t0] = v;
    }
}

SiteArgs make_args(txs_ctx* c, const txs_params& p) {
    SiteArgs a;
    a.nrows = (int)c->nrows; a.ncols = (int)c->ncols; a.R = c->vs_roi;
    a.bsize = std::max(1, c->vs_roi);
    a.nbx = (int)((c->ncols + a.bsize - 1) / a.bsize);
    a.nby = (int)((c->nrows + a.bsize - 1) / a.bsize);
    a.wpr = (c->ncols + 63) / 64;
    a.n = c->vs_n;
    a.stride = c->vs_stride;
    a.max_sel = p.max_selected;
    a.target = p.target_coverage;
    a.total = (double)c->nrows * (double)c->ncols;
    a.cr0 = (int)c->cum_r0; a.cr1 = (int)c->cum_r1;
    a.dpitch = (int)c->dpitch;
    a.prof = (getenv("TXS_SITE_PROFILE") ? 1 : 0) | (getenv("TXS_GAIN_FOLD") ? 2 : 0);
    return a;
}

// accumulate the device time between ev_r0 and ev_r1 (stream already synced)
static void add_round_time(txs_ctx* c) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c->ev_r0, c->ev_r1) == cudaSuccess) c->stats.ms_site_rounds += ms;
}

int blocks_for(int64_t work, int per_block, int cap) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((work + per_block - 1) / per_block, cap));
}

// Full gain pass (popc(v_i & ~cum) for every candidate): bucket-tiled when the
// buckets exist (SITE rounds), hold >= 64 candidates on average and the
// bucket's cum region fits two CTAs per SM (roi <= ~280) -- measured: C5 (244
// per bucket) 4.26 -> 4.97 TB/s; C2 (39) and C3 (5) stream faster with
// k_gain_full, which reads each candidate's cum words from L2.
static bool gain_tiled(const SiteArgs& a, bool buckets, size_t* smem_out) {
    const int64_t rows = (int64_t)a.bsize + 2 * a.R;
    const int64_t pw = (a.bsize + 2 * (int64_t)a.R + 63) / 64 + 1;
    const size_t smem = sizeof(uint64_t) * (size_t)(rows * pw);
    const bool dense = a.n >= 64 * (int64_t)a.nbx * a.nby;
    *smem_out = smem;
    return buckets && dense && smem <= 110 * 1024 && !getenv("TXS_GAIN_REG");
}

// Tile of k_gain_strips: SH rows (TXS_STRIP_ROWS, default 32, <= 128) x TX
// buckets (TXS_STRIP_TX, default 8); the staging ring slot holds the longest
// task (SH window rows, even).  0 when the shared memory would pass 110 KB.
struct StripShape {
    int sh, tx, tile_words, sw;
    size_t smem;
};
static int strip_rows(const SiteArgs& a, StripShape* sp) {
    int sh = 32, t = 8;
    if (const char* e = getenv("TXS_STRIP_ROWS")) sh = std::min(1 << 12, std::max(1, atoi(e)));
    if (const char* e = getenv("TXS_STRIP_TX")) t = std::max(1, atoi(e));
    const int64_t pw = ((int64_t)t * a.bsize + 2 * (int64_t)a.R + 63) / 64 + 2;
    const int64_t nwr_max = (2 * (int64_t)a.R + 63) / 64 + 1;
    const int64_t tile_words = (pw * sh + 1) & ~(int64_t)1;
    const int64_t sw = (std::min<int64_t>(sh, 2 * (int64_t)a.R + 1) * nwr_max + 3) & ~(int64_t)1;
    const int64_t bytes = 8 * (tile_words + (int64_t)(kStripThreads / 32) * kStripSlots * sw);
    if (bytes > 110 * 1024 || nwr_max >= 4096 || sw > (1 << 20)) return 0;
    sp->sh = sh; sp->tx = t; sp->tile_words = (int)tile_words; sp->sw = (int)sw; sp->smem = (size_t)bytes;
    return sh;
}

static StripGeo strip_geo(const SiteArgs& a, const StripShape& sp) {
    StripGeo g;
    g.SH = sp.sh; g.TX = sp.tx;
    g.r_lo = std::max(0, a.cr0); g.r_hi = std::min(a.nrows, a.cr1);
    g.nstrips = std::max(0, (g.r_hi - g.r_lo + g.SH - 1) / g.SH);
    g.ntx = (a.nbx + g.TX - 1) / g.TX;
    return g;
}

// the task list of the current candidate set for this shape (count, scan, fill)
static txs_status build_strip_tasks(txs_ctx* c, const SiteArgs& a, const StripShape& sp) {
    const StripGeo g = strip_geo(a, sp);
    const int64_t tiles = (int64_t)g.nstrips * g.ntx;
    const int64_t cap = a.n * ((2 * (int64_t)a.R + 1 + g.SH - 1) / g.SH + 1);
    const int64_t alg_at = (2 * (tiles + 1) + 1) & ~(int64_t)1;   // u64 slot after the two int arrays
    if (ensure(c, "site", (void**)&c->d_strip_start, &c->strip_start_cap, sizeof(int32_t) * (size_t)(alg_at + 2)) != TXS_OK ||
        ensure(c, "site", (void**)&c->d_strip_tasks, &c->strip_tasks_cap, sizeof(int4) * (size_t)std::max<int64_t>(1, cap)) != TXS_OK)
        return TXS_ERR_OUT_OF_MEMORY;
    if (cap > INT32_MAX) return fail(c, TXS_ERR_RANGE, "site", "strip task list too long");
    int32_t* start = c->d_strip_start;
    int32_t* cursor = c->d_strip_start + tiles + 1;
    unsigned long long* alg = (unsigned long long*)(c->d_strip_start + alg_at);
    TXS_CUDA(c, "site", cudaMemsetAsync(cursor, 0, sizeof(int32_t) * (size_t)(tiles + 1), c->stream));
    TXS_CUDA(c, "site", cudaMemsetAsync(alg, 0, sizeof(unsigned long long), c->stream));
    const int blocks = blocks_for(a.n, 256, c->num_sms * 8);
    k_strip_tasks<false><<<blocks, 256, 0, c->stream>>>(a, g, c->d_win, c->d_ccol, cursor, nullptr, alg);
    TXS_LAUNCHED(c, "site");
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cursor, start, (int)(tiles + 1), c->stream);
    void* tmp = nullptr;
    TXS_CUDA(c, "site", cudaMallocAsync(&tmp, tb, c->stream));
    TXS_CUDA(c, "site", cub::DeviceScan::ExclusiveSum(tmp, tb, cursor, start, (int)(tiles + 1), c->stream));
    TXS_CUDA(c, "site", cudaFreeAsync(tmp, c->stream));
    TXS_CUDA(c, "site", cudaMemcpyAsync(cursor, start, sizeof(int32_t) * (size_t)(tiles + 1), cudaMemcpyDeviceToDevice, c->stream));
    k_strip_tasks<true><<<blocks, 256, 0, c->stream>>>(a, g, c->d_win, c->d_ccol, cursor, c->d_strip_tasks, nullptr);
    TXS_LAUNCHED(c, "site");
    TXS_CUDA(c, "site", cudaMemcpyAsync(&c->site_alg_bytes, alg, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    TXS_CUDA(c, "site", cudaStreamSynchronize(c->stream));
    return TXS_OK;
}

// The t8 shadow (tile words of every viewshed + the tile cum) for the current
// candidate set; built once per viewshed set (t8_valid), the tile cum zeroed or
// converted from the row-padded cum by the caller.  false when HBM is short.
static bool t8_fits(txs_ctx* c, const SiteArgs& a) {
    if (c->t8_valid) return true;
    const size_t need = sizeof(uint64_t) * (size_t)(std::max<int64_t>(1, a.n) * t8_stride(a.R));
    if (c->t8_words_cap >= need) return true;
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return false;
    return fr > need + (need >> 3) + ((size_t)1 << 30);
}

static txs_status build_t8(txs_ctx* c, const SiteArgs& a) {
    const int th = (a.nrows + 7) >> 3, tw = (a.ncols + 7) >> 3;
    if (ensure(c, "site", (void**)&c->d_t8_cum, &c->t8_cum_cap, sizeof(uint64_t) * (size_t)((int64_t)th * tw + 1)) != TXS_OK)
        return TXS_ERR_OUT_OF_MEMORY;
    if (c->t8_valid) return TXS_OK;
    const int64_t ts = t8_stride(a.R);
    if (ensure(c, "site", (void**)&c->d_t8_words, &c->t8_words_cap, sizeof(uint64_t) * (size_t)(std::max<int64_t>(1, a.n) * ts)) != TXS_OK ||
        ensure(c, "site", (void**)&c->d_t8_win, &c->t8_win_cap, sizeof(int4) * (size_t)std::max<int64_t>(1, a.n)) != TXS_OK)
        return TXS_ERR_OUT_OF_MEMORY;
    if (a.n > 0) {
        k_words_to_t8<<<blocks_for(a.n * 32, 256, c->num_sms * 16), 256, 0, c->stream>>>(a.n, c->d_win, c->d_words, a.stride,
                                                                                       c->d_t8_words, ts, c->d_t8_win);
        TXS_LAUNCHED(c, "site");
    }
    c->t8_valid = true;
    return TXS_OK;
}

// TXS_GAIN_PASS=full|tiled|strips|t8 overrides the measured choice (A/B only;
// k_gain_strips measured slower than k_gain_full at c2-c4 and equal to
// k_gain_tiled at c5, profiles/README.md).  Kinds: 0 cum-aligned rows, 1
// bucket-tiled cum in shared memory, 2 strips, 3 the 8x8-tile shadow.
static int gain_pass_kind(txs_ctx* c, const SiteArgs& a, bool buckets, size_t* smem, StripShape* sp) {
    size_t ts = 0;
    const bool tiled = gain_tiled(a, buckets, &ts);
    const int rows = buckets ? strip_rows(a, sp) : 0;
    // t8: SITE rounds on a whole-grid cum only (the shadow is per viewshed set)
    const bool t8ok = buckets && a.cr0 == 0 && a.cr1 == a.nrows && a.n > 0 && t8_fits(c, a);
    int kind = t8ok ? 3 : (tiled ? 1 : 0);   // measured: t8 >= tiled at c5 (5.41 vs 5.15 TB/s), >= rows at c2-c4
    if (const char* e = getenv("TXS_GAIN_PASS")) {
        if (!strcmp(e, "full")) kind = 0;
        else if (!strcmp(e, "tiled") && buckets) kind = 1;
        else if (!strcmp(e, "strips") && rows > 0) kind = 2;
        else if (!strcmp(e, "t8") && t8ok) kind = 3;
    }
    *smem = kind == 1 ? ts : kind == 2 ? sp->smem : 0;
    return kind;
}

// CTAs per SM of the per-candidate passes' grid (TXS_GAIN_GRID, A/B).  Five
// 256-thread CTAs are resident per SM: 16 per SM made 3.2 waves with an idle
// tail; measured 5 / 16 / 64 / 256 per SM, TB/s: c3 t8 4.09 / 4.10 / 4.34 /
// 4.21, c4 rows 3.44 / 3.32 / 3.65 / 3.54, c5 t8 5.17 / 4.94 / 5.41 / 5.46
static int gain_grid_mult() {
    const char* e = getenv("TXS_GAIN_GRID");
    return e ? std::max(1, atoi(e)) : 64;
}

// t8 pass: candidates of look-ahead for the tile-cum L2 prefetch (< 0 = none):
// only when the tile cum cannot stay in L2 between passes (c4: 269 MB);
// TXS_GAIN_PF_AHEAD overrides (A/B)
static int64_t t8_prefetch_ahead(txs_ctx*, const SiteArgs& a) {
    if (const char* e = getenv("TXS_GAIN_PF_AHEAD")) return std::max<long long>(-1, atoll(e));
    const int64_t cum_bytes = (int64_t)((a.nrows + 7) >> 3) * ((a.ncols + 7) >> 3) * 8;
    return cum_bytes > (int64_t)96 << 20 ? 0 : -1;
}

template <typename G>
static void launch_gain_pass(txs_ctx* c, const SiteArgs& a, const SiteState* st, const uint64_t* cum, G* gain,
                             unsigned long long* counters, bool buckets) {
    size_t smem = 0;
    StripShape sp{};
    const int kind = gain_pass_kind(c, a, buckets, &smem, &sp);
    if (kind == 3) {   // `cum` is not read: the tile cum shadows it (build_t8 / k_commit_t8 / k_cum_to_t8)
        SiteArgs t = a;
        t.stride = t8_stride(a.R);
        t.wpr = (a.ncols + 7) >> 3;
        k_gain_full<G, true><<<blocks_for(a.n * 32, 256, c->num_sms * gain_grid_mult()), 256, 0, c->stream>>>(
            t, st, c->d_t8_win, c->d_t8_words, c->d_t8_cum, gain, counters, c->d_win, t8_prefetch_ahead(c, a));
    } else if (kind == 2) {
        k_zero_gains<G><<<blocks_for(a.n, 256, c->num_sms * 4), 256, 0, c->stream>>>(st, gain, a.n);
        auto kern = k_gain_strips<G>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const StripGeo g = strip_geo(a, sp);
        const int64_t tiles = (int64_t)g.nstrips * g.ntx;
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kStripThreads, smem);
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)c->num_sms * std::max(1, per_sm)));
        kern<<<grid, kStripThreads, smem, c->stream>>>(a, g, st, c->d_words, cum, c->d_strip_start, c->d_strip_tasks,
                                                       gain, counters, c->site_alg_bytes, sp.tile_words, sp.sw);
    } else if (kind == 1) {
        auto kern = k_gain_tiled<G>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int64_t nbk = (int64_t)a.nbx * a.nby;
        const int grid = (int)std::min<int64_t>(nbk, (int64_t)c->num_sms * 2 * 8);
        kern<<<grid, kTiledThreads, smem, c->stream>>>(a, st, c->d_win, c->d_words, cum, c->d_bucket_start,
                                                       c->d_bucket_items, gain, counters);
    } else {
        k_gain_full<G, false><<<blocks_for(a.n * 32, 256, c->num_sms * gain_grid_mult()), 256, 0, c->stream>>>(
            a, st, c->d_win, c->d_words, cum, gain, counters, nullptr, -1);
    }
}

// ---- batched exact greedy (site_mode 0): every local maximum per round ------------------
// The greedy sequence is serial only along chains of overlapping windows.  If
// candidate X has the largest key (gain << 32 | ~index) among all candidates
// whose windows overlap X's, no overlapping candidate can be picked before X
// (their keys only fall and X's stays until something overlapping is picked),
// so X WILL be the greedy pick with exactly its current gain once every
// larger key elsewhere is used up -- and committing it now changes nothing
// for the picks in between: they do not overlap X, and X's neighbours, whose
// gains drop early, stay below X.  Successive greedy picks have strictly
// falling keys, so the greedy ORDER is the committed picks sorted by key.
// Per round: (1) k_batch_bmax: per neighbour bucket (side R) the best key, the
// global best kappa and a gain histogram; (2) k_batch_decide: the stop test on
// the known prefix (logged picks with key > kappa) and the rank threshold;
// (3) k_batch_winners: every bucket champion that beats the champions of all
// buckets within 2R of it (a superset of the overlapping candidates) is a
// winner -- winners are pairwise non-overlapping; (4) k_batch_delta: each
// winner's newly covered bits D = v_w & ~cum go to its own delta window, into
// cum and its key into the log; (5) k_batch_update: gain_z -= popc(v_z & D_w)
// for the winners' neighbours.  The run ends once the stop rule (decision D9)
// fires inside the known prefix.  Winners whose key turns out to lie past the
// stop were committed needlessly: the rank threshold (only candidates among
// the `remaining` largest current gains may win, besides the global maximum)
// keeps them to one histogram bin; the step list is cut at the stop and the
// cum rebuilt from the kept picks.  c3: 4096 serial rounds -> tens of rounds.
struct BatchState {
    unsigned long long kappa_acc;   // running max of the uncommitted keys (k_batch_bmax)
    unsigned long long kappa;       // the round's global max key
    long long logn;                 // committed picks in the log
    long long nvalid, svalid;       // logged picks with key > kappa: count, gain sum
    int nx;                         // winners of the current round besides the global maximum (may exceed cap - 1)
    int cap;                        // winner slots per round
    int tau;                        // gain threshold of the winners other than the global maximum
    int done, rounds;
};
constexpr int kHistBins = 4096;
constexpr int kBatchUpdThreads = 128;
constexpr int kBatchMaxRanges = 8;

__device__ __forceinline__ int batch_nw(const BatchState* S) { return 1 + min(S->nx, S->cap - 1); }

__global__ void __launch_bounds__(256) k_batch_bmax(SiteArgs a, BatchState* S, const int32_t* __restrict__ bstart,
                                                    const int32_t* __restrict__ items, const int32_t* __restrict__ gain,
                                                    unsigned long long* __restrict__ bmax, unsigned int* __restrict__ hist,
                                                    int hshift) {
    if (S->done) return;
    __shared__ unsigned int s_hist[kHistBins];
    const bool use_hist = a.max_sel > 0;
    if (use_hist) {
        for (int k = threadIdx.x; k < kHistBins; k += blockDim.x) s_hist[k] = 0u;
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    const int64_t nbk = (int64_t)a.nbx * a.nby, nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long cta_best = 0ull;
    for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nbk; b += nwarps) {
        const int s0 = bstart[b], s1 = bstart[b + 1];
        unsigned long long best = 0ull;
        for (int s = s0 + lane; s < s1; s += 32) {
            const int i = items[s], g = gain[i];
            if (g > 0) {
                best = umax64(best, ((unsigned long long)(uint32_t)g << 32) | (0xffffffffull - (uint64_t)(uint32_t)i));
                if (use_hist) atomicAdd(&s_hist[min(g >> hshift, kHistBins - 1)], 1u);
            }
        }
        for (int o = 16; o; o >>= 1) best = umax64(best, __shfl_xor_sync(kFull, best, o));
        if (lane == 0) bmax[b] = best;
        cta_best = umax64(cta_best, best);
    }
    if (lane == 0 && cta_best) atomicMax(&S->kappa_acc, cta_best);
    if (use_hist) {
        __syncthreads();
        for (int k = threadIdx.x; k < kHistBins; k += blockDim.x) {
            const unsigned int h = s_hist[k];
            if (h) atomicAdd(&hist[k], h);
        }
    }
}

// one CTA: the stop test on the known prefix, the next rank threshold, resets
__global__ void __launch_bounds__(1024) k_batch_decide(SiteArgs a, BatchState* S, const unsigned long long* __restrict__ log,
                                                       unsigned int* __restrict__ hist, int hshift) {
    if (S->done) return;
    __shared__ long long s_cnt[32], s_sum[32];
    __shared__ unsigned int s_h[32];
    __shared__ int s_tau;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long logn = S->logn + (S->rounds > 0 ? batch_nw(S) : 0);   // the previous round's winners are in the log now
    const unsigned long long kappa = S->kappa_acc;
    long long cnt = 0, sum = 0;
    for (long long k = tid; k < logn; k += blockDim.x) {
        const unsigned long long key = log[k];
        if (key > kappa) { ++cnt; sum += (long long)(key >> 32); }
    }
    for (int o = 16; o; o >>= 1) { cnt += __shfl_xor_sync(kFull, cnt, o); sum += __shfl_xor_sync(kFull, sum, o); }
    if (lane == 0) { s_cnt[warp] = cnt; s_sum[warp] = sum; }
    // counts of the gain histogram from the top bin down: thread t owns bins [top, top + 3], top = 4 (1023 - t)
    const int top = (kHistBins / 4 - 1 - tid) * 4;
    const unsigned int h3 = hist[top + 3], h2 = hist[top + 2], h1 = hist[top + 1], h0 = hist[top];
    const unsigned int mine = h0 + h1 + h2 + h3;
    unsigned int incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned int t = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_h[warp] = incl;
    if (tid == 0) s_tau = 1;
    __syncthreads();
    cnt = 0; sum = 0;
    for (int q = 0; q < 32; ++q) { cnt += s_cnt[q]; sum += s_sum[q]; }
    unsigned int before = 0;   // candidates in higher bins than this thread's
    for (int q = 0; q < warp; ++q) before += s_h[q];
    before += incl - mine;
    const long long remaining = a.max_sel > 0 ? a.max_sel - cnt : (long long)1 << 40;
    // the bin where the count from the top reaches `remaining`: its lower edge is the threshold
    if (remaining > 0 && (long long)before < remaining && (long long)before + mine >= remaining) {
        long long c2 = before;
        int bin = top;
        const unsigned int hh[4] = {h3, h2, h1, h0};
        for (int k = 0; k < 4; ++k) {
            c2 += hh[k];
            if (c2 >= remaining) { bin = top + 3 - k; break; }
        }
        s_tau = max(1, bin << hshift);
    }
    __syncthreads();
    for (int k = tid; k < kHistBins; k += blockDim.x) hist[k] = 0u;
    if (tid == 0) {
        const long long g = (long long)(kappa >> 32);
        const bool stop = (a.max_sel > 0 && cnt >= a.max_sel) || (double)sum / a.total >= a.target || g <= 0;
        S->kappa = kappa;
        S->kappa_acc = 0ull;
        S->logn = logn;
        S->nvalid = cnt;
        S->svalid = sum;
        S->nx = 0;
        S->tau = s_tau;
        S->rounds += 1;
        if (stop) S->done = 1;
    }
}

// slot 0 is the global maximum's (always a winner: progress every round)
__global__ void k_batch_winners(SiteArgs a, BatchState* S, const unsigned long long* __restrict__ bmax,
                                const int32_t* __restrict__ crow, const int32_t* __restrict__ ccol,
                                int32_t* __restrict__ wl, unsigned long long* __restrict__ wkey) {
    if (S->done) return;
    const int64_t nbk = (int64_t)a.nbx * a.nby;
    const unsigned long long kappa = S->kappa;
    const int tau = S->tau, cap = S->cap;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nbk; b += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = bmax[b];
        if (!key) continue;
        if ((int)(key >> 32) < tau && key != kappa) continue;
        const int i = (int)(0xffffffffull - (key & 0xffffffffull));
        const int r = crow[i], c = ccol[i];
        const int by0 = max(0, (r - 2 * a.R) / a.bsize), by1 = min(a.nby - 1, (r + 2 * a.R) / a.bsize);
        const int bx0 = max(0, (c - 2 * a.R) / a.bsize), bx1 = min(a.nbx - 1, (c + 2 * a.R) / a.bsize);
        bool top = true;
        for (int by = by0; by <= by1 && top; ++by)
            for (int bx = bx0; bx <= bx1; ++bx)
                if (bmax[(int64_t)by * a.nbx + bx] > key) { top = false; break; }
        if (!top) continue;
        int slot = 0;
        if (key != kappa) {
            slot = 1 + atomicAdd(&S->nx, 1);
            if (slot >= cap) continue;   // no slot this round: it wins again next round
        }
        wl[slot] = i;
        wkey[slot] = key;
    }
}

// one CTA per winner: D = v_w & ~cum into the winner's delta window (+ per-row spans of its
// non-zero words), cum |= D, key into the log.  Winners' windows are disjoint, but two may
// share a cum word at their edges: the bits each one tests and sets are its own.
__global__ void __launch_bounds__(256) k_batch_delta(SiteArgs a, const BatchState* S, const int32_t* __restrict__ wl,
                                                     const unsigned long long* __restrict__ wkey,
                                                     const int4* __restrict__ wins, const uint64_t* __restrict__ words,
                                                     uint64_t* cum, uint64_t* __restrict__ dwin, int2* __restrict__ dspan,
                                                     unsigned long long* __restrict__ log) {
    if (S->done) return;
    const int nw = batch_nw(S), side = 2 * a.R + 1;
    for (int w = blockIdx.x; w < nw; w += gridDim.x) {
        const int X = wl[w];
        const int4 wx = wins[X];
        const uint64_t* v = words + (int64_t)X * a.stride;
        uint64_t* dw = dwin + (int64_t)w * side * a.dpitch;
        int2* ds = dspan + (int64_t)w * side;
        const int nwr = win_nwr(wx.y, wx.w), wlo = wx.y >> 6;
        for (int y = threadIdx.x; y < side; y += blockDim.x) ds[y] = make_int2(0x7fffffff, -1);
        __syncthreads();
        for (int t = threadIdx.x; t < wx.z * nwr; t += blockDim.x) {
            const int y = t / nwr, b = t - y * nwr;
            const int64_t o = (int64_t)(wx.x + y) * a.wpr + wlo + b;
            const uint64_t d = v[t] & ~__ldcg(cum + o);
            dw[(int64_t)y * a.dpitch + b] = d;
            if (d) {
                atomicOr((unsigned long long*)(cum + o), (unsigned long long)d);
                atomicMin(&ds[y].x, b);
                atomicMax(&ds[y].y, b);
            }
        }
        if (threadIdx.x == 0) log[S->logn + w] = wkey[w];
        __syncthreads();
    }
}

// virtual CTA (winner w, slot x of XS): the neighbours f = x, x + XS, ... of winner w.  XS shrinks as
// the winners grow so that the grid holds about one virtual CTA per real one.
__global__ void __launch_bounds__(kBatchUpdThreads) k_batch_update(SiteArgs a, const BatchState* S,
                                                                    const int32_t* __restrict__ wl,
                                                                    const int32_t* __restrict__ crow,
                                                                    const int32_t* __restrict__ ccol,
                                                                    const int32_t* __restrict__ bstart,
                                                                    const int32_t* __restrict__ items,
                                                                    const int4* __restrict__ wins,
                                                                    const uint64_t* __restrict__ words,
                                                                    const uint64_t* __restrict__ dwin,
                                                                    const int2* __restrict__ dspan,
                                                                    int32_t* __restrict__ gain,
                                                                    unsigned long long* __restrict__ counters) {
    if (S->done) return;
    __shared__ int s_red[kBatchUpdThreads / 32], s_cnt[kBatchUpdThreads / 32], s_start[kBatchMaxRanges], s_len[kBatchMaxRanges],
        s_pref[kBatchMaxRanges + 1];
    const int nw = batch_nw(S), side = 2 * a.R + 1;
    const int XS = max(1, min(64, (int)gridDim.x / nw));
    unsigned long long bytes = 0;
    for (int64_t vf = blockIdx.x; vf < (int64_t)nw * XS; vf += gridDim.x) {
        const int w = (int)(vf / XS), x = (int)(vf - (int64_t)w * XS);
        const int X = wl[w];
        const int4 wx = wins[X];
        const int r = crow[X], c = ccol[X];
        const int by0 = max(0, (r - 2 * a.R) / a.bsize), by1 = min(a.nby - 1, (r + 2 * a.R) / a.bsize);
        const int bx0 = max(0, (c - 2 * a.R) / a.bsize), bx1 = min(a.nbx - 1, (c + 2 * a.R) / a.bsize);
        const int nb = min(kBatchMaxRanges, by1 - by0 + 1);
        __syncthreads();
        if (threadIdx.x < nb) {
            const int s0 = bstart[(int64_t)(by0 + threadIdx.x) * a.nbx + bx0], s1 = bstart[(int64_t)(by0 + threadIdx.x) * a.nbx + bx1 + 1];
            s_start[threadIdx.x] = s0;
            s_len[threadIdx.x] = s1 - s0;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int pref = 0;
            for (int k = 0; k < nb; ++k) { s_pref[k] = pref; pref += s_len[k]; }
            s_pref[nb] = pref;
        }
        __syncthreads();
        bytes += update_body<true>(a, wx.x, wx.y, wx.z, wx.w, nb, s_start, s_pref, wins, words,
                                   dwin + (int64_t)w * side * a.dpitch, dspan + (int64_t)w * side, items, gain, x, XS, s_red, s_cnt);
    }
    if (threadIdx.x == 0 && bytes) atomicAdd(counters + kSiteBytes, bytes);
}

// cum |= v_w for the first `count` listed candidates (the rebuild after an over-commit)
__global__ void k_batch_rebuild(SiteArgs a, int64_t count, const int32_t* __restrict__ wl, const int4* __restrict__ wins,
                                const uint64_t* __restrict__ words, uint64_t* __restrict__ cum) {
    for (int64_t w = blockIdx.x; w < count; w += gridDim.x) {
        const int X = wl[w];
        const int4 wx = wins[X];
        const uint64_t* v = words + (int64_t)X * a.stride;
        const int nwr = win_nwr(wx.y, wx.w), wlo = wx.y >> 6;
        for (int t = threadIdx.x; t < wx.z * nwr; t += blockDim.x) {
            const uint64_t x = v[t];
            const int y = t / nwr, b = t - y * nwr;
            if (x) atomicOr((unsigned long long*)(cum + (int64_t)(wx.x + y) * a.wpr + wlo + b), (unsigned long long)x);
        }
    }
}

__global__ void k_batch_emit(int64_t count, const unsigned long long* __restrict__ sorted, const int32_t* __restrict__ crow,
                             const int32_t* __restrict__ ccol, txs_step* __restrict__ steps, int32_t* __restrict__ idx_out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = sorted[k];
        const int i = (int)(0xffffffffull - (key & 0xffffffffull));
        steps[k] = txs_step{(int64_t)i, crow[i], ccol[i], (int64_t)(key >> 32), 0.0};
        idx_out[k] = i;
    }
}

// cum over the held region rows [r0, r1) (whole grid unless sharded) + delta list
txs_status alloc_bitmaps(txs_ctx* c, int64_t r0, int64_t r1) {
    c->wpr = (c->ncols + 63) / 64;
    c->cum_r0 = r0;
    c->cum_r1 = r1;
    const size_t bytes = sizeof(uint64_t) * (size_t)((r1 - r0) * c->wpr + 1);
    if (ensure(c, "site", (void**)&c->d_cum, &c->bitmap_cap, bytes) != TXS_OK) return TXS_ERR_OUT_OF_MEMORY;
    // delta window: (2R+1) rows x dpitch words, plus per-row spans
    const int64_t side = 2 * (int64_t)std::max(1, c->vs_roi) + 1;
    c->dpitch = (side + 63) / 64 + 1;
    if (ensure(c, "site", (void**)&c->d_dwin, &c->dwin_cap, sizeof(uint64_t) * (size_t)(side * c->dpitch)) != TXS_OK ||
        ensure(c, "site", (void**)&c->d_dspan, &c->dspan_cap, sizeof(int2) * (size_t)(2 * side)) != TXS_OK)
        return TXS_ERR_OUT_OF_MEMORY;
    return TXS_OK;
}


// gains <- popcounts; CSR buckets (side roi) over the candidates' positions
txs_status init_gains_buckets(txs_ctx* c, const SiteArgs& a, void* d_scan_tmp, size_t scan_bytes) {
    const int64_t n = a.n, nbk = (int64_t)a.nbx * a.nby;
    const int sms = c->num_sms;
    if (n == 0) return TXS_OK;
    k_init_gains<<<blocks_for(n, 256, sms * 8), 256, 0, c->stream>>>(c->d_pop, c->d_gain, n);
    TXS_LAUNCHED(c, "site");
    int32_t* counts = c->d_bucket_start;            // nbk+1
    int32_t* cursor = c->d_bucket_start + nbk + 1;  // nbk+1
    TXS_CUDA(c, "site", cudaMemsetAsync(counts, 0, sizeof(int32_t) * (nbk + 1), c->stream));
    k_bucket_count<<<blocks_for(n, 256, sms * 8), 256, 0, c->stream>>>(c->d_crow, c->d_ccol, n, a.bsize, a.nbx, counts);
    TXS_LAUNCHED(c, "site");
    TXS_CUDA(c, "site", cub::DeviceScan::ExclusiveSum(d_scan_tmp, scan_bytes, counts, cursor, (int)(nbk + 1), c->stream));
    TXS_CUDA(c, "site", cudaMemcpyAsync(counts, cursor, sizeof(int32_t) * (nbk + 1), cudaMemcpyDeviceToDevice, c->stream));
    k_bucket_fill<<<blocks_for(n, 256, sms * 8), 256, 0, c->stream>>>(c->d_crow, c->d_ccol, n, a.bsize, a.nbx, cursor, c->d_bucket_items);
    TXS_LAUNCHED(c, "site");
    return TXS_OK;
}

// Batched exact greedy (kernels above): graphs of kBatchRoundsPerGraph rounds until the device
// stop flag, then the log sorted by key is the greedy order; decision D9's stop rules are
// replayed over it on the host (exactly the serial loop's tests, pick by pick).
constexpr int kBatchRoundsPerGraph = 8;

static txs_status run_site_batched(txs_ctx* c, const txs_params& p, const SiteArgs& a, txs_step* d_steps,
                                   std::vector<txs_step>& out, int32_t* stop) {
    const int64_t n = a.n, nbk = (int64_t)a.nbx * a.nby;
    const int sms = c->num_sms, side = 2 * a.R + 1;
    // winner slots per round: one per bucket at most; the delta windows are capped at 1 GB
    const int64_t dwin_words = (int64_t)side * a.dpitch;
    int64_t cap = std::min<int64_t>(nbk, std::max<int64_t>(64, ((int64_t)1 << 30) / (8 * dwin_words)));
    cap = std::max<int64_t>(1, std::min<int64_t>(cap, n));
    if (const char* e = getenv("TXS_SITE_BATCH_CAP")) cap = std::max<int64_t>(1, std::min<int64_t>(cap, atoll(e)));
    size_t sort_bytes = 0;
    cub::DeviceRadixSort::SortKeysDescending(nullptr, sort_bytes, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                             (int)n, 0, 64, c->stream);
    auto al = [](size_t x) { return (x + 255) / 256 * 256; };
    const size_t o_bmax = 0, o_hist = o_bmax + al(8 * (size_t)nbk), o_wl = o_hist + al(4 * kHistBins),
                 o_wkey = o_wl + al(4 * (size_t)cap), o_log = o_wkey + al(8 * (size_t)cap), o_sorted = o_log + al(8 * (size_t)n),
                 o_idx = o_sorted + al(8 * (size_t)n), o_sort = o_idx + al(4 * (size_t)n), o_dspan = o_sort + al(sort_bytes),
                 o_dwin = o_dspan + al(sizeof(int2) * (size_t)(cap * side)), total = o_dwin + al(8 * (size_t)(cap * dwin_words));
    if (ensure(c, "site", &c->d_batch, &c->batch_cap, total) != TXS_OK) return TXS_ERR_OUT_OF_MEMORY;
    char* base = (char*)c->d_batch;
    unsigned long long* bmax = (unsigned long long*)(base + o_bmax);
    unsigned int* hist = (unsigned int*)(base + o_hist);
    int32_t* wl = (int32_t*)(base + o_wl);
    unsigned long long* wkey = (unsigned long long*)(base + o_wkey);
    unsigned long long* log = (unsigned long long*)(base + o_log);
    unsigned long long* sorted = (unsigned long long*)(base + o_sorted);
    int32_t* idx = (int32_t*)(base + o_idx);
    int2* dspan = (int2*)(base + o_dspan);
    uint64_t* dwin = (uint64_t*)(base + o_dwin);
    static_assert(sizeof(BatchState) <= sizeof(SiteState), "BatchState lives in the SiteState buffers");
    BatchState* S = (BatchState*)c->d_state;
    BatchState* hS = (BatchState*)c->h_state;
    std::memset(hS, 0, sizeof(BatchState));
    hS->cap = (int)cap;
    TXS_CUDA(c, "site", cudaMemcpyAsync(S, hS, sizeof(BatchState), cudaMemcpyHostToDevice, c->stream));
    TXS_CUDA(c, "site", cudaMemsetAsync(hist, 0, 4 * kHistBins, c->stream));
    int hshift = 0;
    while ((((int64_t)side * side) >> hshift) >= kHistBins) ++hshift;
    const int bm_blocks = blocks_for(nbk * 32, 256, sms * 4);
    const int wn_blocks = blocks_for(nbk, 128, sms * 4);
    const int dl_blocks = (int)std::min<int64_t>(cap, sms * 8);
    int up_blocks = sms * 8;
    if (const char* e = getenv("TXS_BATCH_UPD_MULT")) up_blocks = sms * std::max(1, atoi(e));
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    TXS_CUDA(c, "site", cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    for (int r = 0; r < kBatchRoundsPerGraph; ++r) {
        k_batch_bmax<<<bm_blocks, 256, 0, c->stream>>>(a, S, c->d_bucket_start, c->d_bucket_items, c->d_gain, bmax, hist, hshift);
        k_batch_decide<<<1, 1024, 0, c->stream>>>(a, S, log, hist, hshift);
        k_batch_winners<<<wn_blocks, 128, 0, c->stream>>>(a, S, bmax, c->d_crow, c->d_ccol, wl, wkey);
        k_batch_delta<<<dl_blocks, 256, 0, c->stream>>>(a, S, wl, wkey, c->d_win, c->d_words, c->d_cum, dwin, dspan, log);
        k_batch_update<<<up_blocks, kBatchUpdThreads, 0, c->stream>>>(a, S, wl, c->d_crow, c->d_ccol, c->d_bucket_start,
                                                                      c->d_bucket_items, c->d_win, c->d_words, dwin, dspan,
                                                                      c->d_gain, c->d_counters);
    }
    cudaError_t ce = cudaStreamEndCapture(c->stream, &graph);
    if (ce != cudaSuccess) return cuda_fail(c, "site", ce);
    ce = cudaGraphInstantiate(&exec, graph, 0);
    if (ce != cudaSuccess) { cudaGraphDestroy(graph); return cuda_fail(c, "site", ce); }
    txs_status st = TXS_OK;
    int64_t graphs = 0;
    for (;;) {
        cudaEventRecord(c->ev_r0, c->stream);
        ce = cudaGraphLaunch(exec, c->stream);
        if (ce != cudaSuccess) { st = cuda_fail(c, "site", ce); break; }
        cudaEventRecord(c->ev_r1, c->stream);
        ++graphs;
        ce = cudaMemcpyAsync(hS, S, sizeof(BatchState), cudaMemcpyDeviceToHost, c->stream);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(c->stream);
        if (ce == cudaSuccess) add_round_time(c);
        if (ce != cudaSuccess) { st = cuda_fail(c, "site", ce); break; }
        if (hS->done) break;
        if (graphs * kBatchRoundsPerGraph > n + 2 * kBatchRoundsPerGraph) { st = fail(c, TXS_ERR_STATE, "site", "batched loop did not terminate"); break; }
    }
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    if (st != TXS_OK) return st;
    c->launches += graphs * kBatchRoundsPerGraph * 5;
    c->stats.site_launches += graphs * kBatchRoundsPerGraph * 5;
    const int64_t logn = hS->logn, rounds = hS->rounds;
    const unsigned long long kappa = hS->kappa;
    if (getenv("TXS_SITE_BATCH_VERBOSE"))
        fprintf(stderr, "[txs] batched SITE: %lld rounds, %lld picks logged, %lld in the known prefix\n", (long long)rounds,
                (long long)logn, (long long)hS->nvalid);
    out.clear();
    *stop = (kappa >> 32) == 0 ? (logn >= n ? TXS_STOP_EXHAUSTED : TXS_STOP_ZERO_GAIN) : TXS_STOP_ZERO_GAIN;
    int64_t kept = 0;
    if (logn > 0) {
        TXS_CUDA(c, "site", cub::DeviceRadixSort::SortKeysDescending(base + o_sort, sort_bytes, (const unsigned long long*)log, sorted,
                                                                     (int)logn, 0, 64, c->stream));
        k_batch_emit<<<blocks_for(logn, 256, sms * 4), 256, 0, c->stream>>>(logn, sorted, c->d_crow, c->d_ccol, d_steps, idx);
        TXS_LAUNCHED(c, "site");
        out.resize((size_t)logn);
        TXS_CUDA(c, "site", cudaMemcpyAsync(out.data(), d_steps, sizeof(txs_step) * logn, cudaMemcpyDeviceToHost, c->stream));
        TXS_CUDA(c, "site", cudaStreamSynchronize(c->stream));
        // D9 in the serial loop's order: a pick is made while a positive gain is left; after
        // it, target coverage is tested before the observer cap
        long long covered = 0;
        bool stopped = false;
        for (int64_t k = 0; k < logn; ++k) {
            covered += out[k].gain;
            const double cov = (double)covered / a.total;
            out[k].coverage = cov;
            kept = k + 1;
            if (cov >= a.target) { *stop = TXS_STOP_TARGET_REACHED; stopped = true; break; }
            if (a.max_sel > 0 && k + 1 >= a.max_sel) { *stop = TXS_STOP_MAX_SELECTED; stopped = true; break; }
        }
        if (!stopped && (kappa >> 32) != 0) return fail(c, TXS_ERR_STATE, "site", "batched loop ended before a stop rule");
        out.resize((size_t)kept);
        if (kept < logn) {   // picks past the stop were committed: the cum is the kept picks' union
            const size_t bm = sizeof(uint64_t) * (size_t)((c->cum_r1 - c->cum_r0) * c->wpr + 1);
            TXS_CUDA(c, "site", cudaMemsetAsync(c->d_cum, 0, bm, c->stream));
            k_batch_rebuild<<<(int)std::min<int64_t>(kept, sms * 8), 256, 0, c->stream>>>(a, kept, idx, c->d_win, c->d_words, c->d_cum);
            TXS_LAUNCHED(c, "site");
            TXS_CUDA(c, "site", cudaStreamSynchronize(c->stream));
        }
    }
    c->stats.site_iterations += kept;
    return TXS_OK;
}

}  // namespace

txs_status run_site(txs_ctx* c, const txs_params& p, std::vector<txs_step>& out, int32_t* stop) {
    TXS_CUDA(c, "site", cudaStreamSynchronize(c->stream));
    if (alloc_bitmaps(c, 0, c->nrows) != TXS_OK) return TXS_ERR_OUT_OF_MEMORY;
    const SiteArgs a = make_args(c, p);
    const int64_t n = a.n;
    uint64_t* cumv = c->d_cum;   // region starts at row 0
    if (ensure(c, "site", (void**)&c->d_gain, &c->gain_cap, sizeof(int32_t) * std::max<int64_t>(1, n)) != TXS_OK)
        return TXS_ERR_OUT_OF_MEMORY;
    const int64_t nbk = (int64_t)a.nbx * a.nby;
    if (ensure(c, "site", (void**)&c->d_bucket_start, &c->bucket_cap, sizeof(int32_t) * (nbk + 1) * 2) != TXS_OK ||
        ensure(c, "site", (void**)&c->d_bucket_items, &c->bucket_items_cap, sizeof(int32_t) * std::max<int64_t>(1, n)) != TXS_OK)
        return TXS_ERR_OUT_OF_MEMORY;
    // device step log
    txs_step* d_steps = nullptr;
    size_t scan_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int32_t*)nullptr, (int32_t*)nullptr, (int)(nbk + 1));
    const size_t steps_bytes = sizeof(txs_step) * (size_t)std::max<int64_t>(1, n);
    if (ensure(c, "site", &c->d_scratch, &c->scratch_cap, steps_bytes + scan_bytes + 256) != TXS_OK) return TXS_ERR_OUT_OF_MEMORY;
    d_steps = (txs_step*)c->d_scratch;
    void* d_scan_tmp = (char*)c->d_scratch + ((steps_bytes + 255) / 256) * 256;

    const size_t bm = sizeof(uint64_t) * (size_t)((c->cum_r1 - c->cum_r0) * c->wpr + 1);
    TXS_CUDA(c, "site", cudaMemsetAsync(c->d_cum, 0, bm, c->stream));
    TXS_CUDA(c, "site", cudaMemsetAsync(c->d_state, 0, sizeof(SiteState), c->stream));
    const int sms = c->num_sms;
    if (init_gains_buckets(c, a, d_scan_tmp, scan_bytes) != TXS_OK) return TXS_ERR_CUDA;
    const LoopPtrs lp0{c->d_crow, c->d_ccol, c->d_win, c->d_bucket_start, d_steps};
    // Batched exact greedy (every local maximum per round) when the grid holds enough
    // independent (4R+1)^2 neighbourhoods for a round to commit several picks (measured:
    // c3 1670 regions 21.9 -> 1.9 ms, c5 268 regions 79.6 -> 46.4, c2 26 regions 6.8 -> 3.8;
    // c1's 6 regions 0.41 -> 0.82 ms, so small grids keep the serial loop).  TXS_SITE_BATCH=0|1
    // forces the choice; the serial loops' A/B knobs imply 0.
    {
        const double regions = (double)c->nrows * (double)c->ncols / ((4.0 * a.R + 1.0) * (4.0 * a.R + 1.0));
        bool batch = regions >= 16.0;
        for (const char* k : {"TXS_SITE_CLUSTER", "TXS_SITE_PERSISTENT", "TXS_SITE_GRAPH", "TXS_SITE_LOOP3", "TXS_SITE_LOOP_CTAS",
                              "TXS_SITE_PROFILE"})
            if (getenv(k)) batch = false;
        if (const char* e = getenv("TXS_SITE_BATCH")) batch = atoi(e) != 0;
        if (batch && p.site_mode == 0 && n > 0) return run_site_batched(c, p, a, d_steps, out, stop);
    }
    // Persistent loop vs graph of per-round kernels (measured, profiles/): the
    // persistent kernel wins while a round touches few neighbours (C1 0.72 vs
    // 1.28 ms, C3 47 vs 62 ms); with thousands of neighbours per round (C5) the
    // per-round kernels' wider update grid wins (109 vs 197 ms).
    const double span = 4.0 * a.R + 1.0;
    const double expected_nb = (double)n * span * span / ((double)c->nrows * (double)c->ncols);
    const bool persistent = p.site_mode == 0 && (expected_nb <= 1000.0 || getenv("TXS_SITE_PERSISTENT")) &&
                            !getenv("TXS_SITE_GRAPH");
    // the loop inside one thread-block cluster (cluster barrier + partials through
    // distributed shared memory): A/B only, TXS_SITE_CLUSTER=8|16.  Measured slower
    // than the grid loop (profiles/README.md: the barrier drops from 2.7 to 0.75 us
    // per round, but 16 SMs carry the neighbour updates 3x slower: c3 27.1 vs 21.9 ms,
    // c4 24.2 vs 23.0)
    if (persistent && !getenv("TXS_SITE_LOOP3") && n > 0) {
        int want_cs = 0;
        if (const char* e = getenv("TXS_SITE_CLUSTER")) want_cs = std::max(0, std::min(kLcMaxCluster, atoi(e)));
        for (int cs = want_cs; cs >= 8; cs >>= 1) {
            const int64_t mmax = (n + cs - 1) / cs;
            const int64_t nchunk = (mmax + 31) / 32;
            const size_t smem = (size_t)(mmax + 1) * 12 + (size_t)nchunk * 12 + (size_t)mmax * 2 + 32;
            if (mmax > 65535 || smem > 216 * 1024 || c->nrows > 65535 || c->ncols > 65535 ||
                4 * (int64_t)a.R / a.bsize + 2 > kLcMaxRanges)
                continue;
            if (cs > 8 && cudaFuncSetAttribute(k_site_loopc, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
                cudaGetLastError();
                continue;
            }
            if (cudaFuncSetAttribute(k_site_loopc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
                cudaGetLastError();
                continue;
            }
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3((unsigned)cs);
            cfg.blockDim = dim3(kLcThreads);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = c->stream;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = (unsigned)cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.attrs = at; cfg.numAttrs = 1;
            int nclusters = 0;
            if (cudaOccupancyMaxActiveClusters(&nclusters, k_site_loopc, &cfg) != cudaSuccess || nclusters < 1) {
                cudaGetLastError();
                continue;
            }
            cudaEventRecord(c->ev_r0, c->stream);
            TXS_CUDA(c, "site", cudaLaunchKernelEx(&cfg, k_site_loopc, a, c->d_state, lp0, (const int32_t*)c->d_pop, c->d_gain,
                                                   (const int32_t*)c->d_bucket_items, (const uint64_t*)c->d_words, cumv,
                                                   c->d_counters));
            TXS_LAUNCHED(c, "site");
            cudaEventRecord(c->ev_r1, c->stream);
            c->stats.site_launches += 1;
            TXS_CUDA(c, "site", cudaMemcpyAsync(c->h_state, c->d_state, sizeof(SiteState), cudaMemcpyDeviceToHost, c->stream));
            TXS_CUDA(c, "site", cudaStreamSynchronize(c->stream));
            add_round_time(c);
            const int64_t ns = c->h_state->nsel;
            c->stats.site_iterations += ns;
            out.resize((size_t)ns);
            if (ns > 0) {
                TXS_CUDA(c, "site", cudaMemcpyAsync(out.data(), d_steps, sizeof(txs_step) * ns, cudaMemcpyDeviceToHost, c->stream));
                TXS_CUDA(c, "site", cudaStreamSynchronize(c->stream));
            }
            *stop = c->h_state->stop;
            return TXS_OK;
        }
    }
    if (persistent && !getenv("TXS_SITE_LOOP3")) {
        // one-barrier persistent loop (k_site_loop1): owned gains/windows in shared memory
        // CTAs per SM (measured, profiles/README.md): one when few neighbours change per
        // round (fewer partials to reduce: c3 23.2 -> 21.9 ms, c4 23.8 -> 23.0), two
        // when the neighbour updates dominate (c2, ~630 per round: 6.8 vs 9.3 ms)
        int want = expected_nb < 300.0 ? 1 : 2;
        if (const char* e = getenv("TXS_SITE_LOOP_CTAS")) want = std::max(1, atoi(e));
        int grid = 0, per_sm = 0;
        size_t smem = 0;
        for (int w = want; w >= 1; --w) {
            const int g = w * sms;
            const int64_t m = (n + g - 1) / g;
            smem = (size_t)m * (sizeof(int4) + sizeof(int2) + 2 * sizeof(int));
            if (smem > 200 * 1024) continue;
            if (smem > 48 * 1024)
                TXS_CUDA(c, "site", cudaFuncSetAttribute(k_site_loop1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            TXS_CUDA(c, "site", cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_site_loop1, kL1Threads, smem));
            if (per_sm >= w) { grid = g; break; }
        }
        if (grid > 0) {
            if (ensure(c, "site", (void**)&c->d_partials, &c->partials_cap, 2 * sizeof(SitePart) * (size_t)grid) != TXS_OK)
                return TXS_ERR_OUT_OF_MEMORY;
            SiteArgs aa = a;
            LoopPtrs lpp = lp0;
            SiteState* st_ = c->d_state;
            const int32_t* pop_ = c->d_pop;
            int32_t* g_ = c->d_gain;
            const uint64_t* w_ = c->d_words;
            uint64_t* cu_ = cumv;
            SitePart* pa_ = (SitePart*)c->d_partials;
            unsigned long long* co_ = c->d_counters;
            void* args[] = {&aa, &st_, &lpp, &pop_, &g_, &w_, &cu_, &pa_, &co_};
            cudaEventRecord(c->ev_r0, c->stream);
            TXS_CUDA(c, "site", cudaLaunchCooperativeKernel((void*)k_site_loop1, grid, kL1Threads, args, smem, c->stream));
            TXS_LAUNCHED(c, "site");
            cudaEventRecord(c->ev_r1, c->stream);
            c->stats.site_launches += 1;
            TXS_CUDA(c, "site", cudaMemcpyAsync(c->h_state, c->d_state, sizeof(SiteState), cudaMemcpyDeviceToHost, c->stream));
            TXS_CUDA(c, "site", cudaStreamSynchronize(c->stream));
            add_round_time(c);
            const int64_t ns = c->h_state->nsel;
            c->stats.site_iterations += ns;
            out.resize((size_t)ns);
            if (ns > 0) {
                TXS_CUDA(c, "site", cudaMemcpyAsync(out.data(), d_steps, sizeof(txs_step) * ns, cudaMemcpyDeviceToHost, c->stream));
                TXS_CUDA(c, "site", cudaStreamSynchronize(c->stream));
            }
            *stop = c->h_state->stop;
            return TXS_OK;
        }
    }
    if (persistent) {
        // persistent cooperative loop: as many co-resident CTAs as fit, <= 2 per SM
        int per_sm = 0;
        TXS_CUDA(c, "site", cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_site_loop, kLoopThreads, 0));
        // CTAs per SM (measured, profiles/README.md): 4 when a round updates
        // hundreds of neighbours (C2: 10.2 -> 9.1 ms), else 2 (C3: grid syncs dominate)
        int want = expected_nb >= 400.0 ? 4 : 2;
        if (const char* e = getenv("TXS_SITE_LOOP_CTAS")) want = std::max(1, atoi(e));
        const int grid = std::max(1, std::min(per_sm, want)) * sms;
        if (ensure(c, "site", (void**)&c->d_partials, &c->partials_cap, sizeof(unsigned long long) * grid) != TXS_OK)
            return TXS_ERR_OUT_OF_MEMORY;
        int2* sp1 = c->d_dspan + (2 * a.R + 1);
        SiteArgs aa = a;
        LoopPtrs lpp = lp0;
        int32_t* g_ = c->d_gain; const int32_t* it_ = c->d_bucket_items; const uint64_t* w_ = c->d_words;
        uint64_t* cu_ = cumv; uint64_t* dw_ = c->d_dwin; int2* s0_ = c->d_dspan; unsigned long long* pa_ = c->d_partials;
        unsigned long long* co_ = c->d_counters; SiteState* st_ = c->d_state;
        void* args[] = {&aa, &st_, &lpp, &g_, &it_, &w_, &cu_, &dw_, &s0_, &sp1, &pa_, &co_};
        cudaEventRecord(c->ev_r0, c->stream);
        TXS_CUDA(c, "site", cudaLaunchCooperativeKernel((void*)k_site_loop, grid, kLoopThreads, args, 0, c->stream));
        TXS_LAUNCHED(c, "site");
        cudaEventRecord(c->ev_r1, c->stream);
        c->stats.site_launches += 1;
        TXS_CUDA(c, "site", cudaMemcpyAsync(c->h_state, c->d_state, sizeof(SiteState), cudaMemcpyDeviceToHost, c->stream));
        TXS_CUDA(c, "site", cudaStreamSynchronize(c->stream));
        add_round_time(c);
        const int64_t ns = c->h_state->nsel;
        c->stats.site_iterations += ns;
        out.resize((size_t)ns);
        if (ns > 0) {
            TXS_CUDA(c, "site", cudaMemcpyAsync(out.data(), d_steps, sizeof(txs_step) * ns, cudaMemcpyDeviceToHost, c->stream));
            TXS_CUDA(c, "site", cudaStreamSynchronize(c->stream));
        }
        *stop = c->h_state->stop;
        return TXS_OK;
    }
    // graph of kRoundsPerGraph rounds
    // neighbour-update grid: 32 CTAs/SM (measured, c5 112.2 -> 91.9 ms; rounds
    // touch ~3900 neighbours, one CTA each)
    int am_mult = 2, up_mult = kUpdPerSm;
    if (const char* e = getenv("TXS_ARGMAX_MULT")) am_mult = std::max(1, atoi(e));
    if (const char* e = getenv("TXS_UPD_MULT")) up_mult = std::max(1, atoi(e));
    const int am_blocks = blocks_for(n, 256 * 4, sms * am_mult);
    const int cm_blocks = 16;
    const int up_blocks = sms * up_mult;
    const LoopPtrs lp{c->d_crow, c->d_ccol, c->d_win, c->d_bucket_start, d_steps};
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    size_t gp_smem = 0;
    StripShape gp_shape{};
    const int gp_kind = p.site_mode == 1 ? gain_pass_kind(c, a, true, &gp_smem, &gp_shape) : -1;
    if (gp_kind == 2) {
        const txs_status bs = build_strip_tasks(c, a, gp_shape);
        if (bs != TXS_OK) return bs;
    }
    const int t8w = (a.ncols + 7) >> 3, t8h = (a.nrows + 7) >> 3;
    if (gp_kind == 3) {
        const txs_status bs = build_t8(c, a);
        if (bs != TXS_OK) return bs;
        TXS_CUDA(c, "site", cudaMemsetAsync(c->d_t8_cum, 0, sizeof(uint64_t) * (size_t)((int64_t)t8h * t8w), c->stream));
    }
    TXS_CUDA(c, "site", cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    for (int r = 0; r < kRoundsPerGraph; ++r) {
        if (p.site_mode == 1) launch_gain_pass<int32_t>(c, a, c->d_state, cumv, c->d_gain, c->d_counters, true);
        k_argmax<<<am_blocks, 256, 0, c->stream>>>(c->d_gain, a, c->d_state, lp, c->d_dspan);
        k_commit<<<cm_blocks, 256, 0, c->stream>>>(a, c->d_state, c->d_words, cumv, c->d_dwin, c->d_dspan, nullptr);
        if (gp_kind == 3)
            k_commit_t8<<<cm_blocks, 256, 0, c->stream>>>(c->d_state, c->d_t8_win, c->d_t8_words, t8_stride(a.R), c->d_t8_cum, t8w);
        if (p.site_mode != 1)
            k_update<<<up_blocks, kUpdThreads, 0, c->stream>>>(a, c->d_state, c->d_win, c->d_words, c->d_dwin,
                                                               c->d_dspan, c->d_bucket_items, c->d_gain, c->d_counters);
    }
    cudaError_t ce = cudaStreamEndCapture(c->stream, &graph);
    if (ce != cudaSuccess) return cuda_fail(c, "site", ce);
    ce = cudaGraphInstantiate(&exec, graph, 0);
    if (ce != cudaSuccess) { cudaGraphDestroy(graph); return cuda_fail(c, "site", ce); }
    const int per_round = (gp_kind == 2 || gp_kind == 3) ? 4 : 3;
    txs_status st = TXS_OK;
    int64_t graphs = 0;
    for (;;) {
        cudaEventRecord(c->ev_r0, c->stream);
        ce = cudaGraphLaunch(exec, c->stream);
        if (ce != cudaSuccess) { st = cuda_fail(c, "site", ce); break; }
        cudaEventRecord(c->ev_r1, c->stream);
        ++graphs;
        ce = cudaMemcpyAsync(c->h_state, c->d_state, sizeof(SiteState), cudaMemcpyDeviceToHost, c->stream);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(c->stream);
        if (ce == cudaSuccess) add_round_time(c);
        if (ce != cudaSuccess) { st = cuda_fail(c, "site", ce); break; }
        if (c->h_state->done) break;
        if (graphs * kRoundsPerGraph > n + 2 * kRoundsPerGraph) { st = fail(c, TXS_ERR_STATE, "site", "loop did not terminate"); break; }
    }
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    if (st != TXS_OK) return st;
    c->launches += graphs * kRoundsPerGraph * per_round;
    c->stats.site_launches += graphs * kRoundsPerGraph * per_round;
    const int64_t ns = c->h_state->nsel;
    c->stats.site_iterations += ns;
    out.resize((size_t)ns);
    if (ns > 0) {
        TXS_CUDA(c, "site", cudaMemcpyAsync(out.data(), d_steps, sizeof(txs_step) * ns, cudaMemcpyDeviceToHost, c->stream));
        TXS_CUDA(c, "site", cudaStreamSynchronize(c->stream));
    }
    *stop = c->h_state->stop;
    return TXS_OK;
}

txs_status launch_marginal_gains(txs_ctx* c, const uint64_t* d_cum_dense, int64_t* d_gains) {
    txs_params p{};
    p.target_coverage = 1.0;
    SiteArgs a = make_args(c, p);
    a.cr0 = 0; a.cr1 = (int)c->nrows;
    c->wpr = (c->ncols + 63) / 64;
    uint64_t* pad = nullptr;
    TXS_CUDA(c, "site", cudaMallocAsync((void**)&pad, sizeof(uint64_t) * (size_t)(c->nrows * c->wpr + 1), c->stream));
    k_dense_to_padded<<<blocks_for(c->nrows * c->wpr, 256, c->num_sms * 16), 256, 0, c->stream>>>(d_cum_dense, pad, c->nrows, c->ncols, c->wpr);
    TXS_LAUNCHED(c, "site");
    if (a.n > 0) {
        launch_gain_pass<int64_t>(c, a, nullptr, pad, d_gains, nullptr, false);
        TXS_LAUNCHED(c, "site");
    }
    TXS_CUDA(c, "site", cudaFreeAsync(pad, c->stream));
    return TXS_OK;
}

txs_status time_gain_pass(txs_ctx* c, int32_t reps, double* ms, int64_t* bytes) {
    txs_params p{};
    p.target_coverage = 1.0;
    const SiteArgs a = make_args(c, p);
    uint64_t* cumv = c->d_cum - c->cum_r0 * c->wpr;
    size_t gp_smem = 0;
    StripShape gp_shape{};
    const int gp_kind = gain_pass_kind(c, a, true, &gp_smem, &gp_shape);
    if (gp_kind == 2) {
        const txs_status bs = build_strip_tasks(c, a, gp_shape);
        if (bs != TXS_OK) return bs;
    }
    if (gp_kind == 3) {   // the tile cum from the current row-padded cum
        const txs_status bs = build_t8(c, a);
        if (bs != TXS_OK) return bs;
        const int t8w = (a.ncols + 7) >> 3, t8h = (a.nrows + 7) >> 3;
        k_cum_to_t8<<<blocks_for((int64_t)t8h * t8w, 256, c->num_sms * 16), 256, 0, c->stream>>>(cumv, a.wpr, a.cr0, a.cr1, t8h,
                                                                                                t8w, c->d_t8_cum);
        TXS_LAUNCHED(c, "site");
    }
    TXS_CUDA(c, "site", cudaMemsetAsync(c->d_counters + kSiteBytes, 0, sizeof(unsigned long long), c->stream));
    launch_gain_pass<int32_t>(c, a, nullptr, cumv, c->d_gain, c->d_counters, true);   // warm-up (+ byte count)
    TXS_LAUNCHED(c, "site");
    unsigned long long b = 0;
    TXS_CUDA(c, "site", cudaMemcpyAsync(&b, c->d_counters + kSiteBytes, sizeof(b), cudaMemcpyDeviceToHost, c->stream));
    cudaEventRecord(c->ev_r0, c->stream);
    for (int k = 0; k < reps; ++k) {
        launch_gain_pass<int32_t>(c, a, nullptr, cumv, c->d_gain, nullptr, true);
        TXS_LAUNCHED(c, "site");
    }
    cudaEventRecord(c->ev_r1, c->stream);
    TXS_CUDA(c, "site", cudaEventSynchronize(c->ev_r1));
    float t = 0.f;
    cudaEventElapsedTime(&t, c->ev_r0, c->ev_r1);
    *ms = reps > 0 ? (double)t / reps : 0.0;
    *bytes = (int64_t)b;
    return TXS_OK;
}

txs_status download_cum(txs_ctx* c, uint64_t* host_dense) {
    const int64_t nw = (c->nrows * c->ncols + 63) / 64;
    // persistent staging buffer (a stream-ordered malloc/free per call stalled
    // the download for up to hundreds of ms when the pool returned its memory)
    if (ensure(c, "site", (void**)&c->d_cum_dense, &c->cum_dense_cap, sizeof(uint64_t) * (size_t)std::max<int64_t>(1, nw)) != TXS_OK)
        return TXS_ERR_OUT_OF_MEMORY;
    uint64_t* dense = c->d_cum_dense;
    k_padded_to_dense<<<blocks_for(nw, 256, c->num_sms * 16), 256, 0, c->stream>>>(
        c->d_cum - c->cum_r0 * c->wpr, dense, c->nrows, c->ncols, c->wpr, c->cum_r0, c->cum_r1, 0, nw);
    TXS_LAUNCHED(c, "site");
    TXS_CUDA(c, "site", cudaMemcpyAsync(host_dense, dense, sizeof(uint64_t) * nw, cudaMemcpyDeviceToHost, c->stream));
    TXS_CUDA(c, "site", cudaStreamSynchronize(c->stream));
    return TXS_OK;
}

// Rows [rb, re) of the cum into the caller's whole-grid dense bitmap: the
// interior words by one D2H straight into place, the two shared edge words
// OR-ed atomically (row bands of several contexts assemble concurrently).
txs_status download_cum_rows(txs_ctx* c, int64_t rb, int64_t re, uint64_t* host_dense) {
    const int64_t total = c->nrows * c->ncols;
    const int64_t b0 = rb * c->ncols, b1 = re * c->ncols;
    if (b1 <= b0) return TXS_OK;
    const int64_t t0 = b0 >> 6, t1 = (b1 + 63) >> 6, m = t1 - t0;
    if (ensure(c, "site", (void**)&c->d_cum_dense, &c->cum_dense_cap, sizeof(uint64_t) * (size_t)m) != TXS_OK)
        return TXS_ERR_OUT_OF_MEMORY;
    k_padded_to_dense<<<blocks_for(m, 256, c->num_sms * 16), 256, 0, c->stream>>>(
        c->d_cum - c->cum_r0 * c->wpr, c->d_cum_dense, c->nrows, c->ncols, c->wpr, std::max(rb, c->cum_r0),
        std::min(re, c->cum_r1), t0, t1);
    TXS_LAUNCHED(c, "site");
    // words shared with rows outside [rb, re) (the last word's tail past the grid is padding)
    const bool e0 = (b0 & 63) != 0, e1 = (b1 & 63) != 0 && b1 < total;
    const int64_t i0 = e0 ? 1 : 0, i1 = e1 ? m - 1 : m;
    if (i1 > i0)
        TXS_CUDA(c, "site", cudaMemcpyAsync(host_dense + t0 + i0, c->d_cum_dense + i0, sizeof(uint64_t) * (i1 - i0),
                                            cudaMemcpyDeviceToHost, c->stream));
    uint64_t edge[2] = {0, 0};
    if (e0) TXS_CUDA(c, "site", cudaMemcpyAsync(&edge[0], c->d_cum_dense, 8, cudaMemcpyDeviceToHost, c->stream));
    if (e1) TXS_CUDA(c, "site", cudaMemcpyAsync(&edge[1], c->d_cum_dense + m - 1, 8, cudaMemcpyDeviceToHost, c->stream));
    TXS_CUDA(c, "site", cudaStreamSynchronize(c->stream));
    if (e0) __atomic_fetch_or(&host_dense[t0], edge[0], __ATOMIC_RELAXED);       // OR is idempotent: m == 1
    if (e1) __atomic_fetch_or(&host_dense[t1 - 1], edge[1], __ATOMIC_RELAXED);   // with both edges is fine
    return TXS_OK;
}

// ---- replicated SITE: records <-> resident candidates (one warp per record) -----------
__global__ void k_pack_records(int64_t n, int64_t slots, int64_t gid0, const int32_t* __restrict__ cgid,
                               const int32_t* __restrict__ crow, const int32_t* __restrict__ ccol,
                               const int32_t* __restrict__ cscore, const int4* __restrict__ cwin,
                               const int32_t* __restrict__ cpop,
                               const uint64_t* __restrict__ words, int64_t stride, uint64_t* __restrict__ rec) {
    const int lane = threadIdx.x & 31;
    const int64_t rw = kRecHead + stride;
    for (int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < slots;
         s += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        uint64_t* r = rec + s * rw;
        if (s >= n) {
            if (lane == 0) r[0] = ~0ull;   // padding
            continue;
        }
        const int4 w = cwin[s];
        if (lane == 0) {
            r[0] = (uint64_t)(cgid ? (int64_t)cgid[s] : gid0 + s);
            r[1] = (uint64_t)(uint32_t)crow[s] | ((uint64_t)(uint32_t)ccol[s] << 32);
            r[2] = (uint64_t)(uint32_t)w.x | ((uint64_t)(uint32_t)w.y << 32);
            r[3] = (uint64_t)(uint32_t)w.z | ((uint64_t)(uint32_t)w.w << 32);
            r[4] = (uint64_t)(uint32_t)cpop[s] | ((uint64_t)(uint32_t)cscore[s] << 32);
        }
        const int64_t nw = (int64_t)w.z * win_nwr(w.y, w.w);
        for (int64_t t = lane; t < nw; t += 32) r[kRecHead + t] = words[s * stride + t];
    }
}

__global__ void k_unpack_records(int64_t nrec, int64_t n_total, const uint64_t* __restrict__ rec, int64_t stride,
                                 int32_t* __restrict__ crow, int32_t* __restrict__ ccol, int32_t* __restrict__ cscore,
                                 int4* __restrict__ cwin, int32_t* __restrict__ cpop, uint64_t* __restrict__ words) {
    const int lane = threadIdx.x & 31;
    const int64_t rw = kRecHead + stride;
    for (int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < nrec;
         s += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const uint64_t* r = rec + s * rw;
        const int64_t g = (int64_t)r[0];
        if (g < 0 || g >= n_total) continue;
        const int4 w = make_int4((int)(uint32_t)r[2], (int)(uint32_t)(r[2] >> 32), (int)(uint32_t)r[3],
                                 (int)(uint32_t)(r[3] >> 32));
        if (lane == 0) {
            crow[g] = (int32_t)(uint32_t)r[1];
            ccol[g] = (int32_t)(uint32_t)(r[1] >> 32);
            cwin[g] = w;
            cpop[g] = (int32_t)(uint32_t)r[4];
            cscore[g] = (int32_t)(uint32_t)(r[4] >> 32);
        }
        const int64_t nw = (int64_t)w.z * win_nwr(w.y, w.w);
        for (int64_t t = lane; t < nw; t += 32) words[g * stride + t] = __ldcs(r + kRecHead + t);
    }
}

txs_status pack_records(txs_ctx* c, int64_t slots, uint64_t* d_rec) {
    if (slots <= 0) return TXS_OK;
    k_pack_records<<<blocks_for(slots * 32, 256, c->num_sms * 16), 256, 0, c->stream>>>(
        c->vs_n, slots, c->cand_gid0, c->h_cgid.empty() ? nullptr : c->d_cgid, c->d_crow, c->d_ccol, c->d_cscore, c->d_win,
        c->d_pop, c->d_words, c->vs_stride, d_rec);
    TXS_LAUNCHED(c, "site");
    return TXS_OK;
}

txs_status unpack_records(txs_ctx* c, int64_t nrec, const uint64_t* d_rec) {
    if (nrec <= 0) return TXS_OK;
    k_unpack_records<<<blocks_for(nrec * 32, 256, c->num_sms * 16), 256, 0, c->stream>>>(
        nrec, c->vs_n, d_rec, c->vs_stride, c->d_crow, c->d_ccol, c->d_cscore, c->d_win, c->d_pop, c->d_words);
    TXS_LAUNCHED(c, "site");
    return TXS_OK;
}

// ---- sharded SITE rounds -------------------------------------------
namespace {

__global__ void k_shard_best(const int32_t* __restrict__ gain, const int32_t* __restrict__ cgid, int64_t gid0,
                             int64_t n, SiteState* st) {
    __shared__ unsigned long long s_red[32];
    unsigned long long best = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t gid = cgid ? (uint64_t)cgid[i] : (uint64_t)(gid0 + i);
        best = umax64(best, ((unsigned long long)(uint32_t)gain[i] << 32) | (0xffffffffull - gid));
    }
    for (int o = 16; o; o >>= 1) best = umax64(best, __shfl_xor_sync(kFull, best, o));
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k) best = umax64(best, s_red[k]);
        best = umax64(best, s_red[0]);
        if (best) atomicMax(&st->shard_key, best);
    }
}

__global__ void k_shard_prep(SiteArgs a, SiteState* st, int r, int c, int4 win, const int32_t* __restrict__ bstart,
                             int2* __restrict__ dspan) {
    for (int y = threadIdx.x; y < 2 * a.R + 1; y += blockDim.x) dspan[y] = make_int2(0x7fffffff, -1);
    if (threadIdx.x != 0) return;
    st->done = 0; st->finish = 0; st->w_idx = -1;
    st->w_row0 = win.x; st->w_col0 = win.y; st->w_h = win.z; st->w_w = win.w;
    const int by0 = max(0, (r - 2 * a.R) / a.bsize), by1 = min(a.nby - 1, (r + 2 * a.R) / a.bsize);
    const int bx0 = max(0, (c - 2 * a.R) / a.bsize), bx1 = min(a.nbx - 1, (c + 2 * a.R) / a.bsize);
    int nb = 0, pref = 0;
    for (int by = by0; by <= by1 && nb < kMaxNb; ++by) {
        const int s0 = bstart[by * a.nbx + bx0], e0 = bstart[by * a.nbx + bx1 + 1];
        st->nb_start[nb] = s0;
        st->nb_pref[nb] = pref;
        pref += e0 - s0;
        ++nb;
    }
    st->nb_pref[nb] = pref;
    st->nb_count = nb;
}

// ---- device-resident shard rounds ----
// Best local key, or 0 once this context's SITE stopped (done / final pick made).
__global__ void k_shard_best_dev(const int32_t* __restrict__ gain, const int32_t* __restrict__ cgid, int64_t gid0,
                                 int64_t n, const SiteState* st, unsigned long long* __restrict__ d_key) {
    if (st->done || st->finish) return;
    __shared__ unsigned long long s_red[32];
    unsigned long long best = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t gid = cgid ? (uint64_t)cgid[i] : (uint64_t)(gid0 + i);
        best = umax64(best, ((unsigned long long)(uint32_t)gain[i] << 32) | (0xffffffffull - gid));
    }
    for (int o = 16; o; o >>= 1) best = umax64(best, __shfl_xor_sync(kFull, best, o));
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k) best = umax64(best, s_red[k]);
        best = umax64(best, s_red[0]);
        if (best) atomicMax(d_key, best);
    }
}

// One CTA: zero the payload; the rank holding the reduced key's candidate
// writes {row, col, row0, col0, h, w, cum-aligned words} (the same layout on
// every rank: aligned words are anchored to global terrain columns).
__global__ void k_shard_export_dev(const SiteState* st, const unsigned long long* __restrict__ d_key,
                                   const int32_t* __restrict__ cgid, int64_t gid0, int64_t n,
                                   const int32_t* __restrict__ crow, const int32_t* __restrict__ ccol,
                                   const int4* __restrict__ wins, const uint64_t* __restrict__ words, int64_t stride,
                                   uint64_t* __restrict__ payload, int64_t pwords) {
    __shared__ int64_t s_li;
    for (int64_t t = threadIdx.x; t < pwords; t += blockDim.x) payload[t] = 0ull;
    if (threadIdx.x == 0) {
        s_li = -1;
        const unsigned long long key = *d_key;
        if (!st->done && !st->finish && (key >> 32) > 0) {
            const int64_t gid = (int64_t)(0xffffffffull - (key & 0xffffffffull));
            if (!cgid) {
                if (gid >= gid0 && gid < gid0 + n) s_li = gid - gid0;
            } else {   // sorted global draw indices
                int64_t lo = 0, hi = n;
                while (lo < hi) {
                    const int64_t mid = (lo + hi) >> 1;
                    if ((int64_t)cgid[mid] < gid) lo = mid + 1; else hi = mid;
                }
                if (lo < n && (int64_t)cgid[lo] == gid) s_li = lo;
            }
        }
    }
    __syncthreads();
    const int64_t li = s_li;
    if (li < 0) return;
    const int4 win = wins[li];
    const int total = win.z * win_nwr(win.y, win.w);
    if (threadIdx.x == 0) {
        payload[0] = (uint64_t)(uint32_t)crow[li];
        payload[1] = (uint64_t)(uint32_t)ccol[li];
        payload[2] = (uint64_t)(uint32_t)win.x;
        payload[3] = (uint64_t)(uint32_t)win.y;
        payload[4] = (uint64_t)(uint32_t)win.z;
        payload[5] = (uint64_t)(uint32_t)win.w;
    }
    const uint64_t* v = words + li * stride;
    for (int t = threadIdx.x; t < total; t += blockDim.x) payload[6 + t] = v[t];
}

// One CTA: the round's decision from the reduced key and payload (identical on
// every rank), step record, winner window and neighbour ranges; k_commit and
// k_update follow and no-op once done.
__global__ void k_shard_decide_dev(SiteArgs a, SiteState* st, const unsigned long long* __restrict__ d_key,
                                   const uint64_t* __restrict__ payload, int64_t total_cand,
                                   const int32_t* __restrict__ bstart, int2* __restrict__ dspan,
                                   txs_step* __restrict__ steps, int64_t steps_cap) {
    if (st->done) return;
    if (st->finish) {   // the previous round committed the final pick
        if (threadIdx.x == 0) st->done = 1;
        return;
    }
    for (int y = threadIdx.x; y < 2 * a.R + 1; y += blockDim.x) dspan[y] = make_int2(0x7fffffff, -1);
    if (threadIdx.x != 0) return;
    if (st->nsel >= total_cand) { st->done = 1; st->stop = TXS_STOP_EXHAUSTED; return; }
    const unsigned long long key = *d_key;
    const long long g = (long long)(key >> 32);
    if (g <= 0) { st->done = 1; st->stop = TXS_STOP_ZERO_GAIN; return; }
    const int64_t gid = (int64_t)(0xffffffffull - (key & 0xffffffffull));
    const int r = (int)(uint32_t)payload[0], c = (int)(uint32_t)payload[1];
    st->w_row0 = (int)(uint32_t)payload[2]; st->w_col0 = (int)(uint32_t)payload[3];
    st->w_h = (int)(uint32_t)payload[4]; st->w_w = (int)(uint32_t)payload[5];
    st->w_idx = -1;
    st->covered += g;
    const double cov = (double)st->covered / a.total;
    const long long k = st->nsel;
    if (k < steps_cap) steps[k] = txs_step{gid, r, c, (int64_t)g, cov};
    st->nsel = k + 1;
    if (cov >= a.target) { st->finish = 1; st->stop = TXS_STOP_TARGET_REACHED; }
    else if (a.max_sel > 0 && k + 1 >= a.max_sel) { st->finish = 1; st->stop = TXS_STOP_MAX_SELECTED; }
    const int by0 = max(0, (r - 2 * a.R) / a.bsize), by1 = min(a.nby - 1, (r + 2 * a.R) / a.bsize);
    const int bx0 = max(0, (c - 2 * a.R) / a.bsize), bx1 = min(a.nbx - 1, (c + 2 * a.R) / a.bsize);
    int nb = 0, pref = 0;
    for (int by = by0; by <= by1 && nb < kMaxNb; ++by) {
        const int s0 = bstart[by * a.nbx + bx0], e0 = bstart[by * a.nbx + bx1 + 1];
        st->nb_start[nb] = s0;
        st->nb_pref[nb] = pref;
        pref += e0 - s0;
        ++nb;
    }
    st->nb_pref[nb] = pref;
    st->nb_count = nb;
}

}  // namespace

txs_status viewsheds_to_dense(txs_ctx* c, int64_t first, int64_t count, uint64_t* d_dense, int64_t dstride) {
    if (count <= 0) return TXS_OK;
    k_aligned_to_dense<<<blocks_for(count * dstride, 256, c->num_sms * 16), 256, 0, c->stream>>>(
        c->d_words + first * c->vs_stride, c->vs_stride, c->d_win + first, count, d_dense, dstride);
    TXS_LAUNCHED(c, "viewshed");
    return TXS_OK;
}

txs_status viewsheds_from_dense(txs_ctx* c, const uint64_t* d_dense, int64_t dstride, const int4* d_wins,
                                uint64_t* d_aligned, int64_t astride, int64_t count) {
    if (count <= 0) return TXS_OK;
    k_dense_to_aligned<<<blocks_for(count * astride, 256, c->num_sms * 16), 256, 0, c->stream>>>(
        d_dense, dstride, d_wins, count, d_aligned, astride);
    TXS_LAUNCHED(c, "site");
    return TXS_OK;
}

txs_status shard_site_begin(txs_ctx* c, const txs_params& p) {
    TXS_CUDA(c, "site", cudaStreamSynchronize(c->stream));
    const int64_t R = c->vs_roi;
    if (alloc_bitmaps(c, std::max<int64_t>(0, c->band_r0 - R), std::min<int64_t>(c->nrows, c->band_r1 + R)) != TXS_OK)
        return TXS_ERR_OUT_OF_MEMORY;
    const SiteArgs a = make_args(c, p);
    const int64_t n = a.n, nbk = (int64_t)a.nbx * a.nby;
    if (ensure(c, "site", (void**)&c->d_gain, &c->gain_cap, sizeof(int32_t) * std::max<int64_t>(1, n)) != TXS_OK ||
        ensure(c, "site", (void**)&c->d_bucket_start, &c->bucket_cap, sizeof(int32_t) * (nbk + 1) * 2) != TXS_OK ||
        ensure(c, "site", (void**)&c->d_bucket_items, &c->bucket_items_cap, sizeof(int32_t) * std::max<int64_t>(1, n)) != TXS_OK)
        return TXS_ERR_OUT_OF_MEMORY;
    size_t scan_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int32_t*)nullptr, (int32_t*)nullptr, (int)(nbk + 1));
    if (ensure(c, "site", &c->d_scratch, &c->scratch_cap, scan_bytes + 256) != TXS_OK) return TXS_ERR_OUT_OF_MEMORY;
    TXS_CUDA(c, "site", cudaMemsetAsync(c->d_cum, 0, sizeof(uint64_t) * ((c->cum_r1 - c->cum_r0) * c->wpr + 1), c->stream));
    TXS_CUDA(c, "site", cudaMemsetAsync(c->d_state, 0, sizeof(SiteState), c->stream));
    if (init_gains_buckets(c, a, c->d_scratch, scan_bytes) != TXS_OK) return TXS_ERR_CUDA;
    if (!c->h_cgid.empty()) {
        if (ensure(c, "site", (void**)&c->d_cgid, &c->cgid_cap, sizeof(int32_t) * c->h_cgid.size()) != TXS_OK)
            return TXS_ERR_OUT_OF_MEMORY;
        TXS_CUDA(c, "site", cudaMemcpyAsync(c->d_cgid, c->h_cgid.data(), sizeof(int32_t) * c->h_cgid.size(),
                                            cudaMemcpyHostToDevice, c->stream));
    }
    const int64_t mw = max_window_words(R) + 2 + aligned_stride(R) + 2;
    if (ensure(c, "site", (void**)&c->d_xfer, &c->xfer_cap, sizeof(uint64_t) * mw) != TXS_OK) return TXS_ERR_OUT_OF_MEMORY;
    TXS_CUDA(c, "site", cudaStreamSynchronize(c->stream));
    c->shard_target = p.target_coverage;
    c->shard_max_sel = p.max_selected;
    c->site_valid = true;
    return TXS_OK;
}

txs_status shard_site_best(txs_ctx* c, uint64_t* key) {
    const int64_t n = c->vs_n;
    TXS_CUDA(c, "site", cudaMemsetAsync(&c->d_state->shard_key, 0, sizeof(unsigned long long), c->stream));
    if (n > 0) {
        k_shard_best<<<blocks_for(n, 1024, c->num_sms * 2), 256, 0, c->stream>>>(
            c->d_gain, c->h_cgid.empty() ? nullptr : c->d_cgid, c->cand_gid0, n, c->d_state);
        TXS_LAUNCHED(c, "site");
    }
    unsigned long long k = 0;
    TXS_CUDA(c, "site", cudaMemcpyAsync(&k, &c->d_state->shard_key, sizeof(k), cudaMemcpyDeviceToHost, c->stream));
    TXS_CUDA(c, "site", cudaStreamSynchronize(c->stream));
    *key = k;
    return TXS_OK;
}

txs_status shard_site_apply(txs_ctx* c, int32_t row, int32_t col, const txs_window& win, const uint64_t* words) {
    txs_params p{};
    p.target_coverage = 1.0;
    const SiteArgs a = make_args(c, p);
    const int64_t nw = ((int64_t)win.h * win.w + 63) / 64, dstr = max_window_words(c->vs_roi);
    const int64_t astr = aligned_stride(c->vs_roi);
    if (nw > dstr || win.h > 2 * c->vs_roi + 1 || win.w > 2 * c->vs_roi + 1)
        return fail(c, TXS_ERR_INVALID_ARGUMENT, "site", "window larger than the engine's roi");
    // xfer = [dense words (dstr+2)] [aligned words (astr)] [window int4]
    uint64_t* xd = c->d_xfer;
    uint64_t* xa = c->d_xfer + dstr + 2;
    int4* xw = (int4*)(xa + astr);
    const int4 w4 = make_int4(win.row0, win.col0, win.h, win.w);
    TXS_CUDA(c, "site", cudaMemcpyAsync(xd, words, sizeof(uint64_t) * nw, cudaMemcpyHostToDevice, c->stream));
    TXS_CUDA(c, "site", cudaMemsetAsync(xd + nw, 0, sizeof(uint64_t) * (dstr + 2 - nw), c->stream));
    TXS_CUDA(c, "site", cudaMemcpyAsync(xw, &w4, sizeof(int4), cudaMemcpyHostToDevice, c->stream));
    if (viewsheds_from_dense(c, xd, dstr, xw, xa, astr, 1) != TXS_OK) return TXS_ERR_CUDA;
    k_shard_prep<<<1, 256, 0, c->stream>>>(a, c->d_state, row, col, make_int4(win.row0, win.col0, win.h, win.w),
                                          c->d_bucket_start, c->d_dspan);
    TXS_LAUNCHED(c, "site");
    uint64_t* cumv = c->d_cum - c->cum_r0 * c->wpr;
    k_commit<<<16, 256, 0, c->stream>>>(a, c->d_state, c->d_words, cumv, c->d_dwin, c->d_dspan, xa);
    TXS_LAUNCHED(c, "site");
    k_update<<<c->num_sms * kUpdPerSm, kUpdThreads, 0, c->stream>>>(a, c->d_state, c->d_win, c->d_words, c->d_dwin, c->d_dspan,
                                                           c->d_bucket_items, c->d_gain, c->d_counters);
    TXS_LAUNCHED(c, "site");
    c->stats.site_iterations += 1;
    return TXS_OK;
}

int64_t shard_payload_words(const txs_ctx* c) { return 6 + aligned_stride(c->vs_roi); }

// The gathered {key, payload} entries of every rank: the largest key (the
// allreduce(MAX) winner) and its payload, copied for txs_site_shard_apply_dev.
__global__ void k_shard_select_dev(const uint64_t* __restrict__ g, int nranks, int64_t pw,
                                   unsigned long long* __restrict__ key, uint64_t* __restrict__ payload) {
    __shared__ int s_best;
    if (threadIdx.x == 0) {
        int b = 0;
        for (int k = 1; k < nranks; ++k)
            if (g[(int64_t)k * (pw + 1)] > g[(int64_t)b * (pw + 1)]) b = k;
        s_best = b;
        *key = g[(int64_t)b * (pw + 1)];
    }
    __syncthreads();
    const uint64_t* src = g + (int64_t)s_best * (pw + 1) + 1;
    for (int64_t t = threadIdx.x; t < pw; t += blockDim.x) payload[t] = src[t];
}

txs_status shard_site_select_dev(txs_ctx* c, const uint64_t* d_gathered, int32_t nranks, uint64_t* d_key,
                                 uint64_t* d_payload) {
    k_shard_select_dev<<<1, 256, 0, c->stream>>>(d_gathered, nranks, shard_payload_words(c),
                                                 (unsigned long long*)d_key, d_payload);
    TXS_LAUNCHED(c, "site");
    return TXS_OK;
}

// Peer-memory exchange (txs_group, TXS_XCHG_P2P): mail[k] points at rank k's
// mailbox {key, payload} -- on its own device, read here over NVLink.  All N keys
// are read, then only the winner's header and window rows (h * nwr aligned words,
// not the whole payload stride) cross the link.
__global__ void k_shard_select_peers(const uint64_t* const* __restrict__ mail, int nranks,
                                     unsigned long long* __restrict__ key, uint64_t* __restrict__ payload) {
    __shared__ int s_best;
    __shared__ int64_t s_len;
    if (threadIdx.x == 0) {
        int b = 0;
        uint64_t bk = *(volatile const uint64_t*)mail[0];
        for (int k = 1; k < nranks; ++k) {
            const uint64_t v = *(volatile const uint64_t*)mail[k];
            if (v > bk) { bk = v; b = k; }
        }
        s_best = b;
        *key = bk;
        const uint64_t* src = mail[b] + 1;
        const int h = (int)(uint32_t)src[4], c0 = (int)(uint32_t)src[3], w = (int)(uint32_t)src[5];
        s_len = bk ? 6 + (int64_t)h * win_nwr(c0, w) : 6;
    }
    __syncthreads();
    const uint64_t* src = mail[s_best] + 1;
    for (int64_t t = threadIdx.x; t < s_len; t += blockDim.x) payload[t] = src[t];
}

txs_status shard_site_select_peers(txs_ctx* c, const uint64_t* const* d_mail, int32_t nranks, uint64_t* d_key,
                                   uint64_t* d_payload) {
    k_shard_select_peers<<<1, 256, 0, c->stream>>>(d_mail, nranks, (unsigned long long*)d_key, d_payload);
    TXS_LAUNCHED(c, "site");
    return TXS_OK;
}

txs_status shard_site_best_dev(txs_ctx* c, uint64_t* d_key) {
    const int64_t n = c->vs_n;
    TXS_CUDA(c, "site", cudaMemsetAsync(d_key, 0, sizeof(uint64_t), c->stream));
    if (n > 0) {
        k_shard_best_dev<<<blocks_for(n, 1024, c->num_sms * 2), 256, 0, c->stream>>>(
            c->d_gain, c->h_cgid.empty() ? nullptr : c->d_cgid, c->cand_gid0, n, c->d_state,
            (unsigned long long*)d_key);
        TXS_LAUNCHED(c, "site");
    }
    return TXS_OK;
}

txs_status shard_site_export_dev(txs_ctx* c, const uint64_t* d_key, uint64_t* d_payload) {
    k_shard_export_dev<<<1, 256, 0, c->stream>>>(c->d_state, (const unsigned long long*)d_key,
                                                 c->h_cgid.empty() ? nullptr : c->d_cgid, c->cand_gid0, c->vs_n,
                                                 c->d_crow, c->d_ccol, c->d_win, c->d_words, c->vs_stride, d_payload,
                                                 shard_payload_words(c));
    TXS_LAUNCHED(c, "site");
    return TXS_OK;
}

txs_status shard_site_apply_dev(txs_ctx* c, const uint64_t* d_key, const uint64_t* d_payload, int64_t total) {
    txs_params p{};
    p.target_coverage = c->shard_target;
    p.max_selected = c->shard_max_sel;
    const SiteArgs a = make_args(c, p);
    const int64_t cap = std::max<int64_t>(1, total);
    if (ensure(c, "site", (void**)&c->d_shard_steps, &c->shard_steps_cap, sizeof(txs_step) * cap) != TXS_OK)
        return TXS_ERR_OUT_OF_MEMORY;
    k_shard_decide_dev<<<1, 256, 0, c->stream>>>(a, c->d_state, (const unsigned long long*)d_key, d_payload, total,
                                                 c->d_bucket_start, c->d_dspan, c->d_shard_steps, cap);
    TXS_LAUNCHED(c, "site");
    uint64_t* cumv = c->d_cum - c->cum_r0 * c->wpr;
    k_commit<<<16, 256, 0, c->stream>>>(a, c->d_state, c->d_words, cumv, c->d_dwin, c->d_dspan, d_payload + 6);
    TXS_LAUNCHED(c, "site");
    k_update<<<c->num_sms * kUpdPerSm, kUpdThreads, 0, c->stream>>>(a, c->d_state, c->d_win, c->d_words, c->d_dwin, c->d_dspan,
                                                           c->d_bucket_items, c->d_gain, c->d_counters);
    TXS_LAUNCHED(c, "site");
    return TXS_OK;
}

}  // namespace txs
