// Internal state of a txs_ctx: everything resident in HBM between stages.
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <string>
#include <vector>

#include "../../include/txsite_b200.h"
#include "common.cuh"

namespace txs {

// D5 ray template in host form (built by raytemplate.cpp).
struct RayTemplate {
    int32_t roi = 0;
    std::vector<int32_t> p, q;          // primitive directions, angle order
    std::vector<int64_t> cell_begin;    // rays+1
    std::vector<int32_t> ca, cb;        // owned cells sorted by projection
};
const RayTemplate& ray_template(int32_t roi);

// Device copy: rays[r] = {p, q, cell_begin, cell_count}; cells packed (a & 0xffff) | (b << 16).
// For roi <= kEvMaxRoi also the merged per-ray event stream (see raytemplate.cpp):
// 32-lane groups of neighbouring rays, events interleaved [step][lane], each
// event = {word (type, offsets, weight, byrow bit), y (line index or cell dot)}.
constexpr int kEvMaxRoi = 250;
enum EvType : uint32_t { kEvRow = 0, kEvCol = 1, kEvPost = 2, kEvCell = 3, kEvNop = 4 };
struct RayTemplateDev {
    int32_t roi = 0, nrays = 0;
    int64_t ncells = 0;
    int4* rays = nullptr;
    uint32_t* cells = nullptr;
    int32_t ngroups = 0;
    int2* groups = nullptr;      // {first event row (x32 lanes), steps}
    uint2* events = nullptr;
    uint2* events3 = nullptr;    // the same stream in the interior-sweep encoding (raytemplate.cpp, pack_ev3)
    int64_t nevents = 0;
};
// host-side event stream (exposed for tests through txs_event_template)
struct EventTemplate {
    std::vector<int2> groups;
    std::vector<uint2> events;
    std::vector<uint2> events3;   // interior encoding (pack_ev3), same order
};
// interior-sweep event types (events3)
enum Ev3Type : uint32_t { kEv3Cross = 0, kEv3Cell = 1, kEv3Nop = 2 };
const EventTemplate& event_template(int32_t roi);

// Device-side SITE loop state (one struct, read/written by the loop kernels).
constexpr int kMaxNb = 64;   // neighbour bucket ranges per winner
struct SiteState {
    unsigned long long best_key;   // (gain << 32) | (0xffffffff - idx), atomicMax target
    unsigned int blocks_done;      // last-block detection in k_argmax
    long long nsel;
    long long covered;
    int done;                      // no more commits
    int finish;                    // commit this round, then done
    int stop;
    int w_idx, w_gain;
    int w_row0, w_col0, w_h, w_w;   // current winner window
    int nb_count;
    int nb_start[kMaxNb];
    int nb_pref[kMaxNb + 1];
    unsigned long long shard_key;  // sharded SITE: local best key
    unsigned long long phase_ns[5];   // k_site_loop1 phases (TXS_SITE_PROFILE=1): winner, commit, update, partial, barrier
};

// device counter slots
enum Counter : int {
    kVixLos = 0, kVixCrossFull, kVsCross, kVsCells, kSiteBytes,
    kVixNext,   // work counter of the persistent VIX kernel (reset per launch)
    kVixTies,   // VIX segments visible with an exact grazing tie (fp64 tie list entries)
    kVsTies,    // VIEWSHED (observer, ray) pairs with a grazing tie at a cell (fp64 tie list)
    kVixTiesFlipped, kVsTiesFlipped,   // decisions the fp64 re-test changed
    kVixSelFail, kVixSelTotal, kVixSel,   // k_vix_sample: sampled segments failing a 32-step skip test / sampled; chosen log2 group size
    kNumCounters
};

}  // namespace txs

struct txs_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    int num_sms = 148;

    // terrain: row-major int16 in HBM.  nrows/ncols are the
    // GLOBAL grid; the context holds rows [z_off, z_off + z_rows) of it (all of
    // it unless sharded) and owns the band [band_r0, band_r1).
    int64_t nrows = 0, ncols = 0;
    int16_t* d_z = nullptr;
    size_t z_cap = 0;
    int64_t z_off = 0, z_rows = 0, band_r0 = 0, band_r1 = 0;
    bool sharded = false;
    const int16_t* zv() const { return d_z - z_off * ncols; }   // indexed by global row
    int16_t* d_zt = nullptr;      // column-major copy (VIX global path)
    size_t zt_cap = 0;
    void* d_pairs = nullptr;      // VIX quad planes / VIEWSHED pair planes (per-call scratch)
    uint8_t* d_gcd = nullptr;     // 256x256 gcd table (VIX crossing statistic)
    int4* d_ties = nullptr;       // fp64 tie lists (VIX segments / VIEWSHED rays), per-call scratch
    size_t ties_cap = 0;
    int64_t vix_tie_min = 0, vs_tie_min = 0;   // tie-list sizes after an overflow (re-run)
    size_t pairs_cap = 0;

    // VixMap: one byte per post
    uint8_t* d_vix = nullptr;
    size_t vix_cap = 0;
    bool vix_valid = false;

    // candidates, in candidate-index order; global id of local
    // candidate i = cand_gid0 + i, or h_cgid[i] when set (sharded random observers)
    int64_t ncand = 0;
    int64_t cand_gid0 = 0;
    std::vector<int32_t> h_cgid;
    int32_t* d_cgid = nullptr;
    size_t cgid_cap = 0;
    int32_t *d_crow = nullptr, *d_ccol = nullptr, *d_cscore = nullptr;
    size_t cand_cap = 0;
    bool cand_valid = false;

    // viewsheds: fixed stride of max window words per candidate
    int32_t vs_roi = 0;
    int64_t vs_n = 0, vs_stride = 0;
    uint64_t* d_words = nullptr;
    size_t words_cap = 0;
    int4* d_win = nullptr;        // {row0, col0, h, w}
    int32_t* d_pop = nullptr;     // popcount per viewshed
    size_t win_cap = 0, pop_cap = 0;
    bool vs_valid = false;
    std::map<int32_t, txs::RayTemplateDev> templates;

    // SITE: row-padded bitmaps (wpr words per terrain row) over
    // the cum region rows [cum_r0, cum_r1) (whole grid unless sharded)
    int64_t wpr = 0;
    int64_t cum_r0 = 0, cum_r1 = 0;
    uint64_t* d_xfer = nullptr;          // sharded SITE: the broadcast winner window
    size_t xfer_cap = 0;
    txs_step* d_shard_steps = nullptr;   // sharded SITE (device rounds): step log
    size_t shard_steps_cap = 0;
    double shard_target = 1.0;           // sharded SITE: stop rules of txs_site_shard_begin
    int64_t shard_max_sel = 0;
    uint64_t* d_cum = nullptr;
    uint64_t* d_cum_dense = nullptr;     // SPEC-dense staging of txs_get_cumulative
    size_t cum_dense_cap = 0;
    // per-round delta: newly covered words over the winner window (row pitch
    // dpitch words) and per-row [lo, hi] spans of non-zero words
    uint64_t* d_dwin = nullptr;
    int2* d_dspan = nullptr;
    size_t dwin_cap = 0, dspan_cap = 0;
    int64_t dpitch = 0;
    unsigned long long* d_partials = nullptr;   // persistent SITE loop: per-CTA argmax
    size_t partials_cap = 0;
    void* d_batch = nullptr;             // batched SITE (site.cu): bucket maxima, winner lists, delta windows, pick log
    size_t batch_cap = 0;
    size_t bitmap_cap = 0;
    int32_t* d_gain = nullptr;
    size_t gain_cap = 0;
    txs::SiteState* d_state = nullptr;
    txs::SiteState* h_state = nullptr;   // pinned mirror
    int32_t* d_bucket_start = nullptr;   // CSR over candidate buckets
    int32_t* d_bucket_items = nullptr;
    size_t bucket_cap = 0, bucket_items_cap = 0;
    int4* d_strip_tasks = nullptr;       // k_gain_strips task list (site.cu), grouped by tile
    int32_t* d_strip_start = nullptr;    // tiles+1 (+ tiles+1 fill cursors)
    size_t strip_tasks_cap = 0, strip_start_cap = 0;
    unsigned long long site_alg_bytes = 0;   // SPEC-layout bytes of the candidate set's viewsheds
    // 8x8-tile shadow of the viewsheds and the cum for the streaming gain pass
    // (site.cu, "t8" layout); t8_valid: d_t8_words / d_t8_win match d_words
    uint64_t* d_t8_words = nullptr;
    int4* d_t8_win = nullptr;
    uint64_t* d_t8_cum = nullptr;
    size_t t8_words_cap = 0, t8_win_cap = 0, t8_cum_cap = 0;
    bool t8_valid = false;
    bool site_valid = false;

    // txs_run_pipeline_host: terrain rows arriving on copy_stream in chunks
    // (event up_ev[k] after chunk k, which ends at row up_end[k]); VIX starts on the first
    // row bands while the rest is still in flight
    cudaStream_t copy_stream = nullptr;
    std::vector<cudaEvent_t> up_ev;
    std::vector<int64_t> up_end;   // chunk k holds rows [up_end[k-1], up_end[k])
    bool up_pending = false;

    // stats
    txs_stats stats{};
    unsigned long long* d_counters = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t ev_r0 = nullptr, ev_r1 = nullptr;   // SITE round-loop timer
    cudaEvent_t ev_k0 = nullptr, ev_k1 = nullptr;   // the stage's main kernel alone (VIX / VIEWSHED)
    cudaEvent_t user_ev[16] = {};
    int64_t launches = 0;
    int64_t dev_bytes = 0, dev_bytes_peak = 0;   // context buffers (txs::ensure), live and high-water
    // VIX crossing statistic (txs_stats.vix_crossings_full): a function of the grid,
    // band, roi, S and seed only, so it is counted on the first launch with a
    // given key and added from this cache afterwards (k_vix_lanes)
    uint64_t vix_cross_key = 0;
    unsigned long long vix_cross_count = 0;
    bool vix_cross_valid = false;

    // scratch
    void* d_scratch = nullptr;
    size_t scratch_cap = 0;
};

namespace txs {

txs_status fail(txs_ctx* ctx, txs_status st, const char* stage, const std::string& msg);
txs_status cuda_fail(txs_ctx* ctx, const char* stage, cudaError_t e);
// (re)allocate *p to at least bytes; contents not preserved
txs_status ensure(txs_ctx* ctx, const char* stage, void** p, size_t* cap, size_t bytes);
txs_status check_params(txs_ctx* ctx, const char* stage, const txs_params* p, bool need_vix);
txs_status get_template(txs_ctx* ctx, int32_t roi, RayTemplateDev** out);
// SPEC layout (decision D8): window rows packed densely, LSB-first.
inline int64_t max_window_words(int64_t roi) { return ((2 * roi + 1) * (2 * roi + 1) + 63) / 64; }
// Engine-internal layout ("cum-aligned rows"): window row y occupies the
// terrain's own 64-bit column words (col0>>6) .. ((col0+w-1)>>6), so cell
// (y, x) is bit (col0+x)&63 of word y*nwr + ((col0+x)>>6) - (col0>>6); bits
// outside the window are zero.  Every SITE kernel then ANDs whole words with
// the row-padded cumulative bitmap.  Converted to/from the SPEC layout at the
// C-ABI (txs_get_viewsheds / txs_set_viewsheds).
__host__ __device__ inline int win_nwr(int col0, int w) { return ((col0 + w - 1) >> 6) - (col0 >> 6) + 1; }
inline int64_t aligned_stride(int64_t roi) { return (2 * roi + 1) * ((2 * roi + 63) / 64 + 1); }

// stage launchers (one .cu each)
txs_status launch_generate(txs_ctx*, int64_t nrows, int64_t ncols, double roughness, uint64_t seed,
                           int32_t zmin, int32_t zmax);   // writes held rows [z_off, z_off+z_rows)
txs_status launch_fill_rows(txs_ctx*, int64_t rb, int64_t re, int16_t v);
txs_status launch_vix(txs_ctx*, const txs_params& p);
// txs_run_pipeline_host: make the context stream wait until terrain rows [0, row_end) have arrived
txs_status wait_terrain_rows(txs_ctx*, int64_t row_end);
txs_status launch_los_batch(txs_ctx*, const int32_t* d_pairs, int64_t n, int32_t ht, int32_t hr,
                            int32_t arith, uint8_t* d_out);
txs_status launch_findmax(txs_ctx*, const txs_params& p, int64_t bw);
txs_status launch_random_observers(txs_ctx*, int64_t n, uint64_t seed);
txs_status launch_viewsheds(txs_ctx*, const txs_params& p);
txs_status run_site(txs_ctx*, const txs_params& p, std::vector<txs_step>& steps, int32_t* stop);
txs_status launch_marginal_gains(txs_ctx*, const uint64_t* d_cum_dense, int64_t* d_gains);
txs_status time_gain_pass(txs_ctx*, int32_t reps, double* ms, int64_t* bytes);
txs_status download_cum(txs_ctx*, uint64_t* host_dense);
txs_status shard_site_begin(txs_ctx*, const txs_params& p);
// layout conversion for candidates [first, first+count): aligned (resident) <-> dense (SPEC)
txs_status viewsheds_to_dense(txs_ctx*, int64_t first, int64_t count, uint64_t* d_dense, int64_t dstride);
txs_status viewsheds_from_dense(txs_ctx*, const uint64_t* d_dense, int64_t dstride, const int4* d_wins,
                                uint64_t* d_aligned, int64_t astride, int64_t count);
txs_status shard_site_best(txs_ctx*, uint64_t* key);
txs_status shard_site_apply(txs_ctx*, int32_t row, int32_t col, const txs_window& win, const uint64_t* words);
txs_status shard_site_best_dev(txs_ctx*, uint64_t* d_key);
txs_status shard_site_export_dev(txs_ctx*, const uint64_t* d_key, uint64_t* d_payload);
txs_status shard_site_apply_dev(txs_ctx*, const uint64_t* d_key, const uint64_t* d_payload, int64_t total);
int64_t shard_payload_words(const txs_ctx*);
txs_status shard_site_select_dev(txs_ctx*, const uint64_t* d_gathered, int32_t nranks, uint64_t* d_key,
                                 uint64_t* d_payload);
// txs_group's peer-memory exchange: d_mail = device array of the N ranks' mailboxes
txs_status shard_site_select_peers(txs_ctx*, const uint64_t* const* d_mail, int32_t nranks, uint64_t* d_key,
                                   uint64_t* d_payload);
txs_status download_cum_rows(txs_ctx*, int64_t row_begin, int64_t row_end, uint64_t* host_dense);
// replicated SITE: resident viewsheds -> records; gathered records -> the
// context's candidate / viewshed arrays at their global ids
constexpr int kRecHead = 5;
txs_status pack_records(txs_ctx*, int64_t slots, uint64_t* d_rec);
txs_status unpack_records(txs_ctx*, int64_t nrec, const uint64_t* d_rec);

}  // namespace txs

#define TXS_CUDA(ctx, stage, call)                                   \
    do {                                                             \
        cudaError_t _e = (call);                                     \
        if (_e != cudaSuccess) return txs::cuda_fail(ctx, stage, _e); \
    } while (0)

#define TXS_LAUNCHED(ctx, stage)                                                \
    do {                                                                        \
        ++(ctx)->launches;                                                      \
        cudaError_t _e = cudaGetLastError();                                    \
        if (_e != cudaSuccess) return txs::cuda_fail(ctx, stage, _e);           \
    } while (0)
