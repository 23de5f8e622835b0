/*
 * txsite_b200.h — C-ABI drop-in boundary of the B200-native multiple-observer
 * siting engine (arXiv 2006.16783; contract /root/reference/SPEC.md).
 *
 * The reference's boundary is the C++ stage API of namespace txsite
 * (SPEC.md:176 estimate_vix, :228 partition, :238 find_candidates,
 * :305 compute_all_viewsheds, :364 site, :433 run_pipeline) inside static lib
 * txsite_core (proj/CMakeLists.txt:13-26).  The reference ships no binary ABI
 * and no FFI (src/ is absent), so each entry point below names
 * the SPEC operation it replaces; include/txsite/txsite.hpp re-exposes them as
 * that C++ API and INTEGRATION.md shows the bindings (C++, ctypes).
 *
 * Conventions
 *  - plain pointers and sizes only; host buffers are owned by the caller;
 *  - every function returns txs_status; on failure txs_last_error(ctx) holds a
 *    stage-tagged message ("stage-tagged message");
 *  - stage outputs stay resident in HBM inside the context; the *_out host
 *    pointers are optional copies (NULL = keep on device only);
 *  - calls are synchronous at stage granularity; a context is not thread-safe;
 *  - there is no CPU fallback: without a usable sm_100 device txs_create fails.
 */
#ifndef TXSITE_B200_H
#define TXSITE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TXS_ABI_VERSION 1

typedef enum txs_status {
    TXS_OK = 0,
    TXS_ERR_INVALID_ARGUMENT = 1, /* roi < 1, roi < 3 for partition (:232), zmin > zmax (:65) ... */
    TXS_ERR_OFF_GRID = 2,         /* off-grid base point                                        */
    TXS_ERR_STATE = 3,            /* a stage called before its input exists                                     */
    TXS_ERR_CUDA = 4,             /* CUDA runtime / no sm_100 device                                            */
    TXS_ERR_OUT_OF_MEMORY = 5,
    TXS_ERR_RANGE = 6,            /* exceeds the exact-integer arithmetic envelope (DESIGN.md §2 D2)            */
    TXS_ERR_SIZE_MISMATCH = 7,
    TXS_ERR_NODATA = 8            /* NODATA sentinel -32768 rejected                              */
} txs_status;

/* SitingResult.stop_reason + max_selected. */
typedef enum txs_stop {
    TXS_STOP_TARGET_REACHED = 0,
    TXS_STOP_ZERO_GAIN = 1,
    TXS_STOP_EXHAUSTED = 2,
    TXS_STOP_MAX_SELECTED = 3
} txs_stop;

/* LOS arithmetic (txs_params.los_arith; DESIGN.md §2 D2).  TXS_LOS_FP64 is
 * SPEC.md:147's formula ("All LOS arithmetic in double-precision floating
 * point"): VIX/LOS decisions and viewshed bits identical to the fp64 oracle.
 * TXS_LOS_EXACT is SPEC.md:120's real-number predicate in exact integers; the
 * two differ only where the terrain touches the LOS exactly (grazing ties,
 * ~1e-4 of LOS decisions), which fp64 rounding decides either way. */
typedef enum txs_los_arith { TXS_LOS_FP64 = 0, TXS_LOS_EXACT = 1 } txs_los_arith;

/* SiteParams plus the knobs the BASELINE configs need. */
typedef struct txs_params {
    int32_t roi;               /* radius of interest in posts, >= 1                       */
    int32_t tx_height;         /* h_t, integer elevation units, >= 0                       */
    int32_t rx_height;         /* h_r                                                      */
    int32_t samples_per_point; /* VIX samples per post (default 10), 1..255                */
    int32_t per_block;         /* FINDMAX top-k per block (default 20)                     */
    int32_t block_width;       /* 0 => ceil(roi/3); BASELINE fixes it        */
    int32_t site_mode;         /* 0 = exact incremental gains, 1 = full rescan each round  */
    int32_t los_arith;         /* TXS_LOS_FP64 (0, default) or TXS_LOS_EXACT (1), below      */
    double target_coverage;    /* (0,1]                                                    */
    int64_t max_selected;      /* 0 => unlimited                             */
    uint64_t seed;             /* VIX sampling seed                          */
} txs_params;

typedef struct txs_candidate { int32_t row, col, score, _pad; } txs_candidate;
typedef struct txs_window { int32_t row0, col0, h, w; } txs_window;
typedef struct txs_step {
    int64_t index;    /* candidate index (block order) */
    int32_t row, col; /* transmitter base                            */
    int64_t gain;     /* marginal gain in cells                      */
    double coverage;  /* cumulative coverage after this step         */
} txs_step;

/* Per-stage device timings (CUDA events on the context stream) and the
 * algorithmic work counters the roofline figures are computed from. */
typedef struct txs_stats {
    double ms_terrain, ms_vix, ms_findmax, ms_viewshed, ms_site;
    int64_t vix_los;                /* sampled LOS segments tested                          */
    int64_t vix_crossings_full;     /* interior crossings of those segments, no early exit  */
    int64_t viewshed_crossings;     /* R2 ray crossings evaluated (in-grid, no early exit)  */
    int64_t viewshed_cells;         /* disk cells tested                                    */
    int64_t site_iterations;
    int64_t site_bytes;             /* packed viewshed bytes streamed by the gain kernels    */
    int64_t site_launches;          /* kernels launched by the SITE loop                     */
    int64_t candidates;
    int64_t kernel_launches;        /* every kernel this context launched since reset        */
    double ms_site_rounds;          /* device time of the SITE round loop alone (no setup)   */
    /* fp64 LOS arithmetic (TXS_LOS_FP64): exact grazing ties found by the exact
     * walks and re-decided with SPEC.md:147's formula, and how many of those
     * decisions fp64 rounding changed (VIX: segments; VIEWSHED: rays / bits). */
    int64_t vix_fp64_ties, vix_fp64_flips;
    int64_t vs_fp64_ties, vs_fp64_flips;
    /* device time of the stage's main kernel alone (k_vix_quads / k_vix, the
     * VIEWSHED sweep), CUDA events on the context stream around that launch */
    double ms_vix_kernel, ms_viewshed_kernel;
    /* HBM held by the context's resident buffers (terrain, planes, VixMap,
     * candidates, viewsheds, bitmaps, SITE state): now, and the high-water mark
     * since creation (RunReport's peak memory estimate) */
    int64_t device_bytes, device_bytes_peak;
    /* persistent SITE loop, CTA 0's device time per phase over the whole loop
     * (set with TXS_SITE_PROFILE=1, else 0): winner reduction, commit of the
     * previous winner, neighbour updates, partial argmax, grid barrier */
    int64_t site_phase_ns[5];
} txs_stats;

typedef struct txs_ctx txs_ctx;

int txs_abi_version(void);
/* 1 if a CUDA device with compute capability 10.x is visible. */
int txs_device_ok(void);

txs_status txs_create(int device, txs_ctx** out);
void txs_destroy(txs_ctx* ctx);
const char* txs_last_error(const txs_ctx* ctx);
txs_status txs_get_stats(txs_ctx* ctx, txs_stats* out);
txs_status txs_reset_stats(txs_ctx* ctx);
txs_status txs_synchronize(txs_ctx* ctx);
/* Device-side timing on the context stream: record event `slot` (0..15) now;
 * elapsed milliseconds between two recorded slots (waits for slot b). */
txs_status txs_event_record(txs_ctx* ctx, int slot);
txs_status txs_event_elapsed(txs_ctx* ctx, int slot_a, int slot_b, double* ms);

/* ---- terrain module ---------------------------------------- */
/* load_binary's in-memory result: row-major int16, copied to HBM. */
txs_status txs_set_terrain(txs_ctx* ctx, const int16_t* z, int64_t nrows, int64_t ncols);
/* generate_fractal, decision D10; generated directly in HBM. */
txs_status txs_generate_fractal(txs_ctx* ctx, int64_t nrows, int64_t ncols, double roughness,
                                uint64_t seed, int32_t zmin, int32_t zmax);
/* Config-3 water clamp: rows [row_begin,row_end) set to value. */
txs_status txs_fill_rows(txs_ctx* ctx, int64_t row_begin, int64_t row_end, int16_t value);
txs_status txs_get_terrain(txs_ctx* ctx, int16_t* z_out);
txs_status txs_terrain_dims(const txs_ctx* ctx, int64_t* nrows, int64_t* ncols);

/* ---- los module — batch form for parity tests --------------- */
/* pairs: n x {tx_row, tx_col, rx_row, rx_col}; out: n bytes 0/1; los_arith as
 * in txs_params. */
txs_status txs_is_visible_batch(txs_ctx* ctx, const int32_t* pairs, int64_t n, int32_t tx_height,
                                int32_t rx_height, int32_t los_arith, uint8_t* out);

/* ---- vix module (SPEC.md:176 estimate_vix) ------------------------------------ */
txs_status txs_estimate_vix(txs_ctx* ctx, const txs_params* p, uint8_t* scores_out);
txs_status txs_set_vix(txs_ctx* ctx, const uint8_t* scores);  /* inject a VixMap */
/* copy rows [row_begin, row_end) of the resident VixMap (band rows when sharded) */
txs_status txs_get_vix(txs_ctx* ctx, int64_t row_begin, int64_t row_end, uint8_t* scores_out);

/* ---- candidates module (SPEC.md:228 partition, :238 find_candidates) ------- */
txs_status txs_partition(int64_t nrows, int64_t ncols, int32_t roi, int32_t block_width,
                         int64_t* bw_out, int64_t* blocks_x, int64_t* blocks_y);
txs_status txs_find_candidates(txs_ctx* ctx, const txs_params* p, int64_t* n_out,
                               txs_candidate* out, int64_t cap);
txs_status txs_set_candidates(txs_ctx* ctx, const txs_candidate* c, int64_t n);
/* Config 5: n uniformly random observers, row = next_below(nrows) then
 * col = next_below(ncols) from SplitMix64(seed) (decision D11). */
txs_status txs_random_observers(txs_ctx* ctx, int64_t n, uint64_t seed);
txs_status txs_get_candidates(txs_ctx* ctx, txs_candidate* out, int64_t cap, int64_t* n_out);
/* Global candidate ids of the resident candidates (index i -> base + i, or the
 * draw index of a sharded random observer): the ids SITE steps report. */
txs_status txs_get_candidate_ids(txs_ctx* ctx, int64_t* ids_out, int64_t cap, int64_t* n_out);

/* ---- viewshed module (SPEC.md:305 compute_all_viewsheds) ------------------- */
txs_status txs_compute_viewsheds(txs_ctx* ctx, const txs_params* p);
/* words_stride >= ceil((2roi+1)^2/64); popcounts optional. */
txs_status txs_get_viewsheds(txs_ctx* ctx, int64_t first, int64_t count, txs_window* wins,
                             uint64_t* words, int64_t words_stride, int64_t* popcounts);
/* Inject packed viewsheds (for SITE parity on given input). */
txs_status txs_set_viewsheds(txs_ctx* ctx, int32_t roi, int64_t n, const int32_t* rows,
                             const int32_t* cols, const txs_window* wins, const uint64_t* words,
                             int64_t words_stride);

/* ---- siting module (SPEC.md:364 site, :374 marginal_gain, :384 coverage) --- */
txs_status txs_site(txs_ctx* ctx, const txs_params* p, txs_step* steps, int64_t cap,
                    int64_t* nsteps, int32_t* stop_reason);
/* CumulativeShed words: dense row-major, (nrows*ncols+63)/64. */
txs_status txs_get_cumulative(txs_ctx* ctx, uint64_t* words_out);
/* marginal_gain of every resident viewshed against a caller cum (dense). */
txs_status txs_marginal_gains(txs_ctx* ctx, const uint64_t* cum_dense, int64_t* gains_out);
/* Measurement: `reps` full gain passes (popc(v_i & ~cum) for every candidate, the
 * full-rescan SITE kernel) against the context's current cumulative bitmap (after
 * txs_site), timed with CUDA events on the context stream; the incremental gains
 * are overwritten.  ms_per_pass = mean device time of one pass, bytes_per_pass =
 * packed viewshed bytes streamed (SPEC layout, algorithmic). */
txs_status txs_time_gain_pass(txs_ctx* ctx, int32_t reps, double* ms_per_pass, int64_t* bytes_per_pass);
/* Measurement: L2-resident read bandwidth (GB/s) -- `reps` passes of 16-byte
 * loads over a `bytes` buffer that fits the L2, timed with CUDA events on the
 * context stream (the peak the VIX / VIEWSHED LOS-sample figures are set
 * against). */
txs_status txs_measure_cache_read(txs_ctx* ctx, int64_t bytes, int32_t reps, double* gbs);

/* ---- cli module (SPEC.md:433 run_pipeline) ---------------------------------- */
/* vix -> findmax -> viewshed -> site on the resident terrain, device-resident
 * in between; stage_ms[4] = {vix, findmax, viewshed, site}. */
txs_status txs_run_pipeline(txs_ctx* ctx, const txs_params* p, txs_step* steps, int64_t cap,
                            int64_t* nsteps, int32_t* stop_reason, double* stage_ms);

/* run_pipeline straight from a host terrain (load_binary's result, SPEC.md:41 +
 * :433): the rows go up in ~16 chunks on a copy stream while VIX runs band by
 * band behind them (each band waits only for the rows its walks and skip-map
 * corners reach), so the upload overlaps the dominant stage; NODATA is checked
 * once the rows are in.  Same results as txs_set_terrain + txs_run_pipeline
 * (which it is, on a sharded context).  z should be pinned for the overlap. */
txs_status txs_run_pipeline_host(txs_ctx* ctx, const int16_t* z, int64_t nrows, int64_t ncols, const txs_params* p,
                                 txs_step* steps, int64_t cap, int64_t* nsteps, int32_t* stop_reason, double* stage_ms);

/* ---- multi-GPU row-band shards ---------------------------------
 * A sharded context owns rows [row_begin,row_end) of a global nrows x ncols grid
 * and holds terrain rows [max(0,row_begin-halo), min(nrows,row_end+halo)).
 * Terrain input is those rows (txs_set_terrain) or the global generator
 * (txs_generate_fractal with the global dims, cropped on the device).  VIX and
 * FINDMAX cover the band only (bands align to FINDMAX block rows); candidate
 * global ids are base + local index (txs_set_candidate_base), or the global
 * draw index for txs_random_observers.  SITE runs as rounds driven by the
 * caller: every rank reports its local best key, the caller reduces the max
 * across ranks (the one collective), the owner exports the winner's window,
 * every rank applies it.  No collective runs inside the engine. */
txs_status txs_set_shard(txs_ctx* ctx, int64_t nrows, int64_t ncols, int64_t row_begin, int64_t row_end,
                         int32_t halo);
txs_status txs_shard_info(const txs_ctx* ctx, int64_t* held_row0, int64_t* held_rows, int64_t* band_begin,
                          int64_t* band_end);
txs_status txs_set_candidate_base(txs_ctx* ctx, int64_t gid0);
txs_status txs_site_shard_begin(txs_ctx* ctx, const txs_params* p);
/* key = (gain << 32) | (0xffffffff - global id) of the best local candidate, 0 if none */
txs_status txs_site_shard_best(txs_ctx* ctx, uint64_t* key);
/* If this rank owns global id gid: *owned = 1 and its observer position,
 * window and packed words (words_stride u64) are written. */
txs_status txs_site_shard_export(txs_ctx* ctx, int64_t gid, int32_t* owned, int32_t* row, int32_t* col,
                                 txs_window* win, uint64_t* words, int64_t words_stride);
/* OR the winner window into the held cum rows and update the local gains. */
txs_status txs_site_shard_apply(txs_ctx* ctx, int32_t row, int32_t col, const txs_window* win,
                                const uint64_t* words);

/* Device-resident form of the same round (no host round trip; for
 * collectives issued on the context stream, e.g. NCCL through
 * torch.distributed on txs_stream()):
 *   txs_site_shard_best_dev    d_key[0] = this rank's best key (0 once stopped)
 *   -- caller: allreduce(MAX) of d_key over the ranks --
 *   txs_site_shard_export_dev  d_payload = the winner's {row, col, row0, col0, h, w,
 *                              cum-aligned words} if this rank owns it, else zeros
 *                              (txs_site_shard_payload_words() u64)
 *   -- caller: allreduce(SUM) of d_payload (a broadcast from the data-dependent owner) --
 *   txs_site_shard_apply_dev   stop rules (decision D9, total_candidates = global
 *                              count), step record, cum OR + local gain updates;
 *                              rounds after the stop are no-ops
 * txs_site_shard_result copies the recorded steps and the stop reason (-1 while
 * running).  All three calls are stream-ordered and return without waiting. */
txs_status txs_site_shard_best_dev(txs_ctx* ctx, uint64_t* d_key);
txs_status txs_site_shard_export_dev(txs_ctx* ctx, const uint64_t* d_key, uint64_t* d_payload);
txs_status txs_site_shard_apply_dev(txs_ctx* ctx, const uint64_t* d_key, const uint64_t* d_payload,
                                    int64_t total_candidates);
int64_t txs_site_shard_payload_words(const txs_ctx* ctx);
/* One-collective form of the same round (one allgather instead of the two
 * allreduces above):
 *   txs_site_shard_best_dev
 *   txs_site_shard_export_keyed_dev  d_out[0] = d_key[0] (this rank's best key),
 *                                    d_out[1..] = that candidate's payload
 *                                    (1 + txs_site_shard_payload_words() u64)
 *   -- caller: allgather of d_out over the ranks, rank-major --
 *   txs_site_shard_select_dev        d_key / d_payload = the entry with the largest
 *                                    key (gain desc, global id asc: the allreduce(MAX)
 *                                    winner), its payload
 *   txs_site_shard_apply_dev */
txs_status txs_site_shard_export_keyed_dev(txs_ctx* ctx, const uint64_t* d_key, uint64_t* d_out);
txs_status txs_site_shard_select_dev(txs_ctx* ctx, const uint64_t* d_gathered, int32_t nranks, uint64_t* d_key,
                                     uint64_t* d_payload);
txs_status txs_site_shard_result(txs_ctx* ctx, txs_step* steps, int64_t cap, int64_t* nsteps, int32_t* stop_reason);
/* The context's CUDA stream (a cudaStream_t), for ordering external work with it. */
void* txs_stream(txs_ctx* ctx);

/* ---- replicated SITE over gathered viewsheds -------------------
 * The other multi-GPU SITE form: one allgather of every band's candidates and
 * packed viewsheds, then the single-GPU SITE loop (no collective per round) on
 * the gathered set -- the same picks, bit for bit, since the gathered set IS the
 * single-GPU candidate list.  A record is txs_viewshed_record_words(roi) u64:
 *   [0] global candidate id (-1: padding)   [1] row | col << 32
 *   [2..3] window {row0, col0, h, w} (int32) [4] popcount | FINDMAX score << 32
 *   [5..] the engine's cum-aligned row words (txs_viewsheds_device layout)
 * txs_viewsheds_pack writes the context's resident viewsheds as `slots`
 * records into a device buffer (padding past its count), stream-ordered on
 * txs_stream (for collectives issued there). */
int64_t txs_viewshed_record_words(int32_t roi);
txs_status txs_viewsheds_pack(txs_ctx* ctx, int64_t slots, uint64_t* d_records, int64_t* n_out);
/* SITE (p's stop rules) on `nrec` gathered records holding the
 * n_total candidates of the whole grid (each placed at its global id).  The
 * context's own candidates and viewsheds are replaced; afterwards
 * txs_get_cumulative returns the whole grid's cumulative viewshed. */
txs_status txs_site_gathered(txs_ctx* ctx, const txs_params* p, int64_t nrec, int64_t n_total, const uint64_t* d_records,
                             txs_step* steps, int64_t cap, int64_t* nsteps, int32_t* stop_reason);
/* OR the bits of global rows [row_begin, row_end) of the context's cumulative
 * viewshed (the held cum rows; rows outside them read as 0) into `dense_out`,
 * the caller's SPEC-dense bitmap of the WHOLE grid ((nrows*ncols+63)/64 words,
 * SPEC.md:351).  Words wholly inside the rows are overwritten, the (at most two)
 * words shared with neighbouring rows are OR-ed atomically, so row bands of
 * several contexts may be assembled into one buffer concurrently.  The dense
 * words are formed on the device; only the band's words cross PCIe. */
txs_status txs_get_cumulative_rows(txs_ctx* ctx, int64_t row_begin, int64_t row_end, uint64_t* dense_out);

/* ---- native multi-GPU group (SURVEY §8(b) txs_create(ngpus, devices)) ----
 * One process, one host thread per call, N contexts (one per device, or several
 * on one device for testing).  The group plans the row bands (FINDMAX block rows,
 * roi+1 halo), runs VIX / FINDMAX / VIEWSHED on every band concurrently (one
 * worker thread per rank: no collective), assigns global candidate ids by the
 * prefix of band counts, and drives the SITE rounds with one of three winner
 * exchanges:
 *   TXS_XCHG_P2P   every rank writes {its best key, payload} into its
 *                  own device mailbox; every rank's select kernel reads the N
 *                  keys and then the winner's window words straight out of the
 *                  winner rank's mailbox over NVLink peer memory (cross-device
 *                  ordering by CUDA events, double-buffered mailboxes); the
 *                  rounds of all ranks are captured as ONE multi-device CUDA
 *                  graph of 16 rounds and replayed until the device stop flag;
 *   TXS_XCHG_NCCL  one ncclAllGather of {key, payload} per round over the
 *                  group's communicators (ncclCommInitAll; distinct devices),
 *                  also graph-captured;
 *   TXS_XCHG_HOST  host-staged rounds (keys and the owner's window through host
 *                  memory; txs_site_shard_best/export/apply) -- the reference
 *                  formulation, and the only exchange available with custom ops;
 *   TXS_XCHG_REPLICATE (default, below) gathers the viewsheds once instead.
 * All three give the single-context pick sequence and cumulative bitmap. */
typedef enum txs_exchange {
    TXS_XCHG_P2P = 0, TXS_XCHG_NCCL = 1, TXS_XCHG_HOST = 2,
    /* no exchange per round: every band's packed viewsheds are copied once to
     * rank 0 (peer copies) and rank 0 runs the single-GPU SITE loop on them
     * (txs_site_gathered) -- the default: ~6 us per round at roi 100 against
     * a cross-GPU exchange's latency per round */
    TXS_XCHG_REPLICATE = 3
} txs_exchange;

/* Stage entry points the group drives (defaults: the functions above).  A test
 * may substitute a CPU stand-in; only TXS_XCHG_HOST works with substituted ops. */
typedef struct txs_engine_ops {
    txs_status (*create)(int device, txs_ctx** out);
    void (*destroy)(txs_ctx* ctx);
    const char* (*last_error)(const txs_ctx* ctx);
    txs_status (*set_shard)(txs_ctx*, int64_t nrows, int64_t ncols, int64_t row_begin, int64_t row_end, int32_t halo);
    txs_status (*shard_info)(const txs_ctx*, int64_t* held_row0, int64_t* held_rows, int64_t* band_begin, int64_t* band_end);
    txs_status (*set_terrain)(txs_ctx*, const int16_t* z, int64_t nrows, int64_t ncols);
    txs_status (*generate_fractal)(txs_ctx*, int64_t nrows, int64_t ncols, double roughness, uint64_t seed,
                                   int32_t zmin, int32_t zmax);
    txs_status (*fill_rows)(txs_ctx*, int64_t row_begin, int64_t row_end, int16_t value);
    txs_status (*estimate_vix)(txs_ctx*, const txs_params* p, uint8_t* scores_out);
    txs_status (*find_candidates)(txs_ctx*, const txs_params* p, int64_t* n_out, txs_candidate* out, int64_t cap);
    txs_status (*random_observers)(txs_ctx*, int64_t n, uint64_t seed);
    txs_status (*get_candidates)(txs_ctx*, txs_candidate* out, int64_t cap, int64_t* n_out);
    txs_status (*set_candidate_base)(txs_ctx*, int64_t gid0);
    txs_status (*compute_viewsheds)(txs_ctx*, const txs_params* p);
    txs_status (*site_shard_begin)(txs_ctx*, const txs_params* p);
    txs_status (*site_shard_best)(txs_ctx*, uint64_t* key);
    txs_status (*site_shard_export)(txs_ctx*, int64_t gid, int32_t* owned, int32_t* row, int32_t* col,
                                    txs_window* win, uint64_t* words, int64_t words_stride);
    txs_status (*site_shard_apply)(txs_ctx*, int32_t row, int32_t col, const txs_window* win, const uint64_t* words);
    txs_status (*get_cumulative_rows)(txs_ctx*, int64_t row_begin, int64_t row_end, uint64_t* dense_out);
    txs_status (*get_stats)(txs_ctx*, txs_stats* out);
} txs_engine_ops;
const txs_engine_ops* txs_default_ops(void);

typedef struct txs_group txs_group;
/* Row bands of nrows over `world` ranks by whole FINDMAX block rows (the split
 * of shard.py's plan_bands): out[2k], out[2k+1] = rank k's [row_begin, row_end).
 * Host-only.  TXS_ERR_INVALID_ARGUMENT when world exceeds the block rows. */
txs_status txs_plan_bands(int64_t nrows, int64_t block, int32_t world, int64_t* out);
txs_status txs_group_create(int ngpus, const int* devices, txs_group** out);
txs_status txs_group_create_with_ops(int ngpus, const int* devices, const txs_engine_ops* ops, txs_group** out);
void txs_group_destroy(txs_group* g);
const char* txs_group_last_error(const txs_group* g);
int32_t txs_group_size(const txs_group* g);
txs_ctx* txs_group_context(txs_group* g, int32_t rank);
txs_status txs_group_set_exchange(txs_group* g, int32_t exchange);
/* Plan the bands (block = p->block_width, or ceil(roi/3); halo roi+1) and make
 * every rank a shard of the nrows x ncols grid.  Call before the terrain. */
txs_status txs_group_set_grid(txs_group* g, int64_t nrows, int64_t ncols, const txs_params* p);
txs_status txs_group_band(const txs_group* g, int32_t rank, int64_t* row_begin, int64_t* row_end);
/* Terrain: the whole row-major grid from the host (each rank copies its band +
 * halo rows), or the D10 generator on every rank's device (cropped). */
txs_status txs_group_set_terrain(txs_group* g, const int16_t* z);
txs_status txs_group_generate_fractal(txs_group* g, double roughness, uint64_t seed, int32_t zmin, int32_t zmax);
txs_status txs_group_fill_rows(txs_group* g, int64_t row_begin, int64_t row_end, int16_t value);
/* Config 5: the n global draws of decision D11; every rank keeps its band's
 * observers (ids = draw index).  The next txs_group_run_pipeline then skips
 * VIX/FINDMAX. */
txs_status txs_group_random_observers(txs_group* g, int64_t n, uint64_t seed);
/* VIX -> FINDMAX -> VIEWSHED on every band, then the SITE rounds; stage_ms[4] =
 * device ms of {vix, findmax, viewshed, site} (max over ranks; site = the
 * rounds incl. the exchange). */
txs_status txs_group_run_pipeline(txs_group* g, const txs_params* p, txs_step* steps, int64_t cap,
                                  int64_t* nsteps, int32_t* stop_reason, double* stage_ms);
/* Global dense cumulative bitmap, assembled from every rank's band rows. */
txs_status txs_group_get_cumulative(txs_group* g, uint64_t* dense_out);

/* ---- host-only helpers (no GPU needed; used by the CPU test-suite) -------- */
/* The frozen D5 ray template for roi: returns ray count; arrays filled when the
 * caps suffice.  cell_begin has rays+1 entries. */
int64_t txs_ray_template(int32_t roi, int32_t* p, int32_t* q, int64_t* cell_begin, int32_t* ca,
                         int32_t* cb, int64_t cap_rays, int64_t cap_cells, int64_t* ncells);
/* Size of the VIEWSHED event stream for roi (<= 250): events, events incl.
 * warp padding, 32-ray groups.  0 = ok. */
int txs_event_template_info(int32_t roi, int64_t* real_events, int64_t* padded_events, int32_t* groups);
/* Self-test of host-side integer helpers (exact 64-bit division magic). 0 = ok. */
int txs_selftest(void);

#ifdef __cplusplus
}
#endif
#endif /* TXSITE_B200_H */
