// C++ stage API of the reference (include/txsite/txsite.hpp) over the B200
// engine's C-ABI.  Host code only: every LOS / viewshed / gain evaluation runs
// in the sm_100a kernels behind include/txsite_b200.h.
#include "txsite/txsite.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <mutex>
#include <sstream>

#include "txsite_b200.h"

namespace txsite {

namespace {

void check(txs_ctx* c, txs_status st) {
    if (st != TXS_OK) throw Error((int)st, c ? txs_last_error(c) : "txsite: invalid argument");
}

txs_params to_params(const SiteParams& p, uint64_t seed = 0) {
    txs_params q{};
    q.roi = p.roi;
    q.tx_height = p.tx_height;
    q.rx_height = p.rx_height;
    q.samples_per_point = p.samples_per_point;
    q.per_block = p.per_block;
    q.block_width = p.block_width;
    q.site_mode = p.site_mode;
    q.los_arith = p.los_arith;
    q.target_coverage = p.target_coverage;
    q.max_selected = p.max_selected;
    q.seed = seed;
    return q;
}

// the shared context behind the value-type calls
std::mutex g_mu;
txs_ctx* g_ctx = nullptr;
txs_ctx* shared_ctx() {
    if (!g_ctx) {
        txs_status st = txs_create(0, &g_ctx);
        if (st != TXS_OK) throw Error((int)st, "txsite: no usable sm_100 device (the engine has no CPU fallback)");
    }
    return g_ctx;
}

void upload(txs_ctx* c, const TerrainGrid& g) {
    if ((int64_t)g.elevations.size() != g.nrows * g.ncols)
        throw Error(TXS_ERR_SIZE_MISMATCH, "[read] elevations size != nrows*ncols");
    check(c, txs_set_terrain(c, g.elevations.data(), g.nrows, g.ncols));
}

std::vector<Viewshed> download_viewsheds(txs_ctx* c, int32_t roi, int64_t n) {
    const int64_t stride = ((2 * (int64_t)roi + 1) * (2 * (int64_t)roi + 1) + 63) / 64;
    std::vector<txs_window> wins((size_t)n);
    std::vector<uint64_t> words((size_t)(n * stride));
    std::vector<txs_candidate> cand((size_t)n);
    int64_t nc = 0;
    if (n) {
        check(c, txs_get_viewsheds(c, 0, n, wins.data(), words.data(), stride, nullptr));
        check(c, txs_get_candidates(c, cand.data(), n, &nc));
    }
    std::vector<Viewshed> out((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        Viewshed& v = out[(size_t)i];
        v.origin = {cand[(size_t)i].row, cand[(size_t)i].col};
        v.roi = roi;
        v.row0 = wins[(size_t)i].row0; v.col0 = wins[(size_t)i].col0; v.h = wins[(size_t)i].h; v.w = wins[(size_t)i].w;
        const int64_t nw = ((int64_t)v.h * v.w + 63) / 64;
        v.words.assign(words.begin() + i * stride, words.begin() + i * stride + nw);
    }
    return out;
}

SitingResult run_site(txs_ctx* c, const SiteParams& p, int64_t ncand, bool with_cum) {
    const txs_params q = to_params(p);
    std::vector<txs_step> steps((size_t)ncand + 1);
    int64_t ns = 0;
    int32_t stop = 0;
    check(c, txs_site(c, &q, steps.data(), (int64_t)steps.size(), &ns, &stop));
    SitingResult r;
    std::vector<txs_candidate> cand((size_t)std::max<int64_t>(ncand, 1));
    int64_t nc = 0;
    if (ncand) check(c, txs_get_candidates(c, cand.data(), ncand, &nc));
    for (int64_t k = 0; k < ns; ++k) {
        const txs_step& s = steps[(size_t)k];
        r.selected.push_back({s.index, {{s.row, s.col}, cand[(size_t)s.index].score}, s.gain, s.coverage});
    }
    r.stop_reason = (StopReason)stop;
    r.final_coverage = r.selected.empty() ? 0.0 : r.selected.back().cumulative_coverage;
    if (with_cum) {
        int64_t nr = 0, ncol = 0;
        check(c, txs_terrain_dims(c, &nr, &ncol));
        r.cumulative.nrows = nr;
        r.cumulative.ncols = ncol;
        r.cumulative.words.resize((size_t)((nr * ncol + 63) / 64));
        check(c, txs_get_cumulative(c, r.cumulative.words.data()));
    }
    return r;
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

// ---- terrain -----------------------------------------------------------------------
TerrainGrid load_binary(const std::string& path, int64_t nrows, int64_t ncols) {
    std::ifstream f(path, std::ios::binary | std::ios::ate);
    if (!f) throw Error(TXS_ERR_INVALID_ARGUMENT, "[read] file-missing: " + path);
    const std::streamsize bytes = f.tellg();
    if (bytes != (std::streamsize)(nrows * ncols * 2))
        throw Error(TXS_ERR_SIZE_MISMATCH, "[read] size-mismatch: " + path);
    TerrainGrid g;
    g.nrows = nrows;
    g.ncols = ncols;
    g.elevations.resize((size_t)(nrows * ncols));
    f.seekg(0);
    f.read(reinterpret_cast<char*>(g.elevations.data()), bytes);   // little-endian hosts
    for (int16_t v : g.elevations)
        if (v == -32768) throw Error(TXS_ERR_NODATA, "[read] NODATA sentinel -32768");
    return g;
}

void write_binary(const TerrainGrid& g, const std::string& path) {
    std::ofstream f(path, std::ios::binary);
    f.write(reinterpret_cast<const char*>(g.elevations.data()), (std::streamsize)(g.elevations.size() * 2));
}

TerrainGrid load_ascii_grid(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw Error(TXS_ERR_INVALID_ARGUMENT, "[read] file-missing: " + path);
    std::string k1, k2;
    TerrainGrid g;
    if (!(f >> k1 >> g.nrows >> k2 >> g.ncols) || k1 != "nrows" || k2 != "ncols")
        throw Error(TXS_ERR_INVALID_ARGUMENT, "[read] parse-failure at line 1 (header \"nrows N ncols M\")");
    g.elevations.resize((size_t)(g.nrows * g.ncols));
    for (size_t i = 0; i < g.elevations.size(); ++i) {
        long v;
        if (!(f >> v)) throw Error(TXS_ERR_INVALID_ARGUMENT, "[read] parse-failure at value " + std::to_string(i));
        g.elevations[i] = (int16_t)v;
    }
    return g;
}

void write_ascii_grid(const TerrainGrid& g, const std::string& path) {
    std::ofstream f(path);
    f << "nrows " << g.nrows << " ncols " << g.ncols << "\n";
    for (int64_t r = 0; r < g.nrows; ++r) {
        for (int64_t c = 0; c < g.ncols; ++c) f << (c ? " " : "") << g.at(r, c);
        f << "\n";
    }
}

TerrainGrid generate_fractal(int64_t nrows, int64_t ncols, double roughness, uint64_t seed, int32_t zmin, int32_t zmax) {
    std::lock_guard<std::mutex> lk(g_mu);
    txs_ctx* c = shared_ctx();
    check(c, txs_generate_fractal(c, nrows, ncols, roughness, seed, zmin, zmax));
    TerrainGrid g;
    g.nrows = nrows;
    g.ncols = ncols;
    g.elevations.resize((size_t)(nrows * ncols));
    check(c, txs_get_terrain(c, g.elevations.data()));
    return g;
}

double elevation_between(const TerrainGrid& g, GridPoint p, GridPoint q, double frac) {
    const int64_t d = std::llabs(p.row - q.row) + std::llabs(p.col - q.col);
    if (d > 1) throw Error(TXS_ERR_INVALID_ARGUMENT, "[los] elevation_between: non-adjacent posts");
    return g.at(p.row, p.col) * (1.0 - frac) + g.at(q.row, q.col) * frac;
}

// ---- los -----------------------------------------------------------------------------
std::vector<uint8_t> is_visible_batch(const TerrainGrid& g, const std::vector<GridPoint>& tx,
                                      const std::vector<GridPoint>& rx, int32_t ht, int32_t hr,
                                      int32_t los_arith) {
    if (tx.size() != rx.size()) throw Error(TXS_ERR_SIZE_MISMATCH, "[los] tx/rx size mismatch");
    std::vector<int32_t> pairs(4 * tx.size());
    for (size_t i = 0; i < tx.size(); ++i) {
        pairs[4 * i] = (int32_t)tx[i].row; pairs[4 * i + 1] = (int32_t)tx[i].col;
        pairs[4 * i + 2] = (int32_t)rx[i].row; pairs[4 * i + 3] = (int32_t)rx[i].col;
    }
    std::lock_guard<std::mutex> lk(g_mu);
    txs_ctx* c = shared_ctx();
    upload(c, g);
    std::vector<uint8_t> out(tx.size());
    check(c, txs_is_visible_batch(c, pairs.data(), (int64_t)tx.size(), ht, hr, los_arith, out.data()));
    return out;
}

bool is_visible(const TerrainGrid& g, const ObserverSpec& tx, const ObserverSpec& rx) {
    return is_visible_batch(g, {tx.base}, {rx.base}, tx.height, rx.height)[0] != 0;
}

// ---- vix -----------------------------------------------------------------------------
VixMap estimate_vix(const TerrainGrid& g, const SiteParams& p, uint64_t seed) {
    std::lock_guard<std::mutex> lk(g_mu);
    txs_ctx* c = shared_ctx();
    upload(c, g);
    VixMap v;
    v.nrows = g.nrows;
    v.ncols = g.ncols;
    v.samples_per_point = p.samples_per_point;
    v.scores.resize((size_t)(g.nrows * g.ncols));
    const txs_params q = to_params(p, seed);
    check(c, txs_estimate_vix(c, &q, v.scores.data()));
    return v;
}

// ---- candidates ---------------------------------------------------------------------
BlockPartition partition(int64_t nrows, int64_t ncols, int32_t roi, int32_t block_width) {
    BlockPartition b;
    check(nullptr, txs_partition(nrows, ncols, roi, block_width, &b.block_width, &b.blocks_x, &b.blocks_y));
    return b;
}

std::vector<Candidate> find_candidates(const VixMap& vix, const BlockPartition& part, int32_t per_block) {
    std::lock_guard<std::mutex> lk(g_mu);
    txs_ctx* c = shared_ctx();
    int64_t nr = 0, nc = 0;
    txs_terrain_dims(c, &nr, &nc);
    if (nr != vix.nrows || nc != vix.ncols) {   // FINDMAX needs only the VixMap: a flat placeholder terrain
        std::vector<int16_t> zero((size_t)(vix.nrows * vix.ncols), 0);
        check(c, txs_set_terrain(c, zero.data(), vix.nrows, vix.ncols));
    }
    check(c, txs_set_vix(c, vix.scores.data()));
    txs_params q{};
    q.roi = std::max<int32_t>(3, (int32_t)part.block_width);
    q.block_width = (int32_t)part.block_width;
    q.per_block = per_block;
    int64_t n = 0;
    check(c, txs_find_candidates(c, &q, &n, nullptr, 0));
    std::vector<txs_candidate> buf((size_t)n);
    if (n) check(c, txs_get_candidates(c, buf.data(), n, nullptr));
    std::vector<Candidate> out((size_t)n);
    for (int64_t i = 0; i < n; ++i) out[(size_t)i] = {{buf[(size_t)i].row, buf[(size_t)i].col}, buf[(size_t)i].score};
    return out;
}

// ---- viewshed ------------------------------------------------------------------------
std::vector<Viewshed> compute_all_viewsheds(const TerrainGrid& g, const std::vector<Candidate>& cands,
                                            const SiteParams& p) {
    std::lock_guard<std::mutex> lk(g_mu);
    txs_ctx* c = shared_ctx();
    upload(c, g);
    std::vector<txs_candidate> buf(cands.size());
    for (size_t i = 0; i < cands.size(); ++i)
        buf[i] = txs_candidate{(int32_t)cands[i].base.row, (int32_t)cands[i].base.col, cands[i].score, 0};
    check(c, txs_set_candidates(c, buf.data(), (int64_t)buf.size()));
    const txs_params q = to_params(p);
    check(c, txs_compute_viewsheds(c, &q));
    return download_viewsheds(c, p.roi, (int64_t)cands.size());
}

Viewshed compute_viewshed(const TerrainGrid& g, GridPoint tx, const SiteParams& p) {
    return compute_all_viewsheds(g, {Candidate{tx, 0}}, p).at(0);
}

int64_t popcount(const Viewshed& v) {
    int64_t s = 0;
    for (uint64_t w : v.words) s += __builtin_popcountll(w);
    return s;
}

// ---- siting --------------------------------------------------------------------------
const char* stop_reason_name(StopReason s) {
    switch (s) {
        case StopReason::TargetReached: return "target-reached";
        case StopReason::ZeroGain: return "zero-gain";
        case StopReason::CandidatesExhausted: return "candidates-exhausted";
        case StopReason::MaxSelected: return "max-selected";
    }
    return "?";
}

static void inject(txs_ctx* c, const std::vector<Viewshed>& v, int64_t nrows, int64_t ncols) {
    const int32_t roi = v.empty() ? 1 : v[0].roi;
    const int64_t stride = ((2 * (int64_t)roi + 1) * (2 * (int64_t)roi + 1) + 63) / 64;
    std::vector<int32_t> rows(v.size()), cols(v.size());
    std::vector<txs_window> wins(v.size());
    std::vector<uint64_t> words(v.size() * stride, 0);
    for (size_t i = 0; i < v.size(); ++i) {
        if (v[i].roi != roi) throw Error(TXS_ERR_INVALID_ARGUMENT, "[site] mixed roi viewsheds");
        rows[i] = (int32_t)v[i].origin.row; cols[i] = (int32_t)v[i].origin.col;
        wins[i] = txs_window{v[i].row0, v[i].col0, v[i].h, v[i].w};
        std::copy(v[i].words.begin(), v[i].words.end(), words.begin() + i * stride);
    }
    std::vector<int16_t> zero((size_t)(nrows * ncols), 0);
    check(c, txs_set_terrain(c, zero.data(), nrows, ncols));
    check(c, txs_set_viewsheds(c, roi, (int64_t)v.size(), rows.data(), cols.data(), wins.data(), words.data(), stride));
}

SitingResult site(const std::vector<Viewshed>& v, int64_t nrows, int64_t ncols, const SiteParams& p) {
    std::lock_guard<std::mutex> lk(g_mu);
    txs_ctx* c = shared_ctx();
    inject(c, v, nrows, ncols);
    SitingResult r = run_site(c, p, (int64_t)v.size(), true);
    for (auto& s : r.selected) s.candidate.base = v[(size_t)s.index].origin;
    return r;
}

int64_t marginal_gain(const Viewshed& shed, const CumulativeShed& cum) {
    std::lock_guard<std::mutex> lk(g_mu);
    txs_ctx* c = shared_ctx();
    inject(c, {shed}, cum.nrows, cum.ncols);
    int64_t g = 0;
    check(c, txs_marginal_gains(c, cum.words.data(), &g));
    return g;
}

double coverage(const CumulativeShed& cum) {
    int64_t s = 0;
    for (uint64_t w : cum.words) s += __builtin_popcountll(w);
    return (double)s / (double)(cum.nrows * cum.ncols);
}

// ---- Pipeline (device-resident) ------------------------------------------------------
Pipeline::Pipeline(int device) {
    txs_status st = txs_create(device, &ctx_);
    if (st != TXS_OK) throw Error((int)st, "txsite: no usable sm_100 device (the engine has no CPU fallback)");
}
Pipeline::~Pipeline() { txs_destroy(ctx_); }
void Pipeline::set_terrain(const TerrainGrid& g) { upload(ctx_, g); }
void Pipeline::generate_fractal(int64_t nr, int64_t nc, double rough, uint64_t seed, int32_t zmin, int32_t zmax) {
    check(ctx_, txs_generate_fractal(ctx_, nr, nc, rough, seed, zmin, zmax));
}
void Pipeline::estimate_vix(const SiteParams& p, uint64_t seed) {
    const txs_params q = to_params(p, seed);
    check(ctx_, txs_estimate_vix(ctx_, &q, nullptr));
}
int64_t Pipeline::find_candidates(const SiteParams& p) {
    const txs_params q = to_params(p);
    int64_t n = 0;
    check(ctx_, txs_find_candidates(ctx_, &q, &n, nullptr, 0));
    return n;
}
void Pipeline::fill_rows(int64_t rb, int64_t re, int16_t v) { check(ctx_, txs_fill_rows(ctx_, rb, re, v)); }
int64_t Pipeline::random_observers(int64_t n, uint64_t seed) {
    check(ctx_, txs_random_observers(ctx_, n, seed));
    return n;
}
void Pipeline::compute_all_viewsheds(const SiteParams& p) {
    const txs_params q = to_params(p);
    check(ctx_, txs_compute_viewsheds(ctx_, &q));
}
SitingResult Pipeline::site(const SiteParams& p, bool with_cum) {
    int64_t n = 0;
    check(ctx_, txs_get_candidates(ctx_, nullptr, 0, &n));
    return run_site(ctx_, p, n, with_cum);
}

// ---- cli ---------------------------------------------------------------------------------
std::string RunReport::to_string() const {
    std::ostringstream o;
    o << "stage_seconds read=" << read_s << " vix=" << vix_s << " findmax=" << findmax_s
      << " viewshed=" << viewshed_s << " site=" << site_s << " total=" << total_s << "\n"
      << "candidates=" << candidates << " selected=" << result.selected.size()
      << " final_coverage=" << result.final_coverage << " stop=" << stop_reason_name(result.stop_reason) << "\n"
      << "peak_memory_estimate device_bytes=" << device_bytes_peak << " (max over " << gpus
      << " GPU(s) of resident HBM buffers) host_bytes=" << host_bytes_peak << "\n"
      << "params " << params_echo << "\n";
    return o.str();
}

void render_cumshed(const CumulativeShed& cum, const std::string& path) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw Error(TXS_ERR_INVALID_ARGUMENT, "[render] unwritable path: " + path);
    f << "P5\n" << cum.ncols << " " << cum.nrows << "\n255\n";
    std::vector<unsigned char> row((size_t)cum.ncols);
    for (int64_t r = 0; r < cum.nrows; ++r) {
        for (int64_t c = 0; c < cum.ncols; ++c) {
            const int64_t k = r * cum.ncols + c;
            row[(size_t)c] = ((cum.words[(size_t)(k >> 6)] >> (k & 63)) & 1) ? 255 : 0;
        }
        f.write(reinterpret_cast<const char*>(row.data()), (std::streamsize)row.size());
    }
}

void render_snapshots(const SitingResult& r, const std::vector<Viewshed>& v, int64_t nrows, int64_t ncols,
                      const std::vector<int64_t>& schedule, const std::string& dir) {
    CumulativeShed cum;
    cum.nrows = nrows;
    cum.ncols = ncols;
    cum.words.assign((size_t)((nrows * ncols + 63) / 64), 0);
    size_t done = 0;
    for (int64_t k : schedule) {
        const size_t upto = std::min<size_t>((size_t)std::max<int64_t>(k, 0), r.selected.size());
        if ((size_t)k > r.selected.size())
            std::fprintf(stderr, "[render] warning: snapshot %lld > %zu selected, clamped\n", (long long)k, r.selected.size());
        for (; done < upto; ++done) {
            const Viewshed& s = v[(size_t)r.selected[done].index];
            for (int64_t y = 0; y < s.h; ++y)
                for (int64_t x = 0; x < s.w; ++x) {
                    const int64_t b = y * s.w + x;
                    if ((s.words[(size_t)(b >> 6)] >> (b & 63)) & 1) {
                        const int64_t t = (s.row0 + y) * ncols + s.col0 + x;
                        cum.words[(size_t)(t >> 6)] |= 1ull << (t & 63);
                    }
                }
        }
        render_cumshed(cum, dir + "/cumshed_" + std::to_string(k) + ".pgm");
    }
}

namespace {

std::string params_echo(const RunConfig& c, int gpus) {
    std::ostringstream o;
    o << "input=" << (c.synth || c.input.empty() ? std::string("synth") : c.input) << " nrows=" << c.nrows
      << " ncols=" << c.ncols << " seed=" << c.seed << " roughness=" << c.roughness << " zmin=" << c.zmin
      << " zmax=" << c.zmax << " water_rows=" << c.water_rows << " observers_random=" << c.observers_random
      << " observer_seed=" << c.observer_seed << " roi=" << c.params.roi << " tx_height=" << c.params.tx_height
      << " rx_height=" << c.params.rx_height << " coverage=" << c.params.target_coverage
      << " samples=" << c.params.samples_per_point << " per_block=" << c.params.per_block
      << " block_width=" << c.params.block_width << " max_selected=" << c.params.max_selected
      << " site_mode=" << c.params.site_mode << " los_arith=" << (c.params.los_arith == TXS_LOS_EXACT ? "exact" : "fp64")
      << " vix_seed=" << c.vix_seed << " gpus=" << gpus;
    if (gpus > 1)
        o << " exchange=" << (c.exchange == TXS_XCHG_NCCL ? "nccl" : c.exchange == TXS_XCHG_HOST ? "host"
                              : c.exchange == TXS_XCHG_P2P ? "p2p" : "replicate");
    return o.str();
}

int64_t host_rss_peak() {
    std::ifstream f("/proc/self/status");
    std::string line;
    while (std::getline(f, line))
        if (line.rfind("VmHWM:", 0) == 0) return std::atoll(line.c_str() + 6) * 1024;
    return 0;
}

// the resident candidates of each context in global-id order, plus the owner
// (context, local index) of every global id a step may name
struct Owners {
    std::vector<txs_ctx*> ctx;
    std::vector<std::vector<int64_t>> ids;      // per context, sorted global ids
    std::vector<std::vector<txs_candidate>> cand;
    bool find(int64_t gid, size_t* k, int64_t* li) const {
        for (size_t i = 0; i < ids.size(); ++i) {
            auto it = std::lower_bound(ids[i].begin(), ids[i].end(), gid);
            if (it != ids[i].end() && *it == gid) { *k = i; *li = it - ids[i].begin(); return true; }
        }
        return false;
    }
};

Owners owners_of(const std::vector<txs_ctx*>& ctxs) {
    Owners o;
    o.ctx = ctxs;
    for (txs_ctx* c : ctxs) {
        int64_t n = 0;
        check(c, txs_get_candidate_ids(c, nullptr, 0, &n));
        std::vector<int64_t> ids((size_t)n);
        std::vector<txs_candidate> cand((size_t)n);
        if (n) {
            check(c, txs_get_candidate_ids(c, ids.data(), n, nullptr));
            check(c, txs_get_candidates(c, cand.data(), n, nullptr));
        }
        o.ids.push_back(std::move(ids));
        o.cand.push_back(std::move(cand));
    }
    return o;
}

SitingResult to_result(const std::vector<txs_step>& steps, int32_t stop, const Owners& o) {
    SitingResult r;
    for (const txs_step& s : steps) {
        size_t k = 0;
        int64_t li = 0;
        const int32_t score = o.find(s.index, &k, &li) ? o.cand[k][(size_t)li].score : 0;
        r.selected.push_back({s.index, {{s.row, s.col}, score}, s.gain, s.coverage});
    }
    r.stop_reason = (StopReason)stop;
    r.final_coverage = r.selected.empty() ? 0.0 : r.selected.back().cumulative_coverage;
    return r;
}

// the selected transmitters' viewsheds only (SPEC layout), in step order
std::vector<Viewshed> selected_viewsheds(const SitingResult& r, const Owners& o, int32_t roi) {
    const int64_t stride = ((2 * (int64_t)roi + 1) * (2 * (int64_t)roi + 1) + 63) / 64;
    std::vector<Viewshed> out;
    std::vector<uint64_t> words((size_t)stride);
    for (const Selected& s : r.selected) {
        size_t k = 0;
        int64_t li = 0;
        if (!o.find(s.index, &k, &li)) throw Error(TXS_ERR_STATE, "[render] selected id not resident");
        txs_window w{};
        check(o.ctx[k], txs_get_viewsheds(o.ctx[k], li, 1, &w, words.data(), stride, nullptr));
        Viewshed v;
        v.origin = s.candidate.base;
        v.roi = roi;
        v.row0 = w.row0; v.col0 = w.col0; v.h = w.h; v.w = w.w;
        v.words.assign(words.begin(), words.begin() + ((int64_t)w.h * w.w + 63) / 64);
        out.push_back(std::move(v));
    }
    return out;
}

// band_ctx[k] holds VixMap rows bands[k] (every context of a group; the owners
// of the candidates may be fewer: a replicated SITE gathers them on rank 0)
void write_dumps(const RunConfig& cfg, const Owners& o, const std::vector<txs_ctx*>& band_ctx,
                 const std::vector<std::pair<int64_t, int64_t>>& bands) {
    const std::string& d = cfg.out_dir;
    if (cfg.dump_vix && cfg.observers_random == 0) {   // SPEC.md:201 row-major score bytes
        std::vector<uint8_t> v((size_t)(cfg.nrows * cfg.ncols));
        for (size_t k = 0; k < band_ctx.size(); ++k)
            check(band_ctx[k], txs_get_vix(band_ctx[k], bands[k].first, bands[k].second,
                                           v.data() + bands[k].first * cfg.ncols));
        std::ofstream(d + "/vix.u8", std::ios::binary).write(reinterpret_cast<const char*>(v.data()), (std::streamsize)v.size());
    }
    // candidates / viewsheds in global id order (ranks hold contiguous id ranges
    // in band order, or interleaved draw indices: merge by id)
    std::vector<std::pair<int64_t, std::pair<size_t, int64_t>>> order;
    for (size_t k = 0; k < o.ids.size(); ++k)
        for (size_t i = 0; i < o.ids[k].size(); ++i) order.push_back({o.ids[k][i], {k, (int64_t)i}});
    std::sort(order.begin(), order.end());
    if (cfg.dump_candidates) {
        std::ofstream f(d + "/candidates.csv");
        f << "row,col,score\n";
        for (const auto& e : order) {
            const txs_candidate& c = o.cand[e.second.first][(size_t)e.second.second];
            f << c.row << "," << c.col << "," << c.score << "\n";
        }
    }
    if (cfg.dump_viewsheds) {    // window header + packed words, little-endian
        const int32_t roi = cfg.params.roi;
        const int64_t stride = ((2 * (int64_t)roi + 1) * (2 * (int64_t)roi + 1) + 63) / 64;
        const int64_t chunk = std::max<int64_t>(1, (int64_t)(64 << 20) / (8 * stride));
        std::ofstream f(d + "/viewsheds.bin", std::ios::binary);
        std::vector<txs_window> wins;
        std::vector<uint64_t> words;
        // ranks' id ranges are each sorted: stream every rank in chunks, emit in id order
        std::vector<std::vector<std::pair<txs_window, std::vector<uint64_t>>>> cache(o.ctx.size());
        std::vector<int64_t> cached_from(o.ctx.size(), -1);
        for (const auto& e : order) {
            const size_t k = e.second.first;
            const int64_t li = e.second.second;
            if (cached_from[k] < 0 || li >= cached_from[k] + (int64_t)cache[k].size()) {
                const int64_t m = std::min<int64_t>(chunk, (int64_t)o.ids[k].size() - li);
                wins.resize((size_t)m);
                words.resize((size_t)(m * stride));
                check(o.ctx[k], txs_get_viewsheds(o.ctx[k], li, m, wins.data(), words.data(), stride, nullptr));
                cache[k].clear();
                for (int64_t i = 0; i < m; ++i) {
                    const int64_t nw = ((int64_t)wins[(size_t)i].h * wins[(size_t)i].w + 63) / 64;
                    cache[k].push_back({wins[(size_t)i], std::vector<uint64_t>(words.begin() + i * stride,
                                                                               words.begin() + i * stride + nw)});
                }
                cached_from[k] = li;
            }
            const auto& v = cache[k][(size_t)(li - cached_from[k])];
            const int32_t hdr[4] = {v.first.row0, v.first.col0, v.first.w, v.first.h};
            f.write(reinterpret_cast<const char*>(hdr), sizeof hdr);
            f.write(reinterpret_cast<const char*>(v.second.data()), (std::streamsize)(8 * v.second.size()));
        }
    }
}

void write_outputs(const RunConfig& cfg, RunReport& rep, const Owners& o, const std::vector<txs_ctx*>& band_ctx,
                   const std::vector<std::pair<int64_t, int64_t>>& bands) {
    if (cfg.out_dir.empty()) return;
    std::ofstream csv(cfg.out_dir + "/result.csv");
    if (!csv) throw Error(TXS_ERR_INVALID_ARGUMENT, "[render] unwritable out-dir: " + cfg.out_dir);
    csv << "rank,row,col,marginal_gain,cumulative_coverage\n";
    for (size_t k = 0; k < rep.result.selected.size(); ++k) {
        const Selected& s = rep.result.selected[k];
        char line[160];
        std::snprintf(line, sizeof line, "%zu,%lld,%lld,%lld,%.17g\n", k + 1, (long long)s.candidate.base.row,
                      (long long)s.candidate.base.col, (long long)s.marginal_gain, s.cumulative_coverage);
        csv << line;
    }
    if (cfg.images) render_cumshed(rep.result.cumulative, cfg.out_dir + "/cumshed.pgm");
    if (!cfg.snapshots.empty()) {
        SitingResult byrank = rep.result;   // snapshot k = union of the first k selected viewsheds
        for (size_t k = 0; k < byrank.selected.size(); ++k) byrank.selected[k].index = (int64_t)k;
        render_snapshots(byrank, selected_viewsheds(rep.result, o, cfg.params.roi), cfg.nrows, cfg.ncols,
                         cfg.snapshots, cfg.out_dir);
    }
    write_dumps(cfg, o, band_ctx, bands);
    std::ofstream(cfg.out_dir + "/report.txt") << rep.to_string();
}

RunReport run_single(const RunConfig& cfg) {
    RunReport rep;
    Pipeline pl(cfg.device);
    const double t0 = now_s();
    if (cfg.synth || cfg.input.empty()) pl.generate_fractal(cfg.nrows, cfg.ncols, cfg.roughness, cfg.seed, cfg.zmin, cfg.zmax);
    else pl.set_terrain(load_binary(cfg.input, cfg.nrows, cfg.ncols));
    if (cfg.water_rows > 0) pl.fill_rows(0, std::min(cfg.water_rows, cfg.nrows), 0);
    txs_synchronize(pl.handle());
    const double t1 = now_s();
    if (cfg.observers_random == 0) pl.estimate_vix(cfg.params, cfg.vix_seed);
    const double t2 = now_s();
    rep.candidates = cfg.observers_random > 0 ? pl.random_observers(cfg.observers_random, cfg.observer_seed)
                                              : pl.find_candidates(cfg.params);
    const double t3 = now_s();
    pl.compute_all_viewsheds(cfg.params);
    const double t4 = now_s();
    rep.result = pl.site(cfg.params, true);
    const double t5 = now_s();
    rep.read_s = t1 - t0; rep.vix_s = t2 - t1; rep.findmax_s = t3 - t2; rep.viewshed_s = t4 - t3; rep.site_s = t5 - t4;
    rep.total_s = t5 - t0;
    const Owners o = owners_of({pl.handle()});
    txs_stats st{};
    check(pl.handle(), txs_get_stats(pl.handle(), &st));
    rep.gpus = 1;
    rep.device_bytes_peak = st.device_bytes_peak;
    rep.params_echo = params_echo(cfg, 1);
    rep.host_bytes_peak = host_rss_peak();
    write_outputs(cfg, rep, o, {pl.handle()}, {{0, cfg.nrows}});
    return rep;
}

RunReport run_group(const RunConfig& cfg) {
    RunReport rep;
    const int n = (int)cfg.devices.size();
    txs_group* g = nullptr;
    txs_status st0 = txs_group_create(n, cfg.devices.data(), &g);
    if (st0 != TXS_OK) throw Error((int)st0, "txsite: txs_group_create failed (no usable sm_100 devices?)");
    struct Guard { txs_group* g; ~Guard() { txs_group_destroy(g); } } guard{g};
    auto gchk = [&](txs_status st) { if (st != TXS_OK) throw Error((int)st, txs_group_last_error(g)); };
    gchk(txs_group_set_exchange(g, cfg.exchange));
    const txs_params q = to_params(cfg.params, cfg.vix_seed);
    const double t0 = now_s();
    gchk(txs_group_set_grid(g, cfg.nrows, cfg.ncols, &q));
    if (cfg.synth || cfg.input.empty()) gchk(txs_group_generate_fractal(g, cfg.roughness, cfg.seed, cfg.zmin, cfg.zmax));
    else gchk(txs_group_set_terrain(g, load_binary(cfg.input, cfg.nrows, cfg.ncols).elevations.data()));
    if (cfg.water_rows > 0) gchk(txs_group_fill_rows(g, 0, std::min(cfg.water_rows, cfg.nrows), 0));
    if (cfg.observers_random > 0) gchk(txs_group_random_observers(g, cfg.observers_random, cfg.observer_seed));
    const double t1 = now_s();
    std::vector<txs_step> steps;
    int64_t ns = 0;
    int32_t stop = 0;
    double ms[4] = {0, 0, 0, 0};
    int64_t cap = cfg.params.max_selected > 0 ? cfg.params.max_selected + 1 : 1 << 20;
    steps.resize((size_t)cap);
    gchk(txs_group_run_pipeline(g, &q, steps.data(), cap, &ns, &stop, ms));
    const double t2 = now_s();
    steps.resize((size_t)std::min(ns, cap));
    std::vector<txs_ctx*> ctxs;
    std::vector<std::pair<int64_t, int64_t>> bands;
    for (int k = 0; k < n; ++k) {
        ctxs.push_back(txs_group_context(g, k));
        int64_t a = 0, b = 0;
        gchk(txs_group_band(g, k, &a, &b));
        bands.push_back({a, b});
    }
    // replicated SITE: rank 0 holds every candidate (at its global id); else the bands do
    const Owners o = cfg.exchange == TXS_XCHG_REPLICATE ? owners_of({ctxs[0]}) : owners_of(ctxs);
    rep.result = to_result(steps, stop, o);
    rep.result.cumulative.nrows = cfg.nrows;
    rep.result.cumulative.ncols = cfg.ncols;
    rep.result.cumulative.words.resize((size_t)((cfg.nrows * cfg.ncols + 63) / 64));
    gchk(txs_group_get_cumulative(g, rep.result.cumulative.words.data()));
    for (const auto& ids : o.ids) rep.candidates += (int64_t)ids.size();
    // stage times: device time of each stage's slowest band; total: wall clock
    rep.read_s = t1 - t0; rep.vix_s = ms[0] / 1e3; rep.findmax_s = ms[1] / 1e3; rep.viewshed_s = ms[2] / 1e3;
    rep.site_s = ms[3] / 1e3;
    rep.total_s = t2 - t0;
    rep.gpus = n;
    for (txs_ctx* c : ctxs) {
        txs_stats st{};
        check(c, txs_get_stats(c, &st));
        rep.device_bytes_peak = std::max(rep.device_bytes_peak, st.device_bytes_peak);
    }
    rep.params_echo = params_echo(cfg, n);
    rep.host_bytes_peak = host_rss_peak();
    write_outputs(cfg, rep, o, ctxs, bands);
    return rep;
}

}  // namespace

RunReport run_pipeline(const RunConfig& cfg) {
    if (cfg.devices.size() > 1) return run_group(cfg);
    RunConfig c = cfg;
    if (c.devices.size() == 1) c.device = c.devices[0];
    return run_single(c);
}

}  // namespace txsite
