// txsite/txsite.hpp — the reference's C++ stage API (namespace txsite,
// /root/reference/SPEC.md modules terrain/los/vix/candidates/viewshed/siting/
// cli), re-exposed over the B200 engine's C-ABI (include/txsite_b200.h).
//
// A caller of the reference's txsite_core (proj/CMakeLists.txt:13-26) links
// libtxsite_host.a + libtxsite_b200.so instead and keeps its call sites:
// same type names, same operation names, same argument meaning, errors as
// exceptions carrying SPEC's stage-tagged message.  Value-type
// calls (estimate_vix(grid,...) etc.) run on a shared device context and copy
// results back; Pipeline keeps every stage's output resident in HBM.
#pragma once
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../txsite_b200.h"

namespace txsite {

struct Error : std::runtime_error {
    int status;
    Error(int st, const std::string& m) : std::runtime_error(m), status(st) {}
};

// ---- terrain ---------------------------------------------------
struct GridPoint { int64_t row = 0, col = 0; };
struct TerrainGrid {
    int64_t nrows = 0, ncols = 0;
    std::vector<int16_t> elevations;   // row-major, int16 as in the files
    int32_t at(int64_t r, int64_t c) const { return elevations[(size_t)(r * ncols + c)]; }
};
TerrainGrid load_binary(const std::string& path, int64_t nrows, int64_t ncols);
void write_binary(const TerrainGrid& g, const std::string& path);
TerrainGrid load_ascii_grid(const std::string& path);
void write_ascii_grid(const TerrainGrid& g, const std::string& path);
TerrainGrid generate_fractal(int64_t nrows, int64_t ncols, double roughness, uint64_t seed,
                             int32_t zmin, int32_t zmax);
double elevation_between(const TerrainGrid& g, GridPoint p, GridPoint q, double frac);

// ---- los -------------------------------------------------------
struct ObserverSpec { GridPoint base; int32_t height = 0; };
bool is_visible(const TerrainGrid& g, const ObserverSpec& tx, const ObserverSpec& rx);
std::vector<uint8_t> is_visible_batch(const TerrainGrid& g, const std::vector<GridPoint>& tx,
                                      const std::vector<GridPoint>& rx, int32_t ht, int32_t hr,
                                      int32_t los_arith = TXS_LOS_FP64);

// ---- params ----------------------------------------------------------
struct SiteParams {
    int32_t roi = 30;
    int32_t tx_height = 10, rx_height = 10;
    double target_coverage = 0.95;
    int32_t samples_per_point = 10;
    int32_t per_block = 20;
    int32_t block_width = 0;     // 0 => ceil(roi/3)
    int64_t max_selected = 0;    // 0 => unlimited
    int32_t site_mode = 0;       // 0 incremental exact gains, 1 full rescan
    int32_t los_arith = TXS_LOS_FP64;   // SPEC.md:147 fp64 (default) or TXS_LOS_EXACT
};

// ---- vix ---------------------------------------------------------
struct VixMap {
    int64_t nrows = 0, ncols = 0;
    std::vector<uint8_t> scores;
    int32_t samples_per_point = 0;
};
VixMap estimate_vix(const TerrainGrid& g, const SiteParams& p, uint64_t seed);

// ---- candidates ----------------------------------------------
struct Candidate { GridPoint base; int32_t score = 0; };
struct BlockPartition { int64_t block_width = 0, blocks_x = 0, blocks_y = 0; };
BlockPartition partition(int64_t nrows, int64_t ncols, int32_t roi, int32_t block_width = 0);
std::vector<Candidate> find_candidates(const VixMap& vix, const BlockPartition& part, int32_t per_block);

// ---- viewshed --------------------------------------------------
struct Viewshed {
    GridPoint origin;
    int32_t roi = 0;
    int32_t row0 = 0, col0 = 0, h = 0, w = 0;   // clipped window
    std::vector<uint64_t> words;                // row-major, LSB-first (D8)
};
Viewshed compute_viewshed(const TerrainGrid& g, GridPoint tx, const SiteParams& p);
std::vector<Viewshed> compute_all_viewsheds(const TerrainGrid& g, const std::vector<Candidate>& c,
                                            const SiteParams& p);
int64_t popcount(const Viewshed& v);

// ---- siting ------------------------------------------------------
struct CumulativeShed {
    int64_t nrows = 0, ncols = 0;
    std::vector<uint64_t> words;   // dense row-major
};
enum class StopReason { TargetReached = 0, ZeroGain = 1, CandidatesExhausted = 2, MaxSelected = 3 };
const char* stop_reason_name(StopReason s);
struct Selected { int64_t index = 0; Candidate candidate; int64_t marginal_gain = 0; double cumulative_coverage = 0; };
struct SitingResult {
    std::vector<Selected> selected;
    double final_coverage = 0;
    StopReason stop_reason = StopReason::CandidatesExhausted;
    CumulativeShed cumulative;
};
SitingResult site(const std::vector<Viewshed>& v, int64_t nrows, int64_t ncols, const SiteParams& p);
int64_t marginal_gain(const Viewshed& shed, const CumulativeShed& cum);
double coverage(const CumulativeShed& cum);

// ---- cli -----------------------------------------------------------
struct RunConfig {
    std::string input;          // raw int16 file, or empty with synth
    int64_t nrows = 1000, ncols = 1000;
    bool synth = true;
    uint64_t seed = 1;
    double roughness = 0.5;
    int32_t zmin = 0, zmax = 4000;
    int64_t water_rows = 0;     // rows [0, water_rows) clamped to 0 (BASELINE config 3)
    int64_t observers_random = 0;   // > 0: that many random observers (decision D11) replace VIX + FINDMAX (config 5)
    uint64_t observer_seed = 0;
    SiteParams params;
    uint64_t vix_seed = 1;
    std::string out_dir;        // result CSV, report, PGMs when non-empty
    std::vector<int64_t> snapshots;
    bool images = true;             // out_dir/cumshed.pgm; --no-images skips it
    bool dump_vix = false;          // out_dir/vix.u8: row-major score bytes
    bool dump_candidates = false;   // out_dir/candidates.csv: "row,col,score"
    bool dump_viewsheds = false;    // out_dir/viewsheds.bin: per viewshed {row0, col0, w, h} int32 + packed u64 words, LE
    int device = 0;
    std::vector<int> devices;   // > 1 entries: the native multi-GPU group (row bands, txs_group_*)
    int32_t exchange = TXS_XCHG_REPLICATE;   // group SITE: gathered viewsheds (default) or a per-round exchange
};
struct RunReport {
    double read_s = 0, vix_s = 0, findmax_s = 0, viewshed_s = 0, site_s = 0, total_s = 0;
    int64_t candidates = 0;
    int32_t gpus = 1;
    int64_t device_bytes_peak = 0;   // peak memory estimate: max over GPUs of resident HBM buffers
    int64_t host_bytes_peak = 0;     // process max RSS
    std::string params_echo;         // parameter echo
    SitingResult result;
    std::string to_string() const;
};
RunReport run_pipeline(const RunConfig& cfg);
void render_cumshed(const CumulativeShed& cum, const std::string& path);
void render_snapshots(const SitingResult& r, const std::vector<Viewshed>& v, int64_t nrows, int64_t ncols,
                      const std::vector<int64_t>& schedule, const std::string& dir);

// Device-resident pipeline (one txs_ctx): stage outputs stay in HBM between calls.
class Pipeline {
public:
    explicit Pipeline(int device = 0);
    ~Pipeline();
    Pipeline(const Pipeline&) = delete;
    Pipeline& operator=(const Pipeline&) = delete;
    void set_terrain(const TerrainGrid& g);
    void generate_fractal(int64_t nrows, int64_t ncols, double roughness, uint64_t seed, int32_t zmin, int32_t zmax);
    void estimate_vix(const SiteParams& p, uint64_t seed);
    int64_t find_candidates(const SiteParams& p);
    void fill_rows(int64_t row_begin, int64_t row_end, int16_t value);
    int64_t random_observers(int64_t n, uint64_t seed);
    void compute_all_viewsheds(const SiteParams& p);
    SitingResult site(const SiteParams& p, bool with_cumulative = true);
    txs_ctx* handle() const { return ctx_; }
private:
    txs_ctx* ctx_ = nullptr;
};

}  // namespace txsite
