// txsite CLI (SPEC.md:468 flags; the reference's tools/txsite_main.cpp,
// proj/CMakeLists.txt:28): runs VIX -> FINDMAX -> VIEWSHED -> SITE on the
// B200 engine and writes the result CSV, report and PGM images.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "txsite/txsite.hpp"

static void usage() {
    std::fprintf(stderr,
                 "usage: txsite (--input FILE --nrows N --ncols M | --synth [--nrows N --ncols M --seed S --roughness R "
                 "--zmin A --zmax B]) [--roi R] [--tx-height H] [--rx-height H] [--coverage F] [--samples K] "
                 "[--per-block K] [--block-width W] [--max-selected N] [--vix-seed S] [--site-mode 0|1] "
                 "[--out-dir DIR] [--snapshots a,b,c|pow2] [--threads T (ignored: GPU engine)] [--device D] "
                 "[--water-rows K] [--observers-random N --observer-seed S] [--los-arith fp64|exact] "
                 "[--gpus N | --devices a,b,...] [--exchange replicate|p2p|nccl|host] [--dump-vix] [--dump-candidates] "
                 "[--dump-viewsheds] [--no-images]\n");
}

int main(int argc, char** argv) {
    txsite::RunConfig cfg;
    bool pow2 = false;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        auto val = [&]() -> const char* {
            if (i + 1 >= argc) { usage(); std::exit(2); }
            return argv[++i];
        };
        if (a == "--input") { cfg.input = val(); cfg.synth = false; }
        else if (a == "--synth") cfg.synth = true;
        else if (a == "--nrows") cfg.nrows = std::atoll(val());
        else if (a == "--ncols") cfg.ncols = std::atoll(val());
        else if (a == "--seed") cfg.seed = std::strtoull(val(), nullptr, 10);
        else if (a == "--roughness") cfg.roughness = std::atof(val());
        else if (a == "--zmin") cfg.zmin = std::atoi(val());
        else if (a == "--zmax") cfg.zmax = std::atoi(val());
        else if (a == "--roi") cfg.params.roi = std::atoi(val());
        else if (a == "--tx-height") cfg.params.tx_height = std::atoi(val());
        else if (a == "--rx-height") cfg.params.rx_height = std::atoi(val());
        else if (a == "--coverage") cfg.params.target_coverage = std::atof(val());
        else if (a == "--samples") cfg.params.samples_per_point = std::atoi(val());
        else if (a == "--per-block") cfg.params.per_block = std::atoi(val());
        else if (a == "--block-width") cfg.params.block_width = std::atoi(val());
        else if (a == "--max-selected") cfg.params.max_selected = std::atoll(val());
        else if (a == "--site-mode") cfg.params.site_mode = std::atoi(val());
        else if (a == "--vix-seed") cfg.vix_seed = std::strtoull(val(), nullptr, 10);
        else if (a == "--out-dir") cfg.out_dir = val();
        else if (a == "--device") cfg.device = std::atoi(val());
        else if (a == "--water-rows") cfg.water_rows = std::atoll(val());
        else if (a == "--observers-random") cfg.observers_random = std::atoll(val());
        else if (a == "--observer-seed") cfg.observer_seed = std::strtoull(val(), nullptr, 10);
        else if (a == "--los-arith") {
            const std::string m = val();
            if (m != "fp64" && m != "exact") { usage(); return 2; }
            cfg.params.los_arith = m == "exact" ? TXS_LOS_EXACT : TXS_LOS_FP64;
        } else if (a == "--gpus") {
            const int n = std::atoi(val());
            cfg.devices.clear();
            for (int k = 0; k < n; ++k) cfg.devices.push_back(k);
        } else if (a == "--devices") {   // e.g. 0,0 : two row bands on device 0 (testing)
            const std::string d = val();
            cfg.devices.clear();
            size_t p = 0;
            while (p < d.size()) {
                size_t q = d.find(',', p);
                if (q == std::string::npos) q = d.size();
                cfg.devices.push_back(std::atoi(d.substr(p, q - p).c_str()));
                p = q + 1;
            }
        } else if (a == "--exchange") {
            const std::string m = val();
            if (m == "p2p") cfg.exchange = TXS_XCHG_P2P;
            else if (m == "nccl") cfg.exchange = TXS_XCHG_NCCL;
            else if (m == "host") cfg.exchange = TXS_XCHG_HOST;
            else if (m == "replicate") cfg.exchange = TXS_XCHG_REPLICATE;
            else { usage(); return 2; }
        }
        else if (a == "--no-images") cfg.images = false;
        else if (a == "--dump-vix") cfg.dump_vix = true;
        else if (a == "--dump-candidates") cfg.dump_candidates = true;
        else if (a == "--dump-viewsheds") cfg.dump_viewsheds = true;
        else if (a == "--threads") (void)val();
        else if (a == "--snapshots") {
            const std::string s = val();
            if (s == "pow2") pow2 = true;
            else {
                size_t p = 0;
                while (p < s.size()) {
                    size_t q = s.find(',', p);
                    if (q == std::string::npos) q = s.size();
                    cfg.snapshots.push_back(std::atoll(s.substr(p, q - p).c_str()));
                    p = q + 1;
                }
            }
        } else if (a == "-h" || a == "--help") { usage(); return 0; }
        else { std::fprintf(stderr, "unknown flag %s\n", a.c_str()); usage(); return 2; }
    }
    try {
        if (pow2) for (int64_t k = 1; k <= (int64_t)1 << 20; k <<= 1) cfg.snapshots.push_back(k);
        const txsite::RunReport rep = txsite::run_pipeline(cfg);
        std::fputs(rep.to_string().c_str(), stdout);
        return 0;
    } catch (const txsite::Error& e) {
        std::fprintf(stderr, "txsite: %s\n", e.what());
        return 1;
    }
}
