// Exercises the reference-shaped C++ value-type API (include/txsite/txsite.hpp,
// namespace txsite -- the calls a user of the reference's txsite_core makes)
// on a small synthetic grid and prints every stage's result as plain text for
// tests/test_gpu_cli.py to compare with the CPU oracle.  Built by the top-level
// Makefile as paper_2006_16783_b200/bin/txsite_api_check.
#include <cstdio>
#include <string>
#include <vector>

#include "txsite/txsite.hpp"

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : ".";
    using namespace txsite;
    try {
        TerrainGrid g = generate_fractal(160, 140, 0.5, 3, 0, 2000);
        write_binary(g, dir + "/terrain.bin");
        const TerrainGrid g2 = load_binary(dir + "/terrain.bin", 160, 140);
        std::printf("roundtrip %d\n", g2.elevations == g.elevations ? 1 : 0);
        try {
            load_binary(dir + "/terrain.bin", 160, 141);
            std::printf("size_mismatch none\n");
        } catch (const Error& e) {
            std::printf("size_mismatch %d %s\n", e.status, e.what());
        }
        std::printf("elev %.17g\n", elevation_between(g, {10, 10}, {10, 11}, 0.25));
        std::printf("visible %d %d\n", is_visible(g, {{20, 30}, 10}, {{60, 90}, 5}) ? 1 : 0,
                    is_visible(g, {{100, 20}, 0}, {{101, 21}, 0}) ? 1 : 0);
        SiteParams p;
        p.roi = 15; p.tx_height = 10; p.rx_height = 5; p.samples_per_point = 7; p.per_block = 3;
        p.block_width = 20; p.target_coverage = 0.9; p.max_selected = 30;
        const VixMap v = estimate_vix(g, p, 11);
        unsigned long long h = 1469598103934665603ull;
        for (uint8_t s : v.scores) h = (h ^ s) * 1099511628211ull;
        std::printf("vix %llu\n", h);
        const BlockPartition part = partition(g.nrows, g.ncols, p.roi, p.block_width);
        std::printf("partition %lld %lld %lld\n", (long long)part.block_width, (long long)part.blocks_x,
                    (long long)part.blocks_y);
        const std::vector<Candidate> c = find_candidates(v, part, p.per_block);
        std::printf("candidates %zu", c.size());
        for (const Candidate& x : c) std::printf(" %lld,%lld,%d", (long long)x.base.row, (long long)x.base.col, x.score);
        std::printf("\n");
        const std::vector<Viewshed> vs = compute_all_viewsheds(g, c, p);
        long long pc = 0;
        for (const Viewshed& x : vs) pc += popcount(x);
        std::printf("viewsheds %zu %lld\n", vs.size(), pc);
        const SitingResult r = site(vs, g.nrows, g.ncols, p);
        std::printf("site %s %zu", stop_reason_name(r.stop_reason), r.selected.size());
        for (const Selected& s : r.selected) std::printf(" %lld:%lld", (long long)s.index, (long long)s.marginal_gain);
        std::printf("\n");
        std::printf("coverage %.17g %.17g\n", coverage(r.cumulative), r.final_coverage);
        CumulativeShed empty;
        empty.nrows = g.nrows; empty.ncols = g.ncols;
        empty.words.assign((size_t)((g.nrows * g.ncols + 63) / 64), 0);
        std::printf("gain %lld %lld\n", (long long)marginal_gain(vs[0], empty),
                    (long long)marginal_gain(vs[0], r.cumulative));
    } catch (const Error& e) {
        std::fprintf(stderr, "api_check: %s\n", e.what());
        return 1;
    }
    return 0;
}
