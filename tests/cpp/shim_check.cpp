// Exercises the drop-in C++ interface (include/mrf_b200/mrf.hpp) the way a
// reference user would: same types, same calls, same exceptions.
// Exit 0 = all checks passed.  Run on a B200 (the compute goes to the GPU).
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "mrf_b200/mrf.hpp"

using namespace mrf;
static int fails = 0;
#define EXPECT(c)                                                    \
    do {                                                             \
        if (!(c)) {                                                  \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #c); \
            ++fails;                                                 \
        }                                                            \
    } while (0)

int main() {
    // schedule + digest (sequence.hpp, dictionary.hpp:67)
    Schedule s500 = build_schedule(500, 1);
    EXPECT(digest_hex(schedule_digest(s500)) ==
           "99b129a4b97065d83595554534b6434b0c5cbe05b7223af5981b79ec6965bc8e");
    // generic 1-D zoom over a caller objective (host path)
    std::vector<long> seen;
    std::vector<long> steps{4, 1};
    long r = zoom_1d([&](long x) { seen.push_back(x); return -std::abs(double(x - 7)); }, 0, 20, 10, steps);
    EXPECT(r == 7 && (seen == std::vector<long>{10, 6, 2, 10, 5, 7, 6, 8}));

    // GPU: lattice targets, quantify vs brute force over a generated dictionary
    Schedule s = build_schedule(60, 15);
    SearchRanges ranges{{600, 1000, 10}, {80, 160, 5}, {-20, 30, 2}};
    ParameterGrid grid = grid_from_ranges(ranges.t1_ms, ranges.t2_ms, ranges.df_hz);
    EXPECT(grid.total() == 40u * 16u * 25u);
    ZoomConfig cfg;
    cfg.df_coarse_hz = 2;
    Dictionary dict = generate(grid, s);
    BlochSimulator sim(s);
    std::vector<Fingerprint> q;
    for (int k = 0; k < 4; ++k) {
        TissueParams t = grid.params_at(7 + 9 * k, 3 + 3 * k, 2 + 6 * k);
        Fingerprint fp = sim.simulate(t);
        for (auto& v : fp.s) v *= 1.7;
        q.push_back(fp);
        QuantResult z = quantify(fp, ranges, cfg, s);
        Match b = brute_force_search(fp, dict);
        EXPECT(z.params.t1 == b.params.t1 && z.params.t2 == b.params.t2 && z.params.df == b.params.df);
        EXPECT(z.params.t1 == t.t1 && z.params.df == t.df);
        EXPECT(std::abs(z.params.pd - 1.7) < 1e-9);
        EXPECT(z.evaluations > 0 && z.evaluations < grid.total());
        std::size_t traced = 0;  // test_zoom.cpp:334-336
        for (const auto& st : z.trace) traced += st.evaluations;
        EXPECT(traced == z.evaluations);
        EXPECT(!z.trace.empty() && z.trace.front().stage == "df.coarse" && z.trace.back().stage == "t1t2.final");
    }
    ScanOutcome sc = scan_grid(grid, s, q, Metric::cc, 1, 7);
    for (std::size_t k = 0; k < q.size(); ++k) {
        Match b = brute_force_search(q[k], dict);
        EXPECT(sc.matches[k].params.t1 == b.params.t1 && sc.matches[k].score == b.score);
        EXPECT(sc.matches[k].evaluations == grid.total());
    }
    // Objective (zoom.hpp:72-110): the memo the search runs on; its value at
    // quantify's answer is quantify's score, repeats are free, metric
    // switches reuse the entry, range errors are out_of_range
    {
        Fingerprint fp = q[1];
        QuantResult z = quantify(fp, ranges, cfg, s);
        Objective obj(fp, grid, s, Objective::Options{});
        const long i1 = std::lround((z.params.t1 * 1e3 - grid.t1_ms.min) / grid.t1_ms.step);
        const long i2 = std::lround((z.params.t2 * 1e3 - grid.t2_ms.min) / grid.t2_ms.step);
        const long idf = std::lround((z.params.df - grid.df_hz.min) / grid.df_hz.step);
        EXPECT(obj.eval(i1, i2, idf, Metric::cc) == z.score);
        EXPECT(obj.evaluations() == 1);
        obj.eval(i1, i2, idf, Metric::euclidean);
        obj.eval_df_stage(i1, i2, idf, Metric::cc);
        EXPECT(obj.evaluations() == 1);
        Fingerprint ideal = obj.ideal_at(i1, i2, idf);
        EXPECT(std::abs(estimate_pd(fp, ideal) - z.params.pd) < 1e-15);
        bool oor = false;
        try {
            obj.eval(-1, 0, 0, Metric::cc);
        } catch (const std::out_of_range&) {
            oor = true;
        }
        EXPECT(oor);
        // a full dictionary: the objective scores the stored float entries
        Objective::Options o;
        o.full_dict = &dict;
        Objective od(fp, grid, s, o);
        const double vd = od.eval(i1, i2, idf, Metric::cc);
        EXPECT(std::abs(vd - z.score) < 1e-6 && od.evaluations() == 1);
    }
    // cc_map streams every score in order
    std::size_t got = 0;
    cc_map(q[0], grid, s, [&](std::size_t first, std::span<const float> v) {
        EXPECT(first == got);
        got += v.size();
    }, 1, 1000);
    EXPECT(got == grid.total());
    // slice with and without priors (zoom.hpp:174-178)
    int nx = 4, ny = 3;
    std::vector<std::uint8_t> mask(12, 1);
    mask[0] = mask[11] = 0;
    std::vector<Fingerprint> fps(12);
    for (int v = 0; v < 12; ++v)
        if (mask[v]) fps[v] = sim.simulate(grid.params_at(20 + v % 2, 8 + v % 3, 10));
    SliceResult a = quantify_slice(fps, mask, nx, ny, ranges, cfg, s, false);
    SliceResult c = quantify_slice(fps, mask, nx, ny, ranges, cfg, s, true);
    for (int v = 0; v < 12; ++v) EXPECT(a.t1_ms[v] == c.t1_ms[v] && a.df_hz[v] == c.df_hz[v]);
    EXPECT(c.total_evaluations < a.total_evaluations);
    // the reference's exceptions
    bool threw = false;
    try {
        Fingerprint bad;
        bad.s.assign(59, {1, 0});
        brute_force_search(bad, dict);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    EXPECT(threw);
    threw = false;
    try {
        std::vector<Fingerprint> none;
        scan_grid(grid, s, none);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    EXPECT(threw);
    // .mrfd / .mrfc files (dictionary.hpp:87-96, 130-132)
    {
        const std::filesystem::path dir = std::filesystem::temp_directory_path();
        const auto pd = dir / "shim_check.mrfd", pc = dir / "shim_check.mrfc";
        save_generated(grid, s, pd, 1, 777);
        Dictionary back = load(pd);
        EXPECT(back.digest == dict.digest && back.entry_len == dict.entry_len);
        EXPECT(back.grid.total() == grid.total() && back.data == dict.data);
        save(dict, dir / "shim_check2.mrfd");
        EXPECT(load(dir / "shim_check2.mrfd").data == dict.data);
        cc_map_to_file(q[0], grid, s, pc);
        EXPECT(std::filesystem::file_size(pc) == 4 + 4 + 32 + 72 + 8 + 4 * grid.total());
        threw = false;
        try {
            load(pc);  // an .mrfc is not a dictionary
        } catch (const std::runtime_error&) {
            threw = true;
        }
        EXPECT(threw);
        std::filesystem::remove(pd);
        std::filesystem::remove(pc);
        std::filesystem::remove(dir / "shim_check2.mrfd");
    }
    // noise calibration, smoothing, fingerprint CSV (fingerprint.hpp:45-75)
    {
        Fingerprint f0 = sim.simulate(grid.params_at(12, 9, 4));
        const double sg = calibrate_noise(f0, 0.5, 3);
        EXPECT(std::abs(cc(f0, add_noise(f0, sg, 3)) - 0.5) <= 0.02);
        CalibratedNoise cn = make_calibrated_noise(f0, 0.5, 3);
        EXPECT(cn.sigma == sg && cn.seed == 3);
        Fingerprint sm = smooth(f0, 5);
        EXPECT(sm.size() == f0.size());
        const auto pf = std::filesystem::temp_directory_path() / "shim_check_fp.csv";
        save_csv(f0, pf);
        Fingerprint rl = load_fingerprint_csv(pf);
        EXPECT(rl.size() == f0.size() && std::abs(rl.s[7] - f0.s[7]) < 1e-8);
        std::filesystem::remove(pf);
        threw = false;
        try {
            smooth(f0, 4);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        EXPECT(threw);
    }
    std::printf("%s (%d failures)\n", fails ? "FAILED" : "OK", fails);
    return fails ? 1 : 0;
}
