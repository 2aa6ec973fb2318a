// test_shim.cpp -- reference-style C++ tests written against the drop-in
// shim (include/ccwsim_gpu.hpp), i.e. exactly as a reference user's code
// reads (proj/tests/test_{wavelet,matcher,simulator}.cpp), checked against
// the oracle restatement (oracle/ccw_oracle.h, plain C -- no name clash).
//
// Build (tests/test_cpp_shim.py does this):
//   g++ -std=c++20 -O2 -Iinclude -Ioracle tests/cpp/test_shim.cpp \
//       -Lpaper_2404_00441_b200 -lccwgpu -Loracle/_build -lccworacle
#include <cstdio>
#include <cstdlib>
#include <random>
#include <set>

#include "ccwsim_gpu.hpp"
extern "C" {
#include "ccw_oracle.h"
}

using namespace ccwsim;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        ++g_checks;                                                              \
        if (!(cond)) {                                                           \
            ++g_fail;                                                            \
            std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                        \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                              \
    do {                                                                         \
        ++g_checks;                                                              \
        bool ok_ = false;                                                        \
        try {                                                                    \
            (void)(expr);                                                        \
        } catch (const type&) {                                                  \
            ok_ = true;                                                          \
        } catch (...) {                                                          \
        }                                                                        \
        if (!ok_) {                                                              \
            ++g_fail;                                                            \
            std::fprintf(stderr, "%s:%d: expected %s from %s\n", __FILE__, __LINE__, #type, #expr); \
        }                                                                        \
    } while (0)

static RealPlane random_plane(int h, int w, std::mt19937_64& rng) {
    std::vector<double> v(static_cast<std::size_t>(h) * w);
    for (double& x : v) x = static_cast<double>(bounded(rng, 2000)) / 1000.0 - 1.0;
    return RealPlane(h, w, std::move(v));
}

static CategoricalGrid random_grid(int h, int w, int nf, std::mt19937_64& rng) {
    std::vector<int> c(static_cast<std::size_t>(h) * w);
    for (int& x : c) x = static_cast<int>(bounded(rng, nf));
    return CategoricalGrid(h, w, nf, std::move(c));
}

// blocky TI: many exactly tied windows (the fp64 tie-breaking stress case)
static CategoricalGrid blocky_grid(int h, int w, int nf, int b, std::mt19937_64& rng) {
    std::vector<int> c(static_cast<std::size_t>(h) * w);
    std::vector<int> blk(static_cast<std::size_t>(h / b + 1) * (w / b + 1));
    for (int& x : blk) x = static_cast<int>(bounded(rng, nf));
    for (int r = 0; r < h; ++r)
        for (int q = 0; q < w; ++q) c[static_cast<std::size_t>(r) * w + q] = blk[(r / b) * (w / b + 1) + q / b];
    return CategoricalGrid(h, w, nf, std::move(c));
}

static void test_wavelet() {
    // test_wavelet.cpp:81-88, :90-103, :116-119, :152-157
    const SingleLevelDwt d = dwt2_single(RealPlane(2, 2, {1.0, 1.0, 0.0, 0.0}));
    CHECK(std::abs(d.approx.at(0, 0) - 1.0) < 1e-12 && std::abs(d.detail_h.at(0, 0) - 1.0) < 1e-12);
    CHECK(std::abs(d.detail_v.at(0, 0)) < 1e-12 && std::abs(d.detail_d.at(0, 0)) < 1e-12);
    const SingleLevelDwt c = dwt2_single(RealPlane(6, 4, 3.25));
    CHECK(c.approx.height() == 3 && c.approx.width() == 2);
    for (double v : c.approx.values()) CHECK(std::abs(v - 6.5) < 1e-12);
    CHECK_THROWS_AS(dwt2_single(RealPlane(3, 4)), DimensionError);
    CHECK_THROWS_AS(dwt2(RealPlane(12, 16), 3), DimensionError);
    const WaveletPyramid cp = dwt2(RealPlane(8, 8, 1.5), 3);
    for (double v : cp.apex.values()) CHECK(std::abs(v - 12.0) < 1e-12);
    // bit-exact vs the oracle + perfect reconstruction (test_wavelet.cpp:191-204)
    std::mt19937_64 rng(25);
    for (int trial = 0; trial < 30; ++trial) {
        const int lv = 1 + static_cast<int>(bounded(rng, 3)), b = 1 << lv;
        const int h = b * (1 + static_cast<int>(bounded(rng, 64 / b)));
        const int w = b * (1 + static_cast<int>(bounded(rng, 64 / b)));
        const RealPlane p = random_plane(h, w, rng);
        const WaveletPyramid pyr = dwt2(p, lv);
        std::vector<double> apex(static_cast<std::size_t>(h >> lv) * (w >> lv));
        ccwo_dwt2(p.values().data(), h, w, lv, apex.data(), nullptr);
        CHECK(apex == pyr.apex.values());
        const RealPlane back = idwt2(pyr);
        double m = 0;
        for (std::size_t i = 0; i < back.values().size(); ++i)
            m = std::max(m, std::abs(back.values()[i] - p.values()[i]));
        CHECK(m < 1e-9);
    }
}

static void test_matcher() {
    // test_matcher.cpp:164-183, :209-214
    const CandidateSet s = top_k(ScoreMap{RealPlane(2, 2, {3.0, 1.0, 2.0, 5.0})}, 2);
    CHECK(s.size() == 2 && s.entries[0].row == 1 && s.entries[0].col == 1 && s.entries[0].score == 5.0);
    CHECK(s.entries[1].row == 0 && s.entries[1].col == 0 && s.entries[1].score == 3.0);
    const CandidateSet t = top_k(ScoreMap{RealPlane(2, 3, 4.0)}, 3);
    CHECK(t.entries[0].col == 0 && t.entries[1].col == 1 && t.entries[2].col == 2);
    CHECK(top_k(ScoreMap{RealPlane(2, 2, 1.0)}, 10).size() == 4);
    CHECK_THROWS_AS(top_k(ScoreMap{RealPlane(2, 2, 1.0)}, 0), ConfigError);
    CHECK_THROWS_AS(top_k(ScoreMap{}, 3), EmptyInputError);
    // CCF bit-exact vs the oracle on random planes and masks (test_matcher.cpp:81-101)
    std::mt19937_64 rng(33);
    for (int trial = 0; trial < 25; ++trial) {
        const int th = 2 + static_cast<int>(bounded(rng, 4)), tw = 2 + static_cast<int>(bounded(rng, 4));
        const RealPlane ti = random_plane(th + 4 + static_cast<int>(bounded(rng, 9)),
                                          tw + 4 + static_cast<int>(bounded(rng, 9)), rng);
        RealPlane mask(th, tw, 0.0);
        for (int r = 0; r < th; ++r)
            for (int c = 0; c < tw; ++c)
                if (bounded(rng, 2)) mask.set(r, c, 1.0);
        mask.set(0, 0, 1.0);
        RealPlane tm = random_plane(th, tw, rng);
        for (int r = 0; r < th; ++r)
            for (int c = 0; c < tw; ++c)
                if (mask.at(r, c) == 0.0) tm.set(r, c, 0.0);
        const ScoreMap m = ccw_score_map(ti, tm, mask);
        std::vector<double> o(m.scores.values().size());
        ccwo_score_map_channels(ti.values().data(), tm.values().data(), 1, ti.height(), ti.width(),
                                th, tw, mask.values().data(), 0, o.data());
        CHECK(o == m.scores.values());
    }
    CHECK_THROWS_AS(ccw_score_map(RealPlane(8, 8, 1.0), RealPlane(3, 3, 0.0), RealPlane(3, 4, 1.0)),
                    StructureError);
    CHECK_THROWS_AS(ccw_score_map(RealPlane(8, 8, 1.0), RealPlane(9, 3, 0.0), RealPlane(9, 3, 1.0)),
                    DimensionError);
}

static SimConfig base_config() {  // test_simulator.cpp:15-25
    SimConfig cfg;
    cfg.sg_height = cfg.sg_width = 64;
    cfg.template_size = 16;
    cfg.overlap = 4;
    cfg.dwt_level = 2;
    cfg.candidates = 4;
    cfg.n_realizations = 1;
    cfg.master_seed = 1234;
    return cfg;
}

static bool same_as_oracle(const CategoricalGrid& ti, const SimConfig& cfg, std::uint64_t seed) {
    const SimResult r = simulate_one(ti, cfg, seed);
    const std::vector<std::uint8_t> cells = ti.bytes();
    ccwo_sim_config oc{};
    const ccw_sim_config c = cfg.to_c();
    oc.sg_height = c.sg_height;
    oc.sg_width = c.sg_width;
    oc.template_size = c.template_size;
    oc.overlap = c.overlap;
    oc.dwt_level = c.dwt_level;
    oc.candidates = c.candidates;
    oc.n_realizations = c.n_realizations;
    oc.scoring = c.scoring;
    oc.facies_mode = c.facies_mode;
    oc.min_cut = c.min_cut;
    oc.master_seed = c.master_seed;
    std::vector<std::int32_t> hd;
    if (cfg.hard_data)
        for (const HardDatum& d : cfg.hard_data->points) hd.insert(hd.end(), {d.row, d.col, d.facies});
    std::vector<std::uint8_t> out(static_cast<std::size_t>(cfg.sg_height) * cfg.sg_width);
    ccwo_diag od{};
    if (ccwo_simulate_one(cells.data(), ti.height(), ti.width(), ti.num_facies(), &oc,
                          cfg.hard_data ? hd.data() : nullptr,
                          cfg.hard_data ? static_cast<int>(cfg.hard_data->size()) : 0, seed,
                          out.data(), &od, nullptr))
        return false;
    return std::vector<int>(out.begin(), out.end()) == r.realization.cells() &&
           od.pre_overwrite_mismatches == r.diagnostics.pre_overwrite_mismatches;
}

static void test_simulator() {
    // config validation names the key (test_simulator.cpp:29-71)
    SimConfig cfg = base_config();
    cfg.overlap = 6;
    cfg.template_size = 32;
    try {
        cfg.validate();
        CHECK(false);
    } catch (const ConfigError& e) {
        CHECK(std::string(e.what()).find("overlap") != std::string::npos);
    }
    cfg = base_config();
    CHECK_THROWS_AS(cfg.validate_against(CategoricalGrid(8, 8, 2, 0)), ConfigError);
    // plan geometry (test_simulator.cpp:74-106)
    cfg = base_config();
    cfg.sg_height = cfg.sg_width = 512;
    cfg.template_size = 32;
    cfg.overlap = 8;
    std::mt19937_64 r1(1);
    const PlacementPlan plan = plan_raster_path(cfg, r1);
    CHECK(plan.work_height == 512 && plan.placements.size() == 441);
    std::set<std::pair<int, bool>> seen;
    for (std::uint64_t s = 0; s < 64; ++s) {
        std::mt19937_64 r(s);
        const PlacementPlan p = plan_raster_path(base_config(), r);
        seen.emplace(static_cast<int>(p.origin), p.column_major);
    }
    CHECK(seen.size() == 8);
    // constant TI -> constant realization; same seed identical (test_simulator.cpp:401-421)
    cfg = base_config();
    cfg.sg_height = cfg.sg_width = 48;
    const SimResult cres = simulate_one(CategoricalGrid(32, 32, 2, 1), cfg, 999);
    for (int v : cres.realization.cells()) CHECK(v == 1);
    std::mt19937_64 rng(3);
    const CategoricalGrid ti = random_grid(64, 64, 3, rng);
    CHECK(simulate_one(ti, base_config(), 31337).realization == simulate_one(ti, base_config(), 31337).realization);
    // provenance: every pasted block is a block-aligned TI crop (test_simulator.cpp:449-460)
    SimTrace trace;
    simulate_one(ti, base_config(), 77, &trace);
    CHECK(!trace.events.empty());
    for (const auto& ev : trace.events)
        CHECK(ev.ti_row % 4 == 0 && ev.ti_col % 4 == 0 && ev.pasted == crop(ti, ev.ti_row, ev.ti_col, 16, 16));
    // ensemble == simulate_one with mix64 seeds, any `workers` (test_simulator.cpp:529-551)
    SimConfig ec = base_config();
    ec.n_realizations = 4;
    const auto ens = simulate_ensemble(ti, ec, 4);
    for (int r = 0; r < 4; ++r)
        CHECK(ens[r].realization == simulate_one(ti, ec, mix64(ec.master_seed, r + 1)).realization);
    // bit-exact vs the oracle across modes, K, J, min-cut, hard data, blocky ties
    std::mt19937_64 g(2026);
    for (int trial = 0; trial < 24; ++trial) {
        const int J = 1 + static_cast<int>(bounded(g, 3)), b = 1 << J;
        SimConfig c = base_config();
        c.dwt_level = J;
        c.template_size = b * (2 + static_cast<int>(bounded(g, 4)));
        c.overlap = b * (1 + static_cast<int>(bounded(g, static_cast<std::uint64_t>(c.template_size / b - 1))));
        c.candidates = 1 + static_cast<int>(bounded(g, 10));
        c.sg_height = c.template_size + static_cast<int>(bounded(g, 60));
        c.sg_width = c.template_size + static_cast<int>(bounded(g, 60));
        c.min_cut = bounded(g, 2) == 1;
        c.facies_mode = bounded(g, 3) == 0 ? FaciesMode::raw_codes : FaciesMode::indicator;
        c.scoring = bounded(g, 5) == 0 ? ScoringMode::normalized : ScoringMode::raw;
        const int nf = 1 + static_cast<int>(bounded(g, 4));
        const int H = b * (c.template_size / b + 1 + static_cast<int>(bounded(g, 96 / b)));
        const CategoricalGrid t = trial % 2 ? random_grid(H, H, nf, g) : blocky_grid(H, H, nf, b, g);
        if (trial % 3 == 0) {
            HardDataSet hd;
            std::set<std::pair<int, int>> used;
            while (hd.points.size() < 12) {
                const int rr = static_cast<int>(bounded(g, c.sg_height)), cc = static_cast<int>(bounded(g, c.sg_width));
                if (used.emplace(rr, cc).second) hd.points.push_back({rr, cc, static_cast<int>(bounded(g, nf))});
            }
            c.hard_data = hd;
        }
        CHECK(same_as_oracle(t, c, g()));
    }
}

int main() {
    test_wavelet();
    test_matcher();
    test_simulator();
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
