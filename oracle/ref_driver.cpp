// ref_driver.cpp -- C-ABI driver over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file against
// /root/reference/proj/include (the reference sources where they lie, never
// copied) into oracle/_ref/libccwref.so.  It is used (a) to pin the C
// restatement in ccw_oracle.c (tests/golden fixtures, oracle/gen_golden.py)
// and (b) as the "reference" CPU baseline in bench.py (--impl reference).
//
// The signatures mirror ccw_oracle.h with a ccwr_ prefix so the two CPU
// implementations are interchangeable behind oracle/pyoracle.py.  All symbols
// except the extern "C" ones are hidden (-fvisibility=hidden), so the
// reference's inline ccwsim:: definitions never interpose with anything else
// loaded in the same process.

#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <random>
#include <span>
#include <string>
#include <vector>

#include "ccwsim/errors.hpp"
#include "ccwsim/grid.hpp"
#include "ccwsim/matcher.hpp"
#include "ccwsim/rng.hpp"
#include "ccwsim/simulator.hpp"
#include "ccwsim/wavelet.hpp"
#include "support/synthetic.hpp"

extern "C" {
#include "ccw_oracle.h"
}

#define EXPORT extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

int code_of(const std::exception& e) {
    if (dynamic_cast<const ccwsim::BoundsError*>(&e)) return CCWO_BOUNDS;
    if (dynamic_cast<const ccwsim::DimensionError*>(&e)) return CCWO_DIMENSION;
    if (dynamic_cast<const ccwsim::StructureError*>(&e)) return CCWO_STRUCTURE;
    if (dynamic_cast<const ccwsim::ConfigError*>(&e)) return CCWO_CONFIG;
    if (dynamic_cast<const ccwsim::EmptyInputError*>(&e)) return CCWO_EMPTY;
    if (dynamic_cast<const ccwsim::IoError*>(&e)) return CCWO_IO;
    return CCWO_ERROR;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return CCWO_OK;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

ccwsim::RealPlane plane_of(const double* p, int h, int w) {
    return ccwsim::RealPlane(h, w, std::vector<double>(p, p + static_cast<std::size_t>(h) * w));
}

void put(const ccwsim::RealPlane& p, double* out) {
    std::memcpy(out, p.values().data(), p.values().size() * sizeof(double));
}

ccwsim::CategoricalGrid grid_of(const uint8_t* cells, int h, int w, int nf) {
    std::vector<int> v(cells, cells + static_cast<std::size_t>(h) * w);
    return ccwsim::CategoricalGrid(h, w, nf, std::move(v));
}

ccwsim::SimConfig config_of(const ccwo_sim_config* c, const int32_t* hd, int n_hd) {
    if (c->any_support)  // the literal-config extension is not the reference's behaviour
        throw ccwsim::ConfigError("any_support: the reference has no literal-config extension");
    ccwsim::SimConfig cfg;
    cfg.sg_height = c->sg_height;
    cfg.sg_width = c->sg_width;
    cfg.template_size = c->template_size;
    cfg.overlap = c->overlap;
    cfg.dwt_level = c->dwt_level;
    cfg.candidates = c->candidates;
    cfg.n_realizations = c->n_realizations;
    cfg.master_seed = c->master_seed;
    cfg.scoring = c->scoring ? ccwsim::ScoringMode::normalized : ccwsim::ScoringMode::raw;
    cfg.facies_mode =
        c->facies_mode ? ccwsim::FaciesMode::raw_codes : ccwsim::FaciesMode::indicator;
    cfg.min_cut = c->min_cut != 0;
    if (hd) {
        ccwsim::HardDataSet set;
        for (int i = 0; i < n_hd; ++i)
            set.points.push_back({hd[3 * i], hd[3 * i + 1], hd[3 * i + 2]});
        cfg.hard_data = set;
    }
    return cfg;
}

void put_diag(const ccwsim::SimDiagnostics& d, ccwo_diag* o) {
    o->seed = d.seed;
    o->origin = static_cast<int32_t>(d.origin);
    o->column_major = d.column_major;
    o->work_height = d.work_height;
    o->work_width = d.work_width;
    o->placement_count = d.placement_count;
    o->hard_data_count = d.hard_data_count;
    o->pre_overwrite_mismatches = d.pre_overwrite_mismatches;
    o->_pad = 0;
    o->wall_seconds = d.wall_seconds;
}

void put_grid(const ccwsim::CategoricalGrid& g, uint8_t* out) {
    const auto& c = g.cells();
    for (std::size_t i = 0; i < c.size(); ++i) out[i] = static_cast<uint8_t>(c[i]);
}

}  // namespace

EXPORT const char* ccwr_last_error(void) { return g_err.c_str(); }

EXPORT uint64_t ccwr_mix64(uint64_t seed, uint64_t index) { return ccwsim::mix64(seed, index); }

EXPORT void ccwr_mt64_draws(uint64_t seed, uint64_t* out, int n) {
    std::mt19937_64 g(seed);
    for (int i = 0; i < n; ++i) out[i] = g();
}

EXPORT void ccwr_bounded_draws(uint64_t seed, const uint64_t* ns, uint64_t* out, int n) {
    std::mt19937_64 g(seed);
    for (int i = 0; i < n; ++i) out[i] = ccwsim::bounded(g, ns[i]);
}

EXPORT int ccwr_dwt2_single(const double* in, int h, int w, double* a, double* dh, double* dv,
                            double* dd) {
    return guarded([&] {
        const auto r = ccwsim::dwt2_single(plane_of(in, h, w));
        put(r.approx, a);
        put(r.detail_h, dh);
        put(r.detail_v, dv);
        put(r.detail_d, dd);
    });
}

EXPORT int ccwr_idwt2_single(const double* a, const double* dh, const double* dv,
                             const double* dd, int hh, int hw, double* out) {
    return guarded([&] {
        put(ccwsim::idwt2_single(plane_of(a, hh, hw), plane_of(dh, hh, hw), plane_of(dv, hh, hw),
                                 plane_of(dd, hh, hw)),
            out);
    });
}

EXPORT int ccwr_dwt2(const double* in, int h, int w, int levels, double* apex, double* details) {
    return guarded([&] {
        const auto pyr = ccwsim::dwt2(plane_of(in, h, w), levels);
        put(pyr.apex, apex);
        if (details) {
            std::size_t off = 0;
            for (const auto& sb : pyr.details) {
                put(sb.detail_h, details + off);
                off += sb.detail_h.values().size();
                put(sb.detail_v, details + off);
                off += sb.detail_v.values().size();
                put(sb.detail_d, details + off);
                off += sb.detail_d.values().size();
            }
        }
    });
}

EXPORT int ccwr_idwt2(const double* apex, const double* details, int h, int w, int levels,
                      double* out) {
    return guarded([&] {
        ccwsim::WaveletPyramid pyr;
        pyr.levels = levels;
        pyr.original_height = h;
        pyr.original_width = w;
        pyr.apex = plane_of(apex, h >> levels, w >> levels);
        std::size_t off = 0;
        for (int j = 1; j <= levels; ++j) {
            const int ph = h >> j, pw = w >> j;
            const std::size_t n = static_cast<std::size_t>(ph) * pw;
            ccwsim::SubbandSet sb{plane_of(details + off, ph, pw),
                                  plane_of(details + off + n, ph, pw),
                                  plane_of(details + off + 2 * n, ph, pw)};
            off += 3 * n;
            pyr.details.push_back(std::move(sb));
        }
        put(ccwsim::idwt2(pyr), out);
    });
}

EXPORT int ccwr_score_map_channels(const double* ti, const double* tmpl, int nch, int ti_h,
                                   int ti_w, int t_h, int t_w, const double* mask, int scoring,
                                   double* out) {
    return guarded([&] {
        std::vector<ccwsim::RealPlane> a, b;
        for (int f = 0; f < nch; ++f) {
            a.push_back(plane_of(ti + static_cast<std::size_t>(f) * ti_h * ti_w, ti_h, ti_w));
            b.push_back(plane_of(tmpl + static_cast<std::size_t>(f) * t_h * t_w, t_h, t_w));
        }
        const auto map = ccwsim::ccw_score_map_channels(
            a, b, plane_of(mask, t_h, t_w),
            scoring ? ccwsim::ScoringMode::normalized : ccwsim::ScoringMode::raw);
        put(map.scores, out);
    });
}

EXPORT int ccwr_top_k(const double* scores, int h, int w, int k, int32_t* rows, int32_t* cols,
                      double* vals, int* n_out) {
    return guarded([&] {
        ccwsim::ScoreMap map;
        if (h > 0 && w > 0) map.scores = plane_of(scores, h, w);
        const auto set = ccwsim::top_k(map, k);
        for (std::size_t i = 0; i < set.entries.size(); ++i) {
            rows[i] = set.entries[i].row;
            cols[i] = set.entries[i].col;
            vals[i] = set.entries[i].score;
        }
        *n_out = static_cast<int>(set.entries.size());
    });
}

EXPORT int ccwr_select_conditional(const int32_t* rows, const int32_t* cols, const double* vals,
                                   int n_cands, const int32_t* hd, int n_hd, const uint8_t* ti,
                                   int ti_h, int ti_w, int levels, int* pick, int* mismatches) {
    return guarded([&] {
        ccwsim::CandidateSet set;
        for (int i = 0; i < n_cands; ++i) set.entries.push_back({rows[i], cols[i], vals[i]});
        std::vector<ccwsim::HardDatum> loc;
        for (int i = 0; i < n_hd; ++i) loc.push_back({hd[3 * i], hd[3 * i + 1], hd[3 * i + 2]});
        int nf = 1;
        for (std::size_t i = 0; i < static_cast<std::size_t>(ti_h) * ti_w; ++i)
            nf = std::max(nf, static_cast<int>(ti[i]) + 1);
        const auto p =
            ccwsim::select_conditional(set, loc, grid_of(ti, ti_h, ti_w, nf), levels);
        *pick = 0;
        for (int i = 0; i < n_cands; ++i)
            if (set.entries[i].row == p.candidate.row && set.entries[i].col == p.candidate.col) {
                *pick = i;
                break;
            }
        *mismatches = p.mismatches;
    });
}

EXPORT int ccwr_plan_raster_path(const ccwo_sim_config* c, uint64_t seed, int* origin,
                                 int* column_major, int* work_h, int* work_w, int32_t* tops,
                                 int32_t* lefts, int32_t* shapes, int capacity, int* count) {
    return guarded([&] {
        std::mt19937_64 rng(seed);
        const auto plan = ccwsim::plan_raster_path(config_of(c, nullptr, 0), rng);
        *origin = static_cast<int>(plan.origin);
        *column_major = plan.column_major;
        *work_h = plan.work_height;
        *work_w = plan.work_width;
        *count = static_cast<int>(plan.placements.size());
        for (int i = 0; i < *count && i < capacity; ++i) {
            tops[i] = plan.placements[i].top;
            lefts[i] = plan.placements[i].left;
            shapes[i] = static_cast<int32_t>(plan.placements[i].or_shape);
        }
    });
}

EXPORT int ccwr_min_cost_seam(const int32_t* cost, int layers, int width, int32_t* seam) {
    return guarded([&] {
        std::vector<std::vector<int>> c(layers, std::vector<int>(width));
        for (int l = 0; l < layers; ++l)
            for (int j = 0; j < width; ++j) c[l][j] = cost[l * width + j];
        const auto s = ccwsim::detail::min_cost_seam(c);
        for (int l = 0; l < layers; ++l) seam[l] = s[l];
    });
}

EXPORT int ccwr_min_cut_stitch(const uint8_t* existing, const uint8_t* incoming, int t,
                               int shape, int vertical_on_left, int horizontal_on_top,
                               int overlap, uint8_t* out) {
    return guarded([&] {
        int nf = 1;
        for (int i = 0; i < t * t; ++i)
            nf = std::max({nf, static_cast<int>(existing[i]) + 1, static_cast<int>(incoming[i]) + 1});
        ccwsim::OrGeometry g;
        g.shape = static_cast<ccwsim::OrShape>(shape);
        g.vertical_on_left = vertical_on_left != 0;
        g.horizontal_on_top = horizontal_on_top != 0;
        g.overlap = overlap;
        put_grid(ccwsim::min_cut_stitch(grid_of(existing, t, t, nf), grid_of(incoming, t, t, nf), g),
                 out);
    });
}

EXPORT int ccwr_simulate_one(const uint8_t* ti, int ti_h, int ti_w, int nf,
                             const ccwo_sim_config* c, const int32_t* hd, int n_hd, uint64_t seed,
                             uint8_t* out, ccwo_diag* diag, ccwo_trace* trace) {
    return guarded([&] {
        ccwsim::SimTrace tr;
        const auto res = ccwsim::simulate_one(grid_of(ti, ti_h, ti_w, nf), config_of(c, hd, n_hd),
                                              seed, trace ? &tr : nullptr);
        put_grid(res.realization, out);
        if (diag) put_diag(res.diagnostics, diag);
        if (trace) {
            trace->count = 0;
            for (const auto& ev : tr.events) {
                if (trace->count >= trace->capacity) break;
                const int e = trace->count++;
                trace->top[e] = ev.placement.top;
                trace->left[e] = ev.placement.left;
                trace->shape[e] = static_cast<int32_t>(ev.placement.or_shape);
                trace->ti_row[e] = ev.ti_row;
                trace->ti_col[e] = ev.ti_col;
                if (trace->pasted)
                    put_grid(ev.pasted, trace->pasted + static_cast<std::size_t>(e) *
                                                          ev.pasted.height() * ev.pasted.width());
            }
        }
    });
}

EXPORT int ccwr_simulate_ensemble(const uint8_t* ti, int ti_h, int ti_w, int nf,
                                  const ccwo_sim_config* c, const int32_t* hd, int n_hd,
                                  int workers, uint8_t* out, ccwo_diag* diags) {
    return guarded([&] {
        const auto res = ccwsim::simulate_ensemble(grid_of(ti, ti_h, ti_w, nf),
                                                   config_of(c, hd, n_hd), workers);
        const std::size_t sg = static_cast<std::size_t>(c->sg_height) * c->sg_width;
        for (std::size_t r = 0; r < res.size(); ++r) {
            put_grid(res[r].realization, out + r * sg);
            if (diags) put_diag(res[r].diagnostics, &diags[r]);
        }
    });
}

// tests/support/synthetic.hpp:19-44 -- the reference tests' channel TI.
EXPORT void ccwr_make_channel_ti(int h, int w, uint64_t seed, uint8_t* out) {
    put_grid(testsupport::make_channel_ti(h, w, seed), out);
}

// tests/support/synthetic.hpp:46-59
EXPORT void ccwr_random_grid(int h, int w, int nf, uint64_t seed, uint8_t* out) {
    std::mt19937_64 rng(seed);
    put_grid(testsupport::random_grid(h, w, nf, rng), out);
}

EXPORT void ccwr_random_plane(int h, int w, uint64_t seed, double* out) {
    std::mt19937_64 rng(seed);
    put(testsupport::random_plane(h, w, rng), out);
}
