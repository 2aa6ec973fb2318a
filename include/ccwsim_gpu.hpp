// ccwsim_gpu.hpp -- drop-in C++ shim: the reference's `namespace ccwsim`
// hot-path API (proj/include/ccwsim/{errors,rng,grid,wavelet,matcher,
// simulator}.hpp) re-declared over the C-ABI of libccwgpu.so.
//
// A program written against the reference headers compiles against this one
// unchanged for the hot path: same type names, member names, free functions,
// exception classes and messages.  Every numeric operator and the simulation
// run on the GPU (include/ccwgpu.h); what stays on the host is host logic by
// nature: the containers, crop/paste of caller-side grids, the caller's
// std::mt19937_64 draws (bounded, select_unconditional, the two plan draws).
//
// Never include this together with the reference headers in one program
// (same names, different definitions).  Link with -lccwgpu.
//
// Concurrency: each host thread gets its own device context (thread_local),
// on device $CCWSIM_DEVICE (default 0).  simulate_ensemble's `workers`
// argument is accepted and ignored -- all realizations run in one batched
// device call, and the reference guarantees worker-count-invariant output
// (simulator.hpp:521-522), so results are identical.
#pragma once

#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <optional>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>
#include <thread>
#include <mutex>
#include <exception>
#include <algorithm>

#include "ccwgpu.h"

namespace ccwsim {

// ------------------------------------------------------------ errors.hpp --
class Error : public std::runtime_error {
public:
    explicit Error(const std::string& msg) : std::runtime_error(msg) {}
};
class BoundsError : public Error { public: using Error::Error; };
class DimensionError : public Error { public: using Error::Error; };
class StructureError : public Error { public: using Error::Error; };
class ConfigError : public Error { public: using Error::Error; };
class EmptyInputError : public Error { public: using Error::Error; };
class DegeneracyError : public Error { public: using Error::Error; };
class IoError : public Error { public: using Error::Error; };
// CUDA failures inside libccwgpu.so (status >= 100); no reference twin.
class DeviceError : public Error { public: using Error::Error; };

namespace gpu_detail {

[[noreturn]] inline void raise(int code, const std::string& msg) {
    switch (code) {
        case CCW_ERR_BOUNDS: throw BoundsError(msg);
        case CCW_ERR_DIMENSION: throw DimensionError(msg);
        case CCW_ERR_STRUCTURE: throw StructureError(msg);
        case CCW_ERR_CONFIG: throw ConfigError(msg);
        case CCW_ERR_EMPTY: throw EmptyInputError(msg);
        case CCW_ERR_IO: throw IoError(msg);
        case CCW_ERR_GENERIC: throw Error(msg);
        default: throw DeviceError(msg);
    }
}

struct Ctx {
    ccw_ctx* h = nullptr;
    Ctx() {
        const char* e = std::getenv("CCWSIM_DEVICE");
        const int dev = e ? std::atoi(e) : 0;
        const int rc = ccw_ctx_create(dev, &h);
        if (rc) raise(rc, ccw_last_error(nullptr));
    }
    ~Ctx() { ccw_ctx_destroy(h); }
    Ctx(const Ctx&) = delete;
    Ctx& operator=(const Ctx&) = delete;
};

inline ccw_ctx* ctx() {
    thread_local Ctx c;
    return c.h;
}

inline void check(int rc) {
    if (rc) raise(rc, ccw_last_error(ctx()));
}

}  // namespace gpu_detail

// --------------------------------------------------------------- rng.hpp --
inline std::uint64_t mix64(std::uint64_t seed, std::uint64_t index) { return ccw_mix64(seed, index); }

inline std::uint64_t bounded(std::mt19937_64& rng, std::uint64_t n) {
    const std::uint64_t threshold = (0 - n) % n;  // rng.hpp:21-28
    for (;;) {
        const std::uint64_t r = rng();
        if (r >= threshold) return r % n;
    }
}

// -------------------------------------------------------------- grid.hpp --
class CategoricalGrid {
public:
    CategoricalGrid() = default;
    CategoricalGrid(int height, int width, int num_facies, int fill = 0)
        : height_(height), width_(width), num_facies_(num_facies) {
        check_shape();
        if (fill < 0 || fill >= num_facies_)
            throw BoundsError("fill code " + std::to_string(fill) + " outside [0, " +
                              std::to_string(num_facies_) + ")");
        cells_.assign(static_cast<std::size_t>(height_) * width_, fill);
    }
    CategoricalGrid(int height, int width, int num_facies, std::vector<int> cells)
        : height_(height), width_(width), num_facies_(num_facies), cells_(std::move(cells)) {
        check_shape();
        if (cells_.size() != static_cast<std::size_t>(height_) * width_)
            throw StructureError("cell count " + std::to_string(cells_.size()) + " does not match " +
                                 std::to_string(height_) + "x" + std::to_string(width_));
        for (std::size_t i = 0; i < cells_.size(); ++i)
            if (cells_[i] < 0 || cells_[i] >= num_facies_)
                throw BoundsError("cell " + std::to_string(i) + " holds code " +
                                  std::to_string(cells_[i]) + " outside [0, " +
                                  std::to_string(num_facies_) + ")");
    }
    int height() const noexcept { return height_; }
    int width() const noexcept { return width_; }
    int num_facies() const noexcept { return num_facies_; }
    std::int64_t area() const noexcept { return static_cast<std::int64_t>(height_) * width_; }
    int at(int r, int c) const { return cells_[index(r, c)]; }
    void set(int r, int c, int code) {
        if (code < 0 || code >= num_facies_)
            throw BoundsError("code " + std::to_string(code) + " outside [0, " +
                              std::to_string(num_facies_) + ")");
        cells_[index(r, c)] = code;
    }
    const std::vector<int>& cells() const noexcept { return cells_; }
    bool operator==(const CategoricalGrid& o) const = default;

    std::vector<std::uint8_t> bytes() const {
        return std::vector<std::uint8_t>(cells_.begin(), cells_.end());
    }

private:
    void check_shape() const {
        if (height_ <= 0 || width_ <= 0) throw DimensionError("grid dimensions must be positive");
        if (num_facies_ <= 0) throw DimensionError("num_facies must be positive");
    }
    std::size_t index(int r, int c) const {
        if (r < 0 || r >= height_ || c < 0 || c >= width_)
            throw BoundsError("cell (" + std::to_string(r) + ", " + std::to_string(c) + ") outside " +
                              std::to_string(height_) + "x" + std::to_string(width_) + " grid");
        return static_cast<std::size_t>(r) * width_ + c;
    }
    int height_ = 0, width_ = 0, num_facies_ = 1;
    std::vector<int> cells_;
};

class RealPlane {
public:
    RealPlane() = default;
    RealPlane(int height, int width, double fill = 0.0) : height_(height), width_(width) {
        if (height_ <= 0 || width_ <= 0) throw DimensionError("plane dimensions must be positive");
        values_.assign(static_cast<std::size_t>(height_) * width_, fill);
    }
    RealPlane(int height, int width, std::vector<double> values)
        : height_(height), width_(width), values_(std::move(values)) {
        if (height_ <= 0 || width_ <= 0) throw DimensionError("plane dimensions must be positive");
        if (values_.size() != static_cast<std::size_t>(height_) * width_)
            throw StructureError("value count does not match " + std::to_string(height_) + "x" +
                                 std::to_string(width_));
        for (double v : values_)
            if (!std::isfinite(v)) throw StructureError("plane values must be finite");
    }
    int height() const noexcept { return height_; }
    int width() const noexcept { return width_; }
    double at(int r, int c) const { return values_[index(r, c)]; }
    void set(int r, int c, double v) { values_[index(r, c)] = v; }
    const double* row(int r) const { return values_.data() + static_cast<std::size_t>(r) * width_; }
    double* row(int r) { return values_.data() + static_cast<std::size_t>(r) * width_; }
    const std::vector<double>& values() const noexcept { return values_; }
    std::vector<double>& values() noexcept { return values_; }

private:
    std::size_t index(int r, int c) const {
        if (r < 0 || r >= height_ || c < 0 || c >= width_)
            throw BoundsError("plane cell (" + std::to_string(r) + ", " + std::to_string(c) +
                              ") outside " + std::to_string(height_) + "x" + std::to_string(width_));
        return static_cast<std::size_t>(r) * width_ + c;
    }
    int height_ = 0, width_ = 0;
    std::vector<double> values_;
};

struct HardDatum {
    int row = 0, col = 0, facies = 0;
    bool operator==(const HardDatum&) const = default;
};

struct HardDataSet {
    std::vector<HardDatum> points;
    bool empty() const noexcept { return points.empty(); }
    std::size_t size() const noexcept { return points.size(); }
};

namespace gpu_detail {
inline std::vector<std::int32_t> triples(const std::vector<HardDatum>& pts) {
    std::vector<std::int32_t> v;
    v.reserve(pts.size() * 3);
    for (const HardDatum& p : pts) {
        v.push_back(p.row);
        v.push_back(p.col);
        v.push_back(p.facies);
    }
    return v;
}
}  // namespace gpu_detail

inline CategoricalGrid crop(const CategoricalGrid& grid, int top, int left, int h, int w) {
    if (h <= 0 || w <= 0) throw DimensionError("crop size must be positive");
    if (top < 0 || left < 0 || top + h > grid.height() || left + w > grid.width())
        throw BoundsError("crop rectangle (" + std::to_string(top) + ", " + std::to_string(left) +
                          ", " + std::to_string(h) + "x" + std::to_string(w) + ") outside " +
                          std::to_string(grid.height()) + "x" + std::to_string(grid.width()) + " grid");
    std::vector<int> out;
    out.reserve(static_cast<std::size_t>(h) * w);
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c) out.push_back(grid.at(top + r, left + c));
    return CategoricalGrid(h, w, grid.num_facies(), std::move(out));
}

inline RealPlane crop(const RealPlane& plane, int top, int left, int h, int w) {
    if (h <= 0 || w <= 0) throw DimensionError("crop size must be positive");
    if (top < 0 || left < 0 || top + h > plane.height() || left + w > plane.width())
        throw BoundsError("crop rectangle outside " + std::to_string(plane.height()) + "x" +
                          std::to_string(plane.width()) + " plane");
    RealPlane out(h, w);
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c) out.set(r, c, plane.at(top + r, left + c));
    return out;
}

inline void paste_into(CategoricalGrid& grid, const CategoricalGrid& patch, int top, int left) {
    if (top < 0 || left < 0 || top + patch.height() > grid.height() ||
        left + patch.width() > grid.width())
        throw BoundsError("patch footprint overflows grid");
    if (patch.num_facies() > grid.num_facies())
        throw StructureError("patch facies count exceeds target grid's");
    for (int r = 0; r < patch.height(); ++r)
        for (int c = 0; c < patch.width(); ++c) grid.set(top + r, left + c, patch.at(r, c));
}

inline CategoricalGrid paste(const CategoricalGrid& grid, const CategoricalGrid& patch, int top,
                             int left) {
    CategoricalGrid out = grid;
    paste_into(out, patch, top, left);
    return out;
}

inline std::vector<RealPlane> to_indicator_planes(const CategoricalGrid& grid) {
    std::vector<RealPlane> planes;
    for (int f = 0; f < grid.num_facies(); ++f) planes.emplace_back(grid.height(), grid.width(), 0.0);
    for (std::size_t i = 0; i < grid.cells().size(); ++i) planes[grid.cells()[i]].values()[i] = 1.0;
    return planes;
}

inline RealPlane to_real_plane(const CategoricalGrid& grid) {
    RealPlane out(grid.height(), grid.width());
    for (std::size_t i = 0; i < grid.cells().size(); ++i)
        out.values()[i] = static_cast<double>(grid.cells()[i]);
    return out;
}

// ----------------------------------------------------------- wavelet.hpp --
struct HaarFilterBank {
    static constexpr double kInvSqrt2 = 0.70710678118654752440084436210485;
    static constexpr std::array<double, 2> analysis_low{kInvSqrt2, kInvSqrt2};
    static constexpr std::array<double, 2> analysis_high{kInvSqrt2, -kInvSqrt2};
    static constexpr std::array<double, 2> synthesis_low{kInvSqrt2, kInvSqrt2};
    static constexpr std::array<double, 2> synthesis_high{kInvSqrt2, -kInvSqrt2};
};

struct SubbandSet {
    RealPlane detail_h, detail_v, detail_d;
};

struct WaveletPyramid {
    int levels = 0;
    int original_height = 0;
    int original_width = 0;
    RealPlane apex;
    std::vector<SubbandSet> details;
};

struct SingleLevelDwt {
    RealPlane approx, detail_h, detail_v, detail_d;
};

inline SingleLevelDwt dwt2_single(const RealPlane& plane) {
    const int h = plane.height(), w = plane.width();
    if (h % 2 != 0 || w % 2 != 0)
        throw DimensionError("dwt2_single requires even dimensions, got " + std::to_string(h) + "x" +
                             std::to_string(w));
    SingleLevelDwt o{RealPlane(h / 2, w / 2), RealPlane(h / 2, w / 2), RealPlane(h / 2, w / 2),
                     RealPlane(h / 2, w / 2)};
    gpu_detail::check(ccw_dwt2_single_f64(gpu_detail::ctx(), plane.values().data(), h, w,
                                          o.approx.values().data(), o.detail_h.values().data(),
                                          o.detail_v.values().data(), o.detail_d.values().data()));
    return o;
}

inline RealPlane idwt2_single(const RealPlane& approx, const RealPlane& detail_h,
                              const RealPlane& detail_v, const RealPlane& detail_d) {
    const int hh = approx.height(), hw = approx.width();
    auto same = [&](const RealPlane& p) { return p.height() == hh && p.width() == hw; };
    if (!same(detail_h) || !same(detail_v) || !same(detail_d))
        throw StructureError("subband sizes disagree");
    RealPlane out(2 * hh, 2 * hw);
    gpu_detail::check(ccw_idwt2_single_f64(gpu_detail::ctx(), approx.values().data(),
                                           detail_h.values().data(), detail_v.values().data(),
                                           detail_d.values().data(), hh, hw, out.values().data()));
    return out;
}

inline WaveletPyramid dwt2(const RealPlane& plane, int levels) {
    if (levels < 1) throw DimensionError("decomposition level must be >= 1");
    const int div = 1 << std::min(levels, 30);
    if (plane.height() % div != 0 || plane.width() % div != 0)
        throw DimensionError("plane " + std::to_string(plane.height()) + "x" +
                             std::to_string(plane.width()) + " not divisible by 2^" +
                             std::to_string(levels));
    const int h = plane.height(), w = plane.width();
    std::size_t nd = 0;
    for (int j = 1; j <= levels; ++j) nd += 3 * static_cast<std::size_t>(h >> j) * (w >> j);
    std::vector<double> det(nd);
    WaveletPyramid pyr;
    pyr.levels = levels;
    pyr.original_height = h;
    pyr.original_width = w;
    pyr.apex = RealPlane(h >> levels, w >> levels);
    gpu_detail::check(ccw_dwt2_f64(gpu_detail::ctx(), plane.values().data(), h, w, levels,
                                   pyr.apex.values().data(), det.data()));
    std::size_t off = 0;
    for (int j = 1; j <= levels; ++j) {
        const int ph = h >> j, pw = w >> j;
        const std::size_t n = static_cast<std::size_t>(ph) * pw;
        auto slice = [&](std::size_t o) {
            return RealPlane(ph, pw, std::vector<double>(det.begin() + o, det.begin() + o + n));
        };
        pyr.details.push_back(SubbandSet{slice(off), slice(off + n), slice(off + 2 * n)});
        off += 3 * n;
    }
    return pyr;
}

inline RealPlane idwt2(const WaveletPyramid& pyr) {
    if (pyr.levels < 1 || pyr.details.size() != static_cast<std::size_t>(pyr.levels))
        throw StructureError("pyramid level count inconsistent");
    int h = pyr.original_height >> pyr.levels, w = pyr.original_width >> pyr.levels;
    if (pyr.apex.height() != h || pyr.apex.width() != w)
        throw StructureError("apex size does not match original/2^levels");
    std::vector<double> det;
    for (int j = 1; j <= pyr.levels; ++j) {
        const SubbandSet& sb = pyr.details[static_cast<std::size_t>(j) - 1];
        const int ph = pyr.original_height >> j, pw = pyr.original_width >> j;
        for (const RealPlane* p : {&sb.detail_h, &sb.detail_v, &sb.detail_d}) {
            if (p->height() != ph || p->width() != pw)
                throw StructureError("level " + std::to_string(j) + " subband size inconsistent");
            det.insert(det.end(), p->values().begin(), p->values().end());
        }
    }
    RealPlane out(pyr.original_height, pyr.original_width);
    gpu_detail::check(ccw_idwt2_f64(gpu_detail::ctx(), pyr.apex.values().data(), det.data(),
                                    pyr.original_height, pyr.original_width, pyr.levels,
                                    out.values().data()));
    return out;
}

inline std::pair<int, int> coarse_to_fine(std::pair<int, int> coord, int levels) {
    return {coord.first << levels, coord.second << levels};
}

// ----------------------------------------------------------- matcher.hpp --
enum class ScoringMode { raw, normalized };

struct ScoreMap {
    RealPlane scores;
};

struct Candidate {
    int row = 0;
    int col = 0;
    double score = 0.0;
};

struct CandidateSet {
    std::vector<Candidate> entries;
    bool empty() const noexcept { return entries.empty(); }
    std::size_t size() const noexcept { return entries.size(); }
};

inline ScoreMap ccw_score_map_channels(std::span<const RealPlane> ti_channels,
                                       std::span<const RealPlane> or_channels,
                                       const RealPlane& or_mask,
                                       ScoringMode mode = ScoringMode::raw) {
    if (ti_channels.empty() || ti_channels.size() != or_channels.size())
        throw StructureError("channel counts disagree");
    const int th = or_channels[0].height(), tw = or_channels[0].width();
    for (std::size_t f = 0; f < or_channels.size(); ++f)
        if (or_mask.height() != or_channels[f].height() || or_mask.width() != or_channels[f].width())
            throw StructureError("mask size " + std::to_string(or_mask.height()) + "x" +
                                 std::to_string(or_mask.width()) + " does not match template " +
                                 std::to_string(or_channels[f].height()) + "x" +
                                 std::to_string(or_channels[f].width()));
    const int ih = ti_channels[0].height(), iw = ti_channels[0].width();
    std::vector<double> ti, tm;
    for (std::size_t f = 0; f < ti_channels.size(); ++f) {
        ti.insert(ti.end(), ti_channels[f].values().begin(), ti_channels[f].values().end());
        tm.insert(tm.end(), or_channels[f].values().begin(), or_channels[f].values().end());
    }
    if (th > ih || tw > iw)
        throw DimensionError("template " + std::to_string(th) + "x" + std::to_string(tw) +
                             " larger than TI coefficients " + std::to_string(ih) + "x" +
                             std::to_string(iw));
    ScoreMap map{RealPlane(ih - th + 1, iw - tw + 1)};
    gpu_detail::check(ccw_score_map_f64(gpu_detail::ctx(), ti.data(), tm.data(),
                                        static_cast<int>(ti_channels.size()), ih, iw, th, tw,
                                        or_mask.values().data(), mode == ScoringMode::normalized,
                                        map.scores.values().data()));
    return map;
}

inline ScoreMap ccw_score_map(const RealPlane& ti_approx, const RealPlane& or_approx,
                              const RealPlane& or_mask) {
    const RealPlane* a = &ti_approx;
    const RealPlane* b = &or_approx;
    return ccw_score_map_channels(std::span<const RealPlane>(a, 1), std::span<const RealPlane>(b, 1),
                                  or_mask, ScoringMode::raw);
}

inline CandidateSet top_k(const ScoreMap& map, int k) {
    if (map.scores.values().empty()) throw EmptyInputError("top_k on empty score map");
    if (k < 1) throw ConfigError("candidate count must be >= 1");
    const int h = map.scores.height(), w = map.scores.width();
    const int kk = static_cast<int>(std::min<std::int64_t>(k, static_cast<std::int64_t>(h) * w));
    std::vector<std::int32_t> rows(kk), cols(kk);
    std::vector<double> vals(kk);
    int n = 0;
    gpu_detail::check(ccw_top_k_f64(gpu_detail::ctx(), map.scores.values().data(), h, w, k,
                                    rows.data(), cols.data(), vals.data(), &n));
    CandidateSet set;
    for (int i = 0; i < n; ++i) set.entries.push_back({rows[i], cols[i], vals[i]});
    return set;
}

inline Candidate select_unconditional(const CandidateSet& cands, std::mt19937_64& rng) {
    if (cands.empty()) throw EmptyInputError("select_unconditional on empty candidate set");
    return cands.entries[bounded(rng, cands.entries.size())];
}

struct ConditionalPick {
    Candidate candidate;
    int mismatches = 0;
};

inline ConditionalPick select_conditional(const CandidateSet& cands,
                                          const std::vector<HardDatum>& hd_in_footprint,
                                          const CategoricalGrid& ti, int levels) {
    if (cands.empty()) throw EmptyInputError("select_conditional on empty candidate set");
    std::vector<std::int32_t> rows, cols;
    for (const Candidate& c : cands.entries) {
        rows.push_back(c.row);
        cols.push_back(c.col);
    }
    const std::vector<std::int32_t> hd = gpu_detail::triples(hd_in_footprint);
    const std::vector<std::uint8_t> cells = ti.bytes();
    int pick = 0, mis = 0;
    gpu_detail::check(ccw_select_conditional(gpu_detail::ctx(), rows.data(), cols.data(),
                                             static_cast<int>(rows.size()), hd.data(),
                                             static_cast<int>(hd_in_footprint.size()), cells.data(),
                                             ti.height(), ti.width(), levels, &pick, &mis));
    return ConditionalPick{cands.entries[static_cast<std::size_t>(pick)], mis};
}

// --------------------------------------------------------- simulator.hpp --
enum class FaciesMode { indicator, raw_codes };

struct SimConfig {
    int sg_height = 0;
    int sg_width = 0;
    int template_size = 0;
    int overlap = 0;
    int dwt_level = 1;
    int candidates = 1;
    int n_realizations = 1;
    std::uint64_t master_seed = 0;
    ScoringMode scoring = ScoringMode::raw;
    FaciesMode facies_mode = FaciesMode::indicator;
    bool min_cut = false;
    std::optional<HardDataSet> hard_data;
    // extension (not a reference member): the literal-config any-support mask,
    // include/ccwgpu.h ccw_sim_config::any_support
    bool any_support = false;

    int block() const noexcept { return 1 << dwt_level; }
    int stride() const noexcept { return template_size - overlap; }

    ccw_sim_config to_c() const {
        ccw_sim_config c{};
        c.sg_height = sg_height;
        c.sg_width = sg_width;
        c.template_size = template_size;
        c.overlap = overlap;
        c.dwt_level = dwt_level;
        c.candidates = candidates;
        c.n_realizations = n_realizations;
        c.scoring = scoring == ScoringMode::normalized;
        c.facies_mode = facies_mode == FaciesMode::raw_codes;
        c.min_cut = min_cut;
        c.master_seed = master_seed;
        c.any_support = any_support;
        return c;
    }
    void validate() const {
        const ccw_sim_config c = to_c();
        char msg[512];
        const int rc = ccw_validate_config(&c, 0, 0, 0, nullptr, 0, msg, sizeof msg);
        if (rc) gpu_detail::raise(rc, msg);
    }
    void validate_against(const CategoricalGrid& ti) const {
        const ccw_sim_config c = to_c();
        const std::vector<std::int32_t> hd =
            hard_data ? gpu_detail::triples(hard_data->points) : std::vector<std::int32_t>{};
        char msg[512];
        const int rc = ccw_validate_config(&c, ti.height(), ti.width(), ti.num_facies(),
                                           hard_data ? hd.data() : nullptr,
                                           hard_data ? static_cast<int>(hard_data->size()) : 0, msg,
                                           sizeof msg);
        if (rc) gpu_detail::raise(rc, msg);
    }
};

enum class OrShape { none, vertical_strip, horizontal_strip, l_shaped };

struct Placement {
    int top = 0;
    int left = 0;
    OrShape or_shape = OrShape::none;
};

enum class Corner { top_left, top_right, bottom_left, bottom_right };

inline const char* corner_name(Corner c) {
    switch (c) {
        case Corner::top_left: return "top_left";
        case Corner::top_right: return "top_right";
        case Corner::bottom_left: return "bottom_left";
        default: return "bottom_right";
    }
}

struct PlacementPlan {
    Corner origin = Corner::top_left;
    bool column_major = false;
    int work_height = 0;
    int work_width = 0;
    std::vector<Placement> placements;
    bool vertical_on_left() const noexcept {
        return origin == Corner::top_left || origin == Corner::bottom_left;
    }
    bool horizontal_on_top() const noexcept {
        return origin == Corner::top_left || origin == Corner::top_right;
    }
};

// Consumes exactly two draws from rng (simulator.hpp:154-155).
inline PlacementPlan plan_raster_path(const SimConfig& cfg, std::mt19937_64& rng) {
    cfg.validate();
    PlacementPlan plan;
    plan.origin = static_cast<Corner>(bounded(rng, 4));
    plan.column_major = bounded(rng, 2) == 1;
    const ccw_sim_config c = cfg.to_c();
    const int s = cfg.stride();
    const int cap = ((cfg.sg_height + s) / s + 2) * ((cfg.sg_width + s) / s + 2);
    std::vector<std::int32_t> tops(cap), lefts(cap), shapes(cap);
    int n = 0;
    char msg[512];
    const int rc = ccw_plan_raster_path(&c, static_cast<int>(plan.origin), plan.column_major,
                                        &plan.work_height, &plan.work_width, tops.data(),
                                        lefts.data(), shapes.data(), cap, &n, msg, sizeof msg);
    if (rc) gpu_detail::raise(rc, msg);
    for (int i = 0; i < n; ++i)
        plan.placements.push_back({tops[i], lefts[i], static_cast<OrShape>(shapes[i])});
    return plan;
}

struct OrGeometry {
    OrShape shape = OrShape::none;
    bool vertical_on_left = true;
    bool horizontal_on_top = true;
    int overlap = 0;
};

inline CategoricalGrid min_cut_stitch(const CategoricalGrid& existing,
                                      const CategoricalGrid& incoming, const OrGeometry& geom) {
    if (existing.height() != incoming.height() || existing.width() != incoming.width())
        throw StructureError("existing and incoming patch sizes disagree");
    if (geom.shape == OrShape::none) return incoming;
    const int t = incoming.height();
    if (geom.overlap < 1 || geom.overlap >= t) throw StructureError("overlap band width out of range");
    const std::vector<std::uint8_t> e = existing.bytes(), i = incoming.bytes();
    std::vector<std::uint8_t> o(static_cast<std::size_t>(t) * t);
    gpu_detail::check(ccw_min_cut_stitch(gpu_detail::ctx(), e.data(), i.data(), t,
                                         static_cast<int>(geom.shape), geom.vertical_on_left,
                                         geom.horizontal_on_top, geom.overlap, o.data()));
    return CategoricalGrid(t, t, std::max(existing.num_facies(), incoming.num_facies()),
                           std::vector<int>(o.begin(), o.end()));
}

struct SimDiagnostics {
    std::uint64_t seed = 0;
    Corner origin = Corner::top_left;
    bool column_major = false;
    int work_height = 0;
    int work_width = 0;
    int placement_count = 0;
    int hard_data_count = 0;
    int pre_overwrite_mismatches = 0;
    double wall_seconds = 0.0;
    double pre_overwrite_mismatch_rate() const noexcept {
        return hard_data_count > 0 ? static_cast<double>(pre_overwrite_mismatches) / hard_data_count : 0.0;
    }
};

struct SimTrace {
    struct PasteEvent {
        Placement placement;
        int ti_row = 0;
        int ti_col = 0;
        CategoricalGrid pasted;
    };
    std::vector<PasteEvent> events;
};

struct SimResult {
    CategoricalGrid realization;
    SimDiagnostics diagnostics;
};

namespace gpu_detail {

// fn(i) for i in [0, n) on up to 16 host threads (boundary glue: converting
// the library's byte grids into the reference's int grids).
template <class F>
inline void parallel_for(int n, F&& fn) {
    const int nt = std::max(1, std::min({n, 16, static_cast<int>(std::thread::hardware_concurrency())}));
    if (nt <= 1) {
        for (int i = 0; i < n; ++i) fn(i);
        return;
    }
    std::vector<std::thread> th;
    std::exception_ptr err;
    std::mutex mu;
    for (int t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            try {
                for (int i = t; i < n; i += nt) fn(i);
            } catch (...) {
                std::lock_guard<std::mutex> lk(mu);
                if (!err) err = std::current_exception();
            }
        });
    for (auto& x : th) x.join();
    if (err) std::rethrow_exception(err);
}

// One device TI handle (pyramid built once on the GPU).
struct TiHandle {
    ccw_ti* h = nullptr;
    TiHandle(const CategoricalGrid& ti, const SimConfig& cfg) {
        const std::vector<std::uint8_t> cells = ti.bytes();
        check(ccw_ti_create(ctx(), cells.data(), ti.height(), ti.width(), ti.num_facies(),
                            cfg.dwt_level, cfg.facies_mode == FaciesMode::raw_codes, &h));
    }
    ~TiHandle() { ccw_ti_destroy(h); }
    TiHandle(const TiHandle&) = delete;
    TiHandle& operator=(const TiHandle&) = delete;
};

inline std::vector<SimResult> run(const CategoricalGrid& ti, const SimConfig& cfg,
                                  const std::vector<std::uint64_t>& seeds,
                                  std::vector<SimTrace>* traces) {
    cfg.validate_against(ti);
    const auto t0 = std::chrono::steady_clock::now();
    TiHandle th(ti, cfg);
    const ccw_sim_config c = cfg.to_c();
    const int n = static_cast<int>(seeds.size());
    const std::size_t sg = static_cast<std::size_t>(cfg.sg_height) * cfg.sg_width;
    std::vector<std::uint8_t> out(sg * n);
    std::vector<ccw_diag> diags(n);
    const std::vector<std::int32_t> hd =
        cfg.hard_data ? triples(cfg.hard_data->points) : std::vector<std::int32_t>{};
    const int t = cfg.template_size, s = cfg.stride();
    const int cap = ((cfg.sg_height + s) / s + 2) * ((cfg.sg_width + s) / s + 2);
    std::vector<std::vector<std::int32_t>> tb;
    std::vector<std::vector<std::uint8_t>> pb;
    std::vector<ccw_trace> ct;
    if (traces) {
        tb.assign(static_cast<std::size_t>(n) * 5, std::vector<std::int32_t>(cap));
        pb.assign(n, std::vector<std::uint8_t>(static_cast<std::size_t>(cap) * t * t));
        for (int r = 0; r < n; ++r)
            ct.push_back(ccw_trace{cap, 0, tb[5 * r].data(), tb[5 * r + 1].data(), tb[5 * r + 2].data(),
                                   tb[5 * r + 3].data(), tb[5 * r + 4].data(), pb[r].data()});
    }
    check(ccw_simulate(ctx(), th.h, &c, seeds.data(), n, cfg.hard_data ? hd.data() : nullptr,
                       cfg.hard_data ? static_cast<int>(cfg.hard_data->size()) : 0, out.data(),
                       diags.data(), traces ? ct.data() : nullptr));
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::vector<SimResult> res(n);
    // the realizations as the reference's std::vector<int> grids: one host
    // thread per realization range (100 M ints for config 1)
    parallel_for(n, [&](int r) {
        res[r].realization = CategoricalGrid(
            cfg.sg_height, cfg.sg_width, ti.num_facies(),
            std::vector<int>(out.begin() + static_cast<std::ptrdiff_t>(sg * r),
                             out.begin() + static_cast<std::ptrdiff_t>(sg * (r + 1))));
    });
    for (int r = 0; r < n; ++r) {
        SimDiagnostics& d = res[r].diagnostics;
        d.seed = diags[r].seed;
        d.origin = static_cast<Corner>(diags[r].origin);
        d.column_major = diags[r].column_major != 0;
        d.work_height = diags[r].work_height;
        d.work_width = diags[r].work_width;
        d.placement_count = diags[r].placement_count;
        d.hard_data_count = diags[r].hard_data_count;
        d.pre_overwrite_mismatches = diags[r].pre_overwrite_mismatches;
        d.wall_seconds = wall;
        if (traces) {
            SimTrace& tr = (*traces)[r];
            tr.events.clear();
            for (int e = 0; e < ct[r].count; ++e) {
                const std::uint8_t* p = pb[r].data() + static_cast<std::size_t>(e) * t * t;
                tr.events.push_back({Placement{ct[r].top[e], ct[r].left[e], static_cast<OrShape>(ct[r].shape[e])},
                                     ct[r].ti_row[e], ct[r].ti_col[e],
                                     CategoricalGrid(t, t, ti.num_facies(), std::vector<int>(p, p + t * t))});
            }
        }
    }
    return res;
}

}  // namespace gpu_detail

inline SimResult simulate_one(const CategoricalGrid& ti, const SimConfig& cfg, std::uint64_t seed,
                              SimTrace* trace = nullptr) {
    std::vector<SimTrace> tr(1);
    auto res = gpu_detail::run(ti, cfg, {seed}, trace ? &tr : nullptr);
    if (trace) *trace = std::move(tr[0]);
    return std::move(res[0]);
}

inline std::vector<SimResult> simulate_ensemble(const CategoricalGrid& ti, const SimConfig& cfg,
                                                int workers = 1) {
    (void)workers;  // one batched device call; output is worker-count invariant
    cfg.validate_against(ti);
    std::vector<std::uint64_t> seeds;
    for (int r = 0; r < cfg.n_realizations; ++r)
        seeds.push_back(mix64(cfg.master_seed, static_cast<std::uint64_t>(r) + 1));
    return gpu_detail::run(ti, cfg, seeds, nullptr);
}

}  // namespace ccwsim
