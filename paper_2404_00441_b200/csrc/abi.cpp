// abi.cpp -- the extern "C" boundary of libccwgpu.so plus the host-side
// logic that stays on the CPU by nature: configuration validation, the raster
// plan and the mt19937_64 draw schedule.  Messages match the reference's
// exception texts (tests match substrings such as "overlap" / "template").
#include <algorithm>
#include <atomic>
#include <thread>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <atomic>
#include <map>
#include <utility>

#include "ccf_tc.hpp"
#include "internal.hpp"

using ccwgpu::Fail;

namespace {

thread_local std::string g_err;  // errors raised before a context exists

std::string fmt(const char* f, ...) __attribute__((format(printf, 1, 2)));
std::string fmt(const char* f, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, f);
    vsnprintf(buf, sizeof buf, f, ap);
    va_end(ap);
    return buf;
}

template <typename F>
ccw_status guarded(ccw_ctx* ctx, F&& f) {
    try {
        if (ctx) CCW_CUDA(cudaSetDevice(ctx->device));
        f();
        return CCW_OK;
    } catch (const Fail& e) {
        (ctx ? ctx->err : g_err) = e.what();
        return e.code;
    } catch (const std::exception& e) {
        (ctx ? ctx->err : g_err) = e.what();
        return CCW_ERR_GENERIC;
    }
}

void copy_msg(char* msg, size_t len, const std::string& s) {
    if (msg && len) {
        std::snprintf(msg, len, "%s", s.c_str());
    }
}

}  // namespace

namespace ccwgpu {

// simulator.hpp:46-69
void validate_config(const ccw_sim_config& c) {
    if (c.sg_height < 1 || c.sg_width < 1)
        throw Fail(CCW_ERR_CONFIG, "sg_size: dimensions must be positive");
    if (c.dwt_level < 1) throw Fail(CCW_ERR_CONFIG, "dwt_level: must be >= 1");
    // (the reference has no upper bound; 1 << dwt_level must stay an int)
    if (c.dwt_level > 30) throw Fail(CCW_ERR_CONFIG, "dwt_level: must be <= 30");
    if (c.template_size < 2) throw Fail(CCW_ERR_CONFIG, "template: must be >= 2");
    if (c.overlap < 1 || c.overlap >= c.template_size)
        throw Fail(CCW_ERR_CONFIG, "overlap: must be in [1, template)");
    const int b = 1 << c.dwt_level;
    if (c.template_size % b != 0)
        throw Fail(CCW_ERR_CONFIG, fmt("template: %d not divisible by 2^dwt_level = %d",
                                       c.template_size, b));
    if (c.overlap % b != 0 && !c.any_support)  // (any_support: literal-config extension)
        throw Fail(CCW_ERR_CONFIG,
                   fmt("overlap: %d not divisible by 2^dwt_level = %d", c.overlap, b));
    if (c.candidates < 1) throw Fail(CCW_ERR_CONFIG, "candidates: must be >= 1");
    if (c.n_realizations < 1) throw Fail(CCW_ERR_CONFIG, "realizations: must be >= 1");
    if (c.template_size > c.sg_height || c.template_size > c.sg_width)
        throw Fail(CCW_ERR_CONFIG, fmt("template: %d exceeds simulation grid %dx%d",
                                       c.template_size, c.sg_height, c.sg_width));
    if (c.scoring != 0 && c.scoring != 1) throw Fail(CCW_ERR_CONFIG, "scoring: must be raw or normalized");
    if (c.facies_mode != 0 && c.facies_mode != 1)
        throw Fail(CCW_ERR_CONFIG, "facies_mode: must be indicator or raw-codes");
}

// grid.hpp:151-170
static void validate_hard_data(const int32_t* hd, int n_hd, int h, int w, int nf) {
    // one bit per cell (a 4000^2 grid is 2 MB); the earlier entry of a
    // duplicate is looked up only when reporting it
    std::vector<uint64_t> seen;
    if (n_hd > 0) seen.assign((static_cast<size_t>(h) * w + 63) / 64, 0);
    for (int i = 0; i < n_hd; ++i) {
        const int r = hd[3 * i], c = hd[3 * i + 1], f = hd[3 * i + 2];
        if (r < 0 || r >= h || c < 0 || c >= w)
            throw Fail(CCW_ERR_BOUNDS,
                       fmt("hard datum %d at (%d, %d) outside %dx%d grid", i, r, c, h, w));
        if (f < 0 || f >= nf)
            throw Fail(CCW_ERR_BOUNDS,
                       fmt("hard datum %d has facies %d outside [0, %d)", i, f, nf));
        const size_t cell = static_cast<size_t>(r) * w + c;
        uint64_t& word = seen[cell >> 6];
        const uint64_t bit = 1ull << (cell & 63);
        if (word & bit) {
            int s = 0;
            while (hd[3 * s] != r || hd[3 * s + 1] != c) ++s;
            throw Fail(CCW_ERR_STRUCTURE,
                       fmt("duplicate hard data at (%d, %d): entries %d and %d", r, c, s, i));
        }
        word |= bit;
    }
}

// simulator.hpp:72-84
void validate_against(const ccw_sim_config& c, int ti_h, int ti_w, int nf, const int32_t* hd,
                      int n_hd) {
    validate_config(c);
    const int b = 1 << c.dwt_level;
    // any_support (literal-config extension): the TI is used at its top-left
    // floor(d / 2^J) * 2^J crop, the only cells a block-aligned window reaches
    const int uh = c.any_support ? ti_h / b * b : ti_h, uw = c.any_support ? ti_w / b * b : ti_w;
    if (c.template_size > uh || c.template_size > uw)
        throw Fail(CCW_ERR_CONFIG, fmt("template: %d exceeds training image %dx%d",
                                       c.template_size, ti_h, ti_w));
    if (!c.any_support && (ti_h % b != 0 || ti_w % b != 0))
        throw Fail(CCW_ERR_CONFIG,
                   fmt("training image %dx%d not divisible by 2^dwt_level = %d", ti_h, ti_w, b));
    if (hd) validate_hard_data(hd, n_hd, c.sg_height, c.sg_width, nf);
}

// 3D extension (oracle/ccw3d_oracle.h: simulator.hpp:46-84 and
// grid.hpp:151-170 over three axes); same messages as the 2D checks.
void validate_config3d(const ccw_sim3d_config& c, const int32_t* ti, int nf, const int32_t* hd, int n_hd) {
    if (c.sg[0] < 1 || c.sg[1] < 1 || c.sg[2] < 1) throw Fail(CCW_ERR_CONFIG, "sg_size: dimensions must be positive");
    if (c.dwt_level < 1) throw Fail(CCW_ERR_CONFIG, "dwt_level: must be >= 1");
    if (c.dwt_level > 10) throw Fail(CCW_ERR_CONFIG, "dwt_level: must be <= 10");
    if (c.template_size < 2) throw Fail(CCW_ERR_CONFIG, "template: must be >= 2");
    if (c.overlap < 1 || c.overlap >= c.template_size) throw Fail(CCW_ERR_CONFIG, "overlap: must be in [1, template)");
    const int b = 1 << c.dwt_level;
    if (c.template_size % b != 0)
        throw Fail(CCW_ERR_CONFIG, fmt("template: %d not divisible by 2^dwt_level = %d", c.template_size, b));
    if (!c.any_support && c.overlap % b != 0)
        throw Fail(CCW_ERR_CONFIG, fmt("overlap: %d not divisible by 2^dwt_level = %d", c.overlap, b));
    if (c.candidates < 1) throw Fail(CCW_ERR_CONFIG, "candidates: must be >= 1");
    if (c.n_realizations < 1) throw Fail(CCW_ERR_CONFIG, "realizations: must be >= 1");
    for (int a = 0; a < 3; ++a)
        if (c.template_size > c.sg[a])
            throw Fail(CCW_ERR_CONFIG, fmt("template: %d exceeds simulation grid %dx%dx%d", c.template_size, c.sg[0],
                                           c.sg[1], c.sg[2]));
    if (!ti) return;
    if (ti[0] < 1 || ti[1] < 1 || ti[2] < 1) throw Fail(CCW_ERR_DIMENSION, "grid dimensions must be positive");
    if (nf < 1 || nf > 16) throw Fail(CCW_ERR_DIMENSION, "num_facies must be in [1, 16] for the 3D path");
    for (int a = 0; a < 3; ++a) {
        const int used = c.any_support ? ti[a] / b * b : ti[a];
        if (c.template_size > used)
            throw Fail(CCW_ERR_CONFIG, fmt("template: %d exceeds training image %dx%dx%d", c.template_size, ti[0],
                                           ti[1], ti[2]));
    }
    if (!c.any_support && (ti[0] % b || ti[1] % b || ti[2] % b))
        throw Fail(CCW_ERR_CONFIG, fmt("training image %dx%dx%d not divisible by 2^dwt_level = %d", ti[0], ti[1],
                                       ti[2], b));
    if (n_hd > 0 && !hd) throw Fail(CCW_ERR_GENERIC, "null hard data");
    std::vector<uint64_t> seen;
    const size_t n = static_cast<size_t>(c.sg[0]) * c.sg[1] * c.sg[2];
    if (n_hd > 0) seen.assign((n + 63) / 64, 0);
    for (int i = 0; i < n_hd; ++i) {
        const int32_t* d = hd + 4 * i;
        if (d[0] < 0 || d[0] >= c.sg[0] || d[1] < 0 || d[1] >= c.sg[1] || d[2] < 0 || d[2] >= c.sg[2])
            throw Fail(CCW_ERR_BOUNDS, fmt("hard datum %d at (%d, %d, %d) outside %dx%dx%d grid", i, d[0], d[1], d[2],
                                           c.sg[0], c.sg[1], c.sg[2]));
        if (d[3] < 0 || d[3] >= nf)
            throw Fail(CCW_ERR_BOUNDS, fmt("hard datum %d has facies %d outside [0, %d)", i, d[3], nf));
        const size_t cell = (static_cast<size_t>(d[0]) * c.sg[1] + d[1]) * c.sg[2] + d[2];
        if (seen[cell >> 6] & (1ull << (cell & 63)))
            throw Fail(CCW_ERR_STRUCTURE, fmt("duplicate hard data at (%d, %d, %d)", d[0], d[1], d[2]));
        seen[cell >> 6] |= 1ull << (cell & 63);
    }
}

uint64_t bounded(std::mt19937_64& rng, uint64_t n) {
    const uint64_t threshold = (0 - n) % n;
    for (;;) {
        const uint64_t r = rng();
        if (r >= threshold) return r % n;
    }
}

static int padded_extent(int sg, int t, int stride) {  // simulator.hpp:125-131
    if (sg == t) return t;
    const int steps = (sg - t + stride - 1) / stride;
    return t + steps * stride;
}

Plan make_plan(const ccw_sim_config& c, std::mt19937_64& rng) {
    validate_config(c);
    const int origin = static_cast<int>(bounded(rng, 4));
    const bool column_major = bounded(rng, 2) == 1;
    return make_plan_from(c, origin, column_major);
}

Plan make_plan_from(const ccw_sim_config& c, int origin, bool column_major) {
    validate_config(c);
    const int t = c.template_size, stride = t - c.overlap;
    Plan p;
    p.origin = origin;
    p.column_major = column_major;
    p.work_h = padded_extent(c.sg_height, t, stride);
    p.work_w = padded_extent(c.sg_width, t, stride);
    const bool rows_asc = p.origin == CCW_TOP_LEFT || p.origin == CCW_TOP_RIGHT;
    const bool cols_asc = p.origin == CCW_TOP_LEFT || p.origin == CCW_BOTTOM_LEFT;
    std::vector<int> rp, cp;
    for (int q = 0; q + t <= p.work_h; q += stride) rp.push_back(q);
    for (int q = 0; q + t <= p.work_w; q += stride) cp.push_back(q);
    if (!rows_asc) std::reverse(rp.begin(), rp.end());
    if (!cols_asc) std::reverse(cp.begin(), cp.end());
    const std::vector<int>& outer = p.column_major ? cp : rp;
    const std::vector<int>& inner = p.column_major ? rp : cp;
    p.n_outer = static_cast<int>(outer.size());
    p.n_inner = static_cast<int>(inner.size());
    const size_t n = outer.size() * inner.size();
    p.tops.reserve(n);
    p.lefts.reserve(n);
    p.shapes.reserve(n);
    for (int o = 0; o < p.n_outer; ++o)
        for (int i = 0; i < p.n_inner; ++i) {
            p.tops.push_back(p.column_major ? inner[i] : outer[o]);
            p.lefts.push_back(p.column_major ? outer[o] : inner[i]);
            int sh;
            if (o == 0 && i == 0)
                sh = CCW_OR_NONE;
            else if (o == 0)
                sh = p.column_major ? CCW_OR_HORIZONTAL : CCW_OR_VERTICAL;
            else if (i == 0)
                sh = p.column_major ? CCW_OR_VERTICAL : CCW_OR_HORIZONTAL;
            else
                sh = CCW_OR_L;
            p.shapes.push_back(sh);
            p.outer_idx.push_back(o);
            p.inner_idx.push_back(i);
        }
    return p;
}

namespace {
struct DevCache {
    std::mutex mu;
    std::map<void*, std::pair<int, size_t>> live;                   // ptr -> (device, bytes)
    std::multimap<std::pair<int, size_t>, void*> idle;              // (device, bytes) -> ptr
};
DevCache& dev_cache() {
    static DevCache* c = new DevCache();  // intentionally leaked: outlives static destructors
    return *c;
}
}  // namespace

void* cache_alloc(int device, size_t bytes) {
    bytes = std::max<size_t>(bytes, 1);
    DevCache& c = dev_cache();
    {
        std::lock_guard<std::mutex> lk(c.mu);
        auto it = c.idle.find({device, bytes});
        if (it != c.idle.end()) {
            void* p = it->second;
            c.idle.erase(it);
            c.live[p] = {device, bytes};
            return p;
        }
    }
    void* p = nullptr;
    CCW_CUDA(cudaMalloc(&p, bytes));
    std::lock_guard<std::mutex> lk(c.mu);
    c.live[p] = {device, bytes};
    return p;
}

void cache_free(void* p) {
    if (!p) return;
    DevCache& c = dev_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.live.find(p);
    if (it == c.live.end()) return;
    c.idle.emplace(it->second, p);
    c.live.erase(it);
}

}  // namespace ccwgpu

// ================================================================ C-ABI ===

extern "C" {

ccw_status ccw_ctx_create(int device, ccw_ctx** out) {
    if (!out) {
        g_err = "ccw_ctx_create: null output pointer";
        return CCW_ERR_GENERIC;
    }
    *out = nullptr;
    auto* ctx = new ccw_ctx();
    ctx->device = device;
    ccw_status st = guarded(nullptr, [&] {
        int n = 0;
        CCW_CUDA(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n)
            throw Fail(CCW_ERR_CUDA, fmt("device %d not present (%d visible)", device, n));
        CCW_CUDA(cudaSetDevice(device));
        CCW_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    });
    if (st != CCW_OK) {
        delete ctx;
        return st;
    }
    *out = ctx;
    return CCW_OK;
}

void ccw_ctx_destroy(ccw_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (cudaStream_t s : ctx->gstreams) cudaStreamSynchronize(s);
    for (cudaStream_t s : ctx->copy_streams) cudaStreamSynchronize(s);
    ccwgpu::nccl_comm_destroy(ctx->nccl_comm);
    for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
    if (ctx->upload_done) cudaEventDestroy(ctx->upload_done);
    for (auto& sl : ctx->aslot)
        for (cudaEvent_t e : {sl.done, sl.t0, sl.t1})
            if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : ctx->stage_ev)
        if (e) cudaEventDestroy(e);
    for (cudaStream_t s : ctx->gstreams) cudaStreamDestroy(s);
    for (cudaStream_t s : ctx->copy_streams) cudaStreamDestroy(s);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;  // every DevBuf / HostBuf member frees its memory (RAII)
}

const char* ccw_last_error(const ccw_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

void* ccw_ctx_stream(ccw_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

ccw_status ccw_ctx_set_profiling(ccw_ctx* ctx, int enabled) {
    if (!ctx) return CCW_ERR_GENERIC;
    ctx->profiling = enabled != 0;
    return CCW_OK;
}

ccw_status ccw_ctx_last_timing(ccw_ctx* ctx, ccw_timing* out) {
    if (!ctx || !out) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        ccwgpu::async_settle(ctx, true);  // (an asynchronous call's counters)
        *out = ctx->timing;
    });
}

ccw_status ccw_ctx_set_ccf_variant(ccw_ctx* ctx, int variant) {
    if (!ctx) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        if (variant < 0 || variant > 2)
            throw Fail(CCW_ERR_CONFIG, fmt("ccf variant %d unknown", variant));
        ctx->ccf_variant = variant;
    });
}

ccw_status ccw_nccl_unique_id(uint8_t* id128) {
    if (!id128) {
        g_err = "ccw_nccl_unique_id: null output pointer";
        return CCW_ERR_GENERIC;
    }
    return guarded(nullptr, [&] { ccwgpu::nccl_unique_id(id128); });
}

ccw_status ccw_ctx_set_position_shards(ccw_ctx* ctx, int nranks, int rank, const uint8_t* nccl_id,
                                       int virtual_shards) {
    if (!ctx) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        if (nranks < 1 || rank < 0 || rank >= nranks)
            throw Fail(CCW_ERR_CONFIG, fmt("position shards: rank %d of %d is invalid", rank, nranks));
        if (virtual_shards < 1 || virtual_shards > 64)
            throw Fail(CCW_ERR_CONFIG, fmt("position shards: %d virtual shards (1-64)", virtual_shards));
        if (nranks > 1 && !nccl_id)
            throw Fail(CCW_ERR_CONFIG, "position shards: more than one rank needs an NCCL unique id");
        CCW_CUDA(cudaStreamSynchronize(ctx->stream));
        for (cudaStream_t s : ctx->gstreams) CCW_CUDA(cudaStreamSynchronize(s));
        // the old sharding state is dropped first; the new one is committed only
        // once its communicator exists, so a failed init leaves sharding off
        ccwgpu::nccl_comm_destroy(ctx->nccl_comm);
        ctx->nccl_comm = nullptr;
        ctx->shard_nranks = 1;
        ctx->shard_rank = 0;
        ctx->shard_virtual = 1;
        void* comm = nccl_id ? ccwgpu::nccl_comm_init(nranks, rank, nccl_id) : nullptr;
        ctx->nccl_comm = comm;
        ctx->shard_nranks = nranks;
        ctx->shard_rank = rank;
        ctx->shard_virtual = virtual_shards;
    });
}

ccw_status ccw_ctx_set_option(ccw_ctx* ctx, const char* name, long long value) {
    if (!ctx) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        int* slot = name ? ccwgpu::option_slot(ctx->opt, name) : nullptr;
        if (!slot) throw Fail(CCW_ERR_CONFIG, fmt("option: unknown name '%s'", name ? name : "(null)"));
        if (value < 0 || value > (1 << 20)) throw Fail(CCW_ERR_CONFIG, fmt("option %s: value out of range", name));
        *slot = static_cast<int>(value);
    });
}

ccw_status ccw_measure_fp32_peak(ccw_ctx* ctx, double* tflops) {
    if (!ctx || !tflops) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] { *tflops = ccwgpu::measure_ffma_peak(ctx); });
}

ccw_status ccw_measure_int_peak(ccw_ctx* ctx, int kind, double* tops) {
    if (!ctx || !tops) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        if (kind != 0 && kind != 1) throw Fail(CCW_ERR_CONFIG, "int peak: kind must be 0 (IMAD) or 1 (dp4a)");
        *tops = ccwgpu::measure_int_peak(ctx, kind);
    });
}

ccw_status ccw_measure_ccf_screen(ccw_ctx* ctx, ccw_ti* ti, int template_size, int njobs, int iters,
                                  double* ms_per_launch) {
    if (!ctx || !ti || !ms_per_launch) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        const int Tc = template_size >> ti->J;
        if (Tc < 1 || Tc > std::min(ti->hc, ti->wc) || njobs < 1 || iters < 1)
            throw Fail(CCW_ERR_CONFIG, "ccw_measure_ccf_screen: bad template size, job or iteration count");
        if (ti->nscr < 1) throw Fail(CCW_ERR_CONFIG, "ccw_measure_ccf_screen: this TI has no screen planes");
        *ms_per_launch = ccwgpu::measure_ccf_screen(ti, Tc, njobs, iters, ctx->stream);
    });
}

ccw_status ccw_measure_i8_peak(ccw_ctx* ctx, double* tops) {
    if (!ctx || !tops) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] { *tops = ccwgpu::measure_i8_peak(ctx->stream); });
}

uint64_t ccw_mix64(uint64_t seed, uint64_t index) {  // rng.hpp:11-16
    uint64_t z = seed + index * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// A large host upload: the context's host threads copy chunks into pinned
// staging and each chunk leaves with its own async copy as soon as it is
// staged (a pageable cudaMemcpy goes through the driver's bounce buffer one
// chunk at a time, ~4x slower for a 32 MB 3D training image).  The staging
// buffer is reused by the next upload only after these copies complete.
static void upload_host(ccw_ctx* ctx, void* d, const void* h, size_t n) {
    constexpr size_t kSmall = 1u << 20, kChunk = 2u << 20;
    if (n < kSmall) {
        CCW_CUDA(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, ctx->stream));
        return;
    }
    if (ctx->upload_done) CCW_CUDA(cudaEventSynchronize(ctx->upload_done));
    uint8_t* stage = static_cast<uint8_t*>(ctx->h_upload.get(n));
    const int nchunk = static_cast<int>((n + kChunk - 1) / kChunk);
    // chunks are staged in parallel; copies are issued in chunk order on the
    // context stream as each one is ready
    std::vector<std::atomic<int>> ready(nchunk);
    for (auto& r : ready) r.store(0);
    const int device = ctx->device;
    cudaError_t issue_err = cudaSuccess;  // (the issuer's first error, rethrown by the caller)
    std::thread issuer([&] {
        cudaSetDevice(device);
        for (int i = 0; i < nchunk; ++i) {
            while (!ready[i].load(std::memory_order_acquire)) std::this_thread::yield();
            const size_t o = static_cast<size_t>(i) * kChunk;
            const cudaError_t e = cudaMemcpyAsync(static_cast<uint8_t*>(d) + o, stage + o, std::min(kChunk, n - o),
                                                  cudaMemcpyHostToDevice, ctx->stream);
            if (e != cudaSuccess && issue_err == cudaSuccess) issue_err = e;
        }
    });
    ctx->pool.run(nchunk, [&](int i) {
        const size_t o = static_cast<size_t>(i) * kChunk;
        std::memcpy(stage + o, static_cast<const uint8_t*>(h) + o, std::min(kChunk, n - o));
        ready[i].store(1, std::memory_order_release);
    });
    issuer.join();
    if (issue_err != cudaSuccess)
        throw Fail(CCW_ERR_CUDA, std::string("cudaMemcpyAsync (staged upload): ") + cudaGetErrorString(issue_err));
    if (!ctx->upload_done) CCW_CUDA(cudaEventCreateWithFlags(&ctx->upload_done, cudaEventDisableTiming));
    CCW_CUDA(cudaEventRecord(ctx->upload_done, ctx->stream));
    CCW_CUDA(cudaGetLastError());
}

static ccw_status ti_create_impl(ccw_ctx* ctx, const uint8_t* cells, bool device_ptr, int h,
                                 int w, int nf, int levels, int mode, ccw_ti** out) {
    if (!ctx || !out) return CCW_ERR_GENERIC;
    *out = nullptr;
    auto* ti = new ccw_ti();
    ccw_status st = guarded(ctx, [&] {
        if (h <= 0 || w <= 0) throw Fail(CCW_ERR_DIMENSION, "grid dimensions must be positive");
        if (nf <= 0) throw Fail(CCW_ERR_DIMENSION, "num_facies must be positive");
        if (nf > 255) throw Fail(CCW_ERR_DIMENSION, "num_facies must be <= 255 (uint8 codes)");
        if (levels < 1) throw Fail(CCW_ERR_DIMENSION, "decomposition level must be >= 1");
        // extents 2^J does not divide are kept (the pyramid covers the top-left
        // floor(d / 2^J) blocks); simulate rejects them unless the config
        // enables the literal-config extension (validate_against)
        if (levels > 30 || (h >> levels) < 1 || (w >> levels) < 1)
            throw Fail(CCW_ERR_CONFIG,
                       fmt("training image %dx%d smaller than one 2^dwt_level = %d block", h, w,
                           1 << std::min(levels, 30)));
        if (mode != 0 && mode != 1) throw Fail(CCW_ERR_CONFIG, "facies_mode: unknown");
        ti->ctx = ctx;
        ti->device = ctx->device;
        ti->h = h;
        ti->w = w;
        ti->F = nf;
        ti->J = levels;
        ti->mode = mode;
        ti->hc = h >> levels;
        ti->wc = w >> levels;
        ti->nch = mode == 0 ? nf : 1;
        ti->nscr = mode == 0 ? nf - 1 : 1;
        const size_t n = static_cast<size_t>(h) * w;
        const size_t nc = static_cast<size_t>(ti->hc) * ti->wc;
        ti->d_codes = static_cast<uint8_t*>(ccwgpu::cache_alloc(ti->device, n));
        ti->d_ti64 = static_cast<double*>(ccwgpu::cache_alloc(ti->device, sizeof(double) * nc * ti->nch));
        ti->d_scr = static_cast<float*>(ccwgpu::cache_alloc(ti->device, sizeof(float) * nc * std::max(ti->nscr, 1)));
        // content key: host cells hashed with the shape; device cells get a unique id
        uint64_t key = 0x9E3779B97F4A7C15ull ^ (static_cast<uint64_t>(h) << 40) ^
                       (static_cast<uint64_t>(w) << 16) ^ (static_cast<uint64_t>(nf) << 8) ^
                       (static_cast<uint64_t>(levels) << 4) ^ static_cast<uint64_t>(mode);
        if (!device_ptr) {
            // four independent multiply-rotate lanes, folded at the end
            uint64_t a[4] = {key, key + 1, key + 2, key + 3};
            constexpr uint64_t kM = 0x9FB21C651E98DF25ull;
            size_t i = 0;
            for (; i + 32 <= n; i += 32)
                for (int l = 0; l < 4; ++l) {
                    uint64_t v;
                    std::memcpy(&v, cells + i + 8 * l, 8);
                    a[l] = ((a[l] ^ v) * kM);
                    a[l] ^= a[l] >> 29;
                }
            for (; i < n; ++i) a[0] = (a[0] ^ cells[i]) * kM;
            key = ccwgpu::mix_key(a[0] ^ ccwgpu::mix_key(a[1] ^ ccwgpu::mix_key(a[2] ^ ccwgpu::mix_key(a[3]))));
        } else {
            static std::atomic<uint64_t> next_id{1};
            key = ccwgpu::mix_key(key ^ (next_id.fetch_add(1) << 1 | 1));
        }
        ti->key = key;
        if (device_ptr) {
            CCW_CUDA(cudaMemcpyAsync(ti->d_codes, cells, n, cudaMemcpyDeviceToDevice, ctx->stream));
        } else {
            upload_host(ctx, ti->d_codes, cells, n);
            // grid.hpp:36-40 code-range check, on the device (the device-pointer path trusts its caller)
            const size_t bad = ccwgpu::first_bad_code(ti->d_codes, n, nf, ctx->stream, ctx->chk.as<unsigned long long>(1));
            if (bad < n)
                throw Fail(CCW_ERR_BOUNDS, fmt("cell %zu holds code %d outside [0, %d)", bad,
                                               static_cast<int>(cells[bad]), nf));
        }
        ccwgpu::build_pyramid(ti, ctx->stream);
    });
    if (st != CCW_OK) {
        ccw_ti_destroy(ti);
        return st;
    }
    *out = ti;
    return CCW_OK;
}

ccw_status ccw_ti_create(ccw_ctx* ctx, const uint8_t* cells, int h, int w, int nf, int levels,
                         int mode, ccw_ti** out) {
    return ti_create_impl(ctx, cells, false, h, w, nf, levels, mode, out);
}

ccw_status ccw_ti_create_device(ccw_ctx* ctx, const uint8_t* d_cells, int h, int w, int nf,
                                int levels, int mode, ccw_ti** out) {
    return ti_create_impl(ctx, d_cells, true, h, w, nf, levels, mode, out);
}

void ccw_ti_destroy(ccw_ti* ti) {
    if (!ti) return;
    // The owning context may already be gone: drain the device, then hand
    // the buffers back to the process-wide cache.
    cudaSetDevice(ti->device);
    cudaDeviceSynchronize();
    ccwgpu::cache_free(ti->d_codes);
    ccwgpu::cache_free(ti->d_ti64);
    ccwgpu::cache_free(ti->d_scr);
    for (auto& kv : ti->im2col) ccwgpu::cache_free(kv.second);
    for (auto& kv : ti->nnmap) ccwgpu::cache_free(kv.second);
    for (auto& kv : ti->umap) ccwgpu::cache_free(kv.second);
    delete ti;
}

ccw_status ccw_ti_apex(ccw_ti* ti, double* out) {
    if (!ti) return CCW_ERR_GENERIC;
    return guarded(ti->ctx, [&] {
        CCW_CUDA(cudaMemcpyAsync(out, ti->d_ti64,
                                 sizeof(double) * ti->nch * static_cast<size_t>(ti->hc) * ti->wc,
                                 cudaMemcpyDeviceToHost, ti->ctx->stream));
        CCW_CUDA(cudaStreamSynchronize(ti->ctx->stream));
    });
}

static void check_ti_cfg(ccw_ti* ti, const ccw_sim_config* cfg, const int32_t* hd, int n_hd) {
    if (!cfg) throw Fail(CCW_ERR_GENERIC, "null config");
    ccwgpu::validate_against(*cfg, ti->h, ti->w, ti->F, hd, n_hd);
    if (cfg->dwt_level != ti->J)
        throw Fail(CCW_ERR_CONFIG, fmt("dwt_level: %d does not match the TI pyramid level %d",
                                       cfg->dwt_level, ti->J));
    if (cfg->facies_mode != ti->mode)
        throw Fail(CCW_ERR_CONFIG, "facies_mode: does not match the TI pyramid");
}

ccw_status ccw_simulate(ccw_ctx* ctx, ccw_ti* ti, const ccw_sim_config* cfg,
                        const uint64_t* seeds, int n_real, const int32_t* hd, int n_hd,
                        uint8_t* out, ccw_diag* diag, ccw_trace* traces) {
    if (!ctx || !ti) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        check_ti_cfg(ti, cfg, hd, n_hd);
        if (n_real < 1) throw Fail(CCW_ERR_CONFIG, "realizations: must be >= 1");
        ccwgpu::run_simulation(ctx, ti, *cfg, seeds, n_real, hd, n_hd, nullptr, out, diag,
                               traces);
    });
}

ccw_status ccw_simulate_device(ccw_ctx* ctx, ccw_ti* ti, const ccw_sim_config* cfg,
                               const uint64_t* seeds, int n_real, const int32_t* hd, int n_hd,
                               uint8_t* d_out, ccw_diag* diag) {
    if (!ctx || !ti) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        check_ti_cfg(ti, cfg, hd, n_hd);
        if (n_real < 1) throw Fail(CCW_ERR_CONFIG, "realizations: must be >= 1");
        ccwgpu::run_simulation(ctx, ti, *cfg, seeds, n_real, hd, n_hd, d_out, nullptr, diag,
                               nullptr);
    });
}

ccw_status ccw_simulate_device_async(ccw_ctx* ctx, ccw_ti* ti, const ccw_sim_config* cfg,
                                     const uint64_t* seeds, int n_real, const int32_t* hd, int n_hd,
                                     uint8_t* d_out) {
    if (!ctx || !ti) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        check_ti_cfg(ti, cfg, hd, n_hd);
        if (n_real < 1) throw Fail(CCW_ERR_CONFIG, "realizations: must be >= 1");
        if (!d_out) throw Fail(CCW_ERR_GENERIC, "null output");
        ccwgpu::run_simulation(ctx, ti, *cfg, seeds, n_real, hd, n_hd, d_out, nullptr, nullptr, nullptr, true);
    });
}

ccw_status ccw_ctx_synchronize(ccw_ctx* ctx) {
    if (!ctx) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        CCW_CUDA(cudaStreamSynchronize(ctx->stream));
        ccwgpu::async_settle(ctx, true);
        if (!ctx->async_err.empty()) {
            const std::string e = ctx->async_err;
            ctx->async_err.clear();
            throw Fail(CCW_ERR_GENERIC, e);
        }
    });
}

ccw_status ccw_simulate_ensemble(ccw_ctx* ctx, ccw_ti* ti, const ccw_sim_config* cfg,
                                 const int32_t* hd, int n_hd, uint8_t* out, ccw_diag* diag) {
    if (!ctx || !ti) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        check_ti_cfg(ti, cfg, hd, n_hd);
        std::vector<uint64_t> seeds(static_cast<size_t>(cfg->n_realizations));
        for (int r = 0; r < cfg->n_realizations; ++r)
            seeds[r] = ccw_mix64(cfg->master_seed, static_cast<uint64_t>(r) + 1);
        ccwgpu::run_simulation(ctx, ti, *cfg, seeds.data(), cfg->n_realizations, hd, n_hd,
                               nullptr, out, diag, nullptr);
    });
}

ccw_status ccw_dwt2_single_f64(ccw_ctx* ctx, const double* in, int h, int w, double* a,
                               double* dh, double* dv, double* dd) {
    if (!ctx) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        if (h <= 0 || w <= 0) throw Fail(CCW_ERR_DIMENSION, "plane dimensions must be positive");
        if (h % 2 != 0 || w % 2 != 0)
            throw Fail(CCW_ERR_DIMENSION,
                       fmt("dwt2_single requires even dimensions, got %dx%d", h, w));
        ccwgpu::op_dwt2_single(ctx, in, h, w, a, dh, dv, dd);
    });
}

ccw_status ccw_idwt2_single_f64(ccw_ctx* ctx, const double* a, const double* dh,
                                const double* dv, const double* dd, int hh, int hw,
                                double* out) {
    if (!ctx) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        if (hh <= 0 || hw <= 0) throw Fail(CCW_ERR_DIMENSION, "plane dimensions must be positive");
        ccwgpu::op_idwt2_single(ctx, a, dh, dv, dd, hh, hw, out);
    });
}

ccw_status ccw_dwt2_f64(ccw_ctx* ctx, const double* in, int h, int w, int levels, double* apex,
                        double* details) {
    if (!ctx) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        if (h <= 0 || w <= 0) throw Fail(CCW_ERR_DIMENSION, "plane dimensions must be positive");
        if (levels < 1) throw Fail(CCW_ERR_DIMENSION, "decomposition level must be >= 1");
        if (levels > 30 || h % (1 << levels) != 0 || w % (1 << levels) != 0)
            throw Fail(CCW_ERR_DIMENSION,
                       fmt("plane %dx%d not divisible by 2^%d", h, w, levels));
        ccwgpu::op_dwt2(ctx, in, h, w, levels, apex, details);
    });
}

ccw_status ccw_idwt2_f64(ccw_ctx* ctx, const double* apex, const double* details, int h, int w,
                         int levels, double* out) {
    if (!ctx) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        if (levels < 1 || levels > 30 || h <= 0 || w <= 0 || (h >> levels) < 1 ||
            (w >> levels) < 1 || h % (1 << levels) != 0 || w % (1 << levels) != 0)
            throw Fail(CCW_ERR_STRUCTURE, "pyramid level count inconsistent");
        if (!details) throw Fail(CCW_ERR_STRUCTURE, "pyramid level count inconsistent");
        ccwgpu::op_idwt2(ctx, apex, details, h, w, levels, out);
    });
}

ccw_status ccw_score_map_f64(ccw_ctx* ctx, const double* ti, const double* tmpl, int nch,
                             int ti_h, int ti_w, int t_h, int t_w, const double* mask,
                             int scoring, double* out) {
    if (!ctx) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        if (nch < 1) throw Fail(CCW_ERR_STRUCTURE, "channel counts disagree");
        // matcher.hpp:102-123
        if (t_h > ti_h || t_w > ti_w)
            throw Fail(CCW_ERR_DIMENSION,
                       fmt("template %dx%d larger than TI coefficients %dx%d", t_h, t_w, ti_h, ti_w));
        for (int f = 0; f < nch; ++f)
            for (int i = 0; i < t_h * t_w; ++i) {
                const double m = mask[i];
                if (m != 0.0 && m != 1.0) throw Fail(CCW_ERR_STRUCTURE, "mask values must be 0 or 1");
                if (m == 0.0 && tmpl[static_cast<size_t>(f) * t_h * t_w + i] != 0.0)
                    throw Fail(CCW_ERR_STRUCTURE,
                               "template carries nonzero values outside the mask");
            }
        ccwgpu::op_score_map(ctx, ti, tmpl, nch, ti_h, ti_w, t_h, t_w, mask, scoring, out);
    });
}

ccw_status ccw_top_k_f64(ccw_ctx* ctx, const double* scores, int h, int w, int k, int32_t* rows,
                         int32_t* cols, double* vals, int* n_out) {
    if (!ctx) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        if (h <= 0 || w <= 0 || !scores) throw Fail(CCW_ERR_EMPTY, "top_k on empty score map");
        if (k < 1) throw Fail(CCW_ERR_CONFIG, "candidate count must be >= 1");
        ccwgpu::op_top_k(ctx, scores, h, w, k, rows, cols, vals, n_out);
    });
}

ccw_status ccw_select_conditional(ccw_ctx* ctx, const int32_t* rows, const int32_t* cols,
                                  int n_cands, const int32_t* hd, int n_hd, const uint8_t* ti,
                                  int ti_h, int ti_w, int levels, int* pick, int* mismatches) {
    if (!ctx) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        if (n_cands < 1) throw Fail(CCW_ERR_EMPTY, "select_conditional on empty candidate set");
        // CategoricalGrid::at bounds (grid.hpp:69-75)
        for (int i = 0; i < n_cands; ++i)
            for (int d = 0; d < n_hd; ++d) {
                const int r = (rows[i] << levels) + hd[3 * d];
                const int c = (cols[i] << levels) + hd[3 * d + 1];
                if (r < 0 || r >= ti_h || c < 0 || c >= ti_w)
                    throw Fail(CCW_ERR_BOUNDS, fmt("cell (%d, %d) outside %dx%d grid", r, c,
                                                   ti_h, ti_w));
            }
        ccwgpu::op_select_conditional(ctx, rows, cols, n_cands, hd, n_hd, ti, ti_h, ti_w, levels,
                                      pick, mismatches);
    });
}

ccw_status ccw_min_cut_stitch(ccw_ctx* ctx, const uint8_t* existing, const uint8_t* incoming,
                              int t, int shape, int vleft, int htop, int overlap, uint8_t* out) {
    if (!ctx) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        if (t <= 0) throw Fail(CCW_ERR_DIMENSION, "crop size must be positive");
        if (shape < 0 || shape > 3) throw Fail(CCW_ERR_STRUCTURE, "unknown overlap shape");
        if (shape != CCW_OR_NONE && (overlap < 1 || overlap >= t))
            throw Fail(CCW_ERR_STRUCTURE, "overlap band width out of range");
        ccwgpu::op_min_cut_stitch(ctx, existing, incoming, t, shape, vleft, htop, overlap, out);
    });
}

// ------------------------------------------------------------- 3D ----

ccw_status ccw_ti3d_create(ccw_ctx* ctx, const uint8_t* cells, int d0, int d1, int d2, int nf, int levels,
                           ccw_ti3d** out) {
    if (!ctx || !out) return CCW_ERR_GENERIC;
    *out = nullptr;
    auto* ti = new ccw_ti3d();
    ccw_status st = guarded(ctx, [&] {
        if (d0 <= 0 || d1 <= 0 || d2 <= 0) throw Fail(CCW_ERR_DIMENSION, "grid dimensions must be positive");
        if (nf < 1 || nf > 16) throw Fail(CCW_ERR_DIMENSION, "num_facies must be in [1, 16] for the 3D path");
        if (levels < 1 || levels > 10) throw Fail(CCW_ERR_DIMENSION, "decomposition level must be in [1, 10]");
        if (!cells) throw Fail(CCW_ERR_GENERIC, "null cells");
        const size_t n = static_cast<size_t>(d0) * d1 * d2;
        const int b = 1 << levels;
        ti->ctx = ctx;
        ti->device = ctx->device;
        ti->d[0] = d0;
        ti->d[1] = d1;
        ti->d[2] = d2;
        for (int a = 0; a < 3; ++a) ti->c[a] = ti->d[a] / b;
        if (ti->c[0] < 1 || ti->c[1] < 1 || ti->c[2] < 1)
            throw Fail(CCW_ERR_DIMENSION, "training image smaller than one 2^dwt_level block");
        ti->F = nf;
        ti->J = levels;
        ti->nscr = std::max(nf - 1, 1);
        ti->mode = (b <= 4 && ti->nscr <= 4) ? 0 : 1;
        const size_t nc = static_cast<size_t>(ti->c[0]) * ti->c[1] * ti->c[2];
        ti->d_codes = static_cast<uint8_t*>(ccwgpu::cache_alloc(ti->device, n));
        ti->d_pk = static_cast<int32_t*>(
            ccwgpu::cache_alloc(ti->device, sizeof(int32_t) * nc * (ti->mode == 0 ? 1 : ti->nscr)));
        upload_host(ctx, ti->d_codes, cells, n);
        const size_t bad = ccwgpu::first_bad_code(ti->d_codes, n, nf, ctx->stream, ctx->chk.as<unsigned long long>(1));  // (grid.hpp:36-40)
        if (bad < n)
            throw Fail(CCW_ERR_BOUNDS, fmt("cell %zu holds code %d outside [0, %d)", bad, static_cast<int>(cells[bad]), nf));
        ccwgpu::build_pyramid3d(ti, ctx->stream);
    });
    if (st != CCW_OK) {
        ccw_ti3d_destroy(ti);
        return st;
    }
    *out = ti;
    return CCW_OK;
}

void ccw_ti3d_destroy(ccw_ti3d* ti) {
    if (!ti) return;
    cudaSetDevice(ti->device);
    cudaDeviceSynchronize();
    ccwgpu::cache_free(ti->d_codes);
    ccwgpu::cache_free(ti->d_pk);
    for (auto& kv : ti->im2col) ccwgpu::cache_free(kv.second);
    delete ti;
}

ccw_status ccw_validate_config3d(const ccw_sim3d_config* cfg, const int32_t* ti_dims, int nf, const int32_t* hd,
                                 int n_hd, char* msg, size_t msg_len) {
    try {
        if (!cfg) throw Fail(CCW_ERR_GENERIC, "null config");
        ccwgpu::validate_config3d(*cfg, ti_dims, nf, hd, n_hd);
        copy_msg(msg, msg_len, "");
        return CCW_OK;
    } catch (const Fail& e) {
        copy_msg(msg, msg_len, e.what());
        g_err = e.what();
        return e.code;
    }
}

static void check_ti3d(ccw_ti3d* ti, const ccw_sim3d_config* cfg, const int32_t* hd, int n_hd) {
    if (!cfg) throw Fail(CCW_ERR_GENERIC, "null config");
    ccwgpu::validate_config3d(*cfg, ti->d, ti->F, hd, n_hd);
    if (cfg->dwt_level != ti->J)
        throw Fail(CCW_ERR_CONFIG, fmt("dwt_level: %d does not match the TI pyramid level %d", cfg->dwt_level, ti->J));
}

ccw_status ccw_simulate3d(ccw_ctx* ctx, ccw_ti3d* ti, const ccw_sim3d_config* cfg, const uint64_t* seeds, int n_real,
                          const int32_t* hd, int n_hd, uint8_t* out, ccw_diag3d* diag) {
    if (!ctx || !ti) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        check_ti3d(ti, cfg, hd, n_hd);
        if (n_real < 1) throw Fail(CCW_ERR_CONFIG, "realizations: must be >= 1");
        ccwgpu::run_simulation3d(ctx, ti, *cfg, seeds, n_real, hd, n_hd, nullptr, out, diag);
    });
}

ccw_status ccw_simulate3d_trace(ccw_ctx* ctx, ccw_ti3d* ti, const ccw_sim3d_config* cfg, const uint64_t* seeds,
                                int n_real, const int32_t* hd, int n_hd, uint8_t* out, ccw_diag3d* diag,
                                int32_t* ti_origins, int capacity) {
    if (!ctx || !ti) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        check_ti3d(ti, cfg, hd, n_hd);
        if (n_real < 1) throw Fail(CCW_ERR_CONFIG, "realizations: must be >= 1");
        if (!ti_origins || capacity < 1) throw Fail(CCW_ERR_GENERIC, "trace: null buffer or zero capacity");
        ccwgpu::run_simulation3d(ctx, ti, *cfg, seeds, n_real, hd, n_hd, nullptr, out, diag, ti_origins, capacity);
    });
}

ccw_status ccw_simulate3d_device(ccw_ctx* ctx, ccw_ti3d* ti, const ccw_sim3d_config* cfg, const uint64_t* seeds,
                                 int n_real, const int32_t* hd, int n_hd, uint8_t* d_out, ccw_diag3d* diag) {
    if (!ctx || !ti) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        check_ti3d(ti, cfg, hd, n_hd);
        if (n_real < 1) throw Fail(CCW_ERR_CONFIG, "realizations: must be >= 1");
        ccwgpu::run_simulation3d(ctx, ti, *cfg, seeds, n_real, hd, n_hd, d_out, nullptr, diag);
    });
}

ccw_status ccw_simulate3d_ensemble(ccw_ctx* ctx, ccw_ti3d* ti, const ccw_sim3d_config* cfg, const int32_t* hd,
                                   int n_hd, uint8_t* out, ccw_diag3d* diag) {
    if (!ctx || !ti) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        check_ti3d(ti, cfg, hd, n_hd);
        std::vector<uint64_t> seeds(static_cast<size_t>(cfg->n_realizations));
        for (int r = 0; r < cfg->n_realizations; ++r) seeds[r] = ccw_mix64(cfg->master_seed, static_cast<uint64_t>(r) + 1);
        ccwgpu::run_simulation3d(ctx, ti, *cfg, seeds.data(), cfg->n_realizations, hd, n_hd, nullptr, out, diag);
    });
}

// ------------------------------------------------------- metrics (f3) --

static void check_grids(const uint8_t* g, int n, int h, int w) {
    if (!g) throw Fail(CCW_ERR_GENERIC, "null grids");
    if (n < 1) throw Fail(CCW_ERR_EMPTY, "ensemble_average on empty ensemble");
    if (h < 1 || w < 1) throw Fail(CCW_ERR_DIMENSION, "grid dimensions must be positive");
}

static void check_lag(int direction, int h, int w, int max_lag) {  // metrics.hpp:70-73
    if (direction != 0 && direction != 1) throw Fail(CCW_ERR_CONFIG, "direction: must be east_west or north_south");
    const int extent = direction == 0 ? w : h;
    if (max_lag < 1 || max_lag >= extent)
        throw Fail(CCW_ERR_DIMENSION, fmt("max_lag must be in [1, extent) = [1, %d)", extent));
}

ccw_status ccw_variogram(ccw_ctx* ctx, const uint8_t* grids, int on_device, int n, int h, int w, int facies,
                         int direction, int max_lag, double* gamma, int32_t* present) {
    if (!ctx || !gamma) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        check_grids(grids, n, h, w);
        check_lag(direction, h, w, max_lag);
        ccwgpu::metric_variogram(ctx, grids, on_device != 0, n, h, w, facies, direction, max_lag, gamma, present);
    });
}

ccw_status ccw_connectivity(ccw_ctx* ctx, const uint8_t* grids, int on_device, int n, int h, int w, int facies,
                            int direction, int max_lag, double* prob) {
    if (!ctx || !prob) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        check_grids(grids, n, h, w);
        check_lag(direction, h, w, max_lag);
        if (static_cast<int64_t>(h) * w >= (int64_t(1) << 31)) throw Fail(CCW_ERR_DIMENSION, "grid too large");
        ccwgpu::metric_connectivity(ctx, grids, on_device != 0, n, h, w, facies, direction, max_lag, prob);
    });
}

ccw_status ccw_ensemble_average(ccw_ctx* ctx, const uint8_t* grids, int on_device, int n, int h, int w, int facies,
                                double* out) {
    if (!ctx || !out) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        if (n < 1) throw Fail(CCW_ERR_EMPTY, "ensemble_average on empty ensemble");
        check_grids(grids, n, h, w);
        ccwgpu::metric_ensemble_average(ctx, grids, on_device != 0, n, h, w, facies, out);
    });
}

ccw_status ccw_downsample_majority(ccw_ctx* ctx, const uint8_t* grid, int on_device, int h, int w, int nf, int factor,
                                   uint8_t* out) {
    if (!ctx || !out) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        check_grids(grid, 1, h, w);
        if (factor < 1) throw Fail(CCW_ERR_DIMENSION, "downsample factor must be >= 1");  // metrics.hpp:290
        if (h / factor < 1 || w / factor < 1)
            throw Fail(CCW_ERR_DIMENSION, fmt("downsample factor %d too large for %dx%d", factor, h, w));
        if (nf < 1 || nf > 256) throw Fail(CCW_ERR_DIMENSION, "num_facies must be in [1, 256]");
        ccwgpu::metric_downsample(ctx, grid, on_device != 0, h, w, nf, factor, out, false);
    });
}

ccw_status ccw_pattern_histogram(ccw_ctx* ctx, const uint8_t* grid, int on_device, int h, int w, int nf, int window,
                                 int stride, ccw_phist** out) {
    if (!ctx || !out) return CCW_ERR_GENERIC;
    *out = nullptr;
    return guarded(ctx, [&] {
        check_grids(grid, 1, h, w);
        if (window < 1 || window > h || window > w)  // metrics.hpp:232-237
            throw Fail(CCW_ERR_DIMENSION, fmt("window %d does not fit %dx%d grid", window, h, w));
        if (stride < 1) throw Fail(CCW_ERR_DIMENSION, "stride must be >= 1");
        if (nf > 256) throw Fail(CCW_ERR_STRUCTURE, "byte pattern keys require num_facies <= 256");
        *out = ccwgpu::metric_pattern_histogram(ctx, grid, on_device != 0, h, w, std::max(nf, 1), window, stride);
    });
}

ccw_status ccw_phist_info(const ccw_phist* hist, int64_t* distinct, int64_t* total, int* window) {
    if (!hist) return CCW_ERR_GENERIC;
    if (distinct) *distinct = hist->n;
    if (total) *total = static_cast<int64_t>(hist->total);
    if (window) *window = hist->window;
    return CCW_OK;
}

ccw_status ccw_phist_copy(ccw_ctx* ctx, const ccw_phist* hist, uint8_t* keys, uint64_t* counts) {
    if (!ctx || !hist) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] { ccwgpu::metric_phist_copy(ctx, hist, keys, counts); });
}

void ccw_phist_destroy(ccw_phist* hist) { ccwgpu::metric_phist_destroy(hist); }

ccw_status ccw_js_divergence(ccw_ctx* ctx, const ccw_phist* p, const ccw_phist* q, double* out) {
    if (!ctx || !p || !q || !out) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        if (p->window != q->window)  // metrics.hpp:259-262
            throw Fail(CCW_ERR_STRUCTURE, fmt("window sizes disagree: %d vs %d", p->window, q->window));
        if (p->total == 0 || q->total == 0) throw Fail(CCW_ERR_EMPTY, "js_divergence on empty histogram");
        *out = ccwgpu::metric_js(ctx, p, q);
    });
}

ccw_status ccw_anodi(ccw_ctx* ctx, const uint8_t* ga, int na, const uint8_t* gb, int nb, int on_device, int h, int w,
                     const uint8_t* ti, int th, int tw, int nf, int levels, int window, const double* weights,
                     double* out, double* aggregate) {
    if (!ctx || !out || !aggregate) return CCW_ERR_GENERIC;
    return guarded(ctx, [&] {
        if (na < 2 || nb < 2) throw Fail(CCW_ERR_EMPTY, "anodi requires at least 2 realizations per ensemble");
        if (levels < 1) throw Fail(CCW_ERR_DIMENSION, "anodi requires levels >= 1");
        if (!ga || !gb || !ti) throw Fail(CCW_ERR_GENERIC, "null grids");
        if (h < 1 || w < 1 || th < 1 || tw < 1) throw Fail(CCW_ERR_DIMENSION, "grid dimensions must be positive");
        if (window < 1) throw Fail(CCW_ERR_DIMENSION, "window must be >= 1");
        if (nf < 1 || nf > 256) throw Fail(CCW_ERR_DIMENSION, "num_facies must be in [1, 256]");
        ccwgpu::metric_anodi(ctx, ga, na, gb, nb, on_device != 0, h, w, ti, th, tw, nf, levels, window, weights, out,
                             aggregate);
    });
}

ccw_status ccw_validate_config(const ccw_sim_config* cfg, int ti_h, int ti_w, int nf,
                               const int32_t* hd, int n_hd, char* msg, size_t msg_len) {
    try {
        if (!cfg) throw Fail(CCW_ERR_GENERIC, "null config");
        if (ti_h <= 0 || ti_w <= 0) {
            ccwgpu::validate_config(*cfg);
        } else {
            ccwgpu::validate_against(*cfg, ti_h, ti_w, nf, hd, n_hd);
        }
        copy_msg(msg, msg_len, "");
        return CCW_OK;
    } catch (const Fail& e) {
        copy_msg(msg, msg_len, e.what());
        g_err = e.what();
        return e.code;
    }
}

ccw_status ccw_plan_raster_path(const ccw_sim_config* cfg, int origin, int column_major,
                                int* work_h, int* work_w, int32_t* tops, int32_t* lefts,
                                int32_t* shapes, int capacity, int* count, char* msg,
                                size_t msg_len) {
    try {
        if (!cfg) throw Fail(CCW_ERR_GENERIC, "null config");
        if (origin < 0 || origin > 3) throw Fail(CCW_ERR_CONFIG, "origin: must be in [0, 4)");
        const ccwgpu::Plan p = ccwgpu::make_plan_from(*cfg, origin, column_major != 0);
        *work_h = p.work_h;
        *work_w = p.work_w;
        *count = static_cast<int>(p.tops.size());
        for (int i = 0; i < *count && i < capacity; ++i) {
            tops[i] = p.tops[i];
            lefts[i] = p.lefts[i];
            shapes[i] = p.shapes[i];
        }
        copy_msg(msg, msg_len, "");
        return CCW_OK;
    } catch (const Fail& e) {
        copy_msg(msg, msg_len, e.what());
        g_err = e.what();
        return e.code;
    }
}

}  // extern "C"
