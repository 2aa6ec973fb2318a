// internal.hpp -- host-side internals of libccwgpu.so (not part of the ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <exception>
#include <functional>
#include <map>
#include <mutex>
#include <thread>
#include <tuple>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/ccwgpu.h"

namespace ccwgpu {

// Internal exception; converted to a ccw_status at the ABI boundary.
struct Fail : std::runtime_error {
    int code;
    Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CCW_CUDA(expr)                                                                     \
    do {                                                                                   \
        cudaError_t e_ = (expr);                                                           \
        if (e_ != cudaSuccess)                                                             \
            throw ::ccwgpu::Fail(CCW_ERR_CUDA, std::string(#expr) + ": " +                 \
                                                   cudaGetErrorString(e_));                \
    } while (0)

// Launch with programmatic stream serialization (PDL): the kernel may start
// while its stream predecessor drains; it must pdl_wait() before reading the
// predecessor's output.
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CCW_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// Grow-only device buffer owned by a context (freed with it).
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void* get(size_t bytes) {
        if (bytes > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            CCW_CUDA(cudaMalloc(&p, bytes));
            cap = bytes;
        }
        return p;
    }
    template <typename T>
    T* as(size_t n) {
        return static_cast<T*>(get(n * sizeof(T) + 16));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

// Pinned host staging buffer (freed with its owner).
struct HostBuf {
    void* p = nullptr;
    size_t cap = 0;
    HostBuf() = default;
    HostBuf(const HostBuf&) = delete;
    HostBuf& operator=(const HostBuf&) = delete;
    ~HostBuf() { release(); }
    void* get(size_t bytes) {
        if (bytes > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = 0;
            CCW_CUDA(cudaMallocHost(&p, bytes));
            cap = bytes;
        }
        return p;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
};

// 64-bit finalizer (splitmix64 style) for content keys.
inline uint64_t mix_key(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Process-wide caching device allocator (exact-size reuse, per device):
// training-image buffers come and go with every ccw_ti; returning them to
// the driver (cudaFree) would unmap memory and stall on every destroy.
void* cache_alloc(int device, size_t bytes);
// device code-range check of an uploaded grid: the first index holding a code >= nf, n if none (ops.cu)
size_t first_bad_code(const uint8_t* d, size_t n, int nf, cudaStream_t st, unsigned long long* d_scratch);
void cache_free(void* p);
// packed cells (1, 2 or 4 bits each, first cell in the low bits) -> bytes (sim.cu)
void unpack_cells(uint8_t* d, const uint8_t* s, size_t n, int bits);

// Persistent host worker pool (one per context): run(n, fn) calls fn(i) for
// every i in [0, n) on the workers and the calling thread, then rethrows the
// first exception.  Keeps thread start-up out of every simulate call.
class HostPool {
public:
    HostPool() = default;
    HostPool(const HostPool&) = delete;
    HostPool& operator=(const HostPool&) = delete;
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : thr_) t.join();
    }
    template <class F>
    void run(int n, F&& fn, int max_threads = 1 << 30) {
        if (n <= 0) return;
        const int want = std::min({n / 2, max_workers(), max_threads - 1});
        if (want <= 0) {
            for (int i = 0; i < n; ++i) fn(i);
            return;
        }
        while (static_cast<int>(thr_.size()) < want) {
            const int idx = static_cast<int>(thr_.size());
            thr_.emplace_back([this, idx, g = gen_] { worker(idx, g); });
        }
        std::function<void(int)> job(std::forward<F>(fn));
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_ = &job;
            n_ = n;
            active_ = want;  // workers [0, want) join; the rest check in and wait
            next_.store(0);
            busy_ = static_cast<int>(thr_.size());
            err_ = nullptr;
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [this] { return busy_ == 0; });
        job_ = nullptr;
        if (err_) std::rethrow_exception(err_);
    }

private:
    static int max_workers() {
        const int hw = static_cast<int>(std::thread::hardware_concurrency());
        return std::max(0, std::min(hw, 16) - 1);
    }
    void work() {
        for (;;) {
            const int i = next_.fetch_add(1);
            if (i >= n_) return;
            try {
                (*job_)(i);
            } catch (...) {
                std::lock_guard<std::mutex> lk(mu_);
                if (!err_) err_ = std::current_exception();
                next_.store(n_);
            }
        }
    }
    void worker(int idx, uint64_t seen) {
        for (;;) {
            bool join = false;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                join = idx < active_;
            }
            if (join) work();
            std::lock_guard<std::mutex> lk(mu_);
            if (--busy_ == 0) done_.notify_all();
        }
    }
    std::vector<std::thread> thr_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    std::function<void(int)>* job_ = nullptr;
    int n_ = 0, busy_ = 0, active_ = 0;
    std::atomic<int> next_{0};
    uint64_t gen_ = 0;
    bool stop_ = false;
    std::exception_ptr err_;
};

// Per-context tuning / test options (ccw_ctx_set_option).  Every default is
// the production setting; tests flip them to force rarely taken paths.
struct Options {
    int groups = 0;            // realization groups on separate streams (0 = auto: 2)
    int sched_replay = 0;      // 1: every unconditional pick takes the sequential replay (tests)
    int norm_screen = 1;       // normalized scoring screened on the int8 GEMM
    int shard_fast = 1;        // position shards may take the fast select
    int uniform = 1;           // uniform-window reduction of large tie groups
    int s16 = 1;               // int16 score rows when every screen score fits
    int bulk = 1;              // bulk (CTA-wide) tie-group rescoring kernel
    int help_min = 32;         // equal-score groups >= this are rescored by helper CTAs (0 = off)
    int stream_out = 1;        // progressive band finalize + copy for host results
    int pack = 1;              // bit-packed streamed bands
    int stream_bands = 6;      // streaming checkpoints per call
    int place_threads = 0;     // host unpack threads (0 = auto)
    int wave = 0;              // fused wave kernel (wave.cu) where it applies (experimental)
    int wave_cs = 0;           // its CTAs per cluster (0 = auto)
    int flagprep = 1;          // OR prep waits on per-placement dependency flags, not the whole select
    int tc3d = 1;              // 3D: tcgen05 int8 screen where the block counts fit int8 (sim3d.cu)
};

// Known option names (for ccw_ctx_set_option); returns nullptr if unknown.
inline int* option_slot(Options& o, const std::string& name) {
    if (name == "groups") return &o.groups;
    if (name == "sched_replay") return &o.sched_replay;
    if (name == "norm_screen") return &o.norm_screen;
    if (name == "shard_fast") return &o.shard_fast;
    if (name == "uniform") return &o.uniform;
    if (name == "s16") return &o.s16;
    if (name == "bulk") return &o.bulk;
    if (name == "help_min") return &o.help_min;
    if (name == "stream_out") return &o.stream_out;
    if (name == "pack") return &o.pack;
    if (name == "stream_bands") return &o.stream_bands;
    if (name == "place_threads") return &o.place_threads;
    if (name == "wave") return &o.wave;
    if (name == "wave_cs") return &o.wave_cs;
    if (name == "flagprep") return &o.flagprep;
    if (name == "tc3d") return &o.tc3d;
    return nullptr;
}

// Diagnostics-only environment switches (timelines, phase clocks): compiled
// in only with -DCCW_DEBUG_KNOBS; a production build never reads them.
inline const char* debug_env(const char* name) {
#ifdef CCW_DEBUG_KNOBS
    return getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}

}  // namespace ccwgpu

struct ccw_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    bool profiling = false;
    int ccf_variant = 0;
    ccwgpu::Options opt;
    ccw_timing timing{};
    // scratch
    ccwgpu::DevBuf wave_w, depflag, chk, cjob, depcnt, defer, bulk_sync, bulk_keys, bulk_idx, hdoff, hdent, jobs, work, hd, wts, wts8, tm64, scores, summary, chosen, pasted, mism, out,
        stats, src, mtab, roff, seeds, lattice, sched_err, sched_outs, sched_replay, jdump, band_off, band_stage, hboards, hpos, hkeys, hdone, tmaxnu, jvar, ops_a, ops_b, ops_c, ops_d, ops_e, tc3_w, tc3_sc, tc3_tm;
    long long mtab_key = -1;  // (Tc, OVc, nch) of the mask tables in mtab
    ccwgpu::HostBuf h_stage;
    ccwgpu::HostBuf h_out_stage;  // pinned landing zone when the caller's result buffer is pageable
    ccwgpu::HostBuf h_upload;     // pinned staging of large host uploads (upload_host, abi.cpp)
    cudaEvent_t upload_done = nullptr;  // the last staged upload's copies
    ccwgpu::HostPool pool;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<cudaStream_t> gstreams;  // realization-group streams
    std::vector<cudaStream_t> copy_streams;  // per group: progressive device->host copies of final bands
    // launch plan memory: (TI content key, Tc, OVc, K, T) whose last call
    // deferred no placement to the bulk tie select skip its per-wave launch
    // (re-enabled when the warp select reports a would-be deferral)
    std::map<std::tuple<uint64_t, int, int, int, int>, bool> bulk_off;
    // ... and whose last call deferred many placements (a tie storm: the
    // screen then also keeps per-tile non-uniform maxima for the bulk kernel)
    std::map<std::tuple<uint64_t, int, int, int, int>, bool> tie_storm;
    // asynchronous device calls (ccw_simulate_device_async): two result slots
    // alternate by call parity; a slot's counters land in pinned memory and are
    // folded into the timing and the plan memory later (ccwgpu::async_settle)
    struct AsyncSlot {
        bool valid = false;
        cudaEvent_t done = nullptr, t0 = nullptr, t1 = nullptr;
        ccwgpu::HostBuf res;  // [kNumStats] stats, then the schedule error flag
        ccw_timing timing{};  // every field but the counters read back
        std::tuple<uint64_t, int, int, int, int> key{};
        bool use_wave = false, bulk_launch = false;
    } aslot[2];
    int async_par = 0;
    std::string async_err;     // the first device-side error an async call reported
    ccwgpu::HostBuf h_stage2;  // second roff staging half (calls alternate)
    cudaEvent_t stage_ev[2] = {nullptr, nullptr};  // the staging half's upload completed
    // candidate-position sharding (ccw_ctx_set_position_shards)
    int shard_nranks = 1, shard_rank = 0, shard_virtual = 1;
    void* nccl_comm = nullptr;  // ncclComm_t when shard_nranks > 1 (or an explicit id was given)
    ccwgpu::DevBuf xrec;        // exchange buffer: [S][jobs][K] shard top-K records
};

struct ccw_ti {
    ccw_ctx* ctx = nullptr;
    int device = 0;
    int h = 0, w = 0, F = 0, J = 0, mode = 0;
    int hc = 0, wc = 0, nch = 0, nscr = 0;
    uint8_t* d_codes = nullptr;  // h*w
    double* d_ti64 = nullptr;    // nch*hc*wc
    float* d_scr = nullptr;      // nscr*hc*wc
    std::map<int, int8_t*> im2col;  // per template size Tc: npos x kpad int8 (tcgen05 screen)
    std::map<std::pair<int, int>, int32_t*> nnmap;  // per (Tc, OVc): normalized-screen norms
    std::map<std::pair<int, int>, int8_t*> umap;    // per (Tc, OVc): uniform-window classes (8 mask variants)
    uint64_t key = 0;  // content key (hash of cells + shape) for per-context plan memory
};

// 3D training image (extension, ccw_ti3d_create): codes and level-J block
// counts (mode 0: int8x4 packed channels, counts <= 64; mode 1: int32 planes).
struct ccw_ti3d {
    ccw_ctx* ctx = nullptr;
    int device = 0;
    int d[3] = {0, 0, 0};  // fine extents
    int c[3] = {0, 0, 0};  // coarse extents (floor(d / 2^J))
    int F = 0, J = 0, nscr = 0, mode = 0;
    uint8_t* d_codes = nullptr;
    int32_t* d_pk = nullptr;
    // im2col of the packed counts for the tcgen05 screen, keyed by the coarse
    // template size (sim3d.cu ti3d_im2col); freed with the TI
    std::map<int, int8_t*> im2col;
};

// On-device pattern histogram (ccw_pattern_histogram): distinct exact window
// keys (codes packed bpc bits each, 128 bits as (hi, lo)) in (hi, lo) order
// with their multiplicities.
struct ccw_phist {
    int device = 0;
    int window = 0, bpc = 0;
    int64_t n = 0;       // distinct keys
    uint64_t total = 0;  // windows
    uint64_t* lo = nullptr;
    uint64_t* hi = nullptr;
    uint64_t* cnt = nullptr;
};

namespace ccwgpu {

// --- host logic shared by the ABI (abi.cpp) ------------------------------
void validate_config(const ccw_sim_config& c);
void validate_against(const ccw_sim_config& c, int ti_h, int ti_w, int nf, const int32_t* hd,
                      int n_hd);

struct Plan {
    int origin = 0;
    bool column_major = false;
    int work_h = 0, work_w = 0;
    int n_outer = 0, n_inner = 0;
    std::vector<int32_t> tops, lefts, shapes, outer_idx, inner_idx;
    bool vertical_on_left() const { return origin == CCW_TOP_LEFT || origin == CCW_BOTTOM_LEFT; }
    bool horizontal_on_top() const { return origin == CCW_TOP_LEFT || origin == CCW_TOP_RIGHT; }
};

// rng.hpp:21-28 (std::mt19937_64's sequence is pinned by the C++ standard).
uint64_t bounded(std::mt19937_64& rng, uint64_t n);
// plan_raster_path (simulator.hpp:148-190): consumes exactly two draws.
Plan make_plan(const ccw_sim_config& c, std::mt19937_64& rng);
Plan make_plan_from(const ccw_sim_config& c, int origin, bool column_major);

// --- NCCL (shard.cpp; libnccl.so.2 loaded on first use) -------------------
void nccl_unique_id(uint8_t* out128);
void* nccl_comm_init(int nranks, int rank, const uint8_t* id128);
void nccl_comm_destroy(void* comm);
void nccl_all_gather_bytes(void* comm, const void* send, void* recv, size_t bytes, cudaStream_t st);

// --- device entry points (sim.cu / ops.cu / peak.cu) ----------------------
double measure_ffma_peak(ccw_ctx* ctx);
double measure_int_peak(ccw_ctx* ctx, int kind);
void build_pyramid(ccw_ti* ti, cudaStream_t s);
void async_settle(ccw_ctx* ctx, bool block);
void run_simulation(ccw_ctx* ctx, ccw_ti* ti, const ccw_sim_config& cfg, const uint64_t* seeds,
                    int n_real, const int32_t* hd, int n_hd, uint8_t* d_out, uint8_t* h_out,
                    ccw_diag* diag, ccw_trace* traces, bool async_call = false);

void build_pyramid3d(ccw_ti3d* ti, cudaStream_t s);
void run_simulation3d(ccw_ctx* ctx, ccw_ti3d* ti, const ccw_sim3d_config& cfg, const uint64_t* seeds, int n_real,
                      const int32_t* hd, int n_hd, uint8_t* d_out, uint8_t* h_out, ccw_diag3d* diag,
                      int32_t* trace = nullptr, int trace_cap = 0);
void validate_config3d(const ccw_sim3d_config& c, const int32_t* ti_dims, int nf, const int32_t* hd, int n_hd);

// metrics.cu (metrics.hpp:68-311 on device)
void metric_variogram(ccw_ctx* ctx, const uint8_t* grids, bool on_device, int n, int h, int w, int facies,
                      int direction, int max_lag, double* gamma, int32_t* present);
void metric_connectivity(ccw_ctx* ctx, const uint8_t* grids, bool on_device, int n, int h, int w, int facies,
                         int direction, int max_lag, double* prob);
void metric_ensemble_average(ccw_ctx* ctx, const uint8_t* grids, bool on_device, int n, int h, int w, int facies,
                             double* out);
void metric_downsample(ccw_ctx* ctx, const uint8_t* grid, bool on_device, int h, int w, int nf, int factor,
                       uint8_t* out, bool out_on_device);
ccw_phist* metric_pattern_histogram(ccw_ctx* ctx, const uint8_t* grid, bool on_device, int h, int w, int nf,
                                    int win, int stride);
double metric_js(ccw_ctx* ctx, const ccw_phist* p, const ccw_phist* q);
void metric_phist_copy(ccw_ctx* ctx, const ccw_phist* h, uint8_t* keys, uint64_t* counts);
void metric_phist_destroy(ccw_phist* h);
void metric_anodi(ccw_ctx* ctx, const uint8_t* ga, int na, const uint8_t* gb, int nb, bool on_device, int h, int w,
                  const uint8_t* ti, int th, int tw, int nf, int levels, int win, const double* weights, double* out,
                  double* aggregate);

void op_dwt2_single(ccw_ctx* ctx, const double* in, int h, int w, double* a, double* dh,
                    double* dv, double* dd);
void op_idwt2_single(ccw_ctx* ctx, const double* a, const double* dh, const double* dv,
                     const double* dd, int hh, int hw, double* out);
void op_dwt2(ccw_ctx* ctx, const double* in, int h, int w, int levels, double* apex,
             double* details);
void op_idwt2(ccw_ctx* ctx, const double* apex, const double* details, int h, int w, int levels,
              double* out);
void op_score_map(ccw_ctx* ctx, const double* ti, const double* tmpl, int nch, int ti_h, int ti_w,
                  int t_h, int t_w, const double* mask, int scoring, double* out);
void op_top_k(ccw_ctx* ctx, const double* scores, int h, int w, int k, int32_t* rows,
              int32_t* cols, double* vals, int* n_out);
void op_select_conditional(ccw_ctx* ctx, const int32_t* rows, const int32_t* cols, int n_cands,
                           const int32_t* hd, int n_hd, const uint8_t* ti, int ti_h, int ti_w,
                           int levels, int* pick, int* mismatches);
void op_min_cut_stitch(ccw_ctx* ctx, const uint8_t* existing, const uint8_t* incoming, int t,
                       int shape, int vleft, int htop, int overlap, uint8_t* out);

}  // namespace ccwgpu
