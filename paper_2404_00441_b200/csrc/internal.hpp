// internal.hpp -- host-side internals of libccwgpu.so (not part of the ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
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

// Grow-only device buffer owned by a context.
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
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

// Pinned host staging buffer.
struct HostBuf {
    void* p = nullptr;
    size_t cap = 0;
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

}  // namespace ccwgpu

struct ccw_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    bool profiling = false;
    int ccf_variant = 0;
    ccw_timing timing{};
    // scratch
    ccwgpu::DevBuf defer, bulk_sync, bulk_keys, bulk_idx, hdoff, hdent, jobs, work, hd, wts, wts8, tm64, scores, summary, chosen, pasted, mism, out,
        stats, src, ops_a, ops_b, ops_c, ops_d, ops_e;
    ccwgpu::HostBuf h_stage;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<cudaStream_t> gstreams;  // realization-group streams
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
    // launch plan memory: geometries whose last call deferred no placement to
    // the bulk tie select skip its per-wave launch (re-enabled on demand)
    std::map<std::tuple<int, int, int, int>, bool> bulk_off;
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

// --- device entry points (sim.cu / ops.cu / peak.cu) ----------------------
double measure_ffma_peak(ccw_ctx* ctx);
void build_pyramid(ccw_ti* ti, cudaStream_t s);
void run_simulation(ccw_ctx* ctx, ccw_ti* ti, const ccw_sim_config& cfg, const uint64_t* seeds,
                    int n_real, const int32_t* hd, int n_hd, uint8_t* d_out, uint8_t* h_out,
                    ccw_diag* diag, ccw_trace* traces);

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
