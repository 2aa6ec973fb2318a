// sim_kernels.cuh -- the simulation path's shared device building blocks,
// sizes and kernel declarations (prep.cu, ccf_direct.cu, select.cu, sim.cu).
#pragma once

#include <climits>
#include <cstdint>

#include "ccf_tc.hpp"
#include "ccw_device.cuh"
#include "internal.hpp"

namespace ccwgpu {

// ------------------------------------------------------------ or_prep ----

// Normalized screen: C_job = B^2 * sum over the mask of the OR's last-facies
// block count, so the screen S' (F-1 channels) plus C_job is the full
// count score S (indicator mode; 0 in raw-codes mode).
__device__ __forceinline__ void store_cjob(int32_t* cjob, int mode, int B, int slot, int csum) {
    __shared__ int red[32];
    for (int o = 16; o > 0; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
    __syncthreads();  // (red may be in use by an earlier call)
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = csum;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
        cjob[slot] = mode == 0 ? B * B * t : 0;
    }
}

// Screen weights: indicator mode uses F-1 channels with w_f = n_f - n_{F-1}
// (n = OR block counts).  Because every fine cell holds exactly one facies,
//   S = sum_f sum_mask N_f * n_f = sum_{f<F-1} sum_mask N_f * w_f + B * sum_mask n_{F-1}
// and the last term is the same for every TI window, so ranking by the F-1
// channel sum is ranking by S.  Raw-codes mode uses the code sums directly.
// Fast path (no min-cut): every work block is a verbatim block-aligned TI
// block (pastes are block aligned, simulator.hpp:452-453, 480-483), so the OR's
// counts and reference-order apex values are gathers from the TI pyramid at
// the recorded source block -- identical values, no recomputation.
// One placement's OR preparation from the source-block map (every thread of
// the calling CTA takes part; the CTA size is free).  Outputs go to the given
// per-slot bases: the int8 screen weights (w8base, or the int32 weights of the
// fp32 screen when w8base is null), the fp64 template and C_job.
__device__ __forceinline__ void prep_src_job(const SimParams& P, const Job& jb, int slot, int8_t* w8base,
                                             double* tmbase, int32_t* cjobbase) {
    const int Tc = P.Tc, B = P.B, nc = P.hc * P.wc;
    const int J = P.J;  // (B = 2^J: block coordinates by shifts)
    const int32_t* src = P.src + static_cast<size_t>(jb.real) * (P.wh >> J) * P.swc +
                         static_cast<size_t>(jb.top >> J) * P.swc + (jb.left >> J);
    const bool tc_pow2 = (Tc & (Tc - 1)) == 0;
    const int tc_log = __ffs(Tc) - 1;
    int32_t* wts = w8base ? nullptr : P.wts + static_cast<size_t>(slot) * P.nscr * Tc * Tc;
    double* tm = tmbase ? tmbase + static_cast<size_t>(slot) * P.nch * Tc * Tc : nullptr;
    int8_t* w8 = w8base ? w8base + static_cast<size_t>(slot) * P.kpad : nullptr;
    if (w8)
        for (int k = P.nscr * Tc * Tc + threadIdx.x; k < P.kpad; k += blockDim.x) w8[k] = 0;
    int csum = 0;
    constexpr int kCh = 8, kCpt = 2;  // batched path: <= 8 channels, 2 cells per thread
    if (P.nch <= kCh && P.nscr <= kCh) {
        // every load of a thread's cells in flight at once: the map entries, then
        // the screen planes and apex values at the source blocks
        for (int c0 = threadIdx.x; c0 < Tc * Tc; c0 += kCpt * blockDim.x) {
            int sb[kCpt];
            bool in[kCpt];
#pragma unroll
            for (int u = 0; u < kCpt; ++u) {
                const int c = c0 + u * blockDim.x;
                const int s = tc_pow2 ? c >> tc_log : c / Tc, t = c - s * Tc;
                int t0 = 0, t1 = 0;
                if (c < Tc * Tc) mask_row_run(jb.shape, jb.vleft, jb.htop, Tc, P.OVc, s, t0, t1);
                in[u] = c < Tc * Tc && t >= t0 && t < t1;
                sb[u] = in[u] ? src[static_cast<size_t>(s) * P.swc + t] : 0;
            }
            float n[kCpt][kCh];
            double a[kCpt][kCh];
#pragma unroll
            for (int u = 0; u < kCpt; ++u)
#pragma unroll
                for (int f = 0; f < kCh; ++f) {
                    n[u][f] = f < P.nscr ? P.tiscr[static_cast<size_t>(f) * nc + sb[u]] : 0.f;
                    a[u][f] = f < P.nch && in[u] ? P.ti64[static_cast<size_t>(f) * nc + sb[u]] : 0.0;
                }
#pragma unroll
            for (int u = 0; u < kCpt; ++u) {
                const int c = c0 + u * blockDim.x;
                if (c >= Tc * Tc) continue;
                int last = B * B;
                if (P.mode == 0)
#pragma unroll
                    for (int f = 0; f < kCh; ++f)
                        if (f < P.nscr) last -= static_cast<int>(n[u][f]);
                if (in[u]) csum += last;
#pragma unroll
                for (int f = 0; f < kCh; ++f) {
                    if (f >= P.nscr) break;
                    const int v = in[u] ? (P.mode == 0 ? static_cast<int>(n[u][f]) - last : static_cast<int>(n[u][f])) : 0;
                    if (w8)
                        w8[f * Tc * Tc + c] = static_cast<int8_t>(v);
                    else
                        wts[f * Tc * Tc + c] = v;
                }
                if (tm)
#pragma unroll
                    for (int ch = 0; ch < kCh; ++ch)
                        if (ch < P.nch) tm[ch * Tc * Tc + c] = a[u][ch];
            }
        }
        if (cjobbase) store_cjob(cjobbase, P.mode, P.B, slot, csum);
        return;
    }
    for (int c = threadIdx.x; c < Tc * Tc; c += blockDim.x) {
        const int s = tc_pow2 ? c >> tc_log : c / Tc, t = c - s * Tc;
        int t0, t1;
        mask_row_run(jb.shape, jb.vleft, jb.htop, Tc, P.OVc, s, t0, t1);
        const bool in = t >= t0 && t < t1;
        const int sb = in ? src[static_cast<size_t>(s) * P.swc + t] : 0;
        int last = B * B;
        if (P.mode == 0)
            for (int f = 0; f < P.nscr; ++f) last -= static_cast<int>(P.tiscr[static_cast<size_t>(f) * nc + sb]);
        if (in) csum += last;
        for (int f = 0; f < P.nscr; ++f) {
            const int n = static_cast<int>(P.tiscr[static_cast<size_t>(f) * nc + sb]);
            const int v = in ? (P.mode == 0 ? n - last : n) : 0;
            if (w8)
                w8[f * Tc * Tc + c] = static_cast<int8_t>(v);
            else
                wts[f * Tc * Tc + c] = v;
        }
        for (int ch = 0; ch < P.nch; ++ch)
            tm[ch * Tc * Tc + c] = in ? P.ti64[static_cast<size_t>(ch) * nc + sb] : 0.0;
    }
    if (cjobbase) store_cjob(cjobbase, P.mode, P.B, slot, csum);
}

// --------------------------------------------------------- CCF screen ----

constexpr int CCF_TX = 16;  // output rows per CTA
constexpr int CCF_TY = 64;  // output columns per CTA
constexpr int CCF_RY = 8;   // consecutive outputs per thread
constexpr int CCF_THREADS = CCF_TX * CCF_TY / CCF_RY;

__host__ __device__ constexpr int ccf_sw(int Tc) { return ((CCF_TY + Tc + 4) + 3) & ~3; }
__host__ __device__ constexpr int ccf_wp(int Tc) { return (Tc + 3) & ~3; }


// ------------------------------------------------------- select+paste ----

constexpr int SEL_T = 256;
constexpr int GCAP = 1024;
constexpr int KMAX = 8192;
constexpr int RSUM_CAP = 4096;  // (window, run) partial sums staged per rescoring group

struct SelLayout {
    size_t hist, misc, redd, redi, gkey, gidx, tkey, tidx, runs, tmpl, rsum, rnrm, exist, outp,
        from, dp, seam, total;
};

__host__ __device__ inline SelLayout sel_layout(int K, int T, int OV, int nch = 1, int Tc = 1,
                                                int normalized = 0) {
    SelLayout L{};
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o = (o + bytes + 15) & ~static_cast<size_t>(15);
        return at;
    };
    L.hist = take(256 * 4);
    L.misc = take(16 * 4);
    L.redd = take(32 * 8);
    L.redi = take(64 * 4);
    L.gkey = take(static_cast<size_t>(GCAP + SEL_T + K) * 8);
    L.gidx = take(static_cast<size_t>(GCAP + SEL_T + K) * 4);
    L.tkey = take(static_cast<size_t>(K) * 8);
    L.tidx = take(static_cast<size_t>(K) * 4);
    L.runs = take(static_cast<size_t>(nch) * Tc * 16);
    L.tmpl = take(static_cast<size_t>(nch) * Tc * Tc * 8);
    L.rsum = take(static_cast<size_t>(RSUM_CAP) * 8);
    L.rnrm = take(normalized ? static_cast<size_t>(RSUM_CAP) * 8 : 0);
    L.exist = take(static_cast<size_t>(T) * T);
    L.outp = take(static_cast<size_t>(T) * T);
    L.from = take(static_cast<size_t>(T) * OV * 2);
    L.dp = take(static_cast<size_t>(2) * OV * 4);
    L.seam = take(static_cast<size_t>(T) * 4);
    L.total = o;
    return L;
}

// Normalized screen.  Mask variant of a placement:
// L (vleft, htop) 0-3, vertical strip 4 + vleft, horizontal strip 6 + htop.
__host__ __device__ inline int mask_variant(int shape, int vleft, int htop) {
    return shape == kL ? (vleft ? 2 : 0) + (htop ? 1 : 0)
                       : (shape == kVertical ? 4 + (vleft ? 1 : 0) : 6 + (htop ? 1 : 0));
}

// ------------------------------------------------------------ fast select --
//
// The common case (raw scoring, K <= kTcQ, tcgen05 screen, no min-cut): the
// tile-maximum bound M_K, the (score, position) list of windows >= M_K, the
// exact K-th score S_K, fp64 rescoring of the candidates, ranking, pick --
// select_fast_kernel below; placements whose list overflows go to
// select_bulk_kernel.
constexpr int SC_LC = 256;     // list / candidate capacity per placement
constexpr int SC_TB = 8;       // qualifying tiles read per round trip
#ifndef CCW_PK_TMC
#define CCW_PK_TMC 1024
#endif
constexpr int PK_TMC = CCW_PK_TMC;   // fp64 template values staged in shared memory (when they fit)
constexpr int PK_MAXTC = 64;   // template rows tabulated

// ---------------------------------------------------- fused fast select --
//
// One 128-thread CTA per placement: warp 0 scans (scan_job) while warps 1-3
// stage the fp64 template, the mask rows and the rescoring work items; then
// every (candidate, run group) item is rescored by one thread -- a run group
// is up to FS_G cells of consecutive mask rows of one channel with the same
// column run, whose operands are loaded in one round trip and whose run sums
// are formed left to right (matcher.hpp:72-76); per-window folds in
// row-major run order (matcher.hpp:77, 160-161); reference ranking; pick;
// source-block map.
constexpr int FS_T = 128;
constexpr int FS_G = 16;       // cells per rescoring item
#ifndef CCW_FS_MAXG
#define CCW_FS_MAXG 512
#endif
constexpr int FS_MAXG = CCW_FS_MAXG;   // run groups per placement
// Per mask variant (mask_variant), built once on the host: int4 (rows, groups,
// any run longer than FS_G, 0), the mask rows (short4 (s, t0, t1, 0), two per
// int4) and the rescoring run groups (see select_fast_kernel).
constexpr int MT_ROWS4 = PK_MAXTC / 2;
constexpr int MT_STRIDE = 1 + MT_ROWS4 + FS_MAXG;
#ifndef CCW_FS_RS
#define CCW_FS_RS 1536
#endif
constexpr int FS_RS = CCW_FS_RS;    // (window, run) partial sums per batch

// ------------------------------------------------------- bulk tie select --
//
// Placements whose exact-screen tie group is large (a binary TI with K = 1
// can tie thousands of windows at the maximum) are deferred here by the warp
// select.  S CTAs serve each deferred placement: they take position blocks of
// bulk_bx x bulk_by windows from a per-placement counter; a block holding a
// window at or above the threshold stages the TI apex tile it reads into
// shared memory (cp.async) and every thread rescores whole windows in the
// reference's operation order (matcher.hpp:72-77, 160-161), BK_W independent
// windows interleaved to hide the dependent fp64 chain.  Each CTA publishes
// its top-K; the last CTA to finish merges them by the reference ranking
// (matcher.hpp:189-198), chooses and pastes like the warp select.
#ifndef CCW_BK_T
#define CCW_BK_T 256
#endif
#ifndef CCW_BK_W
#define CCW_BK_W 4
#endif
constexpr int BK_T = CCW_BK_T;
constexpr int BK_W = CCW_BK_W;
constexpr int BK_V = 16;     // positions per thread per scan pass
constexpr int BK_SMAX = 32;  // CTAs per placement (upper bound)
constexpr int BK_STAGE_MIN = 512;  // windows of a block worth staging its apex tile for

struct BulkLayout {
    size_t stage, tm, rows, cand, ukey, misc, total;
    int sh, sw;
};

__host__ __device__ inline BulkLayout bulk_layout(int nch, int Tc, int bx, int by) {
    BulkLayout L{};
    L.sh = bx + Tc - 1;
    L.sw = (by + Tc - 1) | 1;  // odd row stride spreads rows over the banks
    size_t o = 0;
    L.stage = o;
    o += static_cast<size_t>(nch) * L.sh * L.sw * sizeof(double);
    // the per-thread top-K lists reuse the stage area at the end
    o = std::max(o, static_cast<size_t>(BK_T) * kTcQ * (sizeof(double) + sizeof(int)));
    L.tm = o;
    o += static_cast<size_t>(nch) * Tc * Tc * sizeof(double);
    L.rows = o;
    o += static_cast<size_t>(Tc) * sizeof(short4);
    L.cand = o;
    o += (static_cast<size_t>(bx) * by + BK_T) * sizeof(int);
    o = (o + 15) & ~static_cast<size_t>(15);
    L.ukey = o;   // fp64 key of each uniform class for this placement
    o += 16 * sizeof(double);
    L.misc = o;
    o += 320 + static_cast<size_t>(BK_SMAX) * kTcQ * (sizeof(double) + sizeof(int));
    L.total = o;
    return L;
}

// ------------------------------------------------------------ wave ----
//
// The fused wave kernel (wave.cu): OR prep, implicit-im2col tcgen05 screen,
// exact top-K' in the epilogue, fp64 tie ranking, pick and paste in one
// launch per wave (source-block-map path, raw scoring, K <= 16, Tc <= 16).
struct WaveArgs {
    const int8_t* strips;  // ti_strips: [out_w][nmb][nscr][144][16] int8
    int nmb;               // position blocks per column
    int nb;                // positions per block (a multiple of 16, <= 128)
    int8_t* wglob;         // per set: the A operand (screen weights) staged in global memory
    int dbg;               // debug builds only (CCW_WAVE_DBG): 1 no prep loads, 2 no list work, 4 no MMA
};
bool wave_supported(int nscr, int Tc, int nch, int K, int T, int OV);
const int8_t* ti_strips(ccw_ti* ti, int Tc, cudaStream_t st, int* nmb_out, int* nb_out);
int wave_pick_cs(const SimParams& P, int nj, int want);
int wave_jobs_per_set();
void wave_prepare(const SimParams& P);
void launch_wave(const SimParams& P, const Job* jobs, int job0, int nj, const int8_t* strips, int nmb, int nb, int cs,
                 int8_t* wglob, cudaStream_t st);
size_t wave_wglob_bytes(const SimParams& P, int nj);

// ---------------------------------------------------------- kernels -----

// prep.cu
// Device schedule (schedule.cu): one thread per realization replays its
// mt19937_64 draws and writes its jobs at their wave-ordered slots.
enum { kTopLeft = 0, kTopRight = 1, kBottomLeft = 2, kBottomRight = 3 };  // simulator.hpp:97-104
struct SchedParams {
    const uint64_t* seeds;
    const int32_t* vid;        // host's path variant per realization (origin * 2 + column-major), checked
    const int32_t* roff;       // [n_real][nkeys] first flat slot of each realization in each wave
    const uint8_t* lattice_hd; // stride-lattice cells holding hard data (null: none)
    int* err;                  // set when the device draws disagree with vid
    uint64_t* outs;            // [n_real][nout] tempered generator outputs (scratch)
    uint64_t* replay;          // [n_real][313] generator state for the sequential replay (scratch)
    int n_real, nkeys, keymul, nout;
    int nlr, nlc, stride, B, Kp;
    uint64_t nfr, nfc;         // first placement: block-aligned TI origins per axis
    uint64_t thr_fr, thr_fc, thr_k;  // bounded() rejection thresholds (2^64 - n) mod n
};
__global__ void build_jobs_kernel(SchedParams S, Job* __restrict__ jobs);

__global__ void or_prep_src_kernel(SimParams P, const Job* __restrict__ jobs, int job0);
__global__ void or_prep_kernel(SimParams P, const Job* __restrict__ jobs, int job0);
const int32_t* ti_nnmap(ccw_ti* ti, int Tc, int OVc, cudaStream_t st);
const int8_t* ti_umap(ccw_ti* ti, int Tc, int OVc, cudaStream_t st);
int umap_stride(int npos);
const double* ti_pure_apex(ccw_ti* ti, int Tc, int OVc, cudaStream_t st);
const int* ti_uniform_first(ccw_ti* ti, int Tc, int OVc, cudaStream_t st);
const uint32_t* ti_uniform_bits(ccw_ti* ti, int Tc, int OVc, cudaStream_t st);
void fill_i32(int32_t* p, size_t n, int32_t v, cudaStream_t st);
// ccf_direct.cu
size_t ccf_smem_bytes(int Tc, int nscr);
__global__ void ccf_direct_kernel(SimParams P, const Job* __restrict__ jobs, int job0);
// select.cu
__global__ void select_paste_kernel(SimParams P, const Job* __restrict__ jobs, int job0, int use_screen);
__global__ void shard_merge_kernel(SimParams P, const Job* __restrict__ jobs, int job0, int nshards);
template <bool S16>
__global__ void select_fast_kernel(const __grid_constant__ SimParams P, const Job* __restrict__ jobs, int job0, int nj);
__global__ void select_bulk_kernel(SimParams P, const Job* __restrict__ jobs, int job0, int nj, int S);

}  // namespace ccwgpu
