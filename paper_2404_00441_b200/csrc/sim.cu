// sim.cu -- the batched, wavefront-scheduled CCWSIM simulation on sm_100a.
//
// One ccw_simulate call runs every realization in lock-step.  Placements of
// all realizations are grouped into waves by the key (d+1)*o + i of their
// raster coordinates (o outer, i inner; d = how many stride steps a footprint
// reaches), which orders every pair of overlapping footprints exactly as the
// reference's raster loop does (simulator.hpp:447-496) while letting the
// placements of one wave run concurrently.  Per wave:
//
//   or_prep        overlap region -> exact-integer screen weights and the
//                  reference-order fp64 OR apex (simulator.hpp:455-460)
//   ccf_direct     exact-integer CCF screen over every TI window, fp32 FFMA
//                  on CUDA cores (matcher.hpp:64-81 up to a per-job constant)
//   select_paste   exact K-th-largest threshold, fp64 reference-order
//                  rescoring of the tie group, top-K ordering
//                  (matcher.hpp:177-204), unconditional / conditional pick
//                  (matcher.hpp:207-241), optional min-cut stitch
//                  (simulator.hpp:286-374) and the paste (simulator.hpp:483-493)
//
// and once per call a finalize kernel applies the hard-data overwrite and
// crops the work grid (simulator.hpp:506-515).
#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <exception>
#include <mutex>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <climits>
#include <cstring>

#include "ccf_tc.hpp"
#include "ccw_device.cuh"
#include "internal.hpp"

namespace ccwgpu {

// ------------------------------------------------------------ pyramid ----

// TI pyramid, once per TI: reference-order apex per channel (wavelet.hpp:147-171
// applied to to_indicator_planes / to_real_plane, simulator.hpp:429-435) and the
// exact-integer screen planes (block counts of facies 0..F-2, or code sums).
__global__ void pyramid_kernel(const uint8_t* __restrict__ codes, int w, int hc, int wc, int J,
                               int mode, int nscr, double* __restrict__ ti64,
                               float* __restrict__ scr) {
    const int cell = blockIdx.x * blockDim.x + threadIdx.x;
    const int ch = blockIdx.y;
    if (cell >= hc * wc) return;
    const int i = cell / wc, j = cell - i * wc;
    const int B = 1 << J;
    const uint8_t* base = codes + static_cast<size_t>(i * B) * w + j * B;
    ti64[static_cast<size_t>(ch) * hc * wc + cell] = haar_apex_block(base, w, J, mode, ch);
    if (ch < nscr)
        scr[static_cast<size_t>(ch) * hc * wc + cell] = static_cast<float>(block_stat(base, w, B, mode, ch));
}

void build_pyramid(ccw_ti* ti, cudaStream_t s) {
    const int n = ti->hc * ti->wc;
    dim3 grid((n + 127) / 128, ti->nch);
    pyramid_kernel<<<grid, 128, 0, s>>>(ti->d_codes, ti->w, ti->hc, ti->wc, ti->J, ti->mode,
                                        ti->nscr, ti->d_ti64, ti->d_scr);
    CCW_CUDA(cudaGetLastError());
}

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
    const int32_t* src = P.src + static_cast<size_t>(jb.real) * (P.wh / B) * P.swc;
    int32_t* wts = w8base ? nullptr : P.wts + static_cast<size_t>(slot) * P.nscr * Tc * Tc;
    double* tm = tmbase + static_cast<size_t>(slot) * P.nch * Tc * Tc;
    int8_t* w8 = w8base ? w8base + static_cast<size_t>(slot) * P.kpad : nullptr;
    if (w8)
        for (int k = P.nscr * Tc * Tc + threadIdx.x; k < P.kpad; k += blockDim.x) w8[k] = 0;
    int csum = 0;
    for (int c = threadIdx.x; c < Tc * Tc; c += blockDim.x) {
        const int s = c / Tc, t = c - s * Tc;
        int t0, t1;
        mask_row_run(jb.shape, jb.vleft, jb.htop, Tc, P.OVc, s, t0, t1);
        const bool in = t >= t0 && t < t1;
        const int sb = in ? src[static_cast<size_t>(jb.top / B + s) * P.swc + jb.left / B + t] : 0;
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

__global__ void or_prep_src_kernel(SimParams P, const Job* __restrict__ jobs, int job0) {
    pdl_trigger();
    const int slot = blockIdx.x;
    const Job jb = jobs[job0 + slot];
    tl_mark(P.tl, 2);
    pdl_wait();
    tl_mark(P.tl, 0);
    prep_src_job(P, jb, slot, P.wts8, P.tm64, P.cjob);
    tl_mark(P.tl, 1);
}

__global__ void or_prep_kernel(SimParams P, const Job* __restrict__ jobs, int job0) {
    pdl_trigger();
    const int slot = blockIdx.x;
    const Job jb = jobs[job0 + slot];
    pdl_wait();
    const int Tc = P.Tc, B = P.B;
    const uint8_t* grid = P.work + static_cast<size_t>(jb.real) * P.wh * P.ww;
    int32_t* wts = P.wts + static_cast<size_t>(slot) * P.nscr * Tc * Tc;
    double* tm = P.tm64 + static_cast<size_t>(slot) * P.nch * Tc * Tc;
    if (P.wts8)  // zero the K padding of this job's int8 weight row
        for (int k = P.nscr * Tc * Tc + threadIdx.x; k < P.kpad; k += blockDim.x)
            P.wts8[static_cast<size_t>(slot) * P.kpad + k] = 0;
    int csum = 0;
    for (int c = threadIdx.x; c < Tc * Tc; c += blockDim.x) {
        const int s = c / Tc, t = c - s * Tc;
        int t0, t1;
        mask_row_run(jb.shape, jb.vleft, jb.htop, Tc, P.OVc, s, t0, t1);
        const bool in = t >= t0 && t < t1;
        const uint8_t* base = grid + static_cast<size_t>(jb.top + s * B) * P.ww + jb.left + t * B;
        int8_t* w8 = P.wts8 ? P.wts8 + static_cast<size_t>(slot) * P.kpad : nullptr;
        if (P.mode == 0) {
            const int last = in ? block_stat(base, P.ww, B, 0, P.F - 1) : 0;
            csum += last;
            for (int f = 0; f < P.nscr; ++f) {
                const int v = in ? block_stat(base, P.ww, B, 0, f) - last : 0;
                wts[f * Tc * Tc + c] = v;
                if (w8) w8[f * Tc * Tc + c] = static_cast<int8_t>(v);
            }
        } else {
            const int v = in ? block_stat(base, P.ww, B, 1, 0) : 0;
            wts[c] = v;
            if (w8) w8[c] = static_cast<int8_t>(v);
        }
        for (int ch = 0; ch < P.nch; ++ch)
            tm[ch * Tc * Tc + c] = in ? haar_apex_block(base, P.ww, P.J, P.mode, ch) : 0.0;
    }
    if (P.cjob) store_cjob(P.cjob, P.mode, P.B, slot, csum);
}

// --------------------------------------------------------- CCF screen ----

constexpr int CCF_TX = 16;  // output rows per CTA
constexpr int CCF_TY = 64;  // output columns per CTA
constexpr int CCF_RY = 8;   // consecutive outputs per thread
constexpr int CCF_THREADS = CCF_TX * CCF_TY / CCF_RY;

struct Rect {
    int s0, t0, h, w;
};

// The strip / L overlap masks are the union of at most two disjoint
// rectangles: the horizontal strip (full width) and the rest of the vertical
// strip.  (Any summation order is exact for the integer screen.)
__device__ __forceinline__ int mask_rects(const Job& jb, int Tc, int OVc, Rect* r) {
    const bool vert = jb.shape == kVertical || jb.shape == kL;
    const bool horz = jb.shape == kHorizontal || jb.shape == kL;
    int n = 0;
    if (horz) r[n++] = {jb.htop ? 0 : Tc - OVc, 0, OVc, Tc};
    if (vert) {
        const int c0 = jb.vleft ? 0 : Tc - OVc;
        if (horz)
            r[n++] = {jb.htop ? OVc : 0, c0, Tc - OVc, OVc};
        else
            r[n++] = {0, c0, Tc, OVc};
    }
    return n;
}

__host__ __device__ constexpr int ccf_sw(int Tc) { return ((CCF_TY + Tc + 4) + 3) & ~3; }
__host__ __device__ constexpr int ccf_wp(int Tc) { return (Tc + 3) & ~3; }

size_t ccf_smem_bytes(int Tc, int nscr) {
    const int SH = CCF_TX + Tc - 1, SW = ccf_sw(Tc), WP = ccf_wp(Tc);
    return sizeof(float) * (static_cast<size_t>(nscr) * SH * SW + static_cast<size_t>(nscr) * 2 * Tc * WP);
}

// Direct correlation of the job's integer weights with the TI screen planes,
// fp32 on CUDA cores.  Every operand is a small integer and every partial sum
// is bounded by mask * B^2 < 2^24 (checked on the host), so FFMA is exact.
// Tiling: one CTA = 16 x 64 outputs of one job; thread = 1 x 8 outputs with a
// sliding 11-register TI window per 4-wide weight chunk.
__global__ void __launch_bounds__(CCF_THREADS) ccf_direct_kernel(SimParams P,
                                                                 const Job* __restrict__ jobs,
                                                                 int job0) {
    extern __shared__ __align__(16) float ccf_sm[];
    pdl_trigger();
    const int slot = blockIdx.z;
    const Job jb = jobs[job0 + slot];
    pdl_wait();
    const int Tc = P.Tc, hc = P.hc, wc = P.wc, nscr = P.nscr;
    const int SH = CCF_TX + Tc - 1, SW = ccf_sw(Tc), WP = ccf_wp(Tc);
    float* tile = ccf_sm;
    float* wpk = ccf_sm + nscr * SH * SW;
    Rect rc[2];
    const int nr = mask_rects(jb, Tc, P.OVc, rc);
    const int x0 = blockIdx.y * CCF_TX, y0 = blockIdx.x * CCF_TY;

    const int tn = nscr * SH * SW;
    for (int e = threadIdx.x; e < tn; e += CCF_THREADS) {
        const int f = e / (SH * SW);
        const int rem = e - f * SH * SW;
        const int r = rem / SW, c = rem - r * SW;
        const int gx = x0 + r, gy = y0 + c;
        tile[e] = (gx < hc && gy < wc) ? P.tiscr[static_cast<size_t>(f) * hc * wc + gx * wc + gy] : 0.f;
    }
    const int32_t* wg = P.wts + static_cast<size_t>(slot) * nscr * Tc * Tc;
    const int wn = nscr * 2 * Tc * WP;
    for (int e = threadIdx.x; e < wn; e += CCF_THREADS) {
        const int f = e / (2 * Tc * WP);
        const int k = (e / (Tc * WP)) & 1;
        const int i = (e / WP) % Tc;
        const int j = e % WP;
        float v = 0.f;
        if (k < nr && i < rc[k].h && j < rc[k].w)
            v = static_cast<float>(wg[f * Tc * Tc + (rc[k].s0 + i) * Tc + rc[k].t0 + j]);
        wpk[e] = v;
    }
    __syncthreads();

    const int tr = threadIdx.x >> 3, tcg = (threadIdx.x & 7) * CCF_RY;
    float acc[CCF_RY];
#pragma unroll
    for (int b = 0; b < CCF_RY; ++b) acc[b] = 0.f;
    for (int f = 0; f < nscr; ++f) {
        for (int k = 0; k < nr; ++k) {
            const Rect R = rc[k];
            const float* tb = tile + f * SH * SW + (tr + R.s0) * SW + tcg + R.t0;
            const float* wb = wpk + (f * 2 + k) * Tc * WP;
            for (int i = 0; i < R.h; ++i) {
                const float* trow = tb + i * SW;
                const float* wrow = wb + i * WP;
                for (int j = 0; j < R.w; j += 4) {
                    const float4 w4 = *reinterpret_cast<const float4*>(wrow + j);
                    float v[CCF_RY + 3];
#pragma unroll
                    for (int q = 0; q < CCF_RY + 3; ++q) v[q] = trow[j + q];
#pragma unroll
                    for (int b = 0; b < CCF_RY; ++b) {
                        acc[b] = fmaf(v[b], w4.x, acc[b]);
                        acc[b] = fmaf(v[b + 1], w4.y, acc[b]);
                        acc[b] = fmaf(v[b + 2], w4.z, acc[b]);
                        acc[b] = fmaf(v[b + 3], w4.w, acc[b]);
                    }
                }
            }
        }
    }
    const int x = x0 + tr;
    if (x < P.out_h) {
        int32_t* out = P.scores + static_cast<size_t>(slot) * P.sld + static_cast<size_t>(x) * P.out_w;
#pragma unroll
        for (int b = 0; b < CCF_RY; ++b) {
            const int y = y0 + tcg + b;
            if (y < P.out_w) out[y] = __float2int_rn(acc[b]);
        }
    }
}

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

// Exact K-th largest value (with multiplicity) of n int32 values, skipping
// INT_MIN padding: block-wide radix select over the offset range, 8 bits per
// pass, warp-aggregated shared-memory histograms.
// (No __restrict__: the normalized screen rewrites its input in the same kernel.)
__device__ int radix_kth_largest(const int32_t* sc, int n, int K, int* hist,
                                 int* misc, int* redi, int stride = 1) {
    int lo = INT_MAX, hi = INT_MIN;
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
        const int v = sc[static_cast<size_t>(p) * stride];
        if (v == INT_MIN) continue;
        lo = min(lo, v);
        hi = max(hi, v);
    }
    lo = block_reduce(lo, [](int a, int b) { return min(a, b); }, redi);
    hi = block_reduce(hi, [](int a, int b) { return max(a, b); }, redi);
    const uint32_t range = static_cast<uint32_t>(hi) - static_cast<uint32_t>(lo);
    if (range == 0) return lo;
    const int nbits = 32 - __clz(range);
    const int passes = (nbits + 7) / 8;
    uint32_t prefix = 0;
    int krem = K;
    for (int ps = passes - 1; ps >= 0; --ps) {
        const int shift = ps * 8;
        for (int e = threadIdx.x; e < 256; e += blockDim.x) hist[e] = 0;
        __syncthreads();
        for (int base = 0; base < n; base += blockDim.x) {
            const int p = base + threadIdx.x;
            bool match = false;
            int dg = 0;
            if (p < n && sc[static_cast<size_t>(p) * stride] != INT_MIN) {
                const uint32_t u = static_cast<uint32_t>(sc[static_cast<size_t>(p) * stride]) - static_cast<uint32_t>(lo);
                match = (static_cast<uint64_t>(u) >> (shift + 8)) ==
                        (static_cast<uint64_t>(prefix) >> (shift + 8));
                dg = (u >> shift) & 255;
            }
            const unsigned mm = __ballot_sync(0xffffffffu, match);
            if (match) {
                const unsigned grp = __match_any_sync(mm, dg);
                if ((threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&hist[dg], __popc(grp));
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int cum = 0, d = 255;
            for (; d > 0; --d) {
                if (cum + hist[d] >= krem) break;
                cum += hist[d];
            }
            misc[0] = d;
            misc[1] = krem - cum;
        }
        __syncthreads();
        prefix |= static_cast<uint32_t>(misc[0]) << shift;
        krem = misc[1];
        __syncthreads();
    }
    return static_cast<int>(static_cast<uint32_t>(lo) + prefix);
}

struct RunDesc {
    int ch, s, t0, t1;
};

// fp64 rescoring of `cnt` windows in the reference's exact order
//   acc = 0; for f: for run (row-major): sum = 0; sum += ti*or over the run;
//   acc += sum          (matcher.hpp:64-81, 158-161)
// plus, for normalized scoring, the masked squares and acc / sqrt(norm)
// (matcher.hpp:84-100, 163-171).  Parallel over (window, run) pairs: each
// thread forms one run's sum (the reference's inner chain), then one thread
// per window folds the run sums in order -- the same operations in the same
// order as the reference, so the result is bit-identical.
__device__ void rescore_group(const SimParams& P, const RunDesc* runs, int R,
                              const double* tmpl, const int* gidx, double* gkey, int cnt,
                              double* rsum, double* rnrm) {
    const int EG = max(1, RSUM_CAP / R);
    const bool norm = P.scoring == 1;
    for (int e0 = 0; e0 < cnt; e0 += EG) {
        const int ng = min(EG, cnt - e0);
        for (int w = threadIdx.x; w < ng * R; w += blockDim.x) {
            const int e = e0 + w / R, r = w - (w / R) * R;
            const int pos = gidx[e];
            const int x = pos / P.out_w, y = pos - x * P.out_w;
            const RunDesc rd = runs[r];
            const double* a = P.ti64 + static_cast<size_t>(rd.ch) * P.hc * P.wc +
                              static_cast<size_t>(x + rd.s) * P.wc + y;
            const double* b = tmpl + (rd.ch * P.Tc + rd.s) * P.Tc;
            double sum = 0.0, nsum = 0.0;
            for (int t = rd.t0; t < rd.t1; ++t) {
                const double av = __ldg(a + t);
                sum = __dadd_rn(sum, __dmul_rn(av, b[t]));
                if (norm) nsum = __dadd_rn(nsum, __dmul_rn(av, av));
            }
            rsum[w] = sum;
            if (norm) rnrm[w] = nsum;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < ng; e += blockDim.x) {
            double acc = 0.0;
            for (int r = 0; r < R; ++r) acc = __dadd_rn(acc, rsum[e * R + r]);
            if (norm) {
                double n = 0.0;
                for (int r = 0; r < R; ++r) n = __dadd_rn(n, rnrm[e * R + r]);
                acc = n > 0.0 ? __ddiv_rn(acc, __dsqrt_rn(n)) : 0.0;
            }
            gkey[e0 + e] = acc;
        }
        __syncthreads();
    }
}

// Reference ranking: higher score first, earlier row-major location on ties
// (matcher.hpp:189-198 -- the result is a prefix of the stable sort).
__device__ __forceinline__ bool better(double ka, int ia, double kb, int ib) {
    return ka > kb || (ka == kb && ia < ib);
}

// Monotone min-cost seam (simulator.hpp:286-320) with the reference tie rules;
// dp rows in shared memory, one thread per band column, thread 0 backtracks.
template <typename CostF>
__device__ void seam_dp(int layers, int width, CostF cost, int16_t* from, int* dp, int* seam) {
    for (int j = threadIdx.x; j < width; j += blockDim.x) dp[j] = cost(0, j);
    __syncthreads();
    for (int l = 1; l < layers; ++l) {
        const int* prev = dp + ((l - 1) & 1) * width;
        int* cur = dp + (l & 1) * width;
        for (int j = threadIdx.x; j < width; j += blockDim.x) {
            int best = prev[j], arg = j;
            if (j > 0 && prev[j - 1] < best) {
                best = prev[j - 1];
                arg = j - 1;
            }
            if (j + 1 < width && prev[j + 1] < best) {
                best = prev[j + 1];
                arg = j + 1;
            }
            if (j > 0 && prev[j - 1] == best && j - 1 < arg) arg = j - 1;
            cur[j] = cost(l, j) + best;
            from[l * width + j] = static_cast<int16_t>(arg);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int* last = dp + ((layers - 1) & 1) * width;
        int end = 0;
        for (int j = 1; j < width; ++j)
            if (last[j] < last[end]) end = j;
        seam[layers - 1] = end;
        for (int l = layers - 1; l > 0; --l) seam[l - 1] = from[l * width + seam[l]];
    }
    __syncthreads();
}

// min_cut_stitch (simulator.hpp:328-374) on T x T patches in shared memory:
// `outp` holds the incoming patch on entry and the stitched patch on exit.
__device__ void min_cut_device(const uint8_t* exist, uint8_t* outp, int T, int OV, int shape,
                               int vleft, int htop, int16_t* from, int* dp, int* seam) {
    if (shape == kNone) return;
    if (shape == kVertical || shape == kL) {
        const int c0 = vleft ? 0 : T - OV;
        seam_dp(T, OV,
                [&](int r, int j) { return exist[r * T + c0 + j] != outp[r * T + c0 + j] ? 1 : 0; },
                from, dp, seam);
        for (int e = threadIdx.x; e < T * OV; e += blockDim.x) {
            const int r = e / OV, j = e - r * OV;
            const bool keep = vleft ? j < seam[r] : j > seam[r];
            if (keep) outp[r * T + c0 + j] = exist[r * T + c0 + j];
        }
        __syncthreads();
    }
    if (shape == kHorizontal || shape == kL) {
        const int r0 = htop ? 0 : T - OV;
        seam_dp(T, OV,
                [&](int c, int j) { return exist[(r0 + j) * T + c] != outp[(r0 + j) * T + c] ? 1 : 0; },
                from, dp, seam);
        for (int e = threadIdx.x; e < T * OV; e += blockDim.x) {
            const int c = e / OV, j = e - c * OV;
            const bool keep = htop ? j < seam[c] : j > seam[c];
            if (keep) outp[(r0 + j) * T + c] = exist[(r0 + j) * T + c];
        }
        __syncthreads();
    }
}

// Rescore the gathered windows and merge them with the running top-K list
// (K rounds of a block-wide argmax under the reference ranking).
__device__ void flush_candidates(const SimParams& P, const RunDesc* runs, int R,
                                 const double* tmpl, int* gidx, double* gkey, int& cnt,
                                 double* tkey, int* tidx, int& ntop, int K, double* rsum,
                                 double* rnrm, double* redd, int* redi) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (P.stats && tid == 0) atomicAdd(&P.stats[0], static_cast<unsigned long long>(cnt));
    rescore_group(P, runs, R, tmpl, gidx, gkey, cnt, rsum, rnrm);
    for (int e = tid; e < ntop; e += SEL_T) {
        gkey[cnt + e] = tkey[e];
        gidx[cnt + e] = tidx[e];
    }
    __syncthreads();
    const int n = cnt + ntop;
    const int keep = min(K, n);
    for (int round = 0; round < keep; ++round) {
        double bk = 0.0;
        int bi = INT_MAX, bp = -1;
        for (int e = tid; e < n; e += SEL_T) {
            const int ix = gidx[e];
            if (ix >= 0 && (bp < 0 || better(gkey[e], ix, bk, bi))) {
                bk = gkey[e];
                bi = ix;
                bp = e;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            const int op = __shfl_xor_sync(0xffffffffu, bp, o);
            if (op >= 0 && (bp < 0 || better(ok, oi, bk, bi))) {
                bk = ok;
                bi = oi;
                bp = op;
            }
        }
        if (lane == 0) {
            redd[wid] = bk;
            redi[wid] = bi;
            redi[32 + wid] = bp;
        }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < SEL_T / 32; ++w) {
                if (redi[32 + w] >= 0 && (bp < 0 || better(redd[w], redi[w], bk, bi))) {
                    bk = redd[w];
                    bi = redi[w];
                    bp = redi[32 + w];
                }
            }
            tkey[round] = bk;
            tidx[round] = bi;
            gidx[bp] = -1;
        }
        __syncthreads();
    }
    ntop = keep;
    cnt = 0;
    __syncthreads();
}

// Normalized screen.  Mask variant of a placement:
// L (vleft, htop) 0-3, vertical strip 4 + vleft, horizontal strip 6 + htop.
__host__ __device__ inline int mask_variant(int shape, int vleft, int htop) {
    return shape == kL ? (vleft ? 2 : 0) + (htop ? 1 : 0)
                       : (shape == kVertical ? 4 + (vleft ? 1 : 0) : 6 + (htop ? 1 : 0));
}

// NN[v][p] = sum over mask variant v's cells and over every channel of the
// squared TI block count: the reference's normalization sum_f sum_mask ti_f^2
// (matcher.hpp:84-100, 163-171) times 4^J, exact in integers.
__global__ void nn_map_kernel(const float* __restrict__ scr, int nscr, int mode, int B, int hc, int wc,
                              int Tc, int OVc, int out_w, int npos, int32_t* __restrict__ out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const int v = blockIdx.y;
    if (p >= npos) return;
    const int shape = v < 4 ? kL : (v < 6 ? kVertical : kHorizontal);
    const int vleft = v < 4 ? (v >> 1) : (v < 6 ? v - 4 : 0);
    const int htop = v < 4 ? (v & 1) : (v < 6 ? 0 : v - 6);
    const int x = p / out_w, y = p - x * out_w;
    const size_t nc = static_cast<size_t>(hc) * wc;
    int acc = 0;
    for (int s = 0; s < Tc; ++s) {
        int t0, t1;
        mask_row_run(shape, vleft, htop, Tc, OVc, s, t0, t1);
        for (int t = t0; t < t1; ++t) {
            const size_t idx = static_cast<size_t>(x + s) * wc + y + t;
            if (mode == 0) {
                int rest = B * B;  // the last facies' count
                for (int f = 0; f < nscr; ++f) {
                    const int n = static_cast<int>(scr[f * nc + idx]);
                    acc += n * n;
                    rest -= n;
                }
                acc += rest * rest;
            } else {
                const int n = static_cast<int>(scr[idx]);
                acc += n * n;
            }
        }
    }
    out[static_cast<size_t>(v) * npos + p] = acc;
}

__global__ void __launch_bounds__(SEL_T) select_paste_kernel(SimParams P,
                                                             const Job* __restrict__ jobs,
                                                             int job0, int use_screen) {
    extern __shared__ __align__(16) unsigned char sel_sm[];
    const SelLayout L = sel_layout(P.K, P.T, P.OV, P.nch, P.Tc, P.scoring == 1);
    int* hist = reinterpret_cast<int*>(sel_sm + L.hist);
    int* misc = reinterpret_cast<int*>(sel_sm + L.misc);
    double* redd = reinterpret_cast<double*>(sel_sm + L.redd);
    int* redi = reinterpret_cast<int*>(sel_sm + L.redi);
    double* gkey = reinterpret_cast<double*>(sel_sm + L.gkey);
    int* gidx = reinterpret_cast<int*>(sel_sm + L.gidx);
    double* tkey = reinterpret_cast<double*>(sel_sm + L.tkey);
    int* tidx = reinterpret_cast<int*>(sel_sm + L.tidx);
    RunDesc* runs = reinterpret_cast<RunDesc*>(sel_sm + L.runs);
    double* tmpl = reinterpret_cast<double*>(sel_sm + L.tmpl);
    double* rsum = reinterpret_cast<double*>(sel_sm + L.rsum);
    double* rnrm = reinterpret_cast<double*>(sel_sm + L.rnrm);
    uint8_t* exist = sel_sm + L.exist;
    uint8_t* outp = sel_sm + L.outp;
    int16_t* from = reinterpret_cast<int16_t*>(sel_sm + L.from);
    int* dp = reinterpret_cast<int*>(sel_sm + L.dp);
    int* seam = reinterpret_cast<int*>(sel_sm + L.seam);

    pdl_trigger();
    const int gj = job0 + blockIdx.x;
    const Job jb = jobs[gj];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    pdl_wait();
    int fr, fc;
    if (jb.shape == kNone) {
        fr = jb.fr;
        fc = jb.fc;
    } else {
        const int Tc = P.Tc;
        const int32_t* sc = P.scores + static_cast<size_t>(blockIdx.x) * P.sld;
        const double* tm = P.tm64 + static_cast<size_t>(blockIdx.x) * P.nch * Tc * Tc;
        const int K = P.K;
        // stage the job's fp64 template and its run list (matcher.hpp:44-61 order)
        for (int e = tid; e < P.nch * Tc * Tc; e += SEL_T) tmpl[e] = tm[e];
        int R = 0;
        {
            int rows = 0;
            for (int s = 0; s < Tc; ++s) {
                int t0, t1;
                mask_row_run(jb.shape, jb.vleft, jb.htop, Tc, P.OVc, s, t0, t1);
                rows += t1 > t0;
            }
            R = rows * P.nch;
            if (tid == 0) {
                int r = 0;
                for (int ch = 0; ch < P.nch; ++ch)
                    for (int s = 0; s < Tc; ++s) {
                        int t0, t1;
                        mask_row_run(jb.shape, jb.vleft, jb.htop, Tc, P.OVc, s, t0, t1);
                        if (t1 > t0) runs[r++] = {ch, s, t0, t1};
                    }
            }
        }
        // 1. exact screen threshold: every window whose integer score reaches
        //    the K-th largest can appear in the reference's top-K.
        const bool all = !use_screen;
        const int32_t* tmx = P.tmax ? P.tmax + static_cast<size_t>(blockIdx.x) * P.ntiles : nullptr;
        int thr = 0;
        if (use_screen == 2) {
            // normalized: R = S / sqrt(NN) with S = S' + C_job and NN exact
            // integers; keys = R rounded down to float32 (monotone as int32
            // for R >= 0).  Every window the reference's fp64 score (relative
            // error << 1e-9) can rank in the top-K has R >= R_K (1 - 1e-9),
            // hence key >= the threshold below: a superset, rescored exactly.
            int32_t* scw = P.scores + static_cast<size_t>(blockIdx.x) * P.sld;
            const int32_t* nn = P.nnmap + static_cast<size_t>(mask_variant(jb.shape, jb.vleft, jb.htop)) * P.npos;
            const int cj = P.cjob[blockIdx.x];
            for (int p = tid; p < P.npos; p += SEL_T) {
                const int n = nn[p];
                const double R = n > 0 ? static_cast<double>(scw[p] + cj) / sqrt(static_cast<double>(n)) : 0.0;
                scw[p] = __float_as_int(__double2float_rd(R));
            }
            __syncthreads();
            const int kk = radix_kth_largest(sc, P.npos, K, hist, misc, redi);
            thr = __float_as_int(__double2float_rd(static_cast<double>(__int_as_float(kk)) * (1.0 - 1e-9)));
            tmx = nullptr;  // the tile maxima bound S', not the keys
        } else if (!all) {
            thr = radix_kth_largest(sc, P.npos, K, hist, misc, redi);
        }
        if (P.stats && tid == 0) atomicAdd(&P.stats[1], 1ull);
        __syncthreads();
        // 2. gather the tie group in row-major order, rescore in fp64, keep the
        //    running top-K by (fp64 desc, index asc).
        const int span = tmx ? kTcTile : SEL_T;
        const int nspans = (P.npos + span - 1) / span;
        int ntop = 0, cnt = 0;
        for (int sp = 0; sp < nspans; ++sp) {
            if (!all && tmx && tmx[sp] < thr) continue;  // uniform
            for (int sub = 0; sub < span; sub += SEL_T) {
                const int p = sp * span + sub + tid;
                const bool q = sub + tid < span && p < P.npos && (all || sc[p] >= thr);
                const unsigned bal = __ballot_sync(0xffffffffu, q);
                if (lane == 0) redi[wid] = __popc(bal);
                __syncthreads();
                int off = 0, tot = 0;
                for (int w = 0; w < SEL_T / 32; ++w) {
                    if (w < wid) off += redi[w];
                    tot += redi[w];
                }
                if (q) gidx[cnt + off + __popc(bal & ((1u << lane) - 1))] = p;
                cnt += tot;
                __syncthreads();
                if (cnt + SEL_T > GCAP)
                    flush_candidates(P, runs, R, tmpl, gidx, gkey, cnt, tkey, tidx, ntop, K, rsum,
                                     rnrm, redd, redi);
            }
        }
        if (cnt > 0)
            flush_candidates(P, runs, R, tmpl, gidx, gkey, cnt, tkey, tidx, ntop, K, rsum, rnrm,
                             redd, redi);
        // 3. choose (matcher.hpp:207-241)
        int pick = jb.pick;
        if (pick < 0) {
            int best = 0, best_mis = INT_MAX;
            pick = -1;
            const int cell = (jb.top / P.stride) * P.lat_nlc + jb.left / P.stride;
            const int e0 = P.hd_off[cell], e1 = P.hd_off[cell + 1];
            for (int c = 0; c < ntop; ++c) {
                const int pos = tidx[c];
                const int cfr = (pos / P.out_w) << P.J, cfc = (pos % P.out_w) << P.J;
                int mis = 0;
                for (int e = e0 + tid; e < e1; e += SEL_T) {
                    const uint32_t u = P.hd_ent[e];
                    const int rc = static_cast<int>(u >> 8), r = rc / P.T, cc = rc - r * P.T;
                    mis += P.ti[static_cast<size_t>(cfr + r) * P.ti_w + cfc + cc] != (u & 255u);
                }
                mis = block_reduce(mis, [](int a, int b) { return a + b; }, redi);
                if (mis == 0) {
                    pick = c;
                    break;
                }
                if (mis < best_mis) {
                    best = c;
                    best_mis = mis;
                }
            }
            if (pick < 0) pick = best;
        }
        const int pos = tidx[pick];
        fr = (pos / P.out_w) << P.J;
        fc = (pos % P.out_w) << P.J;
        __syncthreads();
    }

    // 4. crop + optional stitch + paste (simulator.hpp:483-493)
    const int T = P.T;
    uint8_t* g = P.work ? P.work + static_cast<size_t>(jb.real) * P.wh * P.ww : nullptr;
    uint8_t* trace = P.pasted ? P.pasted + static_cast<size_t>(gj) * T * T : nullptr;
    if (P.min_cut && jb.shape != kNone) {
        for (int e = tid; e < T * T; e += SEL_T) {
            const int r = e / T, c = e - r * T;
            exist[e] = g[static_cast<size_t>(jb.top + r) * P.ww + jb.left + c];
            outp[e] = P.ti[static_cast<size_t>(fr + r) * P.ti_w + fc + c];
        }
        __syncthreads();
        min_cut_device(exist, outp, T, P.OV, jb.shape, jb.vleft, jb.htop, from, dp, seam);
        for (int e = tid; e < T * T; e += SEL_T) {
            const int r = e / T, c = e - r * T;
            g[static_cast<size_t>(jb.top + r) * P.ww + jb.left + c] = outp[e];
            if (trace) trace[e] = outp[e];
        }
    } else if (P.work || trace) {  // (no work grid: the source-block map is the realization)
        for (int e = tid; e < T * T; e += SEL_T) {
            const int r = e / T, c = e - r * T;
            const uint8_t v = P.ti[static_cast<size_t>(fr + r) * P.ti_w + fc + c];
            if (P.work) g[static_cast<size_t>(jb.top + r) * P.ww + jb.left + c] = v;
            if (trace) trace[e] = v;
        }
    }
    if (P.src) {
        int32_t* sm = P.src + static_cast<size_t>(jb.real) * (P.wh / P.B) * P.swc;
        for (int e = tid; e < P.Tc * P.Tc; e += SEL_T) {
            const int a = e / P.Tc, b = e - a * P.Tc;
            sm[static_cast<size_t>(jb.top / P.B + a) * P.swc + jb.left / P.B + b] =
                (fr / P.B + a) * P.wc + fc / P.B + b;
        }
    }
    if (tid == 0) {
        P.chosen[2 * gj] = fr;
        P.chosen[2 * gj + 1] = fc;
    }
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

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}

// K-th largest (with multiplicity) of the union of the lanes' sorted top
// lists (INT_MIN padded): rounds of warp max over the lanes' heads.
__device__ __forceinline__ int warp_kth(const int (&top)[kTcQ], int K, int lane) {
    int ptr = 0, acc = 0;
    for (int round = 0; round < kTcQ + 1; ++round) {
        int head = INT_MIN;
#pragma unroll
        for (int i = 0; i < kTcQ; ++i)
            if (i == ptr) head = top[i];
        int m = head;
        for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        int c = 0;
#pragma unroll
        for (int i = 0; i < kTcQ; ++i)
            if (i >= ptr && top[i] == m) ++c;
        ptr += c;
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        acc += c;
        if (acc >= K || m == INT_MIN) return m;
    }
    return INT_MIN;
}

// Conditional / unconditional choice among the ranked top-K (matcher.hpp:207-241):
// the host-drawn index, or the first zero-mismatch candidate against the hard
// data, else the fewest mismatches.  Warp-level; every warp of a job may run
// it redundantly (identical inputs, identical result).
__device__ __forceinline__ int choose_pick(const SimParams& P, const Job& jb, const int* tidx, int ntop,
                                        int lane) {
    int pick = jb.pick;
    if (pick < 0) {
        int best = 0, best_mis = INT_MAX;
        const int cell = (jb.top / P.stride) * P.lat_nlc + jb.left / P.stride;
        const int e0 = P.hd_off[cell], e1 = P.hd_off[cell + 1];
        for (int c = 0; c < ntop; ++c) {
            const int pos = tidx[c];
            const int cfr = (pos / P.out_w) << P.J, cfc = (pos % P.out_w) << P.J;
            int mis = 0;
            for (int e = e0 + lane; e < e1; e += 32) {
                const uint32_t u = P.hd_ent[e];
                const int rc = static_cast<int>(u >> 8), r = rc / P.T, cc = rc - r * P.T;
                mis += P.ti[static_cast<size_t>(cfr + r) * P.ti_w + cfc + cc] != (u & 255u);
            }
            for (int o = 16; o > 0; o >>= 1) mis += __shfl_xor_sync(0xffffffffu, mis, o);
            if (mis == 0) {
                pick = c;
                break;
            }
            if (mis < best_mis) {
                best = c;
                best_mis = mis;
            }
        }
        if (pick < 0) pick = best;
    }
    return tidx[pick];
}

// Paste the chosen TI crop (simulator.hpp:483-493), record the trace and the
// source-block map; JT threads cooperate (jt = 0..JT-1).
template <int JT>
__device__ __forceinline__ void paste_job(const SimParams& P, const Job& jb, int gj, int fr, int fc,
                                          int jt) {
    const int Tc = P.Tc;
    const int T = P.T;
    uint8_t* trace = P.pasted ? P.pasted + static_cast<size_t>(gj) * T * T : nullptr;
    // Without a work grid (source-block map mode) the realization is rebuilt
    // from the map at finalize: only the map (and a requested trace) is written.
    uint8_t* g = P.work ? P.work + static_cast<size_t>(jb.real) * P.wh * P.ww : nullptr;
    const int wpr = T >> 2;  // 32-bit words per row
    const bool vec4 = ((fc | jb.left | P.ti_w | P.ww | T) & 3) == 0 && wpr <= JT && (JT % wpr) == 0;
    if (!g && !trace) {
    } else if (vec4) {
        // thread -> (row phase, word); every row it copies loaded in one round trip
        const int rpi = JT / wpr, rsub = jt / wpr, cw = jt - rsub * wpr;
        const uint8_t* srcp = P.ti + static_cast<size_t>(fr) * P.ti_w + fc + 4 * cw;
        uint8_t* dstp = g ? g + static_cast<size_t>(jb.top) * P.ww + jb.left + 4 * cw : nullptr;
        for (int r0 = rsub; r0 < T; r0 += rpi * 32) {
            uint32_t v[32];  // every row this lane copies, loaded in one round trip
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int r = r0 + i * rpi;
                if (r < T) v[i] = *reinterpret_cast<const uint32_t*>(srcp + static_cast<size_t>(r) * P.ti_w);
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int r = r0 + i * rpi;
                if (r < T) {
                    if (g) *reinterpret_cast<uint32_t*>(dstp + static_cast<size_t>(r) * P.ww) = v[i];
                    if (trace) *reinterpret_cast<uint32_t*>(trace + r * T + 4 * cw) = v[i];
                }
            }
        }
    } else {
        // unaligned rows: byte copies, 16 loads in flight per thread
        constexpr int BB = 16;
        for (int e0 = 0; e0 < T * T; e0 += JT * BB) {
            uint8_t v[BB];
#pragma unroll
            for (int i = 0; i < BB; ++i) {
                const int e = e0 + i * JT + jt;
                const int r = e / T, c = e - r * T;
                if (e < T * T) v[i] = P.ti[static_cast<size_t>(fr + r) * P.ti_w + fc + c];
            }
#pragma unroll
            for (int i = 0; i < BB; ++i) {
                const int e = e0 + i * JT + jt;
                const int r = e / T, c = e - r * T;
                if (e < T * T) {
                    if (g) g[static_cast<size_t>(jb.top + r) * P.ww + jb.left + c] = v[i];
                    if (trace) trace[e] = v[i];
                }
            }
        }
    }
    if (P.src) {  // Tc x Tc map entries spread over every thread
        int32_t* sm = P.src + static_cast<size_t>(jb.real) * (P.wh / P.B) * P.swc +
                      static_cast<size_t>(jb.top / P.B) * P.swc + jb.left / P.B;
        const int s0 = (fr / P.B) * P.wc + fc / P.B;
        for (int e = jt; e < Tc * Tc; e += JT) {
            const int a = e / Tc, b = e - a * Tc;
            sm[static_cast<size_t>(a) * P.swc + b] = s0 + a * P.wc + b;
        }
    }
}

struct ScanWarp {
    int lv[SC_LC];
    int lp[SC_LC];
    int tq[SC_TB];  // queued qualifying tiles
};

// Warp-level scan of one placement (every lane of the warp calls it): the
// tile-maximum bound M_K, the (score, position) list of windows >= M_K, the
// exact K-th score S_K and the candidate positions (>= S_K) into out[].
// Returns the candidate count, or -1 when the list overflowed (then every
// window >= mk_out must be rescored -- a superset, still exact).
__device__ __forceinline__ int scan_job(const SimParams& P, int slot, ScanWarp& W, int* out, int& mk_out,
                                        long long* sclk, int* out_s = nullptr) {
    const int lane = threadIdx.x & 31;
    const int K = P.K;
    const int32_t* sc = P.scores + static_cast<size_t>(slot) * P.sld;
    const int32_t* tmx = P.tmax + static_cast<size_t>(slot) * P.ntiles;
    // 1. M_K = K-th largest tile maximum (with multiplicity): a lower bound of
    //    the K-th largest screen score S_K (the K best tiles each hold a
    //    window scoring at least M_K).  Tile maxima stay in registers.
    constexpr int kTM = 16;  // tile maxima per lane (512 tiles per placement)
    const bool regs = P.ntiles <= 32 * kTM;  // else: stream the maxima (sorted per-lane top lists)
    int tv[kTM];
#pragma unroll
    for (int i = 0; i < kTM; ++i) {
        const int e = i * 32 + lane;
        tv[i] = regs && e < P.ntiles ? tmx[e] : INT_MIN;
    }
    int mk = INT_MIN;
    if (!regs) {
        int top[kTcQ];
#pragma unroll
        for (int i = 0; i < kTcQ; ++i) top[i] = INT_MIN;
        for (int e = lane; e < P.ntiles; e += 32) {
            int v = tmx[e];
            if (v > top[kTcQ - 1]) {
#pragma unroll
                for (int j = 0; j < kTcQ; ++j)
                    if (v > top[j]) {
                        const int t = top[j];
                        top[j] = v;
                        v = t;
                    }
            }
        }
        mk = warp_kth(top, K, lane);
    } else {
        int cur = INT_MAX, acc = 0;
        for (int round = 0; round < K; ++round) {
            int m = INT_MIN;
#pragma unroll
            for (int i = 0; i < kTM; ++i)
                if (tv[i] < cur) m = max(m, tv[i]);
            m = __reduce_max_sync(0xffffffffu, m);
            int c = 0;
#pragma unroll
            for (int i = 0; i < kTM; ++i) c += tv[i] == m;
            acc += static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(c)));
            mk = m;
            if (acc >= K || m == INT_MIN) break;
            cur = m;
        }
    }
    sclk[1] = clock64();
    // 2. every window scoring >= M_K, from the tiles whose maximum reaches it,
    //    into a (score, position) list.  Qualifying tiles are queued across the
    //    32-tile groups and loaded SC_TB per round trip.
    int nl = 0, ntl = 0;
    bool over = false;
    auto flush_tiles = [&]() {
        __syncwarp();
        int tl[SC_TB], v[SC_TB][4];
#pragma unroll
        for (int u = 0; u < SC_TB; ++u) tl[u] = u < ntl ? W.tq[u] : -1;
#pragma unroll
        for (int u = 0; u < SC_TB; ++u) {
            const int p0 = tl[u] * kTcTile + lane * 4;
#pragma unroll
            for (int i = 0; i < 4; ++i) v[u][i] = INT_MIN;
            if (tl[u] >= 0 && p0 < P.npos) {  // rows are padded to a multiple of 4
                const int4 a4 = *reinterpret_cast<const int4*>(sc + p0);
                v[u][0] = a4.x;
                v[u][1] = p0 + 1 < P.npos ? a4.y : INT_MIN;
                v[u][2] = p0 + 2 < P.npos ? a4.z : INT_MIN;
                v[u][3] = p0 + 3 < P.npos ? a4.w : INT_MIN;
            }
        }
#pragma unroll
        for (int u = 0; u < SC_TB; ++u)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const bool q = v[u][i] != INT_MIN && v[u][i] >= mk;  // scores are never INT_MIN
                const unsigned bal = __ballot_sync(0xffffffffu, q);
                if (!bal) continue;
                if (nl + __popc(bal) > SC_LC) {
                    over = true;
                    continue;
                }
                if (q) {
                    const int o = nl + __popc(bal & ((1u << lane) - 1));
                    W.lv[o] = v[u][i];
                    W.lp[o] = tl[u] * kTcTile + lane * 4 + i;
                }
                nl += __popc(bal);
            }
        ntl = 0;
        __syncwarp();
    };
#pragma unroll 1
    for (int i0 = 0; i0 * 32 < P.ntiles && !over; ++i0) {
        const int t0 = i0 * 32;
        int mine = INT_MIN;
        if (regs) {
#pragma unroll
            for (int i = 0; i < kTM; ++i)
                if (i == i0) mine = tv[i];
        } else if (t0 + lane < P.ntiles) {
            mine = tmx[t0 + lane];
        }
        unsigned tiles = __ballot_sync(0xffffffffu, mine != INT_MIN && mine >= mk);
        while (tiles && !over) {
            if (lane == 0) W.tq[ntl] = t0 + __ffs(tiles) - 1;
            tiles &= tiles - 1;
            if (++ntl == SC_TB) flush_tiles();
        }
    }
    if (ntl > 0 && !over) flush_tiles();
    __syncwarp();
    sclk[2] = clock64();
#ifdef CCW_DBG_STATS
    if (P.stats) {
        int nq = 0;
        for (int t0 = 0; t0 < P.ntiles; t0 += 32)
            nq += __popc(__ballot_sync(0xffffffffu, t0 + lane < P.ntiles && tmx[t0 + lane] >= mk));
        if (lane == 0) {
            atomicAdd(&P.stats[5], static_cast<unsigned long long>(nq));
            atomicAdd(&P.stats[6], static_cast<unsigned long long>(nl));
        }
    }
#endif
    if (P.stats && lane == 0) atomicAdd(&P.stats[1], 1ull);
    mk_out = mk;
    if (over) {
        if (lane == 0 && P.stats) atomicAdd(&P.stats[2], 1ull);
        return -1;
    }
    // 3. exact S_K from the list (rounds of warp max with multiplicity)
    int lvr[SC_LC / 32];
#pragma unroll
    for (int j2 = 0; j2 < SC_LC / 32; ++j2) {
        const int e = j2 * 32 + lane;
        lvr[j2] = e < nl ? W.lv[e] : INT_MIN;
    }
    int thr = mk, cur = INT_MAX, acc = 0;
    for (int round = 0; round < K; ++round) {
        int m = INT_MIN;
#pragma unroll
        for (int j2 = 0; j2 < SC_LC / 32; ++j2)
            if (lvr[j2] < cur) m = max(m, lvr[j2]);
        m = __reduce_max_sync(0xffffffffu, m);
        int c = 0;
#pragma unroll
        for (int j2 = 0; j2 < SC_LC / 32; ++j2) c += lvr[j2] == m;
        acc += static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(c)));
        thr = m;
        if (acc >= K || m == INT_MIN) break;
        cur = m;
    }
    sclk[3] = clock64();
    // 4. the candidates: every listed window >= S_K
    int* cd = out;
    int cnt = 0;
    for (int e0 = 0; e0 < nl; e0 += 32) {
        const int e = e0 + lane;
        const bool q = e < nl && W.lv[e] >= thr;
        const unsigned bal = __ballot_sync(0xffffffffu, q);
        if (q) {
            const int o = cnt + __popc(bal & ((1u << lane) - 1));
            cd[o] = W.lp[e];
            if (out_s) out_s[o] = W.lv[e];
        }
        cnt += __popc(bal);
    }
    return cnt;
}

// Fused OR prep (select epilogue): after this placement's source-block map
// is written, count it against each next-wave placement that reads it; the
// CTA that completes a dependent's count prepares that dependent (its OR
// weights, template and C_job) into the next wave's buffers.  Every thread
// of the CTA calls this (it synchronizes).
__device__ __forceinline__ void prep_dependents(const SimParams& P, const Job* __restrict__ jobs,
                                                const Job& jb, int* flag) {
    if (!P.depcnt) return;
    __syncthreads();  // this CTA's map writes are issued
    for (int q = 0; q < 2; ++q) {
        const int d = q == 0 ? jb.dep0 : jb.dep1;  // uniform
        if (d < 0) continue;
        if (threadIdx.x == 0) {
            __threadfence();  // release the map writes before counting
            const int need = jobs[d].ndep;
            const int old = atomicAdd(&P.depcnt[d - P.next_j0], 1);
            *flag = old == need - 1;
            if (*flag) {
                P.depcnt[d - P.next_j0] = 0;  // reset for the next use of this slot
                __threadfence();              // acquire the other dependency's writes
            }
        }
        __syncthreads();
        if (*flag) prep_src_job(P, jobs[d], d - P.next_j0, P.n_wts8, P.n_tm64, P.n_cjob);
        __syncthreads();
    }
}

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
#ifndef CCW_FS_RS
#define CCW_FS_RS 1536
#endif
constexpr int FS_RS = CCW_FS_RS;    // (window, run) partial sums per batch

struct FastSmem {
    double tm[PK_TMC];
    double rsum[FS_RS];
    double key[SC_LC + kTcQ];
    int cidx[SC_LC + kTcQ];
    int cs[SC_LC];          // the candidates' screen scores
    int tie[32];            // candidates sharing their screen score (positions)
    int tslot[32];          // candidate -> its entry in tie[] (or -1)
    ScanWarp sw;
    int4 grp[FS_MAXG];      // (channel, first row-table index, rows, t0 << 8 | len)
    short4 rows[PK_MAXTC];  // mask rows (s, t0, t1, -)
    double tkey[kTcQ];
    int tidx[kTcQ];
    double rk[FS_T / 32];
    int ri[FS_T / 32], rp[FS_T / 32], wc[FS_T / 32];
    int misc[8];
};

// Rescore S.cidx[0, cnt) and merge with the running top-K (ntop entries).
// fp64 keys of the windows cidx[0, cnt) (reference order, see fast_batch).
__device__ __forceinline__ void rescore_keys(const SimParams& P, FastSmem& S, const double* tmS, int nr,
                                             int ngrp, const int* cidx, int cnt, double* keys) {
    const int tid = threadIdx.x;
    const int R = nr * P.nch;
    const int EB = max(1, FS_RS / R);
    const size_t plane = static_cast<size_t>(P.hc) * P.wc;
    if (P.stats && tid == 0) atomicAdd(&P.stats[0], static_cast<unsigned long long>(cnt));
    for (int e0 = 0; e0 < cnt; e0 += EB) {
        const int ng = min(EB, cnt - e0);
        for (int it = tid; it < ng * ngrp; it += FS_T) {
            const int e = it / ngrp, g = it - e * ngrp;
            const int4 G = S.grp[g];
            const int ch = G.x, k0 = G.y, nk = G.z, t0 = G.w >> 8, len = G.w & 255;
            const int pos = cidx[e0 + e];
            const int x = pos / P.out_w, y = pos - x * P.out_w;
            const double* base = P.ti64 + ch * plane + static_cast<size_t>(x) * P.wc + y + t0;
            const double* tb = tmS + ch * P.Tc * P.Tc + t0;
            double* rs = S.rsum + e * R + ch * nr + k0;
            if (len > FS_G) {  // one long run (nk == 1), FS_G operands per round trip
                const int s = S.rows[k0].x;
                const double* a = base + static_cast<size_t>(s) * P.wc;
                const double* b = tb + s * P.Tc;
                double sum = 0.0;
                for (int c0 = 0; c0 < len; c0 += FS_G) {
                    double av[FS_G];
#pragma unroll
                    for (int c = 0; c < FS_G; ++c) av[c] = c0 + c < len ? __ldg(a + c0 + c) : 0.0;
#pragma unroll
                    for (int c = 0; c < FS_G; ++c)
                        if (c0 + c < len) sum = __dadd_rn(sum, __dmul_rn(av[c], b[c0 + c]));
                }
                rs[0] = sum;
                continue;
            }
            double av[FS_G];
            {
                int kk = 0, t = 0;
#pragma unroll
                for (int c = 0; c < FS_G; ++c) {
                    av[c] = kk < nk ? __ldg(base + static_cast<size_t>(S.rows[k0 + kk].x) * P.wc + t) : 0.0;
                    if (++t == len) {
                        t = 0;
                        ++kk;
                    }
                }
            }
            double sum = 0.0;
            int kk = 0, t = 0;
#pragma unroll
            for (int c = 0; c < FS_G; ++c) {
                if (kk < nk) {
                    sum = __dadd_rn(sum, __dmul_rn(av[c], tb[S.rows[k0 + kk].x * P.Tc + t]));
                    if (++t == len) {
                        rs[kk] = sum;
                        sum = 0.0;
                        t = 0;
                        ++kk;
                    }
                }
            }
        }
        __syncthreads();
        for (int e = tid; e < ng; e += FS_T) {
            // the fold is one sequential chain; its operands load 8 at a time
            const double* rp = S.rsum + e * R;
            double acc = 0.0;
            int r = 0;
            for (; r + 8 <= R; r += 8) {
                double x[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) x[i] = rp[r + i];
#pragma unroll
                for (int i = 0; i < 8; ++i) acc = __dadd_rn(acc, x[i]);
            }
            for (; r < R; ++r) acc = __dadd_rn(acc, rp[r]);
            keys[e0 + e] = acc;
        }
        __syncthreads();
    }
}

// Rescore S.cidx[0, cnt) and merge with the running top-K (ntop entries).
__device__ __forceinline__ void fast_batch(const SimParams& P, FastSmem& S, const double* tmS, int nr,
                                           int ngrp, int cnt, int& ntop, int K) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    rescore_keys(P, S, tmS, nr, ngrp, S.cidx, cnt, S.key);
    // merge: the batch plus the running top-K (reference ranking)
    for (int e = tid; e < ntop; e += FS_T) {
        S.key[cnt + e] = S.tkey[e];
        S.cidx[cnt + e] = S.tidx[e];
    }
    __syncthreads();
    const int n = cnt + ntop;
    const int keep = min(K, n);
    if (n <= 32) {
        if (wid == 0) {
            const double mk = lane < n ? S.key[lane] : 0.0;
            const int mi = lane < n ? S.cidx[lane] : INT_MAX;
            int rank = 0;
            for (int j = 0; j < n; ++j) {
                const double ok = __shfl_sync(0xffffffffu, mk, j);
                const int oi = __shfl_sync(0xffffffffu, mi, j);
                rank += better(ok, oi, mk, mi);
            }
            if (lane < n && rank < keep) {
                S.tkey[rank] = mk;
                S.tidx[rank] = mi;
            }
        }
    } else {
        for (int round = 0; round < keep; ++round) {
            double bk = 0.0;
            int bi = INT_MAX, bp = -1;
            for (int e = tid; e < n; e += FS_T) {
                const int ix = S.cidx[e];
                if (ix >= 0 && (bp < 0 || better(S.key[e], ix, bk, bi))) {
                    bk = S.key[e];
                    bi = ix;
                    bp = e;
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                const int op = __shfl_xor_sync(0xffffffffu, bp, o);
                if (op >= 0 && (bp < 0 || better(ok, oi, bk, bi))) {
                    bk = ok;
                    bi = oi;
                    bp = op;
                }
            }
            if (lane == 0) {
                S.rk[wid] = bk;
                S.ri[wid] = bi;
                S.rp[wid] = bp;
            }
            __syncthreads();
            if (tid == 0) {
                for (int w = 1; w < FS_T / 32; ++w)
                    if (S.rp[w] >= 0 && (bp < 0 || better(S.rk[w], S.ri[w], bk, bi))) {
                        bk = S.rk[w];
                        bi = S.ri[w];
                        bp = S.rp[w];
                    }
                S.tkey[round] = bk;
                S.tidx[round] = bi;
                S.cidx[bp] = -1;
            }
            __syncthreads();
        }
    }
    ntop = keep;
    __syncthreads();
}

#ifndef CCW_FS_MINB
#define CCW_FS_MINB 4
#endif
__global__ void __launch_bounds__(FS_T, CCW_FS_MINB)
    select_fast_kernel(SimParams P, const Job* __restrict__ jobs, int job0, int nj) {
    __shared__ FastSmem S;
    const int slot = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    pdl_trigger();
    tl_mark(P.tl, 2);
    pdl_wait();
    tl_mark(P.tl, 0);
    if (slot >= nj) return;
    const int gj = job0 + slot;
    const Job jb = jobs[gj];
    const int Tc = P.Tc;
    long long fclk[5] = {clock64(), 0, 0, 0, 0};
    int fr, fc;
    if (jb.shape == kNone) {
        fr = jb.fr;
        fc = jb.fc;
    } else {
        const int K = P.K;
        const double* tmg = P.tm64 + static_cast<size_t>(slot) * P.nch * Tc * Tc;
        const int ntm = P.nch * Tc * Tc;
        const double* tmS = ntm <= PK_TMC ? S.tm : tmg;
        int mk = INT_MIN;
        if (wid == 0) {
            long long sclk[5];
            sclk[0] = clock64();
            const int n = scan_job(P, slot, S.sw, S.cidx, mk, sclk, S.cs);
            if (lane == 0) {
                S.misc[0] = n;
                S.misc[1] = mk;
                if (P.stats && P.tl && n >= 0) {
                    sclk[4] = clock64();
                    for (int q = 0; q < 4; ++q)
                        atomicAdd(&P.stats[8 + q], static_cast<unsigned long long>(sclk[q + 1] - sclk[q]));
                }
            }
        } else {
            // stage the template (matcher.hpp:44-61 order), the mask rows and the run groups
            if (ntm <= PK_TMC)
                for (int e = tid - 32; e < ntm; e += FS_T - 32) cp_async8(&S.tm[e], tmg + e);
            if (wid == 1) {
                int nr = 0;
                for (int s0 = 0; s0 < Tc; s0 += 32) {
                    const int s = s0 + lane;
                    int t0 = 0, t1 = 0;
                    if (s < Tc) mask_row_run(jb.shape, jb.vleft, jb.htop, Tc, P.OVc, s, t0, t1);
                    const unsigned m = __ballot_sync(0xffffffffu, t1 > t0);
                    if (t1 > t0) S.rows[nr + __popc(m & ((1u << lane) - 1))] = make_short4(s, t0, t1, 0);
                    nr += __popc(m);
                }
                __syncwarp();
                if (lane == 0) {
                    int ng = 0;
                    for (int ch = 0; ch < P.nch; ++ch) {
                        int k = 0;
                        while (k < nr) {
                            const int t0 = S.rows[k].y, len = S.rows[k].z - S.rows[k].y;
                            int nk = 1;
                            while (k + nk < nr && S.rows[k + nk].y == t0 && S.rows[k + nk].z - t0 == len &&
                                   (nk + 1) * len <= FS_G)
                                ++nk;
                            if (len > FS_G) {  // a long run stays one item (one sequential sum)
                                if (ng < FS_MAXG) S.grp[ng++] = make_int4(ch, k, 1, (t0 << 8) | len);
                                nk = 1;
                            } else if (ng < FS_MAXG) {
                                S.grp[ng++] = make_int4(ch, k, nk, (t0 << 8) | len);
                            }
                            k += nk;
                        }
                    }
                    S.misc[2] = nr;
                    S.misc[3] = ng;
                }
            }
            cp_async_wait_all();
        }
        __syncthreads();
        fclk[1] = clock64();
        const int n = S.misc[0], nr = S.misc[2], ngrp = S.misc[3];
        mk = S.misc[1];
        int ntop = 0;
        if (n < 0 && P.defer) {  // a large tie group: the bulk kernel rescores every window >= M_K
            if (tid == 0) P.defer[slot] = max(mk, INT_MIN + 1);  // (INT_MIN marks "not deferred")
            return;
        }
        if (P.defer && tid == 0) P.defer[slot] = INT_MIN;
        if (n >= 0 && n <= 32) {
            // Windows with different screen scores never swap in fp64 (§3 of
            // DESIGN.md): only candidates that share their score are rescored;
            // the ranking is (S desc, fp64 desc within equal S, index asc).
            if (wid == 0) {
                const int sv = lane < n ? S.cs[lane] : INT_MIN;
                const unsigned grp = __match_any_sync(0xffffffffu, sv);
                const bool tie = lane < n && __popc(grp) > 1;
                const unsigned tb = __ballot_sync(0xffffffffu, tie);
                const int o = __popc(tb & ((1u << lane) - 1));
                if (tie) S.tie[o] = S.cidx[lane];
                if (lane < n) S.tslot[lane] = tie ? o : -1;
                if (lane == 0) S.misc[6] = __popc(tb);
            }
            __syncthreads();
            const int nt = S.misc[6];
            if (nt > 0) rescore_keys(P, S, tmS, nr, ngrp, S.tie, nt, S.key);
            if (wid == 0) {
                const int si = lane < n ? S.cs[lane] : INT_MIN;
                const int ii = lane < n ? S.cidx[lane] : INT_MAX;
                const double ki = lane < n && S.tslot[lane] >= 0 ? S.key[S.tslot[lane]] : 0.0;
                int rank = 0;
                for (int j = 0; j < n; ++j) {
                    const int sj = __shfl_sync(0xffffffffu, si, j);
                    const int ij = __shfl_sync(0xffffffffu, ii, j);
                    const double kj = __shfl_sync(0xffffffffu, ki, j);
                    rank += sj > si || (sj == si && better(kj, ij, ki, ii));
                }
                if (lane < n && rank < K) {
                    S.tidx[rank] = ii;
                    S.tkey[rank] = ki;
                }
            }
            ntop = min(K, n);
            __syncthreads();
        } else if (n >= 0) {
            fast_batch(P, S, tmS, nr, ngrp, n, ntop, K);
        } else {
            // list overflow without the bulk kernel: every window >= M_K, in batches
            const int32_t* sc = P.scores + static_cast<size_t>(slot) * P.sld;
            const int32_t* tmx = P.tmax + static_cast<size_t>(slot) * P.ntiles;
            int cnt = 0;
            for (int t = 0; t < P.ntiles; ++t) {
                if (tmx[t] < mk) continue;  // uniform
                const int p = t * kTcTile + tid;  // FS_T == kTcTile
                const bool q = p < P.npos && sc[p] >= mk;
                const unsigned bal = __ballot_sync(0xffffffffu, q);
                if (lane == 0) S.wc[wid] = __popc(bal);
                __syncthreads();
                int off = 0, tot = 0;
                for (int w = 0; w < FS_T / 32; ++w) {
                    off += w < wid ? S.wc[w] : 0;
                    tot += S.wc[w];
                }
                __syncthreads();
                if (cnt + tot > SC_LC) {
                    fast_batch(P, S, tmS, nr, ngrp, cnt, ntop, K);
                    cnt = 0;
                }
                if (q) S.cidx[cnt + off + __popc(bal & ((1u << lane) - 1))] = p;
                cnt += tot;
                __syncthreads();
            }
            if (cnt > 0) fast_batch(P, S, tmS, nr, ngrp, cnt, ntop, K);
        }
        fclk[2] = clock64();
        // choose (matcher.hpp:207-241)
        if (wid == 0) {
            const int pos = choose_pick(P, jb, S.tidx, ntop, lane);
            if (lane == 0) S.misc[4] = pos;
        }
        __syncthreads();
        fclk[3] = clock64();
        const int pos = S.misc[4];
        fr = (pos / P.out_w) << P.J;
        fc = (pos % P.out_w) << P.J;
    }
    paste_job<FS_T>(P, jb, gj, fr, fc, tid);
    prep_dependents(P, jobs, jb, &S.misc[5]);
    if (tid == 0) {
        P.chosen[2 * gj] = fr;
        P.chosen[2 * gj + 1] = fc;
        if (P.stats && P.tl && fclk[3]) {
            fclk[4] = clock64();
            atomicAdd(&P.stats[12], static_cast<unsigned long long>(fclk[1] - fclk[0]));
            atomicAdd(&P.stats[13], static_cast<unsigned long long>(fclk[2] - fclk[1]));
            atomicAdd(&P.stats[4], static_cast<unsigned long long>(fclk[4] - fclk[2]));
            atomicAdd(&P.stats[5], static_cast<unsigned long long>(fclk[3] - fclk[2]));  // choose
        }
    }
    tl_mark(P.tl, 1);
}

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
constexpr int BK_T = 256;
constexpr int BK_W = 4;
constexpr int BK_V = 8;      // positions per thread per scan pass
constexpr int BK_SMAX = 8;   // CTAs per placement (upper bound)

struct BulkLayout {
    size_t stage, tm, rows, cand, misc, total;
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
    L.misc = o;
    o += 320 + static_cast<size_t>(BK_SMAX) * kTcQ * (sizeof(double) + sizeof(int));
    L.total = o;
    return L;
}

__global__ void __launch_bounds__(BK_T, 1)
    select_bulk_kernel(SimParams P, const Job* __restrict__ jobs, int job0, int nj, int S) {
    extern __shared__ __align__(16) unsigned char bk_sm[];
    pdl_trigger();
    tl_mark(P.tl, 2);
    pdl_wait();
    tl_mark(P.tl, 0);
    const int slot = blockIdx.y, part = blockIdx.x;
    if (slot >= nj) return;
    const int thr = P.defer[slot];
    if (thr == INT_MIN) return;  // handled by the warp select
    const int gj = job0 + slot;
    const Job jb = jobs[gj];
    const int Tc = P.Tc, nch = P.nch, K = P.K;
    const int bx = P.bulk_bx, by = P.bulk_by;
    const BulkLayout L = bulk_layout(nch, Tc, bx, by);
    double* stg = reinterpret_cast<double*>(bk_sm + L.stage);
    double* tmS = reinterpret_cast<double*>(bk_sm + L.tm);
    short4* rows = reinterpret_cast<short4*>(bk_sm + L.rows);
    int* cand = reinterpret_cast<int*>(bk_sm + L.cand);
    unsigned char* misc = bk_sm + L.misc;
    int* wcnt = reinterpret_cast<int*>(misc);               // [8]
    double* rk = reinterpret_cast<double*>(misc + 64);     // [8]
    int* ri = reinterpret_cast<int*>(misc + 128);          // [8]
    int* rp = reinterpret_cast<int*>(misc + 160);          // [8]
    double* tkey = reinterpret_cast<double*>(misc + 192);  // [kTcQ]
    int* tidx = reinterpret_cast<int*>(misc + 256);        // [kTcQ]
    int* shv = reinterpret_cast<int*>(misc + 288);         // [4] broadcast scalars
    double* mk = reinterpret_cast<double*>(misc + 320);    // [BK_SMAX * kTcQ] merge keys
    int* mi = reinterpret_cast<int*>(misc + 320 + 8 * BK_SMAX * kTcQ);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int32_t* sc = P.scores + static_cast<size_t>(slot) * P.sld;
    const int32_t* tmx = P.tmax + static_cast<size_t>(slot) * P.ntiles;
    const double* tm = P.tm64 + static_cast<size_t>(slot) * nch * Tc * Tc;
    long long clk_stage = 0, clk_comp = 0;
    const long long clk_start = clock64();
    for (int e = tid; e < nch * Tc * Tc; e += BK_T) tmS[e] = tm[e];
    int nrows = 0;
    for (int s0 = 0; s0 < Tc; s0 += 32) {
        const int s = s0 + lane;
        int t0 = 0, t1 = 0;
        if (s < Tc) mask_row_run(jb.shape, jb.vleft, jb.htop, Tc, P.OVc, s, t0, t1);
        const unsigned m = __ballot_sync(0xffffffffu, t1 > t0);
        if (wid == 0 && t1 > t0) rows[nrows + __popc(m & ((1u << lane) - 1))] = make_short4(s, t0, t1, 0);
        nrows += __popc(m);
    }
    double tk[kTcQ];
    int tix[kTcQ];
#pragma unroll
    for (int j = 0; j < kTcQ; ++j) {
        tk[j] = -INFINITY;
        tix[j] = INT_MAX;
    }
    unsigned long long rescored = 0;
    const int nbx = (P.out_h + bx - 1) / bx, nby = (P.out_w + by - 1) / by;
    int* next = P.bulk_sync + 2 * slot;  // [0] next block, [1] finished CTAs
    for (;;) {
        __syncthreads();  // previous block's stage / candidates consumed
        if (tid == 0) shv[0] = atomicAdd(next, 1);
        __syncthreads();
        const int kb = shv[0];
        if (kb >= nbx * nby) break;
        const int xb = (kb / nby) * bx, yb = (kb % nby) * by;
        const int bxa = min(bx, P.out_h - xb), bya = min(by, P.out_w - yb);
        // skip blocks whose tiles all stay below the threshold
        const int tf = (xb * P.out_w + yb) / kTcTile;
        const int tl = ((xb + bxa - 1) * P.out_w + yb + bya - 1) / kTcTile;
        bool any = false;
        for (int t = tf + tid; t <= tl; t += BK_T) any |= tmx[t] >= thr;
        if (!__syncthreads_or(any)) continue;
        // windows of the block at or above the threshold (block-local index)
        const long long c_st = clock64();
        int cnt = 0;
        const int nb = bxa * bya;
        for (int e0 = 0; e0 < nb; e0 += BK_T * BK_V) {
            int v[BK_V];
#pragma unroll
            for (int i = 0; i < BK_V; ++i) {
                const int e = e0 + tid * BK_V + i;
                v[i] = INT_MIN;
                if (e < nb) {
                    const int lx = e / bya, ly = e - lx * bya;
                    v[i] = sc[(xb + lx) * P.out_w + yb + ly];
                }
            }
            int c = 0;
#pragma unroll
            for (int i = 0; i < BK_V; ++i) c += v[i] >= thr;
            int incl = c;  // warp inclusive scan
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) wcnt[wid] = incl;
            __syncthreads();
            int off = incl - c, tot = 0;
#pragma unroll
            for (int w = 0; w < BK_T / 32; ++w) {
                off += w < wid ? wcnt[w] : 0;
                tot += wcnt[w];
            }
            off += cnt;
#pragma unroll
            for (int i = 0; i < BK_V; ++i)
                if (v[i] >= thr) cand[off++] = e0 + tid * BK_V + i;
            cnt += tot;
            __syncthreads();
        }
        if (cnt == 0) continue;
        rescored += cnt;
        // stage the apex tile the block's windows read
        const int sha = bxa + Tc - 1, swa = bya + Tc - 1;
        for (int ch = 0; ch < nch; ++ch) {
            const double* src = P.ti64 + static_cast<size_t>(ch) * P.hc * P.wc +
                                static_cast<size_t>(xb) * P.wc + yb;
            double* dst = stg + static_cast<size_t>(ch) * L.sh * L.sw;
            for (int e = tid; e < sha * swa; e += BK_T) {
                const int r = e / swa, c = e - r * swa;
                cp_async8(dst + r * L.sw + c, src + static_cast<size_t>(r) * P.wc + c);
            }
        }
        cp_async_wait_all();
        __syncthreads();
        const long long c_cp = clock64();
        clk_stage += c_cp - c_st;
        for (int i0 = tid; i0 < cnt; i0 += BK_T * BK_W) {
            int base[BK_W], pidx[BK_W];
            bool ok[BK_W];
#pragma unroll
            for (int k = 0; k < BK_W; ++k) {
                const int i = i0 + k * BK_T;
                ok[k] = i < cnt;
                const int e = cand[ok[k] ? i : i0];
                const int lx = e / bya, ly = e - lx * bya;
                base[k] = lx * L.sw + ly;
                pidx[k] = (xb + lx) * P.out_w + yb + ly;
            }
            double acc[BK_W];
#pragma unroll
            for (int k = 0; k < BK_W; ++k) acc[k] = 0.0;
            for (int ch = 0; ch < nch; ++ch) {
                const double* sp = stg + static_cast<size_t>(ch) * L.sh * L.sw;
                const double* tp = tmS + ch * Tc * Tc;
                for (int r = 0; r < nrows; ++r) {
                    const short4 rw = rows[r];
                    const double* a = sp + rw.x * L.sw + rw.y;
                    const double* b = tp + rw.x * Tc + rw.y;
                    const int len = rw.z - rw.y;
                    double sum[BK_W];
#pragma unroll
                    for (int k = 0; k < BK_W; ++k) sum[k] = 0.0;
                    // sum += ti*or left to right (matcher.hpp:72-76)
#pragma unroll 4
                    for (int t = 0; t < len; ++t) {
                        const double bv = b[t];
#pragma unroll
                        for (int k = 0; k < BK_W; ++k) sum[k] = __dadd_rn(sum[k], __dmul_rn(a[base[k] + t], bv));
                    }
#pragma unroll
                    for (int k = 0; k < BK_W; ++k) acc[k] = __dadd_rn(acc[k], sum[k]);
                }
            }
#pragma unroll
            for (int k = 0; k < BK_W; ++k) {
                if (!ok[k]) continue;
                double ck = acc[k];
                int ci = pidx[k];
#pragma unroll
                for (int j = 0; j < kTcQ; ++j)
                    if (j < K && better(ck, ci, tk[j], tix[j])) {
                        const double t0 = tk[j];
                        const int t1 = tix[j];
                        tk[j] = ck;
                        tix[j] = ci;
                        ck = t0;
                        ci = t1;
                    }
            }
        }
        clk_comp += clock64() - c_cp;
    }
    // this CTA's top-K: K rounds of a block-wide arg-best over the per-thread lists
    double* lk = stg;
    int* li = reinterpret_cast<int*>(stg + BK_T * kTcQ);
#pragma unroll
    for (int j = 0; j < kTcQ; ++j) {
        lk[j * BK_T + tid] = tk[j];
        li[j * BK_T + tid] = tix[j];
    }
    int head = 0;
    for (int round = 0; round < K; ++round) {
        double bk = head < K ? lk[head * BK_T + tid] : -INFINITY;
        int bi = head < K ? li[head * BK_T + tid] : INT_MAX;
        int bt = tid;
        for (int o = 16; o > 0; o >>= 1) {
            const double ok2 = __shfl_xor_sync(0xffffffffu, bk, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
            if (better(ok2, oi, bk, bi)) {
                bk = ok2;
                bi = oi;
                bt = ot;
            }
        }
        if (lane == 0) {
            rk[wid] = bk;
            ri[wid] = bi;
            rp[wid] = bt;
        }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < BK_T / 32; ++w)
                if (better(rk[w], ri[w], bk, bi)) {
                    bk = rk[w];
                    bi = ri[w];
                    bt = rp[w];
                }
            tkey[round] = bk;
            tidx[round] = bi;
            shv[1] = bt;
        }
        __syncthreads();
        if (tid == shv[1]) ++head;
    }
    if (tid == 0) {
        double* gk = P.bulk_keys + (static_cast<size_t>(slot) * BK_SMAX + part) * kTcQ;
        int* gi = P.bulk_idx + (static_cast<size_t>(slot) * BK_SMAX + part) * kTcQ;
        for (int j = 0; j < K; ++j) {
            gk[j] = tkey[j];
            gi[j] = tidx[j];
        }
        if (P.stats) {
            atomicAdd(&P.stats[14], static_cast<unsigned long long>(clk_stage));
            atomicAdd(&P.stats[15], static_cast<unsigned long long>(clk_comp));
            atomicAdd(&P.stats[7], static_cast<unsigned long long>(clock64() - clk_start));
            if (rescored) atomicAdd(&P.stats[0], rescored);
        }
        __threadfence();
        shv[2] = atomicAdd(next + 1, 1);
    }
    __syncthreads();
    if (shv[2] != S - 1) return;  // not the last CTA of this placement
    // last CTA: merge the S lists (reference ranking), choose, paste
    __threadfence();
    const int nm = S * K;
    for (int e = tid; e < nm; e += BK_T) {
        const int p = e / K, j = e - p * K;
        mk[e] = __ldcg(P.bulk_keys + (static_cast<size_t>(slot) * BK_SMAX + p) * kTcQ + j);
        mi[e] = __ldcg(P.bulk_idx + (static_cast<size_t>(slot) * BK_SMAX + p) * kTcQ + j);
    }
    __syncthreads();
    int ntop = 0;
    if (wid == 0) {
        for (int round = 0; round < K; ++round) {
            double bk = -INFINITY;
            int bi = INT_MAX, bp = -1;
            for (int e = lane; e < nm; e += 32)
                if (mi[e] != INT_MAX && better(mk[e], mi[e], bk, bi)) {
                    bk = mk[e];
                    bi = mi[e];
                    bp = e;
                }
            for (int o = 16; o > 0; o >>= 1) {
                const double ok2 = __shfl_xor_sync(0xffffffffu, bk, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                const int op = __shfl_xor_sync(0xffffffffu, bp, o);
                if (better(ok2, oi, bk, bi)) {
                    bk = ok2;
                    bi = oi;
                    bp = op;
                }
            }
            if (bp < 0) break;
            if (lane == 0) {
                tkey[round] = bk;
                tidx[round] = bi;
                mi[bp] = INT_MAX;
            }
            __syncwarp();
            ntop = round + 1;
        }
        const int pos = choose_pick(P, jb, tidx, ntop, lane);
        if (lane == 0) {
            shv[3] = pos;
            next[0] = 0;  // reset the placement's counters for the next launch
            next[1] = 0;
            if (P.stats) atomicAdd(&P.stats[3], 1ull);
        }
    }
    __syncthreads();
    const int pos = shv[3];
    const int fr = (pos / P.out_w) << P.J, fc = (pos % P.out_w) << P.J;
    paste_job<BK_T>(P, jb, gj, fr, fc, tid);
    prep_dependents(P, jobs, jb, shv + 4);  // (misc + 304: free)
    if (tid == 0) {
        P.chosen[2 * gj] = fr;
        P.chosen[2 * gj + 1] = fc;
    }
    tl_mark(P.tl, 1);
}

// ----------------------------------------------------------- finalize ----

__global__ void hd_scatter_kernel(const int32_t* __restrict__ hd, int n_hd, uint8_t* plane, int ww) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_hd) plane[static_cast<size_t>(hd[3 * i]) * ww + hd[3 * i + 1]] = static_cast<uint8_t>(hd[3 * i + 2]);
}

// Hard-data overwrite with pre-overwrite mismatch count, then the crop to
// the simulation grid (simulator.hpp:506-515).
// Without a work grid the cell is read from the TI through the source-block
// map (every work block is a verbatim copy of the TI block it was last pasted
// from).
__global__ void finalize_kernel(const uint8_t* __restrict__ work, int wh, int ww,
                                const int32_t* __restrict__ src, int B, int J, int swc,
                                const uint8_t* __restrict__ ti, int ti_w, int wc,
                                const uint8_t* __restrict__ hd, int sg_h, int sg_w,
                                uint8_t* __restrict__ out, int* mism) {
    pdl_wait();
    const size_t n = static_cast<size_t>(sg_h) * sg_w;
    const int r = blockIdx.y;
    const uint8_t* g = work ? work + static_cast<size_t>(r) * wh * ww : nullptr;
    const int32_t* sm = src ? src + static_cast<size_t>(r) * (wh >> J) * swc : nullptr;
    int local = 0;
    for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int y = static_cast<int>(e / sg_w), x = static_cast<int>(e - static_cast<size_t>(y) * sg_w);
        uint8_t v;
        if (g) {
            v = g[static_cast<size_t>(y) * ww + x];
        } else {
            const int b = sm[static_cast<size_t>(y >> J) * swc + (x >> J)];
            const int by = b / wc, bx = b - by * wc;
            v = ti[static_cast<size_t>((by << J) + (y & (B - 1))) * ti_w + (bx << J) + (x & (B - 1))];
        }
        if (hd) {
            const uint8_t h = hd[static_cast<size_t>(y) * ww + x];
            if (h != kNoDatum) {
                local += v != h;
                v = h;
            }
        }
        out[static_cast<size_t>(r) * n + e] = v;
    }
    if (hd) {
        for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
        if ((threadIdx.x & 31) == 0 && local) atomicAdd(&mism[r], local);
    }
}

// Progressive finalize: band descriptors (realization, axis, lo, hi) in
// output coordinates -- axis 0: rows [lo, hi) x every column; axis 1: every
// row x columns [lo, hi).  A band is final once every placement covering it
// is done (run_simulation's checkpoints), so it is rebuilt and copied to the
// host while later waves still compute.
__global__ void finalize_band_kernel(const int4* __restrict__ bands, const uint8_t* __restrict__ work,
                                     int wh, int ww, const int32_t* __restrict__ src, int B, int J,
                                     int swc, const uint8_t* __restrict__ ti, int ti_w, int wc,
                                     const uint8_t* __restrict__ hd, int sg_h, int sg_w,
                                     uint8_t* __restrict__ out, int* mism, unsigned long long* tl) {
    tl_mark(tl, 2);
    pdl_wait();
    tl_mark(tl, 0);
    const int4 bd = bands[blockIdx.y];
    const int r = bd.x;
    const int rows = bd.y == 0 ? bd.w - bd.z : sg_h;  // (axis 2: a column band, copied whole later)
    const int cols = bd.y == 0 ? sg_w : bd.w - bd.z;
    const int y0 = bd.y == 0 ? bd.z : 0, x0 = bd.y == 0 ? 0 : bd.z;
    const size_t n = static_cast<size_t>(rows) * cols;
    const uint8_t* g = work ? work + static_cast<size_t>(r) * wh * ww : nullptr;
    const int32_t* sm = src ? src + static_cast<size_t>(r) * (wh >> J) * swc : nullptr;
    int local = 0;
    for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int y = y0 + static_cast<int>(e / cols), x = x0 + static_cast<int>(e % cols);
        uint8_t v;
        if (g) {
            v = g[static_cast<size_t>(y) * ww + x];
        } else {
            const int b = sm[static_cast<size_t>(y >> J) * swc + (x >> J)];
            const int by = b / wc, bx = b - by * wc;
            v = ti[static_cast<size_t>((by << J) + (y & (B - 1))) * ti_w + (bx << J) + (x & (B - 1))];
        }
        if (hd) {
            const uint8_t h = hd[static_cast<size_t>(y) * ww + x];
            if (h != kNoDatum) {
                local += v != h;
                v = h;
            }
        }
        out[(static_cast<size_t>(r) * sg_h + y) * sg_w + x] = v;
    }
    if (hd) {
        for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
        if ((threadIdx.x & 31) == 0 && local) atomicAdd(&mism[r], local);
    }
    tl_mark(tl, 1);
}

// min_cut_stitch as a stand-alone operator (the drop-in API surface).
__global__ void __launch_bounds__(256) min_cut_op_kernel(const uint8_t* __restrict__ ex,
                                                         const uint8_t* __restrict__ inc, int T,
                                                         int OV, int shape, int vleft, int htop,
                                                         uint8_t* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char mc_sm[];
    const SelLayout L = sel_layout(1, T, OV);
    uint8_t* exist = mc_sm + L.exist;
    uint8_t* outp = mc_sm + L.outp;
    int16_t* from = reinterpret_cast<int16_t*>(mc_sm + L.from);
    int* dp = reinterpret_cast<int*>(mc_sm + L.dp);
    int* seam = reinterpret_cast<int*>(mc_sm + L.seam);
    for (int e = threadIdx.x; e < T * T; e += blockDim.x) {
        exist[e] = ex[e];
        outp[e] = inc[e];
    }
    __syncthreads();
    min_cut_device(exist, outp, T, OV, shape, vleft, htop, from, dp, seam);
    for (int e = threadIdx.x; e < T * T; e += blockDim.x) out[e] = outp[e];
}

void op_min_cut_stitch(ccw_ctx* ctx, const uint8_t* existing, const uint8_t* incoming, int t,
                       int shape, int vleft, int htop, int overlap, uint8_t* out) {
    const size_t n = static_cast<size_t>(t) * t;
    const int ov = std::max(overlap, 1);
    uint8_t* d = ctx->ops_a.as<uint8_t>(3 * n);
    CCW_CUDA(cudaMemcpyAsync(d, existing, n, cudaMemcpyHostToDevice, ctx->stream));
    CCW_CUDA(cudaMemcpyAsync(d + n, incoming, n, cudaMemcpyHostToDevice, ctx->stream));
    const size_t smem = sel_layout(1, t, ov).total;
    if (smem > 227 * 1024) throw Fail(CCW_ERR_DIMENSION, "patch too large for the stitch kernel");
    CCW_CUDA(cudaFuncSetAttribute(min_cut_op_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    min_cut_op_kernel<<<1, 256, smem, ctx->stream>>>(d, d + n, t, ov, shape, vleft, htop, d + 2 * n);
    CCW_CUDA(cudaGetLastError());
    CCW_CUDA(cudaMemcpyAsync(out, d + 2 * n, n, cudaMemcpyDeviceToHost, ctx->stream));
    CCW_CUDA(cudaStreamSynchronize(ctx->stream));
}

// ------------------------------------------------------- host driver -----

namespace {

struct EventTimer {
    ccw_ctx* ctx;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ccf, sel;
    size_t next = 0;
    cudaEvent_t get() {
        if (next == ctx->ev_pool.size()) {
            cudaEvent_t e;
            CCW_CUDA(cudaEventCreate(&e));
            ctx->ev_pool.push_back(e);
        }
        return ctx->ev_pool[next++];
    }
};

double pair_ms(const std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v) {
    double t = 0;
    for (auto& p : v) {
        float ms = 0;
        cudaEventElapsedTime(&ms, p.first, p.second);
        t += ms;
    }
    return t;
}

}  // namespace

// NN maps of a TI for template Tc / overlap OVc (8 mask variants), cached on the TI.
const int32_t* ti_nnmap(ccw_ti* ti, int Tc, int OVc, cudaStream_t st) {
    const auto key = std::make_pair(Tc, OVc);
    auto it = ti->nnmap.find(key);
    if (it != ti->nnmap.end()) return it->second;
    const int out_h = ti->hc - Tc + 1, out_w = ti->wc - Tc + 1, npos = out_h * out_w;
    int32_t* m = static_cast<int32_t*>(cache_alloc(ti->device, sizeof(int32_t) * 8 * static_cast<size_t>(npos)));
    nn_map_kernel<<<dim3((npos + 255) / 256, 8), 256, 0, st>>>(ti->d_scr, ti->nscr, ti->mode, 1 << ti->J, ti->hc,
                                                             ti->wc, Tc, OVc, out_w, npos, m);
    CCW_CUDA(cudaGetLastError());
    ti->nnmap[key] = m;
    return m;
}

void run_simulation(ccw_ctx* ctx, ccw_ti* ti, const ccw_sim_config& cfg, const uint64_t* seeds,
                    int n_real, const int32_t* hd, int n_hd, uint8_t* d_out, uint8_t* h_out,
                    ccw_diag* diag, ccw_trace* traces) {
    const auto wall0 = std::chrono::steady_clock::now();
    cudaStream_t st = ctx->stream;
    const int T = cfg.template_size, OV = cfg.overlap, J = cfg.dwt_level, B = 1 << J;
    const int stride = T - OV;
    const int Tc = T >> J, OVc = OV >> J;
    const int out_h = ti->hc - Tc + 1, out_w = ti->wc - Tc + 1;
    const int npos = out_h * out_w;
    const int Kp = std::min(cfg.candidates, npos);
    if (Kp > KMAX)
        throw Fail(CCW_ERR_CONFIG, "candidates: more than 8192 effective candidates unsupported");
    const int reach = (T + stride - 1) / stride - 1;  // footprints overlap up to `reach` steps
    const int keymul = reach + 1;

    // ---- host schedule: raster paths, hard-data lattice, mt19937_64 draws.
    // A raster path (simulator.hpp:148-190) is one of 8 variants (origin x
    // major order); each realization draws its variant, then its per-placement
    // draws.  Jobs are written straight into pinned staging memory in
    // (group, wave, realization, placement) order.
    std::vector<Plan> variants(8);
    std::vector<char> have(8, 0);
    std::vector<int> vid(n_real);
    std::vector<std::mt19937_64> rngs(n_real);
    for (int r = 0; r < n_real; ++r) {
        rngs[r].seed(seeds[r]);
        const int origin = static_cast<int>(bounded(rngs[r], 4));
        const bool cm = bounded(rngs[r], 2) == 1;
        const int v = origin * 2 + (cm ? 1 : 0);
        if (!have[v]) {
            variants[v] = make_plan_from(cfg, origin, cm);
            have[v] = 1;
        }
        vid[r] = v;
    }
    int wh = 0, ww = 0, nlr = 0, nlc = 0;
    {
        const Plan& p0 = variants[vid[0]];  // geometry (identical for every variant)
        wh = p0.work_h;
        ww = p0.work_w;
        nlr = (wh - T) / stride + 1;
        nlc = (ww - T) / stride + 1;
    }
    // hard data per lattice cell (placements sit on the stride lattice for
    // every raster path): CSR lists of (cell in footprint, facies), so the
    // conditional choice reads only the cells that hold data
    std::vector<uint8_t> lattice_hd;
    std::vector<int32_t> hd_off;
    std::vector<uint32_t> hd_ent;
    if (hd && n_hd > 0) {
        const size_t ncell = static_cast<size_t>(nlr) * nlc;
        lattice_hd.assign(ncell, 0);
        hd_off.assign(ncell + 1, 0);
        auto each_cell = [&](int i, auto&& fn) {
            const int r = hd[3 * i], c = hd[3 * i + 1];
            const int qr0 = std::max(0, (r - T + 1 + stride - 1) / stride);
            const int qc0 = std::max(0, (c - T + 1 + stride - 1) / stride);
            for (int qr = qr0; qr <= std::min(nlr - 1, r / stride); ++qr)
                for (int qc = qc0; qc <= std::min(nlc - 1, c / stride); ++qc)
                    if (r >= qr * stride && r < qr * stride + T && c >= qc * stride && c < qc * stride + T)
                        fn(static_cast<size_t>(qr) * nlc + qc, r - qr * stride, c - qc * stride, hd[3 * i + 2]);
        };
        for (int i = 0; i < n_hd; ++i)
            each_cell(i, [&](size_t q, int, int, int) { ++hd_off[q + 1]; });
        for (size_t q = 0; q < ncell; ++q) {
            lattice_hd[q] = hd_off[q + 1] > 0;
            hd_off[q + 1] += hd_off[q];
        }
        hd_ent.resize(hd_off[ncell]);
        std::vector<int32_t> fill(hd_off.begin(), hd_off.end() - 1);
        for (int i = 0; i < n_hd; ++i)
            each_cell(i, [&](size_t q, int lr, int lc, int v) {
                hd_ent[fill[q]++] = (static_cast<uint32_t>(lr * T + lc) << 8) | static_cast<uint32_t>(v);
            });
    }
    int max_key = 0;
    for (int v = 0; v < 8; ++v)
        if (have[v]) max_key = std::max(max_key, keymul * (variants[v].n_outer - 1) + variants[v].n_inner - 1);
    const int nkeys = max_key + 1;
    // per-variant wave histograms
    std::vector<std::vector<int>> vhist(8);
    for (int v = 0; v < 8; ++v)
        if (have[v]) {
            vhist[v].assign(nkeys, 0);
            const Plan& p = variants[v];
            for (size_t k = 0; k < p.tops.size(); ++k) ++vhist[v][keymul * p.outer_idx[k] + p.inner_idx[k]];
        }

    // Realizations are split into G independent groups, each on its own
    // stream, so one group's latency-bound select overlaps another group's
    // tensor-core screen.  Within a group, waves run in order.
    int G = std::max(1, std::min(n_real, 2));
    if (const char* e = getenv("CCW_GROUPS")) G = std::max(1, std::min(n_real, atoi(e)));
    auto group_of = [&](int r) { return static_cast<int>(static_cast<int64_t>(r) * G / n_real); };
    std::vector<size_t> bucket(static_cast<size_t>(G) * nkeys + 1, 0);
    size_t total_jobs = 0;
    for (int r = 0; r < n_real; ++r) {
        const size_t g = group_of(r);
        for (int k = 0; k < nkeys; ++k) bucket[g * nkeys + k + 1] += vhist[vid[r]][k];
        total_jobs += variants[vid[r]].tops.size();
    }
    for (size_t i = 1; i < bucket.size(); ++i) bucket[i] += bucket[i - 1];
    std::vector<std::vector<size_t>> wave_off(G);  // per group, absolute offsets into flat
    size_t max_wave = 1;
    for (int g = 0; g < G; ++g) {
        for (int k = 0; k <= nkeys; ++k) wave_off[g].push_back(bucket[static_cast<size_t>(g) * nkeys + std::min(k, nkeys)]);
        for (int k = 0; k < nkeys; ++k) max_wave = std::max(max_wave, wave_off[g][k + 1] - wave_off[g][k]);
    }
    // each realization's first slot in every wave bucket
    std::vector<size_t> roff(static_cast<size_t>(n_real) * nkeys);
    {
        std::vector<size_t> fill(bucket.begin(), bucket.end() - 1);
        for (int r = 0; r < n_real; ++r) {
            const size_t g = group_of(r);
            for (int k = 0; k < nkeys; ++k) {
                roff[static_cast<size_t>(r) * nkeys + k] = fill[g * nkeys + k];
                fill[g * nkeys + k] += vhist[vid[r]][k];
            }
        }
    }
    Job* flat = static_cast<Job*>(ctx->h_stage.get(sizeof(Job) * total_jobs));
    auto build_one = [&](int r) {
        std::mt19937_64& rng = rngs[r];
        const Plan& p = variants[vid[r]];
        size_t* off = roff.data() + static_cast<size_t>(r) * nkeys;
        const int cnt = static_cast<int>(p.tops.size());
        // flat index of every placement (in placement order within each wave bucket)
        std::vector<int32_t> fi(cnt);
        {
            std::vector<size_t> o2(off, off + nkeys);
            for (int k = 0; k < cnt; ++k) fi[k] = static_cast<int32_t>(o2[keymul * p.outer_idx[k] + p.inner_idx[k]]++);
        }
        const int ni = p.n_inner, no = p.n_outer;
        for (int k = 0; k < cnt; ++k) {
            Job jb;
            {  // raster neighbours (k = o * n_inner + i): next-wave readers, previous-wave writers
                const int o = p.outer_idx[k], i = p.inner_idx[k];
                jb.dep0 = i + 1 < ni ? fi[k + 1] : -1;
                jb.dep1 = (o + 1 < no && i >= 1) ? fi[k + ni - 1] : -1;
                jb.ndep = (i >= 1 ? 1 : 0) + (o >= 1 && i + 1 < ni ? 1 : 0);
            }
            jb.real = r;
            jb.place = k;
            jb.top = p.tops[k];
            jb.left = p.lefts[k];
            jb.shape = p.shapes[k];
            jb.vleft = p.vertical_on_left();
            jb.htop = p.horizontal_on_top();
            jb.pick = 0;
            jb.fr = jb.fc = 0;
            if (jb.shape == kNone) {  // simulator.hpp:450-453
                jb.fr = static_cast<int>(bounded(rng, static_cast<uint64_t>((ti->h - T) / B + 1))) * B;
                jb.fc = static_cast<int>(bounded(rng, static_cast<uint64_t>((ti->w - T) / B + 1))) * B;
            } else {
                const bool cond = !lattice_hd.empty() &&
                                  lattice_hd[static_cast<size_t>(jb.top / stride) * nlc + jb.left / stride];
                jb.pick = cond ? -1 : static_cast<int>(bounded(rng, static_cast<uint64_t>(Kp)));
            }
            flat[off[keymul * p.outer_idx[k] + p.inner_idx[k]]++] = jb;
        }
    };
    ctx->pool.run(n_real, build_one);
    const double host_prep_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();

    // ---- exactness guard for the fp32 screen
    const double maxw = ti->mode == 0 ? B : static_cast<double>(ti->F - 1) * B;
    const double mask_cells = static_cast<double>(Tc) * OVc + static_cast<double>(Tc - OVc) * OVc;
    const bool use_screen = cfg.scoring == 0 && ti->nscr > 0;
    // normalized scoring: screened on the int8 tensor-core GEMM when it applies
    // (otherwise every window is rescored in fp64)
    bool norm_screen = cfg.scoring == 1 && ti->nscr > 0 && !getenv("CCW_NO_NORM_SCREEN") &&
                       mask_cells * ti->nch * maxw * maxw * maxw * maxw < 2147483647.0;
    if (use_screen && mask_cells * maxw * maxw * std::max(1, ti->nscr) >= 16777216.0)
        throw Fail(CCW_ERR_CONFIG, "configuration exceeds the exact fp32 screen range (mask*B^2 >= 2^24)");

    // ---- device buffers
    Job* d_jobs = ctx->jobs.as<Job>(total_jobs);
    CCW_CUDA(cudaMemcpyAsync(d_jobs, flat, sizeof(Job) * total_jobs, cudaMemcpyHostToDevice, st));
    const size_t plane = static_cast<size_t>(wh) * ww;
    // the work grid exists only with min-cut (seams read the grid); otherwise
    // the source-block map is the realization until finalize
    uint8_t* d_work = nullptr;
    if (cfg.min_cut) {
        d_work = ctx->work.as<uint8_t>(plane * n_real);
        CCW_CUDA(cudaMemsetAsync(d_work, 0, plane * n_real, st));
    }
    uint8_t* d_hd = nullptr;
    const int32_t* P_hd_off = nullptr;
    const uint32_t* P_hd_ent = nullptr;
    if (hd && n_hd > 0) {
        d_hd = ctx->hd.as<uint8_t>(plane);
        CCW_CUDA(cudaMemsetAsync(d_hd, kNoDatum, plane, st));
        int32_t* d_hdl = reinterpret_cast<int32_t*>(ctx->ops_e.get(sizeof(int32_t) * 3 * n_hd));
        CCW_CUDA(cudaMemcpyAsync(d_hdl, hd, sizeof(int32_t) * 3 * n_hd, cudaMemcpyHostToDevice, st));
        hd_scatter_kernel<<<(n_hd + 255) / 256, 256, 0, st>>>(d_hdl, n_hd, d_hd, ww);
        CCW_CUDA(cudaGetLastError());
        int32_t* d_off = ctx->hdoff.as<int32_t>(hd_off.size());
        uint32_t* d_ent = ctx->hdent.as<uint32_t>(std::max<size_t>(1, hd_ent.size()));
        CCW_CUDA(cudaMemcpyAsync(d_off, hd_off.data(), sizeof(int32_t) * hd_off.size(), cudaMemcpyHostToDevice, st));
        if (!hd_ent.empty())
            CCW_CUDA(cudaMemcpyAsync(d_ent, hd_ent.data(), sizeof(uint32_t) * hd_ent.size(),
                                     cudaMemcpyHostToDevice, st));
        P_hd_off = d_off;
        P_hd_ent = d_ent;
    }
    const int sld = (npos + 3) & ~3;  // (score rows exist only for the block-select path)
    const size_t score_budget = (static_cast<size_t>(512) << 20) / G;
    const size_t maxj = std::max<size_t>(1, std::min<size_t>(max_wave, score_budget / (sizeof(int32_t) * sld)));
    int32_t* d_scores = ctx->scores.as<int32_t>(G * maxj * sld);
    int32_t* d_wts = ctx->wts.as<int32_t>(G * maxj * std::max(ti->nscr, 1) * Tc * Tc);
    // prep outputs (template, screen weights) have two parity halves: with the
    // fused OR prep, wave w's select writes wave w+1's half while wave w reads its own
    double* d_tm = ctx->tm64.as<double>(2 * G * maxj * ti->nch * Tc * Tc);
    int32_t* d_chosen = ctx->chosen.as<int32_t>(2 * total_jobs);
    uint8_t* d_pasted = traces ? ctx->pasted.as<uint8_t>(total_jobs * T * T) : nullptr;
    int* d_mism = ctx->mism.as<int>(n_real);
    CCW_CUDA(cudaMemsetAsync(d_mism, 0, sizeof(int) * n_real, st));

    SimParams P{};
    P.ti = ti->d_codes;
    P.ti64 = ti->d_ti64;
    P.tiscr = ti->d_scr;
    P.ti_h = ti->h;
    P.ti_w = ti->w;
    P.hc = ti->hc;
    P.wc = ti->wc;
    P.F = ti->F;
    P.J = J;
    P.mode = ti->mode;
    P.nch = ti->nch;
    P.nscr = ti->nscr;
    P.T = T;
    P.OV = OV;
    P.Tc = Tc;
    P.OVc = OVc;
    P.B = B;
    P.out_h = out_h;
    P.out_w = out_w;
    P.npos = npos;
    P.K = Kp;
    P.scoring = cfg.scoring;
    P.min_cut = cfg.min_cut;
    P.work = d_work;
    P.wh = wh;
    P.ww = ww;
    P.hd = d_hd;
    P.hd_off = P_hd_off;
    P.hd_ent = P_hd_ent;
    P.lat_nlc = nlc;
    P.stride = stride;
    P.sld = sld;
    P.chosen = d_chosen;
    P.pasted = d_pasted;

    // screen variant: tcgen05 int8 implicit GEMM when every operand fits int8
    const int maxv = ti->mode == 0 ? B * B : (ti->F - 1) * B * B;
    const bool tc_ok = (use_screen || norm_screen) && maxv <= 127;
    if (ctx->ccf_variant == 2 && use_screen && !tc_ok)
        throw Fail(CCW_ERR_CONFIG, "tcgen05 int8 screen needs block statistics <= 127");
    const bool use_tc = tc_ok && ctx->ccf_variant != 1;
    norm_screen = norm_screen && use_tc;  // the normalized screen rides on the int8 GEMM only
    const bool any_screen = use_screen || norm_screen;
    const int kpad = tc_kpad(ti->nscr, Tc);
    const int ntiles = tc_tiles(npos);
    const int8_t* d_x = nullptr;
    int8_t* d_w8 = nullptr;
    int32_t* d_tmax = nullptr;
    if (use_tc) {
        d_x = ti_im2col(ti, Tc, st);
        d_w8 = ctx->wts8.as<int8_t>(2 * G * maxj * kpad);
        d_tmax = ctx->summary.as<int32_t>(G * maxj * ntiles);
    }
    int32_t* d_cjob = nullptr;
    if (norm_screen) {
        P.nnmap = ti_nnmap(ti, Tc, OVc, st);
        d_cjob = ctx->cjob.as<int32_t>(G * maxj);
    }
    unsigned long long* d_stats = ctx->stats.as<unsigned long long>(16);
    CCW_CUDA(cudaMemsetAsync(d_stats, 0, 16 * sizeof(unsigned long long), st));
    // source-block map (fast or_prep), valid whenever pastes are verbatim TI blocks
    const int swc = ww / B;
    int32_t* d_src = nullptr;
    if (!cfg.min_cut) {
        d_src = ctx->src.as<int32_t>(static_cast<size_t>(n_real) * (wh / B) * swc);
    }
    P.src = d_src;
    P.swc = swc;
    const bool warp_select = use_tc && Kp <= kTcQ && !cfg.min_cut && cfg.scoring == 0 &&
                             ti->nch * Tc <= FS_MAXG && Tc <= PK_MAXTC;
    P.kpad = kpad;
    P.ntiles = ntiles;
    P.stats = d_stats;
    P.im2col = d_x;
    // bulk tie select: largest window block whose apex tile fits the shared-memory budget
    size_t bulk_smem = 0;
    if (warp_select && !getenv("CCW_NOBULK")) {
        constexpr size_t kBudget = 200 * 1024;
        for (int by = std::min(out_w, 256); by >= 8 && !bulk_smem; by /= 2) {
            int bx = std::min(out_h, 64);
            while (bx > 1 && bulk_layout(ti->nch, Tc, bx, by).total > kBudget) --bx;
            if (bulk_layout(ti->nch, Tc, bx, by).total <= kBudget && (bx >= 4 || bx == out_h)) {
                P.bulk_bx = bx;
                P.bulk_by = by;
                bulk_smem = bulk_layout(ti->nch, Tc, bx, by).total;
            }
        }
    }
    const auto bulk_key = std::make_tuple(ti->key, Tc, OVc, Kp, T);
    const bool bulk_launch = bulk_smem && !ctx->bulk_off.count(bulk_key);
    int* d_defer = bulk_launch ? ctx->defer.as<int>(G * maxj) : nullptr;
    int bulk_S = 1;
    if (bulk_launch) {
        // CTAs per deferred placement: enough to cover the SMs when a wave
        // chunk defers a third of its placements
        bulk_S = std::max(1, std::min(BK_SMAX, 3 * tc_num_sms() / std::max<int>(1, static_cast<int>(std::min<size_t>(maxj, max_wave)))));
        int* d_bsync = ctx->bulk_sync.as<int>(2 * G * maxj);
        CCW_CUDA(cudaMemsetAsync(d_bsync, 0, sizeof(int) * 2 * G * maxj, st));
        P.bulk_sync = d_bsync;
        P.bulk_keys = ctx->bulk_keys.as<double>(G * maxj * BK_SMAX * kTcQ);
        P.bulk_idx = ctx->bulk_idx.as<int>(G * maxj * BK_SMAX * kTcQ);
    }
    if (bulk_smem)
        CCW_CUDA(cudaFuncSetAttribute(select_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(bulk_smem)));
    std::vector<SimParams> GP(G, P);
    for (int g = 0; g < G; ++g) {
        GP[g].scores = d_scores + g * maxj * sld;
        GP[g].wts = d_wts + g * maxj * std::max(ti->nscr, 1) * Tc * Tc;
        GP[g].tm64 = d_tm + g * maxj * ti->nch * Tc * Tc;
        GP[g].wts8 = d_w8 ? d_w8 + g * maxj * kpad : nullptr;
        GP[g].tmax = d_tmax ? d_tmax + g * maxj * ntiles : nullptr;
        GP[g].cjob = d_cjob ? d_cjob + g * maxj : nullptr;
        GP[g].defer = d_defer ? d_defer + g * maxj : nullptr;
        if (d_defer) {
            GP[g].bulk_sync = P.bulk_sync + 2 * g * maxj;
            GP[g].bulk_keys = P.bulk_keys + g * maxj * BK_SMAX * kTcQ;
            GP[g].bulk_idx = P.bulk_idx + g * maxj * BK_SMAX * kTcQ;
        }
    }

    // fused OR prep (opt-in, CCW_FUSE_PREP=1): applies with the fast select,
    // one-step wavefront neighbours (keymul 2) and waves that fit one launch
    // (the slot of a dependent is its index in the next wave).  Measured r1:
    // slower (config 1 5.2 -> 5.5 ms, config 2 39 -> 45 ms) -- the completing
    // CTA's preps lengthen the select's critical path by more than the
    // separate, fully parallel prep kernel costs.
    const bool fuse_prep = warp_select && keymul == 2 && max_wave <= maxj && d_src &&
                           getenv("CCW_FUSE_PREP") != nullptr;
    int* d_depcnt = nullptr;
    if (fuse_prep) {
        d_depcnt = ctx->depcnt.as<int>(G * maxj);
        CCW_CUDA(cudaMemsetAsync(d_depcnt, 0, sizeof(int) * G * maxj, st));
    }
    // per (group, parity) parameter sets
    std::vector<std::array<SimParams, 2>> GPP(G);
    const size_t tm_half = G * maxj * ti->nch * Tc * Tc, w8_half = G * maxj * kpad;
    for (int g = 0; g < G; ++g)
        for (int par = 0; par < 2; ++par) {
            SimParams& Q = GPP[g][par];
            Q = GP[g];
            Q.tm64 = GP[g].tm64 + par * tm_half;
            Q.wts8 = GP[g].wts8 ? GP[g].wts8 + par * w8_half : nullptr;
            if (fuse_prep) {
                Q.depcnt = d_depcnt + g * maxj;
                Q.n_tm64 = GP[g].tm64 + (1 - par) * tm_half;
                Q.n_wts8 = GP[g].wts8 ? GP[g].wts8 + (1 - par) * w8_half : nullptr;
                Q.n_cjob = nullptr;  // (raw scoring only)
            }
        }

    const size_t ccf_smem = ccf_smem_bytes(Tc, ti->nscr);
    const size_t sel_smem = sel_layout(Kp, T, OV, ti->nch, Tc, cfg.scoring == 1).total;
    if (ccf_smem > 227 * 1024 || sel_smem > 227 * 1024)
        throw Fail(CCW_ERR_CONFIG, "configuration exceeds the per-CTA shared-memory budget");
    CCW_CUDA(cudaFuncSetAttribute(ccf_direct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(ccf_smem)));
    CCW_CUDA(cudaFuncSetAttribute(select_paste_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sel_smem)));

    unsigned long long* d_probe = nullptr;
    if (getenv("CCW_TC_PROBE")) {
        d_probe = reinterpret_cast<unsigned long long*>(ctx->ops_d.get(8 * sizeof(unsigned long long)));
        CCW_CUDA(cudaMemsetAsync(d_probe, 0, 8 * sizeof(unsigned long long), st));
    }
    tc_probe_buffer = d_probe;
    std::vector<std::array<TcPlan, 2>> tcplans(G);
    if (use_tc)
        for (int g = 0; g < G; ++g)
            for (int par = 0; par < 2; ++par)
                tcplans[g][par] = plan_ccf_tc(GPP[g][par].wts8, static_cast<int>(maxj), d_x, npos, kpad);
    // group streams, forked from / joined back to the context stream
    while (static_cast<int>(ctx->copy_streams.size()) < G) {  // one per group: final copies overlap
        cudaStream_t s3;
        CCW_CUDA(cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking));
        ctx->copy_streams.push_back(s3);
    }
    while (static_cast<int>(ctx->gstreams.size()) < G) {
        cudaStream_t s2;
        CCW_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        ctx->gstreams.push_back(s2);
    }
    // timing experiments only (results are wrong when set): skip a kernel class
    const char* skip_env = getenv("CCW_DEBUG_SKIP");
    const std::string skip = skip_env ? skip_env : "";
    const bool skip_prep = skip.find("prep") != std::string::npos;
    const bool skip_ccf = skip.find("ccf") != std::string::npos;
    const bool skip_sel = skip.find("sel") != std::string::npos;
    EventTimer tm{ctx, {}, {}, 0};
    cudaEvent_t ev0 = tm.get(), ev1 = tm.get();
    CCW_CUDA(cudaEventRecord(ev0, st));
    for (int g = 0; g < G; ++g) CCW_CUDA(cudaStreamWaitEvent(ctx->gstreams[g], ev0, 0));
    // ---- progressive output (host results): bands of every realization that
    // no remaining placement covers are finalized and copied back at a few
    // checkpoint waves, overlapping the copy with the remaining waves
    uint8_t* fin = d_out ? d_out : ctx->out.as<uint8_t>(static_cast<size_t>(cfg.sg_height) * cfg.sg_width * n_real);
    const size_t out_bytes = static_cast<size_t>(cfg.sg_height) * cfg.sg_width * n_real;
    // device->host copies need page-locked memory to run asynchronously: a
    // pageable destination gets a pinned staging buffer, copied out at the end
    uint8_t* h_dst = h_out;
    if (h_out) {
        cudaPointerAttributes pa{};
        const bool pinned = cudaPointerGetAttributes(&pa, h_out) == cudaSuccess && pa.type == cudaMemoryTypeHost;
        cudaGetLastError();
        if (!pinned) h_dst = static_cast<uint8_t*>(ctx->h_out_stage.get(out_bytes));
    }
    const bool stream_out = h_out && !getenv("CCW_NO_STREAM_OUT");
    std::vector<int4> bands;                                   // all checkpoints, in launch order
    std::vector<std::vector<std::pair<int, std::pair<size_t, size_t>>>> band_at(G);  // per group: (wave, [off, off+n))
    if (stream_out) {
        int nck = 4;
        if (const char* e = getenv("CCW_STREAM_BANDS")) nck = std::max(1, atoi(e));
        const int delta = std::max(1, (max_key + 1 + nck - 1) / nck);
        // column-major raster paths free whole columns: strided copies, slower
        // per byte -- emitted whole at the last wave (CCW_STREAM_COLS=1: every
        // other checkpoint; measured slower end to end, r1)
        const char* ce = getenv("CCW_STREAM_COLS");
        const bool stream_cols = ce && atoi(ce) != 0;  // measured slower (r1): off by default
        std::vector<int> done(n_real, 0);  // raster-outer extent already emitted
        int ck = 0;
        for (int w = 0; w <= max_key; ++w) {
            if ((w + 1) % delta != 0 && w != max_key) continue;
            const bool col_ck = w == max_key || (stream_cols && (ck & 1));
            ++ck;
            for (int g = 0; g < G; ++g) {
                const size_t off = bands.size();
                for (int r = 0; r < n_real; ++r) {
                    if (group_of(r) != g) continue;
                    const Plan& p = variants[vid[r]];
                    // column bands: strided copies at col_ck checkpoints (CCW_STREAM_COLS,
                    // axis 1), or finalized on the device at every checkpoint and the whole
                    // realization copied at the last wave (axis 2: the final band, possibly
                    // empty, carries the copy)
                    if (p.column_major && stream_cols && !col_ck) continue;
                    const int axis = !p.column_major ? 0 : (stream_cols ? 1 : 2);
                    const bool asc = axis == 0 ? (p.origin == CCW_TOP_LEFT || p.origin == CCW_TOP_RIGHT)
                                               : (p.origin == CCW_TOP_LEFT || p.origin == CCW_BOTTOM_LEFT);
                    const int extent = axis == 0 ? wh : ww, sg_ext = axis == 0 ? cfg.sg_height : cfg.sg_width;
                    int O = w >= p.n_inner - 1 ? (w - (p.n_inner - 1)) / keymul : -1;
                    O = std::min(O, p.n_outer - 1);
                    const int U = (w == max_key || O == p.n_outer - 1) ? extent : (O + 1) * stride;
                    const bool carry = axis == 2 && w == max_key;
                    if (U <= done[r] && !carry) continue;
                    int lo = asc ? done[r] : extent - U, hi = asc ? U : extent - done[r];
                    done[r] = std::max(done[r], U);
                    lo = std::max(lo, 0);
                    hi = std::min(hi, sg_ext);
                    if (hi > lo || carry) bands.push_back(make_int4(r, axis, lo, std::max(lo, hi)));
                }
                if (bands.size() > off) band_at[g].push_back({w, {off, bands.size()}});
            }
        }
    }
    int4* d_bands = nullptr;
    if (!bands.empty()) {
        d_bands = reinterpret_cast<int4*>(ctx->ops_b.get(sizeof(int4) * bands.size()));
        CCW_CUDA(cudaMemcpyAsync(d_bands, bands.data(), sizeof(int4) * bands.size(), cudaMemcpyHostToDevice, st));
    }
    std::vector<size_t> band_next(G, 0);
    struct CopyMark {
        int w, g;
        cudaEvent_t ev;
    };
    std::vector<CopyMark> copy_marks;

    // debug timeline: [resident, past-wait, end] per launch
    const bool want_tl = getenv("CCW_TIMELINE") != nullptr;
    std::vector<std::array<int, 3>> tl_tag;  // (wave, group, kind 0 prep / 1 ccf / 2 select)
    unsigned long long* d_tl = nullptr;
    const size_t tl_cap = static_cast<size_t>(max_key + 1) * G * 4 * 8;
    if (want_tl) {
        d_tl = reinterpret_cast<unsigned long long*>(ctx->ops_c.get(tl_cap * 4 * sizeof(unsigned long long)));
        std::vector<unsigned long long> init(tl_cap * 4);
        for (size_t i = 0; i < tl_cap; ++i) {
            init[4 * i] = ~0ull;
            init[4 * i + 1] = 0;
            init[4 * i + 2] = ~0ull;
            init[4 * i + 3] = 0;
        }
        CCW_CUDA(cudaMemcpy(d_tl, init.data(), init.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice));
    }
    auto tl_next = [&](int w, int g, int kind) -> unsigned long long* {
        if (!d_tl || tl_tag.size() >= tl_cap) return nullptr;
        tl_tag.push_back({w, g, kind});
        return d_tl + 4 * (tl_tag.size() - 1);
    };
    int64_t launches = 0, ccf_launches = 0;
    double ccf_flop = 0, ccf_flop_ref = 0, ccf_mma_flop = 0;
    const dim3 ccf_grid_xy((out_w + CCF_TY - 1) / CCF_TY, (out_h + CCF_TX - 1) / CCF_TX);
    for (int w = 0; w <= max_key; ++w) {
        for (int g = 0; g < G; ++g) {
            cudaStream_t gs = ctx->gstreams[g];
            const int par = fuse_prep ? (w & 1) : 0;
            SimParams Q = GPP[g][par];
            Q.next_j0 = static_cast<int>(wave_off[g][std::min(w + 1, nkeys)]);
            for (size_t j0 = wave_off[g][w]; j0 < wave_off[g][w + 1]; j0 += maxj) {
                const int nj = static_cast<int>(std::min(maxj, wave_off[g][w + 1] - j0));
                const bool first_wave = flat[j0].shape == kNone;
                if (!first_wave) {
                    Q.tl = tl_next(w, g, 0);
                    if (!skip_prep && !fuse_prep) {  // (fused: prepared by the previous wave's select)
                        if (d_src)
                            launch_pdl(or_prep_src_kernel, dim3(nj), dim3(128), 0, gs, Q,
                                       static_cast<const Job*>(d_jobs), static_cast<int>(j0));
                        else
                            launch_pdl(or_prep_kernel, dim3(nj), dim3(128), 0, gs, Q,
                                       static_cast<const Job*>(d_jobs), static_cast<int>(j0));
                        ++launches;
                    }
                    if (any_screen) {
                        cudaEvent_t a = nullptr, b = nullptr;
                        if (ctx->profiling) {
                            a = tm.get();
                            b = tm.get();
                            CCW_CUDA(cudaEventRecord(a, gs));
                        }
                        if (skip_ccf) {
                        } else if (use_tc) {
                            launch_ccf_tc(tcplans[g][par], npos, sld, kpad, nj, Q.scores, Q.tmax, gs,
                                          tl_next(w, g, 1));
                        } else {
                            launch_pdl(ccf_direct_kernel, dim3(ccf_grid_xy.x, ccf_grid_xy.y, nj),
                                       dim3(CCF_THREADS), ccf_smem, gs, Q,
                                       static_cast<const Job*>(d_jobs), static_cast<int>(j0));
                        }
                        ++launches;
                        ++ccf_launches;
                        if (ctx->profiling) {
                            CCW_CUDA(cudaEventRecord(b, gs));
                            tm.ccf.push_back({a, b});
                        }
                        ccf_mma_flop += 2.0 * kpad * static_cast<double>(npos) * nj;
                        for (int q = 0; q < nj; ++q) {
                            const int sh = flat[j0 + q].shape;
                            const double m = sh == kL ? mask_cells : static_cast<double>(Tc) * OVc;
                            ccf_flop += 2.0 * ti->nscr * npos * m;
                            ccf_flop_ref += 2.0 * ti->nch * npos * m;
                        }
                    }
                }
                cudaEvent_t a = nullptr, b = nullptr;
                if (ctx->profiling) {
                    a = tm.get();
                    b = tm.get();
                    CCW_CUDA(cudaEventRecord(a, gs));
                }
                Q.tl = tl_next(w, g, 2);
                if (skip_sel && !first_wave) {
                } else if (warp_select || (first_wave && !cfg.min_cut)) {
                    const Job* dj = d_jobs;
                    launch_pdl(select_fast_kernel, dim3(nj), dim3(FS_T), 0, gs, Q, dj,
                               static_cast<int>(j0), nj);
                    if (Q.defer && !first_wave) {
                        Q.tl = tl_next(w, g, 5);
                        launch_pdl(select_bulk_kernel, dim3(bulk_S, nj), dim3(BK_T), bulk_smem, gs, Q, dj,
                                   static_cast<int>(j0), nj, bulk_S);
                        ++launches;
                    }
                }
                else
                    launch_pdl(select_paste_kernel, dim3(nj), dim3(SEL_T), sel_smem, gs, Q,
                               static_cast<const Job*>(d_jobs), static_cast<int>(j0),
                               use_screen ? 1 : (norm_screen ? 2 : 0));
                ++launches;
                if (ctx->profiling) {
                    CCW_CUDA(cudaEventRecord(b, gs));
                    tm.sel.push_back({a, b});
                }
            }
            if (band_next[g] < band_at[g].size() && band_at[g][band_next[g]].first == w) {
                const auto rng = band_at[g][band_next[g]++].second;
                const int nb = static_cast<int>(rng.second - rng.first);
                size_t most = 1;  // cells of the largest band: enough CTAs to cover it
                for (size_t q = rng.first; q < rng.second; ++q)
                    most = std::max(most, static_cast<size_t>(bands[q].w - bands[q].z) *
                                              (bands[q].y == 0 ? cfg.sg_width : cfg.sg_height));
                const int bxb = static_cast<int>(std::min<size_t>((most + 255) / 256, 1024));
                // final bands are never written again: rebuild and copy them on the copy
                // stream, off the group's critical path
                cudaEvent_t be = tm.get();
                CCW_CUDA(cudaEventRecord(be, gs));
                CCW_CUDA(cudaStreamWaitEvent(ctx->copy_streams[g], be, 0));
                launch_pdl(finalize_band_kernel, dim3(bxb, nb), dim3(256), 0, ctx->copy_streams[g],
                           static_cast<const int4*>(d_bands + rng.first), static_cast<const uint8_t*>(d_work),
                           wh, ww, static_cast<const int32_t*>(d_src), B, J, swc,
                           static_cast<const uint8_t*>(ti->d_codes), ti->w, ti->wc,
                           static_cast<const uint8_t*>(d_hd), cfg.sg_height, cfg.sg_width, fin, d_mism, tl_next(w, g, 4));
                ++launches;
                // copies straight into the caller's buffer; adjacent ranges merged
                const size_t n = static_cast<size_t>(cfg.sg_height) * cfg.sg_width;
                size_t o0 = 0, o1 = 0;
                auto flush = [&] {
                    if (o1 > o0)
                        CCW_CUDA(cudaMemcpyAsync(h_dst + o0, fin + o0, o1 - o0, cudaMemcpyDeviceToHost,
                                                 ctx->copy_streams[g]));
                    o0 = o1 = 0;
                };
                for (size_t q = rng.first; q < rng.second; ++q) {
                    const int4 bd = bands[q];
                    const size_t base = static_cast<size_t>(bd.x) * n;
                    if (bd.y == 2 && w != max_key) continue;  // device-only column band
                    const bool full = (bd.y == 0 && bd.z == 0 && bd.w == cfg.sg_height) ||
                                      (bd.y == 1 && bd.z == 0 && bd.w == cfg.sg_width) || bd.y == 2;
                    if (bd.y == 1 && !full) {  // a column band: one strided copy
                        flush();
                        CCW_CUDA(cudaMemcpy2DAsync(h_dst + base + bd.z, cfg.sg_width, fin + base + bd.z,
                                                   cfg.sg_width, bd.w - bd.z, cfg.sg_height,
                                                   cudaMemcpyDeviceToHost, ctx->copy_streams[g]));
                        continue;
                    }
                    const size_t a0 = full ? base : base + static_cast<size_t>(bd.z) * cfg.sg_width;
                    const size_t a1 = full ? base + n : base + static_cast<size_t>(bd.w) * cfg.sg_width;
                    if (a0 != o1) flush();
                    if (o1 == 0) o0 = a0;
                    o1 = a1;
                }
                flush();
                if (want_tl) {  // debug: copy-stream progress per checkpoint
                    cudaEvent_t ce = tm.get();
                    CCW_CUDA(cudaEventRecord(ce, ctx->copy_streams[g]));
                    copy_marks.push_back({w, g, ce});
                }
            }
        }
    }
    CCW_CUDA(cudaGetLastError());
    for (int g = 0; g < G; ++g) {
        cudaEvent_t e = tm.get();
        CCW_CUDA(cudaEventRecord(e, ctx->gstreams[g]));
        CCW_CUDA(cudaStreamWaitEvent(st, e, 0));
    }
    if (stream_out)
        for (int g = 0; g < G; ++g) {
            cudaEvent_t e = tm.get();
            CCW_CUDA(cudaEventRecord(e, ctx->copy_streams[g]));
            CCW_CUDA(cudaStreamWaitEvent(st, e, 0));
        }

    // ---- finalize (device results, or host results without streaming)
    if (!stream_out) {
        const size_t n = static_cast<size_t>(cfg.sg_height) * cfg.sg_width;
        const int bx = static_cast<int>(std::min<size_t>((n + 255) / 256, 1024));
        finalize_kernel<<<dim3(bx, n_real), 256, 0, st>>>(d_work, wh, ww, d_src, B, J, swc, ti->d_codes,
                                                          ti->w, ti->wc, d_hd, cfg.sg_height,
                                                          cfg.sg_width, fin, d_mism);
        ++launches;
        CCW_CUDA(cudaGetLastError());
    }
    CCW_CUDA(cudaEventRecord(ev1, st));
    if (h_out && !stream_out)
        CCW_CUDA(cudaMemcpyAsync(h_dst, fin, out_bytes, cudaMemcpyDeviceToHost, st));
    unsigned long long stats[16] = {0};
    CCW_CUDA(cudaMemcpyAsync(stats, d_stats, sizeof(stats), cudaMemcpyDeviceToHost, st));
    std::vector<int> mism(n_real, 0);
    CCW_CUDA(cudaMemcpyAsync(mism.data(), d_mism, sizeof(int) * n_real, cudaMemcpyDeviceToHost, st));
    std::vector<int32_t> chosen;
    std::vector<uint8_t> pasted;
    if (traces) {
        chosen.resize(2 * total_jobs);
        CCW_CUDA(cudaMemcpyAsync(chosen.data(), d_chosen, sizeof(int32_t) * chosen.size(),
                                 cudaMemcpyDeviceToHost, st));
        pasted.resize(total_jobs * T * T);
        CCW_CUDA(cudaMemcpyAsync(pasted.data(), d_pasted, pasted.size(), cudaMemcpyDeviceToHost, st));
    }
    CCW_CUDA(cudaStreamSynchronize(st));
    if (h_out && h_dst != h_out) {  // pinned staging -> the caller's pageable buffer, in parallel
        constexpr size_t kChunk = 4u << 20;
        const int nchunk = static_cast<int>((out_bytes + kChunk - 1) / kChunk);
        ctx->pool.run(nchunk, [&](int i) {
            const size_t o = static_cast<size_t>(i) * kChunk;
            std::memcpy(h_out + o, h_dst + o, std::min(kChunk, out_bytes - o));
        });
    }

    {
        float ms = 0;
        cudaEventElapsedTime(&ms, ev0, ev1);
        ctx->timing.total_ms = ms;
        ctx->timing.ccf_ms = ctx->profiling ? pair_ms(tm.ccf) : 0.0;
        ctx->timing.select_ms = ctx->profiling ? pair_ms(tm.sel) : 0.0;
    }
    ctx->timing.ccf_launches = ccf_launches;
    ctx->timing.launches = launches + (d_hd ? 1 : 0) + 0;
    ctx->timing.ccf_flop = ccf_flop;
    ctx->timing.ccf_flop_ref = ccf_flop_ref;
    ctx->timing.waves = static_cast<int64_t>(max_key + 1);
    ctx->timing.groups = G;
    ctx->timing.host_prep_ms = host_prep_ms;
    ctx->timing.jobs = static_cast<int64_t>(total_jobs);
    ctx->timing.rescored = static_cast<int64_t>(stats[0]);
    for (const CopyMark& cm : copy_marks) {
        float ms = 0;
        cudaEventElapsedTime(&ms, ev0, cm.ev);
        fprintf(stderr, "copy stream: wave %d group %d bands copied at %.3f ms\n", cm.w, cm.g, ms);
    }
    if (d_tl) {
        std::vector<unsigned long long> h(tl_tag.size() * 4);
        CCW_CUDA(cudaMemcpy(h.data(), d_tl, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        unsigned long long t0 = ~0ull;
        for (size_t i = 0; i < tl_tag.size(); ++i) t0 = std::min(t0, h[4 * i + 2]);
        fprintf(stderr, "timeline (us from first resident CTA): wave group kind resident start end last_start\n");
        for (size_t i = 0; i < tl_tag.size(); ++i) {
            if (h[4 * i + 1] == 0) continue;
            fprintf(stderr, "TL %d %d %d %.2f %.2f %.2f %.2f\n", tl_tag[i][0], tl_tag[i][1], tl_tag[i][2],
                    (h[4 * i + 2] - t0) * 1e-3, (h[4 * i] - t0) * 1e-3, (h[4 * i + 1] - t0) * 1e-3,
                    (h[4 * i + 3] - t0) * 1e-3);
        }
    }
    if (d_probe) {
        unsigned long long pr[8];
        CCW_CUDA(cudaMemcpy(pr, d_probe, sizeof(pr), cudaMemcpyDeviceToHost));
        const double n = static_cast<double>(std::max(1ull, pr[7]));
        fprintf(stderr, "ccf probe (mean cycles from CTA start over %llu CTAs): setup %.0f pdl_wait %.0f first_stage %.0f "
                "last_stage %.0f acc_ready %.0f epilogue_done %.0f end %.0f\n", pr[7], pr[0] / n, pr[1] / n,
                pr[2] / n, pr[3] / n, pr[4] / n, pr[5] / (8 * n), pr[6] / n);
        tc_probe_buffer = nullptr;
    }
    if (getenv("CCW_PHASES"))
        fprintf(stderr, "phase clocks: scan[M_K %llu list %llu S_K %llu cand %llu] fast[scan+stage %llu batch %llu choose+map %llu]"
                " | bulk total %llu stage %llu compute %llu | tiles>=M_K %llu list %llu\n",
                stats[8], stats[9], stats[10], stats[11], stats[12], stats[13], stats[4], stats[7], stats[14],
                stats[15], stats[5], stats[6]);
    ctx->timing.screened_jobs = static_cast<int64_t>(stats[1]);
    ctx->timing.list_overflows = static_cast<int64_t>(stats[2]);
    ctx->timing.bulk_jobs = static_cast<int64_t>(stats[3]);
    if (bulk_launch && stats[3] == 0)
        ctx->bulk_off[bulk_key] = true;
    else if (!bulk_launch && stats[2] > 0)  // a list overflowed: bring the bulk kernel back
        ctx->bulk_off.erase(bulk_key);
    ctx->timing.ccf_variant = any_screen ? (use_tc ? 2 : 1) : 0;
    ctx->timing.ccf_mma_flop = use_tc ? ccf_mma_flop : 0.0;

    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
    for (int r = 0; r < n_real; ++r) {
        if (diag) {
            ccw_diag& d = diag[r];
            d.seed = seeds[r];
            d.origin = variants[vid[r]].origin;
            d.column_major = variants[vid[r]].column_major;
            d.work_height = wh;
            d.work_width = ww;
            d.placement_count = static_cast<int>(variants[vid[r]].tops.size());
            d.hard_data_count = hd ? n_hd : 0;
            d.pre_overwrite_mismatches = mism[r];
            d._pad = 0;
            d.wall_seconds = wall;
        }
        if (traces) {
            ccw_trace& tr = traces[r];
            tr.count = 0;
            (void)tr;
        }
    }
    if (traces) {
        // flat is wave-ordered; rebuild each realization's raster-ordered trace
        for (size_t g = 0; g < total_jobs; ++g) {
            const Job& jb = flat[g];
            ccw_trace& tr = traces[jb.real];
            if (jb.place >= tr.capacity) continue;
            tr.top[jb.place] = jb.top;
            tr.left[jb.place] = jb.left;
            tr.shape[jb.place] = jb.shape;
            tr.ti_row[jb.place] = chosen[2 * g];
            tr.ti_col[jb.place] = chosen[2 * g + 1];
            if (tr.pasted)
                std::memcpy(tr.pasted + static_cast<size_t>(jb.place) * T * T, pasted.data() + g * T * T,
                            static_cast<size_t>(T) * T);
        }
        for (int r = 0; r < n_real; ++r)
            traces[r].count = std::min(traces[r].capacity, static_cast<int>(variants[vid[r]].tops.size()));
    }
}

}  // namespace ccwgpu
