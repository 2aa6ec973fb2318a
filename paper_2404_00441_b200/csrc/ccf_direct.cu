// ccf_direct.cu -- the exact-integer CCF screen on CUDA cores (fp32 FFMA over
// integer-valued operands), used when the int8 tensor-core screen does not
// apply (ccw_ctx_set_ccf_variant 1, or block statistics above 127).
#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <thread>

#include "sim_kernels.cuh"

namespace ccwgpu {

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
    // (position shards: the grid covers the rows of [p0, p0 + npos) only)
    const int x0 = P.p0 / P.out_w + blockIdx.y * CCF_TX, y0 = blockIdx.x * CCF_TY;

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
        int32_t* out = P.scores + static_cast<size_t>(slot) * P.sld;
#pragma unroll
        for (int b = 0; b < CCF_RY; ++b) {
            const int y = y0 + tcg + b;
            const int p = x * P.out_w + y - P.p0;  // shard-local position
            if (y < P.out_w && p >= 0 && p < P.npos) out[p] = __float2int_rn(acc[b]);
        }
    }
}

}  // namespace ccwgpu
