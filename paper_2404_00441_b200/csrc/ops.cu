// ops.cu -- the reference's fp64 operator surface on the device, bit-identical
// to wavelet.hpp / matcher.hpp for arbitrary real planes (the
// drop-in ccw_score_map(RealPlane...) API is pinned to 1e-9 on generic
// doubles, so it cannot use the integer screen of the simulator).
#include <algorithm>
#include <cfloat>
#include <climits>
#include <vector>

#include "ccw_device.cuh"
#include "internal.hpp"

namespace ccwgpu {

namespace {

constexpr double S = kInvSqrt2;

// One analysis level (wavelet.hpp:69-106): row pass lo = s*x0 + s*x1,
// hi = s*x0 + (-s)*x1 (HaarFilterBank::analyze, :25-32), then column pass
// a = s*(l0 + l1), dh = s*(l0 - l1), dv = s*(h0 + h1), dd = s*(h0 - h1).
__global__ void dwt_level_kernel(const double* __restrict__ in, int h, int w, double* a,
                                 double* dh, double* dv, double* dd) {
    const int hw = w / 2, hh = h / 2;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= hh * hw) return;
    const int i = idx / hw, j = idx - i * hw;
    const double* r0 = in + static_cast<size_t>(2 * i) * w + 2 * j;
    const double* r1 = r0 + w;
    const double l0 = __dadd_rn(__dmul_rn(S, r0[0]), __dmul_rn(S, r0[1]));
    const double h0 = __dadd_rn(__dmul_rn(S, r0[0]), __dmul_rn(-S, r0[1]));
    const double l1 = __dadd_rn(__dmul_rn(S, r1[0]), __dmul_rn(S, r1[1]));
    const double h1 = __dadd_rn(__dmul_rn(S, r1[0]), __dmul_rn(-S, r1[1]));
    a[idx] = __dmul_rn(S, __dadd_rn(l0, l1));
    if (dh) dh[idx] = __dmul_rn(S, __dsub_rn(l0, l1));
    if (dv) dv[idx] = __dmul_rn(S, __dadd_rn(h0, h1));
    if (dd) dd[idx] = __dmul_rn(S, __dsub_rn(h0, h1));
}

// One synthesis level (wavelet.hpp:108-143): l0 = s*(a + dh), l1 = s*(a - dh),
// h0 = s*(dv + dd), h1 = s*(dv - dd); x0 = s*lo + s*hi, x1 = s*lo + (-s)*hi.
__global__ void idwt_level_kernel(const double* __restrict__ a, const double* __restrict__ dh,
                                  const double* __restrict__ dv, const double* __restrict__ dd,
                                  int hh, int hw, double* out) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= hh * hw) return;
    const int i = idx / hw, j = idx - i * hw;
    const int w = 2 * hw;
    const double l0 = __dmul_rn(S, __dadd_rn(a[idx], dh[idx]));
    const double l1 = __dmul_rn(S, __dsub_rn(a[idx], dh[idx]));
    const double h0 = __dmul_rn(S, __dadd_rn(dv[idx], dd[idx]));
    const double h1 = __dmul_rn(S, __dsub_rn(dv[idx], dd[idx]));
    double* o0 = out + static_cast<size_t>(2 * i) * w + 2 * j;
    double* o1 = o0 + w;
    o0[0] = __dadd_rn(__dmul_rn(S, l0), __dmul_rn(S, h0));
    o0[1] = __dadd_rn(__dmul_rn(S, l0), __dmul_rn(-S, h0));
    o1[0] = __dadd_rn(__dmul_rn(S, l1), __dmul_rn(S, h1));
    o1[1] = __dadd_rn(__dmul_rn(S, l1), __dmul_rn(-S, h1));
}

// Generic fp64 CCF (matcher.hpp:147-173), one thread per window, reference
// order: for f, for run, sum over the run, acc += sum.
__global__ void score_map_kernel(const double* __restrict__ ti, const double* __restrict__ tmpl,
                                 int nch, int ti_h, int ti_w, int t_h, int t_w,
                                 const int3* __restrict__ runs, int nruns, int scoring,
                                 double* __restrict__ out) {
    const int out_h = ti_h - t_h + 1, out_w = ti_w - t_w + 1;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= out_h * out_w) return;
    const int x = idx / out_w, y = idx - x * out_w;
    double acc = 0.0;
    for (int f = 0; f < nch; ++f) {
        const double* tp = ti + static_cast<size_t>(f) * ti_h * ti_w;
        const double* mp = tmpl + static_cast<size_t>(f) * t_h * t_w;
        for (int k = 0; k < nruns; ++k) {
            const int3 r = runs[k];
            const double* a = tp + static_cast<size_t>(x + r.x) * ti_w + y;
            const double* b = mp + static_cast<size_t>(r.x) * t_w;
            double sum = 0.0;
            for (int t = r.y; t < r.z; ++t) sum = __dadd_rn(sum, __dmul_rn(a[t], b[t]));
            acc = __dadd_rn(acc, sum);
        }
    }
    if (scoring == 1) {
        double n = 0.0;
        for (int f = 0; f < nch; ++f) {
            const double* tp = ti + static_cast<size_t>(f) * ti_h * ti_w;
            for (int k = 0; k < nruns; ++k) {
                const int3 r = runs[k];
                const double* a = tp + static_cast<size_t>(x + r.x) * ti_w + y;
                double sum = 0.0;
                for (int t = r.y; t < r.z; ++t) sum = __dadd_rn(sum, __dmul_rn(a[t], a[t]));
                n = __dadd_rn(n, sum);
            }
        }
        acc = n > 0.0 ? __ddiv_rn(acc, __dsqrt_rn(n)) : 0.0;
    }
    out[idx] = acc;
}

__device__ __forceinline__ bool ranks_before(double ka, int ia, double kb, int ib) {
    return ka > kb || (ka == kb && ia < ib);
}

// top_k (matcher.hpp:177-204) = prefix of the stable descending sort: round r
// picks the best entry ranked strictly after round r-1's winner.
__global__ void __launch_bounds__(1024) top_k_kernel(const double* __restrict__ s, int n, int k,
                                                     int* __restrict__ idx_out,
                                                     double* __restrict__ val_out) {
    __shared__ double rk[32];
    __shared__ int ri[32];
    __shared__ double prev_k;
    __shared__ int prev_i;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) {
        prev_k = 0.0;
        prev_i = -1;
    }
    __syncthreads();
    for (int round = 0; round < k; ++round) {
        const double pk = prev_k;
        const int pi = prev_i;
        double bk = 0.0;
        int bi = -1;
        for (int e = threadIdx.x; e < n; e += blockDim.x) {
            const double v = s[e];
            if (pi >= 0 && !ranks_before(pk, pi, v, e)) continue;
            if (bi < 0 || ranks_before(v, e, bk, bi)) {
                bk = v;
                bi = e;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (oi >= 0 && (bi < 0 || ranks_before(ok, oi, bk, bi))) {
                bk = ok;
                bi = oi;
            }
        }
        if (lane == 0) {
            rk[wid] = bk;
            ri[wid] = bi;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < nw; ++w)
                if (ri[w] >= 0 && (bi < 0 || ranks_before(rk[w], ri[w], bk, bi))) {
                    bk = rk[w];
                    bi = ri[w];
                }
            idx_out[round] = bi;
            val_out[round] = bk;
            prev_k = bk;
            prev_i = bi;
        }
        __syncthreads();
    }
}

// select_conditional (matcher.hpp:222-241): first zero-mismatch candidate,
// else the first with the fewest mismatches.
__global__ void __launch_bounds__(256) select_conditional_kernel(
    const int32_t* __restrict__ rows, const int32_t* __restrict__ cols, int n_cands,
    const int32_t* __restrict__ hd, int n_hd, const uint8_t* __restrict__ ti, int ti_w, int levels,
    int* out) {
    __shared__ int red[32];
    int best = 0, best_mis = INT_MAX, pick = -1;
    for (int c = 0; c < n_cands; ++c) {
        const int fr = rows[c] << levels, fc = cols[c] << levels;
        int mis = 0;
        for (int d = threadIdx.x; d < n_hd; d += blockDim.x)
            mis += ti[static_cast<size_t>(fr + hd[3 * d]) * ti_w + fc + hd[3 * d + 1]] != hd[3 * d + 2];
        mis = block_reduce(mis, [](int a, int b) { return a + b; }, red);
        if (mis == 0) {
            pick = c;
            best_mis = 0;
            break;
        }
        if (mis < best_mis) {
            best = c;
            best_mis = mis;
        }
    }
    if (threadIdx.x == 0) {
        out[0] = pick >= 0 ? pick : best;
        out[1] = best_mis;
    }
}

template <typename T>
T* upload(ccw_ctx* ctx, DevBuf& buf, const T* src, size_t n) {
    T* d = buf.as<T>(n);
    if (n) CCW_CUDA(cudaMemcpyAsync(d, src, sizeof(T) * n, cudaMemcpyHostToDevice, ctx->stream));
    return d;
}

template <typename T>
void download(ccw_ctx* ctx, T* dst, const T* src, size_t n) {
    if (n) CCW_CUDA(cudaMemcpyAsync(dst, src, sizeof(T) * n, cudaMemcpyDeviceToHost, ctx->stream));
}

int blocks(size_t n, int t) { return static_cast<int>((n + t - 1) / t); }

}  // namespace

void op_dwt2_single(ccw_ctx* ctx, const double* in, int h, int w, double* a, double* dh,
                    double* dv, double* dd) {
    const size_t n = static_cast<size_t>(h) * w, q = n / 4;
    const double* d_in = upload(ctx, ctx->ops_a, in, n);
    double* d_o = ctx->ops_b.as<double>(4 * q);
    dwt_level_kernel<<<blocks(q, 256), 256, 0, ctx->stream>>>(d_in, h, w, d_o, d_o + q, d_o + 2 * q,
                                                              d_o + 3 * q);
    CCW_CUDA(cudaGetLastError());
    download(ctx, a, d_o, q);
    download(ctx, dh, d_o + q, q);
    download(ctx, dv, d_o + 2 * q, q);
    download(ctx, dd, d_o + 3 * q, q);
    CCW_CUDA(cudaStreamSynchronize(ctx->stream));
}

void op_idwt2_single(ccw_ctx* ctx, const double* a, const double* dh, const double* dv,
                     const double* dd, int hh, int hw, double* out) {
    const size_t q = static_cast<size_t>(hh) * hw;
    double* d_in = ctx->ops_a.as<double>(4 * q);
    CCW_CUDA(cudaMemcpyAsync(d_in, a, sizeof(double) * q, cudaMemcpyHostToDevice, ctx->stream));
    CCW_CUDA(cudaMemcpyAsync(d_in + q, dh, sizeof(double) * q, cudaMemcpyHostToDevice, ctx->stream));
    CCW_CUDA(cudaMemcpyAsync(d_in + 2 * q, dv, sizeof(double) * q, cudaMemcpyHostToDevice, ctx->stream));
    CCW_CUDA(cudaMemcpyAsync(d_in + 3 * q, dd, sizeof(double) * q, cudaMemcpyHostToDevice, ctx->stream));
    double* d_o = ctx->ops_b.as<double>(4 * q);
    idwt_level_kernel<<<blocks(q, 256), 256, 0, ctx->stream>>>(d_in, d_in + q, d_in + 2 * q,
                                                               d_in + 3 * q, hh, hw, d_o);
    CCW_CUDA(cudaGetLastError());
    download(ctx, out, d_o, 4 * q);
    CCW_CUDA(cudaStreamSynchronize(ctx->stream));
}

// dwt2 (wavelet.hpp:147-171): dwt2_single re-applied to the previous apex.
void op_dwt2(ccw_ctx* ctx, const double* in, int h, int w, int levels, double* apex,
             double* details) {
    const size_t n = static_cast<size_t>(h) * w;
    double* cur = upload(ctx, ctx->ops_a, in, n);
    double* nxt = ctx->ops_b.as<double>(n);
    size_t dtot = 0;
    for (int j = 1; j <= levels; ++j) dtot += 3 * static_cast<size_t>(h >> j) * (w >> j);
    double* d_det = ctx->ops_c.as<double>(std::max<size_t>(dtot, 1));
    int ch = h, cw = w;
    size_t off = 0;
    for (int j = 1; j <= levels; ++j) {
        const size_t q = static_cast<size_t>(ch / 2) * (cw / 2);
        dwt_level_kernel<<<blocks(q, 256), 256, 0, ctx->stream>>>(cur, ch, cw, nxt, d_det + off,
                                                                  d_det + off + q, d_det + off + 2 * q);
        CCW_CUDA(cudaGetLastError());
        off += 3 * q;
        std::swap(cur, nxt);
        ch /= 2;
        cw /= 2;
    }
    download(ctx, apex, cur, static_cast<size_t>(ch) * cw);
    if (details) download(ctx, details, d_det, dtot);
    CCW_CUDA(cudaStreamSynchronize(ctx->stream));
}

// idwt2 (wavelet.hpp:174-191).
void op_idwt2(ccw_ctx* ctx, const double* apex, const double* details, int h, int w, int levels,
              double* out) {
    size_t dtot = 0;
    std::vector<size_t> offs(levels + 1, 0);
    for (int j = 1; j <= levels; ++j) {
        offs[j] = dtot;
        dtot += 3 * static_cast<size_t>(h >> j) * (w >> j);
    }
    const double* d_det = upload(ctx, ctx->ops_c, details, dtot);
    const size_t n = static_cast<size_t>(h) * w;
    double* cur = ctx->ops_a.as<double>(n);
    double* nxt = ctx->ops_b.as<double>(n);
    int ch = h >> levels, cw = w >> levels;
    CCW_CUDA(cudaMemcpyAsync(cur, apex, sizeof(double) * ch * cw, cudaMemcpyHostToDevice, ctx->stream));
    for (int j = levels; j >= 1; --j) {
        const size_t q = static_cast<size_t>(ch) * cw;
        const double* dj = d_det + offs[j];
        idwt_level_kernel<<<blocks(q, 256), 256, 0, ctx->stream>>>(cur, dj, dj + q, dj + 2 * q, ch,
                                                                   cw, nxt);
        CCW_CUDA(cudaGetLastError());
        std::swap(cur, nxt);
        ch *= 2;
        cw *= 2;
    }
    download(ctx, out, cur, n);
    CCW_CUDA(cudaStreamSynchronize(ctx->stream));
}

void op_score_map(ccw_ctx* ctx, const double* ti, const double* tmpl, int nch, int ti_h, int ti_w,
                  int t_h, int t_w, const double* mask, int scoring, double* out) {
    // mask_runs (matcher.hpp:44-61) on the host: pure index bookkeeping
    std::vector<int3> runs;
    for (int s = 0; s < t_h; ++s) {
        int t = 0;
        while (t < t_w) {
            if (mask[static_cast<size_t>(s) * t_w + t] == 1.0) {
                const int t0 = t;
                while (t < t_w && mask[static_cast<size_t>(s) * t_w + t] == 1.0) ++t;
                runs.push_back(make_int3(s, t0, t));
            } else {
                ++t;
            }
        }
    }
    const double* d_ti = upload(ctx, ctx->ops_a, ti, static_cast<size_t>(nch) * ti_h * ti_w);
    const double* d_tm = upload(ctx, ctx->ops_b, tmpl, static_cast<size_t>(nch) * t_h * t_w);
    const int3* d_runs = upload(ctx, ctx->ops_c, runs.data(), runs.size());
    const size_t nout = static_cast<size_t>(ti_h - t_h + 1) * (ti_w - t_w + 1);
    double* d_out = ctx->ops_d.as<double>(nout);
    score_map_kernel<<<blocks(nout, 128), 128, 0, ctx->stream>>>(
        d_ti, d_tm, nch, ti_h, ti_w, t_h, t_w, d_runs, static_cast<int>(runs.size()), scoring, d_out);
    CCW_CUDA(cudaGetLastError());
    download(ctx, out, d_out, nout);
    CCW_CUDA(cudaStreamSynchronize(ctx->stream));
}

void op_top_k(ccw_ctx* ctx, const double* scores, int h, int w, int k, int32_t* rows,
              int32_t* cols, double* vals, int* n_out) {
    const int n = h * w;
    const int kk = std::min(k, n);
    const double* d_s = upload(ctx, ctx->ops_a, scores, static_cast<size_t>(n));
    int* d_i = ctx->ops_b.as<int>(kk);
    double* d_v = ctx->ops_c.as<double>(kk);
    top_k_kernel<<<1, 1024, 0, ctx->stream>>>(d_s, n, kk, d_i, d_v);
    CCW_CUDA(cudaGetLastError());
    std::vector<int> idx(kk);
    download(ctx, idx.data(), d_i, kk);
    download(ctx, vals, d_v, kk);
    CCW_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < kk; ++i) {
        rows[i] = idx[i] / w;
        cols[i] = idx[i] % w;
    }
    *n_out = kk;
}

void op_select_conditional(ccw_ctx* ctx, const int32_t* rows, const int32_t* cols, int n_cands,
                           const int32_t* hd, int n_hd, const uint8_t* ti, int ti_h, int ti_w,
                           int levels, int* pick, int* mismatches) {
    const int32_t* d_r = upload(ctx, ctx->ops_a, rows, n_cands);
    const int32_t* d_c = upload(ctx, ctx->ops_b, cols, n_cands);
    const int32_t* d_h = upload(ctx, ctx->ops_c, hd, static_cast<size_t>(3) * n_hd);
    const uint8_t* d_t = upload(ctx, ctx->ops_d, ti, static_cast<size_t>(ti_h) * ti_w);
    int* d_o = ctx->ops_e.as<int>(2);
    select_conditional_kernel<<<1, 256, 0, ctx->stream>>>(d_r, d_c, n_cands, d_h, n_hd, d_t, ti_w,
                                                          levels, d_o);
    CCW_CUDA(cudaGetLastError());
    int o[2];
    download(ctx, o, d_o, 2);
    CCW_CUDA(cudaStreamSynchronize(ctx->stream));
    *pick = o[0];
    *mismatches = o[1];
}

// First cell whose code is >= nf (n if none): the code-range check of an
// uploaded grid (grid.hpp:36-40), on the device.
__global__ void first_bad_code_kernel(const uint8_t* __restrict__ c, size_t n, int nf,
                                      unsigned long long* __restrict__ first) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x * 16;
    for (size_t i0 = (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 16; i0 < n; i0 += stride) {
        if (i0 + 16 <= n && (reinterpret_cast<uintptr_t>(c + i0) & 15) == 0) {
            const uint4 v = *reinterpret_cast<const uint4*>(c + i0);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 16; ++k)
                if (static_cast<int>((w[k >> 2] >> (8 * (k & 3))) & 255u) >= nf) {
                    atomicMin(first, static_cast<unsigned long long>(i0 + k));
                    break;
                }
        } else {
            for (size_t i = i0; i < n && i < i0 + 16; ++i)
                if (c[i] >= nf) {
                    atomicMin(first, static_cast<unsigned long long>(i));
                    break;
                }
        }
    }
}

size_t first_bad_code(const uint8_t* d, size_t n, int nf, cudaStream_t st, unsigned long long* d_first) {
    if (nf >= 256 || n == 0) return n;
    const unsigned long long init = n;
    CCW_CUDA(cudaMemcpyAsync(d_first, &init, sizeof(init), cudaMemcpyHostToDevice, st));
    const size_t threads = (n + 15) / 16;
    const unsigned nb = static_cast<unsigned>(std::min<size_t>((threads + 255) / 256, 148 * 16));
    first_bad_code_kernel<<<nb, 256, 0, st>>>(d, n, nf, d_first);
    CCW_CUDA(cudaGetLastError());
    unsigned long long got = n;
    CCW_CUDA(cudaMemcpyAsync(&got, d_first, sizeof(got), cudaMemcpyDeviceToHost, st));
    CCW_CUDA(cudaStreamSynchronize(st));
    return static_cast<size_t>(got);
}

}  // namespace ccwgpu
