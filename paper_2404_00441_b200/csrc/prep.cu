// prep.cu -- per-TI and per-wave preparation: the TI pyramid (reference-order
// apex values and exact block-count screen planes), the overlap-region prep
// of every placement (screen weights, fp64 template) and the normalized
// screen's norm maps.
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

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Dependency flags (P.depflag, option flagprep): a placement's prep starts as
// soon as the previous-wave placements it reads have pasted (their select
// CTAs count them here after the map writes), not when the whole previous
// launch has ended -- the prep overlaps the select's tail.  The launch has
// one extra CTA that waits for the previous launch in full, so this
// launch's completion still implies it (the screen that follows rewrites
// the score rows that launch reads).
__global__ void or_prep_src_kernel(SimParams P, const Job* __restrict__ jobs, int job0) {
    pdl_trigger();
    const int slot = blockIdx.x;
    if (P.depflag && slot == static_cast<int>(gridDim.x) - 1) {
        pdl_wait();
        return;
    }
    const Job jb = jobs[job0 + slot];
    if (P.jvar && threadIdx.x == 0) P.jvar[slot] = static_cast<int8_t>(mask_variant(jb.shape, jb.vleft, jb.htop));
    tl_mark(P.tl, 2);
    if (P.depflag && jb.ndep > 0) {
        if (threadIdx.x == 0) {
            const int* f = P.depflag + job0 + slot;
            long long spins = 0;
            while (ld_acquire(f) < jb.ndep) {
                __nanosleep(32);
                if (++spins > (1ll << 27)) __trap();  // (a missing signal is a bug: fail, do not hang)
            }
            __threadfence();
        }
        __syncthreads();
    } else {
        pdl_wait();
    }
    tl_mark(P.tl, 0);
    prep_src_job(P, jb, slot, P.wts8, P.tm64, P.cjob);
    tl_mark(P.tl, 1);
}

__global__ void or_prep_kernel(SimParams P, const Job* __restrict__ jobs, int job0) {
    pdl_trigger();
    const int slot = blockIdx.x;
    const Job jb = jobs[job0 + slot];
    pdl_wait();
    if (P.jvar && threadIdx.x == 0) P.jvar[slot] = static_cast<int8_t>(mask_variant(jb.shape, jb.vleft, jb.htop));
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
        // literal-config extension: blocks the overlap only partly covers
        // count / transform just their supported cells
        auto stat = [&](int mode, int f) {
            return P.any_support ? block_stat_sup(base, P.ww, B, mode, f, s * B, t * B, jb.shape, jb.vleft, jb.htop,
                                                  P.T, P.OV)
                                 : block_stat(base, P.ww, B, mode, f);
        };
        if (P.mode == 0) {
            const int last = in ? stat(0, P.F - 1) : 0;
            csum += last;
            for (int f = 0; f < P.nscr; ++f) {
                const int v = in ? stat(0, f) - last : 0;
                wts[f * Tc * Tc + c] = v;
                if (w8) w8[f * Tc * Tc + c] = static_cast<int8_t>(v);
            }
        } else {
            const int v = in ? stat(1, 0) : 0;
            wts[c] = v;
            if (w8) w8[c] = static_cast<int8_t>(v);
        }
        for (int ch = 0; ch < P.nch; ++ch)
            tm[ch * Tc * Tc + c] =
                !in ? 0.0
                    : P.any_support ? haar_apex_block_sup(base, P.ww, P.J, P.mode, ch, s * B, t * B, jb.shape, jb.vleft,
                                                          jb.htop, P.T, P.OV)
                                    : haar_apex_block(base, P.ww, P.J, P.mode, ch);
    }
    if (P.cjob) store_cjob(P.cjob, P.mode, P.B, slot, csum);
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

// Pure coarse blocks: the facies all B x B fine cells of the block hold, -1 if mixed.
__global__ void pure_block_kernel(const uint8_t* __restrict__ codes, int w, int hc, int wc, int B,
                                  int8_t* __restrict__ out) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= hc * wc) return;
    const int br = b / wc, bc = b - br * wc;
    const uint8_t* c0 = codes + static_cast<size_t>(br) * B * w + static_cast<size_t>(bc) * B;
    const int f = c0[0];
    bool pure = f < 16;
    for (int r = 0; r < B && pure; ++r)
        for (int c = 0; c < B; ++c) pure &= c0[static_cast<size_t>(r) * w + c] == f;
    out[b] = pure ? static_cast<int8_t>(f) : static_cast<int8_t>(-1);
}

// U[v][p]: the facies f when every coarse block of window p under mask
// variant v is pure f, else -1.  Such windows have the all-f block's apex
// values on every masked cell in every channel (indicator or raw codes), so
// their fp64 scores (matcher.hpp:64-81) are bit-identical for any template.
__global__ void uniform_map_kernel(const int8_t* __restrict__ pure, int wc, int Tc, int OVc, int out_w, int npos,
                                   int ustride, int8_t* __restrict__ out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const int v = blockIdx.y;
    if (p >= npos) return;
    const int shape = v < 4 ? kL : (v < 6 ? kVertical : kHorizontal);
    const int vleft = v < 4 ? (v >> 1) : (v < 6 ? v - 4 : 0);
    const int htop = v < 4 ? (v & 1) : (v < 6 ? 0 : v - 6);
    const int x = p / out_w, y = p - x * out_w;
    int cls = -2;  // (no masked cell seen yet)
    for (int s = 0; s < Tc && cls != -1; ++s) {
        int t0, t1;
        mask_row_run(shape, vleft, htop, Tc, OVc, s, t0, t1);
        for (int t = t0; t < t1; ++t) {
            const int f = pure[static_cast<size_t>(x + s) * wc + y + t];
            if (f < 0 || (cls >= 0 && f != cls)) {
                cls = -1;
                break;
            }
            cls = f;
        }
    }
    out[static_cast<size_t>(v) * ustride + p] = static_cast<int8_t>(cls < 0 ? -1 : cls);
}

// first[f] = the lowest-index pure block of facies f (INT_MAX: none)
__global__ void first_pure_kernel(const int8_t* __restrict__ pure, int nb, int* __restrict__ first) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nb && pure[b] >= 0) atomicMin(&first[pure[b]], b);
}

// out[f][ch] = the apex of a pure-f block in channel ch: every pure-f block
// holds the same cells, so the reference-order Haar tree gives one value
__global__ void pure_apex_kernel(const int* __restrict__ first, const double* __restrict__ ti64, int nb, int nch,
                                 double* __restrict__ out) {
    const int f = threadIdx.x / nch, ch = threadIdx.x % nch;
    if (f >= 16) return;
    out[f * nch + ch] = first[f] < nb ? ti64[static_cast<size_t>(ch) * nb + first[f]] : 0.0;
}

// first[v][f][0, kTcQ): the kTcQ lowest window positions of uniform class f
// under mask variant v (INT_MAX pads).  One CTA per (f, v): each thread keeps
// the first matches of its contiguous chunk, chunks are merged in order.
__global__ void __launch_bounds__(256) uniform_first_kernel(const int8_t* __restrict__ umap, int npos, int ustride,
                                                            int* __restrict__ first) {
    const int f = blockIdx.x, v = blockIdx.y;
    __shared__ int loc[256][kTcQ];
    __shared__ int nloc[256];
    const int8_t* u = umap + static_cast<size_t>(v) * ustride;
    const int chunk = (npos + blockDim.x - 1) / blockDim.x;
    const int p0 = threadIdx.x * chunk, p1 = min(npos, p0 + chunk);
    int n = 0;
    for (int p = p0; p < p1 && n < kTcQ; ++p)
        if (u[p] == f) loc[threadIdx.x][n++] = p;
    nloc[threadIdx.x] = n;
    __syncthreads();
    if (threadIdx.x == 0) {
        int* out = first + (static_cast<size_t>(v) * 16 + f) * kTcQ;
        int k = 0;
        for (int t = 0; t < static_cast<int>(blockDim.x) && k < kTcQ; ++t)
            for (int i = 0; i < nloc[t] && k < kTcQ; ++i) out[k++] = loc[t][i];
        for (; k < kTcQ; ++k) out[k] = INT_MAX;
    }
}

// Non-uniform windows as bits: [8][ustride / 32] words, bit i of word k set
// when window 32 k + i of the variant is non-uniform (the screen's tmax_nu).
__global__ void uniform_bits_kernel(const int8_t* __restrict__ umap, int npos, int ustride, uint32_t* __restrict__ bits) {
    const int nw = ustride / 32;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= 8 * nw) return;
    const int v = e / nw, k = e - v * nw;
    const int8_t* u = umap + static_cast<size_t>(v) * ustride + 32 * k;
    uint32_t b = 0;
    for (int i = 0; i < 32; ++i) b |= static_cast<uint32_t>(32 * k + i < npos && u[i] < 0) << i;
    bits[e] = b;
}

// Uniform-window classes of a TI for template Tc / overlap OVc, cached on the
// TI, followed by the pure blocks, (8-byte aligned) the pure-block apex table
// [16][nch] (ti_pure_apex) and the first positions of every class
// [8][16][kTcQ] (ti_uniform_first).
template <typename T>
static T* align16(T* p) {  // (the screen epilogue reads the bits as uint4)
    return reinterpret_cast<T*>((reinterpret_cast<uintptr_t>(p) + 15) & ~static_cast<uintptr_t>(15));
}

int umap_stride(int npos) { return (npos + 255) & ~255; }  // (whole 256-position screen tiles)
static size_t umap_apex_offset(size_t npos, size_t nb) {
    return (8 * static_cast<size_t>(umap_stride(static_cast<int>(npos))) + nb + 8 + 7) & ~static_cast<size_t>(7);
}

const int8_t* ti_umap(ccw_ti* ti, int Tc, int OVc, cudaStream_t st) {
    const auto key = std::make_pair(Tc, OVc);
    auto it = ti->umap.find(key);
    if (it != ti->umap.end()) return it->second;
    const int out_h = ti->hc - Tc + 1, out_w = ti->wc - Tc + 1, npos = out_h * out_w;
    const size_t nb = static_cast<size_t>(ti->hc) * ti->wc;
    const size_t ao = umap_apex_offset(npos, nb);
    int8_t* m = static_cast<int8_t*>(cache_alloc(ti->device, ao + sizeof(double) * 16 * ti->nch + 16 * sizeof(int) +
                                                              sizeof(int) * 8 * 16 * kTcQ +
                                                              sizeof(uint32_t) * 8 * (umap_stride(npos) / 32) + 16));
    const int us = umap_stride(npos);
    int8_t* pure = m + 8 * static_cast<size_t>(us);
    CCW_CUDA(cudaMemsetAsync(m, 0xFF, 8 * static_cast<size_t>(us), st));  // (padding: non-uniform)
    pure_block_kernel<<<static_cast<unsigned>((nb + 255) / 256), 256, 0, st>>>(ti->d_codes, ti->w, ti->hc, ti->wc,
                                                                              1 << ti->J, pure);
    uniform_map_kernel<<<dim3((npos + 255) / 256, 8), 256, 0, st>>>(pure, ti->wc, Tc, OVc, out_w, npos, us, m);
    double* apex = reinterpret_cast<double*>(m + ao);
    int* first = reinterpret_cast<int*>(apex + 16 * ti->nch);
    fill_i32(first, 16, INT_MAX, st);
    first_pure_kernel<<<static_cast<unsigned>((nb + 255) / 256), 256, 0, st>>>(pure, static_cast<int>(nb), first);
    pure_apex_kernel<<<1, 16 * ti->nch, 0, st>>>(first, ti->d_ti64, static_cast<int>(nb), ti->nch, apex);
    uniform_first_kernel<<<dim3(16, 8), 256, 0, st>>>(m, npos, us, first + 16);
    uint32_t* ubits = align16(reinterpret_cast<uint32_t*>(first + 16 + 8 * 16 * kTcQ));
    uniform_bits_kernel<<<(8 * (us / 32) + 255) / 256, 256, 0, st>>>(m, npos, us, ubits);
    CCW_CUDA(cudaGetLastError());
    ti->umap[key] = m;
    return m;
}

const uint32_t* ti_uniform_bits(ccw_ti* ti, int Tc, int OVc, cudaStream_t st) {
    return align16(reinterpret_cast<const uint32_t*>(ti_uniform_first(ti, Tc, OVc, st) + 8 * 16 * kTcQ));
}

const int* ti_uniform_first(ccw_ti* ti, int Tc, int OVc, cudaStream_t st) {
    const double* apex = ti_pure_apex(ti, Tc, OVc, st);
    return reinterpret_cast<const int*>(apex + 16 * ti->nch) + 16;
}

const double* ti_pure_apex(ccw_ti* ti, int Tc, int OVc, cudaStream_t st) {
    const int8_t* m = ti_umap(ti, Tc, OVc, st);
    const int npos = (ti->hc - Tc + 1) * (ti->wc - Tc + 1);
    return reinterpret_cast<const double*>(m + umap_apex_offset(npos, static_cast<size_t>(ti->hc) * ti->wc));
}

}  // namespace ccwgpu
