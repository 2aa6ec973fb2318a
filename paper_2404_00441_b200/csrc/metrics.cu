// metrics.cu -- on-device validation metrics of simulated ensembles
// (proj/include/ccwsim/metrics.hpp:68-311): indicator variograms,
// connectivity functions, the ensemble average, block-majority
// downsampling, pattern histograms and their Jensen-Shannon divergence.
// They read realizations where ccw_simulate_device left them in HBM (or copy
// host grids once), so a 100-realization ensemble is validated without a
// CPU pass.
//
//   variogram     indicator planes bit-packed 64 cells per word; a lag is an
//                 XOR of a row with itself shifted (east-west) or with the row
//                 `lag` below (north-south), then popcounts
//   connectivity  4-connected components by lock-free union-find (CAS on the
//                 parent array, smaller index wins -- the reference's roots,
//                 metrics.hpp:116-154), then per-lag label comparisons with
//                 warp reductions
//   histograms    exact window keys (codes packed ceil(log2 F) bits each,
//                 <= 128 bits), radix-sorted, run-length counted on device
//   JS            merge of two sorted histograms by binary search, fp64 terms
//                 summed per block and then in block order (deterministic)
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "ccw_device.cuh"
#include "internal.hpp"

namespace ccwgpu {

namespace {

// ------------------------------------------------------------ inputs -----
// Host grids are copied once; device grids are read in place.
struct GridInput {
    const uint8_t* d = nullptr;
    uint8_t* owned = nullptr;
    GridInput(const uint8_t* p, bool on_device, size_t bytes, cudaStream_t st) {
        if (on_device) {
            d = p;
        } else {
            CCW_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&owned), std::max<size_t>(bytes, 1), st));
            CCW_CUDA(cudaMemcpyAsync(owned, p, bytes, cudaMemcpyHostToDevice, st));
            d = owned;
        }
    }
    void release(cudaStream_t st) {
        if (owned) cudaFreeAsync(owned, st);
        owned = nullptr;
    }
};

template <typename T>
struct Scratch {  // stream-ordered device scratch, freed with the scope
    T* p = nullptr;
    cudaStream_t st;
    Scratch(size_t n, cudaStream_t s) : st(s) {
        CCW_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), std::max<size_t>(n, 1) * sizeof(T), st));
    }
    ~Scratch() {
        if (p) cudaFreeAsync(p, st);
    }
};

// ---------------------------------------------------------- variogram ----
__global__ void pack_indicator_kernel(const uint8_t* __restrict__ g, int n, int h, int w, int nw, int facies,
                                      unsigned long long* __restrict__ bits) {
    const size_t total = static_cast<size_t>(n) * h * nw;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int k = static_cast<int>(e % nw);
        const size_t row = e / nw;  // (realization, row)
        const uint8_t* src = g + row * w + static_cast<size_t>(k) * 64;
        const int m = min(64, w - k * 64);
        unsigned long long v = 0;
        for (int j = 0; j < m; ++j) v |= static_cast<unsigned long long>(src[j] == facies) << j;
        bits[e] = v;
    }
}

__device__ __forceinline__ unsigned long long low_bits(int m) {
    return m >= 64 ? ~0ull : (m <= 0 ? 0ull : ((1ull << m) - 1));
}

// word k of row `rb` shifted down by `lag` cells (cells [64k + lag, 64k + lag + 64))
__device__ __forceinline__ unsigned long long shifted_word(const unsigned long long* rb, int nw, int k, int lag) {
    const int q = k + lag / 64, s = lag % 64;
    const unsigned long long a = q < nw ? rb[q] : 0ull;
    if (s == 0) return a;
    const unsigned long long b = q + 1 < nw ? rb[q + 1] : 0ull;
    return (a >> s) | (b << (64 - s));
}

__global__ void variogram_kernel(const unsigned long long* __restrict__ bits, int h, int w, int nw, int direction,
                                 double* __restrict__ gamma, int max_lag) {
    const int r = blockIdx.x, lag = blockIdx.y + 1;
    const unsigned long long* b = bits + static_cast<size_t>(r) * h * nw;
    long long diff = 0;
    if (direction == 0) {  // east_west: pairs (row, c), (row, c + lag), c + lag < w
        for (int e = threadIdx.x; e < h * nw; e += blockDim.x) {
            const int row = e / nw, k = e - row * nw;
            const unsigned long long* rb = b + static_cast<size_t>(row) * nw;
            const unsigned long long valid = low_bits(w - lag - 64 * k);
            diff += __popcll((rb[k] ^ shifted_word(rb, nw, k, lag)) & valid);
        }
    } else {  // north_south: pairs (row, c), (row + lag, c)
        for (int e = threadIdx.x; e < (h - lag) * nw; e += blockDim.x) {
            const int row = e / nw, k = e - row * nw;
            const unsigned long long valid = low_bits(w - 64 * k);
            diff += __popcll((b[static_cast<size_t>(row) * nw + k] ^ b[static_cast<size_t>(row + lag) * nw + k]) & valid);
        }
    }
    __shared__ long long red[32];
    for (int o = 16; o > 0; o >>= 1) diff += __shfl_xor_sync(0xffffffffu, diff, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = diff;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long s = 0;
        for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) s += red[i];
        const long long pairs = direction == 0 ? static_cast<long long>(h) * (w - lag)
                                               : static_cast<long long>(h - lag) * w;
        // metrics.hpp:107-108: 0.5 * sum_sq / pairs (indicator differences are 0 or 1)
        gamma[static_cast<size_t>(r) * max_lag + lag - 1] =
            pairs > 0 ? 0.5 * static_cast<double>(s) / static_cast<double>(pairs) : 0.0;
    }
}

__global__ void present_kernel(const unsigned long long* __restrict__ bits, size_t words_per_grid,
                               int* __restrict__ present) {
    const int r = blockIdx.x;
    int any = 0;
    for (size_t e = threadIdx.x; e < words_per_grid; e += blockDim.x) any |= bits[r * words_per_grid + e] != 0;
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) present[r] = any;
}

// ------------------------------------------------------- connectivity ----
__device__ __forceinline__ int uf_find(const int* parent, int x) {
    int p = __ldcg(parent + x);  // (L2: other SMs relink roots concurrently)
    while (p != x) {
        x = p;
        p = __ldcg(parent + x);
    }
    return x;
}

// link the roots of a and b: the larger root points at the smaller one
__device__ __forceinline__ void uf_union(int* parent, int a, int b) {
    for (;;) {
        a = uf_find(parent, a);
        b = uf_find(parent, b);
        if (a == b) return;
        if (a < b) {
            const int t = a;
            a = b;
            b = t;
        }
        const int old = atomicCAS(&parent[a], a, b);
        if (old == a) return;
        a = old;
    }
}

__global__ void ccl_init_kernel(const uint8_t* __restrict__ g, size_t cells, int facies, int* __restrict__ lab) {
    const int r = blockIdx.y;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < cells;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        lab[r * cells + i] = g[r * cells + i] == facies ? static_cast<int>(i) : -1;
}

__global__ void ccl_merge_kernel(const uint8_t* __restrict__ g, int h, int w, int facies, int* __restrict__ lab) {
    const int r = blockIdx.y;
    const size_t cells = static_cast<size_t>(h) * w;
    const uint8_t* gg = g + r * cells;
    int* parent = lab + r * cells;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < cells;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        if (gg[i] != facies) continue;
        const int c = static_cast<int>(i % w), row = static_cast<int>(i / w);
        if (c + 1 < w && gg[i + 1] == facies) uf_union(parent, static_cast<int>(i), static_cast<int>(i + 1));
        if (row + 1 < h && gg[i + w] == facies) uf_union(parent, static_cast<int>(i), static_cast<int>(i + w));
    }
}

__global__ void ccl_flatten_kernel(size_t cells, int* __restrict__ lab) {
    const int r = blockIdx.y;
    int* parent = lab + r * cells;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < cells;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        if (parent[i] >= 0) parent[i] = uf_find(parent, static_cast<int>(i));
}

// per (realization, lag): pairs of labelled cells, pairs in one component
__global__ void connectivity_kernel(const int* __restrict__ lab, int h, int w, int direction, int max_lag,
                                    unsigned long long* __restrict__ both, unsigned long long* __restrict__ conn) {
    extern __shared__ unsigned long long cs[];  // [2][max_lag]
    const int r = blockIdx.y;
    const size_t cells = static_cast<size_t>(h) * w;
    const int* L = lab + r * cells;
    for (int i = threadIdx.x; i < 2 * max_lag; i += blockDim.x) cs[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    // a warp walks 32 consecutive cells of one row at a time
    const size_t nchunk = (cells + 31) / 32;
    for (size_t ch = blockIdx.x * static_cast<size_t>(blockDim.x >> 5) + (threadIdx.x >> 5); ch < nchunk;
         ch += static_cast<size_t>(gridDim.x) * (blockDim.x >> 5)) {
        const size_t i = ch * 32 + lane;
        const bool in = i < cells;
        const int la = in ? L[i] : -1;
        const int c = in ? static_cast<int>(i % w) : 0, row = in ? static_cast<int>(i / w) : 0;
        if (!__any_sync(0xffffffffu, la >= 0)) continue;
        for (int lag = 1; lag <= max_lag; ++lag) {
            int lb = -1;
            if (la >= 0) {
                if (direction == 0) {
                    if (c + lag < w) lb = L[i + lag];
                } else if (row + lag < h) {
                    lb = L[i + static_cast<size_t>(lag) * w];
                }
            }
            const unsigned b = __ballot_sync(0xffffffffu, la >= 0 && lb >= 0);
            const unsigned e = __ballot_sync(0xffffffffu, la >= 0 && lb >= 0 && la == lb);
            if (lane == 0 && b) {
                atomicAdd(&cs[lag - 1], static_cast<unsigned long long>(__popc(b)));
                atomicAdd(&cs[max_lag + lag - 1], static_cast<unsigned long long>(__popc(e)));
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < max_lag; i += blockDim.x) {
        if (cs[i]) atomicAdd(&both[static_cast<size_t>(r) * max_lag + i], cs[i]);
        if (cs[max_lag + i]) atomicAdd(&conn[static_cast<size_t>(r) * max_lag + i], cs[max_lag + i]);
    }
}

// ----------------------------------------------------- ensemble average --
__global__ void ensemble_average_kernel(const uint8_t* __restrict__ g, int n, size_t cells, int facies,
                                        double* __restrict__ out) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < cells;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        double v = 0.0;  // metrics.hpp:220-224: += 1.0 per hit, then / n
        for (int r = 0; r < n; ++r)
            if (g[r * cells + i] == facies) v += 1.0;
        out[i] = v / static_cast<double>(n);
    }
}

// ----------------------------------------------------- downsampling ------
__global__ void downsample_kernel(const uint8_t* __restrict__ g, int h, int w, int nf, int factor,
                                  uint8_t* __restrict__ out) {
    const int oh = h / factor, ow = w / factor;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < static_cast<size_t>(oh) * ow;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(e / ow), j = static_cast<int>(e % ow);
        int cnt[256];
        for (int f = 0; f < nf; ++f) cnt[f] = 0;
        for (int r = 0; r < factor; ++r)
            for (int c = 0; c < factor; ++c) ++cnt[g[static_cast<size_t>(i * factor + r) * w + j * factor + c]];
        int best = 0;
        for (int f = 1; f < nf; ++f)
            if (cnt[f] > cnt[best]) best = f;  // ties keep the lowest code (metrics.hpp:305-307)
        out[e] = static_cast<uint8_t>(best);
    }
}

// ------------------------------------------------------- histograms ------
__global__ void window_keys_kernel(const uint8_t* __restrict__ g, int w, int win, int stride, int nx, int ny,
                                   int bpc, uint64_t* __restrict__ lo, uint64_t* __restrict__ hi) {
    const size_t n = static_cast<size_t>(nx) * ny;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int top = static_cast<int>(e / ny) * stride, left = static_cast<int>(e % ny) * stride;
        uint64_t a = 0, b = 0;
        int bit = 0;
        for (int r = 0; r < win; ++r)
            for (int c = 0; c < win; ++c, bit += bpc) {
                const uint64_t v = g[static_cast<size_t>(top + r) * w + left + c];
                if (bit < 64) {
                    a |= v << bit;
                    if (bit + bpc > 64) b |= v >> (64 - bit);
                } else {
                    b |= v << (bit - 64);
                }
            }
        lo[e] = a;
        hi[e] = b;
    }
}

__global__ void head_flags_kernel(const uint64_t* __restrict__ lo, const uint64_t* __restrict__ hi, size_t n,
                                  int* __restrict__ head) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        head[i] = i == 0 || lo[i] != lo[i - 1] || hi[i] != hi[i - 1];
}

__global__ void compact_kernel(const uint64_t* __restrict__ lo, const uint64_t* __restrict__ hi, size_t n,
                               const int* __restrict__ head, const int* __restrict__ pos, uint64_t* __restrict__ ulo,
                               uint64_t* __restrict__ uhi, uint64_t* __restrict__ start) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        if (head[i]) {
            ulo[pos[i]] = lo[i];
            uhi[pos[i]] = hi[i];
            start[pos[i]] = i;
        }
}

// multiplicity of each distinct key: distance to the next key's first window
__global__ void counts_kernel(const uint64_t* __restrict__ start, int64_t nu, uint64_t total,
                              uint64_t* __restrict__ cnt) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nu;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        cnt[i] = (i + 1 < nu ? start[i + 1] : total) - start[i];
}

// JS terms (metrics.hpp:269-282): for every key of `a`, its frequency in `b`
__global__ void js_terms_kernel(const uint64_t* __restrict__ alo, const uint64_t* __restrict__ ahi,
                                const uint64_t* __restrict__ acnt, int64_t na, double at,
                                const uint64_t* __restrict__ blo, const uint64_t* __restrict__ bhi,
                                const uint64_t* __restrict__ bcnt, int64_t nb, double bt, double* __restrict__ part) {
    double s = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < na;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t kh = ahi[i], kl = alo[i];
        int64_t lo = 0, hi = nb;  // first entry >= key in (hi, lo) order
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            const bool less = bhi[mid] < kh || (bhi[mid] == kh && blo[mid] < kl);
            if (less)
                lo = mid + 1;
            else
                hi = mid;
        }
        const double pp = static_cast<double>(acnt[i]) / at;
        const double qq = (lo < nb && bhi[lo] == kh && blo[lo] == kl) ? static_cast<double>(bcnt[lo]) / bt : 0.0;
        s += 0.5 * pp * log2(2.0 * pp / (pp + qq));
    }
    __shared__ double red[32];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < static_cast<int>(blockDim.x >> 5); ++k) t += red[k];
        part[blockIdx.x] = t;
    }
}

__global__ void sum_parts_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += part[i];
        *out = s;
    }
}

// One histogram of a batch (ANODI): device arrays + counts.
struct HistDesc {
    const uint64_t* lo;
    const uint64_t* hi;
    const uint64_t* cnt;
    int64_t n;
    double total;
};

// JS divergence of every listed histogram pair, one CTA per pair: the terms of
// js_terms_kernel, reduced per CTA in a fixed order.
__global__ void js_pairs_kernel(const HistDesc* __restrict__ hd, const int2* __restrict__ pairs,
                                double* __restrict__ out) {
    const int2 pr = pairs[blockIdx.x];
    __shared__ double red[32];
    double s = 0.0;
    for (int side = 0; side < 2; ++side) {
        const HistDesc a = hd[side ? pr.y : pr.x], b = hd[side ? pr.x : pr.y];
        for (int64_t i = threadIdx.x; i < a.n; i += blockDim.x) {
            const uint64_t kh = a.hi[i], kl = a.lo[i];
            int64_t lo = 0, hi = b.n;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                const bool less = b.hi[mid] < kh || (b.hi[mid] == kh && b.lo[mid] < kl);
                if (less)
                    lo = mid + 1;
                else
                    hi = mid;
            }
            const double pp = static_cast<double>(a.cnt[i]) / a.total;
            const double qq = (lo < b.n && b.hi[lo] == kh && b.lo[lo] == kl) ? static_cast<double>(b.cnt[lo]) / b.total
                                                                             : 0.0;
            s += 0.5 * pp * log2(2.0 * pp / (pp + qq));
        }
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < static_cast<int>(blockDim.x >> 5); ++k) t += red[k];
        out[blockIdx.x] = fmin(fmax(t, 0.0), 1.0);  // metrics.hpp:283
    }
}

int grid_for(size_t n) { return static_cast<int>(std::min<size_t>((n + 255) / 256, 148 * 16)); }

}  // namespace

void metric_variogram(ccw_ctx* ctx, const uint8_t* grids, bool on_device, int n, int h, int w, int facies,
                      int direction, int max_lag, double* gamma, int32_t* present) {
    cudaStream_t st = ctx->stream;
    GridInput in(grids, on_device, static_cast<size_t>(n) * h * w, st);
    const int nw = (w + 63) / 64;
    Scratch<unsigned long long> bits(static_cast<size_t>(n) * h * nw, st);
    Scratch<double> dg(static_cast<size_t>(n) * max_lag, st);
    Scratch<int> dp(n, st);
    pack_indicator_kernel<<<grid_for(static_cast<size_t>(n) * h * nw), 256, 0, st>>>(in.d, n, h, w, nw, facies,
                                                                                   bits.p);
    variogram_kernel<<<dim3(n, max_lag), 256, 0, st>>>(bits.p, h, w, nw, direction, dg.p, max_lag);
    present_kernel<<<n, 256, 0, st>>>(bits.p, static_cast<size_t>(h) * nw, dp.p);
    CCW_CUDA(cudaGetLastError());
    CCW_CUDA(cudaMemcpyAsync(gamma, dg.p, sizeof(double) * n * max_lag, cudaMemcpyDeviceToHost, st));
    if (present) CCW_CUDA(cudaMemcpyAsync(present, dp.p, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
    in.release(st);
    CCW_CUDA(cudaStreamSynchronize(st));
}

void metric_connectivity(ccw_ctx* ctx, const uint8_t* grids, bool on_device, int n, int h, int w, int facies,
                         int direction, int max_lag, double* prob) {
    cudaStream_t st = ctx->stream;
    const size_t cells = static_cast<size_t>(h) * w;
    GridInput in(grids, on_device, n * cells, st);
    Scratch<int> lab(n * cells, st);
    Scratch<unsigned long long> cnt(2 * static_cast<size_t>(n) * max_lag, st);
    CCW_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long) * 2 * n * max_lag, st));
    const dim3 g2(std::min<unsigned>(static_cast<unsigned>((cells + 255) / 256), 1024u), n);
    ccl_init_kernel<<<g2, 256, 0, st>>>(in.d, cells, facies, lab.p);
    ccl_merge_kernel<<<g2, 256, 0, st>>>(in.d, h, w, facies, lab.p);
    ccl_flatten_kernel<<<g2, 256, 0, st>>>(cells, lab.p);
    const size_t smem = sizeof(unsigned long long) * 2 * max_lag;
    if (smem > 200 * 1024) throw Fail(CCW_ERR_DIMENSION, "max_lag too large for the on-device connectivity");
    CCW_CUDA(cudaFuncSetAttribute(connectivity_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    const dim3 g3(std::min<unsigned>(static_cast<unsigned>((cells + 255) / 256), 256u), n);
    connectivity_kernel<<<g3, 256, smem, st>>>(lab.p, h, w, direction, max_lag, cnt.p, cnt.p + n * max_lag);
    CCW_CUDA(cudaGetLastError());
    std::vector<unsigned long long> hc(2 * static_cast<size_t>(n) * max_lag);
    CCW_CUDA(cudaMemcpyAsync(hc.data(), cnt.p, sizeof(unsigned long long) * hc.size(), cudaMemcpyDeviceToHost, st));
    in.release(st);
    CCW_CUDA(cudaStreamSynchronize(st));
    for (size_t i = 0; i < static_cast<size_t>(n) * max_lag; ++i) {
        const unsigned long long both = hc[i], conn = hc[static_cast<size_t>(n) * max_lag + i];
        // metrics.hpp:199-201: undefined lags stay unset (NaN here)
        prob[i] = both > 0 ? static_cast<double>(conn) / static_cast<double>(both) : NAN;
    }
}

void metric_ensemble_average(ccw_ctx* ctx, const uint8_t* grids, bool on_device, int n, int h, int w, int facies,
                             double* out) {
    cudaStream_t st = ctx->stream;
    const size_t cells = static_cast<size_t>(h) * w;
    GridInput in(grids, on_device, n * cells, st);
    Scratch<double> d(cells, st);
    ensemble_average_kernel<<<grid_for(cells), 256, 0, st>>>(in.d, n, cells, facies, d.p);
    CCW_CUDA(cudaGetLastError());
    CCW_CUDA(cudaMemcpyAsync(out, d.p, sizeof(double) * cells, cudaMemcpyDeviceToHost, st));
    in.release(st);
    CCW_CUDA(cudaStreamSynchronize(st));
}

void metric_downsample(ccw_ctx* ctx, const uint8_t* grid, bool on_device, int h, int w, int nf, int factor,
                       uint8_t* out, bool out_on_device) {
    cudaStream_t st = ctx->stream;
    GridInput in(grid, on_device, static_cast<size_t>(h) * w, st);
    const size_t on = static_cast<size_t>(h / factor) * (w / factor);
    Scratch<uint8_t> d(out_on_device ? 0 : on, st);
    uint8_t* dst = out_on_device ? out : d.p;
    downsample_kernel<<<grid_for(on), 256, 0, st>>>(in.d, h, w, nf, factor, dst);
    CCW_CUDA(cudaGetLastError());
    if (!out_on_device) CCW_CUDA(cudaMemcpyAsync(out, d.p, on, cudaMemcpyDeviceToHost, st));
    in.release(st);
    CCW_CUDA(cudaStreamSynchronize(st));
}

ccw_phist* metric_pattern_histogram(ccw_ctx* ctx, const uint8_t* grid, bool on_device, int h, int w, int nf,
                                    int win, int stride) {
    cudaStream_t st = ctx->stream;
    int bpc = 1;
    while ((1 << bpc) < nf) ++bpc;
    if (win * win * bpc > 128)
        throw Fail(CCW_ERR_DIMENSION, "window too large for exact 128-bit on-device pattern keys");
    GridInput in(grid, on_device, static_cast<size_t>(h) * w, st);
    const int nx = (h - win) / stride + 1, ny = (w - win) / stride + 1;
    const size_t n = static_cast<size_t>(nx) * ny;
    Scratch<uint64_t> klo(n, st), khi(n, st), slo(n, st), shi(n, st), tlo(n, st), thi(n, st);
    window_keys_kernel<<<grid_for(n), 256, 0, st>>>(in.d, w, win, stride, nx, ny, bpc, klo.p, khi.p);
    CCW_CUDA(cudaGetLastError());
    // (hi, lo) order: stable LSD radix sort by lo, then by hi
    size_t tmp_bytes = 0, t2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, klo.p, tlo.p, khi.p, thi.p, static_cast<int64_t>(n), 0, 64, st);
    cub::DeviceRadixSort::SortPairs(nullptr, t2, thi.p, shi.p, tlo.p, slo.p, static_cast<int64_t>(n), 0, 64, st);
    Scratch<uint8_t> tmp(std::max(tmp_bytes, t2), st);
    tmp_bytes = std::max(tmp_bytes, t2);
    const int hib = std::max(0, win * win * bpc - 64);  // significant bits of hi
    CCW_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, klo.p, tlo.p, khi.p, thi.p, static_cast<int64_t>(n), 0,
                                             std::min(64, win * win * bpc), st));
    if (hib > 0)
        CCW_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, thi.p, shi.p, tlo.p, slo.p, static_cast<int64_t>(n),
                                                 0, hib, st));
    const uint64_t* lo = hib > 0 ? slo.p : tlo.p;
    const uint64_t* hi = hib > 0 ? shi.p : thi.p;
    Scratch<int> head(n, st), pos(n, st);
    head_flags_kernel<<<grid_for(n), 256, 0, st>>>(lo, hi, n, head.p);
    size_t sb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, sb, head.p, pos.p, static_cast<int64_t>(n), st);
    Scratch<uint8_t> stmp(sb, st);
    CCW_CUDA(cub::DeviceScan::ExclusiveSum(stmp.p, sb, head.p, pos.p, static_cast<int64_t>(n), st));
    int last_pos = 0, last_head = 0;
    CCW_CUDA(cudaMemcpyAsync(&last_pos, pos.p + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    CCW_CUDA(cudaMemcpyAsync(&last_head, head.p + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    CCW_CUDA(cudaStreamSynchronize(st));
    const int64_t nu = static_cast<int64_t>(last_pos) + last_head;
    auto* hist = new ccw_phist();
    hist->device = ctx->device;
    hist->window = win;
    hist->bpc = bpc;
    hist->n = nu;
    hist->total = n;
    try {
        CCW_CUDA(cudaMalloc(&hist->lo, sizeof(uint64_t) * std::max<int64_t>(nu, 1)));
        CCW_CUDA(cudaMalloc(&hist->hi, sizeof(uint64_t) * std::max<int64_t>(nu, 1)));
        CCW_CUDA(cudaMalloc(&hist->cnt, sizeof(uint64_t) * std::max<int64_t>(nu, 1)));
        Scratch<uint64_t> start(nu, st);
        compact_kernel<<<grid_for(n), 256, 0, st>>>(lo, hi, n, head.p, pos.p, hist->lo, hist->hi, start.p);
        counts_kernel<<<grid_for(static_cast<size_t>(nu)), 256, 0, st>>>(start.p, nu, n, hist->cnt);
        CCW_CUDA(cudaGetLastError());
        in.release(st);
        CCW_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
        cudaFree(hist->lo);
        cudaFree(hist->hi);
        cudaFree(hist->cnt);
        delete hist;
        throw;
    }
    return hist;
}

double metric_js(ccw_ctx* ctx, const ccw_phist* p, const ccw_phist* q) {
    cudaStream_t st = ctx->stream;
    const int bp = static_cast<int>(std::min<int64_t>((p->n + 255) / 256, 1024));
    const int bq = static_cast<int>(std::min<int64_t>((q->n + 255) / 256, 1024));
    Scratch<double> part(bp + bq + 1, st);
    js_terms_kernel<<<std::max(bp, 1), 256, 0, st>>>(p->lo, p->hi, p->cnt, p->n, static_cast<double>(p->total), q->lo,
                                                     q->hi, q->cnt, q->n, static_cast<double>(q->total), part.p);
    js_terms_kernel<<<std::max(bq, 1), 256, 0, st>>>(q->lo, q->hi, q->cnt, q->n, static_cast<double>(q->total), p->lo,
                                                     p->hi, p->cnt, p->n, static_cast<double>(p->total),
                                                     part.p + std::max(bp, 1));
    sum_parts_kernel<<<1, 32, 0, st>>>(part.p, std::max(bp, 1) + std::max(bq, 1), part.p + bp + bq);
    CCW_CUDA(cudaGetLastError());
    double s = 0.0;
    CCW_CUDA(cudaMemcpyAsync(&s, part.p + bp + bq, sizeof(double), cudaMemcpyDeviceToHost, st));
    CCW_CUDA(cudaStreamSynchronize(st));
    return std::clamp(s, 0.0, 1.0);  // metrics.hpp:283
}

// anodi (metrics.hpp:318-384, without MDS).  out: levels x 8 doubles.
void metric_anodi(ccw_ctx* ctx, const uint8_t* ga, int na, const uint8_t* gb, int nb, bool on_device, int h, int w,
                  const uint8_t* ti, int th, int tw, int nf, int levels, int win, const double* weights, double* out,
                  double* aggregate) {
    cudaStream_t st = ctx->stream;
    const size_t cells = static_cast<size_t>(h) * w;
    GridInput ia(ga, on_device, na * cells, st), ib(gb, on_device, nb * cells, st);
    GridInput it(ti, false, static_cast<size_t>(th) * tw, st);
    *aggregate = 0.0;
    for (int p = 1; p <= levels; ++p) {
        const int factor = 1 << (p - 1);
        const int oh = h / factor, ow = w / factor, toh = th / factor, tow = tw / factor;
        if (oh < win || ow < win || toh < win || tow < win)
            throw Fail(CCW_ERR_DIMENSION, "window does not fit the level-" + std::to_string(p) + " grids");
        Scratch<uint8_t> da(factor > 1 ? static_cast<size_t>(na) * oh * ow : 0, st),
            db(factor > 1 ? static_cast<size_t>(nb) * oh * ow : 0, st), dt(static_cast<size_t>(toh) * tow, st);
        // downsample_majority of every grid (the level-1 grids are used as they are)
        auto down = [&](const uint8_t* src, int hh, int ww, uint8_t* dst) {
            metric_downsample(ctx, src, true, hh, ww, nf, factor, dst, true);
        };
        std::vector<const uint8_t*> pa(na), pb(nb);
        for (int r = 0; r < na; ++r) {
            if (factor > 1) down(ia.d + r * cells, h, w, da.p + static_cast<size_t>(r) * oh * ow);
            pa[r] = factor > 1 ? da.p + static_cast<size_t>(r) * oh * ow : ia.d + r * cells;
        }
        for (int r = 0; r < nb; ++r) {
            if (factor > 1) down(ib.d + r * cells, h, w, db.p + static_cast<size_t>(r) * oh * ow);
            pb[r] = factor > 1 ? db.p + static_cast<size_t>(r) * oh * ow : ib.d + r * cells;
        }
        if (factor > 1)
            down(it.d, th, tw, dt.p);
        else
            CCW_CUDA(cudaMemcpyAsync(dt.p, it.d, static_cast<size_t>(th) * tw, cudaMemcpyDeviceToDevice, st));
        // pattern histograms: [A..., B..., TI]
        std::vector<ccw_phist*> hs;
        struct Free {
            std::vector<ccw_phist*>& v;
            ~Free() {
                for (ccw_phist* x : v) metric_phist_destroy(x);
            }
        } free_hs{hs};
        for (int r = 0; r < na; ++r) hs.push_back(metric_pattern_histogram(ctx, pa[r], true, oh, ow, nf, win, 1));
        for (int r = 0; r < nb; ++r) hs.push_back(metric_pattern_histogram(ctx, pb[r], true, oh, ow, nf, win, 1));
        hs.push_back(metric_pattern_histogram(ctx, dt.p, true, toh, tow, nf, win, 1));
        std::vector<HistDesc> desc;
        for (ccw_phist* x : hs) desc.push_back({x->lo, x->hi, x->cnt, x->n, static_cast<double>(x->total)});
        // pairs in the reference's order: A pairs, B pairs, A vs TI, B vs TI
        std::vector<int2> pairs;
        for (int i = 0; i < na; ++i)
            for (int j = i + 1; j < na; ++j) pairs.push_back(make_int2(i, j));
        for (int i = 0; i < nb; ++i)
            for (int j = i + 1; j < nb; ++j) pairs.push_back(make_int2(na + i, na + j));
        const int tix = na + nb;
        for (int i = 0; i < na; ++i) pairs.push_back(make_int2(i, tix));
        for (int i = 0; i < nb; ++i) pairs.push_back(make_int2(na + i, tix));
        Scratch<HistDesc> ddesc(desc.size(), st);
        Scratch<int2> dpairs(pairs.size(), st);
        Scratch<double> djs(pairs.size(), st);
        CCW_CUDA(cudaMemcpyAsync(ddesc.p, desc.data(), sizeof(HistDesc) * desc.size(), cudaMemcpyHostToDevice, st));
        CCW_CUDA(cudaMemcpyAsync(dpairs.p, pairs.data(), sizeof(int2) * pairs.size(), cudaMemcpyHostToDevice, st));
        js_pairs_kernel<<<static_cast<unsigned>(pairs.size()), 256, 0, st>>>(ddesc.p, dpairs.p, djs.p);
        CCW_CUDA(cudaGetLastError());
        std::vector<double> js(pairs.size());
        CCW_CUDA(cudaMemcpyAsync(js.data(), djs.p, sizeof(double) * js.size(), cudaMemcpyDeviceToHost, st));
        CCW_CUDA(cudaStreamSynchronize(st));
        // means in the reference's summation order (metrics.hpp:340-356)
        size_t k = 0;
        double s = 0.0;
        const size_t npa = static_cast<size_t>(na) * (na - 1) / 2, npb = static_cast<size_t>(nb) * (nb - 1) / 2;
        for (size_t q = 0; q < npa; ++q) s += js[k++];
        const double between_a = s / static_cast<double>(npa);
        s = 0.0;
        for (size_t q = 0; q < npb; ++q) s += js[k++];
        const double between_b = s / static_cast<double>(npb);
        s = 0.0;
        for (int q = 0; q < na; ++q) s += js[k++];
        const double within_a = s / na;
        s = 0.0;
        for (int q = 0; q < nb; ++q) s += js[k++];
        const double within_b = s / nb;
        double* o = out + static_cast<size_t>(p - 1) * 8;
        o[0] = between_a;
        o[1] = between_b;
        o[2] = within_a;
        o[3] = within_b;
        o[7] = weights ? weights[p - 1] : 1.0 / levels;
        if (within_a == 0.0 || within_b == 0.0)
            throw Fail(CCW_ERR_DEGENERACY, "realizations identical to TI at level " + std::to_string(p));
        if (between_b == 0.0)
            throw Fail(CCW_ERR_DEGENERACY,
                       "ensemble B has zero between-realization variability at level " + std::to_string(p));
        o[4] = between_a / between_b;
        o[5] = within_a / within_b;
        o[6] = o[4] / o[5];
        *aggregate += o[7] * o[6];
    }
    ia.release(st);
    ib.release(st);
    it.release(st);
    CCW_CUDA(cudaStreamSynchronize(st));
}

void metric_phist_copy(ccw_ctx* ctx, const ccw_phist* h, uint8_t* keys, uint64_t* counts) {
    cudaStream_t st = ctx->stream;
    std::vector<uint64_t> lo(static_cast<size_t>(h->n)), hi(static_cast<size_t>(h->n));
    CCW_CUDA(cudaMemcpyAsync(lo.data(), h->lo, sizeof(uint64_t) * h->n, cudaMemcpyDeviceToHost, st));
    CCW_CUDA(cudaMemcpyAsync(hi.data(), h->hi, sizeof(uint64_t) * h->n, cudaMemcpyDeviceToHost, st));
    if (counts) CCW_CUDA(cudaMemcpyAsync(counts, h->cnt, sizeof(uint64_t) * h->n, cudaMemcpyDeviceToHost, st));
    CCW_CUDA(cudaStreamSynchronize(st));
    if (!keys) return;
    const int kw = h->window * h->window, bpc = h->bpc;
    const uint64_t m = (1ull << bpc) - 1;
    for (int64_t i = 0; i < h->n; ++i)
        for (int k = 0; k < kw; ++k) {
            const int bit = k * bpc;
            uint64_t v;
            if (bit + bpc <= 64)
                v = lo[i] >> bit;
            else if (bit >= 64)
                v = hi[i] >> (bit - 64);
            else
                v = (lo[i] >> bit) | (hi[i] << (64 - bit));
            keys[static_cast<size_t>(i) * kw + k] = static_cast<uint8_t>(v & m);
        }
}

void metric_phist_destroy(ccw_phist* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    cudaFree(h->lo);
    cudaFree(h->hi);
    cudaFree(h->cnt);
    delete h;
}

}  // namespace ccwgpu
