// sim.cu -- the batched, wavefront-scheduled CCWSIM simulation on sm_100a:
// the host driver (run_simulation) and the finalize kernels.
//
// One ccw_simulate call runs every realization in lock-step.  Placements of
// all realizations are grouped into waves by the key (d+1)*o + i of their
// raster coordinates (o outer, i inner; d = how many stride steps a footprint
// reaches), which orders every pair of overlapping footprints exactly as the
// reference's raster loop does (simulator.hpp:447-496) while letting the
// placements of one wave run concurrently.  Per wave and realization group:
//
//   or_prep      overlap region -> exact-integer screen weights and the
//                reference-order fp64 OR apex (simulator.hpp:455-460)   prep.cu
//   ccf_tc       exact-integer CCF screen over every TI window, int8 tcgen05
//                GEMM (matcher.hpp:64-81 up to a per-job constant)       ccf_tc.cu
//                (ccf_direct: the CUDA-core fallback)                    ccf_direct.cu
//   select       exact K-th-largest threshold, fp64 reference-order
//                rescoring of equal-score candidates, top-K ordering
//                (matcher.hpp:177-204), unconditional / conditional pick
//                (matcher.hpp:207-241), optional min-cut stitch
//                (simulator.hpp:286-374), paste / source-block map     select.cu
//
// and finalize rebuilds the realizations (progressively for host results),
// applies the hard-data overwrite and crops (simulator.hpp:506-515).
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

#include <immintrin.h>

#include "sim_kernels.cuh"

namespace ccwgpu {

// ----------------------------------------------------------- finalize ----

__global__ void fill_i32_kernel(int32_t* __restrict__ p, size_t n, int32_t v) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        p[i] = v;
}

void fill_i32(int32_t* p, size_t n, int32_t v, cudaStream_t st) {
    if (!p || n == 0) return;
    fill_i32_kernel<<<static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 4 * 148)), 256, 0, st>>>(p, n, v);
    CCW_CUDA(cudaGetLastError());
}

__global__ void hd_scatter_kernel(const int32_t* __restrict__ hd, int n_hd, uint8_t* plane, int ww) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_hd) plane[static_cast<size_t>(hd[3 * i]) * ww + hd[3 * i + 1]] = static_cast<uint8_t>(hd[3 * i + 2]);
}

// Hard-data CSR per stride-lattice cell (a placement's footprint origin):
// entries (footprint cell r * T + c) << 8 | facies.  Count, scan, fill; the
// order inside a cell is free (the conditional choice sums mismatches).
__device__ __forceinline__ void hd_cells(const int32_t* hd, int i, int T, int stride, int nlr, int nlc, int& qr0,
                                         int& qr1, int& qc0, int& qc1) {
    const int r = hd[3 * i], c = hd[3 * i + 1];
    qr0 = max(0, (r - T + 1 + stride - 1) / stride);
    qc0 = max(0, (c - T + 1 + stride - 1) / stride);
    qr1 = min(nlr - 1, r / stride);
    qc1 = min(nlc - 1, c / stride);
}

__global__ void hd_count_kernel(const int32_t* __restrict__ hd, int n, int T, int stride, int nlr, int nlc,
                                int32_t* __restrict__ cnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int qr0, qr1, qc0, qc1;
    hd_cells(hd, i, T, stride, nlr, nlc, qr0, qr1, qc0, qc1);
    const int r = hd[3 * i], c = hd[3 * i + 1];
    for (int qr = qr0; qr <= qr1; ++qr)
        for (int qc = qc0; qc <= qc1; ++qc)
            if (r >= qr * stride && r < qr * stride + T && c >= qc * stride && c < qc * stride + T)
                atomicAdd(&cnt[static_cast<size_t>(qr) * nlc + qc], 1);
}

// One CTA: off[0..ncell] (off[q + 1] holds cell q's count on entry) becomes the
// exclusive scan; cursors = a copy of the starts; lattice[q] = cell q holds data.
__global__ void hd_scan_kernel(int32_t* __restrict__ off, int ncell, int32_t* __restrict__ cursors,
                               uint8_t* __restrict__ lattice) {
    __shared__ int part[32];
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int base = 0; base < ncell; base += blockDim.x) {
        const int q = base + threadIdx.x;
        const int v = q < ncell ? off[q + 1] : 0;
        if (q < ncell) lattice[q] = v > 0;
        int x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) part[wid] = x;
        __syncthreads();
        if (wid == 0) {
            int p = lane < static_cast<int>(blockDim.x >> 5) ? part[lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, p, o);
                if (lane >= o) p += y;
            }
            part[lane] = p;
        }
        __syncthreads();
        const int incl = x + (wid > 0 ? part[wid - 1] : 0) + carry;
        if (q < ncell) {
            off[q + 1] = incl;
            cursors[q] = incl - v;
        }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) off[0] = 0;
}

__global__ void hd_fill_kernel(const int32_t* __restrict__ hd, int n, int T, int stride, int nlr, int nlc,
                               int32_t* __restrict__ cursors, uint32_t* __restrict__ ent) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int qr0, qr1, qc0, qc1;
    hd_cells(hd, i, T, stride, nlr, nlc, qr0, qr1, qc0, qc1);
    const int r = hd[3 * i], c = hd[3 * i + 1], v = hd[3 * i + 2];
    for (int qr = qr0; qr <= qr1; ++qr)
        for (int qc = qc0; qc <= qc1; ++qc)
            if (r >= qr * stride && r < qr * stride + T && c >= qc * stride && c < qc * stride + T) {
                const int at = atomicAdd(&cursors[static_cast<size_t>(qr) * nlc + qc], 1);
                ent[at] = (static_cast<uint32_t>((r - qr * stride) * T + (c - qc * stride)) << 8) | static_cast<uint32_t>(v);
            }
}

// Rebuild (and hard-data overwrite) the output cells of rows [y0, y1) x columns
// [x0, x1) of realization r.  With the source-block map, one thread per
// coarse block: one map entry, then the B x B TI patch (BT = B for 2/4/8; 0 =
// one thread per cell, for min-cut's work grid or large blocks).
template <int BT>
__device__ __forceinline__ void finalize_region(int r, int y0, int y1, int x0, int x1,
                                                const uint8_t* __restrict__ work, int wh, int ww,
                                                const int32_t* __restrict__ src, int B, int J, int swc,
                                                const uint8_t* __restrict__ ti, int ti_w, int wc,
                                                const uint8_t* __restrict__ hd, int sg_h, int sg_w,
                                                uint8_t* __restrict__ obase, int opitch, int& local) {
    // cell (y, x) of the region goes to obase[(y - y0) * opitch + (x - x0)]
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    const uint8_t* hp = hd;
    if constexpr (BT == 0) {
        const uint8_t* g = work ? work + static_cast<size_t>(r) * wh * ww : nullptr;
        const int32_t* sm = src ? src + static_cast<size_t>(r) * (wh >> J) * swc : nullptr;
        const int cols = x1 - x0;
        const size_t n = static_cast<size_t>(y1 - y0) * cols;
        for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += stride) {
            const int y = y0 + static_cast<int>(e / cols), x = x0 + static_cast<int>(e % cols);
            uint8_t v;
            if (g) {
                v = g[static_cast<size_t>(y) * ww + x];
            } else {
                const int b = sm[static_cast<size_t>(y >> J) * swc + (x >> J)];
                const int by = b / wc, bx = b - by * wc;
                v = ti[static_cast<size_t>((by << J) + (y & (B - 1))) * ti_w + (bx << J) + (x & (B - 1))];
            }
            if (hp) {
                const uint8_t h = hp[static_cast<size_t>(y) * ww + x];
                if (h != kNoDatum) {
                    local += v != h;
                    v = h;
                }
            }
            obase[static_cast<size_t>(y - y0) * opitch + (x - x0)] = v;
        }
    } else {
        const int32_t* sm = src + static_cast<size_t>(r) * (wh >> J) * swc;
        const int by0 = y0 / BT, by1 = (y1 + BT - 1) / BT, bx0 = x0 / BT, bx1 = (x1 + BT - 1) / BT;
        const int nbw = bx1 - bx0;
        const size_t nb = static_cast<size_t>(by1 - by0) * nbw;
        for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < nb; e += stride) {
            const int cby = by0 + static_cast<int>(e / nbw), cbx = bx0 + static_cast<int>(e % nbw);
            const int b = sm[static_cast<size_t>(cby) * swc + cbx];
            const int tby = b / wc, tbx = b - tby * wc;
            const uint8_t* tp = ti + static_cast<size_t>(tby * BT) * ti_w + tbx * BT;
            uint8_t v[BT][BT];
#pragma unroll
            for (int i = 0; i < BT; ++i)
#pragma unroll
                for (int j = 0; j < BT; ++j) v[i][j] = tp[static_cast<size_t>(i) * ti_w + j];
#pragma unroll
            for (int i = 0; i < BT; ++i) {
                const int y = cby * BT + i;
                if (y < y0 || y >= y1) continue;
#pragma unroll
                for (int j = 0; j < BT; ++j) {
                    const int x = cbx * BT + j;
                    if (x < x0 || x >= x1) continue;
                    uint8_t w = v[i][j];
                    if (hp) {
                        const uint8_t h = hp[static_cast<size_t>(y) * ww + x];
                        if (h != kNoDatum) {
                            local += w != h;
                            w = h;
                        }
                    }
                    obase[static_cast<size_t>(y - y0) * opitch + (x - x0)] = w;
                }
            }
        }
    }
}

template <int BT>
__global__ void finalize_kernel(const uint8_t* __restrict__ work, int wh, int ww,
                                const int32_t* __restrict__ src, int B, int J, int swc,
                                const uint8_t* __restrict__ ti, int ti_w, int wc,
                                const uint8_t* __restrict__ hd, int sg_h, int sg_w,
                                uint8_t* __restrict__ out, int* mism) {
    pdl_wait();
    const int r = blockIdx.y;
    int local = 0;
    finalize_region<BT>(r, 0, sg_h, 0, sg_w, work, wh, ww, src, B, J, swc, ti, ti_w, wc, hd, sg_h, sg_w,
                        out + static_cast<size_t>(r) * sg_h * sg_w, sg_w, local);
    if (hd) {
        for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
        if ((threadIdx.x & 31) == 0 && local) atomicAdd(&mism[r], local);
    }
}

// Progressive finalize: band descriptors (realization, axis, lo, hi) in
// output coordinates -- axis 0: rows [lo, hi) x every column; axis 1: every
// row x columns [lo, hi).  A band is final once every placement covering it
// is done (run_simulation's checkpoints), so it is rebuilt and copied to the
// host while later waves still compute.  With boff the band is written packed
// at out + boff[band] (axis 0: its rows; axis 1: rows of hi - lo bytes), so a
// checkpoint's bands leave in one contiguous copy; without, in place in the
// row-major realizations.
template <int BT>
__global__ void finalize_band_kernel(const int4* __restrict__ bands, const long long* __restrict__ boff,
                                     const uint8_t* __restrict__ work,
                                     int wh, int ww, const int32_t* __restrict__ src, int B, int J,
                                     int swc, const uint8_t* __restrict__ ti, int ti_w, int wc,
                                     const uint8_t* __restrict__ hd, int sg_h, int sg_w,
                                     uint8_t* __restrict__ out, int* mism, unsigned long long* tl) {
    tl_mark(tl, 2);
    pdl_wait();
    tl_mark(tl, 0);
    const int4 bd = bands[blockIdx.y];
    const int r = bd.x;
    const size_t rb = static_cast<size_t>(r) * sg_h * sg_w;
    int local = 0;
    if (bd.y == 0)
        finalize_region<BT>(r, bd.z, bd.w, 0, sg_w, work, wh, ww, src, B, J, swc, ti, ti_w, wc, hd, sg_h, sg_w,
                            boff ? out + boff[blockIdx.y] : out + rb + static_cast<size_t>(bd.z) * sg_w, sg_w,
                            local);
    else
        finalize_region<BT>(r, 0, sg_h, bd.z, bd.w, work, wh, ww, src, B, J, swc, ti, ti_w, wc, hd, sg_h, sg_w,
                            boff ? out + boff[blockIdx.y] : out + rb + bd.z, boff ? bd.w - bd.z : sg_w, local);
    if (hd) {
        for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
        if ((threadIdx.x & 31) == 0 && local) atomicAdd(&mism[r], local);
    }
    tl_mark(tl, 1);
}

// Streamed bands with few facies: the same cells as finalize_band_kernel
// (map -> TI cell, hard-data overwrite, mismatch count), written BITS per
// cell (1, 2 or 4; cell c of a byte in bits [c*BITS, (c+1)*BITS)), each
// band row padded to whole bytes -- the device->host copy shrinks 8/BITS-fold
// and the host unpacks while placing the bands.
template <int BITS>
__global__ void pack_band_kernel(const int4* __restrict__ bands, const long long* __restrict__ boff,
                                 const uint8_t* __restrict__ work, int wh, int ww, const int32_t* __restrict__ src,
                                 int B, int J, int swc, const uint8_t* __restrict__ ti, int ti_w, int wc,
                                 const uint8_t* __restrict__ hd, int sg_h, int sg_w, uint8_t* __restrict__ out,
                                 int* mism, unsigned long long* tl) {
    constexpr int CPB = 8 / BITS;
    tl_mark(tl, 2);
    pdl_wait();
    tl_mark(tl, 0);
    const int4 bd = bands[blockIdx.y];
    const int r = bd.x;
    const int y0 = bd.y == 0 ? bd.z : 0, y1 = bd.y == 0 ? bd.w : sg_h;
    const int x0 = bd.y == 0 ? 0 : bd.z, x1 = bd.y == 0 ? sg_w : bd.w;
    const int rowb = (x1 - x0 + CPB - 1) / CPB;
    const size_t nbytes = static_cast<size_t>(y1 - y0) * rowb;
    uint8_t* o = out + boff[blockIdx.y];
    const uint8_t* g = work ? work + static_cast<size_t>(r) * wh * ww : nullptr;
    const int32_t* sm = src ? src + static_cast<size_t>(r) * (wh >> J) * swc : nullptr;
    int local = 0;
    for (size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < nbytes;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int y = y0 + static_cast<int>(e / rowb);
        const int xb = x0 + static_cast<int>(e % rowb) * CPB;
        unsigned v = 0;
#pragma unroll
        for (int c = 0; c < CPB; ++c) {
            const int x = xb + c;
            if (x >= x1) break;
            unsigned cell;
            if (g) {
                cell = g[static_cast<size_t>(y) * ww + x];
            } else {
                const int b = sm[static_cast<size_t>(y >> J) * swc + (x >> J)];
                const int by = b / wc, bx = b - by * wc;
                cell = ti[static_cast<size_t>((by << J) + (y & (B - 1))) * ti_w + (bx << J) + (x & (B - 1))];
            }
            if (hd) {
                const uint8_t h = hd[static_cast<size_t>(y) * ww + x];
                if (h != kNoDatum) {
                    local += cell != h;
                    cell = h;
                }
            }
            v |= cell << (c * BITS);
        }
        o[e] = static_cast<uint8_t>(v);
    }
    if (hd) {
        for (int q = 16; q > 0; q >>= 1) local += __shfl_xor_sync(0xffffffffu, local, q);
        if ((threadIdx.x & 31) == 0 && local) atomicAdd(&mism[r], local);
    }
    tl_mark(tl, 1);
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

// Raster-path variant (origin * 2 + column-major) of a realization: its
// mt19937_64's first two outputs through bounded(4) and bounded(2)
// (simulator.hpp:148-152).  Powers of two are never rejected by bounded()
// (threshold (2^64 - n) mod n = 0), and outputs 0 and 1 read only state words
// 0-2 and 156-157 of the seeded state, so the seeding recurrence stops at 157.
int path_variant_of_seed(uint64_t seed) {
    uint64_t x[158];
    x[0] = seed;
    for (int i = 1; i < 158; ++i) x[i] = 6364136223846793005ULL * (x[i - 1] ^ (x[i - 1] >> 62)) + i;
    auto out = [&](int k) {
        const uint64_t y = (x[k] & 0xFFFFFFFF80000000ULL) | (x[k + 1] & 0x7FFFFFFFULL);
        uint64_t v = x[k + 156] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ULL : 0);
        v ^= (v >> 29) & 0x5555555555555555ULL;
        v ^= (v << 17) & 0x71D67FFFEDA60000ULL;
        v ^= (v << 37) & 0xFFF7EEE000000000ULL;
        v ^= v >> 43;
        return v;
    };
    const int origin = static_cast<int>(out(0) % 4);
    const int cm = static_cast<int>(out(1) % 2);
    return origin * 2 + cm;
}

// A packed band (pack_band_kernel's layout: rows of rowb bytes, CPB cells per
// byte) -> rows x wdt cells at d with pitch ld.  BMI2 deposits 8 cells per
// instruction (whole rows are written with non-temporal stores); without
// BMI2 a byte -> cells table.
template <int CPB>
__attribute__((target("bmi2"))) void unpack_band_pdep(uint8_t* d, size_t ld, const uint8_t* sp, size_t rowb,
                                                      size_t rows, size_t wdt, const uint64_t* lut) {
    constexpr int kBits = 8 / CPB;  // bits per cell = input bytes per 8 cells
    constexpr uint64_t kMask = kBits == 1 ? 0x0101010101010101ULL : kBits == 2 ? 0x0303030303030303ULL
                                                                               : 0x0F0F0F0F0F0F0F0FULL;
    for (size_t y = 0; y < rows; ++y, d += ld, sp += rowb) {
        const uint8_t* s = sp;
        size_t x = 0;
        // Whole 64-byte lines of the destination are written around the caches
        // (no read-for-ownership); the partial lines at either end of a
        // column-band row take cached stores (non-temporal stores to partial
        // lines are ~10x slower than cached ones).  8 cells per input word.
#define CCW_PUT8(NT)                                                                             \
    do {                                                                                         \
        uint32_t in = 0;                                                                         \
        std::memcpy(&in, s, kBits);                                                              \
        const uint64_t cells = _pdep_u64(in, kMask);                                             \
        if (NT)                                                                                  \
            _mm_stream_si64(reinterpret_cast<long long*>(d + x), static_cast<long long>(cells)); \
        else                                                                                     \
            std::memcpy(d + x, &cells, 8);                                                       \
        x += 8;                                                                                  \
        s += kBits;                                                                              \
    } while (0)
        const size_t head = (64 - (reinterpret_cast<uintptr_t>(d) & 63)) & 63;  // bytes to the first line
        if ((head & 7) == 0) {
            while (x < head && x + 8 <= wdt) CCW_PUT8(false);
            const size_t body = x + (wdt - x) / 64 * 64;
            while (x < body) CCW_PUT8(true);
        }
        while (x + 8 <= wdt) CCW_PUT8(false);
#undef CCW_PUT8
        for (; x < wdt; ++x) {  // the row's last partial group of 8
            const size_t c = x & 7;
            d[x] = static_cast<uint8_t>((s[c / CPB] >> ((c % CPB) * kBits)) & ((1u << kBits) - 1));
        }
    }
    _mm_sfence();
}

template <int CPB>
void unpack_band(uint8_t* d, size_t ld, const uint8_t* sp, size_t rowb, size_t rows, size_t wdt,
                 const uint64_t* lut) {
    static const bool bmi2 = __builtin_cpu_supports("bmi2");
    if (bmi2) return unpack_band_pdep<CPB>(d, ld, sp, rowb, rows, wdt, lut);
    for (size_t y = 0; y < rows; ++y, d += ld, sp += rowb) {
        const uint8_t* s = sp;
        for (size_t x = 0; x < wdt; x += CPB, ++s) {
            const uint64_t cells = lut[*s];
            std::memcpy(d + x, &cells, std::min<size_t>(CPB, wdt - x));
        }
    }
}

// Mask tables of the fast select (MT_STRIDE int4 per mask variant): the mask
// rows of the placement and its rescoring run groups -- up to FS_G cells of
// consecutive rows of one channel with the same column run (a run longer than
// FS_G is a group of its own, summed sequentially), as int4 (channel, first
// row-table index | first row << 16, rows | row-end cell mask << 8, t0 << 8 |
// run length).
void build_mask_tables(int Tc, int OVc, int nch, std::vector<int4>& tab) {
    tab.assign(static_cast<size_t>(8) * MT_STRIDE, make_int4(0, 0, 0, 0));
    const int shapes[8][3] = {{kL, 0, 0}, {kL, 0, 1}, {kL, 1, 0}, {kL, 1, 1},
                              {kVertical, 0, 0}, {kVertical, 1, 0}, {kHorizontal, 0, 0}, {kHorizontal, 0, 1}};
    for (const auto& sh : shapes) {
        const int v = mask_variant(sh[0], sh[1], sh[2]);
        int4* mt = tab.data() + static_cast<size_t>(v) * MT_STRIDE;
        short4* rows = reinterpret_cast<short4*>(mt + 1);
        int4* grp = mt + 1 + MT_ROWS4;
        int nr = 0, lng = 0;
        for (int s = 0; s < Tc; ++s) {
            int t0, t1;
            mask_row_run(sh[0], sh[1], sh[2], Tc, OVc, s, t0, t1);
            if (t1 > t0) {
                rows[nr++] = make_short4(static_cast<short>(s), static_cast<short>(t0), static_cast<short>(t1), 0);
                lng |= t1 - t0 > FS_G;
            }
        }
        int ng = 0;
        for (int ch = 0; ch < nch; ++ch) {
            int k = 0;
            while (k < nr) {
                const int t0 = rows[k].y, len = rows[k].z - rows[k].y;
                int nk = 1;
                while (k + nk < nr && rows[k + nk].x == rows[k].x + nk && rows[k + nk].y == t0 &&
                       rows[k + nk].z - t0 == len && (nk + 1) * len <= FS_G)
                    ++nk;
                if (len > FS_G) nk = 1;
                int endm = 0;  // cells that end a row (nk * len <= FS_G)
                if (len <= FS_G)
                    for (int q = 0; q < nk; ++q) endm |= 1 << (q * len + len - 1);
                if (ng < FS_MAXG) grp[ng++] = make_int4(ch, k | (rows[k].x << 16), nk | (endm << 8), (t0 << 8) | len);
                k += nk;
            }
        }
        mt[0] = make_int4(nr, ng, lng, 0);
    }
}

}  // namespace

// n cells packed `bits` per cell (1, 2 or 4; 8 / bits cells per byte, first
// cell in the low bits) -> one byte per cell at d (the 3D result path).
void unpack_cells(uint8_t* d, const uint8_t* s, size_t n, int bits) {
    static uint64_t lut[3][256];
    static std::once_flag once;
    std::call_once(once, [] {
        for (int k = 0; k < 3; ++k) {
            const int b = 1 << k, cpb = 8 / b;
            for (int v = 0; v < 256; ++v) {
                uint64_t o = 0;
                for (int c = 0; c < cpb; ++c) o |= static_cast<uint64_t>((v >> (c * b)) & ((1 << b) - 1)) << (8 * c);
                lut[k][v] = o;
            }
        }
    });
    if (bits == 1) unpack_band<8>(d, 0, s, 0, 1, n, lut[0]);
    else if (bits == 2) unpack_band<4>(d, 0, s, 0, 1, n, lut[1]);
    else unpack_band<2>(d, 0, s, 0, 1, n, lut[2]);
}

namespace {
}  // namespace

// The per-context plan memory (sim.cu run_simulation): after a call, whether
// its TI/shape deferred tie groups (bulk kernel on/off) or stormed (keep the
// select + bulk kernels instead of the wave kernel).
static void learn_plan(ccw_ctx* ctx, const std::tuple<uint64_t, int, int, int, int>& key, bool use_wave,
                       bool bulk_launch, const unsigned long long* stats) {
    if (use_wave) {
        if (stats[1] > 0 && stats[2] * 50 > stats[1]) ctx->tie_storm[key] = true;
    } else if (bulk_launch && stats[1] > 0 && stats[3] * 50 > stats[1])  // > 2 % of the screened placements
        ctx->tie_storm[key] = true;
    else
        ctx->tie_storm.erase(key);
    if (bulk_launch && stats[3] == 0)
        ctx->bulk_off[key] = true;
    else if (!bulk_launch && stats[2] > 0)  // a list overflowed: bring the bulk kernel back
        ctx->bulk_off.erase(key);
}

// Fold finished asynchronous calls into the context: timing, plan memory and
// device-side errors (oldest first; block = wait for them).
void async_settle(ccw_ctx* ctx, bool block) {
    for (int k = 0; k < 2; ++k) {
        ccw_ctx::AsyncSlot& sl = ctx->aslot[k == 0 ? ctx->async_par : 1 - ctx->async_par];
        if (!sl.valid) continue;
        if (block) {
            CCW_CUDA(cudaEventSynchronize(sl.done));
        } else if (cudaEventQuery(sl.done) != cudaSuccess) {
            cudaGetLastError();
            break;  // (the newer slot cannot be done before the older one)
        }
        const unsigned long long* st = static_cast<const unsigned long long*>(sl.res.p);
        ccw_timing t = sl.timing;
        float ms = 0;
        cudaEventElapsedTime(&ms, sl.t0, sl.t1);
        t.total_ms = ms;
        t.rescored = static_cast<int64_t>(st[0]);
        t.screened_jobs = static_cast<int64_t>(st[1]);
        t.list_overflows = static_cast<int64_t>(st[2]);
        t.bulk_jobs = static_cast<int64_t>(st[3]);
        t.shared_groups = static_cast<int64_t>(st[32]);
        ctx->timing = t;
        learn_plan(ctx, sl.key, sl.use_wave, sl.bulk_launch, st);
        if (st[kNumStats] != 0 && ctx->async_err.empty())
            ctx->async_err = "internal: device schedule disagrees with the host path draws";
        sl.valid = false;
    }
}

void run_simulation(ccw_ctx* ctx, ccw_ti* ti, const ccw_sim_config& cfg, const uint64_t* seeds,
                    int n_real, const int32_t* hd, int n_hd, uint8_t* d_out, uint8_t* h_out,
                    ccw_diag* diag, ccw_trace* traces, bool async_call) {
    const auto wall0 = std::chrono::steady_clock::now();
    // earlier asynchronous calls: a synchronous call settles them all; an
    // asynchronous one settles what has finished (its own slot was used two
    // calls ago and is normally done)
    async_settle(ctx, !async_call);
    if (async_call && ctx->aslot[ctx->async_par].valid) {
        CCW_CUDA(cudaEventSynchronize(ctx->aslot[ctx->async_par].done));
        async_settle(ctx, false);
    }
    const int apar = ctx->async_par;
    cudaStream_t st = ctx->stream;
    const int T = cfg.template_size, OV = cfg.overlap, J = cfg.dwt_level, B = 1 << J;
    const int stride = T - OV;
    // literal-config extension (any_support): the coarse mask keeps every block
    // the fine overlap touches, ceil(OV / B) coarse cells deep
    const int Tc = T >> J, OVc = cfg.any_support ? (OV + B - 1) >> J : OV >> J;
    // pastes land on whole TI blocks but, with an overlap 2^J does not
    // divide, not on whole work-grid blocks: the work grid then holds the
    // realization (as with min-cut) instead of the source-block map
    const bool grid_mode = cfg.min_cut || (cfg.any_support && (T - OV) % B != 0);
    const int out_h = ti->hc - Tc + 1, out_w = ti->wc - Tc + 1;
    const int npos = out_h * out_w;
    const int Kp = std::min(cfg.candidates, npos);
    if (Kp > KMAX)
        throw Fail(CCW_ERR_CONFIG, "candidates: more than 8192 effective candidates unsupported");
    const int reach = (T + stride - 1) / stride - 1;  // footprints overlap up to `reach` steps
    const int keymul = reach + 1;

    // ---- host schedule: raster paths, hard-data lattice, wave layout.  A
    // raster path (simulator.hpp:148-190) is one of 8 variants (origin x major
    // order) drawn first by each realization's mt19937_64; the per-placement
    // draws and the jobs themselves are made on the device (schedule.cu) in
    // (group, wave, realization, placement) order.
    std::vector<Plan> variants(8);
    std::vector<char> have(8, 0);
    std::vector<int32_t> vid(n_real);
    for (int r = 0; r < n_real; ++r) vid[r] = path_variant_of_seed(seeds[r]);
    const double t_seed = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();
    for (int r = 0; r < n_real; ++r)
        if (!have[vid[r]]) {
            variants[vid[r]] = make_plan_from(cfg, vid[r] / 2, (vid[r] & 1) != 0);
            have[vid[r]] = 1;
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
    // conditional choice reads only the cells that hold data -- built on the
    // device (hd_count / hd_scan / hd_fill kernels below)
    const bool have_hd = hd && n_hd > 0;
    int max_key = 0;
    for (int v = 0; v < 8; ++v)
        if (have[v]) max_key = std::max(max_key, keymul * (variants[v].n_outer - 1) + variants[v].n_inner - 1);
    const int nkeys = max_key + 1;
    // per-variant wave histograms
    std::vector<std::vector<int>> vhist(8), vhistL(8);  // placements (L-shaped ones) per wave
    for (int v = 0; v < 8; ++v)
        if (have[v]) {
            vhist[v].assign(nkeys, 0);
            const Plan& p = variants[v];
            vhistL[v].assign(nkeys, 0);
            for (size_t k = 0; k < p.tops.size(); ++k) {
                ++vhist[v][keymul * p.outer_idx[k] + p.inner_idx[k]];
                if (p.shapes[k] == kL) ++vhistL[v][keymul * p.outer_idx[k] + p.inner_idx[k]];
            }
        }

    // Realizations are split into G independent groups, each on its own
    // stream, so one group's latency-bound select overlaps another group's
    // tensor-core screen.  Within a group, waves run in order.
    // candidate-position sharding (ccw_ctx_set_position_shards): S shards of the
    // window positions, S_virt of them in this rank; one group (the per-wave
    // exchange is one collective on one stream)
    const int S_virt = ctx->shard_virtual, S_ranks = ctx->shard_nranks;
    const int S_all = S_virt * S_ranks;
    const bool sharded = S_all > 1 || ctx->nccl_comm != nullptr;
    if (sharded && npos < S_all)
        throw Fail(CCW_ERR_CONFIG, "position shards: more shards than TI window positions");
    int G = std::max(1, std::min(n_real, 2));
    if (ctx->opt.groups > 0) G = std::max(1, std::min(n_real, ctx->opt.groups));
    if (sharded) G = 1;
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
    // each realization's first slot in every wave bucket (uploaded for the device schedule)
    // (pinned staging halves alternate by call: the previous call's upload from
    // the other half may still be queued behind its predecessor)
    ccwgpu::HostBuf& hstage = apar == 0 ? ctx->h_stage : ctx->h_stage2;
    if (ctx->stage_ev[apar]) CCW_CUDA(cudaEventSynchronize(ctx->stage_ev[apar]));
    int32_t* roff = static_cast<int32_t*>(hstage.get(sizeof(int32_t) * (static_cast<size_t>(n_real) * nkeys + n_real)));
    int32_t* vid_stage = roff + static_cast<size_t>(n_real) * nkeys;
    std::copy(vid.begin(), vid.end(), vid_stage);
    {
        std::vector<size_t> fill(bucket.begin(), bucket.end() - 1);
        for (int r = 0; r < n_real; ++r) {
            const size_t g = group_of(r);
            for (int k = 0; k < nkeys; ++k) {
                roff[static_cast<size_t>(r) * nkeys + k] = static_cast<int32_t>(fill[g * nkeys + k]);
                fill[g * nkeys + k] += vhist[vid[r]][k];
            }
        }
    }
    const double t_sched = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();
    const double host_prep_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();

    // ---- exactness guard for the fp32 screen
    const double maxw = ti->mode == 0 ? B : static_cast<double>(ti->F - 1) * B;
    const double mask_cells = static_cast<double>(Tc) * OVc + static_cast<double>(Tc - OVc) * OVc;
    bool use_screen = cfg.scoring == 0 && ti->nscr > 0;
    // normalized scoring: screened on the int8 tensor-core GEMM when it applies
    // (otherwise every window is rescored in fp64)
    bool norm_screen = cfg.scoring == 1 && ti->nscr > 0 && ctx->opt.norm_screen &&
                       mask_cells * ti->nch * maxw * maxw * maxw * maxw < 2147483647.0;

    // ---- device buffers
    EventTimer tm{ctx, {}, {}, 0};
    cudaEvent_t ev_sched = tm.get();
    CCW_CUDA(cudaEventRecord(ev_sched, st));
    int32_t* d_hdl = nullptr;
    uint8_t* d_lat = nullptr;
    const int32_t* P_hd_off = nullptr;
    const uint32_t* P_hd_ent = nullptr;
    if (have_hd) {
        const size_t ncell = static_cast<size_t>(nlr) * nlc;
        const int cover = (T + stride - 1) / stride;  // lattice positions per axis covering one cell
        d_hdl = reinterpret_cast<int32_t*>(ctx->ops_e.get(sizeof(int32_t) * 3 * n_hd));
        CCW_CUDA(cudaMemcpyAsync(d_hdl, hd, sizeof(int32_t) * 3 * n_hd, cudaMemcpyHostToDevice, st));
        int32_t* d_off = ctx->hdoff.as<int32_t>(2 * (ncell + 1));  // offsets, then the fill cursors
        uint32_t* d_ent = ctx->hdent.as<uint32_t>(std::max<size_t>(1, static_cast<size_t>(n_hd) * cover * cover));
        d_lat = ctx->lattice.as<uint8_t>(ncell);
        CCW_CUDA(cudaMemsetAsync(d_off, 0, sizeof(int32_t) * 2 * (ncell + 1), st));
        const unsigned nb = static_cast<unsigned>((n_hd + 255) / 256);
        hd_count_kernel<<<nb, 256, 0, st>>>(d_hdl, n_hd, T, stride, nlr, nlc, d_off + 1);
        hd_scan_kernel<<<1, 1024, 0, st>>>(d_off, static_cast<int>(ncell), d_off + ncell + 1, d_lat);
        hd_fill_kernel<<<nb, 256, 0, st>>>(d_hdl, n_hd, T, stride, nlr, nlc, d_off + ncell + 1, d_ent);
        CCW_CUDA(cudaGetLastError());
        P_hd_off = d_off;
        P_hd_ent = d_ent;
    }
    Job* d_jobs = ctx->jobs.as<Job>(total_jobs);
    {
        const size_t nstage = static_cast<size_t>(n_real) * nkeys + n_real;
        int32_t* d_roff = ctx->roff.as<int32_t>(nstage);
        CCW_CUDA(cudaMemcpyAsync(d_roff, roff, sizeof(int32_t) * nstage, cudaMemcpyHostToDevice, st));
        if (!ctx->stage_ev[apar]) CCW_CUDA(cudaEventCreateWithFlags(&ctx->stage_ev[apar], cudaEventDisableTiming));
        CCW_CUDA(cudaEventRecord(ctx->stage_ev[apar], st));
        int* d_err = ctx->sched_err.as<int>(1);
        CCW_CUDA(cudaMemsetAsync(d_err, 0, sizeof(int), st));
        SchedParams SP{};
        SP.seeds = static_cast<const uint64_t*>(ctx->seeds.get(sizeof(uint64_t) * n_real));
        CCW_CUDA(cudaMemcpyAsync(const_cast<uint64_t*>(SP.seeds), seeds, sizeof(uint64_t) * n_real,
                                 cudaMemcpyHostToDevice, st));
        SP.vid = d_roff + static_cast<size_t>(n_real) * nkeys;
        SP.roff = d_roff;
        if (d_lat) SP.lattice_hd = d_lat;
        SP.err = d_err;
        SP.n_real = n_real;
        SP.nkeys = nkeys;
        SP.keymul = keymul;
        SP.nlr = nlr;
        SP.nlc = nlc;
        SP.stride = stride;
        SP.B = B;
        SP.Kp = Kp;
        SP.nfr = static_cast<uint64_t>((ti->hc * B - T) / B + 1);  // (the used TI: whole blocks)
        SP.nfc = static_cast<uint64_t>((ti->wc * B - T) / B + 1);
        SP.thr_fr = (0 - SP.nfr) % SP.nfr;
        SP.thr_fc = (0 - SP.nfc) % SP.nfc;
        SP.thr_k = (0 - static_cast<uint64_t>(Kp)) % static_cast<uint64_t>(Kp);
        if (ctx->opt.sched_replay) SP.thr_k = ~0ull;  // tests: every pick "rejected" -> sequential replay
        SP.nout = 4 + nlr * nlc;  // the path, the first placement's two, one per other placement
        SP.outs = ctx->sched_outs.as<uint64_t>(static_cast<size_t>(n_real) * SP.nout);
        SP.replay = ctx->sched_replay.as<uint64_t>(static_cast<size_t>(n_real) * 313);
        build_jobs_kernel<<<n_real, 32, 0, st>>>(SP, d_jobs);
        CCW_CUDA(cudaGetLastError());
    }
    const size_t plane = static_cast<size_t>(wh) * ww;
    // the work grid exists only with min-cut (seams read the grid); otherwise
    // the source-block map is the realization until finalize
    uint8_t* d_work = nullptr;
    if (grid_mode) {
        d_work = ctx->work.as<uint8_t>(plane * n_real);
        CCW_CUDA(cudaMemsetAsync(d_work, 0, plane * n_real, st));
    }
    uint8_t* d_hd = nullptr;
    if (have_hd) {
        d_hd = ctx->hd.as<uint8_t>(plane);
        CCW_CUDA(cudaMemsetAsync(d_hd, kNoDatum, plane, st));
        hd_scatter_kernel<<<(n_hd + 255) / 256, 256, 0, st>>>(d_hdl, n_hd, d_hd, ww);
        CCW_CUDA(cudaGetLastError());
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
    P.any_support = cfg.any_support;
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
    // the fp32 CUDA-core screen is exact only while every partial sum stays
    // below 2^24; beyond that every window is scored in fp64 (select mode 0)
    if (use_screen && !use_tc && mask_cells * maxw * maxw * std::max(1, ti->nscr) >= 16777216.0)
        use_screen = false;
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
    unsigned long long* d_stats = ctx->stats.as<unsigned long long>(kNumStats);
    CCW_CUDA(cudaMemsetAsync(d_stats, 0, kNumStats * sizeof(unsigned long long), st));
    // source-block map (fast or_prep), valid whenever pastes are verbatim TI blocks
    const int swc = ww / B;
    int32_t* d_src = nullptr;
    if (!grid_mode) {
        d_src = ctx->src.as<int32_t>(static_cast<size_t>(n_real) * (wh / B) * swc);
    }
    P.src = d_src;
    P.swc = swc;
    const bool fast_ok = use_tc && Kp <= kTcQ && !cfg.min_cut && cfg.scoring == 0 &&
                         ti->nch * Tc <= FS_MAXG && Tc <= PK_MAXTC;
    // position shards take the fast select when every shard (boundaries at
    // multiples of one 256-position MMA tile) holds at least K tile maxima of
    // its own; the other shards' tiles read INT_MIN and are never candidates
    const bool shard_fast = sharded && fast_ok && ctx->opt.shard_fast &&
                            npos / S_all >= 256 + 128 * Kp;
    const bool warp_select = !sharded && fast_ok;
    if (warp_select || shard_fast) {
        const long long key = Tc | (static_cast<long long>(OVc) << 16) | (static_cast<long long>(ti->nch) << 32);
        int4* d_mt = ctx->mtab.as<int4>(static_cast<size_t>(8) * MT_STRIDE);
        if (ctx->mtab_key != key) {
            std::vector<int4> tab;
            build_mask_tables(Tc, OVc, ti->nch, tab);
            CCW_CUDA(cudaMemcpyAsync(d_mt, tab.data(), tab.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
            CCW_CUDA(cudaStreamSynchronize(st));  // tab is freed on return
            ctx->mtab_key = key;
        }
        P.mtab = d_mt;
        if (ctx->opt.uniform) {
            P.umap = ti_umap(ti, Tc, OVc, st);
            P.ustride = umap_stride(npos);
            P.pure_apex = ti_pure_apex(ti, Tc, OVc, st);
            P.ufirst = ti_uniform_first(ti, Tc, OVc, st);
        }
    }
    // int16 score rows for the fast select when every screen score fits:
    // |S'| <= mask cells * (largest weight) * (largest block statistic)
    const bool s16 = warp_select && mask_cells * static_cast<double>(maxv) * maxv < 32767.0 &&
                     ctx->opt.s16;
    P.s16 = s16 ? 1 : 0;
    P.kpad = kpad;
    P.ntiles = ntiles;
    P.stats = d_stats;
    P.im2col = d_x;
    // bulk tie select: largest window block whose apex tile fits the shared-memory budget
    size_t bulk_smem = 0;
    if ((warp_select || shard_fast) && ctx->opt.bulk) {
        // (measured r2, config 2: blocks of up to 64 x 256 windows beat 32 x 64
        // ones, 19.0 vs 25.0 ms -- every block costs a tile-max round trip)
        constexpr size_t kBudget = 200 * 1024;
#ifndef CCW_BK_BY
#define CCW_BK_BY 256
#define CCW_BK_BX 64
#endif
        for (int by = std::min(out_w, CCW_BK_BY); by >= 8 && !bulk_smem; by /= 2) {
            int bx = std::min(out_h, CCW_BK_BX);
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
    // thresholds [G][maxj], deferred-slot lists [G][maxj], list counters [G][2]
    int* d_defer = bulk_launch ? ctx->defer.as<int>(2 * G * maxj + 2 * G) : nullptr;
    int* d_dcnt = d_defer ? d_defer + 2 * G * maxj : nullptr;
    if (d_dcnt) CCW_CUDA(cudaMemsetAsync(d_dcnt, 0, sizeof(int) * 2 * G, st));
    std::vector<int> dpar(G, 0);  // per group: which list counter the next select / bulk pair uses
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
    // tie-storm placements: the screen also keeps per-tile maxima over the
    // non-uniform windows, so the bulk kernel reads only the tiles that can
    // hold a non-uniform candidate (the uniform classes are class constants)
    int32_t* d_tmaxnu = nullptr;
    int8_t* d_jvar = nullptr;
    const uint32_t* d_ubits = nullptr;
    if (bulk_launch && warp_select && P.umap && P.ufirst && use_tc && ctx->tie_storm.count(bulk_key)) {
        d_ubits = ti_uniform_bits(ti, Tc, OVc, st);
        d_tmaxnu = ctx->tmaxnu.as<int32_t>(G * maxj * ntiles);
        d_jvar = ctx->jvar.as<int8_t>(G * maxj);
    }
    // fused wave kernel (wave.cu): one launch per wave for the source-block-map
    // path with the int8 screen; TIs whose last call was a tie storm keep the
    // select + bulk kernels (the wave kernel's fallback is exact but slow)
    const bool use_wave = !sharded && use_tc && use_screen && d_src && !cfg.min_cut && cfg.scoring == 0 &&
                          ctx->opt.wave && wave_supported(ti->nscr, Tc, ti->nch, Kp, T, OV) &&
                          !ctx->tie_storm.count(bulk_key);
    const int8_t* d_strips = nullptr;
    int wave_nmb = 1, wave_nb = 16;
    int8_t* d_wave_w = nullptr;
    size_t wave_w_per_group = 0;
    if (use_wave) {
        d_strips = ti_strips(ti, Tc, st, &wave_nmb, &wave_nb);
        wave_w_per_group = wave_wglob_bytes(P, static_cast<int>(maxj));
        d_wave_w = ctx->wave_w.as<int8_t>(G * wave_w_per_group);
        wave_prepare(P);
    }
    if (bulk_smem)
        CCW_CUDA(cudaFuncSetAttribute(select_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(bulk_smem)));
    // dependency flags between a wave's select and the next wave's OR prep
    // (option flagprep; or_prep_src_kernel): needs every paste in the select
    // (no bulk deferrals), the raster neighbours of keymul 2 and the map path
    const bool flag_prep = ctx->opt.flagprep && warp_select && keymul == 2 && d_src && !bulk_launch && !use_wave &&
                           debug_env("CCW_FUSE_PREP") == nullptr;
    if (flag_prep) {
        int* d_depflag = ctx->depflag.as<int>(total_jobs);
        CCW_CUDA(cudaMemsetAsync(d_depflag, 0, sizeof(int) * total_jobs, st));
        P.depflag = d_depflag;
    }
    std::vector<SimParams> GP(G, P);
    for (int g = 0; g < G; ++g) {
        GP[g].scores = d_scores + g * maxj * sld;
        GP[g].wts = d_wts + g * maxj * std::max(ti->nscr, 1) * Tc * Tc;
        GP[g].tm64 = d_tm + g * maxj * ti->nch * Tc * Tc;
        GP[g].wts8 = d_w8 ? d_w8 + g * maxj * kpad : nullptr;
        GP[g].tmax = d_tmax ? d_tmax + g * maxj * ntiles : nullptr;
        GP[g].tmax_nu = d_tmaxnu ? d_tmaxnu + g * maxj * ntiles : nullptr;
        GP[g].jvar = d_jvar ? d_jvar + g * maxj : nullptr;
        GP[g].cjob = d_cjob ? d_cjob + g * maxj : nullptr;
        GP[g].defer = d_defer ? d_defer + g * maxj : nullptr;
        GP[g].defer_list = d_defer ? d_defer + G * maxj + g * maxj : nullptr;
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
                           debug_env("CCW_FUSE_PREP") != nullptr;
    int* d_depcnt = nullptr;
    if (fuse_prep) {
        d_depcnt = ctx->depcnt.as<int>(G * maxj);
        CCW_CUDA(cudaMemsetAsync(d_depcnt, 0, sizeof(int) * G * maxj, st));
    }
    // shared rescoring of large equal-score groups (select_fast_kernel): two
    // boards per group, alternating between its select launches
    HelpBoard* d_boards = nullptr;
    int4* d_hslots = nullptr;
    if (warp_select) {
        const int help_min = ctx->opt.help_min;
        if (help_min > 0) {
            d_boards = ctx->hboards.as<HelpBoard>(2 * G);
            CCW_CUDA(cudaMemsetAsync(d_boards, 0, sizeof(HelpBoard) * 2 * G, st));
            d_hslots = ctx->hdone.as<int4>(2 * G * maxj);
            CCW_CUDA(cudaMemsetAsync(d_hslots, 0, sizeof(int4) * 2 * G * maxj, st));
            int* d_hpos = ctx->hpos.as<int>(G * maxj * SC_LC);
            double* d_hkeys = ctx->hkeys.as<double>(G * maxj * SC_LC);
            for (int g = 0; g < G; ++g) {
                GP[g].hpos = d_hpos + g * maxj * SC_LC;
                GP[g].hkeys = d_hkeys + g * maxj * SC_LC;
                GP[g].hs_n = static_cast<int>(maxj);
                GP[g].help_min = help_min;
            }
        }
    }
    std::vector<int> hb_par(G, 0);
    const char* jdump_path = debug_env("CCW_TAIL_DUMP");
    unsigned long long* d_jdump = nullptr;
    if (jdump_path) {
        d_jdump = ctx->jdump.as<unsigned long long>(8 * total_jobs);
        CCW_CUDA(cudaMemsetAsync(d_jdump, 0, sizeof(unsigned long long) * 8 * total_jobs, st));
        for (int g = 0; g < G; ++g) GP[g].jdump = d_jdump;
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
    if (debug_env("CCW_TC_PROBE")) {
        d_probe = reinterpret_cast<unsigned long long*>(ctx->ops_d.get(8 * sizeof(unsigned long long)));
        CCW_CUDA(cudaMemsetAsync(d_probe, 0, 8 * sizeof(unsigned long long), st));
    }
    tc_probe_buffer = d_probe;
    std::vector<std::array<TcPlan, 2>> tcplans(G);
    if (use_tc)
        for (int g = 0; g < G; ++g)
            for (int par = 0; par < 2; ++par)
                tcplans[g][par] = plan_ccf_tc(GPP[g][par].wts8, static_cast<int>(maxj), d_x, npos, kpad);
    // position shards of this rank: window ranges, shard-local score rows and
    // tile maxima, TMA plans over the im2col row slice, the exchange buffer
    struct ShardPart {
        int s, p0, n, sld, ntiles;
        int32_t *scores, *tmax;
        TcPlan plan;
    };
    std::vector<ShardPart> parts;
    ShardRec* d_xrec = nullptr;
    if (sharded) {
        size_t sc_tot = 0, tm_tot = 0;
        auto cut = [&](int s) {  // shard boundary (256-aligned for the fast select)
            const int64_t p = static_cast<int64_t>(npos) * s / S_all;
            return static_cast<int>(shard_fast && s < S_all ? p / 256 * 256 : p);
        };
        for (int v = 0; v < S_virt; ++v) {
            ShardPart sp{};
            sp.s = ctx->shard_rank * S_virt + v;
            sp.p0 = cut(sp.s);
            sp.n = cut(sp.s + 1) - sp.p0;
            // fast select: full-length rows in global positions, INT_MIN outside the shard
            sp.sld = shard_fast ? sld : (sp.n + 3) & ~3;
            sp.ntiles = shard_fast ? ntiles : tc_tiles(sp.n);
            sc_tot += maxj * sp.sld;
            tm_tot += maxj * sp.ntiles;
            parts.push_back(sp);
        }
        int32_t* sc = ctx->scores.as<int32_t>(sc_tot);
        int32_t* tmx = use_tc ? ctx->summary.as<int32_t>(tm_tot) : nullptr;
        if (shard_fast) {
            fill_i32(sc, sc_tot, INT_MIN, st);
            fill_i32(tmx, tm_tot, INT_MIN, st);
        }
        for (ShardPart& sp : parts) {
            sp.scores = sc;
            sc += maxj * sp.sld;
            if (tmx) {
                sp.tmax = tmx;
                tmx += maxj * sp.ntiles;
                sp.plan = plan_ccf_tc(GPP[0][0].wts8, static_cast<int>(maxj), d_x + static_cast<size_t>(sp.p0) * kpad,
                                      sp.n, kpad);
            }
        }
        d_xrec = ctx->xrec.as<ShardRec>(static_cast<size_t>(S_all) * maxj * Kp);
        CCW_CUDA(cudaFuncSetAttribute(shard_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(sel_smem)));
    }
    // group streams, forked from / joined back to the context stream
    // (stream priorities measured r1, config 1 end to end: waves first 22.6 G
    // cells/s -- starving the band finalize kernels delays the host's
    // unpacking; copies first within noise of none; so none)
    int least = 0, greatest = 0;
    CCW_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    const int wave_prio = least, copy_prio = least;
    while (static_cast<int>(ctx->copy_streams.size()) < G) {  // one per group: final copies overlap
        cudaStream_t s3;
        CCW_CUDA(cudaStreamCreateWithPriority(&s3, cudaStreamNonBlocking, copy_prio));
        ctx->copy_streams.push_back(s3);
    }
    while (static_cast<int>(ctx->gstreams.size()) < G) {
        cudaStream_t s2;
        CCW_CUDA(cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, wave_prio));
        ctx->gstreams.push_back(s2);
    }
    cudaEvent_t ev0 = tm.get(), ev1 = tm.get();
    CCW_CUDA(cudaEventRecord(ev0, st));
    if (async_call) {  // (this call's span on events the next call does not reuse)
        ccw_ctx::AsyncSlot& sl = ctx->aslot[apar];
        for (cudaEvent_t* e : {&sl.done, &sl.t0, &sl.t1})
            if (!*e) CCW_CUDA(cudaEventCreate(e));
        CCW_CUDA(cudaEventRecord(sl.t0, st));
    }
    for (int g = 0; g < G; ++g) CCW_CUDA(cudaStreamWaitEvent(ctx->gstreams[g], ev0, 0));
    const bool host_t = debug_env("CCW_HOSTT") != nullptr;
    auto host_ms = [&]() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count(); };
    const double t_ev0 = host_t ? host_ms() : 0.0;
    // finalize granularity: one thread per coarse block (B = 2, 4, 8) with the map
    const int fin_bt = d_src && (B == 2 || B == 4 || B == 8) ? B : 0;
    const size_t fin_cells = fin_bt ? static_cast<size_t>(B) * B : 1;
    // ---- progressive output (host results): bands of every realization that
    // no remaining placement covers are finalized and copied back at a few
    // checkpoint waves, overlapping the copy with the remaining waves
    uint8_t* fin = d_out ? d_out : ctx->out.as<uint8_t>(static_cast<size_t>(cfg.sg_height) * cfg.sg_width * n_real);
    const size_t out_bytes = static_cast<size_t>(cfg.sg_height) * cfg.sg_width * n_real;
    const bool stream_out = h_out && !d_out && ctx->opt.stream_out;
    // device->host copies need page-locked memory to run asynchronously: a
    // pageable destination without streaming gets a pinned staging buffer,
    // copied out at the end
    uint8_t* h_dst = h_out;
    if (h_out && !stream_out) {
        cudaPointerAttributes pa{};
        const bool pinned = cudaPointerGetAttributes(&pa, h_out) == cudaSuccess && pa.type == cudaMemoryTypeHost;
        cudaGetLastError();
        if (!pinned) h_dst = static_cast<uint8_t*>(ctx->h_out_stage.get(out_bytes));
    }
    // Streaming: at each checkpoint wave, every band no remaining placement
    // covers (rows of a row-major path, columns of a column-major one) is
    // finalized while later waves compute.  Row bands into a page-locked
    // caller buffer are contiguous there: finalized in place and copied
    // directly.  Column bands (and every band of a pageable buffer) are
    // finalized packed -- pack_bits per cell -- into a device staging area;
    // a checkpoint's packed bands leave in one contiguous copy into pinned
    // host staging and host threads unpack them into the caller's buffer.
    // Checkpoints thicken towards the end, where the last rows / columns
    // (direct row bands measured slower, r1: one copy per realization band
    // lengthens the launch loop, and 8-bit rows quadruple the PCIe bytes)
    const bool direct_rows = debug_env("CCW_DIRECT_ROWS") != nullptr;
    // CTAs per band of a finalize launch: few while waves still run (the
    // bands are not urgent and the waves need the SMs), many for the last
    // checkpoint, which the call waits for (measured r2, config 1 e2e:
    // 16 -> 3.18 ms vs 1024 -> 3.31 ms per call)
#ifndef CCW_BAND_LAST
#define CCW_BAND_LAST 1024
#endif
    const size_t band_cap_mid = 16, band_cap_last = CCW_BAND_LAST;
    bool h_pinned = false;
    if (stream_out) {
        cudaPointerAttributes pa{};
        h_pinned = cudaPointerGetAttributes(&pa, h_out) == cudaSuccess && pa.type == cudaMemoryTypeHost;
        cudaGetLastError();
    }
    struct Checkpoint {
        int w;
        size_t b0, bm, b1;  // bands [b0, bm) direct, [bm, b1) packed
    };
    std::vector<int4> bands;                                   // all checkpoints, in launch order
    std::vector<long long> band_off;                           // packed bands: offset in the staging
    std::vector<std::vector<Checkpoint>> band_at(G);           // per group, in wave order
    uint8_t* h_stage = nullptr;
    uint8_t* d_stage = nullptr;
    // cells per streamed byte: the realizations' codes fit in 1, 2 or 4 bits for F <= 2, 4, 16
    const int pack_bits = !ctx->opt.pack ? 8 : ti->F <= 2 ? 1 : ti->F <= 4 ? 2 : ti->F <= 16 ? 4 : 8;
    const int pack_cpb = 8 / pack_bits;
    auto band_rowb = [&](const int4& bd) {  // packed bytes per band row
        const int wdt = bd.y == 0 ? cfg.sg_width : bd.w - bd.z;
        return static_cast<size_t>((wdt + pack_cpb - 1) / pack_cpb);
    };
    auto band_rows = [&](const int4& bd) { return static_cast<size_t>(bd.y == 0 ? bd.w - bd.z : cfg.sg_height); };
    if (stream_out) {
        std::vector<int> cks;
        // evenly spaced (measured r1: 6 beats both fewer and more, and beats
        // checkpoints crowded towards the end -- thin column bands cost the
        // host more per byte than the later landing costs)
        const int nck = std::max(1, ctx->opt.stream_bands);
        for (int k = 1; k <= nck; ++k) cks.push_back((max_key * k) / nck);
        // extra checkpoints one raster-outer step apart before the end shrink
        // the bands that can only leave after the last wave
        int ntail = 0;
        if (const char* e = debug_env("CCW_STREAM_TAIL")) ntail = std::max(0, atoi(e));
        for (int k = 1; k <= ntail; ++k) cks.push_back(max_key - k * keymul);
        std::vector<int> done(n_real, 0);  // raster-outer extent already emitted
        long long off = 0;
        for (int w = 0; w <= max_key; ++w) {
            if (w != max_key && std::find(cks.begin(), cks.end(), w) == cks.end()) continue;
            for (int g = 0; g < G; ++g) {
                const size_t b0 = bands.size();
                size_t bm = b0;
                for (int pass = 0; pass < 2; ++pass)  // direct bands first, then packed ones
                for (int r = 0; r < n_real; ++r) {
                    if (group_of(r) != g) continue;
                    const Plan& p = variants[vid[r]];
                    const int axis = p.column_major ? 1 : 0;
                    const bool direct = axis == 0 && h_pinned && direct_rows;
                    if (direct != (pass == 0)) continue;
                    const bool asc = axis == 0 ? (p.origin == CCW_TOP_LEFT || p.origin == CCW_TOP_RIGHT)
                                               : (p.origin == CCW_TOP_LEFT || p.origin == CCW_BOTTOM_LEFT);
                    const int extent = axis == 0 ? wh : ww, sg_ext = axis == 0 ? cfg.sg_height : cfg.sg_width;
                    int O = w >= p.n_inner - 1 ? (w - (p.n_inner - 1)) / keymul : -1;
                    O = std::min(O, p.n_outer - 1);
                    const int U = (w == max_key || O == p.n_outer - 1) ? extent : (O + 1) * stride;
                    if (U <= done[r]) continue;
                    int lo = asc ? done[r] : extent - U, hi = asc ? U : extent - done[r];
                    done[r] = std::max(done[r], U);
                    lo = std::max(lo, 0);
                    hi = std::min(hi, sg_ext);
                    if (hi <= lo) continue;
                    bands.push_back(make_int4(r, axis, lo, hi));
                    if (direct) {
                        band_off.push_back(-1);
                        bm = bands.size();
                    } else {
                        band_off.push_back(off);
                        off += static_cast<long long>(band_rows(bands.back()) * band_rowb(bands.back()));
                    }
                }
                if (bands.size() > b0) band_at[g].push_back({w, b0, bm, bands.size()});
            }
        }
    }
    if (stream_out) {
        h_stage = static_cast<uint8_t*>(ctx->h_out_stage.get(out_bytes));
        d_stage = ctx->band_stage.as<uint8_t>(out_bytes);
    }
    int4* d_bands = nullptr;
    long long* d_boff = nullptr;
    if (!bands.empty()) {
        d_bands = reinterpret_cast<int4*>(ctx->ops_b.get(sizeof(int4) * bands.size()));
        CCW_CUDA(cudaMemcpyAsync(d_bands, bands.data(), sizeof(int4) * bands.size(), cudaMemcpyHostToDevice, st));
        d_boff = ctx->band_off.as<long long>(band_off.size());
        CCW_CUDA(cudaMemcpyAsync(d_boff, band_off.data(), sizeof(long long) * band_off.size(),
                                 cudaMemcpyHostToDevice, st));
    }
    std::vector<size_t> band_next(G, 0);
    struct CopyMark {
        int w, g;
        cudaEvent_t ev;
    };
    std::vector<CopyMark> copy_marks;
    struct Arrival {  // one checkpoint's packed bands of one group, landed in h_stage once ev completes
        size_t b0, b1;
        cudaEvent_t ev;
    };
    auto band_bytes = [&](size_t q) { return band_rows(bands[q]) * band_rowb(bands[q]); };
    // every packed checkpoint, in landing (band) order, with its event made
    // up front: a placer thread consumes them while the waves are launched
    std::vector<Arrival> arrivals;
    for (int g = 0; g < G; ++g)
        for (const Checkpoint& ck : band_at[g])
            if (ck.b1 > ck.bm) arrivals.push_back({ck.bm, ck.b1, tm.get()});
    std::sort(arrivals.begin(), arrivals.end(), [](const Arrival& a, const Arrival& b) { return a.b0 < b.b0; });
    std::unique_ptr<std::atomic<int>[]> arr_ready(new std::atomic<int>[arrivals.size() + 1]);
    for (size_t k = 0; k < arrivals.size(); ++k) arr_ready[k].store(0);
    auto arrival_index = [&](size_t b0) {
        return static_cast<size_t>(std::lower_bound(arrivals.begin(), arrivals.end(), b0,
                                                    [](const Arrival& a, size_t v) { return a.b0 < v; }) -
                                   arrivals.begin());
    };
    uint64_t unpack_lut[256];  // byte -> its pack_cpb cells, one per byte (little endian)
    for (int b = 0; b < 256; ++b) {
        uint64_t v = 0;
        for (int c = 0; c < pack_cpb && pack_bits < 8; ++c)
            v |= static_cast<uint64_t>((b >> (c * pack_bits)) & ((1 << pack_bits) - 1)) << (8 * c);
        unpack_lut[b] = v;
    }
    std::vector<size_t> packed_q;  // packed bands in landing order, and their arrivals
    std::vector<int> packed_arrival;
    for (size_t k = 0; k < arrivals.size(); ++k)
        for (size_t q = arrivals[k].b0; q < arrivals[k].b1; ++q) {
            packed_q.push_back(q);
            packed_arrival.push_back(static_cast<int>(k));
        }
    std::atomic<long long> t_wait{0}, t_unpack{0};
    // Placement: host workers take the packed bands in landing order; each
    // waits (polling, so the launching thread keeps its core) until the copy
    // carrying its band has landed, then unpacks it into the caller's buffer.
    auto place_band = [&](int qi) {
        const size_t q = packed_q[static_cast<size_t>(qi)];
        const auto tw0 = std::chrono::steady_clock::now();
        const size_t k = static_cast<size_t>(packed_arrival[static_cast<size_t>(qi)]);
        for (int spin = 0;; ++spin) {  // recorded, then landed: short pause-spins, then naps
            if (arr_ready[k].load(std::memory_order_acquire)) {
                const cudaError_t e = cudaEventQuery(arrivals[k].ev);
                if (e == cudaSuccess) break;
                if (e != cudaErrorNotReady) CCW_CUDA(e);
            }
            if (spin < 64)
                for (int i = 0; i < 64; ++i) _mm_pause();
            else
                std::this_thread::sleep_for(std::chrono::microseconds(10));
        }
        const auto tw1 = std::chrono::steady_clock::now();
        t_wait += std::chrono::duration_cast<std::chrono::nanoseconds>(tw1 - tw0).count();
        const int4 bd = bands[q];
        const uint8_t* srcp = h_stage + band_off[q];
        uint8_t* dst = h_out + static_cast<size_t>(bd.x) * cfg.sg_height * cfg.sg_width;
        const int y0 = bd.y == 0 ? bd.z : 0, x0 = bd.y == 0 ? 0 : bd.z;
        const size_t wdt = static_cast<size_t>(bd.y == 0 ? cfg.sg_width : bd.w - bd.z);
        const size_t rowb = band_rowb(bd), rows = band_rows(bd);
        uint8_t* d = dst + static_cast<size_t>(y0) * cfg.sg_width + x0;
        if (pack_bits == 8)
            for (size_t y = 0; y < rows; ++y) std::memcpy(d + y * cfg.sg_width, srcp + y * rowb, wdt);
        else if (pack_cpb == 8) unpack_band<8>(d, cfg.sg_width, srcp, rowb, rows, wdt, unpack_lut);
        else if (pack_cpb == 4) unpack_band<4>(d, cfg.sg_width, srcp, rowb, rows, wdt, unpack_lut);
        else unpack_band<2>(d, cfg.sg_width, srcp, rowb, rows, wdt, unpack_lut);
        t_unpack += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - tw1).count();
    };
    int place_threads = std::max(1, static_cast<int>(std::thread::hardware_concurrency()) - 2);
    if (ctx->opt.place_threads > 0) place_threads = ctx->opt.place_threads;
    std::exception_ptr place_err;
    std::thread placer;
    if (!packed_q.empty())
        placer = std::thread([&] {
            try {
                ctx->pool.run(static_cast<int>(packed_q.size()), place_band, place_threads);
            } catch (...) {
                place_err = std::current_exception();
            }
        });
    struct PlacerJoin {  // the placer never outlives this frame, even on an exception
        std::thread& t;
        std::atomic<int>* ready;
        size_t n;
        ~PlacerJoin() {
            if (t.joinable()) {
                for (size_t k = 0; k < n; ++k) ready[k].store(1);
                t.join();
            }
        }
    } placer_join{placer, arr_ready.get(), arrivals.size()};

    // debug timeline: [resident, past-wait, end] per launch
    const bool want_tl = debug_env("CCW_TIMELINE") != nullptr;
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
            // parity halves of the prep outputs: with the fused prep or the flag
            // prep, wave w+1's prep runs while wave w's select may still read its
            // fp64 templates (rescoring, helpers), so the waves alternate halves
            const int par = (fuse_prep || flag_prep) ? (w & 1) : 0;
            SimParams Q = GPP[g][par];
            Q.next_j0 = static_cast<int>(wave_off[g][std::min(w + 1, nkeys)]);
            for (size_t j0 = wave_off[g][w]; j0 < wave_off[g][w + 1]; j0 += maxj) {
                const int nj = static_cast<int>(std::min(maxj, wave_off[g][w + 1] - j0));
                const bool first_wave = w == 0;  // (wave 0 is every realization's first placement)
                if (sharded) {
                    // per shard: screen its window range, local top-K into the
                    // exchange buffer; all-gather across ranks; merge, pick, paste
                    if (!first_wave) {
                        launch_pdl(d_src ? or_prep_src_kernel : or_prep_kernel, dim3(nj), dim3(128), 0, gs, Q,
                                   static_cast<const Job*>(d_jobs), static_cast<int>(j0));
                        ++launches;
                        for (const ShardPart& sp : parts) {
                            SimParams QV = Q;
                            if (!shard_fast) {  // (fast: global positions, full-length rows)
                                QV.p0 = sp.p0;
                                QV.npos = sp.n;
                                QV.K = std::min(Kp, sp.n);
                                QV.sld = sp.sld;
                                QV.ntiles = sp.ntiles;
                            }
                            QV.scores = sp.scores;
                            QV.tmax = sp.tmax;
                            QV.xrec = d_xrec;
                            QV.xnj = nj;
                            QV.xk = Kp;
                            QV.xshard = sp.s;
                            if (any_screen) {
                                cudaEvent_t a = nullptr, b = nullptr;
                                if (ctx->profiling) {
                                    a = tm.get();
                                    b = tm.get();
                                    CCW_CUDA(cudaEventRecord(a, gs));
                                }
                                if (shard_fast) {
                                    launch_ccf_tc(sp.plan, sp.n, sp.sld, kpad, nj, sp.scores + sp.p0,
                                                  sp.tmax + sp.p0 / kTcTile, gs, nullptr, sp.ntiles);
                                } else if (use_tc) {
                                    launch_ccf_tc(sp.plan, sp.n, sp.sld, kpad, nj, sp.scores, sp.tmax, gs);
                                } else {  // fp32 direct screen over the rows holding the shard's range
                                    const int xr0 = sp.p0 / out_w, xr1 = (sp.p0 + sp.n - 1) / out_w;
                                    const unsigned gy = static_cast<unsigned>((xr1 - xr0 + CCF_TX) / CCF_TX);
                                    launch_pdl(ccf_direct_kernel, dim3(ccf_grid_xy.x, gy, nj), dim3(CCF_THREADS),
                                               ccf_smem, gs, QV, static_cast<const Job*>(d_jobs),
                                               static_cast<int>(j0));
                                }
                                if (ctx->profiling) {
                                    CCW_CUDA(cudaEventRecord(b, gs));
                                    tm.ccf.push_back({a, b});
                                }
                                ++launches;
                                ++ccf_launches;
                                if (use_tc) ccf_mma_flop += 2.0 * kpad * static_cast<double>(sp.n) * nj;
                            }
                            if (shard_fast) {
                                if (QV.defer) {
                                    QV.defer_cnt = d_dcnt + 2 * g + dpar[g];
                                    QV.defer_cnt_next = d_dcnt + 2 * g + (1 - dpar[g]);
                                    dpar[g] ^= 1;
                                }
                                launch_pdl(select_fast_kernel<false>, dim3(nj), dim3(FS_T), 0, gs, QV,
                                           static_cast<const Job*>(d_jobs), static_cast<int>(j0), nj);
                                if (QV.defer) {
                                    launch_pdl(select_bulk_kernel, dim3(tc_num_sms()), dim3(BK_T),
                                               bulk_smem, gs, QV, static_cast<const Job*>(d_jobs), static_cast<int>(j0),
                                               nj, bulk_S);
                                    ++launches;
                                }
                            } else {
                                launch_pdl(select_paste_kernel, dim3(nj), dim3(SEL_T), sel_smem, gs, QV,
                                           static_cast<const Job*>(d_jobs), static_cast<int>(j0),
                                           use_screen ? 1 : (norm_screen ? 2 : 0));
                            }
                            ++launches;
                        }
                        if (any_screen && j0 == wave_off[g][w]) {
                            double nL = 0, nS = 0, mine = 0;
                            for (const ShardPart& sp : parts) mine += sp.n;
                            for (int r = 0; r < n_real; ++r) {
                                nL += vhistL[vid[r]][w];
                                nS += vhist[vid[r]][w] - vhistL[vid[r]][w];
                            }
                            const double m = nL * mask_cells + nS * static_cast<double>(Tc) * OVc;
                            ccf_flop += 2.0 * ti->nscr * mine * m;
                            ccf_flop_ref += 2.0 * ti->nch * mine * m;
                        }
                        if (ctx->nccl_comm) {
                            const size_t chunk = static_cast<size_t>(S_virt) * nj * Kp;
                            nccl_all_gather_bytes(ctx->nccl_comm, d_xrec + ctx->shard_rank * chunk, d_xrec,
                                                  chunk * sizeof(ShardRec), gs);
                        }
                    }
                    SimParams QM = Q;
                    QM.xrec = d_xrec;
                    QM.xnj = nj;
                    QM.xk = Kp;
                    launch_pdl(shard_merge_kernel, dim3(nj), dim3(SEL_T), sel_smem, gs, QM,
                               static_cast<const Job*>(d_jobs), static_cast<int>(j0), S_all);
                    ++launches;
                    continue;
                }
                if (use_wave && !first_wave) {
                    cudaEvent_t a = nullptr, b = nullptr;
                    if (ctx->profiling) {
                        a = tm.get();
                        b = tm.get();
                        CCW_CUDA(cudaEventRecord(a, gs));
                    }
                    SimParams QW = Q;
                    QW.tl = tl_next(w, g, 1);
                    const int cs = wave_pick_cs(QW, nj, ctx->opt.wave_cs);
                    launch_wave(QW, d_jobs, static_cast<int>(j0), nj, d_strips, wave_nmb, wave_nb, cs, d_wave_w + g * wave_w_per_group, gs);
                    if (ctx->profiling) {
                        CCW_CUDA(cudaEventRecord(b, gs));
                        tm.ccf.push_back({a, b});
                    }
                    ++launches;
                    ++ccf_launches;
                    const int jps = wave_jobs_per_set();
                    ccf_mma_flop += 2.0 * ((nj + jps - 1) / jps) * jps * (static_cast<double>(wave_nb) * wave_nmb * out_w) *
                                    (ti->nscr * ((Tc + 1) & ~1) * 16.0);
                    if (j0 == wave_off[g][w]) {
                        double nL = 0, nS = 0;
                        for (int r = 0; r < n_real; ++r)
                            if (group_of(r) == g) {
                                nL += vhistL[vid[r]][w];
                                nS += vhist[vid[r]][w] - vhistL[vid[r]][w];
                            }
                        const double m = nL * mask_cells + nS * static_cast<double>(Tc) * OVc;
                        ccf_flop += 2.0 * ti->nscr * npos * m;
                        ccf_flop_ref += 2.0 * ti->nch * npos * m;
                    }
                    continue;
                }
                if (!first_wave) {
                    Q.tl = tl_next(w, g, 0);
                    if (!fuse_prep) {  // (fused: prepared by the previous wave's select)
                        if (d_src)  // (+1 CTA with flag_prep: it waits for the previous launch in full)
                            launch_pdl(or_prep_src_kernel, dim3(nj + (flag_prep ? 1 : 0)), dim3(128), 0, gs, Q,
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
                        if (use_tc) {
                            launch_ccf_tc(tcplans[g][par], npos, sld, kpad, nj, Q.scores, Q.tmax, gs,
                                          tl_next(w, g, 1), -1, Q.s16, Q.tmax_nu, d_ubits, P.ustride, Q.jvar);
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
                        if (j0 == wave_off[g][w]) {  // the whole wave's mask cells, at its first launch
                            double nL = 0, nS = 0;
                            for (int r = 0; r < n_real; ++r)
                                if (group_of(r) == g) {
                                    nL += vhistL[vid[r]][w];
                                    nS += vhist[vid[r]][w] - vhistL[vid[r]][w];
                                }
                            const double m = nL * mask_cells + nS * static_cast<double>(Tc) * OVc;
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
                if (warp_select || (first_wave && !cfg.min_cut)) {
                    const Job* dj = d_jobs;
                    if (d_boards) {
                        Q.hb = d_boards + 2 * g + hb_par[g];
                        Q.hs = d_hslots + (2 * g + hb_par[g]) * maxj;
                        Q.hb_reset = d_boards + 2 * g + (1 - hb_par[g]);
                        Q.hs_reset = d_hslots + (2 * g + (1 - hb_par[g])) * maxj;
                        hb_par[g] ^= 1;
                    }
                    if (Q.defer && !first_wave) {
                        Q.defer_cnt = d_dcnt + 2 * g + dpar[g];
                        Q.defer_cnt_next = d_dcnt + 2 * g + (1 - dpar[g]);
                        dpar[g] ^= 1;
                    }
                    launch_pdl(Q.s16 ? select_fast_kernel<true> : select_fast_kernel<false>, dim3(nj), dim3(FS_T), 0, gs, Q, dj,
                               static_cast<int>(j0), nj);
                    if (Q.defer && !first_wave) {
                        Q.tl = tl_next(w, g, 5);
                        launch_pdl(select_bulk_kernel, dim3(tc_num_sms()), dim3(BK_T), bulk_smem,
                                   gs, Q, dj, static_cast<int>(j0), nj, bulk_S);
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
            if (band_next[g] < band_at[g].size() && band_at[g][band_next[g]].w == w) {
                const Checkpoint ck = band_at[g][band_next[g]++];
                // final bands are never written again: rebuild and copy them on the copy
                // stream, off the group's critical path
                cudaEvent_t be = tm.get();
                CCW_CUDA(cudaEventRecord(be, gs));
                CCW_CUDA(cudaStreamWaitEvent(ctx->copy_streams[g], be, 0));
                auto launch_bands = [&](size_t q0, size_t q1, bool packed) {
                    size_t most = 1;  // cells of the largest band: enough CTAs to cover it
                    for (size_t q = q0; q < q1; ++q)
                        most = std::max(most, static_cast<size_t>(bands[q].w - bands[q].z) *
                                                  (bands[q].y == 0 ? cfg.sg_width : cfg.sg_height));
                    const size_t per_thread = packed && pack_bits < 8 ? static_cast<size_t>(pack_cpb) : fin_cells;
                    const size_t band_cap = ck.w == max_key ? band_cap_last : band_cap_mid;
                    const int bxb = static_cast<int>(std::min<size_t>((most / per_thread + 255) / 256 + 1, band_cap));
                    auto band = [&](auto kern) {
                        launch_pdl(kern, dim3(bxb, static_cast<unsigned>(q1 - q0)), dim3(256), 0, ctx->copy_streams[g],
                                   static_cast<const int4*>(d_bands + q0),
                                   static_cast<const long long*>(packed ? d_boff + q0 : nullptr),
                                   static_cast<const uint8_t*>(d_work), wh, ww, static_cast<const int32_t*>(d_src), B,
                                   J, swc, static_cast<const uint8_t*>(ti->d_codes), ti->w, ti->wc,
                                   static_cast<const uint8_t*>(d_hd), cfg.sg_height, cfg.sg_width,
                                   packed ? d_stage : fin, d_mism, tl_next(w, g, 4));
                    };
                    if (packed && pack_bits == 1) band(pack_band_kernel<1>);
                    else if (packed && pack_bits == 2) band(pack_band_kernel<2>);
                    else if (packed && pack_bits == 4) band(pack_band_kernel<4>);
                    else if (fin_bt == 2) band(finalize_band_kernel<2>);
                    else if (fin_bt == 4) band(finalize_band_kernel<4>);
                    else if (fin_bt == 8) band(finalize_band_kernel<8>);
                    else band(finalize_band_kernel<0>);
                    ++launches;
                };
                if (ck.bm > ck.b0) {  // row bands, finalized in place and copied straight to the caller
                    launch_bands(ck.b0, ck.bm, false);
                    const size_t n = static_cast<size_t>(cfg.sg_height) * cfg.sg_width;
                    size_t o0 = 0, o1 = 0;
                    auto flush = [&] {
                        if (o1 > o0)
                            CCW_CUDA(cudaMemcpyAsync(h_out + o0, fin + o0, o1 - o0, cudaMemcpyDeviceToHost,
                                                     ctx->copy_streams[g]));
                        o0 = o1 = 0;
                    };
                    for (size_t q = ck.b0; q < ck.bm; ++q) {
                        const int4 bd = bands[q];
                        const size_t a0 = static_cast<size_t>(bd.x) * n + static_cast<size_t>(bd.z) * cfg.sg_width;
                        const size_t a1 = static_cast<size_t>(bd.x) * n + static_cast<size_t>(bd.w) * cfg.sg_width;
                        if (a0 != o1) flush();
                        if (o1 == 0) o0 = a0;
                        o1 = a1;
                    }
                    flush();
                }
                if (ck.b1 > ck.bm) {  // packed bands: one contiguous copy into the host staging
                    launch_bands(ck.bm, ck.b1, true);
                    const size_t p0 = static_cast<size_t>(band_off[ck.bm]);
                    const size_t p1 = static_cast<size_t>(band_off[ck.b1 - 1]) + band_bytes(ck.b1 - 1);
                    CCW_CUDA(cudaMemcpyAsync(h_stage + p0, d_stage + p0, p1 - p0, cudaMemcpyDeviceToHost,
                                             ctx->copy_streams[g]));
                    const size_t k = arrival_index(ck.bm);
                    CCW_CUDA(cudaEventRecord(arrivals[k].ev, ctx->copy_streams[g]));
                    arr_ready[k].store(1, std::memory_order_release);
                }
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
        const size_t n = static_cast<size_t>(cfg.sg_height) * cfg.sg_width / fin_cells + 1;
        const int bx = static_cast<int>(std::min<size_t>((n + 255) / 256, 1024));
        auto full = [&](auto kern) {
            kern<<<dim3(bx, n_real), 256, 0, st>>>(d_work, wh, ww, d_src, B, J, swc, ti->d_codes, ti->w, ti->wc,
                                                 d_hd, cfg.sg_height, cfg.sg_width, fin, d_mism);
        };
        if (fin_bt == 2) full(finalize_kernel<2>);
        else if (fin_bt == 4) full(finalize_kernel<4>);
        else if (fin_bt == 8) full(finalize_kernel<8>);
        else full(finalize_kernel<0>);
        ++launches;
        CCW_CUDA(cudaGetLastError());
    }
    if (host_t)
        fprintf(stderr, "host ms: seed %.3f sched %.3f prep %.3f ev0 %.3f launched %.3f\n", t_seed, t_sched, host_prep_ms,
                t_ev0, host_ms());
    const double t_launched = host_t ? host_ms() : 0.0;
    CCW_CUDA(cudaEventRecord(ev1, st));
    if (async_call) {
        // device output, no diagnostics: the counters go to this call's pinned
        // slot and are folded in by a later call or ccw_ctx_synchronize
        ccw_ctx::AsyncSlot& sl = ctx->aslot[apar];
        CCW_CUDA(cudaEventRecord(sl.t1, st));
        unsigned long long* res = static_cast<unsigned long long*>(sl.res.get(sizeof(unsigned long long) * (kNumStats + 1)));
        res[kNumStats] = 0;
        CCW_CUDA(cudaMemcpyAsync(res, d_stats, sizeof(unsigned long long) * kNumStats, cudaMemcpyDeviceToHost, st));
        CCW_CUDA(cudaMemcpyAsync(res + kNumStats, ctx->sched_err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        CCW_CUDA(cudaEventRecord(sl.done, st));
        sl.timing = ccw_timing{};
        sl.timing.ccf_launches = ccf_launches;
        sl.timing.launches = launches + (d_hd ? 1 : 0);
        sl.timing.ccf_flop = ccf_flop;
        sl.timing.ccf_flop_ref = ccf_flop_ref;
        sl.timing.waves = static_cast<int64_t>(max_key + 1);
        sl.timing.groups = G;
        sl.timing.host_prep_ms = host_prep_ms;
        sl.timing.jobs = static_cast<int64_t>(total_jobs);
        sl.timing.ccf_variant = any_screen ? (use_wave ? 5 : (use_tc ? 2 : 1)) : 0;
        sl.timing.ccf_mma_flop = use_tc ? ccf_mma_flop : 0.0;
        sl.key = bulk_key;
        sl.use_wave = use_wave;
        sl.bulk_launch = bulk_launch;
        sl.valid = true;
        ctx->async_par = 1 - apar;
        return;
    }
    if (placer.joinable()) placer.join();
    if (place_err) std::rethrow_exception(place_err);
    if (host_t)
        fprintf(stderr, "host ms: bands placed %.3f (thread-ms waiting %.3f, unpacking %.3f, bands %zu)\n", host_ms(),
                t_wait * 1e-6, t_unpack * 1e-6, packed_q.size());
    if (h_out && !stream_out)
        CCW_CUDA(cudaMemcpyAsync(h_dst, fin, out_bytes, cudaMemcpyDeviceToHost, st));
    unsigned long long stats[kNumStats] = {0};
    CCW_CUDA(cudaMemcpyAsync(stats, d_stats, sizeof(stats), cudaMemcpyDeviceToHost, st));
    std::vector<int> mism(n_real, 0);
    CCW_CUDA(cudaMemcpyAsync(mism.data(), d_mism, sizeof(int) * n_real, cudaMemcpyDeviceToHost, st));
    std::vector<int32_t> chosen;
    std::vector<uint8_t> pasted;
    std::vector<Job> flat_jobs;
    int sched_err = 0;
    CCW_CUDA(cudaMemcpyAsync(&sched_err, ctx->sched_err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    if (traces) {
        chosen.resize(2 * total_jobs);
        CCW_CUDA(cudaMemcpyAsync(chosen.data(), d_chosen, sizeof(int32_t) * chosen.size(),
                                 cudaMemcpyDeviceToHost, st));
        flat_jobs.resize(total_jobs);
        CCW_CUDA(cudaMemcpyAsync(flat_jobs.data(), d_jobs, sizeof(Job) * total_jobs, cudaMemcpyDeviceToHost, st));
        pasted.resize(total_jobs * T * T);
        CCW_CUDA(cudaMemcpyAsync(pasted.data(), d_pasted, pasted.size(), cudaMemcpyDeviceToHost, st));
    }
    CCW_CUDA(cudaStreamSynchronize(st));
    if (sched_err) throw Fail(CCW_ERR_GENERIC, "internal: device schedule disagrees with the host path draws");
    if (d_jdump) {  // debug: per-job select timing, with each job's group and wave
        std::vector<unsigned long long> jd(8 * total_jobs);
        CCW_CUDA(cudaMemcpy(jd.data(), d_jdump, sizeof(unsigned long long) * jd.size(), cudaMemcpyDeviceToHost));
        if (FILE* f = fopen(jdump_path, "wb")) {
            std::vector<int32_t> gw(2 * total_jobs);
            for (int g = 0; g < G; ++g)
                for (int w = 0; w < nkeys; ++w)
                    for (size_t j = wave_off[g][w]; j < wave_off[g][w + 1]; ++j) {
                        gw[2 * j] = g;
                        gw[2 * j + 1] = w;
                    }
            const uint64_t tj = total_jobs;
            fwrite(&tj, sizeof(tj), 1, f);
            fwrite(jd.data(), sizeof(unsigned long long), jd.size(), f);
            fwrite(gw.data(), sizeof(int32_t), gw.size(), f);
            fclose(f);
        }
    }
    if (host_t) {
        float sms = 0;
        cudaEventElapsedTime(&sms, ev_sched, ev0);
        fprintf(stderr, "device schedule (uploads + build_jobs) %.3f ms; host waited %.3f ms after launching\n", sms,
                host_ms() - t_launched);
    }
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
    {
        size_t d2h = h_out && !stream_out ? out_bytes : 0;
        for (size_t q = 0; q < bands.size(); ++q)
            d2h += band_off[q] < 0 ? band_rows(bands[q]) * cfg.sg_width : band_bytes(q);
        ctx->timing.d2h_bytes = static_cast<int64_t>(d2h);
    }
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
    if (debug_env("CCW_TAIL"))
        fprintf(stderr, "select jobs: ties %llu avg %.0f max %llu cycles | no ties %llu avg %.0f max %llu cycles\n",
                stats[16], stats[16] ? double(stats[17]) / stats[16] : 0.0, stats[18], stats[19],
                stats[19] ? double(stats[20]) / stats[19] : 0.0, stats[21]);
    if (debug_env("CCW_TAIL"))
        fprintf(stderr, "select cycles histogram <10k %llu <20k %llu <40k %llu <80k %llu >=80k %llu | long jobs: scan+stage %llu batch %llu choose+map %llu candidates %llu\n",
                stats[22], stats[23], stats[24], stats[25], stats[26], stats[27], stats[28], stats[29], stats[30]);
    if (debug_env("CCW_TAIL"))
        fprintf(stderr, "shared rescoring: posts %llu, chunks %llu (own %llu), owner help cycles %llu wait cycles %llu\n",
                stats[32], stats[33], stats[34], stats[35], stats[36]);
    if (debug_env("CCW_TAIL"))
        fprintf(stderr, "small groups (g < 8): %llu, rescore+select cycles avg %.0f (items %.0f), scan->group cycles avg %.0f\n",
                stats[37], stats[37] ? double(stats[38]) / stats[37] : 0.0, stats[37] ? double(stats[40]) / stats[37] : 0.0,
                stats[37] ? double(stats[39]) / stats[37] : 0.0);
    if (debug_env("CCW_TAIL"))
        fprintf(stderr, "small-group item (thread 0): loads+products %.0f chain+stores %.0f cycles over %llu\n",
                stats[43] ? double(stats[41]) / stats[43] : 0.0, stats[43] ? double(stats[42]) / stats[43] : 0.0, stats[43]);
    if (debug_env("CCW_PHASES") && use_wave && stats[14])
        fprintf(stderr, "wave CTA phases (mean cycles from CTA start over %llu CTAs): dep-wait %.0f prep-own %.0f prep+sync %.0f screen %.0f "
                "lists-sync %.0f post+sync %.0f end %.0f\n", stats[14], stats[8] / double(stats[14]), stats[24] / double(stats[14]),
                stats[9] / double(stats[14]), stats[10] / double(stats[14]), stats[11] / double(stats[14]),
                stats[12] / double(stats[14]), stats[13] / double(stats[14]));
    if (debug_env("CCW_PHASES") && use_wave && stats[14])
        fprintf(stderr, "wave screen per CTA: mma waits acc %.0f full %.0f issue %.0f | epilogue(q0) waits %.0f work %.0f (ldtm %.0f) | "
                "compactions per tile %.3f | tiles per CTA %.1f\n", stats[16] / double(stats[14]), stats[17] / double(stats[14]),
                stats[22] / double(stats[14]), stats[18] / double(stats[14]), stats[19] / double(stats[14]), stats[23] / double(stats[14]), stats[20] / double(std::max(1ull, stats[21])),
                stats[21] / double(stats[14]));
    if (debug_env("CCW_PHASES") && use_wave && stats[14])
        fprintf(stderr, "wave epilogue(q0) split per CTA: ldtm %.0f first-tile insert %.0f filter %.0f list %.0f bound-read %.0f "
                "bound-publish %.0f\n", stats[25] / double(stats[14]), stats[26] / double(stats[14]), stats[27] / double(stats[14]),
                stats[28] / double(stats[14]), stats[29] / double(stats[14]), stats[30] / double(stats[14]));
    if (debug_env("CCW_PHASES"))
        fprintf(stderr, "bulk CTA phases: setup %llu loop %llu (max CTA %llu) last-CTA merge+paste %llu cycles\n",
                stats[44], stats[45], stats[46], stats[47]);
    if (debug_env("CCW_PHASES"))
        fprintf(stderr, "phase clocks: scan[M_K %llu list %llu S_K %llu cand %llu] fast[scan+stage %llu batch %llu choose+map %llu]"
                " | bulk total %llu stage %llu compute %llu | tiles>=M_K %llu list %llu\n",
                stats[8], stats[9], stats[10], stats[11], stats[12], stats[13], stats[4], stats[7], stats[14],
                stats[15], stats[5], stats[6]);
    ctx->timing.screened_jobs = static_cast<int64_t>(stats[1]);
    ctx->timing.list_overflows = static_cast<int64_t>(stats[2]);
    ctx->timing.bulk_jobs = static_cast<int64_t>(stats[3]);
    ctx->timing.shared_groups = static_cast<int64_t>(stats[32]);
    learn_plan(ctx, bulk_key, use_wave, bulk_launch, stats);
    ctx->timing.ccf_variant = any_screen ? (use_wave ? 5 : (use_tc ? 2 : 1)) : 0;
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
            const Job& jb = flat_jobs[g];
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
