// sim3d.cu -- the 3D CCWSIM extension (BASELINE configs 3 and 4) on sm_100a.
//
// The reference has no 3D; oracle/ccw3d_oracle.h is the
// normative definition: the 2D algorithm of
// simulator.hpp:148-252,418-519 / matcher.hpp:64-81,177-241 /
// wavelet.hpp:69-106 generalized to three axes, scored EXACTLY from
// per-facies block counts (a level-J 3D Haar apex is count / (2 sqrt 2)^J),
// ranked by (score desc, row-major position asc).
//
// Device pipeline per placement wave (waves as in 2D: key
// (d+1)^2 io + (d+1) im + ii orders every overlapping pair as the raster loop
// does and lets the rest of a wave run concurrently):
//
//   prep3d    overlap block counts of every job from the resident work grid
//             -> integer weights (n_f - n_{F-1}, the one-hot TI makes the
//             F-1 channel sum rank exactly like the F channel sum)
//   screen3d  exact integer CCF of a batch of up to 8 jobs sharing one mask
//             over a box of TI window positions: the box's TI block counts
//             staged in shared memory (row pitch padded so a warp's loads hit
//             32 distinct banks), packed int8x4 channels + dp4a when every
//             count fits int8 (J <= 2), int32 IMAD per channel otherwise; the
//             box's top-K packed keys (score << 32 | ~position) per job
//   [ncclAllGather of the shards' box lists when positions are sharded]
//   select3d  merge of the box lists -> the job's top-K, conditional /
//             unconditional pick, T^3 paste into the work grid
//
// and finalize3d crops the realizations and forces the hard data.
#include <algorithm>
#include <chrono>
#include <climits>
#include <cstring>

#include "ccf_tc.hpp"
#include "ccw_device.cuh"
#include "internal.hpp"

namespace ccwgpu {

namespace {

constexpr int JB = 8;       // jobs per screen batch (one mask)
constexpr int KMAX3 = 16;   // candidates per job (3D path)
constexpr int S3_THREADS = 256;

struct Job3 {
    int32_t real, place;
    int32_t P[3];     // footprint origin in the work grid
    int32_t mask;     // mask id = corner * 8 + shape (shape: bit a = slab on axis a)
    int32_t bmask;    // the screen batch's mask: corner * 8 + union of its jobs' shapes
    int32_t pick;     // unconditional draw; -1 conditional; -2 first placement
    int32_t fr[3];    // first placement's TI origin
    int32_t lat;      // lattice cell of the footprint (hard-data lists)
};

struct Batch3 {
    int32_t j0, n, mask, pad;
};

struct Geo3 {
    int c[3];      // TI coarse extents used
    int o[3];      // window positions per axis
    int tc, B, J, T, OV, nscr, F;
    int ti[3];     // TI fine extents (array dims)
    int W[3];      // work grid extents
    int sg[3];
    int any_support;
    int mode;      // 0: int8x4 counts + dp4a, 1: int32 per channel
    int aligned4;  // paste may move 4-byte words
};

// ----------------------------------------------------------- pyramid -----
// block counts of channels 0..nscr-1 (facies codes); mode 0: int8x4 packed
// (counts <= 64), mode 1: int32 planes [ch][cell].
__global__ void pyramid3d_kernel(const uint8_t* __restrict__ ti, int d0, int d1, int d2, int c0, int c1,
                                 int c2, int B, int nscr, int mode, int32_t* __restrict__ out) {
    const size_t nc = static_cast<size_t>(c0) * c1 * c2;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < nc;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int q0 = static_cast<int>(e / (static_cast<size_t>(c1) * c2));
        const int q1 = static_cast<int>((e / c2) % c1), q2 = static_cast<int>(e % c2);
        int cnt[16] = {0};
        for (int x0 = 0; x0 < B; ++x0)
            for (int x1 = 0; x1 < B; ++x1) {
                const uint8_t* row = ti + (static_cast<size_t>(q0 * B + x0) * d1 + q1 * B + x1) * d2 + q2 * B;
                for (int x2 = 0; x2 < B; ++x2) {
                    const int f = row[x2];
#pragma unroll
                    for (int ch = 0; ch < 16; ++ch)
                        if (ch == f) ++cnt[ch];
                }
            }
        if (mode == 0) {
            uint32_t v = 0;
            for (int ch = 0; ch < nscr && ch < 4; ++ch) v |= (static_cast<uint32_t>(cnt[ch]) & 0xFFu) << (8 * ch);
            out[e] = static_cast<int32_t>(v);
        } else {
            for (int ch = 0; ch < nscr; ++ch) out[ch * nc + e] = ch < 16 ? cnt[ch] : 0;
        }
    }
}

// ------------------------------------------------------------- prep ------
// One CTA per job, one warp per mask cell at a time: the overlap's facies
// counts over the block's supported fine cells (simulator.hpp:225-272 in 3D).
__global__ void __launch_bounds__(256) prep3d_kernel(Geo3 g, const Job3* __restrict__ jobs, int j0,
                                                     const int* __restrict__ mask_off,
                                                     const int* __restrict__ mask_cells,
                                                     const uint8_t* __restrict__ work, int32_t* __restrict__ wbuf,
                                                     int wstride, int tcrow) {
    // tcrow > 0 (tcgen05 screen of 9-bit counts, see im2col3d_digits_kernel):
    // wbuf holds THREE int8 GEMM rows per job (row stride wstride * 4 / 3
    // bytes), two digit bytes per (window cell, channel) over all tcrow = tc^3
    // window cells (zero off the job's own overlap support); else one int32
    // entry per cell of the batch's mask and channel.
    pdl_trigger();
    pdl_wait();
    const Job3 jb = jobs[j0 + blockIdx.x];
    const int corner = jb.mask >> 3, shape = jb.mask & 7;  // the job's own overlap support
    const int m_lo = mask_off[jb.bmask];
    const int nm = tcrow > 0 ? tcrow : mask_off[jb.bmask + 1] - m_lo;  // cells of its batch's mask
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int B = g.B, B3 = B * B * B;
    const uint8_t* wk = work + static_cast<size_t>(jb.real) * g.W[0] * g.W[1] * g.W[2];
    int32_t* wout = wbuf + static_cast<size_t>(blockIdx.x) * wstride;
    const int nw = blockDim.x >> 5;
    for (int i = blockIdx.y * nw + warp; i < nm; i += gridDim.y * nw) {
        int m0, m1, m2;
        int B3e = B3;  // (0: the block touches none of the job's slabs, nothing to count)
        if (tcrow > 0) {
            m2 = i % g.tc, m1 = (i / g.tc) % g.tc, m0 = i / (g.tc * g.tc);
            const int m[3] = {m0, m1, m2};
            bool any = false;
#pragma unroll
            for (int a = 0; a < 3; ++a)
                if ((shape >> a) & 1) any |= !((corner >> a) & 1) ? m[a] * B < g.OV : m[a] * B + B > g.T - g.OV;
            if (!any) B3e = 0;
        } else {
            const int cell = mask_cells[m_lo + i];
            m0 = cell >> 16, m1 = (cell >> 8) & 0xFF, m2 = cell & 0xFF;
        }
        int wv[16];
        const int last = g.F - 1;
        int nlast = 0;
        if (B3 <= 4096) {
            // byte counters, four facies per word (a lane sees <= 128 cells),
            // summed over the warp as 16-bit halves (<= 4096); B = 2^J: shifts
            uint32_t c4[4] = {0, 0, 0, 0};
            const int J = g.J, bm = B - 1;
            const bool fast8 = B == 8 && g.aligned4;
            if (fast8 && B3e) {
                // B = 8, aligned rows: the block is 64 rows of two 4-byte words; a
                // lane loads its four words up front (independent, inside the
                // work grid) and counts a facies as byte-equality masks under
                // the word's support mask (as prep3d_cell_kernel)
                int lo3[3], hi3[3];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const bool on = (shape >> a) & 1, asc = !((corner >> a) & 1);
                    lo3[a] = !on ? 1 : asc ? 0 : g.T - g.OV;
                    hi3[a] = !on ? 0 : asc ? g.OV : g.T;
                }
                uint32_t wd[4], sm[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int wi = lane + 32 * k, row = wi >> 1, half = wi & 1;
                    const int X0 = m0 * 8 + (row >> 3), X1 = m1 * 8 + (row & 7), X2 = m2 * 8 + half * 4;
                    wd[k] = *reinterpret_cast<const uint32_t*>(
                        wk + (static_cast<size_t>(jb.P[0] + X0) * g.W[1] + jb.P[1] + X1) * g.W[2] + jb.P[2] + X2);
                    uint32_t m = 0;
                    if ((X0 >= lo3[0] && X0 < hi3[0]) || (X1 >= lo3[1] && X1 < hi3[1])) {
                        m = 0xFFFFFFFFu;
                    } else {
#pragma unroll
                        for (int b = 0; b < 4; ++b)
                            if (X2 + b >= lo3[2] && X2 + b < hi3[2]) m |= 0xFFu << (8 * b);
                    }
                    sm[k] = m;
                }
#pragma unroll
                for (int ch = 0; ch < 16; ++ch)
                    if (ch < g.F) {  // (uniform)
                        int n = 0;
#pragma unroll
                        for (int k = 0; k < 4; ++k) n += __popc(__vcmpeq4(wd[k], 0x01010101u * ch) & sm[k]);
                        c4[ch >> 2] += static_cast<uint32_t>(n >> 3) << (8 * (ch & 3));
                    }
            }
            for (int e = lane; e < (fast8 ? 0 : B3e); e += 32) {
                const int x0 = m0 * B + (e >> (2 * J)), x1 = m1 * B + ((e >> J) & bm), x2 = m2 * B + (e & bm);
                const int x[3] = {x0, x1, x2};
                bool sup = false;
#pragma unroll
                for (int a = 0; a < 3; ++a)
                    if ((shape >> a) & 1) {
                        const bool asc = !((corner >> a) & 1);
                        sup |= asc ? x[a] < g.OV : x[a] >= g.T - g.OV;
                    }
                if (!sup) continue;
                const int f = wk[(static_cast<size_t>(jb.P[0] + x0) * g.W[1] + jb.P[1] + x1) * g.W[2] + jb.P[2] + x2];
                const uint32_t inc = 1u << ((f & 3) * 8);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if ((f >> 2) == q) c4[q] += inc;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t lo = 0, hi = 0;
                if (4 * q < g.F) {  // (uniform: F is a launch constant)
                    lo = __reduce_add_sync(0xffffffffu, c4[q] & 0x00FF00FFu);
                    hi = __reduce_add_sync(0xffffffffu, (c4[q] >> 8) & 0x00FF00FFu);
                }
                wv[4 * q] = lo & 0xFFFF;
                wv[4 * q + 1] = hi & 0xFFFF;
                wv[4 * q + 2] = lo >> 16;
                wv[4 * q + 3] = hi >> 16;
            }
#pragma unroll
            for (int ch = 0; ch < 16; ++ch)
                if (ch == last) nlast = wv[ch];
        } else {
            int cnt[16] = {0};
            for (int e = lane; e < B3e; e += 32) {
                const int x0 = m0 * B + e / (B * B), x1 = m1 * B + (e / B) % B, x2 = m2 * B + e % B;
                const int x[3] = {x0, x1, x2};
                bool sup = false;
#pragma unroll
                for (int a = 0; a < 3; ++a)
                    if ((shape >> a) & 1) {
                        const bool asc = !((corner >> a) & 1);
                        sup |= asc ? x[a] < g.OV : x[a] >= g.T - g.OV;
                    }
                if (!sup) continue;
                const int f = wk[(static_cast<size_t>(jb.P[0] + x0) * g.W[1] + jb.P[1] + x1) * g.W[2] + jb.P[2] + x2];
#pragma unroll
                for (int ch = 0; ch < 16; ++ch)
                    if (ch == f) ++cnt[ch];
            }
#pragma unroll
            for (int ch = 0; ch < 16; ++ch) {
                const int s = ch < g.F ? __reduce_add_sync(0xffffffffu, cnt[ch]) : 0;  // (uniform)
                if (ch == last) nlast = s;
                wv[ch] = s;
            }
        }
#ifdef CCW_DEBUG3D
        if (lane == 0 && blockIdx.x == 0) printf("prep job %d cell %d (%d,%d,%d) counts %d %d %d %d\n", j0, i, m0, m1, m2, wv[0], wv[1], wv[2], wv[3]);
#endif
        if (lane == 0) {
            if (tcrow > 0) {
                // w = 32 hi + lo, lo in [0, 32), |hi| <= 16; against x = 32 xh + xl:
                // row 1 . X = sum hi xh, row 2 . X = sum (lo xh + hi xl), row 3 . X = sum lo xl
                const int kbytes = wstride * 4 / 3;
                int8_t* r1 = reinterpret_cast<int8_t*>(wout);
#pragma unroll
                for (int ch = 0; ch < 16; ++ch)
                    if (ch < g.nscr) {
                        const int w = g.F > 1 ? wv[ch] - nlast : 0;
                        const uint32_t wl = static_cast<uint32_t>(w & 31), wh = static_cast<uint32_t>(w >> 5) & 0xFFu;
                        const int off = (i * g.nscr + ch) * 2;
                        *reinterpret_cast<uint16_t*>(r1 + off) = static_cast<uint16_t>(wh);
                        *reinterpret_cast<uint16_t*>(r1 + kbytes + off) = static_cast<uint16_t>(wl | (wh << 8));
                        *reinterpret_cast<uint16_t*>(r1 + 2 * kbytes + off) = static_cast<uint16_t>(wl << 8);
                    }
            } else if (g.mode == 0) {  // int8x4
                uint32_t v = 0;
#pragma unroll
                for (int ch = 0; ch < 4; ++ch)
                    if (ch < g.nscr) {
                        const int w = g.F > 1 ? wv[ch] - nlast : 0;
                        v |= (static_cast<uint32_t>(w) & 0xFFu) << (8 * ch);
                    }
                wout[i] = static_cast<int32_t>(v);
            } else {
#pragma unroll
                for (int ch = 0; ch < 16; ++ch)
                    if (ch < g.nscr) wout[i * g.nscr + ch] = g.F > 1 ? wv[ch] - nlast : 0;
            }
        }
    }
}

// The same weights for B <= 4 with B threads per coarse cell (one x0 plane of
// the block each, <= 4 rows of <= 4 facies bytes): every row is loaded before
// anything is counted (independent loads, always inside the work grid), a
// facies' cells are counted as byte-equality masks (__vcmpeq4 + popc) under
// the row's support mask, and the planes are summed with shuffles on byte
// counters (a block has <= 64 cells).  The warp-per-cell kernel above is
// instruction- and latency-bound at these block sizes.  W4: aligned 4-byte rows.
template <int B, bool W4>
__global__ void __launch_bounds__(128) prep3d_cell_kernel(Geo3 g, const Job3* __restrict__ jobs, int j0,
                                                          const int* __restrict__ mask_off,
                                                          const int* __restrict__ mask_cells,
                                                          const uint8_t* __restrict__ work,
                                                          int32_t* __restrict__ wbuf, int wstride, int tcrow) {
    pdl_trigger();
    pdl_wait();
    const Job3 jb = jobs[j0 + blockIdx.x];
    const int corner = jb.mask >> 3, shape = jb.mask & 7;
    const int m_lo = mask_off[jb.bmask];
    const int nm = tcrow > 0 ? tcrow : mask_off[jb.bmask + 1] - m_lo;
    const int gi = blockIdx.y * blockDim.x + threadIdx.x;
    const int i = gi / B, x0 = gi % B;  // (a cell's B threads share a warp)
    int32_t* wout = wbuf + static_cast<size_t>(blockIdx.x) * wstride;
    int m0 = 0, m1 = 0, m2 = 0;
    bool live = i < nm;
    if (live) {
        if (tcrow > 0) {
            m2 = i % g.tc, m1 = (i / g.tc) % g.tc, m0 = i / (g.tc * g.tc);
        } else {
            const int cell = mask_cells[m_lo + i];
            m0 = cell >> 16, m1 = (cell >> 8) & 0xFF, m2 = cell & 0xFF;
        }
    }
    // per axis: fine coordinates [lo, hi) of the template lie in the job's slab
    int lo[3], hi[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const bool on = (shape >> a) & 1, asc = !((corner >> a) & 1);
        lo[a] = !on ? 1 : asc ? 0 : g.T - g.OV;
        hi[a] = !on ? 0 : asc ? g.OV : g.T;
    }
    uint32_t rw[B];  // this plane's rows, B facies bytes each
    uint32_t sm[B];  // 0xFF in the bytes of supported cells
#pragma unroll
    for (int x1 = 0; x1 < B; ++x1) rw[x1] = sm[x1] = 0;
    if (live) {
        const uint8_t* wk = work + static_cast<size_t>(jb.real) * g.W[0] * g.W[1] * g.W[2];
        const uint8_t* base = wk + (static_cast<size_t>(jb.P[0] + m0 * B + x0) * g.W[1] + jb.P[1] + m1 * B) * g.W[2] +
                              jb.P[2] + m2 * B;
#pragma unroll
        for (int x1 = 0; x1 < B; ++x1) {
            const uint8_t* row = base + static_cast<size_t>(x1) * g.W[2];
            if constexpr (W4) {
                rw[x1] = *reinterpret_cast<const uint32_t*>(row);
            } else {
                uint32_t w = 0;
#pragma unroll
                for (int x2 = 0; x2 < B; ++x2) w |= static_cast<uint32_t>(row[x2]) << (8 * x2);
                rw[x1] = w;
            }
        }
        const int X0 = m0 * B + x0;
        const bool s0 = X0 >= lo[0] && X0 < hi[0];
        uint32_t m2mask = 0, all = 0;
#pragma unroll
        for (int x2 = 0; x2 < B; ++x2) {
            const int X2 = m2 * B + x2;
            all |= 0xFFu << (8 * x2);
            if (X2 >= lo[2] && X2 < hi[2]) m2mask |= 0xFFu << (8 * x2);
        }
#pragma unroll
        for (int x1 = 0; x1 < B; ++x1) {
            const int X1 = m1 * B + x1;
            sm[x1] = (s0 || (X1 >= lo[1] && X1 < hi[1])) ? all : m2mask;
        }
    }
    uint32_t c4[4] = {0, 0, 0, 0};  // byte counters, four facies per word
#pragma unroll
    for (int ch = 0; ch < 16; ++ch)
        if (ch < g.F) {  // (uniform: F is a launch constant)
            int n = 0;
#pragma unroll
            for (int x1 = 0; x1 < B; ++x1) n += __popc(__vcmpeq4(rw[x1], 0x01010101u * ch) & sm[x1]);
            c4[ch >> 2] += static_cast<uint32_t>(n >> 3) << (8 * (ch & 3));
        }
#pragma unroll
    for (int q = 0; q < 4; ++q)
        if (4 * q < g.F) {
#pragma unroll
            for (int o = 1; o < B; o <<= 1) c4[q] += __shfl_xor_sync(0xffffffffu, c4[q], o);
        }
    if (x0 != 0 || i >= nm) return;
    int wv[16];
    int nlast = 0;
#pragma unroll
    for (int ch = 0; ch < 16; ++ch) {
        wv[ch] = (c4[ch >> 2] >> (8 * (ch & 3))) & 0xFF;
        if (ch == g.F - 1) nlast = wv[ch];
    }
    if (g.mode == 0) {  // int8x4
        uint32_t v = 0;
#pragma unroll
        for (int ch = 0; ch < 4; ++ch)
            if (ch < g.nscr) {
                const int w = g.F > 1 ? wv[ch] - nlast : 0;
                v |= (static_cast<uint32_t>(w) & 0xFFu) << (8 * ch);
            }
        if (tcrow > 0) {  // GEMM row: max(nscr, 1) channel bytes per window cell
            const int bpc = max(g.nscr, 1);
            int8_t* r8 = reinterpret_cast<int8_t*>(wout) + i * bpc;
#pragma unroll
            for (int ch = 0; ch < 4; ++ch)
                if (ch < bpc) r8[ch] = static_cast<int8_t>((v >> (8 * ch)) & 0xFFu);
        } else {
            wout[i] = static_cast<int32_t>(v);
        }
    } else {
#pragma unroll
        for (int ch = 0; ch < 16; ++ch)
            if (ch < g.nscr) wout[i * g.nscr + ch] = g.F > 1 ? wv[ch] - nlast : 0;
    }
}

// ----------------------------------------------------------- screen ------
struct Screen3Args {
    Geo3 g;
    const Job3* jobs;
    const Batch3* batches;
    int bt0;              // first batch of the wave
    int j0;               // first job of the wave (wbuf / xbuf rows are wave-relative)
    const int* mask_off;
    const int* mask_cells;
    const int32_t* tipk;  // packed TI block counts
    const int32_t* wbuf;  // [job in wave][wstride]
    int wstride;
    int P0, P1, P2, W1;   // box shape (P1 = 4 W1, P0 = 8 / W1, P2 = 8 NP)
    int nb[3];            // boxes per axis
    int box0, box1;       // this launch's box range (one shard)
    int bps;              // boxes per shard slot
    int shard;            // shard slot of box0
    int K;
    int nj;               // jobs in the wave
    unsigned long long* xbuf;  // [shard][nj][bps][K]
};

__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) {
    return a > b ? a : b;
}

__device__ __forceinline__ unsigned long long warp_max64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = umax64(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// The CCF of one box for JBT jobs (JBT >= the batch's job count): NP
// positions per thread strided by 8 along axis 2, JBT accumulators each; then
// each warp's top-K packed keys per job into wk[j][warp][K].
template <int MODE, int NP, int JBT>
__device__ __forceinline__ void screen_body(const Screen3Args& a, const Batch3& bt, const int32_t* region,
                                            const int32_t* moff, const int32_t* wsm, int nm, int RV, int R1,
                                            int R2p, int B0, int B1, int B2, int32_t* s3) {
    const Geo3& g = a.g;
    const int nch = MODE == 0 ? 1 : g.nscr;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t0 = warp / a.W1, t1 = (warp % a.W1) * 4 + (lane >> 3), l2 = lane & 7;
    const int base = (t0 * R1 + t1) * R2p + l2;
    int acc[NP][JBT];
#pragma unroll
    for (int k = 0; k < NP; ++k)
#pragma unroll
        for (int j = 0; j < JBT; ++j) acc[k][j] = 0;
    auto weights = [&](int row, int (&wv)[JBT]) {
        const int* w = wsm + row * JB;
        if constexpr (JBT == 8) {
            const int4 w0 = *reinterpret_cast<const int4*>(w), w1 = *reinterpret_cast<const int4*>(w + 4);
            wv[0] = w0.x; wv[1] = w0.y; wv[2] = w0.z; wv[3] = w0.w;
            wv[4] = w1.x; wv[5] = w1.y; wv[6] = w1.z; wv[7] = w1.w;
        } else if constexpr (JBT == 4) {
            const int4 w0 = *reinterpret_cast<const int4*>(w);
            wv[0] = w0.x; wv[1] = w0.y; wv[2] = w0.z; wv[3] = w0.w;
        } else if constexpr (JBT == 2) {
            const int2 w0 = *reinterpret_cast<const int2*>(w);
            wv[0] = w0.x; wv[1] = w0.y;
        } else {
            wv[0] = w[0];
        }
    };
#pragma unroll 2
    for (int i = 0; i < nm; ++i) {
        const int o = base + moff[i];
        if constexpr (MODE == 0) {
            int wv[JBT];
            weights(i, wv);
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                const int v = region[o + 8 * k];
#pragma unroll
                for (int j = 0; j < JBT; ++j) acc[k][j] = __dp4a(v, wv[j], acc[k][j]);
            }
        } else {
            for (int ch = 0; ch < nch; ++ch) {
                int wv[JBT];
                weights(i * nch + ch, wv);
#pragma unroll
                for (int k = 0; k < NP; ++k) {
                    const int v = region[ch * RV + o + 8 * k];
#pragma unroll
                    for (int j = 0; j < JBT; ++j) acc[k][j] += v * wv[j];
                }
            }
        }
    }
    // packed keys: exact score (biased) above the complemented position, so
    // the larger key is the better candidate (earlier position on ties)
    const int p0 = B0 + t0, p1 = B1 + t1;
    const bool row_ok = p0 < g.o[0] && p1 < g.o[1];
    __syncthreads();  // (the region is reused below as the per-warp key lists)
    unsigned long long* wk = reinterpret_cast<unsigned long long*>(s3);  // [JB][8 warps][K]
    const int K = a.K;
#pragma unroll
    for (int j = 0; j < JBT; ++j) {
        if (j >= bt.n) break;
        unsigned long long key[NP];
#pragma unroll
        for (int k = 0; k < NP; ++k) {
            const int p2 = B2 + l2 + 8 * k;
            key[k] = 0;
            if (row_ok && p2 < g.o[2]) {
                const uint32_t pos = static_cast<uint32_t>((p0 * g.o[1] + p1) * g.o[2] + p2);
                key[k] = (static_cast<unsigned long long>(static_cast<uint32_t>(acc[k][j]) ^ 0x80000000u) << 32) |
                         (0xFFFFFFFFu - pos);
            }
        }
        for (int r = 0; r < K; ++r) {
            unsigned long long m = 0;
#pragma unroll
            for (int k = 0; k < NP; ++k) m = umax64(m, key[k]);
            const unsigned long long wm = warp_max64(m);
#pragma unroll
            for (int k = 0; k < NP; ++k)
                if (key[k] == wm) key[k] = 0;  // keys are unique: one lane drops it
            if (lane == 0) wk[(j * 8 + warp) * K + r] = wm;
        }
    }
}

template <int MODE, int NP>
__global__ void __launch_bounds__(S3_THREADS) screen3d_kernel(Screen3Args a) {
    extern __shared__ __align__(16) int32_t s3[];
    pdl_trigger();
    const Geo3& g = a.g;
    const Batch3 bt = a.batches[a.bt0 + blockIdx.y];
    const int box = a.box0 + blockIdx.x;
    const int bx2 = box % a.nb[2], bx1 = (box / a.nb[2]) % a.nb[1], bx0 = box / (a.nb[2] * a.nb[1]);
    const int B0 = bx0 * a.P0, B1 = bx1 * a.P1, B2 = bx2 * a.P2;
    const int R0 = a.P0 + g.tc - 1, R1 = a.P1 + g.tc - 1, R2 = a.P2 + g.tc - 1;
    const int R2p = R2 + ((8 - R2 % 32) + 32) % 32;  // row pitch = 8 mod 32 (conflict-free rows)
    const int RV = R0 * R1 * R2p;                    // one channel's region
    const int nch = MODE == 0 ? 1 : g.nscr;
    const int m_lo = a.mask_off[bt.mask], nm = a.mask_off[bt.mask + 1] - m_lo;
    int32_t* region = s3;
    int32_t* moff = region + RV * nch;
    int32_t* wsm = moff + ((nm + 3) & ~3);  // [nm][nch][JB]
    const size_t ncell = static_cast<size_t>(g.c[0]) * g.c[1] * g.c[2];
    // TI block counts of the box's window region (independent of earlier kernels)
    for (int e = threadIdx.x; e < RV * nch; e += blockDim.x) {
        const int ch = e / RV, r = e - ch * RV;
        const int r2 = r % R2p, r1 = (r / R2p) % R1, r0 = r / (R2p * R1);
        const int q0 = B0 + r0, q1 = B1 + r1, q2 = B2 + r2;
        int32_t v = 0;
        if (r2 < R2 && q0 < g.c[0] && q1 < g.c[1] && q2 < g.c[2])
            v = a.tipk[ch * ncell + (static_cast<size_t>(q0) * g.c[1] + q1) * g.c[2] + q2];
        region[e] = v;
    }
    for (int i = threadIdx.x; i < nm; i += blockDim.x) {
        const int cell = a.mask_cells[m_lo + i];
        moff[i] = ((cell >> 16) * R1 + ((cell >> 8) & 0xFF)) * R2p + (cell & 0xFF);
    }
    pdl_wait();  // weights (prep3d) ready; the previous select has read xbuf
    for (int e = threadIdx.x; e < nm * nch * JB; e += blockDim.x) {
        const int jb = e % JB, ich = e / JB;
        wsm[e] = jb < bt.n ? a.wbuf[static_cast<size_t>(bt.j0 - a.j0 + jb) * a.wstride + ich] : 0;
    }
    __syncthreads();
#ifdef CCW_DEBUG3D
    if (threadIdx.x == 0 && blockIdx.x == 0) printf("screen bt j0 %d n %d mask %d nm %d w0 %x region0 %x P %d %d %d\n", bt.j0, bt.n, bt.mask, nm, wsm[0], region[0], a.P0, a.P1, a.P2);
#endif

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // the batch's job count picks the accumulator width (no MACs on empty slots)
    if (bt.n > 4)
        screen_body<MODE, NP, 8>(a, bt, region, moff, wsm, nm, RV, R1, R2p, B0, B1, B2, s3);
    else if (bt.n > 2)
        screen_body<MODE, NP, 4>(a, bt, region, moff, wsm, nm, RV, R1, R2p, B0, B1, B2, s3);
    else if (bt.n > 1)
        screen_body<MODE, NP, 2>(a, bt, region, moff, wsm, nm, RV, R1, R2p, B0, B1, B2, s3);
    else
        screen_body<MODE, NP, 1>(a, bt, region, moff, wsm, nm, RV, R1, R2p, B0, B1, B2, s3);
    __syncthreads();
    // warp j merges job j's 8 warp lists
    const unsigned long long* wk = reinterpret_cast<const unsigned long long*>(s3);
    const int K = a.K;
    if (warp < bt.n) {
        const int j = warp;
        const int n = 8 * K;
        unsigned long long c[(8 * KMAX3 + 31) / 32];
#pragma unroll
        for (int q = 0; q < (8 * KMAX3 + 31) / 32; ++q) {
            const int e = lane + 32 * q;
            c[q] = e < n ? wk[j * 8 * K + e] : 0;
        }
        unsigned long long* dst = a.xbuf + ((static_cast<size_t>(a.shard + (box - a.box0) / a.bps) * a.nj +
                                             (bt.j0 - a.j0 + j)) * a.bps + (box - a.box0) % a.bps) * K;
        for (int r = 0; r < K; ++r) {
            unsigned long long m = 0;
#pragma unroll
            for (int q = 0; q < (8 * KMAX3 + 31) / 32; ++q) m = umax64(m, c[q]);
            const unsigned long long wm = warp_max64(m);
#pragma unroll
            for (int q = 0; q < (8 * KMAX3 + 31) / 32; ++q)
                if (c[q] == wm) c[q] = 0;
            if (lane == 0) dst[r] = wm;
        }
    }
}

// ------------------------------------------- tcgen05 screen (mode 0) ------
// Where the block counts fit int8 (mode 0: B <= 4, <= 4 screen channels) the
// 3D CCF is the same implicit GEMM as the 2D screen (ccf_tc.cu): placements x
// window positions over K = tc^3 cells x 4 packed channel bytes.  The window
// matrix is an explicit im2col of the packed TI counts, built once per TI and
// coarse template size; the prep writes one packed weight word per window cell
// (zero off the job's overlap support, so the full-window product equals the
// masked sum of screen3d_kernel bit for bit).
__global__ void im2col3d_kernel(const int32_t* __restrict__ tipk, int c1, int c2, int o1, int o2, int tc,
                                int npos, int bpc, int kbytes, int8_t* __restrict__ X) {
    // bpc = screen channels (1..4): byte cell * bpc + ch of a position's row is
    // channel ch's count of window cell (m0, m1, m2), cell = (m0 tc + m1) tc + m2;
    // the row padding up to kbytes was zeroed by the caller
    const int tc3 = tc * tc * tc;
    const size_t total = static_cast<size_t>(npos) * tc3;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int pos = static_cast<int>(e / tc3), cell = static_cast<int>(e - static_cast<size_t>(pos) * tc3);
        const int m2 = cell % tc, m1 = (cell / tc) % tc, m0 = cell / (tc * tc);
        const int p2 = pos % o2, p1 = (pos / o2) % o1, p0 = pos / (o2 * o1);
        const uint32_t v = static_cast<uint32_t>(tipk[(static_cast<size_t>(p0 + m0) * c1 + p1 + m1) * c2 + p2 + m2]);
        int8_t* x = X + static_cast<size_t>(pos) * kbytes + cell * bpc;
        for (int ch = 0; ch < bpc; ++ch) x[ch] = static_cast<int8_t>((v >> (8 * ch)) & 0xFFu);
    }
}

// Counts up to 512 (J = 3: mode 1) as two int8 digits, x = 32 xh + xl: per
// (window cell, channel) the bytes (xh, xl), K = 2 nscr tc^3 bytes.  With the
// prep's three weight rows per job the exact score is
// 1024 row1 + 32 row2 + row3 (keys3d_digits_kernel).
__global__ void im2col3d_digits_kernel(const int32_t* __restrict__ tipk, size_t ncell, int c1, int c2, int o1,
                                       int o2, int tc, int nscr, int npos, int kbytes, int8_t* __restrict__ X) {
    const int per = tc * tc * tc * nscr;
    const size_t total = static_cast<size_t>(npos) * per;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int pos = static_cast<int>(e / per), k = static_cast<int>(e - static_cast<size_t>(pos) * per);
        const int ch = k % nscr, cell = k / nscr;
        const int m2 = cell % tc, m1 = (cell / tc) % tc, m0 = cell / (tc * tc);
        const int p2 = pos % o2, p1 = (pos / o2) % o1, p0 = pos / (o2 * o1);
        const int x = tipk[ch * ncell + (static_cast<size_t>(p0 + m0) * c1 + p1 + m1) * c2 + p2 + m2];
        *reinterpret_cast<uint16_t*>(X + static_cast<size_t>(pos) * kbytes + 2 * k) =
            static_cast<uint16_t>((x >> 5) | ((x & 31) << 8));
    }
}

// Per job and position chunk: the K best packed keys of the combined score
// 1024 row1 + 32 row2 + row3, as one "box" list of select3d's merge.
__global__ void __launch_bounds__(256) keys3d_digits_kernel(const int32_t* __restrict__ sc, int sld, int npos,
                                                            int K, unsigned long long* __restrict__ xbuf) {
    __shared__ unsigned long long red[8];
    pdl_trigger();
    pdl_wait();
    const int j = blockIdx.x, ns = gridDim.y, s = blockIdx.y, tid = threadIdx.x;
    const int32_t* r1 = sc + static_cast<size_t>(3 * j) * sld;
    const int32_t* r2 = r1 + sld;
    const int32_t* r3 = r2 + sld;
    const int chunk = (npos + ns - 1) / ns;
    const int p_lo = s * chunk, p_hi = min(npos, p_lo + chunk);
    unsigned long long prev = ~0ull;
    for (int r = 0; r < K; ++r) {
        unsigned long long m = 0;
        for (int p = p_lo + tid; p < p_hi; p += 256) {
            const int S = 1024 * r1[p] + 32 * r2[p] + r3[p];
            const unsigned long long key =
                (static_cast<unsigned long long>(static_cast<uint32_t>(S) ^ 0x80000000u) << 32) |
                (0xFFFFFFFFu - static_cast<uint32_t>(p));
            if (key < prev) m = umax64(m, key);
        }
        m = warp_max64(m);
        __syncthreads();
        if ((tid & 31) == 0) red[tid >> 5] = m;
        __syncthreads();
        m = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) m = umax64(m, red[w]);
        if (tid == 0) xbuf[(static_cast<size_t>(j) * ns + s) * K + r] = m;
        prev = m;
    }
}

// ----------------------------------------------------------- select ------
struct Select3Args {
    Geo3 g;
    const Job3* jobs;
    int j0, nj;
    const unsigned long long* xbuf;  // [S][nj][bps][K]
    int S, bps, nbox, K, Kp;
    // tcgen05 screen: exact score rows and their 128-position tile maxima
    // instead of the boxes' key lists (null: off)
    const int32_t* sc;  // [nj][sld]
    const int32_t* tm;  // [nj][tld]
    int sld, tld, npos;
    const int* hd_off;          // CSR per lattice cell (may be null)
    const uint32_t* hd_ent;     // (x0 << 20 | x1 << 10 | x2) local offset, facies in a second word
    const uint8_t* hd_fac;
    const uint8_t* ti;
    uint8_t* work;
    int32_t* chosen;            // [job][3]
};

__device__ __forceinline__ unsigned long long block_max64(unsigned long long v, unsigned long long* red) {
    v = warp_max64(v);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    unsigned long long m = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) m = umax64(m, red[w]);
    return m;
}

__device__ __forceinline__ int block_sum(int v, int* red) {
    v = __reduce_add_sync(0xffffffffu, v);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    int s = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += red[w];
    return s;
}

__device__ __forceinline__ unsigned long long key64(int score, uint32_t idx) {
    return (static_cast<unsigned long long>(static_cast<uint32_t>(score) ^ 0x80000000u) << 32) | (0xFFFFFFFFu - idx);
}

// The K best packed keys (score desc, position asc) of one score row of the
// tcgen05 screen.  Only tiles whose maximum reaches the K-th largest tile
// maximum can hold a top-K window: those tiles are listed, then K rounds of
// "largest key below the last" over the listed tiles' positions.
constexpr int TLCAP = 128;
__device__ void row_top_keys(const int32_t* __restrict__ sc, const int32_t* __restrict__ tm, int npos, int K,
                             unsigned long long* cands, unsigned long long* red, int* tl, int* ntl) {
    const int tid = threadIdx.x, nth = blockDim.x;
    const int nt = (npos + kTcTile - 1) / kTcTile;
    int thr = INT_MIN;
    if (nt > K) {
        unsigned long long prev = ~0ull, m = 0;
        for (int r = 0; r < K; ++r) {
            m = 0;
            for (int t = tid; t < nt; t += nth) {
                const unsigned long long key = key64(tm[t], static_cast<uint32_t>(t));
                if (key < prev) m = umax64(m, key);
            }
            m = block_max64(m, red);
            prev = m;
        }
        thr = static_cast<int>(static_cast<uint32_t>(m >> 32) ^ 0x80000000u);
        if (K == 1) {
            // the best window is in the first tile that holds the row maximum
            const int t = static_cast<int>(0xFFFFFFFFu - static_cast<uint32_t>(m & 0xFFFFFFFFull));
            unsigned long long b = 0;
            for (int p = t * kTcTile + tid; p < min(npos, (t + 1) * kTcTile); p += nth)
                b = umax64(b, key64(sc[p], static_cast<uint32_t>(p)));
            b = block_max64(b, red);
            if (tid == 0) cands[0] = b;
            return;
        }
    }
    if (tid == 0) *ntl = 0;
    __syncthreads();
    for (int t = tid; t < nt; t += nth)
        if (tm[t] >= thr) {
            const int q = atomicAdd(ntl, 1);
            if (q < TLCAP) tl[q] = t;
        }
    __syncthreads();
    const int n = *ntl;
    unsigned long long prev = ~0ull;
    for (int r = 0; r < K; ++r) {
        unsigned long long m = 0;
        auto tile = [&](int t) {
            for (int p = t * kTcTile + tid; p < min(npos, (t + 1) * kTcTile); p += nth) {
                const unsigned long long key = key64(sc[p], static_cast<uint32_t>(p));
                if (key < prev) m = umax64(m, key);
            }
        };
        if (n <= TLCAP) {
            for (int q = 0; q < n; ++q) tile(tl[q]);
        } else {  // a tie storm over many tiles: every qualifying tile, unlisted
            for (int t = 0; t < nt; ++t)
                if (tm[t] >= thr) tile(t);
        }
        m = block_max64(m, red);
        if (tid == 0) cands[r] = m;
        prev = m;
    }
}

__global__ void __launch_bounds__(128) select3d_kernel(Select3Args a) {
    __shared__ unsigned long long red[4];
    __shared__ int redi[4];
    __shared__ unsigned long long cands[KMAX3];
    __shared__ int fr_s[3];
    __shared__ int tl_s[TLCAP];
    __shared__ int ntl_s;
    pdl_trigger();
    pdl_wait();
    const Geo3& g = a.g;
    const int jw = blockIdx.x;
    const Job3 jb = a.jobs[a.j0 + jw];
    if (jb.pick == -2) {
        if (threadIdx.x < 3) fr_s[threadIdx.x] = jb.fr[threadIdx.x];
    } else {
        // top-K of the boxes' lists: K rounds of "largest key below the last"
        const int per = a.bps * a.K;
        const int total = a.S * per;
        unsigned long long prev = ~0ull;
        if (a.sc)  // (tcgen05 screen: straight from the score row)
            row_top_keys(a.sc + static_cast<size_t>(jw) * a.sld, a.tm + static_cast<size_t>(jw) * a.tld, a.npos,
                         a.Kp, cands, red, tl_s, &ntl_s);
        for (int r = 0; r < (a.sc ? 0 : a.Kp); ++r) {
            unsigned long long m = 0;
            for (int e = threadIdx.x; e < total; e += blockDim.x) {
                const int s = e / per, rem = e - s * per;
                if (s * a.bps + rem / a.K >= a.nbox) continue;
                const unsigned long long v = a.xbuf[(static_cast<size_t>(s) * a.nj + jw) * per + rem];
                if (v < prev) m = umax64(m, v);
            }
            m = block_max64(m, red);
            if (threadIdx.x == 0) cands[r] = m;
            prev = m;
        }
        __syncthreads();
#ifdef CCW_DEBUG3D
        if (threadIdx.x == 0) printf("select job %d cands %llx %llx total %d per %d nbox %d\n", a.j0 + jw, cands[0], a.Kp > 1 ? cands[1] : 0ull, total, per, a.nbox);
#endif
        int pick = jb.pick;
        if (pick < 0) {  // select_conditional (matcher.hpp:222-241)
            const int h0 = a.hd_off[jb.lat], nh = a.hd_off[jb.lat + 1] - h0;
            int best = 0, best_m = nh + 1;
            for (int ci = 0; ci < a.Kp; ++ci) {
                const uint32_t pos = 0xFFFFFFFFu - static_cast<uint32_t>(cands[ci] & 0xFFFFFFFFull);
                const int q2 = pos % g.o[2], q1 = (pos / g.o[2]) % g.o[1], q0 = pos / (g.o[2] * g.o[1]);
                int mm = 0;
                for (int e = threadIdx.x; e < nh; e += blockDim.x) {
                    const uint32_t off = a.hd_ent[h0 + e];
                    const int x0 = off >> 20, x1 = (off >> 10) & 1023, x2 = off & 1023;
                    const size_t t = (static_cast<size_t>(q0 * g.B + x0) * g.ti[1] + q1 * g.B + x1) * g.ti[2] +
                                     q2 * g.B + x2;
                    mm += a.ti[t] != a.hd_fac[h0 + e];
                }
                mm = block_sum(mm, redi);
                if (mm == 0) {
                    best = ci;
                    break;
                }
                if (mm < best_m) {
                    best_m = mm;
                    best = ci;
                }
            }
            pick = best;
        }
        if (threadIdx.x == 0) {
            const uint32_t pos = 0xFFFFFFFFu - static_cast<uint32_t>(cands[pick] & 0xFFFFFFFFull);
            fr_s[2] = pos % g.o[2] * g.B;
            fr_s[1] = (pos / g.o[2]) % g.o[1] * g.B;
            fr_s[0] = pos / (g.o[2] * g.o[1]) * g.B;
        }
    }
    __syncthreads();
    const int f0 = fr_s[0], f1 = fr_s[1], f2 = fr_s[2];
    if (threadIdx.x < 3 && blockIdx.y == 0) a.chosen[3 * (a.j0 + jw) + threadIdx.x] = fr_s[threadIdx.x];
    // crop + paste_into (grid.hpp:172-230): T^3 cells, 4-byte words where
    // aligned; the gridDim.y CTAs of a job (each made the same pick) paste
    // one slab of x0 each
    uint8_t* wk = a.work + static_cast<size_t>(jb.real) * g.W[0] * g.W[1] * g.W[2];
    const int T = g.T;
    const int xa = static_cast<int>(static_cast<int64_t>(T) * blockIdx.y / gridDim.y);
    const int xb = static_cast<int>(static_cast<int64_t>(T) * (blockIdx.y + 1) / gridDim.y);
    const size_t rows = static_cast<size_t>(xb - xa) * T;
    if (g.aligned4) {  // every row start is 4-byte aligned on both sides
        const int T4 = T >> 2;
        for (size_t e = threadIdx.x; e < rows * T4; e += blockDim.x) {
            const int x2 = static_cast<int>(e % T4) * 4;
            const size_t rr = e / T4;
            const int x1 = static_cast<int>(rr % T), x0 = xa + static_cast<int>(rr / T);
            *reinterpret_cast<uint32_t*>(wk + (static_cast<size_t>(jb.P[0] + x0) * g.W[1] + jb.P[1] + x1) * g.W[2] +
                                         jb.P[2] + x2) =
                *reinterpret_cast<const uint32_t*>(a.ti + (static_cast<size_t>(f0 + x0) * g.ti[1] + f1 + x1) * g.ti[2] +
                                                   f2 + x2);
        }
        return;
    }
    for (size_t e = threadIdx.x; e < rows * T; e += blockDim.x) {
        const int x2 = static_cast<int>(e % T);
        const size_t rr = e / T;
        const int x1 = static_cast<int>(rr % T), x0 = xa + static_cast<int>(rr / T);
        wk[(static_cast<size_t>(jb.P[0] + x0) * g.W[1] + jb.P[1] + x1) * g.W[2] + jb.P[2] + x2] =
            a.ti[(static_cast<size_t>(f0 + x0) * g.ti[1] + f1 + x1) * g.ti[2] + f2 + x2];
    }
}

// --------------------------------------------------------- finalize ------
__global__ void finalize3d_kernel(const uint8_t* __restrict__ work, int W0, int W1, int W2, int s0, int s1,
                                  int s2, uint8_t* __restrict__ out) {
    pdl_wait();
    const int r = blockIdx.y;
    const size_t n = static_cast<size_t>(s0) * s1 * s2;
    const uint8_t* wk = work + static_cast<size_t>(r) * W0 * W1 * W2;
    uint8_t* o = out + static_cast<size_t>(r) * n;
    if (s2 % 4 == 0 && W2 % 4 == 0 && (reinterpret_cast<uintptr_t>(out) & 3) == 0 &&
        (reinterpret_cast<uintptr_t>(work) & 3) == 0) {  // 4-byte words: every row start is aligned on both sides
        const int q2 = s2 >> 2;
        for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < n / 4;
             e += static_cast<size_t>(gridDim.x) * blockDim.x) {
            const int x2 = static_cast<int>(e % q2) * 4;
            const size_t rr = e / q2;
            const int x1 = static_cast<int>(rr % s1), x0 = static_cast<int>(rr / s1);
            *reinterpret_cast<uint32_t*>(o + 4 * e) =
                *reinterpret_cast<const uint32_t*>(wk + (static_cast<size_t>(x0) * W1 + x1) * W2 + x2);
        }
        return;
    }
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int x2 = static_cast<int>(e % s2);
        const size_t rr = e / s2;
        const int x1 = static_cast<int>(rr % s1), x0 = static_cast<int>(rr / s1);
        o[e] = wk[(static_cast<size_t>(x0) * W1 + x1) * W2 + x2];
    }
}

// Result codes packed `bits` per cell (8 / bits cells per byte, first cell in
// the low bits) for the device -> host copy; the host unpacks (unpack_cells).
template <int BITS>
__global__ void pack3d_kernel(const uint8_t* __restrict__ in, size_t n, uint8_t* __restrict__ out) {
    constexpr int CPB = 8 / BITS;
    const size_t nb = (n + CPB - 1) / CPB;
    for (size_t b = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; b < nb;
         b += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t c0 = b * CPB;
        uint32_t v = 0;
        if (c0 + CPB <= n && (reinterpret_cast<uintptr_t>(in) & 7) == 0) {
            uint64_t w;  // CPB aligned cells in one load
            if constexpr (CPB == 8) w = *reinterpret_cast<const uint64_t*>(in + c0);
            else if constexpr (CPB == 4) w = *reinterpret_cast<const uint32_t*>(in + c0);
            else w = *reinterpret_cast<const uint16_t*>(in + c0);
#pragma unroll
            for (int c = 0; c < CPB; ++c) v |= static_cast<uint32_t>((w >> (8 * c)) & ((1u << BITS) - 1)) << (c * BITS);
        } else {
            for (int c = 0; c < CPB && c0 + c < n; ++c) v |= static_cast<uint32_t>(in[c0 + c] & ((1u << BITS) - 1)) << (c * BITS);
        }
        out[b] = static_cast<uint8_t>(v);
    }
}

// hard-data overwrite with the pre-overwrite mismatch count (simulator.hpp:506-513)
__global__ void hd3d_kernel(const int32_t* __restrict__ hd, int n_hd, int s0, int s1, int s2, uint8_t* out,
                            int* mism) {
    const int r = blockIdx.y;
    const size_t n = static_cast<size_t>(s0) * s1 * s2;
    int local = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_hd; i += gridDim.x * blockDim.x) {
        const int* d = hd + 4 * i;
        uint8_t* c = out + r * n + (static_cast<size_t>(d[0]) * s1 + d[1]) * s2 + d[2];
        local += *c != d[3];
        *c = static_cast<uint8_t>(d[3]);
    }
    local = __reduce_add_sync(0xffffffffu, local);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(&mism[r], local);
}

int padded_extent3(int sg, int t, int stride) {  // simulator.hpp:125-131
    if (sg == t) return t;
    return t + (sg - t + stride - 1) / stride * stride;
}

const int kOrders[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};

}  // namespace

// ------------------------------------------------------------ host -------

void build_pyramid3d(ccw_ti3d* ti, cudaStream_t st) {
    const size_t nc = static_cast<size_t>(ti->c[0]) * ti->c[1] * ti->c[2];
    const int nb = static_cast<int>(std::min<size_t>((nc + 255) / 256, 4096));
    pyramid3d_kernel<<<std::max(nb, 1), 256, 0, st>>>(ti->d_codes, ti->d[0], ti->d[1], ti->d[2], ti->c[0], ti->c[1],
                                                     ti->c[2], 1 << ti->J, ti->nscr, ti->mode,
                                                     ti->d_pk);
    CCW_CUDA(cudaGetLastError());
}

// im2col of the packed TI counts for the tcgen05 screen (cached on the TI):
// [npos][kbytes] int8, bpc channel bytes per window cell.
static const int8_t* ti3d_im2col(ccw_ti3d* ti, const Geo3& g, int npos, int bpc, int kbytes, cudaStream_t st) {
    auto it = ti->im2col.find(g.tc);
    if (it != ti->im2col.end()) return it->second;
    const size_t bytes = static_cast<size_t>(npos) * kbytes;
    int8_t* X = static_cast<int8_t*>(cache_alloc(ti->device, bytes));
    CCW_CUDA(cudaMemsetAsync(X, 0, bytes, st));
    const size_t total = static_cast<size_t>(npos) * g.tc * g.tc * g.tc;
    const unsigned nb = static_cast<unsigned>(std::min<size_t>((total + 255) / 256, 148 * 32));
    im2col3d_kernel<<<std::max(nb, 1u), 256, 0, st>>>(ti->d_pk, g.c[1], g.c[2], g.o[1], g.o[2], g.tc, npos, bpc, kbytes, X);
    CCW_CUDA(cudaGetLastError());
    ti->im2col[g.tc] = X;
    return X;
}

void run_simulation3d(ccw_ctx* ctx, ccw_ti3d* ti, const ccw_sim3d_config& cfg, const uint64_t* seeds, int n_real,
                      const int32_t* hd, int n_hd, uint8_t* d_out, uint8_t* h_out, ccw_diag3d* diag,
                      int32_t* trace, int trace_cap) {
    const auto wall0 = std::chrono::steady_clock::now();
    cudaStream_t st = ctx->stream;
    Geo3 g{};
    g.J = cfg.dwt_level;
    g.B = 1 << g.J;
    g.T = cfg.template_size;
    g.OV = cfg.overlap;
    g.tc = g.T >> g.J;
    g.nscr = ti->nscr;
    g.F = ti->F;
    g.any_support = cfg.any_support;
    g.mode = ti->mode;
    const int stride = g.T - g.OV;
    for (int a = 0; a < 3; ++a) {
        g.c[a] = ti->c[a];
        g.o[a] = g.c[a] - g.tc + 1;
        g.ti[a] = ti->d[a];
        g.sg[a] = cfg.sg[a];
        g.W[a] = padded_extent3(cfg.sg[a], g.T, stride);
    }
    g.aligned4 = (g.W[2] % 4 == 0 && g.ti[2] % 4 == 0 && stride % 4 == 0 && g.B % 4 == 0 && g.T % 4 == 0) ? 1 : 0;
    const int64_t npos64 = static_cast<int64_t>(g.o[0]) * g.o[1] * g.o[2];
    if (npos64 >= (int64_t(1) << 31)) throw Fail(CCW_ERR_CONFIG, "3D: too many TI window positions");
    const int npos = static_cast<int>(npos64);
    const int Kp = static_cast<int>(std::min<int64_t>(cfg.candidates, npos));
    if (Kp > KMAX3) throw Fail(CCW_ERR_CONFIG, "candidates: the 3D path supports at most 16 candidates");
    if (g.tc > 255 || g.T >= 1024) throw Fail(CCW_ERR_CONFIG, "3D: template too large");
    // exactness of the int32 screen: |S'| <= mask * B^3 * B^3 <= T^3 * B^3
    if (static_cast<double>(g.T) * g.T * g.T * g.B * g.B * g.B >= 2147483647.0)
        throw Fail(CCW_ERR_CONFIG, "3D: template^3 * block^3 exceeds the exact int32 screen range");
    const int n_lat[3] = {(g.W[0] - g.T) / stride + 1, (g.W[1] - g.T) / stride + 1, (g.W[2] - g.T) / stride + 1};
    const int reach = (g.T + stride - 1) / stride - 1;
    const int km = reach + 1;

    // ---- host schedule: plans, draws (the whole mt19937_64 sequence is a
    // function of the geometry: conditional placements draw nothing) ----
    const size_t nlat = static_cast<size_t>(n_lat[0]) * n_lat[1] * n_lat[2];
    std::vector<int32_t> hd_off(nlat + 1, 0);
    std::vector<uint32_t> hd_ent;
    std::vector<uint8_t> hd_fac;
    if (hd && n_hd > 0) {
        auto each = [&](int i, auto&& fn) {
            const int* d = hd + 4 * i;
            int lo[3], hi[3];
            for (int a = 0; a < 3; ++a) {
                lo[a] = std::max(0, (d[a] - g.T + 1 + stride - 1) / stride);
                hi[a] = std::min(n_lat[a] - 1, d[a] / stride);
            }
            for (int q0 = lo[0]; q0 <= hi[0]; ++q0)
                for (int q1 = lo[1]; q1 <= hi[1]; ++q1)
                    for (int q2 = lo[2]; q2 <= hi[2]; ++q2) {
                        const int q[3] = {q0, q1, q2};
                        bool in = true;
                        for (int a = 0; a < 3; ++a) in &= d[a] >= q[a] * stride && d[a] < q[a] * stride + g.T;
                        if (in)
                            fn((static_cast<size_t>(q0) * n_lat[1] + q1) * n_lat[2] + q2, d[0] - q0 * stride,
                               d[1] - q1 * stride, d[2] - q2 * stride, d[3]);
                    }
        };
        for (int i = 0; i < n_hd; ++i) each(i, [&](size_t q, int, int, int, int) { ++hd_off[q + 1]; });
        for (size_t q = 0; q < nlat; ++q) hd_off[q + 1] += hd_off[q];
        hd_ent.resize(hd_off[nlat]);
        hd_fac.resize(hd_off[nlat]);
        std::vector<int32_t> fill(hd_off.begin(), hd_off.end() - 1);
        for (int i = 0; i < n_hd; ++i)
            each(i, [&](size_t q, int x0, int x1, int x2, int f) {
                hd_ent[fill[q]] = (static_cast<uint32_t>(x0) << 20) | (static_cast<uint32_t>(x1) << 10) |
                                  static_cast<uint32_t>(x2);
                hd_fac[fill[q]++] = static_cast<uint8_t>(f);
            });
    }
    struct Pl {
        int wave, mask;
        Job3 j;
    };
    std::vector<Pl> pls;
    std::vector<int> corners(n_real), orders(n_real), counts(n_real);
    int max_key = 0;
    std::vector<char> mask_used(64, 0);
    for (int r = 0; r < n_real; ++r) {
        std::mt19937_64 rng(seeds[r]);
        const int corner = static_cast<int>(bounded(rng, 8));
        const int order = static_cast<int>(bounded(rng, 6));
        corners[r] = corner;
        orders[r] = order;
        const int* ord = kOrders[order];
        const int n0 = n_lat[ord[0]], n1 = n_lat[ord[1]], n2 = n_lat[ord[2]];
        counts[r] = n0 * n1 * n2;
        int place = 0;
        for (int io = 0; io < n0; ++io)
            for (int im = 0; im < n1; ++im)
                for (int ii = 0; ii < n2; ++ii, ++place) {
                    int idx[3];
                    idx[ord[0]] = io;
                    idx[ord[1]] = im;
                    idx[ord[2]] = ii;
                    Pl p{};
                    p.j.real = r;
                    p.j.place = place;
                    int sh = 0, lat[3];
                    for (int a = 0; a < 3; ++a) {
                        const bool asc = !((corner >> a) & 1);
                        lat[a] = asc ? idx[a] : n_lat[a] - 1 - idx[a];
                        p.j.P[a] = lat[a] * stride;
                        if (idx[a] > 0) sh |= 1 << a;
                    }
                    p.j.lat = static_cast<int>((static_cast<size_t>(lat[0]) * n_lat[1] + lat[1]) * n_lat[2] + lat[2]);
                    p.j.mask = corner * 8 + sh;
                    p.mask = p.j.mask;
                    p.wave = km * km * io + km * im + ii;
                    max_key = std::max(max_key, p.wave);
                    if (sh == 0) {
                        p.j.pick = -2;
                        for (int a = 0; a < 3; ++a)
                            p.j.fr[a] = static_cast<int>(bounded(rng, static_cast<uint64_t>((ti->c[a] * g.B - g.T) / g.B + 1))) * g.B;
                    } else {
                        const bool cond = !hd_off.empty() && hd_off[p.j.lat + 1] > hd_off[p.j.lat];
                        p.j.pick = cond ? -1 : static_cast<int>(bounded(rng, static_cast<uint64_t>(Kp)));
                    }
                    pls.push_back(p);
                }
    }
    // (wave, corner, shape) order: a batch holds up to JB jobs of one corner,
    // screened against the union of their overlap masks (a job's weights are
    // zero on the cells outside its own overlap)
    std::stable_sort(pls.begin(), pls.end(), [](const Pl& x, const Pl& y) {
        return x.wave != y.wave ? x.wave < y.wave : x.mask < y.mask;
    });
    const size_t njobs = pls.size();
    std::vector<Job3> jobs(njobs);
    std::vector<Batch3> batches;
    std::vector<int> wave_j0(max_key + 2, 0), wave_b0(max_key + 2, 0);
    {
        size_t k = 0;
        for (int w = 0; w <= max_key; ++w) {
            wave_j0[w] = static_cast<int>(k);
            wave_b0[w] = static_cast<int>(batches.size());
            while (k < njobs && pls[k].wave == w) {
                size_t e = k;
                while (e < njobs && pls[e].wave == w && (pls[e].mask >> 3) == (pls[k].mask >> 3) && e - k < JB) ++e;
                int bm = pls[k].mask;
                for (size_t q = k; q < e; ++q) bm |= pls[q].mask & 7;
                for (size_t q = k; q < e; ++q) pls[q].j.bmask = bm;
                if (pls[k].j.pick != -2) {
                    batches.push_back({static_cast<int>(k), static_cast<int>(e - k), bm, 0});
                    mask_used[bm] = 1;
                }
                k = e;
            }
        }
        wave_j0[max_key + 1] = static_cast<int>(njobs);
        wave_b0[max_key + 1] = static_cast<int>(batches.size());
        for (size_t i = 0; i < njobs; ++i) jobs[i] = pls[i].j;
    }
    // mask cell lists (row-major coarse cells of the block-level mask)
    std::vector<int> mask_off(65, 0), mask_cells;
    int max_nm = 0;
    for (int id = 0; id < 64; ++id) {
        mask_off[id] = static_cast<int>(mask_cells.size());
        if (mask_used[id]) {
            const int corner = id >> 3, sh = id & 7;
            const int tc = g.tc, B = g.B;
            for (int m0 = 0; m0 < tc; ++m0)
                for (int m1 = 0; m1 < tc; ++m1)
                    for (int m2 = 0; m2 < tc; ++m2) {
                        const int m[3] = {m0, m1, m2};
                        bool any = false;
                        for (int a = 0; a < 3; ++a)
                            if ((sh >> a) & 1) {
                                const bool asc = !((corner >> a) & 1);
                                // block [m*B, m*B+B) touches the slab [0, OV) / [T-OV, T)
                                any |= asc ? m[a] * B < g.OV : m[a] * B + B > g.T - g.OV;
                            }
                        if (any) mask_cells.push_back((m0 << 16) | (m1 << 8) | m2);
                    }
        }
        max_nm = std::max(max_nm, static_cast<int>(mask_cells.size()) - mask_off[id]);
    }
    mask_off[64] = static_cast<int>(mask_cells.size());
    // waves -> batches of jobs sharing one mask
    int max_wave = 1;
    for (int w = 0; w <= max_key; ++w) max_wave = std::max(max_wave, wave_j0[w + 1] - wave_j0[w]);

    // ---- box shape: P2 = 8 NP along axis 2, P1 = 4 W1, P0 = 8 / W1 ----
    int best_np = 2, best_w1 = 2;
    double best_v = 1e300;
    for (int np : {4, 2, 1})
        for (int w1 : {1, 2, 4, 8}) {
            const int P[3] = {8 / w1, 4 * w1, 8 * np};
            double v = 1;
            for (int a = 0; a < 3; ++a) v *= static_cast<double>((g.o[a] + P[a] - 1) / P[a]) * P[a];
            v *= (np == 1 ? 1.25 : 1.0) + 0.02 * (4 - np);  // NP = 1 is load-bound; more positions per thread on ties
            if (v < best_v) {
                best_v = v;
                best_np = np;
                best_w1 = w1;
            }
        }
    const int P0 = 8 / best_w1, P1 = 4 * best_w1, P2 = 8 * best_np;
    const int nb[3] = {(g.o[0] + P0 - 1) / P0, (g.o[1] + P1 - 1) / P1, (g.o[2] + P2 - 1) / P2};
    const int nbox = nb[0] * nb[1] * nb[2];
    const int mode = ti->mode;
    const int nch = mode == 0 ? 1 : g.nscr;
    const int R0 = P0 + g.tc - 1, R1 = P1 + g.tc - 1, R2 = P2 + g.tc - 1;
    const int R2p = R2 + ((8 - R2 % 32) + 32) % 32;
    const size_t smem = sizeof(int32_t) * (static_cast<size_t>(R0) * R1 * R2p * nch + ((max_nm + 3) & ~3) +
                                           static_cast<size_t>(max_nm) * nch * JB);
    const size_t smem_keys = sizeof(unsigned long long) * JB * 8 * KMAX3;
    const size_t smem_tot = std::max(smem, smem_keys);
    if (smem_tot > 227 * 1024) throw Fail(CCW_ERR_CONFIG, "3D: screen tile exceeds the shared-memory budget");

    // ---- position shards (ccw_ctx_set_position_shards) ----
    const int S_virt = ctx->shard_virtual, S_ranks = ctx->shard_nranks, S = S_virt * S_ranks;
    if (nbox < S) throw Fail(CCW_ERR_CONFIG, "position shards: more shards than 3D screen boxes");
    const int bps = (nbox + S - 1) / S;
    // ---- tcgen05 screen (option tc3d): int8 block counts, unsharded ----
    const int tc3 = g.tc * g.tc * g.tc;
    const int bpc = std::max(g.nscr, 1);                  // channel bytes per window cell
    const int kbytes = ((tc3 * bpc + 127) / 128) * 128;  // K, whole 128-byte stages
    const int sld = (npos + 3) & ~3;
    const int tld = tc_tiles(npos);
    const bool use_tc = ctx->opt.tc3d && mode == 0 && S == 1 && !ctx->nccl_comm && Kp >= 1 &&
                        static_cast<size_t>(npos) * kbytes <= (size_t(4) << 30) &&
                        static_cast<size_t>(max_wave) * sld * 4 <= (size_t(2) << 30);
    // ... and 9-bit counts (mode 1 at B = 8: config 4; B <= 4 with more than 4
    // screen channels keeps the CUDA-core screen) as two int8 digits,
    // three GEMM rows per job (im2col3d_digits_kernel)
    const int kdig = ((2 * g.nscr * tc3 + 127) / 128) * 128;  // K bytes
    const int nsplit = 32;                                     // position chunks per job (keys3d_digits_kernel)
    const bool use_dig = ctx->opt.tc3d && mode == 1 && g.B == 8 && S == 1 && !ctx->nccl_comm &&
                         Kp >= 1 && static_cast<size_t>(npos) * kdig <= (size_t(4) << 30) &&
                         static_cast<size_t>(max_wave) * 3 * sld * 4 <= (size_t(2) << 30);

    const bool host_t = debug_env("CCW_HOSTT") != nullptr;
    auto host_ms = [&]() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count(); };
    const double t_plan = host_t ? host_ms() : 0.0;
    // ---- device buffers ----
    const size_t wvol = static_cast<size_t>(g.W[0]) * g.W[1] * g.W[2];
    uint8_t* d_work = ctx->work.as<uint8_t>(wvol * n_real);
    CCW_CUDA(cudaMemsetAsync(d_work, 0, wvol * n_real, st));
    Job3* d_jobs = reinterpret_cast<Job3*>(ctx->jobs.get(sizeof(Job3) * njobs + 16));
    CCW_CUDA(cudaMemcpyAsync(d_jobs, jobs.data(), sizeof(Job3) * njobs, cudaMemcpyHostToDevice, st));
    Batch3* d_bt = reinterpret_cast<Batch3*>(ctx->ops_a.get(sizeof(Batch3) * std::max<size_t>(1, batches.size())));
    if (!batches.empty())
        CCW_CUDA(cudaMemcpyAsync(d_bt, batches.data(), sizeof(Batch3) * batches.size(), cudaMemcpyHostToDevice, st));
    int* d_moff = reinterpret_cast<int*>(ctx->ops_b.get(sizeof(int) * (65 + mask_cells.size() + 1)));
    int* d_mcells = d_moff + 65;
    CCW_CUDA(cudaMemcpyAsync(d_moff, mask_off.data(), sizeof(int) * 65, cudaMemcpyHostToDevice, st));
    if (!mask_cells.empty())
        CCW_CUDA(cudaMemcpyAsync(d_mcells, mask_cells.data(), sizeof(int) * mask_cells.size(), cudaMemcpyHostToDevice,
                                 st));
    const int wstride = std::max(1, max_nm * nch);
    int32_t* d_w = ctx->wts.as<int32_t>(static_cast<size_t>(max_wave) * wstride);
    unsigned long long* d_x =
        ctx->xrec.as<unsigned long long>(static_cast<size_t>(S) * max_wave * bps * std::max(Kp, 1));
    int32_t* d_chosen = ctx->chosen.as<int32_t>(3 * njobs);
    int* d_hdoff = nullptr;
    uint32_t* d_hdent = nullptr;
    uint8_t* d_hdfac = nullptr;
    int32_t* d_hd = nullptr;
    if (hd && n_hd > 0) {
        d_hdoff = ctx->hdoff.as<int32_t>(hd_off.size());
        CCW_CUDA(cudaMemcpyAsync(d_hdoff, hd_off.data(), sizeof(int32_t) * hd_off.size(), cudaMemcpyHostToDevice, st));
        d_hdent = ctx->hdent.as<uint32_t>(std::max<size_t>(1, hd_ent.size()) * 2);
        d_hdfac = reinterpret_cast<uint8_t*>(d_hdent + std::max<size_t>(1, hd_ent.size()));
        if (!hd_ent.empty()) {
            CCW_CUDA(cudaMemcpyAsync(d_hdent, hd_ent.data(), sizeof(uint32_t) * hd_ent.size(), cudaMemcpyHostToDevice,
                                     st));
            CCW_CUDA(cudaMemcpyAsync(d_hdfac, hd_fac.data(), hd_fac.size(), cudaMemcpyHostToDevice, st));
        }
        d_hd = reinterpret_cast<int32_t*>(ctx->hd.get(sizeof(int32_t) * 4 * n_hd));
        CCW_CUDA(cudaMemcpyAsync(d_hd, hd, sizeof(int32_t) * 4 * n_hd, cudaMemcpyHostToDevice, st));
    }
    int* d_mism = ctx->mism.as<int>(n_real);
    CCW_CUDA(cudaMemsetAsync(d_mism, 0, sizeof(int) * n_real, st));
    const size_t sgvol = static_cast<size_t>(cfg.sg[0]) * cfg.sg[1] * cfg.sg[2];
    uint8_t* fin = d_out ? d_out : ctx->out.as<uint8_t>(sgvol * n_real);

    TcPlan tcplan{};
    int32_t* d_w8 = nullptr;
    int32_t* d_sc = nullptr;
    int32_t* d_tm = nullptr;
    if (use_tc) {
        const int maxj = ((max_wave + 127) / 128) * 128;
        d_w8 = ctx->tc3_w.as<int32_t>(static_cast<size_t>(maxj) * kbytes / 4);
        CCW_CUDA(cudaMemsetAsync(d_w8, 0, static_cast<size_t>(maxj) * kbytes, st));  // (K padding stays zero)
        d_sc = ctx->tc3_sc.as<int32_t>(static_cast<size_t>(max_wave) * sld);
        d_tm = ctx->tc3_tm.as<int32_t>(static_cast<size_t>(max_wave) * tld);
        const int8_t* X = ti3d_im2col(ti, g, npos, bpc, kbytes, st);
        tcplan = plan_ccf_tc(reinterpret_cast<const int8_t*>(d_w8), maxj, X, npos, kbytes);
    }
    if (use_dig) {
        const int maxj = ((3 * max_wave + 127) / 128) * 128;
        d_w8 = ctx->tc3_w.as<int32_t>(static_cast<size_t>(maxj) * kdig / 4);
        CCW_CUDA(cudaMemsetAsync(d_w8, 0, static_cast<size_t>(maxj) * kdig, st));  // (K padding stays zero)
        d_sc = ctx->tc3_sc.as<int32_t>(static_cast<size_t>(3 * max_wave) * sld);
        d_tm = ctx->tc3_tm.as<int32_t>(static_cast<size_t>(3 * max_wave) * tld);
        auto it = ti->im2col.find(-g.tc);  // (digit layout: keyed by -tc)
        int8_t* X = it != ti->im2col.end() ? it->second : nullptr;
        if (!X) {
            const size_t bytes = static_cast<size_t>(npos) * kdig;
            X = static_cast<int8_t*>(cache_alloc(ti->device, bytes));
            CCW_CUDA(cudaMemsetAsync(X, 0, bytes, st));
            const size_t total = static_cast<size_t>(npos) * tc3 * g.nscr;
            im2col3d_digits_kernel<<<static_cast<unsigned>(std::min<size_t>((total + 255) / 256, 148 * 32)), 256, 0, st>>>(
                ti->d_pk, static_cast<size_t>(g.c[0]) * g.c[1] * g.c[2], g.c[1], g.c[2], g.o[1], g.o[2], g.tc, g.nscr,
                npos, kdig, X);
            CCW_CUDA(cudaGetLastError());
            ti->im2col[-g.tc] = X;
        }
        tcplan = plan_ccf_tc(reinterpret_cast<const int8_t*>(d_w8), maxj, X, npos, kdig);
        d_x = ctx->xrec.as<unsigned long long>(
            std::max(static_cast<size_t>(S) * max_wave * bps, static_cast<size_t>(max_wave) * nsplit) * std::max(Kp, 1));
    }
    void (*screen)(Screen3Args) = nullptr;
    if (mode == 0)
        screen = best_np == 4 ? screen3d_kernel<0, 4> : best_np == 2 ? screen3d_kernel<0, 2> : screen3d_kernel<0, 1>;
    else
        screen = best_np == 4 ? screen3d_kernel<1, 4> : best_np == 2 ? screen3d_kernel<1, 2> : screen3d_kernel<1, 1>;
    CCW_CUDA(cudaFuncSetAttribute(screen, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_tot)));

    Screen3Args sa{};
    sa.g = g;
    sa.jobs = d_jobs;
    sa.batches = d_bt;
    sa.mask_off = d_moff;
    sa.mask_cells = d_mcells;
    sa.tipk = ti->d_pk;
    sa.wbuf = d_w;
    sa.wstride = wstride;
    sa.P0 = P0;
    sa.P1 = P1;
    sa.P2 = P2;
    sa.W1 = best_w1;
    for (int a = 0; a < 3; ++a) sa.nb[a] = nb[a];
    sa.bps = bps;
    sa.K = std::max(Kp, 1);
    sa.xbuf = d_x;
    Select3Args se{};
    se.g = g;
    se.jobs = d_jobs;
    se.xbuf = d_x;
    se.S = S;
    se.bps = bps;
    se.nbox = nbox;
    se.K = std::max(Kp, 1);
    se.Kp = Kp;
    se.hd_off = d_hdoff;
    se.hd_ent = d_hdent;
    se.hd_fac = d_hdfac;
    se.ti = ti->d_codes;
    se.work = d_work;
    se.chosen = d_chosen;

    cudaEvent_t ev0, ev1;
    CCW_CUDA(cudaEventCreate(&ev0));
    CCW_CUDA(cudaEventCreate(&ev1));
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ccf_ev;
    CCW_CUDA(cudaEventRecord(ev0, st));
    const double t_ev0 = host_t ? host_ms() : 0.0;
    int64_t launches = 0, ccf_launches = 0;
    double ccf_flop = 0;
    for (int w = 0; w <= max_key; ++w) {
        const int j0 = wave_j0[w], nj = wave_j0[w + 1] - j0;
        if (nj == 0) continue;
        const int b0 = wave_b0[w], nbt = wave_b0[w + 1] - b0;
        if (nbt > 0) {
            // (latency-bound: one or two cells per warp, up to 16 CTAs per SM)
            const int pcells = use_tc ? tc3 : max_nm;
            const int psplit = std::max(1, std::min((pcells + 7) / 8, (16 * 148 + nj - 1) / nj));
            if (g.B <= 4) {  // one thread per coarse cell
                const int py = (pcells * g.B + 127) / 128;
                auto pk = g.B == 4 ? (g.aligned4 ? prep3d_cell_kernel<4, true> : prep3d_cell_kernel<4, false>)
                                   : prep3d_cell_kernel<2, false>;
                launch_pdl(pk, dim3(nj, py), dim3(128), 0, st, g, static_cast<const Job3*>(d_jobs), j0,
                           static_cast<const int*>(d_moff), static_cast<const int*>(d_mcells),
                           static_cast<const uint8_t*>(d_work), use_tc ? d_w8 : d_w, use_tc ? kbytes / 4 : wstride,
                           use_tc ? tc3 : 0);
            } else if (use_dig) {  // three digit rows per job, written in place
                const int ps = std::max(1, std::min((tc3 + 7) / 8, (16 * 148 + nj - 1) / nj));
                launch_pdl(prep3d_kernel, dim3(nj, ps), dim3(256), 0, st, g, static_cast<const Job3*>(d_jobs), j0,
                           static_cast<const int*>(d_moff), static_cast<const int*>(d_mcells),
                           static_cast<const uint8_t*>(d_work), d_w8, 3 * kdig / 4, tc3);
            } else
                launch_pdl(prep3d_kernel, dim3(nj, psplit), dim3(256), 0, st, g, static_cast<const Job3*>(d_jobs), j0,
                           static_cast<const int*>(d_moff), static_cast<const int*>(d_mcells),
                           static_cast<const uint8_t*>(d_work), d_w, wstride, 0);
            ++launches;
            cudaEvent_t ea = nullptr, eb = nullptr;
            if (ctx->profiling) {
                CCW_CUDA(cudaEventCreate(&ea));
                CCW_CUDA(cudaEventCreate(&eb));
                CCW_CUDA(cudaEventRecord(ea, st));
            }
            Screen3Args q = sa;
            q.bt0 = b0;
            q.j0 = j0;
            q.nj = nj;
            if (use_tc) {
                launch_ccf_tc(tcplan, npos, sld, kbytes, nj, d_sc, d_tm, st);
                launches += 1;
                ++ccf_launches;
            }
            if (use_dig) {
                launch_ccf_tc(tcplan, npos, sld, kdig, 3 * nj, d_sc, d_tm, st);
                launch_pdl(keys3d_digits_kernel, dim3(nj, nsplit), dim3(256), 0, st, static_cast<const int32_t*>(d_sc),
                           sld, npos, sa.K, d_x);
                launches += 2;
                ++ccf_launches;
            }
            for (int v = 0; v < (use_tc || use_dig ? 0 : S_virt); ++v) {
                const int s = ctx->shard_rank * S_virt + v;
                q.box0 = std::min(nbox, s * bps);
                q.box1 = std::min(nbox, (s + 1) * bps);
                q.shard = s;
                if (q.box1 <= q.box0) continue;
                launch_pdl(screen, dim3(q.box1 - q.box0, nbt), dim3(S3_THREADS), smem_tot, st, q);
                ++launches;
                ++ccf_launches;
            }
            if (ctx->profiling) {
                CCW_CUDA(cudaEventRecord(eb, st));
                ccf_ev.push_back({ea, eb});
            }
            for (int b = b0; b < b0 + nbt; ++b) {
                const int nm = mask_off[batches[b].mask + 1] - mask_off[batches[b].mask];
                ccf_flop += 2.0 * g.F * static_cast<double>(npos) * nm * batches[b].n;
            }
            if (ctx->nccl_comm) {
                const size_t chunk = static_cast<size_t>(S_virt) * nj * bps * sa.K;
                nccl_all_gather_bytes(ctx->nccl_comm, d_x + ctx->shard_rank * chunk, d_x,
                                      chunk * sizeof(unsigned long long), st);
            }
        }
        Select3Args q = se;
        q.j0 = j0;
        q.nj = nj;
        if (use_tc) {  // the score rows and tile maxima instead of key lists
            q.sc = d_sc;
            q.tm = d_tm;
            q.sld = sld;
            q.tld = tld;
            q.npos = npos;
        }
        if (use_dig) {  // keys3d_digits_kernel's chunk lists
            q.S = 1;
            q.bps = q.nbox = nsplit;
        }
        const int ssplit = std::max(1, std::min(g.T, (16 * 148 + nj - 1) / nj));
        launch_pdl(select3d_kernel, dim3(nj, ssplit), dim3(128), 0, st, q);
        ++launches;
    }
    {
        const size_t n = sgvol;
        const int bx = static_cast<int>(std::min<size_t>((n + 255) / 256, 2048));
        launch_pdl(finalize3d_kernel, dim3(bx, n_real), dim3(256), 0, st, static_cast<const uint8_t*>(d_work), g.W[0],
                   g.W[1], g.W[2], cfg.sg[0], cfg.sg[1], cfg.sg[2], fin);
        ++launches;
        if (d_hd) {
            hd3d_kernel<<<dim3(std::min((n_hd + 255) / 256, 256), n_real), 256, 0, st>>>(
                d_hd, n_hd, cfg.sg[0], cfg.sg[1], cfg.sg[2], fin, d_mism);
            CCW_CUDA(cudaGetLastError());
            ++launches;
        }
    }
    CCW_CUDA(cudaEventRecord(ev1, st));
    if (host_t) fprintf(stderr, "3D host ms: plan %.3f ev0 %.3f launched %.3f\n", t_plan, t_ev0, host_ms());
    // Host result, opt-in (option `pack` = 2): codes packed 1 / 2 / 4 bits per
    // cell on the device, copied in chunks to pinned staging and unpacked into
    // the caller's buffer by the context's host threads as the chunks land.
    // Off by default: with a pinned result buffer the plain copy is faster on
    // the 16-core bench hosts (config 3 e2e 17.2 vs 13.2 G cells/s packed).
    const size_t out_cells = sgvol * n_real;
    const int pbits = g.F <= 2 ? 1 : g.F <= 4 ? 2 : 4;
    const bool packed_out = h_out && ctx->opt.pack >= 2 && g.F <= 16 && out_cells >= (size_t(1) << 16);
    std::vector<cudaEvent_t> pk_ev;
    uint8_t* h_pk = nullptr;
    size_t pk_chunk = 0;  // cells per chunk (a multiple of 64 cells and of whole bytes)
    if (packed_out) {
        const int cpb = 8 / pbits;
        const size_t pbytes = (out_cells + cpb - 1) / cpb;
        uint8_t* d_pk = ctx->band_stage.as<uint8_t>(pbytes);
        h_pk = static_cast<uint8_t*>(ctx->h_out_stage.get(pbytes));
        const unsigned nb = static_cast<unsigned>(std::min<size_t>((pbytes + 255) / 256, 148 * 16));
        if (pbits == 1) pack3d_kernel<1><<<nb, 256, 0, st>>>(fin, out_cells, d_pk);
        else if (pbits == 2) pack3d_kernel<2><<<nb, 256, 0, st>>>(fin, out_cells, d_pk);
        else pack3d_kernel<4><<<nb, 256, 0, st>>>(fin, out_cells, d_pk);
        CCW_CUDA(cudaGetLastError());
        ++launches;
        const int nchunk = 32;
        pk_chunk = ((out_cells + nchunk - 1) / nchunk + 511) / 512 * 512;
        for (size_t c0 = 0; c0 < out_cells; c0 += pk_chunk) {
            const size_t c1 = std::min(out_cells, c0 + pk_chunk);
            CCW_CUDA(cudaMemcpyAsync(h_pk + c0 / cpb, d_pk + c0 / cpb, (c1 - c0 + cpb - 1) / cpb, cudaMemcpyDeviceToHost, st));
            cudaEvent_t e;
            CCW_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            CCW_CUDA(cudaEventRecord(e, st));
            pk_ev.push_back(e);
        }
    } else if (h_out) {
        CCW_CUDA(cudaMemcpyAsync(h_out, fin, out_cells, cudaMemcpyDeviceToHost, st));
    }
    std::vector<int> mism(n_real, 0);
    CCW_CUDA(cudaMemcpyAsync(mism.data(), d_mism, sizeof(int) * n_real, cudaMemcpyDeviceToHost, st));
    std::vector<int32_t> chosen;
    if (trace) {
        chosen.resize(3 * njobs);
        CCW_CUDA(cudaMemcpyAsync(chosen.data(), d_chosen, sizeof(int32_t) * chosen.size(), cudaMemcpyDeviceToHost, st));
    }
    if (packed_out) {
        const int cpb = 8 / pbits;
        ctx->pool.run(static_cast<int>(pk_ev.size()), [&](int c) {
            CCW_CUDA(cudaEventSynchronize(pk_ev[c]));
            const size_t c0 = static_cast<size_t>(c) * pk_chunk, c1 = std::min(out_cells, c0 + pk_chunk);
            unpack_cells(h_out + c0, h_pk + c0 / cpb, c1 - c0, pbits);
        });
        for (auto e : pk_ev) cudaEventDestroy(e);
    }
    CCW_CUDA(cudaStreamSynchronize(st));
    if (trace)  // provenance: TI fine origin of every placement, raster order per realization
        for (size_t k = 0; k < njobs; ++k)
            if (jobs[k].place < trace_cap)
                for (int a = 0; a < 3; ++a)
                    trace[(static_cast<size_t>(jobs[k].real) * trace_cap + jobs[k].place) * 3 + a] = chosen[3 * k + a];
    float ms = 0;
    cudaEventElapsedTime(&ms, ev0, ev1);
    double ccf_ms = 0;
    for (auto& e : ccf_ev) {
        float m = 0;
        cudaEventElapsedTime(&m, e.first, e.second);
        ccf_ms += m;
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    ctx->timing = ccw_timing{};
    ctx->timing.total_ms = ms;
    ctx->timing.ccf_ms = ccf_ms;
    ctx->timing.ccf_launches = static_cast<int64_t>(ccf_ev.size());
    ctx->timing.launches = launches;
    ctx->timing.ccf_flop = ccf_flop;
    ctx->timing.ccf_flop_ref = ccf_flop;
    ctx->timing.waves = max_key + 1;
    ctx->timing.jobs = static_cast<int64_t>(njobs);
    ctx->timing.screened_jobs = static_cast<int64_t>(njobs) - n_real;
    ctx->timing.ccf_variant = use_tc ? 6 : use_dig ? 7 : mode == 0 ? 3 : 4;
    ctx->timing.groups = 1;
    ctx->timing.d2h_bytes = !h_out ? 0 : packed_out ? static_cast<int64_t>((out_cells + 8 / pbits - 1) / (8 / pbits))
                                                    : static_cast<int64_t>(out_cells);
    (void)ccf_launches;
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
    if (diag)
        for (int r = 0; r < n_real; ++r) {
            ccw_diag3d& d = diag[r];
            d.seed = seeds[r];
            d.corner = corners[r];
            d.order = orders[r];
            for (int a = 0; a < 3; ++a) d.work[a] = g.W[a];
            d.placement_count = counts[r];
            d.hard_data_count = hd ? n_hd : 0;
            d.pre_overwrite_mismatches = mism[r];
            d.wall_seconds = wall;
        }
}

}  // namespace ccwgpu
