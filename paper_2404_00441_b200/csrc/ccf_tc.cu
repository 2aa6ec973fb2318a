// ccf_tc.cu -- the CCF screen as an int8 implicit GEMM on the 5th-generation
// tensor cores (tcgen05.mma kind::i8, int32 accumulators in TMEM).
//
// For one wave of placements (jobs) the exact-integer screen is
//
//   S[job, pos] = sum_k W[job, k] * X[pos, k],   k = (channel, s, t) over the
//                                                 Tc x Tc coarse template window
//
// with X the im2col of the TI block-count planes (built once per TI and Tc,
// int8: counts <= 4^J <= 64) and W the per-job OR weights (int8 in [-4^J, 4^J],
// zero off the overlap mask).  int8 x int8 -> int32 is exact, so S equals the
// fp32 CUDA-core screen (ccf_direct_kernel) bit for bit.  Off-mask template
// cells cost MMA work but no correctness (their weights are zero).
//
// Tile: M = 128 jobs x N = 256 positions, K in 128-byte stages, a TMA ->
// shared-memory (128B swizzle) ring feeding a single-thread MMA issuer; the
// accumulator (128 lanes x 256 columns int32) lives in TMEM.  The epilogue
// (8 warps, one TMEM lane per job) transposes each 32 x 32 block through
// shared memory so the score rows are written with row-contiguous stores,
// and keeps the maximum of every 128-position tile, from which the select
// kernel bounds the K-th largest score without rescanning every position.
#include <cuda.h>

#include <algorithm>
#include <climits>
#include <mutex>

#include "ccw_device.cuh"
#include "ccf_tc.hpp"
#include "internal.hpp"

namespace ccwgpu {

namespace {

constexpr int kM = 128;
constexpr int kN = 256;
constexpr int kKC = 128;  // bytes of K per stage (one 128B swizzle atom)
#ifndef CCW_TC_STAGES
#define CCW_TC_STAGES 3
#endif
#ifndef CCW_TC_ACC
#define CCW_TC_ACC 2
#endif
constexpr int kStages = CCW_TC_STAGES;
constexpr int kAcc = CCW_TC_ACC;  // TMEM accumulators (kAcc x 256 columns)
constexpr int kABytes = kM * kKC;
constexpr int kBBytes = kN * kKC;
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kEpiWarps = 8;  // two warps per TMEM lane quarter, 128 columns each
constexpr int kThreads = 64 + 32 * kEpiWarps;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}

// UMMA shared-memory descriptor, K-major operand in the canonical 128B-swizzle
// layout TMA writes: 8-row x 128-byte swizzle atoms, SBO = 1024 bytes between
// 8-row groups, LBO unused (1), version 1 (tcgen05), layout SWIZZLE_128B (2).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(1024 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}

// kind::i8 instruction descriptor: D s32, A s8, B s8, both K-major.
__host__ __device__ constexpr uint32_t i8_idesc(int M, int N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     bar)
                 : "memory");
}

#define LDTM_X32(taddr, r)                                                                         \
    asm volatile(                                                                                  \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"   \
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"         \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),      \
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),  \
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),            \
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),            \
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])             \
        : "r"(taddr))

// One (job tile, half position tile) of accumulators, drained from TMEM:
// the exact scores and the tile maximum.  stage = this warp's 4 KB of shared
// memory (32 rows x 128 B, 16-byte chunks swizzled by row) for the transpose.
template <bool S16, bool NU>
__device__ __forceinline__ void tc_epilogue(const TcArgs& a, uint32_t tbuf, int m0, int n0,
                                            int warp, int lane, uint32_t stage) {
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int job = m0 + q * 32 + lane;
    const uint32_t trow = tbuf + (static_cast<uint32_t>(q * 32) << 16) + half * (kN / 2);
    const int pbase = n0 + half * (kN / 2);
    const int ntile = (n0 / kN) * 2 + half;
    int mx = INT_MIN, mxn = INT_MIN;
    const bool nu = NU && job < a.nj;
    uint4 ub = make_uint4(0, 0, 0, 0);  // this job's non-uniform bits of the 128 positions (tmax_nu)
    if (NU && nu) ub = *reinterpret_cast<const uint4*>(a.ubits + static_cast<size_t>(a.jvar[job]) * (a.ustride / 32) + pbase / 32);
    // store phase: lane -> (row r0 + 4 i, 16-byte chunk lane & 7)
    const int srow = lane >> 3, schunk = lane & 7;
#ifndef CCW_TC_LDTM1  // (measured r1: two chunks per wait is ~2% faster end to end)
#define CCW_TC_LDTM2
#endif
#ifdef CCW_TC_LDTM2
    uint32_t rr[2][32];  // two 32-column chunks per TMEM round trip (more registers)
#endif
#pragma unroll
    for (int c = 0; c < kN / 64; ++c) {
#ifdef CCW_TC_LDTM2
        if ((c & 1) == 0) {
            LDTM_X32(trow + c * 32, rr[0]);
            LDTM_X32(trow + (c + 1) * 32, rr[1]);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        }
        uint32_t (&r)[32] = rr[c & 1];
#else
        uint32_t r[32];
        LDTM_X32(trow + c * 32, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#endif
        const int p0 = pbase + c * 32;
        const int lim = a.npos - p0;  // valid columns of this chunk
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (i < lim) mx = max(mx, static_cast<int>(r[i]));
        if (NU && nu) {  // (the bits are 0 past npos: ustride covers whole tiles)
            const uint32_t bm = c == 0 ? ub.x : c == 1 ? ub.y : c == 2 ? ub.z : ub.w;
#pragma unroll
            for (int i = 0; i < 32; ++i)
                if ((bm >> i) & 1u) mxn = max(mxn, static_cast<int>(r[i]));
        }
#pragma unroll
        for (int v = 0; v < 8; ++v) {
            const uint32_t addr = stage + lane * 128 + ((v ^ (lane & 7)) << 4);
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(r[4 * v]),
                         "r"(r[4 * v + 1]), "r"(r[4 * v + 2]), "r"(r[4 * v + 3])
                         : "memory");
        }
        __syncwarp();
        const int pos = p0 + schunk * 4;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int row = 4 * i + srow;
            const uint32_t addr = stage + row * 128 + ((schunk ^ (row & 7)) << 4);
            int4 v;
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                         : "r"(addr)
                         : "memory");
            const int jr = m0 + q * 32 + row;
            // rows are padded to sld (a multiple of 4) >= npos: a chunk that
            // starts inside the row is stored whole
            if (jr < a.nj && pos < a.npos) {
                if (S16) {  // (exact: every score fits int16, checked on the host)
                    const uint2 h = make_uint2((static_cast<uint32_t>(v.x) & 0xffffu) | (static_cast<uint32_t>(v.y) << 16),
                                               (static_cast<uint32_t>(v.z) & 0xffffu) | (static_cast<uint32_t>(v.w) << 16));
                    *reinterpret_cast<uint2*>(reinterpret_cast<int16_t*>(a.scores) + static_cast<size_t>(jr) * a.sld + pos) = h;
                } else {
                    *reinterpret_cast<int4*>(a.scores + static_cast<size_t>(jr) * a.sld + pos) = v;
                }
            }
        }
        __syncwarp();
    }
    if (job < a.nj) a.tmax[static_cast<size_t>(job) * a.ntiles + ntile] = mx;
    if (NU && nu) a.tmax_nu[static_cast<size_t>(job) * a.ntiles + ntile] = mxn;
}

// Persistent implicit GEMM: one CTA per SM loops over (job tile, position
// tile) pairs; warp 0 streams K stages through a 4-deep TMA ring, warp 1
// issues the MMAs into one of two TMEM accumulators, warps 2..9 drain the
// other accumulator -- the epilogue of tile i overlaps the loads and MMAs of
// tile i+1.
#ifndef CCW_TC_MINB
#define CCW_TC_MINB 1
#endif
// S16: int16 score rows; NU: per-tile non-uniform maxima too (tie-storm TIs)
// -- separate instances keep the common one's registers unchanged
template <bool S16, bool NU>
__global__ void __launch_bounds__(kThreads, CCW_TC_MINB)
    ccf_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  TcArgs a) {
    extern __shared__ __align__(1024) uint8_t tc_sm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_sm_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + kStages * kStageBytes);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;   // [2] accumulator ready
    uint64_t* tempty = tfull + 2;        // [2] accumulator drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    // 4 KB per epilogue warp: after the ring when CTAs loop over tiles; in the
    // ring itself when each CTA drains a single tile (its MMAs have read every
    // stage before the accumulator is signalled full, and nothing is loaded
    // after them), which halves the footprint so two CTAs share an SM
    const uint32_t epi_stage = a.epi_in_ring ? smem_u32(sm) : smem_u32(sm + kStages * kStageBytes + 256);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_mt = (a.nj + kM - 1) / kM, n_nt = (a.npos + kN - 1) / kN;
    const long long pc0 = clock64();
    auto probe = [&](int k) {
        if (a.probe) atomicAdd(&a.probe[k], static_cast<unsigned long long>(clock64() - pc0));
    };
    pdl_trigger();
    const int ntot = n_mt * n_nt;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&tfull[b]), 1);
            mbar_init(smem_u32(&tempty[b]), kEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)));
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)));
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
            smem_u32(tmem_slot)), "n"(kAcc * kN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) probe(0);
    // The dependency wait (griddepcontrol.wait) is per role: the producer's B
    // operand (the TI im2col) does not depend on earlier kernels, so the first
    // ring of B tiles is requested before it; the weights (A, written by
    // or_prep) and the epilogue's stores (score rows the previous select read)
    // wait.  The MMA warp touches no global memory.

    if (warp == 0) {
        if (lane == 0) {  // TMA producer: K stages of every tile, one ring
            // prologue: the first ring's B tiles, before the dependency wait
            int npre = 0;
            for (int t = blockIdx.x; t < ntot && npre < kStages; t += gridDim.x) {
                const int n0 = (t / n_mt) * kN;
                for (int kc = 0; kc < a.nk && npre < kStages; ++kc, ++npre) {
                    const uint32_t bar = smem_u32(&full[npre]);
                    mbar_expect_tx(bar, kStageBytes);
                    tma_load_2d(smem_u32(sm + npre * kStageBytes + kABytes), &tmB, kc * kKC, n0, bar);
                }
            }
            tl_mark(a.tl, 2);
            pdl_wait();  // the weights (or_prep) are complete
            tl_mark(a.tl, 0);
            probe(1);
            int it = 0;
            for (int t = blockIdx.x; t < ntot; t += gridDim.x) {
                const int m0 = (t % n_mt) * kM, n0 = (t / n_mt) * kN;
                for (int kc = 0; kc < a.nk; ++kc, ++it) {
                    const int s = it % kStages;
                    const uint32_t bar = smem_u32(&full[s]);
                    if (it >= npre) {
                        if (it >= kStages) mbar_wait(smem_u32(&empty[s]), ((it / kStages) - 1) & 1);
                        mbar_expect_tx(bar, kStageBytes);
                        tma_load_2d(smem_u32(sm + s * kStageBytes + kABytes), &tmB, kc * kKC, n0, bar);
                    }
                    tma_load_2d(smem_u32(sm + s * kStageBytes), &tmA, kc * kKC, m0, bar);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // single-thread MMA issuer
            constexpr uint32_t idesc = i8_idesc(kM, kN);
            int it = 0, lt = 0;
            for (int t = blockIdx.x; t < ntot; t += gridDim.x, ++lt) {
                const int b = lt % kAcc;
                if (lt >= kAcc) mbar_wait(smem_u32(&tempty[b]), ((lt / kAcc) - 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t acc = tmem + b * kN;
                for (int kc = 0; kc < a.nk; ++kc, ++it) {
                    const int s = it % kStages;
                    mbar_wait(smem_u32(&full[s]), (it / kStages) & 1);
                    if (it == 0) probe(2);
                    if (it == a.nk - 1) probe(3);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint64_t ad = sw128_desc(smem_u32(sm + s * kStageBytes));
                    const uint64_t bd = sw128_desc(smem_u32(sm + s * kStageBytes + kABytes));
#pragma unroll
                    for (int k = 0; k < kKC / 32; ++k)  // K = 32 bytes per kind::i8 MMA
                        mma_i8(acc, ad + 2 * k, bd + 2 * k, idesc, (kc | k) != 0);
                    mma_commit(smem_u32(&empty[s]));
                }
                mma_commit(smem_u32(&tfull[b]));
            }
        }
    } else {  // epilogue warps 2..9
        pdl_wait();  // the previous wave's select has read the score rows
        int lt = 0;
        for (int t = blockIdx.x; t < ntot; t += gridDim.x, ++lt) {
            const int b = lt % kAcc;
            mbar_wait(smem_u32(&tfull[b]), (lt / kAcc) & 1);
            if (lt == 0 && warp == 2 && lane == 0) probe(4);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int m0 = (t % n_mt) * kM, n0 = (t / n_mt) * kN;
            tc_epilogue<S16, NU>(a, tmem + b * kN, m0, n0, warp, lane, epi_stage + (warp - 2) * 4096);
            if (lt == 0 && lane == 0) probe(5);  // summed over the 8 epilogue warps
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[b])) : "memory");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    tl_mark(a.tl, 1);
    if (threadIdx.x == 0) {
        probe(6);
        if (a.probe) atomicAdd(&a.probe[7], 1ull);
    }
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kAcc * kN));
}

// Tensor-core peak probe: back-to-back kind::i8 MMAs of the screen's shape
// (M=128, N=256, K=32, cta_group::1) on shared-memory operands, one CTA per SM.
__global__ void __launch_bounds__(128, 1) i8_peak_kernel(int iters) {
    extern __shared__ __align__(1024) uint8_t pk_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(pk_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + kABytes + kBBytes);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (kABytes + kBBytes) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u;
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(bar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *slot;
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = i8_idesc(kM, kN);
        const uint64_t ad = sw128_desc(smem_u32(sm)), bd = sw128_desc(smem_u32(sm + kABytes));
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int k = 0; k < 4; ++k) mma_i8(tmem, ad + 2 * k, bd + 2 * k, idesc, (i | k) != 0);
        mma_commit(smem_u32(bar));
        mbar_wait(smem_u32(bar), 0);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

// im2col of the TI screen planes: row = score-map position, column k =
// (ch, s, t); values are exact small integers, stored as int8.
__global__ void im2col_kernel(const float* __restrict__ scr, int nscr, int hc, int wc, int Tc,
                              int out_w, int npos, int kpad, int8_t* __restrict__ X) {
    const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t total = static_cast<size_t>(npos) * kpad;
    if (idx >= total) return;
    const int p = static_cast<int>(idx / kpad), k = static_cast<int>(idx - static_cast<size_t>(p) * kpad);
    const int x = p / out_w, y = p - x * out_w;
    int8_t v = 0;
    if (k < nscr * Tc * Tc) {
        const int ch = k / (Tc * Tc), rem = k - ch * Tc * Tc;
        const int s = rem / Tc, t = rem - s * Tc;
        v = static_cast<int8_t>(__float2int_rn(scr[static_cast<size_t>(ch) * hc * wc +
                                                   static_cast<size_t>(x + s) * wc + y + t]));
    }
    X[idx] = v;
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    if (!fn) throw Fail(CCW_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

CUtensorMap make_map(void* base, uint64_t cols_bytes, uint64_t rows, uint32_t box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {cols_bytes, rows};
    const cuuint64_t strides[1] = {cols_bytes};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(kKC), box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Fail(CCW_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    return m;
}

}  // namespace

size_t ccf_tc_smem_bytes(bool epi_in_ring) {
    static_assert(kStages * kStageBytes >= kEpiWarps * 4096, "epilogue staging must fit in the ring");
    return kStages * kStageBytes + 1024 + 256 + (epi_in_ring ? 0 : kEpiWarps * 4096);
}

int tc_num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    return sms;
}

unsigned long long* tc_probe_buffer = nullptr;

int tc_kpad(int nscr, int Tc) { return ((nscr * Tc * Tc + 15) / 16) * 16; }

const int8_t* ti_im2col(ccw_ti* ti, int Tc, cudaStream_t st) {
    auto it = ti->im2col.find(Tc);
    if (it != ti->im2col.end()) return it->second;
    const int out_h = ti->hc - Tc + 1, out_w = ti->wc - Tc + 1;
    const int npos = out_h * out_w;
    const int kpad = tc_kpad(ti->nscr, Tc);
    int8_t* X = static_cast<int8_t*>(cache_alloc(ti->device, static_cast<size_t>(npos) * kpad));
    const size_t total = static_cast<size_t>(npos) * kpad;
    im2col_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(
        ti->d_scr, ti->nscr, ti->hc, ti->wc, Tc, out_w, npos, kpad, X);
    CCW_CUDA(cudaGetLastError());
    ti->im2col[Tc] = X;
    return X;
}

double measure_i8_peak(cudaStream_t st) {
    const int sms = tc_num_sms();
    const size_t smem = kABytes + kBBytes + 1024 + 64;
    CCW_CUDA(cudaFuncSetAttribute(i8_peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    cudaEvent_t a, b;
    CCW_CUDA(cudaEventCreate(&a));
    CCW_CUDA(cudaEventCreate(&b));
    const int iters = 4096;
    double best = 0;
    for (int rep = 0; rep < 4; ++rep) {
        CCW_CUDA(cudaEventRecord(a, st));
        i8_peak_kernel<<<sms, 128, smem, st>>>(iters);
        CCW_CUDA(cudaEventRecord(b, st));
        CCW_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        CCW_CUDA(cudaEventElapsedTime(&ms, a, b));
        const double ops = 2.0 * kM * kN * 32.0 * 4.0 * iters * sms;
        if (rep > 0) best = std::max(best, ops / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return best;
}

// Throughput of the screen kernel alone: `njobs` placements' worth of int8
// weights (all ones) against the TI's im2col, `iters` back-to-back launches
// with no dependency between them.  Milliseconds per launch.
double measure_ccf_screen(ccw_ti* ti, int Tc, int njobs, int iters, cudaStream_t st) {
    const int out_h = ti->hc - Tc + 1, out_w = ti->wc - Tc + 1, npos = out_h * out_w;
    const int kpad = tc_kpad(ti->nscr, Tc), sld = (npos + 3) & ~3;
    const int8_t* X = ti_im2col(ti, Tc, st);
    int8_t* W = nullptr;
    int32_t *sc = nullptr, *tmx = nullptr;
    CCW_CUDA(cudaMalloc(&W, static_cast<size_t>(njobs) * kpad));
    CCW_CUDA(cudaMalloc(&sc, sizeof(int32_t) * static_cast<size_t>(njobs) * sld));
    CCW_CUDA(cudaMalloc(&tmx, sizeof(int32_t) * static_cast<size_t>(njobs) * tc_tiles(npos)));
    CCW_CUDA(cudaMemsetAsync(W, 1, static_cast<size_t>(njobs) * kpad, st));
    const TcPlan pl = plan_ccf_tc(W, njobs, X, npos, kpad);
    cudaEvent_t a, b;
    CCW_CUDA(cudaEventCreate(&a));
    CCW_CUDA(cudaEventCreate(&b));
    launch_ccf_tc(pl, npos, sld, kpad, njobs, sc, tmx, st);  // warm-up
    CCW_CUDA(cudaEventRecord(a, st));
    for (int i = 0; i < iters; ++i) launch_ccf_tc(pl, npos, sld, kpad, njobs, sc, tmx, st);
    CCW_CUDA(cudaEventRecord(b, st));
    CCW_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    CCW_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(W);
    cudaFree(sc);
    cudaFree(tmx);
    return ms / iters;
}

TcPlan plan_ccf_tc(const int8_t* d_w8, int maxj, const int8_t* d_x, int npos, int kpad) {
    TcPlan pl;
    pl.ma = make_map(const_cast<int8_t*>(d_w8), kpad, maxj, kM);
    pl.mb = make_map(const_cast<int8_t*>(d_x), kpad, npos, kN);
    for (auto k : {ccf_tc_kernel<false, false>, ccf_tc_kernel<true, false>, ccf_tc_kernel<false, true>,
                   ccf_tc_kernel<true, true>})
        CCW_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(ccf_tc_smem_bytes())));
    return pl;
}

void launch_ccf_tc(const TcPlan& pl, int npos, int sld, int kpad, int nj, int32_t* scores,
                   int32_t* tmax, cudaStream_t st, unsigned long long* tl, int tmax_ld, int s16, int32_t* tmax_nu,
                   const uint32_t* ubits, int ustride, const int8_t* jvar) {
    TcArgs a{};
    a.tmax_nu = tmax_nu;
    a.ubits = ubits;
    a.ustride = ustride;
    a.jvar = jvar;
    a.nj = nj;
    a.npos = npos;
    a.sld = sld;
    a.nk = (kpad + kKC - 1) / kKC;
    a.ntiles = tmax_ld >= 0 ? tmax_ld : tc_tiles(npos);  // (row stride of tmax)
    a.s16 = s16;
    a.scores = scores;
    a.tmax = tmax;
    a.probe = tc_probe_buffer;
    a.tl = tl;
    const int ntot = ((npos + kN - 1) / kN) * ((nj + kM - 1) / kM);
    // CTAs resident at once: CCW_TC_MINB per SM when the footprint allows
    const int slots = tc_num_sms() * CCW_TC_MINB;
    int cap = slots;
    if (const char* e = debug_env("CCW_TC_GRID")) cap = std::max(1, std::min(slots, atoi(e)));
    a.epi_in_ring = ntot <= cap;
    dim3 grid(std::min(ntot, cap));
    auto k = s16 ? (tmax_nu ? ccf_tc_kernel<true, true> : ccf_tc_kernel<true, false>)
                 : (tmax_nu ? ccf_tc_kernel<false, true> : ccf_tc_kernel<false, false>);
    launch_pdl(k, grid, dim3(kThreads), ccf_tc_smem_bytes(a.epi_in_ring), st, pl.ma, pl.mb, a);
}

int tc_tiles(int npos) { return 2 * ((npos + kN - 1) / kN); }  // tile maxima per score row

}  // namespace ccwgpu
