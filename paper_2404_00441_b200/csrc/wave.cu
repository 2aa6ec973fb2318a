// wave.cu -- the fused wave kernel: for one wave of placements a cluster of
// CTAs prepares the overlap regions, screens every TI window on the tensor
// cores, keeps the exact top-K' of the screen in the epilogue, rescores
// equal-score groups in fp64, picks and pastes -- one launch per wave instead
// of prep -> screen -> select, and no score rows in memory.
//
// The screen is an implicit-im2col int8 GEMM.  Positions p = (r, c) of the
// score map (matcher.hpp:132-173) are taken a column c at a time: the TI
// block-count planes restricted to columns [c, c + 16) form a "strip" of
// 16-byte rows, strip[r'][t] = plane[r'][c + t], and the template window of
// position (r, c) at K = (channel, s, t) is strip[r + s][t].  Consecutive
// positions r are the same bytes shifted by one 16-byte row, which the
// canonical no-swizzle K-major UMMA layout expresses directly: core matrices
// of 8 rows x 16 bytes at row stride 16 (SBO = 128), the next K core matrix
// (s + 1) 16 bytes further (LBO = 16).  So one 2.3 KB strip per channel feeds
// a 128-position x 16-placement x (channels x 16 x 16) tcgen05.mma kind::i8
// tile -- the explicit im2col (npos x kpad bytes) never exists.  Strips are
// cut once per TI (ti_strips) and streamed with 1D bulk copies.
//
// Exact top-K' in the epilogue: every epilogue warp owns a quarter of the
// positions (its TMEM lane quarter) and keeps, per placement, a list of
// (score, position) >= a running threshold; when the list fills, a warp-level
// K'-th-largest raises the threshold to the warp's own K'-th largest score,
// which bounds the global S_K' from below -- so the union of the lists holds
// every window with S >= S_K' (ties included).  K' = pick + 1 for an
// unconditional pick (matcher.hpp:207-211; ranks past the pick never matter),
// K for a conditional one.  Ranking is (S desc, fp64 reference score desc,
// index asc): windows with different S never swap, so
// only equal-S groups are rescored in fp64 in the reference's exact operation
// order (matcher.hpp:64-81, 158-161, 189-198).  A list that overflows (a tie
// storm) sends its placement to the in-kernel fallback: the cluster recomputes
// the placement's full score row on the CUDA cores and runs the generic CTA
// select (select_common.cuh), which is exact for any tie group.
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <map>

#include "select_common.cuh"

namespace cg = cooperative_groups;

namespace ccwgpu {

namespace {

constexpr int WV_NJ = 16;     // placements per cluster (the MMA's N)
constexpr int WV_T = 256;     // threads per CTA (= SEL_T for the fallback)
constexpr int WV_SR = 144;    // strip rows: 128 positions + up to 16 template rows
constexpr int WV_CAP = 64;    // list capacity per (epilogue warp, placement)
constexpr int WV_ST = 6;      // strip ring stages
constexpr int WV_NACC = 4;    // TMEM accumulators (16 columns each)
constexpr int WV_GCAP = 128;  // equal-score group members rescored per warp
constexpr int WV_RS = 256;    // (member, run) partial sums per chunk
constexpr int WV_MAXCS = 4;   // CTAs per cluster (position column ranges)
constexpr int WV_KMAX = 16;   // largest K (and K') this path takes
#ifndef CCW_WV_MINB
#define CCW_WV_MINB 1
#endif

static_assert(WV_T == SEL_T, "the fallback runs the generic select with every thread");

__device__ __forceinline__ uint32_t su(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
// no-swizzle K-major UMMA shared-memory descriptor (version 1, layout 0)
__device__ __forceinline__ uint64_t ns_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (static_cast<uint64_t>(1) << 46);
}
// kind::i8: D s32, A s8, B s8, both K-major
__host__ __device__ constexpr uint32_t wv_idesc(int M, int N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void ldtm16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Per-warp scratch of the post-scan (group rescoring and the ranked list).
struct WvWarp {
    int gpos[WV_GCAP];
    double gkey[WV_GCAP];
    double rsum[WV_RS];
    int4 runs[64];  // (channel, s, t0, t1), reference order
    int tidx[WV_KMAX];
    int misc[4];
};

struct WvLayout {
    int stage_bytes, tsp;
    size_t u, b, lists, cnt, thr, ov, sthr, kq, fb, jobs, bar, total;
};

__host__ __device__ inline WvLayout wv_layout(int nscr, int Tc, int nch, int K, int T, int OV) {
    WvLayout L{};
    L.tsp = (Tc + 1) & ~1;
    L.stage_bytes = nscr * WV_SR * 16;
    size_t u = static_cast<size_t>(WV_ST) * L.stage_bytes;
    u = u > 8 * sizeof(WvWarp) ? u : 8 * sizeof(WvWarp);
    const size_t sl = sel_layout(K, T, OV, nch, Tc, 0).total;
    u = u > sl ? u : sl;
    size_t o = 0;
    L.u = o;
    o += (u + 1023) & ~static_cast<size_t>(1023);
    L.b = o;  // B operand: [nscr * tsp core-matrix columns][16 placements][16 bytes]
    o += static_cast<size_t>(nscr) * L.tsp * WV_NJ * 16;
    L.lists = o;  // [4 quarters][16 placements][WV_CAP] (score, position)
    o += static_cast<size_t>(4) * WV_NJ * WV_CAP * sizeof(int2);
    L.cnt = o;  // [4][16] list lengths
    o += 4 * WV_NJ * sizeof(int);
    L.thr = o;  // [4][16] list thresholds
    o += 4 * WV_NJ * sizeof(int);
    L.ov = o;  // [4][16] largest value dropped from a list (INT_MIN: none)
    o += 4 * WV_NJ * sizeof(int);
    L.sthr = o;  // [16] shared lower bound of S_K' (max of the quarters' K'-th largest)
    o += WV_NJ * sizeof(int);
    L.kq = o;  // [16] K' per placement
    o += WV_NJ * sizeof(int);
    L.fb = o;  // fallback bits of the placements this CTA owns
    o += 4 * sizeof(int);
    L.jobs = o;
    o += WV_NJ * sizeof(Job);
    o = (o + 15) & ~static_cast<size_t>(15);
    L.bar = o;  // full[ST], empty[ST], tfull[NACC], tempty[NACC], tmem slot
    o += (2 * WV_ST + 2 * WV_NACC) * sizeof(uint64_t) + 16;
    L.total = o + 1024;  // (base alignment slack)
    return L;
}

// Raise a list's threshold to its K'-th largest score (or the shared bound,
// whichever is higher) and keep the entries at or above it (warp-wide).  When
// the entries tying at the threshold do not fit, they are dropped and the
// threshold moves past them: the returned .z is the dropped value (INT_MIN
// if none) -- a lower bound of S_K', so the post-scan knows the lists are
// complete above it.  Returns (length, threshold, dropped value).
__device__ __forceinline__ int4 wv_compact(int2* L, int cnt, int kq, int thr) {
    const int lane = threadIdx.x & 31;
    const int2 e0 = lane < cnt ? L[lane] : make_int2(INT_MIN, -1);
    const int2 e1 = lane + 32 < cnt ? L[lane + 32] : make_int2(INT_MIN, -1);
    int cur = INT_MAX, acc = 0, m = INT_MIN;
    for (int r = 0; r < kq; ++r) {
        const int a = max(e0.y >= 0 && e0.x < cur ? e0.x : INT_MIN, e1.y >= 0 && e1.x < cur ? e1.x : INT_MIN);
        m = __reduce_max_sync(0xffffffffu, a);
        if (m == INT_MIN) break;
        acc += __popc(__ballot_sync(0xffffffffu, e0.y >= 0 && e0.x == m)) +
               __popc(__ballot_sync(0xffffffffu, e1.y >= 0 && e1.x == m));
        if (acc >= kq) break;
        cur = m;
    }
    if (acc >= kq) thr = max(thr, m);
    bool k0 = e0.y >= 0 && e0.x >= thr, k1 = e1.y >= 0 && e1.x >= thr;
    int dropped = INT_MIN;
    if (__popc(__ballot_sync(0xffffffffu, k0)) + __popc(__ballot_sync(0xffffffffu, k1)) > WV_CAP - 32) {
        dropped = thr;  // (thr is a lower bound of S_K': a local K'-th largest or the shared bound)
        k0 = k0 && e0.x > thr;
        k1 = k1 && e1.x > thr;
        thr = thr + 1;
    }
    const unsigned b0 = __ballot_sync(0xffffffffu, k0), b1 = __ballot_sync(0xffffffffu, k1);
    const unsigned lt = (1u << lane) - 1;
    __syncwarp();
    if (k0) L[__popc(b0 & lt)] = e0;
    if (k1) L[__popc(b0) + __popc(b1 & lt)] = e1;
    __syncwarp();
    return make_int4(__popc(b0) + __popc(b1), thr, dropped, 0);
}

// fp64 reference scores (matcher.hpp:64-81, 158-161) of the windows
// W.gpos[0, g) for placement jb: one lane per (window, run) forms the run's
// sum left to right, then one lane per window folds the run sums in order.
__device__ __noinline__ void wv_rescore(const SimParams& P, const Job& jb, WvWarp& W, int g, int R) {
    const int lane = threadIdx.x & 31;
    const size_t nc = static_cast<size_t>(P.hc) * P.wc;
    const int32_t* src = P.src + static_cast<size_t>(jb.real) * (P.wh / P.B) * P.swc +
                         static_cast<size_t>(jb.top / P.B) * P.swc + jb.left / P.B;
    const int EG = max(1, WV_RS / R);
    for (int e0 = 0; e0 < g; e0 += EG) {
        const int ng = min(EG, g - e0);
        for (int w = lane; w < ng * R; w += 32) {
            const int e = e0 + w / R, r = w - (w / R) * R;
            const int pos = W.gpos[e];
            const int x = pos / P.out_w, y = pos - x * P.out_w;
            const int4 rd = W.runs[r];
            const double* a = P.ti64 + static_cast<size_t>(rd.x) * nc + static_cast<size_t>(x + rd.y) * P.wc + y;
            const int32_t* sr = src + static_cast<size_t>(rd.y) * P.swc;
            const int n = rd.w - rd.z;
            double av[16], bv[16];
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if (i < n) {
                    av[i] = __ldg(a + rd.z + i);
                    bv[i] = P.ti64[static_cast<size_t>(rd.x) * nc + sr[rd.z + i]];
                }
            double sum = 0.0;
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if (i < n) sum = __dadd_rn(sum, __dmul_rn(av[i], bv[i]));
            W.rsum[w] = sum;
        }
        __syncwarp();
        for (int e = lane; e < ng; e += 32) {
            double acc = 0.0;
            for (int r = 0; r < R; ++r) acc = __dadd_rn(acc, W.rsum[e * R + r]);
            W.gkey[e0 + e] = acc;
        }
        __syncwarp();
    }
    if (P.stats && lane == 0) atomicAdd(&P.stats[0], static_cast<unsigned long long>(g));
}

// The post-scan of placement j (one warp): the union of the cluster's lists,
// S_K', the ranked candidates up to rank `need`, the pick, the paste.
// Returns false when the placement needs the fallback.
template <int CS>
__device__ __noinline__ bool wv_post(const SimParams& P, const Job& jb, int gj, int j, int kq, const int2* lists,
                        const int* cnts, const int* ovs, WvWarp& W) {
    const int lane = threadIdx.x & 31;
    cg::cluster_group cl = cg::this_cluster();
    constexpr int NL = 4 * CS;
    int v[NL], p[NL];
    int dmax = INT_MIN;  // largest value any list dropped: the lists are complete above it
#pragma unroll
    for (int li = 0; li < NL; ++li) {
        const int r = li >> 2, q = li & 3;
        const int2* rl = cl.map_shared_rank(lists, r) + (q * WV_NJ + j) * WV_CAP;
        const int n = *(cl.map_shared_rank(cnts, r) + q * WV_NJ + j);
        dmax = max(dmax, *(cl.map_shared_rank(ovs, r) + q * WV_NJ + j));
        const int2 e = lane < n ? rl[lane] : make_int2(INT_MIN, -1);
        v[li] = e.x;
        p[li] = e.y;
    }
    // the ranking up to rank `need` (matcher.hpp:177-204): equal-S groups in
    // descending S; a group of one needs no fp64 key
    const int pick = jb.pick;
    const int need = kq;
    int R = 0;
    int above = 0, cur = INT_MAX;
    bool runs_ready = false;
    while (above < need) {
        int a = INT_MIN;
#pragma unroll
        for (int li = 0; li < NL; ++li)
            if (p[li] >= 0 && v[li] < cur) a = max(a, v[li]);
        const int m = __reduce_max_sync(0xffffffffu, a);
        if (m == INT_MIN) {  // fewer listed windows than `need`
            if (dmax != INT_MIN) return false;
            break;  // (npos < K)
        }
        if (m <= dmax) return false;  // windows of this score may have been dropped: the generic select
        int g = 0;
#pragma unroll
        for (int li = 0; li < NL; ++li) g += __popc(__ballot_sync(0xffffffffu, p[li] >= 0 && v[li] == m));
        cur = m;
        if (pick >= 0 && above + g <= pick) {  // ranks before the pick: order irrelevant
            above += g;
            continue;
        }
        if (g == 1) {
#pragma unroll
            for (int li = 0; li < NL; ++li)
                if (p[li] >= 0 && v[li] == m) W.tidx[above] = p[li];
            above += 1;
            __syncwarp();
            continue;
        }
        if (g > WV_GCAP) return false;  // a tie storm: the generic select
        int o = 0;
#pragma unroll
        for (int li = 0; li < NL; ++li) {
            const unsigned bl = __ballot_sync(0xffffffffu, p[li] >= 0 && v[li] == m);
            if (bl & (1u << lane)) W.gpos[o + __popc(bl & ((1u << lane) - 1))] = p[li];
            o += __popc(bl);
        }
        if (!runs_ready) {  // the mask's runs in reference order (channel-major, rows ascending)
            if (lane == 0) {
                int r = 0;
                for (int ch = 0; ch < P.nch; ++ch)
                    for (int s = 0; s < P.Tc; ++s) {
                        int t0, t1;
                        mask_row_run(jb.shape, jb.vleft, jb.htop, P.Tc, P.OVc, s, t0, t1);
                        if (t1 > t0) W.runs[r++] = make_int4(ch, s, t0, t1);
                    }
                W.misc[0] = r;
            }
            __syncwarp();
            R = W.misc[0];
            runs_ready = true;
        }
        __syncwarp();
        wv_rescore(P, jb, W, g, R);
        // members in (fp64 desc, index asc) order; ranks past `need` are dropped
        for (int e = lane; e < g; e += 32) {
            const double k = W.gkey[e];
            const int ps = W.gpos[e];
            int rank = 0;
            for (int f = 0; f < g; ++f) {
                const double kf = W.gkey[f];
                rank += kf > k || (kf == k && W.gpos[f] < ps);
            }
            if (above + rank < need) W.tidx[above + rank] = ps;
        }
        above += g;
        __syncwarp();
    }
    __syncwarp();
    const int ntop = min(above, need);
    int pos;
    if (pick >= 0)
        pos = W.tidx[min(pick, ntop - 1)];
    else
        pos = choose_pick(P, jb, W.tidx, ntop, lane);
    const int fr = (pos / P.out_w) << P.J, fc = (pos % P.out_w) << P.J;
    paste_job<32>(P, jb, gj, fr, fc, lane);
    if (lane == 0) {
        P.chosen[2 * gj] = fr;
        P.chosen[2 * gj + 1] = fc;
        if (P.stats) atomicAdd(&P.stats[1], 1ull);
    }
    return true;
}

// The epilogue of one TMEM lane quarter q (one warp): every tile's 16
// placement scores of 32 positions; a placement's list takes the windows at or
// above its threshold.  Kept compact (thresholds and lengths in shared memory,
// a loop over the placements a tile actually lists): the common tile is a
// TMEM load, 16 compares and one warp reduction.
__device__ __noinline__ void wv_epilogue(const SimParams& P, const WaveArgs& A, const WvLayout& L, uint32_t tmem, int q,
                                         int c0, int ntile, int2* lists, int* cnts, int* thrs, int* ovs, int* sthr,
                                         const int* kqs, uint64_t* tfull, uint64_t* tempty) {
    const int lane = threadIdx.x & 31;
    int* wthr = thrs + q * WV_NJ;
    int* wcnt = cnts + q * WV_NJ;
    if (lane < WV_NJ) {
        wthr[lane] = kqs[lane] > 0 ? INT_MIN : INT_MAX;  // (absent placements never list)
        wcnt[lane] = 0;
    }
    __syncwarp();
    int2* myl = lists + q * WV_NJ * WV_CAP;
    long long e_wait = 0, e_work = 0, ncomp = 0, e_ld = 0;
    const unsigned lt = (1u << lane) - 1;
    for (int i = 0; i < ntile; ++i) {
        const int b = i % WV_NACC;
        const long long k0 = clock64();
        mbar_wait(su(&tfull[b]), (i / WV_NACC) & 1);
        const long long k1 = clock64();
        e_wait += k1 - k0;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        uint32_t v[16];
        ldtm16(tmem + (static_cast<uint32_t>(q * 32) << 16) + b * 16, v);
        e_ld += clock64() - k1;
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(su(&tempty[b]));
        const int c = c0 + i / A.nmb, mb = i - (i / A.nmb) * A.nmb;
        const int r = mb * 128 + q * 32 + lane;
        const bool valid = r < P.out_h && !(A.dbg & 2);
        const int pos = r * P.out_w + c;
        unsigned hit = 0;
        const int4* t4 = reinterpret_cast<const int4*>(wthr);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const int4 t = t4[g];
            hit |= (static_cast<int>(v[4 * g]) >= t.x ? 1u : 0u) << (4 * g);
            hit |= (static_cast<int>(v[4 * g + 1]) >= t.y ? 1u : 0u) << (4 * g + 1);
            hit |= (static_cast<int>(v[4 * g + 2]) >= t.z ? 1u : 0u) << (4 * g + 2);
            hit |= (static_cast<int>(v[4 * g + 3]) >= t.w ? 1u : 0u) << (4 * g + 3);
        }
        if (!valid) hit = 0;
        unsigned jobs_hit = __reduce_or_sync(0xffffffffu, hit);
        if (jobs_hit == 0) {
            e_work += clock64() - k1;
            continue;
        }
        int val[WV_NJ];  // (dynamic pick below: a select chain, not local memory)
#pragma unroll
        for (int j = 0; j < WV_NJ; ++j) val[j] = static_cast<int>(v[j]);
        while (jobs_hit) {
            const int j = __ffs(jobs_hit) - 1;
            jobs_hit &= jobs_hit - 1;
            int vj = val[0];
#pragma unroll
            for (int k = 1; k < WV_NJ; ++k) vj = k == j ? val[k] : vj;
            const bool pr = (hit >> j) & 1u;
            const unsigned bal = __ballot_sync(0xffffffffu, pr);
            int cnt = wcnt[j];
            if (pr) myl[j * WV_CAP + cnt + __popc(bal & lt)] = make_int2(vj, pos);
            cnt += __popc(bal);
            __syncwarp();
            if (cnt > WV_CAP - 32) {
                ++ncomp;
                const int4 rr = wv_compact(myl + j * WV_CAP, cnt, kqs[j], max(wthr[j], sthr[j]));
                cnt = rr.x;
                if (lane == 0) {
                    wthr[j] = rr.y;
                    if (rr.z != INT_MIN) {
                        ovs[q * WV_NJ + j] = max(ovs[q * WV_NJ + j], rr.z);
                        atomicMax(&sthr[j], rr.z);
                    } else if (rr.y != INT_MIN) {
                        atomicMax(&sthr[j], rr.y);
                    }
                }
            }
            if (lane == 0) wcnt[j] = cnt;
            __syncwarp();
        }
        if ((i & 7) == 7 && lane < WV_NJ) wthr[lane] = max(wthr[lane], sthr[lane]);  // the other quarters' bounds
        __syncwarp();
        e_work += clock64() - k1;
    }
    if (P.tl && P.stats && lane == 0 && q == 0) {
        atomicAdd(&P.stats[18], static_cast<unsigned long long>(e_wait));
        atomicAdd(&P.stats[19], static_cast<unsigned long long>(e_work));
        atomicAdd(&P.stats[20], static_cast<unsigned long long>(ncomp));
        atomicAdd(&P.stats[21], static_cast<unsigned long long>(ntile));
        atomicAdd(&P.stats[23], static_cast<unsigned long long>(e_ld));
    }
}

// The generic select of one placement (out of line: the wave kernel's hot
// code stays small).
__device__ __noinline__ void wv_fallback(const SimParams& Q, const Job* __restrict__ jobs, int job0, int slot,
                                         unsigned char* sm) {
    select_paste_body(Q, jobs, job0, slot, 1, sm);
}

template <int CS>
__global__ void __launch_bounds__(WV_T, CCW_WV_MINB)
    wave_kernel(const __grid_constant__ SimParams P, const Job* __restrict__ jobs, int job0, int nj, WaveArgs A) {
    extern __shared__ __align__(1024) uint8_t wv_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(wv_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const WvLayout L = wv_layout(P.nscr, P.Tc, P.nch, P.K, P.T, P.OV);
    uint8_t* ring = sm + L.u;
    int8_t* Bs = reinterpret_cast<int8_t*>(sm + L.b);
    int2* lists = reinterpret_cast<int2*>(sm + L.lists);
    int* cnts = reinterpret_cast<int*>(sm + L.cnt);
    int* thrs = reinterpret_cast<int*>(sm + L.thr);
    int* ovs = reinterpret_cast<int*>(sm + L.ov);
    int* sthr = reinterpret_cast<int*>(sm + L.sthr);
    int* kqs = reinterpret_cast<int*>(sm + L.kq);
    int* fbm = reinterpret_cast<int*>(sm + L.fb);
    Job* js = reinterpret_cast<Job*>(sm + L.jobs);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + L.bar);
    uint64_t* empty = full + WV_ST;
    uint64_t* tfull = empty + WV_ST;
    uint64_t* tempty = tfull + WV_NACC;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + WV_NACC);

    cg::cluster_group cl = cg::this_cluster();
    const int rank = static_cast<int>(cl.block_rank());
    const int set = static_cast<int>(blockIdx.x) / CS;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int js0 = set * WV_NJ;                     // first job slot of the set
    const int njs = min(WV_NJ, nj - js0);            // placements of this set
    const int cpc = (P.out_w + CS - 1) / CS;         // columns per CTA
    const int c0 = min(P.out_w, rank * cpc), c1 = min(P.out_w, c0 + cpc);
    const int ntile = (c1 - c0) * A.nmb;
    const int tsp = L.tsp, nk = P.nscr * (tsp / 2);  // MMAs per tile (K = 32 bytes each)

    const long long pc0 = clock64();
    auto phase = [&](int k) {  // debug timeline runs only: cycles from CTA start per phase, summed
        if (P.tl && P.stats && tid == 0) atomicAdd(&P.stats[8 + k], static_cast<unsigned long long>(clock64() - pc0));
    };
    pdl_trigger();
    if (tid == 0) {
        for (int s = 0; s < WV_ST; ++s) {
            mbar_init(su(&full[s]), 1);
            mbar_init(su(&empty[s]), 1);
        }
        for (int b = 0; b < WV_NACC; ++b) {
            mbar_init(su(&tfull[b]), 1);
            mbar_init(su(&tempty[b]), 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su(tslot)), "n"(WV_NACC * 16));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int e = tid; e < P.nscr * tsp * WV_NJ; e += WV_T)  // zero B (K padding, absent placements)
        reinterpret_cast<int4*>(Bs)[e] = make_int4(0, 0, 0, 0);
    if (tid < 4 * WV_NJ) ovs[tid] = INT_MIN;
    if (tid < WV_NJ) {
        sthr[tid] = INT_MIN;
        if (tid < njs) js[tid] = jobs[job0 + js0 + tid];
    }
    if (tid < 4) fbm[tid] = 0;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;
    // the TI strips do not depend on earlier launches: the first ring is
    // requested before the dependency wait
    if (warp == 0 && lane == 0)
        for (int i = 0; i < min(ntile, WV_ST); ++i) {
            const int c = c0 + i / A.nmb, mb = i - (i / A.nmb) * A.nmb;
            mbar_expect_tx(su(&full[i]), L.stage_bytes);
            bulk_load(su(ring + static_cast<size_t>(i) * L.stage_bytes),
                      A.strips + (static_cast<size_t>(c) * A.nmb + mb) * L.stage_bytes, L.stage_bytes, su(&full[i]));
        }
    tl_mark(P.tl, 2);
    pdl_wait();  // the previous wave's pastes (the source-block map) are complete
    tl_mark(P.tl, 0);
    phase(0);

    // ---- OR prep: int8 screen weights of the set's placements into B ----------
    // (prep_src_job's arithmetic; thread = template cell, every placement's map
    //  entry then every screen plane in flight at once)
    {
        const int Tc = P.Tc, B = P.B;
        const size_t nc = static_cast<size_t>(P.hc) * P.wc;
        const int c = tid, s = c / Tc, t = c - s * Tc;
        if (c < Tc * Tc) {
            int sb[WV_NJ];
            unsigned inm = 0;
#pragma unroll
            for (int j = 0; j < WV_NJ; ++j) {
                sb[j] = 0;
                if (j < njs) {
                    const Job& jb = js[j];
                    int t0, t1;
                    mask_row_run(jb.shape, jb.vleft, jb.htop, Tc, P.OVc, s, t0, t1);
                    if (t >= t0 && t < t1) {
                        inm |= 1u << j;
                        if (!(A.dbg & 1))
                            sb[j] = P.src[static_cast<size_t>(jb.real) * (P.wh / B) * P.swc +
                                          static_cast<size_t>(jb.top / B + s) * P.swc + jb.left / B + t];
                    }
                }
            }
            for (int f0 = 0; f0 < P.nscr; f0 += 2) {  // two screen planes per round trip
                float n[WV_NJ][2];
#pragma unroll
                for (int j = 0; j < WV_NJ; ++j)
#pragma unroll
                    for (int u = 0; u < 2; ++u)
                        n[j][u] = ((inm >> j) & 1u) && f0 + u < P.nscr && !(A.dbg & 1) ? P.tiscr[(f0 + u) * nc + sb[j]] : 0.f;
#pragma unroll
                for (int j = 0; j < WV_NJ; ++j) {
                    if (!((inm >> j) & 1u)) continue;
                    int last = B * B;
                    if (P.mode == 0)  // the last facies' count: every cell holds one facies
                        for (int f = 0; f < P.nscr; ++f)
                            last -= static_cast<int>(f >= f0 && f < f0 + 2 ? n[j][f - f0] : P.tiscr[f * nc + sb[j]]);
#pragma unroll
                    for (int u = 0; u < 2; ++u)
                        if (f0 + u < P.nscr) {
                            const int v = static_cast<int>(n[j][u]);
                            Bs[(((f0 + u) * tsp + s) * WV_NJ + j) * 16 + t] = static_cast<int8_t>(P.mode == 0 ? v - last : v);
                        }
                }
            }
        }
        if (tid < WV_NJ) {
            int kq = 0;
            if (tid < njs) {
                const Job& jb = js[tid];
                kq = jb.pick >= 0 ? min(jb.pick + 1, P.K) : P.K;
            }
            kqs[tid] = kq;
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // B: generic writes -> the MMA's async proxy
    __syncthreads();
    phase(1);

    // ---- screen: strips -> tcgen05 -> exact top-K' lists ----------------------
    if (warp == 0) {
        if (lane == 0)  // producer: the rest of the strips through the ring
            for (int i = WV_ST; i < ntile; ++i) {
                const int s = i % WV_ST;
                mbar_wait(su(&empty[s]), ((i / WV_ST) - 1) & 1);
                const int c = c0 + i / A.nmb, mb = i - (i / A.nmb) * A.nmb;
                mbar_expect_tx(su(&full[s]), L.stage_bytes);
                bulk_load(su(ring + static_cast<size_t>(s) * L.stage_bytes),
                          A.strips + (static_cast<size_t>(c) * A.nmb + mb) * L.stage_bytes, L.stage_bytes, su(&full[s]));
            }
    } else if (warp == 1) {
        if (lane == 0) {  // single-thread MMA issuer
            constexpr uint32_t idesc = wv_idesc(128, WV_NJ);
            constexpr int KM = 32;  // MMAs per tile: nscr * tsp / 2 <= 4 * 8
            uint64_t ad0[KM], bd[KM];
            const uint32_t abase = su(ring), bbase = su(Bs);
#pragma unroll
            for (int k = 0; k < KM; ++k) {
                const int ch = k / 8, sp = k % 8;  // (tsp / 2 <= 8: s pairs padded to 8 per channel)
                ad0[k] = ns_desc(abase + ch * (WV_SR * 16) + sp * 32, 16, 128);
                bd[k] = ns_desc(bbase + (ch * tsp + 2 * sp) * (WV_NJ * 16), WV_NJ * 16, 128);
            }
            const int hs = tsp / 2;
            long long w_acc = 0, w_full = 0, w_iss = 0;
            for (int i = 0; i < ntile; ++i) {
                const int s = i % WV_ST, b = i % WV_NACC;
                const long long k0 = clock64();
                if (i >= WV_NACC) mbar_wait(su(&tempty[b]), ((i / WV_NACC) - 1) & 1);
                const long long k1 = clock64();
                mbar_wait(su(&full[s]), (i / WV_ST) & 1);
                w_acc += k1 - k0;
                const long long k2 = clock64();
                w_full += k2 - k1;
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint64_t aoff = static_cast<uint64_t>((s * L.stage_bytes) >> 4);
                const uint32_t d = tmem + b * 16;
#pragma unroll
                for (int k = 0; k < KM; ++k)
                    if ((k / 8) < P.nscr && (k % 8) < hs) mma_i8(d, ad0[k] + aoff, bd[k], idesc, k == 0 ? 0u : 1u);
                mma_commit(su(&empty[s]));
                mma_commit(su(&tfull[b]));
                w_iss += clock64() - k2;
            }
            if (P.tl && P.stats) {
                atomicAdd(&P.stats[22], static_cast<unsigned long long>(w_iss));
                atomicAdd(&P.stats[16], static_cast<unsigned long long>(w_acc));
                atomicAdd(&P.stats[17], static_cast<unsigned long long>(w_full));
            }
        }
    } else if (warp < 6) {  // epilogue: warp w reads TMEM lanes 32 (w % 4) ..
        wv_epilogue(P, A, L, tmem, warp & 3, c0, ntile, lists, cnts, thrs, ovs, sthr, kqs, tfull, tempty);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    phase(2);
    cl.sync();  // every list of the cluster is final
    phase(3);

    // ---- post-scan: the placements this CTA owns, one warp each --------------
    WvWarp& W = reinterpret_cast<WvWarp*>(ring)[warp];
    for (int j = rank + CS * warp; j < njs && !(A.dbg & 2); j += CS * 8) {
        const bool ok = wv_post<CS>(P, js[j], job0 + js0 + j, j, kqs[j], lists, cnts, ovs, W);
        if (!ok && lane == 0) atomicOr(&fbm[0], 1 << j);
    }
    __syncthreads();
    cl.sync();  // remote list reads done; fallback bits published
    int fb = 0;
#pragma unroll
    for (int r = 0; r < CS; ++r) fb |= *cl.map_shared_rank(fbm, r);
    cl.sync();  // no CTA leaves while another reads its shared memory
    phase(4);

    // ---- fallback (tie storms): full score rows, then the generic select -----
    if (fb) {
        const int Tc = P.Tc;
        const size_t nc = static_cast<size_t>(P.hc) * P.wc;
        for (int j = 0; j < njs; ++j) {
            if (!((fb >> j) & 1)) continue;
            const int slot = js0 + j;
            int32_t* row = P.scores + static_cast<size_t>(slot) * P.sld;
            for (int e = tid; e < (c1 - c0) * P.out_h; e += WV_T) {
                const int c = c0 + e / P.out_h, r = e - (e / P.out_h) * P.out_h;
                const int mb = r >> 7, rl = r & 127;
                const int8_t* st = A.strips + (static_cast<size_t>(c) * A.nmb + mb) * L.stage_bytes;
                int acc = 0;
                for (int f = 0; f < P.nscr; ++f)
                    for (int s = 0; s < tsp; ++s) {
                        const int4 a = *reinterpret_cast<const int4*>(st + (f * WV_SR + rl + s) * 16);
                        const int4 w = *reinterpret_cast<const int4*>(Bs + ((f * tsp + s) * WV_NJ + j) * 16);
                        acc = __dp4a(a.x, w.x, acc);
                        acc = __dp4a(a.y, w.y, acc);
                        acc = __dp4a(a.z, w.z, acc);
                        acc = __dp4a(a.w, w.w, acc);
                    }
                row[r * P.out_w + c] = acc;
            }
            if (j % CS == rank) {  // the owner stages the placement's fp64 template
                const Job& jb = js[j];
                const int32_t* src = P.src + static_cast<size_t>(jb.real) * (P.wh / P.B) * P.swc;
                double* tm = P.tm64 + static_cast<size_t>(slot) * P.nch * Tc * Tc;
                for (int c = tid; c < Tc * Tc; c += WV_T) {
                    const int s = c / Tc, t = c - s * Tc;
                    int t0, t1;
                    mask_row_run(jb.shape, jb.vleft, jb.htop, Tc, P.OVc, s, t0, t1);
                    const bool in = t >= t0 && t < t1;
                    const int sb = in ? src[static_cast<size_t>(jb.top / P.B + s) * P.swc + jb.left / P.B + t] : 0;
                    for (int ch = 0; ch < P.nch; ++ch) tm[ch * Tc * Tc + c] = in ? P.ti64[ch * nc + sb] : 0.0;
                }
            }
        }
        __threadfence();
        cl.sync();  // every column range of the rows is written
        SimParams Q = P;
        Q.tmax = nullptr;
        for (int j = rank; j < njs; j += CS)
            if ((fb >> j) & 1) {
                __syncthreads();
                wv_fallback(Q, jobs, job0, js0 + j, ring);
                if (tid == 0 && P.stats) atomicAdd(&P.stats[2], 1ull);
            }
    }
    __syncthreads();
    phase(5);
    if (P.tl && P.stats && tid == 0) atomicAdd(&P.stats[14], 1ull);
    tl_mark(P.tl, 1);
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(WV_NACC * 16));
}

__global__ void strips_kernel(const float* __restrict__ scr, int nscr, int hc, int wc, int out_w, int nmb,
                              int8_t* __restrict__ out) {
    // out[c][mb][ch][WV_SR][16] = plane[ch][mb * 128 + row][c + t], 0 outside
    const size_t per = static_cast<size_t>(nscr) * WV_SR * 16;
    const size_t total = static_cast<size_t>(out_w) * nmb * per;
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t cm = i / per, rem = i - cm * per;
        const int c = static_cast<int>(cm / nmb), mb = static_cast<int>(cm - static_cast<size_t>(c) * nmb);
        const int ch = static_cast<int>(rem / (WV_SR * 16)), rr = static_cast<int>(rem % (WV_SR * 16));
        const int row = mb * 128 + rr / 16, col = c + rr % 16;
        int8_t v = 0;
        if (row < hc && col < wc) v = static_cast<int8_t>(__float2int_rn(scr[(static_cast<size_t>(ch) * hc + row) * wc + col]));
        out[i] = v;
    }
}

}  // namespace

int wave_max_cs() { return WV_MAXCS; }
int wave_jobs_per_set() { return WV_NJ; }

bool wave_supported(int nscr, int Tc, int nch, int K, int T, int OV) {
    if (nscr < 1 || nscr > 4 || Tc > 16 || Tc < 1 || K > WV_KMAX || K < 1 || nch * Tc > 64) return false;
    return wv_layout(nscr, Tc, nch, K, T, OV).total <= 227 * 1024;
}

const int8_t* ti_strips(ccw_ti* ti, int Tc, cudaStream_t st, int* nmb_out) {
    const int out_h = ti->hc - Tc + 1, out_w = ti->wc - Tc + 1;
    const int nmb = (out_h + 127) / 128;
    *nmb_out = nmb;
    const int key = -1000 - Tc;  // (shares the per-TI cache map with the im2col, keyed apart)
    auto it = ti->im2col.find(key);
    if (it != ti->im2col.end()) return it->second;
    const size_t bytes = static_cast<size_t>(out_w) * nmb * ti->nscr * WV_SR * 16;
    int8_t* X = static_cast<int8_t*>(cache_alloc(ti->device, bytes));
    strips_kernel<<<static_cast<unsigned>(std::min<size_t>((bytes + 255) / 256, 148 * 8)), 256, 0, st>>>(
        ti->d_scr, ti->nscr, ti->hc, ti->wc, out_w, nmb, X);
    CCW_CUDA(cudaGetLastError());
    ti->im2col[key] = X;
    return X;
}

int wave_pick_cs(const SimParams& P, int nj, int want) {
    const int sets = (nj + WV_NJ - 1) / WV_NJ;
    if (want > 0) return std::max(1, std::min(WV_MAXCS, want));
    int cs = WV_MAXCS;
    while (cs > 1 && sets * cs > 148) --cs;
    (void)P;
    return cs;
}

// Once per simulate call: the kernels' dynamic shared-memory ceiling.
void wave_prepare(const SimParams& P) {
    const int bytes = static_cast<int>(wv_layout(P.nscr, P.Tc, P.nch, P.K, P.T, P.OV).total);
    CCW_CUDA(cudaFuncSetAttribute(wave_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    CCW_CUDA(cudaFuncSetAttribute(wave_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    CCW_CUDA(cudaFuncSetAttribute(wave_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    CCW_CUDA(cudaFuncSetAttribute(wave_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

void launch_wave(const SimParams& P, const Job* jobs, int job0, int nj, const int8_t* strips, int nmb, int cs,
                 cudaStream_t st) {
    const WvLayout L = wv_layout(P.nscr, P.Tc, P.nch, P.K, P.T, P.OV);
    WaveArgs A{};
    A.strips = strips;
    A.nmb = nmb;
    if (const char* e = debug_env("CCW_WAVE_DBG")) A.dbg = atoi(e);
    const int sets = (nj + WV_NJ - 1) / WV_NJ;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(sets * cs));
    cfg.blockDim = dim3(WV_T);
    cfg.dynamicSmemBytes = L.total;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = static_cast<unsigned>(cs);
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    if (debug_env("CCW_WAVE_NOPDL")) {
        at[0] = at[1];
        cfg.numAttrs = 1;
    }
    auto go = [&](auto kern) { CCW_CUDA(cudaLaunchKernelEx(&cfg, kern, P, jobs, job0, nj, A)); };
    switch (cs) {
        case 1: go(wave_kernel<1>); break;
        case 2: go(wave_kernel<2>); break;
        case 3: go(wave_kernel<3>); break;
        default: go(wave_kernel<4>); break;
    }
}

}  // namespace ccwgpu
