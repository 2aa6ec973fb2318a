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

#include "select_common.cuh"

namespace cg = cooperative_groups;

namespace ccwgpu {

namespace {

constexpr int WV_M = 128;     // placements per cluster (the MMA's M, one TMEM lane each)
constexpr int WV_T = 256;     // threads per CTA (= SEL_T for the fallback)
constexpr int WV_NB = 128;    // positions per strip block (the MMA's N <= 128)
constexpr int WV_SR = WV_NB + 16;  // strip rows: a block of positions + up to 16 template rows
constexpr int WV_LC = 32;     // list capacity per placement and CTA
constexpr int WV_LS = WV_LC + 1;  // list row stride (int2): spreads the lanes' rows over the banks
constexpr int WV_ST = 4;      // strip ring stages
constexpr int WV_NACC = 4;    // TMEM accumulators (WV_NB columns each)
constexpr int WV_GCAP = 128;  // equal-score group members rescored per warp
constexpr int WV_RS = 256;    // (member, run) partial sums per chunk
constexpr int WV_MAXCS = 16;  // CTAs per cluster (position column ranges)
constexpr int WV_KMAX = 8;    // largest K (and K') this path takes

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
    int stage_bytes, tsp, nb;
    size_t u, a, lists, cnt, drop, gthr, fb, jobs, bar, total;
};

// nb: positions per strip block (a multiple of 16, <= WV_NB)
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
    L.a = o;  // A operand (weights): [nscr * tsp core-matrix columns][128 placements][16 bytes]
    o += static_cast<size_t>(nscr) * L.tsp * WV_M * 16;
    L.lists = o;  // [128 placements][WV_LS] (score, position)
    o += static_cast<size_t>(WV_M) * WV_LS * sizeof(int2);
    L.cnt = o;  // [128] list lengths
    o += WV_M * sizeof(int);
    L.drop = o;  // [128] largest value dropped from the list (INT_MIN: none)
    o += WV_M * sizeof(int);
    L.gthr = o;  // [128] (rank 0) the cluster's shared lower bound of S_K'
    o += WV_M * sizeof(int);
    L.fb = o;  // fallback bits of the placements this CTA owns
    o += 4 * sizeof(int);
    L.jobs = o;  // the placements this CTA owns (j = rank + CS * i)
    o += (WV_M / 2) * sizeof(Job);
    o = (o + 15) & ~static_cast<size_t>(15);
    L.bar = o;  // full[ST], empty[ST], tfull[NACC], tempty[NACC], tmem slot
    o += (2 * WV_ST + 2 * WV_NACC + 1) * sizeof(uint64_t) + 16;
    L.total = o + 1024;  // (base alignment slack)
    return L;
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
// the ranking up to rank K' (matcher.hpp:177-204), the pick, the paste.
// Returns false when the placement needs the fallback.
template <int CS>
__device__ __noinline__ bool wv_post(const SimParams& P, const Job& jb, int gj, int j, const int2* lists,
                                     const int* cnts, const int* drops, WvWarp& W) {
    const int lane = threadIdx.x & 31;
    cg::cluster_group cl = cg::this_cluster();
    int v[CS], p[CS];
    int dmax = INT_MIN;  // largest value any list dropped: the lists are complete above it
#pragma unroll
    for (int r = 0; r < CS; ++r) {
        const int2* rl = cl.map_shared_rank(lists, r) + j * WV_LS;
        const int n = *(cl.map_shared_rank(cnts, r) + j);
        dmax = max(dmax, *(cl.map_shared_rank(drops, r) + j));
        const int2 e = lane < n ? rl[lane] : make_int2(INT_MIN, -1);
        v[r] = e.x;
        p[r] = e.y;
    }
    const int pick = jb.pick;
    const int need = pick >= 0 ? min(pick + 1, P.K) : P.K;
    int R = 0;
    int above = 0, cur = INT_MAX;
    bool runs_ready = false;
    while (above < need) {
        int a = INT_MIN;
#pragma unroll
        for (int r = 0; r < CS; ++r)
            if (p[r] >= 0 && v[r] < cur) a = max(a, v[r]);
        const int m = __reduce_max_sync(0xffffffffu, a);
        if (m == INT_MIN) {  // fewer listed windows than `need`
            if (dmax != INT_MIN) return false;
            break;  // (npos < K)
        }
        if (m <= dmax) return false;  // windows of this score may have been dropped: the generic select
        int g = 0;
#pragma unroll
        for (int r = 0; r < CS; ++r) g += __popc(__ballot_sync(0xffffffffu, p[r] >= 0 && v[r] == m));
        cur = m;
        if (pick >= 0 && above + g <= pick) {  // ranks before the pick: order irrelevant
            above += g;
            continue;
        }
        if (g == 1) {
#pragma unroll
            for (int r = 0; r < CS; ++r)
                if (p[r] >= 0 && v[r] == m) W.tidx[above] = p[r];
            above += 1;
            __syncwarp();
            continue;
        }
        if (g > WV_GCAP) return false;  // a tie storm: the generic select
        int o = 0;
#pragma unroll
        for (int r = 0; r < CS; ++r) {
            const unsigned bl = __ballot_sync(0xffffffffu, p[r] >= 0 && v[r] == m);
            if (bl & (1u << lane)) W.gpos[o + __popc(bl & ((1u << lane) - 1))] = p[r];
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

// OR prep of the placements this CTA owns (j = rank + CS * i): their int8
// screen weights (prep_src_job's arithmetic), one (placement, template row)
// per thread, as 16-byte rows of the set's A operand in global memory
// (A.wglob, the shared-memory layout); every CTA of the cluster then bulk-loads
// the whole operand.  Rows past Tc and absent placements are written as zeros,
// so every row is written exactly once.
template <int CS>
__device__ __noinline__ void wv_prep(const SimParams& P, const WaveArgs& A, const Job* js, int njs, int rank,
                                     int8_t* wg, int tsp) {
    const int Tc = P.Tc, B = P.B;
    const size_t nc = static_cast<size_t>(P.hc) * P.wc;
    constexpr int NOWN = WV_M / CS;
    for (int it = threadIdx.x; it < NOWN * tsp; it += WV_T) {
        const int i = it / tsp, s = it - i * tsp;
        const int j = rank + CS * i;
        int w[4][16];
#pragma unroll
        for (int f = 0; f < 4; ++f)
#pragma unroll
            for (int t = 0; t < 16; ++t) w[f][t] = 0;
        if (j < njs && s < Tc) {
            const Job& jb = js[i];
            int t0, t1;
            mask_row_run(jb.shape, jb.vleft, jb.htop, Tc, P.OVc, s, t0, t1);
            const int32_t* srow = P.src + static_cast<size_t>(jb.real) * (P.wh / B) * P.swc +
                                  static_cast<size_t>(jb.top / B + s) * P.swc + jb.left / B;
            int sb[16];
#pragma unroll
            for (int t = 0; t < 16; ++t) sb[t] = t >= t0 && t < t1 && !(A.dbg & 1) ? srow[t] : -1;
            float n[4][16];
#pragma unroll
            for (int f = 0; f < 4; ++f)
#pragma unroll
                for (int t = 0; t < 16; ++t) n[f][t] = f < P.nscr && sb[t] >= 0 ? P.tiscr[f * nc + sb[t]] : 0.f;
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                if (t < t0 || t >= t1) continue;
                int last = B * B;
#pragma unroll
                for (int f = 0; f < 4; ++f)
                    if (f < P.nscr) last -= static_cast<int>(n[f][t]);
#pragma unroll
                for (int f = 0; f < 4; ++f) {
                    const int c = static_cast<int>(n[f][t]);
                    w[f][t] = P.mode == 0 ? c - last : c;
                }
            }
        }
#pragma unroll
        for (int f = 0; f < 4; ++f) {
            if (f >= P.nscr) break;
            int4 row;
            row.x = (w[f][0] & 255) | ((w[f][1] & 255) << 8) | ((w[f][2] & 255) << 16) | (w[f][3] << 24);
            row.y = (w[f][4] & 255) | ((w[f][5] & 255) << 8) | ((w[f][6] & 255) << 16) | (w[f][7] << 24);
            row.z = (w[f][8] & 255) | ((w[f][9] & 255) << 8) | ((w[f][10] & 255) << 16) | (w[f][11] << 24);
            row.w = (w[f][12] & 255) | ((w[f][13] & 255) << 8) | ((w[f][14] & 255) << 16) | (w[f][15] << 24);
            *reinterpret_cast<int4*>(wg + (static_cast<size_t>(f * tsp + s) * WV_M + j) * 16) = row;
        }
    }
}

// The epilogue of one TMEM lane quarter (one warp, one placement per thread):
// every tile's scores of its placement, a running top-K' of the values seen
// (sorted, in registers) whose K'-th entry is the list threshold, and the
// list of (score, position) at or above it in shared memory.  The cluster
// shares the thresholds (gthr at rank 0: the max over CTAs of their K'-th
// largest, still a lower bound of S_K'), so after a CTA's first tile a
// 16-value chunk is almost always dismissed by its maximum alone.
__device__ __forceinline__ void wv_insert(int val, int (&top)[WV_KMAX], int kq) {
    int x = val;
#pragma unroll
    for (int k = 0; k < WV_KMAX; ++k)
        if (k < kq && x > top[k]) {
            const int y = top[k];
            top[k] = x;
            x = y;
        }
}

// A full list: the K'-th largest of its windows (top rebuilt from them)
// raises the threshold; a tie group at it that still does not fit is dropped
// and the threshold moves past it (the post-scan checks the dropped value).
// Returns (length, threshold, dropped value).
__device__ __noinline__ int4 wv_make_room(int2* my, int cnt, int kq, int thr, int drop) {
    // K'-th largest (with multiplicity) of the listed scores: rounds of "largest
    // below the previous round", each one pass over the list
    int cur = INT_MAX, acc = 0, kth = INT_MIN;
    for (int r = 0; r < kq; ++r) {
        int m = INT_MIN, c = 0;
        for (int e = 0; e < cnt; ++e) {
            const int x = my[e].x;
            if (x < cur && x > m) {
                m = x;
                c = 1;
            } else if (x == m) {
                ++c;
            }
        }
        if (m == INT_MIN) break;
        acc += c;
        if (acc >= kq) {
            kth = m;
            break;
        }
        cur = m;
    }
    thr = max(thr, kth);
    int n2 = 0;
    for (int e = 0; e < cnt; ++e) {
        const int2 x = my[e];
        if (x.x >= thr) my[n2++] = x;
    }
    if (n2 > WV_LC - 16) {  // a tie group at the threshold leaves no room: drop it
        drop = max(drop, thr);
        int n3 = 0;
        for (int e = 0; e < n2; ++e) {
            const int2 x = my[e];
            if (x.x > thr) my[n3++] = x;
        }
        n2 = n3;
        thr = thr + 1;
    }
    return make_int4(n2, thr, drop, kth);
}

__device__ __noinline__ void wv_epilogue(const SimParams& P, const WaveArgs& A, const WvLayout& L, uint32_t tmem, int q,
                                         int c0, int ntile, int njs, const Job* __restrict__ jobs, int gj0, int2* lists,
                                         int* cnts, int* drops, int* gthr, uint64_t* tfull, uint64_t* tempty) {
    const int lane = threadIdx.x & 31;
    const int j = q * 32 + lane;
    cg::cluster_group cl = cg::this_cluster();
    int* gt = cl.map_shared_rank(gthr, 0) + j;  // the cluster's shared bound for this placement
    int kq = 0;
    if (j < njs) {
        const int pick = jobs[gj0 + j].pick;
        kq = pick >= 0 ? min(pick + 1, P.K) : P.K;
    }
    int top[WV_KMAX];
#pragma unroll
    for (int k = 0; k < WV_KMAX; ++k) top[k] = INT_MIN;
    // thr: windows below it are never listed; a lower bound of S_K' (this
    // CTA's K'-th largest so far, the cluster's bound, or past a dropped tie)
    int thr = kq > 0 ? INT_MIN : INT_MAX, drop = INT_MIN, cnt = 0, kpub = INT_MIN;
    int2* my = lists + j * WV_LS;
    long long e_wait = 0, e_work = 0, ncomp = 0, t_ld = 0, t_ins = 0, t_flt = 0, t_st = 0, t_gt = 0, t_pub = 0;
    auto kth_of = [&]() {
        int t = INT_MIN;
#pragma unroll
        for (int k = 0; k < WV_KMAX; ++k)
            if (k == kq - 1) t = top[k];
        return t;
    };
    for (int i = 0; i < ntile; ++i) {
        const int b = i % WV_NACC;
        const long long k0 = clock64();
        mbar_wait(su(&tfull[b]), (i / WV_NACC) & 1);
        const long long k1 = clock64();
        e_wait += k1 - k0;
        long long q0 = clock64();
        if (i > 0 && kq > 0 && !(A.dbg & 8)) thr = max(thr, *gt);  // the other CTAs' bounds
        t_gt += clock64() - q0;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int c = c0 + i / A.nmb, mb = i - (i / A.nmb) * A.nmb;
        const int r0 = mb * A.nb;
        const uint32_t tb = tmem + (static_cast<uint32_t>(q * 32) << 16) + b * WV_NB;
        for (int ch = 0; ch < A.nb; ch += 16) {
            uint32_t vv[16];
            long long q1 = clock64();
            ldtm16(tb + ch, vv);
            t_ld += clock64() - q1;
            q1 = clock64();
            if (ch + 16 >= A.nb) {  // the accumulator is drained: the MMA may reuse it
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(su(&tempty[b]));
            }
            const int nv = min(16, P.out_h - (r0 + ch));  // valid rows of the chunk
            int cm0 = INT_MIN, cm1 = INT_MIN, cm2 = INT_MIN, cm3 = INT_MIN;
#pragma unroll
            for (int u = 0; u < 16; u += 4) {
                cm0 = max(cm0, u < nv ? static_cast<int>(vv[u]) : INT_MIN);
                cm1 = max(cm1, u + 1 < nv ? static_cast<int>(vv[u + 1]) : INT_MIN);
                cm2 = max(cm2, u + 2 < nv ? static_cast<int>(vv[u + 2]) : INT_MIN);
                cm3 = max(cm3, u + 3 < nv ? static_cast<int>(vv[u + 3]) : INT_MIN);
            }
            const int cm = max(max(cm0, cm1), max(cm2, cm3));
            const bool anyc = __any_sync(0xffffffffu, cm >= thr);
            t_flt += clock64() - q1;
            if (!anyc) continue;
            const long long q2 = clock64();
            // list the chunk's windows at or above the threshold
            unsigned m = 0;
#pragma unroll
            for (int u = 0; u < 16; ++u) m |= (u < nv && static_cast<int>(vv[u]) >= thr ? 1u : 0u) << u;
            if (m && cnt + __popc(m) > WV_LC) {
                ++ncomp;
                const int4 st = wv_make_room(my, cnt, kq, thr, drop);
                cnt = st.x;
                thr = st.y;
                drop = st.z;
                kpub = max(kpub, st.w);
                m = 0;
#pragma unroll
                for (int u = 0; u < 16; ++u) m |= (u < nv && static_cast<int>(vv[u]) >= thr ? 1u : 0u) << u;
                if (cnt + __popc(m) > WV_LC) {  // ties at the raised threshold still do not fit
                    drop = max(drop, thr);
                    thr = thr + 1;
                    m = 0;
#pragma unroll
                    for (int u = 0; u < 16; ++u) m |= (u < nv && static_cast<int>(vv[u]) >= thr ? 1u : 0u) << u;
                }
            }
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if ((m >> u) & 1u) my[cnt + __popc(m & ((1u << u) - 1))] = make_int2(static_cast<int>(vv[u]), (r0 + ch + u) * P.out_w + c);
            cnt += __popc(m);
            t_st += clock64() - q2;
        }
        const long long q3 = clock64();
        if (kq > 0 && !(A.dbg & 8)) {  // publish this CTA's bound (a K'-th largest it has seen)
            if (kpub != INT_MIN) atomicMax(gt, kpub);
        }
        t_pub += clock64() - q3;
        e_work += clock64() - k1;
    }
    cnts[j] = cnt;
    drops[j] = drop;
    if (P.tl && P.stats && lane == 0 && q == 0) {
        atomicAdd(&P.stats[18], static_cast<unsigned long long>(e_wait));
        atomicAdd(&P.stats[19], static_cast<unsigned long long>(e_work));
        atomicAdd(&P.stats[20], static_cast<unsigned long long>(ncomp));
        atomicAdd(&P.stats[21], static_cast<unsigned long long>(ntile));
        atomicAdd(&P.stats[25], static_cast<unsigned long long>(t_ld));
        atomicAdd(&P.stats[26], static_cast<unsigned long long>(t_ins));
        atomicAdd(&P.stats[27], static_cast<unsigned long long>(t_flt));
        atomicAdd(&P.stats[28], static_cast<unsigned long long>(t_st));
        atomicAdd(&P.stats[29], static_cast<unsigned long long>(t_gt));
        atomicAdd(&P.stats[30], static_cast<unsigned long long>(t_pub));
    }
}

// The generic select of one placement (out of line: the wave kernel's hot
// code stays small).
__device__ __noinline__ void wv_fallback(const SimParams& Q, const Job* __restrict__ jobs, int job0, int slot,
                                         unsigned char* sm) {
    select_paste_body(Q, jobs, job0, slot, 1, sm);
}

template <int CS>
__global__ void __launch_bounds__(WV_T, 1)
    wave_kernel(const __grid_constant__ SimParams P, const Job* __restrict__ jobs, int job0, int nj, WaveArgs A) {
    extern __shared__ __align__(1024) uint8_t wv_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(wv_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const WvLayout L = wv_layout(P.nscr, P.Tc, P.nch, P.K, P.T, P.OV);
    uint8_t* ring = sm + L.u;
    int8_t* Abuf = reinterpret_cast<int8_t*>(sm + L.a);
    int2* lists = reinterpret_cast<int2*>(sm + L.lists);
    int* cnts = reinterpret_cast<int*>(sm + L.cnt);
    int* drops = reinterpret_cast<int*>(sm + L.drop);
    int* gthr = reinterpret_cast<int*>(sm + L.gthr);
    int* fbm = reinterpret_cast<int*>(sm + L.fb);
    Job* js = reinterpret_cast<Job*>(sm + L.jobs);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + L.bar);
    uint64_t* empty = full + WV_ST;
    uint64_t* tfull = empty + WV_ST;
    uint64_t* tempty = tfull + WV_NACC;
    uint64_t* abar = tempty + WV_NACC;  // the A operand landed
    uint32_t* tslot = reinterpret_cast<uint32_t*>(abar + 1);

    cg::cluster_group cl = cg::this_cluster();
    const int rank = static_cast<int>(cl.block_rank());
    const int set = static_cast<int>(blockIdx.x) / CS;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int js0 = set * WV_M;                      // first job slot of the set
    const int njs = min(WV_M, nj - js0);             // placements of this set
    const int cpc = (P.out_w + CS - 1) / CS;         // columns per CTA
    const int c0 = min(P.out_w, rank * cpc), c1 = min(P.out_w, c0 + cpc);
    const int ntile = (c1 - c0) * A.nmb;
    const int tsp = L.tsp;
    constexpr int NOWN = WV_M / CS;

    const long long pc0 = clock64();
    auto phase = [&](int k) {  // debug timeline runs only: cycles from CTA start per phase, summed
        if (P.tl && P.stats && tid == 0) atomicAdd(&P.stats[k < 6 ? 8 + k : 24], static_cast<unsigned long long>(clock64() - pc0));
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
        mbar_init(su(abar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su(tslot)), "n"(WV_NACC * WV_NB));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid < NOWN) {
        const int j = rank + CS * tid;
        if (j < njs) js[tid] = jobs[job0 + js0 + j];
    }
    if (tid < 4) fbm[tid] = 0;
    if (tid < WV_M) gthr[tid] = INT_MIN;
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

    const int abytes = P.nscr * tsp * WV_M * 16;
    int8_t* wg = A.wglob + static_cast<size_t>(set) * abytes;
    wv_prep<CS>(P, A, js, njs, rank, wg, tsp);
    asm volatile("fence.proxy.async.global;" ::: "memory");  // (generic writes -> the bulk copy's async proxy)
    phase(6);
    cl.sync();  // every row of the set's A operand is in global memory (gthr initialised too)
    if (tid == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        mbar_expect_tx(su(abar), abytes);
        for (int o = 0; o < abytes; o += 32768)
            bulk_load(su(Abuf + o), wg + o, min(32768, abytes - o), su(abar));
    }
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
        if (lane == 0) {  // single-thread MMA issuer: D[placement][position] += W[placement][k] * strip[position][k]
            const uint32_t idesc = wv_idesc(WV_M, A.nb);
            constexpr int KM = 16;  // MMAs per tile: nscr * tsp / 2 (<= 16: K <= 512 bytes)
            uint64_t ad[KM], bd0[KM];
            const uint32_t abase = su(Abuf), bbase = su(ring);
            const int hs = tsp / 2;
#pragma unroll
            for (int k = 0; k < KM; ++k) {
                const int ch = k / hs, sp = k - ch * hs;
                ad[k] = ns_desc(abase + (ch * tsp + 2 * sp) * (WV_M * 16), WV_M * 16, 128);
                bd0[k] = ns_desc(bbase + ch * (WV_SR * 16) + sp * 32, 16, 128);
            }
            const int nk = P.nscr * hs;
            mbar_wait(su(abar), 0);
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
                const uint64_t boff = static_cast<uint64_t>((s * L.stage_bytes) >> 4);
                const uint32_t d = tmem + b * WV_NB;
#pragma unroll
                for (int k = 0; k < KM; ++k)
                    if (k < nk) mma_i8(d, ad[k], bd0[k] + boff, idesc, k == 0 ? 0u : 1u);
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
    } else if (warp < 6) {  // epilogue: warp w reads TMEM lanes 32 (w % 4) .. = placements
        wv_epilogue(P, A, L, tmem, warp & 3, c0, ntile, njs, jobs, job0 + js0, lists, cnts, drops, gthr, tfull, tempty);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    phase(2);
    cl.sync();  // every list of the cluster is final
    phase(3);

    // ---- post-scan: the placements this CTA owns, one warp each --------------
    WvWarp& W = reinterpret_cast<WvWarp*>(ring)[warp];
    for (int i = warp; i < NOWN && !(A.dbg & 2); i += 8) {
        const int j = rank + CS * i;
        if (j >= njs) break;
        const bool ok = wv_post<CS>(P, js[i], job0 + js0 + j, j, lists, cnts, drops, W);
        if (!ok && lane == 0) atomicOr(&fbm[i >> 5], 1 << (i & 31));
    }
    __syncthreads();
    cl.sync();  // remote list reads done; fallback bits published
    int fb[CS];
    bool anyfb = false;
#pragma unroll
    for (int r = 0; r < CS; ++r) {
        fb[r] = *cl.map_shared_rank(fbm, r);
        anyfb |= fb[r] != 0;
    }
    cl.sync();  // no CTA leaves while another reads its shared memory
    phase(4);

    // ---- fallback (tie storms): full score rows, then the generic select -----
    if (anyfb) {
        mbar_wait(su(abar), 0);
        const int Tc = P.Tc;
        const size_t nc = static_cast<size_t>(P.hc) * P.wc;
        for (int r = 0; r < CS; ++r)
            for (int i = 0; i < NOWN; ++i) {
                if (!((fb[r] >> i) & 1)) continue;
                const int j = r + CS * i, slot = js0 + j;
                int32_t* row = P.scores + static_cast<size_t>(slot) * P.sld;
                for (int e = tid; e < (c1 - c0) * P.out_h; e += WV_T) {
                    const int c = c0 + e / P.out_h, rr = e - (e / P.out_h) * P.out_h;
                    const int mb = rr / A.nb, rl = rr - mb * A.nb;
                    const int8_t* st = A.strips + (static_cast<size_t>(c) * A.nmb + mb) * L.stage_bytes;
                    int acc = 0;
                    for (int f = 0; f < P.nscr; ++f)
                        for (int s = 0; s < tsp; ++s) {
                            const int4 a = *reinterpret_cast<const int4*>(st + (f * WV_SR + rl + s) * 16);
                            const int4 w = *reinterpret_cast<const int4*>(Abuf + (static_cast<size_t>(f * tsp + s) * WV_M + j) * 16);
                            acc = __dp4a(a.x, w.x, acc);
                            acc = __dp4a(a.y, w.y, acc);
                            acc = __dp4a(a.z, w.z, acc);
                            acc = __dp4a(a.w, w.w, acc);
                        }
                    row[rr * P.out_w + c] = acc;
                }
                if (r == rank) {  // the owner stages the placement's fp64 template
                    const Job& jb = js[i];
                    const int32_t* src = P.src + static_cast<size_t>(jb.real) * (P.wh / P.B) * P.swc;
                    double* tm = P.tm64 + static_cast<size_t>(slot) * P.nch * Tc * Tc;
                    for (int cc = tid; cc < Tc * Tc; cc += WV_T) {
                        const int s = cc / Tc, t = cc - s * Tc;
                        int t0, t1;
                        mask_row_run(jb.shape, jb.vleft, jb.htop, Tc, P.OVc, s, t0, t1);
                        const bool in = t >= t0 && t < t1;
                        const int sb = in ? src[static_cast<size_t>(jb.top / P.B + s) * P.swc + jb.left / P.B + t] : 0;
                        for (int chn = 0; chn < P.nch; ++chn) tm[chn * Tc * Tc + cc] = in ? P.ti64[chn * nc + sb] : 0.0;
                    }
                }
            }
        __threadfence();
        cl.sync();  // every column range of the rows is written
        SimParams Q = P;
        Q.tmax = nullptr;
        for (int i = 0; i < NOWN; ++i)
            if ((fb[rank] >> i) & 1) {
                __syncthreads();
                wv_fallback(Q, jobs, job0, js0 + rank + CS * i, ring);
                if (tid == 0 && P.stats) atomicAdd(&P.stats[2], 1ull);
            }
    }
    __syncthreads();
    phase(5);
    if (P.tl && P.stats && tid == 0) atomicAdd(&P.stats[14], 1ull);
    tl_mark(P.tl, 1);
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(WV_NACC * WV_NB));
}

__global__ void strips_kernel(const float* __restrict__ scr, int nscr, int hc, int wc, int out_w, int nmb, int nb,
                              int8_t* __restrict__ out) {
    // out[c][mb][ch][WV_SR][16] = plane[ch][mb * nb + row][c + t], 0 outside
    const size_t per = static_cast<size_t>(nscr) * WV_SR * 16;
    const size_t total = static_cast<size_t>(out_w) * nmb * per;
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t cm = i / per, rem = i - cm * per;
        const int c = static_cast<int>(cm / nmb), mb = static_cast<int>(cm - static_cast<size_t>(c) * nmb);
        const int ch = static_cast<int>(rem / (WV_SR * 16)), rr = static_cast<int>(rem % (WV_SR * 16));
        const int row = mb * nb + rr / 16, col = c + rr % 16;
        int8_t v = 0;
        if (row < hc && col < wc) v = static_cast<int8_t>(__float2int_rn(scr[(static_cast<size_t>(ch) * hc + row) * wc + col]));
        out[i] = v;
    }
}

}  // namespace

int wave_jobs_per_set() { return WV_M; }

bool wave_supported(int nscr, int Tc, int nch, int K, int T, int OV) {
    const int tsp = (Tc + 1) & ~1;
    if (nscr < 1 || nscr > 4 || nscr * tsp > 32 || Tc > 16 || Tc < 1 || K > WV_KMAX || K < 1 || nch * Tc > 64)
        return false;
    return wv_layout(nscr, Tc, nch, K, T, OV).total <= 227 * 1024;
}

// Position blocks of a column: nb positions (a multiple of 16, <= 128) each.
static void wave_blocks(int out_h, int* nmb, int* nb) {
    *nmb = (out_h + WV_NB - 1) / WV_NB;
    const int per = (out_h + *nmb - 1) / *nmb;
    *nb = (per + 15) & ~15;
}

const int8_t* ti_strips(ccw_ti* ti, int Tc, cudaStream_t st, int* nmb_out, int* nb_out) {
    const int out_h = ti->hc - Tc + 1, out_w = ti->wc - Tc + 1;
    int nmb, nb;
    wave_blocks(out_h, &nmb, &nb);
    *nmb_out = nmb;
    *nb_out = nb;
    const int key = -1000 - Tc;  // (shares the per-TI cache map with the im2col, keyed apart)
    auto it = ti->im2col.find(key);
    if (it != ti->im2col.end()) return it->second;
    const size_t bytes = static_cast<size_t>(out_w) * nmb * ti->nscr * WV_SR * 16;
    int8_t* X = static_cast<int8_t*>(cache_alloc(ti->device, bytes));
    strips_kernel<<<static_cast<unsigned>(std::min<size_t>((bytes + 255) / 256, 148 * 8)), 256, 0, st>>>(
        ti->d_scr, ti->nscr, ti->hc, ti->wc, out_w, nmb, nb, X);
    CCW_CUDA(cudaGetLastError());
    ti->im2col[key] = X;
    return X;
}

int wave_pick_cs(const SimParams& P, int nj, int want) {
    const int sets = (nj + WV_M - 1) / WV_M;
    if (want == 4 || want == 8 || want == 16) return want;
    (void)P;
    return sets * 16 <= 148 ? 16 : (sets * 8 <= 148 ? 8 : 4);
}

// Once per simulate call: the kernels' dynamic shared-memory ceiling and
// (cluster size 16) the non-portable cluster permission.
void wave_prepare(const SimParams& P) {
    const int bytes = static_cast<int>(wv_layout(P.nscr, P.Tc, P.nch, P.K, P.T, P.OV).total);
    CCW_CUDA(cudaFuncSetAttribute(wave_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    CCW_CUDA(cudaFuncSetAttribute(wave_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    CCW_CUDA(cudaFuncSetAttribute(wave_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    CCW_CUDA(cudaFuncSetAttribute(wave_kernel<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
}

size_t wave_wglob_bytes(const SimParams& P, int nj) {
    const int tsp = (P.Tc + 1) & ~1;
    return static_cast<size_t>((nj + WV_M - 1) / WV_M) * P.nscr * tsp * WV_M * 16;
}

void launch_wave(const SimParams& P, const Job* jobs, int job0, int nj, const int8_t* strips, int nmb, int nb, int cs,
                 int8_t* wglob, cudaStream_t st) {
    const WvLayout L = wv_layout(P.nscr, P.Tc, P.nch, P.K, P.T, P.OV);
    WaveArgs A{};
    A.strips = strips;
    A.nmb = nmb;
    A.nb = nb;
    A.wglob = wglob;
    if (const char* e = debug_env("CCW_WAVE_DBG")) A.dbg = atoi(e);
    const int sets = (nj + WV_M - 1) / WV_M;
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
        case 4: go(wave_kernel<4>); break;
        case 8: go(wave_kernel<8>); break;
        default: go(wave_kernel<16>); break;
    }
}

}  // namespace ccwgpu
