// select.cu -- choosing and pasting each placement's TI patch: the generic
// CTA select (radix threshold, fp64 rescoring, min-cut), the fast select
// (tile-maximum bound, equal-score rescoring) and the bulk tie select.
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
#include "select_common.cuh"

// Rarely executed select paths (fp64 rescoring, batches, shared rescoring,
// the streaming scan).  Measured r1: out of line (-DCCW_COLD_CALLS) they cost
// more in calls and generic shared-memory accesses than they save in
// instruction fetch (config 1: 2.27 -> 2.48 ms), so they stay inlined.
#ifdef CCW_COLD_CALLS
#define CCW_COLD __noinline__
#else
#define CCW_COLD __forceinline__
#endif

namespace ccwgpu {

__global__ void __launch_bounds__(SEL_T) select_paste_kernel(SimParams P,
                                                             const Job* __restrict__ jobs,
                                                             int job0, int use_screen) {
    extern __shared__ __align__(16) unsigned char sel_sm[];
    pdl_trigger();
    pdl_wait();
    select_paste_body(P, jobs, job0, static_cast<int>(blockIdx.x), use_screen, sel_sm);
}

// Candidate-position sharding, after the exchange: merge the S shard lists
// of each placement (xrec, [S][nj][xk]) into the reference's top-K, then
// choose and paste exactly as select_paste_kernel does.  Every rank runs this
// on identical lists, so every rank pastes the same patch.
__global__ void __launch_bounds__(SEL_T) shard_merge_kernel(SimParams P, const Job* __restrict__ jobs,
                                                            int job0, int nshards) {
    extern __shared__ __align__(16) unsigned char sel_sm[];
    const SelLayout L = sel_layout(P.K, P.T, P.OV, P.nch, P.Tc, P.scoring == 1);
    double* redd = reinterpret_cast<double*>(sel_sm + L.redd);
    int* redi = reinterpret_cast<int*>(sel_sm + L.redi);
    double* gkey = reinterpret_cast<double*>(sel_sm + L.gkey);
    int* gidx = reinterpret_cast<int*>(sel_sm + L.gidx);
    double* tkey = reinterpret_cast<double*>(sel_sm + L.tkey);
    int* tidx = reinterpret_cast<int*>(sel_sm + L.tidx);
    uint8_t* exist = sel_sm + L.exist;
    uint8_t* outp = sel_sm + L.outp;
    int16_t* from = reinterpret_cast<int16_t*>(sel_sm + L.from);
    int* dp = reinterpret_cast<int*>(sel_sm + L.dp);
    int* seam = reinterpret_cast<int*>(sel_sm + L.seam);

    pdl_trigger();
    const int gj = job0 + blockIdx.x;
    const Job jb = jobs[gj];
    const int tid = threadIdx.x;
    pdl_wait();
    int fr = jb.fr, fc = jb.fc;
    if (jb.shape != kNone) {
        RunDesc* runs = reinterpret_cast<RunDesc*>(sel_sm + L.runs);
        double* tmpl = reinterpret_cast<double*>(sel_sm + L.tmpl);
        double* rsum = reinterpret_cast<double*>(sel_sm + L.rsum);
        double* rnrm = reinterpret_cast<double*>(sel_sm + L.rnrm);
        const int Tc = P.Tc;
        // the fp64 template and run list, for keys the fast select left out
        const double* tm = P.tm64 + static_cast<size_t>(blockIdx.x) * P.nch * Tc * Tc;
        for (int e = tid; e < P.nch * Tc * Tc; e += SEL_T) tmpl[e] = tm[e];
        int R = 0;
        for (int ch = 0; ch < P.nch; ++ch)
            for (int s = 0; s < Tc; ++s) {
                int t0, t1;
                mask_row_run(jb.shape, jb.vleft, jb.htop, Tc, P.OVc, s, t0, t1);
                if (t1 > t0) {
                    if (tid == 0) runs[R] = {ch, s, t0, t1};
                    ++R;
                }
            }
        __shared__ int nvalid, nabsent;
        int ntop = 0, cnt = 0;
        const int n = nshards * P.xk;
        for (int e0 = 0; e0 < n; e0 += GCAP) {
            const int m = min(GCAP, n - e0);
            if (tid == 0) {
                nvalid = 0;
                nabsent = 0;
            }
            __syncthreads();
            for (int e = tid; e < m; e += SEL_T) {
                const int s = (e0 + e) / P.xk, k = (e0 + e) - s * P.xk;
                const ShardRec r = P.xrec[(static_cast<size_t>(s) * P.xnj + blockIdx.x) * P.xk + k];
                if (r.pos >= 0) {  // (empty slots of a short shard list are skipped; the
                                   //  merge orders by (key, position), so slot order is free)
                    const int at = atomicAdd(&nvalid, 1);
                    gkey[at] = r.key;
                    gidx[at] = r.pos;
                    if (!r.valid) nabsent = 1;
                }
            }
            __syncthreads();
            cnt = nvalid;
            // absent keys: rescore the chunk in the reference's order (the keys
            // that were present are recomputed bit-identically)
            if (nabsent) rescore_group(P, runs, R, tmpl, gidx, gkey, cnt, rsum, rnrm);
            if (cnt > 0) merge_top(gkey, gidx, cnt, tkey, tidx, ntop, P.K, redd, redi);
            __syncthreads();
        }
        const int pos = choose_candidate(P, jb, tidx, ntop, redi);
        fr = (pos / P.out_w) << P.J;
        fc = (pos % P.out_w) << P.J;
        __syncthreads();
    }
    paste_placement(P, jb, gj, fr, fc, exist, outp, from, dp, seam);
}

struct ScanWarp {
    int lv[SC_LC];
    int lp[SC_LC];
    int tq[SC_TB];  // queued qualifying tiles
};

constexpr int kTM = 16;  // tile maxima per lane in registers (512 tiles per placement)

// K-th largest (with multiplicity) of the warp's register-held values (NT
// per lane; rounds of warp max and count, each reduced as a tree so a round's
// dependent chain is log2(NT) deep).
template <int NT>
__device__ __forceinline__ int regs_kth(const int (&tv)[NT], int K) {
    int cur = INT_MAX, acc = 0, mk = INT_MIN;
    for (int round = 0; round < K; ++round) {
        int m[NT], c[NT];
#pragma unroll
        for (int i = 0; i < NT; ++i) m[i] = tv[i] < cur ? tv[i] : INT_MIN;
#pragma unroll
        for (int w = NT / 2; w > 0; w >>= 1)
#pragma unroll
            for (int i = 0; i < w; ++i) m[i] = max(m[i], m[i + w]);
        const int mx = __reduce_max_sync(0xffffffffu, m[0]);
#pragma unroll
        for (int i = 0; i < NT; ++i) c[i] = tv[i] == mx;
#pragma unroll
        for (int w = NT / 2; w > 0; w >>= 1)
#pragma unroll
            for (int i = 0; i < w; ++i) c[i] += c[i + w];
        acc += static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(c[0])));
        mk = mx;
        if (acc >= K || mx == INT_MIN) break;
        cur = mx;
    }
    return mk;
}

// Steps 3-4 of the scan (one warp): the exact K-th score S_K of the list
// W.lv[0, nl) and the candidate positions (>= S_K) into out[].  NV list
// values per lane (NV * 32 >= nl).
template <int NV>
__device__ __forceinline__ int scan_finish_nv(const SimParams& P, const ScanWarp& W, int nl, int mk, int* out,
                                              long long* sclk, int* out_s, int K) {
    const int lane = threadIdx.x & 31;
    // 3. exact S_K from the list (rounds of warp max with multiplicity)
    int lvr[NV];
#pragma unroll
    for (int j2 = 0; j2 < NV; ++j2) {
        const int e = j2 * 32 + lane;
        lvr[j2] = e < nl ? W.lv[e] : INT_MIN;
    }
    const int thr = nl > 0 ? regs_kth<NV>(lvr, K) : mk;
    sclk[3] = clock64();
    // 4. the candidates: every listed window >= S_K
    int* cd = out;
    int cnt = 0;
#pragma unroll
    for (int j2 = 0; j2 < NV; ++j2) {
        const int e = j2 * 32 + lane;
        const bool q = e < nl && lvr[j2] >= thr;
        const unsigned bal = __ballot_sync(0xffffffffu, q);
        if (q) {
            const int o = cnt + __popc(bal & ((1u << lane) - 1));
            cd[o] = W.lp[e];
            if (out_s) out_s[o] = lvr[j2];
        }
        cnt += __popc(bal);
    }
    return cnt;
}

__device__ __forceinline__ int scan_finish(const SimParams& P, const ScanWarp& W, int nl, int mk, int* out,
                                           long long* sclk, int* out_s, int K) {
    return nl <= 32 ? scan_finish_nv<1>(P, W, nl, mk, out, sclk, out_s, K)
                    : scan_finish_nv<SC_LC / 32>(P, W, nl, mk, out, sclk, out_s, K);
}

// Warp-level scan of one placement (every lane of the warp calls it): the
// tile-maximum bound M_K, the (score, position) list of windows >= M_K, the
// exact K-th score S_K and the candidate positions (>= S_K) into out[].
// Returns the candidate count, or -1 when the list overflowed (then every
// window >= mk_out must be rescored -- a superset, still exact).
template <bool S16>
__device__ CCW_COLD int scan_job(const SimParams& P, int slot, ScanWarp& W, int* out, int& mk_out,
                                        long long* sclk, int* out_s = nullptr) {
    const int lane = threadIdx.x & 31;
    const int K = P.K;
    const int32_t* tmx = P.tmax + static_cast<size_t>(slot) * P.ntiles;
    // 1. M_K = K-th largest tile maximum (with multiplicity): a lower bound of
    //    the K-th largest screen score S_K (the K best tiles each hold a
    //    window scoring at least M_K).  Tile maxima stay in registers.
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
        mk = regs_kth<kTM>(tv, K);
    }
    sclk[1] = clock64();
    // 2. every window scoring >= M_K, from the tiles whose maximum reaches it,
    //    into a (score, position) list.  Qualifying tiles are queued across the
    //    32-tile groups and loaded SC_TB per round trip.
    int nl = 0, ntl = 0;
    bool over = false;
    {  // more qualifying tiles than list slots: an overflow before any score is read
        int nq = 0;
        if (regs) {
#pragma unroll
            for (int i = 0; i < kTM; ++i) nq += __popc(__ballot_sync(0xffffffffu, tv[i] != INT_MIN && tv[i] >= mk));
        } else {
            for (int t0 = 0; t0 < P.ntiles; t0 += 32)
                nq += __popc(__ballot_sync(0xffffffffu, t0 + lane < P.ntiles && tmx[t0 + lane] >= mk));
        }
        over = nq > SC_LC;
    }
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
                const int4 a4 = load_score4<S16>(P, slot, p0);
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
    return scan_finish(P, W, nl, mk, out, sclk, out_s, K);
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

struct FastSmem {
    double tm[PK_TMC];
    double rsum[FS_RS];
    double key[SC_LC + kTcQ];
    int cidx[SC_LC + kTcQ];
    int cs[SC_LC];          // the candidates' screen scores
    int tie[SC_LC];         // candidates sharing their screen score (positions)
    int tslot[32];          // candidate -> its entry in tie[] (or -1)
    ScanWarp sw;
    int4 grp[FS_MAXG];      // (channel, first row index | first row << 16, rows, t0 << 8 | len)
    double tkey[kTcQ];
    int tidx[kTcQ];
    double rk[FS_T / 32];
    int ri[FS_T / 32], rp[FS_T / 32], wc[FS_T / 32];
    int misc[8];
    int tqa[32 * kTM];      // cooperative scan: the tiles whose maximum reaches M_K
    int nq, lcnt, lover;    // their count, the list length, list overflow
    int lean;               // lean_scan: 0 not taken, 1 list done, 2 group settled too
    // uniform-window reduction of a large equal-score group (uniform_reduce)
    int utmp[SC_LC];
    signed char ucl[SC_LC], ucl2[SC_LC];
    int urep[16], urs[16], ucnt[2];
#ifdef CCW_DBG_TAIL
    long long dbg[8];
#endif
};

// Large equal-score groups are often windows made entirely of pure blocks of
// one facies (a background region): their fp64 scores are bit-identical
// (P.umap), so one representative per facies is rescored.  Reorders S.tie[0,
// g) so the members to rescore come first and returns their count; the others'
// keys are copied from their representative by uniform_fill.  The ranking is by
// (key, position), so the order of S.tie is free.
constexpr int UD_MIN = 8;
__device__ CCW_COLD int uniform_reduce(const SimParams& P, FastSmem& S, int g, int var) {
    const int tid = threadIdx.x;
    const int8_t* um = P.umap + static_cast<size_t>(var) * P.ustride;
    if (tid < 16) S.urep[tid] = INT_MAX;
    if (tid < 2) S.ucnt[tid] = 0;
    __syncthreads();
    for (int e = tid; e < g; e += FS_T) {
        const int c = __ldg(um + S.tie[e]);
        S.ucl[e] = static_cast<signed char>(c);
        if (c >= 0) atomicMin(&S.urep[c], e);
    }
    __syncthreads();
    for (int e = tid; e < g; e += FS_T) {
        const int c = S.ucl[e];
        if (c < 0 || S.urep[c] == e) {
            const int k = atomicAdd(&S.ucnt[0], 1);
            S.utmp[k] = S.tie[e];
            if (c >= 0) S.urs[c] = k;
        } else {
            const int d = g - 1 - atomicAdd(&S.ucnt[1], 1);
            S.utmp[d] = S.tie[e];
            S.ucl2[d] = static_cast<signed char>(c);
        }
    }
    __syncthreads();
    for (int e = tid; e < g; e += FS_T) S.tie[e] = S.utmp[e];
    const int gr = S.ucnt[0];
    __syncthreads();
    return gr;
}

__device__ CCW_COLD void uniform_fill(FastSmem& S, int gr, int g) {
    for (int j = gr + threadIdx.x; j < g; j += FS_T) S.key[j] = S.key[S.urs[S.ucl2[j]]];
    __syncthreads();
}

// Cooperative scan (ntiles <= 32 * kTM), step 1 on warp 0: M_K (as scan_job)
// and the queue of tiles whose maximum reaches it, in tile order.
template <int NT>
__device__ __forceinline__ void coop_head_nt(const SimParams& P, int slot, FastSmem& S, int K) {
    const int lane = threadIdx.x & 31;
    const int32_t* tmx = P.tmax + static_cast<size_t>(slot) * P.ntiles;
    int tv[NT];
#pragma unroll
    for (int i = 0; i < NT; ++i) {
        const int e = i * 32 + lane;
        tv[i] = e < P.ntiles ? tmx[e] : INT_MIN;
    }
#ifdef CCW_DBG_TAIL
    {
        int sdbg = 0;
#pragma unroll
        for (int i = 0; i < NT; ++i) sdbg ^= tv[i];
        const long long c = clock64();
        if (lane == 0) S.dbg[0] = c + (sdbg == 0x12345 ? 1 : 0);
    }
#endif
    const int mk = regs_kth<NT>(tv, K);
#ifdef CCW_DBG_TAIL
    if (lane == 0) S.dbg[1] = clock64();
#endif
    int nq = 0;
#pragma unroll
    for (int i = 0; i < NT; ++i) {
        const bool q = tv[i] != INT_MIN && tv[i] >= mk;
        const unsigned bal = __ballot_sync(0xffffffffu, q);
        if (q) S.tqa[nq + __popc(bal & ((1u << lane) - 1))] = i * 32 + lane;
        nq += __popc(bal);
    }
    if (lane == 0) {
        S.misc[1] = mk;
        S.nq = nq;
        S.lcnt = 0;
        // every queued tile holds a window >= M_K: more tiles than list slots
        // is an overflow before a single score is read
        S.lover = nq > SC_LC ? 1 : 0;
    }
}

__device__ __forceinline__ void coop_head(const SimParams& P, int slot, FastSmem& S, int K) {
    if (P.ntiles <= 32 * 4)
        coop_head_nt<4>(P, slot, S, K);
    else
        coop_head_nt<kTM>(P, slot, S, K);
}

// Step 2 on every warp: the windows >= M_K of the queued tiles (SC_TB tiles per
// round trip per warp) appended to the shared (score, position) list.  The
// list order is irrelevant: every later ranking is a total order on (S, fp64
// key, index).  Overflow iff the list would exceed SC_LC, as in scan_job.
template <bool S16>
__device__ __forceinline__ void coop_list(const SimParams& P, int slot, FastSmem& S) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nq = S.nq, mk = S.misc[1];
    if (S.lover) return;  // (coop_head: the list cannot fit)
    for (int q0 = wid * SC_TB; q0 < nq; q0 += (FS_T / 32) * SC_TB) {
        int tl[SC_TB], v[SC_TB][4];
#pragma unroll
        for (int u = 0; u < SC_TB; ++u) tl[u] = q0 + u < nq ? S.tqa[q0 + u] : -1;
#ifdef CCW_DBG_TAIL
        if (q0 == 0 && lane == 0) S.dbg[5] = clock64() + (tl[0] == 0x7fffffff);
#endif
#pragma unroll
        for (int u = 0; u < SC_TB; ++u) {
            const int p0 = tl[u] * kTcTile + lane * 4;
#pragma unroll
            for (int i = 0; i < 4; ++i) v[u][i] = INT_MIN;
            if (tl[u] >= 0 && p0 < P.npos) {  // rows are padded to a multiple of 4
                const int4 a4 = load_score4<S16>(P, slot, p0);
                v[u][0] = a4.x;
                v[u][1] = p0 + 1 < P.npos ? a4.y : INT_MIN;
                v[u][2] = p0 + 2 < P.npos ? a4.z : INT_MIN;
                v[u][3] = p0 + 3 < P.npos ? a4.w : INT_MIN;
            }
        }
#ifdef CCW_DBG_TAIL
        if (q0 == 0) {
            int sdbg = 0;
#pragma unroll
            for (int u = 0; u < SC_TB; ++u) sdbg ^= v[u][0];
            const long long cl = clock64();
            if (lane == 0) S.dbg[2] = cl + (sdbg == 0x12345 ? 1 : 0);
        }
#endif
        int c = 0;
#pragma unroll
        for (int u = 0; u < SC_TB; ++u)
#pragma unroll
            for (int i = 0; i < 4; ++i) c += v[u][i] != INT_MIN && v[u][i] >= mk;
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        if (tot == 0) continue;
        int base = 0;
        if (lane == 0) base = atomicAdd(&S.lcnt, tot);
        base = __shfl_sync(0xffffffffu, base, 0);
#ifdef CCW_DBG_TAIL
        if (q0 == 0 && lane == 0) S.dbg[6] = clock64() + (base == 0x7fffffff);
#endif
        if (base + tot > SC_LC) {
            if (lane == 0) S.lover = 1;
            continue;
        }
        int o = base + incl - c;
#pragma unroll
        for (int u = 0; u < SC_TB; ++u)
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (v[u][i] != INT_MIN && v[u][i] >= mk) {
                    S.sw.lv[o] = v[u][i];
                    S.sw.lp[o] = tl[u] * kTcTile + lane * 4 + i;
                    ++o;
                }
    }
}

// The (window, run group) items of rescore_keys: every operand is loaded and
// multiplied before the sequential sums (tb: the staged template in shared
// memory, or the global one).
template <typename TB>
__device__ __forceinline__ void rescore_items(const SimParams& P, FastSmem& S, TB tb, int nr, int ngrp,
                                              const int* cidx, int e0, int ng, int R) {
    const size_t plane = static_cast<size_t>(P.hc) * P.wc;
    for (int it = threadIdx.x; it < ng * ngrp; it += FS_T) {
#ifdef CCW_DBG_TAIL
        long long z0 = clock64();
#endif
        const int e = it / ngrp, g = it - e * ngrp;
        const int4 G = S.grp[g];  // rows s0 .. s0 + nk - 1, columns t0 .. t0 + len - 1
        const int ch = G.x, k0 = G.y & 0xffff, s0 = G.y >> 16, nk = G.z & 255, t0 = G.w >> 8, len = G.w & 255;
        const int pos = cidx[e0 + e];
        const int x = pos / P.out_w, y = pos - x * P.out_w;
        const double* a0 = P.ti64 + ch * plane + static_cast<size_t>(x + s0) * P.wc + y + t0;
        const int b0 = ch * P.Tc * P.Tc + s0 * P.Tc + t0;
        double* rs = S.rsum + e * R + ch * nr + k0;
        double pv[FS_G];
        if (len > FS_G) {  // one long run (nk == 1), FS_G products per round trip
            double sum = 0.0;
            for (int c0 = 0; c0 < len; c0 += FS_G) {
#pragma unroll
                for (int c = 0; c < FS_G; ++c)
                    pv[c] = c0 + c < len ? __dmul_rn(__ldg(a0 + c0 + c), tb[b0 + c0 + c]) : 0.0;
#pragma unroll
                for (int c = 0; c < FS_G; ++c)
                    if (c0 + c < len) sum = __dadd_rn(sum, pv[c]);
            }
            rs[0] = sum;
            continue;
        }
        // Cells past nk * len read a clamped in-window address and are never
        // stored, so no load needs a predicate and all FS_G are in flight at once.
        const int inv = (4096 + len - 1) / len;  // c / len == (c * inv) >> 12 for c < 16
#pragma unroll
        for (int c = 0; c < FS_G; ++c) {
            const int kq = (c * inv) >> 12, t = c - kq * len, kk = min(kq, nk - 1);
#ifdef CCW_DBG_NOTI  // timing experiment only: no TI reads (wrong results)
            pv[c] = __dmul_rn(tb[(b0 + kk * P.Tc + t + 7) & 255], tb[b0 + kk * P.Tc + t]);
#else
            pv[c] = __dmul_rn(__ldg(a0 + kk * P.wc + t), tb[b0 + kk * P.Tc + t]);
#endif
        }
#ifdef CCW_DBG_TAIL
        double chk = 0;
        for (int c = 0; c < FS_G; ++c) chk += pv[c];
        long long z1 = clock64();
        if (chk == 12345.678) z1 = 0;  // (keeps the products computed before z1)
#endif
        const int endm = G.z >> 8;  // cells that end a row
        double sum = 0.0;
        int kk = 0;
#pragma unroll
        for (int c = 0; c < FS_G; ++c) {
            sum = __dadd_rn(sum, pv[c]);
            if ((endm >> c) & 1) {
                rs[kk++] = sum;
                sum = 0.0;
            }
        }
#ifdef CCW_DBG_TAIL
        if (threadIdx.x == 0 && P.stats && ng < 8 && cidx != S.utmp) {
            const long long z2 = clock64();
            atomicAdd(&P.stats[41], static_cast<unsigned long long>(z1 - z0));
            atomicAdd(&P.stats[42], static_cast<unsigned long long>(z2 - z1));
            atomicAdd(&P.stats[43], 1ull);
        }
#endif
    }
}

// fp64 keys of the windows cidx[0, cnt) (reference order, see fast_batch).
// (tmg: the placement's template in global memory; staged in S.tm when it
// fits, unless own_tm is false -- a chunk of another placement.)
__device__ CCW_COLD void rescore_keys(const SimParams& P, FastSmem& S, const double* tmg, int nr,
                                             int ngrp, const int* cidx, int cnt, double* keys,
                                             bool own_tm = true) {
    const int tid = threadIdx.x;
    const int R = nr * P.nch;
    const int EB = max(1, FS_RS / R);
    const bool tm_smem = own_tm && P.nch * P.Tc * P.Tc <= PK_TMC;
    if (P.stats && tid == 0) atomicAdd(&P.stats[0], static_cast<unsigned long long>(cnt));
#ifdef CCW_DBG_TAIL
    long long r0 = clock64();
#endif
    for (int e0 = 0; e0 < cnt; e0 += EB) {
        const int ng = min(EB, cnt - e0);
        rescore_items(P, S, tm_smem ? static_cast<const double*>(S.tm) : tmg, nr, ngrp, cidx, e0, ng, R);
        __syncthreads();
#ifdef CCW_DBG_TAIL
        if (tid == 0 && e0 == 0) S.dbg[5] = clock64();
#endif
#ifdef CCW_DBG_TAIL
        if (tid == 0 && P.stats && cnt < 8) {
            atomicAdd(&P.stats[40], static_cast<unsigned long long>(clock64() - r0));
            r0 = clock64();
        }
#endif
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
#ifdef CCW_DBG_TAIL
        if (tid == 0 && e0 == 0) S.dbg[6] = clock64();
#endif
    }
}

// Rescore S.cidx[0, cnt) and merge with the running top-K (ntop entries).
__device__ CCW_COLD void fast_batch(const SimParams& P, FastSmem& S, const double* tmg, int nr,
                                           int ngrp, int cnt, int& ntop, int K) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    rescore_keys(P, S, tmg, nr, ngrp, S.cidx, cnt, S.key);
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


// ---- shared rescoring (HelpBoard, ccw_device.cuh) ----

// Rescore chunk c of slot's posted group (every thread calls; uses S.grp,
// S.cs, S.rsum, S.key) and count it finished.
__device__ __forceinline__ void hb_chunk(const SimParams& P, FastSmem& S, int slot, int c, int4 info) {
    const int tid = threadIdx.x;
    const int cw = info.w & 0xffff, var = info.w >> 16;
    const int e0 = c * cw, n = min(cw, info.z - e0);
    const int4* mt = P.mtab + static_cast<size_t>(var) * MT_STRIDE;
    const int4 mi = __ldg(mt);
    for (int e = tid; e < mi.y; e += FS_T) S.grp[e] = __ldg(mt + 1 + MT_ROWS4 + e);
    for (int e = tid; e < n; e += FS_T) S.cs[e] = __ldcg(P.hpos + static_cast<size_t>(slot) * SC_LC + e0 + e);
    __syncthreads();
    const double* tmg = P.tm64 + static_cast<size_t>(slot) * P.nch * P.Tc * P.Tc;
    rescore_keys(P, S, tmg, mi.x, mi.y, S.cs, n, S.key, false);
    for (int e = tid; e < n; e += FS_T) P.hkeys[static_cast<size_t>(slot) * SC_LC + e0 + e] = S.key[e];
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicAdd(&P.hs[slot].y, 1);
#ifdef CCW_DBG_TAIL
    if (tid == 0 && P.stats) {
        atomicAdd(&P.stats[33], 1ull);
        if (slot == static_cast<int>(blockIdx.x)) atomicAdd(&P.stats[34], 1ull);
    }
#endif
}

// Claim chunks of slot's posted group until none is left (every thread calls).
__device__ __forceinline__ void hb_drain(const SimParams& P, FastSmem& S, int slot, int4 info) {
    const int nchunk = (info.z + (info.w & 0xffff) - 1) / (info.w & 0xffff);
    while (true) {
        if (threadIdx.x == 0) {  // (a plain read first: most helpers arrive after the last claim)
            const int seen = *reinterpret_cast<volatile int*>(&P.hs[slot].x);
            S.misc[0] = seen >= nchunk ? seen : atomicAdd(&P.hs[slot].x, 1);
        }
        __syncthreads();
        const int c = S.misc[0];
        __syncthreads();
        if (c >= nchunk) return;
        hb_chunk(P, S, slot, c, info);
    }
}

// Help with every group posted so far in this launch (every thread calls).
__device__ CCW_COLD void hb_help(const SimParams& P, FastSmem& S) {
    const int tid = threadIdx.x;
    if (tid == 0) S.misc[1] = *reinterpret_cast<volatile int*>(&P.hb->nposts);
    __syncthreads();
    const int np = min(S.misc[1], HB_CAP);
    for (int q = 0; q < np; ++q) {
        __syncthreads();
        if (tid == 0) {
            volatile int* pp = &P.hb->posts[q];
            int v;
            while ((v = *pp) == 0) {  // (its poster is running and writes it next)
            }
            __threadfence();
            const int slot = v - 1;
            const int4 info = __ldcg(&P.hs[slot]);
            S.misc[2] = slot;
            S.misc[4] = info.z;
            S.misc[5] = info.w;
        }
        __syncthreads();
        const int slot = S.misc[2];
        hb_drain(P, S, slot, make_int4(0, 0, S.misc[4], S.misc[5]));
    }
}

// Rescore S.tie[0, g) of this placement with the launch's help: post the
// group, rescore its chunks until none is left (helpers claim the others),
// wait for the helpers' chunks, gather the keys into S.key.  Returns false
// (nothing posted) when the board is full.  Every thread calls.
__device__ CCW_COLD bool hb_rescore(const SimParams& P, FastSmem& S, int slot, int g, int ngrp,
                                           int var) {
    const int tid = threadIdx.x;
    const int cw = max(1, FS_T / ngrp);  // windows per chunk: one round of items
    const int nchunk = (g + cw - 1) / cw;
    const int4 info = make_int4(0, 0, g, cw | var << 16);
    for (int e = tid; e < g; e += FS_T) P.hpos[static_cast<size_t>(slot) * SC_LC + e] = S.tie[e];
    if (tid == 0) {
        P.hs[slot].z = info.z;
        P.hs[slot].w = info.w;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const int q = atomicAdd(&P.hb->nposts, 1);
        if (q < HB_CAP) atomicExch(&P.hb->posts[q], slot + 1);
        S.misc[3] = q < HB_CAP;
    }
    __syncthreads();
    if (!S.misc[3]) return false;
#ifdef CCW_DBG_TAIL
    const long long h0 = clock64();
#endif
    hb_drain(P, S, slot, info);
#ifdef CCW_DBG_TAIL
    const long long h1 = clock64();
#endif
    if (tid == 0) {
        volatile int* done = &P.hs[slot].y;
        while (*done < nchunk) {
        }
        __threadfence();
        if (P.stats) atomicAdd(&P.stats[32], 1ull);
#ifdef CCW_DBG_TAIL
        if (P.stats) {
            atomicAdd(&P.stats[35], static_cast<unsigned long long>(h1 - h0));
            atomicAdd(&P.stats[36], static_cast<unsigned long long>(clock64() - h1));
        }
#endif
    }
    __syncthreads();
    for (int e = tid; e < g; e += FS_T) S.key[e] = __ldcg(P.hkeys + static_cast<size_t>(slot) * SC_LC + e);
    __syncthreads();
    return true;
}

#ifndef CCW_COOP_SCAN
#define CCW_COOP_SCAN 1
#endif
#ifndef CCW_FS_MINB
#define CCW_FS_MINB 4
#endif
// Lean scan of an unconditional pick (warp 0; every lane calls it), after
// coop_head queued the nq tiles whose maximum reaches mk: when they fit one
// round trip (nq <= SC_TB) the warp reads their rows itself -- no other warp,
// no shared-memory atomics, no block barrier -- and, when the list of windows
// >= mk fits one per lane, settles the equal-score group holding rank `pick`
// in the same rounds that find S_{pick+1} (pick_group's outputs, S.lean =
// 2).  Returns false (nothing written) when the queue is too long for it.
template <bool S16>
__device__ __forceinline__ bool lean_scan(const SimParams& P, int slot, FastSmem& S, int pick, int K,
                                          long long* sclk) {
    const int lane = threadIdx.x & 31;
    const int nq = S.nq, mk = S.misc[1];
    if (nq > SC_TB || S.lover) return false;
    int tl[SC_TB], v[SC_TB][4];
#pragma unroll
    for (int u = 0; u < SC_TB; ++u) tl[u] = u < nq ? S.tqa[u] : -1;
#pragma unroll
    for (int u = 0; u < SC_TB; ++u) {
        const int p0 = tl[u] * kTcTile + lane * 4;
#pragma unroll
        for (int i = 0; i < 4; ++i) v[u][i] = INT_MIN;
        if (tl[u] >= 0 && p0 < P.npos) {  // rows are padded to a multiple of 4
            const int4 a4 = load_score4<S16>(P, slot, p0);
            v[u][0] = a4.x;
            v[u][1] = p0 + 1 < P.npos ? a4.y : INT_MIN;
            v[u][2] = p0 + 2 < P.npos ? a4.z : INT_MIN;
            v[u][3] = p0 + 3 < P.npos ? a4.w : INT_MIN;
        }
    }
#ifdef CCW_DBG_TAIL
    {
        int sdbg = 0;
#pragma unroll
        for (int u = 0; u < SC_TB; ++u) sdbg ^= v[u][0];
        const long long cl = clock64();
        if (lane == 0) S.dbg[2] = cl + (sdbg == 0x12345 ? 1 : 0);
    }
#endif
    // the (score, position) list of windows >= mk, in lane order
    int c = 0;
#pragma unroll
    for (int u = 0; u < SC_TB; ++u)
#pragma unroll
        for (int i = 0; i < 4; ++i) c += v[u][i] != INT_MIN && v[u][i] >= mk;
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int nl = __shfl_sync(0xffffffffu, incl, 31);
    if (P.stats && lane == 0) atomicAdd(&P.stats[1], 1ull);
    if (nl > SC_LC) {  // (the general path's overflow: deferred with threshold mk)
        if (lane == 0) {
            S.misc[0] = -1;
            S.lean = 1;
            if (P.stats) atomicAdd(&P.stats[2], 1ull);
        }
        return true;
    }
    int o = incl - c;
#pragma unroll
    for (int u = 0; u < SC_TB; ++u)
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (v[u][i] != INT_MIN && v[u][i] >= mk) {
                S.sw.lv[o] = v[u][i];
                S.sw.lp[o] = tl[u] * kTcTile + lane * 4 + i;
                ++o;
            }
    __syncwarp();
    sclk[2] = clock64();
    if (nl > 32) {  // the general finish over the list
        const int n = scan_finish(P, S.sw, nl, mk, S.cidx, sclk, S.cs, K);
        if (lane == 0) {
            S.misc[0] = n;
            S.lean = 1;
        }
        return true;
    }
    // one window per lane: rounds of (max, count) down to the group holding
    // rank `pick`; its score is S_{pick+1}, the candidates are the windows >= it
    const int lv = lane < nl ? S.sw.lv[lane] : INT_MIN;
    const int lp = lane < nl ? S.sw.lp[lane] : -1;
    int cur = INT_MAX, acc = 0, sp = INT_MIN, above = 0;
    for (int round = 0; round <= pick && round < nl; ++round) {
        const int m = __reduce_max_sync(0xffffffffu, lv < cur ? lv : INT_MIN);
        const int cn = __popc(__ballot_sync(0xffffffffu, lane < nl && lv == m));
        sp = m;
        above = acc;
        if (acc + cn > pick) break;
        acc += cn;
        cur = m;
    }
    sclk[3] = clock64();
    const bool cand = lane < nl && lv >= sp;
    const unsigned cb = __ballot_sync(0xffffffffu, cand);
    if (cand) {
        const int e = __popc(cb & ((1u << lane) - 1));
        S.cidx[e] = lp;
        S.cs[e] = lv;
    }
    const bool q = lane < nl && lv == sp;
    const unsigned gb = __ballot_sync(0xffffffffu, q);
    if (q) S.tie[__popc(gb & ((1u << lane) - 1))] = lp;
    if (lane == 0) {
        S.misc[0] = __popc(cb);
        S.misc[6] = __popc(gb);
        S.misc[5] = pick - above;  // rank inside the group
        S.lean = 2;
    }
    return true;
}

// Unconditional pick (one warp): the equal-score group of the candidates
// S.cs/S.cidx[0, n) that holds rank `pick` of (S desc, ...) into S.tie, its
// size into S.misc[6] and the rank inside it into S.misc[5].  KV candidates
// per lane (KV * 32 >= n).
template <int KV>
__device__ __forceinline__ void pick_group(FastSmem& S, int n, int pick, int lane) {
    int v[KV];
#pragma unroll
    for (int j = 0; j < KV; ++j) {
        const int e = j * 32 + lane;
        v[j] = e < n ? S.cs[e] : INT_MIN;
    }
    int cur = INT_MAX, acc = 0, sp = INT_MIN, above = 0;
    for (int round = 0; round <= pick && round < n; ++round) {
        int m = INT_MIN;
#pragma unroll
        for (int j = 0; j < KV; ++j)
            if (v[j] < cur) m = max(m, v[j]);
        m = __reduce_max_sync(0xffffffffu, m);
        int c = 0;
#pragma unroll
        for (int j = 0; j < KV; ++j) c += v[j] == m;
        c = static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(c)));
        sp = m;
        above = acc;
        if (acc + c > pick) break;
        acc += c;
        cur = m;
    }
    int g = 0;
#pragma unroll
    for (int j = 0; j < KV; ++j) {
        const int e = j * 32 + lane;
        const bool q = e < n && v[j] == sp;
        const unsigned bal = __ballot_sync(0xffffffffu, q);
        if (q) S.tie[g + __popc(bal & ((1u << lane) - 1))] = S.cidx[e];
        g += __popc(bal);
    }
    if (lane == 0) {
        S.misc[6] = g;
        S.misc[5] = pick - above;  // rank inside the group
    }
}

template <bool S16>  // int16 score rows (P.s16); one instance each keeps the code lean
__global__ void __launch_bounds__(FS_T, CCW_FS_MINB)
    select_fast_kernel(const __grid_constant__ SimParams P, const Job* __restrict__ jobs, int job0, int nj) {
    __shared__ FastSmem S;
    const int slot = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
#ifdef CCW_DBG_TAIL
    if (tid < 8) S.dbg[tid] = 0;
#endif
    pdl_trigger();
    tl_mark(P.tl, 2);
#ifdef CCW_TI_PREFETCH
    // keep the fp64 TI apex planes (the tie rescoring's operands, rarely read)
    // in L2: each CTA of the launch touches its slice, before the wait
    if (wid == 1 && P.ti64) {
        const size_t lines = (static_cast<size_t>(P.nch) * P.hc * P.wc * sizeof(double) + 127) / 128;
        const size_t l0 = lines * slot / gridDim.x, l1 = lines * (slot + 1) / gridDim.x;
        for (size_t l = l0 + lane; l < l1; l += 32)
            asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(reinterpret_cast<const char*>(P.ti64) + l * 128));
    }
#endif
#ifdef CCW_DBG_TLB  // experiment: touch this slot's score row before the wait (translation only)
    if (wid == 1 && slot < nj) {
        const char* r = reinterpret_cast<const char*>(P.scores) + static_cast<size_t>(slot) * P.sld * (P.s16 ? 2 : 4);
        unsigned x;
        asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(x) : "l"(r + lane * 768));
        if (x == 0x12345677u) S.misc[0] = 0;
    }
#endif
    pdl_wait();
    tl_mark(P.tl, 0);
    if (P.hb_reset && slot == 0) {  // the next launch's board (the last launch that used it is complete)
        for (int i = tid; i < HB_CAP; i += FS_T) P.hb_reset->posts[i] = 0;
        for (int i = tid; i < P.hs_n; i += FS_T) P.hs_reset[i] = make_int4(0, 0, 0, 0);
        if (tid == 0) P.hb_reset->nposts = 0;
    }
    if (slot >= nj) return;
    const int gj = job0 + slot;
    const Job jb = jobs[gj];
    if (P.xrec && jb.shape == kNone) {  // (position shards: the merge places first patches)
        if (P.defer && tid == 0) P.defer[slot] = INT_MIN;
        return;
    }
    const int Tc = P.Tc;
    long long fclk[5] = {clock64(), 0, 0, 0, 0};
#ifdef CCW_DBG_TAIL
    const unsigned long long dbg_t0 = gtimer();
    int dbg_n = -2, dbg_g = 0;
    long long pc[8] = {clock64(), 0, 0, 0, 0, 0, 0, 0};  // head, list, finish, resolve, choose, paste, deps
#define PCLK(i) pc[i] = clock64()
#else
#define PCLK(i)
#endif
    int fr, fc;
    if (jb.shape == kNone) {
        fr = jb.fr;
        fc = jb.fc;
    } else {
        const int K = P.K;
        const double* tmg = P.tm64 + static_cast<size_t>(slot) * P.nch * Tc * Tc;
        const int ntm = P.nch * Tc * Tc;
        int mk = INT_MIN;
        // the scan: warp 0 alone (scan_job), or with the list step spread over
        // every warp when the tile maxima fit in registers
        const bool coop = CCW_COOP_SCAN && P.ntiles <= 32 * kTM;
        // An unconditional pick (matcher.hpp:207-211) needs only the top
        // pick + 1 windows in rank order: every window at or above rank `pick`
        // scores >= the (pick+1)-th largest score S_{pick+1} >= the (pick+1)-th
        // largest tile maximum, so the scan runs with K' = pick + 1 -- fewer
        // rounds, fewer qualifying tiles, and the list (and a deferral's
        // threshold) is still a superset of the ranks that matter.
        const bool upick = jb.pick >= 0 && !P.xrec;
        const int Ks = upick ? min(jb.pick + 1, K) : K;
        long long sclk[5];
        if (wid == 0) {
            sclk[0] = clock64();
            if (coop) {
                coop_head(P, slot, S, Ks);
                sclk[1] = clock64();
                PCLK(1);
                __syncwarp();
                if (!(upick && lean_scan<S16>(P, slot, S, jb.pick, Ks, sclk)) && lane == 0) S.lean = 0;
            } else {
                const int n = scan_job<S16>(P, slot, S.sw, S.cidx, mk, sclk, S.cs);
                if (lane == 0) {
                    S.misc[0] = n;
                    S.misc[1] = mk;
                    if (P.stats && P.tl && n >= 0) {
                        sclk[4] = clock64();
                        for (int q = 0; q < 4; ++q)
                            atomicAdd(&P.stats[8 + q], static_cast<unsigned long long>(sclk[q + 1] - sclk[q]));
                    }
                }
            }
        } else {
            // stage the template (matcher.hpp:44-61 order), the mask rows and the run groups
            if (ntm <= PK_TMC)
                for (int e = tid - 32; e < ntm; e += FS_T - 32) cp_async8(&S.tm[e], tmg + e);
            // the run groups of this mask variant (host tables)
            const int4* mt = P.mtab + static_cast<size_t>(mask_variant(jb.shape, jb.vleft, jb.htop)) * MT_STRIDE;
            const int4 info = __ldg(mt);
            for (int e = tid - 32; e < info.y; e += FS_T - 32) cp_async16(&S.grp[e], mt + 1 + MT_ROWS4 + e);
            if (tid == 32) {
                S.misc[2] = info.x;
                S.misc[3] = info.y;
                S.misc[7] = info.z;
            }
            cp_async_wait_all();
#ifdef CCW_DBG_TAIL
            if (tid == 32) S.dbg[3] = clock64();
#endif
        }
        __syncthreads();
#ifdef CCW_DBG_TAIL
        if (tid == 0) S.dbg[4] = clock64();
#endif
        const int lean = coop ? S.lean : 0;
        if (coop && !lean) {
            coop_list<S16>(P, slot, S);
            __syncthreads();
            PCLK(2);
            if (wid == 0) {
                sclk[2] = clock64();
                const int nl = S.lcnt, mk0 = S.misc[1];
                if (P.stats && lane == 0) atomicAdd(&P.stats[1], 1ull);
                int n = -1;
                if (S.lover) {
                    if (P.stats && lane == 0) atomicAdd(&P.stats[2], 1ull);
                } else {
                    n = scan_finish(P, S.sw, nl, mk0, S.cidx, sclk, S.cs, Ks);
                }
                if (lane == 0) {
                    S.misc[0] = n;
                    if (P.stats && P.tl && n >= 0) {
                        sclk[4] = clock64();
                        for (int q = 0; q < 4; ++q)
                            atomicAdd(&P.stats[8 + q], static_cast<unsigned long long>(sclk[q + 1] - sclk[q]));
                    }
                }
            }
            __syncthreads();
        }
        fclk[1] = clock64();
        PCLK(3);
        const int n = S.misc[0], nr = S.misc[2], ngrp = S.misc[3];
#ifdef CCW_DBG_TAIL
        dbg_n = n;
#endif
        mk = S.misc[1];
        int ntop = 0;
        if (n < 0 && P.defer) {  // a large tie group: the bulk kernel rescores every window >= M_K
            if (tid == 0) {
                P.defer[slot] = max(mk, INT_MIN + 1);  // (INT_MIN marks "not deferred")
                if (P.defer_list) P.defer_list[atomicAdd(P.defer_cnt, 1)] = slot;
            }
            return;
        }
        if (P.defer && tid == 0) P.defer[slot] = INT_MIN;
        int picked = -1;  // the chosen position when settled without the ranked list
        if (n >= 0 && jb.pick >= 0 && !P.xrec) {
            // Unconditional pick (matcher.hpp:207-211): only the candidate at rank
            // `pick` of (S desc, fp64 desc, index asc) matters, and windows with
            // different S never swap in fp64 -- so only the equal-S group that
            // holds rank `pick` can need fp64 keys, and none when it is a single window.
            if (wid == 0 && lean != 2) {
                if (n <= 32)
                    pick_group<1>(S, n, jb.pick, lane);
                else
                    pick_group<SC_LC / 32>(S, n, jb.pick, lane);
            }
            if (lean != 2) __syncthreads();
            const int g = S.misc[6], rk = S.misc[5];
#ifdef CCW_DBG_TAIL
            dbg_g = g;
#endif
            if (g == 1) {
                picked = S.tie[0];
            } else {
#ifdef CCW_DBG_TAIL
                const long long q0 = clock64();
#endif
                const int var = mask_variant(jb.shape, jb.vleft, jb.htop);
#ifdef CCW_DBG_TAIL
                if (tid == 0) S.dbg[3] = clock64();
#endif
#ifdef CCW_DBG_WARM  // experiment: a dry run on other windows first (warm code, cold data)
                if (g < 8) {
                    for (int e = tid; e < g; e += FS_T) S.utmp[e] = (S.tie[e] + 7919) % P.npos;
                    __syncthreads();
                    rescore_keys(P, S, tmg, nr, ngrp, S.utmp, g, S.key + 64);
                    if (tid == 0 && P.stats) atomicAdd(&P.stats[39], static_cast<unsigned long long>(clock64() - q0));
                }
#endif
                const int gr = P.umap && g >= UD_MIN ? uniform_reduce(P, S, g, var) : g;
                if (!(P.hb && gr >= P.help_min && hb_rescore(P, S, slot, gr, ngrp, var)))
                    rescore_keys(P, S, tmg, nr, ngrp, S.tie, gr, S.key);
                if (gr < g) uniform_fill(S, gr, g);
#ifdef CCW_DBG_TAIL
                if (tid == 0 && P.stats && g < 8) {
                    atomicAdd(&P.stats[37], 1ull);
                    atomicAdd(&P.stats[38], static_cast<unsigned long long>(clock64() - q0));
                    atomicAdd(&P.stats[39], static_cast<unsigned long long>(q0 - fclk[1]));
                }
#endif
                if (g <= FS_T) {  // the rk-th best of the group by (fp64 desc, index asc): direct ranks
                    if (tid < g) {
                        const double ke = S.key[tid];
                        const int ie = S.tie[tid];
                        int rank = 0;
                        for (int j = 0; j < g; ++j) rank += better(S.key[j], S.tie[j], ke, ie);
                        if (rank == rk) S.misc[4] = ie;
                    }
                } else if (wid == 0) {
                    for (int round = 0; round <= rk; ++round) {
                        double bk = 0.0;
                        int bi = INT_MAX, bp = -1;
                        for (int e = lane; e < g; e += 32) {
                            const int ix = S.tie[e];
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
                        if (round == rk) {
                            if (lane == 0) S.misc[4] = bi;
                        } else if (lane == 0) {
                            S.tie[bp] = -1;
                        }
                        __syncwarp();
                    }
                }
                __syncthreads();
#ifdef CCW_DBG_TAIL
                if (tid == 0) S.dbg[7] = clock64();
#endif
                picked = S.misc[4];
            }
        } else if (n >= 0 && n <= 32) {
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
            if (nt > 0) rescore_keys(P, S, tmg, nr, ngrp, S.tie, nt, S.key);
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
                    // (position shards: a key that was not computed is marked NaN)
                    S.tkey[rank] = P.xrec && S.tslot[lane] < 0 ? __longlong_as_double(0x7ff8000000000000ll) : ki;
                }
            }
            ntop = min(K, n);
            __syncthreads();
        } else if (n >= 0) {
            fast_batch(P, S, tmg, nr, ngrp, n, ntop, K);
        } else {
            // list overflow without the bulk kernel: every window >= M_K, in batches
            const int32_t* tmx = P.tmax + static_cast<size_t>(slot) * P.ntiles;
            int cnt = 0;
            for (int t = 0; t < P.ntiles; ++t) {
                if (tmx[t] < mk) continue;  // uniform
                const int p = t * kTcTile + tid;  // FS_T == kTcTile
                const bool q = p < P.npos && (S16 ? static_cast<int>(reinterpret_cast<const int16_t*>(P.scores)[static_cast<size_t>(slot) * P.sld + p]) : P.scores[static_cast<size_t>(slot) * P.sld + p]) >= mk;
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
                    fast_batch(P, S, tmg, nr, ngrp, cnt, ntop, K);
                    cnt = 0;
                }
                if (q) S.cidx[cnt + off + __popc(bal & ((1u << lane) - 1))] = p;
                cnt += tot;
                __syncthreads();
            }
            if (cnt > 0) fast_batch(P, S, tmg, nr, ngrp, cnt, ntop, K);
        }
        fclk[2] = clock64();
        PCLK(4);
        if (P.xrec) {  // position shard: hand the local top-K to the exchange
            ShardRec* xr = P.xrec + (static_cast<size_t>(P.xshard) * P.xnj + slot) * P.xk;
            for (int k = tid; k < P.xk; k += FS_T) {
                const double key = k < ntop ? S.tkey[k] : 0.0;
                xr[k] = k < ntop ? ShardRec{key, S.tidx[k], isnan(key) ? 0 : 1} : ShardRec{0.0, -1, 0};
            }
            return;
        }
        // choose (matcher.hpp:207-241)
        if (picked < 0 && wid == 0) {
            const int pos = choose_pick(P, jb, S.tidx, ntop, lane);
            if (lane == 0) S.misc[4] = pos;
        }
        __syncthreads();
        fclk[3] = clock64();
        PCLK(5);
        const int pos = picked >= 0 ? picked : S.misc[4];
        fr = (pos / P.out_w) << P.J;
        fc = (pos % P.out_w) << P.J;
    }
    paste_job<FS_T>(P, jb, gj, fr, fc, tid);
    PCLK(6);
    prep_dependents(P, jobs, jb, &S.misc[5]);
    if (P.depflag) {  // the next wave's OR prep of each dependent waits for these map writes
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            if (jb.dep0 >= 0) atomicAdd(&P.depflag[jb.dep0], 1);
            if (jb.dep1 >= 0) atomicAdd(&P.depflag[jb.dep1], 1);
        }
    }
    PCLK(7);
    if (tid == 0) {
        P.chosen[2 * gj] = fr;
        P.chosen[2 * gj + 1] = fc;
        if (P.stats && P.tl && fclk[3]) {
            fclk[4] = clock64();
            atomicAdd(&P.stats[12], static_cast<unsigned long long>(fclk[1] - fclk[0]));
            atomicAdd(&P.stats[13], static_cast<unsigned long long>(fclk[2] - fclk[1]));
            atomicAdd(&P.stats[4], static_cast<unsigned long long>(fclk[4] - fclk[2]));
            atomicAdd(&P.stats[5], static_cast<unsigned long long>(fclk[3] - fclk[2]));  // choose
#ifdef CCW_DBG_TAIL
            const bool had_tie = S.misc[6] > 0;
            const unsigned long long tot = static_cast<unsigned long long>(fclk[4] - fclk[0]);
            atomicAdd(&P.stats[had_tie ? 16 : 19], 1ull);
            atomicAdd(&P.stats[had_tie ? 17 : 20], tot);
            atomicMax(&P.stats[had_tie ? 18 : 21], tot);
            atomicAdd(&P.stats[22 + (tot < 10000 ? 0 : tot < 20000 ? 1 : tot < 40000 ? 2 : tot < 80000 ? 3 : 4)], 1ull);
            // where the long ones spend it: scan, batch, choose+map
            if (tot >= 40000) {
                atomicAdd(&P.stats[30], static_cast<unsigned long long>(S.misc[0]));  // candidates
                atomicAdd(&P.stats[27], static_cast<unsigned long long>(fclk[1] - fclk[0]));
                atomicAdd(&P.stats[28], static_cast<unsigned long long>(fclk[2] - fclk[1]));
                atomicAdd(&P.stats[29], static_cast<unsigned long long>(fclk[4] - fclk[2]));
            }
#endif
        }
    }
#ifdef CCW_DBG_TAIL
    const unsigned long long dbg_t1 = gtimer();
#endif
    if (P.hb) hb_help(P, S);  // rescore posted chunks of this launch's large groups
#ifdef CCW_DBG_TAIL
    if (P.jdump && tid == 0) {
        unsigned long long* d = P.jdump + 8 * static_cast<size_t>(gj);
        d[0] = dbg_t0;
        d[1] = dbg_t1;
        d[2] = gtimer();
        d[3] = static_cast<unsigned long long>(static_cast<unsigned>(dbg_n)) |
               (static_cast<unsigned long long>(dbg_g) << 32);
        for (int q = 1; q < 8; ++q) {  // cycle deltas from the start, 16 bits each (saturated)
            const long long dv = pc[q] ? min(pc[q] - pc[0], 65535ll) : 0;
            d[4 + (q >> 2)] |= static_cast<unsigned long long>(dv) << (16 * (q & 3));
        }
        for (int q = 0; q < 8; ++q) {  // 0 tmax loaded, 1 M_K, 2 rows loaded, 3 staging done, 4 sync, 5 tl read, 6 atomic
            const long long dv = S.dbg[q] > pc[0] ? min(S.dbg[q] - pc[0], 65535ll) : 0;
            d[6 + (q >> 2)] |= static_cast<unsigned long long>(dv) << (16 * (q & 3));
        }
    }
#endif
    tl_mark(P.tl, 1);
#undef PCLK
}

template __global__ void select_fast_kernel<false>(const __grid_constant__ SimParams, const Job* __restrict__, int, int);
template __global__ void select_fast_kernel<true>(const __grid_constant__ SimParams, const Job* __restrict__, int, int);

// One CTA's share (part of S) of one deferred placement.
__device__ __forceinline__ void bulk_part(const SimParams& P, const Job* __restrict__ jobs, int job0, int slot,
                                          int part, int S, unsigned char* bk_sm) {
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
    auto offer = [&](double ck, int ci) {  // per-thread top-K under the reference ranking
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
    };
    // Uniform-class windows (every masked coarse block pure facies f, P.umap)
    // carry the all-f block's apex on every masked cell, so their fp64 score is
    // one value per class: computed once here in the reference's order
    // (matcher.hpp:72-77, 160-161) and never rescored per window.
    double* ukey = reinterpret_cast<double*>(bk_sm + L.ukey);
    const bool uni = P.umap != nullptr && P.pure_apex != nullptr && P.ufirst != nullptr;
    const int var = mask_variant(jb.shape, jb.vleft, jb.htop);
    const int8_t* um = uni ? P.umap + static_cast<size_t>(var) * P.ustride : nullptr;
    __syncthreads();  // (template and mask rows staged)
    if (uni && tid < 16) {
        double acc = 0.0;
        for (int ch = 0; ch < nch; ++ch) {
            const double c = P.pure_apex[tid * nch + ch];
            const double* tp = tmS + ch * Tc * Tc;
            for (int r = 0; r < nrows; ++r) {
                const short4 rw = rows[r];
                double sum = 0.0;
                for (int t = rw.y; t < rw.z; ++t) sum = __dadd_rn(sum, __dmul_rn(c, tp[rw.x * Tc + t]));
                acc = __dadd_rn(acc, sum);
            }
        }
        ukey[tid] = acc;
        // every member of a class shares its score and key, so the class's
        // candidates are its K lowest positions -- offered once per placement
        // (by CTA 0), when the class reaches the threshold
        const int* fp = P.ufirst + (static_cast<size_t>(var) * 16 + tid) * kTcQ;
        if (part == 0 && fp[0] != INT_MAX && load_score(P, slot, fp[0]) >= thr)
            for (int j = 0; j < K; ++j)
                if (fp[j] != INT_MAX) offer(acc, fp[j]);
    }
    unsigned long long rescored = 0;
#ifdef CCW_DEBUG_KNOBS
    const long long dbg_c0 = clock64();
#endif
    const int nbx = (P.out_h + bx - 1) / bx, nby = (P.out_w + by - 1) / by;
    int* next = P.bulk_sync + 2 * slot;  // [0] next block, [1] finished CTAs
    if (P.tmax_nu && uni) {
        // Only a tile whose maximum over NON-uniform windows reaches the
        // threshold can hold a candidate the class keys do not cover: this
        // CTA's share (tiles part, part + S, ...) is filtered on the screen's
        // tmax_nu, and each qualifying tile's windows are checked by one
        // thread each and rescored straight from L2 (reference order).
        const int32_t* tn = P.tmax_nu + static_cast<size_t>(slot) * P.ntiles;
        int* tq = cand;
        if (tid == 0) wcnt[0] = 0;
        __syncthreads();
        for (int t = part + S * tid; t < P.ntiles; t += S * BK_T)
            if (tn[t] >= thr) tq[atomicAdd(&wcnt[0], 1)] = t;
        __syncthreads();
        const int nq = wcnt[0];
        constexpr int kTpp = BK_T / kTcTile;  // tiles per pass
        for (int q0 = 0; q0 < nq; q0 += kTpp) {
            const int qi = q0 + tid / kTcTile;
            if (qi >= nq) continue;
            const int p = tq[qi] * kTcTile + tid % kTcTile;
            if (p >= P.npos || um[p] >= 0 || load_score(P, slot, p) < thr) continue;
            const int x = p / P.out_w, y = p - x * P.out_w;
            double acc = 0.0;
            for (int ch = 0; ch < nch; ++ch) {
                const double* sp = P.ti64 + static_cast<size_t>(ch) * P.hc * P.wc + static_cast<size_t>(x) * P.wc + y;
                const double* tp = tmS + ch * Tc * Tc;
                for (int r = 0; r < nrows; ++r) {
                    const short4 rw = rows[r];
                    const double* a = sp + rw.x * P.wc + rw.y;
                    const double* b = tp + rw.x * Tc + rw.y;
                    double sum = 0.0;  // sum += ti*or left to right (matcher.hpp:72-76)
                    for (int t = 0; t < rw.z - rw.y; ++t) sum = __dadd_rn(sum, __dmul_rn(__ldg(a + t), b[t]));
                    acc = __dadd_rn(acc, sum);
                }
            }
            offer(acc, p);
            if (P.stats) atomicAdd(&P.stats[0], 1ull);
        }
    }
    for (;;) {
        if (P.tmax_nu && uni) break;  // (the tile path above covered this placement)
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
            // every load of the pass in flight at once (score and class are
            // independent: one round trip per pass)
            int v[BK_V];
            int8_t u[BK_V];
#pragma unroll
            for (int i = 0; i < BK_V; ++i) {
                const int e = e0 + tid * BK_V + i;
                v[i] = INT_MIN;
                u[i] = -1;
                if (e < nb) {
                    const int lx = e / bya, ly = e - lx * bya;
                    const size_t p = static_cast<size_t>(xb + lx) * P.out_w + yb + ly;
                    v[i] = load_score(P, slot, p);
                    if (uni) u[i] = um[p];
                }
            }
            // (uniform-class windows were offered per class above)
#pragma unroll
            for (int i = 0; i < BK_V; ++i)
                if (u[i] >= 0) v[i] = INT_MIN;
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
        // stage the apex tile the block's windows read -- worth it only for
        // many windows; a few are rescored straight from L2
        const bool staged = cnt >= BK_STAGE_MIN;
        const int pitch = staged ? L.sw : P.wc;
        if (staged) {
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
        }
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
                base[k] = lx * pitch + ly;
                pidx[k] = (xb + lx) * P.out_w + yb + ly;
            }
            double acc[BK_W];
#pragma unroll
            for (int k = 0; k < BK_W; ++k) acc[k] = 0.0;
            for (int ch = 0; ch < nch; ++ch) {
                const double* sp = staged ? stg + static_cast<size_t>(ch) * L.sh * L.sw
                                          : P.ti64 + static_cast<size_t>(ch) * P.hc * P.wc +
                                                static_cast<size_t>(xb) * P.wc + yb;
                const double* tp = tmS + ch * Tc * Tc;
                for (int r = 0; r < nrows; ++r) {
                    const short4 rw = rows[r];
                    const double* a = sp + rw.x * pitch + rw.y;
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
            for (int k = 0; k < BK_W; ++k)
                if (ok[k]) offer(acc[k], pidx[k]);
        }
        clk_comp += clock64() - c_cp;
    }
#ifdef CCW_DEBUG_KNOBS
    const long long dbg_c1 = clock64();
    if (tid == 0 && P.stats) {
        atomicAdd(&P.stats[44], static_cast<unsigned long long>(dbg_c0 - clk_start));
        atomicAdd(&P.stats[45], static_cast<unsigned long long>(dbg_c1 - dbg_c0));
        atomicMax(&P.stats[46], static_cast<unsigned long long>(dbg_c1 - clk_start));
    }
#endif
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
#ifdef CCW_DEBUG_KNOBS
    const long long dbg_c2 = clock64();
#endif
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
        if (P.xrec) {  // position shard: the merged list goes to the exchange (every key exact)
            ShardRec* xr = P.xrec + (static_cast<size_t>(P.xshard) * P.xnj + slot) * P.xk;
            for (int k = lane; k < P.xk; k += 32)
                xr[k] = k < ntop ? ShardRec{tkey[k], tidx[k], 1} : ShardRec{0.0, -1, 0};
        } else {
            const int pos = choose_pick(P, jb, tidx, ntop, lane);
            if (lane == 0) shv[3] = pos;
        }
        if (lane == 0) {
            next[0] = 0;  // reset the placement's counters for the next launch
            next[1] = 0;
            if (P.stats) atomicAdd(&P.stats[3], 1ull);
        }
    }
    if (P.xrec) return;
    __syncthreads();
    const int pos = shv[3];
    const int fr = (pos / P.out_w) << P.J, fc = (pos % P.out_w) << P.J;
    paste_job<BK_T>(P, jb, gj, fr, fc, tid);
    prep_dependents(P, jobs, jb, shv + 4);  // (misc + 304: free)
    if (tid == 0) {
        P.chosen[2 * gj] = fr;
        P.chosen[2 * gj + 1] = fc;
#ifdef CCW_DEBUG_KNOBS
        if (P.stats) atomicAdd(&P.stats[47], static_cast<unsigned long long>(clock64() - dbg_c2));
#endif
    }
}

// Persistent over the launch's deferred placements (the fast select lists
// them): CTA b takes work items b, b + gridDim.x, ... = (placement, part).
// Without a list (defer_list null) the grid is (S, nj) as one item per CTA.
__global__ void __launch_bounds__(BK_T, 1)
    select_bulk_kernel(SimParams P, const Job* __restrict__ jobs, int job0, int nj, int S) {
    extern __shared__ __align__(16) unsigned char bk_sm[];
    pdl_trigger();
    tl_mark(P.tl, 2);
    pdl_wait();
    tl_mark(P.tl, 0);
    if (!P.defer_list) {
        if (static_cast<int>(blockIdx.y) < nj) bulk_part(P, jobs, job0, blockIdx.y, blockIdx.x, S, bk_sm);
        tl_mark(P.tl, 1);
        return;
    }
    const int ndef = __ldcg(P.defer_cnt);
    if (blockIdx.x == 0 && threadIdx.x == 0) *P.defer_cnt_next = 0;  // (the next launch's list)
    // as many CTAs per deferred placement as the grid covers (the same S in
    // every CTA: each placement's last CTA is its (S-1)-th finisher)
#ifndef CCW_BK_CAP
#define CCW_BK_CAP 8
#endif
    const int Sd = max(1, min(CCW_BK_CAP, static_cast<int>(gridDim.x) / max(ndef, 1)));
    (void)S;
    for (int w = blockIdx.x; w < ndef * Sd; w += gridDim.x) {
        __syncthreads();  // (the previous item's shared memory is consumed)
        bulk_part(P, jobs, job0, __ldcg(P.defer_list + w / Sd), w % Sd, Sd, bk_sm);
    }
    tl_mark(P.tl, 1);
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

}  // namespace ccwgpu
