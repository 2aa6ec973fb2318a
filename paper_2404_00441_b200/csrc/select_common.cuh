// select_common.cuh -- the generic CTA select (radix threshold, fp64 rescoring,
// min-cut, choose, paste) and the warp-level choose / paste helpers, shared by
// select.cu (select_paste_kernel, the fast and bulk selects) and wave.cu (the
// fused wave kernel, whose rare fallback runs the generic select in-kernel).
#pragma once

#include <climits>

#include "sim_kernels.cuh"

namespace ccwgpu {

// Exact K-th largest value (with multiplicity) of n int32 values, skipping
// INT_MIN padding: block-wide radix select over the offset range, 8 bits per
// pass, warp-aggregated shared-memory histograms.
// (No __restrict__: the normalized screen rewrites its input in the same kernel.)
static __device__ int radix_kth_largest(const int32_t* sc, int n, int K, int* hist,
                                 int* misc, int* redi, int stride = 1) {
    int lo = INT_MAX, hi = INT_MIN;
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
        const int v = sc[static_cast<size_t>(p) * stride];
        if (v == INT_MIN) continue;
        lo = min(lo, v);
        hi = max(hi, v);
    }
    lo = block_reduce(lo, [](int a, int b) { return min(a, b); }, redi);
    hi = block_reduce(hi, [](int a, int b) { return max(a, b); }, redi);
    const uint32_t range = static_cast<uint32_t>(hi) - static_cast<uint32_t>(lo);
    if (range == 0) return lo;
    const int nbits = 32 - __clz(range);
    const int passes = (nbits + 7) / 8;
    uint32_t prefix = 0;
    int krem = K;
    for (int ps = passes - 1; ps >= 0; --ps) {
        const int shift = ps * 8;
        for (int e = threadIdx.x; e < 256; e += blockDim.x) hist[e] = 0;
        __syncthreads();
        for (int base = 0; base < n; base += blockDim.x) {
            const int p = base + threadIdx.x;
            bool match = false;
            int dg = 0;
            if (p < n && sc[static_cast<size_t>(p) * stride] != INT_MIN) {
                const uint32_t u = static_cast<uint32_t>(sc[static_cast<size_t>(p) * stride]) - static_cast<uint32_t>(lo);
                match = (static_cast<uint64_t>(u) >> (shift + 8)) ==
                        (static_cast<uint64_t>(prefix) >> (shift + 8));
                dg = (u >> shift) & 255;
            }
            const unsigned mm = __ballot_sync(0xffffffffu, match);
            if (match) {
                const unsigned grp = __match_any_sync(mm, dg);
                if ((threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&hist[dg], __popc(grp));
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int cum = 0, d = 255;
            for (; d > 0; --d) {
                if (cum + hist[d] >= krem) break;
                cum += hist[d];
            }
            misc[0] = d;
            misc[1] = krem - cum;
        }
        __syncthreads();
        prefix |= static_cast<uint32_t>(misc[0]) << shift;
        krem = misc[1];
        __syncthreads();
    }
    return static_cast<int>(static_cast<uint32_t>(lo) + prefix);
}

struct RunDesc {
    int ch, s, t0, t1;
};

// fp64 rescoring of `cnt` windows in the reference's exact order
//   acc = 0; for f: for run (row-major): sum = 0; sum += ti*or over the run;
//   acc += sum          (matcher.hpp:64-81, 158-161)
// plus, for normalized scoring, the masked squares and acc / sqrt(norm)
// (matcher.hpp:84-100, 163-171).  Parallel over (window, run) pairs: each
// thread forms one run's sum (the reference's inner chain), then one thread
// per window folds the run sums in order -- the same operations in the same
// order as the reference, so the result is bit-identical.
static __device__ void rescore_group(const SimParams& P, const RunDesc* runs, int R,
                              const double* tmpl, const int* gidx, double* gkey, int cnt,
                              double* rsum, double* rnrm) {
    const int EG = max(1, RSUM_CAP / R);
    const bool norm = P.scoring == 1;
    for (int e0 = 0; e0 < cnt; e0 += EG) {
        const int ng = min(EG, cnt - e0);
        for (int w = threadIdx.x; w < ng * R; w += blockDim.x) {
            const int e = e0 + w / R, r = w - (w / R) * R;
            const int pos = gidx[e];
            const int x = pos / P.out_w, y = pos - x * P.out_w;
            const RunDesc rd = runs[r];
            const double* a = P.ti64 + static_cast<size_t>(rd.ch) * P.hc * P.wc +
                              static_cast<size_t>(x + rd.s) * P.wc + y;
            const double* b = tmpl + (rd.ch * P.Tc + rd.s) * P.Tc;
            double sum = 0.0, nsum = 0.0;
            for (int t = rd.t0; t < rd.t1; ++t) {
                const double av = __ldg(a + t);
                sum = __dadd_rn(sum, __dmul_rn(av, b[t]));
                if (norm) nsum = __dadd_rn(nsum, __dmul_rn(av, av));
            }
            rsum[w] = sum;
            if (norm) rnrm[w] = nsum;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < ng; e += blockDim.x) {
            double acc = 0.0;
            for (int r = 0; r < R; ++r) acc = __dadd_rn(acc, rsum[e * R + r]);
            if (norm) {
                double n = 0.0;
                for (int r = 0; r < R; ++r) n = __dadd_rn(n, rnrm[e * R + r]);
                acc = n > 0.0 ? __ddiv_rn(acc, __dsqrt_rn(n)) : 0.0;
            }
            gkey[e0 + e] = acc;
        }
        __syncthreads();
    }
}

// Reference ranking: higher score first, earlier row-major location on ties
// (matcher.hpp:189-198 -- the result is a prefix of the stable sort).
__device__ __forceinline__ bool better(double ka, int ia, double kb, int ib) {
    return ka > kb || (ka == kb && ia < ib);
}

// Monotone min-cost seam (simulator.hpp:286-320) with the reference tie rules;
// dp rows in shared memory, one thread per band column, thread 0 backtracks.
template <typename CostF>
static __device__ void seam_dp(int layers, int width, CostF cost, int16_t* from, int* dp, int* seam) {
    for (int j = threadIdx.x; j < width; j += blockDim.x) dp[j] = cost(0, j);
    __syncthreads();
    for (int l = 1; l < layers; ++l) {
        const int* prev = dp + ((l - 1) & 1) * width;
        int* cur = dp + (l & 1) * width;
        for (int j = threadIdx.x; j < width; j += blockDim.x) {
            int best = prev[j], arg = j;
            if (j > 0 && prev[j - 1] < best) {
                best = prev[j - 1];
                arg = j - 1;
            }
            if (j + 1 < width && prev[j + 1] < best) {
                best = prev[j + 1];
                arg = j + 1;
            }
            if (j > 0 && prev[j - 1] == best && j - 1 < arg) arg = j - 1;
            cur[j] = cost(l, j) + best;
            from[l * width + j] = static_cast<int16_t>(arg);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int* last = dp + ((layers - 1) & 1) * width;
        int end = 0;
        for (int j = 1; j < width; ++j)
            if (last[j] < last[end]) end = j;
        seam[layers - 1] = end;
        for (int l = layers - 1; l > 0; --l) seam[l - 1] = from[l * width + seam[l]];
    }
    __syncthreads();
}

// min_cut_stitch (simulator.hpp:328-374) on T x T patches in shared memory:
// `outp` holds the incoming patch on entry and the stitched patch on exit.
static __device__ void min_cut_device(const uint8_t* exist, uint8_t* outp, int T, int OV, int shape,
                               int vleft, int htop, int16_t* from, int* dp, int* seam) {
    if (shape == kNone) return;
    if (shape == kVertical || shape == kL) {
        const int c0 = vleft ? 0 : T - OV;
        seam_dp(T, OV,
                [&](int r, int j) { return exist[r * T + c0 + j] != outp[r * T + c0 + j] ? 1 : 0; },
                from, dp, seam);
        for (int e = threadIdx.x; e < T * OV; e += blockDim.x) {
            const int r = e / OV, j = e - r * OV;
            const bool keep = vleft ? j < seam[r] : j > seam[r];
            if (keep) outp[r * T + c0 + j] = exist[r * T + c0 + j];
        }
        __syncthreads();
    }
    if (shape == kHorizontal || shape == kL) {
        const int r0 = htop ? 0 : T - OV;
        seam_dp(T, OV,
                [&](int c, int j) { return exist[(r0 + j) * T + c] != outp[(r0 + j) * T + c] ? 1 : 0; },
                from, dp, seam);
        for (int e = threadIdx.x; e < T * OV; e += blockDim.x) {
            const int c = e / OV, j = e - c * OV;
            const bool keep = htop ? j < seam[c] : j > seam[c];
            if (keep) outp[(r0 + j) * T + c] = exist[(r0 + j) * T + c];
        }
        __syncthreads();
    }
}

// Merge cnt keyed windows (gkey, gidx) with the running top-K list (tkey,
// tidx, ntop): K rounds of a block-wide argmax under the reference ranking.
static __device__ void merge_top(double* gkey, int* gidx, int& cnt, double* tkey, int* tidx, int& ntop,
                          int K, double* redd, int* redi) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int e = tid; e < ntop; e += SEL_T) {
        gkey[cnt + e] = tkey[e];
        gidx[cnt + e] = tidx[e];
    }
    __syncthreads();
    const int n = cnt + ntop;
    const int keep = min(K, n);
    for (int round = 0; round < keep; ++round) {
        double bk = 0.0;
        int bi = INT_MAX, bp = -1;
        for (int e = tid; e < n; e += SEL_T) {
            const int ix = gidx[e];
            if (ix >= 0 && (bp < 0 || better(gkey[e], ix, bk, bi))) {
                bk = gkey[e];
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
            redd[wid] = bk;
            redi[wid] = bi;
            redi[32 + wid] = bp;
        }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < SEL_T / 32; ++w) {
                if (redi[32 + w] >= 0 && (bp < 0 || better(redd[w], redi[w], bk, bi))) {
                    bk = redd[w];
                    bi = redi[w];
                    bp = redi[32 + w];
                }
            }
            tkey[round] = bk;
            tidx[round] = bi;
            gidx[bp] = -1;
        }
        __syncthreads();
    }
    ntop = keep;
    cnt = 0;
    __syncthreads();
}

// Rescore the gathered windows in fp64 and merge them with the running top-K.
static __device__ void flush_candidates(const SimParams& P, const RunDesc* runs, int R,
                                 const double* tmpl, int* gidx, double* gkey, int& cnt,
                                 double* tkey, int* tidx, int& ntop, int K, double* rsum,
                                 double* rnrm, double* redd, int* redi) {
    if (P.stats && threadIdx.x == 0) atomicAdd(&P.stats[0], static_cast<unsigned long long>(cnt));
    rescore_group(P, runs, R, tmpl, gidx, gkey, cnt, rsum, rnrm);
    merge_top(gkey, gidx, cnt, tkey, tidx, ntop, K, redd, redi);
}

// select_unconditional / select_conditional (matcher.hpp:207-241) over the
// ranked list: the job's precomputed draw, or the first candidate whose TI
// patch matches every hard datum of the footprint (else the fewest
// mismatches, earliest first).  Returns the chosen window position.
static __device__ int choose_candidate(const SimParams& P, const Job& jb, const int* tidx, int ntop, int* redi) {
    int pick = jb.pick;
    if (pick < 0) {
        int best = 0, best_mis = INT_MAX;
        pick = -1;
        const int cell = (jb.top / P.stride) * P.lat_nlc + jb.left / P.stride;
        const int e0 = P.hd_off[cell], e1 = P.hd_off[cell + 1];
        for (int c = 0; c < ntop; ++c) {
            const int pos = tidx[c];
            const int cfr = (pos / P.out_w) << P.J, cfc = (pos % P.out_w) << P.J;
            int mis = 0;
            for (int e = e0 + threadIdx.x; e < e1; e += SEL_T) {
                const uint32_t u = P.hd_ent[e];
                const int rc = static_cast<int>(u >> 8), r = rc / P.T, cc = rc - r * P.T;
                mis += P.ti[static_cast<size_t>(cfr + r) * P.ti_w + cfc + cc] != (u & 255u);
            }
            mis = block_reduce(mis, [](int a, int b) { return a + b; }, redi);
            if (mis == 0) {
                pick = c;
                break;
            }
            if (mis < best_mis) {
                best = c;
                best_mis = mis;
            }
        }
        if (pick < 0) pick = best;
    }
    return tidx[pick];
}

// crop + optional stitch + paste (simulator.hpp:483-493) of the TI patch at
// fine origin (fr, fc), the source-block map entries and the chosen origin.
static __device__ void paste_placement(const SimParams& P, const Job& jb, int gj, int fr, int fc, uint8_t* exist,
                                uint8_t* outp, int16_t* from, int* dp, int* seam) {
    const int tid = threadIdx.x;
    const int T = P.T;
    uint8_t* g = P.work ? P.work + static_cast<size_t>(jb.real) * P.wh * P.ww : nullptr;
    uint8_t* trace = P.pasted ? P.pasted + static_cast<size_t>(gj) * T * T : nullptr;
    if (P.min_cut && jb.shape != kNone) {
        for (int e = tid; e < T * T; e += SEL_T) {
            const int r = e / T, c = e - r * T;
            exist[e] = g[static_cast<size_t>(jb.top + r) * P.ww + jb.left + c];
            outp[e] = P.ti[static_cast<size_t>(fr + r) * P.ti_w + fc + c];
        }
        __syncthreads();
        min_cut_device(exist, outp, T, P.OV, jb.shape, jb.vleft, jb.htop, from, dp, seam);
        for (int e = tid; e < T * T; e += SEL_T) {
            const int r = e / T, c = e - r * T;
            g[static_cast<size_t>(jb.top + r) * P.ww + jb.left + c] = outp[e];
            if (trace) trace[e] = outp[e];
        }
    } else if (P.work || trace) {  // (no work grid: the source-block map is the realization)
        for (int e = tid; e < T * T; e += SEL_T) {
            const int r = e / T, c = e - r * T;
            const uint8_t v = P.ti[static_cast<size_t>(fr + r) * P.ti_w + fc + c];
            if (P.work) g[static_cast<size_t>(jb.top + r) * P.ww + jb.left + c] = v;
            if (trace) trace[e] = v;
        }
    }
    if (P.src) {  // (block coordinates by shifts: B = 2^J)
        const int J = P.J, Tc = P.Tc;
        int32_t* sm = P.src + static_cast<size_t>(jb.real) * (P.wh >> J) * P.swc +
                      static_cast<size_t>(jb.top >> J) * P.swc + (jb.left >> J);
        const int s0 = (fr >> J) * P.wc + (fc >> J);
        for (int e = tid; e < Tc * Tc; e += SEL_T) {
            const int a = e / Tc, b = e - a * Tc;
            sm[static_cast<size_t>(a) * P.swc + b] = s0 + a * P.wc + b;
        }
    }
    if (tid == 0) {
        P.chosen[2 * gj] = fr;
        P.chosen[2 * gj + 1] = fc;
    }
}

// The generic select + paste of the placement in job slot `slot` by the
// calling CTA (SEL_T threads): also the wave kernel's fallback (wave.cu).
static __device__ void select_paste_body(const SimParams& P, const Job* __restrict__ jobs, int job0, int slot,
                                  int use_screen, unsigned char* sel_sm) {
    const SelLayout L = sel_layout(P.K, P.T, P.OV, P.nch, P.Tc, P.scoring == 1);
    int* hist = reinterpret_cast<int*>(sel_sm + L.hist);
    int* misc = reinterpret_cast<int*>(sel_sm + L.misc);
    double* redd = reinterpret_cast<double*>(sel_sm + L.redd);
    int* redi = reinterpret_cast<int*>(sel_sm + L.redi);
    double* gkey = reinterpret_cast<double*>(sel_sm + L.gkey);
    int* gidx = reinterpret_cast<int*>(sel_sm + L.gidx);
    double* tkey = reinterpret_cast<double*>(sel_sm + L.tkey);
    int* tidx = reinterpret_cast<int*>(sel_sm + L.tidx);
    RunDesc* runs = reinterpret_cast<RunDesc*>(sel_sm + L.runs);
    double* tmpl = reinterpret_cast<double*>(sel_sm + L.tmpl);
    double* rsum = reinterpret_cast<double*>(sel_sm + L.rsum);
    double* rnrm = reinterpret_cast<double*>(sel_sm + L.rnrm);
    uint8_t* exist = sel_sm + L.exist;
    uint8_t* outp = sel_sm + L.outp;
    int16_t* from = reinterpret_cast<int16_t*>(sel_sm + L.from);
    int* dp = reinterpret_cast<int*>(sel_sm + L.dp);
    int* seam = reinterpret_cast<int*>(sel_sm + L.seam);

    const int gj = job0 + slot;
    const Job jb = jobs[gj];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (P.xrec && jb.shape == kNone) return;  // (position shards: the merge places first patches)
    int fr, fc;
    if (jb.shape == kNone) {
        fr = jb.fr;
        fc = jb.fc;
    } else {
        const int Tc = P.Tc;
        const int32_t* sc = P.scores + static_cast<size_t>(slot) * P.sld;
        const double* tm = P.tm64 + static_cast<size_t>(slot) * P.nch * Tc * Tc;
        const int K = P.K;
        // stage the job's fp64 template and its run list (matcher.hpp:44-61 order)
        for (int e = tid; e < P.nch * Tc * Tc; e += SEL_T) tmpl[e] = tm[e];
        int R = 0;
        {
            int rows = 0;
            for (int s = 0; s < Tc; ++s) {
                int t0, t1;
                mask_row_run(jb.shape, jb.vleft, jb.htop, Tc, P.OVc, s, t0, t1);
                rows += t1 > t0;
            }
            R = rows * P.nch;
            if (tid == 0) {
                int r = 0;
                for (int ch = 0; ch < P.nch; ++ch)
                    for (int s = 0; s < Tc; ++s) {
                        int t0, t1;
                        mask_row_run(jb.shape, jb.vleft, jb.htop, Tc, P.OVc, s, t0, t1);
                        if (t1 > t0) runs[r++] = {ch, s, t0, t1};
                    }
            }
        }
        // 1. exact screen threshold: every window whose integer score reaches
        //    the K-th largest can appear in the reference's top-K.
        const bool all = !use_screen;
        const int32_t* tmx = P.tmax ? P.tmax + static_cast<size_t>(slot) * P.ntiles : nullptr;
        int thr = 0;
        if (use_screen == 2) {
            // normalized: R = S / sqrt(NN) with S = S' + C_job and NN exact
            // integers; keys = R rounded down to float32 (monotone as int32
            // for R >= 0).  Every window the reference's fp64 score (relative
            // error << 1e-9) can rank in the top-K has R >= R_K (1 - 1e-9),
            // hence key >= the threshold below: a superset, rescored exactly.
            int32_t* scw = P.scores + static_cast<size_t>(slot) * P.sld;
            const int32_t* nn = P.nnmap + static_cast<size_t>(mask_variant(jb.shape, jb.vleft, jb.htop)) * (P.out_h * P.out_w) + P.p0;
            const int cj = P.cjob[slot];
            for (int p = tid; p < P.npos; p += SEL_T) {
                const int n = nn[p];
                const double R = n > 0 ? static_cast<double>(scw[p] + cj) / sqrt(static_cast<double>(n)) : 0.0;
                scw[p] = __float_as_int(__double2float_rd(R));
            }
            __syncthreads();
            const int kk = radix_kth_largest(sc, P.npos, K, hist, misc, redi);
            thr = __float_as_int(__double2float_rd(static_cast<double>(__int_as_float(kk)) * (1.0 - 1e-9)));
            tmx = nullptr;  // the tile maxima bound S', not the keys
        } else if (!all) {
            thr = radix_kth_largest(sc, P.npos, K, hist, misc, redi);
        }
        if (P.stats && tid == 0) atomicAdd(&P.stats[1], 1ull);
        __syncthreads();
        // 2. gather the tie group in row-major order, rescore in fp64, keep the
        //    running top-K by (fp64 desc, index asc).
        const int span = tmx ? kTcTile : SEL_T;
        const int nspans = (P.npos + span - 1) / span;
        int ntop = 0, cnt = 0;
        for (int sp = 0; sp < nspans; ++sp) {
            if (!all && tmx && tmx[sp] < thr) continue;  // uniform
            for (int sub = 0; sub < span; sub += SEL_T) {
                const int p = sp * span + sub + tid;
                const bool q = sub + tid < span && p < P.npos && (all || sc[p] >= thr);
                const unsigned bal = __ballot_sync(0xffffffffu, q);
                if (lane == 0) redi[wid] = __popc(bal);
                __syncthreads();
                int off = 0, tot = 0;
                for (int w = 0; w < SEL_T / 32; ++w) {
                    if (w < wid) off += redi[w];
                    tot += redi[w];
                }
                if (q) gidx[cnt + off + __popc(bal & ((1u << lane) - 1))] = p + P.p0;
                cnt += tot;
                __syncthreads();
                if (cnt + SEL_T > GCAP)
                    flush_candidates(P, runs, R, tmpl, gidx, gkey, cnt, tkey, tidx, ntop, K, rsum,
                                     rnrm, redd, redi);
            }
        }
        if (cnt > 0)
            flush_candidates(P, runs, R, tmpl, gidx, gkey, cnt, tkey, tidx, ntop, K, rsum, rnrm,
                             redd, redi);
        if (P.xrec) {  // position shard: hand the local top-K to the exchange
            ShardRec* xr = P.xrec + (static_cast<size_t>(P.xshard) * P.xnj + slot) * P.xk;
            for (int k = tid; k < P.xk; k += SEL_T)
                xr[k] = k < ntop ? ShardRec{tkey[k], tidx[k], 1} : ShardRec{0.0, -1, 0};
            return;
        }
        // 3. choose (matcher.hpp:207-241)
        const int pos = choose_candidate(P, jb, tidx, ntop, redi);
        fr = (pos / P.out_w) << P.J;
        fc = (pos % P.out_w) << P.J;
        __syncthreads();
    }
    // 4. crop + optional stitch + paste (simulator.hpp:483-493)
    paste_placement(P, jb, gj, fr, fc, exist, outp, from, dp, seam);
}


__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}

// K-th largest (with multiplicity) of the union of the lanes' sorted top
// lists (INT_MIN padded): rounds of warp max over the lanes' heads.
__device__ __forceinline__ int warp_kth(const int (&top)[kTcQ], int K, int lane) {
    int ptr = 0, acc = 0;
    for (int round = 0; round < kTcQ + 1; ++round) {
        int head = INT_MIN;
#pragma unroll
        for (int i = 0; i < kTcQ; ++i)
            if (i == ptr) head = top[i];
        int m = head;
        for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        int c = 0;
#pragma unroll
        for (int i = 0; i < kTcQ; ++i)
            if (i >= ptr && top[i] == m) ++c;
        ptr += c;
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        acc += c;
        if (acc >= K || m == INT_MIN) return m;
    }
    return INT_MIN;
}

// Conditional / unconditional choice among the ranked top-K (matcher.hpp:207-241):
// the host-drawn index, or the first zero-mismatch candidate against the hard
// data, else the fewest mismatches.  Warp-level; every warp of a job may run
// it redundantly (identical inputs, identical result).
__device__ __forceinline__ int choose_pick(const SimParams& P, const Job& jb, const int* tidx, int ntop,
                                        int lane) {
    int pick = jb.pick;
    if (pick < 0) {
        int best = 0, best_mis = INT_MAX;
        const int cell = (jb.top / P.stride) * P.lat_nlc + jb.left / P.stride;
        const int e0 = P.hd_off[cell], e1 = P.hd_off[cell + 1];
        for (int c = 0; c < ntop; ++c) {
            const int pos = tidx[c];
            const int cfr = (pos / P.out_w) << P.J, cfc = (pos % P.out_w) << P.J;
            int mis = 0;
            for (int e = e0 + lane; e < e1; e += 32) {
                const uint32_t u = P.hd_ent[e];
                const int rc = static_cast<int>(u >> 8), r = rc / P.T, cc = rc - r * P.T;
                mis += P.ti[static_cast<size_t>(cfr + r) * P.ti_w + cfc + cc] != (u & 255u);
            }
            for (int o = 16; o > 0; o >>= 1) mis += __shfl_xor_sync(0xffffffffu, mis, o);
            if (mis == 0) {
                pick = c;
                break;
            }
            if (mis < best_mis) {
                best = c;
                best_mis = mis;
            }
        }
        if (pick < 0) pick = best;
    }
    return tidx[pick];
}

// Paste the chosen TI crop (simulator.hpp:483-493), record the trace and the
// source-block map; JT threads cooperate (jt = 0..JT-1).
template <int JT>
__device__ __forceinline__ void paste_copy(const SimParams& P, const Job& jb, int gj, int fr, int fc, int jt) {
    const int Tc = P.Tc;
    const int T = P.T;
    uint8_t* trace = P.pasted ? P.pasted + static_cast<size_t>(gj) * T * T : nullptr;
    // Without a work grid (source-block map mode) the realization is rebuilt
    // from the map at finalize: only the map (and a requested trace) is written.
    uint8_t* g = P.work ? P.work + static_cast<size_t>(jb.real) * P.wh * P.ww : nullptr;
    const int wpr = T >> 2;  // 32-bit words per row
    const bool vec4 = ((fc | jb.left | P.ti_w | P.ww | T) & 3) == 0 && wpr <= JT && (JT % wpr) == 0;
    if (vec4) {
        // thread -> (row phase, word); every row it copies loaded in one round trip
        const int rpi = JT / wpr, rsub = jt / wpr, cw = jt - rsub * wpr;
        const uint8_t* srcp = P.ti + static_cast<size_t>(fr) * P.ti_w + fc + 4 * cw;
        uint8_t* dstp = g ? g + static_cast<size_t>(jb.top) * P.ww + jb.left + 4 * cw : nullptr;
        for (int r0 = rsub; r0 < T; r0 += rpi * 32) {
            uint32_t v[32];  // every row this lane copies, loaded in one round trip
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int r = r0 + i * rpi;
                if (r < T) v[i] = *reinterpret_cast<const uint32_t*>(srcp + static_cast<size_t>(r) * P.ti_w);
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int r = r0 + i * rpi;
                if (r < T) {
                    if (g) *reinterpret_cast<uint32_t*>(dstp + static_cast<size_t>(r) * P.ww) = v[i];
                    if (trace) *reinterpret_cast<uint32_t*>(trace + r * T + 4 * cw) = v[i];
                }
            }
        }
    } else {
        // unaligned rows: byte copies, 16 loads in flight per thread
        constexpr int BB = 16;
        for (int e0 = 0; e0 < T * T; e0 += JT * BB) {
            uint8_t v[BB];
#pragma unroll
            for (int i = 0; i < BB; ++i) {
                const int e = e0 + i * JT + jt;
                const int r = e / T, c = e - r * T;
                if (e < T * T) v[i] = P.ti[static_cast<size_t>(fr + r) * P.ti_w + fc + c];
            }
#pragma unroll
            for (int i = 0; i < BB; ++i) {
                const int e = e0 + i * JT + jt;
                const int r = e / T, c = e - r * T;
                if (e < T * T) {
                    if (g) g[static_cast<size_t>(jb.top + r) * P.ww + jb.left + c] = v[i];
                    if (trace) trace[e] = v[i];
                }
            }
        }
    }
}

template <int JT>
__device__ __forceinline__ void paste_job(const SimParams& P, const Job& jb, int gj, int fr, int fc,
                                          int jt) {
    const int Tc = P.Tc;
    // Without a work grid (source-block map mode) the realization is rebuilt
    // from the map at finalize: only the map (and a requested trace) is written.
    if (P.work || P.pasted) paste_copy<JT>(P, jb, gj, fr, fc, jt);
    if (P.src) {  // Tc x Tc map entries spread over every thread
        // (B = 2^J: shifts, not integer divisions -- this is on every
        //  placement's critical path; a power-of-two Tc splits e by shifts too)
        const int J = P.J;
        int32_t* sm = P.src + static_cast<size_t>(jb.real) * (P.wh >> J) * P.swc +
                      static_cast<size_t>(jb.top >> J) * P.swc + (jb.left >> J);
        const int s0 = (fr >> J) * P.wc + (fc >> J);
        const bool pow2 = (Tc & (Tc - 1)) == 0;
        const int lt = __ffs(Tc) - 1;
        for (int e = jt; e < Tc * Tc; e += JT) {
            const int a = pow2 ? e >> lt : e / Tc, b = e - a * Tc;
            sm[static_cast<size_t>(a) * P.swc + b] = s0 + a * P.wc + b;
        }
    }
}


}  // namespace ccwgpu
