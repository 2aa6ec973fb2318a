// ccw_device.cuh -- device-side building blocks shared by the kernels.
//
// Exactness contract: everything that reproduces a reference
// double uses explicit round-to-nearest intrinsics (__dmul_rn / __dadd_rn /
// __ddiv_rn / __dsqrt_rn), so nvcc can never contract it into an FMA, and
// follows the reference's operation order literally.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ccwgpu {

constexpr double kInvSqrt2 = 0.70710678118654752440084436210485;  // wavelet.hpp:17
constexpr int kMaxLevels = 12;
constexpr uint8_t kNoDatum = 255;

enum OrShape : int { kNone = 0, kVertical = 1, kHorizontal = 2, kL = 3 };  // simulator.hpp:87

// One placement of one realization, as scheduled on the device.
struct Job {
    int32_t real;    // realization index within the call
    int32_t place;   // placement index in the reference raster order
    int32_t top;     // fine-grid footprint origin in the work grid
    int32_t left;
    int32_t shape;   // OrShape
    int32_t vleft;   // vertical strip on the left (plan.vertical_on_left())
    int32_t htop;    // horizontal strip on top (plan.horizontal_on_top())
    int32_t pick;    // unconditional: precomputed bounded(rng, K') draw; -1 = conditional
    int32_t fr;      // first placement: precomputed block-aligned TI origin
    int32_t fc;
    int32_t dep0;    // fused OR prep: flat index of a next-wave placement that reads this
    int32_t dep1;    //   one's paste ((o, i+1) and (o+1, i-1)), -1 = none
    int32_t ndep;    //   previous-wave placements this one reads ((o, i-1), (o-1, i+1))
};

// Candidate-position sharding: one entry of a shard's top-K list (fp64
// reference score, global row-major window position; pos < 0 = empty slot).
// valid = 0: the fast select ranked the window by its exact screen score
// alone (no other local candidate shares it), so key is absent and the merge
// rescores it -- windows of different shards may share a screen score.
struct ShardRec {
    double key;
    int32_t pos;
    int32_t valid;
};

// Parameters shared by every job of one simulate call.
constexpr int kNumStats = 48;  // device counters per simulation call (SimParams::stats)

// Shared rescoring (select_fast_kernel): a placement with a large equal-score
// group posts it in chunks; the launch's CTAs that finish their own placement
// claim and rescore chunks.  One board (+ per-slot counters) per launch.
constexpr int HB_CAP = 1024;  // posts per board
struct HelpBoard {
    int nposts;
    int pad[3];
    int posts[HB_CAP];  // slot + 1 (0: being written)
};
// per slot of a board: int4 (next chunk, finished chunks, windows,
// windows per chunk | mask variant << 16)

struct SimParams {
    // training image
    const uint8_t* ti;       // h*w codes
    const double* ti64;      // nch planes hc*wc: reference-order apex values
    const float* tiscr;      // nscr planes hc*wc: exact block-sum screen planes
    int ti_h, ti_w, hc, wc;
    int F, J, mode;          // mode 0 indicator, 1 raw_codes
    int nch, nscr;
    // geometry
    int T, OV, Tc, OVc, B;   // B = 2^J
    int out_h, out_w, npos;  // score-map extent
    int K;                   // min(candidates, npos)
    int scoring;             // 0 raw, 1 normalized
    int min_cut;
    int any_support;         // literal-config extension: OV may not be a multiple of B; the
                             // overlap prep counts only the supported fine cells of a block
    // simulation grid
    uint8_t* work;           // n_real planes of wh*ww
    int wh, ww;
    const uint8_t* hd;       // wh*ww plane, kNoDatum = none; may be null
    const int32_t* hd_off;   // per stride-lattice cell: CSR offsets into hd_ent (null without hard data)
    const uint32_t* hd_ent;  // (footprint cell r*T+c) << 8 | facies
    int lat_nlc, stride;     // lattice columns, placement stride T - OV
    int32_t* src;            // n_real planes of (wh/B)*(ww/B): TI coarse index each work block
                             // was pasted from (null with min-cut, whose blocks mix sources)
    int swc;                 // ww / B
    // per-job scratch (indexed by job slot within a launch chunk)
    int32_t* wts;            // nscr*Tc*Tc integer screen weights (fp32 screen)
    int8_t* wts8;            // kpad int8 screen weights per job (tcgen05 screen), may be null
    const int8_t* im2col;    // npos x kpad int8 TI windows (tcgen05 screen), may be null
    int kpad;
    int32_t* tmax;           // per job: ntiles tile maxima of the screen (tcgen05), may be null
    int ntiles;
    unsigned long long* stats;  // [0] windows rescored in fp64, [1] screened jobs
    double* tm64;            // nch*Tc*Tc reference-order OR apex values
    int32_t* scores;         // npos screen scores per job, row stride sld (16-byte rows)
    int sld;
    int s16;                 // fast select: score rows hold int16 (exact when |S| < 2^15, host-checked)
    int* defer;              // per job slot: threshold handed to select_bulk_kernel, INT_MIN = none
    int* defer_list;         // deferred job slots of this launch (appended by the fast select)
    int* defer_cnt;          //   ... their count (two counters alternate by launch parity:
    int* defer_cnt_next;     //   the bulk launch zeroes the next launch's)
    // fused OR prep: the select of wave w prepares the placements of wave w+1
    // once both of their wave-w dependencies have pasted (null: separate launch)
    int* depcnt;             // per next-wave slot: dependencies that have pasted
    int* depflag;            // dependency flags (option flagprep): per flat job, the previous-wave
                             // placements it reads that have pasted (select -> OR prep of the next wave)
    int next_j0;             // flat index of the next wave's first job (this group)
    int8_t* n_wts8;          // next wave's prep outputs (the other parity buffers)
    double* n_tm64;
    int32_t* n_cjob;
    unsigned long long* tl;  // debug timeline slot of this launch (null unless CCW_TIMELINE)
    int bulk_bx, bulk_by;    // select_bulk_kernel window block (positions per shared-memory tile)
    int32_t* cjob;           // normalized screen: per job slot, S = S' + cjob (null otherwise)
    const int4* mtab;        // fast select: mask rows and run groups per mask variant
    int ustride;             // row stride of umap (a multiple of 256 >= npos)
    int8_t* jvar;            // per job slot: mask variant (written by the OR prep; null: unused)
    int32_t* tmax_nu;        // per job slot: per tile the max score over non-uniform windows (null: off)
    const double* pure_apex; // [16][nch] apex values of a pure block of facies f (any: they are equal)
    const int* ufirst;       // [8 variants][16 classes][kTcQ] lowest window positions of each uniform class
    const int8_t* umap;      // fast select: [8 mask variants][npos] uniform class of each window --
                             // the facies every masked coarse block is made of (pure blocks), -1 if
                             // none; same class => bit-identical fp64 score (null: off)
    const int32_t* nnmap;    // normalized screen: [8 mask variants][npos] sum over mask and
                             // channels of squared TI block counts (null otherwise)
    HelpBoard* hb;           // shared rescoring board of this launch (null: off)
    int4* hs;                //   ... its per-slot counters
    HelpBoard* hb_reset;     // board of the next launch (reset by block 0)
    int4* hs_reset;          //   ... its per-slot counters
    int hs_n;                // slots per board
    int* hpos;               // per job slot: SC_LC posted window positions
    double* hkeys;           //   ... their fp64 keys
    int help_min;            // smallest group that is shared
    unsigned long long* jdump;  // debug (CCW_DBG_TAIL builds, CCW_TAIL_DUMP): per job t0, t1, t_end, n | g << 32
    int* bulk_sync;          // per job slot: [next position block, finished CTAs]
    double* bulk_keys;       // per job slot x CTA: that CTA's top-K keys
    int* bulk_idx;           //   ... and positions
    // candidate-position sharding: the select screens window positions
    // [p0, p0 + npos) (scores / tmax rows are shard-local) and writes its
    // top-K to xrec[(xshard * xnj + slot) * xk + k] instead of pasting
    int p0;
    ShardRec* xrec;          // null: normal select
    int xnj, xk, xshard;
    // outputs
    int32_t* chosen;         // per job (global job id): fr, fc
    uint8_t* pasted;         // optional trace of pasted patches (global job id * T*T)
};

// Screen scores of job slot `slot` (int32 rows, or int16 rows when P.s16):
// four at p0 (a multiple of 4), or one.
template <bool S16>
__device__ __forceinline__ int4 load_score4(const SimParams& P, int slot, int p0) {
    const size_t o = static_cast<size_t>(slot) * P.sld + p0;
    if (S16) {
        const uint2 u = *reinterpret_cast<const uint2*>(reinterpret_cast<const int16_t*>(P.scores) + o);
        return make_int4(static_cast<int16_t>(u.x & 0xffffu), static_cast<int16_t>(u.x >> 16),
                         static_cast<int16_t>(u.y & 0xffffu), static_cast<int16_t>(u.y >> 16));
    }
    return *reinterpret_cast<const int4*>(P.scores + o);
}
__device__ __forceinline__ int load_score(const SimParams& P, int slot, size_t p) {
    const size_t o = static_cast<size_t>(slot) * P.sld + p;
    return P.s16 ? static_cast<int>(reinterpret_cast<const int16_t*>(P.scores)[o]) : P.scores[o];
}

// Row-major run of the coarse overlap mask in template row s: [t0, t1).
// Every simulator mask (strip or L, simulator.hpp:194-215) has at most one
// maximal run per row, so mask_runs (matcher.hpp:44-61) reduces to this.
__host__ __device__ __forceinline__ void mask_row_run(int shape, int vleft, int htop, int Tc, int OVc,
                                             int s, int& t0, int& t1) {
    const bool vert = shape == kVertical || shape == kL;
    const bool horz = shape == kHorizontal || shape == kL;
    const bool in_h = horz && (htop ? s < OVc : s >= Tc - OVc);
    if (in_h) {
        t0 = 0;
        t1 = Tc;
    } else if (vert) {
        t0 = vleft ? 0 : Tc - OVc;
        t1 = t0 + OVc;
    } else {
        t0 = 0;
        t1 = 0;
    }
}

// Level-J Haar apex of one 2^J x 2^J block in the reference's exact order.
// The reference transforms whole planes level by level (wavelet.hpp:163-168);
// by locality each apex value depends only on its block, through the tree
//   a = s*((s*A00 + s*A01) + (s*A10 + s*A11))      (wavelet.hpp:29, :99)
// over the four level-(j-1) quadrant values.  Visiting the leaves in Morton
// order and folding every completed quartet reproduces that tree exactly.
// leaf(code) is the indicator (mode 0, facies f) or the raw code (mode 1).
__device__ __forceinline__ double haar_apex_block(const uint8_t* cells, int ld, int J, int mode,
                                                  int f) {
    double st[kMaxLevels][4];
    int cnt[kMaxLevels];
    for (int l = 0; l < J; ++l) cnt[l] = 0;
    const int n = 1 << (2 * J);
    for (int k = 0; k < n; ++k) {
        int r = 0, c = 0;
        for (int b = 0; b < J; ++b) {
            c |= ((k >> (2 * b)) & 1) << b;
            r |= ((k >> (2 * b + 1)) & 1) << b;
        }
        const int code = cells[r * ld + c];
        double x = mode == 0 ? (code == f ? 1.0 : 0.0) : (double)code;
        int l = 0;
        st[0][cnt[0]++] = x;
        while (cnt[l] == 4) {
            const double lo0 = __dadd_rn(__dmul_rn(kInvSqrt2, st[l][0]), __dmul_rn(kInvSqrt2, st[l][1]));
            const double lo1 = __dadd_rn(__dmul_rn(kInvSqrt2, st[l][2]), __dmul_rn(kInvSqrt2, st[l][3]));
            const double a = __dmul_rn(kInvSqrt2, __dadd_rn(lo0, lo1));
            cnt[l] = 0;
            ++l;
            if (l == J) return a;
            st[l][cnt[l]++] = a;
        }
    }
    return 0.0;  // unreachable for J >= 1
}

// Exact-integer block statistic used by the screen: the count of facies f
// (mode 0) or the sum of codes (mode 1) over one 2^J x 2^J block.
__device__ __forceinline__ int block_stat(const uint8_t* cells, int ld, int B, int mode, int f) {
    int acc = 0;
    for (int r = 0; r < B; ++r)
        for (int c = 0; c < B; ++c) {
            const int code = cells[r * ld + c];
            acc += mode == 0 ? (code == f) : code;
        }
    return acc;
}

// Fine-cell overlap support of a template (simulator.hpp:194-215): strips of
// width OV on the origin's sides.
__device__ __forceinline__ bool fine_support(int shape, int vleft, int htop, int T, int OV, int r, int c) {
    const bool vert = shape == kVertical || shape == kL;
    const bool horz = shape == kHorizontal || shape == kL;
    return (vert && (vleft ? c < OV : c >= T - OV)) || (horz && (htop ? r < OV : r >= T - OV));
}

// haar_apex_block / block_stat over only the supported fine cells of a block
// at template offset (r0, c0): extract_or's zeros stand for the others
// (simulator.hpp:225-252) -- the literal-config extension's partial blocks.
__device__ __forceinline__ double haar_apex_block_sup(const uint8_t* cells, int ld, int J, int mode, int f, int r0,
                                                      int c0, int shape, int vleft, int htop, int T, int OV) {
    double st[kMaxLevels][4];
    int cnt[kMaxLevels];
    for (int l = 0; l < J; ++l) cnt[l] = 0;
    const int n = 1 << (2 * J);
    for (int k = 0; k < n; ++k) {
        int r = 0, c = 0;
        for (int b = 0; b < J; ++b) {
            c |= ((k >> (2 * b)) & 1) << b;
            r |= ((k >> (2 * b + 1)) & 1) << b;
        }
        double x = 0.0;
        if (fine_support(shape, vleft, htop, T, OV, r0 + r, c0 + c)) {
            const int code = cells[r * ld + c];
            x = mode == 0 ? (code == f ? 1.0 : 0.0) : (double)code;
        }
        int l = 0;
        st[0][cnt[0]++] = x;
        while (cnt[l] == 4) {
            const double lo0 = __dadd_rn(__dmul_rn(kInvSqrt2, st[l][0]), __dmul_rn(kInvSqrt2, st[l][1]));
            const double lo1 = __dadd_rn(__dmul_rn(kInvSqrt2, st[l][2]), __dmul_rn(kInvSqrt2, st[l][3]));
            const double a = __dmul_rn(kInvSqrt2, __dadd_rn(lo0, lo1));
            cnt[l] = 0;
            ++l;
            if (l == J) return a;
            st[l][cnt[l]++] = a;
        }
    }
    return 0.0;
}

__device__ __forceinline__ int block_stat_sup(const uint8_t* cells, int ld, int B, int mode, int f, int r0, int c0,
                                              int shape, int vleft, int htop, int T, int OV) {
    int acc = 0;
    for (int r = 0; r < B; ++r)
        for (int c = 0; c < B; ++c) {
            if (!fine_support(shape, vleft, htop, T, OV, r0 + r, c0 + c)) continue;
            const int code = cells[r * ld + c];
            acc += mode == 0 ? (code == f) : code;
        }
    return acc;
}

// Programmatic dependent launch (PDL): a kernel lets its stream successor
// start launching early, and waits for its predecessor's completion (and
// memory) before reading what the predecessor wrote.  Both are no-ops for a
// kernel launched without the programmatic-serialization attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Debug timeline (CCW_TIMELINE): per launch [first CTA past its dependency
// wait, last CTA end, first CTA resident] in globaltimer ns.
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void tl_mark(unsigned long long* tl, int k) {
    if (tl && threadIdx.x == 0) {
        const unsigned long long t = gtimer();
        if (k == 1) {
            atomicMax(&tl[1], t);
        } else {
            atomicMin(&tl[k], t);
            if (k == 0) atomicMax(&tl[3], t);  // last CTA past its wait
        }
    }
}

// Block-wide reductions for blockDim.x a multiple of 32 (<= 1024).
template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, Op op, T* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    T r = red[0];
    for (int i = 1; i < nw; ++i) r = op(r, red[i]);
    return r;
}

}  // namespace ccwgpu
