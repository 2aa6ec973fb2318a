// Device-side schedule: every realization's placement jobs, built on the GPU.
//
// The reference plans each realization on the host (simulator.hpp:148-190,
// 440-470): a std::mt19937_64 seeded with the realization seed draws the
// raster path (origin, major order), then one draw per unconditional
// placement (the rank of the pick among the K candidates) and two for the
// first placement (its block-aligned TI origin).  Here one thread per
// realization replays that exact sequence -- std::mt19937_64 is pinned by the
// C++ standard ([rand.eng.mers], [rand.predef]) and bounded() is
// rng.hpp:21-28 -- and writes the jobs straight into the wave-ordered job
// array, so the host neither builds nor uploads them.
#include "sim_kernels.cuh"

namespace ccwgpu {

namespace {

constexpr int kMtN = 312, kMtM = 156;

struct Mt64 {
    uint64_t x[kMtN];
    int i;
};

__device__ __forceinline__ void mt_seed(Mt64& m, uint64_t s) {
    m.x[0] = s;
    for (int i = 1; i < kMtN; ++i) m.x[i] = 6364136223846793005ULL * (m.x[i - 1] ^ (m.x[i - 1] >> 62)) + i;
    m.i = kMtN;
}

__device__ __forceinline__ void mt_twist(Mt64& m) {
    constexpr uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL, kA = 0xB5026F5AA96619E9ULL;
    int k = 0;
    for (; k < kMtN - kMtM; ++k) {
        const uint64_t y = (m.x[k] & kUpper) | (m.x[k + 1] & kLower);
        m.x[k] = m.x[k + kMtM] ^ (y >> 1) ^ ((y & 1) ? kA : 0);
    }
    for (; k < kMtN - 1; ++k) {
        const uint64_t y = (m.x[k] & kUpper) | (m.x[k + 1] & kLower);
        m.x[k] = m.x[k + kMtM - kMtN] ^ (y >> 1) ^ ((y & 1) ? kA : 0);
    }
    const uint64_t y = (m.x[kMtN - 1] & kUpper) | (m.x[0] & kLower);
    m.x[kMtN - 1] = m.x[kMtM - 1] ^ (y >> 1) ^ ((y & 1) ? kA : 0);
    m.i = 0;
}

__device__ __forceinline__ uint64_t mt_next(Mt64& m) {
    if (m.i >= kMtN) mt_twist(m);
    uint64_t y = m.x[m.i++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

// rng.hpp:21-28: rejection below (2^64 - n) mod n, then r mod n.
__device__ __forceinline__ uint64_t mt_bounded(Mt64& m, uint64_t n) {
    const uint64_t threshold = (0 - n) % n;
    for (;;) {
        const uint64_t r = mt_next(m);
        if (r >= threshold) return r % n;
    }
}

}  // namespace

namespace {

struct PathGeom {
    bool cm, rows_asc, cols_asc, vleft, htop;
    int no, ni;
};

__device__ __forceinline__ PathGeom path_geom(const SchedParams& S, int origin, bool cm) {
    PathGeom g;
    g.cm = cm;
    g.rows_asc = origin == kTopLeft || origin == kTopRight;
    g.cols_asc = origin == kTopLeft || origin == kBottomLeft;
    g.vleft = origin == kTopLeft || origin == kBottomLeft;
    g.htop = origin == kTopLeft || origin == kTopRight;
    g.no = cm ? S.nlc : S.nlr;
    g.ni = cm ? S.nlr : S.nlc;
    return g;
}

// Placement (o, i) of realization r as a job (make_plan_from order, k = o * ni + i).
__device__ __forceinline__ Job make_job(const SchedParams& S, const PathGeom& g, int r, int o, int i, int pick,
                                        int fr, int fc) {
    const int ro = g.cm ? i : o, co = g.cm ? o : i;  // row / column lattice index in path order
    const int rq = g.rows_asc ? ro : S.nlr - 1 - ro, cq = g.cols_asc ? co : S.nlc - 1 - co;
    Job jb;
    jb.real = r;
    jb.place = o * g.ni + i;
    jb.top = rq * S.stride;
    jb.left = cq * S.stride;
    jb.shape = o == 0 && i == 0 ? kNone
               : o == 0         ? (g.cm ? kHorizontal : kVertical)
               : i == 0         ? (g.cm ? kVertical : kHorizontal)
                                : kL;
    jb.vleft = g.vleft;
    jb.htop = g.htop;
    jb.pick = pick;
    jb.fr = fr;
    jb.fc = fc;
    return jb;
}

__device__ __forceinline__ bool is_cond(const SchedParams& S, const PathGeom& g, int o, int i) {
    if (!S.lattice_hd) return false;
    const int ro = g.cm ? i : o, co = g.cm ? o : i;
    const int rq = g.rows_asc ? ro : S.nlr - 1 - ro, cq = g.cols_asc ? co : S.nlc - 1 - co;
    return S.lattice_hd[static_cast<size_t>(rq) * S.nlc + cq] != 0;
}

// flat index of placement (o, i): its realization's first slot in wave
// keymul*o + i, plus its earlier placements (o' < o) in the same wave
__device__ __forceinline__ int flat_index(const SchedParams& S, const int32_t* roff, int ni, int o, int i) {
    const int km = S.keymul, key = km * o + i;
    const int lo = key - ni + 1 <= 0 ? 0 : (key - ni + 1 + km - 1) / km;
    const int hi = min(o - 1, key / km);
    return roff[key] + max(0, hi - lo + 1);
}

__device__ __forceinline__ void write_job(const SchedParams& S, Job* jobs, const int32_t* roff, const PathGeom& g,
                                          int r, int o, int i, int pick, int fr, int fc) {
    Job jb = make_job(S, g, r, o, i, pick, fr, fc);
    jb.dep0 = i + 1 < g.ni ? flat_index(S, roff, g.ni, o, i + 1) : -1;
    jb.dep1 = (o + 1 < g.no && i >= 1) ? flat_index(S, roff, g.ni, o + 1, i - 1) : -1;
    jb.ndep = (i >= 1 ? 1 : 0) + (o >= 1 && i + 1 < g.ni ? 1 : 0);
    jobs[flat_index(S, roff, g.ni, o, i)] = jb;
}

__device__ __forceinline__ uint64_t temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

}  // namespace

// One warp per realization.  The generator state is twisted by the whole warp
// (the recurrence is parallel within a block of 312 words), the outputs are
// tempered into scratch, and each placement reads its draws at its offset in
// the draw sequence -- exact whenever no draw is rejected by bounded(), which
// the warp checks; otherwise lane 0 replays the realization sequentially.
__global__ void __launch_bounds__(32) build_jobs_kernel(SchedParams S, Job* __restrict__ jobs) {
    __shared__ uint64_t x[kMtN];
    const int r = blockIdx.x, lane = threadIdx.x;
    if (r >= S.n_real) return;
    const int32_t* roff = S.roff + static_cast<size_t>(r) * S.nkeys;
    uint64_t* outs = S.outs + static_cast<size_t>(r) * S.nout;
    constexpr uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL, kA = 0xB5026F5AA96619E9ULL;
    if (lane == 0) {
        uint64_t v = S.seeds[r];
        x[0] = v;
        for (int q = 1; q < kMtN; ++q) {
            v = 6364136223846793005ULL * (v ^ (v >> 62)) + q;
            x[q] = v;
        }
    }
    __syncwarp();
    for (int b = 0; b * kMtN < S.nout; ++b) {  // twist (three dependent phases) and temper one block
        uint64_t nv[5];
#pragma unroll
        for (int u = 0; u < 5; ++u) {
            const int q = lane + 32 * u;
            if (q < kMtN - kMtM) {
                const uint64_t y = (x[q] & kUpper) | (x[q + 1] & kLower);
                nv[u] = x[q + kMtM] ^ (y >> 1) ^ ((y & 1) ? kA : 0);
            }
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 5; ++u) {
            const int q = lane + 32 * u;
            if (q < kMtN - kMtM) x[q] = nv[u];
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 5; ++u) {
            const int q = kMtN - kMtM + lane + 32 * u;
            if (q < kMtN - 1) {
                const uint64_t y = (x[q] & kUpper) | (x[q + 1] & kLower);
                nv[u] = x[q - (kMtN - kMtM)] ^ (y >> 1) ^ ((y & 1) ? kA : 0);
            }
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 5; ++u) {
            const int q = kMtN - kMtM + lane + 32 * u;
            if (q < kMtN - 1) x[q] = nv[u];
        }
        __syncwarp();
        if (lane == 0) {
            const uint64_t y = (x[kMtN - 1] & kUpper) | (x[0] & kLower);
            x[kMtN - 1] = x[kMtM - 1] ^ (y >> 1) ^ ((y & 1) ? kA : 0);
        }
        __syncwarp();
        for (int q = lane; q < kMtN && b * kMtN + q < S.nout; q += 32) outs[b * kMtN + q] = temper(x[q]);
        __syncwarp();
    }
    // draws 0, 1: the path (bounded(4), bounded(2) never reject)
    const uint64_t o0 = outs[0], o1 = outs[1];
    const int origin = static_cast<int>(o0 % 4);
    const bool cm = o1 % 2 == 1;
    if (lane == 0 && origin * 2 + (cm ? 1 : 0) != S.vid[r]) atomicExch(S.err, 1);
    const PathGeom g = path_geom(S, origin, cm);
    const int cnt = g.no * g.ni;
    // placements in chunks of 32: draw counts, their offsets, the draws
    int dc = 2;
    bool reject = false;
    for (int k0 = 0; k0 < cnt; k0 += 32) {
        const int k = k0 + lane;
        const int o = k / g.ni, i = k - o * g.ni;
        const bool in = k < cnt;
        const bool cond = in && k > 0 && is_cond(S, g, o, i);
        const int nd = !in ? 0 : k == 0 ? 2 : cond ? 0 : 1;
        int incl = nd;
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, s);
            if (lane >= s) incl += y;
        }
        const int base = dc + incl - nd;
        dc += __shfl_sync(0xffffffffu, incl, 31);
        int pick = 0, fr = 0, fc = 0;
        bool rej = false;
        if (in && base + nd <= S.nout) {
            if (k == 0) {  // simulator.hpp:450-453
                const uint64_t a = outs[base], c = outs[base + 1];
                rej = a < S.thr_fr || c < S.thr_fc;
                fr = static_cast<int>(a % S.nfr) * S.B;
                fc = static_cast<int>(c % S.nfc) * S.B;
            } else if (cond) {
                pick = -1;
            } else {
                const uint64_t a = outs[base];
                rej = a < S.thr_k;
                pick = static_cast<int>(a % static_cast<uint64_t>(S.Kp));
            }
        } else if (in) {
            rej = true;  // (past the generated outputs: only after rejections)
        }
        reject |= __any_sync(0xffffffffu, rej);
        if (in) write_job(S, jobs, roff, g, r, o, i, pick, fr, fc);
    }
    if (!reject) return;
    __syncwarp();
    if (lane == 0) {  // a draw was rejected: replay the realization sequentially (rng.hpp:21-28)
        Mt64& m = *reinterpret_cast<Mt64*>(S.replay + static_cast<size_t>(r) * (kMtN + 1));
        mt_seed(m, S.seeds[r]);
        mt_bounded(m, 4);
        mt_bounded(m, 2);
        for (int k = 0; k < cnt; ++k) {
            const int o = k / g.ni, i = k - o * g.ni;
            int pick = 0, fr = 0, fc = 0;
            if (k == 0) {
                fr = static_cast<int>(mt_bounded(m, S.nfr)) * S.B;
                fc = static_cast<int>(mt_bounded(m, S.nfc)) * S.B;
            } else if (is_cond(S, g, o, i)) {
                pick = -1;
            } else {
                pick = static_cast<int>(mt_bounded(m, static_cast<uint64_t>(S.Kp)));
            }
            write_job(S, jobs, roff, g, r, o, i, pick, fr, fc);
        }
    }
}

}  // namespace ccwgpu
