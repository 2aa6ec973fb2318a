// ccf_tc.hpp -- host interface of the tcgen05 int8 CCF screen (ccf_tc.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

struct ccw_ti;

namespace ccwgpu {

constexpr int kTcQ = 8;       // largest K the warp / bulk selects take (top-K kept in registers)
constexpr int kTcTile = 128;  // positions per tile maximum (half a tcgen05 N tile)

struct TcArgs {
    int nj;          // jobs in this launch chunk (rows of W)
    int npos;        // score-map positions (rows of X)
    int sld;         // row stride of scores (multiple of 4 ints)
    int nk;          // K stages of 128 bytes
    int ntiles;      // tiles of kTcTile positions
    int32_t* scores;   // [nj][sld] exact screen scores
    int32_t* tmax;     // [nj][ntiles] maximum score of each tile
    unsigned long long* probe;  // debug phase clocks (null unless CCW_TC_PROBE)
    unsigned long long* tl;     // debug timeline slot (null unless CCW_TIMELINE)
    int s16;                    // score rows as int16 (exact: the host checks |S| < 2^15)
    int epi_in_ring;            // every CTA drains one tile: the epilogue's transpose
                                // staging reuses the (then idle) TMA ring
    // optional: per tile the maximum over NON-uniform windows (tie-storm
    // placements skip the uniform classes, whose scores are class constants)
    int32_t* tmax_nu;           // [nj][ntiles] (null: off)
    const uint32_t* ubits;      // [8][ustride / 32] non-uniform windows as bits
    int ustride;
    const int8_t* jvar;         // [nj] mask variant of each job
};

size_t ccf_tc_smem_bytes(bool epi_in_ring = false);
extern unsigned long long* tc_probe_buffer;  // debug: ccf phase clocks (CCW_TC_PROBE)
int tc_kpad(int nscr, int Tc);
int tc_tiles(int npos);
int tc_num_sms();
// im2col of the TI screen planes for template size Tc (cached on the TI).
const int8_t* ti_im2col(ccw_ti* ti, int Tc, cudaStream_t st);
// Measured dense int8 tcgen05 rate of the screen's MMA shape (TOPS).
double measure_i8_peak(cudaStream_t st);
// The screen kernel alone on njobs placements, back-to-back launches (ms per launch).
double measure_ccf_screen(ccw_ti* ti, int Tc, int njobs, int iters, cudaStream_t st);

// TMA descriptors, built once per simulate call and group.
struct TcPlan {
    CUtensorMap ma, mb;
};
TcPlan plan_ccf_tc(const int8_t* d_w8, int maxj, const int8_t* d_x, int npos, int kpad);
void launch_ccf_tc(const TcPlan& pl, int npos, int sld, int kpad, int nj, int32_t* scores,
                   int32_t* tmax, cudaStream_t st, unsigned long long* tl = nullptr,
                   int tmax_ld = -1,   // tmax row stride (default: this launch's tile count)
                   int s16 = 0, int32_t* tmax_nu = nullptr, const uint32_t* ubits = nullptr, int ustride = 0,
                   const int8_t* jvar = nullptr);       // store int16 score rows

}  // namespace ccwgpu
