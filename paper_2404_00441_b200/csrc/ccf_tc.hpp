// ccf_tc.hpp -- host interface of the tcgen05 int8 CCF screen (ccf_tc.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

struct ccw_ti;

namespace ccwgpu {

constexpr int kTcQ = 8;     // per-(job, tile) summary slots: top scores with multiplicity
constexpr int kTcTile = 128;  // positions per summary (half a tcgen05 N tile)

struct TcArgs {
    int nj;          // jobs in this launch chunk (rows of W)
    int npos;        // score-map positions (rows of X)
    int sld;         // row stride of scores (multiple of 4 ints)
    int nk;          // K stages of 128 bytes
    int ntiles;      // summary tiles of kTcTile positions
    int32_t* scores;   // [nj][sld] exact screen scores (block-select path), or null
    int32_t* ovf;      // [nj][sld] scores of tie-overflowing half tiles only (warp path), or null
    int2* summary;     // [nj][ntiles][kTcQ] top-Q (score, position) per tile ordered by
                       // (score desc, position asc), INT_MIN padded; position -2 marks a
                       // tile whose ties overflowed the list (its scores are in ovf)
};

size_t ccf_tc_smem_bytes();
int tc_kpad(int nscr, int Tc);
int tc_tiles(int npos);
int tc_num_sms();
int tc_qdepth(int K);
// im2col of the TI screen planes for template size Tc (cached on the TI).
const int8_t* ti_im2col(ccw_ti* ti, int Tc, cudaStream_t st);
// Measured dense int8 tcgen05 rate of the screen's MMA shape (TOPS).
double measure_i8_peak(cudaStream_t st);

// TMA descriptors + kernel choice, built once per simulate call and group.
struct TcPlan {
    CUtensorMap ma, mb;
    int q;
};
TcPlan plan_ccf_tc(const int8_t* d_w8, int maxj, const int8_t* d_x, int npos, int kpad, int K);
void launch_ccf_tc(const TcPlan& pl, int npos, int sld, int kpad, int nj, int32_t* scores,
                   int32_t* ovf, int2* summary, cudaStream_t st);

}  // namespace ccwgpu
