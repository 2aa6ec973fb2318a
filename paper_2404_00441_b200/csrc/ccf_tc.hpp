// ccf_tc.hpp -- host interface of the tcgen05 int8 CCF screen (ccf_tc.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

struct ccw_ti;

namespace ccwgpu {

constexpr int kTcQ = 8;     // per-(job, tile) summary depth: top-8 scores with multiplicity
constexpr int kTcTile = 128;  // positions per summary (half a tcgen05 N tile)

struct TcArgs {
    int nj;          // jobs in this launch chunk (rows of W)
    int npos;        // score-map positions (rows of X)
    int sld;         // row stride of scores (multiple of 4 ints)
    int nk;          // K stages of 128 bytes
    int ntiles;      // summary tiles of kTcTile positions
    int32_t* scores;   // [nj][sld] exact screen scores
    int32_t* summary;  // [nj][ntiles][kTcQ] descending top-Q per tile (INT_MIN padded)
};

size_t ccf_tc_smem_bytes();
int tc_kpad(int nscr, int Tc);
int tc_tiles(int npos);
// im2col of the TI screen planes for template size Tc (cached on the TI).
const int8_t* ti_im2col(ccw_ti* ti, int Tc, cudaStream_t st);
void launch_ccf_tc(const int8_t* d_w8, int maxj, const int8_t* d_x, int npos, int sld, int kpad, int nj,
                   int K, int32_t* scores, int32_t* summary, cudaStream_t st);

}  // namespace ccwgpu
