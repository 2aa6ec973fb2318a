// peak.cu -- in-run FP32 FFMA peak microbenchmark (the CCF screen's roofline
// denominator: MEASURED_PEAKS.json records only HBM and bf16 tensor peaks).
#include <algorithm>

#include "internal.hpp"

namespace ccwgpu {

// 8 independent FMA chains per thread; one operand is an immediate, the form
// the B300/B200 FMA pipe issues at full rate.
__global__ void __launch_bounds__(256) ffma_peak_kernel(float* out, int iters, float seed) {
    float a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
    float a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            a0 = fmaf(a0, 0.9999f, 0.0001f);
            a1 = fmaf(a1, 0.9999f, 0.0001f);
            a2 = fmaf(a2, 0.9999f, 0.0001f);
            a3 = fmaf(a3, 0.9999f, 0.0001f);
            a4 = fmaf(a4, 0.9999f, 0.0001f);
            a5 = fmaf(a5, 0.9999f, 0.0001f);
            a6 = fmaf(a6, 0.9999f, 0.0001f);
            a7 = fmaf(a7, 0.9999f, 0.0001f);
        }
    }
    const float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 12345.678f) out[blockIdx.x] = s;  // keep the chains alive
}

double measure_ffma_peak(ccw_ctx* ctx) {
    int sms = 0;
    CCW_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    float* d = nullptr;
    const int blocks = sms * 8;
    CCW_CUDA(cudaMalloc(&d, sizeof(float) * blocks));
    cudaEvent_t a, b;
    CCW_CUDA(cudaEventCreate(&a));
    CCW_CUDA(cudaEventCreate(&b));
    const int iters = 4096;
    double best = 0;
    for (int rep = 0; rep < 5; ++rep) {
        CCW_CUDA(cudaEventRecord(a, ctx->stream));
        ffma_peak_kernel<<<blocks, 256, 0, ctx->stream>>>(d, iters, 1.0f);
        CCW_CUDA(cudaEventRecord(b, ctx->stream));
        CCW_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        CCW_CUDA(cudaEventElapsedTime(&ms, a, b));
        const double flop = 2.0 * 8 * 16 * static_cast<double>(iters) * blocks * 256;
        if (rep > 0) best = std::max(best, flop / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(d);
    return best;
}

// Integer peaks of the 3D screen's inner loops: IMAD (one int32 MAC per lane)
// and dp4a (four int8 MACs per lane), 8 independent chains per thread.
template <int DP4A>
__global__ void __launch_bounds__(256) int_peak_kernel(int* out, int iters, int seed) {
    int a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = seed + threadIdx.x + k;
    const int w = 0x01020304 ^ seed;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                if (DP4A)
                    a[c] = __dp4a(a[c], w, a[c]);
                else
                    a[c] = a[c] * w + c;
            }
    }
    int s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345678) out[blockIdx.x] = s;
}

// ops per second (2 per MAC) in TOPS; kind 0 IMAD, 1 dp4a
double measure_int_peak(ccw_ctx* ctx, int kind) {
    int sms = 0;
    CCW_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    int* d = nullptr;
    const int blocks = sms * 8;
    CCW_CUDA(cudaMalloc(&d, sizeof(int) * blocks));
    cudaEvent_t a, b;
    CCW_CUDA(cudaEventCreate(&a));
    CCW_CUDA(cudaEventCreate(&b));
    const int iters = 2048;
    double best = 0;
    for (int rep = 0; rep < 5; ++rep) {
        CCW_CUDA(cudaEventRecord(a, ctx->stream));
        if (kind == 1)
            int_peak_kernel<1><<<blocks, 256, 0, ctx->stream>>>(d, iters, 3);
        else
            int_peak_kernel<0><<<blocks, 256, 0, ctx->stream>>>(d, iters, 3);
        CCW_CUDA(cudaEventRecord(b, ctx->stream));
        CCW_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        CCW_CUDA(cudaEventElapsedTime(&ms, a, b));
        const double ops = 2.0 * (kind == 1 ? 4 : 1) * 8 * 16 * static_cast<double>(iters) * blocks * 256;
        if (rep > 0) best = std::max(best, ops / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(d);
    return best;
}

}  // namespace ccwgpu
