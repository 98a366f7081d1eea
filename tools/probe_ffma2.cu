// FP32 FMA throughput by instruction form on this GPU: FFMA with constant-bank
// operands, FFMA with three register operands, and the packed FFMA2 (float2)
// of sm_100 (__ffma2_rn).  nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/probe_ffma2.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 16;

__global__ void __launch_bounds__(256) ffma_const(float* out, int iters, float a, float b) {
    float x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3f + c;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = fmaf(x[c], a, b);
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 12345.678f) out[0] = s;
}

__global__ void __launch_bounds__(256) ffma_reg(float* out, int iters, float a, float b) {
    float x[CH], y[CH], z[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        x[c] = threadIdx.x * 1e-3f + c;
        y[c] = a + c * 1e-7f * threadIdx.x;
        z[c] = b - c * 1e-7f * threadIdx.x;
    }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = fmaf(x[c], y[c], z[c]);
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c] + y[c] + z[c];
    if (s == 12345.678f) out[0] = s;
}

__global__ void __launch_bounds__(256) ffma2_reg(float* out, int iters, float a, float b) {
    float2 x[CH / 2], y[CH / 2], z[CH / 2];
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) {
        x[c] = make_float2(threadIdx.x * 1e-3f + c, threadIdx.x * 2e-3f + c);
        y[c] = make_float2(a + c * 1e-7f * threadIdx.x, a - c * 1e-7f * threadIdx.x);
        z[c] = make_float2(b - c * 1e-7f * threadIdx.x, b + c * 1e-7f * threadIdx.x);
    }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < CH / 2; ++c) x[c] = __ffma2_rn(x[c], y[c], z[c]);
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) s += x[c].x + x[c].y + y[c].x + z[c].y;
    if (s == 12345.678f) out[0] = s;
}

template <class K>
double run(K kern, float* out, int sms) {
    const int iters = 1 << 15, blocks = sms * 8, threads = 256;
    kern<<<blocks, threads>>>(out, 256, 0.999f, 1e-3f);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        kern<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double fmas = (double)blocks * threads * iters * CH;
    return 2.0 * fmas / (best * 1e-3) / 1e12;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, 4);
    std::printf("{\"ffma_const_tflops\": %.2f, \"ffma_reg_tflops\": %.2f, \"ffma2_reg_tflops\": %.2f}\n",
                run(ffma_const, out, sms), run(ffma_reg, out, sms), run(ffma2_reg, out, sms));
    return 0;
}
