// FP32 SIMT FMA peak on this GPU (the roofline denominator of the register
// recursion kernels, which MEASURED_PEAKS.json does not carry).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/probe_fp32_peak.cu -o /tmp/fp32peak
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void __launch_bounds__(256) fma_kernel(float* out, int iters, float a, float b) {
    float x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3f + c;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) x[c] = fmaf(x[c], a, b);
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += x[c];
    if (s == 12345.678f) out[0] = s;  // keep the chains alive
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, 4);
    constexpr int CH = 16;
    const int iters = 1 << 16;
    const int blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    fma_kernel<CH><<<blocks, threads>>>(out, 1024, 0.999f, 1e-3f);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        fma_kernel<CH><<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * CH * (double)iters * blocks * threads;
    printf("{\"fp32_fma_tflops\": %.2f, \"sms\": %d, \"ms\": %.3f}\n", flops / best / 1e9, sms, best);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
