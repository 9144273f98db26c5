// probe.cu -- pipe-throughput microbenchmarks for the roofline denominators.
// FP32: 8 independent FFMA chains per thread, and 8 independent packed FFMA2 (f32x2)
// chains (sm_100: same FLOP rate, half the issue slots; the faster is the peak);
// MUFU: 8 independent ex2 chains.
#include "common.cuh"

namespace bf {
namespace {

__global__ void __launch_bounds__(256) ffma_probe(float *out, int iters, float a, float b) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678f) out[0] = s;
}

__global__ void __launch_bounds__(256) ffma2_probe(float *out, int iters, float a0, float b0) {
    unsigned long long x[8], a, b;
    asm("mov.b64 %0, {%1, %1};" : "=l"(a) : "f"(a0));
    asm("mov.b64 %0, {%1, %1};" : "=l"(b) : "f"(b0));
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float u = threadIdx.x * 1e-3f + i, v = u + 0.5f;
        asm("mov.b64 %0, {%1, %2};" : "=l"(x[i]) : "f"(u), "f"(v));
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i)
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(a), "l"(b));
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float u, v;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(u), "=f"(v) : "l"(x[i]));
        s += u + v;
    }
    if (s == 12345.678f) out[0] = s;
}

__global__ void __launch_bounds__(256) mufu_probe(float *out, int iters) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-6f + i * 1e-3f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678f) out[0] = s;
}

}  // namespace
}  // namespace bf

extern "C" int bf_probe_peaks(int device, double *fp32_tflops, double *mufu_tops) {
    using namespace bf;
    BF_TRY_CUDA(cudaSetDevice(device));
    cudaDeviceProp p;
    BF_TRY_CUDA(cudaGetDeviceProperties(&p, device));
    float *out;
    BF_TRY_CUDA(cudaMalloc(&out, 16));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = p.multiProcessorCount * 8, threads = 256;
    const int fi = 4096, mi = 512;
    float best_f = 1e30f, best_m = 1e30f, best_f2 = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        float ms;
        cudaEventRecord(e0);
        ffma_probe<<<blocks, threads>>>(out, fi, 0.999f, 1e-3f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) best_f = ms < best_f ? ms : best_f;
        cudaEventRecord(e0);
        mufu_probe<<<blocks, threads>>>(out, mi);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) best_m = ms < best_m ? ms : best_m;
        cudaEventRecord(e0);
        ffma2_probe<<<blocks, threads>>>(out, fi, 0.999f, 1e-3f);  // 2 x 8 x 8 FMA per iteration
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) best_f2 = ms < best_f2 ? ms : best_f2;
    }
    note_launch(12);
    cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    BF_TRY_CUDA(err);
    const double n = (double)blocks * threads * 16 * 8;
    const double ffma = 2.0 * n * fi / (best_f * 1e-3) / 1e12;
    const double ffma2 = 2.0 * (double)blocks * threads * 128 * fi / (best_f2 * 1e-3) / 1e12;
    *fp32_tflops = ffma > ffma2 ? ffma : ffma2;
    *mufu_tops = n * mi / (best_m * 1e-3) / 1e12;
    return BF_OK;
}
