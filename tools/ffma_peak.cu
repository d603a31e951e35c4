// FP32 FFMA peak microbenchmark for the "alu" roofline of the direct path
// (MEASURED_PEAKS.json has no FP32 entry; the builder measures it).
//
// Each thread runs 8 independent FFMA chains (enough ILP to hide the 4-cycle
// FMA latency at full occupancy) for `iters` rounds; grid = 148 SMs x 8 CTAs x 256
// threads (16 warps/SM... x 4 = 64 warps/SM).  Timed with CUDA events after a
// warm-up launch; the best of 10 launches is reported together with the SM clock
// the launches ran at (clock64 delta / event time).  Output: one JSON line.
//
// Build:  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o ffma_peak tools/ffma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void __launch_bounds__(256) k_ffma(float *out, int iters, float a, float b,
                                              long long *cycles)
{
    float v0 = threadIdx.x * 1e-7f, v1 = v0 + 1e-6f, v2 = v0 + 2e-6f, v3 = v0 + 3e-6f;
    float v4 = v0 + 4e-6f, v5 = v0 + 5e-6f, v6 = v0 + 6e-6f, v7 = v0 + 7e-6f;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            v0 = fmaf(v0, a, b); v1 = fmaf(v1, a, b); v2 = fmaf(v2, a, b); v3 = fmaf(v3, a, b);
            v4 = fmaf(v4, a, b); v5 = fmaf(v5, a, b); v6 = fmaf(v6, a, b); v7 = fmaf(v7, a, b);
        }
    }
    long long t1 = clock64();
    float s = ((v0 + v1) + (v2 + v3)) + ((v4 + v5) + (v6 + v7));
    if (s == 12345.f) out[threadIdx.x] = s;      // keeps the chains live
    if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
}

int main()
{
    int dev = 0, sms = 0, clk_khz = 0;
    CK(cudaSetDevice(dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
    float *out;
    long long *cyc;
    CK(cudaMalloc(&out, 1024 * sizeof(float)));
    CK(cudaMalloc(&cyc, sizeof(long long)));
    const int threads = 256, per_sm = 8, iters = 4096;
    const int blocks = sms * per_sm;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    k_ffma<<<blocks, threads>>>(out, iters, 0.999999f, 1e-7f, cyc);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
        CK(cudaEventRecord(e0));
        k_ffma<<<blocks, threads>>>(out, iters, 0.999999f, 1e-7f, cyc);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        long long c;
        CK(cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost));
        (void)c;
        if (ms < best) best = ms;
    }
    const double fma = (double)blocks * threads * iters * 16 * 8;
    const double tfma = fma / (best * 1e-3) / 1e12;
    const double nominal = (double)sms * 128 * clk_khz * 1e3 / 1e12;
    printf("{\"ffma_tfma_s\": %.3f, \"fp32_tflops\": %.3f, \"ms\": %.4f, \"sms\": %d, "
           "\"threads\": %d, \"blocks\": %d, \"fma_per_launch\": %.6e, "
           "\"nominal_tfma_s_at_max_clock\": %.3f, \"max_clock_mhz\": %.1f, "
           "\"frac_of_nominal\": %.4f}\n",
           tfma, 2 * tfma, best, sms, threads, blocks, fma, nominal, clk_khz / 1e3,
           tfma / nominal);
    return 0;
}
