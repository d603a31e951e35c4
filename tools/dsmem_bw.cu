// Distributed-shared-memory bandwidth on B200 (the quantity that decides whether a
// cluster-transposed, on-chip 2-D FFT could beat the two-pass design).
//
// Clusters of C CTAs (one CTA per SM, 96 KB smem each, 512 threads); every CTA streams
// 16-byte st.shared::cluster stores into the shared memory of CTA (rank + 1) % C for R
// rounds of 64 KB (the producer-pays pattern of a transpose), a cluster barrier at the end.  Reported: bytes moved per SM per cycle
// and summed over the GPU (best of 5 launches, CUDA events), and the same traffic into the
// CTA's own shared memory for comparison.
//
// Build:  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/dsmem_bw tools/dsmem_bw.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int NTH = 512, BUF = 64 * 1024;

template <int MODE>   // 0: remote stores, 1: remote loads, 2: local stores
__global__ void __launch_bounds__(NTH) k_dsmem(int rounds, float *sink) {
    extern __shared__ __align__(16) float4 buf[];
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank(), cs = cl.num_blocks();
    for (int i = threadIdx.x; i < BUF / 16; i += NTH) buf[i] = make_float4(i, rank, 0, 0);
    cl.sync();
    // shared::cluster address of buf in the peer CTA (or this CTA)
    const uint32_t local = (uint32_t)__cvta_generic_to_shared(buf);
    uint32_t base = local;
    if (MODE != 2)
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(base) : "r"(local), "r"((rank + 1) % cs));
    float acc = 0.f;
    for (int r = 0; r < rounds; ++r) {
        const float fr = (float)r;
#pragma unroll 8
        for (int i = threadIdx.x; i < BUF / 16; i += NTH) {
            const uint32_t a = base + 16u * (uint32_t)i;
            if (MODE == 1) {
                float x, y, z, w;
                asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(a) : "memory");
                acc += x + w;
            } else {
                asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};"
                             :: "r"(a), "f"(fr), "f"((float)i), "f"((float)rank), "f"(acc) : "memory");
            }
        }
    }
    cl.sync();
    if (acc == 12345.f) sink[threadIdx.x] = acc;
}

template <int MODE>
static int run(int C, int sms, int clk_khz, float *sink) {
    cudaLaunchConfig_t cfg = {};
    const int nclusters = sms / C;
    cfg.gridDim = dim3(nclusters * C);
    cfg.blockDim = dim3(NTH);
    cfg.dynamicSmemBytes = 96 * 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaFuncSetAttribute(k_dsmem<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    if (C > 8) CK(cudaFuncSetAttribute(k_dsmem<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    const int rounds = 200;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaLaunchKernelEx(&cfg, k_dsmem<MODE>, rounds, sink));
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int i = 0; i < 5; ++i) {
        CK(cudaEventRecord(e0));
        CK(cudaLaunchKernelEx(&cfg, k_dsmem<MODE>, rounds, sink));
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
    }
    const double bytes_cta = (double)rounds * BUF, ctas = nclusters * C;
    const double per_sm = bytes_cta / (best * 1e-3);                     // B/s per CTA (= per SM)
    const char *names[3] = {"remote_store", "remote_load", "local_store"};
    printf("{\"mode\": \"%s\", \"cluster\": %d, \"ctas\": %d, \"ms\": %.4f, \"GBps_per_sm\": %.1f, "
           "\"B_per_clk_per_sm\": %.2f, \"TBps_total\": %.3f}\n",
           names[MODE], C, (int)ctas, best, per_sm / 1e9, per_sm / (clk_khz * 1e3), per_sm * ctas / 1e12);
    return 0;
}

int main() {
    int sms = 0, clk = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    float *sink;
    CK(cudaMalloc(&sink, NTH * sizeof(float)));
    // (remote loads are not reported: ptxas turns the unused components of the v4 load into
    // narrower generic loads, so that mode does not measure the transpose pattern)
    for (int C : {2, 4, 8, 16})
        if (run<0>(C, sms, clk, sink)) return 1;
    return run<2>(2, sms, clk, sink);
}
