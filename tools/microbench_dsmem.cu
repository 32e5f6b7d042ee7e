// Random 4-byte loads from distributed shared memory (cluster of 2, each CTA holding
// 32Ki floats = 128 KiB): half local, half remote, 8 independent loads per step.
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ uint32_t hash32(uint32_t x) { x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x; }
__global__ void __cluster_dims__(2, 1, 1) k(int steps, float* out, int remote_frac_pct) {
    extern __shared__ float sw[];
    cg::cluster_group cl = cg::this_cluster();
    for (int i = threadIdx.x; i < 32768; i += blockDim.x) sw[i] = (float)i;
    cl.sync();
    const int me = cl.block_rank();
    const float* other = cl.map_shared_rank(sw, me ^ 1);
    uint32_t s = hash32(blockIdx.x * blockDim.x + threadIdx.x);
    float acc = 0.f;
    for (int b = 0; b < steps; b += 8) {
        float x[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            s = s * 1664525u + 1013904223u;
            const uint32_t j = s >> 17;
            const bool rem = ((s >> 8) % 100) < (uint32_t)remote_frac_pct;
            x[t] = rem ? other[j] : sw[j];
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) acc += x[t];
    }
    if (acc == 1.234f) out[0] = acc;
    cl.sync();
}
int main() {
    float* out; cudaMalloc(&out, 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int pct : {0, 50, 100}) {
        const int blocks = (sms / 2) * 2, threads = 1024, steps = 1024;
        k<<<blocks, threads, 131072>>>(steps, out, pct);
        cudaEventRecord(e0);
        k<<<blocks, threads, 131072>>>(steps, out, pct);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"bench\":\"rand4_dsmem_cluster2\",\"remote_pct\":%d,\"loads_per_s\":%.3e,\"err\":\"%s\"}\n", pct,
               (double)blocks * threads * steps / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
