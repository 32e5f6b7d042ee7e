// tools/microbench.cu — access-pattern ceilings on this B200 (roofline context
// for DESIGN.md §5.1).  Standalone: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o tools/microbench tools/microbench.cu ; ./tools/microbench
//
//  copy     : streaming float4 copy (cross-check of MEASURED_PEAKS.json hbm_gbs)
//  gather64 : in-place-gather pattern of k_gather_rows16: 64-byte rows, a
//             fraction f of rows rewritten from a random row of the same 4 MiB
//             block (algorithmic bytes = 2 x 64 x moved rows + 4 B/row of index)
//  rand4_l2 : warp-wide random 4-byte loads from 256 KiB windows (L2-resident):
//             the Metropolis proposal pattern, loads per second
//  rand4_smem: the same from shared memory (upper bound for smem-resident w)
//  l2_stream: float4 reads (ld.global.cg) of an L2-resident buffer, repeated (L2 read bandwidth:
//             the roofline denominator of the L2-resident C2 working set)
//  l2_sector: random 32-byte sector reads of an L2-resident buffer (the random-sector rate that
//             bounds the multinomial bucket searches and the Metropolis proposals)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}

// perm[i] = source row (== i when not moved)
__global__ void k_make_perm(int32_t* perm, int64_t rows, int block_rows, float frac) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t h = hash32((uint32_t)i * 2654435761u + 12345u);
        const bool moved = (h & 0xFFFFFF) < (uint32_t)(frac * 16777216.0f);
        const int64_t b0 = (i / block_rows) * block_rows;
        perm[i] = moved ? (int32_t)(b0 + hash32(h) % block_rows) : (int32_t)i;
    }
}

// thread per 16-byte chunk (4 per 64-byte row), 4 chunks in flight
__global__ void k_gather64(const int4* __restrict__ X, int4* __restrict__ Y, const int32_t* __restrict__ perm, int64_t rows) {
    const int64_t total = rows * 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t g0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g0 < total; g0 += 4 * stride) {
        int4 v[4];
        int64_t dst[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t g = g0 + u * stride;
            dst[u] = -1;
            if (g < total) {
                const int64_t r = g >> 2;
                const int32_t p = __ldg(perm + r);
                if (p != r) { v[u] = __ldg(X + (int64_t)p * 4 + (g & 3)); dst[u] = r * 4 + (g & 3); }
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) if (dst[u] >= 0) Y[dst[u]] = v[u];
    }
}

__global__ void k_rand4(const float* __restrict__ w, int64_t nwin, int steps, float* out) {
    // each warp works in one 64Ki-float window; 8 independent loads per step
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const float* win = w + (gw % nwin) * 65536;
    uint32_t s = hash32((uint32_t)(blockIdx.x * blockDim.x + threadIdx.x));
    float acc = 0.f;
    for (int b = 0; b < steps; b += 8) {
        float x[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) { s = s * 1664525u + 1013904223u; x[t] = __ldg(win + (s >> 16)); }
#pragma unroll
        for (int t = 0; t < 8; ++t) acc += x[t];
    }
    if (acc == 12345.f) out[0] = acc;
}

__global__ void k_l2_stream(const float4* __restrict__ a, int64_t n4, int reps, float* out) {
    float acc = 0.f;
    for (int r = 0; r < reps; ++r)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
            const float4 v = __ldcg(a + i);
            acc += v.x + v.y + v.z + v.w;
        }
    if (acc == 12345.f) out[0] = acc;
}

// each thread reads 8 independent random 32-byte sectors (two float4 each) per step
__global__ void k_l2_sector(const float4* __restrict__ a, int64_t nsec, int steps, float* out) {
    uint32_t s = hash32((uint32_t)(blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 7u);
    float acc = 0.f;
    for (int b = 0; b < steps; ++b) {
        float4 x[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            s = s * 1664525u + 1013904223u;
            x[t] = __ldcg(a + 2 * (int64_t)(hash32(s) % (uint32_t)nsec));
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) acc += x[t].x;
    }
    if (acc == 12345.f) out[0] = acc;
}

__global__ void k_rand4_smem(const float* __restrict__ w, int steps, float* out) {
    extern __shared__ float sw[];
    for (int i = threadIdx.x; i < 32768; i += blockDim.x) sw[i] = w[i];
    __syncthreads();
    uint32_t s = hash32((uint32_t)(blockIdx.x * blockDim.x + threadIdx.x));
    float acc = 0.f;
    for (int b = 0; b < steps; b += 8) {
        float x[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) { s = s * 1664525u + 1013904223u; x[t] = sw[s >> 17]; }
#pragma unroll
        for (int t = 0; t < 8; ++t) acc += x[t];
    }
    if (acc == 12345.f) out[0] = acc;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0;
    // ---- copy: 2 GiB -> 2 GiB
    const size_t n4 = (size_t)1 << 27;  // float4s = 2 GiB
    float4 *a, *b;
    CK(cudaMalloc(&a, n4 * 16));
    CK(cudaMalloc(&b, n4 * 16));
    CK(cudaMemset(a, 0, n4 * 16));
    for (int it = 0; it < 3; ++it) k_copy<<<sms * 8, 256>>>(a, b, n4);
    cudaEventRecord(e0);
    for (int it = 0; it < 10; ++it) k_copy<<<sms * 8, 256>>>(a, b, n4);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"bench\":\"copy\",\"GBs\":%.1f}\n", 2.0 * n4 * 16 * 10 / (ms * 1e-3) / 1e9);
    // ---- gather64: 2^26 rows x 64 B = 4 GiB state, blocks of 2^16 rows (4 MiB)
    const int64_t rows = (int64_t)1 << 26;
    int32_t* perm;
    CK(cudaMalloc(&perm, rows * 4));
    int4* X = reinterpret_cast<int4*>(a);  // reuse: 2 GiB each -> use 2^25 rows
    const int64_t r2 = rows / 2;
    for (float frac : {0.10f, 0.383f, 0.60f}) {
        k_make_perm<<<sms * 8, 256>>>(perm, r2, 65536, frac);
        for (int it = 0; it < 3; ++it) k_gather64<<<sms * 16, 256>>>(X, X, perm, r2);
        cudaEventRecord(e0);
        for (int it = 0; it < 10; ++it) k_gather64<<<sms * 16, 256>>>(X, X, perm, r2);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = (4.0 + 2.0 * 64.0 * frac) * r2;
        printf("{\"bench\":\"gather64_inplace\",\"moved_fraction\":%.3f,\"alg_GBs\":%.1f}\n", frac, bytes * 10 / (ms * 1e-3) / 1e9);
    }
    // ---- random 4-byte loads, L2-resident windows (1024 x 256 KiB = 256 MiB total, warps spread)
    float* w = reinterpret_cast<float*>(b);
    float* out;
    CK(cudaMalloc(&out, 4));
    const int steps = 256;
    for (int64_t nwin : {(int64_t)64, (int64_t)1024}) {
        const int blocks = sms * 8, threads = 256;
        k_rand4<<<blocks, threads>>>(w, nwin, steps, out);
        cudaEventRecord(e0);
        k_rand4<<<blocks, threads>>>(w, nwin, steps, out);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"bench\":\"rand4_global\",\"windows_256KiB\":%lld,\"loads_per_s\":%.3e}\n", (long long)nwin,
               (double)blocks * threads * steps / (ms * 1e-3));
    }
    CK(cudaFuncSetAttribute(k_rand4_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
    {
        const int blocks = sms, threads = 1024;
        k_rand4_smem<<<blocks, threads, 131072>>>(w, steps, out);
        cudaEventRecord(e0);
        k_rand4_smem<<<blocks, threads, 131072>>>(w, steps * 4, out);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"bench\":\"rand4_smem\",\"loads_per_s\":%.3e}\n", (double)blocks * threads * steps * 4 / (ms * 1e-3));
    }
    // ---- L2: 32 MiB resident buffer
    {
        const int64_t n4 = (int64_t(32) << 20) / 16;
        const int reps = 20;
        k_l2_stream<<<sms * 8, 256>>>(reinterpret_cast<const float4*>(b), n4, 2, out);
        cudaEventRecord(e0);
        k_l2_stream<<<sms * 8, 256>>>(reinterpret_cast<const float4*>(b), n4, reps, out);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"bench\":\"l2_stream\",\"MiB\":32,\"GBs\":%.1f}\n", (double)n4 * 16 * reps / (ms * 1e-3) / 1e9);
        const int64_t nsec = (int64_t(32) << 20) / 32;
        const int steps = 64;
        k_l2_sector<<<sms * 8, 256>>>(reinterpret_cast<const float4*>(b), nsec, 4, out);
        cudaEventRecord(e0);
        k_l2_sector<<<sms * 8, 256>>>(reinterpret_cast<const float4*>(b), nsec, steps, out);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        const double sectors = (double)sms * 8 * 256 * steps * 8;
        printf("{\"bench\":\"l2_random_sector\",\"MiB\":32,\"sectors_per_s\":%.3e,\"GBs_32B\":%.1f}\n",
               sectors / (ms * 1e-3), sectors * 32 / (ms * 1e-3) / 1e9);
    }
    return 0;
}
