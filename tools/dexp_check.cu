// Exhaustive check that the device dexp() / weight2() of pf_device.cuh are bit-identical to the
// literal NS-4 transcription below (steps 1-7 as written) for every float32 t <= 0
// (all 2^31 patterns with the sign bit set, NaNs included) and t = +0.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1202_6163_b200/csrc \
//        tools/dexp_check.cu -o tools/dexp_check && tools/dexp_check
#include <cstdio>
#include <cstdint>
#include "pf_device.cuh"

__device__ __forceinline__ float ns4_literal(float t) {
    const float kTiny = __uint_as_float(0x00800000u);
    const bool kill = !(t >= -88.0f);                                      // step 1
    float tt = kill ? 0.0f : t;
    tt = (fabsf(tt) < kTiny) ? 0.0f : tt;                                  // step 2
    const float n = rintf(__fmul_rn(tt, __uint_as_float(0x3FB8AA3Bu)));   // step 3
    float r = __fmaf_rn(-n, __uint_as_float(0x3F317200u), tt);            // step 4
    r = __fmaf_rn(-n, __uint_as_float(0x35BFBE8Eu), r);
    float p = __uint_as_float(0x39500D01u);                                // step 5
    p = __fmaf_rn(p, r, __uint_as_float(0x3AB60B61u));
    p = __fmaf_rn(p, r, __uint_as_float(0x3C088889u));
    p = __fmaf_rn(p, r, __uint_as_float(0x3D2AAAABu));
    p = __fmaf_rn(p, r, __uint_as_float(0x3E2AAAABu));
    p = __fmaf_rn(p, r, 0.5f);
    p = __fmaf_rn(p, r, 1.0f);
    p = __fmaf_rn(p, r, 1.0f);
    const int ni = static_cast<int>(n);                                    // step 6
    const uint32_t sbits = (ni >= -126) ? (static_cast<uint32_t>(ni + 127) << 23) : 0u;
    float w = __fmul_rn(p, __uint_as_float(sbits));
    w = (kill || w < kTiny) ? 0.0f : w;                                    // step 7
    return fminf(w, 1.0f);
}

__global__ void check(unsigned long long* bad, uint32_t* first_bad) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    unsigned long long nb = 0;
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k <= (1ull << 31); k += stride) {
        const uint32_t b = (k == (1ull << 31)) ? 0u : (0x80000000u | static_cast<uint32_t>(k));
        const float t = __uint_as_float(b);
        const uint32_t ref = __float_as_uint(ns4_literal(t));
        const uint32_t got = __float_as_uint(pf::dexp(t));
        // weight2 with lmax = 0 (fl(t - 0) = t), the partner lane a rotated pattern
        const float t2 = __uint_as_float(0x80000000u | ((b * 2654435761u) >> 1));
        float w0, w1;
        pf::weight2(t, t2, 0.0f, w0, w1);
        const bool ok = got == ref && __float_as_uint(w0) == ref && __float_as_uint(w1) == __float_as_uint(ns4_literal(t2));
        if (!ok) {
            ++nb;
            atomicMin(first_bad, b);
            if (nb <= 2)
                printf("t %08x ref %08x dexp %08x w0 %08x | t2 %08x ref2 %08x w1 %08x\n", b, ref, got,
                       __float_as_uint(w0), __float_as_uint(t2), __float_as_uint(ns4_literal(t2)), __float_as_uint(w1));
        }
    }
    if (nb) atomicAdd(bad, nb);
}

int main() {
    unsigned long long* bad;
    uint32_t* fb;
    cudaMallocManaged(&bad, 8);
    cudaMallocManaged(&fb, 4);
    *bad = 0;
    *fb = 0xFFFFFFFFu;
    check<<<148 * 16, 256>>>(bad, fb);
    const cudaError_t e = cudaDeviceSynchronize();
    printf("{\"inputs\": %llu, \"mismatches\": %llu, \"first_bad\": \"0x%08x\", \"cuda\": \"%s\"}\n",
           (1ull << 31) + 1, *bad, *fb, cudaGetErrorString(e));
    return (e == cudaSuccess && *bad == 0) ? 0 : 1;
}
