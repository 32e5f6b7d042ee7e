// pf_f64.cu — binary64 log-weights (NS-3d, R-21; the paper computes in double,
// P:199).  The difference to the filter's maximum is taken in binary64 and rounded once to
// binary32; everything after it is the float32 path on those differences (their maximum is
// exactly 0).  Two full-GPU passes over the doubles:
//   k_max64    per (filter, chunk) CTA: max + NaN/+inf flag of its chunk -> one atomicMax on
//              an order-preserving u64 key and one atomicOr per CTA and filter
//   k_shift64  t_i = fl32(logw_i - lmax) (NaN everywhere for an invalid filter, so that the
//              float path flags it and writes the NS-1 outputs)
// and, after the float path, k_lse64 adds the binary64 maximum to lse (the float path's lse
// is 0 + ln S).  HBM: 8 + 8 B read + 4 B written per particle.
#include "pf_device.cuh"
#include "pf_internal.h"

namespace pf {
namespace {

constexpr int kT64 = 256;        // threads per CTA
constexpr int kChunk64 = 4096;   // particles per CTA chunk (16 per thread)

// order-preserving map of non-NaN doubles to u64 (-inf -> 0x000F..F > 0, so a zeroed key is
// "nothing seen yet" and every value beats it)
__device__ __forceinline__ unsigned long long okey(double v) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double okey_inv(unsigned long long k) {
    const unsigned long long b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    return __longlong_as_double(static_cast<long long>(b));
}

template <bool VEC>
__global__ void __launch_bounds__(kT64) k_max64(const double* __restrict__ logw, int64_t ld, int32_t P, int cpf,
                                                unsigned long long* __restrict__ key, int32_t* __restrict__ bad) {
    const int64_t b = blockIdx.x;
    const int64_t n = b / cpf;
    const int64_t c = b % cpf;
    const int64_t i0 = c * kChunk64, i1 = min(static_cast<int64_t>(P), i0 + kChunk64);
    const double* row = logw + n * ld;
    double m = -INFINITY;
    int flag = 0;
    if (VEC) {
        // i0 is a multiple of 4096 and ld even: double2 loads from an aligned row
        for (int64_t i = i0 + 2 * threadIdx.x; i < i1; i += 2 * kT64) {
            if (i + 1 < i1) {
                const double2 v = __ldcs(reinterpret_cast<const double2*>(row + i));
                flag |= (isnan(v.x) || v.x == INFINITY || isnan(v.y) || v.y == INFINITY) ? 1 : 0;
                m = fmax(m, fmax(v.x, v.y));  // fmax drops NaN; a NaN filter is invalid anyway
            } else {
                const double v = __ldcs(row + i);
                flag |= (isnan(v) || v == INFINITY) ? 1 : 0;
                m = fmax(m, v);
            }
        }
    } else {
        for (int64_t i = i0 + threadIdx.x; i < i1; i += kT64) {
            const double v = __ldcs(row + i);
            flag |= (isnan(v) || v == INFINITY) ? 1 : 0;
            m = fmax(m, v);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        m = fmax(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
        flag |= __shfl_xor_sync(0xFFFFFFFFu, flag, o);
    }
    __shared__ double s_m[kT64 / 32];
    __shared__ int s_b[kT64 / 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { s_m[warp] = m; s_b[warp] = flag; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kT64 / 32; ++w) { m = fmax(m, s_m[w]); flag |= s_b[w]; }
        atomicMax(key + n, okey(m));
        if (flag) atomicOr(bad + n, 1);
    }
}

template <bool VEC>
__global__ void __launch_bounds__(kT64) k_shift64(const double* __restrict__ logw, int64_t ld, int32_t P, int cpf,
                                                  const unsigned long long* __restrict__ key,
                                                  const int32_t* __restrict__ bad, float* __restrict__ t,
                                                  int64_t ldt) {
    const int64_t b = blockIdx.x;
    const int64_t n = b / cpf;
    const int64_t c = b % cpf;
    const int64_t i0 = c * kChunk64, i1 = min(static_cast<int64_t>(P), i0 + kChunk64);
    const double* row = logw + n * ld;
    float* trow = t + n * ldt;
    const double lm = okey_inv(key[n]);
    const bool invalid = bad[n] != 0 || lm == -INFINITY;
    // NS-3d: one binary64 subtraction, one round-to-nearest conversion (-inf below float range)
    if (VEC) {
        for (int64_t i = i0 + 2 * threadIdx.x; i < i1; i += 2 * kT64) {
            if (i + 1 < i1) {
                const double2 v = __ldcs(reinterpret_cast<const double2*>(row + i));
                float2 r;
                r.x = invalid ? NAN : __double2float_rn(__dsub_rn(v.x, lm));
                r.y = invalid ? NAN : __double2float_rn(__dsub_rn(v.y, lm));
                *reinterpret_cast<float2*>(trow + i) = r;
            } else {
                trow[i] = invalid ? NAN : __double2float_rn(__dsub_rn(__ldcs(row + i), lm));
            }
        }
    } else {
        for (int64_t i = i0 + threadIdx.x; i < i1; i += kT64)
            trow[i] = invalid ? NAN : __double2float_rn(__dsub_rn(__ldcs(row + i), lm));
    }
}

__global__ void k_lse64(const unsigned long long* __restrict__ key, int32_t N, double* __restrict__ lse) {
    const int64_t n = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (n < N) lse[n] = __dadd_rn(okey_inv(key[n]), lse[n]);  // NaN (invalid filter) stays NaN
}

}  // namespace

size_t f64_ws_bytes(int32_t N, int32_t P) {
    const size_t ldt = (static_cast<size_t>(P) + 3) / 4 * 4;
    const size_t tb = (static_cast<size_t>(N) * ldt * 4 + 255) / 256 * 256;
    return tb + (static_cast<size_t>(N) * 12 + 255) / 256 * 256;
}

cudaError_t launch_shift64(const double* logw, int64_t ld, int32_t N, int32_t P, void* ws, float** t_out,
                           int64_t* ldt_out, unsigned long long** key_out, cudaStream_t s, uint64_t* launches) {
    const int64_t ldt = (static_cast<int64_t>(P) + 3) / 4 * 4;
    const size_t tb = (static_cast<size_t>(N) * static_cast<size_t>(ldt) * 4 + 255) / 256 * 256;
    float* t = static_cast<float*>(ws);
    auto* key = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + tb);
    auto* bad = reinterpret_cast<int32_t*>(key + N);
    cudaError_t e = cudaMemsetAsync(key, 0, static_cast<size_t>(N) * 12, s);
    if (e != cudaSuccess) return e;
    const int cpf = static_cast<int>((static_cast<int64_t>(P) + kChunk64 - 1) / kChunk64);
    const unsigned grid = static_cast<unsigned>(static_cast<int64_t>(N) * cpf);
    const bool vec = (reinterpret_cast<uintptr_t>(logw) & 15) == 0 && (ld % 2 == 0);
    {
        ProfScope ps_("k_max64", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 8u);
        if (vec) k_max64<true><<<grid, kT64, 0, s>>>(logw, ld, P, cpf, key, bad);
        else k_max64<false><<<grid, kT64, 0, s>>>(logw, ld, P, cpf, key, bad);
    }
    {
        ProfScope ps_("k_shift64", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 12u);
        if (vec) k_shift64<true><<<grid, kT64, 0, s>>>(logw, ld, P, cpf, key, bad, t, ldt);
        else k_shift64<false><<<grid, kT64, 0, s>>>(logw, ld, P, cpf, key, bad, t, ldt);
    }
    *launches += 2;
    *t_out = t;
    *ldt_out = ldt;
    *key_out = key;
    return cudaPeekAtLastError();
}

cudaError_t launch_lse64(const unsigned long long* key, int32_t N, double* lse, cudaStream_t s,
                         uint64_t* launches) {
    ProfScope ps_("k_lse64", s);
    k_lse64<<<static_cast<unsigned>((N + 255) / 256), 256, 0, s>>>(key, N, lse);
    ++*launches;
    return cudaPeekAtLastError();
}

}  // namespace pf
