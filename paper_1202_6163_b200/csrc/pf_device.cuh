// pf_device.cuh — device primitives of libpfresample (sm_100a).
//
// Implements the numeric spec of DESIGN.md §3 (NS-n) for the GPU.  Shares no
// code with oracle/ (which implements the same text on the host); bit-exact
// agreement is the parity test.  Every float operation that decides an
// integer is spelled out with an explicit IEEE intrinsic (__fmul_rn,
// __fmaf_rn, __fsub_rn) so that nvcc can neither contract nor reorder it.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pf {

// ---------------------------------------------------------------- NS-6
// Philox4x32-10 (Salmon et al., SC'11).  Counter (c0, c1, tag, filter),
// key (lo32(seed), hi32(seed)).
struct u32x4 {
    uint32_t x, y, z, w;
};

__device__ __forceinline__ u32x4 philox10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                           uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c0;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ k0;
        const uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return {c0, c1, c2, c3};
}

struct Key {
    uint32_t k0, k1;
};
__host__ __device__ __forceinline__ Key make_key(uint64_t seed) {
    return {static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)};
}

__device__ __forceinline__ uint64_t lo_word(const u32x4& v) {
    return (static_cast<uint64_t>(v.y) << 32) | v.x;
}
__device__ __forceinline__ uint64_t hi_word(const u32x4& v) {
    return (static_cast<uint64_t>(v.w) << 32) | v.z;
}

// ---------------------------------------------------------------- NS-4
// Deterministic float32 exp of t <= 0; constants are the NS-4 bit patterns.  Written without
// branches, and with three steps folded into cheaper equivalents, each bit-identical for every
// t <= 0 and NaN (all 2^31 + 1 such inputs checked exhaustively against the literal NS-4
// transcription by tools/dexp_check.cu):
//  - step 1 (t < -88 or NaN -> 0) becomes a clamp t >= -100: below -88 the scale 2^n is 0
//    (n <= -127), so w = p * 0 = 0 while r and p stay finite; step 7 then returns 0;
//  - step 2 (|t| < 2^-126 -> 0) is dropped: such a t gives n = 0, r = t and p = fl(1 + t) = 1,
//    the value t = 0 gives;
//  - step 3's rint of fl(t * log2e) by the add-and-subtract of 1.5 * 2^23 (round to nearest
//    even in [2^23, 2^24), the rint of the product for |t * log2e| < 2^22), which also yields
//    n as an integer from the sum's bit pattern (no float-to-int conversion);
//  - step 6's scale bits max(n + 127, 0) << 23 (n >= -145 after the clamp).
constexpr float kRintMagic = 12582912.0f;  // 1.5 * 2^23, bit pattern 0x4B400000
__device__ __forceinline__ float dexp(float t) {
    const float kTiny = __uint_as_float(0x00800000u);  // 2^-126
    const float tt = fmaxf(t, -100.0f);                 // step 1 (also -inf and NaN)
    const float m = __fadd_rn(__fmul_rn(tt, __uint_as_float(0x3FB8AA3Bu)), kRintMagic);  // step 3
    const float n = __fadd_rn(m, -kRintMagic);
    float r = __fmaf_rn(-n, __uint_as_float(0x3F317200u), tt);  // step 4
    r = __fmaf_rn(-n, __uint_as_float(0x35BFBE8Eu), r);
    float p = __uint_as_float(0x39500D01u);  // step 5
    p = __fmaf_rn(p, r, __uint_as_float(0x3AB60B61u));
    p = __fmaf_rn(p, r, __uint_as_float(0x3C088889u));
    p = __fmaf_rn(p, r, __uint_as_float(0x3D2AAAABu));
    p = __fmaf_rn(p, r, __uint_as_float(0x3E2AAAABu));
    p = __fmaf_rn(p, r, 0.5f);
    p = __fmaf_rn(p, r, 1.0f);
    p = __fmaf_rn(p, r, 1.0f);
    // step 6: n + 127 = bits(m) - (0x4B400000 - 127)
    const int e = max(static_cast<int>(__float_as_uint(m)) - (0x4B400000 - 127), 0);
    float w = __fmul_rn(p, __uint_as_float(static_cast<uint32_t>(e) << 23));
    w = (w < kTiny) ? 0.0f : w;  // step 7
    return fminf(w, 1.0f);
}

// NS-4 for two weights at once with the Blackwell packed FP32 instructions (FFMA2 / FMUL2 /
// FADD2: fma.rn / mul.rn / add.rn .f32x2, each lane an IEEE round-to-nearest operation), so the
// result is bit-identical to two dexp() calls while the arithmetic issues half the
// instructions.  Same steps as dexp(); the clamps and selects stay per lane.
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t f2_splat(uint32_t bits) {
    return (static_cast<uint64_t>(bits) << 32) | bits;
}

// w = dexp(fl(logw - lmax)) for two log-weights (NS-3 + NS-4), bit-identical to weight()
__device__ __forceinline__ void weight2(float l0, float l1, float lmax, float& w0, float& w1) {
    const float kTiny = __uint_as_float(0x00800000u);  // 2^-126
    float t0, t1;
    f2_unpack(f2_add(f2_pack(l0, l1), f2_pack(-lmax, -lmax)), t0, t1);  // fl(logw - lmax): exact negation
    const uint64_t tt = f2_pack(fmaxf(t0, -100.0f), fmaxf(t1, -100.0f));  // step 1
    // step 3: m = fl(fl(t log2e) + 1.5 2^23), n = m - 1.5 2^23 (exact).  Per lane: ptxas
    // contracts a mul.rn.f32x2 feeding an add.rn.f32x2 into one FFMA2 (a single rounding,
    // which changes the rint of half-way products; tools/dexp_check.cu caught it)
    float s0, s1;
    f2_unpack(tt, s0, s1);
    const float m0 = __fadd_rn(__fmul_rn(s0, __uint_as_float(0x3FB8AA3Bu)), kRintMagic);
    const float m1 = __fadd_rn(__fmul_rn(s1, __uint_as_float(0x3FB8AA3Bu)), kRintMagic);
    const uint64_t m = f2_pack(m0, m1);
    const uint64_t n = f2_add(m, f2_splat(0xCB400000u));
    // step 4: fma(-n, c, t) == fma(n, -c, t) exactly (negation is exact)
    uint64_t r = f2_fma(n, f2_splat(0x3F317200u ^ 0x80000000u), tt);
    r = f2_fma(n, f2_splat(0x35BFBE8Eu ^ 0x80000000u), r);
    uint64_t p = f2_splat(0x39500D01u);                                  // step 5
    p = f2_fma(p, r, f2_splat(0x3AB60B61u));
    p = f2_fma(p, r, f2_splat(0x3C088889u));
    p = f2_fma(p, r, f2_splat(0x3D2AAAABu));
    p = f2_fma(p, r, f2_splat(0x3E2AAAABu));
    p = f2_fma(p, r, f2_splat(0x3F000000u));                             // 0.5
    p = f2_fma(p, r, f2_splat(0x3F800000u));                             // 1
    p = f2_fma(p, r, f2_splat(0x3F800000u));                             // 1
    // step 6: the scale bits max(n + 127, 0) << 23 from the bit patterns of m
    const int e0 = max(static_cast<int>(static_cast<uint32_t>(m)) - (0x4B400000 - 127), 0);
    const int e1 = max(static_cast<int>(static_cast<uint32_t>(m >> 32)) - (0x4B400000 - 127), 0);
    float x0, x1;
    f2_unpack(f2_mul(p, (static_cast<uint64_t>(static_cast<uint32_t>(e1) << 23) << 32) |
                            (static_cast<uint32_t>(e0) << 23)),
              x0, x1);
    x0 = (x0 < kTiny) ? 0.0f : x0;  // step 7
    x1 = (x1 < kTiny) ? 0.0f : x1;
    w0 = fminf(x0, 1.0f);
    w1 = fminf(x1, 1.0f);
}

// ---------------------------------------------------------------- NS-5
// q = trunc(w * 2^kfx): w is 0 or a normal float in [2^-126, 1] (NS-4 flushes).
__device__ __forceinline__ uint64_t quantise(float w, int kfx) {
    // w * 2^kfx is exact in float (a power-of-two scale of a normal float in [2^-126, 1] with
    // 30 <= kfx <= 61 stays normal and below 2^62), and the conversion truncates toward zero:
    // q = trunc(w 2^kfx) exactly, as NS-5 defines it
    const float scaled = __fmul_rn(w, __uint_as_float(static_cast<uint32_t>(127 + kfx) << 23));
    return static_cast<uint64_t>(__float2ull_rz(scaled));
}

// w_i = dexp(fl(logw_i - lmax)) (NS-3)
__device__ __forceinline__ float weight(float logw, float lmax) { return dexp(__fsub_rn(logw, lmax)); }

// ---------------------------------------------------------------- NS-7..10
__device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b) { return __umul64hi(a, b); }

// ---------------------------------------------------------------- warp helpers
__device__ __forceinline__ uint64_t warp_incl_scan_u64(uint64_t v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t t = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}

// ---------------------------------------------------------------- lookback status words
// 64-bit word: [63:62] flag (0 empty, 1 aggregate, 2 inclusive prefix), [61:0] value.
// Values are <= 2^61 (NS-5) or packed pairs < 2^62 (permute).
constexpr uint64_t kFlagShift = 62;
constexpr uint64_t kFlagAgg = 1ull << kFlagShift;
constexpr uint64_t kFlagInc = 2ull << kFlagShift;
constexpr uint64_t kValueMask = (1ull << kFlagShift) - 1;

__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// Flag and value share one 64-bit word, so the lookback needs no acquire per
// probe: a relaxed (L1-bypassing) load sees a consistent (flag, value) pair.
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Warp-cooperative decoupled lookback (Merrill & Garland 2016) over the
// status words of tiles [0, tile) of one segment.  Returns the exclusive
// prefix of `tile`.  Must be called by a full warp.
__device__ __forceinline__ uint64_t lookback(const uint64_t* status, int64_t tile, int lane) {
    uint64_t prefix = 0;
    int64_t pred = tile - 1;
    while (true) {
        const int64_t idx = pred - lane;
        uint64_t s = (idx >= 0) ? ld_relaxed(status + idx) : kFlagInc;
        while (__any_sync(0xFFFFFFFFu, (s >> kFlagShift) == 0)) {
            if ((s >> kFlagShift) == 0) s = ld_relaxed(status + idx);
        }
        const uint32_t inc = __ballot_sync(0xFFFFFFFFu, (s >> kFlagShift) == 2);
        if (inc) {
            const int L = __ffs(inc) - 1;  // nearest inclusive predecessor
            const uint64_t v = (lane <= L) ? (s & kValueMask) : 0ull;
            prefix += warp_sum_u64(v);
            return prefix;
        }
        prefix += warp_sum_u64(s & kValueMask);
        pred -= 32;
    }
}

// ---------------------------------------------------------------- NS-12 (a6)
// Deterministic binary64 log of x in (0, 1]: x = m 2^e, m in [sqrt(1/2), sqrt 2),
// log m = 2 atanh(s), s = (m - 1)/(m + 1), series to s^19 (NS-12 constants).
__device__ __forceinline__ double ddlog(double x) {
    const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(x));
    int e = static_cast<int>((bits >> 52) & 0x7FF) - 1023;
    double m = __longlong_as_double(static_cast<long long>((bits & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull));
    if (m > __longlong_as_double(0x3FF6A09E667F3BCDll)) {
        m = __dmul_rn(m, 0.5);
        e = e + 1;
    }
    const double f = __dsub_rn(m, 1.0);
    const double s = __ddiv_rn(f, __dadd_rn(m, 1.0));
    const double z = __dmul_rn(s, s);
    double p = __longlong_as_double(0x3faaf286bca1af28ll);
    p = __fma_rn(p, z, __longlong_as_double(0x3fae1e1e1e1e1e1ell));
    p = __fma_rn(p, z, __longlong_as_double(0x3fb1111111111111ll));
    p = __fma_rn(p, z, __longlong_as_double(0x3fb3b13b13b13b14ll));
    p = __fma_rn(p, z, __longlong_as_double(0x3fb745d1745d1746ll));
    p = __fma_rn(p, z, __longlong_as_double(0x3fbc71c71c71c71cll));
    p = __fma_rn(p, z, __longlong_as_double(0x3fc2492492492492ll));
    p = __fma_rn(p, z, __longlong_as_double(0x3fc999999999999all));
    p = __fma_rn(p, z, __longlong_as_double(0x3fd5555555555555ll));
    const double t = __dmul_rn(2.0, s);
    const double r = __dmul_rn(t, z);
    const double logm = __fma_rn(r, p, t);
    const double de = static_cast<double>(e);
    const double lo = __dmul_rn(de, __longlong_as_double(0x3DEA39EF35793C76ll));
    const double b = __dadd_rn(lo, logm);
    const double hi = __dmul_rn(de, __longlong_as_double(0x3FE62E42FEE00000ll));
    return __dadd_rn(hi, b);
}

// e = trunc(-ddlog(U) 2^24) + 1 for the 32-bit draw r, U = (r + 1/2) 2^-32
__device__ __forceinline__ uint64_t spacing_from_word(uint32_t r) {
    const double U = __dmul_rn(__dadd_rn(static_cast<double>(r), 0.5), __longlong_as_double(0x3DF0000000000000ll));
    const double E = -ddlog(U);
    return static_cast<uint64_t>(__dmul_rn(E, 16777216.0)) + 1ull;
}

// floor(a * b / d) with the per-(b, d) constants ratio = b / d and inv_d = 1 / d precomputed
// (double): the same estimate + two coarse corrections + exact 128-bit fix-up as
// muldiv_floor below, without a double division per call
__device__ __forceinline__ uint64_t muldiv_floor_pre(uint64_t a, uint64_t b, uint64_t d, double ratio, double inv_d) {
    const uint64_t plo = a * b, phi = __umul64hi(a, b);
    uint64_t q = static_cast<uint64_t>(__dmul_rn(static_cast<double>(a), ratio));
    for (int it = 0; it < 2; ++it) {
        const uint64_t tlo = q * d, thi = __umul64hi(q, d);
        const uint64_t rlo = plo - tlo;
        const int64_t rhi = static_cast<int64_t>(phi - thi - (plo < tlo ? 1ull : 0ull));
        const double rd = __dadd_rn(__dmul_rn(static_cast<double>(rhi), 18446744073709551616.0),
                                    static_cast<double>(rlo));
        const double dq = floor(__dmul_rn(rd, inv_d));
        q = static_cast<uint64_t>(static_cast<int64_t>(q) + static_cast<int64_t>(dq));
    }
    for (int it = 0; it < 3; ++it) {
        const uint64_t tlo = q * d, thi = __umul64hi(q, d);
        if (thi > phi || (thi == phi && tlo > plo)) { --q; continue; }
        const uint64_t ulo = tlo + d, uhi = thi + (ulo < tlo ? 1ull : 0ull);
        if (uhi < phi || (uhi == phi && ulo <= plo)) { ++q; continue; }
        break;
    }
    return q;
}

// floor(a * b / d) for a < d (so the quotient is < b), exact: double estimate,
// then two exact 128-bit corrections.
__device__ __forceinline__ uint64_t muldiv_floor(uint64_t a, uint64_t b, uint64_t d) {
    const uint64_t plo = a * b, phi = __umul64hi(a, b);
    uint64_t q = static_cast<uint64_t>(__dmul_rn(static_cast<double>(a), __ddiv_rn(static_cast<double>(b),
                                                                                 static_cast<double>(d))));
    for (int it = 0; it < 2; ++it) {
        // r = p - q d as signed 128-bit; coarse correction by r / d in double
        const uint64_t tlo = q * d, thi = __umul64hi(q, d);
        const uint64_t rlo = plo - tlo;
        const int64_t rhi = static_cast<int64_t>(phi - thi - (plo < tlo ? 1ull : 0ull));
        const double rd = __dadd_rn(__dmul_rn(static_cast<double>(rhi), 18446744073709551616.0),
                                    static_cast<double>(rlo));
        const double dq = floor(__ddiv_rn(rd, static_cast<double>(d)));
        q = static_cast<uint64_t>(static_cast<int64_t>(q) + static_cast<int64_t>(dq));
    }
    // final exact fix-up: ensure q d <= p < (q + 1) d
    for (int it = 0; it < 3; ++it) {
        const uint64_t tlo = q * d, thi = __umul64hi(q, d);
        if (thi > phi || (thi == phi && tlo > plo)) { --q; continue; }
        const uint64_t ulo = tlo + d, uhi = thi + (ulo < tlo ? 1ull : 0ull);
        if (uhi < phi || (uhi == phi && ulo <= plo)) { ++q; continue; }
        break;
    }
    return q;
}

// ---------------------------------------------------------------- CTA-wide expansion helpers
// Head marks in shared memory (8 consecutive slots per thread) and their CTA-wide max-scan:
// a_k = max{i : head at or before k}, the expansion of run lengths into indices.
__device__ __forceinline__ void cta_clear8(int32_t* s_head, int tid) {
    int4* h4 = reinterpret_cast<int4*>(s_head);
    h4[2 * tid] = make_int4(-1, -1, -1, -1);
    h4[2 * tid + 1] = make_int4(-1, -1, -1, -1);
}

// CTA-wide inclusive max-scan of the kXS marks in s_head, 8 consecutive per thread (the
// caller has synchronised after marking): h[t] = max(carry, marks [0, 8 tid + t]); carry
// (block-uniform) becomes the chunk maximum.  One barrier.
template <int FW>
__device__ __forceinline__ void cta_max_scan8(const int32_t* s_head, int32_t* s_wmax, int32_t h[8], int32_t& carry,
                                              int tid, int warp, int lane) {
    const int4* h4 = reinterpret_cast<const int4*>(s_head);
    const int4 lo = h4[2 * tid], hi = h4[2 * tid + 1];
    h[0] = lo.x; h[1] = lo.y; h[2] = lo.z; h[3] = lo.w; h[4] = hi.x; h[5] = hi.y; h[6] = hi.z; h[7] = hi.w;
#pragma unroll
    for (int t = 1; t < 8; ++t) h[t] = max(h[t], h[t - 1]);
    int32_t incl = h[7];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t u = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl = max(incl, u);
    }
    if (lane == 31) s_wmax[warp] = incl;
    __syncthreads();
    int32_t w = (lane < FW) ? s_wmax[lane] : -1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t u = __shfl_up_sync(0xFFFFFFFFu, w, o);
        if (lane >= o) w = max(w, u);
    }
    const int32_t wpre = __shfl_sync(0xFFFFFFFFu, w, (warp + 31) & 31);  // inclusive of warp - 1
    const int32_t tot = __shfl_sync(0xFFFFFFFFu, w, 31);
    int32_t pre = __shfl_up_sync(0xFFFFFFFFu, incl, 1);
    pre = (lane == 0) ? -1 : pre;
    pre = max(max(pre, carry), (warp == 0) ? -1 : wpre);
#pragma unroll
    for (int t = 0; t < 8; ++t) h[t] = max(h[t], pre);
    carry = max(carry, tot);
}

// Host/device shared integer helpers (no method arithmetic beyond NS-5/NS-7 sizes).
__host__ __device__ __forceinline__ int ceil_log2(int64_t P) {
    int m = 0;
    while ((int64_t{1} << m) < P) ++m;
    return m;
}

}  // namespace pf
