/*
 * oracle/pfo.c — plain, slow, single-threaded CPU oracle for the resampling
 * hot path of arXiv 1202.6163 ("particle filter resampling on GPUs").
 *
 * TEST INFRASTRUCTURE ONLY (see pfo.h).  Never linked by the product path.
 *
 * Written step by step from PAPER.md (P:n) and the numeric spec DESIGN.md §3
 * (NS-n).  No blocking, no fusion, no reordering: every function follows the
 * definition in the order the text states it.  Build flags (see
 * __graft_entry__.build): -O2 -ffp-contract=off -fno-fast-math, so that every
 * float operation below is one IEEE-754 binary32 operation, round-to-nearest.
 *
 * Pins (what fixes each function other than itself) are listed in DESIGN.md
 * §4 and implemented in tests/test_oracle_*.py.
 */
#include "pfo.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* NS-6  Philox4x32-10 (Salmon, Moraes, Dror, Shaw 2011; Random123).        */
/* Round: (hi(M1*c2)^c1^k0, lo(M1*c2), hi(M0*c0)^c3^k1, lo(M0*c0)); the key   */
/* is bumped by the Weyl constants between rounds.                           */
/* ------------------------------------------------------------------------ */
void pfo_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t prod0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t prod1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t n0 = (uint32_t)(prod1 >> 32) ^ c1 ^ k0;
        uint32_t n1 = (uint32_t)prod1;
        uint32_t n2 = (uint32_t)(prod0 >> 32) ^ c3 ^ k1;
        uint32_t n3 = (uint32_t)prod0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* NS-6: one Philox call with key = (lo32(seed), hi32(seed)) and counter
 * (c0, c1, tag, filter_index). */
static void philox_draw(uint64_t seed, uint32_t c0, uint32_t c1, uint32_t tag,
                        uint32_t filter_index, uint32_t out[4])
{
    uint32_t ctr[4] = { c0, c1, tag, filter_index };
    uint32_t key[2] = { (uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32) };
    pfo_philox4x32_10(ctr, key, out);
}

/* NS-6: 64-bit word "half h" of a Philox output. */
static uint64_t philox_half(const uint32_t x[4], int h)
{
    if (h == 0) return ((uint64_t)x[1] << 32) | (uint64_t)x[0];
    return ((uint64_t)x[3] << 32) | (uint64_t)x[2];
}

/* ------------------------------------------------------------------------ */
/* NS-4  dexp: deterministic float32 exp for t <= 0.                        */
/* ------------------------------------------------------------------------ */
static float f32_from_bits(uint32_t b)
{
    float f;
    memcpy(&f, &b, sizeof f);
    return f;
}

float pfo_dexp(float t)
{
    /* constants of NS-4, given by their binary32 bit patterns */
    const float LOG2E = f32_from_bits(0x3FB8AA3Bu);  /* 1.44269502       */
    const float LN2_HI = f32_from_bits(0x3F317200u); /* 0.693145751953125 */
    const float LN2_LO = f32_from_bits(0x35BFBE8Eu); /* 1.42860677e-06   */
    const float C2 = f32_from_bits(0x3F000000u);     /* 1/2   */
    const float C3 = f32_from_bits(0x3E2AAAABu);     /* 1/6   */
    const float C4 = f32_from_bits(0x3D2AAAABu);     /* 1/24  */
    const float C5 = f32_from_bits(0x3C088889u);     /* 1/120 */
    const float C6 = f32_from_bits(0x3AB60B61u);     /* 1/720 */
    const float C7 = f32_from_bits(0x39500D01u);     /* 1/5040 */
    const float TINY = f32_from_bits(0x00800000u);   /* 2^-126 */

    /* step 1: exp(t) < 2^-126 for t < -88, and -inf means zero weight */
    if (!(t >= -88.0f)) return 0.0f;
    /* step 2: subnormal t behaves as 0 (independent of FTZ/DAZ) */
    if (fabsf(t) < TINY) t = 0.0f;
    /* step 3: n = rint(t * log2 e) */
    float tl = t * LOG2E;
    float n = rintf(tl);
    /* step 4: Cody-Waite reduction r = t - n*ln2 in two fma steps */
    float r = fmaf(-n, LN2_HI, t);
    r = fmaf(-n, LN2_LO, r);
    /* step 5: degree-7 Taylor polynomial, Horner in fma */
    float p = C7;
    p = fmaf(p, r, C6);
    p = fmaf(p, r, C5);
    p = fmaf(p, r, C4);
    p = fmaf(p, r, C3);
    p = fmaf(p, r, C2);
    p = fmaf(p, r, 1.0f);
    p = fmaf(p, r, 1.0f);
    /* step 6: scale by 2^n (n in [-127, 0]); 2^-127 is below the flush limit */
    int ni = (int)n;
    if (ni < -126) return 0.0f;
    float scale = f32_from_bits((uint32_t)(ni + 127) << 23);
    float w = p * scale;
    /* step 7: explicit flush below 2^-126 and clamp to 1 */
    if (w < TINY) return 0.0f;
    if (w > 1.0f) w = 1.0f;
    return w;
}

/* ------------------------------------------------------------------------ */
/* NS-1 / NS-2  validation and log-weight maximum.                          */
/* ------------------------------------------------------------------------ */
int pfo_lmax(const float* logw, int32_t P, float* lmax)
{
    float m = -INFINITY;
    int bad = 0;
    for (int32_t i = 0; i < P; ++i) {
        float v = logw[i];
        if (isnan(v) || (isinf(v) && v > 0)) bad = 1;
        else if (v > m) m = v;
    }
    *lmax = m;
    if (bad || m == -INFINITY) return PFO_FILTER_INVALID_WEIGHTS;
    return PFO_FILTER_OK;
}

/* NS-3 / NS-4 with a given maximum (used for a shard of a larger filter) */
void pfo_weights_with(const float* logw, int32_t P, float lmax, float* w)
{
    for (int32_t i = 0; i < P; ++i) {
        float t = logw[i] - lmax; /* one binary32 subtraction, RN */
        w[i] = pfo_dexp(t);
    }
}

/* NS-3 / NS-4 */
int pfo_weights(const float* logw, int32_t P, float* w)
{
    float lmax;
    int st = pfo_lmax(logw, P, &lmax);
    if (st != PFO_FILTER_OK) return st;
    pfo_weights_with(logw, P, lmax, w);
    return PFO_FILTER_OK;
}

/* NS-5 */
static int ceil_log2(int64_t P)
{
    int m = 0;
    while (((int64_t)1 << m) < P) ++m;
    return m;
}

int pfo_kfx(int32_t P) { return 61 - ceil_log2(P); }

/* NS-5 with a given maximum and fraction bits: inclusive scan of q_i */
void pfo_cumulative_with(const float* logw, int32_t P, float lmax, int kfx, uint64_t* Q)
{
    float* w = (float*)malloc(sizeof(float) * (size_t)(P > 0 ? P : 1));
    pfo_weights_with(logw, P, lmax, w);
    double scale = ldexp(1.0, kfx); /* 2^k_fx */
    uint64_t acc = 0;
    for (int32_t i = 0; i < P; ++i) {
        /* exact: a 24-bit mantissa times a power of two, then truncate */
        uint64_t q = (uint64_t)((double)w[i] * scale);
        acc += q;
        Q[i] = acc;
    }
    free(w);
}

int pfo_cumulative(const float* logw, int32_t P, uint64_t* Q)
{
    float lmax;
    int st = pfo_lmax(logw, P, &lmax);
    if (st == PFO_FILTER_OK) pfo_cumulative_with(logw, P, lmax, pfo_kfx(P), Q);
    return st;
}

/* ------------------------------------------------------------------------ */
/* NS-7..NS-10  positions on the weight circle (Fig. 1).          */
/* ------------------------------------------------------------------------ */
static uint64_t mulhi64(uint64_t a, uint64_t b)
{
    return (uint64_t)(((unsigned __int128)a * (unsigned __int128)b) >> 64);
}

/* NS-7: stratum width as a 64-bit fraction, P >= 2 */
static uint64_t stratum_width(int32_t P)
{
    if ((P & (P - 1)) == 0) return (uint64_t)1 << (64 - ceil_log2(P));
    return UINT64_MAX / (uint64_t)P;
}

uint64_t pfo_position(int scheme, int32_t P, uint64_t Qtot, uint64_t seed,
                      uint32_t filter_index, int64_t k)
{
    uint32_t x[4];
    if (scheme == PFO_MULTINOMIAL) {
        /* NS-8, Fig. 1(a): i.i.d. uniform position per slot */
        philox_draw(seed, (uint32_t)(k >> 1), 0u, PFO_MULTINOMIAL, filter_index, x);
        uint64_t R = philox_half(x, (int)(k & 1));
        return mulhi64(R, Qtot);
    }
    uint64_t D = stratum_width(P);
    uint64_t rho;
    if (scheme == PFO_STRATIFIED) {
        /* NS-9, Fig. 1(b): own random offset per stratum */
        philox_draw(seed, (uint32_t)(k >> 1), 0u, PFO_STRATIFIED, filter_index, x);
        rho = mulhi64(philox_half(x, (int)(k & 1)), D);
    } else {
        /* NS-10, Fig. 1(c): the same offset in every stratum */
        philox_draw(seed, 0u, 0u, PFO_SYSTEMATIC, filter_index, x);
        rho = mulhi64(philox_half(x, 0), D);
    }
    uint64_t S = (uint64_t)k * D + rho;
    return mulhi64(S, Qtot);
}

int32_t pfo_upper_bound(const uint64_t* Q, int32_t P, uint64_t x)
{
    /* smallest i with Q[i] > x; Q is nondecreasing and Q[P-1] > x */
    int32_t lo = 0, hi = P - 1;
    while (lo < hi) {
        int32_t mid = lo + (hi - lo) / 2;
        if (Q[mid] > x) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

void pfo_systematic_from_R(const uint64_t* Q, int32_t P, uint64_t R, int32_t* anc)
{
    uint64_t D = stratum_width(P);
    uint64_t rho = mulhi64(R, D);
    for (int32_t k = 0; k < P; ++k) {
        uint64_t S = (uint64_t)k * D + rho;
        anc[k] = pfo_upper_bound(Q, P, mulhi64(S, Q[P - 1]));
    }
}

/* ------------------------------------------------------------------------ */
/* NS-11  Metropolis resampler.                      */
/* ------------------------------------------------------------------------ */
void pfo_metropolis_chains(const float* w, int32_t P, int64_t slot0, int32_t nslots,
                           uint64_t seed, int32_t B, uint32_t filter_index, int32_t* anc)
{
    for (int32_t s = 0; s < nslots; ++s) {
        int64_t i = slot0 + s;
        int64_t k = i;       /* G3: chain starts at its own particle */
        float wk = w[k];
        uint32_t x[4] = { 0, 0, 0, 0 };
        for (int32_t b = 0; b < B; ++b) {
            if ((b & 1) == 0)
                philox_draw(seed, (uint32_t)i, (uint32_t)(b >> 1), PFO_METROPOLIS, filter_index, x);
            uint32_t rj = (b & 1) ? x[2] : x[0];
            uint32_t ru = (b & 1) ? x[3] : x[1];
            /* proposal: uniform over all particle indices (line:proposal) */
            int64_t j = (int64_t)(((uint64_t)rj * (uint64_t)P) >> 32);
            /* u on the 24-bit grid of [0,1) */
            float u = (float)(ru >> 8) * f32_from_bits(0x33800000u); /* 2^-24 */
            float wj = w[j];
            /* Metropolis criterion (line:accept): accept j iff u*w_k < w_j */
            float uw = u * wk;
            if (uw < wj) {
                k = j;
                wk = wj;
            }
        }
        anc[s] = (int32_t)k;
    }
}

/* ------------------------------------------------------------------------ */
/* Full single-filter resampling: P:64-68 problem statement.                */
/* ------------------------------------------------------------------------ */
int pfo_resample(int scheme, const float* logw, int32_t P, uint64_t seed, int32_t B,
                 uint32_t filter_index, int32_t* anc, double* lse, float* normw, double* ess)
{
    float lmax;
    int st = pfo_lmax(logw, P, &lmax);
    if (st != PFO_FILTER_OK) {
        /* NS-1: invalid input -> identity ancestors, NaN side outputs */
        for (int32_t i = 0; i < P; ++i) anc[i] = i;
        if (lse) *lse = NAN;
        if (ess) *ess = NAN;
        if (normw) for (int32_t i = 0; i < P; ++i) normw[i] = NAN;
        return st;
    }
    float* w = (float*)malloc(sizeof(float) * (size_t)P);
    pfo_weights(logw, P, w);

    /* NS-13 side outputs: sequential double sums */
    double S = 0.0, S2 = 0.0;
    for (int32_t i = 0; i < P; ++i) {
        S += (double)w[i];
        S2 += (double)w[i] * (double)w[i];
    }
    if (lse) *lse = (double)lmax + log(S);
    if (ess) *ess = S * S / S2;
    if (normw) for (int32_t i = 0; i < P; ++i) normw[i] = (float)((double)w[i] / S);

    if (scheme == PFO_METROPOLIS) {
        pfo_metropolis_chains(w, P, 0, P, seed, B, filter_index, anc);
        free(w);
        return PFO_FILTER_OK;
    }
    if (P == 1) { /* NS-7 */
        anc[0] = 0;
        free(w);
        return PFO_FILTER_OK;
    }
    uint64_t* Q = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)P);
    pfo_cumulative(logw, P, Q);
    uint64_t Qtot = Q[P - 1];
    for (int32_t k = 0; k < P; ++k) {
        uint64_t xk = pfo_position(scheme, P, Qtot, seed, filter_index, k);
        anc[k] = pfo_upper_bound(Q, P, xk);
    }
    free(Q);
    free(w);
    return PFO_FILTER_OK;
}

void pfo_resample_batched(int scheme, const float* logw, int64_t ld_logw, int32_t N, int32_t P,
                          uint64_t seed, uint32_t first_filter, int32_t B,
                          int32_t* anc, int64_t ld_anc, int32_t* status)
{
    for (int32_t n = 0; n < N; ++n) {
        int st = pfo_resample(scheme, logw + (int64_t)n * ld_logw, P, seed, B,
                              first_filter + (uint32_t)n, anc + (int64_t)n * ld_anc,
                              NULL, NULL, NULL);
        if (status) status[n] = st;
    }
}

/* ------------------------------------------------------------------------ */
/* NS-12  sorted-uniform multinomial (variant a6): exponential spacings.     */
/* The P order statistics of P i.i.d. uniforms are G_k / G_P, k < P, where   */
/* G_k = e_0 + ... + e_k and e_j are i.i.d. exponentials; here fixed point.  */
/* ------------------------------------------------------------------------ */
static double f64_from_bits(uint64_t b)
{
    double d;
    memcpy(&d, &b, sizeof d);
    return d;
}

/* deterministic natural log of x in (0, 1]: x = m 2^e, m in [sqrt(1/2), sqrt 2),
 * log m = 2 atanh(s), s = (m - 1)/(m + 1), series to s^19; every operation is
 * one IEEE binary64 operation (NS-12) */
double pfo_dlog(double x)
{
    uint64_t bits;
    memcpy(&bits, &x, sizeof bits);
    int e = (int)((bits >> 52) & 0x7FF) - 1023;
    double m = f64_from_bits((bits & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull); /* [1, 2) */
    if (m > f64_from_bits(0x3FF6A09E667F3BCDull)) { /* sqrt 2 */
        m = m * 0.5;
        e = e + 1;
    }
    double f = m - 1.0;
    double s = f / (m + 1.0);
    double z = s * s;
    double p = f64_from_bits(0x3faaf286bca1af28ull);            /* 1/19 */
    p = fma(p, z, f64_from_bits(0x3fae1e1e1e1e1e1eull));       /* 1/17 */
    p = fma(p, z, f64_from_bits(0x3fb1111111111111ull));       /* 1/15 */
    p = fma(p, z, f64_from_bits(0x3fb3b13b13b13b14ull));       /* 1/13 */
    p = fma(p, z, f64_from_bits(0x3fb745d1745d1746ull));       /* 1/11 */
    p = fma(p, z, f64_from_bits(0x3fbc71c71c71c71cull));       /* 1/9  */
    p = fma(p, z, f64_from_bits(0x3fc2492492492492ull));       /* 1/7  */
    p = fma(p, z, f64_from_bits(0x3fc999999999999aull));       /* 1/5  */
    p = fma(p, z, f64_from_bits(0x3fd5555555555555ull));       /* 1/3  */
    double t = 2.0 * s;
    double r = t * z;
    double logm = fma(r, p, t);
    double de = (double)e;
    double lo = de * f64_from_bits(0x3DEA39EF35793C76ull);     /* e ln2_lo */
    double b = lo + logm;
    double hi = de * f64_from_bits(0x3FE62E42FEE00000ull);     /* e ln2_hi (exact) */
    return hi + b;
}

/* e_k = trunc(-dlog(U_k) 2^24) + 1, U_k = (r_k + 1/2) 2^-32, r_k = word (k & 3) of
 * Philox(k >> 2, 0, tag 5, filter) */
uint64_t pfo_spacing(uint64_t seed, uint32_t filter_index, int64_t k)
{
    uint32_t x[4];
    philox_draw(seed, (uint32_t)(k >> 2), 0u, 5u, filter_index, x);
    double U = ((double)x[k & 3] + 0.5) * f64_from_bits(0x3DF0000000000000ull); /* 2^-32 */
    double E = -pfo_dlog(U);
    return (uint64_t)(E * 16777216.0) + 1u;
}

/* G_k = e_0 + ... + e_k for k = 0..P (P + 1 values) */
void pfo_spacings(int32_t P, uint64_t seed, uint32_t filter_index, uint64_t* G)
{
    uint64_t acc = 0;
    for (int64_t k = 0; k <= P; ++k) {
        acc += pfo_spacing(seed, filter_index, k);
        G[k] = acc;
    }
}

/* slot k < P: position x_k = floor(G_k Q / G_P); a_k = min{i : Q_i > x_k} */
int pfo_resample_sorted_multinomial(const float* logw, int32_t P, uint64_t seed, uint32_t filter_index,
                                    int32_t* anc)
{
    uint64_t* Q = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)P);
    int st = pfo_cumulative(logw, P, Q);
    if (st != PFO_FILTER_OK) {
        for (int32_t i = 0; i < P; ++i) anc[i] = i;
        free(Q);
        return st;
    }
    uint64_t* G = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)P + 1));
    pfo_spacings(P, seed, filter_index, G);
    uint64_t Qtot = Q[P - 1], GP = G[P];
    for (int32_t k = 0; k < P; ++k) {
        uint64_t x = (uint64_t)(((unsigned __int128)G[k] * (unsigned __int128)Qtot) / (unsigned __int128)GP);
        anc[k] = pfo_upper_bound(Q, P, x);
    }
    free(G);
    free(Q);
    return PFO_FILTER_OK;
}

/* ------------------------------------------------------------------------ */
/* NS-3d  binary64 log-weights (the paper computes in double;        */
/* reading R-21).  NS-1 validation and the NS-2 max on the doubles; then    */
/* t_i = the binary64 difference logw_i - lmax rounded ONCE to binary32      */
/* (nearest; below -FLT_MAX it is -inf, and any t < -88 weighs 0 by NS-4),  */
/* and the float32 path NS-3..NS-12 runs on t, whose maximum is exactly 0.  */
/* lse = lmax + ln S (NS-13 with the double maximum).                       */
/* ------------------------------------------------------------------------ */
int pfo_shift_f64(const double* logw, int32_t P, float* t, double* lmax)
{
    double m = -INFINITY;
    int bad = 0;
    for (int32_t i = 0; i < P; ++i) {
        double v = logw[i];
        if (isnan(v) || (isinf(v) && v > 0)) bad = 1;
        else if (v > m) m = v;
    }
    *lmax = m;
    if (bad || m == -INFINITY) {
        for (int32_t i = 0; i < P; ++i) t[i] = NAN; /* invalid for the float path too (NS-1) */
        return PFO_FILTER_INVALID_WEIGHTS;
    }
    for (int32_t i = 0; i < P; ++i) {
        double d = logw[i] - m; /* one binary64 subtraction, RN */
        t[i] = (d < -FLT_MAX) ? -INFINITY : (float)d;
    }
    return PFO_FILTER_OK;
}

int pfo_resample_f64(int scheme, int sorted, const double* logw, int32_t P, uint64_t seed, int32_t B,
                     uint32_t filter_index, int32_t* anc, double* lse, float* normw, double* ess)
{
    float* t = (float*)malloc(sizeof(float) * (size_t)P);
    double lm;
    int st = pfo_shift_f64(logw, P, t, &lm);
    if (sorted) {
        pfo_resample_sorted_multinomial(t, P, seed, filter_index, anc);
        if (lse || normw || ess) { /* side outputs do not depend on the positions */
            int32_t* scratch = (int32_t*)malloc(sizeof(int32_t) * (size_t)P);
            pfo_resample(PFO_SYSTEMATIC, t, P, seed, 0, filter_index, scratch, lse, normw, ess);
            free(scratch);
        }
    } else {
        pfo_resample(scheme, t, P, seed, B, filter_index, anc, lse, normw, ess);
    }
    if (lse && st == PFO_FILTER_OK) *lse = lm + *lse; /* the float path's lse is 0 + ln S */
    free(t);
    return st;
}

/* ------------------------------------------------------------------------ */
/* NS-17  pre-sorted weights (the paper's "sorting enabled" series,         */
/* P:226-231; reading R-14).  sigma = the indices in DESCENDING order of    */
/* logw, equal values (+0 == -0) in ascending index order; the float32 path */
/* resamples y_j = logw[sigma_j] (same seed and filter index) into b, and   */
/* a_k = sigma[b_k]; v_{sigma_j} = the normalised weight of y_j.  Invalid   */
/* filters (NS-1) give the identity.                                        */
/* ------------------------------------------------------------------------ */
static const float* g_sort_keys; /* qsort context (single-threaded oracle) */

static int desc_then_index(const void* pa, const void* pb)
{
    int32_t a = *(const int32_t*)pa, b = *(const int32_t*)pb;
    float x = g_sort_keys[a], y = g_sort_keys[b];
    if (x > y) return -1;
    if (x < y) return 1;
    return (a < b) ? -1 : (a > b); /* equal values (incl. +0 / -0): index order */
}

int pfo_resample_sorted_weights(int scheme, const float* logw, int32_t P, uint64_t seed, uint32_t filter_index,
                                int32_t* anc, double* lse, float* normw, double* ess)
{
    float lm;
    int st = pfo_lmax(logw, P, &lm);
    if (st != PFO_FILTER_OK) /* NS-1 outputs, no sort */
        return pfo_resample(scheme, logw, P, seed, 0, filter_index, anc, lse, normw, ess);
    int32_t* sigma = (int32_t*)malloc(sizeof(int32_t) * (size_t)P);
    for (int32_t i = 0; i < P; ++i) sigma[i] = i;
    g_sort_keys = logw;
    qsort(sigma, (size_t)P, sizeof(int32_t), desc_then_index);
    float* y = (float*)malloc(sizeof(float) * (size_t)P);
    for (int32_t j = 0; j < P; ++j) y[j] = logw[sigma[j]];
    int32_t* b = (int32_t*)malloc(sizeof(int32_t) * (size_t)P);
    float* vy = normw ? (float*)malloc(sizeof(float) * (size_t)P) : NULL;
    pfo_resample(scheme, y, P, seed, 0, filter_index, b, lse, vy, ess);
    for (int32_t k = 0; k < P; ++k) anc[k] = sigma[b[k]];
    if (normw) {
        for (int32_t j = 0; j < P; ++j) normw[sigma[j]] = vy[j];
        free(vy);
    }
    free(b);
    free(y);
    free(sigma);
    return PFO_FILTER_OK;
}

/* ------------------------------------------------------------------------ */
/* NS-14 conversions ("Converting between the two is straightforward"). */
/* ------------------------------------------------------------------------ */
void pfo_ancestors_to_offspring(const int32_t* anc, int32_t P, int32_t* o)
{
    for (int32_t i = 0; i < P; ++i) o[i] = 0;
    for (int32_t k = 0; k < P; ++k) o[anc[k]] += 1;
}

void pfo_offspring_to_ancestors(const int32_t* o, int32_t P, int32_t* anc)
{
    /* cumulative convention */
    int32_t k = 0;
    for (int32_t i = 0; i < P; ++i)
        for (int32_t c = 0; c < o[i]; ++c) anc[k++] = i;
}

/* ------------------------------------------------------------------------ */
/* NS-15 canonical permutation: survivors stay in their own slot; the r-th  */
/* free slot (ascending) receives the r-th extra copy (ascending survivor).  */
/* ------------------------------------------------------------------------ */
void pfo_permute(const int32_t* anc, int32_t P, int32_t* perm)
{
    int32_t* o = (int32_t*)malloc(sizeof(int32_t) * (size_t)P);
    pfo_ancestors_to_offspring(anc, P, o);
    /* survivors */
    for (int32_t i = 0; i < P; ++i) perm[i] = (o[i] > 0) ? i : -1;
    /* walk the extras list and the free-slot list together */
    int32_t f = 0; /* next free-slot candidate */
    for (int32_t i = 0; i < P; ++i) {
        for (int32_t c = 1; c < o[i]; ++c) {
            while (o[f] != 0) ++f;
            perm[f] = i;
            ++f;
        }
    }
    free(o);
}

/* NS-16 */
void pfo_gather_inplace(void* X, int64_t row_bytes, int64_t ld_bytes, int32_t P, const int32_t* perm)
{
    char* base = (char*)X;
    for (int32_t i = 0; i < P; ++i)
        if (perm[i] != i)
            memcpy(base + (int64_t)i * ld_bytes, base + (int64_t)perm[i] * ld_bytes, (size_t)row_bytes);
}

void pfo_gather_out(const void* X, void* Y, int64_t row_bytes, int64_t ld_x, int64_t ld_y,
                    int32_t P, const int32_t* anc)
{
    const char* xs = (const char*)X;
    char* ys = (char*)Y;
    for (int32_t i = 0; i < P; ++i)
        memcpy(ys + (int64_t)i * ld_y, xs + (int64_t)anc[i] * ld_x, (size_t)row_bytes);
}

/* ------------------------------------------------------------------------ */
/* P:142-186 two-state chain, Eq. (2) alpha, beta = 1/P, Eq. (5).           */
/* ------------------------------------------------------------------------ */
/* Readings (R-22): B >= 1 (B = max(1, ceil(Eq. (5)))); w_max < 1/P
 * lies outside Eq. (2)'s domain and a B beyond int32 is not representable:
 * both return -1. */
int32_t pfo_metropolis_required_B(int64_t P, double w_max, double eps)
{
    double beta = 1.0 / (double)P;
    if (w_max * (double)P < 1.0 - 1e-12) return -1;            /* w_max >= 1/P */
    double alpha = (1.0 - w_max) / ((double)P * w_max);         /* Eq. (2) */
    double lambda = 1.0 - alpha - beta;
    double mx = alpha > beta ? alpha : beta;
    double target = eps * (alpha + beta) / mx;                  /* Eq. (4) */
    if (target >= 1.0) return 1;                                /* S:250 clamp */
    if (lambda <= 0.0) return 1;
    double B = ceil(log(target) / log(lambda));                 /* Eq. (5) */
    if (B > 2147483647.0) return -1;
    return B < 1.0 ? 1 : (int32_t)B;
}
