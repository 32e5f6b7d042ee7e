// pf_kernels.cu — sm_100a kernels of libpfresample.
//
// Stage map:
//   k_max       a1      log-weight max-reduce + validation           HBM 4 B/particle
//   k_scan      a2+a3   dexp -> u64 fixed point -> decoupled-lookback inclusive scan
//                                                                    HBM 4 B in + 8 B out
//   k_merge     a4+a5   merge-path search of sorted positions (stratified / systematic)
//                                                                    HBM 8 B in + 4 B out
//   k_merge<ModeBuckets> + k_bsearch_buckets  a4+a5  multinomial (bucket index + short per-slot searches)
//   k_mexp/k_metro a7   Metropolis: weights once, then B-step chains (no collective)
//   k_hist      a8      ancestors -> offspring (warp-aggregated atomics)
//   k_pscan+k_merge a9  canonical in-place permutation
//   k_gather_*  a10     state gather (16-byte vectors)
// Every kernel takes the filter index n as part of a flat grid, so a batch of
// N independent filters (a11) is one launch per stage.
#include <cfloat>
#include <cmath>

#include "pf_device.cuh"
#include "pf_internal.h"

namespace pf {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ============================================================================ a1: max
template <bool VEC>
__global__ void __launch_bounds__(kThreads) k_max(const float* __restrict__ logw, int64_t ld, int32_t P,
                                                  int cpf, int64_t chunk, Ws ws, int32_t* status_out,
                                                  float* lmax_out, int32_t* bad_out) {
    __shared__ float s_m[kThreads / 32];
    __shared__ int s_b[kThreads / 32];
    __shared__ int s_last;
    const int n = blockIdx.x / cpf;
    const int c = blockIdx.x - n * cpf;
    const int tid = threadIdx.x;
    const float* row = logw + static_cast<int64_t>(n) * ld;
    const int64_t beg = static_cast<int64_t>(c) * chunk;
    const int64_t end = min(static_cast<int64_t>(P), beg + chunk);
    float m = -INFINITY;
    int bad = 0;
    auto upd = [&](float v) {
        if (isnan(v) || v == INFINITY) bad = 1;
        else m = fmaxf(m, v);
    };
    int64_t i = beg + tid;
    if (VEC) {
        const float4* r4 = reinterpret_cast<const float4*>(row + beg);
        const int64_t n4 = (end > beg) ? (end - beg) / 4 : 0;
        for (int64_t t = tid; t < n4; t += kThreads) {
            const float4 v = __ldg(r4 + t);
            upd(v.x); upd(v.y); upd(v.z); upd(v.w);
        }
        i = beg + n4 * 4 + tid;
    }
    for (; i < end; i += kThreads) upd(__ldg(row + i));
    // block reduce
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
        bad |= __shfl_xor_sync(kFull, bad, o);
    }
    const int warp = tid >> 5, lane = tid & 31;
    if (lane == 0) { s_m[warp] = m; s_b[warp] = bad; }
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < kThreads / 32; ++w) { m = fmaxf(m, s_m[w]); bad |= s_b[w]; }
        bool finalize = true;
        if (cpf > 1) {
            ws.max_part[static_cast<int64_t>(n) * cpf + c] = m;
            ws.max_bad[static_cast<int64_t>(n) * cpf + c] = bad;
            __threadfence();
            const unsigned prev = atomicAdd(ws.max_cnt + n, 1u);
            finalize = (prev == static_cast<unsigned>(cpf - 1));
        }
        s_last = finalize ? 1 : 0;
    }
    __syncthreads();
    if (!s_last) return;
    if (cpf > 1) {
        __threadfence();
        m = -INFINITY;
        bad = 0;
        for (int t = tid; t < cpf; t += kThreads) {
            m = fmaxf(m, __ldcg(ws.max_part + static_cast<int64_t>(n) * cpf + t));
            bad |= __ldcg(ws.max_bad + static_cast<int64_t>(n) * cpf + t);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
            bad |= __shfl_xor_sync(kFull, bad, o);
        }
        __syncthreads();
        if (lane == 0) { s_m[warp] = m; s_b[warp] = bad; }
        __syncthreads();
        if (tid == 0) for (int w = 0; w < kThreads / 32; ++w) { m = fmaxf(m, s_m[w]); bad |= s_b[w]; }
    }
    if (tid == 0) {
        const int st = (bad || m == -INFINITY) ? 1 : 0;
        ws.lmax[n] = m;
        ws.fstatus[n] = st;
        if (status_out) status_out[n] = st;
        if (lmax_out) lmax_out[n] = m;
        if (bad_out) bad_out[n] = bad;
    }
}

// ============================================================================ a2+a3: scan
// One tile = 4096 particles = 8 warps x 4 rows x (32 lanes x 4 contiguous items).
// Tiles are taken in order from an atomic counter (forward progress of the
// lookback), never straddle filters, and publish (aggregate | inclusive) words.
template <bool VEC>
__global__ void __launch_bounds__(kThreads, 4) k_scan(const float* __restrict__ logw, int64_t ld, int32_t P, int T,
                                                   int kfx, Ws ws, int64_t ldq, int write_q, double* lse_out,
                                                   double* ess_out) {
    __shared__ uint32_t s_tile;
    __shared__ uint64_t s_wtot[kThreads / 32];
    __shared__ double s_sw[kThreads / 32], s_sw2[kThreads / 32];
    __shared__ uint64_t s_off[kThreads / 32];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) s_tile = atomicAdd(ws.tile_ctr, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int n = static_cast<int>(tile / T);
    const int j = static_cast<int>(tile - static_cast<int64_t>(n) * T);
    if (ws.fstatus[n] != 0) {
        if (j == T - 1 && tid == 0) {
            if (lse_out) lse_out[n] = NAN;
            if (ess_out) ess_out[n] = NAN;
            ws.S[n] = NAN;
        }
        return;
    }
    const float lm = ws.lmax[n];
    const float* row = logw + static_cast<int64_t>(n) * ld;
    const int64_t base = static_cast<int64_t>(j) * kTile + warp * 512;

    // Pass 1: load all 16 log-weights first (4 x 16-byte loads in flight), then
    // weights.  Registers hold only w (16 floats) and the per-row exclusive
    // lane offsets (4 x u64); q is recomputed after the tile prefix arrives.
    float w[16];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int64_t i0 = base + r * 128 + lane * 4;
        if (VEC && i0 + 3 < P) {
            const float4 t = __ldcs(reinterpret_cast<const float4*>(row + i0));
            w[r * 4 + 0] = t.x; w[r * 4 + 1] = t.y; w[r * 4 + 2] = t.z; w[r * 4 + 3] = t.w;
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) w[r * 4 + c] = (i0 + c < P) ? row[i0 + c] : -INFINITY;
        }
    }
    double sw = 0.0, sw2 = 0.0;
    uint64_t excl[4];
    uint64_t carry = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        uint64_t loc = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const float wv = weight(w[r * 4 + c], lm);
            w[r * 4 + c] = wv;
            sw += static_cast<double>(wv);
            sw2 += static_cast<double>(wv) * static_cast<double>(wv);
            loc += quantise(wv, kfx);
        }
        const uint64_t incl = warp_incl_scan_u64(loc, lane);
        excl[r] = incl - loc + carry;
        carry += __shfl_sync(kFull, incl, 31);
    }
    sw = warp_sum_f64(sw);
    sw2 = warp_sum_f64(sw2);
    if (lane == 0) { s_wtot[warp] = carry; s_sw[warp] = sw; s_sw2[warp] = sw2; }
    __syncthreads();
    if (warp == 0) {
        const uint64_t wv = (lane < kThreads / 32) ? s_wtot[lane] : 0ull;
        const uint64_t wi = warp_incl_scan_u64(wv, lane);
        const uint64_t agg = __shfl_sync(kFull, wi, kThreads / 32 - 1);
        uint64_t* st = ws.tstatus + static_cast<int64_t>(n) * T;
        if (lane == 0) {
            double a = 0.0, b = 0.0;
            for (int k = 0; k < kThreads / 32; ++k) { a += s_sw[k]; b += s_sw2[k]; }
            ws.tsum[tile] = a;
            ws.tsum2[tile] = b;
        }
        uint64_t prefix = 0;
        if (j == 0) {
            if (lane == 0) st_release(st, kFlagInc | agg);
        } else {
            if (lane == 0) st_release(st + j, kFlagAgg | agg);
            prefix = lookback(st, j, lane);
            if (lane == 0) st_release(st + j, kFlagInc | (prefix + agg));
        }
        if (lane < kThreads / 32) s_off[lane] = prefix + wi - wv;
        if (j == T - 1) {
            // last tile of the filter: every predecessor wrote its partial sums before its first
            // status release; an acquire load of each predecessor's (non-empty) status word
            // synchronises with that release directly, so the sums read after it are visible
            // (no reliance on transitive relaxed chains through the lookback).
            __syncwarp();  // this tile's own sums (lane 0's stores) for the lane that reads them
            double a = 0.0, b = 0.0;
            const int64_t t0 = static_cast<int64_t>(n) * T;
            for (int t = lane; t < T; t += 32) {
                if (t != j)
                    while ((ld_acquire(st + t) >> kFlagShift) == 0) {
                    }
                a += __ldcg(ws.tsum + t0 + t);
                b += __ldcg(ws.tsum2 + t0 + t);
            }
            a = warp_sum_f64(a);
            b = warp_sum_f64(b);
            if (lane == 0) {
                ws.Qtot[n] = prefix + agg;
                ws.S[n] = a;
                if (lse_out) lse_out[n] = static_cast<double>(lm) + log(a);
                if (ess_out) ess_out[n] = a * a / b;
            }
        }
    }
    if (!write_q) return;
    __syncthreads();
    const uint64_t off = s_off[warp];
    uint64_t* qrow = ws.Q + static_cast<int64_t>(n) * ldq;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int64_t i0 = base + r * 128 + lane * 4;
        uint64_t run = off + excl[r];
        uint64_t q4[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            run += quantise(w[r * 4 + c], kfx);
            q4[c] = run;
        }
        if (i0 + 3 < P) {
            ulonglong2* dst = reinterpret_cast<ulonglong2*>(qrow + i0);
            __stcg(dst, make_ulonglong2(q4[0], q4[1]));
            __stcg(dst + 1, make_ulonglong2(q4[2], q4[3]));
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (i0 + c < P) qrow[i0 + c] = q4[c];
        }
    }
}

// CTA-per-filter form of the scan for batches that fill the GPU (N >= SMs, P <= 2^17): a
// 512-thread CTA walks its filter in 4096-particle tiles with a running carry, so there is no
// decoupled lookback (whose latency bounds k_scan) and no tile-status traffic.  Same outputs as
// k_scan (Q, Qtot, S, lse, ESS; invalid filters: NaN side outputs).
constexpr int kScanCtaT = 512;
template <bool VEC>
__global__ void __launch_bounds__(kScanCtaT, 2) k_scan_cta(const float* __restrict__ logw, int64_t ld, int32_t N,
                                                           int32_t P, int kfx, Ws ws, int64_t ldq, int write_q,
                                                           double* lse_out, double* ess_out) {
    constexpr int W = kScanCtaT / 32;
    __shared__ uint64_t s_wt[W];
    __shared__ double s_a[W], s_b[W];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int n = blockIdx.x; n < N; n += gridDim.x) {
        if (ws.fstatus[n] != 0) {
            if (tid == 0) {
                if (lse_out) lse_out[n] = NAN;
                if (ess_out) ess_out[n] = NAN;
                ws.S[n] = NAN;
            }
            continue;
        }
        const float lm = ws.lmax[n];
        const float* row = logw + static_cast<int64_t>(n) * ld;
        uint64_t* qrow = ws.Q + static_cast<int64_t>(n) * ldq;
        uint64_t carry = 0;
        double sw = 0.0, sw2 = 0.0;
        for (int base = 0; base < P; base += 8 * kScanCtaT) {
            const int i0 = base + 8 * tid;
            float w[8];
            if (VEC && i0 + 7 < P) {
                const float4 t0 = __ldg(reinterpret_cast<const float4*>(row + i0));
                const float4 t1 = __ldg(reinterpret_cast<const float4*>(row + i0 + 4));
                w[0] = t0.x; w[1] = t0.y; w[2] = t0.z; w[3] = t0.w; w[4] = t1.x; w[5] = t1.y; w[6] = t1.z; w[7] = t1.w;
            } else {
#pragma unroll
                for (int c = 0; c < 8; ++c) w[c] = (i0 + c < P) ? row[i0 + c] : -INFINITY;
            }
            uint64_t loc = 0;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                w[c] = weight(w[c], lm);
                sw += static_cast<double>(w[c]);
                sw2 += static_cast<double>(w[c]) * static_cast<double>(w[c]);
                loc += quantise(w[c], kfx);
            }
            const uint64_t incl = warp_incl_scan_u64(loc, lane);
            if (lane == 31) s_wt[warp] = incl;
            __syncthreads();
            uint64_t wpre = 0, tot = 0;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                const uint64_t t = s_wt[k];
                wpre += (k < warp) ? t : 0ull;
                tot += t;
            }
            __syncthreads();  // s_wt is rewritten by the next tile
            if (write_q) {
                uint64_t run = carry + wpre + incl - loc;
                uint64_t q8[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    run += quantise(w[c], kfx);
                    q8[c] = run;
                }
                if (i0 + 7 < P) {
                    ulonglong2* dst = reinterpret_cast<ulonglong2*>(qrow + i0);
#pragma unroll
                    for (int c = 0; c < 4; ++c) __stcg(dst + c, make_ulonglong2(q8[2 * c], q8[2 * c + 1]));
                } else {
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        if (i0 + c < P) qrow[i0 + c] = q8[c];
                }
            }
            carry += tot;
        }
        sw = warp_sum_f64(sw);
        sw2 = warp_sum_f64(sw2);
        if (lane == 0) { s_a[warp] = sw; s_b[warp] = sw2; }
        __syncthreads();
        if (tid == 0) {
            double a = 0.0, b = 0.0;
            for (int k = 0; k < W; ++k) { a += s_a[k]; b += s_b[k]; }
            ws.Qtot[n] = carry;
            ws.S[n] = a;
            if (lse_out) lse_out[n] = static_cast<double>(lm) + log(a);
            if (ess_out) ess_out[n] = a * a / b;
        }
        __syncthreads();  // s_a / s_b reuse
    }
}

// ============================================================================ a4+a5: merge path
// Merged sequence of A (positions x_k, sorted) and B (cumulative Q_i, sorted);
// B_i precedes A_k iff Q_i <= x_k, so when x_k is emitted the number of B
// consumed is #{i : Q_i <= x_k} = min{i : Q_i > x_k} = a_k (G6).
struct SortedCtx {
    int n;
    uint64_t Qtot, D, rho;
    uint32_t filt;
    const uint64_t* Q;
};

template <int SCHEME>  // PF_STRATIFIED = 2, PF_SYSTEMATIC = 3
struct ModeSorted {
    const uint64_t* Q;
    int64_t ldq;
    const uint64_t* Qtot;
    const int32_t* fstatus;
    uint64_t D;
    Key key;
    uint32_t filt0;
    int32_t P;
    int32_t* anc;
    int64_t ld_anc;

    using Ctx = SortedCtx;
    __device__ Ctx ctx(int n) const {
        Ctx c;
        c.n = n;
        c.Qtot = Qtot[n];
        c.D = D;
        c.filt = filt0 + static_cast<uint32_t>(n);
        c.Q = Q + static_cast<int64_t>(n) * ldq;
        c.rho = 0;
        if (SCHEME == 3) c.rho = mulhi64(lo_word(philox10(0u, 0u, 3u, c.filt, key.k0, key.k1)), D);
        return c;
    }
    __device__ bool valid(int n) const { return fstatus[n] == 0; }
    __device__ int64_t nA(const Ctx&) const { return P; }
    __device__ uint64_t x(const Ctx& c, int64_t k) const {
        uint64_t rho = c.rho;
        if (SCHEME == 2) {
            const u32x4 r = philox10(static_cast<uint32_t>(k >> 1), 0u, 2u, c.filt, key.k0, key.k1);
            rho = mulhi64((k & 1) ? hi_word(r) : lo_word(r), c.D);
        }
        return mulhi64(static_cast<uint64_t>(k) * c.D + rho, c.Qtot);
    }
    __device__ uint64_t b(const Ctx& c, int64_t i) const { return __ldg(c.Q + i); }
    __device__ void fill_a(const Ctx& c, int64_t ka0, int na, uint64_t* s) const {
        if (SCHEME == 2) {
            const int64_t k_even = ka0 & ~int64_t{1};
            const int npairs = static_cast<int>((ka0 + na - k_even + 1) >> 1);
            for (int p = threadIdx.x; p < npairs; p += kThreads) {
                const int64_t k = k_even + 2 * p;
                const u32x4 r = philox10(static_cast<uint32_t>(k >> 1), 0u, 2u, c.filt, key.k0, key.k1);
                if (k >= ka0)
                    s[k - ka0] = mulhi64(static_cast<uint64_t>(k) * c.D + mulhi64(lo_word(r), c.D), c.Qtot);
                if (k + 1 < ka0 + na)
                    s[k + 1 - ka0] = mulhi64(static_cast<uint64_t>(k + 1) * c.D + mulhi64(hi_word(r), c.D), c.Qtot);
            }
        } else {
            for (int t = threadIdx.x; t < na; t += kThreads) s[t] = x(c, ka0 + t);
        }
    }
    __device__ void emit(const Ctx& c, int64_t ka0, int na, const int32_t* s_out) const {
        int32_t* dst = anc + static_cast<int64_t>(c.n) * ld_anc + ka0;
        for (int t = threadIdx.x; t < na; t += kThreads) dst[t] = s_out[t];
    }
    __device__ void identity(int n, int c, int cpf) const {
        const int64_t per = cdiv(P, cpf);
        const int64_t b0 = c * per, b1 = min(static_cast<int64_t>(P), b0 + per);
        int32_t* dst = anc + static_cast<int64_t>(n) * ld_anc;
        for (int64_t k = b0 + threadIdx.x; k < b1; k += kThreads) dst[k] = static_cast<int32_t>(k);
    }
};

template <class Mode>
__device__ __forceinline__ int64_t merge_split(const Mode& md, const typename Mode::Ctx& c, int64_t d, int64_t nA,
                                               int64_t nB, int lane) {
    int64_t lo = max(int64_t{0}, d - nB), hi = min(d, nA);
    while (hi > lo) {
        const int64_t step = (hi - lo + 31) / 32;
        const int64_t m = lo + lane * step;
        bool p = false;
        if (m < hi) p = md.x(c, m) < md.b(c, d - 1 - m);
        const int L = __popc(__ballot_sync(kFull, p));
        const int64_t nlo = (L == 0) ? lo : lo + static_cast<int64_t>(L - 1) * step + 1;
        const int64_t mL = lo + static_cast<int64_t>(L) * step;
        hi = (mL < hi) ? mL : hi;
        lo = nlo;
    }
    return lo;
}

// Sliding-window merge: CTA cb owns the merged diagonals [cb*chunk, +chunk).
// One warp-parallel global search finds the start split; afterwards every
// window of kWin merged items starts where the previous one ended, so the
// window only needs the next kWin items of each list (smem) and a per-thread
// diagonal search in shared memory.
constexpr int kWin = 2048;
constexpr int kWinItems = kWin / kThreads;  // 8 merged items per thread

template <class Mode>
__global__ void __launch_bounds__(kThreads) k_merge(Mode md, int cpf, int64_t chunk) {
    __shared__ uint64_t sA[kWin];
    __shared__ uint64_t sB[kWin];
    __shared__ int32_t s_out[kWin];
    __shared__ int64_t s_split[2];
    const int n = blockIdx.x / cpf;
    const int cb = blockIdx.x - n * cpf;
    if (!md.valid(n)) {
        md.identity(n, cb, cpf);
        return;
    }
    const typename Mode::Ctx c = md.ctx(n);
    const int64_t nA = md.nA(c), nB = md.P;
    const int64_t total = nA + nB;
    const int64_t d0 = static_cast<int64_t>(cb) * chunk;
    if (d0 >= total) return;
    const int64_t d1 = min(d0 + chunk, total);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) {
        const int64_t ka = merge_split(md, c, d0, nA, nB, lane);
        if (lane == 0) { s_split[0] = ka; s_split[1] = d0 - ka; }
    }
    __syncthreads();
    int64_t ka = s_split[0], ib = s_split[1];
    for (int64_t d = d0; d < d1; d += kWin) {
        const int wlen = static_cast<int>(min(static_cast<int64_t>(kWin), d1 - d));
        const int na = static_cast<int>(min(static_cast<int64_t>(wlen), nA - ka));
        const int nb = static_cast<int>(min(static_cast<int64_t>(wlen), nB - ib));
        md.fill_a(c, ka, na, sA);
        for (int t = tid; t < nb; t += kThreads) sB[t] = md.b(c, ib + t);
        __syncthreads();
        const int dd = tid * kWinItems;
        if (dd < wlen) {
            int lo = max(0, dd - nb), hi = min(dd, na);
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (sA[mid] < sB[dd - 1 - mid]) lo = mid + 1;
                else hi = mid;
            }
            int a = lo, b = dd - lo;
            const int end = min(dd + kWinItems, wlen);
            uint64_t xa = (a < na) ? sA[a] : 0ull;
            uint64_t xb = (b < nb) ? sB[b] : 0ull;
            const int32_t ibase = static_cast<int32_t>(ib);
#pragma unroll
            for (int it = 0; it < kWinItems; ++it) {
                if (dd + it < end) {
                    const bool take_b = (b < nb) && (a >= na || xb <= xa);
                    if (take_b) {
                        ++b;
                        xb = (b < nb) ? sB[b] : 0ull;
                    } else {
                        s_out[a] = ibase + b;
                        ++a;
                        xa = (a < na) ? sA[a] : 0ull;
                    }
                }
            }
            if (end == wlen && dd + kWinItems >= wlen) { s_split[0] = a; s_split[1] = b; }
        }
        __syncthreads();
        const int a_end = static_cast<int>(s_split[0]);
        const int b_end = static_cast<int>(s_split[1]);
        md.emit(c, ka, a_end, s_out);
        ka += a_end;
        ib += b_end;
        __syncthreads();
    }
}

// ============================================================================ a6: spacings
// Inclusive scan of the exponential spacings e_0..e_P (NS-12) of each filter,
// same tile / lookback structure as k_scan; the values come from Philox
// (tag 5, one call per 4 consecutive k) and the deterministic double log.
__global__ void __launch_bounds__(kThreads, 4) k_gscan(int32_t P, int T2, Ws ws, int64_t ldg, Key key,
                                                       uint32_t filt0) {
    __shared__ uint32_t s_tile;
    __shared__ uint64_t s_wtot[kThreads / 32];
    __shared__ uint64_t s_off[kThreads / 32];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) s_tile = atomicAdd(ws.tile_ctr2, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int n = static_cast<int>(tile / T2);
    const int j = static_cast<int>(tile - static_cast<int64_t>(n) * T2);
    const int64_t base = static_cast<int64_t>(j) * kTile + warp * 512;
    const uint32_t filt = filt0 + static_cast<uint32_t>(n);
    uint64_t v[16];
    uint64_t excl[4];
    uint64_t carry = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int64_t i0 = base + r * 128 + lane * 4;
        uint64_t loc = 0;
        if (i0 <= P) {
            const u32x4 x = philox10(static_cast<uint32_t>(i0 >> 2), 0u, 5u, filt, key.k0, key.k1);
            const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                v[r * 4 + c] = (i0 + c <= P) ? spacing_from_word(w4[c]) : 0ull;
                loc += v[r * 4 + c];
            }
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) v[r * 4 + c] = 0ull;
        }
        const uint64_t incl = warp_incl_scan_u64(loc, lane);
        excl[r] = incl - loc + carry;
        carry += __shfl_sync(kFull, incl, 31);
    }
    if (lane == 0) s_wtot[warp] = carry;
    __syncthreads();
    if (warp == 0) {
        const uint64_t wv = (lane < kThreads / 32) ? s_wtot[lane] : 0ull;
        const uint64_t wi = warp_incl_scan_u64(wv, lane);
        const uint64_t agg = __shfl_sync(kFull, wi, kThreads / 32 - 1);
        uint64_t* st = ws.tstatus2 + static_cast<int64_t>(n) * T2;
        uint64_t prefix = 0;
        if (j == 0) {
            if (lane == 0) st_release(st, kFlagInc | agg);
        } else {
            if (lane == 0) st_release(st + j, kFlagAgg | agg);
            prefix = lookback(st, j, lane);
            if (lane == 0) st_release(st + j, kFlagInc | (prefix + agg));
        }
        if (lane < kThreads / 32) s_off[lane] = prefix + wi - wv;
    }
    __syncthreads();
    const uint64_t off = s_off[warp];
    uint64_t* grow = ws.G + static_cast<int64_t>(n) * ldg;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int64_t i0 = base + r * 128 + lane * 4;
        uint64_t run = off + excl[r];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            run += v[r * 4 + c];
            if (i0 + c <= P) grow[i0 + c] = run;
            if (i0 + c == P) ws.Gtot[n] = run;
        }
    }
}

struct SpacCtx {
    int n;
    uint64_t Qtot, GP;
    const uint64_t* Q;
    const uint64_t* G;
    double ratio, inv_d;  // Q / G_P and 1 / G_P (estimates only; the division is exact)
};

// a6 merge: slot k's position is x_k = floor(G_k Q / G_P) (exact 128/64 division);
// a_k = min{i : Q_i > x_k} as for the other sorted schemes.
struct ModeSpacings {
    const uint64_t* Q;
    int64_t ldq;
    const uint64_t* Qtot;
    const int32_t* fstatus;
    const uint64_t* G;
    int64_t ldg;
    const uint64_t* Gtot;
    int32_t P;
    int32_t* anc;
    int64_t ld_anc;

    using Ctx = SpacCtx;
    __device__ Ctx ctx(int n) const {
        const uint64_t qt = Qtot[n], gp = Gtot[n];
        return {n, qt, gp, Q + static_cast<int64_t>(n) * ldq, G + static_cast<int64_t>(n) * ldg,
                __ddiv_rn(static_cast<double>(qt), static_cast<double>(gp)), __drcp_rn(static_cast<double>(gp))};
    }
    __device__ bool valid(int n) const { return fstatus[n] == 0; }
    __device__ int64_t nA(const Ctx&) const { return P; }
    __device__ uint64_t x(const Ctx& c, int64_t k) const {
        return muldiv_floor_pre(__ldg(c.G + k), c.Qtot, c.GP, c.ratio, c.inv_d);
    }
    __device__ uint64_t b(const Ctx& c, int64_t i) const { return __ldg(c.Q + i); }
    __device__ void fill_a(const Ctx& c, int64_t ka0, int na, uint64_t* s) const {
        for (int t = threadIdx.x; t < na; t += kThreads) s[t] = x(c, ka0 + t);
    }
    __device__ void emit(const Ctx& c, int64_t ka0, int na, const int32_t* s_out) const {
        int32_t* dst = anc + static_cast<int64_t>(c.n) * ld_anc + ka0;
        for (int t = threadIdx.x; t < na; t += kThreads) dst[t] = s_out[t];
    }
    __device__ void identity(int n, int cb, int cpf) const {
        const int64_t per = cdiv(P, cpf);
        const int64_t b0 = cb * per, b1 = min(static_cast<int64_t>(P), b0 + per);
        int32_t* dst = anc + static_cast<int64_t>(n) * ld_anc;
        for (int64_t k = b0 + threadIdx.x; k < b1; k += kThreads) dst[k] = static_cast<int32_t>(k);
    }
};

// ============================================================================ a4+a5: multinomial (bucketed)
// Bucket index of the multinomial search: NB = 2^ceil(log2 P) equal buckets of
// the 64-bit uniform R; bucket b covers positions [floor(b Q / NB), floor((b+1) Q / NB)]
// (x = mulhi64(R, Q) is monotone in R), so idx[b] = min{i : Q_i > floor(b Q / NB)}
// bounds the ancestor of every slot whose R falls in bucket b:
// idx[b] <= a_k <= idx[b+1].  The index is the merge of those NB sorted values
// with Q (k_merge<ModeBuckets>).
struct BucketCtx {
    int n;
    uint64_t Qtot;
    const uint64_t* Q;
};

struct ModeBuckets {
    const uint64_t* Q;
    int64_t ldq;
    const uint64_t* Qtot;
    const int32_t* fstatus;
    int lgNB;
    int32_t NB;
    int32_t P;  // particles (the B list)
    int32_t* idx;
    int64_t ldb;

    using Ctx = BucketCtx;
    __device__ Ctx ctx(int n) const { return {n, Qtot[n], Q + static_cast<int64_t>(n) * ldq}; }
    __device__ bool valid(int n) const { return fstatus[n] == 0; }
    __device__ int64_t nA(const Ctx&) const { return NB; }
    __device__ uint64_t x(const Ctx& c, int64_t b) const {
        return lgNB == 0 ? 0ull : mulhi64(static_cast<uint64_t>(b) << (64 - lgNB), c.Qtot);
    }
    __device__ uint64_t b(const Ctx& c, int64_t i) const { return __ldg(c.Q + i); }
    __device__ void fill_a(const Ctx& c, int64_t ka0, int na, uint64_t* s) const {
        for (int t = threadIdx.x; t < na; t += kThreads) s[t] = x(c, ka0 + t);
    }
    __device__ void emit(const Ctx& c, int64_t ka0, int na, const int32_t* s_out) const {
        int32_t* dst = idx + static_cast<int64_t>(c.n) * ldb + ka0;
        for (int t = threadIdx.x; t < na; t += kThreads) dst[t] = s_out[t];
    }
    __device__ void identity(int, int, int) const {}
};

// per slot: bucket from the top bits of R_k, then a binary search in the
// (usually 1-3 particle) range [idx[b], idx[b+1]]; 8 slots per thread.
__global__ void __launch_bounds__(kThreads) k_bsearch_buckets(int32_t N, int32_t P, Ws ws, int64_t ldq, int64_t ldb,
                                                              int lgNB, Key key, uint32_t filt0, int32_t* anc,
                                                              int64_t ld_anc) {
    const int64_t per_row = cdiv(P, 8);
    const int64_t total = static_cast<int64_t>(N) * per_row;
    for (int64_t g = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; g < total;
         g += static_cast<int64_t>(gridDim.x) * kThreads) {
        const int64_t n = g / per_row;
        const int64_t kb = (g - n * per_row) * 8;
        int32_t* arow = anc + n * ld_anc;
        if (ws.fstatus[n] != 0) {
            for (int t = 0; t < 8; ++t)
                if (kb + t < P) arow[kb + t] = static_cast<int32_t>(kb + t);
            continue;
        }
        const uint64_t* Q = ws.Q + n * ldq;
        const int32_t* bi = ws.bidx + n * ldb;
        const uint64_t Qtot = ws.Qtot[n];
        const uint32_t filt = filt0 + static_cast<uint32_t>(n);
        uint64_t pos[8];
        int32_t lo[8], hi[8];
#pragma unroll
        for (int t = 0; t < 8; t += 2) {
            const u32x4 r = philox10(static_cast<uint32_t>((kb + t) >> 1), 0u, 1u, filt, key.k0, key.k1);
            const uint64_t R0 = lo_word(r), R1 = hi_word(r);
            pos[t] = mulhi64(R0, Qtot);
            pos[t + 1] = mulhi64(R1, Qtot);
            const int64_t b0 = lgNB ? static_cast<int64_t>(R0 >> (64 - lgNB)) : 0;
            const int64_t b1 = lgNB ? static_cast<int64_t>(R1 >> (64 - lgNB)) : 0;
            lo[t] = __ldg(bi + b0);
            hi[t] = (b0 + 1 < (int64_t{1} << lgNB)) ? min(__ldg(bi + b0 + 1), P - 1) : P - 1;
            lo[t + 1] = __ldg(bi + b1);
            hi[t + 1] = (b1 + 1 < (int64_t{1} << lgNB)) ? min(__ldg(bi + b1 + 1), P - 1) : P - 1;
        }
        bool more = true;
        while (more) {
            more = false;
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                if (lo[t] < hi[t]) {
                    const int32_t mid = (lo[t] + hi[t]) >> 1;
                    if (__ldg(Q + mid) > pos[t]) hi[t] = mid;
                    else lo[t] = mid + 1;
                    more |= lo[t] < hi[t];
                }
            }
        }
        if (kb + 8 <= P && ((reinterpret_cast<uintptr_t>(arow + kb) & 15) == 0)) {
            int4* dst = reinterpret_cast<int4*>(arow + kb);
            dst[0] = make_int4(lo[0], lo[1], lo[2], lo[3]);
            dst[1] = make_int4(lo[4], lo[5], lo[6], lo[7]);
        } else {
#pragma unroll
            for (int t = 0; t < 8; ++t)
                if (kb + t < P) arow[kb + t] = lo[t];
        }
    }
}

// ============================================================================ a7: Metropolis
__global__ void __launch_bounds__(kThreads) k_mexp(const float* __restrict__ logw, int64_t ld, int32_t N,
                                                   int32_t P, Ws ws, int64_t ldq) {
    const int64_t total = static_cast<int64_t>(N) * P;
    for (int64_t g = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; g < total;
         g += static_cast<int64_t>(gridDim.x) * kThreads) {
        const int64_t n = g / P, i = g - n * P;
        ws.w[n * ldq + i] = weight(__ldcs(logw + n * ld + i), ws.lmax[n]);
    }
}

__global__ void __launch_bounds__(kThreads) k_mexp_vec(const float4* __restrict__ logw, int64_t ld4, int32_t N,
                                                       int32_t P4, Ws ws, int64_t ldq4) {
    const int64_t total = static_cast<int64_t>(N) * P4;
    float4* w4 = reinterpret_cast<float4*>(ws.w);
    for (int64_t g = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; g < total;
         g += static_cast<int64_t>(gridDim.x) * kThreads) {
        const int64_t n = g / P4, i = g - n * P4;
        const float lm = ws.lmax[n];
        const float4 v = __ldcs(logw + n * ld4 + i);
        w4[n * ldq4 + i] = make_float4(weight(v.x, lm), weight(v.y, lm), weight(v.z, lm), weight(v.w, lm));
    }
}

// NS-11's proposal j = (r P) >> 32 is r >> (32 - m) when P = 2^m (m >= 1): the same value
// without a multiply on the integer-multiply pipe that the Philox rounds saturate (the binding
// pipe of these kernels, profiles/r02_ncu_metro.md).  PSH = the shift, or 0: general P.
template <bool POW2>
__device__ __forceinline__ uint32_t metro_j(uint32_t r, uint32_t P, int sh) {
    return POW2 ? (r >> sh) : __umulhi(r, P);
}

template <bool POW2>
__global__ void __launch_bounds__(kThreads) k_metro(int32_t N, int32_t P, Ws ws, int64_t ldq, Key key,
                                                    uint32_t filt0, int32_t B, int32_t* anc, int64_t ld_anc,
                                                    int sh) {
    const int64_t g = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x;
    if (g >= static_cast<int64_t>(N) * P) return;
    const int n = static_cast<int>(g / P);
    const int32_t i = static_cast<int32_t>(g - static_cast<int64_t>(n) * P);
    int32_t* out = anc + static_cast<int64_t>(n) * ld_anc + i;
    if (B == 0 || ws.fstatus[n] != 0) {
        *out = i;
        return;
    }
    const float* w = ws.w + static_cast<int64_t>(n) * ldq;
    const uint32_t filt = filt0 + static_cast<uint32_t>(n);
    int32_t k = i;
    float wk = __ldg(w + i);
    const float kU = __uint_as_float(0x33800000u);  // 2^-24
    for (int32_t b = 0; b < B; b += 8) {
        uint32_t j[8];
        float u[8], wj[8];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const u32x4 r = philox10(static_cast<uint32_t>(i), static_cast<uint32_t>((b >> 1) + t), 4u, filt,
                                     key.k0, key.k1);
            j[2 * t] = metro_j<POW2>(r.x, static_cast<uint32_t>(P), sh);
            u[2 * t] = __fmul_rn(static_cast<float>(r.y >> 8), kU);
            j[2 * t + 1] = metro_j<POW2>(r.z, static_cast<uint32_t>(P), sh);
            u[2 * t + 1] = __fmul_rn(static_cast<float>(r.w >> 8), kU);
        }
#pragma unroll
        for (int s = 0; s < 8; ++s) wj[s] = (b + s < B) ? __ldg(w + j[s]) : 0.0f;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            if (b + s < B && __fmul_rn(u[s], wk) < wj[s]) {
                k = static_cast<int32_t>(j[s]);
                wk = wj[s];
            }
        }
    }
    *out = k;
}

// Filter-per-CTA form: one 1024-thread CTA per SM walks whole filters, so an SM's L1 holds (most
// of) one filter's weight vector and the B random proposals per chain hit L1 instead of L2
// (the kernel is launched with the maximum L1 carve-out).  Same chains, same results as k_metro.
template <bool POW2>
__global__ void __launch_bounds__(1024, 1) k_metro_fpc(int32_t N, int32_t P, Ws ws, int64_t ldq, Key key,
                                                        uint32_t filt0, int32_t B, int32_t* anc, int64_t ld_anc,
                                                        int sh) {
    const float kU = __uint_as_float(0x33800000u);  // 2^-24
    for (int n = blockIdx.x; n < N; n += gridDim.x) {
        int32_t* out = anc + static_cast<int64_t>(n) * ld_anc;
        if (B == 0 || ws.fstatus[n] != 0) {
            for (int32_t i = threadIdx.x; i < P; i += blockDim.x) out[i] = i;
            continue;
        }
        const float* w = ws.w + static_cast<int64_t>(n) * ldq;
        const uint32_t filt = filt0 + static_cast<uint32_t>(n);
        for (int32_t i = threadIdx.x; i < P; i += blockDim.x) {
            int32_t k = i;
            float wk = __ldg(w + i);
            for (int32_t b = 0; b < B; b += 8) {
                uint32_t j[8];
                float u[8], wj[8];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const u32x4 r = philox10(static_cast<uint32_t>(i), static_cast<uint32_t>((b >> 1) + t), 4u, filt,
                                             key.k0, key.k1);
                    j[2 * t] = metro_j<POW2>(r.x, static_cast<uint32_t>(P), sh);
                    u[2 * t] = __fmul_rn(static_cast<float>(r.y >> 8), kU);
                    j[2 * t + 1] = metro_j<POW2>(r.z, static_cast<uint32_t>(P), sh);
                    u[2 * t + 1] = __fmul_rn(static_cast<float>(r.w >> 8), kU);
                }
#pragma unroll
                for (int t = 0; t < 8; ++t) wj[t] = (b + t < B) ? __ldg(w + j[t]) : 0.0f;
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    if (b + t < B && __fmul_rn(u[t], wk) < wj[t]) {
                        k = static_cast<int32_t>(j[t]);
                        wk = wj[t];
                    }
                }
            }
            out[i] = k;
        }
    }
}

// ============================================================================ a12: normalised weights
__global__ void __launch_bounds__(kThreads) k_normw(const float* __restrict__ logw, int64_t ld, int32_t N,
                                                    int32_t P, Ws ws, float* normw) {
    const int64_t total = static_cast<int64_t>(N) * P;
    for (int64_t g = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; g < total;
         g += static_cast<int64_t>(gridDim.x) * kThreads) {
        const int64_t n = g / P, i = g - n * P;
        float v = NAN;
        if (ws.fstatus[n] == 0)
            v = static_cast<float>(static_cast<double>(weight(logw[n * ld + i], ws.lmax[n])) / ws.S[n]);
        normw[g] = v;
    }
}

__global__ void __launch_bounds__(kThreads) k_identity(int32_t N, int32_t P, int32_t* anc, int64_t ld_anc) {
    const int64_t total = static_cast<int64_t>(N) * P;
    for (int64_t g = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; g < total;
         g += static_cast<int64_t>(gridDim.x) * kThreads) {
        const int64_t n = g / P, i = g - n * P;
        anc[n * ld_anc + i] = static_cast<int32_t>(i);
    }
}

// ============================================================================ a8: offspring
__global__ void __launch_bounds__(kThreads) k_hist(const int32_t* __restrict__ anc, int64_t ld_anc, int32_t N,
                                                   int32_t P, int32_t* o, int64_t ld_o) {
    const int64_t total = static_cast<int64_t>(N) * P;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
    const int64_t g0 = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x;
    const int64_t rounds = cdiv(total, stride);
    for (int64_t r = 0; r < rounds; ++r) {  // warp-uniform trip count for __match_any_sync
        const int64_t g = g0 + r * stride;
        int32_t* addr = nullptr;
        if (g < total) {
            const int64_t n = g / P, k = g - n * P;
            const int32_t a = __ldcs(anc + n * ld_anc + k);
            if (a >= 0 && a < P) addr = o + n * ld_o + a;
        }
        const unsigned peers = __match_any_sync(kFull, reinterpret_cast<unsigned long long>(addr));
        if (addr && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(addr, __popc(peers));
    }
}

// Offspring histogram over one filter row with P % 4 == 0 and 16-byte aligned
// rows: each warp takes 128 consecutive ancestors (one int4 per lane) and
// issues one reduction per run of equal values (a run head adds the distance
// to the next head), so sorted ancestors (stratified / systematic) cost one
// atomic per surviving particle and unsorted ones one per slot.
// Shared-memory histogram for batches of filters with P <= 65536: two CTAs per filter, each
// counting the ancestors that fall in its half of the particle range (<= 32768 u32 counters,
// 128 KB), reading the filter's ancestors once each (the second read is L2-resident); no global
// atomics, no memset, and the counts are written with coalesced stores.
constexpr int kHistT = 1024;
__global__ void __launch_bounds__(kHistT) k_hist_smem(const int32_t* __restrict__ anc, int64_t ld_anc, int32_t N,
                                                       int32_t P, int32_t* o, int64_t ld_o, int vec) {
    extern __shared__ uint32_t s_cnt[];
    const int half = (P + 1) / 2;
    for (int64_t job = blockIdx.x; job < 2LL * N; job += gridDim.x) {
        const int64_t n = job >> 1;
        const int lo = (job & 1) ? half : 0;
        const int hi = (job & 1) ? P : half;
        for (int i = threadIdx.x; i < hi - lo; i += kHistT) s_cnt[i] = 0u;
        __syncthreads();
        const int32_t* arow = anc + n * ld_anc;
        if (vec) {
            const int4* a4 = reinterpret_cast<const int4*>(arow);
            for (int k = threadIdx.x; k < P / 4; k += kHistT) {
                const int4 v = __ldg(a4 + k);
                const int32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (vv[c] >= lo && vv[c] < hi) atomicAdd(&s_cnt[vv[c] - lo], 1u);
            }
            for (int k = (P / 4) * 4 + threadIdx.x; k < P; k += kHistT) {
                const int32_t v = __ldg(arow + k);
                if (v >= lo && v < hi) atomicAdd(&s_cnt[v - lo], 1u);
            }
        } else {
            for (int k = threadIdx.x; k < P; k += kHistT) {
                const int32_t v = __ldg(arow + k);
                if (v >= lo && v < hi) atomicAdd(&s_cnt[v - lo], 1u);
            }
        }
        __syncthreads();
        int32_t* orow = o + n * ld_o;
        for (int i = threadIdx.x; i < hi - lo; i += kHistT) orow[lo + i] = static_cast<int32_t>(s_cnt[i]);
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kThreads) k_hist_runs(const int32_t* __restrict__ anc, int64_t ld_anc,
                                                        int32_t N, int32_t P, int32_t* o, int64_t ld_o) {
    const int lane = threadIdx.x & 31;
    const int64_t per_row = P / 128 + ((P % 128) ? 1 : 0);  // warp-blocks per filter
    const int64_t nblk = static_cast<int64_t>(N) * per_row;
    const int64_t wstride = static_cast<int64_t>(gridDim.x) * (kThreads / 32);
    for (int64_t blk = blockIdx.x * static_cast<int64_t>(kThreads / 32) + (threadIdx.x >> 5); blk < nblk;
         blk += wstride) {
        const int64_t n = blk / per_row;
        const int64_t k0 = (blk - n * per_row) * 128 + lane * 4;
        int32_t v[4] = {-1, -1, -1, -1};
        if (k0 < P) {  // P % 4 == 0: a lane's 4 items are all valid or all beyond P
            const int4 t = __ldcs(reinterpret_cast<const int4*>(anc + n * ld_anc + k0));
            v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
        }
        const int32_t prev = __shfl_up_sync(kFull, v[3], 1);
        // head bits of this lane's 4 items
        unsigned h = 0;
        h |= (lane == 0 || v[0] != prev) ? 1u : 0u;
        h |= (v[1] != v[0]) ? 2u : 0u;
        h |= (v[2] != v[1]) ? 4u : 0u;
        h |= (v[3] != v[2]) ? 8u : 0u;
        // position of the first head in later lanes (suffix min over lanes > lane)
        int first = h ? (lane * 4 + __ffs(h) - 1) : 128;
        int nxt = 128;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int t = __shfl_down_sync(kFull, first, off);
            if (lane + off < 32) first = min(first, t);
        }
        // first now = min over lanes >= lane; shift by one lane for "strictly later"
        nxt = __shfl_down_sync(kFull, first, 1);
        if (lane == 31) nxt = 128;
        int32_t* row = o + n * ld_o;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (!(h & (1u << c)) || v[c] < 0 || v[c] >= P) continue;
            // run end: next head inside this lane, else the first head of a later lane
            int end = nxt;
#pragma unroll
            for (int d = 3; d > c; --d)
                if (h & (1u << d)) end = lane * 4 + d;
            int len = end - (lane * 4 + c);
            // the window may end before P: clip to valid items
            const int64_t lim = P - (k0 - lane * 4);
            if (end > lim) len = static_cast<int>(lim) - (lane * 4 + c);
            atomicAdd(row + v[c], len);
        }
    }
}

// ============================================================================ a9: permutation scan
// Packed pair per particle: bits [0,31) free flag (o_i == 0), bits [31,62)
// extras e_i = max(o_i - 1, 0).  Exclusive free rank and inclusive extras
// offsets come out of one u64 lookback scan (both halves < 2^31, no carry).
__global__ void __launch_bounds__(kThreads, 5) k_pscan(int32_t P, int T, Ws ws, int64_t ldq, const int32_t* o_in,
                                                       int64_t ld_o, int o_vec, int32_t* perm, int64_t ld_perm) {
    __shared__ uint32_t s_tile;
    __shared__ uint64_t s_wtot[kThreads / 32];
    __shared__ uint64_t s_off[kThreads / 32];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) s_tile = atomicAdd(ws.tile_ctr, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int n = static_cast<int>(tile / T);
    const int j = static_cast<int>(tile - static_cast<int64_t>(n) * T);
    const int64_t base = static_cast<int64_t>(j) * kTile + warp * 512;
    const int32_t* orow = o_in + static_cast<int64_t>(n) * ld_o;
    int32_t ov[16];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int64_t i0 = base + r * 128 + lane * 4;
        if (o_vec && i0 + 3 < P) {
            const int4 t = __ldcg(reinterpret_cast<const int4*>(orow + i0));
            ov[r * 4 + 0] = t.x; ov[r * 4 + 1] = t.y; ov[r * 4 + 2] = t.z; ov[r * 4 + 3] = t.w;
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) ov[r * 4 + c] = (i0 + c < P) ? __ldcg(orow + i0 + c) : 1;
        }
    }
    auto packed = [](int32_t o) -> uint64_t {
        const uint64_t e = (o > 1) ? static_cast<uint64_t>(o - 1) : 0ull;
        return (e << 31) | (o == 0 ? 1ull : 0ull);
    };
    uint64_t excl[4];
    uint64_t carry = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        uint64_t loc = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) loc += packed(ov[r * 4 + c]);
        const uint64_t incl = warp_incl_scan_u64(loc, lane);
        excl[r] = incl - loc + carry;
        carry += __shfl_sync(kFull, incl, 31);
    }
    if (lane == 0) s_wtot[warp] = carry;
    __syncthreads();
    if (warp == 0) {
        const uint64_t wv = (lane < kThreads / 32) ? s_wtot[lane] : 0ull;
        const uint64_t wi = warp_incl_scan_u64(wv, lane);
        const uint64_t agg = __shfl_sync(kFull, wi, kThreads / 32 - 1);
        uint64_t* st = ws.tstatus + static_cast<int64_t>(n) * T;
        uint64_t prefix = 0;
        if (j == 0) {
            if (lane == 0) st_release(st, kFlagInc | agg);
        } else {
            if (lane == 0) st_release(st + j, kFlagAgg | agg);
            prefix = lookback(st, j, lane);
            if (lane == 0) st_release(st + j, kFlagInc | (prefix + agg));
        }
        if (lane < kThreads / 32) s_off[lane] = prefix + wi - wv;
        if (j == T - 1 && lane == 0) ws.F[n] = static_cast<int32_t>((prefix + agg) & 0x7FFFFFFFull);
    }
    __syncthreads();
    const uint64_t off = s_off[warp];
    uint32_t* qe = ws.Qe + static_cast<int64_t>(n) * ldq;
    int32_t* fs = ws.freeslot + static_cast<int64_t>(n) * ldq;
    int32_t* pr = perm + static_cast<int64_t>(n) * ld_perm;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int64_t i0 = base + r * 128 + lane * 4;
        uint64_t run = off + excl[r];
        uint32_t e4[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int64_t i = i0 + c;
            run += packed(ov[r * 4 + c]);
            e4[c] = static_cast<uint32_t>(run >> 31);
            if (i < P) {
                if (ov[r * 4 + c] > 0) {
                    pr[i] = static_cast<int32_t>(i);
                } else {
                    const uint64_t rank_excl = (run & 0x7FFFFFFFull) - 1;  // this item is free: its own flag is 1
                    fs[rank_excl] = static_cast<int32_t>(i);
                }
            }
        }
        if (i0 + 3 < P) {
            __stcg(reinterpret_cast<uint4*>(qe + i0), make_uint4(e4[0], e4[1], e4[2], e4[3]));
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (i0 + c < P) qe[i0 + c] = e4[c];
        }
    }
}

// ============================================================================ a9: push
// Completes the canonical permutation: the extras of a block of 128
// consecutive particles occupy the contiguous free ranks [R0, R0 + S)
// (R0 = exclusive extras prefix of the block's first particle).  Each warp
// expands its block's extras list in 256-rank chunks with a head-mark +
// max-scan in shared memory (owner of rank r = max{j : off_j <= r}) and writes
// perm[freeslot[R0 + r]] = owner with coalesced free-slot reads.
constexpr int kPushChunk = 256;
__global__ void __launch_bounds__(kThreads) k_push(int32_t N, int32_t P, Ws ws, int64_t ldq, const int32_t* o_in,
                                                   int64_t ld_o, int o_vec, int32_t* perm, int64_t ld_perm) {
    __shared__ __align__(16) int32_t s_buf[kThreads / 32][kPushChunk];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t per_filter = cdiv(P, 128);
    const int64_t nblk = static_cast<int64_t>(N) * per_filter;
    const int64_t wstride = static_cast<int64_t>(gridDim.x) * (kThreads / 32);
    int4* b4 = reinterpret_cast<int4*>(s_buf[warp]);
    for (int64_t blk = blockIdx.x * static_cast<int64_t>(kThreads / 32) + warp; blk < nblk; blk += wstride) {
        const int64_t n = blk / per_filter;
        const int64_t i0 = (blk - n * per_filter) * 128 + lane * 4;
        const int32_t* orow = o_in + n * ld_o;
        int32_t ov[4] = {1, 1, 1, 1};
        if (o_vec && i0 + 3 < P) {
            const int4 t = __ldcs(reinterpret_cast<const int4*>(orow + i0));
            ov[0] = t.x; ov[1] = t.y; ov[2] = t.z; ov[3] = t.w;
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (i0 + c < P) ov[c] = orow[i0 + c];
        }
        uint32_t e[4], loc = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            e[c] = ov[c] > 1 ? static_cast<uint32_t>(ov[c] - 1) : 0u;
            loc += e[c];
        }
        uint32_t incl = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += t;
        }
        const uint32_t S = __shfl_sync(kFull, incl, 31);
        if (S == 0) continue;
        const uint32_t lane_off = incl - loc;  // block-relative offset of this lane's first extra
        // R0: exclusive extras prefix of the block's first particle (from the inclusive Qe of lane 0's first)
        uint32_t R0 = 0;
        if (lane == 0) R0 = __ldcg(ws.Qe + n * ldq + i0) - e[0];
        R0 = __shfl_sync(kFull, R0, 0);
        const int32_t* fs = ws.freeslot + n * ldq + R0;
        int32_t* prow = perm + n * ld_perm;
        int32_t carry = -1;
        for (uint32_t c0 = 0; c0 < S; c0 += kPushChunk) {
            b4[2 * lane] = make_int4(-1, -1, -1, -1);
            b4[2 * lane + 1] = make_int4(-1, -1, -1, -1);
            __syncwarp();
            uint32_t off = lane_off;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint32_t rel = off - c0;
                if (e[c] > 0 && rel < static_cast<uint32_t>(kPushChunk)) s_buf[warp][rel] = static_cast<int32_t>(i0 + c);
                off += e[c];
            }
            __syncwarp();
            const int4 lo = b4[2 * lane], hi = b4[2 * lane + 1];
            int32_t h[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
            for (int t = 1; t < 8; ++t) h[t] = max(h[t], h[t - 1]);
            int32_t run = h[7];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t u = __shfl_up_sync(kFull, run, o);
                if (lane >= o) run = max(run, u);
            }
            int32_t pre = __shfl_up_sync(kFull, run, 1);
            pre = max(carry, lane == 0 ? -1 : pre);
            carry = max(carry, __shfl_sync(kFull, run, 31));
            const uint32_t r0 = c0 + 8 * lane;
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                if (r0 + t < S) prow[__ldcg(fs + r0 + t)] = max(h[t], pre);
            }
            __syncwarp();
        }
    }
}

// ============================================================================ a10: gather
template <int CH>  // chunk bytes: 16, 4 or 1
struct Chunk;
template <> struct Chunk<16> { using T = int4; };
template <> struct Chunk<4> { using T = int32_t; };
template <> struct Chunk<1> { using T = char; };

template <int CH>
__global__ void __launch_bounds__(kThreads) k_gather_inplace(char* X, int64_t ld_bytes, int64_t ld_filter_bytes,
                                                             int32_t N, int32_t P, int64_t cpr,
                                                             const int32_t* __restrict__ perm, int64_t ld_perm) {
    using T = typename Chunk<CH>::T;
    const int64_t total = static_cast<int64_t>(N) * P * cpr;
    for (int64_t g = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; g < total;
         g += static_cast<int64_t>(gridDim.x) * kThreads) {
        const int64_t row = g / cpr, c = g - row * cpr;
        const int64_t n = row / P, i = row - n * P;
        const int32_t p = __ldg(perm + n * ld_perm + i);
        if (p == i) continue;
        char* base = X + n * ld_filter_bytes;
        const T v = *reinterpret_cast<const T*>(base + p * ld_bytes + c * CH);
        *reinterpret_cast<T*>(base + i * ld_bytes + c * CH) = v;
    }
}

// In-place gather, 16-byte chunks, warp-cooperative: each warp takes 128
// consecutive rows of one filter (one int4 of permutation entries per lane),
// compacts the moved rows (perm[i] != i) into a per-warp (dst, src) list, then
// copies their chunks with kGU 16-byte loads in flight per lane before the
// stores.  Safe in place: loads only touch survivor rows, stores only
// non-survivor rows.  Requires P % 4 == 0 and 16-byte aligned rows.
constexpr int kGU = 4;
__global__ void __launch_bounds__(kThreads, 8) k_gather_rows16(char* X, int64_t ld_bytes, int64_t ld_filter_bytes,
                                                               int32_t N, int32_t P, int cpr,
                                                               const int32_t* __restrict__ perm, int64_t ld_perm) {
    __shared__ int2 s_ds[kThreads / 32][128];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int per_filter = (P + 127) / 128;
    const int64_t nblk = static_cast<int64_t>(N) * per_filter;
    const int64_t wstride = static_cast<int64_t>(gridDim.x) * (kThreads / 32);
    for (int64_t blk = blockIdx.x * static_cast<int64_t>(kThreads / 32) + warp; blk < nblk; blk += wstride) {
        const int n = static_cast<int>(blk / per_filter);
        const int i0 = static_cast<int>(blk - static_cast<int64_t>(n) * per_filter) * 128 + lane * 4;
        int4 pv = make_int4(0, 1, 2, 3);  // identity for rows past P (not moved)
        if (i0 < P) pv = __ldg(reinterpret_cast<const int4*>(perm + n * ld_perm + i0));
        else pv = make_int4(i0, i0 + 1, i0 + 2, i0 + 3);
        const int m0 = (pv.x != i0), m1 = (pv.y != i0 + 1), m2 = (pv.z != i0 + 2), m3 = (pv.w != i0 + 3);
        const int moved = m0 + m1 + m2 + m3;
        int incl = moved;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += t;
        }
        const int nmoved = __shfl_sync(kFull, incl, 31);
        int at = incl - moved;
        if (m0) s_ds[warp][at++] = make_int2(i0, pv.x);
        if (m1) s_ds[warp][at++] = make_int2(i0 + 1, pv.y);
        if (m2) s_ds[warp][at++] = make_int2(i0 + 2, pv.z);
        if (m3) s_ds[warp][at++] = make_int2(i0 + 3, pv.w);
        __syncwarp();
        char* base = X + n * ld_filter_bytes;
        const int items = nmoved * cpr;
        for (int it0 = 0; it0 < items; it0 += 32 * kGU) {
            int4 v[kGU];
#pragma unroll
            for (int u = 0; u < kGU; ++u) {
                const int it = it0 + u * 32 + lane;
                if (it < items) {
                    const int rw = it / cpr, ch = it - rw * cpr;
                    v[u] = *reinterpret_cast<const int4*>(base + static_cast<int64_t>(s_ds[warp][rw].y) * ld_bytes + ch * 16);
                }
            }
#pragma unroll
            for (int u = 0; u < kGU; ++u) {
                const int it = it0 + u * 32 + lane;
                if (it < items) {
                    const int rw = it / cpr, ch = it - rw * cpr;
                    __stcs(reinterpret_cast<int4*>(base + static_cast<int64_t>(s_ds[warp][rw].x) * ld_bytes + ch * 16), v[u]);
                }
            }
        }
        __syncwarp();
    }
}

template <int CH>
__global__ void __launch_bounds__(kThreads) k_gather_out(const char* __restrict__ X, char* __restrict__ Y,
                                                         int64_t ld_x, int64_t ld_y, int32_t P, int64_t cpr,
                                                         const int32_t* __restrict__ anc) {
    using T = typename Chunk<CH>::T;
    const int64_t total = static_cast<int64_t>(P) * cpr;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
    for (int64_t g0 = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; g0 < total; g0 += 4 * stride) {
        T v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t g = g0 + u * stride;
            if (g < total) {
                const int64_t i = g / cpr, c = g - i * cpr;
                const int32_t p = __ldg(anc + i);
                v[u] = __ldg(reinterpret_cast<const T*>(X + p * ld_x + c * CH));
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t g = g0 + u * stride;
            if (g < total) {
                const int64_t i = g / cpr, c = g - i * cpr;
                *reinterpret_cast<T*>(Y + i * ld_y + c * CH) = v[u];
            }
        }
    }
}

// ============================================================================ shards (C5)
struct ShardCtxDev {
    int64_t k_lo, k_hi;
    uint64_t off, Qtot, T;
    int32_t invalid;
};

template <int SCHEME>
__device__ __forceinline__ uint64_t shard_position(int64_t k, uint64_t D, uint64_t rho, uint64_t Qtot, Key key,
                                                   uint32_t filt) {
    if (SCHEME == 2) {
        const u32x4 r = philox10(static_cast<uint32_t>(k >> 1), 0u, 2u, filt, key.k0, key.k1);
        rho = mulhi64((k & 1) ? hi_word(r) : lo_word(r), D);
    }
    return mulhi64(static_cast<uint64_t>(k) * D + rho, Qtot);
}

// One warp: offsets from the all-gathered totals, validity, and the slot range
// [k_lo, k_hi) = [#{k : x_k < off}, #{k : x_k < off + T}) by 32-ary searches.
template <int SCHEME>
__global__ void k_shard_range(const uint64_t* totals, int nshards, int shard, const float* gmax,
                              const int32_t* gbad, int64_t P_global, uint64_t D, Key key, uint32_t filt,
                              ShardCtxDev* ctx, int64_t* range_out) {
    const int lane = threadIdx.x & 31;
    uint64_t off = 0, tot = 0;
    for (int h = 0; h < nshards; ++h) {
        const uint64_t t = totals[h];
        if (h < shard) off += t;
        tot += t;
    }
    const uint64_t T = totals[shard];
    const int invalid = (*gbad != 0 || *gmax == -INFINITY) ? 1 : 0;
    uint64_t rho = 0;
    if (SCHEME == 3) rho = mulhi64(lo_word(philox10(0u, 0u, 3u, filt, key.k0, key.k1)), D);
    int64_t kk[2];
    for (int w = 0; w < 2; ++w) {
        const uint64_t v = w ? off + T : off;
        int64_t lo = 0, hi = P_global;
        while (hi > lo) {
            const int64_t step = (hi - lo + 31) / 32;
            const int64_t m = lo + lane * step;
            const bool p = (m < hi) && (shard_position<SCHEME>(m, D, rho, tot, key, filt) < v);
            const int L = __popc(__ballot_sync(kFull, p));
            const int64_t nlo = (L == 0) ? lo : lo + static_cast<int64_t>(L - 1) * step + 1;
            const int64_t mL = lo + static_cast<int64_t>(L) * step;
            hi = (mL < hi) ? mL : hi;
            lo = nlo;
        }
        kk[w] = lo;
    }
    if (lane == 0) {
        ctx->k_lo = invalid ? 0 : kk[0];
        ctx->k_hi = invalid ? 0 : kk[1];
        ctx->off = off;
        ctx->Qtot = tot;
        ctx->T = T;
        ctx->invalid = invalid;
        range_out[0] = ctx->k_lo;
        range_out[1] = ctx->k_hi;
    }
}

struct ShardCtx {
    int n;
    int64_t k_lo, nA;
    uint64_t off, Qtot, D, rho;
    uint32_t filt;
};

template <int SCHEME>
struct ModeShard {
    const uint64_t* Q;
    const ShardCtxDev* dctx;
    uint64_t D;
    Key key;
    uint32_t filt;
    int32_t P;  // particles of this shard (the B list)
    int64_t p0;
    int32_t* anc;

    using Ctx = ShardCtx;
    __device__ Ctx ctx(int) const {
        Ctx c;
        c.n = 0;
        c.k_lo = dctx->k_lo;
        c.nA = dctx->k_hi - dctx->k_lo;
        c.off = dctx->off;
        c.Qtot = dctx->Qtot;
        c.D = D;
        c.filt = filt;
        c.rho = 0;
        if (SCHEME == 3) c.rho = mulhi64(lo_word(philox10(0u, 0u, 3u, filt, key.k0, key.k1)), D);
        return c;
    }
    __device__ bool valid(int) const { return dctx->invalid == 0; }
    __device__ int64_t nA(const Ctx& c) const { return c.nA; }
    __device__ uint64_t x(const Ctx& c, int64_t m) const {
        return shard_position<SCHEME>(c.k_lo + m, c.D, c.rho, c.Qtot, key, c.filt);
    }
    __device__ uint64_t b(const Ctx& c, int64_t i) const { return c.off + __ldg(Q + i); }
    __device__ void fill_a(const Ctx& c, int64_t ka0, int na, uint64_t* s) const {
        for (int t = threadIdx.x; t < na; t += kThreads) s[t] = x(c, ka0 + t);
    }
    __device__ void emit(const Ctx& c, int64_t ka0, int na, const int32_t* s_out) const {
        int32_t* dst = anc + c.k_lo + ka0;
        for (int t = threadIdx.x; t < na; t += kThreads) dst[t] = static_cast<int32_t>(p0 + s_out[t]);
    }
    __device__ void identity(int, int cb, int cpf) const {
        const int64_t per = cdiv(P, cpf);
        const int64_t b0 = cb * per, b1 = min(static_cast<int64_t>(P), b0 + per);
        for (int64_t k = b0 + threadIdx.x; k < b1; k += kThreads) anc[p0 + k] = static_cast<int32_t>(p0 + k);
    }
};

// Multinomial shard: every shard regenerates all positions (NS-8) and keeps
// those in its cumulative-weight range [off, off + T); binary search in d_Q.
__global__ void __launch_bounds__(kThreads) k_shard_multinomial(const uint64_t* __restrict__ Q, int32_t Pl,
                                                                int64_t p0, int64_t P_global,
                                                                const ShardCtxDev* dctx, Key key, uint32_t filt,
                                                                int32_t* anc) {
    const ShardCtxDev c = *dctx;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
    const int64_t g0 = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x;
    if (c.invalid) {
        for (int64_t k = g0; k < Pl; k += stride) anc[p0 + k] = static_cast<int32_t>(p0 + k);
        return;
    }
    const int64_t npairs = (P_global + 1) / 2;
    for (int64_t pr = g0; pr < npairs; pr += stride) {
        const u32x4 r = philox10(static_cast<uint32_t>(pr), 0u, 1u, filt, key.k0, key.k1);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t k = 2 * pr + h;
            if (k >= P_global) break;
            const uint64_t x = mulhi64(h ? hi_word(r) : lo_word(r), c.Qtot);
            if (x < c.off || x - c.off >= c.T) continue;
            const uint64_t xl = x - c.off;  // local position; local Q is relative to the shard
            int64_t lo = 0, hi = Pl - 1;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (__ldg(Q + mid) > xl) hi = mid;
                else lo = mid + 1;
            }
            anc[k] = static_cast<int32_t>(p0 + lo);
        }
    }
}

// ---- Routed multinomial: rank g generates only the positions of
// its own slot shard [k0, k1) (NS-8) and sends each to the shard whose cumulative-weight range
// holds it (one variable all-to-all); the owner searches its local Q.  Work per rank ~ P/G.
struct RouteRanges {
    uint64_t off[kMaxRouteShards + 1];  // exclusive prefix of the shard totals
    uint64_t Qtot;
    int32_t invalid;
};

__device__ __forceinline__ void route_ranges(const uint64_t* totals, int nshards, const float* gmax,
                                             const int32_t* gbad, RouteRanges* r) {
    uint64_t c = 0;
    for (int h = 0; h < nshards; ++h) {
        r->off[h] = c;
        c += totals[h];
    }
    r->off[nshards] = c;
    r->Qtot = c;
    r->invalid = (*gbad != 0 || *gmax == -INFINITY) ? 1 : 0;
}

// owner shard of position x: the h with off[h] <= x < off[h + 1] (empty ranges never match)
__device__ __forceinline__ int route_owner(const RouteRanges& r, int nshards, uint64_t x) {
    int h = 0;
    for (int g = 1; g < nshards; ++g) h = (r.off[g] <= x) ? g : h;
    return h;
}

// pass 1: positions of the slot shard per owner (counts[nshards], zeroed by the caller);
// pass 2 (cursor != nullptr): (x, k) pairs grouped by owner, group h starting at the exclusive
// prefix of counts (order inside a group is arbitrary; each pair carries its slot)
__global__ void __launch_bounds__(kThreads) k_route(const uint64_t* totals, int nshards, const float* gmax,
                                                    const int32_t* gbad, int64_t P_global, int64_t k0, int64_t k1,
                                                    Key key, uint32_t filt, unsigned long long* counts,
                                                    unsigned long long* cursor, uint64_t* send_x, int32_t* send_k) {
    __shared__ RouteRanges s_r;
    __shared__ unsigned long long s_base[kMaxRouteShards];
    if (threadIdx.x == 0) route_ranges(totals, nshards, gmax, gbad, &s_r);
    if (cursor != nullptr && threadIdx.x < nshards) {
        unsigned long long b = 0;
        for (int h = 0; h < static_cast<int>(threadIdx.x); ++h) b += counts[h];
        s_base[threadIdx.x] = b;
    }
    __syncthreads();
    if (s_r.invalid) return;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
    // pairs of slots (one Philox call, NS-8); the loop is warp-uniform for the aggregation
    const int64_t pr0 = k0 >> 1, pr1 = (k1 + 1) >> 1;
    const int64_t rounds = (pr1 - pr0 + stride - 1) / stride;
    for (int64_t rr = 0; rr < rounds; ++rr) {
        const int64_t pr = pr0 + rr * stride + blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x;
        u32x4 r = {0u, 0u, 0u, 0u};
        if (pr < pr1) r = philox10(static_cast<uint32_t>(pr), 0u, 1u, filt, key.k0, key.k1);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int64_t k = 2 * pr + hh;
            const bool mine = pr < pr1 && k >= k0 && k < k1;
            const uint64_t x = mine ? mulhi64(hh ? hi_word(r) : lo_word(r), s_r.Qtot) : 0;
            const int h = mine ? route_owner(s_r, nshards, x) : -1;
            // warp-aggregated: one atomic per (warp, owner)
            const unsigned peers = __match_any_sync(0xFFFFFFFFu, h);
            const int leader = __ffs(peers) - 1;
            const int rank = __popc(peers & ((1u << (threadIdx.x & 31)) - 1u));
            unsigned long long base = 0;
            if (mine && (threadIdx.x & 31) == leader)
                base = atomicAdd(cursor ? cursor + h : counts + h, static_cast<unsigned long long>(__popc(peers)));
            base = __shfl_sync(0xFFFFFFFFu, base, leader);
            if (mine && cursor) {
                const unsigned long long at = s_base[h] + base + rank;
                send_x[at] = x;
                send_k[at] = static_cast<int32_t>(k);
            }
        }
    }
}

// received (x, k): anc[k] = p0 + min{i : Q_i > x - off_shard}; invalid filter: the identity over
// the shard's own particles (every rank writes its own, as the other schemes do)
__global__ void __launch_bounds__(kThreads) k_route_search(const uint64_t* __restrict__ Q, int32_t Pl, int64_t p0,
                                                           const uint64_t* totals, int nshards, int shard,
                                                           const float* gmax, const int32_t* gbad,
                                                           const uint64_t* __restrict__ rx,
                                                           const int32_t* __restrict__ rk, int64_t nrecv,
                                                           int32_t* anc) {
    __shared__ RouteRanges s_r;
    if (threadIdx.x == 0) route_ranges(totals, nshards, gmax, gbad, &s_r);
    __syncthreads();
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
    const int64_t g0 = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x;
    if (s_r.invalid) {
        for (int64_t i = g0; i < Pl; i += stride) anc[p0 + i] = static_cast<int32_t>(p0 + i);
        return;
    }
    const uint64_t off = s_r.off[shard];
    for (int64_t t = g0; t < nrecv; t += stride) {
        const uint64_t xl = __ldg(rx + t) - off;
        int64_t lo = 0, hi = Pl - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (__ldg(Q + mid) > xl) hi = mid;
            else lo = mid + 1;
        }
        anc[__ldg(rk + t)] = static_cast<int32_t>(p0 + lo);
    }
}

__global__ void __launch_bounds__(kThreads) k_shard_weights(const float* __restrict__ logw, int32_t Pl,
                                                            const float* gmax, float* w) {
    const float lm = *gmax;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; i < Pl;
         i += static_cast<int64_t>(gridDim.x) * kThreads)
        w[i] = weight(__ldcs(logw + i), lm);
}

// Metropolis chains slot0 .. slot0 + nslots - 1 over the full weight vector (NS-11).
__global__ void __launch_bounds__(kThreads) k_metro_slots(const float* __restrict__ w, int64_t P_global,
                                                          int64_t slot0, int32_t nslots, Key key, uint32_t filt,
                                                          int32_t B, const float* gmax, const int32_t* gbad,
                                                          int32_t* anc) {
    const int64_t s = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x;
    if (s >= nslots) return;
    const int64_t i = slot0 + s;
    const bool invalid = (gbad && *gbad != 0) || (gmax && *gmax == -INFINITY);
    if (invalid || B == 0) {
        anc[s] = static_cast<int32_t>(i);
        return;
    }
    int64_t k = i;
    float wk = __ldg(w + i);
    const float kU = __uint_as_float(0x33800000u);
    for (int32_t b = 0; b < B; b += 8) {
        uint32_t j[8];
        float u[8], wj[8];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const u32x4 r = philox10(static_cast<uint32_t>(i), static_cast<uint32_t>((b >> 1) + t), 4u, filt, key.k0,
                                     key.k1);
            j[2 * t] = static_cast<uint32_t>((static_cast<uint64_t>(r.x) * static_cast<uint64_t>(P_global)) >> 32);
            u[2 * t] = __fmul_rn(static_cast<float>(r.y >> 8), kU);
            j[2 * t + 1] = static_cast<uint32_t>((static_cast<uint64_t>(r.z) * static_cast<uint64_t>(P_global)) >> 32);
            u[2 * t + 1] = __fmul_rn(static_cast<float>(r.w >> 8), kU);
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) wj[t] = (b + t < B) ? __ldg(w + j[t]) : 0.0f;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            if (b + t < B && __fmul_rn(u[t], wk) < wj[t]) {
                k = j[t];
                wk = wj[t];
            }
        }
    }
    anc[s] = static_cast<int32_t>(k);
}

// ============================================================================ a6 shards (C5 sorted multinomial)
// SURVEY §8(e) "Giant filter: sorted multinomial": the P + 1 spacings e_0..e_P
// (NS-12) are split into nshards contiguous spacing shards [s_h, s_{h+1}),
// s_h = min(P + 1, h * ceil((P + 1) / nshards)); rank h contributes the total of
// its spacing shard, the totals are all-gathered, so every rank knows
// G_{s_h - 1} = sum_{h' < h} etot_h' and G_P = sum of all.  Rank g's slots are
// those with x_k = floor(G_k Q / G_P) in [off_g, off_g + T_g); it regenerates
// and scans only the spacing shards that contain them.
__device__ __forceinline__ uint64_t spacing_at(int64_t k, uint32_t filt, Key key) {
    const u32x4 r = philox10(static_cast<uint32_t>(k >> 2), 0u, 5u, filt, key.k0, key.k1);
    const int c = static_cast<int>(k & 3);
    return spacing_from_word(c == 0 ? r.x : c == 1 ? r.y : c == 2 ? r.z : r.w);
}

__host__ __device__ __forceinline__ int64_t spacing_shard_begin(int64_t P, int nshards, int h) {
    const int64_t per = (P + 1 + nshards - 1) / nshards;
    return min(P + 1, static_cast<int64_t>(h) * per);
}

// sum of e_k over k in [k0, k1) into *etot (zeroed by the caller; integer atomics: order-free)
__global__ void __launch_bounds__(kThreads) k_spacings_total(int64_t k0, int64_t k1, Key key, uint32_t filt,
                                                             unsigned long long* etot) {
    __shared__ uint64_t s_w[kThreads / 32];
    uint64_t sum = 0;
    const int64_t g0 = k0 >> 2, g1 = (k1 + 3) >> 2;  // groups of 4 spacings (one Philox call)
    for (int64_t g = g0 + blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; g < g1;
         g += static_cast<int64_t>(gridDim.x) * kThreads) {
        const u32x4 r = philox10(static_cast<uint32_t>(g), 0u, 5u, filt, key.k0, key.k1);
        const uint32_t w4[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int64_t k = 4 * g + c;
            if (k >= k0 && k < k1) sum += spacing_from_word(w4[c]);
        }
    }
    sum = warp_sum_u64(sum);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) s_w[warp] = sum;
    __syncthreads();
    if (warp == 0) {
        uint64_t v = (lane < kThreads / 32) ? s_w[lane] : 0ull;
        v = warp_sum_u64(v);
        if (lane == 0 && v) atomicAdd(etot, static_cast<unsigned long long>(v));
    }
}

struct SpacShardDev {
    int64_t sa, sb;       // scanned slot range [sa, sb): G_ws[k - sa] = G_k
    int64_t hlo[2];       // spacing shard holding the crossing of off and off + T
    int64_t k_lo, k_hi;   // this rank's slots
    uint64_t off, Qtot, T, GP, Gbase;
    uint64_t ntiles;
    int32_t invalid;
};

// a * b < c * d for u64 operands (exact 128-bit products)
__device__ __forceinline__ bool lt128(uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    const uint64_t h1 = __umul64hi(a, b), h2 = __umul64hi(c, d);
    return h1 < h2 || (h1 == h2 && a * b < c * d);
}

// One warp: offsets, G at the spacing-shard boundaries, and the range of spacing
// shards to scan.  crossing shard of v: h(v) = max{h : h == 0 or G_{s_h - 1} Q < v G_P}
// (every slot before s_h has x < v; the first slot with x >= v lies in [s_h, s_{h+1}]).
__global__ void k_spac_shard_plan(const uint64_t* totals, const uint64_t* etotals, int nshards, int shard,
                                  const float* gmax, const int32_t* gbad, int64_t P, SpacShardDev* ctx) {
    if (threadIdx.x != 0) return;
    uint64_t off = 0, Qt = 0, GP = 0;
    for (int h = 0; h < nshards; ++h) {
        if (h < shard) off += totals[h];
        Qt += totals[h];
        GP += etotals[h];
    }
    const uint64_t T = totals[shard];
    const int invalid = (*gbad != 0 || *gmax == -INFINITY) ? 1 : 0;
    int64_t hv[2];
    for (int w = 0; w < 2; ++w) {
        const uint64_t v = w ? off + T : off;
        int hb = 0;
        uint64_t Gb = 0;  // G_{s_h - 1}
        for (int h = 1; h < nshards; ++h) {
            Gb += etotals[h - 1];
            if (spacing_shard_begin(P, nshards, h) < P && lt128(Gb, Qt, v, GP)) hb = h;
        }
        hv[w] = hb;
    }
    uint64_t Gbase = 0;
    for (int h = 0; h < hv[0]; ++h) Gbase += etotals[h];
    const int64_t sa = spacing_shard_begin(P, nshards, static_cast<int>(hv[0]));
    const int64_t sb = min(P, spacing_shard_begin(P, nshards, static_cast<int>(hv[1]) + 1));
    ctx->sa = sa;
    ctx->sb = (invalid || T == 0) ? sa : max(sa, sb);
    ctx->hlo[0] = hv[0];
    ctx->hlo[1] = hv[1];
    ctx->off = off;
    ctx->Qtot = Qt;
    ctx->T = T;
    ctx->GP = GP;
    ctx->Gbase = Gbase;
    ctx->ntiles = static_cast<uint64_t>(cdiv(ctx->sb - ctx->sa, kTile));
    ctx->invalid = invalid;
    ctx->k_lo = ctx->k_hi = 0;
}

// Persistent decoupled-lookback scan of e_k over [sa, sb) (the plan's range, read on
// the device): G_ws[k - sa] = Gbase + e_sa + ... + e_k.  Tiles are taken in order from a
// global counter, so a CTA only ever waits on tiles held by running CTAs.
__global__ void __launch_bounds__(kThreads, 4) k_gscan_range(const SpacShardDev* ctx, Key key, uint32_t filt,
                                                             uint32_t* tile_ctr, uint64_t* status, uint64_t* G) {
    __shared__ uint32_t s_tile;
    __shared__ uint64_t s_wtot[kThreads / 32];
    __shared__ uint64_t s_off[kThreads / 32];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t sa = ctx->sa, len = ctx->sb - ctx->sa;
    const uint64_t ntiles = ctx->ntiles, Gbase = ctx->Gbase;
    for (;;) {
        if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
        __syncthreads();
        const int64_t tile = s_tile;
        if (static_cast<uint64_t>(tile) >= ntiles) break;
        const int64_t base = tile * kTile + warp * 512;  // relative to sa
        uint64_t v[16];
        uint64_t excl[4];
        uint64_t carry = 0;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int64_t i0 = base + r * 128 + lane * 4;
            uint64_t loc = 0;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                v[r * 4 + c] = (i0 + c < len) ? spacing_at(sa + i0 + c, filt, key) : 0ull;
                loc += v[r * 4 + c];
            }
            const uint64_t incl = warp_incl_scan_u64(loc, lane);
            excl[r] = incl - loc + carry;
            carry += __shfl_sync(kFull, incl, 31);
        }
        if (lane == 0) s_wtot[warp] = carry;
        __syncthreads();
        if (warp == 0) {
            const uint64_t wv = (lane < kThreads / 32) ? s_wtot[lane] : 0ull;
            const uint64_t wi = warp_incl_scan_u64(wv, lane);
            const uint64_t agg = __shfl_sync(kFull, wi, kThreads / 32 - 1);
            uint64_t prefix = 0;
            if (tile == 0) {
                if (lane == 0) st_release(status, kFlagInc | agg);
            } else {
                if (lane == 0) st_release(status + tile, kFlagAgg | agg);
                prefix = lookback(status, tile, lane);
                if (lane == 0) st_release(status + tile, kFlagInc | (prefix + agg));
            }
            if (lane < kThreads / 32) s_off[lane] = prefix + wi - wv;
        }
        __syncthreads();
        const uint64_t off = Gbase + s_off[warp];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int64_t i0 = base + r * 128 + lane * 4;
            uint64_t run = off + excl[r];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                run += v[r * 4 + c];
                if (i0 + c < len) G[i0 + c] = run;
            }
        }
    }
}

// One warp: k(v) = #{k < P : G_k Q < v G_P} for v = off, off + T, searching the scanned
// crossing shard (32-ary search over G_ws).
__global__ void k_spac_shard_range(SpacShardDev* ctx, const uint64_t* G, int64_t P, int nshards,
                                   int64_t* range_out) {
    const int lane = threadIdx.x & 31;
    const int64_t sa = ctx->sa, sb = ctx->sb;
    const uint64_t Qt = ctx->Qtot, GP = ctx->GP;
    int64_t kk[2];
    for (int w = 0; w < 2; ++w) {
        const uint64_t v = w ? ctx->off + ctx->T : ctx->off;
        const int h = static_cast<int>(ctx->hlo[w]);
        // every k < s_h is below v; the crossing is in [s_h, min(s_{h+1}, P)]
        int64_t lo = max(sa, spacing_shard_begin(P, nshards, h));
        int64_t hi = min(sb, spacing_shard_begin(P, nshards, h + 1));
        hi = max(lo, hi);
        while (hi > lo) {
            const int64_t step = (hi - lo + 31) / 32;
            const int64_t m = lo + lane * step;
            const bool p = (m < hi) && lt128(G[m - sa], Qt, v, GP);
            const int L = __popc(__ballot_sync(kFull, p));
            const int64_t nlo = (L == 0) ? lo : lo + static_cast<int64_t>(L - 1) * step + 1;
            const int64_t mL = lo + static_cast<int64_t>(L) * step;
            hi = (mL < hi) ? mL : hi;
            lo = nlo;
        }
        kk[w] = lo;
    }
    if (lane == 0) {
        const bool empty = ctx->invalid || ctx->T == 0;
        ctx->k_lo = empty ? 0 : kk[0];
        ctx->k_hi = empty ? 0 : kk[1];
        range_out[0] = ctx->k_lo;
        range_out[1] = ctx->k_hi;
    }
}

struct SpacShardCtx {
    int n;
    int64_t k_lo, nA, sa;
    uint64_t off, Qtot, GP;
};

struct ModeShardSpacings {
    const uint64_t* Q;
    const SpacShardDev* dctx;
    const uint64_t* G;
    int32_t P;  // particles of this shard (the B list)
    int64_t p0;
    int32_t* anc;

    using Ctx = SpacShardCtx;
    __device__ Ctx ctx(int) const {
        Ctx c;
        c.n = 0;
        c.k_lo = dctx->k_lo;
        c.nA = dctx->k_hi - dctx->k_lo;
        c.sa = dctx->sa;
        c.off = dctx->off;
        c.Qtot = dctx->Qtot;
        c.GP = dctx->GP;
        return c;
    }
    __device__ bool valid(int) const { return dctx->invalid == 0; }
    __device__ int64_t nA(const Ctx& c) const { return c.nA; }
    __device__ uint64_t x(const Ctx& c, int64_t m) const {
        return muldiv_floor(__ldg(G + (c.k_lo + m - c.sa)), c.Qtot, c.GP);
    }
    __device__ uint64_t b(const Ctx& c, int64_t i) const { return c.off + __ldg(Q + i); }
    __device__ void fill_a(const Ctx& c, int64_t ka0, int na, uint64_t* s) const {
        for (int t = threadIdx.x; t < na; t += kThreads) s[t] = x(c, ka0 + t);
    }
    __device__ void emit(const Ctx& c, int64_t ka0, int na, const int32_t* s_out) const {
        int32_t* dst = anc + c.k_lo + ka0;
        for (int t = threadIdx.x; t < na; t += kThreads) dst[t] = static_cast<int32_t>(p0 + s_out[t]);
    }
    __device__ void identity(int, int cb, int cpf) const {
        const int64_t per = cdiv(P, cpf);
        const int64_t b0 = cb * per, b1 = min(static_cast<int64_t>(P), b0 + per);
        for (int64_t k = b0 + threadIdx.x; k < b1; k += kThreads) anc[p0 + k] = static_cast<int32_t>(p0 + k);
    }
};

// ============================================================================ C4 demo model
__device__ __forceinline__ void box_muller4(const u32x4& r, float z[4]) {
    const float k = 2.3283064365386963e-10f;  // 2^-32
    const float u1 = (static_cast<float>(r.x) + 0.5f) * k, u2 = (static_cast<float>(r.y) + 0.5f) * k;
    const float u3 = (static_cast<float>(r.z) + 0.5f) * k, u4 = (static_cast<float>(r.w) + 0.5f) * k;
    const float a = sqrtf(-2.0f * logf(u1)), b = sqrtf(-2.0f * logf(u3));
    float s1, c1, s2, c2;
    sincospif(2.0f * u2, &s1, &c1);
    sincospif(2.0f * u4, &s2, &c2);
    z[0] = a * c1; z[1] = a * s1; z[2] = b * c2; z[3] = b * s2;
}

__global__ void __launch_bounds__(kThreads) k_lg_init(float* X, int64_t ld, int32_t P, int32_t D, float sd,
                                                      Key key) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x;
    if (i >= P) return;
    float* row = X + i * ld;
    const int nb = (D + 3) / 4;
    for (int b = 0; b < nb; ++b) {
        float z[4];
        box_muller4(philox10(static_cast<uint32_t>(i), static_cast<uint32_t>(b), 7u, 0u, key.k0, key.k1), z);
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (4 * b + q < D) row[4 * b + q] = sd * z[q];
    }
}

__global__ void __launch_bounds__(kThreads) k_lg_step(float* X, int64_t ld, int32_t P, int32_t D, float phi,
                                                      float sx, float inv2vy, float y, Key key, int32_t t,
                                                      float* logw, int vec) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x;
    if (i >= P) return;
    float* row = X + i * ld;
    const int nb = (D + 3) / 4;
    float x0 = 0.0f;
    for (int b = 0; b < nb; ++b) {
        float z[4];
        box_muller4(philox10(static_cast<uint32_t>(i), static_cast<uint32_t>(t * nb + b), 6u, 0u, key.k0, key.k1), z);
        if (vec && 4 * b + 3 < D) {
            float4 v = reinterpret_cast<float4*>(row)[b];
            v.x = phi * v.x + sx * z[0];
            v.y = phi * v.y + sx * z[1];
            v.z = phi * v.z + sx * z[2];
            v.w = phi * v.w + sx * z[3];
            reinterpret_cast<float4*>(row)[b] = v;
            if (b == 0) x0 = v.x;
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (4 * b + q < D) {
                    const float nv = phi * row[4 * b + q] + sx * z[q];
                    row[4 * b + q] = nv;
                    if (b == 0 && q == 0) x0 = nv;
                }
            }
        }
    }
    const float d = y - x0;
    logw[i] = -d * d * inv2vy;
}

__global__ void k_lg_accumulate(const double* lse, double c, double* loglik) {
    if (threadIdx.x == 0) loglik[0] += lse[0] - c;
}

int64_t grid_for(int64_t work, int per_sm = 8) {
    const int64_t cap = static_cast<int64_t>(sm_count()) * per_sm;
    const int64_t need = cdiv(work, kThreads);
    return std::max<int64_t>(1, std::min(cap, need));
}

}  // namespace

int sm_count() {
    static std::atomic<int> cache[kMaxDevices];
    return cached_per_device(cache, [] {
        int sms = 0;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, current_device()) != cudaSuccess ||
            sms <= 0) {
            cudaGetLastError();
            sms = 148;
        }
        return sms;
    });
}


// ============================================================================ host side
Layout make_layout(int32_t N, int32_t P, unsigned need) {
    Layout L{};
    const int64_t target = static_cast<int64_t>(sm_count()) * 4;
    int64_t cpf = cdiv(target, N);
    cpf = std::min<int64_t>(cpf, cdiv(P, 2048));
    L.cpf_max = static_cast<int>(std::max<int64_t>(1, cpf));
    L.T = static_cast<int>(cdiv(P, kTile));
    L.ldq = (P + 3) / 4 * 4;
    const int64_t NT = static_cast<int64_t>(N) * L.T;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        off = align_up(off, 256);
        const size_t at = off;
        off += bytes;
        return at;
    };
    L.lmax = take(sizeof(float) * N);
    L.fstatus = take(sizeof(int32_t) * N);
    L.max_part = take(sizeof(float) * N * L.cpf_max);
    L.max_bad = take(sizeof(int32_t) * N * L.cpf_max);
    L.zero_begin = take(0);
    L.max_cnt = take(sizeof(uint32_t) * N);
    L.tile_ctr = take(sizeof(uint32_t));
    L.tstatus = take(sizeof(uint64_t) * NT);
    L.T2 = static_cast<int>(cdiv(static_cast<int64_t>(P) + 1, kTile));
    L.ldg = (static_cast<int64_t>(P) + 1 + 3) / 4 * 4;
    L.tile_ctr2 = (need & kNeedG) ? take(sizeof(uint32_t)) : 0;
    L.tstatus2 = (need & kNeedG) ? take(sizeof(uint64_t) * static_cast<int64_t>(N) * L.T2) : 0;
    L.zero_end = align_up(off, 256);
    L.tsum = take(sizeof(double) * NT);
    L.tsum2 = take(sizeof(double) * NT);
    L.Qtot = take(sizeof(uint64_t) * N);
    L.S = take(sizeof(double) * N);
    L.F = take(sizeof(int32_t) * N);
    const size_t rows = static_cast<size_t>(N) * L.ldq;
    L.Q = (need & kNeedQ) ? take(sizeof(uint64_t) * rows) : 0;
    L.w = (need & kNeedW) ? take(sizeof(float) * rows) : 0;
    L.o = (need & kNeedPermute) ? take(sizeof(int32_t) * rows) : 0;
    L.Qe = (need & kNeedPermute) ? take(sizeof(uint32_t) * rows) : 0;
    L.freeslot = (need & kNeedPermute) ? take(sizeof(int32_t) * rows) : 0;
    L.G = (need & kNeedG) ? take(sizeof(uint64_t) * static_cast<size_t>(N) * L.ldg) : 0;
    L.ldb = int64_t{1} << ceil_log2(P);
    L.bidx = (need & kNeedBuckets) ? take(sizeof(int32_t) * static_cast<size_t>(N) * L.ldb) : 0;
    L.Gtot = (need & kNeedG) ? take(sizeof(uint64_t) * N) : 0;
    L.total = align_up(off, 256);
    return L;
}

Ws carve(void* base, const Layout& L) {
    char* b = static_cast<char*>(base);
    Ws w{};
    w.lmax = reinterpret_cast<float*>(b + L.lmax);
    w.fstatus = reinterpret_cast<int32_t*>(b + L.fstatus);
    w.max_part = reinterpret_cast<float*>(b + L.max_part);
    w.max_bad = reinterpret_cast<int32_t*>(b + L.max_bad);
    w.max_cnt = reinterpret_cast<uint32_t*>(b + L.max_cnt);
    w.tile_ctr = reinterpret_cast<uint32_t*>(b + L.tile_ctr);
    w.tstatus = reinterpret_cast<uint64_t*>(b + L.tstatus);
    w.tsum = reinterpret_cast<double*>(b + L.tsum);
    w.tsum2 = reinterpret_cast<double*>(b + L.tsum2);
    w.Qtot = reinterpret_cast<uint64_t*>(b + L.Qtot);
    w.S = reinterpret_cast<double*>(b + L.S);
    w.F = reinterpret_cast<int32_t*>(b + L.F);
    w.Q = L.Q ? reinterpret_cast<uint64_t*>(b + L.Q) : nullptr;
    w.w = L.w ? reinterpret_cast<float*>(b + L.w) : nullptr;
    w.o = L.o ? reinterpret_cast<int32_t*>(b + L.o) : nullptr;
    w.Qe = L.Qe ? reinterpret_cast<uint32_t*>(b + L.Qe) : nullptr;
    w.freeslot = L.freeslot ? reinterpret_cast<int32_t*>(b + L.freeslot) : nullptr;
    w.tile_ctr2 = L.tile_ctr2 ? reinterpret_cast<uint32_t*>(b + L.tile_ctr2) : nullptr;
    w.tstatus2 = L.tstatus2 ? reinterpret_cast<uint64_t*>(b + L.tstatus2) : nullptr;
    w.G = L.G ? reinterpret_cast<uint64_t*>(b + L.G) : nullptr;
    w.Gtot = L.Gtot ? reinterpret_cast<uint64_t*>(b + L.Gtot) : nullptr;
    w.bidx = L.bidx ? reinterpret_cast<int32_t*>(b + L.bidx) : nullptr;
    return w;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

cudaError_t launch_max(const float* logw, int64_t ld, int32_t N, int32_t P, const Layout& L, const Ws& ws,
                       int32_t* status_out, cudaStream_t s, uint64_t* launches, float* lmax_out, int32_t* bad_out) {
    const int cpf = L.cpf_max;
    int64_t chunk = cdiv(P, cpf);
    chunk = (chunk + 3) / 4 * 4;
    const bool vec = aligned16(logw) && (ld % 4 == 0);
    const dim3 grid(static_cast<unsigned>(static_cast<int64_t>(N) * cpf));
    if (vec) { ProfScope ps_("k_max", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 4u); k_max<true><<<grid, kThreads, 0, s>>>(logw, ld, P, cpf, chunk, ws, status_out, lmax_out, bad_out); }
    else { ProfScope ps_("k_max", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 4u); k_max<false><<<grid, kThreads, 0, s>>>(logw, ld, P, cpf, chunk, ws, status_out, lmax_out, bad_out); }
    ++*launches;
    return cudaPeekAtLastError();
}

cudaError_t launch_scan(const float* logw, int64_t ld, int32_t N, int32_t P, const Layout& L, const Ws& ws,
                        bool write_q, double* lse_out, double* ess_out, cudaStream_t s, uint64_t* launches,
                        int kfx_override) {
    const int kfx = (kfx_override >= 0) ? kfx_override : 61 - ceil_log2(P);
    const bool vec = aligned16(logw) && (ld % 4 == 0);
    if (N >= sm_count() && P <= (1 << 17)) {
        // a CTA per filter (no lookback): 2 CTAs per SM, persistent over the filters
        const unsigned g = static_cast<unsigned>(std::min<int64_t>(N, 2LL * sm_count()));
        ProfScope ps_("k_scan", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * (write_q ? 12u : 4u));
        if (vec) k_scan_cta<true><<<g, kScanCtaT, 0, s>>>(logw, ld, N, P, kfx, ws, L.ldq, write_q ? 1 : 0, lse_out, ess_out);
        else k_scan_cta<false><<<g, kScanCtaT, 0, s>>>(logw, ld, N, P, kfx, ws, L.ldq, write_q ? 1 : 0, lse_out, ess_out);
        ++*launches;
        return cudaPeekAtLastError();
    }
    const dim3 grid(static_cast<unsigned>(static_cast<int64_t>(N) * L.T));
    if (vec)
        { ProfScope ps_("k_scan", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * (write_q ? 12u : 4u)); k_scan<true><<<grid, kThreads, 0, s>>>(logw, ld, P, L.T, kfx, ws, L.ldq, write_q ? 1 : 0, lse_out, ess_out); }
    else
        { ProfScope ps_("k_scan", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * (write_q ? 12u : 4u)); k_scan<false><<<grid, kThreads, 0, s>>>(logw, ld, P, L.T, kfx, ws, L.ldq, write_q ? 1 : 0, lse_out, ess_out); }
    ++*launches;
    return cudaPeekAtLastError();
}

// merged items per merge CTA: enough CTAs for ~10 per SM, at most 16 windows each
static int64_t merge_chunk(int32_t N, int32_t P) {
    const int64_t total = static_cast<int64_t>(N) * 2 * P;
    int64_t ch = cdiv(total, static_cast<int64_t>(sm_count()) * 10);
    ch = cdiv(ch, kWin) * kWin;
    return std::max<int64_t>(kWin, std::min<int64_t>(ch, 16 * kWin));
}

static uint64_t stratum_width(int32_t P) {
    const int m = ceil_log2(P);
    if ((P & (P - 1)) == 0) return uint64_t{1} << (64 - m);
    return UINT64_MAX / static_cast<uint64_t>(P);
}

// the multinomial's per-slot searches against Q and the bucket index (ws.Q, ws.bidx, ws.Qtot,
// ws.fstatus written by k_merge<ModeBuckets> after the scan, or by the cluster kernel's bucket mode)
cudaError_t launch_bsearch_buckets(int32_t N, int32_t P, const Layout& L, const Ws& ws, uint64_t seed,
                                   uint32_t first_filter, int32_t* anc, int64_t ld_anc, cudaStream_t s,
                                   uint64_t* launches) {
    const int lgNB = ceil_log2(P);
    {
        ProfScope ps_("k_bsearch", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 12u);  // Q read once, ancestors written
        k_bsearch_buckets<<<static_cast<unsigned>(grid_for(static_cast<int64_t>(N) * cdiv(P, 8), 8)), kThreads, 0,
                            s>>>(N, P, ws, L.ldq, L.ldb, lgNB, make_key(seed), first_filter, anc, ld_anc);
    }
    ++*launches;
    return cudaPeekAtLastError();
}

cudaError_t launch_search(int scheme, int32_t N, int32_t P, const Layout& L, const Ws& ws, uint64_t seed,
                          uint32_t first_filter, int32_t* anc, int64_t ld_anc, cudaStream_t s,
                          uint64_t* launches) {
    const Key key = make_key(seed);
    if (scheme == 1) {
        const int lgNB = ceil_log2(P);
        const int32_t NB = 1 << lgNB;
        const int64_t chunk = merge_chunk(N, P);
        const int cpf = static_cast<int>(cdiv(static_cast<int64_t>(NB) + P, chunk));
        ModeBuckets md{ws.Q, L.ldq, ws.Qtot, ws.fstatus, lgNB, NB, P, ws.bidx, L.ldb};
        {
            ProfScope ps_("k_merge_buckets", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 8u + static_cast<uint64_t>(N) * static_cast<uint64_t>(NB) * 4u);
            k_merge<ModeBuckets><<<static_cast<unsigned>(static_cast<int64_t>(N) * cpf), kThreads, 0, s>>>(md, cpf,
                                                                                                        chunk);
        }
        ++*launches;
        return launch_bsearch_buckets(N, P, L, ws, seed, first_filter, anc, ld_anc, s, launches);
    } else {
        const int64_t chunk = merge_chunk(N, P);
        const int cpf = static_cast<int>(cdiv(2 * static_cast<int64_t>(P), chunk));
        const dim3 grid(static_cast<unsigned>(static_cast<int64_t>(N) * cpf));
        if (scheme == 2) {
            ModeSorted<2> md{ws.Q, L.ldq, ws.Qtot, ws.fstatus, stratum_width(P), key, first_filter, P, anc, ld_anc};
            { ProfScope ps_("k_merge", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 12u); k_merge<ModeSorted<2>><<<grid, kThreads, 0, s>>>(md, cpf, chunk); }
        } else {
            ModeSorted<3> md{ws.Q, L.ldq, ws.Qtot, ws.fstatus, stratum_width(P), key, first_filter, P, anc, ld_anc};
            { ProfScope ps_("k_merge", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 12u); k_merge<ModeSorted<3>><<<grid, kThreads, 0, s>>>(md, cpf, chunk); }
        }
    }
    ++*launches;
    return cudaPeekAtLastError();
}

cudaError_t launch_metropolis(const float* logw, int64_t ld, int32_t N, int32_t P, const Layout& L,
                              const Ws& ws, uint64_t seed, uint32_t first_filter, int32_t B, int32_t* anc,
                              int64_t ld_anc, cudaStream_t s, uint64_t* launches) {
    const int64_t total = static_cast<int64_t>(N) * P;
    if (B > 0) {
        if (aligned16(logw) && ld % 4 == 0 && P % 4 == 0) {
            { ProfScope ps_("k_mexp_vec", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 8u); k_mexp_vec<<<static_cast<unsigned>(grid_for(total / 4)), kThreads, 0, s>>>(
                reinterpret_cast<const float4*>(logw), ld / 4, N, P / 4, ws, L.ldq / 4); }
        } else {
            { ProfScope ps_("k_mexp", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 8u); k_mexp<<<static_cast<unsigned>(grid_for(total)), kThreads, 0, s>>>(logw, ld, N, P, ws, L.ldq); }
        }
        ++*launches;
    }
    // batches that fill the GPU: the filter-per-CTA kernel (L1-resident weights; C3: 6.84 ->
    // 4.28 ms at B = 32, tools/metro_times.py); fewer filters: one thread per chain over all SMs
    const bool pow2 = P > 1 && (P & (P - 1)) == 0;
    const int sh = pow2 ? 32 - ceil_log2(P) : 0;
    if (N >= sm_count()) {
        ProfScope ps_("k_metro", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 8u);  // w read once, ancestors written
        const unsigned g = static_cast<unsigned>(std::min<int64_t>(N, sm_count()));
        if (pow2) k_metro_fpc<true><<<g, 1024, 0, s>>>(N, P, ws, L.ldq, make_key(seed), first_filter, B, anc, ld_anc, sh);
        else k_metro_fpc<false><<<g, 1024, 0, s>>>(N, P, ws, L.ldq, make_key(seed), first_filter, B, anc, ld_anc, 0);
    } else {
        ProfScope ps_("k_metro", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 8u);
        const unsigned g = static_cast<unsigned>(cdiv(total, kThreads));
        if (pow2) k_metro<true><<<g, kThreads, 0, s>>>(N, P, ws, L.ldq, make_key(seed), first_filter, B, anc, ld_anc, sh);
        else k_metro<false><<<g, kThreads, 0, s>>>(N, P, ws, L.ldq, make_key(seed), first_filter, B, anc, ld_anc, 0);
    }
    ++*launches;
    return cudaPeekAtLastError();
}

cudaError_t launch_normw(const float* logw, int64_t ld, int32_t N, int32_t P, const Ws& ws, float* normw,
                         cudaStream_t s, uint64_t* launches) {
    const int64_t total = static_cast<int64_t>(N) * P;
    { ProfScope ps_("k_normw", s); k_normw<<<static_cast<unsigned>(grid_for(total)), kThreads, 0, s>>>(logw, ld, N, P, ws, normw); }
    ++*launches;
    return cudaPeekAtLastError();
}

cudaError_t launch_identity(int32_t N, int32_t P, int32_t* anc, int64_t ld_anc, cudaStream_t s,
                            uint64_t* launches) {
    const int64_t total = static_cast<int64_t>(N) * P;
    { ProfScope ps_("k_identity", s); k_identity<<<static_cast<unsigned>(grid_for(total)), kThreads, 0, s>>>(N, P, anc, ld_anc); }
    ++*launches;
    return cudaPeekAtLastError();
}

cudaError_t launch_offspring(const int32_t* anc, int64_t ld_anc, int32_t N, int32_t P, int32_t* o, int64_t ld_o,
                             cudaStream_t s, uint64_t* launches) {
    if (N >= sm_count() / 2 && P >= 2 && P <= 65536) {
        const int half = (P + 1) / 2;
        const size_t smem = static_cast<size_t>(half) * 4;
        static std::atomic<int> attr_set[kMaxDevices];
        cached_per_device(attr_set, [] {
            cudaFuncSetAttribute(k_hist_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 * 4);
            return 1;
        });
        const int vec = ((reinterpret_cast<uintptr_t>(anc) & 15) == 0 && ld_anc % 4 == 0) ? 1 : 0;
        const unsigned g = static_cast<unsigned>(std::min<int64_t>(2LL * N, sm_count()));
        ProfScope ps_("k_hist", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 8u);
        k_hist_smem<<<g, kHistT, smem, s>>>(anc, ld_anc, N, P, o, ld_o, vec);
        ++*launches;
        return cudaPeekAtLastError();
    }
    cudaError_t e = cudaMemset2DAsync(o, static_cast<size_t>(ld_o) * 4, 0, static_cast<size_t>(P) * 4,
                                      static_cast<size_t>(N), s);
    if (e != cudaSuccess) return e;
    const int64_t total = static_cast<int64_t>(N) * P;
    const bool runs = (P % 4 == 0) && ((reinterpret_cast<uintptr_t>(anc) & 15) == 0) && (ld_anc % 4 == 0);
    if (runs) {
        const int64_t nblk = static_cast<int64_t>(N) * cdiv(P, 128);
        const unsigned g = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(cdiv(nblk, kThreads / 32),
                                                                                     sm_count() * 8)));
        ProfScope ps_("k_hist", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 8u);
        k_hist_runs<<<g, kThreads, 0, s>>>(anc, ld_anc, N, P, o, ld_o);
    } else {
        ProfScope ps_("k_hist", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 8u);
        k_hist<<<static_cast<unsigned>(grid_for(total, 16)), kThreads, 0, s>>>(anc, ld_anc, N, P, o, ld_o);
    }
    ++*launches;
    return cudaPeekAtLastError();
}

cudaError_t launch_permute_from_offspring(const int32_t* o, int64_t ld_o, int32_t N, int32_t P, const Layout& L,
                                         const Ws& ws, int32_t* perm, int64_t ld_perm, cudaStream_t s,
                                         uint64_t* launches) {
    const int o_vec = ((reinterpret_cast<uintptr_t>(o) & 15) == 0 && ld_o % 4 == 0) ? 1 : 0;
    { ProfScope ps_("k_pscan", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 12u);  // o read, permutation (survivors) + free list written
      k_pscan<<<static_cast<unsigned>(static_cast<int64_t>(N) * L.T), kThreads, 0, s>>>(P, L.T, ws, L.ldq, o, ld_o, o_vec, perm,
                                                                                     ld_perm); }
    ++*launches;
    {
        ProfScope ps_("k_push", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 8u);  // o and the free list read
        const int64_t nblk = static_cast<int64_t>(N) * cdiv(P, 128);
        const unsigned g = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(cdiv(nblk, kThreads / 32),
                                                                                     sm_count() * 8)));
        k_push<<<g, kThreads, 0, s>>>(N, P, ws, L.ldq, o, ld_o, o_vec, perm, ld_perm);
    }
    ++*launches;
    return cudaPeekAtLastError();
}

cudaError_t launch_permute(const int32_t* anc, int64_t ld_anc, int32_t N, int32_t P, const Layout& L,
                           const Ws& ws, int32_t* perm, int64_t ld_perm, cudaStream_t s, uint64_t* launches) {
    cudaError_t e = launch_offspring(anc, ld_anc, N, P, ws.o, L.ldq, s, launches);
    if (e != cudaSuccess) return e;
    return launch_permute_from_offspring(ws.o, L.ldq, N, P, L, ws, perm, ld_perm, s, launches);
}

cudaError_t launch_gather_inplace(void* X, int64_t row_bytes, int64_t ld_bytes, int64_t ld_filter_bytes, int32_t N,
                                  int32_t P, const int32_t* perm, int64_t ld_perm, cudaStream_t s,
                                  uint64_t* launches) {
    char* x = static_cast<char*>(X);
    const bool a16 = aligned16(x) && row_bytes % 16 == 0 && ld_bytes % 16 == 0 && ld_filter_bytes % 16 == 0;
    const bool a4 = (reinterpret_cast<uintptr_t>(x) & 3) == 0 && row_bytes % 4 == 0 && ld_bytes % 4 == 0 &&
                    ld_filter_bytes % 4 == 0;
    const int ch = a16 ? 16 : (a4 ? 4 : 1);
    const int64_t cpr = row_bytes / ch;
    const int64_t total = static_cast<int64_t>(N) * P * cpr;
    const unsigned grid = static_cast<unsigned>(grid_for(total, 16));
    const bool vec_perm = ((reinterpret_cast<uintptr_t>(perm) & 15) == 0 && ld_perm % 4 == 0 && P % 4 == 0);
    if (ch == 16 && cpr <= 64 && vec_perm) {
        const int64_t nblk = static_cast<int64_t>(N) * cdiv(P, 128);
        const unsigned g2 = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(cdiv(nblk, kThreads / 32),
                                                                                      sm_count() * 8)));
        ProfScope ps_("k_gather_inplace", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 4u, 2u * static_cast<uint64_t>(row_bytes));
        k_gather_rows16<<<g2, kThreads, 0, s>>>(x, ld_bytes, ld_filter_bytes, N, P, static_cast<int>(cpr), perm,
                                                ld_perm);
    }
    else if (ch == 16) { ProfScope ps_("k_gather_inplace", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 4u, 2u * static_cast<uint64_t>(row_bytes)); k_gather_inplace<16><<<grid, kThreads, 0, s>>>(x, ld_bytes, ld_filter_bytes, N, P, cpr, perm, ld_perm); }
    else if (ch == 4) { ProfScope ps_("k_gather_inplace", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 4u, 2u * static_cast<uint64_t>(row_bytes)); k_gather_inplace<4><<<grid, kThreads, 0, s>>>(x, ld_bytes, ld_filter_bytes, N, P, cpr, perm, ld_perm); }
    else { ProfScope ps_("k_gather_inplace", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 4u, 2u * static_cast<uint64_t>(row_bytes)); k_gather_inplace<1><<<grid, kThreads, 0, s>>>(x, ld_bytes, ld_filter_bytes, N, P, cpr, perm, ld_perm); }
    ++*launches;
    return cudaPeekAtLastError();
}

cudaError_t launch_gather_out(const void* X, void* Y, int64_t row_bytes, int64_t ld_x, int64_t ld_y, int32_t P,
                              const int32_t* anc, cudaStream_t s, uint64_t* launches) {
    const char* x = static_cast<const char*>(X);
    char* y = static_cast<char*>(Y);
    const bool a16 = aligned16(x) && aligned16(y) && row_bytes % 16 == 0 && ld_x % 16 == 0 && ld_y % 16 == 0;
    const bool a4 = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 3) == 0 &&
                    row_bytes % 4 == 0 && ld_x % 4 == 0 && ld_y % 4 == 0;
    const int ch = a16 ? 16 : (a4 ? 4 : 1);
    const int64_t cpr = row_bytes / ch;
    const int64_t total = static_cast<int64_t>(P) * cpr;
    const unsigned grid = static_cast<unsigned>(grid_for(total, 16));
    if (ch == 16) { ProfScope ps_("k_gather_out", s, static_cast<uint64_t>(P) * (4u + 2u * static_cast<uint64_t>(row_bytes))); k_gather_out<16><<<grid, kThreads, 0, s>>>(x, y, ld_x, ld_y, P, cpr, anc); }
    else if (ch == 4) { ProfScope ps_("k_gather_out", s, static_cast<uint64_t>(P) * (4u + 2u * static_cast<uint64_t>(row_bytes))); k_gather_out<4><<<grid, kThreads, 0, s>>>(x, y, ld_x, ld_y, P, cpr, anc); }
    else { ProfScope ps_("k_gather_out", s, static_cast<uint64_t>(P) * (4u + 2u * static_cast<uint64_t>(row_bytes))); k_gather_out<1><<<grid, kThreads, 0, s>>>(x, y, ld_x, ld_y, P, cpr, anc); }
    ++*launches;
    return cudaPeekAtLastError();
}

// ---------------------------------------------------------------- shard launchers
cudaError_t launch_shard_search(int scheme, const uint64_t* Q, int32_t Pl, int64_t p0, int64_t P_global,
                                const uint64_t* totals, int nshards, int shard, const float* gmax,
                                const int32_t* gbad, uint64_t seed, uint32_t filt, int32_t* anc,
                                int64_t* range_out, void* ctx_mem, cudaStream_t s, uint64_t* launches) {
    const Key key = make_key(seed);
    ShardCtxDev* dctx = static_cast<ShardCtxDev*>(ctx_mem);
    const uint64_t D = (P_global <= 1) ? 0 : stratum_width(static_cast<int32_t>(P_global));
    // the range kernel evaluates sorted positions; multinomial only needs the offsets from it
    {
        ProfScope ps_("k_shard_range", s);
        if (scheme == 2) k_shard_range<2><<<1, 32, 0, s>>>(totals, nshards, shard, gmax, gbad, P_global, D, key, filt, dctx, range_out);
        else k_shard_range<3><<<1, 32, 0, s>>>(totals, nshards, shard, gmax, gbad, P_global, D, key, filt, dctx, range_out);
    }
    ++*launches;
    if (scheme == 1) {
        ProfScope ps_("k_shard_multinomial", s, static_cast<uint64_t>(Pl) * 12u);
        k_shard_multinomial<<<static_cast<unsigned>(grid_for((P_global + 1) / 2, 8)), kThreads, 0, s>>>(
            Q, Pl, p0, P_global, dctx, key, filt, anc);
        ++*launches;
        return cudaPeekAtLastError();
    }
    const int64_t chunk = merge_chunk(1, static_cast<int32_t>(std::min<int64_t>(P_global, INT32_MAX / 2)));
    const int cpf = static_cast<int>(cdiv(P_global + Pl, chunk));
    if (scheme == 2) {
        ModeShard<2> md{Q, dctx, D, key, filt, Pl, p0, anc};
        ProfScope ps_("k_merge", s, static_cast<uint64_t>(Pl) * 12u);  // Q read, ~Pl slots written
        k_merge<ModeShard<2>><<<static_cast<unsigned>(cpf), kThreads, 0, s>>>(md, cpf, chunk);
    } else {
        ModeShard<3> md{Q, dctx, D, key, filt, Pl, p0, anc};
        ProfScope ps_("k_merge", s, static_cast<uint64_t>(Pl) * 12u);
        k_merge<ModeShard<3>><<<static_cast<unsigned>(cpf), kThreads, 0, s>>>(md, cpf, chunk);
    }
    ++*launches;
    return cudaPeekAtLastError();
}

cudaError_t launch_shard_weights(const float* logw, int32_t Pl, const float* gmax, float* w, cudaStream_t s,
                                 uint64_t* launches) {
    ProfScope ps_("k_shard_weights", s, static_cast<uint64_t>(Pl) * 8u);
    k_shard_weights<<<static_cast<unsigned>(grid_for(Pl)), kThreads, 0, s>>>(logw, Pl, gmax, w);
    ++*launches;
    return cudaPeekAtLastError();
}

cudaError_t launch_metro_slots(const float* w, int64_t P_global, int64_t slot0, int32_t nslots, uint64_t seed,
                               int32_t B, uint32_t filt, const float* gmax, const int32_t* gbad, int32_t* anc,
                               cudaStream_t s, uint64_t* launches) {
    ProfScope ps_("k_metro_slots", s, static_cast<uint64_t>(nslots) * 8u);
    k_metro_slots<<<static_cast<unsigned>(cdiv(nslots, kThreads)), kThreads, 0, s>>>(w, P_global, slot0, nslots,
                                                                                     make_key(seed), filt, B, gmax,
                                                                                     gbad, anc);
    ++*launches;
    return cudaPeekAtLastError();
}

size_t shard_ctx_bytes() { return sizeof(ShardCtxDev); }

// ---------------------------------------------------------------- a6 shard launchers
cudaError_t launch_spacings_total(int64_t P_global, int nshards, int shard, uint64_t seed, uint32_t filt,
                                  uint64_t* etot, cudaStream_t s, uint64_t* launches) {
    const int64_t k0 = spacing_shard_begin(P_global, nshards, shard);
    const int64_t k1 = spacing_shard_begin(P_global, nshards, shard + 1);
    cudaError_t e = cudaMemsetAsync(etot, 0, sizeof(uint64_t), s);
    if (e != cudaSuccess || k1 <= k0) return e;
    const int64_t groups = ((k1 + 3) >> 2) - (k0 >> 2);
    {
        ProfScope ps_("k_spacings_total", s);
        k_spacings_total<<<static_cast<unsigned>(grid_for(groups, 8)), kThreads, 0, s>>>(
            k0, k1, make_key(seed), filt, reinterpret_cast<unsigned long long*>(etot));
    }
    ++*launches;
    return cudaPeekAtLastError();
}

struct SpacShardLayout {
    size_t ctx, ctr, status, G, zero_begin, zero_end, total;
};

static SpacShardLayout spac_shard_layout(int64_t P_global) {
    SpacShardLayout L{};
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align_up(off + bytes, 256);
        return o;
    };
    L.ctx = take(sizeof(SpacShardDev));
    L.zero_begin = off;
    L.ctr = take(sizeof(uint32_t));
    L.status = take(sizeof(uint64_t) * static_cast<size_t>(cdiv(P_global, kTile)));
    L.zero_end = off;
    L.G = take(sizeof(uint64_t) * static_cast<size_t>(P_global));
    L.total = off;
    return L;
}

size_t spac_shard_workspace_bytes(int64_t P_global) { return spac_shard_layout(P_global).total; }

// slot shard of rank `shard`: [shard ceil(P/G), ...) as shard_range in paper_1202_6163_b200/shard.py
static void route_slots(int64_t P_global, int nshards, int shard, int64_t* k0, int64_t* k1) {
    const int64_t per = (P_global + nshards - 1) / nshards;
    *k0 = std::min<int64_t>(P_global, static_cast<int64_t>(shard) * per);
    *k1 = std::min<int64_t>(P_global, *k0 + per);
}

cudaError_t launch_route(const uint64_t* totals, int nshards, int shard, const float* gmax, const int32_t* gbad,
                         int64_t P_global, uint64_t seed, uint32_t filt, int64_t* counts, int64_t* cursor,
                         uint64_t* send_x, int32_t* send_k, cudaStream_t s, uint64_t* launches) {
    int64_t k0, k1;
    route_slots(P_global, nshards, shard, &k0, &k1);
    const int64_t pairs = std::max<int64_t>(1, ((k1 + 1) >> 1) - (k0 >> 1));
    const unsigned grid = static_cast<unsigned>(grid_for(pairs, 4));
    cudaError_t e = cudaMemsetAsync(cursor ? cursor : counts, 0, sizeof(int64_t) * nshards, s);
    if (e != cudaSuccess) return e;
    {
        ProfScope ps_(cursor ? "k_route_pack" : "k_route_count", s, cursor ? static_cast<uint64_t>(k1 - k0) * 12u : 0u);
        k_route<<<grid, kThreads, 0, s>>>(totals, nshards, gmax, gbad, P_global, k0, k1, make_key(seed), filt,
                                          reinterpret_cast<unsigned long long*>(counts),
                                          reinterpret_cast<unsigned long long*>(cursor), send_x, send_k);
    }
    ++*launches;
    return cudaPeekAtLastError();
}

cudaError_t launch_route_search(const uint64_t* Q, int32_t Pl, int64_t p0, const uint64_t* totals, int nshards,
                                int shard, const float* gmax, const int32_t* gbad, const uint64_t* rx,
                                const int32_t* rk, int64_t nrecv, int32_t* anc, cudaStream_t s, uint64_t* launches) {
    const unsigned grid = static_cast<unsigned>(grid_for(std::max<int64_t>(std::max<int64_t>(nrecv, Pl), 1), 4));
    {
        ProfScope ps_("k_route_search", s, static_cast<uint64_t>(nrecv) * 16u);  // (x, k) read, ancestor written
        k_route_search<<<grid, kThreads, 0, s>>>(Q, Pl, p0, totals, nshards, shard, gmax, gbad, rx, rk, nrecv, anc);
    }
    ++*launches;
    return cudaPeekAtLastError();
}

cudaError_t launch_shard_search_sorted(const uint64_t* Q, int32_t Pl, int64_t p0, int64_t P_global,
                                       const uint64_t* totals, const uint64_t* etotals, int nshards, int shard,
                                       const float* gmax, const int32_t* gbad, uint64_t seed, uint32_t filt,
                                       int32_t* anc, int64_t* range_out, void* ws, cudaStream_t s,
                                       uint64_t* launches) {
    const SpacShardLayout L = spac_shard_layout(P_global);
    char* b = static_cast<char*>(ws);
    SpacShardDev* dctx = reinterpret_cast<SpacShardDev*>(b + L.ctx);
    uint64_t* G = reinterpret_cast<uint64_t*>(b + L.G);
    const Key key = make_key(seed);
    cudaError_t e = cudaMemsetAsync(b + L.zero_begin, 0, L.zero_end - L.zero_begin, s);
    if (e != cudaSuccess) return e;
    { ProfScope ps_("k_spac_shard_plan", s); k_spac_shard_plan<<<1, 32, 0, s>>>(totals, etotals, nshards, shard, gmax, gbad, P_global, dctx); }
    ++*launches;
    {
        ProfScope ps_("k_gscan_range", s);
        const int64_t grid = std::min<int64_t>(static_cast<int64_t>(sm_count()) * 4, std::max<int64_t>(1, cdiv(P_global, kTile)));
        k_gscan_range<<<static_cast<unsigned>(grid), kThreads, 0, s>>>(dctx, key, filt,
                                                                      reinterpret_cast<uint32_t*>(b + L.ctr),
                                                                      reinterpret_cast<uint64_t*>(b + L.status), G);
    }
    ++*launches;
    { ProfScope ps_("k_spac_shard_range", s); k_spac_shard_range<<<1, 32, 0, s>>>(dctx, G, P_global, nshards, range_out); }
    ++*launches;
    const int64_t chunk = merge_chunk(1, static_cast<int32_t>(std::min<int64_t>(P_global, INT32_MAX / 2)));
    const int cpf = static_cast<int>(cdiv(P_global + Pl, chunk));
    ModeShardSpacings md{Q, dctx, G, Pl, p0, anc};
    {
        ProfScope ps_("k_merge", s, static_cast<uint64_t>(Pl) * 20u);  // Q and G read, ~Pl slots written
        k_merge<ModeShardSpacings><<<static_cast<unsigned>(cpf), kThreads, 0, s>>>(md, cpf, chunk);
    }
    ++*launches;
    return cudaPeekAtLastError();
}

cudaError_t launch_sorted_multinomial(int32_t N, int32_t P, const Layout& L, const Ws& ws, uint64_t seed,
                                      uint32_t first_filter, int32_t* anc, int64_t ld_anc, cudaStream_t s,
                                      uint64_t* launches, bool spacings_only) {
    const Key key = make_key(seed);
    if (spacings_only) {
        ProfScope ps_("k_gscan", s, (static_cast<uint64_t>(N) * static_cast<uint64_t>(P) + N) * 8u);  // G_0..G_P written
        k_gscan<<<static_cast<unsigned>(static_cast<int64_t>(N) * L.T2), kThreads, 0, s>>>(P, L.T2, ws, L.ldg, key,
                                                                                          first_filter);
        ++*launches;
        return cudaPeekAtLastError();
    }
    const int64_t chunk = merge_chunk(N, P);
    const int cpf = static_cast<int>(cdiv(2 * static_cast<int64_t>(P), chunk));
    ModeSpacings md{ws.Q, L.ldq, ws.Qtot, ws.fstatus, ws.G, L.ldg, ws.Gtot, P, anc, ld_anc};
    {
        ProfScope ps_("k_merge_spacings", s, static_cast<uint64_t>(N) * static_cast<uint64_t>(P) * 20u);  // Q and G read, ancestors written
        k_merge<ModeSpacings><<<static_cast<unsigned>(static_cast<int64_t>(N) * cpf), kThreads, 0, s>>>(md, cpf,
                                                                                                     chunk);
    }
    ++*launches;
    return cudaPeekAtLastError();
}

cudaError_t launch_lg_init(float* X, int64_t ld, int32_t P, int32_t D, float phi, float sigma_x, uint64_t seed,
                           cudaStream_t s, uint64_t* launches) {
    const float sd = sigma_x / sqrtf(1.0f - phi * phi);
    ProfScope ps_("k_lg_init", s);
    k_lg_init<<<static_cast<unsigned>(cdiv(P, kThreads)), kThreads, 0, s>>>(X, ld, P, D, sd, make_key(seed));
    ++*launches;
    return cudaPeekAtLastError();
}

cudaError_t launch_lg_step(float* X, int64_t ld, int32_t P, int32_t D, float phi, float sigma_x, float sigma_y,
                           float y, uint64_t seed, int32_t t, float* logw, cudaStream_t s, uint64_t* launches) {
    const int vec = ((reinterpret_cast<uintptr_t>(X) & 15) == 0 && ld % 4 == 0) ? 1 : 0;
    ProfScope ps_("k_lg_step", s);
    k_lg_step<<<static_cast<unsigned>(cdiv(P, kThreads)), kThreads, 0, s>>>(
        X, ld, P, D, phi, sigma_x, 0.5f / (sigma_y * sigma_y), y, make_key(seed), t, logw, vec);
    ++*launches;
    return cudaPeekAtLastError();
}

cudaError_t launch_lg_accumulate(const double* lse, int32_t P, float sigma_y, double* loglik, cudaStream_t s,
                                 uint64_t* launches) {
    const double c = std::log(static_cast<double>(P)) +
                     0.5 * std::log(2.0 * 3.14159265358979323846 * static_cast<double>(sigma_y) * sigma_y);
    ProfScope ps_("k_lg_accumulate", s);
    k_lg_accumulate<<<1, 32, 0, s>>>(lse, c, loglik);
    ++*launches;
    return cudaPeekAtLastError();
}

}  // namespace pf
