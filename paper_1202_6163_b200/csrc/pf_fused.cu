// pf_fused.cu — one-launch resampler for batches of small/medium filters.
//
// One thread-block CLUSTER per filter (CL = ceil(P / 16384) CTAs, <= 8), a
// persistent loop over filters.  CTA c of the cluster owns particles
// [c*PP, (c+1)*PP) and keeps their inclusive fixed-point cumulative weights
// Q_i (NS-5) in shared memory (PP <= 16384 -> <= 128 KiB).  Per filter:
//   A  log-weights -> registers (float4, coalesced); local max; cluster max
//      through DSMEM (a1, NS-1/NS-2)
//   B  w = dexp, q = trunc(w 2^kfx) (a2, NS-3..NS-5); block scan in
//      registers + shared memory; cluster exchange of the CTA totals gives
//      the CTA's offset O_c and the filter total Q (a3, the "collective
//      prefix-sum" of P:125-128, here inside one launch); lse / ESS /
//      normalised weights fused (a12)
//   C  slots whose positions fall in [O_c, O_c + T_c) form a contiguous range
//      [k_lo, k_hi) (positions are sorted, NS-9/NS-10), found by a
//      warp-parallel search over k; each thread takes 16 consecutive slots,
//      generates their positions (Philox, NS-6) and finds a_k = min{i : Q_i >
//      x_k} by a binary search for the first slot and a galloping search from
//      the previous answer for the rest (a4+a5).
// HBM traffic: 4 B/particle in (logw) + 4 B out (ancestors) (+4 B normw).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "pf_device.cuh"
#include "pf_internal.h"

namespace cg = cooperative_groups;

namespace pf {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kFT = 512;               // threads per CTA
constexpr int kFW = kFT / 32;          // warps per CTA
constexpr int kFI = 32;                // particles per thread
constexpr int kFR = kFI / 4;           // float4 rows per thread
constexpr int kPP = kFT * kFI;         // 16384 particles per CTA (max)
constexpr int kSlotsPerThread = 16;

struct Exchange {
    float m;
    int bad;
    uint64_t tot;
    double sw, sw2;
};

struct FusedArgs {
    const float* logw;
    int64_t ld;
    int32_t N, P, CL, PP;
    uint64_t D;
    Key key;
    uint32_t filt0;
    int kfx;
    int vec;  // logw rows 16-byte aligned and PP % 4 == 0
    int32_t* anc;
    int64_t ld_anc;
    int anc_vec;  // ancestor rows 16-byte aligned
    double* lse_out;
    double* ess_out;
    float* normw;
    int32_t* status_out;
};

template <int SCHEME>
__device__ __forceinline__ uint64_t position(const FusedArgs& a, uint32_t filt, uint64_t Qtot, uint64_t rho,
                                             int64_t k) {
    if (SCHEME == 2) {
        const u32x4 r = philox10(static_cast<uint32_t>(k >> 1), 0u, 2u, filt, a.key.k0, a.key.k1);
        rho = mulhi64((k & 1) ? hi_word(r) : lo_word(r), a.D);
    }
    return mulhi64(static_cast<uint64_t>(k) * a.D + rho, Qtot);
}

// #{k in [0, P) : x_k < v} by a 32-ary warp search (x_k nondecreasing in k).
template <int SCHEME>
__device__ int64_t count_below(const FusedArgs& a, uint32_t filt, uint64_t Qtot, uint64_t rho, uint64_t v,
                               int lane) {
    int64_t lo = 0, hi = a.P;
    while (hi > lo) {
        const int64_t step = (hi - lo + 31) / 32;
        const int64_t m = lo + lane * step;
        const bool p = (m < hi) && (position<SCHEME>(a, filt, Qtot, rho, m) < v);
        const int L = __popc(__ballot_sync(kFull, p));
        const int64_t nlo = (L == 0) ? lo : lo + static_cast<int64_t>(L - 1) * step + 1;
        const int64_t mL = lo + static_cast<int64_t>(L) * step;
        hi = (mL < hi) ? mL : hi;
        lo = nlo;
    }
    return lo;
}

template <int SCHEME>
__global__ void __launch_bounds__(kFT, 1) k_fused_sorted(FusedArgs a) {
    extern __shared__ __align__(16) uint64_t sQ[];
    __shared__ Exchange s_x;
    __shared__ float s_f[kFW];
    __shared__ int s_i[kFW];
    __shared__ double s_d[2][kFW];
    __shared__ uint64_t s_wt[kFR][kFW];
    __shared__ float s_lmax;
    __shared__ int s_bad;
    __shared__ uint64_t s_off, s_tot, s_Qtot;
    __shared__ double s_S, s_S2;
    __shared__ int64_t s_k[2];

    cg::cluster_group cluster = cg::this_cluster();
    const int c = static_cast<int>(cluster.block_rank());
    const int CL = a.CL;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int num_clusters = gridDim.x / CL;
    const int cid = blockIdx.x / CL;

    for (int n = cid; n < a.N; n += num_clusters) {
        const int64_t p0 = static_cast<int64_t>(c) * a.PP;
        const int64_t p1 = min(static_cast<int64_t>(a.P), p0 + a.PP);
        const int np = static_cast<int>(max(int64_t{0}, p1 - p0));
        const float* row = a.logw + static_cast<int64_t>(n) * a.ld + p0;
        const uint32_t filt = a.filt0 + static_cast<uint32_t>(n);

        // ---------------- A: load + max
        float v[kFI];
#pragma unroll
        for (int j = 0; j < kFR; ++j) {
            const int i0 = j * (kFT * 4) + tid * 4;
            if (a.vec && i0 + 3 < np) {
                const float4 t = __ldcs(reinterpret_cast<const float4*>(row + i0));
                v[j * 4 + 0] = t.x; v[j * 4 + 1] = t.y; v[j * 4 + 2] = t.z; v[j * 4 + 3] = t.w;
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) v[j * 4 + q] = (i0 + q < np) ? __ldcs(row + i0 + q) : -INFINITY;
            }
        }
        float m = -INFINITY;
        int bad = 0;
#pragma unroll
        for (int t = 0; t < kFI; ++t) {
            if (isnan(v[t]) || v[t] == INFINITY) bad = 1;
            else m = fmaxf(m, v[t]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
            bad |= __shfl_xor_sync(kFull, bad, o);
        }
        if (lane == 0) { s_f[warp] = m; s_i[warp] = bad; }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < kFW; ++w) { m = fmaxf(m, s_f[w]); bad |= s_i[w]; }
            s_x.m = m;
            s_x.bad = bad;
        }
        cluster.sync();  // #1
        if (tid == 0) {
            float gm = -INFINITY;
            int gb = 0;
            for (int r = 0; r < CL; ++r) {
                const Exchange* rx = cluster.map_shared_rank(&s_x, r);
                gm = fmaxf(gm, rx->m);
                gb |= rx->bad;
            }
            s_lmax = gm;
            s_bad = (gb || gm == -INFINITY) ? 1 : 0;
        }
        __syncthreads();
        if (s_bad) {
            // NS-1: invalid filter -> identity ancestors, NaN side outputs
            int32_t* arow = a.anc + static_cast<int64_t>(n) * a.ld_anc;
            for (int64_t k = p0 + tid; k < p1; k += kFT) arow[k] = static_cast<int32_t>(k);
            if (a.normw)
                for (int64_t k = p0 + tid; k < p1; k += kFT) a.normw[static_cast<int64_t>(n) * a.P + k] = NAN;
            if (c == 0 && tid == 0) {
                if (a.lse_out) a.lse_out[n] = NAN;
                if (a.ess_out) a.ess_out[n] = NAN;
                if (a.status_out) a.status_out[n] = 1;
            }
            cluster.sync();  // readers of s_x.m are done before the next filter writes it
            continue;
        }
        const float lm = s_lmax;

        // ---------------- B: weights, quantise, block scan, cluster offsets
        double sw = 0.0, sw2 = 0.0;
        uint64_t rs[kFR];
#pragma unroll
        for (int j = 0; j < kFR; ++j) {
            uint64_t loc = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float w = weight(v[j * 4 + q], lm);
                v[j * 4 + q] = w;
                sw += static_cast<double>(w);
                sw2 += static_cast<double>(w) * static_cast<double>(w);
                loc += quantise(w, a.kfx);
            }
            rs[j] = loc;
        }
        uint64_t ex[kFR];
#pragma unroll
        for (int j = 0; j < kFR; ++j) {
            const uint64_t incl = warp_incl_scan_u64(rs[j], lane);
            ex[j] = incl - rs[j];
            const uint64_t wt = __shfl_sync(kFull, incl, 31);
            if (lane == 0) s_wt[j][warp] = wt;
        }
        sw = warp_sum_f64(sw);
        sw2 = warp_sum_f64(sw2);
        if (lane == 0) { s_d[0][warp] = sw; s_d[1][warp] = sw2; }
        __syncthreads();
        if (warp == 0) {
            // exclusive scan of the kFR x kFW warp totals in (row, warp) order: 4 per lane
            uint64_t t4[4];
            uint64_t tsum = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int idx = lane * 4 + q;
                t4[q] = s_wt[idx / kFW][idx % kFW];
                tsum += t4[q];
            }
            const uint64_t incl = warp_incl_scan_u64(tsum, lane);
            uint64_t run = incl - tsum;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int idx = lane * 4 + q;
                s_wt[idx / kFW][idx % kFW] = run;
                run += t4[q];
            }
            if (lane == 31) s_tot = incl;
            if (lane == 0) {
                double A = 0.0, Bv = 0.0;
                for (int w = 0; w < kFW; ++w) { A += s_d[0][w]; Bv += s_d[1][w]; }
                s_x.sw = A;
                s_x.sw2 = Bv;
            }
        }
        __syncthreads();
        if (tid == 0) s_x.tot = s_tot;
        cluster.sync();  // #2
        if (tid == 0) {
            uint64_t off = 0, tot = 0;
            double S = 0.0, S2 = 0.0;
            for (int r = 0; r < CL; ++r) {
                const Exchange* rx = cluster.map_shared_rank(&s_x, r);
                if (r < c) off += rx->tot;
                tot += rx->tot;
                S += rx->sw;
                S2 += rx->sw2;
            }
            s_off = off;
            s_Qtot = tot;
            s_S = S;
            s_S2 = S2;
        }
        __syncthreads();
        const uint64_t O = s_off;
        const uint64_t Qtot = s_Qtot;
        // inclusive Q into shared memory (natural order)
#pragma unroll
        for (int j = 0; j < kFR; ++j) {
            const int i0 = j * (kFT * 4) + tid * 4;
            uint64_t run = O + s_wt[j][warp] + ex[j];
            uint64_t q4[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                run += quantise(v[j * 4 + q], a.kfx);
                q4[q] = run;
            }
            if (i0 + 3 < np) {
                reinterpret_cast<ulonglong2*>(sQ + i0)[0] = make_ulonglong2(q4[0], q4[1]);
                reinterpret_cast<ulonglong2*>(sQ + i0)[1] = make_ulonglong2(q4[2], q4[3]);
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (i0 + q < np) sQ[i0 + q] = q4[q];
            }
        }
        if (a.normw) {
            const double S = s_S;
            float* nrow = a.normw + static_cast<int64_t>(n) * a.P + p0;
#pragma unroll
            for (int j = 0; j < kFR; ++j) {
                const int i0 = j * (kFT * 4) + tid * 4;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (i0 + q < np) nrow[i0 + q] = static_cast<float>(static_cast<double>(v[j * 4 + q]) / S);
            }
        }
        if (c == 0 && tid == 0) {
            if (a.lse_out) a.lse_out[n] = static_cast<double>(lm) + log(s_S);
            if (a.ess_out) a.ess_out[n] = s_S * s_S / s_S2;
            if (a.status_out) a.status_out[n] = 0;
        }

        // ---------------- C: slots of this CTA and their ancestors
        uint64_t rho = 0;
        if (SCHEME == 3) rho = mulhi64(lo_word(philox10(0u, 0u, 3u, filt, a.key.k0, a.key.k1)), a.D);
        if (a.P == 1) {
            if (tid == 0) a.anc[static_cast<int64_t>(n) * a.ld_anc] = 0;
        } else if (np > 0) {
            if (warp < 2) {
                int64_t k;
                if (warp == 0) k = (c == 0) ? 0 : count_below<SCHEME>(a, filt, Qtot, rho, O, lane);
                else k = (c == CL - 1 || p1 == a.P) ? a.P : count_below<SCHEME>(a, filt, Qtot, rho, O + s_tot, lane);
                if (lane == 0) s_k[warp] = k;
            }
            __syncthreads();
            const int64_t k_lo = s_k[0], k_hi = s_k[1];
            int32_t* arow = a.anc + static_cast<int64_t>(n) * a.ld_anc;
            const int64_t b_first = k_lo / kSlotsPerThread;
            const int64_t b_last = (k_hi + kSlotsPerThread - 1) / kSlotsPerThread;  // exclusive
            for (int64_t b = b_first + tid; b < b_last; b += kFT) {
                const int64_t kb = b * kSlotsPerThread;
                uint64_t x[kSlotsPerThread];
                if (SCHEME == 2) {
#pragma unroll
                    for (int t = 0; t < kSlotsPerThread; t += 2) {
                        const u32x4 r = philox10(static_cast<uint32_t>((kb + t) >> 1), 0u, 2u, filt, a.key.k0,
                                                 a.key.k1);
                        x[t] = mulhi64(static_cast<uint64_t>(kb + t) * a.D + mulhi64(lo_word(r), a.D), Qtot);
                        x[t + 1] = mulhi64(static_cast<uint64_t>(kb + t + 1) * a.D + mulhi64(hi_word(r), a.D), Qtot);
                    }
                } else {
#pragma unroll
                    for (int t = 0; t < kSlotsPerThread; ++t)
                        x[t] = mulhi64(static_cast<uint64_t>(kb + t) * a.D + rho, Qtot);
                }
                int32_t out[kSlotsPerThread];
                int cur = -1;  // local index of the previous answer
#pragma unroll
                for (int t = 0; t < kSlotsPerThread; ++t) {
                    const int64_t k = kb + t;
                    out[t] = 0;
                    if (k < k_lo || k >= k_hi) continue;
                    const uint64_t xv = x[t];
                    int lo, hi;
                    if (cur < 0) {
                        lo = 0;
                        hi = np - 1;
                    } else if (sQ[cur] > xv) {
                        lo = hi = cur;
                    } else {
                        // gallop: find hi with sQ[hi] > xv
                        int step = 1;
                        lo = cur + 1;
                        hi = min(cur + step, np - 1);
                        while (hi < np - 1 && sQ[hi] <= xv) {
                            lo = hi + 1;
                            step <<= 1;
                            hi = min(cur + step, np - 1);
                        }
                    }
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (sQ[mid] > xv) hi = mid;
                        else lo = mid + 1;
                    }
                    cur = lo;
                    out[t] = static_cast<int32_t>(p0 + lo);
                }
                if (a.anc_vec && kb >= k_lo && kb + kSlotsPerThread <= k_hi) {
                    int4* dst = reinterpret_cast<int4*>(arow + kb);
#pragma unroll
                    for (int t = 0; t < kSlotsPerThread; t += 4)
                        __stcs(dst + t / 4, make_int4(out[t], out[t + 1], out[t + 2], out[t + 3]));
                } else {
#pragma unroll
                    for (int t = 0; t < kSlotsPerThread; ++t)
                        if (kb + t >= k_lo && kb + t < k_hi) arow[kb + t] = out[t];
                }
            }
        }
        __syncthreads();  // sQ and s_k are reused by the next filter
    }
    cluster.sync();  // keep this CTA's shared memory alive for remote readers
}

int device_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

template <int SCHEME>
cudaError_t launch_fused_t(const FusedArgs& a, cudaStream_t s) {
    const size_t smem = static_cast<size_t>(a.PP) * sizeof(uint64_t);
    auto kern = k_fused_sorted<SCHEME>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kPP * static_cast<int>(sizeof(uint64_t)));
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
        attr_set = true;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = a.CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kFT, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(a.CL, 1, 1);
    int max_clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1) {
        cudaGetLastError();
        max_clusters = std::max(1, device_sms() / a.CL);
    }
    const int clusters = std::max(1, std::min(a.N, max_clusters));
    cfg.gridDim = dim3(static_cast<unsigned>(clusters * a.CL), 1, 1);
    return cudaLaunchKernelEx(&cfg, kern, a);
}

}  // namespace

bool fused_supported(int scheme, int32_t P) {
    return (scheme == 2 || scheme == 3) && P >= 1 && P <= 8 * kPP;
}

cudaError_t launch_fused_sorted(int scheme, const float* logw, int64_t ld, int32_t N, int32_t P, uint64_t seed,
                                uint32_t first_filter, int32_t* anc, int64_t ld_anc, double* lse_out,
                                double* ess_out, float* normw, int32_t* status_out, cudaStream_t s,
                                uint64_t* launches) {
    FusedArgs a{};
    a.logw = logw;
    a.ld = ld;
    a.N = N;
    a.P = P;
    a.CL = static_cast<int32_t>((P + kPP - 1) / kPP);
    int64_t pp = (P + a.CL - 1) / a.CL;
    pp = (pp + 3) / 4 * 4;
    a.PP = static_cast<int32_t>(pp);
    const int m = ceil_log2(P);
    a.D = (P <= 1) ? 0 : (((P & (P - 1)) == 0) ? (uint64_t{1} << (64 - m)) : (UINT64_MAX / static_cast<uint64_t>(P)));
    a.key = make_key(seed);
    a.filt0 = first_filter;
    a.kfx = 61 - m;
    a.vec = ((reinterpret_cast<uintptr_t>(logw) & 15) == 0 && ld % 4 == 0) ? 1 : 0;
    a.anc = anc;
    a.ld_anc = ld_anc;
    a.anc_vec = ((reinterpret_cast<uintptr_t>(anc) & 15) == 0 && ld_anc % 4 == 0) ? 1 : 0;
    a.lse_out = lse_out;
    a.ess_out = ess_out;
    a.normw = normw;
    a.status_out = status_out;
    ProfScope ps_("k_fused_sorted", s);
    cudaError_t e = (scheme == 2) ? launch_fused_t<2>(a, s) : launch_fused_t<3>(a, s);
    ++*launches;
    if (e != cudaSuccess) return e;
    return cudaPeekAtLastError();
}

}  // namespace pf
