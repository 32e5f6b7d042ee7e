// tools/gather_ceiling.cu — how fast can the in-place state gather of the C3 step go on B200?
//
// Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_ceiling tools/gather_ceiling.cu
//
// The pattern is the real one of the bench step: 1024 filters x 2^16 particles,
// Gaussian log-weights sigma^2 = 1, systematic resampling, the canonical permutation NS-15: the
// r-th extra copy (owners ascending) goes to the r-th free slot (ascending); 64-byte rows
// (D = 16 float32).  Host-generated (plain double arithmetic; only the access pattern matters
// here, not bit-exactness).  Each variant copies X[slot] <- X[owner] for every (slot, owner) pair
// of every filter, units of 256 pairs of one filter per warp (the fused kernel's granularity).
//
//   ldg U   : per-lane 16-byte LDG/STG, U chunks in flight per lane (copy_rows_warp, U = 4 today)
//   bulk K  : per-lane cp.async.bulk global->shared of one 64-byte row (mbarrier complete_tx),
//             then cp.async.bulk shared->global; K stages of 32 rows in flight per warp
//   stream  : contiguous float4 copy of the same byte count (the streaming ceiling)
// Algorithmic bytes = 2 x 64 x pairs.  One JSON line per variant.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

struct Unit { int32_t n, start, len, pad; };

template <int U>
__global__ void __launch_bounds__(512) k_ldg(char* X, int64_t xfld, const int2* __restrict__ pairs, int64_t P,
                                             const Unit* __restrict__ units, int nunits) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const uint32_t ch = (lane & 3) * 16u;
    for (int u = gw; u < nunits; u += nw) {
        const Unit un = units[u];
        char* Xf = X + static_cast<int64_t>(un.n) * xfld;
        const int2* pr = pairs + static_cast<int64_t>(un.n) * P + un.start;
        int p = lane >> 2;
        for (; p + (U - 1) * 8 < un.len; p += U * 8) {
            int4 v[U];
            int2 q[U];
#pragma unroll
            for (int k = 0; k < U; ++k) q[k] = pr[p + k * 8];
#pragma unroll
            for (int k = 0; k < U; ++k) v[k] = __ldcg(reinterpret_cast<const int4*>(Xf + static_cast<uint32_t>(q[k].y) * 64u + ch));
#pragma unroll
            for (int k = 0; k < U; ++k) __stcg(reinterpret_cast<int4*>(Xf + static_cast<uint32_t>(q[k].x) * 64u + ch), v[k]);
        }
        for (; p < un.len; p += 8) {
            const int2 q = pr[p];
            __stcg(reinterpret_cast<int4*>(Xf + static_cast<uint32_t>(q.x) * 64u + ch),
                   __ldcg(reinterpret_cast<const int4*>(Xf + static_cast<uint32_t>(q.y) * 64u + ch)));
        }
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// K stages x 32 rows x 64 B per warp, one mbarrier per (stage, lane)
template <int K, int WPC>
__global__ void __launch_bounds__(WPC * 32) k_bulk(char* X, int64_t xfld, const int2* __restrict__ pairs, int64_t P,
                                                   const Unit* __restrict__ units, int nunits) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* buf = sm + static_cast<size_t>(warp) * K * 32 * 64;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + static_cast<size_t>(WPC) * K * 32 * 64) + warp * K * 32;
#pragma unroll
    for (int s = 0; s < K; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + s * 32 + lane)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    uint32_t phase = 0;  // bit s: parity of stage s
    const int gw = blockIdx.x * WPC + warp;
    const int nw = gridDim.x * WPC;
    int dst_pending[K];
    char* dst_ptr[K];
#pragma unroll
    for (int s = 0; s < K; ++s) { dst_pending[s] = 0; dst_ptr[s] = nullptr; }
    int st = 0;  // next stage to fill
    int inflight = 0;
    int drain = 0;  // next stage to drain
    auto drain_one = [&]() {
        const int s = drain;
        if (dst_pending[s]) {
            const uint32_t b = smem_u32(bar + s * 32 + lane);
            const uint32_t par = (phase >> s) & 1u;
            asm volatile(
                "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(b),
                "r"(par) : "memory");
            phase ^= 1u << s;
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 64;" ::"l"(dst_ptr[s]),
                         "r"(smem_u32(buf + (s * 32 + lane) * 64)) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            dst_pending[s] = 0;
        }
        drain = (drain + 1 == K) ? 0 : drain + 1;
        --inflight;
    };
    for (int u = gw; u < nunits; u += nw) {
        const Unit un = units[u];
        char* Xf = X + static_cast<int64_t>(un.n) * xfld;
        const int2* pr = pairs + static_cast<int64_t>(un.n) * P + un.start;
        for (int r0 = 0; r0 < un.len; r0 += 32) {
            if (inflight == K) drain_one();
            // the stage's smem must have been read by its previous store: <= K-1 groups pending
            asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(K - 1) : "memory");
            const int r = r0 + lane;
            if (r < un.len) {
                const int2 q = pr[r];
                const uint32_t b = smem_u32(bar + st * 32 + lane);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 64;" ::"r"(b) : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 64, [%2];" ::"r"(
                        smem_u32(buf + (st * 32 + lane) * 64)),
                    "l"(Xf + static_cast<int64_t>(q.y) * 64), "r"(b)
                    : "memory");
                dst_pending[st] = 1;
                dst_ptr[st] = Xf + static_cast<int64_t>(q.x) * 64;
            } else {
                dst_pending[st] = 0;
            }
            st = (st + 1 == K) ? 0 : st + 1;
            ++inflight;
        }
    }
    while (inflight > 0) drain_one();
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// one copy "engine" warp per CTA (the rest of the SM would be compute): cp.async 16-byte chunks
// into a staging ring of NB batches (K x 8 rows each), completion per batch on an mbarrier
// (32 lane arrivals), retired in order with LDS + STG; up to NB batches in flight.  The pairs
// of a 256-pair unit sit in shared memory (as the resampler's ring would hold them); the next
// unit's pairs are loaded into registers one unit ahead.
template <int NB, int K>
__global__ void __launch_bounds__(32) k_engine(char* X, int64_t xfld, const int2* __restrict__ pairs, int64_t P,
                                               const Unit* __restrict__ units, int nunits) {
    extern __shared__ __align__(128) unsigned char sm[];
    int4* stage = reinterpret_cast<int4*>(sm);
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + NB * K * 32 * 16);
    int2* up = reinterpret_cast<int2*>(bar + NB);  // [2][256] pairs of the current / previous unit
    int* un_n = reinterpret_cast<int*>(up + 512);   // [2] filter of each buffer
    const int lane = threadIdx.x;
    if (lane < NB) asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(smem_u32(bar + lane)));
    __syncwarp();
    const uint32_t ch = (lane & 3) * 16u;
    const int sub = lane >> 2;
    int head = 0, tail = 0;
    uint32_t phase = 0;
    int bbuf[NB], boff[NB], bcnt[NB];
    // register prefetch of a unit's pairs: 8 per lane
    int2 pre[8];
    int pre_len = 0, pre_n = 0;
    int u = blockIdx.x;
    auto prefetch = [&](int uu) {
        pre_len = 0;
        if (uu < nunits) {
            const Unit un = units[uu];
            pre_len = un.len;
            pre_n = un.n;
            const int2* pr = pairs + static_cast<int64_t>(un.n) * P + un.start;
#pragma unroll
            for (int t = 0; t < 8; ++t) pre[t] = (lane * 8 + t < un.len) ? pr[lane * 8 + t] : make_int2(0, 0);
        }
    };
    prefetch(u);
    int cur = 0, cur_len = 0, r0 = 0;
    auto next_unit = [&]() -> bool {  // current unit exhausted: move the prefetched one into smem
        if (pre_len == 0) return false;
        cur ^= 1;
        // the buffer being overwritten may still be referenced by in-flight batches: the caller
        // retires all batches of the old buffer first (at most one unit in flight)
#pragma unroll
        for (int t = 0; t < 8; ++t) up[cur * 256 + lane * 8 + t] = pre[t];
        if (lane == 0) un_n[cur] = pre_n;
        cur_len = pre_len;
        r0 = 0;
        __syncwarp();
        u += gridDim.x;
        prefetch(u);
        return true;
    };
    auto retire = [&]() {
        const int b = head % NB;
        const uint32_t par = (phase >> b) & 1u;
        asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(
                         smem_u32(bar + b)), "r"(par) : "memory");
        phase ^= 1u << b;
        char* Xf = X + static_cast<int64_t>(un_n[bbuf[b]]) * xfld;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int rr = k * 8 + sub;
            if (rr < bcnt[b]) {
                const int2 q = up[bbuf[b] * 256 + boff[b] + rr];
                __stcg(reinterpret_cast<int4*>(Xf + static_cast<int64_t>(q.x) * 64 + ch), stage[(b * K + k) * 32 + lane]);
            }
        }
        ++head;
    };
    int old_inflight_of_prev = 0;  // batches of the other buffer still in flight
    bool have = next_unit();
    while (have || head != tail) {
        if (have && r0 < cur_len && tail - head < NB) {
            const int b = tail % NB;
            const int cnt = min(K * 8, cur_len - r0);
            const char* Xf = X + static_cast<int64_t>(un_n[cur]) * xfld;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int rr = k * 8 + sub;
                if (rr < cnt) {
                    const int2 q = up[cur * 256 + r0 + rr];
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(stage + (b * K + k) * 32 + lane)),
                                 "l"(Xf + static_cast<int64_t>(q.y) * 64 + ch) : "memory");
                }
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];" ::"r"(smem_u32(bar + b)) : "memory");
            bbuf[b] = cur;
            boff[b] = r0;
            bcnt[b] = cnt;
            r0 += cnt;
            ++tail;
            continue;
        }
        if (have && r0 >= cur_len) {
            // switch units: batches of the buffer about to be overwritten must be retired
            while (head != tail && bbuf[head % NB] != cur) retire();
            have = next_unit();
            (void)old_inflight_of_prev;
            continue;
        }
        retire();
    }
}

__global__ void k_stream(const int4* __restrict__ a, int4* __restrict__ b, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        b[i] = __ldcs(a + i);
}

int main(int argc, char** argv) {
    const int N = 1024, P = 1 << 16;
    const double sigma = 1.0;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    // ---- host pattern: systematic resampling + NS-15 pairs per filter
    std::vector<int2> pairs(static_cast<size_t>(N) * P);
    std::vector<int32_t> cnt(N);
    std::vector<Unit> units;
    std::mt19937_64 rng(0x12026163);
    std::normal_distribution<double> nd;
    std::uniform_real_distribution<double> ud;
    std::vector<double> w(P);
    std::vector<int32_t> o(P), freel, extr;
    int64_t total = 0;
    for (int n = 0; n < N; ++n) {
        double S = 0;
        for (int i = 0; i < P; ++i) { w[i] = std::exp(sigma * nd(rng)); S += w[i]; }
        const double u = ud(rng);
        double C = 0;
        int64_t prev = 0;
        for (int i = 0; i < P; ++i) {
            C += w[i] / S;
            int64_t e = static_cast<int64_t>(std::floor(C * P - u)) + 1;  // #{k : (k + u)/P < C}
            e = std::min<int64_t>(std::max<int64_t>(e, 0), P);
            if (i == P - 1) e = P;
            o[i] = static_cast<int32_t>(e - prev);
            prev = e;
        }
        freel.clear();
        extr.clear();
        for (int i = 0; i < P; ++i) {
            if (o[i] == 0) freel.push_back(i);
            for (int k = 1; k < o[i]; ++k) extr.push_back(i);
        }
        const size_t m = std::min(freel.size(), extr.size());
        cnt[n] = static_cast<int32_t>(m);
        for (size_t r = 0; r < m; ++r) pairs[static_cast<size_t>(n) * P + r] = make_int2(freel[r], extr[r]);
        for (size_t s0 = 0; s0 < m; s0 += 256) units.push_back({n, static_cast<int32_t>(s0), static_cast<int32_t>(std::min<size_t>(256, m - s0)), 0});
        total += static_cast<int64_t>(m);
    }
    printf("{\"pattern\":\"C3 systematic sigma2=1\",\"moved_fraction\":%.4f,\"units\":%zu}\n", double(total) / (double(N) * P), units.size());
    int2* d_pairs;
    Unit* d_units;
    char* X;
    CK(cudaMalloc(&d_pairs, pairs.size() * sizeof(int2)));
    CK(cudaMalloc(&d_units, units.size() * sizeof(Unit)));
    const int64_t xfld = static_cast<int64_t>(P) * 64;
    CK(cudaMalloc(&X, xfld * N));
    CK(cudaMemset(X, 1, xfld * N));
    CK(cudaMemcpy(d_pairs, pairs.data(), pairs.size() * sizeof(int2), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_units, units.data(), units.size() * sizeof(Unit), cudaMemcpyHostToDevice));
    const int nunits = static_cast<int>(units.size());
    const double bytes = 2.0 * 64.0 * double(total);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char* name, int param, auto launch) -> int {
        for (int i = 0; i < 3; ++i) launch();
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        float best = 1e30f, sum = 0;
        const int reps = 10;
        for (int i = 0; i < reps; ++i) {
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = std::min(best, ms);
            sum += ms;
        }
        printf("{\"variant\":\"%s\",\"param\":%d,\"ms_best\":%.4f,\"ms_mean\":%.4f,\"alg_GBs\":%.1f}\n", name, param, best,
               sum / reps, bytes / (sum / reps * 1e-3) / 1e9);
        fflush(stdout);
        return 0;
    };
    for (int occ : {2, 4}) {
        timeit("ldg4", occ, [&] { k_ldg<4><<<sms * occ, 512>>>(X, xfld, d_pairs, P, d_units, nunits); });
        timeit("ldg8", occ, [&] { k_ldg<8><<<sms * occ, 512>>>(X, xfld, d_pairs, P, d_units, nunits); });
    }
    timeit("ldg16", 2, [&] { k_ldg<16><<<sms * 2, 512>>>(X, xfld, d_pairs, P, d_units, nunits); });
    timeit("ldg4_low_occ", 1, [&] { k_ldg<4><<<sms, 512>>>(X, xfld, d_pairs, P, d_units, nunits); });
    {
        constexpr int K = 4, WPC = 8;
        const int smem = WPC * K * 32 * 64 + WPC * K * 32 * 8;
        CK(cudaFuncSetAttribute(k_bulk<K, WPC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (int occ : {1, 2, 3})
            timeit("bulk_K4_W8", occ, [&] { k_bulk<K, WPC><<<sms * occ, WPC * 32, smem>>>(X, xfld, d_pairs, P, d_units, nunits); });
    }
    {
        constexpr int K = 8, WPC = 4;
        const int smem = WPC * K * 32 * 64 + WPC * K * 32 * 8;
        CK(cudaFuncSetAttribute(k_bulk<K, WPC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (int occ : {1, 2, 3})
            timeit("bulk_K8_W4", occ, [&] { k_bulk<K, WPC><<<sms * occ, WPC * 32, smem>>>(X, xfld, d_pairs, P, d_units, nunits); });
    }
    {
        constexpr int K = 16, WPC = 2;
        const int smem = WPC * K * 32 * 64 + WPC * K * 32 * 8;
        CK(cudaFuncSetAttribute(k_bulk<K, WPC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (int occ : {2, 4, 6})
            timeit("bulk_K16_W2", occ, [&] { k_bulk<K, WPC><<<sms * occ, WPC * 32, smem>>>(X, xfld, d_pairs, P, d_units, nunits); });
    }
    // one engine warp per CTA, `occ` CTAs per SM (what a warp-specialised resampler could dedicate)
    {
        constexpr int NB = 8, K = 4;
        const int smem = NB * K * 32 * 16 + NB * 8 + 512 * 8 + 16;
        CK(cudaFuncSetAttribute(k_engine<NB, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (int occ : {3, 4, 6, 8})
            timeit("engine_NB8_K4", occ, [&] { k_engine<NB, K><<<sms * occ, 32, smem>>>(X, xfld, d_pairs, P, d_units, nunits); });
    }
    {
        constexpr int NB = 16, K = 4;
        const int smem = NB * K * 32 * 16 + NB * 8 + 512 * 8 + 16;
        CK(cudaFuncSetAttribute(k_engine<NB, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (int occ : {2, 3, 4})
            timeit("engine_NB16_K4", occ, [&] { k_engine<NB, K><<<sms * occ, 32, smem>>>(X, xfld, d_pairs, P, d_units, nunits); });
    }
    // streaming copy of the same number of bytes (half read, half written)
    {
        const int64_t n16 = static_cast<int64_t>(bytes / 2 / 16);
        int4* Y;
        CK(cudaMalloc(&Y, n16 * 16));
        timeit("stream", 0, [&] { k_stream<<<sms * 8, 256>>>(reinterpret_cast<const int4*>(X), Y, n16); });
        CK(cudaFree(Y));
    }
    return 0;
}
