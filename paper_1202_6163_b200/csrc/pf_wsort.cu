// pf_wsort.cu — pre-sorted weights (PF_SORT_WEIGHTS; NS-17 / R-14): the paper's
// "sorting enabled" series, where the weights are sorted in descending order so
// that the searches of the heavy particles end early.  Here: a segmented, stable LSD radix
// sort of every filter's log-weights (8 passes of 4-bit digits over order-preserving u32
// keys, descending, equal values in index order), the float path on the sorted weights, and
// a_k = sigma[b_k] back in the original indices.
//
// One pass = three launches over (filter, 4096-item tile) CTAs of 256 threads x 16 items
// (blocked: thread t holds items 16t..16t+15 of its tile, so thread order is index order):
//   k_rhist     digit counts of the tile -> H[n][digit][tile]
//   k_rscan     per filter: exclusive scan of H in (digit, tile) order (global digit offsets)
//   k_rscatter  per-thread digit counts -> CTA exclusive scan in (digit, thread) order ->
//               stable positions; pass 0 reads the float log-weights and builds (key, index),
//               the last pass writes the sorted float weights instead of the keys.
// HBM per pass: 8 B read twice + 8 B written per particle (the sort is the series' cost,
// which the paper found to outweigh the faster search).
#include <algorithm>

#include "pf_device.cuh"
#include "pf_internal.h"

namespace pf {
namespace {

constexpr int kRT = 256;              // threads
constexpr int kRI = 16;               // items per thread
constexpr int kRTile = kRT * kRI;     // 4096 items per tile
constexpr int kRadixBits = 4;
constexpr int kDigits = 1 << kRadixBits;
constexpr int kPasses = 32 / kRadixBits;
constexpr int kSortSmem = (kDigits * kRT + 2 * kRTile) * 4;  // counters + the tile's keys and values

// descending order key: equal floats (+0 == -0) get equal keys; -inf sorts last among numbers
__device__ __forceinline__ uint32_t sort_key(float f) {
    uint32_t b = __float_as_uint(f == 0.0f ? 0.0f : f);
    b = (b >> 31) ? ~b : (b | 0x80000000u);  // ascending order of the float value
    return ~b;                              // descending
}
__device__ __forceinline__ float key_value(uint32_t k) {
    const uint32_t a = ~k;
    return __uint_as_float((a >> 31) ? (a & 0x7FFFFFFFu) : ~a);
}

struct SortArgs {
    const float* logw;  // pass 0 input
    int64_t ld;
    int32_t N, P, T;
    int64_t ldk;        // stride of the key / value planes
    const uint32_t* kin;
    const int32_t* vin;
    uint32_t* kout;     // last pass: the sorted float weights (as bits)
    int32_t* vout;
    uint32_t* H;        // [N][kDigits][T]
    int shift;
};

// 16 items of thread t of tile `tile` of filter n: keys and original indices
template <bool FIRST>
__device__ __forceinline__ int load_items(const SortArgs& a, int64_t n, int tile, uint32_t* k, int32_t* v) {
    const int64_t i0 = static_cast<int64_t>(tile) * kRTile + threadIdx.x * kRI;
    const int cnt = static_cast<int>(max(int64_t{0}, min(int64_t{kRI}, static_cast<int64_t>(a.P) - i0)));
    if (!FIRST && cnt == kRI) {
        // planes have 16-byte aligned rows (ldk % 4 == 0) and i0 % 16 == 0
        const uint4* kp = reinterpret_cast<const uint4*>(a.kin + n * a.ldk + i0);
        const int4* vp = reinterpret_cast<const int4*>(a.vin + n * a.ldk + i0);
#pragma unroll
        for (int q = 0; q < kRI / 4; ++q) {
            const uint4 kk = kp[q];
            const int4 vv = vp[q];
            k[4 * q] = kk.x; k[4 * q + 1] = kk.y; k[4 * q + 2] = kk.z; k[4 * q + 3] = kk.w;
            v[4 * q] = vv.x; v[4 * q + 1] = vv.y; v[4 * q + 2] = vv.z; v[4 * q + 3] = vv.w;
        }
        return cnt;
    }
#pragma unroll
    for (int j = 0; j < kRI; ++j) {
        if (j < cnt) {
            if (FIRST) {
                k[j] = sort_key(a.logw[n * a.ld + i0 + j]);
                v[j] = static_cast<int32_t>(i0 + j);
            } else {
                k[j] = a.kin[n * a.ldk + i0 + j];
                v[j] = a.vin[n * a.ldk + i0 + j];
            }
        } else {
            k[j] = 0;
            v[j] = 0;
        }
    }
    return cnt;
}

// packed per-thread digit counts: 8-bit fields, digits 0..7 in lo, 8..15 in hi
__device__ __forceinline__ void count_digits(const uint32_t* k, int cnt, int shift, uint64_t& lo, uint64_t& hi) {
    lo = 0;
    hi = 0;
#pragma unroll
    for (int j = 0; j < kRI; ++j) {
        const uint32_t d = (k[j] >> shift) & (kDigits - 1);
        const uint64_t one = (j < cnt) ? 1ull : 0ull;
        lo += (d < 8) ? (one << (8 * d)) : 0ull;
        hi += (d >= 8) ? (one << (8 * (d - 8))) : 0ull;
    }
}
__device__ __forceinline__ uint32_t field(uint64_t lo, uint64_t hi, int d) {
    return static_cast<uint32_t>(((d < 8) ? (lo >> (8 * d)) : (hi >> (8 * (d - 8)))) & 0xFFu);
}

// the histogram does not depend on the order of the items: coalesced striped loads (float4 /
// uint4 where the rows allow), 16 items per thread
template <bool FIRST>
__global__ void __launch_bounds__(kRT) k_rhist(SortArgs a) {
    const int64_t n = blockIdx.x / a.T;
    const int tile = static_cast<int>(blockIdx.x % a.T);
    const int64_t t0 = static_cast<int64_t>(tile) * kRTile;
    const int tc = static_cast<int>(min(int64_t{kRTile}, static_cast<int64_t>(a.P) - t0));
    uint32_t k[kRI];
    int cnt = 0;
    const bool vec = FIRST ? ((reinterpret_cast<uintptr_t>(a.logw) & 15) == 0 && (a.ld & 3) == 0) : true;
    if (vec && tc == kRTile) {
#pragma unroll
        for (int q = 0; q < kRI / 4; ++q) {
            const int64_t i = t0 + (q * kRT + threadIdx.x) * 4;
            if (FIRST) {
                const float4 f = __ldcs(reinterpret_cast<const float4*>(a.logw + n * a.ld + i));
                k[4 * q] = sort_key(f.x); k[4 * q + 1] = sort_key(f.y);
                k[4 * q + 2] = sort_key(f.z); k[4 * q + 3] = sort_key(f.w);
            } else {
                const uint4 u = *reinterpret_cast<const uint4*>(a.kin + n * a.ldk + i);
                k[4 * q] = u.x; k[4 * q + 1] = u.y; k[4 * q + 2] = u.z; k[4 * q + 3] = u.w;
            }
        }
        cnt = kRI;
    } else {
#pragma unroll
        for (int j = 0; j < kRI; ++j) {
            const int r = j * kRT + threadIdx.x;  // striped
            k[j] = 0;
            if (r < tc) {
                k[j] = FIRST ? sort_key(a.logw[n * a.ld + t0 + r]) : a.kin[n * a.ldk + t0 + r];
                cnt = j + 1;
            }
        }
    }
    uint64_t lo, hi;
    count_digits(k, cnt, a.shift, lo, hi);
    __shared__ uint32_t s_c[kDigits];
    if (threadIdx.x < kDigits) s_c[threadIdx.x] = 0;
    __syncthreads();
    // per digit: the warp's sum of the per-thread fields (<= 16 each), one smem atomic per warp
#pragma unroll
    for (int d = 0; d < kDigits; ++d) {
        uint32_t c = field(lo, hi, d);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
        if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s_c[d], c);
    }
    __syncthreads();
    if (threadIdx.x < kDigits) a.H[(n * kDigits + threadIdx.x) * a.T + tile] = s_c[threadIdx.x];
}

// per filter: exclusive scan of H[n][0..kDigits*T) in place
__global__ void __launch_bounds__(kRT) k_rscan(uint32_t* H, int32_t T) {
    const int64_t n = blockIdx.x;
    uint32_t* h = H + n * kDigits * T;
    const int64_t len = static_cast<int64_t>(kDigits) * T;
    __shared__ uint32_t s_w[kRT / 32];
    __shared__ uint32_t s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t base = 0; base < len; base += kRT) {
        const int64_t i = base + threadIdx.x;
        const uint32_t x = (i < len) ? h[i] : 0u;
        uint32_t inc = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, inc, o);
            if (lane >= o) inc += u;
        }
        if (lane == 31) s_w[warp] = inc;
        __syncthreads();
        uint32_t wpre = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < kRT / 32; ++w) {
            const uint32_t t = s_w[w];
            wpre += (w < warp) ? t : 0u;
            tot += t;
        }
        const uint32_t carry = s_carry;
        if (i < len) h[i] = carry + wpre + inc - x;
        __syncthreads();
        if (threadIdx.x == 0) s_carry = carry + tot;
        __syncthreads();
    }
}

// s_cnt[d * kRT + t] <- number of items of digit d in threads < t plus in digits < d over the
// whole tile: the CTA-wide exclusive scan of the per-thread digit counts in (digit, thread)
// order, i.e. the position in the tile's stable digit order of thread t's first digit-d item
__device__ __forceinline__ void tile_digit_scan(uint64_t lo, uint64_t hi, uint32_t* s_cnt, uint32_t* s_w, int tid) {
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int d = 0; d < kDigits; ++d) s_cnt[d * kRT + tid] = field(lo, hi, d);
    __syncthreads();
    // thread t owns the entries [16t, 16t + 16) of the flat (digit, thread) array
    uint32_t run[kRI];
    uint32_t sum = 0;
#pragma unroll
    for (int j = 0; j < kRI; ++j) {
        run[j] = sum;
        sum += s_cnt[tid * kRI + j];
    }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= o) inc += u;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    uint32_t wpre = 0;
#pragma unroll
    for (int w = 0; w < kRT / 32; ++w) wpre += (w < warp) ? s_w[w] : 0u;
    const uint32_t excl = wpre + inc - sum;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kRI; ++j) s_cnt[tid * kRI + j] = excl + run[j];
    __syncthreads();
}

// Filters of P <= 4096 (one tile): all eight passes in shared memory, one launch, one CTA per
// filter; writes the sorted weights and sigma like the last multi-tile pass.
__global__ void __launch_bounds__(kRT) k_rsort_tile(SortArgs a) {
    extern __shared__ __align__(16) uint32_t s_dyn[];
    uint32_t* s_cnt = s_dyn;                                       // kDigits * kRT
    uint32_t* s_k = s_dyn + kDigits * kRT;                         // kRTile
    int32_t* s_v = reinterpret_cast<int32_t*>(s_k + kRTile);       // kRTile
    __shared__ uint32_t s_w[kRT / 32];
    const int64_t n = blockIdx.x;
    const int tid = threadIdx.x;
    uint32_t k[kRI];
    int32_t v[kRI];
    const int cnt = load_items<true>(a, n, 0, k, v);
    for (int pass = 0; pass < kPasses; ++pass) {
        const int shift = pass * kRadixBits;
        uint64_t lo, hi;
        count_digits(k, cnt, shift, lo, hi);
        tile_digit_scan(lo, hi, s_cnt, s_w, tid);
#pragma unroll
        for (int j = 0; j < kRI; ++j) {
            if (j < cnt) {
                const uint32_t d = (k[j] >> shift) & (kDigits - 1);
                const uint32_t pos = s_cnt[d * kRT + tid]++;
                s_k[pos] = k[j];
                s_v[pos] = v[j];
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kRI; ++j) {
            if (j < cnt) {
                k[j] = s_k[tid * kRI + j];
                v[j] = s_v[tid * kRI + j];
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < kRI; ++j) {
        if (j < cnt) {
            const int64_t o = n * a.ldk + tid * kRI + j;
            a.kout[o] = __float_as_uint(key_value(k[j]));
            a.vout[o] = v[j];
        }
    }
}

template <bool FIRST, bool LAST>
__global__ void __launch_bounds__(kRT) k_rscatter(SortArgs a) {
    const int64_t n = blockIdx.x / a.T;
    const int tile = static_cast<int>(blockIdx.x % a.T);
    const int tid = threadIdx.x;
    uint32_t k[kRI];
    int32_t v[kRI];
    const int cnt = load_items<FIRST>(a, n, tile, k, v);
    uint64_t lo, hi;
    count_digits(k, cnt, a.shift, lo, hi);
    extern __shared__ __align__(16) uint32_t s_dyn[];
    uint32_t* s_cnt = s_dyn;                                  // (digit, thread) order
    uint32_t* s_k = s_dyn + kDigits * kRT;                    // the tile in digit order
    int32_t* s_v = reinterpret_cast<int32_t*>(s_k + kRTile);
    __shared__ uint32_t s_w[kRT / 32];
    __shared__ int64_t s_goff[kDigits];
    tile_digit_scan(lo, hi, s_cnt, s_w, tid);
    // a tile item at digit-order position p goes to the filter's position H[d][tile] + p - start[d]
    if (tid < kDigits)
        s_goff[tid] = static_cast<int64_t>(a.H[(n * kDigits + tid) * a.T + tile]) - s_cnt[tid * kRT];
    __syncthreads();
    // stable local sort of the tile by the digit (thread order = index order), in shared memory
#pragma unroll
    for (int j = 0; j < kRI; ++j) {
        if (j < cnt) {
            const uint32_t d = (k[j] >> a.shift) & (kDigits - 1);
            const uint32_t pos = s_cnt[d * kRT + tid]++;  // column of this thread: no conflicts
            s_k[pos] = k[j];
            s_v[pos] = v[j];
        }
    }
    __syncthreads();
    // coalesced stores: consecutive positions of one digit are consecutive in the filter
    const int tc = static_cast<int>(min(int64_t{kRTile}, static_cast<int64_t>(a.P) - static_cast<int64_t>(tile) * kRTile));
    for (int p = tid; p < tc; p += kRT) {
        const uint32_t key = s_k[p];
        const int64_t o = n * a.ldk + s_goff[(key >> a.shift) & (kDigits - 1)] + p;
        a.kout[o] = LAST ? __float_as_uint(key_value(key)) : key;
        a.vout[o] = s_v[p];
    }
}

// a_k = sigma[b_k] (identity for invalid filters, NS-1); normw back to the original order
__global__ void __launch_bounds__(kRT) k_unsort(const int32_t* __restrict__ sigma, int64_t ldk,
                                                const int32_t* __restrict__ b, const int32_t* __restrict__ fst,
                                                int32_t N, int32_t P, int32_t* __restrict__ anc, int64_t ld_anc,
                                                const float* __restrict__ vs, float* __restrict__ normw) {
    const int64_t total = static_cast<int64_t>(N) * P;
    for (int64_t g = static_cast<int64_t>(blockIdx.x) * kRT + threadIdx.x; g < total;
         g += static_cast<int64_t>(gridDim.x) * kRT) {
        const int64_t n = g / P, k = g % P;
        const bool ok = fst[n] == 0;
        const int32_t* sg = sigma + n * ldk;
        anc[n * ld_anc + k] = ok ? sg[b[n * ldk + k]] : static_cast<int32_t>(k);
        if (normw) normw[n * P + sg[k]] = vs[n * P + k];
    }
}

}  // namespace

size_t wsort_ws_bytes(int32_t N, int32_t P, bool normw) {
    const int64_t ldk = (static_cast<int64_t>(P) + 3) / 4 * 4;
    const int64_t T = (P + kRTile - 1) / kRTile;
    auto al = [](size_t x) { return (x + 255) / 256 * 256; };
    const size_t plane = al(static_cast<size_t>(N) * static_cast<size_t>(ldk) * 4);
    return 5 * plane + al(static_cast<size_t>(N) * kDigits * static_cast<size_t>(T) * 4) +
           al(static_cast<size_t>(N) * 4) + (normw ? al(static_cast<size_t>(N) * static_cast<size_t>(P) * 4) : 0);
}

cudaError_t launch_wsort(const float* logw, int64_t ld, int32_t N, int32_t P, void* ws, bool normw, WsortBufs* out,
                         cudaStream_t s, uint64_t* launches) {
    const int64_t ldk = (static_cast<int64_t>(P) + 3) / 4 * 4;
    const int32_t T = static_cast<int32_t>((P + kRTile - 1) / kRTile);
    auto al = [](size_t x) { return (x + 255) / 256 * 256; };
    const size_t plane = al(static_cast<size_t>(N) * static_cast<size_t>(ldk) * 4);
    char* p = static_cast<char*>(ws);
    uint32_t* kA = reinterpret_cast<uint32_t*>(p);
    int32_t* vA = reinterpret_cast<int32_t*>(p + plane);
    uint32_t* kB = reinterpret_cast<uint32_t*>(p + 2 * plane);
    int32_t* vB = reinterpret_cast<int32_t*>(p + 3 * plane);
    int32_t* b = reinterpret_cast<int32_t*>(p + 4 * plane);
    uint32_t* H = reinterpret_cast<uint32_t*>(p + 5 * plane);
    int32_t* fst = reinterpret_cast<int32_t*>(p + 5 * plane + al(static_cast<size_t>(N) * kDigits * T * 4));
    float* vs = normw ? reinterpret_cast<float*>(reinterpret_cast<char*>(fst) + al(static_cast<size_t>(N) * 4))
                      : nullptr;
    SortArgs a{logw, ld, N, P, T, ldk, nullptr, nullptr, nullptr, nullptr, H, 0};
    const unsigned grid = static_cast<unsigned>(static_cast<int64_t>(N) * T);
    {
        // dynamic shared memory above 48 KB (per device; idempotent, so a racing first call on
        // one device just sets the same values twice)
        static std::atomic<int> done[kMaxDevices];
        std::atomic<int>& d = done[current_device()];
        if (!d.load(std::memory_order_relaxed)) {
            cudaFuncSetAttribute(k_rsort_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, kSortSmem);
            cudaFuncSetAttribute(k_rscatter<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSortSmem);
            cudaFuncSetAttribute(k_rscatter<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSortSmem);
            cudaFuncSetAttribute(k_rscatter<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSortSmem);
            d.store(1, std::memory_order_relaxed);
        }
    }
    for (int pass = 0; pass < kPasses && T == 1; ++pass) {  // one tile: a single launch
        a.kout = kB;
        a.vout = vB;
        ProfScope ps_("k_rsort_tile", s);
        k_rsort_tile<<<static_cast<unsigned>(N), kRT, kSortSmem, s>>>(a);
        ++*launches;
        break;
    }
    for (int pass = 0; pass < kPasses && T > 1; ++pass) {
        a.shift = pass * kRadixBits;
        const bool first = pass == 0, last = pass == kPasses - 1;
        a.kin = (pass & 1) ? kA : kB;
        a.vin = (pass & 1) ? vA : vB;
        a.kout = (pass & 1) ? kB : kA;
        a.vout = (pass & 1) ? vB : vA;
        {
            ProfScope ps_("k_rhist", s);
            if (first) k_rhist<true><<<grid, kRT, 0, s>>>(a);
            else k_rhist<false><<<grid, kRT, 0, s>>>(a);
        }
        {
            ProfScope ps_("k_rscan", s);
            k_rscan<<<static_cast<unsigned>(N), kRT, 0, s>>>(H, T);
        }
        {
            ProfScope ps_("k_rscatter", s);
            if (first) k_rscatter<true, false><<<grid, kRT, kSortSmem, s>>>(a);
            else if (last) k_rscatter<false, true><<<grid, kRT, kSortSmem, s>>>(a);
            else k_rscatter<false, false><<<grid, kRT, kSortSmem, s>>>(a);
        }
        *launches += 3;
    }
    static_assert(kPasses % 2 == 0, "the sorted planes end in kB / vB");
    out->y = reinterpret_cast<float*>(kB);
    out->sigma = vB;
    out->ldk = ldk;
    out->b = b;
    out->fstatus = fst;
    out->vs = vs;
    return cudaPeekAtLastError();
}

cudaError_t launch_unsort(const WsortBufs& w, int32_t N, int32_t P, int32_t* anc, int64_t ld_anc, float* normw,
                          cudaStream_t s, uint64_t* launches) {
    const int64_t total = static_cast<int64_t>(N) * P;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>((total + kRT - 1) / kRT, 8LL * sm_count()));
    ProfScope ps_("k_unsort", s);
    k_unsort<<<grid, kRT, 0, s>>>(w.sigma, w.ldk, w.b, w.fstatus, N, P, anc, ld_anc, w.vs, normw);
    ++*launches;
    return cudaPeekAtLastError();
}

}  // namespace pf
