// pf_migrate.cu — cross-GPU particle migration of a sharded filter (include/pf.h 4a-4d;
// SURVEY §8(f) NEXT-4).
//
// The canonical permutation NS-15 of the whole filter, shard by shard: each shard packs its
// own extras (particle i repeated o_i - 1 times, ascending i) and fills its own free slots
// (o_i = 0, ascending) from the rows the all-to-all delivers.  Both lists are built per
// 2048-particle tile from a tile-level exclusive scan, then expanded item by item (one
// 4/16-byte chunk of one row per thread), so the copies are coalesced on the packed side; the
// pack side walks work items of 2048 extras ranks (a skewed tile is split over many CTAs).
#include <algorithm>
#include <cmath>
#include <cstdint>

#include "pf_internal.h"

namespace pf {
namespace {

constexpr int kMigItems = 8;
constexpr int kMigTile = kThreads * kMigItems;  // particles per tile
constexpr unsigned kFullMask = 0xffffffffu;

template <int CH>
struct MigChunk;
template <> struct MigChunk<16> { using T = int4; };
template <> struct MigChunk<4> { using T = int32_t; };
template <> struct MigChunk<1> { using T = char; };

__host__ __device__ inline int64_t mig_cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Exclusive block scan of one value per thread (kThreads threads); returns the block total.
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* excl, int64_t* s_warp) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int64_t t = __shfl_up_sync(kFullMask, inc, d);
        if (lane >= d) inc += t;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    int64_t before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
        const int64_t s = s_warp[w];
        if (w < warp) before += s;
        total += s;
    }
    *excl = before + inc - v;
    __syncthreads();  // s_warp reusable
    return total;
}

// 4a: histogram of the window's ancestors; warp-aggregated atomics (unsorted ancestors).
__global__ void __launch_bounds__(kThreads) k_mig_offspring(const int32_t* __restrict__ anc, int64_t n_anc,
                                                            int64_t win0, int32_t Pw, const float* gmax,
                                                            const int32_t* gbad, int32_t* __restrict__ o) {
    const bool invalid = gbad != nullptr && (*gbad != 0 || *gmax == -INFINITY);
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
    if (invalid) {
        for (int64_t i = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; i < Pw; i += stride) o[i] = 1;
        return;
    }
    const int lane = threadIdx.x & 31;
    // warp-uniform trip count so __match_any_sync sees the whole warp
    for (int64_t base = blockIdx.x * static_cast<int64_t>(kThreads) + (threadIdx.x & ~31); base < n_anc;
         base += stride) {
        const int64_t k = base + lane;
        int32_t v = -1;
        if (k < n_anc) {
            const int64_t a = static_cast<int64_t>(__ldg(anc + k)) - win0;
            if (a >= 0 && a < Pw) v = static_cast<int32_t>(a);
        }
        const unsigned peers = __match_any_sync(kFullMask, v);
        if (v >= 0 && lane == __ffs(peers) - 1) atomicAdd(o + v, static_cast<int32_t>(__popc(peers)));
    }
}

// 4a with a slot range (stratified, systematic, sorted multinomial): the range's ancestors are
// nondecreasing, so o_a is the length of a's run.  Per warp of 32 slots: run boundaries from
// neighbour shuffles; a run that starts and ends inside the warp is stored by its first lane
// (no atomics); a run crossing a warp boundary is summed from per-warp pieces with atomics.
__global__ void __launch_bounds__(kThreads) k_mig_offspring_runs(const int32_t* __restrict__ anc, int64_t n_anc,
                                                                 const int64_t* __restrict__ range, int64_t win0,
                                                                 int32_t Pw, const float* gmax, const int32_t* gbad,
                                                                 int32_t* __restrict__ o) {
    const bool invalid = gbad != nullptr && (*gbad != 0 || *gmax == -INFINITY);
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
    if (invalid) {
        for (int64_t i = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; i < Pw; i += stride) o[i] = 1;
        return;
    }
    const int lane = threadIdx.x & 31;
    const int64_t lo = max(range[0], static_cast<int64_t>(0)), hi = min(range[1], n_anc);
    for (int64_t base = lo + blockIdx.x * static_cast<int64_t>(kThreads) + (threadIdx.x & ~31); base < hi;
         base += stride) {
        const int64_t k = base + lane;
        const bool in = k < hi;
        const int32_t a = in ? __ldg(anc + k) : 0;
        int32_t prev = __shfl_up_sync(kFullMask, a, 1), next = __shfl_down_sync(kFullMask, a, 1);
        if (lane == 0 && in && k > lo) prev = __ldg(anc + k - 1);
        if (lane == 31 && k + 1 < hi) next = __ldg(anc + k + 1);
        const bool start = in && (k == lo || prev != a);
        const bool end = in && (k == hi - 1 || next != a);
        const unsigned ends = __ballot_sync(kFullMask, end);
        const int64_t v = static_cast<int64_t>(a) - win0;
        if (!in || v < 0 || v >= Pw) continue;
        if (start) {
            const unsigned m = ends >> lane;  // ends at this lane or later
            if (m != 0) o[v] = __ffs(m);      // the whole run is inside the warp
            else atomicAdd(o + v, 32 - lane);
        } else if (lane == 0) {  // the warp's first run began in an earlier warp
            atomicAdd(o + v, ends != 0 ? __ffs(ends) : 32);
        }
    }
}

// Per-tile counts: tE[t] = sum max(o - 1, 0), tF[t] = #{o = 0} over tile t.
__global__ void __launch_bounds__(kThreads) k_mig_tile_counts(const int32_t* __restrict__ o, int32_t Pl,
                                                              int64_t* __restrict__ tE, int64_t* __restrict__ tF) {
    __shared__ int64_t s_warp[kThreads / 32];
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kMigTile + threadIdx.x * kMigItems;
    int64_t e = 0, f = 0;
#pragma unroll
    for (int j = 0; j < kMigItems; ++j) {
        const int64_t i = i0 + j;
        if (i < Pl) {
            const int32_t v = __ldg(o + i);
            e += v > 1 ? v - 1 : 0;
            f += v == 0;
        }
    }
    int64_t ex;
    const int64_t E = block_excl_scan(e, &ex, s_warp);
    const int64_t F = block_excl_scan(f, &ex, s_warp);
    if (threadIdx.x == 0) {
        tE[blockIdx.x] = E;
        tF[blockIdx.x] = F;
    }
}

// One CTA: exclusive scans of tE and tF in place; totals into counts[0..1].  Thread t owns
// kScanPer consecutive tiles of each round of 1024 * kScanPer (all loads issued at once).
constexpr int kScanPer = 16;
// The pack stage's work items: tile t's extras are cut into ceil(E_t / kMigTile) chunks of
// kMigTile ranks; tC (ntiles + 1 entries) = their exclusive prefix, tC[ntiles] = the total.
__global__ void __launch_bounds__(1024) k_mig_tile_scan(int64_t* __restrict__ tE, int64_t* __restrict__ tF,
                                                        int64_t* __restrict__ tC, int64_t ntiles,
                                                        int64_t* __restrict__ counts) {
    __shared__ int64_t s_warp[3][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t cE = 0, cF = 0, cC = 0;
    for (int64_t r0 = 0; r0 < ntiles; r0 += 1024 * kScanPer) {
        const int64_t b = r0 + static_cast<int64_t>(threadIdx.x) * kScanPer;
        int64_t vE[kScanPer], vF[kScanPer];
        int64_t sE = 0, sF = 0, sC = 0;
#pragma unroll
        for (int u = 0; u < kScanPer; ++u) {
            const bool in = b + u < ntiles;
            vE[u] = in ? tE[b + u] : 0;
            vF[u] = in ? tF[b + u] : 0;
            sE += vE[u];
            sF += vF[u];
            sC += mig_cdiv(vE[u], kMigTile);
        }
        int64_t iE = sE, iF = sF, iC = sC;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int64_t a = __shfl_up_sync(kFullMask, iE, d), c = __shfl_up_sync(kFullMask, iF, d);
            const int64_t k = __shfl_up_sync(kFullMask, iC, d);
            if (lane >= d) {
                iE += a;
                iF += c;
                iC += k;
            }
        }
        if (lane == 31) {
            s_warp[0][warp] = iE;
            s_warp[1][warp] = iF;
            s_warp[2][warp] = iC;
        }
        __syncthreads();
        int64_t bE = 0, bF = 0, bC = 0, TE = 0, TF = 0, TC = 0;
#pragma unroll 8
        for (int w = 0; w < 32; ++w) {
            const int64_t a = s_warp[0][w], c = s_warp[1][w], k = s_warp[2][w];
            if (w < warp) {
                bE += a;
                bF += c;
                bC += k;
            }
            TE += a;
            TF += c;
            TC += k;
        }
        int64_t rE = cE + bE + iE - sE, rF = cF + bF + iF - sF, rC = cC + bC + iC - sC;
#pragma unroll
        for (int u = 0; u < kScanPer; ++u) {
            if (b + u < ntiles) {
                tE[b + u] = rE;
                tF[b + u] = rF;
                tC[b + u] = rC;
            }
            rE += vE[u];
            rF += vF[u];
            rC += mig_cdiv(vE[u], kMigTile);
        }
        cE += TE;
        cF += TF;
        cC += TC;
        __syncthreads();  // s_warp reused by the next round
    }
    if (threadIdx.x == 0) {
        tC[ntiles] = cC;
        if (counts != nullptr) {
            counts[0] = cE;
            counts[1] = cF;
        }
    }
}

// Row copies of one tile: row j of the tile's list (j < n) goes from src_row(j) to dst_row(j).
// When a row is cpr = 2^lg <= 32 chunks, each row is handled by a group of cpr lanes and each
// thread keeps 4 rows' loads in flight; otherwise one chunk per thread and iteration.
template <int CH, class Src, class Dst>
__device__ __forceinline__ void copy_tile_rows(int64_t n, int64_t cpr, int lg, Src src_row, Dst dst_row) {
    using T = typename MigChunk<CH>::T;
    if (lg >= 0) {
        const int c = threadIdx.x & ((1 << lg) - 1);
        const int64_t step = kThreads >> lg;
        int64_t j = threadIdx.x >> lg;
        for (; j + 3 * step < n; j += 4 * step) {
            T v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldcs(reinterpret_cast<const T*>(src_row(j + u * step)) + c);
#pragma unroll
            for (int u = 0; u < 4; ++u) reinterpret_cast<T*>(dst_row(j + u * step))[c] = v[u];
        }
        for (; j < n; j += step) reinterpret_cast<T*>(dst_row(j))[c] = __ldcs(reinterpret_cast<const T*>(src_row(j)) + c);
        return;
    }
    for (int64_t g = threadIdx.x; g < n * cpr; g += kThreads) {
        const int64_t j = g / cpr, c = g - j * cpr;
        reinterpret_cast<T*>(dst_row(j))[c] = __ldcs(reinterpret_cast<const T*>(src_row(j)) + c);
    }
}

// 4c: the extras in NS-15 order, cut into work items of kMigTile ranks (a tile's extras are
// its particles' o_i - 1 copies in order; tile t holds items [tC[t], tC[t+1])).  A persistent
// grid walks the items, so a tile that holds a heavy particle's thousands of extras is copied
// by as many CTAs as it has items (one CTA per tile serialised skewed shards).
// Each item rescans its tile's extras counts and tabulates the owner of each of its ranks.
template <int CH>
__global__ void __launch_bounds__(kThreads) k_mig_pack(const char* __restrict__ X, int64_t ld, int64_t row_bytes,
                                                       int lg, int32_t Pl, int64_t p0, const int32_t* __restrict__ o,
                                                       const int64_t* __restrict__ tE, const int64_t* __restrict__ tC,
                                                       int64_t ntiles, char* __restrict__ send,
                                                       int32_t* __restrict__ send_src) {
    __shared__ int16_t s_map[kMigTile];
    __shared__ int64_t s_warp[kThreads / 32];
    const int64_t items = tC[ntiles];
    for (int64_t w = blockIdx.x; w < items; w += gridDim.x) {
        int64_t lo = 0, hi = ntiles - 1;  // the tile of item w: the last t with tC[t] <= w
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (__ldg(tC + mid) <= w) lo = mid;
            else hi = mid - 1;
        }
        const int64_t t = lo;
        const int64_t t0 = t * kMigTile;
        int32_t e[kMigItems];
        int32_t sum = 0;
#pragma unroll
        for (int j = 0; j < kMigItems; ++j) {
            const int64_t i = t0 + threadIdx.x * kMigItems + j;
            const int32_t v = i < Pl ? __ldg(o + i) : 1;
            e[j] = v > 1 ? v - 1 : 0;
            sum += e[j];
        }
        int64_t ex;
        const int64_t Et = block_excl_scan(sum, &ex, s_warp);
        const int64_t r0 = (w - __ldg(tC + t)) * kMigTile;
        const int64_t r1 = min(Et, r0 + kMigTile);
        int64_t run = ex;
#pragma unroll
        for (int j = 0; j < kMigItems; ++j) {
            const int q = threadIdx.x * kMigItems + j;
            const int64_t a = max(run, r0), b = min(run + e[j], r1);
            for (int64_t c = a; c < b; ++c) s_map[c - r0] = static_cast<int16_t>(q);
            run += e[j];
        }
        __syncthreads();
        const int64_t n = r1 - r0;
        const int64_t base = __ldg(tE + t) + r0;
        if (send_src != nullptr)
            for (int64_t j = threadIdx.x; j < n; j += kThreads)
                send_src[base + j] = static_cast<int32_t>(p0 + t0 + s_map[j]);
        if (row_bytes != 0)
            copy_tile_rows<CH>(n, row_bytes / CH, lg, [&](int64_t j) { return X + (t0 + s_map[j]) * ld; },
                               [&](int64_t j) { return send + (base + j) * row_bytes; });
        __syncthreads();  // s_map is rewritten by the next item
    }
}

// 4d: the tile's free slots take rows tF[t] + r, r = their rank in the tile.
template <int CH>
__global__ void __launch_bounds__(kThreads) k_mig_unpack(char* __restrict__ X, int64_t ld, int64_t row_bytes, int lg,
                                                         int32_t Pl, int64_t p0, const int32_t* __restrict__ o,
                                                         const int64_t* __restrict__ tF,
                                                         const char* __restrict__ recv,
                                                         const int32_t* __restrict__ recv_src,
                                                         int32_t* __restrict__ perm) {
    __shared__ int16_t s_free[kMigTile];
    __shared__ int32_t s_perm[kMigTile];
    __shared__ int64_t s_warp[kThreads / 32];
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kMigTile;
    const int64_t base = tF[blockIdx.x];
    bool fr[kMigItems];
    int32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < kMigItems; ++j) {
        const int64_t i = t0 + threadIdx.x * kMigItems + j;
        fr[j] = i < Pl && __ldg(o + i) == 0;
        cnt += fr[j];
    }
    int64_t ex;
    const int64_t Ft = block_excl_scan(cnt, &ex, s_warp);
    int32_t r = static_cast<int32_t>(ex);
#pragma unroll
    for (int j = 0; j < kMigItems; ++j) {
        const int q = threadIdx.x * kMigItems + j;
        if (perm != nullptr) s_perm[q] = fr[j] ? __ldg(recv_src + base + r) : static_cast<int32_t>(p0 + t0 + q);
        if (fr[j]) s_free[r++] = static_cast<int16_t>(q);
    }
    __syncthreads();
    if (perm != nullptr)
        for (int q = threadIdx.x; q < kMigTile && t0 + q < Pl; q += kThreads) perm[t0 + q] = s_perm[q];
    if (row_bytes == 0 || Ft == 0) return;
    copy_tile_rows<CH>(Ft, row_bytes / CH, lg, [&](int64_t j) { return recv + (base + j) * row_bytes; },
                       [&](int64_t j) { return X + (t0 + s_free[j]) * ld; });
}

int mig_chunk(const void* a, const void* b, int64_t row_bytes, int64_t ld) {
    const uintptr_t p = reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b);
    if ((p & 15) == 0 && row_bytes % 16 == 0 && ld % 16 == 0) return 16;
    if ((p & 3) == 0 && row_bytes % 4 == 0 && ld % 4 == 0) return 4;
    return 1;
}

// log2 of the chunks per row when that is a power of two <= 32, else -1
int mig_lg(int64_t cpr) {
    for (int lg = 0; lg <= 5; ++lg)
        if (cpr == (int64_t{1} << lg)) return lg;
    return -1;
}

}  // namespace

// plan: tE [ntiles], tF [ntiles], tC [ntiles + 1] (int64)
size_t mig_plan_bytes(int32_t Pl) { return sizeof(int64_t) * (3 * static_cast<size_t>(mig_cdiv(Pl, kMigTile)) + 1); }

cudaError_t launch_mig_offspring(const int32_t* anc, int64_t n_anc, const int64_t* range, int64_t win0, int32_t Pw,
                                 const float* gmax, const int32_t* gbad, int32_t* o, cudaStream_t s,
                                 uint64_t* launches) {
    cudaError_t e = cudaMemsetAsync(o, 0, sizeof(int32_t) * static_cast<size_t>(Pw), s);
    if (e != cudaSuccess) return e;
    const int64_t work = std::max<int64_t>(n_anc, Pw);
    const unsigned grid = static_cast<unsigned>(
        std::max<int64_t>(1, std::min<int64_t>(mig_cdiv(work, kThreads), static_cast<int64_t>(sm_count()) * 8)));
    ProfScope ps_("k_mig_offspring", s);
    if (range != nullptr) k_mig_offspring_runs<<<grid, kThreads, 0, s>>>(anc, n_anc, range, win0, Pw, gmax, gbad, o);
    else k_mig_offspring<<<grid, kThreads, 0, s>>>(anc, n_anc, win0, Pw, gmax, gbad, o);
    ++*launches;
    return cudaPeekAtLastError();
}

// the plan = the tiles' exclusive prefixes (tE = plan, tF = plan + ntiles) and the pack work
// items' prefix (tC = plan + 2 ntiles, ntiles + 1 entries); counts nullable
cudaError_t launch_mig_plan(const int32_t* o, int32_t Pl, void* plan, int64_t* counts, cudaStream_t s,
                            uint64_t* launches) {
    const int64_t nt = mig_cdiv(Pl, kMigTile);
    int64_t* tE = static_cast<int64_t*>(plan);
    int64_t* tF = tE + nt;
    {
        ProfScope ps_("k_mig_tile_counts", s);
        k_mig_tile_counts<<<static_cast<unsigned>(nt), kThreads, 0, s>>>(o, Pl, tE, tF);
    }
    {
        ProfScope ps_("k_mig_tile_scan", s);
        k_mig_tile_scan<<<1, 1024, 0, s>>>(tE, tF, tF + nt, nt, counts);
    }
    *launches += 2;
    return cudaPeekAtLastError();
}

cudaError_t launch_mig_pack(const void* X, int64_t row_bytes, int64_t ld, int32_t Pl, int64_t p0, const int32_t* o,
                            const void* plan, void* send, int32_t* send_src, cudaStream_t s, uint64_t* launches) {
    const int64_t nt = mig_cdiv(Pl, kMigTile);
    const int64_t* tE = static_cast<const int64_t*>(plan);
    const int64_t* tC = tE + 2 * nt;
    const char* x = static_cast<const char*>(X);
    char* y = static_cast<char*>(send);
    const int ch = row_bytes > 0 ? mig_chunk(x, y, row_bytes, std::max<int64_t>(ld, row_bytes)) : 16;
    const int lg = row_bytes > 0 ? mig_lg(row_bytes / ch) : 0;
    // persistent over the work items (their count is on the device): enough CTAs for the
    // balanced case, and every SM busy when one tile holds most of the extras
    const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(
        std::max<int64_t>(nt, static_cast<int64_t>(sm_count()) * 4), static_cast<int64_t>(sm_count()) * 8)));
    ProfScope ps_("k_mig_pack", s);
    if (ch == 16) k_mig_pack<16><<<grid, kThreads, 0, s>>>(x, ld, row_bytes, lg, Pl, p0, o, tE, tC, nt, y, send_src);
    else if (ch == 4) k_mig_pack<4><<<grid, kThreads, 0, s>>>(x, ld, row_bytes, lg, Pl, p0, o, tE, tC, nt, y, send_src);
    else k_mig_pack<1><<<grid, kThreads, 0, s>>>(x, ld, row_bytes, lg, Pl, p0, o, tE, tC, nt, y, send_src);
    ++*launches;
    return cudaPeekAtLastError();
}

cudaError_t launch_mig_unpack(void* X, int64_t row_bytes, int64_t ld, int32_t Pl, int64_t p0, const int32_t* o,
                              const void* plan, const void* recv, const int32_t* recv_src, int32_t* perm,
                              cudaStream_t s, uint64_t* launches) {
    const int64_t* tF = static_cast<const int64_t*>(plan) + mig_cdiv(Pl, kMigTile);
    char* x = static_cast<char*>(X);
    const char* y = static_cast<const char*>(recv);
    const int ch = row_bytes > 0 ? mig_chunk(x, y, row_bytes, std::max<int64_t>(ld, row_bytes)) : 16;
    const int lg = row_bytes > 0 ? mig_lg(row_bytes / ch) : 0;
    const unsigned grid = static_cast<unsigned>(mig_cdiv(Pl, kMigTile));
    ProfScope ps_("k_mig_unpack", s);
    if (ch == 16) k_mig_unpack<16><<<grid, kThreads, 0, s>>>(x, ld, row_bytes, lg, Pl, p0, o, tF, y, recv_src, perm);
    else if (ch == 4) k_mig_unpack<4><<<grid, kThreads, 0, s>>>(x, ld, row_bytes, lg, Pl, p0, o, tF, y, recv_src, perm);
    else k_mig_unpack<1><<<grid, kThreads, 0, s>>>(x, ld, row_bytes, lg, Pl, p0, o, tF, y, recv_src, perm);
    ++*launches;
    return cudaPeekAtLastError();
}

}  // namespace pf
