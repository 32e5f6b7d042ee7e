// pf_fused.cu — one-launch resamplers (
// NEXT-2): k_fused_sorted (a cluster per filter, P <= 8 x 8192), k_coop_sorted
// (a cooperative grid per filter, larger P), k_small (a warp per filter, P <= 256).
//
// k_fused_sorted: one thread-block CLUSTER per filter (CL = ceil(P / 8192) CTAs of
// 512 threads, 16 particles each), persistent over filters.  CTA c owns particles
// [c*PP, (c+1)*PP).
//   A  log-weights -> registers (float4, coalesced); CTA max; cluster max
//      through distributed shared memory (a1, NS-1, NS-2).
//   B  w = dexp, q = trunc(w 2^kfx) (a2, NS-3..5); block scan of q in
//      registers + shared memory; a DSMEM exchange of the CTA totals gives the
//      CTA offset O_c and the filter total Q (a3 — the paper's "collective
//      prefix-sum", without a second launch); lse / ESS / v_i fused
//      (a12, NS-13).
//   C  positions are sorted (NS-9, NS-10), so the slots landing in particle i
//      are [E_{i-1}, E_i) with E_i = c(Q_i) = #{k : x_k < Q_i}.  c() has a
//      closed form: x_k < v  <=>  k*D + rho_k < v 2^64 / Q; a double-precision
//      estimate of k* = (v 2^64/Q - rho)/D is within 2^-19 of the truth, so one
//      exact integer position check decides the count (the boundary case takes
//      a second check).  Per chunk of 8 slots per thread, particle i marks
//      heads[E_{i-1}] = i when E_i > E_{i-1}, and a CTA-wide max-scan gives every
//      ancestor a_k = max{i : E_{i-1} <= k} = min{i : Q_i > x_k} (a4+a5); the
//      offspring o_i = E_i - E_{i-1} is a free by-product (a8).
//   D  (optional) canonical permutation (a9, NS-15): a packed (extras, free) scan
//      across the cluster, every CTA's free-slot list in its shared memory, and a
//      CTA-wide head-mark + max-scan over its extras ranks; the r-th extra goes to
//      the r-th free slot, read from the owning CTA's list through DSMEM.
// HBM traffic: 4 B/particle in (logw) + 4 B out per output array.  No workspace.
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <type_traits>
#include <cstdlib>
#include <cmath>

#include "pf_device.cuh"
#include "pf_internal.h"

namespace cg = cooperative_groups;

namespace pf {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
// threads per CTA of the cooperative kernel and of the cluster kernel up to P = 65536: 512
// (2 CTAs / SM, so one CTA's barriers overlap the other's work; measured 4% faster than
// 1024 x 1 at C3 and 1.4x at single filters of 2^18-2^20).  The cluster kernel takes 1024
// threads (16384 particles per CTA, clusters of up to 16) for 65536 < P <= 262144.
constexpr int kFT = 512;
constexpr int kMaxCL = 16;  // largest cluster (non-portable above 8)
constexpr int kFW = kFT / 32;      // warps per CTA
constexpr int kFI = 16;            // particles per thread
constexpr int kFR = kFI / 4;       // 4 float4 rows
constexpr int kPP = kFT * kFI;     // particles per CTA (max): 8192
constexpr int kChunk = 256;        // slots per warp max-scan pass (8 per lane)
constexpr int kXS = kFW * kChunk;   // slots (ranks) per CTA-wide expansion chunk: 8 per thread
static_assert(kXS == 8 * kFT, "CTA-wide expansion assumes 8 slots per thread");
static_assert(kFW <= 32, "the cross-warp max-scan reads one warp total per lane");
static_assert(kFR * kFW % 32 == 0, "phase-B totals scan assumes a multiple of 32 (row, warp) totals");

struct Exchange {
    float m;
    int bad;
    double m64;  // binary64 input (NS-3d): the CTA's max of the doubles
    uint64_t tot;
    double sw, sw2;
    uint64_t ptot;  // packed (extras << 31 | free) total of the CTA (phase D)
};

// SCHEME value of the cluster kernel's multinomial bucket mode: the systematic machinery with
// rho = 0 over NB = 2^ceil(log2 P) slots at b 2^(64 - m) gives the bucket index of the
// multinomial search, idx[b] = min{i : Q_i > floor(b Q / NB)} (pf_kernels.cu ModeBuckets), and
// Q is written
constexpr int kBuckets = 5;
// SCHEME value of the permutation-from-offspring mode: phases A-C are replaced by reading the
// offspring counts (a8's output, e.g. the histogram of the multinomial's or Metropolis' unsorted
// ancestors); phase D builds the canonical permutation NS-15 and gathers the state NS-16
constexpr int kFromOffspring = 6;

struct FusedArgs {
    const float* logw;
    uint64_t* Qout;      // kBuckets: Q [N][ldq] and the filter totals
    int64_t ldq;
    int32_t S;           // kBuckets: bucket count NB = 2^ceil(log2 P) (the slots of the expansion)
    uint64_t* Qtot_out;
    const double* logw64;  // F64 instantiations: binary64 log-weights (NS-3d), same ld
    int64_t ld;
    int32_t N, P, CL, PP;
    uint64_t D;
    Key key;
    uint32_t filt0;
    int kfx;
    int vec;       // logw rows 16-byte aligned
    int sums;      // lse / ess / normw requested
    int32_t* anc;
    int64_t ld_anc;
    int anc_vec;   // ancestor rows 16-byte aligned
    double* lse_out;
    double* ess_out;
    float* normw;
    int32_t* status_out;
    int32_t* off;   // offspring out (row stride ld_anc), nullable
    const int32_t* off_in;  // kFromOffspring: the offspring counts (row stride ld_off_in)
    int64_t ld_off_in;
    int32_t* perm;  // canonical permutation out (row stride ld_anc), nullable
    char* X;        // state rows gathered in place (PERM), nullable: filter n at X + n * xfld
    int64_t xld;    // bytes between rows
    int64_t xfld;   // bytes between filters
    int xlg;        // log2 of the 16-byte chunks per row (row bytes = 16 << xlg)
};

#ifndef PF_STRAT_DBL
#define PF_STRAT_DBL 1  // stratified check decided in double away from the boundary
#endif
struct Pos {
    uint64_t D, Qtot, rho;
    Key key;
    uint32_t filt;
    int64_t P;
    double A, Bc;  // k* = v * A - Bc
    double C;      // A 2^kfx: k* advances by about w C per particle of weight w (PF_KF_RUN)
};

template <int SCHEME>
__device__ __forceinline__ uint64_t xpos(const Pos& z, int64_t k) {
    uint64_t rho = z.rho;
    if (SCHEME == 2) {
        const u32x4 r = philox10(static_cast<uint32_t>(k >> 1), 0u, 2u, z.filt, z.key.k0, z.key.k1);
        rho = mulhi64((k & 1) ? hi_word(r) : lo_word(r), z.D);
    }
    return mulhi64(static_cast<uint64_t>(k) * z.D + rho, z.Qtot);
}

// c(v) = #{k in [0, P) : x_k < v}
template <int SCHEME>
__device__ __forceinline__ uint32_t count_below(const Pos& z, uint64_t v) {
    const double kf = fma(static_cast<double>(v), z.A, -z.Bc);
    const double fl = floor(kf);
    const double fr = kf - fl;
    int64_t c;
    if (fr > 0x1p-12 && fr < 1.0 - 0x1p-12) {
        const int64_t n = static_cast<int64_t>(fl);
        if (SCHEME == 3) {
            c = n + 1;  // k* in (n, n+1): exactly the k <= n count (clamped below)
        } else {
            // strata k < n lie below v, k > n above; stratum n decides itself
            c = (n < 0) ? 0 : ((n >= z.P) ? z.P : n + (xpos<SCHEME>(z, n) < v ? 1 : 0));
        }
    } else {
        const int64_t m0 = llrint(kf);
        if (SCHEME == 3) {
            c = m0 + ((m0 >= 0 && m0 < z.P && xpos<SCHEME>(z, m0) < v) ? 1 : 0);
        } else {
            const int64_t a = m0 - 1;
            c = min(max(a, int64_t{0}), z.P);
            if (a >= 0 && a < z.P && xpos<SCHEME>(z, a) < v) ++c;
            if (m0 >= 0 && m0 < z.P && xpos<SCHEME>(z, m0) < v) ++c;
        }
    }
    return static_cast<uint32_t>(min(max(c, int64_t{0}), z.P));
}

// Systematic: the common case of count_below without branches (32-bit clamp); *slow is set
// when k* is within 2^-12 of an integer, where the caller recomputes with count_below.
__device__ __forceinline__ uint32_t count_below_sys_fast(const Pos& z, uint64_t v, bool* slow) {
    const double kf = fma(static_cast<double>(v), z.A, -z.Bc);
    const double fl = floor(kf);
    const double fr = kf - fl;
    *slow = !(fr > 0x1p-12 && fr < 1.0 - 0x1p-12);
    const int n1 = static_cast<int>(fl) + 1;  // kf in [-1, P]: fits in 32 bits
    return static_cast<uint32_t>(min(max(n1, 0), static_cast<int>(z.P)));
}

// Stratified: the common case (k* not within 2^-12 of an integer), branch-free: stratum n
// decides itself by one exact position check (strata below n lie below v, above n above).
template <bool SD = false>
__device__ __forceinline__ uint32_t count_below_strat_fast(const Pos& z, uint64_t v, bool* slow) {
    const double kf = fma(static_cast<double>(v), z.A, -z.Bc);
    const double fl = floor(kf);
    const double fr = kf - fl;
    *slow = !(fr > 0x1p-12 && fr < 1.0 - 0x1p-12);
    const int P = static_cast<int>(z.P);
    const int n = static_cast<int>(fl);
    const int nc = min(max(n, 0), P - 1);
    const u32x4 r = philox10(static_cast<uint32_t>(nc >> 1), 0u, 2u, z.filt, z.key.k0, z.key.k1);
    const uint64_t R = (nc & 1) ? hi_word(r) : lo_word(r);
    // x_n < v  <=>  rho_n < fr D  <=>  rho_n / D < fr, and rho_n / D = mulhi(R, D) / D lies in
    // (R 2^-64 - 1/D, R 2^-64]: decided in double away from the boundary (|kf| error < 2^-19 for
    // k* < 2^31, 1/D <= 2^-33, so a 2^-18 band is safe), exactly within it (rare)
    uint32_t below;
    const double u = static_cast<double>(R) * 0x1p-64;
    if (SD && u + 0x1p-18 < fr) {
        below = 1u;
    } else if (SD && u > fr + 0x1p-18) {
        below = 0u;
    } else {
        const uint64_t rho = mulhi64(R, z.D);
        below = (mulhi64(static_cast<uint64_t>(nc) * z.D + rho, z.Qtot) < v) ? 1u : 0u;
    }
    return (n < 0) ? 0u : (n >= P ? static_cast<uint32_t>(P) : static_cast<uint32_t>(n) + below);
}

#ifndef PF_EARLY_RHO
#define PF_EARLY_RHO 1
#endif
#ifndef PF_KF_RUN
#define PF_KF_RUN 1  // systematic slot counts: k* estimate advanced by w C (count_row<3, true>)
#endif
// E for the 4 particles of a row: running sum from run0, fast paths with an exact redo of the
// (rare) rows holding a near-integer k*
template <int SCHEME, bool KFR = false, bool SD = false>
__device__ __forceinline__ void count_row(const Pos& z, uint64_t run0, const float* w4, int kfx, uint32_t* E4) {
    if (SCHEME == 3) {
        bool any_slow = false;
        uint64_t run = run0;
        if (KFR && z.A < 0x1p-16) {
            // the estimate of k* from the row's exact start, advanced by w C per particle
            // instead of quantising each weight and converting each Q_i: it differs from the
            // per-particle estimate by the quantiser's truncations (< 1 unit of q each, i.e.
            // < A in k*; A = 2^64 / (D Q) <= S 2^-kfx, at most 2^-23 for S <= 2^18, and the
            // filter-uniform test A < 2^-16 keeps four of them below 2^-14 at any P) and by
            // roundings (<= 2^-20 for k* < 2^31): inside the 2^-12 margin that sends
            // near-integer k* to the exact recount below
            double kf = fma(static_cast<double>(run0), z.A, -z.Bc);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                kf = fma(static_cast<double>(w4[q]), z.C, kf);
                const double fl = floor(kf);
                const double fr = kf - fl;
                any_slow |= !(fr > 0x1p-12 && fr < 1.0 - 0x1p-12);
                const int n1 = static_cast<int>(fl) + 1;
                E4[q] = static_cast<uint32_t>(min(max(n1, 0), static_cast<int>(z.P)));
            }
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                run += quantise(w4[q], kfx);
                bool sl;
                E4[q] = count_below_sys_fast(z, run, &sl);
                any_slow |= sl;
            }
        }
        if (any_slow) {
            run = run0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                run += quantise(w4[q], kfx);
                E4[q] = count_below<SCHEME>(z, run);
            }
        }
    } else {
        bool any_slow = false;
        uint64_t run = run0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            run += quantise(w4[q], kfx);
            bool sl;
            E4[q] = count_below_strat_fast<SD>(z, run, &sl);
            any_slow |= sl;
        }
        if (any_slow) {
            run = run0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                run += quantise(w4[q], kfx);
                E4[q] = count_below<SCHEME>(z, run);
            }
        }
    }
}

// Cluster-wide barrier without a cluster-scope release on every thread: only the threads that
// wrote data other CTAs (or other threads) read after the barrier fence their writes
// (fence.acq_rel.cluster, the documented release pattern for barrier.cluster.arrive.relaxed);
// the wait keeps its acquire semantics.  Every other thread skips the memory barrier, which
// otherwise waits for all of its outstanding global stores (the state copies, the outputs).
__device__ __forceinline__ void cluster_sync_publish(bool publisher) {
    if (publisher) asm volatile("fence.acq_rel.cluster;" ::: "memory");
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

// a10 fused: one warp copies npairs rows X[slot[p]] <- X[owner[p]] of filter n
// ((16 << xlg) bytes each), 16 bytes per lane, kCopyU chunks in flight per lane.
#ifndef PF_COPY_U
#define PF_COPY_U 4
#endif
constexpr int kCopyU = PF_COPY_U;
// Deferred state copy (max-ahead instantiations with the gather): every warp keeps the (free
// slot, owner) pairs it produced in phase D in a private ring and copies their rows in "ticks"
// spread over the NEXT filter's phases: a tick stores the rows staged by the previous tick
// (cp.async, 16 bytes per lane, into shared memory: no registers held while in flight) and
// stages the next kCU x (32 / chunks-per-row) rows.  The copy's memory latency hides under
// the compute of the following phases instead of stalling the warp at the end of phase D.
#ifndef PF_COPY_CU
#define PF_COPY_CU 3
#endif
#ifndef PF_COPY_CU256
#define PF_COPY_CU256 8
#endif
// chunks per lane per tick: 256-thread CTAs with the gather run 3 per SM (85 registers, room
// for larger staged batches)
template <int FT>
__host__ __device__ constexpr int copy_cu() {
    return FT == 256 ? PF_COPY_CU256 : PF_COPY_CU;
}
// the deferred copy runs in the systematic instantiations (stratified's per-particle Philox in
// phase C leaves no registers for the ticks: its step was 1.96 -> 2.40 ms with them)
template <int SCHEME, int PERM, int FT, bool F64>
__host__ __device__ constexpr bool fused_deferred_copy() {
#ifndef PF_DC_OFFIN
#define PF_DC_OFFIN 0  // from offspring the copy has no later phases to hide under: in-line copy (1.59 -> 1.42 ms at C3 multinomial)
#endif
    return FT <= 512 && !F64 && PERM == 2 && (SCHEME == 3 || (PF_DC_OFFIN && SCHEME == kFromOffspring));
}
#ifndef PF_FT256_DC_BLOCKS
#define PF_FT256_DC_BLOCKS 3
#endif
template <int FT, int PERM>
__host__ __device__ constexpr int fused_min_blocks() {
    return (FT == 256 && PERM == 2) ? PF_FT256_DC_BLOCKS : 1024 / FT;
}
constexpr int kRQ = 256;  // ring entries per warp: packed (slot << 16 | owner), P <= 65536
#ifndef PF_ROW_SKIP
#define PF_ROW_SKIP 1  // expansion marks: skip a thread's rows whose slots miss the chunk
#endif
#ifndef PF_PF_L2
#define PF_PF_L2 1  // deferred copy: L2 prefetch of each pair's owner row when the pair is queued
                    // (C3 step 1.350 -> 1.333 ms; prefetching every owner at once instead -- at
                    // the end of phase C, or before the in-line copies of other schemes -- floods
                    // L2 and the memory system: 1.58 ms, stratified step 2.0 -> 2.4 ms)
#endif
#ifndef PF_COOP_RESIDENT
#define PF_COOP_RESIDENT 1  // cooperative kernel: one sub-tile per CTA keeps its values in registers
#endif
#ifndef PF_ROWSCAN
#define PF_ROWSCAN 1  // the four row scans of phases B and D as one transposed warp scan
#endif
#ifndef PF_FFMA2
#define PF_FFMA2 1  // phase B's dexp on packed f32x2 (FFMA2 / FMUL2)
#endif
#ifndef PF_TICK_B
#define PF_TICK_B 1  // a tick after each row of phase B
#endif
#ifndef PF_TICK_C
#define PF_TICK_C 1  // a tick after each row's slot counts in phase C
#endif
#ifndef PF_PREFETCH_NEXT
#define PF_PREFETCH_NEXT 1
#endif
template <class Args>
__device__ __forceinline__ void copy_rows_warp(const Args& a, int n, const int32_t* owner, const int32_t* slot,
                                               int npairs, int lane) {
    char* Xf = a.X + static_cast<int64_t>(n) * a.xfld;
    // a lane always handles the same 16-byte chunk of a row (32 is a multiple of the chunks per
    // row); rows of one filter are < 2^32 bytes apart (P <= 65536 rows of <= 512 bytes)
    const uint32_t ch = static_cast<uint32_t>(lane & ((1 << a.xlg) - 1)) * 16u;
    const int rstep = 32 >> a.xlg;  // rows per warp instruction
    const uint32_t xld = static_cast<uint32_t>(a.xld);
    int p = lane >> a.xlg;
    // full rounds without per-item predicates (no divergent branches around the loads), then
    // the tail item by item
    for (; p + (kCopyU - 1) * rstep < npairs; p += kCopyU * rstep) {
        int4 v[kCopyU];
#pragma unroll
        for (int u = 0; u < kCopyU; ++u)
            v[u] = __ldcg(reinterpret_cast<const int4*>(Xf + (static_cast<uint32_t>(owner[p + u * rstep]) * xld + ch)));
#pragma unroll
        for (int u = 0; u < kCopyU; ++u)
            __stcg(reinterpret_cast<int4*>(Xf + (static_cast<uint32_t>(slot[p + u * rstep]) * xld + ch)), v[u]);
    }
    for (; p < npairs; p += rstep)
        __stcg(reinterpret_cast<int4*>(Xf + (static_cast<uint32_t>(slot[p]) * xld + ch)),
               __ldcg(reinterpret_cast<const int4*>(Xf + (static_cast<uint32_t>(owner[p]) * xld + ch))));
}

// Max-ahead mode (512-thread float32 instantiations): the CTA's slice of the NEXT filter's
// log-weights arrives in shared memory by one bulk asynchronous copy (cp.async.bulk, mbarrier
// completion) issued as soon as the current filter's values are in registers; its CTA maximum
// is formed during phase B and travels with the scan totals at the cluster exchange, so a
// filter needs one cluster barrier without the permutation (was two) and two with it (was
// four: the free-slot lists are built before the packed totals are exchanged).  The exchange
// words are double-buffered by filter parity, which makes one barrier per filter enough.
template <int FT, bool F64>
__host__ __device__ constexpr bool fused_max_ahead() {
    return FT <= 512 && !F64;
}

// Exclusive prefix sums across the warp's lanes of R rows at once (R = 2 or 4): ex[j] = sum
// over lanes l' < lane of loc[j] (what R warp_incl_scan_u64 calls give), through the warp's
// R x 256 B of shared memory buf (16-byte aligned, warp-private): lane l sums the R-lane
// segment l % (32 / R) of row l / (32 / R) serially, a (32 / R)-lane shuffle scan runs over the
// segments, and the prefixes go back through buf.  One 3- (4-) step 64-bit shuffle scan
// instead of four (two) 5-step ones.  *rowtot: the total of row l / (32 / R), valid on the last
// lane of each row's group.
template <int R>
__device__ __forceinline__ void warp_rows_excl_scan(const uint64_t* loc, uint64_t* ex, uint64_t* buf, int lane,
                                                    uint64_t* rowtot) {
    static_assert(R == 2 || R == 4, "two or four rows");
    constexpr int kSeg = 32 / R;  // segments per row = lanes per row group
#pragma unroll
    for (int j = 0; j < R; ++j) buf[j * 32 + lane] = loc[j];
    __syncwarp();
    const int seg = lane % kSeg;
    ulonglong2* p = reinterpret_cast<ulonglong2*>(buf + (lane / kSeg) * 32 + seg * R);
    uint64_t e[R];  // inclusive partial sums of the segment
    const ulonglong2 a = p[0];
    e[0] = a.x;
    e[1] = a.x + a.y;
    if (R == 4) {
        const ulonglong2 b = p[1];
        e[2 % R] = e[1] + b.x;
        e[3 % R] = e[2 % R] + b.y;
    }
    const uint64_t T = e[R - 1];
    uint64_t inc = T;
#pragma unroll
    for (int o = 1; o < kSeg; o <<= 1) {
        const uint64_t t = __shfl_up_sync(0xFFFFFFFFu, inc, o, kSeg);
        if (seg >= o) inc += t;
    }
    *rowtot = inc;
    const uint64_t base = inc - T;
    __syncwarp();
    p[0] = make_ulonglong2(base, base + e[0]);
    if (R == 4) p[1] = make_ulonglong2(base + e[1], base + e[2 % R]);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < R; ++j) ex[j] = buf[j * 32 + lane];
    __syncwarp();
}

// IEEE max that propagates NaN (max.NaN.f32): the max of a set is NaN iff a member is
__device__ __forceinline__ float fmax_nan(float a, float b) {
    float d;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}" ::"r"(
            smem_addr(bar)),
        "r"(parity)
        : "memory");
}
// one thread: bytes (a multiple of 16, 16-byte aligned ends) from global src into shared dst,
// completion counted on bar (the caller waits on the barrier's current phase)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of dst
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

// PERM: 0 ancestors (+ offspring) only, 1 + canonical permutation, 2 + in-place state gather
template <int SCHEME, bool SUMS, int PERM, int FT, int FI, bool F64 = false>
__global__ void __launch_bounds__(FT, (fused_min_blocks<FT, PERM>())) k_fused_sorted(FusedArgs a) {
    // geometry of this instantiation: FT threads x FI particles per thread (FT = 512, FI = 16:
    // 8192 particles per CTA, clusters of <= 8; FT = 1024, FI = 16: 16384 per CTA, clusters of
    // <= 16 for 65536 < P <= 262144)
    constexpr int kFT = FT;
    constexpr int kFW = FT / 32;
    constexpr int kFI = FI;
    constexpr int kFR = FI / 4;
    constexpr int kPP = FT * FI;
    constexpr int kTPL = kFR * kFW / 32;
    constexpr int kXS = kFW * kChunk;
    constexpr bool OFFIN = (SCHEME == kFromOffspring);
    constexpr bool MA = fused_max_ahead<FT, F64>() && !OFFIN;  // the next filter's slice in s_lw
    constexpr bool MD = fused_max_ahead<FT, F64>();             // phase D with 16-bit lists, one barrier
    constexpr int kCU = copy_cu<FT>();
    static_assert(kXS == 8 * kFT && kFW <= 32 && kFR * kFW % 32 == 0, "fused kernel geometry");
    // rho and rho / D at the top of each filter by the last warp (PF_EARLY_RHO), except in the
    // ancestors-only 256-thread form, where the 8 warps cannot hide that warp's extra latency
    // (measured: step 1.312 -> 1.281 ms, permutation 0.701 -> 0.688 ms, ancestors-only
    // 0.382 -> 0.391 ms, which therefore keeps them after the exchange)
    constexpr bool kEarlyRho = PF_EARLY_RHO && !(FT == 256 && PERM == 0);
    static_assert((kFR == 2 || kFR == 4) && kChunk * 4 >= kFR * 32 * 8, "warp_rows_excl_scan: rows of s_buf per warp");
    // phase D's packed scan transposed too, except in the gather-from-offspring form (measured
    // 0.02 ms slower at the C3 multinomial step: its registers spill more)
    constexpr bool RS_D = PF_ROWSCAN && !(SCHEME == kFromOffspring && PERM == 2);
    extern __shared__ __align__(16) int32_t s_dyn[];
    float* s_lw = reinterpret_cast<float*>(s_dyn);  // MA: this CTA's slice of the next filter's log-weights
    // PERM: this CTA's free-slot list (kPP entries; 16-bit slots in the max-ahead mode, P <= 65536;
    // from offspring: two lists, by filter parity, as only one cluster barrier separates filters)
    using FsT = std::conditional_t<MD, uint16_t, int32_t>;
    constexpr bool DC = fused_deferred_copy<SCHEME, PERM, FT, F64>();  // deferred, asynchronous state copy
    constexpr int kFsN = OFFIN ? 2 : 1;
    FsT* const s_fs0 = reinterpret_cast<FsT*>(s_dyn + (MA ? kPP : 0));
    FsT* s_fs = s_fs0;
    int32_t* s_pslot = reinterpret_cast<int32_t*>(s_fs0 + kFsN * kPP);  // PERM == 2 (not DC): free slot per extras rank
    uint32_t* s_ring = reinterpret_cast<uint32_t*>(s_fs0 + kFsN * kPP);  // DC: kFW rings of kRQ pairs
    int4* s_stage = reinterpret_cast<int4*>(s_ring + kFW * kRQ); // DC: kFW x kCU x 32 staged chunks
    __shared__ Exchange s_xx[2];                    // MA: double-buffered by filter parity
    __shared__ uint64_t s_mbar;
    __shared__ uint32_t s_rf[kMaxCL + 1];
    __shared__ uint64_t s_poff;
    __shared__ float s_f[kFW];
    __shared__ int s_i[kFW];
    __shared__ double s_d[2][kFW];
    __shared__ uint64_t s_wt[kFR][kFW];
    __shared__ uint32_t s_lastE[kFR][kFW];
    __shared__ __align__(16) int32_t s_buf[kFW][kChunk];
    __shared__ int32_t s_wmax[kFW];
    __shared__ float s_lmax;
    __shared__ double s_lmax64;
    __shared__ double s_m64[kFW];
    __shared__ int s_bad;
    __shared__ uint64_t s_off, s_tot, s_Qtot;
    __shared__ double s_S, s_S2;
    __shared__ uint32_t s_klo;
    __shared__ uint64_t s_rho;
    __shared__ double s_zA, s_zBc;

    cg::cluster_group cluster = cg::this_cluster();
    const int c = static_cast<int>(cluster.block_rank());
    const int CL = a.CL;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int num_clusters = gridDim.x / CL;
    const int cid = blockIdx.x / CL;
    // this CTA's particle range is the same for every filter
    const int64_t p0 = static_cast<int64_t>(c) * a.PP;
    const int64_t p1 = min(static_cast<int64_t>(a.P), p0 + a.PP);
    const int np = static_cast<int>(max(int64_t{0}, p1 - p0));

    // ---- MA helpers: the next filter's slice into s_lw, its CTA max / invalid flag from s_lw
    const bool lw_bulk = MA && a.vec && np > 0 && (np & 3) == 0;
    uint32_t lw_phase = 0;
    auto lw_issue = [&](int nn) {  // all threads, after a barrier that ends every read of s_lw
        const float* src = a.logw + static_cast<int64_t>(nn) * a.ld + p0;
        if (lw_bulk) {
            if (tid == 0) bulk_g2s(s_lw, src, static_cast<uint32_t>(np) * 4u, &s_mbar);
        } else {
            for (int i = tid; i < np; i += kFT) s_lw[i] = __ldcs(src + i);
        }
    };
    auto lw_wait = [&]() {  // all threads
        if (lw_bulk) {
            mbar_wait(&s_mbar, lw_phase);
            lw_phase ^= 1u;
        } else {
            __syncthreads();
        }
    };
    // CTA partials of max / invalid flag of the slice in s_lw into s_f / s_i (the caller
    // synchronises before warp 0 reads them)
    auto lw_partials = [&]() {
        float m = -INFINITY;
        bool bad = false;
#pragma unroll
        for (int j = 0; j < kFR; ++j) {
            const int i0 = j * (kFT * 4) + tid * 4;
            float x[4];
            if (i0 + 3 < np) {
                const float4 t = *reinterpret_cast<const float4*>(s_lw + i0);
                x[0] = t.x; x[1] = t.y; x[2] = t.z; x[3] = t.w;
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) x[q] = (i0 + q < np) ? s_lw[i0 + q] : -INFINITY;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) m = fmax_nan(m, x[q]);  // a NaN anywhere stays NaN
        }
        bad = !(m <= FLT_MAX);  // NaN or +inf among the values (one test, not one per value)
        int b = bad ? 1 : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
            b |= __shfl_xor_sync(kFull, b, o);
        }
        if (lane == 0) { s_f[warp] = m; s_i[warp] = b; }
    };
    // warp 0 after the barrier that follows lw_partials: CTA max / flag into the exchange
    auto lw_cta_reduce = [&](Exchange& x) {
        float mm = (lane < kFW) ? s_f[lane] : -INFINITY;
        int bb = (lane < kFW) ? s_i[lane] : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mm = fmaxf(mm, __shfl_xor_sync(kFull, mm, o));
            bb |= __shfl_xor_sync(kFull, bb, o);
        }
        if (lane == 0) { x.m = mm; x.bad = bb; }
    };
    // warp 0 after the cluster barrier: the filter maximum / invalid flag from every CTA's exchange
    auto lw_cluster_reduce = [&](int xb) {
        float gm = -INFINITY;
        int gb = 0;
        if (lane < CL) {
            const Exchange* rx = cluster.map_shared_rank(&s_xx[xb], lane);
            gm = rx->m;
            gb = rx->bad;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            gm = fmaxf(gm, __shfl_xor_sync(kFull, gm, o));
            gb |= __shfl_xor_sync(kFull, gb, o);
        }
        if (lane == 0) {
            s_lmax = gm;
            s_bad = (gb || gm == -INFINITY) ? 1 : 0;
        }
    };
    // ---- DC: this warp's ring of (slot, owner) pairs of filter rq_n and its staged batch
    uint32_t rq_head = 0, rq_tail = 0, rq_nb = 0;  // pairs stored, produced, staged (in flight)
    int rq_n = 0;
    const int cxl = a.xlg;
    const int rstep = 32 >> cxl;                          // rows per warp instruction
    const uint32_t cch = static_cast<uint32_t>(lane & ((1 << cxl) - 1)) * 16u;  // this lane's chunk
    const uint32_t csub = static_cast<uint32_t>(lane >> cxl);                   // this lane's row
    const uint32_t cxld = static_cast<uint32_t>(a.xld);
    uint32_t* const ring = s_ring + warp * kRQ;
    int4* const stage = s_stage + warp * (kCU * 32);
    // a tick: wait for the batch staged by the previous tick (each lane reads back only its own
    // chunks, so the lane's cp.async wait is all it needs), store its rows to their free slots,
    // then stage the next batch of the ring.  Whole warp, uniform.
    auto tick = [&]() {
        if constexpr (DC) {
            if (rq_nb) {
                asm volatile("cp.async.wait_all;" ::: "memory");
                char* Xf = a.X + static_cast<int64_t>(rq_n) * a.xfld;
#pragma unroll
                for (int u = 0; u < kCU; ++u) {
                    const uint32_t k = static_cast<uint32_t>(u * rstep) + csub;
                    if (k < rq_nb) {
                        const uint32_t e = ring[(rq_head + k) & (kRQ - 1)];
                        __stcg(reinterpret_cast<int4*>(Xf + ((e >> 16) * cxld + cch)), stage[u * 32 + lane]);
                    }
                }
                rq_head += rq_nb;
                rq_nb = 0;
            }
            const uint32_t avail = rq_tail - rq_head;
            if (avail) {
                rq_nb = min(avail, static_cast<uint32_t>(kCU * rstep));
                const char* Xf = a.X + static_cast<int64_t>(rq_n) * a.xfld;
#pragma unroll
                for (int u = 0; u < kCU; ++u) {
                    const uint32_t k = static_cast<uint32_t>(u * rstep) + csub;
                    if (k < rq_nb) {
                        const uint32_t e = ring[(rq_head + k) & (kRQ - 1)];
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(stage + u * 32 + lane)),
                                     "l"(Xf + ((e & 0xFFFFu) * cxld + cch))
                                     : "memory");
                    }
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
            }
        }
    };
    auto drain_all = [&]() {
        if constexpr (DC) {
            while (rq_nb || rq_tail != rq_head) tick();
        }
    };
    int it = 0;
    if (MA) {
        if (tid == 0) mbar_init(&s_mbar);
        __syncthreads();
        if (cid < a.N) {
            // prologue: the first filter's slice, its maximum through one cluster exchange
            lw_issue(cid);
            lw_wait();
            lw_partials();
            __syncthreads();
            if (warp == 0) lw_cta_reduce(s_xx[1]);
            cluster_sync_publish(warp == 0 && lane == 0);
            if (warp == 0) lw_cluster_reduce(1);
            __syncthreads();
        }
    }

    for (int n = cid; n < a.N; n += num_clusters, ++it) {
        const int xb = MD ? (it & 1) : 0;
        Exchange& s_x = s_xx[xb];
        if (OFFIN) s_fs = s_fs0 + (it & 1) * kPP;
        uint32_t E[kFI];
        const int32_t idbase = static_cast<int32_t>(p0) + tid * 4;
        if constexpr (OFFIN) {
            // the offspring counts of this CTA's particles (padding: 0, and not a free slot)
            const int32_t* orow_in = a.off_in + static_cast<int64_t>(n) * a.ld_off_in + p0;
#pragma unroll
            for (int j = 0; j < kFR; ++j) {
                const int i0 = j * (kFT * 4) + tid * 4;
                if (a.anc_vec && i0 + 3 < np) {
                    const int4 t = __ldcs(reinterpret_cast<const int4*>(orow_in + i0));
                    E[j * 4 + 0] = t.x; E[j * 4 + 1] = t.y; E[j * 4 + 2] = t.z; E[j * 4 + 3] = t.w;
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) E[j * 4 + q] = (i0 + q < np) ? __ldcs(orow_in + i0 + q) : 0u;
                }
            }
        } else {
        const float* row = a.logw + static_cast<int64_t>(n) * a.ld + p0;
        const uint32_t filt = a.filt0 + static_cast<uint32_t>(n);
        if (kEarlyRho && warp == kFW - 1 && lane == 0) {
            // the filter's weight-free position constants rho and rho / D (a Philox call and a
            // double division), by one thread of the last warp while the filter starts: read
            // after the scan exchange's barriers, so off the path that every warp waits on there
            // (computed after the exchange by warp 0 they were 14% of the stall samples)
            const uint64_t rho =
                (SCHEME == 3) ? mulhi64(lo_word(philox10(0u, 0u, 3u, filt, a.key.k0, a.key.k1)), a.D) : 0ull;
            s_rho = rho;
            s_zBc = (SCHEME == 3) ? static_cast<double>(rho) / static_cast<double>(a.D) : 0.0;
        }
        const bool has_next = n + num_clusters < a.N;

        // ---------------- A: load + max
        float v[kFI];
        const double* row64 = F64 ? a.logw64 + static_cast<int64_t>(n) * a.ld + p0 : nullptr;
        if (MA) {
            // the values arrived in shared memory during the previous filter (or the prologue),
            // and its maximum / flag came with the previous exchange
#pragma unroll
            for (int j = 0; j < kFR; ++j) {
                const int i0 = j * (kFT * 4) + tid * 4;
                if (i0 + 3 < np) {
                    const float4 t = *reinterpret_cast<const float4*>(s_lw + i0);
                    v[j * 4 + 0] = t.x; v[j * 4 + 1] = t.y; v[j * 4 + 2] = t.z; v[j * 4 + 3] = t.w;
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) v[j * 4 + q] = (i0 + q < np) ? s_lw[i0 + q] : -INFINITY;
                }
            }
            tick();
        } else if (F64) {
            // NS-3d: the max and the NaN / +inf flag on the doubles; the shifted float32 weights
            // are formed in phase B from a second (L2) read of the same rows
            double m = -INFINITY;
            int bad = 0;
#pragma unroll
            for (int j = 0; j < kFR; ++j) {
                const int i0 = j * (kFT * 4) + tid * 4;
                double x[4];
                if (a.vec && i0 + 3 < np) {
                    const double2 t0 = __ldcg(reinterpret_cast<const double2*>(row64 + i0));
                    const double2 t1 = __ldcg(reinterpret_cast<const double2*>(row64 + i0 + 2));
                    x[0] = t0.x; x[1] = t0.y; x[2] = t1.x; x[3] = t1.y;
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) x[q] = (i0 + q < np) ? __ldcg(row64 + i0 + q) : -INFINITY;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    bad |= (isnan(x[q]) || x[q] == INFINITY) ? 1 : 0;
                    m = fmax(m, x[q]);
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                m = fmax(m, __shfl_xor_sync(kFull, m, o));
                bad |= __shfl_xor_sync(kFull, bad, o);
            }
            if (lane == 0) { s_m64[warp] = m; s_i[warp] = bad; }
            __syncthreads();
            if (warp == 0) {
                double mm = (lane < kFW) ? s_m64[lane] : -INFINITY;
                int bb = (lane < kFW) ? s_i[lane] : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    mm = fmax(mm, __shfl_xor_sync(kFull, mm, o));
                    bb |= __shfl_xor_sync(kFull, bb, o);
                }
                if (lane == 0) { s_x.m64 = mm; s_x.bad = bb; }
            }
        } else {
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
                bad |= (isnan(v[t]) || v[t] == INFINITY) ? 1 : 0;
                m = fmaxf(m, v[t]);  // fmaxf ignores NaN; +inf makes the filter invalid anyway
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
                bad |= __shfl_xor_sync(kFull, bad, o);
            }
            if (lane == 0) { s_f[warp] = m; s_i[warp] = bad; }
            __syncthreads();
            if (warp == 0) {
                float mm = (lane < kFW) ? s_f[lane] : -INFINITY;
                int bb = (lane < kFW) ? s_i[lane] : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    mm = fmaxf(mm, __shfl_xor_sync(kFull, mm, o));
                    bb |= __shfl_xor_sync(kFull, bb, o);
                }
                if (lane == 0) { s_x.m = mm; s_x.bad = bb; }
            }
        }
        if (MA) {
            __syncthreads();  // every read of s_lw, s_lmax and s_bad of this filter is done
            if (has_next) lw_issue(n + num_clusters);
        } else {
            cluster_sync_publish(warp == 0 && lane == 0);  // #1 (s_x.m, s_x.bad)
            if (warp == 0) {
                if (F64) {
                    double gm = -INFINITY;
                    int gb = 0;
                    if (lane < CL) {
                        const Exchange* rx = cluster.map_shared_rank(&s_x, lane);
                        gm = rx->m64;
                        gb = rx->bad;
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        gm = fmax(gm, __shfl_xor_sync(kFull, gm, o));
                        gb |= __shfl_xor_sync(kFull, gb, o);
                    }
                    if (lane == 0) {
                        s_lmax64 = gm;
                        s_lmax = 0.0f;  // the shifted weights' maximum is exactly 0 (NS-3d)
                        s_bad = (gb || gm == -INFINITY) ? 1 : 0;
                    }
                } else {
                    lw_cluster_reduce(xb);
                }
            }
            __syncthreads();
        }
        const float lm = s_lmax;
        if (s_bad) {
            // NS-1: invalid filter -> identity ancestors, NaN side outputs
            int32_t* arow = a.anc + static_cast<int64_t>(n) * a.ld_anc;
            for (int64_t k = p0 + tid; k < p1; k += kFT) arow[k] = static_cast<int32_t>(k);
            if (a.off)
                for (int64_t k = p0 + tid; k < p1; k += kFT) a.off[static_cast<int64_t>(n) * a.ld_anc + k] = 1;
            if (PERM)
                if (a.perm)
                    for (int64_t k = p0 + tid; k < p1; k += kFT) a.perm[static_cast<int64_t>(n) * a.ld_anc + k] = static_cast<int32_t>(k);
            if (a.normw)
                for (int64_t k = p0 + tid; k < p1; k += kFT) a.normw[static_cast<int64_t>(n) * a.P + k] = NAN;
            if (c == 0 && tid == 0) {
                if (a.lse_out) a.lse_out[n] = NAN;
                if (a.ess_out) a.ess_out[n] = NAN;
                if (a.status_out) a.status_out[n] = 1;
            }
            if (MA) {
                // the next filter's maximum still travels through this filter's exchange
                if (has_next) {
                    lw_wait();
                    lw_partials();
                }
                __syncthreads();
                if (warp == 0 && has_next) lw_cta_reduce(s_x);
                cluster_sync_publish(warp == 0 && lane == 0);
                if (warp == 0 && has_next) lw_cluster_reduce(xb);
                __syncthreads();
            } else {
                cluster_sync_publish(false);  // remote readers of s_x are done before the next filter writes it
            }
            continue;
        }
        if (F64) {
            // NS-3d: t_i = fl32(logw_i - lmax) (binary64 subtraction, one rounding); padding -inf
            const double lm64 = s_lmax64;
#pragma unroll
            for (int j = 0; j < kFR; ++j) {
                const int i0 = j * (kFT * 4) + tid * 4;
                double x[4];
                if (a.vec && i0 + 3 < np) {
                    const double2 t0 = __ldcg(reinterpret_cast<const double2*>(row64 + i0));
                    const double2 t1 = __ldcg(reinterpret_cast<const double2*>(row64 + i0 + 2));
                    x[0] = t0.x; x[1] = t0.y; x[2] = t1.x; x[3] = t1.y;
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) x[q] = (i0 + q < np) ? __ldcg(row64 + i0 + q) : -INFINITY;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) v[j * 4 + q] = __double2float_rn(__dsub_rn(x[q], lm64));
            }
        }
#if PF_PREFETCH_NEXT
        // the next filter's log-weights of this CTA into L2 (one bulk prefetch), so its phase A
        // loads come from L2 instead of HBM (the max-ahead mode copies them to shared memory)
        if (!MA && tid == 0 && has_next && a.vec && (np & 3) == 0 && np > 0) {
            const int64_t off = static_cast<int64_t>(n + num_clusters) * a.ld + p0;
            const void* nrow = F64 ? static_cast<const void*>(a.logw64 + off) : static_cast<const void*>(a.logw + off);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nrow),
                         "r"(static_cast<uint32_t>(np) * (F64 ? 8u : 4u))
                         : "memory");
        }
#endif

        // ---------------- B: weights, quantise, block scan, cluster offsets
        double sw = 0.0, sw2 = 0.0;
        uint64_t ex[kFR];
        uint64_t locs[kFR];
#pragma unroll
        for (int j = 0; j < kFR; ++j) {
            uint64_t loc = 0;
            if (PF_FFMA2) {
                // two weights per packed f32x2 evaluation (bit-identical to weight())
                weight2(v[j * 4 + 0], v[j * 4 + 1], lm, v[j * 4 + 0], v[j * 4 + 1]);
                weight2(v[j * 4 + 2], v[j * 4 + 3], lm, v[j * 4 + 2], v[j * 4 + 3]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float w = PF_FFMA2 ? v[j * 4 + q] : weight(v[j * 4 + q], lm);
                v[j * 4 + q] = w;
                if (SUMS) {
                    sw += static_cast<double>(w);
                    sw2 += static_cast<double>(w) * static_cast<double>(w);
                }
                loc += quantise(w, a.kfx);
            }
            if (PF_ROWSCAN) {
                locs[j] = loc;
            } else {
                const uint64_t incl = warp_incl_scan_u64(loc, lane);
                ex[j] = incl - loc;
                const uint64_t wt = __shfl_sync(kFull, incl, 31);
                if (lane == 0) s_wt[j][warp] = wt;
            }
            if (PF_TICK_B) tick();
        }
        if (PF_ROWSCAN) {
            uint64_t rt;
            warp_rows_excl_scan<kFR>(locs, ex, reinterpret_cast<uint64_t*>(&s_buf[warp][0]), lane, &rt);
            if (lane % (32 / kFR) == 32 / kFR - 1) s_wt[lane / (32 / kFR)][warp] = rt;
        }
        if (SUMS) {
            sw = warp_sum_f64(sw);
            sw2 = warp_sum_f64(sw2);
            if (lane == 0) { s_d[0][warp] = sw; s_d[1][warp] = sw2; }
        }
        if (MA && has_next) {
            // the next filter's slice has landed (issued at the top of this filter)
            lw_wait();
            lw_partials();
            tick();
        }
        __syncthreads();
        if (warp == 0) {
            // exclusive scan of the (row, warp) totals in (row, warp) order: kTPL per lane
            uint64_t t4[kTPL];
            uint64_t tsum = 0;
#pragma unroll
            for (int q = 0; q < kTPL; ++q) {
                const int idx = lane * kTPL + q;
                t4[q] = s_wt[idx / kFW][idx % kFW];
                tsum += t4[q];
            }
            const uint64_t incl = warp_incl_scan_u64(tsum, lane);
            uint64_t run = incl - tsum;
#pragma unroll
            for (int q = 0; q < kTPL; ++q) {
                const int idx = lane * kTPL + q;
                s_wt[idx / kFW][idx % kFW] = run;
                run += t4[q];
            }
            double A = 0.0, Bv = 0.0;
            if (SUMS) {
                A = (lane < kFW) ? s_d[0][lane] : 0.0;  // fixed-order tree over the warp partials
                Bv = (lane < kFW) ? s_d[1][lane] : 0.0;
                A = warp_sum_f64(A);
                Bv = warp_sum_f64(Bv);
            }
            if (lane == 31) {
                s_x.tot = incl;
                s_tot = incl;
            }
            if (lane == 0) {
                s_x.sw = A;
                s_x.sw2 = Bv;
            }
            if (MA && has_next) lw_cta_reduce(s_x);
        }
        cluster_sync_publish(warp == 0);  // #2 (s_wt, s_x.tot / sw / sw2, s_tot; MA: next max)
        if (warp == 0) {
            uint64_t tot = 0, off = 0;
            double S = 0.0, S2 = 0.0;
            if (lane < CL) {
                const Exchange* rx = cluster.map_shared_rank(&s_x, lane);
                tot = rx->tot;
                off = (lane < c) ? tot : 0ull;
                S = rx->sw;
                S2 = rx->sw2;
            }
            // fixed rank order for the double sums (deterministic): serial over lanes
            double Sr = 0.0, S2r = 0.0;
            for (int r = 0; r < CL; ++r) {
                Sr += __shfl_sync(kFull, S, r);
                S2r += __shfl_sync(kFull, S2, r);
            }
            tot = warp_sum_u64(tot);
            off = warp_sum_u64(off);
            if (lane == 0) {
                s_off = off;
                s_Qtot = tot;
                s_S = Sr;
                s_S2 = S2r;
                if (!kEarlyRho) {
                    const uint64_t rho = (SCHEME == 3)
                                             ? mulhi64(lo_word(philox10(0u, 0u, 3u, filt, a.key.k0, a.key.k1)), a.D)
                                             : 0ull;
                    s_rho = rho;
                    s_zBc = (SCHEME == 3) ? static_cast<double>(rho) / static_cast<double>(a.D) : 0.0;
                }
                // A = 2^64 / (D Q) (the double estimate k* = v A - rho / D): a float reciprocal
                // refined by two Newton steps (relative error ~2^-52) instead of a double
                // division on the path every warp waits on; A only steers the estimate, whose
                // near-integer cases the exact recount decides
                const double den = static_cast<double>(a.D) * static_cast<double>(tot);
                double r = static_cast<double>(__frcp_rn(static_cast<float>(den)));
                r = fma(r, fma(-den, r, 1.0), r);
                r = fma(r, fma(-den, r, 1.0), r);
                s_zA = 0x1p64 * r;
            }
            if (MA && has_next) lw_cluster_reduce(xb);  // the next filter's lmax / flag
        }
        __syncthreads();
        const uint64_t O = s_off;
        Pos z;
        z.D = a.D;
        z.Qtot = s_Qtot;
        z.key = a.key;
        z.filt = filt;
        z.P = (SCHEME == kBuckets) ? a.S : a.P;  // slots: the P resampled particles, or the NB buckets
        z.rho = s_rho;
        z.A = s_zA;
        z.C = ldexp(s_zA, a.kfx);
        z.Bc = s_zBc;
        if (c == 0 && tid == 0) {
            if (a.lse_out) a.lse_out[n] = (F64 ? s_lmax64 : static_cast<double>(lm)) + log(s_S);
            if (a.ess_out) a.ess_out[n] = s_S * s_S / s_S2;
            if (a.status_out) a.status_out[n] = 0;
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
        if (a.P == 1) {
            if (tid == 0) a.anc[static_cast<int64_t>(n) * a.ld_anc] = 0;
            if (tid == 0 && a.off) a.off[static_cast<int64_t>(n) * a.ld_anc] = 1;
            if (PERM && a.perm && tid == 0) a.perm[static_cast<int64_t>(n) * a.ld_anc] = 0;
            __syncthreads();
            continue;
        }
        // ---------------- C: E_i = c(Q_i), heads, max-scan
#pragma unroll
        for (int j = 0; j < kFR; ++j) {
            // the w C estimate: measured faster without the permutation in CTAs of <= 512
            // threads (C3 resample 0.3845 -> 0.381 ms, bucket mode 1.116 -> 1.10 ms) and slower
            // with it, in 1024-thread CTAs or in the cooperative kernel (more live registers)
            // (and the stratified check in double away from its boundary, without the state
            // gather: C3 stratified resample 0.775 -> 0.738 ms, with the gather 1.905 -> 2.12 ms)
            count_row<(SCHEME == kBuckets ? 3 : SCHEME), PF_KF_RUN && PERM == 0 && FT <= 512,
                      PF_STRAT_DBL && PERM < 2>(z, O + s_wt[j][warp] + ex[j], v + j * 4, a.kfx, E + j * 4);
            if (SCHEME == kBuckets) {
                // the multinomial's search structure: Q_i of every particle (u64, 2 x 16-byte stores)
                uint64_t r = O + s_wt[j][warp] + ex[j];
                uint64_t q4[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    r += quantise(v[j * 4 + q], a.kfx);
                    q4[q] = r;
                }
                const int i0 = j * (kFT * 4) + tid * 4;
                uint64_t* qrow = a.Qout + static_cast<int64_t>(n) * a.ldq + p0 + i0;
                if (i0 + 3 < np) {
                    reinterpret_cast<ulonglong2*>(qrow)[0] = make_ulonglong2(q4[0], q4[1]);
                    reinterpret_cast<ulonglong2*>(qrow)[1] = make_ulonglong2(q4[2], q4[3]);
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (i0 + q < np) qrow[q] = q4[q];
                }
            }
            if (lane == 31) s_lastE[j][warp] = E[j * 4 + 3];
            if (PF_TICK_C) tick();
        }
        if (tid == 0) s_klo = count_below<(SCHEME == kBuckets ? 3 : SCHEME)>(z, O);
        if (SCHEME == kBuckets && c == 0 && tid == 0) a.Qtot_out[n] = z.Qtot;
        __syncthreads();
        const uint32_t k_lo = s_klo;
        // E_{i-1} of the first particle of each 4-chunk (natural order: row j, warp, lane, q);
        // the other three predecessors are the chunk's own E values.
        uint32_t first[kFR];
#pragma unroll
        for (int j = 0; j < kFR; ++j) {
            const uint32_t up = __shfl_up_sync(kFull, E[j * 4 + 3], 1);
            if (lane > 0) first[j] = up;
            else if (warp > 0) first[j] = s_lastE[j][warp - 1];
            else if (j > 0) first[j] = s_lastE[j - 1][kFW - 1];
            else first[j] = k_lo;
        }
        if (a.off) {
            // a8 fused: o_i = E_i - E_{i-1}
            int32_t* orow = a.off + static_cast<int64_t>(n) * a.ld_anc + p0;
#pragma unroll
            for (int j = 0; j < kFR; ++j) {
                const int i0 = j * (kFT * 4) + tid * 4;
                const int32_t o0 = static_cast<int32_t>(E[j * 4 + 0] - first[j]);
                const int32_t o1 = static_cast<int32_t>(E[j * 4 + 1] - E[j * 4 + 0]);
                const int32_t o2 = static_cast<int32_t>(E[j * 4 + 2] - E[j * 4 + 1]);
                const int32_t o3 = static_cast<int32_t>(E[j * 4 + 3] - E[j * 4 + 2]);
                if (a.anc_vec && (p0 & 3) == 0 && i0 + 3 < np) {
                    __stcs(reinterpret_cast<int4*>(orow + i0), make_int4(o0, o1, o2, o3));
                } else {
                    if (i0 + 0 < np) orow[i0 + 0] = o0;
                    if (i0 + 1 < np) orow[i0 + 1] = o1;
                    if (i0 + 2 < np) orow[i0 + 2] = o2;
                    if (i0 + 3 < np) orow[i0 + 3] = o3;
                }
            }
        }
        int32_t* arow = a.anc + static_cast<int64_t>(n) * a.ld_anc;
        int32_t* s_head = &s_buf[0][0];
        // The CTA's slots are [k_lo, K1).  Per 8192-slot chunk (8 per thread): heads[E_{i-1}] = i
        // for every particle with o_i > 0, then a CTA-wide max-scan gives
        // a_k = max{i : E_{i-1} <= k}; aligned vector stores except at the CTA's two ends.
        {
            const uint32_t K1 = s_lastE[kFR - 1][kFW - 1];
            int32_t carry = -1;
            for (uint32_t c0 = k_lo & ~7u; c0 < K1; c0 += kXS) {
                cta_clear8(s_head, tid);
                __syncthreads();
#pragma unroll
                for (int j = 0; j < kFR; ++j) {
                    // the row's heads lie in [first[j], E[j*4+3]): skip rows outside this chunk
                    if (PF_ROW_SKIP && (E[j * 4 + 3] <= c0 || first[j] >= c0 + static_cast<uint32_t>(kXS))) continue;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t pe = (q == 0) ? first[j] : E[j * 4 + q - 1];
                        const uint32_t rel = pe - c0;  // wraps when pe < c0
                        if (E[j * 4 + q] > pe && rel < static_cast<uint32_t>(kXS))
                            s_head[rel] = idbase + j * (kFT * 4) + q;
                    }
                }
                __syncthreads();
                int32_t h[8];
                cta_max_scan8<kFW>(s_head, s_wmax, h, carry, tid, warp, lane);
                const uint32_t k0 = c0 + 8 * tid;
                if (a.anc_vec && k0 >= k_lo && k0 + 8 <= K1) {
                    int4* dst = reinterpret_cast<int4*>(arow + k0);
                    __stcs(dst, make_int4(h[0], h[1], h[2], h[3]));
                    __stcs(dst + 1, make_int4(h[4], h[5], h[6], h[7]));
                } else if (k0 + 8 > k_lo && k0 < K1) {
#pragma unroll
                    for (int t = 0; t < 8; ++t)
                        if (k0 + t >= k_lo && k0 + t < K1) arow[k0 + t] = h[t];
                }
                tick();
            }
        }
        if (PERM) {
            // E becomes the offspring in place (first[] dies here: fewer live registers in D)
#pragma unroll
            for (int j = 0; j < kFR; ++j) {
#pragma unroll
                for (int q = 3; q > 0; --q) E[j * 4 + q] -= E[j * 4 + q - 1];
                E[j * 4] -= first[j];
            }
        }
        }  // phases A-C (not in the permutation-from-offspring mode)
        if (PERM) {
            int32_t* s_head = &s_buf[0][0];
            // ---------------- D: canonical permutation (NS-15) from the offspring o_i
            // packed value per particle: (extras << 31) | free; padding particles are neither.
            uint32_t* const O4 = E;  // O4[j * 4 + q] = o of particle (j, q)
            uint64_t pex[kFR];
            if (DC) {
                drain_all();  // the ring now takes this filter's pairs
                rq_n = n;
            }
            __syncthreads();  // s_wt is reused
            uint64_t plocs[kFR];
#pragma unroll
            for (int j = 0; j < kFR; ++j) {
                uint64_t loc = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t o = O4[j * 4 + q];
                    const bool real = (j * (kFT * 4) + tid * 4 + q) < np;
                    loc += (static_cast<uint64_t>(o > 1 ? o - 1 : 0) << 31) | ((o == 0 && real) ? 1ull : 0ull);
                }
                if (RS_D) {
                    plocs[j] = loc;
                } else {
                    const uint64_t incl = warp_incl_scan_u64(loc, lane);
                    pex[j] = incl - loc;
                    const uint64_t wt = __shfl_sync(kFull, incl, 31);
                    if (lane == 0) s_wt[j][warp] = wt;
                }
            }
            if (RS_D) {
                uint64_t rt;
                warp_rows_excl_scan<kFR>(plocs, pex, reinterpret_cast<uint64_t*>(&s_buf[warp][0]), lane, &rt);
                if (lane % (32 / kFR) == 32 / kFR - 1) s_wt[lane / (32 / kFR)][warp] = rt;
            }
            __syncthreads();
            if (warp == 0) {
                uint64_t t4[kTPL];
                uint64_t tsum = 0;
#pragma unroll
                for (int q = 0; q < kTPL; ++q) {
                    const int idx = lane * kTPL + q;
                    t4[q] = s_wt[idx / kFW][idx % kFW];
                    tsum += t4[q];
                }
                const uint64_t incl = warp_incl_scan_u64(tsum, lane);
                uint64_t run = incl - tsum;
#pragma unroll
                for (int q = 0; q < kTPL; ++q) {
                    const int idx = lane * kTPL + q;
                    s_wt[idx / kFW][idx % kFW] = run;
                    run += t4[q];
                }
                if (lane == 31) s_x.ptot = incl;
            }
            int32_t* prow = a.perm + static_cast<int64_t>(n) * a.ld_anc;
            // survivors keep their slot: the identity over the CTA's range (aligned vector stores;
            // the free slots are overwritten by their owners after the next cluster barrier)
            if (a.perm) {
#pragma unroll
                for (int j = 0; j < kFR; ++j) {
                    const int i0 = j * (kFT * 4) + tid * 4;
                    const int32_t id0 = static_cast<int32_t>(p0) + i0;
                    if (a.anc_vec && i0 + 3 < np) {
                        __stcg(reinterpret_cast<int4*>(prow + p0 + i0), make_int4(id0, id0 + 1, id0 + 2, id0 + 3));
                    } else {
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            if (i0 + q < np) prow[p0 + i0 + q] = id0 + q;
                    }
                }
            }
            uint64_t poff;
            if (MD) {
                // the CTA's free-slot list (local free ranks) before the exchange, so one cluster
                // barrier publishes both the packed totals and the lists
                __syncthreads();
#pragma unroll
                for (int j = 0; j < kFR; ++j) {
                    uint64_t run = s_wt[j][warp] + pex[j];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int i = j * (kFT * 4) + tid * 4 + q;
                        const uint32_t o = O4[j * 4 + q];
                        if (o == 0 && i < np) s_fs[static_cast<uint32_t>(run & 0x7FFFFFFFull)] = static_cast<FsT>(p0 + i);
                        run += (static_cast<uint64_t>(o > 1 ? o - 1 : 0) << 31) | ((o == 0 && i < np) ? 1ull : 0ull);
                    }
                }
                __syncthreads();
                cluster_sync_publish(tid == 0);  // #3 packed totals and free-slot lists published
            } else {
                cluster_sync_publish(warp == 0);  // #3 packed CTA totals (s_wt, s_x.ptot) published
            }
            if (warp == 0) {
                uint64_t pt = 0;
                if (lane < CL) pt = cluster.map_shared_rank(&s_x, lane)->ptot;
                // free-rank prefix of every CTA (for the owner lookup) and this CTA's packed offset
                uint64_t incl = pt;
#pragma unroll
                for (int o2 = 1; o2 < 32; o2 <<= 1) {
                    const uint64_t u = __shfl_up_sync(kFull, incl, o2);
                    if (lane >= o2) incl += u;
                }
                const uint64_t excl = incl - pt;
                if (lane <= CL) s_rf[lane] = static_cast<uint32_t>(excl & 0x7FFFFFFFull);
                if (lane == c) s_poff = excl;
            }
            __syncthreads();
            poff = s_poff;
            if (!MD) {
                const uint32_t rf_c = s_rf[c];
#pragma unroll
                for (int j = 0; j < kFR; ++j) {
                    uint64_t run = poff + s_wt[j][warp] + pex[j];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int i = j * (kFT * 4) + tid * 4 + q;
                        const uint32_t o = O4[j * 4 + q];
                        if (o == 0 && i < np) s_fs[static_cast<uint32_t>(run & 0x7FFFFFFFull) - rf_c] = static_cast<FsT>(p0 + i);
                        run += (static_cast<uint64_t>(o > 1 ? o - 1 : 0) << 31) | ((o == 0 && i < np) ? 1ull : 0ull);
                    }
                }
                __syncthreads();
                cluster_sync_publish(tid == 0);  // #4 every CTA's free-slot list complete
            }
            // Survivors' extra copies, CTA-wide: the CTA's extras ranks are [XC0, XC0 + XC).  Per
            // 8192-rank chunk: heads[first extras rank of i] = i, CTA max-scan gives the owner of
            // every rank r; the r-th global free slot (this CTA's list or a peer's, DSMEM) gets it.
            {
                const uint32_t XC0 = static_cast<uint32_t>(poff >> 31);
                const uint32_t XC = static_cast<uint32_t>(s_x.ptot >> 31);
                int32_t carry = -1;
                for (uint32_t c0 = 0; c0 < XC; c0 += kXS) {
                    cta_clear8(s_head, tid);
                    __syncthreads();
#pragma unroll
                    for (int j = 0; j < kFR; ++j) {
                        uint64_t run = poff + s_wt[j][warp] + pex[j];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const uint32_t o = O4[j * 4 + q];
                            const uint32_t rel = static_cast<uint32_t>(run >> 31) - XC0 - c0;
                            if (o > 1 && rel < static_cast<uint32_t>(kXS)) s_head[rel] = idbase + j * (kFT * 4) + q;
                            run += static_cast<uint64_t>(o > 1 ? o - 1 : 0) << 31;  // the free bit never carries
                        }
                    }
                    __syncthreads();
                    int32_t h[8];
                    cta_max_scan8<kFW>(s_head, s_wmax, h, carry, tid, warp, lane);
                    const uint32_t r0 = c0 + 8 * tid;
                    // this warp's pairs of the chunk: extras ranks [c0 + 256 warp, ...) of XC
                    const int64_t wfirst = static_cast<int64_t>(c0) + 256 * warp;
                    const int npairs = static_cast<int>(
                        min(int64_t{256}, max(int64_t{0}, static_cast<int64_t>(XC) - wfirst)));
                    if (DC) {
                        while (rq_tail + static_cast<uint32_t>(npairs) - rq_head > static_cast<uint32_t>(kRQ)) tick();
                    }
                    if (r0 < XC) {
                        uint32_t R = XC0 + r0;  // global free rank of this thread's first extra
                        int cc = 0;
#pragma unroll
                        for (int q2 = 1; q2 < kMaxCL; ++q2) cc += (q2 < CL && s_rf[q2] <= R) ? 1 : 0;
                        uint32_t rb = s_rf[cc], nxt = s_rf[cc + 1];
                        const FsT* rfs = (cc == c) ? s_fs : cluster.map_shared_rank(s_fs, cc);
#pragma unroll
                        for (int t = 0; t < 8; ++t) {
                            if (r0 + t < XC) {
                                while (R >= nxt) {  // next CTA's free list (rare)
                                    ++cc;
                                    rb = nxt;
                                    nxt = s_rf[cc + 1];
                                    rfs = (cc == c) ? s_fs : cluster.map_shared_rank(s_fs, cc);
                                }
                                const int32_t slot = static_cast<int32_t>(rfs[R - rb]);
                                prow[slot] = h[t];
                                if (DC) {
                                    ring[(rq_tail + 8 * lane + t) & (kRQ - 1)] =
                                        (static_cast<uint32_t>(slot) << 16) | static_cast<uint32_t>(h[t]);
                                    if (PF_PF_L2 && (t == 0 || h[t] != h[t - 1])) {
                                        const char* src = a.X + static_cast<int64_t>(n) * a.xfld +
                                                          static_cast<int64_t>(h[t]) * a.xld;
                                        for (int b = 0; b < (16 << cxl); b += 128)
                                            asm volatile("prefetch.global.L2 [%0];" ::"l"(src + b));
                                    }
                                } else if (PERM == 2) {
                                    s_pslot[8 * tid + t] = slot;
                                }
                                ++R;
                            }
                        }
                    }
                    if (DC) {
                        __syncwarp();  // the ring entries are read by other lanes of the warp
                        rq_tail += static_cast<uint32_t>(npairs);
                        tick();
                    } else if (PERM == 2) {
                        // a10 fused (NS-16): X[free slot] <- X[owner] for this warp's (slot, owner)
                        // pairs; reads touch survivor rows only, writes free rows only
                        int4* hh = reinterpret_cast<int4*>(s_head);
                        hh[2 * tid] = make_int4(h[0], h[1], h[2], h[3]);
                        hh[2 * tid + 1] = make_int4(h[4], h[5], h[6], h[7]);
                        __syncwarp();
                        copy_rows_warp(a, n, s_head + 256 * warp, s_pslot + 256 * warp, npairs, lane);
                        __syncwarp();
                    }
                }
            }
        }
        // no barrier here: the next filter first writes shared memory (s_f, s_i, s_x.m) that no
        // thread reads any more in this filter, and its first barrier follows its loads, so warps
        // that finish their copies early start the next filter's loads under the stragglers' copies
    }
    drain_all();
    cluster.sync();  // keep this CTA's shared memory alive for remote readers
}

// ============================================================================ cooperative
// One-launch resampler for LARGE filters (P > 8 x 8192): a cooperative grid of
// G co-resident CTAs, CTA c owning the contiguous chunk [c*CH, (c+1)*CH) of
// every filter, processed in 8192-particle sub-tiles.
//   A  chunk max -> global array -> grid sync -> every CTA reduces the G maxima
//   B  chunk sum of q (log-weights re-read, L2-resident up to ~2^24 particles)
//      -> grid sync -> chunk offset O_c = sum of earlier chunk totals
//   C  sub-tiles in order with a running carry: dexp, quantise, block scan,
//      E_i = c(Q_i), per-warp head-mark + max-scan expansion of the runs
//      [E_{i-1}, E_i) straight into the ancestors (no Q array in HBM).
// HBM: 4 B/particle in (+2 L2 re-reads) + 4 B out.  Two grid syncs per filter.
struct CoopArgs {
    const float* logw;
    int64_t ld;
    int32_t N, P;
    int64_t CH;  // particles per CTA chunk (multiple of kPP)
    uint64_t D;
    Key key;
    uint32_t filt0;
    int kfx;
    int vec;
    int32_t* anc;
    int64_t ld_anc;
    int anc_vec;
    double* lse_out;
    double* ess_out;
    int32_t* status_out;
    int32_t* off;  // offspring out (row stride ld_anc), nullable (required with PERM)
    int32_t* perm;  // canonical permutation out (row stride ld_anc), PERM
    int32_t* freelist;  // scratch [P]: the filter's free slots in rank order (PERM)
    uint64_t* Qout;     // kBuckets: Q [N][ldq], the totals, and the bucket count S
    int64_t ldq;
    uint64_t* Qtot_out;
    int32_t S;
    uint64_t* g_ptot;   // scratch [G]: packed (extras, free) totals of the chunks (PERM)
    uint4* heavy;       // scratch [2][heavy_cap]: deferred runs {kind, start, end, particle} per filter parity
    uint32_t* heavy_n;  // scratch [2]: their counts
    int32_t heavy_cap;
    // scratch (device): [G] per-CTA values
    float* g_max;
    int32_t* g_bad;
    uint64_t* g_tot;
    double* g_sw;
    double* g_sw2;
};

// packed (extras << 31 | free) value of a particle with offspring o (NS-15)
__device__ __forceinline__ uint64_t packed_of(int32_t o, bool real) {
    return (static_cast<uint64_t>(o > 1 ? o - 1 : 0) << 31) | ((o == 0 && real) ? 1ull : 0ull);
}

// this thread's FI offspring of the sub-tile at t0 (rows of 4, natural order), 0 past c1
template <int FI>
__device__ __forceinline__ void coop_load_o(const int32_t* orow, int64_t t0, int64_t c1, int tid, int vec,
                                            int32_t* ov) {
    constexpr int kFR = FI / 4;
#pragma unroll
    for (int j = 0; j < kFR; ++j) {
        const int64_t i0 = t0 + j * (kFT * 4) + tid * 4;
        if (vec && i0 + 3 < c1) {
            const int4 t = __ldcg(reinterpret_cast<const int4*>(orow + i0));
            ov[j * 4 + 0] = t.x; ov[j * 4 + 1] = t.y; ov[j * 4 + 2] = t.z; ov[j * 4 + 3] = t.w;
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) ov[j * 4 + q] = (i0 + q < c1) ? __ldcg(orow + i0 + q) : 0;
        }
    }
}

// block exclusive scan of the packed values of a sub-tile: pex[j] = this lane's offset in row j's
// warp segment, s_wt[j][warp] = the (row, warp) segment offset, *total = the sub-tile's total
template <int FI>
__device__ __forceinline__ void coop_packed_scan(const int32_t* ov, int64_t t0, int64_t c1, int tid, int warp,
                                                 int lane, uint64_t (*s_wt)[kFW], uint64_t* s_u64, uint64_t* pex,
                                                 uint64_t* total, uint64_t* wbuf) {
    // wbuf: this warp's 1 KB of free shared memory (the row scans as one transposed scan)
    constexpr int kFR = FI / 4;
    constexpr int kTPL = kFR * kFW / 32;
    uint64_t locs[kFR];
#pragma unroll
    for (int j = 0; j < kFR; ++j) {
        uint64_t loc = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) loc += packed_of(ov[j * 4 + q], t0 + j * (kFT * 4) + tid * 4 + q < c1);
        if (PF_ROWSCAN) {
            locs[j] = loc;
        } else {
            const uint64_t incl = warp_incl_scan_u64(loc, lane);
            pex[j] = incl - loc;
            const uint64_t wt = __shfl_sync(kFull, incl, 31);
            if (lane == 0) s_wt[j][warp] = wt;
        }
    }
    if (PF_ROWSCAN) {
        uint64_t rt;
        warp_rows_excl_scan<kFR>(locs, pex, wbuf, lane, &rt);
        if (lane % (32 / kFR) == 32 / kFR - 1) s_wt[lane / (32 / kFR)][warp] = rt;
    }
    __syncthreads();
    if (warp == 0) {
        uint64_t t4[kTPL];
        uint64_t tsum = 0;
#pragma unroll
        for (int q = 0; q < kTPL; ++q) {
            const int idx = lane * kTPL + q;
            t4[q] = s_wt[idx / kFW][idx % kFW];
            tsum += t4[q];
        }
        const uint64_t incl = warp_incl_scan_u64(tsum, lane);
        uint64_t run = incl - tsum;
#pragma unroll
        for (int q = 0; q < kTPL; ++q) {
            const int idx = lane * kTPL + q;
            s_wt[idx / kFW][idx % kFW] = run;
            run += t4[q];
        }
        if (lane == 31) s_u64[2] = incl;
    }
    __syncthreads();
    *total = s_u64[2];
}

// Slot-balanced expansion under skew (the cooperative kernel): a run of one particle that
// covers whole kXS-slot expansion chunks of its CTA (o_i >= kXS slots, or o_i - 1 >= kXS extras
// ranks) is not expanded by that CTA chunk by chunk; its covered chunks [cs, ce) go to a
// deferred list and, after the filter's closing grid barrier, every CTA of the grid fills a
// 1/G share of every listed run.  A heavy particle of a skewed filter (sigma^2 = 10 at P = 2^20:
// one particle ~3.5e4 slots) therefore costs the grid ce - cs stores instead of one CTA
// (ce - cs) / kXS serial expansion chunks.
constexpr int kMaxHeavy = 16;  // per sub-tile (more are expanded the ordinary way)
struct HeavyRun {
    uint32_t s, e;
    int32_t id;
};
enum { kRunSlots = 0, kRunExtras = 1 };

// the sub-tile's particles with runs of >= kXS (slots or extras ranks) into s_h (tid 0 reads
// the count after the caller's barrier); run ends are relative to the caller's rank space
__device__ __forceinline__ void heavy_note(uint32_t s, uint32_t e, int32_t id, HeavyRun* s_h, uint32_t* s_nh) {
    if (e - s >= static_cast<uint32_t>(kXS)) {
        const uint32_t k = atomicAdd(s_nh, 1u);
        if (k < static_cast<uint32_t>(kMaxHeavy)) s_h[k] = {s, e, id};
    }
}

// if chunk [q0, q0 + kXS) lies inside a listed run: the end of the run's covered chunks (so the
// caller jumps there) and the run's particle in *id (the max-scan carry after the jump: its head
// may sit in a skipped chunk), after listing those chunks for the deferred fill (thread 0);
// else q0
__device__ __forceinline__ uint32_t heavy_skip(uint32_t q0, const HeavyRun* s_h, uint32_t nh, const CoopArgs& a,
                                               int parity, uint32_t kind, uint32_t base, int32_t* id) {
    for (uint32_t h = 0; h < nh; ++h) {
        if (s_h[h].s <= q0 && q0 + kXS <= s_h[h].e) {
            *id = s_h[h].id;
            const uint32_t nc = (s_h[h].e - q0) / kXS;  // whole chunks covered from q0 on
            if (threadIdx.x == 0) {
                // one entry per chunk: the grid then shares the fill evenly however long the run
                const uint32_t k = atomicAdd(a.heavy_n + parity, nc);
                for (uint32_t m = 0; m < nc && static_cast<int64_t>(k) + m < a.heavy_cap; ++m)
                    a.heavy[static_cast<int64_t>(parity) * a.heavy_cap + k + m] =
                        make_uint4(kind, base + q0 + m * kXS, 0u, static_cast<uint32_t>(s_h[h].id));
            }
            return q0 + nc * kXS;
        }
    }
    return q0;
}

// PERM: 0 ancestors (+ offspring), 1 + the canonical permutation (offspring required)
template <int SCHEME, bool SUMS, int PERM, int FI>
__global__ void __launch_bounds__(kFT, 1024 / kFT) k_coop_sorted(CoopArgs a) {
    // FI particles per thread: sub-tiles of kPP = 512 x FI particles (16: 8192, 8: 4096, so that
    // filters of 2^18..2^20 spread over 64..256 CTAs instead of 32..128)
    constexpr int kFI = FI;
    constexpr int kFR = FI / 4;
    constexpr int kPP = kFT * FI;
    constexpr int kTPL = kFR * kFW / 32;
    static_assert(kFR * kFW % 32 == 0, "phase-B totals scan assumes a multiple of 32 (row, warp) totals");
    static_assert((kFR == 2 || kFR == 4) && kChunk * 4 >= kFR * 32 * 8, "warp_rows_excl_scan: rows of s_buf per warp");
    __shared__ float s_f[kFW];
    __shared__ int s_i[kFW];
    __shared__ double s_d[2][kFW];
    __shared__ uint64_t s_wt[kFR][kFW];
    __shared__ uint32_t s_lastE[kFR][kFW];
    __shared__ __align__(16) int32_t s_buf[kFW][kChunk];
    __shared__ float s_lmax;
    __shared__ int s_bad;
    __shared__ uint64_t s_u64[4];
    __shared__ uint32_t s_prevE;
    __shared__ int32_t s_wmax[kFW];
    __shared__ uint64_t s_crho;
    __shared__ double s_cA, s_cBc;
    __shared__ HeavyRun s_h[kMaxHeavy];
    __shared__ uint32_t s_nh;
    cg::grid_group grid = cg::this_grid();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int G = gridDim.x, c = blockIdx.x;
    if (c == 0 && tid < 2) a.heavy_n[tid] = 0;  // appended only after the first filter's second grid barrier
    for (int n = 0; n < a.N; ++n) {
        const int hp = n & 1;  // this filter's deferred-run list
        const float* frow = a.logw + static_cast<int64_t>(n) * a.ld;
        const int64_t c0 = static_cast<int64_t>(c) * a.CH;
        const int64_t c1 = min(static_cast<int64_t>(a.P), c0 + a.CH);
        const uint32_t filt = a.filt0 + static_cast<uint32_t>(n);
        if (PF_EARLY_RHO && warp == kFW - 1 && lane == 0) {
            // rho and rho / D (weight-free) while phase A loads, not after the scan's grid barrier
            // where every warp waits for them (as in k_fused_sorted); read after that barrier
            const uint64_t rho =
                (SCHEME == 3) ? mulhi64(lo_word(philox10(0u, 0u, 3u, filt, a.key.k0, a.key.k1)), a.D) : 0ull;
            s_crho = rho;
            s_cBc = (SCHEME == 3) ? static_cast<double>(rho) / static_cast<double>(a.D) : 0.0;
        }
        // ---------------- A: chunk max
        float m = -INFINITY;
        int bad = 0;
        // resident (a CTA's chunk is one sub-tile): the values stay in registers from A to C,
        // and phase C reuses phase B's weights (one load and one dexp per particle, not three / two)
        // (8 particles per thread only: with 16 the live values cost registers on every path)
        const bool resident = PF_COOP_RESIDENT && kFI == 8 && a.CH <= kPP;
        float rv[kFI];
        for (int64_t t0 = c0; t0 < c1; t0 += kPP) {
#pragma unroll
            for (int j = 0; j < kFR; ++j) {
                const int64_t i0 = t0 + j * (kFT * 4) + tid * 4;
                float v4[4];
                if (a.vec && i0 + 3 < c1) {
                    const float4 t = __ldg(reinterpret_cast<const float4*>(frow + i0));
                    v4[0] = t.x; v4[1] = t.y; v4[2] = t.z; v4[3] = t.w;
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) v4[q] = (i0 + q < c1) ? __ldg(frow + i0 + q) : -INFINITY;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    m = fmax_nan(m, v4[q]);  // a NaN anywhere stays NaN
                    if (kFI == 8) rv[j * 4 + q] = v4[q];
                }
            }
        }
        bad = !(m <= FLT_MAX) ? 1 : 0;  // NaN or +inf among this thread's values
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
            bad |= __shfl_xor_sync(kFull, bad, o);
        }
        if (lane == 0) { s_f[warp] = m; s_i[warp] = bad; }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < kFW; ++w) { m = fmaxf(m, s_f[w]); bad |= s_i[w]; }
            a.g_max[c] = m;
            a.g_bad[c] = bad;
        }
        grid.sync();
        // every CTA has filled the previous filter's runs (list 1 - hp) before reaching the barrier
        if (c == 0 && tid == 0) a.heavy_n[1 - hp] = 0;
        if (warp == 0) {
            float gm = -INFINITY;
            int gb = 0;
            for (int r = lane; r < G; r += 32) { gm = fmaxf(gm, __ldcg(a.g_max + r)); gb |= __ldcg(a.g_bad + r); }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                gm = fmaxf(gm, __shfl_xor_sync(kFull, gm, o));
                gb |= __shfl_xor_sync(kFull, gb, o);
            }
            if (lane == 0) { s_lmax = gm; s_bad = (gb || gm == -INFINITY) ? 1 : 0; }
        }
        __syncthreads();
        const float lm = s_lmax;
        int32_t* arow = a.anc + static_cast<int64_t>(n) * a.ld_anc;
        if (s_bad) {
            for (int64_t k = c0 + tid; k < c1; k += kFT) arow[k] = static_cast<int32_t>(k);
            if (a.off)
                for (int64_t k = c0 + tid; k < c1; k += kFT) a.off[static_cast<int64_t>(n) * a.ld_anc + k] = 1;
            if (c == 0 && tid == 0) {
                if (a.lse_out) a.lse_out[n] = NAN;
                if (a.ess_out) a.ess_out[n] = NAN;
                if (a.status_out) a.status_out[n] = 1;
            }
            grid.sync();  // g_max/g_bad are rewritten by the next filter
            continue;
        }
        // ---------------- B: chunk totals
        uint64_t tot = 0;
        double sw = 0.0, sw2 = 0.0;
        for (int64_t t0 = c0; t0 < c1; t0 += kPP) {
#pragma unroll
            for (int j = 0; j < kFR; ++j) {
                const int64_t i0 = t0 + j * (kFT * 4) + tid * 4;
                float v4[4];
                if (resident) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) v4[q] = rv[j * 4 + q];
                } else if (a.vec && i0 + 3 < c1) {
                    const float4 t = __ldg(reinterpret_cast<const float4*>(frow + i0));
                    v4[0] = t.x; v4[1] = t.y; v4[2] = t.z; v4[3] = t.w;
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) v4[q] = (i0 + q < c1) ? __ldg(frow + i0 + q) : -INFINITY;
                }
                if (PF_FFMA2) {
                    weight2(v4[0], v4[1], lm, v4[0], v4[1]);
                    weight2(v4[2], v4[3], lm, v4[2], v4[3]);
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float w = PF_FFMA2 ? v4[q] : weight(v4[q], lm);
                    if (kFI == 8) rv[j * 4 + q] = w;
                    tot += quantise(w, a.kfx);
                    if (SUMS) {
                        sw += static_cast<double>(w);
                        sw2 += static_cast<double>(w) * static_cast<double>(w);
                    }
                }
            }
        }
        tot = warp_sum_u64(tot);
        if (SUMS) { sw = warp_sum_f64(sw); sw2 = warp_sum_f64(sw2); }
        if (lane == 0) { s_wt[0][warp] = tot; s_d[0][warp] = sw; s_d[1][warp] = sw2; }
        __syncthreads();
        if (tid == 0) {
            uint64_t t = 0;
            double A = 0.0, Bv = 0.0;
            for (int w = 0; w < kFW; ++w) { t += s_wt[0][w]; A += s_d[0][w]; Bv += s_d[1][w]; }
            a.g_tot[c] = t;
            a.g_sw[c] = A;
            a.g_sw2[c] = Bv;
        }
        grid.sync();
        if (warp == 0) {
            uint64_t off = 0, all = 0;
            for (int r = lane; r < G; r += 32) {
                const uint64_t t = __ldcg(a.g_tot + r);
                all += t;
                if (r < c) off += t;
            }
            off = warp_sum_u64(off);
            all = warp_sum_u64(all);
            if (lane == 0) {
                s_u64[0] = off;
                s_u64[1] = all;
                // the filter's position constants, once per CTA (as in k_fused_sorted)
                if (!PF_EARLY_RHO) {
                    const uint64_t rho = (SCHEME == 3)
                                             ? mulhi64(lo_word(philox10(0u, 0u, 3u, filt, a.key.k0, a.key.k1)), a.D)
                                             : 0ull;
                    s_crho = rho;
                    s_cBc = (SCHEME == 3) ? static_cast<double>(rho) / static_cast<double>(a.D) : 0.0;
                }
                const double den = static_cast<double>(a.D) * static_cast<double>(all);
                double r = static_cast<double>(__frcp_rn(static_cast<float>(den)));
                r = fma(r, fma(-den, r, 1.0), r);
                r = fma(r, fma(-den, r, 1.0), r);
                s_cA = 0x1p64 * r;
                if (SUMS && c == 0) {
                    double S = 0.0, S2 = 0.0;
                    for (int r = 0; r < G; ++r) { S += __ldcg(a.g_sw + r); S2 += __ldcg(a.g_sw2 + r); }
                    if (a.lse_out) a.lse_out[n] = static_cast<double>(lm) + log(S);
                    if (a.ess_out) a.ess_out[n] = S * S / S2;
                }
                if (c == 0 && a.status_out) a.status_out[n] = 0;
                if (SCHEME == kBuckets && c == 0) a.Qtot_out[n] = all;
            }
        }
        __syncthreads();
        Pos z;
        z.D = a.D;
        z.Qtot = s_u64[1];
        z.key = a.key;
        z.filt = filt;
        z.P = (SCHEME == kBuckets) ? a.S : a.P;  // slots: the particles, or the NB buckets
        z.rho = s_crho;
        z.A = s_cA;
        z.C = ldexp(s_cA, a.kfx);
        z.Bc = s_cBc;
        uint64_t carry = s_u64[0];
        if (tid == 0) s_prevE = count_below<(SCHEME == kBuckets ? 3 : SCHEME)>(z, carry);
        // ---------------- C: sub-tiles in order
        uint64_t ploc_c = 0;  // PERM: packed (extras << 31 | free) total of this thread's particles
        for (int64_t t0 = c0; t0 < c1; t0 += kPP) {
            float v[kFI];
#pragma unroll
            for (int j = 0; j < kFR; ++j) {
                const int64_t i0 = t0 + j * (kFT * 4) + tid * 4;
                if (resident) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) v[j * 4 + q] = rv[j * 4 + q];  // phase B's weights
                } else if (a.vec && i0 + 3 < c1) {
                    const float4 t = __ldg(reinterpret_cast<const float4*>(frow + i0));
                    v[j * 4 + 0] = t.x; v[j * 4 + 1] = t.y; v[j * 4 + 2] = t.z; v[j * 4 + 3] = t.w;
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) v[j * 4 + q] = (i0 + q < c1) ? __ldg(frow + i0 + q) : -INFINITY;
                }
            }
            uint64_t ex[kFR];
            uint64_t locs[kFR];
#pragma unroll
            for (int j = 0; j < kFR; ++j) {
                uint64_t loc = 0;
                if (PF_FFMA2 && !resident) {
                    weight2(v[j * 4 + 0], v[j * 4 + 1], lm, v[j * 4 + 0], v[j * 4 + 1]);
                    weight2(v[j * 4 + 2], v[j * 4 + 3], lm, v[j * 4 + 2], v[j * 4 + 3]);
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float w = (PF_FFMA2 || resident) ? v[j * 4 + q] : weight(v[j * 4 + q], lm);
                    v[j * 4 + q] = w;
                    loc += quantise(w, a.kfx);
                }
                if (PF_ROWSCAN) {
                    locs[j] = loc;
                } else {
                    const uint64_t incl = warp_incl_scan_u64(loc, lane);
                    ex[j] = incl - loc;
                    const uint64_t wt = __shfl_sync(kFull, incl, 31);
                    if (lane == 0) s_wt[j][warp] = wt;
                }
            }
            if (PF_ROWSCAN) {
                // s_buf's last readers (the previous sub-tile's expansion) passed the barrier
                // inside its final max-scan
                uint64_t rt;
                warp_rows_excl_scan<kFR>(locs, ex, reinterpret_cast<uint64_t*>(&s_buf[warp][0]), lane, &rt);
                if (lane % (32 / kFR) == 32 / kFR - 1) s_wt[lane / (32 / kFR)][warp] = rt;
            }
            __syncthreads();
            if (warp == 0) {
                uint64_t t4[kTPL];
                uint64_t tsum = 0;
#pragma unroll
                for (int q = 0; q < kTPL; ++q) {
                    const int idx = lane * kTPL + q;
                    t4[q] = s_wt[idx / kFW][idx % kFW];
                    tsum += t4[q];
                }
                const uint64_t incl = warp_incl_scan_u64(tsum, lane);
                uint64_t run = incl - tsum;
#pragma unroll
                for (int q = 0; q < kTPL; ++q) {
                    const int idx = lane * kTPL + q;
                    s_wt[idx / kFW][idx % kFW] = run;
                    run += t4[q];
                }
                if (lane == 31) s_u64[2] = incl;  // sub-tile total
            }
            __syncthreads();
            uint32_t E[kFI];
#pragma unroll
            for (int j = 0; j < kFR; ++j) {
                count_row<(SCHEME == kBuckets ? 3 : SCHEME)>(z, carry + s_wt[j][warp] + ex[j], v + j * 4, a.kfx,
                                                             E + j * 4);
                if (SCHEME == kBuckets) {
                    // the multinomial's search structure: Q_i of every particle of the sub-tile
                    uint64_t r = carry + s_wt[j][warp] + ex[j];
                    const int64_t i0 = t0 + j * (kFT * 4) + tid * 4;
                    uint64_t* qrow = a.Qout + static_cast<int64_t>(n) * a.ldq + i0;
                    uint64_t q4[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        r += quantise(v[j * 4 + q], a.kfx);
                        q4[q] = r;
                    }
                    if (i0 + 3 < c1) {
                        reinterpret_cast<ulonglong2*>(qrow)[0] = make_ulonglong2(q4[0], q4[1]);
                        reinterpret_cast<ulonglong2*>(qrow)[1] = make_ulonglong2(q4[2], q4[3]);
                    } else {
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            if (i0 + q < c1) qrow[q] = q4[q];
                    }
                }
                if (lane == 31) s_lastE[j][warp] = E[j * 4 + 3];
            }
            __syncthreads();
            uint32_t first[kFR];
#pragma unroll
            for (int j = 0; j < kFR; ++j) {
                const uint32_t up = __shfl_up_sync(kFull, E[j * 4 + 3], 1);
                if (lane > 0) first[j] = up;
                else if (warp > 0) first[j] = s_lastE[j][warp - 1];
                else if (j > 0) first[j] = s_lastE[j - 1][kFW - 1];
                else first[j] = s_prevE;
            }
            const int32_t idbase = static_cast<int32_t>(t0) + tid * 4;
            if (a.off) {
                int32_t* orow = a.off + static_cast<int64_t>(n) * a.ld_anc;
#pragma unroll
                for (int j = 0; j < kFR; ++j) {
                    const int64_t i0 = t0 + j * (kFT * 4) + tid * 4;
                    const int32_t o0 = static_cast<int32_t>(E[j * 4 + 0] - first[j]);
                    const int32_t o1 = static_cast<int32_t>(E[j * 4 + 1] - E[j * 4 + 0]);
                    const int32_t o2 = static_cast<int32_t>(E[j * 4 + 2] - E[j * 4 + 1]);
                    const int32_t o3 = static_cast<int32_t>(E[j * 4 + 3] - E[j * 4 + 2]);
                    if (PERM)
                        ploc_c += packed_of(o0, i0 + 0 < c1) + packed_of(o1, i0 + 1 < c1) + packed_of(o2, i0 + 2 < c1) +
                                  packed_of(o3, i0 + 3 < c1);
                    if (a.anc_vec && i0 + 3 < c1) {
                        // phase D reads them back: keep them in L2 (streaming stores otherwise)
                        if (PERM) __stcg(reinterpret_cast<int4*>(orow + i0), make_int4(o0, o1, o2, o3));
                        else __stcs(reinterpret_cast<int4*>(orow + i0), make_int4(o0, o1, o2, o3));
                    } else {
                        if (i0 + 0 < c1) orow[i0 + 0] = o0;
                        if (i0 + 1 < c1) orow[i0 + 1] = o1;
                        if (i0 + 2 < c1) orow[i0 + 2] = o2;
                        if (i0 + 3 < c1) orow[i0 + 3] = o3;
                    }
                }
            }
            // the sub-tile's slots [K0, K1): CTA-wide chunks of kXS slots, head marks + max-scan,
            // aligned vector stores except at the two ends (as in k_fused_sorted phase C)
            {
                int32_t* s_head = &s_buf[0][0];
                const uint32_t K0 = s_prevE, K1 = s_lastE[kFR - 1][kFW - 1];
                if (tid == 0) s_nh = 0;
                __syncthreads();
#pragma unroll
                for (int j = 0; j < kFR; ++j) {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        heavy_note((q == 0) ? first[j] : E[j * 4 + q - 1], E[j * 4 + q], idbase + j * (kFT * 4) + q,
                                   s_h, &s_nh);
                }
                __syncthreads();
                const uint32_t nh = min(s_nh, static_cast<uint32_t>(kMaxHeavy));
                int32_t cy = -1;
                for (uint32_t q0 = K0 & ~7u; q0 < K1; q0 += kXS) {
                    if (nh) {
                        int32_t hid;
                        const uint32_t qs = heavy_skip(q0, s_h, nh, a, hp, kRunSlots, 0u, &hid);
                        if (qs != q0) {
                            // the skipped chunks all hold the run's particle: it is the max-scan
                            // carry of the slots that follow (ancestors grow with the slot)
                            cy = hid;
                            q0 = qs - kXS;
                            continue;
                        }
                    }
                    cta_clear8(s_head, tid);
                    __syncthreads();
#pragma unroll
                    for (int j = 0; j < kFR; ++j) {
                        if (PF_ROW_SKIP && (E[j * 4 + 3] <= q0 || first[j] >= q0 + static_cast<uint32_t>(kXS))) continue;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const uint32_t pe = (q == 0) ? first[j] : E[j * 4 + q - 1];
                            const uint32_t rel = pe - q0;
                            if (E[j * 4 + q] > pe && rel < static_cast<uint32_t>(kXS))
                                s_head[rel] = idbase + j * (kFT * 4) + q;
                        }
                    }
                    __syncthreads();
                    int32_t h[8];
                    cta_max_scan8<kFW>(s_head, s_wmax, h, cy, tid, warp, lane);
                    const uint32_t k0 = q0 + 8 * tid;
                    if (a.anc_vec && k0 >= K0 && k0 + 8 <= K1) {
                        int4* dst = reinterpret_cast<int4*>(arow + k0);
                        __stcs(dst, make_int4(h[0], h[1], h[2], h[3]));
                        __stcs(dst + 1, make_int4(h[4], h[5], h[6], h[7]));
                    } else if (k0 + 8 > K0 && k0 < K1) {
#pragma unroll
                        for (int t = 0; t < 8; ++t)
                            if (k0 + t >= K0 && k0 + t < K1) arow[k0 + t] = h[t];
                    }
                }
            }
            carry += s_u64[2];
            __syncthreads();
            if (tid == 0) s_prevE = s_lastE[kFR - 1][kFW - 1];
            __syncthreads();
        }
        if (PERM) {
            // ---------------- D: canonical permutation (NS-15) of this filter from the offspring
            // written in phase C
            // (this CTA's own chunk: visible to it after the barrier)
            __syncthreads();
            const int32_t* orow = a.off + static_cast<int64_t>(n) * a.ld_anc;
            int32_t* prow = a.perm + static_cast<int64_t>(n) * a.ld_anc;
            // D1: packed (extras << 31 | free) total of the chunk (each thread's part summed in
            // phase C from the offspring in registers)
            uint64_t ploc = warp_sum_u64(ploc_c);
            if (lane == 0) s_wt[0][warp] = ploc;
            __syncthreads();
            if (tid == 0) {
                uint64_t t = 0;
                for (int w = 0; w < kFW; ++w) t += s_wt[0][w];
                a.g_ptot[c] = t;
            }
            grid.sync();
            if (warp == 0) {
                uint64_t off = 0;
                for (int r = lane; r < c; r += 32) off += __ldcg(a.g_ptot + r);
                off = warp_sum_u64(off);
                if (lane == 0) s_u64[3] = off;
            }
            __syncthreads();
            // D2: survivors keep their slot; free slots into the global free list (rank order)
            {
                uint64_t run0 = s_u64[3];
                for (int64_t t0 = c0; t0 < c1; t0 += kPP) {
                    int32_t ov[kFI];
                    coop_load_o<FI>(orow, t0, c1, tid, a.anc_vec, ov);
                    uint64_t pex[kFR], stot;
                    coop_packed_scan<FI>(ov, t0, c1, tid, warp, lane, s_wt, s_u64, pex, &stot,
                                         reinterpret_cast<uint64_t*>(&s_buf[warp][0]));
#pragma unroll
                    for (int j = 0; j < kFR; ++j) {
                        uint64_t run = run0 + s_wt[j][warp] + pex[j];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int64_t i = t0 + j * (kFT * 4) + tid * 4 + q;
                            const int32_t o = ov[j * 4 + q];
                            if (i < c1) {
                                if (o > 0) prow[i] = static_cast<int32_t>(i);
                                else a.freelist[run & 0x7FFFFFFFull] = static_cast<int32_t>(i);
                            }
                            run += packed_of(o, i < c1);
                        }
                    }
                    run0 += stot;
                    __syncthreads();  // s_wt is reused by the next sub-tile
                }
            }
            grid.sync();  // the filter's free list is complete
            // D3: the r-th extra copy goes to the r-th free slot
            {
                uint64_t run0 = s_u64[3];
                int32_t* s_head = &s_buf[0][0];
                for (int64_t t0 = c0; t0 < c1; t0 += kPP) {
                    int32_t ov[kFI];
                    coop_load_o<FI>(orow, t0, c1, tid, a.anc_vec, ov);
                    uint64_t pex[kFR], stot;
                    coop_packed_scan<FI>(ov, t0, c1, tid, warp, lane, s_wt, s_u64, pex, &stot,
                                         reinterpret_cast<uint64_t*>(&s_buf[warp][0]));
                    const uint32_t XS = static_cast<uint32_t>(run0 >> 31);          // first extras rank
                    const uint32_t XT = static_cast<uint32_t>((run0 + stot) >> 31) - XS;
                    const int32_t idbase = static_cast<int32_t>(t0) + tid * 4;
                    if (tid == 0) s_nh = 0;
                    __syncthreads();
#pragma unroll
                    for (int j = 0; j < kFR; ++j) {
                        uint64_t run = run0 + s_wt[j][warp] + pex[j];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int32_t o = ov[j * 4 + q];
                            const uint32_t r = static_cast<uint32_t>(run >> 31) - XS;
                            if (o > 1) heavy_note(r, r + static_cast<uint32_t>(o - 1), idbase + j * (kFT * 4) + q, s_h, &s_nh);
                            run += static_cast<uint64_t>(o > 1 ? o - 1 : 0) << 31;
                        }
                    }
                    __syncthreads();
                    const uint32_t nh = min(s_nh, static_cast<uint32_t>(kMaxHeavy));
                    int32_t cy = -1;
                    for (uint32_t q0 = 0; q0 < XT; q0 += kXS) {
                        if (nh) {
                            int32_t hid;
                            const uint32_t qs = heavy_skip(q0, s_h, nh, a, hp, kRunExtras, XS, &hid);
                            if (qs != q0) {
                                cy = hid;
                                q0 = qs - kXS;
                                continue;
                            }
                        }
                        cta_clear8(s_head, tid);
                        __syncthreads();
#pragma unroll
                        for (int j = 0; j < kFR; ++j) {
                            uint64_t run = run0 + s_wt[j][warp] + pex[j];
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const int32_t o = ov[j * 4 + q];
                                const uint32_t rel = static_cast<uint32_t>(run >> 31) - XS - q0;
                                if (o > 1 && rel < static_cast<uint32_t>(kXS)) s_head[rel] = idbase + j * (kFT * 4) + q;
                                run += static_cast<uint64_t>(o > 1 ? o - 1 : 0) << 31;
                            }
                        }
                        __syncthreads();
                        int32_t h[8];
                        cta_max_scan8<kFW>(s_head, s_wmax, h, cy, tid, warp, lane);
                        const uint32_t r0 = q0 + 8 * tid;
#pragma unroll
                        for (int t = 0; t < 8; ++t)
                            if (r0 + t < XT) prow[__ldcg(a.freelist + XS + r0 + t)] = h[t];
                        __syncthreads();  // s_head is cleared by the next chunk
                    }
                    run0 += stot;
                }
            }
        }
        grid.sync();  // scratch arrays are rewritten by the next filter
        // the filter's deferred chunks (list hp is complete), round-robin over the grid: chunk
        // entries {kind, first slot / extras rank, -, particle}, kXS ranks each
        {
            const uint32_t nr = min(__ldcg(a.heavy_n + hp), static_cast<uint32_t>(a.heavy_cap));
            int32_t* arow = a.anc + static_cast<int64_t>(n) * a.ld_anc;
            int32_t* prow = PERM ? a.perm + static_cast<int64_t>(n) * a.ld_anc : nullptr;
            for (uint32_t r = c; r < nr; r += G) {
                const uint4 h = __ldcg(a.heavy + static_cast<int64_t>(hp) * a.heavy_cap + r);
                const int32_t id = static_cast<int32_t>(h.w);
                if (h.x == kRunSlots) {
                    if (a.anc_vec) {  // the chunk grid is 8-slot aligned
                        int4* dst = reinterpret_cast<int4*>(arow + h.y);
                        for (int k = tid; k < kXS / 4; k += kFT) __stcs(dst + k, make_int4(id, id, id, id));
                    } else {
                        for (int k = tid; k < kXS; k += kFT) arow[h.y + k] = id;
                    }
                } else if (PERM) {
                    for (int k = tid; k < kXS; k += kFT) prow[__ldcg(a.freelist + h.y + k)] = id;
                }
            }
        }
    }
}

// ============================================================================ small filters
// One WARP per filter for P <= 256 (8 particles per lane): every scheme in one
// launch with warp-level synchronisation only (BASELINE C1: P = 16; batches of
// small filters).  Q (u64) and w (f32) of the filter live in shared memory.
constexpr int kSmallP = 256;
constexpr int kSmallWarps = 8;

struct SmallArgs {
    const float* logw;
    int64_t ld;
    int32_t N, P, scheme, B, sorted;
    int kfx;
    uint64_t D;
    Key key;
    uint32_t filt0;
    int32_t* anc;
    int64_t ld_anc;
    double* lse_out;
    double* ess_out;
    float* normw;
    int32_t* status_out;
    int32_t* off;
};

__device__ __forceinline__ int small_upper_bound(const uint64_t* Q, int P, uint64_t x) {
    int lo = 0, n = P;  // first i with Q[i] > x (Q[P-1] > x)
    while (n > 1) {
        const int half = n >> 1;
        lo += (Q[lo + half - 1] <= x) ? half : 0;
        n -= half;
    }
    return lo;
}

__global__ void __launch_bounds__(kSmallWarps * 32) k_small(SmallArgs a) {
    __shared__ uint64_t s_q[kSmallWarps][kSmallP + 4];
    __shared__ float s_w[kSmallWarps][kSmallP];
    __shared__ int32_t s_o[kSmallWarps][kSmallP];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = blockIdx.x * kSmallWarps + warp;
    if (n >= a.N) return;
    const int P = a.P;
    const float* row = a.logw + static_cast<int64_t>(n) * a.ld;
    int32_t* arow = a.anc + static_cast<int64_t>(n) * a.ld_anc;
    const uint32_t filt = a.filt0 + static_cast<uint32_t>(n);
    uint64_t* Q = s_q[warp];
    float* W = s_w[warp];
    // a1: max + validation
    float v[8];
    float m = -INFINITY;
    int bad = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const int i = lane * 8 + t;
        v[t] = (i < P) ? row[i] : -INFINITY;
        bad |= (isnan(v[t]) || v[t] == INFINITY) ? 1 : 0;
        m = fmaxf(m, v[t]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
        bad |= __shfl_xor_sync(kFull, bad, o);
    }
    const bool invalid = bad || m == -INFINITY;
    if (invalid) {
        for (int i = lane; i < P; i += 32) {
            arow[i] = i;
            if (a.off) a.off[static_cast<int64_t>(n) * a.ld_anc + i] = 1;
            if (a.normw) a.normw[static_cast<int64_t>(n) * P + i] = NAN;
        }
        if (lane == 0) {
            if (a.lse_out) a.lse_out[n] = NAN;
            if (a.ess_out) a.ess_out[n] = NAN;
            if (a.status_out) a.status_out[n] = 1;
        }
        return;
    }
    // a2+a3: weights, fixed point, warp scan (8 consecutive per lane)
    double sw = 0.0, sw2 = 0.0;
    uint64_t loc = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const float w = weight(v[t], m);
        v[t] = w;
        sw += static_cast<double>(w);
        sw2 += static_cast<double>(w) * static_cast<double>(w);
        loc += quantise(w, a.kfx);
    }
    const uint64_t incl = warp_incl_scan_u64(loc, lane);
    uint64_t run = incl - loc;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const int i = lane * 8 + t;
        run += quantise(v[t], a.kfx);
        if (i < P) { Q[i] = run; W[i] = v[t]; }
        if (i < kSmallP) s_o[warp][i] = 0;
    }
    sw = warp_sum_f64(sw);
    sw2 = warp_sum_f64(sw2);
    const uint64_t Qtot = __shfl_sync(kFull, incl, 31);
    __syncwarp();
    if (lane == 0) {
        if (a.lse_out) a.lse_out[n] = static_cast<double>(m) + log(sw);
        if (a.ess_out) a.ess_out[n] = sw * sw / sw2;
        if (a.status_out) a.status_out[n] = 0;
    }
    if (a.normw)
        for (int i = lane; i < P; i += 32)
            a.normw[static_cast<int64_t>(n) * P + i] = static_cast<float>(static_cast<double>(W[i]) / sw);
    // a4+a5 / a6 / a7: slot k = lane * 8 + t
    int32_t out[8];
    if (a.scheme == 4) {
        // chains i = lane + 32 t: small filters keep every lane busy
        const float kU = __uint_as_float(0x33800000u);
        for (int t = 0; t < 8; ++t) {
            const int i = lane + 32 * t;
            if (i >= P) break;
            int32_t k = i;
            float wk = W[i];
            for (int32_t b = 0; b < a.B; b += 2) {
                const u32x4 r = philox10(static_cast<uint32_t>(i), static_cast<uint32_t>(b >> 1), 4u, filt, a.key.k0,
                                         a.key.k1);
                const uint32_t j0 = __umulhi(r.x, static_cast<uint32_t>(P));
                const float u0 = __fmul_rn(static_cast<float>(r.y >> 8), kU);
                const float w0 = W[j0];
                if (__fmul_rn(u0, wk) < w0) { k = j0; wk = w0; }
                if (b + 1 < a.B) {
                    const uint32_t j1 = __umulhi(r.z, static_cast<uint32_t>(P));
                    const float u1 = __fmul_rn(static_cast<float>(r.w >> 8), kU);
                    const float w1 = W[j1];
                    if (__fmul_rn(u1, wk) < w1) { k = j1; wk = w1; }
                }
            }
            arow[i] = k;
            if (a.off) atomicAdd(&s_o[warp][k], 1);
        }
        if (a.off) {
            __syncwarp();
            for (int i = lane; i < P; i += 32) a.off[static_cast<int64_t>(n) * a.ld_anc + i] = s_o[warp][i];
        }
        return;
    } else if (P == 1) {
#pragma unroll
        for (int t = 0; t < 8; ++t) out[t] = 0;
    } else if (a.sorted) {
        // a6: spacings e_0..e_P (P + 1 <= 257 values) scanned by the warp, 9 per lane
        uint64_t e[9], gl = 0;
#pragma unroll
        for (int t = 0; t < 9; ++t) {
            const int k = lane * 9 + t;
            e[t] = 0;
            if (k <= P) {
                const u32x4 r = philox10(static_cast<uint32_t>(k >> 2), 0u, 5u, filt, a.key.k0, a.key.k1);
                const uint32_t wd = ((k & 3) == 0) ? r.x : ((k & 3) == 1) ? r.y : ((k & 3) == 2) ? r.z : r.w;
                e[t] = spacing_from_word(wd);
            }
            gl += e[t];
        }
        const uint64_t gincl = warp_incl_scan_u64(gl, lane);
        const uint64_t GP = __shfl_sync(kFull, gincl, 31);
        uint64_t gr = gincl - gl;
        // positions of this lane's spacing indices, then a shuffle to the slot owners
        uint64_t xk[9];
#pragma unroll
        for (int t = 0; t < 9; ++t) {
            gr += e[t];
            xk[t] = muldiv_floor(gr, Qtot, GP);  // only used for k < P (G_k < G_P)
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const int k = lane * 8 + t;         // slot owned by this lane
            const int src = k / 9, idx = k - src * 9;
            uint64_t x = 0;
#pragma unroll
            for (int tt = 0; tt < 9; ++tt) {
                const uint64_t cand = __shfl_sync(kFull, xk[tt], src & 31);
                if (tt == idx) x = cand;
            }
            out[t] = (k < P) ? small_upper_bound(Q, P, x) : 0;
        }
    } else {
        uint64_t rho = 0;
        if (a.scheme == 3) rho = mulhi64(lo_word(philox10(0u, 0u, 3u, filt, a.key.k0, a.key.k1)), a.D);
#pragma unroll
        for (int t = 0; t < 8; t += 2) {
            const int k = lane * 8 + t;
            const u32x4 r = philox10(static_cast<uint32_t>(k >> 1), 0u, static_cast<uint32_t>(a.scheme), filt,
                                     a.key.k0, a.key.k1);
            uint64_t x0, x1;
            if (a.scheme == 1) {
                x0 = mulhi64(lo_word(r), Qtot);
                x1 = mulhi64(hi_word(r), Qtot);
            } else {
                const uint64_t r0 = (a.scheme == 2) ? mulhi64(lo_word(r), a.D) : rho;
                const uint64_t r1 = (a.scheme == 2) ? mulhi64(hi_word(r), a.D) : rho;
                x0 = mulhi64(static_cast<uint64_t>(k) * a.D + r0, Qtot);
                x1 = mulhi64(static_cast<uint64_t>(k + 1) * a.D + r1, Qtot);
            }
            out[t] = (k < P) ? small_upper_bound(Q, P, x0) : 0;
            out[t + 1] = (k + 1 < P) ? small_upper_bound(Q, P, x1) : 0;
        }
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const int k = lane * 8 + t;
        if (k < P) {
            arow[k] = out[t];
            if (a.off) atomicAdd(&s_o[warp][out[t]], 1);
        }
    }
    if (a.off) {
        __syncwarp();
        for (int i = lane; i < P; i += 32) a.off[static_cast<int64_t>(n) * a.ld_anc + i] = s_o[warp][i];
    }
}

// ============================================================================ medium filters
// k_medium: ONE CTA per filter for 256 < P <= 8192, every scheme, everything in shared
// memory (one launch; the latency path for single and few filters, Fig. 2's P range):
//   a1   max + validation over float4 loads (log-weights kept in smem)
//   a2+3 4-item-per-thread tiles: dexp, quantise, block scan with a running carry -> Q (smem)
//   a6   the same tile scan of the spacings e_0..e_P -> G (smem)
//   a4+5 slot k: its position (NS-8..NS-10, NS-12), a_k = upper_bound(Q, x_k) by binary
//        search in smem (13 probes at 8192); Metropolis (a7): chains over the smem weights
//   a8   offspring by shared-memory atomics
// (256 threads up to P = 2048, 1024 threads above: the per-filter latency is serial work per
// thread, profiles/r01_dispatch.md)
constexpr int kMedP = 8192;

template <int kMedT>
__device__ __forceinline__ uint64_t med_block_excl_scan(uint64_t v, uint64_t* s_wt, int tid, uint64_t* total) {
    constexpr int kMedW = kMedT / 32;
    const int lane = tid & 31, warp = tid >> 5;
    const uint64_t incl = warp_incl_scan_u64(v, lane);
    if (lane == 31) s_wt[warp] = incl;
    __syncthreads();
    uint64_t wpre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kMedW; ++w) {
        const uint64_t t = s_wt[w];
        wpre += (w < warp) ? t : 0ull;
        tot += t;
    }
    __syncthreads();  // s_wt is reused by the next tile
    *total = tot;
    return wpre + incl - v;
}

template <int kMedT>
__global__ void __launch_bounds__(kMedT) k_medium(SmallArgs a) {
    constexpr int kMedW = kMedT / 32;
    extern __shared__ __align__(16) unsigned char s_med[];
    __shared__ uint64_t s_wt[kMedW];
    __shared__ float s_fm[kMedW];
    __shared__ int s_ib[kMedW];
    __shared__ double s_dd[2][kMedW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int P = a.P;
    const int P4 = (P + 3) & ~3;
    uint64_t* Q = reinterpret_cast<uint64_t*>(s_med);               // [P4]
    float* W = reinterpret_cast<float*>(Q + P4);                    // [P4]  logw, then w
    int32_t* O = reinterpret_cast<int32_t*>(W + P4);                // [P4]  offspring counts
    uint64_t* G = reinterpret_cast<uint64_t*>(O + P4);              // [P4 + 4] spacings scan (a6)
    for (int n = blockIdx.x; n < a.N; n += gridDim.x) {
        const float* row = a.logw + static_cast<int64_t>(n) * a.ld;
        int32_t* arow = a.anc + static_cast<int64_t>(n) * a.ld_anc;
        int32_t* orow = a.off ? a.off + static_cast<int64_t>(n) * a.ld_anc : nullptr;
        const uint32_t filt = a.filt0 + static_cast<uint32_t>(n);
        // ---- a1
        float m = -INFINITY;
        int bad = 0;
        const bool vec = ((reinterpret_cast<uintptr_t>(row) & 15) == 0);
        for (int i0 = 4 * tid; i0 < P4; i0 += 4 * kMedT) {
            float4 t;
            if (vec && i0 + 3 < P) {
                t = __ldcs(reinterpret_cast<const float4*>(row + i0));
            } else {
                t.x = (i0 + 0 < P) ? row[i0 + 0] : -INFINITY;
                t.y = (i0 + 1 < P) ? row[i0 + 1] : -INFINITY;
                t.z = (i0 + 2 < P) ? row[i0 + 2] : -INFINITY;
                t.w = (i0 + 3 < P) ? row[i0 + 3] : -INFINITY;
            }
            reinterpret_cast<float4*>(W)[i0 >> 2] = t;
            const float q4[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                bad |= (isnan(q4[c]) || q4[c] == INFINITY) ? 1 : 0;
                m = fmaxf(m, q4[c]);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
            bad |= __shfl_xor_sync(kFull, bad, o);
        }
        if (lane == 0) { s_fm[warp] = m; s_ib[warp] = bad; }
        __syncthreads();
        m = -INFINITY;
        bad = 0;
#pragma unroll
        for (int w = 0; w < kMedW; ++w) { m = fmaxf(m, s_fm[w]); bad |= s_ib[w]; }
        if (bad || m == -INFINITY) {
            for (int i = tid; i < P; i += kMedT) {
                arow[i] = i;
                if (orow) orow[i] = 1;
                if (a.normw) a.normw[static_cast<int64_t>(n) * P + i] = NAN;
            }
            if (tid == 0) {
                if (a.lse_out) a.lse_out[n] = NAN;
                if (a.ess_out) a.ess_out[n] = NAN;
                if (a.status_out) a.status_out[n] = 1;
            }
            __syncthreads();
            continue;
        }
        // ---- a2+a3: tiles of 4 x kMedT, running carry
        double sw = 0.0, sw2 = 0.0;
        uint64_t carry = 0;
        for (int base = 0; base < P4; base += 4 * kMedT) {
            const int i0 = base + 4 * tid;
            uint64_t q[4] = {0, 0, 0, 0};
            if (i0 < P4) {
                float4 t = reinterpret_cast<float4*>(W)[i0 >> 2];
                float* tv = reinterpret_cast<float*>(&t);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float w = weight(tv[c], m);
                    tv[c] = w;
                    sw += static_cast<double>(w);
                    sw2 += static_cast<double>(w) * static_cast<double>(w);
                    q[c] = quantise(w, a.kfx);
                }
                reinterpret_cast<float4*>(W)[i0 >> 2] = t;
            }
            uint64_t tot;
            uint64_t run = carry + med_block_excl_scan<kMedT>(q[0] + q[1] + q[2] + q[3], s_wt, tid, &tot);
            if (i0 < P4) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    run += q[c];
                    Q[i0 + c] = run;
                }
            }
            carry += tot;
        }
        const uint64_t Qtot = carry;
        // sums in a fixed order: warp trees, then warps in order (deterministic)
        sw = warp_sum_f64(sw);
        sw2 = warp_sum_f64(sw2);
        if (lane == 0) { s_dd[0][warp] = sw; s_dd[1][warp] = sw2; }
        if (a.off)
            for (int i = tid; i < P; i += kMedT) O[i] = 0;
        __syncthreads();
        double S = 0.0, S2 = 0.0;
#pragma unroll
        for (int w = 0; w < kMedW; ++w) { S += s_dd[0][w]; S2 += s_dd[1][w]; }
        if (tid == 0) {
            if (a.lse_out) a.lse_out[n] = static_cast<double>(m) + log(S);
            if (a.ess_out) a.ess_out[n] = S * S / S2;
            if (a.status_out) a.status_out[n] = 0;
        }
        if (a.normw)
            for (int i = tid; i < P; i += kMedT)
                a.normw[static_cast<int64_t>(n) * P + i] = static_cast<float>(static_cast<double>(W[i]) / S);
        // ---- a4+a5 / a6 / a7
        if (a.scheme == 4) {
            const float kU = __uint_as_float(0x33800000u);
            for (int i = tid; i < P; i += kMedT) {
                int32_t k = i;
                float wk = W[i];
                for (int32_t b = 0; b < a.B; b += 2) {
                    const u32x4 r = philox10(static_cast<uint32_t>(i), static_cast<uint32_t>(b >> 1), 4u, filt,
                                             a.key.k0, a.key.k1);
                    const uint32_t j0 = __umulhi(r.x, static_cast<uint32_t>(P));
                    const float u0 = __fmul_rn(static_cast<float>(r.y >> 8), kU);
                    const float w0 = W[j0];
                    if (__fmul_rn(u0, wk) < w0) { k = j0; wk = w0; }
                    if (b + 1 < a.B) {
                        const uint32_t j1 = __umulhi(r.z, static_cast<uint32_t>(P));
                        const float u1 = __fmul_rn(static_cast<float>(r.w >> 8), kU);
                        const float w1 = W[j1];
                        if (__fmul_rn(u1, wk) < w1) { k = j1; wk = w1; }
                    }
                }
                arow[i] = k;
                if (a.off) atomicAdd(&O[k], 1);
            }
        } else if (a.sorted) {
            // spacings e_0..e_P (NS-12), tile scan into G
            uint64_t gc = 0;
            const int PG = P + 1;
            for (int base = 0; base < PG; base += 4 * kMedT) {
                const int k0 = base + 4 * tid;
                uint64_t e[4] = {0, 0, 0, 0};
                if (k0 < PG) {
                    const u32x4 r = philox10(static_cast<uint32_t>(k0 >> 2), 0u, 5u, filt, a.key.k0, a.key.k1);
                    const uint32_t wd[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
                    for (int c = 0; c < 4; ++c) e[c] = (k0 + c < PG) ? spacing_from_word(wd[c]) : 0ull;
                }
                uint64_t tot;
                uint64_t run = gc + med_block_excl_scan<kMedT>(e[0] + e[1] + e[2] + e[3], s_wt, tid, &tot);
                if (k0 < PG) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        run += e[c];
                        if (k0 + c < PG) G[k0 + c] = run;
                    }
                }
                gc += tot;
            }
            __syncthreads();
            const uint64_t GP = gc;
            for (int k = tid; k < P; k += kMedT) {
                const int32_t anc = small_upper_bound(Q, P, muldiv_floor(G[k], Qtot, GP));
                arow[k] = anc;
                if (a.off) atomicAdd(&O[anc], 1);
            }
        } else {
            __syncthreads();  // Q complete
            uint64_t rho = 0;
            if (a.scheme == 3) rho = mulhi64(lo_word(philox10(0u, 0u, 3u, filt, a.key.k0, a.key.k1)), a.D);
            for (int k = 2 * tid; k < P; k += 2 * kMedT) {
                const u32x4 r = (a.scheme == 3) ? u32x4{0u, 0u, 0u, 0u}
                                                : philox10(static_cast<uint32_t>(k >> 1), 0u,
                                                           static_cast<uint32_t>(a.scheme), filt, a.key.k0, a.key.k1);
                uint64_t x0, x1;
                if (a.scheme == 1) {
                    x0 = mulhi64(lo_word(r), Qtot);
                    x1 = mulhi64(hi_word(r), Qtot);
                } else {
                    const uint64_t r0 = (a.scheme == 2) ? mulhi64(lo_word(r), a.D) : rho;
                    const uint64_t r1 = (a.scheme == 2) ? mulhi64(hi_word(r), a.D) : rho;
                    x0 = mulhi64(static_cast<uint64_t>(k) * a.D + r0, Qtot);
                    x1 = mulhi64(static_cast<uint64_t>(k + 1) * a.D + r1, Qtot);
                }
                const int32_t a0 = small_upper_bound(Q, P, x0);
                arow[k] = a0;
                if (a.off) atomicAdd(&O[a0], 1);
                if (k + 1 < P) {
                    const int32_t a1 = small_upper_bound(Q, P, x1);
                    arow[k + 1] = a1;
                    if (a.off) atomicAdd(&O[a1], 1);
                }
            }
        }
        if (a.off) {
            __syncthreads();
            for (int i = tid; i < P; i += kMedT) orow[i] = O[i];
        }
        __syncthreads();  // smem reused by the next filter
    }
}

int device_sms() { return sm_count(); }

template <int SCHEME, int PERM, int FT, int FI, bool F64 = false>
constexpr size_t fused_smem() {
    // max-ahead: [the next filter's log-weight slice, float] [PERM: free-slot list, u16]
    //            [deferred copy: kFW pair rings of kRQ u32, kFW x kCU x 32 staged 16-byte chunks |
    //             PERM 2 otherwise: free slot per extras rank of a chunk, int32]
    // otherwise: [PERM: free-slot list, int32] [PERM 2: free slot per extras rank of a chunk]
    constexpr size_t pslot = (PERM == 2) ? static_cast<size_t>(FT / 32) * kChunk * 4 : 0;
    constexpr bool offin = SCHEME == kFromOffspring;  // no log-weight slice; two free-slot lists
    return fused_max_ahead<FT, F64>()
               ? (offin ? 0 : static_cast<size_t>(FT * FI) * 4) +
                     (PERM ? static_cast<size_t>(FT * FI) * 2 * (offin ? 2 : 1) : 0) +
                     (fused_deferred_copy<SCHEME, PERM, FT, F64>()
                          ? static_cast<size_t>(FT / 32) * (kRQ * 4 + copy_cu<FT>() * 32 * 16)
                          : pslot)
               : (PERM ? static_cast<size_t>(FT * FI) * 4 + pslot : 0);
}

template <int SCHEME, bool SUMS, int PERM, int FT, int FI, bool F64 = false>
void fused_set_attributes() {
    // per-device function attributes: set once per device
    static std::atomic<int> attr_set[kMaxDevices];
    cached_per_device(attr_set, [] {
        auto kern = k_fused_sorted<SCHEME, SUMS, PERM, FT, FI, F64>;
        if (fused_smem<SCHEME, PERM, FT, FI, F64>() > 0)
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(fused_smem<SCHEME, PERM, FT, FI, F64>()));
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaGetLastError();
        return 1;
    });
}

template <int SCHEME, bool SUMS, int PERM, int FT, int FI, bool F64 = false>
int fused_max_clusters(int CL) {
    // occupancy of (kernel, cluster size) is a device constant: query once (host cost ~us);
    // -1 = a cluster of this size cannot be scheduled on this device (0 = not queried yet)
    static std::atomic<int> cached[kMaxCL + 1][kMaxDevices];
    return cached_per_device(cached[CL], [&] {
        fused_set_attributes<SCHEME, SUMS, PERM, FT, FI, F64>();
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CL;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.blockDim = dim3(FT, 1, 1);
        cfg.dynamicSmemBytes = fused_smem<SCHEME, PERM, FT, FI, F64>();
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(CL, 1, 1);
        int mc = 0;
        if (cudaOccupancyMaxActiveClusters(&mc, k_fused_sorted<SCHEME, SUMS, PERM, FT, FI, F64>, &cfg) != cudaSuccess ||
            mc < 1) {
            cudaGetLastError();
            mc = -1;
        }
        return mc;
    });
}

template <int SCHEME, bool SUMS, int PERM, int FT, int FI, bool F64 = false>
cudaError_t launch_fused_t(const FusedArgs& a, cudaStream_t s) {
    fused_set_attributes<SCHEME, SUMS, PERM, FT, FI, F64>();
    const int max_clusters = fused_max_clusters<SCHEME, SUMS, PERM, FT, FI, F64>(a.CL);
    if (max_clusters < 1) return cudaErrorNotSupported;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = a.CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(FT, 1, 1);
    cfg.dynamicSmemBytes = fused_smem<SCHEME, PERM, FT, FI, F64>();
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int clusters = std::max(1, std::min(a.N, max_clusters));
    cfg.gridDim = dim3(static_cast<unsigned>(clusters * a.CL), 1, 1);
    return cudaLaunchKernelEx(&cfg, k_fused_sorted<SCHEME, SUMS, PERM, FT, FI, F64>, a);
}

template <int FT, int FI, bool F64 = false>
cudaError_t launch_fused_ft(int scheme, int pm, const FusedArgs& a, cudaStream_t s) {
    if constexpr (FT == 512 && !F64) {
        if (scheme == kBuckets)
            return a.sums ? launch_fused_t<kBuckets, true, 0, FT, FI>(a, s) : launch_fused_t<kBuckets, false, 0, FT, FI>(a, s);
        if (scheme == kFromOffspring)
            return pm == 2 ? launch_fused_t<kFromOffspring, false, 2, FT, FI>(a, s)
                           : launch_fused_t<kFromOffspring, false, 1, FT, FI>(a, s);
    }
    if (scheme == 2) {
        if (pm == 2)
            return a.sums ? launch_fused_t<2, true, 2, FT, FI, F64>(a, s) : launch_fused_t<2, false, 2, FT, FI, F64>(a, s);
        if (pm == 1)
            return a.sums ? launch_fused_t<2, true, 1, FT, FI, F64>(a, s) : launch_fused_t<2, false, 1, FT, FI, F64>(a, s);
        return a.sums ? launch_fused_t<2, true, 0, FT, FI, F64>(a, s) : launch_fused_t<2, false, 0, FT, FI, F64>(a, s);
    }
    if (pm == 2)
        return a.sums ? launch_fused_t<3, true, 2, FT, FI, F64>(a, s) : launch_fused_t<3, false, 2, FT, FI, F64>(a, s);
    if (pm == 1)
        return a.sums ? launch_fused_t<3, true, 1, FT, FI, F64>(a, s) : launch_fused_t<3, false, 1, FT, FI, F64>(a, s);
    return a.sums ? launch_fused_t<3, true, 0, FT, FI, F64>(a, s) : launch_fused_t<3, false, 0, FT, FI, F64>(a, s);
}

// can a 16-CTA cluster of 1024-thread CTAs be scheduled (one per GPC)?  cached per device
bool big_clusters_ok() {
    static std::atomic<int> ok[kMaxDevices];
    return cached_per_device(ok, [] { return fused_max_clusters<3, false, 2, 1024, 16>(kMaxCL) >= 1 ? 1 : -1; }) > 0;
}

}  // namespace

// The cooperative kernel handles one filter at a time: ~19 us of grid-sync latency per
// filter up to P ~ 2^20, then ~8.4e10 particles/s; the multi-launch path processes a
// whole batch at ~6.5e10 particles/s after ~20 us of launches (tools/quick_times.py
// --coop-vs-unfused, profiles/r01_dispatch.md).  Take the cooperative kernel when it
// is expected to be faster; both give identical results.
bool coop_supported(int scheme, int32_t N, int32_t P) {
    if (!(scheme == 2 || scheme == 3) || P <= 8 * kPP) return false;
    const double per_filter_excess_us = 19.0 - static_cast<double>(P) / 65000.0;
    return N == 1 || per_filter_excess_us <= 0.0 || static_cast<double>(N) * per_filter_excess_us < 20.0;
}

// deferred runs per filter: at most (slots + extras ranks) / kXS of them
int32_t coop_heavy_cap(int32_t P) { return static_cast<int32_t>(2 * (static_cast<int64_t>(P) / kXS) + 2 * kMaxHeavy); }
size_t coop_scratch_bytes(int32_t P) {
    return static_cast<size_t>(4096) * (4 + 4 + 8 + 8 + 8 + 8) + static_cast<size_t>(P) * 4 + 256 +
           2 * static_cast<size_t>(coop_heavy_cap(P)) * sizeof(uint4) + 16;
}

template <int SCHEME, bool SUMS, int PERM, int FI>
int coop_occupancy() {
    static std::atomic<int> per_sm[kMaxDevices];
    return cached_per_device(per_sm, [] {
        int o = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_coop_sorted<SCHEME, SUMS, PERM, FI>, kFT, 0) !=
                cudaSuccess ||
            o < 1) {
            cudaGetLastError();
            o = 1;
        }
        return o;
    });
}

// particles per thread of the cooperative kernel: 8 (4096-particle sub-tiles) while the filter
// has no more 4096-tiles than co-resident CTAs, so that every CTA holds one short sub-tile; 16
// above (fewer, longer sub-tiles amortise the per-sub-tile barriers).  PF_COOP_FI=8|16 forces one.
int coop_fi(int32_t P, int g_max) {
    static const int forced = [] {
        const char* e = std::getenv("PF_COOP_FI");
        return e ? std::atoi(e) : 0;
    }();
    if (forced == 8 || forced == 16) return forced;
    return (static_cast<int64_t>(P) + kFT * 8 - 1) / (kFT * 8) <= g_max ? 8 : 16;
}

template <int SCHEME, bool SUMS, int PERM, int FI>
cudaError_t launch_coop_fi(CoopArgs& a, cudaStream_t s) {
    constexpr int64_t kSub = static_cast<int64_t>(kFT) * FI;
    int G = std::min(device_sms() * coop_occupancy<SCHEME, SUMS, PERM, FI>(), 4096);
    // chunks are whole sub-tiles; never more CTAs than sub-tiles
    const int64_t tiles = (static_cast<int64_t>(a.P) + kSub - 1) / kSub;
    G = static_cast<int>(std::min<int64_t>(G, tiles));
    const int64_t per = (tiles + G - 1) / G;
    a.CH = per * kSub;
    G = static_cast<int>((static_cast<int64_t>(a.P) + a.CH - 1) / a.CH);
    void* args[] = {&a};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_coop_sorted<SCHEME, SUMS, PERM, FI>), dim3(G),
                                       dim3(kFT), args, 0, s);
}

template <int SCHEME, bool SUMS, int PERM>
cudaError_t launch_coop_t(CoopArgs& a, cudaStream_t s) {
    const int g8 = std::min(device_sms() * coop_occupancy<SCHEME, SUMS, PERM, 8>(), 4096);
    return coop_fi(a.P, g8) == 8 ? launch_coop_fi<SCHEME, SUMS, PERM, 8>(a, s)
                                 : launch_coop_fi<SCHEME, SUMS, PERM, 16>(a, s);
}

template <int PERM>
cudaError_t launch_coop_p(int scheme, bool sums, CoopArgs& a, cudaStream_t s) {
    if constexpr (PERM == 0) {
        if (scheme == kBuckets)
            return sums ? launch_coop_t<kBuckets, true, 0>(a, s) : launch_coop_t<kBuckets, false, 0>(a, s);
    }
    if (scheme == 2) return sums ? launch_coop_t<2, true, PERM>(a, s) : launch_coop_t<2, false, PERM>(a, s);
    return sums ? launch_coop_t<3, true, PERM>(a, s) : launch_coop_t<3, false, PERM>(a, s);
}

cudaError_t launch_coop_sorted(int scheme, const float* logw, int64_t ld, int32_t N, int32_t P, uint64_t seed,
                               uint32_t first_filter, int32_t* anc, int64_t ld_anc, double* lse_out,
                               double* ess_out, int32_t* status_out, int32_t* offspring, int32_t* permuted,
                               void* X, int64_t x_row_bytes, int64_t x_ld, int64_t x_fld, void* scratch,
                               cudaStream_t s, uint64_t* launches, uint64_t* Qout, int64_t ldq, uint64_t* Qtot_out) {
    CoopArgs a{};
    const bool sums = lse_out || ess_out;
    a.logw = logw;
    a.ld = ld;
    a.N = N;
    a.P = P;
    const int m = ceil_log2(P);
    a.D = ((P & (P - 1)) == 0) ? (uint64_t{1} << (64 - m)) : (UINT64_MAX / static_cast<uint64_t>(P));
    a.S = P;
    a.Qout = Qout;
    a.ldq = ldq;
    a.Qtot_out = Qtot_out;
    if (scheme == kBuckets) {  // NB = 2^m bucket boundaries b 2^(64-m) as the slots (ModeBuckets)
        a.S = 1 << m;
        a.D = uint64_t{1} << (64 - m);
    }
    a.key = make_key(seed);
    a.filt0 = first_filter;
    a.kfx = 61 - m;
    a.vec = ((reinterpret_cast<uintptr_t>(logw) & 15) == 0 && ld % 4 == 0) ? 1 : 0;
    a.anc = anc;
    a.ld_anc = ld_anc;
    a.anc_vec = ((reinterpret_cast<uintptr_t>(anc) & 15) == 0 && ld_anc % 4 == 0 &&
                 (!offspring || (reinterpret_cast<uintptr_t>(offspring) & 15) == 0)) ? 1 : 0;
    a.lse_out = lse_out;
    a.ess_out = ess_out;
    a.status_out = status_out;
    a.off = offspring;
    a.perm = permuted;
    (void)x_row_bytes;
    (void)x_ld;
    (void)x_fld;
    char* sc = static_cast<char*>(scratch);
    a.g_max = reinterpret_cast<float*>(sc);
    a.g_bad = reinterpret_cast<int32_t*>(sc + 4096 * 4);
    a.g_tot = reinterpret_cast<uint64_t*>(sc + 4096 * 8);
    a.g_sw = reinterpret_cast<double*>(sc + 4096 * 16);
    a.g_sw2 = reinterpret_cast<double*>(sc + 4096 * 24);
    a.g_ptot = reinterpret_cast<uint64_t*>(sc + 4096 * 32);
    a.freelist = reinterpret_cast<int32_t*>(sc + 4096 * 40);
    {
        const size_t hoff = (static_cast<size_t>(4096) * 40 + static_cast<size_t>(P) * 4 + 255) / 256 * 256;
        a.heavy_cap = coop_heavy_cap(P);
        a.heavy = reinterpret_cast<uint4*>(sc + hoff);
        a.heavy_n = reinterpret_cast<uint32_t*>(sc + hoff + 2 * static_cast<size_t>(a.heavy_cap) * sizeof(uint4));
    }
    const uint64_t NP = static_cast<uint64_t>(N) * static_cast<uint64_t>(P);
    const uint64_t alg = NP * 4u * (1u + (scheme != kBuckets ? 1u : 0u) + (offspring ? 1u : 0u) + (permuted ? 1u : 0u)) +
                         (scheme == kBuckets ? NP * 8u + static_cast<uint64_t>(N) * static_cast<uint64_t>(a.S) * 4u : 0u);
    ProfScope ps_("k_coop_sorted", s, alg);
    if (X) return cudaErrorNotSupported;  // the state gather runs as its own kernel (pf_api.cu)
    cudaError_t e = permuted ? launch_coop_p<1>(scheme, sums, a, s) : launch_coop_p<0>(scheme, sums, a, s);
    ++*launches;
    if (e != cudaSuccess) return e;
    return cudaPeekAtLastError();
}

bool small_supported(int32_t P) { return P >= 1 && P <= kSmallP; }

cudaError_t launch_small(int scheme, bool sorted, const float* logw, int64_t ld, int32_t N, int32_t P, uint64_t seed,
                         uint32_t first_filter, int32_t B, int32_t* anc, int64_t ld_anc, double* lse_out,
                         double* ess_out, float* normw, int32_t* status_out, int32_t* offspring, cudaStream_t s,
                         uint64_t* launches) {
    SmallArgs a{};
    a.logw = logw;
    a.ld = ld;
    a.N = N;
    a.P = P;
    a.scheme = scheme;
    a.B = B;
    a.sorted = sorted ? 1 : 0;
    const int m = ceil_log2(P);
    a.kfx = 61 - m;
    a.D = (P <= 1) ? 0 : (((P & (P - 1)) == 0) ? (uint64_t{1} << (64 - m)) : (UINT64_MAX / static_cast<uint64_t>(P)));
    a.key = make_key(seed);
    a.filt0 = first_filter;
    a.anc = anc;
    a.ld_anc = ld_anc;
    a.lse_out = lse_out;
    a.ess_out = ess_out;
    a.normw = normw;
    a.status_out = status_out;
    a.off = offspring;
    const unsigned grid = static_cast<unsigned>((static_cast<int64_t>(N) + kSmallWarps - 1) / kSmallWarps);
    {
        ProfScope ps_("k_small", s,
                      static_cast<uint64_t>(N) * P * 4u * (2u + (offspring ? 1u : 0u) + (normw ? 1u : 0u)));
        k_small<<<grid, kSmallWarps * 32, 0, s>>>(a);
    }
    ++*launches;
    return cudaPeekAtLastError();
}

bool medium_supported(int32_t P) { return P >= 1 && P <= kMedP; }

template <int T>
cudaError_t launch_medium_t(const SmallArgs& a, size_t smem, cudaStream_t s, uint64_t* launches) {
    static std::atomic<int> attr_set[kMaxDevices];
    cached_per_device(attr_set, [] {
        cudaFuncSetAttribute(k_medium<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kMedP * (8 + 4 + 4) + (kMedP + 4) * 8));
        return 1;
    });
    // occupancy per (device, shared-memory size in KiB)
    constexpr int kKiB = (kMedP * (8 + 4 + 4) + (kMedP + 4) * 8) / 1024 + 2;
    static std::atomic<int> occ_cache[kKiB][kMaxDevices];
    const size_t kib = (smem + 1023) / 1024;
    const int occ = cached_per_device(occ_cache[kib], [&] {
        int o = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_medium<T>, T, kib * 1024) != cudaSuccess || o < 1) {
            cudaGetLastError();
            o = 1;
        }
        return o;
    });
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(a.N, static_cast<int64_t>(device_sms()) * occ));
    {
        ProfScope ps_("k_medium", s,
                      static_cast<uint64_t>(a.N) * a.P * 4u * (2u + (a.off ? 1u : 0u) + (a.normw ? 1u : 0u)));
        k_medium<T><<<grid, T, smem, s>>>(a);
    }
    ++*launches;
    return cudaPeekAtLastError();
}

cudaError_t launch_medium(int scheme, bool sorted, const float* logw, int64_t ld, int32_t N, int32_t P, uint64_t seed,
                          uint32_t first_filter, int32_t B, int32_t* anc, int64_t ld_anc, double* lse_out,
                          double* ess_out, float* normw, int32_t* status_out, int32_t* offspring, cudaStream_t s,
                          uint64_t* launches) {
    SmallArgs a{};
    a.logw = logw;
    a.ld = ld;
    a.N = N;
    a.P = P;
    a.scheme = scheme;
    a.B = B;
    a.sorted = sorted ? 1 : 0;
    const int m = ceil_log2(P);
    a.kfx = 61 - m;
    a.D = (P <= 1) ? 0 : (((P & (P - 1)) == 0) ? (uint64_t{1} << (64 - m)) : (UINT64_MAX / static_cast<uint64_t>(P)));
    a.key = make_key(seed);
    a.filt0 = first_filter;
    a.anc = anc;
    a.ld_anc = ld_anc;
    a.lse_out = lse_out;
    a.ess_out = ess_out;
    a.normw = normw;
    a.status_out = status_out;
    a.off = offspring;
    const size_t P4 = (static_cast<size_t>(P) + 3) & ~size_t{3};
    const size_t smem = P4 * (8 + 4 + 4) + (sorted ? (P4 + 4) * 8 : 0);
    return (P <= 2048) ? launch_medium_t<256>(a, smem, s, launches) : launch_medium_t<1024>(a, smem, s, launches);
}

// the in-place state gather fuses into k_fused_sorted for rows of 16 << k bytes (k <= 5),
// 16-byte aligned rows
bool fused_gather_supported(const void* X, int64_t row_bytes, int64_t ld, int64_t fld) {
    if (!X || row_bytes < 16 || row_bytes > 512 || (row_bytes & (row_bytes - 1)) != 0) return false;
    // row offsets inside a filter are computed in 32 bits: (16 x 16384) rows x ld <= 2^32
    return (reinterpret_cast<uintptr_t>(X) & 15) == 0 && ld % 16 == 0 && fld % 16 == 0 &&
           ld * static_cast<int64_t>(kMaxCL * 1024 * kFI) <= (int64_t{1} << 32);
}

int fused_cluster_ctas(int32_t P) {
    const int FT = (P <= 8 * 512 * kFI) ? 512 : 1024;
    return static_cast<int>((P + FT * kFI - 1) / (FT * kFI));
}

// P <= 65536: any batch.  65536 < P <= 262144 (clusters of 5..16 CTAs of 1024 threads): only
// batches that span the GPU; a single big cluster per filter runs on <= 16 SMs, where the
// cooperative kernel uses all of them (C4: 55.7 vs 62.6 us per PF step).
// multinomial: the bucket index + Q from one cluster-kernel launch (kBuckets: the rho = 0
// systematic machinery over NB = 2^ceil(log2 P) slots of width 2^(64 - m)), then the per-slot
// searches; above the sizes the CTA-per-filter kernel takes
bool buckets_fused_supported(int32_t P) { return P > 2048 && P <= 8 * 512 * kFI; }

bool fused_supported(int scheme, int32_t N, int32_t P) {
    if (!(scheme == 2 || scheme == 3) || P < 1) return false;
    if (P <= 8 * 512 * kFI) return true;
    return P <= kMaxCL * 1024 * kFI && static_cast<int64_t>(N) * fused_cluster_ctas(P) >= sm_count() &&
           big_clusters_ok();
}

cudaError_t launch_fused_sorted(int scheme, const float* logw, int64_t ld, int32_t N, int32_t P, uint64_t seed,
                                uint32_t first_filter, int32_t* anc, int64_t ld_anc, double* lse_out,
                                double* ess_out, float* normw, int32_t* status_out, int32_t* offspring,
                                int32_t* permuted, void* X, int64_t x_row_bytes, int64_t x_ld, int64_t x_fld,
                                cudaStream_t s, uint64_t* launches, const double* logw64, uint64_t* Qout,
                                int64_t ldq, uint64_t* Qtot_out) {
    FusedArgs a{};
    a.logw = logw;
    a.logw64 = logw64;
    a.Qout = Qout;
    a.ldq = ldq;
    a.Qtot_out = Qtot_out;
    a.ld = ld;
    a.N = N;
    a.P = P;
    // geometry: 512 threads (8192 particles per CTA) up to 8 CTAs, else 1024 threads (16384).
    // Systematic filters of 16385..65536 particles without the state gather: 256 threads (4096
    // per CTA, clusters of 5..16, 4 CTAs per SM; C3 resample 0.469 -> 0.452 ms, with the
    // permutation 0.850 -> 0.773 ms: more, smaller CTAs per SM hide each cluster's barrier
    // skew).  PF_FUSED_FT=256|512 forces one where both apply (diagnostics).
    static const int ft_env = [] {
        const char* e = std::getenv("PF_FUSED_FT");
        return e ? std::atoi(e) : 0;
    }();
    const bool ft256_ok = !logw64 && P <= 16 * 256 * kFI && scheme != kBuckets;
    const bool ft256_default = ft256_ok && scheme == 3 && !X && P > 4 * 256 * kFI;
    int FT = ((ft_env == 256 && ft256_ok) || (ft_env != 512 && ft256_default))
                 ? 256
                 : ((P <= 8 * 512 * kFI) ? 512 : 1024);
    auto set_geometry = [&](int ft) {
        a.CL = static_cast<int32_t>((P + ft * kFI - 1) / (ft * kFI));
        int64_t pp = (P + a.CL - 1) / a.CL;
        pp = (pp + 3) / 4 * 4;
        a.PP = static_cast<int32_t>(pp);
    };
    set_geometry(FT);
    const int m = ceil_log2(P);
    a.D = (P <= 1) ? 0 : (((P & (P - 1)) == 0) ? (uint64_t{1} << (64 - m)) : (UINT64_MAX / static_cast<uint64_t>(P)));
    a.S = P;
    if (scheme == kBuckets) {
        // NB = 2^m equal buckets of the 64-bit uniform: positions b 2^(64-m) (ModeBuckets)
        a.S = 1 << m;
        a.D = uint64_t{1} << (64 - m);
    }
    a.key = make_key(seed);
    a.filt0 = first_filter;
    a.kfx = 61 - m;
    a.vec = logw64 ? (((reinterpret_cast<uintptr_t>(logw64) & 15) == 0 && ld % 2 == 0) ? 1 : 0)
                   : (((reinterpret_cast<uintptr_t>(logw) & 15) == 0 && ld % 4 == 0) ? 1 : 0);
    a.sums = (lse_out || ess_out || normw) ? 1 : 0;
    a.anc = anc;
    a.ld_anc = ld_anc;
    a.anc_vec = ((reinterpret_cast<uintptr_t>(anc) & 15) == 0 && ld_anc % 4 == 0) ? 1 : 0;
    a.lse_out = lse_out;
    a.ess_out = ess_out;
    a.normw = normw;
    a.status_out = status_out;
    a.off = offspring;
    a.perm = permuted;
    a.X = static_cast<char*>(X);
    a.xld = x_ld;
    a.xfld = x_fld;
    a.xlg = 0;
    while ((int64_t{16} << a.xlg) < x_row_bytes) ++a.xlg;
    // algorithmic bytes: log-weights once, each requested output once (bucket mode: Q and the
    // bucket index), plus one read and one write per moved state row
    const uint64_t NP = static_cast<uint64_t>(N) * static_cast<uint64_t>(P);
    const uint64_t alg = NP * (logw64 ? 8u : 4u) +
                         NP * 4u * ((scheme != kBuckets ? 1u : 0u) + (offspring ? 1u : 0u) + (permuted ? 1u : 0u) +
                                    (normw ? 1u : 0u)) +
                         (scheme == kBuckets ? NP * 8u + static_cast<uint64_t>(N) * static_cast<uint64_t>(a.S) * 4u : 0u);
    ProfScope ps_("k_fused_sorted", s, alg, X ? 2u * static_cast<uint64_t>(x_row_bytes) : 0u);
    cudaError_t e;
    const int pm = a.X ? 2 : (a.perm ? 1 : 0);
    if (logw64) {
        if (FT != 512) return cudaErrorNotSupported;  // binary64 fused for P <= 65536 only (f64_fused_supported)
        e = launch_fused_ft<512, 16, true>(scheme, pm, a, s);
    } else {
        if (FT == 256) {
            e = launch_fused_ft<256, 16>(scheme, pm, a, s);
            if (e == cudaErrorNotSupported) {  // 16-CTA clusters not schedulable here: 512 threads
                FT = 512;
                set_geometry(FT);
            }
        }
        if (FT != 256)
            e = (FT == 512) ? launch_fused_ft<512, 16>(scheme, pm, a, s) : launch_fused_ft<1024, 16>(scheme, pm, a, s);
    }
    ++*launches;
    if (e != cudaSuccess) return e;
    return cudaPeekAtLastError();
}

// The canonical permutation (NS-15) and the in-place state gather (NS-16) of a batch from its
// offspring counts, in one cluster-kernel launch (phase D of k_fused_sorted on counts read from
// memory): the fused a9 + a10 for the schemes whose ancestors are unsorted (multinomial,
// Metropolis) and for pf_permute_offspring.  X nullable (permutation only).
bool fused_from_offspring_supported(int32_t P) { return P >= 1 && P <= 8 * 512 * kFI; }

cudaError_t launch_fused_from_offspring(const int32_t* off, int64_t ld_off, int32_t N, int32_t P, int32_t* perm,
                                        int64_t ld_perm, void* X, int64_t x_row_bytes, int64_t x_ld, int64_t x_fld,
                                        cudaStream_t s, uint64_t* launches) {
    FusedArgs a{};
    a.N = N;
    a.P = P;
    a.CL = static_cast<int32_t>((P + 512 * kFI - 1) / (512 * kFI));
    int64_t pp = (P + a.CL - 1) / a.CL;
    a.PP = static_cast<int32_t>((pp + 3) / 4 * 4);
    a.off_in = off;
    a.ld_off_in = ld_off;
    a.perm = perm;
    a.ld_anc = ld_perm;
    a.anc_vec = ((reinterpret_cast<uintptr_t>(perm) & 15) == 0 && ld_perm % 4 == 0 &&
                 (reinterpret_cast<uintptr_t>(off) & 15) == 0 && ld_off % 4 == 0) ? 1 : 0;
    a.X = static_cast<char*>(X);
    a.xld = x_ld;
    a.xfld = x_fld;
    a.xlg = 0;
    while ((int64_t{16} << a.xlg) < x_row_bytes) ++a.xlg;
    const uint64_t NP = static_cast<uint64_t>(N) * static_cast<uint64_t>(P);
    ProfScope ps_("k_fused_perm", s, NP * 8u, X ? 2u * static_cast<uint64_t>(x_row_bytes) : 0u);
    const cudaError_t e = launch_fused_ft<512, 16>(kFromOffspring, X ? 2 : 1, a, s);
    ++*launches;
    if (e != cudaSuccess) return e;
    return cudaPeekAtLastError();
}

}  // namespace pf
