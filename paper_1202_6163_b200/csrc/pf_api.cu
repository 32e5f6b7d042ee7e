// pf_api.cu — C ABI of libpfresample (include/pf.h): argument validation,
// the (device, stream)-keyed workspace pool ("pooled memory") and
// the stage sequence of each entry point.  No torch types, no host sync.
#include <atomic>
#include <cmath>
#include <map>
#include <mutex>
#include <cstring>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "../../include/pf.h"
#include "pf_device.cuh"
#include "pf_internal.h"

namespace {

std::atomic<uint64_t> g_launches{0};
std::atomic<bool> g_no_fusion{false};  // pf_set_fusion(0): diagnostics, multi-launch paths everywhere

struct PoolBlock {
    void* ptr = nullptr;
    size_t bytes = 0;
};

std::mutex g_pool_mu;
std::map<std::tuple<int, void*, int>, PoolBlock>& pool() {
    static auto* m = new std::map<std::tuple<int, void*, int>, PoolBlock>();
    return *m;
}

// Returns a device workspace of >= bytes for (current device, stream, slot).  Growth
// is stream-ordered (cudaFreeAsync / cudaMallocAsync) and happens only when a
// call needs more than any earlier call on that stream.  Slot 1 holds the binary64
// entry points' shifted log-weights, which stay live while the float path uses slot 0.
pf_status pool_get(size_t bytes, cudaStream_t s, void** out, int slot = 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return PF_ERR_CUDA;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    PoolBlock& b = pool()[{dev, static_cast<void*>(s), slot}];
    if (b.bytes < bytes) {
        if (b.ptr) cudaFreeAsync(b.ptr, s);
        b.ptr = nullptr;
        b.bytes = 0;
        const size_t want = bytes + bytes / 4 + (1u << 20);
        if (cudaMallocAsync(&b.ptr, want, s) != cudaSuccess) {
            cudaGetLastError();
            b.ptr = nullptr;
            return PF_ERR_WORKSPACE;
        }
        b.bytes = want;
    }
    *out = b.ptr;
    return PF_OK;
}

pf_status get_workspace(const pf_opts* opts, size_t bytes, cudaStream_t s, void** out) {
    if (opts && opts->workspace) {
        if (opts->workspace_bytes < bytes || (reinterpret_cast<uintptr_t>(opts->workspace) & 255) != 0)
            return PF_ERR_WORKSPACE;
        *out = opts->workspace;
        return PF_OK;
    }
    return pool_get(bytes, s, out);
}

// ---------------------------------------------------------------- tracing
struct ProfRecord {
    const char* name;
    cudaEvent_t start, stop;
    uint64_t alg_bytes, row_bytes;
};
std::atomic<bool> g_prof_on{false};
std::mutex g_prof_mu;
std::vector<ProfRecord>& prof_records() {
    static auto* v = new std::vector<ProfRecord>();
    return *v;
}
std::vector<cudaEvent_t>& prof_free_events() {
    static auto* v = new std::vector<cudaEvent_t>();
    return *v;
}
cudaEvent_t prof_event() {
    auto& fr = prof_free_events();
    if (!fr.empty()) {
        cudaEvent_t e = fr.back();
        fr.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

pf_status cuda_status(cudaError_t e) { return e == cudaSuccess ? PF_OK : PF_ERR_CUDA; }

unsigned needs_for(int scheme) {
    if (scheme == PF_METROPOLIS) return pf::kNeedW;
    if (scheme == PF_MULTINOMIAL) return pf::kNeedQ | pf::kNeedBuckets;
    return pf::kNeedQ;
}

// k_medium (one CTA per filter) against the cluster kernel and the multi-launch path, from
// the measured table in profiles/r01_dispatch.md: it wins everywhere up to P = 2048 (the
// cluster kernel idles most of its 8192-slot CTAs there), stays ahead for stratified and
// small multinomial batches up to 4096, and loses above (a single CTA per filter limits the
// parallelism of one filter to one SM).  Metropolis: only up to P = 1024.
// P <= 256: the warp-per-filter kernel packs 8 filters per CTA and wins for batches of
// >= 256 filters; below that the CTA-per-filter kernel has the lower latency
// (3.3-3.8 us vs 5-8 us at N <= 64, profiles/r01_dispatch.md)
#ifndef PF_SMALL_MIN_N
#define PF_SMALL_MIN_N 256
#endif
bool medium_preferred(int scheme, int32_t N, int32_t P) {
    if (P <= 1024) return true;
    if (P <= 2048) return scheme != PF_METROPOLIS;
    if (P <= 4096) return scheme == PF_STRATIFIED || (scheme == PF_MULTINOMIAL && N <= 128);
    return false;
}

// one launch per batch: cluster-per-filter kernel (ancestors, offspring, permutation and the
// state gather), no workspace except the permutation when the state is gathered without
// permuted_out (pf_fused.cu).  logw64 non-null: the binary64 instantiation (NS-3d), P <= 65536.
pf_status fused_branch(int scheme, const float* logw, const double* logw64, int64_t ld, int32_t N, int32_t P,
                       uint64_t seed, uint32_t first_filter, int32_t* anc, int64_t ld_anc, const pf_opts* opts,
                       cudaStream_t s) {
    double* lse = opts ? opts->lse_out : nullptr;
    double* ess = opts ? opts->ess_out : nullptr;
    float* normw = opts ? opts->normw_out : nullptr;
    int32_t* status_out = opts ? opts->status_out : nullptr;
    int32_t* offspring_out = opts ? opts->offspring_out : nullptr;
    int32_t* permuted_out = opts ? opts->permuted_out : nullptr;
    void* state = opts ? opts->state : nullptr;
    const int64_t x_row = opts ? opts->state_row_bytes : 0, x_ld = opts ? opts->state_ld_bytes : 0;
    const int64_t x_fld = opts ? opts->state_filter_ld_bytes : 0;
    // The cluster kernel gathers the state itself when the batch spans the GPU; a batch of few
    // filters (one cluster each) would copy its rows through a handful of SMs, so there the
    // permutation is fused and the gather runs as its own full-GPU kernel.
    const bool fuse_gather = state && pf::fused_gather_supported(state, x_row, x_ld, x_fld) &&
                             static_cast<int64_t>(N) * pf::fused_cluster_ctas(P) >= pf::sm_count();
    int32_t* perm = permuted_out;
    void* fstate = fuse_gather ? state : nullptr;
    if (state && !perm) {
        void* p = nullptr;
        const pf_status st = get_workspace(opts, static_cast<size_t>(N) * static_cast<size_t>(ld_anc) * 4, s, &p);
        if (st != PF_OK) return st;
        perm = static_cast<int32_t*>(p);
    }
    uint64_t nl = 0;
    cudaError_t e = pf::launch_fused_sorted(scheme, logw, ld, N, P, seed, first_filter, anc, ld_anc, lse, ess, normw,
                                            status_out, offspring_out, perm, fstate, x_row, x_ld, x_fld, s, &nl,
                                            logw64);
    if (e == cudaSuccess && state && !fstate)
        e = pf::launch_gather_inplace(state, x_row, x_ld, x_fld, N, P, perm, ld_anc, s, &nl);
    g_launches += nl;
    return cuda_status(e);
}

// Canonical permutation (+ the in-place gather) from offspring counts in one cluster-kernel
// launch when the batch spans the GPU (P <= 65536; pf_fused.cu launch_fused_from_offspring);
// false: the caller takes the lookback path (k_pscan + k_push, then k_gather_rows16).
bool fused_permute_preferred(int32_t N, int32_t P) {
    return !g_no_fusion.load() && pf::fused_from_offspring_supported(P) &&
           static_cast<int64_t>(N) * pf::fused_cluster_ctas(P) >= pf::sm_count();
}

cudaError_t permute_gather_from_offspring(const int32_t* off, int64_t ld_off, int32_t N, int32_t P, int32_t* perm,
                                          int64_t ld_perm, void* state, int64_t x_row, int64_t x_ld, int64_t x_fld,
                                          cudaStream_t s, uint64_t* nl) {
    const bool fuse_gather = state && pf::fused_gather_supported(state, x_row, x_ld, x_fld);
    cudaError_t e = pf::launch_fused_from_offspring(off, ld_off, N, P, perm, ld_perm, fuse_gather ? state : nullptr,
                                                    x_row, x_ld, x_fld, s, nl);
    if (e == cudaSuccess && state && !fuse_gather)
        e = pf::launch_gather_inplace(state, x_row, x_ld, x_fld, N, P, perm, ld_perm, s, nl);
    return e;
}

pf_status resample_core(int scheme, const float* logw, int64_t ld, int32_t N, int32_t P, uint64_t seed,
                        uint32_t first_filter, int32_t B, int32_t* anc, int64_t ld_anc, const pf_opts* opts,
                        cudaStream_t s) {
    if (!logw || !anc) return PF_ERR_INVALID_ARG;
    if (scheme < PF_MULTINOMIAL || scheme > PF_METROPOLIS) return PF_ERR_INVALID_ARG;
    if (N < 1 || P < 1 || B < 0 || ld < P || ld_anc < P) return PF_ERR_INVALID_ARG;
    if (opts && (opts->flags & ~static_cast<uint32_t>(PF_NO_FUSION | PF_SORTED)) != 0) return PF_ERR_UNSUPPORTED;
    const bool sorted_multi = opts && (opts->flags & PF_SORTED);
    if (sorted_multi && scheme != PF_MULTINOMIAL) return PF_ERR_UNSUPPORTED;
    double* lse = opts ? opts->lse_out : nullptr;
    double* ess = opts ? opts->ess_out : nullptr;
    float* normw = opts ? opts->normw_out : nullptr;
    int32_t* status_out = opts ? opts->status_out : nullptr;
    int32_t* offspring_out = opts ? opts->offspring_out : nullptr;
    int32_t* permuted_out = opts ? opts->permuted_out : nullptr;

    void* state = opts ? opts->state : nullptr;
    const int64_t x_row = opts ? opts->state_row_bytes : 0, x_ld = opts ? opts->state_ld_bytes : 0;
    const int64_t x_fld = opts ? opts->state_filter_ld_bytes : 0;
    if (state && (x_row < 1 || x_ld < x_row || (N > 1 && x_fld < x_ld * static_cast<int64_t>(P))))
        return PF_ERR_INVALID_ARG;

    const bool no_fusion = (opts && (opts->flags & PF_NO_FUSION)) || g_no_fusion.load();
    if (!no_fusion && pf::small_supported(P) && !permuted_out && !state && N >= PF_SMALL_MIN_N) {
        // one warp per filter, every scheme, one launch (pf_fused.cu k_small)
        uint64_t nl = 0;
        const cudaError_t e = pf::launch_small(scheme, sorted_multi, logw, ld, N, P, seed, first_filter, B, anc, ld_anc,
                                               lse, ess, normw, status_out, offspring_out, s, &nl);
        g_launches += nl;
        return cuda_status(e);
    }
    if (!no_fusion && pf::medium_supported(P) && !permuted_out && !state && medium_preferred(scheme, N, P)) {
        // one CTA per filter, every scheme, one launch (pf_fused.cu k_medium)
        uint64_t nl = 0;
        const cudaError_t e = pf::launch_medium(scheme, sorted_multi, logw, ld, N, P, seed, first_filter, B, anc,
                                                ld_anc, lse, ess, normw, status_out, offspring_out, s, &nl);
        g_launches += nl;
        return cuda_status(e);
    }
    if (!no_fusion && pf::fused_supported(scheme, N, P))
        return fused_branch(scheme, logw, nullptr, ld, N, P, seed, first_filter, anc, ld_anc, opts, s);
    if ((permuted_out || state) && !no_fusion && !normw && pf::coop_supported(scheme, N, P)) {
        // large filters, few of them: the cooperative kernel writes the permutation too (and gathers
        // the state when the rows allow it); scratch = [coop scratch + free list | offspring | perm]
        const size_t plane = static_cast<size_t>(N) * static_cast<size_t>(ld_anc) * 4;
        const size_t o1 = (pf::coop_scratch_bytes(P) + 255) / 256 * 256;
        const size_t o2 = o1 + (offspring_out ? 0 : (plane + 255) / 256 * 256);
        const size_t need = o2 + (permuted_out ? 0 : plane);
        void* big = nullptr;
        const pf_status st0 = get_workspace(opts, need, s, &big);
        if (st0 != PF_OK) return st0;
        char* b = static_cast<char*>(big);
        int32_t* off = offspring_out ? offspring_out : reinterpret_cast<int32_t*>(b + o1);
        int32_t* perm = permuted_out ? permuted_out : reinterpret_cast<int32_t*>(b + o2);
        // the state gather runs as its own full-GPU kernel: inside the cooperative kernel the copies
        // of each CTA's chunk serialise behind its permutation work (P = 2^18: 51.7 vs 41.2 us;
        // 2^20: 66.2 vs 61.2 us, profiles/r01_dispatch.md)
        uint64_t nl = 0;
        cudaError_t e = pf::launch_coop_sorted(scheme, logw, ld, N, P, seed, first_filter, anc, ld_anc, lse, ess,
                                               status_out, off, perm, nullptr, 0, 0, 0, big, s, &nl);
        if (e == cudaSuccess && state)
            e = pf::launch_gather_inplace(state, x_row, x_ld, x_fld, N, P, perm, ld_anc, s, &nl);
        g_launches += nl;
        return cuda_status(e);
    }
    if (permuted_out || state) {
        // not fused for this size/scheme/row layout: resample (offspring as a side output), then
        // the canonical permutation from the offspring (k_pscan + k_push), then the gather.  One
        // pool block holds [permutation scratch | offspring (if the caller gave none) | permutation
        // (if the caller gave none) | resample workspace].
        if (opts && opts->workspace) return PF_ERR_UNSUPPORTED;
        const pf::Layout LP = pf::make_layout(N, P, pf::kNeedPermute);
        const pf::Layout LR = pf::make_layout(N, P, needs_for(scheme) | (sorted_multi ? pf::kNeedG : 0u));
        const size_t plane = static_cast<size_t>(N) * static_cast<size_t>(ld_anc) * 4;
        const size_t off_bytes = offspring_out ? 0 : plane;
        const size_t perm_bytes = permuted_out ? 0 : plane;
        const size_t o1 = (LP.total + 255) / 256 * 256;
        const size_t o1p = (o1 + off_bytes + 255) / 256 * 256;
        const size_t o2b = (o1p + perm_bytes + 255) / 256 * 256;
        void* big = nullptr;
        pf_status st0 = pool_get(o2b + LR.total, s, &big);
        if (st0 != PF_OK) return st0;
        const pf::Ws wp = pf::carve(big, LP);
        int32_t* off = offspring_out ? offspring_out : reinterpret_cast<int32_t*>(static_cast<char*>(big) + o1);
        int32_t* perm = permuted_out ? permuted_out : reinterpret_cast<int32_t*>(static_cast<char*>(big) + o1p);
        pf_opts o2 = opts ? *opts : pf_opts{};
        o2.permuted_out = nullptr;
        o2.state = nullptr;
        o2.offspring_out = off;
        o2.workspace = static_cast<char*>(big) + o2b;
        o2.workspace_bytes = LR.total;
        pf_status st2 = resample_core(scheme, logw, ld, N, P, seed, first_filter, B, anc, ld_anc, &o2, s);
        if (st2 != PF_OK) return st2;
        uint64_t nl = 0;
        if (!no_fusion && fused_permute_preferred(N, P)) {
            // a9 + a10 fused: the cluster kernel's phase D on the offspring (one launch)
            const cudaError_t e = permute_gather_from_offspring(off, ld_anc, N, P, perm, ld_anc, state, x_row, x_ld,
                                                                x_fld, s, &nl);
            g_launches += nl;
            return cuda_status(e);
        }
        cudaError_t e = cudaMemsetAsync(static_cast<char*>(big) + LP.zero_begin, 0, LP.zero_end - LP.zero_begin, s);
        if (e == cudaSuccess) e = pf::launch_permute_from_offspring(off, ld_anc, N, P, LP, wp, perm, ld_anc, s, &nl);
        if (e == cudaSuccess && state)
            e = pf::launch_gather_inplace(state, x_row, x_ld, x_fld, N, P, perm, ld_anc, s, &nl);
        g_launches += nl;
        return cuda_status(e);
    }
    if (!no_fusion && !normw && pf::coop_supported(scheme, N, P)) {
        // one cooperative launch for large filters (pf_fused.cu); tiny scratch from the pool
        void* sc = nullptr;
        pf_status st2 = get_workspace(opts, pf::coop_scratch_bytes(P), s, &sc);
        if (st2 != PF_OK) return st2;
        uint64_t nl = 0;
        const cudaError_t e = pf::launch_coop_sorted(scheme, logw, ld, N, P, seed, first_filter, anc, ld_anc, lse,
                                                     ess, status_out, offspring_out, nullptr, nullptr, 0, 0, 0, sc,
                                                     s, &nl);
        g_launches += nl;
        return cuda_status(e);
    }
    const pf::Layout L = pf::make_layout(N, P, needs_for(scheme) | (sorted_multi ? pf::kNeedG : 0u));
    void* base = nullptr;
    pf_status st = get_workspace(opts, L.total, s, &base);
    if (st != PF_OK) return st;
    const pf::Ws ws = pf::carve(base, L);
    uint64_t nl = 0;
    if (!no_fusion && scheme == PF_MULTINOMIAL && !sorted_multi && pf::buckets_fused_supported(P)) {
        // one cluster-kernel launch writes Q, the totals, the status, the side outputs and the
        // bucket index (the rho = 0 systematic positions); then the per-slot searches
        cudaError_t e = pf::launch_fused_sorted(pf::kFusedBuckets, logw, ld, N, P, seed, first_filter, ws.bidx, L.ldb,
                                                lse, ess, normw, ws.fstatus, nullptr, nullptr, nullptr, 0, 0, 0, s, &nl,
                                                nullptr, ws.Q, L.ldq, ws.Qtot);
        if (e == cudaSuccess) e = pf::launch_bsearch_buckets(N, P, L, ws, seed, first_filter, anc, ld_anc, s, &nl);
        if (e == cudaSuccess && status_out)
            e = cudaMemcpyAsync(status_out, ws.fstatus, static_cast<size_t>(N) * 4, cudaMemcpyDeviceToDevice, s);
        if (offspring_out && e == cudaSuccess)
            e = pf::launch_offspring(anc, ld_anc, N, P, offspring_out, ld_anc, s, &nl);
        g_launches += nl;
        return cuda_status(e);
    }
    if (!no_fusion && scheme == PF_MULTINOMIAL && !sorted_multi && !normw && !(opts && opts->workspace) &&
        pf::coop_supported(PF_SYSTEMATIC, N, P)) {
        // large filters, few of them: the cooperative kernel's bucket mode (Q, totals, status, lse /
        // ESS and the bucket index in one launch), then the per-slot searches
        void* sc = nullptr;
        pf_status st2 = pool_get(pf::coop_scratch_bytes(P), s, &sc, 3);
        if (st2 != PF_OK) return st2;
        cudaError_t e = pf::launch_coop_sorted(pf::kFusedBuckets, logw, ld, N, P, seed, first_filter, ws.bidx, L.ldb,
                                               lse, ess, ws.fstatus, nullptr, nullptr, nullptr, 0, 0, 0, sc, s, &nl,
                                               ws.Q, L.ldq, ws.Qtot);
        if (e == cudaSuccess) e = pf::launch_bsearch_buckets(N, P, L, ws, seed, first_filter, anc, ld_anc, s, &nl);
        if (e == cudaSuccess && status_out)
            e = cudaMemcpyAsync(status_out, ws.fstatus, static_cast<size_t>(N) * 4, cudaMemcpyDeviceToDevice, s);
        if (offspring_out && e == cudaSuccess)
            e = pf::launch_offspring(anc, ld_anc, N, P, offspring_out, ld_anc, s, &nl);
        g_launches += nl;
        return cuda_status(e);
    }
    cudaError_t e = cudaMemsetAsync(static_cast<char*>(base) + L.zero_begin, 0, L.zero_end - L.zero_begin, s);
    if (sorted_multi && e == cudaSuccess)  // spacings do not depend on the weights: first
        e = pf::launch_sorted_multinomial(N, P, L, ws, seed, first_filter, anc, ld_anc, s, &nl, true);
    if (e == cudaSuccess) e = pf::launch_max(logw, ld, N, P, L, ws, status_out, s, &nl);
    const bool side = lse || ess || normw;
    if (scheme != PF_METROPOLIS) {
        if (e == cudaSuccess) e = pf::launch_scan(logw, ld, N, P, L, ws, P > 1, lse, ess, s, &nl);
        if (e == cudaSuccess) {
            if (P == 1) e = pf::launch_identity(N, P, anc, ld_anc, s, &nl);
            else if (sorted_multi)
                e = pf::launch_sorted_multinomial(N, P, L, ws, seed, first_filter, anc, ld_anc, s, &nl, false);
            else e = pf::launch_search(scheme, N, P, L, ws, seed, first_filter, anc, ld_anc, s, &nl);
        }
    } else {
        if (side && e == cudaSuccess) e = pf::launch_scan(logw, ld, N, P, L, ws, false, lse, ess, s, &nl);
        if (e == cudaSuccess)
            e = pf::launch_metropolis(logw, ld, N, P, L, ws, seed, first_filter, B, anc, ld_anc, s, &nl);
    }
    if (normw && e == cudaSuccess) e = pf::launch_normw(logw, ld, N, P, ws, normw, s, &nl);
    if (offspring_out && e == cudaSuccess) e = pf::launch_offspring(anc, ld_anc, N, P, offspring_out, ld_anc, s, &nl);
    g_launches += nl;
    return cuda_status(e);
}

// NS-17 (PF_SORT_WEIGHTS): segmented radix sort of the log-weights (descending) into a
// slot-2 pool block, the float path on the sorted weights (ancestors b in sorted space), then
// a_k = sigma[b_k] and normw back in the original order; offspring / permutation / state run
// on the mapped ancestors (histogram, k_pscan + k_push, gather).
pf_status resample_sorted_weights(int scheme, const float* logw, int64_t ld, int32_t N, int32_t P, uint64_t seed,
                                  uint32_t first_filter, int32_t* anc, int64_t ld_anc, const pf_opts* opts,
                                  cudaStream_t s) {
    if (!logw || !anc) return PF_ERR_INVALID_ARG;
    if (scheme < PF_MULTINOMIAL || scheme > PF_METROPOLIS) return PF_ERR_INVALID_ARG;
    if (N < 1 || P < 1 || ld < P || ld_anc < P) return PF_ERR_INVALID_ARG;
    const uint32_t flags = opts->flags;
    if ((flags & ~static_cast<uint32_t>(PF_NO_FUSION | PF_SORT_WEIGHTS)) != 0 || scheme == PF_METROPOLIS)
        return PF_ERR_UNSUPPORTED;
    void* state = opts->state;
    const int64_t x_row = opts->state_row_bytes, x_ld = opts->state_ld_bytes, x_fld = opts->state_filter_ld_bytes;
    if (state && (x_row < 1 || x_ld < x_row || (N > 1 && x_fld < x_ld * static_cast<int64_t>(P))))
        return PF_ERR_INVALID_ARG;
    const size_t sort_bytes = (pf::wsort_ws_bytes(N, P, opts->normw_out != nullptr) + 255) / 256 * 256;
    const bool own_perm = state && !opts->permuted_out;
    void* ws = nullptr;
    pf_status st = pool_get(sort_bytes + (own_perm ? static_cast<size_t>(N) * static_cast<size_t>(ld_anc) * 4 : 0),
                            s, &ws, 2);
    if (st != PF_OK) return st;
    pf::WsortBufs w{};
    uint64_t nl = 0;
    cudaError_t e = pf::launch_wsort(logw, ld, N, P, ws, opts->normw_out != nullptr, &w, s, &nl);
    g_launches += nl;
    if (e != cudaSuccess) return cuda_status(e);
    pf_opts o2{};
    o2.flags = flags & PF_NO_FUSION;
    o2.lse_out = opts->lse_out;
    o2.ess_out = opts->ess_out;
    o2.status_out = w.fstatus;
    o2.normw_out = w.vs;
    o2.workspace = opts->workspace;
    o2.workspace_bytes = opts->workspace_bytes;
    st = resample_core(scheme, w.y, w.ldk, N, P, seed, first_filter, 0, w.b, w.ldk, &o2, s);
    if (st != PF_OK) return st;
    nl = 0;
    e = pf::launch_unsort(w, N, P, anc, ld_anc, opts->normw_out, s, &nl);
    g_launches += nl;
    if (e == cudaSuccess && opts->status_out)
        e = cudaMemcpyAsync(opts->status_out, w.fstatus, static_cast<size_t>(N) * 4, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_status(e);
    if (opts->offspring_out) {
        st = pf_ancestors_to_offspring_batched(anc, ld_anc, N, P, opts->offspring_out, ld_anc, s);
        if (st != PF_OK) return st;
    }
    if (opts->permuted_out || state) {
        int32_t* perm = own_perm ? reinterpret_cast<int32_t*>(static_cast<char*>(ws) + sort_bytes) : opts->permuted_out;
        st = pf_permute_batched(anc, ld_anc, N, P, perm, ld_anc, s);
        if (st == PF_OK && state) st = pf_gather_state_batched(state, x_row, x_ld, x_fld, N, P, perm, ld_anc, s);
    }
    return st;
}

pf_status resample_impl(int scheme, const float* logw, int64_t ld, int32_t N, int32_t P, uint64_t seed,
                        uint32_t first_filter, int32_t B, int32_t* anc, int64_t ld_anc, const pf_opts* opts,
                        cudaStream_t s) {
    if (opts && (opts->flags & PF_SORT_WEIGHTS))
        return resample_sorted_weights(scheme, logw, ld, N, P, seed, first_filter, anc, ld_anc, opts, s);
    return resample_core(scheme, logw, ld, N, P, seed, first_filter, B, anc, ld_anc, opts, s);
}

// NS-3d: binary64 log-weights -> t = fl32(logw - lmax) in a slot-1 pool block -> the float32
// path on t (every dispatch of resample_impl applies) -> lse += lmax
pf_status resample_f64_impl(int scheme, const double* logw, int64_t ld, int32_t N, int32_t P, uint64_t seed,
                            uint32_t first_filter, int32_t B, int32_t* anc, int64_t ld_anc, const pf_opts* opts,
                            cudaStream_t s) {
    if (!logw || !anc) return PF_ERR_INVALID_ARG;
    if (scheme < PF_MULTINOMIAL || scheme > PF_METROPOLIS) return PF_ERR_INVALID_ARG;
    if (N < 1 || P < 1 || B < 0 || ld < P || ld_anc < P) return PF_ERR_INVALID_ARG;
    if (opts && (opts->flags & ~static_cast<uint32_t>(PF_NO_FUSION | PF_SORTED | PF_SORT_WEIGHTS)) != 0)
        return PF_ERR_UNSUPPORTED;
    if (opts && (opts->flags & PF_SORTED) && scheme != PF_MULTINOMIAL) return PF_ERR_UNSUPPORTED;
    const uint32_t fl = opts ? opts->flags : 0u;
    void* state = opts ? opts->state : nullptr;
    if (state && (opts->state_row_bytes < 1 || opts->state_ld_bytes < opts->state_row_bytes ||
                  (N > 1 && opts->state_filter_ld_bytes < opts->state_ld_bytes * static_cast<int64_t>(P))))
        return PF_ERR_INVALID_ARG;
    // stratified / systematic batches of 4097..65536-particle filters: the cluster kernel reads the
    // doubles itself (max, then t_i = fl32(logw_i - lmax) from a second, L2-resident read)
    if (!(fl & (PF_NO_FUSION | PF_SORT_WEIGHTS)) && !g_no_fusion.load() &&
        (scheme == PF_STRATIFIED || scheme == PF_SYSTEMATIC) && P > 4096 && P <= pf::kFusedF64MaxP)
        return fused_branch(scheme, nullptr, logw, ld, N, P, seed, first_filter, anc, ld_anc, opts, s);
    void* ws = nullptr;
    pf_status st = pool_get(pf::f64_ws_bytes(N, P), s, &ws, 1);
    if (st != PF_OK) return st;
    float* t = nullptr;
    int64_t ldt = 0;
    unsigned long long* key = nullptr;
    uint64_t nl = 0;
    cudaError_t e = pf::launch_shift64(logw, ld, N, P, ws, &t, &ldt, &key, s, &nl);
    g_launches += nl;
    if (e != cudaSuccess) return cuda_status(e);
    st = resample_impl(scheme, t, ldt, N, P, seed, first_filter, B, anc, ld_anc, opts, s);
    if (st != PF_OK || !opts || !opts->lse_out) return st;
    nl = 0;
    e = pf::launch_lse64(key, N, opts->lse_out, s, &nl);
    g_launches += nl;
    return cuda_status(e);
}

}  // namespace

namespace pf {
ProfScope::ProfScope(const char* name, cudaStream_t s, uint64_t alg_bytes, uint64_t row_bytes) : slot(-1), stream(s) {
    if (!g_prof_on.load(std::memory_order_relaxed)) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    ProfRecord r{name, prof_event(), prof_event(), alg_bytes, row_bytes};
    cudaEventRecord(r.start, s);
    prof_records().push_back(r);
    slot = static_cast<int>(prof_records().size()) - 1;
}
ProfScope::~ProfScope() {
    if (slot < 0) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEventRecord(prof_records()[slot].stop, stream);
}
}  // namespace pf

extern "C" {

void pf_profile_enable(int32_t on) { g_prof_on.store(on != 0); }

void pf_set_fusion(int32_t on) { g_no_fusion.store(on == 0); }

int32_t pf_profile_collect(pf_kernel_time* out, int32_t max_entries) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    struct Agg {
        std::string name;
        uint64_t launches;
        double ms;
        uint64_t alg_bytes, row_bytes;
    };
    std::vector<Agg> agg;
    int32_t rc = 0;
    for (auto& r : prof_records()) {
        float ms = 0.0f;
        if (cudaEventSynchronize(r.stop) != cudaSuccess || cudaEventElapsedTime(&ms, r.start, r.stop) != cudaSuccess)
            rc = -1;
        bool found = false;
        for (auto& a : agg)
            if (a.name == r.name) {
                a.launches += 1;
                a.ms += ms;
                a.alg_bytes += r.alg_bytes;
                a.row_bytes += r.row_bytes;
                found = true;
            }
        if (!found) agg.push_back({r.name, 1, static_cast<double>(ms), r.alg_bytes, r.row_bytes});
        prof_free_events().push_back(r.start);
        prof_free_events().push_back(r.stop);
    }
    prof_records().clear();
    if (rc < 0) return -1;
    int32_t n = 0;
    for (auto& a : agg) {
        if (n >= max_entries) break;
        std::memset(out[n].name, 0, sizeof(out[n].name));
        std::strncpy(out[n].name, a.name.c_str(), sizeof(out[n].name) - 1);
        out[n].launches = a.launches;
        out[n].total_ms = a.ms;
        out[n].alg_bytes = a.alg_bytes;
        out[n].row_bytes = a.row_bytes;
        ++n;
    }
    return static_cast<int32_t>(agg.size());
}


pf_status pf_resample_ex(pf_scheme scheme, const float* logw, int32_t P, uint64_t seed, int32_t B,
                         int32_t* ancestors, const pf_opts* opts, pf_stream_t stream) {
    const uint32_t f = opts ? opts->filter_index : 0u;
    return resample_impl(scheme, logw, P, 1, P, seed, f, B, ancestors, P, opts, static_cast<cudaStream_t>(stream));
}

pf_status pf_resample_multinomial(const float* logw, int32_t P, uint64_t seed, int32_t B, int32_t* ancestors,
                                  pf_stream_t stream) {
    return pf_resample_ex(PF_MULTINOMIAL, logw, P, seed, B, ancestors, nullptr, stream);
}
pf_status pf_resample_stratified(const float* logw, int32_t P, uint64_t seed, int32_t B, int32_t* ancestors,
                                 pf_stream_t stream) {
    return pf_resample_ex(PF_STRATIFIED, logw, P, seed, B, ancestors, nullptr, stream);
}
pf_status pf_resample_systematic(const float* logw, int32_t P, uint64_t seed, int32_t B, int32_t* ancestors,
                                 pf_stream_t stream) {
    return pf_resample_ex(PF_SYSTEMATIC, logw, P, seed, B, ancestors, nullptr, stream);
}
pf_status pf_resample_metropolis(const float* logw, int32_t P, uint64_t seed, int32_t B, int32_t* ancestors,
                                 pf_stream_t stream) {
    return pf_resample_ex(PF_METROPOLIS, logw, P, seed, B, ancestors, nullptr, stream);
}

pf_status pf_resample_batched(pf_scheme scheme, const float* logw, int64_t ld_logw, int32_t N, int32_t P,
                              uint64_t seed, uint32_t first_filter, int32_t B, int32_t* ancestors, int64_t ld_anc,
                              const pf_opts* opts, pf_stream_t stream) {
    return resample_impl(scheme, logw, ld_logw, N, P, seed, first_filter, B, ancestors, ld_anc, opts,
                         static_cast<cudaStream_t>(stream));
}

pf_status pf_resample_ex_f64(pf_scheme scheme, const double* logw, int32_t P, uint64_t seed, int32_t B,
                             int32_t* ancestors, const pf_opts* opts, pf_stream_t stream) {
    const uint32_t f = opts ? opts->filter_index : 0u;
    return resample_f64_impl(scheme, logw, P, 1, P, seed, f, B, ancestors, P, opts, static_cast<cudaStream_t>(stream));
}

pf_status pf_resample_batched_f64(pf_scheme scheme, const double* logw, int64_t ld_logw, int32_t N, int32_t P,
                                  uint64_t seed, uint32_t first_filter, int32_t B, int32_t* ancestors, int64_t ld_anc,
                                  const pf_opts* opts, pf_stream_t stream) {
    return resample_f64_impl(scheme, logw, ld_logw, N, P, seed, first_filter, B, ancestors, ld_anc, opts,
                             static_cast<cudaStream_t>(stream));
}

size_t pf_workspace_bytes_ex(pf_scheme scheme, int32_t N, int32_t P, uint32_t flags, int64_t ld_anc) {
    if (N < 1 || P < 1 || ld_anc < P || scheme < PF_MULTINOMIAL || scheme > PF_METROPOLIS) return 0;
    const bool sorted_multi = (flags & PF_SORTED) && scheme == PF_MULTINOMIAL;
    // the largest need over the paths a call with these arguments may take: the multi-launch
    // layout, the cooperative kernel's scratch, and the permutation the cluster kernel writes
    // when the state is gathered without permuted_out
    size_t need = pf::make_layout(N, P, needs_for(scheme) | (sorted_multi ? pf::kNeedG : 0u)).total;
    const size_t plane = (static_cast<size_t>(N) * static_cast<size_t>(ld_anc) * 4 + 255) / 256 * 256;
    need = std::max(need, (pf::coop_scratch_bytes(P) + 255) / 256 * 256 + 2 * plane);
    return need;
}

size_t pf_workspace_bytes(pf_scheme scheme, int32_t N, int32_t P) {
    return pf_workspace_bytes_ex(scheme, N, P, 0u, P);
}

pf_status pf_ancestors_to_offspring_batched(const int32_t* anc, int64_t ld_anc, int32_t N, int32_t P,
                                            int32_t* offspring, int64_t ld_off, pf_stream_t stream) {
    if (!anc || !offspring || N < 1 || P < 1 || ld_anc < P || ld_off < P) return PF_ERR_INVALID_ARG;
    uint64_t nl = 0;
    const cudaError_t e =
        pf::launch_offspring(anc, ld_anc, N, P, offspring, ld_off, static_cast<cudaStream_t>(stream), &nl);
    g_launches += nl;
    return cuda_status(e);
}

pf_status pf_ancestors_to_offspring(const int32_t* anc, int32_t P, int32_t* offspring, pf_stream_t stream) {
    return pf_ancestors_to_offspring_batched(anc, P, 1, P, offspring, P, stream);
}

pf_status pf_permute_batched(const int32_t* anc, int64_t ld_anc, int32_t N, int32_t P, int32_t* permuted,
                             int64_t ld_perm, pf_stream_t stream) {
    if (!anc || !permuted || N < 1 || P < 1 || ld_anc < P || ld_perm < P) return PF_ERR_INVALID_ARG;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const pf::Layout L = pf::make_layout(N, P, pf::kNeedPermute);
    void* base = nullptr;
    pf_status st = pool_get(L.total, s, &base);
    if (st != PF_OK) return st;
    const pf::Ws ws = pf::carve(base, L);
    uint64_t nl = 0;
    if (fused_permute_preferred(N, P)) {
        // offspring histogram into the workspace, then the cluster kernel's phase D on it
        cudaError_t e = pf::launch_offspring(anc, ld_anc, N, P, ws.o, L.ldq, s, &nl);
        if (e == cudaSuccess)
            e = pf::launch_fused_from_offspring(ws.o, L.ldq, N, P, permuted, ld_perm, nullptr, 0, 0, 0, s, &nl);
        g_launches += nl;
        return cuda_status(e);
    }
    cudaError_t e = cudaMemsetAsync(static_cast<char*>(base) + L.zero_begin, 0, L.zero_end - L.zero_begin, s);
    if (e == cudaSuccess) e = pf::launch_permute(anc, ld_anc, N, P, L, ws, permuted, ld_perm, s, &nl);
    g_launches += nl;
    return cuda_status(e);
}

pf_status pf_permute_offspring_batched(const int32_t* offspring, int64_t ld_off, int32_t N, int32_t P,
                                       int32_t* permuted, int64_t ld_perm, pf_stream_t stream) {
    if (!offspring || !permuted || N < 1 || P < 1 || ld_off < P || ld_perm < P) return PF_ERR_INVALID_ARG;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const pf::Layout L = pf::make_layout(N, P, pf::kNeedPermute);
    void* base = nullptr;
    pf_status st = pool_get(L.total, s, &base);
    if (st != PF_OK) return st;
    const pf::Ws ws = pf::carve(base, L);
    uint64_t nl = 0;
    if (fused_permute_preferred(N, P)) {
        const cudaError_t e =
            pf::launch_fused_from_offspring(offspring, ld_off, N, P, permuted, ld_perm, nullptr, 0, 0, 0, s, &nl);
        g_launches += nl;
        return cuda_status(e);
    }
    cudaError_t e = cudaMemsetAsync(static_cast<char*>(base) + L.zero_begin, 0, L.zero_end - L.zero_begin, s);
    if (e == cudaSuccess)
        e = pf::launch_permute_from_offspring(offspring, ld_off, N, P, L, ws, permuted, ld_perm, s, &nl);
    g_launches += nl;
    return cuda_status(e);
}

pf_status pf_permute_offspring(const int32_t* offspring, int32_t P, int32_t* permuted, pf_stream_t stream) {
    return pf_permute_offspring_batched(offspring, P, 1, P, permuted, P, stream);
}

pf_status pf_permute(const int32_t* anc, int32_t P, int32_t* permuted, pf_stream_t stream) {
    return pf_permute_batched(anc, P, 1, P, permuted, P, stream);
}

pf_status pf_gather_state_batched(void* X, int64_t row_bytes, int64_t ld_bytes, int64_t ld_filter_bytes, int32_t N,
                                  int32_t P, const int32_t* permuted, int64_t ld_perm, pf_stream_t stream) {
    if (!X || !permuted || N < 1 || P < 1 || row_bytes < 1 || ld_bytes < row_bytes || ld_perm < P)
        return PF_ERR_INVALID_ARG;
    if (N > 1 && ld_filter_bytes < ld_bytes * P) return PF_ERR_INVALID_ARG;
    uint64_t nl = 0;
    const cudaError_t e = pf::launch_gather_inplace(X, row_bytes, ld_bytes, ld_filter_bytes, N, P, permuted, ld_perm,
                                                    static_cast<cudaStream_t>(stream), &nl);
    g_launches += nl;
    return cuda_status(e);
}

pf_status pf_gather_state(void* X, int64_t row_bytes, int64_t ld_bytes, int32_t P, const int32_t* permuted,
                          pf_stream_t stream) {
    return pf_gather_state_batched(X, row_bytes, ld_bytes, ld_bytes * P, 1, P, permuted, P, stream);
}

pf_status pf_gather_state_out(const void* X, void* Y, int64_t row_bytes, int64_t ld_x, int64_t ld_y, int32_t P,
                              const int32_t* anc, pf_stream_t stream) {
    if (!X || !Y || !anc || P < 1 || row_bytes < 1 || ld_x < row_bytes || ld_y < row_bytes)
        return PF_ERR_INVALID_ARG;
    uint64_t nl = 0;
    const cudaError_t e =
        pf::launch_gather_out(X, Y, row_bytes, ld_x, ld_y, P, anc, static_cast<cudaStream_t>(stream), &nl);
    g_launches += nl;
    return cuda_status(e);
}

// ---------------------------------------------------------------- giant-filter shards
pf_status pf_shard_max(const float* logw, int32_t Pl, float* d_lmax, int32_t* d_bad, pf_stream_t stream) {
    if (!logw || !d_lmax || !d_bad || Pl < 1) return PF_ERR_INVALID_ARG;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const pf::Layout L = pf::make_layout(1, Pl, 0u);
    void* base = nullptr;
    pf_status st = pool_get(L.total, s, &base);
    if (st != PF_OK) return st;
    const pf::Ws ws = pf::carve(base, L);
    uint64_t nl = 0;
    cudaError_t e = cudaMemsetAsync(static_cast<char*>(base) + L.zero_begin, 0, L.zero_end - L.zero_begin, s);
    if (e == cudaSuccess) e = pf::launch_max(logw, Pl, 1, Pl, L, ws, nullptr, s, &nl, d_lmax, d_bad);
    g_launches += nl;
    return cuda_status(e);
}

pf_status pf_shard_scan(const float* logw, int32_t Pl, int64_t P_global, const float* d_gmax, uint64_t* d_Q,
                        uint64_t* d_total, double* d_wsum, pf_stream_t stream) {
    if (!logw || !d_gmax || !d_Q || !d_total || Pl < 1 || P_global < Pl || P_global > INT32_MAX)
        return PF_ERR_INVALID_ARG;
    if ((reinterpret_cast<uintptr_t>(d_Q) & 15) != 0) return PF_ERR_INVALID_ARG;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const pf::Layout L = pf::make_layout(1, Pl, 0u);
    void* base = nullptr;
    pf_status st = pool_get(L.total, s, &base);
    if (st != PF_OK) return st;
    pf::Ws ws = pf::carve(base, L);
    ws.Q = d_Q;
    uint64_t nl = 0;
    cudaError_t e = cudaMemsetAsync(static_cast<char*>(base) + L.zero_begin, 0, L.zero_end - L.zero_begin, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(ws.fstatus, 0, sizeof(int32_t), s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(ws.lmax, d_gmax, sizeof(float), cudaMemcpyDeviceToDevice, s);
    const int kfx = 61 - pf::ceil_log2(P_global);
    if (e == cudaSuccess) e = pf::launch_scan(logw, Pl, 1, Pl, L, ws, true, nullptr, nullptr, s, &nl, kfx);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_total, ws.Qtot, sizeof(uint64_t), cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess && d_wsum) e = cudaMemcpyAsync(d_wsum, ws.S, sizeof(double), cudaMemcpyDeviceToDevice, s);
    g_launches += nl;
    return cuda_status(e);
}

pf_status pf_shard_search(pf_scheme scheme, const uint64_t* d_Q, int32_t Pl, int64_t p0, int64_t P_global,
                          const uint64_t* d_totals, int32_t nshards, int32_t shard, const float* d_gmax,
                          const int32_t* d_gbad, uint64_t seed, uint32_t filter_index, int32_t* anc_out,
                          int64_t* d_slot_range, pf_stream_t stream) {
    if (!d_Q || !d_totals || !d_gmax || !d_gbad || !anc_out || !d_slot_range) return PF_ERR_INVALID_ARG;
    if (scheme < PF_MULTINOMIAL || scheme > PF_SYSTEMATIC) return PF_ERR_UNSUPPORTED;
    if (Pl < 1 || p0 < 0 || P_global < p0 + Pl || P_global > INT32_MAX || nshards < 1 || shard < 0 ||
        shard >= nshards)
        return PF_ERR_INVALID_ARG;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    void* ctx = nullptr;
    pf_status st = pool_get(pf::shard_ctx_bytes(), s, &ctx);
    if (st != PF_OK) return st;
    uint64_t nl = 0;
    const cudaError_t e = pf::launch_shard_search(scheme, d_Q, Pl, p0, P_global, d_totals, nshards, shard, d_gmax,
                                                  d_gbad, seed, filter_index, anc_out, d_slot_range, ctx, s, &nl);
    g_launches += nl;
    return cuda_status(e);
}

pf_status pf_shard_route_count(const uint64_t* d_totals, int32_t nshards, int32_t shard, int64_t P_global,
                               const float* d_gmax, const int32_t* d_gbad, uint64_t seed, uint32_t filter_index,
                               int64_t* d_counts, pf_stream_t stream) {
    if (!d_totals || !d_gmax || !d_gbad || !d_counts) return PF_ERR_INVALID_ARG;
    if (P_global < 1 || P_global > INT32_MAX || nshards < 1 || nshards > pf::kMaxRouteShards || shard < 0 ||
        shard >= nshards)
        return PF_ERR_INVALID_ARG;
    uint64_t nl = 0;
    const cudaError_t e = pf::launch_route(d_totals, nshards, shard, d_gmax, d_gbad, P_global, seed, filter_index,
                                           d_counts, nullptr, nullptr, nullptr, static_cast<cudaStream_t>(stream), &nl);
    g_launches += nl;
    return cuda_status(e);
}

pf_status pf_shard_route_pack(const uint64_t* d_totals, int32_t nshards, int32_t shard, int64_t P_global,
                              const float* d_gmax, const int32_t* d_gbad, uint64_t seed, uint32_t filter_index,
                              const int64_t* d_counts, uint64_t* send_x, int32_t* send_k, pf_stream_t stream) {
    if (!d_totals || !d_gmax || !d_gbad || !d_counts || !send_x || !send_k) return PF_ERR_INVALID_ARG;
    if (P_global < 1 || P_global > INT32_MAX || nshards < 1 || nshards > pf::kMaxRouteShards || shard < 0 ||
        shard >= nshards)
        return PF_ERR_INVALID_ARG;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    void* cur = nullptr;
    const pf_status st = pool_get(sizeof(int64_t) * pf::kMaxRouteShards, s, &cur);
    if (st != PF_OK) return st;
    uint64_t nl = 0;
    const cudaError_t e = pf::launch_route(d_totals, nshards, shard, d_gmax, d_gbad, P_global, seed, filter_index,
                                           const_cast<int64_t*>(d_counts), static_cast<int64_t*>(cur), send_x, send_k,
                                           s, &nl);
    g_launches += nl;
    return cuda_status(e);
}

pf_status pf_shard_route_search(const uint64_t* d_Q, int32_t Pl, int64_t p0, int64_t P_global,
                                const uint64_t* d_totals, int32_t nshards, int32_t shard, const float* d_gmax,
                                const int32_t* d_gbad, const uint64_t* recv_x, const int32_t* recv_k, int64_t nrecv,
                                int32_t* anc_out, pf_stream_t stream) {
    if (!d_Q || !d_totals || !d_gmax || !d_gbad || !anc_out || nrecv < 0 || (nrecv > 0 && (!recv_x || !recv_k)))
        return PF_ERR_INVALID_ARG;
    if (Pl < 1 || p0 < 0 || P_global < p0 + Pl || P_global > INT32_MAX || nshards < 1 ||
        nshards > pf::kMaxRouteShards || shard < 0 || shard >= nshards)
        return PF_ERR_INVALID_ARG;
    uint64_t nl = 0;
    const cudaError_t e = pf::launch_route_search(d_Q, Pl, p0, d_totals, nshards, shard, d_gmax, d_gbad, recv_x, recv_k,
                                                  nrecv, anc_out, static_cast<cudaStream_t>(stream), &nl);
    g_launches += nl;
    return cuda_status(e);
}

pf_status pf_shard_spacings_total(int64_t P_global, int32_t nshards, int32_t shard, uint64_t seed,
                                  uint32_t filter_index, uint64_t* d_etotal, pf_stream_t stream) {
    if (!d_etotal || P_global < 1 || P_global > INT32_MAX || nshards < 1 || shard < 0 || shard >= nshards)
        return PF_ERR_INVALID_ARG;
    uint64_t nl = 0;
    const cudaError_t e = pf::launch_spacings_total(P_global, nshards, shard, seed, filter_index, d_etotal,
                                                    static_cast<cudaStream_t>(stream), &nl);
    g_launches += nl;
    return cuda_status(e);
}

size_t pf_shard_search_sorted_workspace_bytes(int64_t P_global) {
    if (P_global < 1 || P_global > INT32_MAX) return 0;
    return pf::spac_shard_workspace_bytes(P_global);
}

pf_status pf_shard_search_sorted(const uint64_t* d_Q, int32_t Pl, int64_t p0, int64_t P_global,
                                 const uint64_t* d_totals, const uint64_t* d_etotals, int32_t nshards, int32_t shard,
                                 const float* d_gmax, const int32_t* d_gbad, uint64_t seed, uint32_t filter_index,
                                 int32_t* anc_out, int64_t* d_slot_range, void* workspace, size_t workspace_bytes,
                                 pf_stream_t stream) {
    if (!d_Q || !d_totals || !d_etotals || !d_gmax || !d_gbad || !anc_out || !d_slot_range)
        return PF_ERR_INVALID_ARG;
    if (Pl < 1 || p0 < 0 || P_global < p0 + Pl || P_global > INT32_MAX || nshards < 1 || shard < 0 ||
        shard >= nshards)
        return PF_ERR_INVALID_ARG;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t need = pf::spac_shard_workspace_bytes(P_global);
    void* ws = workspace;
    if (ws) {
        if (workspace_bytes < need || (reinterpret_cast<uintptr_t>(ws) & 255) != 0) return PF_ERR_WORKSPACE;
    } else {
        const pf_status st = pool_get(need, s, &ws);
        if (st != PF_OK) return st;
    }
    uint64_t nl = 0;
    const cudaError_t e = pf::launch_shard_search_sorted(d_Q, Pl, p0, P_global, d_totals, d_etotals, nshards, shard,
                                                         d_gmax, d_gbad, seed, filter_index, anc_out, d_slot_range,
                                                         ws, s, &nl);
    g_launches += nl;
    return cuda_status(e);
}

pf_status pf_shard_weights(const float* logw, int32_t Pl, const float* d_gmax, float* w_out, pf_stream_t stream) {
    if (!logw || !d_gmax || !w_out || Pl < 1) return PF_ERR_INVALID_ARG;
    uint64_t nl = 0;
    const cudaError_t e = pf::launch_shard_weights(logw, Pl, d_gmax, w_out, static_cast<cudaStream_t>(stream), &nl);
    g_launches += nl;
    return cuda_status(e);
}

pf_status pf_metropolis_from_weights(const float* w_full, int64_t P_global, int64_t slot0, int32_t nslots,
                                     uint64_t seed, int32_t B, uint32_t filter_index, const float* d_gmax,
                                     const int32_t* d_gbad, int32_t* anc, pf_stream_t stream) {
    if (!w_full || !anc || P_global < 1 || P_global > INT32_MAX || slot0 < 0 || nslots < 0 ||
        slot0 + nslots > P_global || B < 0)
        return PF_ERR_INVALID_ARG;
    if (nslots == 0) return PF_OK;
    uint64_t nl = 0;
    const cudaError_t e = pf::launch_metro_slots(w_full, P_global, slot0, nslots, seed, B, filter_index, d_gmax,
                                                 d_gbad, anc, static_cast<cudaStream_t>(stream), &nl);
    g_launches += nl;
    return cuda_status(e);
}

// ---------------------------------------------------------------- particle migration (4a-4d)
pf_status pf_shard_offspring(const int32_t* anc, int64_t n_anc, const int64_t* d_slot_range, int64_t win0,
                             int32_t Pw, const float* d_gmax, const int32_t* d_gbad, int32_t* offspring,
                             pf_stream_t stream) {
    if (!offspring || Pw < 1 || n_anc < 0 || (n_anc > 0 && !anc) || win0 < 0 || (!d_gmax) != (!d_gbad))
        return PF_ERR_INVALID_ARG;
    uint64_t nl = 0;
    const cudaError_t e = pf::launch_mig_offspring(anc, n_anc, d_slot_range, win0, Pw, d_gmax, d_gbad, offspring,
                                                   static_cast<cudaStream_t>(stream), &nl);
    g_launches += nl;
    return cuda_status(e);
}

size_t pf_shard_migration_plan_bytes(int32_t Pl) { return Pl < 1 ? 0 : pf::mig_plan_bytes(Pl); }

pf_status pf_shard_migration_counts(const int32_t* offspring, int32_t Pl, void* plan, int64_t* d_counts,
                                    pf_stream_t stream) {
    if (!offspring || !plan || !d_counts || Pl < 1 || (reinterpret_cast<uintptr_t>(plan) & 7) != 0)
        return PF_ERR_INVALID_ARG;
    uint64_t nl = 0;
    const cudaError_t e =
        pf::launch_mig_plan(offspring, Pl, plan, d_counts, static_cast<cudaStream_t>(stream), &nl);
    g_launches += nl;
    return cuda_status(e);
}

pf_status pf_shard_migrate_pack(const void* X, int64_t row_bytes, int64_t ld_bytes, int32_t Pl, int64_t p0,
                                const int32_t* offspring, const void* plan, void* send_rows, int32_t* send_src,
                                pf_stream_t stream) {
    if (!offspring || !plan || Pl < 1 || p0 < 0 || p0 + Pl > INT32_MAX || row_bytes < 0 ||
        (row_bytes > 0 && (!X || !send_rows || ld_bytes < row_bytes)) || (row_bytes == 0 && !send_src))
        return PF_ERR_INVALID_ARG;
    uint64_t nl = 0;
    const cudaError_t e = pf::launch_mig_pack(X, row_bytes, ld_bytes, Pl, p0, offspring, plan, send_rows, send_src,
                                              static_cast<cudaStream_t>(stream), &nl);
    g_launches += nl;
    return cuda_status(e);
}

pf_status pf_shard_migrate_unpack(void* X, int64_t row_bytes, int64_t ld_bytes, int32_t Pl, int64_t p0,
                                  const int32_t* offspring, const void* plan, const void* recv_rows,
                                  const int32_t* recv_src, int32_t* perm_out, pf_stream_t stream) {
    if (!offspring || !plan || Pl < 1 || p0 < 0 || p0 + Pl > INT32_MAX || row_bytes < 0 ||
        (row_bytes > 0 && (!X || ld_bytes < row_bytes)) || (row_bytes == 0 && !perm_out))
        return PF_ERR_INVALID_ARG;
    uint64_t nl = 0;
    const cudaError_t e = pf::launch_mig_unpack(X, row_bytes, ld_bytes, Pl, p0, offspring, plan, recv_rows, recv_src,
                                                perm_out, static_cast<cudaStream_t>(stream), &nl);
    g_launches += nl;
    return cuda_status(e);
}

// ---------------------------------------------------------------- C4 demo model
pf_status pf_lg_init(float* X, int64_t ld, int32_t P, int32_t D, float phi, float sigma_x, uint64_t seed,
                     pf_stream_t stream) {
    if (!X || P < 1 || D < 1 || ld < D || !(phi * phi < 1.0f) || !(sigma_x >= 0.0f)) return PF_ERR_INVALID_ARG;
    uint64_t nl = 0;
    const cudaError_t e = pf::launch_lg_init(X, ld, P, D, phi, sigma_x, seed, static_cast<cudaStream_t>(stream), &nl);
    g_launches += nl;
    return cuda_status(e);
}

pf_status pf_lg_propagate_weight(float* X, int64_t ld, int32_t P, int32_t D, float phi, float sigma_x,
                                 float sigma_y, float y, uint64_t seed, int32_t t, float* logw, pf_stream_t stream) {
    if (!X || !logw || P < 1 || D < 1 || ld < D || !(sigma_y > 0.0f) || t < 0) return PF_ERR_INVALID_ARG;
    uint64_t nl = 0;
    const cudaError_t e = pf::launch_lg_step(X, ld, P, D, phi, sigma_x, sigma_y, y, seed, t, logw,
                                             static_cast<cudaStream_t>(stream), &nl);
    g_launches += nl;
    return cuda_status(e);
}

pf_status pf_lg_accumulate(const double* lse, int32_t P, float sigma_y, double* loglik, pf_stream_t stream) {
    if (!lse || !loglik || P < 1 || !(sigma_y > 0.0f)) return PF_ERR_INVALID_ARG;
    uint64_t nl = 0;
    const cudaError_t e = pf::launch_lg_accumulate(lse, P, sigma_y, loglik, static_cast<cudaStream_t>(stream), &nl);
    g_launches += nl;
    return cuda_status(e);
}

int32_t pf_metropolis_required_B(int64_t P, double w_max, double eps) {
    if (P < 1 || !(w_max > 0.0) || w_max > 1.0 || !(eps > 0.0)) return -1;
    // w_max >= 1/P: the maximum of P normalised weights (outside Eq. (2)'s domain otherwise)
    if (w_max * static_cast<double>(P) < 1.0 - 1e-12) return -1;
    const double beta = 1.0 / static_cast<double>(P);
    const double alpha = (1.0 - w_max) / (static_cast<double>(P) * w_max);    // Eq. (2)
    const double lambda = 1.0 - alpha - beta;
    const double bound = eps * (alpha + beta) / (alpha > beta ? alpha : beta);  // Eq. (4)
    if (bound >= 1.0 || lambda <= 0.0) return 1;  // at least one step (DESIGN R-22)
    const double B = std::ceil(std::log(bound) / std::log(lambda));           // Eq. (5)
    if (B > 2147483647.0) return -1;  // not representable (e.g. w_max -> 1 at P = 2^28)
    return B < 1.0 ? 1 : static_cast<int32_t>(B);
}

const char* pf_status_string(pf_status s) {
    switch (s) {
        case PF_OK: return "PF_OK";
        case PF_ERR_INVALID_ARG: return "PF_ERR_INVALID_ARG";
        case PF_ERR_WORKSPACE: return "PF_ERR_WORKSPACE";
        case PF_ERR_CUDA: return "PF_ERR_CUDA";
        case PF_ERR_UNSUPPORTED: return "PF_ERR_UNSUPPORTED";
    }
    return "PF_ERR_UNKNOWN";
}

uint64_t pf_launch_count(void) { return g_launches.load(); }

const char* pf_version(void) { return "libpfresample 0.1 (sm_100a)"; }

void pf_release(void) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    for (auto& kv : pool()) {
        if (kv.second.ptr) cudaFree(kv.second.ptr);
    }
    pool().clear();
}

}  // extern "C"
