// pf_internal.h — internal launcher interface between the C ABI (pf_api.cu)
// and the kernels (pf_kernels.cu).  Not installed; no torch types.
#pragma once
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace pf {

// Per-device cache of launch-geometry constants (SM count, occupancy): thread-safe (relaxed
// atomics; a racing first use computes the same value twice) and correct for processes that
// drive several devices.
constexpr int kMaxDevices = 64;
inline int current_device() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) {
        cudaGetLastError();
        d = 0;
    }
    return (d >= 0 && d < kMaxDevices) ? d : 0;
}
template <class F>
inline int cached_per_device(std::atomic<int>* slots, F&& compute) {
    std::atomic<int>& slot = slots[current_device()];
    int v = slot.load(std::memory_order_relaxed);
    if (v == 0) {
        v = compute();
        slot.store(v, std::memory_order_relaxed);
    }
    return v;
}
int sm_count();  // SMs of the current device

constexpr int kThreads = 256;           // every kernel: 8 warps
constexpr int kItems = 16;              // items per thread in scan / merge tiles
constexpr int kTile = kThreads * kItems;  // 4096 particles per scan tile

// Per-kernel event tracing (pf_profile_enable); a no-op unless enabled.
// alg_bytes: the launch's algorithmic HBM bytes known at launch (inputs read once, outputs
// written once); row_bytes: the extra algorithmic bytes per moved state row (data-dependent:
// the caller multiplies by the rows its gather moved).  Both are reported per kernel name by
// pf_profile_collect, so a roofline is computed from what each launch actually moved.
struct ProfScope {
    ProfScope(const char* name, cudaStream_t s, uint64_t alg_bytes = 0, uint64_t row_bytes = 0);
    ~ProfScope();
    int slot;
    cudaStream_t stream;
};

// Per-call device workspace (carved from the pool or a caller buffer).
struct Ws {
    float* lmax;         // [N]
    int32_t* fstatus;    // [N]
    float* max_part;     // [N*cpf]
    int32_t* max_bad;    // [N*cpf]
    uint32_t* max_cnt;   // [N]       zeroed per call
    uint32_t* tile_ctr;  // [1]       zeroed per call
    uint64_t* tstatus;   // [N*T]     zeroed per call
    double* tsum;        // [N*T]
    double* tsum2;       // [N*T]
    uint64_t* Q;         // [N*ldq]   inclusive fixed-point scan
    uint64_t* Qtot;      // [N]
    double* S;           // [N]       sum of w (double)
    float* w;            // [N*ldq]   Metropolis weights
    int32_t* o;          // [N*ldq]   permute: offspring
    uint32_t* Qe;        // [N*ldq]   permute: inclusive extras count
    int32_t* freeslot;   // [N*ldq]   permute: r-th free slot
    int32_t* F;          // [N]       permute: number of free slots
    uint32_t* tile_ctr2; // [1]       zeroed per call (spacings scan)
    uint64_t* tstatus2;  // [N*T2]    zeroed per call
    uint64_t* G;         // [N*ldg]   a6: inclusive spacings sums G_0..G_P
    uint64_t* Gtot;      // [N]       a6: G_P
    int32_t* bidx;       // [N*ldb]   multinomial bucket index idx[b] = min{i : Q_i > floor(b Q / NB)}
};

struct Layout {
    size_t lmax, fstatus, max_part, max_bad, zero_begin, max_cnt, tile_ctr, tstatus, zero_end;
    size_t tsum, tsum2, Q, Qtot, S, w, o, Qe, freeslot, F, tile_ctr2, tstatus2, G, Gtot, bidx, total;
    int64_t ldb;  // bucket-index row length NB = 2^ceil(log2 P)
    int cpf_max;  // CTAs per filter of k_max
    int T;        // scan tiles per filter
    int T2;       // spacings-scan tiles per filter (P + 1 values)
    int64_t ldq;  // padded row length (multiple of 4)
    int64_t ldg;  // padded spacings row length (P + 1 rounded to 4)
};

enum Need : unsigned { kNeedQ = 1u, kNeedW = 2u, kNeedPermute = 4u, kNeedG = 8u, kNeedBuckets = 16u };

Layout make_layout(int32_t N, int32_t P, unsigned need);
Ws carve(void* base, const Layout& L);

// Launchers: enqueue on `s`; return cudaPeekAtLastError().  `launches` is
// incremented by the number of kernels enqueued.
cudaError_t launch_max(const float* logw, int64_t ld, int32_t N, int32_t P, const Layout& L, const Ws& ws,
                       int32_t* status_out, cudaStream_t s, uint64_t* launches, float* lmax_out = nullptr,
                       int32_t* bad_out = nullptr);
cudaError_t launch_scan(const float* logw, int64_t ld, int32_t N, int32_t P, const Layout& L, const Ws& ws,
                        bool write_q, double* lse_out, double* ess_out, cudaStream_t s, uint64_t* launches,
                        int kfx_override = -1);
cudaError_t launch_search(int scheme, int32_t N, int32_t P, const Layout& L, const Ws& ws, uint64_t seed,
                          uint32_t first_filter, int32_t* anc, int64_t ld_anc, cudaStream_t s,
                          uint64_t* launches);
cudaError_t launch_sorted_multinomial(int32_t N, int32_t P, const Layout& L, const Ws& ws, uint64_t seed,
                                      uint32_t first_filter, int32_t* anc, int64_t ld_anc, cudaStream_t s,
                                      uint64_t* launches, bool spacings_only);
cudaError_t launch_metropolis(const float* logw, int64_t ld, int32_t N, int32_t P, const Layout& L,
                              const Ws& ws, uint64_t seed, uint32_t first_filter, int32_t B, int32_t* anc,
                              int64_t ld_anc, cudaStream_t s, uint64_t* launches);
cudaError_t launch_normw(const float* logw, int64_t ld, int32_t N, int32_t P, const Ws& ws, float* normw,
                         cudaStream_t s, uint64_t* launches);
cudaError_t launch_identity(int32_t N, int32_t P, int32_t* anc, int64_t ld_anc, cudaStream_t s,
                            uint64_t* launches);
cudaError_t launch_offspring(const int32_t* anc, int64_t ld_anc, int32_t N, int32_t P, int32_t* o, int64_t ld_o,
                             cudaStream_t s, uint64_t* launches);
cudaError_t launch_permute(const int32_t* anc, int64_t ld_anc, int32_t N, int32_t P, const Layout& L,
                           const Ws& ws, int32_t* perm, int64_t ld_perm, cudaStream_t s, uint64_t* launches);
cudaError_t launch_permute_from_offspring(const int32_t* o, int64_t ld_o, int32_t N, int32_t P, const Layout& L,
                                         const Ws& ws, int32_t* perm, int64_t ld_perm, cudaStream_t s,
                                         uint64_t* launches);
cudaError_t launch_gather_inplace(void* X, int64_t row_bytes, int64_t ld_bytes, int64_t ld_filter_bytes, int32_t N,
                                  int32_t P, const int32_t* perm, int64_t ld_perm, cudaStream_t s,
                                  uint64_t* launches);
cudaError_t launch_gather_out(const void* X, void* Y, int64_t row_bytes, int64_t ld_x, int64_t ld_y, int32_t P,
                              const int32_t* anc, cudaStream_t s, uint64_t* launches);

// Giant-filter shard stages (C5).
cudaError_t launch_shard_search(int scheme, const uint64_t* Q, int32_t Pl, int64_t p0, int64_t P_global,
                                const uint64_t* totals, int nshards, int shard, const float* gmax,
                                const int32_t* gbad, uint64_t seed, uint32_t filt, int32_t* anc,
                                int64_t* range_out, void* ctx_mem, cudaStream_t s, uint64_t* launches);
cudaError_t launch_shard_weights(const float* logw, int32_t Pl, const float* gmax, float* w, cudaStream_t s,
                                 uint64_t* launches);
cudaError_t launch_metro_slots(const float* w, int64_t P_global, int64_t slot0, int32_t nslots, uint64_t seed,
                               int32_t B, uint32_t filt, const float* gmax, const int32_t* gbad, int32_t* anc,
                               cudaStream_t s, uint64_t* launches);
constexpr int kMaxRouteShards = 64;  // ranks of a routed multinomial (one node and beyond)
cudaError_t launch_route(const uint64_t* totals, int nshards, int shard, const float* gmax, const int32_t* gbad,
                         int64_t P_global, uint64_t seed, uint32_t filt, int64_t* counts, int64_t* cursor,
                         uint64_t* send_x, int32_t* send_k, cudaStream_t s, uint64_t* launches);
cudaError_t launch_route_search(const uint64_t* Q, int32_t Pl, int64_t p0, const uint64_t* totals, int nshards,
                                int shard, const float* gmax, const int32_t* gbad, const uint64_t* rx,
                                const int32_t* rk, int64_t nrecv, int32_t* anc, cudaStream_t s, uint64_t* launches);
size_t shard_ctx_bytes();
// a6 (sorted multinomial) shards.
cudaError_t launch_spacings_total(int64_t P_global, int nshards, int shard, uint64_t seed, uint32_t filt,
                                  uint64_t* etot, cudaStream_t s, uint64_t* launches);
size_t spac_shard_workspace_bytes(int64_t P_global);
cudaError_t launch_shard_search_sorted(const uint64_t* Q, int32_t Pl, int64_t p0, int64_t P_global,
                                       const uint64_t* totals, const uint64_t* etotals, int nshards, int shard,
                                       const float* gmax, const int32_t* gbad, uint64_t seed, uint32_t filt,
                                       int32_t* anc, int64_t* range_out, void* ws, cudaStream_t s,
                                       uint64_t* launches);

// C4 demo model (linear-Gaussian bootstrap filter).
cudaError_t launch_lg_init(float* X, int64_t ld, int32_t P, int32_t D, float phi, float sigma_x, uint64_t seed,
                           cudaStream_t s, uint64_t* launches);
cudaError_t launch_lg_step(float* X, int64_t ld, int32_t P, int32_t D, float phi, float sigma_x, float sigma_y,
                           float y, uint64_t seed, int32_t t, float* logw, cudaStream_t s, uint64_t* launches);
cudaError_t launch_lg_accumulate(const double* lse, int32_t P, float sigma_y, double* loglik, cudaStream_t s,
                                 uint64_t* launches);

// One-launch cluster-per-filter resampler for stratified/systematic (pf_fused.cu).
bool fused_supported(int scheme, int32_t N, int32_t P);
bool fused_gather_supported(const void* X, int64_t row_bytes, int64_t ld, int64_t fld);
int fused_cluster_ctas(int32_t P);  // CTAs per filter (cluster size) of the cluster kernel
cudaError_t launch_fused_sorted(int scheme, const float* logw, int64_t ld, int32_t N, int32_t P, uint64_t seed,
                                uint32_t first_filter, int32_t* anc, int64_t ld_anc, double* lse_out,
                                double* ess_out, float* normw, int32_t* status_out, int32_t* offspring,
                                int32_t* permuted, void* X, int64_t x_row_bytes, int64_t x_ld, int64_t x_fld,
                                cudaStream_t s, uint64_t* launches, const double* logw64 = nullptr,
                                uint64_t* Qout = nullptr, int64_t ldq = 0, uint64_t* Qtot_out = nullptr);
// scheme id of launch_fused_sorted's multinomial bucket mode (Q + bucket index, pf_fused.cu)
bool fused_from_offspring_supported(int32_t P);
cudaError_t launch_fused_from_offspring(const int32_t* off, int64_t ld_off, int32_t N, int32_t P, int32_t* perm,
                                        int64_t ld_perm, void* X, int64_t x_row_bytes, int64_t x_ld, int64_t x_fld,
                                        cudaStream_t s, uint64_t* launches);
constexpr int kFusedBuckets = 5;
bool buckets_fused_supported(int32_t P);
cudaError_t launch_bsearch_buckets(int32_t N, int32_t P, const Layout& L, const Ws& ws, uint64_t seed,
                                   uint32_t first_filter, int32_t* anc, int64_t ld_anc, cudaStream_t s,
                                   uint64_t* launches);

// One-warp-per-filter kernel for P <= 256, every scheme (pf_fused.cu).
bool small_supported(int32_t P);
cudaError_t launch_small(int scheme, bool sorted, const float* logw, int64_t ld, int32_t N, int32_t P, uint64_t seed,
                         uint32_t first_filter, int32_t B, int32_t* anc, int64_t ld_anc, double* lse_out,
                         double* ess_out, float* normw, int32_t* status_out, int32_t* offspring, cudaStream_t s,
                         uint64_t* launches);

// One-CTA-per-filter kernel for 256 < P <= 8192, every scheme (pf_fused.cu).
bool medium_supported(int32_t P);
cudaError_t launch_medium(int scheme, bool sorted, const float* logw, int64_t ld, int32_t N, int32_t P, uint64_t seed,
                          uint32_t first_filter, int32_t B, int32_t* anc, int64_t ld_anc, double* lse_out,
                          double* ess_out, float* normw, int32_t* status_out, int32_t* offspring, cudaStream_t s,
                          uint64_t* launches);

// One-launch cooperative resampler for large filters (pf_fused.cu).
bool coop_supported(int scheme, int32_t N, int32_t P);
size_t coop_scratch_bytes(int32_t P);  // includes the free list of the permutation (4 P bytes)
// with permuted (and optionally X, rows gathered in place as FusedArgs) the kernel also writes
// the canonical permutation; then offspring must be non-null (scratch is fine)
cudaError_t launch_coop_sorted(int scheme, const float* logw, int64_t ld, int32_t N, int32_t P, uint64_t seed,
                               uint32_t first_filter, int32_t* anc, int64_t ld_anc, double* lse_out,
                               double* ess_out, int32_t* status_out, int32_t* offspring, int32_t* permuted,
                               void* X, int64_t x_row_bytes, int64_t x_ld, int64_t x_fld, void* scratch,
                               cudaStream_t s, uint64_t* launches, uint64_t* Qout = nullptr, int64_t ldq = 0,
                               uint64_t* Qtot_out = nullptr);

// Cross-GPU particle migration of a sharded filter (pf_migrate.cu; include/pf.h 4a-4d).
size_t mig_plan_bytes(int32_t Pl);  // the tiles' prefixes of extras / free slots
cudaError_t launch_mig_offspring(const int32_t* anc, int64_t n_anc, const int64_t* range, int64_t win0, int32_t Pw,
                                 const float* gmax, const int32_t* gbad, int32_t* o, cudaStream_t s,
                                 uint64_t* launches);
cudaError_t launch_mig_plan(const int32_t* o, int32_t Pl, void* plan, int64_t* counts, cudaStream_t s,
                            uint64_t* launches);
cudaError_t launch_mig_pack(const void* X, int64_t row_bytes, int64_t ld, int32_t Pl, int64_t p0, const int32_t* o,
                            const void* plan, void* send, int32_t* send_src, cudaStream_t s, uint64_t* launches);
cudaError_t launch_mig_unpack(void* X, int64_t row_bytes, int64_t ld, int32_t Pl, int64_t p0, const int32_t* o,
                              const void* plan, const void* recv, const int32_t* recv_src, int32_t* perm,
                              cudaStream_t s, uint64_t* launches);

// pf_f64.cu: binary64 log-weights (NS-3d).  ws holds f64_ws_bytes(N, P): t [N][ldt] float
// (ldt = P rounded up to 4), then the per-filter max keys (u64) and bad flags (i32).
size_t f64_ws_bytes(int32_t N, int32_t P);
constexpr int32_t kFusedF64MaxP = 65536;  // binary64 instantiation of the cluster kernel: 8 x 8192
cudaError_t launch_shift64(const double* logw, int64_t ld, int32_t N, int32_t P, void* ws, float** t_out,
                           int64_t* ldt_out, unsigned long long** key_out, cudaStream_t s, uint64_t* launches);
cudaError_t launch_lse64(const unsigned long long* key, int32_t N, double* lse, cudaStream_t s,
                         uint64_t* launches);

// pf_wsort.cu: pre-sorted weights (PF_SORT_WEIGHTS, NS-17).  ws holds wsort_ws_bytes(N, P, normw).
struct WsortBufs {
    float* y;          // [N][ldk] log-weights sorted in descending order
    int32_t* sigma;    // [N][ldk] original index of each sorted position
    int64_t ldk;
    int32_t* b;        // [N][ldk] ancestors in sorted space (written by the float path)
    int32_t* fstatus;  // [N] filter status (written by the float path)
    float* vs;         // [N][P] normalised weights in sorted order (nullable)
};
size_t wsort_ws_bytes(int32_t N, int32_t P, bool normw);
cudaError_t launch_wsort(const float* logw, int64_t ld, int32_t N, int32_t P, void* ws, bool normw, WsortBufs* out,
                         cudaStream_t s, uint64_t* launches);
cudaError_t launch_unsort(const WsortBufs& w, int32_t N, int32_t P, int32_t* anc, int64_t ld_anc, float* normw,
                          cudaStream_t s, uint64_t* launches);

}  // namespace pf
