/*
 * pf.h — C ABI of libpfresample: B200 (sm_100a) particle-filter resampling,
 * after Murray, "GPU acceleration of the particle filter: the Metropolis
 * resampler" (arXiv 1202.6163).
 *
 * Citation keys: P:n = PAPER.md line n (the paper's text); NS-n / R-n =
 * DESIGN.md §3 numeric spec / §3.2 readings.  The problem statement is P:64-68:
 * "Redraw, with replacement, P samples from the weighted sample set, using
 * weights as unnormalised probabilities".
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Every data pointer is CALLER-OWNED DEVICE memory (cudaMalloc / torch),
 *    unless stated otherwise.  The library never frees caller memory.
 *  - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *    Calls only ENQUEUE work: they never synchronise the stream, never abort
 *    and never throw.  Results are ready when the stream reaches them.
 *  - Argument errors (NULL pointer, P < 1, N < 1, B < 0, ld < P, bad scheme,
 *    too-small explicit workspace) are reported synchronously by the return
 *    value and nothing is enqueued.  A failed launch returns PF_ERR_CUDA
 *    (cudaPeekAtLastError after the launch).
 *  - Data-dependent errors are reported asynchronously, per filter, in the
 *    optional device array status_out (PF_FILTER_*): any NaN or +inf
 *    log-weight, or all log-weights -inf, is invalid (NS-1); the ancestors of
 *    an invalid filter are the identity and its lse/ess/normw are NaN.
 *  - Log-weights are float32; -inf means zero weight.  Ancestors, offspring
 *    and permutations are int32, 0-based.
 *  - Randomness is a pure function of (seed, scheme, filter_index, slot): the
 *    Philox4x32-10 counter is (c0, c1, scheme tag, filter_index) and the key
 *    is the 64-bit seed (NS-6).  Results are bit-identical to the CPU oracle
 *    (oracle/pfo.c) and independent of launch configuration and GPU count.
 *  - Workspace: by default the library uses its own pool keyed by (device,
 *    stream), grown on demand outside steady state ("pooled memory").
 *    The device is the CURRENT device (cudaGetDevice) of the calling thread:
 *    make it the device of the buffers and of the stream (the Python binding
 *    does so around every call).
 *  - Thread safety: concurrent calls are safe on distinct streams.  Calls that
 *    share a stream from several host threads must be serialised by the caller,
 *    even with explicit workspaces: the binary64 shift buffer, PF_SORT_WEIGHTS,
 *    pf_permute*, pf_gather_state* and every pf_shard_* stage always draw
 *    scratch from the (device, stream) pool.
 */
#ifndef PF_H
#define PF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* pf_stream_t; /* cudaStream_t */

typedef enum {
    PF_OK = 0,
    PF_ERR_INVALID_ARG = 1,
    PF_ERR_WORKSPACE = 2,
    PF_ERR_CUDA = 3,
    PF_ERR_UNSUPPORTED = 4
} pf_status;

/* Scheme ids double as the Philox counter tag c2 (NS-6). */
typedef enum {
    PF_MULTINOMIAL = 1, /* Fig. 1(a): i.i.d. uniform positions      */
    PF_STRATIFIED = 2,  /* Fig. 1(b): one offset per stratum       */
    PF_SYSTEMATIC = 3,  /* Fig. 1(c): one shared offset (Kitagawa) */
    PF_METROPOLIS = 4   /* Fig. 1(d): B-step chains    */
} pf_scheme;

enum { PF_FILTER_OK = 0, PF_FILTER_INVALID_WEIGHTS = 1 };

/* pf_opts.flags bits */
enum {
    /* with PF_MULTINOMIAL: the sorted-uniform multinomial (NS-12):
     * positions are the uniform order statistics G_k / G_P of exponential
     * spacings (Philox tag 5, deterministic double log), so the ancestors come
     * out nondecreasing and the search is a merge instead of per-slot binary
     * searches.  Same law as PF_MULTINOMIAL (Fig. 1(a)), different random stream. */
    PF_SORTED = 1u << 0,
    /* diagnostics: force the multi-launch path (max -> lookback scan -> search)
     * even where the one-launch cluster kernel applies.  Results are identical. */
    PF_NO_FUSION = 1u << 1,
    /* with PF_MULTINOMIAL / PF_STRATIFIED / PF_SYSTEMATIC: the paper's pre-sorted weight
     * series (NS-17): each filter's log-weights are stably sorted in
     * descending order (equal values, +0 = -0, in index order) by a segmented radix sort,
     * resampled by the same scheme, seed and filter index, and the ancestors are mapped back
     * to the original indices (a_k = sigma[b_k]); normw_out / offspring_out / permuted_out /
     * state are in the original order.  Same law as the unsorted scheme; the paper found the
     * sort to cost more than the faster search saves.  Not with PF_SORTED or
     * PF_METROPOLIS (-> PF_ERR_UNSUPPORTED).  Its scratch (~20 B per particle) always comes from
     * the library pool. */
    PF_SORT_WEIGHTS = 1u << 2
};

/*
 * Optional outputs and controls of pf_resample_ex / pf_resample_batched.
 * All device pointers are nullable.  A zero-initialised struct means "none".
 */
typedef struct {
    uint32_t filter_index; /* Philox c3 of a single-filter call (batched: first_filter+n) */
    uint32_t flags;        /* PF_SORTED (multinomial only) | PF_NO_FUSION | PF_SORT_WEIGHTS; other bits -> PF_ERR_UNSUPPORTED */
    double* lse_out;       /* [N] ln sum_i exp(logw_i)  (NS-13; 1e-6 rel. of oracle)       */
    float* normw_out;      /* [N][P] (row stride P) v_i = w_i / sum_j w_j  (NS-13)          */
    double* ess_out;       /* [N] (sum w)^2 / sum w^2                          */
    int32_t* status_out;   /* [N] PF_FILTER_* per filter                                    */
    int32_t* offspring_out; /* [N][P] (row stride = ancestors' ld) o_i = #{k : a_k = i} (NS-14);
                              the cluster and cooperative kernels derive it from their slot
                              counts at no extra pass, the warp / CTA-per-filter kernels count
                              in shared memory, the multi-launch path runs a histogram      */
    int32_t* permuted_out;  /* [N][P] (row stride = ancestors' ld) the canonical in-place
                              permutation of the ancestors (NS-15, = pf_permute(ancestors));
                              stratified/systematic: written by the cluster kernel (P <= 65536,
                              or P <= 262144 for batches spanning the GPU) or the cooperative
                              kernel (large filters, few of them); otherwise computed from the
                              offspring after the search                                    */
    void* workspace;       /* device, 256-byte aligned, nullable -> library pool            */
    size_t workspace_bytes;
    /* Optional fused state gather (a10, NS-16; "redraw"): if state is non-NULL, after
     * resampling every filter's rows are gathered IN PLACE with the canonical permutation a'
     * (NS-15): row i <- row a'_i for the non-survivors, survivors untouched.  Filter n's rows
     * start at state + n * state_filter_ld_bytes, row i at + i * state_ld_bytes, each
     * state_row_bytes long (device).  Same result as pf_permute + pf_gather_state_batched;
     * fused into the cluster kernel for power-of-two rows of 16..512 bytes (16-byte aligned
     * strides), otherwise run as a separate gather after the permutation.  Requires
     * state_ld_bytes >= state_row_bytes and non-overlapping filters. */
    void* state;
    int64_t state_row_bytes;
    int64_t state_ld_bytes;
    int64_t state_filter_ld_bytes;
} pf_opts;

/*
 * Single-filter resamplers with the north-star signature.
 *   logw      [P] float32 log-weights (device).
 *   P         particle count, 1 <= P <= 2^31-1.
 *   seed      64-bit Philox key.
 *   B         Metropolis steps per chain; ignored (must be >= 0)
 *             by the prefix-sum schemes.  B = 0 yields the identity.
 *   ancestors [P] int32 output (device): a_k = ancestor of slot k.
 * The multinomial, stratified and systematic schemes compute the exact u64
 * fixed-point inclusive scan of the weights and search it
 * (NS-5..NS-10); stratified and systematic ancestors are nondecreasing.
 * The Metropolis scheme needs no collective (NS-11).
 */
pf_status pf_resample_multinomial(const float* logw, int32_t P, uint64_t seed, int32_t B,
                                  int32_t* ancestors, pf_stream_t stream);
pf_status pf_resample_stratified(const float* logw, int32_t P, uint64_t seed, int32_t B,
                                 int32_t* ancestors, pf_stream_t stream);
pf_status pf_resample_systematic(const float* logw, int32_t P, uint64_t seed, int32_t B,
                                 int32_t* ancestors, pf_stream_t stream);
pf_status pf_resample_metropolis(const float* logw, int32_t P, uint64_t seed, int32_t B,
                                 int32_t* ancestors, pf_stream_t stream);

/* Same with a scheme id and optional outputs (opts nullable). */
pf_status pf_resample_ex(pf_scheme scheme, const float* logw, int32_t P, uint64_t seed, int32_t B,
                         int32_t* ancestors, const pf_opts* opts, pf_stream_t stream);

/*
 * Batched resampling of N independent filters (PMCMC): filter n reads
 * logw[n*ld_logw .. +P) and writes ancestors[n*ld_anc .. +P).  Filter n is
 * bit-identical to pf_resample_ex with filter_index = first_filter + n, so
 * disjoint filter ranges may be resampled on different GPUs.
 * opts->filter_index is ignored here.
 */
pf_status pf_resample_batched(pf_scheme scheme, const float* logw, int64_t ld_logw, int32_t N, int32_t P,
                              uint64_t seed, uint32_t first_filter, int32_t B,
                              int32_t* ancestors, int64_t ld_anc, const pf_opts* opts, pf_stream_t stream);

/*
 * Binary64 log-weights (the paper's precision; NS-3d / R-21).  Same
 * arguments, outputs and error behaviour as pf_resample_ex / pf_resample_batched, with logw
 * double [N][ld_logw] (device).  The filter's maximum is taken in binary64 (NaN, +inf or
 * all -inf -> invalid, NS-1), t_i = logw_i - lmax is computed in binary64 and rounded once
 * to binary32, and the float32 path runs on t (every option, flag and kernel applies); lse
 * = lmax + ln sum_i w_i keeps the binary64 maximum.  Use it when the log-weights carry a
 * large common offset (an accumulated log-likelihood) that float32 would round away.  The
 * shifted weights (4 B per particle + 12 B per filter) always come from the library pool
 * (pf_opts.workspace, when given, serves the float path only).  Stratified / systematic
 * filters of 4097..65536 particles (no PF_NO_FUSION / PF_SORT_WEIGHTS) run in one launch of
 * the cluster kernel's binary64 instantiation, which reads the doubles itself; every other
 * call takes two extra launches (max, shift) before the float path and one after it when
 * lse_out is set.  Results are identical either way.
 */
pf_status pf_resample_ex_f64(pf_scheme scheme, const double* logw, int32_t P, uint64_t seed, int32_t B,
                             int32_t* ancestors, const pf_opts* opts, pf_stream_t stream);
pf_status pf_resample_batched_f64(pf_scheme scheme, const double* logw, int64_t ld_logw, int32_t N, int32_t P,
                                  uint64_t seed, uint32_t first_filter, int32_t B,
                                  int32_t* ancestors, int64_t ld_anc, const pf_opts* opts, pf_stream_t stream);

/* Workspace bytes a call with these sizes needs (for explicit workspaces, pf_opts.workspace):
 * the maximum over every path the call may take.  _ex takes the pf_opts.flags (PF_SORTED needs
 * the spacings scan) and the ancestors' row stride; pf_workspace_bytes(s, N, P) =
 * pf_workspace_bytes_ex(s, N, P, 0, P).  Returns 0 for invalid arguments.  An explicit workspace
 * is not supported together with permuted_out or state on the multi-launch path (multinomial,
 * Metropolis, P above the cluster kernel): those calls return PF_ERR_UNSUPPORTED. */
size_t pf_workspace_bytes(pf_scheme scheme, int32_t N, int32_t P);
size_t pf_workspace_bytes_ex(pf_scheme scheme, int32_t N, int32_t P, uint32_t flags, int64_t ld_anc);

/*
 * Ancestors -> offspring (NS-14): offspring[i] = #{k : anc[k] == i}.
 * anc entries must lie in [0, P).  Batched form: N rows with strides.
 */
pf_status pf_ancestors_to_offspring(const int32_t* anc, int32_t P, int32_t* offspring, pf_stream_t stream);
pf_status pf_ancestors_to_offspring_batched(const int32_t* anc, int64_t ld_anc, int32_t N, int32_t P,
                                            int32_t* offspring, int64_t ld_off, pf_stream_t stream);

/*
 * In-place permutation (NS-15; BJ north_star): permuted is a permutation of
 * the multiset anc with permuted[i] == i for every surviving particle i
 * (offspring > 0); the free slots, ascending, receive the extra copies in
 * ascending survivor order.  Unique given the offspring; independent of the
 * order of anc.  Batched form: N rows with strides.
 */
pf_status pf_permute(const int32_t* anc, int32_t P, int32_t* permuted, pf_stream_t stream);
pf_status pf_permute_batched(const int32_t* anc, int64_t ld_anc, int32_t N, int32_t P,
                             int32_t* permuted, int64_t ld_perm, pf_stream_t stream);

/*
 * Canonical permutation from offspring counts (NS-15): identical result to
 * pf_permute(anc) for any ancestors with these offspring.  offspring[i] >= 0
 * and sum_i offspring[i] == P are required (not checked).  Use with
 * pf_opts.offspring_out to skip the ancestor histogram.
 */
pf_status pf_permute_offspring(const int32_t* offspring, int32_t P, int32_t* permuted, pf_stream_t stream);
pf_status pf_permute_offspring_batched(const int32_t* offspring, int64_t ld_off, int32_t N, int32_t P,
                                       int32_t* permuted, int64_t ld_perm, pf_stream_t stream);

/*
 * State gather in place (NS-16): for each i with permuted[i] != i,
 * row i of X (row_bytes bytes at X + i*ld_bytes) <- row permuted[i].  Safe in
 * place ONLY for a pf_permute output (reads touch survivors, writes touch
 * non-survivors).  Batched: filter n's rows start at X + n*ld_filter_bytes and
 * its permutation at permuted + n*ld_perm.
 */
pf_status pf_gather_state(void* X, int64_t row_bytes, int64_t ld_bytes, int32_t P,
                          const int32_t* permuted, pf_stream_t stream);
pf_status pf_gather_state_batched(void* X, int64_t row_bytes, int64_t ld_bytes, int64_t ld_filter_bytes,
                                  int32_t N, int32_t P, const int32_t* permuted, int64_t ld_perm,
                                  pf_stream_t stream);

/* Out-of-place gather for arbitrary ancestors: Y[i] <- X[anc[i]]. X and Y must not overlap. */
pf_status pf_gather_state_out(const void* X, void* Y, int64_t row_bytes, int64_t ld_x, int64_t ld_y,
                              int32_t P, const int32_t* anc, pf_stream_t stream);

/*
 * Giant-filter sharding.  One filter of P_global
 * particles is split into contiguous shards; shard g owns particles
 * [p0, p0 + Pl).  The stages below run on the shard's GPU; the caller issues
 * the collectives between them (torch.distributed / NCCL):
 *   1 pf_shard_max          -> all_reduce(MAX) of lmax, all_reduce(MAX) of bad
 *   2 pf_shard_scan         -> all_gather of the 8-byte local totals (and sums)
 *   3 pf_shard_search       (stratified / systematic / multinomial)
 *   Metropolis: pf_shard_weights -> all_gather of the weights ->
 *               pf_metropolis_from_weights on any slot range.
 * Every stage evaluates the single-filter numeric spec (NS-2..NS-11) with the
 * GLOBAL max and k_fx(P_global), so the assembled ancestors are bit-identical
 * to pf_resample_ex on the whole filter (filter_index, seed as given).
 */
/* d_lmax[0] = max of the shard's log-weights (-inf if none); d_bad[0] = 1 if
 * any NaN or +inf (else 0).  Device outputs. */
pf_status pf_shard_max(const float* logw, int32_t Pl, float* d_lmax, int32_t* d_bad, pf_stream_t stream);
/* d_Q[Pl] (u64, device, caller-owned) = inclusive fixed-point scan of the shard
 * with the global max *d_gmax and k_fx = 61 - ceil(log2 P_global) (NS-5);
 * d_total[0] = Q of the shard's last particle; d_wsum[0] = sum of the shard's
 * w_i in double (lse = gmax + ln sum over shards, NS-13).  d_wsum nullable. */
pf_status pf_shard_scan(const float* logw, int32_t Pl, int64_t P_global, const float* d_gmax, uint64_t* d_Q,
                        uint64_t* d_total, double* d_wsum, pf_stream_t stream);
/* Ancestors of the slots whose positions fall in this shard's range of the
 * cumulative weights.  d_totals[nshards] = every shard's d_total (all-gathered,
 * device).  d_gmax / d_gbad = all-reduced max and bad flag (device).  Writes
 * anc_out[k] = global ancestor index for each slot k of this shard (anc_out has
 * P_global entries; other entries untouched) and d_slot_range[0..1] = [k_lo,
 * k_hi).  Stratified/systematic: positions are sorted, the slot range is found
 * by search and merged with d_Q (work ~ Pl + slots).  Multinomial: every shard
 * regenerates all P_global positions and keeps its own (replicated position
 * generation; exact, not work-optimal: the routed stages below are).  An invalid global filter (bad or all
 * -inf) writes the identity for slots [p0, p0 + Pl).  P_global <= 2^31 - 1. */
pf_status pf_shard_search(pf_scheme scheme, const uint64_t* d_Q, int32_t Pl, int64_t p0, int64_t P_global,
                          const uint64_t* d_totals, int32_t nshards, int32_t shard, const float* d_gmax,
                          const int32_t* d_gbad, uint64_t seed, uint32_t filter_index, int32_t* anc_out,
                          int64_t* d_slot_range, pf_stream_t stream);

/*
 * Routed unsorted multinomial (Fig. 1(a)): the
 * work-optimal alternative to pf_shard_search's replicated position generation.  Shard g
 * generates only the positions x_k (NS-8) of its own SLOT shard [g ceil(P/G), ...) and each goes
 * to the shard whose cumulative-weight range [off_h, off_h + T_h) holds it:
 *   pf_shard_route_count   d_counts[nshards] (int64, device) = this slot shard's positions per
 *                          owner shard (all zero for an invalid filter)
 *   (caller: all_gather of the counts -> the split sizes of one variable all_to_all)
 *   pf_shard_route_pack    send_x (u64) / send_k (int32) = the pairs (x_k, k) grouped by owner in
 *                          shard order (group h starts at sum_{h' < h} d_counts[h']; the order
 *                          inside a group is unspecified); d_counts from pf_shard_route_count
 *   (caller: all_to_all of the pairs)
 *   pf_shard_route_search  for the nrecv received pairs: anc_out[k] = p0 + min{i : Q_i > x - off}
 *                          (the same value pf_shard_search writes); an invalid filter writes the
 *                          identity for slots [p0, p0 + Pl).
 * Work per rank ~ P_global / nshards generated positions + its received ones.  nshards <= 64,
 * P_global <= 2^31 - 1.  d_totals / d_gmax / d_gbad as for pf_shard_search. */
pf_status pf_shard_route_count(const uint64_t* d_totals, int32_t nshards, int32_t shard, int64_t P_global,
                               const float* d_gmax, const int32_t* d_gbad, uint64_t seed, uint32_t filter_index,
                               int64_t* d_counts, pf_stream_t stream);
pf_status pf_shard_route_pack(const uint64_t* d_totals, int32_t nshards, int32_t shard, int64_t P_global,
                              const float* d_gmax, const int32_t* d_gbad, uint64_t seed, uint32_t filter_index,
                              const int64_t* d_counts, uint64_t* send_x, int32_t* send_k, pf_stream_t stream);
pf_status pf_shard_route_search(const uint64_t* d_Q, int32_t Pl, int64_t p0, int64_t P_global,
                                const uint64_t* d_totals, int32_t nshards, int32_t shard, const float* d_gmax,
                                const int32_t* d_gbad, const uint64_t* recv_x, const int32_t* recv_k, int64_t nrecv,
                                int32_t* anc_out, pf_stream_t stream);
/*
 * Sorted-uniform multinomial (a6, NS-12) over shards: work-optimal.
 * The P_global + 1 spacings e_0..e_P are split into nshards contiguous SPACING
 * shards [s_h, s_{h+1}), s_h = min(P+1, h * ceil((P+1)/nshards)) (independent of
 * the particle shards' sizes).  Stages after pf_shard_scan:
 *   2b pf_shard_spacings_total -> all_gather of the 8-byte spacing totals
 *   3  pf_shard_search_sorted
 * Bit-identical to pf_resample_ex(PF_MULTINOMIAL, flags = PF_SORTED) on the whole filter.
 */
/* d_etotal[0] (device) = e_{s_h} + ... + e_{s_{h+1}-1} for h = shard (NS-12 e_k from
 * Philox tag 5 of filter_index and seed).  0 <= shard < nshards. */
pf_status pf_shard_spacings_total(int64_t P_global, int32_t nshards, int32_t shard, uint64_t seed,
                                  uint32_t filter_index, uint64_t* d_etotal, pf_stream_t stream);
/* Bytes of device workspace pf_shard_search_sorted needs (8 (P_global + P_global / 4096) + 1 KiB:
 * the scanned G range is at most P_global slots, e.g. when one shard holds all the weight). */
size_t pf_shard_search_sorted_workspace_bytes(int64_t P_global);
/* Sorted multinomial ancestors of the slots whose positions x_k = floor(G_k Q / G_P)
 * fall in this particle shard's range [off, off + T) of the cumulative weights.
 * d_totals[nshards] / d_etotals[nshards]: all-gathered pf_shard_scan totals and
 * pf_shard_spacings_total values (device).  The shard regenerates and scans only the
 * spacing shards containing its slots (the plan is computed on the device), then
 * merges the positions with d_Q.  anc_out (P_global entries, device) receives the
 * global ancestor of each of its slots; d_slot_range[0..1] = [k_lo, k_hi).
 * workspace: device, 256-byte aligned, >= pf_shard_search_sorted_workspace_bytes, or NULL for the
 * library pool.  Invalid global filter: identity for slots [p0, p0 + Pl). */
pf_status pf_shard_search_sorted(const uint64_t* d_Q, int32_t Pl, int64_t p0, int64_t P_global,
                                 const uint64_t* d_totals, const uint64_t* d_etotals, int32_t nshards, int32_t shard,
                                 const float* d_gmax, const int32_t* d_gbad, uint64_t seed, uint32_t filter_index,
                                 int32_t* anc_out, int64_t* d_slot_range, void* workspace, size_t workspace_bytes,
                                 pf_stream_t stream);
/* Metropolis weights of the shard: w_out[Pl] = dexp(logw - *d_gmax) (NS-4). */
pf_status pf_shard_weights(const float* logw, int32_t Pl, const float* d_gmax, float* w_out, pf_stream_t stream);
/* Metropolis chains (NS-11) for slots [slot0, slot0 + nslots) of a filter whose
 * full weight vector w_full[P_global] is on this device; anc[s] = final state of
 * chain slot0 + s.  Bit-identical to the same chains of pf_resample_metropolis.
 * d_gmax / d_gbad (nullable, device): the all-reduced max and bad flag; an
 * invalid filter (bad, or max = -inf) gives the identity (NS-1). */
pf_status pf_metropolis_from_weights(const float* w_full, int64_t P_global, int64_t slot0, int32_t nslots,
                                     uint64_t seed, int32_t B, uint32_t filter_index, const float* d_gmax,
                                     const int32_t* d_gbad, int32_t* anc, pf_stream_t stream);

/*
 * Cross-GPU particle migration of a sharded filter:
 * the in-place permutation (a9, NS-15) and state gather (a10, NS-16) of the WHOLE filter,
 * applied shard by shard.  After resampling, shard g's particles [p0, p0 + Pl) have
 * offspring o_i; the global extras list (particle i repeated o_i - 1 times, ascending i)
 * is the concatenation of the shards' own extras lists, and the global free-slot list
 * (o_i = 0, ascending) the concatenation of their own free lists, so the r-th global
 * extra goes to the r-th global free slot exactly as NS-15 on the whole filter:
 *   4a pf_shard_offspring         o_i of the shard's particles (prefix-sum schemes: every
 *                                 ancestor of a particle of shard g was written by rank g)
 *                                 (Metropolis: histogram the rank's slots over the whole
 *                                 filter, then reduce_scatter(SUM) of the counts)
 *   4b pf_shard_migration_counts  d_counts = {E_g extras, F_g free slots} + the tile plan
 *      -> all_gather of the counts; exclusive prefixes give each rank's ranges of the
 *         global extras / free lists, hence the split sizes of one variable all-to-all
 *   4c pf_shard_migrate_pack      the shard's extra rows (+ their global indices), in order
 *      -> all_to_all of the rows (rank g receives exactly its F_g rows, in global order)
 *   4d pf_shard_migrate_unpack    received rows into the free slots; survivors stay
 * Afterwards shard g holds rows [p0, p0 + Pl) of pf_gather_state(X, pf_permute(anc)) on the
 * whole filter, and perm_out[i] = pf_permute(anc)[p0 + i].  Rows that stay on their shard
 * go through the all-to-all's self-copy.  Sum over shards of E_g = sum of F_g.
 */
/* offspring[Pw] (device) = #{k in the slot window : anc[k] - win0 = i} for i in [0, Pw).
 * anc[n_anc] (device) holds global ancestor indices; the slot window is
 * [d_slot_range[0], d_slot_range[1]) clamped to [0, n_anc) (d_slot_range: device, as
 * written by pf_shard_search for stratified / systematic or pf_shard_search_sorted; the
 * entries in it must be NONDECREASING, as those searches write them: each run's length is
 * stored without atomics), or all n_anc entries, in any order, when d_slot_range is NULL
 * (the unsorted multinomial, whose shard writes scattered slots, entries it did not write
 * lying outside [win0, win0 + Pw), e.g. -1; Metropolis slot histograms).  Entries outside
 * [win0, win0 + Pw) are ignored.  d_gmax / d_gbad (device, both or neither): when they
 * mark the global filter invalid (bad, or max = -inf), offspring = 1 everywhere (the
 * identity ancestors NS-1 gives; the searches then report an empty slot range). */
pf_status pf_shard_offspring(const int32_t* anc, int64_t n_anc, const int64_t* d_slot_range, int64_t win0,
                             int32_t Pw, const float* d_gmax, const int32_t* d_gbad, int32_t* offspring,
                             pf_stream_t stream);
/* Bytes of the migration plan of a shard of Pl particles (24 per 2048-particle tile + 8). */
size_t pf_shard_migration_plan_bytes(int32_t Pl);
/* d_counts[0] = E = sum_i max(o_i - 1, 0), d_counts[1] = F = #{i : o_i = 0} (device int64);
 * plan (device, caller-owned, 8-byte aligned, >= pf_shard_migration_plan_bytes(Pl)) receives
 * every tile's offsets into the shard's extras and free lists, read by 4c and 4d (the
 * offspring must not change in between). */
pf_status pf_shard_migration_counts(const int32_t* offspring, int32_t Pl, void* plan, int64_t* d_counts,
                                    pf_stream_t stream);
/* send_rows[E][row_bytes] (device, packed) = the shard's extra rows in NS-15 order: for
 * ascending i with o_i > 1, o_i - 1 copies of X[i]; send_src[E] (device int32, nullable) =
 * their global indices p0 + i.  X: [Pl] rows of row_bytes at stride ld_bytes; X and
 * send_rows may be NULL when row_bytes = 0 (indices only).  Must not overlap. */
pf_status pf_shard_migrate_pack(const void* X, int64_t row_bytes, int64_t ld_bytes, int32_t Pl, int64_t p0,
                                const int32_t* offspring, const void* plan, void* send_rows, int32_t* send_src,
                                pf_stream_t stream);
/* In place: the r-th free slot (o_i = 0, ascending i) of the shard <- recv_rows[r]
 * (packed rows, F of them, device); survivors are untouched.  perm_out[Pl] (device int32,
 * nullable unless row_bytes = 0) = p0 + i for survivors, recv_src[r] for the r-th free
 * slot.  recv_rows (when row_bytes > 0) and recv_src (when perm_out is given) must hold F
 * entries; they are not read, and may be NULL, when F = 0.  X may be NULL when row_bytes = 0. */
pf_status pf_shard_migrate_unpack(void* X, int64_t row_bytes, int64_t ld_bytes, int32_t Pl, int64_t p0,
                                  const int32_t* offspring, const void* plan, const void* recv_rows,
                                  const int32_t* recv_src, int32_t* perm_out, pf_stream_t stream);

/*
 * Bootstrap particle filter demo model (BASELINE config C4; P:43-68 steps 1-3;
 * DESIGN.md R-20): a diagonal AR(1) state in D dimensions, x_t = phi x_{t-1} +
 * sigma_x eps_t, observed through y_t = x_t[0] + sigma_y eta_t.  X is float32
 * [P][ld] row-major (ld >= D, device).  Noise: Philox4x32-10 (tag 6 for the
 * transition, 7 for the initial draw; counter (particle, step * ceil(D/4) + block,
 * tag, 0)) -> Box-Muller normals (float32 intrinsics; not part of the bit-exact
 * resampling contract).
 */
/* x_0 ~ N(0, sigma_x^2 / (1 - phi^2)) in every dimension (stationary start). */
pf_status pf_lg_init(float* X, int64_t ld, int32_t P, int32_t D, float phi, float sigma_x, uint64_t seed,
                     pf_stream_t stream);
/* Propagate (step 2) and weight (step 3): x <- phi x + sigma_x eps, then
 * logw_i = -(y - x_i[0])^2 / (2 sigma_y^2).  t = time index (1-based). */
pf_status pf_lg_propagate_weight(float* X, int64_t ld, int32_t P, int32_t D, float phi, float sigma_x,
                                 float sigma_y, float y, uint64_t seed, int32_t t, float* logw, pf_stream_t stream);
/* loglik[0] += lse[0] - ln P - ln(2 pi sigma_y^2) / 2: the log of the bootstrap
 * likelihood increment p(y_t | y_1:t-1) (lse from pf_resample_ex lse_out). */
pf_status pf_lg_accumulate(const double* lse, int32_t P, float sigma_y, double* loglik, pf_stream_t stream);

/*
 * Host helper: minimum B with lambda^B <= eps (alpha+beta)/max(alpha,beta)
 * (Eq. (4)-(5)), alpha = (1 - w_max)/(P w_max) (Eq. (2)), beta = 1/P.  Returns at least 1
 * (a resampler takes at least one step: 1 when Eq. (4) holds already or lambda <= 0;
 * DESIGN R-22), -1 on invalid arguments: P < 1, eps <= 0, w_max outside [1/P, 1] (a maximum
 * of P normalised weights is >= 1/P), or a B beyond INT32_MAX.  Host-only, no GPU.
 */
int32_t pf_metropolis_required_B(int64_t P, double w_max, double eps);

const char* pf_status_string(pf_status s);

/* Number of kernels this library has launched in this process (diagnostics / bench). */
uint64_t pf_launch_count(void);

/*
 * Per-kernel tracing (SURVEY §5 "tracing"): when enabled, every kernel launch
 * is bracketed by two CUDA events recorded on its own stream (the launching
 * stream, so the interval is that kernel's device duration).
 * pf_profile_collect waits for the recorded events, writes up to max_entries
 * aggregated {kernel name, launches, total milliseconds, algorithmic bytes}
 * records, clears the record and returns the number of distinct kernels (or -1
 * on a CUDA error).  alg_bytes sums, over the kernel's launches, the HBM bytes
 * each launch must move by what it was asked to read and write (inputs once,
 * outputs once; 0 = not stated for that kernel); row_bytes sums the extra bytes
 * per moved state row of launches that gather a state (2 x row bytes: one read,
 * one write), which the caller multiplies by the rows that moved (data-
 * dependent).  Not for use inside CUDA-graph capture.
 */
typedef struct {
    char name[32];
    uint64_t launches;
    double total_ms;
    uint64_t alg_bytes;
    uint64_t row_bytes;
} pf_kernel_time;
void pf_profile_enable(int32_t on);
int32_t pf_profile_collect(pf_kernel_time* out, int32_t max_entries);

/*
 * Diagnostics: pf_set_fusion(0) makes every entry point use its multi-launch
 * path (lookback scans, merge-path searches) even where a one-launch cluster
 * kernel applies; pf_set_fusion(1) (default) re-enables them.  Results are
 * identical either way; only speed differs.  Process-wide.
 */
void pf_set_fusion(int32_t on);

/* Library version string. */
const char* pf_version(void);

/* Free the library workspace pool (all devices/streams).  Must not race with calls. */
void pf_release(void);

#ifdef __cplusplus
}
#endif
#endif /* PF_H */
