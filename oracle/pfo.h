/*
 * oracle/pfo.h — CPU ORACLE for particle-filter resampling (arXiv 1202.6163).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may link or call this
 * library.  It shares no code, header, table or constant generator with the
 * CUDA product path (paper_1202_6163_b200/csrc); both implement the numeric
 * spec written out in DESIGN.md §3 ("NS-n") independently.
 *
 * Citation keys:  P:n = /root/reference/PAPER.md line n,  NS-n = DESIGN.md §3.
 * All pointers are host pointers; no function allocates caller memory.
 */
#ifndef PFO_H
#define PFO_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { PFO_MULTINOMIAL = 1, PFO_STRATIFIED = 2, PFO_SYSTEMATIC = 3, PFO_METROPOLIS = 4 };
enum { PFO_FILTER_OK = 0, PFO_FILTER_INVALID_WEIGHTS = 1 };

/* NS-6: Philox4x32-10 block function (counter ctr[4], key key[2]) -> out[4]. */
void pfo_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* NS-4: deterministic float32 exp of t <= 0. */
float pfo_dexp(float t);

/* NS-1/NS-2: validate and reduce; returns PFO_FILTER_* and writes lmax. */
int pfo_lmax(const float* logw, int32_t P, float* lmax);

/* NS-3/NS-4: w_i = dexp(fl(logw_i - lmax)); returns filter status. */
int pfo_weights(const float* logw, int32_t P, float* w);

/* NS-3/NS-4 with an explicit (e.g. global) maximum: w_i = dexp(fl(logw_i - lmax)). */
void pfo_weights_with(const float* logw, int32_t P, float lmax, float* w);

/* NS-5 with explicit maximum and fraction bits (a shard of a larger filter). */
void pfo_cumulative_with(const float* logw, int32_t P, float lmax, int kfx, uint64_t* Q);

/* NS-5: fixed-point fraction bits k_fx = 61 - ceil(log2 P). */
int pfo_kfx(int32_t P);

/* NS-5: Q_i = sum_{j<=i} q_j (inclusive, u64).  Returns filter status. */
int pfo_cumulative(const float* logw, int32_t P, uint64_t* Q);

/* NS-7..NS-10: position x_k of slot k in [0, Q_total) for the prefix-sum schemes. */
uint64_t pfo_position(int scheme, int32_t P, uint64_t Qtot, uint64_t seed,
                      uint32_t filter_index, int64_t k);

/* a = min{ i : Q_i > x }  (G6: half-open [Q_{i-1}, Q_i)). */
int32_t pfo_upper_bound(const uint64_t* Q, int32_t P, uint64_t x);

/* Systematic search with an explicit 64-bit offset fraction R (SPEC S:171 example). */
void pfo_systematic_from_R(const uint64_t* Q, int32_t P, uint64_t R, int32_t* anc);

/* NS-11: Metropolis chains for slots [slot0, slot0+nslots) over weights w[P]. */
void pfo_metropolis_chains(const float* w, int32_t P, int64_t slot0, int32_t nslots,
                           uint64_t seed, int32_t B, uint32_t filter_index, int32_t* anc);

/*
 * Full resampling of one filter (NS-1..NS-13).  anc[P] always written
 * (identity when invalid).  lse/normw/ess may be NULL.  Returns PFO_FILTER_*.
 */
int pfo_resample(int scheme, const float* logw, int32_t P, uint64_t seed, int32_t B,
                 uint32_t filter_index, int32_t* anc, double* lse, float* normw, double* ess);

/* Batched: filter n uses filter_index first_filter + n; rows strided. */
void pfo_resample_batched(int scheme, const float* logw, int64_t ld_logw, int32_t N, int32_t P,
                          uint64_t seed, uint32_t first_filter, int32_t B,
                          int32_t* anc, int64_t ld_anc, int32_t* status);

/* NS-12 sorted-uniform multinomial (variant a6). */
double pfo_dlog(double x);
uint64_t pfo_spacing(uint64_t seed, uint32_t filter_index, int64_t k);
void pfo_spacings(int32_t P, uint64_t seed, uint32_t filter_index, uint64_t* G);
int pfo_resample_sorted_multinomial(const float* logw, int32_t P, uint64_t seed, uint32_t filter_index,
                                    int32_t* anc);

/* NS-3d (reading R-21): binary64 log-weights.  t[P] = fl32(logw_i - lmax) with
 * the binary64 max (NaN everywhere when invalid); returns PFO_FILTER_*. */
int pfo_shift_f64(const double* logw, int32_t P, float* t, double* lmax);
/* The float32 path on t; lse = lmax + ln S.  sorted != 0: the a6 multinomial. */
int pfo_resample_f64(int scheme, int sorted, const double* logw, int32_t P, uint64_t seed, int32_t B,
                     uint32_t filter_index, int32_t* anc, double* lse, float* normw, double* ess);

/* NS-17 (R-14): pre-sorted weights (descending, ties by index), resampled by the
 * float32 path, ancestors mapped back to the original indices.  Prefix-sum schemes. */
int pfo_resample_sorted_weights(int scheme, const float* logw, int32_t P, uint64_t seed, uint32_t filter_index,
                                int32_t* anc, double* lse, float* normw, double* ess);

/* NS-14 / SPEC S:60-77 conversions. */
void pfo_ancestors_to_offspring(const int32_t* anc, int32_t P, int32_t* o);
void pfo_offspring_to_ancestors(const int32_t* o, int32_t P, int32_t* anc);

/* NS-15 canonical in-place permutation. */
void pfo_permute(const int32_t* anc, int32_t P, int32_t* perm);

/* NS-16 gathers (rows of row_bytes, strides in bytes). */
void pfo_gather_inplace(void* X, int64_t row_bytes, int64_t ld_bytes, int32_t P, const int32_t* perm);
void pfo_gather_out(const void* X, void* Y, int64_t row_bytes, int64_t ld_x, int64_t ld_y,
                    int32_t P, const int32_t* anc);

/* P:168-186 Eq. (5) (with Eq. (3) corrected, R11): minimum B. */
int32_t pfo_metropolis_required_B(int64_t P, double w_max, double eps);

#ifdef __cplusplus
}
#endif
#endif
