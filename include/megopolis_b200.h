/*
 * megopolis_b200.h -- C ABI of libmgp.so, the B200 (sm_100a) implementation of the
 * resampling hot path of arXiv 2109.13504 ("The Megopolis Resampler").
 *
 * The reference (pkg/src/megores, "M/" below) is a pure-Python/numba package; its
 * plug-in surface for this path is the Python resampler API
 *     fn(w: WeightVector, b: int, seed) -> np.int64[N]      (M/resample.py:431-455)
 * Each entry point below names the reference interface it replaces.  The Python
 * package paper_2109_13504_b200 binds these with ctypes and mirrors the reference
 * API (names, arguments, defaults, errors); INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - Plain pointers and sizes only.  "d_" pointers are device (HBM) pointers,
 *     "h_" pointers are host pointers (pinned for asynchronous copies).
 *   - stream: a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Device-pointer calls are asynchronous on that stream and run on the calling
 *     thread's current device.
 *   - dtype: MGP_F32 / MGP_F64 weights (the reference's "single" / "double",
 *     M/weights.py:39).  Ancestors and offspring counts are int64 (the reference's
 *     np.int64 results, M/resample.py:128, 368).
 *   - rng: MGP_RNG_MEGORES is the reference's keyed splitmix64 stream
 *     (M/rng.py:85-121), bit-exact with the reference; MGP_RNG_PHILOX is
 *     Philox4x32-10 with the same counter layout.
 *   - Return codes: 0 = ok; MGP_EINVAL (< 0) = invalid argument, the reference's
 *     ValueError (message via mgp_last_error(), same text as the reference);
 *     MGP_EUNSUPPORTED = size/feature outside this build; > 0 = cudaError_t.
 *   - Thread-safe; mgp_last_error() is thread-local.  Scratch is stream-ordered
 *     (cudaMallocFromPoolAsync) from a private per-device cudaMemPool owned by the library;
 *     the device's default pool and the host application's allocator settings are never
 *     touched.  Library-internal caches (the per-device pool, per-thread host-path streams,
 *     the bounded LRU of float32 weight texture objects) sit behind mutexes or are
 *     thread-local.
 *   - partition_bytes counts 4-byte words (n_w = partition_bytes / 4, the reference's
 *     default word_bytes = 4, M/resample.py:64, 84-87); hosts with another word size pass
 *     n_w * 4 (the Python layer's abi_partition_bytes).
 *   - Host buffers: page-locked memory lets the ancestor download overlap the compute
 *     chunk by chunk; pageable memory works too (every chunk kernel is queued first, then
 *     the downloads), at the driver's pageable copy rate.
 *   - Particle counts are limited to N < 2^31 (32-bit index arithmetic on device).
 */
#ifndef MEGOPOLIS_B200_H
#define MEGOPOLIS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MGP_ABI_VERSION 1

enum { MGP_F32 = 0, MGP_F64 = 1 };
enum { MGP_RNG_MEGORES = 0, MGP_RNG_PHILOX = 1 };
enum { MGP_KIND_METROPOLIS = 0, MGP_KIND_C1 = 1, MGP_KIND_C2 = 2, MGP_KIND_MEGOPOLIS = 3 };
/* prefix-sum resamplers (M/resample.py:285-336): b is ignored, rng must be MGP_RNG_MEGORES */
enum { MGP_KIND_MULTINOMIAL = 4, MGP_KIND_SYSTEMATIC = 5 };
enum { MGP_OK = 0, MGP_EINVAL = -1, MGP_EUNSUPPORTED = -2 };

/* flags: MGP_FLAG_NONZERO asserts that no weight is zero (mgp_weight_stats:
 * n_zero == 0), so the both-zero rejection of the acceptance rule
 * (M/resample.py:118-122) can never fire and is compiled out.  Results are
 * identical with or without the flag when it holds. */
enum { MGP_FLAG_NONZERO = 1 };
/* MGP_FLAG_NO_STAGE: C1 reads its partition from global memory instead of staging it in shared
 * memory (a benchmarking knob for SURVEY config 3; results are identical). */
enum { MGP_FLAG_NO_STAGE = 2 };

/* Weight statistics (device-resident result).  sum/mean are bit-identical to
 * numpy's np.asarray(w, float64).sum()/.mean() (pairwise summation), which feeds
 * the B rule at M/bench.py:119-120 and T/conftest.py:29-30. */
typedef struct {
    double sum;
    double mean;
    double max;          /* float64 max (M/bench.py:120) */
    int64_t n_pos;       /* w > 0 and finite           */
    int64_t n_zero;      /* w == 0 (incl. -0.0)        */
    int64_t n_neg;       /* w < 0                      */
    int64_t n_nonfinite; /* inf / nan                  */
    int64_t n_notnormal; /* zero, subnormal, negative or non-finite */
} mgp_weight_stats_t;

int mgp_abi_version(void);
const char *mgp_last_error(void);

/* WeightVector's host-side validation (M/weights.py:53-59) in one parallel pass over host memory
 * (no device work): counts[0..3] = non-finite, negative (finite, < 0; -0.0 is not), zero and
 * positive elements. */
int mgp_check_host_weights(const void *h_w, int dtype, int64_t n, int64_t *counts);

/* Return the library's cached scratch memory on `device` (-1: the current device) to the
 * driver: trims the private stream-ordered pool (cudaMemPoolTrimTo(pool, 0)). */
int mgp_release_cached_memory(int device);

/* Replaces the f64 mean/max scan feeding compute_iterations (M/weights.py:114-131,
 * M/bench.py:119-120) and the WeightVector / _check_weights scans
 * (M/weights.py:49-59, M/resample.py:96-100).  One fused HBM pass. */
int mgp_weight_stats(const void *d_w, int dtype, int64_t n, mgp_weight_stats_t *d_out, void *stream);

/* B = ceil(ln eps / ln(1 - mean/max)), clamped >= 1 (M/weights.py:114-131; same
 * ValueErrors).  Host arithmetic, libm log as the reference's math.log. */
int mgp_compute_iterations(double epsilon, double mean_w, double max_w, int32_t *b_out);

/* megopolis_offsets (M/resample.py:263-265): B offsets on GLOBAL_OFFSET_LANE. */
int mgp_offsets_host(uint64_t seed, int64_t n, int32_t b, int rng, int64_t *h_off);
int mgp_offsets(uint64_t seed, int64_t n, int32_t b, int rng, int64_t *d_off, void *stream);

/* Resamplers (device pointers).  Preconditions are checked like the reference
 * wrappers check them (B >= 1, strict N % W, partition geometry); the
 * data-dependent "all weights are zero" check (M/resample.py:96-100) needs the
 * weight statistics and is done by the caller (the Python package does it) or by
 * mgp_resample_host. */
/* megopolis(w, b, warp, seed, strict)          M/resample.py:268-282 */
int mgp_megopolis(const void *d_w, int dtype, int64_t n, int32_t b, uint64_t seed, int32_t warp, int strict,
                  int rng, int flags, int64_t *d_anc, void *stream);
/* metropolis(w, b, seed)                       M/resample.py:201-206 */
int mgp_metropolis(const void *d_w, int dtype, int64_t n, int32_t b, uint64_t seed, int rng, int flags,
                   int64_t *d_anc, void *stream);
/* metropolis_c1(w, b, part, warp, seed, strict) M/resample.py:209-225; partition_bytes
 * is PartitionConfig.partition_bytes, word size 4 bytes (M/resample.py:64, 84-93) */
int mgp_metropolis_c1(const void *d_w, int dtype, int64_t n, int32_t b, uint64_t seed, int32_t warp,
                      int32_t partition_bytes, int strict, int rng, int flags, int64_t *d_anc, void *stream);
/* metropolis_c2(w, b, part, warp, seed, strict) M/resample.py:228-244 */
int mgp_metropolis_c2(const void *d_w, int dtype, int64_t n, int32_t b, uint64_t seed, int32_t warp,
                      int32_t partition_bytes, int strict, int rng, int flags, int64_t *d_anc, void *stream);

/* Particle slice [p0, p1) of any resampler (sharded multi-GPU / pipelined use):
 * ancestors for particle i land in d_anc_slice[i - p0]; the weights are the full
 * (replicated) array.  For the W = 32 paths p0 must be a multiple of 32. */
int mgp_resample_range(int kind, const void *d_w, int dtype, int64_t n, int32_t b, uint64_t seed, int32_t warp,
                       int32_t partition_bytes, int strict, int rng, int flags, int64_t p0, int64_t p1,
                       int64_t *d_anc_slice, void *stream);

/* Resample AND apply the ancestors in one kernel (apply_ancestors, M/resample.py:371-377, fused):
 * each resampled particle's state row is read directly from its owner h_peer_rows[owner] -- local
 * memory or NVLink-mapped peer memory of the rank that owns the row (sharded particle states).
 * layout 0 (contiguous): particles [p0, p1) into d_anc_out / d_rows_out[i - p0];
 *   owner = anc / rows_local.
 * layout 1 (stripes): particles [p0, p1) and N/2 + [p0, p1) into [L lower | L upper] (as
 *   mgp_resample_stripes); owner r holds [r*h, (r+1)*h) then N/2 + [r*h, (r+1)*h), h = rows_local/2.
 * h_peer_rows: host array of npeers device pointers; rows of row_bytes.  W = 32 resamplers with
 * 4-byte-aligned rows copy the row in the kernel's final store; other shapes run a peer-gather
 * kernel with the same owner mapping afterwards. */
int mgp_resample_gather(int kind, const void *d_w, int dtype, int64_t n, int32_t b, uint64_t seed, int32_t warp,
                        int32_t partition_bytes, int strict, int rng, int flags, int layout, int64_t p0, int64_t p1,
                        const void *const *h_peer_rows, int npeers, int64_t rows_local, int64_t row_bytes,
                        int64_t *d_anc_out, void *d_rows_out, void *stream);

/* Single-process multi-device resample from host buffers (SURVEY 8b mgp_megopolis_multi; for C hosts
 * without torch.distributed).  The weights (host, n elements) are replicated to devs[0..ndev)
 * (device-to-device copies peer to peer), B comes from the numpy-exact stats on devs[0] (b <= 0:
 * the epsilon rule; *b_used receives it), and device d resamples stripe d of each half (contiguous
 * slices when N does not split into 32-aligned stripes), writing into h_anc[n].  Same results as
 * the single-device call; a device may appear more than once in devs. */
int mgp_resample_multi(int kind, const void *h_w, int dtype, int64_t n, int32_t b, double epsilon, uint64_t seed,
                       int32_t warp, int32_t partition_bytes, int strict, int rng, int ndev, const int *devs,
                       int64_t *h_anc, int32_t *b_used);

/* Two-stripe particle range: particles [lo0, lo1) and [N/2 + lo0, N/2 + lo1) (0 <= lo0 <= lo1
 * <= N/2, N even) into d_anc_local[0, L) and d_anc_local[L, 2L), L = lo1 - lo0.  This is the
 * sharded "stripes" layout (rank r owns stripe r of each half), under which every rank can run
 * the half-split Megopolis kernel. */
int mgp_resample_stripes(int kind, const void *d_w, int dtype, int64_t n, int32_t b, uint64_t seed, int32_t warp,
                         int32_t partition_bytes, int strict, int rng, int flags, int64_t lo0, int64_t lo1,
                         int64_t *d_anc_local, void *stream);

/* Host-buffer drop-in for make_resampler(kind, ...)(w, b, seed) (M/resample.py:431-455):
 * copies h_w to the device, validates (WeightVector + _check_weights), derives B
 * from epsilon when b <= 0 (reporting it in *b_used), resamples, and streams the
 * ancestors back into h_anc overlapped with the remaining compute.  device: the CUDA device
 * to run on (-1: the calling thread's current device, which is left unchanged either way). */
int mgp_resample_host(int kind, const void *h_w, int dtype, int64_t n, int32_t b, double epsilon, uint64_t seed,
                      int32_t warp, int32_t partition_bytes, int strict, int rng, int64_t *h_anc, int32_t *b_used,
                      int device);

/* Independent resamples of `count` host weight vectors of n elements (h_w[k] -> h_anc[k], seeds[k];
 * b <= 0: each job's B from epsilon, reported in b_used[k]), pipelined over two device buffer slots:
 * job k+1's upload and statistics and job k-1's download overlap job k's kernel.  Same ancestors
 * as `count` calls of mgp_resample_host.  The overlap needs page-locked host buffers (pageable ones
 * are correct, their copies synchronous).  Output buffers may repeat every other job. */
int mgp_resample_host_batch(int kind, const void *const *h_w, int dtype, int64_t n, int32_t count, int32_t b,
                            double epsilon, const uint64_t *seeds, int32_t warp, int32_t partition_bytes, int strict,
                            int rng, int64_t *const *h_anc, int32_t *b_used, int device);

/* ancestors_to_offspring (M/resample.py:361-368): d_counts[j] = #{i : anc[i] == j};
 * *d_bad set to 1 if an ancestor is outside [0, n) (the reference's ValueError). */
int mgp_offspring(const int64_t *d_anc, int64_t n_anc, int64_t n, int64_t *d_counts, int32_t *d_bad,
                  void *stream);

/* QualityAccumulator (M/metrics.py:55-110), float64, bit-identical to numpy:
 *   expected:  d_e = N * w / sum(w)              (_expected_offspring, :55-60)
 *   add:       sum += o; sum_sq += o*o; se_total += sum((o - e)^2)      (:86-93)
 *   finalize:  variance = sum(sum_sq/k - mean^2), bias_sq = sum((mean - e)^2) (:95-110) */
int mgp_expected_offspring(const void *d_w, int dtype, int64_t n, double *d_e, double *d_total, void *stream);
/* _expected_offspring for a slice of a sharded population: d_e = n_all * w / total over the
 * n_slice local weights, total = the global float64 sum (numpy order) computed elsewhere. */
int mgp_expected_offspring_slice(const void *d_w, int dtype, int64_t n_slice, int64_t n_all, double total,
                                 double *d_e, void *stream);
int mgp_quality_add(const int64_t *d_counts, const double *d_e, int64_t n, double *d_sum, double *d_sumsq,
                    double *d_se_total, double *d_se_run, void *stream);
int mgp_quality_finalize(const double *d_sum, const double *d_sumsq, const double *d_e, int64_t n, int64_t k,
                         double *d_variance, double *d_bias_sq, void *stream);
/* K runs of a resampler accumulated on the device (the inner loop of the quality grids,
 * M/bench.py:121-126): for each h_seeds[r]: ancestors = kind(w, b, seed) -> offspring ->
 * QualityAccumulator.add into d_sum / d_sumsq / *d_se_total (d_e from mgp_expected_offspring).
 * Same results as K separate calls, without a host round trip per run. */
int mgp_quality_runs(int kind, const void *d_w, int dtype, int64_t n, int32_t b, const uint64_t *h_seeds, int32_t k,
                     int32_t warp, int32_t partition_bytes, int strict, int rng, int flags, const double *d_e,
                     double *d_sum, double *d_sumsq, double *d_se_total, void *stream);
/* squared_error (M/metrics.py:63-68) for one offspring vector */
int mgp_squared_error(const int64_t *d_counts, const double *d_e, int64_t n, double *d_out, void *stream);

/* apply_ancestors (M/resample.py:371-377): out[i] = states[anc[i]], rows of row_bytes */
int mgp_gather(const void *d_states, int64_t row_bytes, const int64_t *d_anc, int64_t n, void *d_out, void *stream);

/* Sharded apply_ancestors over peer memory: rank r owns rows [r*n_local, (r+1)*n_local)
 * at peer_states[r] (device pointers valid on the calling device: NVLink P2P /
 * symmetric-memory mappings); out[i] = row anc[i] read directly from its owner. */
int mgp_gather_peers(const void *const *peer_states, int npeers, int64_t n_local, int64_t row_bytes,
                     const int64_t *d_anc, int64_t n, void *d_out, void *stream);

/* Comparison-index replay (comparison_indices, M/resample.py:384-428): d_out[r * n + i] = the
 * weight index particle i reads at round r, for kind 0-3, reference (megores) stream; B x N int64.
 * word_bytes is WarpConfig.word_bytes (the C1/C2 partition width is partition_bytes / word_bytes). */
int mgp_comparison_indices(int kind, int64_t n, int32_t b, uint64_t seed, int32_t warp, int32_t partition_bytes,
                           int32_t word_bytes, int64_t *d_out, void *stream);
/* The warp transaction model (traffic_report, M/warpsim.py:94-111) over a rows x width trace of
 * word indices, groups of `warp` consecutive entries of a row: d_out[0] = total transactions
 * (distinct aligned segments per group, summed), d_out[1] = the largest per-group count,
 * d_out[2] = unnecessary words (segments * words_per_segment - distinct words, summed). */
int mgp_traffic_report(const int64_t *d_idx, int64_t rows, int64_t width, int32_t warp, int32_t word_bytes,
                       int32_t segment_bytes, int64_t *d_out, void *stream);

/* Peer mappings for the two entry points above (CUDA IPC; no reference counterpart -- the
 * reference is single-process).  mgp_ipc_export: the 64-byte cudaIpcMemHandle_t of the
 * allocation holding d_ptr and d_ptr's offset in it.  mgp_ipc_open (in another process,
 * any device with peer access): the mapped pointer to the same bytes, peer access enabled
 * lazily.  mgp_ipc_close(mapped pointer, offset) unmaps.  The exporting process keeps
 * the allocation alive while it is mapped. */
int mgp_ipc_export(const void *d_ptr, void *handle_out, int64_t *offset_out);
int mgp_ipc_open(const void *handle, int64_t offset, void **d_ptr_out);
int mgp_ipc_close(void *d_ptr, int64_t offset);

/* np.mean of a float64 / float32 vector (numpy pairwise order), e.g. the filter estimate
 * (M/pfilter.py:162). */
int mgp_mean(const void *d_x, int dtype, int64_t n, double *d_out, void *stream);

/* SIR particle filter stages (M/pfilter.py:129-165), float64:
 *   mgp_pf_init: x_i = gaussian_at(seed, i, 0) * sqrt(process_var)          (init_state)
 *   mgp_pf_predict_update: noise = gaussian_at(seed, i, 0) * sqrt(process_var);
 *     x' = transition(x, t, noise) with cos_term = 8 cos(1.2 t) (M/pfilter.py:86-89);
 *     w = max(likelihood(z, x', obs_var), tiny) cast to dtype (M/pfilter.py:92-103);
 *     *d_any_pos |= 1 if any weight is > 0 (nullable; the resampler's all-zero check,
 *     M/resample.py:96-100, without a host round trip). */
int mgp_pf_init(int64_t n, uint64_t seed, double sqrt_process_var, double *d_x, void *stream);
int mgp_pf_predict_update(const double *d_x, int64_t n, double cos_term, double sqrt_process_var, uint64_t seed,
                          double z, double obs_var, int dtype, double *d_xpred, void *d_w, int32_t *d_any_pos,
                          void *stream);

/* estimate_ratio (M/weights.py:134-154) statistics: d_out = {mean, max} (float64) of the
 * subset formed by the first `subset` entries of the stable argsort of uniform01_at(seed, i, 0)
 * (the full array when subset == n).  ratio = mean / max is formed by the caller. */
int mgp_estimate_ratio_stats(const void *d_w, int dtype, int64_t n, int64_t subset, uint64_t seed, double *d_out,
                             void *stream);

/* gen_gaussian_weights (M/weights.py:100-104) on the device (synthetic inputs) */
int mgp_gen_gaussian(double y, int64_t n, uint64_t seed, int dtype, void *d_out, void *stream);

/* gen_gamma_weights (M/weights.py:107-111): d_out[i] = scipy.stats.gamma.ppf(u_i, a=alpha,
 * scale=1/beta) with u_i = uniform_open01_at(seed, i, 0) (M/rng.py:134-137), evaluated in HBM
 * (incomplete-gamma inversion in float64, ~1e-14 relative to scipy; not bit-exact). */
int mgp_gen_gamma(double alpha, double beta, int64_t n, uint64_t seed, int dtype, void *d_out, void *stream);

/* Prefix-sum resamplers (M/resample.py:285-336).  mgp_cumsum is np.cumsum(values) in the
 * weights' dtype (M/resample.py:288-291) -- numpy's sequential left-to-right rounding,
 * reproduced bit for bit by a parallel exact scan.
 *   multinomial(w, seed)          M/resample.py:295-304
 *   systematic_improved(w, seed)  M/resample.py:307-336
 * Also reachable as kinds MGP_KIND_MULTINOMIAL / MGP_KIND_SYSTEMATIC of mgp_resample_range
 * and mgp_resample_host (b ignored). */
int mgp_cumsum(const void *d_w, int dtype, int64_t n, void *d_out, void *stream);
int mgp_multinomial(const void *d_w, int dtype, int64_t n, uint64_t seed, int64_t *d_anc, void *stream);
int mgp_systematic(const void *d_w, int dtype, int64_t n, uint64_t seed, int64_t *d_anc, void *stream);

/* systematic_oracle(w, u) (M/resample.py:339-354) for an explicit u in [0, 1): the reference's
 * sequential stratified selection, with its comparison semantics (float32 weights compare in
 * float32 against float32(target), NumPy 2 weak-scalar promotion). */
int mgp_systematic_oracle(const void *d_w, int dtype, int64_t n, double u, int64_t *d_anc, void *stream);

/* Self-check: our Philox4x32-10 vs curand_Philox4x32_10 for counters {i, c1, c2, c3}.
 * Writes 4*n words each; returns the number of mismatching words in *h_mismatch. */
int mgp_philox_selftest(uint64_t key, uint32_t c1, uint32_t c2, uint32_t c3, int64_t n, int64_t *h_mismatch);

/* Diagnostic: the number of particles whose megores-stream float32 decision bracket (Megopolis,
 * Metropolis-C1 and -C2 on float32 weights) was ambiguous in some round and that were re-run with
 * the exact float64 rule (the current device, since the last reset).  reset != 0 zeroes the
 * counter after reading it. */
int mgp_debug_megores_fallbacks(int64_t *h_count, int reset);
/* Exact-cumsum resolver profile (16 counters; non-zero only in a -DMGP_PX_PROF build of the
 * library, scripts/mb/px_prof.sh): super windows, chunk windows, crossing chunks, block passes,
 * sequential tails and their cycles. */
int mgp_debug_px_prof(int64_t *h_out16, int reset);

/* Measurement switch for mgp_offspring: 0 = the queued shared-memory histogram (default), 1 = the
 * int32 global-atomic histogram (round 1), 2 = the count-matrix bucketed histogram.  Process-wide;
 * for A/B timing and tests only. */
int mgp_debug_offspring_mode(int mode);

#ifdef __cplusplus
}
#endif
#endif /* MEGOPOLIS_B200_H */
