/*
 * kmedoids.h -- C ABI of the B200-native FastPAM SWAP library (libkmedoids.so).
 *
 * The problem: given a dissimilarity matrix D
 * and k, find k medoids M, the assignment of every object to its nearest
 * medoid, and the total deviation TD = sum_o min_j d(x_o, m_j) (Eq. eqn:td,
 * P:112-118).  The library implements PAM BUILD (Alg.1), the
 * FastPAM1 SWAP iteration (Alg.3, Eq. eqn:better-change3
 * P:797-837) and the FastPAM2 multi-swap iteration (P:861-862, P:945-947,
 * DESIGN.md reading R6) on one B200 or on a column-sharded set of B200s.
 *
 * Conventions that hold for every entry point:
 *  - d(x_o, x_c) = D[o][c]: row = object o, column = medoid/candidate c
 *    (reading R0).  D needs no symmetry and no triangle inequality
 *     but must be >= 0 with d(x,x) = 0 on the diagonal.
 *  - D is BORROWED: device memory owned by the caller, alive and unmodified
 *    for the handle's lifetime.  The library never frees it.  Row stride
 *    `ld` (elements) must be a multiple of 4 and D 16-byte aligned (128-bit
 *    loads).  Element (o, c) of the local slab is D[o*ld + (c - col_begin)].
 *  - Sharding: rank r of R holds the column slab [col_begin, col_end) of all
 *    n rows (candidates are columns).  A single GPU has col_begin = 0,
 *    col_end = n.  Sharded runs are driven through the phase entry points
 *    below; every rank calls every function with the same arguments.
 *  - Medoids live in k slots; a swap replaces slot i in place.
 *    assignment[o] is the slot of o's nearest medoid; ties go to the smaller
 *    slot (reading R2).  The best swap is the lexicographic minimum of
 *    (dTD, slot, candidate) (reading R1).
 *  - TD / dTD values are int64 for KM_U32 inputs (exact) and double for
 *    KM_F32 inputs (fp64 sums of f32 values); `td_out` points to an int64_t
 *    or a double accordingly.  A swap is accepted iff dTD < 0 (U32) or
 *    dTD < -1e-12*|TD| (F32, reading R5).
 *  - Errors: every function returns a km_status; nothing is thrown.
 *    kmedoids_last_error() returns a thread-local description of the last
 *    failure.  KM_ECUDA leaves the handle unusable (destroy it).
 *  - All work is enqueued on the handle's CUDA stream; functions that return
 *    host values synchronise that stream before returning.
 */
#ifndef KMEDOIDS_H
#define KMEDOIDS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    KM_OK = 0,
    KM_CONVERGED = 1,      /* not an error: the best dTD does not improve (Alg.2) */
    KM_NOT_CONVERGED = 2,  /* max_iter passes ran without convergence */
    KM_EINVAL = 10,        /* bad argument (sizes, duplicate/out-of-range medoids, alignment, state) */
    KM_ENOMEM = 11,        /* device or host allocation failed */
    KM_ECUDA = 12,         /* a CUDA call failed; the handle must be destroyed */
    KM_ECOMM = 13          /* the sharded exchange was used inconsistently */
} km_status;

typedef enum { KM_U32 = 0, KM_F32 = 1 } km_dtype;
/* KM_FASTERPAM: FasterPAM's eager swapping (Alg.4; readings
 * F1-F5 in DESIGN.md), evaluated exactly on the GPU by speculative candidate
 * batches. */
/* KM_FASTPAM1_INC: the same swaps as KM_FASTPAM1 (Alg.3's best swap per
 * iteration, reading R1; bit-exact on U32), computed incrementally: the
 * k-vectors of every candidate are kept (one FastPAM2-mode stream of D) and
 * corrected after each swap from the rows of the objects whose nearest /
 * second changed, instead of re-streaming D (DESIGN.md "incremental
 * FastPAM1"; extra device memory k*n*8 bytes).  Single GPU. */
typedef enum { KM_FASTPAM1 = 0, KM_FASTPAM2 = 1, KM_FASTERPAM = 2, KM_FASTPAM1_INC = 3 } km_variant;

typedef struct km_handle km_handle;  /* opaque; owns only its scratch buffers */

/* Create a handle over the borrowed device slab D (see conventions).
 *   n: number of objects (rows), 3 <= n < 2^31;  k: medoids, 2 <= k < n
 *   (BUILD also allows k = 1 through kmedoids_init_build);
 *   cuda_stream: a cudaStream_t (NULL = legacy default stream).
 * Allocates O(k*n + n*P) bytes of device scratch (P = internal row parts).
 * Errors: KM_EINVAL for bad sizes/alignment, KM_ENOMEM, KM_ECUDA. */
km_status kmedoids_create(km_handle** out, const void* D, km_dtype dtype, int64_t n, int64_t ld,
                          int64_t col_begin, int64_t col_end, int32_t k, void* cuda_stream);

/* Release the handle's scratch (never D).  Safe on NULL. */
km_status kmedoids_destroy(km_handle* h);

/* Thread-local message describing the last non-OK status ("" if none). */
const char* kmedoids_last_error(void);

/* Set the k initial medoids (host array, distinct point indices in [0, n),
 * slot order) and compute the nearest/second cache (Alg.3) and TD.
 * Single GPU only; a sharded handle uses kmedoids_shard_set_medoids.
 * Errors: KM_EINVAL for duplicates / out of range. */
km_status kmedoids_set_medoids(km_handle* h, const int32_t* medoids);

/* Declare D exactly symmetric (symmetric = 1): d(x_o, x_c) == d(x_c, x_o)
 * bitwise for all o, c < n -- true of every metric dissimilarity matrix.
 * Verified by one tiled pass over D (KM_EINVAL and the flag stays off if any
 * pair differs).  With it, the FastPAM2 sequential phase reads candidate c's
 * distances as row c (4n contiguous bytes) instead of the strided column
 * (n separate sectors); results are unchanged.  symmetric = 0 turns it off.
 * Single GPU only (a column slab holds no whole rows: KM_EINVAL). */
km_status kmedoids_set_symmetric(km_handle* h, int32_t symmetric);

/* PAM BUILD (Alg.1; readings R3/R4) on the device; leaves the
 * handle ready for SWAP.  medoids_out (host, k entries) and td_out
 * (int64_t* or double*) may be NULL.  Single GPU only (sharded BUILD is
 * driven through kmedoids_build_step*). */
km_status kmedoids_init_build(km_handle* h, int32_t* medoids_out, void* td_out);

/* NEXT-4 initialisations, single GPU.  Random numbers are
 * caller inputs (the oracle uses the same), so runs are reproducible.
 *  kmedoids_init_weighted: distance-weighted seeding ("k-means++" adapted to
 *    arbitrary dissimilarities; reading I1).  u: host
 *    array of k uniforms in [0, 1): seed 0 = floor(u[0] n); seed i = the first
 *    object whose running sum of w(o) = min_j d(x_o, m_j) exceeds u[i] * W.
 *  kmedoids_init_lab: LAB (reading I2).  seq: host array of k
 *    rows of (s + k) indices in [0, n) or -1 (padding), distinct per row;
 *    step i samples the first s non-medoids of row i and takes BUILD's choice
 *    on that sample (s = 10 + ceil(sqrt(n))).
 * Both leave the handle ready for SWAP (cache and TD as kmedoids_set_medoids);
 * medoids_out[k] / td_out may be NULL.  Errors: KM_EINVAL (k < 2, u outside
 * [0, 1), s outside [1, n], indices out of range, sharded handle). */
km_status kmedoids_init_weighted(km_handle* h, const double* u, int32_t* medoids_out, void* td_out);
km_status kmedoids_init_lab(km_handle* h, int32_t s, const int32_t* seq, int32_t* medoids_out, void* td_out);

/* NEXT-3 FastCLARA (reading C1), single GPU.  For each
 * of the nsamples caller-drawn samples (host array samples[nsamples][s] of
 * distinct indices in [0, n); P:1122 suggests s = 80 + 4k): PAM on the s x s
 * sub-matrix (BUILD, then SWAP with `variant` to convergence), medoids mapped
 * back to point indices, TD over all n objects; the sample with the smallest
 * (TD, sample index) wins.  The handle is left on the winning medoids (cache,
 * TD); medoids_out[k], td_out, best_sample_out may be NULL.  Scratch: s x s
 * sub-matrix + one nested handle (allocated on first use; s fixed per handle).
 * Errors: KM_EINVAL (s <= k or s > n, bad or duplicate indices, sharded). */
km_status kmedoids_clara(km_handle* h, int32_t nsamples, int32_t s, const int32_t* samples, km_variant variant,
                         int32_t* medoids_out, void* td_out, int32_t* best_sample_out);

/* One SWAP iteration (FastPAM1: Alg.3; FastPAM2: reading R6;
 * FasterPAM: one pass of Alg.4's candidate scan) from the
 * current state.  *swaps_done_out (may be NULL) receives the number of
 * swaps applied (0 or 1 for FastPAM1, 0..k for FastPAM2, 0..n-k for a
 * FasterPAM pass); *td_out the TD after the iteration.  Returns KM_CONVERGED
 * when no swap improves (FasterPAM: when n consecutive scan positions
 * passed without a swap, reading F2; a pass that ends that way returns
 * KM_CONVERGED, and later calls return KM_CONVERGED without work).
 * Single GPU only. */
km_status kmedoids_swap_iter(km_handle* h, km_variant variant, int32_t* swaps_done_out, void* td_out);

/* Up to `count` FastPAM1 iterations (Alg.3), each exactly one
 * kmedoids_swap_iter(KM_FASTPAM1), enqueued back to back: the next iteration
 * is queued on the device while the host reads the outcome of the current one
 * (a pass without an improving swap makes every pass queued behind it a
 * no-op), so no host round trip separates iterations.  Stops after the first
 * non-improving pass (counted).  iters_out / swaps_out: passes
 * and swaps done by this call; td_out (int64_t* or double*) the TD after
 * them; any may be NULL.  Returns KM_CONVERGED if the last pass made no swap,
 * else KM_OK.  kmedoids_run uses the same path for KM_FASTPAM1.  Single GPU. */
km_status kmedoids_swap_iters(km_handle* h, int32_t count, int32_t* iters_out, int32_t* swaps_out, void* td_out);
/* The same for KM_FASTPAM2 (reading R6) as well as
 * KM_FASTPAM1: up to `count` iterations, each exactly one
 * kmedoids_swap_iter(variant), the next queued on the device while the host
 * reads the current one's outcome from pinned memory; a FastPAM2 pass with no
 * improving slot sets a sticky flag, so passes queued behind it plan, swap and
 * count nothing.  Outputs and return value as kmedoids_swap_iters;
 * kmedoids_run uses this path for both variants.  Errors: KM_EINVAL (count
 * < 1, another variant, no medoids, sharded handle), KM_ECUDA.  Single GPU. */
km_status kmedoids_swap_iters_variant(km_handle* h, km_variant variant, int32_t count, int32_t* iters_out,
                                      int32_t* swaps_out, void* td_out);

/* BUILD (if use_build) or the medoids already set, then SWAP iterations until
 * convergence or max_iter passes (max_iter <= 0 means 2000).  Outputs are
 * host arrays (any may be NULL): medoids_out[k], assignment_out[n] (slot of
 * the nearest medoid), td_out, n_iter_out (passes including the final
 * non-improving one), n_swaps_out.
 * Returns KM_OK (converged) or KM_NOT_CONVERGED.  Single GPU only. */
km_status kmedoids_run(km_handle* h, int32_t use_build, km_variant variant, int32_t max_iter,
                       int32_t* medoids_out, int32_t* assignment_out, void* td_out,
                       int32_t* n_iter_out, int32_t* n_swaps_out);

/* Whole job from HOST memory: copies D_host (n x n, row stride ld elements,
 * preferably pinned) to a device buffer the call allocates and frees, then
 * behaves as kmedoids_run (use_build, variant, max_iter as there).
 * initial_medoids (host, k) is used when use_build == 0.  Outputs are host
 * arrays as in kmedoids_run.  Everything (H2D, BUILD, SWAP, D2H) runs on
 * cuda_stream. */
km_status kmedoids_run_host(const void* D_host, km_dtype dtype, int64_t n, int64_t ld, int32_t k,
                            int32_t use_build, const int32_t* initial_medoids, km_variant variant,
                            int32_t max_iter, void* cuda_stream, int32_t* medoids_out,
                            int32_t* assignment_out, void* td_out, int32_t* n_iter_out,
                            int32_t* n_swaps_out);

/* kmedoids_run_host keeps its device copy of D between calls (one buffer per
 * process, reused while large enough, so repeated jobs pay no allocation),
 * and kmedoids_clara_points its per-sample scratch; this frees both.  Safe to call at any time from any thread; KM_OK if there
 * was nothing to free. */
km_status kmedoids_release_host_cache(void);

/* Copy the current state to host arrays (any may be NULL): medoids[k],
 * assignment[n], td, counters.  Synchronises the stream. */
km_status kmedoids_get_state(km_handle* h, int32_t* medoids_out, int32_t* assignment_out, void* td_out,
                             int32_t* n_iter_out, int32_t* n_swaps_out);

/* Copy the nearest/second cache to host: nearest[n], second[n] (slots),
 * dn[n], ds[n] (in D's element type).  Any may be NULL. */
km_status kmedoids_get_cache(km_handle* h, int32_t* nearest_out, int32_t* second_out, void* dn_out,
                             void* ds_out);

/* Diagnostics for parity tests: after kmedoids_eval_candidates, copies the
 * per-candidate result of the last FastPAM1 evaluation for the local columns
 * [col_begin, col_end): dtd[c] = min_i dTD(m_i, x_c) (int64/double), slot[c]
 * = its lexicographic argmin slot; medoid columns get slot -1. */
km_status kmedoids_eval_candidates(km_handle* h, void* dtd_out, int32_t* slot_out);

/* The swaps applied by the last kmedoids_swap_iter call, in application
 * order: slots_out[j], cands_out[j] (global point index) and dtds_out[j]
 * (int64_t / double) for j < min(*count_out, cap).  Any output may be NULL. */
km_status kmedoids_last_swaps(km_handle* h, int32_t* slots_out, int32_t* cands_out, void* dtds_out, int32_t cap,
                              int32_t* count_out);

/* Diagnostics of the last KM_FASTPAM2 iteration (reading R6, P:861-862,
 * P:945-947): v_out[k] (int64_t or double) and c_out[k] = the per-slot best
 * (v_i, c_i) = lexicographic min over non-medoid c of (dTD(m_i, x_c), c)
 * (c_i = -1, v_i = 0 if the slot had no candidate); order_out (capacity k)
 * receives the m_out improving slots in ascending (v_i, i), the order the
 * sequential phase visits them.  Any output may be NULL.  Synchronises the
 * handle's stream.  Errors: KM_EINVAL before the first FastPAM2 iteration. */
km_status kmedoids_fp2_last_plan(km_handle* h, void* v_out, int32_t* c_out, int32_t* order_out, int32_t* m_out);

/* Profiling: enable (1) / disable (0) CUDA-event timing of the SWAP-delta
 * stream kernel on the handle's stream; kmedoids_stream_time returns the
 * accumulated milliseconds and launch count since the last reset. */
km_status kmedoids_set_profiling(km_handle* h, int32_t enable);
km_status kmedoids_stream_time(km_handle* h, double* ms_out, int64_t* launches_out, int32_t reset);

/* Number of CUDA kernel launches this handle has issued (all kernels). */
/* Name of the SWAP-delta stream kernel this handle launches (static string;
 * measurement/reporting aid). */
km_status kmedoids_stream_kernel(km_handle* h, const char** name_out);
km_status kmedoids_launch_count(km_handle* h, int64_t* count_out);

/* ---------------- dissimilarity materialisation -----
 * The dissimilarity matrix the method starts from ("computed in
 * advance"; its cost dominates FasterPAM on MNIST), written
 * directly in the layout a handle borrows: the column slab
 * [col_begin, col_end) of all n rows, D[o*ld + (c - col_begin)].
 *   KM_METRIC_L2_F32: X float32 (n x d, row-major, device), D float32,
 *     d(x, y) = sqrt(max(0, |x|^2 + |y|^2 - 2 <x, y>)), inner products on the
 *     tensor cores (tcgen05, tf32 hi/lo split: ~f32 accuracy), d <= 64,
 *     D 16-byte aligned, ld % 4 == 0.  Diagonal exactly 0.  The points are
 *     centred on their mean first (mu).  Accuracy: the squared distance is
 *     within ~(6d + 16) 2^-24 (|x - mu|^2 + |y - mu|^2) of the exact one --
 *     relative errors up to ~3e-4 on the closest (within-cluster) pairs of
 *     the config recipes, where the expansion cancels (the tensor cores'
 *     fp32 accumulation).
 *   KM_METRIC_L2_F32_EXACT: as KM_METRIC_L2_F32, plus every pair with
 *     d^2 < (|x - mu|^2 + |y - mu|^2) / 16 recomputed in the epilogue from
 *     the points by the definition (f32 differences, fp32 accumulation,
 *     correctly rounded sqrt: relative error <= (d + 2) 2^-24 on d^2).
 *     Measured on the C2-C4 recipes: every pair within 1e-5 relative of the
 *     fp64 definition; cost ~2x the plain L2 at C4 (1.2 % of the pairs
 *     recomputed).
 *   KM_METRIC_L1_U32: X int32 integer coordinates (n x d), D uint32,
 *     d(x, y) = sum_t |x_t - y_t| exactly (caller keeps sums < 2^32).  The
 *     arithmetic is chosen on the device from the coordinate ranges, always
 *     exact: packed 16-bit (every range < 2^16), fp32 (sum of ranges < 2^24)
 *     or 32-bit integer; KM_DIST_L1=int / f32 restricts the choice (tests).
 * Asynchronous on cuda_stream (it never waits for the GPU); X and D are
 * borrowed; the library keeps one grow-only scratch buffer per device,
 * ordered across streams by an event.  Errors: KM_EINVAL (sizes,
 * alignment, d > 64 for L2), KM_ENOMEM, KM_ECUDA. */
typedef enum { KM_METRIC_L2_F32 = 0, KM_METRIC_L1_U32 = 1, KM_METRIC_L2_F32_EXACT = 2 } km_metric;
km_status kmedoids_dissimilarity(const void* X, km_metric metric, int64_t n, int32_t d, void* D, int64_t ld,
                                 int64_t col_begin, int64_t col_end, void* cuda_stream);

/* NEXT-3 FastCLARA from points, without the n x n matrix ("the
 * remaining objects are assigned to their closest medoid", P:1109-1129,
 * P:618-620; reading C2), single GPU.  X (device, n x d row-major,
 * 1 <= d <= 128): float32 coordinates for KM_METRIC_L2_F32, int32 for
 * KM_METRIC_L1_U32.  For each of the nsamples caller-drawn samples (host
 * samples[nsamples][s], distinct indices in [0, n), k < s <= n
 * suggests s = 80 + 4k): the s x s dissimilarity matrix of the sample's
 * points by the definitions (L2: fp64 sums, sqrt, rounded to float32; L1:
 * exact, stored as uint32), PAM on it (BUILD, then SWAP with `variant` to
 * convergence), medoids mapped back to point indices, and TD over ALL n
 * objects with every distance recomputed from the points the same way (L2:
 * double of the float32 distance; L1 int64).  The smallest (TD, sample
 * index) wins.  Outputs (host, each may be NULL): medoids_out[k],
 * td_out (double* for L2, int64_t* for L1), best_sample_out, assignment_out[n]
 * (slot of each object's closest winning medoid, smallest slot on ties).
 * Device memory: O(8 s^2 + n) scratch (up to 8 s x s buffers and nested
 * handles), kept between calls with the same (device, s, k, n) so later
 * samples replay each nested BUILD from its CUDA graph; freed by
 * kmedoids_release_host_cache.
 * Samples run concurrently (up to 8, each on its own stream); X must stay
 * unchanged during the call, which synchronises cuda_stream first.
 * Errors: KM_EINVAL (sizes, bad or duplicate indices, metric), KM_ENOMEM,
 * KM_ECUDA. */
km_status kmedoids_clara_points(const void* X, km_metric metric, int64_t n, int32_t d, int32_t k, int32_t nsamples,
                                int32_t s, const int32_t* samples, km_variant variant, void* cuda_stream,
                                int32_t* medoids_out, void* td_out, int32_t* best_sample_out,
                                int32_t* assignment_out);

/* ---------------- sharded (column-slab) phase API ----------------------
 * A sharded SWAP iteration on R ranks is, on every rank:
 *   1. kmedoids_shard_eval(h)          local candidates -> 16-byte record
 *   2. all-gather the records          (caller, e.g. NCCL over NVLink)
 *   3. kmedoids_shard_select(h, ...)   lexicographic reduce of the R records
 *   4. if *found: the owner rank (*owner) packs column c* with
 *      kmedoids_shard_pack_column, the caller broadcasts the n-element
 *      column buffer from *owner, and every rank calls
 *      kmedoids_shard_apply(h) (update M, TD and the nearest/second cache).
 * Buffers are device memory owned by the handle; the caller moves bytes
 * between them.  BUILD follows the same pattern with the build_* calls. */
typedef struct {
    void* record_send;     /* this rank's record (record_bytes) */
    void* record_recv;     /* R records, rank order (R*record_bytes), filled by the caller */
    size_t record_bytes;
    void* column;          /* n elements of D's type: column c* (owner packs, others receive) */
    size_t column_bytes;
} km_exchange;

km_status kmedoids_shard_exchange(km_handle* h, int32_t nranks, km_exchange* out);
/* Set the medoids on a sharded handle; columns[j*n + o] = d(x_o, m_j) must
 * be provided by the caller (device, k*n elements), gathered from owners. */
km_status kmedoids_shard_set_medoids(km_handle* h, const int32_t* medoids, const void* columns_dev);
km_status kmedoids_shard_eval(km_handle* h);
/* Reads the R gathered records; writes (host) *found (1 if an improving
 * swap exists), *slot, *cand (global index), *owner (rank owning cand given
 * the column ranges passed to kmedoids_shard_exchange... computed from
 * rank_col_begin[R+1], the column boundaries of all ranks), *dtd (int64_t*
 * or double*).  Returns KM_CONVERGED when nothing improves. */
km_status kmedoids_shard_select(km_handle* h, const int64_t* rank_col_begin, int32_t* found, int32_t* slot,
                                int32_t* cand, int32_t* owner, void* dtd);
/* The owner of point `cand` (col_begin <= cand < col_end) copies column
 * d(., x_cand) into the exchange column buffer (n elements). */
km_status kmedoids_shard_pack_column(km_handle* h, int32_t cand);
km_status kmedoids_shard_apply(km_handle* h);

/* Device-decided sharded FastPAM1 iteration (Alg.3 P:874-904 over column
 * slabs, readings R1/R5), with no host round trip inside an iteration:
 *   1. kmedoids_shard_eval(h)            local candidates -> 16-byte record
 *   2. all-gather the R records          (caller)
 *   3. kmedoids_shard_decide(h)          lexicographic min of the records on the
 *      device (M, TD, the decision); the rank owning c* copies column c* into
 *      the exchange column buffer, every other rank writes zeros
 *   4. SUM all-reduce of the column buffers (caller; elements of D's type --
 *      float32 or the uint32 bits as int32: x + 0 = x exactly)
 *   5. kmedoids_shard_apply_async(h)     MC, nearest/second cache
 * All five are asynchronous on the handle's stream.  The decision is sticky:
 * once an iteration finds no improving swap, later iterations change nothing
 * and are not counted, so a caller may keep iterations queued ahead of the
 * one it inspects.  kmedoids_shard_status reads the run's status (pinned
 * mirror written by step 3): *converged, *n_iter (the converging iteration
 * included, as P:1390-1392), *n_swaps, *td (int64_t* or double*) as of a
 * definite iteration, so every rank reads the same status: wait = 1 after
 * all enqueued work (the last iteration), 2 after the iteration before the
 * most recently enqueued one (blocks only until that one is done), 0 no
 * synchronisation (the last iteration's copy if already written, else an
 * older one -- a hint, not for collective decisions).  kmedoids_shard_trace copies the applied
 * swaps of the run (slot, candidate, dTD; up to 4096 recorded) to host
 * arrays of cap entries, *count = swaps of the run.  The status restarts at
 * kmedoids_shard_set_medoids and at the end of a sharded BUILD.  Errors:
 * KM_ECOMM before kmedoids_shard_exchange, KM_EINVAL (wait), KM_ECUDA. */
/* The same for a sharded BUILD step (Alg.1, reading R3):
 * kmedoids_build_eval(h, step), all-gather the records, kmedoids_build_decide
 * (lexicographic min (gain, c) on the device; the owner packs column c*,
 * other ranks zeros), SUM all-reduce of the column buffers,
 * kmedoids_build_apply_async(h, step).  No host round trip in any of the k
 * steps; the chosen medoids are read with kmedoids_get_state afterwards.
 * Errors: KM_ECOMM before kmedoids_shard_exchange, KM_EINVAL (step out of
 * order / range), KM_ECUDA. */
km_status kmedoids_build_decide(km_handle* h, int32_t step);
km_status kmedoids_build_apply_async(km_handle* h, int32_t step);
km_status kmedoids_shard_decide(km_handle* h);
km_status kmedoids_shard_apply_async(km_handle* h);
km_status kmedoids_shard_status(km_handle* h, int32_t wait, int32_t* converged, int32_t* n_iter, int32_t* n_swaps,
                                void* td_out);
km_status kmedoids_shard_trace(km_handle* h, int32_t* slots_out, int32_t* cands_out, void* dtds_out, int32_t cap,
                               int32_t* count_out);
/* After the five calls above were captured once into a CUDA graph on the
 * handle's stream (with the caller's collectives) and the graph replayed:
 * waits for the handle's stream and takes the number of decide steps from
 * the device status (the host did not see the replays), so
 * kmedoids_shard_status / kmedoids_shard_trace read the right mirror.
 * *calls_out (may be NULL): decide steps since the last reset.  The launch
 * counter does not count replayed kernels.  Errors: KM_EINVAL (NULL handle),
 * KM_ECUDA. */
km_status kmedoids_shard_resync(km_handle* h, int32_t* calls_out);

/* Sharded FastPAM2 (reading R6) iteration, on every rank:
 *   1. kmedoids_fp2_shard_eval(h)      per-slot best (v_i, i, c_i) over the local
 *                                      candidates -> record_send (k records)
 *   2. all-gather the records           (caller; k*16 bytes per rank)
 *   3. kmedoids_fp2_shard_plan(h, rcb, &m, &maxcnt)
 *                                      per-slot min over ranks, improving slots in
 *                                      (v_i, i) order (m of them; 0 = converged),
 *                                      this rank's planned candidate columns
 *                                      packed into col_send (maxcnt columns)
 *   4. if m > 0: all-gather maxcnt*n elements per rank from col_send into
 *      col_recv (rank order), then kmedoids_fp2_shard_apply(h, ...) runs the
 *      sequential phase redundantly on every rank (identical results).
 * Buffers are device memory owned by the handle.  The column buffers hold
 * col_capacity columns per rank and grow on demand: when step 3 returns a
 * maxcnt above the capacity last returned by kmedoids_fp2_shard_exchange,
 * the buffers were reallocated and the caller calls it again for the new
 * pointers before step 4. */
typedef struct {
    void* record_send;          /* k records of 16 bytes */
    void* record_recv;          /* R*k records, rank order */
    size_t record_bytes;        /* k*16 */
    void* col_send;             /* col_capacity columns of n elements */
    void* col_recv;             /* R*col_capacity columns (use R*maxcnt) */
    size_t col_bytes_per_column;
    int32_t col_capacity;       /* columns per rank the buffers hold now (<= k) */
} km_fp2_exchange;

km_status kmedoids_fp2_shard_exchange(km_handle* h, int32_t nranks, km_fp2_exchange* out);
km_status kmedoids_fp2_shard_eval(km_handle* h);
km_status kmedoids_fp2_shard_plan(km_handle* h, const int64_t* rank_col_begin, int32_t* m_out, int32_t* maxcnt_out);
km_status kmedoids_fp2_shard_apply(km_handle* h, int32_t* swaps_done_out, void* td_out);

/* Sharded FastPAM2, owner-side form of step 4 (reading R6 unchanged;
 * parallel.fp2_iter(mode="owner")).  After step 3 returned m > 0 (no column
 * all-gather), repeat on every rank until *more_out == 0:
 *   a. kmedoids_fp2_round_eval(h)   this rank re-evaluates, on the current
 *      state, its own unskipped plan entries from the round's first position
 *      in plan order (later swaps are re-checked) and publishes
 *      its first improving one -- plan position, dTD, slot, candidate and the
 *      candidate's n-element column -- into its round buffer (32-byte header
 *      {int32 pos (INT32_MAX = none), int32 pad, dTD (int64/double), int32
 *      slot, int32 c, 8 pad bytes}, then the column); round 0 publishes plan
 *      entry 0 as is (it is FastPAM1's swap);
 *   b. all-gather the round buffers: stride bytes per rank, rank order
 *      (caller; send -> recv of kmedoids_fp2_round_buffers);
 *   c. kmedoids_fp2_round_apply(h, &more, &swaps, td)  applies the published
 *      entry with the smallest plan position (identical on every rank); when
 *      none is published the iteration is over: *more_out = 0, *swaps_done_out
 *      = swaps of the iteration, *td_out (int64_t* / double*) = TD.
 * Same trace, medoids and TD as kmedoids_fp2_shard_apply and as one GPU
 * (same per-entry arithmetic and summation tree); one column per applied
 * swap crosses the interconnect instead of every planned candidate's.
 * Buffers are device memory owned by the handle (valid until destroy).
 * Errors: KM_ECOMM before kmedoids_fp2_shard_exchange, KM_EINVAL without a
 * plan / with an empty plan (converged: use kmedoids_fp2_shard_apply),
 * KM_ECUDA. */
km_status kmedoids_fp2_round_buffers(km_handle* h, void** send_out, void** recv_out, size_t* stride_out);
km_status kmedoids_fp2_round_eval(km_handle* h);
km_status kmedoids_fp2_round_apply(km_handle* h, int32_t* more_out, int32_t* swaps_done_out, void* td_out);

/* Sharded BUILD: step 0 evaluates the distance sums (first medoid), steps
 * 1..k-1 the BUILD gains of the local candidates into record_send; after the
 * gather, kmedoids_build_select picks the global (value, c) minimum, the
 * owner packs the column, the caller broadcasts it and kmedoids_build_apply
 * adds the medoid. */
km_status kmedoids_build_eval(km_handle* h, int32_t step);
km_status kmedoids_build_select(km_handle* h, const int64_t* rank_col_begin, int32_t* cand,
                                int32_t* owner, void* gain);
km_status kmedoids_build_apply(km_handle* h, int32_t step);

#ifdef __cplusplus
}
#endif

#endif /* KMEDOIDS_H */
