/*
 * spamm_gpu.h -- C ABI of the B200-native SpAMM hot path.
 *
 * This is the drop-in boundary under the reference's C++ API
 * (/root/reference/proj/core/include/spamm/{quadtree,multiply,error_control}.hpp).
 * Plain pointers, sizes and status codes only: no C++ types, no torch types,
 * no exception crosses it.  The C++ drop-in (include/spamm/*.hpp, namespace
 * spamm) and the Python bindings (paper_2005_10680_b200/_native.py) both sit
 * on top of exactly these entry points.
 *
 * Each entry point names the reference interface it replaces (file:line,
 * relative to /root/reference/proj/core).
 *
 * Ownership: the caller owns every host buffer; the library owns every
 * device buffer behind the opaque handles.  Matrices are immutable once built
 * (quadtree.hpp:30-33).  Calls on one context are serialised by the library.
 *
 * Errors: every function returns SPG_OK or a negative-free status code;
 * spg_last_error() gives the thread-local message of the last failure.  The
 * codes map onto the reference's exception types:
 *   SPG_EINVAL  std::invalid_argument  (dimension/leaf mismatch multiply.cpp:94-98,
 *               error_control.cpp:161-163; tau < 0 multiply.cpp:112;
 *               delta <= 0 error_control.cpp:205; grid error_control.cpp:139-150;
 *               duplicate coordinates quadtree.cpp:213-216)
 *   SPG_ERANGE  std::out_of_range      (coordinates quadtree.cpp:202-208)
 */
#ifndef SPAMM_GPU_H
#define SPAMM_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPG_OK 0
#define SPG_EINVAL 1
#define SPG_ERANGE 2
#define SPG_ENOMEM 3
#define SPG_ECUDA 4
#define SPG_ENCCL 5
#define SPG_EINTERNAL 6

typedef struct spg_context spg_context; /* one device + one stream + workspace */
typedef struct spg_matrix spg_matrix;   /* device-resident quadtree matrix     */

typedef struct {
  int32_t dimension;        /* QuadTreeMatrix::dimension()         quadtree.hpp:65 */
  int32_t padded_dimension; /* QuadTreeMatrix::padded_dimension()  quadtree.hpp:66 */
  int32_t leaf_size;        /* QuadTreeMatrix::leaf_size()         quadtree.hpp:67 */
  int32_t depth;            /* log2(padded / leaf)                               */
  int64_t nnz_blocks;       /* QuadTreeMatrix::nnz_blocks()        quadtree.hpp:79 */
  double frobenius_norm;    /* QuadTreeMatrix::frobenius_norm()    quadtree.hpp:72 */
} spg_matrix_info;

typedef struct {
  int64_t candidates;    /* non-null leaf pairs (A(i,k), B(k,j))                 */
  int64_t survivors;     /* leaf products performed, |S(tau)|                    */
  int64_t output_blocks; /* C blocks with at least one surviving product        */
  double flops;          /* 2 * L^3 * survivors                                  */
  float ms_tasklist;     /* device time: skip test + compaction + grouping       */
  float ms_gemm;         /* device time: leaf GEMM kernel                         */
  float ms_finalize;     /* device time: C norms, zero-collapse, norm pyramid    */
} spg_spamm_stats;

typedef struct {
  double tau;            /* ControlledProduct::chosen_tau   error_control.hpp:66 */
  int32_t tau_index;     /* grid index, -1 = exact fallback (tau = 0)           */
  double bound;          /* ControlledProduct::bound        error_control.hpp:68 */
  double cse_seconds;    /* ControlledProduct::cse_seconds  error_control.hpp:69 */
  double spamm_seconds;  /* ControlledProduct::spamm_seconds error_control.hpp:70 */
  float ms_cse;          /* device time of the tau-sweep kernels                 */
  spg_spamm_stats spamm;
} spg_controlled_stats;

/* ---- library / context -------------------------------------------------- */
const char* spg_last_error(void);
int spg_version(void);
int spg_device_count(int* count);
int spg_context_create(int device, spg_context** out);
int spg_context_destroy(spg_context* ctx);
/* cudaStream_t of the context, for callers that time kernels with events. */
int spg_context_stream(spg_context* ctx, void** stream);
int spg_context_synchronize(spg_context* ctx);
/* Kernel launches issued by this context so far (evidence counter). */
int spg_context_launch_count(spg_context* ctx, int64_t* launches);
/* Products larger than the device's memory (the reference's spamm_multiply
 * has no size cap, multiply.cpp:109-116): when a product's task list (16 B
 * per candidate leaf product, 24 B for the L = 32 super-block entries; ~40 /
 * ~96 B where the expansion + sort builder runs: depth < 3, chunks
 * thinner than 8 block rows) would exceed `bytes` -- 0 (default):
 * half of the free HBM plus the context's cached pool -- the product is run
 * in 2^c row chunks, one task list at a time, into one C; bitwise the same C
 * (same products, same per-block k order). */
int spg_context_set_task_budget(spg_context* ctx, int64_t bytes);
/* Return the context's cached (freed) device blocks to the driver; live
 * matrices are untouched.  Allocation failures trim by themselves first. */
int spg_context_trim(spg_context* ctx);

/* ---- matrices (quadtree.hpp / quadtree.cpp) ------------------------------ */
/* Replaces QuadTreeMatrix::from_coordinates at leaf granularity
 * (quadtree.cpp:198-222): `n_leaves` dense L*L column-major blocks at block
 * coordinates (block_rows[t], block_cols[t]).  All-zero blocks collapse
 * (node_ops.hpp:40-53); norms are cached bottom-up (node_ops.hpp:24-36).
 * Host buffers. */
int spg_matrix_upload(spg_context* ctx, int32_t dimension, int32_t leaf_size, int64_t n_leaves,
                      const int32_t* block_rows, const int32_t* block_cols, const double* payload,
                      spg_matrix** out);
/* Same with device-resident inputs (the matrix takes a private copy). */
/* Staged upload: the same as spg_matrix_upload, split in two.  stage()
 * queues the host->device copies on the context's upload stream and returns
 * at once (the pinned host buffers must stay unchanged until the matching
 * stage_finish() returns); stage_finish() makes the context's work wait for
 * the copies and builds the matrix (norms, pyramid).  Lets a caller stream
 * the next input in while the current product runs.  stage_finish() (or
 * spg_staged_free()) releases the staging object. */
typedef struct spg_staged spg_staged;
int spg_matrix_stage(spg_context* ctx, int32_t dimension, int32_t leaf_size, int64_t n_leaves,
                     const int32_t* block_rows, const int32_t* block_cols, const double* payload,
                     spg_staged** out);
int spg_matrix_stage_finish(spg_staged* staged, spg_matrix** out);
void spg_staged_free(spg_staged* staged);
int spg_matrix_upload_device(spg_context* ctx, int32_t dimension, int32_t leaf_size,
                             int64_t n_leaves, const int32_t* d_block_rows,
                             const int32_t* d_block_cols, const double* d_payload,
                             spg_matrix** out);
/* QuadTreeMatrix::from_dense (quadtree.cpp:224-229); host row-major n x n. */
int spg_matrix_from_dense(spg_context* ctx, int32_t dimension, int32_t leaf_size,
                          const double* dense_rowmajor, spg_matrix** out);
/* QuadTreeMatrix::zero (quadtree.cpp:237-240). */
int spg_matrix_zero(spg_context* ctx, int32_t dimension, int32_t leaf_size, spg_matrix** out);
int spg_matrix_get_info(const spg_matrix* m, spg_matrix_info* out);
/* Non-null leaves in Morton order (child index 2*row+col, quadtree.cpp:103-106):
 * block coordinates, L*L column-major payload and cached norms.  Any output
 * may be NULL.  Host buffers of nnz_blocks entries. */
int spg_matrix_download(const spg_matrix* m, int32_t* block_rows, int32_t* block_cols,
                        double* payload, double* norms);
/* QuadTreeMatrix::to_dense (quadtree.cpp:243-247); host row-major n x n. */
int spg_matrix_to_dense(const spg_matrix* m, double* dense_rowmajor);
/* Cached node norms of one tree level as a dense Morton grid of 4^level
 * doubles; -1.0 marks an identically-zero (null) quadrant. */
int spg_matrix_level_norms(const spg_matrix* m, int32_t level, double* out);
int spg_matrix_free(spg_matrix* m);

/* ---- hot path (error_control.hpp / multiply.hpp) ------------------------- */
/* Validation of ToleranceGrid(std::vector<double>) (error_control.cpp:139-150). */
int spg_tolerance_grid_check(const double* taus, int32_t n_taus);
/* spamm::cse (error_control.hpp:44, error_control.cpp:160-166).  Bit-identical
 * bounds.  `bounds` is a host buffer of n_taus doubles. */
int spg_cse(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, const double* taus,
            int32_t n_taus, double* bounds);
/* spamm::select_tolerance (error_control.hpp:48-49, error_control.cpp:168-172).
 * Host-only; *tau = 0 and *index = -1 when no candidate qualifies. */
int spg_select_tolerance(const double* bounds, const double* taus, int32_t n_taus, double delta,
                         double* tau, int32_t* index);
/* spamm::spamm_multiply (multiply.hpp:28-29, multiply.cpp:109-116). */
int spg_spamm(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, double tau,
              spg_matrix** c, spg_spamm_stats* stats);
/* spamm::multiply_exact (multiply.hpp:22, multiply.cpp:102-107). */
int spg_multiply_exact(spg_context* ctx, const spg_matrix* a, const spg_matrix* b,
                       spg_matrix** c, spg_spamm_stats* stats);
/* spamm::spamm_with_error_control (error_control.hpp:76-77,
 * error_control.cpp:203-220).  `bounds` (optional, n_taus doubles) receives
 * the sweep. */
int spg_spamm_with_error_control(spg_context* ctx, const spg_matrix* a, const spg_matrix* b,
                                 double delta, const double* taus, int32_t n_taus,
                                 spg_matrix** c, double* bounds, spg_controlled_stats* stats);
/* spg_spamm_with_error_control with C delivered to host buffers: the leaf
 * GEMM runs in chunks and each finished chunk is copied D2H while the next
 * one computes (use pinned buffers for the overlap).  Outputs equal
 * spg_spamm_with_error_control + spg_matrix_download: *c_count non-null
 * leaves in Morton order (capacity >= number of output blocks). */
int spg_spamm_with_error_control_to_host(spg_context* ctx, const spg_matrix* a,
                                         const spg_matrix* b, double delta, const double* taus,
                                         int32_t n_taus, int64_t capacity, int32_t* c_rows,
                                         int32_t* c_cols, double* c_payload, double* c_norms,
                                         int64_t* c_count, double* bounds,
                                         spg_controlled_stats* stats);
/* The surviving leaf-product set of spamm_multiply(a, b, tau) (the leaves the
 * recursion of multiply.cpp:70-92 reaches) as (i, k, j) block triples sorted
 * by (Morton(i, j), k).  Writes min(count, capacity) triples. */
int spg_survivors(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, double tau,
                  int64_t* count, int32_t* triples, int64_t capacity);

/* Survivor-set digest of A*B at tau restricted to the output block rows of
 * shard `shard` of 2^level (level 0: the whole product), from the product's
 * own task-list builder: count and sum over the surviving (i, k, j) of
 * mix64(i << 42 | k << 21 | j) mod 2^64 (mix64 = SplitMix64 finaliser).  The
 * sum is order-free and additive over disjoint shards, so per-shard digests
 * of a sharded run add up to the whole product's -- the form in which the
 * survivor SET is pinned against the reference at configs 2-5 sizes. */
int spg_survivor_digest(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, double tau,
                        int32_t level, int32_t shard, int64_t* count, uint64_t* digest);

/* Parity audit: of all candidate leaf products (non-null
 * A(i,k) x B(k,j)), how many have |fl(nA*nB) - tau| <= ulps * ulp(tau) --
 * the decisions a one-ulp norm difference could flip. */
int spg_parity_audit(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, double tau,
                     int32_t ulps, int64_t* near_ties, int64_t* candidates);

/* Self-test of the sweep kernels' branch-free square root (csrc/cse.cu
 * sqrt_fast + its out-of-line slow path) against the correctly rounded
 * sqrt.rn.f64 the reference's std::sqrt stands for (error_control.cpp:77):
 * 2n seeded bit patterns over every exponent, sign and special value plus
 * perfect squares +-1 ulp; *mismatches counts differing result bits. */
int spg_selftest_sqrt(spg_context* ctx, int64_t n, uint64_t seed, int64_t* mismatches);

/* ---- callers of the hot path (SURVEY.md 8f "next" row 1) ----------------- */
/* truncate (error_control.hpp:59-62, error_control.cpp:174-201): remove whole
 * leaves greedily in ascending (norm, row-major position) order while the
 * removed norm stays strictly below delta.  The result shares x's payload. */
int spg_truncate(spg_context* ctx, const spg_matrix* x, double delta, spg_matrix** out,
                 double* removed_norm_bound, int64_t* removed_block_count);

#define SPG_VARIANT_TRUNCMUL 0 /* multiply_exact + truncate(delta)              */
#define SPG_VARIANT_SPAMM 1    /* spamm_with_error_control(delta)                */
#define SPG_VARIANT_HYBRID 2   /* spamm_with_error_control(delta/2) + truncate(delta/2) */

typedef struct {
  int32_t variant;
  double chosen_tau;         /* RunRecord::chosen_tau (0 for truncmul)        */
  int64_t nnz_blocks_mid;    /* leaves of the product before truncation       */
  int64_t removed_blocks;    /* leaves removed by truncation                  */
  double removed_norm_bound; /* sqrt of the removed squared norms             */
  double t_mul, t_cse, t_spamm, t_trunc; /* host seconds per phase (RunRecord) */
  double flops;              /* leaf-GEMM flops performed                     */
} spg_square_stats;

/* approximate_square (experiment.cpp:47-82): X*X by one of the variants. */
int spg_approximate_square(spg_context* ctx, const spg_matrix* x, int32_t variant, double delta,
                           const double* taus, int32_t n_taus, spg_matrix** out,
                           spg_square_stats* stats);

/* ---- device matrix algebra for the callers (quadtree.cpp:128-171,254-261) */
/* QuadTreeMatrix::trace: same association as node_trace (quadtree.cpp:128-138). */
int spg_matrix_trace(const spg_matrix* m, double* out);
/* QuadTreeMatrix::nnz: stored entries != 0 (quadtree.cpp:140-151). */
int spg_matrix_nnz(const spg_matrix* m, int64_t* out);
/* add(a.scale(alpha), b.scale(beta)) (quadtree.cpp:24-36,249-261); b may be
 * NULL (scale only).  All-zero leaves collapse. */
int spg_matrix_axpby(spg_context* ctx, double alpha, const spg_matrix* a, double beta,
                     const spg_matrix* b, spg_matrix** out);
/* QuadTreeMatrix::identity (quadtree.cpp:231-235). */
int spg_matrix_identity(spg_context* ctx, int32_t dimension, int32_t leaf_size, spg_matrix** out);
/* diag(d): leaves on the block diagonal holding d (host array of length n). */
int spg_matrix_from_diagonal(spg_context* ctx, int32_t dimension, int32_t leaf_size,
                             const double* diag, spg_matrix** out);
/* Per row i (host arrays of length n, either may be NULL): the diagonal entry
 * and sum_j |a_ij| (ascending j) -- Gershgorin data for spectral bounds. */
int spg_matrix_rows(const spg_matrix* m, double* diag, double* abs_row_sums);
/* Gershgorin spectral bounds (reference oracle.cpp:191-200 on the dense
 * matrix): low = min_i (a_ii - r_i), high = max_i (a_ii + r_i), r_i = sum over
 * j != i of |a_ij| in ascending j -- bitwise the reference's values, computed
 * from the device leaves (no dense copy). */
int spg_matrix_gershgorin(const spg_matrix* m, double* low, double* high);

/* ---- SP2 purification over the GPU product (purification.cpp:49-202;
 * SURVEY.md 8f row 2, BASELINE config 3) ----------------------------------- */
#define SPG_STATUS_OK 0
#define SPG_STATUS_VIOLATION 1
#define SPG_STATUS_CONVERGED 2

typedef struct {
  int32_t variant;               /* SPG_VARIANT_*                               */
  int32_t occupation;            /* PurificationConfig::occupation             */
  int32_t max_iterations;
  double epsilon;
  double idempotency_threshold;  /* 0 -> epsilon / 10                          */
  const double* taus;            /* tolerance grid of the controlled products  */
  int32_t n_taus;
  double initial_delta;          /* ErrorBudget::initial_delta                 */
  const double* deltas;          /* ErrorBudget::deltas (>= max_iterations)    */
  int32_t n_deltas;
  int32_t measure_error;         /* realized error vs an exact product (RunRecord) */
} spg_purify_config;

/* RunRecord (run_record.hpp:16-32), one per iteration (0 = initial truncation) */
typedef struct {
  int32_t iteration;
  int32_t status;      /* SPG_STATUS_*                          */
  int32_t polynomial;  /* 0: x^2, 1: 2x - x^2 (sp2_step)         */
  double tolerance, chosen_tau, t_mul, t_trunc, t_spamm, t_cse;
  int64_t nnz_in, nnz_mid, nnz_out, nnz_blocks_out;
  double realized_error; /* -1 when not measured                 */
  double trace;
  double flops;          /* leaf-GEMM flops of the iteration's square */
} spg_run_record;

/* ErrorBudget::geometric (purification.cpp:66-82): deltas[iterations]. */
int spg_error_budget_geometric(double epsilon, int32_t iterations, double ratio,
                               double* initial_delta, double* deltas);
/* purify (purification.cpp:90-202).  *density: the final iterate (or the last
 * iterate before convergence, like the reference). */
int spg_purify(spg_context* ctx, const spg_matrix* x0, const spg_purify_config* cfg,
               spg_matrix** density, spg_run_record* log, int32_t log_capacity, int32_t* n_log,
               int32_t* converged, int32_t* iterations);

/* ---- row shards across GPUs (new, the reference is single-
 * process) --------------------------------------------------------------
 * A shard at `level` s owns output block-rows [shard*nb/2^s, (shard+1)*nb/2^s)
 * (power-of-two aligned), shard in [0, 2^s).  Bounds assembled from all
 * shards are bit-identical to spg_cse; the union of the shard products is
 * spg_spamm's C, block for block. */
/* The shard's level-s partial bound vectors: 4^s x n_taus doubles, vector of
 * pair (shard, K, J) at index (K * 2^s + J) * n_taus; zeros for null pairs. */
int spg_cse_shard(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, const double* taus,
                  int32_t n_taus, int32_t level, int32_t shard, double* partial);
/* Host-only: combine the gathered partials (2^s shards in order, each as
 * above) through the top s levels in reference order (cse_node,
 * error_control.cpp:46-79).  a/b_top_norms: node norms of levels 0..s-1,
 * concatenated Morton grids (spg_matrix_top_norms). */
int spg_cse_finish(int32_t level, const double* a_top_norms, const double* b_top_norms,
                   int32_t n_taus, const double* partials, double* bounds);
/* Concatenated Morton norm grids of levels 0..levels-1 ((4^levels-1)/3 doubles). */
int spg_matrix_top_norms(const spg_matrix* m, int32_t levels, double* out);
/* spamm_multiply restricted to the shard's output block-rows. */
int spg_spamm_shard(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, double tau,
                    int32_t level, int32_t shard, spg_matrix** c, spg_spamm_stats* stats);

/* ---- B resident in host memory, streamed in panels (SURVEY.md 8e, configs
 * 4/5: operands larger than one GPU's HBM) -----------------------------------
 * The leaves of B are given sorted by block row (ties in any order) and stay
 * in the caller's host buffer, which must outlive the stream object.  Panel
 * p holds block rows [p*panel_block_rows, (p+1)*panel_block_rows).  Creation
 * streams the panels through the leaf-norm kernel once to build B's norm
 * pyramid; the products then copy each panel (double-buffered, overlapping
 * the GEMM of the previous one) and continue every output block's
 * accumulator over the panel's k range.  Results are bitwise identical to
 * the same call with B resident (spg_matrix_upload + spg_spamm / spg_cse).
 * register_host != 0 page-locks the caller's buffer for the stream's
 * lifetime (asynchronous copies); 0 leaves it as is. */
typedef struct spg_bstream spg_bstream;
int spg_bstream_create(spg_context* ctx, int32_t dimension, int32_t leaf_size, int64_t n_leaves,
                       const int32_t* block_rows, const int32_t* block_cols,
                       const double* payload, int32_t panel_block_rows, int32_t register_host,
                       spg_bstream** out);
/* B's norm-only matrix: valid for spg_cse, spg_matrix_get_info,
 * spg_matrix_level_norms, spg_matrix_download without payload; SPG_EINVAL
 * where leaf values are needed. Owned by the stream object. */
int spg_bstream_matrix(const spg_bstream* bs, const spg_matrix** norms);
int spg_bstream_panels(const spg_bstream* bs, int32_t* n_panels, int64_t* max_panel_leaves);
void spg_bstream_free(spg_bstream* bs);
/* spamm_multiply (multiply.cpp:109-116) with B streamed from host memory. */
int spg_spamm_streamed(spg_context* ctx, const spg_matrix* a, const spg_bstream* b, double tau,
                       spg_matrix** c, spg_spamm_stats* stats);
/* spamm_with_error_control (error_control.cpp:203-220) with B streamed. */
int spg_spamm_with_error_control_streamed(spg_context* ctx, const spg_matrix* a,
                                          const spg_bstream* b, double delta, const double* taus,
                                          int32_t n_taus, spg_matrix** c, double* bounds,
                                          spg_controlled_stats* stats);

/* ---- panel plans: B arriving in block-row panels from any source (host
 * memory, the GPU owning those rows over NCCL) --------------------------------
 * B is a norm-only matrix whose leaf slots are sorted by block row
 * (spg_matrix_from_leaf_norms, spg_bstream_matrix).  A plan holds the task
 * list of A*B (or of a row shard of it, as spg_spamm_shard) and an all-zero
 * C; spg_plan_accumulate adds the products whose k lies in block rows
 * [row_begin, row_end) given B's leaves of those rows (slots
 * spg_plan_panel_slots(...)) in device memory.  Panels must tile
 * [0, ceil(n/L)) in ascending order (empty rows may pass d_panel = NULL);
 * the resulting C is bitwise identical to the resident product.
 * `stream` (a cudaStream_t, or NULL): the library's work waits for the work
 * already queued on it, and work queued on it later waits for the library's
 * use of d_panel, so a caller filling panel buffers on its own stream needs
 * no host synchronisation. */
typedef struct spg_plan spg_plan;
/* a_norms (or NULL): the whole A's norms (spg_matrix_from_leaf_norms) when
 * `a` holds only the shard's block rows -- the skip tests above the shard
 * level need the global ancestor norms. */
int spg_plan_create(spg_context* ctx, const spg_matrix* a, const spg_matrix* a_norms,
                    const spg_matrix* b, double tau, int32_t level, int32_t shard,
                    spg_plan** plan);
int spg_plan_panel_slots(const spg_plan* plan, int32_t row_begin, int32_t row_end,
                         int64_t* slot_begin, int64_t* count);
int spg_plan_accumulate(spg_plan* plan, int32_t row_begin, int32_t row_end,
                        const double* d_panel, void* stream);
int spg_plan_finish(spg_plan* plan, spg_matrix** c, spg_spamm_stats* stats);
void spg_plan_free(spg_plan* plan);
/* The whole panel loop in one call, with the row chunking of
 * spg_context_set_task_budget (each chunk receives every panel again): B's
 * panels of `panel_rows` block rows (never crossing a multiple of
 * `owner_rows`, 0 = no owners) are requested from fetch(user, row_begin,
 * row_end, d_dst, count, stream), which fills d_dst with the `count` leaves of
 * those rows in (row, col) order on `stream` (asynchronously is fine: the
 * GEMM waits for the stream; the buffer is not refilled before its GEMM is
 * done).  Two panels are in flight.  The context is unlocked while fetch
 * runs.  Returns the shard's rows of C~ -- bitwise the resident product's. */
typedef int (*spg_panel_fetch_fn)(void* user, int32_t row_begin, int32_t row_end, double* d_dst,
                                  int64_t count, void* stream);
int spg_spamm_panels(spg_context* ctx, const spg_matrix* a, const spg_matrix* a_norms,
                     const spg_matrix* b_norms, double tau, int32_t level, int32_t shard,
                     int32_t panel_rows, int32_t owner_rows, spg_panel_fetch_fn fetch,
                     void* user, spg_matrix** c, spg_spamm_stats* stats);
/* All of the plan's products in ONE GEMM launch, B leaf t read in place
 * from owner_base[slot_owner[t]] + slot_local[t] * L*L: the owners' leaf
 * payloads, local or another GPU's memory opened with spg_ipc_open (NVLink
 * peer loads inside the GEMM -- no staging copy, no broadcast).  Host arrays
 * of B's leaf count (slots of the norm-only B); replaces the panels. */
int spg_plan_run_table(spg_plan* plan, int32_t n_owners, const double* const* owner_base,
                       const int32_t* slot_owner, const int32_t* slot_local, void* stream);
/* One timed pass of the leaf-norm kernel (K1, block_norm) over every leaf
 * of m (results discarded): *ms = device time.  For roofline reporting. */
int spg_matrix_norm_pass(const spg_matrix* m, float* ms);
/* Device address of a matrix's leaf payload (slot t at base + t * L*L). */
int spg_matrix_payload(const spg_matrix* m, const double** base);
/* Payload slot of every non-null leaf, in spg_matrix_download order. */
int spg_matrix_payload_slots(const spg_matrix* m, int32_t* slots);
/* CUDA IPC of a matrix's leaf payload (64-byte handle) for the processes of
 * one node; the exporting matrix must outlive every importer's use. */
int spg_ipc_export(const spg_matrix* m, void* handle);
int spg_ipc_open(spg_context* ctx, const void* handle, const double** base);
int spg_ipc_close(spg_context* ctx, const double* base);
/* Norm-only matrix from a leaf table (host arrays, sorted by (block row, block
 * col), no duplicates -- SPG_EINVAL otherwise; slot
 * t = leaf t).  nonzero may be NULL (every leaf non-null).  Norms are taken
 * as given: pass the block_norm values the owning GPU computed (download
 * norms) for bit-exact bounds. */
int spg_matrix_from_leaf_norms(spg_context* ctx, int32_t dimension, int32_t leaf_size,
                               int64_t n_leaves, const int32_t* block_rows,
                               const int32_t* block_cols, const double* norms,
                               const uint8_t* nonzero, spg_matrix** out);
/* The non-null leaves of block rows [row_begin, row_end) in (row, column)
 * order into device memory (at most `capacity` leaves; no host sync -- the
 * caller knows the count from the leaf table).  `stream` as above. */
int spg_matrix_gather_rows(const spg_matrix* m, int32_t row_begin, int32_t row_end,
                           double* d_out, int64_t capacity, void* stream);

/* ---- multi-GPU inside the library: communicator + sharded products
 * (replaces the reference's fork-join over host threads,
 * execution.cpp:11-23, multiply.cpp:79-84, error_control.cpp:59-66) ---------
 * One process per GPU; 2^s ranks shard the output block rows: rank r owns
 * rows [r nb/2^s, (r+1) nb/2^s).  The sweep runs below level s per rank, the
 * level-s partial vectors are all-gathered and every rank finishes the top s
 * levels in reference order: bounds and tau are bit-identical to one GPU on
 * every rank, and so are the rank's rows of C~ (per-block k order unchanged).
 * Transports: NCCL (loaded with dlopen; SPG_NCCL_LIB overrides the library
 * name; collectives on the context's stream, over NVLink / NVSwitch) or a
 * host all-gather callback (the caller's own collective: gloo, MPI, tests). */
typedef struct spg_comm spg_comm;
#define SPG_COMM_ID_BYTES 128
/* All-gather `bytes` from every rank into recv (nranks * bytes, rank order);
 * return 0 on success. */
typedef int (*spg_host_allgather_fn)(void* user, const void* send, size_t bytes, void* recv);
/* ncclGetUniqueId: rank 0 creates it and hands the 128 bytes to the others. */
int spg_comm_unique_id(void* id_out);
int spg_comm_create_nccl(spg_context* ctx, int32_t nranks, int32_t rank, const void* id,
                         spg_comm** out);
int spg_comm_create_host(spg_context* ctx, int32_t nranks, int32_t rank,
                         spg_host_allgather_fn fn, void* user, spg_comm** out);
int spg_comm_info(const spg_comm* comm, int32_t* nranks, int32_t* rank, int32_t* uses_nccl);
int spg_comm_destroy(spg_comm* comm);
/* cse (error_control.cpp:160-166) of the whole product, sharded: bounds on
 * every rank. */
int spg_cse_sharded(spg_comm* comm, const spg_matrix* a, const spg_matrix* b, const double* taus,
                    int32_t n_taus, double* bounds);
/* spamm_multiply (skip_test = 1) / multiply_exact (skip_test = 0), sharded:
 * the rank's rows of C, or with gather = 1 the whole C on every rank
 * (all-gather of the rows' leaves). */
int spg_spamm_sharded(spg_comm* comm, const spg_matrix* a, const spg_matrix* b, double tau,
                      int32_t skip_test, int32_t gather, spg_matrix** c, spg_spamm_stats* stats);
/* spamm_with_error_control (error_control.cpp:203-220), sharded as above;
 * stats->spamm counts this rank's rows; bounds (may be NULL) the whole
 * problem's. */
int spg_spamm_with_error_control_sharded(spg_comm* comm, const spg_matrix* a,
                                         const spg_matrix* b, double delta, const double* taus,
                                         int32_t n_taus, int32_t gather, spg_matrix** c,
                                         double* bounds, spg_controlled_stats* stats);
/* Every rank's row shard (disjoint block rows) -> the whole matrix on every rank. */
int spg_matrix_gather_shards(spg_comm* comm, const spg_matrix* shard, spg_matrix** out);

#ifdef __cplusplus
}
#endif

#endif /* SPAMM_GPU_H */
