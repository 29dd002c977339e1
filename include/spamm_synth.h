/*
 * spamm_synth.h -- seeded synthetic inputs for the BASELINE.json configs.
 *
 * NOT part of the hot path and not a reference interface: these generate the
 * decay matrices BASELINE.json's configs describe (the reference generates
 * its own with oracle.cpp:156-189; the configs' matrices are not in the
 * reference).  The exact recipe is specified in DESIGN.md "Inputs".
 *
 * Values use a counter-based hash, so every entry is a pure function of
 * (seed, min(i,j), max(i,j)).  The host and device generators share every
 * integer and IEEE add/mul/div/sqrt step; they differ only through exp()
 * (glibc vs CUDA libdevice), so parity tests always ship one generator's bits
 * to both sides, never regenerate.
 */
#ifndef SPAMM_SYNTH_H
#define SPAMM_SYNTH_H

#include <stdint.h>

#include "spamm_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Config 1: 1-D chain, A_ij = u_ij * exp(-|i-j| / ell), |A_ij| < drop -> 0.
 * Host generator.  Writes non-null leaves (Morton order) up to `capacity`;
 * *n_leaves = total non-null leaves.  Pass payload = NULL to count only. */
int spg_synth_chain_host(int32_t n, int32_t leaf_size, double ell, uint64_t seed, double drop,
                         int64_t capacity, int32_t* block_rows, int32_t* block_cols,
                         double* payload, int64_t* n_leaves);

/* Configs 2-5: 3-D cluster.  n/4 sites uniform in a cube of density
 * `density` sites/A^3 (positions from site_seed), Morton-ordered, 4 basis
 * functions per site; A_ij = u_ij * exp(-d_ij / ell) with u from value_seed;
 * divided by the largest absolute row sum; |A_ij| < drop -> 0.  Host. */
int spg_synth_cluster_host(int32_t n, int32_t leaf_size, double ell, double density,
                           uint64_t site_seed, uint64_t value_seed, double drop, int64_t capacity,
                           int32_t* block_rows, int32_t* block_cols, double* payload,
                           int64_t* n_leaves);

/* Device generators: build the matrix directly in HBM (same recipe). */
int spg_synth_chain_device(spg_context* ctx, int32_t n, int32_t leaf_size, double ell,
                           uint64_t seed, double drop, spg_matrix** out);
int spg_synth_cluster_device(spg_context* ctx, int32_t n, int32_t leaf_size, double ell,
                             double density, uint64_t site_seed, uint64_t value_seed, double drop,
                             spg_matrix** out);
/* The same matrices restricted to block rows [row_begin, row_end) (a row
 * shard; the other rows are null).  Values are those of the full generator
 * (the cluster scale is the global largest row sum). */
int spg_synth_chain_device_rows(spg_context* ctx, int32_t n, int32_t leaf_size, double ell,
                                uint64_t seed, double drop, int32_t row_begin, int32_t row_end,
                                spg_matrix** out);
int spg_synth_cluster_device_rows(spg_context* ctx, int32_t n, int32_t leaf_size, double ell,
                                  double density, uint64_t site_seed, uint64_t value_seed,
                                  double drop, int32_t row_begin, int32_t row_end,
                                  spg_matrix** out);
/* The cluster generator's global scale (largest absolute row sum), and the
 * row-range generator with that scale passed in: generating many row panels
 * of one matrix (e.g. B streamed panel by panel) then skips the O(n^2) row
 * sums per call.  With scale = spg_synth_cluster_scale(...) the output is
 * bit-identical to spg_synth_cluster_device_rows. */
int spg_synth_cluster_scale(spg_context* ctx, int32_t n, double ell, double density,
                            uint64_t site_seed, uint64_t value_seed, double* scale);
int spg_synth_cluster_device_rows_scaled(spg_context* ctx, int32_t n, int32_t leaf_size,
                                         double ell, double density, uint64_t site_seed,
                                         uint64_t value_seed, double drop, double scale,
                                         int32_t row_begin, int32_t row_end, spg_matrix** out);

#ifdef __cplusplus
}
#endif

#endif /* SPAMM_SYNTH_H */
