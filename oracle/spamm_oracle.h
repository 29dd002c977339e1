/*
 * spamm_oracle.h -- CPU restatement of the reference SpAMM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2005_10680_b200/)
 * links, loads or calls this library; only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg use it, and only as the checker.
 *
 * Plain C99 restatement of the reference (`spamm-ec`, /root/reference/proj)
 * algorithms on this path.  Every function cites the reference file:line it
 * follows.  Arithmetic is written with separate multiplies and adds and the
 * library is compiled with -ffp-contract=off and no -march, so the bits match
 * the reference build.  Pinned against the reference itself
 * (oracle/_ref, compiled from the reference sources) and against the golden
 * fixtures in tests/golden/.
 *
 * Data model (quadtree.hpp:34-49): a node is either NULL (identically zero
 * quadrant), a leaf (dense L x L column-major block) or an inner node with
 * four children indexed [2*row + col]; every node caches its Frobenius norm.
 */
#ifndef SPAMM_ORACLE_H
#define SPAMM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ora_tree ora_tree;

/* Build from a leaf list (block row, block col, L*L column-major payload per
 * leaf).  All-zero leaves collapse to NULL (node_ops.hpp:40-53); inner nodes
 * with four NULL children collapse (node_ops.hpp:57-63).  Returns NULL on
 * invalid input (out-of-range or duplicate block coordinates). */
ora_tree* ora_build(int dimension, int leaf_size, int64_t n_leaves, const int32_t* block_rows,
                    const int32_t* block_cols, const double* payload);

/* Norm-only tree for large-N CSE: leaf norms given, no payload.
 * Negative norm = absent leaf. */
ora_tree* ora_build_norm_only(int dimension, int leaf_size, int64_t n_leaves,
                              const int32_t* block_rows, const int32_t* block_cols,
                              const double* leaf_norms);

void ora_free(ora_tree* t);

int ora_dimension(const ora_tree* t);
int ora_padded_dimension(const ora_tree* t);
int ora_leaf_size(const ora_tree* t);
int ora_depth(const ora_tree* t);
int64_t ora_nnz_blocks(const ora_tree* t);
double ora_frobenius(const ora_tree* t);

/* Leaves in Morton order (child index 2*row+col at every level). Any output
 * pointer may be NULL. payload needs nnz_blocks*L*L doubles. */
void ora_leaves(const ora_tree* t, int32_t* rows, int32_t* cols, double* payload, double* norms);

/* Dense Morton-ordered grid of node norms at `level` (0 = root); 4^level
 * entries; -1.0 marks a NULL node. */
void ora_level_norms(const ora_tree* t, int level, double* out);

/* CSE sweep (error_control.cpp:34-79,160-166). Returns 0, or -1 on mismatch. */
int ora_cse(const ora_tree* a, const ora_tree* b, const double* taus, int n_taus, double* bounds);

/* cse_node (error_control.cpp:46-79) for the pair A(I,K) x B(K,J) at `level`
 * (the partial vector a row shard contributes). */
int ora_cse_subtree(const ora_tree* a, const ora_tree* b, const double* taus, int n_taus, int level,
                    int32_t I, int32_t K, int32_t J, double* out);

/* First k with bounds[k] < delta (error_control.cpp:81-87); -1 if none. */
int ora_select_index(const double* bounds, int n_taus, double delta);

/* SpAMM product (multiply.cpp:70-92,109-116).  NULL result tree is never
 * returned for valid input; *status = 0 ok, -1 invalid. */
ora_tree* ora_spamm(const ora_tree* a, const ora_tree* b, double tau, int* status);

/* Exact product (multiply.cpp:34-56,102-107). */
ora_tree* ora_multiply_exact(const ora_tree* a, const ora_tree* b, int* status);

/* Leaf products the recursion of multiply.cpp:70-92 performs, as (i,k,j)
 * block triples sorted by (Morton(i,j), k).  Returns the count; writes at most
 * `capacity` triples (3 int32 each) when `triples` is non-NULL. */
int64_t ora_survivors(const ora_tree* a, const ora_tree* b, double tau, int32_t* triples,
                      int64_t capacity);

/* Number of non-null leaf pairs (candidates T_cand, SURVEY 8 notation). */
int64_t ora_candidates(const ora_tree* a, const ora_tree* b);

/* truncate (error_control.cpp:93-134,174-201): returns the truncated tree
 * (a new tree; leaves copied), the removed norm bound and count; NULL with
 * *status = -1 for delta < 0. */
ora_tree* ora_truncate(const ora_tree* x, double delta, double* removed_norm,
                       int64_t* removed_count, int* status);

/* Leaf norm rule alone (node_ops.hpp:24-28), for kernel-level pins. */
double ora_block_norm(const double* block, int64_t count);

#ifdef __cplusplus
}
#endif

#endif
