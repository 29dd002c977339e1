/*
 * spamm_oracle.c -- CPU restatement of the reference SpAMM hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see spamm_oracle.h).  Compiled with
 * -ffp-contract=off and without -march so every multiply and add rounds
 * separately, exactly like the reference Release build.
 */
#include "spamm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef struct ora_node {
  double norm;
  double* block; /* leaf payload, column-major L*L; NULL on inner nodes / norm-only leaves */
  struct ora_node* child[4];
} ora_node;

struct ora_tree {
  int dimension;
  int padded;
  int leaf_size;
  int depth;
  int norm_only;
  ora_node* root;
};

/* ---------------------------------------------------------------------------
 * node_ops.hpp restated
 * ------------------------------------------------------------------------- */

/* block_norm: node_ops.hpp:24-28 -- ascending storage order, then sqrt. */
double ora_block_norm(const double* block, int64_t count) {
  double sumsq = 0.0;
  for (int64_t t = 0; t < count; ++t) sumsq += block[t] * block[t];
  return sqrt(sumsq);
}

/* combine_child_norms: node_ops.hpp:30-36 -- children 0..3, NULL skipped. */
static double combine_child_norms(ora_node* const child[4]) {
  double sumsq = 0.0;
  for (int c = 0; c < 4; ++c)
    if (child[c]) sumsq += child[c]->norm * child[c]->norm;
  return sqrt(sumsq);
}

static ora_node* new_node(void) { return (ora_node*)calloc(1, sizeof(ora_node)); }

/* make_leaf: node_ops.hpp:40-53 -- takes ownership of `block`; all-zero -> NULL. */
static ora_node* make_leaf(double* block, int64_t count) {
  int all_zero = 1;
  for (int64_t t = 0; t < count; ++t)
    if (block[t] != 0.0) {
      all_zero = 0;
      break;
    }
  if (all_zero) {
    free(block);
    return NULL;
  }
  ora_node* n = new_node();
  n->norm = ora_block_norm(block, count);
  n->block = block;
  return n;
}

/* make_inner: node_ops.hpp:57-63 -- four NULL children -> NULL. */
static ora_node* make_inner(ora_node* child[4]) {
  if (!child[0] && !child[1] && !child[2] && !child[3]) return NULL;
  ora_node* n = new_node();
  n->norm = combine_child_norms(child);
  for (int c = 0; c < 4; ++c) n->child[c] = child[c];
  return n;
}

static void free_node(ora_node* n) {
  if (!n) return;
  for (int c = 0; c < 4; ++c) free_node(n->child[c]);
  free(n->block);
  free(n);
}

/* padded_dimension_for: quadtree.cpp:15-22. */
static int padded_dimension_for(int dimension, int leaf_size) {
  int padded = leaf_size;
  while (padded < dimension) {
    if (padded > (1 << 29)) return -1;
    padded *= 2;
  }
  return padded;
}

/* ---------------------------------------------------------------------------
 * Construction (quadtree.cpp:60-108 semantics from a leaf list)
 * ------------------------------------------------------------------------- */

static uint64_t morton2(uint32_t r, uint32_t c, int depth) {
  uint64_t key = 0;
  for (int b = depth - 1; b >= 0; --b) key = (key << 2) | (((r >> b) & 1u) << 1) | ((c >> b) & 1u);
  return key;
}

typedef struct {
  uint64_t key;
  int64_t index;
} keyed;

static int cmp_keyed(const void* x, const void* y) {
  const keyed* a = (const keyed*)x;
  const keyed* b = (const keyed*)y;
  if (a->key != b->key) return a->key < b->key ? -1 : 1;
  return a->index < b->index ? -1 : (a->index > b->index);
}

typedef struct {
  const keyed* order;
  const double* payload; /* or norms in norm-only mode */
  int depth;
  int64_t block;         /* L*L */
  int norm_only;
} build_ctx;

static ora_node* build_range(const build_ctx* bc, int64_t lo, int64_t hi, int level) {
  if (lo >= hi) return NULL;
  if (level == bc->depth) {
    const int64_t src = bc->order[lo].index;
    if (bc->norm_only) {
      const double nrm = bc->payload[src];
      if (nrm < 0.0) return NULL;
      ora_node* n = new_node();
      n->norm = nrm;
      return n;
    }
    double* blk = (double*)malloc(sizeof(double) * (size_t)bc->block);
    memcpy(blk, bc->payload + src * bc->block, sizeof(double) * (size_t)bc->block);
    return make_leaf(blk, bc->block);
  }
  const int shift = 2 * (bc->depth - level - 1);
  ora_node* child[4];
  int64_t start = lo;
  for (int c = 0; c < 4; ++c) {
    int64_t end = start;
    while (end < hi && (int)((bc->order[end].key >> shift) & 3u) == c) ++end;
    child[c] = build_range(bc, start, end, level + 1);
    start = end;
  }
  return make_inner(child);
}

static ora_tree* build_common(int dimension, int leaf_size, int64_t n_leaves, const int32_t* rows,
                              const int32_t* cols, const double* data, int norm_only) {
  if (dimension <= 0 || leaf_size <= 0) return NULL;
  const int padded = padded_dimension_for(dimension, leaf_size);
  if (padded < 0) return NULL;
  int depth = 0;
  while ((leaf_size << depth) < padded) ++depth;
  const int64_t limit = (dimension + leaf_size - 1) / leaf_size;
  keyed* order = (keyed*)malloc(sizeof(keyed) * (size_t)(n_leaves > 0 ? n_leaves : 1));
  for (int64_t t = 0; t < n_leaves; ++t) {
    if (rows[t] < 0 || cols[t] < 0 || rows[t] >= limit || cols[t] >= limit) {
      free(order);
      return NULL;
    }
    order[t].key = morton2((uint32_t)rows[t], (uint32_t)cols[t], depth);
    order[t].index = t;
  }
  qsort(order, (size_t)n_leaves, sizeof(keyed), cmp_keyed);
  for (int64_t t = 1; t < n_leaves; ++t)
    if (order[t].key == order[t - 1].key) {
      free(order);
      return NULL;
    }
  build_ctx bc = {order, data, depth, (int64_t)leaf_size * leaf_size, norm_only};
  ora_tree* tree = (ora_tree*)calloc(1, sizeof(ora_tree));
  tree->dimension = dimension;
  tree->padded = padded;
  tree->leaf_size = leaf_size;
  tree->depth = depth;
  tree->norm_only = norm_only;
  tree->root = build_range(&bc, 0, n_leaves, 0);
  free(order);
  return tree;
}

ora_tree* ora_build(int dimension, int leaf_size, int64_t n_leaves, const int32_t* block_rows,
                    const int32_t* block_cols, const double* payload) {
  return build_common(dimension, leaf_size, n_leaves, block_rows, block_cols, payload, 0);
}

ora_tree* ora_build_norm_only(int dimension, int leaf_size, int64_t n_leaves,
                              const int32_t* block_rows, const int32_t* block_cols,
                              const double* leaf_norms) {
  return build_common(dimension, leaf_size, n_leaves, block_rows, block_cols, leaf_norms, 1);
}

void ora_free(ora_tree* t) {
  if (!t) return;
  free_node(t->root);
  free(t);
}

int ora_dimension(const ora_tree* t) { return t->dimension; }
int ora_padded_dimension(const ora_tree* t) { return t->padded; }
int ora_leaf_size(const ora_tree* t) { return t->leaf_size; }
int ora_depth(const ora_tree* t) { return t->depth; }
double ora_frobenius(const ora_tree* t) { return t->root ? t->root->norm : 0.0; }

static int64_t count_leaves(const ora_node* n, int level, int depth) {
  if (!n) return 0;
  if (level == depth) return 1;
  int64_t s = 0;
  for (int c = 0; c < 4; ++c) s += count_leaves(n->child[c], level + 1, depth);
  return s;
}

int64_t ora_nnz_blocks(const ora_tree* t) { return count_leaves(t->root, 0, t->depth); }

typedef struct {
  int32_t* rows;
  int32_t* cols;
  double* payload;
  double* norms;
  int64_t next;
  int64_t block;
  int depth;
} leaf_walk;

static void walk_leaves(leaf_walk* w, const ora_node* n, int level, int32_t r, int32_t c) {
  if (!n) return;
  if (level == w->depth) {
    const int64_t at = w->next++;
    if (w->rows) w->rows[at] = r;
    if (w->cols) w->cols[at] = c;
    if (w->norms) w->norms[at] = n->norm;
    if (w->payload) {
      if (n->block)
        memcpy(w->payload + at * w->block, n->block, sizeof(double) * (size_t)w->block);
      else
        memset(w->payload + at * w->block, 0, sizeof(double) * (size_t)w->block);
    }
    return;
  }
  for (int q = 0; q < 4; ++q)
    walk_leaves(w, n->child[q], level + 1, 2 * r + (q >> 1), 2 * c + (q & 1));
}

void ora_leaves(const ora_tree* t, int32_t* rows, int32_t* cols, double* payload, double* norms) {
  leaf_walk w = {rows, cols, payload, norms, 0, (int64_t)t->leaf_size * t->leaf_size, t->depth};
  walk_leaves(&w, t->root, 0, 0, 0);
}

static void walk_level(const ora_node* n, int level, int target, uint64_t key, double* out) {
  if (!n) return;
  if (level == target) {
    out[key] = n->norm;
    return;
  }
  for (int q = 0; q < 4; ++q) walk_level(n->child[q], level + 1, target, key * 4 + (uint64_t)q, out);
}

void ora_level_norms(const ora_tree* t, int level, double* out) {
  const uint64_t count = 1ull << (2 * level);
  for (uint64_t i = 0; i < count; ++i) out[i] = -1.0;
  walk_level(t->root, 0, level, 0, out);
}

static int conformable(const ora_tree* a, const ora_tree* b) {
  return a->dimension == b->dimension && a->leaf_size == b->leaf_size;
}

/* ---------------------------------------------------------------------------
 * CSE sweep: error_control.cpp:34-79 (cse_quadrant / cse_node), :160-166
 * ------------------------------------------------------------------------- */

typedef struct {
  const double* taus;
  int n;
  int depth;
  double* scratch; /* per level: 4 contributions + 1 temporary */
} cse_ctx;

static void cse_node(const cse_ctx* cx, const ora_node* a, const ora_node* b, int level,
                     double* errors /* zeroed */) {
  if (!a || !b) return;                       /* :49 */
  const double norm_product = a->norm * b->norm; /* :50 */
  if (norm_product == 0.0) return;            /* :51 */
  const int n = cx->n;
  if (level == cx->depth) {                   /* :52-55 */
    for (int k = 0; k < n; ++k)
      if (norm_product < cx->taus[k]) errors[k] = norm_product;
    return;
  }
  double* contribution = cx->scratch + (size_t)level * 5 * n;
  double* e1 = contribution + 4 * (size_t)n;
  for (int row = 0; row < 2; ++row)
    for (int col = 0; col < 2; ++col) {
      /* cse_quadrant, :34-44: E_0 from k-half 0 plus E_1 from k-half 1 */
      double* e0 = contribution + (size_t)(2 * row + col) * n;
      memset(e0, 0, sizeof(double) * (size_t)n);
      cse_node(cx, a->child[2 * row + 0], b->child[2 * 0 + col], level + 1, e0);
      memset(e1, 0, sizeof(double) * (size_t)n);
      cse_node(cx, a->child[2 * row + 1], b->child[2 * 1 + col], level + 1, e1);
      for (int k = 0; k < n; ++k) e0[k] += e1[k];
    }
  /* :73-77 fixed quadrant order, then sqrt */
  for (int q = 0; q < 4; ++q) {
    const double* c = contribution + (size_t)q * n;
    for (int k = 0; k < n; ++k) errors[k] += c[k] * c[k];
  }
  for (int k = 0; k < n; ++k) errors[k] = sqrt(errors[k]);
}

int ora_cse(const ora_tree* a, const ora_tree* b, const double* taus, int n_taus, double* bounds) {
  if (!conformable(a, b) || n_taus < 1) return -1;
  cse_ctx cx = {taus, n_taus, a->depth, NULL};
  cx.scratch = (double*)malloc(sizeof(double) * 5 * (size_t)n_taus * (size_t)(a->depth + 1));
  memset(bounds, 0, sizeof(double) * (size_t)n_taus);
  cse_node(&cx, a->root, b->root, 0, bounds);
  free(cx.scratch);
  return 0;
}

static const ora_node* node_at(const ora_node* n, int level, int32_t r, int32_t c) {
  for (int l = level - 1; l >= 0 && n; --l) n = n->child[2 * ((r >> l) & 1) + ((c >> l) & 1)];
  return n;
}

int ora_cse_subtree(const ora_tree* a, const ora_tree* b, const double* taus, int n_taus, int level,
                    int32_t I, int32_t K, int32_t J, double* out) {
  if (!conformable(a, b) || n_taus < 1 || level < 0 || level > a->depth) return -1;
  cse_ctx cx = {taus, n_taus, a->depth, NULL};
  cx.scratch = (double*)malloc(sizeof(double) * 5 * (size_t)n_taus * (size_t)(a->depth + 1));
  memset(out, 0, sizeof(double) * (size_t)n_taus);
  cse_node(&cx, node_at(a->root, level, I, K), node_at(b->root, level, K, J), level, out);
  free(cx.scratch);
  return 0;
}

/* select_index: error_control.cpp:81-87. */
int ora_select_index(const double* bounds, int n_taus, double delta) {
  for (int k = 0; k < n_taus; ++k)
    if (bounds[k] < delta) return k;
  return -1;
}

/* ---------------------------------------------------------------------------
 * Products: multiply.cpp:16-20, 34-56, 61-92; quadtree.cpp:24-49
 * ------------------------------------------------------------------------- */

/* leaf_gemm: quadtree.cpp:38-49 -- j, k, i loop order, zero b skipped. */
static void leaf_gemm(const double* a, const double* b, double* c, int L) {
  for (int j = 0; j < L; ++j) {
    double* cj = c + (size_t)j * L;
    for (int k = 0; k < L; ++k) {
      const double bkj = b[k + (size_t)j * L];
      if (bkj == 0.0) continue;
      const double* ak = a + (size_t)k * L;
      for (int i = 0; i < L; ++i) cj[i] += ak[i] * bkj;
    }
  }
}

/* leaf_product: multiply.cpp:16-20. */
static ora_node* leaf_product(const ora_node* a, const ora_node* b, int L) {
  double* blk = (double*)calloc((size_t)L * L, sizeof(double));
  leaf_gemm(a->block, b->block, blk, L);
  return make_leaf(blk, (int64_t)L * L);
}

/* add_nodes: quadtree.cpp:24-36, consuming both (owned) operands. */
static ora_node* add_owned(ora_node* a, ora_node* b, int level, int depth, int L) {
  if (!a) return b;
  if (!b) return a;
  if (level == depth) {
    const int64_t count = (int64_t)L * L;
    double* sum = (double*)malloc(sizeof(double) * (size_t)count);
    for (int64_t i = 0; i < count; ++i) sum[i] = a->block[i] + b->block[i];
    free_node(a);
    free_node(b);
    return make_leaf(sum, count);
  }
  ora_node* child[4];
  for (int c = 0; c < 4; ++c) child[c] = add_owned(a->child[c], b->child[c], level + 1, depth, L);
  free(a->block);
  free(b->block);
  free(a);
  free(b);
  return make_inner(child);
}

typedef struct {
  double tau;
  int skip_test; /* 0 for multiply_exact */
  int depth;
  int L;
} mul_ctx;

/* spamm_node (multiply.cpp:70-92) / multiply_exact_node (:34-56). */
static ora_node* mul_node(const mul_ctx* m, const ora_node* a, const ora_node* b, int level) {
  if (!a || !b) return NULL;                                  /* :72 */
  if (m->skip_test && a->norm * b->norm < m->tau) return NULL; /* :73 */
  if (level == m->depth) return leaf_product(a, b, m->L);     /* :74 */
  ora_node* child[4];
  for (int row = 0; row < 2; ++row)
    for (int col = 0; col < 2; ++col) {
      /* spamm_quadrant :61-68 -- T0 from k-half 0, T1 from k-half 1, T0 + T1 */
      ora_node* t0 = mul_node(m, a->child[2 * row + 0], b->child[2 * 0 + col], level + 1);
      ora_node* t1 = mul_node(m, a->child[2 * row + 1], b->child[2 * 1 + col], level + 1);
      child[2 * row + col] = add_owned(t0, t1, level + 1, m->depth, m->L);
    }
  return make_inner(child);
}

static ora_tree* wrap(const ora_tree* like, ora_node* root) {
  ora_tree* t = (ora_tree*)calloc(1, sizeof(ora_tree));
  t->dimension = like->dimension;
  t->padded = like->padded;
  t->leaf_size = like->leaf_size;
  t->depth = like->depth;
  t->root = root;
  return t;
}

ora_tree* ora_spamm(const ora_tree* a, const ora_tree* b, double tau, int* status) {
  /* check_conformable :94-98; negative tau :112 */
  if (!conformable(a, b) || tau < 0.0 || a->norm_only || b->norm_only) {
    if (status) *status = -1;
    return NULL;
  }
  mul_ctx m = {tau, 1, a->depth, a->leaf_size};
  if (status) *status = 0;
  return wrap(a, mul_node(&m, a->root, b->root, 0));
}

ora_tree* ora_multiply_exact(const ora_tree* a, const ora_tree* b, int* status) {
  if (!conformable(a, b) || a->norm_only || b->norm_only) {
    if (status) *status = -1;
    return NULL;
  }
  mul_ctx m = {0.0, 0, a->depth, a->leaf_size};
  if (status) *status = 0;
  return wrap(a, mul_node(&m, a->root, b->root, 0));
}

/* ---------------------------------------------------------------------------
 * Surviving leaf-product set: the leaves mul_node reaches (multiply.cpp:70-92)
 * ------------------------------------------------------------------------- */

typedef struct {
  double tau;
  int depth;
  int skip_test;
  int zero_test; /* not used by spamm; ora_candidates counts every non-null pair */
  int64_t count;
  int64_t capacity;
  int32_t* out;
} surv_ctx;

static void surv_node(surv_ctx* s, const ora_node* a, const ora_node* b, int level, int32_t I,
                      int32_t K, int32_t J) {
  if (!a || !b) return;
  if (s->skip_test && a->norm * b->norm < s->tau) return;
  if (level == s->depth) {
    if (s->out && s->count < s->capacity) {
      s->out[3 * s->count + 0] = I;
      s->out[3 * s->count + 1] = K;
      s->out[3 * s->count + 2] = J;
    }
    ++s->count;
    return;
  }
  for (int row = 0; row < 2; ++row)
    for (int col = 0; col < 2; ++col)
      for (int h = 0; h < 2; ++h)
        surv_node(s, a->child[2 * row + h], b->child[2 * h + col], level + 1, 2 * I + row,
                  2 * K + h, 2 * J + col);
}

typedef struct {
  uint64_t key;
  int32_t t[3];
} surv_rec;

static int cmp_surv(const void* x, const void* y) {
  const surv_rec* a = (const surv_rec*)x;
  const surv_rec* b = (const surv_rec*)y;
  if (a->key != b->key) return a->key < b->key ? -1 : 1;
  return (a->t[1] > b->t[1]) - (a->t[1] < b->t[1]);
}

int64_t ora_survivors(const ora_tree* a, const ora_tree* b, double tau, int32_t* triples,
                      int64_t capacity) {
  surv_ctx s = {tau, a->depth, 1, 0, 0, 0, NULL};
  surv_node(&s, a->root, b->root, 0, 0, 0, 0);
  const int64_t total = s.count;
  if (!triples || capacity <= 0) return total;
  int32_t* raw = (int32_t*)malloc(sizeof(int32_t) * 3 * (size_t)(total > 0 ? total : 1));
  surv_ctx w = {tau, a->depth, 1, 0, 0, total, raw};
  surv_node(&w, a->root, b->root, 0, 0, 0, 0);
  surv_rec* rec = (surv_rec*)malloc(sizeof(surv_rec) * (size_t)(total > 0 ? total : 1));
  for (int64_t i = 0; i < total; ++i) {
    rec[i].t[0] = raw[3 * i];
    rec[i].t[1] = raw[3 * i + 1];
    rec[i].t[2] = raw[3 * i + 2];
    rec[i].key = morton2((uint32_t)rec[i].t[0], (uint32_t)rec[i].t[2], a->depth);
  }
  qsort(rec, (size_t)total, sizeof(surv_rec), cmp_surv);
  const int64_t n = total < capacity ? total : capacity;
  for (int64_t i = 0; i < n; ++i) memcpy(triples + 3 * i, rec[i].t, sizeof(int32_t) * 3);
  free(rec);
  free(raw);
  return total;
}

int64_t ora_candidates(const ora_tree* a, const ora_tree* b) {
  surv_ctx s = {0.0, a->depth, 0, 0, 0, 0, NULL};
  surv_node(&s, a->root, b->root, 0, 0, 0, 0);
  return s.count;
}

/* ---------------------------------------------------------------------------
 * Truncation: error_control.cpp:93-134 (collect_leaves / drop_leaves),
 * :174-201 (truncate)
 * ------------------------------------------------------------------------- */

typedef struct {
  double norm;
  int64_t position; /* block_row * blocks_per_side + block_col */
  int64_t index;    /* Morton-order leaf index */
} leaf_ref;

static int cmp_leaf_ref(const void* x, const void* y) {
  const leaf_ref* a = (const leaf_ref*)x;
  const leaf_ref* b = (const leaf_ref*)y;
  if (a->norm != b->norm) return a->norm < b->norm ? -1 : 1;
  return (a->position > b->position) - (a->position < b->position);
}

ora_tree* ora_truncate(const ora_tree* x, double delta, double* removed_norm,
                       int64_t* removed_count, int* status) {
  if (delta < 0.0) {
    if (status) *status = -1;
    return NULL;
  }
  const int64_t n = ora_nnz_blocks(x);
  const int64_t L2 = (int64_t)x->leaf_size * x->leaf_size;
  const int64_t side = (int64_t)1 << x->depth;
  int32_t* rows = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  int32_t* cols = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  double* norms = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double* payload = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n * L2 : 1));
  ora_leaves(x, rows, cols, payload, norms);
  leaf_ref* refs = (leaf_ref*)malloc(sizeof(leaf_ref) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    refs[i].norm = norms[i];
    refs[i].position = (int64_t)rows[i] * side + cols[i];
    refs[i].index = i;
  }
  qsort(refs, (size_t)n, sizeof(leaf_ref), cmp_leaf_ref);
  char* removed = (char*)calloc((size_t)(n > 0 ? n : 1), 1);
  double sumsq = 0.0;
  int64_t count = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (!(sqrt(sumsq + refs[i].norm * refs[i].norm) < delta)) break;
    sumsq += refs[i].norm * refs[i].norm;
    removed[refs[i].index] = 1;
    ++count;
  }
  int64_t kept = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (removed[i]) continue;
    rows[kept] = rows[i];
    cols[kept] = cols[i];
    memmove(payload + kept * L2, payload + i * L2, sizeof(double) * (size_t)L2);
    ++kept;
  }
  ora_tree* out = ora_build(x->dimension, x->leaf_size, kept, rows, cols, payload);
  free(rows);
  free(cols);
  free(norms);
  free(payload);
  free(refs);
  free(removed);
  if (removed_norm) *removed_norm = sqrt(sumsq);
  if (removed_count) *removed_count = count;
  if (status) *status = 0;
  return out;
}
