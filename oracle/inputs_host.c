/* inputs_host.c -- host generator of the seeded synthetic BASELINE inputs
 * (TEST / BENCH INFRASTRUCTURE ONLY: the reference arm of bench.py and the
 * CPU tests build their inputs with it, so the reference's timing never loads
 * the product library).
 *
 * It produces exactly the bits of the product's host generator
 * (spg_synth_chain_host / spg_synth_cluster_host, csrc/synth.cu; recipe in
 * DESIGN.md "Inputs"), multi-threaded: every entry is an independent function
 * of (seed, i, j), row sums are per-row sequential in ascending j, the scale
 * is their maximum, so the thread count never changes a bit.  It differs from
 * the DEVICE generator only through exp() (glibc vs libdevice).
 *
 *   u(seed, a, b) = (mix64(mix64(seed) ^ (a << 32 | b)) >> 11) * 2^-53
 *   chain:   A_ij = (2u - 1) * exp(-|i-j| / ell)
 *   cluster: n/4 sites uniform in a cube of side cbrt((n/4)/density), sorted by
 *            the Morton key of their 10-bit quantised coordinates; basis b sits
 *            on site b/4; A_ij = (2u - 1) * exp(-d_ij / ell) / max_i sum_j |.|
 *   |A_ij| < drop -> 0; all-zero blocks are left out; leaves in Morton order,
 *   column-major payload.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static double u01(uint64_t sm, uint32_t a, uint32_t b) {
  const uint64_t h = mix64(sm ^ (((uint64_t)a << 32) | b));
  return (double)(h >> 11) * 0x1.0p-53;
}

static double signed_u(uint64_t sm, uint32_t i, uint32_t j) {
  const uint32_t lo = i < j ? i : j, hi = i < j ? j : i;
  return 2.0 * u01(sm, lo, hi) - 1.0;
}

static uint64_t spread3(uint32_t x) {
  uint64_t v = x & 0x3ff;
  v = (v | (v << 16)) & 0x030000FFull;
  v = (v | (v << 8)) & 0x0300F00Full;
  v = (v | (v << 4)) & 0x030C30C3ull;
  v = (v | (v << 2)) & 0x09249249ull;
  return v;
}

static uint32_t compact2(uint64_t x) {
  x &= 0x5555555555555555ull;
  x = (x | (x >> 1)) & 0x3333333333333333ull;
  x = (x | (x >> 2)) & 0x0F0F0F0F0F0F0F0Full;
  x = (x | (x >> 4)) & 0x00FF00FF00FF00FFull;
  x = (x | (x >> 8)) & 0x0000FFFF0000FFFFull;
  x = (x | (x >> 16)) & 0x00000000FFFFFFFFull;
  return (uint32_t)x;
}

typedef struct {
  uint64_t key;
  int32_t idx;
} KeyIdx;

static int cmp_keyidx(const void* pa, const void* pb) {
  const KeyIdx* a = (const KeyIdx*)pa;
  const KeyIdx* b = (const KeyIdx*)pb;
  if (a->key != b->key) return a->key < b->key ? -1 : 1;
  return (a->idx > b->idx) - (a->idx < b->idx);
}

/* ---- the generator state shared by the worker threads ------------------- */
typedef struct {
  int kind; /* 0 chain, 1 cluster */
  int32_t n, L, nb, depth;
  double ell, drop, scale;
  uint64_t sm;
  const double* sites; /* cluster: 3 per site, Morton-sorted */
  /* block work list */
  const uint64_t* keys;
  int64_t n_keys;
  double* payload;   /* n_keys * L*L scratch, block t at t*L*L */
  uint8_t* nonzero;  /* per block */
  double* rowsum;    /* cluster pass 1 */
  int threads;
} Gen;

static double site_distance(const double* p, const double* q) {
  volatile double dx = p[0] - q[0], dy = p[1] - q[1], dz = p[2] - q[2];
  volatile double xx = dx * dx, yy = dy * dy, zz = dz * dz;
  volatile double s = xx + yy;
  s = s + zz;
  return sqrt((double)s);
}

static double raw_value(const Gen* g, int32_t i, int32_t j) {
  if (g->kind == 0) {
    const double d = (double)(i > j ? i - j : j - i);
    volatile double e = exp(-(d / g->ell));
    volatile double v = signed_u(g->sm, (uint32_t)i, (uint32_t)j) * e;
    return (double)v;
  }
  const double d = site_distance(&g->sites[3 * (i >> 2)], &g->sites[3 * (j >> 2)]);
  volatile double e = exp(-(d / g->ell));
  volatile double v = signed_u(g->sm, (uint32_t)i, (uint32_t)j) * e;
  return (double)v;
}

typedef struct {
  Gen* g;
  int t;
  int pass;
} Job;

static void* worker(void* arg) {
  Job* job = (Job*)arg;
  Gen* g = job->g;
  if (job->pass == 0) { /* cluster row sums, rows t, t+T, ... */
    for (int32_t i = job->t; i < g->n; i += g->threads) {
      double s = 0.0;
      for (int32_t j = 0; j < g->n; ++j) s += fabs(raw_value(g, i, j));
      g->rowsum[i] = s;
    }
    return NULL;
  }
  const int64_t LL = (int64_t)g->L * g->L;
  for (int64_t b = job->t; b < g->n_keys; b += g->threads) {
    const int32_t br = (int32_t)compact2(g->keys[b] >> 1), bc = (int32_t)compact2(g->keys[b]);
    double* blk = g->payload + b * LL;
    int any = 0;
    for (int32_t j = 0; j < g->L; ++j)
      for (int32_t i = 0; i < g->L; ++i) {
        const int32_t gi = br * g->L + i, gj = bc * g->L + j;
        double v = 0.0;
        if (gi < g->n && gj < g->n) {
          v = raw_value(g, gi, gj);
          if (g->kind == 1) {
            volatile double w = v / g->scale;
            v = (double)w;
          }
          if (fabs(v) < g->drop) v = 0.0;
        }
        blk[i + (int64_t)j * g->L] = v;
        any = any || v != 0.0;
      }
    g->nonzero[b] = (uint8_t)any;
  }
  return NULL;
}

static void run_pass(Gen* g, int pass) {
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)g->threads);
  Job* jobs = (Job*)malloc(sizeof(Job) * (size_t)g->threads);
  for (int t = 0; t < g->threads; ++t) {
    jobs[t].g = g;
    jobs[t].t = t;
    jobs[t].pass = pass;
    pthread_create(&th[t], NULL, worker, &jobs[t]);
  }
  for (int t = 0; t < g->threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
}

static int shape(int32_t n, int32_t L, int32_t* nb, int32_t* depth) {
  if (n <= 0 || L <= 0) return -1;
  int64_t padded = L;
  int d = 0;
  while (padded < n) {
    padded *= 2;
    ++d;
  }
  if (d > 20) return -1;
  *nb = (n + L - 1) / L;
  *depth = d;
  return 0;
}

/* Morton keys of the logical blocks (optionally only those `keep` accepts) */
static uint64_t* block_keys(const Gen* g, int64_t* count) {
  const uint64_t total = (uint64_t)1 << (2 * g->depth);
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(total ? total : 1));
  int64_t c = 0;
  for (uint64_t key = 0; key < total; ++key) {
    const uint32_t r = compact2(key >> 1), col = compact2(key);
    if (r >= (uint32_t)g->nb || col >= (uint32_t)g->nb) continue;
    if (g->kind == 0 && g->drop > 0.0) { /* chain: blocks that may hold an entry >= drop */
      const int64_t diff = (int64_t)r - (int64_t)col;
      int64_t gap = (diff < 0 ? -diff : diff) * g->L - (g->L - 1);
      if (gap < 0) gap = 0;
      if (!(exp(-((double)gap / g->ell)) >= g->drop * 0.5)) continue;
    }
    keys[c++] = key;
  }
  *count = c;
  return keys;
}

/* Generate, compact non-null blocks into the outputs (capacity in leaves).
 * Returns the number of non-null leaves, or -1 on bad arguments. */
static int64_t generate(Gen* g, int64_t capacity, int32_t* rows, int32_t* cols, double* payload) {
  int64_t n_keys = 0;
  uint64_t* keys = block_keys(g, &n_keys);
  const int64_t LL = (int64_t)g->L * g->L;
  g->keys = keys;
  g->n_keys = n_keys;
  /* generate straight into the caller's payload when it can hold every
   * candidate block, else into scratch */
  double* scratch = NULL;
  if (payload && capacity >= n_keys) {
    g->payload = payload;
  } else {
    scratch = (double*)malloc(sizeof(double) * (size_t)(n_keys ? n_keys : 1) * (size_t)LL);
    g->payload = scratch;
  }
  g->nonzero = (uint8_t*)malloc((size_t)(n_keys ? n_keys : 1));
  if (n_keys) run_pass(g, 1);
  int64_t out = 0;
  for (int64_t b = 0; b < n_keys; ++b) {
    if (!g->nonzero[b]) continue;
    if (payload && out < capacity) {
      rows[out] = (int32_t)compact2(keys[b] >> 1);
      cols[out] = (int32_t)compact2(keys[b]);
      if (g->payload + b * LL != payload + out * LL)
        memmove(payload + out * LL, g->payload + b * LL, sizeof(double) * (size_t)LL);
    }
    ++out;
  }
  free(g->nonzero);
  free(scratch);
  free(keys);
  return out;
}

int inp_chain(int32_t n, int32_t L, double ell, uint64_t seed, double drop, int threads,
              int64_t capacity, int32_t* rows, int32_t* cols, double* payload,
              int64_t* n_leaves) {
  Gen g;
  memset(&g, 0, sizeof g);
  if (!n_leaves || !(ell > 0.0) || shape(n, L, &g.nb, &g.depth)) return -1;
  g.kind = 0;
  g.n = n;
  g.L = L;
  g.ell = ell;
  g.drop = drop;
  g.sm = mix64(seed);
  g.threads = threads < 1 ? 1 : threads;
  *n_leaves = generate(&g, capacity, rows, cols, payload);
  return 0;
}

int inp_cluster(int32_t n, int32_t L, double ell, double density, uint64_t site_seed,
                uint64_t value_seed, double drop, int threads, int64_t capacity, int32_t* rows,
                int32_t* cols, double* payload, int64_t* n_leaves) {
  Gen g;
  memset(&g, 0, sizeof g);
  if (!n_leaves || n % 4 != 0 || !(ell > 0.0) || !(density > 0.0) ||
      shape(n, L, &g.nb, &g.depth))
    return -1;
  const int32_t n_sites = n / 4;
  const double box = cbrt((double)n_sites / density);
  const uint64_t ssm = mix64(site_seed);
  double* xyz = (double*)malloc(sizeof(double) * 3 * (size_t)n_sites);
  double* sorted = (double*)malloc(sizeof(double) * 3 * (size_t)n_sites);
  KeyIdx* order = (KeyIdx*)malloc(sizeof(KeyIdx) * (size_t)n_sites);
  for (int32_t s = 0; s < n_sites; ++s) {
    uint32_t q[3];
    for (int a = 0; a < 3; ++a) {
      const double x = box * u01(ssm, (uint32_t)s, (uint32_t)a);
      xyz[3 * s + a] = x;
      int64_t qi = (int64_t)(x / box * 1024.0);
      if (qi < 0) qi = 0;
      if (qi > 1023) qi = 1023;
      q[a] = (uint32_t)qi;
    }
    order[s].key = (spread3(q[0]) << 2) | (spread3(q[1]) << 1) | spread3(q[2]);
    order[s].idx = s;
  }
  qsort(order, (size_t)n_sites, sizeof(KeyIdx), cmp_keyidx);
  for (int32_t r = 0; r < n_sites; ++r)
    for (int a = 0; a < 3; ++a) sorted[3 * r + a] = xyz[3 * order[r].idx + a];
  free(xyz);
  free(order);
  g.kind = 1;
  g.n = n;
  g.L = L;
  g.ell = ell;
  g.drop = drop;
  g.sm = mix64(value_seed);
  g.sites = sorted;
  g.threads = threads < 1 ? 1 : threads;
  g.rowsum = (double*)malloc(sizeof(double) * (size_t)n);
  run_pass(&g, 0);
  double scale = 0.0;
  for (int32_t i = 0; i < n; ++i) scale = scale > g.rowsum[i] ? scale : g.rowsum[i];
  free(g.rowsum);
  g.rowsum = NULL;
  g.scale = scale;
  *n_leaves = generate(&g, capacity, rows, cols, payload);
  free(sorted);
  return 0;
}
