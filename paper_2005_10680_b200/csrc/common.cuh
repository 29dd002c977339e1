// common.cuh -- shared state, error plumbing and index helpers for the
// B200-native SpAMM library (libspamm_gpu.so).
//
// GPU quadtree layout:
//   * leaf payload: n_slots dense L x L FP64 blocks, column-major
//     (quadtree.cpp:93-99), in upload order; `slots` maps the Morton-sorted
//     non-null leaves to payload slots.
//   * grid_slot: dense Morton grid (4^depth int32) of the leaf level, payload
//     slot or -1 for an identically-zero (null) quadrant.
//   * pyramid: dense Morton grids of node norms for every level 0..depth,
//     concatenated (level l has 4^l doubles at offset (4^l - 1) / 3); -1.0
//     marks null.  Children of Morton node m at level l are 4m..4m+3 at level
//     l+1 in child-index order 2*row+col (node_ops.hpp:20), so every subtree
//     is a contiguous range at every level.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <stdexcept>
#include <string>
#include <vector>

#include "spamm_gpu.h"

namespace spg {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail(int code, const std::string& msg);
void set_last_error(const std::string& msg);

#define SPG_CUDA(expr)                                                                     \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      ::spg::fail(SPG_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e) + " (" +  \
                                 __FILE__ + ":" + std::to_string(__LINE__) + ")");         \
  } while (0)

#define SPG_CHECK_LAUNCH(ctx)                \
  do {                                       \
    SPG_CUDA(cudaGetLastError());            \
    (ctx)->launches++;                       \
  } while (0)

constexpr int kMaxDepth = 14;  // 4^14 Morton grid entries = 268M (2.1 GB norms) at most

}  // namespace spg

namespace spg {
// Per-context caching allocator.  Every kernel of a context runs on its one
// stream, so a freed block can be handed to the next request immediately
// (stream order makes the reuse safe).  The driver is only called while the
// working set grows (warm-up); steady-state calls never allocate, which keeps
// step times free of driver-pool stalls (measured up to 1.3 s with the
// stream-ordered pool).
struct DevicePool {
  std::multimap<size_t, void*> free_blocks;
  std::unordered_map<void*, size_t> live;
  size_t reserved = 0;
  void* alloc(size_t bytes, cudaStream_t s);
  void release(void* p);
  void trim(cudaStream_t s);
};
}  // namespace spg

struct spg_context {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // D2H of product chunks overlapping the GEMM
  cudaStream_t aux_stream = nullptr;   // second compute stream for chunked GEMMs
  cudaStream_t h2d_stream = nullptr;   // staged uploads (next input while this product runs)
  cudaEvent_t ev[8] = {};
  std::mutex mu;
  int64_t launches = 0;   // own kernels launched (evidence counter)
  int64_t lib_calls = 0;  // CUB primitives invoked
  int64_t task_budget = 0;  // task-list bytes per product before row chunking (0: free HBM)
  spg::DevicePool pool;
};

struct spg_matrix {
  spg_context* ctx = nullptr;
  int32_t dimension = 0, padded = 0, leaf = 0, depth = 0;
  int64_t nnzb = 0;     // non-null leaves
  int64_t n_slots = 0;  // payload slots (>= nnzb)
  double* payload = nullptr;    // n_slots * L * L (owned through payload_ref)
  std::shared_ptr<double> payload_ref;  // shared by matrices derived without copying (truncate)
  uint64_t* keys = nullptr;     // nnzb Morton keys, ascending
  int32_t* slots = nullptr;     // nnzb payload slots, aligned with keys
  int32_t* grid_slot = nullptr; // 4^depth
  double* pyramid = nullptr;    // sum_l 4^l
  double frob = 0.0;
  bool norms_only = false;      // norms of a host-resident B (spg_bstream): no payload
  const double** leaf_ptrs = nullptr;  // n_slots leaf addresses (GEMM B table), built on first use
  // norms_only: leaves (slots) sorted by block row; slots of block rows
  // [r0, r1) are [row_slot_begin[r0], row_slot_begin[r1]) (2^depth + 1 entries)
  std::vector<int64_t> row_slot_begin;
};

// B kept in host memory and streamed to the GPU in panels of block rows
// (SURVEY.md 8e, configs 4/5): leaves sorted by block row, panel p = block
// rows [panel_row[p], panel_row[p+1]) = leaves [panel_leaf[p], panel_leaf[p+1]).
// `norms` is a norm-only matrix whose grid_slot holds the sorted leaf index.
struct spg_bstream {
  spg_context* ctx = nullptr;
  spg_matrix* norms = nullptr;
  const double* host_payload = nullptr;
  bool registered = false;  // host payload page-locked by spg_bstream_create
  std::vector<int32_t> panel_row;
  std::vector<int64_t> panel_leaf;
  int64_t max_panel_leaves = 0;
};

namespace spg {

__host__ __device__ inline int64_t level_offset(int level) { return ((int64_t(1) << (2 * level)) - 1) / 3; }
__host__ __device__ inline int64_t pyramid_size(int depth) { return level_offset(depth + 1); }

__host__ __device__ inline uint64_t spread2(uint32_t x) {
  uint64_t v = x;
  v = (v | (v << 16)) & 0x0000FFFF0000FFFFull;
  v = (v | (v << 8)) & 0x00FF00FF00FF00FFull;
  v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0Full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}
__host__ __device__ inline uint32_t compact2(uint64_t v) {
  v &= 0x5555555555555555ull;
  v = (v | (v >> 1)) & 0x3333333333333333ull;
  v = (v | (v >> 2)) & 0x0F0F0F0F0F0F0F0Full;
  v = (v | (v >> 4)) & 0x00FF00FF00FF00FFull;
  v = (v | (v >> 8)) & 0x0000FFFF0000FFFFull;
  v = (v | (v >> 16)) & 0x00000000FFFFFFFFull;
  return static_cast<uint32_t>(v);
}
// Morton key with the row bit above the column bit at every level, so the
// two key bits of a level are the child index 2*row+col (node_ops.hpp:20).
__host__ __device__ inline uint64_t morton2(uint32_t row, uint32_t col) {
  return (spread2(row) << 1) | spread2(col);
}
__host__ __device__ inline uint32_t morton_row(uint64_t key) { return compact2(key >> 1); }
__host__ __device__ inline uint32_t morton_col(uint64_t key) { return compact2(key); }

// Device buffer owned by a context's pool.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  spg_context* c = nullptr;
  DevBuf() = default;
  DevBuf(size_t count, spg_context* ctx) : n(count), c(ctx) {
    if (count) p = static_cast<T*>(ctx->pool.alloc(count * sizeof(T), ctx->stream));
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), c(o.c) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    reset();
    p = o.p; n = o.n; c = o.c;
    o.p = nullptr; o.n = 0;
    return *this;
  }
  ~DevBuf() { reset(); }
  void reset() {
    if (p) c->pool.release(p);
    p = nullptr;
    n = 0;
  }
  // adopt a pool block allocated elsewhere
  static DevBuf adopt(T* ptr, size_t count, spg_context* ctx) {
    DevBuf b;
    b.p = ptr; b.n = count; b.c = ctx;
    return b;
  }
  T* release() { T* r = p; p = nullptr; n = 0; return r; }
  T* get() const { return p; }
};

template <typename T>
T* dev_alloc(size_t count, spg_context* ctx) {
  return count ? static_cast<T*>(ctx->pool.alloc(count * sizeof(T), ctx->stream)) : nullptr;
}
inline void dev_free(void* p, spg_context* ctx) {
  if (p) ctx->pool.release(p);
}

inline unsigned grid_for(int64_t work, int threads, int64_t cap = (int64_t(1) << 30)) {
  int64_t g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

// Scoped context lock + device guard.
struct CtxGuard {
  std::lock_guard<std::mutex> lock;
  explicit CtxGuard(spg_context* c) : lock(c->mu) { SPG_CUDA(cudaSetDevice(c->device)); }
};

// --- internal entry points shared between translation units -------------
// norms.cu
void leaf_norms(spg_context* ctx, const double* payload, int64_t n_slots, int leaf,
                int32_t dimension, int32_t nb_logical, const int32_t* slot_rows,
                const int32_t* slot_cols, double* norms, uint8_t* nonzero, int* bad_padding,
                cudaStream_t st = nullptr);
void build_pyramid(spg_context* ctx, spg_matrix* m, const double* slot_norms,
                   const uint8_t* slot_nonzero);
// matrix.cu
spg_matrix* matrix_from_device_leaves(spg_context* ctx, int32_t dimension, int32_t leaf,
                                      int64_t n_leaves, const int32_t* d_rows,
                                      const int32_t* d_cols, double* d_payload_owned);
spg_matrix* matrix_from_morton_blocks(spg_context* ctx, int32_t dimension, int32_t leaf,
                                      int64_t n_blocks, uint64_t* d_keys_owned,
                                      double* d_payload_owned);
void matrix_destroy(spg_matrix* m);
// one matrix from row chunks (disjoint block rows) -- leaves copied, norms recomputed (K1)
spg_matrix* concat_row_chunks(spg_context* ctx, const std::vector<spg_matrix*>& parts);
// New matrix over x's payload (shared) keeping the slots with keep[slot] != 0;
// slot_norms[slot] = cached leaf norm (K1 result) for kept slots.
spg_matrix* matrix_keep_slots(spg_context* ctx, const spg_matrix* x, const double* slot_norms,
                              const uint8_t* keep);
spg_matrix* controlled_product(spg_context* ctx, const spg_matrix* a, const spg_matrix* b,
                               double delta, const double* taus, int n_taus, double* bounds,
                               spg_controlled_stats* stats);
// algebra.cu
double trace_device(spg_context* ctx, const spg_matrix* m);
int64_t nnz_device(spg_context* ctx, const spg_matrix* m);
spg_matrix* axpby_device(spg_context* ctx, double alpha, const spg_matrix* a, double beta,
                         const spg_matrix* b);
spg_matrix* identity_device(spg_context* ctx, int32_t dimension, int32_t leaf);
// truncate.cu
spg_matrix* truncate_device(spg_context* ctx, const spg_matrix* x, double delta,
                            double* removed_norm, int64_t* removed_count);
void check_shape(int32_t dimension, int32_t leaf, int32_t* padded, int32_t* depth);
// Row shard of a product: level 0 = the whole matrix.
struct Shard {
  int level = 0;
  int index = 0;
};
// cse.cu -- with shard.level > 0, `out` receives the level-s partial bound
// vectors of the shard (4^level x n_taus, dense (K, J) order) instead of bounds
void cse_device(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, const double* taus,
                int n_taus, double* out, float* ms, Shard shard = {});
// spamm.cu -- with `host` set, C is streamed to the caller's host buffers
// chunk by chunk while the GEMM runs and no device matrix is returned
struct HostOut {
  int64_t capacity = 0;
  int32_t* rows = nullptr;
  int32_t* cols = nullptr;
  double* payload = nullptr;
  double* norms = nullptr;
  int64_t count = 0;
};
spg_matrix* spamm_device(spg_context* ctx, const spg_matrix* a, const spg_matrix* b, double tau,
                         bool skip_test, spg_spamm_stats* stats, Shard shard = {},
                         HostOut* host = nullptr);

int64_t copy_scalar_to_host_i64(spg_context* ctx, const int64_t* d);
// the matrix's leaf address table (payload + t L^2), built once on ctx->stream
const double* const* leaf_table(spg_context* ctx, const spg_matrix* m);
__global__ void leaf_ptr_kernel(const double* payload, int64_t n, int64_t LL, const double** out);

// the product with B streamed panel by panel from host memory; C identical
// (bitwise) to spamm_device with B resident
spg_matrix* spamm_streamed_device(spg_context* ctx, const spg_matrix* a, const spg_bstream* b,
                                  double tau, spg_spamm_stats* stats);
// matrix.cu: norm-only matrix from per-leaf norms (slot = leaf index);
// h_rows: the same block rows on the host, sorted ascending
spg_matrix* matrix_from_leaf_norms(spg_context* ctx, int32_t dimension, int32_t leaf,
                                   int64_t n_leaves, const int32_t* h_rows,
                                   const int32_t* d_rows, const int32_t* d_cols,
                                   const double* d_norms, const uint8_t* d_nonzero);

inline void require_payload(const spg_matrix* m) {
  if (m && m->norms_only)
    fail(SPG_EINVAL, "matrix holds the norms of a host-resident B only (use spg_spamm_streamed)");
}

// SPG_TRACE=1: synchronising host-side phase timer printed to stderr
// (diagnostics only; off by default, never used for reported numbers).
struct PhaseTrace {
  spg_context* ctx;
  const char* what;
  double t0;
  bool on;
  PhaseTrace(spg_context* c, const char* w);
  ~PhaseTrace();
};

}  // namespace spg

// Wrap an API body: translate exceptions to status codes + last error.
#define SPG_API_BEGIN try {
#define SPG_API_END                                        \
  return SPG_OK;                                           \
  }                                                        \
  catch (const ::spg::Error& e) {                          \
    ::spg::set_last_error(e.what());                       \
    return e.code;                                         \
  }                                                        \
  catch (const std::bad_alloc&) {                          \
    ::spg::set_last_error("out of host memory");           \
    return SPG_ENOMEM;                                     \
  }                                                        \
  catch (const std::exception& e) {                        \
    ::spg::set_last_error(e.what());                       \
    return SPG_EINTERNAL;                                  \
  }
