// matrix.cu -- device-resident quadtree matrices: build (upload), inspect,
// download; the context and error plumbing of the C ABI.
//
// Reference interfaces replaced: QuadTreeMatrix::from_coordinates /
// from_dense / zero / to_dense / nnz_blocks / frobenius_norm
// (quadtree.hpp:52-83, quadtree.cpp:198-247).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>

#include <thrust/iterator/counting_iterator.h>

#include "common.cuh"

namespace spg {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

[[noreturn]] void fail(int code, const std::string& msg) { throw Error(code, msg); }

static bool trace_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SPG_TRACE");
    return e && e[0] == '1';
  }();
  return on;
}
static double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
PhaseTrace::PhaseTrace(spg_context* c, const char* w) : ctx(c), what(w), t0(0), on(trace_enabled()) {
  if (on) {
    cudaStreamSynchronize(ctx->stream);
    t0 = now_ms();
  }
}
PhaseTrace::~PhaseTrace() {
  if (on) {
    cudaStreamSynchronize(ctx->stream);
    std::fprintf(stderr, "[spg] %-28s %9.3f ms\n", what, now_ms() - t0);
  }
}

// Block sizes between 1 MB and 16 GB are rounded up to eight classes per
// octave (at most 12.5 % over the request): task-list buffers follow the
// survivor count, which differs a little from product to product, and exact
// sizes missed the cache -- a cudaMalloc (and, with the device nearly full, a
// trim of the whole cache) between two kernels showed up as 200-500 ms
// task-list times on single cells.  Larger blocks (operand and product
// payloads of configs 4/5, within a few GB of the device's capacity) stay
// exact.
static size_t size_class(size_t bytes) {
  if (bytes < (size_t(1) << 20) || bytes >= (size_t(16) << 30)) return bytes;
  size_t step = size_t(1) << 17;  // octave / 8 for the first octave (1 MB)
  while ((step << 4) <= bytes) step <<= 1;
  return (bytes + step - 1) / step * step;
}

void* DevicePool::alloc(size_t bytes, cudaStream_t s) {
  bytes = size_class((bytes + 511) & ~size_t(511));
  // best fit among cached blocks, wasting at most half of a small block and
  // an eighth of a large one (config-4-sized products run within a few GB of
  // the device's capacity: 2x blocks of several GB each exhausted it)
  auto it = free_blocks.lower_bound(bytes);
  const size_t slack = bytes < (size_t(256) << 20) ? bytes + (size_t(1) << 20) : bytes / 8;
  if (it != free_blocks.end() && it->first <= bytes + slack) {
    void* p = it->second;
    live[p] = it->first;
    free_blocks.erase(it);
    return p;
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaErrorMemoryAllocation && !free_blocks.empty()) {
    // out of memory: return cached blocks to the driver, largest first, only
    // until the request fits
    cudaGetLastError();
    cudaStreamSynchronize(s);
    while (e == cudaErrorMemoryAllocation && !free_blocks.empty()) {
      auto last = std::prev(free_blocks.end());
      cudaFree(last->second);
      reserved -= last->first;
      free_blocks.erase(last);
      e = cudaMalloc(&p, bytes);
      if (e == cudaErrorMemoryAllocation) cudaGetLastError();
    }
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(e == cudaErrorMemoryAllocation ? SPG_ENOMEM : SPG_ECUDA,
         std::string("device allocation of ") + std::to_string(bytes) +
             " bytes failed: " + cudaGetErrorString(e));
  }
  reserved += bytes;
  live[p] = bytes;
  return p;
}

void DevicePool::release(void* p) {
  auto it = live.find(p);
  if (it == live.end()) return;
  free_blocks.emplace(it->second, p);
  live.erase(it);
}

void DevicePool::trim(cudaStream_t s) {
  cudaStreamSynchronize(s);
  for (auto& kv : free_blocks) {
    cudaFree(kv.second);
    reserved -= kv.first;
  }
  free_blocks.clear();
}

int64_t copy_scalar_to_host_i64(spg_context* ctx, const int64_t* d) {
  int64_t h = 0;
  SPG_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  return h;
}

// padded_dimension_for (quadtree.cpp:15-22) + validate_shape (:55-58).
void check_shape(int32_t dimension, int32_t leaf, int32_t* padded, int32_t* depth) {
  if (dimension <= 0) fail(SPG_EINVAL, "dimension must be positive");
  if (leaf <= 0) fail(SPG_EINVAL, "leaf_size must be positive");
  int64_t p = leaf;
  int d = 0;
  while (p < dimension) {
    if (p > (int64_t(1) << 29)) fail(SPG_EINVAL, "dimension too large to pad");
    p *= 2;
    ++d;
  }
  if (d > kMaxDepth) fail(SPG_EINVAL, "quadtree depth exceeds the device grid limit");
  *padded = static_cast<int32_t>(p);
  *depth = d;
}

namespace {

// Scatter uploaded leaves into the Morton grid; detects range errors
// (std::out_of_range, quadtree.cpp:202-208) and duplicates
// (std::invalid_argument, quadtree.cpp:213-216).
__global__ void scatter_leaves(const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                               int64_t n, int32_t nb_logical, int32_t* __restrict__ grid_slot,
                               int* __restrict__ flags) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int32_t r = rows[t], c = cols[t];
  if (r < 0 || c < 0 || r >= nb_logical || c >= nb_logical) {
    atomicOr(flags, 1);
    return;
  }
  const uint64_t key = morton2(static_cast<uint32_t>(r), static_cast<uint32_t>(c));
  const int32_t prev = atomicCAS(grid_slot + key, -1, static_cast<int32_t>(t));
  if (prev != -1) atomicOr(flags, 2);
}

__global__ void scatter_keys(const uint64_t* __restrict__ keys, int64_t n,
                             int32_t* __restrict__ grid_slot, int32_t* __restrict__ rows,
                             int32_t* __restrict__ cols) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const uint64_t key = keys[t];
  grid_slot[key] = static_cast<int32_t>(t);
  rows[t] = static_cast<int32_t>(morton_row(key));
  cols[t] = static_cast<int32_t>(morton_col(key));
}

struct NonNull {
  const int32_t* grid;
  __host__ __device__ bool operator()(const uint64_t& p) const { return grid[p] >= 0; }
};

__global__ void gather_slots(const uint64_t* __restrict__ keys, int64_t n,
                             const int32_t* __restrict__ grid_slot, int32_t* __restrict__ slots) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  slots[t] = grid_slot[keys[t]];
}

// Compact the non-null grid positions into (keys, slots), ascending Morton.
void compact_leaves(spg_context* ctx, spg_matrix* m) {
  const int64_t count = int64_t(1) << (2 * m->depth);
  DevBuf<uint64_t> keys(std::max<int64_t>(count, 1), ctx);
  DevBuf<int64_t> n_sel(1, ctx);
  thrust::counting_iterator<uint64_t> it(0);
  size_t tmp_bytes = 0;
  SPG_CUDA(cub::DeviceSelect::If(nullptr, tmp_bytes, it, keys.get(), n_sel.get(), count,
                                 NonNull{m->grid_slot}, ctx->stream));
  DevBuf<uint8_t> tmp(tmp_bytes, ctx);
  SPG_CUDA(cub::DeviceSelect::If(tmp.get(), tmp_bytes, it, keys.get(), n_sel.get(), count,
                                 NonNull{m->grid_slot}, ctx->stream));
  ctx->lib_calls++;  // CUB device-wide primitive (library kernels)
  m->nnzb = copy_scalar_to_host_i64(ctx, n_sel.get());
  m->keys = dev_alloc<uint64_t>(std::max<int64_t>(m->nnzb, 1), ctx);
  m->slots = dev_alloc<int32_t>(std::max<int64_t>(m->nnzb, 1), ctx);
  if (m->nnzb) {
    SPG_CUDA(cudaMemcpyAsync(m->keys, keys.get(), m->nnzb * sizeof(uint64_t),
                             cudaMemcpyDeviceToDevice, ctx->stream));
    gather_slots<<<grid_for(m->nnzb, 256), 256, 0, ctx->stream>>>(m->keys, m->nnzb, m->grid_slot,
                                                                  m->slots);
    SPG_CHECK_LAUNCH(ctx);
  }
}

spg_matrix* new_matrix(spg_context* ctx, int32_t dimension, int32_t leaf) {
  auto m = std::make_unique<spg_matrix>();
  m->ctx = ctx;
  m->dimension = dimension;
  m->leaf = leaf;
  check_shape(dimension, leaf, &m->padded, &m->depth);
  const int64_t cells = int64_t(1) << (2 * m->depth);
  m->grid_slot = dev_alloc<int32_t>(cells, ctx);
  SPG_CUDA(cudaMemsetAsync(m->grid_slot, 0xff, cells * sizeof(int32_t), ctx->stream));
  m->pyramid = dev_alloc<double>(pyramid_size(m->depth), ctx);
  return m.release();
}

void finish_matrix(spg_context* ctx, spg_matrix* m, const int32_t* slot_rows,
                   const int32_t* slot_cols, bool check_padding) {
  const int32_t nb_logical = (m->dimension + m->leaf - 1) / m->leaf;
  DevBuf<double> norms(std::max<int64_t>(m->n_slots, 1), ctx);
  DevBuf<uint8_t> nonzero(std::max<int64_t>(m->n_slots, 1), ctx);
  DevBuf<int> bad(1, ctx);
  SPG_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), ctx->stream));
  leaf_norms(ctx, m->payload, m->n_slots, m->leaf, m->dimension, nb_logical,
             check_padding ? slot_rows : nullptr, slot_cols, norms.get(), nonzero.get(),
             bad.get());
  int h_bad = 0;
  SPG_CUDA(cudaMemcpyAsync(&h_bad, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  build_pyramid(ctx, m, norms.get(), nonzero.get());
  compact_leaves(ctx, m);  // synchronises
  if (h_bad) fail(SPG_EINVAL, "nonzero entry in the padding region of a boundary leaf");
  double root = -1.0;
  SPG_CUDA(cudaMemcpyAsync(&root, m->pyramid, sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  m->frob = root < 0.0 ? 0.0 : root;
}

__global__ void gather_payload(const double* __restrict__ payload,
                               const int32_t* __restrict__ slots, int64_t n, int64_t elems,
                               double* __restrict__ out) {
  const int64_t leaf = blockIdx.y + static_cast<int64_t>(gridDim.y) * blockIdx.z;
  if (leaf >= n) return;
  const double* src = payload + static_cast<int64_t>(slots[leaf]) * elems;
  double* dst = out + leaf * elems;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < elems;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[e] = src[e];
}

__global__ void gather_norms(const uint64_t* __restrict__ keys, int64_t n,
                             const double* __restrict__ level, double* __restrict__ out) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  out[t] = level[keys[t]];
}

// Non-null leaves of block rows [r0, r0 + rows) in (row, col) order: cell
// (r, c) of the panel in row-major order is flagged when its grid slot is
// non-null (within a block row, Morton order is column order).
__global__ void panel_cell_flags(const int32_t* __restrict__ grid_slot, int32_t r0, int32_t rows,
                                 int32_t nbp, uint8_t* __restrict__ flags) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<int64_t>(rows) * nbp) return;
  const uint32_t r = static_cast<uint32_t>(r0 + t / nbp), c = static_cast<uint32_t>(t % nbp);
  flags[t] = grid_slot[morton2(r, c)] >= 0;
}

__global__ void panel_gather(const double* __restrict__ payload,
                             const int32_t* __restrict__ grid_slot,
                             const int64_t* __restrict__ cells, const int64_t* __restrict__ n_sel,
                             int32_t r0, int32_t nbp, int64_t capacity, int64_t elems,
                             double* __restrict__ out) {
  const int64_t n = *n_sel < capacity ? *n_sel : capacity;
  for (int64_t i = blockIdx.y; i < n; i += gridDim.y) {
    const int64_t t = cells[i];
    const uint32_t r = static_cast<uint32_t>(r0 + t / nbp), c = static_cast<uint32_t>(t % nbp);
    const double* src = payload + static_cast<int64_t>(grid_slot[morton2(r, c)]) * elems;
    double* dst = out + i * elems;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < elems;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x)
      dst[e] = src[e];
  }
}

}  // namespace

__global__ void leaf_ptr_kernel(const double* payload, int64_t n, int64_t LL,
                                const double** out) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n) out[t] = payload + t * LL;
}

const double* const* leaf_table(spg_context* ctx, const spg_matrix* m) {
  // cached in the matrix, from its own context's pool: only on that context
  // (another context's call may run concurrently with the owner's)
  if (!m->payload || m->n_slots == 0 || m->ctx != ctx) return nullptr;
  auto* mm = const_cast<spg_matrix*>(m);  // cache: built once, read-only afterwards
  if (!mm->leaf_ptrs) {
    mm->leaf_ptrs = dev_alloc<const double*>(m->n_slots, ctx);
    leaf_ptr_kernel<<<grid_for(m->n_slots, 256), 256, 0, ctx->stream>>>(
        m->payload, m->n_slots, static_cast<int64_t>(m->leaf) * m->leaf, mm->leaf_ptrs);
    SPG_CHECK_LAUNCH(ctx);
  }
  return mm->leaf_ptrs;
}

void matrix_destroy(spg_matrix* m) {
  if (!m) return;
  spg_context* ctx = m->ctx;
  dev_free(m->leaf_ptrs, ctx);
  m->payload_ref.reset();  // returns the payload to the pool with its last user
  dev_free(m->keys, ctx);
  dev_free(m->slots, ctx);
  dev_free(m->grid_slot, ctx);
  dev_free(m->pyramid, ctx);
  delete m;
}

spg_matrix* matrix_from_device_leaves(spg_context* ctx, int32_t dimension, int32_t leaf,
                                      int64_t n_leaves, const int32_t* d_rows,
                                      const int32_t* d_cols, double* d_payload_owned) {
  std::unique_ptr<spg_matrix, void (*)(spg_matrix*)> m(nullptr, matrix_destroy);
  try {
    m.reset(new_matrix(ctx, dimension, leaf));
  } catch (...) {
    dev_free(d_payload_owned, ctx);
    throw;
  }
  m->payload = d_payload_owned;
  m->payload_ref = std::shared_ptr<double>(d_payload_owned,
                                           [ctx](double* p) { dev_free(p, ctx); });
  m->n_slots = n_leaves;
  if (n_leaves > (int64_t(1) << 31) - 1) fail(SPG_EINVAL, "too many leaves");
  const int32_t nb_logical = (dimension + leaf - 1) / leaf;
  DevBuf<int> flags(1, ctx);
  SPG_CUDA(cudaMemsetAsync(flags.get(), 0, sizeof(int), ctx->stream));
  if (n_leaves) {
    scatter_leaves<<<grid_for(n_leaves, 256), 256, 0, ctx->stream>>>(
        d_rows, d_cols, n_leaves, nb_logical, m->grid_slot, flags.get());
    SPG_CHECK_LAUNCH(ctx);
  }
  int h_flags = 0;
  SPG_CUDA(cudaMemcpyAsync(&h_flags, flags.get(), sizeof(int), cudaMemcpyDeviceToHost,
                           ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h_flags & 1) fail(SPG_ERANGE, "block coordinate outside the matrix dimension");
  if (h_flags & 2) fail(SPG_EINVAL, "duplicate block coordinate");
  finish_matrix(ctx, m.get(), d_rows, d_cols, true);
  return m.release();
}

spg_matrix* matrix_from_leaf_norms(spg_context* ctx, int32_t dimension, int32_t leaf,
                                   int64_t n_leaves, const int32_t* h_rows,
                                   const int32_t* d_rows, const int32_t* d_cols,
                                   const double* d_norms, const uint8_t* d_nonzero) {
  std::unique_ptr<spg_matrix, void (*)(spg_matrix*)> m(new_matrix(ctx, dimension, leaf),
                                                       matrix_destroy);
  m->norms_only = true;
  m->n_slots = n_leaves;
  const int32_t nbp = 1 << m->depth;
  m->row_slot_begin.resize(static_cast<size_t>(nbp) + 1);
  for (int32_t r = 0; r <= nbp; ++r)
    m->row_slot_begin[r] = std::lower_bound(h_rows, h_rows + n_leaves, r) - h_rows;
  if (n_leaves > (int64_t(1) << 31) - 1) fail(SPG_EINVAL, "too many leaves");
  const int32_t nb_logical = (dimension + leaf - 1) / leaf;
  DevBuf<int> flags(1, ctx);
  SPG_CUDA(cudaMemsetAsync(flags.get(), 0, sizeof(int), ctx->stream));
  if (n_leaves) {
    scatter_leaves<<<grid_for(n_leaves, 256), 256, 0, ctx->stream>>>(
        d_rows, d_cols, n_leaves, nb_logical, m->grid_slot, flags.get());
    SPG_CHECK_LAUNCH(ctx);
  }
  int h_flags = 0;
  SPG_CUDA(cudaMemcpyAsync(&h_flags, flags.get(), sizeof(int), cudaMemcpyDeviceToHost,
                           ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h_flags & 1) fail(SPG_ERANGE, "block coordinate outside the matrix dimension");
  if (h_flags & 2) fail(SPG_EINVAL, "duplicate block coordinate");
  build_pyramid(ctx, m.get(), d_norms, d_nonzero);
  compact_leaves(ctx, m.get());
  double root = -1.0;
  SPG_CUDA(cudaMemcpyAsync(&root, m->pyramid, sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  m->frob = root < 0.0 ? 0.0 : root;
  return m.release();
}

spg_matrix* matrix_keep_slots(spg_context* ctx, const spg_matrix* x, const double* slot_norms,
                              const uint8_t* keep) {
  std::unique_ptr<spg_matrix, void (*)(spg_matrix*)> m(new_matrix(ctx, x->dimension, x->leaf),
                                                       matrix_destroy);
  m->payload = x->payload;
  m->payload_ref = x->payload_ref;
  m->n_slots = x->n_slots;
  const int64_t cells = int64_t(1) << (2 * x->depth);
  SPG_CUDA(cudaMemcpyAsync(m->grid_slot, x->grid_slot, cells * sizeof(int32_t),
                           cudaMemcpyDeviceToDevice, ctx->stream));
  build_pyramid(ctx, m.get(), slot_norms, keep);  // removed slots -> null
  compact_leaves(ctx, m.get());
  double root = -1.0;
  SPG_CUDA(cudaMemcpyAsync(&root, m->pyramid, sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  m->frob = root < 0.0 ? 0.0 : root;
  return m.release();
}

spg_matrix* matrix_from_morton_blocks(spg_context* ctx, int32_t dimension, int32_t leaf,
                                      int64_t n_blocks, uint64_t* d_keys_owned,
                                      double* d_payload_owned) {
  std::unique_ptr<spg_matrix, void (*)(spg_matrix*)> m(nullptr, matrix_destroy);
  try {
    m.reset(new_matrix(ctx, dimension, leaf));
  } catch (...) {
    dev_free(d_payload_owned, ctx);
    dev_free(d_keys_owned, ctx);
    throw;
  }
  m->payload = d_payload_owned;
  m->payload_ref = std::shared_ptr<double>(d_payload_owned,
                                           [ctx](double* p) { dev_free(p, ctx); });
  m->n_slots = n_blocks;
  DevBuf<uint64_t> keys = DevBuf<uint64_t>::adopt(d_keys_owned, n_blocks, ctx);
  DevBuf<int32_t> rows(std::max<int64_t>(n_blocks, 1), ctx);
  DevBuf<int32_t> cols(std::max<int64_t>(n_blocks, 1), ctx);
  if (n_blocks) {
    scatter_keys<<<grid_for(n_blocks, 256), 256, 0, ctx->stream>>>(
        d_keys_owned, n_blocks, m->grid_slot, rows.get(), cols.get());
    SPG_CHECK_LAUNCH(ctx);
  }
  finish_matrix(ctx, m.get(), rows.get(), cols.get(), false);
  return m.release();
}

namespace {
__global__ void pack_chunk(const uint64_t* __restrict__ keys, const int32_t* __restrict__ slots,
                           int64_t n, const double* __restrict__ payload, int64_t LL,
                           uint64_t* __restrict__ out_keys, double* __restrict__ out) {
  for (int64_t t = blockIdx.x; t < n; t += gridDim.x) {
    if (threadIdx.x == 0) out_keys[t] = keys[t];
    const double* src = payload + static_cast<int64_t>(slots[t]) * LL;
    for (int64_t e = threadIdx.x; e < LL; e += blockDim.x) out[t * LL + e] = src[e];
  }
}
}  // namespace

spg_matrix* concat_row_chunks(spg_context* ctx, const std::vector<spg_matrix*>& parts) {
  if (parts.empty()) fail(SPG_EINTERNAL, "concat: no parts");
  const spg_matrix* f = parts[0];
  const int64_t LL = static_cast<int64_t>(f->leaf) * f->leaf;
  int64_t total = 0;
  for (const spg_matrix* m : parts) total += m->nnzb;
  double* pay = dev_alloc<double>(std::max<int64_t>(total * LL, 1), ctx);
  uint64_t* keys = nullptr;
  try {
    keys = dev_alloc<uint64_t>(std::max<int64_t>(total, 1), ctx);
    int64_t off = 0;
    for (const spg_matrix* m : parts) {
      if (m->nnzb) {
        pack_chunk<<<grid_for(m->nnzb, 1, 1 << 20), 256, 0, ctx->stream>>>(
            m->keys, m->slots, m->nnzb, m->payload, LL, keys + off, pay + off * LL);
        SPG_CHECK_LAUNCH(ctx);
      }
      off += m->nnzb;
    }
  } catch (...) {
    dev_free(pay, ctx);
    if (keys) dev_free(keys, ctx);
    throw;
  }
  return matrix_from_morton_blocks(ctx, f->dimension, f->leaf, total, keys, pay);
}

}  // namespace spg

using namespace spg;

extern "C" {

const char* spg_last_error(void) { return spg::g_last_error.c_str(); }

int spg_version(void) { return 1; }

int spg_device_count(int* count) {
  SPG_API_BEGIN
  if (!count) fail(SPG_EINVAL, "null output");
  *count = 0;
  SPG_CUDA(cudaGetDeviceCount(count));
  SPG_API_END
}

int spg_context_create(int device, spg_context** out) {
  SPG_API_BEGIN
  if (!out) fail(SPG_EINVAL, "null output");
  *out = nullptr;
  auto ctx = std::make_unique<spg_context>();
  ctx->device = device;
  SPG_CUDA(cudaSetDevice(device));
  SPG_CUDA(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device));
  SPG_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  SPG_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  SPG_CUDA(cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking));
  SPG_CUDA(cudaStreamCreateWithFlags(&ctx->h2d_stream, cudaStreamNonBlocking));
  for (auto& e : ctx->ev) SPG_CUDA(cudaEventCreate(&e));
  *out = ctx.release();
  SPG_API_END
}

int spg_context_destroy(spg_context* ctx) {
  SPG_API_BEGIN
  if (!ctx) return SPG_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  ctx->pool.trim(ctx->stream);
  for (auto& kv : ctx->pool.live) cudaFree(kv.first);
  ctx->pool.live.clear();
  for (auto& e : ctx->ev) cudaEventDestroy(e);
  cudaStreamDestroy(ctx->stream);
  cudaStreamDestroy(ctx->copy_stream);
  cudaStreamDestroy(ctx->aux_stream);
  cudaStreamDestroy(ctx->h2d_stream);
  delete ctx;
  SPG_API_END
}

int spg_context_stream(spg_context* ctx, void** stream) {
  SPG_API_BEGIN
  if (!ctx || !stream) fail(SPG_EINVAL, "null argument");
  *stream = ctx->stream;
  SPG_API_END
}

int spg_context_synchronize(spg_context* ctx) {
  SPG_API_BEGIN
  if (!ctx) fail(SPG_EINVAL, "null context");
  CtxGuard g(ctx);
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  SPG_API_END
}

int spg_context_set_task_budget(spg_context* ctx, int64_t bytes) {
  SPG_API_BEGIN
  if (!ctx) fail(SPG_EINVAL, "null context");
  if (bytes < 0) fail(SPG_EINVAL, "task budget must be >= 0");
  ctx->task_budget = bytes;
  SPG_API_END
}

int spg_context_trim(spg_context* ctx) {
  SPG_API_BEGIN
  if (!ctx) fail(SPG_EINVAL, "null context");
  std::lock_guard<std::mutex> lock(ctx->mu);
  ctx->pool.trim(ctx->stream);
  SPG_API_END
}

int spg_context_launch_count(spg_context* ctx, int64_t* launches) {
  SPG_API_BEGIN
  if (!ctx || !launches) fail(SPG_EINVAL, "null argument");
  *launches = ctx->launches;
  SPG_API_END
}

int spg_matrix_upload(spg_context* ctx, int32_t dimension, int32_t leaf_size, int64_t n_leaves,
                      const int32_t* block_rows, const int32_t* block_cols, const double* payload,
                      spg_matrix** out) {
  SPG_API_BEGIN
  if (!ctx || !out) fail(SPG_EINVAL, "null argument");
  *out = nullptr;
  if (n_leaves < 0) fail(SPG_EINVAL, "negative leaf count");
  if (n_leaves && (!block_rows || !block_cols || !payload)) fail(SPG_EINVAL, "null leaf arrays");
  CtxGuard g(ctx);
  int32_t padded, depth;
  check_shape(dimension, leaf_size, &padded, &depth);
  const int64_t elems = static_cast<int64_t>(leaf_size) * leaf_size;
  DevBuf<int32_t> rows(std::max<int64_t>(n_leaves, 1), ctx);
  DevBuf<int32_t> cols(std::max<int64_t>(n_leaves, 1), ctx);
  double* d_payload = dev_alloc<double>(std::max<int64_t>(n_leaves * elems, 1), ctx);
  DevBuf<double> payload_guard = DevBuf<double>::adopt(d_payload, 1, ctx);
  if (n_leaves) {
    SPG_CUDA(cudaMemcpyAsync(rows.get(), block_rows, n_leaves * sizeof(int32_t),
                             cudaMemcpyHostToDevice, ctx->stream));
    SPG_CUDA(cudaMemcpyAsync(cols.get(), block_cols, n_leaves * sizeof(int32_t),
                             cudaMemcpyHostToDevice, ctx->stream));
    SPG_CUDA(cudaMemcpyAsync(d_payload, payload, n_leaves * elems * sizeof(double),
                             cudaMemcpyHostToDevice, ctx->stream));
  }
  payload_guard.release();
  *out = matrix_from_device_leaves(ctx, dimension, leaf_size, n_leaves, rows.get(), cols.get(),
                                   d_payload);
  SPG_API_END
}

// ---- staged uploads: the copies run on the context's h2d stream, so the
// next input streams in while the current product computes
}  // extern "C"

struct spg_staged {
  spg_context* ctx = nullptr;
  int32_t dimension = 0, leaf = 0;
  int64_t n = 0;
  spg::DevBuf<int32_t> rows, cols;
  double* payload = nullptr;
  cudaEvent_t done = nullptr;
  ~spg_staged() {
    if (payload) spg::dev_free(payload, ctx);
    if (done) cudaEventDestroy(done);
  }
};

extern "C" {

int spg_matrix_stage(spg_context* ctx, int32_t dimension, int32_t leaf_size, int64_t n_leaves,
                     const int32_t* block_rows, const int32_t* block_cols, const double* payload,
                     spg_staged** out) {
  SPG_API_BEGIN
  if (!ctx || !out) fail(SPG_EINVAL, "null argument");
  *out = nullptr;
  if (n_leaves < 0) fail(SPG_EINVAL, "negative leaf count");
  if (n_leaves && (!block_rows || !block_cols || !payload)) fail(SPG_EINVAL, "null leaf arrays");
  CtxGuard g(ctx);
  int32_t padded, depth;
  check_shape(dimension, leaf_size, &padded, &depth);
  auto st = std::make_unique<spg_staged>();
  st->ctx = ctx;
  st->dimension = dimension;
  st->leaf = leaf_size;
  st->n = n_leaves;
  const int64_t elems = static_cast<int64_t>(leaf_size) * leaf_size;
  st->rows = DevBuf<int32_t>(std::max<int64_t>(n_leaves, 1), ctx);
  st->cols = DevBuf<int32_t>(std::max<int64_t>(n_leaves, 1), ctx);
  st->payload = dev_alloc<double>(std::max<int64_t>(n_leaves * elems, 1), ctx);
  SPG_CUDA(cudaEventCreateWithFlags(&st->done, cudaEventDisableTiming));
  // pool blocks are handed out in ctx->stream order: start after it
  SPG_CUDA(cudaEventRecord(st->done, ctx->stream));
  SPG_CUDA(cudaStreamWaitEvent(ctx->h2d_stream, st->done, 0));
  if (n_leaves) {
    SPG_CUDA(cudaMemcpyAsync(st->rows.get(), block_rows, n_leaves * sizeof(int32_t),
                             cudaMemcpyHostToDevice, ctx->h2d_stream));
    SPG_CUDA(cudaMemcpyAsync(st->cols.get(), block_cols, n_leaves * sizeof(int32_t),
                             cudaMemcpyHostToDevice, ctx->h2d_stream));
    SPG_CUDA(cudaMemcpyAsync(st->payload, payload, n_leaves * elems * sizeof(double),
                             cudaMemcpyHostToDevice, ctx->h2d_stream));
  }
  SPG_CUDA(cudaEventRecord(st->done, ctx->h2d_stream));
  *out = st.release();
  SPG_API_END
}

int spg_matrix_stage_finish(spg_staged* st, spg_matrix** out) {
  SPG_API_BEGIN
  if (!st || !out) fail(SPG_EINVAL, "null argument");
  *out = nullptr;
  std::unique_ptr<spg_staged> own(st);
  spg_context* ctx = st->ctx;
  CtxGuard g(ctx);
  SPG_CUDA(cudaStreamWaitEvent(ctx->stream, st->done, 0));
  double* p = st->payload;
  st->payload = nullptr;  // owned by the matrix from here on
  *out = matrix_from_device_leaves(ctx, st->dimension, st->leaf, st->n, st->rows.get(),
                                   st->cols.get(), p);
  SPG_API_END
}

void spg_staged_free(spg_staged* st) {
  if (!st) return;
  try {
    CtxGuard g(st->ctx);
    SPG_CUDA(cudaEventSynchronize(st->done));
    delete st;
  } catch (...) {
  }
}

int spg_matrix_upload_device(spg_context* ctx, int32_t dimension, int32_t leaf_size,
                             int64_t n_leaves, const int32_t* d_block_rows,
                             const int32_t* d_block_cols, const double* d_payload,
                             spg_matrix** out) {
  SPG_API_BEGIN
  if (!ctx || !out) fail(SPG_EINVAL, "null argument");
  *out = nullptr;
  if (n_leaves < 0) fail(SPG_EINVAL, "negative leaf count");
  CtxGuard g(ctx);
  int32_t padded, depth;
  check_shape(dimension, leaf_size, &padded, &depth);
  const int64_t elems = static_cast<int64_t>(leaf_size) * leaf_size;
  double* copy = dev_alloc<double>(std::max<int64_t>(n_leaves * elems, 1), ctx);
  if (n_leaves)
    SPG_CUDA(cudaMemcpyAsync(copy, d_payload, n_leaves * elems * sizeof(double),
                             cudaMemcpyDeviceToDevice, ctx->stream));
  *out = matrix_from_device_leaves(ctx, dimension, leaf_size, n_leaves, d_block_rows,
                                   d_block_cols, copy);
  SPG_API_END
}

int spg_matrix_from_dense(spg_context* ctx, int32_t dimension, int32_t leaf_size,
                          const double* dense, spg_matrix** out) {
  SPG_API_BEGIN
  if (!ctx || !out || !dense) fail(SPG_EINVAL, "null argument");
  *out = nullptr;
  int32_t padded, depth;
  check_shape(dimension, leaf_size, &padded, &depth);
  // build_from_dense (quadtree.cpp:89-108): leaf blocks inside the logical
  // dimension, column-major; padding stays zero; all-zero leaves dropped.
  const int32_t nb = (dimension + leaf_size - 1) / leaf_size;
  const int64_t elems = static_cast<int64_t>(leaf_size) * leaf_size;
  std::vector<int32_t> rows, cols;
  std::vector<double> payload;
  std::vector<double> blk(static_cast<size_t>(elems));
  for (int32_t br = 0; br < nb; ++br)
    for (int32_t bc = 0; bc < nb; ++bc) {
      std::fill(blk.begin(), blk.end(), 0.0);
      const int r = std::min(leaf_size, dimension - br * leaf_size);
      const int c = std::min(leaf_size, dimension - bc * leaf_size);
      bool any = false;
      for (int j = 0; j < c; ++j)
        for (int i = 0; i < r; ++i) {
          const double v =
              dense[static_cast<int64_t>(br * leaf_size + i) * dimension + bc * leaf_size + j];
          blk[i + static_cast<size_t>(j) * leaf_size] = v;
          any = any || v != 0.0;
        }
      if (!any) continue;
      rows.push_back(br);
      cols.push_back(bc);
      payload.insert(payload.end(), blk.begin(), blk.end());
    }
  return spg_matrix_upload(ctx, dimension, leaf_size, static_cast<int64_t>(rows.size()),
                           rows.data(), cols.data(), payload.data(), out);
  SPG_API_END
}

int spg_matrix_zero(spg_context* ctx, int32_t dimension, int32_t leaf_size, spg_matrix** out) {
  return spg_matrix_upload(ctx, dimension, leaf_size, 0, nullptr, nullptr, nullptr, out);
}

int spg_matrix_get_info(const spg_matrix* m, spg_matrix_info* out) {
  SPG_API_BEGIN
  if (!m || !out) fail(SPG_EINVAL, "null argument");
  out->dimension = m->dimension;
  out->padded_dimension = m->padded;
  out->leaf_size = m->leaf;
  out->depth = m->depth;
  out->nnz_blocks = m->nnzb;
  out->frobenius_norm = m->frob;
  SPG_API_END
}

int spg_matrix_download(const spg_matrix* m, int32_t* block_rows, int32_t* block_cols,
                        double* payload, double* norms) {
  SPG_API_BEGIN
  if (!m) fail(SPG_EINVAL, "null matrix");
  if (payload) require_payload(m);
  spg_context* ctx = m->ctx;
  CtxGuard g(ctx);
  if (m->nnzb == 0) return SPG_OK;
  std::vector<uint64_t> keys(static_cast<size_t>(m->nnzb));
  SPG_CUDA(cudaMemcpyAsync(keys.data(), m->keys, m->nnzb * sizeof(uint64_t),
                           cudaMemcpyDeviceToHost, ctx->stream));
  if (payload) {
    const int64_t elems = static_cast<int64_t>(m->leaf) * m->leaf;
    // chunked gather + copy keeps the staging buffer bounded
    const int64_t chunk = std::max<int64_t>(1, (int64_t(256) << 20) / (elems * 8));
    DevBuf<double> stage(std::min(chunk, m->nnzb) * elems, ctx);
    for (int64_t lo = 0; lo < m->nnzb; lo += chunk) {
      const int64_t n = std::min(chunk, m->nnzb - lo);
      dim3 grid(static_cast<unsigned>(std::min<int64_t>((elems + 255) / 256, 64)),
                static_cast<unsigned>(std::min<int64_t>(n, 65535)),
                static_cast<unsigned>((n + 65534) / 65535));
      gather_payload<<<grid, 256, 0, ctx->stream>>>(m->payload, m->slots + lo, n, elems,
                                                    stage.get());
      SPG_CHECK_LAUNCH(ctx);
      SPG_CUDA(cudaMemcpyAsync(payload + lo * elems, stage.get(), n * elems * sizeof(double),
                               cudaMemcpyDeviceToHost, ctx->stream));
    }
  }
  if (norms) {
    DevBuf<double> d_norms(m->nnzb, ctx);
    gather_norms<<<grid_for(m->nnzb, 256), 256, 0, ctx->stream>>>(
        m->keys, m->nnzb, m->pyramid + level_offset(m->depth), d_norms.get());
    SPG_CHECK_LAUNCH(ctx);
    SPG_CUDA(cudaMemcpyAsync(norms, d_norms.get(), m->nnzb * sizeof(double),
                             cudaMemcpyDeviceToHost, ctx->stream));
  }
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int64_t t = 0; t < m->nnzb; ++t) {
    if (block_rows) block_rows[t] = static_cast<int32_t>(morton_row(keys[t]));
    if (block_cols) block_cols[t] = static_cast<int32_t>(morton_col(keys[t]));
  }
  SPG_API_END
}

int spg_matrix_to_dense(const spg_matrix* m, double* dense) {
  SPG_API_BEGIN
  if (!m || !dense) fail(SPG_EINVAL, "null argument");
  require_payload(m);
  const int64_t n = m->dimension, L = m->leaf, elems = L * L;
  std::vector<int32_t> rows(static_cast<size_t>(m->nnzb)), cols(static_cast<size_t>(m->nnzb));
  std::vector<double> payload(static_cast<size_t>(m->nnzb * elems));
  int rc = spg_matrix_download(m, rows.data(), cols.data(), payload.data(), nullptr);
  if (rc != SPG_OK) return rc;
  std::memset(dense, 0, sizeof(double) * static_cast<size_t>(n * n));
  for (int64_t t = 0; t < m->nnzb; ++t) {
    const int64_t r0 = rows[t] * L, c0 = cols[t] * L;
    for (int64_t j = 0; j < L && c0 + j < n; ++j)
      for (int64_t i = 0; i < L && r0 + i < n; ++i)
        dense[(r0 + i) * n + c0 + j] = payload[t * elems + i + j * L];
  }
  SPG_API_END
}

int spg_matrix_level_norms(const spg_matrix* m, int32_t level, double* out) {
  SPG_API_BEGIN
  if (!m || !out) fail(SPG_EINVAL, "null argument");
  if (level < 0 || level > m->depth) fail(SPG_EINVAL, "level outside the tree");
  spg_context* ctx = m->ctx;
  CtxGuard g(ctx);
  SPG_CUDA(cudaMemcpyAsync(out, m->pyramid + level_offset(level),
                           (int64_t(1) << (2 * level)) * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  SPG_API_END
}

int spg_matrix_free(spg_matrix* m) {
  SPG_API_BEGIN
  if (!m) return SPG_OK;
  std::lock_guard<std::mutex> lock(m->ctx->mu);
  matrix_destroy(m);
  SPG_API_END
}


int spg_matrix_from_leaf_norms(spg_context* ctx, int32_t dimension, int32_t leaf_size,
                               int64_t n_leaves, const int32_t* block_rows,
                               const int32_t* block_cols, const double* norms,
                               const uint8_t* nonzero, spg_matrix** out) {
  SPG_API_BEGIN
  if (!ctx || !out) fail(SPG_EINVAL, "null argument");
  *out = nullptr;
  if (n_leaves < 0) fail(SPG_EINVAL, "negative leaf count");
  if (n_leaves && (!block_rows || !block_cols || !norms)) fail(SPG_EINVAL, "null argument");
  // (row, col) strictly ascending: panel plans (spg_matrix_gather_rows emits
  // (row, col) order) pair B slots with this table's order
  for (int64_t t = 1; t < n_leaves; ++t)
    if (block_rows[t] < block_rows[t - 1] ||
        (block_rows[t] == block_rows[t - 1] && block_cols[t] <= block_cols[t - 1]))
      fail(SPG_EINVAL, "leaf norms: leaves must be sorted by (block row, block col) without "
                       "duplicates");
  int32_t padded = 0, depth = 0;
  check_shape(dimension, leaf_size, &padded, &depth);
  CtxGuard g(ctx);
  const int64_t n1 = std::max<int64_t>(n_leaves, 1);
  DevBuf<int32_t> r(n1, ctx), c(n1, ctx);
  DevBuf<double> nr(n1, ctx);
  DevBuf<uint8_t> nz(n1, ctx);
  if (n_leaves) {
    SPG_CUDA(cudaMemcpyAsync(r.get(), block_rows, n_leaves * sizeof(int32_t),
                             cudaMemcpyHostToDevice, ctx->stream));
    SPG_CUDA(cudaMemcpyAsync(c.get(), block_cols, n_leaves * sizeof(int32_t),
                             cudaMemcpyHostToDevice, ctx->stream));
    SPG_CUDA(cudaMemcpyAsync(nr.get(), norms, n_leaves * sizeof(double), cudaMemcpyHostToDevice,
                             ctx->stream));
    if (nonzero)
      SPG_CUDA(cudaMemcpyAsync(nz.get(), nonzero, n_leaves, cudaMemcpyHostToDevice, ctx->stream));
    else
      SPG_CUDA(cudaMemsetAsync(nz.get(), 1, n_leaves, ctx->stream));
  }
  *out = matrix_from_leaf_norms(ctx, dimension, leaf_size, n_leaves, block_rows, r.get(),
                                c.get(), nr.get(), nz.get());
  SPG_API_END
}

int spg_matrix_gather_rows(const spg_matrix* m, int32_t row_begin, int32_t row_end,
                           double* d_out, int64_t capacity, void* stream) {
  SPG_API_BEGIN
  if (!m) fail(SPG_EINVAL, "null matrix");
  require_payload(m);
  const int32_t nbp = 1 << m->depth;
  if (row_begin < 0 || row_end < row_begin || row_end > nbp)
    fail(SPG_EINVAL, "gather_rows: bad block row range");
  if (capacity > 0 && !d_out) fail(SPG_EINVAL, "null output");
  spg_context* ctx = m->ctx;
  CtxGuard g(ctx);
  const int32_t rows = row_end - row_begin;
  const int64_t cells = static_cast<int64_t>(rows) * nbp;
  if (cells == 0 || capacity <= 0) return SPG_OK;
  cudaStream_t foreign = static_cast<cudaStream_t>(stream);
  cudaEvent_t ev = nullptr;
  if (foreign && foreign != ctx->stream) {
    SPG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    SPG_CUDA(cudaEventRecord(ev, foreign));
    SPG_CUDA(cudaStreamWaitEvent(ctx->stream, ev, 0));
  }
  DevBuf<uint8_t> flags(cells, ctx);
  DevBuf<int64_t> sel(cells, ctx), n_sel(1, ctx);
  panel_cell_flags<<<grid_for(cells, 256), 256, 0, ctx->stream>>>(m->grid_slot, row_begin, rows,
                                                                  nbp, flags.get());
  SPG_CHECK_LAUNCH(ctx);
  thrust::counting_iterator<int64_t> it(0);
  size_t bytes = 0;
  SPG_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, flags.get(), sel.get(), n_sel.get(),
                                      cells, ctx->stream));
  DevBuf<uint8_t> tmp(bytes, ctx);
  SPG_CUDA(cub::DeviceSelect::Flagged(tmp.get(), bytes, it, flags.get(), sel.get(), n_sel.get(),
                                      cells, ctx->stream));
  ctx->lib_calls++;  // CUB device-wide primitive (library kernels)
  const int64_t elems = static_cast<int64_t>(m->leaf) * m->leaf;
  const int64_t ylim = std::min<int64_t>(std::min(capacity, cells), 65535);
  dim3 grid(static_cast<unsigned>(std::min<int64_t>((elems + 255) / 256, 16)),
            static_cast<unsigned>(ylim));
  panel_gather<<<grid, 256, 0, ctx->stream>>>(m->payload, m->grid_slot, sel.get(), n_sel.get(),
                                              row_begin, nbp, capacity, elems, d_out);
  SPG_CHECK_LAUNCH(ctx);
  if (ev) {
    SPG_CUDA(cudaEventRecord(ev, ctx->stream));
    SPG_CUDA(cudaStreamWaitEvent(foreign, ev, 0));
    cudaEventDestroy(ev);  // released once the recorded work completes
  }
  SPG_API_END
}


int spg_matrix_norm_pass(const spg_matrix* m, float* ms) {
  SPG_API_BEGIN
  if (!m || !ms) fail(SPG_EINVAL, "null argument");
  require_payload(m);
  spg_context* ctx = m->ctx;
  CtxGuard g(ctx);
  const int64_t n = m->n_slots;
  DevBuf<double> norms(std::max<int64_t>(n, 1), ctx);
  DevBuf<uint8_t> nz(std::max<int64_t>(n, 1), ctx);
  const int32_t nb = (m->dimension + m->leaf - 1) / m->leaf;
  SPG_CUDA(cudaEventRecord(ctx->ev[6], ctx->stream));
  leaf_norms(ctx, m->payload, n, m->leaf, m->dimension, nb, nullptr, nullptr, norms.get(),
             nz.get(), nullptr);
  SPG_CUDA(cudaEventRecord(ctx->ev[7], ctx->stream));
  SPG_CUDA(cudaEventSynchronize(ctx->ev[7]));
  SPG_CUDA(cudaEventElapsedTime(ms, ctx->ev[6], ctx->ev[7]));
  SPG_API_END
}

int spg_matrix_payload(const spg_matrix* m, const double** base) {
  SPG_API_BEGIN
  if (!m || !base) fail(SPG_EINVAL, "null argument");
  require_payload(m);
  *base = m->payload;
  SPG_API_END
}

int spg_matrix_payload_slots(const spg_matrix* m, int32_t* slots) {
  SPG_API_BEGIN
  if (!m || !slots) fail(SPG_EINVAL, "null argument");
  require_payload(m);
  CtxGuard g(m->ctx);
  if (m->nnzb)
    SPG_CUDA(cudaMemcpyAsync(slots, m->slots, m->nnzb * sizeof(int32_t), cudaMemcpyDeviceToHost,
                             m->ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(m->ctx->stream));
  SPG_API_END
}

int spg_ipc_export(const spg_matrix* m, void* handle) {
  SPG_API_BEGIN
  if (!m || !handle) fail(SPG_EINVAL, "null argument");
  require_payload(m);
  if (!m->payload) fail(SPG_EINVAL, "matrix has no leaves to export");
  CtxGuard g(m->ctx);
  cudaIpcMemHandle_t h;
  SPG_CUDA(cudaIpcGetMemHandle(&h, m->payload));
  std::memcpy(handle, &h, sizeof h);
  SPG_API_END
}

int spg_ipc_open(spg_context* ctx, const void* handle, const double** base) {
  SPG_API_BEGIN
  if (!ctx || !handle || !base) fail(SPG_EINVAL, "null argument");
  CtxGuard g(ctx);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  void* p = nullptr;
  SPG_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  *base = static_cast<const double*>(p);
  SPG_API_END
}

int spg_ipc_close(spg_context* ctx, const double* base) {
  SPG_API_BEGIN
  if (!ctx || !base) fail(SPG_EINVAL, "null argument");
  CtxGuard g(ctx);
  SPG_CUDA(cudaIpcCloseMemHandle(const_cast<double*>(base)));
  SPG_API_END
}

}  // extern "C"
