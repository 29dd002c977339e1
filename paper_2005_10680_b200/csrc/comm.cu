// comm.cu -- multi-GPU inside the C ABI: a communicator over
// the ranks of one job (one process per GPU) and the output-block-row-sharded
// controlled product on top of it.
//
// The reference parallelises every call through its thread knob
// (execution.cpp:11-23, fork-join at multiply.cpp:79-84 and
// error_control.cpp:59-66).  Here the unit of parallelism is a GPU: with
// 2^s ranks, rank r owns output block rows [r nb/2^s, (r+1) nb/2^s):
//   1. cse_device(shard s, r): the level-s partial bound vectors of its rows
//      (4^s x N_tau doubles, <= 512 KB at s = 3, 128 tau);
//   2. all-gather of the partials;
//   3. spg_cse_finish on every rank: the top s levels in reference order ->
//      bounds and tau bit-identical to one GPU on every rank;
//   4. spamm_device(shard s, r): the rank's rows of C~ (per-block k order
//      unchanged, so C~'s bits do not depend on the rank count);
//   5. optionally an all-gather of the rows' leaves, so every rank holds the
//      whole C~ (the value semantics of the reference API).
//
// Transports:
//   * NCCL (ncclAllGather on the library stream, over NVLink / NVSwitch),
//     loaded with dlopen at communicator creation -- the library itself does
//     not link NCCL and still loads on machines without it;
//   * a host callback (the caller's own collective, e.g. gloo or MPI): used
//     by the tests, which run two ranks on one GPU.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <memory>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

struct spg_comm {
  spg_context* ctx = nullptr;
  int32_t nranks = 1, rank = 0;
  // NCCL transport
  ncclComm_t nccl = nullptr;
  // host transport
  spg_host_allgather_fn host_fn = nullptr;
  void* host_user = nullptr;
};

namespace spg {
namespace {

// ---- NCCL, resolved at run time ---------------------------------------------
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string error;
};

const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    const char* env = std::getenv("SPG_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      if (!n) continue;
      a.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (!a.h) {
      a.error = std::string("cannot load NCCL (libnccl.so.2): ") + dlerror();
      return a;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(a.h, name));
      if (!fn && a.error.empty()) a.error = std::string("NCCL symbol missing: ") + name;
    };
    sym(a.get_unique_id, "ncclGetUniqueId");
    sym(a.init_rank, "ncclCommInitRank");
    sym(a.all_gather, "ncclAllGather");
    sym(a.destroy, "ncclCommDestroy");
    sym(a.error_string, "ncclGetErrorString");
    return a;
  }();
  return api;
}

const NcclApi& require_nccl() {
  const NcclApi& a = nccl_api();
  if (!a.error.empty()) fail(SPG_ENCCL, a.error);
  return a;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(SPG_ENCCL, std::string(what) + ": " + nccl_api().error_string(r));
}

// ---- all-gather of equal-size byte blocks from every rank --------------------
// d_send / d_recv on the device (recv: nranks * bytes, rank order)
void allgather_device(spg_comm* comm, const void* d_send, void* d_recv, size_t bytes) {
  spg_context* ctx = comm->ctx;
  if (comm->nranks == 1) {
    if (bytes)
      SPG_CUDA(cudaMemcpyAsync(d_recv, d_send, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    return;
  }
  if (comm->nccl) {
    nccl_check(nccl_api().all_gather(d_send, d_recv, bytes, ncclUint8, comm->nccl, ctx->stream),
               "ncclAllGather");
    return;
  }
  // host transport: stage through host memory
  std::vector<unsigned char> hs(bytes), hr(bytes * comm->nranks);
  if (bytes) {
    SPG_CUDA(cudaMemcpyAsync(hs.data(), d_send, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  if (comm->host_fn(comm->host_user, hs.data(), bytes, hr.data()) != 0)
    fail(SPG_ENCCL, "host all-gather callback failed");
  if (bytes)
    SPG_CUDA(cudaMemcpyAsync(d_recv, hr.data(), hr.size(), cudaMemcpyHostToDevice, ctx->stream));
}

// host buffers in and out (small payloads: counts, partial bound vectors)
void allgather_host(spg_comm* comm, const void* send, void* recv, size_t bytes) {
  if (comm->nranks == 1) {
    std::memcpy(recv, send, bytes);
    return;
  }
  if (!comm->nccl) {
    if (comm->host_fn(comm->host_user, send, bytes, recv) != 0)
      fail(SPG_ENCCL, "host all-gather callback failed");
    return;
  }
  spg_context* ctx = comm->ctx;
  DevBuf<unsigned char> ds(std::max<size_t>(bytes, 1), ctx),
      dr(std::max<size_t>(bytes * comm->nranks, 1), ctx);
  SPG_CUDA(cudaMemcpyAsync(ds.get(), send, bytes, cudaMemcpyHostToDevice, ctx->stream));
  allgather_device(comm, ds.get(), dr.get(), bytes);
  SPG_CUDA(cudaMemcpyAsync(recv, dr.get(), bytes * comm->nranks, cudaMemcpyDeviceToHost,
                           ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
}

int shard_level(const spg_comm* comm, const spg_matrix* a) {
  const int s = 31 - __builtin_clz(static_cast<unsigned>(comm->nranks));
  if ((1 << s) != comm->nranks)
    fail(SPG_EINVAL, "sharded product: the rank count must be a power of two");
  if (s > a->depth || s > 8)
    fail(SPG_EINVAL, "sharded product: more ranks than block rows (or > 256 ranks)");
  return s;
}

// bounds of the whole problem from the rank's shard + the gathered partials
void cse_sharded(spg_comm* comm, const spg_matrix* a, const spg_matrix* b, const double* taus,
                 int n_taus, int s, double* bounds, float* ms) {
  spg_context* ctx = comm->ctx;
  if (s == 0) {
    cse_device(ctx, a, b, taus, n_taus, bounds, ms);
    return;
  }
  const size_t per = (size_t(1) << (2 * s)) * n_taus;
  std::vector<double> mine(per), all(per * comm->nranks);
  cse_device(ctx, a, b, taus, n_taus, mine.data(), ms, Shard{s, comm->rank});
  allgather_host(comm, mine.data(), all.data(), per * sizeof(double));
  const int64_t top = level_offset(s);
  std::vector<double> at(top), bt(top);
  SPG_CUDA(cudaMemcpyAsync(at.data(), a->pyramid, top * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
  SPG_CUDA(cudaMemcpyAsync(bt.data(), b->pyramid, top * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  const int rc = spg_cse_finish(s, at.data(), bt.data(), n_taus, all.data(), bounds);
  if (rc != SPG_OK) fail(rc, spg_last_error());
}

__global__ void pack_leaves(const uint64_t* __restrict__ keys, const int32_t* __restrict__ slots,
                            int64_t n, const double* __restrict__ payload, int64_t LL,
                            int32_t* __restrict__ rows, int32_t* __restrict__ cols,
                            double* __restrict__ out) {
  for (int64_t t = blockIdx.x; t < n; t += gridDim.x) {
    if (threadIdx.x == 0) {
      rows[t] = static_cast<int32_t>(morton_row(keys[t]));
      cols[t] = static_cast<int32_t>(morton_col(keys[t]));
    }
    const double* src = payload + static_cast<int64_t>(slots[t]) * LL;
    double* dst = out + t * LL;
    for (int64_t e = threadIdx.x; e < LL; e += blockDim.x) dst[e] = src[e];
  }
}

__global__ void compact_ranks(const int32_t* __restrict__ rows_in,
                              const int32_t* __restrict__ cols_in,
                              const double* __restrict__ pay_in, const int64_t* __restrict__ src,
                              int64_t n, int64_t LL, int32_t* __restrict__ rows,
                              int32_t* __restrict__ cols, double* __restrict__ pay) {
  for (int64_t t = blockIdx.x; t < n; t += gridDim.x) {
    const int64_t s = src[t];
    if (threadIdx.x == 0) {
      rows[t] = rows_in[s];
      cols[t] = cols_in[s];
    }
    for (int64_t e = threadIdx.x; e < LL; e += blockDim.x) pay[t * LL + e] = pay_in[s * LL + e];
  }
}

// every rank's leaves of its shard -> the whole matrix on every rank
spg_matrix* gather_rows(spg_comm* comm, const spg_matrix* mine) {
  spg_context* ctx = comm->ctx;
  const int64_t LL = static_cast<int64_t>(mine->leaf) * mine->leaf;
  const int R = comm->nranks;
  int64_t n = mine->nnzb;
  std::vector<int64_t> counts(R);
  allgather_host(comm, &n, counts.data(), sizeof(int64_t));
  const int64_t cap = std::max<int64_t>(*std::max_element(counts.begin(), counts.end()), 1);
  int64_t total = 0;
  for (int64_t c : counts) total += c;
  DevBuf<int32_t> r1(cap, ctx), c1(cap, ctx), rr(cap * R, ctx), cr(cap * R, ctx);
  DevBuf<double> p1(cap * LL, ctx), pr(cap * R * LL, ctx);
  if (n) {
    pack_leaves<<<grid_for(n, 1, 1 << 20), 256, 0, ctx->stream>>>(
        mine->keys, mine->slots, n, mine->payload, LL, r1.get(), c1.get(), p1.get());
    SPG_CHECK_LAUNCH(ctx);
  }
  allgather_device(comm, r1.get(), rr.get(), cap * sizeof(int32_t));
  allgather_device(comm, c1.get(), cr.get(), cap * sizeof(int32_t));
  allgather_device(comm, p1.get(), pr.get(), cap * LL * sizeof(double));
  // drop the padding: rank g's leaves sit at [g cap, g cap + counts[g])
  std::vector<int64_t> src(static_cast<size_t>(std::max<int64_t>(total, 1)));
  int64_t t = 0;
  for (int g = 0; g < R; ++g)
    for (int64_t i = 0; i < counts[g]; ++i) src[t++] = g * cap + i;
  DevBuf<int64_t> dsrc(std::max<int64_t>(total, 1), ctx);
  DevBuf<int32_t> rows(std::max<int64_t>(total, 1), ctx), cols(std::max<int64_t>(total, 1), ctx);
  double* pay = dev_alloc<double>(std::max<int64_t>(total * LL, 1), ctx);
  if (total) {
    SPG_CUDA(cudaMemcpyAsync(dsrc.get(), src.data(), total * sizeof(int64_t),
                             cudaMemcpyHostToDevice, ctx->stream));
    compact_ranks<<<grid_for(total, 1, 1 << 20), 256, 0, ctx->stream>>>(
        rr.get(), cr.get(), pr.get(), dsrc.get(), total, LL, rows.get(), cols.get(), pay);
    SPG_CHECK_LAUNCH(ctx);
  }
  return matrix_from_device_leaves(ctx, mine->dimension, mine->leaf, total, rows.get(),
                                   cols.get(), pay);
}

using Clock = std::chrono::steady_clock;

}  // namespace
}  // namespace spg

using namespace spg;

extern "C" {

int spg_comm_unique_id(void* id_out) {
  SPG_API_BEGIN
  if (!id_out) fail(SPG_EINVAL, "null argument");
  ncclUniqueId id;
  nccl_check(require_nccl().get_unique_id(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == SPG_COMM_ID_BYTES, "NCCL unique id size");
  std::memcpy(id_out, &id, sizeof id);
  SPG_API_END
}

int spg_comm_create_nccl(spg_context* ctx, int32_t nranks, int32_t rank, const void* id,
                         spg_comm** out) {
  SPG_API_BEGIN
  if (!ctx || !id || !out) fail(SPG_EINVAL, "null argument");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(SPG_EINVAL, "bad rank / rank count");
  const NcclApi& api = require_nccl();
  CtxGuard g(ctx);
  auto* c = new spg_comm;
  c->ctx = ctx;
  c->nranks = nranks;
  c->rank = rank;
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  const ncclResult_t r = api.init_rank(&c->nccl, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    nccl_check(r, "ncclCommInitRank");
  }
  *out = c;
  SPG_API_END
}

int spg_comm_create_host(spg_context* ctx, int32_t nranks, int32_t rank,
                         spg_host_allgather_fn fn, void* user, spg_comm** out) {
  SPG_API_BEGIN
  if (!ctx || !fn || !out) fail(SPG_EINVAL, "null argument");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(SPG_EINVAL, "bad rank / rank count");
  auto* c = new spg_comm;
  c->ctx = ctx;
  c->nranks = nranks;
  c->rank = rank;
  c->host_fn = fn;
  c->host_user = user;
  *out = c;
  SPG_API_END
}

int spg_comm_info(const spg_comm* comm, int32_t* nranks, int32_t* rank, int32_t* uses_nccl) {
  SPG_API_BEGIN
  if (!comm) fail(SPG_EINVAL, "null argument");
  if (nranks) *nranks = comm->nranks;
  if (rank) *rank = comm->rank;
  if (uses_nccl) *uses_nccl = comm->nccl != nullptr;
  SPG_API_END
}

int spg_comm_destroy(spg_comm* comm) {
  SPG_API_BEGIN
  if (!comm) return SPG_OK;
  if (comm->nccl) {
    CtxGuard g(comm->ctx);
    SPG_CUDA(cudaStreamSynchronize(comm->ctx->stream));
    nccl_api().destroy(comm->nccl);
  }
  delete comm;
  SPG_API_END
}

int spg_cse_sharded(spg_comm* comm, const spg_matrix* a, const spg_matrix* b, const double* taus,
                    int32_t n_taus, double* bounds) {
  SPG_API_BEGIN
  if (!comm || !a || !b || !bounds) fail(SPG_EINVAL, "null argument");
  int rc = spg_tolerance_grid_check(taus, n_taus);
  if (rc != SPG_OK) return rc;
  if (a->dimension != b->dimension || a->leaf != b->leaf)
    fail(SPG_EINVAL, "cse: dimension or leaf size mismatch");
  CtxGuard g(comm->ctx);
  cse_sharded(comm, a, b, taus, n_taus, shard_level(comm, a), bounds, nullptr);
  SPG_API_END
}

int spg_spamm_sharded(spg_comm* comm, const spg_matrix* a, const spg_matrix* b, double tau,
                      int32_t skip_test, int32_t gather, spg_matrix** c, spg_spamm_stats* stats) {
  SPG_API_BEGIN
  if (!comm || !a || !b || !c) fail(SPG_EINVAL, "null argument");
  *c = nullptr;
  if (a->dimension != b->dimension || a->leaf != b->leaf)
    fail(SPG_EINVAL, "multiply: dimension or leaf size mismatch");
  if (tau < 0.0) fail(SPG_EINVAL, "spamm: tau must be nonnegative");
  CtxGuard g(comm->ctx);
  const int s = shard_level(comm, a);
  spg_matrix* mine = spamm_device(comm->ctx, a, b, tau, skip_test != 0, stats,
                                  Shard{s, comm->rank});
  if (gather && comm->nranks > 1) {
    std::unique_ptr<spg_matrix, void (*)(spg_matrix*)> own(mine, matrix_destroy);
    *c = gather_rows(comm, mine);
  } else {
    *c = mine;
  }
  SPG_API_END
}

int spg_spamm_with_error_control_sharded(spg_comm* comm, const spg_matrix* a,
                                         const spg_matrix* b, double delta, const double* taus,
                                         int32_t n_taus, int32_t gather, spg_matrix** c,
                                         double* bounds, spg_controlled_stats* stats) {
  SPG_API_BEGIN
  if (!comm || !a || !b || !c) fail(SPG_EINVAL, "null argument");
  *c = nullptr;
  if (!(delta > 0.0)) fail(SPG_EINVAL, "spamm_with_error_control: delta must be positive");
  int rc = spg_tolerance_grid_check(taus, n_taus);
  if (rc != SPG_OK) return rc;
  if (a->dimension != b->dimension || a->leaf != b->leaf)
    fail(SPG_EINVAL, "cse: dimension or leaf size mismatch");
  spg_context* ctx = comm->ctx;
  CtxGuard g(ctx);
  const int s = shard_level(comm, a);
  std::vector<double> local(static_cast<size_t>(n_taus));
  double* bv = bounds ? bounds : local.data();
  float cse_ms = 0.0f;
  const auto t0 = Clock::now();
  cse_sharded(comm, a, b, taus, n_taus, s, bv, &cse_ms);
  const double cse_seconds = std::chrono::duration<double>(Clock::now() - t0).count();
  int32_t k = -1;
  for (int32_t i = 0; i < n_taus; ++i)
    if (bv[i] < delta) {
      k = i;
      break;
    }
  const double tau = k >= 0 ? taus[k] : 0.0;
  spg_spamm_stats ss{};
  const auto t1 = Clock::now();
  spg_matrix* mine = spamm_device(ctx, a, b, tau, true, &ss, Shard{s, comm->rank});
  if (gather && comm->nranks > 1) {
    std::unique_ptr<spg_matrix, void (*)(spg_matrix*)> own(mine, matrix_destroy);
    *c = gather_rows(comm, mine);
  } else {
    *c = mine;
  }
  SPG_CUDA(cudaStreamSynchronize(ctx->stream));
  const double spamm_seconds = std::chrono::duration<double>(Clock::now() - t1).count();
  if (stats) {
    stats->tau = tau;
    stats->tau_index = k;
    stats->bound = k >= 0 ? bv[k] : 0.0;
    stats->cse_seconds = cse_seconds;
    stats->spamm_seconds = spamm_seconds;
    stats->ms_cse = cse_ms;
    stats->spamm = ss;
  }
  SPG_API_END
}

int spg_matrix_gather_shards(spg_comm* comm, const spg_matrix* shard, spg_matrix** out) {
  SPG_API_BEGIN
  if (!comm || !shard || !out) fail(SPG_EINVAL, "null argument");
  *out = nullptr;
  require_payload(shard);
  CtxGuard g(comm->ctx);
  *out = gather_rows(comm, shard);
  SPG_API_END
}

}  // extern "C"
