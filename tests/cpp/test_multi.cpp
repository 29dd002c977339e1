// test_multi.cpp -- the drop-in's multi-GPU mode (include/spamm/distributed.hpp)
// through the UNCHANGED reference API: two ranks (forked processes, each with
// its own context on the one GPU of the box, no rank ever waits on another's
// kernels), joined by a host all-gather over shared memory.  Every rank's
// cse bounds, spamm_with_error_control (tau, bound, C~), spamm_multiply and
// multiply_exact results must be BITWISE those of the single-GPU calls.
#include <pthread.h>
#include <sys/mman.h>
#include <sys/wait.h>
#include <unistd.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

#include "spamm/distributed.hpp"
#include "spamm/error_control.hpp"
#include "spamm/multiply.hpp"
#include "spamm/quadtree.hpp"

using namespace spamm;

namespace {

constexpr int kRanks = 2;
constexpr std::size_t kArea = std::size_t(256) << 20;

struct Shared {
  pthread_barrier_t barrier;
  unsigned char data[1];  // kArea bytes follow
};

int shm_allgather(void* user, const void* send, std::size_t bytes, void* recv) {
  static int rank = -1;
  auto* sh = static_cast<Shared*>(user);
  if (rank < 0) rank = distributed::rank();
  if (bytes * kRanks > kArea) return 1;
  std::memcpy(sh->data + rank * bytes, send, bytes);
  pthread_barrier_wait(&sh->barrier);
  std::memcpy(recv, sh->data, bytes * kRanks);
  pthread_barrier_wait(&sh->barrier);
  return 0;
}

DenseMatrix decay(int n, std::uint64_t seed, double ell) {
  std::mt19937_64 rng(seed);
  DenseMatrix d(n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) {
      const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53 * 2.0 - 1.0;
      const double v = u * std::exp(-std::abs(i - j) / ell);
      d(i, j) = d(j, i) = std::abs(v) < 1e-12 ? 0.0 : v;
    }
  return d;
}

bool same(const QuadTreeMatrix& x, const QuadTreeMatrix& y) {
  return x.dimension() == y.dimension() && x.nnz_blocks() == y.nnz_blocks() &&
         x.to_dense_padded() == y.to_dense_padded() &&
         std::memcmp(&x.root()->norm, &y.root()->norm, sizeof(double)) == 0;
}

int checks = 0, failures = 0;
void check(bool ok, const char* what, int rank) {
  ++checks;
  if (!ok) {
    ++failures;
    std::fprintf(stderr, "FAIL rank %d: %s\n", rank, what);
  }
}

int run_rank(int rank, Shared* sh) {
  const int n = 1000, leaf = 32;  // ragged: padded 1024, 32 block rows
  const QuadTreeMatrix a = QuadTreeMatrix::from_dense(decay(n, 11, 25.0), leaf);
  const QuadTreeMatrix b = QuadTreeMatrix::from_dense(decay(n, 12, 12.0), leaf);
  const ToleranceGrid grid = ToleranceGrid::geometric(1.0, 0.7, 60);
  // single GPU first
  const ErrorBoundVector e1 = cse(a, b, grid);
  const ControlledProduct p1 = spamm_with_error_control(a, b, 1e-6, grid);
  const QuadTreeMatrix s1 = spamm_multiply(a, b, SpammTolerance{1e-5});
  const QuadTreeMatrix x1 = multiply_exact(a, b);
  // then the same calls as rank `rank` of kRanks
  distributed::init_host(rank, kRanks, shm_allgather, sh);
  check(distributed::active() && distributed::size() == kRanks && distributed::rank() == rank,
        "communicator", rank);
  const ErrorBoundVector e2 = cse(a, b, grid);
  check(std::memcmp(e1.bounds.data(), e2.bounds.data(), e1.bounds.size() * 8) == 0, "cse bounds",
        rank);
  const ControlledProduct p2 = spamm_with_error_control(a, b, 1e-6, grid);
  check(p1.chosen_tau.tau == p2.chosen_tau.tau && p1.bound == p2.bound, "tau / bound", rank);
  check(p1.chosen_tau.tau > 0.0, "tau skips something", rank);
  check(same(p1.matrix, p2.matrix), "controlled product C~", rank);
  check(same(s1, spamm_multiply(a, b, SpammTolerance{1e-5})), "spamm_multiply", rank);
  check(same(x1, multiply_exact(a, b)), "multiply_exact", rank);
  distributed::finalize();
  check(!distributed::active() && distributed::size() == 1, "finalize", rank);
  std::printf("rank %d: %d checks, %d failures\n", rank, checks, failures);
  return failures ? 1 : 0;
}

}  // namespace

int main() {
  void* mem = mmap(nullptr, sizeof(Shared) + kArea, PROT_READ | PROT_WRITE,
                   MAP_SHARED | MAP_ANONYMOUS, -1, 0);
  if (mem == MAP_FAILED) return 2;
  auto* sh = static_cast<Shared*>(mem);
  pthread_barrierattr_t attr;
  pthread_barrierattr_init(&attr);
  pthread_barrierattr_setpshared(&attr, PTHREAD_PROCESS_SHARED);
  pthread_barrier_init(&sh->barrier, &attr, kRanks);
  pid_t pids[kRanks];
  for (int r = 0; r < kRanks; ++r) {
    pids[r] = fork();
    if (pids[r] == 0) _exit(run_rank(r, sh));  // CUDA is first touched in the child
  }
  int bad = 0;
  for (int r = 0; r < kRanks; ++r) {
    int status = 0;
    waitpid(pids[r], &status, 0);
    if (!WIFEXITED(status) || WEXITSTATUS(status) != 0) ++bad;
  }
  std::printf("%d of %d ranks failed\n", bad, kRanks);
  return bad ? 1 : 0;
}
