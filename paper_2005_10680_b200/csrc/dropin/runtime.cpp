// runtime.cpp -- drop-in glue: device context, error mapping, exec knob.
#include "runtime.hpp"

#include <atomic>
#include <cstdlib>
#include <new>
#include <stdexcept>

#include "spamm/execution.hpp"

namespace spamm::b200 {

spg_context* context() {
  static spg_context* ctx = [] {
    const char* env = std::getenv("SPAMM_B200_DEVICE");
    spg_context* c = nullptr;
    check(spg_context_create(env ? std::atoi(env) : 0, &c));
    return c;  // intentionally never destroyed: matrices may outlive main()
  }();
  return ctx;
}

void check(int rc) {
  if (rc == SPG_OK) return;
  const std::string msg = spg_last_error();
  switch (rc) {
    case SPG_EINVAL: throw std::invalid_argument(msg);
    case SPG_ERANGE: throw std::out_of_range(msg);
    case SPG_ENOMEM: throw std::bad_alloc();
    default: throw std::runtime_error("spamm-b200: " + msg);
  }
}

}  // namespace spamm::b200

spamm::QuadTreeMatrix::State::~State() {
  if (dev) spg_matrix_free(dev);
}

// Thread knob (execution.hpp:15-22).  Kept for source compatibility; the GPU
// hot path does not use host threads, so results never depend on it.
namespace spamm::exec {
namespace {
std::atomic<int> g_threads{1};
}
void set_max_threads(int threads) { g_threads.store(threads < 1 ? 1 : threads); }
int max_threads() noexcept { return g_threads.load(); }
int spawn_levels() noexcept {
  int levels = 0;
  for (int cap = 1; cap < max_threads() && levels < 3; cap *= 4) ++levels;
  return levels;
}
}  // namespace spamm::exec
