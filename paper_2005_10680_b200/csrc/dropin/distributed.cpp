// distributed.cpp -- the drop-in's multi-GPU mode (include/spamm/distributed.hpp):
// a process-wide communicator over the C ABI (spg_comm_*).  multiply.cpp and
// error_control.cpp route the reference calls through the sharded entry points
// while it is set.
#include "spamm/distributed.hpp"

#include <mutex>
#include <stdexcept>

#include "runtime.hpp"

namespace spamm::b200 {

namespace {
std::mutex g_mu;
spg_comm* g_comm = nullptr;
}  // namespace

spg_comm* communicator() {
  std::lock_guard<std::mutex> lock(g_mu);
  return g_comm;
}

}  // namespace spamm::b200

namespace spamm::distributed {

namespace {
void install(spg_comm* c) {
  std::lock_guard<std::mutex> lock(b200::g_mu);
  if (b200::g_comm) spg_comm_destroy(b200::g_comm);
  b200::g_comm = c;
}
}  // namespace

UniqueId nccl_unique_id() {
  UniqueId id{};
  b200::check(spg_comm_unique_id(id.data()));
  return id;
}

void init_nccl(int rank, int nranks, const UniqueId& id) {
  spg_comm* c = nullptr;
  b200::check(spg_comm_create_nccl(b200::context(), nranks, rank, id.data(), &c));
  install(c);
}

void init_host(int rank, int nranks, HostAllGather fn, void* user) {
  spg_comm* c = nullptr;
  b200::check(spg_comm_create_host(b200::context(), nranks, rank, fn, user, &c));
  install(c);
}

void finalize() { install(nullptr); }

bool active() { return b200::communicator() != nullptr; }

int rank() {
  spg_comm* c = b200::communicator();
  int32_t r = 0;
  if (c) b200::check(spg_comm_info(c, nullptr, &r, nullptr));
  return r;
}

int size() {
  spg_comm* c = b200::communicator();
  int32_t n = 1;
  if (c) b200::check(spg_comm_info(c, &n, nullptr, nullptr));
  return n;
}

}  // namespace spamm::distributed
