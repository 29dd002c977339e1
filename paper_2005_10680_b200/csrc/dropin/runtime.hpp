// runtime.hpp -- internal glue of the C++ drop-in: the process-wide device
// context, status -> exception mapping, and the shared matrix state.
#pragma once

#include <mutex>
#include <string>

#include "spamm/quadtree.hpp"
#include "spamm_gpu.h"

namespace spamm::b200 {

/// Process-wide context on device $SPAMM_B200_DEVICE (default 0).
spg_context* context();

/// The multi-GPU communicator (spamm::distributed), or null: single GPU.
spg_comm* communicator();

/// Map a C-ABI status onto the reference's exception types
/// (std::invalid_argument / std::out_of_range, include/spamm_gpu.h).
void check(int rc);

}  // namespace spamm::b200

struct spamm::QuadTreeMatrix::State {
  std::mutex mu;
  spg_matrix* dev = nullptr;  // owned device matrix (may be built lazily from `host`)
  NodePtr host;               // host tree (materialised lazily from `dev`)
  bool host_ready = false;
  ~State();
};
