#pragma once
//
// spamm-b200 drop-in, B200 extension: multi-GPU for the reference's callers.
//
// The reference spreads a product over host threads with its process-wide
// knob exec::set_max_threads (execution.hpp:15, execution.cpp:11-23).  The
// B200 analogue is one process per GPU: after init_nccl / init_host on every
// rank, the UNCHANGED reference calls
//     spamm_with_error_control, spamm_multiply, multiply_exact, cse
// run as output-block-row shards over the ranks' GPUs (2^s ranks; rank r
// computes block rows [r nb/2^s, (r+1) nb/2^s)), and every rank still gets the
// whole result (an all-gather of the rows' leaves): the reference's value
// semantics.  Bounds, tau and C~ are bitwise the single-GPU ones on every
// rank.  Collectives go through include/spamm_gpu.h's communicator (NCCL over
// NVLink / NVSwitch, or the caller's own all-gather).
//
#include <array>
#include <cstddef>

namespace spamm::distributed {

using UniqueId = std::array<unsigned char, 128>;

/// ncclGetUniqueId on one rank; hand the bytes to every other rank (MPI,
/// a file, torch.distributed ...).
UniqueId nccl_unique_id();

/// Join the job as `rank` of `nranks` over NCCL.  Throws std::runtime_error
/// when NCCL is unavailable, std::invalid_argument on a bad rank.
void init_nccl(int rank, int nranks, const UniqueId& id);

/// Join with the caller's own all-gather: fn(user, send, bytes, recv) must
/// place every rank's `bytes` into recv in rank order and return 0.
using HostAllGather = int (*)(void* user, const void* send, std::size_t bytes, void* recv);
void init_host(int rank, int nranks, HostAllGather fn, void* user);

/// Back to single-GPU operation.
void finalize();

bool active();
int rank();
int size();

}  // namespace spamm::distributed
