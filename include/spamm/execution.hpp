#pragma once
//
// spamm-b200 drop-in: thread knob of the reference
// (/root/reference/proj/core/include/spamm/execution.hpp:15-22).
//
// The GPU path does not use host threads for the hot path; the knob is kept
// so callers compile and behave unchanged.  Results are bitwise independent
// of it (as in the reference, execution.hpp:11-13).
//
namespace spamm::exec {

void set_max_threads(int threads);
int max_threads() noexcept;
int spawn_levels() noexcept;

}  // namespace spamm::exec
