// The kernel seam (proj/include/ooc/kernel_exec.hpp:12-30): one par_loop over one
// sub-range against dense row-major views. Here the loop runs as an sm_100a kernel
// (the device layer's ooc_launch_loop); the views must be device-accessible — device
// memory, or this build's page-locked Dataset::host buffers (mapped into the GPU's
// address space). ExecPolicy is kept for source compatibility: every policy runs on
// the GPU.
#pragma once

#include <vector>

#include "ooc/core.hpp"

namespace ooc {

enum class ExecPolicy { serial, openmp };
inline ExecPolicy default_exec_policy() { return ExecPolicy::openmp; }

struct ArgView {
  double* data = nullptr;  // element box.lo, row-major over `box`
  Extent box;
};

/// Evaluates every write tape of `loop` at each point of `range` (all reads of a point
/// before any of its writes, as proj/src/kernel_exec.cpp:133-198) on GPU `gpu`, and
/// combines the range's reduction into *reduction_acc (parallel tree: within 1e-12 of
/// the reference's sequential fold). Synchronous: returns when the kernel is done.
void apply_loop(const ParLoop& loop, const Extent& range, const std::vector<ArgView>& views,
                ExecPolicy policy = default_exec_policy(), double* reduction_acc = nullptr, int gpu = 0);

}  // namespace ooc
