// The executor seam (proj/include/ooc/explicit_exec.hpp:14-65): run_chain_explicit with
// the reference's signature, executed by the B200 streaming engine — three HBM slots,
// H2D / compute+D2D / D2H CUDA streams, pinned host memory, edge carry on the device,
// write-first / read-only / cyclic skipping, speculative first-tile prefetch. The
// reference's own Runtime::execute (proj/src/runtime.cpp:112-125) can call it unchanged.
#pragma once

#include <map>
#include <memory>
#include <vector>

#include "ooc/chain.hpp"
#include "ooc/command.hpp"
#include "ooc/device_config.hpp"
#include "ooc/kernel_exec.hpp"
#include "ooc/tiler.hpp"

namespace ooc {

class GpuEngine;

struct ExecOptions {
  bool cyclic = false;    // discard write-first data instead of downloading
  bool prefetch = false;  // speculatively upload the next chain's first tile
  ExecPolicy policy = ExecPolicy::serial;
};

/// Per-(dataset, tile) byte audit; tile == tile_count marks speculative uploads staged
/// for the next chain (proj/include/ooc/explicit_exec.hpp:20-24).
struct AuditRow {
  DatasetId dataset = -1;
  int tile = -1;
  index_t uploaded = 0, downloaded = 0, d2d = 0;
};

struct ExecResult {
  Timeline timeline;                 // measured (when the state records one), else empty
  std::vector<AuditRow> audit;
  std::map<int, double> reductions;  // loop id -> value
  index_t faults = 0;                // unified mode of the reference: always 0 here
};

/// Device-side state that survives between chains (proj/include/ooc/explicit_exec.hpp:39-54):
/// the GPU engine itself — its streams, slot rotation and the speculative uploads staged
/// for the next chain stay live in HBM between calls.
struct DeviceState {
  int gpu = 0;             // CUDA device the engine runs on
  bool timeline = false;   // record the measured command timeline into ExecResult
  int slot_cursor = 0;     // mirrors the engine's slot rotation after each chain
  struct Staged {
    Extent region;
  };
  std::map<DatasetId, Staged> staged;  // mirrors the engine's staged first tiles
  std::shared_ptr<GpuEngine> engine;

  void invalidate_staged(DatasetId d);
};

/// Runs a planned chain through the three-slot pipeline on the GPU. Host buffers of
/// `mesh` (page-locked) are updated in place and current when the call returns, except
/// cyclically discarded datasets (marked stale, proj/src/explicit_exec.cpp:236-258).
/// Throws CapacityError when 3 * slot_bytes exceeds cfg.capacity_bytes (:61-62).
ExecResult run_chain_explicit(Mesh& mesh, const LoopChain& chain, const TilePlan& plan,
                              const Footprints& fp, const DeviceConfig& cfg,
                              const ExecOptions& opts, DeviceState& state);

}  // namespace ooc
