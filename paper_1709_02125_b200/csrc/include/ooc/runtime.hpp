// Lazy loop-chain runtime with B200 executors.
//
// Source-compatible with the reference Runtime (proj/include/ooc/runtime.hpp:53-137):
// declare / enqueue_loop / fetch_dataset / fetch_reduction / set_cyclic_flag /
// flush / finish and the same flush semantics (proj/src/runtime.cpp:5-39). What
// changes is what a flush runs on:
//
//   ExecutorKind::tiled_explicit  the out-of-core streaming engine: Algorithm 1 of
//                                 the paper over three HBM slots and three CUDA
//                                 streams (H2D / compute+D2D / D2H), pinned host
//                                 memory, tile-edge reuse device-to-device, no
//                                 upload of write-first data, no download of
//                                 read-only data, cyclic discard of temporaries.
//   ExecutorKind::resident        in-core: datasets stay in HBM across chains;
//                                 optionally skew-tiled to an L2-sized budget.
//   ExecutorKind::reference       the reference's whole-range semantics, run as
//                                 resident with one tile (there is no CPU path).
//   ExecutorKind::plan_only       flush = plan + record only; nothing executes (CPU
//                                 planner checks; no results can be fetched).
//   tiled_cache / unified         KNL/UM cost models of the reference: out of scope.
#pragma once

#include <map>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "ooc/command.hpp"
#include "ooc/core.hpp"
#include "ooc/device_config.hpp"
#include "ooc/explicit_exec.hpp"
#include "ooc/kernel_exec.hpp"
#include "ooc/metrics.hpp"
#include "ooc/tiler.hpp"

namespace ooc {

enum class ExecutorKind { reference, tiled_cache, tiled_explicit, unified, resident, plan_only };

inline const char* executor_name(ExecutorKind k) {
  switch (k) {
    case ExecutorKind::reference:
      return "reference";
    case ExecutorKind::tiled_cache:
      return "cache";
    case ExecutorKind::tiled_explicit:
      return "explicit";
    case ExecutorKind::unified:
      return "unified";
    case ExecutorKind::resident:
      return "resident";
    default:
      return "plan_only";
  }
}

struct RuntimeOptions {
  ExecutorKind executor = ExecutorKind::reference;
  DeviceConfig device;
  int tiles = 0;  // 0 = choose by capacity (explicit) / 1 (resident)
  int tiled_dim = 0;
  bool prefetch = false;
  ExecPolicy policy = default_exec_policy();
  bool record_chains = false;
  // ---- B200 additions
  int gpu = 0;                      // CUDA device ordinal of this runtime
  index_t resident_budget = 0;      // resident: >0 picks T with 3*slot <= budget (L2 tiling)
  bool profile_loops = false;       // per-launch CUDA events -> per-loop device time
  int arena_fill = 0;               // debug: 0 none, 1 zero (reference behaviour), 2 NaN poison
  bool fuse = true;                 // run point-wise-dependent consecutive loops in one launch
  bool timeline = false;            // record a real event timeline of every command
  bool exact_reductions = false;    // debug: fold reductions in the reference's sequential
                                    // row-major order (bitwise equal; one thread per fold)
  // ---- slab decomposition (multi-GPU, one runtime per GPU): this rank owns rows
  // [own_lo, own_hi) of dimension 0 and recomputes `ghost` rows on each side. Any
  // program runs unchanged: declared datasets and loop ranges are clipped to the
  // rank's window, ghost bands are exchanged after each chain, reductions fold the
  // owned rows and are all-reduced. own_hi <= own_lo: no decomposition.
  int dist_rank = 0, dist_world = 1;
  index_t own_lo = 0, own_hi = 0;
  index_t ghost = 0;
};

/// Ghost-band exchange of one dataset after a chain (rows of dimension 0).
struct HaloXfer {
  DatasetId dataset;
  index_t send_left[2], recv_left[2], send_right[2], recv_right[2];  // [lo, hi) rows
};

struct FlushRecord {
  int chain_id;
  FlushReason reason;
  int loop_count;
};

/// One command of the real event timeline (schema of the reference's simulated
/// Timeline, proj/include/ooc/command.hpp:93-108). kind: 0 h2d, 1 d2h, 2 d2d, 3 kernel.
struct TimelineRow {
  int command_id;
  int kind;
  int queue;
  index_t bytes;
  double issue, start, end;  // seconds from the first recorded command
  DatasetId dataset;
  int tile;
  int loop;
};

/// One executed chain as measured on the device (CUDA events).
struct ChainTiming {
  int chain_id = -1;
  int tiles = 1;
  int loops = 0;
  index_t metric_bytes = 0;
  index_t uploaded = 0, downloaded = 0, d2d = 0;
  double seconds = 0.0;  // first device op of the chain -> last (H2D..D2H)
};

class GpuEngine;  // device-side state: context, slots, resident buffers, events

class Runtime {
 public:
  explicit Runtime(RuntimeOptions opts = {});
  ~Runtime();
  Runtime(const Runtime&) = delete;
  Runtime& operator=(const Runtime&) = delete;

  Mesh& mesh() { return mesh_; }
  const Mesh& mesh() const { return mesh_; }
  const RuntimeOptions& options() const { return opts_; }

  DatasetId declare(const std::string& name, const Extent& core, Point halo, index_t elem_bytes,
                    double fill) {
    return declare_dataset(mesh_, name, window_core(core), halo, elem_bytes, fill);
  }
  DatasetId declare(const std::string& name, const Extent& core, Point halo, index_t elem_bytes,
                    const std::function<double(Point)>& fill) {
    return declare_dataset(mesh_, name, window_core(core), halo, elem_bytes, fill);
  }

  // ---- slab decomposition
  bool windowed() const { return opts_.own_hi > opts_.own_lo; }
  /// The part of a global core this rank stores (owned rows +- ghost rows).
  Extent window_core(const Extent& core) const;
  /// Rows of dimension 0 a chain needs correct beyond the owned rows at its start
  /// (backward sweep of the stencil extents); must not exceed `ghost`.
  index_t dependency_depth(const LoopChain& chain) const;
  /// Ghost-band exchanges after `chain` (datasets it writes that are not write-first).
  std::vector<HaloXfer> halo_plan(const LoopChain& chain);
  /// Join the NCCL communicator of the slab decomposition (128-byte unique id).
  void comm_init(const void* unique_id);
  /// Join the CUDA-IPC transport instead (ranks of one node; same `name` on every rank).
  void comm_init_ipc(const std::string& name);

  void enqueue_loop(ParLoop loop);
  std::vector<double> fetch_dataset(DatasetId d);
  /// Flushing fetch into caller memory (no intermediate std::vector).
  void fetch_dataset_into(DatasetId d, double* out, std::size_t n);
  double fetch_reduction(const std::string& name);

  void set_cyclic_flag(bool on) { cyclic_ = on; }
  /// Exact reductions (RuntimeOptions::exact_reductions) for the chains flushed from now on.
  void set_exact_reductions(bool on);
  bool cyclic_flag() const { return cyclic_; }

  void flush(FlushReason reason = FlushReason::explicit_flush);
  void finish();
  /// Wait for every queued device operation (no host copy-back).
  void sync();
  /// Copy every dataset whose newest values live on the device back to host.
  void sync_host();

  int pending_loops() const { return static_cast<int>(pending_.size()); }
  int chains_flushed() const { return next_chain_id_; }
  const std::vector<FlushRecord>& flush_log() const { return flush_log_; }
  const std::vector<LoopMetric>& loop_metrics();
  const std::vector<AuditRow>& audit_rows() const { return audit_; }
  index_t uploaded() const { return uploaded_; }
  index_t downloaded() const { return downloaded_; }
  index_t d2d_bytes() const { return d2d_; }
  PlanCache& plan_cache() { return plans_; }
  const std::optional<LoopChain>& last_chain() const { return last_chain_; }
  const std::vector<LoopChain>& chain_log() const { return chain_log_; }
  int last_tile_count() const { return last_tiles_; }
  /// Device-measured chain times (forces a device sync to resolve events).
  const std::vector<ChainTiming>& chain_timings();
  RunReport report();
  GpuEngine& engine();
  /// Real event timeline rows resolved so far (RuntimeOptions::timeline).
  const std::vector<TimelineRow>& timeline();
  /// The same rows in the reference's TimelineEntry schema (proj/include/ooc/runtime.hpp:93).
  const std::vector<TimelineEntry>& timeline_entries();
  /// Device-side state shared with run_chain_explicit callers (the GPU engine).
  DeviceState& device_state();
  // CSVs in the reference's schemas (proj/src/metrics.cpp:46-79, command.cpp:160-168)
  std::string report_csv(const std::string& app = "", const std::string& size = "", int iters = 0);
  std::string loops_csv();
  std::string audit_csv() const;
  std::string timeline_csv();

 private:
  void execute(LoopChain&& chain);
  const PlanCache::Entry& plan_for(const LoopChain& chain);

  RuntimeOptions opts_;
  Mesh mesh_;
  std::vector<ParLoop> pending_;
  bool cyclic_ = false;
  int next_loop_id_ = 0;
  int next_chain_id_ = 0;
  PlanCache plans_;
  std::map<std::string, int> tile_choice_;  // choose_tile_count results per structure+budget
  std::vector<FlushRecord> flush_log_;
  std::vector<LoopMetric> loop_metrics_;
  std::map<int, std::size_t> metric_index_;
  std::vector<AuditRow> audit_;
  index_t uploaded_ = 0, downloaded_ = 0, d2d_ = 0;
  int last_tiles_ = 1;
  std::optional<LoopChain> last_chain_;
  std::vector<LoopChain> chain_log_;
  std::map<std::string, int> red_slot_;  // reduction name -> device accumulator slot
  std::map<int, index_t> owned_bytes_;   // windowed runs: metric bytes of the owned rows
  std::vector<ChainTiming> timings_;
  std::vector<TimelineRow> timeline_;
  std::vector<TimelineEntry> timeline_entries_;
  double last_kernel_end_ = 0.0;
  DeviceState device_;  // device_.engine: the GPU engine (created at first use)
};

}  // namespace ooc
