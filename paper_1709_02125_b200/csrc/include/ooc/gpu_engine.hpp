// B200 execution engine behind ooc::Runtime: the out-of-core streaming executor
// (paper Algorithm 1; reference run_chain_explicit, proj/src/explicit_exec.cpp:55-281)
// and the in-core resident executor, both driving the device layer through the C
// ABI in include/ooc_device.h.
#pragma once

#include <chrono>
#include <functional>
#include <map>
#include <string>
#include <vector>

#include "ooc/runtime.hpp"
#include "ooc_device.h"

namespace ooc {

void device_check(int rc, const char* what);  // throws DeviceError on failure

/// Lowered loop: flattened tapes in the device ABI format, reused per tile.
struct LoweredLoop {
  std::vector<ooc_ins> tape;
  std::vector<int> write_arg, write_len;
  int reduce_op = OOC_RED_NONE;
  int reduce_len = 0;
};
LoweredLoop lower_loop(const ParLoop& loop);

/// Loop-fusion legality (see gpu_engine.cpp): can `b` join `group` (total tape
/// length `group_tape`) in one launch without changing any observable value?
bool can_fuse(const std::vector<const ParLoop*>& group, std::size_t group_tape, const ParLoop& b,
              bool enabled);

/// Process-wide: admit row-recompute fusion (default on; OOC_ROW_RECOMPUTE=0 disables).
void set_row_recompute(bool on);

/// Fusion partition of a chain into consecutive launch groups: starts[j] = 1 where a
/// launch begins. Among all partitions whose groups pass `can_fuse` (as the engine
/// checks them, prefix by prefix) it picks the one with the least estimated DRAM
/// traffic plus a per-launch cost — greedy first-fit can strand loops in extra
/// launches that re-read what the previous launch just wrote.
std::vector<char> plan_fusion(const Mesh& mesh, const std::vector<ParLoop>& loops,
                              const std::vector<std::size_t>& tape_len, bool enabled);

/// Dense (optionally row-padded) device layout of a box.
struct BoxLayout {
  Extent box;       // the largest box the layout must hold (per-dim max lengths)
  Point stride{0, 0, 0};
  index_t elems = 0;
};
BoxLayout padded_layout(const Extent& box, index_t pad_elems = 16);
ooc_view view_at(double* data, const Extent& box, const Point& stride);
ooc_view host_view(Dataset& ds);
ooc_loop make_call(const LoweredLoop& lw, const Extent& sub, const std::vector<ooc_view>& views, int red_slot);
/// A run of consecutive loops [a, b) executed by one row-sweep launch; `dead` = the
/// datasets it writes whose values are overwritten before anyone reads them.
struct SweepRun {
  std::size_t a = 0, b = 0;
  std::vector<DatasetId> dead;
};
/// Row-sweep partition of an untiled chain: the least-traffic split into sweep runs
/// (>= 2 loops each, accepted by ooc_sweep_check) and loops left to the other kernels.
std::vector<SweepRun> plan_sweeps(const Mesh& mesh, const std::vector<ParLoop>& loops, bool exact_reductions,
                                  const std::vector<ooc_loop>& calls);
std::string sweep_key(const Mesh& mesh, const LoopChain& chain);
bool sweep_enabled();  // OOC_SWEEP=0 disables
void set_sweep(bool on);  // process-wide override

class GpuEngine {
 public:
  explicit GpuEngine(const RuntimeOptions& opts);
  ~GpuEngine();

  struct ChainOut {
    std::vector<AuditRow> audit;
    std::map<int, int> reduction_slot;  // loop id -> accumulator slot
  };

  void run_explicit(Mesh& mesh, const LoopChain& chain, const TilePlan& plan,
                    const Footprints& fp, bool cyclic, ChainOut& out,
                    const std::vector<HaloXfer>* halos = nullptr);
  void run_resident(Mesh& mesh, const LoopChain& chain, const TilePlan* plan,
                    const Footprints* fp, ChainOut& out,
                    const std::vector<HaloXfer>* halos = nullptr);
  /// Join the NCCL communicator of the slab decomposition.
  void comm_init(int rank, int world, const void* unique_id);
  /// Join the CUDA-IPC transport of the slab decomposition (ranks of one node; `name`
  /// identifies the job's shared-memory rendezvous).
  void comm_init_ipc(int rank, int world, const std::string& name);
  int rank() const { return rank_; }
  int world() const { return world_; }
  bool comm_ready() const { return comm_ready_; }

  /// Resident mode: newest values of `d` are on the device (host copy stale).
  bool host_outdated(DatasetId d) const;
  void download_resident(Mesh& mesh, DatasetId d);
  void forget_resident(DatasetId d);
  /// A fetched dataset's staged first tile may be modified before the next chain
  /// (reference Runtime::fetch_dataset, proj/src/runtime.cpp:17).
  void invalidate_staged(DatasetId d);
  /// Block until the reduction written to `slot` has reached host memory.
  double reduction_value(int slot);
  void sync();
  /// Record a timing event on the compute queue; wait on the D2H queue first so a
  /// mark also covers every download issued so far.
  int mark();
  double mark_elapsed(int a, int b);
  std::vector<ChainTiming> take_timings();
  std::map<int, double> take_loop_times();
  /// Profiled launches (profile_loops): first loop id, #loops, metric bytes, seconds.
  struct LaunchRecord {
    int first_loop, nloops;
    index_t bytes;
    double seconds;
  };
  std::vector<LaunchRecord> launch_log;
  /// Resolve the real event timeline recorded so far (RuntimeOptions::timeline).
  std::vector<TimelineRow> take_timeline();
  ooc_ctx* ctx() { return ctx_; }
  /// ExecOptions::prefetch per call (run_chain_explicit seam).
  void set_prefetch(bool on) { opts_.prefetch = on; }
  /// Exact reductions: reducing loops run alone through the contribution path and one
  /// thread folds them in row-major order; sweeps stop before them, graphs are off.
  void set_exact_reductions(bool on);
  bool exact_reductions() const { return opts_.exact_reductions; }
  int slot_cursor() const { return slot_cursor_; }
  /// Datasets whose next-chain first tile is staged in HBM, with the staged region.
  std::map<DatasetId, Extent> staged_regions() const {
    std::map<DatasetId, Extent> m;
    for (const auto& [d, s] : staged_) m[d] = s.region;
    return m;
  }
  const ooc_dev_props& props() const { return props_; }

 private:
  struct Resident {
    double* dev = nullptr;
    double* shadow = nullptr;  // second buffer for out-of-place sweep outputs (swapped with dev)
    BoxLayout layout;
    bool dev_valid = false;
    bool host_outdated = false;
    const double* host_ptr = nullptr;
  };
  struct PendingChain {
    ChainTiming t;
    ooc_event* start = nullptr;
    ooc_event* end = nullptr;
  };
  struct PendingLoop {
    std::vector<std::pair<int, double>> weights;  // loop id -> share of the launch time
    index_t bytes = 0;                            // metric bytes of the launch
    ooc_event* a;
    ooc_event* b;
  };
  struct Group {  // loops collected for one fused launch
    std::vector<ooc_loop> calls;
    std::vector<const ParLoop*> loops;
    std::vector<index_t> bytes;
    std::size_t tape_len = 0;
  };

  ooc_event* ev(std::vector<ooc_event*>& pool, std::size_t i, bool timing = false);
  ooc_event* fresh_timing_event();
  void recycle(ooc_event* e);
  int alloc_red_slot();
  void launch(int queue, bool group_start, int tile, const ParLoop& loop, const LoweredLoop& lw,
              const Extent& sub,
              const std::vector<ooc_view>& views, int red_slot);
  bool fusable(const ParLoop& b) const;
  void flush_group(int queue);
  void issue_instrumented(int queue, const std::vector<const ParLoop*>& loops, const std::vector<index_t>& bytes,
                          const std::function<void()>& issue);
  /// One row-sweep launch; false (nothing launched) when HBM has no room for a shadow.
  bool run_sweep(Mesh& mesh, const LoopChain& chain, const SweepRun& run, const std::vector<LoweredLoop>& lowered,
                 std::vector<DatasetId>& flipped, const std::map<int, int>& red_slots);
  index_t loop_bytes_per_point_views(const ParLoop& loop) const;
  void ensure_pool(index_t elems);
  void ensure_resident(Mesh& mesh, DatasetId d);
  void finish_chain(const LoopChain& chain, const std::map<int, int>& red, PendingChain pc,
                    int end_queue = OOC_Q_COMPUTE);

  RuntimeOptions opts_;
  ooc_ctx* ctx_ = nullptr;
  ooc_dev_props props_{};
  // explicit-mode slot pool (three slots)
  double* pool_ = nullptr;
  index_t pool_elems_ = 0;
  int slot_cursor_ = 0;
  // per-tile events, double-buffered by chain parity so the next chain can wait on
  // the previous chain's downloads while recording its own
  std::vector<ooc_event*> ev_h2d_[2], ev_k_[2], ev_q0_[2], ev_d2h_[2];
  ooc_event* chain_done_[2] = {nullptr, nullptr};
  long long chain_count_ = 0;
  // last users of each slot (may belong to the previous chain)
  ooc_event* slot_q0_[3] = {nullptr, nullptr, nullptr};
  ooc_event* slot_d2h_[3] = {nullptr, nullptr, nullptr};
  // host rows the previous chain downloaded, per dataset: (box, tile)
  std::vector<std::vector<std::pair<Extent, int>>> prev_down_;
  // speculative first-tile stages for the next chain (reference DeviceState::staged)
  struct Staged {
    Extent region;
    ooc_view view;
  };
  std::map<DatasetId, Staged> staged_;
  double* staging_ = nullptr;
  index_t staging_elems_ = 0;
  void ensure_staging(index_t elems);
  /// Out-of-core slabs: refresh the host ghost bands of `halos` from the neighbours'
  /// owned rows (after this chain's downloads): H2D of the send bands into a device
  /// scratch, exchange, D2H of the received bands.
  void exchange_host_bands(Mesh& mesh, const std::vector<HaloXfer>& halos);
  double* band_stage_ = nullptr;
  index_t band_stage_elems_ = 0;
  struct TLPending {
    int kind, queue;
    index_t bytes;
    DatasetId dataset;
    int tile;
    std::vector<std::pair<int, index_t>> loops;
    double issue;
    ooc_event* a;
    ooc_event* b;
  };
  void timeline_cmd(int kind, int queue, index_t bytes, DatasetId d, int tile,
                    std::vector<std::pair<int, index_t>> loops, const std::function<void()>& issue);
  std::vector<TLPending> tl_pending_;
  // CUDA graphs of repeated resident chains (key: everything a launch bakes in)
  // Two graphs per chain structure, alternating, each with its own reduction slots
  // (from the upper half of the slot range) so a replay never waits on the previous chain.
  struct GraphEntry {
    int seen = 0;
    int flip = 0;
    bool settled = false;  // the last direct run made no tuning launch
    ooc_graph* g[2] = {nullptr, nullptr};
    std::vector<int> slots[2];
    std::vector<DatasetId> flips;  // datasets whose buffers the chain's sweeps swap (odd count)
  };
  std::map<std::string, GraphEntry> graphs_;
  int next_graph_slot_ = OOC_REDUCE_SLOTS / 2;
  std::string graph_key(const LoopChain& chain, const TilePlan* plan, bool pointers = true) const;
  std::map<std::string, int> struct_seen_;  // sightings per chain structure (all buffer states)
  ooc_event* tl_base_ = nullptr;
  std::chrono::steady_clock::time_point tl_host0_;
  int next_cmd_ = 0;
  int cur_tile_ = 0;
  // resident buffers by dataset id
  std::vector<Resident> res_;
  // reductions: device accumulator slot -> pinned host mirror
  double* red_host_ = nullptr;
  int next_red_slot_ = 0;
  std::map<int, ooc_event*> red_ready_;  // slot -> event after its D2H
  std::vector<ooc_event*> free_timing_;
  std::vector<PendingChain> pending_chains_;
  std::vector<PendingLoop> pending_loops_;
  std::vector<ooc_event*> marks_;
  Group group_;
  int rank_ = 0, world_ = 1;
  bool comm_ready_ = false;
};

}  // namespace ooc
