// Lazy loop-chain runtime (flush semantics of proj/src/runtime.cpp:5-148) over the
// B200 engine.
#include "ooc/runtime.hpp"

#include <algorithm>
#include <sstream>

#include "ooc/gpu_engine.hpp"
#include "ooc_device.h"

namespace ooc {

Runtime::Runtime(RuntimeOptions opts) : opts_(opts) {
  // this runtime's datasets (declared on this thread) are pinned next to its GPU
  ooc_host_numa_device(opts_.gpu);
  if (opts_.executor == ExecutorKind::tiled_cache || opts_.executor == ExecutorKind::unified)
    throw ValidationError(std::string("executor '") + executor_name(opts_.executor) +
                          "' (a KNL cache / unified-memory cost model of the reference) is not "
                          "part of the B200 build; use tiled_explicit or resident");
}

Runtime::~Runtime() = default;

GpuEngine& Runtime::engine() {
  if (!device_.engine) {
    device_.engine = std::make_shared<GpuEngine>(opts_);
    device_.gpu = opts_.gpu;
  }
  return *device_.engine;
}

void Runtime::set_exact_reductions(bool on) {
  opts_.exact_reductions = on;  // applies to every chain executed from now on
  if (device_.engine) device_.engine->set_exact_reductions(on);
}

DeviceState& Runtime::device_state() {
  engine();
  return device_;
}

const std::vector<TimelineEntry>& Runtime::timeline_entries() {
  const std::vector<TimelineRow>& rows = timeline();
  for (std::size_t i = timeline_entries_.size(); i < rows.size(); ++i) {
    const TimelineRow& r = rows[i];
    timeline_entries_.push_back({r.command_id, static_cast<CmdKind>(r.kind), r.queue, r.bytes, r.issue, r.start,
                                 r.end, r.dataset, r.tile, r.loop});
  }
  return timeline_entries_;
}

Extent Runtime::window_core(const Extent& core) const {
  if (!windowed()) return core;
  Extent c = core;
  c.lo[0] = std::max(core.lo[0], opts_.own_lo - opts_.ghost);
  c.hi[0] = std::min(core.hi[0], opts_.own_hi + opts_.ghost);
  if (c.lo[0] >= c.hi[0])
    throw ValidationError("dataset core " + core.str() + " lies outside this rank's rows [" +
                          std::to_string(opts_.own_lo - opts_.ghost) + "," +
                          std::to_string(opts_.own_hi + opts_.ghost) + ")");
  return c;
}

void Runtime::enqueue_loop(ParLoop loop) {  // runtime.cpp:5-11
  if (windowed()) {
    // owned rows carry the metric (so ranks sum to the global metric); reductions
    // fold only owned rows; every other loop runs on the whole window
    Extent owned = loop.range;
    owned.lo[0] = std::max(owned.lo[0], opts_.own_lo);
    owned.hi[0] = std::min(owned.hi[0], opts_.own_hi);
    Extent run = owned;
    if (!loop.has_reduction()) {
      run = loop.range;
      run.lo[0] = std::max(run.lo[0], opts_.own_lo - opts_.ghost);
      run.hi[0] = std::min(run.hi[0], opts_.own_hi + opts_.ghost);
      // near the window edge a loop shrinks by its own stencil reach (rows it cannot
      // read locally); dependency_depth() <= ghost keeps the owned rows exact
      for (const LoopArg& a : loop.args) {
        if (a.dataset < 0 || a.dataset >= static_cast<int>(mesh_.datasets.size())) continue;
        const Dataset& ds = mesh_[a.dataset];
        if (access_reads(a.mode)) {
          auto [slo, shi] = stencil_extents(a.stencil);
          run.lo[0] = std::max(run.lo[0], ds.alloc().lo[0] - slo[0]);
          run.hi[0] = std::min(run.hi[0], ds.alloc().hi[0] - shi[0]);
        }
        if (access_writes(a.mode)) {
          run.lo[0] = std::max(run.lo[0], ds.core.lo[0]);
          run.hi[0] = std::min(run.hi[0], ds.core.hi[0]);
        }
      }
    }
    if (run.empty() || owned.empty())
      throw ValidationError("loop range " + loop.range.str() +
                            " does not reach this rank's owned rows (slab too thin)");
    loop.range = run;
    validate_loop(mesh_, loop);
    loop.id = next_loop_id_;
    owned_bytes_[loop.id] = owned.size() * loop_bytes_per_point(mesh_, loop);
  }
  validate_loop(mesh_, loop);
  loop.id = next_loop_id_++;
  const bool reduces = loop.has_reduction();
  pending_.push_back(std::move(loop));
  if (reduces) flush(FlushReason::reduction_fetch);
}

std::vector<double> Runtime::fetch_dataset(DatasetId d) {  // runtime.cpp:13-19
  if (d < 0 || d >= static_cast<DatasetId>(mesh_.datasets.size()))
    throw ValidationError("fetch of an unknown dataset");
  std::vector<double> out(mesh_[d].host.size());
  fetch_dataset_into(d, out.data(), out.size());
  return out;
}

void Runtime::fetch_dataset_into(DatasetId d, double* dst, std::size_t n) {
  flush(FlushReason::data_fetch);
  if (d < 0 || d >= static_cast<DatasetId>(mesh_.datasets.size()))
    throw ValidationError("fetch of an unknown dataset");
  if (opts_.executor == ExecutorKind::plan_only && next_chain_id_ > 0)
    throw ValidationError("plan_only runtime executes nothing; no results to fetch");
  Dataset& ds = mesh_[d];
  if (ds.host_stale) throw StaleDataError(ds.name, ds.stale_chain);
  if (n != ds.host.size()) throw ValidationError("fetch buffer has the wrong length");
  if (device_.engine) {
    if (device_.engine->host_outdated(d))
      device_.engine->download_resident(mesh_, d);
    else
      device_.engine->sync();  // streamed downloads of earlier chains must have landed
    device_.engine->invalidate_staged(d);  // runtime.cpp:17
  }
  std::copy(ds.host.begin(), ds.host.end(), dst);
}

double Runtime::fetch_reduction(const std::string& name) {  // runtime.cpp:21-26
  flush(FlushReason::data_fetch);
  if (opts_.executor == ExecutorKind::plan_only)
    throw ValidationError("plan_only runtime executes nothing; no results to fetch");
  auto it = red_slot_.find(name);
  if (it == red_slot_.end()) throw ValidationError("unknown reduction '" + name + "'");
  return engine().reduction_value(it->second);
}

void Runtime::flush(FlushReason reason) {  // runtime.cpp:28-39
  if (pending_.empty()) return;
  LoopChain chain;
  chain.chain_id = next_chain_id_++;
  chain.reason = reason;
  chain.loops = std::move(pending_);
  pending_.clear();
  flush_log_.push_back({chain.chain_id, reason, static_cast<int>(chain.loops.size())});
  last_chain_ = chain;
  if (opts_.record_chains) chain_log_.push_back(chain);
  execute(std::move(chain));
}

void Runtime::finish() {
  flush(FlushReason::program_end);
  sync_host();
}

void Runtime::sync() {
  if (device_.engine) device_.engine->sync();
}

void Runtime::sync_host() {
  if (!device_.engine) return;
  for (std::size_t d = 0; d < mesh_.datasets.size(); ++d)
    if (device_.engine->host_outdated(static_cast<DatasetId>(d)))
      device_.engine->download_resident(mesh_, static_cast<DatasetId>(d));
  device_.engine->sync();
}

const PlanCache::Entry& Runtime::plan_for(const LoopChain& chain) {  // runtime.cpp:41-62
  if (opts_.tiles > 0) return plans_.get(mesh_, chain, opts_.tiles, opts_.tiled_dim);
  index_t budget = opts_.device.capacity_bytes;
  // resident (in-core) tiling has no slot rotation: one tile's working set must fit
  // the budget (e.g. L2), so choose the smallest T with slot_bytes <= budget.
  if (opts_.executor == ExecutorKind::resident) budget = 3 * opts_.resident_budget;
  // the linear scan is O(T) plans: remember its answer per chain structure and budget
  const std::string key = chain_structural_key(mesh_, chain) + "|" + std::to_string(budget);
  auto it = tile_choice_.find(key);
  if (it == tile_choice_.end())
    it = tile_choice_.emplace(key, choose_tile_count(mesh_, chain, budget, opts_.tiled_dim).tile_count).first;
  return plans_.get(mesh_, chain, it->second, opts_.tiled_dim);
}

void Runtime::execute(LoopChain&& chain) {  // runtime.cpp:64-148
  for (const ParLoop& l : chain.loops) {
    auto it = metric_index_.find(l.id);
    if (it != metric_index_.end()) continue;
    LoopMetric m;
    m.loop_id = l.id;
    m.points = l.range.size();
    auto ob = owned_bytes_.find(l.id);
    m.bytes = ob != owned_bytes_.end() ? ob->second : l.range.size() * loop_bytes_per_point(mesh_, l);
    metric_index_[l.id] = loop_metrics_.size();
    loop_metrics_.push_back(m);
  }
  if (opts_.executor == ExecutorKind::plan_only) {
    const PlanCache::Entry& e = plan_for(chain);
    last_tiles_ = e.plan.tile_count;
    return;
  }
  GpuEngine& g = engine();
  // slab decomposition: every chain's owned rows must be exact (ghost rows >= the chain's
  // dependency depth) and, with neighbours, refreshed and combined after it — never run
  // a multi-rank slab silently without its exchange
  const bool slabbed = windowed() && opts_.dist_world > 1;
  if (slabbed && opts_.exact_reductions)
    throw ValidationError("exact reductions fold on one rank; the slab decomposition all-reduces per-rank folds");
  if (slabbed && !g.comm_ready())
    throw ValidationError("slab decomposition over " + std::to_string(opts_.dist_world) +
                          " ranks needs a communicator (comm_init / comm_init_ipc) before its first chain");
  std::vector<HaloXfer> halos;
  if (windowed()) {
    const index_t depth = dependency_depth(chain);
    if (depth > opts_.ghost)
      throw ValidationError("chain " + std::to_string(chain.chain_id) + " needs " + std::to_string(depth) +
                            " ghost rows; the slab has " + std::to_string(opts_.ghost));
    if (g.comm_ready()) halos = halo_plan(chain);
  }
  GpuEngine::ChainOut out;
  if (opts_.executor == ExecutorKind::tiled_explicit) {
    const PlanCache::Entry& e = plan_for(chain);
    last_tiles_ = e.plan.tile_count;
    // a chain that would upload cyclically discarded data would ship garbage
    for (std::size_t d = 0; d < e.footprints.per_dataset.size(); ++d) {
      const auto& pd = e.footprints.per_dataset[d];
      const Dataset& ds = mesh_[static_cast<DatasetId>(d)];
      if (pd.accessed && ds.host_stale && !pd.write_first)
        throw StaleDataError(ds.name, ds.stale_chain);
    }
    g.run_explicit(mesh_, chain, e.plan, e.footprints, cyclic_, out, g.comm_ready() ? &halos : nullptr);
  } else {
    const bool tiled = opts_.executor == ExecutorKind::resident &&
                       (opts_.tiles > 1 || (opts_.tiles == 0 && opts_.resident_budget > 0));
    if (tiled && windowed())
      throw ValidationError("resident tiling (tiles > 1 or resident_budget) cannot be combined with the "
                            "slab decomposition; use the untiled resident or the tiled_explicit executor");
    if (tiled) {
      const PlanCache::Entry& e = plan_for(chain);
      last_tiles_ = e.plan.tile_count;
      g.run_resident(mesh_, chain, &e.plan, &e.footprints, out);
    } else if (windowed() && g.comm_ready()) {
      last_tiles_ = 1;
      g.run_resident(mesh_, chain, nullptr, nullptr, out, &halos);
    } else {
      last_tiles_ = 1;
      g.run_resident(mesh_, chain, nullptr, nullptr, out);
    }
  }
  for (const ParLoop& l : chain.loops)
    if (l.has_reduction()) red_slot_[l.kernel.reduce_name] = out.reduction_slot.at(l.id);
  for (const AuditRow& r : out.audit) {
    audit_.push_back(r);
    uploaded_ += r.uploaded;
    downloaded_ += r.downloaded;
    d2d_ += r.d2d;
  }
}

// Rows of dimension 0 each dataset must be correct beyond the owned rows at the
// start of the chain so the owned rows are exact at its end: a backward sweep like
// the planner's (tiler.cpp:100-134) — a loop that must produce rows owned+-e reads
// its stencil's reach beyond that.
index_t Runtime::dependency_depth(const LoopChain& chain) const {
  std::vector<index_t> need(mesh_.datasets.size(), 0);
  for (std::size_t jj = chain.loops.size(); jj-- > 0;) {
    const ParLoop& l = chain.loops[jj];
    index_t e = 0;
    for (const LoopArg& a : l.args)
      if (access_writes(a.mode)) e = std::max(e, need[static_cast<std::size_t>(a.dataset)]);
    for (const LoopArg& a : l.args) {
      if (!access_reads(a.mode)) continue;
      auto [lo, hi] = stencil_extents(a.stencil);
      const index_t reach = e + std::max(-lo[0], hi[0]);
      auto& n = need[static_cast<std::size_t>(a.dataset)];
      n = std::max(n, reach);
    }
  }
  index_t d = 0;
  for (index_t v : need) d = std::max(d, v);
  return d;
}

std::vector<HaloXfer> Runtime::halo_plan(const LoopChain& chain) {
  std::vector<HaloXfer> out;
  std::vector<char> written(mesh_.datasets.size(), 0);
  for (const ParLoop& l : chain.loops)
    for (const LoopArg& a : l.args)
      if (access_writes(a.mode)) written[static_cast<std::size_t>(a.dataset)] = 1;
  const index_t lo = opts_.own_lo, hi = opts_.own_hi;
  const bool left = opts_.dist_rank > 0, right = opts_.dist_rank + 1 < opts_.dist_world;
  for (std::size_t d = 0; d < written.size(); ++d) {
    if (!written[d]) continue;  // untouched data keeps its (globally correct) values
    const Dataset& ds = mesh_[static_cast<DatasetId>(d)];
    const Extent a = ds.alloc();
    const index_t band = opts_.ghost + ds.halo[0];
    auto clip = [&](index_t r0, index_t r1, index_t* dst) {
      dst[0] = std::max(r0, a.lo[0]);
      dst[1] = std::max(dst[0], std::min(r1, a.hi[0]));
    };
    HaloXfer h{};
    h.dataset = static_cast<DatasetId>(d);
    if (left) {
      clip(lo, lo + band, h.send_left);
      clip(lo - band, lo, h.recv_left);
    }
    if (right) {
      clip(hi - band, hi, h.send_right);
      clip(hi, hi + band, h.recv_right);
    }
    out.push_back(h);
  }
  return out;
}

void Runtime::comm_init(const void* unique_id) {
  engine().comm_init(opts_.dist_rank, opts_.dist_world, unique_id);
}

void Runtime::comm_init_ipc(const std::string& name) {
  engine().comm_init_ipc(opts_.dist_rank, opts_.dist_world, name);
}

const std::vector<ChainTiming>& Runtime::chain_timings() {
  if (device_.engine)
    for (ChainTiming& t : device_.engine->take_timings()) timings_.push_back(t);
  return timings_;
}

const std::vector<LoopMetric>& Runtime::loop_metrics() {
  if (device_.engine && opts_.timeline) {
    timeline();
  } else if (device_.engine) {
    for (const auto& [id, s] : device_.engine->take_loop_times()) {
      auto it = metric_index_.find(id);
      if (it == metric_index_.end()) continue;
      LoopMetric& m = loop_metrics_[it->second];
      m.time_s += s;
      m.bandwidth = m.time_s > 0 ? static_cast<double>(m.bytes) / m.time_s : 0.0;
    }
  }
  return loop_metrics_;
}

// Real-timeline loop attribution (restates proj/src/metrics.cpp:14-32 over measured
// rows): kernel rows sorted by (start, command_id); each gets max(0, end - prev_end).
const std::vector<TimelineRow>& Runtime::timeline() {
  if (!device_.engine) return timeline_;
  std::vector<TimelineRow> rows = device_.engine->take_timeline();
  std::vector<const TimelineRow*> k;
  for (const TimelineRow& r : rows)
    if (r.kind == 3) k.push_back(&r);
  std::sort(k.begin(), k.end(), [](const TimelineRow* a, const TimelineRow* b) {
    if (a->start != b->start) return a->start < b->start;
    return a->command_id < b->command_id;
  });
  for (const TimelineRow* e : k) {
    const double span = std::max(0.0, e->end - last_kernel_end_);
    if (e->end > last_kernel_end_) last_kernel_end_ = e->end;
    auto it = metric_index_.find(e->loop);
    if (it == metric_index_.end()) continue;
    LoopMetric& m = loop_metrics_[it->second];
    m.time_s += span;
    m.bandwidth = m.time_s > 0 ? static_cast<double>(m.bytes) / m.time_s : 0.0;
  }
  timeline_.insert(timeline_.end(), rows.begin(), rows.end());
  return timeline_;
}

static const char* kind_name(int k) {
  static const char* n[] = {"h2d", "d2h", "d2d", "kernel"};
  return k >= 0 && k < 4 ? n[k] : "unknown";
}

std::string Runtime::timeline_csv() {
  std::ostringstream os;  // proj/src/command.cpp:160-168
  os << "command_id,kind,queue,bytes,issue,start,end\n";
  os.precision(12);
  for (const TimelineRow& e : timeline())
    os << e.command_id << "," << kind_name(e.kind) << "," << e.queue << "," << e.bytes << ","
       << e.issue << "," << e.start << "," << e.end << "\n";
  return os.str();
}

std::string Runtime::report_csv(const std::string& app, const std::string& size, int iters) {
  RunReport r = report();  // proj/src/metrics.cpp:46-60
  r.app = app;
  r.size = size;
  r.iters = iters;
  std::ostringstream os;
  os << "#oocstencil-report-v1\n"
        "app,size,iters,mode,tiles,capacity,average_bandwidth,total_bytes,total_time,"
        "makespan,uploaded,downloaded,d2d,efficiency,hit_rate,faults,error\n";
  os.precision(12);
  os << r.app << "," << r.size << "," << r.iters << "," << r.mode << "," << r.tiles << ","
     << r.capacity << "," << r.average_bandwidth << "," << r.total_bytes << "," << r.total_time
     << "," << r.makespan << "," << r.uploaded << "," << r.downloaded << "," << r.d2d << ","
     << r.efficiency << "," << r.hit_rate << "," << r.faults << "," << r.error << "\n";
  return os.str();
}

std::string Runtime::loops_csv() {
  std::ostringstream os;  // proj/src/metrics.cpp:62-70
  os << "#oocstencil-report-v1\nloop,points,bytes,time,bandwidth\n";
  os.precision(12);
  for (const LoopMetric& l : loop_metrics())
    os << l.loop_id << "," << l.points << "," << l.bytes << "," << l.time_s << "," << l.bandwidth
       << "\n";
  return os.str();
}

std::string Runtime::audit_csv() const {
  std::ostringstream os;  // proj/src/metrics.cpp:72-79
  os << "dataset,tile,uploaded,downloaded,d2d\n";
  for (const AuditRow& r : audit_)
    os << mesh_[r.dataset].name << "," << r.tile << "," << r.uploaded << "," << r.downloaded << ","
       << r.d2d << "\n";
  return os.str();
}

RunReport Runtime::report() {
  RunReport r;
  r.mode = executor_name(opts_.executor);
  r.tiles = opts_.tiles > 0 ? opts_.tiles : last_tiles_;
  for (const LoopMetric& m : loop_metrics()) r.total_bytes += m.bytes;
  for (const ChainTiming& t : chain_timings()) r.total_time += t.seconds;
  r.makespan = r.total_time;
  if (r.total_time > 0) r.average_bandwidth = static_cast<double>(r.total_bytes) / r.total_time;
  r.uploaded = uploaded_;
  r.downloaded = downloaded_;
  r.d2d = d2d_;
  r.capacity = opts_.device.capacity_bytes;
  return r;
}

}  // namespace ooc
