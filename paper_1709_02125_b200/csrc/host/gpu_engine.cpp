// The B200 streaming engine (paper Alg. 1) and the resident in-core executor.
//
// Streaming executor — restates the data movement of the reference's
// run_chain_explicit (proj/src/explicit_exec.cpp:55-281) on real hardware:
//   * three slots in HBM, slot(t) = (cursor + t) % 3 (explicit_exec.cpp:75, 273);
//   * tile 0 uploads full[0], tile t+1 uploads right_fp[t+1] on the H2D queue while
//     tile t computes (explicit_exec.cpp:174-186);
//   * kernels of tile t on the compute queue, then the right edge is carried
//     device-to-device into slot(t+1) (explicit_exec.cpp:206-231);
//   * left_fp[t] of written datasets downloads on the D2H queue
//     (explicit_exec.cpp:233-242): read-only data never travels back, write-first
//     data never travels up (:86, :235), cyclic drops write-first data (:236-239).
// Every cross-queue hazard is an explicit CUDA event wait, including the
// compute-waits-for-its-upload dependency the reference's simulated timeline
// omits (kernels of tile t wait for the H2D of tile t).
#include "ooc/gpu_engine.hpp"

#include <cstdio>
#include <cstdlib>
#include <map>

#include <cmath>
#include <cstring>

namespace ooc {

void device_check(int rc, const char* what) {
  if (rc == OOC_OK) return;
  std::string msg = std::string(what) + ": " + ooc_dev_last_error();
  if (rc == OOC_ERR_CAPACITY) throw CapacityError(-1, -1);
  throw DeviceError(rc, msg);
}

#define DEV(call) device_check((call), #call)

// ---------------------------------------------------------------- lowering / layouts

LoweredLoop lower_loop(const ParLoop& loop) {
  LoweredLoop lw;
  auto put = [&](const ExprTape& t) {
    for (const auto& in : t.ins) {
      ooc_ins o{};
      o.op = static_cast<int32_t>(in.op);
      o.arg = in.arg;
      o.value = in.value;
      for (int d = 0; d < 3; ++d) o.offset[d] = in.offset[d];
      lw.tape.push_back(o);
    }
    return static_cast<int>(t.ins.size());
  };
  for (std::size_t w = 0; w < loop.kernel.writes.size(); ++w) {
    lw.write_arg.push_back(loop.kernel.writes[w].arg);
    lw.write_len.push_back(put(loop.write_tapes[w]));
  }
  if (loop.has_reduction()) {
    lw.reduce_op = loop.kernel.reduce == ReduceOp::sum   ? OOC_RED_SUM
                   : loop.kernel.reduce == ReduceOp::min ? OOC_RED_MIN
                                                         : OOC_RED_MAX;
    lw.reduce_len = put(loop.reduce_tape);
  }
  return lw;
}

BoxLayout padded_layout(const Extent& box, index_t pad) {
  BoxLayout L;
  L.box = box;
  const int nd = box.ndim;
  const index_t n0 = box.len(0), n1 = box.len(1), n2 = box.len(2);
  auto up = [&](index_t v) { return (v + pad - 1) / pad * pad; };
  if (nd == 1) {
    L.stride = {1, 1, 1};
    L.elems = n0;
  } else if (nd == 2) {
    L.stride = {up(n1), 1, 1};
    L.elems = L.stride[0] * n0;
  } else {
    L.stride = {up(n2) * n1, up(n2), 1};
    L.elems = L.stride[0] * n0;
  }
  return L;
}

ooc_view view_at(double* data, const Extent& box, const Point& stride) {
  ooc_view v{};
  v.data = data;
  for (int d = 0; d < 3; ++d) {
    v.lo[d] = box.lo[d];
    v.hi[d] = box.hi[d];
    v.stride[d] = stride[d];
  }
  return v;
}

ooc_view host_view(Dataset& ds) {
  const Extent a = ds.alloc();
  return view_at(ds.host.data(), a, a.strides());
}

// ---------------------------------------------------------------- engine

GpuEngine::GpuEngine(const RuntimeOptions& opts) : opts_(opts) {
  DEV(ooc_ctx_create(opts.gpu, &ctx_));
  DEV(ooc_ctx_props(ctx_, &props_));
  DEV(ooc_set_reduce_exact(ctx_, opts.exact_reductions ? 1 : 0));
  void* p = nullptr;
  DEV(ooc_host_alloc(sizeof(double) * OOC_REDUCE_SLOTS, &p));
  red_host_ = static_cast<double*>(p);
  std::memset(red_host_, 0, sizeof(double) * OOC_REDUCE_SLOTS);
}

void GpuEngine::set_exact_reductions(bool on) {
  opts_.exact_reductions = on;
  DEV(ooc_set_reduce_exact(ctx_, on ? 1 : 0));
}

GpuEngine::~GpuEngine() {
  if (!ctx_) return;
  ooc_ctx_sync(ctx_);
  for (auto& [k, e] : graphs_) {
    ooc_graph_destroy(e.g[0]);
    ooc_graph_destroy(e.g[1]);
  }
  auto drop = [&](std::vector<ooc_event*>& v) {
    for (auto* e : v) ooc_event_destroy(ctx_, e);
    v.clear();
  };
  for (int p = 0; p < 2; ++p) {
    drop(ev_h2d_[p]);
    drop(ev_k_[p]);
    drop(ev_q0_[p]);
    drop(ev_d2h_[p]);
    if (chain_done_[p]) ooc_event_destroy(ctx_, chain_done_[p]);
  }
  drop(free_timing_);
  for (auto& pc : pending_chains_) {
    ooc_event_destroy(ctx_, pc.start);
    ooc_event_destroy(ctx_, pc.end);
  }
  for (auto& pl : pending_loops_) {
    ooc_event_destroy(ctx_, pl.a);
    ooc_event_destroy(ctx_, pl.b);
  }
  for (auto& [slot, e] : red_ready_) ooc_event_destroy(ctx_, e);
  for (auto* e : marks_) ooc_event_destroy(ctx_, e);
  if (red_host_) ooc_host_free(red_host_);
  ooc_ctx_destroy(ctx_);  // frees pool and resident buffers tracked by the manager
}

ooc_event* GpuEngine::ev(std::vector<ooc_event*>& pool, std::size_t i, bool timing) {
  while (pool.size() <= i) {
    ooc_event* e = nullptr;
    DEV(ooc_event_create(ctx_, timing ? 1 : 0, &e));
    pool.push_back(e);
  }
  return pool[i];
}

ooc_event* GpuEngine::fresh_timing_event() {
  if (!free_timing_.empty()) {
    ooc_event* e = free_timing_.back();
    free_timing_.pop_back();
    return e;
  }
  ooc_event* e = nullptr;
  DEV(ooc_event_create(ctx_, 1, &e));
  return e;
}

void GpuEngine::recycle(ooc_event* e) {
  if (e) free_timing_.push_back(e);
}

int GpuEngine::alloc_red_slot() {
  int s = next_red_slot_;
  next_red_slot_ = (next_red_slot_ + 1) % (OOC_REDUCE_SLOTS / 2);  // upper half: graphs
  auto it = red_ready_.find(s);
  if (it != red_ready_.end()) {  // slot reuse: its previous value must have landed
    DEV(ooc_event_sync(ctx_, it->second));
  }
  return s;
}

// Loop fusion: consecutive loops run in one launch when every value a point consumes
// is either (a) read from memory that no loop of the launch writes at another point,
// or (b) produced earlier in the launch by the same thread — at the point itself
// (forwarded in registers) or, for reads at row (B = dim ndim-2) offsets, by
// re-evaluating the unique earlier writer's expression on the shifted row from inputs
// no loop of the launch rewrites ("row recompute"). The matching WAR rule: no loop
// overwrites what an earlier loop reads at a neighbour, directly or through a
// recomputation. Reducing loops always run alone.
namespace {

// Row recompute trades DRAM bytes for re-evaluated expressions. The register-staged
// kernel template spills on such groups (8-loop miniflow2d group: 226-255 regs); the
// shared-memory/TMA template runs them at 44-128 regs, and the autotuner picks
// whichever is faster. Default on; OOC_ROW_RECOMPUTE=0 disables.
int g_row_recompute = -1;  // -1: from the environment
bool row_recompute_enabled() {
  if (g_row_recompute < 0) {
    const char* e = std::getenv("OOC_ROW_RECOMPUTE");
    g_row_recompute = !(e && std::atoi(e) == 0);
  }
  return g_row_recompute != 0;
}

bool row_only(const Stencil& st, int ndim) {
  const int b = ndim - 2;
  if (b < 0 || !row_recompute_enabled()) return false;
  for (const Point& o : st.offsets)
    for (int d = 0; d < 3; ++d)
      if (d != b && o[d] != 0) return false;
  return true;
}

bool writes_dataset(const ParLoop& l, DatasetId d) {
  for (const LoopArg& a : l.args)
    if (a.dataset == d && access_writes(a.mode)) return true;
  return false;
}

// Datasets the recomputation of dataset d before position `pos` reads from memory;
// false when it cannot be recomputed (several writers, non-row offsets, or an input
// that some loop from the writer on rewrites).
bool recompute_inputs(const std::vector<const ParLoop*>& all, DatasetId d, std::size_t pos,
                      std::vector<DatasetId>& inputs, int depth = 0) {
  if (depth > 8) return false;
  std::size_t x = all.size();
  int nw = 0;
  for (std::size_t k = 0; k < pos; ++k)
    if (writes_dataset(*all[k], d)) {
      x = k;
      ++nw;
    }
  if (nw != 1) return false;
  const ParLoop& w = *all[x];
  for (const LoopArg& a : w.args) {
    if (!access_reads(a.mode)) continue;
    bool earlier = false;
    for (std::size_t k = 0; k < x; ++k) earlier = earlier || writes_dataset(*all[k], a.dataset);
    if (earlier) {
      if (!a.stencil.is_point() && !row_only(a.stencil, w.range.ndim)) return false;
      if (!recompute_inputs(all, a.dataset, x, inputs, depth + 1)) return false;
      continue;
    }
    for (std::size_t k = x; k < all.size(); ++k)
      if (writes_dataset(*all[k], a.dataset)) return false;
    inputs.push_back(a.dataset);
  }
  return true;
}

}  // namespace

void set_row_recompute(bool on) { g_row_recompute = on ? 1 : 0; }

bool can_fuse(const std::vector<const ParLoop*>& group, std::size_t group_tape, const ParLoop& b,
              bool enabled) {
  if (group.empty()) return true;
  if (!enabled || b.has_reduction() || group.size() >= 8) return false;
  std::size_t tape = group_tape;
  for (const auto& t : b.write_tapes) tape += t.ins.size();
  if (tape > 200) return false;
  std::vector<const ParLoop*> all(group);
  all.push_back(&b);
  for (const ParLoop* a : group) {
    if (a->has_reduction() || a->range.ndim != b.range.ndim) return false;
    for (const LoopArg& x : a->args)
      for (const LoopArg& y : b.args) {
        if (x.dataset != y.dataset) continue;
        if (access_reads(x.mode) && access_writes(y.mode) && !x.stencil.is_point()) return false;
      }
  }
  // b's neighbour reads of values written in the launch: row recompute only
  for (const LoopArg& y : b.args) {
    if (!access_reads(y.mode) || y.stencil.is_point()) continue;
    bool written = false;
    for (const ParLoop* a : group) written = written || writes_dataset(*a, y.dataset);
    if (!written) continue;
    if (!row_only(y.stencil, b.range.ndim) || writes_dataset(b, y.dataset)) return false;
    std::vector<DatasetId> in;
    if (!recompute_inputs(all, y.dataset, group.size(), in)) return false;
  }
  // b must not overwrite an input of a recomputation an earlier loop relies on
  for (std::size_t j = 0; j < group.size(); ++j)
    for (const LoopArg& y : group[j]->args) {
      if (!access_reads(y.mode) || y.stencil.is_point()) continue;
      bool written = false;
      for (std::size_t k = 0; k < j; ++k) written = written || writes_dataset(*group[k], y.dataset);
      if (!written) continue;
      std::vector<DatasetId> in;
      if (!recompute_inputs(all, y.dataset, j, in)) return false;
    }
  return true;
}

std::vector<char> plan_fusion(const Mesh& mesh, const std::vector<ParLoop>& loops,
                              const std::vector<std::size_t>& tape_len, bool enabled) {
  const std::size_t L = loops.size();
  std::vector<char> starts(L, 1);
  if (!enabled || L < 2) return starts;
  // longest legal group from each start (exactly the engine's incremental check)
  std::vector<std::size_t> maxj(L);
  for (std::size_t i = 0; i < L; ++i) {
    std::vector<const ParLoop*> g{&loops[i]};
    std::size_t tape = tape_len[i], j = i + 1;
    if (!loops[i].has_reduction())
      for (; j < L && can_fuse(g, tape, loops[j], true); ++j) {
        g.push_back(&loops[j]);
        tape += tape_len[j];
      }
    maxj[i] = j;
  }
  // estimated DRAM bytes of a group: each dataset read once if its first access in
  // the group reads it, written once if any loop writes it; plus a launch cost
  constexpr double kLaunchBytes = 24e6;  // ~4 us of HBM time per extra launch
  auto cost = [&](std::size_t i, std::size_t j) {
    std::map<DatasetId, std::pair<int, index_t>> m;  // dataset -> (reads+writes, points)
    std::map<DatasetId, bool> seen, wrote;
    for (std::size_t k = i; k < j; ++k)
      for (const LoopArg& a : loops[k].args) {
        auto& e = m[a.dataset];
        if (!seen[a.dataset]) {
          seen[a.dataset] = true;
          e.first += access_reads(a.mode) ? 1 : 0;
        }
        if (access_writes(a.mode) && !wrote[a.dataset]) {
          wrote[a.dataset] = true;
          e.first += 1;
        }
        e.second = std::max(e.second, loops[k].range.size());
      }
    double b = kLaunchBytes;
    for (const auto& [d, e] : m) b += static_cast<double>(e.first) * e.second * mesh[d].elem_bytes;
    return b;
  };
  std::vector<double> best(L + 1, 1e300);
  std::vector<std::size_t> from(L + 1, 0);
  best[0] = 0;
  for (std::size_t j = 1; j <= L; ++j)
    for (std::size_t i = j; i-- > 0;) {
      if (j - i > 8) break;
      if (maxj[i] < j) continue;
      const double c = best[i] + cost(i, j);
      if (c < best[j]) {
        best[j] = c;
        from[j] = i;
      }
    }
  std::fill(starts.begin(), starts.end(), 0);
  for (std::size_t j = L; j > 0; j = from[j]) starts[from[j]] = 1;
  return starts;
}

bool GpuEngine::fusable(const ParLoop& b) const {
  return can_fuse(group_.loops, group_.tape_len, b, opts_.fuse);
}

void GpuEngine::issue_instrumented(int queue, const std::vector<const ParLoop*>& loops,
                                   const std::vector<index_t>& bytes, const std::function<void()>& issue) {
  if (opts_.timeline) {
    std::vector<std::pair<int, index_t>> ls;
    index_t total = 0;
    for (std::size_t i = 0; i < loops.size(); ++i) {
      ls.push_back({loops[i]->id, bytes[i]});
      total += bytes[i];
    }
    timeline_cmd(3, queue, total, -1, cur_tile_, std::move(ls), issue);
  } else if (opts_.profile_loops) {
    PendingLoop pl{{}, 0, fresh_timing_event(), fresh_timing_event()};
    double total = 0;
    for (index_t b : bytes) total += static_cast<double>(b);
    for (std::size_t i = 0; i < loops.size(); ++i)
      pl.weights.push_back({loops[i]->id, total > 0 ? bytes[i] / total : 1.0});
    pl.bytes = static_cast<index_t>(total);
    DEV(ooc_event_record(ctx_, pl.a, queue));
    issue();
    DEV(ooc_event_record(ctx_, pl.b, queue));
    pending_loops_.push_back(std::move(pl));
  } else {
    issue();
  }
}

void GpuEngine::flush_group(int queue) {
  if (group_.calls.empty()) return;
  issue_instrumented(queue, group_.loops, group_.bytes, [&] {
    DEV(ooc_launch_group(ctx_, queue, group_.calls.data(), static_cast<int>(group_.calls.size())));
  });
  group_ = Group{};
}

ooc_loop make_call(const LoweredLoop& lw, const Extent& sub, const std::vector<ooc_view>& views, int red_slot) {
  ooc_loop L{};
  L.ndim = sub.ndim;
  for (int d = 0; d < 3; ++d) {
    L.lo[d] = sub.lo[d];
    L.hi[d] = sub.hi[d];
  }
  L.nargs = static_cast<int32_t>(views.size());
  for (std::size_t a = 0; a < views.size(); ++a) L.args[a] = views[a];
  L.nwrites = static_cast<int32_t>(lw.write_arg.size());
  for (std::size_t w = 0; w < lw.write_arg.size(); ++w) {
    L.write_arg[w] = lw.write_arg[w];
    L.write_len[w] = lw.write_len[w];
  }
  L.reduce_op = lw.reduce_op;
  L.reduce_len = lw.reduce_len;
  L.reduce_slot = red_slot;
  L.ntape = static_cast<int32_t>(lw.tape.size());
  L.tape = lw.tape.data();
  return L;
}

namespace {
// Dead after [a, b): the first access of d after the run is a write (not a read) whose
// range covers every point the run writes.
bool dead_after(const std::vector<ParLoop>& loops, std::size_t a, std::size_t b, DatasetId d) {
  Extent u;
  bool any = false;
  for (std::size_t k = a; k < b; ++k)
    for (const LoopArg& x : loops[k].args)
      if (x.dataset == d && access_writes(x.mode)) {
        const Extent& r = loops[k].range;
        if (!any) {
          u = r;
        } else {
          for (int q = 0; q < 3; ++q) {
            u.lo[q] = std::min(u.lo[q], r.lo[q]);
            u.hi[q] = std::max(u.hi[q], r.hi[q]);
          }
        }
        any = true;
      }
  if (!any) return false;
  for (std::size_t k = b; k < loops.size(); ++k) {
    bool rd = false, wr = false;
    for (const LoopArg& x : loops[k].args)
      if (x.dataset == d) {
        rd = rd || access_reads(x.mode);
        wr = wr || access_writes(x.mode);
      }
    if (rd) return false;
    if (wr) return loops[k].range.contains(u);
  }
  return false;  // live at the end of the chain
}
}  // namespace

std::vector<SweepRun> plan_sweeps(const Mesh& mesh, const std::vector<ParLoop>& loops, bool exact_reductions,
                                  const std::vector<ooc_loop>& calls) {
  // Least-traffic partition (dynamic programming) of the chain into sweep runs and
  // single loops left to the other kernels. A run costs one read of every dataset it
  // loads plus one write of every dataset it writes that is still live after it; a
  // launch costs ~4 us of HBM time.
  const std::size_t L = calls.size();
  constexpr double kLaunchBytes = 24e6;
  auto bytes_of = [&](DatasetId d) { return static_cast<double>(mesh[d].alloc().size()) * mesh[d].elem_bytes; };
  std::vector<std::vector<std::pair<std::size_t, double>>> runs(L);  // i -> (j, cost)
  std::vector<int> flags;
  for (std::size_t i = 0; i < L; ++i)
    for (std::size_t j = i + 2; j <= L; ++j) {
      if (exact_reductions && loops[j - 1].has_reduction()) break;  // folded on its own
      flags.assign((j - i) * OOC_MAX_ARGS, 0);
      if (ooc_sweep_check(&calls[i], static_cast<int>(j - i), flags.data()) != 1) {
        if (j > i + 2 || ooc_sweep_check(&calls[i], 1, nullptr) != 1) break;
        continue;
      }
      std::map<DatasetId, int> f;
      for (std::size_t k = i; k < j; ++k)
        for (std::size_t x = 0; x < loops[k].args.size(); ++x)
          f[loops[k].args[x].dataset] |= flags[(k - i) * OOC_MAX_ARGS + x];
      double c = kLaunchBytes;
      for (const auto& [d, fl] : f) {
        if (fl & 2) c += bytes_of(d);
        if ((fl & 4) && !dead_after(loops, i, j, d)) c += bytes_of(d);
      }
      runs[i].push_back({j, c});
    }
  std::vector<double> best(L + 1, 1e300);
  std::vector<std::size_t> from(L + 1, 0);
  best[0] = 0;
  for (std::size_t i = 0; i < L; ++i) {
    if (best[i] >= 1e299) continue;
    double single = kLaunchBytes;  // the loop launched on its own
    for (const LoopArg& x : loops[i].args)
      single += bytes_of(x.dataset) * (x.mode == AccessMode::read_write ? 2 : 1);
    if (best[i] + single < best[i + 1]) {
      best[i + 1] = best[i] + single;
      from[i + 1] = i;
    }
    for (const auto& [j, c] : runs[i])
      if (best[i] + c < best[j]) {
        best[j] = best[i] + c;
        from[j] = i;
      }
  }
  std::vector<SweepRun> out;
  for (std::size_t j = L; j > 0; j = from[j]) {
    const std::size_t i = from[j];
    if (j - i >= 2) {
      SweepRun r{i, j, {}};
      std::vector<DatasetId> seen;
      for (std::size_t k = i; k < j; ++k)
        for (const LoopArg& x : loops[k].args)
          if (access_writes(x.mode) && std::find(seen.begin(), seen.end(), x.dataset) == seen.end()) {
            seen.push_back(x.dataset);
            if (dead_after(loops, i, j, x.dataset)) r.dead.push_back(x.dataset);
          }
      out.push_back(r);
    }
  }
  std::reverse(out.begin(), out.end());
  return out;
}

namespace {
int g_sweep = -1;  // -1: from the environment (OOC_SWEEP=0 disables)
}
bool sweep_enabled() {
  if (g_sweep < 0) {
    const char* e = std::getenv("OOC_SWEEP");
    g_sweep = !(e && std::atoi(e) == 0);
  }
  return g_sweep != 0;
}
void set_sweep(bool on) { g_sweep = on ? 1 : 0; }

void GpuEngine::launch(int queue, bool group_start, int tile, const ParLoop& loop,
                       const LoweredLoop& lw, const Extent& sub,
                       const std::vector<ooc_view>& views, int red_slot) {
  if (group_start || !fusable(loop)) flush_group(queue);
  cur_tile_ = tile;
  group_.calls.push_back(make_call(lw, sub, views, red_slot));
  group_.loops.push_back(&loop);
  group_.bytes.push_back(sub.size() * loop_bytes_per_point_views(loop));
  group_.tape_len += lw.tape.size();
  if (loop.has_reduction()) flush_group(queue);
}

index_t GpuEngine::loop_bytes_per_point_views(const ParLoop& loop) const {
  index_t n = 0;
  for (const LoopArg& a : loop.args) n += 8 * (a.mode == AccessMode::read_write ? 2 : 1);
  return n;
}

void GpuEngine::ensure_pool(index_t elems) {
  if (elems <= pool_elems_) return;
  if (pool_) {
    DEV(ooc_ctx_sync(ctx_));  // earlier chains may still read the old pool
    DEV(ooc_mem_free(ctx_, pool_));
    pool_ = nullptr;
  }
  void* p = nullptr;
  DEV(ooc_mem_alloc(ctx_, static_cast<std::size_t>(elems) * sizeof(double), &p));
  pool_ = static_cast<double*>(p);
  pool_elems_ = elems;
}

void GpuEngine::finish_chain(const LoopChain& chain, const std::map<int, int>& red,
                             PendingChain pc, int end_queue) {
  // reductions: one 8-byte D2H per reducing loop, on the compute queue after its kernels
  if (!red.empty()) {
    for (const auto& [loop_id, slot] : red) {
      DEV(ooc_reduce_fetch(ctx_, OOC_Q_COMPUTE, slot, red_host_ + slot));
      ooc_event*& e = red_ready_[slot];
      if (!e) DEV(ooc_event_create(ctx_, 0, &e));
      DEV(ooc_event_record(ctx_, e, OOC_Q_COMPUTE));
    }
  }
  DEV(ooc_event_record(ctx_, pc.end, end_queue));
  pc.t.chain_id = chain.chain_id;
  pc.t.loops = static_cast<int>(chain.loops.size());
  pending_chains_.push_back(pc);
}

// ---------------------------------------------------------------- streaming executor

void GpuEngine::run_explicit(Mesh& mesh, const LoopChain& chain, const TilePlan& plan,
                             const Footprints& fp, bool cyclic, ChainOut& out,
                             const std::vector<HaloXfer>* halos) {
  const int T = plan.tile_count;
  const int dim = plan.tiled_dim;
  if (3 * fp.slot_bytes > opts_.device.capacity_bytes)  // explicit_exec.cpp:61-62
    throw CapacityError(3 * fp.slot_bytes, opts_.device.capacity_bytes);

  std::vector<DatasetId> used;
  for (std::size_t d = 0; d < fp.per_dataset.size(); ++d)
    if (fp.per_dataset[d].accessed) used.push_back(static_cast<DatasetId>(d));
  auto P = [&](DatasetId d) -> const Footprints::PerDataset& {
    return fp.per_dataset[static_cast<std::size_t>(d)];
  };

  // Slot layout: every dataset gets a region able to hold its largest tile box
  // (per-dim max over tiles of full[t]); rows padded to 128 B.
  std::vector<BoxLayout> lay(mesh.datasets.size());
  std::vector<index_t> off(mesh.datasets.size(), 0);
  index_t slot_elems = 0;
  // Arena boxes span the dataset's full allocation across the non-tiled dimensions: a
  // tile box that stops a column or two short of the allocation (e.g. a dataset read
  // through a row-only stencil) would make every upload a pitched copy; uploading the
  // whole rows instead is one contiguous DMA at full PCIe rate (the extra columns are
  // never read, never downloaded, and not counted: audit and timeline keep the
  // reference's boxes).
  auto widen = [&](DatasetId d, const Extent& e) {
    Extent w = e;
    if (e.empty()) return w;
    const Extent a = mesh[d].alloc();
    for (int k = 0; k < e.ndim; ++k)
      if (k != dim) {
        w.lo[k] = a.lo[k];
        w.hi[k] = a.hi[k];
      }
    return w;
  };
  for (DatasetId d : used) {
    Extent big = Extent::none(mesh[d].core.ndim);
    for (const Extent& f0 : P(d).full)
      if (const Extent f = widen(d, f0); !f.empty()) {
        if (big.empty()) {
          big = f;
        } else {
          for (int k = 0; k < 3; ++k) {
            index_t len = std::max(big.len(k), f.len(k));
            big.lo[k] = 0;
            big.hi[k] = len;
          }
        }
      }
    if (big.empty()) continue;
    // rows padded to 16 B only (TMA stride rule): an arena row then matches the host
    // row whenever the tile box spans the dataset's full inner extent, and the box
    // copies collapse to 1-D DMA (ooc_copy_box)
    lay[static_cast<std::size_t>(d)] = padded_layout(big, 2);
    off[static_cast<std::size_t>(d)] = slot_elems;
    slot_elems += (lay[static_cast<std::size_t>(d)].elems + 31) / 32 * 32;  // 256-B aligned
  }
  ensure_pool(3 * std::max<index_t>(slot_elems, 32));

  const int par = static_cast<int>(chain_count_ & 1);  // this chain's event pools
  auto E = [&](std::vector<ooc_event*>* pools, int t) { return ev(pools[par], static_cast<std::size_t>(t)); };
  auto slot_of = [&](int t) { return (slot_cursor_ + t) % 3; };
  auto arena = [&](DatasetId d, int t) {
    return view_at(pool_ + static_cast<index_t>(slot_of(t)) * slot_elems + off[static_cast<std::size_t>(d)],
                   widen(d, P(d).full[t]), lay[static_cast<std::size_t>(d)].stride);
  };
  std::map<std::pair<DatasetId, int>, AuditRow> audit;
  auto row = [&](DatasetId d, int t) -> AuditRow& {
    AuditRow& r = audit[{d, t}];
    r.dataset = d;
    r.tile = t;
    return r;
  };
  auto copy = [&](int q, int kind, const ooc_view& s, const ooc_view& dv, const Extent& region,
                  DatasetId d, int tile, const Extent* dma = nullptr) {
    int64_t lo[3], hi[3];
    for (int k = 0; k < 3; ++k) {
      lo[k] = dma ? dma->lo[k] : region.lo[k];
      hi[k] = dma ? dma->hi[k] : region.hi[k];
    }
    const int cmd = kind == OOC_COPY_H2D ? 0 : kind == OOC_COPY_D2H ? 1 : 2;  // CmdKind order
    timeline_cmd(cmd, q, region.size() * mesh[d].elem_bytes, d, tile, {},
                 [&] { DEV(ooc_copy_box(ctx_, q, kind, &s, &dv, lo, hi)); });
  };
  auto fill_tile = [&](int t, int q) {
    if (!opts_.arena_fill) return;
    const double v = opts_.arena_fill == 2 ? std::nan("") : 0.0;
    for (DatasetId d : used) {
      if (P(d).full[t].empty()) continue;
      ooc_view a = arena(d, t);
      DEV(ooc_fill_box(ctx_, q, &a, v));
    }
  };
  // A queue about to write slot s waits for the slot's previous users (kernels and
  // edge carry on the compute queue, the download) — possibly of the previous chain.
  auto wait_slot_free = [&](int q, int s) {
    if (slot_q0_[s]) DEV(ooc_queue_wait(ctx_, q, slot_q0_[s]));
    if (slot_d2h_[s]) DEV(ooc_queue_wait(ctx_, q, slot_d2h_[s]));
  };
  // Host read-after-write across chains: an upload of rows `r` of dataset d waits
  // for the previous chain's download of those rows (latest intersecting tile).
  auto wait_host_rows = [&](DatasetId d, const Extent& r) {
    const auto& downs = prev_down_[static_cast<std::size_t>(d)];
    int last = -1;
    for (const auto& [box, t] : downs)
      if (!box.intersect(r).empty()) last = std::max(last, t);
    if (last >= 0) DEV(ooc_queue_wait(ctx_, OOC_Q_H2D, ev(ev_d2h_[1 - par], static_cast<std::size_t>(last))));
  };
  if (prev_down_.size() < mesh.datasets.size()) prev_down_.resize(mesh.datasets.size());

  PendingChain pc;
  pc.start = fresh_timing_event();
  pc.end = fresh_timing_event();
  pc.t.tiles = T;
  DEV(ooc_event_record(ctx_, pc.start, OOC_Q_COMPUTE));
  // chains older than the previous one are fully downloaded before this one uploads
  // (the previous chain is tracked row by row in wait_host_rows)
  if (chain_done_[par]) DEV(ooc_queue_wait(ctx_, OOC_Q_H2D, chain_done_[par]));

  // reduction accumulators (explicit_exec.cpp:159-162)
  for (const ParLoop& l : chain.loops)
    if (l.has_reduction()) {
      int s = alloc_red_slot();
      out.reduction_slot[l.id] = s;
      DEV(ooc_reduce_reset(ctx_, OOC_Q_COMPUTE, s, lower_loop(l).reduce_op));
    }

  std::vector<Extent> down_hull(mesh.datasets.size()), skip_hull(mesh.datasets.size());
  for (DatasetId d : used) {
    down_hull[static_cast<std::size_t>(d)] = Extent::none(mesh[d].alloc().ndim);
    skip_hull[static_cast<std::size_t>(d)] = Extent::none(mesh[d].alloc().ndim);
  }
  std::vector<std::vector<std::pair<Extent, int>>> this_down(mesh.datasets.size());
  // tapes are lowered once per chain; ooc_launch_loop copies them into kernel params
  std::vector<LoweredLoop> lowered_store(chain.loops.size());
  for (std::size_t j = 0; j < chain.loops.size(); ++j) lowered_store[j] = lower_loop(chain.loops[j]);
  std::vector<std::size_t> tape_len(chain.loops.size());
  for (std::size_t j = 0; j < chain.loops.size(); ++j) tape_len[j] = lowered_store[j].tape.size();
  const std::vector<char> starts = plan_fusion(mesh, chain.loops, tape_len, opts_.fuse);
  std::vector<ooc_view> hviews(mesh.datasets.size());
  for (DatasetId d : used) hviews[static_cast<std::size_t>(d)] = host_view(mesh[d]);

  for (int t = 0; t < T; ++t) {
    if (t == 0) {
      wait_slot_free(OOC_Q_H2D, slot_of(0));
      fill_tile(0, OOC_Q_H2D);
      for (DatasetId d : used) {
        const auto& pd = P(d);
        if (pd.write_first || pd.full[0].empty()) continue;
        const Extent& region = pd.full[0];
        const index_t eb = mesh[d].elem_bytes;
        // consume what the previous chain staged speculatively when it only differs
        // along the tiled dimension (explicit_exec.cpp:135-157)
        auto st = staged_.find(d);
        bool splits = false;
        Extent common;
        if (st != staged_.end()) {
          common = region.intersect(st->second.region);
          splits = !common.empty();
          for (int k = 0; k < 3 && splits; ++k)
            if (k != dim && (common.lo[k] != region.lo[k] || common.hi[k] != region.hi[k])) splits = false;
        }
        if (splits) {
          copy(OOC_Q_H2D, OOC_COPY_D2D, st->second.view, arena(d, 0), common, d, 0);
          Extent lo_part = region.with_dim(dim, region.lo[dim], common.lo[dim]);
          Extent hi_part = region.with_dim(dim, common.hi[dim], region.hi[dim]);
          for (const Extent& part : {lo_part, hi_part})
            if (part.lo[dim] < part.hi[dim]) {
              wait_host_rows(d, part);
              const Extent wpart = widen(d, part);
              copy(OOC_Q_H2D, OOC_COPY_H2D, hviews[static_cast<std::size_t>(d)], arena(d, 0), part, d, 0, &wpart);
              row(d, 0).uploaded += part.size() * eb;
            }
        } else {
          wait_host_rows(d, region);
          const Extent wregion = widen(d, region);
          copy(OOC_Q_H2D, OOC_COPY_H2D, hviews[static_cast<std::size_t>(d)], arena(d, 0), region, d, 0, &wregion);
          row(d, 0).uploaded += region.size() * eb;
        }
      }
      staged_.clear();  // anything not consumed is for a chain that never came (:178)
      DEV(ooc_event_record(ctx_, E(ev_h2d_, 0), OOC_Q_H2D));
    }
    if (t + 1 < T) {
      wait_slot_free(OOC_Q_H2D, slot_of(t + 1));
      fill_tile(t + 1, OOC_Q_H2D);
      for (DatasetId d : used) {
        const auto& pd = P(d);
        if (pd.write_first || pd.right_fp[t + 1].empty()) continue;
        wait_host_rows(d, pd.right_fp[t + 1]);
        const Extent wfp = widen(d, pd.right_fp[t + 1]);
        copy(OOC_Q_H2D, OOC_COPY_H2D, hviews[static_cast<std::size_t>(d)], arena(d, t + 1), pd.right_fp[t + 1], d,
             t + 1, &wfp);
        row(d, t + 1).uploaded += pd.right_fp[t + 1].size() * mesh[d].elem_bytes;
      }
      DEV(ooc_event_record(ctx_, E(ev_h2d_, t + 1), OOC_Q_H2D));
    }

    // kernels of tile t wait for tile t's upload (missing from the reference model)
    DEV(ooc_queue_wait(ctx_, OOC_Q_COMPUTE, E(ev_h2d_, t)));
    for (std::size_t j = 0; j < chain.loops.size(); ++j) {
      const ParLoop& loop = chain.loops[j];
      const Extent sub = plan.subrange(static_cast<int>(j), t);
      if (sub.empty()) continue;
      std::vector<ooc_view> views;
      views.reserve(loop.args.size());
      for (const LoopArg& a : loop.args) {
        views.push_back(arena(a.dataset, t));
        if (access_writes(a.mode)) mesh[a.dataset].ever_written = true;
      }
      auto rs = out.reduction_slot.find(loop.id);
      launch(OOC_Q_COMPUTE, starts[j] != 0, t, loop, lowered_store[j], sub, views,
             rs == out.reduction_slot.end() ? 0 : rs->second);
    }
    flush_group(OOC_Q_COMPUTE);
    DEV(ooc_event_record(ctx_, E(ev_k_, t), OOC_Q_COMPUTE));

    if (t + 1 < T) {
      // the edge carry writes slot(t+1): its previous download must be done
      if (slot_d2h_[slot_of(t + 1)]) DEV(ooc_queue_wait(ctx_, OOC_Q_COMPUTE, slot_d2h_[slot_of(t + 1)]));
      for (DatasetId d : used) {
        const auto& pd = P(d);
        if (pd.right_edge[t].empty()) continue;
        copy(OOC_Q_COMPUTE, OOC_COPY_D2D, arena(d, t), arena(d, t + 1), pd.right_edge[t], d, t + 1);
        row(d, t + 1).d2d += pd.right_edge[t].size() * mesh[d].elem_bytes;
      }
    }
    DEV(ooc_event_record(ctx_, E(ev_q0_, t), OOC_Q_COMPUTE));
    slot_q0_[slot_of(t)] = E(ev_q0_, t);

    DEV(ooc_queue_wait(ctx_, OOC_Q_D2H, E(ev_k_, t)));
    for (DatasetId d : used) {
      const auto& pd = P(d);
      if (!pd.written_any) continue;  // read-only data never travels back
      if (cyclic && pd.write_first) {  // cyclic: temporaries are dropped
        skip_hull[static_cast<std::size_t>(d)] = skip_hull[static_cast<std::size_t>(d)].hull(pd.left_fp[t]);
        continue;
      }
      if (!pd.left_fp[t].empty()) {
        copy(OOC_Q_D2H, OOC_COPY_D2H, arena(d, t), hviews[static_cast<std::size_t>(d)], pd.left_fp[t], d, t);
        row(d, t).downloaded += pd.left_fp[t].size() * mesh[d].elem_bytes;
        this_down[static_cast<std::size_t>(d)].push_back({pd.left_fp[t], t});
      }
      down_hull[static_cast<std::size_t>(d)] = down_hull[static_cast<std::size_t>(d)].hull(pd.left_fp[t]);
    }
    DEV(ooc_event_record(ctx_, E(ev_d2h_, t), OOC_Q_D2H));
    slot_d2h_[slot_of(t)] = E(ev_d2h_, t);
  }

  // speculative upload of this chain's first tile for the next chain
  // (explicit_exec.cpp:188-204, 260-271): issued once every download that writes
  // those host rows has landed, into a staging region outside the three slots
  if (opts_.prefetch) {
    index_t need = 0;
    std::vector<std::pair<DatasetId, BoxLayout>> st_lay;
    for (DatasetId d : used) {
      const auto& pd = P(d);
      if (pd.write_first || pd.full[0].empty()) continue;
      st_lay.push_back({d, padded_layout(widen(d, pd.full[0]), 2)});
      need += (st_lay.back().second.elems + 31) / 32 * 32;
    }
    ensure_staging(need);
    index_t at = 0;
    for (const auto& [d, L] : st_lay) {
      const Extent& region = P(d).full[0];
      const Extent wregion = widen(d, region);  // whole rows: one contiguous DMA
      int last = -1;
      for (const auto& [box, t] : this_down[static_cast<std::size_t>(d)])
        if (!box.intersect(wregion).empty()) last = std::max(last, t);
      if (last >= 0) DEV(ooc_queue_wait(ctx_, OOC_Q_H2D, E(ev_d2h_, last)));
      Staged s;
      s.region = region;
      s.view = view_at(staging_ + at, wregion, L.stride);
      at += (L.elems + 31) / 32 * 32;
      copy(OOC_Q_H2D, OOC_COPY_H2D, hviews[static_cast<std::size_t>(d)], s.view, region, d, T, &wregion);
      row(d, T).uploaded += region.size() * mesh[d].elem_bytes;
      staged_[d] = s;
    }
  }

  // host staleness bookkeeping (explicit_exec.cpp:245-258)
  for (DatasetId d : used) {
    Dataset& ds = mesh[d];
    const Extent& sk = skip_hull[static_cast<std::size_t>(d)];
    const Extent& dn = down_hull[static_cast<std::size_t>(d)];
    if (!sk.empty()) {
      ds.stale_region = ds.host_stale ? ds.stale_region.hull(sk) : sk;
      ds.host_stale = true;
      ds.stale_chain = chain.chain_id;
    } else if (ds.host_stale && !dn.empty() && dn.contains(ds.stale_region)) {
      ds.host_stale = false;
      ds.stale_chain = -1;
      ds.stale_region = Extent::none(ds.alloc().ndim);
    }
  }
  slot_cursor_ = (slot_cursor_ + T) % 3;
  for (std::size_t d = 0; d < prev_down_.size(); ++d)
    prev_down_[d] = d < this_down.size() ? std::move(this_down[d]) : std::vector<std::pair<Extent, int>>{};
  // everything of this chain has landed in host memory once this event completes
  ooc_event*& done = chain_done_[par];
  if (!done) DEV(ooc_event_create(ctx_, 0, &done));
  DEV(ooc_event_record(ctx_, done, OOC_Q_D2H));
  ++chain_count_;

  for (auto& [k, r] : audit) {
    out.audit.push_back(r);
    pc.t.uploaded += r.uploaded;
    pc.t.downloaded += r.downloaded;
    pc.t.d2d += r.d2d;
  }
  for (const ParLoop& l : chain.loops) pc.t.metric_bytes += l.range.size() * loop_bytes_per_point(mesh, l);
  // the chain ends when its last download has landed; the compute queue does not
  // wait for it, so the next chain's first tiles overlap this chain's last downloads
  DEV(ooc_queue_wait(ctx_, OOC_Q_D2H, E(ev_q0_, T - 1)));
  if (halos && comm_ready_) {
    // slab decomposition out of core: the neighbours' owned rows land in this rank's host
    // ghost bands (from their host slabs, after their downloads), then the reductions
    // are combined — the next chain uploads the refreshed rows like any others
    exchange_host_bands(mesh, *halos);
    for (const ParLoop& l : chain.loops)
      if (l.has_reduction())
        DEV(ooc_reduce_allreduce(ctx_, OOC_Q_COMPUTE, out.reduction_slot.at(l.id), lower_loop(l).reduce_op));
  }
  finish_chain(chain, out.reduction_slot, pc, OOC_Q_D2H);
}

void GpuEngine::exchange_host_bands(Mesh& mesh, const std::vector<HaloXfer>& halos) {
  DEV(ooc_ctx_sync(ctx_));  // the chain's downloads have landed: owned rows are current
  struct Band {
    DatasetId d;
    index_t r0, r1, off;
  };
  std::vector<Band> send, recv;
  std::vector<ooc_xfer> xs;
  index_t total = 0;
  auto band = [&](DatasetId d, const index_t* rr, std::vector<Band>& into) -> std::pair<index_t, index_t> {
    const Extent a = mesh[d].alloc();
    const index_t plane = a.size() / std::max<index_t>(1, a.hi[0] - a.lo[0]);
    const index_t n = std::max<index_t>(0, rr[1] - rr[0]) * plane;
    into.push_back({d, rr[0], rr[1], total});
    total += n;
    return {into.back().off, n};
  };
  struct Pend {
    int peer;
    index_t so, sn, ro, rn;
  };
  std::vector<Pend> pend;
  for (const HaloXfer& h : halos) {
    const Dataset& ds = mesh[h.dataset];
    if (ds.host_stale) continue;  // cyclic temporaries were never downloaded (same on every rank)
    if (rank_ > 0) {
      auto s = band(h.dataset, h.send_left, send);
      auto r = band(h.dataset, h.recv_left, recv);
      pend.push_back({rank_ - 1, s.first, s.second, r.first, r.second});
    }
    if (rank_ + 1 < world_) {
      auto s = band(h.dataset, h.send_right, send);
      auto r = band(h.dataset, h.recv_right, recv);
      pend.push_back({rank_ + 1, s.first, s.second, r.first, r.second});
    }
    invalidate_staged(h.dataset);  // a speculative first tile may hold the old ghost rows
  }
  if (pend.empty()) return;
  if (total > band_stage_elems_) {
    if (band_stage_) DEV(ooc_mem_free(ctx_, band_stage_));
    void* p = nullptr;
    DEV(ooc_mem_alloc(ctx_, static_cast<std::size_t>(total) * sizeof(double), &p));
    band_stage_ = static_cast<double*>(p);
    band_stage_elems_ = total;
  }
  auto copy = [&](const Band& b, int kind) {
    if (b.r1 <= b.r0) return;
    Dataset& ds = mesh[b.d];
    Extent box = ds.alloc();
    box.lo[0] = b.r0;
    box.hi[0] = b.r1;
    const BoxLayout L = padded_layout(box, 1);
    ooc_view hv = host_view(ds);
    ooc_view dv = view_at(band_stage_ + b.off, box, L.stride);
    if (kind == OOC_COPY_H2D)
      DEV(ooc_copy_box(ctx_, OOC_Q_COMPUTE, kind, &hv, &dv, dv.lo, dv.hi));
    else
      DEV(ooc_copy_box(ctx_, OOC_Q_COMPUTE, kind, &dv, &hv, dv.lo, dv.hi));
  };
  for (const Band& b : send) copy(b, OOC_COPY_H2D);
  for (const Pend& p : pend)
    xs.push_back({p.peer, band_stage_ + p.so, p.sn, band_stage_ + p.ro, p.rn});
  DEV(ooc_comm_exchange(ctx_, OOC_Q_COMPUTE, xs.data(), static_cast<int>(xs.size())));
  for (const Band& b : recv) copy(b, OOC_COPY_D2H);
  DEV(ooc_queue_sync(ctx_, OOC_Q_COMPUTE));
}

// Real event timeline (replaces the reference's simulated one, command.cpp:35-126):
// every command bracketed by timing events on its queue; fused launches are split
// into per-loop sub-intervals in proportion to their metric bytes.
void GpuEngine::timeline_cmd(int kind, int queue, index_t bytes, DatasetId d, int tile,
                             std::vector<std::pair<int, index_t>> loops,
                             const std::function<void()>& issue) {
  if (!opts_.timeline) {
    issue();
    return;
  }
  if (!tl_base_) {
    DEV(ooc_event_create(ctx_, 1, &tl_base_));
    DEV(ooc_event_record(ctx_, tl_base_, OOC_Q_COMPUTE));
    tl_host0_ = std::chrono::steady_clock::now();
  }
  TLPending p{kind, queue, bytes, d, tile, std::move(loops), 0.0, fresh_timing_event(),
              fresh_timing_event()};
  p.issue = std::chrono::duration<double>(std::chrono::steady_clock::now() - tl_host0_).count();
  DEV(ooc_event_record(ctx_, p.a, queue));
  issue();
  DEV(ooc_event_record(ctx_, p.b, queue));
  tl_pending_.push_back(std::move(p));
}

std::vector<TimelineRow> GpuEngine::take_timeline() {
  std::vector<TimelineRow> out;
  for (TLPending& p : tl_pending_) {
    DEV(ooc_event_sync(ctx_, p.b));
    float a = 0.f, b = 0.f;
    DEV(ooc_event_elapsed_ms(tl_base_, p.a, &a));
    DEV(ooc_event_elapsed_ms(tl_base_, p.b, &b));
    const double s = a * 1e-3, e = b * 1e-3;
    if (p.loops.empty()) {
      out.push_back({next_cmd_++, p.kind, p.queue, p.bytes, p.issue, s, e, p.dataset, p.tile, -1});
    } else {
      double t = s;
      for (const auto& [loop, lb] : p.loops) {
        const double span = p.bytes > 0 ? (e - s) * static_cast<double>(lb) / p.bytes
                                        : (e - s) / p.loops.size();
        out.push_back({next_cmd_++, p.kind, p.queue, lb, p.issue, t, t + span, -1, p.tile, loop});
        t += span;
      }
    }
    recycle(p.a);
    recycle(p.b);
  }
  tl_pending_.clear();
  return out;
}

void GpuEngine::ensure_staging(index_t elems) {
  if (elems <= staging_elems_) return;
  if (staging_) {
    DEV(ooc_ctx_sync(ctx_));
    DEV(ooc_mem_free(ctx_, staging_));
    staging_ = nullptr;
  }
  void* p = nullptr;
  DEV(ooc_mem_alloc(ctx_, static_cast<std::size_t>(elems) * sizeof(double), &p));
  staging_ = static_cast<double*>(p);
  staging_elems_ = elems;
}

void GpuEngine::invalidate_staged(DatasetId d) { staged_.erase(d); }

// ---------------------------------------------------------------- resident executor

void GpuEngine::ensure_resident(Mesh& mesh, DatasetId d) {
  if (res_.size() < mesh.datasets.size()) res_.resize(mesh.datasets.size());
  Resident& r = res_[static_cast<std::size_t>(d)];
  Dataset& ds = mesh[d];
  if (r.dev && r.host_ptr != ds.host.data()) {  // mesh replaced underneath us
    DEV(ooc_ctx_sync(ctx_));
    DEV(ooc_mem_free(ctx_, r.dev));
    if (r.shadow) DEV(ooc_mem_free(ctx_, r.shadow));
    r = Resident{};
  }
  if (!r.dev) {
    r.layout = padded_layout(ds.alloc());
    void* p = nullptr;
    int rc = ooc_mem_alloc(ctx_, static_cast<std::size_t>(r.layout.elems) * sizeof(double), &p);
    if (rc == OOC_ERR_CAPACITY) {
      long long in_use = 0;
      ooc_mem_usage(ctx_, &in_use, nullptr);
      throw CapacityError(in_use + r.layout.elems * 8, props_.hbm_bytes);
    }
    DEV(rc);
    r.dev = static_cast<double*>(p);
    r.host_ptr = ds.host.data();
  }
  if (!r.dev_valid) {
    ooc_view hv = host_view(ds);
    ooc_view dv = view_at(r.dev, ds.alloc(), r.layout.stride);
    timeline_cmd(0, OOC_Q_COMPUTE, ds.alloc().size() * ds.elem_bytes, d, 0, {}, [&] {
      DEV(ooc_copy_box(ctx_, OOC_Q_COMPUTE, OOC_COPY_H2D, &hv, &dv, hv.lo, hv.hi));
    });
    r.dev_valid = true;
    r.host_outdated = false;
  }
}

bool GpuEngine::host_outdated(DatasetId d) const {
  return static_cast<std::size_t>(d) < res_.size() && res_[static_cast<std::size_t>(d)].host_outdated;
}

void GpuEngine::download_resident(Mesh& mesh, DatasetId d) {
  if (!host_outdated(d)) return;
  Resident& r = res_[static_cast<std::size_t>(d)];
  Dataset& ds = mesh[d];
  ooc_view hv = host_view(ds);
  ooc_view dv = view_at(r.dev, ds.alloc(), r.layout.stride);
  DEV(ooc_copy_box(ctx_, OOC_Q_COMPUTE, OOC_COPY_D2H, &dv, &hv, hv.lo, hv.hi));
  DEV(ooc_queue_sync(ctx_, OOC_Q_COMPUTE));
  r.host_outdated = false;
}

void GpuEngine::forget_resident(DatasetId d) {
  if (static_cast<std::size_t>(d) < res_.size()) res_[static_cast<std::size_t>(d)].dev_valid = false;
}

void GpuEngine::run_resident(Mesh& mesh, const LoopChain& chain, const TilePlan* plan,
                             const Footprints* fp, ChainOut& out,
                             const std::vector<HaloXfer>* halos) {
  (void)fp;
  PendingChain pc;
  pc.start = fresh_timing_event();
  pc.end = fresh_timing_event();
  pc.t.tiles = plan ? plan->tile_count : 1;
  std::vector<char> used(mesh.datasets.size(), 0);
  for (const ParLoop& l : chain.loops)
    for (const LoopArg& a : l.args) used[static_cast<std::size_t>(a.dataset)] = 1;
  // first touch of a dataset uploads it (in order on the compute queue, before the
  // chain's start event, so uploads are not part of the chain's device time)
  index_t up = 0;
  for (std::size_t d = 0; d < used.size(); ++d)
    if (used[d]) {
      bool had = d < res_.size() && res_[d].dev_valid;
      ensure_resident(mesh, static_cast<DatasetId>(d));
      if (!had) up += mesh[static_cast<DatasetId>(d)].alloc().size() * mesh[static_cast<DatasetId>(d)].elem_bytes;
    }
  pc.t.uploaded = up;
  DEV(ooc_event_record(ctx_, pc.start, OOC_Q_COMPUTE));
  // A chain whose launches repeat exactly (same loops, constants, plan, buffers and
  // reduction slots — e.g. every steady-state chain of an app) is captured into a CUDA
  // graph on its third sighting, once tile-shape tuning has settled, and replayed with
  // one launch from then on: the host cost of thousands of small launches (L2-tiled
  // chains) disappears.
  static const bool graphs_on = [] {
    const char* e = std::getenv("OOC_GRAPHS");
    return !(e && std::atoi(e) == 0);
  }();
  const bool graphs_ok = graphs_on && !(halos && comm_ready_) && !opts_.profile_loops && !opts_.timeline &&
                        !opts_.exact_reductions;  // the contribution buffer grows outside captures
  GraphEntry* ge = nullptr;
  int par = 0, sseen = 0;
  if (graphs_ok) {
    // sightings count per chain structure; graphs are kept per buffer state (sweeps that
    // swap an odd number of times make consecutive chains alternate between two states)
    sseen = ++struct_seen_[graph_key(chain, plan, false)];
    ge = &graphs_[graph_key(chain, plan)];
    ++ge->seen;
    par = ge->flip;
    ge->flip ^= 1;
    if (ge->slots[par].empty()) {
      int need = 0;
      for (const ParLoop& l : chain.loops) need += l.has_reduction() ? 1 : 0;
      if (next_graph_slot_ + need > OOC_REDUCE_SLOTS) {
        ge = nullptr;  // slot range exhausted: this structure runs without graphs
      } else {
        for (int r = 0; r < need; ++r) ge->slots[par].push_back(next_graph_slot_++);
        if (need == 0) ge->slots[par].push_back(-1);  // mark as assigned
      }
    }
  }
  {
    std::size_t r = 0;
    for (const ParLoop& l : chain.loops)
      if (l.has_reduction()) {
        if (ge) {
          const int s = ge->slots[par][r++];
          auto it = red_ready_.find(s);  // the chain two back used it: its value has landed?
          if (it != red_ready_.end()) DEV(ooc_event_sync(ctx_, it->second));
          out.reduction_slot[l.id] = s;
        } else {
          out.reduction_slot[l.id] = alloc_red_slot();
        }
      }
  }
  auto mark_written = [&] {
    for (const ParLoop& l : chain.loops)
      for (const LoopArg& a : l.args)
        if (access_writes(a.mode)) {
          mesh[a.dataset].ever_written = true;
          res_[static_cast<std::size_t>(a.dataset)].host_outdated = true;
        }
  };
  if (ge && ge->g[par]) {
    DEV(ooc_graph_launch(ctx_, OOC_Q_COMPUTE, ge->g[par]));
    mark_written();
    for (DatasetId d : ge->flips) {  // the buffers the captured sweeps swapped
      Resident& r = res_[static_cast<std::size_t>(d)];
      std::swap(r.dev, r.shadow);
    }
    for (const ParLoop& l : chain.loops) pc.t.metric_bytes += l.range.size() * loop_bytes_per_point(mesh, l);
    finish_chain(chain, out.reduction_slot, pc);
    return;
  }
  // capture on the third sighting (tuning-complete chains from the second); shapes
  // still being tuned are frozen at the fastest measured
  const bool capture = ge && (ge->settled || sseen >= 3);
  static const bool gdbg = std::getenv("OOC_GRAPH_DEBUG") != nullptr;
  if (gdbg)
    std::fprintf(stderr, "graph: chain %d loops %zu ok %d entry %d seen %d par %d settled %d graphs %zu\n",
                 chain.chain_id, chain.loops.size(), graphs_ok ? 1 : 0, ge ? 1 : 0, ge ? ge->seen : -1, par,
                 ge && ge->settled ? 1 : 0, graphs_.size());
  long long unsettled0 = 0;
  if (ge && !capture) {
    ooc_dev_stats st{};
    DEV(ooc_stats(ctx_, &st));
    unsettled0 = st.jit_unsettled;
  }
  if (capture) {
    ooc_jit_freeze(1);
    DEV(ooc_graph_begin(ctx_, OOC_Q_COMPUTE));
  }
  for (const ParLoop& l : chain.loops)
    if (l.has_reduction())
      DEV(ooc_reduce_reset(ctx_, OOC_Q_COMPUTE, out.reduction_slot.at(l.id), lower_loop(l).reduce_op));
  std::vector<LoweredLoop> lowered_store(chain.loops.size());
  for (std::size_t j = 0; j < chain.loops.size(); ++j) {
    lowered_store[j] = lower_loop(chain.loops[j]);
    for (const LoopArg& a : chain.loops[j].args)
      if (access_writes(a.mode)) {
        mesh[a.dataset].ever_written = true;
        res_[static_cast<std::size_t>(a.dataset)].host_outdated = true;
      }
  }
  // views are taken at launch time: a sweep launch swaps the buffers of the datasets it
  // rewrites out of place
  auto views_of = [&](const ParLoop& l) {
    std::vector<ooc_view> v;
    for (const LoopArg& a : l.args) {
      const Resident& r = res_[static_cast<std::size_t>(a.dataset)];
      v.push_back(view_at(r.dev, mesh[a.dataset].alloc(), r.layout.stride));
    }
    return v;
  };
  std::vector<std::size_t> tape_len(chain.loops.size());
  for (std::size_t j = 0; j < chain.loops.size(); ++j) tape_len[j] = lowered_store[j].tape.size();
  const std::vector<char> starts = plan_fusion(mesh, chain.loops, tape_len, opts_.fuse);
  const int T = plan ? plan->tile_count : 1;
  // untiled chains: runs of loops the row-sweep kernel accepts stream through shared
  // memory in one launch each (csrc/device/sweep.cu)
  static std::map<std::string, std::vector<SweepRun>> sweep_cache;  // per chain structure
  const std::vector<SweepRun>* sweeps = nullptr;
  static const std::vector<SweepRun> no_sweeps;
  if (T == 1 && opts_.fuse && sweep_enabled()) {
    // the partition depends on the specialisation policy too (size threshold, OOC_JIT)
    int jm = 1;
    long long jmin = 0;
    ooc_jit_policy(&jm, &jmin);
    const std::string key = sweep_key(mesh, chain) + "|" + std::to_string(jm) + "|" + std::to_string(jmin) + "|" +
                            std::to_string(ooc_sweep_3d_enabled()) + "|" +
                            std::to_string(opts_.exact_reductions ? 1 : 0);
    auto it = sweep_cache.find(key);
    if (it == sweep_cache.end()) {
      std::vector<ooc_loop> calls;
      for (std::size_t j = 0; j < chain.loops.size(); ++j)
        calls.push_back(make_call(lowered_store[j], chain.loops[j].range, views_of(chain.loops[j]), 0));
      it = sweep_cache.emplace(key, plan_sweeps(mesh, chain.loops, opts_.exact_reductions, calls)).first;
    }
    sweeps = &it->second;
  } else {
    sweeps = &no_sweeps;
  }
  std::vector<DatasetId> flipped;
  std::size_t next_sweep = 0;
  for (int t = 0; t < T; ++t)
    for (std::size_t j = 0; j < chain.loops.size(); ++j) {
      if (next_sweep < sweeps->size() && (*sweeps)[next_sweep].a == j) {
        const SweepRun& run = (*sweeps)[next_sweep];
        const std::size_t b = run.b;
        ++next_sweep;
        flush_group(OOC_Q_COMPUTE);
        if (run_sweep(mesh, chain, run, lowered_store, flipped, out.reduction_slot)) {
          j = b - 1;
          continue;
        }
        // no HBM left for a shadow buffer: this run's loops go through the fused launches
      }
      const ParLoop& l = chain.loops[j];
      const Extent sub = plan ? plan->subrange(static_cast<int>(j), t) : l.range;
      if (sub.empty()) continue;
      auto rs = out.reduction_slot.find(l.id);
      const bool after_sweep = next_sweep > 0 && (*sweeps)[next_sweep - 1].b == j;
      launch(OOC_Q_COMPUTE, starts[j] != 0 || after_sweep, t, l, lowered_store[j], sub, views_of(l),
             rs == out.reduction_slot.end() ? 0 : rs->second);
    }
  flush_group(OOC_Q_COMPUTE);
  if (capture) {
    ooc_jit_freeze(0);
    DEV(ooc_graph_end(ctx_, OOC_Q_COMPUTE, -1, &ge->g[par]));
    ge->flips = flipped;
    DEV(ooc_graph_launch(ctx_, OOC_Q_COMPUTE, ge->g[par]));
  } else if (ge) {
    ooc_dev_stats st{};
    DEV(ooc_stats(ctx_, &st));
    ge->settled = sseen >= 2 && st.jit_unsettled == unsettled0;
  }
  if (halos && comm_ready_) {
    // slab decomposition: refresh every ghost band from the neighbours' owned rows,
    // then combine the ranks' reductions — both stream-ordered after the kernels
    std::vector<ooc_xfer> xs;
    for (const HaloXfer& h : *halos) {
      const Resident& r = res_[static_cast<std::size_t>(h.dataset)];
      const Extent a = mesh[h.dataset].alloc();
      const index_t row = r.layout.stride[0];
      auto at = [&](index_t r0) { return r.dev + (r0 - a.lo[0]) * row; };
      if (rank_ > 0)
        xs.push_back({rank_ - 1, at(h.send_left[0]), (h.send_left[1] - h.send_left[0]) * row,
                      at(h.recv_left[0]), (h.recv_left[1] - h.recv_left[0]) * row});
      if (rank_ + 1 < world_)
        xs.push_back({rank_ + 1, at(h.send_right[0]), (h.send_right[1] - h.send_right[0]) * row,
                      at(h.recv_right[0]), (h.recv_right[1] - h.recv_right[0]) * row});
    }
    if (!xs.empty()) DEV(ooc_comm_exchange(ctx_, OOC_Q_COMPUTE, xs.data(), static_cast<int>(xs.size())));
    for (const ParLoop& l : chain.loops)
      if (l.has_reduction())
        DEV(ooc_reduce_allreduce(ctx_, OOC_Q_COMPUTE, out.reduction_slot.at(l.id),
                                 lower_loop(l).reduce_op));
  }
  for (const ParLoop& l : chain.loops) pc.t.metric_bytes += l.range.size() * loop_bytes_per_point(mesh, l);
  finish_chain(chain, out.reduction_slot, pc);
}

std::string sweep_key(const Mesh& mesh, const LoopChain& chain) {
  // everything the sweep partition depends on: ranges, datasets (+ allocations),
  // access modes, tape structure (opcodes, arguments, offsets; not constant values)
  std::string k;
  auto put_i = [&](long long v) { k.append(reinterpret_cast<const char*>(&v), sizeof v); };
  for (const ParLoop& l : chain.loops) {
    put_i(l.range.ndim);
    for (int d = 0; d < 3; ++d) {
      put_i(l.range.lo[d]);
      put_i(l.range.hi[d]);
    }
    put_i(l.has_reduction() ? 1 : 0);
    for (const LoopArg& a : l.args) {
      put_i(a.dataset);
      put_i(static_cast<long long>(a.mode));
      const Extent al = mesh[a.dataset].alloc();
      for (int d = 0; d < 3; ++d) {
        put_i(al.lo[d]);
        put_i(al.hi[d]);
      }
    }
    const LoweredLoop lw = lower_loop(l);
    for (const ooc_ins& in : lw.tape) {
      put_i(in.op);
      put_i(in.arg);
      for (int d = 0; d < 3; ++d) put_i(in.offset[d]);
    }
    for (int w : lw.write_len) put_i(w);
  }
  return k;
}

bool GpuEngine::run_sweep(Mesh& mesh, const LoopChain& chain, const SweepRun& run,
                          const std::vector<LoweredLoop>& lowered, std::vector<DatasetId>& flipped,
                          const std::map<int, int>& red_slots) {
  std::vector<ooc_loop> calls;
  std::vector<const ParLoop*> loops;
  std::vector<index_t> bytes;
  for (std::size_t j = run.a; j < run.b; ++j) {
    const ParLoop& l = chain.loops[j];
    std::vector<ooc_view> v;
    for (const LoopArg& x : l.args) {
      const Resident& r = res_[static_cast<std::size_t>(x.dataset)];
      v.push_back(view_at(r.dev, mesh[x.dataset].alloc(), r.layout.stride));
    }
    auto rs = red_slots.find(l.id);
    calls.push_back(make_call(lowered[j], l.range, v, rs == red_slots.end() ? 0 : rs->second));
    loops.push_back(&l);
    bytes.push_back(l.range.size() * loop_bytes_per_point_views(l));
  }
  std::vector<int> flags(calls.size() * OOC_MAX_ARGS, 0);
  if (ooc_sweep_check(calls.data(), static_cast<int>(calls.size()), flags.data()) != 1)
    throw DeviceError(OOC_ERR_UNSUPPORTED, "sweep group no longer sweepable");
  std::vector<DatasetId> outs;  // live out-of-place outputs: written to the shadow, then swapped
  for (std::size_t i = 0; i < calls.size(); ++i)
    for (std::size_t x = 0; x < loops[i]->args.size(); ++x) {
      const DatasetId d = loops[i]->args[x].dataset;
      if ((flags[i * OOC_MAX_ARGS + x] & 1) && std::find(outs.begin(), outs.end(), d) == outs.end() &&
          std::find(run.dead.begin(), run.dead.end(), d) == run.dead.end())
        outs.push_back(d);
    }
  std::vector<ooc_redirect> red;
  for (DatasetId d : run.dead) red.push_back({res_[static_cast<std::size_t>(d)].dev, nullptr});
  for (DatasetId d : outs) {
    Resident& r = res_[static_cast<std::size_t>(d)];
    if (!r.shadow) {
      void* p = nullptr;
      int rc = ooc_mem_alloc(ctx_, static_cast<std::size_t>(r.layout.elems) * sizeof(double), &p);
      if (rc == OOC_ERR_CAPACITY) return false;  // caller falls back to the fused launches
      DEV(rc);
      r.shadow = static_cast<double*>(p);
    }
    red.push_back({r.dev, r.shadow});
  }
  int rc = OOC_OK;
  issue_instrumented(OOC_Q_COMPUTE, loops, bytes, [&] {
    rc = ooc_launch_sweep(ctx_, OOC_Q_COMPUTE, calls.data(), static_cast<int>(calls.size()), red.data(),
                          static_cast<int>(red.size()));
  });
  if (rc == OOC_ERR_UNSUPPORTED) {  // e.g. the kernel could not be built: fused launches instead
    static bool warned = false;
    if (!warned) std::fprintf(stderr, "ooc: row sweep unavailable (%s); using fused launches\n", ooc_dev_last_error());
    warned = true;
    // the instrumented span bracketed no launch: drop it, the fused launches record their own
    if (opts_.timeline && !tl_pending_.empty()) {
      recycle(tl_pending_.back().a);
      recycle(tl_pending_.back().b);
      tl_pending_.pop_back();
    } else if (opts_.profile_loops && !pending_loops_.empty()) {
      recycle(pending_loops_.back().a);
      recycle(pending_loops_.back().b);
      pending_loops_.pop_back();
    }
    return false;
  }
  DEV(rc);
  for (DatasetId d : outs) {
    Resident& r = res_[static_cast<std::size_t>(d)];
    std::swap(r.dev, r.shadow);
    auto it = std::find(flipped.begin(), flipped.end(), d);
    if (it == flipped.end()) flipped.push_back(d);
    else flipped.erase(it);
  }
  return true;
}

std::string GpuEngine::graph_key(const LoopChain& chain, const TilePlan* plan, bool pointers) const {
  std::string k;
  auto put = [&](const void* p, std::size_t n) { k.append(static_cast<const char*>(p), n); };
  auto put_i = [&](long long v) { put(&v, sizeof v); };
  put_i(static_cast<long long>(chain.loops.size()));
  put_i(opts_.fuse ? 1 : 0);
  for (const ParLoop& l : chain.loops) {
    put_i(l.range.ndim);
    for (int d = 0; d < 3; ++d) {
      put_i(l.range.lo[d]);
      put_i(l.range.hi[d]);
    }
    for (const LoopArg& a : l.args) {
      put_i(a.dataset);
      put_i(static_cast<long long>(a.mode));
      if (pointers) {
        const double* dev = res_[static_cast<std::size_t>(a.dataset)].dev;
        put(&dev, sizeof dev);
      }
      put_i(static_cast<long long>(a.stencil.offsets.size()));
      for (const Point& o : a.stencil.offsets) put(o.data(), sizeof(index_t) * 3);
    }
    const LoweredLoop lw = lower_loop(l);
    for (const ooc_ins& in : lw.tape) {  // field by field: no struct padding in the key
      put_i(in.op);
      put_i(in.arg);
      put(&in.value, sizeof in.value);
      for (int d = 0; d < 3; ++d) put_i(in.offset[d]);
    }
    put_i(lw.reduce_op);
  }
  if (plan) {  // plans live in the runtime's PlanCache (never evicted): identity suffices
    put(&plan, sizeof plan);
    put_i(plan->tile_count);
  }
  return k;
}

void GpuEngine::comm_init(int rank, int world, const void* id) {
  DEV(ooc_comm_init(ctx_, rank, world, id));
  rank_ = rank;
  world_ = world;
  comm_ready_ = true;
}

void GpuEngine::comm_init_ipc(int rank, int world, const std::string& name) {
  DEV(ooc_comm_init_ipc(ctx_, rank, world, name.c_str()));
  rank_ = rank;
  world_ = world;
  comm_ready_ = true;
}

double GpuEngine::reduction_value(int slot) {
  auto it = red_ready_.find(slot);
  if (it != red_ready_.end()) DEV(ooc_event_sync(ctx_, it->second));
  return red_host_[slot];
}

void GpuEngine::sync() { DEV(ooc_ctx_sync(ctx_)); }

int GpuEngine::mark() {
  ooc_event* tail = nullptr;
  DEV(ooc_event_create(ctx_, 0, &tail));
  DEV(ooc_event_record(ctx_, tail, OOC_Q_D2H));
  DEV(ooc_queue_wait(ctx_, OOC_Q_COMPUTE, tail));
  DEV(ooc_event_destroy(ctx_, tail));
  ooc_event* e = nullptr;
  DEV(ooc_event_create(ctx_, 1, &e));
  DEV(ooc_event_record(ctx_, e, OOC_Q_COMPUTE));
  marks_.push_back(e);
  return static_cast<int>(marks_.size()) - 1;
}

double GpuEngine::mark_elapsed(int a, int b) {
  if (a < 0 || b < 0 || a >= static_cast<int>(marks_.size()) || b >= static_cast<int>(marks_.size()))
    throw ValidationError("unknown timing mark");
  DEV(ooc_event_sync(ctx_, marks_[static_cast<std::size_t>(b)]));
  float ms = 0.f;
  DEV(ooc_event_elapsed_ms(marks_[static_cast<std::size_t>(a)], marks_[static_cast<std::size_t>(b)], &ms));
  return ms * 1e-3;
}

std::vector<ChainTiming> GpuEngine::take_timings() {
  std::vector<ChainTiming> out;
  for (auto& pc : pending_chains_) {
    DEV(ooc_event_sync(ctx_, pc.end));
    float ms = 0.f;
    DEV(ooc_event_elapsed_ms(pc.start, pc.end, &ms));
    pc.t.seconds = ms * 1e-3;
    out.push_back(pc.t);
    recycle(pc.start);
    recycle(pc.end);
  }
  pending_chains_.clear();
  return out;
}

std::map<int, double> GpuEngine::take_loop_times() {
  std::map<int, double> out;
  for (auto& pl : pending_loops_) {
    DEV(ooc_event_sync(ctx_, pl.b));
    float ms = 0.f;
    DEV(ooc_event_elapsed_ms(pl.a, pl.b, &ms));
    for (const auto& [id, w] : pl.weights) out[id] += w * ms * 1e-3;
    if (!pl.weights.empty())
      launch_log.push_back({pl.weights.front().first, static_cast<int>(pl.weights.size()), pl.bytes, ms * 1e-3});
    recycle(pl.a);
    recycle(pl.b);
  }
  pending_loops_.clear();
  return out;
}

}  // namespace ooc
