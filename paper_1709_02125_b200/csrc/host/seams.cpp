// The reference's two execution seams, implemented over the B200 engine:
//   run_chain_explicit (proj/include/ooc/explicit_exec.hpp:63-65) — the three-slot
//     streaming executor; DeviceState keeps the GpuEngine (streams, slot rotation,
//     staged prefetch) alive across chains like the reference's DeviceState (:39-54);
//   apply_loop (proj/include/ooc/kernel_exec.hpp:29-30) — one par_loop over one range
//     as an sm_100a kernel on device-accessible views.
#include <mutex>

#include "ooc/explicit_exec.hpp"
#include "ooc/gpu_engine.hpp"
#include "ooc/kernel_exec.hpp"
#include "ooc/runtime.hpp"

namespace ooc {

void DeviceState::invalidate_staged(DatasetId d) {
  staged.erase(d);
  if (engine) engine->invalidate_staged(d);
}

ExecResult run_chain_explicit(Mesh& mesh, const LoopChain& chain, const TilePlan& plan, const Footprints& fp,
                              const DeviceConfig& cfg, const ExecOptions& opts, DeviceState& state) {
  if (!state.engine) {
    RuntimeOptions ro;
    ro.executor = ExecutorKind::tiled_explicit;
    ro.device = cfg;
    ro.prefetch = opts.prefetch;
    ro.gpu = state.gpu;
    ro.timeline = state.timeline;
    state.engine = std::make_shared<GpuEngine>(ro);
  }
  GpuEngine& g = *state.engine;
  if (3 * fp.slot_bytes > cfg.capacity_bytes)  // explicit_exec.cpp:61-62, against this call's config
    throw CapacityError(3 * fp.slot_bytes, cfg.capacity_bytes);
  g.set_prefetch(opts.prefetch);
  GpuEngine::ChainOut out;
  g.run_explicit(mesh, chain, plan, fp, opts.cyclic, out);
  g.sync();  // the reference returns with the host buffers updated
  ExecResult res;
  res.audit = std::move(out.audit);
  for (const auto& [loop, slot] : out.reduction_slot) res.reductions[loop] = g.reduction_value(slot);
  if (state.timeline) {
    for (const TimelineRow& r : g.take_timeline()) {
      res.timeline.entries.push_back(
          {r.command_id, static_cast<CmdKind>(r.kind), r.queue, r.bytes, r.issue, r.start, r.end, r.dataset, r.tile, r.loop});
      res.timeline.makespan = std::max(res.timeline.makespan, r.end);
      if (r.kind == 0) res.timeline.uploaded += r.bytes;
      if (r.kind == 1) res.timeline.downloaded += r.bytes;
      if (r.kind == 2) res.timeline.d2d_bytes += r.bytes;
      if (r.kind == 3) res.timeline.kernel_bytes += r.bytes;
    }
  }
  state.slot_cursor = g.slot_cursor();
  state.staged.clear();
  for (const auto& [d, region] : g.staged_regions()) state.staged[d] = DeviceState::Staged{region};
  return res;
}

namespace {
struct LoopCtx {
  ooc_ctx* ctx = nullptr;
  double* red_host = nullptr;
};
std::mutex g_loop_mu;
LoopCtx& loop_ctx(int gpu) {
  static std::map<int, LoopCtx> ctxs;
  LoopCtx& c = ctxs[gpu];
  if (!c.ctx) {
    device_check(ooc_ctx_create(gpu, &c.ctx), "apply_loop: ooc_ctx_create");
    void* p = nullptr;
    device_check(ooc_host_alloc(sizeof(double), &p), "apply_loop: ooc_host_alloc");
    c.red_host = static_cast<double*>(p);
  }
  return c;
}
}  // namespace

void apply_loop(const ParLoop& loop, const Extent& range, const std::vector<ArgView>& views, ExecPolicy,
                double* reduction_acc, int gpu) {
  if (views.size() != loop.args.size()) throw ValidationError("apply_loop: one view per loop argument");
  if (range.empty()) return;
  std::lock_guard<std::mutex> lk(g_loop_mu);
  LoopCtx& c = loop_ctx(gpu);
  const LoweredLoop lw = lower_loop(loop);
  std::vector<ooc_view> v;
  for (std::size_t i = 0; i < views.size(); ++i) {
    const ArgView& a = views[i];
    // every point the loop touches through this argument must lie in its view
    // (proj/src/kernel_exec.cpp:97-101 check_containment)
    auto [slo, shi] = stencil_extents(loop.args[i].stencil);
    if (!a.data || a.box.ndim != range.ndim || !a.box.contains(range.expand(slo, shi)))
      throw ValidationError("apply_loop: argument " + std::to_string(i) + " view " + a.box.str() +
                            " does not contain the range " + range.str() + " and its stencil");
    v.push_back(view_at(a.data, a.box, padded_layout(a.box, 1).stride));
  }
  const int slot = 0;
  if (lw.reduce_op != OOC_RED_NONE) device_check(ooc_reduce_reset(c.ctx, OOC_Q_COMPUTE, slot, lw.reduce_op), "apply_loop");
  const ooc_loop call = make_call(lw, range, v, slot);
  device_check(ooc_launch_loop(c.ctx, OOC_Q_COMPUTE, &call), "apply_loop: ooc_launch_loop");
  if (lw.reduce_op != OOC_RED_NONE) device_check(ooc_reduce_fetch(c.ctx, OOC_Q_COMPUTE, slot, c.red_host), "apply_loop");
  device_check(ooc_queue_sync(c.ctx, OOC_Q_COMPUTE), "apply_loop: sync");
  if (lw.reduce_op != OOC_RED_NONE && reduction_acc)
    *reduction_acc = reduce_combine(loop.kernel.reduce, *reduction_acc, *c.red_host);
}

}  // namespace ooc
