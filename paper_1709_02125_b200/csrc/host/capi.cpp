// C ABI of the runtime (include/ooc_stencil.h). Exceptions of the reference's
// types become negative status codes; messages go to a thread-local buffer.
#include "ooc_stencil.h"

#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>

#include "json_writer.hpp"
#include "ooc/apps.hpp"
#include "ooc/gpu_engine.hpp"
#include "ooc/chain_file.hpp"
#include "ooc/runtime.hpp"

struct ooc_runtime {
  std::unique_ptr<ooc::Runtime> rt;
};

namespace {

thread_local std::string g_err;
thread_local std::string g_out;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ooc::StaleDataError& e) {
    g_err = std::string("StaleDataError: ") + e.what();
    return OOC_E_STALE;
  } catch (const ooc::InfeasibleError& e) {
    g_err = std::string("InfeasibleError: ") + e.what();
    return OOC_E_INFEASIBLE;
  } catch (const ooc::CapacityError& e) {
    g_err = std::string("CapacityError: ") + e.what();
    return OOC_E_CAPACITY;
  } catch (const ooc::ValidationError& e) {
    g_err = std::string("ValidationError: ") + e.what();
    return OOC_E_VALIDATION;
  } catch (const ooc::DeviceError& e) {
    g_err = std::string("DeviceError: ") + e.what();
    return OOC_E_DEVICE;
  } catch (const std::exception& e) {
    g_err = std::string("Error: ") + e.what();
    return OOC_E_OTHER;
  }
}

const char* out_str(std::string s) {
  g_out = std::move(s);
  return g_out.c_str();
}

const char* err_json() {
  ooc::JsonWriter w;
  w.begin_object().key("error").value(g_err).end_object();
  return out_str(w.str());
}

ooc::Extent extent_of(int ndim, const int64_t lo[3], const int64_t hi[3]) {
  return ooc::Extent::make(ndim, {lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]});
}

// Coordinate-only fill expression evaluated with the tape of the expression,
// the same stack order as the reference's chain-file fill (chain_file.cpp:72-115).
std::function<double(ooc::Point)> fill_from_expr(const std::string& text) {
  using namespace ooc;
  ExprTape tape = ExprTape::compile(parse_prefix_expr(text, /*allow_coords=*/true));
  for (const auto& in : tape.ins)
    if (in.op == ExprOp::read) throw ValidationError("fill expressions cannot read datasets");
  return [tape](Point p) {
    double st[OOC_MAX_STACK];
    int sp = 0;
    for (const auto& in : tape.ins) {
      switch (in.op) {
        case ExprOp::constant:
          st[sp++] = in.value;
          break;
        case ExprOp::coord:
          st[sp++] = static_cast<double>(p[in.arg]);
          break;
        case ExprOp::add:
          --sp;
          st[sp - 1] = st[sp - 1] + st[sp];
          break;
        case ExprOp::sub:
          --sp;
          st[sp - 1] = st[sp - 1] - st[sp];
          break;
        case ExprOp::mul:
          --sp;
          st[sp - 1] = st[sp - 1] * st[sp];
          break;
        case ExprOp::divide:
          --sp;
          st[sp - 1] = st[sp - 1] / st[sp];
          break;
        case ExprOp::min:
          --sp;
          st[sp - 1] = st[sp] < st[sp - 1] ? st[sp] : st[sp - 1];
          break;
        case ExprOp::max:
          --sp;
          st[sp - 1] = st[sp - 1] < st[sp] ? st[sp] : st[sp - 1];
          break;
        default:
          break;
      }
    }
    return st[0];
  };
}

}  // namespace

extern "C" {

void ooc_rt_default_options(ooc_runtime_options* o) {
  std::memset(o, 0, sizeof *o);
  o->executor = OOC_EXEC_REFERENCE;
  o->capacity_bytes = 16000000000LL;
}

const char* ooc_rt_last_error(void) { return g_err.c_str(); }

int ooc_rt_create(const ooc_runtime_options* o, ooc_runtime** out) {
  return guard([&] {
    ooc::RuntimeOptions ro;
    ro.executor = static_cast<ooc::ExecutorKind>(o->executor);
    ro.tiles = o->tiles;
    ro.tiled_dim = o->tiled_dim;
    if (o->capacity_bytes > 0) ro.device.capacity_bytes = o->capacity_bytes;
    ro.resident_budget = o->resident_budget;
    ro.prefetch = o->prefetch != 0;
    ro.record_chains = o->record_chains != 0;
    ro.gpu = o->gpu;
    ro.profile_loops = o->profile_loops != 0;
    ro.arena_fill = o->arena_fill;
    ro.fuse = o->no_fuse == 0;
    ro.dist_rank = o->dist_rank;
    ro.dist_world = o->dist_world > 0 ? o->dist_world : 1;
    ro.own_lo = o->own_lo;
    ro.own_hi = o->own_hi;
    ro.ghost = o->ghost;
    ro.timeline = o->timeline != 0;
    auto* h = new ooc_runtime;
    h->rt = std::make_unique<ooc::Runtime>(ro);
    *out = h;
  });
}

void ooc_rt_destroy(ooc_runtime* h) { delete h; }

int ooc_rt_declare(ooc_runtime* h, const char* name, int ndim, const int64_t lo[3],
                   const int64_t hi[3], const int64_t halo[3], int64_t elem_bytes,
                   const char* fill_expr, double fill_value, const double* init, int* id_out) {
  return guard([&] {
    ooc::Extent core = extent_of(ndim, lo, hi);
    ooc::Point h3{halo[0], halo[1], halo[2]};
    int id;
    if (init) {
      id = h->rt->declare(name, core, h3, elem_bytes, 0.0);
      ooc::Dataset& ds = h->rt->mesh()[id];
      std::memcpy(ds.host.data(), init, ds.host.size() * sizeof(double));
    } else if (fill_expr && *fill_expr) {
      id = h->rt->declare(name, core, h3, elem_bytes, fill_from_expr(fill_expr));
    } else {
      id = h->rt->declare(name, core, h3, elem_bytes, fill_value);
    }
    if (id_out) *id_out = id;
  });
}

int ooc_rt_enqueue_loop(ooc_runtime* h, int ndim, const int64_t lo[3], const int64_t hi[3],
                        int nargs, const int* dataset, const int* mode, const int* noffsets,
                        const int64_t* offsets, int nwrites, const int* write_args,
                        const char* const* write_exprs, int reduce_op, const char* reduce_expr,
                        const char* reduce_name) {
  return guard([&] {
    ooc::ParLoop loop;
    loop.range = extent_of(ndim, lo, hi);
    const int64_t* o = offsets;
    for (int a = 0; a < nargs; ++a) {
      ooc::LoopArg arg;
      arg.dataset = dataset[a];
      if (mode[a] < 0 || mode[a] > 2) throw ooc::ValidationError("bad access mode");
      arg.mode = static_cast<ooc::AccessMode>(mode[a]);
      for (int k = 0; k < noffsets[a]; ++k, o += 3) arg.stencil.offsets.push_back({o[0], o[1], o[2]});
      loop.args.push_back(std::move(arg));
    }
    for (int w = 0; w < nwrites; ++w)
      loop.kernel.writes.push_back({write_args[w], ooc::parse_prefix_expr(write_exprs[w])});
    if (reduce_op != OOC_REDUCE_NONE) {
      loop.kernel.reduce = static_cast<ooc::ReduceOp>(reduce_op);
      if (reduce_expr) loop.kernel.reduce_expr = ooc::parse_prefix_expr(reduce_expr);
      loop.kernel.reduce_name = reduce_name ? reduce_name : "";
    }
    h->rt->enqueue_loop(std::move(loop));
  });
}

int ooc_rt_flush(ooc_runtime* h) {
  return guard([&] { h->rt->flush(); });
}
int ooc_rt_finish(ooc_runtime* h) {
  return guard([&] { h->rt->finish(); });
}
int ooc_rt_sync(ooc_runtime* h) {
  return guard([&] { h->rt->sync(); });
}
int ooc_rt_set_cyclic(ooc_runtime* h, int on) {
  return guard([&] { h->rt->set_cyclic_flag(on != 0); });
}
int ooc_rt_fetch_dataset(ooc_runtime* h, int d, double* out, int64_t n) {
  return guard([&] { h->rt->fetch_dataset_into(d, out, static_cast<std::size_t>(n)); });
}
int ooc_rt_fetch_reduction(ooc_runtime* h, const char* name, double* out) {
  return guard([&] { *out = h->rt->fetch_reduction(name); });
}

int ooc_rt_num_datasets(ooc_runtime* h) { return static_cast<int>(h->rt->mesh().datasets.size()); }

int ooc_rt_dataset_info(ooc_runtime* h, int d, int64_t* len, int* stale, int* ndim, int64_t lo[3],
                        int64_t hi[3]) {
  return guard([&] {
    if (d < 0 || d >= static_cast<int>(h->rt->mesh().datasets.size()))
      throw ooc::ValidationError("unknown dataset id");
    const ooc::Dataset& ds = h->rt->mesh()[d];
    if (len) *len = static_cast<int64_t>(ds.host.size());
    if (stale) *stale = ds.host_stale ? 1 : 0;
    const ooc::Extent a = ds.alloc();
    if (ndim) *ndim = a.ndim;
    for (int k = 0; k < 3; ++k) {
      if (lo) lo[k] = a.lo[k];
      if (hi) hi[k] = a.hi[k];
    }
  });
}

int ooc_rt_find_dataset(ooc_runtime* h, const char* name) { return h->rt->mesh().find(name); }

int ooc_rt_host_data(ooc_runtime* h, int d, double** data, int64_t* len) {
  return guard([&] {
    ooc::Dataset& ds = h->rt->mesh()[d];
    *data = ds.host.data();
    *len = static_cast<int64_t>(ds.host.size());
  });
}

int ooc_rt_run_app(ooc_runtime* h, const char* name, int64_t nx, int64_t ny, int64_t nz, int iters,
                   int span, int cyclic) {
  return guard([&] {
    ooc::AppParams p;
    p.name = name;
    p.nx = nx;
    p.ny = ny;
    p.nz = nz;
    p.iters = iters;
    p.tile_span = span;
    p.cyclic = cyclic != 0;
    ooc::run_app(*h->rt, p);
  });
}

int ooc_rt_declare_app(ooc_runtime* h, const char* name, int64_t nx, int64_t ny, int64_t nz,
                       int span) {
  return guard([&] {
    ooc::AppParams p;
    p.name = name;
    p.nx = nx;
    p.ny = ny;
    p.nz = nz;
    p.tile_span = span;
    ooc::declare_app(*h->rt, p);
  });
}

int ooc_rt_app_iterations(ooc_runtime* h, const char* name, int64_t nx, int64_t ny, int64_t nz,
                           int span, int cyclic, int it0, int it1) {
  return guard([&] {
    ooc::AppParams p;
    p.name = name;
    p.nx = nx;
    p.ny = ny;
    p.nz = nz;
    p.tile_span = span;
    p.cyclic = cyclic != 0;
    ooc::app_iterations(*h->rt, p, it0, it1);
  });
}

int64_t ooc_app_problem_bytes(const char* name, int64_t nx, int64_t ny, int64_t nz, int span) {
  int64_t out = -1;
  guard([&] {
    ooc::AppParams p;
    p.name = name;
    p.nx = nx;
    p.ny = ny;
    p.nz = nz;
    p.tile_span = span;
    out = ooc::app_problem_bytes(p);
  });
  return out;
}

int ooc_rt_mark(ooc_runtime* h) {
  int id = -1;
  int rc = guard([&] { id = h->rt->engine().mark(); });
  return rc ? rc : id;
}

int ooc_rt_mark_elapsed(ooc_runtime* h, int a, int b, double* seconds) {
  return guard([&] { *seconds = h->rt->engine().mark_elapsed(a, b); });
}

const char* ooc_rt_flush_log_json(ooc_runtime* h) {
  ooc::JsonWriter w;
  w.begin_array();
  for (const auto& f : h->rt->flush_log())
    w.begin_array().value(f.chain_id).value(ooc::flush_reason_name(f.reason)).value(f.loop_count).end_array();
  w.end_array();
  return out_str(w.str());
}

const char* ooc_rt_audit_json(ooc_runtime* h) {
  ooc::JsonWriter w;
  w.begin_array();
  for (const auto& r : h->rt->audit_rows())
    w.begin_array().value(r.dataset).value(r.tile).value(r.uploaded).value(r.downloaded).value(r.d2d).end_array();
  w.end_array();
  return out_str(w.str());
}

void ooc_rt_set_row_recompute(int on) { ooc::set_row_recompute(on != 0); }
void ooc_rt_set_sweep(int on) { ooc::set_sweep(on != 0); }

int ooc_rt_set_exact_reductions(ooc_runtime* h, int on) {
  return guard([&] { h->rt->set_exact_reductions(on != 0); });
}

const char* ooc_rt_report_csv(ooc_runtime* h, const char* app, const char* size, int iters) {
  std::string s;
  int rc = guard([&] { s = h->rt->report_csv(app ? app : "", size ? size : "", iters); });
  return rc ? nullptr : out_str(s);
}

const char* ooc_rt_loops_csv(ooc_runtime* h) {
  std::string s;
  int rc = guard([&] { s = h->rt->loops_csv(); });
  return rc ? nullptr : out_str(s);
}

const char* ooc_rt_audit_csv(ooc_runtime* h) {
  std::string s;
  int rc = guard([&] { s = h->rt->audit_csv(); });
  return rc ? nullptr : out_str(s);
}

const char* ooc_rt_timeline_csv(ooc_runtime* h) {
  std::string s;
  int rc = guard([&] { s = h->rt->timeline_csv(); });
  return rc ? nullptr : out_str(s);
}

const char* ooc_rt_report_json(ooc_runtime* h) {
  std::string s;
  int rc = guard([&] {
    ooc::RunReport r = h->rt->report();
    ooc::JsonWriter w;
    w.begin_object();
    w.key("mode").value(r.mode);
    w.key("tiles").value(r.tiles);
    w.key("average_bandwidth").value(r.average_bandwidth);
    w.key("total_bytes").value(r.total_bytes);
    w.key("total_time").value(r.total_time);
    w.key("uploaded").value(r.uploaded);
    w.key("downloaded").value(r.downloaded);
    w.key("d2d").value(r.d2d);
    w.key("capacity").value(r.capacity);
    w.key("chains").value(h->rt->chains_flushed());
    w.end_object();
    s = w.str();
  });
  return rc ? err_json() : out_str(s);
}

const char* ooc_rt_chain_timings_json(ooc_runtime* h) {
  std::string s;
  int rc = guard([&] {
    ooc::JsonWriter w;
    w.begin_array();
    for (const auto& t : h->rt->chain_timings()) {
      w.begin_object();
      w.key("chain").value(t.chain_id);
      w.key("tiles").value(t.tiles);
      w.key("loops").value(t.loops);
      w.key("metric_bytes").value(t.metric_bytes);
      w.key("uploaded").value(t.uploaded);
      w.key("downloaded").value(t.downloaded);
      w.key("d2d").value(t.d2d);
      w.key("seconds").value(t.seconds);
      w.end_object();
    }
    w.end_array();
    s = w.str();
  });
  return rc ? err_json() : out_str(s);
}

const char* ooc_rt_loop_metrics_json(ooc_runtime* h) {
  std::string s;
  int rc = guard([&] {
    ooc::JsonWriter w;
    w.begin_array();
    for (const auto& m : h->rt->loop_metrics())
      w.begin_array().value(m.loop_id).value(m.points).value(m.bytes).value(m.time_s).end_array();
    w.end_array();
    s = w.str();
  });
  return rc ? err_json() : out_str(s);
}

const char* ooc_rt_launch_log_json(ooc_runtime* h) {
  std::string s;
  int rc = guard([&] {
    h->rt->loop_metrics();  // resolves pending launch events into the log
    ooc::JsonWriter w;
    w.begin_array();
    for (const auto& r : h->rt->engine().launch_log)
      w.begin_array().value(r.first_loop).value(r.nloops).value(r.bytes).value(r.seconds).end_array();
    w.end_array();
    h->rt->engine().launch_log.clear();
    s = w.str();
  });
  return rc ? err_json() : out_str(s);
}

const char* ooc_rt_device_json(ooc_runtime* h) {
  std::string s;
  int rc = guard([&] {
    ooc::GpuEngine& g = h->rt->engine();
    const ooc_dev_props& p = g.props();
    ooc_dev_stats st{};
    ooc_stats(g.ctx(), &st);
    long long in_use = 0, peak = 0;
    ooc_mem_usage(g.ctx(), &in_use, &peak);
    ooc::JsonWriter w;
    w.begin_object();
    w.key("name").value(std::string(p.name));
    w.key("sm_count").value(p.sm_count);
    w.key("cc").value(std::to_string(p.cc_major) + "." + std::to_string(p.cc_minor));
    w.key("l2_bytes").value(p.l2_bytes);
    w.key("hbm_bytes").value(p.hbm_bytes);
    w.key("kernel_launches").value(st.kernel_launches);
    w.key("interp_launches").value(st.interp_launches);
    w.key("special_launches").value(st.special_launches);
    w.key("h2d_bytes").value(st.h2d_bytes);
    w.key("d2h_bytes").value(st.d2h_bytes);
    w.key("d2d_bytes").value(st.d2d_bytes);
    w.key("copy_calls").value(st.copy_calls);
    w.key("jit_launches").value(st.jit_launches);
    w.key("jit_compiles").value(st.jit_compiles);
    w.key("jit_compile_ms").value(st.jit_compile_ms);
    w.key("jit_host_us").value(st.jit_host_us);
    w.key("graph_launches").value(st.graph_launches);
    w.key("sweep_launches").value(st.sweep_launches);
    w.key("sweep_host_us").value(st.sweep_host_us);
    w.key("comm_bytes").value(st.comm_bytes);
    w.key("mem_in_use").value(in_use);
    w.key("mem_peak").value(peak);
    w.key("build").value(std::string(ooc_dev_build_info()));
    w.end_object();
    s = w.str();
  });
  return rc ? err_json() : out_str(s);
}

int ooc_rt_num_chains(ooc_runtime* h) { return static_cast<int>(h->rt->chain_log().size()); }

const char* ooc_rt_chain_plan_json(ooc_runtime* h, int chain, int tiles, int64_t budget, int dump) {
  std::string s;
  int rc = guard([&] {
    const auto& log = h->rt->chain_log();
    if (chain < 0 || chain >= static_cast<int>(log.size()))
      throw ooc::ValidationError("no such recorded chain");
    const ooc::LoopChain& c = log[static_cast<std::size_t>(chain)];
    const ooc::Mesh& m = h->rt->mesh();
    if (tiles > 0) {
      ooc::TilePlan plan = ooc::compute_tile_plan(m, c, tiles, h->rt->options().tiled_dim);
      ooc::Footprints fp = ooc::compute_footprints(m, c, plan);
      s = dump ? ooc::plan_dump_json(m, c, plan, fp) : ooc::plan_full_json(m, plan, fp);
    } else {
      ooc::TileChoice ch = ooc::choose_tile_count(m, c, budget, h->rt->options().tiled_dim);
      s = dump ? ooc::plan_dump_json(m, c, ch.plan, ch.footprints)
               : ooc::plan_full_json(m, ch.plan, ch.footprints);
    }
  });
  return rc ? err_json() : out_str(s);
}

const char* ooc_rt_chain_sweep_check(ooc_runtime* h, int chain, int compile) {
  std::string s;
  int rc = guard([&] {
    const ooc::LoopChain& c = h->rt->chain_log().at(static_cast<std::size_t>(chain));
    const ooc::Mesh& m = h->rt->mesh();
    std::vector<ooc_view> views(m.datasets.size());
    for (std::size_t d = 0; d < m.datasets.size(); ++d) {
      const ooc::Extent a = m.datasets[d].alloc();
      ooc::BoxLayout L = ooc::padded_layout(a);
      views[d] = ooc::view_at(reinterpret_cast<double*>((d + 1) << 32), a, L.stride);
    }
    std::vector<ooc::LoweredLoop> low;
    for (const auto& l : c.loops) low.push_back(ooc::lower_loop(l));
    std::vector<ooc_loop> calls;
    for (std::size_t j = 0; j < c.loops.size(); ++j) {
      std::vector<ooc_view> v;
      for (const auto& a : c.loops[j].args) v.push_back(views[static_cast<std::size_t>(a.dataset)]);
      calls.push_back(ooc::make_call(low[j], c.loops[j].range, v, 0));
    }
    ooc::JsonWriter w;
    w.begin_array();
    for (const ooc::SweepRun& run : ooc::plan_sweeps(m, c.loops, false, calls)) {
      const std::size_t a = run.a, b = run.b;
      std::vector<ooc_redirect> dead;
      for (ooc::DatasetId d : run.dead) dead.push_back({views[static_cast<std::size_t>(d)].data, nullptr});
      std::vector<char> log(1 << 20);
      int r = ooc_sweep_describe(calls.data() + a, static_cast<int>(b - a), dead.data(), static_cast<int>(dead.size()),
                                 log.data(), static_cast<int>(log.size()), compile);
      w.begin_object().key("first").value(static_cast<long long>(a)).key("loops").value(static_cast<long long>(b - a));
      w.key("ok").value(r == OOC_OK).key("plan").value(std::string(log.data()));
      w.key("dead").begin_array();
      for (ooc::DatasetId d : run.dead) w.value(static_cast<long long>(d));
      w.end_array();
      w.end_object();
    }
    w.end_array();
    s = w.str();
  });
  return rc ? err_json() : out_str(s);
}

const char* ooc_rt_chain_jit_check(ooc_runtime* h, int chain, int fuse) {
  std::string s;
  int rc = guard([&] {
    const ooc::LoopChain& c = h->rt->chain_log().at(static_cast<std::size_t>(chain));
    const ooc::Mesh& m = h->rt->mesh();
    // stand-in device views: distinct fake bases per dataset, the resident layout
    std::vector<ooc_view> views(m.datasets.size());
    for (std::size_t d = 0; d < m.datasets.size(); ++d) {
      const ooc::Extent a = m.datasets[d].alloc();
      ooc::BoxLayout L = ooc::padded_layout(a);
      views[d] = ooc::view_at(reinterpret_cast<double*>((d + 1) << 32), a, L.stride);
    }
    std::vector<ooc::LoweredLoop> low;
    for (const auto& l : c.loops) low.push_back(ooc::lower_loop(l));
    ooc::JsonWriter w;
    w.begin_array();
    std::vector<const ooc::ParLoop*> grp;
    std::vector<ooc_loop> calls;
    std::size_t tape = 0;
    auto flush = [&] {
      if (calls.empty()) return;
      std::vector<char> log(1 << 16);
      int r = ooc_jit_compile_check(calls.data(), static_cast<int>(calls.size()), log.data(),
                                    static_cast<int>(log.size()));
      w.begin_object().key("loops").value(static_cast<long long>(calls.size()));
      w.key("ok").value(r == OOC_OK);
      if (r != OOC_OK || std::getenv("OOC_JIT_DUMP")) w.key("log").value(std::string(log.data()));
      w.end_object();
      grp.clear();
      calls.clear();
      tape = 0;
    };
    std::vector<std::size_t> tape_len(c.loops.size());
    for (std::size_t j = 0; j < c.loops.size(); ++j) tape_len[j] = low[j].tape.size();
    const std::vector<char> starts = ooc::plan_fusion(m, c.loops, tape_len, fuse != 0);
    for (std::size_t j = 0; j < c.loops.size(); ++j) {
      const ooc::ParLoop& l = c.loops[j];
      if (starts[j] || !ooc::can_fuse(grp, tape, l, fuse != 0)) flush();
      ooc_loop L{};
      L.ndim = l.range.ndim;
      for (int d = 0; d < 3; ++d) {
        L.lo[d] = l.range.lo[d];
        L.hi[d] = l.range.hi[d];
      }
      L.nargs = static_cast<int32_t>(l.args.size());
      for (std::size_t a = 0; a < l.args.size(); ++a) L.args[a] = views[static_cast<std::size_t>(l.args[a].dataset)];
      const ooc::LoweredLoop& lw = low[j];
      L.nwrites = static_cast<int32_t>(lw.write_arg.size());
      for (std::size_t k = 0; k < lw.write_arg.size(); ++k) {
        L.write_arg[k] = lw.write_arg[k];
        L.write_len[k] = lw.write_len[k];
      }
      L.reduce_op = lw.reduce_op;
      L.reduce_len = lw.reduce_len;
      L.ntape = static_cast<int32_t>(lw.tape.size());
      L.tape = lw.tape.data();
      calls.push_back(L);
      grp.push_back(&l);
      tape += lw.tape.size();
      if (l.has_reduction()) flush();
    }
    flush();
    w.end_array();
    s = w.str();
  });
  return rc ? err_json() : out_str(s);
}

int ooc_rt_load_chain_json(ooc_runtime* h, const char* text, int* loops_enqueued) {
  return guard([&] {
    const ooc::ChainFileResult r = ooc::load_chain_json(*h->rt, text ? text : "");
    if (loops_enqueued) *loops_enqueued = r.loops_enqueued;
  });
}

int ooc_rt_comm_init_ipc(ooc_runtime* h, const char* name) {
  return guard([&] { h->rt->comm_init_ipc(name ? name : ""); });
}

int ooc_rt_comm_init(ooc_runtime* h, const void* unique_id) {
  return guard([&] { h->rt->comm_init(unique_id); });
}

const char* ooc_rt_chain_export_json(ooc_runtime* h, int chain) {
  std::string s;
  int rc = guard([&] {
    const ooc::LoopChain& c = h->rt->chain_log().at(static_cast<std::size_t>(chain));
    const ooc::Mesh& m = h->rt->mesh();
    ooc::JsonWriter w;
    w.begin_array();
    for (const ooc::ParLoop& l : c.loops) {
      w.begin_object();
      w.key("id").value(l.id);
      w.key("lo").begin_array();
      for (int d = 0; d < l.range.ndim; ++d) w.value(l.range.lo[d]);
      w.end_array();
      w.key("hi").begin_array();
      for (int d = 0; d < l.range.ndim; ++d) w.value(l.range.hi[d]);
      w.end_array();
      w.key("args").begin_array();
      for (const ooc::LoopArg& a : l.args) {
        w.begin_object().key("dataset").value(m[a.dataset].name).key("mode").value(ooc::access_name(a.mode));
        w.key("offsets").begin_array();
        for (const ooc::Point& o : a.stencil.offsets) w.begin_array().value(o[0]).value(o[1]).value(o[2]).end_array();
        w.end_array().end_object();
      }
      w.end_array();
      w.key("writes").begin_object();
      for (const auto& wr : l.kernel.writes) w.key(std::to_string(wr.arg)).value(ooc::expr_to_string(wr.expr));
      w.end_object();
      if (l.has_reduction()) {
        const char* op = l.kernel.reduce == ooc::ReduceOp::sum ? "SUM" : l.kernel.reduce == ooc::ReduceOp::min ? "MIN" : "MAX";
        w.key("reduction").begin_object().key("op").value(op).key("expr").value(ooc::expr_to_string(l.kernel.reduce_expr))
            .key("name").value(l.kernel.reduce_name).end_object();
      }
      w.end_object();
    }
    w.end_array();
    s = w.str();
  });
  return rc ? err_json() : out_str(s);
}

const char* ooc_rt_dist_plan_json(ooc_runtime* h, int chain) {
  std::string s;
  int rc = guard([&] {
    const ooc::LoopChain& c = h->rt->chain_log().at(static_cast<std::size_t>(chain));
    const ooc::Mesh& m = h->rt->mesh();
    ooc::JsonWriter w;
    w.begin_object();
    w.key("depth").value(h->rt->dependency_depth(c));
    w.key("ghost").value(h->rt->options().ghost);
    w.key("halos").begin_array();
    for (const ooc::HaloXfer& x : h->rt->halo_plan(c)) {
      w.begin_object().key("dataset").value(m[x.dataset].name);
      const std::pair<const char*, const ooc::index_t*> f[] = {
          {"send_left", x.send_left}, {"recv_left", x.recv_left}, {"send_right", x.send_right}, {"recv_right", x.recv_right}};
      for (const auto& [k, v] : f) w.key(k).begin_array().value(v[0]).value(v[1]).end_array();
      w.end_object();
    }
    w.end_array();
    w.end_object();
    s = w.str();
  });
  return rc ? err_json() : out_str(s);
}

const char* ooc_rt_chain_plan_text(ooc_runtime* h, int chain, int tiles) {
  std::string s;
  int rc = guard([&] {
    const ooc::LoopChain& c = h->rt->chain_log().at(static_cast<std::size_t>(chain));
    const ooc::Mesh& m = h->rt->mesh();
    ooc::TilePlan plan = ooc::compute_tile_plan(m, c, tiles, h->rt->options().tiled_dim);
    s = ooc::plan_dump_text(m, c, plan, ooc::compute_footprints(m, c, plan));
  });
  return rc ? err_json() : out_str(s);
}

const char* ooc_rt_chain_oracle_json(ooc_runtime* h, int chain, int tiles) {
  std::string s;
  int rc = guard([&] {
    const ooc::LoopChain& c = h->rt->chain_log().at(static_cast<std::size_t>(chain));
    const ooc::Mesh& m = h->rt->mesh();
    ooc::TilePlan plan = ooc::compute_tile_plan(m, c, tiles, h->rt->options().tiled_dim);
    ooc::OracleResult r = ooc::dependency_oracle(m, c, plan);
    ooc::JsonWriter w;
    w.begin_object();
    w.key("ok").value(r.ok);
    w.key("tile").value(r.tile);
    w.key("loop").value(r.loop);
    w.key("dataset").value(r.dataset);
    w.key("point").begin_array().value(r.point[0]).value(r.point[1]).value(r.point[2]).end_array();
    w.key("message").value(r.message);
    w.end_object();
    s = w.str();
  });
  return rc ? err_json() : out_str(s);
}

}  // extern "C"
