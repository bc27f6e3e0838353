// oracle/ref/ref_capi.cpp — TEST INFRASTRUCTURE ONLY (never part of the product path).
//
// A thin C ABI over the *unmodified* reference library compiled from
// /root/reference/proj/src (see oracle/ref/Makefile). Tests, golden-vector
// generation and bench.py's CPU-baseline leg load the resulting
// oracle/_ref/libooc_ref.so through ctypes; nothing in the product links it.
//
// Programs are the reference's own chain-file JSON (proj/src/chain_file.cpp:58-162)
// extended with an "ops" list so flushes / cyclic toggles can sit between loops:
//   {"datasets": [...], "stencils": [...],
//    "ops": [{"op": "loop", <chain-file loop object>}, {"op": "flush"},
//            {"op": "cyclic", "on": true}, {"op": "finish"}]}
// Every loop is fed through the reference's load_chain_json so the reference's
// own parser and fill evaluator define the semantics.
#include <cstring>
#include <memory>
#include <sstream>
#include <string>

#include "json.hpp"
#include "ooc/apps.hpp"
#include "ooc/chain_file.hpp"
#include "ooc/runtime.hpp"
#include "ooc/tiler.hpp"

using nlohmann::json;
using namespace ooc;

namespace {

thread_local std::string g_err;
thread_local std::string g_str;

struct Handle {
  std::unique_ptr<Runtime> rt;
};

json ext_json(const Extent& e) {
  return json::array({e.ndim, e.lo[0], e.lo[1], e.lo[2], e.hi[0], e.hi[1], e.hi[2]});
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const StaleDataError& e) {
    g_err = std::string("StaleDataError: ") + e.what();
    return -2;
  } catch (const InfeasibleError& e) {
    g_err = std::string("InfeasibleError: ") + e.what();
    return -3;
  } catch (const CapacityError& e) {
    g_err = std::string("CapacityError: ") + e.what();
    return -4;
  } catch (const ValidationError& e) {
    g_err = std::string("ValidationError: ") + e.what();
    return -1;
  } catch (const std::exception& e) {
    g_err = std::string("error: ") + e.what();
    return -9;
  }
}

json full_plan_json(const Mesh& mesh, const TilePlan& plan, const Footprints& fp) {
  json j;
  j["T"] = plan.tile_count;
  j["tiled_dim"] = plan.tiled_dim;
  j["nominal_ends"] = plan.nominal_ends;
  j["ends"] = plan.ends;
  j["warnings"] = plan.warnings.size();
  j["slot_bytes"] = fp.slot_bytes;
  json ds = json::array();
  for (size_t d = 0; d < fp.per_dataset.size(); ++d) {
    const auto& pd = fp.per_dataset[d];
    json jd;
    jd["name"] = mesh.datasets[d].name;
    jd["accessed"] = pd.accessed;
    if (pd.accessed) {
      jd["written_any"] = pd.written_any;
      jd["write_first"] = pd.write_first;
      jd["max_tile_bytes"] = pd.max_tile_bytes;
      std::vector<int> mod(pd.modified.begin(), pd.modified.end());
      jd["modified"] = mod;
      for (const char* key : {"full", "left_edge", "right_edge", "left_fp", "right_fp"}) {
        const std::vector<Extent>& v = std::string(key) == "full"         ? pd.full
                                       : std::string(key) == "left_edge"  ? pd.left_edge
                                       : std::string(key) == "right_edge" ? pd.right_edge
                                       : std::string(key) == "left_fp"    ? pd.left_fp
                                                                          : pd.right_fp;
        json arr = json::array();
        for (const auto& e : v) arr.push_back(ext_json(e));
        jd[key] = arr;
      }
    }
    ds.push_back(jd);
  }
  j["datasets"] = ds;
  return j;
}

}  // namespace

extern "C" {

const char* refo_last_error() { return g_err.c_str(); }

// executor: 0 reference, 2 tiled_explicit (ExecutorKind order, proj/include/ooc/runtime.hpp:18)
void* refo_create(int executor, int tiles, long long capacity, int openmp, int prefetch,
                  int record) {
  RuntimeOptions o;
  o.executor = static_cast<ExecutorKind>(executor);
  o.tiles = tiles;
  if (capacity > 0) o.device.capacity_bytes = capacity;
  o.policy = openmp ? ExecPolicy::openmp : ExecPolicy::serial;
  o.prefetch = prefetch != 0;
  o.record_chains = record != 0;
  auto* h = new Handle;
  h->rt = std::make_unique<Runtime>(o);
  return h;
}

void refo_destroy(void* p) { delete static_cast<Handle*>(p); }

int refo_load_program(void* p, const char* text) {
  Runtime& rt = *static_cast<Handle*>(p)->rt;
  return guarded([&] {
    json doc = json::parse(text);
    json decl;
    decl["datasets"] = doc.value("datasets", json::array());
    load_chain_json(rt, decl.dump());
    json stencils = doc.value("stencils", json::array());
    json ops = doc.contains("ops") ? doc["ops"] : json::array();
    if (!doc.contains("ops"))
      for (const auto& l : doc.value("loops", json::array())) {
        json op = l;
        op["op"] = "loop";
        ops.push_back(op);
      }
    for (const auto& op : ops) {
      std::string kind = op.at("op").get<std::string>();
      if (kind == "loop") {
        json one;
        one["stencils"] = stencils;
        json l = op;
        l.erase("op");
        one["loops"] = json::array({l});
        load_chain_json(rt, one.dump());
      } else if (kind == "flush") {
        rt.flush();
      } else if (kind == "finish") {
        rt.finish();
      } else if (kind == "cyclic") {
        rt.set_cyclic_flag(op.value("on", true));
      } else {
        throw ValidationError("unknown program op '" + kind + "'");
      }
    }
  });
}

int refo_run_app(void* p, const char* name, long long nx, long long ny, int iters, int span,
                 int cyclic) {
  Runtime& rt = *static_cast<Handle*>(p)->rt;
  return guarded([&] {
    AppParams ap;
    ap.name = name;
    ap.nx = nx;
    ap.ny = ny;
    ap.iters = iters;
    ap.tile_span = span;
    ap.cyclic = cyclic != 0;
    run_app(rt, ap);
  });
}

long long refo_app_problem_bytes(const char* name, long long nx, long long ny, int span) {
  AppParams ap;
  ap.name = name;
  ap.nx = nx;
  ap.ny = ny;
  ap.tile_span = span;
  return app_problem_bytes(ap);
}

int refo_flush(void* p) {
  return guarded([&] { static_cast<Handle*>(p)->rt->flush(); });
}
int refo_finish(void* p) {
  return guarded([&] { static_cast<Handle*>(p)->rt->finish(); });
}

int refo_num_datasets(void* p) {
  return static_cast<int>(static_cast<Handle*>(p)->rt->mesh().datasets.size());
}
const char* refo_dataset_name(void* p, int d) {
  g_str = static_cast<Handle*>(p)->rt->mesh().datasets.at(d).name;
  return g_str.c_str();
}
long long refo_dataset_len(void* p, int d) {
  return static_cast<long long>(static_cast<Handle*>(p)->rt->mesh().datasets.at(d).host.size());
}
int refo_dataset_stale(void* p, int d) {
  return static_cast<Handle*>(p)->rt->mesh().datasets.at(d).host_stale ? 1 : 0;
}
// Raw host copy (no flush, no stale check) — the buffer the reference holds.
int refo_copy_dataset(void* p, int d, double* out) {
  const auto& h = static_cast<Handle*>(p)->rt->mesh().datasets.at(d).host;
  std::memcpy(out, h.data(), h.size() * sizeof(double));
  return 0;
}
// Zero-copy address of the buffer the reference holds (bench parity at full size).
const double* refo_dataset_ptr(void* p, int d) {
  return static_cast<Handle*>(p)->rt->mesh().datasets.at(d).host.data();
}
// Flushing fetch with the reference's stale semantics (runtime.cpp:13-19).
int refo_fetch_dataset(void* p, int d, double* out) {
  Runtime& rt = *static_cast<Handle*>(p)->rt;
  return guarded([&] {
    auto v = rt.fetch_dataset(d);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
  });
}
int refo_fetch_reduction(void* p, const char* name, double* out) {
  Runtime& rt = *static_cast<Handle*>(p)->rt;
  return guarded([&] { *out = rt.fetch_reduction(name); });
}

// totals: uploaded, downloaded, d2d, total_metric_bytes, chains_flushed, last_tiles
int refo_totals(void* p, long long* out, double* time_out) {
  Runtime& rt = *static_cast<Handle*>(p)->rt;
  out[0] = rt.uploaded();
  out[1] = rt.downloaded();
  out[2] = rt.d2d_bytes();
  long long bytes = 0;
  double t = 0;
  for (const auto& m : rt.loop_metrics()) {
    bytes += m.bytes;
    t += m.time_s;
  }
  out[3] = bytes;
  out[4] = rt.chains_flushed();
  out[5] = rt.last_tile_count();
  *time_out = t;
  return 0;
}

const char* refo_flush_log_json(void* p) {
  Runtime& rt = *static_cast<Handle*>(p)->rt;
  json a = json::array();
  for (const auto& f : rt.flush_log())
    a.push_back({f.chain_id, flush_reason_name(f.reason), f.loop_count});
  g_str = a.dump();
  return g_str.c_str();
}

const char* refo_audit_json(void* p) {
  Runtime& rt = *static_cast<Handle*>(p)->rt;
  json a = json::array();
  for (const auto& r : rt.audit_rows())
    a.push_back({r.dataset, r.tile, r.uploaded, r.downloaded, r.d2d});
  g_str = a.dump();
  return g_str.c_str();
}

const char* refo_reductions_json(void* p) {
  // latest value per reduction name is only reachable through fetch_reduction;
  // callers pass names explicitly, so this returns the per-loop metric rows instead
  Runtime& rt = *static_cast<Handle*>(p)->rt;
  json a = json::array();
  for (const auto& m : rt.loop_metrics()) a.push_back({m.loop_id, m.points, m.bytes, m.time_s});
  g_str = a.dump();
  return g_str.c_str();
}

int refo_num_chains(void* p) {
  return static_cast<int>(static_cast<Handle*>(p)->rt->chain_log().size());
}

// Full plan + footprint dump of a recorded chain. tiles > 0 plans with that
// count; otherwise choose_tile_count(budget) picks it (tiler.cpp:383-402).
const char* refo_chain_plan_json(void* p, int chain_index, int tiles, long long budget) {
  Runtime& rt = *static_cast<Handle*>(p)->rt;
  int rc = guarded([&] {
    const LoopChain& chain = rt.chain_log().at(chain_index);
    if (tiles > 0) {
      TilePlan plan = compute_tile_plan(rt.mesh(), chain, tiles, 0);
      Footprints fp = compute_footprints(rt.mesh(), chain, plan);
      g_str = full_plan_json(rt.mesh(), plan, fp).dump();
    } else {
      TileChoice c = choose_tile_count(rt.mesh(), chain, budget, 0);
      g_str = full_plan_json(rt.mesh(), c.plan, c.footprints).dump();
    }
  });
  if (rc != 0) g_str = json({{"error", g_err}}).dump();
  return g_str.c_str();
}

const char* refo_chain_plan_dump_json(void* p, int chain_index, int tiles) {
  Runtime& rt = *static_cast<Handle*>(p)->rt;
  int rc = guarded([&] {
    const LoopChain& chain = rt.chain_log().at(chain_index);
    TilePlan plan = compute_tile_plan(rt.mesh(), chain, tiles, 0);
    Footprints fp = compute_footprints(rt.mesh(), chain, plan);
    g_str = plan_dump_json(rt.mesh(), chain, plan, fp);
  });
  if (rc != 0) g_str = json({{"error", g_err}}).dump();
  return g_str.c_str();
}

}  // extern "C"
