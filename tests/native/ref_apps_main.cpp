// Drop-in proof for the reference's own application code: the reference's
// proj/src/apps.cpp (heat2d, miniflow2d, rk3chain, app_baseline_bandwidth,
// scaling_sweep), compiled UNCHANGED against this repo's ooc/*.hpp and linked with
// libooc.so, drives the B200 runtime. Built by tests/native/Makefile where the
// reference sources exist; run by tests/test_gpu_native_api.py, which compares the
// output with the reference library's golden records (tests/golden/apps.json).
//
//   ref_apps_b200 <app> <nx> <ny> <iters> <span> <executor: reference|explicit>
//                 <tiles> <capacity> <cyclic 0|1> <prefetch 0|1>
//
// Prints one JSON record: per-dataset checksums (the oracle's 64-bit mix,
// oracle/ooc_oracle.py checksum), stale flags, reductions (hex floats), audit rows,
// transfer/metric totals and the flush log — or {"error": "<exception type>"}.
#include <cstdint>
#include <cstdio>
#include <string>

#include "ooc/apps.hpp"
#include "ooc/metrics.hpp"
#include "ooc/runtime.hpp"

namespace {

std::string checksum(const double* p, std::size_t n) {
  std::uint64_t h = 0, s = 0;
  for (std::size_t i = 0; i < n; ++i) {
    std::uint64_t x;
    __builtin_memcpy(&x, p + i, 8);
    const std::uint64_t k = (static_cast<std::uint64_t>(i) * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull) | 1ull;
    const std::uint64_t m = (x ^ (x >> 29)) * k;
    h ^= m ^ (m >> 32);
    s += m;
  }
  char buf[40];
  std::snprintf(buf, sizeof buf, "%016llx%016llx", static_cast<unsigned long long>(h),
                static_cast<unsigned long long>(s));
  return buf;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 11) {
    std::fprintf(stderr, "usage: %s app nx ny iters span executor tiles capacity cyclic prefetch\n", argv[0]);
    return 2;
  }
  ooc::RuntimeOptions o;
  const std::string ex = argv[6];
  o.executor = ex == "explicit" ? ooc::ExecutorKind::tiled_explicit : ooc::ExecutorKind::reference;
  o.tiles = std::atoi(argv[7]);
  o.device.capacity_bytes = std::atoll(argv[8]);
  o.prefetch = std::atoi(argv[10]) != 0;
  ooc::AppParams p;
  p.name = argv[1];
  p.nx = std::atoll(argv[2]);
  p.ny = std::atoll(argv[3]);
  p.iters = std::atoi(argv[4]);
  p.tile_span = std::atoi(argv[5]);
  p.cyclic = std::atoi(argv[9]) != 0;
  std::string out;
  try {
    ooc::Runtime rt(o);
    ooc::run_app(rt, p);  // the reference's run_app (its apps.cpp, unchanged)
    rt.sync();
    out = "{\"buffers\":[";
    for (std::size_t d = 0; d < rt.mesh().datasets.size(); ++d) {
      const ooc::Dataset& ds = rt.mesh().datasets[d];
      out += (d ? ",\"" : "\"") + checksum(ds.host.data(), ds.host.size()) + "\"";
    }
    out += "],\"stale\":[";
    for (std::size_t d = 0; d < rt.mesh().datasets.size(); ++d)
      out += std::string(d ? "," : "") + (rt.mesh().datasets[d].host_stale ? "true" : "false");
    out += "],\"reductions\":{";
    if (p.name == "miniflow2d" && p.iters >= 10) {
      char hx[64];
      std::snprintf(hx, sizeof hx, "%a", rt.fetch_reduction("fieldsum"));
      out += std::string("\"fieldsum\":\"") + hx + "\"";
    }
    out += "},\"audit\":[";
    bool first = true;
    for (const ooc::AuditRow& r : rt.audit_rows()) {
      out += (first ? "[" : ",[") + std::to_string(r.dataset) + "," + std::to_string(r.tile) + "," +
             std::to_string(r.uploaded) + "," + std::to_string(r.downloaded) + "," + std::to_string(r.d2d) + "]";
      first = false;
    }
    const ooc::RunReport rep = rt.report();
    out += "],\"totals\":[" + std::to_string(rep.uploaded) + "," + std::to_string(rep.downloaded) + "," +
           std::to_string(rep.d2d) + "," + std::to_string(rep.total_bytes) + "],\"flush_log\":[";
    first = true;
    for (const ooc::FlushRecord& f : rt.flush_log()) {
      out += (first ? "[" : ",[") + std::to_string(f.chain_id) + ",\"" + ooc::flush_reason_name(f.reason) + "\"," +
             std::to_string(f.loop_count) + "]";
      first = false;
    }
    // the reference's report CSV functions (metrics.hpp) over this runtime's report
    out += "],\"report_csv\":\"" + std::to_string(ooc::report_csv_header().size() + ooc::report_csv_row(rep).size()) +
           "\"}";
  } catch (const ooc::InfeasibleError&) {
    out = "{\"error\":\"InfeasibleError\"}";
  } catch (const ooc::CapacityError&) {
    out = "{\"error\":\"CapacityError\"}";
  } catch (const ooc::StaleDataError&) {
    out = "{\"error\":\"StaleDataError\"}";
  } catch (const ooc::ValidationError& e) {
    out = std::string("{\"error\":\"ValidationError\",\"what\":\"") + e.what() + "\"}";
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 1;
  }
  std::printf("%s\n", out.c_str());
  return 0;
}
