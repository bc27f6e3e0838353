// The reference's executor seam, driven the way its Runtime::execute drives it
// (proj/src/runtime.cpp:64-148): plan a chain (choose_tile_count under a capacity),
// then run_chain_explicit(mesh, chain, plan, footprints, DeviceConfig, ExecOptions,
// DeviceState&) — here executed by the B200 streaming engine. DeviceState persists
// across chains (slot rotation, speculative first tile), ExecResult carries the audit
// and reductions. INTEGRATION.md §2 quotes this file; tests/test_gpu_native_api.py
// compiles it and checks its output bitwise against the oracle.
//   usage: executor_seam N ITERS CHAINS -> final field u (raw doubles) on stdout
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ooc/explicit_exec.hpp"
#include "ooc/metrics.hpp"
#include "ooc/runtime.hpp"

using namespace ooc;

int main(int argc, char** argv) {
  const index_t n = argc > 1 ? std::atoll(argv[1]) : 96;
  const int iters = argc > 2 ? std::atoi(argv[2]) : 4;
  const int chains = argc > 3 ? std::atoi(argv[3]) : 3;
  Mesh mesh;
  DatasetId u = declare_dataset(mesh, "u", Extent::rect(0, n, 0, n), {1, 1, 0}, 8,
                                [](Point p) { return 1.0 + 0.125 * double(p[0] + p[1]); });
  DatasetId tmp = declare_dataset(mesh, "tmp", Extent::rect(0, n, 0, n), {1, 1, 0}, 8, 0.0);
  index_t problem = 0;
  for (const Dataset& ds : mesh.datasets) problem += ds.alloc().size() * ds.elem_bytes;
  DeviceConfig cfg;
  cfg.capacity_bytes = problem / 3;  // out of core: three slots of a third each at most
  ExecOptions eo;
  eo.prefetch = true;
  DeviceState state;  // lives across chains, like the reference Runtime's device_
  using namespace ex;
  int next_id = 0;
  index_t up = 0, down = 0, metric = 0;
  double usum = 0.0;
  for (int ci = 0; ci < chains; ++ci) {
    LoopChain chain;
    chain.chain_id = ci;
    chain.reason = FlushReason::reduction_fetch;
    for (int it = 0; it < iters; ++it) {
      ParLoop l1;
      l1.range = Extent::rect(1, n - 1, 1, n - 1);
      l1.args = {{u, Stencil::star(2, 1), AccessMode::read}, {tmp, Stencil::point(), AccessMode::write}};
      l1.kernel.writes.push_back({1, mul(c(0.25), add(add(r(0, -1, 0), r(0, 1, 0)), add(r(0, 0, -1), r(0, 0, 1))))});
      ParLoop l2;
      l2.range = Extent::rect(1, n - 1, 1, n - 1);
      l2.args = {{tmp, Stencil::point(), AccessMode::read}, {u, Stencil::point(), AccessMode::write}};
      l2.kernel.writes.push_back({1, r(0, 0, 0)});
      for (ParLoop* l : {&l1, &l2}) {
        validate_loop(mesh, *l);
        l->id = next_id++;
        chain.loops.push_back(std::move(*l));
      }
    }
    ParLoop red;
    red.range = Extent::rect(0, n, 0, n);
    red.args = {{u, Stencil::point(), AccessMode::read}};
    red.kernel.reduce = ReduceOp::sum;
    red.kernel.reduce_expr = r(0, 0, 0);
    red.kernel.reduce_name = "usum";
    validate_loop(mesh, red);
    red.id = next_id++;
    chain.loops.push_back(std::move(red));
    // --- the seam: plan, then run_chain_explicit (proj/src/runtime.cpp:112-125)
    const TileChoice tc = choose_tile_count(mesh, chain, cfg.capacity_bytes);
    ExecResult res = run_chain_explicit(mesh, chain, tc.plan, tc.footprints, cfg, eo, state);
    for (const AuditRow& a : res.audit) {
      up += a.uploaded;
      down += a.downloaded;
    }
    for (const ParLoop& l : chain.loops) metric += loop_metric_bytes(mesh, l);
    usum = res.reductions.at(chain.loops.back().id);
    std::fprintf(stderr, "chain %d T=%d slot_cursor=%d staged=%zu\n", ci, tc.tile_count, state.slot_cursor,
                 state.staged.size());
  }
  std::fprintf(stderr, "usum %.17g uploaded %lld downloaded %lld metric %lld\n", usum, static_cast<long long>(up),
               static_cast<long long>(down), static_cast<long long>(metric));
  const auto& v = mesh[u].host;  // page-locked std::vector<double, PinnedAllocator>
  std::fwrite(v.data(), sizeof(double), v.size(), stdout);
  return 0;
}
