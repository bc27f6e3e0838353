// A loop chain written against the reference's C++ API (the shape of
// proj/tests/test_chain_file.cpp:38-79 "by_hand"), compiled unchanged against the
// ooc-b200 headers and run on the B200 streaming engine.
//   usage: heat_chain N ITERS TILES  -> prints the final field (raw doubles) to stdout
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ooc/runtime.hpp"

using namespace ooc;

int main(int argc, char** argv) {
  const index_t n = argc > 1 ? std::atoll(argv[1]) : 64;
  const int iters = argc > 2 ? std::atoi(argv[2]) : 6;
  const int tiles = argc > 3 ? std::atoi(argv[3]) : 3;
  RuntimeOptions opts;
  opts.executor = ExecutorKind::tiled_explicit;
  opts.tiles = tiles;
  Runtime rt(opts);
  DatasetId u = rt.declare("u", Extent::rect(0, n, 0, n), {1, 1, 0}, 8,
                           [](Point p) { return 1.0 + 0.125 * double(p[0] + p[1]); });
  DatasetId tmp = rt.declare("tmp", Extent::rect(0, n, 0, n), {1, 1, 0}, 8, 0.0);
  using namespace ex;
  for (int it = 0; it < iters; ++it) {
    ParLoop l1;
    l1.range = Extent::rect(1, n - 1, 1, n - 1);
    l1.args = {{u, Stencil::star(2, 1), AccessMode::read}, {tmp, Stencil::point(), AccessMode::write}};
    l1.kernel.writes.push_back(
        {1, mul(c(0.25), add(add(r(0, -1, 0), r(0, 1, 0)), add(r(0, 0, -1), r(0, 0, 1))))});
    rt.enqueue_loop(std::move(l1));
    ParLoop l2;
    l2.range = Extent::rect(1, n - 1, 1, n - 1);
    l2.args = {{tmp, Stencil::point(), AccessMode::read}, {u, Stencil::point(), AccessMode::write}};
    l2.kernel.writes.push_back({1, r(0, 0, 0)});
    rt.enqueue_loop(std::move(l2));
  }
  ParLoop red;
  red.range = Extent::rect(0, n, 0, n);
  red.args = {{u, Stencil::point(), AccessMode::read}};
  red.kernel.reduce = ReduceOp::sum;
  red.kernel.reduce_expr = r(0, 0, 0);
  red.kernel.reduce_name = "usum";
  rt.enqueue_loop(std::move(red));
  std::vector<double> v = rt.fetch_dataset(u);
  std::fprintf(stderr, "usum %.17g chains %d tiles %d\n", rt.fetch_reduction("usum"),
               rt.chains_flushed(), rt.last_tile_count());
  std::fwrite(v.data(), sizeof(double), v.size(), stdout);
  return 0;
}
