// The reference's kernel seam (proj/include/ooc/kernel_exec.hpp:29-30):
//   apply_loop(const ParLoop&, const Extent& range, const std::vector<ArgView>&, ExecPolicy, double* acc)
// here one sm_100a launch over device-accessible views — the page-locked Dataset::host
// buffers of a Mesh, read and written by the GPU through the host mapping. The program
// applies a 5-point average and a SUM reduction and checks both against a plain host
// evaluation (same operation order, no FMA: bit-identical field, sum within 1e-12).
//   usage: kernel_seam N   -> prints "ok" (exit 0) or the first mismatch (exit 1)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ooc/kernel_exec.hpp"
#include "ooc/runtime.hpp"

using namespace ooc;

int main(int argc, char** argv) {
  const index_t n = argc > 1 ? std::atoll(argv[1]) : 64;
  Mesh mesh;
  DatasetId u = declare_dataset(mesh, "u", Extent::rect(0, n, 0, n), {1, 1, 0}, 8,
                                [](Point p) { return 1.0 + 0.01 * double(p[0]) - 0.003 * double(p[1] * p[1]); });
  DatasetId t = declare_dataset(mesh, "t", Extent::rect(0, n, 0, n), {1, 1, 0}, 8, 0.0);
  using namespace ex;
  ParLoop l;
  l.range = Extent::rect(1, n - 1, 1, n - 1);
  l.args = {{u, Stencil::star(2, 1), AccessMode::read}, {t, Stencil::point(), AccessMode::write}};
  l.kernel.writes.push_back({1, mul(c(0.25), add(add(r(0, -1, 0), r(0, 1, 0)), add(r(0, 0, -1), r(0, 0, 1))))});
  l.kernel.reduce = ReduceOp::sum;
  l.kernel.reduce_expr = sub(r(0, 0, 0), r(0, 1, 0));
  l.kernel.reduce_name = "diff";
  validate_loop(mesh, l);
  std::vector<ArgView> views = {{mesh[u].host.data(), mesh[u].alloc()}, {mesh[t].host.data(), mesh[t].alloc()}};
  double acc = 0.0;
  apply_loop(l, l.range, views, ExecPolicy::openmp, &acc);
  // host evaluation, tape order
  const Extent a = mesh[u].alloc();
  const index_t w = a.hi[1] - a.lo[1];
  auto U = [&](index_t i, index_t j) { return mesh[u].host[static_cast<std::size_t>((i - a.lo[0]) * w + (j - a.lo[1]))]; };
  double want_sum = 0.0;
  for (index_t i = 1; i < n - 1; ++i)
    for (index_t j = 1; j < n - 1; ++j) {
      const double want = 0.25 * ((U(i - 1, j) + U(i + 1, j)) + (U(i, j - 1) + U(i, j + 1)));
      const double got = mesh[t].host[static_cast<std::size_t>((i - a.lo[0]) * w + (j - a.lo[1]))];
      if (got != want) {
        std::printf("mismatch at (%lld,%lld): %.17g vs %.17g\n", static_cast<long long>(i), static_cast<long long>(j), got, want);
        return 1;
      }
      want_sum += U(i, j) - U(i + 1, j);  // r(0, 1, 0): one row down (dim 0)
    }
  if (std::fabs(acc - want_sum) > 1e-12 * std::fabs(want_sum)) {
    std::printf("reduction %.17g vs %.17g\n", acc, want_sum);
    return 1;
  }
  std::printf("ok\n");
  return 0;
}
