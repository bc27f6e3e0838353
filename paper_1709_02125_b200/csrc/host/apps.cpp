// Bundled workloads (see ooc/apps.hpp). The 2-D apps restate proj/src/apps.cpp:36-213
// loop for loop; the 3-D ones are the CloverLeaf-3D / OpenSBLI-TGV analogues.
#include "ooc/apps.hpp"

namespace ooc {

namespace {

using namespace ex;

ParLoop loop_of(Extent range, std::vector<LoopArg> args, KernelSpec k) {
  ParLoop l;
  l.range = range;
  l.args = std::move(args);
  l.kernel = std::move(k);
  return l;
}

KernelSpec writes(int arg, ExprPtr e) {
  KernelSpec k;
  k.writes.push_back({arg, std::move(e)});
  return k;
}

ExprPtr avg4(int a) {  // apps.cpp:25-28
  return mul(c(0.25), add(add(r(a, -1, 0), r(a, 1, 0)), add(r(a, 0, -1), r(a, 0, 1))));
}
ExprPtr star5(int a) {  // apps.cpp:30-34
  return mul(c(0.2),
             add(add(add(r(a, -1, 0), r(a, 1, 0)), add(r(a, 0, -1), r(a, 0, 1))), r(a, 0, 0)));
}
ExprPtr avg6(int a) {
  return mul(c(1.0 / 6.0), add(add(add(r(a, -1, 0, 0), r(a, 1, 0, 0)),
                                   add(r(a, 0, -1, 0), r(a, 0, 1, 0))),
                               add(r(a, 0, 0, -1), r(a, 0, 0, 1))));
}
ExprPtr star7(int a) {
  return mul(c(1.0 / 7.0), add(add(add(add(r(a, -1, 0, 0), r(a, 1, 0, 0)),
                                       add(r(a, 0, -1, 0), r(a, 0, 1, 0))),
                                   add(r(a, 0, 0, -1), r(a, 0, 0, 1))),
                               r(a, 0, 0, 0)));
}

constexpr AccessMode R = AccessMode::read, W = AccessMode::write, RW = AccessMode::read_write;

// Each app body runs in three phases so callers can drive it step by step:
// declare (datasets), iterations [it0, it1) (loops + the app's own flushes), finish.
struct Phase {
  bool declare = true;
  int it0 = 0, it1 = 0;
  bool finish = true;
};

void heat2d(Runtime& rt, const AppParams& p, const Phase& ph) {  // apps.cpp:36-55
  const Extent core = Extent::rect(0, p.nx, 0, p.ny);
  if (ph.declare) {
    rt.declare("u", core, {1, 1, 0}, 8, [](Point q) { return 1.0 + 0.001 * q[0] + 0.002 * q[1]; });
    rt.declare("tmp", core, {1, 1, 0}, 8, 0.0);
    if (p.cyclic) rt.set_cyclic_flag(true);
  }
  const DatasetId u = rt.mesh().find("u"), tmp = rt.mesh().find("tmp");
  const Extent inner = Extent::rect(1, p.nx - 1, 1, p.ny - 1);
  const Stencil s5 = Stencil::star(2, 1);
  for (int it = ph.it0; it < ph.it1; ++it) {
    DatasetId src = it % 2 == 0 ? u : tmp, dst = it % 2 == 0 ? tmp : u;
    rt.enqueue_loop(loop_of(inner, {{src, s5, R}, {dst, Stencil::point(), W}}, writes(1, avg4(0))));
    if (p.tile_span > 0 && (it + 1) % p.tile_span == 0) rt.flush();
  }
  if (ph.finish) rt.finish();
}

struct Flow {
  DatasetId rho, e, v, gamma, t1, t2, t3, t4, t5, t6;
};

Flow declare_flow(Runtime& rt, int nd, index_t nx, index_t ny, index_t nz) {
  Flow f;
  const Extent core = nd == 2 ? Extent::rect(0, nx, 0, ny) : Extent::box(0, nx, 0, ny, 0, nz);
  const Extent wide = nd == 2 ? Extent::rect(-1, nx + 1, -1, ny + 1)
                              : Extent::box(-1, nx + 1, -1, ny + 1, -1, nz + 1);
  const Point h2 = nd == 2 ? Point{2, 2, 0} : Point{2, 2, 2};
  if (nd == 2) {
    f.rho = rt.declare("rho", core, h2, 8, [](Point q) { return 1.0 + 0.002 * q[0] - 0.001 * q[1]; });
    f.e = rt.declare("e", core, h2, 8, [](Point q) { return 2.0 + 0.001 * (q[0] + q[1]); });
    f.v = rt.declare("v", core, h2, 8, [](Point q) { return 0.5 + 0.003 * q[0] + 0.001 * q[1]; });
  } else {
    f.rho = rt.declare("rho", core, h2, 8, [](Point q) {
      return 1.0 + 0.002 * static_cast<double>(q[0]) - 0.001 * static_cast<double>(q[1]) +
             0.0005 * static_cast<double>(q[2]);
    });
    f.e = rt.declare("e", core, h2, 8, [](Point q) {
      return 2.0 + 0.001 * (static_cast<double>(q[0]) + static_cast<double>(q[1]) +
                            static_cast<double>(q[2]));
    });
    f.v = rt.declare("v", core, h2, 8, [](Point q) {
      return 0.5 + 0.003 * static_cast<double>(q[0]) + 0.001 * static_cast<double>(q[1]) -
             0.002 * static_cast<double>(q[2]);
    });
  }
  f.gamma = rt.declare("gamma", core, h2, 8, 1.4);
  DatasetId* t[] = {&f.t1, &f.t2, &f.t3, &f.t4, &f.t5, &f.t6};
  const char* names[] = {"t1", "t2", "t3", "t4", "t5", "t6"};
  for (int i = 0; i < 6; ++i) *t[i] = rt.declare(names[i], wide, {0, 0, 0}, 8, 0.0);
  return f;
}

// miniflow2d: apps.cpp:57-154 (14 loops / iteration, fieldsum every 10th).
// miniflow3d: the same chain in 3-D; the e-update reads t6 along z and the last
// v-update reads t3 along y so every direction is exercised.
void miniflow(Runtime& rt, const AppParams& p, int nd, const Phase& ph) {
  const index_t nz = p.nz > 0 ? p.nz : p.nx;
  if (ph.declare) declare_flow(rt, nd, p.nx, p.ny, nz);
  const Mesh& m = rt.mesh();
  const Flow f{m.find("rho"), m.find("e"), m.find("v"), m.find("gamma"), m.find("t1"),
               m.find("t2"),  m.find("t3"), m.find("t4"), m.find("t5"), m.find("t6")};
  const Extent core = nd == 2 ? Extent::rect(0, p.nx, 0, p.ny) : Extent::box(0, p.nx, 0, p.ny, 0, nz);
  const Extent wide = nd == 2 ? Extent::rect(-1, p.nx + 1, -1, p.ny + 1)
                              : Extent::box(-1, p.nx + 1, -1, p.ny + 1, -1, nz + 1);
  const Stencil pt = Stencil::point(), st = Stencil::star(nd, 1);
  const Stencil sx = Stencil::line(0, 1), sy = Stencil::line(1, 1), sz = Stencil::line(2, 1);
  auto off = [nd](int arg, index_t o0, index_t o1, index_t o2 = 0) {
    return nd == 2 ? r(arg, o0, o1) : r(arg, o0, o1, o2);
  };
  auto smooth = [&](int a) { return nd == 2 ? avg4(a) : avg6(a); };
  for (int it = ph.it0; it < ph.it1; ++it) {
    rt.enqueue_loop(loop_of(wide, {{f.rho, st, R}, {f.t1, pt, W}}, writes(1, smooth(0))));
    rt.enqueue_loop(loop_of(wide, {{f.e, sx, R}, {f.t2, pt, W}},
                            writes(1, mul(c(0.5), sub(off(0, 1, 0), off(0, -1, 0))))));
    rt.enqueue_loop(loop_of(wide, {{f.v, sy, R}, {f.t3, pt, W}},
                            writes(1, mul(c(0.5), sub(off(0, 0, 1), off(0, 0, -1))))));
    rt.enqueue_loop(loop_of(wide, {{f.t1, pt, R}, {f.t2, pt, R}, {f.t4, pt, W}},
                            writes(2, add(r(0), r(1)))));
    rt.enqueue_loop(loop_of(wide, {{f.v, st, R}, {f.t5, pt, W}}, writes(1, smooth(0))));
    rt.enqueue_loop(loop_of(wide, {{f.t3, pt, R}, {f.gamma, pt, R}, {f.e, pt, R}, {f.t6, pt, W}},
                            writes(3, add(mul(r(0), r(1)), mul(c(0.001), r(2))))));
    rt.enqueue_loop(loop_of(core, {{f.rho, pt, RW}, {f.t4, sx, R}},
                            writes(0, add(r(0), mul(c(0.01), sub(off(1, 1, 0), off(1, -1, 0)))))));
    if (nd == 2)
      rt.enqueue_loop(loop_of(core, {{f.e, pt, RW}, {f.t6, sy, R}},
                              writes(0, add(r(0), mul(c(0.01), sub(r(1, 0, 1), r(1, 0, -1)))))));
    else
      rt.enqueue_loop(loop_of(core, {{f.e, pt, RW}, {f.t6, sz, R}},
                              writes(0, add(r(0), mul(c(0.01), sub(r(1, 0, 0, 1), r(1, 0, 0, -1)))))));
    rt.enqueue_loop(loop_of(core, {{f.v, pt, RW}, {f.t5, st, R}},
                            writes(0, add(mul(c(0.99), r(0)), mul(c(0.01), smooth(1))))));
    rt.enqueue_loop(loop_of(wide, {{f.t4, pt, R}, {f.t5, pt, R}, {f.t2, pt, W}},
                            writes(2, sub(r(0), r(1)))));
    rt.enqueue_loop(loop_of(wide, {{f.t1, pt, R}, {f.t2, pt, R}, {f.t3, pt, W}},
                            writes(2, ex::min(r(0), r(1)))));
    rt.enqueue_loop(loop_of(core, {{f.rho, pt, RW}, {f.t2, pt, R}},
                            writes(0, add(r(0), mul(c(0.001), r(1))))));
    rt.enqueue_loop(loop_of(core, {{f.e, pt, RW}, {f.t3, pt, R}},
                            writes(0, add(r(0), mul(c(0.002), r(1))))));
    if (nd == 2)
      rt.enqueue_loop(loop_of(core, {{f.v, pt, RW}, {f.t3, sx, R}},
                              writes(0, add(r(0), mul(c(0.005), add(r(1, -1, 0), r(1, 1, 0)))))));
    else
      rt.enqueue_loop(loop_of(core, {{f.v, pt, RW}, {f.t3, sy, R}},
                              writes(0, add(r(0), mul(c(0.005), add(r(1, 0, -1, 0), r(1, 0, 1, 0)))))));
    if ((it + 1) % 10 == 0) {
      ParLoop red = loop_of(core, {{f.rho, pt, R}, {f.e, pt, R}, {f.v, pt, R}, {f.gamma, pt, R}},
                            KernelSpec{});
      red.kernel.reduce = ReduceOp::sum;
      red.kernel.reduce_expr = add(add(r(0), r(1)), add(r(2), r(3)));
      red.kernel.reduce_name = "fieldsum";
      rt.enqueue_loop(std::move(red));
    }
    if (it == 1) {  // settling phase ends; cyclic execution may begin
      rt.flush();
      if (p.cyclic) rt.set_cyclic_flag(true);
    }
    if (p.tile_span > 0 && (it + 1) % p.tile_span == 0) rt.flush();
  }
  if (ph.finish) rt.finish();
}

// rk3chain: apps.cpp:156-213; rk3chain3d: the same scheme over a 7-point star.
void rk3(Runtime& rt, const AppParams& p, int nd, const Phase& ph) {
  const int span = p.tile_span > 0 ? p.tile_span : 1;
  const index_t pad = 3 * static_cast<index_t>(span) - 1;
  const index_t nz = p.nz > 0 ? p.nz : p.nx;
  const Extent core = nd == 2 ? Extent::rect(-pad, p.nx + pad, -pad, p.ny + pad)
                              : Extent::box(-pad, p.nx + pad, -pad, p.ny + pad, -pad, nz + pad);
  const Point h1 = nd == 2 ? Point{1, 1, 0} : Point{1, 1, 1};
  if (ph.declare) {
  if (nd == 2) {
    rt.declare("w", core, h1, 8, [](Point q) { return 1.0 + 0.0015 * q[0] - 0.0005 * q[1]; });
  } else {
    rt.declare("w", core, h1, 8, [](Point q) {
      return 1.0 + 0.0015 * static_cast<double>(q[0]) - 0.0005 * static_cast<double>(q[1]) +
             0.00025 * static_cast<double>(q[2]);
    });
  }
  rt.declare("r", core, {0, 0, 0}, 8, 0.0);
  rt.declare("k", core, {0, 0, 0}, 8, 0.0);
  if (nd == 2) {
    rt.declare("b", core, {0, 0, 0}, 8, [](Point q) { return 1.0 + 0.0001 * (q[0] + 2 * q[1]); });
  } else {
    rt.declare("b", core, {0, 0, 0}, 8, [](Point q) {
      return 1.0 + 0.0001 * (static_cast<double>(q[0]) + 2.0 * static_cast<double>(q[1]) +
                             3.0 * static_cast<double>(q[2]));
    });
  }
  rt.declare("c2", core, {0, 0, 0}, 8, 0.9);
  rt.declare("d3", core, {0, 0, 0}, 8, 0.05);
  if (p.cyclic) rt.set_cyclic_flag(true);
  }
  const Mesh& m = rt.mesh();
  const DatasetId w = m.find("w"), r_ = m.find("r"), k_ = m.find("k"), b = m.find("b"),
                  c2 = m.find("c2"), d3 = m.find("d3");
  const Stencil pt = Stencil::point(), st = Stencil::star(nd, 1);
  const double alpha[3] = {1.0 / 3.0, 0.5, 1.0};
  const double beta[3] = {0.0, -0.6, -0.85};
  // a chain spans `span` timesteps; [it0, it1) are counted in whole chains of the
  // un-split schedule so step-wise driving reproduces run_app exactly
  int done = ph.it0;
  while (done < ph.it1) {
    const int steps = std::min(span, ph.it1 - done);
    for (int tau = 0; tau < steps; ++tau)
      for (int sigma = 0; sigma < 3; ++sigma) {
        const index_t dp = 3 * static_cast<index_t>(steps - 1 - tau) + (2 - sigma);
        const Extent range = nd == 2 ? Extent::rect(-dp, p.nx + dp, -dp, p.ny + dp)
                                     : Extent::box(-dp, p.nx + dp, -dp, p.ny + dp, -dp, nz + dp);
        rt.enqueue_loop(loop_of(range, {{w, st, R}, {b, pt, R}, {r_, pt, W}},
                                writes(2, mul(nd == 2 ? star5(0) : star7(0), r(1)))));
        if (sigma == 0)
          rt.enqueue_loop(loop_of(range, {{r_, pt, R}, {c2, pt, R}, {k_, pt, W}},
                                  writes(2, mul(r(0), r(1)))));
        else
          rt.enqueue_loop(loop_of(range, {{r_, pt, R}, {c2, pt, R}, {k_, pt, RW}},
                                  writes(2, add(mul(c(beta[sigma]), r(2)), mul(r(0), r(1))))));
        rt.enqueue_loop(loop_of(range, {{w, pt, RW}, {k_, pt, R}, {d3, pt, R}},
                                writes(0, add(r(0), mul(c(alpha[sigma]), mul(r(1), r(2)))))));
      }
    done += steps;
    rt.flush();
  }
  if (ph.finish) rt.finish();
}

void dispatch(Runtime& rt, const AppParams& p, const Phase& ph) {
  if (p.name == "heat2d")
    heat2d(rt, p, ph);
  else if (p.name == "miniflow2d")
    miniflow(rt, p, 2, ph);
  else if (p.name == "miniflow3d")
    miniflow(rt, p, 3, ph);
  else if (p.name == "rk3chain")
    rk3(rt, p, 2, ph);
  else if (p.name == "rk3chain3d")
    rk3(rt, p, 3, ph);
  else
    throw ValidationError("unknown app '" + p.name + "'");
}

}  // namespace

std::vector<std::string> app_names() {
  return {"heat2d", "miniflow2d", "rk3chain", "miniflow3d", "rk3chain3d"};
}

void run_app(Runtime& rt, const AppParams& params) {
  dispatch(rt, params, Phase{true, 0, params.iters, true});
}
void declare_app(Runtime& rt, const AppParams& params) {
  dispatch(rt, params, Phase{true, 0, 0, false});
}
void app_iterations(Runtime& rt, const AppParams& params, int it0, int it1) {
  if (it0 < 0 || it1 < it0) throw ValidationError("bad iteration window");
  dispatch(rt, params, Phase{false, it0, it1, false});
}

index_t app_problem_bytes(const AppParams& p) {
  const index_t nz = p.nz > 0 ? p.nz : p.nx;
  if (p.name == "heat2d") return 2 * (p.nx + 2) * (p.ny + 2) * 8;
  if (p.name == "miniflow2d")
    return (4 * (p.nx + 4) * (p.ny + 4) + 6 * (p.nx + 2) * (p.ny + 2)) * 8;
  if (p.name == "miniflow3d")
    return (4 * (p.nx + 4) * (p.ny + 4) * (nz + 4) + 6 * (p.nx + 2) * (p.ny + 2) * (nz + 2)) * 8;
  const index_t pad = 3 * static_cast<index_t>(p.tile_span > 0 ? p.tile_span : 1) - 1;
  if (p.name == "rk3chain")
    return ((p.nx + 2 * pad + 2) * (p.ny + 2 * pad + 2) + 5 * (p.nx + 2 * pad) * (p.ny + 2 * pad)) * 8;
  if (p.name == "rk3chain3d")
    return ((p.nx + 2 * pad + 2) * (p.ny + 2 * pad + 2) * (nz + 2 * pad + 2) +
            5 * (p.nx + 2 * pad) * (p.ny + 2 * pad) * (nz + 2 * pad)) *
           8;
  throw ValidationError("unknown app '" + p.name + "'");
}

}  // namespace ooc
