// Bundled workloads. heat2d / miniflow2d / rk3chain are the reference's apps
// (proj/include/ooc/apps.hpp:10-48, proj/src/apps.cpp:36-213), written against the
// same API. miniflow3d (CloverLeaf-3D-shaped) and rk3chain3d (OpenSBLI-TGV-shaped)
// are their 3-D analogues for BASELINE configs 4-5; oracle/programs.py restates
// every one of them in the reference chain-file format so the unmodified
// reference runs them as the parity oracle.
#pragma once

#include <string>
#include <vector>

#include "ooc/runtime.hpp"

namespace ooc {

struct AppParams {
  std::string name = "heat2d";
  index_t nx = 64, ny = 64, nz = 0;  // nz: 3-D apps only (0 = nx)
  int iters = 10;
  int tile_span = 0;
  bool cyclic = false;
};

std::vector<std::string> app_names();
void run_app(Runtime& rt, const AppParams& params);
/// Declares the app's datasets on `rt` without enqueueing loops.
void declare_app(Runtime& rt, const AppParams& params);
/// Enqueues iterations [it0, it1) of an app declared with declare_app, including
/// the app's own flushes (fieldsum, settling flush, spans); run_app equals
/// declare_app + app_iterations(0, iters) + finish. rk3 apps count timesteps and
/// must be driven in whole spans.
void app_iterations(Runtime& rt, const AppParams& params, int it0, int it1);
/// Bytes of every dataset the app declares (core + halo), as app_problem_bytes
/// (proj/src/apps.cpp:230-238) — computed from the extents, without allocating.
index_t app_problem_bytes(const AppParams& params);

}  // namespace ooc
