// Parameter block of the NVRTC-specialised par_loop kernels (jit.cu). The kernel
// template declares an identical struct.
#pragma once

#include <string>

#include "ooc_device.h"

#define OOC_JMAX_LOOPS 8
#define OOC_JMAX_FAMILIES 48
#define OOC_JMAX_WRITES 24
#define OOC_JMAX_CONST 128
#define OOC_JMAX_VIEWS 16

// A load family: one dataset view read at one (a, c) offset; its rows are loaded
// once per thread tile and shared by every read of that view at any b offset.
struct JitParams {
  long long nA, nB, nC;                    // canonical extents of the launch box (c contiguous)
  double* part;                            // reduction block partials
  int red_op;
  int pad;
  int rng[OOC_JMAX_LOOPS][6];              // per loop: [a0,a1) [b0,b1) [c0,c1) rel. to the box
  const double* fp[OOC_JMAX_FAMILIES];     // family base (box origin, a-offset folded in)
  long long fsA[OOC_JMAX_FAMILIES], fsB[OOC_JMAX_FAMILIES];
  long long fbox[OOC_JMAX_FAMILIES][6];    // safe-load bounds on (a, b, c) rel. to the box
  long long inner[6];                      // interior tiles: a in [0,1), ib0 in [2, 3-Q], block cols in [4,5)
  double* wp[OOC_JMAX_WRITES];
  long long wsA[OOC_JMAX_WRITES], wsB[OOC_JMAX_WRITES];
  double cst[OOC_JMAX_CONST];
  int tv_org[OOC_JMAX_VIEWS][3];           // TMA template: tensor coords (c, b, a) of each staged
                                           // view's box at tile (0, 0, 0)
};

namespace oocdev {
int jit_launch_group(ooc_ctx* c, int q, const ooc_loop* loops, int n, int* blocks_out);
// Generic NVRTC path shared with the row-sweep kernels (sweep.cu): build `kname` from
// `src` for sm_100a with the exact-arithmetic flags; launch with programmatic
// dependent launch on queue q (counts one specialised launch).
int jit_policy(long long* min_points);  // OOC_JIT mode (0/1/2) and its size threshold
bool jit_available(bool load, std::string& why);
// acc[slot] = combine(acc[slot], fixed-order fold of the queue's `blocks` partials)
int launch_fold(ooc_ctx* c, int q, int blocks, int slot, int op);
extern bool g_frozen;  // graph capture in progress: no tuning launches (ooc_jit_freeze)
bool jit_build_kernel(const std::string& src, const char* kname, int block, long long smem, void** fn,
                      int* occ, std::string& err, bool load);
// Tiled f64 tensor map for TMA tensor copies (zero fill out of bounds); false if the driver
// entry point is unavailable or rejects the layout.
bool jit_tensor_map(void* out128, int rank, const double* base, const unsigned long long* gdim,
                    const unsigned long long* gstride_bytes, const unsigned* box);
int jit_launch_kernel(ooc_ctx* c, int q, void* fn, unsigned gx, unsigned gy, unsigned block, unsigned smem,
                      void** args);
}
