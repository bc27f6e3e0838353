// Parameter block of the NVRTC-specialised par_loop kernels (jit.cu). The kernel
// template declares an identical struct.
#pragma once

#include "ooc_device.h"

#define OOC_JMAX_LOOPS 8
#define OOC_JMAX_READS 64
#define OOC_JMAX_WRITES 32
#define OOC_JMAX_CONST 128

struct JitParams {
  long long nA, nB, nC;
  double* part;
  int red_op;
  int pad;
  int rng[OOC_JMAX_LOOPS][6];
  const double* rp[OOC_JMAX_READS];
  long long rsA[OOC_JMAX_READS];
  long long rsB[OOC_JMAX_READS];
  double* wp[OOC_JMAX_WRITES];
  long long wsA[OOC_JMAX_WRITES];
  long long wsB[OOC_JMAX_WRITES];
  double cst[OOC_JMAX_CONST];
};

namespace oocdev {
int jit_launch_group(ooc_ctx* c, int q, const ooc_loop* loops, int n, int* blocks_out);
}
