// Pinned host <-> device box-copy throughput for the layouts the streaming engine uses:
// contiguous, device rows padded (2-D/3-D pitched), host rows strided (a box narrower
// than the allocation). nvcc -O2 -arch=sm_100a copy_probe.cu -o copy_probe
#include <cuda_runtime.h>
#include <cstdio>

static double gbps(size_t bytes, float ms) { return bytes / (ms * 1e-3) / 1e9; }

int main() {
  const size_t n1 = 604, n2 = 604, planes = 200;  // one 3-D tile: 200 planes of 604x604
  const size_t host_elems = planes * n1 * n2;
  double *h, *d;
  cudaHostAlloc(&h, host_elems * 8 * 2, cudaHostAllocPortable);
  cudaMalloc(&d, planes * n1 * 640 * 8 + (64 << 20));
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, cudaMemcpyKind k, size_t dpitch_e, size_t hpitch_e, size_t w_e, size_t rows_per_plane) {
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      cudaMemcpy3DParms p{};
      cudaPitchedPtr hp = make_cudaPitchedPtr(h, hpitch_e * 8, w_e * 8, n1);
      cudaPitchedPtr dp = make_cudaPitchedPtr(d, dpitch_e * 8, w_e * 8, rows_per_plane);
      p.srcPtr = k == cudaMemcpyHostToDevice ? hp : dp;
      p.dstPtr = k == cudaMemcpyHostToDevice ? dp : hp;
      p.extent = make_cudaExtent(w_e * 8, rows_per_plane, planes);
      p.kind = k;
      cudaEventRecord(a, s);
      cudaMemcpy3DAsync(&p, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-44s %s %7.2f GB/s\n", name, k == cudaMemcpyHostToDevice ? "H2D" : "D2H",
           gbps(w_e * rows_per_plane * planes * 8, best));
  };
  auto flat = [&](cudaMemcpyKind k) {
    const size_t bytes = host_elems * 8;
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(a, s);
      if (k == cudaMemcpyHostToDevice) cudaMemcpyAsync(d, h, bytes, k, s);
      else cudaMemcpyAsync(h, d, bytes, k, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-44s %s %7.2f GB/s\n", "1-D contiguous", k == cudaMemcpyHostToDevice ? "H2D" : "D2H", gbps(bytes, best));
  };
  for (cudaMemcpyKind k : {cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost}) {
    flat(k);
    run("3-D same pitch (604/604)", k, 604, 604, 604, 604);
    run("3-D device rows padded 604->608", k, 608, 604, 604, 604);
    run("3-D device rows padded 604->640", k, 640, 604, 604, 604);
    run("3-D host strided (600 of 604), dev 608", k, 608, 604, 600, 600);
    run("3-D host strided (602 of 604), dev 602", k, 602, 604, 602, 602);
  }
  // 2-D: 15364-wide rows
  return 0;
}
