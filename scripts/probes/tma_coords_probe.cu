// Probe: does a tiled 3-D TMA tensor load (f64) accept odd and negative box coordinates
// (out-of-bounds elements zero-filled)? Each case runs in its own process so a fault
// cannot poison the others.   nvcc -gencode arch=compute_100a,code=sm_100a -o p tma_coords_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void probe(const __grid_constant__ CUtensorMap map, int x, int y, int z, double* out, int n) {
  __shared__ __align__(128) double buf[16 * 34];
  __shared__ __align__(8) unsigned long long bar;
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar));
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(buf));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(16 * 34 * 8));
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(d),
        "l"(&map), "r"(x), "r"(y), "r"(z), "r"(b)
        : "memory");
  }
  unsigned done = 0;
  while (!done)
    asm volatile("{\n .reg .pred P1;\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n selp.u32 %0, 1, 0, P1;\n}\n"
                 : "=r"(done)
                 : "r"(b));
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
  const int x = std::atoi(argv[1]), y = std::atoi(argv[2]), z = std::atoi(argv[3]);
  const int NX = 100, NY = 40, NZ = 8, PX = 112;  // padded row pitch (16 doubles)
  std::vector<double> h(static_cast<size_t>(PX) * NY * NZ);
  for (int k = 0; k < NZ; ++k)
    for (int j = 0; j < NY; ++j)
      for (int i = 0; i < PX; ++i) h[(static_cast<size_t>(k) * NY + j) * PX + i] = 1e6 * k + 1e3 * j + i + 1;
  double *dv, *dout;
  cudaMalloc(&dv, h.size() * 8);
  cudaMalloc(&dout, 16 * 34 * 8);
  cudaMemcpy(dv, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  CUtensorMap map;
  cuuint64_t gdim[3] = {static_cast<cuuint64_t>(NX), static_cast<cuuint64_t>(NY), static_cast<cuuint64_t>(NZ)};
  cuuint64_t gstr[2] = {static_cast<cuuint64_t>(PX) * 8, static_cast<cuuint64_t>(PX) * NY * 8};
  cuuint32_t box[3] = {34, 16, 1}, es[3] = {1, 1, 1};
  CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, dv, gdim, gstr, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::printf("encode failed %d\n", static_cast<int>(r));
    return 2;
  }
  probe<<<1, 128>>>(map, x, y, z, dout, 16 * 34);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    std::printf("coords (%d,%d,%d): FAULT %s\n", x, y, z, cudaGetErrorString(e));
    return 1;
  }
  std::vector<double> o(16 * 34);
  cudaMemcpy(o.data(), dout, o.size() * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int j = 0; j < 16; ++j)
    for (int i = 0; i < 34; ++i) {
      const int gx = x + i, gy = y + j, gz = z;
      const double want = (gx >= 0 && gx < NX && gy >= 0 && gy < NY && gz >= 0 && gz < NZ) ? 1e6 * gz + 1e3 * gy + gx + 1 : 0.0;
      if (o[j * 34 + i] != want) ++bad;
    }
  std::printf("coords (%d,%d,%d): %s (%d mismatches)\n", x, y, z, bad ? "WRONG" : "ok", bad);
  return bad ? 3 : 0;
}
