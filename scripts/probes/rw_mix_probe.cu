// HBM bandwidth of streaming read/write mixes (R arrays in, W arrays out, fp64, 128-bit
// accesses): what a store-heavy sweep (the chain's last run: 4 in, 9 out) can reach.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rw_mix_probe rw_mix_probe.cu && ./rw_mix_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int R, int W>
__global__ void mix(const double2* const* in, double2* const* out, long long n2) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x) {
    double2 a = make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double2 v = __ldcs(in[r] + i);
      a.x += v.x;
      a.y += v.y;
    }
#pragma unroll
    for (int w = 0; w < W; ++w) __stcs(out[w] + i, make_double2(a.x + w, a.y - w));
  }
}

template <int R, int W>
void run(double2** din, double2** dout, long long n2) {
  const double2** ip;
  double2** op;
  cudaMalloc(&ip, sizeof(void*) * 16);
  cudaMalloc(&op, sizeof(void*) * 16);
  cudaMemcpy(ip, din, sizeof(void*) * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(op, dout, sizeof(void*) * 16, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int grid : {148 * 4, 148 * 8, 148 * 16}) {
    mix<R, W><<<grid, 256>>>(ip, op, n2);
    cudaEventRecord(a);
    const int reps = 5;
    for (int k = 0; k < reps; ++k) mix<R, W><<<grid, 256>>>(ip, op, n2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = double(R + W) * n2 * 16 * reps;
    std::printf("R=%d W=%d grid=%d: %.1f GB/s\n", R, W, grid, bytes / (ms * 1e-3) / 1e9);
  }
  cudaFree(ip);
  cudaFree(op);
}

int main() {
  const long long n = 1LL << 28;  // 2 GiB per array (doubles)
  const long long n2 = n / 2;
  double2* din[16] = {};
  double2* dout[16] = {};
  for (int i = 0; i < 4; ++i) cudaMalloc(&din[i], n * 8);
  for (int i = 0; i < 9; ++i) cudaMalloc(&dout[i], n * 8);
  for (int i = 0; i < 4; ++i) cudaMemset(din[i], 0, n * 8);
  run<1, 1>(din, dout, n2);
  run<4, 3>(din, dout, n2);
  run<4, 9>(din, dout, n2);
  run<4, 0>(din, dout, n2);
  run<0, 4>(din, dout, n2);
  std::printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
