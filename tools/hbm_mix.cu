// HBM bandwidth against the read : write mix (round 2d).  The STP writes 4-6x what it reads
// (qavg, favg[3], 12 face arrays per element against one q), while MEASURED_PEAKS.json's HBM peak
// is a copy (1 : 1).  Kernel: every thread reads one 16-byte vector of x (R = 1) or nothing
// (R = 0) and writes W vectors (streams y_0 .. y_{W-1}), all 16-byte accesses, grid-stride, arrays
// far beyond the 126 MB L2.  Prints GB/s of DRAM traffic (read + write) per mix.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hbm_mix tools/hbm_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int R, int W, bool CS>
__global__ void mix(const double2* __restrict__ x, double2* __restrict__ y, long long n, double* sink) {
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double2 v = make_double2(1.0 + (double)i, 2.0);
    if (R) v = CS ? __ldcs(x + i) : x[i];
    if (W == 0) acc += v.x + v.y;
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const double2 o = make_double2(v.x * (k + 1), v.y + k);
      if (CS) __stcs(y + k * n + i, o);
      else y[k * n + i] = o;
    }
  }
  if (W == 0 && acc == 123.456) *sink = acc;
}

template <int R, int W, bool CS>
double run(const double2* x, double2* y, long long n, double* sink, int grid) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 2; ++i) mix<R, W, CS><<<grid, 256>>>(x, y, n, sink);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) mix<R, W, CS><<<grid, 256>>>(x, y, n, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return (double)(R + W) * n * 16.0 * reps / (ms * 1e-3) / 1e9;
}

int main() {
  const long long n = 1ll << 26;  // 1 GiB per stream
  double2 *x, *y;
  double* sink;
  cudaMalloc(&x, n * 16);
  cudaMalloc(&y, 6 * n * 16);
  cudaMalloc(&sink, 8);
  cudaMemset(x, 0, n * 16);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mult : {8, 16, 32}) {
    const int grid = sms * mult;
    printf("{\"grid\": %d, \"read_only\": %.0f, \"copy_1r1w\": %.0f, \"write_only_1\": %.0f, \"write_only_4\": %.0f, "
           "\"r1_w2\": %.0f, \"r1_w4\": %.0f, \"r1_w5\": %.0f, \"r1_w6\": %.0f, \"r1_w5_default_cache\": %.0f}\n",
           grid, run<1, 0, true>(x, y, n, sink, grid), run<1, 1, true>(x, y, n, sink, grid),
           run<0, 1, true>(x, y, n, sink, grid), run<0, 4, true>(x, y, n, sink, grid),
           run<1, 2, true>(x, y, n, sink, grid), run<1, 4, true>(x, y, n, sink, grid),
           run<1, 5, true>(x, y, n, sink, grid), run<1, 6, true>(x, y, n, sink, grid),
           run<1, 5, false>(x, y, n, sink, grid));
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
