// fp64 pipe microbenchmark for B200 (sm_100a): DFMA, DMMA (mma.sync m8n8k4 f64)
// and both interleaved in one warp, to decide how the STP contractions are issued.
// Output: one JSON line per test with TFLOP/s (2 flops per FMA).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters, double a, double b) {
  double c0[CHAINS], c1[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { c0[c] = c; c1[c] = -c; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) dmma(c0[c], c1[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += c0[c] + c1[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// interleave: per iteration CHAINS dmma + FCH dfma
template <int CHAINS, int FCH>
__global__ void mixed_kernel(double* out, int iters, double a, double b) {
  double c0[CHAINS], c1[CHAINS], f[FCH];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { c0[c] = c; c1[c] = -c; }
#pragma unroll
  for (int c = 0; c < FCH; ++c) f[c] = c * 0.5;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) dmma(c0[c], c1[c], a, b);
#pragma unroll
    for (int c = 0; c < FCH; ++c) f[c] = fma(f[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += c0[c] + c1[c];
#pragma unroll
  for (int c = 0; c < FCH; ++c) s += f[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

static int g_reps = 5;

template <typename K>
static float time_kernel(K k, int grid, int block, double* out, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) k<<<grid, block>>>(out, iters, 0.999, 1e-9);
  cudaEventRecord(e0);
  const int reps = g_reps;
  for (int r = 0; r < reps; ++r) k<<<grid, block>>>(out, iters, 0.999, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

// usage: fp64_peaks [reps]   (reps = timed launches per test; ~0.7 ms each at 2 blocks/SM)
int main(int argc, char** argv) {
  if (argc > 1) g_reps = atoi(argv[1]);
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d, \"reps\": %d}\n", p.name, sms, clk, g_reps);
  fflush(stdout);
  double* out; CK(cudaMalloc(&out, 4096 * sizeof(double)));
  const int iters = 20000;
  for (int bpsm : {2, 4, 8}) {
    int grid = sms * bpsm, block = 256;
    float ms = time_kernel(dfma_kernel<8>, grid, block, out, iters);
    double fl = 2.0 * 8 * iters * (double)grid * block;
    printf("{\"test\": \"dfma\", \"blocks_per_sm\": %d, \"tflops\": %.2f, \"ms\": %.3f}\n", bpsm, fl / ms / 1e9, ms);
    fflush(stdout);
  }
  for (int bpsm : {2, 4, 8}) {
    int grid = sms * bpsm, block = 256;
    float ms = time_kernel(dmma_kernel<4>, grid, block, out, iters / 4);
    double fl = 2.0 * 256 * 4 * (iters / 4) * (double)grid * (block / 32);
    printf("{\"test\": \"dmma\", \"blocks_per_sm\": %d, \"tflops\": %.2f, \"ms\": %.3f}\n", bpsm, fl / ms / 1e9, ms);
    fflush(stdout);
  }
  for (int bpsm : {4, 8}) {
    int grid = sms * bpsm, block = 256;
    // 2 dmma (512 FMA/warp) + 16 dfma (512 FMA/warp) per iteration
    float ms = time_kernel(mixed_kernel<2, 16>, grid, block, out, iters / 4);
    double fl = 2.0 * (256 * 2 + 32 * 16) * (iters / 4) * (double)grid * (block / 32);
    printf("{\"test\": \"mixed_2dmma_16dfma\", \"blocks_per_sm\": %d, \"tflops\": %.2f, \"ms\": %.3f}\n", bpsm, fl / ms / 1e9, ms);
    fflush(stdout);
  }
  return 0;
}
