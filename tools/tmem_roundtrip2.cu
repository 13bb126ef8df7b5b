// TMEM round trip check: every thread of 10 warps stores 4 x 20 columns of its own values and
// reads them back (the stp_bip_kernel layout).  Prints the mismatch count.
#include <cstdio>
#include <cstdint>
#ifndef OFF
#define OFF 82
#endif
__device__ __forceinline__ void st16(uint32_t ta, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};\n" ::"r"(ta),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}
__device__ __forceinline__ void st4(uint32_t ta, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(ta), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]));
}
__device__ __forceinline__ void ld16(uint32_t ta, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) : "r"(ta));
}
__device__ __forceinline__ void ld4(uint32_t ta, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(ta));
}
__global__ void k(int* bad, uint32_t* basev) {
  __shared__ uint32_t base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(&base)), "n"(256) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (threadIdx.x == 0) basev[blockIdx.x] = base;
  // packed layout with unaligned x16 offsets: warp w uses columns [ (w>>2)*OFF, ... ), blocks of 20 at 20t
  const uint32_t ta = base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * OFF);
  uint32_t r[20];
  for (int t = 0; t < 4; ++t) {
    for (int i = 0; i < 20; ++i) r[i] = blockIdx.x * 100000 + threadIdx.x * 100 + t * 20 + i;
    st16(ta + 20 * t, r);
    st4(ta + 20 * t + 16, r + 16);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  __syncthreads();
  int nb = 0;
  for (int t = 0; t < 4; ++t) {
    ld16(ta + 20 * t, r);
    ld4(ta + 20 * t + 16, r + 16);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    for (int i = 0; i < 20; ++i) nb += r[i] != blockIdx.x * 100000 + threadIdx.x * 100 + t * 20 + i;
  }
  atomicAdd(bad, nb);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(base), "n"(256) : "memory");
}
int main() {
  int* bad; uint32_t* bv;
  cudaMalloc(&bad, 4); cudaMemset(bad, 0, 4);
  cudaMalloc(&bv, 4 * 1000);
  k<<<1000, 320, 100000>>>(bad, bv);
  cudaError_t e = cudaDeviceSynchronize();
  int h; uint32_t hb[4];
  cudaMemcpy(&h, bad, 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hb, bv, 16, cudaMemcpyDeviceToHost);
  printf("err=%s bad=%d base=%x %x %x %x\n", cudaGetErrorString(e), h, hb[0], hb[1], hb[2], hb[3]);
  return 0;
}
