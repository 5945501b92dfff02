// microbenchmark: TMEM load/store throughput per SM (scratch, not product)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void ld16(uint32_t a, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
    : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]) : "r"(a));
}
__device__ __forceinline__ void st16(uint32_t a, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
    :: "r"(a), "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]),"r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]) : "memory");
}
__global__ void k(unsigned long long* out, int iters, int mode) {
  __shared__ uint32_t slot;
  __shared__ float sm[32768];
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t t = slot;
  const uint32_t w = threadIdx.x >> 5;
  const uint32_t base = t + ((32u * (w & 3)) << 16) + 16 * ((w >> 2) & 31);
  uint32_t r[16];
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x + i;
  uint32_t acc = 0;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) {
      ld16(base, r);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc += r[0] ^ r[15];
    } else if (mode == 1) {
      st16(base, r);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      r[0] += 1;
    } else {
      float4 v = reinterpret_cast<float4*>(sm)[(threadIdx.x + it * 7) & 8191];
      acc += __float_as_uint(v.x) ^ __float_as_uint(v.w);
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345) out[1000] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(t));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8 * 2000);
  int iters = 4096;
  for (int mode = 0; mode < 3; ++mode)
    for (int threads : {128, 256, 512, 1024}) {
      k<<<148, threads>>>(d, iters, mode);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      double bytes = (double)threads * 16 * 4 * iters;
      printf("%s threads %4d: %llu cycles, %.1f B/cycle/SM  (%s)\n", mode == 0 ? "LDTM x16" : mode == 1 ? "STTM x16" : "LDS.128 ", threads, h,
             bytes / h, cudaGetErrorString(e));
    }
  return 0;
}
