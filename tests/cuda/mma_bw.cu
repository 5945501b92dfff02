// microbenchmark: tcgen05.mma kind::f16 issue/throughput for small-N shapes (scratch)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t sbo, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;  // SW128
  return d;
}
__device__ __forceinline__ uint32_t idesc(uint32_t M, uint32_t N, bool amn, bool bmn, bool neg) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((neg ? 1u : 0u) << 13) | ((amn ? 1u : 0u) << 15) |
         ((bmn ? 1u : 0u) << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc));
}
__global__ void k(unsigned long long* out, int reps, int mode) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
  unsigned long long t0 = 0, t1 = 0;
  uint32_t phase = 0;
  if (threadIdx.x == 0) {
    t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      for (uint32_t s = 0; s < 8; ++s) {
        const uint32_t fr = sb + 0, fi = sb + 32768, br = sb + 65536, bi = sb + 65536 + 16384;
        const uint32_t ko = (s >> 2) * 16384 + (s & 3) * 32;
        uint64_t dr = desc(fr + ko, 1024, 16), di = desc(fi + ko, 1024, 16);
        if (mode == 0) {  // stage B as in the kernel: N=64, B MN-major, negate, 2 accumulators
          uint64_t xr = desc(br + s * 2048, 1024, 1024), xi = desc(bi + s * 2048, 1024, 1024);
          uint32_t ip = idesc(128, 64, false, true, false), in = idesc(128, 64, false, true, true);
          mma(t, dr, xr, ip, s); mma(t, di, xi, in, 1); mma(t + 64, di, xr, ip, s); mma(t + 64, dr, xi, ip, 1);
        } else if (mode == 1) {  // same, B K-major
          uint64_t xr = desc(br + (s >> 2) * 8192 + (s & 3) * 32, 1024, 16), xi = desc(bi + (s >> 2) * 8192 + (s & 3) * 32, 1024, 16);
          uint32_t ip = idesc(128, 64, false, false, false), in = idesc(128, 64, false, false, true);
          mma(t, dr, xr, ip, s); mma(t, di, xi, in, 1); mma(t + 64, di, xr, ip, s); mma(t + 64, dr, xi, ip, 1);
        } else if (mode == 2) {  // N=128 MN-major (twice the data per MMA), 2 MMAs per k-step
          uint64_t xr = desc(br + s * 2048, 1024, 8192);
          uint32_t ip = idesc(128, 128, false, true, false);
          mma(t, dr, xr, ip, s); mma(t + 128, di, xr, ip, s);
        } else if (mode == 3) {  // N=256 K-major, 1 MMA per k-step
          uint64_t xr = desc(br + (s >> 2) * 32768 + (s & 3) * 32, 1024, 16);
          uint32_t ip = idesc(128, 256, false, false, false);
          mma(t, dr, xr, ip, s);
        } else if (mode == 4) {  // N=64 MN-major, no negate, single accumulator
          uint64_t xr = desc(br + s * 2048, 1024, 1024), xi = desc(bi + s * 2048, 1024, 1024);
          uint32_t ip = idesc(128, 64, false, true, false);
          mma(t, dr, xr, ip, s); mma(t, di, xi, ip, 1); mma(t, di, xr, ip, 1); mma(t, dr, xi, ip, 1);
        } else {  // N=64, 4 distinct accumulators
          uint64_t xr = desc(br + s * 2048, 1024, 1024), xi = desc(bi + s * 2048, 1024, 1024);
          uint32_t ip = idesc(128, 64, false, true, false);
          mma(t, dr, xr, ip, s); mma(t + 64, di, xi, ip, s); mma(t + 128, di, xr, ip, s); mma(t + 192, dr, xi, ip, s);
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
      asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" :: "r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"(phase) : "memory");
      phase ^= 1;
    }
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(t));
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8 * 2000);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* names[] = {"N64 MN-major neg 2acc (kernel)", "N64 K-major neg 2acc", "N128 MN-major 2acc", "N256 K-major 1acc", "N64 MN 1acc no-neg", "N64 MN 4acc"};
  const double flops_per_batch[] = {8*4*2.0*128*64*16, 8*4*2.0*128*64*16, 8*2*2.0*128*128*16, 8*2.0*128*256*16, 8*4*2.0*128*64*16, 8*4*2.0*128*64*16};
  int reps = 2000;
  for (int mode = 0; mode < 6; ++mode) {
    for (int grid : {1, 148}) {
      k<<<grid, 128, 200 * 1024>>>(d, reps, mode);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      double cyc_per_batch = (double)h / reps;
      printf("%-32s grid %3d: %.0f cycles/batch, %.1f flop/cycle/SM (%s)\n", names[mode], grid, cyc_per_batch,
             flops_per_batch[mode] / cyc_per_batch, cudaGetErrorString(e));
    }
  }
  return 0;
}
