// microbenchmark (round 2): tcgen05.mma kind::f16 cycles per instruction,
// A from shared memory (SS) vs A from TMEM (TS), N = 32..256, short batches
// (commit + wait every 16 MMAs, as a single slot does) vs long batches
// (the steady-state pipe rate when several items keep it fed).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_bw2 mma_bw2.cu
#include <cstdint>
#include <cstdio>
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
__host__ __device__ constexpr uint32_t idesc(uint32_t M, uint32_t N, bool amn, bool bmn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((amn ? 1u : 0u) << 15) | ((bmn ? 1u : 0u) << 16) |
         ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
               "r"(a), "l"(b), "r"(id), "r"(acc));
}

// TS: A from TMEM; N; BATCH16: commits every 16 MMAs (else every 256);
// PIPE: wait for the previous batch, not the one just committed
template <int TS, int N>
__global__ void k(unsigned long long* out, int reps, int batch16, int pipelined) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[2];
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
  uint32_t ph[2] = {0, 0};
  if (threadIdx.x == 0) {
    constexpr uint32_t id = idesc(128, N, false, N >= 64);  // N = 32: K-major B
    const int per = batch16 ? 1 : 16;  // 16-MMA groups per commit
    const unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const int b = pipelined ? (r & 1) : 0;
      for (int g = 0; g < per; ++g) {
#pragma unroll
        for (uint32_t i = 0; i < 16; ++i) {
          const uint32_t s = i & 7;
          const uint64_t bd = N >= 64 ? desc(sb + 65536 + s * 2048 * (N / 64), 1024 * (N / 64), 1024)
                                      : desc(sb + 65536 + (s >> 2) * 4096 + (s & 3) * 32, 1024, 16);
          const uint32_t d = t + (i >> 3) * (N <= 128 ? 128 : 0);
          if (TS) mma_ts(d, t + 256 + s * 8, bd, id, s);
          else mma_ss(d, desc(sb + (s >> 2) * 16384 + (s & 3) * 32, 1024, 16), bd, id, s);
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(&bar[b]))
                   : "memory");
      const int w = pipelined ? (b ^ 1) : b;
      if (!pipelined || r > 0) {
        asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&bar[w])),
                     "r"(ph[w])
                     : "memory");
        ph[w] ^= 1;
      }
    }
    if (pipelined) {
      const int w = (reps - 1) & 1;
      asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(&bar[w])),
                   "r"(ph[w])
                   : "memory");
    }
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

template <int TS, int N>
void run(unsigned long long* d) {
  cudaFuncSetAttribute(k<TS, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int b16 = 1; b16 >= 0; --b16)
    for (int pipe = 0; pipe < 2; ++pipe) {
      if (!b16 && pipe) continue;
      const int total = 65536;
      const int reps = total / (b16 ? 16 : 256);
      k<TS, N><<<148, 128, 200 * 1024>>>(d, reps, b16, pipe);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      const double c = (double)h / total;
      printf("%s N=%3d batch=%3d pipe=%d: %6.1f cycles/MMA, %5.1f%% of floor (%s)\n", TS ? "TS" : "SS",
             N, b16 ? 16 : 256, pipe, c, 100.0 * (N / 2.0) / c, cudaGetErrorString(e));
    }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 2000);
  printf("mode N batch pipelined: cycles/MMA (floor N/2), %% of floor\n");
  run<0, 32>(d); run<0, 64>(d); run<0, 128>(d); run<0, 256>(d);
  run<1, 32>(d); run<1, 64>(d); run<1, 128>(d); run<1, 256>(d);
  return 0;
}
