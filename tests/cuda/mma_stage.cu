// microbenchmark (round 2): the exact tcgen05 MMA batches of the config-2
// forward (fb_single_tc.cu stages A, B (three-plane windows), B', A') issued
// back to back on one SM, cycles per batch; plus variants of stage B.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_stage mma_stage.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t sbo, uint32_t lbo = 16) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(uint32_t M, uint32_t N, bool amn, bool bmn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((amn ? 1u : 0u) << 15) | ((bmn ? 1u : 0u) << 16) |
         ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc));
}
constexpr uint32_t SIN = 0, SOP = 32768, SMAT = SOP + 2 * 49152, FA = 0, FR = 16384, FI = 49152;

template <int STAGE>
__device__ __forceinline__ void batch(uint32_t sb, uint32_t d) {
  if constexpr (STAGE == 0) {  // A: data MN-major (LBO 8192) x FA K-major, N128
    constexpr uint32_t id = idesc(128, 128, true, false);
#pragma unroll
    for (uint32_t s = 0; s < 4; ++s)
      mma(d, desc(sb + SIN + s * 2048, 1024, 8192), desc(sb + SMAT + FA + s * 32, 1024), id, s);
  } else if constexpr (STAGE == 1 || STAGE == 2) {  // B / B': three-plane windows, N128
    constexpr uint32_t id = idesc(128, 128, false, true);
    const uint32_t fr = sb + SMAT + FR, fi = sb + SMAT + FI, p0 = sb + SOP, p1 = p0 + 16384;
#pragma unroll
    for (uint32_t s = 0; s < 8; ++s) {
      const uint32_t ko = (s >> 2) * 16384 + (s & 3) * 32;
      const uint64_t w0 = desc(p0 + s * 2048, 1024, 16384), w1 = desc(p1 + s * 2048, 1024, 16384);
      mma(d, desc(fr + ko, 1024), STAGE == 2 ? w0 : w1, id, s);
      mma(d, desc(fi + ko, 1024), STAGE == 2 ? w1 : w0, id, 1);
    }
  } else if constexpr (STAGE == 3) {  // A': data K-major x FA MN-major (LBO 1024), N64
    constexpr uint32_t id = idesc(128, 64, false, true);
#pragma unroll
    for (uint32_t s = 0; s < 8; ++s)
      mma(d, desc(sb + SOP + (s >> 2) * 16384 + (s & 3) * 32, 1024),
          desc(sb + SMAT + FA + s * 2048, 1024, 1024), id, s);
  } else if constexpr (STAGE == 4) {  // B variant: planes adjacent (LBO 1024 -> N128 contiguous 2 KB k-rows)
    constexpr uint32_t id = idesc(128, 128, false, true);
    const uint32_t fr = sb + SMAT + FR, fi = sb + SMAT + FI;
#pragma unroll
    for (uint32_t s = 0; s < 8; ++s) {
      const uint32_t ko = (s >> 2) * 16384 + (s & 3) * 32;
      mma(d, desc(fr + ko, 1024), desc(sb + SOP + s * 4096, 2048, 1024), id, s);
      mma(d, desc(fi + ko, 1024), desc(sb + SOP + 32768 + s * 4096, 2048, 1024), id, 1);
    }
  } else if constexpr (STAGE == 5) {  // B variant: two accumulators (d, d+128) alternate per MMA
    constexpr uint32_t id = idesc(128, 128, false, true);
    const uint32_t fr = sb + SMAT + FR, fi = sb + SMAT + FI, p0 = sb + SOP, p1 = p0 + 16384;
#pragma unroll
    for (uint32_t s = 0; s < 8; ++s) {
      const uint32_t ko = (s >> 2) * 16384 + (s & 3) * 32;
      mma(d, desc(fr + ko, 1024), desc(p1 + s * 2048, 1024, 16384), id, s);
      mma(d + 128, desc(fi + ko, 1024), desc(p0 + s * 2048, 1024, 16384), id, s);
    }
  } else {  // B variant: one MMA per k-step (Fr only), N128
    constexpr uint32_t id = idesc(128, 128, false, true);
    const uint32_t fr = sb + SMAT + FR, p1 = sb + SOP + 16384;
#pragma unroll
    for (uint32_t s = 0; s < 8; ++s) {
      const uint32_t ko = (s >> 2) * 16384 + (s & 3) * 32;
      mma(d, desc(fr + ko, 1024), desc(p1 + s * 2048, 1024, 16384), id, s);
    }
  }
}

template <int STAGE>
__global__ void k(unsigned long long* out, int reps) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[2];
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 210 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
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
    const unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {  // two batches in flight (two slots), waits on the older
      const int b = r & 1;
      batch<STAGE>(sb, t + 256 * b);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(&bar[b])) : "memory");
      if (r > 0) {
        asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&bar[b ^ 1])), "r"(ph[b ^ 1]) : "memory");
        ph[b ^ 1] ^= 1;
      }
    }
    const int w = (reps - 1) & 1;
    asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&bar[w])), "r"(ph[w]) : "memory");
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

template <int STAGE>
void run(unsigned long long* d, const char* name, int mmas, double floor) {
  cudaFuncSetAttribute(k<STAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  const int reps = 4000;
  k<STAGE><<<148, 128, 210 * 1024>>>(d, reps);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double c = (double)h / reps;
  printf("%-44s %7.1f cycles/batch (%d MMAs, floor %.0f: %5.1f%%) %s\n", name, c, mmas, floor,
         100 * floor / c, cudaGetErrorString(e));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 2000);
  run<0>(d, "A  (MN-major data LBO 8K x FA, N128)", 4, 4 * 64);
  run<1>(d, "B  (3-plane windows LBO 16K, N128, 1 acc)", 16, 16 * 64);
  run<2>(d, "B' (3-plane windows, N128, 1 acc)", 16, 16 * 64);
  run<3>(d, "A' (K-major data x FA MN-major, N64)", 8, 8 * 32);
  run<4>(d, "B  var: adjacent planes LBO 1K", 16, 16 * 64);
  run<5>(d, "B  var: 2 accumulators", 16, 16 * 64);
  run<6>(d, "B  var: Fr only (8 MMAs)", 8, 8 * 64);
  return 0;
}
