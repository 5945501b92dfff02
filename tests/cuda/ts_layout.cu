// probe (round 2): operand layout of tcgen05.mma kind::f16 with the A operand
// in TMEM (".ts"): lane m = row m, 32-bit column c of K-step s holds
// (k = 16 s + 2c, 16 s + 2c + 1) as a bf16 pair (low half = even k)?  B is an
// MN-major SW128 smem operand [k][n], N = 64.  Checks D = A.B for K = 32
// (two K-steps, A base advanced by 8 columns per step) against the host.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ts_layout ts_layout.cu
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int M = 128, N = 64, K = 32;

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t sbo, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;  // SW128
  return d;
}
__host__ __device__ constexpr uint32_t idesc(uint32_t m, uint32_t n, bool amn, bool bmn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((amn ? 1u : 0u) << 15) | ((bmn ? 1u : 0u) << 16) |
         ((n >> 3) << 17) | ((m >> 4) << 24);
}
__host__ __device__ inline uint32_t sw(uint32_t lin) { return lin ^ ((lin >> 3) & 0x70u); }
// MN-major, N = 64: [k/8][k%8][n] 128-byte rows
__host__ __device__ inline uint32_t boff(uint32_t k, uint32_t n) { return sw((k >> 3) * 1024 + (k & 7) * 128 + n * 2); }

__global__ void k(const float* A, const float* Bm, float* D) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < K * N; i += blockDim.x) {
    const int kk = i / N, n = i % N;
    *reinterpret_cast<__nv_bfloat16*>(sm + boff(kk, n)) = __float2bfloat16(Bm[kk * N + n]);
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot;
  // A into TMEM columns [128, 128 + K/2): thread = lane
  const uint32_t m = threadIdx.x;
  const uint32_t lane_addr = t + ((32u * (m >> 5)) << 16);
  uint32_t v[K / 2];
  for (int c = 0; c < K / 2; ++c) {
    __nv_bfloat162 h = __floats2bfloat162_rn(A[m * K + 2 * c], A[m * K + 2 * c + 1]);
    v[c] = *reinterpret_cast<uint32_t*>(&h);
  }
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
                   lane_addr + 128),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
               "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
               : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
    for (uint32_t s = 0; s < K / 16; ++s) {
      const uint64_t bd = desc(sb + s * 2048, 1024, 1024);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(t),
                   "r"(t + 128 + 8 * s), "l"(bd), "r"(idesc(M, N, false, true)), "r"(s));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&bar))
                 : "memory");
  }
  asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W_%=;\n\t}" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(&bar))
               : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(lane_addr + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) D[m * N + c0 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(t));
}

int main() {
  static float A[M * K], Bm[K * N], D[M * N];
  for (int i = 0; i < M * K; ++i) A[i] = (float)((i * 7 + 3) % 9 - 4);
  for (int i = 0; i < K * N; ++i) Bm[i] = (float)((i * 5 + 1) % 7 - 3);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, sizeof A);
  cudaMalloc(&dB, sizeof Bm);
  cudaMalloc(&dD, sizeof D);
  cudaMemcpy(dA, A, sizeof A, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, Bm, sizeof Bm, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<<<1, 128, 64 * 1024>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D, dD, sizeof D, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      float ref = 0;
      for (int kk = 0; kk < K; ++kk) ref += A[m * K + kk] * Bm[kk * N + n];
      if (ref != D[m * N + n] && bad++ < 8) printf("m=%d n=%d got %g want %g\n", m, n, D[m * N + n], ref);
    }
  printf("ts_layout: %s, %d mismatches of %d\n", cudaGetErrorString(e), bad, M * N);
  return bad != 0;
}
