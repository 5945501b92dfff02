// tcgen05 layout/descriptor probe: D[128][N] = A[128][K] * B[N][K]^T with
// bf16 K-major operands in SW32 / SW64 / SW128 layouts, checked against a
// host fp32 GEMM.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
//   -std=c++17 -I paper_2302_06646_b200/csrc tests/cuda/tc_probe.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "fb_tc.cuh"

using namespace fb;

template <int SWZ, int K, int N>
__global__ void probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t bar;
  constexpr uint32_t RB = tc::SwzTraits<SWZ>::row_bytes;
  static_assert(RB == K * 2, "row = K");
  unsigned char* sa = sm;
  unsigned char* sb = sm + 128 * RB;
  for (int i = threadIdx.x; i < 128 * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sa + tc::kmajor_off<SWZ>(r, k)) = A[i];
  }
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sb + tc::kmajor_off<SWZ>(r, k)) = B[i];
  }
  if (threadIdx.x < 32) tc::alloc<128>(&taddr_s);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t t = taddr_s;
  if (threadIdx.x == 0) {
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sa);
    const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(sb);
    const uint32_t sbo = tc::SwzTraits<SWZ>::atom;
    for (int ks = 0; ks < K / 16; ++ks) {
      const uint64_t ad = tc::smem_desc(a0 + ks * 32, sbo, SWZ);
      const uint64_t bd = tc::smem_desc(b0 + ks * 32, sbo, SWZ);
      tc::mma_bf16(t, ad, bd, tc::idesc_bf16(128, N), ks > 0);
    }
    tc::commit(&bar);
  }
  // wait
  asm volatile(
      "{\n\t.reg .pred P1;\nW:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
      "@!P1 bra W;\n\t}" ::"r"((uint32_t)__cvta_generic_to_shared(&bar))
      : "memory");
  tc::fence_after();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int c = 0; c < N; c += 32) {
    float v[32];
    tc::ld32(t + ((uint32_t)(warp * 32) << 16) + c, v);
    tc::ld_wait();
    for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * N + c + j] = v[j];
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::dealloc<128>(t);
}

template <int SWZ, int K, int N>
int run(const char* name) {
  std::vector<__nv_bfloat16> A(128 * K), B(N * K);
  std::vector<float> Af(128 * K), Bf(N * K), D(128 * N), R(128 * N, 0.f);
  srand(1);
  for (int i = 0; i < 128 * K; ++i) {
    Af[i] = (float)((rand() % 17) - 8) / 8.f;
    A[i] = __float2bfloat16(Af[i]);
  }
  for (int i = 0; i < N * K; ++i) {
    Bf[i] = (float)((rand() % 13) - 6) / 4.f;
    B[i] = __float2bfloat16(Bf[i]);
  }
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < K; ++k) R[m * N + n] += Af[m * K + k] * Bf[n * K + k];
  __nv_bfloat16 *dA, *dB;
  float* dD;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  const int smem = (128 + N) * K * 2 + 1024;
  cudaFuncSetAttribute(probe<SWZ, K, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<SWZ, K, N><<<1, 128, smem>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int i = 0; i < 128 * N; ++i) maxerr = fmax(maxerr, fabs(D[i] - R[i]));
  printf("%-6s K=%d N=%d: %s maxerr=%g  D[0]=%g R[0]=%g D[last]=%g R[last]=%g\n", name, K, N,
         cudaGetErrorString(e), maxerr, D[0], R[0], D[128 * N - 1], R[128 * N - 1]);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return maxerr < 1e-3 ? 0 : 1;
}

// A MN-major SW128 (M contiguous), full A is [256 m][K]; the MMA uses the
// M tile starting at m0 = 128 (two 64-m blocks in).  B K-major SW64 / SW128.
template <int K, int N, int BSWZ>
__global__ void probe_mn(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t bar;
  constexpr int MT = 256;
  unsigned char* sa = sm;                       // [K/8][MT/64][8][64]
  unsigned char* sb = sm + MT * K * 2;
  for (int i = threadIdx.x; i < MT * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sa + tc::mnmajor_off(m, k, MT)) = A[i];
  }
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sb + tc::kmajor_off<BSWZ>(r, k)) = B[i];
  }
  if (threadIdx.x < 32) tc::alloc<128>(&taddr_s);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t t = taddr_s;
  if (threadIdx.x == 0) {
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sa) + 2 * 1024;  // m0 = 128
    const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(sb);
    for (int ks = 0; ks < K / 16; ++ks) {
      const uint64_t ad = tc::smem_desc(a0 + ks * 2 * (MT / 64) * 1024, (MT / 64) * 1024, tc::kSw128, 1024);
      const uint64_t bd = tc::smem_desc(b0 + ks * 32, tc::SwzTraits<BSWZ>::atom, BSWZ);
      tc::mma_bf16(t, ad, bd, tc::idesc_bf16(128, N) | (1u << 15), ks > 0);
    }
    tc::commit(&bar);
  }
  asm volatile(
      "{\n\t.reg .pred P1;\nW2:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
      "@!P1 bra W2;\n\t}" ::"r"((uint32_t)__cvta_generic_to_shared(&bar))
      : "memory");
  tc::fence_after();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int c = 0; c < N; c += 32) {
    float v[32];
    tc::ld32(t + ((uint32_t)(warp * 32) << 16) + c, v);
    tc::ld_wait();
    for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * N + c + j] = v[j];
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::dealloc<128>(t);
}

template <int K, int N, int BSWZ>
int run_mn(const char* name) {
  constexpr int MT = 256;
  std::vector<__nv_bfloat16> A(MT * K), B(N * K);
  std::vector<float> Af(MT * K), Bf(N * K), D(128 * N), R(128 * N, 0.f);
  srand(2);
  for (int i = 0; i < MT * K; ++i) {
    Af[i] = (float)((rand() % 17) - 8) / 8.f;
    A[i] = __float2bfloat16(Af[i]);
  }
  for (int i = 0; i < N * K; ++i) {
    Bf[i] = (float)((rand() % 13) - 6) / 4.f;
    B[i] = __float2bfloat16(Bf[i]);
  }
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < K; ++k) R[m * N + n] += Af[(128 + m) * K + k] * Bf[n * K + k];
  __nv_bfloat16 *dA, *dB;
  float* dD;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  const int smem = (MT + N) * K * 2 + 1024;
  cudaFuncSetAttribute(probe_mn<K, N, BSWZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_mn<K, N, BSWZ><<<1, 128, smem>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int i = 0; i < 128 * N; ++i) maxerr = fmax(maxerr, fabs(D[i] - R[i]));
  printf("%-8s K=%d N=%d: %s maxerr=%g  D[0]=%g R[0]=%g\n", name, K, N, cudaGetErrorString(e),
         maxerr, D[0], R[0]);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return maxerr < 1e-3 ? 0 : 1;
}

int main() {
  int bad = 0;
  bad += run_mn<32, 32, tc::kSw64>("MN128a");
  bad += run_mn<16, 32, tc::kSw32>("MN128b");
  bad += run_mn<64, 64, tc::kSw128>("MN128c");
  bad += run<tc::kSw32, 16, 64>("SW32");
  bad += run<tc::kSw64, 32, 64>("SW64");
  bad += run<tc::kSw128, 64, 64>("SW128");
  bad += run<tc::kSw64, 32, 32>("SW64");
  bad += run<tc::kSw128, 64, 128>("SW128");
  printf(bad ? "PROBE FAIL\n" : "PROBE OK\n");
  return bad;
}
