// FlashButterfly-B200 three-pass engine (K3 forward, K4b backward, K1
// spectrum in the pass-2 layout) for transforms beyond shared memory:
// n = l * m with l = 8192 (the row length the single-pass machinery runs
// on-chip) and m in {2, 4, 8, 16} (n = 16K ... 128K, i.e. N = 8K ... 64K causal).
//
// Reference: conv_three_pass_ordered (proj/src/three_pass.cpp:225-254) with
// BlockDiagonalButterfly::apply (:101-122) as passes 1/3, middle_block
// (:211-221) as pass 2 and build_three_pass's d_k (:197-203) as the pass-2
// kernel spectrum.  With t = c*l + tau and f = a + m*s:
//   pass 1  X1[a][tau] = w_n^(-a tau) sum_c w_m^(-a c) x[c l + tau]
//           (m-point DFT down each column tau, then the twiddle)
//   pass 2  per row a: Z = FFT_l(X1[a]) = X[a + m s]; Z *= Kf2[a][s];
//           W[a] = IFFT_l(Z)   (Kf2[h][a][s] = K_hat[a + m s] / n)
//   pass 3  y[c l + tau] = sum_a w_m^(+a c) w_n^(+a tau) W[a][tau]
// The reference's B^T / B^-1^T factors are exactly passes 1 and 3 (entry
// exp(-2 pi i k (j l + tau)/n), three_pass.hpp:71-75); its d_k = l K_hat
// permuted is Kf2 up to the 1/(l n) normalisation folded here.
// Each pass streams the buffer once with coalesced, vectorised accesses:
// passes 1/3 give one column tau per thread (consecutive threads =
// consecutive tau), pass 2 moves whole rows by TMA bulk copies.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "fb_common.cuh"
#include "fb_fft.cuh"
#include "fb_internal.h"
#include "fb_ptx.cuh"

namespace fb {

constexpr int kL2 = 13;  // log2(l)
constexpr uint32_t kL = 1u << kL2;
constexpr int kColThreads = 256;

// complex storage element of the intermediates
template <typename ST>
struct CxT {
  ST x, y;
};

// ---------------------------------------------------------------- pass 1
// grid (l/256, H, npairs [or 1 for the kernel spectrum]).  SRC: 0 = signal
// pairs (real channels b0, b1 -> re, im); 1 = two signals (dy, u) at once
// with the dD partial; 2 = the regularized kernel bank (fp32, one channel).
template <typename IO, typename ST, int M, int SRC>
__global__ void __launch_bounds__(kColThreads)
    tp_pass1_kernel(const IO* __restrict__ a_in, const IO* __restrict__ b_in,
                    const float* __restrict__ kbar, CxT<ST>* __restrict__ out_a,
                    CxT<ST>* __restrict__ out_b, float* __restrict__ ddpart,
                    const float2* __restrict__ tab_g, int B, int H, uint32_t N, int causal) {
  __shared__ float red[kColThreads / 32];
  const uint32_t tau = blockIdx.x * kColThreads + threadIdx.x;
  const int h = blockIdx.y, pr = blockIdx.z;
  const int b0 = 2 * pr, b1 = b0 + 1;
  const bool has1 = b1 < B;
  constexpr int MH = M;  // rows that can hold data
  const int cmax = causal ? M / 2 : M;
  float dd = 0.f;
  auto column = [&](const IO* src, float2 (&v)[M]) {
    const IO* r0 = src + ((size_t)b0 * H + h) * N;
    const IO* r1 = src + ((size_t)b1 * H + h) * N;
#pragma unroll
    for (int c = 0; c < MH; ++c) {
      const uint32_t t = c * kL + tau;
      const bool ok = c < cmax && t < N;
      v[c].x = ok ? ld(r0 + t) : 0.f;
      v[c].y = (ok && has1) ? ld(r1 + t) : 0.f;
    }
  };
  float2 v[M];
  if constexpr (SRC == 2) {
    const float* kr = kbar + (size_t)h * N;
#pragma unroll
    for (int c = 0; c < M; ++c) {
      const uint32_t t = c * kL + tau;
      v[c] = make_float2((c < cmax && t < N) ? __ldg(kr + t) : 0.f, 0.f);
    }
  } else {
    column(a_in, v);
  }
  if constexpr (SRC == 1) {
    float2 w[M];
    column(b_in, w);
#pragma unroll
    for (int c = 0; c < M; ++c) dd = fmaf(v[c].x, w[c].x, fmaf(v[c].y, w[c].y, dd));
    dft_reg<-1, M>(w);
    apply_tw_g<-1, M>(w, tab_g, tau);
    CxT<ST>* ob = out_b + ((size_t)pr * H + h) * (size_t)M * kL;
#pragma unroll
    for (int a = 0; a < M; ++a) stc<ST>(&ob[a * kL + tau].x, w[a]);
  }
  dft_reg<-1, M>(v);
  apply_tw_g<-1, M>(v, tab_g, tau);
  CxT<ST>* oa = out_a + ((size_t)pr * H + h) * (size_t)M * kL;
#pragma unroll
  for (int a = 0; a < M; ++a) stc<ST>(&oa[a * kL + tau].x, v[a]);
  if constexpr (SRC == 1) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dd += __shfl_xor_sync(0xffffffffu, dd, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dd;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (int w = 0; w < kColThreads / 32; ++w) t += red[w];
      ddpart[((size_t)h * gridDim.z + pr) * gridDim.x + blockIdx.x] = t;
    }
  }
}

// ---------------------------------------------------------------- pass 2
template <typename ST>
__device__ __forceinline__ void stage_row(CxT<ST>* dst, const CxT<ST>* src, uint64_t* bar) {
  if (threadIdx.x == 0) {
    constexpr uint32_t bytes = kL * sizeof(CxT<ST>);
    ptx::fence_proxy_async_smem();
    ptx::mbar_arrive_expect_tx(bar, bytes);
    ptx::bulk_g2s(dst, src, bytes, bar);
  }
}

__device__ __forceinline__ float2 cx_load(const CxT<float>* p) { return *reinterpret_cast<const float2*>(p); }
__device__ __forceinline__ float2 cx_load(const CxT<__nv_bfloat16>* p) {
  return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p));
}
__device__ __forceinline__ float2 cx_load(const CxT<__half>* p) {
  return __half22float2(*reinterpret_cast<const __half2*>(p));
}

// MODE 0: forward rows  W = IFFT(FFT(X1 row) * Kf2[h][a])   (in place)
// MODE 1: spectrum      Kf2[h][a] = FFT(X1k row) / n
// grid (H*m, chunks); rows of pair pr: X1[((pr*H + h)*m + a)*l ...].
template <typename ST, int MODE>
__global__ void __launch_bounds__(kL / 16, 1)
    tp_pass2_kernel(CxT<ST>* __restrict__ x1, const float2* __restrict__ kf2,
                    float2* kf2_out, const float2* __restrict__ tab_g, int npairs,
                    int H, int m, int ppc, float inv_n, CxT<ST>* __restrict__ usave = nullptr) {
  using S = FftShape<kL2>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[2];
  // k_f row staged in smem for 16-bit storage; fp32 rows need the room for
  // the double-buffered stage, so k_f is read through L2 there.
  constexpr bool KF_SMEM = sizeof(ST) < 4;
  float2* work = reinterpret_cast<float2*>(smem_raw);
  float2* kfs = work + S::work_len;
  float2* tab = kfs + (KF_SMEM ? S::n : 0);
  CxT<ST>* stage = reinterpret_cast<CxT<ST>*>(tab + ((S::tab_len + 1) & ~1u));  // [2][l]
  const int ha = blockIdx.x, h = ha / m, a = ha % m;
  const uint32_t j = threadIdx.x;
  const float2* kfg = kf2 + (size_t)ha * S::n;
  const int p0 = blockIdx.y * ppc, p1 = min(npairs, p0 + ppc);
  if (p0 >= p1) return;
  if (j == 0) {
    ptx::mbar_init(&bars[0], 1);
    ptx::mbar_init(&bars[1], 1);
    ptx::fence_barrier_init();
  }
  for (uint32_t i = j; i < S::tab_len; i += S::T) tab[i] = __ldg(tab_g + i);
  if constexpr (MODE == 0 && KF_SMEM) {
    const float4* src = reinterpret_cast<const float4*>(kfg);
    float4* dst = reinterpret_cast<float4*>(kfs);
    for (uint32_t i = j; i < S::n / 2; i += S::T) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  auto row_ptr = [&](int pr) { return x1 + ((size_t)pr * H + h) * (size_t)m * kL + (size_t)a * kL; };
  stage_row<ST>(stage, row_ptr(p0), &bars[0]);
  for (int pr = p0, it = 0; pr < p1; ++pr, ++it) {
    const int buf = it & 1;
    ptx::mbar_wait(&bars[buf], (it >> 1) & 1);
    if (pr + 1 < p1) stage_row<ST>(stage + (buf ^ 1) * kL, row_ptr(pr + 1), &bars[buf ^ 1]);
    const CxT<ST>* srow = stage + buf * kL;
    float2 v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = cx_load(srow + j + r * S::stride);
    dft_reg<-1, 16>(v);
    bfly_store<16, 1>(work, v, j);
    __syncthreads();
    mid_passes<-1, kL2, 16>(work, tab);
    bfly_load<-1, 16, S::n / 16, kL2>(work, tab, v, j);
    if constexpr (MODE == 1) {
      float2* out = kf2_out + (size_t)ha * S::n;
#pragma unroll
      for (int r = 0; r < 16; ++r) out[j + r * S::stride] = cscale(v[r], inv_n);
    } else {
      if (usave) {  // the row spectrum, kept for the backward (training step)
        CxT<ST>* us = usave + ((size_t)pr * H + h) * (size_t)m * kL + (size_t)a * kL;
#pragma unroll
        for (int r = 0; r < 16; ++r) stc<ST>(&us[j + r * S::stride].x, v[r]);
      }
#pragma unroll
      for (int r = 0; r < 16; ++r)
        v[r] = cmul(v[r], KF_SMEM ? kfs[j + r * S::stride] : __ldg(kfg + j + r * S::stride));
      dft_reg<+1, 16>(v);
      __syncthreads();
      bfly_store<16, 1>(work, v, j);
      __syncthreads();
      mid_passes<+1, kL2, 16>(work, tab);
      bfly_load<+1, 16, S::n / 16, kL2>(work, tab, v, j);
      CxT<ST>* orow = row_ptr(pr);
#pragma unroll
      for (int r = 0; r < 16; ++r) stc<ST>(&orow[j + r * S::stride].x, v[r]);
    }
    __syncthreads();
  }
}

// Backward middle pass, CTA (h, a) over ALL pairs (so the dK spectrum of row
// a is complete in one CTA, fixed order => deterministic):
//   DY = FFT(X1dy), U = FFT(X1u); acc += conj(U) DY; X1dy <- IFFT(DY conj(Kf2))
//   finally wdk[h][a] = IFFT(acc)  (fp32)
// SAVED: x1u holds the forward's row spectra FFT_l(X1u row) (tp_pass2_kernel
// usave) instead of the rows, so each pair costs two transforms, not three.
template <typename ST, bool SAVED = false>
__global__ void __launch_bounds__(kL / 16, 1)
    tp_pass2_bwd_kernel(CxT<ST>* __restrict__ x1dy, const CxT<ST>* __restrict__ x1u,
                        const float2* __restrict__ kf2, float2* __restrict__ wdk,
                        const float2* __restrict__ tab_g, int npairs, int H, int m) {
  using S = FftShape<kL2>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[1];
  float2* work = reinterpret_cast<float2*>(smem_raw);
  float2* acc = work + S::work_len;
  float2* tab = acc + S::n;
  CxT<ST>* stage = reinterpret_cast<CxT<ST>*>(tab + ((S::tab_len + 1) & ~1u));  // [l]
  const int ha = blockIdx.x, h = ha / m, a = ha % m;
  const uint32_t j = threadIdx.x;
  const float2* kh = kf2 + (size_t)ha * S::n;
  if (j == 0) {
    ptx::mbar_init(&bars[0], 1);
    ptx::fence_barrier_init();
  }
  for (uint32_t i = j; i < S::tab_len; i += S::T) tab[i] = __ldg(tab_g + i);
#pragma unroll
  for (int r = 0; r < 16; ++r) acc[j + r * S::stride] = make_float2(0.f, 0.f);
  __syncthreads();
  auto rp = [&](const CxT<ST>* base, int pr) {
    return base + ((size_t)pr * H + h) * (size_t)m * kL + (size_t)a * kL;
  };
  uint32_t phase = 0;
  if (npairs > 0) stage_row<ST>(stage, rp(x1dy, 0), &bars[0]);
  for (int pr = 0; pr < npairs; ++pr) {
    float2 gv[16], v[16];
    ptx::mbar_wait(&bars[0], phase);
    phase ^= 1;
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = cx_load(stage + j + r * S::stride);
    __syncthreads();  // stage consumed
    if constexpr (SAVED) {
      if (pr + 1 < npairs) stage_row<ST>(stage, rp(x1dy, pr + 1), &bars[0]);
    } else {
      stage_row<ST>(stage, rp(x1u, pr), &bars[0]);
    }
    dft_reg<-1, 16>(v);
    bfly_store<16, 1>(work, v, j);
    __syncthreads();
    mid_passes<-1, kL2, 16>(work, tab);
    bfly_load<-1, 16, S::n / 16, kL2>(work, tab, gv, j);
    if constexpr (SAVED) {
      const CxT<ST>* us = rp(x1u, pr);
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = cx_load(us + j + r * S::stride);
    } else {
      ptx::mbar_wait(&bars[0], phase);
      phase ^= 1;
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = cx_load(stage + j + r * S::stride);
      dft_reg<-1, 16>(v);
      __syncthreads();
      if (pr + 1 < npairs) stage_row<ST>(stage, rp(x1dy, pr + 1), &bars[0]);
      bfly_store<16, 1>(work, v, j);
      __syncthreads();
      mid_passes<-1, kL2, 16>(work, tab);
      bfly_load<-1, 16, S::n / 16, kL2>(work, tab, v, j);
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t e = j + r * S::stride;
      acc[e] = cadd(acc[e], cconjmul(v[r], gv[r]));
      v[r] = cmulc(gv[r], __ldg(kh + e));
    }
    dft_reg<+1, 16>(v);
    __syncthreads();
    bfly_store<16, 1>(work, v, j);
    __syncthreads();
    mid_passes<+1, kL2, 16>(work, tab);
    bfly_load<+1, 16, S::n / 16, kL2>(work, tab, v, j);
    CxT<ST>* orow = const_cast<CxT<ST>*>(rp(x1dy, pr));
#pragma unroll
    for (int r = 0; r < 16; ++r) stc<ST>(&orow[j + r * S::stride].x, v[r]);
    __syncthreads();
  }
  // dK spectrum row -> IFFT_l -> wdk (fp32)
  float2 v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = acc[j + r * S::stride];
  dft_reg<+1, 16>(v);
  __syncthreads();
  bfly_store<16, 1>(work, v, j);
  __syncthreads();
  mid_passes<+1, kL2, 16>(work, tab);
  bfly_load<+1, 16, S::n / 16, kL2>(work, tab, v, j);
  float2* orow = wdk + (size_t)ha * S::n;
#pragma unroll
  for (int r = 0; r < 16; ++r) orow[j + r * S::stride] = v[r];
}

// ---------------------------------------------------------------- pass 3
// MODE 0: signal pairs -> out[b][h][t] = y + D * skip[b][h][t]
// MODE 1: dK row per head (fp32 complex) -> dkbar[h][t] = Re(.) * scale
template <typename ST, typename IO, int M, int MODE>
__global__ void __launch_bounds__(kColThreads)
    tp_pass3_kernel(const CxT<ST>* __restrict__ w_in, const IO* __restrict__ skip,
                    IO* __restrict__ out, const float* __restrict__ D, float* __restrict__ dkbar,
                    const float2* __restrict__ tab_g, int B, int H, uint32_t N, int causal,
                    float scale) {
  const uint32_t tau = blockIdx.x * kColThreads + threadIdx.x;
  const int h = blockIdx.y, pr = blockIdx.z;
  float2 v[M];
  const CxT<ST>* src = w_in + ((size_t)pr * H + h) * (size_t)M * kL;
#pragma unroll
  for (int a = 0; a < M; ++a) v[a] = cx_load(src + a * kL + tau);
  apply_tw_g<+1, M>(v, tab_g, tau);
  dft_reg<+1, M>(v);
  const int cmax = causal ? M / 2 : M;
  if constexpr (MODE == 0) {
    const int b0 = 2 * pr, b1 = b0 + 1;
    const bool has1 = b1 < B;
    const float d = __ldg(D + h);
    const size_t o0 = ((size_t)b0 * H + h) * N, o1 = ((size_t)b1 * H + h) * N;
#pragma unroll
    for (int c = 0; c < M; ++c) {
      const uint32_t t = c * kL + tau;
      if (c < cmax && t < N) {
        st(out + o0 + t, fmaf(d, ld(skip + o0 + t), v[c].x));
        if (has1) st(out + o1 + t, fmaf(d, ld(skip + o1 + t), v[c].y));
      }
    }
  } else {
#pragma unroll
    for (int c = 0; c < M; ++c) {
      const uint32_t t = c * kL + tau;
      if (c < cmax && t < N) dkbar[(size_t)h * N + t] = v[c].x * scale;
    }
  }
}

// ---------------------------------------------------------------- streaming column passes
// Passes 1 and 3 for m <= 16 as persistent streaming kernels: a CTA walks
// tiles of TB = 256 columns tau of one (pair, head); each tile's input rows
// arrive by 3-D TMA boxes into a ring of smem stages (kColStages tiles in
// flight per CTA), so HBM latency is hidden behind the other tiles instead of
// each thread's 16 dependent loads.  Thread j owns column tau = tile + j:
// column DFT + twiddle in registers, coalesced stores.
constexpr uint32_t kTB = 256;  // columns per tile (= threads)
constexpr int kColMaxStages = 4;

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];" ::"r"(ptx::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(ptx::smem_u32(bar))
      : "memory");
}

// tile t -> (pair, head, column block): column blocks fastest
struct ColTile {
  int pr, h, tb;
};
__device__ __forceinline__ ColTile col_tile(int t, int H) {
  constexpr int NB = kL / kTB;
  ColTile c;
  c.tb = t % NB;
  c.h = (t / NB) % H;
  c.pr = t / (NB * H);
  return c;
}

// Producer / consumer ring shared by the streaming column kernels: warp
// kCons / 32 only issues the TMA boxes (waiting on the per-stage "empty"
// barriers), the kCons consumer threads wait on "full", copy their two
// adjacent columns to registers, release the stage at once and compute — the
// TMA issue is never on a consumer warp's critical path, and every load and
// store moves a column pair (half the memory instructions of one column per
// thread).
constexpr uint32_t kCons = kTB / 2;

__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ptx::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kCons) : "memory");
}
template <class Issue>
__device__ __forceinline__ void col_producer(int first, int step, int ntiles, int nstages,
                                             uint64_t* empty, Issue&& issue) {
  if (threadIdx.x != kCons) return;
  int k = 0;
  for (int t = first; t < ntiles; t += step, ++k) {
    const int sg = k % nstages;
    if (k >= nstages) ptx::mbar_wait(&empty[sg], (uint32_t)((k / nstages) - 1) & 1);
    issue(t, sg);
  }
}

// two consecutive elements (column pair) in / out
__device__ __forceinline__ float2 ld2s(const float* p) { return *reinterpret_cast<const float2*>(p); }
__device__ __forceinline__ float2 ld2s(const __nv_bfloat16* p) {
  return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p));
}
__device__ __forceinline__ float2 ld2s(const __half* p) {
  return __half22float2(*reinterpret_cast<const __half2*>(p));
}
__device__ __forceinline__ void st2(float* p, float a, float b) {
  *reinterpret_cast<float2*>(p) = make_float2(a, b);
}
__device__ __forceinline__ void st2(__nv_bfloat16* p, float a, float b) {
  *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(a, b);
}
__device__ __forceinline__ void st2(__half* p, float a, float b) {
  *reinterpret_cast<__half2*>(p) = __floats2half2_rn(a, b);
}
__device__ __forceinline__ void st4(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}
__device__ __forceinline__ void st4(__nv_bfloat16* p, float a, float b, float c, float d) {
  const __nv_bfloat162 x = __floats2bfloat162_rn(a, b), y = __floats2bfloat162_rn(c, d);
  *reinterpret_cast<uint2*>(p) =
      make_uint2(*reinterpret_cast<const uint32_t*>(&x), *reinterpret_cast<const uint32_t*>(&y));
}
__device__ __forceinline__ void st4(__half* p, float a, float b, float c, float d) {
  const __half2 x = __floats2half2_rn(a, b), y = __floats2half2_rn(c, d);
  *reinterpret_cast<uint2*>(p) =
      make_uint2(*reinterpret_cast<const uint32_t*>(&x), *reinterpret_cast<const uint32_t*>(&y));
}
// two consecutive complex elements
__device__ __forceinline__ void cx_load2(const CxT<float>* p, float2& a, float2& b) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  a = make_float2(v.x, v.y);
  b = make_float2(v.z, v.w);
}
template <typename H2>
__device__ __forceinline__ float2 h2f(uint32_t v);
template <>
__device__ __forceinline__ float2 h2f<__nv_bfloat16>(uint32_t v) {
  return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&v));
}
template <>
__device__ __forceinline__ float2 h2f<__half>(uint32_t v) {
  return __half22float2(*reinterpret_cast<__half2*>(&v));
}
template <typename T>
__device__ __forceinline__ void cx_load2(const CxT<T>* p, float2& a, float2& b) {
  const uint2 v = *reinterpret_cast<const uint2*>(p);
  a = h2f<T>(v.x);
  b = h2f<T>(v.y);
}

// Pass 1, SRC 0: signal pairs (channels 2 pr, 2 pr + 1 -> re, im);
// SRC 1: dy and u pairs at once, plus the lag-0 dD partial.  Signal maps view
// [B*H][rows][l] with rows = N / l data rows (the causal pad is implicit).
// PLANAR: rows leave as [re l | im l] (the tcgen05 row pass's TMA layout)
template <typename IO, typename ST, int M, int SRC, bool PLANAR = false>
__global__ void __launch_bounds__(kCons + 32)
    tp_col1_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                   CxT<ST>* __restrict__ out_a, CxT<ST>* __restrict__ out_b,
                   float* __restrict__ ddpart, const float2* __restrict__ tab_g, int H, int npairs,
                   int rows, int ntiles, int nstages) {
  extern __shared__ __align__(128) unsigned char csm[];
  __shared__ __align__(8) uint64_t full[kColMaxStages], empty[kColMaxStages];
  __shared__ float red[2][kCons / 32];
  constexpr int NCH = SRC == 1 ? 4 : 2;
  const uint32_t chb = (uint32_t)rows * kTB * sizeof(IO);
  const uint32_t stage_bytes = NCH * chb;
  const int j = threadIdx.x;
  if (j == 0) {
    for (int i = 0; i < nstages; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], kCons);
    }
    ptx::fence_barrier_init();
  }
  __syncthreads();
  const int first = blockIdx.x, step = gridDim.x;
  if (j >= (int)kCons) {
    col_producer(first, step, ntiles, nstages, empty, [&](int t, int st) {
      const ColTile c = col_tile(t, H);
      unsigned char* dst = csm + (size_t)st * stage_bytes;
      ptx::mbar_arrive_expect_tx(&full[st], stage_bytes);
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        const CUtensorMap* mp = (SRC == 1 && ch >= 2) ? &bmap : &amap;
        const int b = 2 * c.pr + (ch & 1);
        tma_load_3d(dst + ch * chb, mp, c.tb * (int)kTB, 0, b * H + c.h, &full[st]);
      }
    });
    return;
  }
  int it = 0;
  for (int t = first; t < ntiles; t += step, ++it) {
    const int sg = it % nstages;
    ptx::mbar_wait(&full[sg], (uint32_t)(it / nstages) & 1);
    const ColTile c = col_tile(t, H);
    const uint32_t tau = c.tb * kTB + 2 * j;
    const IO* sv = reinterpret_cast<const IO*>(csm + (size_t)sg * stage_bytes);
    // columns tau (v0) and tau + 1 (v1) of the channel pair (ch0, ch0 + 1)
    auto columns = [&](int ch0, float2 (&v0)[M], float2 (&v1)[M]) {
#pragma unroll
      for (int r = 0; r < M; ++r) {
        const bool ok = r < rows;
        const float2 a = ok ? ld2s(sv + (ch0 * rows + r) * kTB + 2 * j) : make_float2(0.f, 0.f);
        const float2 b = ok ? ld2s(sv + ((ch0 + 1) * rows + r) * kTB + 2 * j) : make_float2(0.f, 0.f);
        v0[r] = make_float2(a.x, b.x);
        v1[r] = make_float2(a.y, b.y);
      }
    };
    float2 v0[M], v1[M];
    columns(0, v0, v1);
    float dd = 0.f;
    float2 w0[SRC == 1 ? M : 1], w1[SRC == 1 ? M : 1];
    if constexpr (SRC == 1) columns(2, w0, w1);
    mbar_arrive_cta(&empty[sg]);  // this thread's reads of the stage are done
    auto put = [&](CxT<ST>* o, const float2 (&x0)[M], const float2 (&x1)[M]) {
      if constexpr (PLANAR) {
#pragma unroll
        for (int a = 0; a < M; ++a) {
          ST* r = reinterpret_cast<ST*>(o + a * kL);
          st2(r + tau, x0[a].x, x1[a].x);
          st2(r + kL + tau, x0[a].y, x1[a].y);
        }
      } else {
#pragma unroll
        for (int a = 0; a < M; ++a)
          st4(&o[a * kL + tau].x, x0[a].x, x0[a].y, x1[a].x, x1[a].y);
      }
    };
    if constexpr (SRC == 1) {
#pragma unroll
      for (int r = 0; r < M; ++r) {
        dd = fmaf(v0[r].x, w0[r].x, fmaf(v0[r].y, w0[r].y, dd));
        dd = fmaf(v1[r].x, w1[r].x, fmaf(v1[r].y, w1[r].y, dd));
      }
      dft_reg<-1, M>(w0);
      apply_tw_g<-1, M>(w0, tab_g, tau);
      dft_reg<-1, M>(w1);
      apply_tw_g<-1, M>(w1, tab_g, tau + 1);
      put(out_b + ((size_t)c.pr * H + c.h) * (size_t)M * kL, w0, w1);
    }
    dft_reg<-1, M>(v0);
    apply_tw_g<-1, M>(v0, tab_g, tau);
    dft_reg<-1, M>(v1);
    apply_tw_g<-1, M>(v1, tab_g, tau + 1);
    put(out_a + ((size_t)c.pr * H + c.h) * (size_t)M * kL, v0, v1);
    if constexpr (SRC == 1) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dd += __shfl_xor_sync(0xffffffffu, dd, o);
      if ((j & 31) == 0) red[it & 1][j >> 5] = dd;
      consumers_sync();  // red[it & 1] complete (double-buffered by tile parity)
      if (j == 0) {
        float s = 0.f;
        for (int w2 = 0; w2 < (int)(kCons / 32); ++w2) s += red[it & 1][w2];
        ddpart[((size_t)c.h * npairs + c.pr) * (kL / kTB) + c.tb] = s;
      }
    }
  }
}

// Pass 3 (MODE 0): W rows [pair*H + h][M][l] (complex ST) -> out[b][h][c l + tau]
// = Re/Im(column IDFT) + D[h] skip[b][h][c l + tau], c < rows.
template <typename ST, typename IO, int M>
__global__ void __launch_bounds__(kCons + 32)
    tp_col3_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap smap,
                   IO* __restrict__ out, const float* __restrict__ D,
                   const float2* __restrict__ tab_g, int B, int H, uint32_t N, int rows, int ntiles,
                   int nstages) {
  extern __shared__ __align__(128) unsigned char csm[];
  __shared__ __align__(8) uint64_t full[kColMaxStages], empty[kColMaxStages];
  const uint32_t wb = M * kTB * sizeof(CxT<ST>);
  const uint32_t chb = (uint32_t)rows * kTB * sizeof(IO);
  const uint32_t stage_bytes = wb + 2 * chb;
  const int j = threadIdx.x;
  if (j == 0) {
    for (int i = 0; i < nstages; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], kCons);
    }
    ptx::fence_barrier_init();
  }
  __syncthreads();
  const int first = blockIdx.x, step = gridDim.x;
  if (j >= (int)kCons) {
    col_producer(first, step, ntiles, nstages, empty, [&](int t, int st) {
      const ColTile c = col_tile(t, H);
      unsigned char* dst = csm + (size_t)st * stage_bytes;
      ptx::mbar_arrive_expect_tx(&full[st], stage_bytes);
      tma_load_3d(dst, &wmap, c.tb * (int)kTB, 0, c.pr * H + c.h, &full[st]);
#pragma unroll
      for (int ch = 0; ch < 2; ++ch)
        tma_load_3d(dst + wb + ch * chb, &smap, c.tb * (int)kTB, 0, (2 * c.pr + ch) * H + c.h,
                    &full[st]);
    });
    return;
  }
  int it = 0;
  for (int t = first; t < ntiles; t += step, ++it) {
    const int sg = it % nstages;
    ptx::mbar_wait(&full[sg], (uint32_t)(it / nstages) & 1);
    const ColTile c = col_tile(t, H);
    const uint32_t tau = c.tb * kTB + 2 * j;
    const unsigned char* base = csm + (size_t)sg * stage_bytes;
    const CxT<ST>* sw = reinterpret_cast<const CxT<ST>*>(base);
    const IO* sk = reinterpret_cast<const IO*>(base + wb);
    float2 v0[M], v1[M];
#pragma unroll
    for (int a = 0; a < M; ++a) cx_load2(sw + a * kTB + 2 * j, v0[a], v1[a]);
    float2 s0[M], s1[M];  // skip of channels b0 / b1 at (tau, tau + 1)
#pragma unroll
    for (int r = 0; r < M; ++r) {
      s0[r] = r < rows ? ld2s(sk + r * kTB + 2 * j) : make_float2(0.f, 0.f);
      s1[r] = r < rows ? ld2s(sk + (rows + r) * kTB + 2 * j) : make_float2(0.f, 0.f);
    }
    mbar_arrive_cta(&empty[sg]);
    apply_tw_g<+1, M>(v0, tab_g, tau);
    dft_reg<+1, M>(v0);
    apply_tw_g<+1, M>(v1, tab_g, tau + 1);
    dft_reg<+1, M>(v1);
    const int b0 = 2 * c.pr, b1 = b0 + 1;
    const bool has1 = b1 < B;
    const float d = __ldg(D + c.h);
    const size_t o0 = ((size_t)b0 * H + c.h) * N, o1 = ((size_t)b1 * H + c.h) * N;
#pragma unroll
    for (int r = 0; r < M; ++r) {
      if (r < rows) {
        const uint32_t tt = r * kL + tau;
        st2(out + o0 + tt, fmaf(d, s0[r].x, v0[r].x), fmaf(d, s0[r].y, v1[r].x));
        if (has1) st2(out + o1 + tt, fmaf(d, s1[r].x, v0[r].y), fmaf(d, s1[r].y, v1[r].y));
      }
    }
  }
}

__global__ void tp_dd_reduce_kernel(const float* __restrict__ ddpart, float* __restrict__ dD,
                                    int per_head) {
  const int h = blockIdx.x;
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int i = 0; i < per_head; ++i) t += ddpart[(size_t)h * per_head + i];
    dD[h] = t;
  }
}

// ---------------------------------------------------------------- passes 1/3, m > 16
// A CTA owns TAU = 8192/m consecutive columns tau and all m rows: the tile
// (m x TAU complex, fp32) is staged in shared memory with coalesced row
// segments, the TAU independent m-point DFTs run as batched Stockham passes
// (element e of column c at s[pad16(e) * TAU + c]), and the w_n^(a tau)
// twiddle is applied on the way out (pass 1) / in (pass 3) from a two-level
// table  w_n^t = lo[t & 4095] * hi[t >> 12].
constexpr uint32_t kBigTile = 8192;  // complex elements per tile
constexpr uint32_t kBigThreads = kBigTile / 16;

template <int SIGN>
__device__ __forceinline__ float2 tw_big(const float2* __restrict__ tb, uint32_t t) {
  const float2 w = cmul(__ldg(tb + (t & 4095u)), __ldg(tb + 4096u + (t >> 12)));
  return SIGN < 0 ? w : make_float2(w.x, -w.y);
}

template <typename IO, typename ST, int SMALL, int SRC>
__global__ void __launch_bounds__(kBigThreads, 1)
    tp_pass1_big_kernel(const IO* __restrict__ a_in, const IO* __restrict__ b_in,
                        const float* __restrict__ kbar, CxT<ST>* __restrict__ out_a,
                        CxT<ST>* __restrict__ out_b, float* __restrict__ ddpart,
                        const float2* __restrict__ tw_m, const float2* __restrict__ tb, int B,
                        int H, uint32_t N, int causal, uint32_t m) {
  extern __shared__ __align__(16) float2 tsm[];
  __shared__ float red[kBigThreads / 32];
  const uint32_t TAU = kBigTile / m;
  const uint32_t plen = padded_len(m) * TAU;
  float2* sa = tsm;
  float2* sb = tsm + plen;
  const uint32_t tau0 = blockIdx.x * TAU;
  const int h = blockIdx.y, pr = blockIdx.z;
  const int b0 = 2 * pr, b1 = b0 + 1;
  const bool has1 = b1 < B;
  const uint32_t cmax = causal ? m / 2 : m;
  float dd = 0.f;
  for (uint32_t i = threadIdx.x; i < kBigTile; i += kBigThreads) {
    const uint32_t e = pdiv(i, TAU), c = pmod(i, TAU);
    const uint32_t t = e * kL + tau0 + c;
    const bool ok = e < cmax && t < N;
    float2 v = make_float2(0.f, 0.f), w = make_float2(0.f, 0.f);
    if constexpr (SRC == 2) {
      v.x = ok ? __ldg(kbar + (size_t)h * N + t) : 0.f;
    } else {
      const size_t o0 = ((size_t)b0 * H + h) * N, o1 = ((size_t)b1 * H + h) * N;
      v.x = ok ? ld(a_in + o0 + t) : 0.f;
      v.y = (ok && has1) ? ld(a_in + o1 + t) : 0.f;
      if constexpr (SRC == 1) {
        w.x = ok ? ld(b_in + o0 + t) : 0.f;
        w.y = (ok && has1) ? ld(b_in + o1 + t) : 0.f;
        dd = fmaf(v.x, w.x, fmaf(v.y, w.y, dd));
        sb[pad16(e) * TAU + c] = w;
      }
    }
    sa[pad16(e) * TAU + c] = v;
  }
  __syncthreads();
  smem_passes<-1, SMALL>(sa, m, TAU, 1, m, tw_m);
  if constexpr (SRC == 1) smem_passes<-1, SMALL>(sb, m, TAU, 1, m, tw_m);
  CxT<ST>* oa = out_a + ((size_t)pr * H + h) * (size_t)m * kL;
  CxT<ST>* ob = SRC == 1 ? out_b + ((size_t)pr * H + h) * (size_t)m * kL : nullptr;
  for (uint32_t i = threadIdx.x; i < kBigTile; i += kBigThreads) {
    const uint32_t a = pdiv(i, TAU), c = pmod(i, TAU);
    const float2 w = tw_big<-1>(tb, a * (tau0 + c));
    stc<ST>(&oa[(size_t)a * kL + tau0 + c].x, cmul(sa[pad16(a) * TAU + c], w));
    if constexpr (SRC == 1) stc<ST>(&ob[(size_t)a * kL + tau0 + c].x, cmul(sb[pad16(a) * TAU + c], w));
  }
  if constexpr (SRC == 1) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dd += __shfl_xor_sync(0xffffffffu, dd, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dd;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (uint32_t w = 0; w < kBigThreads / 32; ++w) t += red[w];
      ddpart[((size_t)h * gridDim.z + pr) * gridDim.x + blockIdx.x] = t;
    }
  }
}

template <typename ST, typename IO, int SMALL, int MODE>
__global__ void __launch_bounds__(kBigThreads, 1)
    tp_pass3_big_kernel(const CxT<ST>* __restrict__ w_in, const IO* __restrict__ skip,
                        IO* __restrict__ out, const float* __restrict__ D,
                        float* __restrict__ dkbar, const float2* __restrict__ tw_m,
                        const float2* __restrict__ tb, int B, int H, uint32_t N, int causal,
                        float scale, uint32_t m) {
  extern __shared__ __align__(16) float2 tsm[];
  const uint32_t TAU = kBigTile / m;
  const uint32_t tau0 = blockIdx.x * TAU;
  const int h = blockIdx.y, pr = blockIdx.z;
  const CxT<ST>* src = w_in + ((size_t)pr * H + h) * (size_t)m * kL;
  for (uint32_t i = threadIdx.x; i < kBigTile; i += kBigThreads) {
    const uint32_t a = pdiv(i, TAU), c = pmod(i, TAU);
    tsm[pad16(a) * TAU + c] = cmul(cx_load(src + (size_t)a * kL + tau0 + c), tw_big<+1>(tb, a * (tau0 + c)));
  }
  __syncthreads();
  smem_passes<+1, SMALL>(tsm, m, TAU, 1, m, tw_m);
  const uint32_t cmax = causal ? m / 2 : m;
  if constexpr (MODE == 0) {
    const int b0 = 2 * pr, b1 = b0 + 1;
    const bool has1 = b1 < B;
    const float d = __ldg(D + h);
    const size_t o0 = ((size_t)b0 * H + h) * N, o1 = ((size_t)b1 * H + h) * N;
    for (uint32_t i = threadIdx.x; i < cmax * TAU; i += kBigThreads) {
      const uint32_t cc = pdiv(i, TAU), c = pmod(i, TAU);
      const uint32_t t = cc * kL + tau0 + c;
      if (t < N) {
        const float2 v = tsm[pad16(cc) * TAU + c];
        st(out + o0 + t, fmaf(d, ld(skip + o0 + t), v.x));
        if (has1) st(out + o1 + t, fmaf(d, ld(skip + o1 + t), v.y));
      }
    }
  } else {
    for (uint32_t i = threadIdx.x; i < cmax * TAU; i += kBigThreads) {
      const uint32_t cc = pdiv(i, TAU), c = pmod(i, TAU);
      const uint32_t t = cc * kL + tau0 + c;
      if (t < N) dkbar[(size_t)h * N + t] = tsm[pad16(cc) * TAU + c].x * scale;
    }
  }
}

// ---------------------------------------------------------------- streaming big column passes
// Passes 1/3 for m > 16 as persistent kernels: a CTA walks tiles of
// TAU = 8192 / m columns x all m rows of one (pair, head); the next tile's
// input boxes stream in by TMA (2-stage ring, <= 256 rows per box) while the
// current tile runs its batched m-point column FFT in smem.
constexpr int kBigStages = 2;

// column twiddle w^(a (tau0 + c)) for the rows a = a0 + 16 k a thread visits
// (kBigThreads is a multiple of TAU, so c is fixed per thread): two table
// lookups per tile, then a 16-step rotation recurrence (fp32, a few ulp)
template <int SIGN>
struct ColTw {
  float2 w, step;
  __device__ __forceinline__ ColTw(const float2* __restrict__ tb, uint32_t a0, uint32_t tcol,
                                   uint32_t astep) {
    w = tw_big<SIGN>(tb, a0 * tcol);
    step = tw_big<SIGN>(tb, astep * tcol);
  }
  __device__ __forceinline__ float2 next() {
    const float2 r = w;
    w = cmul(w, step);
    return r;
  }
};

// two CTAs per SM where the smem allows it (single-signal pass 1)
// PLANAR: rows leave as [re l | im l] (the tcgen05 row pass's TMA layout)
template <typename IO, typename ST, int SMALL, int SRC, bool PLANAR = false>
__global__ void __launch_bounds__(kBigThreads, SRC == 1 ? 1 : 2)
    tp_bigs1_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                    CxT<ST>* __restrict__ out_a, CxT<ST>* __restrict__ out_b,
                    float* __restrict__ ddpart, const float2* __restrict__ tw_m,
                    const float2* __restrict__ tb, int H, int npairs, int rows, uint32_t m,
                    int ntiles) {
  extern __shared__ __align__(128) float2 tsm[];
  __shared__ __align__(8) uint64_t full[kBigStages];
  __shared__ float red[kBigThreads / 32];
  constexpr int NCH = SRC == 1 ? 4 : (SRC == 2 ? 1 : 2);
  const uint32_t TAU = kBigTile / m, NBk = kL / TAU;
  const uint32_t plen = padded_len(m) * TAU;
  float2* sa = tsm;
  float2* sb = tsm + plen;
  unsigned char* ring = reinterpret_cast<unsigned char*>(tsm + (SRC == 1 ? 2 : 1) * plen);
  const uint32_t chb = (uint32_t)rows * TAU * sizeof(IO);
  const uint32_t stage_bytes = NCH * chb;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kBigStages; ++i) ptx::mbar_init(&full[i], 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  auto tile_of = [&](int t, int& pr, int& h, int& tbk) {
    tbk = t % NBk;
    h = (t / NBk) % H;
    pr = t / (NBk * H);
  };
  auto issue = [&](int t, int sg) {
    int pr, h, tbk;
    tile_of(t, pr, h, tbk);
    unsigned char* dst = ring + (size_t)sg * stage_bytes;
    ptx::mbar_arrive_expect_tx(&full[sg], stage_bytes);
    for (int ch = 0; ch < NCH; ++ch) {
      const CUtensorMap* mp = (SRC == 1 && ch >= 2) ? &bmap : &amap;
      const int row = SRC == 2 ? h : (2 * pr + (ch & 1)) * H + h;
      for (int r0 = 0; r0 < rows; r0 += 256)
        tma_load_3d(dst + ch * chb + (size_t)r0 * TAU * sizeof(IO), mp, tbk * (int)TAU, r0, row,
                    &full[sg]);
    }
  };
  const int first = blockIdx.x, step = gridDim.x;
  if (threadIdx.x == 0 && first < ntiles) issue(first, 0);
  int it = 0;
  for (int t = first; t < ntiles; t += step, ++it) {
    const int sg = it % kBigStages;
    int pr, h, tbk;
    tile_of(t, pr, h, tbk);
    const uint32_t tau0 = tbk * TAU;
    if (threadIdx.x == 0 && t + step < ntiles) issue(t + step, (it + 1) % kBigStages);
    ptx::mbar_wait(&full[sg], (uint32_t)(it / kBigStages) & 1);
    const IO* sv = reinterpret_cast<const IO*>(ring + (size_t)sg * stage_bytes);
    float dd = 0.f;
    for (uint32_t i = threadIdx.x; i < kBigTile; i += kBigThreads) {
      const uint32_t e = pdiv(i, TAU), c = pmod(i, TAU);
      const bool ok = e < (uint32_t)rows;
      float2 v = make_float2(0.f, 0.f);
      if (ok) {
        v.x = tof(sv[e * TAU + c]);
        if constexpr (SRC != 2) v.y = tof(sv[(rows + e) * TAU + c]);
      }
      if constexpr (SRC == 1) {
        float2 w = make_float2(0.f, 0.f);
        if (ok) {
          w.x = tof(sv[(2 * rows + e) * TAU + c]);
          w.y = tof(sv[(3 * rows + e) * TAU + c]);
        }
        dd = fmaf(v.x, w.x, fmaf(v.y, w.y, dd));
        sb[pad16(e) * TAU + c] = w;
      }
      sa[pad16(e) * TAU + c] = v;
    }
    __syncthreads();  // stage sg consumed (refilled two tiles from now)
    smem_passes<-1, SMALL>(sa, m, TAU, 1, m, tw_m);
    if constexpr (SRC == 1) smem_passes<-1, SMALL>(sb, m, TAU, 1, m, tw_m);
    CxT<ST>* oa = out_a + ((size_t)pr * H + h) * (size_t)m * kL;
    CxT<ST>* ob = SRC == 1 ? out_b + ((size_t)pr * H + h) * (size_t)m * kL : nullptr;
    ColTw<-1> ctw(tb, pdiv(threadIdx.x, TAU), tau0 + pmod(threadIdx.x, TAU), pdiv(kBigThreads, TAU));
    for (uint32_t i = threadIdx.x; i < kBigTile; i += kBigThreads) {
      const uint32_t a = pdiv(i, TAU), c = pmod(i, TAU);
      const float2 w = ctw.next();
      if constexpr (PLANAR) {
        const float2 x = cmul(sa[pad16(a) * TAU + c], w);
        ST* r = reinterpret_cast<ST*>(oa + (size_t)a * kL);
        st(r + tau0 + c, x.x);
        st(r + kL + tau0 + c, x.y);
      } else {
        stc<ST>(&oa[(size_t)a * kL + tau0 + c].x, cmul(sa[pad16(a) * TAU + c], w));
      }
      if constexpr (SRC == 1) stc<ST>(&ob[(size_t)a * kL + tau0 + c].x, cmul(sb[pad16(a) * TAU + c], w));
    }
    if constexpr (SRC == 1) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dd += __shfl_xor_sync(0xffffffffu, dd, o);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dd;
    }
    __syncthreads();  // tile buffers free for the next tile
    if constexpr (SRC == 1) {
      if (threadIdx.x == 0) {
        float s = 0.f;
        for (uint32_t w2 = 0; w2 < kBigThreads / 32; ++w2) s += red[w2];
        ddpart[((size_t)h * npairs + pr) * NBk + tbk] = s;
      }
    }
  }
}

template <typename ST, typename IO, int SMALL, int MODE>
__global__ void __launch_bounds__(kBigThreads, 1)
    tp_bigs3_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap smap,
                    IO* __restrict__ out, const float* __restrict__ D, float* __restrict__ dkbar,
                    const float2* __restrict__ tw_m, const float2* __restrict__ tb, int B, int H,
                    uint32_t N, int rows, uint32_t m, float scale, int ntiles) {
  extern __shared__ __align__(128) float2 tsm[];
  __shared__ __align__(8) uint64_t full[kBigStages];
  const uint32_t TAU = kBigTile / m, NBk = kL / TAU;
  const uint32_t plen = padded_len(m) * TAU;
  unsigned char* ring = reinterpret_cast<unsigned char*>(tsm + plen);
  const uint32_t wb = m * TAU * sizeof(CxT<ST>);
  const uint32_t chb = MODE == 0 ? (uint32_t)rows * TAU * sizeof(IO) : 0;
  const uint32_t stage_bytes = wb + 2 * chb;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kBigStages; ++i) ptx::mbar_init(&full[i], 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  auto tile_of = [&](int t, int& pr, int& h, int& tbk) {
    tbk = t % NBk;
    h = (t / NBk) % H;
    pr = t / (NBk * H);
  };
  auto issue = [&](int t, int sg) {
    int pr, h, tbk;
    tile_of(t, pr, h, tbk);
    unsigned char* dst = ring + (size_t)sg * stage_bytes;
    ptx::mbar_arrive_expect_tx(&full[sg], stage_bytes);
    for (uint32_t r0 = 0; r0 < m; r0 += 256)
      tma_load_3d(dst + (size_t)r0 * TAU * sizeof(CxT<ST>), &wmap, tbk * (int)TAU, (int)r0,
                  pr * H + h, &full[sg]);
    if constexpr (MODE == 0)
      for (int ch = 0; ch < 2; ++ch)
        for (int r0 = 0; r0 < rows; r0 += 256)
          tma_load_3d(dst + wb + ch * chb + (size_t)r0 * TAU * sizeof(IO), &smap, tbk * (int)TAU,
                      r0, (2 * pr + ch) * H + h, &full[sg]);
  };
  const int first = blockIdx.x, step = gridDim.x;
  if (threadIdx.x == 0 && first < ntiles) issue(first, 0);
  int it = 0;
  for (int t = first; t < ntiles; t += step, ++it) {
    const int sg = it % kBigStages;
    int pr, h, tbk;
    tile_of(t, pr, h, tbk);
    const uint32_t tau0 = tbk * TAU;
    if (threadIdx.x == 0 && t + step < ntiles) issue(t + step, (it + 1) % kBigStages);
    ptx::mbar_wait(&full[sg], (uint32_t)(it / kBigStages) & 1);
    const unsigned char* base = ring + (size_t)sg * stage_bytes;
    const CxT<ST>* sw = reinterpret_cast<const CxT<ST>*>(base);
    ColTw<+1> ctw(tb, pdiv(threadIdx.x, TAU), tau0 + pmod(threadIdx.x, TAU), pdiv(kBigThreads, TAU));
    for (uint32_t i = threadIdx.x; i < kBigTile; i += kBigThreads) {
      const uint32_t a = pdiv(i, TAU), c = pmod(i, TAU);
      tsm[pad16(a) * TAU + c] = cmul(cx_load(sw + a * TAU + c), ctw.next());
    }
    __syncthreads();
    smem_passes<+1, SMALL>(tsm, m, TAU, 1, m, tw_m);
    if constexpr (MODE == 0) {
      const IO* sk = reinterpret_cast<const IO*>(base + wb);
      const int b0 = 2 * pr, b1 = b0 + 1;
      const bool has1 = b1 < B;
      const float d = __ldg(D + h);
      const size_t o0 = ((size_t)b0 * H + h) * N, o1 = ((size_t)b1 * H + h) * N;
      for (uint32_t i = threadIdx.x; i < (uint32_t)rows * TAU; i += kBigThreads) {
        const uint32_t cc = pdiv(i, TAU), c = pmod(i, TAU);
        const uint32_t tt = cc * kL + tau0 + c;
        const float2 v = tsm[pad16(cc) * TAU + c];
        st(out + o0 + tt, fmaf(d, tof(sk[cc * TAU + c]), v.x));
        if (has1) st(out + o1 + tt, fmaf(d, tof(sk[(rows + cc) * TAU + c]), v.y));
      }
    } else {
      for (uint32_t i = threadIdx.x; i < (uint32_t)rows * TAU; i += kBigThreads) {
        const uint32_t cc = pdiv(i, TAU), c = pmod(i, TAU);
        dkbar[(size_t)h * N + cc * kL + tau0 + c] = tsm[pad16(cc) * TAU + c].x * scale;
      }
    }
    __syncthreads();  // tile and stage sg free
  }
}

// ---------------------------------------------------------------- sequence-sharded passes
// Local passes of the four-step convolution when the transform itself is
// sharded over ranks (config 5-4M, paper_2302_06646_b200/seqshard.py): rank r
// holds columns tau in [tau0, tau0 + lp) of every row c of n = l m, as complex
// fp32 [C][m][lp].  Same arithmetic as passes 1 / 3 (three_pass.cpp:225-254)
// with the global column index in the twiddle:
//   SIGN -1:  out[a][tau] = w_n^(-a tau) sum_c w_m^(-a c) in[c][tau]
//   SIGN +1:  out[c][tau] = scale sum_a w_m^(+a c) w_n^(+a tau) in[a][tau]
// Signal-side variants (the layer's pair packing fused into the passes):
// IO = the signal type; pass 1 (SIGN -1) reads channel (p, h) straight from
// the real signals sig[B][H][half][lp] (channels 2p / 2p+1 as re / im, rows
// >= half the causal zero pad) and pass 3 (SIGN +1) writes re / im of its
// rows < half back as channels 2p / 2p+1 of out[B][H][half][lp], plus
// D[h] skip (optional).  IO = void: complex f32 in / out ([C][m][lp]).
struct ShardSig {
  const void* sig = nullptr;   // pass 1 input signals
  void* out = nullptr;         // pass 3 output signals
  const void* skip = nullptr;  // pass 3: + D[h] skip[b][h][c][tau]
  const float* D = nullptr;
  int B = 0, H = 0, half = 0;
};
template <int SIGN, int SMALL, typename IO = void>
__global__ void __launch_bounds__(kBigThreads, 1)
    tp_shard_cols_kernel(const float2* __restrict__ in, float2* __restrict__ out,
                         const float2* __restrict__ tw_m, const float2* __restrict__ tb, uint32_t m,
                         uint32_t lp, uint32_t tau0, float scale, ShardSig sg) {
  constexpr bool kSig = !std::is_same<IO, void>::value;
  using T = typename std::conditional<kSig, IO, float>::type;
  extern __shared__ __align__(16) float2 tsm[];
  const uint32_t TAU = kBigTile / m;
  const uint32_t c0 = blockIdx.x * TAU;
  const size_t ch = (size_t)blockIdx.y * m * lp;
  const int pr = kSig ? (int)blockIdx.y / sg.H : 0, hh = kSig ? (int)blockIdx.y % sg.H : 0;
  for (uint32_t i = threadIdx.x; i < kBigTile; i += kBigThreads) {
    const uint32_t e = pdiv(i, TAU), c = pmod(i, TAU);
    float2 v;
    if constexpr (kSig && SIGN < 0) {
      v = make_float2(0.f, 0.f);
      if ((int)e < sg.half) {
        const T* sg0 = reinterpret_cast<const T*>(sg.sig);
        const size_t o = ((size_t)(2 * pr) * sg.H + hh) * sg.half * lp + (size_t)e * lp + c0 + c;
        v.x = tof(sg0[o]);
        if (2 * pr + 1 < sg.B) v.y = tof(sg0[o + (size_t)sg.H * sg.half * lp]);
      }
    } else {
      v = __ldg(in + ch + (size_t)e * lp + c0 + c);
    }
    if (SIGN > 0) v = cmul(v, tw_big<+1>(tb, e * (tau0 + c0 + c)));
    tsm[pad16(e) * TAU + c] = v;
  }
  __syncthreads();
  smem_passes<SIGN, SMALL>(tsm, m, TAU, 1, m, tw_m);
  for (uint32_t i = threadIdx.x; i < kBigTile; i += kBigThreads) {
    const uint32_t a = pdiv(i, TAU), c = pmod(i, TAU);
    float2 v = tsm[pad16(a) * TAU + c];
    v = SIGN < 0 ? cmul(v, tw_big<-1>(tb, a * (tau0 + c0 + c))) : cscale(v, scale);
    if constexpr (kSig && SIGN > 0) {
      if ((int)a >= sg.half) continue;
      T* so = reinterpret_cast<T*>(sg.out);
      const T* sk = reinterpret_cast<const T*>(sg.skip);
      const float d = sk ? __ldg(sg.D + hh) : 0.f;
      for (int q = 0; q < 2; ++q) {
        const int b = 2 * pr + q;
        if (b >= sg.B) break;
        const size_t o = ((size_t)b * sg.H + hh) * sg.half * lp + (size_t)a * lp + c0 + c;
        float r = q ? v.y : v.x;
        if (sk) r += d * tof(sk[o]);
        so[o] = cvt<T>(r);
      }
    } else {
      out[ch + (size_t)a * lp + c0 + c] = v;
    }
  }
}

// ---------------------------------------------------------------- host side
namespace {

template <typename ST>
size_t pass2_smem() {
  using S = FftShape<kL2>;
  return (S::work_len + (sizeof(ST) < 4 ? S::n : 0) + ((S::tab_len + 1) & ~1u)) * sizeof(float2) +
         2 * kL * sizeof(CxT<ST>);
}
template <typename ST>
size_t pass2_bwd_smem() {
  using S = FftShape<kL2>;
  return (S::work_len + S::n + ((S::tab_len + 1) & ~1u)) * sizeof(float2) + kL * sizeof(CxT<ST>);
}

template <class F>
void with_m(int64_t m, F&& f) {
  switch (m) {
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    case 8: f(std::integral_constant<int, 8>{}); break;
    default: f(std::integral_constant<int, 16>{}); break;
  }
}
template <class F>
void with_io(int dtype, F&& f) {
  switch (dtype) {
    case FB_F32: f(float{}); break;
    case FB_BF16: f(__nv_bfloat16{}); break;
    default: f(__half{}); break;
  }
}

int log2u(int64_t v) {
  int k = 0;
  while ((int64_t(1) << k) < v) ++k;
  return k;
}

template <class F>
void with_small(int64_t m, F&& f) {
  switch (log2u(m) % 4) {
    case 0: f(std::integral_constant<int, 1>{}); break;
    case 1: f(std::integral_constant<int, 2>{}); break;
    case 2: f(std::integral_constant<int, 4>{}); break;
    default: f(std::integral_constant<int, 8>{}); break;
  }
}

size_t big_smem(int src) {
  return (size_t)(src == 1 ? 2 : 1) * padded_len(kBigTile) * sizeof(float2) + 64 * sizeof(float2);
}

template <typename T>
constexpr CUtensorMapDataType tma_type() {
  if constexpr (std::is_same<T, float>::value) return CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  else if constexpr (std::is_same<T, __nv_bfloat16>::value) return CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  else return CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
}

// signal [B][H][N] as [B*H][rows = N / l][l], box [256][rows][1]
template <typename IO>
int signal_map(CUtensorMap* m, const fb_plan* p, const IO* ptr, int B) {
  const uint64_t rows = (uint64_t)(p->N / kL);
  const uint64_t dims[3] = {kL, rows, (uint64_t)B * p->H};
  const uint64_t strides[2] = {kL * sizeof(IO), (uint64_t)p->N * sizeof(IO)};
  const uint32_t box[3] = {kTB, (uint32_t)rows, 1};
  return encode_map_3d(m, tma_type<IO>(), ptr, dims, strides, box);
}
// intermediates [npairs*H][m][l] complex, box [256][m][1]
template <typename ST>
int inter_map(CUtensorMap* mp, const fb_plan* p, const CxT<ST>* ptr, int npairs) {
  constexpr size_t es = sizeof(CxT<ST>);
  const uint64_t dims[3] = {kL, (uint64_t)p->m, (uint64_t)npairs * p->H};
  const uint64_t strides[2] = {kL * es, (uint64_t)p->m * kL * es};
  const uint32_t box[3] = {kTB, (uint32_t)p->m, 1};
  return encode_map_3d(mp, es == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT64,
                       ptr, dims, strides, box);
}
// [outer][rows][l] view (rows l apart, outer blocks outer_stride elements
// apart) with a {tau, min(rows, 256), 1} box
template <typename T>
int rows_map(CUtensorMap* mp, CUtensorMapDataType type, const T* ptr, uint64_t outer, uint64_t rows,
             uint64_t outer_stride, uint32_t tau) {
  const uint64_t dims[3] = {kL, rows, outer};
  const uint64_t strides[2] = {kL * sizeof(T), outer_stride * sizeof(T)};
  const uint32_t box[3] = {tau, (uint32_t)std::min<uint64_t>(rows, 256), 1};
  return encode_map_3d(mp, type, ptr, dims, strides, box);
}
template <typename ST>
constexpr CUtensorMapDataType cx_type() {
  return sizeof(CxT<ST>) == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT64;
}
// FB_BIGS=0 / 1 / 3 (debug): streaming big-column kernels off / pass 1 only / pass 3 only
int bigs_mask() {
  static int v = [] {
    const char* e = getenv("FB_BIGS");
    return e ? atoi(e) : 3 | 1;
  }();
  return v;
}
size_t bigs_smem(uint32_t m, int tiles, size_t stage) {
  return (size_t)tiles * padded_len(kBigTile) * sizeof(float2) + kBigStages * stage;
}

int col_stages(size_t stage_bytes) {
  return (int)std::max<size_t>(2, std::min<size_t>(kColMaxStages, (52 * 1024) / stage_bytes));
}
// resident CTAs per SM as the ring's smem allows (<= 4), persistent over the tiles
int col_grid(size_t ring_bytes, int ntiles, int sms) {
  const int per = (int)std::max<size_t>(1, std::min<size_t>(4, (220 * 1024) / (ring_bytes + 2048)));
  return std::min(ntiles, per * sms);
}

// pass 1: streaming TMA column kernel (signals, m <= 16), register kernel for
// the kernel bank, tiled smem kernel for m > 16
template <typename IO, typename ST, int SRC>
uint32_t launch_pass1(const fb_plan* p, const IO* a, const IO* b, CxT<ST>* oa, CxT<ST>* ob,
                      float* ddpart, int B, int npairs, cudaStream_t s, bool planar = false) {
  const int causal = p->mode == FB_MODE_CAUSAL;
  if constexpr (SRC == 0) {
    if (planar && p->m <= 16) {  // the tcgen05 row pass's input: streaming column kernel only
      CUtensorMap am;
      if (signal_map<IO>(&am, p, a, B)) {
        set_error("three-pass: planar pass 1 needs a signal tensor map");
        return 0;
      }
      const int rows = (int)(p->N / kL);
      const size_t stage = (size_t)2 * rows * kTB * sizeof(IO);
      const int ns = col_stages(stage);
      const int ntiles = (int)(npairs * p->H * (kL / kTB));
      const int grid = col_grid(stage * ns, ntiles, p->num_sms);
      with_m(p->m, [&](auto mc) {
        constexpr int M = decltype(mc)::value;
        auto k = tp_col1_kernel<IO, ST, M, 0, true>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(stage * ns));
        k<<<grid, kCons + 32, stage * ns, s>>>(am, am, oa, nullptr, nullptr, p->tw_n, (int)p->H,
                                             npairs, rows, ntiles, ns);
      });
      return kL / kTB;
    }
    if (planar && p->m > 16) {  // m = 32 .. 128: the column DFTs as tcgen05 GEMMs
      const int rc = tc_col1(p, a, oa, B, npairs, s);
      if (rc == FB_OK) return kL / 128;
      if (rc != FB_ERR_UNSUPPORTED) return 0;
    }
  }
  if constexpr (SRC != 2) {
    if (p->m <= 16) {
      CUtensorMap am, bm;
      const bool maps = !signal_map<IO>(&am, p, a, B) && !signal_map<IO>(&bm, p, SRC == 1 ? b : a, B);
      const int rows = (int)(p->N / kL);
      const size_t stage = (size_t)(SRC == 1 ? 4 : 2) * rows * kTB * sizeof(IO);
      const int ns = col_stages(stage);
      const int ntiles = (int)(npairs * p->H * (kL / kTB));
      const int grid = col_grid(stage * ns, ntiles, p->num_sms);
      if (maps) with_m(p->m, [&](auto mc) {
        constexpr int M = decltype(mc)::value;
        auto k = tp_col1_kernel<IO, ST, M, SRC>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(stage * ns));
        k<<<grid, kCons + 32, stage * ns, s>>>(am, bm, oa, ob, ddpart, p->tw_n, (int)p->H, npairs,
                                             rows, ntiles, ns);
      });
      if (maps) return kL / kTB;
    }
  }
  if (p->m <= 16) {
    with_m(p->m, [&](auto mc) {
      constexpr int M = decltype(mc)::value;
      tp_pass1_kernel<IO, ST, M, SRC><<<dim3(kL / kColThreads, (unsigned)p->H, (unsigned)npairs),
                                        kColThreads, 0, s>>>(a, b, p->kbar, oa, ob, ddpart, p->tw_n,
                                                             B, (int)p->H, (uint32_t)p->N, causal);
    });
    return kL / kColThreads;
  }
  const uint32_t gx = (uint32_t)(kL / (kBigTile / p->m));
  {
    // streaming big-column kernel (TMA ring)
    const uint32_t TAU = (uint32_t)(kBigTile / p->m);
    const int rows = (int)(p->N / kL);
    CUtensorMap am, bm;
    bool maps;
    if constexpr (SRC == 2) {
      maps = !rows_map<float>(&am, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, p->kbar, (uint64_t)p->H, rows,
                              (uint64_t)p->N, TAU);
      bm = am;
    } else {
      maps = !rows_map<IO>(&am, tma_type<IO>(), a, (uint64_t)B * p->H, rows, (uint64_t)p->N, TAU) &&
             !rows_map<IO>(&bm, tma_type<IO>(), SRC == 1 ? b : a, (uint64_t)B * p->H, rows,
                           (uint64_t)p->N, TAU);
    }
    const int nch = SRC == 1 ? 4 : (SRC == 2 ? 1 : 2);
    const size_t stage = (size_t)nch * rows * TAU * sizeof(IO);
    const size_t sm = bigs_smem((uint32_t)p->m, SRC == 1 ? 2 : 1, stage);
    const int ntiles = (int)((SRC == 2 ? 1 : npairs) * p->H * gx);
    if (maps && sm <= 227 * 1024 && (bigs_mask() & 1)) {
      with_small(p->m, [&](auto sc) {
        constexpr int SM = decltype(sc)::value;
        auto k = tp_bigs1_kernel<IO, ST, SM, SRC>;
        if constexpr (SRC == 0)
          if (planar) k = tp_bigs1_kernel<IO, ST, SM, SRC, true>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        const int per_sm = (SRC != 1 && sm <= 113 * 1024) ? 2 : 1;
        k<<<std::min(ntiles, per_sm * p->num_sms), kBigThreads, sm, s>>>(am, bm, oa, ob, ddpart, p->tw_m,
                                                                p->tw_big, (int)p->H, npairs, rows,
                                                                (uint32_t)p->m, ntiles);
      });
      return gx;
    }
  }
  if (planar) {
    set_error("three-pass: planar pass 1 needs the streaming column kernels");
    return 0;
  }
  with_small(p->m, [&](auto sc) {
    constexpr int SM = decltype(sc)::value;
    auto k = tp_pass1_big_kernel<IO, ST, SM, SRC>;
    const size_t sm = big_smem(SRC);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<dim3(gx, (unsigned)p->H, (unsigned)npairs), kBigThreads, sm, s>>>(
        a, b, p->kbar, oa, ob, ddpart, p->tw_m, p->tw_big, B, (int)p->H, (uint32_t)p->N, causal,
        (uint32_t)p->m);
  });
  return gx;
}

template <typename ST, typename IO, int MODE>
void launch_pass3(const fb_plan* p, const CxT<ST>* w, const IO* skip, IO* out, float* dkbar,
                  int B, int npairs, float scale, cudaStream_t s) {
  const int causal = p->mode == FB_MODE_CAUSAL;
  if constexpr (MODE == 0) {
    if (p->m <= 16) {
      CUtensorMap wm, sm;
      const bool maps = !inter_map<ST>(&wm, p, w, npairs) && !signal_map<IO>(&sm, p, skip, B);
      const int rows = (int)(p->N / kL);
      const size_t stage = p->m * kTB * sizeof(CxT<ST>) + 2 * (size_t)rows * kTB * sizeof(IO);
      const int ns = col_stages(stage);
      const int ntiles = (int)(npairs * p->H * (kL / kTB));
      const int grid = col_grid(stage * ns, ntiles, p->num_sms);
      if (maps) with_m(p->m, [&](auto mc) {
        constexpr int M = decltype(mc)::value;
        auto k = tp_col3_kernel<ST, IO, M>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(stage * ns));
        k<<<grid, kCons + 32, stage * ns, s>>>(wm, sm, out, p->d, p->tw_n, B, (int)p->H,
                                             (uint32_t)p->N, rows, ntiles, ns);
      });
      if (maps) return;  // else: the register column kernel below
    }
    if constexpr (std::is_same_v<ST, __nv_bfloat16>) {
      if (p->m > 16) {  // m = 32 / 64: the inverse column DFTs as tcgen05 GEMMs
        const int rc = tc_col3(p, w, skip, out, B, npairs, s);
        if (rc != FB_ERR_UNSUPPORTED) return;
      }
    }
  }
  if (p->m <= 16) {
    with_m(p->m, [&](auto mc) {
      constexpr int M = decltype(mc)::value;
      tp_pass3_kernel<ST, IO, M, MODE><<<dim3(kL / kColThreads, (unsigned)p->H, (unsigned)npairs),
                                         kColThreads, 0, s>>>(w, skip, out, p->d, dkbar, p->tw_n, B,
                                                              (int)p->H, (uint32_t)p->N, causal,
                                                              scale);
    });
    return;
  }
  const uint32_t gx = (uint32_t)(kL / (kBigTile / p->m));
  {
    const uint32_t TAU = (uint32_t)(kBigTile / p->m);
    const int rows = (int)(p->N / kL);
    const int np = MODE == 0 ? npairs : 1;
    CUtensorMap wm, sm_map;
    bool maps = !rows_map<CxT<ST>>(&wm, cx_type<ST>(), w, (uint64_t)np * p->H, (uint64_t)p->m,
                                   (uint64_t)p->m * kL, TAU);
    if constexpr (MODE == 0)
      maps = maps && !rows_map<IO>(&sm_map, tma_type<IO>(), skip, (uint64_t)B * p->H, rows,
                                   (uint64_t)p->N, TAU);
    else
      sm_map = wm;
    const size_t stage = (size_t)p->m * TAU * sizeof(CxT<ST>) +
                         (MODE == 0 ? 2 * (size_t)rows * TAU * sizeof(IO) : 0);
    const size_t smb = bigs_smem((uint32_t)p->m, 1, stage);
    const int ntiles = (int)(np * p->H * gx);
    if (maps && smb <= 227 * 1024 && (bigs_mask() & 2)) {
      with_small(p->m, [&](auto sc) {
        constexpr int SM = decltype(sc)::value;
        auto k = tp_bigs3_kernel<ST, IO, SM, MODE>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);
        k<<<std::min(ntiles, p->num_sms), kBigThreads, smb, s>>>(
            wm, sm_map, out, p->d, dkbar, p->tw_m, p->tw_big, B, (int)p->H, (uint32_t)p->N, rows,
            (uint32_t)p->m, scale, ntiles);
      });
      return;
    }
  }
  with_small(p->m, [&](auto sc) {
    constexpr int SM = decltype(sc)::value;
    auto k = tp_pass3_big_kernel<ST, IO, SM, MODE>;
    const size_t sm = big_smem(0);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<dim3(gx, (unsigned)p->H, (unsigned)npairs), kBigThreads, sm, s>>>(
        w, skip, out, p->d, dkbar, p->tw_m, p->tw_big, B, (int)p->H, (uint32_t)p->N, causal, scale,
        (uint32_t)p->m);
  });
}

size_t inter_bytes(const fb_plan* p, int64_t npairs) {
  const size_t es = p->dtype == FB_F32 ? 8 : 4;  // complex storage element
  return ((size_t)npairs * p->H * p->n * es + 255) & ~size_t(255);
}

int pass2_chunks(const fb_plan* p, int64_t npairs) {
  const int64_t rows = p->H * p->m;
  int64_t c = (p->num_sms + rows - 1) / rows;
  return (int)std::max<int64_t>(1, std::min<int64_t>(c, npairs));
}

}  // namespace

int tp_prep(fb_plan* p, const float* K, cudaStream_t s) {
  int rc = regularize_bank_dev(p, K, s);
  if (rc) return rc;
  // kernel rows through pass 1 (fp32) straight into the spectrum buffer, then
  // each row's FFT in place (a CTA stages its whole row before writing it)
  auto* x1k = reinterpret_cast<CxT<float>*>(p->kf);
  launch_pass1<float, float, 2>(p, nullptr, nullptr, x1k, nullptr, nullptr, 2, 1, s);
  const size_t sm = pass2_smem<float>();
  auto k = tp_pass2_kernel<float, 1>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k<<<dim3((unsigned)(p->H * p->m), 1), kL / 16, sm, s>>>(x1k, nullptr, p->kf, p->tw_l, 1,
                                                          (int)p->H, (int)p->m, 1,
                                                          1.0f / (float)p->n, nullptr);
  return cuda_status(cudaGetLastError(), "tp_prep");
}

size_t tp_workspace(const fb_plan* p, int64_t B) {
  const int64_t npairs = (B + 1) / 2;
  size_t bytes = 2 * inter_bytes(p, npairs);                            // X1dy/X1u (fwd: X1)
  bytes += ((size_t)p->H * p->n * sizeof(float2) + 255) & ~size_t(255); // dK rows
  bytes += ((size_t)p->H * p->N * sizeof(float) + 255) & ~size_t(255);  // dKbar scratch
  bytes += ((size_t)p->H * npairs * 1024 * sizeof(float) + 255) & ~size_t(255);  // dD partials
  return bytes + 256;
}

size_t tp_saved_size(const fb_plan* p, int64_t B) { return inter_bytes(p, (B + 1) / 2); }

__global__ void tp_dd_lag0_kernel(const float* __restrict__ dkbar, float* __restrict__ dD, int H,
                                  int64_t N) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h < H) dD[h] = dkbar[(size_t)h * N];  // dD = sum_t dy u = dKbar[0] (lag 0)
}

// pass 2 on tcgen05 when the dtype allows it and pass 1 can write planar rows
// (streaming column kernels: m <= 16, or the big-column ring fits in smem)
static bool use_tc_rows(const fb_plan* p) {
  if (!tc_rows_eligible(p)) return false;
  if (p->m <= 16) return true;
  const uint32_t TAU = (uint32_t)(kBigTile / p->m);
  const size_t stage = (size_t)2 * (p->N / kL) * TAU * 2;
  return bigs_smem((uint32_t)p->m, 1, stage) <= 227 * 1024 && (bigs_mask() & 1);
}

bool tp_uses_tc_rows(const fb_plan* p) { return use_tc_rows(p); }

int tp_fwd(fb_plan* p, const void* u, void* y, int64_t B, void* ws, cudaStream_t s, void* usave) {
  const int64_t npairs = (B + 1) / 2;
  if (p->periodic) {
    set_error("three-pass: circular mode needs N == n");
    return FB_ERR_UNSUPPORTED;
  }
  int rc = FB_OK;
  const bool tcr = use_tc_rows(p);
  // intermediates in the I/O precision, except fp16 on the tcgen05 rows:
  // bf16 there (the rows kernels' operand type; no fp16 range limit)
  auto body = [&](auto io, auto st) {
    using IO = decltype(io);
    using ST = decltype(st);
    auto* x1 = reinterpret_cast<CxT<ST>*>(ws);
    if (tcr) {  // pass 2 on tcgen05 (planar rows in, interleaved out)
      if (!launch_pass1<IO, ST, 0>(p, (const IO*)u, nullptr, x1, nullptr, nullptr, (int)B,
                                   (int)npairs, s, true)) {
        rc = FB_ERR_UNSUPPORTED;
        return;
      }
      // pass 1 ran alongside an asynchronous kernel prep
      if ((rc = prep_wait(p, s)) || (rc = tc_rows_fwd(p, x1, usave, npairs, s))) return;
      launch_pass3<ST, IO, 0>(p, x1, (const IO*)u, (IO*)y, nullptr, (int)B, (int)npairs, 1.f, s);
      return;
    }
    launch_pass1<IO, ST, 0>(p, (const IO*)u, nullptr, x1, nullptr, nullptr, (int)B, (int)npairs, s);
    if ((rc = prep_wait(p, s))) return;
    const size_t sm = pass2_smem<ST>();
    auto k2 = tp_pass2_kernel<ST, 0>;
    cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const int chunks = pass2_chunks(p, npairs);
    const int ppc = (int)((npairs + chunks - 1) / chunks);
    prof_mark(p, 0, 0, s);
    k2<<<dim3((unsigned)(p->H * p->m), (unsigned)chunks), kL / 16, sm, s>>>(
        x1, p->kf, nullptr, p->tw_l, (int)npairs, (int)p->H, (int)p->m, ppc, 0.f,
        reinterpret_cast<CxT<ST>*>(usave));
    prof_mark(p, 0, 1, s);
    launch_pass3<ST, IO, 0>(p, x1, (const IO*)u, (IO*)y, nullptr, (int)B, (int)npairs, 1.f, s);
  };
  with_io(p->dtype, [&](auto io) {
    using IO = decltype(io);
    if constexpr (std::is_same<IO, __half>::value) {
      if (tcr) body(io, __nv_bfloat16{});
      else body(io, io);
    } else {
      body(io, io);
    }
  });
  if (rc) return rc;
  return cuda_status(cudaGetLastError(), "tp_fwd");
}

int tp_bwd(fb_plan* p, const void* dy, const void* u, void* du, float* dK, float* dKbar, float* dD,
           int64_t B, void* ws, cudaStream_t s, const void* usave) {
  const int64_t npairs = (B + 1) / 2;
  if (p->periodic) {
    set_error("three-pass: circular mode needs N == n");
    return FB_ERR_UNSUPPORTED;
  }
  char* w = (char*)ws;
  uint32_t gx = 0;
  const size_t ib = inter_bytes(p, npairs);
  char* x1dy_raw = w;
  char* x1u_raw = w + ib;
  float2* wdk = (float2*)(w + 2 * ib);
  size_t off = 2 * ib + (((size_t)p->H * p->n * sizeof(float2) + 255) & ~size_t(255));
  float* dkbar_s = (float*)(w + off);
  off += ((size_t)p->H * p->N * sizeof(float) + 255) & ~size_t(255);
  float* ddpart = (float*)(w + off);
  float* dkbar = dKbar ? dKbar : dkbar_s;
  int rc = FB_OK;
  const bool tcr = use_tc_rows(p);
  auto body = [&](auto io, auto st) {
    using IO = decltype(io);
    using ST = decltype(st);
    auto* x1dy = reinterpret_cast<CxT<ST>*>(x1dy_raw);
    auto* x1u = reinterpret_cast<CxT<ST>*>(x1u_raw);
    const size_t sm = pass2_bwd_smem<ST>();
    if (tcr) {  // rows on tcgen05; without a saved U, recompute it (spectrum-only rows)
      const void* us = usave;
      if (!us) {
        if (!launch_pass1<IO, ST, 0>(p, (const IO*)u, nullptr, x1u, nullptr, nullptr, (int)B,
                                     (int)npairs, s, true)) {
          rc = FB_ERR_UNSUPPORTED;
          return;
        }
        if ((rc = tc_rows_spectrum(p, x1u, npairs, s))) return;
        us = x1u;
      }
      if (!launch_pass1<IO, ST, 0>(p, (const IO*)dy, nullptr, x1dy, nullptr, nullptr, (int)B,
                                   (int)npairs, s, true)) {
        rc = FB_ERR_UNSUPPORTED;
        return;
      }
      if ((rc = tc_rows_bwd(p, x1dy, us, wdk, npairs, s))) return;
    } else if (usave) {  // the forward's row spectra of u: pass 1 and 2 on dy only
      launch_pass1<IO, ST, 0>(p, (const IO*)dy, nullptr, x1dy, nullptr, nullptr, (int)B,
                              (int)npairs, s);
      auto k2 = tp_pass2_bwd_kernel<ST, true>;
      cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      prof_mark(p, 1, 0, s);
      k2<<<(unsigned)(p->H * p->m), kL / 16, sm, s>>>(
          x1dy, reinterpret_cast<const CxT<ST>*>(usave), p->kf, wdk, p->tw_l, (int)npairs,
          (int)p->H, (int)p->m);
      prof_mark(p, 1, 1, s);
    } else {
      gx = launch_pass1<IO, ST, 1>(p, (const IO*)dy, (const IO*)u, x1dy, x1u, ddpart, (int)B,
                                   (int)npairs, s);
      auto k2 = tp_pass2_bwd_kernel<ST, false>;
      cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      prof_mark(p, 1, 0, s);
      k2<<<(unsigned)(p->H * p->m), kL / 16, sm, s>>>(x1dy, x1u, p->kf, wdk, p->tw_l, (int)npairs,
                                                       (int)p->H, (int)p->m);
      prof_mark(p, 1, 1, s);
    }
    // the dK tail (dK rows -> dKbar, dD, regularizer chain rule) on the
    // auxiliary stream, alongside pass 3 of du
    cudaStream_t ts = s;
    if (p->aux && !cudaEventRecord(p->ev_fork, s) && !cudaStreamWaitEvent(p->aux, p->ev_fork, 0))
      ts = p->aux;
    launch_pass3<float, float, 1>(p, reinterpret_cast<const CxT<float>*>(wdk), nullptr, nullptr,
                                  dkbar, 2, 1, 1.0f / (float)p->n, ts);
    if (usave || tcr)
      tp_dd_lag0_kernel<<<(unsigned)((p->H + 127) / 128), 128, 0, ts>>>(dkbar, dD, (int)p->H, p->N);
    else
      tp_dd_reduce_kernel<<<(unsigned)p->H, 32, 0, ts>>>(ddpart, dD, (int)(npairs * gx));
    if (int r2 = regularizer_backward_dev(p, dkbar, dK, ts)) rc = r2;
    launch_pass3<ST, IO, 0>(p, x1dy, (const IO*)dy, (IO*)du, nullptr, (int)B, (int)npairs, 1.f, s);
    if (ts != s) {  // join
      cudaEventRecord(p->ev_join, ts);
      cudaStreamWaitEvent(s, p->ev_join, 0);
    }
  };
  with_io(p->dtype, [&](auto io) {
    using IO = decltype(io);
    if constexpr (std::is_same<IO, __half>::value) {
      if (tcr) body(io, __nv_bfloat16{});
      else body(io, io);
    } else {
      body(io, io);
    }
  });
  if (rc) return rc;
  return cuda_status(cudaGetLastError(), "tp_bwd");
}

}  // namespace fb

// ---------------------------------------------------------------- sequence-sharded C ABI
namespace fb {
int upload_table(float2** dst, int64_t n, int kind);  // fb_capi.cu
}
using namespace fb;

struct fb_shard_plan {
  int64_t l = kL, m = 0, n = 0;
  int device = 0;
  float2* tw_m = nullptr;    // exp(-2 pi i t / m)
  float2* tw_big = nullptr;  // two-level exp(-2 pi i t / n)
  float2* tw_l = nullptr;    // two-level table of the l-point row FFT
};

extern "C" {

int fb_shard_plan_destroy(fb_shard_plan* sp) {
  if (!sp) return FB_OK;
  cudaFree(sp->tw_m);
  cudaFree(sp->tw_big);
  cudaFree(sp->tw_l);
  delete sp;
  return FB_OK;
}

int fb_shard_plan_create(fb_shard_plan** out, int64_t n, int device) {
  if (!out) {
    set_error("fb_shard_plan_create: null output");
    return FB_ERR_ARG;
  }
  *out = nullptr;
  if (n < 16 * (int64_t)kL || (n & (n - 1)) || n / kL > 1024) {
    set_error("fb_shard_plan_create: n must be a power of two with 16 <= n / 8192 <= 1024");
    return FB_ERR_PLAN;
  }
  DevGuard dg_(device);
  int rc = cuda_status(dg_.err, "cudaSetDevice");
  if (rc) return rc;
  auto* sp = new fb_shard_plan();
  sp->n = n;
  sp->m = n / kL;
  sp->device = device;
  rc = upload_table(&sp->tw_m, sp->m, 0);
  if (!rc) rc = upload_table(&sp->tw_big, n, 2);
  if (!rc) rc = upload_table(&sp->tw_l, kL, 1);
  if (rc) {
    fb_shard_plan_destroy(sp);
    return rc;
  }
  *out = sp;
  return FB_OK;
}

int fb_shard_plan_dims(const fb_shard_plan* sp, int64_t* l, int64_t* m) {
  if (!sp) {
    set_error("fb_shard_plan_dims: null plan");
    return FB_ERR_ARG;
  }
  if (l) *l = sp->l;
  if (m) *m = sp->m;
  return FB_OK;
}

int fb_shard_columns(fb_shard_plan* sp, const void* in, void* out, int64_t C, int64_t tau0,
                     int64_t lp, int inverse, void* stream) {
  if (!sp || !in || !out) {
    set_error("fb_shard_columns: null argument");
    return FB_ERR_ARG;
  }
  const uint32_t TAU = (uint32_t)(kBigTile / sp->m);
  if (C < 1 || lp < TAU || lp % TAU || tau0 < 0 || tau0 + lp > sp->l || C > 65535) {
    set_error("fb_shard_columns: bad shard geometry (lp must be a multiple of 8192 / m)");
    return FB_ERR_DIM;
  }
  DevGuard dg_(sp->device);
  int rc = cuda_status(dg_.err, "cudaSetDevice");
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t sm = padded_len(kBigTile) * sizeof(float2);
  const dim3 g((unsigned)(lp / TAU), (unsigned)C);
  const float scale = 1.0f / (float)sp->n;
  with_small(sp->m, [&](auto sc) {
    constexpr int SM = decltype(sc)::value;
    if (inverse) {
      auto k = tp_shard_cols_kernel<+1, SM>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k<<<g, kBigThreads, sm, s>>>((const float2*)in, (float2*)out, sp->tw_m, sp->tw_big,
                                   (uint32_t)sp->m, (uint32_t)lp, (uint32_t)tau0, scale, ShardSig());
    } else {
      auto k = tp_shard_cols_kernel<-1, SM>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k<<<g, kBigThreads, sm, s>>>((const float2*)in, (float2*)out, sp->tw_m, sp->tw_big,
                                   (uint32_t)sp->m, (uint32_t)lp, (uint32_t)tau0, scale, ShardSig());
    }
  });
  return cuda_status(cudaGetLastError(), "fb_shard_columns");
}

// Pass 1 straight from the real signals (pairs packed on the fly) / pass 3
// straight into them (unpacked, + D skip): the layer's glue fused into the
// column passes (see ShardSig).
static int shard_cols_sig(fb_shard_plan* sp, const void* x_in, void* x_out, int dtype, ShardSig sg,
                          int64_t tau0, int64_t lp, int inverse, cudaStream_t s, const char* name) {
  const uint32_t TAU = (uint32_t)(kBigTile / sp->m);
  const int64_t C = ((int64_t)(sg.B + 1) / 2) * sg.H;
  if (sg.B < 1 || sg.H < 1 || sg.half < 1 || sg.half > sp->m || lp < TAU || lp % TAU || tau0 < 0 ||
      tau0 + lp > sp->l || C > 65535) {
    set_error(std::string(name) + ": bad shard geometry");
    return FB_ERR_DIM;
  }
  DevGuard dg_(sp->device);
  int rc = cuda_status(dg_.err, "cudaSetDevice");
  if (rc) return rc;
  const size_t sm = padded_len(kBigTile) * sizeof(float2);
  const dim3 g((unsigned)(lp / TAU), (unsigned)C);
  const float scale = 1.0f / (float)sp->n;
  with_io(dtype, [&](auto io) {
    using IO = decltype(io);
    with_small(sp->m, [&](auto sc) {
      constexpr int SM = decltype(sc)::value;
      if (inverse) {
        auto k = tp_shard_cols_kernel<+1, SM, IO>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k<<<g, kBigThreads, sm, s>>>((const float2*)x_in, nullptr, sp->tw_m, sp->tw_big, (uint32_t)sp->m,
                                     (uint32_t)lp, (uint32_t)tau0, scale, sg);
      } else {
        auto k = tp_shard_cols_kernel<-1, SM, IO>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k<<<g, kBigThreads, sm, s>>>(nullptr, (float2*)x_out, sp->tw_m, sp->tw_big, (uint32_t)sp->m,
                                     (uint32_t)lp, (uint32_t)tau0, scale, sg);
      }
    });
  });
  return cuda_status(cudaGetLastError(), name);
}

int fb_shard_columns_from_signals(fb_shard_plan* sp, const void* sig, int dtype, void* out, int64_t B,
                                  int64_t H, int64_t half, int64_t tau0, int64_t lp, void* stream) {
  if (!sp || !sig || !out) {
    set_error("fb_shard_columns_from_signals: null argument");
    return FB_ERR_ARG;
  }
  ShardSig sg;
  sg.sig = sig;
  sg.B = (int)B;
  sg.H = (int)H;
  sg.half = (int)half;
  return shard_cols_sig(sp, nullptr, out, dtype, sg, tau0, lp, 0, (cudaStream_t)stream,
                        "fb_shard_columns_from_signals");
}

int fb_shard_columns_to_signals(fb_shard_plan* sp, const void* in, void* sig_out, int dtype,
                                const void* skip, const float* D, int64_t B, int64_t H, int64_t half,
                                int64_t tau0, int64_t lp, void* stream) {
  if (!sp || !in || !sig_out || (skip && !D)) {
    set_error("fb_shard_columns_to_signals: null argument");
    return FB_ERR_ARG;
  }
  ShardSig sg;
  sg.out = sig_out;
  sg.skip = skip;
  sg.D = D;
  sg.B = (int)B;
  sg.H = (int)H;
  sg.half = (int)half;
  return shard_cols_sig(sp, in, nullptr, dtype, sg, tau0, lp, 1, (cudaStream_t)stream,
                        "fb_shard_columns_to_signals");
}

int fb_shard_rows(fb_shard_plan* sp, void* rows, const void* kf2, void* kf2_out, int64_t C,
                  int64_t mp, int mode, float scale, void* stream) {
  if (!sp || !rows || (mode == 0 && !kf2) || (mode == 1 && !kf2_out)) {
    set_error("fb_shard_rows: null argument");
    return FB_ERR_ARG;
  }
  if (C < 1 || mp < 1 || C * mp > (int64_t)1 << 31) {
    set_error("fb_shard_rows: bad shard geometry");
    return FB_ERR_DIM;
  }
  DevGuard dg_(sp->device);
  int rc = cuda_status(dg_.err, "cudaSetDevice");
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t sm = pass2_smem<float>();
  auto* x1 = reinterpret_cast<CxT<float>*>(rows);
  if (mode == 0) {
    auto k = tp_pass2_kernel<float, 0>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<dim3((unsigned)(C * mp), 1), kL / 16, sm, s>>>(x1, (const float2*)kf2, nullptr, sp->tw_l,
                                                       1, (int)C, (int)mp, 1, 0.f, nullptr);
  } else {
    auto k = tp_pass2_kernel<float, 1>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<dim3((unsigned)(C * mp), 1), kL / 16, sm, s>>>(x1, nullptr, (float2*)kf2_out, sp->tw_l,
                                                       1, (int)C, (int)mp, 1, scale, nullptr);
  }
  return cuda_status(cudaGetLastError(), "fb_shard_rows");
}

// rows [P][H][mp][l] in place: rows = IFFT_l(FFT_l(rows) kf2[h][a]) (unnormalised),
// the kernel rows [H][mp][l] shared by the P channel pairs of each head
int fb_shard_rows_pairs(fb_shard_plan* sp, void* rows, const void* kf2, int64_t P, int64_t H, int64_t mp,
                        void* stream) {
  if (!sp || !rows || !kf2) {
    set_error("fb_shard_rows_pairs: null argument");
    return FB_ERR_ARG;
  }
  if (P < 1 || H < 1 || mp < 1 || P * H * mp > (int64_t)1 << 31) {
    set_error("fb_shard_rows_pairs: bad shard geometry");
    return FB_ERR_DIM;
  }
  DevGuard dg_(sp->device);
  int rc = cuda_status(dg_.err, "cudaSetDevice");
  if (rc) return rc;
  const size_t sm = pass2_smem<float>();
  auto k = tp_pass2_kernel<float, 0>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, sp->device);
  const int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(P, (2 * sms + H * mp - 1) / (H * mp)));
  const int ppc = (int)((P + chunks - 1) / chunks);
  k<<<dim3((unsigned)(H * mp), (unsigned)chunks), kL / 16, sm, (cudaStream_t)stream>>>(
      reinterpret_cast<CxT<float>*>(rows), (const float2*)kf2, nullptr, sp->tw_l, (int)P, (int)H, (int)mp,
      ppc, 0.f, nullptr);
  return cuda_status(cudaGetLastError(), "fb_shard_rows_pairs");
}

// The sharded backward's row pass, CTA per (h, a) over all P pairs (fixed
// order, deterministic): DY = FFT_l(dy row), U = FFT_l(u row),
// S += conj(U) DY, dy row <- IFFT_l(DY conj(kf2)); finally wdk[h][a] =
// IFFT_l(S) (unnormalised, complex f32 [H][mp][l]).
int fb_shard_rows_bwd(fb_shard_plan* sp, void* dy_rows, const void* u_rows, const void* kf2, void* wdk,
                      int64_t P, int64_t H, int64_t mp, void* stream) {
  if (!sp || !dy_rows || !u_rows || !kf2 || !wdk) {
    set_error("fb_shard_rows_bwd: null argument");
    return FB_ERR_ARG;
  }
  if (P < 1 || H < 1 || mp < 1 || P * H * mp > (int64_t)1 << 31) {
    set_error("fb_shard_rows_bwd: bad shard geometry");
    return FB_ERR_DIM;
  }
  DevGuard dg_(sp->device);
  int rc = cuda_status(dg_.err, "cudaSetDevice");
  if (rc) return rc;
  const size_t sm = pass2_bwd_smem<float>();
  auto k = tp_pass2_bwd_kernel<float, false>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k<<<(unsigned)(H * mp), kL / 16, sm, (cudaStream_t)stream>>>(
      reinterpret_cast<CxT<float>*>(dy_rows), reinterpret_cast<const CxT<float>*>(u_rows), (const float2*)kf2,
      (float2*)wdk, sp->tw_l, (int)P, (int)H, (int)mp);
  return cuda_status(cudaGetLastError(), "fb_shard_rows_bwd");
}

}  // extern "C"
