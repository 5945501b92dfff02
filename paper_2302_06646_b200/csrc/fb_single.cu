// FlashButterfly-B200 single-pass engine (K1 spectrum, K2 forward, K4a
// backward) for transforms that fit in shared memory (n <= 8192, fp32).
//
// Reference path replaced (regularize.cpp:149-190 -> conv_channel :112-138
// -> conv_butterfly butterfly.cpp:187-210 -> apply_plan x3):
//   * the kernel FFT (butterfly.cpp:205, recomputed per channel by the
//     reference) is hoisted into sp_prep_kernel, once per head, scaled by
//     1/n so the inverse needs no extra pass;
//   * two real channels (b, b+1) of one head ride in the real and imaginary
//     parts of one complex signal (K is real, so conv is linear per part);
//   * u is read from HBM once, y written once; the spectrum never leaves the
//     SM: forward passes -> (x) k_f in registers -> inverse passes.
#include <algorithm>

#include "fb_common.cuh"
#include "fb_fft.cuh"
#include "fb_internal.h"

namespace fb {

// Transform-position value of a length-N channel: zero extension (causal,
// or circular kernels) or periodic extension (circular signals, n > N).
template <typename IO>
__device__ __forceinline__ float sig_at(const IO* __restrict__ p, uint32_t t, uint32_t N,
                                        bool periodic) {
  if (t < N) return ld(p + t);
  if (periodic) return ld(p + (t & (N - 1)));
  return 0.f;
}

// ---------------------------------------------------------------- K1 (spectrum)
// kf[h][e] = FFT_n(zero-pad(kbar[h]))[e] / n
template <int SMALL>
__global__ void __launch_bounds__(512) sp_spectrum_kernel(const float* __restrict__ kbar,
                                                           float2* __restrict__ kf,
                                                           const float2* __restrict__ tw,
                                                           uint32_t N, uint32_t n) {
  extern __shared__ float2 smem[];
  const uint32_t h = blockIdx.x, j = threadIdx.x, stride = n / 16;
  const float* kh = kbar + (size_t)h * N;
  float2 v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const uint32_t t = j + r * stride;
    v[r] = make_float2(t < N ? __ldg(kh + t) : 0.f, 0.f);
  }
  dft_reg<-1, 16>(v);
  stockham_store<16>(smem, v, j, 0, 1, 1);
  __syncthreads();
  smem_passes<-1, SMALL>(smem, n, 1, 16, stride, tw);
  stockham_load_twiddle<-1, 16>(smem, v, j, 0, n, 1, stride, tw);
  dft_reg<-1, 16>(v);
  const float inv_n = 1.0f / (float)n;
  float2* out = kf + (size_t)h * n;
#pragma unroll
  for (int r = 0; r < 16; ++r) out[j + r * stride] = cscale(v[r], inv_n);
}

// ---------------------------------------------------------------- K2 forward
// One CTA = one (head h, channel pair b0=2*blockIdx.y, b1=b0+1); T = n/16.
template <typename IO, int SMALL>
__global__ void __launch_bounds__(512) sp_fwd_kernel(const IO* __restrict__ u, IO* __restrict__ y,
                                                      const float2* __restrict__ kf,
                                                      const float* __restrict__ D,
                                                      const float2* __restrict__ tw, int B, int H,
                                                      uint32_t N, uint32_t n, int periodic) {
  extern __shared__ float2 smem[];
  const int h = blockIdx.x;
  const int b0 = 2 * blockIdx.y, b1 = b0 + 1;
  const bool has1 = b1 < B;
  const size_t off0 = ((size_t)b0 * H + h) * N, off1 = ((size_t)b1 * H + h) * N;
  const uint32_t j = threadIdx.x, stride = n / 16;
  float2 v[16];
  // forward pass 1 (Ns = 1) straight from HBM: pair (u[b0], u[b1]) -> complex
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const uint32_t t = j + r * stride;
    v[r].x = sig_at(u + off0, t, N, periodic);
    v[r].y = has1 ? sig_at(u + off1, t, N, periodic) : 0.f;
  }
  dft_reg<-1, 16>(v);
  stockham_store<16>(smem, v, j, 0, 1, 1);
  __syncthreads();
  smem_passes<-1, SMALL>(smem, n, 1, 16, stride, tw);
  // last forward pass (Ns = n/16): thread j ends up owning bins j + r n/16,
  // exactly the points the first inverse pass (Ns = 1) needs: the pointwise
  // product with k_f and the first inverse DFT block stay in registers.
  stockham_load_twiddle<-1, 16>(smem, v, j, 0, n, 1, stride, tw);
  dft_reg<-1, 16>(v);
  const float2* kh = kf + (size_t)h * n;
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = cmul(v[r], __ldg(kh + j + r * stride));
  dft_reg<+1, 16>(v);
  __syncthreads();
  stockham_store<16>(smem, v, j, 0, 1, 1);
  __syncthreads();
  smem_passes<+1, SMALL>(smem, n, 1, 16, stride, tw);
  stockham_load_twiddle<+1, 16>(smem, v, j, 0, n, 1, stride, tw);
  dft_reg<+1, 16>(v);
  // epilogue: y = conv + D u, straight to HBM (u re-read hits L2)
  const float d = __ldg(D + h);
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const uint32_t t = j + r * stride;
    if (t < N) {
      st(y + off0 + t, fmaf(d, ld(u + off0 + t), v[r].x));
      if (has1) st(y + off1 + t, fmaf(d, ld(u + off1 + t), v[r].y));
    }
  }
}

// ---------------------------------------------------------------- K4a backward
// One CTA = one (head h, chunk of channel pairs).  Per pair:
//   DY = FFT(dy pair), U = FFT(u pair)            (2 forward transforms)
//   acc += conj(U) DY        (thread-owned bins, smem, fixed order => determ.)
//   du = IFFT(DY conj(k_f)) + D dy                (1 inverse transform)
// plus dD partial = sum dy u.  Partials per chunk are reduced by
// sp_dk_finalize_kernel in a fixed order.
template <typename IO, int SMALL>
__global__ void __launch_bounds__(512) sp_bwd_kernel(
    const IO* __restrict__ dy, const IO* __restrict__ u, IO* __restrict__ du,
    const float2* __restrict__ kf, const float* __restrict__ D, const float2* __restrict__ tw,
    float2* __restrict__ spart, float* __restrict__ ddpart, int B, int H, uint32_t N, uint32_t n,
    int periodic, int pairs_per_chunk) {
  extern __shared__ float2 smem[];
  float2* acc = smem + padded_len(n);  // [n], thread-owned bins
  __shared__ float red[32];
  const int h = blockIdx.x, chunk = blockIdx.y, chunks = gridDim.y;
  const uint32_t j = threadIdx.x, stride = n / 16;
  const int npairs = (B + 1) / 2;
  const float2* kh = kf + (size_t)h * n;
  const float d = __ldg(D + h);
#pragma unroll
  for (int r = 0; r < 16; ++r) acc[j + r * stride] = make_float2(0.f, 0.f);
  float dd = 0.f;
  const int p_begin = chunk * pairs_per_chunk;
  const int p_end = min(npairs, p_begin + pairs_per_chunk);
  for (int pr = p_begin; pr < p_end; ++pr) {
    const int b0 = 2 * pr, b1 = b0 + 1;
    const bool has1 = b1 < B;
    const size_t off0 = ((size_t)b0 * H + h) * N, off1 = ((size_t)b1 * H + h) * N;
    float2 gv[16], v[16];
    // ---- FFT(dy)
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t t = j + r * stride;
      v[r].x = sig_at(dy + off0, t, N, periodic);
      v[r].y = has1 ? sig_at(dy + off1, t, N, periodic) : 0.f;
      if (t < N) {
        dd = fmaf(v[r].x, ld(u + off0 + t), dd);
        if (has1) dd = fmaf(v[r].y, ld(u + off1 + t), dd);
      }
    }
    dft_reg<-1, 16>(v);
    __syncthreads();
    stockham_store<16>(smem, v, j, 0, 1, 1);
    __syncthreads();
    smem_passes<-1, SMALL>(smem, n, 1, 16, stride, tw);
    stockham_load_twiddle<-1, 16>(smem, gv, j, 0, n, 1, stride, tw);
    dft_reg<-1, 16>(gv);
    // ---- FFT(u)
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t t = j + r * stride;
      v[r].x = sig_at(u + off0, t, N, periodic);
      v[r].y = has1 ? sig_at(u + off1, t, N, periodic) : 0.f;
    }
    dft_reg<-1, 16>(v);
    __syncthreads();
    stockham_store<16>(smem, v, j, 0, 1, 1);
    __syncthreads();
    smem_passes<-1, SMALL>(smem, n, 1, 16, stride, tw);
    stockham_load_twiddle<-1, 16>(smem, v, j, 0, n, 1, stride, tw);
    dft_reg<-1, 16>(v);
    // ---- spectral products
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t e = j + r * stride;
      const float2 a = acc[e];
      acc[e] = cadd(a, cconjmul(v[r], gv[r]));
      v[r] = cmulc(gv[r], __ldg(kh + e));
    }
    // ---- du = IFFT(DY conj(kf)) + D dy
    dft_reg<+1, 16>(v);
    __syncthreads();
    stockham_store<16>(smem, v, j, 0, 1, 1);
    __syncthreads();
    smem_passes<+1, SMALL>(smem, n, 1, 16, stride, tw);
    stockham_load_twiddle<+1, 16>(smem, v, j, 0, n, 1, stride, tw);
    dft_reg<+1, 16>(v);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t t = j + r * stride;
      if (t < N) {
        st(du + off0 + t, fmaf(d, ld(dy + off0 + t), v[r].x));
        if (has1) st(du + off1 + t, fmaf(d, ld(dy + off1 + t), v[r].y));
      }
    }
  }
  // partial spectra + dD (deterministic block reduction)
  float2* sp = spart + ((size_t)h * chunks + chunk) * n;
#pragma unroll
  for (int r = 0; r < 16; ++r) sp[j + r * stride] = acc[j + r * stride];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dd += __shfl_xor_sync(0xffffffffu, dd, o);
  if ((j & 31) == 0) red[j >> 5] = dd;
  __syncthreads();
  if (j == 0) {
    float t = 0.f;
    for (uint32_t w = 0; w < (blockDim.x + 31) / 32; ++w) t += red[w];
    ddpart[(size_t)h * chunks + chunk] = t;
  }
}

// dKbar[h][t] = scale * Re IFFT(sum_c spart[h][c])[t] / n ; dD[h] = sum_c ddpart.
template <int SMALL>
__global__ void __launch_bounds__(512) sp_dk_finalize_kernel(
    const float2* __restrict__ spart, const float* __restrict__ ddpart, int chunks,
    float* __restrict__ dkbar, float* __restrict__ dD, const float2* __restrict__ tw, uint32_t N,
    uint32_t n, float scale) {
  extern __shared__ float2 smem[];
  const uint32_t h = blockIdx.x, j = threadIdx.x, stride = n / 16;
  float2 v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = make_float2(0.f, 0.f);
  for (int c = 0; c < chunks; ++c) {
    const float2* sp = spart + ((size_t)h * chunks + c) * n;
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = cadd(v[r], __ldg(sp + j + r * stride));
  }
  dft_reg<+1, 16>(v);
  stockham_store<16>(smem, v, j, 0, 1, 1);
  __syncthreads();
  smem_passes<+1, SMALL>(smem, n, 1, 16, stride, tw);
  stockham_load_twiddle<+1, 16>(smem, v, j, 0, n, 1, stride, tw);
  dft_reg<+1, 16>(v);
  const float s = scale / (float)n;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const uint32_t t = j + r * stride;
    if (t < N) dkbar[(size_t)h * N + t] = v[r].x * s;
  }
  if (j == 0) {
    float t = 0.f;
    for (int c = 0; c < chunks; ++c) t += ddpart[(size_t)h * chunks + c];
    dD[h] = t;
  }
}

// ---------------------------------------------------------------- host side
namespace {

int log2i(int64_t n) {
  int k = 0;
  while ((int64_t(1) << k) < n) ++k;
  return k;
}

template <int SMALL>
struct SpKernels {
  template <typename IO>
  static void fwd(dim3 g, dim3 b, size_t sm, cudaStream_t s, const void* u, void* y,
                  const fb_plan* p, int B) {
    auto k = sp_fwd_kernel<IO, SMALL>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<g, b, sm, s>>>((const IO*)u, (IO*)y, p->kf, p->d, p->tw_n, B, (int)p->H, (uint32_t)p->N,
                       (uint32_t)p->n, p->periodic ? 1 : 0);
  }
  template <typename IO>
  static void bwd(dim3 g, dim3 b, size_t sm, cudaStream_t s, const void* dy, const void* u,
                  void* du, const fb_plan* p, float2* spart, float* ddpart, int B, int ppc) {
    auto k = sp_bwd_kernel<IO, SMALL>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<g, b, sm, s>>>((const IO*)dy, (const IO*)u, (IO*)du, p->kf, p->d, p->tw_n, spart, ddpart,
                       B, (int)p->H, (uint32_t)p->N, (uint32_t)p->n, p->periodic ? 1 : 0, ppc);
  }
  static void spectrum(dim3 g, dim3 b, size_t sm, cudaStream_t s, const fb_plan* p) {
    auto k = sp_spectrum_kernel<SMALL>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<g, b, sm, s>>>(p->kbar, p->kf, p->tw_n, (uint32_t)p->N, (uint32_t)p->n);
  }
  static void finalize(dim3 g, dim3 b, size_t sm, cudaStream_t s, const fb_plan* p,
                       const float2* spart, const float* ddpart, int chunks, float* dkbar,
                       float* dD) {
    auto k = sp_dk_finalize_kernel<SMALL>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const float scale = p->periodic ? (float)p->N / (float)p->n : 1.0f;
    k<<<g, b, sm, s>>>(spart, ddpart, chunks, dkbar, dD, p->tw_n, (uint32_t)p->N,
                       (uint32_t)p->n, scale);
  }
};

template <class F>
void with_small(int64_t n, F&& f) {
  switch (log2i(n) % 4) {
    case 0: f(SpKernels<1>{}); break;
    case 1: f(SpKernels<2>{}); break;
    case 2: f(SpKernels<4>{}); break;
    default: f(SpKernels<8>{}); break;
  }
}

int chunks_for(const fb_plan* p, int64_t B) {
  // enough CTAs to cover the SMs ~2x while keeping the per-head reduction
  // short; each chunk owns >= 1 pair.
  const int64_t npairs = (B + 1) / 2;
  int64_t c = (2 * p->num_sms + p->H - 1) / p->H;
  c = std::max<int64_t>(1, std::min<int64_t>(c, npairs));
  return (int)c;
}

}  // namespace

int sp_prep(fb_plan* p, const float* K, cudaStream_t s) {
  int rc = regularize_bank_dev(p, K, s);
  if (rc) return rc;
  const size_t sm = padded_len((uint32_t)p->n) * sizeof(float2);
  with_small(p->n, [&](auto ks) { ks.spectrum(dim3((unsigned)p->H), dim3((unsigned)(p->n / 16)), sm, s, p); });
  return cuda_status(cudaGetLastError(), "sp_prep");
}

int sp_fwd(fb_plan* p, const void* u, void* y, int64_t B, cudaStream_t s) {
  const size_t sm = padded_len((uint32_t)p->n) * sizeof(float2);
  const dim3 g((unsigned)p->H, (unsigned)((B + 1) / 2)), b((unsigned)(p->n / 16));
  with_small(p->n, [&](auto ks) {
    switch (p->dtype) {
      case FB_F32: ks.template fwd<float>(g, b, sm, s, u, y, p, (int)B); break;
      case FB_BF16: ks.template fwd<__nv_bfloat16>(g, b, sm, s, u, y, p, (int)B); break;
      default: ks.template fwd<__half>(g, b, sm, s, u, y, p, (int)B); break;
    }
  });
  return cuda_status(cudaGetLastError(), "sp_fwd");
}

size_t sp_workspace(const fb_plan* p, int64_t B) {
  const int c = chunks_for(p, B);
  size_t bytes = (size_t)p->H * c * p->n * sizeof(float2);  // spectral partials
  bytes += (size_t)p->H * c * sizeof(float);                 // dD partials
  bytes = (bytes + 255) & ~size_t(255);
  bytes += (size_t)p->H * p->N * sizeof(float);              // dKbar scratch
  return bytes + 256;
}

int sp_bwd(fb_plan* p, const void* dy, const void* u, void* du, float* dK, float* dKbar, float* dD,
           int64_t B, void* ws, cudaStream_t s) {
  const int chunks = chunks_for(p, B);
  const int64_t npairs = (B + 1) / 2;
  const int ppc = (int)((npairs + chunks - 1) / chunks);
  char* w = (char*)ws;
  float2* spart = (float2*)w;
  size_t off = (size_t)p->H * chunks * p->n * sizeof(float2);
  float* ddpart = (float*)(w + off);
  off += (size_t)p->H * chunks * sizeof(float);
  off = (off + 255) & ~size_t(255);
  float* dkbar = dKbar ? dKbar : (float*)(w + off);
  const size_t sm1 = padded_len((uint32_t)p->n) * sizeof(float2);
  const size_t smb = sm1 + p->n * sizeof(float2);
  const dim3 g((unsigned)p->H, (unsigned)chunks), b((unsigned)(p->n / 16));
  with_small(p->n, [&](auto ks) {
    switch (p->dtype) {
      case FB_F32: ks.template bwd<float>(g, b, smb, s, dy, u, du, p, spart, ddpart, (int)B, ppc); break;
      case FB_BF16: ks.template bwd<__nv_bfloat16>(g, b, smb, s, dy, u, du, p, spart, ddpart, (int)B, ppc); break;
      default: ks.template bwd<__half>(g, b, smb, s, dy, u, du, p, spart, ddpart, (int)B, ppc); break;
    }
    ks.finalize(dim3((unsigned)p->H), b, sm1, s, p, spart, ddpart, chunks, dkbar, dD);
  });
  int rc = cuda_status(cudaGetLastError(), "sp_bwd");
  if (rc) return rc;
  return regularizer_backward_dev(p, dkbar, dK, s);
}

}  // namespace fb
