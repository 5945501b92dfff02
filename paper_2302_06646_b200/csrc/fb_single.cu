// FlashButterfly-B200 single-pass engine (K1 spectrum, K2 forward, K4a
// backward) for transforms that fit in shared memory (n <= 8192, fp32).
//
// Reference path replaced (regularize.cpp:149-190 -> conv_channel :112-138
// -> conv_butterfly butterfly.cpp:187-210 -> apply_plan x3):
//   * the kernel FFT (butterfly.cpp:205, recomputed per channel by the
//     reference) is hoisted into sp_spectrum_kernel, once per head, scaled
//     by 1/n so the inverse needs no extra pass;
//   * two real channels (b, b+1) of one head ride in the real and imaginary
//     parts of one complex signal (K is real, so conv is linear per part);
//   * each CTA owns one head and a run of channel pairs: k_f is staged in
//     shared memory once, the next pair's rows are prefetched by TMA bulk
//     copies (cp.async.bulk + mbarrier) while the current pair transforms;
//   * u is read from HBM once, y written once; the spectrum never leaves the
//     SM: forward passes -> (x) k_f in registers -> inverse passes.
#include <algorithm>

#include "fb_common.cuh"
#include "fb_fft.cuh"
#include "fb_internal.h"
#include "fb_ptx.cuh"
#include "fb_reg.cuh"

namespace fb {

// Staged signal value at transform position t of a length-N row in smem:
// zero extension (causal) or periodic extension (circular with n > N).
template <typename IO>
__device__ __forceinline__ float stage_at(const IO* row, uint32_t t, uint32_t N, bool periodic) {
  if (t < N) return tof(row[t]);
  if (periodic) return tof(row[t & (N - 1)]);
  return 0.f;
}

template <typename IO>
__host__ __device__ constexpr uint32_t row_pitch(uint32_t N) {
  // row stride in elements, 16-byte multiple (TMA bulk granularity)
  return (N + (16 / sizeof(IO)) - 1) / (16 / sizeof(IO)) * (16 / sizeof(IO));
}

// Copy rows [b0, b0+nrows) x head h of `src` ([B][H][N]) into smem rows of
// pitch P.  TMA bulk path when every row is 16-byte aligned, else a
// cooperative (synchronous) copy.  Returns the number of bytes in flight.
template <typename IO>
__device__ __forceinline__ uint32_t stage_rows(IO* dst, const IO* const* srcs, int nrows, uint32_t N,
                                               uint32_t P, bool tma, uint64_t* bar) {
  if (tma) {
    uint32_t bytes = 0;
    if (threadIdx.x == 0) {
      const uint32_t rb = N * (uint32_t)sizeof(IO);
      bytes = rb * nrows;
      ptx::fence_proxy_async_smem();
      ptx::mbar_arrive_expect_tx(bar, bytes);
      for (int r = 0; r < nrows; ++r) ptx::bulk_g2s(dst + r * P, srcs[r], rb, bar);
    }
    return bytes;
  }
  for (int r = 0; r < nrows; ++r)
    for (uint32_t t = threadIdx.x; t < N; t += blockDim.x) dst[r * P + t] = __ldg(srcs[r] + t);
  return 0;
}

template <int LOG2N>
__device__ __forceinline__ void load_table(float2* tab, const float2* __restrict__ g) {
  for (uint32_t i = threadIdx.x; i < FftShape<LOG2N>::tab_len; i += blockDim.x) tab[i] = __ldg(g + i);
}

// ---------------------------------------------------------------- K1 (spectrum)
// One CTA per head, the whole of K1 in one launch: kbar[h] = squash(smooth(
// dropout(K[h]))) (fb_reg.cuh, fp64) is written once for the backward's mask
// and transformed in place: kf[h][f] = FFT_n(zero-pad(kbar[h]))[f] / n.  With
// kf_tc set (tcgen05 path) the spectrum goes out instead in the tensor-core
// layout [h][f1 64][f2 128] (f = f1 + 64 f2) with the skip gain folded in
// as a flat spectrum, k_f' = k_f + D/n, as fp16 pairs scaled by the power
// of two that brings the head's largest component to <= 2^15; kf_scale[h]
// is the inverse (the tensor-core kernels fold it into their output).
// (two CTAs per SM: one wave for H <= 2 x the SM count; per-head work is a
// latency-bound chain, so co-residency is what hides it)
template <int LOG2N>
__global__ void __launch_bounds__(FftShape<LOG2N>::T, 2)
    sp_spectrum_kernel(const float* __restrict__ K, const uint8_t* __restrict__ keep,
                       float* __restrict__ kbar, float2* __restrict__ kf, __half2* __restrict__ kf_tc,
                       float* __restrict__ kf_scale, const float* __restrict__ D,
                       const float2* __restrict__ tab_g, uint32_t N, int64_t p, double lambda,
                       double keep_scale, int freq, int tc_ver) {
  using S = FftShape<LOG2N>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ float red[32];
  float2* work = reinterpret_cast<float2*>(smem_raw);
  float2* tab = work + S::work_len;
  const uint32_t h = blockIdx.x, j = threadIdx.x;
  load_table<LOG2N>(tab, tab_g);
  const size_t base = (size_t)h * N;
  // the fp64 regularizer once per element in a rolled loop (its code inlined
  // sixteen times next to the FFT thrashed the instruction cache), staged in smem
  float* kb = reinterpret_cast<float*>(work);
  if (!freq && (size_t)N * 12 <= (size_t)S::work_len * sizeof(float2)) {
    // time smoothing: dropout(K) converted to fp64 once per element into
    // smem, then reg_value's tap sum (same order, same rounding) from there
    double* kd = reinterpret_cast<double*>(work);
    kb = reinterpret_cast<float*>(kd + N);
    // (unrolled: the K loads of all of a thread's elements in flight at once)
#pragma unroll 8
    for (uint32_t t = j; t < N; t += S::T) kd[t] = dropped(K, keep, keep_scale, base + t);
    __syncthreads();
    const double inv_w = 1.0 / (double)(2 * p + 1);
    const int pp = (int)p, Ni = (int)N;  // N <= 4096 here: 32-bit index math
#pragma unroll 1
    for (uint32_t t = j; t < N; t += S::T) {
      const int ti = (int)t;
      const int lo = ti >= pp ? ti - pp : 0;
      const int hi = (ti + pp < Ni - 1) ? ti + pp : Ni - 1;
      double acc = 0.0;
      for (int q = lo; q <= hi; ++q) acc += kd[q];
      const double sv = acc * inv_w;
      const double mag = fabs(sv) - lambda;
      const float kv = mag > 0.0 ? (float)copysign(mag, sv) : 0.0f;
      kbar[base + t] = kv;
      kb[t] = kv;
    }
  } else {
#pragma unroll 1
    for (uint32_t t = j; t < N; t += S::T) {
      const float kv = reg_value(K, keep, keep_scale, base, t, N, p, lambda, freq);
      kbar[base + t] = kv;
      kb[t] = kv;
    }
  }
  __syncthreads();
  float2 v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const uint32_t t = j + r * S::stride;
    v[r] = make_float2(t < N ? kb[t] : 0.f, 0.f);
  }
  __syncthreads();  // kb read before the FFT overwrites work
  dft_reg<-1, 16>(v);
  bfly_store<16, 1>(work, v, j);
  __syncthreads();
  mid_passes<-1, LOG2N, 16>(work, tab);
  bfly_load<-1, 16, S::n / 16, LOG2N>(work, tab, v, j);
  const float inv_n = 1.0f / (float)S::n;
  if (kf_tc == nullptr) {
    float2* out = kf + (size_t)h * S::n;
#pragma unroll
    for (int r = 0; r < 16; ++r) out[j + r * S::stride] = cscale(v[r], inv_n);
    return;
  }
  // f = j + r * stride -> its tensor-core slot (v2 / v1 layouts below), padded by one per 128
  const float dn = __ldg(D + h) * inv_n;
  float mx = 0.f;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    v[r] = cscale(v[r], inv_n);
    v[r].x += dn;
    mx = fmaxf(mx, fmaxf(fabsf(v[r].x), fabsf(v[r].y)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((j & 31) == 0) red[j >> 5] = mx;
  __syncthreads();
  if (j < 32) {
    float m = j < (S::T + 31) / 32 ? red[j] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (j == 0) red[0] = m;
  }
  __syncthreads();
  int e = 0;
  if (red[0] > 0.f) frexpf(red[0], &e);
  const float sc = red[0] > 0.f ? ldexpf(1.f, 15 - e) : 1.f;
  if (j == 0) kf_scale[h] = red[0] > 0.f ? ldexpf(1.f, e - 15) : 1.f;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const uint32_t f = j + r * S::stride;
    // v2: [f2 / 4][f1][f2 % 4], f1 = f % 128, f2 = f / 128 (coalesced per-lane loads)
    const uint32_t i = tc_ver == 2 ? (((f >> 9) * 128u + (f & 127u)) * 4u + ((f >> 7) & 3u))
                                   : (f & 63u) * 128u + (f >> 6);
    work[i + (i >> 7)] = cscale(v[r], sc);
  }
  __syncthreads();
  __half2* out = kf_tc + (size_t)h * S::n;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const uint32_t i = j + r * S::stride;
    const float2 w = work[i + (i >> 7)];
    out[i] = __floats2half2_rn(w.x, w.y);
  }
}

// ---------------------------------------------------------------- K2 forward
// grid (H, chunks): CTA (h, c) runs channel pairs [c*ppc, (c+1)*ppc).
template <typename IO, int LOG2N>
__global__ void __launch_bounds__(FftShape<LOG2N>::T, 1)
    sp_fwd_kernel(const IO* __restrict__ u, IO* __restrict__ y, const float2* __restrict__ kf,
                  const float* __restrict__ D, const float2* __restrict__ tab_g, int B, int H,
                  uint32_t N, int periodic, int ppc, int tma) {
  using S = FftShape<LOG2N>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[2];
  const uint32_t P = row_pitch<IO>(N);
  float2* work = reinterpret_cast<float2*>(smem_raw);
  float2* kfs = work + S::work_len;
  float2* tab = kfs + S::n;
  IO* stage = reinterpret_cast<IO*>(tab + ((S::tab_len + 1) & ~1u));  // [2][2][P]
  const int h = blockIdx.x, j = threadIdx.x;
  const int npairs = (B + 1) / 2;
  const int p0 = blockIdx.y * ppc, p1 = min(npairs, p0 + ppc);
  if (p0 >= p1) return;
  if (j == 0) {
    ptx::mbar_init(&bars[0], 1);
    ptx::mbar_init(&bars[1], 1);
    ptx::fence_barrier_init();
  }
  load_table<LOG2N>(tab, tab_g);
  {
    const float4* src = reinterpret_cast<const float4*>(kf + (size_t)h * S::n);
    float4* dst = reinterpret_cast<float4*>(kfs);
    for (uint32_t i = j; i < S::n / 2; i += S::T) dst[i] = __ldg(src + i);
  }
  const float d = __ldg(D + h);
  __syncthreads();
  auto issue = [&](int pr, int buf) {
    const int b0 = 2 * pr;
    const IO* rows[2] = {u + ((size_t)b0 * H + h) * N, u + ((size_t)(b0 + 1) * H + h) * N};
    stage_rows<IO>(stage + buf * 2 * P, rows, (b0 + 1 < B) ? 2 : 1, N, P, tma, &bars[buf]);
  };
  if (tma) issue(p0, 0);
  for (int pr = p0, it = 0; pr < p1; ++pr, ++it) {
    const int buf = tma ? (it & 1) : 0;
    const int b0 = 2 * pr, b1 = b0 + 1;
    const bool has1 = b1 < B;
    if (tma) {
      ptx::mbar_wait(&bars[buf], (it >> 1) & 1);
      if (pr + 1 < p1) issue(pr + 1, buf ^ 1);
    } else {
      issue(pr, 0);
      __syncthreads();
    }
    const IO* s0 = stage + buf * 2 * P;
    const IO* s1 = s0 + P;
    float2 v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t t = j + r * S::stride;
      v[r].x = stage_at(s0, t, N, periodic);
      v[r].y = has1 ? stage_at(s1, t, N, periodic) : 0.f;
    }
    dft_reg<-1, 16>(v);
    bfly_store<16, 1>(work, v, j);
    __syncthreads();
    mid_passes<-1, LOG2N, 16>(work, tab);
    // last forward pass (Ns = n/16): thread j owns bins j + r n/16, exactly
    // the points the first inverse pass (Ns = 1) needs, so the product with
    // k_f and the first inverse DFT block stay in registers.
    bfly_load<-1, 16, S::n / 16, LOG2N>(work, tab, v, j);
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = cmul(v[r], kfs[j + r * S::stride]);
    dft_reg<+1, 16>(v);
    __syncthreads();
    bfly_store<16, 1>(work, v, j);
    __syncthreads();
    mid_passes<+1, LOG2N, 16>(work, tab);
    bfly_load<+1, 16, S::n / 16, LOG2N>(work, tab, v, j);
    IO* y0 = y + ((size_t)b0 * H + h) * N;
    IO* y1 = y + ((size_t)b1 * H + h) * N;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t t = j + r * S::stride;
      if (t < N) {
        st(y0 + t, fmaf(d, tof(s0[t]), v[r].x));
        if (has1) st(y1 + t, fmaf(d, tof(s1[t]), v[r].y));
      }
    }
    __syncthreads();  // work + stage[buf] free for the next pair
  }
}

// ---------------------------------------------------------------- K4a backward
// grid (H, chunks).  Per pair:
//   DY = FFT(dy pair), U = FFT(u pair)            (2 forward transforms)
//   acc += conj(U) DY        (thread-owned bins in smem, fixed order)
//   du = IFFT(DY conj(k_f)) + D dy                (1 inverse transform)
// plus dD partial = sum dy u.  Per-chunk partials are reduced by
// sp_dk_finalize_kernel in a fixed order (deterministic, no atomics).
template <typename IO, int LOG2N, int NBUF>
__global__ void __launch_bounds__(FftShape<LOG2N>::T, 1)
    sp_bwd_kernel(const IO* __restrict__ dy, const IO* __restrict__ u, IO* __restrict__ du,
                  const float2* __restrict__ kf, const float* __restrict__ D,
                  const float2* __restrict__ tab_g, float2* __restrict__ spart,
                  float* __restrict__ ddpart, int B, int H, uint32_t N, int periodic, int ppc,
                  int tma) {
  using S = FftShape<LOG2N>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ float red[32];
  const uint32_t P = row_pitch<IO>(N);
  float2* work = reinterpret_cast<float2*>(smem_raw);
  float2* acc = work + S::work_len;  // [n], thread-owned bins
  float2* tab = acc + S::n;
  IO* stage = reinterpret_cast<IO*>(tab + ((S::tab_len + 1) & ~1u));  // [NBUF][4][P]
  const int h = blockIdx.x, chunk = blockIdx.y, chunks = gridDim.y;
  const uint32_t j = threadIdx.x;
  const int npairs = (B + 1) / 2;
  const float2* kh = kf + (size_t)h * S::n;
  const float d = __ldg(D + h);
  if (j == 0) {
    ptx::mbar_init(&bars[0], 1);
    ptx::mbar_init(&bars[1], 1);
    ptx::fence_barrier_init();
  }
  load_table<LOG2N>(tab, tab_g);
#pragma unroll
  for (int r = 0; r < 16; ++r) acc[j + r * S::stride] = make_float2(0.f, 0.f);
  float dd = 0.f;
  const int p0 = chunk * ppc, p1 = min(npairs, p0 + ppc);
  __syncthreads();
  // rows in a stage buffer: dy[b0], dy[b1], u[b0], u[b1]
  auto issue = [&](int pr, int buf) {
    const int b0 = 2 * pr;
    const bool two = b0 + 1 < B;
    IO* dst = stage + buf * 4 * P;
    const IO* rd[2] = {dy + ((size_t)b0 * H + h) * N, dy + ((size_t)(b0 + 1) * H + h) * N};
    const IO* ru[2] = {u + ((size_t)b0 * H + h) * N, u + ((size_t)(b0 + 1) * H + h) * N};
    if (tma) {
      if (j == 0) {
        const uint32_t rb = N * (uint32_t)sizeof(IO);
        const int nr = two ? 2 : 1;
        ptx::fence_proxy_async_smem();
        ptx::mbar_arrive_expect_tx(&bars[buf], 2 * nr * rb);
        for (int r = 0; r < nr; ++r) {
          ptx::bulk_g2s(dst + r * P, rd[r], rb, &bars[buf]);
          ptx::bulk_g2s(dst + (2 + r) * P, ru[r], rb, &bars[buf]);
        }
      }
    } else {
      stage_rows<IO>(dst, rd, two ? 2 : 1, N, P, false, nullptr);
      stage_rows<IO>(dst + 2 * P, ru, two ? 2 : 1, N, P, false, nullptr);
    }
  };
  if (tma && p0 < p1) issue(p0, 0);
  for (int pr = p0, it = 0; pr < p1; ++pr, ++it) {
    const int buf = (NBUF == 2 && tma) ? (it & 1) : 0;
    const int b0 = 2 * pr, b1 = b0 + 1;
    const bool has1 = b1 < B;
    if (tma) {
      ptx::mbar_wait(&bars[buf], NBUF == 2 ? ((it >> 1) & 1) : (it & 1));
      if (NBUF == 2 && pr + 1 < p1) issue(pr + 1, buf ^ 1);
    } else {
      issue(pr, 0);
      __syncthreads();
    }
    const IO* g0 = stage + buf * 4 * P;
    const IO* g1 = g0 + P;
    const IO* u0 = g0 + 2 * P;
    const IO* u1 = g0 + 3 * P;
    float2 gv[16], v[16];
    // ---- FFT(dy), with the dD partial from the staged rows
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t t = j + r * S::stride;
      v[r].x = stage_at(g0, t, N, periodic);
      v[r].y = has1 ? stage_at(g1, t, N, periodic) : 0.f;
      if (t < N) {
        dd = fmaf(v[r].x, tof(u0[t]), dd);
        if (has1) dd = fmaf(v[r].y, tof(u1[t]), dd);
      }
    }
    dft_reg<-1, 16>(v);
    bfly_store<16, 1>(work, v, j);
    __syncthreads();
    mid_passes<-1, LOG2N, 16>(work, tab);
    bfly_load<-1, 16, S::n / 16, LOG2N>(work, tab, gv, j);
    // ---- FFT(u)
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t t = j + r * S::stride;
      v[r].x = stage_at(u0, t, N, periodic);
      v[r].y = has1 ? stage_at(u1, t, N, periodic) : 0.f;
    }
    dft_reg<-1, 16>(v);
    __syncthreads();
    bfly_store<16, 1>(work, v, j);
    __syncthreads();
    mid_passes<-1, LOG2N, 16>(work, tab);
    bfly_load<-1, 16, S::n / 16, LOG2N>(work, tab, v, j);
    // ---- spectral products
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t e = j + r * S::stride;
      acc[e] = cadd(acc[e], cconjmul(v[r], gv[r]));
      v[r] = cmulc(gv[r], __ldg(kh + e));
    }
    // ---- du = IFFT(DY conj(kf)) + D dy
    dft_reg<+1, 16>(v);
    __syncthreads();
    bfly_store<16, 1>(work, v, j);
    __syncthreads();
    mid_passes<+1, LOG2N, 16>(work, tab);
    bfly_load<+1, 16, S::n / 16, LOG2N>(work, tab, v, j);
    IO* d0 = du + ((size_t)b0 * H + h) * N;
    IO* d1 = du + ((size_t)b1 * H + h) * N;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t t = j + r * S::stride;
      if (t < N) {
        st(d0 + t, fmaf(d, tof(g0[t]), v[r].x));
        if (has1) st(d1 + t, fmaf(d, tof(g1[t]), v[r].y));
      }
    }
    __syncthreads();
    if (NBUF == 1 && tma && pr + 1 < p1) issue(pr + 1, 0);
  }
  // partial spectra + dD (deterministic block reduction)
  float2* sp = spart + ((size_t)h * chunks + chunk) * S::n;
#pragma unroll
  for (int r = 0; r < 16; ++r) sp[j + r * S::stride] = acc[j + r * S::stride];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dd += __shfl_xor_sync(0xffffffffu, dd, o);
  if ((j & 31) == 0) red[j >> 5] = dd;
  __syncthreads();
  if (j == 0) {
    float t = 0.f;
    for (uint32_t w = 0; w < (S::T + 31) / 32; ++w) t += red[w];
    ddpart[(size_t)h * chunks + chunk] = t;
  }
}

// Backward tail, one CTA per head: dKbar[h][t] = scale * Re IFFT(sum_c
// spart[h][c])[t] / n (chunk partials summed in a fixed order), staged in
// smem and pushed through the regularizer chain rule (fb_reg.cuh) into
// dK[h]; dD[h] = sum_c ddpart (SIMT) or the lag-0 correlation dKbar[h][0]
// (tcgen05 path, where D is folded into k_f').  dkbar_out is optional.
template <int LOG2N>
__global__ void __launch_bounds__(FftShape<LOG2N>::T, 2)
    sp_dk_finalize_kernel(const float2* __restrict__ spart, const float* __restrict__ ddpart,
                          int chunks, float* __restrict__ dkbar_out, float* __restrict__ dD,
                          const float* __restrict__ kbar, const uint8_t* __restrict__ keep,
                          float* __restrict__ dK, const float2* __restrict__ tab_g, uint32_t N,
                          float scale, int64_t p, double keep_scale, int freq, int dd_lag0,
                          SpartMap map) {
  using S = FftShape<LOG2N>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float2* work = reinterpret_cast<float2*>(smem_raw);
  float2* tab = work + S::work_len;
  const uint32_t h = blockIdx.x, j = threadIdx.x;
  load_table<LOG2N>(tab, tab_g);
  float2 v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = make_float2(0.f, 0.f);
  if (map.ctas > 0) {
    // the CTAs whose shares meet head h's pairs [h np, (h+1) np), in order
    const int64_t G = map.ctas, T = map.total, np = map.npairs;
    // CTA owning pair i: the last c with start(c) <= i
    const int64_t U = (T + 1) / 2;
    auto owner = [&](int64_t i) {
      return map.even ? (int)((((i / 2) + 1) * G - 1) / U) : (int)(((i + 1) * G - 1) / T);
    };
    const int c0 = owner((int64_t)h * np), c1 = owner(((int64_t)h + 1) * np - 1);
    for (int c = c0; c <= c1; ++c) {
      const int64_t start = map.even ? 2 * ((int64_t)c * U / G) : (int64_t)c * T / G;
      const int seg = (int)h - (int)(start / np);
      const float2* sp = spart + ((size_t)c * map.maxseg + seg) * S::n;
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = cadd(v[r], __ldg(sp + j + r * S::stride));
    }
  } else {
    for (int c = 0; c < chunks; ++c) {
      const float2* sp = spart + ((size_t)h * chunks + c) * S::n;
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = cadd(v[r], __ldg(sp + j + r * S::stride));
    }
  }
  dft_reg<+1, 16>(v);
  bfly_store<16, 1>(work, v, j);
  __syncthreads();
  mid_passes<+1, LOG2N, 16>(work, tab);
  bfly_load<+1, 16, S::n / 16, LOG2N>(work, tab, v, j);
  const float s = scale / (float)S::n;
  const size_t base = (size_t)h * N;
  float* row = reinterpret_cast<float*>(work);
  __syncthreads();
  // time smoothing: the squash mask 1[kbar != 0] applied once per element
  // (row holds the masked dKbar; the tap sum below is reg_grad's, same order)
  const bool tsm = !freq;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const uint32_t t = j + r * S::stride;
    if (t < N) {
      const float g = v[r].x * s;
      row[t] = (tsm && __ldg(kbar + base + t) == 0.f) ? 0.f : g;
      if (dkbar_out) dkbar_out[base + t] = g;
      if (t == 0 && dd_lag0) dD[h] = g;
    }
  }
  __syncthreads();
  if (tsm) {
    const double inv_w = 1.0 / (double)(2 * p + 1);
    for (uint32_t t = j; t < N; t += S::T) {
      const int64_t lo = (int64_t)t >= p ? (int64_t)t - p : 0;
      const int64_t hi = ((int64_t)t + p < (int64_t)N - 1) ? (int64_t)t + p : (int64_t)N - 1;
      double acc = 0.0;
      for (int64_t q = lo; q <= hi; ++q) acc += (double)row[q];
      double g = acc * inv_w;
      if (keep) g = keep[base + t] ? g * keep_scale : 0.0;
      dK[base + t] = (float)g;
    }
  } else {
    for (uint32_t t = j; t < N; t += S::T)
      dK[base + t] = reg_grad(kbar + base, row, keep ? keep + base : nullptr, t, N, p, keep_scale,
                              freq);
  }
  if (j == 0 && !dd_lag0) {
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

template <typename IO>
size_t stage_bytes(uint32_t N, int rows) {
  return (size_t)rows * row_pitch<IO>(N) * sizeof(IO);
}

template <int LOG2N>
size_t base_smem(bool with_n_extra) {
  using S = FftShape<LOG2N>;
  return (S::work_len + (with_n_extra ? S::n : 0) + ((S::tab_len + 1) & ~1u)) * sizeof(float2);
}

constexpr size_t kMaxSmem = 227 * 1024;

bool rows_aligned(const void* a, const void* b, uint32_t N, size_t es) {
  return ((N * es) % 16 == 0) && ((uintptr_t)a % 16 == 0) && (b == nullptr || (uintptr_t)b % 16 == 0);
}

template <int LOG2N>
struct Sp {
  template <typename IO>
  static void fwd(cudaStream_t s, const fb_plan* p, const void* u, void* y, int B, int chunks,
                  int ppc) {
    const size_t sm = base_smem<LOG2N>(true) + stage_bytes<IO>((uint32_t)p->N, 4);
    auto k = sp_fwd_kernel<IO, LOG2N>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const int tma = rows_aligned(u, nullptr, (uint32_t)p->N, sizeof(IO)) ? 1 : 0;
    k<<<dim3((unsigned)p->H, (unsigned)chunks), FftShape<LOG2N>::T, sm, s>>>(
        (const IO*)u, (IO*)y, p->kf, p->d, p->tw2, B, (int)p->H, (uint32_t)p->N,
        p->periodic ? 1 : 0, ppc, tma);
  }
  template <typename IO>
  static void bwd(cudaStream_t s, const fb_plan* p, const void* dy, const void* u, void* du,
                  float2* spart, float* ddpart, int B, int chunks, int ppc) {
    const size_t sm2 = base_smem<LOG2N>(true) + stage_bytes<IO>((uint32_t)p->N, 8);
    const int tma = rows_aligned(dy, u, (uint32_t)p->N, sizeof(IO)) ? 1 : 0;
    const dim3 g((unsigned)p->H, (unsigned)chunks);
    if (sm2 <= kMaxSmem) {
      auto k = sp_bwd_kernel<IO, LOG2N, 2>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
      k<<<g, FftShape<LOG2N>::T, sm2, s>>>((const IO*)dy, (const IO*)u, (IO*)du, p->kf, p->d,
                                           p->tw2, spart, ddpart, B, (int)p->H, (uint32_t)p->N,
                                           p->periodic ? 1 : 0, ppc, tma);
    } else {
      const size_t sm1 = base_smem<LOG2N>(true) + stage_bytes<IO>((uint32_t)p->N, 4);
      auto k = sp_bwd_kernel<IO, LOG2N, 1>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
      k<<<g, FftShape<LOG2N>::T, sm1, s>>>((const IO*)dy, (const IO*)u, (IO*)du, p->kf, p->d,
                                           p->tw2, spart, ddpart, B, (int)p->H, (uint32_t)p->N,
                                           p->periodic ? 1 : 0, ppc, tma);
    }
  }
  static void spectrum(cudaStream_t s, const fb_plan* p, const float* K) {
    const size_t sm = base_smem<LOG2N>(false);
    auto k = sp_spectrum_kernel<LOG2N>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<(unsigned)p->H, FftShape<LOG2N>::T, sm, s>>>(
        K, p->use_keep ? p->keep : nullptr, p->kbar, p->kf,
        p->use_tc ? (__half2*)p->kf_tc : nullptr, p->kf_scale, p->d, p->tw2, (uint32_t)p->N, p->p, p->lambda, p->keep_scale,
        p->smooth_domain == FB_SMOOTH_FREQUENCY, p->tc_ver);
  }
  static void finalize(cudaStream_t s, const fb_plan* p, const float2* spart, const float* ddpart,
                       int chunks, float* dkbar, float* dD, float* dK, int dd_lag0,
                       const SpartMap* map) {
    const size_t sm = base_smem<LOG2N>(false);
    auto k = sp_dk_finalize_kernel<LOG2N>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const float scale = p->periodic ? (float)p->N / (float)p->n : 1.0f;
    k<<<(unsigned)p->H, FftShape<LOG2N>::T, sm, s>>>(
        spart, ddpart, chunks, dkbar, dD, p->kbar, p->use_keep ? p->keep : nullptr, dK, p->tw2,
        (uint32_t)p->N, scale, p->p, p->keep_scale, p->smooth_domain == FB_SMOOTH_FREQUENCY,
        dd_lag0, map ? *map : SpartMap{0, 0, 0, 0, 0});
  }
};

template <class F>
void with_log2n(int64_t n, F&& f) {
  switch (log2i(n)) {
    case 8: f(Sp<8>{}); break;
    case 9: f(Sp<9>{}); break;
    case 10: f(Sp<10>{}); break;
    case 11: f(Sp<11>{}); break;
    case 12: f(Sp<12>{}); break;
    default: f(Sp<13>{}); break;
  }
}

// Split the channel pairs of a head into chunks (CTAs per head): enough CTAs
// for ~1 wave while keeping each CTA's k_f staging amortised.  A CTA is
// n / 16 threads, so for n <= 512 (one warp) aim at ~16 CTAs per SM instead
// (measured: sweep N = 256 0.090 -> 0.064 ms; larger n lose with more chunks).
int chunks_for(const fb_plan* p, int64_t B) {
  const int64_t npairs = (B + 1) / 2;
  const int64_t target = (int64_t)p->num_sms * (p->n <= 512 ? 16 : 1);
  int64_t c = (target + p->H - 1) / p->H;
  c = std::max<int64_t>(1, std::min<int64_t>(c, npairs));
  return (int)c;
}

}  // namespace

int sp_prep(fb_plan* p, const float* K, cudaStream_t s) {
  with_log2n(p->n, [&](auto ks) { ks.spectrum(s, p, K); });
  return cuda_status(cudaGetLastError(), "sp_prep");
}

int sp_finalize(fb_plan* p, const float2* spart, const float* ddpart, int chunks, float* dkbar,
                float* dD, float* dK, int dd_lag0, const SpartMap* map, cudaStream_t s) {
  with_log2n(p->n, [&](auto ks) {
    ks.finalize(s, p, spart, ddpart, chunks, dkbar, dD, dK, dd_lag0, map);
  });
  return cuda_status(cudaGetLastError(), "sp_finalize");
}

int sp_fwd(fb_plan* p, const void* u, void* y, int64_t B, cudaStream_t s) {
  if (p->use_tc) return tc_fwd(p, u, y, B, s);
  if (p->use_sc) {
    prof_mark(p, 0, 0, s);
    const int rc = sc_fwd(p, u, y, B, s);
    prof_mark(p, 0, 1, s);
    return rc;
  }
  const int chunks = chunks_for(p, B);
  const int64_t npairs = (B + 1) / 2;
  const int ppc = (int)((npairs + chunks - 1) / chunks);
  prof_mark(p, 0, 0, s);
  with_log2n(p->n, [&](auto ks) {
    switch (p->dtype) {
      case FB_F32: ks.template fwd<float>(s, p, u, y, (int)B, chunks, ppc); break;
      case FB_BF16: ks.template fwd<__nv_bfloat16>(s, p, u, y, (int)B, chunks, ppc); break;
      default: ks.template fwd<__half>(s, p, u, y, (int)B, chunks, ppc); break;
    }
  });
  prof_mark(p, 0, 1, s);
  return cuda_status(cudaGetLastError(), "sp_fwd");
}

size_t sp_workspace(const fb_plan* p, int64_t B) {
  if (p->use_tc) return tc_workspace(p, B);
  if (p->use_sc)  // spectral partials, then dD partials
    return ((size_t)p->H * sc_chunks(p, B) * (p->n * sizeof(float2) + sizeof(float)) + 255) & ~size_t(255);
  const int c = chunks_for(p, B);
  size_t bytes = (size_t)p->H * c * p->n * sizeof(float2);  // spectral partials
  bytes += (size_t)p->H * c * sizeof(float);                 // dD partials
  bytes = (bytes + 255) & ~size_t(255);
  bytes += (size_t)p->H * p->N * sizeof(float);              // dKbar scratch
  return bytes + 256;
}

int sp_bwd(fb_plan* p, const void* dy, const void* u, void* du, float* dK, float* dKbar, float* dD,
           int64_t B, void* ws, cudaStream_t s) {
  if (p->use_tc) return tc_bwd(p, dy, u, du, dK, dKbar, dD, B, ws, s);
  if (p->use_sc) {
    const int c = sc_chunks(p, B);
    float2* spart = (float2*)ws;
    float* ddpart = (float*)((char*)ws + (size_t)p->H * c * p->n * sizeof(float2));
    prof_mark(p, 1, 0, s);
    int rc = sc_bwd(p, dy, u, du, spart, ddpart, B, s);
    prof_mark(p, 1, 1, s);
    if (!rc) rc = sp_finalize(p, spart, ddpart, c, dKbar, dD, dK, 0, nullptr, s);
    return rc;
  }
  const int chunks = chunks_for(p, B);
  const int64_t npairs = (B + 1) / 2;
  const int ppc = (int)((npairs + chunks - 1) / chunks);
  char* w = (char*)ws;
  float2* spart = (float2*)w;
  size_t off = (size_t)p->H * chunks * p->n * sizeof(float2);
  float* ddpart = (float*)(w + off);
  off += (size_t)p->H * chunks * sizeof(float);
  off = (off + 255) & ~size_t(255);
  with_log2n(p->n, [&](auto ks) {
    prof_mark(p, 1, 0, s);
    switch (p->dtype) {
      case FB_F32: ks.template bwd<float>(s, p, dy, u, du, spart, ddpart, (int)B, chunks, ppc); break;
      case FB_BF16: ks.template bwd<__nv_bfloat16>(s, p, dy, u, du, spart, ddpart, (int)B, chunks, ppc); break;
      default: ks.template bwd<__half>(s, p, dy, u, du, spart, ddpart, (int)B, chunks, ppc); break;
    }
    prof_mark(p, 1, 1, s);
    ks.finalize(s, p, spart, ddpart, chunks, dKbar, dD, dK, 0, nullptr);
  });
  return cuda_status(cudaGetLastError(), "sp_bwd");
}

}  // namespace fb
