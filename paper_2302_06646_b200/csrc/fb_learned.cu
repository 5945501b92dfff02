// FlashButterfly-B200 learned butterfly (K5): the DFT blocks of the plan
// become trainable per-head f x f complex matrices (§3.2.1).
//
// Reference: LearnedButterfly / learned_forward / learned_gradients
// (proj/src/butterfly.cpp:221-307) over the stage walk apply_stages
// (:124-163).  Writing the reference's gather / dense block / scatter +
// twiddle of stage s (factor f, segment L, rest = L/f) in matrix form, each
// length-L segment viewed as an f x rest matrix M[p][q] = cur[p*rest + q]
// is updated in place as
//     M'[a][q] = exp(-2 pi i a q / L) * sum_p W_s[a][p] M[p][q]
// (the gather/scatter permutations cancel), and the final output is
// y[i] = cur[output_map[i]] (:161).  The adjoint (:248-307) is
//     w[a][q]  = conj(tw(a,q)) g[a*rest + q]
//     G_s[a][p] += sum_{seg,q} w[a][q] conj(M_s[p][q])        (block grad)
//     g'[p*rest + q] = sum_a conj(W_s[a][p]) w[a][q]          (input grad)
// starting from g[output_map[i]] = upstream[i].
//
// One CTA per head owns the head's blocks in shared memory; the backward CTA
// walks all B rows of its head in order, so dblocks (summed over b) are
// deterministic without atomics.
#include <algorithm>
#include <type_traits>
#include <cmath>
#include <vector>

#include "fb_common.cuh"
#include "fb_fft.cuh"
#include "fb_internal.h"

namespace fb {

constexpr int kLbThreads = 256;
constexpr int kLbMaxStages = 32;

struct LbStages {
  int nstages;
  int f[kLbMaxStages];
  int L[kLbMaxStages];
  int off[kLbMaxStages];  // complex offset of stage block in the per-head params
};

// stage s in place: dst = T .* (W_s x M) per segment (src -> dst buffers)
__device__ __forceinline__ void lb_stage(const float2* __restrict__ src, float2* __restrict__ dst,
                                         const float2* __restrict__ W, int f, int L, uint32_t n,
                                         const float2* __restrict__ tw) {
  const int rest = L / f;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const uint32_t seg = i / L, loc = i % L, a = loc / rest, q = loc % rest;
    const float2* col = src + seg * L + q;
    const float2* wr = W + a * f;
    float2 acc = make_float2(0.f, 0.f);
    for (int p = 0; p < f; ++p) {
      const float2 w = wr[p], x = col[p * rest];
      acc.x = fmaf(w.x, x.x, fmaf(-w.y, x.y, acc.x));
      acc.y = fmaf(w.x, x.y, fmaf(w.y, x.x, acc.y));
    }
    // exp(-2 pi i a q / L) = tw_n[a q (n / L)]
    dst[i] = cmul(acc, __ldg(tw + (size_t)a * q * (n / L)));
  }
}

template <typename IO>
__global__ void __launch_bounds__(kLbThreads)
    lb_fwd_kernel(const float* __restrict__ blocks, const IO* __restrict__ x, IO* __restrict__ y,
                  const uint32_t* __restrict__ omap, const float2* __restrict__ tw, LbStages st,
                  int B, int H, uint32_t n, int P, int rows_per_cta) {
  extern __shared__ __align__(16) float2 lsm[];
  float2* W = lsm;          // [P]
  float2* b0 = W + P;       // [n]
  float2* b1 = b0 + n;      // [n]
  const int h = blockIdx.x;
  const float2* wg = reinterpret_cast<const float2*>(blocks) + (size_t)h * P;
  for (int i = threadIdx.x; i < P; i += blockDim.x) W[i] = wg[i];
  const int r0 = blockIdx.y * rows_per_cta, r1 = min(B, r0 + rows_per_cta);
  for (int b = r0; b < r1; ++b) {
    const IO* xr = x + ((size_t)b * H + h) * 2 * n;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) b0[i] = ldc<IO>(xr + 2 * i);
    __syncthreads();
    float2 *s = b0, *d = b1;
    for (int k = 0; k < st.nstages; ++k) {
      lb_stage(s, d, W + st.off[k], st.f[k], st.L[k], n, tw);
      __syncthreads();
      float2* t = s;
      s = d;
      d = t;
    }
    IO* yr = y + ((size_t)b * H + h) * 2 * n;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) stc<IO>(yr + 2 * i, s[__ldg(omap + i)]);
  }
}

// CTA (h, split): rows b in [split * rows, ...) of head h, in order; the
// block gradient partial of the split goes to gpart[split][h] and
// lb_reduce_kernel sums the splits in a fixed order (deterministic).
template <typename IO>
__global__ void __launch_bounds__(kLbThreads)
    lb_bwd_kernel(const float* __restrict__ blocks, const IO* __restrict__ x,
                  const IO* __restrict__ g, IO* __restrict__ dx, float2* __restrict__ gpart,
                  const uint32_t* __restrict__ omap, const float2* __restrict__ tw, LbStages st,
                  int B, int H, uint32_t n, int P, int rows) {
  extern __shared__ __align__(16) float2 lsm[];
  float2* W = lsm;                          // [P]
  float2* G = W + P;                        // [P] gradient accumulator
  float2* red = G + P;                      // [kLbThreads] column-split partials
  float2* saved = red + kLbThreads;         // [S][n] stage inputs
  float2* ga = saved + (size_t)st.nstages * n;  // [n]
  float2* gb = ga + n;                      // [n]
  const int h = blockIdx.x;
  const int b_begin = blockIdx.y * rows, b_end = min(B, b_begin + rows);
  const float2* wg = reinterpret_cast<const float2*>(blocks) + (size_t)h * P;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    W[i] = wg[i];
    G[i] = make_float2(0.f, 0.f);
  }
  for (int b = b_begin; b < b_end; ++b) {
    const IO* xr = x + ((size_t)b * H + h) * 2 * n;
    const IO* gr = g + ((size_t)b * H + h) * 2 * n;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) saved[i] = ldc<IO>(xr + 2 * i);
    __syncthreads();
    // forward, keeping each stage's input
    for (int k = 0; k + 1 < st.nstages; ++k) {
      lb_stage(saved + (size_t)k * n, saved + (size_t)(k + 1) * n, W + st.off[k], st.f[k], st.L[k],
               n, tw);
      __syncthreads();
    }
    // adjoint of the output permutation
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) ga[__ldg(omap + i)] = ldc<IO>(gr + 2 * i);
    __syncthreads();
    for (int k = st.nstages - 1; k >= 0; --k) {
      const int f = st.f[k], L = st.L[k], rest = L / f;
      const float2* v = saved + (size_t)k * n;
      const float2* Wk = W + st.off[k];
      // w = conj(tw) * g, in place in ga
      for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t loc = i % L, a = loc / rest, q = loc % rest;
        ga[i] = cmulc(ga[i], __ldg(tw + (size_t)a * q * (n / L)));
      }
      __syncthreads();
      // G[a][p] += sum_{seg, q} w[a][q] conj(v[p][q]): entry e = (a, p) by
      // ns threads, each over every ns-th column, then a fixed-order sum
      {
        const int ff = f * f;
        const int ns = ff >= (int)blockDim.x ? 1 : (int)blockDim.x / ff;
        const uint32_t cols = n / f;  // (segment, q) pairs
        for (int t = threadIdx.x; t < ff * ns; t += blockDim.x) {
          const int e = t % ff, grp = t / ff, a = e / f, p = e % f;
          float2 acc = make_float2(0.f, 0.f);
          for (uint32_t cidx = grp; cidx < cols; cidx += ns) {
            const uint32_t off = (cidx / rest) * L + (cidx % rest);
            const float2 wv = ga[off + a * rest], vv = v[off + p * rest];
            acc.x = fmaf(wv.x, vv.x, fmaf(wv.y, vv.y, acc.x));
            acc.y = fmaf(wv.y, vv.x, fmaf(-wv.x, vv.y, acc.y));
          }
          if (ns == 1) G[st.off[k] + e] = cadd(G[st.off[k] + e], acc);
          else red[t] = acc;
        }
        if (ns > 1) {
          __syncthreads();
          for (int e = threadIdx.x; e < ff; e += blockDim.x) {
            float2 acc = G[st.off[k] + e];
            for (int grp = 0; grp < ns; ++grp) acc = cadd(acc, red[grp * ff + e]);
            G[st.off[k] + e] = acc;
          }
        }
      }
      // g' = W^H w
      for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t seg = i / L, loc = i % L, p = loc / rest, q = loc % rest;
        float2 acc = make_float2(0.f, 0.f);
        for (int a = 0; a < f; ++a) {
          const float2 w = Wk[a * f + p], x2 = ga[seg * L + a * rest + q];
          acc.x = fmaf(w.x, x2.x, fmaf(w.y, x2.y, acc.x));
          acc.y = fmaf(w.x, x2.y, fmaf(-w.y, x2.x, acc.y));
        }
        gb[i] = acc;
      }
      __syncthreads();
      float2* t = ga;
      ga = gb;
      gb = t;
    }
    IO* dr = dx + ((size_t)b * H + h) * 2 * n;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) stc<IO>(dr + 2 * i, ga[i]);
  }
  __syncthreads();
  float2* dg = gpart + ((size_t)blockIdx.y * H + h) * P;
  for (int i = threadIdx.x; i < P; i += blockDim.x) dg[i] = G[i];
}

// ---------------------------------------------------------------- fast path
// Power-of-two factor chains with every factor <= 16 (config 4: n = 1024 =
// 16 x 16 x 4) run through specialised kernels: the stage loops are unrolled
// per factor F (templated), R rows of one head go through each stage
// together, index math is shifts and masks, the twiddle table sits in smem,
// and the backward's block gradients are register tiles (4 x 4 entries per
// thread, column groups reduced by shuffles, warps in a fixed order) so
// neither the stage inputs nor the gradients are read with bank conflicts.
// One stage in the forward direction (stage k of apply_stages,
// butterfly.cpp:136-157, in the matrix form of this file's header):
//   dst[seg L + a rest + q] = w_L^(a q) sum_p W[a][p] src[seg L + p rest + q]
// The adjoint pass writes g' = W^H w and immediately applies the next
// (lower) stage's conj twiddle, so every adjoint stage reads its w ready.
constexpr int kLxThreads = 256;
constexpr int kLxMaxF = 16;

struct LxGeo {
  int nst, lgn;
  int lgf[kLbMaxStages];
  int lgL[kLbMaxStages];
  int off[kLbMaxStages];
};

template <int F>
struct Lg2;
template <> struct Lg2<2> { static constexpr int v = 1; };
template <> struct Lg2<4> { static constexpr int v = 2; };
template <> struct Lg2<8> { static constexpr int v = 3; };
template <> struct Lg2<16> { static constexpr int v = 4; };

// column `col` of R rows under stage geometry (lgL, F): element offset of p = 0
// Stage buffers are padded by one float2 per 32 (element e at px(e)): the
// butterfly's power-of-two strides would otherwise put a warp's accesses in
// a few banks (measured 7x bank conflicts on the config-4 forward).
__host__ __device__ __forceinline__ int px(int e) { return e + (e >> 5); }
// a padded buffer of e elements, rounded to 16 bytes (cp.async destinations)
__host__ __device__ __forceinline__ int pxbuf(int e) { return (px(e) + 2) & ~1; }
__device__ __forceinline__ int lx_base(int col, int lgcpr, int lgrest, int lgL, int lgn) {
  const int r = col >> lgcpr, cc = col & ((1 << lgcpr) - 1);
  return (r << lgn) + ((cc >> lgrest) << lgL) + (cc & ((1 << lgrest) - 1));
}

// 16-byte asynchronous global -> shared copies (LDGSTS): every load of a
// phase is in flight at once instead of one dependent round trip per element
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(static_cast<uint64_t>(__cvta_generic_to_global(gmem)))
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
// bytes (multiple of 16, 16-byte aligned both sides) with the whole CTA
__device__ __forceinline__ void cp_async_bytes(void* dst, const void* src, size_t bytes) {
  for (size_t i = threadIdx.x; i < bytes / 16; i += kLxThreads)
    cp_async16(static_cast<char*>(dst) + 16 * i, static_cast<const char*>(src) + 16 * i);
}

template <int F>
__device__ __forceinline__ void lx_fwd_stage(const float2* __restrict__ src, float2* __restrict__ dst,
                                             const float2* __restrict__ W, int lgL, int lgn, int R,
                                             const float2* __restrict__ tw) {
  constexpr int LGF = Lg2<F>::v;
  const int lgrest = lgL - LGF, lgcpr = lgn - LGF;
  const int C = R << lgcpr;
  // fewer columns than threads: split each column's F outputs over `sp` threads
  const int sp = C >= kLxThreads ? 1 : min(F, kLxThreads / C);
  const int part = threadIdx.x / C, per = F / sp;
  if (part >= sp) return;
  for (int col = threadIdx.x % C; col < C; col += kLxThreads / sp) {
    const int base = lx_base(col, lgcpr, lgrest, lgL, lgn);
    const int ts = (col & ((1 << lgrest) - 1)) << (lgn - lgL);  // q n / L
    float2 x[F];
#pragma unroll
    for (int p = 0; p < F; ++p) x[p] = src[px(base + (p << lgrest))];
    // one output row at a time: the W row is a broadcast load (all lanes read
    // the same entry), so a full unroll would only hoist F^2 registers
#pragma unroll 1
    for (int a = part * per; a < (part + 1) * per; ++a) {
      float ar = 0.f, ai = 0.f;
      const float4* wr = reinterpret_cast<const float4*>(W + a * F);  // two entries per load
#pragma unroll
      for (int p = 0; p < F; p += 2) {
        const float4 w2 = wr[p >> 1];
        ar = fmaf(w2.x, x[p].x, fmaf(-w2.y, x[p].y, ar));
        ai = fmaf(w2.x, x[p].y, fmaf(w2.y, x[p].x, ai));
        ar = fmaf(w2.z, x[p + 1].x, fmaf(-w2.w, x[p + 1].y, ar));
        ai = fmaf(w2.z, x[p + 1].y, fmaf(w2.w, x[p + 1].x, ai));
      }
      dst[px(base + (a << lgrest))] = cmul(make_float2(ar, ai), tw[px(a * ts)]);
    }
  }
}

// g'[p] = sum_a conj(W[a][p]) w[a] (WT = the stage block transposed); then
// (plgL >= 0) times conj of the lower
// stage's twiddle at that element, i.e. the lower stage's w
template <int F>
__device__ __forceinline__ void lx_adj_stage(const float2* __restrict__ w, float2* __restrict__ gout,
                                             const float2* __restrict__ WT, int lgL, int lgn, int R,
                                             const float2* __restrict__ tw, int plgL, int plgf) {
  constexpr int LGF = Lg2<F>::v;
  const int lgrest = lgL - LGF, lgcpr = lgn - LGF;
  const int plgrest = plgL - plgf;
  const int C = R << lgcpr;
  const int sp = C >= kLxThreads ? 1 : min(F, kLxThreads / C);
  const int part = threadIdx.x / C, per = F / sp;
  if (part >= sp) return;
  for (int col = threadIdx.x % C; col < C; col += kLxThreads / sp) {
    const int base = lx_base(col, lgcpr, lgrest, lgL, lgn);
    float2 v[F];
#pragma unroll
    for (int a = 0; a < F; ++a) v[a] = w[px(base + (a << lgrest))];
#pragma unroll 1
    for (int p = part * per; p < (part + 1) * per; ++p) {
      float ar = 0.f, ai = 0.f;
      const float4* wr = reinterpret_cast<const float4*>(WT + p * F);  // W^T row p
#pragma unroll
      for (int a = 0; a < F; a += 2) {
        const float4 m2 = wr[a >> 1];  // conj(m) v
        ar = fmaf(m2.x, v[a].x, fmaf(m2.y, v[a].y, ar));
        ai = fmaf(m2.x, v[a].y, fmaf(-m2.y, v[a].x, ai));
        ar = fmaf(m2.z, v[a + 1].x, fmaf(m2.w, v[a + 1].y, ar));
        ai = fmaf(m2.z, v[a + 1].y, fmaf(-m2.w, v[a + 1].x, ai));
      }
      const int idx = base + (p << lgrest);
      float2 o = make_float2(ar, ai);
      if (plgL >= 0) {
        const int loc = idx & ((1 << plgL) - 1);
        const int pa = loc >> plgrest, pq = loc & ((1 << plgrest) - 1);
        o = cmulc(o, tw[px((pa * pq) << (lgn - plgL))]);
      }
      gout[px(idx)] = o;
    }
  }
}

// G[a][p] += sum_cols w[a] conj(v[p]) over the R rows' columns
template <int F>
__device__ __forceinline__ void lx_grad(const float2* __restrict__ w, const float2* __restrict__ v,
                                        float2* __restrict__ G, float2* __restrict__ red, int lgL,
                                        int lgn, int R) {
  constexpr int LGF = Lg2<F>::v;
  constexpr int TS = F < 4 ? F : 4;
  constexpr int NTS = F / TS, NT = NTS * NTS, CG = kLxThreads / NT;
  const int lgrest = lgL - LGF, lgcpr = lgn - LGF;
  const int t = threadIdx.x, tile = t % NT, cg = t / NT;
  const int a0 = (tile / NTS) * TS, p0 = (tile % NTS) * TS;
  float2 acc[TS][TS];
#pragma unroll
  for (int i = 0; i < TS; ++i)
#pragma unroll
    for (int j = 0; j < TS; ++j) acc[i][j] = make_float2(0.f, 0.f);
  const int C = R << lgcpr;
  for (int col = cg; col < C; col += CG) {
    const int base = lx_base(col, lgcpr, lgrest, lgL, lgn);
    float2 wv[TS], vv[TS];
#pragma unroll
    for (int i = 0; i < TS; ++i) {
      wv[i] = w[px(base + ((a0 + i) << lgrest))];
      vv[i] = v[px(base + ((p0 + i) << lgrest))];
    }
#pragma unroll
    for (int i = 0; i < TS; ++i)
#pragma unroll
      for (int j = 0; j < TS; ++j) {
        acc[i][j].x = fmaf(wv[i].x, vv[j].x, fmaf(wv[i].y, vv[j].y, acc[i][j].x));
        acc[i][j].y = fmaf(wv[i].y, vv[j].x, fmaf(-wv[i].x, vv[j].y, acc[i][j].y));
      }
  }
  // lanes l and l ^ o (o a multiple of NT) hold the same tile
#pragma unroll
  for (int o = NT; o < 32; o <<= 1)
#pragma unroll
    for (int i = 0; i < TS; ++i)
#pragma unroll
      for (int j = 0; j < TS; ++j) {
        acc[i][j].x += __shfl_xor_sync(0xffffffffu, acc[i][j].x, o);
        acc[i][j].y += __shfl_xor_sync(0xffffffffu, acc[i][j].y, o);
      }
  const int warp = t >> 5, lane = t & 31;
  if (lane < NT) {
#pragma unroll
    for (int i = 0; i < TS; ++i)
#pragma unroll
      for (int j = 0; j < TS; ++j) red[warp * F * F + (a0 + i) * F + (p0 + j)] = acc[i][j];
  }
  __syncthreads();
  for (int e = t; e < F * F; e += kLxThreads) {
    float2 s = G[e];
    for (int wq = 0; wq < kLxThreads / 32; ++wq) s = cadd(s, red[wq * F * F + e]);
    G[e] = s;
  }
  __syncthreads();
}

// ---------------------------------------------------------------- F = 16 stages on mma.sync
// For the 16-bit modes the F = 16 stages (all but the last of config 4's
// [16, 16, 4]) run on the tensor cores as real-stacked GEMMs with bf16
// operands and fp32 accumulation: a column's update y = W x (16 x 16
// complex) is [yr; yi] = [[Wr, -Wi]; [Wi, Wr]] [xr; xi], i.e. a 32 x 32 A
// operand (kept in registers for the stage) against 8-column B tiles taken
// from smem — four m16n8k16 MMAs per 8 columns instead of 1024 FFMAs per
// column.  The block gradient G += sum_cols w conj(v) is the 32 x 32 product
// [wr; wi] [vr; vi]^T over the columns (Gr = P00 + P11, Gi = P10 - P01),
// reduced over warps in a fixed order.  (mma.sync rather than tcgen05: the
// operands are a few KB per head and scattered by the butterfly's strides;
// the instruction count, not tensor throughput, is what bounds this path.)
__device__ __forceinline__ uint32_t pk_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// A fragments of [[Mr, -Mi]; [Mi, Mr]] with M(o, i) = (CONJT ? conj(W[i][o]) : W[o][i])
template <bool CONJT>
__device__ __forceinline__ void lx_afrag(uint32_t (&A)[2][2][4], const float2* __restrict__ W) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
  auto m = [&](int o, int i) {
    const float2 w = CONJT ? W[i * 16 + o] : W[o * 16 + i];
    return CONJT ? make_float2(w.x, -w.y) : w;
  };
  auto val = [&](int row, int col) {
    const float2 w = m(row & 15, col & 15);
    const bool rr = row < 16, rc = col < 16;
    return rr ? (rc ? w.x : -w.y) : (rc ? w.y : w.x);
  };
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int kt = 0; kt < 2; ++kt)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int row = 16 * mt + g + (r & 1) * 8, col = 16 * kt + 2 * tig + (r >> 1) * 8;
        A[mt][kt][r] = pk_bf16(val(row, col), val(row, col + 1));
      }
}

// dst[col][o] = post(o, col) * sum_i M(o, i) src[col][i] over all columns, F = 16.
// ADJ = false: M = W and post = the stage twiddle (forward);
// ADJ = true:  M = W^H and post = conj of the lower stage's twiddle (plgL >= 0).
template <bool ADJ>
__device__ __forceinline__ void lx_stage_mma16(const float2* __restrict__ src, float2* __restrict__ dst,
                                               const float2* __restrict__ W, int lgL, int lgn, int R,
                                               const float2* __restrict__ tw, int plgL, int plgf) {
  const int lgrest = lgL - 4, lgcpr = lgn - 4;
  const int C = R << lgcpr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
  uint32_t A[2][2][4];
  lx_afrag<ADJ>(A, W);
  const int plgrest = plgL - plgf;
  for (int nt = warp; nt * 8 < C; nt += kLxThreads / 32) {
    const int base = lx_base(nt * 8 + g, lgcpr, lgrest, lgL, lgn);
    const float2 x0 = src[px(base + ((2 * tig) << lgrest))], x1 = src[px(base + ((2 * tig + 1) << lgrest))];
    const float2 x2 = src[px(base + ((2 * tig + 8) << lgrest))], x3 = src[px(base + ((2 * tig + 9) << lgrest))];
    const uint32_t br0 = pk_bf16(x0.x, x1.x), br1 = pk_bf16(x2.x, x3.x);
    const uint32_t bi0 = pk_bf16(x0.y, x1.y), bi1 = pk_bf16(x2.y, x3.y);
    float d[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      mma_bf16_16816(d[mt], A[mt][0], br0, br1);
      mma_bf16_16816(d[mt], A[mt][1], bi0, bi1);
    }
    // all four twiddles loaded before any store (smem loads and stores
    // would otherwise serialise through possible aliasing)
    int idx[4];
    float2 t[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int o = g + (e >> 1) * 8, cn = nt * 8 + 2 * tig + (e & 1);
      idx[e] = lx_base(cn, lgcpr, lgrest, lgL, lgn) + (o << lgrest);
      if (!ADJ) {
        const int q = cn & ((1 << lgrest) - 1);
        t[e] = tw[px(o * (q << (lgn - lgL)))];
      } else if (plgL >= 0) {
        const int loc = idx[e] & ((1 << plgL) - 1);
        const int pa = loc >> plgrest, pq = loc & ((1 << plgrest) - 1);
        t[e] = tw[px((pa * pq) << (lgn - plgL))];
      } else {
        t[e] = make_float2(1.f, 0.f);
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 y = make_float2(d[0][e], d[1][e]);
      dst[px(idx[e])] = ADJ ? cmulc(y, t[e]) : cmul(y, t[e]);
    }
  }
}

// G[a][p] += sum_cols w[a] conj(v[p]), F = 16; red: 8 x 256 float2 scratch
__device__ __forceinline__ void lx_grad_mma16(const float2* __restrict__ w, const float2* __restrict__ v,
                                              float2* __restrict__ G, float2* __restrict__ red,
                                              int lgL, int lgn, int R) {
  const int lgrest = lgL - 4, lgcpr = lgn - 4;
  const int C = R << lgcpr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
  float d[2][4][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) d[mt][nt][e] = 0.f;
  // K chunks of 16 columns; thread's columns k = 2 tig, +1, +8, +9 of the chunk
  for (int kc = warp; kc * 16 < C; kc += kLxThreads / 32) {
    int cb[4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
      cb[r] = lx_base(kc * 16 + 2 * tig + (r & 1) + (r >> 1) * 8, lgcpr, lgrest, lgL, lgn);
    // A = [wr; wi] rows a = g, g + 8; B = [vr; vi]^T columns p = g, g + 8
    float2 wv[2][4], vv[2][4];
#pragma unroll
    for (int h8 = 0; h8 < 2; ++h8)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        wv[h8][r] = w[px(cb[r] + ((g + 8 * h8) << lgrest))];
        vv[h8][r] = v[px(cb[r] + ((g + 8 * h8) << lgrest))];
      }
    uint32_t a[2][4];  // [re/im][reg]: reg = (row g / g+8) x (k lo / hi)
#pragma unroll
    for (int part = 0; part < 2; ++part)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int h8 = r & 1, kk = (r >> 1) * 2;  // k pair {kk, kk+1} of cb[]
        const float2 p0 = wv[h8][kk], p1 = wv[h8][kk + 1];
        a[part][r] = part ? pk_bf16(p0.y, p1.y) : pk_bf16(p0.x, p1.x);
      }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int part = nt >> 1, h8 = nt & 1;  // columns p = 8 h8 + g of vr (part 0) / vi (1)
      const float2 q0 = vv[h8][0], q1 = vv[h8][1], q2 = vv[h8][2], q3 = vv[h8][3];
      const uint32_t b0 = part ? pk_bf16(q0.y, q1.y) : pk_bf16(q0.x, q1.x);
      const uint32_t b1 = part ? pk_bf16(q2.y, q3.y) : pk_bf16(q2.x, q3.x);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) mma_bf16_16816(d[mt][nt], a[mt], b0, b1);
    }
  }
  // this warp's partial: rows a, columns p of each block
#pragma unroll
  for (int h8 = 0; h8 < 2; ++h8)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int aa = g + (e >> 1) * 8, pp = 8 * h8 + 2 * tig + (e & 1);
      const float gr = d[0][h8][e] + d[1][2 + h8][e];   // wr vr + wi vi
      const float gi = d[1][h8][e] - d[0][2 + h8][e];   // wi vr - wr vi
      red[warp * 256 + aa * 16 + pp] = make_float2(gr, gi);
    }
  __syncthreads();
  for (int e = threadIdx.x; e < 256; e += kLxThreads) {
    float2 s = G[e];
    for (int wq = 0; wq < kLxThreads / 32; ++wq) s = cadd(s, red[wq * 256 + e]);
    G[e] = s;
  }
  __syncthreads();
}

template <typename IO>
constexpr bool kTc = !std::is_same<IO, float>::value;  // 16-bit modes: F = 16 stages on mma.sync

#define LX_DISPATCH(lgf, CALL)        \
  switch (lgf) {                      \
    case 1: { constexpr int F = 2; CALL; } break;  \
    case 2: { constexpr int F = 4; CALL; } break;  \
    case 3: { constexpr int F = 8; CALL; } break;  \
    default: { constexpr int F = 16; CALL; } break; \
  }

template <typename IO>
__global__ void __launch_bounds__(kLxThreads)
    lx_fwd_kernel(const float* __restrict__ blocks, const IO* __restrict__ x, IO* __restrict__ y,
                  const uint32_t* __restrict__ omap, const float2* __restrict__ tw_g, LxGeo geo,
                  int B, int H, int P, int R) {
  extern __shared__ __align__(16) float2 lsm[];
  const int n = 1 << geo.lgn;
  float2* W = lsm;
  float2* tw = W + P;
  float2* bufA = tw + pxbuf(n);
  float2* bufB = bufA + pxbuf(R * n);
  const int h = blockIdx.x;
  const float2* wg = reinterpret_cast<const float2*>(blocks) + (size_t)h * P;
  const int b0 = blockIdx.y * R, rows = min(R, B - b0);
  // blocks, twiddles and the raw rows (staged in bufB) all in flight at once
  IO* raw = reinterpret_cast<IO*>(bufB);
  cp_async_bytes(W, wg, (size_t)P * sizeof(float2));
  for (int i = threadIdx.x; i < n; i += kLxThreads) tw[px(i)] = __ldg(tw_g + i);  // padded twiddle table
  for (int r = 0; r < rows; ++r)
    cp_async_bytes(raw + (size_t)r * 2 * n, x + ((size_t)(b0 + r) * H + h) * 2 * n,
                   2 * (size_t)n * sizeof(IO));
  cp_async_wait_all();
  __syncthreads();
  for (int i = threadIdx.x; i < R * n; i += kLxThreads) {
    const int r = i >> geo.lgn;
    bufA[px(i)] = r < rows ? ldc_any<IO>(raw + 2 * (size_t)i) : make_float2(0.f, 0.f);
  }
  __syncthreads();
  float2 *s = bufA, *d = bufB;
  for (int k = 0; k < geo.nst; ++k) {
    if (kTc<IO> && geo.lgf[k] == 4)
      lx_stage_mma16<false>(s, d, W + geo.off[k], geo.lgL[k], geo.lgn, R, tw, -1, 0);
    else
      LX_DISPATCH(geo.lgf[k], (lx_fwd_stage<F>(s, d, W + geo.off[k], geo.lgL[k], geo.lgn, R, tw)));
    __syncthreads();
    float2* tmp = s;
    s = d;
    d = tmp;
  }
  for (int i = threadIdx.x; i < rows * n; i += kLxThreads) {
    const int r = i >> geo.lgn, e = i & (n - 1);
    stc<IO>(y + ((size_t)(b0 + r) * H + h) * 2 * n + 2 * e, s[px((r << geo.lgn) + (int)__ldg(omap + e))]);
  }
}

// CTA (h, split): rows [split * rps, +rps) of head h, R at a time, in order;
// the split's block-gradient partial goes to gpart[split][h] (lb_reduce_kernel
// sums the splits in a fixed order).
template <typename IO>
__global__ void __launch_bounds__(kLxThreads)
    lx_bwd_kernel(const float* __restrict__ blocks, const IO* __restrict__ x,
                  const IO* __restrict__ g, IO* __restrict__ dx, float2* __restrict__ gpart,
                  const uint32_t* __restrict__ omap, const float2* __restrict__ tw_g, LxGeo geo,
                  int B, int H, int P, int R, int rps) {
  extern __shared__ __align__(16) float2 lsm[];
  const int n = 1 << geo.lgn, S = geo.nst;
  float2* W = lsm;
  float2* WT = W + P;  // per stage block transposed (the adjoint's rows)
  float2* G = WT + P;
  float2* tw = G + P;
  const int RNP = pxbuf(R * n);  // one padded stage buffer
  float2* v = tw + pxbuf(n);  // [S][RNP] stage inputs
  float2* ga = v + (size_t)S * RNP;
  float2* gb = ga + RNP;
  const int h = blockIdx.x;
  const float2* wg = reinterpret_cast<const float2*>(blocks) + (size_t)h * P;
  cp_async_bytes(W, wg, (size_t)P * sizeof(float2));
  for (int i = threadIdx.x; i < n; i += kLxThreads) tw[px(i)] = __ldg(tw_g + i);  // padded twiddle table
  cp_async_wait_all();
  __syncthreads();
  for (int i = threadIdx.x; i < P; i += kLxThreads) G[i] = make_float2(0.f, 0.f);
  for (int k = 0; k < S; ++k) {
    const int f = 1 << geo.lgf[k], o = geo.off[k];
    for (int i = threadIdx.x; i < f * f; i += kLxThreads) WT[o + (i % f) * f + i / f] = W[o + i];
  }
  const int lgLt = geo.lgL[S - 1], lgft = geo.lgf[S - 1];
  const int b_end = min(B, (blockIdx.y + 1) * rps);
  for (int b0 = blockIdx.y * rps; b0 < b_end; b0 += R) {
    const int rows = min(R, b_end - b0);
    __syncthreads();
    // raw rows staged in gb (free until the first adjoint pass), all loads of
    // a phase in flight at once: x -> v[0], then g -> ga (permuted + twiddled)
    IO* raw = reinterpret_cast<IO*>(gb);
    for (int phase = 0; phase < 2; ++phase) {
      const IO* src = phase ? g : x;
      for (int r = 0; r < rows; ++r)
        cp_async_bytes(raw + (size_t)r * 2 * n, src + ((size_t)(b0 + r) * H + h) * 2 * n,
                       2 * (size_t)n * sizeof(IO));
      cp_async_wait_all();
      __syncthreads();
      for (int i = threadIdx.x; i < R * n; i += kLxThreads) {
        const int r = i >> geo.lgn, e = i & (n - 1);
        const float2 val = r < rows ? ldc_any<IO>(raw + 2 * (size_t)i) : make_float2(0.f, 0.f);
        if (phase == 0) {
          v[px(i)] = val;
        } else {
          // adjoint of the output permutation, then the top stage's conj twiddle
          const int idx = __ldg(omap + e);
          const int loc = idx & ((1 << lgLt) - 1), lgr = lgLt - lgft;
          const int pa = loc >> lgr, pq = loc & ((1 << lgr) - 1);
          ga[px((r << geo.lgn) + idx)] = cmulc(val, tw[px((pa * pq) << (geo.lgn - lgLt))]);
        }
      }
      __syncthreads();
    }
    for (int k = 0; k + 1 < S; ++k) {
      if (kTc<IO> && geo.lgf[k] == 4)
        lx_stage_mma16<false>(v + (size_t)k * RNP, v + (size_t)(k + 1) * RNP, W + geo.off[k],
                              geo.lgL[k], geo.lgn, R, tw, -1, 0);
      else
      LX_DISPATCH(geo.lgf[k], (lx_fwd_stage<F>(v + (size_t)k * RNP, v + (size_t)(k + 1) * RNP,
                                               W + geo.off[k], geo.lgL[k], geo.lgn, R, tw)));
      __syncthreads();
    }
    for (int k = S - 1; k >= 0; --k) {
      // gb is free until the adjoint pass: it holds the gradient pass's
      // per-warp partials (R n >= 8 f^2 is a condition of the fast path)
      if (kTc<IO> && geo.lgf[k] == 4)
        lx_grad_mma16(ga, v + (size_t)k * RNP, G + geo.off[k], gb, geo.lgL[k], geo.lgn, R);
      else
      LX_DISPATCH(geo.lgf[k], (lx_grad<F>(ga, v + (size_t)k * RNP, G + geo.off[k], gb, geo.lgL[k],
                                          geo.lgn, R)));
      const int plgL = k > 0 ? geo.lgL[k - 1] : -1, plgf = k > 0 ? geo.lgf[k - 1] : 0;
      if (kTc<IO> && geo.lgf[k] == 4)
        lx_stage_mma16<true>(ga, gb, W + geo.off[k], geo.lgL[k], geo.lgn, R, tw, plgL, plgf);
      else
      LX_DISPATCH(geo.lgf[k], (lx_adj_stage<F>(ga, gb, WT + geo.off[k], geo.lgL[k], geo.lgn, R, tw,
                                               plgL, plgf)));
      __syncthreads();
      float2* tmp = ga;
      ga = gb;
      gb = tmp;
    }
    for (int i = threadIdx.x; i < rows * n; i += kLxThreads) {
      const int r = i >> geo.lgn, e = i & (n - 1);
      stc<IO>(dx + ((size_t)(b0 + r) * H + h) * 2 * n + 2 * e, ga[px(i)]);
    }
  }
  __syncthreads();
  float2* dg = gpart + ((size_t)blockIdx.y * H + h) * P;
  for (int i = threadIdx.x; i < P; i += kLxThreads) dg[i] = G[i];
}

// dblocks[i] = sum over the splits in order; two complex entries per thread
// (16-byte accesses when HP is even), the splits' loads in flight together
__global__ void lb_reduce_kernel(const float2* __restrict__ gpart, float2* __restrict__ dblocks,
                                 int splits, size_t HP) {
  const size_t i = 2 * ((size_t)blockIdx.x * blockDim.x + threadIdx.x);
  if (i >= HP) return;
  if ((HP & 1) == 0) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int sp = 0; sp < splits; ++sp) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(gpart + (size_t)sp * HP + i));
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    *reinterpret_cast<float4*>(dblocks + i) = acc;
    return;
  }
  for (size_t e = i; e < i + 2 && e < HP; ++e) {
    float2 acc = make_float2(0.f, 0.f);
    for (int sp = 0; sp < splits; ++sp) acc = cadd(acc, __ldg(gpart + (size_t)sp * HP + e));
    dblocks[e] = acc;
  }
}

struct LbDevice {
  uint32_t* omap = nullptr;
  float2* tw = nullptr;
  LbStages st{};
  bool fast = false;  // power-of-two factors <= 16: the lx_* kernels
  LxGeo geo{};
  bool tc = false;    // 16-bit modes, [16] * stc + [2^lgfl]: the tcgen05 lt_* kernels
  int stc = 0, lgfl = 0;
};

// rows per pass for the fast kernels: the largest R in {4, 2, 1} whose smem
// fits `budget` bytes
inline int lx_rows(size_t fixed, size_t per_row, size_t budget, int64_t min_elems = 0,
                   int64_t n = 1) {
  for (int R = 8; R >= 1; R >>= 1)
    if (fixed + per_row * R <= budget && R * n >= min_elems) return R;
  return 0;
}
inline int64_t lx_maxf(const fb_learned_plan* p) {
  int64_t m = 0;
  for (int i = 0; i < p->nstages; ++i) m = std::max(m, p->factors[i]);
  return m;
}
// (stage buffers padded to pxbuf(R n) float2: n + n / 32 per row plus up to
// two float2 per buffer, the latter counted in the fixed part)
inline size_t lx_fwd_fixed(const fb_learned_plan* p) {
  return (p->param_count + p->n + p->n / 32 + 6) * sizeof(float2);
}
inline size_t lx_fwd_per_row(const fb_learned_plan* p) { return 2 * (size_t)(p->n + p->n / 32) * sizeof(float2); }
inline size_t lx_bwd_fixed(const fb_learned_plan* p) {
  return (3 * p->param_count + p->n + p->n / 32 + 2 + 2 * (p->nstages + 2)) * sizeof(float2);
}
inline size_t lx_bwd_per_row(const fb_learned_plan* p) {
  return (size_t)(p->nstages + 2) * (p->n + p->n / 32) * sizeof(float2);
}

}  // namespace fb

// The C-ABI plan carries the device tables through an opaque extension.
struct fb_learned_ext {
  fb::LbDevice dev;
};

namespace {

using namespace fb;

// Greedy factor chain of build_plan (butterfly.cpp:83-100).
int greedy_factors(int64_t n, int64_t r, std::vector<int64_t>& out) {
  int64_t seg = n;
  while (seg > 1) {
    int64_t f = 0;
    if (seg <= r) {
      f = seg;
    } else {
      for (int64_t d = std::min(seg, r); d >= 2; --d)
        if (seg % d == 0) {
          f = d;
          break;
        }
    }
    if (f == 0) return FB_ERR_PLAN;
    out.push_back(f);
    seg /= f;
  }
  return FB_OK;
}

// Composed output map (butterfly.cpp:103-116).
std::vector<uint32_t> output_map(int64_t n, const std::vector<int64_t>& f) {
  std::vector<uint32_t> m((size_t)n);
  for (int64_t i = 0; i < n; ++i) m[(size_t)i] = (uint32_t)i;
  int64_t L = n;
  for (size_t d = 0; d + 1 < f.size(); ++d) {
    const int64_t rest = L / f[d];
    for (int64_t i = 0; i < n; ++i) {
      const int64_t off = (m[(size_t)i] / L) * L, local = m[(size_t)i] % L;
      const int64_t j2 = local / f[d], j1 = local % f[d];
      m[(size_t)i] = (uint32_t)(off + j1 * rest + j2);
    }
    L = rest;
  }
  return m;
}

fb_learned_ext* ext_of(const fb_learned_plan* p) {
  return static_cast<fb_learned_ext*>(p->ext);
}

}  // namespace

extern "C" {

int fb_learned_plan_create(fb_learned_plan** out, int64_t n, int64_t r, int64_t H, int dtype,
                           int device) {
  if (!out) {
    set_error("fb_learned_plan_create: null output");
    return FB_ERR_ARG;
  }
  *out = nullptr;
  if (n < 1 || H < 1) {
    set_error("learned: n and H must be >= 1");
    return FB_ERR_DIM;
  }
  if (r < 2) {
    set_error("build_plan: block size r must be >= 2");
    return FB_ERR_PLAN;
  }
  if (dtype < FB_F32 || dtype > FB_F16) {
    set_error("learned: bad dtype");
    return FB_ERR_ARG;
  }
  std::vector<int64_t> f;
  if (greedy_factors(n, r, f) != FB_OK) {
    set_error("build_plan: remainder has no factor <= r; pad the input to a power of two");
    return FB_ERR_PLAN;
  }
  if ((int)f.size() > kLbMaxStages - 1) {
    set_error("learned: too many stages");
    return FB_ERR_PLAN;
  }
  DevGuard dg_(device);
  int rc = cuda_status(dg_.err, "cudaSetDevice");
  if (rc) return rc;
  auto* p = new fb_learned_plan();
  p->n = n;
  p->r = r;
  p->H = H;
  p->dtype = dtype;
  p->device = device;
  p->nstages = (int)f.size();
  auto* ext = new fb_learned_ext();
  LbStages& st = ext->dev.st;
  st.nstages = (int)f.size();
  int64_t L = n, off = 0;
  for (size_t i = 0; i < f.size(); ++i) {
    p->factors[i] = f[i];
    st.f[i] = (int)f[i];
    st.L[i] = (int)L;
    st.off[i] = (int)off;
    off += f[i] * f[i];
    L /= f[i];
  }
  p->param_count = off;
  {
    bool fast = (n & (n - 1)) == 0;
    for (int64_t fi : f) fast = fast && fi <= kLxMaxF && (fi & (fi - 1)) == 0 && fi >= 2;
    LxGeo& gg = ext->dev.geo;
    gg.nst = (int)f.size();
    int lg = 0;
    while ((int64_t(1) << lg) < n) ++lg;
    gg.lgn = lg;
    for (size_t i = 0; i < f.size(); ++i) {
      int lf = 0;
      while ((int64_t(1) << lf) < f[i]) ++lf;
      int ll = 0;
      while ((int64_t(1) << ll) < st.L[i]) ++ll;
      gg.lgf[i] = lf;
      gg.lgL[i] = ll;
      gg.off[i] = st.off[i];
    }
    ext->dev.fast = fast && n >= 2;
    ext->dev.tc = lt_config(n, f.data(), (int)f.size(), dtype, &ext->dev.stc, &ext->dev.lgfl);
  }
  std::vector<uint32_t> om = output_map(n, f);
  std::vector<float2> tw((size_t)n);
  for (int64_t t = 0; t < n; ++t) {
    const double a = -2.0 * M_PI * (double)t / (double)n;
    tw[(size_t)t] = make_float2((float)std::cos(a), (float)std::sin(a));
  }
  rc = cuda_status(cudaMalloc(&ext->dev.omap, sizeof(uint32_t) * n), "cudaMalloc(omap)");
  if (!rc) rc = cuda_status(cudaMalloc(&ext->dev.tw, sizeof(float2) * n), "cudaMalloc(tw)");
  if (!rc)
    rc = cuda_status(cudaMemcpy(ext->dev.omap, om.data(), sizeof(uint32_t) * n, cudaMemcpyHostToDevice),
                     "copy omap");
  if (!rc)
    rc = cuda_status(cudaMemcpy(ext->dev.tw, tw.data(), sizeof(float2) * n, cudaMemcpyHostToDevice),
                     "copy tw");
  p->ext = ext;
  if (rc) {
    fb_learned_plan_destroy(p);
    return rc;
  }
  *out = p;
  return FB_OK;
}

int fb_learned_plan_destroy(fb_learned_plan* p) {
  if (!p) return FB_OK;
  fb_learned_ext* ext = ext_of(p);
  if (ext) {
    cudaFree(ext->dev.omap);
    cudaFree(ext->dev.tw);
    delete ext;
  }
  delete p;
  return FB_OK;
}

int fb_learned_plan_factors(const fb_learned_plan* p, int64_t* factors, int64_t* count,
                            int64_t* param_count) {
  if (!p) {
    set_error("fb_learned_plan_factors: null plan");
    return FB_ERR_ARG;
  }
  if (count) *count = p->nstages;
  if (param_count) *param_count = p->param_count;
  if (factors)
    for (int i = 0; i < p->nstages; ++i) factors[i] = p->factors[i];
  return FB_OK;
}

int fb_learned_plan_engine(const fb_learned_plan* p, int* engine) {
  if (!p || !engine) {
    set_error("fb_learned_plan_engine: null argument");
    return FB_ERR_ARG;
  }
  *engine = ext_of(p)->dev.tc ? 2 : ext_of(p)->dev.fast ? 1 : 0;
  return FB_OK;
}

static int lx_bwd_R(const fb_learned_plan* p);
static bool lx_fast_bwd(const fb_learned_plan* p) {
  return ext_of(p)->dev.fast && lx_bwd_R(p) > 0;
}
static int lx_bwd_R(const fb_learned_plan* p) {
  // two CTAs per SM when two rows fit in half the smem, else as many rows as fit
  const int64_t red = (kLxThreads / 32) * lx_maxf(p) * lx_maxf(p);  // gradient partials in gb
  const int R2 = lx_rows(lx_bwd_fixed(p), lx_bwd_per_row(p), 113 * 1024, red, p->n);
  return R2 >= 2 ? R2 : lx_rows(lx_bwd_fixed(p), lx_bwd_per_row(p), 227 * 1024, red, p->n);
}

// Row splits per head for the backward: enough CTAs to fill the SMs (a few
// waves), each split a whole number of the fast kernel's R-row passes.
static int lb_splits(const fb_learned_plan* p, int64_t B) {
  if (ext_of(p)->dev.tc) return (int)((B + lt_rows(p->n) - 1) / lt_rows(p->n));
  int dev_sms = 148;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, p->device);
  if (lx_fast_bwd(p)) {
    const int64_t R = lx_bwd_R(p), passes = (B + R - 1) / R;
    int64_t s = (16 * dev_sms + p->H - 1) / p->H;  // many small CTAs: loads overlap compute
    return (int)std::max<int64_t>(1, std::min<int64_t>(s, passes));
  }
  int64_t s = (2 * dev_sms + p->H - 1) / p->H;
  return (int)std::max<int64_t>(1, std::min<int64_t>(s, B));
}

size_t fb_learned_workspace_size(const fb_learned_plan* p, int64_t B) {
  if (!p || B < 1) return 0;
  return (size_t)lb_splits(p, B) * p->H * p->param_count * sizeof(float2);
}

int fb_learned_fwd(fb_learned_plan* p, const float* blocks, const void* x, void* y, int64_t B,
                   void*, void* stream) {
  if (!p || !blocks || !x || !y) {
    set_error("fb_learned_fwd: null argument");
    return FB_ERR_ARG;
  }
  if (B < 1) {
    set_error("learned_forward: batch must be >= 1");
    return FB_ERR_DIM;
  }
  DevGuard dg_(p->device);
  int rc = cuda_status(dg_.err, "cudaSetDevice");
  if (rc) return rc;
  fb_learned_ext* ext = ext_of(p);
  cudaStream_t s = (cudaStream_t)stream;
  if (ext->dev.tc)
    return cuda_status(lt_fwd(ext->dev.stc, ext->dev.lgfl, p->dtype, blocks, x, y, ext->dev.omap,
                              ext->dev.tw, (int)B, (int)p->H, (int)p->param_count, s),
                       "fb_learned_fwd (tcgen05)");
  if (ext->dev.fast) {
    // small CTAs (four per SM): the stage chain is latency-bound, so more
    // independent CTAs per SM beat wider ones
    const int R = lx_rows(lx_fwd_fixed(p), lx_fwd_per_row(p), 56 * 1024) > 0
                      ? lx_rows(lx_fwd_fixed(p), lx_fwd_per_row(p), 56 * 1024)
                      : lx_rows(lx_fwd_fixed(p), lx_fwd_per_row(p), 227 * 1024);
    if (R > 0) {
      const size_t sm = lx_fwd_fixed(p) + lx_fwd_per_row(p) * R;
      const dim3 g((unsigned)p->H, (unsigned)((B + R - 1) / R));
      auto go = [&](auto io) {
        using IO = decltype(io);
        auto k = lx_fwd_kernel<IO>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k<<<g, kLxThreads, sm, s>>>(blocks, (const IO*)x, (IO*)y, ext->dev.omap, ext->dev.tw,
                                    ext->dev.geo, (int)B, (int)p->H, (int)p->param_count, R);
      };
      if (p->dtype == FB_F32) go(float{});
      else if (p->dtype == FB_BF16) go(__nv_bfloat16{});
      else go(__half{});
      return cuda_status(cudaGetLastError(), "fb_learned_fwd");
    }
  }
  const size_t sm = (p->param_count + 2 * p->n) * sizeof(float2);
  const int rows = 4;
  const dim3 g((unsigned)p->H, (unsigned)((B + rows - 1) / rows));
  auto go = [&](auto io) {
    using IO = decltype(io);
    auto k = lb_fwd_kernel<IO>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<g, kLbThreads, sm, s>>>(blocks, (const IO*)x, (IO*)y, ext->dev.omap, ext->dev.tw,
                                ext->dev.st, (int)B, (int)p->H, (uint32_t)p->n,
                                (int)p->param_count, rows);
  };
  if (p->dtype == FB_F32) go(float{});
  else if (p->dtype == FB_BF16) go(__nv_bfloat16{});
  else go(__half{});
  return cuda_status(cudaGetLastError(), "fb_learned_fwd");
}

int fb_learned_bwd(fb_learned_plan* p, const float* blocks, const void* x, const void* g, void* dx,
                   float* dblocks, int64_t B, void* ws, void* stream) {
  if (!p || !blocks || !x || !g || !dx || !dblocks) {
    set_error("fb_learned_bwd: null argument");
    return FB_ERR_ARG;
  }
  if (B < 1) {
    set_error("learned_gradients: batch must be >= 1");
    return FB_ERR_DIM;
  }
  DevGuard dg_(p->device);
  int rc = cuda_status(dg_.err, "cudaSetDevice");
  if (rc) return rc;
  fb_learned_ext* ext = ext_of(p);
  cudaStream_t s = (cudaStream_t)stream;
  if (!ws) {
    set_error("fb_learned_bwd: workspace required (fb_learned_workspace_size)");
    return FB_ERR_ARG;
  }
  const int splits = lb_splits(p, B);
  if (ext->dev.tc) {
    rc = cuda_status(lt_bwd(ext->dev.stc, ext->dev.lgfl, p->dtype, blocks, x, g, dx, (float2*)ws,
                            ext->dev.omap, ext->dev.tw, (int)B, (int)p->H, (int)p->param_count, s),
                     "fb_learned_bwd (tcgen05)");
    if (rc) return rc;
    const size_t HP = (size_t)p->H * p->param_count;
    lb_reduce_kernel<<<(unsigned)((HP + 511) / 512), 256, 0, s>>>((const float2*)ws,
                                                                 (float2*)dblocks, splits, HP);
    return cuda_status(cudaGetLastError(), "fb_learned_bwd");
  }
  if (lx_fast_bwd(p)) {
    const int R = lx_bwd_R(p);
    const int64_t passes = (B + R - 1) / R;
    const int rps = (int)(((passes + splits - 1) / splits) * R);
    const size_t sm = lx_bwd_fixed(p) + lx_bwd_per_row(p) * R;
    auto go = [&](auto io) {
      using IO = decltype(io);
      auto k = lx_bwd_kernel<IO>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k<<<dim3((unsigned)p->H, (unsigned)splits), kLxThreads, sm, s>>>(
          blocks, (const IO*)x, (const IO*)g, (IO*)dx, (float2*)ws, ext->dev.omap, ext->dev.tw,
          ext->dev.geo, (int)B, (int)p->H, (int)p->param_count, R, rps);
    };
    if (p->dtype == FB_F32) go(float{});
    else if (p->dtype == FB_BF16) go(__nv_bfloat16{});
    else go(__half{});
    const size_t HP = (size_t)p->H * p->param_count;
    lb_reduce_kernel<<<(unsigned)((HP + 511) / 512), 256, 0, s>>>((const float2*)ws,
                                                                 (float2*)dblocks, splits, HP);
    return cuda_status(cudaGetLastError(), "fb_learned_bwd");
  }
  const int rows = (int)((B + splits - 1) / splits);
  const size_t sm = (2 * p->param_count + kLbThreads + (p->nstages + 2) * p->n) * sizeof(float2);
  if (sm > 227 * 1024) {
    set_error("learned_gradients: row too long for the on-chip backward");
    return FB_ERR_UNSUPPORTED;
  }
  auto go = [&](auto io) {
    using IO = decltype(io);
    auto k = lb_bwd_kernel<IO>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<dim3((unsigned)p->H, (unsigned)splits), kLbThreads, sm, s>>>(
        blocks, (const IO*)x, (const IO*)g, (IO*)dx, (float2*)ws, ext->dev.omap, ext->dev.tw,
        ext->dev.st, (int)B, (int)p->H, (uint32_t)p->n, (int)p->param_count, rows);
  };
  if (p->dtype == FB_F32) go(float{});
  else if (p->dtype == FB_BF16) go(__nv_bfloat16{});
  else go(__half{});
  const size_t HP = (size_t)p->H * p->param_count;
  lb_reduce_kernel<<<(unsigned)((HP + 511) / 512), 256, 0, s>>>((const float2*)ws, (float2*)dblocks,
                                                               splits, HP);
  return cuda_status(cudaGetLastError(), "fb_learned_bwd");
}

}  // extern "C"
