// FlashButterfly-B200 learned butterfly (K5) on the tcgen05 tensor cores, for
// the 16-bit modes and the chains build_plan(n, 16) gives for
// n = 16^S x FL (S in {1, 2} stages of factor 16, a last factor FL in
// {2, 4, 8}: n = 32 .. 2048, config 4's n = 1024 = [16, 16, 4]).
//
// Reference: learned_forward / learned_gradients (proj/src/butterfly.cpp:
// 235-307) over apply_stages (:124-163).  In the matrix form of
// fb_learned.cu's header, a factor-16 stage over segment L (rest = L / 16)
// is, for every column (row r, segment, q < rest),
//     out[a] = w_L^(a q) sum_p W[a][p] in[p]           (a, p < 16)
// i.e. one GEMM with the data columns on M and the real-stacked block
// [[Wr, -Wi], [Wi, Wr]] as the N = 32 operand (K = 32: re / im of the 16
// inputs interleaved).  Its adjoint g'[p] = sum_a conj(W[a][p]) w[a] is the
// same GEMM against the conjugate-transposed block, and the block gradient
//     G[a][p] += sum_columns w[a] conj(v[p])
// is the GEMM P = [w components] x [v components]^T over the columns (K),
// Gr = P[2a][2p] + P[2a+1][2p+1], Gi = P[2a+1][2p] - P[2a][2p+1], with both
// operands read MN-major out of the very buffers the stage GEMMs read
// K-major (SW64: a column's 16 complex values are one 64-byte row, and the
// SW64 K-major and MN-major canonical layouts address the same bytes).
//
// One CTA = 256 threads = R = 4096 / n rows of one head (4096 complex
// values, 256 columns per stage, one column per thread in every epilogue).
// Every stage boundary: tcgen05.mma (M = 128 x 2 tiles, N = 32, K = 32) into
// TMEM, tcgen05.ld by the column's thread, twiddle (power chain from one
// table value), bf16 store scattered into the next stage's operand rows.
// The last stage (factor FL <= 8) runs on the CUDA cores.  The backward
// recomputes the forward stage inputs, keeps them in shared memory, and
// accumulates each stage's block gradient over the CTA's columns in TMEM
// (fixed MMA order; CTAs of one head reduced by lb_reduce_kernel in a fixed
// order), so dblocks is deterministic.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "fb_common.cuh"
#include "fb_fft.cuh"
#include "fb_internal.h"
#include "fb_ptx.cuh"
#include "fb_tc.cuh"

namespace fb {
namespace ltc {

constexpr int kThreads = 256;
constexpr int kNB = 4096;                    // complex values per CTA (R rows x n)
constexpr uint32_t kOp = kNB * 4;            // bf16 operand buffer: 256 rows x 64 B (SW64)
constexpr uint32_t kNat = (kNB + kNB / 16) * 4;  // padded natural buffer (4-byte complex)
constexpr uint32_t kTab = 2048;              // one N = 32 x K = 32 block table (SW64)

// natural-order buffers padded FL words per 16 FL: the last tc stage's
// epilogue writes (segment, q) lanes at stride 16 FL, the last stage reads FL
// consecutive values per thread; both conflict-free with this padding
template <int LGFL>
__device__ __forceinline__ int pn(int e) {
  return e + ((e >> (4 + LGFL)) << LGFL);
}

// acc + a b, acc + a conj(b)
__device__ __forceinline__ float2 cfma(float2 a, float2 b, float2 acc) {
  return make_float2(fmaf(a.x, b.x, fmaf(-a.y, b.y, acc.x)), fmaf(a.x, b.y, fmaf(a.y, b.x, acc.y)));
}
__device__ __forceinline__ float2 cfmac(float2 a, float2 b, float2 acc) {
  return make_float2(fmaf(a.x, b.x, fmaf(a.y, b.y, acc.x)), fmaf(a.y, b.x, fmaf(-a.x, b.y, acc.y)));
}

__device__ __forceinline__ uint32_t pack_bf16(float2 v) {
  __nv_bfloat162 h = __floats2bfloat162_rn(v.x, v.y);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float2 unpack_bf16(uint32_t u) {
  return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u));
}
template <typename IO>
__device__ __forceinline__ float2 io_f2(uint32_t u) {
  if constexpr (std::is_same<IO, __nv_bfloat16>::value)
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u));
  else
    return __half22float2(*reinterpret_cast<const __half2*>(&u));
}
template <typename IO>
__device__ __forceinline__ uint32_t f2_io(float2 v) {
  if constexpr (std::is_same<IO, __nv_bfloat16>::value) {
    return pack_bf16(v);
  } else {
    __half2 h = __floats2half2_rn(v.x, v.y);
    return *reinterpret_cast<uint32_t*>(&h);
  }
}
// IO complex -> the bf16 operand value (a raw copy for bf16)
template <typename IO>
__device__ __forceinline__ uint32_t io_op(uint32_t u) {
  if constexpr (std::is_same<IO, __nv_bfloat16>::value) return u;
  else return pack_bf16(io_f2<IO>(u));
}

__device__ __forceinline__ uint32_t op_off(uint32_t row, uint32_t slot) {
  return tc::kmajor_off<tc::kSw64>(row, 2 * slot);  // complex slot = k pair (2 slot, 2 slot + 1)
}

// [[Mr, -Mi], [Mi, Mr]] as the N x K = 32 x 32 K-major SW64 operand, with
// M(o, i) = W[o][i] (forward) or conj(W[i][o]) (adjoint)
template <bool ADJ>
__device__ __forceinline__ void build_table(unsigned char* tab, const float2* __restrict__ W) {
  for (int i = threadIdx.x; i < 32 * 32; i += kThreads) {
    const int nn = i >> 5, k = i & 31;
    const int o = nn >> 1, co = nn & 1, in = k >> 1, ci = k & 1;
    const float2 w = __ldg(ADJ ? W + in * 16 + o : W + o * 16 + in);
    const float mr = w.x, mi = ADJ ? -w.y : w.y;
    const float val = co == 0 ? (ci == 0 ? mr : -mi) : (ci == 0 ? mi : mr);
    *reinterpret_cast<__nv_bfloat16*>(tab + tc::kmajor_off<tc::kSw64>(nn, k)) = __float2bfloat16_rn(val);
  }
}

// D[tile t][col][2a + c] = sum_k op[col][k] tab[2a + c][k], two M = 128 tiles
__device__ __forceinline__ void issue_stage(uint32_t tmem_d, uint32_t op, uint32_t tab) {
  const uint32_t id = tc::idesc_bf16(128, 32);
#pragma unroll
  for (uint32_t t = 0; t < 2; ++t)
#pragma unroll
    for (uint32_t k = 0; k < 2; ++k)
      tc::mma_bf16(tmem_d + 32 * t, tc::smem_desc(op + t * 8192 + k * 32, 512, tc::kSw64),
                   tc::smem_desc(tab + k * 32, 512, tc::kSw64), id, k);
}
// G[m][n] (+)= sum_col w[col][m] v[col][n] over the 256 columns: both operands
// MN-major SW64 (8-column groups 512 B apart); M = 128 with the MN atoms
// aliased (LBO = 0: lanes 32-127 repeat lanes 0-31 and are not read)
__device__ __forceinline__ void issue_grad(uint32_t tmem_g, uint32_t wop, uint32_t vop, bool acc) {
  const uint32_t id = tc::idesc_bf16(128, 32) | (1u << 15) | (1u << 16);
#pragma unroll
  for (uint32_t kk = 0; kk < 16; ++kk)
    tc::mma_bf16(tmem_g, tc::smem_desc(wop + kk * 1024, 512, tc::kSw64, 0),
                 tc::smem_desc(vop + kk * 1024, 512, tc::kSw64, 0), id, (acc || kk) ? 1u : 0u);
}

__device__ __forceinline__ void sync_for_mma() {
  ptx::fence_proxy_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
}
__device__ __forceinline__ void wait_mma(uint64_t* bar, uint32_t& phase) {
  ptx::mbar_wait(bar, phase);
  phase ^= 1;
  tc::fence_after();
}
// this thread's TMEM row of the stage result: tile = warp / 4, lanes of its quarter
__device__ __forceinline__ void load_col(uint32_t tmem_d, float (&v)[32]) {
  const uint32_t w = threadIdx.x >> 5;
  tc::ld32(tmem_d + ((32 * (w & 3)) << 16) + 32 * (w >> 2), v);
  tc::ld_wait();
}

// twiddles t[a] = b * s^a, a < 16 (power chain from two table values)
__device__ __forceinline__ void tw_chain(float2 (&t)[16], float2 b, float2 s) {
  t[0] = b;
#pragma unroll
  for (int a = 1; a < 16; ++a) t[a] = cmul(t[a - 1], s);
}

// forward epilogue of tc stage S: column c = tid, out[a] = w_L^(a q) D[a] to
// the next stage's operand (tc) or the natural buffer (last stage)
template <int LGN, int LGFL, int S, bool NEXT_TC>
__device__ __forceinline__ void fwd_epilogue(uint32_t tmem_d, unsigned char* next,
                                             const float2* __restrict__ tw_g) {
  constexpr int LGL = LGN - 4 * S, LGR = LGL - 4, LGC = LGN - 4;
  const int c = threadIdx.x;
  const int r = c >> LGC, cc = c & ((1 << LGC) - 1), seg = cc >> LGR, q = cc & ((1 << LGR) - 1);
  float v[32];
  load_col(tmem_d, v);
  float2 t[16];
  const float2 t1 = __ldg(tw_g + (q << (LGN - LGL)));
  tw_chain(t, make_float2(1.f, 0.f), t1);
#pragma unroll
  for (int a = 0; a < 16; ++a) {
    const float2 o = cmul(make_float2(v[2 * a], v[2 * a + 1]), t[a]);
    if constexpr (NEXT_TC) {
      constexpr int LGR2 = LGR - 4;
      const int c2 = (r << LGC) + ((seg * 16 + a) << LGR2) + (q & ((1 << LGR2) - 1));
      *reinterpret_cast<uint32_t*>(next + op_off(c2, q >> LGR2)) = pack_bf16(o);
    } else {
      const int e = (r << LGN) + (seg << LGL) + (a << LGR) + q;
      reinterpret_cast<uint32_t*>(next)[pn<LGFL>(e)] = pack_bf16(o);
    }
  }
}

// one forward tc stage: MMA batch, wait, epilogue to stage S + 1 (or the last stage)
template <int LGN, int LGFL, int STC, int S>
__device__ __forceinline__ void run_fwd_stage(uint32_t tm, uint32_t op, uint32_t tab,
                                              unsigned char* X0, unsigned char* V2,
                                              const float2* __restrict__ tw_g, uint64_t* bar,
                                              uint32_t& phase) {
  if (threadIdx.x == 0) {
    issue_stage(tm, op, tab);
    tc::commit(bar);
  }
  wait_mma(bar, phase);
  if constexpr (S + 1 < STC) fwd_epilogue<LGN, LGFL, S, true>(tm, X0 + (S + 1) * kOp, tw_g);
  else fwd_epilogue<LGN, LGFL, S, false>(tm, V2, tw_g);
  sync_for_mma();
}

// x rows (IO) -> stage-0 operand: column c = (r, q), slot p = x[r][p rest0 + q]
template <typename IO, int LGN>
__device__ __forceinline__ void load_x(unsigned char* x0, const IO* __restrict__ x, int B, int H,
                                       int h, int b0) {
  constexpr int LGC = LGN - 4;
  const int c = threadIdx.x, r = c >> LGC, q = c & ((1 << LGC) - 1);
  const int b = b0 + r;
  uint32_t u[16];
  if (b < B) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(x) + ((size_t)b * H + h) * ((size_t)1 << LGN);
#pragma unroll
    for (int p = 0; p < 16; ++p) u[p] = io_op<IO>(__ldg(src + (p << LGC) + q));
  } else {
#pragma unroll
    for (int p = 0; p < 16; ++p) u[p] = 0u;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j)
    *reinterpret_cast<uint4*>(x0 + tc::kmajor_off<tc::kSw64>(c, 8 * j)) =
        make_uint4(u[4 * j], u[4 * j + 1], u[4 * j + 2], u[4 * j + 3]);
}

struct Smem {
  uint64_t bar;
  uint32_t tmem;
};

template <typename IO, int STC, int LGFL>
__global__ void __launch_bounds__(kThreads)
    lt_fwd_kernel(const float* __restrict__ blocks, const IO* __restrict__ x, IO* __restrict__ y,
                  const uint32_t* __restrict__ omap, const float2* __restrict__ tw_g, int B, int H,
                  int P) {
  constexpr int FL = 1 << LGFL, LGN = 4 * STC + LGFL, N = 1 << LGN, R = kNB / N;
  extern __shared__ __align__(1024) unsigned char lt_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(lt_raw) + 1023) &
                                                       ~uintptr_t(1023));
  unsigned char* X0 = sm;                       // stage operands
  unsigned char* V2 = sm + STC * kOp;           // last-stage input (bf16, natural padded)
  unsigned char* OUT = V2 + kNat;               // last-stage output (IO, natural padded)
  unsigned char* TAB = OUT + kNat;              // STC forward tables
  float2* WL = reinterpret_cast<float2*>(TAB + STC * kTab);
  Smem* ss = reinterpret_cast<Smem*>(WL + FL * FL);
  const int h = blockIdx.x, b0 = blockIdx.y * R;
  const float2* W = reinterpret_cast<const float2*>(blocks) + (size_t)h * P;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&ss->bar, 1);
    ptx::fence_barrier_init();
  }
  if (threadIdx.x < 32) tc::alloc<64>(&ss->tmem);
#pragma unroll
  for (int s = 0; s < STC; ++s) build_table<false>(TAB + s * kTab, W + 256 * s);
  if (threadIdx.x < FL * FL) WL[threadIdx.x] = __ldg(W + 256 * STC + threadIdx.x);
  load_x<IO, LGN>(X0, x, B, H, h, b0);
  sync_for_mma();
  const uint32_t tm = ss->tmem, sbase = ptx::smem_u32(sm), tab = ptx::smem_u32(TAB);
  uint32_t phase = 0;
  run_fwd_stage<LGN, LGFL, STC, 0>(tm, sbase, tab, X0, V2, tw_g, &ss->bar, phase);
  if constexpr (STC == 2) run_fwd_stage<LGN, LGFL, STC, 1>(tm, sbase + kOp, tab + kTab, X0, V2, tw_g, &ss->bar, phase);
  // last stage (factor FL, no twiddle): out[a] = sum_p WL[a][p] in[p]
  const uint32_t* v2 = reinterpret_cast<const uint32_t*>(V2);
  uint32_t* out = reinterpret_cast<uint32_t*>(OUT);
  for (int j = threadIdx.x; j < kNB / FL; j += kThreads) {
    float2 in[FL];
#pragma unroll
    for (int p = 0; p < FL; ++p) in[p] = unpack_bf16(v2[pn<LGFL>(j * FL + p)]);
#pragma unroll
    for (int a = 0; a < FL; ++a) {
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int p = 0; p < FL; ++p) acc = cfma(WL[a * FL + p], in[p], acc);
      out[pn<LGFL>(j * FL + a)] = f2_io<IO>(acc);
    }
  }
  __syncthreads();
  // y[i] = cur[output_map[i]] (butterfly.cpp:161)
  for (int i = threadIdx.x; i < kNB; i += kThreads) {
    const int r = i >> LGN, e = i & (N - 1);
    if (b0 + r < B)
      reinterpret_cast<uint32_t*>(y)[((size_t)(b0 + r) * H + h) * N + e] =
          out[pn<LGFL>((r << LGN) + (int)__ldg(omap + e))];
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::dealloc<64>(tm);
}

template <typename IO, int STC, int LGFL>
__global__ void __launch_bounds__(kThreads)
    lt_bwd_kernel(const float* __restrict__ blocks, const IO* __restrict__ x,
                  const IO* __restrict__ g, IO* __restrict__ dx, float2* __restrict__ gpart,
                  const uint32_t* __restrict__ omap, const float2* __restrict__ tw_g, int B, int H,
                  int P) {
  constexpr int FL = 1 << LGFL, LGN = 4 * STC + LGFL, N = 1 << LGN, R = kNB / N;
  constexpr int LGC = LGN - 4;
  extern __shared__ __align__(1024) unsigned char lt_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(lt_raw) + 1023) &
                                                       ~uintptr_t(1023));
  unsigned char* X0 = sm;                        // stage inputs v_s (operands), s < STC
  unsigned char* WB = sm + STC * kOp;            // w of the top tc stage (w of stage 0 reuses X1)
  unsigned char* V2 = WB + kOp;                  // last-stage input (bf16, natural padded)
  unsigned char* GA = V2 + kNat;                 // upstream in stage order (IO, natural padded)
  unsigned char* TAB = GA + kNat;                // [s][fwd, adj] tables
  float2* WL = reinterpret_cast<float2*>(TAB + 2 * STC * kTab);
  float2* RED = WL + FL * FL;                    // [8 warps][<= 32] last-stage gradient partials
  Smem* ss = reinterpret_cast<Smem*>(RED + kThreads);
  const int h = blockIdx.x, b0 = blockIdx.y * R;
  const float2* W = reinterpret_cast<const float2*>(blocks) + (size_t)h * P;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&ss->bar, 1);
    ptx::fence_barrier_init();
  }
  if (threadIdx.x < 32) tc::alloc<128>(&ss->tmem);
#pragma unroll
  for (int s = 0; s < STC; ++s) {
    build_table<false>(TAB + (2 * s) * kTab, W + 256 * s);
    build_table<true>(TAB + (2 * s + 1) * kTab, W + 256 * s);
  }
  if (threadIdx.x < FL * FL) WL[threadIdx.x] = __ldg(W + 256 * STC + threadIdx.x);
  load_x<IO, LGN>(X0, x, B, H, h, b0);
  // upstream, adjoint of y[i] = cur[omap[i]]: GA[omap[i]] = g[i]
  {
    uint32_t* ga = reinterpret_cast<uint32_t*>(GA);
    for (int i = threadIdx.x; i < kNB; i += kThreads) {
      const int r = i >> LGN, e = i & (N - 1);
      const uint32_t val = b0 + r < B ? __ldg(reinterpret_cast<const uint32_t*>(g) +
                                              ((size_t)(b0 + r) * H + h) * N + e)
                                      : 0u;
      ga[pn<LGFL>((r << LGN) + (int)__ldg(omap + e))] = val;
    }
  }
  sync_for_mma();
  const uint32_t tm = ss->tmem, sbase = ptx::smem_u32(sm), tab = ptx::smem_u32(TAB);
  const uint32_t tmg = tm + 64;  // per-stage gradient accumulators, 32 columns each
  uint32_t phase = 0;
  // forward recompute: v_1 .. v_STC (the last stage's input)
  run_fwd_stage<LGN, LGFL, STC, 0>(tm, sbase, tab, X0, V2, tw_g, &ss->bar, phase);
  if constexpr (STC == 2)
    run_fwd_stage<LGN, LGFL, STC, 1>(tm, sbase + kOp, tab + 2 * kTab, X0, V2, tw_g, &ss->bar, phase);
  // last stage (CUDA cores).  Block gradient: thread = one entry (a, p),
  // columns strided; lanes of one entry reduced by shuffles, warps in order.
  const uint32_t* v2 = reinterpret_cast<const uint32_t*>(V2);
  const uint32_t* ga = reinterpret_cast<const uint32_t*>(GA);
  {
    constexpr int E = FL * FL, GROUPS = kThreads / E;
    const int ent = threadIdx.x % E, grp = threadIdx.x / E, a = ent / FL, p = ent % FL;
    float2 acc = make_float2(0.f, 0.f);
    for (int j = grp; j < kNB / FL; j += GROUPS) {
      const float2 w = io_f2<IO>(ga[pn<LGFL>(j * FL + a)]);
      const float2 vv = unpack_bf16(v2[pn<LGFL>(j * FL + p)]);
      acc = cfmac(w, vv, acc);  // w conj(v)
    }
#pragma unroll
    for (int o = E; o < 32; o <<= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    constexpr int PER = E < 32 ? E : 32;  // lanes of a warp holding distinct entries
    if ((threadIdx.x & 31) < PER) RED[(threadIdx.x >> 5) * PER + (threadIdx.x & 31)] = acc;
  }
  // adjoint of the last stage, times conj of the top tc stage's twiddle, to
  // that stage's w operand: element e = seg2 FL + p of a row sits at column
  // (r, seg2 / 16, q = p), slot seg2 % 16 of tc stage STC - 1 (L = 16 FL)
  for (int j = threadIdx.x; j < kNB / FL; j += kThreads) {
    float2 w[FL];
#pragma unroll
    for (int a = 0; a < FL; ++a) w[a] = io_f2<IO>(ga[pn<LGFL>(j * FL + a)]);
    const int r = j >> (LGN - LGFL), seg2 = j & ((1 << (LGN - LGFL)) - 1), a2 = seg2 & 15;
#pragma unroll
    for (int p = 0; p < FL; ++p) {
      float2 o = make_float2(0.f, 0.f);
#pragma unroll
      for (int a = 0; a < FL; ++a) o = cfmac(w[a], WL[a * FL + p], o);  // conj(WL[a][p]) w[a]
      o = cmulc(o, __ldg(tw_g + ((a2 * p) << (LGN - LGFL - 4))));
      const int c2 = (r << LGC) + ((seg2 >> 4) << LGFL) + p;
      *reinterpret_cast<uint32_t*>(WB + op_off(c2, a2)) = pack_bf16(o);
    }
  }
  sync_for_mma();
  // tc stages, top down: block gradient + adjoint GEMMs in one batch
  auto adjoint_stage = [&](auto s_c) {
    constexpr int s = decltype(s_c)::value;
    const uint32_t wop = s == STC - 1 ? ptx::smem_u32(WB) : sbase + (s + 1) * kOp;
    if (threadIdx.x == 0) {
      issue_grad(tmg + 32 * s, wop, sbase + s * kOp, false);
      issue_stage(tm, wop, tab + (2 * s + 1) * kTab);
      tc::commit(&ss->bar);
    }
    wait_mma(&ss->bar, phase);
    if constexpr (s > 0) {
      // column (r, seg, q) of stage s (L = n / 16^s): g'[p] at e = seg L + p rest + q;
      // stage s - 1 (L' = 16 L): a' = seg % 16, q' = p rest + q, column (r, seg / 16, q')
      constexpr int LGL = LGN - 4, LGR = STC == 2 ? LGL - 4 : 0;  // s == 1 (STC == 2)
      const int c = threadIdx.x;
      const int r = c >> LGC, cc = c & ((1 << LGC) - 1), seg = cc >> LGR, q = cc & ((1 << LGR) - 1);
      const int a2 = seg & 15;
      float v[32];
      load_col(tm, v);
      float2 t[16];
      // conj(w_{16L}^(a2 (p rest + q))) = conj(b s^p), b = w^(a2 q), s = w^(a2 rest)
      tw_chain(t, __ldg(tw_g + ((a2 * q) & (N - 1))), __ldg(tw_g + ((a2 << LGR) & (N - 1))));
      unsigned char* wdst = X0 + kOp;  // w of stage 0 over v_1 (consumed above)
#pragma unroll
      for (int p = 0; p < 16; ++p) {
        const float2 o = cmulc(make_float2(v[2 * p], v[2 * p + 1]), t[p]);
        const int c2 = (r << LGC) + ((seg >> 4) << LGL) + (p << LGR) + q;
        *reinterpret_cast<uint32_t*>(wdst + op_off(c2, a2)) = pack_bf16(o);
      }
    } else {
      // stage 0: dx[r][p rest0 + q] = g'[p]
      const int c = threadIdx.x, r = c >> LGC, q = c & ((1 << LGC) - 1);
      float v[32];
      load_col(tm, v);
      if (b0 + r < B) {
        uint32_t* dst = reinterpret_cast<uint32_t*>(dx) + ((size_t)(b0 + r) * H + h) * N;
#pragma unroll
        for (int p = 0; p < 16; ++p) dst[(p << LGC) + q] = f2_io<IO>(make_float2(v[2 * p], v[2 * p + 1]));
      }
    }
    sync_for_mma();
  };
  if constexpr (STC == 2) adjoint_stage(std::integral_constant<int, 1>());
  adjoint_stage(std::integral_constant<int, 0>());
  // block gradients -> gpart[split][h]: tc stages from TMEM (warp 0: lanes
  // m = 2a + c), the last stage from the warp partials
  float2* dg = gpart + ((size_t)blockIdx.y * H + h) * P;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
#pragma unroll 1
    for (int s = 0; s < STC; ++s) {
      float pv[32];
      tc::ld32(tmg + 32 * s, pv);
      tc::ld_wait();
      float qv[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) qv[i] = __shfl_down_sync(0xffffffffu, pv[i], 1);
      if ((lane & 1) == 0) {
        const int a = lane >> 1;
#pragma unroll
        for (int p = 0; p < 16; ++p)
          dg[256 * s + a * 16 + p] = make_float2(pv[2 * p] + qv[2 * p + 1], qv[2 * p] - pv[2 * p + 1]);
      }
    }
  }
  {
    // entry e sits in lane l = e % 32 of every warp whose lanes start at an
    // entry == e - l (mod E); warps summed in order
    constexpr int E = FL * FL, PER = E < 32 ? E : 32;
    for (int e = threadIdx.x; e < E; e += kThreads) {
      const int l = e % PER;
      float2 s = make_float2(0.f, 0.f);
      for (int wq = 0; wq < kThreads / 32; ++wq)
        if ((wq * 32 + l) % E == e) s = cadd(s, RED[wq * PER + l]);
      dg[256 * STC + e] = s;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::dealloc<128>(tm);
}

template <int STC, int LGFL>
constexpr size_t fwd_smem() {
  return 1024 + STC * kOp + 2 * kNat + STC * kTab + (1 << (2 * LGFL)) * 8 + 64;
}
template <int STC, int LGFL>
constexpr size_t bwd_smem() {
  return 1024 + (STC + 1) * kOp + 2 * kNat + 2 * STC * kTab + (1 << (2 * LGFL)) * 8 +
         kThreads * 8 + 64;
}

template <typename IO, int STC, int LGFL>
cudaError_t launch(bool bwd, const float* blocks, const void* x, const void* g, void* out,
                   float2* gpart, const uint32_t* omap, const float2* tw, int B, int H, int P,
                   cudaStream_t s) {
  constexpr int N = 1 << (4 * STC + LGFL), R = kNB / N;
  const dim3 grid((unsigned)H, (unsigned)((B + R - 1) / R));
  if (!bwd) {
    auto k = lt_fwd_kernel<IO, STC, LGFL>;
    constexpr size_t sm = fwd_smem<STC, LGFL>();
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<grid, kThreads, sm, s>>>(blocks, (const IO*)x, (IO*)out, omap, tw, B, H, P);
  } else {
    auto k = lt_bwd_kernel<IO, STC, LGFL>;
    constexpr size_t sm = bwd_smem<STC, LGFL>();
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<grid, kThreads, sm, s>>>(blocks, (const IO*)x, (const IO*)g, (IO*)out, gpart, omap, tw, B,
                                 H, P);
  }
  return cudaGetLastError();
}

template <typename IO>
cudaError_t dispatch(int stc, int lgfl, bool bwd, const float* blocks, const void* x, const void* g,
                     void* out, float2* gpart, const uint32_t* omap, const float2* tw, int B, int H,
                     int P, cudaStream_t s) {
#define LT_CASE(S_, F_)                                                                        \
  if (stc == S_ && lgfl == F_)                                                                 \
    return launch<IO, S_, F_>(bwd, blocks, x, g, out, gpart, omap, tw, B, H, P, s);
  LT_CASE(1, 1) LT_CASE(1, 2) LT_CASE(1, 3) LT_CASE(2, 1) LT_CASE(2, 2) LT_CASE(2, 3)
#undef LT_CASE
  return cudaErrorInvalidValue;
}

}  // namespace ltc

// chains [16] * stc + [2^lgfl], stc in {1, 2}, lgfl in {1, 2, 3}; 16-bit modes
bool lt_config(int64_t n, const int64_t* f, int nst, int dtype, int* stc, int* lgfl) {
  if (dtype == FB_F32 || nst < 2 || nst > 3) return false;
  for (int i = 0; i + 1 < nst; ++i)
    if (f[i] != 16) return false;
  const int64_t fl = f[nst - 1];
  if (fl != 2 && fl != 4 && fl != 8) return false;
  int lg = 0;
  while ((int64_t(1) << lg) < fl) ++lg;
  if ((int64_t(1) << (4 * (nst - 1) + lg)) != n) return false;
  const char* env = std::getenv("FB_LEARNED_TC");
  if (env && env[0] == '0') return false;
  *stc = nst - 1;
  *lgfl = lg;
  return true;
}
int lt_rows(int64_t n) { return (int)(ltc::kNB / n); }

cudaError_t lt_fwd(int stc, int lgfl, int dtype, const float* blocks, const void* x, void* y,
                   const uint32_t* omap, const float2* tw, int B, int H, int P, cudaStream_t s) {
  return dtype == FB_BF16 ? ltc::dispatch<__nv_bfloat16>(stc, lgfl, false, blocks, x, nullptr, y,
                                                          nullptr, omap, tw, B, H, P, s)
                          : ltc::dispatch<__half>(stc, lgfl, false, blocks, x, nullptr, y, nullptr,
                                                  omap, tw, B, H, P, s);
}
cudaError_t lt_bwd(int stc, int lgfl, int dtype, const float* blocks, const void* x, const void* g,
                   void* dx, float2* gpart, const uint32_t* omap, const float2* tw, int B, int H,
                   int P, cudaStream_t s) {
  return dtype == FB_BF16 ? ltc::dispatch<__nv_bfloat16>(stc, lgfl, true, blocks, x, g, dx, gpart,
                                                          omap, tw, B, H, P, s)
                          : ltc::dispatch<__half>(stc, lgfl, true, blocks, x, g, dx, gpart, omap,
                                                  tw, B, H, P, s);
}

}  // namespace fb
