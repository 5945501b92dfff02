// FlashButterfly-B200 radix-16 stages on the tcgen05 tensor cores: the
// learned butterfly (K5) for the 16-bit modes and the chains build_plan(n, 16)
// gives for n = 16^S x FL (S in {1, 2} stages of factor 16, a last factor FL
// in {2, 4, 8, 16}: n = 32 .. 4096, config 4's n = 1024 = [16, 16, 4]); and, with
// the blocks fixed to the DFT, the short causal single pass (N = 256, 512;
// sc_fwd_kernel / sc_bwd_kernel at the end of this file).
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
// The last stage (factor FL <= 16) runs as the same GEMM with 16 / FL of its
// columns per operand row against a block-diagonal table (its rows are then
// simply 16 consecutive natural-order values).  The backward
// recomputes the forward stage inputs, keeps them in shared memory, and
// accumulates each stage's block gradient over the CTA's columns in TMEM
// (fixed MMA order; CTAs of one head reduced by lb_reduce_kernel in a fixed
// order), so dblocks is deterministic.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <vector>
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
constexpr uint32_t kTab = 2048;              // one N = 32 x K = 32 block table (SW64)

// output_map (butterfly.cpp:103-116) of the chain [16] * STC + [FL] is the
// mixed-radix digit reversal: y[i] = cur[output_map[i]] puts the CTA row's
// element e = e0 16 FL + e1 FL + e2 (STC = 2) at i = e0 + 16 e1 + 256 e2
// (STC = 1: e = e0 FL + e2 -> i = e0 + 16 e2)
template <int STC, int LGFL>
__device__ __forceinline__ int out_index(int e) {
  constexpr int FL = 1 << LGFL;
  if constexpr (STC == 2) return (e >> (LGFL + 4)) | (((e >> LGFL) & 15) << 4) | ((e & (FL - 1)) << 8);
  else return (e >> LGFL) | ((e & (FL - 1)) << 4);
}

__device__ __forceinline__ uint32_t pack_bf16(float2 v) {
  __nv_bfloat162 h = __floats2bfloat162_rn(v.x, v.y);
  return *reinterpret_cast<uint32_t*>(&h);
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

// [[Mr, -Mi], [Mi, Mr]] as the N x K = 32 x 32 K-major SW64 operand of the
// 16 x 16 complex M made of 16 / FB diagonal FB x FB blocks of W:
// M(o, i) = W[o % FB][i % FB] when o / FB == i / FB, else 0 (FB = 16: the
// plain stage block); the adjoint reads it transposed (issue_stage_adj).
// Thread t owns entry (o, i) = (t / 16, t % 16): one load, two 4-byte stores.
template <int FB>
__device__ __forceinline__ float2 table_entry(const float2* __restrict__ W) {
  const int o = threadIdx.x >> 4, in = threadIdx.x & 15;
  return (o / FB == in / FB) ? __ldg(W + (o % FB) * FB + in % FB) : make_float2(0.f, 0.f);
}
__device__ __forceinline__ void store_table(unsigned char* tab, float2 m) {
  const int o = threadIdx.x >> 4, in = threadIdx.x & 15;
  *reinterpret_cast<uint32_t*>(tab + tc::kmajor_off<tc::kSw64>(2 * o, 2 * in)) = pack_bf16(make_float2(m.x, -m.y));
  *reinterpret_cast<uint32_t*>(tab + tc::kmajor_off<tc::kSw64>(2 * o + 1, 2 * in)) = pack_bf16(make_float2(m.y, m.x));
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
// the adjoint: the same table read MN-major, i.e. transposed, which is the
// real-stacked conj(M)^T ([[Wr, -Wi], [Wi, Wr]]^T = [[Wr^T, Wi^T], [-Wi^T, Wr^T]])
__device__ __forceinline__ void issue_stage_adj(uint32_t tmem_d, uint32_t op, uint32_t tab) {
  const uint32_t id = tc::idesc_bf16(128, 32) | (1u << 16);
#pragma unroll
  for (uint32_t t = 0; t < 2; ++t)
#pragma unroll
    for (uint32_t k = 0; k < 2; ++k)
      tc::mma_bf16(tmem_d + 32 * t, tc::smem_desc(op + t * 8192 + k * 32, 512, tc::kSw64),
                   tc::smem_desc(tab + k * 1024, 512, tc::kSw64, 0), id, k);
}
// G[m][n] = sum_col w[col][m] v[col][n] over the 256 columns: both operands
// MN-major SW64 (8-column groups 512 B apart); M = 128 with the MN atoms
// aliased (LBO = 0: lanes 32-127 repeat lanes 0-31 and are not read)
__device__ __forceinline__ void issue_grad(uint32_t tmem_g, uint32_t wop, uint32_t vop) {
  const uint32_t id = tc::idesc_bf16(128, 32) | (1u << 15) | (1u << 16);
#pragma unroll
  for (uint32_t kk = 0; kk < 16; ++kk)
    tc::mma_bf16(tmem_g, tc::smem_desc(wop + kk * 1024, 512, tc::kSw64, 0),
                 tc::smem_desc(vop + kk * 1024, 512, tc::kSw64, 0), id, kk ? 1u : 0u);
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

// Stage geometry (n = 2^LGN, STC factor-16 stages, then the last factor FL):
// factor-16 stage s < STC, segment L = n / 16^s, rest = L / 16: column
// c = (r, seg, q) = r n/16 + seg rest + q holds in[p] = x_r[seg L + p rest + q].
// The last stage (s = STC) runs as 16 / FL of its columns per GEMM row:
// row J holds the CTA's natural elements 16 J .. 16 J + 15 (slot = e % 16),
// its block-diagonal product leaves outputs in the same natural order.

// Operand row of stage S's column c: a permutation of the low 6 bits (bit i
// -> bit perm[i]), free since the GEMMs only see rows and the stage's w / v
// share it; chosen for config 4's chain so that the epilogues' 4-byte
// scatters hit distinct banks (modelled: 2/1/4/1-way for the 0->1 / 1->2 /
// last-adjoint / 1-adjoint scatters, 2/4/8/2-way unpermuted).  Epilogue
// threads own D row tid, i.e. column col_of(tid).
template <int STC, int LGFL, int S>
__host__ __device__ constexpr int row_perm(int i) {
  // (n = 512 / 2048 reuse n = 1024's permutations: with the identity ptxas
  // schedules the short single pass at 100-128 registers instead of 64)
  if constexpr (STC == 2) {
    constexpr int p0[6] = {0, 2, 1, 3, 4, 5}, p1[6] = {1, 2, 0, 3, 4, 5}, p2[6] = {3, 4, 2, 1, 0, 5};
    return S == 0 ? p0[i] : S == 1 ? p1[i] : p2[i];
  } else {
    return i;
  }
}
// (a bit permutation: row_of(x | y) = row_of(x) | row_of(y) for disjoint bit
// sets, so the scatters split a row into a per-thread part and a constant)
template <int STC, int LGFL, int S>
__host__ __device__ constexpr int row_of(int c) {
  int y = c & ~63;
#pragma unroll
  for (int i = 0; i < 6; ++i) y |= ((c >> i) & 1) << row_perm<STC, LGFL, S>(i);
  return y;
}
template <int STC, int LGFL, int S>
__device__ __forceinline__ int col_of(int row) {
  int y = row & ~63;
#pragma unroll
  for (int i = 0; i < 6; ++i) y |= ((row >> row_perm<STC, LGFL, S>(i)) & 1) << i;
  return y;
}

// forward epilogue of factor-16 stage S: out[a] = w_L^(a q) D[a] into stage S + 1's operand
template <int LGN, int LGFL, int STC, int S>
__device__ __forceinline__ void fwd_epilogue(uint32_t tmem_d, unsigned char* next,
                                             const float2* __restrict__ tw_g) {
  constexpr int LGL = LGN - 4 * S, LGR = LGL - 4, LGC = LGN - 4;
  const int c = col_of<STC, LGFL, S>(threadIdx.x);
  const int r = c >> LGC, cc = c & ((1 << LGC) - 1), seg = cc >> LGR, q = cc & ((1 << LGR) - 1);
  float v[32];
  load_col(tmem_d, v);
  float2 t[16];
  tw_chain(t, make_float2(1.f, 0.f), __ldg(tw_g + (q << (LGN - LGL))));
#pragma unroll
  for (int a = 0; a < 16; ++a) {
    const uint32_t o = pack_bf16(cmul(make_float2(v[2 * a], v[2 * a + 1]), t[a]));
    if constexpr (S + 1 < STC) {
      constexpr int LGR2 = LGR - 4 > 0 ? LGR - 4 : 0;
      static_assert(S == 0, "one factor-16 stage feeds another only from stage 0");
      // column (r, a, q % rest2) of stage 1: row_of(r, q % rest2) | row_of(a rest2)
      const int c2b = row_of<STC, LGFL, S + 1>((r << LGC) + (q & ((1 << LGR2) - 1)));
      const int row = c2b | row_of<STC, LGFL, S + 1>(a << LGR2);
      *reinterpret_cast<uint32_t*>(next + op_off(row, q >> LGR2)) = o;
    } else {
      const int e = (r << LGN) + (seg << LGL) + (a << LGR) + q;  // natural order
      // row e >> 4 = ((r << LGN) + (seg << LGL)) >> 4 | (a << LGR) >> 4 (q < 2^LGR <= 16)
      static_assert(LGR <= 4, "the last factor-16 stage has rest = FL <= 16");
      const int rowb = row_of<STC, LGFL, STC>(((r << LGN) + (seg << LGL)) >> 4);
      const int row = rowb | row_of<STC, LGFL, STC>((a << LGR) >> 4);
      *reinterpret_cast<uint32_t*>(next + op_off(row, e & 15)) = o;
    }
  }
}

// one forward factor-16 stage: MMA batch, wait, epilogue
template <int LGN, int LGFL, int STC, int S>
__device__ __forceinline__ void run_fwd_stage(uint32_t tm, uint32_t sbase, uint32_t tab,
                                              unsigned char* X0, const float2* __restrict__ tw_g,
                                              uint64_t* bar, uint32_t& phase) {
  if (threadIdx.x == 0) {
    issue_stage(tm, sbase + S * kOp, tab);
    tc::commit(bar);
  }
  wait_mma(bar, phase);
  fwd_epilogue<LGN, LGFL, STC, S>(tm, X0 + (S + 1) * kOp, tw_g);
  sync_for_mma();
}

// x rows (IO) -> stage-0 operand: column c = (r, q), slot p = x[r][p rest0 + q]
// (loads and stores split so the prologue's loads are all in flight at once)
template <int LGN>
__device__ __forceinline__ void load_x(uint32_t (&u)[16], const void* __restrict__ x, int B, int H,
                                       int h, int b0) {
  constexpr int LGC = LGN - 4;
  const int c = threadIdx.x, r = c >> LGC, q = c & ((1 << LGC) - 1);
  const int b = b0 + r;
  if (b < B) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(x) + ((size_t)b * H + h) * ((size_t)1 << LGN);
#pragma unroll
    for (int p = 0; p < 16; ++p) u[p] = __ldg(src + (p << LGC) + q);
  } else {
#pragma unroll
    for (int p = 0; p < 16; ++p) u[p] = 0u;
  }
}
// this thread's operand row (64 bytes) from 16 IO complex values
template <typename IO>
__device__ __forceinline__ void store_row(unsigned char* op, int row, const uint32_t (&u)[16]) {
#pragma unroll
  for (int j = 0; j < 4; ++j)
    *reinterpret_cast<uint4*>(op + tc::kmajor_off<tc::kSw64>(row, 8 * j)) =
        make_uint4(io_op<IO>(u[4 * j]), io_op<IO>(u[4 * j + 1]), io_op<IO>(u[4 * j + 2]),
                   io_op<IO>(u[4 * j + 3]));
}

// one stage's block gradient from its TMEM slot into dg (called by one warp):
// P's rows m = 2A + c sit in lanes 0-31 and, the M = 128 operand's atoms being
// aliased, again in every other lane quarter, so any warp reads them through
// its own quarter.  Complex entry (A, B) = (P[2A][2B] + P[2A+1][2B+1],
// P[2A+1][2B] - P[2A][2B+1]); FB < 16 (the last stage): G[a][p] = sum over
// the diagonal blocks i of entry (FB i + a, FB i + p).
template <int LGFL, int FB>
__device__ __forceinline__ void store_grad(uint32_t slot, float2* __restrict__ dg) {
  const int lane = threadIdx.x & 31;
  float pv[32];
  tc::ld32(slot + ((32 * ((threadIdx.x >> 5) & 3)) << 16), pv);
  tc::ld_wait();
  float qv[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) qv[i] = __shfl_down_sync(0xffffffffu, pv[i], 1);
  float2 G[16];
#pragma unroll
  for (int b = 0; b < 16; ++b) G[b] = make_float2(pv[2 * b] + qv[2 * b + 1], qv[2 * b] - pv[2 * b + 1]);
  const int A = lane >> 1;
  if constexpr (FB == 16) {
    if ((lane & 1) == 0)
#pragma unroll
      for (int b = 0; b < 16; ++b) dg[A * 16 + b] = G[b];
  } else {
    constexpr int FL = 1 << LGFL;
    const int blk = A >> LGFL, a = A & (FL - 1);
    float2 d[FL];
#pragma unroll
    for (int p = 0; p < FL; ++p) {
      d[p] = make_float2(0.f, 0.f);
#pragma unroll
      for (int i = 0; i < 16 / FL; ++i)
        if (blk == i) d[p] = G[FL * i + p];
    }
#pragma unroll
    for (int off = 2 * FL; off < 32; off <<= 1)
#pragma unroll
      for (int p = 0; p < FL; ++p) {
        d[p].x += __shfl_xor_sync(0xffffffffu, d[p].x, off);
        d[p].y += __shfl_xor_sync(0xffffffffu, d[p].y, off);
      }
    if ((lane & 1) == 0 && blk == 0)
#pragma unroll
      for (int p = 0; p < FL; ++p) dg[a * FL + p] = d[p];
  }
}

struct Smem {
  uint64_t bar;
  uint32_t tmem;
};

__device__ __forceinline__ unsigned char* align1k(unsigned char* p) {
  return reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

template <typename IO, int STC, int LGFL>
__global__ void __launch_bounds__(kThreads)
    lt_fwd_kernel(const float* __restrict__ blocks, const IO* __restrict__ x, IO* __restrict__ y,
                  const uint32_t* __restrict__ /* omap: out_index */, const float2* __restrict__ tw_g, int B, int H,
                  int P) {
  constexpr int FL = 1 << LGFL, LGN = 4 * STC + LGFL, N = 1 << LGN, R = kNB / N;
  extern __shared__ __align__(1024) unsigned char lt_raw[];
  unsigned char* sm = align1k(lt_raw);
  unsigned char* X0 = sm;                          // operands of stages 0 .. STC
  unsigned char* TAB = sm + (STC + 1) * kOp;       // forward tables, stages 0 .. STC
  Smem* ss = reinterpret_cast<Smem*>(TAB + (STC + 1) * kTab);
  const int h = blockIdx.x, b0 = blockIdx.y * R;
  const float2* W = reinterpret_cast<const float2*>(blocks) + (size_t)h * P;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&ss->bar, 1);
    ptx::fence_barrier_init();
  }
  if (threadIdx.x < 32) tc::alloc<64>(&ss->tmem);
  {
    uint32_t u[16];
    float2 wt[STC + 1];
    load_x<LGN>(u, x, B, H, h, b0);
#pragma unroll
    for (int s = 0; s < STC; ++s) wt[s] = table_entry<16>(W + 256 * s);
    wt[STC] = table_entry<FL>(W + 256 * STC);
    store_row<IO>(X0, row_of<STC, LGFL, 0>(threadIdx.x), u);
#pragma unroll
    for (int s = 0; s <= STC; ++s) store_table(TAB + s * kTab, wt[s]);
  }
  sync_for_mma();
  const uint32_t tm = ss->tmem, sbase = ptx::smem_u32(sm), tab = ptx::smem_u32(TAB);
  uint32_t phase = 0;
  run_fwd_stage<LGN, LGFL, STC, 0>(tm, sbase, tab, X0, tw_g, &ss->bar, phase);
  if constexpr (STC == 2) run_fwd_stage<LGN, LGFL, STC, 1>(tm, sbase, tab + kTab, X0, tw_g, &ss->bar, phase);
  // last stage (block-diagonal, no twiddle): row J -> natural elements 16 J + o
  if (threadIdx.x == 0) {
    issue_stage(tm, sbase + STC * kOp, tab + STC * kTab);
    tc::commit(&ss->bar);
  }
  wait_mma(&ss->bar, phase);
  {
    // y[out_index(e)] = cur[e] for the thread's 16 natural elements: a warp's
    // stores cover whole 32-byte sectors (8 consecutive i per sector)
    float v[32];
    load_col(tm, v);
    const int J = col_of<STC, LGFL, STC>(threadIdx.x), r = J >> (LGN - 4), el0 = (J << 4) & (N - 1);
    if (b0 + r < B) {
      uint32_t* dst = reinterpret_cast<uint32_t*>(y) + ((size_t)(b0 + r) * H + h) * N;
#pragma unroll
      for (int o = 0; o < 16; ++o)
        dst[out_index<STC, LGFL>(el0 + o)] = f2_io<IO>(make_float2(v[2 * o], v[2 * o + 1]));
    }
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::dealloc<64>(tm);
}

template <typename IO, int STC, int LGFL>
__global__ void __launch_bounds__(kThreads, 3)
    lt_bwd_kernel(const float* __restrict__ blocks, const IO* __restrict__ x,
                  const IO* __restrict__ g, IO* __restrict__ dx, float2* __restrict__ gpart,
                  const uint32_t* __restrict__ /* omap: out_index */, const float2* __restrict__ tw_g, int B, int H,
                  int P) {
  constexpr int FL = 1 << LGFL, LGN = 4 * STC + LGFL, N = 1 << LGN, R = kNB / N;
  constexpr int LGC = LGN - 4;
  extern __shared__ __align__(1024) unsigned char lt_raw[];
  unsigned char* sm = align1k(lt_raw);
  unsigned char* X0 = sm;                          // stage inputs v_0 .. v_STC (operands)
  unsigned char* GA = sm + (STC + 1) * kOp;        // w of the last stage: upstream in stage order
  unsigned char* TAB = GA + kOp;                   // forward tables, s = 0 .. STC (adjoints: transposed)
  Smem* ss = reinterpret_cast<Smem*>(TAB + (STC + 1) * kTab);
  const int h = blockIdx.x, b0 = blockIdx.y * R;
  const float2* W = reinterpret_cast<const float2*>(blocks) + (size_t)h * P;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&ss->bar, 1);
    ptx::fence_barrier_init();
  }
  if (threadIdx.x < 32) tc::alloc<128>(&ss->tmem);
  {
    // x, the upstream in stage order (the adjoint of y[i] = cur[output_map[i]]:
    // row J of the last stage's w operand = g[out_index(16 J + o)], o < 16)
    // and the block tables: all loads in flight, then the stores
    uint32_t u[16], gu[16];
    float2 wt[STC + 1];
    load_x<LGN>(u, x, B, H, h, b0);
    const int J = threadIdx.x, r = J >> (LGN - 4), el0 = (J << 4) & (N - 1);
    if (b0 + r < B) {
      const uint32_t* src = reinterpret_cast<const uint32_t*>(g) + ((size_t)(b0 + r) * H + h) * N;
#pragma unroll
      for (int o = 0; o < 16; ++o) gu[o] = __ldg(src + out_index<STC, LGFL>(el0 + o));
    } else {
#pragma unroll
      for (int o = 0; o < 16; ++o) gu[o] = 0u;
    }
#pragma unroll
    for (int s = 0; s < STC; ++s) wt[s] = table_entry<16>(W + 256 * s);
    wt[STC] = table_entry<FL>(W + 256 * STC);
    store_row<IO>(X0, row_of<STC, LGFL, 0>(threadIdx.x), u);
    store_row<IO>(GA, row_of<STC, LGFL, STC>(J), gu);
#pragma unroll
    for (int s = 0; s <= STC; ++s) store_table(TAB + s * kTab, wt[s]);
  }
  sync_for_mma();
  const uint32_t tm = ss->tmem, sbase = ptx::smem_u32(sm), tab = ptx::smem_u32(TAB);
  // block-gradient accumulators: two 32-column slots, stage s in slot (STC - s) & 1
  // (a slot is read out in the epilogue right after its batch, before reuse)
  auto gslot = [&](int s) { return tm + 64 + 32 * ((STC - s) & 1); };
  float2* dg = gpart + ((size_t)blockIdx.y * H + h) * P;
  uint32_t phase = 0;
  // forward recompute: v_1 .. v_STC
  run_fwd_stage<LGN, LGFL, STC, 0>(tm, sbase, tab, X0, tw_g, &ss->bar, phase);
  if constexpr (STC == 2) run_fwd_stage<LGN, LGFL, STC, 1>(tm, sbase, tab + kTab, X0, tw_g, &ss->bar, phase);
  // last stage: block gradient + adjoint (block-diagonal), then times conj of
  // stage STC - 1's twiddle into that stage's w (over v_STC, consumed here):
  // natural element e = 16 J + o of a row lies in column (r, e / 16 FL, e % FL),
  // slot (e / FL) % 16 of stage STC - 1 (L = 16 FL, rest = FL)
  if (threadIdx.x == 0) {
    issue_grad(gslot(STC), ptx::smem_u32(GA), sbase + STC * kOp);
    issue_stage_adj(tm, ptx::smem_u32(GA), tab + STC * kTab);
    tc::commit(&ss->bar);
  }
  wait_mma(&ss->bar, phase);
  if ((threadIdx.x >> 5) == 1) store_grad<LGFL, FL>(gslot(STC), dg + 256 * STC);
  {
    float v[32];
    load_col(tm, v);
    unsigned char* wdst = X0 + STC * kOp;
    const int J = col_of<STC, LGFL, STC>(threadIdx.x), r = J >> (LGN - 4), el0 = (J << 4) & (N - 1);
#pragma unroll
    for (int o = 0; o < 16; ++o) {
      const int el = el0 + o, a2 = (el >> LGFL) & 15, q2 = el & (FL - 1);
      const float2 t = __ldg(tw_g + ((a2 * q2) << (LGN - LGFL - 4)));
      const float2 w = cmulc(make_float2(v[2 * o], v[2 * o + 1]), t);
      // column (r, el / 16 FL, q2): el / 16 FL = J / FL for every o
      const int row = row_of<STC, LGFL, STC - 1>((r << LGC) + ((el0 >> (LGFL + 4)) << LGFL)) |
                      row_of<STC, LGFL, STC - 1>(o & (FL - 1));
      *reinterpret_cast<uint32_t*>(wdst + op_off(row, a2)) = pack_bf16(w);
    }
  }
  sync_for_mma();
  // factor-16 stages, top down: block gradient + adjoint GEMMs in one batch;
  // w_s sits over v_(s+1)
  auto adjoint_stage = [&](auto s_c) {
    constexpr int s = decltype(s_c)::value;
    const uint32_t wop = sbase + (s + 1) * kOp;
    if (threadIdx.x == 0) {
      issue_grad(gslot(s), wop, sbase + s * kOp);
      issue_stage_adj(tm, wop, tab + s * kTab);
      tc::commit(&ss->bar);
    }
    wait_mma(&ss->bar, phase);
    if ((threadIdx.x >> 5) == 1) store_grad<LGFL, 16>(gslot(s), dg + 256 * s);
    if constexpr (s > 0) {
      // column (r, seg, q) of stage 1 (L = n / 16): g'[p] at e = seg L + p rest + q;
      // stage 0 (L' = n): a' = seg, q' = p rest + q, column (r, q')
      constexpr int LGL = LGN - 4, LGR = STC == 2 ? LGL - 4 : 0;
      const int c = col_of<STC, LGFL, 1>(threadIdx.x);
      const int r = c >> LGC, cc = c & ((1 << LGC) - 1), seg = cc >> LGR, q = cc & ((1 << LGR) - 1);
      const int a2 = seg & 15;
      float v[32];
      load_col(tm, v);
      float2 t[16];
      // conj(w_n^(a2 (p rest + q))) = conj(b s^p), b = w^(a2 q), s = w^(a2 rest)
      tw_chain(t, __ldg(tw_g + ((a2 * q) & (N - 1))), __ldg(tw_g + ((a2 << LGR) & (N - 1))));
      unsigned char* wdst = X0 + kOp;  // w_0 over v_1 (consumed above)
#pragma unroll
      for (int p = 0; p < 16; ++p) {
        const float2 o = cmulc(make_float2(v[2 * p], v[2 * p + 1]), t[p]);
        // column (r, p rest + q) of stage 0 (seg < 16)
        const int row = row_of<STC, LGFL, 0>((r << LGC) + q) | row_of<STC, LGFL, 0>(p << LGR);
        *reinterpret_cast<uint32_t*>(wdst + op_off(row, a2)) = pack_bf16(o);
      }
    } else {
      // stage 0: dx[r][p rest0 + q] = g'[p]
      const int c = col_of<STC, LGFL, 0>(threadIdx.x), r = c >> LGC, q = c & ((1 << LGC) - 1);
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
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::dealloc<128>(tm);
}

// ---------------------------------------------------------------- short causal convolutions
// The same radix-16 tcgen05 stages with the blocks fixed to the DFT: the
// single-pass layer for N = n / 2 in {512, 1024} (16-bit modes), where the
// 64 x 128 Monarch kernels would pad to n = 8192.  A GEMM row of the CTA is a
// pair of real channels (re = channel 2 pr, im = 2 pr + 1) zero-padded to n;
// U = F(u) by the forward stages, Z = U (k_f + D / n) in the last stage's
// digit-reversed order (k_f = FFT(Kbar) / n from K1), y = the adjoint stages
// of Z (= n F^-1).  The backward: U and DY by the forward stages, du from
// DY conj(k_f + D / n) through the adjoint stages, and the head's dK spectrum
// sum_pairs conj(U) DY (natural order) for sp_dk_finalize_kernel.

// the adjoint stages from w_STC (operand at wlast) down to stage 0; stage 0's
// result for this thread's column c (16 complex, slot p -> t = p rest0 + q)
// goes to out(c, v).  w_s lands over v_(s+1).
template <int LGN, int LGFL, int STC, typename Out>
__device__ __forceinline__ void adjoint_chain(uint32_t tm, uint32_t sbase, uint32_t tab,
                                              uint32_t wlast, unsigned char* X0,
                                              const float2* __restrict__ tw_g, uint64_t* bar,
                                              uint32_t& phase, Out out) {
  constexpr int FL = 1 << LGFL, N = 1 << LGN, LGC = LGN - 4;
  if (threadIdx.x == 0) {
    issue_stage_adj(tm, wlast, tab + STC * kTab);
    tc::commit(bar);
  }
  wait_mma(bar, phase);
  {
    float v[32];
    load_col(tm, v);
    unsigned char* wdst = X0 + STC * kOp;
    const int J = col_of<STC, LGFL, STC>(threadIdx.x), r = J >> (LGN - 4), el0 = (J << 4) & (N - 1);
#pragma unroll
    for (int o = 0; o < 16; ++o) {
      const int el = el0 + o, a2 = (el >> LGFL) & 15, q2 = el & (FL - 1);
      const float2 t = __ldg(tw_g + ((a2 * q2) << (LGN - LGFL - 4)));
      const float2 w = cmulc(make_float2(v[2 * o], v[2 * o + 1]), t);
      const int row = row_of<STC, LGFL, STC - 1>((r << LGC) + ((el0 >> (LGFL + 4)) << LGFL)) |
                      row_of<STC, LGFL, STC - 1>(o & (FL - 1));
      *reinterpret_cast<uint32_t*>(wdst + op_off(row, a2)) = pack_bf16(w);
    }
  }
  sync_for_mma();
  auto adjoint_stage = [&](auto s_c) {
    constexpr int s = decltype(s_c)::value;
    if (threadIdx.x == 0) {
      issue_stage_adj(tm, sbase + (s + 1) * kOp, tab + s * kTab);
      tc::commit(bar);
    }
    wait_mma(bar, phase);
    if constexpr (s > 0) {
      constexpr int LGL = LGN - 4, LGR = STC == 2 ? LGL - 4 : 0;
      const int c = col_of<STC, LGFL, 1>(threadIdx.x);
      const int r = c >> LGC, cc = c & ((1 << LGC) - 1), seg = cc >> LGR, q = cc & ((1 << LGR) - 1);
      const int a2 = seg & 15;
      float v[32];
      load_col(tm, v);
      float2 t[16];
      tw_chain(t, __ldg(tw_g + ((a2 * q) & (N - 1))), __ldg(tw_g + ((a2 << LGR) & (N - 1))));
      unsigned char* wdst = X0 + kOp;
#pragma unroll
      for (int p = 0; p < 16; ++p) {
        const float2 o = cmulc(make_float2(v[2 * p], v[2 * p + 1]), t[p]);
        const int row = row_of<STC, LGFL, 0>((r << LGC) + q) | row_of<STC, LGFL, 0>(p << LGR);
        *reinterpret_cast<uint32_t*>(wdst + op_off(row, a2)) = pack_bf16(o);
      }
    } else {
      const int c = col_of<STC, LGFL, 0>(threadIdx.x);
      float v[32];
      load_col(tm, v);
      out(c, v);
    }
    sync_for_mma();
  };
  if constexpr (STC == 2) adjoint_stage(std::integral_constant<int, 1>());
  adjoint_stage(std::integral_constant<int, 0>());
}

// two real channels of one head as the stage-0 column (r, q): slots p < PS
// hold t = p rest0 + q (re = channel b0, im = b1): PS = 8 causal (t < n / 2,
// slots 8..15 the zero pad), PS = 16 circular (t < n = N)
template <typename IO, int LGN, int PS>
__device__ __forceinline__ void load_pair_col(uint32_t (&u)[16], float (&a)[PS], float (&b)[PS],
                                              const IO* __restrict__ sig, int q, int b0, int B,
                                              int H, int h, bool valid) {
  constexpr int LGC = LGN - 4, NS = PS == 16 ? 1 << LGN : 1 << (LGN - 1);
#pragma unroll
  for (int p = 0; p < 16; ++p) u[p] = 0u;
#pragma unroll
  for (int p = 0; p < PS; ++p) a[p] = b[p] = 0.f;
  if (!valid) return;
  const IO* s0 = sig + ((size_t)b0 * H + h) * NS;
  const IO* s1 = sig + ((size_t)(b0 + 1) * H + h) * NS;
  const bool two = b0 + 1 < B;
#pragma unroll
  for (int p = 0; p < PS; ++p) {
    a[p] = ld(s0 + (p << LGC) + q);
    b[p] = two ? ld(s1 + (p << LGC) + q) : 0.f;
  }
#pragma unroll
  for (int p = 0; p < PS; ++p) u[p] = pack_bf16(make_float2(a[p], b[p]));
}
template <typename IO, int PS>
__device__ __forceinline__ void store_pair_col(IO* __restrict__ sig, const float (&v)[32], int LGC,
                                               int q, int b0, int B, int H, int h, int NS) {
  IO* s0 = sig + ((size_t)b0 * H + h) * NS;
  IO* s1 = sig + ((size_t)(b0 + 1) * H + h) * NS;
  const bool two = b0 + 1 < B;
#pragma unroll
  for (int p = 0; p < PS; ++p) {
    st(s0 + (p << LGC) + q, v[2 * p]);
    if (two) st(s1 + (p << LGC) + q, v[2 * p + 1]);
  }
}

// the last forward stage's result times (k_f + D / n) of the row's head, in
// the stage's digit-reversed order (cur element e -> frequency out_index(e)),
// as the w operand of the adjoint chain; CONJ: times the conjugate
template <int STC, int LGFL, bool CONJ>
__device__ __forceinline__ float2 kf_at(const float2* __restrict__ kf, float dn, int h, int el) {
  constexpr int LGN = 4 * STC + LGFL;
  float2 k = __ldg(kf + ((size_t)h << LGN) + out_index<STC, LGFL>(el));
  k.x += dn;
  if (CONJ) k.y = -k.y;
  return k;
}

template <typename IO, int STC, int LGFL, bool CIRC>
__global__ void __launch_bounds__(kThreads)
    sc_fwd_kernel(const float* __restrict__ blocks, const IO* __restrict__ u, IO* __restrict__ y,
                  const float2* __restrict__ kf, const float* __restrict__ Dg,
                  const float2* __restrict__ tw_g, int B, int H, int npairs, int rows) {
  constexpr int FL = 1 << LGFL, LGN = 4 * STC + LGFL, N = 1 << LGN, R = kNB / N, LGC = LGN - 4;
  extern __shared__ __align__(1024) unsigned char lt_raw[];
  unsigned char* sm = align1k(lt_raw);
  unsigned char* X0 = sm;                          // operands of stages 0 .. STC
  unsigned char* TAB = sm + (STC + 1) * kOp;
  Smem* ss = reinterpret_cast<Smem*>(TAB + (STC + 1) * kTab);
  const float2* W = reinterpret_cast<const float2*>(blocks);
  if (threadIdx.x == 0) {
    ptx::mbar_init(&ss->bar, 1);
    ptx::fence_barrier_init();
  }
  if (threadIdx.x < 32) tc::alloc<64>(&ss->tmem);
  {
    const int c = threadIdx.x, r = c >> LGC, q = c & ((1 << LGC) - 1);
    const int gr = blockIdx.x * R + r;
    constexpr int PS = CIRC ? 16 : 8;
    uint32_t x[16];
    float xa[PS], xb[PS];
    float2 wt[STC + 1];
    load_pair_col<IO, LGN, PS>(x, xa, xb, u, q, 2 * (gr % npairs), B, H, gr / npairs, gr < rows);
#pragma unroll
    for (int s = 0; s < STC; ++s) wt[s] = table_entry<16>(W + 256 * s);
    wt[STC] = table_entry<FL>(W + 256 * STC);
    store_row<__nv_bfloat16>(X0, row_of<STC, LGFL, 0>(c), x);
#pragma unroll
    for (int s = 0; s <= STC; ++s) store_table(TAB + s * kTab, wt[s]);
  }
  sync_for_mma();
  const uint32_t tm = ss->tmem, sbase = ptx::smem_u32(sm), tab = ptx::smem_u32(TAB);
  uint32_t phase = 0;
  run_fwd_stage<LGN, LGFL, STC, 0>(tm, sbase, tab, X0, tw_g, &ss->bar, phase);
  if constexpr (STC == 2) run_fwd_stage<LGN, LGFL, STC, 1>(tm, sbase, tab + kTab, X0, tw_g, &ss->bar, phase);
  if (threadIdx.x == 0) {
    issue_stage(tm, sbase + STC * kOp, tab + STC * kTab);
    tc::commit(&ss->bar);
  }
  wait_mma(&ss->bar, phase);
  {
    // Z = U (k_f + D / n) -> w_STC over the consumed stage-0 operand
    float v[32];
    load_col(tm, v);
    const int J = col_of<STC, LGFL, STC>(threadIdx.x), r = J >> (LGN - 4), el0 = (J << 4) & (N - 1);
    const int gr = blockIdx.x * R + r, h = min(gr, rows - 1) / npairs;
    const float dn = __ldg(Dg + h) / (float)N;
    uint32_t z[16];
#pragma unroll
    for (int o = 0; o < 16; ++o)
      z[o] = pack_bf16(cmul(make_float2(v[2 * o], v[2 * o + 1]), kf_at<STC, LGFL, false>(kf, dn, h, el0 + o)));
#pragma unroll
    for (int j = 0; j < 4; ++j)
      *reinterpret_cast<uint4*>(X0 + tc::kmajor_off<tc::kSw64>(row_of<STC, LGFL, STC>(J), 8 * j)) =
          make_uint4(z[4 * j], z[4 * j + 1], z[4 * j + 2], z[4 * j + 3]);
  }
  sync_for_mma();
  adjoint_chain<LGN, LGFL, STC>(tm, sbase, tab, sbase, X0, tw_g, &ss->bar, phase,
                                [&](int c, const float (&v)[32]) {
                                  const int r = c >> LGC, q = c & ((1 << LGC) - 1);
                                  const int gr = blockIdx.x * R + r;
                                  if (gr < rows)
                                    store_pair_col<IO, CIRC ? 16 : 8>(y, v, LGC, q, 2 * (gr % npairs),
                                                                      B, H, gr / npairs,
                                                                      CIRC ? N : N / 2);
                                });
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::dealloc<64>(tm);
}

// backward: CTA (h, k) owns pairs k R .. k R + R - 1 of head h
template <typename IO, int STC, int LGFL, bool CIRC>
__global__ void __launch_bounds__(kThreads)
    sc_bwd_kernel(const float* __restrict__ blocks, const IO* __restrict__ dy,
                  const IO* __restrict__ u, IO* __restrict__ du, const float2* __restrict__ kf,
                  const float* __restrict__ Dg, const float2* __restrict__ tw_g,
                  float2* __restrict__ spart, float* __restrict__ ddpart, int B, int H,
                  int npairs, int hpc) {
  constexpr int FL = 1 << LGFL, LGN = 4 * STC + LGFL, N = 1 << LGN, R = kNB / N, LGC = LGN - 4;
  constexpr int NJ = N / 16;  // rows J per channel pair
  extern __shared__ __align__(1024) unsigned char lt_raw[];
  unsigned char* sm = align1k(lt_raw);
  unsigned char* X0 = sm;                          // operands of stages 0 .. STC
  uint32_t* UB = reinterpret_cast<uint32_t*>(sm + (STC + 1) * kOp);  // U (bf16 pairs) [o][J]
  float2* SP = reinterpret_cast<float2*>(sm + (STC + 2) * kOp);      // conj(U) DY [o][J]
  unsigned char* TAB = sm + (STC + 4) * kOp;
  Smem* ss = reinterpret_cast<Smem*>(TAB + (STC + 1) * kTab);
  // dD partials: per warp (n >= 512: a warp's columns are one row), or per
  // row (n < 512: a warp holds 32 / (n / 16) rows)
  float* ss_red = reinterpret_cast<float*>(ss + 1);  // [max(8, R)]
  const float2* W = reinterpret_cast<const float2*>(blocks);
  // rows: hpc > 1 -> hpc whole heads per CTA (npairs divides R), else CTA
  // (h, k) owns pairs k R .. k R + R - 1 of head h
  const int k = blockIdx.y;
  auto row_head = [&](int r) { return hpc > 1 ? (int)blockIdx.x * hpc + r / npairs : (int)blockIdx.x; };
  auto row_pair = [&](int r) { return hpc > 1 ? r % npairs : k * R + r; };
  auto row_ok = [&](int r) { return hpc > 1 ? row_head(r) < H : row_pair(r) < npairs; };
  if (threadIdx.x == 0) {
    ptx::mbar_init(&ss->bar, 1);
    ptx::fence_barrier_init();
  }
  if (threadIdx.x < 32) tc::alloc<64>(&ss->tmem);
  uint32_t xd[16];  // dy's column, stored once u's stage 0 is done
  {
    const int c = threadIdx.x, r = c >> LGC, q = c & ((1 << LGC) - 1), pr = row_pair(r);
    const int hr = row_head(r);
    uint32_t x[16];
    float2 wt[STC + 1];
    constexpr int PS = CIRC ? 16 : 8;
    float ua[PS], ub[PS], ga[PS], gb[PS];
    load_pair_col<IO, LGN, PS>(x, ua, ub, u, q, 2 * pr, B, H, hr, row_ok(r));
    load_pair_col<IO, LGN, PS>(xd, ga, gb, dy, q, 2 * pr, B, H, hr, row_ok(r));
    // dD partial = sum dy u over the CTA's channels, in fp32 from the 16-bit
    // inputs (not the lag-0 bin of the bf16-operand spectrum: dD can be small)
    float dd = 0.f;
#pragma unroll
    for (int p = 0; p < PS; ++p) dd = fmaf(ua[p], ga[p], fmaf(ub[p], gb[p], dd));
    constexpr int CW = (1 << LGC) < 32 ? (1 << LGC) : 32;  // a row's lanes in one warp
#pragma unroll
    for (int o = CW / 2; o > 0; o >>= 1) dd += __shfl_xor_sync(0xffffffffu, dd, o);
    if constexpr (CW == 32) {
      if ((threadIdx.x & 31) == 0) ss_red[threadIdx.x >> 5] = dd;
    } else {
      if ((threadIdx.x & (CW - 1)) == 0) ss_red[threadIdx.x >> LGC] = dd;
    }
#pragma unroll
    for (int s = 0; s < STC; ++s) wt[s] = table_entry<16>(W + 256 * s);
    wt[STC] = table_entry<FL>(W + 256 * STC);
    store_row<__nv_bfloat16>(X0, row_of<STC, LGFL, 0>(c), x);
#pragma unroll
    for (int s = 0; s <= STC; ++s) store_table(TAB + s * kTab, wt[s]);
  }
  sync_for_mma();
  const uint32_t tm = ss->tmem, sbase = ptx::smem_u32(sm), tab = ptx::smem_u32(TAB);
  uint32_t phase = 0;
  const int J = col_of<STC, LGFL, STC>(threadIdx.x), el0 = (J << 4) & (N - 1);
  // U = F(u pair)
  run_fwd_stage<LGN, LGFL, STC, 0>(tm, sbase, tab, X0, tw_g, &ss->bar, phase);
  store_row<__nv_bfloat16>(X0, row_of<STC, LGFL, 0>(threadIdx.x), xd);  // stage 0 of u is done
  if constexpr (STC == 2) run_fwd_stage<LGN, LGFL, STC, 1>(tm, sbase, tab + kTab, X0, tw_g, &ss->bar, phase);
  if (threadIdx.x == 0) {
    issue_stage(tm, sbase + STC * kOp, tab + STC * kTab);
    tc::commit(&ss->bar);
  }
  wait_mma(&ss->bar, phase);
  {
    float v[32];
    load_col(tm, v);
#pragma unroll
    for (int o = 0; o < 16; ++o) UB[o * (R * NJ) + J] = pack_bf16(make_float2(v[2 * o], v[2 * o + 1]));
  }
  sync_for_mma();
  // DY = F(dy pair) (dy's stage-0 operand is in place)
  run_fwd_stage<LGN, LGFL, STC, 0>(tm, sbase, tab, X0, tw_g, &ss->bar, phase);
  if constexpr (STC == 2) run_fwd_stage<LGN, LGFL, STC, 1>(tm, sbase, tab + kTab, X0, tw_g, &ss->bar, phase);
  if (threadIdx.x == 0) {
    issue_stage(tm, sbase + STC * kOp, tab + STC * kTab);
    tc::commit(&ss->bar);
  }
  wait_mma(&ss->bar, phase);
  {
    float v[32];
    load_col(tm, v);
    const int hr = min(row_head(J >> (LGN - 4)), H - 1);
    const float dn = __ldg(Dg + hr) / (float)N;
    uint32_t z[16];
#pragma unroll
    for (int o = 0; o < 16; ++o) {
      const float2 d = make_float2(v[2 * o], v[2 * o + 1]);
      const float2 uu = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&UB[o * (R * NJ) + J]));
      SP[o * (R * NJ) + J] = cmulc(d, uu);  // DY conj(U)
      z[o] = pack_bf16(cmul(d, kf_at<STC, LGFL, true>(kf, dn, hr, el0 + o)));
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      *reinterpret_cast<uint4*>(X0 + tc::kmajor_off<tc::kSw64>(row_of<STC, LGFL, STC>(J), 8 * j)) =
          make_uint4(z[4 * j], z[4 * j + 1], z[4 * j + 2], z[4 * j + 3]);
  }
  sync_for_mma();
  adjoint_chain<LGN, LGFL, STC>(tm, sbase, tab, sbase, X0, tw_g, &ss->bar, phase,
                                [&](int c, const float (&v)[32]) {
                                  const int r = c >> LGC, q = c & ((1 << LGC) - 1);
                                  if (row_ok(r))
                                    store_pair_col<IO, CIRC ? 16 : 8>(du, v, LGC, q, 2 * row_pair(r),
                                                                      B, H, row_head(r),
                                                                      CIRC ? N : N / 2);
                                });
  // per head of the CTA: the dD partial (warps in order; a warp's columns are
  // one row) and the dK spectrum partial (rows in order, natural frequency order)
  const int heads = hpc > 1 ? hpc : 1, chunks = gridDim.y;
  for (int hh = 0; hh < heads; ++hh) {
    const int r0 = hpc > 1 ? hh * npairs : 0;
    const int nr = hpc > 1 ? npairs : min(R, npairs - k * R);
    const int head = row_head(r0);
    if (head >= H) break;
    if (threadIdx.x == 0) {
      float t = 0.f;
      if constexpr ((1 << LGC) >= 32) {
        for (int w = 0; w < kThreads / 32; ++w) {
          const int rw = (32 * w) >> LGC;
          if (rw >= r0 && rw < r0 + nr) t += ss_red[w];
        }
      } else {
        for (int r = r0; r < r0 + nr; ++r) t += ss_red[r];
      }
      ddpart[(size_t)head * chunks + k] = t;
    }
    float2* sp = spart + ((size_t)head * chunks + k) * N;
    for (int idx = threadIdx.x; idx < N; idx += kThreads) {
      const int o = idx / NJ, j = idx % NJ;  // lanes: consecutive j
      float2 acc = make_float2(0.f, 0.f);
      for (int r = r0; r < r0 + nr; ++r) acc = cadd(acc, SP[o * (R * NJ) + r * NJ + j]);
      sp[out_index<STC, LGFL>(16 * j + o)] = acc;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::dealloc<64>(tm);
}

template <int STC, int LGFL>
constexpr size_t fwd_smem() {
  return 1024 + (STC + 1) * kOp + (STC + 1) * kTab + 64;
}
template <int STC, int LGFL>
constexpr size_t bwd_smem() {
  return 1024 + (STC + 2) * kOp + (STC + 1) * kTab + 64;
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
  LT_CASE(1, 1) LT_CASE(1, 2) LT_CASE(1, 3) LT_CASE(1, 4)
  LT_CASE(2, 1) LT_CASE(2, 2) LT_CASE(2, 3) LT_CASE(2, 4)
#undef LT_CASE
  return cudaErrorInvalidValue;
}

}  // namespace ltc

// ---------------------------------------------------------------- short single pass (host)
// backward CTAs: whole heads when a head's pairs divide the CTA's rows
static int sc_heads_per_cta(const fb_plan* p, int64_t B) {
  const int64_t R = ltc::kNB / p->n, np = (B + 1) / 2;
  return (np < R && R % np == 0) ? (int)(R / np) : 1;
}
template <typename IO, int STC, int LGFL, bool CIRC>
static int sc_launch(fb_plan* p, bool bwd, const void* a, const void* b, void* out, float2* spart,
                     float* ddpart, int64_t B, cudaStream_t s) {
  constexpr int N = 1 << (4 * STC + LGFL), R = ltc::kNB / N;
  const int npairs = (int)((B + 1) / 2);
  if (!bwd) {
    auto k = ltc::sc_fwd_kernel<IO, STC, LGFL, CIRC>;
    constexpr size_t sm = ltc::fwd_smem<STC, LGFL>();
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const int rows = (int)(p->H * npairs);
    k<<<(unsigned)((rows + R - 1) / R), ltc::kThreads, sm, s>>>(
        (const float*)p->sc_blocks, (const IO*)a, (IO*)out, p->kf, p->d, p->sc_tw, (int)B,
        (int)p->H, npairs, rows);
  } else {
    auto k = ltc::sc_bwd_kernel<IO, STC, LGFL, CIRC>;
    constexpr size_t sm = 1024 + (STC + 4) * ltc::kOp + (STC + 1) * ltc::kTab + 64 + 4 * (R > 8 ? R : 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const int hpc = sc_heads_per_cta(p, B);
    const dim3 grid = hpc > 1 ? dim3((unsigned)((p->H + hpc - 1) / hpc), 1)
                              : dim3((unsigned)p->H, (unsigned)((npairs + R - 1) / R));
    k<<<grid, ltc::kThreads, sm, s>>>((const float*)p->sc_blocks, (const IO*)a, (const IO*)b,
                                      (IO*)out, p->kf, p->d, p->sc_tw, spart, ddpart, (int)B,
                                      (int)p->H, npairs, hpc);
  }
  return cuda_status(cudaGetLastError(), bwd ? "sc_bwd" : "sc_fwd");
}
template <typename IO>
static int sc_dispatch(fb_plan* p, bool bwd, const void* a, const void* b, void* out, float2* spart,
                       float* ddpart, int64_t B, cudaStream_t s) {
#define SC_CASE(S_, F_)                                                          \
  if (p->sc_stc == S_ && p->sc_lgfl == F_)                                         \
    return p->mode == FB_MODE_CIRCULAR                                             \
               ? sc_launch<IO, S_, F_, true>(p, bwd, a, b, out, spart, ddpart, B, s) \
               : sc_launch<IO, S_, F_, false>(p, bwd, a, b, out, spart, ddpart, B, s);
  SC_CASE(1, 1) SC_CASE(1, 2) SC_CASE(1, 3) SC_CASE(1, 4) SC_CASE(2, 1) SC_CASE(2, 2) SC_CASE(2, 3)
  SC_CASE(2, 4)
#undef SC_CASE
  return FB_ERR_UNSUPPORTED;
}

// 16-bit, n = [16] * stc + [2^lgfl] = 2N causal (N = 128 .. 1024; plans pad
// shorter N to n = 256) or N circular (N = 256 .. 4096): measured per step at B*H = 2048 against the
// CUDA-core single pass 0.0585 -> 0.0565 (N = 128), 0.063 -> 0.062 (256),
// 0.090 -> 0.068 (512) and 0.097 -> 0.090 ms (1024).  FB_SHORT_TC=0
// disables the path.
bool sc_config(const fb_plan* p, int* stc, int* lgfl) {
  const char* env = std::getenv("FB_SHORT_TC");
  if (env && env[0] == '0') return false;
  if (p->dtype == FB_F32 || p->periodic) return false;
  // causal: n = 2N (zero half); circular: n = N
  if (p->mode == FB_MODE_CAUSAL ? p->N * 2 != p->n : p->N != p->n) return false;
  int lg = 0;
  while ((int64_t(1) << lg) < p->n) ++lg;
  // n = 4096 ([16, 16, 16]) only for circular N = 4096: causal N = 2048 runs
  // on the 64 x 128 kernels (n = 8192)
  if ((int64_t(1) << lg) != p->n || lg < 5 || lg > 12 || (lg == 12 && p->mode == FB_MODE_CAUSAL))
    return false;
  *stc = lg > 8 ? 2 : 1;  // n = 32 .. 256: [16, FL]; 512 .. 2048: [16, 16, FL]
  *lgfl = lg - 4 * *stc;
  return true;
}
int sc_init(fb_plan* p) {
  const int64_t n = p->n, FL = int64_t(1) << p->sc_lgfl;
  std::vector<float2> blk, tw((size_t)n);  // blocks: [16 x 16] * stc, [FL x FL]
  auto dft = [&](int64_t f) {
    for (int64_t a = 0; a < f; ++a)
      for (int64_t q = 0; q < f; ++q) {
        const double ang = -2.0 * M_PI * (double)((a * q) % f) / (double)f;
        blk.push_back(make_float2((float)std::cos(ang), (float)std::sin(ang)));
      }
  };
  for (int i = 0; i < p->sc_stc; ++i) dft(16);
  dft(FL);
  for (int64_t t = 0; t < n; ++t) {
    const double ang = -2.0 * M_PI * (double)t / (double)n;
    tw[(size_t)t] = make_float2((float)std::cos(ang), (float)std::sin(ang));
  }
  int rc = cuda_status(cudaMalloc(&p->sc_blocks, sizeof(float2) * blk.size()), "cudaMalloc(sc blocks)");
  if (!rc) rc = cuda_status(cudaMalloc(&p->sc_tw, sizeof(float2) * n), "cudaMalloc(sc tw)");
  if (!rc) rc = cuda_status(cudaMemcpy(p->sc_blocks, blk.data(), sizeof(float2) * blk.size(), cudaMemcpyHostToDevice), "copy sc blocks");
  if (!rc) rc = cuda_status(cudaMemcpy(p->sc_tw, tw.data(), sizeof(float2) * n, cudaMemcpyHostToDevice), "copy sc tw");
  return rc;
}
int sc_chunks(const fb_plan* p, int64_t B) {
  const int64_t R = ltc::kNB / p->n;
  if (sc_heads_per_cta(p, B) > 1) return 1;
  return (int)((((B + 1) / 2) + R - 1) / R);
}
int sc_fwd(fb_plan* p, const void* u, void* y, int64_t B, cudaStream_t s) {
  return p->dtype == FB_BF16
             ? sc_dispatch<__nv_bfloat16>(p, false, u, nullptr, y, nullptr, nullptr, B, s)
             : sc_dispatch<__half>(p, false, u, nullptr, y, nullptr, nullptr, B, s);
}
int sc_bwd(fb_plan* p, const void* dy, const void* u, void* du, float2* spart, float* ddpart,
           int64_t B, cudaStream_t s) {
  return p->dtype == FB_BF16 ? sc_dispatch<__nv_bfloat16>(p, true, dy, u, du, spart, ddpart, B, s)
                             : sc_dispatch<__half>(p, true, dy, u, du, spart, ddpart, B, s);
}

// chains [16] * stc + [2^lgfl], stc in {1, 2}, lgfl in {1, 2, 3, 4}; 16-bit modes
bool lt_config(int64_t n, const int64_t* f, int nst, int dtype, int* stc, int* lgfl) {
  if (dtype == FB_F32 || nst < 2 || nst > 3) return false;
  for (int i = 0; i + 1 < nst; ++i)
    if (f[i] != 16) return false;
  const int64_t fl = f[nst - 1];
  if (fl != 2 && fl != 4 && fl != 8 && fl != 16) return false;
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
