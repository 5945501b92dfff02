// FlashButterfly-B200 single-pass engine, version 2: the causal length-8192
// transform (N = 4096, 16-bit I/O, BASELINE config 2) as a 128 x 64 Monarch
// whose middle stages keep their data in TMEM.
//
// The reference computes F_n x as dense DFT blocks joined by twiddles
// (apply_stages, proj/src/butterfly.cpp:124-163) and the layer as
// IFFT(FFT(u) FFT(k))[:N] + D u (conv_butterfly :187-210, regularize.cpp:
// 149-190).  Here t = 64 t1 + t2 (t1 < 128, t2 < 64), f = f1 + 128 f2; the
// causal zero pad means t1 < 64 on the way in and only t1 < 64 on the way out:
//
//   X : DFT128 over t1     D[f1][t2 re | t2 im]   M 128  N 128  K 64    (SS)
//       data = the u pair as the MN-major B operand, landed by TMA;
//       [re | im] = C [u_a | u_b] + S [u_b | -u_a]  (the -u_a half through
//       the instruction descriptor's negate bit on an N = 64 MMA)
//       twiddle w^(f1 t2), fp32 -> bf16 pairs written back into TMEM
//   Y : DFT64 over t2      D[f1][f2 re | f2 im]   M 128  N 128  K 128   (TS)
//       A = the X output in TMEM (lane f1, K = t2 re | t2 im), B = the
//       real-stacked DFT64 block in smem: no smem operand traffic for data
//   x k_f' (k_f + D/n: the skip D u is a flat spectrum), conj -> TMEM
//   Y': the same DFT64 block on conj(Z) (IDFT = conj . DFT . conj)    (TS)
//       twiddle w^(-f1 t2) -> the X' operand in smem (the one transpose)
//   X': IDFT128 to t1 < 64 D[t1 re | t1 im][t2]  M 128  N 64   K 256   (SS)
//       A = windows of T = [C'; S'; -C'] (the im half of K reads rows 64..191,
//       the operand's im rows are written negated), so re and im rows of the
//       output are the two real channels of the pair.
//
// Two channel pairs (slots) are in flight per CTA; each slot's chain is
// MMA -> TMEM -> registers -> TMEM/smem -> MMA, and the tensor pipe runs one
// slot's MMAs while the other slot is in an epilogue.  TMEM per slot: P (128
// columns, every accumulator) and Q (64 columns, the bf16 A operand of Y / Y');
// the backward adds the CTA's dK spectrum S (128 columns).  Per pair the
// MMAs read 112 KB of shared memory (X 64 KB, Y and Y' 32 KB each... see
// DESIGN.md) instead of ~450 KB for the 64 x 128 design with the data always
// as an smem operand (fb_single_tc.cu).
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "fb_common.cuh"
#include "fb_fft.cuh"
#include "fb_internal.h"
#include "fb_ptx.cuh"
#include "fb_tc.cuh"

namespace fb {
namespace tc2 {

constexpr uint32_t kN = 8192;
// two slots x 8 warps: a slot's warp w works on TMEM lane quarter w % 4 and
// column group w / 4, i.e. a thread owns kCW of the 64 columns of a stage's
// re (or im) half for one lane
constexpr uint32_t kSlotWarps = 8, kSlotThreads = 32 * kSlotWarps, kThreads = 2 * kSlotThreads;
constexpr uint32_t kGroups = kSlotWarps / 4, kCW = 64 / kGroups;

// ---------------------------------------------------------------- smem map
// constants (host-built image, build_mats2):
//   MX_C, MX_S : cos / sin(2 pi f1 t1 / 128), A operands of X, K-major SW128
//                [f1 128][t1 64] (16 KB each)
//   MY         : real-stacked DFT64, B operand of Y / Y', K-major SW128
//                [n 128 (f2 re | f2 im)][k 128 (t2 re | t2 im)], 2 k-blocks
//   MT         : T = [C'; S'; -C'] (cos / sin(2 pi t1 f1 / 128), t1 < 64), A
//                windows of X', K-major SW128 [row 192][k 128 (f1)], 2 k-blocks
constexpr uint32_t MX_C = 0, MX_S = 16384, MY = 32768, MT = 65536;
constexpr uint32_t MT_KB = 192 * 128;  // one k-block of T
constexpr uint32_t MAT_BYTES = MT + 2 * MT_KB;
// per slot: the input pair as three MN-major planes [t1 64][t2 64]: u_a | u_b
// (TMA) | -u_a (written by the slot), so X's windows [u_a | u_b] and
// [u_b | -u_a] are N = 128 operands; and the X' B operand (MN-major
// [k 256 (f1 re | f1 im)][t2 64]), which afterwards holds the output tiles
constexpr uint32_t SIN_BYTES = 3 * 8192;
constexpr uint32_t SIN = MAT_BYTES;
constexpr uint32_t SXP = SIN + 2 * SIN_BYTES;
constexpr uint32_t STAB = SXP + 2 * 32768;  // w^t two-level table (192 float2)
constexpr uint32_t SMEM = STAB + 192 * 8;

// TMEM columns (512 allocated): slot s: P at 256 s, Q at 256 s + 128.
// Backward: S re at 192, S im at 448 (fp32, [lane f1][f2]); at a segment end
// conj(S)/n is rewritten in place over S re as the bf16 A operand of Y'.
constexpr uint32_t TS_RE = 192, TS_IM = 448;

__host__ __device__ __forceinline__ uint32_t sw128(uint32_t lin) { return lin ^ ((lin >> 3) & 0x70u); }
// K-major SW128, 64-element k-blocks of kb bytes
__host__ __device__ __forceinline__ uint32_t kmaj(uint32_t row, uint32_t k, uint32_t kb) {
  return (k >> 6) * kb + sw128((row >> 3) * 1024 + (row & 7) * 128 + (k & 63) * 2);
}
// MN-major SW128 with N = 64: [k / 8][k % 8][64 n]
__host__ __device__ __forceinline__ uint32_t mn64(uint32_t k, uint32_t n) {
  return sw128((k >> 3) * 1024 + (k & 7) * 128 + n * 2);
}

template <typename T>
struct Fmt;
template <>
struct Fmt<__nv_bfloat16> {
  static constexpr uint32_t ab = 1;
  static constexpr CUtensorMapDataType tma = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  static constexpr float spre = 1.f;  // S pre-scale into the operand (undone at the exit)
};
template <>
struct Fmt<__half> {
  static constexpr uint32_t ab = 0;
  static constexpr CUtensorMapDataType tma = CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  static constexpr float spre = 1.f / 256.f;
};

template <typename T>
__host__ __device__ constexpr uint32_t idesc(uint32_t M, uint32_t N, bool b_mn) {
  return (1u << 4) | (Fmt<T>::ab << 7) | (Fmt<T>::ab << 10) | ((b_mn ? 1u : 0u) << 16) |
         ((N >> 3) << 17) | ((M >> 4) << 24);
}

template <typename T>
__device__ __forceinline__ uint32_t pack2(float a, float b);
template <>
__device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
template <>
__device__ __forceinline__ uint32_t pack2<__half>(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t pack_bf2(float a, float b) { return pack2<__nv_bfloat16>(a, b); }
__device__ __forceinline__ float2 unpack_bf2(uint32_t v) {
  return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&v));
}
__device__ __forceinline__ float2 unpack_h2(uint32_t v) {
  return __half22float2(*reinterpret_cast<__half2*>(&v));
}
__device__ __forceinline__ uint32_t u4_get(const uint4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

// ---------------------------------------------------------------- TMEM / MMA
// tcgen05.ld 32x32b: thread i of the warp gets lane (base + i), NC consecutive columns
template <int NC>
__device__ __forceinline__ void tld(uint32_t taddr, float* v);
template <>
__device__ __forceinline__ void tld<4>(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
template <>
__device__ __forceinline__ void tld<8>(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
template <>
__device__ __forceinline__ void tld<16>(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
template <>
__device__ __forceinline__ void tld<32>(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
template <int NC>
__device__ __forceinline__ void tst(uint32_t taddr, const uint32_t* r);
template <>
__device__ __forceinline__ void tst<16>(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
template <>
__device__ __forceinline__ void tst<4>(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3])
               : "memory");
}
template <>
__device__ __forceinline__ void tst<8>(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
               "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo = 16) {
  return tc::smem_desc(saddr, 1024, tc::kSw128, lbo);
}

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(ptx::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(ptx::smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(ptx::smem_u32(src))
               : "memory");
}
// mbarrier parity wait (suspending try_wait) with a watchdog: a wait that can
// never complete (a broken protocol) reports where it stuck and traps instead
// of hanging the device
__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t parity, int tag) {
  uint32_t ok = 0;
  const long long t0 = clock64();
  for (uint32_t n = 0;; ++n) {
    asm volatile(
#ifndef FB_TC2_SPINWAIT
        "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(ptx::smem_u32(bar)), "r"(parity), "r"(0x989680)
        : "memory");
#else
        "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(ptx::smem_u32(bar)), "r"(parity)
        : "memory");
#endif
    if (ok) return;
#ifndef NO_WD
    if ((n & 15) == 15 && clock64() - t0 > 8000000000ll) {
      if ((threadIdx.x & 31) == 0)
        printf("tc2 watchdog: cta %d thread %d tag %d parity %u\n", (int)blockIdx.x, (int)threadIdx.x,
               tag, parity);
      __trap();
    }
#endif
  }
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ptx::smem_u32(bar)) : "memory");
}

// experiment build (-DFB_TC2_PROF): per (cta, slot) cycle sums of the leader's
// stages, read back through fb_debug_tc2_prof()
#ifdef FB_TC2_PROF
__device__ unsigned long long g_tc2_prof[148 * 2 * 16];
#define PSTART                     \
  long long _tp = clock64();       \
  uint32_t _acc[16];               \
  for (int _i = 0; _i < 16; ++_i) _acc[_i] = 0;
#define PMARK(k)                                 \
  {                                              \
    const long long _t = clock64();              \
    _acc[(k)] += (uint32_t)(_t - _tp);           \
    _tp = _t;                                    \
  }
#define PFLUSH                                                                                   \
  if (c.leader && blockIdx.x < 148)                                                              \
    for (int _i = 0; _i < 16; ++_i)                                                              \
      g_tc2_prof[(blockIdx.x * 2 + threadIdx.x / kSlotThreads) * 16 + _i] += _acc[_i];
#else
#define PSTART
#define PMARK(k)
#define PFLUSH
#endif

// ---------------------------------------------------------------- slot context
struct Slot {
  unsigned char* sm;
  uint32_t smb;       // smem base (shared window address)
  uint32_t tbase;     // TMEM base of the allocation
  uint32_t P, Q;      // TMEM column offsets
  uint32_t sin, sxp;  // smem offsets of the slot's input planes / X' operand
  uint32_t bar_id;    // named barrier
  uint64_t* mma_bar;
  uint32_t phase;
  bool leader;
  // thread coordinates, re-read through volatile asm where used (loop
  // invariant; hoisting everything derived from them costs more registers
  // than recomputing): TMEM lane = f1 (or the t1 re / im row at the X' exit),
  // column group g (columns [kCW g, kCW g + kCW) of a 64-column half), index
  // within the slot
  __device__ __forceinline__ uint32_t tid() const {
    uint32_t t;
    asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
    return t;
  }
  __device__ __forceinline__ uint32_t lane() const { return 32 * ((tid() >> 5) & 3) + (tid() & 31); }
  __device__ __forceinline__ uint32_t grp() const { return (tid() >> 7) & (kGroups - 1); }
  __device__ __forceinline__ uint32_t st() const { return tid() & (kSlotThreads - 1); }
};

__device__ __forceinline__ uint32_t ta(const Slot& c, uint32_t col) {
  return c.tbase + ((32u * ((c.tid() >> 5) & 3)) << 16) + col;
}
__device__ __forceinline__ void slot_sync(const Slot& c) {
  asm volatile("bar.sync %0, %1;" ::"r"(c.bar_id), "n"(kSlotThreads) : "memory");
}
// make the slot's TMEM / smem writes visible to its next MMAs
__device__ __forceinline__ void publish(const Slot& c, bool smem) {
  if (smem) ptx::fence_proxy_async_smem();
  tc::fence_before();
  slot_sync(c);
  tc::fence_after();
}
__device__ __forceinline__ void commit_wait(Slot& c) {
  if (c.leader) tc::commit(c.mma_bar);
  wait_bar(c.mma_bar, c.phase, 1);
  c.phase ^= 1;
  tc::fence_after();
}

// MMA token (forward): the slots' MMA batches alternate on the tensor pipe —
// slot 0's batch j waits for slot 1's batch j - 1, slot 1's batch j for slot
// 0's batch j (while the other slot still has batches) — so one slot's batch
// runs while the other slot is in its epilogue instead of both queueing behind
// each other in phase.  Only the leader waits; `nb` counts the slot's batches.
struct Token {
  uint64_t* other;  // the other slot's MMA barrier
  uint32_t slot, nb, on;  // on: the other slot's batches in this launch
  __device__ __forceinline__ void wait() {
    if (slot == 0) {
      if (nb >= 1 && nb - 1 < on) wait_bar(other, (nb - 1) & 1, 4);
    } else if (nb < on) {
      wait_bar(other, nb & 1, 4);
    }
    ++nb;
  }
};

// X: [re | im] = C [u_a | u_b] + S [u_b | -u_a]  (windows of the three planes)
template <typename T>
__device__ __forceinline__ void mma_X(const Slot& c) {
  const uint32_t d = c.tbase + c.P;
  const uint32_t in = c.smb + c.sin;
#pragma unroll
  for (uint32_t s = 0; s < 4; ++s) {
    mma_ss(d, desc(c.smb + MX_C + s * 32), desc(in + s * 2048, 8192), idesc<T>(128, 128, true), s);
    mma_ss(d, desc(c.smb + MX_S + s * 32), desc(in + 8192 + s * 2048, 8192), idesc<T>(128, 128, true),
           1);
  }
}
// Y / Y': D = A(TMEM columns a_col..+64) x DFT64-stacked
template <typename T>
__device__ __forceinline__ void mma_Y(const Slot& c, uint32_t a_col) {
  const uint32_t d = c.tbase + c.P;
#pragma unroll
  for (uint32_t s = 0; s < 8; ++s)
    mma_ts(d, c.tbase + a_col + 8 * s, desc(c.smb + MY + (s >> 2) * 16384 + (s & 3) * 32),
           idesc<T>(128, 128, false), s);
}
// X': D[t1 re | t1 im][t2] = T-window x operand
template <typename T>
__device__ __forceinline__ void mma_Xp(const Slot& c) {
  const uint32_t d = c.tbase + c.P;
#pragma unroll
  for (uint32_t s = 0; s < 16; ++s) {
    const uint32_t a = c.smb + MT + ((s & 7) >> 2) * MT_KB + (s >= 8 ? 8192u : 0u) + (s & 3) * 32;
    mma_ss(d, desc(a), desc(c.smb + c.sxp + s * 2048), idesc<T>(128, 64, true), s);
  }
}

// ---------------------------------------------------------------- epilogues
// the slot's -u_a plane (a sign flip, exact), one 16-byte chunk per thread
__device__ __forceinline__ void negate_plane(const Slot& c) {
  const uint4* src = reinterpret_cast<const uint4*>(c.sm + c.sin);
  uint4* dst = reinterpret_cast<uint4*>(c.sm + c.sin + 16384);
  for (uint32_t i = c.st(); i < 512; i += kSlotThreads) {
    uint4 v = src[i];
    v.x ^= 0x80008000u;
    v.y ^= 0x80008000u;
    v.z ^= 0x80008000u;
    v.w ^= 0x80008000u;
    dst[i] = v;
  }
}

// The thread's stage-boundary twiddles w^(f1 t2), t2 = kCW g + j, as kCW / 8
// rotation chains: their starts and the step, computed once per kernel and
// kept in registers (exits never touch shared memory for them: the SS MMAs
// keep the smem port busy)
struct Tw {
  float2 st;  // w^f1 (the chain starts are its powers, by repeated squaring)
};
__device__ __forceinline__ Tw make_tw(const Slot& c, const float2* tab) {
  Tw t;
  t.st = tw2<-1>(tab, c.lane());
  return t;
}
// (re, im)[j] x w^(SIGN f1 (kCW g + 16 h + j)), j < 16 (chunk h of the thread's columns)
// packed fp32x2 arithmetic (FFMA2 / FMUL2: two lanes per instruction)
__device__ __forceinline__ unsigned long long f2u(float2 v) {
  return (unsigned long long)__float_as_uint(v.x) | ((unsigned long long)__float_as_uint(v.y) << 32);
}
__device__ __forceinline__ float2 u2f(unsigned long long v) {
  return make_float2(__uint_as_float((uint32_t)v), __uint_as_float((uint32_t)(v >> 32)));
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
  return u2f(d);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(d);
}
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }
// (ar + i ai) (wr + i wi) on two lanes at once
__device__ __forceinline__ void cmul2(float2& ar, float2& ai, float2 wr, float2 wi) {
  const float2 zr = fma2(ai, neg2(wi), mul2(ar, wr));
  const float2 zi = fma2(ar, wi, mul2(ai, wr));
  ar = zr;
  ai = zi;
}

// (re, im)[j] x w^(SIGN f1 (kCW g + 16 hc + j)), j < 16: two rotation chains
// over the element pairs (j, j + 1), stepping by st^2, in packed fp32x2
template <int SIGN>
__device__ __forceinline__ void twiddle16(const Slot& c, const Tw& tw, int hc, float* re, float* im) {
#ifdef FB_TC2_NOTW
  return;
#endif
  const float2 st = SIGN < 0 ? tw.st : make_float2(tw.st.x, -tw.st.y);
  // chain starts st^(kCW g + 16 hc) and st^(kCW g + 16 hc + 8)
  const float2 s2 = cmul(st, st), s4 = cmul(s2, s2), s8 = cmul(s4, s4), s16 = cmul(s8, s8);
  float2 w0 = hc ? s16 : make_float2(1.f, 0.f);
  if (kCW == 32 && c.grp()) w0 = cmul(w0, cmul(s16, s16));
  if (kCW == 16) {
    const uint32_t gg = c.grp();
    if (gg & 1) w0 = cmul(w0, s16);
    if (gg & 2) w0 = cmul(w0, cmul(s16, s16));
  }
  const float2 w8 = cmul(w0, s8);
  const float2 w1 = cmul(w0, st), w9 = cmul(w8, st);
  float2 WR[2] = {make_float2(w0.x, w1.x), make_float2(w8.x, w9.x)};
  float2 WI[2] = {make_float2(w0.y, w1.y), make_float2(w8.y, w9.y)};
  const float2 SR = make_float2(s2.x, s2.x), SI = make_float2(s2.y, s2.y);
#pragma unroll
  for (int p = 0; p < 4; ++p) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int j = 8 * r + 2 * p;
      float2 ar = make_float2(re[j], re[j + 1]), ai = make_float2(im[j], im[j + 1]);
      cmul2(ar, ai, WR[r], WI[r]);
      re[j] = ar.x;
      re[j + 1] = ar.y;
      im[j] = ai.x;
      im[j + 1] = ai.y;
      if (p < 3) cmul2(WR[r], WI[r], SR, SI);
    }
  }
}

// X exit: D[f1][t2] w^(f1 t2) -> Q as bf16/fp16 pairs (k = t2 re | t2 im), 16 columns at a time
template <typename T>
__device__ __forceinline__ void exit_X(const Slot& c, const Tw& tw) {
#ifdef FB_TC2_NOEPI
  return;
#endif
#pragma unroll
  for (int hc = 0; hc < (int)kCW / 16; ++hc) {
    float re[16], im[16];
    tld<16>(ta(c, c.P + kCW * c.grp() + 16 * hc), re);
    tld<16>(ta(c, c.P + 64 + kCW * c.grp() + 16 * hc), im);
    ld_wait();
    twiddle16<-1>(c, tw, hc, re, im);
    uint32_t pr[8], pi[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      pr[j] = pack2<T>(re[2 * j], re[2 * j + 1]);
      pi[j] = pack2<T>(im[2 * j], im[2 * j + 1]);
    }
    tst<8>(ta(c, c.Q + (kCW / 2) * c.grp() + 8 * hc), pr);
    tst<8>(ta(c, c.Q + 32 + (kCW / 2) * c.grp() + 8 * hc), pi);
  }
  st_wait();
}

// Y' exit: conj(D)[f1][t2] w^(-f1 t2) -> the X' operand (row f1: re, row 128 + f1: -im)
template <typename T>
__device__ __forceinline__ void exit_Yp(const Slot& c, const Tw& tw) {
#ifdef FB_TC2_NOEPI
  return;
#endif
  unsigned char* op = c.sm + c.sxp;
#pragma unroll
  for (int hc = 0; hc < (int)kCW / 16; ++hc) {
    float re[16], im[16];
    tld<16>(ta(c, c.P + kCW * c.grp() + 16 * hc), re);
    tld<16>(ta(c, c.P + 64 + kCW * c.grp() + 16 * hc), im);
    ld_wait();
#pragma unroll
    for (int j = 0; j < 16; ++j) im[j] = -im[j];  // the IDFT's output conjugation
    twiddle16<+1>(c, tw, hc, re, im);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const uint32_t n = kCW * c.grp() + 16 * hc + 8 * q;
      uint4 vr, vi;
      vr.x = pack2<T>(re[8 * q + 0], re[8 * q + 1]);
      vr.y = pack2<T>(re[8 * q + 2], re[8 * q + 3]);
      vr.z = pack2<T>(re[8 * q + 4], re[8 * q + 5]);
      vr.w = pack2<T>(re[8 * q + 6], re[8 * q + 7]);
      vi.x = pack2<T>(-im[8 * q + 0], -im[8 * q + 1]);
      vi.y = pack2<T>(-im[8 * q + 2], -im[8 * q + 3]);
      vi.z = pack2<T>(-im[8 * q + 4], -im[8 * q + 5]);
      vi.w = pack2<T>(-im[8 * q + 6], -im[8 * q + 7]);
      *reinterpret_cast<uint4*>(op + mn64(c.lane(), n)) = vr;
      *reinterpret_cast<uint4*>(op + mn64(128 + c.lane(), n)) = vi;
    }
  }
}

// X' exit: lane t1 (re rows -> channel b0, im rows -> b0 + 1), t2 = kCW g + j,
// scaled, into the slot's (now free) X' operand region as two SW128 tiles
// [64 t1][64 t2] (the TMA box layout); store_pair then writes them out with
// two bulk tensor copies (a missing odd partner's rows are out of bounds: skipped)
template <typename T>
__device__ __forceinline__ void exit_Xp(const Slot& c, float sc) {
#ifdef FB_TC2_NOEPI
  return;
#endif
  float v[kCW];
  tld<kCW>(ta(c, c.P + kCW * c.grp()), v);
  ld_wait();
  const uint32_t t1 = c.lane() & 63;
  unsigned char* tile = c.sm + c.sxp + (c.lane() >= 64 ? 8192u : 0u) + t1 * 128;
#pragma unroll
  for (int q = 0; q < (int)kCW / 8; ++q) {
    uint4 w;
    w.x = pack2<T>(v[8 * q + 0] * sc, v[8 * q + 1] * sc);
    w.y = pack2<T>(v[8 * q + 2] * sc, v[8 * q + 3] * sc);
    w.z = pack2<T>(v[8 * q + 4] * sc, v[8 * q + 5] * sc);
    w.w = pack2<T>(v[8 * q + 6] * sc, v[8 * q + 7] * sc);
    *reinterpret_cast<uint4*>(tile + ((((kCW / 8) * c.grp() + q) ^ (t1 & 7)) << 4)) = w;
  }
}
__device__ __forceinline__ void store_pair(const Slot& c, const CUtensorMap* map, int h, int b0, int H) {
  tma_store_2d(map, c.sm + c.sxp, 0, (b0 * H + h) * 64);
  tma_store_2d(map, c.sm + c.sxp + 8192, 0, ((b0 + 1) * H + h) * 64);
  ptx::bulk_commit();
}

// the CTA's share of the pairs (forward: balanced; backward: even-aligned so a
// head segment splits evenly over the two slots — tc_dk_tail's owner() mirrors it)
__device__ __forceinline__ void cta_range(int total, int& i0, int& i1) {
  i0 = (int)(((int64_t)blockIdx.x * total) / gridDim.x);
  i1 = (int)(((int64_t)(blockIdx.x + 1) * total) / gridDim.x);
}
__device__ __forceinline__ void cta_range_even(int total, int& i0, int& i1) {
  const int64_t U = (total + 1) / 2;
  i0 = min(total, (int)(2 * ((int64_t)blockIdx.x * U / gridDim.x)));
  i1 = min(total, (int)(2 * ((int64_t)(blockIdx.x + 1) * U / gridDim.x)));
}

// pair (b0, b0 + 1) of head h: two 8 KB boxes [64 t1][64 t2] (row (b H + h) 64);
// an odd batch's missing partner is out of bounds and lands as zeros
__device__ __forceinline__ void load_pair(unsigned char* dst, const CUtensorMap* map, int h, int b0,
                                          int H, uint64_t* bar) {
  ptx::mbar_arrive_expect_tx(bar, 16384);
  tma_2d(dst, map, 0, (b0 * H + h) * 64, bar);
  tma_2d(dst + 8192, map, 0, ((b0 + 1) * H + h) * 64, bar);
}
// k_f' / U rows of lane f1 in the [f2 / 4][f1][f2 % 4] layouts: a warp's
// 16-byte accesses cover 512 contiguous bytes
__device__ __forceinline__ const uint4* lane_row(const uint4* base, size_t row, const Slot& c) {
  return base + row * (kN / 4) + (kCW / 4) * 128 * c.grp() + c.lane();
}

__device__ __forceinline__ Slot setup(unsigned char* sm, uint32_t* tmem_slot, uint64_t* bars, int nbars,
                                      const uint4* __restrict__ mats, const float2* __restrict__ tab_g) {
  if (reinterpret_cast<uintptr_t>(sm) & 1023) __trap();
  if (threadIdx.x < 32) tc::alloc<512>(tmem_slot);
  if (threadIdx.x == 0) {
    for (int i = 0; i < nbars; ++i) ptx::mbar_init(&bars[i], 1);
    ptx::fence_barrier_init();
  }
  uint4* dm = reinterpret_cast<uint4*>(sm);
  for (uint32_t i = threadIdx.x; i < MAT_BYTES / 16; i += kThreads) dm[i] = __ldg(mats + i);
  float2* tab = reinterpret_cast<float2*>(sm + STAB);
  for (uint32_t i = threadIdx.x; i < 192; i += kThreads) tab[i] = __ldg(tab_g + i);
  ptx::fence_proxy_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  Slot c;
  const uint32_t slot = threadIdx.x / kSlotThreads;
  c.sm = sm;
  c.smb = ptx::smem_u32(sm);
  c.tbase = *tmem_slot;
  c.P = 256 * slot;
  c.Q = 256 * slot + 128;
  c.sin = SIN + SIN_BYTES * slot;
  c.sxp = SXP + 32768 * slot;
  c.bar_id = 1 + slot;
  c.mma_bar = &bars[slot];
  c.phase = 0;
  c.leader = (threadIdx.x & (kSlotThreads - 1)) == 0;
  return c;
}

__device__ __forceinline__ void teardown(uint32_t tmem) {
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (threadIdx.x < 32) tc::dealloc<512>(tmem);
}

// ------------------------------------------------------------------ forward
// Persistent: CTA c owns pairs [i0, i1) (head-major), slot s takes i0 + s,
// i0 + s + 2, ...  usave (training step / recompute scratch): U = F(u) as
// bf16 pairs [pair][f2 / 4][f1][f2 % 4] for the backward.  SPECTRUM: stop
// after Y (U only, no y).
template <typename T, bool SPECTRUM>
__global__ void __launch_bounds__(kThreads, 1)
    tc2_fwd_kernel(const __grid_constant__ CUtensorMap umap, const __grid_constant__ CUtensorMap ymap,
                   const uint4* __restrict__ kf16, const float* __restrict__ kscale,
                   const uint4* __restrict__ mats, const float2* __restrict__ tab_g, int B, int H,
                   int total, uint4* __restrict__ usave, int tok_on) {
  constexpr bool kScaleEarly = std::is_same<T, __half>::value;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bars[4];  // mma[2], in[2]
  const int npairs = (B + 1) / 2;
  int i0, i1;
  cta_range(total, i0, i1);
  Slot c = setup(smem_raw, &tmem_slot, bars, 4, mats, tab_g);
  const Tw tw = make_tw(c, reinterpret_cast<const float2*>(smem_raw + STAB));
  const uint32_t slot = threadIdx.x / kSlotThreads;
  uint64_t* in_bar = &bars[2 + slot];
  int item = i0 + (int)slot;
  if (c.leader && item < i1)
    load_pair(c.sm + c.sin, &umap, item / npairs, 2 * (item % npairs), H, in_bar);
  Token tok{&bars[slot ^ 1], slot, 0, (SPECTRUM ? 2u : 4u) * (uint32_t)((i1 - i0 - (int)(slot ^ 1) + 1) / 2)};
  if (tok_on == 0) tok.on = 0, tok.slot = 1;  // experiment: free issue
  PSTART
  for (uint32_t it = 0; item < i1; item += 2, ++it) {
    const int h = item / npairs, b0 = 2 * (item % npairs);
    // ---- X (every thread has passed this wait before the leader refills the
    // planes: the refill follows the next slot barrier)
    wait_bar(in_bar, it & 1, 2);
    PMARK(0)
    negate_plane(c);
    publish(c, true);
    if (c.leader) {
      tok.wait();
      mma_X<T>(c);
    }
    commit_wait(c);
    PMARK(1)
    exit_X<T>(c, tw);
    PMARK(2)
    publish(c, false);
    PMARK(3)
    // ---- Y
    if (c.leader) {
      tok.wait();
      mma_Y<T>(c, c.Q);
      if (item + 2 < i1)  // the input planes are free again
        load_pair(c.sm + c.sin, &umap, (item + 2) / npairs, 2 * ((item + 2) % npairs), H, in_bar);
    }
    uint4 kq[kCW / 4];  // k_f' [f2 / 4][f1][f2 % 4]
    {
      const uint4* kp = lane_row(kf16, h, c);
#pragma unroll
      for (int q = 0; q < (int)kCW / 4; ++q) kq[q] = __ldg(kp + 128 * q);
    }
    const float sc = __ldg(kscale + h);
    commit_wait(c);
    PMARK(4)
    {
      uint4* us = usave ? const_cast<uint4*>(lane_row(usave, item, c)) : nullptr;
#pragma unroll
      for (int q = 0; q < (int)kCW / 8; ++q) {
        float re[8], im[8];
        tld<8>(ta(c, c.P + kCW * c.grp() + 8 * q), re);
        tld<8>(ta(c, c.P + 64 + kCW * c.grp() + 8 * q), im);
        ld_wait();
        if (us) {  // U = F(u), bf16 pairs: coalesced 16-byte stores
          us[256 * q] = make_uint4(pack_bf2(re[0], im[0]), pack_bf2(re[1], im[1]),
                                   pack_bf2(re[2], im[2]), pack_bf2(re[3], im[3]));
          us[256 * q + 128] = make_uint4(pack_bf2(re[4], im[4]), pack_bf2(re[5], im[5]),
                                         pack_bf2(re[6], im[6]), pack_bf2(re[7], im[7]));
        }
        if constexpr (!SPECTRUM) {
          uint32_t pr[4], pi[4];
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            float zr[2], zi[2];
#pragma unroll
            for (int d = 0; d < 2; ++d) {
              float2 k = unpack_h2(u4_get(kq[2 * q + ((e + d) >> 2)], (e + d) & 3));
              if constexpr (kScaleEarly) {
                k.x *= sc;
                k.y *= sc;
              }
              const float a = re[e + d], b = im[e + d];
              zr[d] = fmaf(a, k.x, -b * k.y);
              zi[d] = -fmaf(a, k.y, b * k.x);  // conj(Z): Y' runs the forward block
            }
            pr[e / 2] = pack2<T>(zr[0], zr[1]);
            pi[e / 2] = pack2<T>(zi[0], zi[1]);
          }
          tst<4>(ta(c, c.Q + (kCW / 2) * c.grp() + 4 * q), pr);
          tst<4>(ta(c, c.Q + 32 + (kCW / 2) * c.grp() + 4 * q), pi);
        }
      }
      if constexpr (!SPECTRUM) st_wait();
    }
    if constexpr (!SPECTRUM) {
      PMARK(5)
      if (c.leader) ptx::bulk_wait_read<0>();  // the previous y tiles left the X' region
      publish(c, false);
      PMARK(6)
      // ---- Y'
      if (c.leader) {
        tok.wait();
        mma_Y<T>(c, c.Q);
      }
      commit_wait(c);
      PMARK(7)
      exit_Yp<T>(c, tw);
      PMARK(8)
      publish(c, true);
      PMARK(9)
      // ---- X'
      if (c.leader) {
        tok.wait();
        mma_Xp<T>(c);
      }
      commit_wait(c);
      PMARK(10)
      exit_Xp<T>(c, kScaleEarly ? 1.f : sc);
      PMARK(11)
      ptx::fence_proxy_async_smem();
    }
    // P free for the next X; the y tiles complete
    tc::fence_before();
    slot_sync(c);
    if constexpr (!SPECTRUM)
      if (c.leader) store_pair(c, &ymap, h, b0, H);
    PMARK(12)
  }
  PFLUSH
  if (c.leader) ptx::bulk_wait<0>();
  teardown(tmem_slot);
}

// ------------------------------------------------------------------ backward
// Persistent like the forward; the CTA walks its pairs head segment by head
// segment, slot s takes local pairs s, s + 2, ...  Per pair: DY = F(dy) (X, Y),
// S += conj(U) DY with U the forward's saved transform (S = the CTA's dK
// spectrum, fp32 in TMEM, updated strictly in the CTA's pair order across the
// slots through two mbarriers, so the sum is deterministic), du =
// F^-1(DY conj(k_f')) (Y', X').  At a segment's last pair its slot turns S into
// the time-domain partial Re F^-1(S)[t < N] on the tensor cores (Y', X' on
// conj(S)/n in place of S) -> tpart[cta][seg][t]; tc_dk_tail (fb_single_tc.cu)
// sums a head's partials in a fixed order and applies the regularizer chain rule.
//
// The slot's items in CTA order: segment (start a, head h, length L), local
// index j (j = slot, slot + 2, ...); cnt = the other slot's pairs in earlier
// segments, so the other slot's S updates before (a, j) number
// cnt + |{j' < j : j' = other (mod 2)}|.
struct SlotIter {
  int a, j, h, L, cnt;
  int i1, npairs, slot;
  __device__ __forceinline__ int other_in(int len) const { return slot ? (len + 1) / 2 : len / 2; }
  __device__ __forceinline__ void settle() {
    while (a < i1) {
      h = a / npairs;
      L = min(i1, (h + 1) * npairs) - a;
      if (j < L) return;
      cnt += other_in(L);
      a += L;
      j = slot;
    }
  }
  __device__ __forceinline__ void next() {
    j += 2;
    settle();
  }
  __device__ __forceinline__ int other_before() const { return cnt + (slot ? (j + 1) / 2 : j / 2); }
};

template <typename T>
__global__ void __launch_bounds__(kThreads, 1)
    tc2_bwd_kernel(const __grid_constant__ CUtensorMap dymap, const __grid_constant__ CUtensorMap dumap,
                   const uint4* __restrict__ kf16, const float* __restrict__ kscale,
                   const uint4* __restrict__ mats, const float2* __restrict__ tab_g,
                   float* __restrict__ tpart, int B, int H, int total, int maxseg,
                   const uint4* __restrict__ usave, int tok_on) {
  constexpr bool kScaleEarly = std::is_same<T, __half>::value;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bars[6];  // mma[2], in[2], S chain[2]
  const int npairs = (B + 1) / 2;
  int i0, i1;
  cta_range_even(total, i0, i1);
  Slot c = setup(smem_raw, &tmem_slot, bars, 6, mats, tab_g);
  const Tw tw = make_tw(c, reinterpret_cast<const float2*>(smem_raw + STAB));
  const int slot = (int)(threadIdx.x / kSlotThreads);
  uint64_t* in_bar = &bars[2 + slot];
  uint64_t* chain_mine = &bars[4 + slot];
  uint64_t* chain_other = &bars[5 - slot];
  const int seg0 = i0 / npairs;
  SlotIter it{i0, slot, 0, 0, 0, i1, npairs, slot};
  it.settle();
  // the other slot's MMA batches: 4 per pair + 2 per segment end it handles
  Token tok{&bars[slot ^ 1], (uint32_t)slot, 0, 0};
  {
    SlotIter o{i0, slot ^ 1, 0, 0, 0, i1, npairs, slot ^ 1};
    o.settle();
    for (; o.a < i1; o.next()) tok.on += (o.j == o.L - 1) ? 6u : 4u;
  }
  if (!tok_on) tok.on = 0, tok.slot = 1;
  if (c.leader && it.a < i1)
    load_pair(c.sm + c.sin, &dymap, it.h, 2 * (it.a + it.j - it.h * npairs), H, in_bar);
  for (uint32_t in_it = 0; it.a < i1; ++in_it) {
    const int h = it.h, item = it.a + it.j, b0 = 2 * (item - h * npairs);
    const bool first = it.j == 0, last = it.j == it.L - 1;
    const int other_before = it.other_before();
    SlotIter nx = it;
    nx.next();
    // ---- X (dy)
    wait_bar(in_bar, in_it & 1, 2);
    negate_plane(c);
    publish(c, true);
    if (c.leader) {
      tok.wait();
      mma_X<T>(c);
    }
    commit_wait(c);
    exit_X<T>(c, tw);
    publish(c, false);
    // ---- Y (dy)
    if (c.leader) {
      tok.wait();
      mma_Y<T>(c, c.Q);
      if (nx.a < i1)
        load_pair(c.sm + c.sin, &dymap, nx.h, 2 * (nx.a + nx.j - nx.h * npairs), H, in_bar);
    }
    uint4 uq[kCW / 4], kq[kCW / 4];
    {
      const uint4* up = lane_row(usave, item, c);
      const uint4* kp = lane_row(kf16, h, c);
#pragma unroll
      for (int q = 0; q < (int)kCW / 4; ++q) {
        uq[q] = __ldg(up + 128 * q);
        kq[q] = __ldg(kp + 128 * q);
      }
    }
    const float sc = __ldg(kscale + h);
    commit_wait(c);
    // ---- Y exit: S (+)= conj(U) DY in the CTA's pair order; Z = DY conj(k_f') -> Q as conj(Z)
    if (other_before > 0) {
      wait_bar(chain_other, (other_before - 1) & 1, 3);
      tc::fence_after();
    }
#pragma unroll
    for (int q = 0; q < (int)kCW / 4; ++q) {
      float dr[4], di[4], sr[4], si[4];
      tld<4>(ta(c, c.P + kCW * c.grp() + 4 * q), dr);
      tld<4>(ta(c, c.P + 64 + kCW * c.grp() + 4 * q), di);
      if (!first) {
        tld<4>(ta(c, TS_RE + kCW * c.grp() + 4 * q), sr);
        tld<4>(ta(c, TS_IM + kCW * c.grp() + 4 * q), si);
      }
      ld_wait();
      uint32_t pz[2], qz[2];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 u = unpack_bf2(u4_get(uq[q], e));
        const float cr = fmaf(u.x, dr[e], u.y * di[e]);
        const float ci = fmaf(u.x, di[e], -u.y * dr[e]);
        sr[e] = first ? cr : sr[e] + cr;
        si[e] = first ? ci : si[e] + ci;
        float2 k = unpack_h2(u4_get(kq[q], e));
        if constexpr (kScaleEarly) {
          k.x *= sc;
          k.y *= sc;
        }
        // Z = DY conj(k); the operand takes conj(Z)
        const float zr = fmaf(dr[e], k.x, di[e] * k.y);
        const float zi = fmaf(di[e], k.x, -dr[e] * k.y);
        dr[e] = zr;
        di[e] = -zi;
      }
      tst<4>(ta(c, TS_RE + kCW * c.grp() + 4 * q), reinterpret_cast<const uint32_t*>(sr));
      tst<4>(ta(c, TS_IM + kCW * c.grp() + 4 * q), reinterpret_cast<const uint32_t*>(si));
      pz[0] = pack2<T>(dr[0], dr[1]);
      pz[1] = pack2<T>(dr[2], dr[3]);
      qz[0] = pack2<T>(di[0], di[1]);
      qz[1] = pack2<T>(di[2], di[3]);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(
                       ta(c, c.Q + (kCW / 2) * c.grp() + 2 * q)),
                   "r"(pz[0]), "r"(pz[1])
                   : "memory");
      asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(
                       ta(c, c.Q + 32 + (kCW / 2) * c.grp() + 2 * q)),
                   "r"(qz[0]), "r"(qz[1])
                   : "memory");
    }
    st_wait();
    if (c.leader) ptx::bulk_wait_read<0>();  // the previous du tiles left the X' region
    if (last) {
      // ---- segment end: conj(S)/n (x spre) as the Y' operand, in place of S re
      publish(c, false);
      float sr[kCW], si[kCW];
      tld<kCW>(ta(c, TS_RE + kCW * c.grp()), sr);
      tld<kCW>(ta(c, TS_IM + kCW * c.grp()), si);
      ld_wait();
      tc::fence_before();
      slot_sync(c);  // every thread's S read before any operand write
      constexpr float kS = Fmt<T>::spre / (float)kN;
      uint32_t pr[kCW / 2], pi[kCW / 2];
#pragma unroll
      for (int e = 0; e < (int)kCW / 2; ++e) {
        pr[e] = pack2<T>(sr[2 * e] * kS, sr[2 * e + 1] * kS);
        pi[e] = pack2<T>(-si[2 * e] * kS, -si[2 * e + 1] * kS);
      }
      tst<kCW / 2>(ta(c, TS_RE + (kCW / 2) * c.grp()), pr);
      tst<kCW / 2>(ta(c, TS_RE + 32 + (kCW / 2) * c.grp()), pi);
      st_wait();
      publish(c, false);
      if (c.leader) {
        tok.wait();
        mma_Y<T>(c, TS_RE);
      }
      commit_wait(c);
      if (c.leader) mbar_arrive(chain_mine);  // S consumed: the next update may overwrite it
      exit_Yp<T>(c, tw);
      publish(c, true);
      if (c.leader) {
        tok.wait();
        mma_Xp<T>(c);
      }
      commit_wait(c);
      {
        float v[kCW];
        tld<kCW>(ta(c, c.P + kCW * c.grp()), v);
        ld_wait();
        if (c.lane() < 64) {
          float4* o = reinterpret_cast<float4*>(tpart + ((size_t)blockIdx.x * maxseg + (h - seg0)) * 4096 +
                                                64 * c.lane() + kCW * c.grp());
          constexpr float kU = 1.f / Fmt<T>::spre;
#pragma unroll
          for (int q = 0; q < (int)kCW / 4; ++q)
            o[q] = make_float4(v[4 * q] * kU, v[4 * q + 1] * kU, v[4 * q + 2] * kU, v[4 * q + 3] * kU);
        }
      }
      tc::fence_before();
      slot_sync(c);
      tc::fence_after();
    } else {
      tc::fence_before();
      slot_sync(c);
      tc::fence_after();
      if (c.leader) mbar_arrive(chain_mine);
    }
    // ---- Y' (du)
    if (c.leader) {
      tok.wait();
      mma_Y<T>(c, c.Q);
    }
    commit_wait(c);
    exit_Yp<T>(c, tw);
    publish(c, true);
    // ---- X'
    if (c.leader) {
      tok.wait();
      mma_Xp<T>(c);
    }
    commit_wait(c);
    exit_Xp<T>(c, kScaleEarly ? 1.f : sc);
    ptx::fence_proxy_async_smem();
    tc::fence_before();
    slot_sync(c);
    if (c.leader) store_pair(c, &dumap, h, b0, H);
    it = nx;
  }
  if (c.leader) ptx::bulk_wait<0>();
  teardown(tmem_slot);
}

}  // namespace tc2

#ifdef FB_TC2_PROF
extern "C" int fb_debug_tc2_prof(unsigned long long* out, int reset) {
  if (reset) {
    static unsigned long long z[148 * 2 * 16] = {0};
    return (int)cudaMemcpyToSymbol(tc2::g_tc2_prof, z, sizeof(z));
  }
  return (int)cudaMemcpyFromSymbol(out, tc2::g_tc2_prof, sizeof(unsigned long long) * 148 * 2 * 16);
}
#endif

// ---------------------------------------------------------------- host side
namespace {
using namespace tc2;

template <typename T>
void put(std::vector<uint8_t>& img, uint32_t off, double v) {
  T h;
  if constexpr (std::is_same<T, __nv_bfloat16>::value) h = __float2bfloat16_rn((float)v);
  else h = __float2half_rn((float)v);
  std::memcpy(&img[off], &h, 2);
}

template <typename T>
std::vector<uint8_t> build_mats2() {
  std::vector<uint8_t> img(MAT_BYTES, 0);
  // X: C / S [f1][t1], angle 2 pi f1 t1 / 128
  for (int f1 = 0; f1 < 128; ++f1)
    for (int t1 = 0; t1 < 64; ++t1) {
      const double a = 2.0 * M_PI * (double)((f1 * t1) % 128) / 128.0;
      put<T>(img, MX_C + kmaj(f1, t1, 16384), std::cos(a));
      put<T>(img, MX_S + kmaj(f1, t1, 16384), std::sin(a));
    }
  // Y: B[k][n], k = t2 re | t2 im, n = f2 re | f2 im:
  //   re out = sum xr c + xi s, im out = sum xi c - xr s  (W64 = c - i s)
  for (int n = 0; n < 128; ++n)
    for (int k = 0; k < 128; ++k) {
      const int t2 = k & 63, f2 = n & 63;
      const double a = 2.0 * M_PI * (double)((t2 * f2) % 64) / 64.0;
      const double cs = std::cos(a), sn = std::sin(a);
      double v;
      if (k < 64) v = n < 64 ? cs : -sn;
      else v = n < 64 ? sn : cs;
      put<T>(img, MY + kmaj(n, k, 16384), v);
    }
  // X': T = [C'; S'; -C'], angle 2 pi t1 f1 / 128, t1 < 64
  for (int r = 0; r < 192; ++r)
    for (int f1 = 0; f1 < 128; ++f1) {
      const int t1 = r & 63;
      const double a = 2.0 * M_PI * (double)((t1 * f1) % 128) / 128.0;
      const double v = r < 64 ? std::cos(a) : (r < 128 ? std::sin(a) : -std::cos(a));
      put<T>(img, MT + kmaj(r, f1, MT_KB), v);
    }
  return img;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);
EncodeFn encode_fn2() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

// signal [B][H][4096] as rows of 64: [B H 64][64]; box [64 t1][64 t2], SW128
template <typename T>
int make_map2(CUtensorMap* map, const void* ptr, int64_t B, int64_t H) {
  EncodeFn enc = encode_fn2();
  if (!enc) {
    set_error("tcgen05 path: cuTensorMapEncodeTiled unavailable");
    return FB_ERR_CUDA;
  }
  const cuuint64_t dims[2] = {64, (cuuint64_t)(B * H * 64)};
  const cuuint64_t strides[1] = {64 * 2};
  const cuuint32_t box[2] = {64, 64};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, Fmt<T>::tma, 2, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return FB_ERR_CUDA;
  }
  return FB_OK;
}
}  // namespace

// experiment switch FB_TC2_TOKEN: bit 0 = MMA token in the forward, bit 1 = in the backward
static int tc2_token() {
  static const int v = [] {
    const char* e = std::getenv("FB_TC2_TOKEN");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}

int tc2_init(fb_plan* p) {
  std::vector<uint8_t> img = p->dtype == FB_BF16 ? build_mats2<__nv_bfloat16>() : build_mats2<__half>();
  int rc = cuda_status(cudaMalloc(&p->tc_mats, img.size()), "cudaMalloc(tc mats)");
  if (!rc)
    rc = cuda_status(cudaMemcpy(p->tc_mats, img.data(), img.size(), cudaMemcpyHostToDevice),
                     "copy tc mats");
  return rc;
}

int tc2_fwd(fb_plan* p, const void* u, void* y, int64_t B, int ctas, int total, cudaStream_t s,
            void* usave, bool spectrum_only) {
  CUtensorMap map, ymap;
  auto go = [&](auto tv) {
    using T = decltype(tv);
    int rc = make_map2<T>(&map, u, B, p->H);
    if (!rc) rc = make_map2<T>(&ymap, y ? y : u, B, p->H);
    if (rc) return rc;
    auto launch = [&](auto k) {
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
      if (!spectrum_only) prof_mark(p, 0, 0, s);
      k<<<(unsigned)ctas, kThreads, SMEM, s>>>(map, ymap, (const uint4*)p->kf_tc, p->kf_scale,
                                               (const uint4*)p->tc_mats, p->tw2, (int)B, (int)p->H,
                                               total, (uint4*)usave, tc2_token() & 1);
      if (!spectrum_only) prof_mark(p, 0, 1, s);
    };
    if (spectrum_only) launch(tc2_fwd_kernel<T, true>);
    else launch(tc2_fwd_kernel<T, false>);
    return cuda_status(cudaGetLastError(), "tc2_fwd");
  };
  return p->dtype == FB_BF16 ? go(__nv_bfloat16{}) : go(__half{});
}

int tc2_bwd(fb_plan* p, const void* dy, void* du, int64_t B, int ctas, int total, int maxseg,
            float* tpart, const void* usave, cudaStream_t s) {
  CUtensorMap map, dumap;
  auto go = [&](auto tv) {
    using T = decltype(tv);
    int rc = make_map2<T>(&map, dy, B, p->H);
    if (!rc) rc = make_map2<T>(&dumap, du, B, p->H);
    if (rc) return rc;
    auto k = tc2_bwd_kernel<T>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    prof_mark(p, 1, 0, s);
    k<<<(unsigned)ctas, kThreads, SMEM, s>>>(map, dumap, (const uint4*)p->kf_tc, p->kf_scale,
                                             (const uint4*)p->tc_mats, p->tw2, tpart, (int)B,
                                             (int)p->H, total, maxseg, (const uint4*)usave,
                                             tc2_token() & 2);
    prof_mark(p, 1, 1, s);
    return cuda_status(cudaGetLastError(), "tc2_bwd");
  };
  return p->dtype == FB_BF16 ? go(__nv_bfloat16{}) : go(__half{});
}

}  // namespace fb
