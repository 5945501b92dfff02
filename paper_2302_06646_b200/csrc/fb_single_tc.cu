// FlashButterfly-B200 single-pass engine on the 5th-gen tensor cores
// (tcgen05 + TMEM + TMA) for the 16-bit I/O modes at n = 8192 (N = 4096,
// causal) — BASELINE config 2.
//
// The reference's butterfly (apply_stages, proj/src/butterfly.cpp:124-163)
// computes F_n x as dense DFT blocks joined by twiddles.  Here F_8192 is the
// two-factor Monarch product n = 64 (t1) x 128 (t2), t = 128 t1 + t2,
// f = f1 + 64 f2:
//   A : DFT64 over t1        D[t2][f1]   M 128 (t2)  N 128 (f1 re|im)  K 64 (t1<32 re|im)
//       twiddle w_8192^(f1 t2)
//   B : DFT128 over t2       D[f2][f1]   M 128 (f2)  N 64 (f1) x {re, im}  K 128 (t2)
//       (the DFT128 block is the A operand: Xr = Fr.Ar - Fi.Ai, Xi = Fi.Ar + Fr.Ai,
//        four real GEMMs, the minus via the instruction descriptor's negate bit)
//   x k_f' = (K_hat + D)/n   (the skip D u is a flat spectrum)
//   B': IDFT128 over f2      D[t2][f1]   (conj block: Fr.Zr + Fi.Zi, Fr.Zi - Fi.Zr)
//       twiddle w_8192^(-f1 t2)
//   A': IDFT64 over f1       D[t2][t1]   M 128  N 64 (t1<32 re|im)  K 128 (f1 re|im)
// Causal zero padding is pruned on both ends (t1 < 32 in A and A').  Every
// dense block is a tcgen05.mma on bf16/fp16 operands with fp32 accumulation
// in TMEM.  Each stage boundary is one TMEM -> register -> smem epilogue in
// which a thread owns 16 consecutive elements of the next operand, so every
// operand write is a pair of 16-byte stores into a 128B-swizzled UMMA
// layout; the u pair arrives by 4-D TMA boxes written straight into the
// MN-major swizzled operand.  Two real channels (b, b+1) of one head ride as
// re/im of one transform.
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "fb_common.cuh"
#include "fb_fft.cuh"
#include "fb_internal.h"
#include "fb_ptx.cuh"
#include "fb_tc.cuh"
#include "fb_reg.cuh"

namespace fb {
namespace tcfft {

constexpr uint32_t kN = 8192;
constexpr uint32_t kThreads = 512;

// ---------------------------------------------------------------- smem map
// Two independent 16-warp slots per CTA; each slot runs its own channel pair
// through A -> B -> (x k_f') -> B' -> A', so one slot's epilogue (CUDA cores)
// overlaps the other slot's MMAs (tensor pipe).
//   SIN  [slot]: u/dy pair, [mb 2][kg 8][8 k][64 m] bf16 (16 KB), kg 0-3 =
//               channel b0 t1 0..31, kg 4-7 = b1 (the TMA box order)
//   SOP  [slot]: 32 KB operand of stages B, B', A' (one live at a time)
//   FA         : stage-A block [128 rows (f1 re|im)][64 k (t1<32 re|im)]
//               K-major SW128; read as an MN-major B operand it is exactly the
//               stage-A' block (conj(F64) restricted to t1 < 32), so A' needs
//               no matrix of its own
//   FR, FI     : DFT128 real / imaginary [128][128] K-major SW128 (2 k-blocks)
//   KF   (bwd) : k_f' as fp16 pairs [f1 64][f2 128] x per-head scale
constexpr uint32_t kSlotThreads = 256;
// a slot's 16 warps: 4 per TMEM lane quarter, so each thread owns 1/kGroups
// of a row's columns (16 of the 64 complex columns of a stage)
constexpr uint32_t kGroups = kSlotThreads / 128;
constexpr uint32_t kColsPer = 64 / kGroups;
constexpr uint32_t SIN = 0;
constexpr uint32_t SOP = SIN + 2 * 16384;
constexpr uint32_t SMAT = SOP + 2 * 32768;
constexpr uint32_t MAT_FA = 0, MAT_FR = 16384, MAT_FI = 49152, MAT_BYTES = 81920;
constexpr uint32_t STAB = SMAT + MAT_BYTES;
// Forward layout: three 16 KB operand planes per slot so each stage-B/B'
// K-step is two N = 128 MMAs (a 2-plane window of [Xr | Xi] or [-Xi | Xr]
// against Fr / Fi) instead of four N = 64 ones — 61 % vs 46 % of the tensor
// peak (profiles/r01_microbench_tcgen05.md).
constexpr uint32_t SOP3 = SIN + 2 * 16384;
constexpr uint32_t SMAT3 = SOP3 + 2 * 49152;
constexpr uint32_t STAB3 = SMAT3 + MAT_BYTES;
constexpr uint32_t SMEM_FWD = STAB3 + 1536;
// Backward: same planes, plus half of k_f' — K-bar and D are real, so
// k_f'[n - f] = conj(k_f'[f]) and rows f2 <= 64 ([f1 64][65] fp16 pairs)
// cover the spectrum.  231168 B of the 231424 B left next to the 1 KB of
// static smem.
constexpr uint32_t KFH_ROW = 65;
constexpr uint32_t SKF3 = STAB3 + 1536;
constexpr uint32_t SMEM_BWD3 = SKF3 + 64 * KFH_ROW * 4;

__device__ __forceinline__ unsigned char* smem_base(unsigned char* raw) {
  if (reinterpret_cast<uintptr_t>(raw) & 1023) __trap();  // swizzle atoms need 1 KB alignment
  return raw;
}

// TMEM columns (512 allocated).  Slot s works in [128 s, 128 s + 128).
// Forward: the slot's k_f' copy at 256 + 128 s (re f1 0..63 | im).
// Backward: U parked as bf16 pairs at 256 + 64 s, the CTA's dK spectrum
// accumulator S at 384..511 (shared by the slots, updated in pair order).
constexpr uint32_t TKF = 256, TPK = 256, TS = 384;

__host__ __device__ __forceinline__ uint32_t sw128(uint32_t lin) { return lin ^ ((lin >> 3) & 0x70u); }
// MN-major B operand with N = 64: [kg][8 k][64 n]
__host__ __device__ __forceinline__ uint32_t off_bmn(uint32_t n, uint32_t k) {
  return sw128((k >> 3) * 1024 + (k & 7) * 128 + n * 2);
}
// K-major SW128 operand with 128-byte rows, K split in 64-element blocks of
// `kblock` bytes: [k / 64][row / 8][row % 8][k % 64]
__host__ __device__ __forceinline__ uint32_t off_kmaj(uint32_t row, uint32_t k, uint32_t kblock) {
  return sw128((k >> 6) * kblock + (row >> 3) * 1024 + (row & 7) * 128 + (k & 63) * 2);
}

template <typename T>
struct Fmt;
template <>
struct Fmt<__nv_bfloat16> {
  static constexpr uint32_t ab = 1;
  static constexpr CUtensorMapDataType tma = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
};
template <>
struct Fmt<__half> {
  static constexpr uint32_t ab = 0;
  static constexpr CUtensorMapDataType tma = CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
};

template <typename T>
__host__ __device__ constexpr uint32_t idesc(uint32_t M, uint32_t N, bool a_mn, bool b_mn,
                                             bool neg_a = false) {
  return (1u << 4) | (Fmt<T>::ab << 7) | (Fmt<T>::ab << 10) | ((neg_a ? 1u : 0u) << 13) |
         ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
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
template <typename T>
__device__ __forceinline__ float2 unpack2(uint32_t v);
template <>
__device__ __forceinline__ float2 unpack2<__nv_bfloat16>(uint32_t v) {
  return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&v));
}
template <>
__device__ __forceinline__ float2 unpack2<__half>(uint32_t v) {
  return __half22float2(*reinterpret_cast<__half2*>(&v));
}
template <typename T>
__device__ __forceinline__ void st8(unsigned char* p, const float* v) {
  uint4 q;
  q.x = pack2<T>(v[0], v[1]);
  q.y = pack2<T>(v[2], v[3]);
  q.z = pack2<T>(v[4], v[5]);
  q.w = pack2<T>(v[6], v[7]);
  *reinterpret_cast<uint4*>(p) = q;
}

template <typename T>
__device__ __forceinline__ void st8n(unsigned char* p, const float* v) {
  uint4 q;
  q.x = pack2<T>(-v[0], -v[1]);
  q.y = pack2<T>(-v[2], -v[3]);
  q.z = pack2<T>(-v[4], -v[5]);
  q.w = pack2<T>(-v[6], -v[7]);
  *reinterpret_cast<uint4*>(p) = q;
}

template <int NC>
__device__ __forceinline__ void tld(uint32_t taddr, float* v);
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
__device__ __forceinline__ void tld<8>(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tst8(uint32_t taddr, const float* v) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
               "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tst_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4, %5}], [%6];" ::"r"(ptx::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(ptx::smem_u32(bar))
      : "memory");
}

// Data rows t1 of a channel: N / 128 = 32 (N = 4096) or 16 (N = 2048, the
// same n = 8192 transform with u zero beyond 2048: stage A skips the K steps
// of rows 16..31, the A' exit stores rows < 16).  Set once per CTA.
__shared__ uint32_t g_rows;
// the CTA's one-time bulk load of its DFT blocks (setup)
__shared__ __align__(8) uint64_t g_setup_bar;

// Channel pair (b0, b0+1) of head h: 4 boxes [64 t2][g_rows t1] (4 KB / 2 KB),
// channel c of 64-row block mb at dst + mb * 8 KB + c * 4 KB.  An odd batch's
// missing partner is out of bounds and arrives as zeros.
__device__ __forceinline__ void load_pair(unsigned char* dst, const CUtensorMap* map, int h, int b0,
                                          uint64_t* bar) {
  ptx::mbar_arrive_expect_tx(bar, 4 * 128 * g_rows);
#pragma unroll
  for (int mb = 0; mb < 2; ++mb)
#pragma unroll
    for (int c = 0; c < 2; ++c) tma_load_4d(dst + mb * 8192 + c * 4096, map, mb * 64, 0, h, b0 + c, bar);
}

// Thread coordinates re-read through volatile asm inside the epilogues (they
// are loop invariant; hoisting the derived addresses costs more registers
// than recomputing them).
__device__ __forceinline__ uint32_t tid_v() {
  uint32_t t;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
  return t;
}
// Slot-local coordinates: TMEM lane row = 32 (warp % 4) + lane (a warp may
// only touch its lane quarter) and column half g (warps 0-3 / 4-7 of the slot).
__device__ __forceinline__ void coords(uint32_t& row, uint32_t& g) {
  const uint32_t t = tid_v();
  row = 32 * ((t >> 5) & 3) + (t & 31);
  g = (t >> 7) & (kGroups - 1);
}
__device__ __forceinline__ bool slot_leader() { return (tid_v() & (kSlotThreads - 1)) == 0; }

struct Ctx {
  unsigned char* sm;
  uint32_t smb;
  uint32_t tmem;    // TMEM base (lane 0, column 0)
  uint32_t tw;      // the slot's working columns
  uint32_t aux;     // fwd: the slot's k_f' columns; bwd: the slot's parked-U columns
  uint32_t in_off;  // the slot's input buffer (bytes into smem)
  uint32_t sop;     // the slot's operand buffer
  uint32_t smat;    // DFT blocks (bytes into smem)
  uint32_t bar_id;  // the slot's named barrier
  uint64_t* mma_bar;
  uint32_t mma_phase;
  const float2* tab;
  // MMA token: the slots' MMA batches alternate on the tensor pipe (slot 0,
  // slot 1, slot 0, ...) so one slot's MMAs run while the other slot is in
  // its epilogue, instead of both slots queueing behind each other and then
  // idling in lock-step.  Batch j of the current segment (nb - seg0) waits
  // for the other slot's batch j - 1 (slot 0) / j (slot 1) to complete, as
  // long as the other slot has that many batches in the segment.
  uint32_t slot;
  uint64_t* other_bar;
  uint32_t nb;       // batches this slot issued so far
  uint32_t seg0;     // nb at the start of the current segment
  uint32_t obase;    // the other slot's batch count at the segment start
  uint32_t on;       // the other slot's batches in the segment
  // MMA-issue lock (experiment switch FB_TC_SCHED=1): a leader issues its
  // whole batch while holding it, so the slots' batches reach the tensor pipe
  // contiguous and first-ready-first-served, without waiting for each
  // other's completion (the token) or interleaving (free issue)
  uint32_t* lock;
};

__device__ __forceinline__ Ctx make_ctx(unsigned char* sm, uint32_t tmem, uint32_t slot,
                                        uint64_t* mma_bar, bool w3 = false) {
  Ctx c;
  c.sm = sm;
  c.smb = ptx::smem_u32(sm);
  c.tmem = tmem;
  c.tw = 128 * slot;
  c.aux = 0;
  c.in_off = SIN + 16384 * slot;
  c.sop = w3 ? SOP3 + 49152 * slot : SOP + 32768 * slot;
  c.smat = w3 ? SMAT3 : SMAT;
  c.bar_id = 1 + slot;
  c.mma_bar = mma_bar;
  c.mma_phase = 0;
  c.tab = reinterpret_cast<const float2*>(sm + (w3 ? STAB3 : STAB));
  c.slot = slot;
  c.other_bar = mma_bar + (slot ? -1 : 1);
  c.nb = c.seg0 = c.obase = c.on = 0;
  c.lock = nullptr;
  return c;
}

__device__ __forceinline__ uint32_t taddr(const Ctx& c, uint32_t col) {
  return c.tmem + ((32u * ((tid_v() >> 5) & 3)) << 16) + col;
}

__device__ __forceinline__ void slot_sync(const Ctx& c) {
  asm volatile("bar.sync %0, %1;" ::"r"(c.bar_id), "n"(kSlotThreads) : "memory");
}
// make the slot's generic smem writes and TMEM reads visible before its next MMAs
__device__ __forceinline__ void publish(const Ctx& c) {
  ptx::fence_proxy_async_smem();
  tc::fence_before();
  slot_sync(c);
  tc::fence_after();
}
__device__ __forceinline__ void mma_wait(Ctx& c) {
  ptx::mbar_wait(c.mma_bar, c.mma_phase);
  c.mma_phase ^= 1;
  tc::fence_after();
}
__device__ __forceinline__ void cta_sync_tc() {
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
}

// ---------------------------------------------------------------- stages
// A: DFT64 over t1 (pruned to t1 < 32), data = MN-major A operand from TMA
template <typename T>
__device__ __forceinline__ void mma_stage_A(const Ctx& c) {
  const uint32_t id = idesc<T>(128, 128, true, false);
  // K steps s: channel s / 2, rows t1 16 (s % 2) .. +15; with 16 data rows the
  // odd steps would only multiply zero padding
  const uint32_t step = g_rows == 32 ? 1 : 2;
#pragma unroll 1
  for (uint32_t s = 0; s < 4; s += step) {
    const uint64_t ad = tc::smem_desc(c.smb + c.in_off + s * 2048, 1024, tc::kSw128, 8192);
    const uint64_t bd = tc::smem_desc(c.smb + c.smat + MAT_FA + s * 32, 1024, tc::kSw128);
    tc::mma_bf16(c.tmem + c.tw, ad, bd, id, s);
  }
}
// B / B': DFT128 with the data as the B operand (MN-major [kg][8][64] in the
// slot's SOP, re plane then im plane 16 KB apart).  INV: conjugate block.
template <typename T, bool INV, bool W3>
__device__ __forceinline__ void mma_stage_B(const Ctx& c) {
  if constexpr (W3) {
    // planes: forward [-Xi | Xr | Xi], inverse [Zr | Zi | -Zr] (16 KB each)
    const uint32_t id = idesc<T>(128, 128, false, true, false);
    const uint32_t fr = c.smb + c.smat + MAT_FR, fi = c.smb + c.smat + MAT_FI;
    const uint32_t p0 = c.smb + c.sop, p1 = p0 + 16384;
    const uint32_t d = c.tmem + c.tw;
#pragma unroll
    for (uint32_t s = 0; s < 8; ++s) {
      const uint32_t ko = (s >> 2) * 16384 + (s & 3) * 32;
      const uint64_t dr = tc::smem_desc(fr + ko, 1024, tc::kSw128);
      const uint64_t di = tc::smem_desc(fi + ko, 1024, tc::kSw128);
      const uint64_t w0 = tc::smem_desc(p0 + s * 2048, 1024, tc::kSw128, 16384);
      const uint64_t w1 = tc::smem_desc(p1 + s * 2048, 1024, tc::kSw128, 16384);
      // forward: [re | im] += Fr [Xr | Xi] + Fi [-Xi | Xr]
      // inverse: [re | im] += Fr [Zr | Zi] + Fi [Zi | -Zr]
      tc::mma_bf16(d, dr, INV ? w0 : w1, id, s);
      tc::mma_bf16(d, di, INV ? w1 : w0, id, 1);
    }
    return;
  }
  const uint32_t id_p = idesc<T>(128, 64, false, true, false);
  const uint32_t id_n = idesc<T>(128, 64, false, true, true);
  const uint32_t fr = c.smb + c.smat + MAT_FR, fi = c.smb + c.smat + MAT_FI;
  const uint32_t br = c.smb + c.sop, bi = br + 16384;
  const uint32_t d = c.tmem + c.tw;
#pragma unroll
  for (uint32_t s = 0; s < 8; ++s) {
    const uint32_t ko = (s >> 2) * 16384 + (s & 3) * 32;
    const uint64_t dr = tc::smem_desc(fr + ko, 1024, tc::kSw128);
    const uint64_t di = tc::smem_desc(fi + ko, 1024, tc::kSw128);
    const uint64_t xr = tc::smem_desc(br + s * 2048, 1024, tc::kSw128, 1024);
    const uint64_t xi = tc::smem_desc(bi + s * 2048, 1024, tc::kSw128, 1024);
    if (!INV) {
      // re = Fr.Ar - Fi.Ai ; im = Fi.Ar + Fr.Ai
      tc::mma_bf16(d, dr, xr, id_p, s);
      tc::mma_bf16(d, di, xi, id_n, 1);
      tc::mma_bf16(d + 64, di, xr, id_p, s);
      tc::mma_bf16(d + 64, dr, xi, id_p, 1);
    } else {
      // conj(F) Z: re = Fr.Zr + Fi.Zi ; im = Fr.Zi - Fi.Zr
      tc::mma_bf16(d, dr, xr, id_p, s);
      tc::mma_bf16(d, di, xi, id_p, 1);
      tc::mma_bf16(d + 64, dr, xi, id_p, s);
      tc::mma_bf16(d + 64, di, xr, id_n, 1);
    }
  }
}
// A': IDFT64 over f1 to t1 < 32; the B operand is FA read MN-major (= the
// conj(F64) block transposed, see the smem map)
template <typename T>
__device__ __forceinline__ void mma_stage_Ap(const Ctx& c) {
  const uint32_t id = idesc<T>(128, 64, false, true);
#pragma unroll
  for (uint32_t s = 0; s < 8; ++s) {
    const uint64_t ad =
        tc::smem_desc(c.smb + c.sop + (s >> 2) * 16384 + (s & 3) * 32, 1024, tc::kSw128);
    const uint64_t bd = tc::smem_desc(c.smb + c.smat + MAT_FA + s * 2048, 1024, tc::kSw128, 1024);
    tc::mma_bf16(c.tmem + c.tw, ad, bd, id, s);
  }
}

// ---- three-pass rows (pass 2): full complex rows, no causal pruning.
// Stage-A block FA split in its two k-blocks around FR / FI, so the FR / FI
// offsets of the single-pass map still hold: [FA re-k | FR | FI | FA im-k].
namespace rows {
constexpr uint32_t SOP = 0;  // [slot] three 16 KB planes; the input row lands in planes 1-2
constexpr uint32_t SMAT = 2 * 49152;
constexpr uint32_t FA_KB1 = 81920, MAT_BYTES = 98304;
constexpr uint32_t STAB = SMAT + MAT_BYTES;
constexpr uint32_t SMEM = STAB + 1536;
// backward: Kf2 row as bf16 pairs [f2 128][f1 64], 16-byte chunks XOR-swizzled by f2 & 7
constexpr uint32_t SKF = SMEM;
constexpr uint32_t SMEM_BWD = SKF + 32768;
}  // namespace rows

// A (full): DFT64 over all t1; data = MN-major A operand [mb 2][kg 16][8][64]
// (kg 0-7 re plane, 8-15 im plane), K = 128
template <typename T>
__device__ __forceinline__ void mma_stage_A_full(const Ctx& c) {
  const uint32_t id = idesc<T>(128, 128, true, false);
#pragma unroll
  for (uint32_t s = 0; s < 8; ++s) {
    const uint64_t ad = tc::smem_desc(c.smb + c.in_off + s * 2048, 1024, tc::kSw128, 16384);
    const uint64_t bd =
        tc::smem_desc(c.smb + c.smat + (s >> 2) * rows::FA_KB1 + (s & 3) * 32, 1024, tc::kSw128);
    tc::mma_bf16(c.tmem + c.tw, ad, bd, id, s);
  }
}
// A' (full): IDFT64 over f1 to all t1 (N = 128: t1 re | t1 im, the two FA
// k-blocks read MN-major)
template <typename T>
__device__ __forceinline__ void mma_stage_Ap_full(const Ctx& c) {
  const uint32_t id = idesc<T>(128, 128, false, true);
#pragma unroll
  for (uint32_t s = 0; s < 8; ++s) {
    const uint64_t ad =
        tc::smem_desc(c.smb + c.sop + (s >> 2) * 16384 + (s & 3) * 32, 1024, tc::kSw128);
    const uint64_t bd = tc::smem_desc(c.smb + c.smat + s * 2048, 1024, tc::kSw128, rows::FA_KB1);
    tc::mma_bf16(c.tmem + c.tw, ad, bd, id, s);
  }
}

#ifdef FB_TC_TIMING
// experiment only: per (cta, slot, stage) cycle sums of epilogue / slot sync /
// MMA issue / MMA completion, read back through fb_debug_tc_timing()
__device__ unsigned long long g_tc_timing[148 * 2 * 32];
__device__ unsigned long long g_last[148 * 2];
#endif

// experiment: time a region into slot counter k (16..31)
#ifdef FB_TC_TIMING
#define TT_BEGIN unsigned long long _tt0 = clock64();
#define TT_END(k)                                                                        \
  if (slot_leader() && blockIdx.x < 148)                                                 \
    g_tc_timing[(blockIdx.x * 2 + (threadIdx.x / kSlotThreads)) * 32 + (k)] += clock64() - _tt0;
#else
#define TT_BEGIN
#define TT_END(k)
#endif

// No-op leader hook for issue()
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

// publish, MMA batch of `stage` by the slot leader, wait for it.  `hook`
// runs in the leader right after the commit, i.e. while the MMAs execute:
// work placed there (the next input's TMA) is off the slot's critical path.
template <typename T, bool W3 = false, class Hook = NoHook>
__device__ __forceinline__ void issue(Ctx& c, int stage, const Hook& hook = Hook()) {
#ifdef FB_TC_TIMING
  const bool tl = slot_leader() && blockIdx.x < 148;
  const uint32_t ts = (blockIdx.x * 2 + (threadIdx.x / kSlotThreads));
  const int sx = stage == 4 ? 0 : (stage == 5 ? 3 : stage);
  unsigned long long t0 = clock64();
  if (tl && g_last[ts]) g_tc_timing[ts * 32 + sx] += t0 - g_last[ts];
#endif
  publish(c);
#ifdef FB_TC_TIMING
  unsigned long long t1 = clock64();
  if (tl) g_tc_timing[ts * 32 + 4 + sx] += t1 - t0;
#endif
  if (slot_leader()) {
    const uint32_t j = c.nb - c.seg0;
    if (c.slot == 0) {
      if (j >= 1 && j - 1 < c.on) ptx::mbar_wait(c.other_bar, (c.obase + j - 1) & 1);
    } else if (j < c.on) {
      ptx::mbar_wait(c.other_bar, (c.obase + j) & 1);
    }
    if (c.lock)
      while (atomicCAS(c.lock, 0u, 1u) != 0u) {
      }
    switch (stage) {
      case 0: mma_stage_A<T>(c); break;
      case 1: mma_stage_B<T, false, W3>(c); break;
      case 2: mma_stage_B<T, true, W3>(c); break;
      case 3: mma_stage_Ap<T>(c); break;
      case 4: mma_stage_A_full<T>(c); break;
      default: mma_stage_Ap_full<T>(c); break;
    }
    tc::commit(c.mma_bar);
    if (c.lock) atomicExch(c.lock, 0u);
    hook();
  }
  ++c.nb;
#ifdef FB_TC_TIMING
  unsigned long long t2 = clock64();
  if (tl) g_tc_timing[ts * 32 + 8 + sx] += t2 - t1;
#endif
  mma_wait(c);
#ifdef FB_TC_TIMING
  unsigned long long t3 = clock64();
  if (tl) {
    g_tc_timing[ts * 32 + 12 + sx] += t3 - t2;
    g_last[ts] = t3;
  }
#endif
}

// (re[j], im[j]) *= w^((off + j) base), j = 0..15: two table lookups, then
// a rotation recurrence (16 steps: a few fp32 ulp, far below the bf16
// operand rounding that follows)
template <int SIGN>
__device__ __forceinline__ void twiddle_row(float* re, float* im, const float2* tab, uint32_t base,
                                            uint32_t off) {
  float2 w = tw2<SIGN>(tab, off * base);
  const float2 st = tw2<SIGN>(tab, base);
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const float a = re[j], b = im[j];
    re[j] = fmaf(a, w.x, -b * w.y);
    im[j] = fmaf(a, w.y, b * w.x);
    if (j < 15) w = cmul(w, st);
  }
}

// A exit: X[t2][f1] w^(f1 t2) -> stage-B operand (MN-major, k = t2, n = f1)
template <typename T, bool W3 = false>
__device__ __forceinline__ void epi_A_exit(const Ctx& c) {
  uint32_t t2, g;
  coords(t2, g);
  unsigned char* op = c.sm + c.sop;
  constexpr uint32_t Q = kColsPer / 16;
  float rr[Q][16], ii[Q][16];  // all of the thread's columns in flight, one wait
#pragma unroll
  for (uint32_t q = 0; q < Q; ++q) {
    tld<16>(taddr(c, c.tw + kColsPer * g + 16 * q), rr[q]);
    tld<16>(taddr(c, c.tw + 64 + kColsPer * g + 16 * q), ii[q]);
  }
  tc::ld_wait();
#pragma unroll
  for (uint32_t q = 0; q < Q; ++q) {
    const uint32_t cb = kColsPer * g + 16 * q;
    float* re = rr[q];
    float* im = ii[q];
    twiddle_row<-1>(re, im, c.tab, t2, cb);
    if constexpr (W3) {  // planes [-Xi | Xr | Xi]
      st8n<T>(op + off_bmn(cb, t2), im);
      st8n<T>(op + off_bmn(cb + 8, t2), im + 8);
      st8<T>(op + 16384 + off_bmn(cb, t2), re);
      st8<T>(op + 16384 + off_bmn(cb + 8, t2), re + 8);
      st8<T>(op + 32768 + off_bmn(cb, t2), im);
      st8<T>(op + 32768 + off_bmn(cb + 8, t2), im + 8);
    } else {
      st8<T>(op + off_bmn(cb, t2), re);
      st8<T>(op + off_bmn(cb + 8, t2), re + 8);
      st8<T>(op + 16384 + off_bmn(cb, t2), im);
      st8<T>(op + 16384 + off_bmn(cb + 8, t2), im + 8);
    }
  }
}

// B' exit: w^(-f1 t2) -> stage-A' operand (K-major rows t2, k = f1 re | im)
template <typename T>
__device__ __forceinline__ void epi_Bp_exit(const Ctx& c) {
  uint32_t t2, g;
  coords(t2, g);
  unsigned char* op = c.sm + c.sop;
  constexpr uint32_t Q = kColsPer / 16;
  float rr[Q][16], ii[Q][16];
#pragma unroll
  for (uint32_t q = 0; q < Q; ++q) {
    tld<16>(taddr(c, c.tw + kColsPer * g + 16 * q), rr[q]);
    tld<16>(taddr(c, c.tw + 64 + kColsPer * g + 16 * q), ii[q]);
  }
  tc::ld_wait();
#pragma unroll
  for (uint32_t q = 0; q < Q; ++q) {
    const uint32_t cb = kColsPer * g + 16 * q;
    float* re = rr[q];
    float* im = ii[q];
    twiddle_row<+1>(re, im, c.tab, t2, cb);
    st8<T>(op + off_kmaj(t2, cb, 16384), re);
    st8<T>(op + off_kmaj(t2, cb + 8, 16384), re + 8);
    st8<T>(op + off_kmaj(t2, 64 + cb, 16384), im);
    st8<T>(op + off_kmaj(t2, 64 + cb + 8, 16384), im + 8);
  }
}

// A' exit: rows t2, z[128 t1 + t2] for t1 = R g + j (re -> b0, im -> b1)
template <typename T>
__device__ __forceinline__ void store_rows(const Ctx& c, T* __restrict__ out, int b0, int B, int H,
                                           int h) {
  uint32_t t2, g;
  coords(t2, g);
  constexpr int R = 32 / kGroups;
  float re[R], im[R];
  tld<R>(taddr(c, c.tw + R * g), re);
  tld<R>(taddr(c, c.tw + 32 + R * g), im);
  tc::ld_wait();
  const uint32_t rows = g_rows, N = 128 * rows;
  if (R * g >= rows) return;  // beyond the data rows (N = 2048)
  T* o0 = out + ((size_t)b0 * H + h) * N + 128 * (R * g) + t2;
#pragma unroll
  for (int j = 0; j < R; ++j) o0[128 * j] = cvt<T>(re[j]);
  if (b0 + 1 < B) {
    T* o1 = out + ((size_t)(b0 + 1) * H + h) * N + 128 * (R * g) + t2;
#pragma unroll
    for (int j = 0; j < R; ++j) o1[128 * j] = cvt<T>(im[j]);
  }
}

__device__ __forceinline__ void setup(unsigned char* sm, uint32_t* tmem_slot, uint64_t* bars,
                                      int nbars, int nbars_slot, const uint4* __restrict__ mats,
                                      const float2* __restrict__ tab_g, uint32_t smat = SMAT,
                                      uint32_t stab = STAB, uint32_t mat_bytes = MAT_BYTES) {
  if (threadIdx.x < 32) tc::alloc<512>(tmem_slot);
  if (threadIdx.x == 0) {
    for (int i = 0; i < nbars; ++i) ptx::mbar_init(&bars[i], i < nbars - nbars_slot ? 1 : kSlotThreads);
    ptx::mbar_init(&g_setup_bar, 1);
    ptx::fence_barrier_init();
    // the DFT blocks (80-96 KB) as a few bulk copies: one L2 round trip
    // instead of a dependent load/store loop per thread (measured ~6 % of
    // the forward's samples there)
    ptx::mbar_arrive_expect_tx(&g_setup_bar, mat_bytes);
    for (uint32_t off = 0; off < mat_bytes; off += 16384)
      ptx::bulk_g2s(sm + smat + off, reinterpret_cast<const char*>(mats) + off,
                    mat_bytes - off < 16384 ? mat_bytes - off : 16384, &g_setup_bar);
  }
  float2* tab = reinterpret_cast<float2*>(sm + stab);
  for (uint32_t i = threadIdx.x; i < 192; i += kThreads) tab[i] = __ldg(tab_g + i);
  ptx::fence_proxy_async_smem();
  cta_sync_tc();
  ptx::mbar_wait(&g_setup_bar, 0);
}

__device__ __forceinline__ void teardown(uint32_t tmem) {
  cta_sync_tc();
  if (threadIdx.x < 32) tc::dealloc<512>(tmem);
}

// The CTA's contiguous share [i0, i1) of the B/2 x H (head-major) channel pairs
// Backward: shares start on even pair indices (heads hold an even number of
// pairs whenever B/2 is even), so each head segment splits evenly over the two
// slots and neither idles a whole pair at the segment barrier.  CTA c starts
// at 2 floor(c U / G), U = ceil(total / 2) (mirrored by the finalize).
__device__ __forceinline__ void cta_range_even(int total, int& i0, int& i1) {
  const int64_t U = (total + 1) / 2;
  i0 = min(total, (int)(2 * ((int64_t)blockIdx.x * U / gridDim.x)));
  i1 = min(total, (int)(2 * ((int64_t)(blockIdx.x + 1) * U / gridDim.x)));
}
__device__ __forceinline__ void cta_range(int total, int& i0, int& i1) {
  i0 = (int)(((int64_t)blockIdx.x * total) / gridDim.x);
  i1 = (int)(((int64_t)(blockIdx.x + 1) * total) / gridDim.x);
}

__device__ __forceinline__ uint32_t pack_bf2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float2 unpack_bf2(uint32_t v) {
  return __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&v));
}
// ------------------------------------------------------------------ forward
// Persistent: CTA c owns pairs [i0, i1) in head-major order; slot s takes
// i0 + s, i0 + s + 2, ...
// TMEM (512 columns): slot s works in [128 s, 128 s + 128); its head's k_f'
// sits as raw fp16 pairs (the K1 image, scaled by 2^e, one column per f1) at
// TKF16 + 64 s; the stage-boundary twiddles w_8192^(f1 t2) are a fp32 table
// at TTW (re f1 0..63 | im f1 0..63, lane = t2) written once per CTA, so the
// A and B' exits cost one complex multiply per element (no recurrence, no
// table arithmetic), and the per-head scale 1/2^e is folded into the store.
constexpr uint32_t TKF16 = 256, TTW = 384;

// the twiddle table, written by slot 0 (a thread: lane t2, its 32 f1) with
// exactly the values twiddle_row's recurrence produces (chunks of 16 from a
// table start), so the backward's recomputed transforms stay bit-identical
__device__ __forceinline__ void init_tw_tmem(const Ctx& c) {
  uint32_t t2, g;
  coords(t2, g);
  const float2 st = tw2<-1>(c.tab, t2);
#pragma unroll
  for (uint32_t q = 0; q < kColsPer / 16; ++q) {
    const uint32_t cb = kColsPer * g + 16 * q;
    float re[16], im[16];
    float2 w = tw2<-1>(c.tab, cb * t2);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      re[j] = w.x;
      im[j] = w.y;
      if (j < 15) w = cmul(w, st);
    }
    tst8(taddr(c, TTW + cb), re);
    tst8(taddr(c, TTW + cb + 8), re + 8);
    tst8(taddr(c, TTW + 64 + cb), im);
    tst8(taddr(c, TTW + 64 + cb + 8), im + 8);
  }
  tst_wait();
}

// k_f' of head h as raw fp16 pairs: column f1, lane f2
__device__ __forceinline__ void load_kf16_tmem(const Ctx& c, const __half2* __restrict__ kf) {
  uint32_t f2, g;
  coords(f2, g);
  const uint32_t* src = reinterpret_cast<const uint32_t*>(kf) + f2;
#pragma unroll
  for (uint32_t q = 0; q < kColsPer / 8; ++q) {
    const uint32_t cb = kColsPer * g + 8 * q;
    uint32_t v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldg(src + (cb + j) * 128);
    tst8(taddr(c, c.aux + cb), reinterpret_cast<const float*>(v));
  }
  tst_wait();
}

// A exit from the TMEM twiddles: X[t2][f1] w^(f1 t2) -> planes [-Xi | Xr | Xi]
template <typename T>
__device__ __forceinline__ void epi_A_exit_tw(const Ctx& c) {
#ifdef FB_TC_NOEPI
  return;
#endif
  uint32_t t2, g;
  coords(t2, g);
  unsigned char* op = c.sm + c.sop;
#pragma unroll
  for (uint32_t q = 0; q < kColsPer / 8; ++q) {
    const uint32_t cb = kColsPer * g + 8 * q;
    float re[8], im[8], wr[8], wi[8];
    tld<8>(taddr(c, c.tw + cb), re);
    tld<8>(taddr(c, c.tw + 64 + cb), im);
    tld<8>(taddr(c, TTW + cb), wr);
    tld<8>(taddr(c, TTW + 64 + cb), wi);
    tc::ld_wait();
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float a = re[j], b = im[j];
      re[j] = fmaf(a, wr[j], -b * wi[j]);
      im[j] = fmaf(a, wi[j], b * wr[j]);
    }
    st8n<T>(op + off_bmn(cb, t2), im);
    st8<T>(op + 16384 + off_bmn(cb, t2), re);
    st8<T>(op + 32768 + off_bmn(cb, t2), im);
  }
}

// B' exit from the TMEM twiddles: w^(-f1 t2) -> stage-A' operand (K-major)
template <typename T>
__device__ __forceinline__ void epi_Bp_exit_tw(const Ctx& c) {
#ifdef FB_TC_NOEPI
  return;
#endif
  uint32_t t2, g;
  coords(t2, g);
  unsigned char* op = c.sm + c.sop;
#pragma unroll
  for (uint32_t q = 0; q < kColsPer / 8; ++q) {
    const uint32_t cb = kColsPer * g + 8 * q;
    float re[8], im[8], wr[8], wi[8];
    tld<8>(taddr(c, c.tw + cb), re);
    tld<8>(taddr(c, c.tw + 64 + cb), im);
    tld<8>(taddr(c, TTW + cb), wr);
    tld<8>(taddr(c, TTW + 64 + cb), wi);
    tc::ld_wait();
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float a = re[j], b = im[j];
      re[j] = fmaf(a, wr[j], b * wi[j]);  // twiddle_row<+1>'s rounding
      im[j] = fmaf(a, -wi[j], b * wr[j]);
    }
    st8<T>(op + off_kmaj(t2, cb, 16384), re);
    st8<T>(op + off_kmaj(t2, 64 + cb, 16384), im);
  }
}

// A' exit with the head's k_f' scale folded in: z[128 t1 + t2], t1 = R g + j
template <typename T>
__device__ __forceinline__ void store_rows_sc(const Ctx& c, T* __restrict__ out, int b0, int B,
                                              int H, int h, float sc) {
#ifdef FB_TC_NOEPI
  return;
#endif
  uint32_t t2, g;
  coords(t2, g);
  constexpr int R = 32 / kGroups;
  float re[R], im[R];
  tld<R>(taddr(c, c.tw + R * g), re);
  tld<R>(taddr(c, c.tw + 32 + R * g), im);
  tc::ld_wait();
  const uint32_t rows = g_rows, N = 128 * rows;
  if (R * g >= rows) return;  // beyond the data rows (N = 2048)
  T* o0 = out + ((size_t)b0 * H + h) * N + 128 * (R * g) + t2;
#pragma unroll
  for (int j = 0; j < R; ++j) o0[128 * j] = cvt<T>(re[j] * sc);
  if (b0 + 1 < B) {
    T* o1 = out + ((size_t)(b0 + 1) * H + h) * N + 128 * (R * g) + t2;
#pragma unroll
    for (int j = 0; j < R; ++j) o1[128 * j] = cvt<T>(im[j] * sc);
  }
}

// saved U layout: bf16 pairs [pair][f1 / 4][f2][f1 % 4] — a thread's four
// consecutive f1 are one 16-byte store / load, a warp's 32 lanes (f2) 512
// contiguous bytes
__host__ __device__ __forceinline__ uint32_t usave_idx(uint32_t f1, uint32_t f2) {
  return ((f1 >> 2) * 128 + f2) * 4 + (f1 & 3);
}

template <typename T>
__global__ void __launch_bounds__(kThreads, 1)
    tc_fwd_kernel(const __grid_constant__ CUtensorMap umap, T* __restrict__ y,
                  const __half2* __restrict__ kf16, const float* __restrict__ kscale,
                  const uint4* __restrict__ mats, const float2* __restrict__ tab_g, int B, int H,
                  int total, uint32_t* __restrict__ usave, int sched, int rows) {
  // bf16 planes take the scaled product (k_f' x 2^e, e <= ~30) and the
  // store undoes the scale; fp16 planes need it applied at the B exit
  constexpr bool kScaleEarly = std::is_same<T, __half>::value;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bars[4];  // mma[2], in[2]
  __shared__ uint32_t mma_lock;
  unsigned char* sm = smem_base(smem_raw);
  const int npairs = (B + 1) / 2;
  int i0, i1;
  cta_range(total, i0, i1);
  if (threadIdx.x == 0) {
    mma_lock = 0;
    g_rows = (uint32_t)rows;
  }
  setup(sm, &tmem_slot, bars, 4, 0, mats, tab_g, SMAT3, STAB3);
  const uint32_t slot = threadIdx.x / kSlotThreads;
  Ctx c = make_ctx(sm, tmem_slot, slot, &bars[slot], true);
  c.aux = TKF16 + 64 * slot;
  if (slot == 0) init_tw_tmem(c);
  cta_sync_tc();
  if (sched == 1) c.lock = &mma_lock;
  else c.on = 4u * (uint32_t)((i1 - i0 + (int)slot) / 2);  // token: the other slot's pairs x 4 stages
  uint64_t* in_bar = &bars[2 + slot];
  const bool lead = slot_leader();
  int item = i0 + (int)slot;
  if (lead && item < i1) load_pair(sm + c.in_off, &umap, item / npairs, 2 * (item % npairs), in_bar);
  int cur_h = -1;
  float sc = 1.f;
  for (uint32_t it = 0; item < i1; item += 2, ++it) {
    const int h = item / npairs, pr = item % npairs;
    if (h != cur_h) {
      { TT_BEGIN load_kf16_tmem(c, kf16 + (size_t)h * kN); TT_END(17) }
      sc = __ldg(kscale + h);
      cur_h = h;
    }
    { TT_BEGIN ptx::mbar_wait(in_bar, it & 1); TT_END(16) }
    issue<T, true>(c, 0);
    { TT_BEGIN epi_A_exit_tw<T>(c); TT_END(18) }
    // the input buffer is free since stage A completed: the next pair's TMA
    // goes out from the leader while the stage-B MMAs run
    issue<T, true>(c, 1, [&] {
      if (item + 2 < i1)
        load_pair(sm + c.in_off, &umap, (item + 2) / npairs, 2 * ((item + 2) % npairs), in_bar);
    });
    // ---- B exit: Z = X * k_f' (unscaled; the scale is folded into the store)
#ifndef FB_TC_NOEPI
    {
      TT_BEGIN
      uint32_t f2, g;
      coords(f2, g);
      unsigned char* op = c.sm + c.sop;
#pragma unroll
      for (uint32_t q = 0; q < kColsPer / 8; ++q) {
        const uint32_t cb = kColsPer * g + 8 * q;
        float re[8], im[8], kk[8];
        tld<8>(taddr(c, c.tw + cb), re);
        tld<8>(taddr(c, c.tw + 64 + cb), im);
        tld<8>(taddr(c, c.aux + cb), kk);
        tc::ld_wait();
        if (usave) {  // U = F(u) for the backward, bf16 pairs (usave_idx layout)
          uint4* us = reinterpret_cast<uint4*>(usave + (size_t)item * kN + usave_idx(cb, f2));
          us[0] = make_uint4(pack_bf2(re[0], im[0]), pack_bf2(re[1], im[1]), pack_bf2(re[2], im[2]),
                             pack_bf2(re[3], im[3]));
          us[128] = make_uint4(pack_bf2(re[4], im[4]), pack_bf2(re[5], im[5]),
                               pack_bf2(re[6], im[6]), pack_bf2(re[7], im[7]));
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float2 k = __half22float2(*reinterpret_cast<const __half2*>(&kk[j]));
          if constexpr (kScaleEarly) {  // fp16 planes: keep Z in the operand range
            k.x *= sc;
            k.y *= sc;
          }
          const float a = re[j], b = im[j];
          re[j] = fmaf(a, k.x, -b * k.y);
          im[j] = fmaf(a, k.y, b * k.x);
        }
        st8<T>(op + off_bmn(cb, f2), re);  // planes [Zr | Zi | -Zr]
        st8<T>(op + 16384 + off_bmn(cb, f2), im);
        st8n<T>(op + 32768 + off_bmn(cb, f2), re);
      }
      TT_END(19)
    }
#endif
    issue<T, true>(c, 2);
    { TT_BEGIN epi_Bp_exit_tw<T>(c); TT_END(20) }
    issue<T, true>(c, 3);
    { TT_BEGIN store_rows_sc<T>(c, y, 2 * pr, B, H, h, kScaleEarly ? 1.f : sc); TT_END(21) }
  }
  teardown(tmem_slot);
}

// ------------------------------------------------------------------ backward
// Persistent like the forward.  The CTA walks its pairs head segment by head
// segment; inside a segment slot s takes local pairs s, s+2, ...  Per pair:
// DY = F(dy); S += conj(U) DY (S = the CTA's dK spectrum, fp32 in TMEM,
// updated strictly in pair order across the slots through two mbarriers so
// the sum is deterministic) and du = F^-1(DY conj(k_f')).  U = F(u) comes
// from the forward's saved transform (SAVED) or is computed here first and
// parked in the workspace (same layout, same values).  At a segment end slot 0
// transforms S back on the tensor cores (B', A': the causal lags t < N,
// real part) into a time-domain partial tpart[cta][seg][t]; tc_dk_tail sums
// a head's partials in a fixed order and applies the regularizer chain rule.
// TMEM: slot s works in [128 s, 128 s + 128); S at TS2 (re f1 | im f1); the
// forward's twiddle table at TTW.
constexpr uint32_t TS2 = 256;

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ptx::smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// A' exit of the S inverse: Re of the lags t = 128 t1 + t2 (t1 < 32), scaled
__device__ __forceinline__ void store_tpart(const Ctx& c, float* __restrict__ dst, float sc) {
  uint32_t t2, g;
  coords(t2, g);
  constexpr int R = 32 / kGroups;
  float re[R];
  tld<R>(taddr(c, c.tw + R * g), re);
  tc::ld_wait();
  float* o = dst + 128 * (R * g) + t2;
#pragma unroll
  for (int j = 0; j < R; ++j) o[128 * j] = re[j] * sc;
}

// SAVED: U comes from the forward's usave (bf16 pairs, usave_idx layout)
// instead of F(u): one transform per pair fewer.
template <typename T, bool SAVED>
__global__ void __launch_bounds__(kThreads, 1)
    tc_bwd_kernel(const __grid_constant__ CUtensorMap dymap, const __grid_constant__ CUtensorMap umap,
                  T* __restrict__ du, const __half2* __restrict__ kf16,
                  const float* __restrict__ kscale, const uint4* __restrict__ mats,
                  const float2* __restrict__ tab_g, float* __restrict__ tpart, int B, int H,
                  int total, int maxseg, const uint32_t* __restrict__ usave,
                  uint32_t* __restrict__ uscratch, int sched, int rows) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bars[6];  // mma[2], in[2], S chain[2] (256 arrivals)
  __shared__ uint32_t mma_lock;
  __shared__ float red[8];
  unsigned char* sm = smem_base(smem_raw);
  const int npairs = (B + 1) / 2;
  int i0, i1;
  cta_range_even(total, i0, i1);
  if (threadIdx.x == 0) {
    mma_lock = 0;
    g_rows = (uint32_t)rows;
  }
  setup(sm, &tmem_slot, bars, 6, 2, mats, tab_g, SMAT3, STAB3);
  const uint32_t slot = threadIdx.x / kSlotThreads;
  Ctx c = make_ctx(sm, tmem_slot, slot, &bars[slot], true);
  if (slot == 0) init_tw_tmem(c);
  cta_sync_tc();
  if (sched == 1) c.lock = &mma_lock;
  uint64_t* in_bar = &bars[2 + slot];
  uint64_t* chain_mine = &bars[4 + slot];
  uint64_t* chain_other = &bars[5 - slot];
  const bool lead = slot_leader();
  const uint32_t* kfs = reinterpret_cast<const uint32_t*>(sm + SKF3);
  const uint32_t* ubase = SAVED ? usave : uscratch;
  uint32_t in_cnt = 0, base0 = 0, base1 = 0;
  int seg = 0;
  for (int a = i0; a < i1; ++seg) {
    const int h = a / npairs;
    const int L = min(i1, (h + 1) * npairs) - a;
    // ---- segment start (whole CTA): k_f' of head h to smem, S = 0
    {
      TT_BEGIN
      const uint32_t* src = reinterpret_cast<const uint32_t*>(kf16 + (size_t)h * kN);
      uint32_t* dst = reinterpret_cast<uint32_t*>(sm + SKF3);
      // all of the gather in flight at once (4-byte cp.async), not one
      // dependent global round trip per element
      for (uint32_t i = threadIdx.x; i < 64 * KFH_ROW; i += kThreads)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(ptx::smem_u32(dst + i)),
                     "l"(static_cast<uint64_t>(
                         __cvta_generic_to_global(src + (i / KFH_ROW) * 128 + i % KFH_ROW)))
                     : "memory");
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
      const uint32_t t = threadIdx.x;
      constexpr uint32_t W = 64 / (kThreads / 128);  // columns per thread
      const uint32_t lane_off = (32u * ((t >> 5) & 3)) << 16, g8 = t >> 7;
      float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (uint32_t q = 0; q < W / 8; ++q) {
        tst8(tmem_slot + lane_off + TS2 + W * g8 + 8 * q, z);
        tst8(tmem_slot + lane_off + TS2 + 64 + W * g8 + 8 * q, z);
      }
      tst_wait();
      cta_sync_tc();
      TT_END(30)
    }
    const float osc = __ldg(kscale + h);
    // the MMA token measured slower here than free interleaving (the backward's
    // epilogues are longer than its MMA batches): c.on stays 0, no waits
    c.seg0 = c.nb;
    if (lead && (int)slot < L) {
      const int it = a + (int)slot;
      load_pair(sm + c.in_off, SAVED ? &dymap : &umap, h, 2 * (it - h * npairs), in_bar);
    }
    for (int j = (int)slot, k = 0; j < L; j += 2, ++k) {
      const int b0 = 2 * (a + j - h * npairs);
      const uint32_t* up = ubase + (size_t)(a + j) * kN;
      if constexpr (SAVED) {
        if (lead) prefetch_l2(up, kN * sizeof(uint32_t));  // read back in the S epilogue
      } else {
        // ---- U = F(u), parked in the workspace (the saved layout)
        { TT_BEGIN ptx::mbar_wait(in_bar, in_cnt & 1); TT_END(22) }
        ++in_cnt;
        issue<T, true>(c, 0);
        { TT_BEGIN epi_A_exit_tw<T>(c); TT_END(25) }
        issue<T, true>(c, 1, [&] { load_pair(sm + c.in_off, &dymap, h, b0, in_bar); });
        uint32_t f2, g;
        coords(f2, g);
#pragma unroll
        for (uint32_t q = 0; q < kColsPer / 8; ++q) {
          const uint32_t cb = kColsPer * g + 8 * q;
          float re[8], im[8];
          tld<8>(taddr(c, c.tw + cb), re);
          tld<8>(taddr(c, c.tw + 64 + cb), im);
          tc::ld_wait();
          uint4* us = reinterpret_cast<uint4*>(uscratch + (size_t)(a + j) * kN + usave_idx(cb, f2));
          us[0] = make_uint4(pack_bf2(re[0], im[0]), pack_bf2(re[1], im[1]), pack_bf2(re[2], im[2]),
                             pack_bf2(re[3], im[3]));
          us[128] = make_uint4(pack_bf2(re[4], im[4]), pack_bf2(re[5], im[5]),
                               pack_bf2(re[6], im[6]), pack_bf2(re[7], im[7]));
        }
      }
      // ---- DY = F(dy)
      { TT_BEGIN ptx::mbar_wait(in_bar, in_cnt & 1); TT_END(23) }
      ++in_cnt;
      issue<T, true>(c, 0);
      { TT_BEGIN epi_A_exit_tw<T>(c); TT_END(25) }
      issue<T, true>(c, 1, [&] {  // next pair's first input, off the critical path
        if (j + 2 < L) load_pair(sm + c.in_off, SAVED ? &dymap : &umap, h, b0 + 4, in_bar);
      });
      // ---- S += conj(U) DY (in pair order), Z = DY conj(k_f') -> B' operand
      // this thread's U values (L2: prefetched at the pair start), software-
      // pipelined one column chunk ahead: the first chunk's loads are in
      // flight across the chain wait, each later one across the previous
      // chunk's math, instead of one exposed L2 round trip per chunk
      uint4 ua_n, ub_n;
      {
        uint32_t f2u, gu;
        coords(f2u, gu);
        const uint4* us = reinterpret_cast<const uint4*>(up + usave_idx(kColsPer * gu, f2u));
        ua_n = __ldcg(us);
        ub_n = __ldcg(us + 128);
      }
      if (j > 0) {
        const uint32_t idx = slot ? base0 + (uint32_t)k : base1 + (uint32_t)k - 1;
        TT_BEGIN ptx::mbar_wait(chain_other, idx & 1); TT_END(24)
        tc::fence_after();
      }
      {
        uint32_t f2, g;
        coords(f2, g);
        unsigned char* op = c.sm + c.sop;
#pragma unroll 1
        for (uint32_t q = 0; q < kColsPer / 8; ++q) {
          const uint32_t col = kColsPer * g + 8 * q;
          float dr[8], di[8], sr[8], si[8];
          // (L2 loads, .cg: the recompute path wrote U moments ago in this kernel)
          const uint4 ua = ua_n, ub = ub_n;
          if (q + 1 < kColsPer / 8) {
            const uint4* us = reinterpret_cast<const uint4*>(up + usave_idx(col + 8, f2));
            ua_n = __ldcg(us);
            ub_n = __ldcg(us + 128);
          }
          const uint32_t pk[8] = {ua.x, ua.y, ua.z, ua.w, ub.x, ub.y, ub.z, ub.w};
          tld<8>(taddr(c, c.tw + col), dr);
          tld<8>(taddr(c, c.tw + 64 + col), di);
          tld<8>(taddr(c, TS2 + col), sr);
          tld<8>(taddr(c, TS2 + 64 + col), si);
          tc::ld_wait();
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const float2 u = unpack_bf2(pk[jj]);
            sr[jj] = fmaf(u.x, dr[jj], fmaf(u.y, di[jj], sr[jj]));
            si[jj] = fmaf(u.x, di[jj], fmaf(-u.y, dr[jj], si[jj]));
            // k_f'[f1 + 64 f2]; upper half (f2 >= 64) by conjugate symmetry
            const uint32_t f1 = col + jj;
            const bool upper = f2 >= 64;
            const uint32_t idx = !upper ? f1 * KFH_ROW + f2
                                        : (f1 ? (64 - f1) * KFH_ROW + (127 - f2) : 128 - f2);
            float2 kv = __half22float2(*reinterpret_cast<const __half2*>(&kfs[idx]));
            kv.x *= osc;
            kv.y *= upper ? -osc : osc;
            const float a0 = dr[jj], b = di[jj];
            dr[jj] = fmaf(a0, kv.x, b * kv.y);
            di[jj] = fmaf(b, kv.x, -a0 * kv.y);
          }
          tst8(taddr(c, TS2 + col), sr);
          tst8(taddr(c, TS2 + 64 + col), si);
          st8<T>(op + off_bmn(col, f2), dr);  // planes [Zr | Zi | -Zr]
          st8<T>(op + 16384 + off_bmn(col, f2), di);
          st8n<T>(op + 32768 + off_bmn(col, f2), dr);
        }
        tst_wait();
        tc::fence_before();
        mbar_arrive(chain_mine);
      }
      issue<T, true>(c, 2);
      { TT_BEGIN epi_Bp_exit_tw<T>(c); TT_END(28) }
      issue<T, true>(c, 3);
      { TT_BEGIN store_rows<T>(c, du, b0, B, H, h); TT_END(29) }
    }
    base0 += (uint32_t)(L + 1) / 2;
    base1 += (uint32_t)L / 2;
    // ---- segment end: slot 0 inverts S on the tensor cores (B', A') into the
    // time-domain partial tpart[cta][seg] (Re, lags t < N, x 1/n)
    { TT_BEGIN cta_sync_tc(); TT_END(31) }
    float ssc = 1.f;
    if (slot == 0) {
      uint32_t f2, g;
      coords(f2, g);
      // fp16 operands need S brought into range: a power-of-two scale from
      // the segment's max |S| (bf16 has fp32's exponent range: scale 1)
      if constexpr (std::is_same<T, __half>::value) {
        float mx = 0.f;
#pragma unroll
        for (uint32_t q = 0; q < kColsPer / 8; ++q) {
          float sr[8], si[8];
          tld<8>(taddr(c, TS2 + kColsPer * g + 8 * q), sr);
          tld<8>(taddr(c, TS2 + 64 + kColsPer * g + 8 * q), si);
          tc::ld_wait();
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) mx = fmaxf(mx, fmaxf(fabsf(sr[jj]), fabsf(si[jj])));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
        slot_sync(c);
        mx = red[0];
#pragma unroll
        for (int w = 1; w < 8; ++w) mx = fmaxf(mx, red[w]);
        int e = 0;
        if (mx > 0.f) frexpf(mx, &e);
        // max |S| -> [2^7, 2^8): the B' exit's 128-term sums stay below 2^15
        ssc = mx > 0.f ? ldexpf(1.f, 8 - e) : 1.f;
      }
      unsigned char* op = c.sm + c.sop;
#pragma unroll
      for (uint32_t q = 0; q < kColsPer / 8; ++q) {
        const uint32_t col = kColsPer * g + 8 * q;
        float sr[8], si[8];
        tld<8>(taddr(c, TS2 + col), sr);
        tld<8>(taddr(c, TS2 + 64 + col), si);
        tc::ld_wait();
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          sr[jj] *= ssc;
          si[jj] *= ssc;
        }
        st8<T>(op + off_bmn(col, f2), sr);  // planes [Zr | Zi | -Zr]
        st8<T>(op + 16384 + off_bmn(col, f2), si);
        st8n<T>(op + 32768 + off_bmn(col, f2), sr);
      }
    }
    // S has been read: slot 1 may start the next segment (k_f' load, S = 0)
    // while slot 0 finishes the inverse
    cta_sync_tc();
    if (slot == 0) {
      issue<T, true>(c, 2);
      epi_Bp_exit_tw<T>(c);
      issue<T, true>(c, 3);
      store_tpart(c, tpart + ((size_t)blockIdx.x * maxseg + seg) * 4096,
                  1.f / (ssc * (float)kN));
    }
    a += L;
  }
  teardown(tmem_slot);
}

// dKbar[h] = sum of the head's time-domain partials (CTA order, fixed), dD =
// dKbar[0] (lag 0), dK = the regularizer chain rule (fp64 tap sums in the
// reference order) — the tail of the tensor-core backward
template <uint32_t N>
__global__ void __launch_bounds__(512)
    tc_dk_tail_kernel(const float* __restrict__ tpart, float* __restrict__ dkbar_out,
                      float* __restrict__ dD, const float* __restrict__ kbar,
                      const uint8_t* __restrict__ keep, float* __restrict__ dK, int64_t p,
                      double keep_scale, int freq, int ctas, int total, int npairs, int maxseg) {
  // 512 threads x kPer consecutive lags; partial rows hold lags 0..4095
  constexpr uint32_t kPer = N / 512, kPitch = 4096;
  static_assert(kPer == 8 || kPer == 4, "N = 4096 or 2048");
  __shared__ float row[N];
  __shared__ const float* src[8];
  __shared__ int s_c0, s_nc;
  const int h = blockIdx.x;
  const int64_t G = ctas, T = total, np = npairs;
  const int64_t U = (T + 1) / 2;
  // the CTA owning pair i under the backward's even-aligned shares (64-bit
  // divisions: once per CTA, not per thread)
  auto owner = [&](int64_t i) { return (int)((((i / 2) + 1) * G - 1) / U); };
  auto part = [&](int c) {  // CTA c's partial row of head h (segment h - its first head)
    const int64_t start = 2 * ((int64_t)c * U / G);
    return tpart + ((size_t)c * maxseg + (h - (int)(start / np))) * kPitch;
  };
  if (threadIdx.x == 0) {
    s_c0 = owner((int64_t)h * np);
    s_nc = owner(((int64_t)h + 1) * np - 1) - s_c0 + 1;
  }
  __syncthreads();
  const int c0 = s_c0, nc = s_nc;
  if (threadIdx.x < (unsigned)min(nc, 8)) src[threadIdx.x] = part(c0 + (int)threadIdx.x);
  __syncthreads();
  const size_t base = (size_t)h * N;
  const uint32_t t0 = threadIdx.x * kPer;
  // sum the partials in CTA order (deterministic), 16-byte loads
  constexpr uint32_t V = kPer / 4;
  float4 gv[V];
#pragma unroll
  for (uint32_t v = 0; v < V; ++v) gv[v] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int c = 0; c < nc; ++c) {
    const float4* sp = reinterpret_cast<const float4*>((c < 8 ? src[c] : part(c0 + c)) + t0);
#pragma unroll
    for (uint32_t v = 0; v < V; ++v) {
      const float4 a = __ldg(sp + v);
      gv[v].x += a.x; gv[v].y += a.y; gv[v].z += a.z; gv[v].w += a.w;
    }
  }
  if (dkbar_out)
#pragma unroll
    for (uint32_t v = 0; v < V; ++v) reinterpret_cast<float4*>(dkbar_out + base + t0)[v] = gv[v];
  if (threadIdx.x == 0) dD[h] = gv[0].x;
  {
#pragma unroll
    for (uint32_t v = 0; v < V; ++v) {
      const float4 k4 = __ldg(reinterpret_cast<const float4*>(kbar + base + t0) + v);
      const float kb[4] = {k4.x, k4.y, k4.z, k4.w}, g[4] = {gv[v].x, gv[v].y, gv[v].z, gv[v].w};
#pragma unroll
      for (uint32_t j = 0; j < 4; ++j) row[t0 + 4 * v + j] = (!freq && kb[j] == 0.f) ? 0.f : g[j];
    }
  }
  __syncthreads();
  if (!freq) {
    const double inv_w = 1.0 / (double)(2 * p + 1);
    const int pp = (int)p;
    float o[kPer];
#pragma unroll
    for (uint32_t j = 0; j < kPer; ++j) {
      const int t = (int)(t0 + j);
      const int lo = t >= pp ? t - pp : 0;
      const int hi = (t + pp < (int)N - 1) ? t + pp : (int)N - 1;
      double acc = 0.0;
      for (int q = lo; q <= hi; ++q) acc += (double)row[q];
      double gg = acc * inv_w;
      if (keep) gg = keep[base + t] ? gg * keep_scale : 0.0;
      o[j] = (float)gg;
    }
#pragma unroll
    for (uint32_t v = 0; v < kPer / 4; ++v)
      reinterpret_cast<float4*>(dK + base + t0)[v] = make_float4(o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
  } else {
    for (uint32_t t = threadIdx.x; t < N; t += blockDim.x)
      dK[base + t] = reg_grad(kbar + base, row, keep ? keep + base : nullptr, t, N, p, keep_scale,
                              freq);
  }
}

// ------------------------------------------------------------------ three-pass rows
// Pass 2 of the three-pass engine (fb_three.cu, middle_block of
// three_pass.cpp:211-221) on the tensor cores: row X1[(pr H + h) m + a] is a
// full complex length-8192 cyclic convolution W = IFFT(FFT(x) Kf2[h][a]) —
// the single-pass Monarch without the causal pruning (stage A K = 128, stage
// A' N = 128).  The row arrives planar ([re 8192 | im 8192] 16-bit, pass 1
// writes it so) by TMA straight into stage A's MN-major operand in the slot's
// operand planes 1-2 (dead until the A exit); W leaves interleaved (re, im)
// in place for pass 3; U = FFT(x) (natural order f = f1 + 64 f2) is kept for
// the backward.  Items run (h a)-major, pairs inner, so a slot reloads its
// Kf2 row (fp32, into TMEM) once per npairs / 2 rows.
__device__ __forceinline__ void load_row(unsigned char* dst, const CUtensorMap* map, int row,
                                         uint64_t* bar) {
  ptx::mbar_arrive_expect_tx(bar, 32768);
#pragma unroll
  for (int mb = 0; mb < 2; ++mb) tma_load_4d(dst + mb * 16384, map, mb * 64, 0, 0, row, bar);
}

__device__ __forceinline__ void load_kf_rows(const Ctx& c, const float2* __restrict__ kf) {
  uint32_t f2, g;
  coords(f2, g);
#pragma unroll
  for (uint32_t q = 0; q < kColsPer / 16; ++q) {
    const uint32_t cb = kColsPer * g + 16 * q;
    const float4* src = reinterpret_cast<const float4*>(kf + 64 * f2 + cb);
    float re[16], im[16];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 v = __ldg(src + j);
      re[2 * j] = v.x;
      im[2 * j] = v.y;
      re[2 * j + 1] = v.z;
      im[2 * j + 1] = v.w;
    }
    tst8(taddr(c, c.aux + cb), re);
    tst8(taddr(c, c.aux + cb + 8), re + 8);
    tst8(taddr(c, c.aux + 64 + cb), im);
    tst8(taddr(c, c.aux + 64 + cb + 8), im + 8);
  }
  tst_wait();
}

// SPEC: spectrum only (U = FFT(x) to usave, which may alias x1: the row is
// in smem before its spectrum is written) — the backward's recompute path.
template <typename T, bool SPEC = false>
__global__ void __launch_bounds__(kThreads, 1)
    tc_rows_fwd_kernel(const __grid_constant__ CUtensorMap xmap, uint32_t* __restrict__ x1,
                       const float2* __restrict__ kf2, const uint4* __restrict__ mats,
                       const float2* __restrict__ tab_g, int npairs, int hm, int total,
                       uint32_t* __restrict__ usave, int token) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bars[4];  // mma[2], in[2]
  unsigned char* sm = smem_base(smem_raw);
  int i0, i1;
  cta_range(total, i0, i1);
  setup(sm, &tmem_slot, bars, 4, 0, mats, tab_g, rows::SMAT, rows::STAB, rows::MAT_BYTES);
  const uint32_t slot = threadIdx.x / kSlotThreads;
  Ctx c = make_ctx(sm, tmem_slot, slot, &bars[slot], true);
  c.sop = rows::SOP + 49152 * slot;
  c.in_off = c.sop + 16384;
  c.smat = rows::SMAT;
  c.tab = reinterpret_cast<const float2*>(sm + rows::STAB);
  c.aux = TKF + 128 * slot;
  c.on = token ? (SPEC ? 2u : 4u) * (uint32_t)((i1 - i0 + (int)slot) / 2) : 0u;
  if (threadIdx.x == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
  uint64_t* in_bar = &bars[2 + slot];
  const bool lead = slot_leader();
  auto row_of = [&](int item) { return (item % npairs) * hm + item / npairs; };
  int item = i0 + (int)slot;
  if (lead && item < i1) load_row(sm + c.in_off, &xmap, row_of(item), in_bar);
  int cur = -1;
  for (uint32_t it = 0; item < i1; item += 2, ++it) {
    const int ha = item / npairs;
    const size_t row = (size_t)row_of(item);
    if (!SPEC && ha != cur) {
      TT_BEGIN
      load_kf_rows(c, kf2 + (size_t)ha * kN);
      TT_END(17)
      cur = ha;
    }
    { TT_BEGIN ptx::mbar_wait(in_bar, it & 1); TT_END(16) }
    issue<T, true>(c, 4);
    { TT_BEGIN epi_A_exit<T, true>(c); TT_END(18) }
    issue<T, true>(c, 1);
    if constexpr (SPEC) {
      if (lead && item + 2 < i1) load_row(sm + c.in_off, &xmap, row_of(item + 2), in_bar);
      uint32_t f2, g;
      coords(f2, g);
#pragma unroll
      for (uint32_t q = 0; q < kColsPer / 8; ++q) {
        const uint32_t cb = kColsPer * g + 8 * q;
        float re[8], im[8];
        tld<8>(taddr(c, c.tw + cb), re);
        tld<8>(taddr(c, c.tw + 64 + cb), im);
        tc::ld_wait();
        uint4* us = reinterpret_cast<uint4*>(usave + row * kN + 64 * f2 + cb);
        us[0] = make_uint4(pack2<T>(re[0], im[0]), pack2<T>(re[1], im[1]), pack2<T>(re[2], im[2]),
                           pack2<T>(re[3], im[3]));
        us[1] = make_uint4(pack2<T>(re[4], im[4]), pack2<T>(re[5], im[5]), pack2<T>(re[6], im[6]),
                           pack2<T>(re[7], im[7]));
      }
      continue;
    }
    {  // B exit: U -> usave; Z = U Kf2 -> planes [Zr | Zi | -Zr]
      TT_BEGIN
      uint32_t f2, g;
      coords(f2, g);
      unsigned char* op = c.sm + c.sop;
#pragma unroll
      for (uint32_t q2 = 0; q2 < kColsPer / 16; ++q2) {
       float re2[2][8], im2[2][8], kr2[2][8], ki2[2][8];  // 16 columns per TMEM wait
#pragma unroll
       for (uint32_t hh = 0; hh < 2; ++hh) {
        const uint32_t cb = kColsPer * g + 16 * q2 + 8 * hh;
        tld<8>(taddr(c, c.tw + cb), re2[hh]);
        tld<8>(taddr(c, c.tw + 64 + cb), im2[hh]);
        tld<8>(taddr(c, c.aux + cb), kr2[hh]);
        tld<8>(taddr(c, c.aux + 64 + cb), ki2[hh]);
       }
       tc::ld_wait();
#pragma unroll
       for (uint32_t hh = 0; hh < 2; ++hh) {
        const uint32_t cb = kColsPer * g + 16 * q2 + 8 * hh;
        float* re = re2[hh];
        float* im = im2[hh];
        const float* kr = kr2[hh];
        const float* ki = ki2[hh];
        if (usave) {
          uint4* us = reinterpret_cast<uint4*>(usave + row * kN + 64 * f2 + cb);
          us[0] = make_uint4(pack2<T>(re[0], im[0]), pack2<T>(re[1], im[1]), pack2<T>(re[2], im[2]),
                             pack2<T>(re[3], im[3]));
          us[1] = make_uint4(pack2<T>(re[4], im[4]), pack2<T>(re[5], im[5]), pack2<T>(re[6], im[6]),
                             pack2<T>(re[7], im[7]));
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float a = re[j], b = im[j];
          re[j] = fmaf(a, kr[j], -b * ki[j]);
          im[j] = fmaf(a, ki[j], b * kr[j]);
        }
        st8<T>(op + off_bmn(cb, f2), re);
        st8<T>(op + 16384 + off_bmn(cb, f2), im);
        st8n<T>(op + 32768 + off_bmn(cb, f2), re);
       }
      }
      TT_END(19)
    }
    issue<T, true>(c, 2);
    { TT_BEGIN epi_Bp_exit<T>(c); TT_END(20) }
    issue<T, true>(c, 5);
    // the operand planes are free again: the slot's next row streams in
    // while this one is stored
    {
      TT_BEGIN
      if (lead && item + 2 < i1) load_row(sm + c.in_off, &xmap, row_of(item + 2), in_bar);
      TT_END(22)
    }
    {  // A' exit: W[128 t1 + t2] (re, im) for t1 = 16 g + j
      TT_BEGIN
      uint32_t t2, g;
      coords(t2, g);
#pragma unroll
      for (uint32_t q = 0; q < kColsPer / 16; ++q) {
        const uint32_t cb = kColsPer * g + 16 * q;
        float re[16], im[16];
        tld<16>(taddr(c, c.tw + cb), re);
        tld<16>(taddr(c, c.tw + 64 + cb), im);
        tc::ld_wait();
        uint32_t* o = x1 + row * kN + 128 * cb + t2;
#pragma unroll
        for (int j = 0; j < 16; ++j) o[128 * j] = pack2<T>(re[j], im[j]);
      }
      TT_END(21)
    }
  }
  teardown(tmem_slot);
}

// Backward rows (tp_pass2_bwd_kernel's contract, saved-U form): CTA c owns
// the (h a) row groups [g0, g1); in a group slot s takes pairs s, s+2, ...:
//   DY = FFT(x1dy row)  (stage A full, B)
//   acc_s += conj(U) DY   (U = the forward's saved spectrum; acc_s fp32 in TMEM)
//   du row = IFFT(DY conj(Kf2))  (B', A'), interleaved, in place
// At the group end slot 0 sums acc_0 + acc_1 (fixed order: deterministic)
// and runs it through B', A' into wdk[h a] (fp32, natural t), while slot 1
// starts the next group.
__device__ __forceinline__ uint32_t kf_swz(uint32_t f2, uint32_t f1) {
  return f2 * 64 + ((((f1 >> 2) ^ (f2 & 7)) << 2) | (f1 & 3));
}

template <typename T>
__global__ void __launch_bounds__(kThreads, 1)
    tc_rows_bwd_kernel(const __grid_constant__ CUtensorMap xmap, uint32_t* __restrict__ x1dy,
                       const uint32_t* __restrict__ usave, const float2* __restrict__ kf2,
                       float2* __restrict__ wdk, const uint4* __restrict__ mats,
                       const float2* __restrict__ tab_g, int npairs, int hm) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bars[4];  // mma[2], in[2]
  unsigned char* sm = smem_base(smem_raw);
  int g0, g1;
  cta_range(hm, g0, g1);
  setup(sm, &tmem_slot, bars, 4, 0, mats, tab_g, rows::SMAT, rows::STAB, rows::MAT_BYTES);
  const uint32_t slot = threadIdx.x / kSlotThreads;
  Ctx c = make_ctx(sm, tmem_slot, slot, &bars[slot], true);
  c.sop = rows::SOP + 49152 * slot;
  c.in_off = c.sop + 16384;
  c.smat = rows::SMAT;
  c.tab = reinterpret_cast<const float2*>(sm + rows::STAB);
  c.aux = 256 + 128 * slot;  // acc_s
  uint64_t* in_bar = &bars[2 + slot];
  const bool lead = slot_leader();
  uint32_t* kfs = reinterpret_cast<uint32_t*>(sm + rows::SKF);
  auto load_kf = [&](int ha, uint32_t t0, uint32_t nt) {
    const float4* src = reinterpret_cast<const float4*>(kf2 + (size_t)ha * kN);
    for (uint32_t i = t0; i < kN / 2; i += nt) {
      const float4 v = __ldg(src + i);
      const uint32_t f = 2 * i;
      kfs[kf_swz(f >> 6, f & 63)] = pack2<T>(v.x, v.y);
      kfs[kf_swz(f >> 6, (f & 63) + 1)] = pack2<T>(v.z, v.w);
    }
  };
  {  // acc_s = 0, first Kf2 row
    uint32_t f2, g;
    coords(f2, g);
    const float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (uint32_t q = 0; q < kColsPer / 8; ++q) {
      tst8(taddr(c, c.aux + kColsPer * g + 8 * q), z);
      tst8(taddr(c, c.aux + 64 + kColsPer * g + 8 * q), z);
    }
    tst_wait();
    if (g0 < g1) load_kf(g0, threadIdx.x, kThreads);
  }
  uint32_t in_cnt = 0;
  cta_sync_tc();  // first Kf2 row in smem, accumulators zeroed
  for (int ha = g0; ha < g1; ++ha) {
    if (lead && (int)slot < npairs) load_row(sm + c.in_off, &xmap, (int)slot * hm + ha, in_bar);
    for (int j = (int)slot; j < npairs; j += 2) {
      const size_t row = (size_t)j * hm + ha;
      if (j + 2 >= npairs && ha + 1 < g1) {  // the slot's half of the next Kf2 row -> L2
        const char* nk = reinterpret_cast<const char*>(kf2 + (size_t)(ha + 1) * kN) +
                         (size_t)(threadIdx.x & (kSlotThreads - 1)) * 256 + slot * 128;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(nk));
      }
      ptx::mbar_wait(in_bar, in_cnt & 1);
      ++in_cnt;
      issue<T, true>(c, 4);
      epi_A_exit<T, true>(c);
      uint32_t f2, g;
      coords(f2, g);
      // U in flight while the stage-B MMAs run
      uint4 up[kColsPer / 4];
      {
        const uint4* us = reinterpret_cast<const uint4*>(usave + row * kN + 64 * f2 + kColsPer * g);
#pragma unroll
        for (uint32_t i = 0; i < kColsPer / 4; ++i) up[i] = __ldg(us + i);
      }
      issue<T, true>(c, 1);
      {
        unsigned char* op = c.sm + c.sop;
#pragma unroll
        for (uint32_t q = 0; q < kColsPer / 8; ++q) {
          const uint32_t cb = kColsPer * g + 8 * q;
          float dr[8], di[8], ar[8], ai[8];
          tld<8>(taddr(c, c.tw + cb), dr);
          tld<8>(taddr(c, c.tw + 64 + cb), di);
          tld<8>(taddr(c, c.aux + cb), ar);
          tld<8>(taddr(c, c.aux + 64 + cb), ai);
          const uint4 k0 = *reinterpret_cast<const uint4*>(kfs + kf_swz(f2, cb));
          const uint4 k1 = *reinterpret_cast<const uint4*>(kfs + kf_swz(f2, cb + 4));
          tc::ld_wait();
          const uint32_t uw[8] = {up[2 * q].x, up[2 * q].y, up[2 * q].z, up[2 * q].w,
                                  up[2 * q + 1].x, up[2 * q + 1].y, up[2 * q + 1].z, up[2 * q + 1].w};
          const uint32_t kw[8] = {k0.x, k0.y, k0.z, k0.w, k1.x, k1.y, k1.z, k1.w};
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const float2 u = unpack2<T>(uw[jj]), k = unpack2<T>(kw[jj]);
            const float a = dr[jj], b = di[jj];
            ar[jj] = fmaf(u.x, a, fmaf(u.y, b, ar[jj]));   // acc += conj(U) DY
            ai[jj] = fmaf(u.x, b, fmaf(-u.y, a, ai[jj]));
            dr[jj] = fmaf(a, k.x, b * k.y);                 // Z = DY conj(Kf2)
            di[jj] = fmaf(b, k.x, -a * k.y);
          }
          tst8(taddr(c, c.aux + cb), ar);
          tst8(taddr(c, c.aux + 64 + cb), ai);
          st8<T>(op + off_bmn(cb, f2), dr);  // planes [Zr | Zi | -Zr]
          st8<T>(op + 16384 + off_bmn(cb, f2), di);
          st8n<T>(op + 32768 + off_bmn(cb, f2), dr);
        }
        tst_wait();
      }
      issue<T, true>(c, 2);
      epi_Bp_exit<T>(c);
      issue<T, true>(c, 5);
      if (lead && j + 2 < npairs) load_row(sm + c.in_off, &xmap, (j + 2) * hm + ha, in_bar);
      {
        uint32_t t2, gg;
        coords(t2, gg);
#pragma unroll
        for (uint32_t q = 0; q < kColsPer / 16; ++q) {
          const uint32_t cb = kColsPer * gg + 16 * q;
          float re[16], im[16];
          tld<16>(taddr(c, c.tw + cb), re);
          tld<16>(taddr(c, c.tw + 64 + cb), im);
          tc::ld_wait();
          uint32_t* o = x1dy + row * kN + 128 * cb + t2;
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) o[128 * jj] = pack2<T>(re[jj], im[jj]);
        }
      }
    }
    { TT_BEGIN cta_sync_tc(); TT_END(24) }  // acc_0, acc_1 complete
    if (slot == 0) {  // acc_0 + acc_1 -> B' operand planes; zero both accumulators
      uint32_t f2, g;
      coords(f2, g);
      unsigned char* op = c.sm + c.sop;
      const float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (uint32_t q = 0; q < kColsPer / 8; ++q) {
        const uint32_t cb = kColsPer * g + 8 * q;
        float r0[8], i0[8], r1[8], i1[8];
        tld<8>(taddr(c, 256 + cb), r0);
        tld<8>(taddr(c, 256 + 64 + cb), i0);
        tld<8>(taddr(c, 384 + cb), r1);
        tld<8>(taddr(c, 384 + 64 + cb), i1);
        tc::ld_wait();
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          r0[jj] += r1[jj];
          i0[jj] += i1[jj];
        }
        st8<T>(op + off_bmn(cb, f2), r0);
        st8<T>(op + 16384 + off_bmn(cb, f2), i0);
        st8n<T>(op + 32768 + off_bmn(cb, f2), r0);
        tst8(taddr(c, 256 + cb), z);
        tst8(taddr(c, 256 + 64 + cb), z);
        tst8(taddr(c, 384 + cb), z);
        tst8(taddr(c, 384 + 64 + cb), z);
      }
      tst_wait();
    }
    // next Kf2 row (prefetched into L2 during the group's last pairs): the
    // whole CTA converts it, slot 0 after reading the accumulators
    if (ha + 1 < g1) load_kf(ha + 1, threadIdx.x, kThreads);
    { TT_BEGIN cta_sync_tc(); TT_END(25) }  // accumulators consumed, next Kf2 row in smem
    if (slot == 0) {  // dK spectrum row -> IFFT -> wdk (fp32)
      TT_BEGIN
      issue<T, true>(c, 2);
      epi_Bp_exit<T>(c);
      issue<T, true>(c, 5);
      uint32_t t2, gg;
      coords(t2, gg);
#pragma unroll
      for (uint32_t q = 0; q < kColsPer / 16; ++q) {
        const uint32_t cb = kColsPer * gg + 16 * q;
        float re[16], im[16];
        tld<16>(taddr(c, c.tw + cb), re);
        tld<16>(taddr(c, c.tw + 64 + cb), im);
        tc::ld_wait();
        float2* o = wdk + (size_t)ha * kN + 128 * cb + t2;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) o[128 * jj] = make_float2(re[jj], im[jj]);
      }
      TT_END(26)
    }
  }
  teardown(tmem_slot);
}

}  // namespace tcfft

// ---------------------------------------------------------------- host side
namespace {

using namespace tcfft;

template <typename T>
void put(std::vector<uint8_t>& img, uint32_t off, double v) {
  T h;
  if constexpr (std::is_same<T, __nv_bfloat16>::value) h = __float2bfloat16_rn((float)v);
  else h = __float2half_rn((float)v);
  std::memcpy(&img[off], &h, 2);
}

template <typename T>
std::vector<uint8_t> build_mats() {
  std::vector<uint8_t> img(MAT_BYTES, 0);
  // stage A: rows f1 re (0..63) | im (64..127); k t1 re (0..31) | im (32..63)
  for (int r = 0; r < 128; ++r) {
    const int f1 = r % 64;
    const bool imag = r >= 64;
    for (int t1 = 0; t1 < 32; ++t1) {
      const double a = -2.0 * M_PI * (double)((f1 * t1) % 64) / 64.0;
      const double fr = std::cos(a), fi = std::sin(a);
      put<T>(img, MAT_FA + off_kmaj(r, t1, 0), imag ? fi : fr);
      put<T>(img, MAT_FA + off_kmaj(r, 32 + t1, 0), imag ? fr : -fi);
    }
  }
  // DFT128: Fr[f2][t2] = cos, Fi = -sin (symmetric; also serves the inverse)
  for (int r = 0; r < 128; ++r)
    for (int k = 0; k < 128; ++k) {
      const double a = -2.0 * M_PI * (double)((r * k) % 128) / 128.0;
      put<T>(img, MAT_FR + off_kmaj(r, k, 16384), std::cos(a));
      put<T>(img, MAT_FI + off_kmaj(r, k, 16384), std::sin(a));
    }
  return img;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
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

}  // namespace

// Plain (unswizzled) 3-D tiled tensor map, shared with the three-pass column
// kernels: dims {d0, d1, d2} elements of `esize` bytes, row strides in bytes.
int encode_map_3d(CUtensorMap* map, CUtensorMapDataType type, const void* ptr, const uint64_t dims[3],
                  const uint64_t strides[2], const uint32_t box[3]) {
  EncodeFn enc = encode_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return FB_ERR_CUDA;
  }
  const cuuint64_t d[3] = {dims[0], dims[1], dims[2]};
  const cuuint64_t st[2] = {strides[0], strides[1]};
  const cuuint32_t bx[3] = {box[0], box[1], box[2]};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(map, type, 3, const_cast<void*>(ptr), d, st, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (3-D) failed (" + std::to_string((int)r) + ")");
    return FB_ERR_CUDA;
  }
  return FB_OK;
}

namespace {

// signal [B][H][N] viewed as [B][H][N/128 t1][128 t2]; box [64 t2][N/128 t1][1][1]
template <typename T>
int make_map(CUtensorMap* map, const void* ptr, int64_t B, int64_t H, int64_t N) {
  EncodeFn enc = encode_fn();
  if (!enc) {
    set_error("tcgen05 path: cuTensorMapEncodeTiled unavailable");
    return FB_ERR_CUDA;
  }
  const cuuint64_t dims[4] = {128, (cuuint64_t)(N / 128), (cuuint64_t)H, (cuuint64_t)B};
  const cuuint64_t strides[3] = {128 * 2, (cuuint64_t)N * 2, (cuuint64_t)H * N * 2};
  const cuuint32_t box[4] = {64, (cuuint32_t)(N / 128), 1, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(map, Fmt<T>::tma, 4, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return FB_ERR_CUDA;
  }
  return FB_OK;
}

// Persistent grid: one CTA per SM (or per pair when there are fewer),
// contiguous head-major shares of the B/2 x H channel pairs.
struct TcGrid {
  int ctas, total, npairs;
  int bctas, maxseg;  // backward: CTAs over even-aligned shares (none empty), segments per CTA
};
TcGrid tc_grid(const fb_plan* p, int64_t B) {
  TcGrid g;
  g.npairs = (int)((B + 1) / 2);
  g.total = (int)(p->H * g.npairs);
  g.ctas = std::max(1, std::min(p->num_sms, g.total));
  const int U = (g.total + 1) / 2;
  g.bctas = std::max(1, std::min(p->num_sms, U));
  const int per = 2 * ((U + g.bctas - 1) / g.bctas);
  g.maxseg = (per + g.npairs - 1) / g.npairs + 1;  // head segments one CTA can touch
  return g;
}

}  // namespace

// experiment switch: 0 = MMA token (forward) / free issue (backward), 1 = issue lock
static int tc_sched() {
  static const int v = [] {
    const char* e = std::getenv("FB_TC_SCHED");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

// N = 4096, and N = 2048 run on the same n = 8192 transform (fb_plan_create
// picks n = 8192 for it): the extra zero padding costs transform work but the
// tensor-core path still beats the CUDA-core one there
bool tc_length_ok(int64_t N) { return N == 4096 || N == 2048; }
bool tc_eligible(const fb_plan* p) {
  return p->mode == FB_MODE_CAUSAL && tc_length_ok(p->N) && p->n == 8192 &&
         (p->dtype == FB_BF16 || p->dtype == FB_F16) && (p->tc_ver == 1 || p->N == 4096);
}

int tc_init(fb_plan* p) {
  if (p->tc_ver == 2) {
    int rc = tc2_init(p);
    if (!rc) rc = cuda_status(cudaMalloc(&p->kf_tc, sizeof(__half2) * p->H * kN), "cudaMalloc(kf_tc)");
    if (!rc) rc = cuda_status(cudaMalloc(&p->kf_scale, sizeof(float) * p->H), "cudaMalloc(kf_scale)");
    return rc;
  }
  std::vector<uint8_t> img = p->dtype == FB_BF16 ? build_mats<__nv_bfloat16>() : build_mats<__half>();
  int rc = cuda_status(cudaMalloc(&p->tc_mats, img.size()), "cudaMalloc(tc mats)");
  if (!rc)
    rc = cuda_status(cudaMemcpy(p->tc_mats, img.data(), img.size(), cudaMemcpyHostToDevice),
                     "copy tc mats");
  if (!rc) rc = cuda_status(cudaMalloc(&p->kf_tc, sizeof(__half2) * p->H * kN), "cudaMalloc(kf_tc)");
  if (!rc) rc = cuda_status(cudaMalloc(&p->kf_scale, sizeof(float) * p->H), "cudaMalloc(kf_scale)");
  return rc;
}

size_t tc_saved_size(const fb_plan* p, int64_t B) {
  return (size_t)tc_grid(p, B).total * kN * sizeof(uint32_t);
}

int tc_fwd(fb_plan* p, const void* u, void* y, int64_t B, cudaStream_t s, void* usave) {
  const TcGrid gr = tc_grid(p, B);
  if (p->tc_ver == 2) return tc2_fwd(p, u, y, B, gr.ctas, gr.total, s, usave, false);
  CUtensorMap map;
  auto go = [&](auto tv) {
    using T = decltype(tv);
    int rc = make_map<T>(&map, u, B, p->H, p->N);
    if (rc) return rc;
    auto k = tc_fwd_kernel<T>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_FWD);
    prof_mark(p, 0, 0, s);
    k<<<(unsigned)gr.ctas, kThreads, SMEM_FWD, s>>>(map, (T*)y, (const __half2*)p->kf_tc,
                                                     p->kf_scale, (const uint4*)p->tc_mats, p->tw2,
                                                     (int)B, (int)p->H, gr.total,
                                                     (uint32_t*)usave, tc_sched(), (int)(p->N / 128));
    prof_mark(p, 0, 1, s);
    return cuda_status(cudaGetLastError(), "tc_fwd");
  };
  return p->dtype == FB_BF16 ? go(__nv_bfloat16{}) : go(__half{});
}

// workspace: time-domain dK partials [ctas][maxseg][4096] f32, then (recompute
// path) the parked U = F(u) in the saved layout
static size_t tpart_bytes(const TcGrid& gr) {
  return ((size_t)gr.bctas * gr.maxseg * 4096 * sizeof(float) + 255) & ~size_t(255);
}
size_t tc_workspace(const fb_plan* p, int64_t B) {
  const TcGrid gr = tc_grid(p, B);
  return tpart_bytes(gr) + tc_saved_size(p, B) + 256;
}

static int dk_tail(const fb_plan* p, const TcGrid& gr, const float* tpart, float* dKbar, float* dD,
                   float* dK, cudaStream_t s) {
  auto k = p->N == 4096 ? tc_dk_tail_kernel<4096> : tc_dk_tail_kernel<2048>;
  k<<<(unsigned)p->H, 512, 0, s>>>(tpart, dKbar, dD, p->kbar, p->use_keep ? p->keep : nullptr, dK,
                                   p->p, p->keep_scale, p->smooth_domain == FB_SMOOTH_FREQUENCY,
                                   gr.bctas, gr.total, gr.npairs, gr.maxseg);
  return cuda_status(cudaGetLastError(), "tc_dk_tail");
}

int tc_bwd(fb_plan* p, const void* dy, const void* u, void* du, float* dK, float* dKbar, float* dD,
           int64_t B, void* ws, cudaStream_t s, const void* usave) {
  const TcGrid gr = tc_grid(p, B);
  float* tpart = (float*)ws;
  uint32_t* uscratch = (uint32_t*)((char*)ws + tpart_bytes(gr));
  if (p->tc_ver == 2) {
    int rc = FB_OK;
    if (!usave) {  // no saved transform: U = F(u) into the workspace first
      rc = tc2_fwd(p, u, nullptr, B, gr.ctas, gr.total, s, uscratch, true);
      usave = uscratch;
    }
    if (!rc) rc = tc2_bwd(p, dy, du, B, gr.bctas, gr.total, gr.maxseg, tpart, usave, s);
    if (rc) return rc;
    return dk_tail(p, gr, tpart, dKbar, dD, dK, s);
  }
  CUtensorMap dmap, umap;
  auto go = [&](auto tv) {
    using T = decltype(tv);
    int rc = make_map<T>(&dmap, dy, B, p->H, p->N);
    if (!rc) rc = make_map<T>(&umap, usave ? dy : u, B, p->H, p->N);
    if (rc) return rc;
    auto launch = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BWD3);
      prof_mark(p, 1, 0, s);
      kern<<<(unsigned)gr.bctas, kThreads, SMEM_BWD3, s>>>(
          dmap, umap, (T*)du, (const __half2*)p->kf_tc, p->kf_scale, (const uint4*)p->tc_mats,
          p->tw2, tpart, (int)B, (int)p->H, gr.total, gr.maxseg, (const uint32_t*)usave,
          uscratch, tc_sched(), (int)(p->N / 128));
      prof_mark(p, 1, 1, s);
    };
    if (usave) launch(tc_bwd_kernel<T, true>);
    else launch(tc_bwd_kernel<T, false>);
    return cuda_status(cudaGetLastError(), "tc_bwd");
  };
  int rc = p->dtype == FB_BF16 ? go(__nv_bfloat16{}) : go(__half{});
  if (rc) return rc;
  return dk_tail(p, gr, tpart, dKbar, dD, dK, s);
}

// ---------------------------------------------------------------- three-pass rows (host)
namespace {
template <typename T>
std::vector<uint8_t> build_mats_rows() {
  std::vector<uint8_t> img(rows::MAT_BYTES, 0);
  // stage A (full): rows f1 re (0..63) | im (64..127); k t1 re (0..63, k-block
  // at 0) | t1 im (64..127, k-block at FA_KB1)
  for (int r = 0; r < 128; ++r) {
    const int f1 = r % 64;
    const bool imag = r >= 64;
    for (int t1 = 0; t1 < 64; ++t1) {
      const double a = -2.0 * M_PI * (double)((f1 * t1) % 64) / 64.0;
      const double fr = std::cos(a), fi = std::sin(a);
      put<T>(img, off_kmaj(r, t1, 0), imag ? fi : fr);
      put<T>(img, rows::FA_KB1 + off_kmaj(r, t1, 0), imag ? fr : -fi);
    }
  }
  for (int r = 0; r < 128; ++r)
    for (int k = 0; k < 128; ++k) {
      const double a = -2.0 * M_PI * (double)((r * k) % 128) / 128.0;
      put<T>(img, MAT_FR + off_kmaj(r, k, 16384), std::cos(a));
      put<T>(img, MAT_FI + off_kmaj(r, k, 16384), std::sin(a));
    }
  return img;
}

// planar rows [R][2 planes][64 t1][128 t2] 16-bit; box [64 t2][64 t1][2 planes][1]
template <typename T>
int make_rows_map(CUtensorMap* map, const void* ptr, int64_t R) {
  EncodeFn enc = encode_fn();
  if (!enc) {
    set_error("tcgen05 rows: cuTensorMapEncodeTiled unavailable");
    return FB_ERR_CUDA;
  }
  const cuuint64_t dims[4] = {128, 64, 2, (cuuint64_t)R};
  const cuuint64_t strides[3] = {128 * 2, 8192 * 2, 16384 * 2};
  const cuuint32_t box[4] = {64, 64, 2, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(map, Fmt<T>::tma, 4, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (rows) failed (" + std::to_string((int)r) + ")");
    return FB_ERR_CUDA;
  }
  return FB_OK;
}

// ---------------------------------------------------------------- three-pass pass 1, m = 32 .. 128
// The m-point column DFTs of pass 1 (three_pass.cpp:82-122 as applied by
// conv_three_pass_ordered :225-254) for the causal 16-bit three-pass plans
// with m = 32 / 64 / 128 (N = 128K / 256K / 512K) as one GEMM per tile of 128
// columns tau of a channel pair (b0, b0 + 1) of head h:
//   D[tau][c' m + a] = sum_{c, e < m/2} X[tau][c rows + e] T[c' m + a][c rows + e]
// X = the two channels' data rows (e < m/2; the causal zero half is skipped),
// straight from TMA as an MN-major SW128 A operand (M = 128 tau, K = m);
// T = the real-stacked DFT_m (re / im of sum_e w_m^(-a e) (x0 + i x1)[e]),
// a K-major B operand built once per CTA (N = 2m).  The epilogue applies
// the column twiddle w_n^(-a tau) and stores the planar rows [re l | im l]
// the tcgen05 row pass reads.  Warp-specialised: warp 8 issues the TMA ring,
// warp 9 the MMAs (two TMEM accumulators), warps 0-7 drain TMEM
// (lane quarter = tau, warp half = rows a).
namespace colc {
constexpr int kStages = 3;
constexpr uint32_t kEpi = 256, kThreads = kEpi + 64;
constexpr uint32_t kRowL = 8192;  // l: the row length of the three-pass split
// CTAs per SM: TMEM holds 2 x 2m accumulator columns per CTA; at most 3 (registers)
constexpr int per_sm(int M) { return 512 / (4 * M) < 3 ? 512 / (4 * M) : 3; }
}  // namespace colc

__device__ __forceinline__ void tma_load_3d_sw(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                               uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];" ::"r"(ptx::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(ptx::smem_u32(bar))
      : "memory");
}

// w_n^(-t) from the two-level table [w^t, t < 4096 | w^(4096 i)]
__device__ __forceinline__ float2 tw_two(const float2* __restrict__ tb, uint32_t t) {
  const float2 lo = __ldg(tb + (t & 4095u)), hi = __ldg(tb + 4096u + (t >> 12));
  return make_float2(lo.x * hi.x - lo.y * hi.y, lo.x * hi.y + lo.y * hi.x);
}

template <typename T, int M>
__global__ void __launch_bounds__(colc::kThreads, colc::per_sm(M))
    tc_col1_kernel(const __grid_constant__ CUtensorMap smap, __nv_bfloat16* __restrict__ x1,
                   const float2* __restrict__ tb, int H, int ntiles) {
  constexpr uint32_t ROWS = M / 2, K = 2 * ROWS, NN = 2 * M;
  constexpr uint32_t ABYTES = 4 * ROWS * 128;       // 2 tau blocks x 2 channels x ROWS x 128 B
  constexpr uint32_t KBLK = NN * 128;               // one 64-wide K block of the table
  constexpr uint32_t TCOLS = 2 * NN;                // two accumulators
  constexpr uint32_t NTB = colc::kRowL / 128;       // tau tiles per row
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = smem_base(raw);
  unsigned char* tabl = sm + colc::kStages * ABYTES;
  __shared__ __align__(8) uint64_t full[colc::kStages], sfree[colc::kStages], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  const uint32_t tid = threadIdx.x, warp = tid >> 5;

  // the real-stacked DFT_m table, (n' = c' M + a, k = c ROWS + e)
  for (uint32_t i = tid; i < NN * K; i += colc::kThreads) {
    const uint32_t np = i / K, k = i % K;
    const uint32_t cp = np / M, a = np % M, c = k / ROWS, e = k % ROWS;
    float sn, cs;
    sincospif(2.f * (float)((a * e) % M) / (float)M, &sn, &cs);
    const float v = cp == 0 ? (c == 0 ? cs : sn) : (c == 0 ? -sn : cs);
    *reinterpret_cast<T*>(tabl + off_kmaj(np, k, KBLK)) = cvt<T>(v);
  }
  if (tid == 0) {
    for (int s = 0; s < colc::kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&sfree[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], colc::kEpi);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 0) tc::alloc<TCOLS>(&tmem_base);
  ptx::fence_proxy_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  const int first = blockIdx.x, step = gridDim.x;

  if (warp == 8) {  // TMA producer
    if ((tid & 31) == 0) {
      int i = 0;
      for (int t = first; t < ntiles; t += step, ++i) {
        const int s = i % colc::kStages;
        if (i >= colc::kStages) ptx::mbar_wait(&sfree[s], (uint32_t)(i / colc::kStages + 1) & 1);
        const int tbk = t % NTB, h = (t / NTB) % H, pr = t / (NTB * H);
        unsigned char* dst = sm + s * ABYTES;
        ptx::mbar_arrive_expect_tx(&full[s], ABYTES);
#pragma unroll
        for (int mb = 0; mb < 2; ++mb)
#pragma unroll
          for (int c = 0; c < 2; ++c)
            tma_load_3d_sw(dst + mb * (2 * ROWS * 128) + c * (ROWS * 128), &smap, tbk * 128 + mb * 64, 0,
                           (2 * pr + c) * H + h, &full[s]);
      }
    }
  } else if (warp == 9) {  // MMA issuer
    if ((tid & 31) == 0) {
      const uint32_t id = idesc<T>(128, NN, true, false);
      const uint32_t sa = ptx::smem_u32(sm), st = ptx::smem_u32(tabl);
      int i = 0;
      for (int t = first; t < ntiles; t += step, ++i) {
        const int s = i % colc::kStages, b = i & 1;
        ptx::mbar_wait(&full[s], (uint32_t)(i / colc::kStages) & 1);
        if (i >= 2) ptx::mbar_wait(&tempty[b], (uint32_t)(i / 2 + 1) & 1);
        tc::fence_after();
#pragma unroll
        for (uint32_t ks = 0; ks < K / 16; ++ks) {
          const uint64_t ad = tc::smem_desc(sa + s * ABYTES + ks * 2048, 1024, tc::kSw128, 2 * ROWS * 128);
          const uint64_t bd = tc::smem_desc(st + (ks * 16 / 64) * KBLK + (ks * 16 % 64) * 2, 1024, tc::kSw128);
          tc::mma_bf16(tmem + b * NN, ad, bd, id, ks);
        }
        tc::commit(&sfree[s]);
        tc::commit(&tfull[b]);
      }
    }
  } else {  // epilogue: tau = 32 (warp % 4) + lane, rows a in [half M/2, (half + 1) M/2)
    const uint32_t q = warp & 3, half = warp >> 2, lane = tid & 31;
    int i = 0;
    for (int t = first; t < ntiles; t += step, ++i) {
      const int b = i & 1;
      const int tbk = t % NTB, h = (t / NTB) % H, pr = t / (NTB * H);
      const uint32_t tau = tbk * 128 + 32 * q + lane;
      ptx::mbar_wait(&tfull[b], (uint32_t)(i / 2) & 1);
      tc::fence_after();
      __nv_bfloat16* rows = x1 + (((size_t)pr * H + h) * M) * (2 * colc::kRowL) + tau;
      const uint32_t ta = tmem + ((32u * q) << 16) + b * NN;
      const float2 stp = tw_two(tb, tau);
#pragma unroll 1
      for (uint32_t a0 = half * (M / 2); a0 < (half + 1) * (M / 2); a0 += 16) {
        float re[16], im[16];
        tld<16>(ta + a0, re);
        tld<16>(ta + M + a0, im);
        tc::ld_wait();
        float2 w = tw_two(tb, a0 * tau);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float xr = re[j] * w.x - im[j] * w.y, xi = re[j] * w.y + im[j] * w.x;
          __nv_bfloat16* r = rows + (size_t)(a0 + j) * (2 * colc::kRowL);
          r[0] = __float2bfloat16_rn(xr);
          r[colc::kRowL] = __float2bfloat16_rn(xi);
          w = make_float2(w.x * stp.x - w.y * stp.y, w.x * stp.y + w.y * stp.x);
        }
      }
      tc::fence_before();
      mbar_arrive(&tempty[b]);
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::dealloc<TCOLS>(tmem);
}

template <typename T, int M>
int col1_launch(const fb_plan* p, const void* sig, void* x1, int64_t B, int64_t npairs, cudaStream_t s) {
  EncodeFn enc = encode_fn();
  if (!enc) {
    set_error("tcgen05 pass 1: cuTensorMapEncodeTiled unavailable");
    return FB_ERR_CUDA;
  }
  constexpr uint32_t ROWS = M / 2;  // box rows; data rows N / l <= ROWS (the rest zero-filled)
  const cuuint64_t dims[3] = {colc::kRowL, (cuuint64_t)(p->N / colc::kRowL), (cuuint64_t)(B * p->H)};
  const cuuint64_t strides[2] = {colc::kRowL * 2, (cuuint64_t)p->N * 2};
  const cuuint32_t box[3] = {64, ROWS, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  CUtensorMap map;
  CUresult r = enc(&map, Fmt<T>::tma, 3, const_cast<void*>(sig), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (pass 1) failed (" + std::to_string((int)r) + ")");
    return FB_ERR_CUDA;
  }
  constexpr uint32_t smem = colc::kStages * 4 * ROWS * 128 + (2 * M) * 128 * ((M + 63) / 64) + 1024;
  constexpr int per_sm = colc::per_sm(M);
  const int ntiles = (int)(npairs * p->H * (colc::kRowL / 128));
  auto k = tc_col1_kernel<T, M>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = std::max(1, std::min(ntiles, per_sm * p->num_sms));
  k<<<(unsigned)grid, colc::kThreads, smem, s>>>(map, (__nv_bfloat16*)x1, p->tw_big, (int)p->H, ntiles);
  return cuda_status(cudaGetLastError(), "tc_col1_kernel");
}

// ---------------------------------------------------------------- three-pass pass 3, m = 32 .. 128
// Pass 3 of the causal 16-bit three-pass forward / du (three_pass.cpp:225-254,
// the B^-1 factor :101-122):  y[c l + tau] = sum_a w_m^(+a c) w_n^(+a tau) W[a][tau]
// for the data rows c < m/2, channel b0 = Re, b1 = Im, plus D u.  The
// twiddle sits on the contraction index, so the A operand is built by the
// worker warps (TMA'd W tile [a][128 tau] -> x w_n^(+a tau) -> bf16
// MN-major SW128, K = [re a | im a]); the inverse DFT_m is a K-major B
// operand (N = m: [Re c | Im c]); the same warps then drain the previous
// tile's accumulator (skip added, 16-bit stores).  Warps 8 / 9 (16 / 17 with the
// sixteen worker warps at m = 128) issue the TMA loads / the MMAs.
namespace colc3 {
constexpr int kStages = 2;
constexpr int per_sm(int M) { return M == 32 ? 3 : (M == 64 ? 2 : 1); }
// rows a per sub-tile: m = 64 / 128 run each tile as two a-halves (W and A
// buffers of 16 / 32 KB) accumulating into one TMEM tile, so the double
// buffers fit (two CTAs per SM at m = 64)
constexpr int half_a(int M) { return M == 32 ? 32 : M / 2; }
// worker warps: 16 at m = 128 (one CTA per SM; the drain splits the rows c)
constexpr uint32_t workers(int M) { return M == 128 ? 512 : 256; }
constexpr uint32_t threads(int M) { return workers(M) + 64; }
}  // namespace colc3

template <typename IO, int M>
__global__ void __launch_bounds__(colc3::threads(M), colc3::per_sm(M))
    tc_col3_kernel(const __grid_constant__ CUtensorMap wmap, const IO* __restrict__ skip,
                   IO* __restrict__ out, const float* __restrict__ D, const float2* __restrict__ tb,
                   int B, int H, int rows, int ntiles) {
  constexpr uint32_t ROWS = M / 2, K = 2 * M, NN = M;
  constexpr uint32_t MH = colc3::half_a(M), SPLIT = M / MH, KC = 2 * MH;  // sub-tile: a-rows, K
  constexpr uint32_t EPI = colc3::workers(M), RW = ROWS / (EPI / 256);     // drain rows per warp
  constexpr uint32_t WBYTES = MH * 128 * 4;       // W sub-tile [a][128 tau] complex bf16
  constexpr uint32_t ABYTES = 128 * KC * 2;       // A [tau / 64][k][64 tau], k = [re a | im a]
  constexpr uint32_t KBLK = NN * 128;
  constexpr uint32_t TCOLS = 2 * NN < 32 ? 32 : 2 * NN;
  constexpr uint32_t NTB = colc::kRowL / 128;
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = smem_base(raw);
  unsigned char* abuf = sm;                                   // 2 x ABYTES
  unsigned char* tabl = sm + 2 * ABYTES;                      // K / 64 x KBLK
  unsigned char* wring = tabl + (K / 64) * KBLK;              // kStages x WBYTES
  __shared__ __align__(8) uint64_t wfull[colc3::kStages], wempty[colc3::kStages], afull[2], afree[2],
      tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  const uint32_t tid = threadIdx.x, warp = tid >> 5;

  // inverse DFT_m, (n' = c' ROWS + c, k = [re a | im a])
  for (uint32_t i = tid; i < NN * K; i += EPI + 64) {
    const uint32_t np = i / K, k = i % K;
    const uint32_t cp = np / ROWS, c = np % ROWS, a = k % M, im = k / M;
    float sn, cs;
    sincospif(2.f * (float)((a * c) % M) / (float)M, &sn, &cs);
    const float v = cp == 0 ? (im ? -sn : cs) : (im ? cs : sn);
    *reinterpret_cast<__nv_bfloat16*>(tabl + off_kmaj(np, k, KBLK)) = __float2bfloat16_rn(v);
  }
  if (tid == 0) {
    for (int s = 0; s < colc3::kStages; ++s) {
      ptx::mbar_init(&wfull[s], 1);
      ptx::mbar_init(&wempty[s], EPI);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&afull[b], EPI);
      ptx::mbar_init(&afree[b], 1);
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], EPI);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 0) tc::alloc<TCOLS>(&tmem_base);
  ptx::fence_proxy_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  const int first = blockIdx.x, step = gridDim.x;

  if (warp == EPI / 32) {  // TMA producer: W tiles
    if ((tid & 31) == 0) {
      int g = 0;
      for (int t = first; t < ntiles; t += step)
        for (uint32_t part = 0; part < SPLIT; ++part, ++g) {
          const int s = g % colc3::kStages;
          if (g >= colc3::kStages) ptx::mbar_wait(&wempty[s], (uint32_t)(g / colc3::kStages + 1) & 1);
          const int tbk = t % NTB, hp = t / NTB;  // hp = pr * H + h
          ptx::mbar_arrive_expect_tx(&wfull[s], WBYTES);
          tma_load_3d_sw(wring + s * WBYTES, &wmap, tbk * 128, (int)(part * MH), hp, &wfull[s]);
        }
    }
  } else if (warp == EPI / 32 + 1) {  // MMA issuer
    if ((tid & 31) == 0) {
      const uint32_t id = idesc<__nv_bfloat16>(128, NN, true, false);
      const uint32_t sa = ptx::smem_u32(abuf), st = ptx::smem_u32(tabl);
      int i = 0, g = 0;
      for (int t = first; t < ntiles; t += step, ++i) {
        const int tb2 = i & 1;
        for (uint32_t part = 0; part < SPLIT; ++part, ++g) {
          const int b = g & 1;
          ptx::mbar_wait(&afull[b], (uint32_t)(g / 2) & 1);
          if (part == 0 && i >= 2) ptx::mbar_wait(&tempty[tb2], (uint32_t)(i / 2 + 1) & 1);
          tc::fence_after();
#pragma unroll
          for (uint32_t ks = 0; ks < KC / 16; ++ks) {
            const uint32_t kk = ks * 16, k = kk < MH ? part * MH + kk : M + part * MH + (kk - MH);
            const uint64_t ad = tc::smem_desc(sa + b * ABYTES + ks * 2048, 1024, tc::kSw128, KC * 128);
            const uint64_t bd = tc::smem_desc(st + (k / 64) * KBLK + (k % 64) * 2, 1024, tc::kSw128);
            tc::mma_bf16(tmem + tb2 * NN, ad, bd, id, (part | ks) ? 1u : 0u);
          }
          tc::commit(&afree[b]);
        }
        tc::commit(&tfull[tb2]);
      }
    }
  } else {  // workers
    const uint32_t q = warp & 3, half = (warp >> 2) & 1, c_lo = (warp >> 3) * RW, lane = tid & 31;
    int i = 0, g = 0, tprev = -1;
    for (int t = first;; t += step, ++i) {
      const bool have = t < ntiles;
      for (uint32_t part = 0; have && part < SPLIT; ++part, ++g) {  // A operand of tile i
        const int s = g % colc3::kStages, b = g & 1;
        const uint32_t tau0 = (uint32_t)(t % NTB) * 128;
        ptx::mbar_wait(&wfull[s], (uint32_t)(g / colc3::kStages) & 1);
        if (g >= 2) ptx::mbar_wait(&afree[b], (uint32_t)(g / 2 + 1) & 1);
        const unsigned char* ws = wring + s * WBYTES;
        unsigned char* ab = abuf + b * ABYTES;
#pragma unroll 1
        for (uint32_t j = tid; j < MH * 16; j += EPI) {
          const uint32_t al = j >> 4, a = part * MH + al, tc8 = (j & 15) * 8;
          // half-chunk order alternates every 4 chunks so one load instruction
          // covers all 8 16-byte bank groups (conflict-free 512 B per warp)
          const uint32_t sel = (j >> 2) & 1;
          const unsigned char* rp = ws + al * 512 + tc8 * 4;
          const uint4 x0 = *reinterpret_cast<const uint4*>(rp + 16 * sel);
          const uint4 x1 = *reinterpret_cast<const uint4*>(rp + 16 * (sel ^ 1));
          const uint4 v0 = sel ? x1 : x0, v1 = sel ? x0 : x1;
          const uint32_t vv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
          float2 w = tw_two(tb, a * (tau0 + tc8));
          const float2 sp = tw_two(tb, a);
          w.y = -w.y;  // w_n^(+a tau)
          float re[8], im[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float2 z = unpack2<__nv_bfloat16>(vv[e]);
            re[e] = z.x * w.x - z.y * w.y;
            im[e] = z.x * w.y + z.y * w.x;
            w = make_float2(w.x * sp.x + w.y * sp.y, w.y * sp.x - w.x * sp.y);  // x conj(sp)
          }
          const uint32_t base = (tc8 >> 6) * (KC * 128) + (tc8 & 63) * 2;
          st8<__nv_bfloat16>(ab + sw128(base + al * 128), re);
          st8<__nv_bfloat16>(ab + sw128(base + (MH + al) * 128), im);
        }
        ptx::fence_proxy_async_smem();
        mbar_arrive(&wempty[s]);
        mbar_arrive(&afull[b]);
      }
      if (tprev >= 0) {  // drain tile i - 1: warps w % 8 < 4 channel b0 (Re), else b1 (Im); w / 8 picks the rows
        const int ip = i - 1, b = ip & 1;
        const int tbk = tprev % NTB, h = (tprev / NTB) % H, pr = tprev / (NTB * H);
        const uint32_t tau = tbk * 128 + 32 * q + lane;
        const int bc = 2 * pr + (int)half;
        const bool live = bc < B;
        const size_t o =
            ((size_t)bc * H + h) * ((size_t)rows * colc::kRowL) + tau + (size_t)c_lo * colc::kRowL;
        const int nr = rows - (int)c_lo;  // data rows c < rows of this warp's range
        // skip rows of the next chunk in flight while this one drains (the
        // first chunk's before the accumulator wait)
        IO sk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) sk[j] = (live && j < nr) ? skip[o + (size_t)j * colc::kRowL] : IO{};
        const float d = __ldg(D + h);
        ptx::mbar_wait(&tfull[b], (uint32_t)(ip / 2) & 1);
        tc::fence_after();
        const uint32_t ta = tmem + ((32u * q) << 16) + b * NN + half * ROWS + c_lo;
#pragma unroll 1
        for (uint32_t c0 = 0; c0 < RW; c0 += 16) {
          float v[16];
          tld<16>(ta + c0, v);
          tc::ld_wait();
          float y[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) y[j] = fmaf(d, tof(sk[j]), v[j]);
          if (c0 + 16 < RW) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              sk[j] = (live && (int)(c0 + 16) + j < nr) ? skip[o + (size_t)(c0 + 16 + j) * colc::kRowL] : IO{};
          }
          if (live) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if ((int)c0 + j < nr) out[o + (size_t)(c0 + j) * colc::kRowL] = cvt<IO>(y[j]);
          }
        }
        tc::fence_before();
        mbar_arrive(&tempty[b]);
      }
      if (!have) break;
      tprev = t;
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::dealloc<TCOLS>(tmem);
}

template <typename IO, int M>
int col3_launch(const fb_plan* p, const void* w, const void* skip, void* out, int64_t B, int64_t npairs,
                cudaStream_t s) {
  EncodeFn enc = encode_fn();
  if (!enc) {
    set_error("tcgen05 pass 3: cuTensorMapEncodeTiled unavailable");
    return FB_ERR_CUDA;
  }
  // W = x1 [npairs H][m][l] complex bf16 as 32-bit elements; box [128 tau][m a][1]
  const cuuint64_t dims[3] = {colc::kRowL, (cuuint64_t)M, (cuuint64_t)(npairs * p->H)};
  const cuuint64_t strides[2] = {colc::kRowL * 4, (cuuint64_t)M * colc::kRowL * 4};
  const cuuint32_t box[3] = {128, (cuuint32_t)colc3::half_a(M), 1};
  const cuuint32_t es[3] = {1, 1, 1};
  CUtensorMap map;
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<void*>(w), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (pass 3) failed (" + std::to_string((int)r) + ")");
    return FB_ERR_CUDA;
  }
  constexpr uint32_t MH = colc3::half_a(M);
  constexpr uint32_t smem = 2 * (128 * 2 * MH * 2) + (2 * M / 64) * (M * 128) + colc3::kStages * MH * 512 + 1024;
  const int ntiles = (int)(npairs * p->H * (colc::kRowL / 128));
  auto k = tc_col3_kernel<IO, M>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = std::max(1, std::min(ntiles, colc3::per_sm(M) * p->num_sms));
  k<<<(unsigned)grid, colc3::threads(M), smem, s>>>(map, (const IO*)skip, (IO*)out, p->d, p->tw_big, (int)B,
                                                    (int)p->H, (int)(p->N / colc::kRowL), ntiles);
  return cuda_status(cudaGetLastError(), "tc_col3_kernel");
}
}  // namespace

// pass 3 (forward y / backward du) of the same plans for m = 32 / 64 / 128 on the
// tensor cores; FB_ERR_UNSUPPORTED outside that range
int tc_col3(const fb_plan* p, const void* w, const void* skip, void* out, int64_t B, int64_t npairs,
            cudaStream_t s) {
  static const int off = [] {
    const char* e = std::getenv("FB_COL3_TC");
    return e && e[0] == '0';
  }();
  if (off || p->mode != FB_MODE_CAUSAL || p->l != colc::kRowL || p->N % colc::kRowL ||
      p->N / colc::kRowL > p->m / 2 || (p->dtype != FB_BF16 && p->dtype != FB_F16))
    return FB_ERR_UNSUPPORTED;
  const bool bf = p->dtype == FB_BF16;
  switch (p->m) {
    case 32: return bf ? col3_launch<__nv_bfloat16, 32>(p, w, skip, out, B, npairs, s)
                       : col3_launch<__half, 32>(p, w, skip, out, B, npairs, s);
    case 64: return bf ? col3_launch<__nv_bfloat16, 64>(p, w, skip, out, B, npairs, s)
                       : col3_launch<__half, 64>(p, w, skip, out, B, npairs, s);
    case 128: return bf ? col3_launch<__nv_bfloat16, 128>(p, w, skip, out, B, npairs, s)
                        : col3_launch<__half, 128>(p, w, skip, out, B, npairs, s);
    default: return FB_ERR_UNSUPPORTED;
  }
}

// pass 1 of the causal 16-bit three-pass plans with m = 32 / 64 / 128 on the
// tensor cores (planar bf16 rows for the tcgen05 row pass); FB_ERR_UNSUPPORTED
// when the plan is outside that range (the caller runs the CUDA-core kernel)
int tc_col1(const fb_plan* p, const void* sig, void* x1, int64_t B, int64_t npairs, cudaStream_t s) {
  static const int off = [] {
    const char* e = std::getenv("FB_COL1_TC");
    return e && e[0] == '0';
  }();
  if (off || p->mode != FB_MODE_CAUSAL || p->l != colc::kRowL || p->N % colc::kRowL ||
      p->N / colc::kRowL > p->m / 2 || (p->dtype != FB_BF16 && p->dtype != FB_F16))
    return FB_ERR_UNSUPPORTED;
  const bool bf = p->dtype == FB_BF16;
  switch (p->m) {
    case 32: return bf ? col1_launch<__nv_bfloat16, 32>(p, sig, x1, B, npairs, s)
                       : col1_launch<__half, 32>(p, sig, x1, B, npairs, s);
    case 64: return bf ? col1_launch<__nv_bfloat16, 64>(p, sig, x1, B, npairs, s)
                       : col1_launch<__half, 64>(p, sig, x1, B, npairs, s);
    case 128: return bf ? col1_launch<__nv_bfloat16, 128>(p, sig, x1, B, npairs, s)
                        : col1_launch<__half, 128>(p, sig, x1, B, npairs, s);
    default: return FB_ERR_UNSUPPORTED;
  }
}

bool tc_rows_eligible(const fb_plan* p) {
  static const int off = [] {
    const char* e = std::getenv("FB_ROWS_TC");
    return e && e[0] == '0';
  }();
  // fp16 I/O runs the same bf16 rows (fb_three.cu keeps its intermediates in bf16 then)
  return !off && (p->dtype == FB_BF16 || p->dtype == FB_F16) && p->l == 8192;
}

// x1: npairs x H x m planar bf16 rows in, interleaved (re, im) rows out
static int rows_token() {
  static const int t = [] {
    const char* e = std::getenv("FB_ROWS_TOKEN");
    return e ? std::atoi(e) : 1;
  }();
  return t;
}

static int rows_mats(fb_plan* p) {
  if (p->tcr_mats) return FB_OK;
  std::vector<uint8_t> img = build_mats_rows<__nv_bfloat16>();
  int rc = cuda_status(cudaMalloc(&p->tcr_mats, img.size()), "cudaMalloc(tc rows mats)");
  if (!rc)
    rc = cuda_status(cudaMemcpy(p->tcr_mats, img.data(), img.size(), cudaMemcpyHostToDevice),
                     "copy tc rows mats");
  return rc;
}

int tc_rows_fwd(fb_plan* p, void* x1, void* usave, int64_t npairs, cudaStream_t s) {
  if (int rc = rows_mats(p)) return rc;
  const int hm = (int)(p->H * p->m);
  const int total = (int)(npairs * hm);
  CUtensorMap map;
  int rc = make_rows_map<__nv_bfloat16>(&map, x1, total);
  if (rc) return rc;
  auto k = tc_rows_fwd_kernel<__nv_bfloat16>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rows::SMEM);
  const int ctas = std::max(1, std::min(p->num_sms, total));
  prof_mark(p, 0, 0, s);
  k<<<(unsigned)ctas, kThreads, rows::SMEM, s>>>(map, (uint32_t*)x1, p->kf, (const uint4*)p->tcr_mats,
                                                 p->tw_l, (int)npairs, hm, total, (uint32_t*)usave,
                                                 rows_token());
  prof_mark(p, 0, 1, s);
  return cuda_status(cudaGetLastError(), "tc_rows_fwd");
}

int tc_rows_spectrum(fb_plan* p, void* x1, int64_t npairs, cudaStream_t s) {
  if (int rc = rows_mats(p)) return rc;
  const int hm = (int)(p->H * p->m);
  const int total = (int)(npairs * hm);
  CUtensorMap map;
  int rc = make_rows_map<__nv_bfloat16>(&map, x1, total);
  if (rc) return rc;
  auto k = tc_rows_fwd_kernel<__nv_bfloat16, true>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rows::SMEM);
  const int ctas = std::max(1, std::min(p->num_sms, total));
  k<<<(unsigned)ctas, kThreads, rows::SMEM, s>>>(map, (uint32_t*)x1, p->kf, (const uint4*)p->tcr_mats,
                                                 p->tw_l, (int)npairs, hm, total, (uint32_t*)x1,
                                                 rows_token());
  return cuda_status(cudaGetLastError(), "tc_rows_spectrum");
}

int tc_rows_bwd(fb_plan* p, void* x1dy, const void* usave, float2* wdk, int64_t npairs,
                cudaStream_t s) {
  if (int rc = rows_mats(p)) return rc;
  const int hm = (int)(p->H * p->m);
  CUtensorMap map;
  int rc = make_rows_map<__nv_bfloat16>(&map, x1dy, npairs * hm);
  if (rc) return rc;
  auto k = tc_rows_bwd_kernel<__nv_bfloat16>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rows::SMEM_BWD);
  const int ctas = std::max(1, std::min(p->num_sms, hm));
  prof_mark(p, 1, 0, s);
  k<<<(unsigned)ctas, kThreads, rows::SMEM_BWD, s>>>(map, (uint32_t*)x1dy, (const uint32_t*)usave,
                                                     p->kf, wdk, (const uint4*)p->tcr_mats, p->tw_l,
                                                     (int)npairs, hm);
  prof_mark(p, 1, 1, s);
  return cuda_status(cudaGetLastError(), "tc_rows_bwd");
}

#ifdef FB_TC_TIMING
extern "C" int fb_debug_tc_timing(unsigned long long* out, int reset) {
  if (reset) {
    static unsigned long long z[148 * 2 * 32] = {0};
    cudaMemcpyToSymbol(tcfft::g_tc_timing, z, sizeof(z));
    cudaMemcpyToSymbol(tcfft::g_last, z, sizeof(unsigned long long) * 296);
    return 0;
  }
  return (int)cudaMemcpyFromSymbol(out, tcfft::g_tc_timing, sizeof(unsigned long long) * 148 * 2 * 32);
}
#endif
}  // namespace fb
