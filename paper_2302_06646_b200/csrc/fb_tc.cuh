// FlashButterfly-B200: tcgen05 / TMEM building blocks (sm_100a inline PTX).
//
// Operand layouts are the canonical UMMA K-major layouts (in 16-byte units,
// CuTe mma_traits_sm100.hpp make_umma_desc):
//   SW128: ((8,n),2):((8,SBO),1)  rows 128 B apart, 16B-chunk ^= (row & 7)
//   SW64 : ((8,n),2):((4,SBO),1)  rows  64 B apart, 16B-chunk ^= (row >> 1) & 3
//   SW32 : ((8,n),2):((2,SBO),1)  rows  32 B apart, 16B-chunk ^= (row >> 2) & 1
// i.e. the swizzle XORs address bits [4, 4+B) with bits [7, 7+B) (B = 3/2/1).
// One MMA consumes K = 16 bf16 (32 bytes); the next K step advances the
// descriptor start address by 32 bytes.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fb {
namespace tc {

enum Swz : int { kSwNone = 0, kSw128 = 2, kSw64 = 4, kSw32 = 6 };

template <int SWZ>
struct SwzTraits;
template <>
struct SwzTraits<kSw128> {
  static constexpr uint32_t row_bytes = 128, atom = 1024, bits = 3;
};
template <>
struct SwzTraits<kSw64> {
  static constexpr uint32_t row_bytes = 64, atom = 512, bits = 2;
};
template <>
struct SwzTraits<kSw32> {
  static constexpr uint32_t row_bytes = 32, atom = 256, bits = 1;
};

// Byte offset of element (row, k) (16-bit elements) in a K-major swizzled
// operand whose rows hold exactly row_bytes (K = row_bytes / 2 elements).
template <int SWZ>
__host__ __device__ __forceinline__ uint32_t kmajor_off(uint32_t row, uint32_t k) {
  using T = SwzTraits<SWZ>;
  const uint32_t lin = (row >> 3) * T::atom + (row & 7) * T::row_bytes + k * 2;
  const uint32_t mask = ((1u << T::bits) - 1u) << 4;
  return lin ^ ((lin >> 3) & mask);
}

// Byte offset of element (m, k) in an MN-major SW128 operand of MT rows
// (MT % 64 == 0): atoms of 8 k x 64 m (1024 B), laid out
// [k / 8][m / 64][k % 8][m % 64]  =>  LBO (MN-block stride) = 1024 B,
// SBO (8-k group stride) = (MT / 64) * 1024 B; canonical
// ((8,n),(8,k)):((1,LBO),(8,SBO)) in 16-byte units.
__host__ __device__ __forceinline__ uint32_t mnmajor_off(uint32_t m, uint32_t k, uint32_t MT) {
  const uint32_t lin = (k >> 3) * (MT / 64) * 1024 + (m >> 6) * 1024 + (k & 7) * 128 + (m & 63) * 2;
  return lin ^ ((lin >> 3) & 0x70u);
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t sbo_bytes, int swz,
                                              uint32_t lbo_bytes = 16) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (sm100)
  d |= (uint64_t)(swz & 7) << 61;
  return d;
}

// kind::f16 instruction descriptor: bf16 x bf16 -> f32, both K-major.
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t M, uint32_t N) {
  return (1u << 4)            // c_format = F32
         | (1u << 7)          // a_format = BF16
         | (1u << 10)         // b_format = BF16
         | ((N >> 3) << 17)   // n_dim
         | ((M >> 4) << 24);  // m_dim
}

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
               : "memory");
}

__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// One warp allocates `cols` TMEM columns (power of two >= 32); address -> *dst.
template <uint32_t COLS>
__device__ __forceinline__ void alloc(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst_smem))),
               "n"(COLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t COLS>
__device__ __forceinline__ void dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(COLS)
               : "memory");
}

// 32 lanes x 32 columns (32-bit): thread i of the warp gets lane (base+i),
// columns [col, col+32).
__device__ __forceinline__ void ld32(uint32_t taddr, float (&v)[32]) {
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
__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

}  // namespace tc
}  // namespace fb
