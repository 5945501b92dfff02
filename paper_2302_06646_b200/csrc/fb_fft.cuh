// FlashButterfly-B200: fp32 register/shared-memory FFT building blocks.
//
// The reference's apply_stages (proj/src/butterfly.cpp:124-163) walks the
// plan as gather -> dense f x f DFT block -> scatter + twiddle, one stage at
// a time over the whole vector.  On the GPU the same mixed-radix
// factorisation is executed as Stockham autosort passes: each thread gathers
// R strided points from shared memory, applies the DIT twiddle, runs the
// dense R-point DFT block in registers (radix-2 network with compile-time
// roots) and scatters the R outputs.  Output order is natural, so the
// spectrum layout equals the reference's (output_map composed away).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fb {

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
// conj(a) * b
__device__ __forceinline__ float2 cconjmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.x, b.y, -a.y * b.x));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }

template <int IDX>
struct Root32 {  // cos/sin(2 pi IDX / 32) as compile-time constants
  static constexpr float c[9] = {1.000000000e+00f, 9.807852804e-01f, 9.238795325e-01f,
                                 8.314696123e-01f, 7.071067812e-01f, 5.555702330e-01f,
                                 3.826834324e-01f, 1.950903220e-01f, 0.0f};
  // IDX in [0, 16): cos(2 pi IDX/32) = +-c[...], sin = ...
  static constexpr float cosv = IDX <= 8 ? c[IDX] : -c[16 - IDX];
  static constexpr float sinv = IDX <= 8 ? c[8 - IDX] : c[IDX - 8];
};

// v * exp(SIGN * 2 pi i * K / L), K < L/2, L | 32, compile-time.
template <int SIGN, int K, int L>
__device__ __forceinline__ float2 twiddle_const(float2 v) {
  constexpr int idx = K * (32 / L);
  if constexpr (idx == 0) {
    return v;
  } else if constexpr (idx == 8) {  // * (SIGN i)
    return SIGN > 0 ? make_float2(-v.y, v.x) : make_float2(v.y, -v.x);
  } else {
    constexpr float c = Root32<idx>::cosv;
    constexpr float s = SIGN * Root32<idx>::sinv;
    return make_float2(fmaf(v.x, c, -v.y * s), fmaf(v.x, s, v.y * c));
  }
}

template <int R>
struct Log2 {
  static constexpr int v = R <= 1 ? 0 : 1 + Log2<R / 2>::v;
};

template <int R, int B>
struct BitRev {
  static constexpr int v = B == 0 ? 0 : ((R & 1) << (B - 1)) | BitRev<(R >> 1), B - 1>::v;
};
template <int R>
struct BitRev<R, 0> {
  static constexpr int v = 0;
};

// One radix-2 DIF layer of span S over a length-R register array.
template <int SIGN, int R, int S, int START, int K>
__device__ __forceinline__ void dif_butterfly(float2 (&v)[R]) {
  if constexpr (START < R) {
    if constexpr (K < S) {
      const float2 a = v[START + K], b = v[START + K + S];
      v[START + K] = cadd(a, b);
      v[START + K + S] = twiddle_const<SIGN, K, 2 * S>(csub(a, b));
      dif_butterfly<SIGN, R, S, START, K + 1>(v);
    } else {
      dif_butterfly<SIGN, R, S, START + 2 * S, 0>(v);
    }
  }
}
template <int SIGN, int R, int S>
__device__ __forceinline__ void dif_layers(float2 (&v)[R]) {
  if constexpr (S >= 1) {
    dif_butterfly<SIGN, R, S, 0, 0>(v);
    dif_layers<SIGN, R, S / 2>(v);
  }
}
template <int R, int I>
__device__ __forceinline__ void bitrev_copy(const float2 (&a)[R], float2 (&b)[R]) {
  if constexpr (I < R) {
    b[I] = a[BitRev<I, Log2<R>::v>::v];
    bitrev_copy<R, I + 1>(a, b);
  }
}

// In-register R-point DFT: v[k] <- sum_t v[t] exp(SIGN 2 pi i t k / R).
// This is the dense f x f block of the reference plan (butterfly.cpp:13-20,
// applied at :146-152), evaluated with a radix-2 network.
template <int SIGN, int R>
__device__ __forceinline__ void dft_reg(float2 (&v)[R]) {
  if constexpr (R > 1) {
    dif_layers<SIGN, R, R / 2>(v);
    float2 t[R];
    bitrev_copy<R, 0>(v, t);
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = t[i];
  }
}

// Shared-memory slot of logical element e: one pad slot per 16 elements so
// the radix-16 scatter of the first pass (stride-16 stores) is bank
// conflict free.
__device__ __forceinline__ uint32_t pad16(uint32_t e) { return e + (e >> 4); }
__host__ __device__ constexpr uint32_t padded_len(uint32_t n) { return n + (n >> 4); }

// Division / remainder by a runtime power of two (every transform size,
// batch and column-tile width here is one): a shift and a mask instead of the
// integer-division sequence.
__device__ __forceinline__ uint32_t pdiv(uint32_t a, uint32_t b) { return a >> (__ffs(b) - 1); }
__device__ __forceinline__ uint32_t pmod(uint32_t a, uint32_t b) { return a & (b - 1); }

// Twiddle lookup exp(SIGN * 2 pi i * t / n) from a table of exp(-2 pi i t/n).
template <int SIGN>
__device__ __forceinline__ float2 tw_lookup(const float2* __restrict__ tw, uint32_t t) {
  const float2 w = __ldg(tw + t);
  return SIGN < 0 ? w : make_float2(w.x, -w.y);
}

// One Stockham pass of radix R over a batch of length-n transforms stored
// element-major in shared memory (element e of transform c at s[e*batch+c]).
// Butterfly q (q = c + batch * j, j in [0, n/R)) reads s[(j + r n/R)], applies
// the DIT twiddle w^(r (j mod Ns)), w = exp(SIGN 2 pi i / (Ns R)), runs the
// R-point DFT and writes to s[(j/Ns) Ns R + j mod Ns + r Ns].  Reads complete
// (syncthreads) before writes, so the pass is in place.
template <int SIGN, int R>
__device__ __forceinline__ void stockham_load_twiddle(const float2* s, float2 (&v)[R], uint32_t j,
                                                      uint32_t c, uint32_t n, uint32_t batch,
                                                      uint32_t Ns, const float2* __restrict__ tw) {
  const uint32_t stride = pdiv(n, R);
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = s[pad16(j + r * stride) * batch + c];
  if (Ns > 1) {
    const uint32_t base = pmod(j, Ns) * pdiv(n, Ns * R);
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], tw_lookup<SIGN>(tw, r * base));
  }
}

template <int R>
__device__ __forceinline__ void stockham_store(float2* s, const float2 (&v)[R], uint32_t j,
                                               uint32_t c, uint32_t batch, uint32_t Ns) {
  const uint32_t idxD = pdiv(j, Ns) * Ns * R + pmod(j, Ns);
#pragma unroll
  for (int r = 0; r < R; ++r) s[pad16(idxD + r * Ns) * batch + c] = v[r];
}

// Apply the DIT twiddle of a pass to registers already loaded.
template <int SIGN, int R>
__device__ __forceinline__ void stockham_twiddle(float2 (&v)[R], uint32_t j, uint32_t n, uint32_t Ns,
                                                 const float2* __restrict__ tw) {
  if (Ns > 1) {
    const uint32_t base = pmod(j, Ns) * pdiv(n, Ns * R);
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], tw_lookup<SIGN>(tw, r * base));
  }
}

// Full in-place middle passes: runs radix-16 passes (and one radix-SMALL
// pass when SMALL > 1) for Ns from ns_begin up to (but excluding) ns_end.
// Each thread owns EPT = 16 points per pass: T = n*batch/16 threads.
// The pass order is: [16, SMALL, 16, 16, ...]: the small radix sits at
// Ns == 16 (second pass) when present.
template <int SIGN, int SMALL>
__device__ __forceinline__ void smem_passes(float2* s, uint32_t n, uint32_t batch, uint32_t ns_begin,
                                           uint32_t ns_end, const float2* __restrict__ tw) {
  const uint32_t tid = threadIdx.x;
  for (uint32_t Ns = ns_begin; Ns < ns_end;) {
    const bool small = (SMALL > 1) && (Ns == 16);
    if (small) {
      if constexpr (SMALL > 1) {
        constexpr int G = 16 / SMALL;  // butterflies per thread
        float2 v[G][SMALL];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const uint32_t q = tid + g * blockDim.x;
          const uint32_t c = pmod(q, batch), j = pdiv(q, batch);
          stockham_load_twiddle<SIGN, SMALL>(s, v[g], j, c, n, batch, Ns, tw);
          dft_reg<SIGN, SMALL>(v[g]);
        }
        __syncthreads();
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const uint32_t q = tid + g * blockDim.x;
          stockham_store<SMALL>(s, v[g], pdiv(q, batch), pmod(q, batch), batch, Ns);
        }
        __syncthreads();
      }
      Ns *= SMALL;
    } else {
      float2 v[16];
      const uint32_t c = pmod(tid, batch), j = pdiv(tid, batch);
      stockham_load_twiddle<SIGN, 16>(s, v, j, c, n, batch, Ns, tw);
      dft_reg<SIGN, 16>(v);
      __syncthreads();
      stockham_store<16>(s, v, j, c, batch, Ns);
      __syncthreads();
      Ns *= 16;
    }
  }
}


// ---------------------------------------------------------------------------
// Compile-time-size Stockham passes (v2): n = 2^LOG2N points per transform,
// T = n/16 threads, pass order [16, SMALL?, 16, ..., 16] with SMALL =
// 2^(LOG2N mod 4) at Ns == 16.  Twiddles come from a two-level smem table
//   tab[i] = w^i (i < 64),  tab[64 + i] = w^(64 i) (i < n/64),  w = e^{-2 pi i/n}
// so w^t = tab[t & 63] * tab[64 + (t >> 6)].
// ---------------------------------------------------------------------------
template <int LOG2N>
struct FftShape {
  static constexpr uint32_t n = 1u << LOG2N;
  static constexpr uint32_t T = n / 16;
  static constexpr uint32_t stride = n / 16;
  static constexpr int SMALL = 1 << (LOG2N % 4);
  static constexpr uint32_t tab_len = 64 + n / 64;
  static constexpr uint32_t work_len = n + n / 16;  // padded float2 slots
};

template <int SIGN>
__device__ __forceinline__ float2 tw2(const float2* tab, uint32_t t) {
  const float2 w = cmul(tab[t & 63u], tab[64u + (t >> 6)]);
  return SIGN < 0 ? w : make_float2(w.x, -w.y);
}

// v[r] *= w^(r * base) for r in [1, R): four table lookups, the rest by
// products (depth <= 3), so twiddle error stays at a few ulp.
template <int SIGN, int R>
__device__ __forceinline__ void apply_tw(float2 (&v)[R], const float2* tab, uint32_t base) {
  const float2 w1 = tw2<SIGN>(tab, base);
  v[1] = cmul(v[1], w1);
  if constexpr (R >= 4) {
    const float2 w2 = tw2<SIGN>(tab, 2 * base);
    const float2 w3 = cmul(w1, w2);
    v[2] = cmul(v[2], w2);
    v[3] = cmul(v[3], w3);
    if constexpr (R >= 8) {
      const float2 w4 = tw2<SIGN>(tab, 4 * base);
      v[4] = cmul(v[4], w4);
      v[5] = cmul(v[5], cmul(w1, w4));
      v[6] = cmul(v[6], cmul(w2, w4));
      const float2 w7 = cmul(w3, w4);
      v[7] = cmul(v[7], w7);
      if constexpr (R >= 16) {
        const float2 w8 = tw2<SIGN>(tab, 8 * base);
        v[8] = cmul(v[8], w8);
        v[9] = cmul(v[9], cmul(w1, w8));
        v[10] = cmul(v[10], cmul(w2, w8));
        v[11] = cmul(v[11], cmul(w3, w8));
        v[12] = cmul(v[12], cmul(w4, w8));
        v[13] = cmul(v[13], cmul(cmul(w1, w4), w8));
        v[14] = cmul(v[14], cmul(cmul(w2, w4), w8));
        v[15] = cmul(v[15], cmul(w7, w8));
      }
    }
  }
}

// Same as apply_tw, from a full global table tw[t] = w^t (t < n): four
// L1/L2-resident lookups per column instead of a per-CTA smem table.
template <int SIGN, int R>
__device__ __forceinline__ void apply_tw_g(float2 (&v)[R], const float2* __restrict__ tw,
                                           uint32_t base) {
  const float2 w1 = tw_lookup<SIGN>(tw, base);
  v[1] = cmul(v[1], w1);
  if constexpr (R >= 4) {
    const float2 w2 = tw_lookup<SIGN>(tw, 2 * base);
    const float2 w3 = cmul(w1, w2);
    v[2] = cmul(v[2], w2);
    v[3] = cmul(v[3], w3);
    if constexpr (R >= 8) {
      const float2 w4 = tw_lookup<SIGN>(tw, 4 * base);
      v[4] = cmul(v[4], w4);
      v[5] = cmul(v[5], cmul(w1, w4));
      v[6] = cmul(v[6], cmul(w2, w4));
      const float2 w7 = cmul(w3, w4);
      v[7] = cmul(v[7], w7);
      if constexpr (R >= 16) {
        const float2 w8 = tw_lookup<SIGN>(tw, 8 * base);
        v[8] = cmul(v[8], w8);
        v[9] = cmul(v[9], cmul(w1, w8));
        v[10] = cmul(v[10], cmul(w2, w8));
        v[11] = cmul(v[11], cmul(w3, w8));
        v[12] = cmul(v[12], cmul(w4, w8));
        v[13] = cmul(v[13], cmul(cmul(w1, w4), w8));
        v[14] = cmul(v[14], cmul(cmul(w2, w4), w8));
        v[15] = cmul(v[15], cmul(w7, w8));
      }
    }
  }
}

// Load + twiddle + DFT of one radix-R butterfly j of the pass at Ns = NS.
template <int SIGN, int R, uint32_t NS, int LOG2N>
__device__ __forceinline__ void bfly_load(const float2* s, const float2* tab, float2 (&v)[R],
                                          uint32_t j) {
  constexpr uint32_t n = 1u << LOG2N, str = n / R;
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = s[pad16(j + r * str)];
  if constexpr (NS > 1) apply_tw<SIGN, R>(v, tab, (j % NS) * (n / (NS * R)));
  dft_reg<SIGN, R>(v);
}
template <int R, uint32_t NS>
__device__ __forceinline__ void bfly_store(float2* s, const float2 (&v)[R], uint32_t j) {
  const uint32_t idxD = (j / NS) * NS * R + (j % NS);
#pragma unroll
  for (int r = 0; r < R; ++r) s[pad16(idxD + r * NS)] = v[r];
}

// All passes with NS in [NS0, n/16): in place, __syncthreads between.
template <int SIGN, int LOG2N, uint32_t NS>
__device__ __forceinline__ void mid_passes(float2* s, const float2* tab) {
  using S = FftShape<LOG2N>;
  if constexpr (NS < S::n / 16) {
    const uint32_t tid = threadIdx.x;
    if constexpr (S::SMALL > 1 && NS == 16) {
      constexpr int R = S::SMALL, G = 16 / R;
      float2 v[G][R];
#pragma unroll
      for (int g = 0; g < G; ++g) bfly_load<SIGN, R, NS, LOG2N>(s, tab, v[g], tid + g * S::T);
      __syncthreads();
#pragma unroll
      for (int g = 0; g < G; ++g) bfly_store<R, NS>(s, v[g], tid + g * S::T);
      __syncthreads();
      mid_passes<SIGN, LOG2N, NS * R>(s, tab);
    } else {
      float2 v[16];
      bfly_load<SIGN, 16, NS, LOG2N>(s, tab, v, tid);
      __syncthreads();
      bfly_store<16, NS>(s, v, tid);
      __syncthreads();
      mid_passes<SIGN, LOG2N, NS * 16>(s, tab);
    }
  }
}

}  // namespace fb
