// FlashButterfly-B200: host-side plan object and internal launcher API.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/flashbutterfly.h"

struct fb_plan {
  int64_t N = 0, H = 0;
  int64_t n = 0;       // transform length
  int64_t l = 0, m = 1;  // three-pass split (single: l = n, m = 1)
  int mode = FB_MODE_CAUSAL, dtype = FB_F32, engine = FB_ENGINE_SINGLE, device = 0;
  bool periodic = false;  // circular with n > N: u periodically extended
  float2* tw_n = nullptr;  // exp(-2 pi i t / n), t < n
  float2* tw2 = nullptr;   // two-level table for n: [w^i, i<64 | w^(64 i), i<n/64]
  float2* tw_l = nullptr;  // two-level table for l (three-pass pass 2)
  float2* tw_m = nullptr;  // full table exp(-2 pi i t / m)      (three-pass, m > 16)
  float2* tw_big = nullptr; // [w^t, t < 4096 | w^(4096 i), i < n/4096], w = e^{-2 pi i/n}
  float2* kf = nullptr;    // per-head spectrum / n: single [H][n]; three [H][m][l]
  float* kbar = nullptr;   // [H][N] regularized kernels
  uint8_t* keep = nullptr; // [H][N] dropout keep flags (training only)
  float* d = nullptr;      // [H] skip gains
  bool use_tc = false;       // tcgen05 single-pass path (fb_single_tc.cu)
  int tc_ver = 1;            // 1: 64 x 128 Monarch (fb_single_tc.cu); 2: 128 x 64, TMEM-resident middle stages (fb_tc2.cu)
  void* tc_mats = nullptr;   // DFT blocks in UMMA smem images
  void* kf_tc = nullptr;     // k_f' = k_f + D/n as fp16 pairs, scaled: v2 [H][f1 128][f2 64]
                             // (f = f1 + 128 f2), v1 [H][f1 64][f2 128] (f = f1 + 64 f2)
  float* kf_scale = nullptr; // [H] inverse of that per-head power-of-two scale
  void* tcr_mats = nullptr;  // three-pass rows on tcgen05: DFT blocks (fb_single_tc.cu)
  // short single pass (N = n / 2 <= 1024, 16-bit) on the radix-16 tcgen05
  // stages of fb_learned_tc.cu with the DFT as blocks: chain [16] * sc_stc + [2^sc_lgfl]
  bool use_sc = false;
  int sc_stc = 0, sc_lgfl = 0;
  float2* sc_blocks = nullptr;  // the chain's DFT blocks [16 x 16, 16 x 16, FL x FL]
  float2* sc_tw = nullptr;      // exp(-2 pi i t / n), t < n
  bool prepared = false;
  bool use_keep = false;
  double lambda = 0.0, keep_scale = 1.0;
  int64_t p = 0;
  int smooth_domain = FB_SMOOTH_TIME;
  int num_sms = 148;
  int64_t head0 = 0;  // first global head of this plan (dropout child streams)
  // three-pass: the kernel prep and the backward's dK tail run on an auxiliary
  // stream, overlapping pass 1 / pass 3 of the signals (fork / join by events)
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_prep = nullptr, ev_join = nullptr;
  bool prep_async = false;  // ev_prep guards kbar / kf / D / keep
  // one-shot caller events around the next launch of the forward's / the
  // backward's main kernel (fb_plan_profile_events; bench.py's roofline)
  cudaEvent_t prof[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  // three-pass: the caller's K, copied on the caller's stream before the prep
  // forks onto the auxiliary stream ([H][N] f32; the caller may reuse K at once)
  float* kraw = nullptr;
  // causal three-pass with N % l != 0: the work runs on `inner`, the same
  // transform for N' = ceil(N / l) l, through zero-padded staging copies
  // (signals in the workspace, K in kraw [H][N']); outputs are cropped to N
  fb_plan* inner = nullptr;
};

struct fb_learned_plan {
  int64_t n = 0, r = 0, H = 0;
  int dtype = FB_F32, device = 0;
  int nstages = 0;
  int64_t factors[32] = {0};
  int64_t param_count = 0;
  void* ext = nullptr;  // device tables (fb_learned.cu)
};

namespace fb {
// Restores the calling thread's current device when an entry point returns
// (entry points run on the plan's device, the caller's context is kept).
struct DevGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DevGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) err = cudaSetDevice(dev);
  }
  ~DevGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

void set_error(const std::string& msg);
int cuda_status(cudaError_t e, const char* where);

// single-pass (fb_single.cu)
int sp_prep(fb_plan* p, const float* K, cudaStream_t s);
int sp_fwd(fb_plan* p, const void* u, void* y, int64_t B, cudaStream_t s);
size_t sp_workspace(const fb_plan* p, int64_t B);
int sp_bwd(fb_plan* p, const void* dy, const void* u, void* du, float* dK, float* dKbar, float* dD,
           int64_t B, void* ws, cudaStream_t s);

// Where the persistent tcgen05 backward leaves its dK spectrum partials:
// spart[cta * maxseg + seg] for the CTAs' contiguous shares of the
// total = H x npairs head-major pairs (fb_single_tc.cu).
struct SpartMap {
  int ctas, total, npairs, maxseg;
  int even = 0;  // CTA shares start at 2 floor(c ceil(total/2) / ctas)
};
int sp_finalize(fb_plan* p, const float2* spart, const float* ddpart, int chunks, float* dkbar,
                float* dD, float* dK, int dd_lag0, const SpartMap* map, cudaStream_t s);

// Unswizzled 3-D TMA tensor map (fb_single_tc.cu)
int encode_map_3d(CUtensorMap* map, CUtensorMapDataType type, const void* ptr, const uint64_t dims[3],
                  const uint64_t strides[2], const uint32_t box[3]);

// tcgen05 single-pass (fb_single_tc.cu)
bool tc_eligible(const fb_plan* p);
// three-pass pass 2 on tcgen05 (bf16, m <= 16): planar rows in, interleaved out
bool tc_rows_eligible(const fb_plan* p);
int tc_rows_fwd(fb_plan* p, void* x1, void* usave, int64_t npairs, cudaStream_t s);
// three-pass pass 1 on tcgen05 (causal, 16-bit, m = 32 / 64 / 128): planar bf16 rows
int tc_col1(const fb_plan* p, const void* sig, void* x1, int64_t B, int64_t npairs, cudaStream_t s);
// pass 3 (y / du) of the same plans for m = 32 / 64 (W = interleaved complex bf16 rows)
int tc_col3(const fb_plan* p, const void* w, const void* skip, void* out, int64_t B, int64_t npairs,
            cudaStream_t s);
// backward rows (saved U): planar dy rows in, du rows out in place, wdk = IFFT_l(dK spectrum)
int tc_rows_spectrum(fb_plan* p, void* x1, int64_t npairs, cudaStream_t s);  // U in place
int tc_rows_bwd(fb_plan* p, void* x1dy, const void* usave, float2* wdk, int64_t npairs,
                cudaStream_t s);
int tc_init(fb_plan* p);
// version 2 (fb_tc2.cu)
int tc2_init(fb_plan* p);
bool tc_length_ok(int64_t N);
bool tp_uses_tc_rows(const fb_plan* p);  // fb_three.cu: pass 2 on the tcgen05 rows
int tc2_fwd(fb_plan* p, const void* u, void* y, int64_t B, int ctas, int total, cudaStream_t s,
            void* usave, bool spectrum_only);
int tc2_bwd(fb_plan* p, const void* dy, void* du, int64_t B, int ctas, int total, int maxseg,
            float* tpart, const void* usave, cudaStream_t s);
// usave (optional): the forward writes U = F(u) there (tc_saved_size bytes)
// and the backward reads it instead of recomputing (u may then be null)
size_t tc_saved_size(const fb_plan* p, int64_t B);
int tc_fwd(fb_plan* p, const void* u, void* y, int64_t B, cudaStream_t s, void* usave = nullptr);
size_t tc_workspace(const fb_plan* p, int64_t B);
int tc_bwd(fb_plan* p, const void* dy, const void* u, void* du, float* dK, float* dKbar, float* dD,
           int64_t B, void* ws, cudaStream_t s, const void* usave = nullptr);

// three-pass (fb_three.cu)
int tp_prep(fb_plan* p, const float* K, cudaStream_t s);
// usave: the forward keeps its pass-2 row spectra of u (tp_saved_size bytes) and the
// backward reads them instead of transforming u (u may then be null)
size_t tp_saved_size(const fb_plan* p, int64_t B);
int tp_fwd(fb_plan* p, const void* u, void* y, int64_t B, void* ws, cudaStream_t s,
           void* usave = nullptr);
size_t tp_workspace(const fb_plan* p, int64_t B);
int tp_bwd(fb_plan* p, const void* dy, const void* u, void* du, float* dK, float* dKbar, float* dD,
           int64_t B, void* ws, cudaStream_t s, const void* usave = nullptr);

// shared K1 pieces (fb_prep.cu)
int regularize_bank_dev(fb_plan* p, const float* K, cudaStream_t s);
int dropout_keep_dev(fb_plan* p, double rate, uint64_t seed, cudaStream_t s);
// init_kernels (regularize.cpp:73-91) on the device; any output may be null
int init_kernels_dev(int kind, int64_t H, int64_t N, uint64_t seed, float* K, float* D, double* K64,
                     double* D64, int device, cudaStream_t s);
// dK = chain(dKbar) through dropout/smooth/squash, per head; dkbar_in [H][N]
int regularizer_backward_dev(fb_plan* p, const float* dkbar, float* dK, cudaStream_t s);
// record (and clear) the caller's profiling event `e` (0 begin, 1 end) of main kernel k
inline void prof_mark(fb_plan* p, int k, int e, cudaStream_t s) {
  if (p->prof[k][e]) {
    cudaEventRecord(p->prof[k][e], s);
    p->prof[k][e] = nullptr;
  }
}
// make `s` wait for an asynchronous kernel prep (no-op otherwise)
inline int prep_wait(const fb_plan* p, cudaStream_t s) {
  if (p->prep_async) return cuda_status(cudaStreamWaitEvent(s, p->ev_prep, 0), "prep wait");
  return FB_OK;
}

// learned (fb_learned.cu)
size_t lb_workspace(const fb_learned_plan* p, int64_t B);
int lb_fwd(fb_learned_plan* p, const float* blocks, const void* x, void* y, int64_t B, void* ws,
           cudaStream_t s);
int lb_bwd(fb_learned_plan* p, const float* blocks, const void* x, const void* g, void* dx,
           float* dblocks, int64_t B, void* ws, cudaStream_t s);
// learned butterfly on tcgen05 (fb_learned_tc.cu): chains [16] * stc + [2^lgfl]
bool lt_config(int64_t n, const int64_t* f, int nst, int dtype, int* stc, int* lgfl);
int lt_rows(int64_t n);
// short causal single pass on the same stages (fb_learned_tc.cu)
bool sc_config(const fb_plan* p, int* stc, int* lgfl);
int sc_init(fb_plan* p);
int sc_chunks(const fb_plan* p, int64_t B);
int sc_fwd(fb_plan* p, const void* u, void* y, int64_t B, cudaStream_t s);
int sc_bwd(fb_plan* p, const void* dy, const void* u, void* du, float2* spart, float* ddpart,
           int64_t B, cudaStream_t s);
cudaError_t lt_fwd(int stc, int lgfl, int dtype, const float* blocks, const void* x, void* y,
                   const uint32_t* omap, const float2* tw, int B, int H, int P, cudaStream_t s);
cudaError_t lt_bwd(int stc, int lgfl, int dtype, const float* blocks, const void* x, const void* g,
                   void* dx, float2* gpart, const uint32_t* omap, const float2* tw, int B, int H,
                   int P, cudaStream_t s);
}  // namespace fb
