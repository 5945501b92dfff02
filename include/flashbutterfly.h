/* flashbutterfly.h — C ABI of the B200-native FlashButterfly long convolution
 * (libflashbutterfly.so, built from paper_2302_06646_b200/csrc for sm_100a).
 *
 * This is the drop-in boundary for the reference `longconv` hot path
 * (/root/reference/proj/include/longconv).  Each entry point names the
 * reference interface it replaces.  Plain C: pointers, sizes, a cudaStream_t
 * passed as void*.  No torch types.  All device pointers are caller-owned,
 * row-major with the length dimension innermost, exactly like the
 * reference's containers:
 *   signals  [B][H][N]   (SignalBatch, types.hpp:37-57)
 *   kernels  [H][N] f32, skip gains D[H] f32   (KernelBank, types.hpp:60-75)
 *
 * Errors: every function returns FB_OK (0) or an FB_ERR_* code and sets a
 * thread-local message readable through fb_last_error().  The codes map to
 * the reference exception types: FB_ERR_DIM <-> DimensionError, FB_ERR_PLAN
 * <-> PlanError (errors.hpp:9-26).  There is no CPU fallback: a missing or
 * failing device returns FB_ERR_CUDA.
 *
 * Streams: every launch is asynchronous on the given stream.  A plan may be
 * used by one stream at a time; results are deterministic for a fixed plan
 * (no atomics: the dK batch reduction runs in a fixed order).
 */
#ifndef FLASHBUTTERFLY_H
#define FLASHBUTTERFLY_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FB_VERSION 100

enum fb_status {
  FB_OK = 0,
  FB_ERR_DIM = 1,   /* DimensionError (errors.hpp:10-12)                 */
  FB_ERR_PLAN = 2,  /* PlanError (errors.hpp:15-17)                      */
  FB_ERR_CUDA = 3,  /* device / launch failure                           */
  FB_ERR_NCCL = 4,  /* collective failure (sequence-sharded path)        */
  FB_ERR_ARG = 5,   /* invalid argument (null pointer, bad enum, ...)    */
  FB_ERR_UNSUPPORTED = 6
};

/* ConvMode (butterfly.hpp:69): same numeric order as the reference enum. */
enum fb_mode { FB_MODE_CIRCULAR = 0, FB_MODE_CAUSAL = 1 };

/* Engine (regularize.hpp:17) minus kNaive (the O(N^2) oracle stays in
 * oracle/): AUTO picks single-pass when the transform fits in shared memory.
 * SINGLE uses the tcgen05 tensor-core kernels when the shape/dtype allow
 * (16-bit I/O, causal, N = 4096); SINGLE_SIMT forces the fp32 CUDA-core
 * single-pass kernels. */
enum fb_engine {
  FB_ENGINE_AUTO = 0,
  FB_ENGINE_SINGLE = 1,
  FB_ENGINE_THREE = 2,
  FB_ENGINE_SINGLE_SIMT = 3
};

/* I/O element type of u, y, dy, du. K, D, dK, dD are always f32. */
enum fb_dtype { FB_F32 = 0, FB_BF16 = 1, FB_F16 = 2 };

/* SmoothDomain (regularize.hpp:16). */
enum fb_smooth { FB_SMOOTH_TIME = 0, FB_SMOOTH_FREQUENCY = 1 };

/* RegularizationConfig (regularize.hpp:19-25). */
typedef struct fb_reg_config {
  double lambda;        /* soft threshold >= 0                     */
  int64_t smooth_width; /* p; window 2p+1                          */
  double dropout_rate;  /* in [0,1)                                */
  int smooth_domain;    /* fb_smooth                               */
  uint64_t seed;        /* dropout stream (SeededRng(seed).child(h)) */
} fb_reg_config;

typedef struct fb_plan fb_plan;

typedef struct fb_plan_info {
  int64_t N, H;
  int64_t n;       /* transform length (2N causal, N circular; >= 256)  */
  int64_t l, m;    /* three-pass split n = l*m (l = n, m = 1 single)    */
  int engine;      /* resolved fb_engine                                */
  int dtype, mode;
  int tensor_cores; /* 1 when the tcgen05 kernels run this plan         */
} fb_plan_info;

/* Plan for a bank of H kernels of length N.  Replaces the per-call
 * build_plan(2N, 16) / build_three_pass(...) of regularized_long_conv
 * (regularize.cpp:161-174, butterfly.cpp:72-118, three_pass.cpp:183-205).
 * Allocates the per-head kernel spectrum and twiddle tables on `device`. */
int fb_plan_create(fb_plan** plan, int64_t N, int64_t H, int mode, int dtype, int engine,
                   int device);
int fb_plan_destroy(fb_plan* plan);
int fb_plan_get_info(const fb_plan* plan, fb_plan_info* info);

/* Kernel preparation (K1).  Replaces regularize_bank (regularize.hpp:62-63,
 * regularize.cpp:93-107: dropout -> smooth -> squash) fused with the kernel
 * transform that conv_butterfly recomputes per channel (butterfly.cpp:205)
 * and build_three_pass precomputes per head (three_pass.cpp:197-203).
 * K: [H][N] f32 device, D: [H] f32 device.  The regularized bank Kbar is kept
 * in the plan (fb_plan_copy_kbar) for the backward. */
int fb_kernel_prep(fb_plan* plan, const float* K, const float* D, const fb_reg_config* cfg,
                   int training, void* stream);

/* InitKind (regularize.hpp:27). */
enum fb_init_kind { FB_INIT_RANDOM = 0, FB_INIT_GEOMETRIC = 1 };
/* init_kernels (regularize.hpp:55, regularize.cpp:73-91) on the device:
 * K[h][i] = draw i of SeededRng(seed).child(h).normal() (times the geometric
 * envelope exp(-(i/N) (H/2)^(h/H)) for FB_INIT_GEOMETRIC), D[h] = draw h of
 * child(H) — the reference's streams exactly (xoshiro256++ with GF(2)
 * jump-ahead so each head's stream splits over many threads).  fp64 values;
 * K, D receive them rounded to f32, K64, D64 (optional, may be NULL) as f64. */
int fb_init_kernels(int kind, int64_t H, int64_t N, uint64_t seed, float* K, float* D, double* K64,
                    double* D64, int device, void* stream);
/* Copy the plan's regularized kernels Kbar [H][N] f32 into dst (device),
 * stream-ordered after fb_kernel_prep. */
int fb_plan_copy_kbar(const fb_plan* plan, float* dst, void* stream);

/* Scratch bytes fb_fwd / fb_bwd need for a batch of B (caller allocates). */
size_t fb_workspace_size(const fb_plan* plan, int64_t B);

/* Forward (K2 single-pass / K3 three-pass).  Replaces regularized_long_conv
 * (regularize.hpp:67-70, regularize.cpp:149-190) after fb_kernel_prep:
 *   y[b,h] = conv(u[b,h], Kbar[h]) + D[h] u[b,h].
 * u, y: [B][H][N] in the plan dtype (device). */
int fb_fwd(fb_plan* plan, const void* u, void* y, int64_t B, void* workspace, void* stream);

/* Backward (K4a / K4b).  No reference counterpart (the reference is
 * forward-only); restates the composed oracle of SURVEY.md §8c:
 *   du = corr(dy, Kbar) + D dy,  dKbar = sum_b corr(dy, u),  dD = sum dy u,
 *   dK = dropout'(K) * smooth(1[Kbar != 0] * dKbar)   (chain through K1).
 * dK: [H][N] f32 (gradient w.r.t. the RAW K passed to fb_kernel_prep);
 * dKbar (optional, may be NULL): [H][N] f32; dD: [H] f32. */
int fb_bwd(fb_plan* plan, const void* dy, const void* u, void* du, float* dK, float* dKbar,
           float* dD, int64_t B, void* workspace, void* stream);

/* Training-step variant: fb_fwd_save also writes the forward's own
 * transform of u (U = F(u), bf16 pairs, fb_saved_size bytes, caller-owned)
 * and fb_bwd_saved reads it instead of transforming u again — the saved
 * activation of an autograd step.  Results are identical to fb_fwd / fb_bwd
 * (the recompute path parks exactly these bf16 values).  fb_saved_size is 0
 * for plans without the tensor-core path; both calls then fall back to
 * fb_fwd / fb_bwd (and fb_bwd_saved needs u). */
size_t fb_saved_size(const fb_plan* plan, int64_t B);
int fb_fwd_save(fb_plan* plan, const void* u, void* y, void* saved, int64_t B, void* workspace,
                void* stream);
int fb_bwd_saved(fb_plan* plan, const void* dy, const void* u, const void* saved, void* du,
                 float* dK, float* dKbar, float* dD, int64_t B, void* workspace, void* stream);

/* Measurement hook (not part of the reference interface): the plan records
 * the caller's CUDA events `begin` / `end` (cudaEvent_t as void*) on the
 * launching stream immediately before / after the NEXT launch of its main
 * forward kernel (which = 0: tc_fwd_kernel, sp_fwd_kernel, or the three-pass
 * row kernel) or main backward kernel (which = 1: tc_bwd_kernel,
 * sp_bwd_kernel, or the three-pass backward row kernel), then forgets them.
 * bench.py times the dominant kernel alone this way (roofline). */
int fb_plan_profile_events(fb_plan* plan, int which, void* begin, void* end);

/* Host-buffer layer runner: the whole regularized_long_conv forward +
 * backward (regularize.hpp:67-70 with the SURVEY.md §8c backward) on HOST
 * arrays, pipelined.  The H heads are independent, so the runner walks them
 * in chunks of Hc (a divisor of H): while chunk c computes, chunk c+1's
 * inputs copy in and chunk c-1's results copy out (three CUDA streams,
 * double-buffered device staging), which overlaps both PCIe directions with
 * the kernels.  Host pointers should be pinned (cudaHostAlloc /
 * torch.pin_memory) for the copies to be asynchronous.
 *   u, dy, y, du: [B][H][N] in the plan dtype;  K, dK: [H][N] f32;
 *   D, dD: [H] f32.
 * fb_host_runner_run is stream-ordered: it starts after the work already on
 * `stream` and `stream` waits for all of it (so CUDA events recorded on
 * `stream` around the call time the whole step, copies included). */
typedef struct fb_host_runner fb_host_runner;
int fb_host_runner_create(fb_host_runner** runner, int64_t N, int64_t H, int mode, int dtype,
                          int engine, int device, int64_t B, int64_t heads_per_chunk);
int fb_host_runner_destroy(fb_host_runner* runner);
/* heads actually used per chunk (the largest divisor of H <= the request) */
int64_t fb_host_runner_chunk_heads(const fb_host_runner* runner);
int fb_host_runner_run(fb_host_runner* runner, const fb_reg_config* cfg, int training,
                       const void* u, const void* dy, const float* K, const float* D, void* y,
                       void* du, float* dK, float* dD, void* stream);

/* Sequence-sharded local passes (config 5-4M: the transform n = l m itself
 * split over ranks, paper_2302_06646_b200/seqshard.py; three_pass.cpp:225-254
 * with the all-to-all transposes between the passes).  l = 8192 and
 * 16 <= m = n / l <= 1024.  Data is complex f32 (interleaved re, im).
 *   fb_shard_columns: [C][m][lp] columns tau0 .. tau0+lp of every row;
 *     inverse = 0:  out[a][t] = w_n^(-a tau) sum_c w_m^(-a c) in[c][t]   (pass 1)
 *     inverse = 1:  out[c][t] = (1/n) sum_a w_m^(+a c) w_n^(+a tau) in[a][t]  (pass 3)
 *   fb_shard_rows: [C][mp][l] rows, in place:
 *     mode 0:  rows = sum_s w_l^(+s t) FFT_l(rows)[s] kf2[s]   (kf2 [C][mp][l])
 *     mode 1:  kf2_out = scale FFT_l(rows)                      (spectrum rows) */
typedef struct fb_shard_plan fb_shard_plan;
int fb_shard_plan_create(fb_shard_plan** plan, int64_t n, int device);
int fb_shard_plan_destroy(fb_shard_plan* plan);
int fb_shard_plan_dims(const fb_shard_plan* plan, int64_t* l, int64_t* m);
int fb_shard_columns(fb_shard_plan* plan, const void* in, void* out, int64_t C, int64_t tau0,
                     int64_t lp, int inverse, void* stream);
int fb_shard_rows(fb_shard_plan* plan, void* rows, const void* kf2, void* kf2_out, int64_t C,
                  int64_t mp, int mode, float scale, void* stream);

/* The sharded layer's row passes over channel pairs and its glue (seqshard.py):
 *   fb_shard_rows_pairs: rows [P][H][mp][l] in place, rows = IFFT_l(FFT_l(rows)
 *     kf2[h][a]) with the kernel rows kf2 [H][mp][l] shared by the P pairs
 *   fb_shard_rows_bwd: per (h, a) over the P pairs: dy row <- IFFT_l(DY conj(kf2)),
 *     wdk[h][a] = IFFT_l(sum_p conj(U) DY) (fixed order; unnormalised transforms)
 *   fb_shard_stage: out[b][a][x] = in[a][b][x] on complex elements (f32 or bf16
 *     pairs each side): the all-to-all send / receive layouts */
int fb_shard_rows_pairs(fb_shard_plan* plan, void* rows, const void* kf2, int64_t P, int64_t H, int64_t mp,
                        void* stream);
/* Column passes fused with the layer's pair (un)packing: pass 1 of the
 * channel pairs read straight from the real signals sig [B][H][half][lp]
 * (dtype; rows >= half are the causal zero pad) into complex [P][H][m][lp];
 * pass 3 of complex [P][H][m][lp] written straight back as real signals
 * [B][H][half][lp] (dtype) plus D[h] skip (skip optional). */
int fb_shard_columns_from_signals(fb_shard_plan* plan, const void* sig, int dtype, void* out, int64_t B,
                                  int64_t H, int64_t half, int64_t tau0, int64_t lp, void* stream);
int fb_shard_columns_to_signals(fb_shard_plan* plan, const void* in, void* sig_out, int dtype,
                                const void* skip, const float* D, int64_t B, int64_t H, int64_t half,
                                int64_t tau0, int64_t lp, void* stream);
int fb_shard_rows_bwd(fb_shard_plan* plan, void* dy_rows, const void* u_rows, const void* kf2, void* wdk,
                      int64_t P, int64_t H, int64_t mp, void* stream);
int fb_shard_stage(const void* in, void* out, int64_t A, int64_t Bd, int64_t X, int in_dtype, int out_dtype,
                   void* stream);
/* Learned butterfly (K5).  Replaces learned_forward / learned_gradients
 * (butterfly.hpp:88-108, butterfly.cpp:221-307) batched over rows: rows
 * [B][H] of complex length n, with per-head block parameters (one factor x
 * factor complex matrix per stage of build_plan(n, r), concatenated; P =
 * sum_s f_s^2 complex values per head).  Complex data is interleaved f32
 * (re, im).  x, y, g, dx: [B][H][n] complex in the plan dtype;
 * blocks, dblocks: [H][P] complex f32.  dblocks = sum over b (per head). */
typedef struct fb_learned_plan fb_learned_plan;
int fb_learned_plan_create(fb_learned_plan** plan, int64_t n, int64_t r, int64_t H, int dtype,
                           int device);
int fb_learned_plan_destroy(fb_learned_plan* plan);
/* Number of stages and their factors (build_plan greedy chain,
 * butterfly.cpp:83-100); returns P through *param_count. */
int fb_learned_plan_factors(const fb_learned_plan* plan, int64_t* factors, int64_t* count,
                            int64_t* param_count);
/* Kernel family the plan runs: 0 = generic stage walk (any chain), 1 = the
 * factor-specialised CUDA-core kernels (power-of-two factors <= 16), 2 =
 * tcgen05 (16-bit modes, chains [16] * S + [2|4|8|16], n = 32 .. 4096). */
int fb_learned_plan_engine(const fb_learned_plan* plan, int* engine);
size_t fb_learned_workspace_size(const fb_learned_plan* plan, int64_t B);
int fb_learned_fwd(fb_learned_plan* plan, const float* blocks, const void* x, void* y, int64_t B,
                   void* workspace, void* stream);
int fb_learned_bwd(fb_learned_plan* plan, const float* blocks, const void* x, const void* g,
                   void* dx, float* dblocks, int64_t B, void* workspace, void* stream);

/* Complex row transforms / convolutions through the butterfly plan: the
 * device side of the reference's single-row entry points build_plan +
 * apply_plan (butterfly.hpp:74-79), conv_butterfly (butterfly.hpp:82-83) and
 * conv_three_pass's circular convolution with a precomputed spectrum
 * (three_pass.hpp:119-120).  Rows of complex f32, interleaved (re, im).
 * fb_dft_plan_create validates n and r like build_plan (FB_ERR_PLAN for
 * n < 1, r < 2, or a remainder with no factor <= r) and runs the plan's own
 * greedy stage chain with the exact DFT blocks (butterfly.cpp:13-20), so any
 * buildable n works (n > 8192 as a four-step composition of two stage chains).
 *   fb_dft:   y = F_n x (inverse = 0) or conj(F_n conj(x)) / n (inverse = 1)
 *   fb_conv_rows: y = conv(u, k) per row; mode FB_MODE_CIRCULAR needs n == N,
 *     FB_MODE_CAUSAL n == 2N (zero-padded, first N outputs); k has k_rows rows
 *     (1: shared by every row, or rows)
 *   fb_conv_rows_spectrum: the same with the kernel given as its forward
 *     spectrum kspec [k_rows][n] (e.g. build_three_pass's K_hat = F_n k).
 * Workspace: fb_dft_workspace_size(plan, rows, 0) bytes for fb_dft,
 * fb_dft_workspace_size(plan, rows, k_rows) for the convolutions. */
typedef struct fb_dft_plan fb_dft_plan;
int fb_dft_plan_create(fb_dft_plan** plan, int64_t n, int64_t r, int device);
int fb_dft_plan_destroy(fb_dft_plan* plan);
int fb_dft_plan_factors(const fb_dft_plan* plan, int64_t* factors, int64_t* count);
size_t fb_dft_workspace_size(const fb_dft_plan* plan, int64_t rows, int64_t k_rows);
int fb_dft(fb_dft_plan* plan, const float* x, float* y, int64_t rows, int inverse, void* workspace,
           void* stream);
int fb_conv_rows(fb_dft_plan* plan, const float* u, const float* k, float* y, int64_t N, int64_t rows,
                 int64_t k_rows, int mode, void* workspace, void* stream);
int fb_conv_rows_spectrum(fb_dft_plan* plan, const float* u, const float* kspec, float* y, int64_t N,
                          int64_t rows, int64_t k_rows, int mode, void* workspace, void* stream);
/* Learned-butterfly long convolution: the paper's extension
 * with the Butterfly matrices of the FlashButterfly transform learned.  Per
 * head h, with L(W, .) = learned_forward (butterfly.cpp:235-246) over the
 * build_plan(n, r) scaffolding and IL(W, z) = conj(L(W, conj z)) / n:
 *   y[b,h] = Re IL(Wi[h], L(Wf[h], pad u[b,h]) * L(Wf[h], pad Kbar[h]))[:N] + D[h] u[b,h]
 * n = 2N (causal) or N (circular); f32 I/O; Wf, Wi, dWf, dWi: [H][P] complex f32
 * (fb_lconv_plan_dims: P per head).  With Wf = Wi = the DFT blocks
 * (LearnedButterfly::from_plan) this equals regularized_long_conv.  The
 * backward returns du, dKbar (w.r.t. the regularized bank), dD, dWf, dWi. */
typedef struct fb_lconv_plan fb_lconv_plan;
int fb_lconv_plan_create(fb_lconv_plan** plan, int64_t N, int64_t H, int64_t r, int mode, int device);
int fb_lconv_plan_destroy(fb_lconv_plan* plan);
int fb_lconv_plan_dims(const fb_lconv_plan* plan, int64_t* n, int64_t* param_count);
size_t fb_lconv_workspace_size(const fb_lconv_plan* plan, int64_t B);
int fb_lconv_fwd(fb_lconv_plan* plan, const float* u, const float* kbar, const float* D, const float* Wf,
                 const float* Wi, float* y, int64_t B, void* workspace, void* stream);
int fb_lconv_bwd(fb_lconv_plan* plan, const float* dy, const float* u, const float* kbar, const float* D,
                 const float* Wf, const float* Wi, float* du, float* dkbar, float* dD, float* dWf,
                 float* dWi, int64_t B, void* workspace, void* stream);
const char* fb_last_error(void);
int fb_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FLASHBUTTERFLY_H */
