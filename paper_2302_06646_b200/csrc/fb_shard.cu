// FlashButterfly-B200: the all-to-all staging layouts of the
// sequence-sharded four-step layer (config 5-4M, paper_2302_06646_b200/
// seqshard.py), optionally bf16 on the wire.  (The batch-pair packing and the
// unpack with the skip D u are fused into the column passes, fb_three.cu:
// fb_shard_columns_from_signals / _to_signals.)  The reference's analogue is the
// three-pass data flow of three_pass.cpp:225-254 (the mixer passes gather /
// scatter whole columns; here the columns live on different GPUs).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "fb_common.cuh"
#include "fb_internal.h"

namespace fb {
namespace {

unsigned blocks_for(int64_t count) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, 148 * 32));
}

// out[b][a][x] = in[a][b][x] on complex elements, f32 or bf16 pairs either side
template <typename TI, typename TO>
__global__ void stage_kernel(const TI* __restrict__ in, TO* __restrict__ out, int64_t A, int64_t Bd,
                             int64_t X) {
  const int64_t count = A * Bd * X;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = i % X, a = (i / X) % A, b = i / (X * A);
    const float2 v = ldc_any<typename TI::elem>(&in[(a * Bd + b) * X + x].v);
    stc<typename TO::elem>(&out[i].v, v);
  }
}
struct CF32 {
  using elem = float;
  float v, w;
};
struct CBF16 {
  using elem = __nv_bfloat16;
  __nv_bfloat16 v, w;
};

}  // namespace
}  // namespace fb

using namespace fb;

extern "C" {

int fb_shard_stage(const void* in, void* out, int64_t A, int64_t Bd, int64_t X, int in_dtype, int out_dtype,
                   void* stream) {
  if (!in || !out || A < 1 || Bd < 1 || X < 1 || (in_dtype != FB_F32 && in_dtype != FB_BF16) ||
      (out_dtype != FB_F32 && out_dtype != FB_BF16)) {
    set_error("fb_shard_stage: bad arguments");
    return FB_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned g = blocks_for(A * Bd * X);
  if (in_dtype == FB_F32 && out_dtype == FB_F32)
    stage_kernel<CF32, CF32><<<g, 256, 0, s>>>((const CF32*)in, (CF32*)out, A, Bd, X);
  else if (in_dtype == FB_F32)
    stage_kernel<CF32, CBF16><<<g, 256, 0, s>>>((const CF32*)in, (CBF16*)out, A, Bd, X);
  else if (out_dtype == FB_F32)
    stage_kernel<CBF16, CF32><<<g, 256, 0, s>>>((const CBF16*)in, (CF32*)out, A, Bd, X);
  else
    stage_kernel<CBF16, CBF16><<<g, 256, 0, s>>>((const CBF16*)in, (CBF16*)out, A, Bd, X);
  return cuda_status(cudaGetLastError(), "fb_shard_stage");
}

}  // extern "C"
