// FlashButterfly-B200 three-pass engine (placeholder; implemented next).
#include "fb_internal.h"
namespace fb {
int tp_prep(fb_plan*, const float*, cudaStream_t) { set_error("three-pass: not built yet"); return FB_ERR_UNSUPPORTED; }
int tp_fwd(fb_plan*, const void*, void*, int64_t, void*, cudaStream_t) { set_error("three-pass: not built yet"); return FB_ERR_UNSUPPORTED; }
size_t tp_workspace(const fb_plan*, int64_t) { return 256; }
int tp_bwd(fb_plan*, const void*, const void*, void*, float*, float*, float*, int64_t, void*, cudaStream_t) { set_error("three-pass: not built yet"); return FB_ERR_UNSUPPORTED; }
}
