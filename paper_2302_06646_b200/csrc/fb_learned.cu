// FlashButterfly-B200 learned butterfly (placeholder; implemented next).
#include "fb_internal.h"
extern "C" {
int fb_learned_plan_create(fb_learned_plan** p, int64_t, int64_t, int64_t, int, int) { if (p) *p = nullptr; fb::set_error("learned: not built yet"); return FB_ERR_UNSUPPORTED; }
int fb_learned_plan_destroy(fb_learned_plan*) { return FB_OK; }
int fb_learned_plan_factors(const fb_learned_plan*, int64_t*, int64_t*, int64_t*) { return FB_ERR_UNSUPPORTED; }
size_t fb_learned_workspace_size(const fb_learned_plan*, int64_t) { return 0; }
int fb_learned_fwd(fb_learned_plan*, const float*, const void*, void*, int64_t, void*, void*) { return FB_ERR_UNSUPPORTED; }
int fb_learned_bwd(fb_learned_plan*, const float*, const void*, const void*, void*, float*, int64_t, void*, void*) { return FB_ERR_UNSUPPORTED; }
}
