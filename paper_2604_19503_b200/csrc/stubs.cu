// stubs.cu — entry points not implemented yet (return REALB_EUNSUPPORTED).
#include "common.cuh"
using namespace realb;
#define STUB(name) { set_error(#name ": not implemented in this build"); return REALB_EUNSUPPORTED; }
extern "C" int realb_router_topk_stats(const void*, const void*, const float*, const uint8_t*, int, int, int, int, int, float, float, float*, int32_t*, float*, int32_t*, void*) STUB(realb_router_topk_stats)
extern "C" int64_t realb_layout_words(int E, int nchunks) { return LayoutView::words(E, nchunks); }
extern "C" int realb_moe_align(const int32_t*, int, int, const uint8_t*, int32_t*, int32_t*, void*) STUB(realb_moe_align)
extern "C" int realb_dispatch_permute(const void*, const int32_t*, int, int, int, int, const uint8_t*, const int32_t*, int, int64_t, int32_t*, void*, uint8_t*, uint8_t*, int32_t*, void*) STUB(realb_dispatch_permute)
extern "C" int realb_grouped_gemm_nvfp4(const uint8_t*, const uint8_t*, const uint8_t*, const uint8_t*, int64_t, int, int, int, const int32_t*, int, void*, uint8_t*, uint8_t*, int, void*) STUB(realb_grouped_gemm_nvfp4)
extern "C" int realb_combine(const void*, const int32_t*, const float*, int, int, int, void*, void*) STUB(realb_combine)
