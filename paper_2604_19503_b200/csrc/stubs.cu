// stubs.cu — entry points not implemented yet (return REALB_EUNSUPPORTED).
#include "common.cuh"
using namespace realb;
#define STUB(name) { set_error(#name ": not implemented in this build"); return REALB_EUNSUPPORTED; }
extern "C" int realb_grouped_gemm_nvfp4(const uint8_t*, const uint8_t*, const uint8_t*, const uint8_t*, int64_t, int, int, int, const int32_t*, int, void*, uint8_t*, uint8_t*, int, void*) STUB(realb_grouped_gemm_nvfp4)
