// runtime.cu — C-ABI plumbing (errors, device queries, TMA descriptor
// encoding) and the host precision policy P1.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.cuh"

namespace realb {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return REALB_OK;
  set_error("%s: CUDA error %d (%s)", where, (int)e, cudaGetErrorString(e));
  return REALB_ECUDA;
}

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cached[dev] = n;
  }
  return cached[dev];
}

int set_smem_once(const void* kernel, int bytes, const char* where) {
  static std::mutex mu;
  static std::vector<std::tuple<const void*, int, int>> done;  // (kernel, device, bytes)
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  for (auto& d : done)
    if (std::get<0>(d) == kernel && std::get<1>(d) == dev && std::get<2>(d) >= bytes) return REALB_OK;
  int rc = cuda_status(
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), where);
  if (rc == REALB_OK) done.emplace_back(kernel, dev, bytes);
  return rc;
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

int make_tmap_3d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, const uint64_t dims[3],
                 const uint64_t strides_bytes[2], const uint32_t box[3], CUtensorMapSwizzle swz) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
    return REALB_ECUDA;
  }
  cuuint64_t d[3] = {dims[0], dims[1], dims[2]};
  cuuint64_t st[2] = {strides_bytes[0], strides_bytes[1]};
  cuuint32_t b[3] = {box[0], box[1], box[2]};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, dt, 3, const_cast<void*>(base), d, st, b, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (3d) failed (%d): dims=%llu,%llu,%llu box=%u,%u,%u", (int)r,
              (unsigned long long)dims[0], (unsigned long long)dims[1], (unsigned long long)dims[2], box[0], box[1],
              box[2]);
    return REALB_EINVAL;
  }
  return REALB_OK;
}

int make_tmap_2d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t inner,
                 uint64_t outer, uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
                 CUtensorMapSwizzle swz) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
    return REALB_ECUDA;
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): inner=%llu outer=%llu row_bytes=%llu box=%ux%u",
              (int)r, (unsigned long long)inner, (unsigned long long)outer,
              (unsigned long long)row_bytes, box_inner, box_outer);
    return REALB_EINVAL;
  }
  return REALB_OK;
}

}  // namespace realb

using namespace realb;

extern "C" int realb_abi_version(void) { return REALB_ABI_VERSION; }
extern "C" const char* realb_last_error(void) { return g_err; }
extern "C" int realb_num_sms(void) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, 0) != cudaSuccess) {
    cudaGetLastError();
    set_error("no CUDA device");
    return REALB_ECUDA;
  }
  return n;
}

// P1 — plan_realb (balancers.py:89-122) with the reference's fp64 op order:
//   total = sum(r.total); gate: total < threshold or total == 0 -> inactive
//   ideal = total / R;  hot: r.total / ideal > C
//   vision-heavy: total_r > 0 and v_r / total_r > M_d  (isolated: total_r > 0)
extern "C" int realb_plan(const int64_t* rank_vt, int R, double capacity_factor,
                          double modality_threshold, int64_t global_batch_threshold,
                          int modality_isolated, uint8_t* out_prec, uint8_t* out_flags) {
  if (!rank_vt || !out_prec || R < 1) {
    set_error("realb_plan: bad arguments");
    return REALB_EINVAL;
  }
  if (!(capacity_factor > 0.0) || !(modality_threshold >= 0.0 && modality_threshold <= 1.0) ||
      global_batch_threshold < 0) {
    set_error("realb_plan: invalid RealbParams");  // RealbParams.__post_init__, :42-48
    return REALB_EINVAL;
  }
  int64_t total = 0;
  for (int r = 0; r < R; ++r) {
    if (rank_vt[2 * r] < 0 || rank_vt[2 * r + 1] < 0) {
      set_error("realb_plan: token counts must be >= 0");  // RankLoad, core.py:76-78
      return REALB_EINVAL;
    }
    total += rank_vt[2 * r] + rank_vt[2 * r + 1];
  }
  for (int r = 0; r < R; ++r) {
    out_prec[r] = REALB_PREC_W16A16;
    if (out_flags) out_flags[r] = 0;
  }
  if (total < global_batch_threshold || total == 0) return 0;
  const double ideal = (double)total / (double)R;
  for (int r = 0; r < R; ++r) {
    const int64_t tr = rank_vt[2 * r] + rank_vt[2 * r + 1];
    const bool hot = (double)tr / ideal > capacity_factor;
    bool vis;
    if (modality_isolated)
      vis = tr > 0;
    else
      vis = tr > 0 && ((double)rank_vt[2 * r] / (double)tr) > modality_threshold;
    if (out_flags) out_flags[r] = (uint8_t)((hot ? 1 : 0) | (vis ? 2 : 0));
    if (hot && vis) out_prec[r] = REALB_PREC_W4A4;
  }
  return 1;
}
