// quant.cu — K3: on-the-fly BF16 -> NVFP4 weight quantiser (also used for the
// fp32/fp64 parity path). HBM-bound: 2.5625 B/element for bf16 input
// (2 read + 0.5 codes + 0.0625 scale).
//
// Work unit = a 128-row x 4-block (64-column) tile: exactly one 512-byte
// scale-factor atom of the tcgen05 block-scale layout, so the atom is written
// as one contiguous, coalesced 512-byte run. Thread -> (row = b / 4,
// kb = b % 4): four consecutive threads read one row's 128 contiguous input
// bytes (bf16) and write its 32 contiguous code bytes.
#include "common.cuh"
#include "fp4_rule.cuh"

namespace realb {

template <typename T>
struct Loader;

template <>
struct Loader<__nv_bfloat16> {
  static __device__ __forceinline__ void load16(const __nv_bfloat16* p, float (&v)[16]) {
    const uint4* q = reinterpret_cast<const uint4*>(p);
    uint4 a = __ldg(q), b = __ldg(q + 1);
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
};
template <>
struct Loader<float> {
  static __device__ __forceinline__ void load16(const float* p, float (&v)[16]) {
    const float4* q = reinterpret_cast<const float4*>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float4 t = __ldg(q + i);
      v[4 * i] = t.x; v[4 * i + 1] = t.y; v[4 * i + 2] = t.z; v[4 * i + 3] = t.w;
    }
  }
};

__device__ __forceinline__ void flag_nonfinite(int32_t* flag) {
  if (flag) atomicOr(flag, 1);
}

// One 128-row x 64-column tile (one 512-B scale atom) of a bf16 matrix: each
// thread quantises 2 blocks, both loads issued before any compute. Non-finite
// input is detected from the block amax bits (|bits| >= 0x7F80).
template <int LAYOUT>
__device__ __forceinline__ void quant_tile_bf16(const __nv_bfloat16* __restrict__ x, int64_t rows,
                                                int64_t cols, int64_t nkb, int64_t tm, int64_t tk,
                                                uint8_t* __restrict__ codes,
                                                uint8_t* __restrict__ sf, int32_t* flag,
                                                const float2* tab) {
  // thread -> (row r0 + 64h, k-block kb): the two blocks are 64 rows apart
  const int r_in = threadIdx.x >> 2, kq = threadIdx.x & 3;
  const int64_t r0 = tm * 128 + r_in, kb = tk * 4 + kq;
  const bool kok = kb < nkb;
  const __nv_bfloat16* xp = x + r0 * cols + kb * 16;
  const int64_t xstep = 64 * cols;
  uint32_t w[2][8];
  bool ok[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    ok[h] = kok && r0 + 64 * h < rows;
    if (ok[h]) {
      const uint4* q = reinterpret_cast<const uint4*>(xp + h * xstep);
      const uint4 a = __ldg(q), c = __ldg(q + 1);
      w[h][0] = a.x; w[h][1] = a.y; w[h][2] = a.z; w[h][3] = a.w;
      w[h][4] = c.x; w[h][5] = c.y; w[h][6] = c.z; w[h][7] = c.w;
    }
  }
  uint8_t* cp = codes + r0 * (cols >> 1) + kb * 8;
  const int64_t cstep = 64 * (cols >> 1);
  // MMA layout: rows r and r+64 land in the same 512-B atom, byte +8 apart
  const int64_t so0 = LAYOUT == REALB_SF_FLAT ? r0 * nkb + kb : sf_mma_offset(r0, kb, nkb);
  const int64_t sstep = LAYOUT == REALB_SF_FLAT ? 64 * nkb : 8;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (!ok[h]) continue;
    uint32_t sbits;
    bool nf;
    const uint2 c = quant_block16_bf16_tab(w[h], sbits, nf, tab);
    if (nf) flag_nonfinite(flag);
    *reinterpret_cast<uint2*>(cp + h * cstep) = c;
    sf[so0 + h * sstep] = (uint8_t)sbits;
  }
}

template <int LAYOUT>
__global__ void __launch_bounds__(256) quant_kernel_bf16(const __nv_bfloat16* __restrict__ x,
                                                          int64_t rows, int64_t cols,
                                                          uint8_t* __restrict__ codes,
                                                          uint8_t* __restrict__ sf, int32_t* flag) {
  __shared__ float2 tab[128];
  sf_table_init(tab);
  __syncthreads();
  const int64_t nkb = cols >> 4;
  const int tiles_k = (int)((nkb + 3) >> 2);
  const int tiles = (int)((rows + 127) >> 7) * tiles_k;
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int tm = tile / tiles_k, tk = tile - tm * tiles_k;
    quant_tile_bf16<LAYOUT>(x, rows, cols, nkb, tm, tk, codes, sf, flag, tab);
  }
}

// K3 on the device-side plan: quantise only the rows of experts whose
// precision code is W4A4 (rows_per_expert % 128 == 0, so a tile never straddles
// two experts); MMA scale layout.
__global__ void __launch_bounds__(256) quant_experts_kernel(
    const __nv_bfloat16* __restrict__ x, int64_t rows_per_expert, int64_t cols, int E,
    const uint8_t* __restrict__ prec, uint8_t* __restrict__ codes, uint8_t* __restrict__ sf,
    int32_t* flag) {
  const int64_t nkb = cols >> 4;
  const int tiles_k = (int)(nkb >> 2);
  const int mt_per_expert = (int)(rows_per_expert >> 7);
  const int tiles_per_expert = mt_per_expert * tiles_k;
  // enumerate only the W4A4 experts' tiles: tile -> (j-th W4A4 expert, local tile)
  __shared__ int s_list[256];
  __shared__ int s_n;
  __shared__ float2 tab[128];
  sf_table_init(tab);
  if (threadIdx.x == 0) {
    int n = 0;
    for (int e = 0; e < E; ++e)
      if (prec[e] == REALB_PREC_W4A4) s_list[n++] = e;
    s_n = n;
  }
  __syncthreads();
  const int tiles = s_n * tiles_per_expert;
  const int64_t rows = (int64_t)E * rows_per_expert;
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int j = tile / tiles_per_expert, lt = tile - j * tiles_per_expert;
    const int lm = lt / tiles_k;
    quant_tile_bf16<REALB_SF_MMA128x4>(x, rows, cols, nkb, (int64_t)s_list[j] * mt_per_expert + lm,
                                        lt - lm * tiles_k, codes, sf, flag, tab);
  }
}

// resident CTAs per SM x SMs (no partial last wave); capped by the work
static int quant_grid(const void* kern, int64_t tiles, int max_ctas) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    per_sm = 4;
  }
  int64_t grid = (int64_t)num_sms() * per_sm;
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  if (grid > tiles) grid = tiles;
  return (int)(grid < 1 ? 1 : grid);
}

template <typename T, int LAYOUT>
__global__ void __launch_bounds__(256) quant_kernel(const T* __restrict__ x, int64_t rows,
                                                     int64_t cols, uint8_t* __restrict__ codes,
                                                     uint8_t* __restrict__ sf, int32_t* flag) {
  const int64_t nkb = cols >> 4;
  const int64_t tiles_k = (nkb + 3) >> 2;
  const int64_t tiles = ((rows + 127) >> 7) * tiles_k;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t tm = tile / tiles_k, tk = tile - tm * tiles_k;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int b = threadIdx.x + half * 256;
      const int64_t r = tm * 128 + (b >> 2);
      const int64_t kb = tk * 4 + (b & 3);
      if (r >= rows || kb >= nkb) continue;
      float v[16];
      Loader<T>::load16(x + r * cols + kb * 16, v);
      bool finite = true;
#pragma unroll
      for (int i = 0; i < 16; ++i) finite &= isfinite(v[i]);
      if (!finite) flag_nonfinite(flag);
      uint32_t sbits;
      uint2 c = quant_block16_f32(v, sbits);
      *reinterpret_cast<uint2*>(codes + r * (cols >> 1) + kb * 8) = c;
      const int64_t so = LAYOUT == REALB_SF_FLAT ? r * nkb + kb : sf_mma_offset(r, kb, nkb);
      sf[so] = (uint8_t)sbits;
    }
  }
}

// fp64 input: the reference's own arithmetic width (parity path only).
template <int LAYOUT>
__global__ void __launch_bounds__(256) quant_kernel_f64(const double* __restrict__ x, int64_t rows,
                                                         int64_t cols, uint8_t* __restrict__ codes,
                                                         uint8_t* __restrict__ sf, int32_t* flag) {
  const int64_t nkb = cols >> 4;
  const int64_t tiles_k = (nkb + 3) >> 2;
  const int64_t tiles = ((rows + 127) >> 7) * tiles_k;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t tm = tile / tiles_k, tk = tile - tm * tiles_k;
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
      const int b = threadIdx.x + half * 256;
      const int64_t r = tm * 128 + (b >> 2);
      const int64_t kb = tk * 4 + (b & 3);
      if (r >= rows || kb >= nkb) continue;
      const double2* q = reinterpret_cast<const double2*>(x + r * cols + kb * 16);
      double v[16];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        double2 t = __ldg(q + i);
        v[2 * i] = t.x; v[2 * i + 1] = t.y;
      }
      double amax = 0.0;
      bool finite = true;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        finite &= isfinite(v[i]);
        amax = fmax(amax, fabs(v[i]));
      }
      if (!finite) flag_nonfinite(flag);
      const uint32_t sbits = block_scale_bits_f64(amax);
      uint2 c = make_uint2(0u, 0u);
      if (sbits) {
        const double sc = (double)e4m3_decode(sbits);
#pragma unroll
        for (int i = 0; i < 8; ++i) c.x |= e2m1_code<double>(v[i], sc) << (4 * i);
#pragma unroll
        for (int i = 0; i < 8; ++i) c.y |= e2m1_code<double>(v[8 + i], sc) << (4 * i);
      }
      *reinterpret_cast<uint2*>(codes + r * (cols >> 1) + kb * 8) = c;
      const int64_t so = LAYOUT == REALB_SF_FLAT ? r * nkb + kb : sf_mma_offset(r, kb, nkb);
      sf[so] = (uint8_t)sbits;
    }
  }
}

template <typename T>
static int launch_quant(void (*kernel)(const T*, int64_t, int64_t, uint8_t*, uint8_t*, int32_t*),
                        const void* x, int64_t rows, int64_t cols, uint8_t* codes,
                        uint8_t* sf, int32_t* flag, int max_ctas, cudaStream_t st) {
  const int64_t tiles = ((rows + 127) / 128) * (((cols / 16) + 3) / 4);
  if (tiles < 1) return REALB_OK;
  const int grid = quant_grid(reinterpret_cast<const void*>(kernel), tiles, max_ctas);
  kernel<<<(unsigned)grid, 256, 0, st>>>(static_cast<const T*>(x), rows, cols, codes, sf, flag);
  return check_launch("realb_quantize_nvfp4");
}

}  // namespace realb

using namespace realb;

extern "C" int realb_quantize_nvfp4(const void* d_x, int dtype, int64_t rows, int64_t cols,
                                    uint8_t* d_codes, uint8_t* d_sf, int sf_layout,
                                    int32_t* d_flag, int max_ctas, void* stream) {
  if (!d_x || !d_codes || !d_sf || rows < 0 || cols <= 0 || cols % 16) {
    set_error("realb_quantize_nvfp4: bad arguments (rows=%lld cols=%lld; cols must be a "
              "positive multiple of 16)", (long long)rows, (long long)cols);
    return REALB_EINVAL;
  }
  if (sf_layout != REALB_SF_FLAT && sf_layout != REALB_SF_MMA128x4) {
    set_error("realb_quantize_nvfp4: unknown sf_layout %d", sf_layout);
    return REALB_EINVAL;
  }
  if (sf_layout == REALB_SF_MMA128x4 && (rows % 128 || cols % 64)) {
    set_error("realb_quantize_nvfp4: MMA scale layout needs rows%%128==0 and cols%%64==0 "
              "(rows=%lld cols=%lld)", (long long)rows, (long long)cols);
    return REALB_EINVAL;
  }
  if (rows == 0) return REALB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const bool flat = sf_layout == REALB_SF_FLAT;
  switch (dtype) {
    case REALB_DT_BF16:
      return flat ? launch_quant(quant_kernel_bf16<REALB_SF_FLAT>, d_x, rows, cols, d_codes,
                                 d_sf, d_flag, max_ctas, st)
                  : launch_quant(quant_kernel_bf16<REALB_SF_MMA128x4>, d_x, rows, cols, d_codes,
                                 d_sf, d_flag, max_ctas, st);
    case REALB_DT_F32:
      return flat ? launch_quant(quant_kernel<float, REALB_SF_FLAT>, d_x, rows, cols, d_codes,
                                 d_sf, d_flag, max_ctas, st)
                  : launch_quant(quant_kernel<float, REALB_SF_MMA128x4>, d_x, rows, cols, d_codes,
                                 d_sf, d_flag, max_ctas, st);
    case REALB_DT_F64:
      return flat ? launch_quant(quant_kernel_f64<REALB_SF_FLAT>, d_x, rows, cols, d_codes, d_sf,
                                 d_flag, max_ctas, st)
                  : launch_quant(quant_kernel_f64<REALB_SF_MMA128x4>, d_x, rows, cols, d_codes,
                                 d_sf, d_flag, max_ctas, st);
    default:
      set_error("realb_quantize_nvfp4: unknown dtype %d", dtype);
      return REALB_EINVAL;
  }
}

extern "C" int realb_quantize_experts_nvfp4(const void* d_w, int E, int64_t rows_per_expert,
                                            int64_t cols, const uint8_t* d_expert_prec,
                                            uint8_t* d_codes, uint8_t* d_sf, int32_t* d_flag,
                                            int max_ctas, void* stream) {
  if (!d_w || !d_expert_prec || !d_codes || !d_sf || E < 1 || E > 256 || rows_per_expert <= 0 ||
      rows_per_expert % 128 || cols <= 0 || cols % 64) {
    set_error("realb_quantize_experts_nvfp4: bad arguments (E=%d rows/expert=%lld cols=%lld)", E,
              (long long)rows_per_expert, (long long)cols);
    return REALB_EINVAL;
  }
  const int grid = quant_grid(reinterpret_cast<const void*>(quant_experts_kernel),
                             (int64_t)E * (rows_per_expert / 128) * (cols / 64), max_ctas);
  quant_experts_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const __nv_bfloat16*>(d_w), rows_per_expert, cols, E, d_expert_prec,
      d_codes, d_sf, d_flag);
  return check_launch("realb_quantize_experts_nvfp4");
}
