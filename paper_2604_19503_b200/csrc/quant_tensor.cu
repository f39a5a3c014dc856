// quant_tensor.cu — Q5/Q6 on the device: the reference's flat-tensor quantiser
// with its error summary, and the block decoder.
//
//   realb_quantize_tensor_nvfp4   quantize_tensor + ErrorSummary (fp4.py:130-170):
//       n flat values -> ceil(n/16) blocks, the last zero-padded; every block in
//       the 9-byte FP4REF01 record of pack_block (fp4.py:246-252: 8 code bytes,
//       element 2i in the low nibble, then the E4M3 scale byte), so the output is
//       the body write_blocks (fp4.py:265-270) would write. Error statistics over
//       the unpadded elements only, in fp64 as the reference computes them:
//         sums[0] += (x - d)^2, sums[1] += x^2          (fp4.py:157-162)
//         max_rel[b] = max over x != 0 of |x - d| / |x| (fp4.py:163-165)
//       The block rule is evaluated in fp64 (the reference's arithmetic) for every
//       input dtype; codes, scales and per-block max relative errors are bit-exact,
//       the two sums differ from the reference's sequential order only in the last
//       bits (device tree reduction).
//   realb_dequantize_blocks      dequantize_blocks (fp4.py:230-243): packed codes +
//       flat scale bytes -> code magnitude x decoded scale, exact in f32 and f64.
//
// Neither is on the layer's hot path (K3/K4 are); they give the W4A4 ranks'
// weight-error summary (the per-layer accuracy proxy) and the golden-file format.
#include "common.cuh"
#include "fp4_rule.cuh"

namespace realb {

template <typename T>
__device__ __forceinline__ double load_f64(const T* p, int64_t i) {
  if constexpr (sizeof(T) == 2) return (double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
  else return (double)p[i];
}

__device__ __forceinline__ double e2m1_mag(uint32_t c) {  // 0, .5, 1, 1.5, 2, 3, 4, 6
  const uint32_t m = c & 7u;
  return m < 4u ? 0.5 * (double)m : (m == 4u ? 2.0 : (m == 5u ? 3.0 : (m == 6u ? 4.0 : 6.0)));
}

template <typename T>
__global__ void __launch_bounds__(256) quant_tensor_kernel(const T* __restrict__ x, int64_t n,
                                                           uint8_t* __restrict__ rec, double* __restrict__ max_rel,
                                                           double* __restrict__ sums, int32_t* flag) {
  const int64_t nb = (n + 15) >> 4;
  double se = 0.0, sv = 0.0;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    double v[16];
    const int64_t i0 = b * 16;
    const int nreal = n - i0 < 16 ? (int)(n - i0) : 16;
    double amax = 0.0;
    bool nonfinite = false;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      v[i] = i < nreal ? load_f64(x, i0 + i) : 0.0;
      nonfinite |= !isfinite(v[i]);
      amax = fmax(amax, fabs(v[i]));
    }
    if (nonfinite) {
      if (flag) atomicOr(flag, 1);
      amax = 0.0;
    }
    const uint32_t sbits = nonfinite ? 0u : block_scale_bits_f64(amax);
    const double sc = (double)e4m3_decode(sbits);
    uint32_t lo = 0u, hi = 0u;
    double mr = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint32_t c = sbits ? e2m1_code<double>(v[i], sc) : 0u;
      if (i < 8) lo |= c << (4 * i);
      else hi |= c << (4 * (i - 8));
      const double d = (c & 8u) ? -e2m1_mag(c) * sc : e2m1_mag(c) * sc;
      if (i < nreal) {
        const double e = v[i] - d;
        se += e * e;
        sv += v[i] * v[i];
        if (v[i] != 0.0) mr = fmax(mr, fabs(e) / fabs(v[i]));
      }
    }
    uint8_t* r = rec + b * 9;
#pragma unroll
    for (int i = 0; i < 4; ++i) r[i] = (uint8_t)(lo >> (8 * i));
#pragma unroll
    for (int i = 0; i < 4; ++i) r[4 + i] = (uint8_t)(hi >> (8 * i));
    r[8] = (uint8_t)sbits;
    if (max_rel) max_rel[b] = mr;
  }
  if (sums) {
    __shared__ double red[2][8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      se += __shfl_xor_sync(0xffffffffu, se, o);
      sv += __shfl_xor_sync(0xffffffffu, sv, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { red[0][w] = se; red[1][w] = sv; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = 0.0, c = 0.0;
      for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { a += red[0][i]; c += red[1][i]; }
      atomicAdd(&sums[0], a);
      atomicAdd(&sums[1], c);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) dequant_blocks_kernel(const uint8_t* __restrict__ codes,
                                                             const uint8_t* __restrict__ sf, int64_t nb,
                                                             T* __restrict__ out) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const uint2 w = *reinterpret_cast<const uint2*>(codes + b * 8);
    const double sc = (double)e4m3_decode(sf[b]);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint32_t c = ((i < 8 ? w.x : w.y) >> (4 * (i & 7))) & 0xFu;
      const double d = (c & 8u) ? -e2m1_mag(c) * sc : e2m1_mag(c) * sc;
      out[b * 16 + i] = (T)d;
    }
  }
}

}  // namespace realb

using namespace realb;

extern "C" int realb_quantize_tensor_nvfp4(const void* d_x, int dtype, int64_t n, uint8_t* d_records,
                                           double* d_block_max_rel, double* d_sums, int32_t* d_flag,
                                           void* stream) {
  if (!d_x || !d_records || n <= 0 || (dtype != REALB_DT_BF16 && dtype != REALB_DT_F32 && dtype != REALB_DT_F64)) {
    set_error("realb_quantize_tensor_nvfp4: bad arguments (n=%lld dtype=%d)", (long long)n, dtype);
    return REALB_EINVAL;
  }
  const int64_t nb = (n + 15) / 16;
  int64_t grid = (nb + 255) / 256;
  if (grid > (int64_t)num_sms() * 8) grid = (int64_t)num_sms() * 8;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == REALB_DT_BF16)
    quant_tensor_kernel<__nv_bfloat16><<<(unsigned)grid, 256, 0, st>>>(
        reinterpret_cast<const __nv_bfloat16*>(d_x), n, d_records, d_block_max_rel, d_sums, d_flag);
  else if (dtype == REALB_DT_F32)
    quant_tensor_kernel<float><<<(unsigned)grid, 256, 0, st>>>(reinterpret_cast<const float*>(d_x), n, d_records,
                                                               d_block_max_rel, d_sums, d_flag);
  else
    quant_tensor_kernel<double><<<(unsigned)grid, 256, 0, st>>>(reinterpret_cast<const double*>(d_x), n, d_records,
                                                                d_block_max_rel, d_sums, d_flag);
  return check_launch("realb_quantize_tensor_nvfp4");
}

extern "C" int realb_dequantize_blocks(const uint8_t* d_codes, const uint8_t* d_sf, int64_t nblocks, int dtype_out,
                                       void* d_out, void* stream) {
  if (!d_codes || !d_sf || !d_out || nblocks < 0 || (dtype_out != REALB_DT_F32 && dtype_out != REALB_DT_F64)) {
    set_error("realb_dequantize_blocks: bad arguments");
    return REALB_EINVAL;
  }
  if (nblocks == 0) return REALB_OK;
  int64_t grid = (nblocks + 255) / 256;
  if (grid > (int64_t)num_sms() * 8) grid = (int64_t)num_sms() * 8;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype_out == REALB_DT_F32)
    dequant_blocks_kernel<float><<<(unsigned)grid, 256, 0, st>>>(d_codes, d_sf, nblocks, reinterpret_cast<float*>(d_out));
  else
    dequant_blocks_kernel<double><<<(unsigned)grid, 256, 0, st>>>(d_codes, d_sf, nblocks,
                                                                   reinterpret_cast<double*>(d_out));
  return check_launch("realb_dequantize_blocks");
}
