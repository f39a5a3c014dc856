// fp4_rule.cuh — the reference NVFP4 block rule, restated for the device with
// exact arithmetic (no division on elements), bit-exact with
// moesim.fp4.quantize_blocks (fp4.py:173-227) / quantize_block (fp4.py:108-122).
//
//   scale_bits = E4M3_RNE(amax / 6)   (encode_e4m3, fp4.py:36-56; sat 448 -> 0x7E)
//   amax == 0  -> scale 0, all codes 0           (fp4.py:115-116)
//   scale_bits == 0 for a nonzero block -> 1     (fp4.py:118-119)
//   code = nearest E2M1 magnitude of v / scale, ties to the even index,
//          no negative zero                      (fp4.py:69-82, :222-226)
//
// Element codes: instead of dividing, |v| is compared with the exact products
// mid_i * scale (mid_i in {0.25,0.75,1.25,1.75,2.5,3.5,5}; scale has <= 4
// significant bits so every product is exact in fp32/fp64). For even i the
// test is strict (>), for odd i it is (>=): that is the reference's
// searchsorted(side="left") plus its odd-index tie bump. The reference's own
// fp64 quotient can never round onto a midpoint it does not equal (DESIGN.md
// §Q), so the comparisons are equivalent.
#pragma once
#include <stdint.h>

namespace realb {

// E4M3 decode (decode_e4m3, fp4.py:59-66); exact in fp32.
__device__ __forceinline__ float e4m3_decode(uint32_t bits) {
  uint32_t e = bits >> 3, m = bits & 7u;
  if (e == 0) return (float)m * 0.001953125f;  // m * 2^-9
  // (1 + m/8) * 2^(e-7): build the fp32 directly
  uint32_t fb = ((e - 7u + 127u) << 23) | (m << 20);
  return __uint_as_float(fb);
}

// E4M3 round-to-nearest-even of a non-negative fp32 x, saturating at 448
// (encode_e4m3, fp4.py:36-56), integer-exact.
__device__ __forceinline__ uint32_t e4m3_encode_f32(float x) {
  if (x >= 448.0f) return 0x7Eu;
  if (x < 0.015625f) {  // subnormal: m = rint(x / 2^-9), exact scaling
    float m = rintf(x * 512.0f);
    return m >= 8.0f ? 0x08u : (uint32_t)m;
  }
  uint32_t b = __float_as_uint(x);
  int e = (int)((b >> 23) & 0xFF) - 127;
  uint32_t mant = b & 0x7FFFFFu;
  uint32_t m = mant >> 20, rem = mant & 0xFFFFFu;
  if (rem > 0x80000u || (rem == 0x80000u && (m & 1u))) m += 1;
  if (m == 8u) { m = 0; e += 1; }
  if (e > 8 || (e == 8 && m > 6u)) return 0x7Eu;
  return ((uint32_t)(e + 7) << 3) | m;
}

// Same rule on an fp64 value (the reference computes in float64; used for
// fp64 inputs whose amax is not exactly representable in fp32).
__device__ __forceinline__ uint32_t e4m3_encode_f64(double x) {
  if (x >= 448.0) return 0x7Eu;
  if (x < 0.015625) {
    double m = rint(x * 512.0);
    return m >= 8.0 ? 0x08u : (uint32_t)m;
  }
  unsigned long long b = __double_as_longlong(x);
  int e = (int)((b >> 52) & 0x7FF) - 1023;
  unsigned long long mant = b & 0xFFFFFFFFFFFFFull;
  uint32_t m = (uint32_t)(mant >> 49);
  unsigned long long rem = mant & ((1ull << 49) - 1);
  const unsigned long long half = 1ull << 48;
  if (rem > half || (rem == half && (m & 1u))) m += 1;
  if (m == 8u) { m = 0; e += 1; }
  if (e > 8 || (e == 8 && m > 6u)) return 0x7Eu;
  return ((uint32_t)(e + 7) << 3) | m;
}

// block scale bits from amax (fp32 path: amax exactly representable in fp32)
__device__ __forceinline__ uint32_t block_scale_bits_f32(float amax) {
  if (amax == 0.0f) return 0u;
  uint32_t s = e4m3_encode_f32(__fdiv_rn(amax, 6.0f));  // IEEE division, DESIGN.md §Q
  return s == 0u ? 1u : s;
}
// Same for a bf16-representable amax without the IEEE-division slow path:
// q = amax * rn(1/6) refined by one FMA residual step is the correctly rounded
// amax / 6 for normal results; results below 2^-10 (where subnormal rounding
// could differ) all encode to scale bits 0 -> 1 regardless. Verified over every
// positive finite bf16 amax (tests/test_quant_gpu.py::test_all_bf16_amax_bf16_path).
__device__ __forceinline__ uint32_t block_scale_bits_bf16amax(float amax) {
  if (amax == 0.0f) return 0u;
  const float r6 = 0.16666667163372039794921875f;  // rn(1/6)
  const float q0 = amax * r6;
  const float q = fmaf(fmaf(-q0, 6.0f, amax), r6, q0);
  uint32_t s = e4m3_encode_f32(q);
  return s == 0u ? 1u : s;
}
__device__ __forceinline__ uint32_t block_scale_bits_f64(double amax) {
  if (amax == 0.0) return 0u;
  uint32_t s = e4m3_encode_f64(__ddiv_rn(amax, 6.0));
  return s == 0u ? 1u : s;
}

// E2M1 code of v for a block with decoded scale `sc` (> 0).
template <typename F>
__device__ __forceinline__ uint32_t e2m1_code(F v, F sc) {
  F mag = v < F(0) ? -v : v;
  uint32_t idx = (uint32_t)(mag > F(0.25) * sc) + (uint32_t)(mag >= F(0.75) * sc) +
                 (uint32_t)(mag > F(1.25) * sc) + (uint32_t)(mag >= F(1.75) * sc) +
                 (uint32_t)(mag > F(2.5) * sc) + (uint32_t)(mag >= F(3.5) * sc) +
                 (uint32_t)(mag > F(5.0) * sc);
  return (v < F(0) && idx > 0u) ? (idx | 8u) : idx;
}

// Quantise 16 fp32 values (one block). Returns packed codes (element 2i in the
// low nibble of byte i) as two 32-bit words; writes the scale bits.
__device__ __forceinline__ uint2 quant_block16_f32(const float (&v)[16], uint32_t& sbits) {
  float amax = 0.0f;
#pragma unroll
  for (int i = 0; i < 16; ++i) amax = fmaxf(amax, fabsf(v[i]));
  sbits = block_scale_bits_f32(amax);
  uint2 out = make_uint2(0u, 0u);
  if (sbits != 0u) {
    const float sc = e4m3_decode(sbits);
#pragma unroll
    for (int i = 0; i < 8; ++i) out.x |= e2m1_code<float>(v[i], sc) << (4 * i);
#pragma unroll
    for (int i = 0; i < 8; ++i) out.y |= e2m1_code<float>(v[8 + i], sc) << (4 * i);
  }
  return out;
}

// ---------------------------------------------------------------------------
// bf16 fast path (the product path: weights, activations, SwiGLU output).
// For bf16 inputs (8 significant bits) and E4M3 scales (4 bits) the quotient
// v / scale is either exactly an E2M1 rounding midpoint or at least 2^-9
// (relative) away from every midpoint. q1 = q0 + (v - q0*sc) * rcp(sc) with
// q0 = v * rcp(sc) is exact at the midpoints and within a few fp32 ulps
// elsewhere, so the hardware RNE conversion cvt.rn.satfinite.e2m1x2.f32 of q1
// reproduces the reference's ties-to-even-index decision (verified over the
// exhaustive bf16 x scale table, tests/test_quant_gpu.py). The conversion can
// emit negative zero (0x8); it is canonicalised to 0 (fp4.py:80-81).
__device__ __forceinline__ uint32_t cvt_e2m1x4(float a0, float a1, float a2, float a3) {
  uint32_t out;
  asm("{\n\t.reg .b8 b0, b1;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b0, %2, %1;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b1, %4, %3;\n\t"
      "mov.b32 %0, {b0, b1, 0, 0};\n\t}"
      : "=r"(out)
      : "f"(a0), "f"(a1), "f"(a2), "f"(a3));
  return out;
}
// 8 nibbles: any code with zero magnitude becomes +0
__device__ __forceinline__ uint32_t canon_neg_zero(uint32_t x) {
  const uint32_t mag = x & 0x77777777u;
  const uint32_t nz = (mag + 0x77777777u) & 0x88888888u;  // bit 3 of a nibble set iff mag != 0
  return mag | (x & nz);
}
__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// amax of 16 bf16 values held as 8 bf16x2 words (exact: integer max of |bits|).
// Returns the 16-bit magnitude pattern; >= 0x7F80 means an Inf/NaN is present.
__device__ __forceinline__ uint32_t amax_bits_bf16x16(const uint32_t (&w)[8]) {
  uint32_t m = w[0] & 0x7FFF7FFFu;
#pragma unroll
  for (int i = 1; i < 8; ++i) {
    const uint32_t a = w[i] & 0x7FFF7FFFu;
    asm("max.u16x2 %0, %0, %1;" : "+r"(m) : "r"(a));
  }
  const uint32_t lo = m & 0xFFFFu, hi = m >> 16;
  return lo > hi ? lo : hi;
}
__device__ __forceinline__ float amax_bf16x16(const uint32_t (&w)[8]) {
  return __uint_as_float(amax_bits_bf16x16(w) << 16);
}

__device__ __forceinline__ float q1_div(float v, float sc, float r) {
  const float q0 = v * r;
  const float rho = fmaf(-q0, sc, v);
  return fmaf(rho, r, q0);
}

// one block of 16 bf16 (8 words) -> packed codes (element 2i low nibble), scale bits;
// `nonfinite` is set when the block holds an Inf/NaN (QuantizationDomainError)
__device__ __forceinline__ uint2 quant_block16_bf16(const uint32_t (&w)[8], uint32_t& sbits,
                                                    bool& nonfinite) {
  const uint32_t ab = amax_bits_bf16x16(w);
  nonfinite = ab >= 0x7F80u;
  const float amax = __uint_as_float(ab << 16);
  sbits = block_scale_bits_bf16amax(amax);
  if (sbits == 0u) return make_uint2(0u, 0u);
  const float sc = e4m3_decode(sbits);
  const float r = __frcp_rn(sc);
  uint32_t c[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    c[i] = cvt_e2m1x4(q1_div(bf16lo(w[2 * i]), sc, r), q1_div(bf16hi(w[2 * i]), sc, r),
                      q1_div(bf16lo(w[2 * i + 1]), sc, r), q1_div(bf16hi(w[2 * i + 1]), sc, r));
  return make_uint2(canon_neg_zero(c[0] | (c[1] << 16)), canon_neg_zero(c[2] | (c[3] << 16)));
}

// quant_block16_bf16 with the decoded scale and its correctly rounded reciprocal
// taken from a 128-entry (scale bits -> (sc, rn(1/sc))) table in shared memory
// (sf_table_init): the same arithmetic, ~20 fewer instructions per block for the
// HBM-bound weight quantiser.
__device__ __forceinline__ void sf_table_init(float2* tab) {
  for (int i = threadIdx.x; i < 128; i += blockDim.x) {
    const float sc = e4m3_decode((uint32_t)i);
    tab[i] = make_float2(sc, i ? __frcp_rn(sc) : 0.0f);
  }
}
__device__ __forceinline__ uint2 quant_block16_bf16_tab(const uint32_t (&w)[8], uint32_t& sbits,
                                                        bool& nonfinite, const float2* tab) {
  const uint32_t ab = amax_bits_bf16x16(w);
  nonfinite = ab >= 0x7F80u;
  const float amax = __uint_as_float(ab << 16);
  sbits = block_scale_bits_bf16amax(amax);
  if (sbits == 0u) return make_uint2(0u, 0u);
  const float2 t = tab[sbits];
  const float sc = t.x, r = t.y;
  uint32_t c[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    c[i] = cvt_e2m1x4(q1_div(bf16lo(w[2 * i]), sc, r), q1_div(bf16hi(w[2 * i]), sc, r),
                      q1_div(bf16lo(w[2 * i + 1]), sc, r), q1_div(bf16hi(w[2 * i + 1]), sc, r));
  return make_uint2(canon_neg_zero(c[0] | (c[1] << 16)), canon_neg_zero(c[2] | (c[3] << 16)));
}

// same for 16 fp32 values that are known to be bf16-representable
__device__ __forceinline__ uint2 quant_block16_bf16vals(const float (&v)[16], uint32_t& sbits) {
  float amax = 0.0f;
#pragma unroll
  for (int i = 0; i < 16; ++i) amax = fmaxf(amax, fabsf(v[i]));
  sbits = block_scale_bits_bf16amax(amax);
  if (sbits == 0u) return make_uint2(0u, 0u);
  const float sc = e4m3_decode(sbits);
  const float r = __frcp_rn(sc);
  uint32_t c[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    c[i] = cvt_e2m1x4(q1_div(v[4 * i], sc, r), q1_div(v[4 * i + 1], sc, r),
                      q1_div(v[4 * i + 2], sc, r), q1_div(v[4 * i + 3], sc, r));
  return make_uint2(canon_neg_zero(c[0] | (c[1] << 16)), canon_neg_zero(c[2] | (c[3] << 16)));
}

// ---------------------------------------------------------------------------
// Packed-FP32 (FFMA2 / FMUL2, sm_100) form of quant_block16_bf16_tab: the same
// q1 = q0 + (v - q0*sc) * r residual step, two elements per instruction.
__device__ __forceinline__ uint64_t f32x2_pack(float lo, float hi) {
  return ((uint64_t)__float_as_uint(hi) << 32) | __float_as_uint(lo);
}
// one bf16x2 word -> the f32x2 pair (lo element, hi element)
__device__ __forceinline__ uint64_t bf16x2_to_f32x2(uint32_t w) {
  return ((uint64_t)(w & 0xFFFF0000u) << 32) | (uint64_t)(w << 16);
}
__device__ __forceinline__ uint64_t q1_div2(uint64_t v, uint64_t r2, uint64_t nsc2) {
  uint64_t q0, rho, q1;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(q0) : "l"(v), "l"(r2));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rho) : "l"(q0), "l"(nsc2), "l"(v));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(q1) : "l"(rho), "l"(r2), "l"(q0));
  return q1;
}
// two f32x2 quotients (4 elements, in order) -> 4 E2M1 codes in the low 16 bits
__device__ __forceinline__ uint32_t cvt_e2m1x4_2(uint64_t a, uint64_t b) {
  uint32_t out;
  asm("{\n\t.reg .b8 b0, b1;\n\t.reg .f32 a0, a1, a2, a3;\n\t"
      "mov.b64 {a0, a1}, %1;\n\tmov.b64 {a2, a3}, %2;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b0, a1, a0;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b1, a3, a2;\n\t"
      "mov.b32 %0, {b0, b1, 0, 0};\n\t}"
      : "=r"(out)
      : "l"(a), "l"(b));
  return out;
}
// E4M3 scale bits by the hardware conversion: cvt.rn.satfinite.e4m3x2.f32 is RNE
// with subnormals and saturation at 448 (0x7E), i.e. encode_e4m3 (fp4.py:36-56)
// for every non-negative finite input (checked over every bf16 amax,
// tests/test_quant_gpu.py::test_all_bf16_amax_bf16_path); nonzero -> at least 1.
__device__ __forceinline__ uint32_t block_scale_bits_bf16amax_hw(float amax) {
  const float r6 = 0.16666667163372039794921875f;  // rn(1/6)
  const float q0 = amax * r6;
  const float q = fmaf(fmaf(-q0, 6.0f, amax), r6, q0);  // rn(amax / 6) for bf16 amax
  uint16_t h;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %1;" : "=h"(h) : "f"(q));
  const uint32_t b = h & 0xFFu;
  return (b == 0u && amax > 0.0f) ? 1u : b;
}

__device__ __forceinline__ uint2 quant_block16_bf16_x2(const uint32_t (&w)[8], uint32_t& sbits,
                                                       bool& nonfinite, const float2* tab) {
  const uint32_t ab = amax_bits_bf16x16(w);
  nonfinite = ab >= 0x7F80u;
  sbits = block_scale_bits_bf16amax_hw(__uint_as_float(ab << 16));
  if (sbits == 0u) return make_uint2(0u, 0u);
  const float2 t = tab[sbits];
  const uint64_t r2 = f32x2_pack(t.y, t.y), nsc2 = f32x2_pack(-t.x, -t.x);
  uint32_t c[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    c[i] = cvt_e2m1x4_2(q1_div2(bf16x2_to_f32x2(w[2 * i]), r2, nsc2),
                        q1_div2(bf16x2_to_f32x2(w[2 * i + 1]), r2, nsc2));
  return make_uint2(canon_neg_zero(c[0] | (c[1] << 16)), canon_neg_zero(c[2] | (c[3] << 16)));
}

// byte offset of scale (row r, k-block kb) in the REALB_SF_MMA128x4 layout
__host__ __device__ __forceinline__ int64_t sf_mma_offset(int64_t r, int64_t kb, int64_t nkb) {
  const int64_t atom = (r >> 7) * (nkb >> 2) + (kb >> 2);
  return atom * 512 + (r & 31) * 16 + ((r >> 5) & 3) * 4 + (kb & 3);
}


// ---------------------------------------------------------------------------
// Correctly rounded reciprocals of every E4M3 scale, computed at compile time
// (IEEE float division in the constant evaluator; equal to __frcp_rn for all 127
// nonzero scale codes, checked against numpy's float32 division when this table was
// written): the activation-side rule (K4 producers, the K6 SwiGLU re-quantisation)
// reads it instead of evaluating __frcp_rn, an IEEE multi-instruction sequence.
struct E4M3Rcp {
  float v[128];
};
constexpr float e4m3_decode_ce(uint32_t b) {
  const uint32_t e = b >> 3, m = b & 7u;
  if (e == 0) return (float)m * 0.001953125f;
  float f = 1.0f + (float)m * 0.125f;
  for (int i = 7; i < (int)e; ++i) f *= 2.0f;
  for (int i = (int)e; i < 7; ++i) f *= 0.5f;
  return f;
}
constexpr E4M3Rcp make_e4m3_rcp() {
  E4M3Rcp t{};
  for (uint32_t b = 1; b < 128; ++b) t.v[b] = 1.0f / e4m3_decode_ce(b);
  return t;
}
static __device__ const E4M3Rcp g_e4m3_rcp = make_e4m3_rcp();

// the block rule on 8 packed pairs (f32x2: element 2i low, 2i+1 high) of
// bf16-representable values whose amax bits are known: hardware scale encode,
// table reciprocal, packed-FP32 residual step, hardware E2M1 conversion
__device__ __forceinline__ uint2 quant_block16_pairs(const uint64_t (&p)[8], float amax, uint32_t& sbits) {
  sbits = block_scale_bits_bf16amax_hw(amax);
  if (sbits == 0u) return make_uint2(0u, 0u);
  const float sc = e4m3_decode(sbits);
  const float r = __ldg(&g_e4m3_rcp.v[sbits]);
  const uint64_t r2 = f32x2_pack(r, r), nsc2 = f32x2_pack(-sc, -sc);
  uint32_t c[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i] = cvt_e2m1x4_2(q1_div2(p[2 * i], r2, nsc2), q1_div2(p[2 * i + 1], r2, nsc2));
  return make_uint2(canon_neg_zero(c[0] | (c[1] << 16)), canon_neg_zero(c[2] | (c[3] << 16)));
}
// quant_block16_bf16 (16 bf16 as 8 words) by the packed path
__device__ __forceinline__ uint2 quant_block16_bf16_fast(const uint32_t (&w)[8], uint32_t& sbits, bool& nonfinite) {
  const uint32_t ab = amax_bits_bf16x16(w);
  nonfinite = ab >= 0x7F80u;
  uint64_t p[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = bf16x2_to_f32x2(w[i]);
  return quant_block16_pairs(p, __uint_as_float(ab << 16), sbits);
}
// quant_block16_bf16vals (16 fp32 holding bf16 values) by the packed path
__device__ __forceinline__ uint2 quant_block16_bf16vals_fast(const float (&v)[16], uint32_t& sbits) {
  float amax = 0.0f;
#pragma unroll
  for (int i = 0; i < 16; ++i) amax = fmaxf(amax, fabsf(v[i]));
  uint64_t p[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = f32x2_pack(v[2 * i], v[2 * i + 1]);
  return quant_block16_pairs(p, amax, sbits);
}

}  // namespace realb
