/*
 * fp4_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library.
 *
 * Plain-C restatement of the reference NVFP4 quantiser, following its
 * vectorised algorithm step by step in float64:
 *   moesim.fp4.quantize_blocks   /root/reference/pkg/src/moesim/fp4.py:173-227
 *     amax  = max |v|                           fp4.py:188
 *     raw   = amax / 6                          fp4.py:189
 *     sub   = raw < 2^-6 -> m = rint(raw/2^-9), m>=8 -> 0x08      fp4.py:193-195
 *     norm  = frexp(raw) -> e = exp-1, sig = 2*mant,
 *             m = rint((sig-1)*8), carry, saturate -> 0x7E      fp4.py:196-206
 *     raw >= 448 -> 0x7E                         fp4.py:207
 *     nonzero & bits==0 -> 1                     fp4.py:208-209
 *     scale = decode(bits)                       fp4.py:212-216
 *     codes: searchsorted(mids, |v/scale|, left) + odd-index tie bump,
 *            sign only when idx > 0              fp4.py:219-226
 *   dequantize_blocks                            fp4.py:230-243
 * Parity of this file with the reference is pinned by tests/test_oracle.py
 * against fixtures generated from the reference itself
 * (tests/golden/make_golden.py) and the reference's own golden SHA-256.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

static const double MIDS[7] = {0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0};
static const double MAGS[8] = {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0};

static double decode_e4m3(unsigned bits) {
  unsigned se = bits >> 3, sm = bits & 7u;
  if (se == 0) return (double)sm * 0.001953125; /* 2^-9 */
  return (1.0 + (double)sm / 8.0) * exp2((double)se - 7.0);
}

static unsigned encode_scale(double raw) {
  if (raw >= 448.0) return 0x7E;
  if (raw < 0.015625) {
    double m = rint(raw / 0.001953125);
    return m >= 8.0 ? 0x08u : (unsigned)m;
  }
  int exp2i = 0;
  double mant = frexp(raw, &exp2i); /* raw = mant * 2^exp2i, mant in [0.5, 1) */
  int e = exp2i - 1;
  double sig = mant * 2.0;
  long m = (long)rint((sig - 1.0) * 8.0);
  if (m == 8) {
    e += 1;
    m = 0;
  }
  if (e > 8 || (e == 8 && m > 6)) return 0x7E;
  return (unsigned)(((e + 7) << 3) | m);
}

/* returns 0, or -1 if any value is non-finite (QuantizationDomainError) */
int oracle_quantize_blocks(const double* values, int64_t n, uint8_t* codes, uint8_t* scale_bits) {
  for (int64_t i = 0; i < n * 16; ++i)
    if (!isfinite(values[i])) return -1;
  for (int64_t b = 0; b < n; ++b) {
    const double* v = values + b * 16;
    double amax = 0.0;
    for (int i = 0; i < 16; ++i) amax = fmax(amax, fabs(v[i]));
    unsigned bits = encode_scale(amax / 6.0);
    if (amax > 0.0 && bits == 0) bits = 1;
    if (amax == 0.0) bits = 0; /* raw == 0 encodes to 0 anyway */
    scale_bits[b] = (uint8_t)bits;
    const double scale = decode_e4m3(bits);
    for (int i = 0; i < 16; ++i) {
      double sig = amax > 0.0 ? v[i] / scale : 0.0;
      double mag = fabs(sig);
      int idx = 0;
      while (idx < 7 && MIDS[idx] < mag) ++idx; /* searchsorted side="left" */
      if (idx < 7 && mag == MIDS[idx] && (idx & 1)) ++idx;
      codes[b * 16 + i] = (uint8_t)((sig < 0.0 && idx > 0) ? (idx | 8) : idx);
    }
  }
  return 0;
}

void oracle_dequantize_blocks(const uint8_t* codes, const uint8_t* scale_bits, int64_t n,
                              double* out) {
  for (int64_t b = 0; b < n; ++b) {
    const double scale = decode_e4m3(scale_bits[b]);
    for (int i = 0; i < 16; ++i) {
      unsigned c = codes[b * 16 + i];
      double m = MAGS[c & 7];
      out[b * 16 + i] = ((c & 8) ? -m : m) * scale;
    }
  }
}

/* Host-side bf16 fast path used as the CPU baseline: bf16 bits -> same rule.
 * x: uint16 bf16 [rows][cols]; codes packed [rows][cols/2]; sf flat [rows][cols/16]. */
int oracle_quantize_bf16(const uint16_t* x, int64_t rows, int64_t cols, uint8_t* codes_packed,
                         uint8_t* sf) {
  double v[16];
  uint8_t c[16];
  int bad = 0;
  const int64_t nkb = cols / 16;
  for (int64_t r = 0; r < rows; ++r) {
    for (int64_t kb = 0; kb < nkb; ++kb) {
      for (int i = 0; i < 16; ++i) {
        uint32_t w = (uint32_t)x[r * cols + kb * 16 + i] << 16;
        float f;
        memcpy(&f, &w, 4);
        v[i] = (double)f;
      }
      uint8_t s;
      if (oracle_quantize_blocks(v, 1, c, &s)) bad = 1;
      sf[r * nkb + kb] = s;
      for (int i = 0; i < 8; ++i)
        codes_packed[r * (cols / 2) + kb * 8 + i] = (uint8_t)(c[2 * i] | (c[2 * i + 1] << 4));
    }
  }
  return bad ? -1 : 0;
}
