// quant.cu — K3: on-the-fly BF16 -> NVFP4 weight quantiser (also used for the
// fp32/fp64 parity path). HBM-bound: 2.5625 B/element for bf16 input
// (2 read + 0.5 codes + 0.0625 scale).
//
// Work unit = a 128-row x 4-block (64-column) tile: exactly one 512-byte
// scale-factor atom of the tcgen05 block-scale layout, so the atom is written
// as one contiguous, coalesced 512-byte run. Thread -> (row = b / 4,
// kb = b % 4): four consecutive threads read one row's 128 contiguous input
// bytes (bf16) and write its 32 contiguous code bytes.
#include <cstdlib>
#include <climits>

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

// ---------------------------------------------------------------------------
// K3 (v2): persistent and register double-buffered. Tiles are 128 rows x 64
// columns (one 512-B scale atom), enumerated group by group (an expert's rows
// are a group; only the groups the device plan made W4A4, or all of them), k-tile
// fastest; CTA c owns a CONTIGUOUS range of tiles and walks it incrementally (no
// per-tile divisions). Thread -> (row = tid / 2, half = tid % 2): its 2 blocks are
// 64 contiguous input bytes (4 x 16-B loads; a warp reads 16 full 128-B lines),
// 16 contiguous code bytes (one 16-B store) and 2 adjacent scale bytes (one 16-bit
// store into the atom). The NEXT tile's loads are issued before the current tile
// is converted, so every thread keeps 64 B in flight through the conversion, and
// the conversion runs two elements per instruction (FFMA2 / FMUL2).
// one whole block (16 bf16 = one 32-B sector) per load: LDG.256 (sm_100), so no
// sector is requested twice (16-B loads without L1 allocation split every sector
// into two L2 requests)
__device__ __forceinline__ void ldg_nc_v8(uint32_t (&v)[8], const void* p) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "l"(p));
}

// A K3 segment: one [G x rows_per_group, cols] bf16 matrix and its NVFP4 outputs. A
// launch covers up to two segments (an expert's gate_up and down weights) as ONE
// contiguous tile range, so the two matrices share one ramp-up and one tail.
struct QSeg {
  const __nv_bfloat16* x;
  int64_t rows, cols;
  int mt_per_group;
  uint8_t* codes;
  uint8_t* sf;
};
constexpr int kQMaxSegs = 2;
struct QSegs {
  QSeg s[kQMaxSegs];
  int n;
  int dbg;  // timing probes (REALB_DBG_K3): 1 = stores without the conversion, 2 = loads only
};
static int k3_dbg() {
  const char* e = getenv("REALB_DBG_K3");
  return e ? atoi(e) : 0;
}

template <int LAYOUT>
__global__ void __launch_bounds__(256) quant_tiles_kernel(const __grid_constant__ QSegs segs, int G,
                                                          const uint8_t* __restrict__ prec, int32_t* flag) {
  __shared__ float2 tab[128];
  __shared__ int s_list[256];
  __shared__ int s_n;
  sf_table_init(tab);
  if (threadIdx.x == 0) {
    int n = 0;
    for (int g = 0; g < G; ++g)
      if (!prec || prec[g] == REALB_PREC_W4A4) s_list[n++] = g;
    s_n = n;
  }
  __syncthreads();
  static_assert(kQMaxSegs == 2, "the walk below handles two segments");
  const int64_t tiles0 = (int64_t)s_n * segs.s[0].mt_per_group * (segs.s[0].cols >> 6);
  const int64_t tiles = tiles0 + (segs.n > 1 ? (int64_t)s_n * segs.s[1].mt_per_group * (segs.s[1].cols >> 6) : 0);
  const int64_t q = tiles / gridDim.x, rem = tiles % gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * q + min((int64_t)blockIdx.x, rem);
  const int64_t t1 = t0 + q + ((int64_t)blockIdx.x < rem ? 1 : 0);
  if (t0 >= t1) return;
  const int row_in = threadIdx.x >> 1, half = threadIdx.x & 1;
  // walk state: segment si, group g, m-tile mt, k-tile kt
  int64_t w0 = t0;
  const QSeg* S = &segs.s[0];
  if (w0 >= tiles0) { w0 -= tiles0; S = &segs.s[1]; }
  int tiles_k = (int)(S->cols >> 6);
  int per_group = S->mt_per_group * tiles_k;
  int g = (int)(w0 / per_group);
  const int wg = (int)(w0 - (int64_t)g * per_group);
  int mt = wg / tiles_k, kt = wg - (wg / tiles_k) * tiles_k;
  auto row_of = [&](const QSeg* s_, int gg, int mm) {
    return ((int64_t)s_list[gg] * s_->mt_per_group + mm) * 128 + row_in;
  };
  int64_t r = row_of(S, g, mt);
  bool ok = r < S->rows;
  uint32_t cur[2][8], nxt[2][8];
  if (ok) {
    const uint8_t* p = reinterpret_cast<const uint8_t*>(S->x + r * S->cols + kt * 64 + half * 32);
    ldg_nc_v8(cur[0], p);
    ldg_nc_v8(cur[1], p + 32);
  }
  for (int64_t t = t0; t < t1; ++t) {
    const QSeg* S2 = S;
    int g2 = g, mt2 = mt, kt2 = kt + 1;
    if (kt2 == tiles_k) {
      kt2 = 0;
      if (++mt2 == S->mt_per_group) {
        mt2 = 0;
        if (++g2 == s_n) { g2 = 0; S2 = S + 1; }  // next segment (only reached if t + 1 < t1)
      }
    }
    int64_t r2 = 0;
    bool ok2 = false;
    if (t + 1 < t1) {
      r2 = row_of(S2, g2, mt2);
      ok2 = r2 < S2->rows;
      if (ok2) {
        const uint8_t* p = reinterpret_cast<const uint8_t*>(S2->x + r2 * S2->cols + kt2 * 64 + half * 32);
        ldg_nc_v8(nxt[0], p);
        ldg_nc_v8(nxt[1], p + 32);
      }
    }
    if (ok && segs.dbg == 2) {  // probe: keep the loads alive without converting or storing
      if ((cur[0][0] ^ cur[1][7]) == 0x7fc17fc1u) flag_nonfinite(flag);
    } else if (ok) {
      uint32_t sa, sb;
      bool nfa = false, nfb = false;
      uint2 ca, cb;
      if (segs.dbg == 1) {  // probe: the stores without the conversion
        ca = make_uint2(cur[0][0] ^ cur[0][1], cur[0][2] ^ cur[0][3]);
        cb = make_uint2(cur[1][0] ^ cur[1][1], cur[1][2] ^ cur[1][3]);
        sa = cur[0][4] & 0xff; sb = cur[1][4] & 0xff;
      } else {
        ca = quant_block16_bf16_x2(cur[0], sa, nfa, tab);
        cb = quant_block16_bf16_x2(cur[1], sb, nfb, tab);
      }
      if (nfa || nfb) flag_nonfinite(flag);
      const int64_t cols = S->cols, nkb = cols >> 4;
      *reinterpret_cast<uint4*>(S->codes + r * (cols >> 1) + kt * 32 + half * 16) =
          make_uint4(ca.x, ca.y, cb.x, cb.y);
      const int64_t kb0 = (int64_t)kt * 4 + half * 2;
      const int64_t so = LAYOUT == REALB_SF_FLAT ? r * nkb + kb0 : sf_mma_offset(r, kb0, nkb);
      *reinterpret_cast<uint16_t*>(S->sf + so) = (uint16_t)(sa | (sb << 8));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      cur[0][i] = nxt[0][i];
      cur[1][i] = nxt[1][i];
    }
    if (S2 != S) {
      S = S2;
      tiles_k = (int)(S->cols >> 6);
    }
    g = g2; mt = mt2; kt = kt2; r = r2; ok = ok2;
  }
}

// ---------------------------------------------------------------------------
// K3 (v3): TMA-fed, full-row stages. One persistent CTA per SM. Warp 16 streams
// the CTA's CONTIGUOUS range of 8-row slices of the weight matrix (8 whole rows
// = one contiguous run of 8 x cols x 2 bytes, so every DRAM page is read in one
// pass) into a 5-8-stage shared-memory ring with ONE cp.async.bulk.tensor per
// stage: a 3-D box [64 columns] x [cols/64 k-tiles] x [8 rows], SWIZZLE_128B. Two
// groups of 8 converter warps take alternate stages. Converter item (row r,
// k-tile j) = one 128-B line of the stage: the 4 blocks of row r in k-tile j = one
// row of one scale atom; a quarter-warp reads 8 consecutive lines (swizzled,
// conflict-free); it writes 32 contiguous code bytes (one 32-B store; a warp writes
// 1 KB contiguous) and the atom row's 4 scale bytes (one 32-bit store). No register cost
// for the bytes in flight, no address arithmetic on the converting threads
// beyond the item's row and column.
constexpr int kQ3MaxStages = 8;
constexpr int kQ3MaxCols = 2560;                    // 40 boxes: 40 KB per stage
constexpr int kQ3RingBytes = 200 * 1024;            // stages = ring / stage bytes (5..8)
constexpr int kQ3Threads = 544;  // 2 converter groups of 8 warps + the producer warp

__device__ __forceinline__ void stg_v8(void* p, const uint32_t (&v)[8]) {
  asm volatile("st.global.v8.u32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

__global__ void __launch_bounds__(kQ3Threads, 1) quant_tma_kernel(const __grid_constant__ CUtensorMap tmx,
                                                                  int64_t cols, int slices_per_group, int G,
                                                                  const uint8_t* __restrict__ prec,
                                                                  uint8_t* __restrict__ codes,
                                                                  uint8_t* __restrict__ sf, int32_t* flag) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kQ3RingBytes);
  uint64_t* empty = full + kQ3MaxStages;
  float2* tab = reinterpret_cast<float2*>(empty + kQ3MaxStages);
  int* s_list = reinterpret_cast<int*>(tab + 128);
  int* s_n = s_list + 256;
  const int64_t nkb = cols >> 4;
  const int nbox = (int)(cols >> 6);
  const uint32_t stage_bytes = (uint32_t)nbox * 1024u;
  const int kQ3Stages = min(kQ3MaxStages, (int)(kQ3RingBytes / stage_bytes));
  const uint32_t kQ3StageBytes = stage_bytes;
  sf_table_init(tab);
  if (threadIdx.x == 0) {
    int n = 0;
    for (int g = 0; g < G; ++g)
      if (!prec || prec[g] == REALB_PREC_W4A4) s_list[n++] = g;
    *s_n = n;
    for (int i = 0; i < kQ3Stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 8);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t slices = (int64_t)(*s_n) * slices_per_group;
  const int64_t q = slices / gridDim.x, rem = slices % gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * q + min((int64_t)blockIdx.x, rem);
  const int n_t = (int)(q + ((int64_t)blockIdx.x < rem ? 1 : 0));
  if (n_t <= 0) return;
  const int warp = threadIdx.x >> 5;
  auto row0_of = [&](int i) -> int64_t {  // first row of this CTA's slice i
    const int64_t t = t0 + i;
    const int g = (int)(t / slices_per_group);
    return ((int64_t)s_list[g] * slices_per_group + (t - (int64_t)g * slices_per_group)) * 8;
  };
  if (warp == 16) {  // ------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch_desc(&tmx);
      for (int i = 0; i < n_t; ++i) {
        const int stage = i % kQ3Stages;
        mbar_wait(&empty[stage], ((i / kQ3Stages) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[stage], stage_bytes);
        const int row0 = (int)row0_of(i);
        // one 3-D box per stage: [64 columns] x [cols/64 k-tiles] x [8 rows]
        tma_load_3d(smem + stage * kQ3StageBytes, &tmx, &full[stage], 0, 0, row0);
      }
    }
    return;
  }
  // ------------------------------------------------------------------ converters
  const int cg = warp >> 3, tt = threadIdx.x & 255;
  bool nonfinite = false;
  for (int i = cg; i < n_t; i += 2) {
    const int stage = i % kQ3Stages;
    const int64_t row0 = row0_of(i);
    mbar_wait(&full[stage], (i / kQ3Stages) & 1);
    const uint32_t sbase = smem_u32(smem + stage * kQ3StageBytes);
    for (int L = tt; L < nbox * 8; L += 256) {
      // 128-B line L of the stage = (row r_in, k-tile j); a quarter-warp reads 8
      // consecutive lines, whose swizzled chunks hit 8 distinct bank groups
      const int r_in = L / nbox, j = L - r_in * nbox;
      const uint32_t rowbase = sbase + (uint32_t)L * 128u;
      uint32_t w[4][8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint4 v = ld_shared_v4(rowbase + ((uint32_t)(c ^ (L & 7)) << 4));
        w[c >> 1][(c & 1) * 4 + 0] = v.x;
        w[c >> 1][(c & 1) * 4 + 1] = v.y;
        w[c >> 1][(c & 1) * 4 + 2] = v.z;
        w[c >> 1][(c & 1) * 4 + 3] = v.w;
      }
      uint32_t cw[8], sw = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        uint32_t sb;
        bool nf;
        const uint2 c = quant_block16_bf16_x2(w[b], sb, nf, tab);
        nonfinite |= nf;
        cw[2 * b] = c.x;
        cw[2 * b + 1] = c.y;
        sw |= sb << (8 * b);
      }
      const int64_t r = row0 + r_in;
      stg_v8(codes + r * (cols >> 1) + (int64_t)j * 32, cw);
      *reinterpret_cast<uint32_t*>(sf + sf_mma_offset(r, (int64_t)j * 4, nkb)) = sw;
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[stage]);  // this warp is done with the stage
  }
  if (nonfinite) flag_nonfinite(flag);
}

// v3 launch over a [groups x rows_per_group, cols] bf16 matrix (rows_per_group % 8 == 0,
// cols % 64 == 0, cols <= kQ3MaxCols)
static int launch_quant_tma(const void* x, int64_t rows, int64_t cols, int64_t rows_per_group, int G,
                            const uint8_t* prec, uint8_t* codes, uint8_t* sf, int32_t* flag, int max_ctas,
                            cudaStream_t st) {
  CUtensorMap tm;
  const uint64_t dims[3] = {64, (uint64_t)cols / 64, (uint64_t)rows};
  const uint64_t strides[2] = {128, (uint64_t)cols * 2};
  const uint32_t box[3] = {64, (uint32_t)(cols / 64), 8};
  int rc = make_tmap_3d(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, x, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  constexpr int smem = kQ3RingBytes + 2 * kQ3MaxStages * 8 + 128 * 8 + 257 * 4 + 1024;
  static_assert(smem <= 227 * 1024, "K3 v3 shared memory");
  rc = set_smem_once(reinterpret_cast<const void*>(quant_tma_kernel), smem, "quant_tma_kernel: smem attribute");
  if (rc) return rc;
  int grid = num_sms();
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  quant_tma_kernel<<<grid, kQ3Threads, smem, st>>>(tm, cols, (int)(rows_per_group / 8), G, prec, codes, sf, flag);
  return check_launch("realb_quantize (K3 v3)");
}

// K3 form (REALB_K3_VERSION, for A/B runs; scripts/bench_quant.py). Measured on the
// EP8 hot rank's Kimi weights (ncu, gate_up / down): v1 30.6 / 19.3 us, v2 27.1 / 17.8,
// v3 26.8 / 20.6 -> v2 is the default (K3).
static int k3_version() {
  const char* e = getenv("REALB_K3_VERSION");
  if (e && (e[0] == '1' || e[0] == '2' || e[0] == '3')) return e[0] - '0';
  return 2;
}

static bool k3_v1() { return k3_version() == 1; }

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
      if (!flat && cols % 64 == 0 && cols <= kQ3MaxCols && rows % 128 == 0 && k3_version() == 3 &&
          rows / 8 <= INT32_MAX)
        return launch_quant_tma(d_x, rows, cols, rows, 1, nullptr, d_codes, d_sf, d_flag, max_ctas, st);
      if (cols % 64 == 0 && !k3_v1() && (rows + 127) / 128 <= INT32_MAX / 64) {
        const int64_t mt = (rows + 127) / 128;
        auto kern = flat ? quant_tiles_kernel<REALB_SF_FLAT> : quant_tiles_kernel<REALB_SF_MMA128x4>;
        const int grid = quant_grid(reinterpret_cast<const void*>(kern), mt * (cols / 64), max_ctas);
        QSegs sg{};
        sg.s[0] = QSeg{reinterpret_cast<const __nv_bfloat16*>(d_x), rows, cols, (int)mt, d_codes, d_sf};
        sg.n = 1;
        kern<<<grid, 256, 0, st>>>(sg, 1, nullptr, d_flag);
        return check_launch("realb_quantize_nvfp4");
      }
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
  if (cols <= kQ3MaxCols && k3_version() == 3 && rows_per_expert / 8 <= INT32_MAX)
    return launch_quant_tma(d_w, (int64_t)E * rows_per_expert, cols, rows_per_expert, E, d_expert_prec, d_codes,
                            d_sf, d_flag, max_ctas, (cudaStream_t)stream);
  if (!k3_v1()) {
    auto kern = quant_tiles_kernel<REALB_SF_MMA128x4>;
    const int grid = quant_grid(reinterpret_cast<const void*>(kern),
                               (int64_t)E * (rows_per_expert / 128) * (cols / 64), max_ctas);
    QSegs sg{};
    sg.s[0] = QSeg{reinterpret_cast<const __nv_bfloat16*>(d_w), (int64_t)E * rows_per_expert, cols,
                   (int)(rows_per_expert / 128), d_codes, d_sf};
    sg.n = 1;
    sg.dbg = k3_dbg();
    kern<<<grid, 256, 0, (cudaStream_t)stream>>>(sg, E, d_expert_prec, d_flag);
    return check_launch("realb_quantize_experts_nvfp4");
  }
  const int grid = quant_grid(reinterpret_cast<const void*>(quant_experts_kernel),
                             (int64_t)E * (rows_per_expert / 128) * (cols / 64), max_ctas);
  quant_experts_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const __nv_bfloat16*>(d_w), rows_per_expert, cols, E, d_expert_prec,
      d_codes, d_sf, d_flag);
  return check_launch("realb_quantize_experts_nvfp4");
}

extern "C" int realb_quantize_experts2_nvfp4(const void* d_w0, int64_t rows0_per_expert, int64_t cols0,
                                             uint8_t* d_codes0, uint8_t* d_sf0, const void* d_w1,
                                             int64_t rows1_per_expert, int64_t cols1, uint8_t* d_codes1,
                                             uint8_t* d_sf1, int E, const uint8_t* d_expert_prec,
                                             int32_t* d_flag, int max_ctas, void* stream) {
  if (!d_w0 || !d_w1 || !d_expert_prec || !d_codes0 || !d_sf0 || !d_codes1 || !d_sf1 || E < 1 || E > 256 ||
      rows0_per_expert <= 0 || rows0_per_expert % 128 || cols0 <= 0 || cols0 % 64 || rows1_per_expert <= 0 ||
      rows1_per_expert % 128 || cols1 <= 0 || cols1 % 64 || rows0_per_expert / 128 > INT32_MAX / 64 ||
      rows1_per_expert / 128 > INT32_MAX / 64) {
    set_error("realb_quantize_experts2_nvfp4: bad arguments (E=%d rows/expert=%lld,%lld cols=%lld,%lld)", E,
              (long long)rows0_per_expert, (long long)rows1_per_expert, (long long)cols0, (long long)cols1);
    return REALB_EINVAL;
  }
  if (k3_version() != 2) {  // A/B forms (v1 / v3) quantise the two matrices in two launches
    int rc = realb_quantize_experts_nvfp4(d_w0, E, rows0_per_expert, cols0, d_expert_prec, d_codes0, d_sf0, d_flag,
                                          max_ctas, stream);
    if (rc) return rc;
    return realb_quantize_experts_nvfp4(d_w1, E, rows1_per_expert, cols1, d_expert_prec, d_codes1, d_sf1, d_flag,
                                        max_ctas, stream);
  }
  auto kern = quant_tiles_kernel<REALB_SF_MMA128x4>;
  const int64_t tiles = (int64_t)E * ((rows0_per_expert / 128) * (cols0 / 64) + (rows1_per_expert / 128) * (cols1 / 64));
  const int grid = quant_grid(reinterpret_cast<const void*>(kern), tiles, max_ctas);
  QSegs sg{};
  sg.s[0] = QSeg{reinterpret_cast<const __nv_bfloat16*>(d_w0), (int64_t)E * rows0_per_expert, cols0,
                 (int)(rows0_per_expert / 128), d_codes0, d_sf0};
  sg.s[1] = QSeg{reinterpret_cast<const __nv_bfloat16*>(d_w1), (int64_t)E * rows1_per_expert, cols1,
                 (int)(rows1_per_expert / 128), d_codes1, d_sf1};
  sg.n = 2;
  sg.dbg = k3_dbg();
  kern<<<grid, 256, 0, (cudaStream_t)stream>>>(sg, E, d_expert_prec, d_flag);
  return check_launch("realb_quantize_experts2_nvfp4");
}
