// gemm_bf16.cu — K5: grouped BF16 expert GEMM on the 5th-gen tensor cores.
//
//   out[r, n] = sum_k A[r, k] * W[g*N + n, k]      (A, W both K-major bf16)
//
// Persistent warp-specialised kernel, one CTA per SM (148):
//   warp 0      TMA producer: A 128x64 and W BNx64 tiles, SWIZZLE_128B, into a
//               STAGES-deep smem ring (full/empty mbarriers)
//   warp 1      MMA issuer: one thread issues tcgen05.mma.cta_group::1.kind::f16
//               (M=128, N=BN, K=16) x4 per stage into a TMEM accumulator;
//               tcgen05.commit releases smem stages and publishes the tile
//   warp 2      TMEM allocator (2 x BN fp32 columns: double-buffered accumulator
//               so the epilogue of tile i overlaps the mainloop of tile i+1)
//   warps 4-7   epilogue: tcgen05.ld 32x32b -> registers -> (SwiGLU) -> bf16
//               -> global; each warp owns TMEM lane quadrant (warp % 4)
// Roofline: tensor-bound, 2*M*N*K flop per tile.
#include "common.cuh"
#include "grouped.cuh"

namespace realb {

constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 bf16 = 128 B rows = one SWIZZLE_128B atom width

template <int BN, int STAGES>
struct SmemBf16 {
  static constexpr int A_BYTES = kBM * kBK * 2;
  static constexpr int B_BYTES = BN * kBK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;  // + barriers + alignment slack
};

__device__ __forceinline__ float silu_mul(float g, float u) {
  return g / (1.0f + __expf(-g)) * u;
}

template <int BN, int STAGES, int EPI>
__global__ void __launch_bounds__(256, 1)
    grouped_gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA,
                             const __grid_constant__ CUtensorMap tmB, const int32_t* layout,
                             int E, int prec, int N, int K, __nv_bfloat16* __restrict__ out) {
  using S = SmemBf16<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id(), lane = lane_id();
  const GroupedSched sched = GroupedSched::make(layout, E, prec, N, BN);
  const int total = sched.total();
  const int nkb = K / kBK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<2 * BN>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const TileCoord c = sched.coord(t);
        const int brow = c.group * N + c.n0;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * S::STAGE_BYTES;
          mbar_arrive_expect_tx(&full[stage], S::STAGE_BYTES);
          tma_load_2d(sa, &tmA, &full[stage], kb * kBK, c.a_row);
          tma_load_2d(sa + S::A_BYTES, &tmB, &full[stage], kb * kBK, brow);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t idesc = idesc_bf16(kBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t dtmem = tmem_base + acc * BN;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * S::STAGE_BYTES);
          const uint64_t adesc = umma_desc_sw128(sa);
          const uint64_t bdesc = umma_desc_sw128(sa + S::A_BYTES);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            // advance the start address by 32 B (16 bf16) inside the 128-B swizzle atom
            umma_bf16(dtmem, adesc + (uint64_t)(k * 2), bdesc + (uint64_t)(k * 2), idesc,
                      (kb | k) != 0);
          }
          tc_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue
    const int q = warp & 3;  // TMEM lane quadrant
    const int row_in_tile = q * 32 + lane;
    int it = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
      const TileCoord c = sched.coord(t);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + acc * BN + ((uint32_t)(q * 32) << 16);
      const int64_t r = (int64_t)c.a_row + row_in_tile;
      if constexpr (EPI == REALB_EPI_STORE) {
        __nv_bfloat16* orow = out + r * N + c.n0;
#pragma unroll 1
        for (int cc = 0; cc < BN; cc += 32) {
          uint32_t v[32];
          tmem_ld32(tbase + cc, v);
          tmem_wait_ld();
          uint32_t p[16];
#pragma unroll
          for (int i = 0; i < 16; ++i)
            p[i] = pack_bf16x2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
#pragma unroll
          for (int i = 0; i < 4; ++i)
            st_global_v4(orow + cc + 8 * i, p[4 * i], p[4 * i + 1], p[4 * i + 2], p[4 * i + 3]);
        }
      } else {  // SwiGLU: columns [0, BN/2) gate, [BN/2, BN) up of the same outputs
        const int NO = N / 2;
        __nv_bfloat16* orow = out + r * NO + c.n0 / 2;
#pragma unroll 1
        for (int cc = 0; cc < BN / 2; cc += 16) {
          uint32_t g[16], u[16];
          tmem_ld16(tbase + cc, g);
          tmem_ld16(tbase + BN / 2 + cc, u);
          tmem_wait_ld();
          uint32_t p[8];
#pragma unroll
          for (int i = 0; i < 8; ++i)
            p[i] = pack_bf16x2(silu_mul(__uint_as_float(g[2 * i]), __uint_as_float(u[2 * i])),
                               silu_mul(__uint_as_float(g[2 * i + 1]), __uint_as_float(u[2 * i + 1])));
          st_global_v4(orow + cc, p[0], p[1], p[2], p[3]);
          st_global_v4(orow + cc + 8, p[4], p[5], p[6], p[7]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<2 * BN>(tmem_base);
}

template <int BN, int STAGES, int EPI>
static int launch_grouped_bf16(const void* a, const void* w, int64_t rows_cap, int N, int K, int E,
                               const int32_t* layout, int prec, void* out, int max_ctas,
                               cudaStream_t st) {
  CUtensorMap ta, tb;
  int rc = make_tmap_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a, K, rows_cap, (uint64_t)K * 2, kBK,
                        kBM, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  rc = make_tmap_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, w, K, (uint64_t)E * N, (uint64_t)K * 2,
                    kBK, BN, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  auto kern = grouped_gemm_bf16_kernel<BN, STAGES, EPI>;
  const int smem = SmemBf16<BN, STAGES>::TOTAL;
  rc = cuda_status(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                   "grouped_gemm_bf16: smem attribute");
  if (rc) return rc;
  int grid = num_sms();
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  kern<<<grid, 256, smem, st>>>(ta, tb, layout, E, prec, N, K,
                                reinterpret_cast<__nv_bfloat16*>(out));
  return check_launch("realb_grouped_gemm_bf16");
}

}  // namespace realb

using namespace realb;

extern "C" int realb_grouped_gemm_bf16(const void* d_a, const void* d_w, int64_t rows_cap, int N,
                                       int K, int E, const int32_t* d_layout, int prec,
                                       int epilogue, void* d_out, int max_ctas, void* stream) {
  if (!d_a || !d_w || !d_layout || !d_out || rows_cap <= 0 || rows_cap % 128 || E <= 0 ||
      (prec != REALB_PREC_W16A16 && prec != REALB_PREC_W4A4)) {
    set_error("realb_grouped_gemm_bf16: bad arguments");
    return REALB_EINVAL;
  }
  if (K % kBK || N % 256) {
    set_error("realb_grouped_gemm_bf16: needs K %% 64 == 0 and N %% 256 == 0 (N=%d K=%d)", N, K);
    return REALB_EUNSUPPORTED;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (epilogue == REALB_EPI_STORE)
    return launch_grouped_bf16<256, 4, REALB_EPI_STORE>(d_a, d_w, rows_cap, N, K, E, d_layout,
                                                        prec, d_out, max_ctas, st);
  if (epilogue == REALB_EPI_SWIGLU)
    return launch_grouped_bf16<256, 4, REALB_EPI_SWIGLU>(d_a, d_w, rows_cap, N, K, E, d_layout,
                                                         prec, d_out, max_ctas, st);
  set_error("realb_grouped_gemm_bf16: unknown epilogue %d", epilogue);
  return REALB_EINVAL;
}
