// gemm_fp4_pair.cu — K6 v2 for the bf16-STORE (down) GEMM: grouped NVFP4 x NVFP4
// on 2-SM tcgen05 pairs with the A operand RESIDENT in shared memory.
//
// Why (measured, DESIGN.md §4 K6): on the EP8 hot rank the K6 down GEMM is bound by
// the L2 -> SM fabric, not by the tensor pipe. The v1 kernel (1-CTA 128x256 tiles)
// re-reads its A tile for every n-tile and the whole W tile per SM: 2.75 GB of
// L2 -> SM traffic for the Kimi down GEMM, and its 561 MB bf16 output then competes
// with that traffic (the stores cost 30 % of the kernel). Here:
//   * a work unit is (m-tile pair, run of n-tiles): each CTA of the pair loads its
//     128 A rows x K ONCE per unit (K/256 chunks of 16 KB, SWIZZLE_128B) and its
//     A scales once per unit (one TMA box, then tcgen05.cp into TMEM);
//   * per n-tile only W streams: the pair MMA (cta_group::2, M = 256, N = 256) reads
//     128 W rows from each CTA's smem, so an SM receives 16 KB of codes + 4 KB of
//     scales per K = 256 step for 128 x 256 x 256 MACs (v1: 54 KB).
// N stays 256: a pair MMA with N = 128 measured as slow as N = 256 per instruction
// (half the FLOP rate), so the accumulator is single-buffered (256 of the 512 TMEM
// columns; the rest holds the unit's A scales and two W-scale stage buffers). The
// hand-off to the epilogue is cheap with RELAXED arrives (common.cuh: the release
// form compiles to MEMBAR.ALL.GPU, which waited for the epilogue's stores).
// A chunks of the next unit load as the last tile of the current unit releases them
// (per-chunk empty barriers), interleaved with the first tile's W stages; the next
// unit's A rows and scales are prefetched into L2 one unit ahead.
//
// Warp roles (both CTAs of the pair):
//   warp 0      producer (elected lane): A chunks, A scales, W stages (both CTAs
//               load their own halves, completing on the leader's barriers)
//   warp 1      MMA issuer (leader CTA only)
//   warp 2      TMEM allocator (512 columns, cta_group::2)
//   warps 4..   epilogue, lane quadrant q = warp % 4. STORE: 8 warps, 32 rows x 128
//               columns each: tcgen05.ld, release, bf16 convert, SWIZZLE_128B smem
//               staging, two 128-B-wide TMA stores per tile. SWIGLU: 16 warps, 32 rows
//               x 32 outputs each: SwiGLU + NVFP4 re-quantisation (K4), stored from
//               registers (16 code bytes + 2 scale bytes per row)
// Roofline: tensor-bound at the dense NVFP4 rate once the feed fits.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "fp4_rule.cuh"
#include "grouped.cuh"

namespace realb {

constexpr int kPBN = 256;          // N per tile (pair MMA M = 256, N = 256)
constexpr int kPBKB = 128;         // bytes of K per A chunk / W stage = 256 E2M1 values
// epilogue warps: 8 for the bf16 STORE (32 rows x 128 columns each); 16 for SWIGLU,
// whose SwiGLU + NVFP4 re-quantisation of a tile took longer than the tile's MMAs on
// 8 warps (32 rows x 32 outputs each)
template <int EPI>
constexpr int pair_epi_warps() { return EPI == REALB_EPI_SWIGLU ? 16 : 8; }
template <int EPI>
constexpr int pair_threads() { return 32 * (4 + pair_epi_warps<EPI>()); }
constexpr int kPRing = 4;          // unit-id ring depth
constexpr int kPMaxSmem = 232448;  // 227 KB opt-in dynamic smem per CTA

template <int NCH, int EPI>
struct PairSmem {
  static constexpr int A_CHUNK = 128 * kPBKB;        // 16 KB: 128 rows x 128 B
  static constexpr int B_HALF = (kPBN / 2) * kPBKB;  // 16 KB: this CTA's 128 W rows
  static constexpr int SFB_STAGE = 8 * 512;          // 2 x 4 scale atoms (256 W rows x K = 256)
  static constexpr int EPI_WARP = 32 * 128;          // 32 rows x 64 bf16 columns
  static constexpr int SFA_BYTES = NCH * 2048;       // the unit's A scales (K/64 atoms)
  static constexpr int EPI_BYTES = EPI == REALB_EPI_SWIGLU ? 0 : 8 * EPI_WARP;  // SwiGLU stores from registers
  static constexpr int FIXED = NCH * A_CHUNK + SFA_BYTES + EPI_BYTES + 512 + 1024;
  static constexpr int STAGES_FIT = (kPMaxSmem - FIXED) / (B_HALF + SFB_STAGE);
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static constexpr int A_OFF = 0;
  static constexpr int B_OFF = NCH * A_CHUNK;
  static constexpr int SFB_OFF = B_OFF + STAGES * B_HALF;
  static constexpr int SFA_OFF = SFB_OFF + STAGES * SFB_STAGE;
  static constexpr int EPI_OFF = SFA_OFF + SFA_BYTES;
  static constexpr int BAR_OFF = EPI_OFF + EPI_BYTES;
  static constexpr int TOTAL = BAR_OFF + 512 + 1024;
  static_assert(STAGES >= 3, "too few W stages");
  static_assert(TOTAL <= kPMaxSmem, "smem");
};

struct PairArgs {
  const int32_t* layout;
  int E, N, K;
  int run;                   // n-tiles per work unit
  uint32_t sf_lbo, sf_sbo;
  uint32_t dbg;              // REALB_DBG_FP4 bit 1: no epilogue stores (timing probe)
  __nv_bfloat16* out;        // SWIGLU: optional bf16 SwiGLU values (parity hook)
  uint8_t* out_codes;        // SWIGLU: E2M1 [rows][N/4]
  uint8_t* out_sf;           // SWIGLU: MMA-layout scales of the [rows][N/2] result
  unsigned long long* prof;  // debug: [2 ranks][16] wait cycles per call site, or null
};

__device__ __forceinline__ uint64_t sf_desc_p(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)(lbo >> 4) << 16;
  d |= (uint64_t)(sbo >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// barrier wait; with args.prof set (REALB_DBG_PROF), the cycles spent waiting are
// accumulated per call site (debug timing, printed by fp4_pair_store)
#define PW(id, bar, par)               \
  do {                                 \
    if (prof) {                        \
      const long long t0_ = clock64(); \
      mbar_wait(bar, par);             \
      pcyc[id] += clock64() - t0_;     \
    } else {                           \
      mbar_wait(bar, par);             \
    }                                  \
  } while (0)

template <int NCH, int EPI>
__global__ void __launch_bounds__(pair_threads<EPI>(), 1)
    grouped_gemm_fp4_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                                 const __grid_constant__ CUtensorMap tmSfa,
                                 const __grid_constant__ CUtensorMap tmSfb,
                                 const __grid_constant__ CUtensorMap tmOut, const PairArgs args) {
  using S = PairSmem<NCH, EPI>;
  constexpr int STAGES = S::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* afull = empty + STAGES;
  uint64_t* aempty = afull + NCH;
  uint64_t* sfafull = aempty + NCH;
  uint64_t* sfaempty = sfafull + 1;
  uint64_t* tfull = sfaempty + 1;
  uint64_t* tempty = tfull + 1;
  uint64_t* slot_full = tempty + 1;
  uint64_t* slot_empty = slot_full + kPRing;
  int32_t* slot_tile = reinterpret_cast<int32_t*>(slot_empty + kPRing);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(slot_tile + kPRing);

  const int warp = warp_id(), lane = lane_id();
  const uint32_t crank = cluster_ctarank();
  unsigned long long* prof = args.prof;
  long long pcyc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) pcyc[i] = 0;
  const long long tstart = clock64();
  const int N = args.N, K = args.K;
  const GroupedSched sched = GroupedSched::make(args.layout, args.E, REALB_PREC_W4A4, N, kPBN);
  const int n_tiles = N / kPBN;
  const int run = args.run;
  const int nruns = (n_tiles + run - 1) / run;
  const int m_units = sched.G > 0 ? sched.pprefix[sched.G] : 0;
  const int total_units = m_units * nruns;
  const int kbytes = K / 2;
  const int atoms = K / 64;  // A-scale atoms per 128-row tile
  const uint32_t sfa_bytes = (uint32_t)atoms * 512u;
  constexpr uint16_t kBoth = 0x3;
  constexpr int EW = pair_epi_warps<EPI>();
  constexpr uint32_t kSlotConsumers = 2 + 2 * EW;  // leader MMA + both CTAs' epilogue warps + peer producer

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmSfa);
    tma_prefetch_desc(&tmSfb);
    tma_prefetch_desc(&tmOut);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int c = 0; c < NCH; ++c) {
      mbar_init(&afull[c], 1);
      mbar_init(&aempty[c], 1);
    }
    mbar_init(sfafull, 1);
    mbar_init(sfaempty, 1);
    mbar_init(tfull, 1);
    mbar_init(tempty, 2 * EW);
    for (int i = 0; i < kPRing; ++i) {
      mbar_init(&slot_full[i], 1);
      mbar_init(&slot_empty[i], kSlotConsumers);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2sm<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto unit_of = [&](int u, int& nt0, int& nt1) {
    const int mp = u / nruns, r = u - mp * nruns;
    nt0 = r * run;
    nt1 = min(n_tiles, nt0 + run);
    return mp;
  };

  if (warp == 0) {  // ---------------------------------------------------- producer
    const bool leader = elect_one();
    int* ctr = GroupedSched::counters(args.layout, REALB_PREC_W4A4);
    const uint32_t full0 = mapa_shared(&full[0], 0), afull0 = mapa_shared(&afull[0], 0);
    const uint32_t sfafull0 = mapa_shared(sfafull, 0);
    int stage = 0;
    uint32_t phase = 0;
    // unit ids are fetched ONE UNIT AHEAD (leader: atomic counter, published to both
    // CTAs' rings; peer: read from its ring), so the next unit's A rows and A scales
    // are prefetched into L2 while this unit runs
    auto fetch = [&](int i) -> int {
      const int slot = i % kPRing;
      int u = 0;
      if (crank == 0) {
        PW(0, &slot_empty[slot], ((i / kPRing) & 1) ^ 1);
        if (leader) {
          u = atomicAdd(ctr, 1);
          if (u >= total_units) u = -1;
          slot_tile[slot] = u;
          st_cluster_u32(mapa_shared(&slot_tile[slot], 1), (uint32_t)u);
          mbar_arrive_cluster(mapa_shared(&slot_full[slot], 1));  // release: publishes slot_tile
          mbar_arrive(&slot_full[slot]);
        }
        u = __shfl_sync(0xffffffffu, u, 0);
      } else {
        PW(1, &slot_full[slot], (i / kPRing) & 1);
        u = __shfl_sync(0xffffffffu, slot_tile[slot], 0);
        __syncwarp();
        if (leader) mbar_arrive_cluster_relaxed(mapa_shared(&slot_empty[slot], 0));
      }
      return u;
    };
    // A scales of unit #j (id uj): one box of K/64 atoms per CTA into the single smem
    // buffer, after the MMA warp's copy of unit #j-1's scales released it
    auto load_sfa = [&](int j, int uj) {
      int n0_, n1_;
      const int mpj = unit_of(uj, n0_, n1_);
      bool dj = false, dj1 = false;
      const TileCoord cj = sched.coord_pair(mpj * n_tiles, (int)crank, dj);
      if (crank == 0) { bool d1; (void)sched.coord_pair(mpj * n_tiles, 1, d1); dj1 = d1; }
      const int rj = __shfl_sync(0xffffffffu, cj.a_row, 0);
      dj = __shfl_sync(0xffffffffu, (int)dj, 0) != 0;
      dj1 = __shfl_sync(0xffffffffu, (int)dj1, 0) != 0;
      PW(2, sfaempty, (uint32_t)(j & 1) ^ 1);
      if (leader) {
        if (crank == 0) mbar_arrive_expect_tx(sfafull, (dj1 ? 1u : 2u) * sfa_bytes);
        if (!dj) tma_load_2d_2sm(smem + S::SFA_OFF, &tmSfa, sfafull0, 0, (rj >> 7) * atoms * 2);
      }
      __syncwarp();
    };
    int u_next = fetch(0);
    for (int i = 0;; ++i) {
      const int u = u_next;
      if (u < 0) break;
      u_next = fetch(i + 1);
      if (u_next >= 0) {  // L2 prefetch of the next unit's A rows + A scales (this CTA's half)
        int n0_, n1_;
        bool dn;
        const TileCoord cn = sched.coord_pair(unit_of(u_next, n0_, n1_) * n_tiles, (int)crank, dn);
        const int nrow = __shfl_sync(0xffffffffu, cn.a_row, 0);
        dn = __shfl_sync(0xffffffffu, (int)dn, 0) != 0;
        if (leader && !dn) {
          for (int kb = 0; kb < NCH; ++kb) tma_prefetch_l2_2d(&tmA, kb * kPBKB, nrow);
          tma_prefetch_l2_2d(&tmSfa, 0, (nrow >> 7) * atoms * 2);
        }
        __syncwarp();
      }
      int nt0, nt1;
      const int mp = unit_of(u, nt0, nt1);
      bool dummy = false, dummy1 = false;
      const TileCoord c = sched.coord_pair(mp * n_tiles, (int)crank, dummy);
      if (crank == 0) { bool d1; (void)sched.coord_pair(mp * n_tiles, 1, d1); dummy1 = d1; }
      const int a_row = __shfl_sync(0xffffffffu, c.a_row, 0);
      const int group = __shfl_sync(0xffffffffu, c.group, 0);
      dummy = __shfl_sync(0xffffffffu, (int)dummy, 0) != 0;
      dummy1 = __shfl_sync(0xffffffffu, (int)dummy1, 0) != 0;
      const uint32_t ucnt = dummy1 ? 1u : 2u;  // CTAs of the pair that load A rows
      const uint32_t up = (uint32_t)(i & 1);
      if (i == 0) load_sfa(0, u);  // later units' A scales are loaded during the unit before
      for (int nt = nt0; nt < nt1; ++nt) {
        const int brow = group * N + nt * kPBN;
        const int sfb_row = (brow >> 7) * atoms * 2;
        // the NEXT unit's A scales, once the MMA warp has copied this unit's into TMEM
        // (one tile in, the producer's lead of STAGES stages is behind that copy)
        if (nt == min(nt0 + 1, nt1 - 1) && u_next >= 0) load_sfa(i + 1, u_next);
        for (int kb = 0; kb < NCH; ++kb) {
          if (nt == nt0) {  // A chunk kb of this unit, as soon as the last unit's last tile released it
            PW(3, &aempty[kb], up ^ 1);
            if (leader) {
              if (crank == 0) mbar_arrive_expect_tx(&afull[kb], ucnt * S::A_CHUNK);
              if (!dummy)
                tma_load_2d_2sm(smem + S::A_OFF + kb * S::A_CHUNK, &tmA, afull0 + (uint32_t)kb * 8u, kb * kPBKB,
                                a_row);
            }
            __syncwarp();
          }
          PW(4, &empty[stage], phase ^ 1);
          if (leader) {
            if (crank == 0) mbar_arrive_expect_tx(&full[stage], 2 * (S::B_HALF + S::SFB_STAGE));
            const uint32_t fb = full0 + (uint32_t)stage * 8u;
            tma_load_2d_2sm(smem + S::B_OFF + stage * S::B_HALF, &tmB, fb, kb * kPBKB, brow + (int)crank * (kPBN / 2));
            uint8_t* ssfb = smem + S::SFB_OFF + stage * S::SFB_STAGE;  // W rows 0-127 | 128-255 of the tile
            tma_load_2d_2sm(ssfb, &tmSfb, fb, 0, sfb_row + kb * 8);
            tma_load_2d_2sm(ssfb + 2048, &tmSfb, fb, 0, sfb_row + atoms * 2 + kb * 8);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1 && crank == 0) {  // ------------------------------- MMA issuer
    // Whole warp on the path with warp-uniform values; one elected lane issues (the
    // same shape as gemm_fp4.cu, which ptxas compiles to straight uniform-datapath code).
    const bool leader = elect_one();
    constexpr uint32_t idesc = idesc_nvfp4(256, kPBN);
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t tsfa = tbase + kPBN;                // the unit's A scales: K/16 columns
    const uint32_t tsfb0 = tsfa + (uint32_t)(K / 16);  // 2 x 32 columns of stage W scales
    const uint32_t s0 = smem_u32(smem);
    const uint64_t adesc0 = umma_desc_sw128(s0 + S::A_OFF);
    const uint64_t bdesc0 = umma_desc_sw128(s0 + S::B_OFF);
    const uint64_t sfadesc0 = sf_desc_p(s0 + S::SFA_OFF, args.sf_lbo, args.sf_sbo);
    const uint64_t sfbdesc0 = sf_desc_p(s0 + S::SFB_OFF, args.sf_lbo, args.sf_sbo);
    int stage = 0;
    uint32_t phase = 0, sfsel = 0;
    int tile_it = 0;
    for (int it = 0;; ++it) {
      const int slot = it % kPRing;
      PW(5, &slot_full[slot], (it / kPRing) & 1);
      const int u = __shfl_sync(0xffffffffu, slot_tile[slot], 0);
      __syncwarp();
      if (leader) mbar_arrive_relaxed(&slot_empty[slot]);
      if (u < 0) break;
      int nt0, nt1;
      (void)unit_of(u, nt0, nt1);
      const uint32_t up = (uint32_t)(it & 1);
      for (int nt = nt0; nt < nt1; ++nt, ++tile_it) {
        // single accumulator: the previous tile drained => every earlier MMA completed
        PW(7, tempty, (tile_it & 1) ^ 1);
        tc_fence_after();
        if (nt == nt0) {  // the unit's A scales -> TMEM (the previous unit's MMAs are done)
          PW(6, sfafull, up);
          tc_fence_after();
          if (leader) {
            for (int a = 0; a < atoms; ++a) utccp_32x128b_warpx4_2sm(tsfa + 4 * a, sfadesc0 + 32 * a);
            tc_commit_2sm_mc(sfaempty, kBoth);
          }
          __syncwarp();
        }
        const bool last = nt == nt1 - 1;
        for (int kb = 0; kb < NCH; ++kb) {
          const int nmma = min(kPBKB, kbytes - kb * kPBKB) / 32;  // K = 64 steps (last chunk may be short)
          PW(8, &afull[kb], up);
          PW(9, &full[stage], phase);
          tc_fence_after();
          const uint64_t soff_b = (uint64_t)((uint32_t)(stage * S::B_HALF) >> 4);
          const uint64_t soff_sf = (uint64_t)((uint32_t)(stage * S::SFB_STAGE) >> 4);
          const uint64_t aoff = (uint64_t)(kb * (S::A_CHUNK >> 4));
          const uint32_t tsfb = tsfb0 + sfsel * 32;
          if (leader) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (j < nmma) {
                utccp_32x128b_warpx4_2sm(tsfb + 8 * j, sfbdesc0 + soff_sf + 32 * j);
                utccp_32x128b_warpx4_2sm(tsfb + 8 * j + 4, sfbdesc0 + soff_sf + 128 + 32 * j);
              }
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (j < nmma)
                umma_nvfp4_2sm(tbase, adesc0 + aoff + 2 * j, bdesc0 + soff_b + 2 * j, idesc, tsfa + (kb * 4 + j) * 4,
                               tsfb + 8 * j, (kb | j) != 0);
            tc_commit_2sm_mc(&empty[stage], kBoth);
            if (last) tc_commit_2sm_mc(&aempty[kb], kBoth);
          }
          __syncwarp();
          sfsel ^= 1;
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (leader) tc_commit_2sm_mc(tfull, kBoth);
        __syncwarp();
      }
    }
  } else if (warp >= 4) {  // -------------------------------------------- epilogue
    const int q = warp & 3, h = (warp - 4) >> 2;  // h: column half (STORE) / output quarter (SWIGLU)
    const uint32_t ebuf = smem_u32(smem + S::EPI_OFF + (warp - 4) * S::EPI_WARP);
    const bool store = !(args.dbg & 1u);
    int tile_it = 0;
    for (int it = 0;; ++it) {
      const int slot = it % kPRing;
      PW(10, &slot_full[slot], (it / kPRing) & 1);
      const int u = slot_tile[slot];
      __syncwarp();
      if (lane == 0) {  // the slot's value is in registers: relaxed
        if (crank == 0) mbar_arrive_relaxed(&slot_empty[slot]);
        else mbar_arrive_cluster_relaxed(mapa_shared(&slot_empty[slot], 0));
      }
      if (u < 0) break;
      int nt0, nt1;
      const int mp = unit_of(u, nt0, nt1);
      bool dummy;
      const TileCoord c = sched.coord_pair(mp * n_tiles, (int)crank, dummy);
      for (int nt = nt0; nt < nt1; ++nt, ++tile_it) {
        PW(11, tfull, tile_it & 1);
        tc_fence_after();
        uint32_t v[4][32];
        if constexpr (EPI == REALB_EPI_SWIGLU) {  // gate columns [h*32, +32), up columns 128 + the same
          const uint32_t tb = tmem_base + (uint32_t)(h * 32) + ((uint32_t)(q * 32) << 16);
          tmem_ld32(tb, v[0]);
          tmem_ld32(tb + 128, v[1]);
        } else {
          const uint32_t tb = tmem_base + (uint32_t)(h * 128) + ((uint32_t)(q * 32) << 16);
#pragma unroll
          for (int i = 0; i < 4; ++i) tmem_ld32(tb + 32 * i, v[i]);
        }
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {  // accumulator free: the next tile's MMAs may start (relaxed: TMEM reads only)
          if (crank == 0) mbar_arrive_relaxed(tempty);
          else mbar_arrive_cluster_relaxed(mapa_shared(tempty, 0));
        }
        if (dummy || !store) continue;
        if constexpr (EPI == REALB_EPI_SWIGLU) {
          // outputs [nt*128 + h*32, +32) of row r: h = bf16(silu(g) * u), then NVFP4 with
          // the reference block rule (K4 fused; same code as gemm_fp4.cu)
          const int I = N / 2;
          const int64_t r = (int64_t)c.a_row + q * 32 + lane;
          const int ocol = nt * (kPBN / 2) + h * 32;
          uint32_t sfw = 0;
          uint2 cw[2];
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            float hv[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float g = __uint_as_float(v[0][b * 16 + i]);
              const float uu = __uint_as_float(v[1][b * 16 + i]);
              hv[i] = __bfloat162float(__float2bfloat16_rn(__fdividef(g, 1.0f + __expf(-g)) * uu));
            }
            uint32_t sb;
            cw[b] = quant_block16_bf16vals_fast(hv, sb);
            sfw |= sb << (8 * b);
            if (args.out) {  // parity hook: the bf16 SwiGLU values the re-quantisation consumed
              uint32_t hp[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) hp[i] = pack_bf16x2(hv[2 * i], hv[2 * i + 1]);
              uint4* hd = reinterpret_cast<uint4*>(args.out + r * I + ocol + b * 16);
              hd[0] = make_uint4(hp[0], hp[1], hp[2], hp[3]);
              hd[1] = make_uint4(hp[4], hp[5], hp[6], hp[7]);
            }
          }
          *reinterpret_cast<uint4*>(args.out_codes + r * (I / 2) + ocol / 2) = make_uint4(cw[0].x, cw[0].y, cw[1].x, cw[1].y);
          *reinterpret_cast<uint16_t*>(args.out_sf + sf_mma_offset(r, ocol / 16, I / 16)) = (uint16_t)sfw;
          continue;
        }
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {  // two 64-column halves through one 4 KB staging buffer
          {
            const long long t0 = prof ? clock64() : 0;
            if (lane == 0) bulk_wait_group_read<0>();  // the previous store has read the buffer
            __syncwarp();
            if (prof) pcyc[12] += clock64() - t0;
          }
          // row = lane: 128 B of bf16 = 8 x 16-B pieces, piece p at p ^ (row & 7) (SWIZZLE_128B)
#pragma unroll
          for (int p = 0; p < 8; ++p) {
            const uint32_t* src = v[2 * hh + (p >> 2)] + 8 * (p & 3);
            st_shared_v4(ebuf + lane * 128 + ((p ^ (lane & 7)) << 4),
                         pack_bf16x2(__uint_as_float(src[0]), __uint_as_float(src[1])),
                         pack_bf16x2(__uint_as_float(src[2]), __uint_as_float(src[3])),
                         pack_bf16x2(__uint_as_float(src[4]), __uint_as_float(src[5])),
                         pack_bf16x2(__uint_as_float(src[6]), __uint_as_float(src[7])));
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmOut, smem + S::EPI_OFF + (warp - 4) * S::EPI_WARP, nt * kPBN + h * 128 + hh * 64,
                         c.a_row + q * 32);
            bulk_commit_group();
          }
          __syncwarp();
        }
      }
    }
    if (EPI != REALB_EPI_SWIGLU && lane == 0) bulk_wait_group<0>();
  }
  if (prof && lane == 0 && (warp <= 1 || warp >= 4)) {
    pcyc[warp == 0 ? 13 : warp == 1 ? 14 : 15] = clock64() - tstart;  // role's loop time
    for (int i = 0; i < 16; ++i)
      if (pcyc[i]) atomicAdd(prof + crank * 16 + i, (unsigned long long)pcyc[i]);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no peer may still load / arrive / read our smem or TMEM
  tc_fence_after();
  if (warp == 2) tmem_dealloc_2sm<512>(tmem_base);
  if (threadIdx.x == 0) GroupedSched::finish(args.layout, REALB_PREC_W4A4);
}

template <int NCH, int EPI>
static int launch_pair(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tsa, const CUtensorMap& tsb,
                       const CUtensorMap& to, const PairArgs& args, int grid, cudaStream_t st) {
  auto kern = grouped_gemm_fp4_pair_kernel<NCH, EPI>;
  const int smem = PairSmem<NCH, EPI>::TOTAL;
  int rc = set_smem_once(reinterpret_cast<const void*>(kern), smem, "grouped_gemm_nvfp4 (pair): smem attribute");
  if (rc) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(pair_threads<EPI>());
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  rc = cuda_status(cudaLaunchKernelEx(&cfg, kern, ta, tb, tsa, tsb, to, args), "realb_grouped_gemm_nvfp4 (pair) launch");
  if (rc) return rc;
  return check_launch("realb_grouped_gemm_nvfp4 (pair)");
}

// TMEM: 256 accumulator + K/16 A-scale + 2 x 32 W-scale columns <= 512; smem: the
// resident A (K/256 chunks of 16 KB) leaves >= 3 W stages up to K = 1792 with the
// STORE epilogue's staging, up to K = 2048 without it (SWIGLU)
int fp4_pair_supported(int epilogue, int N, int K) {
  if (K % 64 || N % 256) return 0;
  if (epilogue == REALB_EPI_STORE) return K <= 1792;
  if (epilogue == REALB_EPI_SWIGLU) return K <= 2048 && (N / 2) % 64 == 0;
  return 0;
}

int fp4_pair(int epilogue, const uint8_t* a, const uint8_t* a_sf, const uint8_t* w, const uint8_t* w_sf,
             int64_t rows_cap, int N, int K, int E, const int32_t* layout, void* out, uint8_t* out_codes,
             uint8_t* out_sf, int max_ctas, uint32_t sf_lbo, uint32_t sf_sbo, uint32_t dbg, cudaStream_t st) {
  CUtensorMap ta, tb, tsa, tsb, to;
  int rc = make_tmap_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT8, a, (uint64_t)K / 2, rows_cap, (uint64_t)K / 2, kPBKB, 128,
                        CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  rc = make_tmap_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, w, (uint64_t)K / 2, (uint64_t)E * N, (uint64_t)K / 2, kPBKB,
                    kPBN / 2, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  // scale bytes viewed as [bytes / 256][256]: the A box is one 128-row tile's K/64 atoms,
  // the W box 4 atoms (one 128-row tile x K = 256)
  const uint64_t sa_bytes = (uint64_t)rows_cap * (uint64_t)(K / 16);
  rc = make_tmap_2d(&tsa, CU_TENSOR_MAP_DATA_TYPE_UINT8, a_sf, 256, sa_bytes / 256, 256, 256, (uint32_t)(K / 32),
                    CU_TENSOR_MAP_SWIZZLE_NONE);
  if (rc) return rc;
  const uint64_t sb_bytes = (uint64_t)E * N * (uint64_t)(K / 16);
  rc = make_tmap_2d(&tsb, CU_TENSOR_MAP_DATA_TYPE_UINT8, w_sf, 256, sb_bytes / 256, 256, 256, 8,
                    CU_TENSOR_MAP_SWIZZLE_NONE);
  if (rc) return rc;
  if (epilogue == REALB_EPI_STORE) {
    rc = make_tmap_2d(&to, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, out, N, rows_cap, (uint64_t)N * 2, 64, 32,
                      CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  } else {
    to = ta;  // unused
  }
  PairArgs args;
  args.layout = layout;
  args.E = E;
  args.N = N;
  args.K = K;
  // units of <= 4 n-tiles: the A reload at a unit boundary is hidden behind the tile
  // before it, and ~15 units per pair keep the dynamic schedule's tail short
  const char* run_env = getenv("REALB_K6_RUN");
  const int max_run = run_env && run_env[0] ? atoi(run_env) : 3;
  const int nt = N / kPBN, nruns = (nt + max_run - 1) / max_run;
  args.run = (nt + nruns - 1) / nruns;
  args.sf_lbo = sf_lbo;
  args.sf_sbo = sf_sbo;
  args.dbg = dbg;
  args.out = reinterpret_cast<__nv_bfloat16*>(out);
  args.out_codes = out_codes;
  args.out_sf = out_sf;
  args.prof = nullptr;
  static unsigned long long* d_prof = nullptr;
  const bool want_prof = getenv("REALB_DBG_PROF") != nullptr;
  if (want_prof) {
    if (!d_prof) cudaMalloc(&d_prof, 32 * sizeof(unsigned long long));
    cudaMemsetAsync(d_prof, 0, 32 * sizeof(unsigned long long), st);
    args.prof = d_prof;
  }
  int grid = num_sms();
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  grid = grid / 2 * 2;
  if (grid < 2) grid = 2;
#define REALB_PAIR_CASE(NC)                                                                   \
  case NC:                                                                                    \
    rc = epilogue == REALB_EPI_SWIGLU                                                         \
             ? launch_pair<NC, REALB_EPI_SWIGLU>(ta, tb, tsa, tsb, to, args, grid, st)       \
             : launch_pair<(NC < 8 ? NC : 7), REALB_EPI_STORE>(ta, tb, tsa, tsb, to, args, grid, st); \
    break;
  switch ((K + 255) / 256) {
    REALB_PAIR_CASE(1)
    REALB_PAIR_CASE(2)
    REALB_PAIR_CASE(3)
    REALB_PAIR_CASE(4)
    REALB_PAIR_CASE(5)
    REALB_PAIR_CASE(6)
    REALB_PAIR_CASE(7)
    REALB_PAIR_CASE(8)
    default:
      set_error("realb_grouped_gemm_nvfp4 (pair): unsupported K=%d", K);
      return REALB_EUNSUPPORTED;
  }
#undef REALB_PAIR_CASE
  if (want_prof && rc == 0) {  // debug: mean wait cycles per warp and call site, per pair rank
    unsigned long long hbuf[32];
    cudaStreamSynchronize(st);
    cudaMemcpy(hbuf, d_prof, sizeof(hbuf), cudaMemcpyDeviceToHost);
    const char* names[16] = {"P.slot_empty", "P.slot_full", "P.sfaempty", "P.aempty", "P.empty", "M.slot_full",
                             "M.sfafull", "M.tempty", "M.afull", "M.full", "E.slot_full", "E.tfull", "E.storewait",
                             "P.loop", "M.loop", "E.loop"};
    const double ew = epilogue == REALB_EPI_SWIGLU ? 16 : 8;
    const double per[16] = {1, 1, 1, 1, 1, 1, 1, 1, 1, 1, ew, ew, ew, 1, 1, ew};
    const int ctas = grid / 2;
    for (int r = 0; r < 2; ++r) {
      fprintf(stderr, "[pair prof rank %d] mean kcycles per warp:", r);
      for (int i = 0; i < 16; ++i)
        if (hbuf[r * 16 + i]) fprintf(stderr, " %s=%.1f", names[i], hbuf[r * 16 + i] / (per[i] * ctas) / 1000.0);
      fprintf(stderr, "\n");
    }
  }
  return rc;
}

}  // namespace realb
