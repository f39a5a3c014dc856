// gemm_fp4.cu — K6: grouped NVFP4 x NVFP4 expert GEMM on tcgen05
// (kind::mxf4nvf4.block_scale.scale_vec::4X: E2M1 operands, one UE4M3 scale
// per 16 elements along K for both A and W, FP32 accumulation in TMEM).
//
// Persistent, warp-specialised, one CTA per SM, 384 threads:
//   warp 0     TMA producer: A 128x256 and W 256x256 E2M1 tiles (128-B rows,
//              SWIZZLE_128B) + their scale-factor atoms (TMA over the scale
//              bytes viewed as 256-byte rows; the quantisers write scales directly
//              in the 128x4-atom layout, so a stage's scales are contiguous 2 KB runs)
//   warp 1     MMA issuer: tcgen05.cp (smem -> TMEM, 32x128b.warpx4) of the
//              stage's scale atoms, then 4 x tcgen05.mma (K=64 each)
//   warp 2     TMEM allocator (512 columns: 256 accumulator, the m-tile's A
//              scales for the whole K (K/16 columns, RESIDENT across the unit's
//              n-tiles) and 2 x 32 columns of streamed W scales)
// Work unit = (m-tile, run of up to 4 n-tiles): the A-side scales are copied to
// TMEM once per unit, so a steady-state stage issues 8 tcgen05.cp instead of 12
// (measured on B200: 4 MMAs = 512 cycles; +8 copies = 665; +12 copies = 836).
//   warps 4-11 epilogue: the 8 warps copy the whole accumulator into registers
//              (quadrant = warp % 4, column half = (warp - 4) / 4), release TMEM
//              to the MMA warp at once, then run SwiGLU (+ NVFP4 re-quantisation
//              of the bf16 result with the reference block rule, K4 fused) or the
//              bf16 store from registers while the next tile's mainloop runs.
//
// CL = 2 (large experts): a 2-CTA cluster is one tcgen05 CTA pair, M = 256
// (cta_group::2). CTA r stages ITS 128 A rows, HALF of the W tile (rows
// 128r..128r+127 of the 256), its A scales and the full W scales; the leader
// issues the pair's scale copies (each CTA's smem -> its own TMEM) and MMAs.
// Halving the W bytes each SM receives per stage (54 -> 38 KB per 512 MMA cycles)
// lifts the TMA-feed bound the 1-CTA kernel runs into (TMA-only time was 0.67 of
// the kernel on the EP8 hot rank's gate_up).
// Roofline: tensor-bound at the dense FP4 rate (4x BF16 per MMA cycle).
#include <cstdlib>

#include "common.cuh"
#include "fp4_rule.cuh"
#include "grouped.cuh"

namespace realb {

constexpr int kF4BM = 128, kF4BN = 256;
constexpr int kF4BKB = 128;               // bytes of K per stage = 256 E2M1 values
constexpr int kF4Threads = 384;
constexpr int kSfBoxRows = 8;             // scale TMA box: 8 x 256 B = 2 KB = 4 atoms
constexpr int kF4EpiBufs = 3;             // TMA-store staging buffers per epilogue warp (STORE)

// XST (experiment): 4 operand stages and NO epilogue staging for the STORE kernel,
// valid only with the epilogue stores skipped (REALB_DBG_FP4 bit 1): measures how
// much of the down GEMM is the operand feed of a 3-stage ring (K6)
template <int EPI, int CL, int XST = 0>
struct SmemFp4 {
  // STORE (bf16 out) needs 48 KB of TMA-store staging
  static constexpr int STAGES = XST ? XST : CL == 1 ? (EPI != REALB_EPI_SWIGLU ? 3 : 4) : (EPI != REALB_EPI_SWIGLU ? 4 : 5);
  static constexpr int A_BYTES = kF4BM * kF4BKB;              // 16 KB
  static constexpr int B_BYTES = (kF4BN / CL) * kF4BKB;       // 32 KB (16 KB per CTA of a pair)
  static constexpr int SFA_BYTES = 4 * 512;                   // 128 rows x 16 scales
  static constexpr int SFB_BYTES = 2 * 4 * 512;               // 256 rows x 16 scales (full W tile)
  static constexpr int STAGE = A_BYTES + B_BYTES + SFA_BYTES + SFB_BYTES;
  static constexpr int EPI_OFF = STAGES * STAGE;    // 8 warps x kF4EpiBufs x 2 KB (STORE only)
  static constexpr int EPI_BYTES = (EPI != REALB_EPI_SWIGLU && !XST) ? 8 * kF4EpiBufs * 2048 : 0;
  static constexpr int BAR_OFF = EPI_OFF + EPI_BYTES;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};
constexpr uint32_t kTmemAcc = 0, kTmemSfa = 256;  // SFB buffers follow the resident SFA
constexpr int kNPerUnit = 4;                           // n-tiles per work unit
constexpr int kF4Ring = 4;

struct Fp4Args {
  const uint8_t* a_sf;
  const uint8_t* w_sf;
  const int32_t* layout;
  int E, N, K;
  __nv_bfloat16* out;   // STORE: bf16 [rows][N]
  uint8_t* out_codes;   // SWIGLU: E2M1 [rows][N/4]
  uint8_t* out_sf;      // SWIGLU: MMA-layout scales of the [rows][N/2] result
  uint32_t sf_lbo, sf_sbo;
  uint32_t dbg;  // REALB_DBG_FP4 bits: 1 skip epilogue math/stores, 2 skip scale copies, 4 skip MMAs,
                 // 8 release the accumulator without reading it, 16 no accumulator hand-off at
                 // all (MMA never waits, epilogue idle; wrong results: the mainloop alone), 32 STORE
                 // epilogue stages its chunks but issues no TMA store, 64 every TMA store writes
                 // output tile 0 (L2-resident: no HBM write-back)
  RowScatter scat;  // kEpiScatter: per-row destinations (down GEMM fused with the EP return)
};

__device__ __forceinline__ uint64_t sf_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)(lbo >> 4) << 16;
  d |= (uint64_t)(sbo >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

template <int EPI, int CL, int XST = 0>
__global__ void __launch_bounds__(kF4Threads, 1)
    grouped_gemm_fp4_kernel(const __grid_constant__ CUtensorMap tmA,
                            const __grid_constant__ CUtensorMap tmB,
                            const __grid_constant__ CUtensorMap tmSfa,
                            const __grid_constant__ CUtensorMap tmSfb,
                            const __grid_constant__ CUtensorMap tmOut, const Fp4Args args) {
  using S = SmemFp4<EPI, CL, XST>;
  constexpr int kF4Stages = S::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint64_t* empty = full + kF4Stages;
  uint64_t* tfull = empty + kF4Stages;
  uint64_t* tempty = tfull + 1;
  uint64_t* slot_full = tempty + 1;
  uint64_t* slot_empty = slot_full + kF4Ring;
  int32_t* slot_tile = reinterpret_cast<int32_t*>(slot_empty + kF4Ring);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(slot_tile + kF4Ring);

  const int warp = warp_id(), lane = lane_id();
  const uint32_t crank = CL == 2 ? cluster_ctarank() : 0u;
  const int N = args.N, K = args.K;
  const GroupedSched sched = GroupedSched::make(args.layout, args.E, REALB_PREC_W4A4, N, kF4BN);
  const int n_tiles = N / kF4BN;
  const int nchunks = (n_tiles + kNPerUnit - 1) / kNPerUnit;
  const int m_units = sched.G > 0 ? (CL == 2 ? sched.pprefix[sched.G] : sched.prefix[sched.G]) : 0;
  const int total_units = m_units * nchunks;
  const uint32_t sfa_cols = (uint32_t)(K / 16);  // resident A scales: 4 columns per K=64
  const int kbytes = K / 2;
  const int nkb = (kbytes + kF4BKB - 1) / kF4BKB;
  const int atoms_per_row_tile = K / 64;  // 4-scale atoms per 128-row tile
  constexpr uint16_t kBoth = 0x3;
  // consumers of a unit slot: 1-CTA: MMA + 8 epilogue warps; pair: leader MMA + 8
  // leader epilogue warps + peer producer + 8 peer epilogue warps
  constexpr uint32_t kSlotConsumers = CL == 2 ? 18 : 9;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmSfa);
    tma_prefetch_desc(&tmSfb);
    for (int s = 0; s < kF4Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 8 * CL);
    for (int i = 0; i < kF4Ring; ++i) {
      mbar_init(&slot_full[i], 1);
      mbar_init(&slot_empty[i], kSlotConsumers);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (CL == 2) tmem_alloc_2sm<512>(tmem_slot);
    else tmem_alloc<512>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CL == 2) cluster_sync();  // peer barriers / TMEM ready before any remote op
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // m-unit index -> this CTA's 128-row m-tile (dummy: the pair's expert has an odd
  // m-tile count and this rank-1 CTA has no rows of its own in this unit)
  auto mtile_of = [&](int mu, int rank, bool& dummy) -> TileCoord {
    if constexpr (CL == 2) return sched.coord_pair(mu * n_tiles, rank, dummy);
    dummy = false;
    return sched.coord(mu * n_tiles);
  };
  auto arrive_leader = [&](uint64_t* bar) {
    // relaxed: these arrives only signal "slot value read" / "TMEM drained" (no memory
    // writes to publish); a release arrive waits for the warp's outstanding stores
    if constexpr (CL == 2) mbar_arrive_cluster_relaxed(mapa_shared(bar, 0));
    else mbar_arrive_relaxed(bar);
  };

  // Producer and MMA roles run on their WHOLE warp: every lane computes the same
  // (hence provably warp-uniform) values and one elected lane issues the TMA /
  // tcgen05 instructions. Issuing from `lane == 0` code makes the compiler wrap
  // each tcgen05 instruction in an ELECT/R2UR waterfall loop, which made the
  // single issuing thread, not the tensor pipe, the bottleneck.
  if (warp == 0) {  // ---------------- producer + dynamic unit fetch
    const bool leader = elect_one();
    int* ctr = GroupedSched::counters(args.layout, REALB_PREC_W4A4);
    const uint32_t full0 = CL == 2 ? mapa_shared(&full[0], 0) : smem_u32(&full[0]);
    int stage = 0;
    uint32_t phase = 0;
    for (int i = 0;; ++i) {
      const int slot = i % kF4Ring;
      int u = 0;
      if (crank == 0) {  // the (pair) leader fetches and publishes the unit
        mbar_wait(&slot_empty[slot], ((i / kF4Ring) & 1) ^ 1);
        if (leader) {
          u = atomicAdd(ctr, 1);
          if (u >= total_units) u = -1;
          slot_tile[slot] = u;
          if constexpr (CL == 2) {
            st_cluster_u32(mapa_shared(&slot_tile[slot], 1), (uint32_t)u);
            mbar_arrive_cluster(mapa_shared(&slot_full[slot], 1));
          }
          mbar_arrive(&slot_full[slot]);
        }
        u = __shfl_sync(0xffffffffu, u, 0);
      } else {
        mbar_wait(&slot_full[slot], (i / kF4Ring) & 1);
        u = __shfl_sync(0xffffffffu, slot_tile[slot], 0);
        __syncwarp();
        if (leader) arrive_leader(&slot_empty[slot]);
      }
      if (u < 0) break;
      const int mu = u / nchunks, nt0 = (u - mu * nchunks) * kNPerUnit;
      const int nt1 = min(n_tiles, nt0 + kNPerUnit);
      bool dummy = false, dummy1 = false;
      const TileCoord c = mtile_of(mu, (int)crank, dummy);
      if constexpr (CL == 2) {
        if (crank == 0) { bool d1; (void)mtile_of(mu, 1, d1); dummy1 = d1; }
      }
      const int a_row = __shfl_sync(0xffffffffu, c.a_row, 0);
      const int group = __shfl_sync(0xffffffffu, c.group, 0);
      dummy = __shfl_sync(0xffffffffu, (int)dummy, 0) != 0;
      dummy1 = __shfl_sync(0xffffffffu, (int)dummy1, 0) != 0;
      const int sfa_row = (a_row >> 7) * atoms_per_row_tile * 2;  // 256-byte rows of the A-scale view
      for (int nt = nt0; nt < nt1; ++nt) {
        const int brow = group * N + nt * kF4BN;
        const int sfb_row = (brow >> 7) * atoms_per_row_tile * 2;
        const bool load_a_sf = nt == nt0;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) {
            uint8_t* sa = smem + stage * S::STAGE;
            uint8_t* sb = sa + S::A_BYTES;
            uint8_t* ssfa = sb + S::B_BYTES;
            uint8_t* ssfb = ssfa + S::SFA_BYTES;
            const int k_sf_row = kb * 8;  // 4 atoms of 512 B per stage = 8 rows of 256 B
            if constexpr (CL == 2) {
              const uint32_t fb = full0 + (uint32_t)stage * 8u;
              if (crank == 0) {
                const uint32_t a_cnt = 1 + (dummy1 ? 0 : 1);
                mbar_arrive_expect_tx(&full[stage], 2 * S::B_BYTES + 2 * S::SFB_BYTES +
                                                        a_cnt * S::A_BYTES +
                                                        (load_a_sf ? a_cnt * S::SFA_BYTES : 0));
              }
              if (!dummy) {
                tma_load_2d_2sm(sa, &tmA, fb, kb * kF4BKB, a_row);
                if (load_a_sf) tma_load_2d_2sm(ssfa, &tmSfa, fb, 0, sfa_row + k_sf_row);
              }
              tma_load_2d_2sm(sb, &tmB, fb, kb * kF4BKB, brow + (int)crank * (kF4BN / 2));
              tma_load_2d_2sm(ssfb, &tmSfb, fb, 0, sfb_row + k_sf_row);
              tma_load_2d_2sm(ssfb + 2048, &tmSfb, fb, 0, sfb_row + atoms_per_row_tile * 2 + k_sf_row);
            } else {
              // 1-CTA: the scale runs are plain bulk copies (no 2-SM signalling needed), one
              // 512-B atom per 64-wide k-group of this stage: a short last stage (K % 256)
              // must not read past its row tile's scales (or past the end of the buffer)
              const uint32_t sf_bytes = (uint32_t)min(4, K / 64 - kb * 4) * 512u;
              mbar_arrive_expect_tx(&full[stage], S::A_BYTES + S::B_BYTES + 2 * sf_bytes +
                                                      (load_a_sf ? sf_bytes : 0));
              tma_load_2d(sa, &tmA, &full[stage], kb * kF4BKB, a_row);
              tma_load_2d(sb, &tmB, &full[stage], kb * kF4BKB, brow);
              if (load_a_sf) bulk_load(ssfa, args.a_sf + (int64_t)(sfa_row + k_sf_row) * 256, sf_bytes, &full[stage]);
              bulk_load(ssfb, args.w_sf + (int64_t)(sfb_row + k_sf_row) * 256, sf_bytes, &full[stage]);
              bulk_load(ssfb + 2048, args.w_sf + (int64_t)(sfb_row + atoms_per_row_tile * 2 + k_sf_row) * 256,
                        sf_bytes, &full[stage]);
            }
          }
          __syncwarp();
          if (++stage == kF4Stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1 && crank == 0) {  // ---------------- MMA issuer (pair leader)
    const bool leader = elect_one();
    constexpr uint32_t idesc = idesc_nvfp4(kF4BM * CL, kF4BN);
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t tsfa = tbase + kTmemSfa;
    const uint32_t tsfb0 = tsfa + sfa_cols;
    const uint32_t s0 = smem_u32(smem);
    const uint64_t adesc0 = umma_desc_sw128(s0);
    const uint64_t bdesc0 = umma_desc_sw128(s0 + S::A_BYTES);
    const uint64_t sfadesc0 = sf_desc(s0 + S::A_BYTES + S::B_BYTES, args.sf_lbo, args.sf_sbo);
    const uint64_t sfbdesc0 = sf_desc(s0 + S::A_BYTES + S::B_BYTES + S::SFA_BYTES, args.sf_lbo, args.sf_sbo);
    const bool copy_sf = !(args.dbg & 2u);
    auto utccp = [&](uint32_t t, uint64_t d) {
      if constexpr (CL == 2) utccp_32x128b_warpx4_2sm(t, d);
      else utccp_32x128b_warpx4(t, d);
    };
    int stage = 0;
    uint32_t phase = 0, sfsel = 0;
    int tile_it = 0;  // accumulator use count (one per n-tile)
    for (int it = 0;; ++it) {
      const int slot = it % kF4Ring;
      mbar_wait(&slot_full[slot], (it / kF4Ring) & 1);
      const int u = __shfl_sync(0xffffffffu, slot_tile[slot], 0);
      __syncwarp();
      if (leader) mbar_arrive_relaxed(&slot_empty[slot]);
      if (u < 0) break;
      const int mu = u / nchunks, nt0 = (u - mu * nchunks) * kNPerUnit;
      const int nt1 = min(n_tiles, nt0 + kNPerUnit);
      for (int nt = nt0; nt < nt1; ++nt, ++tile_it) {
        // previous n-tile drained by the epilogue(s) => every earlier MMA completed,
        // so the resident A scales may be rewritten at the start of a new unit
        if (!(args.dbg & 16u)) mbar_wait(tempty, (tile_it & 1) ^ 1);  // dbg 16: no accumulator hand-off
        tc_fence_after();
        const bool load_a_sf = nt == nt0;
        for (int kb = 0; kb < nkb; ++kb) {
          const int nmma = min(kF4BKB, kbytes - kb * kF4BKB) / 32;
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t soff = (uint64_t)((uint32_t)(stage * S::STAGE) >> 4);
          const uint32_t tsfb = tsfb0 + sfsel * 32;
          if (leader) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if (j < nmma && copy_sf) {
                if (load_a_sf) utccp(tsfa + (kb * 4 + j) * 4, sfadesc0 + soff + 32 * j);
                utccp(tsfb + 8 * j, sfbdesc0 + soff + 32 * j);
                utccp(tsfb + 8 * j + 4, sfbdesc0 + soff + 128 + 32 * j);
              }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (j < nmma && !(args.dbg & 4u)) {
                if constexpr (CL == 2)
                  umma_nvfp4_2sm(tbase + kTmemAcc, adesc0 + soff + 2 * j, bdesc0 + soff + 2 * j, idesc,
                                 tsfa + (kb * 4 + j) * 4, tsfb + 8 * j, (kb | j) != 0);
                else
                  umma_nvfp4(tbase + kTmemAcc, adesc0 + soff + 2 * j, bdesc0 + soff + 2 * j, idesc,
                             tsfa + (kb * 4 + j) * 4, tsfb + 8 * j, (kb | j) != 0);
              }
            if constexpr (CL == 2) tc_commit_2sm_mc(&empty[stage], kBoth);
            else tc_commit(&empty[stage]);
          }
          __syncwarp();
          sfsel ^= 1;
          if (++stage == kF4Stages) { stage = 0; phase ^= 1; }
        }
        if (leader && !(args.dbg & 16u)) {
          if constexpr (CL == 2) tc_commit_2sm_mc(tfull, kBoth);
          else tc_commit(tfull);
        }
        __syncwarp();
      }
    }
    if (args.dbg & 16u) {  // debug: nobody else waited for the MMAs; drain them before the TMEM dealloc
      if (leader) {
        if constexpr (CL == 2) tc_commit_2sm_mc(tfull, kBoth);
        else tc_commit(tfull);
      }
      __syncwarp();
      mbar_wait(tfull, 0);
    }
  } else if (warp >= 4) {  // ---------------- epilogue (8 warps per CTA)
    const int q = warp & 3, half = (warp - 4) >> 2;
    const int row_in_tile = q * 32 + lane;
    int tile_it = 0;
    int sbuf = 0;  // next STORE staging buffer of this warp
    for (int it = 0;; ++it) {
      const int slot = it % kF4Ring;
      mbar_wait(&slot_full[slot], (it / kF4Ring) & 1);
      const int u = slot_tile[slot];
      __syncwarp();
      if (lane == 0) arrive_leader(&slot_empty[slot]);
      if (u < 0) break;
      const int mu = u / nchunks, nt0 = (u - mu * nchunks) * kNPerUnit;
      const int nt1 = min(n_tiles, nt0 + kNPerUnit);
      bool dummy;
      const TileCoord cm = mtile_of(mu, (int)crank, dummy);
      for (int nt = nt0; nt < nt1; ++nt, ++tile_it) {
      TileCoord c = cm;
      c.n0 = nt * kF4BN;
      if (args.dbg & 16u) continue;  // debug: no accumulator hand-off (mainloop alone)
      mbar_wait(tfull, tile_it & 1);
      tc_fence_after();
      const uint32_t tb = tmem_base + kTmemAcc + ((uint32_t)(q * 32) << 16);
      if (args.dbg & 8u) {  // debug: release the accumulator unread (cost of the TMEM drain)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_leader(tempty);
        continue;
      }
      uint32_t v[4][32];
      if constexpr (EPI == REALB_EPI_SWIGLU) {
        tmem_ld32(tb + half * 64, v[0]);
        tmem_ld32(tb + half * 64 + 32, v[1]);
        tmem_ld32(tb + 128 + half * 64, v[2]);
        tmem_ld32(tb + 128 + half * 64 + 32, v[3]);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) tmem_ld32(tb + half * 128 + 32 * i, v[i]);
      }
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_leader(tempty);  // accumulator free: next mainloop may start
      if ((args.dbg & 1u) || dummy) continue;
      const int64_t r = (int64_t)c.a_row + row_in_tile;
      if constexpr (EPI == kEpiScatter) {  // bf16 rows straight to their sources' return windows
        const int32_t smap = row_in_tile < c.valid ? __ldg(args.scat.row_map + r) : -1;
        const uint32_t ebuf = smem_u32(smem + S::EPI_OFF + (warp - 4) * (kF4EpiBufs * 2048));
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t p[16];
#pragma unroll
          for (int j = 0; j < 16; ++j)
            p[j] = pack_bf16x2(__uint_as_float(v[i][2 * j]), __uint_as_float(v[i][2 * j + 1]));
          const uint32_t b = ebuf + (i & 1) * 2048;  // two chunks staged -> 128-B row segments
#pragma unroll
          for (int cc = 0; cc < 4; ++cc)
            st_shared_v4(b + lane * 64 + ((cc ^ ((lane >> 1) & 3)) << 4), p[4 * cc], p[4 * cc + 1],
                         p[4 * cc + 2], p[4 * cc + 3]);
          if (i & 1) {
            __syncwarp();
            scatter_chunks<2>(ebuf, args.scat, smap, (int64_t)(c.n0 + half * 128 + 32 * (i - 1)) * 2);
            __syncwarp();
          }
        }
        continue;
      }
      if constexpr (EPI == REALB_EPI_SWIGLU) {
        // outputs [n0/2 + half*64, +64): h = bf16(silu(g) * u), then NVFP4
        const int I = N / 2;
        const int ocol = c.n0 / 2 + half * 64;
        uint32_t sfw = 0;
        uint2 cw[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          float h[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int col = b * 16 + i;  // 0..63
            const float g = __uint_as_float(v[col >> 5][col & 31]);
            const float u = __uint_as_float(v[2 + (col >> 5)][col & 31]);
            h[i] = __bfloat162float(__float2bfloat16_rn(__fdividef(g, 1.0f + __expf(-g)) * u));
          }
          uint32_t sb;
          cw[b] = quant_block16_bf16vals_fast(h, sb);
          sfw |= sb << (8 * b);
          if (args.out) {  // parity hook: the bf16 SwiGLU values the re-quantisation consumed
            uint32_t hp[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) hp[i] = pack_bf16x2(h[2 * i], h[2 * i + 1]);
            uint4* hd = reinterpret_cast<uint4*>(args.out + r * I + ocol + b * 16);
            hd[0] = make_uint4(hp[0], hp[1], hp[2], hp[3]);
            hd[1] = make_uint4(hp[4], hp[5], hp[6], hp[7]);
          }
        }
        uint4* cdst = reinterpret_cast<uint4*>(args.out_codes + r * (I / 2) + ocol / 2);
        cdst[0] = make_uint4(cw[0].x, cw[0].y, cw[1].x, cw[1].y);
        cdst[1] = make_uint4(cw[2].x, cw[2].y, cw[3].x, cw[3].y);
        *reinterpret_cast<uint32_t*>(args.out_sf + sf_mma_offset(r, ocol / 16, I / 16)) = sfw;
      } else {  // bf16 out via smem staging (SWIZZLE_64B) + TMA store, 32 columns at a time
        const int wi = warp - 4;
        const uint32_t ebuf = smem_u32(smem + S::EPI_OFF + wi * (kF4EpiBufs * 2048));
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t p[16];
#pragma unroll
          for (int j = 0; j < 16; ++j)
            p[j] = pack_bf16x2(__uint_as_float(v[i][2 * j]), __uint_as_float(v[i][2 * j + 1]));
          if (lane == 0) bulk_wait_group_read<kF4EpiBufs - 1>();
          __syncwarp();
          const uint32_t buf = ebuf + (uint32_t)(sbuf * 2048);
#pragma unroll
          for (int cc = 0; cc < 4; ++cc)
            st_shared_v4(buf + lane * 64 + ((cc ^ ((lane >> 1) & 3)) << 4), p[4 * cc], p[4 * cc + 1],
                         p[4 * cc + 2], p[4 * cc + 3]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0 && !(args.dbg & 32u)) {  // dbg 32: staged, never stored; 64: every store to tile 0
            const bool same = args.dbg & 64u;
            tma_store_2d(&tmOut, smem + S::EPI_OFF + wi * (kF4EpiBufs * 2048) + sbuf * 2048,
                         same ? 32 * i : c.n0 + half * 128 + 32 * i, same ? q * 32 : c.a_row + q * 32);
            bulk_commit_group();
          }
          sbuf = sbuf + 1 == kF4EpiBufs ? 0 : sbuf + 1;
        }
      }
      }
    }
  }
  if constexpr (EPI == REALB_EPI_STORE) {
    if (warp >= 4 && lane == 0) bulk_wait_group<0>();
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CL == 2) cluster_sync();  // no peer may still load / arrive / read our smem
  tc_fence_after();
  if (warp == 2) {
    if constexpr (CL == 2) tmem_dealloc_2sm<512>(tmem_base);
    else tmem_dealloc<512>(tmem_base);
  }
  if (threadIdx.x == 0) GroupedSched::finish(args.layout, REALB_PREC_W4A4);
}

// gemm_fp4_pair.cu
int fp4_pair_supported(int epilogue, int N, int K);
int fp4_pair(int epilogue, const uint8_t* a, const uint8_t* a_sf, const uint8_t* w, const uint8_t* w_sf,
             int64_t rows_cap, int N, int K, int E, const int32_t* layout, void* out, uint8_t* out_codes,
             uint8_t* out_sf, int max_ctas, uint32_t sf_lbo, uint32_t sf_sbo, uint32_t dbg, cudaStream_t st);

static uint32_t env_u32(const char* name, uint32_t dflt) {
  const char* s = getenv(name);
  return s ? (uint32_t)strtoul(s, nullptr, 0) : dflt;
}

// scale bytes of `rows` x K/16 viewed as [bytes/256][256] for the TMA loads
static int make_sf_map(CUtensorMap* m, const uint8_t* sf, int64_t rows, int K) {
  const uint64_t bytes = (uint64_t)rows * (uint64_t)(K / 16);
  return make_tmap_2d(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, sf, 256, bytes / 256, 256, 256, kSfBoxRows,
                      CU_TENSOR_MAP_SWIZZLE_NONE);
}

template <int EPI, int CL, int XST = 0>
static int launch_fp4(const uint8_t* a, const uint8_t* a_sf, const uint8_t* w, const uint8_t* w_sf,
                      int64_t rows_cap, int N, int K, int E, const int32_t* layout, void* out,
                      uint8_t* out_codes, uint8_t* out_sf, int max_ctas, cudaStream_t st,
                      const RowScatter* scat = nullptr) {
  CUtensorMap ta, tb, tsa, tsb, to;
  int rc = make_tmap_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT8, a, (uint64_t)K / 2, rows_cap,
                        (uint64_t)K / 2, kF4BKB, kF4BM, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  rc = make_tmap_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, w, (uint64_t)K / 2, (uint64_t)E * N,
                    (uint64_t)K / 2, kF4BKB, kF4BN / CL, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  rc = make_sf_map(&tsa, a_sf, rows_cap, K);
  if (rc) return rc;
  rc = make_sf_map(&tsb, w_sf, (int64_t)E * N, K);
  if (rc) return rc;
  if (EPI != REALB_EPI_SWIGLU && out) {
    rc = make_tmap_2d(&to, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, out, N, rows_cap, (uint64_t)N * 2, 32, 32,
                      CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
  } else {
    to = ta;  // unused
  }
  Fp4Args args;
  args.a_sf = a_sf;
  args.w_sf = w_sf;
  args.layout = layout;
  args.E = E;
  args.N = N;
  args.K = K;
  args.out = reinterpret_cast<__nv_bfloat16*>(out);
  args.out_codes = out_codes;
  args.out_sf = out_sf;
  args.sf_lbo = env_u32("REALB_DBG_SF_LBO", 128);
  args.sf_sbo = env_u32("REALB_DBG_SF_SBO", 128);
  args.dbg = env_u32("REALB_DBG_FP4", 0);
  args.scat = scat ? *scat : RowScatter{};
  auto kern = grouped_gemm_fp4_kernel<EPI, CL, XST>;
  const int smem = SmemFp4<EPI, CL, XST>::TOTAL;
  rc = set_smem_once(reinterpret_cast<const void*>(kern), smem, "grouped_gemm_nvfp4: smem attribute");
  if (rc) return rc;
  int grid = num_sms();
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  grid = grid / CL * CL;
  if (grid < CL) grid = CL;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kF4Threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  rc = cuda_status(cudaLaunchKernelEx(&cfg, kern, ta, tb, tsa, tsb, to, args),
                   "realb_grouped_gemm_nvfp4 launch");
  if (rc) return rc;
  return check_launch("realb_grouped_gemm_nvfp4");
}

}  // namespace realb

using namespace realb;

extern "C" int realb_grouped_gemm_nvfp4(const uint8_t* d_a_codes, const uint8_t* d_a_sf,
                                        const uint8_t* d_w_codes, const uint8_t* d_w_sf,
                                        int64_t rows_cap, int N, int K, int E,
                                        const int32_t* d_layout, int epilogue, void* d_out,
                                        uint8_t* d_out_codes, uint8_t* d_out_sf, int max_ctas,
                                        void* stream) {
  if (!d_a_codes || !d_a_sf || !d_w_codes || !d_w_sf || !d_layout || rows_cap <= 0 ||
      rows_cap % 128 || E <= 0) {
    set_error("realb_grouped_gemm_nvfp4: bad arguments");
    return REALB_EINVAL;
  }
  if (N % kF4BN || K % 64 || K > 3072) {
    set_error("realb_grouped_gemm_nvfp4: needs N %% 256 == 0, K %% 64 == 0 and K <= 3072 (resident "
              "A scales: K/16 TMEM columns) (N=%d K=%d)", N, K);
    return REALB_EUNSUPPORTED;
  }
  cudaStream_t st = (cudaStream_t)stream;
  // Kernel choice (all forms give bit-identical results; tests/test_gemm_fp4_gpu.py):
  //  * STORE (down GEMM): K6 v2 (gemm_fp4_pair.cu: 2-SM pairs, the A operand resident in
  //    smem for a unit of n-tiles), measured 0.224 vs 0.257 ms (v1 1-CTA) on the EP8 hot
  //    rank (scripts/bench_k6_v2.py);
  //  * SWIGLU (gate_up): v1 in its 2-CTA pair form. The v2 form has no edge there (the
  //    128 KB A reload per unit stalls as much as the streamed A costs).
  // REALB_K6_VERSION=1 forces v1 (REALB_GEMM_CLUSTER=1|2 then picks its form),
  // REALB_K6_VERSION=2 forces v2 where it is supported.
  const char* cl_env = getenv("REALB_GEMM_CLUSTER");
  const char* ver = getenv("REALB_K6_VERSION");
  const bool cl_set = cl_env && cl_env[0];
  const bool v1_forced = (ver && ver[0] == '1') || cl_set;
  auto use_v2 = [&](int epi) {
    if (!fp4_pair_supported(epi, N, K) || v1_forced) return false;
    return epi == REALB_EPI_STORE || (ver && ver[0] == '2');
  };
  // v1 form: pair unless REALB_GEMM_CLUSTER=1, or REALB_K6_VERSION=1 without a cluster
  // choice (the 1-CTA kernel, as in round 1)
  const bool pair = cl_set ? cl_env[0] == '2' : !(ver && ver[0] == '1');
  if (epilogue == REALB_EPI_STORE) {
    if (!d_out) { set_error("realb_grouped_gemm_nvfp4: STORE needs d_out"); return REALB_EINVAL; }
    if (use_v2(REALB_EPI_STORE))
      return fp4_pair(REALB_EPI_STORE, d_a_codes, d_a_sf, d_w_codes, d_w_sf, rows_cap, N, K, E, d_layout, d_out,
                      nullptr, nullptr, max_ctas, env_u32("REALB_DBG_SF_LBO", 128), env_u32("REALB_DBG_SF_SBO", 128),
                      env_u32("REALB_DBG_FP4", 0), st);
    const char* xst = getenv("REALB_DBG_FP4_STORE4");
    if (xst && xst[0] == '1' && !pair) {
      if (!(env_u32("REALB_DBG_FP4", 0) & 1u)) {
        set_error("REALB_DBG_FP4_STORE4 is an experiment: it needs REALB_DBG_FP4 bit 1 (no epilogue stores)");
        return REALB_EINVAL;
      }
      return launch_fp4<REALB_EPI_STORE, 1, 4>(d_a_codes, d_a_sf, d_w_codes, d_w_sf, rows_cap, N, K, E, d_layout,
                                               d_out, nullptr, nullptr, max_ctas, st);
    }
    return pair ? launch_fp4<REALB_EPI_STORE, 2>(d_a_codes, d_a_sf, d_w_codes, d_w_sf, rows_cap, N, K, E,
                                                 d_layout, d_out, nullptr, nullptr, max_ctas, st)
                : launch_fp4<REALB_EPI_STORE, 1>(d_a_codes, d_a_sf, d_w_codes, d_w_sf, rows_cap, N, K, E,
                                                 d_layout, d_out, nullptr, nullptr, max_ctas, st);
  }
  if (epilogue == REALB_EPI_SWIGLU) {
    if (!d_out_codes || !d_out_sf || (N / 2) % 64) {
      set_error("realb_grouped_gemm_nvfp4: SWIGLU needs d_out_codes/d_out_sf and (N/2) %% 64 == 0");
      return REALB_EINVAL;
    }
    // d_out (optional, SWIGLU): also store the bf16 SwiGLU values the re-quantisation consumed
    if (use_v2(REALB_EPI_SWIGLU))
      return fp4_pair(REALB_EPI_SWIGLU, d_a_codes, d_a_sf, d_w_codes, d_w_sf, rows_cap, N, K, E, d_layout, d_out,
                      d_out_codes, d_out_sf, max_ctas, env_u32("REALB_DBG_SF_LBO", 128),
                      env_u32("REALB_DBG_SF_SBO", 128), env_u32("REALB_DBG_FP4", 0), st);
    return pair ? launch_fp4<REALB_EPI_SWIGLU, 2>(d_a_codes, d_a_sf, d_w_codes, d_w_sf, rows_cap, N, K, E,
                                                  d_layout, d_out, d_out_codes, d_out_sf, max_ctas, st)
                : launch_fp4<REALB_EPI_SWIGLU, 1>(d_a_codes, d_a_sf, d_w_codes, d_w_sf, rows_cap, N, K, E,
                                                  d_layout, d_out, d_out_codes, d_out_sf, max_ctas, st);
  }
  set_error("realb_grouped_gemm_nvfp4: unknown epilogue %d", epilogue);
  return REALB_EINVAL;
}

extern "C" int realb_grouped_gemm_nvfp4_scatter(const uint8_t* d_a_codes, const uint8_t* d_a_sf,
                                                const uint8_t* d_w_codes, const uint8_t* d_w_sf, int64_t rows_cap,
                                                int N, int K, int E, const int32_t* d_layout,
                                                const int32_t* d_row_map, int n_dst, const uint64_t* h_dst_bases,
                                                int max_ctas, void* stream) {
  if (!d_a_codes || !d_a_sf || !d_w_codes || !d_w_sf || !d_layout || !d_row_map || !h_dst_bases ||
      rows_cap <= 0 || rows_cap % 128 || E <= 0 || n_dst < 1 || n_dst > kScatterPeers) {
    set_error("realb_grouped_gemm_nvfp4_scatter: bad arguments");
    return REALB_EINVAL;
  }
  if (N % kF4BN || K % 64 || K > 3072) {
    set_error("realb_grouped_gemm_nvfp4_scatter: needs N %% 256 == 0, K %% 64 == 0 and K <= 3072 (N=%d K=%d)",
              N, K);
    return REALB_EUNSUPPORTED;
  }
  RowScatter sc{};
  for (int d = 0; d < n_dst; ++d) {
    if (h_dst_bases[d] & 15) {
      set_error("realb_grouped_gemm_nvfp4_scatter: destination %d not 16-B aligned", d);
      return REALB_EINVAL;
    }
    sc.base[d] = reinterpret_cast<uint8_t*>(h_dst_bases[d]);
  }
  sc.row_map = d_row_map;
  sc.ld = (int64_t)N * 2;
  return launch_fp4<kEpiScatter, 1>(d_a_codes, d_a_sf, d_w_codes, d_w_sf, rows_cap, N, K, E, d_layout, nullptr,
                                    nullptr, nullptr, max_ctas, (cudaStream_t)stream, &sc);
}
