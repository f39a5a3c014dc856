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
//
// Gather form (realb_grouped_gemm_bf16_gather): A is not a grouped operand but
// the token matrix x itself; grouped row g reads x[row_src[g]]. Warps 2-3 load
// the A tile with 16-B cp.async.cg (each warp 64 rows; lane -> 16-B piece of a
// row, stored at its SWIZZLE_128B position) and signal the stage's full barrier
// with cp.async.mbarrier.arrive.noinc; warp 0 keeps the W tile on TMA. Rows past
// the m-block's valid count are zero-filled (src-size 0). This removes the
// dispatch row copy (2H B written + re-read per pair) and keeps the x rows, read
// up to k times, L2-resident. (TMA tile::gather4 gives the same smem image but
// was measured 2.4x slower here: 32 gather4 per 16 KB stage, ~77 cycles each.)
#include <cstdlib>

#include "common.cuh"
#include "grouped.cuh"

namespace realb {

constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 bf16 = 128 B rows = one SWIZZLE_128B atom width
// TMA-store staging buffers per epilogue warp: a warp reuses a buffer only after
// the store issued kEpiBufs chunks earlier has read it (bulk wait_group.read)
constexpr int kEpiBufs = 4;

template <int BN, int STAGES, int CL>
struct SmemBf16 {
  static constexpr int A_BYTES = kBM * kBK * 2;
  static constexpr int B_BYTES = (BN / CL) * kBK * 2;  // a pair stages half of W per CTA
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int EPI_OFF = STAGES * STAGE_BYTES;       // 4 warps x kEpiBufs x (32 rows x 64 B)
  static constexpr int EPI_BYTES = 4 * kEpiBufs * 2048;
  static constexpr int BAR_OFF = EPI_OFF + EPI_BYTES;
  static constexpr int TOTAL = BAR_OFF + 512 + 1024;  // + barriers/slots + alignment slack
};

constexpr int kTileRing = 4;  // depth of the dynamic tile-id ring (producer -> MMA/epilogue)

// silu(g) * u = g / (1 + e^-g) * u with the approximate divide (MUFU.RCP + FMUL):
// the epilogue's math is on the GEMM's critical path (K5), and the
// IEEE division (or __frcp_rn) costs a multi-instruction sequence per element:
// measured on the Kimi gate_up (interleaved) 0.478 vs 0.494 ms (IEEE division) vs
// 0.482 ms (silu as 0.5 g (1 + tanh.approx(g / 2))); same form as K6's epilogue
__device__ __forceinline__ float silu_mul(float g, float u) {
  return __fdividef(g, 1.0f + __expf(-g)) * u;
}
// 32 rows x 32 bf16 (64 B) staging chunk, TMA SWIZZLE_64B layout: the 16-B piece
// c of row r lives at piece c ^ ((r >> 1) & 3) -> conflict-free 16-B smem stores.
__device__ __forceinline__ void stage_row64(uint32_t buf, int r, const uint32_t (&p)[16]) {
#pragma unroll
  for (int c = 0; c < 4; ++c)
    st_shared_v4(buf + r * 64 + ((c ^ ((r >> 1) & 3)) << 4), p[4 * c], p[4 * c + 1], p[4 * c + 2],
                 p[4 * c + 3]);
}

// CL = 1: one CTA per SM, tcgen05.mma.cta_group::1, M = 128.
// CL = 2: a 2-CTA cluster is one tcgen05 "CTA pair" (cta_group::2, M = 256):
//   CTA r stages ITS 128 A rows and HALF of the W tile (W rows 128r..128r+127);
//   the leader (rank 0) issues the pair MMA, which reads A/W from both CTAs'
//   smem and accumulates rows 128r.. in CTA r's TMEM. Halving the W bytes staged
//   per CTA lets 6 stages fit instead of 4: the 1-CTA kernel was bound by
//   operand bytes in flight (TMA-only time 0.38 of 0.49 ms on the 1-GPU gate_up).
//   Both CTAs' loads complete on the leader's full barrier; the leader's
//   multicast commits release both CTAs' stages and publish both accumulators.
__device__ __forceinline__ void cp_async_16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
constexpr int kGatherWarps = 2;  // warps 2..3 load A in the gather form

// copy-in form: warps 2-3 of every CTA copy the dispatch rows x[row_src[g]] -> A[g]
// (the class's valid rows, in grouped order across the grid) while the mainloop
// runs; per-expert row counters (release) gate the producer's first load of an
// expert's tiles (acquire). The copy overlaps the GEMM instead of preceding it.
__device__ __forceinline__ int ld_acquire_gpu(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
struct CopyIn {
  const __nv_bfloat16* x;  // token rows [*, K]
  const int32_t* row_src;  // grouped row -> token
  __nv_bfloat16* a;        // the A operand [rows_cap, K] (also read by TMA)
  int32_t* ready;          // [E] rows copied per expert (zero on entry; the last CTA re-zeroes)
  int32_t* err;            // bit 2: a producer wait timed out
};

template <int BN, int STAGES, int EPI, int CL, bool GATHER, bool COPYIN = false>
__global__ void __launch_bounds__(256, 1)
    grouped_gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA,
                             const __grid_constant__ CUtensorMap tmB,
                             const __grid_constant__ CUtensorMap tmOut, const int32_t* layout,
                             int E, int prec, int N, int K, uint32_t dbg,
                             const __nv_bfloat16* __restrict__ xsrc, const int32_t* __restrict__ row_src,
                             const __grid_constant__ RowScatter scat, const CopyIn cin) {
  static_assert(!GATHER || CL == 1, "the gather form is 1-CTA only");
  using S = SmemBf16<BN, STAGES, CL>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* slot_full = tempty + 2;
  uint64_t* slot_empty = slot_full + kTileRing;
  int32_t* slot_tile = reinterpret_cast<int32_t*>(slot_empty + kTileRing);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(slot_tile + kTileRing);

  const int warp = warp_id(), lane = lane_id();
  const uint32_t crank = CL == 2 ? cluster_ctarank() : 0u;
  const GroupedSched sched = GroupedSched::make(layout, E, prec, N, BN);
  const int total = CL == 2 ? sched.total_pairs() : sched.total();
  const int nkb = K / kBK;
  constexpr uint16_t kBoth = 0x3;
  // consumers of a tile-id slot: 1-CTA: MMA + 4 epilogue warps; pair: leader MMA +
  // 4 leader epilogue warps + peer producer + 4 peer epilogue warps
  // gather form: + the two A-loader warps
  constexpr uint32_t kSlotConsumers = CL == 2 ? 10 : (GATHER ? 5 + kGatherWarps : 5);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmOut);
    for (int s = 0; s < STAGES; ++s) {
      // gather: + one noinc arrive per loader lane; the pair's no-load probe: one arrive
      // from each CTA's producer, so neither producer can be lapped by the MMA (a waiter
      // two phases behind an mbarrier never sees its phase complete)
      mbar_init(&full[s], GATHER ? 1 + 32 * kGatherWarps : (CL == 2 && (dbg & 2u)) ? 2 : 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4 * CL);
    }
    for (int i = 0; i < kTileRing; ++i) {
      mbar_init(&slot_full[i], 1);
      mbar_init(&slot_empty[i], kSlotConsumers);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (CL == 2) tmem_alloc_2sm<2 * BN>(tmem_slot);
    else tmem_alloc<2 * BN>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CL == 2) cluster_sync();  // peer barriers / TMEM ready before any remote op
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto tile_of = [&](int u, int rank, bool& dummy) -> TileCoord {
    if constexpr (CL == 2) return sched.coord_pair(u, rank, dummy);
    dummy = false;
    return sched.coord(u);
  };
  // arrive on a barrier of the pair leader (local barrier in a 1-CTA launch)
  auto arrive_leader = [&](uint64_t* bar) {
    // relaxed: these arrives only signal "slot value read" / "TMEM drained" (no memory
    // writes to publish); a release arrive waits for the warp's outstanding stores
    if constexpr (CL == 2) mbar_arrive_cluster_relaxed(mapa_shared(bar, 0));
    else mbar_arrive_relaxed(bar);
  };

  // Producer and MMA roles run on their whole warp with warp-uniform values and
  // one elected lane issuing (see gemm_fp4.cu: lane-0-only code makes ptxas wrap
  // every tcgen05 instruction in an ELECT/R2UR waterfall loop).
  if (warp == 0) {  // ---------------- TMA producer + dynamic tile fetch
    const bool leader = elect_one();
    int* ctr = GroupedSched::counters(layout, prec);
    const uint32_t full0 = CL == 2 ? mapa_shared(&full[0], 0) : smem_u32(&full[0]);
    int stage = 0;
    uint32_t phase = 0;
    int ready_group = -1;  // copy-in: last expert whose rows were seen complete
    // The leader claims its NEXT unit (atomic) and resolves its coordinates (a binary
    // search over the layout words) while the current unit's loads stream, so neither
    // latency stalls the loads at a unit boundary (the ring is only STAGES deep).
    bool have_ahead = false;
    int t_ahead = -1;
    TileCoord c_ahead{};
    bool dummy_ahead = false, dummy1_ahead = false;
    for (int i = 0;; ++i) {
      const int slot = i % kTileRing;
      int t = 0;
      if (crank == 0) {  // the (pair) leader fetches and publishes the unit
        mbar_wait(&slot_empty[slot], ((i / kTileRing) & 1) ^ 1);
        if (have_ahead) {
          t = t_ahead;
        } else if (leader) {
          t = atomicAdd(ctr, 1);
          if (t >= total) t = -1;
        }
        if (leader) {
          slot_tile[slot] = t;
          if constexpr (CL == 2) {
            st_cluster_u32(mapa_shared(&slot_tile[slot], 1), (uint32_t)t);
            mbar_arrive_cluster(mapa_shared(&slot_full[slot], 1));
          }
          mbar_arrive(&slot_full[slot]);
        }
        t = __shfl_sync(0xffffffffu, t, 0);
      } else {
        mbar_wait(&slot_full[slot], (i / kTileRing) & 1);
        t = __shfl_sync(0xffffffffu, slot_tile[slot], 0);
        __syncwarp();
        if (leader) arrive_leader(&slot_empty[slot]);
      }
      if (t < 0) break;
      bool dummy = false, dummy1 = false;
      TileCoord c;
      if (have_ahead) {
        c = c_ahead;
        dummy = dummy_ahead;
        dummy1 = dummy1_ahead;
      } else {
        c = tile_of(t, (int)crank, dummy);
        if constexpr (CL == 2) {
          if (crank == 0) { bool d1; (void)tile_of(t, 1, d1); dummy1 = d1; }
        }
      }
      have_ahead = false;
      int t_next = 0;  // leader lane: the atomic's result, consumed two stages later
      const int a_row = __shfl_sync(0xffffffffu, c.a_row, 0);
      const int brow = __shfl_sync(0xffffffffu, c.group * N + c.n0, 0);
      dummy = __shfl_sync(0xffffffffu, (int)dummy, 0) != 0;
      dummy1 = __shfl_sync(0xffffffffu, (int)dummy1, 0) != 0;
      if constexpr (COPYIN) {
        const int grp = __shfl_sync(0xffffffffu, c.group, 0);
        if (grp != ready_group) {
          if (leader) {
            const int need = sched.row_count[grp];
            long long spins = 0;
            while (ld_acquire_gpu(cin.ready + grp) < need) {
              __nanosleep(64);
              if (++spins > (1LL << 24)) {  // ~1 s: report instead of hanging
                atomicOr(cin.err, 4);
                break;
              }
            }
            fence_proxy_async_global();  // generic-proxy row stores -> TMA reads
          }
          __syncwarp();
          ready_group = grp;
        }
      }
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        if constexpr (GATHER) {  // W only; A comes from the loader warps
          if (leader) {
            mbar_arrive_expect_tx(&full[stage], S::B_BYTES);
            tma_load_2d(smem + stage * S::STAGE_BYTES + S::A_BYTES, &tmB, &full[stage], kb * kBK, brow);
          }
        } else if (leader) {
          uint8_t* sa = smem + stage * S::STAGE_BYTES;
          if constexpr (CL == 2) {
            const uint32_t fb = full0 + (uint32_t)stage * 8u;
            if (dbg & 2u) {  // debug: no operand loads (MMA + epilogue only); both producers arrive
              mbar_arrive_cluster(fb);
            } else {
              if (crank == 0)
                mbar_arrive_expect_tx(&full[stage], 2 * S::B_BYTES + S::A_BYTES + (dummy1 ? 0 : S::A_BYTES));
              if (!dummy) tma_load_2d_2sm(sa, &tmA, fb, kb * kBK, a_row);
              tma_load_2d_2sm(sa + S::A_BYTES, &tmB, fb, kb * kBK, brow + (int)crank * (BN / 2));
            }
          } else if (dbg & 2u) {  // debug: no operand loads (MMA + epilogue only)
            mbar_arrive(&full[stage]);
          } else {
            mbar_arrive_expect_tx(&full[stage], S::STAGE_BYTES);
            tma_load_2d(sa, &tmA, &full[stage], kb * kBK, a_row);
            tma_load_2d(sa + S::A_BYTES, &tmB, &full[stage], kb * kBK, brow);
          }
        }
        // (1-CTA form only; the pair form claims at the unit boundary as before)
        if (CL == 1 && !(dbg & 128u)) {  // (debug bit 128: claim at the unit boundary instead)
          if (kb == 0 && leader) t_next = atomicAdd(ctr, 1);  // after this stage's loads
          if (kb == (nkb > 2 ? 2 : nkb - 1)) {
            int tn = __shfl_sync(0xffffffffu, t_next, 0);
            if (tn >= total) tn = -1;
            t_ahead = tn;
            if (tn >= 0) {
              c_ahead = tile_of(tn, 0, dummy_ahead);
              if constexpr (CL == 2) { (void)tile_of(tn, 1, dummy1_ahead); }
            }
            have_ahead = true;
          }
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1 && crank == 0) {  // ---------------- MMA issuer (pair leader)
    const bool leader = elect_one();
    constexpr uint32_t idesc = idesc_bf16(kBM * CL, BN);
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t s0 = smem_u32(smem);
    const uint64_t adesc0 = umma_desc_sw128(s0), bdesc0 = umma_desc_sw128(s0 + S::A_BYTES);
    int stage = 0;
    uint32_t phase = 0;
    for (int i = 0;; ++i) {
      const int slot = i % kTileRing;
      mbar_wait(&slot_full[slot], (i / kTileRing) & 1);
      const int t = __shfl_sync(0xffffffffu, slot_tile[slot], 0);
      __syncwarp();
      if (leader) mbar_arrive_relaxed(&slot_empty[slot]);
      if (t < 0) break;
      const int acc = i & 1;
      mbar_wait(&tempty[acc], ((i >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t dtmem = tbase + acc * BN;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full[stage], phase);
        if constexpr (GATHER) fence_proxy_async_smem();  // cp.async (generic proxy) -> MMA reads
        tc_fence_after();
        const uint64_t soff = (uint64_t)((uint32_t)(stage * S::STAGE_BYTES) >> 4);
        if (leader) {
          if (!(dbg & 4u)) {
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {  // +32 B (16 bf16) inside the 128-B swizzle atom
              if constexpr (CL == 2)
                umma_bf16_2sm(dtmem, adesc0 + soff + 2 * k, bdesc0 + soff + 2 * k, idesc, (kb | k) != 0);
              else
                umma_bf16(dtmem, adesc0 + soff + 2 * k, bdesc0 + soff + 2 * k, idesc, (kb | k) != 0);
            }
          }
          if constexpr (CL == 2) tc_commit_2sm_mc(&empty[stage], kBoth);
          else tc_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (leader) {
        if constexpr (CL == 2) tc_commit_2sm_mc(&tfull[acc], kBoth);
        else tc_commit(&tfull[acc]);
      }
      __syncwarp();
    }
  } else if (COPYIN && (warp == 2 || warp == 3)) {  // ---------------- dispatch row copy (copy-in form)
    // compact index v over the class's valid rows (groups in glist order), strided
    // over every copy warp of the grid: increasing v = increasing grouped row
    const int nw = (int)gridDim.x * 2, wid = (int)blockIdx.x * 2 + (warp - 2);
    const int rowv = K / 8;  // uint4 per row
    int gi = 0, e = -1, cnt = 0, pending = 0;
    int64_t cum0 = 0;
    if (sched.G > 0) { e = sched.glist[0]; cnt = sched.row_count[e]; }
    auto flush = [&]() {
      if (pending) {  // all lanes: make this warp's row stores visible (both proxies), then count them
        fence_proxy_async_global();
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(cin.ready + e, pending);
        pending = 0;
      }
    };
    for (int64_t v = wid;; v += nw) {
      while (gi < sched.G && v >= cum0 + cnt) {
        flush();
        cum0 += cnt;
        if (++gi < sched.G) { e = sched.glist[gi]; cnt = sched.row_count[e]; }
      }
      if (gi >= sched.G) break;
      const int64_t g = sched.row_start[e] + (v - cum0);
      const uint4* src = reinterpret_cast<const uint4*>(cin.x + (int64_t)__ldg(cin.row_src + g) * K);
      uint4* dst = reinterpret_cast<uint4*>(cin.a + g * K);
      for (int i0 = 0; i0 < rowv; i0 += 32 * 8) {  // 8 loads in flight per lane, then the stores
        uint4 r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (i0 + j * 32 + lane < rowv) r[j] = __ldg(src + i0 + j * 32 + lane);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (i0 + j * 32 + lane < rowv) dst[i0 + j * 32 + lane] = r[j];
      }
      ++pending;
    }
    flush();
  } else if (GATHER && (warp == 2 || warp == 3)) {  // ---------------- A loaders (gather form)
    // warp w loads rows 64(w-2) .. +63 of the m-block: instruction i covers rows
    // 4i + lane/8 (16-B piece lane%8 of each), 16 instructions per k-block
    const int rsub = lane >> 3, piece = lane & 7;
    const int rbase = (warp - 2) * 64;
    const uint32_t s0 = smem_u32(smem);
    const int64_t ldx = K;  // x row stride (elements)
    int stage = 0;
    uint32_t phase = 0;
    for (int i = 0;; ++i) {
      const int slot = i % kTileRing;
      mbar_wait(&slot_full[slot], (i / kTileRing) & 1);
      const int t = slot_tile[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive_relaxed(&slot_empty[slot]);
      if (t < 0) break;
      bool dummy;
      const TileCoord c = tile_of(t, 0, dummy);
      const __nv_bfloat16* src[16];
      uint32_t nbytes = 0;  // bit j: row of instruction j is real
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        // padding rows (results never read) repeat a valid row of the tile rather than
        // zero-fill: zero operand rows slow the tensor pipe (data-dependent speed)
        const int r = rbase + 4 * j + rsub;
        const int rv = r < c.valid ? r : r % c.valid;
        src[j] = xsrc + (int64_t)__ldg(row_src + c.a_row + rv) * ldx + piece * 8;
        nbytes |= 1u << j;
      }
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        const uint32_t sa = s0 + stage * S::STAGE_BYTES;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int r = rbase + 4 * j + rsub;
          cp_async_16(sa + r * 128 + ((piece ^ (r & 7)) << 4), src[j] + kb * kBK, ((nbytes >> j) & 1u) * 16u);
        }
        cp_async_arrive_noinc(&full[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue: TMEM -> regs -> smem -> TMA store
    const int q = warp & 3;  // TMEM lane quadrant = 32-row slice of this CTA's 128 rows
    const uint32_t ebuf = smem_u32(smem + S::EPI_OFF + q * (kEpiBufs * 2048));
    int nbuf = 0;
    for (int i = 0;; ++i) {
      const int slot = i % kTileRing;
      mbar_wait(&slot_full[slot], (i / kTileRing) & 1);
      const int t = slot_tile[slot];
      __syncwarp();
      if (lane == 0) arrive_leader(&slot_empty[slot]);
      if (t < 0) break;
      bool dummy;
      const TileCoord c = tile_of(t, (int)crank, dummy);
      const int acc = i & 1;
      mbar_wait(&tfull[acc], (i >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem_base + acc * BN + ((uint32_t)(q * 32) << 16);
      const int row0 = c.a_row + q * 32;
      int32_t smap = -1;  // scatter: this lane's row -> destination (C3 fused)
      if constexpr (EPI == kEpiScatter)
        if (!dummy && q * 32 + lane < c.valid) smap = __ldg(scat.row_map + row0 + lane);
      if ((dbg & 1u) || dummy) {  // nothing to store: release the accumulator at once
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_leader(&tempty[acc]);
        continue;
      }
      constexpr int NCH = EPI == REALB_EPI_SWIGLU ? BN / 64 : BN / 32;
#pragma unroll 1
      for (int ch = 0; ch < NCH; ++ch) {
        uint32_t p[16];
        if constexpr (EPI != REALB_EPI_SWIGLU) {
          uint32_t v[32];
          tmem_ld32(tbase + ch * 32, v);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j)
            p[j] = pack_bf16x2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
        } else {  // SwiGLU: gate columns [0, BN/2), up columns [BN/2, BN) of the same outputs
          uint32_t g[32], u[32];
          tmem_ld32(tbase + ch * 32, g);
          tmem_ld32(tbase + BN / 2 + ch * 32, u);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j)
            p[j] = pack_bf16x2(silu_mul(__uint_as_float(g[2 * j]), __uint_as_float(u[2 * j])),
                               silu_mul(__uint_as_float(g[2 * j + 1]), __uint_as_float(u[2 * j + 1])));
        }
        if constexpr (EPI == kEpiScatter) {  // stage 4 chunks, then 256-B row segments
          static_assert(kEpiBufs == 4, "the scatter epilogue stages four chunks");
          stage_row64(ebuf + (ch & 3) * 2048, lane, p);
          if ((ch & 3) == 3) {
            __syncwarp();
            scatter_chunks<4>(ebuf, scat, smap, (int64_t)(c.n0 + (ch - 3) * 32) * 2);
            __syncwarp();
          }
          continue;
        }
        // the buffer about to be reused must have been read out by its TMA store
        if (lane == 0) bulk_wait_group_read<kEpiBufs - 1>();
        __syncwarp();
        const uint32_t buf = ebuf + nbuf * 2048;
        stage_row64(buf, lane, p);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          const int col = EPI == REALB_EPI_SWIGLU ? c.n0 / 2 + ch * 32 : c.n0 + ch * 32;
          tma_store_2d(&tmOut, smem + S::EPI_OFF + q * (kEpiBufs * 2048) + nbuf * 2048, col, row0);
          bulk_commit_group();
        }
        nbuf = nbuf + 1 == kEpiBufs ? 0 : nbuf + 1;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_leader(&tempty[acc]);
    }
    if (lane == 0) bulk_wait_group<0>();  // all stores of this CTA complete
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CL == 2) cluster_sync();  // no peer may still load / arrive / read our smem
  tc_fence_after();
  if (warp == 2) {
    if constexpr (CL == 2) tmem_dealloc_2sm<2 * BN>(tmem_base);
    else tmem_dealloc<2 * BN>(tmem_base);
  }
  if (threadIdx.x == 0) {
    if constexpr (COPYIN) {  // the last CTA re-zeroes the row counters for the next launch
      int* c = GroupedSched::counters(layout, prec);
      __threadfence();
      if (atomicAdd(c + 1, 1) == (int)gridDim.x - 1) {
        for (int i = 0; i < E; ++i) cin.ready[i] = 0;
        c[0] = 0;
        c[1] = 0;
        __threadfence();
      }
    } else {
      GroupedSched::finish(layout, prec);
    }
  }
}

template <int BN, int STAGES, int EPI, int CL, bool GATHER = false, bool COPYIN = false>
static int launch_grouped_bf16(const void* a, const void* w, int64_t rows_cap, int N, int K, int E,
                               const int32_t* layout, int prec, void* out, int max_ctas,
                               cudaStream_t st, const int32_t* row_src = nullptr,
                               const RowScatter* scat = nullptr, const CopyIn* copyin = nullptr) {
  CUtensorMap ta, tb, to;
  // gather form: A is read by the loader warps (the A map is unused, built over x)
  int rc = make_tmap_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, a, K, GATHER ? 1 : rows_cap, (uint64_t)K * 2,
                        kBK, GATHER ? 1 : kBM, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  rc = make_tmap_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, w, K, (uint64_t)E * N, (uint64_t)K * 2,
                    kBK, BN / CL, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  const int NO = EPI == REALB_EPI_SWIGLU ? N / 2 : N;
  // scatter: no output tensor (the map is built over the A operand, never used)
  rc = make_tmap_2d(&to, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, EPI == kEpiScatter ? a : out, NO,
                    EPI == kEpiScatter ? 1 : rows_cap, (uint64_t)NO * 2, 32, EPI == kEpiScatter ? 1 : 32,
                    CU_TENSOR_MAP_SWIZZLE_64B);
  if (rc) return rc;
  auto kern = grouped_gemm_bf16_kernel<BN, STAGES, EPI, CL, GATHER, COPYIN>;
  const int smem = SmemBf16<BN, STAGES, CL>::TOTAL;
  rc = set_smem_once(reinterpret_cast<const void*>(kern), smem, "grouped_gemm_bf16: smem attribute");
  if (rc) return rc;
  int grid = num_sms();
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  grid = grid / CL * CL;
  if (grid < CL) grid = CL;
  const char* dbg_env = getenv("REALB_DBG_BF16");
  const uint32_t dbg = dbg_env ? (uint32_t)strtoul(dbg_env, nullptr, 0) : 0u;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  RowScatter sc{};
  if (scat) sc = *scat;
  CopyIn ci{};
  if (copyin) ci = *copyin;
  rc = cuda_status(cudaLaunchKernelEx(&cfg, kern, ta, tb, to, layout, E, prec, N, K, dbg,
                                      reinterpret_cast<const __nv_bfloat16*>(a), row_src, sc, ci),
                   "realb_grouped_gemm_bf16 launch");
  if (rc) return rc;
  return check_launch("realb_grouped_gemm_bf16");
}

}  // namespace realb

using namespace realb;

extern "C" int realb_grouped_gemm_bf16(const void* d_a, const void* d_w, int64_t rows_cap, int N,
                                       int K, int E, const int32_t* d_layout, int prec,
                                       int epilogue, void* d_out, int max_ctas, void* stream) {
  // rows_cap only bounds the A / out tensor maps: rows past it read as zero (TMA
  // OOB fill) and are never stored, so a dense operand of any row count works
  if (!d_a || !d_w || !d_layout || !d_out || rows_cap <= 0 || E <= 0 ||
      (prec != REALB_PREC_W16A16 && prec != REALB_PREC_W4A4)) {
    set_error("realb_grouped_gemm_bf16: bad arguments");
    return REALB_EINVAL;
  }
  if (K % kBK || N % 256) {
    set_error("realb_grouped_gemm_bf16: needs K %% 64 == 0 and N %% 256 == 0 (N=%d K=%d)", N, K);
    return REALB_EUNSUPPORTED;
  }
  cudaStream_t st = (cudaStream_t)stream;
  // 1-CTA tiles by default. The 2-CTA pair form (cta_group::2, 6 stages; same
  // results) halves the W bytes per SM and its TMA-only time drops, but measured
  // interleaved against the 1-CTA kernel it was slower on every shape
  // (scripts/bench_gemm.py: Kimi EP8 hot rank gate_up 0.876 vs 0.840 ms, 1-GPU
  // layer 0.493 vs 0.469 ms). REALB_GEMM_CLUSTER=2 selects it.
  const char* cl_env = getenv("REALB_GEMM_CLUSTER");
  const bool pair = cl_env && cl_env[0] == '2';
  if (epilogue == REALB_EPI_STORE)
    return pair ? launch_grouped_bf16<256, 6, REALB_EPI_STORE, 2>(d_a, d_w, rows_cap, N, K, E,
                                                                   d_layout, prec, d_out, max_ctas, st)
                : launch_grouped_bf16<256, 4, REALB_EPI_STORE, 1>(d_a, d_w, rows_cap, N, K, E,
                                                                   d_layout, prec, d_out, max_ctas, st);
  if (epilogue == REALB_EPI_SWIGLU)
    return pair ? launch_grouped_bf16<256, 6, REALB_EPI_SWIGLU, 2>(d_a, d_w, rows_cap, N, K, E,
                                                                    d_layout, prec, d_out, max_ctas, st)
                : launch_grouped_bf16<256, 4, REALB_EPI_SWIGLU, 1>(d_a, d_w, rows_cap, N, K, E,
                                                                    d_layout, prec, d_out, max_ctas, st);
  set_error("realb_grouped_gemm_bf16: unknown epilogue %d", epilogue);
  return REALB_EINVAL;
}

extern "C" int realb_grouped_gemm_bf16_gather(const void* d_x, int64_t n_src, const int32_t* d_row_src,
                                              const void* d_w, int64_t rows_cap, int N, int K, int E,
                                              const int32_t* d_layout, int prec, int epilogue, void* d_out,
                                              int max_ctas, void* stream) {
  if (!d_x || !d_row_src || !d_w || !d_layout || !d_out || n_src <= 0 || n_src >= (1LL << 31) - 1 ||
      rows_cap <= 0 || E <= 0 || (prec != REALB_PREC_W16A16 && prec != REALB_PREC_W4A4)) {
    set_error("realb_grouped_gemm_bf16_gather: bad arguments");
    return REALB_EINVAL;
  }
  if (K % kBK || N % 256) {
    set_error("realb_grouped_gemm_bf16_gather: needs K %% 64 == 0 and N %% 256 == 0 (N=%d K=%d)", N, K);
    return REALB_EUNSUPPORTED;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (epilogue == REALB_EPI_STORE)
    return launch_grouped_bf16<256, 4, REALB_EPI_STORE, 1, true>(d_x, d_w, rows_cap, N, K, E, d_layout, prec,
                                                                 d_out, max_ctas, st, d_row_src);
  if (epilogue == REALB_EPI_SWIGLU)
    return launch_grouped_bf16<256, 4, REALB_EPI_SWIGLU, 1, true>(d_x, d_w, rows_cap, N, K, E, d_layout, prec,
                                                                  d_out, max_ctas, st, d_row_src);
  set_error("realb_grouped_gemm_bf16_gather: unknown epilogue %d", epilogue);
  return REALB_EINVAL;
}

extern "C" int realb_grouped_gemm_bf16_scatter(const void* d_a, const void* d_w, int64_t rows_cap, int N, int K,
                                               int E, const int32_t* d_layout, int prec, const int32_t* d_row_map,
                                               int n_dst, const uint64_t* h_dst_bases, int max_ctas,
                                               void* stream) {
  if (!d_a || !d_w || !d_layout || !d_row_map || !h_dst_bases || rows_cap <= 0 || E <= 0 || n_dst < 1 ||
      n_dst > kScatterPeers || (prec != REALB_PREC_W16A16 && prec != REALB_PREC_W4A4)) {
    set_error("realb_grouped_gemm_bf16_scatter: bad arguments");
    return REALB_EINVAL;
  }
  if (K % kBK || N % 256) {
    set_error("realb_grouped_gemm_bf16_scatter: needs K %% 64 == 0 and N %% 256 == 0 (N=%d K=%d)", N, K);
    return REALB_EUNSUPPORTED;
  }
  RowScatter sc{};
  for (int d = 0; d < n_dst; ++d) {
    if (h_dst_bases[d] & 15) {
      set_error("realb_grouped_gemm_bf16_scatter: destination %d not 16-B aligned", d);
      return REALB_EINVAL;
    }
    sc.base[d] = reinterpret_cast<uint8_t*>(h_dst_bases[d]);
  }
  sc.row_map = d_row_map;
  sc.ld = (int64_t)N * 2;
  return launch_grouped_bf16<256, 4, kEpiScatter, 1>(d_a, d_w, rows_cap, N, K, E, d_layout, prec, nullptr,
                                                     max_ctas, (cudaStream_t)stream, nullptr, &sc);
}

extern "C" int realb_grouped_gemm_bf16_copyin(const void* d_x, const int32_t* d_row_src, void* d_a, const void* d_w,
                                              int64_t rows_cap, int N, int K, int E, const int32_t* d_layout,
                                              int prec, int epilogue, void* d_out, int32_t* d_ready,
                                              int32_t* d_err, int max_ctas, void* stream) {
  if (!d_x || !d_row_src || !d_a || !d_w || !d_layout || !d_out || !d_ready || !d_err || rows_cap <= 0 ||
      E <= 0 || (prec != REALB_PREC_W16A16 && prec != REALB_PREC_W4A4)) {
    set_error("realb_grouped_gemm_bf16_copyin: bad arguments");
    return REALB_EINVAL;
  }
  if (K % kBK || N % 256) {
    set_error("realb_grouped_gemm_bf16_copyin: needs K %% 64 == 0 and N %% 256 == 0 (N=%d K=%d)", N, K);
    return REALB_EUNSUPPORTED;
  }
  CopyIn ci{reinterpret_cast<const __nv_bfloat16*>(d_x), d_row_src, reinterpret_cast<__nv_bfloat16*>(d_a), d_ready,
            d_err};
  cudaStream_t st = (cudaStream_t)stream;
  if (epilogue == REALB_EPI_STORE)
    return launch_grouped_bf16<256, 4, REALB_EPI_STORE, 1, false, true>(d_a, d_w, rows_cap, N, K, E, d_layout, prec,
                                                                        d_out, max_ctas, st, nullptr, nullptr, &ci);
  if (epilogue == REALB_EPI_SWIGLU)
    return launch_grouped_bf16<256, 4, REALB_EPI_SWIGLU, 1, false, true>(d_a, d_w, rows_cap, N, K, E, d_layout,
                                                                         prec, d_out, max_ctas, st, nullptr,
                                                                         nullptr, &ci);
  set_error("realb_grouped_gemm_bf16_copyin: unknown epilogue %d", epilogue);
  return REALB_EINVAL;
}
