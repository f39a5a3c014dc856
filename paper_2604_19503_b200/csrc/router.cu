// router.cu — K1 + K2: gating GEMM, top-k selection, routing weights and
// per-chunk (vision, text) pair statistics in ONE kernel.
//
// One CTA per 64-token chunk (REALB_CHUNK_TOKENS; 128 CTAs at T = 8192 — the
// kernel is HBM-bound and needs the SMs). logits[64, E] = X[64, H] . Wg[E, H]^T
// runs on tcgen05 (kind::f16, M=128 with the upper 64 smem rows unused,
// N=E padded to 16) with TMA-fed smem stages; the
// epilogue thread that owns token row r streams its E fp32 logits out of TMEM
// (tcgen05.ld 32x32b) and performs, in registers:
//   - write logits[r, :]                (the D1 contract selects on these)
//   - top-k on s = logit + bias, strict ">" insertion in expert order, i.e.
//     descending score with ties to the lowest expert id (the reference's only
//     top-k convention, balancers.py:161-165)
//   - routing weights per scoring family
//   - (vision, text) counts of its k pairs into a shared-memory histogram
// and the chunk histogram is written once, without global atomics, to
// chunk_counts[c][E][2] (deterministic; summed by realb_moe_align).
// Roofline: HBM-bound (2H bytes/token read, E <= 256 < ridge), DESIGN.md §K1.
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace realb {

constexpr int kRBK = 64;

constexpr int kKMax = 8;

// Operand stage: the chunk's 64 token rows (8 KB) then the router rows. The MMA is
// M = 128 and reads 128 A rows; rows 64..127 fall on the router-row tile that follows
// (their logits land in TMEM lanes 64..127, which nothing reads), so a stage holds
// only the bytes TMA loads and more stages fit (bytes in flight set this kernel's
// HBM rate: one CTA per 64-token chunk).
template <int EPAD, bool DEEP>
struct RouterSmem {
  static constexpr int A_LOAD = REALB_CHUNK_TOKENS * kRBK * 2;  // 8 KB
  static constexpr int B_BYTES = EPAD * kRBK * 2;
  static constexpr int STAGE = A_LOAD + B_BYTES < 128 * kRBK * 2 ? 128 * kRBK * 2 : A_LOAD + B_BYTES;
  static constexpr int STAGE_TX = A_LOAD + B_BYTES;
  // one CTA per SM when the grid fits the SMs (192 KB of stages), else two per SM
  static constexpr int BUDGET = DEEP ? 192 * 1024 : 96 * 1024;
  static constexpr int STAGES = BUDGET / STAGE < 16 ? BUDGET / STAGE : 16;
  static constexpr int LBOX = (EPAD + 31) / 32;
  static constexpr int LS = EPAD + 1;
  static constexpr int XS = kKMax + 2 + 2 * ((EPAD + 31) / 32);
  static constexpr int SCRATCH = LBOX * 8192 + REALB_CHUNK_TOKENS * (LS + XS) * 4;
  static constexpr int HIST_OFF = (STAGES * STAGE > SCRATCH ? STAGES * STAGE : SCRATCH + 1023) / 1024 * 1024;
  static constexpr int BIAS_OFF = HIST_OFF + 256 * 2 * 4;
  static constexpr int BAR_OFF = BIAS_OFF + 256 * 4;
  static constexpr int TOTAL = BAR_OFF + (2 * STAGES + 4) * 8 + 16 + 1024;
  static constexpr uint32_t TMEM_COLS = EPAD <= 32 ? 32 : EPAD <= 64 ? 64 : EPAD <= 128 ? 128 : 256;
  // epilogue scratch over the dead stages: logits tile for the TMA store
  // (SWIZZLE_128B boxes of 64 rows x 32 fp32), scores [64][EPAD+1], high-half exchange
  static constexpr int LOGIT_OFF = 0;
  static constexpr int SCORE_OFF = LBOX * 8192;
  static constexpr int XCH_OFF = SCORE_OFF + REALB_CHUNK_TOKENS * LS * 4;
  static_assert(XCH_OFF + REALB_CHUNK_TOKENS * XS * 4 <= HIST_OFF, "epilogue scratch must fit in the stages");
};

// byte offset of logit (r, c) in the swizzled logits tile (TMA SWIZZLE_128B image)
__device__ __forceinline__ uint32_t logit_off(int r, int c) {
  return (uint32_t)((c >> 5) * 8192 + r * 128 + ((((c & 31) >> 2) ^ (r & 7)) << 4) + (c & 3) * 4);
}

template <int EPAD, int KK, bool DEEP>
__global__ void __launch_bounds__(256, 1)
    router_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                  const __grid_constant__ CUtensorMap tmL, const float* __restrict__ bias,
                  const uint8_t* __restrict__ modality, int T, int H, int E, int scoring,
                  float routed_scaling, float norm_min, float* __restrict__ logits,
                  int32_t* __restrict__ topk_idx, float* __restrict__ topk_w,
                  int32_t* __restrict__ chunk_counts, uint32_t dbg, int nst) {
  using S = RouterSmem<EPAD, DEEP>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned, derived from the __shared__ array by pointer arithmetic so that
  // the compiler keeps shared-space (LDS/STS, not generic) accesses through it
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  int32_t* hist = reinterpret_cast<int32_t*>(smem + S::HIST_OFF);
  float* bsm = reinterpret_cast<float*>(smem + S::BIAS_OFF);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint64_t* empty = full + S::STAGES;
  uint64_t* done = empty + S::STAGES;
  uint64_t* bias_ready = done + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bias_ready + 1);

  const int warp = warp_id(), lane = lane_id();
  const int chunk = blockIdx.x;
  const int nkb = H / kRBK;
  const bool tma_logits = (E & 3) == 0;  // 16-B row pitch: the logits leave by TMA store

  for (int i = threadIdx.x; i < 2 * E; i += blockDim.x) hist[i] = 0;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmW);
    if (tma_logits) tma_prefetch_desc(&tmL);
    for (int s = 0; s < S::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    mbar_init(bias_ready, 32);
    fence_barrier_init();
  }
  // the producer fills the whole ring before the CTA-wide sync (its barriers are
  // initialised by its own lane above), overlapping the first loads' latency with the
  // TMEM allocation and the sync
  const int npre = nkb < nst ? nkb : nst;
  if (warp == 0) {
    if (lane == 0 && !(dbg & 4u)) {  // the lane that initialised the barriers
      for (int kb = 0; kb < npre; ++kb) {
        uint8_t* sa = smem + kb * S::STAGE;
        mbar_arrive_expect_tx(&full[kb], S::STAGE_TX);
        tma_load_2d(sa, &tmX, &full[kb], kb * kRBK, chunk * REALB_CHUNK_TOKENS);
        tma_load_2d(sa + S::A_LOAD, &tmW, &full[kb], kb * kRBK, 0);
      }
    }
    __syncwarp();
  }
  if (warp == 2) tmem_alloc<S::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  long long ts0 = clock64(), ts[6] = {0, 0, 0, 0, 0, 0};

  // Producer and MMA roles run warp-wide with one elected lane issuing (lane-0-only
  // code makes ptxas wrap each TMA / tcgen05 instruction in an ELECT/R2UR loop).
  if (warp == 0) {  // ---------------- TMA producer
    const bool leader = elect_one();
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      if (kb < npre && !(dbg & 4u)) {  // issued before the sync
        if (++stage == nst) { stage = 0; phase ^= 1; }
        continue;
      }
      mbar_wait(&empty[stage], phase ^ 1);
      if (leader) {
        uint8_t* sa = smem + stage * S::STAGE;
        if (dbg & 4u) {  // debug: no loads
          mbar_arrive(&full[stage]);
        } else {
          mbar_arrive_expect_tx(&full[stage], S::STAGE_TX);
          tma_load_2d(sa, &tmX, &full[stage], kb * kRBK, chunk * REALB_CHUNK_TOKENS);
          tma_load_2d(sa + S::A_LOAD, &tmW, &full[stage], kb * kRBK, 0);
        }
      }
      __syncwarp();
      if (++stage == nst) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 1) {  // ---------------- MMA issuer
    const bool leader = elect_one();
    constexpr uint32_t idesc = idesc_bf16(128, EPAD);
    const uint32_t s0 = smem_u32(smem);
    const uint64_t adesc0 = umma_desc_sw128(s0), bdesc0 = umma_desc_sw128(s0 + S::A_LOAD);
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      const uint64_t soff = (uint64_t)((uint32_t)(stage * S::STAGE) >> 4);
      if (leader) {
#pragma unroll
        for (int kk = 0; kk < kRBK / 16; ++kk)
          if (!(dbg & 8u) || kk == 0)  // debug bit 8: one MMA per stage (timing probe)
            umma_bf16(tbase, adesc0 + soff + (uint64_t)(kk * 2), bdesc0 + soff + (uint64_t)(kk * 2), idesc,
                      (kb | kk) != 0);
        tc_commit(&empty[stage]);
      }
      __syncwarp();
      if (++stage == nst) { stage = 0; phase ^= 1; }
    }
    if (leader) tc_commit(done);
    __syncwarp();
  } else if (warp == 6) {  // ---------------- bias -> shared memory, under the K loop
    for (int i = lane; i < EPAD; i += 32) bsm[i] = (bias && i < E) ? __ldg(bias + i) : 0.f;
    mbar_arrive(bias_ready);
  }
  // ---------------- epilogue: rows 0..63 = TMEM lane quadrants 0 and 1. Each row is
  // served by two threads: warp 4/5 ("primary": expert columns [0, HALF)) and warp 0/1
  // (the producer / MMA warps, free once the MMAs are done: [HALF, EPAD)).
  //   pass 1  each thread streams its columns out of TMEM: fp32 logits into the
  //           swizzled tile (one TMA store per 32 columns), scores s = logit + bias
  //           into shared memory, an online softmax, and the k largest scores kept as
  //           a sorted list by a min/max network (2k FMNMX per score, no data-dependent
  //           branches, so consecutive insertions pipeline).
  //   merge   the primary merges the other half's list -> threshold thr = k-th largest
  //           score, n_gt = how many of the k exceed it.
  //   pass 2  each thread marks its columns with s > thr and s == thr as bit masks.
  //   select  the primary takes every s > thr and the lowest-id ties (the reference's
  //           only tie rule, lowest expert id first, balancers.py:161-165), reads their
  //           scores back, orders them by (score desc, id asc) with a sorting network
  //           and writes ids, weights and the (v, t) histogram.
  if (warp == 0 || warp == 1 || warp == 4 || warp == 5) {
    const int q = warp & 3;
    const bool primary = warp >= 4;
    const int row = q * 32 + lane;
    const int t = chunk * REALB_CHUNK_TOKENS + row;
    const bool valid = t < T;
    mbar_wait(done, 0);
    tc_fence_after();
    ts[0] = clock64();
    const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16);
    if (dbg & 1u) {  // debug: no epilogue work
      named_bar_sync(1, 128);
      tc_fence_before();
      goto router_done;
    }
    mbar_wait(bias_ready, 0);

    constexpr int k = KK;
    constexpr int NG = EPAD / 16;        // 16-column TMEM groups
    constexpr int NG_LO = (NG + 1) / 2;  // groups of the primary (low) half
    constexpr int HALF = NG_LO * 16;     // first column of the high half
    constexpr int LS = S::LS;
    constexpr int XS = S::XS;
    const uint32_t ltile = smem_u32(smem + S::LOGIT_OFF);
    float* srow = reinterpret_cast<float*>(smem + S::SCORE_OFF) + row * LS;
    float* xrow = reinterpret_cast<float*>(smem + S::XCH_OFF) + row * XS;

    float top[KK];  // descending
#pragma unroll
    for (int j = 0; j < KK; ++j) top[j] = -INFINITY;
    float run_max = -INFINITY, run_sum = 0.f;  // online softmax over this half's logits
    const int g0 = primary ? 0 : NG_LO, g1 = primary ? NG_LO : NG;
#pragma unroll 1
    for (int g = g0; g < g1; ++g) {
      const int c0 = g * 16;
      uint32_t v[16];
      tmem_ld16(tb + c0, v);
      float bv[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) bv[i] = bsm[c0 + i];
      tmem_wait_ld();
      if (tma_logits) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          st_shared_v4(ltile + logit_off(row, c0 + 4 * i), v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      } else if (valid && !(dbg & 16u)) {  // debug bit 16: no logits stores
        float* lrow = logits + (int64_t)t * E;
#pragma unroll
        for (int i = 0; i < 16; ++i)  // unrolled with a guard: v must not be indexed dynamically
          if (c0 + i < E) lrow[c0 + i] = __uint_as_float(v[i]);
        // the select step reads logits back from the tile
#pragma unroll
        for (int i = 0; i < 4; ++i)
          st_shared_v4(ltile + logit_off(row, c0 + 4 * i), v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      }
      if (scoring != REALB_SCORE_SIGMOID_RENORM) {  // one rescale per 16 logits
        float m = run_max;
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (c0 + i < E) m = fmaxf(m, __uint_as_float(v[i]));
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (c0 + i < E) acc += __expf(__uint_as_float(v[i]) - m);
        run_sum = run_sum * __expf(run_max - m) + acc;
        run_max = m;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float sc = c0 + i < E ? __uint_as_float(v[i]) + bv[i] : -INFINITY;  // padding never wins
        srow[c0 + i] = sc;
        float x = sc;
#pragma unroll
        for (int j = 0; j < KK; ++j) {
          const float hi = fmaxf(top[j], x);
          x = fminf(top[j], x);
          top[j] = hi;
        }
      }
    }
    if (tma_logits) fence_proxy_async_smem();  // the tile's generic stores -> the TMA store
    if (!primary) {
#pragma unroll
      for (int j = 0; j < KK; ++j) xrow[j] = top[j];
      xrow[KK] = run_max;
      xrow[KK + 1] = run_sum;
    }
    named_bar_sync(1, 128);
    ts[1] = clock64();
    if (tma_logits && warp == 4 && lane == 0 && !(dbg & 16u)) {  // the chunk's logits: one store per 32 columns
#pragma unroll 1
      for (int b = 0; b < S::LBOX; ++b)
        tma_store_2d(&tmL, smem + S::LOGIT_OFF + b * 8192, 32 * b, chunk * REALB_CHUNK_TOKENS);
      bulk_commit_group();
    }
    if (primary) {  // merge the high half's list and softmax state -> threshold
#pragma unroll
      for (int j2 = 0; j2 < KK; ++j2) {
        float x = xrow[j2];
#pragma unroll
        for (int j = 0; j < KK; ++j) {
          const float hi = fmaxf(top[j], x);
          x = fminf(top[j], x);
          top[j] = hi;
        }
      }
      if (scoring != REALB_SCORE_SIGMOID_RENORM) {
        const float m2 = xrow[KK], s2 = xrow[KK + 1];
        const float m = fmaxf(run_max, m2);
        run_sum = (run_sum > 0.f ? run_sum * __expf(run_max - m) : 0.f) +
                  (s2 > 0.f ? s2 * __expf(m2 - m) : 0.f);
        run_max = m;
      }
      xrow[0] = top[KK - 1];  // the threshold, for the high half's pass 2
    }
    named_bar_sync(1, 128);
    ts[2] = clock64();
    const float thr = primary ? top[KK - 1] : xrow[0];
    // pass 2: column c <-> bit c % 32 of word c / 32 (each thread sets its own columns)
    constexpr int NWT = (EPAD + 31) / 32;
    uint32_t gt[NWT], eq[NWT];
#pragma unroll
    for (int w = 0; w < NWT; ++w) { gt[w] = 0; eq[w] = 0; }
    auto mark = [&](auto cb, auto ce) {  // compile-time column range: static word indices
#pragma unroll
      for (int c = decltype(cb)::value; c < decltype(ce)::value; ++c) {
        const float sc = srow[c];
        gt[c / 32] |= (sc > thr ? 1u : 0u) << (c % 32);
        eq[c / 32] |= (sc == thr ? 1u : 0u) << (c % 32);
      }
    };
    if (primary) mark(std::integral_constant<int, 0>{}, std::integral_constant<int, HALF>{});
    else mark(std::integral_constant<int, HALF>{}, std::integral_constant<int, EPAD>{});
    if (!primary) {
#pragma unroll
      for (int w = 0; w < NWT; ++w) {
        xrow[KK + 2 + w] = __uint_as_float(gt[w]);
        xrow[KK + 2 + NWT + w] = __uint_as_float(eq[w]);
      }
    }
    named_bar_sync(1, 128);
    ts[3] = clock64();
    if (primary) {
      // all selected columns: every s > thr (n_gt of the k list entries exceed thr),
      // then the lowest-id ties until k are taken
      int n_gt = 0;
#pragma unroll
      for (int j = 0; j < KK; ++j) n_gt += top[j] > thr ? 1 : 0;
      const int need = k - n_gt;
      uint32_t sel[NWT], tie[NWT];
      int n_tie = 0;
#pragma unroll
      for (int w = 0; w < NWT; ++w) {
        sel[w] = gt[w] | __float_as_uint(xrow[KK + 2 + w]);
        tie[w] = eq[w] | __float_as_uint(xrow[KK + 2 + NWT + w]);
        n_tie += __popc(tie[w]);
      }
      if (n_tie <= need) {  // the usual case: the threshold value occurs once
#pragma unroll
        for (int w = 0; w < NWT; ++w) sel[w] |= tie[w];
      } else {
        int left = need;
#pragma unroll
        for (int w = 0; w < NWT; ++w) {
          uint32_t e = tie[w];
          while (e && left > 0) {
            const uint32_t b = e & (0u - e);
            sel[w] |= b;
            e ^= b;
            --left;
          }
        }
      }
      // the k selected ids in ascending order: k fixed steps, each takes the lowest set bit
      float ss[KK], ls[KK];
      int sid[KK];
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        int e = -1;
#pragma unroll
        for (int w = 0; w < NWT; ++w) {
          if (e < 0 && sel[w]) {
            e = 32 * w + __ffs(sel[w]) - 1;
            sel[w] &= sel[w] - 1;
          }
        }
        sid[j] = e < 0 ? 0 : e;
        ss[j] = e < 0 ? -INFINITY : srow[sid[j]];
        ls[j] = e < 0 ? 0.f : __uint_as_float(ld_shared_u32(ltile + logit_off(row, sid[j])));
      }
      // output slot of each selected id (they arrive in ascending id order): the order
      // is (score desc, id asc), so slot = #(selected scores above it) + #(lower ids
      // with an equal score); top[] is exactly the multiset of the selected scores
      int slot[KK];
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        int r = 0;
#pragma unroll
        for (int m = 0; m < KK; ++m) r += top[m] > ss[j] ? 1 : 0;
#pragma unroll
        for (int i = 0; i < j; ++i) r += ss[i] == ss[j] ? 1 : 0;
        slot[j] = r;
      }
      // routing weights from the selected logits
      float w[KK];
      float wsum = 0.f;
      const float inv_sum = __fdividef(1.0f, run_sum);  // MUFU.RCP (the IEEE __frcp_rn is a long sequence)
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        float p;
        if (scoring == REALB_SCORE_SIGMOID_RENORM)
          p = __fdividef(1.0f, 1.0f + __expf(-ls[j]));
        else
          p = __expf(ls[j] - run_max) * inv_sum;  // softmax probability
        w[j] = p;
        wsum += p;
      }
      float scale;
      if (scoring == REALB_SCORE_SOFTMAX_RENORM) scale = __fdividef(1.0f, wsum);
      else if (scoring == REALB_SCORE_SIGMOID_RENORM) scale = __fdividef(routed_scaling, wsum);
      else scale = __fdividef(1.0f, fmaxf(wsum, norm_min));
      ts[4] = clock64();
      if (valid) {
        const int vis = modality[t] ? 0 : 1;  // hist[e][0] vision, [e][1] text
#pragma unroll
        for (int j = 0; j < KK; ++j) {
          topk_idx[(int64_t)t * k + slot[j]] = sid[j];
          topk_w[(int64_t)t * k + slot[j]] = w[j] * scale;
          atomicAdd(&hist[2 * sid[j] + vis], 1);
        }
      }
    }
    tc_fence_before();
    named_bar_sync(1, 128);
    ts[5] = clock64();
    if ((dbg & 32u) && primary && row == 0 && valid) {  // debug: phase cycles into topk_w of the chunk's first token
      int32_t* dst = reinterpret_cast<int32_t*>(topk_w + (int64_t)t * k);
      const long long d[6] = {ts[0] - ts0, ts[1] - ts[0], ts[2] - ts[1], ts[3] - ts[2], ts[4] - ts[3], ts[5] - ts[4]};
#pragma unroll
      for (int j = 0; j < KK && j < 6; ++j) dst[j] = (int)d[j];
    }
    if (primary) {
      int32_t* out = chunk_counts + (int64_t)chunk * E * 2;
      for (int i = row; i < 2 * E; i += REALB_CHUNK_TOKENS) out[i] = hist[i];
    }
    if (tma_logits && warp == 4 && lane == 0) bulk_wait_group_read<0>();  // tile read out before exit
  }
router_done:
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<S::TMEM_COLS>(tmem_base);
}

template <int EPAD, int KK>
static int launch_router(const void* x, const void* wg, const float* bias, const uint8_t* mod,
                         int T, int H, int E, int k, int scoring, float rs, float nm, float* logits,
                         int32_t* idx, float* w, int32_t* cc, cudaStream_t st) {
  CUtensorMap tx, tw, tl;
  int rc = make_tmap_2d(&tx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, x, H, T, (uint64_t)H * 2, kRBK,
                        REALB_CHUNK_TOKENS, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  rc = make_tmap_2d(&tw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, wg, H, E, (uint64_t)H * 2, kRBK, EPAD,
                    CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  if ((E & 3) == 0) {  // logits [T, E] fp32, stored by 64-row x 32-column boxes
    rc = make_tmap_2d(&tl, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, logits, E, T, (uint64_t)E * 4, 32,
                      REALB_CHUNK_TOKENS, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  } else {
    tl = tx;  // unused: rows of E % 4 != 0 logits are not 16-B aligned, stored directly
  }
  const int grid = (T + REALB_CHUNK_TOKENS - 1) / REALB_CHUNK_TOKENS;
  const char* dbg_env = getenv("REALB_DBG_ROUTER");
  const uint32_t dbg = dbg_env ? (uint32_t)strtoul(dbg_env, nullptr, 0) : 0u;
  const bool deep = grid <= num_sms();
  const char* st_env = getenv("REALB_ROUTER_STAGES");  // A/B: cap the ring depth
  const int nst_cap = st_env ? atoi(st_env) : 0;
  auto launch = [&](auto kern, int smem, int stages) {
    int r = set_smem_once(reinterpret_cast<const void*>(kern), smem, "router smem attribute");
    if (r) return r;
    const int nst = nst_cap > 0 && nst_cap < stages ? nst_cap : stages;
    kern<<<grid, 256, smem, st>>>(tx, tw, tl, bias, mod, T, H, E, scoring, rs, nm, logits, idx, w, cc, dbg, nst);
    return check_launch("realb_router_topk_stats");
  };
  return deep ? launch(router_kernel<EPAD, KK, true>, RouterSmem<EPAD, true>::TOTAL, RouterSmem<EPAD, true>::STAGES)
              : launch(router_kernel<EPAD, KK, false>, RouterSmem<EPAD, false>::TOTAL,
                       RouterSmem<EPAD, false>::STAGES);
}

}  // namespace realb

using namespace realb;

extern "C" int realb_router_topk_stats(const void* d_x, const void* d_wg, const float* d_bias,
                                       const uint8_t* d_modality, int T, int H, int E, int k,
                                       int scoring, float routed_scaling, float norm_min,
                                       float* d_logits, int32_t* d_topk_idx, float* d_topk_w,
                                       int32_t* d_chunk_counts, void* stream) {
  if (T == 0 && E >= 1 && E <= 256 && k >= 1 && k <= kKMax && k <= E && H > 0) return REALB_OK;
  if (!d_x || !d_wg || !d_modality || !d_logits || !d_topk_idx || !d_topk_w || !d_chunk_counts ||
      T < 0 || E < 1 || E > 256 || k < 1 || k > kKMax || k > E || H <= 0 || scoring < 0 ||
      scoring > 2) {
    set_error("realb_router_topk_stats: bad arguments (T=%d H=%d E=%d k=%d scoring=%d)", T, H, E,
              k, scoring);
    return REALB_EINVAL;
  }
  if (H % kRBK) {
    set_error("realb_router_topk_stats: H must be a multiple of 64 (H=%d)", H);
    return REALB_EUNSUPPORTED;
  }
  if (T == 0) return REALB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int epad = (E + 15) / 16 * 16;
  if (k != 1 && k != 2 && k != 4 && k != 6 && k != 8) {
    set_error("realb_router_topk_stats: top-k must be one of 1,2,4,6,8 (k=%d)", k);
    return REALB_EUNSUPPORTED;
  }
#define REALB_ROUTER_K(P, KK)                                                                      \
  if (k == KK)                                                                                     \
    return launch_router<P, KK>(d_x, d_wg, d_bias, d_modality, T, H, E, k, scoring, routed_scaling, \
                                norm_min, d_logits, d_topk_idx, d_topk_w, d_chunk_counts, st);
#define REALB_ROUTER_CASE(P) \
  if (epad <= P) {           \
    REALB_ROUTER_K(P, 1)     \
    REALB_ROUTER_K(P, 2)     \
    REALB_ROUTER_K(P, 4)     \
    REALB_ROUTER_K(P, 6)     \
    REALB_ROUTER_K(P, 8)     \
  }
  REALB_ROUTER_CASE(16)
  REALB_ROUTER_CASE(64)
  REALB_ROUTER_CASE(128)
  REALB_ROUTER_CASE(256)
#undef REALB_ROUTER_CASE
#undef REALB_ROUTER_K
  return REALB_EUNSUPPORTED;
}
