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

#include "common.cuh"

namespace realb {

constexpr int kRBK = 64;

constexpr int kKMax = 8;

template <int EPAD, int NSTAGE>
struct RouterSmem {
  static constexpr int A_BYTES = 128 * kRBK * 2;          // MMA reads 128 rows
  static constexpr int A_LOAD = REALB_CHUNK_TOKENS * kRBK * 2;  // TMA fills 64
  static constexpr int B_BYTES = EPAD * kRBK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGE_TX = A_LOAD + B_BYTES;
  // the router is latency-bound per SM (one CTA per 64 tokens), so bytes in flight
  // set its HBM throughput: 8 stages when the grid fits one CTA per SM, 4 (two
  // CTAs per SM) for larger grids
  static constexpr int STAGES = NSTAGE * STAGE <= 200 * 1024 ? NSTAGE : (200 * 1024) / STAGE;
  static constexpr int HIST_OFF = STAGES * STAGE;
  static constexpr int BAR_OFF = HIST_OFF + 256 * 2 * 4;
  static constexpr int TOTAL = BAR_OFF + 128 + 1024;
  static constexpr uint32_t TMEM_COLS = EPAD <= 32 ? 32 : EPAD <= 64 ? 64 : EPAD <= 128 ? 128 : 256;
};

template <int EPAD, int KK, int NSTAGE>
__global__ void __launch_bounds__(256, 1)
    router_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                  const float* __restrict__ bias, const uint8_t* __restrict__ modality, int T,
                  int H, int E, int scoring, float routed_scaling, float norm_min,
                  float* __restrict__ logits, int32_t* __restrict__ topk_idx,
                  float* __restrict__ topk_w, int32_t* __restrict__ chunk_counts, uint32_t dbg) {
  using S = RouterSmem<EPAD, NSTAGE>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  int32_t* hist = reinterpret_cast<int32_t*>(smem + S::HIST_OFF);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint64_t* empty = full + S::STAGES;
  uint64_t* done = empty + S::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = warp_id(), lane = lane_id();
  const int chunk = blockIdx.x;
  const int nkb = H / kRBK;

  for (int i = threadIdx.x; i < 2 * E; i += blockDim.x) hist[i] = 0;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmW);
    for (int s = 0; s < S::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<S::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {  // ---------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sa = smem + stage * S::STAGE;
        if (dbg & 4u) {  // debug: no loads
          mbar_arrive(&full[stage]);
        } else {
          mbar_arrive_expect_tx(&full[stage], S::STAGE_TX);
          tma_load_2d(sa, &tmX, &full[stage], kb * kRBK, chunk * REALB_CHUNK_TOKENS);
          tma_load_2d(sa + S::A_BYTES, &tmW, &full[stage], kb * kRBK, 0);
        }
        if (++stage == S::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(128, EPAD);
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + stage * S::STAGE);
        const uint64_t adesc = umma_desc_sw128(sa), bdesc = umma_desc_sw128(sa + S::A_BYTES);
#pragma unroll
        for (int kk = 0; kk < kRBK / 16; ++kk)
          if (!(dbg & 8u) || kk == 0)  // debug bit 8: one MMA per stage (timing probe)
            umma_bf16(tmem_base, adesc + (uint64_t)(kk * 2), bdesc + (uint64_t)(kk * 2), idesc,
                      (kb | kk) != 0);
        tc_commit(&empty[stage]);
        if (++stage == S::STAGES) { stage = 0; phase ^= 1; }
      }
      tc_commit(done);
    }
  }
  // ---------------- epilogue: rows 0..63 = TMEM lane quadrants 0 and 1. Each row is
  // served by two warps of its quadrant — warp 4/5 ("primary", the low expert-column
  // half) and warp 0/1 (the producer / MMA warps, free once the MMAs are done: the
  // high half) — so a row's E logits are scanned by two threads in parallel (the scan
  // is a dependent compare/insert chain; one thread per row left it latency-bound).
  // The high half's partial top-k and softmax state goes through shared memory (the
  // operand stages are dead by then) and the primary thread merges it.
  if (warp == 0 || warp == 1 || warp == 4 || warp == 5) {
    const int q = warp & 3;
    const bool primary = warp >= 4;
    const int row = q * 32 + lane;
    const int t = chunk * REALB_CHUNK_TOKENS + row;
    const bool valid = t < T;
    mbar_wait(done, 0);
    tc_fence_after();
    const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16);
    if (dbg & 1u) {  // debug: no epilogue work
      named_bar_sync(1, 128);
      tc_fence_before();
      goto router_done;
    }

    constexpr int k = KK;
    constexpr int NG = EPAD / 16;           // 16-column TMEM groups
    constexpr int NG_LO = (NG + 1) / 2;     // groups of the primary (low) half
    float sval[KK], lsel[KK];
    int sid[KK];
#pragma unroll
    for (int j = 0; j < KK; ++j) { sval[j] = -INFINITY; lsel[j] = 0.f; sid[j] = 0; }
    float run_max = -INFINITY, run_sum = 0.f;  // online softmax over this half's logits
    float* lrow = logits + (int64_t)t * E;
    auto insert = [&](float s, float l, int e) {
      if (s > sval[k - 1]) {  // strict: an equal score keeps the lower expert id
        bool placed = false;
#pragma unroll
        for (int j = KK - 1; j >= 0; --j) {
          if (placed) continue;
          if (j > 0 && sval[j - 1] < s) {
            sval[j] = sval[j - 1]; lsel[j] = lsel[j - 1]; sid[j] = sid[j - 1];
          } else {
            sval[j] = s; lsel[j] = l; sid[j] = e; placed = true;
          }
        }
      }
    };
    const int g0 = primary ? 0 : NG_LO, g1 = primary ? NG_LO : NG;
#pragma unroll 1
    for (int g = g0; g < g1; ++g) {
      const int c0 = g * 16;
      uint32_t v[16];
      tmem_ld16(tb + c0, v);
      tmem_wait_ld();
      if (valid) {
        if (c0 + 16 <= E && (E & 3) == 0) {
          float4* l4 = reinterpret_cast<float4*>(lrow + c0);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            l4[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i)  // unrolled with a guard: v must not be indexed dynamically
            if (c0 + i < E) lrow[c0 + i] = __uint_as_float(v[i]);
        }
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
      // fully unrolled (no early exit): v stays in registers; the 16 bias values are
      // loaded up front rather than inside the dependent insertion chain
      float bv[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) bv[i] = (bias && c0 + i < E) ? __ldg(bias + c0 + i) : 0.f;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int e = c0 + i;
        if (e < E) {
          const float l = __uint_as_float(v[i]);
          insert(l + bv[i], l, e);
        }
      }
    }
    // hand the high half's state to the primary thread of the same row
    float* xs = reinterpret_cast<float*>(smem);  // operand stages are free after `done`
    constexpr int XS = 3 * KK + 2;
    if (!primary) {
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        xs[row * XS + j] = sval[j];
        xs[row * XS + KK + j] = lsel[j];
        xs[row * XS + 2 * KK + j] = __int_as_float(sid[j]);
      }
      xs[row * XS + 3 * KK] = run_max;
      xs[row * XS + 3 * KK + 1] = run_sum;
    }
    named_bar_sync(1, 128);
    if (primary) {
#pragma unroll
      for (int j = 0; j < KK; ++j)  // high-half candidates: descending, higher ids than ours
        insert(xs[row * XS + j], xs[row * XS + KK + j], __float_as_int(xs[row * XS + 2 * KK + j]));
      if (scoring != REALB_SCORE_SIGMOID_RENORM) {
        const float m2 = xs[row * XS + 3 * KK], s2 = xs[row * XS + 3 * KK + 1];
        const float m = fmaxf(run_max, m2);
        run_sum = (run_sum > 0.f ? run_sum * __expf(run_max - m) : 0.f) +
                  (s2 > 0.f ? s2 * __expf(m2 - m) : 0.f);
        run_max = m;
      }
      // routing weights from the selected logits
      float w[KK];
      float wsum = 0.f;
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        float p;
        if (scoring == REALB_SCORE_SIGMOID_RENORM)
          p = 1.0f / (1.0f + __expf(-lsel[j]));
        else
          p = __expf(lsel[j] - run_max) / run_sum;  // softmax probability
        w[j] = p;
        wsum += p;
      }
      float scale;
      if (scoring == REALB_SCORE_SOFTMAX_RENORM) scale = 1.0f / wsum;
      else if (scoring == REALB_SCORE_SIGMOID_RENORM) scale = routed_scaling / wsum;
      else scale = 1.0f / fmaxf(wsum, norm_min);
      if (valid) {
        const int vis = modality[t] ? 0 : 1;  // hist[e][0] vision, [e][1] text
#pragma unroll
        for (int j = 0; j < KK; ++j) {
          topk_idx[(int64_t)t * k + j] = sid[j];
          topk_w[(int64_t)t * k + j] = w[j] * scale;
          atomicAdd(&hist[2 * sid[j] + vis], 1);
        }
      }
    }
    tc_fence_before();
    named_bar_sync(1, 128);
    if (primary) {
      int32_t* out = chunk_counts + (int64_t)chunk * E * 2;
      for (int i = row; i < 2 * E; i += REALB_CHUNK_TOKENS) out[i] = hist[i];
    }
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
  CUtensorMap tx, tw;
  int rc = make_tmap_2d(&tx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, x, H, T, (uint64_t)H * 2, kRBK,
                        REALB_CHUNK_TOKENS, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  rc = make_tmap_2d(&tw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, wg, H, E, (uint64_t)H * 2, kRBK, EPAD,
                    CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  const int grid = (T + REALB_CHUNK_TOKENS - 1) / REALB_CHUNK_TOKENS;
  const char* dbg_env = getenv("REALB_DBG_ROUTER");
  const uint32_t dbg = dbg_env ? (uint32_t)strtoul(dbg_env, nullptr, 0) : 0u;
  const char* st_env = getenv("REALB_ROUTER_STAGES");
  const bool deep = st_env ? atoi(st_env) >= 8 : grid <= num_sms();
  auto launch = [&](auto kern, int smem) {
    int r = set_smem_once(reinterpret_cast<const void*>(kern), smem, "router smem attribute");
    if (r) return r;
    kern<<<grid, 256, smem, st>>>(tx, tw, bias, mod, T, H, E, scoring, rs, nm, logits, idx, w, cc, dbg);
    return check_launch("realb_router_topk_stats");
  };
  return deep ? launch(router_kernel<EPAD, KK, 8>, RouterSmem<EPAD, 8>::TOTAL)
              : launch(router_kernel<EPAD, KK, 4>, RouterSmem<EPAD, 4>::TOTAL);
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
