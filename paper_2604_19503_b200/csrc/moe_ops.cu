// moe_ops.cu — the data-movement kernels around the expert GEMMs:
//   realb_moe_align        per-chunk counts -> expert totals (K2 reduction,
//                          the device form of aggregate_rank_loads' inputs,
//                          core.py:106-130), 128-row padded grouped row space,
//                          per-precision group lists and m-tile prefixes
//   realb_dispatch_permute tokens -> grouped rows (stable: by expert, then
//                          token, then slot), bf16 copy or on-the-fly NVFP4
//                          quantisation (K4, reference block rule) per expert
//   realb_combine          y[t] = sum_j w[t,j] * rows[pos[t,j]]  (C3, local)
// All three are HBM/latency-bound; none uses atomics on global memory, so the
// grouped layout and pair positions are deterministic.
#include "common.cuh"
#include "fp4_rule.cuh"

namespace realb {

// ----------------------------------------------------------------- align (+ P1 on device)
struct PlanParams {
  int enabled;       // 0: use the caller's d_prec; 1: evaluate the strategy below
  int strategy;      // 0 baseline, 1 fp4all, 2 realb (plan_for, balancers.py:202-219)
  int R;             // EP ranks of the contiguous placement (place_experts_static)
  int isolated;      // ClusterConfig.modality_isolated
  double C, Md;      // RealbParams.capacity_factor / modality_threshold
  long long thr;     // RealbParams.global_batch_threshold
};

// plan_realb (balancers.py:89-122) on the device: one thread, the reference's
// fp64 operation order (identical to realb_plan in runtime.cu).
__device__ void plan_on_device(const int32_t* ev, int E, const PlanParams& pp, uint8_t* prec,
                               int32_t* plan_out) {  // ev, prec: shared memory
  const int R = pp.R, epr = E / R;
  long long total = 0;  // integer sums: exact in any order
  for (int e = 0; e < E; ++e) total += (long long)ev[2 * e] + ev[2 * e + 1];
  int active = 0, nacc = 0;
  for (int r = 0; r < R; ++r) {  // per-rank (v, v + t), recomputed: no per-rank arrays on the stack
    long long v = 0, tt = 0;
    for (int e = r * epr; e < (r + 1) * epr; ++e) { v += ev[2 * e]; tt += ev[2 * e + 1]; }
    const long long rv_r = v, rt_r = v + tt;
    uint32_t flags = 0;
    if (pp.strategy == 1) {
      flags = 7u;
    } else if (pp.strategy == 2 && !(total < pp.thr || total == 0)) {
      const double ideal = (double)total / (double)R;
      const bool hot = (double)rt_r / ideal > pp.C;
      const bool vis = pp.isolated ? rt_r > 0 : (rt_r > 0 && (double)rv_r / (double)rt_r > pp.Md);
      flags = (hot ? 1u : 0u) | (vis ? 2u : 0u) | ((hot && vis) ? 4u : 0u);
    }
    if (flags & 4u) ++nacc;
    if (plan_out) plan_out[3 + r] = (int32_t)flags;
    for (int e = r * epr; e < (r + 1) * epr; ++e) prec[e] = (flags & 4u) ? REALB_PREC_W4A4 : REALB_PREC_W16A16;
  }
  if (pp.strategy == 1) active = 1;
  else if (pp.strategy == 2) active = !(total < pp.thr || total == 0);
  if (plan_out) { plan_out[0] = active; plan_out[1] = nacc; plan_out[2] = R; }
}

// 256 threads (whole warps, >= E): E experts x G chunk groups (G = 256 / E) read the
// chunk counts (16 loads in flight per thread) and write the per-chunk offsets; the
// scans over the E <= 256 experts run on all 256 threads (warp shuffles); the plan
// on one thread. (1024 threads measured slower: the kernel is instruction-bound on
// its single SM, and a thread count that is not a multiple of 32 would leave a
// partial warp in the shuffle scans.)
constexpr int kAlignThreads = 256;
__global__ void __launch_bounds__(kAlignThreads) align_kernel(const int32_t* __restrict__ cc, int nchunks,
                                                     int E, uint8_t* __restrict__ prec,
                                                     int32_t* __restrict__ layout,
                                                     int32_t* __restrict__ expert_vt,
                                                     PlanParams pp, int32_t* plan_out, int ra) {
  __shared__ int32_t s_v[1024], s_t[1024], s_scan[7 * 256];
  __shared__ int32_t s_cnt[256], s_start[256], s_vt[512];
  __shared__ uint8_t s_prec[256];
  const int G = blockDim.x / E;  // chunk groups per expert
  const int e = threadIdx.x % E, g = threadIdx.x / E;
  const bool act = g < G;
  // chunk range of group g (contiguous, for the offset scan)
  const int per = (nchunks + G - 1) / G;
  const int c0 = act ? min(nchunks, g * per) : 0, c1 = act ? min(nchunks, c0 + per) : 0;
  // chunk counts in blocks of 8 (all loads of a block in flight; one 8-B load per
  // (chunk, expert) pair of counts)
  constexpr int kAB = 16;
  const int2* cc2 = reinterpret_cast<const int2*>(cc);
  int v = 0, t = 0;
  for (int cb = c0; cb < c1; cb += kAB) {
    int2 q[kAB];
#pragma unroll
    for (int i = 0; i < kAB; ++i) q[i] = cb + i < c1 ? __ldg(cc2 + (int64_t)(cb + i) * E + e) : make_int2(0, 0);
#pragma unroll
    for (int i = 0; i < kAB; ++i) { v += q[i].x; t += q[i].y; }
  }
  s_v[threadIdx.x] = v;
  s_t[threadIdx.x] = t;
  __syncthreads();
  if (threadIdx.x < E) {
    int tv = 0, tt = 0;
    for (int j = 0; j < G; ++j) { tv += s_v[j * E + threadIdx.x]; tt += s_t[j * E + threadIdx.x]; }
    expert_vt[2 * threadIdx.x] = tv;
    expert_vt[2 * threadIdx.x + 1] = tt;
    s_vt[2 * threadIdx.x] = tv;
    s_vt[2 * threadIdx.x + 1] = tt;
    s_cnt[threadIdx.x] = tv + tt;
    s_prec[threadIdx.x] = prec[threadIdx.x];
  }
  __syncthreads();
  if (pp.enabled) {
    if (threadIdx.x == 0) plan_on_device(s_vt, E, pp, s_prec, plan_out);
    __syncthreads();
  }
  // Parallel scans over the E <= 256 experts (threads 0..255): padded row starts
  // and, per precision class, the compacted group list with m-tile and m-tile-pair
  // prefixes. Hillis-Steele in shared memory; one value set per precision.
  {
    const int e = threadIdx.x;
    const bool in = e < E;
    const int cnt = in ? s_cnt[e] : 0;
    const int padded = in ? (cnt + ra - 1) / ra * ra : 0;
    const int m = in ? (cnt + 127) / 128 : 0;
    const int pe = in ? (int)s_prec[e] : -1;
    // 4 scanned quantities: padded rows, and for p in {0,1}: (flag, m-tiles, pairs)
    int v[7] = {padded, pe == 0, pe == 0 ? m : 0, pe == 0 ? (m + 1) / 2 : 0,
                pe == 1, pe == 1 ? m : 0, pe == 1 ? (m + 1) / 2 : 0};
    // inclusive scans: within each warp by shuffles, then the warps' totals
    int incl[7];
    const int ln = e & 31, wp = e >> 5;
#pragma unroll
    for (int j = 0; j < 7; ++j) {
      int x = v[j];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, off);
        if (ln >= off) x += y;
      }
      incl[j] = x;
      if (e < 256 && ln == 31) s_scan[j * 8 + wp] = x;  // warp totals
    }
    __syncthreads();
    if (e < 256) {
#pragma unroll
      for (int j = 0; j < 7; ++j)
        for (int w = 0; w < wp; ++w) incl[j] += s_scan[j * 8 + w];
    }
    if (in) {
      s_start[e] = incl[0] - v[0];
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        if (pe != p) continue;
        const int g = incl[1 + 3 * p] - 1;  // exclusive rank among experts of class p
        layout[LayoutView::off_glist(E, p) + g] = e;
        layout[LayoutView::off_prefix(E, p) + g] = incl[2 + 3 * p] - v[2 + 3 * p];
        layout[LayoutView::off_pprefix(E, p) + g] = incl[3 + 3 * p] - v[3 + 3 * p];
      }
    }
    if (e == E - 1) {
      layout[0] = incl[0];
      for (int w = 3; w < 8; ++w) layout[w] = 0;  // GEMM tile counters (grouped.cuh)
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int G = incl[1 + 3 * p];
        layout[1 + p] = G;
        layout[LayoutView::off_prefix(E, p) + G] = incl[2 + 3 * p];
        layout[LayoutView::off_pprefix(E, p) + G] = incl[3 + 3 * p];
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < E) {
    layout[LayoutView::off_row_start(E) + threadIdx.x] = s_start[threadIdx.x];
    layout[LayoutView::off_row_count(E) + threadIdx.x] = s_cnt[threadIdx.x];
    if (pp.enabled) prec[threadIdx.x] = s_prec[threadIdx.x];
  }
  if (act) {
    // exclusive offset of my chunk range within expert e, then per chunk
    int run = s_start[e];
    for (int j = 0; j < g; ++j) run += s_v[j * E + e] + s_t[j * E + e];
    int32_t* co = layout + LayoutView::off_chunk(E);
    for (int cb = c0; cb < c1; cb += kAB) {  // loads of a block first, then its offsets
      int2 q[kAB];
#pragma unroll
      for (int i = 0; i < kAB; ++i) q[i] = cb + i < c1 ? __ldg(cc2 + (int64_t)(cb + i) * E + e) : make_int2(0, 0);
#pragma unroll
      for (int i = 0; i < kAB; ++i)
        if (cb + i < c1) {
          co[(int64_t)(cb + i) * E + e] = run;
          run += q[i].x + q[i].y;
        }
    }
  }
}

// ----------------------------------------------------------------- dispatch
// One CTA per 64-token chunk (REALB_CHUNK_TOKENS, the router's chunking). Pair ranks inside the
// chunk are computed per warp with __match_any_sync, then offset by a per-warp
// exclusive prefix: pairs of one expert keep (token, slot) order.
constexpr int kPermWarps = 8;

__global__ void __launch_bounds__(256) permute_kernel(
    const int32_t* __restrict__ topk_idx, int T, int E, int k,
    const int32_t* __restrict__ layout, int32_t* __restrict__ pair_pos,
    int32_t* __restrict__ row_src = nullptr) {
  extern __shared__ int32_t sm[];
  int32_t* s_base = sm;                       // [E]
  int32_t* s_cnt = s_base + E;                // [kPermWarps][E]
  int32_t* s_pos = s_cnt + kPermWarps * E;    // [REALB_CHUNK_TOKENS * k]
  int32_t* s_eid = s_pos + REALB_CHUNK_TOKENS * k;  // [REALB_CHUNK_TOKENS * k] expert ids (read once)
  const int chunk = blockIdx.x;
  const int t0 = chunk * REALB_CHUNK_TOKENS;
  const int ntok = min(REALB_CHUNK_TOKENS, T - t0);
  const int P = ntok * k;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t* co = layout + LayoutView::off_chunk(E) + (int64_t)chunk * E;
  for (int i = threadIdx.x; i < E; i += blockDim.x) s_base[i] = co[i];
  for (int i = threadIdx.x; i < kPermWarps * E; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();

  // phase 1: warp-local stable ranks
  const int seg = (P + kPermWarps - 1) / kPermWarps;
  const int p_lo = warp * seg, p_hi = min(P, p_lo + seg);
  for (int p0 = p_lo; p0 < p_hi; p0 += 32) {
    const int p = p0 + lane;
    const bool act = p < p_hi;
    const unsigned am = __ballot_sync(0xffffffffu, act);
    if (!act) continue;
    const int e = topk_idx[(int64_t)t0 * k + p];
    s_eid[p] = e;
    const unsigned grp = __match_any_sync(am, e);
    const int before = __popc(grp & ((1u << lane) - 1u));
    const int base = s_cnt[warp * E + e];
    s_pos[p] = base + before;  // rank within this warp's segment
    __syncwarp(am);
    if (before == 0) s_cnt[warp * E + e] = base + __popc(grp);
    __syncwarp(am);
  }
  __syncthreads();
  // phase 2: exclusive prefix over warps, per expert (+ chunk base)
  for (int i = threadIdx.x; i < E; i += blockDim.x) {
    int run = s_base[i];
    for (int w = 0; w < kPermWarps; ++w) {
      const int c = s_cnt[w * E + i];
      s_cnt[w * E + i] = run;
      run += c;
    }
  }
  __syncthreads();
  // phase 3: final positions
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    const int e = s_eid[p];
    const int pos = s_cnt[(p / seg) * E + e] + s_pos[p];
    s_pos[p] = pos;
    pair_pos[(int64_t)t0 * k + p] = pos;
    if (row_src) row_src[pos] = t0 + p / k;  // inverse map for the gather-form GEMM
  }
  __syncthreads();
}

// Row movement for every (token, slot) pair, one warp per pair over the whole
// grid (the position kernel above is chunk-parallel only).
__global__ void __launch_bounds__(256) gather_rows_kernel(
    const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ topk_idx,
    const int32_t* __restrict__ pair_pos, int64_t P, int H, int k,
    const uint8_t* __restrict__ prec, __nv_bfloat16* __restrict__ a_bf16,
    uint8_t* __restrict__ a_codes, uint8_t* __restrict__ a_sf, int32_t* flag,
    const int32_t* __restrict__ d_count, const int32_t* __restrict__ d_gate) {
  if (d_gate && *d_gate == 0) return;
  if (d_count && (int64_t)*d_count < P) P = *d_count;  // device-side row count (capacity launch)
  const int lane = threadIdx.x & 31;
  const int nkb = H / 16;
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < P;
       p += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t t = p / k;
    const int e = topk_idx[p];
    const int64_t pos = pair_pos[p];
    const uint4* src = reinterpret_cast<const uint4*>(x + t * H);
    if (prec[e] == REALB_PREC_W16A16) {
      if (!a_bf16) continue;  // the gather-form GEMM reads these rows from x itself
      uint4* dst = reinterpret_cast<uint4*>(a_bf16 + pos * H);
      for (int i = lane; i < H / 8; i += 32) dst[i] = __ldg(src + i);
    } else {
      // lane handles 4 consecutive 16-blocks = one 32-bit word of the SF atom
      for (int g = lane; g < nkb / 4; g += 32) {
        uint32_t sfw = 0;
        uint2 cw[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const uint4 u0 = __ldg(src + (g * 4 + b) * 2), u1 = __ldg(src + (g * 4 + b) * 2 + 1);
          const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
          uint32_t sb;
          bool nf;
          cw[b] = quant_block16_bf16_fast(w, sb, nf);
          if (nf && flag) atomicOr(flag, 1);
          sfw |= sb << (8 * b);
        }
        uint4* cdst = reinterpret_cast<uint4*>(a_codes + pos * (H / 2) + g * 32);
        cdst[0] = make_uint4(cw[0].x, cw[0].y, cw[1].x, cw[1].y);
        cdst[1] = make_uint4(cw[2].x, cw[2].y, cw[3].x, cw[3].y);
        *reinterpret_cast<uint32_t*>(a_sf + sf_mma_offset(pos, (int64_t)g * 4, nkb)) = sfw;
      }
    }
  }
}

// ----------------------------------------------------------------- EP receive side
// Received rows arrive source-major: from rank s, the rows of local expert 0,
// then 1, ... (each sender packs by global expert id). regroup builds the local
// grouped layout (128-row padded, per precision) and, per received row, its
// local expert and its position in the grouped row space.
__global__ void __launch_bounds__(256) ep_layout_kernel(const int32_t* __restrict__ cnt, int R,
                                                        int El, const uint8_t* __restrict__ prec,
                                                        int32_t* __restrict__ layout,
                                                        int32_t* __restrict__ base /*[R*El+1]*/) {
  __shared__ int32_t s_tot[256], s_start[256];
  const int e = threadIdx.x;
  if (e < El) {
    int t = 0;
    for (int r = 0; r < R; ++r) t += cnt[r * El + e];
    s_tot[e] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int i = 0; i < El; ++i) {
      s_start[i] = run;
      run += (s_tot[i] + 127) / 128 * 128;
    }
    layout[0] = run;
    for (int w = 3; w < 8; ++w) layout[w] = 0;  // GEMM tile counters (grouped.cuh)
    for (int p = 0; p < 2; ++p) {
      int32_t* gl = layout + LayoutView::off_glist(El, p);
      int32_t* pf = layout + LayoutView::off_prefix(El, p);
      int32_t* pp2 = layout + LayoutView::off_pprefix(El, p);
      int g = 0, mt = 0, np = 0;
      for (int i = 0; i < El; ++i) {
        if ((int)prec[i] != p) continue;
        gl[g] = i;
        pf[g] = mt;
        pp2[g] = np;
        const int m = (s_tot[i] + 127) / 128;
        mt += m;
        np += (m + 1) / 2;
        ++g;
      }
      pf[g] = mt;
      pp2[g] = np;
      layout[1 + p] = g;
    }
    // source-major prefix of received rows (row index space of the recv buffer)
    int pr = 0;
    for (int f = 0; f < R * El; ++f) {
      base[R * El + 1 + f] = pr;  // recv prefix
      pr += cnt[f];
    }
    base[2 * R * El + 1] = pr;
  }
  __syncthreads();
  if (e < El) {
    layout[LayoutView::off_row_start(El) + e] = s_start[e];
    layout[LayoutView::off_row_count(El) + e] = s_tot[e];
    int run = s_start[e];
    for (int r = 0; r < R; ++r) {
      base[r * El + e] = run;  // grouped position of (source r, expert e)'s first row
      run += cnt[r * El + e];
    }
  }
}

__global__ void __launch_bounds__(256) ep_rows_kernel(const int32_t* __restrict__ base, int R,
                                                      int El, int64_t n,
                                                      int32_t* __restrict__ row_expert,
                                                      int32_t* __restrict__ row_pos) {
  const int F = R * El;
  const int32_t* pre = base + F + 1;  // [F+1] source-major prefix
  if ((int64_t)pre[F] < n) n = pre[F];  // n may be an upper bound (device-count mode)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = F - 1;  // largest f with pre[f] <= i
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pre[mid] <= i) lo = mid; else hi = mid - 1;
    }
    row_expert[i] = lo % El;
    row_pos[i] = base[lo] + (int32_t)(i - pre[lo]);
  }
}

// dst[i] = src[idx[i]]  (bf16 rows; return path of the EP combine)
__global__ void __launch_bounds__(256) index_rows_kernel(const __nv_bfloat16* __restrict__ src,
                                                         const int32_t* __restrict__ idx,
                                                         int64_t n, int H,
                                                         __nv_bfloat16* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src + (int64_t)idx[r] * H);
    uint4* d4 = reinterpret_cast<uint4*>(dst + r * H);
    for (int i = lane; i < H / 8; i += 32) d4[i] = __ldg(s4 + i);
  }
}

// ----------------------------------------------------------------- combine
template <int K>
__global__ void __launch_bounds__(256, 1) combine_kernel(const __nv_bfloat16* __restrict__ rows,
                                                      const int32_t* __restrict__ pos,
                                                      const float* __restrict__ w, int T, int H,
                                                      const __nv_bfloat16* __restrict__ addend,
                                                      __nv_bfloat16* __restrict__ y) {
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const uint4* src[K];
  float wt[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    src[j] = reinterpret_cast<const uint4*>(rows + (int64_t)pos[(int64_t)t * K + j] * H);
    wt[j] = w[(int64_t)t * K + j];
  }
  for (int c = lane; c < H / 8; c += 32) {
    uint4 u[K];
#pragma unroll
    for (int j = 0; j < K; ++j) u[j] = __ldg(src[j] + c);  // all K loads in flight
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (addend) {  // shared-expert output (added in fp32 before the one bf16 rounding)
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(addend + (int64_t)t * H) + c);
      const uint32_t av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[2 * i] = bf16lo(av[i]);
        acc[2 * i + 1] = bf16hi(av[i]);
      }
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const uint32_t v[4] = {u[j].x, u[j].y, u[j].z, u[j].w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[2 * i] = fmaf(wt[j], bf16lo(v[i]), acc[2 * i]);
        acc[2 * i + 1] = fmaf(wt[j], bf16hi(v[i]), acc[2 * i + 1]);
      }
    }
    reinterpret_cast<uint4*>(y + (int64_t)t * H)[c] =
        make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]),
                   pack_bf16x2(acc[4], acc[5]), pack_bf16x2(acc[6], acc[7]));
  }
}

// ----------------------------------------------------------------- rank-partial combine
// The EP return with a per-rank partial sum ("rank-partial return"): a
// W4A4 owner rank d sums token t's rows over ITS slots before the return,
//   P_d(t) = bf16( fma-chain over t's slots j (ascending) with owner(e_j) = d of w_j * y_j ),
// and returns one row per (token, owner) instead of one per (token, slot). The combine
//   y(t) = bf16( addend + slots j ascending: W16A16 slot -> fma(w_j, y_j, acc);
//                first slot of a W4A4 owner d -> acc + P_d(t) )
// is the same arithmetic whether P_d is formed here from the local rows (REMOTE = false:
// the single-GPU layer, and the EP collective path that gets every slot's row back) or
// read from the owner's returned row (REMOTE = true: unit row d * unit_stride + t past
// unit_base of the return window), so the EP layer equals the single-GPU layer exactly.
template <int K, bool REMOTE>
__global__ void __launch_bounds__(256) combine_partial_kernel(
    const __nv_bfloat16* __restrict__ rows, const int32_t* __restrict__ pos, const float* __restrict__ w,
    const int32_t* __restrict__ topk_idx, const uint8_t* __restrict__ prec, int El, int T, int H,
    const __nv_bfloat16* __restrict__ addend, int64_t unit_base, int64_t unit_stride, __nv_bfloat16* __restrict__ y) {
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  int own[K];
  bool w4[K], first[K];
  float wt[K];
  const uint4* src[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int e = topk_idx[(int64_t)t * K + j];
    own[j] = e / El;
    w4[j] = prec[e] == REALB_PREC_W4A4;
    wt[j] = w[(int64_t)t * K + j];
    first[j] = true;
#pragma unroll
    for (int i = 0; i < j; ++i) first[j] = first[j] && own[i] != own[j];
    const int64_t row = (REMOTE && w4[j]) ? unit_base + (int64_t)own[j] * unit_stride + t
                                          : (int64_t)pos[(int64_t)t * K + j];
    src[j] = reinterpret_cast<const uint4*>(rows + row * H);
  }
  for (int c = lane; c < H / 8; c += 32) {
    uint4 u[K];
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (!(REMOTE && w4[j] && !first[j])) u[j] = __ldg(src[j] + c);  // every needed row in flight
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (addend) {
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(addend + (int64_t)t * H) + c);
      const uint32_t av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[2 * i] = bf16lo(av[i]);
        acc[2 * i + 1] = bf16hi(av[i]);
      }
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (!w4[j]) {
        const uint32_t v[4] = {u[j].x, u[j].y, u[j].z, u[j].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[2 * i] = fmaf(wt[j], bf16lo(v[i]), acc[2 * i]);
          acc[2 * i + 1] = fmaf(wt[j], bf16hi(v[i]), acc[2 * i + 1]);
        }
      } else if (first[j]) {
        uint32_t pv[4];
        if constexpr (REMOTE) {
          pv[0] = u[j].x; pv[1] = u[j].y; pv[2] = u[j].z; pv[3] = u[j].w;
        } else {  // the owner's partial: its slots in ascending order, one bf16 rounding
          float p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
          for (int jj = j; jj < K; ++jj) {
            if (own[jj] != own[j]) continue;
            const uint32_t v[4] = {u[jj].x, u[jj].y, u[jj].z, u[jj].w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              p[2 * i] = fmaf(wt[jj], bf16lo(v[i]), p[2 * i]);
              p[2 * i + 1] = fmaf(wt[jj], bf16hi(v[i]), p[2 * i + 1]);
            }
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) pv[i] = pack_bf16x2(p[2 * i], p[2 * i + 1]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[2 * i] += bf16lo(pv[i]);
          acc[2 * i + 1] += bf16hi(pv[i]);
        }
      }
    }
    reinterpret_cast<uint4*>(y + (int64_t)t * H)[c] =
        make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]),
                   pack_bf16x2(acc[4], acc[5]), pack_bf16x2(acc[6], acc[7]));
  }
}

// ----------------------------------------------------------------- EP pack (send side, C2)
// One warp per (token, slot) pair: the row goes to destination rank d = e / El,
// at byte offset byte0[d] + (pos - row0[d]) * row_bytes(fmt[d]) of the send
// buffer (pos = the pair's place in the expert-sorted, unpadded order, so each
// destination's rows are one contiguous segment). fmt 0: the bf16 row (2H
// bytes); fmt 1: the row quantised to NVFP4 with the reference block rule along
// H (K4 moved before dispatch) as one packed row:
// [H/2 code bytes][H/16 E4M3 scale bytes] — 0.5625 H bytes instead of 2 H.
constexpr int kMaxEpRanks = 64;
struct EpPackMeta {
  int R, El;
  uint8_t fmt[kMaxEpRanks];
  int32_t row0[kMaxEpRanks];
  int64_t byte0[kMaxEpRanks];
};

__global__ void __launch_bounds__(256) ep_pack_rows_kernel(
    const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ topk_idx,
    const int32_t* __restrict__ pair_pos, int64_t P, int H, int k, const EpPackMeta m,
    uint8_t* __restrict__ dst, int32_t* flag) {
  const int lane = threadIdx.x & 31;
  const int nkb = H / 16;
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < P;
       p += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t t = p / k;
    const int d = topk_idx[p] / m.El;
    const int64_t rel = (int64_t)pair_pos[p] - m.row0[d];
    const uint4* src = reinterpret_cast<const uint4*>(x + t * H);
    if (m.fmt[d] == 0) {
      uint4* o = reinterpret_cast<uint4*>(dst + m.byte0[d] + rel * (2 * (int64_t)H));
      for (int i = lane; i < H / 8; i += 32) o[i] = __ldg(src + i);
    } else {
      uint8_t* row = dst + m.byte0[d] + rel * (int64_t)(H / 2 + H / 16);
      for (int g = lane; g < nkb / 4; g += 32) {
        uint32_t sfw = 0;
        uint2 cw[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const uint4 u0 = __ldg(src + (g * 4 + b) * 2), u1 = __ldg(src + (g * 4 + b) * 2 + 1);
          const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
          uint32_t sb;
          bool nf;
          cw[b] = quant_block16_bf16_fast(w, sb, nf);
          if (nf && flag) atomicOr(flag, 1);
          sfw |= sb << (8 * b);
        }
        uint4* cdst = reinterpret_cast<uint4*>(row + g * 32);
        cdst[0] = make_uint4(cw[0].x, cw[0].y, cw[1].x, cw[1].y);
        cdst[1] = make_uint4(cw[2].x, cw[2].y, cw[3].x, cw[3].y);
        reinterpret_cast<uint32_t*>(row + H / 2)[g] = sfw;
      }
    }
  }
}

// EP receive side of the NVFP4 dispatch: packed rows -> grouped NVFP4 operand
// (codes row-major at the row's grouped position, scales into the tcgen05
// block-scale layout). Pure byte movement: the codes are the sender's.
__global__ void __launch_bounds__(256) gather_packed_fp4_kernel(const uint8_t* __restrict__ src,
                                                                const int32_t* __restrict__ row_pos,
                                                                int64_t n, int H,
                                                                uint8_t* __restrict__ a_codes,
                                                                uint8_t* __restrict__ a_sf,
                                                                const int32_t* __restrict__ d_count,
                                                                const int32_t* __restrict__ d_gate) {
  if (d_gate && *d_gate == 0) return;
  if (d_count && (int64_t)*d_count < n) n = *d_count;
  const int lane = threadIdx.x & 31;
  const int nkb = H / 16;
  const int64_t rb = H / 2 + H / 16;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t pos = row_pos[i];
    const uint8_t* row = src + i * rb;
    const uint4* c4 = reinterpret_cast<const uint4*>(row);
    uint4* o4 = reinterpret_cast<uint4*>(a_codes + pos * (H / 2));
    for (int j = lane; j < H / 32; j += 32) o4[j] = __ldg(c4 + j);
    const uint32_t* s4 = reinterpret_cast<const uint32_t*>(row + H / 2);
    for (int g = lane; g < nkb / 4; g += 32)
      *reinterpret_cast<uint32_t*>(a_sf + sf_mma_offset(pos, (int64_t)g * 4, nkb)) = __ldg(s4 + g);
  }
}

// expert-sorted positions of every (token, slot) pair (the permute step shared by
// dispatch, the EP pack and the peer-memory pack)
int ep_positions(const int32_t* topk_idx, int T, int E, int k, const int32_t* layout, int nchunks,
                 int32_t* pair_pos, void* stream) {
  const int smem = (E + kPermWarps * E + 2 * REALB_CHUNK_TOKENS * k) * 4;
  permute_kernel<<<nchunks, 256, smem, (cudaStream_t)stream>>>(topk_idx, T, E, k, layout, pair_pos);
  return check_launch("pair positions");
}

}  // namespace realb

using namespace realb;

extern "C" int64_t realb_layout_words(int E, int nchunks) {
  if (E < 1 || nchunks < 0) return REALB_EINVAL;
  return LayoutView::words(E, nchunks);
}

extern "C" int realb_moe_align(const int32_t* d_cc, int nchunks, int E, const uint8_t* d_prec,
                               int row_align, int32_t* d_layout, int32_t* d_expert_vt,
                               void* stream) {
  if ((!d_cc && nchunks > 0) || !d_prec || !d_layout || !d_expert_vt || E < 1 || E > 256 ||
      nchunks < 0) {
    set_error("realb_moe_align: bad arguments (E=%d nchunks=%d; E <= 256)", E, nchunks);
    return REALB_EINVAL;
  }
  if (row_align != 1 && row_align != 128) {
    set_error("realb_moe_align: row_align must be 1 or 128 (got %d)", row_align);
    return REALB_EINVAL;
  }
  PlanParams pp{};
  align_kernel<<<1, kAlignThreads, 0, (cudaStream_t)stream>>>(d_cc, nchunks, E, const_cast<uint8_t*>(d_prec),
                                                    d_layout, d_expert_vt, pp, nullptr, row_align);
  return check_launch("realb_moe_align");
}

extern "C" int realb_moe_align_plan(const int32_t* d_cc, int nchunks, int E, int R, int strategy,
                                    double capacity_factor, double modality_threshold,
                                    int64_t global_batch_threshold, int modality_isolated,
                                    uint8_t* d_prec, int32_t* d_plan_out, int32_t* d_layout,
                                    int32_t* d_expert_vt, void* stream) {
  if ((!d_cc && nchunks > 0) || !d_prec || !d_layout || !d_expert_vt || E < 1 || E > 256 ||
      nchunks < 0 || R < 1 ||
      R > 256 || E % R || strategy < 0 || strategy > 2) {
    set_error("realb_moe_align_plan: bad arguments (E=%d R=%d strategy=%d)", E, R, strategy);
    return REALB_EINVAL;
  }
  if (!(capacity_factor > 0.0) || !(modality_threshold >= 0.0 && modality_threshold <= 1.0) ||
      global_batch_threshold < 0) {
    set_error("realb_moe_align_plan: invalid RealbParams");
    return REALB_EINVAL;
  }
  PlanParams pp{1, strategy, R, modality_isolated, capacity_factor, modality_threshold,
                (long long)global_batch_threshold};
  align_kernel<<<1, kAlignThreads, 0, (cudaStream_t)stream>>>(d_cc, nchunks, E, d_prec, d_layout,
                                                    d_expert_vt, pp, d_plan_out, 128);
  return check_launch("realb_moe_align_plan");
}

extern "C" int realb_dispatch_permute(const void* d_x, const int32_t* d_topk_idx, int T, int H,
                                      int E, int k, const uint8_t* d_prec,
                                      const int32_t* d_layout, int nchunks, int64_t rows_cap,
                                      int32_t* d_pair_pos, void* d_a_bf16, uint8_t* d_a_codes,
                                      uint8_t* d_a_sf, int32_t* d_flag, void* stream) {
  if (T == 0 && nchunks == 0) return REALB_OK;
  if (!d_x || !d_topk_idx || !d_prec || !d_layout || !d_pair_pos || !d_a_bf16 || T < 0 ||
      H <= 0 || H % 64 || E < 1 || E > 256 || k < 1 || k > 8 || nchunks != (T + REALB_CHUNK_TOKENS - 1) / REALB_CHUNK_TOKENS) {
    set_error("realb_dispatch_permute: bad arguments (T=%d H=%d E=%d k=%d nchunks=%d)", T, H, E,
              k, nchunks);
    return REALB_EINVAL;
  }
  if (T == 0) return REALB_OK;
  const int smem = (E + kPermWarps * E + 2 * REALB_CHUNK_TOKENS * k) * 4;
  permute_kernel<<<nchunks, 256, smem, (cudaStream_t)stream>>>(d_topk_idx, T, E, k, d_layout,
                                                                d_pair_pos);
  int rc = check_launch("realb_dispatch_permute (positions)");
  if (rc) return rc;
  const int64_t P = (int64_t)T * k;
  int64_t grid = (P + 7) / 8;
  if (grid > (int64_t)num_sms() * 16) grid = (int64_t)num_sms() * 16;
  gather_rows_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const __nv_bfloat16*>(d_x), d_topk_idx, d_pair_pos, P, H, k, d_prec,
      reinterpret_cast<__nv_bfloat16*>(d_a_bf16), d_a_codes, d_a_sf, d_flag, nullptr, nullptr);
  return check_launch("realb_dispatch_permute (rows)");
}

extern "C" int realb_dispatch_index(const void* d_x, const int32_t* d_topk_idx, int T, int H, int E, int k,
                                    const uint8_t* d_prec, const int32_t* d_layout, int nchunks,
                                    int64_t rows_cap, int32_t* d_pair_pos, int32_t* d_row_src,
                                    uint8_t* d_a_codes, uint8_t* d_a_sf, int32_t* d_flag, void* stream) {
  if (T == 0 && nchunks == 0) return REALB_OK;
  if (!d_x || !d_topk_idx || !d_prec || !d_layout || !d_pair_pos || !d_row_src || (!d_a_codes != !d_a_sf) ||
      T < 0 || H <= 0 || H % 64 || E < 1 || E > 256 || k < 1 || k > 8 || rows_cap < (int64_t)T * k ||
      nchunks != (T + REALB_CHUNK_TOKENS - 1) / REALB_CHUNK_TOKENS) {
    set_error("realb_dispatch_index: bad arguments (T=%d H=%d E=%d k=%d nchunks=%d)", T, H, E, k, nchunks);
    return REALB_EINVAL;
  }
  if (T == 0) return REALB_OK;
  const int smem = (E + kPermWarps * E + 2 * REALB_CHUNK_TOKENS * k) * 4;
  permute_kernel<<<nchunks, 256, smem, (cudaStream_t)stream>>>(d_topk_idx, T, E, k, d_layout, d_pair_pos,
                                                                d_row_src);
  int rc = check_launch("realb_dispatch_index (positions)");
  if (rc || !d_a_codes) return rc;
  // only the rows of W4A4 experts move (K4 quantisation into the NVFP4 operand)
  const int64_t P = (int64_t)T * k;
  int64_t grid = (P + 7) / 8;
  if (grid > (int64_t)num_sms() * 16) grid = (int64_t)num_sms() * 16;
  gather_rows_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const __nv_bfloat16*>(d_x), d_topk_idx, d_pair_pos, P, H, k, d_prec, nullptr, d_a_codes,
      d_a_sf, d_flag, nullptr, nullptr);
  return check_launch("realb_dispatch_index (nvfp4 rows)");
}

extern "C" int realb_combine(const void* d_rows, const int32_t* d_pos, const float* d_w, int T,
                             int H, int k, const void* d_addend, void* d_y, void* stream) {
  if (T == 0 && H > 0 && H % 8 == 0 && k >= 1 && k <= 8) return REALB_OK;
  if (!d_rows || !d_pos || !d_w || !d_y || T < 0 || H <= 0 || H % 8 || k < 1 || k > 8) {
    set_error("realb_combine: bad arguments (T=%d H=%d k=%d)", T, H, k);
    return REALB_EINVAL;
  }
  if (T == 0) return REALB_OK;
  const dim3 grid((T + 7) / 8);
  cudaStream_t st = (cudaStream_t)stream;
  auto r = reinterpret_cast<const __nv_bfloat16*>(d_rows);
  auto ad = reinterpret_cast<const __nv_bfloat16*>(d_addend);
  auto y = reinterpret_cast<__nv_bfloat16*>(d_y);
  switch (k) {
    case 1: combine_kernel<1><<<grid, 256, 0, st>>>(r, d_pos, d_w, T, H, ad, y); break;
    case 2: combine_kernel<2><<<grid, 256, 0, st>>>(r, d_pos, d_w, T, H, ad, y); break;
    case 4: combine_kernel<4><<<grid, 256, 0, st>>>(r, d_pos, d_w, T, H, ad, y); break;
    case 6: combine_kernel<6><<<grid, 256, 0, st>>>(r, d_pos, d_w, T, H, ad, y); break;
    case 8: combine_kernel<8><<<grid, 256, 0, st>>>(r, d_pos, d_w, T, H, ad, y); break;
    default:
      set_error("realb_combine: top-k must be one of 1,2,4,6,8 (k=%d)", k);
      return REALB_EUNSUPPORTED;
  }
  return check_launch("realb_combine");
}

extern "C" int realb_combine_partial(const void* d_rows, const int32_t* d_pos, const float* d_w,
                                     const int32_t* d_topk_idx, const uint8_t* d_expert_prec, int El, int T, int H,
                                     int k, const void* d_addend, int64_t unit_base, int64_t unit_stride, void* d_y,
                                     void* stream) {
  if (T == 0 && H > 0 && H % 8 == 0 && k >= 1 && k <= 8 && El >= 1) return REALB_OK;
  if (!d_rows || !d_pos || !d_w || !d_topk_idx || !d_expert_prec || !d_y || T < 0 || H <= 0 || H % 8 || k < 1 ||
      k > 8 || El < 1 || unit_base < -1 || (unit_base >= 0 && unit_stride < T)) {
    set_error("realb_combine_partial: bad arguments (T=%d H=%d k=%d El=%d)", T, H, k, El);
    return REALB_EINVAL;
  }
  if (T == 0) return REALB_OK;
  const dim3 grid((T + 7) / 8);
  cudaStream_t st = (cudaStream_t)stream;
  auto r = reinterpret_cast<const __nv_bfloat16*>(d_rows);
  auto ad = reinterpret_cast<const __nv_bfloat16*>(d_addend);
  auto y = reinterpret_cast<__nv_bfloat16*>(d_y);
  const bool remote = unit_base >= 0;
#define REALB_CP(KK)                                                                                              \
  case KK:                                                                                                        \
    if (remote)                                                                                                   \
      combine_partial_kernel<KK, true><<<grid, 256, 0, st>>>(r, d_pos, d_w, d_topk_idx, d_expert_prec, El, T, H, \
                                                             ad, unit_base, unit_stride, y);                       \
    else                                                                                                          \
      combine_partial_kernel<KK, false><<<grid, 256, 0, st>>>(r, d_pos, d_w, d_topk_idx, d_expert_prec, El, T, H, \
                                                              ad, 0, 0, y);                                         \
    break;
  switch (k) {
    REALB_CP(1)
    REALB_CP(2)
    REALB_CP(4)
    REALB_CP(6)
    REALB_CP(8)
    default:
      set_error("realb_combine_partial: top-k must be one of 1,2,4,6,8 (k=%d)", k);
      return REALB_EUNSUPPORTED;
  }
#undef REALB_CP
  return check_launch("realb_combine_partial");
}

extern "C" int realb_gather_rows(const void* d_x, const int32_t* d_expert, const int32_t* d_pos,
                                 int64_t P, int H, int k, const uint8_t* d_prec, void* d_a_bf16,
                                 uint8_t* d_a_codes, uint8_t* d_a_sf, int32_t* d_flag,
                                 const int32_t* d_count, const int32_t* d_gate, void* stream) {
  if (!d_x || !d_expert || !d_pos || !d_prec || !d_a_bf16 || P < 0 || H <= 0 || H % 64 || k < 1) {
    set_error("realb_gather_rows: bad arguments");
    return REALB_EINVAL;
  }
  if (P == 0) return REALB_OK;
  int64_t grid = (P + 7) / 8;
  if (grid > (int64_t)num_sms() * 16) grid = (int64_t)num_sms() * 16;
  gather_rows_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const __nv_bfloat16*>(d_x), d_expert, d_pos, P, H, k, d_prec,
      reinterpret_cast<__nv_bfloat16*>(d_a_bf16), d_a_codes, d_a_sf, d_flag, d_count, d_gate);
  return check_launch("realb_gather_rows");
}

extern "C" int realb_ep_regroup(const int32_t* d_cnt, int R, int El, const uint8_t* d_prec_local,
                                int64_t n_recv, int32_t* d_layout, int32_t* d_base,
                                int32_t* d_row_expert, int32_t* d_row_pos, void* stream) {
  if (!d_cnt || !d_prec_local || !d_layout || !d_base || R < 1 || El < 1 || El > 256 ||
      R * El > 4096 || n_recv < 0 || (n_recv > 0 && (!d_row_expert || !d_row_pos))) {
    set_error("realb_ep_regroup: bad arguments (R=%d El=%d)", R, El);
    return REALB_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  ep_layout_kernel<<<1, 256, 0, st>>>(d_cnt, R, El, d_prec_local, d_layout, d_base);
  int rc = check_launch("realb_ep_regroup (layout)");
  if (rc || n_recv == 0) return rc;
  int64_t grid = (n_recv + 255) / 256;
  if (grid > (int64_t)num_sms() * 8) grid = (int64_t)num_sms() * 8;
  ep_rows_kernel<<<(unsigned)grid, 256, 0, st>>>(d_base, R, El, n_recv, d_row_expert, d_row_pos);
  return check_launch("realb_ep_regroup (rows)");
}

extern "C" int realb_index_rows(const void* d_src, const int32_t* d_idx, int64_t n, int H,
                                void* d_dst, void* stream) {
  if (!d_src || !d_idx || !d_dst || n < 0 || H <= 0 || H % 8) {
    set_error("realb_index_rows: bad arguments");
    return REALB_EINVAL;
  }
  if (n == 0) return REALB_OK;
  int64_t grid = (n + 7) / 8;
  if (grid > (int64_t)num_sms() * 16) grid = (int64_t)num_sms() * 16;
  index_rows_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const __nv_bfloat16*>(d_src), d_idx, n, H,
      reinterpret_cast<__nv_bfloat16*>(d_dst));
  return check_launch("realb_index_rows");
}

extern "C" int realb_ep_pack(const void* d_x, const int32_t* d_topk_idx, int T, int H, int E, int k,
                             const int32_t* d_layout, int nchunks, int R, const uint8_t* h_rank_fmt,
                             const int32_t* h_rank_row0, const int64_t* h_rank_byte0,
                             int32_t* d_pair_pos, uint8_t* d_send, int32_t* d_flag, void* stream) {
  if (!d_x || !d_topk_idx || !d_layout || !d_pair_pos || !d_send || !h_rank_fmt || !h_rank_row0 ||
      !h_rank_byte0 || T < 0 || H <= 0 || H % 64 || E < 1 || E > 256 || k < 1 || k > 8 || R < 1 ||
      R > kMaxEpRanks || E % R || nchunks != (T + REALB_CHUNK_TOKENS - 1) / REALB_CHUNK_TOKENS) {
    set_error("realb_ep_pack: bad arguments (T=%d H=%d E=%d k=%d R=%d nchunks=%d)", T, H, E, k, R,
              nchunks);
    return REALB_EINVAL;
  }
  EpPackMeta m{};
  m.R = R;
  m.El = E / R;
  for (int d = 0; d < R; ++d) {
    if (h_rank_fmt[d] > 1 || (h_rank_byte0[d] & 15)) {
      set_error("realb_ep_pack: rank %d: format must be 0/1 and byte offsets 16-byte aligned", d);
      return REALB_EINVAL;
    }
    m.fmt[d] = h_rank_fmt[d];
    m.row0[d] = h_rank_row0[d];
    m.byte0[d] = h_rank_byte0[d];
  }
  if (T == 0) return REALB_OK;
  const int smem = (E + kPermWarps * E + 2 * REALB_CHUNK_TOKENS * k) * 4;
  permute_kernel<<<nchunks, 256, smem, (cudaStream_t)stream>>>(d_topk_idx, T, E, k, d_layout,
                                                                d_pair_pos);
  int rc = check_launch("realb_ep_pack (positions)");
  if (rc) return rc;
  const int64_t P = (int64_t)T * k;
  int64_t grid = (P + 7) / 8;
  if (grid > (int64_t)num_sms() * 16) grid = (int64_t)num_sms() * 16;
  ep_pack_rows_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const __nv_bfloat16*>(d_x), d_topk_idx, d_pair_pos, P, H, k, m, d_send, d_flag);
  return check_launch("realb_ep_pack (rows)");
}

extern "C" int realb_gather_rows_nvfp4_packed(const uint8_t* d_src, const int32_t* d_pos, int64_t n,
                                              int H, uint8_t* d_a_codes, uint8_t* d_a_sf,
                                              const int32_t* d_count, const int32_t* d_gate,
                                              void* stream) {
  if (!d_src || !d_pos || !d_a_codes || !d_a_sf || n < 0 || H <= 0 || H % 256) {
    set_error("realb_gather_rows_nvfp4_packed: bad arguments (H=%d; H %% 256 == 0)", H);
    return REALB_EINVAL;
  }
  if (n == 0) return REALB_OK;
  int64_t grid = (n + 7) / 8;
  if (grid > (int64_t)num_sms() * 16) grid = (int64_t)num_sms() * 16;
  gather_packed_fp4_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(d_src, d_pos, n, H,
                                                                             d_a_codes, d_a_sf, d_count,
                                                                             d_gate);
  return check_launch("realb_gather_rows_nvfp4_packed");
}
