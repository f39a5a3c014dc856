// p2p.cu — peer-memory transport of the EP layer (C2 dispatch / C3 return
// without a collective library): every rank exposes a receive window and a
// return window (cudaMalloc'd, shared through CUDA IPC handles: NVLink peer
// memory on a multi-GPU node, plain device memory when the processes share one
// GPU), and the pack / return kernels write rows straight into the peers'
// windows. Completion is signalled with system-scope counters in the
// receiver's window and awaited by a spin kernel, all stream-ordered: no host
// synchronisation and no NCCL call on the data path.
//
// Window offsets are a pure function of the [R][R] pair-count matrix every
// rank holds after C1 (source-major receive order, expert-sorted send order),
// so senders and receivers agree on every row's address without a handshake.
#include <cstddef>
#include <cstring>

#include "common.cuh"
#include "fp4_rule.cuh"

namespace realb {

constexpr int kMaxPeers = 64;

struct PeerRows {
  uint8_t* base[kMaxPeers];  // destination address of the first row bound for peer d
  int32_t row0[kMaxPeers];   // expert-sorted send position of that first row
  uint8_t fmt[kMaxPeers];    // 0 bf16 rows (2H bytes), 1 packed NVFP4 rows (H/2 + H/16)
  int R, El;
};

// one warp per (token, slot) pair: the row goes to peer d = e / El at
// base[d] + (pos - row0[d]) * row_bytes(fmt[d])
__global__ void __launch_bounds__(256) p2p_pack_kernel(const __nv_bfloat16* __restrict__ x,
                                                       const int32_t* __restrict__ topk_idx,
                                                       const int32_t* __restrict__ pair_pos, int64_t P,
                                                       int H, int k, const PeerRows m, int32_t* flag) {
  const int lane = threadIdx.x & 31;
  const int nkb = H / 16;
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < P;
       p += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t t = p / k;
    const int d = topk_idx[p] / m.El;
    const int64_t rel = (int64_t)pair_pos[p] - m.row0[d];
    const uint4* src = reinterpret_cast<const uint4*>(x + t * H);
    if (m.fmt[d] == 0) {
      uint4* o = reinterpret_cast<uint4*>(m.base[d] + rel * (2 * (int64_t)H));
      for (int i = lane; i < H / 8; i += 32) o[i] = __ldg(src + i);
    } else {
      uint8_t* row = m.base[d] + rel * (int64_t)(H / 2 + H / 16);
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

struct PeerReturn {
  __nv_bfloat16* base[kMaxPeers];  // peer s's return window + its first row's offset
  int32_t recv0[kMaxPeers + 1];    // source-major prefix of my received rows
  int R;
};

// received row i (from source s, its j-th) goes back to s's return window at
// row j of the block s expects from me; its data is my grouped row row_pos[i]
__global__ void __launch_bounds__(256) p2p_return_kernel(const __nv_bfloat16* __restrict__ rows,
                                                         const int32_t* __restrict__ row_pos, int64_t n,
                                                         int H, const PeerReturn m) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int s = 0;
    while (s + 1 < m.R && m.recv0[s + 1] <= i) ++s;
    const uint4* src = reinterpret_cast<const uint4*>(rows + (int64_t)row_pos[i] * H);
    uint4* dst = reinterpret_cast<uint4*>(m.base[s] + (i - m.recv0[s]) * (int64_t)H);
    for (int c = lane; c < H / 8; c += 32) dst[c] = __ldg(src + c);
  }
}

struct PeerCounters {
  uint32_t* ctr[kMaxPeers];
  int R;
};

// release: this stream's earlier writes (the pack / return kernels) become
// visible system-wide before each peer's counter is bumped
__global__ void p2p_signal_kernel(const PeerCounters m) {
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int d = 0; d < m.R; ++d) atomicAdd_system(m.ctr[d], 1u);
  }
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr uint64_t kWaitTimeoutNs = 10ull * 1000 * 1000 * 1000;  // a dead peer must not hang the GPU

// acquire spin until *ctr reaches target; after kWaitTimeoutNs without it, raise
// *err (if given) and give up, so a broken transport fails loudly instead of hanging
__device__ __forceinline__ void spin_until(const uint32_t* ctr, uint32_t target, int32_t* err) {
  const uint64_t t0 = global_ns();
  uint32_t v;
  for (;;) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    if ((int32_t)(v - target) >= 0) break;
    if (err && global_ns() - t0 > kWaitTimeoutNs) {
      atomicOr(err, 1);
      break;
    }
    __nanosleep(256);
  }
  __threadfence_system();
}

// acquire: spin until my counter reaches `target` (all peers have signalled)
__global__ void p2p_wait_kernel(const uint32_t* ctr, uint32_t target, int32_t* err) {
  if (threadIdx.x == 0) spin_until(ctr, target, err);
}

// ---------------------------------------------------------------------------
// Host-sync-free form: the C1 counts travel through peer memory too, and every
// rank derives the plan and all window offsets ON THE DEVICE from the gathered
// [R][E][2] counts, so the whole EP layer is stream-ordered and CUDA-graph
// capturable (realb_p2p_publish, realb_p2p_plan_offsets and the *_dev kernels).
struct P2PPlan {
  int32_t row0[kMaxPeers];       // my send-order position of the first row bound for peer d
  int64_t dst_off[kMaxPeers];    // byte offset of my block inside peer d's receive window
  int32_t fmt[kMaxPeers];        // row format towards peer d (0 bf16, 1 packed NVFP4)
  int32_t recv0[kMaxPeers + 1];  // source-major prefix of the rows I receive
  int32_t ret_row0[kMaxPeers];   // row offset of my block inside source s's return window
  int32_t n_recv;                // rows I receive (= recv0[R])
  int32_t w4a4;                  // my precision (W4A4 = 1)
  int32_t gate_bf16, gate_packed;  // which receive-side gather runs
  // direct dispatch: grouped row (the owner's GEMM operand row space, 128-padded
  // per expert, source-major inside an expert) of MY first row of each global expert
  int32_t gpos0[256];
};

__global__ void p2p_publish_kernel(const int32_t* __restrict__ src, int n, const PeerRows dst,
                                   int64_t off_words) {
  for (int d = 0; d < dst.R; ++d) {
    int32_t* o = reinterpret_cast<int32_t*>(dst.base[d]) + off_words;
    for (int i = threadIdx.x; i < n; i += blockDim.x) o[i] = src[i];
  }
}

__global__ void __launch_bounds__(256) p2p_plan_kernel(const int32_t* __restrict__ counts, int R, int E,
                                                        int rank, int H, int fp4_dispatch,
                                                        const uint8_t* __restrict__ prec, P2PPlan* plan,
                                                        int32_t* __restrict__ cnt_local,
                                                        uint8_t* __restrict__ prec_local) {
  __shared__ int32_t pairs[kMaxPeers * kMaxPeers];  // [s][d]
  const int El = E / R;
  for (int i = threadIdx.x; i < R * R; i += blockDim.x) {
    const int s = i / R, d = i - s * R;
    int acc = 0;
    for (int e = d * El; e < (d + 1) * El; ++e) acc += counts[(s * E + e) * 2] + counts[(s * E + e) * 2 + 1];
    pairs[i] = acc;
  }
  for (int i = threadIdx.x; i < R * El; i += blockDim.x) {
    const int s = i / El, le = i - s * El, e = rank * El + le;
    cnt_local[i] = counts[(s * E + e) * 2] + counts[(s * E + e) * 2 + 1];
  }
  for (int i = threadIdx.x; i < El; i += blockDim.x) prec_local[i] = prec[rank * El + i];
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t run = 0;
    for (int d = 0; d < R; ++d) {
      const int f = fp4_dispatch && prec[d * El] == REALB_PREC_W4A4;
      const int64_t units = f ? (H / 2 + H / 16) : 2 * (int64_t)H;
      int64_t before = 0;
      for (int s2 = 0; s2 < rank; ++s2) before += pairs[s2 * R + d];
      plan->row0[d] = run;
      plan->dst_off[d] = before * units;
      plan->fmt[d] = f;
      run += pairs[rank * R + d];
    }
    int32_t pr = 0;
    for (int s2 = 0; s2 < R; ++s2) {
      plan->recv0[s2] = pr;
      pr += pairs[s2 * R + rank];
      int32_t before = 0;
      for (int d = 0; d < rank; ++d) before += pairs[s2 * R + d];
      plan->ret_row0[s2] = before;
    }
    plan->recv0[R] = pr;
    plan->n_recv = pr;
    // the owner's grouped layout (ep_layout_kernel's rule: experts in order, each
    // padded to 128 rows, sources in rank order inside an expert)
    for (int d = 0; d < R; ++d) {
      int32_t start = 0;
      for (int le = 0; le < El; ++le) {
        const int e = d * El + le;
        int32_t tot = 0, before = 0;
        for (int s2 = 0; s2 < R; ++s2) {
          const int32_t c = counts[(s2 * E + e) * 2] + counts[(s2 * E + e) * 2 + 1];
          tot += c;
          if (s2 < rank) before += c;
        }
        plan->gpos0[e] = start + before;
        start += (tot + 127) / 128 * 128;
      }
    }
    const int w4 = prec[rank * El] == REALB_PREC_W4A4;
    plan->w4a4 = w4;
    plan->gate_packed = w4 && fp4_dispatch;
    plan->gate_bf16 = !(w4 && fp4_dispatch);
  }
}

// graph-safe wait: the expected value lives in device memory and advances by
// `inc` (= R signals per layer) on every call, so a captured graph can replay it
__global__ void p2p_wait_next_kernel(uint32_t* expected, uint32_t inc, const uint32_t* ctr, int32_t* err) {
  if (threadIdx.x == 0) {
    const uint32_t target = *expected + inc;
    *expected = target;
    spin_until(ctr, target, err);
  }
}

// pack with the per-peer row offsets / formats read from the device plan
__global__ void __launch_bounds__(256) p2p_pack_dev_kernel(const __nv_bfloat16* __restrict__ x,
                                                           const int32_t* __restrict__ topk_idx,
                                                           const int32_t* __restrict__ pair_pos, int64_t P,
                                                           int H, int k, const PeerRows win,
                                                           const P2PPlan* __restrict__ plan, int32_t* flag) {
  const int lane = threadIdx.x & 31;
  const int nkb = H / 16;
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < P;
       p += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t t = p / k;
    const int d = topk_idx[p] / win.El;
    const int64_t rel = (int64_t)pair_pos[p] - plan->row0[d];
    const uint4* src = reinterpret_cast<const uint4*>(x + t * H);
    uint8_t* base = win.base[d] + plan->dst_off[d];
    if (plan->fmt[d] == 0) {
      uint4* o = reinterpret_cast<uint4*>(base + rel * (2 * (int64_t)H));
      for (int i = lane; i < H / 8; i += 32) o[i] = __ldg(src + i);
    } else {
      uint8_t* row = base + rel * (int64_t)(H / 2 + H / 16);
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

struct PeerOperands {
  __nv_bfloat16* a[kMaxPeers];  // peer d's bf16 GEMM operand rows [rows_cap][H]
  uint8_t* codes[kMaxPeers];    // peer d's NVFP4 operand codes [rows_cap][H/2]
  uint8_t* sf[kMaxPeers];       // peer d's NVFP4 scales, ROW-MAJOR staging [rows_cap][H/16]
  int R, El;
  // rank-partial return (realb_p2p_pack_direct_partial): for a W4A4 destination d the
  // sender also records, per (me, token t, slot j), the grouped row g in d's unit table
  // units[d][(me * ustride + t) * k + j] and the routing weight in wts[d][g]
  int32_t* units[kMaxPeers];
  float* wts[kMaxPeers];
  const float* topk_w;
  int me;
  int64_t ustride;
};

// Direct dispatch: every (token, slot) row is written straight into its
// destination's GEMM operand at its final grouped row — bf16 for a W16A16
// destination, NVFP4 codes (the K4 rule) for a W4A4 one — so the receiver runs
// no row gather. Every warp store is one contiguous 512-B span (wide peer-memory
// writes): the NVFP4 codes are regrouped across lanes with shuffles, and the
// scales go row-major (128 B per row) into a staging window that the receiver
// turns into the MMA 128x4 layout locally (realb_sf_rows_to_mma); written in that
// layout directly, a row's scales would be 32 separate 4-B remote writes.
__global__ void __launch_bounds__(256) p2p_pack_direct_kernel(const __nv_bfloat16* __restrict__ x,
                                                              const int32_t* __restrict__ topk_idx,
                                                              const int32_t* __restrict__ pair_pos,
                                                              const int32_t* __restrict__ send_start,
                                                              int64_t P, int H, int k, const PeerOperands ops,
                                                              const P2PPlan* __restrict__ plan, int32_t* flag) {
  const int lane = threadIdx.x & 31;
  const int nkb = H / 16;
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < P;
       p += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t t = p / k;
    const int e = topk_idx[p];
    const int d = e / ops.El;
    const int64_t g = (int64_t)plan->gpos0[e] + (pair_pos[p] - send_start[e]);
    const uint4* src = reinterpret_cast<const uint4*>(x + t * H);
    if (ops.topk_w && plan->fmt[d] == 1 && lane == 0) {  // rank-partial metadata (W4A4 owner)
      ops.units[d][((int64_t)ops.me * ops.ustride + t) * k + (p - t * k)] = (int32_t)g;
      ops.wts[d][g] = ops.topk_w[p];
    }
    if (plan->fmt[d] == 0) {
      uint4* o = reinterpret_cast<uint4*>(ops.a[d] + g * H);
      for (int i = lane; i < H / 8; i += 32) o[i] = __ldg(src + i);
    } else {
      // lane l quantises 64-element group gi = gi0 + l (32 B of codes, one 4-B scale word);
      // each store instruction then writes 512 contiguous code bytes: lane m stores half
      // (m & 1) of the group held by lane (m >> 1) (+16 for the second instruction)
      uint4* crow = reinterpret_cast<uint4*>(ops.codes[d] + g * (H / 2));
      uint32_t* srow = reinterpret_cast<uint32_t*>(ops.sf[d] + g * (H / 16));
      for (int gi0 = 0; gi0 < nkb / 4; gi0 += 32) {  // H % 64 == 0: nkb / 4 groups per row
        const int gi = gi0 + lane;
        const bool act = gi < nkb / 4;
        uint32_t sfw = 0;
        uint2 cw[4] = {};
        if (act) {
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const uint4 u0 = __ldg(src + (gi * 4 + b) * 2), u1 = __ldg(src + (gi * 4 + b) * 2 + 1);
            const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
            uint32_t sb;
            bool nf;
            cw[b] = quant_block16_bf16_fast(w, sb, nf);
            if (nf && flag) atomicOr(flag, 1);
            sfw |= sb << (8 * b);
          }
          srow[gi] = sfw;  // lanes write consecutive words: 128 contiguous bytes
        }
        const int h = lane & 1;
#pragma unroll
        for (int part = 0; part < 2; ++part) {
          const int srcl = part * 16 + (lane >> 1);
          const uint32_t lo0 = __shfl_sync(0xffffffffu, cw[0].x, srcl), lo1 = __shfl_sync(0xffffffffu, cw[0].y, srcl);
          const uint32_t lo2 = __shfl_sync(0xffffffffu, cw[1].x, srcl), lo3 = __shfl_sync(0xffffffffu, cw[1].y, srcl);
          const uint32_t hi0 = __shfl_sync(0xffffffffu, cw[2].x, srcl), hi1 = __shfl_sync(0xffffffffu, cw[2].y, srcl);
          const uint32_t hi2 = __shfl_sync(0xffffffffu, cw[3].x, srcl), hi3 = __shfl_sync(0xffffffffu, cw[3].y, srcl);
          const int piece = gi0 * 2 + part * 32 + lane;  // 16-B piece index within the row
          if (piece < nkb / 2)
            crow[piece] = h ? make_uint4(hi0, hi1, hi2, hi3) : make_uint4(lo0, lo1, lo2, lo3);
        }
      }
    }
  }
}

// return with the sources' offsets and my received-row count from the device plan
__global__ void __launch_bounds__(256) p2p_return_dev_kernel(const __nv_bfloat16* __restrict__ rows,
                                                             const int32_t* __restrict__ row_pos, int64_t n_cap,
                                                             int H, const PeerRows win,
                                                             const P2PPlan* __restrict__ plan) {
  const int lane = threadIdx.x & 31;
  const int R = win.R;
  const int64_t n = min(n_cap, (int64_t)plan->n_recv);
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int s = 0;
    while (s + 1 < R && plan->recv0[s + 1] <= i) ++s;
    const uint4* src = reinterpret_cast<const uint4*>(rows + (int64_t)row_pos[i] * H);
    uint4* dst = reinterpret_cast<uint4*>(win.base[s] + ((int64_t)plan->ret_row0[s] + (i - plan->recv0[s])) *
                                                            (2 * (int64_t)H));
    for (int c = lane; c < H / 8; c += 32) dst[c] = __ldg(src + c);
  }
}

// Rank-partial return: a W4A4 owner sums each (source s, token t)'s
// rows over ITS slots, in slot order (fma chain, fp32), rounds once to bf16 and stores
// ONE row into s's return window (row unit_base + me * ustride + t) instead of one row
// per slot; realb_combine_partial at the source adds it at t's first slot on this rank.
// Warp per unit (s, t); the unit table is reset to -1 behind itself for the next call.
// A W16A16 owner (device plan) does nothing here: its rows went back with the down GEMM.
__global__ void __launch_bounds__(256) p2p_partial_return_kernel(const __nv_bfloat16* __restrict__ rows,
                                                                 int32_t* __restrict__ units,
                                                                 const float* __restrict__ wts, int R,
                                                                 int64_t ustride, int k, int H, int me,
                                                                 const PeerRows win, int64_t unit_base,
                                                                 const P2PPlan* __restrict__ plan) {
  if (!plan->w4a4) return;
  const int lane = threadIdx.x & 31;
  const int64_t nunits = (int64_t)R * ustride;
  for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < nunits;
       u += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t gl = lane < k ? units[u * k + lane] : -1;
    if (!__any_sync(0xffffffffu, gl >= 0)) continue;
    int32_t g[8];
    float w[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      g[j] = __shfl_sync(0xffffffffu, gl, j);
      w[j] = (j < k && g[j] >= 0) ? wts[g[j]] : 0.f;
    }
    const int s = (int)(u / ustride);
    const int64_t t = u - (int64_t)s * ustride;
    uint4* dst = reinterpret_cast<uint4*>(win.base[s] + (unit_base + (int64_t)me * ustride + t) * (2 * (int64_t)H));
    for (int c = lane; c < H / 8; c += 32) {
      uint4 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < k && g[j] >= 0) v[j] = __ldg(reinterpret_cast<const uint4*>(rows + (int64_t)g[j] * H) + c);
      float p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (!(j < k && g[j] >= 0)) continue;
        const uint32_t vv[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          p[2 * i] = fmaf(w[j], __uint_as_float(vv[i] << 16), p[2 * i]);
          p[2 * i + 1] = fmaf(w[j], __uint_as_float(vv[i] & 0xFFFF0000u), p[2 * i + 1]);
        }
      }
      dst[c] = make_uint4(pack_bf16x2(p[0], p[1]), pack_bf16x2(p[2], p[3]), pack_bf16x2(p[4], p[5]),
                          pack_bf16x2(p[6], p[7]));
    }
    __syncwarp();
    if (lane < k) units[u * k + lane] = -1;
  }
}

// the return map of the fused down-GEMM + return (realb_grouped_gemm_*_scatter):
// grouped row row_pos[i] of received row i (source s, its j-th) -> (s << 25) | row
// of s's return window, the address p2p_return_dev_kernel would copy it to
__global__ void __launch_bounds__(256) p2p_return_map_kernel(const int32_t* __restrict__ row_pos, int64_t n_cap,
                                                             int R, const P2PPlan* __restrict__ plan,
                                                             int32_t* __restrict__ row_map) {
  const int64_t n = min(n_cap, (int64_t)plan->n_recv);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int s = 0;
    while (s + 1 < R && plan->recv0[s + 1] <= i) ++s;
    const int64_t row = (int64_t)plan->ret_row0[s] + (i - plan->recv0[s]);
    row_map[row_pos[i]] = (int32_t)(((int64_t)s << kScatterRowBits) | row);
  }
}

// row-major NVFP4 scales [rows][nkb] -> the MMA 128x4 layout, for the valid rows of the
// groups of one precision class (the layout's group list): one thread per (row, 4-scale word)
__global__ void __launch_bounds__(256) sf_rows_to_mma_kernel(const uint32_t* __restrict__ sf_rows,
                                                             const int32_t* __restrict__ layout, int E,
                                                             int prec, int nkb, uint8_t* __restrict__ sf_mma) {
  const int G = layout[1 + prec];
  const int32_t* glist = layout + LayoutView::off_glist(E, prec);
  const int wpr = nkb / 4;  // words per row
  for (int gi = blockIdx.y; gi < G; gi += gridDim.y) {
    const int e = glist[gi];
    const int64_t r0 = layout[LayoutView::off_row_start(E) + e];
    const int64_t n = (int64_t)layout[LayoutView::off_row_count(E) + e] * wpr;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t r = r0 + i / wpr;
      const int w = (int)(i % wpr);
      *reinterpret_cast<uint32_t*>(sf_mma + sf_mma_offset(r, (int64_t)w * 4, nkb)) = sf_rows[r * wpr + w];
    }
  }
}

}  // namespace realb

using namespace realb;

extern "C" int realb_sf_rows_to_mma(const uint8_t* d_sf_rows, int64_t rows_cap, int K, const int32_t* d_layout,
                                    int E, int prec, uint8_t* d_sf_mma, void* stream) {
  if (!d_sf_rows || !d_layout || !d_sf_mma || rows_cap <= 0 || K <= 0 || K % 64 || E < 1 || E > 256 ||
      (prec != REALB_PREC_W16A16 && prec != REALB_PREC_W4A4)) {
    set_error("realb_sf_rows_to_mma: bad arguments (K=%d E=%d)", K, E);
    return REALB_EINVAL;
  }
  const dim3 grid((unsigned)(num_sms() * 4 / (E < 8 ? E : 8) + 1), (unsigned)(E < 8 ? E : 8));
  sf_rows_to_mma_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(reinterpret_cast<const uint32_t*>(d_sf_rows),
                                                                d_layout, E, prec, K / 16, d_sf_mma);
  return check_launch("realb_sf_rows_to_mma");
}

extern "C" int realb_p2p_return_map(const int32_t* d_row_pos, int64_t n_cap, int R, const void* d_plan,
                                    int32_t* d_row_map, void* stream) {
  if (!d_row_pos || !d_plan || !d_row_map || n_cap < 0 || n_cap >= (1LL << kScatterRowBits) || R < 1 ||
      R > kMaxPeers || R > kScatterPeers) {
    set_error("realb_p2p_return_map: bad arguments (n_cap=%lld R=%d)", (long long)n_cap, R);
    return REALB_EINVAL;
  }
  if (n_cap == 0) return REALB_OK;
  int64_t grid = (n_cap + 255) / 256;
  if (grid > (int64_t)num_sms() * 8) grid = (int64_t)num_sms() * 8;
  p2p_return_map_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(
      d_row_pos, n_cap, R, reinterpret_cast<const P2PPlan*>(d_plan), d_row_map);
  return check_launch("realb_p2p_return_map");
}

extern "C" int realb_ipc_alloc(int64_t bytes, void** d_ptr, uint8_t* handle) {
  if (bytes <= 0 || !d_ptr || !handle) {
    set_error("realb_ipc_alloc: bad arguments");
    return REALB_EINVAL;
  }
  int rc = cuda_status(cudaMalloc(d_ptr, (size_t)bytes), "realb_ipc_alloc (cudaMalloc)");
  if (rc) return rc;
  rc = cuda_status(cudaMemset(*d_ptr, 0, (size_t)bytes), "realb_ipc_alloc (memset)");
  if (rc) return rc;
  cudaIpcMemHandle_t h;
  rc = cuda_status(cudaIpcGetMemHandle(&h, *d_ptr), "realb_ipc_alloc (cudaIpcGetMemHandle)");
  if (rc) return rc;
  memcpy(handle, &h, sizeof(h));
  return REALB_OK;
}

extern "C" int realb_ipc_open(const uint8_t* handle, void** d_ptr) {
  if (!handle || !d_ptr) {
    set_error("realb_ipc_open: bad arguments");
    return REALB_EINVAL;
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return cuda_status(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess),
                     "realb_ipc_open (cudaIpcOpenMemHandle)");
}

extern "C" int realb_ipc_close(void* d_ptr) {
  return cuda_status(cudaIpcCloseMemHandle(d_ptr), "realb_ipc_close");
}

extern "C" int realb_ipc_free(void* d_ptr) { return cuda_status(cudaFree(d_ptr), "realb_ipc_free"); }

extern "C" int realb_p2p_pack(const void* d_x, const int32_t* d_topk_idx, int T, int H, int E, int k,
                              const int32_t* d_layout, int nchunks, int R, const uint8_t* h_rank_fmt,
                              const int32_t* h_rank_row0, const uint64_t* h_rank_dst, int32_t* d_pair_pos,
                              int32_t* d_flag, void* stream) {
  if (T == 0 && nchunks == 0) return REALB_OK;
  if (!d_x || !d_topk_idx || !d_layout || !d_pair_pos || !h_rank_fmt || !h_rank_row0 || !h_rank_dst ||
      T < 0 || H <= 0 || H % 64 || E < 1 || E > 256 || k < 1 || k > 8 || R < 1 || R > kMaxPeers ||
      E % R || nchunks != (T + REALB_CHUNK_TOKENS - 1) / REALB_CHUNK_TOKENS) {
    set_error("realb_p2p_pack: bad arguments (T=%d H=%d E=%d k=%d R=%d)", T, H, E, k, R);
    return REALB_EINVAL;
  }
  PeerRows m{};
  m.R = R;
  m.El = E / R;
  for (int d = 0; d < R; ++d) {
    if (h_rank_fmt[d] > 1 || (h_rank_dst[d] & 15)) {
      set_error("realb_p2p_pack: peer %d: format must be 0/1 and addresses 16-byte aligned", d);
      return REALB_EINVAL;
    }
    m.base[d] = reinterpret_cast<uint8_t*>(h_rank_dst[d]);
    m.row0[d] = h_rank_row0[d];
    m.fmt[d] = h_rank_fmt[d];
  }
  int rc = ep_positions(d_topk_idx, T, E, k, d_layout, nchunks, d_pair_pos, stream);
  if (rc) return rc;
  const int64_t P = (int64_t)T * k;
  int64_t grid = (P + 7) / 8;
  if (grid > (int64_t)num_sms() * 16) grid = (int64_t)num_sms() * 16;
  p2p_pack_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const __nv_bfloat16*>(d_x), d_topk_idx, d_pair_pos, P, H, k, m, d_flag);
  return check_launch("realb_p2p_pack (rows)");
}

extern "C" int realb_p2p_return(const void* d_rows, const int32_t* d_row_pos, int64_t n, int H, int R,
                                const int32_t* h_recv_prefix, const uint64_t* h_src_dst, void* stream) {
  if (n < 0 || H <= 0 || H % 8 || R < 1 || R > kMaxPeers || !h_recv_prefix || !h_src_dst ||
      (n > 0 && (!d_rows || !d_row_pos))) {
    set_error("realb_p2p_return: bad arguments (n=%lld H=%d R=%d)", (long long)n, H, R);
    return REALB_EINVAL;
  }
  if (n == 0) return REALB_OK;
  PeerReturn m{};
  m.R = R;
  for (int s = 0; s < R; ++s) {
    if (h_src_dst[s] & 15) {
      set_error("realb_p2p_return: peer %d address not 16-byte aligned", s);
      return REALB_EINVAL;
    }
    m.base[s] = reinterpret_cast<__nv_bfloat16*>(h_src_dst[s]);
  }
  for (int s = 0; s <= R; ++s) m.recv0[s] = h_recv_prefix[s];
  int64_t grid = (n + 7) / 8;
  if (grid > (int64_t)num_sms() * 16) grid = (int64_t)num_sms() * 16;
  p2p_return_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const __nv_bfloat16*>(d_rows), d_row_pos, n, H, m);
  return check_launch("realb_p2p_return");
}

extern "C" int realb_p2p_signal(const uint64_t* h_peer_counters, int R, void* stream) {
  if (!h_peer_counters || R < 1 || R > kMaxPeers) {
    set_error("realb_p2p_signal: bad arguments (R=%d)", R);
    return REALB_EINVAL;
  }
  PeerCounters m{};
  m.R = R;
  for (int d = 0; d < R; ++d) m.ctr[d] = reinterpret_cast<uint32_t*>(h_peer_counters[d]);
  p2p_signal_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(m);
  return check_launch("realb_p2p_signal");
}

extern "C" int realb_p2p_wait(const uint32_t* d_counter, uint32_t target, int32_t* d_err, void* stream) {
  if (!d_counter) {
    set_error("realb_p2p_wait: bad arguments");
    return REALB_EINVAL;
  }
  p2p_wait_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(d_counter, target, d_err);
  return check_launch("realb_p2p_wait");
}

static int fill_bases(PeerRows& w, const uint64_t* h, int R, const char* fn) {
  if (!h || R < 1 || R > kMaxPeers) {
    set_error("%s: bad peer list (R=%d)", fn, R);
    return REALB_EINVAL;
  }
  for (int d = 0; d < R; ++d) {
    if (h[d] & 15) {
      set_error("%s: peer %d address not 16-byte aligned", fn, d);
      return REALB_EINVAL;
    }
    w.base[d] = reinterpret_cast<uint8_t*>(h[d]);
  }
  w.R = R;
  return REALB_OK;
}

extern "C" int64_t realb_p2p_plan_bytes(void) { return (int64_t)sizeof(P2PPlan); }

extern "C" int realb_p2p_publish(const int32_t* d_src, int n_words, int R, const uint64_t* h_peer_windows,
                                 int64_t offset_words, void* stream) {
  if (!d_src || n_words <= 0 || offset_words < 0) {
    set_error("realb_p2p_publish: bad arguments");
    return REALB_EINVAL;
  }
  PeerRows w{};
  int rc = fill_bases(w, h_peer_windows, R, "realb_p2p_publish");
  if (rc) return rc;
  p2p_publish_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(d_src, n_words, w, offset_words);
  return check_launch("realb_p2p_publish");
}

extern "C" int realb_p2p_plan_offsets(const int32_t* d_counts, int R, int E, int rank, int H, int fp4_dispatch,
                                      const uint8_t* d_prec, void* d_plan, int32_t* d_cnt_local,
                                      uint8_t* d_prec_local, void* stream) {
  if (!d_counts || !d_prec || !d_plan || !d_cnt_local || !d_prec_local || R < 1 || R > kMaxPeers ||
      E < 1 || E % R || rank < 0 || rank >= R || H <= 0) {
    set_error("realb_p2p_plan_offsets: bad arguments (R=%d E=%d rank=%d)", R, E, rank);
    return REALB_EINVAL;
  }
  p2p_plan_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(d_counts, R, E, rank, H, fp4_dispatch, d_prec,
                                                       reinterpret_cast<P2PPlan*>(d_plan), d_cnt_local,
                                                       d_prec_local);
  return check_launch("realb_p2p_plan_offsets");
}

extern "C" int realb_p2p_pack_dev(const void* d_x, const int32_t* d_topk_idx, int T, int H, int E, int k,
                                  const int32_t* d_layout, int nchunks, int R, const uint64_t* h_peer_recv,
                                  const void* d_plan, int32_t* d_pair_pos, int32_t* d_flag, void* stream) {
  if (T == 0 && nchunks == 0) return REALB_OK;
  if (!d_x || !d_topk_idx || !d_layout || !d_plan || !d_pair_pos || T < 0 || H <= 0 || H % 64 || E < 1 ||
      E > 256 || k < 1 || k > 8 || E % R || nchunks != (T + REALB_CHUNK_TOKENS - 1) / REALB_CHUNK_TOKENS) {
    set_error("realb_p2p_pack_dev: bad arguments (T=%d H=%d E=%d k=%d R=%d)", T, H, E, k, R);
    return REALB_EINVAL;
  }
  PeerRows w{};
  int rc = fill_bases(w, h_peer_recv, R, "realb_p2p_pack_dev");
  if (rc) return rc;
  w.El = E / R;
  rc = ep_positions(d_topk_idx, T, E, k, d_layout, nchunks, d_pair_pos, stream);
  if (rc) return rc;
  const int64_t P = (int64_t)T * k;
  int64_t grid = (P + 7) / 8;
  if (grid > (int64_t)num_sms() * 16) grid = (int64_t)num_sms() * 16;
  p2p_pack_dev_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const __nv_bfloat16*>(d_x), d_topk_idx, d_pair_pos, P, H, k, w,
      reinterpret_cast<const P2PPlan*>(d_plan), d_flag);
  return check_launch("realb_p2p_pack_dev");
}

extern "C" int realb_p2p_return_dev(const void* d_rows, const int32_t* d_row_pos, int64_t n_cap, int H, int R,
                                    const uint64_t* h_peer_ret, const void* d_plan, void* stream) {
  if (!d_rows || !d_row_pos || !d_plan || n_cap < 0 || H <= 0 || H % 8) {
    set_error("realb_p2p_return_dev: bad arguments");
    return REALB_EINVAL;
  }
  PeerRows w{};
  int rc = fill_bases(w, h_peer_ret, R, "realb_p2p_return_dev");
  if (rc || n_cap == 0) return rc;
  int64_t grid = (n_cap + 7) / 8;
  if (grid > (int64_t)num_sms() * 16) grid = (int64_t)num_sms() * 16;
  p2p_return_dev_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const __nv_bfloat16*>(d_rows), d_row_pos, n_cap, H, w,
      reinterpret_cast<const P2PPlan*>(d_plan));
  return check_launch("realb_p2p_return_dev");
}

extern "C" int realb_p2p_wait_next(uint32_t* d_expected, uint32_t inc, const uint32_t* d_counter,
                                   int32_t* d_err, void* stream) {
  if (!d_expected || !d_counter) {
    set_error("realb_p2p_wait_next: bad arguments");
    return REALB_EINVAL;
  }
  p2p_wait_next_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(d_expected, inc, d_counter, d_err);
  return check_launch("realb_p2p_wait_next");
}

// [sizeof(P2PPlan), offsetof n_recv, w4a4, gate_bf16, gate_packed]
extern "C" int realb_p2p_plan_layout(int64_t* out5) {
  if (!out5) return REALB_EINVAL;
  out5[0] = (int64_t)sizeof(P2PPlan);
  out5[1] = (int64_t)offsetof(P2PPlan, n_recv);
  out5[2] = (int64_t)offsetof(P2PPlan, w4a4);
  out5[3] = (int64_t)offsetof(P2PPlan, gate_bf16);
  out5[4] = (int64_t)offsetof(P2PPlan, gate_packed);
  return REALB_OK;
}

static int pack_direct_impl(const void* d_x, const int32_t* d_topk_idx, int T, int H, int E, int k,
                            const int32_t* d_layout, int nchunks, int R, const uint64_t* h_peer_a,
                            const uint64_t* h_peer_codes, const uint64_t* h_peer_sf, const void* d_plan,
                            int32_t* d_pair_pos, int32_t* d_flag, const float* d_topk_w, const uint64_t* h_peer_units,
                            const uint64_t* h_peer_wts, int me, int64_t ustride, void* stream);

extern "C" int realb_p2p_pack_direct(const void* d_x, const int32_t* d_topk_idx, int T, int H, int E, int k,
                                     const int32_t* d_layout, int nchunks, int R, const uint64_t* h_peer_a,
                                     const uint64_t* h_peer_codes, const uint64_t* h_peer_sf,
                                     const void* d_plan, int32_t* d_pair_pos, int32_t* d_flag, void* stream) {
  return pack_direct_impl(d_x, d_topk_idx, T, H, E, k, d_layout, nchunks, R, h_peer_a, h_peer_codes, h_peer_sf,
                          d_plan, d_pair_pos, d_flag, nullptr, nullptr, nullptr, 0, 0, stream);
}

extern "C" int realb_p2p_pack_direct_partial(const void* d_x, const int32_t* d_topk_idx, const float* d_topk_w,
                                             int T, int H, int E, int k, const int32_t* d_layout, int nchunks, int R,
                                             const uint64_t* h_peer_a, const uint64_t* h_peer_codes,
                                             const uint64_t* h_peer_sf, const uint64_t* h_peer_units,
                                             const uint64_t* h_peer_wts, int me, int64_t ustride, const void* d_plan,
                                             int32_t* d_pair_pos, int32_t* d_flag, void* stream) {
  if (!d_topk_w || !h_peer_units || !h_peer_wts || me < 0 || me >= R || ustride < T) {
    set_error("realb_p2p_pack_direct_partial: bad arguments (me=%d R=%d ustride=%lld T=%d)", me, R,
              (long long)ustride, T);
    return REALB_EINVAL;
  }
  return pack_direct_impl(d_x, d_topk_idx, T, H, E, k, d_layout, nchunks, R, h_peer_a, h_peer_codes, h_peer_sf,
                          d_plan, d_pair_pos, d_flag, d_topk_w, h_peer_units, h_peer_wts, me, ustride, stream);
}

extern "C" int realb_p2p_partial_return(const void* d_rows, int32_t* d_units, const float* d_wts, int R,
                                        int64_t ustride, int k, int H, int me, const uint64_t* h_ret_bases,
                                        int64_t unit_base, const void* d_plan, void* stream) {
  if (!d_rows || !d_units || !d_wts || !h_ret_bases || !d_plan || R < 1 || R > kMaxPeers || me < 0 || me >= R ||
      ustride < 1 || k < 1 || k > 8 || H <= 0 || H % 8 || unit_base < 0) {
    set_error("realb_p2p_partial_return: bad arguments (R=%d me=%d k=%d H=%d)", R, me, k, H);
    return REALB_EINVAL;
  }
  PeerRows win{};
  win.R = R;
  for (int s = 0; s < R; ++s) {
    if (h_ret_bases[s] & 15) {
      set_error("realb_p2p_partial_return: return window %d misaligned", s);
      return REALB_EINVAL;
    }
    win.base[s] = reinterpret_cast<uint8_t*>(h_ret_bases[s]);
  }
  int64_t grid = ((int64_t)R * ustride + 7) / 8;
  if (grid > (int64_t)num_sms() * 16) grid = (int64_t)num_sms() * 16;
  p2p_partial_return_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const __nv_bfloat16*>(d_rows), d_units, d_wts, R, ustride, k, H, me, win, unit_base,
      reinterpret_cast<const P2PPlan*>(d_plan));
  return check_launch("realb_p2p_partial_return");
}

static int pack_direct_impl(const void* d_x, const int32_t* d_topk_idx, int T, int H, int E, int k,
                            const int32_t* d_layout, int nchunks, int R, const uint64_t* h_peer_a,
                            const uint64_t* h_peer_codes, const uint64_t* h_peer_sf, const void* d_plan,
                            int32_t* d_pair_pos, int32_t* d_flag, const float* d_topk_w, const uint64_t* h_peer_units,
                            const uint64_t* h_peer_wts, int me, int64_t ustride, void* stream) {
  if (T == 0 && nchunks == 0) return REALB_OK;
  if (!d_x || !d_topk_idx || !d_layout || !d_plan || !d_pair_pos || !h_peer_a || !h_peer_codes || !h_peer_sf ||
      T < 0 || H <= 0 || H % 64 || E < 1 || E > 256 || k < 1 || k > 8 || R < 1 || R > kMaxPeers || E % R ||
      nchunks != (T + REALB_CHUNK_TOKENS - 1) / REALB_CHUNK_TOKENS) {
    set_error("realb_p2p_pack_direct: bad arguments (T=%d H=%d E=%d k=%d R=%d)", T, H, E, k, R);
    return REALB_EINVAL;
  }
  PeerOperands o{};
  o.R = R;
  o.El = E / R;
  for (int d = 0; d < R; ++d) {
    if ((h_peer_a[d] | h_peer_codes[d]) & 15 || h_peer_sf[d] & 15) {
      set_error("realb_p2p_pack_direct: peer %d operand addresses misaligned", d);
      return REALB_EINVAL;
    }
    o.a[d] = reinterpret_cast<__nv_bfloat16*>(h_peer_a[d]);
    o.codes[d] = reinterpret_cast<uint8_t*>(h_peer_codes[d]);
    o.sf[d] = reinterpret_cast<uint8_t*>(h_peer_sf[d]);
    if (d_topk_w) {
      o.units[d] = reinterpret_cast<int32_t*>(h_peer_units[d]);
      o.wts[d] = reinterpret_cast<float*>(h_peer_wts[d]);
    }
  }
  o.topk_w = d_topk_w;
  o.me = me;
  o.ustride = ustride;
  int rc = ep_positions(d_topk_idx, T, E, k, d_layout, nchunks, d_pair_pos, stream);
  if (rc) return rc;
  const int64_t P = (int64_t)T * k;
  int64_t grid = (P + 7) / 8;
  if (grid > (int64_t)num_sms() * 16) grid = (int64_t)num_sms() * 16;
  p2p_pack_direct_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const __nv_bfloat16*>(d_x), d_topk_idx, d_pair_pos, d_layout + 8, P, H, k, o,
      reinterpret_cast<const P2PPlan*>(d_plan), d_flag);
  return check_launch("realb_p2p_pack_direct");
}
