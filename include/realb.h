/*
 * realb.h — C-ABI of the B200-native ReaLB MoE-layer hot path (sm_100a).
 *
 * Reference: arXiv 2604.19503 ("ReaLB"); reference package `moesim`
 * (/root/reference/pkg/src/moesim). The reference is pure Python with no FFI,
 * so every entry point below replaces a Python function or an analytic cost
 * formula on the MoE-layer path; the replaced symbol is cited per function.
 *
 * Conventions (all functions):
 *   - Plain pointers and sizes only. Every pointer argument named `d_*` is a
 *     DEVICE pointer owned by the caller; nothing here allocates or frees
 *     device memory (TMEM inside kernels excepted).
 *   - `stream` is a cudaStream_t passed as void*. Every call is stream-ordered,
 *     re-entrant, performs no host synchronisation and keeps no hidden state.
 *   - Return value: REALB_OK (0) or a negative status. A human-readable
 *     message for the last failure on the calling thread is available from
 *     realb_last_error(). No C++ exception crosses this boundary.
 *   - Data errors found on the device (non-finite quantiser input, mirroring
 *     moesim.fp4.QuantizationDomainError, fp4.py:22) are reported through a
 *     caller-provided int32 device flag, checked lazily by the caller.
 */
#ifndef REALB_H_
#define REALB_H_

#include <stdint.h>

#if defined(__GNUC__)
#define REALB_API __attribute__((visibility("default")))
#else
#define REALB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define REALB_ABI_VERSION 1

#define REALB_OK 0
#define REALB_EINVAL (-1)      /* bad argument (shape, alignment, range)      */
#define REALB_ECUDA (-2)       /* CUDA runtime / launch failure               */
#define REALB_EUNSUPPORTED (-3) /* shape outside what the kernels implement   */

/* element types for `dtype` arguments */
#define REALB_DT_BF16 0
#define REALB_DT_F32 1
#define REALB_DT_F64 2

/* scale-factor layouts written by the quantisers */
#define REALB_SF_FLAT 0    /* [rows][cols/16] row-major: moesim's (n,) order   */
#define REALB_SF_MMA128x4 1 /* tcgen05 block-scale layout: 128-row x 4-SF
                               512-byte atoms, byte = (r%32)*16+((r/32)%4)*4+k%4,
                               atoms ordered (r/128, k/4) row-major            */

/* router scoring functions (D1 contract) */
#define REALB_SCORE_SOFTMAX_RENORM 0  /* Qwen3-VL-MoE: softmax, top-k, renorm   */
#define REALB_SCORE_SIGMOID_RENORM 1  /* Kimi-VL (DeepSeek-V3 family): sigmoid,
                                         top-k, renorm, x routed_scaling       */
#define REALB_SCORE_SOFTMAX_CLAMPNORM 2 /* ERNIE-4.5-VL: softmax, top-k,
                                           / max(sum, norm_min)                */

/* token chunk of the router / stats / dispatch kernels: chunk_counts hold one
 * [E][2] histogram per REALB_CHUNK_TOKENS consecutive tokens */
#define REALB_CHUNK_TOKENS 64

/* precision codes: values of moesim.core.Precision (core.py:9-11) */
#define REALB_PREC_W16A16 0
#define REALB_PREC_W4A4 1

REALB_API int realb_abi_version(void);
REALB_API const char* realb_last_error(void);
/* number of SMs of the current device, or <0 */
REALB_API int realb_num_sms(void);

/* ------------------------------------------------------------------------ *
 * K3 / K4 — NVFP4 block quantiser.
 * Replaces moesim.fp4.quantize_blocks (fp4.py:173-227), bit-exact, and its
 * scalar twin quantize_block (fp4.py:108-122). Blocks are 16 consecutive
 * elements along a row of x[rows][cols] (cols % 16 == 0).
 *   d_codes : [rows][cols/2] bytes, element 2i in the low nibble (= pack_block
 *             order, fp4.py:246-252, and the tcgen05 packed-E2M1 order)
 *   d_sf    : E4M3 scale bytes, layout `sf_layout`; REALB_SF_MMA128x4 needs
 *             rows % 128 == 0 and cols % 64 == 0.
 *   d_nonfinite_flag : set to 1 when any element is non-finite
 *             (QuantizationDomainError); may be NULL.
 *   max_ctas: cap on CTAs (0 = auto) so the quantiser can run CTA-limited on
 *             a side stream next to NCCL.
 * ------------------------------------------------------------------------ */
REALB_API int realb_quantize_nvfp4(const void* d_x, int dtype, int64_t rows, int64_t cols,
                         uint8_t* d_codes, uint8_t* d_sf, int sf_layout,
                         int32_t* d_nonfinite_flag, int max_ctas, void* stream);

/* K3 driven by the device-side plan: quantise the bf16 weight rows of every
 * expert whose d_expert_prec code is W4A4 (rows of expert e are
 * [e*rows_per_expert, (e+1)*rows_per_expert); rows_per_expert % 128 == 0),
 * MMA scale layout, other experts untouched. */
REALB_API int realb_quantize_experts_nvfp4(const void* d_w, int E, int64_t rows_per_expert,
                                           int64_t cols, const uint8_t* d_expert_prec,
                                           uint8_t* d_codes, uint8_t* d_sf,
                                           int32_t* d_nonfinite_flag, int max_ctas,
                                           void* stream);

/* K3 over two weight matrices of the same experts in ONE launch (an expert's
 * gate_up [E*rows0_per_expert, cols0] and down [E*rows1_per_expert, cols1]):
 * the W4A4 experts' tiles of both matrices form one contiguous range split over
 * a persistent grid, so the pair pays one ramp-up and one tail. Same rule, codes
 * and MMA scale layout as realb_quantize_experts_nvfp4 on each matrix
 * (replaces fp4.py:173-227 per rank-layer). */
REALB_API int realb_quantize_experts2_nvfp4(const void* d_w0, int64_t rows0_per_expert, int64_t cols0,
                                            uint8_t* d_codes0, uint8_t* d_sf0, const void* d_w1,
                                            int64_t rows1_per_expert, int64_t cols1, uint8_t* d_codes1,
                                            uint8_t* d_sf1, int E, const uint8_t* d_expert_prec,
                                            int32_t* d_nonfinite_flag, int max_ctas, void* stream);

/* Q5 — quantize_tensor + ErrorSummary (fp4.py:130-170) on the device.
 *   d_x        : n flat values (dtype REALB_DT_BF16 / F32 / F64), n > 0; the
 *                last block is zero-padded
 *   d_records  : ceil(n/16) x 9 bytes, each the FP4REF01 block record of
 *                pack_block (fp4.py:246-252): 8 code bytes (element 2i in the low
 *                nibble) + the E4M3 scale byte; i.e. the body of write_blocks
 *   d_block_max_rel : fp64 [ceil(n/16)] max over unpadded x != 0 of |x - d|/|x|
 *                (bit-exact with the reference), or NULL
 *   d_sums     : fp64 [2], ACCUMULATED (zero it first): sum (x - d)^2 and sum x^2
 *                over the unpadded elements -> rmse = sqrt(s0 / n),
 *                relative_rmse = sqrt(s0 / s1) (s1 > 0), or NULL
 *   d_nonfinite_flag : set on Inf/NaN input (QuantizationDomainError), or NULL
 * The block rule runs in fp64 (the reference's arithmetic) for every dtype. */
REALB_API int realb_quantize_tensor_nvfp4(const void* d_x, int dtype, int64_t n, uint8_t* d_records,
                                          double* d_block_max_rel, double* d_sums,
                                          int32_t* d_nonfinite_flag, void* stream);

/* Q4/Q6 decode — dequantize_blocks (fp4.py:230-243): nblocks blocks of packed
 * codes (8 bytes, element 2i in the low nibble) and flat E4M3 scale bytes ->
 * 16 values each, code magnitude x scale (exact), dtype_out REALB_DT_F32 / F64. */
REALB_API int realb_dequantize_blocks(const uint8_t* d_codes, const uint8_t* d_sf, int64_t nblocks,
                                      int dtype_out, void* d_out, void* stream);

/* ------------------------------------------------------------------------ *
 * K1 + K2 — router / top-k / modality statistics (new: the reference
 * synthesises routing, tracegen.py:141-185; the counts it produces feed
 * aggregate_rank_loads, core.py:106-130).
 *   d_x        : bf16 [T][H] hidden states, H % 64 == 0
 *   d_wg       : bf16 [E][H] router weight
 *   d_bias     : fp32 [E] selection bias (e_score_correction_bias) or NULL
 *   d_modality : uint8 [T], 1 = vision token, 0 = text
 *   d_logits   : fp32 [T][E] logits written by the kernel (the D1 contract
 *                selects on exactly these values)
 *   d_topk_idx : int32 [T][k], experts in selection order (score desc, ties
 *                to the lowest expert id)
 *   d_topk_w   : fp32 [T][k] routing weights
 *   d_chunk_counts : int32 [ceil(T/64)][E][2] per-64-token-chunk
 *                (vision, text) pair counts (deterministic, atomic-free)
 * E <= 256, 1 <= k <= 16.
 * ------------------------------------------------------------------------ */
REALB_API int realb_router_topk_stats(const void* d_x, const void* d_wg, const float* d_bias,
                            const uint8_t* d_modality, int T, int H, int E, int k,
                            int scoring, float routed_scaling, float norm_min,
                            float* d_logits, int32_t* d_topk_idx, float* d_topk_w,
                            int32_t* d_chunk_counts, void* stream);

/* ------------------------------------------------------------------------ *
 * Grouped-row layout ("align"): from the per-chunk counts, build the
 * expert-sorted, 128-row-padded row space the grouped GEMMs run on.
 * d_layout is an int32 workspace of realb_layout_words(E, nchunks) words:
 *   [0] padded rows used   [1] #W16A16 groups   [2] #W4A4 groups
 *   [8 + e]          row_start[e]    [8 + E + e]   row_count[e]
 *   [8 + 2E + e]     expert (v,t) totals are in d_expert_vt instead
 *   glist/prefix per precision and per-chunk offsets follow (internal).
 * d_expert_prec : uint8 [E] REALB_PREC_* per expert (the precision plan
 *                 expanded through the placement, balancers.py:113-118).
 * d_expert_vt   : int32 [E][2] global (vision, text) pair counts (output).
 * ------------------------------------------------------------------------ */
REALB_API int64_t realb_layout_words(int E, int nchunks);
REALB_API int realb_moe_align(const int32_t* d_chunk_counts, int nchunks, int E,
                              const uint8_t* d_expert_prec, int row_align, int32_t* d_layout,
                              int32_t* d_expert_vt, void* stream);
/* row_align: 128 for the GEMM row space; 1 for an unpadded, expert-sorted
 * (hence destination-rank-contiguous) EP send buffer. */

/* realb_moe_align with the P1 policy evaluated ON THE DEVICE (no host sync):
 * expert totals -> per-rank (v,t) over the contiguous placement of R ranks
 * (place_experts_static, core.py:92-97; aggregate_rank_loads, core.py:106-130)
 * -> plan_for(strategy) (balancers.py:202-219; plan_realb :89-122 with the
 * reference's fp64 operation order) -> d_expert_prec (output), then the layout.
 *   strategy   : 0 baseline, 1 fp4all, 2 realb / realb-seq
 *   d_plan_out : int32 [3 + R] or NULL: [0] active, [1] #W4A4 ranks, [2] R,
 *                [3 + r] flags (bit0 hot, bit1 vision-heavy, bit2 W4A4) */
REALB_API int realb_moe_align_plan(const int32_t* d_chunk_counts, int nchunks, int E, int R,
                                   int strategy, double capacity_factor,
                                   double modality_threshold, int64_t global_batch_threshold,
                                   int modality_isolated, uint8_t* d_expert_prec,
                                   int32_t* d_plan_out, int32_t* d_layout,
                                   int32_t* d_expert_vt, void* stream);

/* Local dispatch: scatter token rows into the grouped row space.
 *   d_pair_pos : int32 [T][k] output row of every (token, slot) pair
 *   d_a_bf16   : bf16 [rows_cap][H] rows of W16A16 experts (others untouched)
 *   d_a_codes / d_a_sf : W4A4 experts' rows, quantised on the fly with the
 *                reference block rule (fp4.py:108-122) into MMA layout;
 *                may be NULL when no expert is W4A4.
 * Padding rows of every group are zero-filled. */
REALB_API int realb_dispatch_permute(const void* d_x, const int32_t* d_topk_idx, int T, int H,
                           int E, int k, const uint8_t* d_expert_prec,
                           const int32_t* d_layout, int nchunks, int64_t rows_cap,
                           int32_t* d_pair_pos, void* d_a_bf16, uint8_t* d_a_codes,
                           uint8_t* d_a_sf, int32_t* d_nonfinite_flag, void* stream);

/* realb_dispatch_permute without the W16A16 row copy: positions, plus the
 * inverse map d_row_src [rows_cap] (grouped row -> token; entries of padding
 * rows are not written) for realb_grouped_gemm_bf16_gather. Rows of W4A4 experts
 * are still quantised into d_a_codes / d_a_sf (both NULL: none is W4A4). */
REALB_API int realb_dispatch_index(const void* d_x, const int32_t* d_topk_idx, int T, int H, int E, int k,
                                   const uint8_t* d_expert_prec, const int32_t* d_layout, int nchunks,
                                   int64_t rows_cap, int32_t* d_pair_pos, int32_t* d_row_src,
                                   uint8_t* d_a_codes, uint8_t* d_a_sf, int32_t* d_nonfinite_flag,
                                   void* stream);

/* The row-movement half of realb_dispatch_permute, exposed for the EP
 * receive side: row p of x (token p / k) goes to position d_pos[p] of the
 * grouped space as bf16 or, when d_prec[d_expert[p]] is W4A4, as NVFP4 (K4). */
REALB_API int realb_gather_rows(const void* d_x, const int32_t* d_expert, const int32_t* d_pos,
                                int64_t P, int H, int k, const uint8_t* d_prec, void* d_a_bf16,
                                uint8_t* d_a_codes, uint8_t* d_a_sf, int32_t* d_nonfinite_flag,
                                const int32_t* d_count, const int32_t* d_gate, void* stream);
/* d_count (nullable): device row count; P is then an upper bound (capacity launch).
 * d_gate (nullable): the kernel does nothing when *d_gate == 0 (a device-side
 * choice between this gather and realb_gather_rows_nvfp4_packed). */

/* EP receive side (C2): rows arrive source-major, per source ordered by local
 * expert (senders pack by global expert id). From the [R][El] count matrix
 * build the local grouped layout (as realb_moe_align, El experts) and, for
 * every received row, its local expert and grouped position.
 *   n_recv : received rows, or an upper bound (the true count comes from d_cnt)
 *   d_base : int32 workspace [2*R*El + 2] */
REALB_API int realb_ep_regroup(const int32_t* d_cnt, int R, int El, const uint8_t* d_prec_local,
                               int64_t n_recv, int32_t* d_layout, int32_t* d_base,
                               int32_t* d_row_expert, int32_t* d_row_pos, void* stream);

/* EP send side (C2 pack), with the NVFP4 activation dispatch of SURVEY.md
 * §8f-1: expert-sorted positions of every (token, slot) pair (as
 * realb_dispatch_permute over d_layout built with row_align 1), then each row is
 * written into the send buffer segment of its destination rank d = e/(E/R):
 *   byte offset h_rank_byte0[d] + (pos - h_rank_row0[d]) * row_bytes(d)
 *   h_rank_fmt[d] = 0: bf16 row, row_bytes = 2H
 *   h_rank_fmt[d] = 1: NVFP4 row quantised with the reference block rule along H
 *                      (fp4.py:173-227, the K4 rule), packed as [H/2 code bytes]
 *                      [H/16 E4M3 scale bytes], row_bytes = H/2 + H/16
 * h_* are HOST arrays of R entries (read during the call; the plan and the
 * split sizes are host-known after the C1 count exchange); byte offsets 16-byte
 * aligned. R <= 64. Replaces the dispatch term of costmodel.dispatch_latency
 * (costmodel.py:71-76) — bytes to W4A4 ranks drop 3.6x. */
REALB_API int realb_ep_pack(const void* d_x, const int32_t* d_topk_idx, int T, int H, int E, int k,
                            const int32_t* d_layout, int nchunks, int R, const uint8_t* h_rank_fmt,
                            const int32_t* h_rank_row0, const int64_t* h_rank_byte0,
                            int32_t* d_pair_pos, uint8_t* d_send, int32_t* d_nonfinite_flag,
                            void* stream);

/* EP receive side of the NVFP4 dispatch: n packed rows (format of
 * realb_ep_pack, fmt 1) -> codes at row d_pos[i] of d_a_codes [rows][H/2] and
 * scales into the REALB_SF_MMA128x4 layout of d_a_sf. H % 256 == 0. */
REALB_API int realb_gather_rows_nvfp4_packed(const uint8_t* d_src, const int32_t* d_pos, int64_t n,
                                             int H, uint8_t* d_a_codes, uint8_t* d_a_sf,
                                             const int32_t* d_count, const int32_t* d_gate,
                                             void* stream);

/* ------------------------------------------------------------------------ *
 * Peer-memory EP transport (C2 / C3 without a collective library).
 * Windows: realb_ipc_alloc cudaMallocs a zeroed device buffer and returns its
 * 64-byte CUDA IPC handle; peers map it with realb_ipc_open (NVLink peer memory
 * across GPUs of a node; plain device memory for processes sharing one GPU).
 * These four are the only calls that allocate / map device memory: the
 * communication windows (like a collective library's own buffers).
 * realb_p2p_pack   : realb_ep_pack whose destination for peer d is the device
 *                    address h_rank_dst[d] (in d's receive window) instead of a
 *                    local send buffer; same row formats (bf16 / packed NVFP4).
 * realb_p2p_return : received row i (source-major: source s owns rows
 *                    [h_recv_prefix[s], h_recv_prefix[s+1])) copied from my
 *                    grouped row d_row_pos[i] to h_src_dst[s] + (i - prefix[s])
 *                    rows in source s's return window (replaces C3 + index_rows).
 * realb_p2p_signal : after this stream's earlier writes are visible system-wide,
 *                    atomically add 1 to each of the R peer counters.
 * realb_p2p_wait   : stream waits until *d_counter (acquire, system scope)
 *                    reaches target (modular uint32 compare); after 10 s without
 *                    it, sets *d_err (if non-NULL) and gives up instead of hanging.
 * h_* are host arrays (read during the call); addresses 16-byte aligned.
 * ------------------------------------------------------------------------ */
REALB_API int realb_ipc_alloc(int64_t bytes, void** d_ptr, uint8_t* handle64);
REALB_API int realb_ipc_open(const uint8_t* handle64, void** d_ptr);
REALB_API int realb_ipc_close(void* d_ptr);
REALB_API int realb_ipc_free(void* d_ptr);
REALB_API int realb_p2p_pack(const void* d_x, const int32_t* d_topk_idx, int T, int H, int E, int k,
                             const int32_t* d_layout, int nchunks, int R, const uint8_t* h_rank_fmt,
                             const int32_t* h_rank_row0, const uint64_t* h_rank_dst,
                             int32_t* d_pair_pos, int32_t* d_nonfinite_flag, void* stream);
REALB_API int realb_p2p_return(const void* d_rows, const int32_t* d_row_pos, int64_t n, int H, int R,
                               const int32_t* h_recv_prefix, const uint64_t* h_src_dst, void* stream);
REALB_API int realb_p2p_signal(const uint64_t* h_peer_counters, int R, void* stream);
REALB_API int realb_p2p_wait(const uint32_t* d_counter, uint32_t target, int32_t* d_err, void* stream);

/* Host-sync-free form (the EP layer becomes CUDA-graph capturable):
 * realb_p2p_publish      : copy n_words int32 (my [E][2] counts) into every peer
 *                          window h_peer_windows[d] at word offset offset_words (C1).
 * realb_p2p_plan_offsets : from the gathered counts [R][E][2] and the device plan's
 *                          expert precisions, write the P2P plan record (d_plan,
 *                          realb_p2p_plan_bytes() bytes: per-peer send offsets and
 *                          row formats, receive prefix, return offsets, my received
 *                          row count and gather gates), my [R][El] receive counts
 *                          and my experts' precisions.
 * realb_p2p_pack_dev / realb_p2p_return_dev : realb_p2p_pack / realb_p2p_return
 *                          with every offset, format and count read from d_plan;
 *                          h_peer_recv / h_peer_ret are the peers' window bases. */
REALB_API int64_t realb_p2p_plan_bytes(void);
/* [size, offsetof(n_recv), offsetof(w4a4), offsetof(gate_bf16), offsetof(gate_packed)] of the
 * plan record, so callers can point realb_gather_rows' d_count / d_gate into it. */
REALB_API int realb_p2p_plan_layout(int64_t* out5);
/* graph-safe wait: *d_expected += inc, then wait until *d_counter reaches it */
REALB_API int realb_p2p_wait_next(uint32_t* d_expected, uint32_t inc, const uint32_t* d_counter,
                                  int32_t* d_err, void* stream);
REALB_API int realb_p2p_publish(const int32_t* d_src, int n_words, int R, const uint64_t* h_peer_windows,
                                int64_t offset_words, void* stream);
REALB_API int realb_p2p_plan_offsets(const int32_t* d_counts, int R, int E, int rank, int H,
                                     int fp4_dispatch, const uint8_t* d_prec, void* d_plan,
                                     int32_t* d_cnt_local, uint8_t* d_prec_local, void* stream);
REALB_API int realb_p2p_pack_dev(const void* d_x, const int32_t* d_topk_idx, int T, int H, int E, int k,
                                 const int32_t* d_layout, int nchunks, int R,
                                 const uint64_t* h_peer_recv, const void* d_plan, int32_t* d_pair_pos,
                                 int32_t* d_nonfinite_flag, void* stream);
REALB_API int realb_p2p_return_dev(const void* d_rows, const int32_t* d_row_pos, int64_t n_cap, int H,
                                   int R, const uint64_t* h_peer_ret, const void* d_plan, void* stream);

/* The return map of the fused down-GEMM + return: for every received row i
 * (n_cap bounds the device-plan count), d_row_map[d_row_pos[i]] = (s << 25) | j,
 * j = the row of source s's return window realb_p2p_return_dev would write. */
REALB_API int realb_p2p_return_map(const int32_t* d_row_pos, int64_t n_cap, int R, const void* d_plan,
                                   int32_t* d_row_map, void* stream);
/* Direct dispatch: each (token, slot) row goes straight to its destination's GEMM
 * operand at its final grouped row (realb_ep_regroup's layout, derived from the
 * gathered counts in d_plan): bf16 into h_peer_a[d] for a W16A16 destination,
 * NVFP4 codes into h_peer_codes[d] (the K4 rule) for a W4A4 one, with its scales
 * ROW-MAJOR ([rows_cap][H/16] bytes) into h_peer_sf[d]; the W4A4 receiver turns
 * those into the MMA layout with realb_sf_rows_to_mma. Every warp store is one
 * contiguous span (wide peer-memory writes). d_layout: my row_align-1 send layout
 * (expert starts). The receiver runs no row gather. */
REALB_API int realb_p2p_pack_direct(const void* d_x, const int32_t* d_topk_idx, int T, int H, int E, int k,
                                    const int32_t* d_layout, int nchunks, int R, const uint64_t* h_peer_a,
                                    const uint64_t* h_peer_codes, const uint64_t* h_peer_sf,
                                    const void* d_plan, int32_t* d_pair_pos, int32_t* d_nonfinite_flag,
                                    void* stream);

/* Rank-partial return. realb_p2p_pack_direct_partial is
 * realb_p2p_pack_direct plus, for every row bound for a W4A4 owner d (device
 * plan), the grouped row g in d's unit table h_peer_units[d] (int32
 * [R][ustride][k], entry (me, t, j); -1 = no row) and the routing weight
 * d_topk_w[t][j] in h_peer_wts[d][g] (fp32 [rows_cap]). After its down GEMM has
 * stored its W4A4 rows locally (d_rows, grouped order), a W4A4 owner calls
 * realb_p2p_partial_return: per (source s, token t) with rows here, the fma chain
 * over t's slots in order, rounded once to bf16, goes to row unit_base + me *
 * ustride + t of s's return window (h_ret_bases[s]); the unit table is reset to
 * -1 behind it. A W16A16 owner's call is a no-op. The source then combines with
 * realb_combine_partial(unit_base, ustride). */
REALB_API int realb_p2p_pack_direct_partial(const void* d_x, const int32_t* d_topk_idx, const float* d_topk_w,
                                            int T, int H, int E, int k, const int32_t* d_layout, int nchunks,
                                            int R, const uint64_t* h_peer_a, const uint64_t* h_peer_codes,
                                            const uint64_t* h_peer_sf, const uint64_t* h_peer_units,
                                            const uint64_t* h_peer_wts, int me, int64_t ustride,
                                            const void* d_plan, int32_t* d_pair_pos, int32_t* d_nonfinite_flag,
                                            void* stream);
REALB_API int realb_p2p_partial_return(const void* d_rows, int32_t* d_units, const float* d_wts, int R,
                                       int64_t ustride, int k, int H, int me, const uint64_t* h_ret_bases,
                                       int64_t unit_base, const void* d_plan, void* stream);

/* Row-major NVFP4 scales [rows][K/16] -> the MMA 128x4 scale layout, for the valid
 * rows of the groups of precision class `prec` in d_layout (E groups). */
REALB_API int realb_sf_rows_to_mma(const uint8_t* d_sf_rows, int64_t rows_cap, int K, const int32_t* d_layout,
                                   int E, int prec, uint8_t* d_sf_mma, void* stream);

/* dst[i] = src[idx[i]] for bf16 rows of H (EP return path before C3). */
REALB_API int realb_index_rows(const void* d_src, const int32_t* d_idx, int64_t n, int H,
                               void* d_dst, void* stream);

/* ------------------------------------------------------------------------ *
 * K5 — grouped BF16 expert GEMM on tcgen05 (kind::f16, TMA, TMEM).
 *   out[r][n] = sum_k A[r][k] * W[g*N + n][k]  over the groups of precision
 *   `prec` listed in d_layout.
 *   epilogue REALB_EPI_STORE  : out bf16 [rows][N]
 *   epilogue REALB_EPI_SWIGLU : W rows are gate/up interleaved in 128-row
 *        halves (D4); out bf16 [rows][N/2] = silu(gate) * up,
 *        and, when d_out_codes != NULL, also NVFP4-quantised (K4 fused).
 * Replaces the compute term of moesim.costmodel.rank_compute_latency
 * (costmodel.py:60-68).
 * ------------------------------------------------------------------------ */
#define REALB_EPI_STORE 0
#define REALB_EPI_SWIGLU 1
REALB_API int realb_grouped_gemm_bf16(const void* d_a, const void* d_w, int64_t rows_cap,
                            int N, int K, int E, const int32_t* d_layout, int prec,
                            int epilogue, void* d_out, int max_ctas, void* stream);

/* K5, gather form: the A operand is the token matrix itself. Grouped row g of
 * the layout reads x[d_row_src[g]] (bf16 [n_src][K]) through TMA tile::gather4;
 * rows past a group's count are zero. With realb_dispatch_index this replaces
 * realb_dispatch_permute's row copy for W16A16 experts (the dispatch half of
 * moesim's dispatch term, costmodel.py:71-76, done inside the GEMM's loads). */
REALB_API int realb_grouped_gemm_bf16_gather(const void* d_x, int64_t n_src, const int32_t* d_row_src,
                                             const void* d_w, int64_t rows_cap, int N, int K, int E,
                                             const int32_t* d_layout, int prec, int epilogue, void* d_out,
                                             int max_ctas, void* stream);

/* K5, copy-in form: the dispatch row copy runs INSIDE the GEMM. Warps 2-3 of every
 * CTA copy x[d_row_src[g]] -> d_a[g] for the class's valid grouped rows (in grouped
 * order across the grid) while the mainloop runs; the producer's first load of an
 * expert's tiles waits for that expert's rows (per-expert counters d_ready [E],
 * int32, zero on entry and re-zeroed by the kernel). d_err bit 2 is set if a wait
 * timed out. With realb_dispatch_index this replaces realb_dispatch_permute's row
 * copy for W16A16 experts; the copy overlaps the GEMM instead of preceding it. */
REALB_API int realb_grouped_gemm_bf16_copyin(const void* d_x, const int32_t* d_row_src, void* d_a, const void* d_w,
                                             int64_t rows_cap, int N, int K, int E, const int32_t* d_layout,
                                             int prec, int epilogue, void* d_out, int32_t* d_ready,
                                             int32_t* d_err, int max_ctas, void* stream);

/* K5 fused with the EP return (C3 over peer memory): the STORE epilogue, but
 * output row g goes to h_dst_bases[m >> 25] + (m & (2^25 - 1)) * N * 2 with
 * m = d_row_map[g] (int32 [rows_cap]; realb_p2p_return_map builds it), i.e.
 * straight into the token's source rank's return window; no local output
 * buffer and no separate return copy. n_dst <= 64; bases 16-B aligned. */
REALB_API int realb_grouped_gemm_bf16_scatter(const void* d_a, const void* d_w, int64_t rows_cap, int N, int K,
                                              int E, const int32_t* d_layout, int prec, const int32_t* d_row_map,
                                              int n_dst, const uint64_t* h_dst_bases, int max_ctas, void* stream);

/* K6 — grouped NVFP4 x NVFP4 GEMM (tcgen05 kind::mxf4nvf4.block_scale,
 * scale_vec::4X, UE4M3 scales in REALB_SF_MMA128x4 layout) over the W4A4
 * groups of d_layout. Weight rows are indexed by global expert id
 * (W row g*N + n), so only the W4A4 experts' rows need to be quantised.
 * With REALB_EPI_SWIGLU and d_out_codes/d_out_sf non-NULL, the SwiGLU output
 * is written directly as NVFP4 codes + MMA-layout scales for the next GEMM;
 * d_out may then be NULL or a bf16 [rows_cap][N/2] buffer that receives the
 * bf16 SwiGLU values the re-quantisation consumed (parity hook: the codes and
 * scales must equal the reference block rule applied to exactly these values). */
REALB_API int realb_grouped_gemm_nvfp4(const uint8_t* d_a_codes, const uint8_t* d_a_sf,
                             const uint8_t* d_w_codes, const uint8_t* d_w_sf,
                             int64_t rows_cap, int N, int K, int E,
                             const int32_t* d_layout, int epilogue,
                             void* d_out, uint8_t* d_out_codes, uint8_t* d_out_sf,
                             int max_ctas, void* stream);

/* K6 fused with the EP return: the STORE epilogue with per-row destinations,
 * as realb_grouped_gemm_bf16_scatter. */
REALB_API int realb_grouped_gemm_nvfp4_scatter(const uint8_t* d_a_codes, const uint8_t* d_a_sf,
                                               const uint8_t* d_w_codes, const uint8_t* d_w_sf, int64_t rows_cap,
                                               int N, int K, int E, const int32_t* d_layout,
                                               const int32_t* d_row_map, int n_dst, const uint64_t* h_dst_bases,
                                               int max_ctas, void* stream);

/* C3 (local part) — weighted top-k combine:
 *   y[t][h] = addend[t][h] + sum_j topk_w[t][j] * rows[pair_pos[t][j]][h]
 *   (fp32 accumulation, one bf16 rounding). d_addend: bf16 [T][H] or NULL —
 *   the shared-expert output of models that have one (Kimi-VL, ERNIE-4.5-VL). */
REALB_API int realb_combine(const void* d_rows, const int32_t* d_pair_pos, const float* d_topk_w,
                  int T, int H, int k, const void* d_addend, void* d_y, void* stream);

/* Combine with the rank-partial return: W16A16 slots as realb_combine;
 * for a W4A4 owner rank d (d_expert_prec[e] == REALB_PREC_W4A4, owner = e / El) the
 * rows of t's slots on d enter as ONE bf16 partial P_d(t) (their fma chain in slot
 * order, rounded once) at t's first slot on d:
 *   unit_base == -1 : P_d formed here from the rows at d_pos (single-GPU layer, and the
 *                     collective EP path that gets every slot's row back)
 *   unit_base >= 0  : P_d read from row unit_base + d * unit_stride + t of d_rows (the
 *                     return window the owners wrote with realb_p2p_partial_return)
 * Both forms are bit-identical for identical rows. */
REALB_API int realb_combine_partial(const void* d_rows, const int32_t* d_pair_pos, const float* d_topk_w,
                                    const int32_t* d_topk_idx, const uint8_t* d_expert_prec, int El, int T,
                                    int H, int k, const void* d_addend, int64_t unit_base, int64_t unit_stride,
                                    void* d_y, void* stream);

/* ------------------------------------------------------------------------ *
 * P1 — host precision policy, identical fp64 operation order to
 * moesim.balancers.plan_realb (balancers.py:89-122). Host-only (no CUDA).
 *   rank_vt : int64 [R][2] (vision, text) per rank (RankLoad, core.py:70-89)
 *   out_prec: uint8 [R] REALB_PREC_*; out_flags: uint8 [R] bit0 hot,
 *             bit1 vision-heavy.  Returns 1 if the plan is active, 0 if the
 *             batch gate kept it inactive, <0 on error.
 * ------------------------------------------------------------------------ */
REALB_API int realb_plan(const int64_t* rank_vt, int R, double capacity_factor,
               double modality_threshold, int64_t global_batch_threshold,
               int modality_isolated, uint8_t* out_prec, uint8_t* out_flags);

#ifdef __cplusplus
}
#endif
#endif /* REALB_H_ */
