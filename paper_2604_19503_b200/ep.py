"""Expert-parallel ReaLB MoE layer: one process per GPU, NCCL over NVLink.

Per layer on rank r of R (contiguous placement: rank r hosts experts
[r*El, (r+1)*El), place_experts_static, core.py:92-97):

  K1+K2  route the local tokens                         -> top-k, per-expert (v,t)
  C1     all_gather of the [E,2] counts (1 KB)           -> identical global loads on
         every rank (integer sums: identical plans); one host sync, which
         NCCL's all_to_allv needs anyway for its split sizes
  P1     plan_for(strategy) on the global loads (policy.py -> C realb_plan,
         balancers.py:89-122); my precision = plan[r]
  pack   rows sorted by global expert (unpadded): rank-contiguous send buffer;
         rows bound for W4A4 ranks are quantised to packed NVFP4 on the sender
         (fp4_dispatch: 0.5625 H instead of 2 H bytes per row;
         same codes the receiver's K4 would produce, so results are unchanged)
  K3     [side stream] quantise my experts' weights if plan[r] is W4A4 — issued
         before C2 so it runs under the dispatch
  C2     all_to_all_v of the token rows (bytes)
  regroup + K4 + K5/K6   grouped expert MLPs over the received rows
  C3     all_to_all_v back, then the weighted top-k combine

The device work goes through a backend object (``CudaEPOps`` here; the CPU
tests inject an oracle backend) and the collectives through ``EPComm``, so the
host orchestration is one piece of code on GPUs (NCCL), in CPU tests (gloo)
and in the one-GPU, two-process test (gloo staged through the host).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .moe import MoEShape, MoEWeights, operand_noise_
from .policy import STRATEGIES, ClusterConfig, Precision, PrecisionPlan, RealbParams, plan_for, \
    rank_loads_from_counts


# Counter words (byte offsets) in every rank's 256-B counter window. The two
# transports keep separate words: the host-plan path tracks its expected value on
# the host (p2p_epoch * R), the host-sync-free path in device memory (d_expected),
# so calling forward() and forward_device() on the same ops cannot let one path's
# wait pass on the other path's signals.
_DEV_CTR_DISPATCH, _DEV_CTR_RETURN, _DEV_CTR_COUNTS = 0, 4, 8
_HOST_CTR_DISPATCH, _HOST_CTR_RETURN = 16, 20


class PeerWaitTimeout(RuntimeError):
    """A peer-memory wait gave up after 10 s (a peer never signalled): the
    layer's output is invalid."""


# ----------------------------------------------------------------------------- comm
class EPComm:
    """Collectives of the EP layer. ``staged`` copies device tensors through the
    host (gloo on a shared GPU / CPU tests); otherwise tensors go to NCCL as-is."""

    def __init__(self, group=None, staged: bool = False, p2p: bool = False):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.staged = staged
        # p2p: C2/C3 move rows through peer-memory windows (CudaEPOps.setup_p2p);
        # the process group then only carries the C1 count exchange
        self.p2p = p2p

    def all_gather_counts(self, vt_local: torch.Tensor) -> np.ndarray:
        """[E,2] int32 per rank -> host numpy [R,E,2] (the layer's one sync)."""
        src = vt_local.cpu() if self.staged else vt_local
        out = [torch.empty_like(src) for _ in range(self.world)]
        dist.all_gather(out, src.contiguous(), group=self.group)
        return torch.stack(out).cpu().numpy().astype(np.int64)

    def all_to_all_rows(self, out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits):
        out_splits = [int(a) for a in out_splits]
        in_splits = [int(a) for a in in_splits]
        if self.staged:
            o = torch.empty((sum(out_splits),) + tuple(out.shape[1:]), dtype=out.dtype)
            dist.all_to_all_single(o, inp[:sum(in_splits)].cpu(), out_splits, in_splits, group=self.group)
            out[:sum(out_splits)].copy_(o)
        else:
            dist.all_to_all_single(out[:sum(out_splits)], inp[:sum(in_splits)], out_splits, in_splits,
                                   group=self.group)
        return out


# ----------------------------------------------------------------------------- device backend
class CudaEPOps:
    """The sm_100a kernels behind the EP layer (C-ABI library)."""

    def __init__(self, shape: MoEShape, router: torch.Tensor, bias, local: MoEWeights, world: int,
                 max_tokens: int, device="cuda", quant_max_ctas: int = 0):
        self.s, self.router, self.bias, self.local = shape, router, bias, local
        E, k, H, I = shape.num_experts, shape.top_k, shape.hidden, shape.intermediate
        self.E, self.k, self.H, self.I, self.R = E, k, H, I, world
        self.El = E // world
        T = max_tokens
        self.T = T
        dev, i32, bf, u8 = torch.device(device), torch.int32, torch.bfloat16, torch.uint8
        self.dev = dev
        self.nch = (T + 63) // 64
        self.logits = torch.empty(T, E, dtype=torch.float32, device=dev)
        self.topk_idx = torch.empty(T, k, dtype=i32, device=dev)
        self.topk_w = torch.empty(T, k, dtype=torch.float32, device=dev)
        self.cc = torch.empty(self.nch, E, 2, dtype=i32, device=dev)
        self.send_layout = torch.zeros(int(_lib.load().realb_layout_words(E, self.nch)), dtype=i32, device=dev)
        self.vt_local = torch.empty(E, 2, dtype=i32, device=dev)
        self.zero_prec = torch.zeros(E, dtype=u8, device=dev)
        self.send_pos = torch.empty(T, k, dtype=i32, device=dev)
        self.send_buf = torch.empty(T * k * 2 * H, dtype=u8, device=dev)  # byte segments per rank
        self.ret_buf = torch.empty(T * k, H, dtype=bf, device=dev)
        recv_cap = world * T * k  # every token of every rank could pick my experts
        self.recv_cap = recv_cap
        self.recv_buf = torch.empty(recv_cap * 2 * H, dtype=u8, device=dev)
        self.back_buf = torch.empty(recv_cap, H, dtype=bf, device=dev)
        self.row_expert = torch.empty(recv_cap, dtype=i32, device=dev)
        self.row_pos = torch.empty(recv_cap, dtype=i32, device=dev)
        El = self.El
        self.rows_cap = (recv_cap + El * 127 + 127) // 128 * 128
        self.local_layout = torch.zeros(int(_lib.load().realb_layout_words(El, 1)), dtype=i32, device=dev)
        self.base = torch.empty(2 * world * El + 2, dtype=i32, device=dev)
        self.cnt_dev = torch.empty(world, El, dtype=i32, device=dev)
        self.cnt_host = torch.empty(world, El, dtype=i32, pin_memory=True)
        self.prec_local = torch.zeros(El, dtype=u8, device=dev)
        self.a_bf16 = operand_noise_(torch.empty(self.rows_cap, H, dtype=bf, device=dev))
        self.h_bf16 = torch.empty(self.rows_cap, I, dtype=bf, device=dev)
        self.rows_out = torch.empty(self.rows_cap, H, dtype=bf, device=dev)
        self.flag = torch.zeros(1, dtype=i32, device=dev)
        self.quant_max_ctas = quant_max_ctas
        self.side = torch.cuda.Stream(device=dev)
        self._fp4 = None
        self.shared = None
        if shape.shared_intermediate:
            from .moe import SharedExpertMLP

            self.shared = SharedExpertMLP(local.shared_gu, local.shared_d, T, dev)

    def _fp4_ws(self):
        if self._fp4 is None:
            El, H, I, R = self.El, self.H, self.I, self.rows_cap
            u8, dev = torch.uint8, self.dev
            self._fp4 = dict(
                a_codes=operand_noise_(torch.empty(R, H // 2, dtype=u8, device=dev), "codes"),
                a_sf=operand_noise_(torch.empty(R * H // 16, dtype=u8, device=dev), "sf"),
                h_codes=torch.empty(R, I // 2, dtype=u8, device=dev),
                h_sf=torch.empty(R * I // 16, dtype=u8, device=dev),
                wgu_codes=torch.empty(El * 2 * I, H // 2, dtype=u8, device=dev),
                wgu_sf=torch.empty(El * 2 * I * H // 16, dtype=u8, device=dev),
                wd_codes=torch.empty(El * H, I // 2, dtype=u8, device=dev),
                wd_sf=torch.empty(El * H * I // 16, dtype=u8, device=dev),
            )
        return self._fp4

    # K1+K2 and the local counts
    def route(self, x, mod):
        T = x.shape[0]
        s, sp = self.s, _lib.stream_ptr()
        _lib.call("realb_router_topk_stats", x.data_ptr(), self.router.data_ptr(), _lib.ptr(self.bias),
                  mod.data_ptr(), T, self.H, self.E, self.k, s.scoring, float(s.routed_scaling),
                  float(s.norm_min), self.logits.data_ptr(), self.topk_idx.data_ptr(),
                  self.topk_w.data_ptr(), self.cc.data_ptr(), sp)
        _lib.call("realb_moe_align", self.cc.data_ptr(), (T + 63) // 64, self.E, self.zero_prec.data_ptr(),
                  1, self.send_layout.data_ptr(), self.vt_local.data_ptr(), sp)
        return self.topk_idx[:T], self.topk_w[:T], self.vt_local

    # rows sorted by global expert id (unpadded) -> rank-contiguous byte segments
    def pack(self, x, topk_idx, fp4_rows, send_counts):
        """-> (send bytes, send positions [T, k], bytes per row for each destination)."""
        T, H, R = x.shape[0], self.H, self.R
        units = np.array([H // 2 + H // 16 if f else 2 * H for f in fp4_rows], np.int64)
        counts = np.asarray(send_counts, np.int64)
        row0 = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int32)
        byte0 = np.concatenate([[0], np.cumsum(counts * units)[:-1]]).astype(np.int64)
        fmt = np.array(fp4_rows, np.uint8)
        _lib.call("realb_ep_pack", x.data_ptr(), self.topk_idx.data_ptr(), T, H, self.E, self.k,
                  self.send_layout.data_ptr(), (T + 63) // 64, R, fmt.ctypes.data, row0.ctypes.data,
                  byte0.ctypes.data, self.send_pos.data_ptr(), self.send_buf.data_ptr(), self.flag.data_ptr(),
                  _lib.stream_ptr())
        return self.send_buf, self.send_pos[:T], units

    def quantize_local_weights_async(self, timer=None):
        ws = self._fp4_ws()
        main = torch.cuda.current_stream()
        self.side.wait_stream(main)
        with torch.cuda.stream(self.side):
            if timer is not None:
                timer.mark("k3_start", self.side)
            sp = _lib.stream_ptr(self.side)
            El, H, I = self.El, self.H, self.I
            _lib.call("realb_quantize_nvfp4", self.local.w_gu.data_ptr(), _lib.DT_BF16, El * 2 * I, H,
                      ws["wgu_codes"].data_ptr(), ws["wgu_sf"].data_ptr(), _lib.SF_MMA128x4,
                      self.flag.data_ptr(), self.quant_max_ctas, sp)
            _lib.call("realb_quantize_nvfp4", self.local.w_d.data_ptr(), _lib.DT_BF16, El * H, I,
                      ws["wd_codes"].data_ptr(), ws["wd_sf"].data_ptr(), _lib.SF_MMA128x4,
                      self.flag.data_ptr(), self.quant_max_ctas, sp)
            if timer is not None:
                timer.mark("k3_end", self.side)

    def recv_buffer(self):
        return self.recv_buf

    # regroup received rows + local expert MLPs
    def expert_compute(self, recv_buf, cnt: np.ndarray, w4a4: bool, packed_fp4: bool = False,
                       return_rows: bool = True):
        """Regroup + gather the received rows (``recv_buf``: tensor or device address),
        the local expert MLPs, and (return_rows) the copy back into receive order."""
        El, H, I = self.El, self.H, self.I
        n = int(cnt.sum())
        recv_ptr = recv_buf if isinstance(recv_buf, int) else recv_buf.data_ptr()
        sp = _lib.stream_ptr()
        self.cnt_host.numpy()[:] = cnt
        self.cnt_dev.copy_(self.cnt_host, non_blocking=True)
        self.prec_local.fill_(_lib.PREC_W4A4 if w4a4 else _lib.PREC_W16A16)
        _lib.call("realb_ep_regroup", self.cnt_dev.data_ptr(), self.R, El, self.prec_local.data_ptr(), n,
                  self.local_layout.data_ptr(), self.base.data_ptr(), self.row_expert.data_ptr(),
                  self.row_pos.data_ptr(), sp)
        ws = self._fp4_ws() if w4a4 else None
        if packed_fp4:  # rows arrived as NVFP4 (sender-side K4): byte movement only
            _lib.call("realb_gather_rows_nvfp4_packed", recv_ptr, self.row_pos.data_ptr(), n, H,
                      ws["a_codes"].data_ptr(), ws["a_sf"].data_ptr(), None, None, sp)
        else:
            _lib.call("realb_gather_rows", recv_ptr, self.row_expert.data_ptr(), self.row_pos.data_ptr(),
                      n, H, 1, self.prec_local.data_ptr(), self.a_bf16.data_ptr(),
                      _lib.ptr(ws["a_codes"]) if ws else None, _lib.ptr(ws["a_sf"]) if ws else None,
                      self.flag.data_ptr(), None, None, sp)
        lay = self.local_layout.data_ptr()
        if not w4a4:
            _lib.call("realb_grouped_gemm_bf16", self.a_bf16.data_ptr(), self.local.w_gu.data_ptr(),
                      self.rows_cap, 2 * I, H, El, lay, _lib.PREC_W16A16, _lib.EPI_SWIGLU,
                      self.h_bf16.data_ptr(), 0, sp)
            _lib.call("realb_grouped_gemm_bf16", self.h_bf16.data_ptr(), self.local.w_d.data_ptr(),
                      self.rows_cap, H, I, El, lay, _lib.PREC_W16A16, _lib.EPI_STORE,
                      self.rows_out.data_ptr(), 0, sp)
        else:
            torch.cuda.current_stream().wait_stream(self.side)
            _lib.call("realb_grouped_gemm_nvfp4", ws["a_codes"].data_ptr(), ws["a_sf"].data_ptr(),
                      ws["wgu_codes"].data_ptr(), ws["wgu_sf"].data_ptr(), self.rows_cap, 2 * I, H, El,
                      lay, _lib.EPI_SWIGLU, None, ws["h_codes"].data_ptr(), ws["h_sf"].data_ptr(), 0, sp)
            _lib.call("realb_grouped_gemm_nvfp4", ws["h_codes"].data_ptr(), ws["h_sf"].data_ptr(),
                      ws["wd_codes"].data_ptr(), ws["wd_sf"].data_ptr(), self.rows_cap, H, I, El, lay,
                      _lib.EPI_STORE, self.rows_out.data_ptr(), None, None, 0, sp)
        if not return_rows:
            return None
        _lib.call("realb_index_rows", self.rows_out.data_ptr(), self.row_pos.data_ptr(), n, H,
                  self.back_buf.data_ptr(), sp)
        return self.back_buf

    # ------------------------------------------------------------ peer-memory transport
    def setup_p2p(self, comm: "EPComm"):
        """Receive / return windows (CUDA IPC, realb_ipc_alloc) plus two uint32
        counters (dispatch, return) per rank; handles exchanged once over the
        process group; peers' windows mapped (NVLink peer memory across GPUs)."""
        import ctypes as Cty

        R, H, T, k, E = self.R, self.H, self.T, self.k, self.E
        rc = self.rows_cap
        # return window: T*k pair rows, then R*T unit rows of the rank-partial return
        # (owner d's partial for my token t at row T*k + d*T + t)
        sizes = {"recv": R * T * k * 2 * H, "ret": (T * k + R * T) * 2 * H, "ctr": 256, "cnt": R * E * 2 * 4,
                 # rank-partial return: unit table [R sources][T][k] (grouped row or -1) and
                 # the routing weight of every grouped row, written by the senders
                 "units": R * T * k * 4, "wts": rc * 4,
                 # the GEMM operands themselves, written directly by the senders (device-plan path)
                 "opa": rc * H * 2, "opc": rc * (H // 2), "ops": rc * (H // 16),
                 # NVFP4 scales as sent (row-major); converted to "ops" (MMA layout) locally
                 "opsr": rc * (H // 16)}
        # Every rank runs the same collectives whatever fails locally (allocation, mapping),
        # and failures are agreed on, so all ranks raise together and fall back together
        # instead of one rank leaving the others blocked in a collective.
        self._p2p_own, handles, err = {}, {}, None
        try:
            if os.environ.get("REALB_TEST_P2P_FAIL_RANK") == str(comm.rank):  # fault injection (tests)
                raise RuntimeError("injected peer-memory allocation failure")
            for name, nbytes in sizes.items():
                ptr, h = Cty.c_void_p(), (Cty.c_uint8 * 64)()
                _lib.call("realb_ipc_alloc", nbytes, Cty.byref(ptr), h)
                self._p2p_own[name] = ptr.value
                handles[name] = bytes(h)
        except Exception as e:  # noqa: BLE001 - reported to every rank below
            err, handles = f"rank {comm.rank}: {type(e).__name__}: {e}", None
        allh = [None] * R
        dist.all_gather_object(allh, handles, group=comm.group)
        if any(h is None for h in allh):
            self._free_own_windows()
            raise RuntimeError(f"peer-memory windows: allocation failed on some rank ({err or 'peer'})")
        self.p2p = {name: [0] * R for name in sizes}
        self._p2p_opened = []
        try:
            for r in range(R):
                for name in sizes:
                    if r == comm.rank:
                        self.p2p[name][r] = self._p2p_own[name]
                    else:
                        ptr = Cty.c_void_p()
                        _lib.call("realb_ipc_open", allh[r][name], Cty.byref(ptr))
                        self.p2p[name][r] = ptr.value
                        self._p2p_opened.append(ptr.value)
            err = None
        except Exception as e:  # noqa: BLE001
            err = f"rank {comm.rank}: {type(e).__name__}: {e}"
        allerr = [None] * R
        dist.all_gather_object(allerr, err, group=comm.group)
        if any(allerr):
            for ptr in self._p2p_opened:
                _lib.call("realb_ipc_close", ptr)
            self._p2p_opened = []
            self._free_own_windows()
            raise RuntimeError(f"peer-memory windows: mapping failed: {[e for e in allerr if e]}")
        self.p2p_epoch = 0
        self.p2p_rank = comm.rank
        # peers' operand bases (kept alive: the ABI reads them through a host pointer)
        self.op_bases = [np.array(self.p2p[n], np.uint64) for n in ("opa", "opc", "opsr", "units", "wts")]
        self.ret_bases = np.array(self.p2p["ret"], np.uint64)
        # my operand windows (written by the senders) start as in-distribution values,
        # not the allocation's zeros: their padding rows are multiplied too (moe.operand_noise_)
        own = self._p2p_own
        noise = operand_noise_(torch.empty(min(self.rows_cap, 1 << 16), H, dtype=torch.bfloat16, device=self.dev))
        nb = noise.view(torch.uint8).view(-1)
        va = _device_view(own["opa"], sizes["opa"], torch.uint8)
        for i in range(0, va.numel(), nb.numel()):
            n = min(nb.numel(), va.numel() - i)
            va[i:i + n].copy_(nb[:n])
        operand_noise_(_device_view(own["opc"], sizes["opc"], torch.uint8), "codes")
        operand_noise_(_device_view(own["ops"], sizes["ops"], torch.uint8), "sf")
        _device_view(own["units"], sizes["units"] // 4, torch.int32).fill_(-1)  # no rows yet
        del noise, nb
        torch.cuda.synchronize()
        # fused down-GEMM + return: grouped row -> (source, row of its return window)
        self.row_map = torch.empty(self.rows_cap, dtype=torch.int32, device=self.dev)
        # host-sync-free (device-plan) form: plan record, expected-counter words,
        # global expert precisions and the plan kernel's scratch
        dev = self.dev
        lay = (C.c_int64 * 5)()
        _lib.call("realb_p2p_plan_layout", lay)
        self.plan_layout = list(lay)
        self.d_plan = torch.zeros(int(lay[0]) + 64, dtype=torch.uint8, device=dev)
        self.d_expected = torch.zeros(4, dtype=torch.int32, device=dev)
        self.p2p_err = torch.zeros(1, dtype=torch.int32, device=dev)  # set by a timed-out wait
        self.prec_global = torch.zeros(E, dtype=torch.uint8, device=dev)
        self.plan_out = torch.zeros(3 + R, dtype=torch.int32, device=dev)
        self.plan_host = torch.zeros(3 + R, dtype=torch.int32, pin_memory=True)
        self.vt_all_host = torch.zeros(R, E, 2, dtype=torch.int32, pin_memory=True)
        self.gl_layout = torch.zeros(int(_lib.load().realb_layout_words(E, R)), dtype=torch.int32, device=dev)
        self.gl_vt = torch.zeros(E, 2, dtype=torch.int32, device=dev)
        dist.barrier(group=comm.group)

    def p2p_dispatch(self, x, topk_idx, fp4_rows, pairs: np.ndarray, rank: int):
        """C2 over peer memory: rows written straight into every destination's
        receive window (source-major, at offsets derived from the [R][R] pair
        counts), then a system-scope signal per destination and a wait for all
        sources. pairs[s][d]: (token, expert) pairs rank s sends to rank d."""
        T, H, R = x.shape[0], self.H, self.R
        units = np.array([H // 2 + H // 16 if f else 2 * H for f in fp4_rows], np.int64)
        row0 = np.concatenate([[0], np.cumsum(pairs[rank])[:-1]]).astype(np.int32)
        recv_off = np.cumsum(pairs, axis=0) - pairs                     # [s][d] rows before source s at d
        dst = np.array([self.p2p["recv"][d] + int(recv_off[rank, d]) * int(units[d]) for d in range(R)],
                       np.uint64)
        fmt = np.array(fp4_rows, np.uint8)
        sp = _lib.stream_ptr()
        _lib.call("realb_p2p_pack", x.data_ptr(), self.topk_idx.data_ptr(), T, H, self.E, self.k,
                  self.send_layout.data_ptr(), (T + 63) // 64, R, fmt.ctypes.data, row0.ctypes.data,
                  dst.ctypes.data, self.send_pos.data_ptr(), self.flag.data_ptr(), sp)
        self.p2p_epoch += 1
        self._p2p_signal_wait(_HOST_CTR_DISPATCH)
        return self.p2p["recv"][rank], self.send_pos[:T]

    def p2p_return(self, cnt: np.ndarray, pairs: np.ndarray, rank: int):
        """C3 over peer memory: every received row goes from my grouped output
        straight into its source's return window, in the source's send order."""
        R, H = self.R, self.H
        n = int(cnt.sum())
        recv_prefix = np.concatenate([[0], np.cumsum(cnt.sum(axis=1))]).astype(np.int32)
        send_row0 = np.cumsum(pairs, axis=1) - pairs                    # [s][d] rows s sends before d
        dst = np.array([self.p2p["ret"][s_] + int(send_row0[s_, rank]) * 2 * H for s_ in range(R)], np.uint64)
        _lib.call("realb_p2p_return", self.rows_out.data_ptr(), self.row_pos.data_ptr(), n, H, R,
                  recv_prefix.ctypes.data, dst.ctypes.data, _lib.stream_ptr())
        self._p2p_signal_wait(_HOST_CTR_RETURN)
        return self.p2p["ret"][rank]

    def _p2p_signal_wait(self, ctr_off: int):
        R = self.R
        ctrs = np.array([self.p2p["ctr"][d] + ctr_off for d in range(R)], np.uint64)
        sp = _lib.stream_ptr()
        _lib.call("realb_p2p_signal", ctrs.ctypes.data, R, sp)
        _lib.call("realb_p2p_wait", self._p2p_own["ctr"] + ctr_off, (self.p2p_epoch * R) & 0xFFFFFFFF,
                  self.p2p_err.data_ptr(), sp)

    def forward_device(self, x, mod, strategy: str, params: RealbParams, fp4_dispatch: bool,
                       timer=None, rank_partial: bool = False):
        """The whole EP layer with no host synchronisation (CUDA-graph capturable):
        C1 through peer memory, the plan and every window offset derived on the
        device (realb_moe_align_plan over the gathered [R][E][2] counts,
        realb_p2p_plan_offsets), rows dispatched straight into the destinations'
        GEMM operands (NVFP4 towards W4A4 ranks, so the receivers run no gather),
        K3 and both GEMM precisions launched unconditionally and selected by the
        device-side group lists, and the return fused into the down GEMMs (their
        epilogues store every output row into its source's return window).
        -> y; the plan and counts are read back lazily (DevicePlanResult)."""
        from .moe import _STRATEGY_CODE

        R, r, E, El, H, I, k = self.R, self.p2p_rank, self.E, self.El, self.H, self.I, self.k
        T = x.shape[0]
        mark = timer.mark if timer is not None else (lambda *a, **kw: None)
        main = torch.cuda.current_stream()
        sp = _lib.stream_ptr(main)
        mark("start")
        self.route(x, mod)
        self.start_shared(x)
        # C1: my [E][2] counts into every rank's counts window, slot r
        cnt_bases = np.array(self.p2p["cnt"], np.uint64)
        _lib.call("realb_p2p_publish", self.vt_local.data_ptr(), E * 2, R, cnt_bases.ctypes.data, r * E * 2, sp)
        self._signal_wait_dev(_DEV_CTR_COUNTS, 2)
        # P1 on the device over the global counts (R "chunks" of [E][2]), then the window plan
        _lib.call("realb_moe_align_plan", self.p2p["cnt"][r], R, E, R, _STRATEGY_CODE[strategy],
                  float(params.capacity_factor), float(params.modality_threshold),
                  int(params.global_batch_threshold), int(bool(self.s.modality_isolated)),
                  self.prec_global.data_ptr(), self.plan_out.data_ptr(), self.gl_layout.data_ptr(),
                  self.gl_vt.data_ptr(), sp)
        # fp4_dispatch=1: direct dispatch always hands a W4A4 rank its NVFP4 operand
        _lib.call("realb_p2p_plan_offsets", self.p2p["cnt"][r], R, E, r, H, 1,
                  self.prec_global.data_ptr(), self.d_plan.data_ptr(), self.cnt_dev.data_ptr(),
                  self.prec_local.data_ptr(), sp)
        mark("schedule")
        # K3 for my experts if the device plan made them W4A4 (no-op otherwise), under C2
        ws = self._fp4_ws()
        self.side.wait_stream(main)
        with torch.cuda.stream(self.side):
            ssp = _lib.stream_ptr(self.side)
            _lib.call("realb_quantize_experts2_nvfp4",
                      self.local.w_gu.data_ptr(), 2 * I, H, ws["wgu_codes"].data_ptr(), ws["wgu_sf"].data_ptr(),
                      self.local.w_d.data_ptr(), H, I, ws["wd_codes"].data_ptr(), ws["wd_sf"].data_ptr(),
                      El, self.prec_local.data_ptr(), self.flag.data_ptr(), self.quant_max_ctas, ssp)
        # C2, direct: every row lands in its destination's GEMM operand at its final
        # grouped row (bf16, or NVFP4 + MMA-layout scales for a W4A4 destination)
        if rank_partial:  # + each W4A4-bound row's (token, slot) -> grouped row and its weight
            _lib.call("realb_p2p_pack_direct_partial", x.data_ptr(), self.topk_idx.data_ptr(),
                      self.topk_w.data_ptr(), T, H, E, k, self.send_layout.data_ptr(), (T + 63) // 64, R,
                      self.op_bases[0].ctypes.data, self.op_bases[1].ctypes.data, self.op_bases[2].ctypes.data,
                      self.op_bases[3].ctypes.data, self.op_bases[4].ctypes.data, r, self.T,
                      self.d_plan.data_ptr(), self.send_pos.data_ptr(), self.flag.data_ptr(), sp)
        else:
            _lib.call("realb_p2p_pack_direct", x.data_ptr(), self.topk_idx.data_ptr(), T, H, E, k,
                      self.send_layout.data_ptr(), (T + 63) // 64, R,
                      self.op_bases[0].ctypes.data, self.op_bases[1].ctypes.data, self.op_bases[2].ctypes.data,
                      self.d_plan.data_ptr(),
                      self.send_pos.data_ptr(), self.flag.data_ptr(), sp)
        self._signal_wait_dev(_DEV_CTR_DISPATCH, 0)
        mark("dispatch")
        # receive side: only the grouped layout and the row map for the return (no row copies)
        cap = self.recv_cap
        _lib.call("realb_ep_regroup", self.cnt_dev.data_ptr(), R, El, self.prec_local.data_ptr(), cap,
                  self.local_layout.data_ptr(), self.base.data_ptr(), self.row_expert.data_ptr(),
                  self.row_pos.data_ptr(), sp)
        pl = self.d_plan.data_ptr()
        # C3 is fused into the down GEMMs: each output row is stored straight into its
        # source's return window (row_map: grouped row -> source, row), over NVLink
        _lib.call("realb_p2p_return_map", self.row_pos.data_ptr(), cap, R, pl, self.row_map.data_ptr(), sp)
        a_bf16, a_codes, a_sf = self.p2p["opa"][r], self.p2p["opc"][r], self.p2p["ops"][r]
        # the NVFP4 scales arrived row-major: into the MMA layout for the W4A4 groups
        _lib.call("realb_sf_rows_to_mma", self.p2p["opsr"][r], self.rows_cap, H, self.local_layout.data_ptr(),
                  El, _lib.PREC_W4A4, a_sf, sp)
        rb = self.ret_bases.ctypes.data
        # both precisions' GEMMs; each runs only the groups the device plan gave it
        lay = self.local_layout.data_ptr()
        _lib.call("realb_grouped_gemm_bf16", a_bf16, self.local.w_gu.data_ptr(), self.rows_cap,
                  2 * I, H, El, lay, _lib.PREC_W16A16, _lib.EPI_SWIGLU, self.h_bf16.data_ptr(), 0, sp)
        _lib.call("realb_grouped_gemm_bf16_scatter", self.h_bf16.data_ptr(), self.local.w_d.data_ptr(),
                  self.rows_cap, H, I, El, lay, _lib.PREC_W16A16, self.row_map.data_ptr(), R, rb, 0, sp)
        main.wait_stream(self.side)
        _lib.call("realb_grouped_gemm_nvfp4", a_codes, a_sf,
                  ws["wgu_codes"].data_ptr(), ws["wgu_sf"].data_ptr(), self.rows_cap, 2 * I, H, El, lay,
                  _lib.EPI_SWIGLU, None, ws["h_codes"].data_ptr(), ws["h_sf"].data_ptr(), 0, sp)
        if rank_partial:
            # a W4A4 owner: down GEMM rows stay local, then ONE partial row per (source,
            # token) goes back (no-op kernels on a W16A16 owner: no W4A4 groups, gate off)
            _lib.call("realb_grouped_gemm_nvfp4", ws["h_codes"].data_ptr(), ws["h_sf"].data_ptr(),
                      ws["wd_codes"].data_ptr(), ws["wd_sf"].data_ptr(), self.rows_cap, H, I, El, lay,
                      _lib.EPI_STORE, self.rows_out.data_ptr(), None, None, 0, sp)
            _lib.call("realb_p2p_partial_return", self.rows_out.data_ptr(), self._p2p_own["units"],
                      self._p2p_own["wts"], R, self.T, k, H, r, rb, self.T * k, pl, sp)
        else:
            _lib.call("realb_grouped_gemm_nvfp4_scatter", ws["h_codes"].data_ptr(), ws["h_sf"].data_ptr(),
                      ws["wd_codes"].data_ptr(), ws["wd_sf"].data_ptr(), self.rows_cap, H, I, El, lay,
                      self.row_map.data_ptr(), R, rb, 0, sp)
        mark("compute")
        self._signal_wait_dev(_DEV_CTR_RETURN, 1)
        y = torch.empty(T, H, dtype=torch.bfloat16, device=self.dev)
        addend = self.shared.join() if self.shared is not None and T > 0 else None
        if rank_partial:
            _lib.call("realb_combine_partial", self.p2p["ret"][r], self.send_pos.data_ptr(), self.topk_w.data_ptr(),
                      self.topk_idx.data_ptr(), self.prec_global.data_ptr(), El, T, H, k, addend, self.T * k,
                      self.T, y.data_ptr(), sp)
        else:
            _lib.call("realb_combine", self.p2p["ret"][r], self.send_pos.data_ptr(), self.topk_w.data_ptr(),
                      T, H, k, addend, y.data_ptr(), sp)
        mark("combine")
        if torch.cuda.is_current_stream_capturing():
            return y, None
        self.plan_host.copy_(self.plan_out, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(main)
        return y, DevicePlanResult(self, ev)

    def read_counts(self) -> np.ndarray:
        """[R, E, 2] global counts of the last device-plan layer call (own counts window)."""
        view = _device_view(self.p2p["cnt"][self.p2p_rank], self.R * self.E * 2, torch.int32)
        return view.reshape(self.R, self.E, 2).cpu().numpy().astype(np.int64)

    def _signal_wait_dev(self, ctr_off: int, slot: int):
        R = self.R
        ctrs = np.array([self.p2p["ctr"][d] + ctr_off for d in range(R)], np.uint64)
        sp = _lib.stream_ptr()
        _lib.call("realb_p2p_signal", ctrs.ctypes.data, R, sp)
        _lib.call("realb_p2p_wait_next", self.d_expected.data_ptr() + 4 * slot, R,
                  self._p2p_own["ctr"] + ctr_off, self.p2p_err.data_ptr(), sp)

    def _free_own_windows(self):
        for ptr in getattr(self, "_p2p_own", {}).values():
            _lib.call("realb_ipc_free", ptr)
        self._p2p_own = {}

    def close_p2p(self):
        torch.cuda.synchronize()
        for p in getattr(self, "_p2p_opened", []):
            _lib.call("realb_ipc_close", p)
        for p in getattr(self, "_p2p_own", {}).values():
            _lib.call("realb_ipc_free", p)
        self._p2p_opened, self._p2p_own = [], {}

    def ret_buffer(self):
        return self.ret_buf

    def time_gate_up(self, reps: int = 5):
        """(median ms, algorithmic flops, is_fp4) of the local gate_up grouped GEMM
        over the rows of the last forward (valid rows only, padding excluded)."""
        El, H, I = self.El, self.H, self.I
        n = int(self.cnt_dev.sum().item())  # filled by the host (C1 path) or the device plan
        w4a4 = bool(self.prec_local[0].item() == _lib.PREC_W4A4)
        lay, sp = self.local_layout.data_ptr(), _lib.stream_ptr()
        ts = []
        for _ in range(reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            if w4a4:
                ws = self._fp4_ws()
                _lib.call("realb_grouped_gemm_nvfp4", ws["a_codes"].data_ptr(), ws["a_sf"].data_ptr(),
                          ws["wgu_codes"].data_ptr(), ws["wgu_sf"].data_ptr(), self.rows_cap, 2 * I, H, El,
                          lay, _lib.EPI_SWIGLU, None, ws["h_codes"].data_ptr(), ws["h_sf"].data_ptr(), 0, sp)
            else:
                _lib.call("realb_grouped_gemm_bf16", self.a_bf16.data_ptr(), self.local.w_gu.data_ptr(),
                          self.rows_cap, 2 * I, H, El, lay, _lib.PREC_W16A16, _lib.EPI_SWIGLU,
                          self.h_bf16.data_ptr(), 0, sp)
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e))
        return float(sorted(ts)[len(ts) // 2]), 2.0 * n * (2 * I) * H, w4a4

    def start_shared(self, x):
        """Shared-expert MLP of this rank's tokens on its own stream, overlapping
        C1 / plan / dispatch / expert compute / return (§8f-2)."""
        if self.shared is not None and x.shape[0] > 0:
            self.shared.start(x)

    def combine(self, ret_buf, send_pos, topk_w, partial_prec=None):
        """Weighted top-k combine of the returned rows (send order). partial_prec (uint8 [E]
        expert precisions, host): the rank-partial return's arithmetic, formed here from
        every slot's returned row — equal to the device path's owner-side partials."""
        T = send_pos.shape[0]
        y = torch.empty(T, self.H, dtype=torch.bfloat16, device=self.dev)
        ret_ptr = ret_buf if isinstance(ret_buf, int) else ret_buf.data_ptr()
        addend = self.shared.join() if self.shared is not None and T > 0 else None
        if partial_prec is not None:
            self.prec_partial = torch.as_tensor(np.asarray(partial_prec, np.uint8)).to(self.dev)
            _lib.call("realb_combine_partial", ret_ptr, self.send_pos.data_ptr(), self.topk_w.data_ptr(),
                      self.topk_idx.data_ptr(), self.prec_partial.data_ptr(), self.El, T, self.H, self.k, addend,
                      -1, 0, y.data_ptr(), _lib.stream_ptr())
        else:
            _lib.call("realb_combine", ret_ptr, self.send_pos.data_ptr(), self.topk_w.data_ptr(),
                      T, self.H, self.k, addend, y.data_ptr(), _lib.stream_ptr())
        return y


# ----------------------------------------------------------------------------- the EP layer
class EPMoELayer:
    """One EP rank of a ReaLB MoE layer (host orchestration, backend-agnostic).

    ``fp4_dispatch``: rows bound for W4A4 ranks travel as packed NVFP4
    (SURVEY.md §8f-1). ``timer`` (optional) gets ``mark(phase)`` calls at the
    phase boundaries of engine.py's RankPhases (schedule / transform /
    dispatch / compute / combine)."""

    def __init__(self, shape: MoEShape, comm: EPComm, ops, fp4_dispatch: bool = False, rank_partial: bool = False):
        if shape.num_experts % comm.world:
            raise ValueError("experts must divide evenly over the EP ranks")
        self.shape, self.comm, self.ops = shape, comm, ops
        self.R, self.rank = comm.world, comm.rank
        self.El = shape.num_experts // self.R
        self.cluster = ClusterConfig(self.R, 1, self.El, 1, shape.modality_isolated)
        self.fp4_dispatch = fp4_dispatch
        # rank_partial: a W4A4 owner returns ONE bf16 partial row per (token, owner) — its
        # slots pre-summed — instead of one row per (token, slot)
        self.rank_partial = rank_partial

    def forward_device(self, x, mod, strategy: str = "realb", params: RealbParams | None = None, timer=None):
        """Host-sync-free EP layer (peer-memory transport only): -> (y, DevicePlanResult
        or None under graph capture)."""
        if not (self.comm.p2p and hasattr(self.ops, "forward_device")):
            raise ValueError("the device-plan EP layer needs the peer-memory transport")
        if strategy not in STRATEGIES:
            raise ValueError(f"unknown strategy {strategy!r}")
        if not self.fp4_dispatch:
            # direct dispatch writes each row into its owner's GEMM operand in the
            # owner's precision: a W4A4 owner always receives NVFP4 rows
            raise ValueError("the device-plan EP layer always sends NVFP4 rows to W4A4 ranks "
                             "(fp4_dispatch=True); use forward() for bf16 dispatch")
        return self.ops.forward_device(x, mod, strategy, params or RealbParams(), self.fp4_dispatch, timer,
                                       rank_partial=self.rank_partial)

    def forward(self, x, mod, strategy: str = "realb", params: RealbParams | None = None, timer=None):
        R, r, El, E = self.R, self.rank, self.El, self.shape.num_experts
        mark = timer.mark if timer is not None else (lambda *a, **k: None)
        mark("start")
        topk_idx, topk_w, vt_local = self.ops.route(x, mod)
        if hasattr(self.ops, "start_shared"):
            self.ops.start_shared(x)
        vt_all = self.comm.all_gather_counts(vt_local)                      # C1 (host sync)
        plan = plan_for(strategy, rank_loads_from_counts(vt_all.sum(0), self.cluster), self.cluster,
                        params or RealbParams())                             # P1
        w4a4 = plan.per_rank_precision[r] is Precision.W4A4
        fp4_rows = [self.fp4_dispatch and p is Precision.W4A4 for p in plan.per_rank_precision]
        send_counts = vt_all[r].reshape(R, El, 2).sum(axis=(1, 2))
        cnt = vt_all[:, r * El:(r + 1) * El, :].sum(axis=2)                 # [R, El]
        recv_counts = cnt.sum(axis=1)
        mark("schedule")
        if w4a4:
            self.ops.quantize_local_weights_async(timer)                     # K3 under C2
        if self.comm.p2p:  # C2 / C3 through peer-memory windows (no collective on the data path)
            pairs = vt_all.sum(axis=2).reshape(R, R, El).sum(axis=2)         # [s][d] pairs s -> d
            recv_buf, send_pos = self.ops.p2p_dispatch(x, topk_idx, fp4_rows, pairs, r)
            mark("dispatch")
            self.ops.expert_compute(recv_buf, cnt, w4a4, fp4_rows[r], return_rows=False)
            mark("compute")
            ret = self.ops.p2p_return(cnt, pairs, r)
        else:
            send_buf, send_pos, units = self.ops.pack(x, topk_idx, fp4_rows, send_counts)
            recv_buf = self.comm.all_to_all_rows(self.ops.recv_buffer(), send_buf, recv_counts * units[r],
                                                 send_counts * units)        # C2
            mark("dispatch")
            back = self.ops.expert_compute(recv_buf, cnt, w4a4, fp4_rows[r])
            mark("compute")
            ret = self.comm.all_to_all_rows(self.ops.ret_buffer(), back, send_counts, recv_counts)  # C3
        if self.rank_partial:
            from .policy import place_experts_static

            y = self.ops.combine(ret, send_pos, topk_w,
                                 partial_prec=plan.expert_precision(place_experts_static(self.cluster)))
        else:
            y = self.ops.combine(ret, send_pos, topk_w)
        mark("combine")
        return y, plan, vt_all


def _device_view(ptr: int, numel: int, dtype) -> torch.Tensor:
    """Zero-copy torch view of raw device memory (a peer-memory window)."""
    typestr = {torch.int32: "<i4", torch.uint8: "|u1", torch.bfloat16: "<f2"}[dtype]

    class _Arr:
        __cuda_array_interface__ = {"shape": (numel,), "typestr": typestr, "data": (ptr, False),
                                    "version": 3}
    return torch.as_tensor(_Arr(), device="cuda")


class DevicePlanResult:
    """The device plan of a host-sync-free EP layer call, read back on first use."""

    def __init__(self, ops, event):
        self.ops, self.event, self._plan = ops, event, None

    def check(self) -> None:
        """Raise PeerWaitTimeout if a peer-memory wait of this rank timed out."""
        self.event.synchronize()
        if int(self.ops.p2p_err.item()) != 0:
            raise PeerWaitTimeout("a peer-memory wait timed out (a peer never signalled); output invalid")

    @property
    def plan(self) -> PrecisionPlan:
        if self._plan is None:
            self.check()
            po = self.ops.plan_host.numpy()
            R = self.ops.R
            flags = po[3:3 + R]
            self._plan = PrecisionPlan(
                tuple(Precision.W4A4 if f & 4 else Precision.W16A16 for f in flags),
                frozenset(int(i) for i in np.flatnonzero(flags & 1)),
                frozenset(int(i) for i in np.flatnonzero(flags & 2)), bool(po[0]))
        return self._plan


class CudaPhaseTimer:
    """CUDA events at the EP layer's phase boundaries, on the main stream (and the
    side stream for K3) -> RankPhases in ns (engine.py:55-76)."""

    PHASES = ("start", "schedule", "dispatch", "compute", "combine")

    def __init__(self):
        self.ev = {}

    def mark(self, name, stream=None):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        self.ev[name] = e

    def phases(self):
        from .moe import RankPhases

        self.ev["combine"].synchronize()
        ms = lambda a, b: self.ev[a].elapsed_time(self.ev[b]) if a in self.ev and b in self.ev else 0.0
        ns = lambda v: int(round(v * 1e6))
        return RankPhases(ns(ms("start", "schedule")), ns(ms("k3_start", "k3_end")),
                          ns(ms("schedule", "dispatch")), ns(ms("dispatch", "compute")),
                          ns(ms("compute", "combine")))

    def total_ns(self):
        return int(round(self.ev["start"].elapsed_time(self.ev["combine"]) * 1e6))


def split_weights(shape: MoEShape, router, gate_up_hf, down_hf, rank: int, world: int, bias=None,
                  device="cuda", shared=None) -> MoEWeights:
    """The local experts' weights of an EP rank (contiguous placement); the shared
    expert (if any) is replicated on every rank."""
    from dataclasses import replace

    El = shape.num_experts // world
    sl = slice(rank * El, (rank + 1) * El)
    local_shape = replace(shape, num_experts=El)
    return MoEWeights.from_hf(local_shape, router[:El], gate_up_hf[sl], down_hf[sl], device=device,
                              shared=shared)


# ----------------------------------------------------------------------------- bench (N > 1)
def run_bench(args):
    """bench.py under torchrun: one rank per GPU, NCCL, weak scaling (tokens/GPU
    fixed). Prints bench.py's JSON line on rank 0: value = all ranks' tokens /
    max-over-ranks device time; speedup vs the all-BF16 EP run of the same
    kernels; e2e with host buffers; per-phase RankPhases of every rank; the
    critical rank's gate_up GEMM against its precision's peak."""
    import json

    from .clocks import FP4_TFLOPS_MEASURED, ClockSampler, measured_peaks
    from .moe import SHAPES
    from .workload import WorkloadSpec, make_batch, make_experts

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local_rank = int(os.environ.get("LOCAL_RANK", rank))
    # REALB_EP_COMM: "nccl" (NCCL all-to-alls, one GPU per rank); "p2p" (C2/C3
    # through CUDA-IPC peer-memory windows, NCCL only for the C1 counts); "gloo" /
    # "p2p-gloo": validation modes for a one-GPU box (all ranks share cuda:0, C1
    # (and C2/C3 for "gloo") staged through the host).
    # "p2p-graph" / "p2p-graph-gloo": the host-sync-free layer (device plan) replayed as
    # one CUDA graph per step. "auto" (default) / "auto-gloo": set up the peer-memory
    # transport, check on this very box that one host-sync-free layer call equals the
    # NCCL path bit for bit (and that no wait timed out) on every rank, and use it if
    # so; otherwise fall back to the NCCL path. The line reports which one ran.
    mode = os.environ.get("REALB_EP_COMM", "auto")
    if mode == "auto" and torch.cuda.device_count() < world:
        mode = "auto-gloo"  # fewer GPUs than ranks: validation run, ranks share cuda:0
    staged = mode in ("gloo", "p2p-gloo", "p2p-graph-gloo", "auto-gloo")
    auto = mode in ("auto", "auto-gloo")
    p2p = mode in ("p2p", "p2p-gloo", "p2p-graph", "p2p-graph-gloo") or auto
    graph = mode in ("p2p-graph", "p2p-graph-gloo") or auto
    if staged:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    shape = SHAPES[args.config]
    T = args.tokens
    spec = WorkloadSpec(tokens=T, vision_frac=args.vision_frac, num_ranks=world, rank=rank)
    x, mod, router, _ = make_batch(shape, spec)
    gu, dn = make_experts(shape)  # same seed on every rank: identical global weights
    bias = torch.zeros(shape.num_experts, device="cuda") if shape.scoring == _lib.SCORE_SIGMOID_RENORM else None
    from .workload import make_shared_expert

    local = split_weights(shape, router, gu, dn, rank, world, shared=make_shared_expert(shape))
    del gu, dn
    comm = EPComm(staged=staged, p2p=p2p)
    ops = CudaEPOps(shape, router.contiguous(), bias, local, world, T)
    fp4_dispatch = not getattr(args, "bf16_dispatch", False)
    if not fp4_dispatch:
        graph = False  # the host-sync-free layer always sends NVFP4 rows to W4A4 owners
    dev_t = "cpu" if staged else "cuda"
    transport_check = None
    if p2p:
        try:
            ops.setup_p2p(comm)
        except Exception as e:  # no peer mapping on this box: the collective path
            if not auto:
                raise
            p2p = graph = False
            comm = EPComm(staged=staged, p2p=False)
            transport_check = f"peer-memory setup failed ({type(e).__name__}): NCCL path"
    layer = EPMoELayer(shape, comm, ops, fp4_dispatch=fp4_dispatch)
    if auto and p2p:
        # both strategies the bench times, each: NCCL-path layer vs host-sync-free layer
        ref_layer = EPMoELayer(shape, EPComm(staged=staged, p2p=False), ops, fp4_dispatch=fp4_dispatch)
        diag = []
        for strategy in ("realb", "baseline"):
            y_ref, _, _ = ref_layer.forward(x, mod, strategy)
            y_ref = y_ref.clone()
            try:  # a failure here must still reach the agreement below (no rank left waiting)
                y_dev, _ = layer.forward_device(x, mod, strategy)
                torch.cuda.synchronize()
                d = (y_ref.float() - y_dev.float()).abs()
                diag.append([float(d.max().nan_to_num(float("inf"))), int((y_ref != y_dev).sum()),
                             int(ops.p2p_err.item())])
            except Exception as e:  # noqa: BLE001
                diag.append([float("inf"), -1, f"{type(e).__name__}: {str(e)[:120]}"])
        ok = torch.tensor([int(all(m == 0 and n == 0 and e == 0 for m, n, e in diag))], device=dev_t)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()):
            transport_check = ("host-sync-free peer-memory layer == NCCL layer bit for bit on every rank "
                               "(realb and baseline)")
        else:
            alld = [None] * world
            dist.all_gather_object(alld, diag, group=comm.group)
            transport_check = ("peer-memory layer differed from the NCCL layer (or a wait timed out): NCCL "
                               f"path; per rank [[max |diff|, differing elements, wait error] x (realb, "
                               f"baseline)] = {alld}")
            p2p = graph = False
            layer = ref_layer
            comm = layer.comm

    def max_over_ranks(v: float) -> float:
        t = torch.tensor([v], dtype=torch.float64, device=dev_t)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(strategy, steps, warmup, e2e=False):
        """ms per step (max over ranks). e2e: every step uploads x/modality from
        pinned host memory and downloads y, inside the timed region."""
        xh, mh = x.cpu().pin_memory(), mod.cpu().pin_memory()
        yh = torch.empty(T, shape.hidden, dtype=torch.bfloat16).pin_memory()
        xd, md = torch.empty_like(x), torch.empty_like(mod)

        if graph:
            xin, min_ = (xd, md) if e2e else (x, mod)
            xd.copy_(x)
            md.copy_(mod)
            layer.forward_device(xin, min_, strategy)  # eager first: lazy workspaces
            torch.cuda.synchronize()
            dist.barrier()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                yg, _ = layer.forward_device(xin, min_, strategy)

        def step():
            if e2e:
                xd.copy_(xh, non_blocking=True)
                md.copy_(mh, non_blocking=True)
                if graph:
                    g.replay()
                    y = yg
                else:
                    y, _, _ = layer.forward(xd, md, strategy)
                yh.copy_(y, non_blocking=True)
            elif graph:
                g.replay()
            else:
                layer.forward(x, mod, strategy)

        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(steps):
            step()
        e.record()
        torch.cuda.synchronize()
        dist.barrier()
        return max_over_ranks(s.elapsed_time(e)) / steps

    def timed_e2e_pipelined(strategy, steps, warmup):
        """e2e with host buffers as a serving loop runs it (the N = 1 bench's pipeline):
        two graph instances over double-buffered inputs / outputs, H2D and D2H on their
        own streams, so step i+1's upload and step i-1's download overlap step i's layer.
        The timed steps include their own first upload and last download."""
        nb = 2
        xs = [torch.empty_like(x) for _ in range(nb)]
        ms_ = [torch.empty_like(mod) for _ in range(nb)]
        for i in range(nb):
            xs[i].copy_(x)
            ms_[i].copy_(mod)
        layer.forward_device(xs[0], ms_[0], strategy)  # eager first: lazy workspaces
        torch.cuda.synchronize()
        dist.barrier()
        graphs, ys = [], []
        for i in range(nb):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                yg, _ = layer.forward_device(xs[i], ms_[i], strategy)
            graphs.append(g)
            ys.append(yg)
        n = steps + warmup
        xh = [x.cpu().pin_memory() for _ in range(min(n, 4))]
        mh = [mod.cpu().pin_memory() for _ in range(min(n, 4))]
        yh = [torch.empty(T, shape.hidden, dtype=torch.bfloat16).pin_memory() for _ in range(min(n, 4))]
        for a, b in zip(xh, mh):  # first DMA touch of a pinned buffer is slow: untimed
            xs[0].copy_(a, non_blocking=True)
            ms_[0].copy_(b, non_blocking=True)
        for c in yh:
            c.copy_(ys[0], non_blocking=True)
        torch.cuda.synchronize()
        comp = torch.cuda.current_stream()
        up, down = torch.cuda.Stream(), torch.cuda.Stream()
        ev = lambda: torch.cuda.Event(enable_timing=True)
        h2d, cdone, d2h = [ev() for _ in range(n)], [ev() for _ in range(n)], [ev() for _ in range(n)]
        t0, t1 = ev(), ev()
        for i in range(n):
            if i == warmup:
                torch.cuda.synchronize()
                dist.barrier()
                t0.record(up)
            b = i % nb
            with torch.cuda.stream(up):
                if i >= nb:
                    up.wait_event(cdone[i - nb])  # graph i-2 finished reading xs[b]
                xs[b].copy_(xh[i % len(xh)], non_blocking=True)
                ms_[b].copy_(mh[i % len(mh)], non_blocking=True)
                h2d[i].record(up)
            comp.wait_event(h2d[i])
            if i >= nb:
                comp.wait_event(d2h[i - nb])  # ys[b] downloaded before it is rewritten
            graphs[b].replay()
            cdone[i].record(comp)
            with torch.cuda.stream(down):
                down.wait_event(cdone[i])
                yh[i % len(yh)].copy_(ys[b], non_blocking=True)
                d2h[i].record(down)
        t1.record(down)
        torch.cuda.synchronize()
        dist.barrier()
        return max_over_ranks(t0.elapsed_time(t1)) / steps

    # kernels per layer call, counted on one eager call, x timed steps
    _lib.launch_count = 0
    if graph:
        layer.forward_device(x, mod, "realb")
    else:
        layer.forward(x, mod, "realb")
    launches = _lib.launch_count * args.steps
    with ClockSampler(local_rank) as clk:
        ms = timed("realb", args.steps, args.warmup)
    # the speedup over all-BF16 EP from interleaved rounds (realb, baseline, ...): clock /
    # power drift over the run must not favour the arm timed first
    pairs_ab = []
    for _ in range(3):
        a = timed("realb", max(2, args.steps // 3), 1)
        b = timed("baseline", max(2, args.steps // 3), 1)
        pairs_ab.append((a, b))
    speedup_ab = float(sum(b for _, b in pairs_ab) / sum(a for a, _ in pairs_ab))
    ms_bf16 = ms * speedup_ab  # the bf16 arm on the headline's scale
    ms_e2e = (timed_e2e_pipelined("realb", args.steps, max(2, args.warmup // 2)) if graph else
              timed("realb", args.steps, max(1, args.warmup // 2), e2e=True))

    # per-rank phases (engine.py RankPhases) of one extra step of each strategy
    phases = {}
    for strategy in ("realb", "baseline"):
        tm = CudaPhaseTimer()
        if graph:
            _, res = layer.forward_device(x, mod, strategy, timer=tm)
            plan_s, vt_all = res.plan, ops.read_counts()
        else:
            _, plan_s, vt_all = layer.forward(x, mod, strategy, timer=tm)
        ph = tm.phases()
        row = [ph.schedule_ns, ph.transform_ns, ph.dispatch_ns, ph.compute_ns, ph.combine_ns, tm.total_ns()]
        allrows = [None] * world
        dist.all_gather_object(allrows, row)
        phases[strategy] = allrows
        if strategy == "realb":
            plan = plan_s
    # critical rank's gate_up GEMM (the dominant kernel) against its precision's peak
    if graph:
        layer.forward_device(x, mod, "realb")
    else:
        layer.forward(x, mod, "realb")
    torch.cuda.synchronize()
    g_ms, g_flops, g_fp4 = ops.time_gate_up()
    allg = [None] * world
    dist.all_gather_object(allg, (g_ms, g_flops, g_fp4))
    # a timed-out peer-memory wait anywhere voids the run: reported, never hidden
    wait_err = int(ops.p2p_err.item()) if getattr(ops, "_p2p_own", None) else 0
    wait_errs = [None] * world
    dist.all_gather_object(wait_errs, wait_err)
    cpu = None
    if rank == 0 and not getattr(args, "no_cpu_baseline", False):
        import sys as _sys
        from pathlib import Path as _P

        _sys.path.insert(0, str(_P(__file__).resolve().parents[1]))
        from oracle.cpu_arm import CpuLayerArm  # the CPU restatement (test infrastructure), rank 0 only

        arm = CpuLayerArm(args.config, args.cpu_sample_tokens, args.vision_frac, num_ranks=world)
        dt = min(arm.step() for _ in range(2))
        cpu = arm.describe(args.cpu_sample_tokens / dt)
        cpu["quantiser"] = arm.quantiser_rates()
        cpu["policy"] = arm.policy_us_per_layer()
        del arm
    dist.barrier()
    if rank == 0:
        peaks, src = measured_peaks()
        crit = max(range(world), key=lambda i: allg[i][0])
        gm, gf, g4 = allg[crit]
        peak = FP4_TFLOPS_MEASURED if g4 else float(peaks.get("bf16_tflops", 1641.1))
        achieved = gf / (gm / 1e3) / 1e12
        # SURVEY §8(d) layer roofline: t_roof = max_r F_r / Peak(plan_r), F_r = pairs_r x 6HI;
        # full path adds 2 x max_r(bytes received by r) / 900 GB/s (dispatch + return)
        H_, I_ = shape.hidden, shape.intermediate
        rp = vt_all.sum(0).reshape(world, -1, 2).sum(axis=(1, 2))
        w4 = [p is Precision.W4A4 for p in plan.per_rank_precision]
        bf16_peak = float(peaks.get("bf16_tflops", 1641.1)) * 1e12
        t_rank = [float(rp[i]) * 6 * H_ * I_ / ((FP4_TFLOPS_MEASURED * 1e12) if w4[i] else bf16_peak)
                  for i in range(world)]
        row_b = [(H_ // 2 + H_ // 16) if (w4[i] and fp4_dispatch) else 2 * H_ for i in range(world)]
        t_comm = 2.0 * max(float(rp[i]) * row_b[i] for i in range(world)) / 900e9
        layer_roof = {"t_roof_ms": max(t_rank) * 1e3, "t_roof_full_path_ms": (max(t_rank) + t_comm) * 1e3,
                      "t_meas_ms": ms, "frac": max(t_rank) * 1e3 / ms,
                      "frac_full_path": (max(t_rank) + t_comm) * 1e3 / ms,
                      "what": "max_r pairs_r x 6HI / peak(plan_r) (BF16 burst / measured NVFP4); full path adds "
                              "2 x max_r received bytes / 900 GB/s"}
        names = ("schedule_ns", "transform_ns", "dispatch_ns", "compute_ns", "combine_ns", "total_ns")
        out = {"metric": "MoE-layer prefill tokens/s and speedup vs all-BF16 EP at 1/2/4/8 B200",
               "value": world * T / (ms / 1e3), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "bf16 (nvfp4 on W4A4 ranks)", "data": "synthetic",
               "config": {"workload": f"{shape.name} MoE layer prefill, {T} tokens/GPU, EP{world}, "
                                      f"{args.vision_frac:.0%} vision",
                          "strategy": "realb", "ep_ranks": world, "tokens_per_gpu": T,
                          "parallelism": f"ep{world}",
                          "dispatch_rows_to_w4a4": "nvfp4" if fp4_dispatch else "bf16",
                          "l2": "inputs + weights per GPU exceed L2 (not flushed)"},
               "speedup_vs_bf16": speedup_ab, "ms_per_step_bf16": ms_bf16,
               "speedup_timing": "3 interleaved rounds of realb / baseline steps (ratio of sums)",
               "e2e": {"value": world * T / (ms_e2e / 1e3), "unit": "tokens/s",
                       "h2d_bytes_per_step": int(world * (x.numel() * 2 + mod.numel())),
                       "d2h_bytes_per_step": int(world * T * shape.hidden * 2),
                       "pipeline": "double-buffered per rank: H2D(i+1) || graph replay of the host-sync-free "
                                   "layer (i) || D2H(i-1)" if graph else
                                   "serial per step (the C1 count exchange syncs the host)"},
               "roofline": {"kernel": f"grouped GEMM gate_up on the critical rank {crit} "
                                      f"({'NVFP4 K6' if g4 else 'BF16 K5'})",
                            "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                            "frac": achieved / peak, "traffic": None,
                            "peak_source": "measured cuBLASLt NVFP4 (DESIGN.md §4)" if g4
                            else f"{src} bf16_tflops (burst)",
                            "algorithmic_flops_per_launch": gf, "launch_ms": gm, "layer": layer_roof},
               "plan_w4a4_ranks": sorted(plan.accelerated_ranks),
               "p2p_wait_timeouts": wait_errs,
               "cpu_baseline": cpu,
               "rank_pairs": vt_all.sum(0).reshape(world, -1, 2).sum(axis=(1, 2)).tolist(),
               "rank_phases_ns": {s: [dict(zip(names, r)) for r in rows] for s, rows in phases.items()},
               "gpu_launches": int(launches),
               "clocks": clk.summary(),
               "comm": ("peer-memory windows incl. C1, device plan, one CUDA graph per layer" if graph else
                        "peer-memory windows (CUDA IPC / NVLink), host plan" if p2p else
                        "gloo-staged all-to-alls" if staged else "nccl all-to-alls")
                       + (" — ranks share one GPU (validation only)" if staged else ""),
               "transport_check": transport_check}
        print(json.dumps(out), flush=True)
    if getattr(ops, "_p2p_own", None):
        dist.barrier()
        ops.close_p2p()
    dist.destroy_process_group()
