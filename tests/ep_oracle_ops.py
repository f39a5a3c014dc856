"""TEST-ONLY device backend for ep.EPMoELayer built on the CPU oracle
(oracle/moe_ref.py), so the EP host orchestration and collectives run under
gloo on CPU with world_size > 1."""

import numpy as np
import torch

from oracle import moe_ref


class OracleEPOps:
    def __init__(self, shape, router, gate_up, down, rank, world):
        self.s, self.router = shape, router              # numpy float32 (bf16 values)
        self.gu, self.dn = gate_up, down                 # full HF-layout numpy weights
        self.rank, self.R = rank, world
        self.El = shape.num_experts // world

    def route(self, x, mod):
        s = self.s
        self.x = x.float().numpy()
        _, idx, w = moe_ref.route(self.x, self.router, s.top_k, s.scoring, routed_scaling=s.routed_scaling)
        vt = moe_ref.expert_counts(idx, mod.numpy(), s.num_experts)
        return idx, w, torch.from_numpy(vt.astype(np.int32))

    def pack(self, x, idx, fp4_rows, send_counts):
        """float rows (the oracle backend sends fp32 rows; NVFP4 rows would be
        re-quantised to the same codes on the receiver); 1 row unit per row."""
        T, k = idx.shape
        flat = idx.reshape(-1)
        order = np.lexsort((np.arange(T * k), flat))      # by expert, then (token, slot)
        send = self.x[order // k]
        pos = np.empty(T * k, np.int64)
        pos[order] = np.arange(T * k)
        self.send_expert = flat[order]
        return torch.from_numpy(send.astype(np.float32)), pos.reshape(T, k), np.ones(self.R, np.int64)

    def quantize_local_weights_async(self, timer=None):
        pass

    def recv_buffer(self):
        return torch.empty(self.R * 100000, self.s.hidden, dtype=torch.float32)

    def expert_compute(self, recv_buf, cnt, w4a4, packed_fp4=False):
        I = self.s.intermediate
        rows = recv_buf[: int(cnt.sum())].numpy()
        out = np.zeros_like(rows)
        off = 0
        for src in range(self.R):
            for le in range(self.El):
                n = int(cnt[src, le])
                if n:
                    e = self.rank * self.El + le
                    out[off:off + n] = moe_ref.expert_mlp(rows[off:off + n], self.gu[e, :I], self.gu[e, I:],
                                                          self.dn[e], w4a4)
                off += n
        return torch.from_numpy(out)

    def ret_buffer(self):
        return torch.empty(self.R * 100000, self.s.hidden, dtype=torch.float32)

    def combine(self, ret, send_pos, w):
        r = ret.numpy()
        y = (w[:, :, None] * r[send_pos]).sum(axis=1, dtype=np.float32)
        return moe_ref.bf16_round(y)
