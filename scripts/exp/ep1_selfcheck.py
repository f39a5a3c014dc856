"""The host-sync-free peer-memory EP layer with ONE rank (its own windows only):
a single process that runs every peer-memory kernel (publish, plan offsets, direct
dispatch, scale conversion, fused-return GEMMs, signals / waits), for running
under compute-sanitizer. Checked against the single-GPU layer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import torch.distributed as dist

os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29577")
torch.cuda.set_device(0)
dist.init_process_group("gloo", rank=0, world_size=1)
from dataclasses import replace
from paper_2604_19503_b200 import _lib
from paper_2604_19503_b200.ep import CudaEPOps, EPComm, EPMoELayer, split_weights
from paper_2604_19503_b200.moe import SHAPES, MoELayer, MoEWeights
from paper_2604_19503_b200.policy import ClusterConfig, RealbParams
from paper_2604_19503_b200.workload import WorkloadSpec, make_batch, make_experts

for strategy in ("fp4all", "baseline"):
    shape = replace(SHAPES["kimi"], num_experts=16)
    T = 333
    x, mod, router, _ = make_batch(shape, WorkloadSpec(tokens=T, num_ranks=1, rank=0))
    gu, dn = make_experts(shape)
    local = split_weights(shape, router, gu, dn, 0, 1)
    ops = CudaEPOps(shape, router.contiguous(), None, local, 1, T)
    comm = EPComm(staged=True, p2p=True)
    ops.setup_p2p(comm)
    layer = EPMoELayer(shape, comm, ops, fp4_dispatch=True)
    params = RealbParams(global_batch_threshold=0)
    y, _ = layer.forward_device(x, mod, strategy, params)
    torch.cuda.synchronize()
    single = MoELayer(MoEWeights.from_hf(shape, router, gu, dn), max_tokens=T,
                      cluster=ClusterConfig(1, 1, 16, 1, False))
    ref = single.forward(x, mod, strategy, params).y
    torch.cuda.synchronize()
    print(strategy, "equal:", bool(torch.equal(y, ref)), "wait error:", int(ops.p2p_err.item()))
    ops.close_p2p()
dist.destroy_process_group()
