"""EP host orchestration under gloo, world_size 2 (CPU): the expert-parallel
layer (C1 count all_gather, global plan, packed all_to_all_v dispatch, local
expert MLPs, all_to_all_v return, combine) equals the single-process oracle
layer on the union of both ranks' tokens with the same plan."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shape_name, strategy, T, outdir):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from ep_oracle_ops import OracleEPOps
    from paper_2604_19503_b200.ep import EPComm, EPMoELayer
    from paper_2604_19503_b200.moe import SHAPES
    from paper_2604_19503_b200.policy import RealbParams
    from paper_2604_19503_b200.workload import WorkloadSpec, make_batch, make_experts
    from dataclasses import replace

    shape = replace(SHAPES[shape_name], num_experts=16) if shape_name != "tiny" else SHAPES["tiny"]
    x, mod, router, _ = make_batch(shape, WorkloadSpec(tokens=T, num_ranks=world, rank=rank), device="cpu")
    gu, dn = make_experts(shape, device="cpu")
    ops = OracleEPOps(shape, router.float().numpy(), gu.float().numpy(), dn.float().numpy(), rank, world)
    layer = EPMoELayer(shape, EPComm(), ops)
    y, plan, vt_all = layer.forward(x, mod, strategy, RealbParams(global_batch_threshold=0))
    np.savez(os.path.join(outdir, f"r{rank}.npz"), y=y, x=x.float().numpy(), mod=mod.numpy(),
             prec=plan.expert_precision(__import__("paper_2604_19503_b200.policy", fromlist=["x"]).place_experts_static(layer.cluster)),
             vt=vt_all)
    dist.destroy_process_group()


@pytest.mark.parametrize("shape_name,strategy", [("tiny", "realb"), ("tiny", "fp4all"), ("kimi", "realb")])
def test_ep_world2_matches_single_process_oracle(tmp_path, shape_name, strategy):
    world, T = 2, 256
    mp.spawn(_worker, args=(world, _free_port(), shape_name, strategy, T, str(tmp_path)), nprocs=world)
    from dataclasses import replace

    from oracle import moe_ref
    from paper_2604_19503_b200.moe import SHAPES
    from paper_2604_19503_b200.workload import WorkloadSpec, make_batch, make_experts

    shape = replace(SHAPES[shape_name], num_experts=16) if shape_name != "tiny" else SHAPES["tiny"]
    r = [np.load(tmp_path / f"r{i}.npz") for i in range(world)]
    assert (r[0]["prec"] == r[1]["prec"]).all() and (r[0]["vt"] == r[1]["vt"]).all()
    x = np.concatenate([a["x"] for a in r])
    mod = np.concatenate([a["mod"] for a in r])
    _, _, router, _ = make_batch(shape, WorkloadSpec(tokens=T, num_ranks=world, rank=0), device="cpu")
    gu, dn = make_experts(shape, device="cpu")
    ref = moe_ref.moe_layer(x, mod, router.float().numpy(), gu.float().numpy(), dn.float().numpy(),
                            shape.top_k, shape.scoring, expert_prec=r[0]["prec"],
                            routed_scaling=shape.routed_scaling)
    y = np.concatenate([a["y"] for a in r])
    np.testing.assert_allclose(y, ref["y"], rtol=2e-2, atol=1e-3)
    assert np.linalg.norm(y - ref["y"]) / np.linalg.norm(ref["y"]) < 1e-3
    if strategy == "fp4all":
        assert r[0]["prec"].all()
