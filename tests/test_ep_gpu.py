"""EP layer with the real sm_100a kernels: two processes share cuda:0 and
exchange through gloo staged via the host (NCCL needs distinct GPUs; the box
has one). The EP result must equal the single-GPU MoELayer run on the union of
both ranks' tokens with the plan over 2 (virtual) ranks — every kernel is
row-independent, so the match is exact."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(shape_name, E, T, world, rank, device="cuda"):
    from dataclasses import replace

    from paper_2604_19503_b200.moe import SHAPES
    from paper_2604_19503_b200.workload import WorkloadSpec, make_batch, make_experts

    from paper_2604_19503_b200.workload import make_shared_expert

    shape = replace(SHAPES[shape_name], num_experts=E)
    x, mod, router, _ = make_batch(shape, WorkloadSpec(tokens=T, num_ranks=world, rank=rank), device=device)
    gu, dn = make_experts(shape, device=device)
    sh = make_shared_expert(shape, device=device)
    return shape, x, mod, router, gu, dn, sh


def _worker(rank, world, port, shape_name, E, T, strategy, fp4_dispatch, outdir, p2p=False, device_plan=False,
            rank_partial=False):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_19503_b200 import _lib
    from paper_2604_19503_b200.ep import CudaEPOps, EPComm, EPMoELayer, split_weights
    from paper_2604_19503_b200.policy import RealbParams

    shape, x, mod, router, gu, dn, sh = _setup(shape_name, E, T, world, rank)
    bias = torch.zeros(E, device="cuda") if shape.scoring == _lib.SCORE_SIGMOID_RENORM else None
    local = split_weights(shape, router, gu, dn, rank, world, shared=sh)
    ops = CudaEPOps(shape, router.contiguous(), bias, local, world, T)
    comm = EPComm(staged=True, p2p=p2p)
    if p2p:
        ops.setup_p2p(comm)
    layer = EPMoELayer(shape, comm, ops, fp4_dispatch=fp4_dispatch, rank_partial=rank_partial)
    params = RealbParams(global_batch_threshold=0)
    if device_plan:
        # host-sync-free layer: eager twice, then captured as a CUDA graph and replayed
        y0, res = layer.forward_device(x, mod, strategy, params)
        plan = res.plan
        y1, _ = layer.forward_device(x, mod, strategy, params)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            yg, _ = layer.forward_device(x, mod, strategy, params)
        for _ in range(2):
            g.replay()
        torch.cuda.synchronize()
        assert torch.equal(y0, y1) and torch.equal(yg, y0)
        y = yg
        assert int(ops.p2p_err.item()) == 0, "a peer-memory wait timed out"
        res.check()
        _dump_operands(ops, x, outdir, rank)
    else:
        y, plan, vt = layer.forward(x, mod, strategy, params)
        if p2p:  # a second layer call exercises window reuse and the epoch counters
            y, plan, vt = layer.forward(x, mod, strategy, params)
            torch.cuda.synchronize()
            assert int(ops.p2p_err.item()) == 0, "a peer-memory wait timed out"
    torch.cuda.synchronize()
    if p2p:
        dist.barrier()
        ops.close_p2p()
    np.savez(os.path.join(outdir, f"r{rank}.npz"), y=y.float().cpu().numpy(),
             acc=np.array(sorted(plan.accelerated_ranks), dtype=np.int64))
    dist.destroy_process_group()


@pytest.mark.parametrize("shape_name,E,T,strategy,fp4_dispatch", [
    ("tiny", 8, 512, "realb", False), ("kimi", 16, 384, "realb", False), ("qwen", 16, 256, "fp4all", False),
    ("kimi", 16, 384, "baseline", False),
    # NVFP4 rows on the wire to W4A4 ranks (§8f-1): sender-side K4 gives the receiver
    # the same codes it would compute itself, so the layer output is unchanged
    ("kimi", 16, 384, "realb", True), ("qwen", 16, 256, "fp4all", True), ("tiny", 8, 512, "realb", True),
    # the replicated shared expert of Kimi-VL, overlapped with the EP path
    ("kimi_shared", 16, 384, "realb", True)])
def test_ep2_on_one_gpu_equals_single_gpu_layer(tmp_path, shape_name, E, T, strategy, fp4_dispatch):
    _run_and_compare(tmp_path, shape_name, E, T, strategy, fp4_dispatch, p2p=False)


@pytest.mark.parametrize("shape_name,E,T,strategy,fp4_dispatch", [
    ("kimi", 16, 384, "realb", True), ("qwen", 16, 256, "fp4all", False), ("tiny", 8, 512, "baseline", False)])
def test_ep2_peer_memory_transport_equals_single_gpu_layer(tmp_path, shape_name, E, T, strategy, fp4_dispatch):
    """C2/C3 through CUDA-IPC peer-memory windows (realb_p2p_*: rows written into
    the peers' windows, system-scope counters, no collective on the data path);
    the two processes share one GPU, as NVLink peers would share windows."""
    _run_and_compare(tmp_path, shape_name, E, T, strategy, fp4_dispatch, p2p=True)


@pytest.mark.parametrize("shape_name,E,T,strategy,fp4_dispatch", [
    ("kimi", 16, 384, "realb", True), ("kimi", 40, 384, "realb", True), ("qwen", 16, 256, "fp4all", True),
    ("tiny", 8, 512, "baseline", True), ("kimi_shared", 16, 384, "realb", True),
    ("kimi", 16, 203, "fp4all", True)])  # ragged token count (not a multiple of the 64-token chunk)
def test_ep2_host_sync_free_layer_and_graph(tmp_path, shape_name, E, T, strategy, fp4_dispatch):
    """The host-sync-free EP layer: C1 through peer memory, plan and window offsets
    derived on the device, both precisions launched and selected by device-side
    group lists; eager == CUDA-graph replay == the single-GPU layer, exactly."""
    _run_and_compare(tmp_path, shape_name, E, T, strategy, fp4_dispatch, p2p=True, device_plan=True)


@pytest.mark.parametrize("world,shape_name,E,T,strategy,fp4_dispatch", [
    (4, "kimi", 16, 256, "realb", True), (4, "qwen", 32, 192, "fp4all", True)])
def test_ep4_host_sync_free_layer_and_graph(tmp_path, world, shape_name, E, T, strategy, fp4_dispatch):
    """The host-sync-free peer-memory layer with FOUR ranks (processes sharing one
    GPU): plan over 4 ranks, window offsets for 4 sources, direct dispatch and the
    fused return into 4 windows; eager == graph replay == the single-GPU layer."""
    _run_and_compare(tmp_path, shape_name, E, T, strategy, fp4_dispatch, p2p=True, device_plan=True, world=world)


@pytest.mark.parametrize("strategy", ["fp4all", "baseline"])
def test_ep1_host_sync_free_layer_own_windows(tmp_path, strategy):
    """Degenerate EP (one rank, its own windows only): every peer-memory kernel in
    one process (also the configuration scripts/exp/ep1_selfcheck.py runs under
    compute-sanitizer); equals the single-GPU layer."""
    _run_and_compare(tmp_path, "kimi", 16, 333, strategy, True, p2p=True, device_plan=True, world=1)


@pytest.mark.parametrize("world,shape_name,E,T,strategy", [
    (2, "kimi", 16, 384, "realb"), (2, "qwen", 16, 256, "fp4all"), (2, "kimi_shared", 16, 384, "realb"),
    (2, "kimi", 16, 203, "fp4all"), (4, "kimi", 16, 256, "realb"), (2, "tiny", 8, 512, "baseline")])
def test_ep_rank_partial_return_host_sync_free(tmp_path, world, shape_name, E, T, strategy):
    """Rank-partial return (realb_p2p_pack_direct_partial -> local K6 down ->
    realb_p2p_partial_return -> realb_combine_partial): a W4A4 owner sends ONE bf16
    partial row per (token, owner). Equal, bit for bit, to the single-GPU layer with the
    same arithmetic (MoELayer.rank_partial), eager and as a CUDA graph, and within the
    layer bar of the oracle's emulation of the rule."""
    _run_and_compare(tmp_path, shape_name, E, T, strategy, True, p2p=True, device_plan=True, world=world,
                     rank_partial=True)


@pytest.mark.parametrize("p2p", [False, True])
def test_ep_rank_partial_collective_path(tmp_path, p2p):
    """The host-plan EP paths (collective all-to-alls / peer-memory windows) with the
    rank-partial arithmetic formed at the source from every slot's returned row: equal to
    the single-GPU layer (and so to the host-sync-free path, which the bench checks)."""
    _run_and_compare(tmp_path, "kimi", 16, 384, "realb", True, p2p=p2p, world=2, rank_partial=True)


def test_device_plan_layer_rejects_bf16_dispatch():
    """The host-sync-free layer always sends NVFP4 rows to W4A4 owners; asking it
    for bf16 dispatch is an error (not a silently different measurement)."""
    from paper_2604_19503_b200.ep import EPMoELayer
    from paper_2604_19503_b200.moe import SHAPES

    class _Comm:
        world, rank, p2p = 2, 0, True

    class _Ops:
        def forward_device(self, *a):
            raise AssertionError("must not run")

    layer = EPMoELayer(SHAPES["tiny"], _Comm(), _Ops(), fp4_dispatch=False)
    with pytest.raises(ValueError, match="NVFP4"):
        layer.forward_device(None, None, "realb")


def _dump_operands(ops, x, outdir, rank):
    """What direct dispatch wrote into THIS rank's GEMM operand windows (valid
    grouped rows only), with the row map back to (source rank, send-order row),
    plus this rank's own tokens and send positions: the parent process checks
    every received row against the oracle (K4 bit-exactness on the wire)."""
    from paper_2604_19503_b200.ep import _device_view
    from paper_2604_19503_b200.quant import sf_mma_to_flat

    H, rc, El = ops.H, ops.rows_cap, ops.El
    r = ops.p2p_rank
    torch.cuda.synchronize()
    lay = ops.local_layout.cpu().numpy()
    starts, counts = lay[8:8 + El].astype(np.int64), lay[8 + El:8 + 2 * El].astype(np.int64)
    g = np.concatenate([s + np.arange(c) for s, c in zip(starts, counts)]) if counts.sum() else np.zeros(0, np.int64)
    gt = torch.from_numpy(g).cuda()
    opa = _device_view(ops.p2p["opa"][r], rc * H, torch.bfloat16).view(rc, H)
    opc = _device_view(ops.p2p["opc"][r], rc * H // 2, torch.uint8).view(rc, H // 2)
    ops_mma = _device_view(ops.p2p["ops"][r], rc * H // 16, torch.uint8).cpu().numpy()
    np.savez(os.path.join(outdir, f"ops{rank}.npz"), g=g, row_map=ops.row_map[gt].cpu().numpy(),
             a=opa[gt].view(torch.int16).cpu().numpy(), codes=opc[gt].cpu().numpy(),
             sf=sf_mma_to_flat(ops_mma, rc, H)[g], w4a4=ops.prec_local.cpu().numpy(),
             x=x.view(torch.int16).cpu().numpy(), send_pos=ops.send_pos[:x.shape[0]].cpu().numpy())


def _check_direct_dispatch_operands(tmp_path, world):
    """Every row direct dispatch placed in an owner's operand is its source token:
    bf16 bits equal for a W16A16 owner; for a W4A4 owner the NVFP4 codes and the
    scales (after realb_sf_rows_to_mma) equal oracle.quantize_bf16 of the token's
    bf16 row (the reference block rule, fp4.py:173-227), bit for bit."""
    import oracle

    d = [np.load(tmp_path / f"ops{r}.npz") for r in range(world)]
    inv, oq = [], []
    for s in range(world):
        sp = d[s]["send_pos"]
        iv = np.full(sp.size, -1, np.int64)
        iv[sp.reshape(-1)] = np.repeat(np.arange(sp.shape[0]), sp.shape[1])
        inv.append(iv)
        oq.append(oracle.quantize_bf16(d[s]["x"].view(np.uint16)))
    checked = 0
    for r in range(world):
        m = d[r]["row_map"].astype(np.int64)
        src, row = m >> 25, m & ((1 << 25) - 1)
        w4a4 = bool(d[r]["w4a4"].any())
        for s in range(world):
            sel = src == s
            tok = inv[s][row[sel]]
            assert (tok >= 0).all()
            if w4a4:
                assert (d[r]["codes"][sel] == oq[s][0][tok]).all(), (r, s)
                assert (d[r]["sf"][sel] == oq[s][1][tok]).all(), (r, s)
            else:
                assert (d[r]["a"][sel] == d[s]["x"][tok]).all(), (r, s)
            checked += int(sel.sum())
    assert checked > 0


def _run_and_compare(tmp_path, shape_name, E, T, strategy, fp4_dispatch, p2p, device_plan=False, world=2,
                     rank_partial=False):
    mp.spawn(_worker, args=(world, _free_port(), shape_name, E, T, strategy, fp4_dispatch, str(tmp_path), p2p,
                            device_plan, rank_partial), nprocs=world)
    from paper_2604_19503_b200 import _lib
    from paper_2604_19503_b200.moe import MoELayer, MoEWeights
    from paper_2604_19503_b200.policy import ClusterConfig, RealbParams

    parts = [_setup(shape_name, E, T, world, r) for r in range(world)]
    shape, _, _, router, gu, dn, sh = parts[0]
    x = torch.cat([p[1] for p in parts])
    mod = torch.cat([p[2] for p in parts])
    bias = torch.zeros(E, device="cuda") if shape.scoring == _lib.SCORE_SIGMOID_RENORM else None
    single = MoELayer(MoEWeights.from_hf(shape, router, gu, dn, bias=bias, shared=sh), max_tokens=world * T,
                      cluster=ClusterConfig(world, 1, E // world, 1, shape.modality_isolated))
    single.rank_partial = rank_partial
    res = single.forward(x, mod, strategy, RealbParams(global_batch_threshold=0))
    ref = res.y.float().cpu().numpy()
    r = [np.load(tmp_path / f"r{i}.npz") for i in range(world)]
    y = np.concatenate([a["y"] for a in r])
    assert list(r[0]["acc"]) == sorted(res.plan.accelerated_ranks)
    np.testing.assert_array_equal(y, ref)
    # and the EP layer against the CPU oracle directly (same plan, the device logits)
    from oracle import moe_ref

    prec = res.plan.expert_precision(single.placement)
    oref = moe_ref.moe_layer(x.float().cpu().numpy(), mod.cpu().numpy(), router.float().cpu().numpy(),
                             gu.float().cpu().numpy(), dn.float().cpu().numpy(), shape.top_k, shape.scoring,
                             expert_prec=prec, routed_scaling=shape.routed_scaling,
                             logits=single.logits[:world * T].cpu().numpy(),
                             shared=None if sh is None else (sh[0].float().cpu().numpy(), sh[1].float().cpu().numpy()),
                             partial_el=(E // world) if rank_partial else None)
    assert (single.topk_idx[:world * T].cpu().numpy() == oref["idx"]).all()
    err = float(np.linalg.norm(y - oref["y"]) / np.linalg.norm(oref["y"]))
    bar = 1e-3 if (strategy == "fp4all" and sh is None) else 2e-3  # tests/test_layer_gpu.py BAR
    assert err < bar, err
    if device_plan:
        _check_direct_dispatch_operands(tmp_path, world)


def _setup_fail_worker(rank, world, port, outdir):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), REALB_TEST_P2P_FAIL_RANK="1")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_19503_b200.ep import CudaEPOps, EPComm, split_weights

    shape, x, mod, router, gu, dn, sh = _setup("kimi", 16, 128, world, rank)
    ops = CudaEPOps(shape, router.contiguous(), None, split_weights(shape, router, gu, dn, rank, world), world, 128)
    raised = ""
    try:
        ops.setup_p2p(EPComm(staged=True, p2p=True))
    except RuntimeError as e:
        raised = str(e)
    dist.barrier()  # both ranks got here: nobody was left inside a collective
    open(os.path.join(outdir, f"r{rank}.txt"), "w").write(raised)
    dist.destroy_process_group()


def test_p2p_setup_failure_is_agreed_by_all_ranks(tmp_path):
    """A peer-memory setup failure on ONE rank (fault injection) makes every rank
    raise, so the bench's auto transport falls back to the collective path on all
    ranks together instead of leaving the healthy ranks blocked in a collective."""
    mp.spawn(_setup_fail_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2)
    msgs = [(tmp_path / f"r{r}.txt").read_text() for r in range(2)]
    assert all("allocation failed" in m for m in msgs), msgs
