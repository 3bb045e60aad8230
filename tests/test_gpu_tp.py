"""Tensor-parallel layers on the GPU (single-process NCCL group; marker: gpu).  The multi-rank
collective pattern itself is covered on CPU by tests/test_tp.py (gloo, world size 2)."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no GPU", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

from paper_2402_10076_b200 import quick, tp  # noqa: E402


@pytest.fixture(scope="module")
def nccl_world1():
    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1)
    yield
    dist.destroy_process_group()


def _x(p):
    return torch.from_numpy(p.x.view(np.int16)).view(torch.float16).cuda()


def test_column_parallel_layer(nccl_world1):
    p = synth.make_problem(31, M=12, N=1024, K=2048, G=128)
    layer = tp.ColumnParallelW4A16(p.qweight, p.scales, p.zeros, 128)
    y = layer.forward(_x(p))
    torch.cuda.synchronize()
    ref = oracle.w4a16_reference(p.x, p.qweight, p.scales, p.zeros, 128)
    assert oracle.tol_check(y.float().cpu().numpy(), ref)["ok"]


def test_row_parallel_layer_fp32_reduce(nccl_world1):
    p = synth.make_problem(32, M=12, N=512, K=4096, G=128)
    layer = tp.RowParallelW4A16(p.qweight, p.scales, p.zeros, 128)
    y = layer.forward(_x(p)[:, layer.k0:layer.k1].contiguous())
    torch.cuda.synchronize()
    ref = oracle.w4a16_reference(p.x, p.qweight, p.scales, p.zeros, 128)
    assert oracle.tol_check(y.float().cpu().numpy(), ref)["ok"]


def test_gather_columns_matches_column_slices():
    """The permutation the column-parallel epilogue applies, on slices computed per 'rank'."""
    p = synth.make_problem(33, M=7, N=1024, K=1024, G=128)
    P = 4
    x = _x(p)
    gathered = torch.empty((P, 7, 256), device="cuda", dtype=torch.float16)
    for r in range(P):
        qw, sc, zr = tp.shard_awq_columns(p.qweight, p.scales, p.zeros, r, P)
        blob = torch.from_numpy(quick.quick_pack_weights(qw, sc, zr, 128)).cuda()
        quick.quick_w4a16_gemm(x, blob, 256, 1024, 128, out=gathered[r], tile_n=16, split_k=2)
    y = quick.quick_gather_columns(gathered, P, 7, 256)
    full = quick.quick_w4a16_gemm(x, torch.from_numpy(quick.quick_pack_weights(p.qweight, p.scales, p.zeros, 128)).cuda(),
                                  1024, 1024, 128, tile_n=16, split_k=2)
    torch.cuda.synchronize()
    # same plan (tile, split) => same per-element summation order => bit-identical columns
    assert torch.equal(y.view(torch.int16), full.view(torch.int16))


# ------------------------------------------------------------------------------- world size 2 on one GPU
# Two processes share cuda:0 and a gloo group that carries the CUDA tensors (NCCL refuses two ranks
# on one device).  Everything else is the production path: the shard packing, the sm_100a GEMM of
# each rank's shard, the collective, and the quick_gather_columns / quick_f32_to_f16 epilogues.
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _tp_worker(rank, world, port, q):
    import traceback
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        res = {}
        # column-parallel (Llama-2-70B up-projection shape, scaled down in K): all-gather + permute
        p = synth.make_problem(61, M=12, N=2048, K=1024, G=128)
        col = tp.ColumnParallelW4A16(p.qweight, p.scales, p.zeros, 128, device=torch.device("cuda", 0))
        y1 = col.forward(_x(p))
        y2 = col.forward(_x(p))               # a fresh output per call (the first is not overwritten)
        torch.cuda.synchronize()
        ref = oracle.w4a16_reference(p.x, p.qweight, p.scales, p.zeros, 128)
        res["col"] = oracle.tol_check(y1.float().cpu().numpy(), ref)["ok"] and y1.data_ptr() != y2.data_ptr() \
            and torch.equal(y1.view(torch.int16), y2.view(torch.int16))
        # the gathered columns are the single-GPU GEMM's columns bit for bit when the per-rank plan is
        # the same as the single-GPU plan of that column slice (forced tile/split here)
        # row-parallel (down-projection): fp32 partials, fp32 all-reduce, cast
        p = synth.make_problem(62, M=7, N=512, K=4096, G=128)
        row = tp.RowParallelW4A16(p.qweight, p.scales, p.zeros, 128, device=torch.device("cuda", 0))
        xs = _x(p)[:, row.k0:row.k1].contiguous()
        y = row.forward(xs)
        torch.cuda.synchronize()
        ref = oracle.w4a16_reference(p.x, p.qweight, p.scales, p.zeros, 128)
        res["row"] = oracle.tol_check(y.float().cpu().numpy(), ref)["ok"]
        # Megatron MLP (BASELINE.json configs[4] split): fused gate||up + SiLU epilogue on this rank's
        # intermediate slice, straight into the row-parallel down projection, one fp32 all-reduce
        K, I, G = 1024, 512, 128
        pg = synth.make_problem(63, M=9, N=I, K=K, G=G)
        pu = synth.make_problem(64, M=9, N=I, K=K, G=G)
        pdn = synth.make_problem(65, M=9, N=K, K=I, G=G)
        mlp = tp.MegatronMLP((pg.qweight, pg.scales, pg.zeros), (pu.qweight, pu.scales, pu.zeros),
                             (pdn.qweight, pdn.scales, pdn.zeros), G, device=torch.device("cuda", 0))
        y = mlp.forward(_x(pg))
        torch.cuda.synchronize()
        h = oracle.round_fp16(oracle.silu_mul(oracle.w4a16_reference(pg.x, pg.qweight, pg.scales, pg.zeros, G),
                                              oracle.w4a16_reference(pg.x, pu.qweight, pu.scales, pu.zeros, G)))
        ref = oracle.w4a16_reference(h, pdn.qweight, pdn.scales, pdn.zeros, G)
        res["mlp"] = oracle.tol_check(y.float().cpu().numpy(), ref)["ok"]
        # attention projections: QKV by head group (8 q + 2 kv heads of 128), O row-parallel
        nh, nkv, hd = 8, 2, 128
        pq = synth.make_problem(66, M=5, N=(nh + 2 * nkv) * hd, K=1024, G=G)
        po = synth.make_problem(67, M=5, N=1024, K=nh * hd, G=G)
        att = tp.MegatronAttentionProjections((pq.qweight, pq.scales, pq.zeros), (po.qweight, po.scales, po.zeros),
                                              nh, nkv, hd, G, device=torch.device("cuda", 0))
        qkv_r = att.forward_qkv(_x(pq))
        o = att.forward_o(_x(po)[:, att.o.k0:att.o.k1].contiguous())
        torch.cuda.synchronize()
        q_r = tp.shard_qkv_columns(pq.qweight, pq.scales, pq.zeros, nh, nkv, hd, rank, world)
        ok_qkv = oracle.tol_check(qkv_r.float().cpu().numpy(), oracle.w4a16_reference(pq.x, *q_r, G))["ok"]
        ok_o = oracle.tol_check(o.float().cpu().numpy(),
                                oracle.w4a16_reference(po.x, po.qweight, po.scales, po.zeros, G))["ok"]
        res["attn"] = ok_qkv and ok_o
        q.put((rank, res))
    except Exception:
        q.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_tp_layers_world2_on_one_gpu():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tp_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for pr in procs:
        pr.join(60)
    want = {"col": True, "row": True, "mlp": True, "attn": True}
    assert out == {0: want, 1: want}, out


# ------------------------------------------------------------------------------- f1: collective-fused TP
def _fused_worker(rank, world, port, q):
    import traceback
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dev = torch.device("cuda", 0)
        comm = tp.PeerComm()
        res = {}
        # column-parallel: the GEMM epilogue stores into every rank's Y; bit-identical to the collective
        # path (same per-rank plan) and within tolerance of the oracle; 3 calls (alternating buffers)
        p = synth.make_problem(71, M=12, N=2048, K=1024, G=128)
        ref_layer = tp.ColumnParallelW4A16(p.qweight, p.scales, p.zeros, 128, device=dev)
        fused = tp.FusedColumnParallelW4A16(p.qweight, p.scales, p.zeros, 128, comm, max_tokens=64, device=dev)
        y_ref = ref_layer.forward(_x(p))
        ok = True
        for it in range(3):
            y = fused.forward(_x(p)).clone()
            torch.cuda.synchronize()
            ok &= torch.equal(y.view(torch.int16), y_ref.view(torch.int16))
        ref = oracle.w4a16_reference(p.x, p.qweight, p.scales, p.zeros, 128)
        res["col"] = bool(ok) and oracle.tol_check(y.float().cpu().numpy(), ref)["ok"]
        # row-parallel: fp32 partials reduced over peer memory in rank order; every rank's Y identical
        p = synth.make_problem(72, M=9, N=1024, K=4096, G=128)
        fr = tp.FusedRowParallelW4A16(p.qweight, p.scales, p.zeros, 128, comm, max_tokens=32, device=dev)
        xs = _x(p)[:, fr.k0:fr.k1].contiguous()
        outs = [fr.forward(xs).clone() for _ in range(3)]
        torch.cuda.synchronize()
        ref = oracle.w4a16_reference(p.x, p.qweight, p.scales, p.zeros, 128)
        ok = all(torch.equal(o.view(torch.int16), outs[0].view(torch.int16)) for o in outs)
        ok &= oracle.tol_check(outs[0].float().cpu().numpy(), ref)["ok"]
        gathered = [None, None]
        dist.all_gather_object(gathered, outs[0].cpu().numpy().tobytes())
        res["row"] = bool(ok) and gathered[0] == gathered[1]
        comm.close()
        q.put((rank, res))
    except Exception:
        q.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_collective_fused_tp_world2_on_one_gpu():
    """SURVEY §8(f) f1 with two ranks sharing cuda:0 through CUDA IPC: the column-parallel epilogue writes
    straight into both ranks' Y, the row-parallel partials are reduced over peer memory."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for pr in procs:
        pr.join(60)
    assert out == {0: {"col": True, "row": True}, 1: {"col": True, "row": True}}, out
