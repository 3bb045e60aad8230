"""Tensor-parallel host logic on CPU with the gloo backend, world size 2 (no GPU needed).

The per-rank GEMM is the oracle (test infrastructure); what is under test is the product's
sharding (paper_2402_10076_b200.tp) and the collective pattern: column shards + all-gather +
column permutation must reproduce the full result bit for bit, row shards + fp32 all-reduce
within fp64 rounding; and fp16 partial sums would break the tolerance.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2402_10076_b200 import tp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def run_world(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(60)
    return out


def _column_parallel(rank, world):
    p = synth.make_problem(21, M=6, N=512, K=512, G=128)
    qw, sc, zr = tp.shard_awq_columns(p.qweight, p.scales, p.zeros, rank, world)
    y_r = oracle.round_fp16(oracle.w4a16_reference(p.x, qw, sc, zr, 128))       # this rank's [M][N/P]
    gathered = torch.empty((world,) + y_r.shape, dtype=torch.float16)
    dist.all_gather_into_tensor(gathered.view(-1), torch.from_numpy(y_r).view(-1))
    # the permutation quick_gather_columns performs on the GPU: [P][M][Nr] -> [M][P*Nr]
    y = gathered.permute(1, 0, 2).reshape(p.M, -1).numpy()
    ref = oracle.round_fp16(oracle.w4a16_reference(p.x, p.qweight, p.scales, p.zeros, 128))
    return bool(np.array_equal(y.view(np.uint16), ref.view(np.uint16)))


def _row_parallel(rank, world):
    p = synth.make_problem(22, M=5, N=256, K=1024, G=128)
    qw, sc, zr = tp.shard_awq_rows(p.qweight, p.scales, p.zeros, 128, rank, world)
    k0, k1 = tp.row_shard_bounds(1024, 128, world, rank)
    part = torch.from_numpy(oracle.w4a16_reference(p.x[:, k0:k1], qw, sc, zr, 128))
    dist.all_reduce(part, op=dist.ReduceOp.SUM)
    ref = oracle.w4a16_reference(p.x, p.qweight, p.scales, p.zeros, 128)
    return float(np.max(np.abs(part.numpy() - ref)))


def test_column_parallel_gloo_world2_bit_exact():
    res = run_world(_column_parallel)
    assert res == {0: True, 1: True}, res


def test_row_parallel_gloo_world2():
    res = run_world(_row_parallel)
    assert all(isinstance(v, float) and v < 1e-12 for v in res.values()), res


def test_shards_reassemble_exactly():
    p = synth.make_problem(3, M=1, N=1024, K=1024, G=128)
    for world in (2, 4, 8):
        cols = [tp.shard_awq_columns(p.qweight, p.scales, p.zeros, r, world) for r in range(world)]
        assert np.array_equal(np.concatenate([c[0] for c in cols], axis=1), p.qweight)
        assert np.array_equal(np.concatenate([c[1] for c in cols], axis=1).view(np.uint16), p.scales.view(np.uint16))
        assert np.array_equal(np.concatenate([c[2] for c in cols], axis=1), p.zeros)
        rows = [tp.shard_awq_rows(p.qweight, p.scales, p.zeros, 128, r, world) for r in range(world)]
        assert np.array_equal(np.concatenate([r_[0] for r_ in rows], axis=0), p.qweight)
        assert np.array_equal(np.concatenate([r_[2] for r_ in rows], axis=0), p.zeros)


def test_shard_alignment_rules():
    # Llama-2-13B MLP at P = 8: N/P = 1728 is not a multiple of 128; K/P = 13.5 groups
    with pytest.raises(ValueError):
        tp.column_shard_bounds(13824, 8, 0)
    with pytest.raises(ValueError):
        tp.row_shard_bounds(13824, 128, 8, 0)
    # every multi-GPU BASELINE config shards cleanly at P = 2, 4, 8
    for P in (2, 4, 8):
        for N in (28672, 8192, 6144, 4096):
            tp.column_shard_bounds(N, P, P - 1)
        for K in (28672, 14336, 4096, 8192):
            tp.row_shard_bounds(K, 128, P, P - 1)


def test_fp16_partials_would_break_the_tolerance():
    """Why the row-parallel all-reduce carries fp32: rounding each of
    8 K-shard partials to fp16 before summing fails the north-star tolerance at K = 28672."""
    p = synth.make_problem(5, M=16, N=128, K=28672, G=128)
    ref = oracle.w4a16_reference(p.x, p.qweight, p.scales, p.zeros, 128)
    parts = [oracle.w4a16_reference(p.x[:, k0:k0 + 3584], *tp.shard_awq_rows(p.qweight, p.scales, p.zeros, 128, r, 8), 128)
             for r, k0 in enumerate(range(0, 28672, 3584))]
    y16 = sum(oracle.round_fp16(pp).astype(np.float64) for pp in parts)
    y32 = sum(pp.astype(np.float32).astype(np.float64) for pp in parts)
    assert not oracle.tol_check(y16, ref)["ok"]
    assert oracle.tol_check(y32, ref)["ok"]


# ------------------------------------------------------------------ Megatron semantic slicing (configs[4])
def test_qkv_shard_keeps_whole_heads():
    """Scales encode the column index, so the shard's columns can be read back: rank r holds query
    heads [r nh/P, (r+1) nh/P), then its key heads, then its value heads (Mistral-7B ratio 4:1)."""
    nh, nkv, hd, K, G = 8, 2, 128, 256, 128
    N = (nh + 2 * nkv) * hd
    p = synth.make_problem(7, M=1, N=N, K=K, G=G)
    scales = np.tile(np.arange(N, dtype=np.float16)[None, :], (K // G, 1))   # exact up to 2048
    for world in (1, 2):
        cols = []
        for r in range(world):
            qw, sc, zr = tp.shard_qkv_columns(p.qweight, scales, p.zeros, nh, nkv, hd, r, world)
            got = sc[0].astype(np.int64)
            hq, hk = nh // world, nkv // world
            want = np.concatenate([np.arange(r * hq * hd, (r + 1) * hq * hd),
                                   nh * hd + np.arange(r * hk * hd, (r + 1) * hk * hd),
                                   (nh + nkv) * hd + np.arange(r * hk * hd, (r + 1) * hk * hd)])
            assert np.array_equal(got, want)
            codes = oracle.unpack_awq(qw)
            assert np.array_equal(codes, oracle.unpack_awq(p.qweight)[:, want])
            assert np.array_equal(oracle.unpack_awq(zr), oracle.unpack_awq(p.zeros)[:, want])
            cols.append(want)
        assert np.array_equal(np.sort(np.concatenate(cols)), np.arange(N))
    with pytest.raises(ValueError):
        tp.shard_qkv_columns(p.qweight, scales, p.zeros, nh, nkv, hd, 0, 4)   # 2 kv heads over 4 ranks


def _mlp_tp(rank, world):
    """Megatron MLP on CPU (oracle GEMMs): each rank's fused gate||up slice feeds its down rows
    directly; the fp32 all-reduce of the down partials equals the full MLP."""
    K, I, G = 512, 256, 128
    pg = synth.make_problem(31, M=4, N=I, K=K, G=G)
    pu = synth.make_problem(32, M=4, N=I, K=K, G=G)
    pdn = synth.make_problem(33, M=4, N=K, K=I, G=G)
    g_r, u_r = tp.shard_gate_up((pg.qweight, pg.scales, pg.zeros), (pu.qweight, pu.scales, pu.zeros), rank, world)
    h_r = oracle.round_fp16(oracle.silu_mul(oracle.w4a16_reference(pg.x, *g_r, G), oracle.w4a16_reference(pg.x, *u_r, G)))
    d_r = tp.shard_awq_rows(pdn.qweight, pdn.scales, pdn.zeros, G, rank, world)
    part = torch.from_numpy(oracle.w4a16_reference(h_r, *d_r, G))
    dist.all_reduce(part, op=dist.ReduceOp.SUM)
    h = oracle.round_fp16(oracle.silu_mul(oracle.w4a16_reference(pg.x, pg.qweight, pg.scales, pg.zeros, G),
                                          oracle.w4a16_reference(pg.x, pu.qweight, pu.scales, pu.zeros, G)))
    ref = oracle.w4a16_reference(h, pdn.qweight, pdn.scales, pdn.zeros, G)
    return float(np.max(np.abs(part.numpy() - ref)))


def test_megatron_mlp_slicing_gloo_world2():
    res = run_world(_mlp_tp)
    assert all(isinstance(v, float) and v < 1e-9 for v in res.values()), res
