"""Tensor-parallel W4A16 linear layers over NCCL (BASELINE.json north_star (4)).

Two partitions of Y = X . dequant(Wq), one process per GPU, torch.distributed for plumbing:

  column-parallel  rank r owns output columns [r N/P, (r+1) N/P) (a multiple of 128): its
                   AWQ slices are packed with quick_pack_weights, it computes Y_r [M, N/P] with
                   quick_w4a16_gemm straight into its slot of a [P][M][N/P] buffer, an
                   in-place NCCL all-gather fills the other slots, and quick_gather_columns
                   permutes [P][M][N/P] -> [M][N].  No arithmetic crosses ranks.
  row-parallel     rank r owns reduction rows [r K/P, (r+1) K/P) (a multiple of G and 64): it
                   computes the un-rounded fp32 partial Y_r = X[:, K_r] . W[K_r, :] with
                   QUICK_FLAG_OUT_F32, NCCL all-reduce(sum) in fp32 (fp16 partials fail the
                   tolerance), then quick_f32_to_f16.

The shard functions are pure host code (numpy) and exact: concatenating the shards gives the
input tensors back bit for bit (tests/test_tp.py, gloo, world size 2).
"""
import numpy as np


# ----------------------------------------------------------------------------------- sharding
def column_shard_bounds(N: int, world: int, rank: int):
    if N % (128 * world):
        raise ValueError(f"N={N} is not a multiple of 128 x world ({world}): no v1 column shard")
    n_r = N // world
    return rank * n_r, (rank + 1) * n_r


def row_shard_bounds(K: int, G: int, world: int, rank: int):
    unit = int(np.lcm(G, 64))
    if K % (unit * world):
        raise ValueError(f"K={K} is not a multiple of lcm(G, 64) x world = {unit * world}: no row shard")
    k_r = K // world
    return rank * k_r, (rank + 1) * k_r


def shard_awq_columns(qweight, scales, zeros, rank: int, world: int):
    """Column (N) shard of AWQ tensors: qweight [K][N/8], scales [K/G][N], zeros [K/G][N/8]."""
    N = scales.shape[1]
    c0, c1 = column_shard_bounds(N, world, rank)
    return (np.ascontiguousarray(qweight[:, c0 // 8:c1 // 8]), np.ascontiguousarray(scales[:, c0:c1]),
            np.ascontiguousarray(zeros[:, c0 // 8:c1 // 8]))


def shard_awq_rows(qweight, scales, zeros, G: int, rank: int, world: int):
    """Row (K) shard of AWQ tensors; the shard boundary is a group boundary."""
    K = qweight.shape[0]
    k0, k1 = row_shard_bounds(K, G, world, rank)
    return (np.ascontiguousarray(qweight[k0:k1]), np.ascontiguousarray(scales[k0 // G:k1 // G]),
            np.ascontiguousarray(zeros[k0 // G:k1 // G]))


# ----------------------------------------------------------------------------------- layers
class ColumnParallelW4A16:
    """Y[M, N] = X[M, K] . dequant(Wq)[K, N], N split across the process group."""

    def __init__(self, qweight, scales, zeros, group_size: int, group=None, device=None):
        import torch
        import torch.distributed as dist
        from . import quick
        self.quick, self.dist, self.torch = quick, dist, torch
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.K, self.N, self.G = qweight.shape[0], scales.shape[1], group_size
        self.Nr = self.N // self.world
        qw, sc, zr = shard_awq_columns(qweight, scales, zeros, self.rank, self.world)
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.packed = torch.from_numpy(quick.quick_pack_weights(qw, sc, zr, group_size)).to(self.device)
        self._gathered = {}   # internal [P][M][N/P] all-gather buffers per M (never returned)
        self.workspace = None

    def forward(self, x, out=None):
        """A fresh output tensor per call unless `out` is given."""
        t = self.torch
        M = x.shape[0]
        if self.world == 1:
            return self.quick.quick_w4a16_gemm(x, self.packed, self.N, self.K, self.G, out=out,
                                               workspace=self.workspace)
        if M not in self._gathered:
            self._gathered[M] = t.empty((self.world, M, self.Nr), device=self.device, dtype=t.float16)
        gathered = self._gathered[M]
        y = out if out is not None else t.empty((M, self.N), device=self.device, dtype=t.float16)
        local = gathered[self.rank]                     # compute straight into our slot
        self.quick.quick_w4a16_gemm(x, self.packed, self.Nr, self.K, self.G, out=local, workspace=self.workspace)
        # in-place all-gather: the input is this rank's slice of the output buffer
        self.dist.all_gather_into_tensor(gathered.view(-1), local.view(-1), group=self.group)
        self.quick.quick_gather_columns(gathered, self.world, M, self.Nr, dst=y)
        return y


class RowParallelW4A16:
    """Y[M, N] = sum_r X[:, K_r] . dequant(Wq)[K_r, :]; input is this rank's K slice of X."""

    def __init__(self, qweight, scales, zeros, group_size: int, group=None, device=None):
        import torch
        import torch.distributed as dist
        from . import quick
        self.quick, self.dist, self.torch = quick, dist, torch
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        K = qweight.shape[0]
        self.N, self.G = scales.shape[1], group_size
        self.k0, self.k1 = row_shard_bounds(K, group_size, self.world, self.rank)
        self.Kr = self.k1 - self.k0
        qw, sc, zr = shard_awq_rows(qweight, scales, zeros, group_size, self.rank, self.world)
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.packed = torch.from_numpy(quick.quick_pack_weights(qw, sc, zr, group_size)).to(self.device)
        self._partial = {}   # internal fp32 partial per M (never returned)
        self.workspace = None

    def forward(self, x_shard, out=None):
        """A fresh output tensor per call unless `out` is given."""
        t = self.torch
        M = x_shard.shape[0]
        y = out if out is not None else t.empty((M, self.N), device=self.device, dtype=t.float16)
        if self.world == 1:
            return self.quick.quick_w4a16_gemm(x_shard, self.packed, self.N, self.Kr, self.G, out=y,
                                               workspace=self.workspace)
        if M not in self._partial:
            self._partial[M] = t.empty((M, self.N), device=self.device, dtype=t.float32)
        partial = self._partial[M]
        self.quick.quick_w4a16_gemm(x_shard, self.packed, self.N, self.Kr, self.G, out=partial, out_fp32=True,
                                    workspace=self.workspace)
        self.dist.all_reduce(partial, op=self.dist.ReduceOp.SUM, group=self.group)   # fp32 on the wire
        self.quick.quick_f32_to_f16(partial, dst=y)
        return y
