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


def shard_qkv_columns(qweight, scales, zeros, n_heads: int, n_kv_heads: int, head_dim: int, rank: int, world: int):
    """Megatron column shard of a fused QKV projection (SURVEY §8(e) semantic slicing): the AWQ
    tensors' columns are [Q heads | K heads | V heads] (n_heads, n_kv_heads, n_kv_heads heads of
    head_dim columns); rank r keeps its n_heads/P query heads and n_kv_heads/P key and value heads,
    as [q_r | k_r | v_r] (so the attention of its heads needs nothing from other ranks).
    Mistral-7B at P = 8: 4 q + 1 k + 1 v heads = 768 columns."""
    if n_heads % world or n_kv_heads % world:
        raise ValueError(f"heads ({n_heads} q, {n_kv_heads} kv) do not split over {world} ranks")
    N = scales.shape[1]
    if N != (n_heads + 2 * n_kv_heads) * head_dim:
        raise ValueError(f"N={N} != (n_heads + 2 n_kv_heads) x head_dim")
    hq, hk = n_heads // world, n_kv_heads // world
    spans = [(rank * hq * head_dim, (rank + 1) * hq * head_dim)]
    off = n_heads * head_dim
    spans.append((off + rank * hk * head_dim, off + (rank + 1) * hk * head_dim))
    off += n_kv_heads * head_dim
    spans.append((off + rank * hk * head_dim, off + (rank + 1) * hk * head_dim))
    for a, b in spans:
        if a % 8 or b % 8:
            raise ValueError("head_dim must keep shard spans on AWQ word boundaries")
    n_r = sum(b - a for a, b in spans)
    if n_r % 128:
        raise ValueError(f"per-rank QKV width {n_r} is not a multiple of 128 (v1 layout)")
    cat = np.concatenate
    return (np.ascontiguousarray(cat([qweight[:, a // 8:b // 8] for a, b in spans], axis=1)),
            np.ascontiguousarray(cat([scales[:, a:b] for a, b in spans], axis=1)),
            np.ascontiguousarray(cat([zeros[:, a // 8:b // 8] for a, b in spans], axis=1)))


def shard_gate_up(gate, up, rank: int, world: int):
    """Megatron column shard of the MLP's gate and up projections: rank r keeps the
    same I/P columns of both (its slice of the intermediate activation), packed together with
    quick_pack_gate_up so one GEMM + SiLU*mul epilogue produces that slice."""
    I = gate[1].shape[1]
    if I % (64 * world):
        raise ValueError(f"I={I} is not a multiple of 64 x world ({world}): no fused gate||up shard")
    i_r = I // world
    c0, c1 = rank * i_r, (rank + 1) * i_r

    def cut(t):
        qw, sc, zr = t
        return (np.ascontiguousarray(qw[:, c0 // 8:c1 // 8]), np.ascontiguousarray(sc[:, c0:c1]),
                np.ascontiguousarray(zr[:, c0 // 8:c1 // 8]))
    return cut(gate), cut(up)


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
        nvtx = t.cuda.nvtx   # (ranges for nsys / ncu --nvtx; no cost without a profiler)
        with nvtx.range("quick.column.gemm"):
            self.quick.quick_w4a16_gemm(x, self.packed, self.Nr, self.K, self.G, out=local, workspace=self.workspace)
        # in-place all-gather: the input is this rank's slice of the output buffer
        with nvtx.range("quick.column.all_gather"):
            self.dist.all_gather_into_tensor(gathered.view(-1), local.view(-1), group=self.group)
        with nvtx.range("quick.column.gather_columns"):
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
        nvtx = t.cuda.nvtx
        with nvtx.range("quick.row.gemm_fp32"):
            self.quick.quick_w4a16_gemm(x_shard, self.packed, self.N, self.Kr, self.G, out=partial, out_fp32=True,
                                        workspace=self.workspace)
        with nvtx.range("quick.row.all_reduce_fp32"):
            self.dist.all_reduce(partial, op=self.dist.ReduceOp.SUM, group=self.group)   # fp32 on the wire
        with nvtx.range("quick.row.to_fp16"):
            self.quick.quick_f32_to_f16(partial, dst=y)
        return y


class MegatronMLP:
    """The MLP linear stack in the Megatron split (BASELINE.json configs[4]):
    fused gate||up column-parallel GEMM with the SiLU*mul epilogue (QUICK_FLAG_SILU_MUL) producing
    this rank's I/P slice of the activation, then the row-parallel down projection (fp32 partial,
    fp32 all-reduce, cast).  No collective between the two GEMMs."""

    def __init__(self, gate, up, down, group_size: int, group=None, device=None):
        import torch
        import torch.distributed as dist
        from . import quick
        self.quick, self.torch = quick, torch
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.G, self.K = group_size, gate[0].shape[0]
        g_r, u_r = shard_gate_up(gate, up, rank, world)
        self.I_r = g_r[1].shape[1]
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.gate_up = torch.from_numpy(quick.quick_pack_gate_up(g_r, u_r, group_size)).to(self.device)
        self.down = RowParallelW4A16(*down, group_size, group=group, device=self.device)
        if self.down.Kr != self.I_r or self.down.k0 != rank * self.I_r:
            raise ValueError("down projection rows must match this rank's intermediate slice")
        self.workspace = None

    def forward(self, x, out=None):
        h = self.quick.quick_w4a16_gemm(x, self.gate_up, 2 * self.I_r, self.K, self.G,
                                        flags=self.quick.QUICK_FLAG_SILU_MUL, workspace=self.workspace)
        self.down.workspace = self.workspace
        return self.down.forward(h, out=out)


class MegatronAttentionProjections:
    """QKV column-parallel by head group (this rank's heads, no collective) and the O projection
    row-parallel over the same heads (fp32 all-reduce); attention itself is not on the hot path
    (SURVEY §8(d)), so `forward_o` takes this rank's attention output [M, n_heads/P x head_dim]."""

    def __init__(self, qkv, o, n_heads: int, n_kv_heads: int, head_dim: int, group_size: int, group=None,
                 device=None):
        import torch
        import torch.distributed as dist
        from . import quick
        self.quick = quick
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.G, self.K = group_size, qkv[0].shape[0]
        q_r = shard_qkv_columns(*qkv, n_heads, n_kv_heads, head_dim, rank, world)
        self.N_r = q_r[1].shape[1]
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.qkv = torch.from_numpy(quick.quick_pack_weights(*q_r, group_size)).to(self.device)
        self.o = RowParallelW4A16(*o, group_size, group=group, device=self.device)
        if self.o.Kr != (n_heads // world) * head_dim:
            raise ValueError("O projection rows must match this rank's query heads")
        self.workspace = None

    def forward_qkv(self, x, out=None):
        return self.quick.quick_w4a16_gemm(x, self.qkv, self.N_r, self.K, self.G, out=out, workspace=self.workspace)

    def forward_o(self, attn_r, out=None):
        self.o.workspace = self.workspace
        return self.o.forward(attn_r, out=out)


# ----------------------------------------------------------------------------------- fused (peer memory)
class _DeviceBuffer:
    """A torch view of a quick_peer_alloc'd buffer (__cuda_array_interface__; no copy)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class PeerComm:
    """Symmetric peer buffers for the collective-fused TP GEMMs: every rank allocates
    the same buffers with quick_peer_alloc, exports CUDA IPC handles, and the handles are exchanged
    over `group` (any torch.distributed backend: plumbing only); each rank then holds every rank's
    pointer.  One flag array per rank for the barriers (their epochs are counted on the device)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        from . import quick
        self.quick, self.dist, self.group = quick, dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world > 8:
            raise ValueError("at most 8 ranks per node")
        self._owned, self._imported = [], []
        self.flags = self.buffer(256)

    def buffer(self, nbytes: int):
        """Collective: one zeroed device buffer of nbytes per rank; returns every rank's pointer here."""
        local = self.quick.quick_peer_alloc(nbytes)
        self._owned.append(local)
        handles = [None] * self.world
        self.dist.all_gather_object(handles, self.quick.quick_peer_export(local), group=self.group)
        ptrs = []
        for p, h in enumerate(handles):
            if p == self.rank:
                ptrs.append(local)
            else:
                q = self.quick.quick_peer_import(h)
                self._imported.append(q)
                ptrs.append(q)
        return ptrs

    def close(self):
        import torch
        torch.cuda.synchronize()
        self.dist.barrier(group=self.group)
        for q in self._imported:
            self.quick.quick_peer_close(q)
        self.dist.barrier(group=self.group)
        for p in self._owned:
            self.quick.quick_peer_free(p)
        self._owned, self._imported = [], []


class FusedColumnParallelW4A16(ColumnParallelW4A16):
    """Column-parallel layer whose GEMM epilogue writes this rank's slice into every rank's Y over peer
    memory (quick_tp_column_gemm): no all-gather call, no gather kernel.  Y alternates between two
    symmetric buffers (a call's output stays valid until the call after next; the exit barrier of each
    call makes the reuse safe), so `forward` returns a view of the current one, shape [M][N]."""

    def __init__(self, qweight, scales, zeros, group_size: int, comm: PeerComm, max_tokens: int, device=None):
        super().__init__(qweight, scales, zeros, group_size, group=comm.group, device=device)
        self.comm, self.max_tokens = comm, max_tokens
        nbytes = max_tokens * self.N * 2
        self._y = [comm.buffer(nbytes), comm.buffer(nbytes)]
        self._turn = 0

    def forward(self, x, out=None):
        t = self.torch
        M = x.shape[0]
        if M > self.max_tokens:
            raise ValueError(f"M={M} > max_tokens={self.max_tokens}")
        ptrs = self._y[self._turn]
        self._turn ^= 1
        self.quick.quick_tp_column_gemm(x, self.packed, self.Nr, self.K, self.G, ptrs, self.N, self.comm.flags,
                                        self.comm.rank, workspace=self.workspace)
        y = t.as_tensor(_DeviceBuffer(ptrs[self.comm.rank], (M, self.N), "<f2"), device=self.device)
        if out is not None:
            out.copy_(y)
            return out
        return y


class FusedRowParallelW4A16(RowParallelW4A16):
    """Row-parallel layer with the fp32 all-reduce done over peer memory (quick_tp_row_gemm: own fp32
    partial, each rank reduces 1/P of the columns in rank order and stores fp16 into every rank's Y).
    Returns a view of the current one of two symmetric Y buffers, shape [M][N]."""

    def __init__(self, qweight, scales, zeros, group_size: int, comm: PeerComm, max_tokens: int, device=None):
        super().__init__(qweight, scales, zeros, group_size, group=comm.group, device=device)
        if self.N % (8 * comm.world):
            raise ValueError("N must be a multiple of 8 x world")
        self.comm, self.max_tokens = comm, max_tokens
        self._part = comm.buffer(max_tokens * self.N * 4)
        self._y = [comm.buffer(max_tokens * self.N * 2), comm.buffer(max_tokens * self.N * 2)]
        self._turn = 0

    def forward(self, x_shard, out=None):
        t = self.torch
        M = x_shard.shape[0]
        if M > self.max_tokens:
            raise ValueError(f"M={M} > max_tokens={self.max_tokens}")
        ptrs = self._y[self._turn]
        self._turn ^= 1
        self.quick.quick_tp_row_gemm(x_shard, self.packed, self.N, self.Kr, self.G, self._part, ptrs, self.N,
                                     self.comm.flags, self.comm.rank, workspace=self.workspace)
        y = t.as_tensor(_DeviceBuffer(ptrs[self.comm.rank], (M, self.N), "<f2"), device=self.device)
        if out is not None:
            out.copy_(y)
            return out
        return y
